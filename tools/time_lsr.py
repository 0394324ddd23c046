"""Config-1-sized lsr_preconditioned (fp64 A 4,194,304 x 512, CountSketch preconditioner):
device time of the whole solve and of one fused pass A'(b - A w) (CUDA events on the
library stream). python tools/time_lsr.py [rows]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1505_07570_b200 as rn  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 22
d = 512
g = torch.Generator(device="cuda")
g.manual_seed(3)
A = torch.randn(n, d, dtype=torch.float64, device="cuda", generator=g)
xs = torch.randn(d, dtype=torch.float64, device="cuda", generator=g)
b = A @ xs + 0.01 * torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
ctx = rn.Context(0)
stream = torch.cuda.ExternalStream(ctx.stream)


def timed(fn, reps=3):
    fn()
    ctx.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        out = fn()
        e1.record(stream)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts), out


ms, sol = timed(lambda: rn.lsr_preconditioned(A, b, 1e-12, 5, want_kappa=False, ctx=ctx))
err = float(torch.linalg.norm(torch.from_numpy(sol.x).cuda() - xs) / torch.linalg.norm(xs))
passes = sol.iterations + 2  # grad_scale pass + iterations + objective pass
gb = n * d * 8 / 1e9
print(f"n={n} d={d}: solve {ms:.2f} ms, {sol.iterations} iterations, {passes} fused passes "
      f"(~{ms / passes:.3f} ms/pass incl. sketch+QR amortized), x rel err vs x* {err:.2e}")
# one fused pass alone: an iteration-budget-1 run minus the setup is noisy; time the solve at eps=0.5
ms1, sol1 = timed(lambda: rn.lsr_preconditioned(A, b, 0.5, 5, want_kappa=False, ctx=ctx))
ms2, sol2 = timed(lambda: rn.lsr_preconditioned(A, b, 0.05, 5, want_kappa=False, ctx=ctx))
per = (ms2 - ms1) / max(1, sol2.iterations - sol1.iterations)
print(f"per fused pass: {per:.3f} ms -> {gb / per * 1e3:.0f} GB/s of A ({gb:.2f} GB)")
