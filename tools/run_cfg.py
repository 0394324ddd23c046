"""Run one BASELINE config's timed operation N times (profiling driver): python tools/run_cfg.py CFG [N]."""
import os, sys, math
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1505_07570_b200 as rn
cfg = int(sys.argv[1]); reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
ctx = rn.Context(0)
g = torch.Generator(device="cuda"); g.manual_seed(7)
if cfg == 0:
    A = torch.randn(8192, 2048, dtype=torch.float64, device="cuda", generator=g)
    fn = lambda: rn.prototype_ksvd(A, 20, 30, 5, power_iters=1, ctx=ctx)
elif cfg == 3:
    A = torch.randn(262144, 16384, device="cuda", generator=g)
    fn = lambda: rn.prototype_ksvd(A, 100, 150, 5, power_iters=2, ctx=ctx)
elif cfg == 4:
    X = (torch.randn(131072, 64, device="cuda", generator=g) * 3).contiguous()
    view = rn.KernelView(X, rn.KernelSpec(35.0))
    fn = lambda: rn.nystrom_eig(view, 2048, 5, 2048, 64, want_vectors=False, ctx=ctx)
elif cfg == 2:
    A = torch.randn(1 << 20, 1024, device="cuda", generator=g)
    fn = lambda: rn.leverage_sample_rows(A, 4096, 9, ctx=ctx)
for _ in range(reps):
    fn()
ctx.synchronize()
print("ok")
