"""Device time of the config-2 leverage-score row sampling (fp32 2^20 x 1024, p = 4096):
Gram in fp64, Cholesky, scores = row norms of M R^-1, host draw. CUDA events on the
library stream, median of 5 after 2 warm-ups. RNLA_TRACE=1 prints the stage split."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1505_07570_b200 as rn  # noqa: E402

n, d, s = 1 << 20, 1024, 4096
g = torch.Generator(device="cuda")
g.manual_seed(2)
A = torch.randn(n, d, device="cuda", generator=g)
ctx = rn.Context(0)
stream = torch.cuda.ExternalStream(ctx.stream)
seed = rn.derive_seed(rn.derive_seed(42, 202), 2)
for _ in range(2):
    rn.leverage_sample_rows(A, s, seed, ctx=ctx)
ctx.synchronize()
ts = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    rn.leverage_sample_rows(A, s, seed, ctx=ctx)
    e1.record(stream)
    e1.synchronize()
    ts.append(e0.elapsed_time(e1))
ts.sort()
print(f"leverage rows median_ms={ts[len(ts) // 2]:.3f} best_ms={ts[0]:.3f}")
