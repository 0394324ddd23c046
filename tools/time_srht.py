"""Device time of the config-2 SRHT row sketch (fp32 2^20 x 1024 -> 4096), CUDA events
on the library stream, median of 20 after 3 warm-ups. Env knobs pass through to the
library (RNLA_SRHT_STRIP_MB, RNLA_SRHT_NO_TMA, RNLA_SRHT_GENERIC)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1505_07570_b200 as rn  # noqa: E402

n, d, s = 1 << 20, 1024, 4096
A = torch.randn(n, d, device="cuda")
out = torch.empty(s, d, device="cuda")
ctx = rn.Context(0)
spec = rn.SketchSpec.srht(s, rn.derive_seed(42, 202))
stream = torch.cuda.ExternalStream(ctx.stream)
for _ in range(3):
    rn.sketch_rows(A, spec, out=out, ctx=ctx)
ctx.synchronize()
ts = []
for _ in range(20):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    rn.sketch_rows(A, spec, out=out, ctx=ctx)
    e1.record(stream)
    e1.synchronize()
    ts.append(e0.elapsed_time(e1))
ts.sort()
ms = ts[len(ts) // 2]
print(f"strip_mb={os.environ.get('RNLA_SRHT_STRIP_MB', 'default')} median_ms={ms:.3f} best_ms={ts[0]:.3f} "
      f"GB/s={(n * d * 4 + s * d * 4) / ms / 1e6:.0f}")
