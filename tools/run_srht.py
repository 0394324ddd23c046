"""Run the config-2 SRHT row sketch (fp32 2^20 x 1024 -> 4096) a few times (profiling driver)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1505_07570_b200 as rn
n, d, s = 1 << 20, 1024, 4096
A = torch.randn(n, d, device="cuda")
out = torch.empty(s, d, device="cuda")
ctx = rn.Context(0)
spec = rn.SketchSpec.srht(s, rn.derive_seed(42, 202))
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    rn.sketch_rows(A, spec, out=out, ctx=ctx)
ctx.synchronize()
print("ok")
