"""Profiling driver: count-only sketch_rows of the config-1 [A, b] (one full
cs_gather_kernel launch per call), device data. python tools/prof_count.py N."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1505_07570_b200 as rn
import workloads as wl
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
ctx = rn.Context(0)
g = torch.Generator(device="cuda"); g.manual_seed(1)
A = torch.randn(wl.CFG1["n"], wl.CFG1["d"], dtype=torch.float64, device="cuda", generator=g)
b = torch.randn(wl.CFG1["n"], dtype=torch.float64, device="cuda", generator=g)
spec = rn.SketchSpec.count_sketch(wl.CFG1["s_cs"], wl.op_seed(1))
for _ in range(reps):
    rn.sketch_rows(A, spec, extra=b, ctx=ctx)
ctx.synchronize()
print("ok")
