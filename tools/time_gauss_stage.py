"""Device time of the fp64 Gaussian stage alone (config-1 shape: 8192 x 513 -> 2048),
CUDA events on the library stream, median of 20 after 3 warm-ups; RNLA_GAUSS_DMMA=1
selects the DMMA path. Also prints the rel-F difference between the two paths' results
when run with --compare."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1505_07570_b200 as rn
g = torch.Generator(device="cuda"); g.manual_seed(3)
C = (torch.randn(8192, 513, dtype=torch.float64, device="cuda", generator=g) * 22.6).contiguous()
ctx = rn.Context(0)
spec = rn.SketchSpec.gaussian(2048, rn.derive_seed(rn.derive_seed(42, 201), 1))
out = torch.empty(2048, 513, dtype=torch.float64, device="cuda")
stream = torch.cuda.ExternalStream(ctx.stream)
for _ in range(3):
    rn.sketch_rows(C, spec, out=out, ctx=ctx)
ctx.synchronize()
ts = []
for _ in range(20):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream); rn.sketch_rows(C, spec, out=out, ctx=ctx); e1.record(stream); e1.synchronize()
    ts.append(e0.elapsed_time(e1))
ts.sort()
print(f"gauss stage {os.environ.get('RNLA_GAUSS_DMMA') and 'dmma' or 'ozaki'}: median {ts[10]*1e3:.1f} us best {ts[0]*1e3:.1f} us")
if "--compare" in sys.argv:
    ref = C.T.contiguous()  # placeholder to keep shapes obvious
    G = torch.from_numpy(rn.gaussian_matrix(8192, 2048, spec.seed)).cuda() / (2048 ** 0.5)
    exact = G.T @ C
    print("rel-F vs torch fp64:", float(torch.linalg.norm(out - exact) / torch.linalg.norm(exact)))
