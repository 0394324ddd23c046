"""Run one tcgen05 GEMM shape through gaussian_sketch (fp32): python tools/dbg_tc.py m n s order.
Prints the device time and the rel-F error against a torch fp64 reference on a column subset."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1505_07570_b200 as rn  # noqa: E402

m, n, s = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
order = sys.argv[4] if len(sys.argv) > 4 else "C"
g = torch.Generator(device="cuda")
g.manual_seed(1)
A = torch.randn(m, n, device="cuda", generator=g)
if order == "F":
    A = A.t().contiguous().t()
ctx = rn.Context(0)
t0 = time.time()
C = rn.gaussian_sketch(A, s, 7, ctx=ctx)
ctx.synchronize()
t1 = time.time()
G = torch.from_numpy(rn.gaussian_matrix(n, s, 7)).cuda() / s ** 0.5
rows = slice(0, min(m, 4096))
ref = A[rows].double() @ G
err = float(torch.linalg.norm(C[rows].double() - ref) / torch.linalg.norm(ref))
print(f"m={m} n={n} s={s} {order}: {1e3 * (t1 - t0):.1f} ms wall, rel-F {err:.2e}", flush=True)
