"""prototype_ksvd fp32 at one shape (debug ladder): python tools/dbg_ksvd.py m n k s q"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1505_07570_b200 as rn  # noqa: E402

m, n, k, s, q = (int(v) for v in sys.argv[1:6])
g = torch.Generator(device="cuda")
g.manual_seed(1)
A = torch.randn(m, n, device="cuda", generator=g)
ctx = rn.Context(0)
t0 = time.time()
r = rn.prototype_ksvd(A, k, s, 5, power_iters=q, ctx=ctx)
ctx.synchronize()
print(f"m={m} n={n} k={k} s={s} q={q}: {1e3 * (time.time() - t0):.1f} ms, sigma0 {r.factors.singular_values[0]:.6g}",
      flush=True)
