"""Diagnostic: relative Frobenius error of fp32 GEMMs (tcgen05 BF16x3 vs SIMT) against fp64."""
import os, sys, math
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1505_07570_b200 as rn
ctx = rn.Context(0)
g = torch.Generator(device="cuda"); g.manual_seed(3)
for (m, n, s) in [(4096, 16384, 150), (4096, 2048, 150), (65536, 16384, 150)]:
    A = torch.randn(m, n, device="cuda", generator=g)
    # low-rank + noise like cfg3
    C = rn.gaussian_sketch(A, s, 11, ctx=ctx)
    Om = torch.from_numpy(rn.gaussian_matrix(n, s, 11) / math.sqrt(s)).cuda()
    ref = A.double() @ Om
    err = (C.double() - ref).norm() / ref.norm()
    print(f"A.Omega m={m} n={n} s={s}: rel-F err {err.item():.3e}", flush=True)
