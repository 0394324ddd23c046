"""Config-2 leverage scores: time (median of 5) and max relative error vs the fp64 oracle
scores on the full 2^20 x 1024 cfg2 data (RNLA_LIB_PATH selects a library build)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import scipy.linalg as sla
import paper_1505_07570_b200 as rn
import workloads as wl
from oracle import oracle as orc
A = wl.cfg2_device()
ctx = rn.Context(0)
seed = orc.derive_seed(wl.op_seed(2), 2)
stream = torch.cuda.ExternalStream(ctx.stream)
for _ in range(2):
    scores, idx = rn.leverage_sample_rows(A, 4096, seed, ctx=ctx)
ts = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream); scores, idx = rn.leverage_sample_rows(A, 4096, seed, ctx=ctx); e1.record(stream); e1.synchronize()
    ts.append(e0.elapsed_time(e1))
a64 = A.double().cpu().numpy()
r = np.linalg.cholesky(a64.T @ a64).T
ref = np.einsum("ij,ij->i", *(2 * [sla.solve_triangular(r, a64.T, trans="T", lower=False).T]))
rel = np.abs(scores - ref) / ref
print(f"lib={os.environ.get('RNLA_LIB_PATH','default')} ms={sorted(ts)[2]:.3f} max_rel={rel.max():.3e} mean_rel={rel.mean():.3e}")
