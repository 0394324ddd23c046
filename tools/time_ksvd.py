"""Device time of prototype_ksvd fp32: python tools/time_ksvd.py m n k s q"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1505_07570_b200 as rn
m, n, k, s, q = (int(v) for v in sys.argv[1:6])
g = torch.Generator(device="cuda"); g.manual_seed(5)
A = torch.randn(m, n, device="cuda", generator=g)
ctx = rn.Context(0)
stream = torch.cuda.ExternalStream(ctx.stream)
for _ in range(2):
    r = rn.prototype_ksvd(A, k, s, 3, power_iters=q, ctx=ctx)
ctx.synchronize()
ts = []
for _ in range(7):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream); r = rn.prototype_ksvd(A, k, s, 3, power_iters=q, ctx=ctx); e1.record(stream); e1.synchronize()
    ts.append(e0.elapsed_time(e1))
ts.sort()
print(f"ksvd {m}x{n} k={k} s={s} q={q} NO_TS={os.environ.get('RNLA_TC_NO_TS')}: median {ts[3]:.3f} ms best {ts[0]:.3f} ms sigma1 {r.factors.singular_values[0]:.6f}")
