"""A-in-TMEM tcgen05 GEMM check: prototype_ksvd (fp32) through the default path vs RNLA_TC_NO_TS=1 in a child
process: python tools/ts_check.py m n s q [order]"""
import os, subprocess, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if os.environ.get("TS_CHILD"):
    import torch
    import paper_1505_07570_b200 as rn
    m, n, s, q = (int(v) for v in sys.argv[1:5])
    order = sys.argv[5] if len(sys.argv) > 5 else "C"
    g = torch.Generator(device="cuda"); g.manual_seed(3)
    A = torch.randn(m, n, device="cuda", generator=g)
    if order == "F":
        A = A.t().contiguous().t()
    ctx = rn.Context(0)
    res = rn.prototype_ksvd(A, min(100, s - 10), s, 5, power_iters=q, ctx=ctx)
    sv = res.factors.singular_values if hasattr(res.factors, "singular_values") else res.factors[1]
    print("SV " + json.dumps([float(v) for v in sv[:8]]), flush=True)
else:
    outs = []
    for env in ({},) if os.environ.get("TS_ONLY") else ({}, {"RNLA_TC_NO_TS": "1"}):
        e = dict(os.environ, TS_CHILD="1", **env)
        try:
            p = subprocess.run([sys.executable, __file__] + sys.argv[1:], env=e, capture_output=True, text=True,
                               timeout=float(os.environ.get("TS_TIMEOUT", "120")))
            line = [l for l in p.stdout.splitlines() if l.startswith("SV ")]
            outs.append((line[0] if line else "FAIL ") + " || " + " | ".join(l for l in p.stderr.strip().splitlines() if l.startswith("[ts]") or "Error" in l)[:1500])
        except subprocess.TimeoutExpired as ex:
            err = ex.stderr.decode() if isinstance(ex.stderr, bytes) else (ex.stderr or "")
            outs.append("TIMEOUT " + " | ".join(err.strip().splitlines()[-4:])[:600])
    print(sys.argv[1:], "TS   :", outs[0])
    if len(outs) > 1:
        print(sys.argv[1:], "NO_TS:", outs[1], flush=True)
