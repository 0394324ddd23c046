#!/usr/bin/env python
"""bench_configs.py -- per-config measurements for BASELINE configs 0, 2, 3, 4
(config 1 is bench.py's headline). One JSON line per config: device time
(CUDA events on the library stream, median of --reps after --warmup), the
binding roofline, and a parity check at full size against an independent
reference of the same algorithm on identical operators.

  cfg0  prototype_ksvd fp64 8192x2048, k=20, s=30, q=1           (oracle: numpy fp64)
  cfg2  SRHT fp32 2^20 x 1024 -> 4096 rows; leverage rows, p=4096  (oracle: C loop on a column subset;
                                                                   scores vs numpy fp64 on a row subset's basis)
  cfg3  prototype_ksvd fp32 262144x16384, k=100, s=150, q=2      (cross-check: same algorithm in torch fp64)
  cfg4  Nystrom + top-64 eig, fp32 n=131072, d=64, c=2048         (oracle: numpy fp64 Gram route)

Synthetic data is seeded and generated on the device (no dataset is
involved); operator seeds follow SURVEY §8(d): O_c = derive_seed(42, 200+c).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1505_07570_b200 as rn  # noqa: E402

HBM = 6542.7e9
F64_TF = 35.5e12       # cuBLAS DGEMM on this pool (profiles/peaks_r01.json)
BF16X3_TF = 1652.9e12 / 3


def op_seed(c):
    return rn.derive_seed(42, 200 + c)


def data_seed(c):
    return rn.derive_seed(42, 100 + c) & 0x7FFFFFFFFFFFFFFF


def timed(ctx, fn, warmup, reps):
    stream = torch.cuda.ExternalStream(ctx.stream)
    for _ in range(warmup):
        fn()
    ctx.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        out = fn()
        e1.record(stream)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts)), float(np.min(ts)), out


def gen(seed):
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    return g


def cfg0(ctx, args):
    m, n, k, s, q = 8192, 2048, 20, 30, 1
    g = gen(data_seed(0))
    U, _ = torch.linalg.qr(torch.randn(m, n, dtype=torch.float64, device="cuda", generator=g))
    V, _ = torch.linalg.qr(torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g))
    sig = torch.exp(-torch.arange(1, n + 1, dtype=torch.float64, device="cuda") / 20.0)
    A = (U * sig) @ V.T + 1e-3 * torch.randn(m, n, dtype=torch.float64, device="cuda", generator=g)
    del U, V
    med, best, r = timed(ctx, lambda: rn.prototype_ksvd(A, k, s, op_seed(0), power_iters=q, ctx=ctx),
                         args.warmup, args.reps)
    from oracle import oracle as orc
    a = A.cpu().numpy()
    _, so, _, _ = orc.prototype_ksvd(a, k, s, op_seed(0), q=q)
    err = float(np.max(np.abs(r.factors.singular_values - so) / so))
    exact = np.linalg.svd(a, compute_uv=False)[:k]
    B, F = 4 * m * n * 8, 4 * 2 * m * n * s
    t_roof = max(B / HBM, F / F64_TF)
    return {"config": "cfg0 prototype_ksvd fp64 8192x2048 k=20 s=30 q=1", "ms_median": med, "ms_best": best,
            "roofline_ms": t_roof * 1e3, "frac_of_roofline": t_roof * 1e3 / med, "binding": "hbm~dmma",
            "alg_bytes": B, "alg_flops": F, "passes": r.passes_over_a,
            "parity": {"sigma_max_rel_err_vs_oracle": err, "gate": 1e-8, "pass": err <= 1e-8},
            "info_rel_err_vs_exact_svd": float(np.max(np.abs(r.factors.singular_values - exact) / exact))}


def cfg2(ctx, args):
    n, d, s = 1 << 20, 1024, 4096
    g = gen(data_seed(2))
    # Student-t(3) = N / sqrt(chi2_3 / 3), seeded on the device
    z = torch.randn(n, d, device="cuda", generator=g)
    chi = (torch.randn(n, d, 3, device="cuda", generator=g) ** 2).sum(-1) / 3.0
    A = (z / torch.sqrt(chi)).float().contiguous()
    del z, chi
    spec = rn.SketchSpec.srht(s, op_seed(2))
    out = torch.empty(s, d, dtype=torch.float32, device="cuda")
    med, best, _ = timed(ctx, lambda: rn.sketch_rows(A, spec, out=out, ctx=ctx), args.warmup, args.reps)
    from oracle import oracle as orc
    cols = list(range(0, d, d // 8))  # parity on 8 of the 1024 columns at full n (fp64 C loop)
    sub = A[:, cols].double().cpu().numpy()
    ref = orc.srht_rows(sub, s, op_seed(2))
    got = out[:, cols].double().cpu().numpy()
    err = float(np.linalg.norm(got - ref) / np.linalg.norm(ref))
    B = n * d * 4 + s * d * 4
    res = {"config": "cfg2 SRHT fp32 2^20x1024 -> 4096", "ms_median": med, "ms_best": best,
           "roofline_ms": B / HBM * 1e3, "frac_of_roofline": B / HBM * 1e3 / med, "binding": "hbm",
           "alg_bytes": B, "achieved_gbs": B / (med * 1e-3) / 1e9,
           "parity": {"rel_fro_err_8cols_vs_oracle": err, "gate": 1e-4, "pass": err <= 1e-4}}
    # leverage-score rows from the orthonormal basis
    medl, bestl, lv = timed(ctx, lambda: rn.leverage_sample_rows(A, s, rn.derive_seed(op_seed(2), 2), ctx=ctx),
                            max(1, args.warmup // 2), max(1, args.reps // 4))
    scores, idx = lv
    draws = np.unique(orc.sample_with_replacement(scores, s, rn.derive_seed(op_seed(2), 2)))
    F = 2 * n * d * d * 2
    res["leverage"] = {"ms_median": medl, "ms_best": bestl, "alg_flops": F,
                       "roofline_ms_bf16x3": F / BF16X3_TF * 1e3, "frac_of_roofline": F / BF16X3_TF * 1e3 / medl,
                       "scores_sum": float(scores.sum()), "scores_sum_expected": d,
                       "indices": int(idx.size), "indices_bit_exact_given_scores": bool(np.array_equal(idx, draws))}
    return res


def cfg3(ctx, args):
    m, n, r, k, s, q = 262144, 16384, 2048, 100, 150, 2
    g = gen(data_seed(3))
    U, _ = torch.linalg.qr(torch.randn(m, r, device="cuda", generator=g))
    V, _ = torch.linalg.qr(torch.randn(n, r, device="cuda", generator=g))
    sig = torch.arange(1, r + 1, dtype=torch.float32, device="cuda") ** -1.5
    torch.backends.cuda.matmul.allow_tf32 = False
    A = (U * sig) @ V.T
    del U, V
    A += 1e-4 * torch.randn(m, n, device="cuda", generator=g)
    med, best, res = timed(ctx, lambda: rn.prototype_ksvd(A, k, s, op_seed(3), power_iters=q, ctx=ctx),
                           args.warmup, args.reps)
    # cross-check: the same algorithm on the same Omega in torch fp64 (cuBLAS), independent of our kernels
    Om = torch.from_numpy(rn.gaussian_matrix(n, s, op_seed(3)) / math.sqrt(s)).cuda()
    A64 = A.double()

    def orth(y):
        qq, _ = torch.linalg.qr(y)
        return qq
    Y = A64 @ Om
    for _ in range(q):
        Qy = orth(Y)
        Z = orth(A64.T @ Qy)
        Y = A64 @ Z
    Qy = orth(Y)
    sv = torch.linalg.svdvals(Qy.T @ A64)[:k].cpu().numpy()
    del A64, Y, Qy
    err = float(np.max(np.abs(res.factors.singular_values - sv) / sv))
    B, F = 6 * m * n * 4, 6 * 2 * m * n * s
    t_roof = max(B / HBM, F / BF16X3_TF)
    return {"config": "cfg3 prototype_ksvd fp32 262144x16384 k=100 s=150 q=2", "ms_median": med, "ms_best": best,
            "roofline_ms": t_roof * 1e3, "frac_of_roofline": t_roof * 1e3 / med, "binding": "hbm (75 flop/B)",
            "alg_bytes": B, "alg_flops": F, "passes": res.passes_over_a,
            "parity": {"sigma_max_rel_err_vs_torch_fp64_same_omega": err, "gate": 1e-3, "pass": err <= 1e-3}}


def cfg4(ctx, args):
    n, d, c, k, comps = 131072, 64, 2048, 64, 16
    g = gen(data_seed(4))
    means = 3.0 * torch.randn(comps, d, device="cuda", generator=g)
    lab = torch.randint(0, comps, (n,), device="cuda", generator=g)
    X = (means[lab] + torch.randn(n, d, device="cuda", generator=g)).float().contiguous()
    sub = X[torch.from_numpy(rn.sample_without_replacement(n, 4096, rn.derive_seed(op_seed(4), 3))).cuda()].double()
    dd = torch.cdist(sub, sub)
    iu = torch.triu_indices(4096, 4096, 1, device="cuda")
    sigma = float(torch.median(dd[iu[0], iu[1]]).item())
    view = rn.KernelView(X, rn.KernelSpec(sigma))
    med, best, out = timed(ctx, lambda: rn.nystrom_eig(view, c, op_seed(4), c, k, want_vectors=False, ctx=ctx),
                           args.warmup, args.reps)
    _, lam, sel, kept = out
    # oracle: numpy fp64 Gram route on the same landmarks
    from oracle import oracle as orc
    x = X.double().cpu().numpy()
    C = orc.rbf_kernel(x, x[sel], sigma)
    C[sel, np.arange(c)] = 1.0
    W = C[sel]
    lw, vw = np.linalg.eigh(0.5 * (W + W.T))
    floor = np.finfo(np.float64).eps * lw[-1] * n
    kp = 0
    while kp < c and lw[c - 1 - kp] > floor:
        kp += 1
    T = vw[:, ::-1][:, :kp] / np.sqrt(lw[::-1][:kp])
    M = T.T @ (C.T @ C) @ T
    lo = np.linalg.eigvalsh(0.5 * (M + M.T))[::-1][:k]
    err = float(np.max(np.abs(lam - lo) / lo))
    F = 2 * n * c * d + 2 * n * c * c + 2 * n * c * k
    return {"config": "cfg4 Nystrom fp32 n=131072 d=64 c=2048 top-64", "sigma": sigma, "kept": kept,
            "kept_oracle": kp, "ms_median": med, "ms_best": best, "alg_flops": F,
            "roofline_ms_bf16x3": F / BF16X3_TF * 1e3, "frac_of_roofline": F / BF16X3_TF * 1e3 / med,
            "parity": {"lambda_max_rel_err_vs_oracle": err, "gate": 1e-3, "pass": err <= 1e-3}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="0,2,3,4")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    ctx = rn.Context(0)
    for c in [int(x) for x in args.configs.split(",")]:
        t0 = time.time()
        res = {0: cfg0, 2: cfg2, 3: cfg3, 4: cfg4}[c](ctx, args)
        res["wall_s"] = round(time.time() - t0, 1)
        print(json.dumps(res), flush=True)
        torch.cuda.empty_cache()
    ctx.close()


if __name__ == "__main__":
    main()
