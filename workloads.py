"""workloads.py -- the five BASELINE.json configurations as seeded synthetic data.

Shared by bench.py (both arms), bench_configs.py and the full-size parity
tests (tests/test_gpu_fullsize.py), so the GPU path, the CPU oracle and the
reference CPU arm consume identical bytes. No public dataset is involved
(SURVEY §8(d)); seeds follow the survey's convention:

  data seed      D_c = derive_seed(42, 100 + c)
  operator seed  O_c = derive_seed(42, 200 + c)

Configs 0 and 1 are generated on the host with numpy (config 1 in fixed
65536-row blocks on a thread pool, so the bytes do not depend on the thread
count); configs 2-4 are generated on the GPU with torch's seeded Philox
generator (config 3 needs 17.6 TFLOP to form U diag(sigma) V^T, far too slow
on a CPU, as SURVEY §8(d) allows) and copied to the host where the oracle needs
them.
"""
from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

MASK64 = (1 << 64) - 1


def derive_seed(seed: int, stream: int) -> int:
    """include/randnla/rng.hpp:21-24 (splitmix64 of seed ^ (golden + stream * phi))."""
    s = seed ^ ((0x6A09E667F3BCC909 + stream * 0x9E3779B97F4A7C15) & MASK64)
    z = (s + 0x9E3779B97F4A7C15) & MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


MASTER_SEED = 42


def data_seed(c: int) -> int:
    return derive_seed(MASTER_SEED, 100 + c)


def op_seed(c: int) -> int:
    return derive_seed(MASTER_SEED, 200 + c)


# ---- shapes and parameters (BASELINE.json configs[0..4]) -------------------
CFG0 = dict(m=8192, n=2048, k=20, s=30, q=1)
CFG1 = dict(n=4_194_304, d=512, s_cs=8192, s=2048)
CFG2 = dict(n=1 << 20, d=1024, s=4096)
CFG3 = dict(m=262_144, n=16_384, r=2048, k=100, s=150, q=2)
CFG4 = dict(n=131_072, d=64, c=2048, k=64, comps=16, sub=4096)

BLOCK = 65536  # config-1 generation block (rows)


def host_threads() -> int:
    return max(1, os.cpu_count() or 1)


def cfg0_host() -> np.ndarray:
    """fp64 A = U diag(sigma) V^T + 1e-3 N(0,1), 8192 x 2048; U, V = Q of seeded
    Gaussians (cf. src/acceptance.cpp:151-158); sigma_i = exp(-i/20), i = 1..2048."""
    m, n = CFG0["m"], CFG0["n"]
    g = np.random.default_rng(data_seed(0))
    u, _ = np.linalg.qr(g.standard_normal((m, n)))
    v, _ = np.linalg.qr(g.standard_normal((n, n)))
    sig = np.exp(-np.arange(1, n + 1) / 20.0)
    return np.ascontiguousarray((u * sig) @ v.T + 1e-3 * g.standard_normal((m, n)))


def cfg1_host(n: int = CFG1["n"], threads: int = 0, r0: int = 0, r1: int = -1, out_a=None, out_b=None):
    """fp64 A (n x 512) i.i.d. N(0,1), b = A x* + 0.01 N(0,1), x* ~ N(0,1)^512.
    Row block i (65536 rows) is drawn from child i of SeedSequence(D_1), so the
    bytes do not depend on the thread count, and rows [r0, r1) (a rank's shard)
    can be generated alone; smaller n gives the first n rows of the
    4,194,304-row matrix. out_a / out_b (e.g. pinned host memory) receive rows
    [r0, r1). Returns (A[r0:r1], b[r0:r1], x*)."""
    d = CFG1["d"]
    r1 = n if r1 < 0 else r1
    kids = np.random.SeedSequence(data_seed(1)).spawn(max(n, CFG1["n"]) // BLOCK + 2)
    xstar = np.random.default_rng(kids[-1]).standard_normal(d)
    a = np.empty((r1 - r0, d)) if out_a is None else out_a
    b = np.empty(r1 - r0) if out_b is None else out_b

    def fill(i):
        lo, hi = max(r0, i * BLOCK), min(r1, (i + 1) * BLOCK)
        g = np.random.default_rng(kids[i])
        blk = g.standard_normal((BLOCK, d))[lo - i * BLOCK: hi - i * BLOCK]
        noise = g.standard_normal(BLOCK)[lo - i * BLOCK: hi - i * BLOCK]
        a[lo - r0: hi - r0] = blk
        b[lo - r0: hi - r0] = blk @ xstar + 0.01 * noise

    try:
        from threadpoolctl import threadpool_limits
        lim = threadpool_limits(limits=1)
    except Exception:  # pragma: no cover
        lim = None
    try:
        with ThreadPoolExecutor(threads or host_threads()) as ex:
            list(ex.map(fill, range(r0 // BLOCK, (r1 + BLOCK - 1) // BLOCK)))
    finally:
        if lim is not None:
            lim.unregister()
    return a, b, xstar


def _gen(seed: int, device):
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed & 0x7FFFFFFFFFFFFFFF)
    return g


def cfg2_device(device="cuda", n: int = CFG2["n"]):
    """fp32 A (2^20 x 1024), i.i.d. Student-t nu = 3 (= N / sqrt(chi2_3 / 3))."""
    import torch
    d = CFG2["d"]
    g = _gen(data_seed(2), device)
    a = torch.empty(n, d, dtype=torch.float32, device=device)
    step = 1 << 16
    for r0 in range(0, n, step):  # bounded temporaries
        r1 = min(n, r0 + step)
        z = torch.randn(r1 - r0, d, device=device, generator=g)
        chi = (torch.randn(r1 - r0, d, 3, device=device, generator=g) ** 2).sum(-1) / 3.0
        a[r0:r1] = z / torch.sqrt(chi)
    return a


def cfg3_device(device="cuda"):
    """fp32 A (262144 x 16384) = U diag(i^-1.5) V^T + 1e-4 N(0,1); the signal is
    truncated at rank r = 2048 (sigma_r ~ 1e-5, far below the noise edge ~0.064;
    SURVEY §8(d)). U, V = Q of seeded Gaussians."""
    import torch
    m, n, r = CFG3["m"], CFG3["n"], CFG3["r"]
    g = _gen(data_seed(3), device)
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        u, _ = torch.linalg.qr(torch.randn(m, r, device=device, generator=g))
        v, _ = torch.linalg.qr(torch.randn(n, r, device=device, generator=g))
        sig = torch.arange(1, r + 1, dtype=torch.float32, device=device) ** -1.5
        a = (u * sig) @ v.T
        del u, v
        step = 1 << 15
        for r0 in range(0, m, step):
            a[r0:r0 + step] += 1e-4 * torch.randn(min(step, m - r0), n, device=device, generator=g)
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    return a


def cfg4_sigma(x: np.ndarray) -> float:
    """Median pairwise distance over a 4096-point subsample (fp64, host, numpy
    median convention), subsample = sample_without_replacement(n, 4096,
    derive_seed(O_4, 3)) restated with the oracle's libstdc++ draw."""
    from oracle import oracle as orc
    sub = x[orc.sample_without_replacement(x.shape[0], CFG4["sub"], derive_seed(op_seed(4), 3))].astype(np.float64)
    sq = np.einsum("ij,ij->i", sub, sub)
    d2 = np.maximum(sq[:, None] + sq[None, :] - 2.0 * (sub @ sub.T), 0.0)
    iu = np.triu_indices(sub.shape[0], 1)
    return float(np.median(np.sqrt(d2[iu])))


def cfg4_device(device="cuda"):
    """fp32 X (131072 x 64) from a seeded 16-component Gaussian mixture (equal
    weights, unit-variance components, means ~ N(0, 9 I)). Returns (X, sigma)."""
    import torch
    n, d, comps = CFG4["n"], CFG4["d"], CFG4["comps"]
    g = _gen(data_seed(4), device)
    means = 3.0 * torch.randn(comps, d, device=device, generator=g)
    lab = torch.randint(0, comps, (n,), device=device, generator=g)
    x = (means[lab] + torch.randn(n, d, device=device, generator=g)).float().contiguous()
    return x, cfg4_sigma(x.cpu().numpy())


def nystrom_oracle_lambda(x: np.ndarray, sigma: float, c: int, seed: int, k: int, threads: int = 0):
    """Oracle for config 4: nystrom(KernelView(x, sigma), c, seed, target_k = c)
    (src/spsd.cpp:181-222) then approx_eig(L, k) (src/spsd.cpp:257-265), in fp64.
    approx_eig's condensed_svd is evaluated for its singular values only
    (lambda = sigma^2); returns (lambda[k], selected, kept)."""
    from oracle import oracle as orc
    l, sel, lk = orc.nystrom(x, sigma, c, seed, c)
    sv = np.linalg.svd(l, compute_uv=False)
    return sv[:k] ** 2, sel, lk.size
