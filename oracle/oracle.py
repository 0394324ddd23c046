"""TEST INFRASTRUCTURE ONLY -- CPU oracle for the randnla hot path.

Restates the reference algorithms (/root/reference/proj, C++ + Eigen, which
cannot be built here: Eigen3 is absent) so the CUDA library can
be checked on identical inputs and identical random operators:

* operator draws, hashes and the streaming sketches come from the plain-C
  restatement in rnla_oracle.c (pinned against real libstdc++ output in
  tests/golden/libstdcxx_streams.json);
* dense linear algebra is numpy/LAPACK (geqrf/gesdd/syevd in place of Eigen's
  HouseholderQR/BDCSVD/SelfAdjointEigenSolver) with the reference's sign and
  rank conventions. Differences against Eigen are rounding-level.

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may import this
module. The product library never calls it.

Parity status: RNG streams, hashes, count sketch (bit-exact sequential
order), SRHT and FWHT are pinned by golden vectors / known answers AND by
fixtures the reference's own src/rng.cpp + src/sketch.cpp produced when
compiled here unmodified against oracle/ref_shim (tests/golden/
ref_fixtures.json, tests/test_ref_fixtures.py); the power
iteration extension (configs 0/3) is parity-unpinned by reference tests
(the reference has no power iteration, src/randsvd.cpp:88-110).
"""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "librnla_oracle.so")
_lib = None

_I64P = C.POINTER(C.c_int64)
_F64P = C.POINTER(C.c_double)


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE, "all"], check=True)
    return _SO


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            build()
        L = C.CDLL(_SO)
        L.orc_splitmix64.restype = C.c_uint64
        L.orc_splitmix64.argtypes = [C.POINTER(C.c_uint64)]
        L.orc_derive_seed.restype = C.c_uint64
        L.orc_derive_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_count_sketch_hashes.argtypes = [C.c_uint64, C.c_int64, C.c_int64, C.c_int64, _I64P, _F64P]
        L.orc_gaussian_matrix.argtypes = [C.c_uint64, C.c_int64, C.c_int64, _F64P]
        L.orc_sample_without_replacement.argtypes = [C.c_uint64, C.c_int64, C.c_int64, _I64P]
        L.orc_sample_with_replacement.argtypes = [C.c_uint64, _F64P, C.c_int64, C.c_int64, _I64P]
        L.orc_srht_operator.argtypes = [C.c_uint64, C.c_int64, C.c_int64, _F64P, _I64P]
        L.orc_count_sketch.argtypes = [_F64P, _F64P, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_uint64,
                                       C.c_int64, _F64P]
        L.orc_count_sketch_mt.argtypes = [_F64P, _F64P, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_uint64,
                                          C.c_int64, _F64P, C.c_int]
        L.orc_count_sketch_mt.restype = C.c_int
        L.orc_fwht.argtypes = [_F64P, C.c_int64]
        L.orc_srht_sketch.argtypes = [_F64P, C.c_int64, C.c_int64, C.c_int64, C.c_int64, _F64P, _I64P, _F64P]
        L.orc_srht_sketch_mt.argtypes = [_F64P, C.c_int64, C.c_int64, C.c_int64, C.c_int64, _F64P, _I64P, _F64P,
                                         C.c_int]
        L.orc_srht_sketch_mt.restype = C.c_int
        L.orc_mt_next.restype = C.c_uint64
        _lib = L
    return _lib


class MT64(C.Structure):
    _fields_ = [("x", C.c_uint64 * 312), ("i", C.c_int)]


def mt64_stream(seed: int, count: int) -> list:
    L = lib()
    g = MT64()
    L.orc_mt_seed.argtypes = [C.POINTER(MT64), C.c_uint64]
    L.orc_mt_next.argtypes = [C.POINTER(MT64)]
    L.orc_mt_seed(C.byref(g), seed)
    return [int(L.orc_mt_next(C.byref(g))) for _ in range(count)]


class _Normal(C.Structure):
    _fields_ = [("saved", C.c_double), ("has_saved", C.c_int)]


class Engine:
    """A std::mt19937_64 whose state carries over between draws, for
    restating reference call sequences on one Rng (src/rng.cpp:8-65)."""

    def __init__(self, seed: int):
        L = lib()
        L.orc_mt_seed.argtypes = [C.POINTER(MT64), C.c_uint64]
        L.orc_mt_next.argtypes = [C.POINTER(MT64)]
        L.orc_normal_next.argtypes = [C.POINTER(_Normal), C.POINTER(MT64)]
        L.orc_normal_next.restype = C.c_double
        L.orc_uniform_real.argtypes = [C.POINTER(MT64), C.c_double, C.c_double]
        L.orc_uniform_real.restype = C.c_double
        L.orc_sample_without_replacement_g.argtypes = [C.POINTER(MT64), C.c_int64, C.c_int64, _I64P]
        self.g = MT64()
        L.orc_mt_seed(C.byref(self.g), seed)

    def gaussian_matrix(self, rows: int, cols: int) -> np.ndarray:
        nd = _Normal(0.0, 0)  # a fresh normal_distribution per call (rng.cpp:9)
        out = np.empty((rows, cols), order="F")
        for j in range(cols):
            for i in range(rows):
                out[i, j] = lib().orc_normal_next(C.byref(nd), C.byref(self.g))
        return out

    def gaussian_unit_vector(self, dim: int) -> np.ndarray:
        nd = _Normal(0.0, 0)
        while True:
            v = np.array([lib().orc_normal_next(C.byref(nd), C.byref(self.g)) for _ in range(dim)])
            n2 = 0.0
            for x in v:
                n2 += x * x
            if n2 != 0.0:
                return v / math.sqrt(n2)

    def sample_without_replacement(self, n: int, count: int) -> np.ndarray:
        out = np.empty(count, dtype=np.int64)
        lib().orc_sample_without_replacement_g(C.byref(self.g), n, count, _p(out, _I64P))
        return out

    def sample_with_replacement(self, weights, count: int) -> np.ndarray:
        w = np.asarray(weights, dtype=np.float64)
        cum = np.empty_like(w)
        total = 0.0
        for i, x in enumerate(w):  # sequential fp64 prefix sums (rng.cpp:46-52)
            total += float(x)
            cum[i] = total
        out = np.empty(count, dtype=np.int64)
        for t in range(count):
            u = lib().orc_uniform_real(C.byref(self.g), 0.0, total)
            out[t] = min(int(np.searchsorted(cum, u, side="right")), w.size - 1)
        return out


def _p(a, t=_F64P):
    return a.ctypes.data_as(t)


# ---------------------------------------------------------------- seeds/ops
def splitmix64(state: int):
    st = C.c_uint64(state)
    out = lib().orc_splitmix64(C.byref(st))
    return int(out), int(st.value)


def derive_seed(seed: int, stream: int) -> int:
    return int(lib().orc_derive_seed(seed, stream))


def count_sketch_hashes(seed: int, n: int, s: int, j0: int = 0):
    b = np.empty(n, dtype=np.int64)
    g = np.empty(n, dtype=np.float64)
    lib().orc_count_sketch_hashes(seed, j0, n, s, _p(b, _I64P), _p(g))
    return b, g


def gaussian_matrix(rows: int, cols: int, seed: int) -> np.ndarray:
    out = np.empty((rows, cols), dtype=np.float64, order="F")
    lib().orc_gaussian_matrix(seed, rows, cols, _p(out))
    return out


def sample_without_replacement(n: int, count: int, seed: int) -> np.ndarray:
    out = np.empty(count, dtype=np.int64)
    if lib().orc_sample_without_replacement(seed, n, count, _p(out, _I64P)) != 0:
        raise ValueError("sample_without_replacement: count > n")
    return out


def sample_with_replacement(weights, count: int, seed: int) -> np.ndarray:
    w = np.ascontiguousarray(weights, dtype=np.float64)
    out = np.empty(count, dtype=np.int64)
    if lib().orc_sample_with_replacement(seed, _p(w), w.shape[0], count, _p(out, _I64P)) != 0:
        raise ValueError("sample_with_replacement: bad weights")
    return out


def srht_operator(n: int, s: int, seed: int):
    signs = np.empty(n, dtype=np.float64)
    idx = np.empty(s, dtype=np.int64)
    if lib().orc_srht_operator(seed, n, s, _p(signs), _p(idx, _I64P)) != 0:
        raise ValueError("srht_sketch: s > padded dimension")
    return signs, idx


def next_pow2(n: int) -> int:
    p = 1
    while p < n:
        p *= 2
    return p


# ---------------------------------------------------------------- sketches
def count_sketch_rows(m: np.ndarray, s: int, seed: int, extra: Optional[np.ndarray] = None, j0: int = 0,
                      threads: int = 1) -> np.ndarray:
    """S^T [M, extra] for row-major tall M (src/sketch.cpp:83-92 via sketch_rows), fp64, sequential order."""
    m = np.ascontiguousarray(m, dtype=np.float64)
    n, L = m.shape
    x = np.ascontiguousarray(extra, dtype=np.float64).reshape(-1) if extra is not None else None
    out = np.empty((s, L + (1 if x is not None else 0)), dtype=np.float64)
    if threads > 1:
        lib().orc_count_sketch_mt(_p(m), _p(x) if x is not None else None, n, L, L, s, seed, j0, _p(out), threads)
    else:
        lib().orc_count_sketch(_p(m), _p(x) if x is not None else None, n, L, L, s, seed, j0, _p(out))
    return out


def count_sketch(a: np.ndarray, s: int, seed: int) -> np.ndarray:
    """C = A S_count for column-major semantics (src/sketch.cpp:94-97)."""
    return count_sketch_rows(np.asarray(a, dtype=np.float64).T, s, seed).T


def count_sketch_operator(n: int, s: int, seed: int) -> np.ndarray:
    b, g = count_sketch_hashes(seed, n, s)
    op = np.zeros((n, s))
    op[np.arange(n), b] = g
    return op


def gaussian_sketch(a: np.ndarray, s: int, seed: int) -> np.ndarray:
    """C = A (G / sqrt(s)) (src/sketch.cpp:36-42)."""
    a = np.asarray(a, dtype=np.float64)
    g = gaussian_matrix(a.shape[1], s, seed) / math.sqrt(s)
    return a @ g


def fwht(x: np.ndarray) -> np.ndarray:
    y = np.ascontiguousarray(x, dtype=np.float64).copy()
    lib().orc_fwht(_p(y), y.shape[0])
    return y


def srht_sketch(a: np.ndarray, s: int, seed: int, threads: int = 1) -> np.ndarray:
    """C = A S_srht (src/sketch.cpp:57-81): segments are the columns of A."""
    a = np.asarray(a, dtype=np.float64)
    n = a.shape[1]
    signs, idx = srht_operator(n, s, seed)
    segs = np.ascontiguousarray(a.T)  # n segments of length m
    out = np.empty((s, a.shape[0]), dtype=np.float64)
    if threads > 1:
        rc = lib().orc_srht_sketch_mt(_p(segs), n, a.shape[0], a.shape[0], s, _p(signs), _p(idx, _I64P), _p(out),
                                      threads)
        assert rc == 0, rc
    else:
        lib().orc_srht_sketch(_p(segs), n, a.shape[0], a.shape[0], s, _p(signs), _p(idx, _I64P), _p(out))
    return out.T


def srht_rows(m: np.ndarray, s: int, seed: int, threads: int = 1) -> np.ndarray:
    """S^T M for row-major tall M (rows are the segments)."""
    return srht_sketch(np.asarray(m, dtype=np.float64).T, s, seed, threads).T


def combined_sketch(a: np.ndarray, s_cs: int, seed: int, stage2_kind: str, s2: int, seed2: int) -> np.ndarray:
    mid = count_sketch(a, s_cs, seed)
    if stage2_kind == "gaussian":
        return gaussian_sketch(mid, s2, seed2)
    return srht_sketch(mid, s2, seed2)


# ---------------------------------------------------------------- core
def fix_column_signs(m: np.ndarray, p: np.ndarray, pair_cols: bool, tol: float = 1e-12):
    """src/core.cpp:15-33."""
    for j in range(m.shape[1]):
        nz = np.nonzero(np.abs(m[:, j]) > tol)[0]
        if nz.size and m[nz[0], j] < 0.0:
            m[:, j] = -m[:, j]
            if pair_cols:
                p[:, j] = -p[:, j]
            else:
                p[j, :] = -p[j, :]


def thin_qr(a: np.ndarray):
    a = np.asarray(a, dtype=np.float64)
    if a.shape[0] < a.shape[1]:
        raise ValueError("thin_qr: rows < cols")
    q, r = np.linalg.qr(a, mode="reduced")
    q = np.array(q, order="F")
    r = np.triu(r)
    fix_column_signs(q, r, pair_cols=False)
    return q, r


def condensed_svd(a: np.ndarray):
    a = np.asarray(a, dtype=np.float64)
    u, sv, vt = np.linalg.svd(a, full_matrices=False)
    if sv.size == 0 or sv[0] <= 0.0:
        raise ValueError("condensed_svd: zero matrix has rank 0")
    thresh = max(a.shape) * np.finfo(np.float64).eps * sv[0]
    rho = int(np.sum(sv > thresh))
    u = np.array(u[:, :rho], order="F")
    v = np.array(vt[:rho].T, order="F")
    fix_column_signs(u, v, pair_cols=True)
    return u, sv[:rho].copy(), v


def truncated_svd(a: np.ndarray, k: int):
    if not (1 <= k <= min(np.shape(a))):
        raise ValueError("truncated_svd: k out of range")
    u, s, v = condensed_svd(a)
    return u[:, :k], s[:k], v[:, :k]


def pseudo_inverse(a: np.ndarray, tol: float = 1e-12) -> np.ndarray:
    a = np.asarray(a, dtype=np.float64)
    u, sv, vt = np.linalg.svd(a, full_matrices=False)
    if sv.size == 0 or sv[0] <= 0.0:
        return np.zeros((a.shape[1], a.shape[0]))
    inv = np.where(sv > tol * sv[0], 1.0 / np.where(sv > 0, sv, 1.0), 0.0)
    return (vt.T * inv) @ u.T


# ---------------------------------------------------------------- algorithms
def prototype_ksvd(a: np.ndarray, k: int, s: int, seed: int, q: int = 0):
    """src/randsvd.cpp:88-110 + SURVEY Appendix A.6 power iterations (Gaussian spec)."""
    a = np.asarray(a, dtype=np.float64)
    m, n = a.shape
    if not (1 <= k <= s <= min(m, n)):
        raise ValueError("prototype_ksvd: need k <= s <= min(m, n)")
    y = gaussian_sketch(a, s, seed)
    for _ in range(q):
        qy, _ = thin_qr(y)
        z, _ = thin_qr(a.T @ qy)
        y = a @ z
    qy, _ = thin_qr(y)
    b = qy.T @ a
    ub, sv, v = truncated_svd(b, min(k, s, n))
    return qy @ ub, sv, v, 2 + 2 * q


def faster_ksvd(a: np.ndarray, k: int, s: int, p_cs: int, p: int, seed: int):
    """src/randsvd.cpp:112-160: two passes; column count sketch C, then one joint
    combined (count p_cs -> Gaussian p) row sketch of [A, C]."""
    a = np.asarray(a, dtype=np.float64)
    if not (1 <= k < s < p < p_cs):
        raise ValueError("faster_ksvd: need k < s < p < p_cs")
    n = a.shape[1]
    c = count_sketch(a, s, derive_seed(seed, 1))
    mid = count_sketch_rows(np.hstack([a, c]), p_cs, derive_seed(seed, 2))
    mid = gaussian_sketch(mid.T, p, derive_seed(seed, 3)).T  # p x (n + s)
    l, d = mid[:, :n], mid[:, n:]
    qd, rd = thin_qr(d)
    u, sv, v = truncated_svd(qd.T @ l, k)
    back = c @ (pseudo_inverse(rd) @ (u * sv))
    uf, sf, vf = condensed_svd(back)
    return uf, sf, v @ vf, 2


def numerical_rank(m: np.ndarray, thresh: float = 1e-10) -> int:
    sv = np.linalg.svd(m, compute_uv=False)
    return int(np.sum(sv > thresh * sv[0])) if sv.size and sv[0] > 0 else 0


def lsr_preconditioned(a: np.ndarray, b: np.ndarray, eps: float, seed: int, sketch_size: int = 0,
                       use_cg: bool = False, kind: str = "count"):
    """src/regression.cpp:94-198 (sketch-and-precondition; CountSketch by default).
    Returns (x, objective, iterations, kappa_estimate)."""
    import scipy.linalg as sla
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64).reshape(-1)
    n, d = a.shape
    if n < d:
        raise ValueError("lsr_preconditioned: n < d")
    if not (0.0 < eps < 1.0):
        raise ValueError("lsr_preconditioned: eps out of (0,1)")
    s = sketch_size or min(d * d, 20 * d)
    s = min(s, n)
    if s < d:
        raise ValueError("lsr_preconditioned: sketch size < d")
    stacked = np.hstack([a, b[:, None]])
    draw = seed
    for attempt in range(2):
        if kind == "count":
            sk = count_sketch_rows(stacked, s, draw)
        elif kind == "gaussian":
            sk = gaussian_sketch(stacked.T, s, draw).T
        else:
            sk = srht_rows(stacked, s, draw)
        q, r = thin_qr(sk[:, :d])
        dg = np.abs(np.diag(r))
        if dg.max() > 0 and dg.min() > 1e-12 * dg.max():
            break
        if attempt >= 1:
            raise RuntimeError("lsr_preconditioned: sketched matrix singular")
        draw = derive_seed(seed, 0x5E5A)
    sb = sk[:, d]
    t = lambda v: sla.solve_triangular(r, v, lower=False)  # noqa: E731
    tt = lambda v: sla.solve_triangular(r, v, lower=False, trans="T")  # noqa: E731
    z = q.T @ sb
    budget = int(math.ceil(10.0 * math.log10(1.0 / eps)))
    grad_tol = max(1e-15 * np.linalg.norm(tt(a.T @ b)), 1e-300)
    it = 0
    if not use_cg:
        prev = math.inf
        while it < budget:
            grad = tt(a.T @ (b - a @ t(z)))
            z = z + grad
            gn = np.linalg.norm(grad)
            if gn <= grad_tol or gn >= 0.9 * prev:
                it += 1
                break
            prev = gn
            it += 1
    else:
        rr = tt(a.T @ (b - a @ t(z)))
        p = rr.copy()
        rs = rr @ rr
        while it < budget and math.sqrt(rs) > grad_tol:
            ap = tt(a.T @ (a @ t(p)))
            alpha = rs / (p @ ap)
            z = z + alpha * p
            rr = rr - alpha * ap
            rs_new = rr @ rr
            p = rr + (rs_new / rs) * p
            rs = rs_new
            it += 1
    x = t(z)
    res = a @ x - b
    sv = np.linalg.svd(a @ sla.solve_triangular(r, np.eye(d), lower=False), compute_uv=False)
    return x, float(res @ res), it, float(sv[0] / sv[-1])


def lsr_sketched(a: np.ndarray, b: np.ndarray, sk: np.ndarray):
    """Solve with a given sketch sk = S^T [A, b] (src/regression.cpp:80-91)."""
    d = a.shape[1]
    a_sk, b_sk = sk[:, :d], sk[:, d]
    flagged = numerical_rank(a_sk) < d
    if flagged:
        x = pseudo_inverse(a_sk) @ b_sk
    else:
        x = np.linalg.lstsq(a_sk, b_sk, rcond=None)[0]
    r = a @ x - b
    return x, float(r @ r), flagged


def rbf_kernel(x1: np.ndarray, x2: np.ndarray, sigma: float) -> np.ndarray:
    """src/spsd.cpp:33-47."""
    x1 = np.asarray(x1, dtype=np.float64)
    x2 = np.asarray(x2, dtype=np.float64)
    inv = 1.0 / (sigma * sigma)
    sq1 = np.einsum("ij,ij->i", x1, x1)
    sq2 = np.einsum("ij,ij->i", x2, x2)
    return np.exp((x1 @ x2.T - 0.5 * (sq1[:, None] + sq2[None, :])) * inv)


def nystrom(x: np.ndarray, sigma: float, s: int, seed: int, target_k: int = 0):
    """src/spsd.cpp:181-222 on KernelView(x, sigma). Returns (L, selected, lam_kept)."""
    x = np.asarray(x, dtype=np.float64)
    n = x.shape[0]
    kk = target_k if target_k > 0 else int(math.ceil(0.8 * s))
    if not (1 <= kk <= s <= n):
        raise ValueError("nystrom: need k <= s <= n")
    sel = sample_without_replacement(n, s, derive_seed(seed, 1))
    c = rbf_kernel(x, x[sel], sigma)
    c[sel, np.arange(s)] = 1.0
    w = c[sel, :]
    lam, vec = np.linalg.eigh(0.5 * (w + w.T))
    lam_max = lam[-1]
    if lam_max <= 0.0:
        raise RuntimeError("nystrom: kernel block has no positive spectrum")
    floor = np.finfo(np.float64).eps * lam_max * n
    kept = 0
    while kept < kk and lam[s - 1 - kept] > floor:
        kept += 1
    if kept == 0:
        raise RuntimeError("nystrom: no retained eigenvalues")
    u = vec[:, ::-1][:, :kept]
    lk = lam[::-1][:kept]
    return c @ (u / np.sqrt(lk)), sel, lk


def approx_eig(l: np.ndarray, k: int):
    """src/spsd.cpp:257-265."""
    if not (1 <= k <= l.shape[1]):
        raise ValueError("approx_eig: k > cols(L)")
    u, sv, _ = condensed_svd(l)
    if k > sv.size:
        raise ValueError("approx_eig: k exceeds rank(L)")
    return u[:, :k], sv[:k] ** 2


def spsd_faster(x: np.ndarray, sigma: float, s: int, p: int, seed: int, dense: bool = False):
    """src/spsd.cpp:131-168 on a KernelView of x (or on the dense SPSD x when dense=True).
    Returns (Q, Z, selected, secondary, flagged)."""
    x = np.asarray(x, dtype=np.float64)
    n = x.shape[0]
    if not (1 <= s <= p <= n):
        raise ValueError("spsd_faster: need s <= p <= n")
    sel = sample_without_replacement(n, s, derive_seed(seed, 1))
    c = x[:, sel] if dense else rbf_kernel(x, x[sel], sigma)
    if not dense:
        c[sel, np.arange(s)] = 1.0
    q, _ = thin_qr(c)
    if p == n:
        sec = np.arange(n)
    else:
        lev = np.einsum("ij,ij->i", q, q)
        sec = np.union1d(np.unique(sample_with_replacement(lev, p, derive_seed(seed, 2))), sel)
    q_sub = q[sec]
    k_sub = x[np.ix_(sec, sec)] if dense else rbf_kernel(x[sec], x[sec], sigma)
    if not dense:
        np.fill_diagonal(k_sub, 1.0)
    flagged = numerical_rank(q_sub) < s
    pinv = pseudo_inverse(q_sub)
    z = pinv @ k_sub @ pinv.T
    return q, 0.5 * (z + z.T), sel, sec, flagged


def cur_faster(a: np.ndarray, c: int, r: int, seed: int):
    """src/cur.cpp:47-104 with the uniform sampler and default p_c = p_r = 2(c + r);
    the kernel variant (:188-212) calls it on K* = rbf_kernel(xtest, xtrain).
    Returns (C, U, R, col_idx, row_idx, sec_rows, sec_cols, flagged)."""
    a = np.asarray(a, dtype=np.float64)
    m, n = a.shape
    if not (1 <= c <= n):
        raise ValueError("cur: c out of [1, n]")
    if not (1 <= r <= m):
        raise ValueError("cur: r out of [1, m]")
    p_c, p_r = min(2 * (c + r), m), min(2 * (c + r), n)
    ci = sample_without_replacement(n, c, derive_seed(seed, 1))
    ri = sample_without_replacement(m, r, derive_seed(seed, 2))
    pc = np.union1d(sample_without_replacement(m, p_c, derive_seed(seed, 3)), ri)
    pr = np.union1d(sample_without_replacement(n, p_r, derive_seed(seed, 4)), ci)
    cm, rm = a[:, ci], a[ri, :]
    c_sub, r_sub = cm[pc], rm[:, pr]
    flagged = numerical_rank(c_sub) < min(c_sub.shape) or numerical_rank(r_sub) < min(r_sub.shape)
    u = pseudo_inverse(c_sub) @ a[np.ix_(pc, pr)] @ pseudo_inverse(r_sub)
    return cm, u, rm, ci, ri, pc, pr, flagged


def leverage_scores(a: np.ndarray, k: Optional[int] = None) -> np.ndarray:
    u, s, v = truncated_svd(a, k) if k else condensed_svd(a)
    return np.sum(v * v, axis=1)


def row_leverage(m: np.ndarray) -> np.ndarray:
    """||Q_i,:||^2 for Q = thin_qr(M).Q (the src/spsd.cpp:150 pattern)."""
    q, _ = thin_qr(m)
    return np.sum(q * q, axis=1)
