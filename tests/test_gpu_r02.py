"""GPU parity of the round-2 kernels against the oracle: the skinny fp64 DMMA
GEMM (n <= 32 outputs, both A layouts), the one-CTA Jacobi core of the
truncated SVD, the speculative prototype_ksvd pipeline and its cached CUDA
graph (replays must see new data behind the same pointer), and the int8
Ozaki-split fp64 Gaussian stage (dynamic range, zero and non-finite columns).
Reference semantics: src/randsvd.cpp:88-110, src/sketch.cpp:36-42,108-123."""
import numpy as np
import pytest

import paper_1505_07570_b200 as rn
from oracle import oracle as orc

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def relf(a, b):
    return float(np.linalg.norm(np.asarray(a) - b) / max(np.linalg.norm(b), 1e-300))


def lowrank(m, n, seed, decay=20.0, noise=1e-3):
    rng = np.random.default_rng(seed)
    u, _ = np.linalg.qr(rng.standard_normal((m, min(m, n))))
    v, _ = np.linalg.qr(rng.standard_normal((n, min(m, n))))
    sig = np.exp(-np.arange(1, min(m, n) + 1) / decay)
    return (u * sig) @ v.T + noise * rng.standard_normal((m, n))


# ------------------------------------------------------------ skinny DMMA GEMM
@pytest.mark.parametrize("m,n,s,order", [(1000, 333, 30, "C"), (777, 2049, 17, "F"), (129, 4000, 32, "C"),
                                         (5000, 130, 1, "F")])
def test_skinny_gaussian_sketch_layouts(ctx, m, n, s, order):
    """C = A (G / sqrt(s)) with s <= 32 (the skinny kernel) for row- and
    column-major A, ragged m and k, against the oracle (src/sketch.cpp:36-42)."""
    rng = np.random.default_rng(m + n + s)
    a = np.asarray(rng.standard_normal((m, n)), order=order)
    got = rn.gaussian_sketch(dev(a) if order == "C" else a, s, 91 + s, ctx=ctx)
    got = got.cpu().numpy() if hasattr(got, "cpu") else got
    assert relf(got, orc.gaussian_sketch(a, s, 91 + s)) <= 1e-12


# ------------------------------------------------------------ Jacobi core + pipeline
def test_prototype_clustered_spectrum_matches_oracle(ctx):
    """Equal leading singular values (repeated eigenvalues of the s x s core
    Gram) through the Jacobi core: sigma within 1e-8 of the same-Omega oracle."""
    rng = np.random.default_rng(5)
    m, n, k, s = 3000, 400, 12, 30
    u, _ = np.linalg.qr(rng.standard_normal((m, n)))
    v, _ = np.linalg.qr(rng.standard_normal((n, n)))
    sig = np.concatenate([np.ones(6), np.exp(-np.arange(1, n - 5) / 10.0) * 0.5])
    a = (u * sig) @ v.T + 1e-6 * rng.standard_normal((m, n))
    r = rn.prototype_ksvd(dev(a), k, s, 1234, power_iters=1, ctx=ctx)
    _, so, _, _ = orc.prototype_ksvd(a, k, s, 1234, q=1)
    assert np.max(np.abs(r.factors.singular_values - so) / so) <= 1e-8


def test_prototype_graph_replay_and_checked_path(ctx, monkeypatch):
    """The speculative pipeline is captured into a CUDA graph on the first call
    and replayed: replays are bitwise identical, see new data written behind
    the same device pointer, and agree with the checked (synchronizing) path and
    with the oracle."""
    m, n, k, s = 2048, 640, 20, 30
    a = lowrank(m, n, 1)
    da = dev(a)
    runs = [rn.prototype_ksvd(da, k, s, 4242, power_iters=1, ctx=ctx) for _ in range(3)]
    for r in runs[1:]:
        assert np.array_equal(r.factors.singular_values, runs[0].factors.singular_values)
        assert torch.equal(r.factors.U, runs[0].factors.U) and torch.equal(r.factors.V, runs[0].factors.V)
    _, so, _, _ = orc.prototype_ksvd(a, k, s, 4242, q=1)
    assert np.max(np.abs(runs[0].factors.singular_values - so) / so) <= 1e-8
    monkeypatch.setenv("RNLA_KSVD_SYNC", "1")
    chk = rn.prototype_ksvd(da, k, s, 4242, power_iters=1, ctx=ctx)
    monkeypatch.delenv("RNLA_KSVD_SYNC")
    assert np.max(np.abs(chk.factors.singular_values - so) / so) <= 1e-8
    assert np.max(np.abs(chk.factors.singular_values - runs[0].factors.singular_values) / so) <= 1e-12
    # new contents, same pointer: the replayed graph reads them
    b = lowrank(m, n, 2, decay=15.0)
    da.copy_(dev(b))
    rb = rn.prototype_ksvd(da, k, s, 4242, power_iters=1, ctx=ctx)
    _, sb, _, _ = orc.prototype_ksvd(b, k, s, 4242, q=1)
    assert np.max(np.abs(rb.factors.singular_values - sb) / sb) <= 1e-8


@pytest.mark.parametrize("on_device", [True, False])
def test_prototype_rank_deficient_falls_back(ctx, on_device):
    """A rank-deficient sketch breaks the Cholesky factorizations of the
    speculative pipeline; the status words send the call to the checked path,
    which returns the reference's rank and an exact factorization
    (src/core.cpp:48-64, tests/test_randsvd.cpp:39-49)."""
    a = orc.gaussian_matrix(600, 3, 7) @ orc.gaussian_matrix(3, 300, 8)
    r = rn.prototype_ksvd(dev(a) if on_device else a, 3, 30, 11, power_iters=1, ctx=ctx)
    sv = r.factors.singular_values
    assert 1 <= sv.size <= 3
    U = r.factors.U.cpu().numpy() if on_device else r.factors.U
    V = r.factors.V.cpu().numpy() if on_device else r.factors.V
    rec = (U[:, : sv.size] * sv) @ V[:, : sv.size].T
    assert np.linalg.norm(rec - a) <= 1e-8 * np.linalg.norm(a)
    _, so, _, _ = orc.prototype_ksvd(a, 3, 30, 11, q=1)
    assert np.max(np.abs(sv - so[: sv.size]) / so[: sv.size]) <= 1e-8


# ------------------------------------------------------------ tridiagonal eigensolver (32 < s <= 128)
@pytest.mark.parametrize("kind", ["graded", "repeated", "decaying"])
def test_prototype_tridiagonal_core_matches_oracle(ctx, kind):
    """The s x s core Gram for 32 < s <= 128 goes through the one-CTA
    tridiagonal eigensolver (Householder, multisection, twisted factorizations,
    Gram-Schmidt within clusters). Graded singular values put most of the core
    spectrum in one cluster; exactly repeated ones make the twisted vectors
    collapse, so the status word sends the call to the checked path (cuSOLVER).
    sigma within 1e-8 of the same-Omega oracle, U orthonormal."""
    rng = np.random.default_rng(11)
    m, n, k, s = 3000, 500, 40, 96
    u, _ = np.linalg.qr(rng.standard_normal((m, n)))
    v, _ = np.linalg.qr(rng.standard_normal((n, n)))
    if kind == "graded":
        sig = np.arange(1, n + 1) ** -1.5
    elif kind == "repeated":
        sig = np.concatenate([np.ones(8), 0.5 * np.exp(-np.arange(1, n - 7) / 30.0)])
    else:
        sig = np.exp(-np.arange(1, n + 1) / 25.0)
    a = (u * sig) @ v.T
    r = rn.prototype_ksvd(dev(a), k, s, 77, power_iters=1, ctx=ctx)
    _, so, _, _ = orc.prototype_ksvd(a, k, s, 77, q=1)
    assert np.max(np.abs(r.factors.singular_values - so) / so) <= 1e-8
    U = r.factors.U.cpu().numpy()
    assert np.linalg.norm(U.T @ U - np.eye(k)) <= 1e-9


# ------------------------------------------------------------ Ozaki Gaussian stage
def test_ozaki_gaussian_rows_dynamic_range(ctx):
    """fp64 row sketch S'M with s >= 128 (the int8 digit path): columns spanning
    1e-150 .. 1e150 and a zero column keep their own relative accuracy (scales
    are per column), against the oracle."""
    rng = np.random.default_rng(9)
    n, L, s = 3000, 40, 256
    m = rng.standard_normal((n, L))
    scale = 10.0 ** np.linspace(-150, 150, L)
    m *= scale
    m[:, 7] = 0.0
    got = rn.sketch_rows(dev(m), rn.SketchSpec.gaussian(s, 31), ctx=ctx).cpu().numpy()
    ref = orc.gaussian_sketch(m.T, s, 31).T
    assert np.all(got[:, 7] == 0.0)
    for j in range(L):
        if j != 7:  # compared in units of the column's scale (the norms would overflow)
            assert relf(got[:, j] / scale[j], ref[:, j] / scale[j]) <= 1e-11, j


def test_ozaki_gaussian_rows_nonfinite_column(ctx):
    """A NaN in one column makes that output column non-finite and leaves the
    others exact to the gate (as the fp64 GEMM would)."""
    rng = np.random.default_rng(10)
    n, L, s = 2000, 33, 128
    m = rng.standard_normal((n, L))
    m[123, 5] = np.nan
    got = rn.sketch_rows(dev(m), rn.SketchSpec.gaussian(s, 5), ctx=ctx).cpu().numpy()
    assert not np.any(np.isfinite(got[:, 5]))
    keep = [j for j in range(L) if j != 5]
    ref = orc.gaussian_sketch(m[:, keep].T, s, 5).T
    assert relf(got[:, keep], ref) <= 1e-11


@pytest.mark.parametrize("n", [128, 1000, 8193])
def test_ozaki_combined_composition_bitwise(ctx, n):
    """combined == gaussian(count) bitwise with the digit stage on both sides
    (tests/test_sketch.cpp:88-98), ragged K."""
    rng = np.random.default_rng(n)
    a = rng.standard_normal((max(n, 200) * 4, 37))
    s_cs, s2 = n, 128
    seed, seed2 = 17, 29
    cs = rn.sketch_rows(dev(a), rn.SketchSpec.count_sketch(s_cs, seed), ctx=ctx)
    two = rn.sketch_rows(cs, rn.SketchSpec.gaussian(s2, seed2), ctx=ctx).cpu().numpy()
    one = rn.sketch_rows(dev(a), rn.SketchSpec.combined(s_cs, rn.SketchSpec.gaussian(s2, seed2), seed),
                         ctx=ctx).cpu().numpy()
    assert np.array_equal(one, two)
    ref = orc.gaussian_sketch(orc.count_sketch_rows(a, s_cs, seed).T, s2, seed2).T
    assert relf(one, ref) <= 1e-11
