"""GPU parity of spsd.hpp (rbf_kernel, Nystrom, approx_eig) against the
oracle and the reference's tests/test_spsd.cpp properties."""
import math

import numpy as np
import pytest

import paper_1505_07570_b200 as rn
from oracle import oracle as orc

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def test_rbf_unit_diagonal_symmetry(ctx):
    # tests/test_spsd.cpp:20-31: exact unit diagonal, bitwise symmetry
    x = orc.gaussian_matrix(30, 4, 1)
    k = rn.rbf_kernel(x, x, 1.5, ctx=ctx)
    assert np.all(np.diag(k) == 1.0)
    assert np.linalg.norm(k - k.T) == 0.0
    assert k.max() <= 1.0 and k.min() >= 0.0
    d2 = np.sum((x[3] - x[17]) ** 2)
    assert abs(k[3, 17] - math.exp(-d2 / (2 * 1.5 ** 2))) <= 1e-12 * math.exp(-d2 / (2 * 1.5 ** 2))
    assert np.max(np.abs(k - orc.rbf_kernel(x, x, 1.5))) <= 1e-13


def test_rbf_fp32_and_rectangular(ctx):
    rng = np.random.default_rng(2)
    x1 = rng.standard_normal((300, 64)).astype(np.float32) * 3
    x2 = rng.standard_normal((70, 64)).astype(np.float32) * 3
    k = rn.rbf_kernel(dev(x1), dev(x2), 20.0, ctx=ctx).cpu().numpy()
    ref = orc.rbf_kernel(x1.astype(np.float64), x2.astype(np.float64), 20.0)
    assert np.max(np.abs(k - ref)) <= 1e-5
    with pytest.raises(ValueError, match="sigma <= 0"):
        rn.rbf_kernel(x1, x2, 0.0, ctx=ctx)


def test_nystrom_matches_oracle(ctx):
    x = orc.gaussian_matrix(400, 5, 10)
    view = rn.KernelView(x, rn.KernelSpec(2.0))
    f = rn.nystrom(view, 40, 11, ctx=ctx)
    L, sel, lam = orc.nystrom(x, 2.0, 40, 11)
    assert np.array_equal(f.selected, sel)
    assert f.L.shape == L.shape
    assert np.linalg.norm(f.L @ f.L.T - L @ L.T) <= 1e-8 * np.linalg.norm(L @ L.T)
    assert view.entries_evaluated() == 400 * 40
    v2 = rn.KernelView(orc.gaussian_matrix(100, 5, 10), rn.KernelSpec(2.0))
    f2 = rn.nystrom(v2, 10, 11, ctx=ctx)  # default k = ceil(0.8 s)
    assert f2.L.shape[1] <= 8 and f2.L.shape[0] == 100 and f2.selected.size == 10


def test_nystrom_argument_checks(ctx):
    v = rn.KernelView(orc.gaussian_matrix(20, 3, 1), rn.KernelSpec(1.0))
    with pytest.raises(ValueError, match="k <= s <= n"):
        rn.nystrom(v, 30, 1, ctx=ctx)
    with pytest.raises(ValueError, match="sigma <= 0"):
        rn.KernelView(np.ones((3, 2)), rn.KernelSpec(0.0))


def test_approx_eig(ctx):
    # tests/test_spsd.cpp:133-142
    l = orc.gaussian_matrix(30, 6, 17)
    u, lam = rn.approx_eig(l, 4, ctx=ctx)
    g = l @ l.T
    for t in range(4):
        assert np.linalg.norm(g @ u[:, t] - lam[t] * u[:, t]) <= 1e-8 * lam[t]
        if t:
            assert lam[t] <= lam[t - 1]
    uo, lo = orc.approx_eig(l, 4)
    assert np.allclose(lam, lo, rtol=1e-12) and np.allclose(u, uo, atol=1e-10)


def test_nystrom_eig_gram_route_matches_oracle(ctx):
    rng = np.random.default_rng(4)
    x = rng.standard_normal((3000, 8)) * 2
    view = rn.KernelView(x, rn.KernelSpec(3.0))
    u, lam, sel, kept = rn.nystrom_eig(view, 200, 9, 150, 12, ctx=ctx)
    L, sel_o, _ = orc.nystrom(x, 3.0, 200, 9, 150)
    uo, lo = orc.approx_eig(L, 12)
    assert np.array_equal(sel, sel_o) and kept == L.shape[1]
    assert np.max(np.abs(lam - lo) / lo) <= 1e-8
    assert np.max(np.abs(np.abs(u[:, :4]) - np.abs(uo[:, :4]))) <= 1e-6


@pytest.mark.parametrize("n,s,k,sigma", [(3000, 200, 12, 3.0), (6000, 400, 40, 4.0), (2500, 257, 10, 3.0)])
def test_nystrom_eig_full_rank_route(ctx, n, s, k, sigma):
    # target_k = s with a well-conditioned W: the Cholesky route (L' = C R^-1)
    # replaces eig(W); approx_eig outputs must match the reference's eig route.
    rng = np.random.default_rng(n)
    x = rng.standard_normal((n, 8)) * 2
    view = rn.KernelView(x, rn.KernelSpec(sigma))
    u, lam, sel, kept = rn.nystrom_eig(view, s, 9, s, k, ctx=ctx)
    L, sel_o, lam_w = orc.nystrom(x, sigma, s, 9, s)
    uo, lo = orc.approx_eig(L, k)
    assert kept == L.shape[1] == s and np.array_equal(sel, sel_o)
    assert np.max(np.abs(lam - lo) / lo) <= 1e-8
    # sign-fixed columns, compared where the eigenvalue is separated from its neighbours
    rel = np.abs(np.diff(lo)) / lo[1:]
    sep = [t for t in range(k - 1) if rel[t] > 1e-3 and (t == 0 or rel[t - 1] > 1e-3)]
    assert sep
    assert np.max(np.abs(u[:, sep] - uo[:, sep])) <= 1e-6


def test_nystrom_eig_rank_deficient_falls_back(ctx):
    # duplicated points make W singular: the floor drops eigenvalues (kept < s),
    # so the eigendecomposition route must run and match the oracle.
    rng = np.random.default_rng(11)
    base = rng.standard_normal((400, 3))
    x = np.vstack([base, base, base])
    view = rn.KernelView(x, rn.KernelSpec(2.0))
    _, lam, sel, kept = rn.nystrom_eig(view, 300, 5, 300, 6, ctx=ctx)
    L, sel_o, _ = orc.nystrom(x, 2.0, 300, 5, 300)
    _, lo = orc.approx_eig(L, 6)
    assert np.array_equal(sel, sel_o) and kept == L.shape[1] < 300
    assert np.max(np.abs(lam - lo) / lo) <= 1e-6


def test_nystrom_eig_fp32(ctx):
    rng = np.random.default_rng(5)
    means = rng.standard_normal((4, 16)) * 3
    x = (means[rng.integers(0, 4, 8192)] + rng.standard_normal((8192, 16))).astype(np.float32)
    view = rn.KernelView(dev(x), rn.KernelSpec(6.0))
    _, lam, _, _ = rn.nystrom_eig(view, 256, 3, 128, 16, want_vectors=False, ctx=ctx)
    L, _, _ = orc.nystrom(x.astype(np.float64), 6.0, 256, 3, 128)
    _, lo = orc.approx_eig(L, 16)
    assert np.max(np.abs(lam - lo) / lo) <= 1e-3


def test_spsd_faster_entry_budget_and_error(ctx):
    # tests/test_spsd.cpp:58-76
    n, s, p = 120, 10, 40
    x = orc.gaussian_matrix(n, 4, 4)
    view = rn.KernelView(x, rn.KernelSpec(1.5))
    sk = rn.spsd_faster(view, s, p, 6, ctx=ctx)
    assert view.entries_evaluated() <= n * s + len(sk.secondary) ** 2
    assert set(sk.selected.tolist()) <= set(sk.secondary.tolist())
    k = orc.rbf_kernel(x, x, 1.5)
    zb = sk.Q.T @ k @ sk.Q
    best = np.linalg.norm(k - sk.Q @ zb @ sk.Q.T)
    assert np.linalg.norm(k - sk.reconstruct()) <= 2.0 * best + 1e-12
    assert np.array_equal(sk.Z, sk.Z.T)


def test_spsd_faster_full_secondary_is_best_core(ctx):
    # tests/test_spsd.cpp:78-85 (dense K)
    x = orc.gaussian_matrix(50, 3, 5)
    k = orc.rbf_kernel(x, x, 1.0)
    sk = rn.spsd_faster(k, 8, 50, 7, ctx=ctx)
    zb = sk.Q.T @ k @ sk.Q
    assert np.linalg.norm(sk.Z - zb) <= 1e-8 * np.linalg.norm(zb)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_spsd_faster_matches_oracle(ctx, dtype):
    rng = np.random.default_rng(9)
    x = (rng.standard_normal((4000, 8)) * 1.5).astype(dtype)
    sk = rn.spsd_faster(rn.KernelView(dev(x), rn.KernelSpec(2.5)), 60, 400, 31, ctx=ctx)
    q, z, sel, sec, flagged = orc.spsd_faster(x.astype(np.float64), 2.5, 60, 400, 31)
    assert np.array_equal(sk.selected, sel)
    assert sk.flagged == flagged
    Q = sk.Q.cpu().numpy()
    tol = 1e-9 if dtype == np.float64 else 1e-4
    assert np.max(np.abs(Q - q)) <= tol * 10
    if dtype == np.float64:
        # leverage draws are bit-exact given the scores; the scores agree to ~1e-15
        assert np.array_equal(sk.secondary, sec)
        assert np.linalg.norm(sk.Z - z) <= 1e-8 * np.linalg.norm(z)
    with pytest.raises(ValueError, match="s <= p <= n"):
        rn.spsd_faster(rn.KernelView(x, rn.KernelSpec(2.5)), 60, 50, 1, ctx=ctx)


@pytest.mark.parametrize("seed", [17, 18, 19])
def test_cur_faster_kernel_matches_oracle(ctx, seed):
    # tests/test_cur.cpp:74-93: the lazy kernel CUR equals cur_faster on K*
    xtest = orc.gaussian_matrix(45, 3, 15)
    xtrain = orc.gaussian_matrix(60, 3, 16)
    f = rn.cur_faster_kernel(xtest, xtrain, 1.3, 7, 6, seed, ctx=ctx)
    ks = orc.rbf_kernel(xtest, xtrain, 1.3)
    C, U, R, ci, ri, pc, pr, flagged = orc.cur_faster(ks, 7, 6, seed)
    assert np.array_equal(f.col_indices, ci) and np.array_equal(f.row_indices, ri)
    assert np.array_equal(f.secondary_rows, pc) and np.array_equal(f.secondary_cols, pr)
    assert f.flagged == flagged
    assert np.allclose(f.C, C, rtol=0, atol=1e-14) and np.allclose(f.R, R, rtol=0, atol=1e-14)
    assert np.linalg.norm(f.U - U) <= 1e-8 * np.linalg.norm(U)
    assert f.entries_visited <= 45 * 7 + 60 * 6 + len(f.secondary_rows) * len(f.secondary_cols)


def test_cur_faster_kernel_preconditions(ctx):
    # tests/test_cur.cpp:95-103
    xtest = orc.gaussian_matrix(1, 3, 20)
    xtrain = orc.gaussian_matrix(30, 3, 21)
    with pytest.raises(ValueError, match="r out of"):
        rn.cur_faster_kernel(xtest, xtrain, 1.0, 5, 3, 1, ctx=ctx)
    ok = rn.cur_faster_kernel(xtest, xtrain, 1.0, 5, 1, 1, ctx=ctx)
    assert ok.R.shape[0] == 1


def test_cur_faster_kernel_fp32_large(ctx):
    rng = np.random.default_rng(3)
    xtest = rng.standard_normal((3000, 16)).astype(np.float32)
    xtrain = rng.standard_normal((5000, 16)).astype(np.float32)
    f = rn.cur_faster_kernel(dev(xtest), dev(xtrain), 4.0, 80, 60, 9, ctx=ctx)
    ks = orc.rbf_kernel(xtest.astype(np.float64), xtrain.astype(np.float64), 4.0)
    C, U, R, ci, ri, pc, pr, flagged = orc.cur_faster(ks, 80, 60, 9)
    assert np.array_equal(f.secondary_rows, pc) and np.array_equal(f.secondary_cols, pr)
    rec = f.C.cpu().numpy().astype(np.float64) @ f.U @ f.R.cpu().numpy().astype(np.float64)
    ref = C @ U @ R
    assert np.linalg.norm(rec - ref) <= 1e-3 * np.linalg.norm(ref)
