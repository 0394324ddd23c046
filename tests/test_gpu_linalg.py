"""GPU parity of core.hpp / randsvd.hpp against the oracle and the reference's
own property tests (tests/test_core.cpp, tests/test_randsvd.cpp)."""
import numpy as np
import pytest

import paper_1505_07570_b200 as rn
from oracle import oracle as orc

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def test_thin_qr(ctx):
    a = orc.gaussian_matrix(20, 8, 1)
    f = rn.thin_qr(a, ctx=ctx)
    q, r = f.Q, f.R
    assert np.linalg.norm(q @ r - a) <= 1e-12 * np.linalg.norm(a)
    assert np.linalg.norm(q.T @ q - np.eye(8)) <= 1e-12
    assert np.all(np.tril(r, -1) == 0.0)
    for j in range(8):
        nz = np.nonzero(np.abs(q[:, j]) > 1e-12)[0]
        assert q[nz[0], j] > 0
    qo, ro = orc.thin_qr(a)
    assert np.allclose(q, qo, atol=1e-13) and np.allclose(r, ro, atol=1e-12)
    with pytest.raises(ValueError, match="rows < cols"):
        rn.thin_qr(orc.gaussian_matrix(3, 5, 2), ctx=ctx)


def test_condensed_svd_rank_cut(ctx):
    a = orc.gaussian_matrix(30, 4, 3) @ orc.gaussian_matrix(4, 25, 4)
    f = rn.condensed_svd(a, ctx=ctx)
    assert f.rank() == 4
    assert np.linalg.norm(f.reconstruct() - a) <= 1e-10 * np.linalg.norm(a)
    assert np.linalg.norm(f.U.T @ f.U - np.eye(4)) <= 1e-12
    assert np.linalg.norm(f.V.T @ f.V - np.eye(4)) <= 1e-12
    assert np.all(np.diff(f.singular_values) <= 0) and f.singular_values[-1] > 0
    uo, so, vo = orc.condensed_svd(a)
    assert np.allclose(f.singular_values, so, rtol=1e-12)
    assert np.allclose(f.U, uo, atol=1e-10) and np.allclose(f.V, vo, atol=1e-10)
    with pytest.raises(ValueError, match="zero matrix"):
        rn.condensed_svd(np.zeros((4, 3)), ctx=ctx)


@pytest.mark.parametrize("m,n", [(15, 12), (200, 30), (30, 200), (4000, 50)])
def test_truncated_svd_optimal(ctx, m, n):
    a = orc.gaussian_matrix(m, n, 5)
    k = 3
    f = rn.truncated_svd(a, k, ctx=ctx)
    assert f.rank() == k
    sv = np.linalg.svd(a, compute_uv=False)
    err = np.linalg.norm(a - f.reconstruct()) ** 2
    assert abs(err - np.sum(sv[k:] ** 2)) <= 1e-10 * np.sum(sv[k:] ** 2)


def test_pseudo_inverse(ctx):
    a = orc.gaussian_matrix(10, 6, 6)
    p = rn.pseudo_inverse(a, ctx=ctx)
    assert np.linalg.norm(a @ p @ a - a) <= 1e-10 * np.linalg.norm(a)
    assert np.linalg.norm(p @ a @ p - p) <= 1e-10 * np.linalg.norm(p)
    assert np.linalg.norm((a @ p).T - a @ p) <= 1e-10
    z = rn.pseudo_inverse(np.zeros((4, 7)), ctx=ctx)
    assert z.shape == (7, 4) and np.linalg.norm(z) == 0.0


def test_prototype_exact_rank_k(ctx):
    # tests/test_randsvd.cpp:39-49
    a = orc.gaussian_matrix(80, 5, 2) @ orc.gaussian_matrix(5, 60, 22)
    r = rn.prototype_ksvd(a, 5, 20, 3, opts=rn.KsvdOptions(True), ctx=ctx)
    assert r.error_fro <= 1e-8 * np.linalg.norm(a)
    assert r.passes_over_a == 2
    assert r.factors.U.shape[0] == 80 and r.factors.V.shape[0] == 60
    assert r.factors.singular_values.size <= 5


def test_prototype_error_above_optimum_and_deterministic(ctx):
    a = orc.gaussian_matrix(50, 50, 4)
    r = rn.prototype_ksvd(a, 5, 25, 5, opts=rn.KsvdOptions(True), ctx=ctx)
    sv = np.linalg.svd(a, compute_uv=False)
    assert r.error_fro >= np.sqrt(np.sum(sv[5:] ** 2)) - 1e-9
    b = orc.gaussian_matrix(40, 35, 11)
    r1 = rn.prototype_ksvd(b, 4, 12, 99, ctx=ctx)
    r2 = rn.prototype_ksvd(b, 4, 12, 99, ctx=ctx)
    assert np.array_equal(r1.factors.singular_values, r2.factors.singular_values)
    assert np.array_equal(r1.factors.U, r2.factors.U)


@pytest.mark.parametrize("q", [0, 1, 2])
def test_prototype_matches_oracle_same_omega(ctx, q):
    rng = np.random.default_rng(q)
    m, n, k, s = 2048, 512, 20, 30
    u, _ = np.linalg.qr(rng.standard_normal((m, n)))
    v, _ = np.linalg.qr(rng.standard_normal((n, n)))
    sig = np.exp(-np.arange(1, n + 1) / 20.0)
    a = (u * sig) @ v.T + 1e-3 * rng.standard_normal((m, n))
    r = rn.prototype_ksvd(dev(a), k, s, 777, power_iters=q, ctx=ctx)
    uo, so, vo, passes = orc.prototype_ksvd(a, k, s, 777, q=q)
    assert r.passes_over_a == passes == 2 + 2 * q
    assert np.max(np.abs(r.factors.singular_values - so) / so) <= 1e-8
    U = r.factors.U.cpu().numpy()
    # the well-separated leading vectors agree up to rounding
    assert np.max(np.abs(np.abs(U[:, :3]) - np.abs(uo[:, :3]))) <= 1e-6


def test_prototype_fp32(ctx):
    rng = np.random.default_rng(3)
    m, n = 4096, 1024
    u, _ = np.linalg.qr(rng.standard_normal((m, 256)))
    v, _ = np.linalg.qr(rng.standard_normal((n, 256)))
    sig = np.arange(1, 257) ** -1.5
    a = ((u * sig) @ v.T + 1e-4 * rng.standard_normal((m, n))).astype(np.float32)
    r = rn.prototype_ksvd(dev(a), 20, 40, 5, power_iters=2, ctx=ctx)
    _, so, _, _ = orc.prototype_ksvd(a.astype(np.float64), 20, 40, 5, q=2)
    assert np.max(np.abs(r.factors.singular_values - so) / so) <= 1e-3


@pytest.mark.parametrize("m,n,s,q,order", [
    (19000, 2048, 150, 1, "C"),   # 149 row tiles (tail of 56 rows), 4 chunks of 512 k; A'Q split over K with a k tail
    (4096, 8192, 150, 0, "C"),    # several work items per persistent CTA (split K), 15 k-blocks each
    (5000, 3000, 137, 1, "F"),    # column-major A: the [64 k][128 rows] TMA box feeds Y = A Omega
    (9000, 1100, 160, 0, "C"),    # N = 160 tile, K not a multiple of 64
])
def test_prototype_fp32_wide_sketch_tmem_operand(ctx, m, n, s, q, order):
    """fp32 projections with 128 < s <= 160 run the A-in-TMEM tcgen05 kernel
    (gemm_tc.cu, gemm_bf16x3_ts_kernel); sigma against the fp64 oracle with the
    same Omega (src/randsvd.cpp:88-110), gate 1e-3 (north_star fp32)."""
    import torch
    rng = np.random.default_rng(m + n + s)
    r0 = 256
    u, _ = np.linalg.qr(rng.standard_normal((m, r0)))
    v, _ = np.linalg.qr(rng.standard_normal((n, r0)))
    sig = np.arange(1, r0 + 1) ** -1.5
    a = ((u * sig) @ v.T + 1e-4 * rng.standard_normal((m, n))).astype(np.float32)
    da = torch.from_numpy(a).cuda()
    if order == "F":
        da = da.t().contiguous().t()
    k = 100
    r = rn.prototype_ksvd(da, k, s, 11, power_iters=q, ctx=ctx)
    _, so, _, _ = orc.prototype_ksvd(a.astype(np.float64), k, s, 11, q=q)
    assert np.max(np.abs(r.factors.singular_values - so) / so) <= 1e-3
    # deterministic: the same call returns the same bits (the converter/TMA ring has no data race)
    r2 = rn.prototype_ksvd(da, k, s, 11, power_iters=q, ctx=ctx)
    assert np.array_equal(r.factors.singular_values, r2.factors.singular_values)
    assert torch.equal(r.factors.U, r2.factors.U)


def test_prototype_count_spec(ctx):
    a = orc.gaussian_matrix(300, 6, 8) @ orc.gaussian_matrix(6, 200, 9)
    r = rn.prototype_ksvd(a, 6, 30, 4, spec=rn.SketchSpec.count_sketch(30, 4), opts=rn.KsvdOptions(True), ctx=ctx)
    assert r.error_fro <= 1e-8 * np.linalg.norm(a)


def test_prototype_argument_checks(ctx):
    with pytest.raises(ValueError, match="k <= s <= min"):
        rn.prototype_ksvd(np.ones((10, 8)), 5, 9, 1, ctx=ctx)


def test_faster_ksvd_recovers_low_rank(ctx):
    # tests/test_randsvd.cpp:61-72
    a = orc.gaussian_matrix(120, 4, 6) @ orc.gaussian_matrix(4, 100, 60)
    r = rn.faster_ksvd(a, 4, 16, 256, 64, 9, opts=rn.KsvdOptions(True), ctx=ctx)
    assert r.error_fro <= 1e-6 * np.linalg.norm(a)
    assert r.passes_over_a == 2
    U = r.factors.U
    assert np.linalg.norm(U.T @ U - np.eye(U.shape[1])) <= 1e-8


def test_faster_ksvd_argument_checks(ctx):
    # tests/test_randsvd.cpp:74-79
    a = orc.gaussian_matrix(30, 30, 10)
    for args in [(5, 5, 40, 20), (5, 10, 20, 20), (5, 10, 15, 20)]:
        with pytest.raises(ValueError, match="k < s < p < p_cs"):
            rn.faster_ksvd(a, *args, 1, ctx=ctx)


@pytest.mark.parametrize("on_device", [False, True])
def test_faster_ksvd_matches_oracle(ctx, on_device):
    rng = np.random.default_rng(5)
    m, n, k, s, p_cs, p = 3000, 400, 10, 24, 512, 96
    u, _ = np.linalg.qr(rng.standard_normal((m, n)))
    v, _ = np.linalg.qr(rng.standard_normal((n, n)))
    sig = np.exp(-np.arange(1, n + 1) / 8.0)
    a = (u * sig) @ v.T + 1e-6 * rng.standard_normal((m, n))
    r = rn.faster_ksvd(dev(a) if on_device else a, k, s, p_cs, p, 31, opts=rn.KsvdOptions(True), ctx=ctx)
    uo, so, vo, passes = orc.faster_ksvd(a, k, s, p_cs, p, 31)
    assert r.passes_over_a == passes == 2
    sv = r.factors.singular_values
    assert sv.size == so.size
    assert np.max(np.abs(sv - so) / so) <= 1e-8
    U = r.factors.U.cpu().numpy() if on_device else r.factors.U
    V = r.factors.V.cpu().numpy() if on_device else r.factors.V
    assert np.max(np.abs(U[:, :3] - uo[:, :3])) <= 1e-6
    assert np.max(np.abs(V[:, :3] - vo[:, :3])) <= 1e-6
    ref_err = np.linalg.norm(a - (uo * so) @ vo.T)
    assert abs(r.error_fro - ref_err) <= 1e-8 * np.linalg.norm(a)


def test_faster_ksvd_fp32_input(ctx):
    a = (orc.gaussian_matrix(500, 6, 2) @ orc.gaussian_matrix(6, 300, 3)).astype(np.float32)
    r = rn.faster_ksvd(dev(a), 6, 12, 200, 48, 4, opts=rn.KsvdOptions(True), ctx=ctx)
    assert r.factors.U.dtype == torch.float32
    assert r.error_fro <= 1e-5 * np.linalg.norm(a.astype(np.float64))


def _ill_conditioned(n, d, seed, decades=5.0):
    rng = np.random.default_rng(seed)
    u, _ = np.linalg.qr(rng.standard_normal((n, d)))
    v, _ = np.linalg.qr(rng.standard_normal((d, d)))
    a = (u * 10.0 ** (-decades * np.arange(d) / (d - 1))) @ v.T
    return a, rng.standard_normal(n)


def test_lsr_preconditioned_reference_cases(ctx):
    # tests/test_regression.cpp:54-86
    a, _ = orc.thin_qr(orc.gaussian_matrix(300, 6, 10))
    b = orc.gaussian_matrix(300, 1, 11)[:, 0]
    sol = rn.lsr_preconditioned(a, b, 1e-10, 13, rn.PreconditionedOptions(sketch_size=120), ctx=ctx)
    exact = np.linalg.lstsq(a, b, rcond=None)[0]
    assert np.linalg.norm(sol.x - exact) <= 1e-8 * (np.linalg.norm(exact) + 1)
    assert sol.iterations <= 40 and sol.kappa_estimate <= 2.0
    a, b = _ill_conditioned(800, 10, 20)
    exact = np.linalg.lstsq(a, b, rcond=None)[0]
    for cg in (False, True):
        sol = rn.lsr_preconditioned(a, b, 1e-8, 22, rn.PreconditionedOptions(sketch_size=200, use_cg=cg), ctx=ctx)
        assert np.linalg.norm(sol.x - exact) <= 1e-7 * np.linalg.norm(exact)
        assert sol.iterations <= 80
    with pytest.raises(ValueError, match="eps out of"):
        rn.lsr_preconditioned(orc.gaussian_matrix(10, 4, 50), orc.gaussian_matrix(10, 1, 54), 2.0, 1, ctx=ctx)
    with pytest.raises(ValueError, match="n < d"):
        rn.lsr_preconditioned(orc.gaussian_matrix(3, 5, 50), orc.gaussian_matrix(3, 1, 54), 0.1, 1, ctx=ctx)


@pytest.mark.parametrize("kind,cg,dtype", [("count", False, np.float64), ("count", True, np.float64),
                                           ("gaussian", False, np.float64), ("srht", True, np.float64),
                                           ("count", False, np.float32)])
def test_lsr_preconditioned_matches_oracle(ctx, kind, cg, dtype):
    a, b = _ill_conditioned(20000, 48, 3, decades=4.0)
    a, b = a.astype(dtype), b.astype(dtype)
    kinds = {"count": rn.SketchKind.kCountSketch, "gaussian": rn.SketchKind.kGaussian, "srht": rn.SketchKind.kSrht}
    opts = rn.PreconditionedOptions(sketch_size=0, use_cg=cg, sketch_kind=kinds[kind])
    sol = rn.lsr_preconditioned(dev(a), dev(b), 1e-10, 99, opts, ctx=ctx)
    x, obj, it, kappa = orc.lsr_preconditioned(a.astype(np.float64), b.astype(np.float64), 1e-10, 99, kind=kind,
                                               use_cg=cg)
    tol = 1e-9 if dtype == np.float64 else 1e-5
    assert np.linalg.norm(sol.x - x) <= tol * np.linalg.norm(x)
    assert abs(sol.objective - obj) <= 1e-9 * obj
    # the gradient-descent stop ("gradient stalled at the rounding floor",
    # regression.cpp:159-166) is rounding-sensitive: the count may differ by a few
    assert abs(sol.iterations - it) <= max(2, it // 10)
    assert abs(sol.kappa_estimate - kappa) <= (1e-6 if dtype == np.float64 else 1e-4) * kappa


def test_lsr_preconditioned_large_d_fused_pass(ctx):
    # d = 512 (the config-1 width): the fused pass holds 16 fp64 per lane
    rng = np.random.default_rng(8)
    n, d = 60000, 512
    a = rng.standard_normal((n, d))
    b = a @ rng.standard_normal(d) + 0.1 * rng.standard_normal(n)
    sol = rn.lsr_preconditioned(dev(a), dev(b), 1e-12, 4, want_kappa=False, ctx=ctx)
    exact = np.linalg.lstsq(a, b, rcond=None)[0]
    assert np.linalg.norm(sol.x - exact) <= 1e-10 * np.linalg.norm(exact)
    r = a @ exact - b
    assert abs(sol.objective - r @ r) <= 1e-10 * (r @ r)
    assert sol.kappa_estimate is None


def test_lsr_cg_converges_to_exact(ctx):
    # tests/test_regression.cpp:34-42
    a = orc.gaussian_matrix(100, 10, 3)
    b = orc.gaussian_matrix(100, 1, 4)[:, 0]
    exact = np.linalg.lstsq(a, b, rcond=None)[0]
    cg = rn.lsr_cg(a, b, 1e-12, 200, ctx=ctx)
    assert cg.converged
    assert np.linalg.norm(cg.x - exact) <= 1e-8 * np.linalg.norm(exact)
    assert cg.iterations <= 11
    r = a @ exact - b
    assert abs(cg.objective - r @ r) <= 1e-10 * (r @ r)
