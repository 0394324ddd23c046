"""GPU parity of the sketch operators and sketched least squares against the
CPU oracle, through the C ABI (librnla_b200.so).

Bars (BASELINE north_star): integer/index outputs and the fp64 count sketch /
SRHT bit-exact (same per-element operation order as the reference loops);
fp64 dense sketches rel-Frobenius <= 1e-10; fp32 <= 1e-4 against the fp64
oracle run on the fp32-rounded inputs.
"""
import os

import numpy as np
import pytest

import paper_1505_07570_b200 as rn
from oracle import oracle as orc

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def relf(a, b):
    return np.linalg.norm(np.asarray(a, dtype=np.float64) - b) / max(np.linalg.norm(b), 1e-300)


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


# ---------------------------------------------------------------- count sketch
@pytest.mark.parametrize("n,L,s", [(1, 1, 1), (2, 3, 1), (10, 5, 64), (1000, 7, 9), (20000, 33, 512),
                                   (5000, 130, 300), (3000, 513, 1024), (2000, 700, 100), (1500, 1300, 77)])
def test_count_sketch_rows_bit_exact(ctx, n, L, s):
    rng = np.random.default_rng(n + L + s)
    m = rng.standard_normal((n, L))
    seed = 1000 + s
    got = rn.sketch_rows(dev(m), rn.SketchSpec.count_sketch(s, seed), ctx=ctx).cpu().numpy()
    assert np.array_equal(got, orc.count_sketch_rows(m, s, seed))


def test_count_sketch_rows_with_extra_column_and_offset(ctx):
    rng = np.random.default_rng(1)
    m = rng.standard_normal((7000, 64))
    b = rng.standard_normal(7000)
    spec = rn.SketchSpec.count_sketch(256, 9)
    got = rn.sketch_rows(dev(m), spec, extra=dev(b), row_offset=123456, ctx=ctx).cpu().numpy()
    assert np.array_equal(got, orc.count_sketch_rows(m, 256, 9, extra=b, j0=123456))


def test_count_sketch_rows_host_streamed_matches(ctx, monkeypatch):
    # Host (numpy) input goes through the chunked H2D pipeline; chunks
    # accumulate in row order, so the result stays bit-identical.
    rng = np.random.default_rng(2)
    m = rng.standard_normal((9001, 40))
    b = rng.standard_normal(9001)
    monkeypatch.setenv("RNLA_STREAM_CHUNK_ROWS", "1000")
    got = rn.sketch_rows(m, rn.SketchSpec.count_sketch(128, 77), extra=b, ctx=ctx)
    assert np.array_equal(got, orc.count_sketch_rows(m, 128, 77, extra=b))


def test_count_sketch_fp32(ctx):
    rng = np.random.default_rng(3)
    m = rng.standard_normal((20000, 48)).astype(np.float32)
    got = rn.sketch_rows(dev(m), rn.SketchSpec.count_sketch(1000, 5), ctx=ctx).cpu().numpy()
    ref = orc.count_sketch_rows(m.astype(np.float64), 1000, 5)
    assert relf(got, ref) <= 1e-6


def test_count_sketch_column_semantics(ctx):
    # tests/test_sketch.cpp:47-64: C = A S equals A times the materialized operator.
    rng = np.random.default_rng(4)
    a = np.asfortranarray(rng.standard_normal((7, 40)))
    c = rn.count_sketch(a, 9, 77, ctx=ctx)
    assert np.array_equal(c, orc.count_sketch(a, 9, 77))
    op = orc.count_sketch_operator(40, 9, 77)
    assert np.linalg.norm(c - a @ op) <= 1e-14 * np.linalg.norm(a)
    # row-major host input and CUDA input give the same bits
    c2 = rn.count_sketch(np.ascontiguousarray(a), 9, 77, ctx=ctx)
    c3 = rn.count_sketch(dev(np.asfortranarray(a).T).t(), 9, 77, ctx=ctx).cpu().numpy()
    assert np.array_equal(c, c2) and np.array_equal(c, c3)


def test_count_sketch_norm_in_expectation(ctx):
    # tests/test_sketch.cpp:66-74
    a = orc.gaussian_matrix(10, 50, 3)
    tot = sum(np.linalg.norm(rn.count_sketch(a, 25, 5000 + t, ctx=ctx)) ** 2 for t in range(1000))
    assert abs(tot / 1000 / np.linalg.norm(a) ** 2 - 1) < 0.02


def test_count_sketch_large_s_with_empty_buckets(ctx):
    rng = np.random.default_rng(5)
    m = rng.standard_normal((50, 6))
    got = rn.sketch_rows(dev(m), rn.SketchSpec.count_sketch(4096, 3), ctx=ctx).cpu().numpy()
    ref = orc.count_sketch_rows(m, 4096, 3)
    assert np.array_equal(got, ref)
    assert np.count_nonzero(np.any(got != 0, axis=1)) <= 50


# ---------------------------------------------------------------- gaussian
@pytest.mark.parametrize("m,n,s", [(10, 50, 30), (64, 2048, 30), (300, 1000, 129), (5, 3, 2)])
def test_gaussian_sketch_fp64(ctx, m, n, s):
    rng = np.random.default_rng(m * n)
    a = rng.standard_normal((m, n))
    got = rn.gaussian_sketch(a, s, 77 + s, ctx=ctx)
    assert relf(got, orc.gaussian_sketch(a, s, 77 + s)) <= 1e-10


def test_gaussian_sketch_fp32(ctx):
    rng = np.random.default_rng(11)
    a = rng.standard_normal((256, 4096)).astype(np.float32)
    got = rn.gaussian_sketch(dev(a), 150, 9, ctx=ctx).cpu().numpy()
    assert relf(got, orc.gaussian_sketch(a.astype(np.float64), 150, 9)) <= 1e-4


@pytest.mark.parametrize("m,n,s,order", [(256, 16384, 150, "C"), (256, 16384, 150, "F"), (8192, 2048, 30, "C"),
                                         (3000, 4096, 160, "F"), (130, 700, 17, "C")])
def test_tcgen05_bf16x3_gemm_precision(ctx, m, n, s, order):
    # fp32 Gaussian sketch = A * Omega on tcgen05 (BF16x3 split, TMEM partial sums
    # promoted every 512 k): K-contiguous (C) and MN-contiguous (F) operands,
    # split-K and ragged tiles; error stays ~5e-6 independent of K.
    rng = np.random.default_rng(m + n)
    a = np.asarray(rng.standard_normal((m, n)), dtype=np.float32, order=order)
    ta = dev(a) if order == "C" else dev(np.ascontiguousarray(a.T)).t()
    got = rn.gaussian_sketch(ta, s, 31 + s, ctx=ctx).cpu().numpy()
    err = relf(got, orc.gaussian_sketch(a.astype(np.float64), s, 31 + s))
    assert err <= 2e-5, err


def test_gaussian_norm_in_expectation(ctx):
    # tests/test_sketch.cpp:37-45
    a = orc.gaussian_matrix(10, 50, 1)
    tot = sum(np.linalg.norm(rn.gaussian_sketch(a, 30, 1000 + t, ctx=ctx)) ** 2 for t in range(400))
    assert abs(tot / 400 / np.linalg.norm(a) ** 2 - 1) < 0.05


# ---------------------------------------------------------------- srht
@pytest.mark.parametrize("m,n,s", [(6, 100, 64), (1, 2, 1), (13, 1024, 1000), (40, 5000, 4096), (3, 70000, 300)])
def test_srht_sketch_fp64_bit_exact(ctx, m, n, s):
    rng = np.random.default_rng(m + n)
    a = rng.standard_normal((m, n))
    got = rn.srht_sketch(a, s, 11 + s, ctx=ctx)
    assert np.array_equal(got, orc.srht_sketch(a, s, 11 + s))


@pytest.mark.parametrize("n,L,s", [(1 << 18, 20, 1000), (300000, 9, 4096), ((1 << 21) - 5, 3, 333)])
def test_srht_register_path_fp64_bit_exact(ctx, n, L, s):
    # padded sizes 2^18 .. 2^22 take the register-blocked two-pass kernels
    rng = np.random.default_rng(n)
    m = rng.standard_normal((n, L))
    got = rn.sketch_rows(dev(m), rn.SketchSpec.srht(s, 5 + s), ctx=ctx).cpu().numpy()
    assert np.array_equal(got, orc.srht_rows(m, s, 5 + s))


def test_srht_register_path_fp32(ctx):
    rng = np.random.default_rng(21)
    m = rng.standard_t(3, size=((1 << 20), 40)).astype(np.float32)
    got = rn.sketch_rows(dev(m), rn.SketchSpec.srht(4096, 17), ctx=ctx).cpu().numpy()
    assert relf(got, orc.srht_rows(m.astype(np.float64), 4096, 17)) <= 1e-4


@pytest.mark.parametrize("n,L,s,ld", [(4096, 8, 4096, 8), (5000, 1, 1, 4), (70000, 40, 300, 40), (1 << 16, 100, 4096, 104),
                                      ((1 << 17) + 3, 33, 2048, 36), (1 << 18, 256, 4096, 256)])
def test_srht_onepass_fp32(ctx, n, L, s, ld):
    # srht_acc.cu: 4096-row tiles, sampled outputs accumulated in TMEM, runs that
    # cross 32-column quads flushed to partials. Checked against the fp64 oracle
    # and against the two-pass TMA kernels on the same operator.
    rng = np.random.default_rng(n + L)
    full = rng.standard_t(3, size=(n, ld)).astype(np.float32)
    m = torch.from_numpy(full).cuda()[:, :L]
    spec = rn.SketchSpec.srht(s, 900 + L)
    got = rn.sketch_rows(m, spec, ctx=ctx).cpu().numpy()
    ref = orc.srht_rows(full[:, :L].astype(np.float64), s, 900 + L)
    assert relf(got, ref) <= 1e-4
    os.environ["RNLA_SRHT_NO_ACC"] = "1"
    try:
        two = rn.sketch_rows(m, spec, ctx=ctx).cpu().numpy()
    finally:
        del os.environ["RNLA_SRHT_NO_ACC"]
    assert relf(got, two) <= 1e-5


def test_srht_onepass_many_runs(ctx):
    # 2^20 x 72: 3 quads x 256 tiles over 37 runs -> runs span quad boundaries
    rng = np.random.default_rng(3)
    m = rng.standard_normal(((1 << 20), 72)).astype(np.float32)
    got = rn.sketch_rows(dev(m), rn.SketchSpec.srht(4096, 5), ctx=ctx).cpu().numpy()
    assert relf(got, orc.srht_rows(m.astype(np.float64), 4096, 5)) <= 1e-4


def test_srht_rows_fp32(ctx):
    rng = np.random.default_rng(12)
    m = rng.standard_t(3, size=(1 << 14, 96)).astype(np.float32)
    got = rn.sketch_rows(dev(m), rn.SketchSpec.srht(512, 21), ctx=ctx).cpu().numpy()
    assert relf(got, orc.srht_rows(m.astype(np.float64), 512, 21)) <= 1e-4


def test_srht_shape_and_unbiased_scale(ctx):
    # tests/test_sketch.cpp:76-86
    a = orc.gaussian_matrix(6, 100, 4)
    c = rn.srht_sketch(a, 64, 11, ctx=ctx)
    assert c.shape == (6, 64)
    tot = sum(np.linalg.norm(rn.srht_sketch(a, 64, 9000 + t, ctx=ctx)) ** 2 for t in range(300))
    assert abs(tot / 300 / np.linalg.norm(a) ** 2 - 1) < 0.05


def test_srht_rejects_oversized_s(ctx):
    with pytest.raises(ValueError, match="s > padded dimension"):
        rn.srht_sketch(np.ones((2, 100)), 129, 1, ctx=ctx)


# ---------------------------------------------------------------- combined / apply
def test_combined_is_exact_composition(ctx):
    # tests/test_sketch.cpp:88-98: norm(c - gaussian_sketch(count_sketch(a))) == 0
    a = orc.gaussian_matrix(8, 200, 5)
    spec = rn.SketchSpec.combined(64, rn.SketchSpec.gaussian(16, 21), 20)
    c = rn.apply_sketch(a, spec, ctx=ctx)
    assert c.shape == (8, 16)
    mid = rn.count_sketch(a, 64, 20, ctx=ctx)
    assert np.linalg.norm(c - rn.gaussian_sketch(mid, 16, 21, ctx=ctx)) == 0.0
    assert relf(c, orc.combined_sketch(a, 64, 20, "gaussian", 16, 21)) <= 1e-10


@pytest.mark.parametrize("m", [100, 101])
def test_combined_is_exact_composition_large(ctx, m):
    # Gaussian stage large enough for the cp.async DMMA kernel (gemm_dmma.cu);
    # odd m makes the standalone call copy to 16-B aligned rows first.
    a = orc.gaussian_matrix(m, 3000, 9)
    spec = rn.SketchSpec.combined(512, rn.SketchSpec.gaussian(128, 33), 31)
    c = rn.apply_sketch(a, spec, ctx=ctx)
    mid = rn.count_sketch(a, 512, 31, ctx=ctx)
    assert np.linalg.norm(c - rn.gaussian_sketch(mid, 128, 33, ctx=ctx)) == 0.0
    assert relf(c, orc.combined_sketch(a, 512, 31, "gaussian", 128, 33)) <= 1e-10


@pytest.mark.parametrize("n,L,s_cs,s2", [(9000, 77, 1000, 100), (20000, 130, 4500, 70), (5000, 64, 4096, 64)])
def test_combined_rows_dmma_edges(ctx, n, L, s_cs, s2):
    # row-form combined sketch: K = s_cs not a multiple of the 16-k step, odd and
    # even L (16-B row padding of the intermediate), K split into 2048-bucket
    # chunks when s_cs >= 4096; bitwise equal to the two-step composition
    rng = np.random.default_rng(n + L)
    m = rng.standard_normal((n, L))
    b = rng.standard_normal(n)
    spec = rn.SketchSpec.combined(s_cs, rn.SketchSpec.gaussian(s2, 5), 4)
    got = rn.sketch_rows(dev(m), spec, extra=dev(b), ctx=ctx).cpu().numpy()
    mid = rn.sketch_rows(dev(m), rn.SketchSpec.count_sketch(s_cs, 4), extra=dev(b), ctx=ctx)
    two = rn.sketch_rows(mid, rn.SketchSpec.gaussian(s2, 5), ctx=ctx).cpu().numpy()
    assert np.array_equal(got, two)
    mid_ref = orc.count_sketch_rows(m, s_cs, 4, extra=b)
    ref = orc.gaussian_sketch(mid_ref.T, s2, 5).T
    assert relf(got, ref) <= 1e-10


def test_combined_srht_stage(ctx):
    a = orc.gaussian_matrix(9, 300, 6)
    spec = rn.SketchSpec.combined(100, rn.SketchSpec.srht(32, 8), 7)
    assert np.array_equal(rn.apply_sketch(a, spec, ctx=ctx), orc.combined_sketch(a, 100, 7, "srht", 32, 8))


def test_combined_rejects_bad_stage2(ctx):
    with pytest.raises(ValueError, match="s > s_cs"):
        rn.apply_sketch(np.ones((3, 50)), rn.SketchSpec.combined(10, rn.SketchSpec.gaussian(20, 1), 2), ctx=ctx)


def test_sketches_deterministic(ctx):
    # tests/test_sketch.cpp:170-182
    a = orc.gaussian_matrix(6, 80, 16)
    for spec in [rn.SketchSpec.gaussian(32, 55), rn.SketchSpec.srht(32, 55), rn.SketchSpec.count_sketch(32, 55)]:
        assert np.array_equal(rn.apply_sketch(a, spec, ctx=ctx), rn.apply_sketch(a, spec, ctx=ctx))


def test_uniform_columns_verbatim(ctx):
    a = orc.gaussian_matrix(5, 30, 6)
    c, sel = rn.uniform_sample_columns(a, 10, 99, ctx=ctx)
    assert np.array_equal(sel.indices, orc.sample_without_replacement(30, 10, 99))
    assert np.array_equal(c, a[:, sel.indices])


def test_leverage_columns(ctx):
    # tests/test_sketch.cpp:111-133
    low = orc.gaussian_matrix(12, 4, 7) @ orc.gaussian_matrix(4, 20, 8)
    sc = rn.leverage_scores(low, ctx=ctx)
    assert abs(sc.sum() - 4.0) < 4e-8 and sc.min() >= 0
    assert abs(rn.leverage_scores(low, 2, ctx=ctx).sum() - 2.0) < 2e-8
    assert np.allclose(sc, orc.leverage_scores(low), atol=1e-10)
    a = orc.gaussian_matrix(6, 25, 9)
    c, sel = rn.leverage_sample_columns(a, 15, 3, None, True, ctx=ctx)
    scores = orc.leverage_scores(a)
    draws = np.unique(orc.sample_with_replacement(scores, 15, 3))
    assert np.array_equal(sel.indices, draws)
    for t, j in enumerate(sel.indices):
        assert sel.weights[t] > 0
        assert np.linalg.norm(c[:, t] - sel.weights[t] * a[:, j]) <= 1e-12


def test_leverage_rows_given_identical_scores(ctx):
    rng = np.random.default_rng(13)
    m = rng.standard_t(3, size=(4096, 32))
    scores, idx = rn.leverage_sample_rows(dev(m), 512, 77, ctx=ctx)
    ref = orc.row_leverage(m)
    assert np.max(np.abs(scores - ref) / ref) <= 1e-8
    assert abs(scores.sum() - 32) < 1e-8
    # index draw bit-exact given identical scores (SURVEY §7 hard part 2)
    assert np.array_equal(idx, np.unique(orc.sample_with_replacement(scores, 512, 77)))
    m32 = m.astype(np.float32)
    s32, _ = rn.leverage_sample_rows(dev(m32), 512, 77, ctx=ctx)
    assert np.max(np.abs(s32 - orc.row_leverage(m32.astype(np.float64))) / ref) <= 1e-4


@pytest.mark.parametrize("n,d", [(20000, 200), (30000, 384), (9000, 1000)])
def test_leverage_rows_fp32_wide_tmem_operand(ctx, n, d):
    """fp32 row leverage with d > 160: the row norms of M R^-1 run on the A-in-TMEM
    tcgen05 kernel (128-column tiles; d = 200: tile pairs with a column tail, d = 384:
    odd tile count, d = 1000: four pairs). Scores against the fp64 oracle
    (src/spsd.cpp:150 pattern), fp32 gate 1e-4; draws bit-exact given the scores."""
    rng = np.random.default_rng(n + d)
    m32 = rng.standard_t(3, size=(n, d)).astype(np.float32)
    scores, idx = rn.leverage_sample_rows(dev(m32), 600, 5, ctx=ctx)
    ref = orc.row_leverage(m32.astype(np.float64))
    assert np.max(np.abs(scores - ref) / ref) <= 1e-4
    assert abs(scores.sum() - d) <= 1e-4 * d
    assert np.array_equal(idx, np.unique(orc.sample_with_replacement(scores, 600, 5)))
    s2, _ = rn.leverage_sample_rows(dev(m32), 600, 5, ctx=ctx)
    assert np.array_equal(scores, s2)


# ---------------------------------------------------------------- lsr_sketched
def test_lsr_sketched_count_matches_oracle(ctx):
    # tests/test_regression.cpp:44-52 + parity of x against the oracle on the same sketch
    a = orc.gaussian_matrix(2000, 10, 5)
    b = a @ orc.gaussian_matrix(10, 1, 6)[:, 0] + orc.gaussian_matrix(2000, 1, 7)[:, 0]
    spec = rn.SketchSpec.count_sketch(500, 9)
    sol = rn.lsr_sketched(a, b, spec, ctx=ctx)
    x_ref, obj_ref, flagged_ref = orc.lsr_sketched(a, b, orc.count_sketch_rows(a, 500, 9, extra=b))
    assert not sol.flagged and not flagged_ref
    assert np.linalg.norm(sol.x - x_ref) <= 1e-10 * np.linalg.norm(x_ref)
    assert abs(sol.objective - obj_ref) <= 1e-10 * obj_ref
    exact = np.linalg.lstsq(a, b, rcond=None)[0]
    e = float(np.sum((a @ exact - b) ** 2))
    assert e - 1e-9 <= sol.objective <= 1.5 * e


def test_lsr_sketched_combined_device(ctx):
    rng = np.random.default_rng(8)
    n, d = 100000, 64
    a = rng.standard_normal((n, d))
    b = a @ rng.standard_normal(d) + 0.01 * rng.standard_normal(n)
    seed = orc.derive_seed(42, 201)
    seed2 = orc.derive_seed(seed, 1)
    spec = rn.SketchSpec.combined(2048, rn.SketchSpec.gaussian(512, seed2), seed)
    sol = rn.lsr_sketched(dev(a), dev(b), spec, ctx=ctx)
    sk = orc.gaussian_sketch(orc.count_sketch_rows(a, 2048, seed, extra=b).T, 512, seed2).T
    x_ref, obj_ref, _ = orc.lsr_sketched(a, b, sk)
    assert np.linalg.norm(sol.x - x_ref) <= 1e-10 * np.linalg.norm(x_ref)
    assert abs(sol.objective - obj_ref) <= 1e-9 * obj_ref


def test_lsr_sketched_flags_rank_deficiency(ctx):
    rng = np.random.default_rng(9)
    a = rng.standard_normal((3000, 8))
    a[:, 7] = a[:, 0] + a[:, 1]  # rank 7
    b = rng.standard_normal(3000)
    sol = rn.lsr_sketched(a, b, rn.SketchSpec.count_sketch(200, 4), ctx=ctx)
    assert sol.flagged
    x_ref, obj_ref, flagged = orc.lsr_sketched(a, b, orc.count_sketch_rows(a, 200, 4, extra=b))
    assert flagged
    assert np.linalg.norm(sol.x - x_ref) <= 1e-8 * np.linalg.norm(x_ref)


def test_lsr_sketched_argument_checks(ctx):
    with pytest.raises(ValueError, match="s < d"):
        rn.lsr_sketched(np.ones((100, 10)), np.ones(100), rn.SketchSpec.count_sketch(5, 1), ctx=ctx)
    with pytest.raises(ValueError, match="dimension mismatch"):
        rn.lsr_sketched(np.ones((100, 10)), np.ones(99), rn.SketchSpec.count_sketch(50, 1), ctx=ctx)
