"""Full-size parity: every BASELINE.json configuration at its own size, GPU
path (through the C ABI) against the CPU oracle on identical inputs and
identical random operators. Gates are north_star's:

* integer / index outputs bit-exact (count-sketch stage, SRHT sample set,
  Nystrom landmarks, leverage indices given identical scores);
* sketches rel-F <= 1e-10 (fp64) / <= 1e-4 (fp32);
* top-k singular values / eigenvalues rel <= 1e-8 (fp64) / <= 1e-3 (fp32);
* config 1's solution x rel <= 1e-10.

Reference code paths (under /root/reference/proj): src/regression.cpp:68-92
(lsr_sketched), src/sketch.cpp:57-123 (SRHT / count / combined),
src/spsd.cpp:150-155 (row leverage), src/randsvd.cpp:88-110 (+ SURVEY A.6
power iterations), src/spsd.cpp:181-265 (nystrom + approx_eig).
"""
import gc
import math

import numpy as np
import pytest

import workloads as wl
from oracle import oracle as orc

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

THREADS = wl.host_threads()


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))


@pytest.fixture(autouse=True)
def _free():
    yield
    gc.collect()
    torch.cuda.empty_cache()


def test_cfg1_fullsize_count_stage_bitexact_and_lsr_sketched(ctx):
    """cfg1 at n = 4,194,304 x 512 fp64: the CountSketch stage of [A, b] is
    bit-identical to the reference's j-ascending loop; the combined sketch is
    within 1e-10 of the oracle's Gaussian stage; lsr_sketched's x within 1e-10
    of the oracle's solve on its own sketch."""
    import paper_1505_07570_b200 as rn
    n, d, s_cs, s2 = wl.CFG1["n"], wl.CFG1["d"], wl.CFG1["s_cs"], wl.CFG1["s"]
    seed = wl.op_seed(1)
    seed2 = orc.derive_seed(seed, 1)
    a, b, xstar = wl.cfg1_host()
    da, db = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    cs = rn.sketch_rows(da, rn.SketchSpec.count_sketch(s_cs, seed), extra=db, ctx=ctx).cpu().numpy()
    ref_cs = orc.count_sketch_rows(a, s_cs, seed, extra=b, threads=THREADS)
    assert np.array_equal(cs, ref_cs), "count stage differs from the reference loop"
    spec = rn.SketchSpec.combined(s_cs, rn.SketchSpec.gaussian(s2, seed2), seed)
    comb = rn.sketch_rows(da, spec, extra=db, ctx=ctx).cpu().numpy()
    ref_comb = orc.gaussian_sketch(ref_cs.T, s2, seed2).T
    e = _rel(comb, ref_comb)
    assert e <= 1e-10, e
    sol = rn.lsr_sketched(da, db, spec, ctx=ctx)
    x_ref, obj_ref, flagged_ref = orc.lsr_sketched(a, b, ref_comb)
    assert not sol.flagged and not flagged_ref
    ex = _rel(sol.x, x_ref)
    assert ex <= 1e-10, ex
    assert abs(sol.objective - obj_ref) <= 1e-10 * obj_ref
    # statistical sanity of the sketch-and-solve (tests/test_regression.cpp:44-52 style)
    assert _rel(sol.x, xstar) < 1e-3


def test_cfg0_fullsize_prototype_ksvd_q1(ctx):
    """cfg0: prototype_ksvd fp64 8192 x 2048, k = 20, s = 30, q = 1 against the
    same-algorithm oracle on the identical Omega: sigma rel <= 1e-8, and the
    singular vectors (sign convention of src/core.cpp:15-33) agree."""
    import paper_1505_07570_b200 as rn
    c = wl.CFG0
    a = wl.cfg0_host()
    res = rn.prototype_ksvd(torch.from_numpy(a).cuda(), c["k"], c["s"], wl.op_seed(0), power_iters=c["q"], ctx=ctx)
    uo, so, vo, passes = orc.prototype_ksvd(a, c["k"], c["s"], wl.op_seed(0), q=c["q"])
    sv = res.factors.singular_values
    err = float(np.max(np.abs(sv - so) / so))
    assert err <= 1e-8, err
    assert res.passes_over_a == passes == 4
    u = res.factors.U.cpu().numpy()
    v = res.factors.V.cpu().numpy()
    assert float(np.max(np.abs(u - uo))) <= 1e-8
    assert float(np.max(np.abs(v - vo))) <= 1e-8


def test_cfg2_fullsize_srht_all_columns(ctx):
    """cfg2 SRHT: fp32 2^20 x 1024 -> 4096, all 1024 columns against the
    reference's sign/FWHT/sample loop (fp64 on the fp32 input): rel-F <= 1e-4;
    the operator (signs then sorted indices from one engine) bit-exact."""
    import paper_1505_07570_b200 as rn
    n, d, s = wl.CFG2["n"], wl.CFG2["d"], wl.CFG2["s"]
    A = wl.cfg2_device()
    out = rn.sketch_rows(A, rn.SketchSpec.srht(s, wl.op_seed(2)), ctx=ctx)
    got = out.double().cpu().numpy()
    a64 = A.double().cpu().numpy()
    ref = orc.srht_rows(a64, s, wl.op_seed(2), threads=THREADS)
    e = _rel(got, ref)
    assert e <= 1e-4, e
    col_err = np.linalg.norm(got - ref, axis=0) / np.linalg.norm(ref, axis=0)
    assert float(col_err.max()) <= 1e-4
    sg, idx = rn.srht_operator(n, s, wl.op_seed(2))
    sg_o, idx_o = orc.srht_operator(n, s, wl.op_seed(2))
    assert np.array_equal(sg.astype(np.float64), sg_o) and np.array_equal(idx, idx_o)


def test_cfg2_fullsize_leverage_rows(ctx):
    """cfg2 leverage: all 2^20 row scores ||Q_i||^2 (Q = thin_qr(A).Q, the
    src/spsd.cpp:150 pattern) within 1e-4 (fp32) of the fp64 oracle; the 4096
    draws (sorted, unique) bit-exact given identical scores."""
    import paper_1505_07570_b200 as rn
    n, d, s = wl.CFG2["n"], wl.CFG2["d"], wl.CFG2["s"]
    A = wl.cfg2_device()
    seed = orc.derive_seed(wl.op_seed(2), 2)
    scores, idx = rn.leverage_sample_rows(A, s, seed, ctx=ctx)
    a64 = A.double().cpu().numpy()
    del A
    # ||Q_i||^2 = ||a_i R^-1||^2 for any R with R'R = A'A (Fact 6)
    import scipy.linalg as sla
    r = np.linalg.cholesky(a64.T @ a64).T
    ref = np.einsum("ij,ij->i", *(2 * [sla.solve_triangular(r, a64.T, trans="T", lower=False).T]))
    rel = np.abs(scores - ref) / ref
    assert float(rel.max()) <= 1e-4, float(rel.max())
    assert abs(scores.sum() - d) <= 1e-3 * d
    draws = np.unique(orc.sample_with_replacement(scores, s, seed))
    assert np.array_equal(idx, draws)


def test_cfg3_fullsize_prototype_ksvd_q2(ctx):
    """cfg3: prototype_ksvd fp32 262144 x 16384, k = 100, s = 150, q = 2 with
    re-orthonormalization against the fp64 oracle of the same algorithm on the
    fp32-rounded input and the identical Omega: sigma rel <= 1e-3."""
    import paper_1505_07570_b200 as rn
    c = wl.CFG3
    A = wl.cfg3_device()
    res = rn.prototype_ksvd(A, c["k"], c["s"], wl.op_seed(3), power_iters=c["q"], ctx=ctx)
    sv = res.factors.singular_values.copy()
    u_top = res.factors.U[:, :4].double().cpu().numpy()
    del res
    a64 = np.empty(A.shape, dtype=np.float64)
    step = 1 << 14
    for r0 in range(0, A.shape[0], step):
        a64[r0:r0 + step] = A[r0:r0 + step].double().cpu().numpy()
    del A
    torch.cuda.empty_cache()
    uo, so, _, passes = orc.prototype_ksvd(a64, c["k"], c["s"], wl.op_seed(3), q=c["q"])
    err = float(np.max(np.abs(sv - so) / so))
    assert err <= 1e-3, err
    assert passes == 6
    # the separated top singular vectors agree (the bulk is ill-determined, SURVEY hard part 9)
    assert float(np.max(np.abs(np.abs(np.sum(u_top * uo[:, :4], axis=0)) - 1.0))) <= 1e-3


def test_cfg4_fullsize_nystrom_top64(ctx):
    """cfg4: Nystrom of the RBF kernel, n = 131072 points in 64 dims, c = 2048
    uniform landmarks, W+ at the reference floor (target_k = c), then the top 64
    eigenvalues of C W+ C^T: landmarks bit-exact, lambda rel <= 1e-3 (fp32)."""
    import paper_1505_07570_b200 as rn
    c = wl.CFG4
    X, sigma = wl.cfg4_device()
    view = rn.KernelView(X, rn.KernelSpec(sigma))
    _, lam, sel, kept = rn.nystrom_eig(view, c["c"], wl.op_seed(4), c["c"], c["k"], want_vectors=False, ctx=ctx)
    lam_o, sel_o, kept_o = wl.nystrom_oracle_lambda(X.double().cpu().numpy(), sigma, c["c"], wl.op_seed(4), c["k"])
    assert np.array_equal(np.sort(sel), np.sort(sel_o))
    # kept (eigenvalues of W above eps * lam_max * n) may differ in the noise-level
    # tail: fp32 kernel entries perturb W's smallest eigenvalues by ~1e-7 lam_max
    assert kept > 0 and kept_o > 0
    err = float(np.max(np.abs(lam - lam_o) / lam_o))
    assert err <= 1e-3, err


def test_torch_stream_inputs_are_ordered(ctx):
    """an input still being written by torch's current stream is
    complete before the library's stream reads it (rnla_ctx_wait_stream)."""
    import paper_1505_07570_b200 as rn
    n, d, s = 1 << 20, 64, 1024
    for trial in range(3):
        big = torch.randn(8192, 8192, device="cuda")
        A = torch.empty(n, d, dtype=torch.float64, device="cuda")
        for _ in range(4):
            big = big @ big  # keep torch's stream busy
        A.fill_(1.0 + trial)
        out = rn.sketch_rows(A, rn.SketchSpec.count_sketch(s, 5), ctx=ctx)
        torch.cuda.synchronize()
        ref = rn.sketch_rows(A, rn.SketchSpec.count_sketch(s, 5), ctx=ctx)
        assert torch.equal(out, ref)
        del big
