"""The NCCL transport on hardware: a world-1 rnla_ctx_create_dist context owns
a one-rank NCCL communicator, so every row-sharded code path (owner-reduced
Gaussian chunks, allreduced Grams / A'Q / B', global row offsets, the global
sign rule, allgathered landmark points) runs its real ncclReduce /
ncclAllReduce / ncclAllGather calls on the single GPU this build has. Results
must agree with the plain single-GPU context (bitwise for the count stage,
to rounding elsewhere). Multi-rank NCCL (world > 1, one process per GPU) is
the same code with more ranks; bench.py --gpus N launches it."""
import numpy as np
import pytest

import paper_1505_07570_b200 as rn
from oracle import oracle as orc

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def nctx():
    c = rn.Context(0, world=1, rank=0, nccl_id=rn.Context.nccl_unique_id())
    yield c
    c.close()


def _rel(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def test_nccl_world1_combined_sketch_and_lsr(ctx, nctx):
    rng = np.random.default_rng(11)
    n, d = 200_000, 63
    a = torch.from_numpy(rng.standard_normal((n, d))).cuda()
    b = torch.from_numpy(rng.standard_normal(n)).cuda()
    cs = rn.SketchSpec.count_sketch(4096, 3)
    spec = rn.SketchSpec.combined(4096, rn.SketchSpec.gaussian(512, 4), 3)
    assert torch.equal(rn.sketch_rows(a, cs, extra=b, ctx=nctx), rn.sketch_rows(a, cs, extra=b, ctx=ctx))
    y1 = rn.sketch_rows(a, spec, extra=b, ctx=nctx).cpu().numpy()
    y0 = rn.sketch_rows(a, spec, extra=b, ctx=ctx).cpu().numpy()
    assert _rel(y1, y0) <= 1e-13
    s1 = rn.lsr_sketched(a, b, spec, ctx=nctx)
    s0 = rn.lsr_sketched(a, b, spec, ctx=ctx)
    assert _rel(s1.x, s0.x) <= 1e-10 and abs(s1.objective - s0.objective) <= 1e-10 * s0.objective


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_nccl_world1_prototype_ksvd(ctx, nctx, dtype):
    rng = np.random.default_rng(12)
    m, n, k, s = 6000, 700, 10, 24
    a_np = (rng.standard_normal((m, 40)) * np.exp(-np.arange(40) / 6.0)) @ rng.standard_normal((40, n))
    a_np += 1e-3 * rng.standard_normal((m, n))
    a = torch.from_numpy(a_np).to(dtype).cuda()
    r1 = rn.prototype_ksvd(a, k, s, 21, power_iters=1, ctx=nctx)
    r0 = rn.prototype_ksvd(a, k, s, 21, power_iters=1, ctx=ctx)
    _, so, _, _ = orc.prototype_ksvd(a.double().cpu().numpy(), k, s, 21, q=1)
    tol = 1e-10 if dtype == torch.float64 else 1e-3
    assert np.max(np.abs(r1.factors.singular_values - so) / so) <= tol
    assert np.max(np.abs(r1.factors.singular_values - r0.factors.singular_values) / so) <= tol
    assert r1.passes_over_a == 4


def test_nccl_world1_srht_and_leverage(ctx, nctx):
    rng = np.random.default_rng(13)
    n, d, s = 1 << 16, 96, 512
    a = torch.from_numpy(rng.standard_t(3, size=(n, d)).astype(np.float32)).cuda()
    o1 = rn.sketch_rows(a, rn.SketchSpec.srht(s, 8), ctx=nctx).double().cpu().numpy()
    ref = orc.srht_rows(a.double().cpu().numpy(), s, 8)
    assert _rel(o1, ref) <= 1e-4
    sc1, ix1 = rn.leverage_sample_rows(a, s, 9, ctx=nctx)
    sc0, ix0 = rn.leverage_sample_rows(a, s, 9, ctx=ctx)
    assert np.max(np.abs(sc1 - sc0) / sc0) <= 1e-4
    assert np.array_equal(ix1, np.unique(orc.sample_with_replacement(sc1, s, 9)))


def test_nccl_world1_nystrom_eig(ctx, nctx):
    rng = np.random.default_rng(14)
    n, d, c, k = 20000, 16, 256, 8
    x = torch.from_numpy(rng.standard_normal((n, d)) * 2.0).cuda()
    view = rn.KernelView(x, rn.KernelSpec(4.0))
    _, l1, sel1, kept1 = rn.nystrom_eig(view, c, 5, c, k, want_vectors=False, ctx=nctx)
    _, l0, sel0, kept0 = rn.nystrom_eig(view, c, 5, c, k, want_vectors=False, ctx=ctx)
    assert np.array_equal(sel1, sel0) and kept1 == kept0
    assert np.max(np.abs(l1 - l0) / l0) <= 1e-8
