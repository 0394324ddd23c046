"""Reference entry points that are not whole-matrix sketches, through the
Python mirror of the C ABI: count_sketch_stream (src/sketch.cpp:83-92),
fwht_inplace (:44-55), nystrom on a dense K and on caller-evaluated columns
(src/spsd.cpp:181-228)."""
import numpy as np
import pytest

import paper_1505_07570_b200 as rn
from oracle import oracle as orc

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.mark.parametrize("m,n,s,chunk", [(13, 5000, 64, 777), (1, 10, 3, 4), (40, 70000, 1000, 4096)])
def test_count_sketch_stream_bitexact(ctx, m, n, s, chunk):
    a = np.asfortranarray(np.random.default_rng(m).standard_normal((m, n)))
    calls = []

    def column(j):
        calls.append(j)
        return a[:, j]

    c = rn.count_sketch_stream(m, n, s, 17, column, chunk=chunk, ctx=ctx)
    assert calls == list(range(n))  # called exactly once per j, in order
    assert np.array_equal(c, orc.count_sketch(a, s, 17))


def test_count_sketch_stream_errors(ctx):
    with pytest.raises(ValueError):
        rn.count_sketch_stream(3, 5, 0, 1, lambda j: np.zeros(3), ctx=ctx)
    with pytest.raises(ValueError):  # wrong column length
        rn.count_sketch_stream(3, 5, 2, 1, lambda j: np.zeros(4), ctx=ctx)


@pytest.mark.parametrize("n,cols", [(1, 1), (2, 3), (8, 1), (4096, 2), (1 << 16, 3), (1 << 20, 1)])
def test_fwht_inplace_bitexact(ctx, n, cols):
    x = np.asfortranarray(np.random.default_rng(n).standard_normal((n, cols)))
    ref = np.column_stack([orc.fwht(x[:, j]) for j in range(cols)])
    y = x.copy(order="F")
    rn.fwht_inplace(y, ctx=ctx)
    assert np.array_equal(y, ref)
    d = torch.from_numpy(x).cuda()
    rn.fwht_inplace(d, ctx=ctx)
    assert np.array_equal(d.cpu().numpy(), ref)
    e = np.zeros(8)
    e[0] = 1.0
    rn.fwht_inplace(e, ctx=ctx)
    assert np.all(e == 1.0)  # SPEC.md:147 known answer
    with pytest.raises(ValueError):
        rn.fwht_inplace(np.zeros(6), ctx=ctx)


def test_nystrom_dense_and_columns_match_oracle(ctx):
    rng = np.random.default_rng(3)
    x = rng.standard_normal((300, 4))
    sigma = 1.5
    K = orc.rbf_kernel(x, x, sigma)
    f = rn.nystrom(K, 30, 77, ctx=ctx)
    Lo, sel_o, _ = orc.nystrom(x, sigma, 30, 77)
    assert np.array_equal(f.selected, sel_o)
    Kd = np.array(K)
    Lref = Kd[:, sel_o]
    w = Lref[sel_o]
    lam, vec = np.linalg.eigh(0.5 * (w + w.T))
    kk = 24
    top = vec[:, ::-1][:, :kk] / np.sqrt(lam[::-1][:kk])
    Lexp = Lref @ top
    assert f.L.shape[1] == kk
    assert np.linalg.norm(f.L @ f.L.T - Lexp @ Lexp.T) <= 1e-8 * np.linalg.norm(Lexp @ Lexp.T)
    g = rn.nystrom_columns(Kd[:, f.selected], f.selected, ctx=ctx)
    assert np.linalg.norm(g.L @ g.L.T - f.L @ f.L.T) <= 1e-12 * np.linalg.norm(f.L @ f.L.T)
    with pytest.raises(ValueError):
        rn.nystrom(K[:, :200], 30, 77, ctx=ctx)
    with pytest.raises(ValueError):
        rn.nystrom_columns(Kd[:, f.selected], f.selected[::-1].copy(), ctx=ctx)
