"""Fixtures produced by the REFERENCE'S OWN CODE: /root/reference/proj/src/
rng.cpp and src/sketch.cpp compiled unmodified against a minimal Eigen
stand-in (oracle/ref_shim, `make -C oracle ref` -> tests/golden/
ref_fixtures.json). The CPU oracle must reproduce them bit for bit (integer,
element-wise and libstdc++ stream outputs) or to rounding (the dense
Gaussian product, whose summation order is the shim's). The GPU path is
checked against the same fixtures in the -m gpu part of this file."""
import json
import os

import numpy as np
import pytest

from oracle import oracle as orc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def ref():
    with open(os.path.join(ROOT, "tests", "golden", "ref_fixtures.json")) as f:
        return json.load(f)


def mat(ref, key):
    e = ref[key]
    return np.array(e["colmajor"], dtype=np.float64).reshape((e["cols"], e["rows"])).T


def test_ref_rng_streams_on_one_engine(ref):
    g = orc.Engine(42)
    assert np.array_equal(g.gaussian_matrix(7, 3), mat(ref, "gaussian_matrix_seed42_7x3"))
    assert np.array_equal(g.gaussian_matrix(5, 2), mat(ref, "gaussian_matrix_seed42_then_5x2"))
    assert np.array_equal(g.gaussian_unit_vector(6), mat(ref, "gaussian_unit_vector_seed42_then_6")[:, 0])
    assert np.array_equal(g.sample_without_replacement(1000, 17),
                          ref["sample_without_replacement_seed42_then_1000_17"])
    w = np.array([0.5 + ((i * 37) % 11) for i in range(40)], dtype=np.float64)
    assert np.array_equal(orc.Engine(7).sample_with_replacement(w, 25), ref["sample_with_replacement_seed7_w40_25"])
    assert np.array_equal(orc.sample_with_replacement(w, 25, 7), ref["sample_with_replacement_seed7_w40_25"])
    # the seed-taking oracle entry points = fresh engines
    assert np.array_equal(orc.gaussian_matrix(7, 3, 42), mat(ref, "gaussian_matrix_seed42_7x3"))


def test_ref_sketches_bitexact(ref):
    a = mat(ref, "A_6x300")
    assert np.array_equal(a, orc.gaussian_matrix(6, 300, 5))
    assert np.array_equal(orc.count_sketch(a, 32, 11), mat(ref, "count_sketch_s32_seed11"))
    assert np.array_equal(orc.count_sketch(a, 7, 3), mat(ref, "count_sketch_s7_seed3"))
    assert np.array_equal(orc.count_sketch_operator(40, 9, 77), mat(ref, "count_sketch_operator_n40_s9_seed77"))
    assert np.array_equal(orc.srht_sketch(a, 64, 13), mat(ref, "srht_sketch_s64_seed13"))
    assert np.array_equal(orc.srht_sketch(a, 512, 2), mat(ref, "srht_sketch_s512_seed2"))
    x = np.array([np.sin(0.1 * i) + 0.01 * i for i in range(64)])
    assert np.array_equal(orc.fwht(x), mat(ref, "fwht_sin64")[:, 0])
    idx = orc.sample_without_replacement(300, 25, 31)
    assert np.array_equal(idx, ref["uniform_sample_columns_s25_seed31_indices"])
    assert np.array_equal(a[:, idx], mat(ref, "uniform_sample_columns_s25_seed31"))


def test_ref_dense_stages_to_rounding(ref):
    a = mat(ref, "A_6x300")
    g = mat(ref, "gaussian_sketch_s20_seed17")
    assert np.linalg.norm(orc.gaussian_sketch(a, 20, 17) - g) <= 1e-14 * np.linalg.norm(g)
    c = mat(ref, "combined_count64_gauss16")
    assert np.linalg.norm(orc.combined_sketch(a, 64, 20, "gaussian", 16, 21) - c) <= 1e-14 * np.linalg.norm(c)
    c = mat(ref, "combined_count64_srht16")
    assert np.array_equal(orc.combined_sketch(a, 64, 20, "srht", 16, 23), c)


@pytest.mark.gpu
def test_gpu_matches_reference_run(ref, ctx):
    """The CUDA path (through the C ABI) against the reference-run outputs."""
    import paper_1505_07570_b200 as rn
    a = mat(ref, "A_6x300")
    assert np.array_equal(rn.count_sketch(a, 32, 11, ctx=ctx), mat(ref, "count_sketch_s32_seed11"))
    assert np.array_equal(rn.count_sketch(a, 7, 3, ctx=ctx), mat(ref, "count_sketch_s7_seed3"))
    assert np.array_equal(rn.srht_sketch(a, 64, 13, ctx=ctx), mat(ref, "srht_sketch_s64_seed13"))
    assert np.array_equal(rn.srht_sketch(a, 512, 2, ctx=ctx), mat(ref, "srht_sketch_s512_seed2"))
    g = mat(ref, "gaussian_sketch_s20_seed17")
    assert np.linalg.norm(rn.gaussian_sketch(a, 20, 17, ctx=ctx) - g) <= 1e-13 * np.linalg.norm(g)
    spec = rn.SketchSpec.combined(64, rn.SketchSpec.gaussian(16, 21), 20)
    c = mat(ref, "combined_count64_gauss16")
    assert np.linalg.norm(rn.combined_sketch(a, spec, ctx=ctx) - c) <= 1e-13 * np.linalg.norm(c)
    spec = rn.SketchSpec.combined(64, rn.SketchSpec.srht(16, 23), 20)
    assert np.array_equal(rn.combined_sketch(a, spec, ctx=ctx), mat(ref, "combined_count64_srht16"))
    c, sel = rn.uniform_sample_columns(a, 25, 31, ctx=ctx)
    assert np.array_equal(sel.indices, ref["uniform_sample_columns_s25_seed31_indices"])
    assert np.array_equal(c, mat(ref, "uniform_sample_columns_s25_seed31"))
    x = np.array([np.sin(0.1 * i) + 0.01 * i for i in range(64)])
    rn.fwht_inplace(x, ctx=ctx)
    assert np.array_equal(x, mat(ref, "fwht_sin64")[:, 0])
    assert np.array_equal(rn.gaussian_matrix(7, 3, 42), mat(ref, "gaussian_matrix_seed42_7x3"))
    w = np.array([0.5 + ((i * 37) % 11) for i in range(40)], dtype=np.float64)
    assert np.array_equal(rn.sample_with_replacement(w, 25, 7), ref["sample_with_replacement_seed7_w40_25"])
