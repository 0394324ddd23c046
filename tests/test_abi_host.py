"""CPU-side checks of the C ABI library (no GPU needed):

* librnla_b200.so loads and exports exactly what include/rnla.h declares;
* the host operator draws (libstdc++, like the reference) agree with the
  golden vectors and with the oracle's independent C restatement;
* argument checks mirror the reference's require() messages;
* without a GPU the compute entry points fail loudly (no CPU fallback).
"""
import os
import re
import subprocess

import numpy as np
import pytest

import paper_1505_07570_b200 as rn
from paper_1505_07570_b200 import _abi
from oracle import oracle as orc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "rnla.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rnla_[a-z0-9_]+)\s*\(", src)))


def test_header_and_binding_agree():
    assert declared_symbols() == sorted(_abi.SIGNATURES)


def test_library_exports_every_declared_symbol():
    out = subprocess.run(["nm", "-D", "--defined-only", _abi.LIB_PATH], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r"\bT (rnla_[a-z0-9_]+)", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    lib = _abi.lib()
    assert lib.rnla_abi_version() == 1


def test_library_is_sm100a():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _abi.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_host_seed_functions_match_oracle(golden):
    streams = [0, 1, 2, 3, 100, 101, 200, 201, 202, 203, 204]
    assert [str(rn.derive_seed(42, s)) for s in streams] == golden["derive_seed_42"]
    for st in [0, 1, 12345, 2**64 - 1]:
        assert rn.splitmix64(st) == orc.splitmix64(st)


def test_host_hashes_match_oracle():
    for seed, s, j0 in [(1, 9, 0), (orc.derive_seed(42, 201), 8192, 4_000_000), (77, 1000, 3)]:
        b1, g1 = rn.count_sketch_hashes(seed, 5000, s, j0)
        b2, g2 = orc.count_sketch_hashes(seed, 5000, s, j0)
        assert np.array_equal(b1, b2) and np.array_equal(g1.astype(np.float64), g2)


def test_host_gaussian_matrix_matches_golden_and_oracle(golden):
    a = rn.gaussian_matrix(5, 7, 1)
    assert np.array_equal(a.ravel(order="F"), np.array([float.fromhex(h) for h in golden["gaussian_seed1_5x7"]]))
    assert np.array_equal(rn.gaussian_matrix(333, 17, 99), orc.gaussian_matrix(333, 17, 99))


def test_host_sampling_matches_oracle(golden):
    for case in golden["swor"]:
        got = rn.sample_without_replacement(case["n"], case["count"], int(case["seed"]))
        assert np.array_equal(got, orc.sample_without_replacement(case["n"], case["count"], int(case["seed"])))
    w = np.random.default_rng(0).random(1000)
    assert np.array_equal(rn.sample_with_replacement(w, 300, 5), orc.sample_with_replacement(w, 300, 5))
    # zero weights, repeated draws (count > n) and ties: the sorted sweep must
    # return exactly upper_bound, in draw order
    w2 = np.random.default_rng(1).random(5000) ** 4
    w2[::7] = 0.0
    w2[-50:] = 0.0
    for seed, cnt in [(3, 1), (11, 4096), (12, 20000)]:
        assert np.array_equal(rn.sample_with_replacement(w2, cnt, seed), orc.sample_with_replacement(w2, cnt, seed))
    for case in golden["srht"]:
        sg, idx = rn.srht_operator(case["n"], case["s"], int(case["seed"]))
        assert sg.tolist() == case["signs"] and idx.tolist() == case["idx"]


def test_host_argument_checks_mirror_reference():
    with pytest.raises(ValueError, match="count > n"):
        rn.sample_without_replacement(5, 6, 1)
    with pytest.raises(ValueError, match="negative weight"):
        rn.sample_with_replacement(np.array([1.0, -1.0]), 3, 1)
    with pytest.raises(ValueError, match="all weights zero"):
        rn.sample_with_replacement(np.zeros(4), 3, 1)
    with pytest.raises(ValueError, match="s > padded dimension"):
        rn.srht_operator(100, 129, 1)
    with pytest.raises(ValueError, match="s < 1"):
        rn.count_sketch_hashes(1, 10, 0)


def test_shard_rows_partition():
    for n in [0, 1, 7, 4_194_304, 1_000_003]:
        for world in [1, 2, 3, 8]:
            spans = [rn.shard_rows(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            sizes = [e - b for b, e in spans]
            assert max(sizes) - min(sizes) <= 1


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(rn.CudaError):
        rn.Context(0)


def test_operand_views_with_negative_or_zero_strides_are_copied():
    """Inputs with negative / zero strides (a[::-1], np.flipud, broadcasts) are
    copied to a contiguous array before their rnla_mat is built; an rnla_mat is
    never described with a clamped stride (it would read the wrong elements)."""
    a = np.arange(12.0).reshape(4, 3)
    for view in (a[::-1], np.flipud(a), a[:, ::-1], np.broadcast_to(a[:1], (4, 3)), a[::2, ::-1]):
        v2 = rn._as2d(view)
        m = rn._mat(v2)
        got = np.array([[np.frombuffer((np.ctypeslib.as_array(
            (np.ctypeslib.ctypes.c_double * 1).from_address(m.data + 8 * (i * m.row_stride + j * m.col_stride))))
        )[0] for j in range(m.cols)] for i in range(m.rows)])
        assert np.array_equal(got, view)
        assert m.row_stride > 0 and m.col_stride > 0
    with pytest.raises(ValueError):
        rn._mat(a[::-1])


def test_wait_stream_without_gpu_fails_loudly():
    if rn._abi.lib() is None:  # pragma: no cover
        pytest.skip("library missing")
    import ctypes as C
    assert rn._abi.lib().rnla_ctx_wait_stream(None, C.c_void_p(0)) == _abi.RNLA_EINVAL
