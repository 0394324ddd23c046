"""ctypes binding of the C ABI in include/rnla.h (librnla_b200.so).

Only plumbing: every compute entry point runs in the native library. The
library must have been built (``__graft_entry__.build()``); there is no
Python or CPU fallback, and loading fails loudly when it is missing.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# RNLA_LIB_PATH: load an alternative build of the same library (A/B kernel experiments).
LIB_PATH = os.environ.get("RNLA_LIB_PATH") or os.path.join(_HERE, "_lib", "librnla_b200.so")

RNLA_OK, RNLA_EINVAL, RNLA_ENUMERIC, RNLA_ECUDA, RNLA_ENCCL, RNLA_ENOMEM = range(6)
RNLA_F64, RNLA_F32 = 0, 1


class RnlaMat(C.Structure):
    _fields_ = [
        ("data", C.c_void_p),
        ("rows", C.c_int64),
        ("cols", C.c_int64),
        ("row_stride", C.c_int64),
        ("col_stride", C.c_int64),
        ("dtype", C.c_int32),
        ("on_device", C.c_int32),
    ]


class RnlaSketchSpec(C.Structure):
    _fields_ = [
        ("kind", C.c_int32),
        ("s", C.c_int64),
        ("seed", C.c_uint64),
        ("stage2_kind", C.c_int32),
        ("stage2_s", C.c_int64),
        ("stage2_seed", C.c_uint64),
        ("scale_columns", C.c_int32),
        ("leverage_rank", C.c_int64),
    ]


_P = C.c_void_p
_M = C.POINTER(RnlaMat)
_S = C.POINTER(RnlaSketchSpec)
_I64P = C.POINTER(C.c_int64)
_F64P = C.POINTER(C.c_double)
_I32P = C.POINTER(C.c_int32)
_I8P = C.POINTER(C.c_int8)
_U64P = C.POINTER(C.c_uint64)

# name -> (restype, argtypes); the exact list of symbols include/rnla.h declares.
SIGNATURES = {
    "rnla_abi_version": (C.c_int, []),
    "rnla_last_error": (C.c_char_p, []),
    "rnla_ctx_create": (C.c_int, [C.c_int, C.POINTER(_P)]),
    "rnla_ctx_create_dist": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_void_p, C.POINTER(_P)]),
    "rnla_group_create": (C.c_int, [C.c_int, C.POINTER(_P)]),
    "rnla_group_destroy": (None, [_P]),
    "rnla_ctx_create_grouped": (C.c_int, [C.c_int, _P, C.c_int, C.POINTER(_P)]),
    "rnla_nccl_unique_id": (C.c_int, [C.c_void_p]),
    "rnla_ctx_destroy": (None, [_P]),
    "rnla_ctx_synchronize": (C.c_int, [_P]),
    "rnla_ctx_wait_stream": (C.c_int, [_P, C.c_void_p]),
    "rnla_ctx_stream": (C.c_void_p, [_P]),
    "rnla_ctx_launch_count": (C.c_int64, [_P]),
    "rnla_ctx_clear_cache": (None, [_P]),
    "rnla_shard_rows": (None, [C.c_int64, C.c_int, C.c_int, _I64P, _I64P]),
    "rnla_splitmix64": (C.c_uint64, [_U64P]),
    "rnla_derive_seed": (C.c_uint64, [C.c_uint64, C.c_uint64]),
    "rnla_count_sketch_hashes": (C.c_int, [C.c_uint64, C.c_int64, C.c_int64, C.c_int64, _I64P, _I8P]),
    "rnla_gaussian_matrix": (C.c_int, [C.c_uint64, C.c_int64, C.c_int64, _F64P]),
    "rnla_sample_without_replacement": (C.c_int, [C.c_uint64, C.c_int64, C.c_int64, _I64P]),
    "rnla_sample_with_replacement": (C.c_int, [C.c_uint64, _F64P, C.c_int64, C.c_int64, _I64P]),
    "rnla_srht_operator": (C.c_int, [C.c_uint64, C.c_int64, C.c_int64, _I8P, _I64P]),
    "rnla_gaussian_sketch": (C.c_int, [_P, _M, C.c_int64, C.c_uint64, _M]),
    "rnla_srht_sketch": (C.c_int, [_P, _M, C.c_int64, C.c_uint64, _M]),
    "rnla_count_sketch": (C.c_int, [_P, _M, C.c_int64, C.c_uint64, _M]),
    "rnla_combined_sketch": (C.c_int, [_P, _M, _S, _M]),
    "rnla_apply_sketch": (C.c_int, [_P, _M, _S, _M, _I64P]),
    "rnla_sketch_output_cols": (C.c_int64, [_S, C.c_int64]),
    "rnla_sketch_rows": (C.c_int, [_P, _M, _M, _S, C.c_int64, _M]),
    "rnla_count_stream_begin": (C.c_int, [_P, C.c_int64, C.c_int64, C.c_int64, C.c_uint64, C.c_int32, C.POINTER(_P)]),
    "rnla_count_stream_push": (C.c_int, [_P, _M]),
    "rnla_count_stream_end": (C.c_int, [_P, _M]),
    "rnla_count_stream_abort": (None, [_P]),
    "rnla_fwht": (C.c_int, [_P, _M]),
    "rnla_uniform_sample_columns": (C.c_int, [_P, _M, C.c_int64, C.c_uint64, _M, _I64P]),
    "rnla_leverage_scores": (C.c_int, [_P, _M, C.c_int64, _F64P]),
    "rnla_leverage_sample_columns": (
        C.c_int, [_P, _M, C.c_int64, C.c_uint64, C.c_int64, C.c_int, _M, _I64P, _F64P, _I64P]),
    "rnla_leverage_sample_rows": (C.c_int, [_P, _M, C.c_int64, C.c_uint64, _F64P, _I64P, _I64P]),
    "rnla_thin_qr": (C.c_int, [_P, _M, _M, _M]),
    "rnla_condensed_svd": (C.c_int, [_P, _M, _M, _F64P, _M, _I64P]),
    "rnla_truncated_svd": (C.c_int, [_P, _M, C.c_int64, _M, _F64P, _M, _I64P]),
    "rnla_pseudo_inverse": (C.c_int, [_P, _M, C.c_double, _M]),
    "rnla_prototype_ksvd": (
        C.c_int, [_P, _M, C.c_int64, C.c_int64, C.c_uint64, _S, C.c_int32, _M, _F64P, _M, _I64P, _I32P, _F64P]),
    "rnla_faster_ksvd": (
        C.c_int, [_P, _M, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_uint64, _M, _F64P, _M, _I64P, _I32P, _F64P]),
    "rnla_lsr_sketched": (C.c_int, [_P, _M, _M, _S, _F64P, _F64P, _I32P]),
    "rnla_lsr_cg": (C.c_int, [_P, _M, _M, C.c_double, C.c_int32, _F64P, _F64P, _I32P, _I32P]),
    "rnla_lsr_preconditioned": (
        C.c_int, [_P, _M, _M, C.c_double, C.c_uint64, C.c_int64, C.c_int32, C.c_int32, _F64P, _F64P, _I32P, _F64P]),
    "rnla_rbf_kernel": (C.c_int, [_P, _M, _M, C.c_double, _M]),
    "rnla_nystrom": (C.c_int, [_P, _M, C.c_double, C.c_int64, C.c_uint64, C.c_int64, _M, _I64P, _I64P, _I64P]),
    "rnla_nystrom_dense": (C.c_int, [_P, _M, C.c_int64, C.c_uint64, C.c_int64, _M, _I64P, _I64P]),
    "rnla_nystrom_columns": (C.c_int, [_P, _M, _I64P, C.c_int64, _M, _I64P]),
    "rnla_approx_eig": (C.c_int, [_P, _M, C.c_int64, _M, _F64P]),
    "rnla_nystrom_eig": (
        C.c_int, [_P, _M, C.c_double, C.c_int64, C.c_uint64, C.c_int64, C.c_int64, _M, _F64P, _I64P, _I64P]),
    "rnla_spsd_faster": (
        C.c_int, [_P, _M, C.c_double, C.c_int64, C.c_int64, C.c_uint64, _M, _M, _I64P, _I64P, _I64P, _I32P]),
    "rnla_cur_faster_kernel": (
        C.c_int, [_P, _M, _M, C.c_double, C.c_int64, C.c_int64, C.c_uint64, _M, _M, _M, _I64P, _I64P, _I64P, _I64P,
                  _I64P, _I64P, _I64P, _I32P]),
    "rnla_spsd_faster_dense": (
        C.c_int, [_P, _M, C.c_int64, C.c_int64, C.c_uint64, _M, _M, _I64P, _I64P, _I64P, _I32P]),
}


def load(path: str = LIB_PATH) -> C.CDLL:
    if not os.path.exists(path):
        raise ImportError(
            f"librnla_b200.so not found at {path}: build it with "
            "`python -c 'import __graft_entry__ as g; g.build()'` (there is no CPU fallback)")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        _lib = load()
    return _lib
