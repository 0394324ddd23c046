"""paper_1505_07570_b200 -- B200-native randomized sketch / rSVD / Nystrom core.

Python mirror of the reference `randnla` C++ API
(/root/reference/proj/include/randnla/{rng,sketch,core,randsvd,regression,spsd}.hpp):
same function names, argument meaning, results and error behaviour
(std::invalid_argument -> ValueError, std::runtime_error -> NumericError).
Every compute call goes through the C ABI of include/rnla.h into
librnla_b200.so (sm_100a CUDA kernels); there is no CPU fallback.

Matrices are 2-D numpy arrays (host memory; the library moves them over
PCIe) or torch tensors (CUDA tensors stay on the device). Results come back
in the same kind of container, column-major like Eigen for functions with
reference semantics and row-major for sketch_rows.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import enum
import math
from typing import Optional, Tuple

import numpy as np

from . import _abi

__all__ = [
    "Context", "ShardGroup", "default_context", "SketchKind", "SketchSpec", "ColumnSelection", "SvdFactors", "QrFactors",
    "KsvdResult", "KsvdOptions", "LsrSolution", "KernelSpec", "KernelView", "NystromFactor", "NumericError",
    "CudaError", "splitmix64", "derive_seed", "count_sketch_hashes", "gaussian_matrix",
    "sample_without_replacement", "sample_with_replacement", "srht_operator", "gaussian_sketch", "srht_sketch",
    "count_sketch", "count_sketch_stream", "fwht_inplace", "nystrom_columns", "combined_sketch", "apply_sketch", "sketch_rows", "uniform_sample_columns", "leverage_scores",
    "leverage_sample_columns", "leverage_sample_rows", "thin_qr", "condensed_svd", "truncated_svd",
    "pseudo_inverse", "prototype_ksvd", "faster_ksvd", "lsr_sketched", "lsr_cg", "lsr_preconditioned", "PreconditionedOptions", "rbf_kernel", "nystrom", "approx_eig", "nystrom_eig", "SpsdSketch", "spsd_faster", "CurFactors", "cur_faster_kernel",
    "shard_rows",
]


class NumericError(RuntimeError):
    """The reference's std::runtime_error (numerical failure)."""


class CudaError(RuntimeError):
    """CUDA / NCCL / allocation failure inside the native library."""


def _check(status: int) -> None:
    if status == _abi.RNLA_OK:
        return
    msg = (_abi.lib().rnla_last_error() or b"").decode()
    if status == _abi.RNLA_EINVAL:
        raise ValueError(msg)
    if status == _abi.RNLA_ENUMERIC:
        raise NumericError(msg)
    raise CudaError(f"status {status}: {msg}")


# --------------------------------------------------------------------------
# context
# --------------------------------------------------------------------------
class ShardGroup:
    """In-process shard group (rnla_group): `world` contexts driven by `world`
    host threads; collectives are staged through host memory and summed in rank
    order. Create one Context per rank with ``Context(device, group=g, rank=r)``."""

    def __init__(self, world: int):
        h = C.c_void_p()
        _check(_abi.lib().rnla_group_create(int(world), C.byref(h)))
        self._h = h
        self.world = int(world)

    @property
    def handle(self):
        return self._h

    def close(self) -> None:
        if getattr(self, "_h", None):
            _abi.lib().rnla_group_destroy(self._h)
            self._h = None


class Context:
    """One CUDA device: stream, workspace and cached operators (rnla_ctx)."""

    def __init__(self, device: int = 0, world: int = 1, rank: int = 0, nccl_id: Optional[bytes] = None,
                 group: Optional[ShardGroup] = None):
        lib = _abi.lib()
        h = C.c_void_p()
        if group is not None:
            _check(lib.rnla_ctx_create_grouped(device, group.handle, rank, C.byref(h)))
            world = group.world
        elif world > 1 or nccl_id is not None:
            buf = C.create_string_buffer(bytes(nccl_id), 128)
            _check(lib.rnla_ctx_create_dist(device, world, rank, buf, C.byref(h)))
        else:
            _check(lib.rnla_ctx_create(device, C.byref(h)))
        self._h = h
        self.device, self.world, self.rank = device, world, rank

    @property
    def handle(self):
        return self._h

    @property
    def stream(self) -> int:
        return _abi.lib().rnla_ctx_stream(self._h) or 0

    def synchronize(self) -> None:
        _check(_abi.lib().rnla_ctx_synchronize(self._h))

    def launch_count(self) -> int:
        return int(_abi.lib().rnla_ctx_launch_count(self._h))

    def clear_cache(self) -> None:
        _abi.lib().rnla_ctx_clear_cache(self._h)

    def close(self) -> None:
        if getattr(self, "_h", None):
            _abi.lib().rnla_ctx_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover - interpreter teardown order varies
        try:
            self.close()
        except Exception:
            pass

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        _check(_abi.lib().rnla_nccl_unique_id(buf))
        return buf.raw


_default: Optional[Context] = None


def default_context() -> Context:
    global _default
    if _default is None:
        dev = 0
        try:
            import torch
            if torch.cuda.is_available():
                dev = torch.cuda.current_device()
        except Exception:
            pass
        _default = Context(dev)
    return _default


def shard_rows(n: int, world: int, rank: int) -> Tuple[int, int]:
    """Row block [begin, end) of `rank` (rnla_shard_rows)."""
    b, e = C.c_int64(), C.c_int64()
    _abi.lib().rnla_shard_rows(n, world, rank, C.byref(b), C.byref(e))
    return b.value, e.value


# --------------------------------------------------------------------------
# operands
# --------------------------------------------------------------------------
def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def _dtype_code(x) -> int:
    if _is_torch(x):
        import torch
        if x.dtype == torch.float64:
            return _abi.RNLA_F64
        if x.dtype == torch.float32:
            return _abi.RNLA_F32
    else:
        if x.dtype == np.float64:
            return _abi.RNLA_F64
        if x.dtype == np.float32:
            return _abi.RNLA_F32
    raise ValueError(f"unsupported dtype {x.dtype}: float64 or float32 required")


def _mat(x) -> _abi.RnlaMat:
    """rnla_mat view of a 1-D (n x 1) or 2-D numpy array / torch tensor.
    Strides must be positive (inputs pass through _as2d, which copies views
    with negative or zero strides; an output with such strides is rejected)."""
    if _is_torch(x):
        if x.dim() == 1:
            rows, cols, rs, cs = x.shape[0], 1, x.stride(0), 1
        else:
            rows, cols = x.shape
            rs, cs = x.stride()
        rs = rs if rows > 1 else max(rs, 1)
        cs = cs if cols > 1 else max(cs, 1)
        if rs <= 0 or cs <= 0:
            raise ValueError("matrix view with a zero stride: pass a contiguous tensor")
        return _abi.RnlaMat(x.data_ptr(), rows, cols, rs, cs, _dtype_code(x), 1 if x.is_cuda else 0)
    a = x
    if a.ndim == 1:
        rows, cols = a.shape[0], 1
        rs, cs = a.strides[0], a.itemsize
    else:
        rows, cols = a.shape
        rs, cs = a.strides
    if rows <= 1:
        rs = max(rs, a.itemsize)
    if cols <= 1:
        cs = max(cs, a.itemsize)
    if rs <= 0 or cs <= 0 or rs % a.itemsize or cs % a.itemsize:
        raise ValueError("matrix view with a negative, zero or unaligned stride: pass a contiguous array")
    return _abi.RnlaMat(a.ctypes.data, rows, cols, rs // a.itemsize, cs // a.itemsize, _dtype_code(a), 0)


def _bad_strides(x) -> bool:
    if _is_torch(x):
        st, sh = x.stride(), x.shape
        return any(t <= 0 and e > 1 for t, e in zip(st, sh))
    return any((t <= 0 and e > 1) or t % x.itemsize for t, e in zip(x.strides, x.shape))


def _empty_like(x, rows: int, cols: int, order: str = "F", dtype=None):
    if _is_torch(x):
        import torch
        dt = dtype or x.dtype
        if order == "F":
            return torch.empty((cols, rows), dtype=dt, device=x.device).t()
        return torch.empty((rows, cols), dtype=dt, device=x.device)
    return np.empty((rows, cols), dtype=dtype or x.dtype, order=order)


def _as2d(x):
    """2-D input operand; views with negative / zero / unaligned strides (e.g.
    a[::-1], np.flipud, broadcasts) are copied to a contiguous array first."""
    if _is_torch(x):
        x = x if x.dim() == 2 else x.reshape(-1, 1)
        return x.contiguous() if _bad_strides(x) else x
    x = np.asarray(x)
    if x.dtype not in (np.float32, np.float64):
        x = x.astype(np.float64)
    x = x if x.ndim == 2 else x.reshape(-1, 1)
    return np.ascontiguousarray(x) if _bad_strides(x) else x


def _ctx(ctx):
    """The context for a call, ordered after the caller's torch CUDA stream:
    device inputs written asynchronously by torch (e.g. torch.randn on the
    device right before the call) are complete before the library's stream
    reads them (rnla_ctx_wait_stream; no host synchronization)."""
    c = ctx or default_context()
    import sys
    torch = sys.modules.get("torch")
    if torch is not None and torch.cuda.is_initialized():
        st = torch.cuda.current_stream(c.device).cuda_stream
        _check(_abi.lib().rnla_ctx_wait_stream(c.handle, C.c_void_p(st)))
    return c


# --------------------------------------------------------------------------
# rng.hpp: seeds, hashes, operator draws (host)
# --------------------------------------------------------------------------
def splitmix64(state: int) -> Tuple[int, int]:
    """Returns (output, new_state) (include/randnla/rng.hpp:13-18)."""
    st = C.c_uint64(state)
    out = _abi.lib().rnla_splitmix64(C.byref(st))
    return int(out), int(st.value)


def derive_seed(seed: int, stream: int) -> int:
    return int(_abi.lib().rnla_derive_seed(seed, stream))


def count_sketch_hashes(seed: int, n: int, s: int, j0: int = 0):
    b = np.empty(n, dtype=np.int64)
    g = np.empty(n, dtype=np.int8)
    _check(_abi.lib().rnla_count_sketch_hashes(seed, j0, n, s, b.ctypes.data_as(_abi._I64P),
                                               g.ctypes.data_as(_abi._I8P)))
    return b, g


def gaussian_matrix(rows: int, cols: int, seed: int) -> np.ndarray:
    """gaussian_matrix(rows, cols, make_rng(seed)) (src/rng.cpp:8-14), column-major."""
    out = np.empty((rows, cols), dtype=np.float64, order="F")
    _check(_abi.lib().rnla_gaussian_matrix(seed, rows, cols, out.ctypes.data_as(_abi._F64P)))
    return out


def sample_without_replacement(n: int, count: int, seed: int) -> np.ndarray:
    out = np.empty(count, dtype=np.int64)
    _check(_abi.lib().rnla_sample_without_replacement(seed, n, count, out.ctypes.data_as(_abi._I64P)))
    return out


def sample_with_replacement(weights, count: int, seed: int) -> np.ndarray:
    w = np.ascontiguousarray(weights, dtype=np.float64)
    out = np.empty(count, dtype=np.int64)
    _check(_abi.lib().rnla_sample_with_replacement(seed, w.ctypes.data_as(_abi._F64P), w.shape[0], count,
                                                   out.ctypes.data_as(_abi._I64P)))
    return out


def srht_operator(n: int, s: int, seed: int):
    signs = np.empty(n, dtype=np.int8)
    idx = np.empty(s, dtype=np.int64)
    _check(_abi.lib().rnla_srht_operator(seed, n, s, signs.ctypes.data_as(_abi._I8P), idx.ctypes.data_as(_abi._I64P)))
    return signs, idx


# --------------------------------------------------------------------------
# sketch.hpp
# --------------------------------------------------------------------------
class SketchKind(enum.IntEnum):
    kGaussian = 0
    kSrht = 1
    kCountSketch = 2
    kUniformColumns = 3
    kLeverageColumns = 4
    kLandmarkColumns = 5
    kCombined = 6


@dataclasses.dataclass(frozen=True)
class SketchSpec:
    """include/randnla/sketch.hpp:25-54."""
    kind: SketchKind = SketchKind.kGaussian
    s: int = 1
    seed: int = 0
    stage2: Optional["SketchSpec"] = None
    scale_columns: bool = False
    leverage_rank: Optional[int] = None

    @staticmethod
    def gaussian(s: int, seed: int) -> "SketchSpec":
        return SketchSpec(SketchKind.kGaussian, s, seed)

    @staticmethod
    def srht(s: int, seed: int) -> "SketchSpec":
        return SketchSpec(SketchKind.kSrht, s, seed)

    @staticmethod
    def count_sketch(s: int, seed: int) -> "SketchSpec":
        return SketchSpec(SketchKind.kCountSketch, s, seed)

    @staticmethod
    def uniform_columns(s: int, seed: int) -> "SketchSpec":
        return SketchSpec(SketchKind.kUniformColumns, s, seed)

    @staticmethod
    def combined(s_cs: int, dense_stage: "SketchSpec", seed: int) -> "SketchSpec":
        return SketchSpec(SketchKind.kCombined, s_cs, seed, dense_stage)

    def to_c(self) -> _abi.RnlaSketchSpec:
        st = self.stage2
        return _abi.RnlaSketchSpec(
            int(self.kind), int(self.s), int(self.seed) & 0xFFFFFFFFFFFFFFFF,
            int(st.kind) if st else 0, int(st.s) if st else 0, (int(st.seed) & 0xFFFFFFFFFFFFFFFF) if st else 0,
            1 if self.scale_columns else 0, int(self.leverage_rank) if self.leverage_rank else 0)


@dataclasses.dataclass
class ColumnSelection:
    indices: np.ndarray
    weights: Optional[np.ndarray] = None


def _sketch_call(fn_name, a, s_out, *args, ctx=None):
    a = _as2d(a)
    c = _empty_like(a, a.shape[0], s_out, "F")
    am, cm = _mat(a), _mat(c)
    _check(getattr(_abi.lib(), fn_name)(_ctx(ctx).handle, C.byref(am), *args, C.byref(cm)))
    return c


def gaussian_sketch(a, s: int, seed: int, ctx: Optional[Context] = None):
    """C = A * (G / sqrt(s)) (src/sketch.cpp:36-42)."""
    if s < 1:
        raise ValueError("gaussian_sketch: s < 1")
    return _sketch_call("rnla_gaussian_sketch", a, s, C.c_int64(s), C.c_uint64(seed), ctx=ctx)


def srht_sketch(a, s: int, seed: int, ctx: Optional[Context] = None):
    """C = A * S_srht with zero padding to the next power of two (src/sketch.cpp:57-81)."""
    n = _as2d(a).shape[1]
    if s < 1 or s > (1 << max(0, (n - 1).bit_length())):
        raise ValueError("srht_sketch: s > padded dimension")
    return _sketch_call("rnla_srht_sketch", a, s, C.c_int64(s), C.c_uint64(seed), ctx=ctx)


def count_sketch(a, s: int, seed: int, ctx: Optional[Context] = None):
    """C = A * S_count (src/sketch.cpp:83-97)."""
    if s < 1:
        raise ValueError("count_sketch: s < 1")
    return _sketch_call("rnla_count_sketch", a, s, C.c_int64(s), C.c_uint64(seed), ctx=ctx)


def combined_sketch(a, spec: SketchSpec, ctx: Optional[Context] = None):
    """Count sketch to spec.s, then the dense stage (src/sketch.cpp:108-123)."""
    if spec.kind != SketchKind.kCombined or spec.stage2 is None:
        raise ValueError("combined_sketch: spec is not a combined sketch")
    cs = spec.to_c()
    a2 = _as2d(a)
    c = _empty_like(a2, a2.shape[0], spec.stage2.s, "F")
    am, cm = _mat(a2), _mat(c)
    _check(_abi.lib().rnla_combined_sketch(_ctx(ctx).handle, C.byref(am), C.byref(cs), C.byref(cm)))
    return c


def apply_sketch(a, spec: SketchSpec, ctx: Optional[Context] = None):
    """Dispatch on spec.kind (src/sketch.cpp:177-197)."""
    if spec.kind == SketchKind.kGaussian:
        return gaussian_sketch(a, spec.s, spec.seed, ctx)
    if spec.kind == SketchKind.kSrht:
        return srht_sketch(a, spec.s, spec.seed, ctx)
    if spec.kind == SketchKind.kCountSketch:
        return count_sketch(a, spec.s, spec.seed, ctx)
    if spec.kind == SketchKind.kCombined:
        return combined_sketch(a, spec, ctx)
    if spec.kind == SketchKind.kUniformColumns:
        return uniform_sample_columns(a, spec.s, spec.seed, ctx)[0]
    if spec.kind == SketchKind.kLeverageColumns:
        return leverage_sample_columns(a, spec.s, spec.seed, spec.leverage_rank, spec.scale_columns, ctx)[0]
    raise ValueError("apply_sketch: landmark selection (k-means) is out of scope for the B200 core")


def sketch_rows(m, spec: SketchSpec, extra=None, row_offset: int = 0, out=None, ctx: Optional[Context] = None):
    """S^T M for a tall M, or S^T [M, extra] (src/regression.cpp:17-19, :76-78). Row-major result."""
    m2 = _as2d(m)
    s_final = spec.stage2.s if spec.kind == SketchKind.kCombined else spec.s
    cols = m2.shape[1] + (1 if extra is not None else 0)
    if out is None:
        out = _empty_like(m2, s_final, cols, "C")
    mm, om = _mat(m2), _mat(out)
    xm = _mat(_as2d(extra)) if extra is not None else None
    cs = spec.to_c()
    _check(_abi.lib().rnla_sketch_rows(_ctx(ctx).handle, C.byref(mm), C.byref(xm) if xm is not None else None,
                                       C.byref(cs), int(row_offset), C.byref(om)))
    return out


def count_sketch_stream(m: int, n: int, s: int, seed: int, column, chunk: int = 4096, dtype=np.float64,
                        ctx: Optional[Context] = None) -> np.ndarray:
    """Single pass over the n columns delivered by column(j), each called
    exactly once in j order (src/sketch.cpp:83-92); columns are packed into
    chunks and accumulated on the device. Returns C (m x s, column-major);
    fp64 is bit-identical to the reference's sequential loop."""
    if s < 1:
        raise ValueError("count_sketch: s < 1")
    lib = _abi.lib()
    c = _ctx(ctx)
    st = C.c_void_p()
    _check(lib.rnla_count_stream_begin(c.handle, m, n, s, C.c_uint64(seed),
                                       _abi.RNLA_F64 if np.dtype(dtype) == np.float64 else _abi.RNLA_F32,
                                       C.byref(st)))
    try:
        buf = np.empty((m, max(1, min(chunk, n))), dtype=dtype, order="F")
        j = 0
        while j < n:
            k = min(buf.shape[1], n - j)
            for t in range(k):
                buf[:, t] = np.asarray(column(j + t), dtype=dtype).reshape(m)
            bm = _mat(buf[:, :k])
            _check(lib.rnla_count_stream_push(st, C.byref(bm)))
            j += k
    except BaseException:
        lib.rnla_count_stream_abort(st)
        raise
    out = np.empty((m, s), dtype=dtype, order="F")
    om = _mat(out)
    _check(lib.rnla_count_stream_end(st, C.byref(om)))
    return out


def fwht_inplace(x, ctx: Optional[Context] = None):
    """Unnormalized Sylvester-order FWHT of x (length 2^q) or of every column
    of a 2-D x, in place (src/sketch.cpp:44-55); returns x."""
    if _is_torch(x):
        x2 = x if x.dim() == 2 else x.reshape(-1, 1)
    else:
        if not (isinstance(x, np.ndarray) and x.dtype in (np.float32, np.float64)):
            raise ValueError("fwht_inplace: a float32/float64 numpy array or torch tensor is required")
        x2 = x if x.ndim == 2 else x.reshape(-1, 1)
        if _bad_strides(x2):
            raise ValueError("fwht_inplace: x must have positive strides")
    xm = _mat(x2)
    _check(_abi.lib().rnla_fwht(_ctx(ctx).handle, C.byref(xm)))
    return x


def uniform_sample_columns(a, s: int, seed: int, ctx: Optional[Context] = None):
    a2 = _as2d(a)
    c = _empty_like(a2, a2.shape[0], s, "F")
    idx = np.empty(s, dtype=np.int64)
    am, cm = _mat(a2), _mat(c)
    _check(_abi.lib().rnla_uniform_sample_columns(_ctx(ctx).handle, C.byref(am), s, C.c_uint64(seed), C.byref(cm),
                                                  idx.ctypes.data_as(_abi._I64P)))
    return c, ColumnSelection(idx)


def leverage_scores(a, k: Optional[int] = None, ctx: Optional[Context] = None) -> np.ndarray:
    a2 = _as2d(a)
    out = np.empty(a2.shape[1], dtype=np.float64)
    am = _mat(a2)
    _check(_abi.lib().rnla_leverage_scores(_ctx(ctx).handle, C.byref(am), int(k or 0),
                                           out.ctypes.data_as(_abi._F64P)))
    return out


def leverage_sample_columns(a, s: int, seed: int, k: Optional[int] = None, scale: bool = False,
                            ctx: Optional[Context] = None):
    a2 = _as2d(a)
    c = _empty_like(a2, a2.shape[0], s, "F")
    idx = np.empty(s, dtype=np.int64)
    w = np.empty(s, dtype=np.float64)
    cnt = C.c_int64()
    am, cm = _mat(a2), _mat(c)
    _check(_abi.lib().rnla_leverage_sample_columns(
        _ctx(ctx).handle, C.byref(am), s, C.c_uint64(seed), int(k or 0), 1 if scale else 0, C.byref(cm),
        idx.ctypes.data_as(_abi._I64P), w.ctypes.data_as(_abi._F64P), C.byref(cnt)))
    n = cnt.value
    sel = ColumnSelection(idx[:n].copy(), w[:n].copy() if scale else None)
    return c[:, :n], sel


def leverage_sample_rows(m, p: int, seed: int, ctx: Optional[Context] = None):
    """Row leverage of tall M from its orthonormal basis + p weighted draws,
    sorted and deduplicated (pattern of src/spsd.cpp:150-154). Returns (scores, indices)."""
    m2 = _as2d(m)
    scores = np.empty(m2.shape[0], dtype=np.float64)
    idx = np.empty(p, dtype=np.int64)
    cnt = C.c_int64()
    mm = _mat(m2)
    _check(_abi.lib().rnla_leverage_sample_rows(_ctx(ctx).handle, C.byref(mm), p, C.c_uint64(seed),
                                                scores.ctypes.data_as(_abi._F64P), idx.ctypes.data_as(_abi._I64P),
                                                C.byref(cnt)))
    return scores, idx[:cnt.value].copy()


# --------------------------------------------------------------------------
# core.hpp
# --------------------------------------------------------------------------
@dataclasses.dataclass
class SvdFactors:
    U: object
    singular_values: np.ndarray
    V: object

    def rank(self) -> int:
        return int(self.singular_values.shape[0])

    def reconstruct(self):
        U = np.asarray(self.U.cpu() if _is_torch(self.U) else self.U)
        V = np.asarray(self.V.cpu() if _is_torch(self.V) else self.V)
        return (U * self.singular_values) @ V.T


@dataclasses.dataclass
class QrFactors:
    Q: object
    R: object


def thin_qr(a, ctx: Optional[Context] = None) -> QrFactors:
    a2 = _as2d(a)
    m, n = a2.shape
    if m < n:
        raise ValueError("thin_qr: rows < cols")
    q = _empty_like(a2, m, n, "F")
    r = _empty_like(a2, n, n, "F")
    am, qm, rm = _mat(a2), _mat(q), _mat(r)
    _check(_abi.lib().rnla_thin_qr(_ctx(ctx).handle, C.byref(am), C.byref(qm), C.byref(rm)))
    return QrFactors(q, r)


def _svd_call(a, k, ctx):
    a2 = _as2d(a)
    m, n = a2.shape
    r = min(m, n) if k is None else k
    u = _empty_like(a2, m, r, "F")
    v = _empty_like(a2, n, r, "F")
    sv = np.empty(r, dtype=np.float64)
    rank = C.c_int64()
    am, um, vm = _mat(a2), _mat(u), _mat(v)
    if k is None:
        _check(_abi.lib().rnla_condensed_svd(_ctx(ctx).handle, C.byref(am), C.byref(um),
                                             sv.ctypes.data_as(_abi._F64P), C.byref(vm), C.byref(rank)))
    else:
        _check(_abi.lib().rnla_truncated_svd(_ctx(ctx).handle, C.byref(am), k, C.byref(um),
                                             sv.ctypes.data_as(_abi._F64P), C.byref(vm), C.byref(rank)))
    rk = rank.value
    return SvdFactors(u[:, :rk], sv[:rk].copy(), v[:, :rk])


def condensed_svd(a, ctx: Optional[Context] = None) -> SvdFactors:
    return _svd_call(a, None, ctx)


def truncated_svd(a, k: int, ctx: Optional[Context] = None) -> SvdFactors:
    a2 = _as2d(a)
    if not (1 <= k <= min(a2.shape)):
        raise ValueError("truncated_svd: k out of range")
    return _svd_call(a2, k, ctx)


def pseudo_inverse(a, tol: float = 1e-12, ctx: Optional[Context] = None):
    a2 = _as2d(a)
    p = _empty_like(a2, a2.shape[1], a2.shape[0], "F")
    am, pm = _mat(a2), _mat(p)
    _check(_abi.lib().rnla_pseudo_inverse(_ctx(ctx).handle, C.byref(am), float(tol), C.byref(pm)))
    return p


# --------------------------------------------------------------------------
# randsvd.hpp
# --------------------------------------------------------------------------
@dataclasses.dataclass
class KsvdOptions:
    evaluate_error: bool = False


@dataclasses.dataclass
class KsvdResult:
    factors: SvdFactors
    passes_over_a: int
    error_fro: Optional[float] = None


def prototype_ksvd(a, k: int, s: int, seed: int, spec: Optional[SketchSpec] = None,
                   opts: KsvdOptions = KsvdOptions(), power_iters: int = 0,
                   ctx: Optional[Context] = None) -> KsvdResult:
    """Prototype randomized k-SVD (src/randsvd.cpp:88-110) + q power iterations."""
    a2 = _as2d(a)
    m, n = a2.shape
    if not (1 <= k <= s <= min(m, n)):
        raise ValueError("prototype_ksvd: need k <= s <= min(m, n)")
    u = _empty_like(a2, m, k, "F")
    v = _empty_like(a2, n, k, "F")
    sv = np.empty(k, dtype=np.float64)
    rank, passes, err = C.c_int64(), C.c_int32(), C.c_double()
    am, um, vm = _mat(a2), _mat(u), _mat(v)
    cs = spec.to_c() if spec is not None else None
    _check(_abi.lib().rnla_prototype_ksvd(
        _ctx(ctx).handle, C.byref(am), k, s, C.c_uint64(seed), C.byref(cs) if cs is not None else None,
        int(power_iters), C.byref(um), sv.ctypes.data_as(_abi._F64P), C.byref(vm), C.byref(rank), C.byref(passes),
        C.byref(err) if opts.evaluate_error else None))
    rk = rank.value
    return KsvdResult(SvdFactors(u[:, :rk], sv[:rk].copy(), v[:, :rk]), int(passes.value),
                      float(err.value) if opts.evaluate_error else None)


def faster_ksvd(a, k: int, s: int, p_cs: int, p: int, seed: int, opts: KsvdOptions = KsvdOptions(),
                ctx: Optional[Context] = None) -> KsvdResult:
    """Two-pass k-SVD: column count sketch C, joint combined row sketch of [A, C]
    (include/randnla/randsvd.hpp:38-41, src/randsvd.cpp:112-160)."""
    a2 = _as2d(a)
    m, n = a2.shape
    if not (1 <= k < s < p < p_cs):
        raise ValueError("faster_ksvd: need k < s < p < p_cs")
    u = _empty_like(a2, m, k, "F")
    v = _empty_like(a2, n, k, "F")
    sv = np.empty(k, dtype=np.float64)
    rank, passes, err = C.c_int64(), C.c_int32(), C.c_double()
    am, um, vm = _mat(a2), _mat(u), _mat(v)
    _check(_abi.lib().rnla_faster_ksvd(
        _ctx(ctx).handle, C.byref(am), k, s, p_cs, p, C.c_uint64(seed), C.byref(um), sv.ctypes.data_as(_abi._F64P),
        C.byref(vm), C.byref(rank), C.byref(passes), C.byref(err) if opts.evaluate_error else None))
    rk = rank.value
    return KsvdResult(SvdFactors(u[:, :rk], sv[:rk].copy(), v[:, :rk]), int(passes.value),
                      float(err.value) if opts.evaluate_error else None)


# --------------------------------------------------------------------------
# regression.hpp
# --------------------------------------------------------------------------
@dataclasses.dataclass
class LsrSolution:
    x: np.ndarray
    objective: float = 0.0
    iterations: int = 0
    kappa_estimate: Optional[float] = None
    converged: bool = True
    flagged: bool = False


def lsr_sketched(a, b, spec: SketchSpec, ctx: Optional[Context] = None) -> LsrSolution:
    """Sketch [A, b] in one pass, solve the small problem (src/regression.cpp:68-92)."""
    a2 = _as2d(a)
    b2 = _as2d(b)
    x = np.empty(a2.shape[1], dtype=np.float64)
    obj = C.c_double()
    flagged = C.c_int32()
    am, bm = _mat(a2), _mat(b2)
    cs = spec.to_c()
    _check(_abi.lib().rnla_lsr_sketched(_ctx(ctx).handle, C.byref(am), C.byref(bm), C.byref(cs),
                                        x.ctypes.data_as(_abi._F64P), C.byref(obj), C.byref(flagged)))
    return LsrSolution(x=x, objective=float(obj.value), flagged=bool(flagged.value))


def lsr_cg(a, b, tol: float, maxit: int, ctx: Optional[Context] = None) -> LsrSolution:
    """CG on the normal equations (src/regression.cpp:38-66), one fused pass over A per iteration."""
    a2 = _as2d(a)
    b2 = _as2d(b)
    x = np.empty(a2.shape[1], dtype=np.float64)
    obj = C.c_double()
    it, conv = C.c_int32(), C.c_int32()
    am, bm = _mat(a2), _mat(b2)
    _check(_abi.lib().rnla_lsr_cg(_ctx(ctx).handle, C.byref(am), C.byref(bm), float(tol), int(maxit),
                                  x.ctypes.data_as(_abi._F64P), C.byref(obj), C.byref(it), C.byref(conv)))
    return LsrSolution(x=x, objective=float(obj.value), iterations=int(it.value), converged=bool(conv.value))


@dataclasses.dataclass(frozen=True)
class PreconditionedOptions:
    """include/randnla/regression.hpp:37-41."""
    sketch_size: int = 0  # 0: min(d^2, 20 d) capped at n
    use_cg: bool = False  # default: gradient descent with unit step
    sketch_kind: SketchKind = SketchKind.kCountSketch


def lsr_preconditioned(a, b, eps: float, seed: int, opts: PreconditionedOptions = PreconditionedOptions(),
                       want_kappa: bool = True, ctx: Optional[Context] = None) -> LsrSolution:
    """Sketch-and-precondition LSR (src/regression.cpp:94-198): T = R_Y^-1 from the QR of
    Y = S'A, z0 = Q_Y' S'b, then O(log 1/eps) iterations, each one fused pass over A."""
    a2 = _as2d(a)
    b2 = _as2d(b)
    x = np.empty(a2.shape[1], dtype=np.float64)
    obj, kappa = C.c_double(), C.c_double()
    it = C.c_int32()
    am, bm = _mat(a2), _mat(b2)
    _check(_abi.lib().rnla_lsr_preconditioned(
        _ctx(ctx).handle, C.byref(am), C.byref(bm), float(eps), C.c_uint64(seed), int(opts.sketch_size),
        1 if opts.use_cg else 0, int(opts.sketch_kind), x.ctypes.data_as(_abi._F64P), C.byref(obj), C.byref(it),
        C.byref(kappa) if want_kappa else None))
    return LsrSolution(x=x, objective=float(obj.value), iterations=int(it.value),
                       kappa_estimate=float(kappa.value) if want_kappa else None)


# --------------------------------------------------------------------------
# spsd.hpp
# --------------------------------------------------------------------------
@dataclasses.dataclass(frozen=True)
class KernelSpec:
    sigma: float = 1.0


class KernelView:
    """Lazily evaluated RBF kernel over one dataset (include/randnla/spsd.hpp:26-47).
    Entries are evaluated on the device inside nystrom(); entries_evaluated()
    reports what those calls evaluated, like the reference's atomic counter."""

    def __init__(self, data, spec: KernelSpec):
        if not spec.sigma > 0.0:
            raise ValueError("KernelView: sigma <= 0")
        d = _as2d(data)
        arr = np.asarray(d.cpu()) if _is_torch(d) else d
        if not np.all(np.isfinite(arr)):
            raise ValueError("KernelView data: non-finite entries")
        self._data = d
        self._spec = spec
        self._count = 0

    def n(self) -> int:
        return int(self._data.shape[0])

    def data(self):
        return self._data

    def spec(self) -> KernelSpec:
        return self._spec

    def entries_evaluated(self) -> int:
        return self._count

    def _add(self, k: int) -> None:
        self._count += int(k)


@dataclasses.dataclass
class NystromFactor:
    L: object
    selected: np.ndarray


def rbf_kernel(x1, x2, sigma: float, ctx: Optional[Context] = None):
    """K_ij = exp((x1_i . x2_j - (|x1_i|^2 + |x2_j|^2)/2) / sigma^2) (src/spsd.cpp:33-47)."""
    if not sigma > 0.0:
        raise ValueError("rbf_kernel: sigma <= 0")
    a, b = _as2d(x1), _as2d(x2)
    if a.shape[1] != b.shape[1]:
        raise ValueError("rbf_kernel: dimension mismatch")
    k = _empty_like(a, a.shape[0], b.shape[0], "F")
    am, bm, km = _mat(a), _mat(b), _mat(k)
    _check(_abi.lib().rnla_rbf_kernel(_ctx(ctx).handle, C.byref(am), C.byref(bm), float(sigma), C.byref(km)))
    return k


def nystrom(k, s: int, seed: int, target_k: int = 0, ctx: Optional[Context] = None) -> NystromFactor:
    """Nystrom factor L with L L' ~ C W_k^+ C' (src/spsd.cpp:181-228): k is a
    KernelView (kernel columns evaluated on the device, entries counted) or a
    dense SPSD matrix K (the reference's nystrom(const DenseMatrix&, ...))."""
    kk = target_k if target_k > 0 else int(math.ceil(0.8 * s))
    sel = np.empty(s, dtype=np.int64)
    kept = C.c_int64()
    if isinstance(k, KernelView):
        x = k.data()
        n = k.n()
        if not (1 <= kk <= s <= n):
            raise ValueError("nystrom: need k <= s <= n")
        L = _empty_like(x, n, kk, "F")
        entries = C.c_int64()
        xm, lm = _mat(x), _mat(L)
        _check(_abi.lib().rnla_nystrom(_ctx(ctx).handle, C.byref(xm), float(k.spec().sigma), s, C.c_uint64(seed),
                                       int(target_k), C.byref(lm), sel.ctypes.data_as(_abi._I64P), C.byref(kept),
                                       C.byref(entries)))
        k._add(entries.value)
        return NystromFactor(L[:, :kept.value], sel)
    K = _as2d(k)
    n = K.shape[0]
    if K.shape[0] != K.shape[1]:
        raise ValueError("nystrom: K not square")
    if not (1 <= kk <= s <= n):
        raise ValueError("nystrom: need k <= s <= n")
    L = _empty_like(K, n, kk, "F")
    km, lm = _mat(K), _mat(L)
    _check(_abi.lib().rnla_nystrom_dense(_ctx(ctx).handle, C.byref(km), s, C.c_uint64(seed), int(target_k),
                                         C.byref(lm), sel.ctypes.data_as(_abi._I64P), C.byref(kept)))
    return NystromFactor(L[:, :kept.value], sel)


def nystrom_columns(c, selected, target_k: int = 0, ctx: Optional[Context] = None) -> NystromFactor:
    """nystrom(const SpsdSource&, ...) for a caller-side source: c = K[:, selected]
    (n x s) already evaluated; selected strictly increasing (src/spsd.cpp:181-217)."""
    c2 = _as2d(c)
    n, s = c2.shape
    kk = target_k if target_k > 0 else int(math.ceil(0.8 * s))
    if not (1 <= kk <= s <= n):
        raise ValueError("nystrom: need k <= s <= n")
    sel = np.ascontiguousarray(selected, dtype=np.int64)
    L = _empty_like(c2, n, kk, "F")
    kept = C.c_int64()
    cm, lm = _mat(c2), _mat(L)
    _check(_abi.lib().rnla_nystrom_columns(_ctx(ctx).handle, C.byref(cm), sel.ctypes.data_as(_abi._I64P),
                                           int(target_k), C.byref(lm), C.byref(kept)))
    return NystromFactor(L[:, :kept.value], sel.copy())


def approx_eig(l, k: int, ctx: Optional[Context] = None):
    """Top-k eigenpairs of L L' from the SVD of L (src/spsd.cpp:257-265)."""
    l2 = _as2d(l)
    if not (1 <= k <= l2.shape[1]):
        raise ValueError("approx_eig: k > cols(L)")
    u = _empty_like(l2, l2.shape[0], k, "F")
    lam = np.empty(k, dtype=np.float64)
    lm, um = _mat(l2), _mat(u)
    _check(_abi.lib().rnla_approx_eig(_ctx(ctx).handle, C.byref(lm), k, C.byref(um), lam.ctypes.data_as(_abi._F64P)))
    return u, lam


def nystrom_eig(k: KernelView, s: int, seed: int, target_k: int, n_eig: int, want_vectors: bool = True,
                ctx: Optional[Context] = None):
    """approx_eig(nystrom(k, s, seed, target_k).L, n_eig) without forming C or L.
    Returns (U or None, lambdas, selected, kept)."""
    x = k.data()
    n = k.n()
    u = _empty_like(x, n, n_eig, "F") if want_vectors else None
    lam = np.empty(n_eig, dtype=np.float64)
    sel = np.empty(s, dtype=np.int64)
    kept = C.c_int64()
    xm = _mat(x)
    um = _mat(u) if u is not None else None
    _check(_abi.lib().rnla_nystrom_eig(_ctx(ctx).handle, C.byref(xm), float(k.spec().sigma), s, C.c_uint64(seed),
                                       int(target_k), n_eig, C.byref(um) if um is not None else None,
                                       lam.ctypes.data_as(_abi._F64P), sel.ctypes.data_as(_abi._I64P),
                                       C.byref(kept)))
    k._add(n * s)
    return u, lam, sel, kept.value


@dataclasses.dataclass
class SpsdSketch:
    """include/randnla/spsd.hpp:86-94: K ~ Q Z Q'."""
    Q: object
    Z: np.ndarray
    selected: np.ndarray
    secondary: np.ndarray
    flagged: bool = False

    def reconstruct(self):
        q = self.Q.cpu().numpy() if _is_torch(self.Q) else np.asarray(self.Q)
        return q @ self.Z @ q.T


def spsd_faster(k, s: int, p: int, seed: int, ctx: Optional[Context] = None) -> SpsdSketch:
    """Faster SPSD sketch (src/spsd.cpp:131-168) of a KernelView (entries evaluated on the
    device: n*s + |P|^2) or of a dense SPSD matrix."""
    view = k if isinstance(k, KernelView) else None
    x = view.data() if view is not None else _as2d(k)
    n = int(x.shape[0])
    q = _empty_like(x, n, s, "F", dtype=None)
    z = np.empty((s, s), dtype=np.float64, order="F")
    sel = np.empty(s, dtype=np.int64)
    sec = np.empty(max(1, min(n, p + s)), dtype=np.int64)
    nsec, flagged = C.c_int64(), C.c_int32()
    xm, qm, zm = _mat(x), _mat(q), _mat(z)
    args = (C.byref(qm), C.byref(zm), sel.ctypes.data_as(_abi._I64P), sec.ctypes.data_as(_abi._I64P),
            C.byref(nsec), C.byref(flagged))
    if view is not None:
        _check(_abi.lib().rnla_spsd_faster(_ctx(ctx).handle, C.byref(xm), float(view.spec().sigma), s, p,
                                           C.c_uint64(seed), *args))
        view._add(n * s + nsec.value * nsec.value)
    else:
        _check(_abi.lib().rnla_spsd_faster_dense(_ctx(ctx).handle, C.byref(xm), s, p, C.c_uint64(seed), *args))
    return SpsdSketch(q, z, sel, sec[:nsec.value].copy(), bool(flagged.value))


@dataclasses.dataclass
class CurFactors:
    """include/randnla/cur.hpp:12-29: A ~ C U R."""
    C: object
    U: np.ndarray
    R: object
    col_indices: np.ndarray
    row_indices: np.ndarray
    secondary_rows: np.ndarray
    secondary_cols: np.ndarray
    entries_visited: int = 0
    flagged: bool = False

    def reconstruct(self):
        c = self.C.cpu().numpy() if _is_torch(self.C) else np.asarray(self.C)
        r = self.R.cpu().numpy() if _is_torch(self.R) else np.asarray(self.R)
        return c @ (self.U @ r)


def cur_faster_kernel(xtest, xtrain, sigma: float, c: int, r: int, seed: int,
                      ctx: Optional[Context] = None) -> CurFactors:
    """CUR of the implicit RBF cross kernel (src/cur.cpp:188-212), entries evaluated on the device."""
    xt, xr = _as2d(xtest), _as2d(xtrain)
    m, n = int(xt.shape[0]), int(xr.shape[0])
    p = 2 * (c + r)
    cm = _empty_like(xt, m, c, "F", dtype=None)
    um = np.empty((c, r), dtype=np.float64, order="F")
    rm = _empty_like(xt, r, n, "F", dtype=None)
    ci, ri = np.empty(c, dtype=np.int64), np.empty(r, dtype=np.int64)
    sr, sc = np.empty(max(1, min(m, p + r)), dtype=np.int64), np.empty(max(1, min(n, p + c)), dtype=np.int64)
    nsr, nsc, ent, fl = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int32()
    a, b, cc, uu, rr = _mat(xt), _mat(xr), _mat(cm), _mat(um), _mat(rm)
    _check(_abi.lib().rnla_cur_faster_kernel(
        _ctx(ctx).handle, C.byref(a), C.byref(b), float(sigma), c, r, C.c_uint64(seed), C.byref(cc), C.byref(uu),
        C.byref(rr), ci.ctypes.data_as(_abi._I64P), ri.ctypes.data_as(_abi._I64P), sr.ctypes.data_as(_abi._I64P),
        C.byref(nsr), sc.ctypes.data_as(_abi._I64P), C.byref(nsc), C.byref(ent), C.byref(fl)))
    return CurFactors(cm, um, rm, ci, ri, sr[:nsr.value].copy(), sc[:nsc.value].copy(), int(ent.value),
                      bool(fl.value))
