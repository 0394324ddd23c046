// api_stream.cu -- the remaining reference entry points of the sketch API
// that are not whole-matrix calls:
//   * count_sketch_stream (src/sketch.cpp:83-92): columns arrive from a
//     caller callback in j order; the library accumulates each pushed chunk
//     into a device-resident m x s result in the reference's bucket order
//     (fp64: bit-identical to the single sequential pass);
//   * fwht_inplace (src/sketch.cpp:44-55) on columns of a matrix, stage by
//     stage in the reference's order h = 1, 2, 4, ... (bit-identical).
#include "marshal.h"
#include "util.cuh"

struct rnla_count_stream {
  rnla_ctx* ctx = nullptr;
  int64_t m = 0, n = 0, s = 0, next_j = 0;
  uint64_t seed = 0;
  int dtype = RNLA_F64;
  rnla::DevBuf acc;  // s segments of length m (row-major s x m): out[b * m + c]
};

namespace rnla {
namespace {

// Stages h < 2^LOG of every aligned 2^LOG block in shared memory, one block
// per CTA (column `blockIdx.y`), then write back. Same butterflies and the
// same stage order as the reference loop.
template <class T, int LOG>
__global__ void fwht_low_kernel(T* __restrict__ x, int64_t ld, int64_t n) {
  constexpr int B = 1 << LOG;
  __shared__ T buf[B];
  T* col = x + (int64_t)blockIdx.y * ld + (int64_t)blockIdx.x * B;
  for (int i = threadIdx.x; i < B; i += blockDim.x) buf[i] = col[i];
  __syncthreads();
  for (int h = 1; h < B && h < n; h *= 2) {
    for (int p = threadIdx.x; p < B / 2; p += blockDim.x) {
      const int j = (p / h) * 2 * h + (p % h);
      const T a = buf[j], b = buf[j + h];
      buf[j] = a + b;
      buf[j + h] = a - b;
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < B; i += blockDim.x) col[i] = buf[i];
}

// One stage h (>= the shared-memory block) over every pair of every column.
template <class T>
__global__ void fwht_stage_kernel(T* __restrict__ x, int64_t ld, int64_t n, int64_t h) {
  const int64_t pairs = n / 2;
  T* col = x + (int64_t)blockIdx.y * ld;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < pairs; p += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = (p / h) * 2 * h + (p % h);
    const T a = col[j], b = col[j + h];
    col[j] = a + b;
    col[j + h] = a - b;
  }
}

template <class T>
void fwht_columns(rnla_ctx* ctx, T* x, int64_t ld, int64_t n, int64_t cols) {
  constexpr int LOG = sizeof(T) == 8 ? 11 : 12;  // 16 KB of shared memory
  const int64_t B = int64_t(1) << LOG;
  if (n <= 1 || cols == 0) return;
  const int64_t low = std::min(n, B);
  if (low == B) {
    fwht_low_kernel<T, LOG><<<dim3((unsigned)(n / B), (unsigned)cols), 256, 0, ctx->stream>>>(x, ld, n);
  } else {  // n < B: one partial block, the loop stops at h < n
    for (int64_t h = 1; h < n; h *= 2) {
      fwht_stage_kernel<T><<<dim3((unsigned)std::max<int64_t>(1, (n / 2 + 255) / 256), (unsigned)cols), 256, 0,
                             ctx->stream>>>(x, ld, n, h);
      note_launch(ctx);
    }
    RNLA_CUDA(cudaGetLastError());
    return;
  }
  RNLA_CUDA(cudaGetLastError());
  note_launch(ctx);
  const unsigned gx = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n / 2 + 255) / 256, 4 * ctx->num_sms));
  for (int64_t h = B; h < n; h *= 2) {
    fwht_stage_kernel<T><<<dim3(gx, (unsigned)cols), 256, 0, ctx->stream>>>(x, ld, n, h);
    RNLA_CUDA(cudaGetLastError());
    note_launch(ctx);
  }
}

}  // namespace
}  // namespace rnla

using namespace rnla;

extern "C" {

rnla_status rnla_fwht(rnla_ctx* ctx, rnla_mat* x) {
  return guard([&] {
    enter(ctx);
    check_mat(x, "fwht_inplace: x");
    const int64_t n = x->rows;
    require(n >= 1 && (n & (n - 1)) == 0, "fwht_inplace: length is not a power of two");
    OutMat o(ctx, x, x->rows, x->cols, "fwht_inplace: x", false);
    if (o.staged) {  // host buffer: upload into the column-major staging copy
      DevMat src = to_device(ctx, x);
      if (x->dtype == RNLA_F64)
        copy2d<double>(ctx, n, x->cols, src.as<double>(), src.rs, src.cs, o.dev.as<double>(), o.dev.rs, o.dev.cs);
      else
        copy2d<float>(ctx, n, x->cols, src.as<float>(), src.rs, src.cs, o.dev.as<float>(), o.dev.rs, o.dev.cs);
    }
    DevMat w = o.dev.rs == 1 ? DevMat{} : dense_copy(ctx, o.dev, false, o.dev.dtype);
    const DevMat& cm = o.dev.rs == 1 ? o.dev : w;
    if (x->dtype == RNLA_F64) fwht_columns<double>(ctx, cm.as<double>(), cm.cs, n, x->cols);
    else fwht_columns<float>(ctx, cm.as<float>(), cm.cs, n, x->cols);
    if (o.dev.rs != 1) {
      if (x->dtype == RNLA_F64)
        copy2d<double>(ctx, n, x->cols, w.as<double>(), 1, w.cs, o.dev.as<double>(), o.dev.rs, o.dev.cs);
      else
        copy2d<float>(ctx, n, x->cols, w.as<float>(), 1, w.cs, o.dev.as<float>(), o.dev.rs, o.dev.cs);
    }
    o.finish(ctx);
  });
}

rnla_status rnla_count_stream_begin(rnla_ctx* ctx, int64_t m, int64_t n, int64_t s, uint64_t seed, int32_t dtype,
                                    rnla_count_stream** out) {
  return guard([&] {
    enter(ctx);
    require(out != nullptr, "count_sketch_stream: null out");
    require(s >= 1, "count_sketch: s < 1");
    require(m >= 0 && n >= 0, "count_sketch_stream: negative shape");
    require(dtype == RNLA_F64 || dtype == RNLA_F32, "count_sketch_stream: unknown dtype");
    auto st = std::make_unique<rnla_count_stream>();
    st->ctx = ctx;
    st->m = m;
    st->n = n;
    st->s = s;
    st->seed = seed;
    st->dtype = dtype;
    const size_t bytes = esize(dtype) * (size_t)std::max<int64_t>(s * m, 1);
    st->acc = DevBuf(bytes, ctx->stream);
    RNLA_CUDA(cudaMemsetAsync(st->acc.p, 0, bytes, ctx->stream));
    *out = st.release();
  });
}

rnla_status rnla_count_stream_push(rnla_count_stream* st, const rnla_mat* cols) {
  return guard([&] {
    require(st != nullptr, "count_sketch_stream: null stream");
    rnla_ctx* ctx = st->ctx;
    enter(ctx);
    check_mat(cols, "count_sketch_stream: columns");
    require(cols->rows == st->m, "count_sketch_stream: column length differs from m");
    require(cols->dtype == st->dtype, "count_sketch_stream: dtype differs from the stream's");
    const int64_t k = cols->cols;
    require(st->next_j + k <= st->n, "count_sketch_stream: more than n columns pushed");
    if (k == 0) return;
    // columns contiguous on the device: segment j = column j
    DevMat d = as_colmajor(ctx, to_device(ctx, cols));
    const int64_t j0 = st->next_j;
    if (st->dtype == RNLA_F64)
      count_sketch_segments<double>(ctx, d.as<double>(), d.cs, nullptr, 1, k, st->m, st->s, st->seed, j0,
                                    st->acc.as<double>(), st->m, true);
    else
      count_sketch_segments<float>(ctx, d.as<float>(), d.cs, nullptr, 1, k, st->m, st->s, st->seed, j0,
                                   st->acc.as<float>(), st->m, true);
    count_sketch_plan_release(ctx, k, st->s, st->seed, j0);  // chunk plans are used once
    st->next_j += k;
    RNLA_CUDA(cudaStreamSynchronize(ctx->stream));  // the caller may reuse its chunk buffer
  });
}

rnla_status rnla_count_stream_end(rnla_count_stream* st, rnla_mat* c) {
  std::unique_ptr<rnla_count_stream> own(st);
  return guard([&] {
    require(st != nullptr, "count_sketch_stream: null stream");
    rnla_ctx* ctx = st->ctx;
    enter(ctx);
    require(st->next_j == st->n, "count_sketch_stream: fewer than n columns pushed");
    OutMat o(ctx, c, st->m, st->s, "count_sketch_stream: C", false);
    require(o.dev.dtype == st->dtype, "count_sketch_stream: output dtype differs");
    // acc segment b (length m) = column b of C
    if (st->dtype == RNLA_F64)
      copy2d<double>(ctx, st->m, st->s, st->acc.as<double>(), 1, st->m, o.dev.as<double>(), o.dev.rs, o.dev.cs);
    else
      copy2d<float>(ctx, st->m, st->s, st->acc.as<float>(), 1, st->m, o.dev.as<float>(), o.dev.rs, o.dev.cs);
    o.finish(ctx);
  });
}

void rnla_count_stream_abort(rnla_count_stream* st) {
  if (!st) return;
  cudaSetDevice(st->ctx->device);
  cudaStreamSynchronize(st->ctx->stream);
  delete st;
}

}  // extern "C"
