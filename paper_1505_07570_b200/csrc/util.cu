// util.cu -- small device helpers: strided 2-D copies, scaling, the
// least-squares objective pass.
#include "rnla_internal.h"
#include "util.cuh"
#include "algos.h"

namespace rnla {

namespace {

template <class S, class D>
__global__ void copy2d_kernel(int64_t rows, int64_t cols, const S* __restrict__ src, int64_t s_rs, int64_t s_cs,
                              D* __restrict__ dst, int64_t d_rs, int64_t d_cs) {
  const int64_t total = rows * cols;
  // Iterate in destination-contiguous order when the destination is row-major.
  const bool dst_rowmajor = d_cs == 1;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t i, j;
    if (dst_rowmajor) { i = e / cols; j = e % cols; } else { j = e / rows; i = e % rows; }
    dst[i * d_rs + j * d_cs] = (D)src[i * s_rs + j * s_cs];
  }
}

template <class T>
__global__ void scale_kernel(T* p, int64_t count, double divisor) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count; e += (int64_t)gridDim.x * blockDim.x)
    p[e] = (T)((double)p[e] / divisor);
}

// Per-row residual r_i = a_i . x - b_i over a row-major-ish A (one warp per
// row), squared and accumulated in fp64 per block, then one partial per block.
template <class T>
__global__ void residual_sq_kernel(int64_t n, int64_t d, const T* __restrict__ A, int64_t a_rs, int64_t a_cs,
                                   const T* __restrict__ b, int64_t b_rs, const double* __restrict__ x,
                                   double* partial) {
  __shared__ double red[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double local = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * nw + warp; i < n; i += (int64_t)gridDim.x * nw) {
    double dot = 0.0;
    for (int64_t c = lane; c < d; c += 32) dot += (double)__ldcs(A + i * a_rs + c * a_cs) * x[c];
#pragma unroll
    for (int o = 16; o; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
    const double r = dot - (double)b[i * b_rs];
    local += r * r;
  }
  if (lane == 0) red[warp] = local;
  __syncthreads();
  if (warp == 0) {
    double v = lane < nw ? red[lane] : 0.0;
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) partial[blockIdx.x] = v;
  }
}

}  // namespace

void ensure_dyn_smem(const void* kernel, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> cur;
  int dev = 0;
  RNLA_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  size_t& c = cur[{kernel, dev}];
  if (bytes <= c) return;
  RNLA_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  c = bytes;
}

int grid_for(rnla_ctx* ctx, int64_t work, int per_block) {
  const int64_t b = (work + per_block - 1) / per_block;
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, (int64_t)ctx->num_sms * 16));
}

template <class S, class D>
void copy2d_cast(rnla_ctx* ctx, int64_t rows, int64_t cols, const S* src, int64_t s_rs, int64_t s_cs, D* dst,
                 int64_t d_rs, int64_t d_cs) {
  if (rows == 0 || cols == 0) return;
  copy2d_kernel<S, D><<<grid_for(ctx, rows * cols, 256), 256, 0, ctx->stream>>>(rows, cols, src, s_rs, s_cs, dst,
                                                                                 d_rs, d_cs);
  RNLA_CUDA(cudaGetLastError());
  note_launch(ctx);
}

template <class T>
void copy2d(rnla_ctx* ctx, int64_t rows, int64_t cols, const T* src, int64_t s_rs, int64_t s_cs, T* dst, int64_t d_rs,
            int64_t d_cs) {
  copy2d_cast<T, T>(ctx, rows, cols, src, s_rs, s_cs, dst, d_rs, d_cs);
}

template <class T>
void scale_inplace(rnla_ctx* ctx, T* p, int64_t count, double divisor) {
  if (count == 0) return;
  scale_kernel<T><<<grid_for(ctx, count, 256), 256, 0, ctx->stream>>>(p, count, divisor);
  RNLA_CUDA(cudaGetLastError());
  note_launch(ctx);
}

template <class T>
double residual_sq(rnla_ctx* ctx, int64_t n, int64_t d, const T* A, int64_t a_rs, int64_t a_cs, const T* b,
                   int64_t b_rs, const double* x_dev) {
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((n + 7) / 8, (int64_t)ctx->num_sms * 8));
  DevBuf part(sizeof(double) * blocks, ctx->stream);
  residual_sq_kernel<T><<<blocks, 256, 0, ctx->stream>>>(n, d, A, a_rs, a_cs, b, b_rs, x_dev, part.as<double>());
  RNLA_CUDA(cudaGetLastError());
  note_launch(ctx);
  std::vector<double> h(blocks);
  RNLA_CUDA(cudaMemcpyAsync(h.data(), part.p, sizeof(double) * blocks, cudaMemcpyDeviceToHost, ctx->stream));
  RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
  double s = 0.0;
  for (double v : h) s += v;
  return s;
}

template void copy2d_cast<double, float>(rnla_ctx*, int64_t, int64_t, const double*, int64_t, int64_t, float*,
                                         int64_t, int64_t);
template void copy2d_cast<float, double>(rnla_ctx*, int64_t, int64_t, const float*, int64_t, int64_t, double*,
                                         int64_t, int64_t);
template void copy2d<double>(rnla_ctx*, int64_t, int64_t, const double*, int64_t, int64_t, double*, int64_t, int64_t);
template void copy2d<float>(rnla_ctx*, int64_t, int64_t, const float*, int64_t, int64_t, float*, int64_t, int64_t);
template void scale_inplace<double>(rnla_ctx*, double*, int64_t, double);
template void scale_inplace<float>(rnla_ctx*, float*, int64_t, double);
template double residual_sq<double>(rnla_ctx*, int64_t, int64_t, const double*, int64_t, int64_t, const double*,
                                    int64_t, const double*);
template double residual_sq<float>(rnla_ctx*, int64_t, int64_t, const float*, int64_t, int64_t, const float*, int64_t,
                                   const double*);

}  // namespace rnla

// ---- small helpers used by the factorization paths (algos.h) ----
namespace rnla {
namespace {
__global__ void scale_rows_kernel(int64_t r, int64_t n, const double* __restrict__ V, const double* __restrict__ s,
                                  double* __restrict__ out) {
  const int64_t total = r * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % r, j = e / r;
    out[i + j * r] = s[i] * V[j + i * n];
  }
}
__global__ void scale_cols_kernel(int64_t n, int64_t r, const double* __restrict__ V, const double* __restrict__ d,
                                  double* __restrict__ out) {
  const int64_t total = r * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x)
    out[e] = V[e] * d[e / n];
}
__global__ void sumsq_kernel(const double* __restrict__ p, int64_t count, double* partial) {
  __shared__ double red[32];
  double acc = 0.0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count; e += (int64_t)gridDim.x * blockDim.x)
    acc += p[e] * p[e];
#pragma unroll
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) partial[blockIdx.x] = v;
  }
}
__global__ void hash_uniform_kernel(int64_t count, uint64_t seed, double* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count; e += (int64_t)gridDim.x * blockDim.x) {
    uint64_t z = seed ^ (0x9e3779b97f4a7c15ull * (uint64_t)(e + 1));
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    z ^= z >> 31;
    out[e] = (double)(z >> 11) * 0x1.0p-52 - 1.0;
  }
}
// out[j] = |YZ(:, j) - theta[j] * VZ(:, j)|^2, one block per column
__global__ void ritz_residual_kernel(int64_t n, const double* __restrict__ YZ, const double* __restrict__ VZ,
                                     const double* __restrict__ theta, double* __restrict__ out) {
  __shared__ double red[32];
  const int64_t j = blockIdx.x;
  const double t = theta[j];
  double acc = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double r = YZ[i + j * n] - t * VZ[i + j * n];
    acc += r * r;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) out[j] = v;
  }
}
}  // namespace

void hash_uniform_dev(rnla_ctx* ctx, int64_t count, uint64_t seed, double* out) {
  if (count == 0) return;
  hash_uniform_kernel<<<grid_for(ctx, count, 256), 256, 0, ctx->stream>>>(count, seed, out);
  RNLA_CUDA(cudaGetLastError());
  note_launch(ctx);
}
void ritz_residual_dev(rnla_ctx* ctx, int64_t n, int64_t k, const double* YZ, const double* VZ, const double* theta,
                       double* out) {
  if (k == 0) return;
  ritz_residual_kernel<<<(unsigned)k, 256, 0, ctx->stream>>>(n, YZ, VZ, theta, out);
  RNLA_CUDA(cudaGetLastError());
  note_launch(ctx);
}

void scale_rows_dev(rnla_ctx* ctx, int64_t r, int64_t n, const double* V, const double* s, double* out) {
  if (r * n == 0) return;
  scale_rows_kernel<<<grid_for(ctx, r * n, 256), 256, 0, ctx->stream>>>(r, n, V, s, out);
  RNLA_CUDA(cudaGetLastError());
  note_launch(ctx);
}
void scale_cols_dev(rnla_ctx* ctx, int64_t n, int64_t r, const double* V, const double* d, double* out) {
  if (r * n == 0) return;
  scale_cols_kernel<<<grid_for(ctx, r * n, 256), 256, 0, ctx->stream>>>(n, r, V, d, out);
  RNLA_CUDA(cudaGetLastError());
  note_launch(ctx);
}
double sum_squares_dev(rnla_ctx* ctx, const double* p, int64_t count) {
  if (count == 0) return 0.0;
  const int blocks = grid_for(ctx, count, 1024);
  DevBuf part(sizeof(double) * blocks, ctx->stream);
  sumsq_kernel<<<blocks, 256, 0, ctx->stream>>>(p, count, part.as<double>());
  RNLA_CUDA(cudaGetLastError());
  note_launch(ctx);
  std::vector<double> h(blocks);
  RNLA_CUDA(cudaMemcpyAsync(h.data(), part.p, sizeof(double) * blocks, cudaMemcpyDeviceToHost, ctx->stream));
  RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
  double s = 0.0;
  for (double v : h) s += v;
  return s;
}
}  // namespace rnla
