// lsr.cu -- the streaming pass of sketch-and-precondition least squares.
//
// Reference: lsr_preconditioned, /root/reference/proj/src/regression.cpp:94-198.
// Every iteration of its gradient descent / CG needs A*(T z) followed by
// A'(residual) (:159-161, :171-173): two passes over A in the reference. Here
// one kernel does both in ONE pass: each warp loads a row a_i once into
// registers, forms r_i = beta*b_i - a_i . w (warp butterfly, identical bits on
// all lanes) and accumulates r_i * a_i into per-lane fp64 partials of
// g = A'(beta*b - A w); it also accumulates sum r_i^2 (the objective). CTA
// partials are reduced in a fixed order, so results are deterministic.
// HBM-bound: n*d*sizeof(T) bytes per call.
#include "rnla_internal.h"
#include "util.cuh"

namespace rnla {

namespace {

constexpr int kWarps = 8;

template <class T, int VPL>
__global__ void __launch_bounds__(kWarps * 32) normal_gemv_kernel(const T* __restrict__ A, int64_t ld, int64_t n,
                                                                  int d, const T* __restrict__ b, int64_t b_stride,
                                                                  double beta, const double* __restrict__ w,
                                                                  double* __restrict__ g_part,
                                                                  double* __restrict__ rr_part) {
  extern __shared__ double sh[];  // w[d], then the per-warp partials [kWarps][d]
  double* ws = sh;
  double* part = sh + d;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int c = threadIdx.x; c < d; c += blockDim.x) ws[c] = w[c];
  __syncthreads();
  double acc[VPL];
#pragma unroll
  for (int k = 0; k < VPL; ++k) acc[k] = 0.0;
  double rr = 0.0;
  const int64_t gw = (int64_t)blockIdx.x * kWarps + warp, nw = (int64_t)gridDim.x * kWarps;
  for (int64_t i = gw; i < n; i += 2 * nw) {
    const int64_t i2 = i + nw;
    double v1[VPL], v2[VPL];
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
      const int c = lane + 32 * k;
      v1[k] = c < d ? (double)__ldcs(A + i * ld + c) : 0.0;
      v2[k] = (c < d && i2 < n) ? (double)__ldcs(A + i2 * ld + c) : 0.0;
    }
    double d1 = 0.0, d2 = 0.0;
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
      const int c = lane + 32 * k;
      const double wc = c < d ? ws[c] : 0.0;
      d1 = fma(v1[k], wc, d1);
      d2 = fma(v2[k], wc, d2);
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      d1 += __shfl_xor_sync(0xffffffffu, d1, o);
      d2 += __shfl_xor_sync(0xffffffffu, d2, o);
    }
    const double r1 = (beta != 0.0 ? beta * (double)b[i * b_stride] : 0.0) - d1;
    const double r2 = i2 < n ? (beta != 0.0 ? beta * (double)b[i2 * b_stride] : 0.0) - d2 : 0.0;
#pragma unroll
    for (int k = 0; k < VPL; ++k) acc[k] = fma(v2[k], r2, fma(v1[k], r1, acc[k]));
    rr = fma(r2, r2, fma(r1, r1, rr));
  }
#pragma unroll
  for (int k = 0; k < VPL; ++k) {
    const int c = lane + 32 * k;
    if (c < d) part[warp * d + c] = acc[k];
  }
  __syncthreads();
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    double s = 0.0;
    for (int q = 0; q < kWarps; ++q) s += part[q * d + c];
    g_part[(int64_t)blockIdx.x * d + c] = s;
  }
  __syncthreads();
  if (lane == 0) part[warp] = rr;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int q = 0; q < kWarps; ++q) s += part[q];
    rr_part[blockIdx.x] = s;
  }
}

// g[c] = sum over CTAs in order; rr = sum of the CTA residual partials.
__global__ void reduce_parts_kernel(int nblk, int d, const double* __restrict__ g_part,
                                    const double* __restrict__ rr_part, double* __restrict__ g,
                                    double* __restrict__ rr) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c <= d; c += gridDim.x * blockDim.x) {
    double s = 0.0;
    if (c < d) {
      for (int q = 0; q < nblk; ++q) s += g_part[(int64_t)q * d + c];
      g[c] = s;
    } else {
      for (int q = 0; q < nblk; ++q) s += rr_part[q];
      *rr = s;
    }
  }
}

template <class T, int VPL>
void launch_normal_gemv(rnla_ctx* ctx, int nblk, int64_t n, int64_t d, const T* A, int64_t ld, const T* b,
                        int64_t b_stride, double beta, const double* w, double* g_part, double* rr_part) {
  const size_t smem = sizeof(double) * (size_t)(d + kWarps * d);
  auto k = normal_gemv_kernel<T, VPL>;
  ensure_dyn_smem((const void*)k, smem);
  k<<<nblk, kWarps * 32, smem, ctx->stream>>>(A, ld, n, (int)d, b, b_stride, beta, w, g_part, rr_part);
  RNLA_CUDA(cudaGetLastError());
}

}  // namespace

bool normal_gemv_supported(int64_t d) { return d >= 1 && d <= 1024; }

template <class T>
void normal_gemv(rnla_ctx* ctx, int64_t n, int64_t d, const T* A, int64_t ld, const T* b, int64_t b_stride,
                 double beta, const double* w, double* g, double* rr) {
  require(normal_gemv_supported(d), "normal_gemv: d above 1024");
  const int nblk = std::max(1, ctx->num_sms * 2);
  DevBuf g_part(sizeof(double) * (size_t)nblk * d, ctx->stream), rr_part(sizeof(double) * nblk, ctx->stream);
  if (n <= 0) {
    RNLA_CUDA(cudaMemsetAsync(g, 0, sizeof(double) * d, ctx->stream));
    RNLA_CUDA(cudaMemsetAsync(rr, 0, sizeof(double), ctx->stream));
    return;
  }
  const int vpl = (int)((d + 31) / 32);
  if (vpl <= 1) launch_normal_gemv<T, 1>(ctx, nblk, n, d, A, ld, b, b_stride, beta, w, g_part.as<double>(), rr_part.as<double>());
  else if (vpl <= 2) launch_normal_gemv<T, 2>(ctx, nblk, n, d, A, ld, b, b_stride, beta, w, g_part.as<double>(), rr_part.as<double>());
  else if (vpl <= 4) launch_normal_gemv<T, 4>(ctx, nblk, n, d, A, ld, b, b_stride, beta, w, g_part.as<double>(), rr_part.as<double>());
  else if (vpl <= 8) launch_normal_gemv<T, 8>(ctx, nblk, n, d, A, ld, b, b_stride, beta, w, g_part.as<double>(), rr_part.as<double>());
  else if (vpl <= 16) launch_normal_gemv<T, 16>(ctx, nblk, n, d, A, ld, b, b_stride, beta, w, g_part.as<double>(), rr_part.as<double>());
  else launch_normal_gemv<T, 32>(ctx, nblk, n, d, A, ld, b, b_stride, beta, w, g_part.as<double>(), rr_part.as<double>());
  reduce_parts_kernel<<<grid_for(ctx, d + 1, 256), 256, 0, ctx->stream>>>(nblk, (int)d, g_part.as<double>(),
                                                                            rr_part.as<double>(), g, rr);
  RNLA_CUDA(cudaGetLastError());
  note_launch(ctx, 2);
}
template void normal_gemv<double>(rnla_ctx*, int64_t, int64_t, const double*, int64_t, const double*, int64_t, double,
                                  const double*, double*, double*);
template void normal_gemv<float>(rnla_ctx*, int64_t, int64_t, const float*, int64_t, const float*, int64_t, double,
                                 const double*, double*, double*);

}  // namespace rnla
