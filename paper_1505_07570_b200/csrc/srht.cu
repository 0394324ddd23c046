// srht.cu -- subsampled randomized Hadamard transform of n segments.
//
// Reference: srht_sketch + fwht_inplace, /root/reference/proj/src/sketch.cpp:44-81.
// For every position c of the segments: x_j = seg_j[c] * sign_j (zero-padded
// to N = 2^q), unnormalized Sylvester FWHT with stages h = 1, 2, 4, ..., and
// out_t[c] = x[idx_t] / sqrt(s).
//
// B200 design: the transform axis crosses segments, so a
// column strip of W positions is transformed in two shared-memory passes,
// H_N = H_{2^qhi} (x) H_{2^qlo}:
//   pass 1 (lo): CTA per (block of 2^qlo consecutive segments, strip): sign
//          flip fused on load, stages h < 2^qlo in smem, result to scratch T;
//   pass 2 (hi): CTA per (low index il, strip): gathers the 2^qhi segments
//          jh*2^qlo + il of T, stages h >= 2^qlo in smem, and writes ONLY the
//          sampled outputs whose low bits are il (gather-on-store), scaled.
// Stages run in the reference order with the same x+y / x-y operations, so
// the fp64 result is bit-identical to the reference's loop. Strips are
// processed in groups small enough for T to stay resident in the 126 MB L2.
#include "rnla_internal.h"
#include "srht.h"

namespace rnla {

namespace {

template <class T, int W>
__global__ void __launch_bounds__(256) srht_lo_kernel(const T* __restrict__ in, int64_t ld, int64_t n, int64_t L,
                                                      const int8_t* __restrict__ signs, int qlo, int64_t c0,
                                                      T* __restrict__ scratch) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sm = reinterpret_cast<T*>(smem_raw);
  const int R = 1 << qlo;
  const int64_t jb = (int64_t)blockIdx.x << qlo;
  const int64_t cb = c0 + (int64_t)blockIdx.y * W;
  for (int e = threadIdx.x; e < R * W; e += blockDim.x) {
    const int r = e / W, c = e % W;
    const int64_t j = jb + r, col = cb + c;
    T v = T(0);
    if (j < n && col < L) v = __ldcs(in + j * ld + col) * (T)signs[j];
    sm[e] = v;
  }
  __syncthreads();
  for (int h = 1; h < R; h <<= 1) {
    for (int e = threadIdx.x; e < (R / 2) * W; e += blockDim.x) {
      const int pr = e / W, c = e % W;
      const int lo = (pr / h) * (2 * h) + (pr % h);
      const T x = sm[lo * W + c], y = sm[(lo + h) * W + c];
      sm[lo * W + c] = x + y;
      sm[(lo + h) * W + c] = x - y;
    }
    __syncthreads();
  }
  // scratch layout: [N rows][W] per strip tile (tile blockIdx.y)
  T* dst = scratch + ((int64_t)blockIdx.y * ((int64_t)gridDim.x << qlo) + jb) * W;
  for (int e = threadIdx.x; e < R * W; e += blockDim.x) dst[e] = sm[e];
}

// samples grouped by low index: for il, entries [grp_off[il], grp_off[il+1])
// of grp_t (output row t) and grp_hi (high part of idx_t).
template <class T, int W>
__global__ void __launch_bounds__(256) srht_hi_kernel(const T* __restrict__ scratch, int qlo, int qhi, int64_t L,
                                                      int64_t c0, const int32_t* __restrict__ grp_off,
                                                      const int32_t* __restrict__ grp_t,
                                                      const int32_t* __restrict__ grp_hi, double scale,
                                                      T* __restrict__ out, int64_t out_rs, int64_t out_cs) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sm = reinterpret_cast<T*>(smem_raw);
  const int il = blockIdx.x;
  const int g0 = grp_off[il], g1 = grp_off[il + 1];
  if (g0 == g1) return;  // no sampled output has these low bits
  const int R = 1 << qhi;
  const int64_t big_n = (int64_t)1 << (qlo + qhi);
  const T* src = scratch + (int64_t)blockIdx.y * big_n * W;
  for (int e = threadIdx.x; e < R * W; e += blockDim.x) {
    const int r = e / W, c = e % W;
    sm[e] = src[(((int64_t)r << qlo) + il) * W + c];
  }
  __syncthreads();
  for (int h = 1; h < R; h <<= 1) {
    for (int e = threadIdx.x; e < (R / 2) * W; e += blockDim.x) {
      const int pr = e / W, c = e % W;
      const int lo = (pr / h) * (2 * h) + (pr % h);
      const T x = sm[lo * W + c], y = sm[(lo + h) * W + c];
      sm[lo * W + c] = x + y;
      sm[(lo + h) * W + c] = x - y;
    }
    __syncthreads();
  }
  const int64_t cb = c0 + (int64_t)blockIdx.y * W;
  for (int e = threadIdx.x; e < (g1 - g0) * W; e += blockDim.x) {
    const int g = g0 + e / W, c = e % W;
    const int64_t col = cb + c;
    if (col < L) out[(int64_t)grp_t[g] * out_rs + col * out_cs] = (T)((double)sm[grp_hi[g] * W + c] * scale);
  }
}

}  // namespace

SrhtPlan::SrhtPlan(rnla_ctx* ctx, int64_t n_, int64_t s_, uint64_t seed_) : n(n_), s(s_), seed(seed_) {
  big_n = next_pow2(n);
  require(s >= 1 && s <= big_n, "srht_sketch: s > padded dimension");
  q = 0;
  while (((int64_t)1 << q) < big_n) ++q;
  require(q <= 22, "srht_sketch: padded dimension above 2^22 is not supported");
  qlo = (q + 1) / 2;
  qhi = q - qlo;
  std::vector<int8_t> sg((size_t)std::max<int64_t>(n, 1));
  std::vector<int64_t> idx((size_t)s);
  srht_operator_host(seed, n, s, sg.data(), idx.data());
  host_idx = idx;
  const int64_t R = (int64_t)1 << qlo;
  std::vector<int32_t> off((size_t)R + 1, 0), gt((size_t)s), gh((size_t)s);
  for (int64_t t = 0; t < s; ++t) off[(size_t)(idx[(size_t)t] & (R - 1)) + 1]++;
  for (int64_t i = 0; i < R; ++i) off[(size_t)i + 1] += off[(size_t)i];
  std::vector<int32_t> cur(off.begin(), off.end() - 1);
  for (int64_t t = 0; t < s; ++t) {
    const int64_t lo = idx[(size_t)t] & (R - 1);
    const int32_t g = cur[(size_t)lo]++;
    gt[(size_t)g] = (int32_t)t;
    gh[(size_t)g] = (int32_t)(idx[(size_t)t] >> qlo);
  }
  signs = DevBuf(sg.size(), ctx->stream);
  grp_off = DevBuf(sizeof(int32_t) * off.size(), ctx->stream);
  grp_t = DevBuf(sizeof(int32_t) * gt.size(), ctx->stream);
  grp_hi = DevBuf(sizeof(int32_t) * gh.size(), ctx->stream);
  RNLA_CUDA(cudaMemcpyAsync(signs.p, sg.data(), sg.size(), cudaMemcpyHostToDevice, ctx->stream));
  RNLA_CUDA(cudaMemcpyAsync(grp_off.p, off.data(), sizeof(int32_t) * off.size(), cudaMemcpyHostToDevice, ctx->stream));
  RNLA_CUDA(cudaMemcpyAsync(grp_t.p, gt.data(), sizeof(int32_t) * gt.size(), cudaMemcpyHostToDevice, ctx->stream));
  RNLA_CUDA(cudaMemcpyAsync(grp_hi.p, gh.data(), sizeof(int32_t) * gh.size(), cudaMemcpyHostToDevice, ctx->stream));
  RNLA_CUDA(cudaStreamSynchronize(ctx->stream));  // host vectors go out of scope
}

template <class T>
void srht_segments(rnla_ctx* ctx, const SrhtPlan& plan, const T* in, int64_t ld, int64_t L, T* out, int64_t out_rs,
                   int64_t out_cs) {
  if (L == 0) return;
  constexpr int W = sizeof(T) == 8 ? 8 : 16;
  const int64_t big_n = plan.big_n;
  // Column tiles per strip: keep the strip's scratch (big_n * W * tiles) within ~48 MB of L2.
  const int64_t tile_bytes = big_n * W * (int64_t)sizeof(T);
  int64_t tiles_per_strip = std::max<int64_t>(1, ((int64_t)48 << 20) / tile_bytes);
  const int64_t total_tiles = (L + W - 1) / W;
  tiles_per_strip = std::min(tiles_per_strip, total_tiles);
  DevBuf scratch(sizeof(T) * (size_t)(big_n * W * tiles_per_strip), ctx->stream);
  const double scale = 1.0 / std::sqrt((double)plan.s);
  const size_t smem_lo = sizeof(T) * ((size_t)1 << plan.qlo) * W;
  const size_t smem_hi = sizeof(T) * ((size_t)1 << plan.qhi) * W;
  RNLA_CUDA(cudaFuncSetAttribute(srht_lo_kernel<T, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_lo));
  RNLA_CUDA(cudaFuncSetAttribute(srht_hi_kernel<T, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_hi));
  for (int64_t t0 = 0; t0 < total_tiles; t0 += tiles_per_strip) {
    const int64_t nt = std::min(tiles_per_strip, total_tiles - t0);
    const int64_t c0 = t0 * W;
    dim3 g1((unsigned)(big_n >> plan.qlo), (unsigned)nt);
    srht_lo_kernel<T, W><<<g1, 256, smem_lo, ctx->stream>>>(in, ld, plan.n, L, plan.signs.as<int8_t>(), plan.qlo, c0,
                                                             scratch.as<T>());
    RNLA_CUDA(cudaGetLastError());
    dim3 g2((unsigned)((int64_t)1 << plan.qlo), (unsigned)nt);
    srht_hi_kernel<T, W><<<g2, 256, smem_hi, ctx->stream>>>(scratch.as<T>(), plan.qlo, plan.qhi, L, c0,
                                                             plan.grp_off.as<int32_t>(), plan.grp_t.as<int32_t>(),
                                                             plan.grp_hi.as<int32_t>(), scale, out, out_rs, out_cs);
    RNLA_CUDA(cudaGetLastError());
    note_launch(ctx, 2);
  }
}

template void srht_segments<double>(rnla_ctx*, const SrhtPlan&, const double*, int64_t, int64_t, double*, int64_t,
                                    int64_t);
template void srht_segments<float>(rnla_ctx*, const SrhtPlan&, const float*, int64_t, int64_t, float*, int64_t,
                                   int64_t);

}  // namespace rnla
