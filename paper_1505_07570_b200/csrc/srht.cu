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
#include "dist.h"
#include "rnla_internal.h"
#include "srht.h"
#include "util.cuh"

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

constexpr int ilog2c(int v) { return v <= 1 ? 0 : 1 + ilog2c(v / 2); }

// Register-blocked pass over R = 2^LOGR logical rows x W columns, 256 threads.
//  phase A: thread (c = tid % W, rb = tid / W) loads logical rows rb*E..rb*E+E-1
//           of column c straight from global (sign flip fused for the low pass),
//           runs the log2(E) lowest stages in registers, stores to smem;
//  phase B: thread owns groups (lo, c) = logical rows lo + E*m, m < R/E, and
//           runs the remaining stages in registers.
// Low pass (HI = false): logical row i of CTA blk is physical row blk*R + i of
// the input; the result goes to the scratch strip. High pass (HI = true):
// logical row i is physical row i*2^qlo + il (il = blockIdx.x) of the scratch;
// only sampled outputs with low bits il are written (x 1/sqrt(s)). Stages run
// h = 1, 2, 4, ... with x+y / x-y exactly like fwht_inplace.
template <class T>
constexpr int fwht_rows_per_thread() { return sizeof(T) == 8 ? 32 : 64; }
template <class T, int LOGR, int W>
constexpr int fwht_threads() { return (1 << LOGR) * W / fwht_rows_per_thread<T>(); }

template <class T, int LOGR, int W, bool HI>
__global__ void __launch_bounds__(fwht_threads<T, LOGR, W>()) fwht_reg_kernel(const T* __restrict__ src, int64_t ld, int64_t n, int64_t L,
                                                       const int8_t* __restrict__ signs, int qlo, int64_t c0,
                                                       T* __restrict__ scratch, int64_t big_n,
                                                       const int32_t* __restrict__ grp_off,
                                                       const int32_t* __restrict__ grp_t,
                                                       const int32_t* __restrict__ grp_hi, double scale,
                                                       T* __restrict__ out, int64_t out_rs, int64_t out_cs) {
  constexpr int R = 1 << LOGR;
  constexpr int NT = fwht_threads<T, LOGR, W>();
  constexpr int E = R * W / NT;  // rows per thread in phase A
  constexpr int G = R / E;        // rows per group in phase B
  constexpr int NG = E * W;               // groups in phase B
  constexpr int GPT = (NG + NT - 1) / NT;
  // 16-bank shift per E-row block when a row chunk is narrower than the 32 banks
  constexpr int PADB = W * (int)sizeof(T) >= 128 ? 0 : 64 / (int)sizeof(T);
  static_assert(E >= 1 && G >= 1 && GPT >= 1, "bad tile");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sm = reinterpret_cast<T*>(smem_raw);
  auto sidx = [](int i, int c) { return i * W + c + (i / E) * PADB; };
  // Low pass: grid (tile, row block) so the CTAs of neighbouring column tiles
  // run together and consume both halves of each 128-B line; high pass: grid
  // (il, tile) so neighbouring il (adjacent scratch rows) run together.
  const int bx = HI ? blockIdx.x : blockIdx.y;
  const int tile = HI ? blockIdx.y : blockIdx.x;
  int g0 = 0, g1 = 0;
  if (HI) {
    g0 = grp_off[bx];
    g1 = grp_off[bx + 1];
    if (g0 == g1) return;  // no sampled output has these low bits (uniform per CTA)
  }
  const int64_t col_base = c0 + (int64_t)tile * W;
  const T* tsrc = HI ? src + (int64_t)tile * big_n * W : src;
  {
    const int c = threadIdx.x % W, rb = threadIdx.x / W;
    T v[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int i = rb * E + e;
      if (HI) {
        const int64_t j = ((int64_t)i << qlo) + bx;
        v[e] = tsrc[j * W + c];
      } else {
        const int64_t j = (int64_t)bx * R + i, col = col_base + c;
        v[e] = (j < n && col < L) ? __ldcs(src + j * ld + col) * (T)signs[j] : T(0);
      }
    }
#pragma unroll
    for (int h = 1; h < E; h <<= 1)
#pragma unroll
      for (int e = 0; e < E; ++e)
        if (!(e & h)) {
          const T x = v[e], y = v[e + h];
          v[e] = x + y;
          v[e + h] = x - y;
        }
#pragma unroll
    for (int e = 0; e < E; ++e) sm[sidx(rb * E + e, c)] = v[e];
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < GPT; ++k) {
    const int g = threadIdx.x + NT * k;
    if (g >= NG) break;
    const int c = g % W, lo = g / W;
    T u[G];
#pragma unroll
    for (int m = 0; m < G; ++m) u[m] = sm[sidx(lo + E * m, c)];
#pragma unroll
    for (int h = 1; h < G; h <<= 1)
#pragma unroll
      for (int m = 0; m < G; ++m)
        if (!(m & h)) {
          const T x = u[m], y = u[m + h];
          u[m] = x + y;
          u[m + h] = x - y;
        }
    if (HI) {
#pragma unroll
      for (int m = 0; m < G; ++m) sm[sidx(lo + E * m, c)] = u[m];
    } else {
      T* dst = scratch + ((int64_t)tile * big_n + (int64_t)bx * R) * W;
#pragma unroll
      for (int m = 0; m < G; ++m) dst[(int64_t)(lo + E * m) * W + c] = u[m];
    }
  }
  if (HI) {
    __syncthreads();
    for (int e = threadIdx.x; e < (g1 - g0) * W; e += NT) {
      const int g = g0 + e / W, c = e % W;
      const int64_t col = col_base + c;
      if (col < L) out[(int64_t)grp_t[g] * out_rs + col * out_cs] = (T)((double)sm[sidx(grp_hi[g], c)] * scale);
    }
  }
}

template <class T, int LOGR, int W, bool HI>
size_t fwht_reg_smem() {
  constexpr int R = 1 << LOGR, E = fwht_rows_per_thread<T>();
  constexpr int PADB = W * (int)sizeof(T) >= 128 ? 0 : 64 / (int)sizeof(T);
  return sizeof(T) * ((size_t)R * W + (size_t)(R / E) * PADB);
}

template <class T, int LOGR, int W, bool HI>
void launch_fwht_reg(rnla_ctx* ctx, dim3 grid, const T* src, int64_t ld, int64_t n, int64_t L,
                     const int8_t* signs, int qlo, int64_t c0, T* scratch, int64_t big_n, const SrhtPlan& plan,
                     double scale, T* out, int64_t out_rs, int64_t out_cs) {
  const size_t smem = fwht_reg_smem<T, LOGR, W, HI>();
  auto kern = fwht_reg_kernel<T, LOGR, W, HI>;
  ensure_dyn_smem((const void*)kern, smem);
  kern<<<grid, fwht_threads<T, LOGR, W>(), smem, ctx->stream>>>(src, ld, n, L, signs, qlo, c0, scratch, big_n, plan.grp_off.as<int32_t>(),
                                         plan.grp_t.as<int32_t>(), plan.grp_hi.as<int32_t>(), scale, out, out_rs,
                                         out_cs);
  RNLA_CUDA(cudaGetLastError());
  note_launch(ctx);
}

// Fast register path for log2 R in {9, 10, 11} (padded dimension 2^18 .. 2^22).
template <class T, int W>
void srht_fast_w(rnla_ctx* ctx, const SrhtPlan& plan, const T* in, int64_t ld, int64_t L, T* out, int64_t out_rs,
                 int64_t out_cs) {
  const int64_t big_n = plan.big_n;
  const int64_t tile_bytes = big_n * W * (int64_t)sizeof(T);
  // a strip = the column tiles that together cover whole 128-B lines
  // (launched adjacently), sized to ~128 MB of scratch so it mostly stays in L2
  const int64_t line_tiles = std::max<int64_t>(1, 128 / (W * (int64_t)sizeof(T)));
  int64_t tiles_per_strip =
      std::max<int64_t>(line_tiles, (srht_strip_mb() << 20) / tile_bytes / line_tiles * line_tiles);
  const int64_t total_tiles = (L + W - 1) / W;
  tiles_per_strip = std::min(tiles_per_strip, total_tiles);
  DevBuf scratch(sizeof(T) * (size_t)(big_n * W * tiles_per_strip), ctx->stream);
  const double scale = 1.0 / std::sqrt((double)plan.s);
  for (int64_t t0 = 0; t0 < total_tiles; t0 += tiles_per_strip) {
    const int64_t nt = std::min(tiles_per_strip, total_tiles - t0);
    const int64_t c0 = t0 * W;
    const dim3 g1((unsigned)nt, (unsigned)(big_n >> plan.qlo)), g2((unsigned)((int64_t)1 << plan.qlo), (unsigned)nt);
#define RNLA_PASS(LOGR, HI, GRID)                                                                                 \
  launch_fwht_reg<T, LOGR, W, HI>(ctx, GRID, HI ? scratch.as<T>() : in, ld, plan.n, L, plan.signs.as<int8_t>(), \
                                  plan.qlo, c0, scratch.as<T>(), big_n, plan, scale, out, out_rs, out_cs)
    if (plan.qlo == 9) RNLA_PASS(9, false, g1);
    else if (plan.qlo == 10) RNLA_PASS(10, false, g1);
    else RNLA_PASS(11, false, g1);
    if (plan.qhi == 9) RNLA_PASS(9, true, g2);
    else if (plan.qhi == 10) RNLA_PASS(10, true, g2);
    else RNLA_PASS(11, true, g2);
#undef RNLA_PASS
  }
}

// Fast register path for log2 R in {9, 10, 11} (padded dimension 2^18 .. 2^22).
// One tile width for both passes (the scratch layout is [tile][N][W]).
template <class T>
bool srht_fast(rnla_ctx* ctx, const SrhtPlan& plan, const T* in, int64_t ld, int64_t L, T* out, int64_t out_rs,
               int64_t out_cs) {
  auto ok = [](int q) { return q >= 9 && q <= 11; };
  if (!ok(plan.qlo) || !ok(plan.qhi)) return false;
  constexpr int W = 64 / sizeof(T);  // 64-B row chunks; paired tiles cover each 128-B line
  if (plan.qlo == 11 || plan.qhi == 11) srht_fast_w<T, W / 2>(ctx, plan, in, ld, L, out, out_rs, out_cs);
  else srht_fast_w<T, W>(ctx, plan, in, ld, L, out, out_rs, out_cs);
  return true;
}

}  // namespace

SrhtPlan::SrhtPlan(rnla_ctx* ctx, int64_t n_, int64_t s_, uint64_t seed_) : n(n_), s(s_), seed(seed_) {
  big_n = next_pow2(n);
  require(s >= 1 && s <= big_n, "srht_sketch: s > padded dimension");
  std::vector<int8_t> sg((size_t)std::max<int64_t>(n, 1));
  std::vector<int64_t> idx((size_t)s);
  srht_operator_host(seed, n, s, sg.data(), idx.data());
  host_idx = idx;
  build(ctx, sg.data(), idx.data());
}

SrhtPlan::SrhtPlan(rnla_ctx* ctx, const int8_t* block_signs, int64_t present, int64_t block, const int64_t* idx,
                   int64_t s_, int64_t block_off_)
    : n(present), s(s_), big_n(block), block_off(block_off_) {
  std::vector<int64_t> loc((size_t)s);
  std::vector<double> sgn((size_t)s);
  for (int64_t t = 0; t < s; ++t) {
    loc[(size_t)t] = idx[t] & (block - 1);
    sgn[(size_t)t] = (__builtin_popcountll((unsigned long long)(block_off & idx[t])) & 1) ? -1.0 : 1.0;
  }
  host_idx = loc;
  out_sign = DevBuf(sizeof(double) * s, ctx->stream);
  RNLA_CUDA(cudaMemcpyAsync(out_sign.p, sgn.data(), sizeof(double) * s, cudaMemcpyHostToDevice, ctx->stream));
  build(ctx, block_signs, loc.data());
}

void SrhtPlan::build(rnla_ctx* ctx, const int8_t* sg, const int64_t* idx) {
  q = 0;
  while (((int64_t)1 << q) < big_n) ++q;
  require(q <= 22, "srht_sketch: padded dimension above 2^22 is not supported");
  qlo = (q + 1) / 2;
  qhi = q - qlo;
  const int64_t R = (int64_t)1 << qlo;
  std::vector<int32_t> off((size_t)R + 1, 0), gt((size_t)s), gh((size_t)s);
  for (int64_t t = 0; t < s; ++t) off[(size_t)(idx[t] & (R - 1)) + 1]++;
  for (int64_t i = 0; i < R; ++i) off[(size_t)i + 1] += off[(size_t)i];
  std::vector<int32_t> cur(off.begin(), off.end() - 1);
  for (int64_t t = 0; t < s; ++t) {
    const int64_t lo = idx[t] & (R - 1);
    const int32_t g = cur[(size_t)lo]++;
    gt[(size_t)g] = (int32_t)t;
    gh[(size_t)g] = (int32_t)(idx[t] >> qlo);
  }
  const size_t ns = (size_t)std::max<int64_t>(n, 1);
  signs = DevBuf(ns, ctx->stream);
  grp_off = DevBuf(sizeof(int32_t) * off.size(), ctx->stream);
  grp_t = DevBuf(sizeof(int32_t) * gt.size(), ctx->stream);
  grp_hi = DevBuf(sizeof(int32_t) * gh.size(), ctx->stream);
  if (n > 0) RNLA_CUDA(cudaMemcpyAsync(signs.p, sg, (size_t)n, cudaMemcpyHostToDevice, ctx->stream));
  RNLA_CUDA(cudaMemcpyAsync(grp_off.p, off.data(), sizeof(int32_t) * off.size(), cudaMemcpyHostToDevice, ctx->stream));
  RNLA_CUDA(cudaMemcpyAsync(grp_t.p, gt.data(), sizeof(int32_t) * gt.size(), cudaMemcpyHostToDevice, ctx->stream));
  RNLA_CUDA(cudaMemcpyAsync(grp_hi.p, gh.data(), sizeof(int32_t) * gh.size(), cudaMemcpyHostToDevice, ctx->stream));
  RNLA_CUDA(cudaStreamSynchronize(ctx->stream));  // host vectors go out of scope
}

template <class T>
void srht_segments(rnla_ctx* ctx, const SrhtPlan& plan, const T* in, int64_t ld, int64_t L, T* out, int64_t out_rs,
                   int64_t out_cs) {
  if (L == 0) return;
  if constexpr (std::is_same<T, float>::value) {
    if (!std::getenv("RNLA_SRHT_GENERIC") && srht_acc_f32(ctx, plan, in, ld, L, out, out_rs, out_cs)) return;
    if (!std::getenv("RNLA_SRHT_GENERIC") && srht_tma_f32(ctx, plan, in, ld, L, out, out_rs, out_cs)) return;
  }
  if (!std::getenv("RNLA_SRHT_GENERIC") && srht_fast<T>(ctx, plan, in, ld, L, out, out_rs, out_cs)) return;
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
  ensure_dyn_smem((const void*)srht_lo_kernel<T, W>, smem_lo);
  ensure_dyn_smem((const void*)srht_hi_kernel<T, W>, smem_hi);
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

namespace {
template <class T>
__global__ void signed_accumulate_kernel(int64_t s, int64_t L, const T* __restrict__ tmp,
                                         const double* __restrict__ sign, T* __restrict__ acc) {
  const int64_t total = s * L;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x)
    acc[e] += (T)sign[e / L] * tmp[e];
}
}  // namespace

// Row-sharded SRHT. With j = o + jl for a block of
// 2^b rows at an offset o that is a multiple of 2^b, and any t:
//   (-1)^popcount(j & t) = (-1)^popcount(o & t) * (-1)^popcount(jl & (t mod 2^b)),
// so this rank's rows, cut into aligned power-of-two blocks, each contribute
// sign_t * [H_{2^b} (signs . x)]_{t mod 2^b} to every sampled output t. The
// partial outputs are summed over ranks by one allreduce (s x L).
template <class T>
void srht_rows_sharded(rnla_ctx* ctx, const T* in, int64_t ld, int64_t n_local, int64_t L, int64_t row_off,
                       int64_t n_total, int64_t s, uint64_t seed, T* out, int64_t out_rs, int64_t out_cs) {
  const int64_t big_n = next_pow2(n_total);
  require(s >= 1 && s <= big_n, "srht_sketch: s > padded dimension");
  std::vector<int8_t> sg((size_t)std::max<int64_t>(n_total, 1));
  std::vector<int64_t> idx((size_t)s);
  srht_operator_host(seed, n_total, s, sg.data(), idx.data());
  DevBuf acc(sizeof(T) * s * std::max<int64_t>(L, 1), ctx->stream), tmp(sizeof(T) * s * std::max<int64_t>(L, 1),
                                                                          ctx->stream);
  RNLA_CUDA(cudaMemsetAsync(acc.p, 0, sizeof(T) * s * L, ctx->stream));
  const int64_t end = row_off + n_local;
  const int64_t limit = end == n_total ? big_n : end;  // the last rank owns the zero padding
  for (int64_t cur = row_off; cur < end;) {
    int64_t b = cur == 0 ? big_n : (cur & -cur);
    while (cur + b > limit) b >>= 1;
    const int64_t present = std::min(b, end - cur);
    SrhtPlan plan(ctx, sg.data() + cur, present, b, idx.data(), s, cur);
    srht_segments<T>(ctx, plan, in + (cur - row_off) * ld, ld, L, tmp.as<T>(), L, 1);
    signed_accumulate_kernel<T><<<grid_for(ctx, s * L, 256), 256, 0, ctx->stream>>>(s, L, tmp.as<T>(),
                                                                                     plan.out_sign.as<double>(),
                                                                                     acc.as<T>());
    RNLA_CUDA(cudaGetLastError());
    note_launch(ctx);
    cur += b;
  }
  allreduce_sum(ctx, acc.p, (size_t)(s * L), std::is_same<T, double>::value ? RNLA_F64 : RNLA_F32);
  copy2d<T>(ctx, s, L, acc.as<T>(), L, 1, out, out_rs, out_cs);
  RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
}
template void srht_rows_sharded<double>(rnla_ctx*, const double*, int64_t, int64_t, int64_t, int64_t, int64_t, int64_t,
                                        uint64_t, double*, int64_t, int64_t);
template void srht_rows_sharded<float>(rnla_ctx*, const float*, int64_t, int64_t, int64_t, int64_t, int64_t, int64_t,
                                       uint64_t, float*, int64_t, int64_t);

}  // namespace rnla
