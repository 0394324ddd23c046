// srht_tma.cu -- TMA-fed two-pass SRHT for fp32 with padded size 2^18 .. 2^20
// (BASELINE config 2: 2^20 x 1024 -> 4096 rows).
//
// Same algorithm and stage order as srht.cu (reference srht_sketch /
// fwht_inplace, /root/reference/proj/src/sketch.cpp:44-81), different data
// movement: every 2^qlo x 16 tile (64 KB) is moved global -> smem by
// cp.async.bulk.tensor (TMA) boxes of 256 rows x 64 B, transformed out of
// smem, and (low pass) written back with a TMA tensor store. No thread
// holds in-flight loads, so several CTAs per SM keep HBM busy.
//
//  phase A: warp w holds rows 64w..64w+63 of the 16 columns: lane = (row
//           parity p, column c); 32 registers = rows 64w + 2e + p. Stage
//           h = 1 is a warp shuffle (xor 16), stages h = 2..32 in registers.
//  phase B: groups (lo < 64, c) of rows lo + 64m, stages h >= 64 in registers.
// Column tiles are launched in pairs so neighbouring CTAs consume both 64-B
// halves of each 128-B line.
#include <cuda.h>

#include "rnla_internal.h"
#include "srht.h"
#include "util.cuh"

namespace rnla {

namespace {

constexpr int TW = 16;  // fp32 columns per tile (64 B)

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init1(uint32_t bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint32_t bar, uint32_t bytes) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}\n" ::"r"(bar),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait0(uint32_t bar) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "W_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t"
      "@!p bra W_%=;\n\t}\n" ::"r"(bar)
      : "memory");
}
// L2 policies: the input and the last read of the scratch are streamed
// (evict_first); the scratch written by the low pass is kept (evict_last) so
// the high pass finds it in L2.
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ void mbar_wait_parity(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "W_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra W_%=;\n\t}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar,
                                            uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3}], "
      "[%4], %5;\n" ::"r"(dst),
      "l"(map), "r"(c0), "r"(c1), "r"(bar), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            uint32_t bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3, "
      "%4}], [%5], %6;\n" ::"r"(dst),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(bar), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, int c0, int c1, uint32_t src, uint64_t pol) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%1, %2}], [%3], %4;\n" ::"l"(
                   map),
               "r"(c0), "r"(c1), "r"(src), "l"(pol)
               : "memory");
}

// One tile issue (thread 0): the TMA boxes of task (bx, tile) into `sm`, completing on `bar`.
template <int LOGR, bool HI>
__device__ __forceinline__ void fwht_issue(float* sm, uint64_t* bar, const CUtensorMap* src_map, int bx, int tile,
                                           int qlo, int64_t big_n, int64_t c0) {
  constexpr int R = 1 << LOGR;
  mbar_expect(su32(bar), R * TW * 4);
  const uint64_t pol = policy_evict_first();
  for (int b = 0; b < R / 256; ++b) {
    const uint32_t dst = su32(sm + b * 256 * TW);
    if (HI)  // scratch viewed as [jh][il][TW] per strip: rows jh = b*256.. of this il
      tma_load_3d(dst, src_map, 0, bx, tile * (int)(big_n >> qlo) + b * 256, su32(bar), pol);
    else  // input A (row-major n x L): columns c0 + tile*16.., rows bx*R + b*256..
      tma_load_2d(dst, src_map, (int)(c0 + tile * TW), bx * R + b * 256, su32(bar), pol);
  }
}

// The transform of one landed tile (all R/2 threads): phases A and B, then the
// low pass stores the tile to the scratch (TMA) and the high pass writes the
// sampled outputs. Ends with the tile buffer free again.
template <int LOGR, bool HI>
__device__ __forceinline__ void fwht_tile(float* sm, int bx, int tile, int g0, int g1, const CUtensorMap* dst_map,
                                          const int8_t* __restrict__ signs, int64_t n, int64_t big_n, int64_t L,
                                          int64_t c0, const int32_t* __restrict__ grp_t,
                                          const int32_t* __restrict__ grp_hi, float scale, float* __restrict__ out,
                                          int64_t out_rs, int64_t out_cs) {
  constexpr int R = 1 << LOGR;
  constexpr int G = R / 64;  // rows per phase-B group
  constexpr int NT = R / 2;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // ---- phase A ----
  const int p = lane >> 4, c = lane & 15;
  float v[32];
  const int64_t rbase = (int64_t)bx * R;
#pragma unroll
  for (int e = 0; e < 32; ++e) {
    const int r = warp * 64 + 2 * e + p;
    float x = sm[r * TW + c];
    if (!HI) x = (rbase + r < n) ? x * (float)signs[rbase + r] : 0.f;
    v[e] = x;
  }
  // h = 1: partner row differs in bit 0 = the other half-warp
#pragma unroll
  for (int e = 0; e < 32; ++e) {
    const float o = __shfl_xor_sync(0xffffffffu, v[e], 16);
    v[e] = p ? (o - v[e]) : (v[e] + o);  // x + y for the lower row, x - y for the upper
  }
  // h = 2 .. 32: register index bit (h / 2)
#pragma unroll
  for (int hh = 1; hh < 32; hh <<= 1)
#pragma unroll
    for (int e = 0; e < 32; ++e)
      if (!(e & hh)) {
        const float x = v[e], y = v[e + hh];
        v[e] = x + y;
        v[e + hh] = x - y;
      }
  __syncthreads();  // everyone has read the tile
#pragma unroll
  for (int e = 0; e < 32; ++e) sm[(warp * 64 + 2 * e + p) * TW + c] = v[e];
  __syncthreads();

  // ---- phase B: groups (lo, c) = rows lo + 64 m, stages h = 64 .. R/2 ----
#pragma unroll
  for (int k = 0; k < (64 * TW) / NT; ++k) {
    const int g = tid + NT * k;
    const int cc = g & 15, lo = g >> 4;
    float u[G];
#pragma unroll
    for (int m = 0; m < G; ++m) u[m] = sm[(lo + 64 * m) * TW + cc];
#pragma unroll
    for (int hh = 1; hh < G; hh <<= 1)
#pragma unroll
      for (int m = 0; m < G; ++m)
        if (!(m & hh)) {
          const float x = u[m], y = u[m + hh];
          u[m] = x + y;
          u[m + hh] = x - y;
        }
#pragma unroll
    for (int m = 0; m < G; ++m) sm[(lo + 64 * m) * TW + cc] = u[m];
  }
  __syncthreads();
  if (!HI) {
    // tile -> scratch [tile][N][TW] with TMA stores
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      const uint64_t pol = policy_evict_last();
      for (int b = 0; b < R / 256; ++b)
        tma_store_2d(dst_map, 0, (int)(tile * big_n + rbase + b * 256), su32(sm + b * 256 * TW), pol);
      asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
    }
    __syncthreads();
  } else {
    const int64_t col_base = c0 + (int64_t)tile * TW;
    for (int e = tid; e < (g1 - g0) * TW; e += NT) {
      const int g = g0 + e / TW, cc = e % TW;
      const int64_t col = col_base + cc;
      if (col < L) out[(int64_t)grp_t[g] * out_rs + col * out_cs] = sm[grp_hi[g] * TW + cc] * scale;
    }
    __syncthreads();
  }
}

// LOGR = log2 of the rows per tile (9 or 10); R/2 threads; one tile per CTA.
template <int LOGR, bool HI>
__global__ void __launch_bounds__((1 << LOGR) / 2, LOGR == 10 ? 3 : 6) fwht_tma_kernel(
    const __grid_constant__ CUtensorMap src_map, const __grid_constant__ CUtensorMap dst_map,
    const int8_t* __restrict__ signs, int64_t n, int qlo, int64_t big_n, int64_t L, int64_t c0,
    const int32_t* __restrict__ grp_off, const int32_t* __restrict__ grp_t, const int32_t* __restrict__ grp_hi,
    float scale, float* __restrict__ out, int64_t out_rs, int64_t out_cs) {
  extern __shared__ __align__(128) float sm[];  // [R][TW], dense (TMA box layout)
  __shared__ __align__(8) uint64_t bar;
  const int bx = HI ? blockIdx.x : blockIdx.y;   // HI: il; LO: row block
  const int tile = HI ? blockIdx.y : blockIdx.x;  // column tile within the strip
  int g0 = 0, g1 = 0;
  if (HI) {
    g0 = grp_off[bx];
    g1 = grp_off[bx + 1];
    if (g0 == g1) return;  // no sampled output has these low bits (uniform per CTA)
  }
  if (threadIdx.x == 0) {
    mbar_init1(su32(&bar));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) fwht_issue<LOGR, HI>(sm, &bar, &src_map, bx, tile, qlo, big_n, c0);
  mbar_wait0(su32(&bar));
  fwht_tile<LOGR, HI>(sm, bx, tile, g0, g1, &dst_map, signs, n, big_n, L, c0, grp_t, grp_hi, scale, out, out_rs,
                      out_cs);
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
  static EncodeFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<EncodeFn>(p);
  }();
  return fn;
}

void make_map(CUtensorMap* m, void* base, int rank, const cuuint64_t* dims, const cuuint64_t* strides_bytes,
              const cuuint32_t* box) {
  const cuuint32_t es[3] = {1, 1, 1};
  const CUresult r = encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, (cuuint32_t)rank, base, dims, strides_bytes, box,
                                 es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
}

}  // namespace

bool tma_encode_available() { return encode_fn() != nullptr; }

void tma_map_rows_f32(CUtensorMap* m, const float* base, int64_t rows, int64_t cols, int64_t ld, uint32_t box_cols,
                      uint32_t box_rows) {
  const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
  const cuuint32_t box[2] = {box_cols, box_rows};
  make_map(m, const_cast<float*>(base), 2, dims, strides, box);
}

namespace {

template <int LOGR, bool HI>
void launch_pass(rnla_ctx* ctx, dim3 grid, const CUtensorMap& src, const CUtensorMap& dst, const SrhtPlan& plan,
                 int64_t L, int64_t c0, float scale, float* out, int64_t out_rs, int64_t out_cs) {
  constexpr int R = 1 << LOGR;
  const size_t smem = (size_t)R * TW * sizeof(float);
  auto k = fwht_tma_kernel<LOGR, HI>;
  ensure_dyn_smem((const void*)k, smem);
  k<<<grid, R / 2, smem, ctx->stream>>>(src, dst, plan.signs.as<int8_t>(), plan.n, plan.qlo, plan.big_n, L, c0,
                                        plan.grp_off.as<int32_t>(), plan.grp_t.as<int32_t>(),
                                        plan.grp_hi.as<int32_t>(), scale, out, out_rs, out_cs);
  RNLA_CUDA(cudaGetLastError());
  note_launch(ctx);
}

}  // namespace

// fp32, qlo, qhi in {9, 10}, 16-B aligned rows; false when not applicable.
bool srht_tma_f32(rnla_ctx* ctx, const SrhtPlan& plan, const float* in, int64_t ld, int64_t L, float* out,
                  int64_t out_rs, int64_t out_cs) {
  auto ok = [](int q) { return q == 9 || q == 10; };
  if (!ok(plan.qlo) || !ok(plan.qhi) || !encode_fn() || std::getenv("RNLA_SRHT_NO_TMA")) return false;
  if ((reinterpret_cast<uintptr_t>(in) & 15) || ((ld * 4) % 16) || plan.n > (int64_t)INT32_MAX) return false;
  const int64_t big_n = plan.big_n;
  const int64_t total_tiles = (L + TW - 1) / TW;
  // strip of column tiles per launch pair. Measured on cfg2 (2^20 x 1024):
  // 64 MB (L2-sized) 3.82 ms, 128 MB 3.07, 256 MB 2.80, 1 GB 2.58, 4 GB 2.56 --
  // wide launches (no wave tails) beat L2 residency of the scratch.
  const int64_t strip_mb = srht_strip_mb();
  int64_t tps = std::max<int64_t>(1, (strip_mb << 20) / (big_n * TW * 4));
  if (tps > 1) tps = tps / 2 * 2;  // whole 128-B lines per strip
  tps = std::min(tps, total_tiles);
  DevBuf scratch(sizeof(float) * (size_t)(big_n * TW * tps), ctx->stream);
  // input map: dims {L, n} (cols inner), row stride ld*4 bytes, box {16, 256}
  CUtensorMap amap, smap_st, smap_ld;
  {
    const cuuint64_t dims[2] = {(cuuint64_t)L, (cuuint64_t)plan.n};
    const cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
    const cuuint32_t box[2] = {TW, 256};
    make_map(&amap, const_cast<float*>(in), 2, dims, strides, box);
  }
  {  // scratch as 2-D [tps * N][16] for the stores
    const cuuint64_t dims[2] = {TW, (cuuint64_t)(tps * big_n)};
    const cuuint64_t strides[1] = {TW * 4};
    const cuuint32_t box[2] = {TW, 256};
    make_map(&smap_st, scratch.p, 2, dims, strides, box);
  }
  {  // scratch as 3-D [tps * N / 2^qlo][2^qlo][16] for the strided high-pass loads
    const int64_t lo = (int64_t)1 << plan.qlo;
    const cuuint64_t dims[3] = {TW, (cuuint64_t)lo, (cuuint64_t)(tps * big_n / lo)};
    const cuuint64_t strides[2] = {TW * 4, (cuuint64_t)(lo * TW * 4)};
    const cuuint32_t box[3] = {TW, 1, 256};
    make_map(&smap_ld, scratch.p, 3, dims, strides, box);
  }
  const float scale = (float)(1.0 / std::sqrt((double)plan.s));
  for (int64_t t0 = 0; t0 < total_tiles; t0 += tps) {
    const int64_t nt = std::min(tps, total_tiles - t0);
    const int64_t c0 = t0 * TW;
    const dim3 g1((unsigned)nt, (unsigned)(big_n >> plan.qlo)), g2((unsigned)((int64_t)1 << plan.qlo), (unsigned)nt);
    if (plan.qlo == 9) launch_pass<9, false>(ctx, g1, amap, smap_st, plan, L, c0, scale, out, out_rs, out_cs);
    else launch_pass<10, false>(ctx, g1, amap, smap_st, plan, L, c0, scale, out, out_rs, out_cs);
    if (plan.qhi == 9) launch_pass<9, true>(ctx, g2, smap_ld, smap_st, plan, L, c0, scale, out, out_rs, out_cs);
    else launch_pass<10, true>(ctx, g2, smap_ld, smap_st, plan, L, c0, scale, out, out_rs, out_cs);
  }
  return true;
}

}  // namespace rnla
