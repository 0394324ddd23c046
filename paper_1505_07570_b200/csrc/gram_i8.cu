// gram_i8.cu -- exact Gram products of RBF kernel columns on the int8
// tensor cores (tcgen05.mma kind::i8, s32 accumulation in TMEM): the config-4
// Nystrom C'C with C = K[:, S] (hard part 8).
//
// The reference evaluates C entry by entry (src/spsd.cpp:58-72) and forms
// L = C U Lambda^-1/2 (:209-215); approx_eig needs L'L = T'(C'C)T. At the
// reference's eigenvalue floor W^+ keeps eigenvalues down to ~1e-11 lam_max,
// so C'C must be accurate to fp64 level: fp32 (or BF16x3) accumulation fails
// by orders of magnitude (SURVEY hard part 8). Here every kernel entry
// x in [0, 1] is split into three exact base-128 digits
//     x_q = m0 2^-7 + m1 2^-14 + m2 2^-21,   m0 in [0, 128] (u8), m1, m2 in [-64, 64] (s8),
// with |x - x_q| <= 2^-22 (the fp32 entry itself carries ~2.5e-7 of rounding
// from its 64-term dot product). The Gram of the digit matrices is computed
// EXACTLY: the nine digit products accumulate into five s32 TMEM accumulators
// by digit weight (classes s + t = 0..4), which cannot overflow over K chunks
// of 65536 rows (|class sum| <= 20480 per row), and are combined in fp64 as
//     G = sum_k A_k 2^-(7k + 14).
// W = K[S, S] is formed from the same digits (dequantized exactly in fp64), so
// the Gram and W describe the same quantized kernel matrix.
//
// Kernels:
//  * rbf_digits_kernel: 64 x 64 RBF tile (sequential FMA chain per dot, the
//    same arithmetic as rbf_tile_kernel), digits staged in shared memory and
//    stored as three column-major int8 planes plane[d][p * pitch + i];
//  * gram_i8_kernel: one 128 x 96 tile of G over one K chunk; warp 0 = TMA
//    producer (SWIZZLE_64B boxes of 64 k x rows, 3 digit planes of A and B per
//    stage, 5 stages), warp 1 = MMA issuer (2 k-steps x 9 digit pairs per
//    stage), warps 2-5 = epilogue (tcgen05.ld of the 5 accumulators, fp64
//    combination, one fp64 partial tile per K chunk);
//  * gram_reduce_kernel: sums the K-chunk partials in a fixed order and
//    writes G and its mirror (bitwise symmetric, deterministic).
#include <cuda.h>

#include "rbf.cuh"
#include "util.cuh"

namespace rnla {

namespace {

constexpr int GM = 128, GN = 96, GBK = 64, GND = 3, GSTAGES = 5, GCLS = 2 * GND - 1;
constexpr int A_TILE = GM * GBK, B_TILE = GN * GBK;            // bytes per digit plane tile
constexpr int STAGE_BYTES = GND * (A_TILE + B_TILE);           // 43008 (1024-aligned)
constexpr int GRAM_SMEM = GSTAGES * STAGE_BYTES + 1024 + 256;  // + alignment + barriers
constexpr int GRAM_THREADS = 192;
constexpr int64_t KCHUNK = 65536;  // rows per CTA: |class sum| <= 20480 * 65536 < 2^31
static_assert(STAGE_BYTES % 1024 == 0, "stage alignment");

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}\n" ::"r"(bar),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];\n" ::"r"(dst),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
      : "memory");
}
// K-major SWIZZLE_64B smem descriptor: 64-B rows, 8-row atoms (SBO 512 B), version 1.
__device__ __forceinline__ uint64_t desc_sw64(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(512 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)4 << 61;
  return d;
}
// kind::i8 instruction descriptor: D s32, A/B u8 (digit 0) or s8, K-major, M = 128, N = GN.
__host__ __device__ constexpr uint32_t idesc_i8(int a_signed, int b_signed) {
  return (2u << 4) | ((uint32_t)a_signed << 7) | ((uint32_t)b_signed << 10) | ((uint32_t)(GN >> 3) << 17) |
         ((uint32_t)(GM >> 4) << 24);
}
__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(bar)
               : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}

// Three exact balanced base-128 digits of x: N = rint(x 2^21) (one rounding
// conversion), then integer digit extraction N = m0 2^14 + m1 2^7 + m2 with
// m1, m2 in [-64, 63] and m0 in [0, 128] for x in [0, 1]. x_q = N 2^-21, so
// |x - x_q| <= 2^-22; every digit step is exact integer arithmetic (only one
// quarter-rate conversion per entry).
__device__ __forceinline__ void digits3(float x, int& m0, int& m1, int& m2) {
  x = fminf(fmaxf(x, 0.f), 1.9921875f);  // RBF entries lie in [0, 1]; guard rounding
  const int N = __float2int_rn(x * 2097152.f);
  m2 = ((N + 64) & 127) - 64;
  const int N1 = (N - m2) >> 7;
  m1 = ((N1 + 64) & 127) - 64;
  m0 = (N1 - m1) >> 7;
}
__device__ __forceinline__ double dequant3(int m0, int m1, int m2) {
  return (double)m0 * 0.0078125 + (double)m1 * 6.103515625e-05 + (double)m2 * 4.76837158203125e-07;
}

constexpr int TM = 64, TN = 64, TK = 16;

// K(i, j) = exp((x_i . y_j - 0.5 (sqx_i + sqy_j)) * inv) for a 64 x 64 tile,
// the dot as a sequential fp32 FMA chain (rbf_tile_kernel's arithmetic), then
// either three int8 digit planes (planes != nullptr: plane d at
// planes + d * plane_stride, element (i, j) at j * pitch + i) or the exact
// dequantized fp64 value (W: w[i + j * ldw]). diag_of[j] == i forces exp(0) = 1.
__global__ void __launch_bounds__(256) rbf_digits_kernel(int64_t n1, int64_t n2, int64_t d, const float* __restrict__ X,
                                                         int64_t x_rs, int64_t x_cs, const float* __restrict__ Y,
                                                         int64_t y_rs, int64_t y_cs, const float* __restrict__ sqx,
                                                         const float* __restrict__ sqy, float inv,
                                                         const int64_t* __restrict__ diag_of,
                                                         int8_t* __restrict__ planes, int64_t pitch,
                                                         int64_t plane_stride, double* __restrict__ w, int64_t ldw) {
  __shared__ float xs[TK][TM + 1];
  __shared__ float ys[TK][TN + 1];
  __shared__ __align__(16) int8_t stage[GND][TN][TM];  // [digit][column j][row i]
  const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
  const int64_t i0 = (int64_t)blockIdx.y * TM, j0 = (int64_t)blockIdx.x * TN;
  float acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.f;
  for (int64_t k0 = 0; k0 < d; k0 += TK) {
    for (int e = tid; e < TK * TM; e += 256) {
      const int r = e / TK, k = e % TK;
      const int64_t gi = i0 + r, gk = k0 + k, gj = j0 + r;
      xs[k][r] = (gi < n1 && gk < d) ? X[gi * x_rs + gk * x_cs] : 0.f;
      ys[k][r] = (gj < n2 && gk < d) ? Y[gj * y_rs + gk * y_cs] : 0.f;
    }
    __syncthreads();
    const int kmax = (d - k0) < TK ? (int)(d - k0) : TK;
    for (int k = 0; k < kmax; ++k) {
      float xv[4], yv[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) xv[a] = xs[k][ty + 16 * a];
#pragma unroll
      for (int b = 0; b < 4; ++b) yv[b] = ys[k][tx + 16 * b];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = fmaf(xv[a], yv[b], acc[a][b]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int li = ty + 16 * a, lj = tx + 16 * b;
      const int64_t i = i0 + li, j = j0 + lj;
      int m0 = 0, m1 = 0, m2 = 0;
      if (i < n1 && j < n2) {
        const float v = (diag_of && diag_of[j] == i) ? 1.f : expf((acc[a][b] - 0.5f * (sqx[i] + sqy[j])) * inv);
        digits3(v, m0, m1, m2);
        if (w) w[i + j * ldw] = dequant3(m0, m1, m2);
      }
      stage[0][lj][li] = (int8_t)(uint8_t)m0;
      stage[1][lj][li] = (int8_t)m1;
      stage[2][lj][li] = (int8_t)m2;
    }
  if (!planes) return;
  __syncthreads();
  // coalesced stores: 16 B of one column's rows per thread
  for (int e = tid; e < GND * TN * (TM / 16); e += 256) {
    const int dgt = e / (TN * (TM / 16)), rem = e % (TN * (TM / 16)), lj = rem / (TM / 16), q = rem % (TM / 16);
    const int64_t j = j0 + lj, i = i0 + 16 * q;
    if (j >= n2 || i >= n1) continue;
    int8_t* dst = planes + dgt * plane_stride + j * pitch + i;
    if (i + 16 <= n1) {
      *reinterpret_cast<int4*>(dst) = *reinterpret_cast<const int4*>(&stage[dgt][lj][16 * q]);
    } else {
      for (int t = 0; i + t < n1; ++t) dst[t] = stage[dgt][lj][16 * q + t];
    }
  }
}

// Persistent: CTA b processes work items b, b + gridDim.x, ... (item = tile +
// ntiles * chunk: one 128 x 96 tile (ib, jb) of G over rows [k0, k0 + kc) of
// C). The shared-memory ring runs across items; the epilogue of item i hands
// the TMEM accumulators back (acc_empty) before the MMAs of item i + 1 start.
__global__ void __launch_bounds__(GRAM_THREADS, 1)
    gram_i8_kernel(const __grid_constant__ CUtensorMap amap, const __grid_constant__ CUtensorMap bmap,
                   const int2* __restrict__ tiles, int ntiles, int nitems, int64_t n, int64_t kc,
                   double* __restrict__ ws) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + GSTAGES * STAGE_BYTES);  // full[S], empty[S], acc_full, acc_empty
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * GSTAGES + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  auto item_nkb = [&](int w, int2& tile, int64_t& k0) {
    tile = tiles[w % ntiles];
    k0 = (int64_t)(w / ntiles) * kc;
    const int64_t klen = n - k0 < kc ? n - k0 : kc;
    return klen > 0 ? (int)((klen + GBK - 1) / GBK) : 0;
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < GSTAGES; ++s) {
      mbar_init(su32(&bars[s]), 1);
      mbar_init(su32(&bars[GSTAGES + s]), 1);
    }
    mbar_init(su32(&bars[2 * GSTAGES]), 1);
    mbar_init(su32(&bars[2 * GSTAGES + 1]), 128);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer ----------------
      int g = 0;
      for (int w = blockIdx.x; w < nitems; w += gridDim.x) {
        int2 tile;
        int64_t k0;
        const int nkb = item_nkb(w, tile, k0);
        for (int kb = 0; kb < nkb; ++kb, ++g) {
          const int st = g % GSTAGES;
          if (g >= GSTAGES) mbar_wait(su32(&bars[GSTAGES + st]), (uint32_t)(((g / GSTAGES) - 1) & 1));
          const uint32_t full = su32(&bars[st]);
          mbar_expect_tx(full, STAGE_BYTES);
          const uint32_t base = su32(smem + st * STAGE_BYTES);
          const int kx = (int)(k0 + (int64_t)kb * GBK);
#pragma unroll
          for (int dg = 0; dg < GND; ++dg) {
            tma_load_3d(base + dg * A_TILE, &amap, kx, tile.x * GM, dg, full);
            tma_load_3d(base + GND * A_TILE + dg * B_TILE, &bmap, kx, tile.y * GN, dg, full);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer ----------------
      int g = 0, it = 0;
      for (int w = blockIdx.x; w < nitems; w += gridDim.x, ++it) {
        int2 tile;
        int64_t k0;
        const int nkb = item_nkb(w, tile, k0);
        if (it > 0) mbar_wait(su32(&bars[2 * GSTAGES + 1]), (uint32_t)((it - 1) & 1));  // accumulators drained
        asm volatile("tcgen05.fence::after_thread_sync;\n");
        for (int kb = 0; kb < nkb; ++kb, ++g) {
          const int st = g % GSTAGES;
          mbar_wait(su32(&bars[st]), (uint32_t)((g / GSTAGES) & 1));
          asm volatile("tcgen05.fence::after_thread_sync;\n");
          const uint32_t a0 = su32(smem + st * STAGE_BYTES), b0 = a0 + GND * A_TILE;
#pragma unroll
          for (int kk = 0; kk < GBK / 32; ++kk) {
#pragma unroll
            for (int s = 0; s < GND; ++s)
#pragma unroll
              for (int t = 0; t < GND; ++t) {
                const int cls = s + t;
                // first write of accumulator `cls`: the first (s, t) of the class at k = 0
                const bool first = kb == 0 && kk == 0 && (s == 0 || t == GND - 1);
                mma_i8(tmem + (uint32_t)(cls * GN), desc_sw64(a0 + s * A_TILE + kk * 32),
                       desc_sw64(b0 + t * B_TILE + kk * 32), idesc_i8(s > 0, t > 0), first ? 0u : 1u);
              }
          }
          mma_commit(su32(&bars[GSTAGES + st]));  // stage free once these MMAs complete
        }
        mma_commit(su32(&bars[2 * GSTAGES]));  // this item's accumulators final
      }
    }
  } else {  // ---------------- epilogue: warps 2-5 ----------------
    const int q = warp & 3;  // TMEM lane quarter of this warp
    const int row = 32 * q + lane;
    const uint32_t tl = tmem + ((uint32_t)(32 * q) << 16);
    int it = 0;
    for (int w = blockIdx.x; w < nitems; w += gridDim.x, ++it) {
      int2 tile;
      int64_t k0;
      const int nkb = item_nkb(w, tile, k0);
      mbar_wait(su32(&bars[2 * GSTAGES]), (uint32_t)(it & 1));
      asm volatile("tcgen05.fence::after_thread_sync;\n");
      double* out = ws + (int64_t)w * (int64_t)(GN * GM);
#pragma unroll 1
      for (int c0 = 0; c0 < GN; c0 += 16) {
        uint32_t v[GCLS][16];
#pragma unroll
        for (int k = 0; k < GCLS; ++k) tmem_ld16(tl + (uint32_t)(k * GN + c0), v[k]);
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          // G = sum_k A_k 2^-(7k + 14), smallest terms first
          double g = (double)(int)v[GCLS - 1][j];
#pragma unroll
          for (int k = GCLS - 2; k >= 0; --k) g = g * 0.0078125 + (double)(int)v[k][j];
          out[(int64_t)(c0 + j) * GM + row] = nkb > 0 ? g * 6.103515625e-05 : 0.0;
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;\n");
      mbar_arrive(su32(&bars[2 * GSTAGES + 1]));
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 2) {
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512));
  }
}

// G[p, q] = G[q, p] = sum over K chunks (fixed order) of the tile partial holding (min, max).
__global__ void gram_reduce_kernel(int64_t s, int njb, const int* __restrict__ tile_of, int ntiles, int nchunks,
                                   const double* __restrict__ ws, double* __restrict__ G, int accumulate) {
  const int64_t total = s * s;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = e % s, q = e / s;
    if (p > q) continue;
    const int64_t ib = p / GM, jb = q / GN;
    const int t = tile_of[ib * njb + jb];
    double acc = 0.0;
    for (int c = 0; c < nchunks; ++c)
      acc += ws[(((int64_t)c * ntiles + t) * GN + (q - jb * GN)) * GM + (p - ib * GM)];
    if (accumulate) acc += G[p + q * s];
    G[p + q * s] = acc;
    G[q + p * s] = acc;
  }
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeFn encode() {
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

void plane_map(CUtensorMap* m, const int8_t* planes, int64_t n, int64_t s, int64_t pitch, uint32_t box_rows) {
  const cuuint64_t dims[3] = {(cuuint64_t)n, (cuuint64_t)s, (cuuint64_t)GND};
  const cuuint64_t strides[2] = {(cuuint64_t)pitch, (cuuint64_t)(pitch * s)};
  const cuuint32_t box[3] = {(cuuint32_t)GBK, box_rows, 1};
  const cuuint32_t es[3] = {1, 1, 1};
  const CUresult r = encode()(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t*>(planes), dims, strides, box,
                              es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled (int8 digit planes) failed: " + std::to_string((int)r));
}


// ---------------------------------------------------------------------------
// Kernel columns on the tensor cores: D = X X_S' (K = d <= 64) with the 3xTF32
// split (x = hi + lo, both tf32; D = Xh Sh' + Xh Sl' + Xl Sh' accumulated in
// fp32 TMEM, ~2^-22 relative per product, the accuracy of an fp32 dot), then
// the RBF epilogue exp((D - 0.5 (|x_i|^2 + |s_j|^2)) / sigma^2) straight into
// the int8 digit planes. C is never stored in fp32.
//
// Persistent CTA = one 128-landmark column block (B hi/lo resident in shared
// memory) x a strided list of 128-row tiles; A hi/lo double-buffered by TMA
// (SWIZZLE_128B, two 32-column halves per operand); two TMEM accumulators so
// the epilogue of tile t overlaps the MMAs of tile t + 1. Warp 0 = TMA, warp 1
// = MMA, warps 2-9 = epilogue (two warps per TMEM lane quarter, 64 columns each).
constexpr int RT_M = 128, RT_N = 128, RT_K = 64;
constexpr int RT_HALF = RT_M * 128;                  // one 128-row x 32-fp32 SW128 box (16 KB)
constexpr int RT_A_BYTES = 4 * RT_HALF;              // hi/lo x two k halves (64 KB)
constexpr int RT_B_BYTES = 4 * RT_HALF;              // 128 landmarks (64 KB)
constexpr int RT_EPI_WARPS = 16;
constexpr int RT_SMEM = RT_B_BYTES + 2 * RT_A_BYTES + 1024 + 2048;
constexpr int RT_THREADS = 32 * (2 + RT_EPI_WARPS);

__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          dst),
      "l"(map), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
// kind::tf32: D f32, A/B tf32, K-major, M = 128, N = RT_N.
constexpr uint32_t IDESC_TF32 = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(RT_N >> 3) << 17) |
                                ((uint32_t)(RT_M >> 4) << 24);

__global__ void tf32_split_kernel(int64_t n, int64_t d, const float* __restrict__ x, int64_t rs, int64_t cs,
                                  float* __restrict__ hi, float* __restrict__ lo) {
  const int64_t total = n * d;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / d, k = e % d;
    const float v = x[i * rs + k * cs];
    uint32_t h, l;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(v));
    const float r = v - __uint_as_float(h);
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(l) : "f"(r));
    hi[e] = __uint_as_float(h);
    lo[e] = __uint_as_float(l);
  }
}

__global__ void __launch_bounds__(RT_THREADS, 1)
    rbf_tc_digits_kernel(const __grid_constant__ CUtensorMap xh, const __grid_constant__ CUtensorMap xl,
                         const __grid_constant__ CUtensorMap sh, const __grid_constant__ CUtensorMap sl, int64_t n,
                         int64_t s, const float* __restrict__ sqx, const float* __restrict__ sqy, float inv,
                         const int64_t* __restrict__ diag_of, int8_t* __restrict__ planes, int64_t pitch,
                         int64_t plane_stride, int ncb, int nrg) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* bsm = smem;
  uint8_t* asm_ = smem + RT_B_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + RT_B_BYTES + 2 * RT_A_BYTES);
  // bars: [0,1] a_full, [2,3] a_empty, [4,5] t_full, [6,7] t_empty, [8] b_full
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 9);
  float* sq_s = reinterpret_cast<float*>(bars + 16);          // [RT_N], 16-B aligned
  int* dg_s = reinterpret_cast<int*>(sq_s + RT_N);             // [RT_N]: landmark's local row, -1 if none
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cb = blockIdx.x % ncb, rg = blockIdx.x / ncb;
  const int64_t j0 = (int64_t)cb * RT_N;
  const int ntile = (int)((n + RT_M - 1) / RT_M);
  const int my_tiles = rg < ntile ? (ntile - 1 - rg) / nrg + 1 : 0;

  if (threadIdx.x == 0) {
    for (int b = 0; b < 2; ++b) {
      mbar_init(su32(&bars[0 + b]), 1);
      mbar_init(su32(&bars[2 + b]), 1);
      mbar_init(su32(&bars[4 + b]), 1);
      mbar_init(su32(&bars[6 + b]), 32 * RT_EPI_WARPS);
    }
    mbar_init(su32(&bars[8]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  for (int c = threadIdx.x; c < RT_N; c += RT_THREADS) {
    const int64_t j = j0 + c;
    sq_s[c] = j < s ? sqy[j] : 0.f;
    const int64_t dr = j < s && diag_of ? diag_of[j] : -1;
    dg_s[c] = dr >= 0 && dr < n ? (int)dr : -1;
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(tmem_slot)),
                 "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer ----------------
      const uint32_t bb = su32(&bars[8]);
      mbar_expect_tx(bb, RT_B_BYTES);
      const uint32_t b0 = su32(bsm);
      tma_load_2d(b0 + 0 * RT_HALF, &sh, 0, (int)j0, bb);
      tma_load_2d(b0 + 1 * RT_HALF, &sh, 32, (int)j0, bb);
      tma_load_2d(b0 + 2 * RT_HALF, &sl, 0, (int)j0, bb);
      tma_load_2d(b0 + 3 * RT_HALF, &sl, 32, (int)j0, bb);
      for (int t = 0; t < my_tiles; ++t) {
        const int buf = t & 1;
        if (t >= 2) mbar_wait(su32(&bars[2 + buf]), (uint32_t)(((t >> 1) - 1) & 1));
        const uint32_t full = su32(&bars[buf]);
        mbar_expect_tx(full, RT_A_BYTES);
        const uint32_t a0 = su32(asm_ + buf * RT_A_BYTES);
        const int i0 = (rg + t * nrg) * RT_M;
        tma_load_2d(a0 + 0 * RT_HALF, &xh, 0, i0, full);
        tma_load_2d(a0 + 1 * RT_HALF, &xh, 32, i0, full);
        tma_load_2d(a0 + 2 * RT_HALF, &xl, 0, i0, full);
        tma_load_2d(a0 + 3 * RT_HALF, &xl, 32, i0, full);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer ----------------
      mbar_wait(su32(&bars[8]), 0u);
      const uint32_t b0 = su32(bsm);
      for (int t = 0; t < my_tiles; ++t) {
        const int buf = t & 1;
        mbar_wait(su32(&bars[buf]), (uint32_t)((t >> 1) & 1));
        if (t >= 2) mbar_wait(su32(&bars[6 + buf]), (uint32_t)(((t >> 1) - 1) & 1));  // accumulator drained
        asm volatile("tcgen05.fence::after_thread_sync;\n");
        const uint32_t a0 = su32(asm_ + buf * RT_A_BYTES), d = tmem + (uint32_t)(buf * RT_N);
#pragma unroll
        for (int kk = 0; kk < RT_K / 8; ++kk) {
          const uint32_t off = (uint32_t)((kk >> 2) * RT_HALF + (kk & 3) * 32);
          const uint64_t ah = desc_sw128(a0 + off), al = desc_sw128(a0 + 2 * RT_HALF + off);
          const uint64_t bh = desc_sw128(b0 + off), bl = desc_sw128(b0 + 2 * RT_HALF + off);
          mma_tf32(d, ah, bh, IDESC_TF32, kk > 0 ? 1u : 0u);
          mma_tf32(d, ah, bl, IDESC_TF32, 1u);
          mma_tf32(d, al, bh, IDESC_TF32, 1u);
        }
        mma_commit(su32(&bars[2 + buf]));  // A buffer free
        mma_commit(su32(&bars[4 + buf]));  // accumulator ready
      }
    }
  } else {  // ---------------- epilogue: warps 2-17 ----------------
    // warp w: TMEM lane quarter w & 3 (rows 32q .. 32q + 31), columns
    // 32 * part .. + 31. Each lane computes its row's digits for 16 columns,
    // packs them 4 columns per word, and a 4-lane byte transpose (shuffles)
    // turns them into words of 4 consecutive ROWS of one column, stored
    // straight to the column-major digit planes (one full 32-B sector per
    // column per 8 lanes).
    const int q = warp & 3, part = (warp - 2) >> 2;
    const int row = 32 * q + lane, sub = lane & 3, g4 = lane >> 2;
    const uint32_t sel = (uint32_t)sub | ((uint32_t)(4 + sub) << 4);  // byte `sub` of x, byte `sub` of y
    for (int t = 0; t < my_tiles; ++t) {
      const int buf = t & 1;
      const int64_t ibase = (int64_t)(rg + t * nrg) * RT_M + 32 * q;
      const int64_t i = ibase + lane;
      mbar_wait(su32(&bars[4 + buf]), (uint32_t)((t >> 1) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;\n");
      const float sxi = i < n ? sqx[i] : 0.f;
      const int il = (int)(i < n ? i : -2);
      const uint32_t tl = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(buf * RT_N + part * 32);
      uint32_t v[2][16];
      tmem_ld16(tl, v[0]);
      tmem_ld16(tl + 16u, v[1]);
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;\n");
      mbar_arrive(su32(&bars[6 + buf]));  // accumulator drained by this thread
      if (ibase >= n) continue;           // warp-uniform
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int cb = part * 32 + h * 16;
        float sq[16];
        int dg[16];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float4 a4 = *reinterpret_cast<const float4*>(sq_s + cb + 4 * u);
          const int4 d4 = *reinterpret_cast<const int4*>(dg_s + cb + 4 * u);
          sq[4 * u] = a4.x; sq[4 * u + 1] = a4.y; sq[4 * u + 2] = a4.z; sq[4 * u + 3] = a4.w;
          dg[4 * u] = d4.x; dg[4 * u + 1] = d4.y; dg[4 * u + 2] = d4.z; dg[4 * u + 3] = d4.w;
        }
        uint32_t w[3][4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          w[0][u] = w[1][u] = w[2][u] = 0u;
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            const int jj = 4 * u + b;
            const float x =
                dg[jj] == il ? 1.f : exp2f((__uint_as_float(v[h][jj]) - 0.5f * (sxi + sq[jj])) * inv);
            int m0, m1, m2;
            digits3(x, m0, m1, m2);
            w[0][u] |= (uint32_t)(m0 & 0xff) << (8 * b);
            w[1][u] |= (uint32_t)(m1 & 0xff) << (8 * b);
            w[2][u] |= (uint32_t)(m2 & 0xff) << (8 * b);
          }
        }
#pragma unroll
        for (int dgt = 0; dgt < 3; ++dgt)
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            // lane (g4, sub) gathers byte `sub` (column 4u + sub) of rows 4 g4 .. 4 g4 + 3
            const uint32_t x0 = __shfl_sync(0xffffffffu, w[dgt][u], (lane & ~3) | 0);
            const uint32_t x1 = __shfl_sync(0xffffffffu, w[dgt][u], (lane & ~3) | 1);
            const uint32_t x2 = __shfl_sync(0xffffffffu, w[dgt][u], (lane & ~3) | 2);
            const uint32_t x3 = __shfl_sync(0xffffffffu, w[dgt][u], (lane & ~3) | 3);
            const uint32_t T = __byte_perm(__byte_perm(x0, x1, sel), __byte_perm(x2, x3, sel), 0x5410);
            const int64_t j = j0 + cb + 4 * u + sub;
            const int64_t r0 = ibase + 4 * g4;
            if (j < s && r0 < n) {
              int8_t* dst = planes + dgt * plane_stride + j * pitch + r0;
              if (r0 + 4 <= n) {
                *reinterpret_cast<uint32_t*>(dst) = T;
              } else {
                for (int b = 0; r0 + b < n; ++b) dst[b] = (int8_t)((T >> (8 * b)) & 0xff);
              }
            }
          }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 2) {
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(256));
  }
}

// W[a, b] = dequantized digits of C at (row dsel[a], column b) for the
// landmarks this rank owns (dsel[a] >= 0), zero otherwise.
__global__ void w_from_digits_kernel(int64_t s, const int64_t* __restrict__ dsel, const int8_t* __restrict__ planes,
                                     int64_t pitch, int64_t plane_stride, double* __restrict__ W) {
  const int64_t total = s * s;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = e % s, b = e / s;
    const int64_t r = dsel[a];
    double v = 0.0;
    if (r >= 0) {
      const int8_t* p = planes + b * pitch + r;
      v = dequant3((int)(uint8_t)p[0], (int)p[plane_stride], (int)p[2 * plane_stride]);
    }
    W[a + b * s] = v;
  }
}
}  // namespace

bool gram_i8_available() {
  static const bool off = std::getenv("RNLA_NYSTROM_DMMA_GRAM") != nullptr;
  return !off && encode() != nullptr && tc_gemm_enabled();
}

int64_t digit_pitch(int64_t n) { return (n + 63) / 64 * 64; }

void rbf_digits(rnla_ctx* ctx, int64_t n1, int64_t n2, int64_t d, const float* X, int64_t x_rs, int64_t x_cs,
                const float* Y, int64_t y_rs, int64_t y_cs, const float* sqx, const float* sqy, double sigma,
                const int64_t* diag_of, int8_t* planes, int64_t pitch, int64_t plane_stride, double* w, int64_t ldw) {
  if (n1 == 0 || n2 == 0) return;
  const float inv = (float)(1.0 / (sigma * sigma));
  dim3 grid((unsigned)((n2 + TN - 1) / TN), (unsigned)((n1 + TM - 1) / TM));
  rbf_digits_kernel<<<grid, 256, 0, ctx->stream>>>(n1, n2, d, X, x_rs, x_cs, Y, y_rs, y_cs, sqx, sqy, inv, diag_of,
                                                   planes, pitch, plane_stride, w, ldw);
  RNLA_CUDA(cudaGetLastError());
  note_launch(ctx);
}

void gram_i8(rnla_ctx* ctx, const int8_t* planes, int64_t n, int64_t s, int64_t pitch, double* G, bool accumulate,
             int reserve_sms) {
  if (s == 0) return;
  const int nib = (int)((s + GM - 1) / GM), njb = (int)((s + GN - 1) / GN);
  std::vector<int2> tl;
  std::vector<int> tile_of((size_t)nib * njb, -1);
  for (int ib = 0; ib < nib; ++ib)
    for (int jb = 0; jb < njb; ++jb)
      if ((int64_t)jb * GN + GN - 1 >= (int64_t)ib * GM) {  // touches the upper triangle
        tile_of[(size_t)ib * njb + jb] = (int)tl.size();
        tl.push_back(make_int2(ib, jb));
      }
  const int ntiles = (int)tl.size();
  const int ctas_max = std::max(1, ctx->num_sms - std::max(0, reserve_sms));
  // K chunks: at most KCHUNK rows each (s32 range); enough work items to
  // balance the persistent CTAs (chunk is the slow index, so the CTAs running
  // together share one chunk of the digit planes in L2)
  const int cmin = (int)std::max<int64_t>(1, (n + KCHUNK - 1) / KCHUNK);
  int nchunks = cmin;
  double best = 1e300;
  for (int c = cmin; c <= std::max(cmin, 64); ++c) {
    const double rounds = std::ceil((double)ntiles * c / ctas_max);
    const double cost = rounds / c + 0.002 * c;  // per-item epilogue + reduce overhead
    if (cost < best - 1e-12) {
      best = cost;
      nchunks = c;
    }
  }
  const int64_t kc = std::max<int64_t>(GBK, ((n + nchunks - 1) / nchunks + GBK - 1) / GBK * GBK);
  nchunks = (int)std::max<int64_t>(1, (n + kc - 1) / kc);
  const int nitems = ntiles * nchunks;
  DevBuf dtl(sizeof(int2) * tl.size(), ctx->stream), dto(sizeof(int) * tile_of.size(), ctx->stream);
  DevBuf ws(sizeof(double) * (size_t)nitems * GM * GN, ctx->stream);
  RNLA_CUDA(cudaMemcpyAsync(dtl.p, tl.data(), sizeof(int2) * tl.size(), cudaMemcpyHostToDevice, ctx->stream));
  RNLA_CUDA(cudaMemcpyAsync(dto.p, tile_of.data(), sizeof(int) * tile_of.size(), cudaMemcpyHostToDevice, ctx->stream));
  if (n > 0) {
    CUtensorMap amap, bmap;
    plane_map(&amap, planes, n, s, pitch, GM);
    plane_map(&bmap, planes, n, s, pitch, GN);
    ensure_dyn_smem((const void*)gram_i8_kernel, GRAM_SMEM);
    gram_i8_kernel<<<std::min(nitems, ctas_max), GRAM_THREADS, GRAM_SMEM, ctx->stream>>>(
        amap, bmap, dtl.as<int2>(), ntiles, nitems, n, kc, ws.as<double>());
    RNLA_CUDA(cudaGetLastError());
    note_launch(ctx);
  } else {
    RNLA_CUDA(cudaMemsetAsync(ws.p, 0, ws.bytes, ctx->stream));
  }
  gram_reduce_kernel<<<grid_for(ctx, s * s, 256), 256, 0, ctx->stream>>>(s, njb, dto.as<int>(), ntiles, nchunks,
                                                                          ws.as<double>(), G, accumulate ? 1 : 0);
  RNLA_CUDA(cudaGetLastError());
  note_launch(ctx);
  RNLA_CUDA(cudaStreamSynchronize(ctx->stream));  // tl / tile_of leave scope
}

bool rbf_tc_available(int64_t d) { return d >= 1 && d <= RT_K && encode() != nullptr && tc_gemm_enabled(); }

void rbf_tc_digits(rnla_ctx* ctx, int64_t n, int64_t s, int64_t d, const float* X, int64_t x_rs, int64_t x_cs,
                   const float* Xs, int64_t s_rs, int64_t s_cs, const float* sqx, const float* sqy, double sigma,
                   const int64_t* diag_of, int8_t* planes, int64_t pitch, int64_t plane_stride, int reserve_sms) {
  if (n == 0 || s == 0) return;
  require(d >= 1 && d <= RT_K, "rbf_tc_digits: d > 64");
  // tf32 hi/lo images, row-major n x d (16-B aligned rows: d padded to 4)
  const int64_t ld = (d + 3) / 4 * 4;
  DevBuf xh(sizeof(float) * n * ld, ctx->stream), xl(sizeof(float) * n * ld, ctx->stream),
      shb(sizeof(float) * s * ld, ctx->stream), slb(sizeof(float) * s * ld, ctx->stream);
  auto split = [&](int64_t rows, const float* src, int64_t rs, int64_t cs, float* hi, float* lo) {
    if (ld != d) {
      RNLA_CUDA(cudaMemsetAsync(hi, 0, sizeof(float) * rows * ld, ctx->stream));
      RNLA_CUDA(cudaMemsetAsync(lo, 0, sizeof(float) * rows * ld, ctx->stream));
    }
    // split into a dense n x d image, then widen the pitch if needed
    tf32_split_kernel<<<grid_for(ctx, rows * d, 256), 256, 0, ctx->stream>>>(rows, d, src, rs, cs, hi, lo);
    RNLA_CUDA(cudaGetLastError());
    note_launch(ctx);
    if (ld != d) {
      RNLA_CUDA(cudaMemcpy2DAsync(hi, sizeof(float) * ld, hi, sizeof(float) * d, sizeof(float) * d, rows,
                                  cudaMemcpyDeviceToDevice, ctx->stream));
      RNLA_CUDA(cudaMemcpy2DAsync(lo, sizeof(float) * ld, lo, sizeof(float) * d, sizeof(float) * d, rows,
                                  cudaMemcpyDeviceToDevice, ctx->stream));
    }
  };
  split(n, X, x_rs, x_cs, xh.as<float>(), xl.as<float>());
  split(s, Xs, s_rs, s_cs, shb.as<float>(), slb.as<float>());
  auto map = [&](CUtensorMap* m, const float* base, int64_t rows) {
    const cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
    const cuuint32_t box[2] = {32, (cuuint32_t)RT_M};
    const cuuint32_t es[2] = {1, 1};
    const CUresult r = encode()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box,
                                es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled (tf32 images) failed: " + std::to_string((int)r));
  };
  CUtensorMap mxh, mxl, msh, msl;
  map(&mxh, xh.as<float>(), n);
  map(&mxl, xl.as<float>(), n);
  map(&msh, shb.as<float>(), s);
  map(&msl, slb.as<float>(), s);
  const int ncb = (int)((s + RT_N - 1) / RT_N);
  const int ntile = (int)((n + RT_M - 1) / RT_M);
  const int nrg = std::max(1, std::min(ntile, std::max(1, ctx->num_sms - std::max(0, reserve_sms)) / ncb));
  ensure_dyn_smem((const void*)rbf_tc_digits_kernel, RT_SMEM);
  rbf_tc_digits_kernel<<<ncb * nrg, RT_THREADS, RT_SMEM, ctx->stream>>>(
      mxh, mxl, msh, msl, n, s, sqx, sqy, (float)(1.4426950408889634 / (sigma * sigma)), diag_of, planes, pitch,
      plane_stride, ncb, nrg);
  RNLA_CUDA(cudaGetLastError());
  note_launch(ctx);
  RNLA_CUDA(cudaStreamSynchronize(ctx->stream));  // the tf32 images leave scope
}

void w_from_digits(rnla_ctx* ctx, int64_t s, const int64_t* dsel, const int8_t* planes, int64_t pitch,
                   int64_t plane_stride, double* W) {
  if (s == 0) return;
  w_from_digits_kernel<<<grid_for(ctx, s * s, 256), 256, 0, ctx->stream>>>(s, dsel, planes, pitch, plane_stride, W);
  RNLA_CUDA(cudaGetLastError());
  note_launch(ctx);
}

}  // namespace rnla
