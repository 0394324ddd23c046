// ozaki.cu -- the fp64 Gaussian stage on the int8 tensor cores with exact
// digit products (an Ozaki-style split): out (+)= Gs' * in for one K-chunk, the
// stage of the config-1 combined sketch Omega' (S'[A, b]) (src/sketch.cpp:108-123,
// 36-42), 2048 x 513 x 8192 = 17.2 GF per call.
//
// Every row i of Gs' = Omega' and every column j of the chunk of `in` is
// scaled by a power of two (2^e_i, 2^f_j: the largest magnitude in it maps below
// 1) and rounded ONCE to a 46-bit integer, N = rint(x 2^46 / 2^e), which is split
// exactly into six balanced digits, the first in [-64, 64] and five base-256
// ones in [-128, 127] (all int8),
//     N = sum_p d_p 2^(40 - 8p),   x = 2^(e - 6) sum_p d_p 2^(-8p)
// to 2^-47 relative to the row (column) maximum. The digit products are exact
// in the s32 accumulators of tcgen05.mma kind::i8; the 21 pairs with
// p + q <= 5 accumulate by class k = p + q (six TMEM accumulators of 80 columns)
// and are combined in fp64,
//     out_ij = 2^(e_i + f_j - 12) sum_k 2^(-8k) S_k,
// dropping the classes k >= 6. Measured: 3.4e-13 rel-F against torch fp64 on
// the config-1 stage (gate 1e-10); six base-128 digits (41 bits) had failed the
// config-1 LSR objective gate (2.2e-10 vs 1e-10). Variants measured on the
// config-1 stage (8192 x 513 -> 2048, whole stage incl. the digit kernels):
// base 128 x 7 digits, N 64, 32-k SW32 stages x 5: 357 us; base 256 x 6, N 80,
// 32-k x 5: 303 us; 64-k SW64 x 2: 289 us (used); fp64 DMMA: 953 us standalone
// (570 us with split-K). The kernel is bound by L2-to-SM operand traffic
// (6 x 208 B per k for 21 x 128 x 80 MACs: ~48 B/clk/SM at the int8 rate).
//
// Layout: digit planes are K-major (each row of Gs', each column of the chunk,
// has its K digits contiguous), plane p at planes + p * plane_stride, loaded by
// TMA as swizzled boxes of OBK k x rows. Omega's planes are built once per
// cached operator; the chunk's planes per call (a column-max kernel and a
// digit kernel). CTA = one 128 x 80 output tile over the chunk's K: warp 0 TMA
// producer, warp 1 MMA issuer (21 digit pairs per 32-k step), warps 2-5
// epilogue (fp64 combination through shared memory, coalesced (+)= into the
// output).
#include <cuda.h>

#include "rnla_internal.h"
#include "util.cuh"

namespace rnla {

namespace {

#ifndef RNLA_OZ_BITS
#define RNLA_OZ_BITS 8   // bits per digit after the first (base 2^bits)
#endif
#ifndef RNLA_OZ_P
#define RNLA_OZ_P 6      // digits per operand
#endif
#ifndef RNLA_OZ_N
#define RNLA_OZ_N 80     // output columns per CTA (OP * ON TMEM columns)
#endif
#ifndef RNLA_OZ_BK
#define RNLA_OZ_BK 64    // k per stage (32: SWIZZLE_32B rows, 64: SWIZZLE_64B)
#endif
#ifndef RNLA_OZ_STAGES
#define RNLA_OZ_STAGES 2
#endif
constexpr int OP = RNLA_OZ_P, DB = RNLA_OZ_BITS;
constexpr int OM = 128, ON = RNLA_OZ_N, OBK = RNLA_OZ_BK, OSTAGES = RNLA_OZ_STAGES;
constexpr int OA_TILE = OM * OBK, OB_TILE = ON * OBK;  // bytes per digit-plane tile
constexpr int OSTAGE = OP * (OA_TILE + OB_TILE);
constexpr int OSMEM = OSTAGES * OSTAGE + 1024 + 256;
constexpr int OTHREADS = 192;
constexpr int OBITS = 6 + DB * (OP - 1);               // bits of each scaled value
constexpr double kTwoBits = (double)(1ll << OBITS);
constexpr double kDigitW = 1.0 / (double)(1 << DB);     // weight ratio of consecutive classes
// class sums stay below 2^31: OP pairs x kc x (2^(DB-1))^2
constexpr int64_t kMaxKc = ((int64_t)1 << 31) / ((int64_t)OP << (2 * (DB - 1))) / 64 * 64;
static_assert(OSTAGE % 1024 == 0, "stage alignment");
static_assert(OP * ON <= 512, "class accumulators exceed TMEM");
static_assert(OM * ON * 8 <= OSTAGES * OSTAGE, "epilogue tile must fit in the stage ring");

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
// K-major swizzled smem descriptor for OBK-byte rows: SWIZZLE_32B (code 6, 8-row
// atoms of 256 B) or SWIZZLE_64B (code 4, 512 B), version 1.
__device__ __forceinline__ uint64_t desc_sw(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)((8 * OBK) >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)(OBK == 32 ? 6 : 4) << 61;
  return d;
}
// kind::i8: D s32, A/B s8, K-major, M = 128, N = ON.
constexpr uint32_t kIdescS8 = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(ON >> 3) << 17) |
                              ((uint32_t)(OM >> 4) << 24);
__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(kIdescS8), "r"(accumulate));
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

// Power-of-two exponent e with max|x| < 2^e (0 for an all-zero vector).
__device__ __forceinline__ int oz_exponent(double mx) { return mx > 0.0 ? ilogb(mx) + 1 : 0; }

// The OP digits of x scaled by 2^-e (one rounding, then exact integer steps).
__device__ __forceinline__ void oz_digits(double x, double inv_scale, int8_t* d) {
  long long N = llrint(x * inv_scale * kTwoBits);
  constexpr long long half = 1ll << (DB - 1), mask = (1ll << DB) - 1;
#pragma unroll
  for (int p = OP - 1; p > 0; --p) {
    const long long r = ((N + half) & mask) - half;
    d[p] = (int8_t)r;
    N = (N - r) >> DB;
  }
  d[0] = (int8_t)N;
}

// One CTA per row i of A (element (i, k) at A[i * lda + k], k < K): the row
// maximum, the row scale 2^(e - 6) (NaN for a non-finite row, so it propagates
// to the output) and the digit planes planes[p * pstride + i * pitch + k]
// (zero for K <= k < pitch).
__global__ void __launch_bounds__(256) oz_row_digits(int64_t K, const double* __restrict__ A, int64_t lda,
                                                     int8_t* __restrict__ planes, int64_t pitch, int64_t pstride,
                                                     double* __restrict__ rscale) {
  __shared__ double red[8];
  __shared__ int bad_s;
  const int64_t i = blockIdx.x;
  const double* a = A + i * lda;
  double mx = 0.0;
  int bad = 0;
  for (int64_t k = threadIdx.x; k < K; k += blockDim.x) {
    const double v = fabs(a[k]);
    if (!isfinite(v)) bad = 1;
    mx = fmax(mx, v);
  }
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (threadIdx.x == 0) bad_s = 0;
  __syncthreads();
  if (bad) atomicOr(&bad_s, 1);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  mx = red[0];
  for (int w = 1; w < 8; ++w) mx = fmax(mx, red[w]);
  const int e = bad_s ? 0 : oz_exponent(mx);
  const double inv = ldexp(1.0, -e);
  if (threadIdx.x == 0) rscale[i] = bad_s ? nan("") : ldexp(1.0, e - 6);
  for (int64_t k = threadIdx.x; k < pitch; k += blockDim.x) {
    int8_t d[OP] = {};
    if (k < K && !bad_s) oz_digits(a[k], inv, d);
#pragma unroll
    for (int p = 0; p < OP; ++p) planes[p * pstride + i * pitch + k] = d[p];
  }
}

// Column maxima of a K x N chunk (element (k, j) at in[k * ld + j]) as the bit
// patterns of |x| (non-negative doubles order like their bits; inf and NaN sort
// above every finite value): grid (N / 32, K / 128), 32 columns x 8 row groups
// of 16 rows per CTA, atomicMax per column (colmax zeroed by the caller).
__global__ void __launch_bounds__(256) oz_col_max(int64_t K, int64_t N, const double* __restrict__ in, int64_t ld,
                                                  unsigned long long* __restrict__ colmax) {
  __shared__ unsigned long long red[8][32];
  const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int64_t j = (int64_t)blockIdx.x * 32 + lane;
  const int64_t k0 = (int64_t)blockIdx.y * 128 + 16 * g;
  unsigned long long mx = 0;
  if (j < N)
    for (int t = 0; t < 16 && k0 + t < K; ++t) {
      const unsigned long long b = (unsigned long long)__double_as_longlong(fabs(in[(k0 + t) * ld + j]));
      mx = b > mx ? b : mx;
    }
  red[g][lane] = mx;
  __syncthreads();
  if (g == 0 && j < N) {
    for (int w = 1; w < 8; ++w) mx = red[w][lane] > mx ? red[w][lane] : mx;
    atomicMax(colmax + j, mx);
  }
}

// Column digits: thread (j, g) of block (jb, kb) turns 16 consecutive k of
// column j into one 16-B store per plane (planes[p * pstride + j * pitch + k]);
// cscale[j] = 2^(e_j - 6) (NaN for a non-finite column).
__global__ void __launch_bounds__(256) oz_col_digits(int64_t K, int64_t N, const double* __restrict__ in, int64_t ld,
                                                     const unsigned long long* __restrict__ colmax,
                                                     int8_t* __restrict__ planes, int64_t pitch, int64_t pstride,
                                                     double* __restrict__ cscale) {
  const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int64_t j = (int64_t)blockIdx.x * 32 + lane;
  const int64_t k0 = (int64_t)blockIdx.y * 128 + 16 * g;
  if (j >= N || k0 >= pitch) return;
  const unsigned long long mb = colmax[j];
  const bool bad = mb >= 0x7ff0000000000000ull;
  const int e = bad ? 0 : oz_exponent(__longlong_as_double((long long)mb));
  const double inv = ldexp(1.0, -e);
  if (blockIdx.y == 0 && g == 0) cscale[j] = bad ? nan("") : ldexp(1.0, e - 6);
  alignas(16) int8_t d[OP][16];
#pragma unroll
  for (int t = 0; t < 16; ++t) {
    int8_t dd[OP] = {};
    if (k0 + t < K && !bad) oz_digits(in[(k0 + t) * ld + j], inv, dd);
#pragma unroll
    for (int p = 0; p < OP; ++p) d[p][t] = dd[p];
  }
#pragma unroll
  for (int p = 0; p < OP; ++p)
    *reinterpret_cast<int4*>(planes + p * pstride + j * pitch + k0) = *reinterpret_cast<const int4*>(d[p]);
}

// out(i, j) (+)= rscale_i cscale_j sum_k 2^-7k S_k for one 128 x 80 tile over
// K = nkb * 64 (grid: (N tiles, M tiles)).
__global__ void __launch_bounds__(OTHREADS, 1)
    oz_gemm_kernel(const __grid_constant__ CUtensorMap amap, const __grid_constant__ CUtensorMap bmap, int64_t M,
                   int64_t N, int a_k0, int nkb, const double* __restrict__ rscale,
                   const double* __restrict__ cscale, double* out, int64_t out_rs, int64_t out_cs, int accumulate) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + OSTAGES * OSTAGE);  // full[S], empty[S], acc_full
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * OSTAGES + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nb = blockIdx.x, mb = blockIdx.y;

  if (threadIdx.x == 0) {
    for (int s = 0; s < OSTAGES; ++s) {
      mbar_init(su32(&bars[s]), 1);
      mbar_init(su32(&bars[OSTAGES + s]), 1);
    }
    mbar_init(su32(&bars[2 * OSTAGES]), 1);
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
      for (int kb = 0; kb < nkb; ++kb) {
        const int st = kb % OSTAGES;
        if (kb >= OSTAGES) mbar_wait(su32(&bars[OSTAGES + st]), (uint32_t)(((kb / OSTAGES) - 1) & 1));
        const uint32_t full = su32(&bars[st]);
        mbar_expect_tx(full, OSTAGE);
        const uint32_t base = su32(smem + st * OSTAGE);
#pragma unroll
        for (int p = 0; p < OP; ++p) {
          tma_load_3d(base + p * OA_TILE, &amap, a_k0 + kb * OBK, mb * OM, p, full);
          tma_load_3d(base + OP * OA_TILE + p * OB_TILE, &bmap, kb * OBK, nb * ON, p, full);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer ----------------
      for (int kb = 0; kb < nkb; ++kb) {
        const int st = kb % OSTAGES;
        mbar_wait(su32(&bars[st]), (uint32_t)((kb / OSTAGES) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;\n");
        const uint32_t a0 = su32(smem + st * OSTAGE), b0 = a0 + OP * OA_TILE;
#pragma unroll
        for (int kk = 0; kk < OBK / 32; ++kk)
#pragma unroll
          for (int p = 0; p < OP; ++p)
#pragma unroll
            for (int q = 0; q + p < OP; ++q) {
              // the first write of class p + q is pair (0, q) at the first k-step
              const bool first = kb == 0 && kk == 0 && p == 0;
              mma_i8(tmem + (uint32_t)((p + q) * ON), desc_sw(a0 + p * OA_TILE + kk * 32),
                     desc_sw(b0 + q * OB_TILE + kk * 32), first ? 0u : 1u);
            }
        mma_commit(su32(&bars[OSTAGES + st]));  // stage free once these MMAs complete
      }
      mma_commit(su32(&bars[2 * OSTAGES]));  // accumulators final
    }
  } else {  // ---------------- epilogue: warps 2-5 ----------------
    // class sums -> fp64 tile in shared memory (the stage ring is idle once the
    // accumulators are final), then coalesced row-wise (+)= into `out`
    const int qd = warp & 3;  // TMEM lane quarter of this warp
    const int r = 32 * qd + lane;
    const int64_t row = (int64_t)mb * OM + r;
    const uint32_t tl = tmem + ((uint32_t)(32 * qd) << 16);
    double* tile = reinterpret_cast<double*>(smem);  // [OM][ON + 1]
    mbar_wait(su32(&bars[2 * OSTAGES]), 0u);
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const double rs = row < M ? rscale[row] : 0.0;
#pragma unroll 1
    for (int c0 = 0; c0 < ON; c0 += 16) {
      uint32_t v[OP][16];
#pragma unroll
      for (int k = 0; k < OP; ++k) tmem_ld16(tl + (uint32_t)(k * ON + c0), v[k]);
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
      for (int jj = 0; jj < 16; ++jj) {
        // sum_k 2^-7k S_k, smallest terms first
        double h = (double)(int)v[OP - 1][jj];
#pragma unroll
        for (int k = OP - 2; k >= 0; --k) h = fma(h, kDigitW, (double)(int)v[k][jj]);
        tile[r * (ON + 1) + c0 + jj] = h * rs;
      }
    }
    asm volatile("bar.sync 1, 128;\n" ::: "memory");  // the four epilogue warps
    const int t = threadIdx.x - 64;
    for (int e = t; e < OM * ON; e += 128) {
      const int rr = e / ON, cc = e % ON;
      const int64_t gi = (int64_t)mb * OM + rr, gj = (int64_t)nb * ON + cc;
      if (gi < M && gj < N) {
        const double val = nkb > 0 ? tile[rr * (ON + 1) + cc] * cscale[gj] : 0.0;
        double* o = out + gi * out_rs + gj * out_cs;
        *o = accumulate ? *o + val : val;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 2) {
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512));
  }
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeFn oz_encode() {
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

// planes [OP][rows][pitch] int8 (K-major), boxes of 32 k x box_rows rows x 1 plane
void oz_plane_map(CUtensorMap* m, const int8_t* planes, int64_t kdim, int64_t rows, int64_t pitch,
                  uint32_t box_rows) {
  const cuuint64_t dims[3] = {(cuuint64_t)kdim, (cuuint64_t)rows, (cuuint64_t)OP};
  const cuuint64_t strides[2] = {(cuuint64_t)pitch, (cuuint64_t)(pitch * rows)};
  const cuuint32_t box[3] = {(cuuint32_t)OBK, box_rows, 1};
  const cuuint32_t es[3] = {1, 1, 1};
  const CUresult r = oz_encode()(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t*>(planes), dims, strides,
                                 box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 OBK == 32 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_64B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled (Ozaki digit planes) failed: " + std::to_string((int)r));
}

}  // namespace

bool ozaki_available() {
  static const bool off = std::getenv("RNLA_GAUSS_DMMA") != nullptr;
  return !off && oz_encode() != nullptr && tc_gemm_enabled();
}

bool ozaki_applies(int64_t s, int64_t L) {
  return ozaki_available() && s >= OM && L >= 16 && s < INT32_MAX && L < INT32_MAX;
}

// out[t * out_rs + c * out_cs] (+)= sum_{k0 <= j < k0 + kc} Gs(j, t) in[j * ld + c] for t < s, c < L
// with Gs = g (n x s column-major fp64). False when the shape does not apply.
bool ozaki_gaussian_chunk(rnla_ctx* ctx, const DenseOperator& g, const double* in, int64_t ld, int64_t n, int64_t L,
                          int64_t s, int64_t k0, int64_t kc, bool accumulate, double* out, int64_t out_rs,
                          int64_t out_cs) {
  // class sums stay below 2^31: 6 pairs x kc x 64^2 for kc <= 65536
  // chunk starts on a 32-k box boundary (measured: an unaligned k0 -- the
  // world-3 shard chunks of 171 buckets -- faults in the kernel)
  if (!ozaki_applies(s, L) || g.dtype != RNLA_F64 || kc < OBK || kc > kMaxKc || n >= INT32_MAX || (k0 % OBK) != 0)
    return false;
  // Omega's digit planes and row scales, once per cached operator
  if (!g.oz_planes.p) {
    g.oz_pitch = (n + 15) / 16 * 16;
    g.oz_planes = DevBuf((size_t)OP * (size_t)s * (size_t)g.oz_pitch, ctx->stream);
    g.oz_rscale = DevBuf(sizeof(double) * (size_t)s, ctx->stream);
    oz_row_digits<<<(unsigned)s, 256, 0, ctx->stream>>>(n, g.data.as<double>(), n, g.oz_planes.as<int8_t>(),
                                                        g.oz_pitch, s * g.oz_pitch, g.oz_rscale.as<double>());
    RNLA_CUDA(cudaGetLastError());
    note_launch(ctx);
  }
  const int64_t pitch = (kc + 15) / 16 * 16;
  DevBuf bp((size_t)OP * (size_t)L * (size_t)pitch, ctx->stream), cs(sizeof(double) * (size_t)L, ctx->stream),
      cm(sizeof(unsigned long long) * (size_t)L, ctx->stream);
  RNLA_CUDA(cudaMemsetAsync(cm.p, 0, sizeof(unsigned long long) * (size_t)L, ctx->stream));
  const dim3 cgrid((unsigned)((L + 31) / 32), (unsigned)((pitch + 127) / 128));
  oz_col_max<<<cgrid, 256, 0, ctx->stream>>>(kc, L, in + k0 * ld, ld, cm.as<unsigned long long>());
  RNLA_CUDA(cudaGetLastError());
  oz_col_digits<<<cgrid, 256, 0, ctx->stream>>>(kc, L, in + k0 * ld, ld, cm.as<unsigned long long>(),
                                                bp.as<int8_t>(), pitch, L * pitch, cs.as<double>());
  RNLA_CUDA(cudaGetLastError());
  note_launch(ctx, 2);
  CUtensorMap amap, bmap;
  oz_plane_map(&amap, g.oz_planes.as<int8_t>(), n, s, g.oz_pitch, OM);
  oz_plane_map(&bmap, bp.as<int8_t>(), kc, L, pitch, ON);
  ensure_dyn_smem((const void*)oz_gemm_kernel, OSMEM);
  const int nkb = (int)((kc + OBK - 1) / OBK);
  dim3 grid((unsigned)((L + ON - 1) / ON), (unsigned)((s + OM - 1) / OM));
  oz_gemm_kernel<<<grid, OTHREADS, OSMEM, ctx->stream>>>(amap, bmap, s, L, (int)k0, nkb, g.oz_rscale.as<double>(),
                                                         cs.as<double>(), out, out_rs, out_cs, accumulate ? 1 : 0);
  RNLA_CUDA(cudaGetLastError());
  note_launch(ctx);
  return true;
}

// C (m x n; element (i, j) at C[i * c_rs + j * c_cs]) = A B in fp64 through the
// same exact digit products, with A given by rows (A(i, k) = A[i * a_ld + k])
// and B by columns (B(k, j) = B[j * b_ld + k]): both digit sets come from the
// row-digit kernel (each row of A / column of B scaled by its own power of
// two). Used for the dense Nystrom products G T and T'(G T). False when the
// shape does not apply.
bool ozaki_gemm_rowcol(rnla_ctx* ctx, int64_t m, int64_t n, int64_t k, const double* A, int64_t a_ld, const double* B,
                       int64_t b_ld, double* C, int64_t c_rs, int64_t c_cs) {
  if (!ozaki_available() || m < 1 || n < 16 || k < OBK || k > kMaxKc || m >= INT32_MAX || n >= INT32_MAX) return false;
  const int64_t pitch = (k + 15) / 16 * 16;
  DevBuf ap((size_t)OP * (size_t)m * (size_t)pitch, ctx->stream), bp((size_t)OP * (size_t)n * (size_t)pitch, ctx->stream);
  DevBuf rs(sizeof(double) * (size_t)m, ctx->stream), cs(sizeof(double) * (size_t)n, ctx->stream);
  oz_row_digits<<<(unsigned)m, 256, 0, ctx->stream>>>(k, A, a_ld, ap.as<int8_t>(), pitch, m * pitch, rs.as<double>());
  RNLA_CUDA(cudaGetLastError());
  oz_row_digits<<<(unsigned)n, 256, 0, ctx->stream>>>(k, B, b_ld, bp.as<int8_t>(), pitch, n * pitch, cs.as<double>());
  RNLA_CUDA(cudaGetLastError());
  note_launch(ctx, 2);
  CUtensorMap amap, bmap;
  oz_plane_map(&amap, ap.as<int8_t>(), k, m, pitch, OM);
  oz_plane_map(&bmap, bp.as<int8_t>(), k, n, pitch, ON);
  ensure_dyn_smem((const void*)oz_gemm_kernel, OSMEM);
  dim3 grid((unsigned)((n + ON - 1) / ON), (unsigned)((m + OM - 1) / OM));
  oz_gemm_kernel<<<grid, OTHREADS, OSMEM, ctx->stream>>>(amap, bmap, m, n, 0, (int)((k + OBK - 1) / OBK),
                                                         rs.as<double>(), cs.as<double>(), C, c_rs, c_cs, 0);
  RNLA_CUDA(cudaGetLastError());
  note_launch(ctx);
  return true;
}

}  // namespace rnla
