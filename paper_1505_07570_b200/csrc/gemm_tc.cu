// gemm_tc.cu -- fp32 GEMM on the 5th-generation tensor cores (tcgen05, TMEM)
// with the BF16x3 split: x = hi + lo (hi = bf16(x), lo = bf16(x - hi)),
// A*B ~= Ahi*Bhi + Ahi*Blo + Alo*Bhi, fp32 accumulation in TMEM.
//
// Used for the fp32 projections of BASELINE configs 2-4 (rSVD A*Omega,
// A'*Q, A*Z, Q'*A; Gram products). The split costs 3 MMAs but keeps the
// relative error at ~1e-6 (SURVEY §7 hard part 5 measured 4.4e-6 rel-F at the
// config 3 shape; 1-pass BF16 2.3e-3 and 1-pass TF32 2.9e-4 fail the 1e-4
// gate), at an effective 1/3 of the BF16 tensor peak (~550 TF measured).
//
// CTA = one 128 x BN output tile (BN <= 160, multiple of 16) over a K range:
//   warps 0-7  : producers -- load fp32 A/B tiles (64 k per stage) from global,
//                split to bf16 hi/lo and store them in the canonical K-major
//                SWIZZLE_128B smem layout; mbarrier `full[stage]`;
//   warp 12    : one lane issues 4 k-steps x 3 tcgen05.mma (kind::f16, M=128,
//                N=BN, K=16) per stage into TMEM partial buffer X[c & 1] and
//                commits to `empty[stage]`; every TC_PROMOTE_KB stages it
//                commits `xfull` and later waits `xfree` before reusing X;
//   warps 8-11 : epilogue -- tcgen05.ld X, add into the TMEM accumulator Y
//                with fp32 CUDA-core adds (tcgen05.st), final alpha/beta store.
// Global operands may be K-contiguous or MN-contiguous; the converting
// loader always produces K-major smem, so only the K-major descriptor is used.
// The fp32 tile lands by TMA and is split by converter warps: in place into
// shared-memory images (gemm_bf16x3_kernel / _persist) or into TMEM
// (gemm_bf16x3_ts_kernel, the A operand then never touches shared memory again).
#include <cuda.h>
#include <cuda_bf16.h>

#include "rnla_internal.h"
#include "util.cuh"

namespace rnla {

namespace {

// k per pipeline stage: 64 (SWIZZLE_128B bf16 rows). 32 (SWIZZLE_64B) keeps
// twice as many stages in the same shared memory; measured on B200 it is no
// faster (config 3 36.9 vs 36.6 ms, leverage Gram 30.6 vs 30.0 ms) and its
// register-staged fallback spills, so it stays a build option.
#ifndef RNLA_TC_BK
#define RNLA_TC_BK 64
#endif
constexpr int TC_BM = 128, TC_BK = RNLA_TC_BK, TC_STAGES_MAX = 8;
// bf16 pieces per operand in the double-float (fp64-output) mode. 2 (BF16x3
// products, double-float accumulation): the config-2 leverage Gram 8.1 -> 5.0 ms
// with the same worst-row score error vs the fp64 oracle (3.77e-5 vs 3.74e-5
// with the 3-piece BF16x6 split; the M R^-1 row-norm GEMM bounds it).
#ifndef RNLA_TC_DF_PK  // k per TMEM partial sum before the double-float promotion
#define RNLA_TC_DF_PK 256
#endif
#ifndef RNLA_TC_DF_NS
#define RNLA_TC_DF_NS 2
#endif
static_assert(TC_BK == 64 || TC_BK == 32, "TC_BK must be 32 or 64");
constexpr int ROWB = TC_BK * 2;  // bytes per K-major bf16 tile row
constexpr int QPR = TC_BK / 8;   // 16-B chunks per tile row
// physical 16-B chunk of logical chunk q in row r: SW128 (q ^ (r & 7)) or SW64 (q ^ ((r >> 1) & 3))
__host__ __device__ constexpr uint32_t swz(int r, int q) {
  return TC_BK == 64 ? (uint32_t)(q ^ (r & 7)) : (uint32_t)(q ^ ((r >> 1) & 3));
}
__host__ __device__ constexpr uint32_t tile_off(int r, int q) { return (uint32_t)r * ROWB + (swz(r, q) << 4); }
// Producer groups of 4 warps take k-blocks round-robin (more groups = more
// A bytes in flight per SM: the loads are register-staged).
#ifndef RNLA_TC_NGROUPS
#define RNLA_TC_NGROUPS 2
#endif
constexpr int TC_NGROUPS = RNLA_TC_NGROUPS;
constexpr int TC_GROUP = 128;                     // producer group (4 warps) per k-block
constexpr int TC_PRODUCERS = TC_GROUP * TC_NGROUPS;  // warps 0 .. 4*NG-1
constexpr int TC_EPI_WARP0 = 4 * TC_NGROUPS;      // 4 epilogue warps (TMEM lane quarters)
constexpr int TC_MMA_WARP = TC_EPI_WARP0 + 4;     // one MMA-issuing warp
constexpr int TC_THREADS = 32 * (TC_MMA_WARP + 1);

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}\n" ::"r"(bar) : "memory");
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

// Shared-memory matrix descriptor, K-major swizzled: rows of ROWB bytes,
// 8-row atoms of 8*ROWB bytes (SBO), LBO unused (1), version 1 (sm_100);
// layout code 2 = SWIZZLE_128B, 4 = SWIZZLE_64B.
__device__ __forceinline__ uint64_t kmajor_sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;                     // LBO (ignored for swizzled K-major)
  d |= (uint64_t)((8 * ROWB) >> 4) << 32;     // SBO: next 8-row group
  d |= (uint64_t)1 << 46;                     // version = 1
  d |= (uint64_t)(TC_BK == 64 ? 2 : 4) << 61;  // swizzle mode
  return d;
}

// kind::f16 instruction descriptor: D f32, A/B bf16, both K-major, M=128, N.
__host__ __device__ constexpr uint32_t idesc_bf16_f32(int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(bar)
               : "memory");
}

constexpr int TC_PROMOTE_KB = 512 / TC_BK;  // k-blocks per TMEM partial sum (512 k)

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n" ::"r"(
          taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}

// (hi, lo) <- (yh, yl) + x with Knuth's TwoSum on the high words; the
// rounding error of every addition is carried in lo.
__device__ __forceinline__ void two_sum_acc(float yh, float yl, float x, float& hi, float& lo) {
  const float s = __fadd_rn(yh, x);
  const float bp = __fsub_rn(s, yh);
  const float ap = __fsub_rn(s, bp);
  const float e = __fadd_rn(__fsub_rn(yh, ap), __fsub_rn(x, bp));
  hi = s;
  lo = __fadd_rn(yl, e);
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

// Split 8 fp32 values into NS 16-B bf16 chunks: x = p0 + p1 (+ p2), each
// piece the bf16 rounding of the remaining residual.
template <int NS>
__device__ __forceinline__ void split8n(const float* f, uint4* out) {
  float r[8];
#pragma unroll
  for (int t = 0; t < 8; ++t) r[t] = f[t];
#pragma unroll
  for (int p = 0; p < NS; ++p) {
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      w[i] = pack_bf16(r[2 * i], r[2 * i + 1]);
      __nv_bfloat162 hb = *reinterpret_cast<__nv_bfloat162*>(&w[i]);
      r[2 * i] -= __low2float(hb);
      r[2 * i + 1] -= __high2float(hb);
    }
    out[p] = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

// Split 8 fp32 values into 16-B bf16 hi and lo chunks.
__device__ __forceinline__ void split8(const float* f, uint4& hi, uint4& lo) {
  float r[8];
  uint32_t h[4], l[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    h[i] = pack_bf16(f[2 * i], f[2 * i + 1]);
    __nv_bfloat162 hb = *reinterpret_cast<__nv_bfloat162*>(&h[i]);
    r[2 * i] = f[2 * i] - __low2float(hb);
    r[2 * i + 1] = f[2 * i + 1] - __high2float(hb);
    l[i] = pack_bf16(r[2 * i], r[2 * i + 1]);
  }
  hi = make_uint4(h[0], h[1], h[2], h[3]);
  lo = make_uint4(l[0], l[1], l[2], l[3]);
}

// One operand tile: R rows (MN) x 64 k of X(r, k) = X[r*rs + k*ks] with rows
// [r0, r0 + R) valid below `rows`, k valid below `kend`, into K-major SW128
// hi/lo tiles (row r at r*128 B, 16-B chunk q at (q ^ (r & 7)) * 16).
template <bool KCONTIG>
__device__ __forceinline__ void unit_coords(int u, int R, int& r, int& q) {
  if (KCONTIG) {  // QPR lanes cover one row's TC_BK k contiguous
    r = u / QPR;
    q = u % QPR;
  } else {  // lanes run along rows (MN-contiguous in global)
    r = u % R;
    q = u / R;
  }
}

template <bool KCONTIG>
__device__ __forceinline__ void load_unit(const float* __restrict__ X, int64_t rs, int64_t ks, int64_t rows,
                                          int64_t gr, int64_t gk, int64_t kend, float* f) {
  if (gr < rows && gk + 8 <= kend) {
    const float* p = X + gr * rs + gk * ks;
    if (KCONTIG && ((reinterpret_cast<uintptr_t>(p) & 15) == 0)) {
      const float4 a = __ldg(reinterpret_cast<const float4*>(p));
      const float4 b = __ldg(reinterpret_cast<const float4*>(p) + 1);
      f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w; f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
    } else {
#pragma unroll
      for (int t = 0; t < 8; ++t) f[t] = __ldg(p + t * ks);
    }
  } else {
#pragma unroll
    for (int t = 0; t < 8; ++t) f[t] = (gr < rows && gk + t < kend) ? __ldg(X + gr * rs + (gk + t) * ks) : 0.f;
  }
}

#ifndef RNLA_TC_PF
#define RNLA_TC_PF 0  // measured: no gain on the config-3 passes (38.3 vs 38.8 ms); off by default
#endif
// L2 prefetch of one 128-row x 64-k fp32 tile by the 128 threads of a group.
template <bool KCONTIG>
__device__ __forceinline__ void prefetch_tile_l2(const float* __restrict__ X, int64_t rs, int64_t ks, int64_t rows,
                                                 int64_t r0, int64_t k0, int64_t kend, int tid) {
  if (KCONTIG) {  // row r = tid: 64 k = 256 B = two 128-B lines
    const int64_t gr = r0 + tid;
    if (gr < rows) {
      const float* p = X + gr * rs + k0 * ks;
      asm volatile("prefetch.global.L2::evict_last [%0];\n" ::"l"(p));
      if (k0 + 32 < kend) asm volatile("prefetch.global.L2::evict_last [%0];\n" ::"l"(p + 32 * ks));
    }
  } else {  // k-row kk = tid / 2 (64 of them), half h: rows r0 + 64h .. of 128 contiguous floats
    const int kk = tid >> 1, h = tid & 1;
    const int64_t gk = k0 + kk, gr = r0 + 64 * h;
    if (gk < kend && gr < rows) {
      const float* p = X + gr * rs + gk * ks;
      asm volatile("prefetch.global.L2::evict_last [%0];\n" ::"l"(p));
      if (gr + 32 < rows) asm volatile("prefetch.global.L2::evict_last [%0];\n" ::"l"(p + 32 * rs));
    }
  }
}

// All loads of the tile are issued before any conversion (R*8/256 units per
// thread in flight), then each unit is split and stored.
// NS pieces go to tiles base, base + R*128, base + 2*R*128.
template <bool KCONTIG, int R, int NT, int NS>
__device__ __forceinline__ void load_split_tile(const float* __restrict__ X, int64_t rs, int64_t ks, int64_t rows,
                                                int64_t r0, int64_t k0, int64_t kend, uint8_t* base, int tid) {
  constexpr int UNITS = R * QPR;  // (row, 8-k chunk)
  constexpr int UPT = (UNITS + NT - 1) / NT;
  float f[UPT][8];
#pragma unroll
  for (int i = 0; i < UPT; ++i) {
    const int u = tid + i * NT;
    if (UNITS % NT == 0 || u < UNITS) {
      int r, q;
      unit_coords<KCONTIG>(u, R, r, q);
      load_unit<KCONTIG>(X, rs, ks, rows, r0 + r, k0 + 8 * q, kend, f[i]);
    }
  }
#pragma unroll
  for (int i = 0; i < UPT; ++i) {
    const int u = tid + i * NT;
    if (UNITS % NT == 0 || u < UNITS) {
      int r, q;
      unit_coords<KCONTIG>(u, R, r, q);
      uint4 pc[NS];
      split8n<NS>(f[i], pc);
      const uint32_t off = tile_off(r, q);
#pragma unroll
      for (int p = 0; p < NS; ++p) *reinterpret_cast<uint4*>(base + p * (R * ROWB) + off) = pc[p];
    }
  }
}

// B operand prepared once per GEMM: every (n-block, k-block) tile split to
// bf16 hi/lo and stored in global memory as the exact K-major SW128 smem
// image [hi BN x 128 B][lo BN x 128 B], so the main loop moves it with one
// cp.async.bulk per stage (no conversion, no registers). B (Omega, Q, Z) is
// small and re-read by every M tile, so this also halves its L2 traffic vs fp32.
template <int NS>
__global__ void split_b_image(int64_t K, int64_t N, const float* __restrict__ B, int64_t b_rs, int64_t b_cs, int BN,
                              int64_t nkb, int64_t nblk, uint8_t* __restrict__ img) {
  const int64_t total = nblk * nkb * BN * QPR;
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < total; u += (int64_t)gridDim.x * blockDim.x) {
    const int q = (int)(u % QPR);
    const int64_t rest0 = u / QPR;
    const int j = (int)(rest0 % BN);
    const int64_t rest = rest0 / BN;
    const int64_t kb = rest % nkb, nb = rest / nkb;
    const int64_t gj = nb * BN + j, gk = kb * TC_BK + 8 * q;
    float f[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) f[t] = (gj < N && gk + t < K) ? B[(gk + t) * b_rs + gj * b_cs] : 0.f;
    uint4 pc[NS];
    split8n<NS>(f, pc);
    uint8_t* tile = img + (nb * nkb + kb) * (int64_t)(NS * BN * ROWB);
    const uint32_t off = tile_off(j, q);
#pragma unroll
    for (int p = 0; p < NS; ++p) *reinterpret_cast<uint4*>(tile + p * BN * ROWB + off) = pc[p];
  }
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}\n" ::"r"(bar),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void tma_load_2d_g2s(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          dst),
      "l"(map), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}

__device__ __forceinline__ void named_bar_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}

// TMA-fed variant: the fp32 A k-block (128 rows x 64 k) lands in the stage by
// TMA (K-contiguous A: two 128 B-wide SWIZZLE_128B boxes; MN-contiguous A: one
// unswizzled [64 k][128 rows] box), then a producer group reads it from smem,
// splits it and writes the bf16 pieces IN PLACE (the pieces need as many
// bytes as the fp32 tile for NS = 2): the DRAM latency is covered by the TMA
// ring instead of by registers.
template <bool KCONTIG, int NS>
__device__ __forceinline__ void convert_tile_inplace(uint8_t* base, int gtid, int grp) {
  constexpr int UPT = (TC_BM * QPR) / TC_GROUP;
  constexpr int A_TILE = TC_BM * ROWB;
  constexpr int FBOX = TC_BM * 128;  // one TMA box: 128 rows x 32 fp32 (128 B, SWIZZLE_128B)
  // K-contiguous tiles: each 8-lane phase takes one 16-B chunk index q of 8
  // consecutive rows, whose swizzled positions are all distinct, so both the
  // fp32 reads and the bf16 writes are bank-conflict free.
  auto coords = [](int u, int& r, int& q) {
    if (KCONTIG) {
      r = (u & 7) + 8 * (u / (8 * QPR));
      q = (u >> 3) % QPR;
    } else {
      unit_coords<false>(u, TC_BM, r, q);
    }
  };
  float f[UPT][8];
#pragma unroll
  for (int i = 0; i < UPT; ++i) {
    const int u = gtid + i * TC_GROUP;
    int r, q;
    coords(u, r, q);
    if (KCONTIG) {  // fp32 k 8q..8q+7: box q / 4, 16-B granules 2 (q % 4) and +1 of the SW128 row
      const uint8_t* row = base + (q >> 2) * FBOX + r * 128;
      const int g0 = (q & 3) * 2;
      const float4 a = *reinterpret_cast<const float4*>(row + ((g0 ^ (r & 7)) << 4));
      const float4 b = *reinterpret_cast<const float4*>(row + (((g0 + 1) ^ (r & 7)) << 4));
      f[i][0] = a.x; f[i][1] = a.y; f[i][2] = a.z; f[i][3] = a.w;
      f[i][4] = b.x; f[i][5] = b.y; f[i][6] = b.z; f[i][7] = b.w;
    } else {
      const float* tile = reinterpret_cast<const float*>(base);  // [TC_BK k][128 rows]
#pragma unroll
      for (int t = 0; t < 8; ++t) f[i][t] = tile[(8 * q + t) * TC_BM + r];
    }
  }
  named_bar_sync(1 + grp, TC_GROUP);  // the whole fp32 tile is in registers before it is overwritten
#pragma unroll
  for (int i = 0; i < UPT; ++i) {
    const int u = gtid + i * TC_GROUP;
    int r, q;
    coords(u, r, q);
    uint4 pc[NS];
    split8n<NS>(f[i], pc);
    const uint32_t off = tile_off(r, q);
#pragma unroll
    for (int p = 0; p < NS; ++p) *reinterpret_cast<uint4*>(base + p * A_TILE + off) = pc[p];
  }
}

__device__ __forceinline__ void bulk_copy_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

// DF = double-float accumulation: Y kept as an unevaluated fp32 pair (hi, lo)
// updated with TwoSum every 4 k-blocks (256 rows), output in fp64 -- for the
// Nystrom Gram C'C, whose W^+-weighted eigenvalues need fp64-grade
// accumulation across <= 256-row chunks (SURVEY §7 hard part 8).
template <bool A_KC, int BN, int STAGES, bool DF, bool TMA_A>
__global__ void __launch_bounds__(TMA_A ? TC_THREADS + 32 : TC_THREADS, 1)
    gemm_bf16x3_kernel(int64_t M, int64_t N, int64_t K, int64_t kchunk, const float* __restrict__ A, int64_t a_rs,
                       int64_t a_cs, const uint8_t* __restrict__ bimg, int64_t nkb_total, double alpha,
                       double beta, typename std::conditional<DF, double, float>::type* C, int64_t c_rs, int64_t c_cs,
                       typename std::conditional<DF, double, float>::type* ws, int sym,
                       const __grid_constant__ CUtensorMap amap, double* rownorm) {
  using OutT = typename std::conditional<DF, double, float>::type;
  // symmetric products (C = A'A): tiles strictly below the diagonal are skipped
  // (uniformly for the whole CTA, before any barrier) and mirrored afterwards
  // (sym bit 0). Bit 1: B is upper triangular (B(p, j) = 0 for p > j, the
  // leverage-score product M R^-1), so this N tile needs k < n0 + BN only.
  // Bit 4: the grid is (N tiles, M tiles), so the N tiles of one M tile run
  // together and share its A rows through L2.
  const int64_t mblk = (sym & 16) ? blockIdx.y : blockIdx.x, nblk_i = (sym & 16) ? blockIdx.x : blockIdx.y;
  if ((sym & 1) && mblk * TC_BM >= (nblk_i + 1) * BN) return;
  constexpr int PKB = DF ? RNLA_TC_DF_PK / TC_BK : TC_PROMOTE_KB;
  // DF may split three ways (RNLA_TC_DF_NS = 3, BF16x6: hh, hm, mh, hl, lh, mm ~
  // fp32-faithful products, 1.9e-7 rel-F per SURVEY §7 hard part 5); BF16x3 by default.
  constexpr int NS = DF ? RNLA_TC_DF_NS : 2;
  constexpr int A_TILE = TC_BM * ROWB;  // bytes per bf16 tile (128 rows x TC_BK k)
  constexpr int B_TILE = BN * ROWB;
  constexpr int STAGE = NS * (A_TILE + B_TILE);
  // TMEM: two MMA partial-sum buffers X0, X1 and the promoted accumulator Y.
  // The tensor core's fp32 accumulation does not round to nearest (measured:
  // rel-F error 5.7e-5 at K = 16384 in one accumulator vs 4.6e-6 at K ~ 400),
  // so every TC_PROMOTE_KB k-blocks the epilogue adds the finished partial
  // into Y with CUDA-core fp32 adds while the MMAs fill the other buffer.
  constexpr int TCOLS = (DF ? 4 : 3) * BN;
  static_assert(TCOLS <= 512, "BN too large for promoted accumulation");
  constexpr uint32_t TMEM_COLS = TCOLS <= 128 ? 128 : (TCOLS <= 256 ? 256 : 512);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-B alignment of the shared-window offset by pointer arithmetic on the
  // __shared__ array (an integer round trip would turn every tile access into
  // a generic LD.E/ST.E instead of LDS/STS).
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  // full[S], empty[S], xfull[2], xfree[2], tfull[S] (TMA_A: the A tile and B image landed)
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE);
  uint64_t* tfull = bars + 2 * STAGES + 4;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * STAGES + 4);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t m0 = mblk * TC_BM, n0 = nblk_i * BN;
  const int64_t kbeg = (int64_t)blockIdx.z * kchunk;
  const int64_t kend = (sym & 2) ? min(min(K, kbeg + kchunk), n0 + BN) : min(K, kbeg + kchunk);
  const int nkb = (int)((kend - kbeg + TC_BK - 1) / TC_BK);

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      // a producer group (+ the bulk-copy expect_tx arrive when the group issues it)
      mbar_init(smem_u32(&bars[s]), TMA_A ? TC_GROUP : TC_GROUP + 1);
      mbar_init(smem_u32(&bars[STAGES + s]), 1);
      mbar_init(smem_u32(&tfull[s]), 1);
    }
    mbar_init(smem_u32(&bars[2 * STAGES]), 1);      // xfull[0]
    mbar_init(smem_u32(&bars[2 * STAGES + 1]), 1);  // xfull[1]
    mbar_init(smem_u32(&bars[2 * STAGES + 2]), 128);  // xfree[0] (epilogue threads)
    mbar_init(smem_u32(&bars[2 * STAGES + 3]), 128);  // xfree[1]
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == TC_EPI_WARP0) {  // TMEM accumulator: 128 lanes x TMEM_COLS fp32 columns
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = *tmem_slot;

  if (TMA_A && warp < TC_EPI_WARP0) {
    // ---------------- converters: groups take k-blocks round-robin; each waits
    // for its stage's TMA, splits the fp32 tile in place, hands it to the MMA ----------------
    const int grp = warp >> 2, gtid = tid & (TC_GROUP - 1);
    for (int kb = grp; kb < nkb; kb += TC_NGROUPS) {
      const int st = kb % STAGES;
      // TMA completions may land out of order: before the parity wait on tfull,
      // make sure the stage's previous phase (k-block kb - STAGES) was consumed,
      // so this wait cannot alias a phase two steps back.
      if (kb >= STAGES) mbar_wait(smem_u32(&bars[STAGES + st]), (uint32_t)(((kb / STAGES) - 1) & 1));
      mbar_wait(smem_u32(&tfull[st]), (uint32_t)((kb / STAGES) & 1));
      convert_tile_inplace<A_KC, NS>(smem + st * STAGE, gtid, grp);
      // Gram with B = A' (sym bit 3, BN == TC_BM): the B tile is the A operand's
      // tile at column block n0, landed by TMA and split the same way.
      // (A diagonal tile, m0 == n0, has B == A: the MMA reads the A pieces twice.)
      if (BN == TC_BM && (sym & 8) && m0 != n0)
        convert_tile_inplace<A_KC, NS>(smem + st * STAGE + NS * A_TILE, gtid, grp);
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      mbar_arrive(smem_u32(&bars[st]));
    }
  } else if (TMA_A && warp == TC_MMA_WARP + 1) {
    // ---------------- TMA issuer: A boxes + the B image of each stage ----------------
    if (lane == 0) {
      const int64_t kb0 = kbeg / TC_BK;
      const uint8_t* bsrc = bimg + (nblk_i * nkb_total + kb0) * (int64_t)(NS * B_TILE);
      for (int kb = 0; kb < nkb; ++kb) {
        const int st = kb % STAGES;
        if (kb >= STAGES) mbar_wait(smem_u32(&bars[STAGES + st]), (uint32_t)(((kb / STAGES) - 1) & 1));
        uint8_t* base = smem + st * STAGE;
        const uint32_t bar = smem_u32(&tfull[st]);
        const bool b_from_a = BN == TC_BM && (sym & 8);
        const bool b_is_a = b_from_a && m0 == n0;
        mbar_arrive_expect_tx(bar, (uint32_t)(TC_BM * TC_BK * 4 +
                                              (b_is_a ? 0 : (b_from_a ? TC_BM * TC_BK * 4 : NS * B_TILE))));
        const int k0 = (int)(kbeg + (int64_t)kb * TC_BK);
        if (A_KC) {  // one 128-row x 32-fp32 SWIZZLE_128B box per 32 k
#pragma unroll
          for (int b = 0; b < TC_BK / 32; ++b)
            tma_load_2d_g2s(smem_u32(base + b * TC_BM * 128), &amap, k0 + 32 * b, (int)m0, bar);
        } else {
          tma_load_2d_g2s(smem_u32(base), &amap, (int)m0, k0, bar);
        }
        if (b_is_a) {
        } else if (b_from_a) {
          if (A_KC) {
#pragma unroll
            for (int b = 0; b < TC_BK / 32; ++b)
              tma_load_2d_g2s(smem_u32(base + NS * A_TILE + b * TC_BM * 128), &amap, k0 + 32 * b, (int)n0, bar);
          } else {
            tma_load_2d_g2s(smem_u32(base + NS * A_TILE), &amap, (int)n0, k0, bar);
          }
        } else {
          bulk_copy_g2s(smem_u32(base + NS * A_TILE), bsrc + (int64_t)kb * (NS * B_TILE), NS * B_TILE, bar);
        }
      }
    }
    __syncwarp();
  } else if (warp < TC_EPI_WARP0) {
    // ---------------- producers: two groups of 4 warps take alternate k-blocks,
    // so two k-blocks of A loads are in flight per SM ----------------
    const int grp = warp >> 2, gtid = tid & (TC_GROUP - 1);
    const int64_t kb0 = kbeg / TC_BK;
    const uint8_t* bsrc = bimg + (nblk_i * nkb_total + kb0) * (int64_t)(NS * B_TILE);
    for (int kb = grp; kb < nkb; kb += TC_NGROUPS) {
      const int st = kb % STAGES;
#if RNLA_TC_PF > 0
      {  // warm L2 with this group's k-block RNLA_TC_PF rounds ahead (hides DRAM latency
         // of the register-staged loads without more registers)
        const int64_t kp = kbeg + (int64_t)(kb + RNLA_TC_PF * TC_NGROUPS) * TC_BK;
        if (kp < kend) prefetch_tile_l2<A_KC>(A, a_rs, a_cs, M, m0, kp, kend, gtid);
      }
#endif
      if (kb >= STAGES) mbar_wait(smem_u32(&bars[STAGES + st]), (uint32_t)(((kb / STAGES) - 1) & 1));
      uint8_t* base = smem + st * STAGE;
      if (gtid == 0) {
        mbar_arrive_expect_tx(smem_u32(&bars[st]), NS * B_TILE);
        bulk_copy_g2s(smem_u32(base + NS * A_TILE), bsrc + (int64_t)kb * (NS * B_TILE), NS * B_TILE,
                      smem_u32(&bars[st]));
      }
      const int64_t k0 = kbeg + (int64_t)kb * TC_BK;
      load_split_tile<A_KC, TC_BM, TC_GROUP, NS>(A, a_rs, a_cs, M, m0, k0, kend, base, gtid);
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      mbar_arrive(smem_u32(&bars[st]));
    }
  } else if (warp == TC_MMA_WARP) {
    {
      // ---------------- MMA issuer (own warp: it waits on epilogue arrivals) ----------------
      if (lane == 0) {
        constexpr uint32_t idesc = idesc_bf16_f32(BN);
        for (int kb = 0; kb < nkb; ++kb) {
          const int st = kb % STAGES;
          const int chunk = kb / PKB, xb = chunk & 1, kin = kb % PKB;
          if (kin == 0 && chunk >= 2)  // X[xb] drained by the epilogue (chunk - 2)?
            mbar_wait(smem_u32(&bars[2 * STAGES + 2 + xb]), (uint32_t)(((chunk / 2) - 1) & 1));
          mbar_wait(smem_u32(&bars[st]), (uint32_t)((kb / STAGES) & 1));
          asm volatile("tcgen05.fence::after_thread_sync;\n");
          const uint32_t dst = tmem + (uint32_t)(xb * BN);
          const uint32_t base = smem_u32(smem + st * STAGE);
          const uint32_t a0 = base, b0 = (BN == TC_BM && (sym & 8) && m0 == n0) ? base : base + NS * A_TILE;
          // products (i, j) of pieces: (0,0) (0,1) (1,0) [+ (0,2) (2,0) (1,1) for NS = 3]
          constexpr int NP = NS == 3 ? 6 : 3;
          constexpr int PI[6] = {0, 0, 1, 0, 2, 1}, PJ[6] = {0, 1, 0, 2, 0, 1};
#pragma unroll
          for (int kk = 0; kk < TC_BK / 16; ++kk) {
            const uint32_t koff = kk * 32;  // 16 bf16 per UMMA_K
#pragma unroll
            for (int p = 0; p < NP; ++p) {
              const uint32_t acc = (p > 0 || kin > 0 || kk > 0) ? 1u : 0u;
              mma_bf16(dst, kmajor_sw128_desc(a0 + PI[p] * A_TILE + koff),
                       kmajor_sw128_desc(b0 + PJ[p] * B_TILE + koff), idesc, acc);
            }
          }
          mma_commit(smem_u32(&bars[STAGES + st]));  // frees the stage when these MMAs finish
          if (kin == PKB - 1 || kb == nkb - 1) mma_commit(smem_u32(&bars[2 * STAGES + xb]));  // X ready
        }
      }
      __syncwarp();
    }
  } else {
    // ---------------- epilogue (warps 8-11) ----------------
    const int quarter = warp & 3;  // TMEM lanes 32*quarter .. +31
    const int64_t row = m0 + quarter * 32 + lane;
    const uint32_t tlane = tmem + ((uint32_t)(quarter * 32) << 16);
    const uint32_t yaddr = tlane + (uint32_t)(2 * BN);
    const uint32_t yloaddr = tlane + (uint32_t)(3 * BN);  // DF: low word of the double-float accumulator
    const int nchunks = (nkb + PKB - 1) / PKB;
    // chunks 0 .. nchunks-2: Y (+)= X[c & 1] in TMEM; the last chunk is combined on the way out
    for (int c = 0; c + 1 < nchunks; ++c) {
      const int xb = c & 1;
      mbar_wait(smem_u32(&bars[2 * STAGES + xb]), (uint32_t)((c / 2) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;\n");
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 16) {
        uint32_t x[16], y[16];
        tmem_ld16(tlane + (uint32_t)(xb * BN + c0), x);
        if (c > 0) tmem_ld16(yaddr + (uint32_t)c0, y);
        if constexpr (DF) {
          uint32_t yl[16];
          if (c > 0) tmem_ld16(yloaddr + (uint32_t)c0, yl);
          asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            float hi = __uint_as_float(x[j]), lo = 0.f;
            if (c > 0) two_sum_acc(__uint_as_float(y[j]), __uint_as_float(yl[j]), __uint_as_float(x[j]), hi, lo);
            x[j] = __float_as_uint(hi);
            yl[j] = __float_as_uint(lo);
          }
          tmem_st16(yloaddr + (uint32_t)c0, yl);
        } else {
          asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
          if (c > 0) {
#pragma unroll
            for (int j = 0; j < 16; ++j) x[j] = __float_as_uint(__uint_as_float(y[j]) + __uint_as_float(x[j]));
          }
        }
        tmem_st16(yaddr + (uint32_t)c0, x);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;\n");
      mbar_arrive(smem_u32(&bars[2 * STAGES + 2 + xb]));  // X[xb] free for chunk c + 2
    }
    const int last = nchunks - 1;
    if (nchunks > 0) {
      mbar_wait(smem_u32(&bars[2 * STAGES + (last & 1)]), (uint32_t)((last / 2) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;\n");
    }
    double rsq = 0.0;
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 16) {
      uint32_t v[16], y[16], yl[16];
      OutT acc[16];
      if (nchunks > 0) {
        tmem_ld16(tlane + (uint32_t)((last & 1) * BN + c0), v);
        if (last > 0) tmem_ld16(yaddr + (uint32_t)c0, y);
        if (DF && last > 0) tmem_ld16(yloaddr + (uint32_t)c0, yl);
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          if constexpr (DF) {
            float hi = __uint_as_float(v[j]), lo = 0.f;
            if (last > 0) two_sum_acc(__uint_as_float(y[j]), __uint_as_float(yl[j]), __uint_as_float(v[j]), hi, lo);
            acc[j] = (OutT)((double)hi + (double)lo);
          } else {
            acc[j] = last > 0 ? __uint_as_float(y[j]) + __uint_as_float(v[j]) : __uint_as_float(v[j]);
          }
        }
      } else {
#pragma unroll
        for (int j = 0; j < 16; ++j) acc[j] = OutT(0);  // empty K range: the sum is zero
      }
      if (rownorm) {  // row-norm mode: sum of squares of this tile's columns, C not written
#pragma unroll
        for (int j = 0; j < 16; ++j)
          if (n0 + c0 + j < N) {
            const double v = alpha * (double)acc[j];
            rsq += v * v;
          }
      } else if (row < M) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int64_t col = n0 + c0 + j;
          if (col < N) {
            if (ws) {
              ws[(int64_t)blockIdx.z * M * N + row * N + col] = acc[j];
            } else {
              OutT* cp = C + row * c_rs + col * c_cs;
              *cp = beta == 0.0 ? (OutT)(alpha * acc[j]) : (OutT)(alpha * acc[j] + beta * *cp);
            }
          }
        }
      }
    }
    if (rownorm && row < M) rownorm[nblk_i * M + row] = rsq;  // [N tile][row]
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == TC_EPI_WARP0) {
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(TMEM_COLS));
  }
}

// Persistent variant for short K (at most two TC_PROMOTE_KB chunks per tile):
// the leverage-score product M R^-1 (K <= 1024, 8 N tiles per M tile) and the
// CholeskyQR applies Y R^-1 of config 3 (K = 150). A CTA walks tiles
// blockIdx.x, + gridDim.x, ... (N-tile fastest, so the N tiles of one M tile run
// on neighbouring CTAs and share its A rows through L2). The TMA ring and the
// converter groups run across tile boundaries, and the fp32 TMEM accumulators
// are double-buffered by tile parity, so the epilogue of tile i overlaps the
// loads, conversion and MMAs of tile i + 1 (the one-tile kernel serializes
// TMA -> convert -> MMA -> epilogue per 128-row tile and pays its setup per
// tile). Chunk sums are combined exactly as the promoting kernel does (fp32
// adds of the <= 512-k partials). sym bit 1: B upper triangular (k < n0 + BN).
template <bool A_KC, int BN, int STAGES, int CH>
__global__ void __launch_bounds__(TC_THREADS + 32, 1)
    gemm_bf16x3_persist(int64_t M, int64_t N, int64_t K, const float* __restrict__ A, const uint8_t* __restrict__ bimg,
                        int64_t nkb_total, double alpha, double beta, float* C, int64_t c_rs, int64_t c_cs, int sym,
                        const __grid_constant__ CUtensorMap amap, double* rownorm, int ntm, int ntn) {
  constexpr int NS = 2;
  constexpr int A_TILE = TC_BM * ROWB, B_TILE = BN * ROWB, STAGE = NS * (A_TILE + B_TILE);
  constexpr uint32_t TCOLS = 2 * CH * BN;
  constexpr uint32_t TMEM_COLS = TCOLS <= 128 ? 128 : (TCOLS <= 256 ? 256 : 512);
  static_assert(TCOLS <= 512, "double-buffered accumulators exceed TMEM");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  // full[S], empty[S], tfull[S], accfull[2], accfree[2]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE);
  uint64_t* full = bars;
  uint64_t* empty = bars + STAGES;
  uint64_t* tfull = bars + 2 * STAGES;
  uint64_t* accfull = bars + 3 * STAGES;
  uint64_t* accfree = bars + 3 * STAGES + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * STAGES + 4);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ntiles = ntm * ntn;
  auto tile_of = [&](int t, int64_t& m0, int64_t& n0, int& nbi, int& nkb) {
    const int mb = t / ntn;
    nbi = t % ntn;
    m0 = (int64_t)mb * TC_BM;
    n0 = (int64_t)nbi * BN;
    const int64_t kend = (sym & 2) ? min(K, n0 + BN) : K;
    nkb = (int)((kend + TC_BK - 1) / TC_BK);
  };
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(smem_u32(&full[s]), TC_GROUP);
      mbar_init(smem_u32(&empty[s]), 1);
      mbar_init(smem_u32(&tfull[s]), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(smem_u32(&accfull[b]), 1);
      mbar_init(smem_u32(&accfree[b]), 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == TC_EPI_WARP0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = *tmem_slot;

  if (warp < TC_EPI_WARP0) {
    // ---------------- converters: global k-block g goes to group g % NG ----------------
    const int grp = warp >> 2, gtid = tid & (TC_GROUP - 1);
    int g = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      int64_t m0, n0;
      int nbi, nkb;
      tile_of(t, m0, n0, nbi, nkb);
      for (int kb = 0; kb < nkb; ++kb, ++g) {
        if (g % TC_NGROUPS != grp) continue;
        const int st = g % STAGES;
        if (g >= STAGES) mbar_wait(smem_u32(&empty[st]), (uint32_t)(((g / STAGES) - 1) & 1));
        mbar_wait(smem_u32(&tfull[st]), (uint32_t)((g / STAGES) & 1));
        convert_tile_inplace<A_KC, NS>(smem + st * STAGE, gtid, grp);
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        mbar_arrive(smem_u32(&full[st]));
      }
    }
  } else if (warp == TC_MMA_WARP + 1) {
    // ---------------- TMA issuer ----------------
    if (lane == 0) {
      int g = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        int64_t m0, n0;
        int nbi, nkb;
        tile_of(t, m0, n0, nbi, nkb);
        const uint8_t* bsrc = bimg + (int64_t)nbi * nkb_total * (int64_t)(NS * B_TILE);
        for (int kb = 0; kb < nkb; ++kb, ++g) {
          const int st = g % STAGES;
          if (g >= STAGES) mbar_wait(smem_u32(&empty[st]), (uint32_t)(((g / STAGES) - 1) & 1));
          uint8_t* base = smem + st * STAGE;
          const uint32_t bar = smem_u32(&tfull[st]);
          mbar_arrive_expect_tx(bar, (uint32_t)(TC_BM * TC_BK * 4 + NS * B_TILE));
          const int k0 = kb * TC_BK;
          if (A_KC) {
#pragma unroll
            for (int b = 0; b < TC_BK / 32; ++b)
              tma_load_2d_g2s(smem_u32(base + b * TC_BM * 128), &amap, k0 + 32 * b, (int)m0, bar);
          } else {
            tma_load_2d_g2s(smem_u32(base), &amap, (int)m0, k0, bar);
          }
          bulk_copy_g2s(smem_u32(base + NS * A_TILE), bsrc + (int64_t)kb * (NS * B_TILE), NS * B_TILE, bar);
        }
      }
    }
    __syncwarp();
  } else if (warp == TC_MMA_WARP) {
    // ---------------- MMA issuer: tile i into accumulator buffer i & 1 ----------------
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_bf16_f32(BN);
      int g = 0, i = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
        int64_t m0, n0;
        int nbi, nkb;
        tile_of(t, m0, n0, nbi, nkb);
        const int buf = i & 1;
        if (i >= 2) mbar_wait(smem_u32(&accfree[buf]), (uint32_t)(((i / 2) - 1) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;\n");
        for (int kb = 0; kb < nkb; ++kb, ++g) {
          const int st = g % STAGES;
          const int chunk = kb / TC_PROMOTE_KB, kin = kb % TC_PROMOTE_KB;
          mbar_wait(smem_u32(&full[st]), (uint32_t)((g / STAGES) & 1));
          asm volatile("tcgen05.fence::after_thread_sync;\n");
          const uint32_t dst = tmem + (uint32_t)((buf * CH + chunk) * BN);
          const uint32_t a0 = smem_u32(smem + st * STAGE), b0 = a0 + NS * A_TILE;
          constexpr int PI[3] = {0, 0, 1}, PJ[3] = {0, 1, 0};
#pragma unroll
          for (int kk = 0; kk < TC_BK / 16; ++kk) {
            const uint32_t koff = kk * 32;
#pragma unroll
            for (int p = 0; p < 3; ++p) {
              const uint32_t acc = (p > 0 || kin > 0 || kk > 0) ? 1u : 0u;
              mma_bf16(dst, kmajor_sw128_desc(a0 + PI[p] * A_TILE + koff), kmajor_sw128_desc(b0 + PJ[p] * B_TILE + koff),
                       idesc, acc);
            }
          }
          mma_commit(smem_u32(&empty[st]));
        }
        mma_commit(smem_u32(&accfull[buf]));
      }
    }
    __syncwarp();
  } else {
    // ---------------- epilogue (warps 8-11) ----------------
    const int quarter = warp & 3;
    const uint32_t tlane = tmem + ((uint32_t)(quarter * 32) << 16);
    int i = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
      int64_t m0, n0;
      int nbi, nkb;
      tile_of(t, m0, n0, nbi, nkb);
      const int buf = i & 1, nch = (nkb + TC_PROMOTE_KB - 1) / TC_PROMOTE_KB;
      const int64_t row = m0 + quarter * 32 + lane;
      mbar_wait(smem_u32(&accfull[buf]), (uint32_t)((i / 2) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;\n");
      double rsq = 0.0;
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 16) {
        uint32_t x0[16], x1[16];
        tmem_ld16(tlane + (uint32_t)(buf * CH * BN + c0), x0);
        if (CH > 1 && nch > 1) tmem_ld16(tlane + (uint32_t)((buf * CH + 1) * BN + c0), x1);
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
        float acc[16];
#pragma unroll
        for (int j = 0; j < 16; ++j)
          acc[j] = (CH > 1 && nch > 1) ? __uint_as_float(x0[j]) + __uint_as_float(x1[j]) : __uint_as_float(x0[j]);
        if (rownorm) {
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (n0 + c0 + j < N) {
              const double v = alpha * (double)acc[j];
              rsq += v * v;
            }
        } else if (row < M) {
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int64_t col = n0 + c0 + j;
            if (col < N) {
              float* cp = C + row * c_rs + col * c_cs;
              *cp = beta == 0.0 ? (float)(alpha * acc[j]) : (float)(alpha * acc[j] + beta * *cp);
            }
          }
        }
      }
      if (rownorm && row < M) rownorm[nbi * M + row] = rsq;
      asm volatile("tcgen05.fence::before_thread_sync;\n");
      mbar_arrive(smem_u32(&accfree[buf]));
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == TC_EPI_WARP0) {
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(TMEM_COLS));
  }
}

// ---------------------------------------------------------------------------
// A-operand-in-TMEM variant (tcgen05.mma with [a_tmem]): the long-K
// projections of config 3 (Y = A Q, Z = A'Q, 128 < N <= 160 in one tile), other
// non-symmetric products with K > 1024 and 32 < N <= 128, and the leverage
// row norms of config 2 (128-column tiles, triangular B, row-norm epilogue).
//
// Why: the smem-operand kernel above is bound by shared-memory bandwidth, not
// by HBM or the tensor pipe (ncu, config-3 pass: LSU shared wavefronts 60 % of
// peak with half of them arbitration conflicts against the TMA writes and the
// UMMA operand reads; 241 KB of shared-memory traffic per 128 x 64 k-block =
// ~1.9 k cycles at 128 B/clk against a 912-cycle MMA floor). Here the
// converters write the bf16 hi/lo pieces of A straight into TMEM
// (tcgen05.st), so the per-k-block shared-memory traffic drops to the TMA
// write + one LSU read of the fp32 tile and the B pieces (161 KB): no bf16 A
// images in shared memory and no UMMA A-operand reads from it. The raw fp32
// ring is decoupled from the MMA: a stage is free as soon as its rows sit in
// converter registers, so RA tiles of A stay in flight per SM.
//
// TMEM (512 columns): X0 | X1 (fp32 partial sums, BN columns each, double
// buffered by 512-k chunk) | TA stages of the A pieces (32 columns hi + 32
// columns lo per 64-k block, bf16 pairs per column, lane = tile row). The
// promoted accumulator Y lives in the registers of eight epilogue warps
// (lane quarter x column half), added in the same order as the kernel above.
//   warps 0-7  : converters, two groups alternating k-blocks (thread = tile row)
//   warps 8-15 : epilogue
//   warp 16    : MMA issuer; warp 17: TMA issuer of the A boxes; warp 18: bulk copies of the B images
constexpr int TS_RA = 3, TS_RB = 3;
constexpr int TS_EPI_WARP0 = 8, TS_MMA_WARP = 16, TS_TMA_WARP = 17, TS_THREADS = 32 * 19;

__device__ __forceinline__ void mma_bf16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t* v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(taddr));
}

// y[0 .. CH) += TMEM columns taddr .. taddr + CH of this thread's lane (8 columns per load:
// the accumulator already takes most of the 96 registers a thread of this kernel has)
template <int CH>
__device__ __forceinline__ void tmem_add_cols(uint32_t taddr, float* y) {
  static_assert(CH % 8 == 0, "column halves come in multiples of 8");
#pragma unroll
  for (int c0 = 0; c0 < CH; c0 += 8) {
    uint32_t x[8];
    tmem_ld8(taddr + (uint32_t)c0, x);
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
    for (int j = 0; j < 8; ++j) y[c0 + j] += __uint_as_float(x[j]);
  }
}

// Epilogue of one warp: columns [C0, C0 + CW) of its 32 lanes. Chunk partial sums X[c & 1] are
// added into registers in chunk order, then the tile rows are stored.
template <int BN, int C0, int CW>
__device__ __forceinline__ void ts_epilogue(uint32_t tl, int c0, int nchunks, uint64_t* xfull, uint64_t* xfree, int64_t row,
                                            int64_t M, int64_t N, int64_t n0, double alpha, double beta, float* C,
                                            int64_t c_rs, int64_t c_cs, float* wsz, double* rn) {
  float y[CW];
#pragma unroll
  for (int j = 0; j < CW; ++j) y[j] = 0.f;
  for (int c = c0; c < c0 + nchunks; ++c) {
    const int xb = c & 1;
    mbar_wait(smem_u32(&xfull[xb]), (uint32_t)((c / 2) & 1));
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    tmem_add_cols<CW>(tl + (uint32_t)(xb * BN + C0), y);
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    mbar_arrive(smem_u32(&xfree[xb]));
  }
  if (row >= M) return;
  if (rn) {  // row-norm mode: sum of squares of this half tile's columns, C not written
    double rsq = 0.0;
#pragma unroll
    for (int j = 0; j < CW; ++j)
      if (n0 + C0 + j < N) {
        const double v = alpha * (double)y[j];
        rsq += v * v;
      }
    rn[row] = rsq;
    return;
  }
#pragma unroll
  for (int j = 0; j < CW; ++j) {
    const int64_t col = n0 + C0 + j;
    if (col < N) {
      if (wsz) {
        wsz[row * N + col] = y[j];
      } else {
        float* cp = C + row * c_rs + col * c_cs;
        *cp = beta == 0.0 ? (float)(alpha * y[j]) : (float)(alpha * y[j] + beta * *cp);
      }
    }
  }
}

template <bool A_KC, int BN>
__global__ void __launch_bounds__(TS_THREADS, 1)
    gemm_bf16x3_ts_kernel(int64_t M, int64_t N, int64_t K, int64_t kchunk, const uint8_t* __restrict__ bimg,
                          int64_t nkb_total, double alpha, double beta, float* C, int64_t c_rs, int64_t c_cs, float* ws,
                          const __grid_constant__ CUtensorMap amap, int mtiles, int nblk, int total_work, int flags,
                          double* rownorm) {
  static_assert(TC_BK == 64, "the TMEM A stages hold 64-k blocks");
  static_assert(BN % 8 == 0 && BN <= 160, "two fp32 partial buffers + A stages must fit 512 TMEM columns");
  constexpr int PKB = TC_PROMOTE_KB;
  constexpr int A_RAW = TC_BM * TC_BK * 4;  // fp32 tile landed by TMA
  constexpr int B_TILE = BN * ROWB;
  constexpr int B_STAGE = 2 * B_TILE;       // hi | lo images
  constexpr int TA = (512 - 2 * BN) / 64 > 4 ? 4 : (512 - 2 * BN) / 64;
  static_assert(TA >= 2, "at least two TMEM A stages");
  // accumulator columns per epilogue warp: halves [0, CH) and [CH, BN), both starting on
  // an 8-column boundary
  constexpr int CH = (BN / 2 + 7) / 8 * 8;
  constexpr uint32_t COL_A = 2 * BN;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* araw = smem;                      // [TS_RA][A_RAW]
  uint8_t* bring = smem + TS_RA * A_RAW;     // [TS_RB][B_STAGE]
  uint64_t* bars = reinterpret_cast<uint64_t*>(bring + TS_RB * B_STAGE);
  uint64_t* a_full = bars;
  uint64_t* a_empty = a_full + TS_RA;
  uint64_t* b_full = a_empty + TS_RA;
  uint64_t* b_empty = b_full + TS_RB;
  uint64_t* t_full = b_empty + TS_RB;
  uint64_t* t_empty = t_full + TA;
  uint64_t* xfull = t_empty + TA;
  uint64_t* xfree = xfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(xfree + 2);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // Work item w = (split z, N tile, M tile), M tile fastest: the CTAs of the
  // grid walk w = blockIdx.x, + gridDim.x, ... so at any time they share one
  // k range of B through L2. All roles run the same list; ring stages and
  // mbarrier phases follow the running k-block count g and chunk count cg.
  // Triangular B (flags bit 1: B(p, j) = 0 for p > j, the leverage product
  // M R^-1): N tile j needs k < (j + 1) BN only, so a CTA takes the tiles in
  // pairs (j, nblk - 1 - j) of equal total length, the pairs of one M tile on
  // neighbouring CTAs (its A rows are shared through L2).
  struct Work {
    int64_t m0, n0, kbeg;
    int nt, z, nkb;
  };
  const bool tri = (flags & 2) != 0, pairs = tri && nblk % 2 == 0;
  auto item = [&](int t, Work& k) -> bool {
    int mt;
    if (pairs) {
      const int pw = (int)blockIdx.x + (t >> 1) * (int)gridDim.x, hp = nblk / 2;
      if (pw >= total_work / 2) return false;
      mt = pw / hp;
      const int pp = pw - mt * hp;
      k.nt = (t & 1) ? nblk - 1 - pp : pp;
      k.z = 0;
    } else {
      const int w = (int)blockIdx.x + t * (int)gridDim.x;
      if (w >= total_work) return false;
      const int per = mtiles * nblk;
      k.z = w / per;
      const int rem = w - k.z * per;
      k.nt = rem / mtiles;
      mt = rem - k.nt * mtiles;
    }
    k.m0 = (int64_t)mt * TC_BM;
    k.n0 = (int64_t)k.nt * BN;
    k.kbeg = (int64_t)k.z * kchunk;
    int64_t kend = min(K, k.kbeg + kchunk);
    if (tri) kend = min(kend, k.n0 + BN);
    k.nkb = kend > k.kbeg ? (int)((kend - k.kbeg + TC_BK - 1) / TC_BK) : 0;
    return true;
  };

  if (tid == 0) {
    for (int s = 0; s < TS_RA; ++s) {
      mbar_init(smem_u32(&a_full[s]), 1);
      mbar_init(smem_u32(&a_empty[s]), TC_GROUP);
    }
    for (int s = 0; s < TS_RB; ++s) {
      mbar_init(smem_u32(&b_full[s]), 1);
      mbar_init(smem_u32(&b_empty[s]), 1);
    }
    for (int s = 0; s < TA; ++s) {
      mbar_init(smem_u32(&t_full[s]), TC_GROUP);
      mbar_init(smem_u32(&t_empty[s]), 1);
    }
    mbar_init(smem_u32(&xfull[0]), 1);
    mbar_init(smem_u32(&xfull[1]), 1);
    mbar_init(smem_u32(&xfree[0]), 256);
    mbar_init(smem_u32(&xfree[1]), 256);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == TS_EPI_WARP0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = *tmem_slot;

  if (warp < TS_EPI_WARP0) {
    // ---------------- converters: thread = tile row (TMEM lane), group = k-block parity ----------------
    const int grp = warp >> 2, r = (warp & 3) * 32 + lane;
    const uint32_t tl = tmem + ((uint32_t)((warp & 3) * 32) << 16) + COL_A;
    int g0 = 0;
    Work wk;
    for (int t = 0; item(t, wk); ++t) {
      for (int kb = (g0 + grp) & 1; kb < wk.nkb; kb += 2) {
        const int g = g0 + kb;
        const int sa = g % TS_RA, ta = g % TA;
        // The ring stages are shared by the two groups (g - RA belongs to the
        // other group), so a parity wait could alias a phase two steps back:
        // first make sure the previous use of the stage was consumed (then
        // a_full is in, or past, the phase of g).
        if (g >= TS_RA) mbar_wait(smem_u32(&a_empty[sa]), (uint32_t)(((g / TS_RA) - 1) & 1));
        mbar_wait(smem_u32(&a_full[sa]), (uint32_t)((g / TS_RA) & 1));
        const uint8_t* base = araw + sa * A_RAW;
        float f[64];
        if (A_KC) {  // two SWIZZLE_128B boxes of 32 k: row r at r * 128, 16-B granule gr at (gr ^ (r & 7)) * 16
#pragma unroll
          for (int b = 0; b < 2; ++b)
#pragma unroll
            for (int gr = 0; gr < 8; ++gr) {
              const float4 v =
                  *reinterpret_cast<const float4*>(base + b * (TC_BM * 128) + r * 128 + ((gr ^ (r & 7)) << 4));
              f[32 * b + 4 * gr] = v.x; f[32 * b + 4 * gr + 1] = v.y; f[32 * b + 4 * gr + 2] = v.z;
              f[32 * b + 4 * gr + 3] = v.w;
            }
        } else {  // [64 k][128 rows]
          const float* t = reinterpret_cast<const float*>(base);
#pragma unroll
          for (int k = 0; k < 64; ++k) f[k] = t[k * TC_BM + r];
        }
        // split before releasing the raw stage: the arrive below then depends on
        // every loaded value (an arrive right after the loads let the TMA refill
        // the stage under loads still in flight: nondeterministic rows)
        uint32_t hi[32], lo[32];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          uint4 a, b;
          split8(f + 8 * u, a, b);
          hi[4 * u] = a.x; hi[4 * u + 1] = a.y; hi[4 * u + 2] = a.z; hi[4 * u + 3] = a.w;
          lo[4 * u] = b.x; lo[4 * u + 1] = b.y; lo[4 * u + 2] = b.z; lo[4 * u + 3] = b.w;
        }
        {
          uint32_t dep = 0;
#pragma unroll
          for (int u = 0; u < 32; ++u) dep |= lo[u];
          asm volatile("" ::"r"(dep) : "memory");  // all splits done (hence all loads returned)
        }
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        mbar_arrive(smem_u32(&a_empty[sa]));
        if (g >= TA) {  // same for the TMEM stage: g - TA written by the other group, then read by its MMAs
          mbar_wait(smem_u32(&t_full[ta]), (uint32_t)(((g / TA) - 1) & 1));
          mbar_wait(smem_u32(&t_empty[ta]), (uint32_t)(((g / TA) - 1) & 1));
        }
        asm volatile("tcgen05.fence::after_thread_sync;\n");
#pragma unroll
        for (int h = 0; h < 2; ++h) {  // 32 k -> 16 columns of hi and of lo
          tmem_st16(tl + (uint32_t)(ta * 64 + 16 * h), hi + 16 * h);
          tmem_st16(tl + (uint32_t)(ta * 64 + 32 + 16 * h), lo + 16 * h);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;\n");
        mbar_arrive(smem_u32(&t_full[ta]));
      }
      g0 += wk.nkb;
    }
  } else if (warp == TS_TMA_WARP) {
    if (lane == 0) {  // A: fp32 boxes into the raw ring
      int g0 = 0;
      Work wk;
      for (int t = 0; item(t, wk); ++t) {
        for (int kb = 0; kb < wk.nkb; ++kb) {
          const int g = g0 + kb, sa = g % TS_RA;
          if (g >= TS_RA) mbar_wait(smem_u32(&a_empty[sa]), (uint32_t)(((g / TS_RA) - 1) & 1));
          const uint32_t bar = smem_u32(&a_full[sa]);
          mbar_arrive_expect_tx(bar, (uint32_t)A_RAW);
          const int k0 = (int)(wk.kbeg + (int64_t)kb * TC_BK);
          uint8_t* base = araw + sa * A_RAW;
          if (A_KC) {
#pragma unroll
            for (int b = 0; b < 2; ++b)
              tma_load_2d_g2s(smem_u32(base + b * TC_BM * 128), &amap, k0 + 32 * b, (int)wk.m0, bar);
          } else {
            tma_load_2d_g2s(smem_u32(base), &amap, (int)wk.m0, k0, bar);
          }
        }
        g0 += wk.nkb;
      }
    }
  } else if (warp == TS_TMA_WARP + 1) {
    if (lane == 0) {  // B: pre-split hi/lo images
      int g0 = 0;
      Work wk;
      for (int t = 0; item(t, wk); ++t) {
        const uint8_t* bsrc = bimg + ((int64_t)wk.nt * nkb_total + wk.kbeg / TC_BK) * (int64_t)B_STAGE;
        for (int kb = 0; kb < wk.nkb; ++kb) {
          const int g = g0 + kb, sb = g % TS_RB;
          if (g >= TS_RB) mbar_wait(smem_u32(&b_empty[sb]), (uint32_t)(((g / TS_RB) - 1) & 1));
          const uint32_t bar = smem_u32(&b_full[sb]);
          mbar_arrive_expect_tx(bar, (uint32_t)B_STAGE);
          bulk_copy_g2s(smem_u32(bring + sb * B_STAGE), bsrc + (int64_t)kb * B_STAGE, B_STAGE, bar);
        }
        g0 += wk.nkb;
      }
    }
    __syncwarp();
  } else if (warp == TS_MMA_WARP) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_bf16_f32(BN);
      int g0 = 0, c0 = 0;
      Work wk;
      for (int t = 0; item(t, wk); ++t) {
        for (int kb = 0; kb < wk.nkb; ++kb) {
          const int g = g0 + kb, sb = g % TS_RB, ta = g % TA;
          const int cg = c0 + kb / PKB, xb = cg & 1, kin = kb % PKB;
          if (kin == 0 && cg >= 2) mbar_wait(smem_u32(&xfree[xb]), (uint32_t)(((cg / 2) - 1) & 1));
          mbar_wait(smem_u32(&b_full[sb]), (uint32_t)((g / TS_RB) & 1));
          mbar_wait(smem_u32(&t_full[ta]), (uint32_t)((g / TA) & 1));
          asm volatile("tcgen05.fence::after_thread_sync;\n");
          const uint32_t dst = tmem + (uint32_t)(xb * BN);
          const uint32_t acol = tmem + COL_A + (uint32_t)(ta * 64);
          const uint32_t bbase = smem_u32(bring + sb * B_STAGE);
          constexpr int PI[3] = {0, 0, 1}, PJ[3] = {0, 1, 0};  // hi*hi, hi*lo, lo*hi
#pragma unroll
          for (int kk = 0; kk < TC_BK / 16; ++kk) {
#pragma unroll
            for (int p = 0; p < 3; ++p) {
              const uint32_t acc = (p > 0 || kin > 0 || kk > 0) ? 1u : 0u;
              mma_bf16_ts(dst, acol + (uint32_t)(PI[p] * 32 + kk * 8),
                          kmajor_sw128_desc(bbase + PJ[p] * B_TILE + kk * 32), idesc, acc);
            }
          }
          mma_commit(smem_u32(&t_empty[ta]));
          mma_commit(smem_u32(&b_empty[sb]));
          if (kin == PKB - 1 || kb == wk.nkb - 1) mma_commit(smem_u32(&xfull[xb]));
        }
        g0 += wk.nkb;
        c0 += (wk.nkb + PKB - 1) / PKB;
      }
      // drain: the commits to t_empty / b_empty of the last k-blocks must have
      // arrived before the CTA exits
      for (int g = max(0, g0 - TA); g < g0; ++g) mbar_wait(smem_u32(&t_empty[g % TA]), (uint32_t)((g / TA) & 1));
      for (int g = max(0, g0 - TS_RB); g < g0; ++g)
        mbar_wait(smem_u32(&b_empty[g % TS_RB]), (uint32_t)((g / TS_RB) & 1));
    }
    __syncwarp();
  } else if (warp < TS_MMA_WARP) {
    // ---------------- epilogue: Y in registers, lane quarter x column half ----------------
    const int quarter = warp & 3;
    const uint32_t tl = tmem + ((uint32_t)(quarter * 32) << 16);
    int c0 = 0;
    Work wk;
    for (int t = 0; item(t, wk); ++t) {
      const int64_t row = wk.m0 + quarter * 32 + lane;
      const int nchunks = (wk.nkb + PKB - 1) / PKB;
      float* wsz = ws ? ws + (int64_t)wk.z * M * N : nullptr;
      // row norms: [2 nt + column half][row]
      double* rn0 = rownorm ? rownorm + (int64_t)(2 * wk.nt) * M : nullptr;
      if (warp - TS_EPI_WARP0 < 4)
        ts_epilogue<BN, 0, CH>(tl, c0, nchunks, xfull, xfree, row, M, N, wk.n0, alpha, beta, C, c_rs, c_cs, wsz, rn0);
      else
        ts_epilogue<BN, CH, BN - CH>(tl, c0, nchunks, xfull, xfree, row, M, N, wk.n0, alpha, beta, C, c_rs, c_cs, wsz,
                                     rn0 ? rn0 + M : nullptr);
      c0 += nchunks;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == TS_EPI_WARP0) {
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512));
  }
}

template <bool A_KC, int BN>
void launch_tc_ts(rnla_ctx* ctx, int64_t m, int64_t n, int64_t k, int64_t kchunk, int splits, const float* B,
                  int64_t b_rs, int64_t b_cs, double alpha, double beta, float* C, int64_t c_rs, int64_t c_cs, float* ws,
                  const CUtensorMap* amap, int flags = 0, double* rownorm = nullptr) {
  const int64_t nkb = std::max<int64_t>(1, (k + TC_BK - 1) / TC_BK), nblk = (n + BN - 1) / BN;
  DevBuf img(2 * (size_t)BN * ROWB * (size_t)(nkb * nblk), ctx->stream);
  split_b_image<2><<<grid_for(ctx, nblk * nkb * BN * QPR, 256), 256, 0, ctx->stream>>>(k, n, B, b_rs, b_cs, BN, nkb,
                                                                                       nblk, img.as<uint8_t>());
  RNLA_CUDA(cudaGetLastError());
  note_launch(ctx);
  const size_t smem = (size_t)TS_RA * TC_BM * TC_BK * 4 + (size_t)TS_RB * 2 * BN * ROWB + 1024 + 8 * 32 + 16;
  auto kern = gemm_bf16x3_ts_kernel<A_KC, BN>;
  ensure_dyn_smem((const void*)kern, smem);
  const int64_t mtiles = (m + TC_BM - 1) / TC_BM, total = mtiles * nblk * splits;
  const bool pairs = (flags & 2) && nblk % 2 == 0;
  const int grid = (int)std::min<int64_t>(pairs ? total / 2 : total, ctx->num_sms);
  kern<<<grid, TS_THREADS, smem, ctx->stream>>>(m, n, k, kchunk, img.as<uint8_t>(), nkb, alpha, beta, C, c_rs, c_cs, ws,
                                                *amap, (int)mtiles, (int)nblk, (int)total, flags, rownorm);
  RNLA_CUDA(cudaGetLastError());
  note_launch(ctx);
}

// Row norms of A B, B upper triangular, on the A-in-TMEM kernel (128-column
// tiles, two partial sums per tile): the leverage-score product of config 2.
bool ts_rownorm_eligible(int64_t m, int64_t n, int64_t k) {
  static const bool no_ts = std::getenv("RNLA_TC_NO_TS") != nullptr;
  return !no_ts && n > 160 && k >= 1 && ((m + TC_BM - 1) / TC_BM) * ((n + 127) / 128) < ((int64_t)1 << 30);
}

template <bool A_KC, int BN, int STAGES, bool DF, bool TMA_A>
void launch_tc(rnla_ctx* ctx, int64_t m, int64_t n, int64_t k, int64_t kchunk, int splits, const float* A,
               int64_t a_rs, int64_t a_cs, const float* B, int64_t b_rs, int64_t b_cs, double alpha, double beta,
               typename std::conditional<DF, double, float>::type* C, int64_t c_rs, int64_t c_cs,
               typename std::conditional<DF, double, float>::type* ws, int sym, const CUtensorMap* amap,
               double* rownorm) {
  constexpr int NS = DF ? RNLA_TC_DF_NS : 2;
  constexpr size_t STAGE = NS * (TC_BM * ROWB + BN * ROWB);
  const int64_t nkb = std::max<int64_t>(1, (k + TC_BK - 1) / TC_BK), nblk = (n + BN - 1) / BN;
  DevBuf img;
  if (!(sym & 8)) {  // B pre-split into bf16 images (a Gram with B = A' splits its B tiles in the kernel)
    img = DevBuf(NS * (size_t)BN * ROWB * (size_t)(nkb * nblk), ctx->stream);
    split_b_image<NS><<<grid_for(ctx, nblk * nkb * BN * QPR, 256), 256, 0, ctx->stream>>>(k, n, B, b_rs, b_cs, BN,
                                                                                         nkb, nblk, img.as<uint8_t>());
    RNLA_CUDA(cudaGetLastError());
    note_launch(ctx);
  }
  const size_t smem = STAGES * STAGE + 1024 + 8 * (3 * STAGES + 5);
  auto kern = gemm_bf16x3_kernel<A_KC, BN, STAGES, DF, TMA_A>;
  ensure_dyn_smem((const void*)kern, smem);
  const bool nfast = nblk > 1 && (m + TC_BM - 1) / TC_BM <= 65535;
  if (nfast) sym |= 16;
  dim3 grid(nfast ? (unsigned)nblk : (unsigned)((m + TC_BM - 1) / TC_BM),
            nfast ? (unsigned)((m + TC_BM - 1) / TC_BM) : (unsigned)nblk, (unsigned)splits);
  CUtensorMap dummy{};
  kern<<<grid, TMA_A ? TC_THREADS + 32 : TC_THREADS, smem, ctx->stream>>>(
      m, n, k, kchunk, A, a_rs, a_cs, img.as<uint8_t>(), nkb, alpha, beta, C, c_rs, c_cs, ws, sym,
      amap ? *amap : dummy, rownorm);
  RNLA_CUDA(cudaGetLastError());
  note_launch(ctx);
}

template <bool A_KC, int BN, int CH>
void launch_tc_persist(rnla_ctx* ctx, int64_t m, int64_t n, int64_t k, const float* A, const float* B, int64_t b_rs,
                       int64_t b_cs, double alpha, double beta, float* C, int64_t c_rs, int64_t c_cs, int sym,
                       const CUtensorMap* amap, double* rownorm) {
  constexpr int NS = 2;
  constexpr size_t STAGE = NS * (TC_BM * ROWB + BN * ROWB);
  constexpr int STAGES = std::min<int>(TC_STAGES_MAX, (int)((220 * 1024) / STAGE));
  const int64_t nkb = std::max<int64_t>(1, (k + TC_BK - 1) / TC_BK), nblk = (n + BN - 1) / BN;
  DevBuf img(NS * (size_t)BN * ROWB * (size_t)(nkb * nblk), ctx->stream);
  split_b_image<NS><<<grid_for(ctx, nblk * nkb * BN * QPR, 256), 256, 0, ctx->stream>>>(k, n, B, b_rs, b_cs, BN, nkb,
                                                                                       nblk, img.as<uint8_t>());
  RNLA_CUDA(cudaGetLastError());
  note_launch(ctx);
  const size_t smem = STAGES * STAGE + 1024 + 8 * (3 * STAGES + 4) + 16;
  auto kern = gemm_bf16x3_persist<A_KC, BN, STAGES, CH>;
  ensure_dyn_smem((const void*)kern, smem);
  const int ntm = (int)((m + TC_BM - 1) / TC_BM), ntn = (int)nblk;
  const int grid = (int)std::min<int64_t>((int64_t)ntm * ntn, ctx->num_sms);
  kern<<<grid, TC_THREADS + 32, smem, ctx->stream>>>(m, n, k, A, img.as<uint8_t>(), nkb, alpha, beta, C, c_rs, c_cs,
                                                      sym, *amap, rownorm, ntm, ntn);
  RNLA_CUDA(cudaGetLastError());
  note_launch(ctx);
}

// Short-K products without split-K on the persistent kernel; false when the
// shape does not qualify (the one-tile kernel runs).
template <bool A_KC>
bool try_tc_persist(rnla_ctx* ctx, int bn, int64_t m, int64_t n, int64_t k, const float* A, const float* B,
                    int64_t b_rs, int64_t b_cs, double alpha, double beta, float* C, int64_t c_rs, int64_t c_cs,
                    int sym, const CUtensorMap* amap, double* rownorm) {
  const int64_t nkb = (k + TC_BK - 1) / TC_BK;
  if (k < 1 || nkb > 2 * TC_PROMOTE_KB || !amap) return false;
  const int64_t tiles = ((m + TC_BM - 1) / TC_BM) * ((n + bn - 1) / bn);
  if (tiles < 2 * (int64_t)ctx->num_sms) return false;
  const bool one = nkb <= TC_PROMOTE_KB;
#define RNLA_P(BNV, CHV) \
  launch_tc_persist<A_KC, BNV, CHV>(ctx, m, n, k, A, B, b_rs, b_cs, alpha, beta, C, c_rs, c_cs, sym, amap, rownorm)
  if (bn <= 32) RNLA_P(32, 2);
  else if (bn <= 64) RNLA_P(64, 2);
  else if (bn <= 96) RNLA_P(96, 2);
  else if (bn <= 128) RNLA_P(128, 2);
  else if (one && bn <= 152) RNLA_P(152, 1);
  else if (one && bn <= 160) RNLA_P(160, 1);
  else return false;
#undef RNLA_P
  return true;
}

template <bool A_KC, bool DF>
void dispatch_bn(rnla_ctx* ctx, int bn, int64_t m, int64_t n, int64_t k, int64_t kchunk, int splits, const float* A,
                 int64_t a_rs, int64_t a_cs, const float* B, int64_t b_rs, int64_t b_cs, double alpha, double beta,
                 typename std::conditional<DF, double, float>::type* C, int64_t c_rs, int64_t c_cs,
                 typename std::conditional<DF, double, float>::type* ws, int sym, const CUtensorMap* amap,
                 double* rownorm) {
  // as many stages as fit in ~220 KB of shared memory (at most TC_STAGES_MAX)
#define RNLA_ST(BNV) \
  std::min(TC_STAGES_MAX, (220 * 1024) / ((DF ? RNLA_TC_DF_NS : 2) * (TC_BM * ROWB + (BNV) * ROWB)))
#define RNLA_TC(BNV)                                                                                           \
  do {                                                                                                         \
    if (amap)                                                                                                  \
      launch_tc<A_KC, BNV, RNLA_ST(BNV), DF, true>(ctx, m, n, k, kchunk, splits, A, a_rs, a_cs, B, b_rs, b_cs, \
                                                   alpha, beta, C, c_rs, c_cs, ws, sym, amap, rownorm);        \
    else                                                                                                       \
      launch_tc<A_KC, BNV, RNLA_ST(BNV), DF, false>(ctx, m, n, k, kchunk, splits, A, a_rs, a_cs, B, b_rs,      \
                                                    b_cs, alpha, beta, C, c_rs, c_cs, ws, sym, nullptr,        \
                                                    rownorm);                                                  \
  } while (0)
  if constexpr (!DF) {
    // plain products with one wide N tile: the A-in-TMEM kernel (see above)
    static const bool no_ts = std::getenv("RNLA_TC_NO_TS") != nullptr;
    // (128 < N <= 160 always; 32 < N <= 128 for long K, where the A path is the bound)
    if (!no_ts && amap && sym == 0 && !rownorm && (bn > 128 || (bn > 32 && k > 2 * TC_PROMOTE_KB * TC_BK)) &&
        ((m + TC_BM - 1) / TC_BM) * ((n + bn - 1) / bn) * splits < ((int64_t)1 << 30)) {
      if (bn <= 64)
        launch_tc_ts<A_KC, 64>(ctx, m, n, k, kchunk, splits, B, b_rs, b_cs, alpha, beta, C, c_rs, c_cs, ws, amap);
      else if (bn <= 96)
        launch_tc_ts<A_KC, 96>(ctx, m, n, k, kchunk, splits, B, b_rs, b_cs, alpha, beta, C, c_rs, c_cs, ws, amap);
      else if (bn <= 128)
        launch_tc_ts<A_KC, 128>(ctx, m, n, k, kchunk, splits, B, b_rs, b_cs, alpha, beta, C, c_rs, c_cs, ws, amap);
      else if (bn <= 152)
        launch_tc_ts<A_KC, 152>(ctx, m, n, k, kchunk, splits, B, b_rs, b_cs, alpha, beta, C, c_rs, c_cs, ws, amap);
      else
        launch_tc_ts<A_KC, 160>(ctx, m, n, k, kchunk, splits, B, b_rs, b_cs, alpha, beta, C, c_rs, c_cs, ws, amap);
      return;
    }
  }
  if (bn <= 32) RNLA_TC(32);
  else if (bn <= 64) RNLA_TC(64);
  else if (bn <= 96) RNLA_TC(96);
  else if (DF || bn <= 128) RNLA_TC(128);
  else if constexpr (!DF) {
    if (bn <= 152) RNLA_TC(152);
    else RNLA_TC(160);
  }
#undef RNLA_TC
#undef RNLA_ST
}

template <class OutT>
__global__ void splitk_reduce_tc(int64_t m, int64_t n, int splits, const OutT* __restrict__ ws, double alpha,
                                 double beta, OutT* C, int64_t c_rs, int64_t c_cs) {
  const int64_t total = m * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    OutT s = ws[e];
    for (int z = 1; z < splits; ++z) s += ws[(int64_t)z * total + e];
    const int64_t i = e / n, j = e % n;
    OutT* cp = C + i * c_rs + j * c_cs;
    *cp = beta == 0.0 ? (OutT)(alpha * s) : (OutT)(alpha * s + beta * *cp);
  }
}

// TMA map of the fp32 A operand for the TMA-fed kernel, or false when the
// layout does not allow it (then the register-staged loader runs).
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

bool make_a_map(CUtensorMap* map, const float* A, int64_t m, int64_t k, int64_t a_rs, int64_t a_cs) {
  // Default on (RNLA_TC_NO_TMA=1 falls back to the register-staged loader):
  // config 3 37.5 vs 38.8 ms once the converter's 8-lane phases read one chunk
  // of 8 consecutive rows (conflict-free SW128 reads and writes).
  static const bool off = std::getenv("RNLA_TC_NO_TMA") != nullptr;
  if (off || !encode_tiled() || (reinterpret_cast<uintptr_t>(A) & 15) || m >= INT32_MAX || k >= INT32_MAX) return false;
  const cuuint32_t es[2] = {1, 1};
  CUresult r;
  if (a_cs == 1 && a_rs > 0 && (a_rs * 4) % 16 == 0) {  // K-contiguous: dims {k, m}, boxes {32 k, 128 rows}, SW128
    const cuuint64_t dims[2] = {(cuuint64_t)k, (cuuint64_t)m};
    const cuuint64_t strides[1] = {(cuuint64_t)a_rs * 4};
    const cuuint32_t box[2] = {32, (cuuint32_t)TC_BM};
    r = encode_tiled()(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(A), dims, strides, box, es,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else if (a_rs == 1 && a_cs > 0 && (a_cs * 4) % 16 == 0) {  // MN-contiguous: dims {m, k}, box {128 rows, 64 k}
    const cuuint64_t dims[2] = {(cuuint64_t)m, (cuuint64_t)k};
    const cuuint64_t strides[1] = {(cuuint64_t)a_cs * 4};
    const cuuint32_t box[2] = {(cuuint32_t)TC_BM, (cuuint32_t)TC_BK};
    r = encode_tiled()(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(A), dims, strides, box, es,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {
    return false;
  }
  return r == CUDA_SUCCESS;
}

// C(i, j) = C(j, i) for the tiles a symmetric launch skipped.
template <class OutT>
__global__ void mirror_skipped_tiles(int64_t n, int bm, int bn, OutT* C, int64_t c_rs, int64_t c_cs) {
  const int64_t total = n * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / n, j = e % n;
    if ((i / bm) * bm >= (j / bn + 1) * bn) C[i * c_rs + j * c_cs] = C[j * c_rs + i * c_cs];
  }
}

template <bool DF>
void gemm_tc_impl(rnla_ctx* ctx, int64_t m, int64_t n, int64_t k, double alpha, const float* A, int64_t a_rs,
                  int64_t a_cs, const float* B, int64_t b_rs, int64_t b_cs, double beta,
                  typename std::conditional<DF, double, float>::type* C, int64_t c_rs, int64_t c_cs,
                  bool tri_b = false, double* rownorm = nullptr, int* rownorm_parts = nullptr) {
  using OutT = typename std::conditional<DF, double, float>::type;
  if (m == 0 || n == 0) return;
  // one N tile up to 160 columns (3 fp32 accumulators fit TMEM; 128 with the
  // 4 of the double-float mode), else 128-column tiles
  const int cap = DF ? 128 : 160;
  // N granularity 8 above 128 columns (kind::f16, M = 128, cta_group::1): the
  // s = 150 products of config 3 run N = 152 instead of 160 (5 % fewer MMAs)
  const int bn_full = n <= cap ? (int)(n > 128 ? ((n + 7) / 8) * 8 : ((n + 15) / 16) * 16) : 128;
  // Gram products (B = A') are symmetric: upper tiles only, then mirror; the
  // split-K sizing below counts only the tiles that run.
  const int sym = (A == B && m == n && a_rs == b_cs && a_cs == b_rs && !std::getenv("RNLA_TC_NO_SYM")) ? 1 : 0;
  const int bn_eff = bn_full <= 32 ? 32 : bn_full <= 64 ? 64 : bn_full <= 96 ? 96 : (DF || bn_full <= 128) ? 128
                    : bn_full <= 152 ? 152 : 160;
  const int64_t mtiles = (m + TC_BM - 1) / TC_BM, ntiles_eff = (n + bn_eff - 1) / bn_eff;
  int64_t tiles = mtiles * ntiles_eff;
  if (sym) {
    tiles = 0;
    for (int64_t mt = 0; mt < mtiles; ++mt)
      for (int64_t nt = 0; nt < ntiles_eff; ++nt) tiles += (mt * TC_BM < (nt + 1) * bn_eff) ? 1 : 0;
  }
  // Split K so that the CTAs fill whole waves of the 148 SMs (one CTA per SM):
  // the smallest split count reaching >= 97 % wave efficiency among those that
  // give every SM a tile, each split keeping >= 4 k-blocks and the fp32/fp64
  // workspace <= 512 MB. (Measured: A'Q at 16384 x 150, K = 262144 ran 256
  // CTAs = 1.73 waves.)
  int64_t splits = 1;
  if (DF && tiles <= 8) {
    // small double-float Grams keep the one-tile-per-SM rule: short K ranges
    // per CTA accumulate in TMEM for only a few k-blocks, and the partials are
    // summed in fp64 (row-leverage sums stay within ~1e-7)
    if (tiles < ctx->num_sms && k >= 2 * TC_BK)
      splits = std::min<int64_t>((ctx->num_sms + tiles - 1) / tiles, k / TC_BK);
  } else if (k >= 2 * TC_BK) {
    const int64_t sms = ctx->num_sms;
    const int64_t ws_cap = ((int64_t)512 << 20) / std::max<int64_t>(1, m * n * (int64_t)sizeof(OutT));
    const int64_t smax = std::max<int64_t>(1, std::min<int64_t>(std::min<int64_t>(k / (4 * TC_BK), 256), ws_cap));
    double best = -1.0;
    for (int64_t s = 1; s <= smax; ++s) {
      const double w = (double)(tiles * s) / (double)sms;
      const double eff = w / std::ceil(w);
      if (eff > best + 1e-9) {
        best = eff;
        splits = s;
      }
      if (eff >= 0.97) break;
    }
  }
  if (tri_b || rownorm) splits = 1;  // clipped k ranges start at 0; row norms need whole sums
  int64_t kchunk = ((k + splits - 1) / splits + TC_BK - 1) / TC_BK * TC_BK;
  if (k == 0) kchunk = TC_BK;
  splits = std::max<int64_t>(1, (k + kchunk - 1) / kchunk);
  DevBuf wsb;
  OutT* ws = nullptr;
  if (splits > 1) {
    wsb = DevBuf(sizeof(OutT) * (size_t)(splits * m * n), ctx->stream);
    ws = wsb.as<OutT>();
  }
  CUtensorMap amap;
  const bool tma = make_a_map(&amap, A, m, k, a_rs, a_cs);
  // Gram via the TMA path with 128-wide tiles: B tiles come from the same
  // tensor map (the pre-split B image measured slower: 8.7 vs 8.1 ms).
  const bool b_from_a = sym && tma && bn_full == TC_BM;
  const int flags = sym | (tri_b && !sym ? 2 : 0) | (b_from_a ? 8 : 0);
  if constexpr (!DF) {
    if (rownorm && tri_b && !sym && tma && splits == 1 && ts_rownorm_eligible(m, n, k)) {
      if (a_cs == 1)
        launch_tc_ts<true, 128>(ctx, m, n, k, kchunk, 1, B, b_rs, b_cs, alpha, 0.0, nullptr, 0, 0, nullptr, &amap, 2,
                                rownorm);
      else
        launch_tc_ts<false, 128>(ctx, m, n, k, kchunk, 1, B, b_rs, b_cs, alpha, 0.0, nullptr, 0, 0, nullptr, &amap, 2,
                                 rownorm);
      if (rownorm_parts) *rownorm_parts = 2 * (int)((n + 127) / 128);  // two column halves per 128-column tile
      return;
    }
    static const bool no_persist = std::getenv("RNLA_TC_NO_PERSIST") != nullptr;
    if (!no_persist && tma && splits == 1 && !sym) {
      const bool ok = a_cs == 1 ? try_tc_persist<true>(ctx, bn_eff, m, n, k, A, B, b_rs, b_cs, alpha, beta, C, c_rs,
                                                       c_cs, flags, &amap, rownorm)
                                : try_tc_persist<false>(ctx, bn_eff, m, n, k, A, B, b_rs, b_cs, alpha, beta, C, c_rs,
                                                        c_cs, flags, &amap, rownorm);
      if (ok) return;
    }
  }
  if (a_cs == 1)
    dispatch_bn<true, DF>(ctx, bn_full, m, n, k, kchunk, (int)splits, A, a_rs, a_cs, B, b_rs, b_cs, alpha, beta, C,
                          c_rs, c_cs, ws, flags, tma ? &amap : nullptr, rownorm);
  else
    dispatch_bn<false, DF>(ctx, bn_full, m, n, k, kchunk, (int)splits, A, a_rs, a_cs, B, b_rs, b_cs, alpha, beta, C,
                           c_rs, c_cs, ws, flags, tma ? &amap : nullptr, rownorm);
  if (splits > 1) {
    splitk_reduce_tc<OutT><<<grid_for(ctx, m * n, 256), 256, 0, ctx->stream>>>(m, n, (int)splits, ws, alpha, beta, C,
                                                                               c_rs, c_cs);
    RNLA_CUDA(cudaGetLastError());
    note_launch(ctx);
  }
  if (sym && !rownorm) {
    mirror_skipped_tiles<OutT><<<grid_for(ctx, m * n, 256), 256, 0, ctx->stream>>>(m, TC_BM, bn_eff, C, c_rs, c_cs);
    RNLA_CUDA(cudaGetLastError());
    note_launch(ctx);
  }

}

}  // namespace

bool tc_gemm_enabled() {
  static const bool on = std::getenv("RNLA_DISABLE_TCGEN05") == nullptr;
  return on;
}

// C[m x n] = alpha * A[m x k] * B[k x n] + beta * C on tcgen05 (BF16x3).
void gemm_f32_tc(rnla_ctx* ctx, int64_t m, int64_t n, int64_t k, float alpha, const float* A, int64_t a_rs,
                 int64_t a_cs, const float* B, int64_t b_rs, int64_t b_cs, float beta, float* C, int64_t c_rs,
                 int64_t c_cs) {
  gemm_tc_impl<false>(ctx, m, n, k, alpha, A, a_rs, a_cs, B, b_rs, b_cs, beta, C, c_rs, c_cs);
}

// Same with B upper triangular (B(p, j) = 0 for p > j): each N tile stops at
// k = its last column, skipping the zero blocks.
void gemm_f32_tc_tri_b(rnla_ctx* ctx, int64_t m, int64_t n, int64_t k, float alpha, const float* A, int64_t a_rs,
                       int64_t a_cs, const float* B, int64_t b_rs, int64_t b_cs, float beta, float* C, int64_t c_rs,
                       int64_t c_cs) {
  gemm_tc_impl<false>(ctx, m, n, k, alpha, A, a_rs, a_cs, B, b_rs, b_cs, beta, C, c_rs, c_cs, true);
}

// Row norms of C = A B with B upper triangular, C never stored:
// rownorm[t * m + i] = sum over the columns of N tile t of (alpha C(i, j))^2,
// t < ntiles (returned). The caller adds the tiles in order.
int gemm_f32_tc_tri_b_rownorm(rnla_ctx* ctx, int64_t m, int64_t n, int64_t k, float alpha, const float* A,
                              int64_t a_rs, int64_t a_cs, const float* B, int64_t b_rs, int64_t b_cs, double* rownorm) {
  int parts = 0;  // set by the A-in-TMEM path (two partial sums per tile)
  gemm_tc_impl<false>(ctx, m, n, k, alpha, A, a_rs, a_cs, B, b_rs, b_cs, 0.f, nullptr, 0, 0, true, rownorm, &parts);
  if (parts > 0) return parts;
  const int bn = n <= 160 ? (int)(n > 128 ? ((n + 7) / 8) * 8 : ((n + 15) / 16) * 16) : 128;
  const int bn_eff = bn <= 32 ? 32 : bn <= 64 ? 64 : bn <= 96 ? 96 : bn <= 128 ? 128 : bn <= 152 ? 152 : 160;
  return (int)((n + bn_eff - 1) / bn_eff);
}

// Same with double-float accumulation across 256-row chunks and fp64 output.
void gemm_f32_tc_f64acc(rnla_ctx* ctx, int64_t m, int64_t n, int64_t k, double alpha, const float* A, int64_t a_rs,
                        int64_t a_cs, const float* B, int64_t b_rs, int64_t b_cs, double beta, double* C,
                        int64_t c_rs, int64_t c_cs) {
  gemm_tc_impl<true>(ctx, m, n, k, alpha, A, a_rs, a_cs, B, b_rs, b_cs, beta, C, c_rs, c_cs);
}

}  // namespace rnla
