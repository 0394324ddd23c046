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
// The fp32 data is read through registers because it has to be split before
// the MMA anyway (a TMA copy would add an smem round trip).
#include <cuda_bf16.h>

#include "rnla_internal.h"
#include "util.cuh"

namespace rnla {

namespace {

constexpr int TC_BM = 128, TC_BK = 64, TC_STAGES_MAX = 4;
constexpr int TC_PRODUCERS = 256;  // warps 0-7
constexpr int TC_GROUP = 128;      // producer group (4 warps) per k-block
constexpr int TC_MMA_WARP = 12;    // warps 8-11 run the epilogue
constexpr int TC_THREADS = 416;

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

// Shared-memory matrix descriptor, K-major SWIZZLE_128B: rows of 128 B,
// 8-row atoms of 1024 B (SBO), LBO unused (1), version 1 (sm_100).
__device__ __forceinline__ uint64_t kmajor_sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;            // LBO (ignored for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;  // SBO: next 8-row group
  d |= (uint64_t)1 << 46;            // version = 1
  d |= (uint64_t)2 << 61;            // SWIZZLE_128B
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

constexpr int TC_PROMOTE_KB = 8;  // k-blocks (x64 k) per TMEM partial sum

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
  if (KCONTIG) {  // 8 lanes cover one row's 64 k: 256 B contiguous
    r = u >> 3;
    q = u & 7;
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

// All loads of the tile are issued before any conversion (R*8/256 units per
// thread in flight), then each unit is split and stored.
// NS pieces go to tiles base, base + R*128, base + 2*R*128.
template <bool KCONTIG, int R, int NT, int NS>
__device__ __forceinline__ void load_split_tile(const float* __restrict__ X, int64_t rs, int64_t ks, int64_t rows,
                                                int64_t r0, int64_t k0, int64_t kend, uint8_t* base, int tid) {
  constexpr int UNITS = R * 8;  // (row, 8-k chunk)
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
      const uint32_t off = (uint32_t)r * 128u + (uint32_t)((q ^ (r & 7)) << 4);
#pragma unroll
      for (int p = 0; p < NS; ++p) *reinterpret_cast<uint4*>(base + p * (R * 128) + off) = pc[p];
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
  const int64_t total = nblk * nkb * BN * 8;
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < total; u += (int64_t)gridDim.x * blockDim.x) {
    const int q = (int)(u & 7);
    const int64_t rest0 = u >> 3;
    const int j = (int)(rest0 % BN);
    const int64_t rest = rest0 / BN;
    const int64_t kb = rest % nkb, nb = rest / nkb;
    const int64_t gj = nb * BN + j, gk = kb * TC_BK + 8 * q;
    float f[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) f[t] = (gj < N && gk + t < K) ? B[(gk + t) * b_rs + gj * b_cs] : 0.f;
    uint4 pc[NS];
    split8n<NS>(f, pc);
    uint8_t* tile = img + (nb * nkb + kb) * (int64_t)(NS * BN * 128);
    const uint32_t off = (uint32_t)j * 128u + (uint32_t)((q ^ (j & 7)) << 4);
#pragma unroll
    for (int p = 0; p < NS; ++p) *reinterpret_cast<uint4*>(tile + p * BN * 128 + off) = pc[p];
  }
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}\n" ::"r"(bar),
               "r"(bytes)
               : "memory");
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
template <bool A_KC, int BN, int STAGES, bool DF>
__global__ void __launch_bounds__(TC_THREADS, 1)
    gemm_bf16x3_kernel(int64_t M, int64_t N, int64_t K, int64_t kchunk, const float* __restrict__ A, int64_t a_rs,
                       int64_t a_cs, const uint8_t* __restrict__ bimg, int64_t nkb_total, double alpha,
                       double beta, typename std::conditional<DF, double, float>::type* C, int64_t c_rs, int64_t c_cs,
                       typename std::conditional<DF, double, float>::type* ws) {
  using OutT = typename std::conditional<DF, double, float>::type;
  constexpr int PKB = DF ? 4 : TC_PROMOTE_KB;
  // DF also splits three ways (BF16x6: hh, hm, mh, hl, lh, mm ~ fp32-faithful
  // products, 1.9e-7 rel-F per SURVEY §7 hard part 5); otherwise BF16x3.
  constexpr int NS = DF ? 3 : 2;
  constexpr int A_TILE = TC_BM * 128;  // bytes per bf16 tile (128 rows x 64 k)
  constexpr int B_TILE = BN * 128;
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
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  // full[S], empty[S], xfull[2], xfree[2]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 4);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t m0 = (int64_t)blockIdx.x * TC_BM, n0 = (int64_t)blockIdx.y * BN;
  const int64_t kbeg = (int64_t)blockIdx.z * kchunk, kend = min(K, kbeg + kchunk);
  const int nkb = (int)((kend - kbeg + TC_BK - 1) / TC_BK);

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(smem_u32(&bars[s]), TC_GROUP + 1);  // a producer group + the bulk-copy expect_tx arrive
      mbar_init(smem_u32(&bars[STAGES + s]), 1);
    }
    mbar_init(smem_u32(&bars[2 * STAGES]), 1);      // xfull[0]
    mbar_init(smem_u32(&bars[2 * STAGES + 1]), 1);  // xfull[1]
    mbar_init(smem_u32(&bars[2 * STAGES + 2]), 128);  // xfree[0] (epilogue threads)
    mbar_init(smem_u32(&bars[2 * STAGES + 3]), 128);  // xfree[1]
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 8) {  // TMEM accumulator: 128 lanes x TMEM_COLS fp32 columns
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = *tmem_slot;

  if (warp < 8) {
    // ---------------- producers: two groups of 4 warps take alternate k-blocks,
    // so two k-blocks of A loads are in flight per SM ----------------
    const int grp = warp >> 2, gtid = tid & (TC_GROUP - 1);
    const int64_t kb0 = kbeg / TC_BK;
    const uint8_t* bsrc = bimg + ((int64_t)blockIdx.y * nkb_total + kb0) * (int64_t)(NS * B_TILE);
    for (int kb = grp; kb < nkb; kb += 2) {
      const int st = kb % STAGES;
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
          const uint32_t a0 = base, b0 = base + NS * A_TILE;
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
      if (row < M) {
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
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 8) {
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(TMEM_COLS));
  }
}

template <bool A_KC, int BN, int STAGES, bool DF>
void launch_tc(rnla_ctx* ctx, int64_t m, int64_t n, int64_t k, int64_t kchunk, int splits, const float* A,
               int64_t a_rs, int64_t a_cs, const float* B, int64_t b_rs, int64_t b_cs, double alpha, double beta,
               typename std::conditional<DF, double, float>::type* C, int64_t c_rs, int64_t c_cs,
               typename std::conditional<DF, double, float>::type* ws) {
  constexpr int NS = DF ? 3 : 2;
  constexpr size_t STAGE = NS * (TC_BM * 128 + BN * 128);
  const int64_t nkb = std::max<int64_t>(1, (k + TC_BK - 1) / TC_BK), nblk = (n + BN - 1) / BN;
  DevBuf img(NS * (size_t)BN * 128 * (size_t)(nkb * nblk), ctx->stream);
  split_b_image<NS><<<grid_for(ctx, nblk * nkb * BN * 8, 256), 256, 0, ctx->stream>>>(k, n, B, b_rs, b_cs, BN, nkb,
                                                                                       nblk, img.as<uint8_t>());
  RNLA_CUDA(cudaGetLastError());
  note_launch(ctx);
  const size_t smem = STAGES * STAGE + 1024 + 8 * (2 * STAGES + 5);
  auto kern = gemm_bf16x3_kernel<A_KC, BN, STAGES, DF>;
  RNLA_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dim3 grid((unsigned)((m + TC_BM - 1) / TC_BM), (unsigned)nblk, (unsigned)splits);
  kern<<<grid, TC_THREADS, smem, ctx->stream>>>(m, n, k, kchunk, A, a_rs, a_cs, img.as<uint8_t>(), nkb, alpha, beta,
                                                 C, c_rs, c_cs, ws);
  RNLA_CUDA(cudaGetLastError());
  note_launch(ctx);
}

template <bool A_KC, bool DF>
void dispatch_bn(rnla_ctx* ctx, int bn, int64_t m, int64_t n, int64_t k, int64_t kchunk, int splits, const float* A,
                 int64_t a_rs, int64_t a_cs, const float* B, int64_t b_rs, int64_t b_cs, double alpha, double beta,
                 typename std::conditional<DF, double, float>::type* C, int64_t c_rs, int64_t c_cs,
                 typename std::conditional<DF, double, float>::type* ws) {
  // as many stages as fit in ~220 KB of shared memory (at most 4)
#define RNLA_ST(BNV) \
  std::min(4, (220 * 1024) / ((DF ? 3 : 2) * (TC_BM * 128 + (BNV) * 128)))
#define RNLA_TC(BNV) \
  launch_tc<A_KC, BNV, RNLA_ST(BNV), DF>(ctx, m, n, k, kchunk, splits, A, a_rs, a_cs, B, b_rs, b_cs, alpha, beta, C, \
                                         c_rs, c_cs, ws)
  if (bn <= 32) RNLA_TC(32);
  else if (bn <= 64) RNLA_TC(64);
  else if (bn <= 96) RNLA_TC(96);
  else if (DF || bn <= 128) RNLA_TC(128);
  else if constexpr (!DF) RNLA_TC(160);
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

template <bool DF>
void gemm_tc_impl(rnla_ctx* ctx, int64_t m, int64_t n, int64_t k, double alpha, const float* A, int64_t a_rs,
                  int64_t a_cs, const float* B, int64_t b_rs, int64_t b_cs, double beta,
                  typename std::conditional<DF, double, float>::type* C, int64_t c_rs, int64_t c_cs) {
  using OutT = typename std::conditional<DF, double, float>::type;
  if (m == 0 || n == 0) return;
  // one N tile up to 160 columns (3 fp32 accumulators fit TMEM; 128 with the
  // 4 of the double-float mode), else 128-column tiles
  const int cap = DF ? 128 : 160;
  const int bn_full = n <= cap ? (int)(((n + 15) / 16) * 16) : 128;
  const int64_t ntiles = (n + bn_full - 1) / bn_full;
  const int64_t tiles = ((m + TC_BM - 1) / TC_BM) * ntiles;
  // split K until every SM has a tile (K ranges stay multiples of 64)
  int64_t splits = 1;
  if (tiles < ctx->num_sms && k >= 2 * TC_BK)
    splits = std::min<int64_t>((ctx->num_sms + tiles - 1) / tiles, k / TC_BK);
  int64_t kchunk = ((k + splits - 1) / splits + TC_BK - 1) / TC_BK * TC_BK;
  if (k == 0) kchunk = TC_BK;
  splits = std::max<int64_t>(1, (k + kchunk - 1) / kchunk);
  DevBuf wsb;
  OutT* ws = nullptr;
  if (splits > 1) {
    wsb = DevBuf(sizeof(OutT) * (size_t)(splits * m * n), ctx->stream);
    ws = wsb.as<OutT>();
  }
  if (a_cs == 1)
    dispatch_bn<true, DF>(ctx, bn_full, m, n, k, kchunk, (int)splits, A, a_rs, a_cs, B, b_rs, b_cs, alpha, beta, C,
                          c_rs, c_cs, ws);
  else
    dispatch_bn<false, DF>(ctx, bn_full, m, n, k, kchunk, (int)splits, A, a_rs, a_cs, B, b_rs, b_cs, alpha, beta, C,
                           c_rs, c_cs, ws);
  if (splits > 1) {
    splitk_reduce_tc<OutT><<<grid_for(ctx, m * n, 256), 256, 0, ctx->stream>>>(m, n, (int)splits, ws, alpha, beta, C,
                                                                               c_rs, c_cs);
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

// Same with double-float accumulation across 256-row chunks and fp64 output.
void gemm_f32_tc_f64acc(rnla_ctx* ctx, int64_t m, int64_t n, int64_t k, double alpha, const float* A, int64_t a_rs,
                        int64_t a_cs, const float* B, int64_t b_rs, int64_t b_cs, double beta, double* C,
                        int64_t c_rs, int64_t c_cs) {
  gemm_tc_impl<true>(ctx, m, n, k, alpha, A, a_rs, a_cs, B, b_rs, b_cs, beta, C, c_rs, c_cs);
}

}  // namespace rnla
