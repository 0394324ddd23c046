// srht_acc.cu -- one-pass fp32 SRHT: every sampled output is accumulated on
// chip, so A is read from HBM exactly once and nothing of size n is written.
//
// Reference: srht_sketch / fwht_inplace (/root/reference/proj/src/sketch.cpp:44-81):
//   out[t][c] = (1/sqrt(s)) * sum_j (-1)^popcount(idx_t & j) * sign_j * A[j][c].
// With j = 4096*jh + jl and idx_t = 4096*th + tl (Sylvester order):
//   out[t] = (1/sqrt s) * sum_jh (-1)^popcount(th & jh) * Y_jh[tl],
//   Y_jh   = H_4096 (sign . A[4096 jh .. 4096 jh + 4095])       (one tile)
// so each 4096-row tile needs only its own 12-bit transform, and every one of
// the s <= 4096 sampled outputs receives one signed add per tile.
//
// Work: a CTA owns an 8-column slice (one 32-B sector per row) and a run of
// consecutive tiles. The tile lives in registers (512 threads x 64 values):
//   phase 1: thread (g, c) takes rows g + 64e (e < 64) from the TMA ring as
//            the chunks land, sign flip, 6 register stages over e (bits 6-11);
//   phase 2: through a swizzled smem tile, thread (a, c) takes rows 64a + b,
//            6 register stages over b (bits 0-5), Y written back in place;
//   gather : thread t owns samples 8t .. 8t+7 (all 8 columns = 64 fp32) whose
//            running sums live in TMEM (tcgen05.ld / tcgen05.st, 256 columns)
//            and adds (-1)^popcount(th & jh) * Y[tl] from smem.
// Four consecutive CTAs take the four 8-column slices of one 128-B line over
// the same tile run, so each line is fetched from HBM once. A run that crosses
// a slice boundary flushes its sums to a partial buffer; a small finalize
// kernel adds the (<= 3) partials of each slice in a fixed order and scales.
// The stage order differs from the reference loop, so results agree to fp32
// rounding (gate 1e-4 rel-F), not bitwise; the fp64 path stays bit-exact.
#include <cuda.h>

#include "rnla_internal.h"
#include "srht.h"
#include "util.cuh"

namespace rnla {

namespace {

constexpr int LO = 12, ROWS = 1 << LO;  // rows per tile
#ifndef RNLA_SRHT_ACC_CH
#define RNLA_SRHT_ACC_CH 512
#endif
constexpr int CH = RNLA_SRHT_ACC_CH;     // rows per chunk (256-row TMA boxes)
constexpr int NCH = ROWS / CH;           // 8 chunks per tile
constexpr int EPC = CH / 64;             // values per thread per chunk
constexpr int RING = (96 * 1024) / (CH * 32);  // chunk slots: 96 KB (3/4 of a tile) in flight
constexpr int SMAX = 4096;               // sampled outputs held on chip
static_assert((NCH & (NCH - 1)) == 0 && CH % 256 == 0, "power-of-two chunks per tile, whole TMA boxes");

// W fp32 columns per CTA (W = 8: one 32-B sector per row, 512 threads, one CTA
// per SM; W = 4: 16-B rows, 256 threads, two CTAs per SM).
template <int W>
struct Cfg {
  static constexpr int NT = 64 * W;           // 64 row groups x W columns
  static constexpr int GS = 32 / W;           // CTAs (slices) per 128-B line; also the swizzle span
  static constexpr int TMEM_COLS = 32 * W;    // 128 lanes x 32W fp32 = 4096 samples x W columns
  static constexpr int SPT = 64 / W;          // samples per thread in the gather
  static constexpr size_t RING_BYTES = (size_t)RING * CH * W * 4;
  static constexpr size_t TILE_BYTES = (size_t)ROWS * W * 4;
  static constexpr size_t SMEM_BYTES = RING_BYTES + TILE_BYTES + 2 * RING * 8 + 16;
};

struct AccArgs {
  const unsigned long long* mask;  // [JH][64]: bit e of (jh, g) = sign of row 4096 jh + g + 64 e is -1
  const uint32_t* samp;            // [SMAX]: tl | th << 12
  float* part;                     // [KQ * segmax][GS][SMAX][W] running sums per (run segment, slice)
  int64_t qt;                      // line-tiles = Q * JH (Q = 32-column lines of GS slices)
  int jh_count, jh_log, kq, segmax;
};

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint32_t bar, uint32_t bytes) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}\n" ::"r"(bar),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "W_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra W_%=;\n\t}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ bool mbar_test(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}\n"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          dst),
      "l"(map), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t* u = reinterpret_cast<uint32_t*>(v);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]), "=r"(u[7]), "=r"(u[8]),
        "=r"(u[9]), "=r"(u[10]), "=r"(u[11]), "=r"(u[12]), "=r"(u[13]), "=r"(u[14]), "=r"(u[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float* v) {
  const uint32_t* u = reinterpret_cast<const uint32_t*>(v);
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n" ::"r"(
          taddr),
      "r"(u[0]), "r"(u[1]), "r"(u[2]), "r"(u[3]), "r"(u[4]), "r"(u[5]), "r"(u[6]), "r"(u[7]), "r"(u[8]), "r"(u[9]),
      "r"(u[10]), "r"(u[11]), "r"(u[12]), "r"(u[13]), "r"(u[14]), "r"(u[15])
      : "memory");
}

// Physical row of tile row r: the low two bits are XORed with bits 6-7, so the
// four row groups a warp touches in phase 2 (rows 64a + b, a = 4w..4w+3) sit in
// different 8-bank groups; phase 1 (rows g + 64e) stays conflict-free too.
// Physical row of tile row r: r XOR ((r >> 6) mod GS), so the GS row groups a
// warp touches in phase 2 (rows 64a + b) sit in different bank groups while
// phase 1 (rows g + 64e) stays conflict-free. For W = 8, column c of physical
// row p sits at p * 8 + (c ^ (p & 4)): the two 16-B halves of a row swap when
// bit 2 of p is set, so the gather's 16-B loads spread over all eight 4-bank
// groups.
template <int GS>
__host__ __device__ __forceinline__ int swz(int r) { return r ^ ((r >> 6) & (GS - 1)); }

// 64-point butterflies on values held as 32 float2 pairs (v[i] = values 2i, 2i+1):
// stage h = 1 pairs the two halves of one float2 (scalar adds), stages h >= 2
// pair whole float2s, so they run as packed FADD2 (add.rn.f32x2; the
// subtraction is x + (-1) * y with one rounding, i.e. exactly x - y).
__device__ __forceinline__ void butterfly64(float2* v) {
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const float x = v[i].x, y = v[i].y;
    v[i] = make_float2(x + y, x - y);
  }
  const float2 m1 = make_float2(-1.f, -1.f);
#pragma unroll
  for (int h = 1; h < 32; h <<= 1)
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (!(i & h)) {
        const float2 x = v[i], y = v[i + h];
        v[i] = __fadd2_rn(x, y);
        v[i + h] = __ffma2_rn(y, m1, x);
      }
}
__device__ __forceinline__ float& vat(float2* v, int e) { return (e & 1) ? v[e >> 1].y : v[e >> 1].x; }

template <int W>
__global__ void __launch_bounds__(Cfg<W>::NT, 8 / W) srht_acc_kernel(const __grid_constant__ CUtensorMap amap, AccArgs a) {
  using C = Cfg<W>;
  constexpr int NT = C::NT, GS = C::GS, TMEM_COLS = C::TMEM_COLS, SPT = C::SPT;
  constexpr size_t RING_BYTES = C::RING_BYTES, TILE_BYTES = C::TILE_BYTES;
  extern __shared__ __align__(1024) unsigned char smem[];
  float* ring = reinterpret_cast<float*>(smem);               // [RING][CH][W]
  float* tile = reinterpret_cast<float*>(smem + RING_BYTES);  // [ROWS][W], swizzled rows
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + RING_BYTES + TILE_BYTES);  // full[RING], empty[RING]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * RING);
  int& nissue_s = *reinterpret_cast<int*>(tmem_slot + 1);  // producer's next chunk

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = tid / W, c = tid % W;  // phase 1: row group g; phase 2: row group a = g
  const int kq = blockIdx.x / GS, r = blockIdx.x % GS;
  const int64_t start = (int64_t)kq * a.qt / a.kq, end = (int64_t)(kq + 1) * a.qt / a.kq;
  const int ntiles = (int)(end - start);
  const int jhn = a.jh_count;
  const int q_first = (int)(start / jhn);
  const int total_chunks = ntiles * NCH;

  if (tid == 0) {
    for (int i = 0; i < RING; ++i) {
      mbar_init(su32(&bars[i]), 1);              // full: one expect_tx arrival + the bytes
      mbar_init(su32(&bars[RING + i]), NT / 32);  // empty: one arrival per warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = *tmem_slot;
  // this warp's TMEM window: lanes 32 (warp % 4) .., columns 64 (warp / 4) .. (64 per thread)
  const uint32_t taddr = tmem + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(64 * (warp >> 2));

  const int qt0 = (int)start;  // quad-tile indices fit in int (Q * JH <= 2^30 checked on the host)
  // Producer (thread 0): chunk N lands in slot N % RING once chunk N - RING has
  // been read by every warp. During phase 1 it keeps chunks up to G + RING - 2
  // issued (G = the chunk just read; the wait is for G - 2, normally long
  // done); after barrier A every chunk of the tile is read, so it tops the ring
  // up to RING chunks for phase 2 and the gather. Its counter lives in smem.
  auto issue = [&](int N) {
    const int slot = N % RING;
    const int qti = qt0 + N / NCH, kk = N & (NCH - 1);
    const int q = qti >> a.jh_log, jh = qti & (jhn - 1);
    mbar_expect(su32(&bars[slot]), CH * W * 4);
#pragma unroll
    for (int b = 0; b < CH / 256; ++b)
      tma_load_2d(su32(ring + ((size_t)slot * CH + b * 256) * W), &amap, (GS * q + r) * W, jh * ROWS + kk * CH + b * 256,
                  su32(&bars[slot]));
  };
  if (tid == 0) {
    int N = 0;
    for (; N < RING && N < total_chunks; ++N) issue(N);
    nissue_s = N;
  }

  int cslot = 0;
  uint32_t cpar = 0;
  unsigned long long msk = ntiles > 0 ? a.mask[(size_t)(qt0 & (jhn - 1)) * 64 + g] : 0ull;
  float2 v[32];
  for (int i = 0; i < ntiles; ++i) {
    const int qti = qt0 + i;
    const int q = qti >> a.jh_log, jh = qti & (jhn - 1);
    const bool first = (i == 0) || jh == 0, last = (i == ntiles - 1) || jh == jhn - 1;
    const unsigned long long msk_next = i + 1 < ntiles ? a.mask[(size_t)((qti + 1) & (jhn - 1)) * 64 + g] : 0ull;

    // ---- phase 1: rows g + 64e as the chunks land (chunk kk holds e = EPC kk .. EPC kk + EPC - 1) ----
#pragma unroll
    for (int kk = 0; kk < NCH; ++kk) {
      mbar_wait(su32(&bars[cslot]), cpar);
      const float* src = ring + (size_t)cslot * CH * W;
#pragma unroll
      for (int j = 0; j < EPC; ++j) {
        const int e = EPC * kk + j;
        const uint32_t bits = __float_as_uint(src[(g + 64 * j) * W + c]);
        vat(v, e) = __uint_as_float(bits ^ ((uint32_t)(msk >> e) << 31));
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(su32(&bars[RING + cslot]));
      if (tid == 0) {
        const int G = i * NCH + kk, N = nissue_s;
        if (N <= G + RING - 2 && N < total_chunks) {
          const int P = N - RING;  // previous occupant of N's slot, <= G - 2
          mbar_wait(su32(&bars[RING + P % RING]), (uint32_t)((P / RING) & 1));
          issue(N);
          nissue_s = N + 1;
        }
      }
      if (++cslot == RING) {
        cslot = 0;
        cpar ^= 1u;
      }
    }
    msk = msk_next;
    butterfly64(v);
    __syncthreads();  // A: the previous tile's gather has finished reading `tile`; all chunks read
    if (tid == 0) {
      int N = nissue_s;
      for (const int lim = min(total_chunks, (i + 1) * NCH + RING); N < lim; ++N) issue(N);
      nissue_s = N;
    }
#pragma unroll
    for (int e = 0; e < 64; ++e) tile[(64 * e + (g ^ (e & (GS - 1)))) * W + (W == 8 ? (c ^ (g & 4)) : c)] = vat(v, e);
    __syncthreads();  // B
    // ---- phase 2: rows 64a + b (a = g), written back in place ----
#pragma unroll
    for (int b = 0; b < 64; ++b) vat(v, b) = tile[(64 * g + (b ^ (g & (GS - 1)))) * W + (W == 8 ? (c ^ (b & 4)) : c)];
    butterfly64(v);
#pragma unroll
    for (int b = 0; b < 64; ++b) tile[(64 * g + (b ^ (g & (GS - 1)))) * W + (W == 8 ? (c ^ (b & 4)) : c)] = vat(v, b);

    // ---- gather: samples SPT tid .. SPT tid + SPT - 1, all W columns ----
    float acc[64];
    uint4 wv[SPT / 4];
#pragma unroll
    for (int m = 0; m < SPT / 4; ++m) wv[m] = __ldg(reinterpret_cast<const uint4*>(a.samp) + (SPT / 4) * tid + m);
    __syncthreads();  // D: Y complete
    if (first) {
#pragma unroll
      for (int e = 0; e < 64; ++e) acc[e] = 0.f;
    } else {
#pragma unroll
      for (int m = 0; m < 4; ++m) tmem_ld16(taddr + 16 * m, acc + 16 * m);
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
    }
#pragma unroll
    for (int k = 0; k < SPT; ++k) {
      const uint32_t wk = k % 4 == 0 ? wv[k / 4].x : k % 4 == 1 ? wv[k / 4].y : k % 4 == 2 ? wv[k / 4].z : wv[k / 4].w;
      const int p = swz<GS>((int)(wk & (ROWS - 1)));
      const float sg = (__popc((wk >> LO) & (uint32_t)jh) & 1) ? -1.f : 1.f;
#pragma unroll
      for (int h = 0; h < W / 4; ++h) {
        const float4 y = *reinterpret_cast<const float4*>(tile + p * W + (W == 8 ? ((4 * h) ^ (p & 4)) : 0));
        float* o = acc + W * k + 4 * h;
        o[0] = fmaf(sg, y.x, o[0]);
        o[1] = fmaf(sg, y.y, o[1]);
        o[2] = fmaf(sg, y.z, o[2]);
        o[3] = fmaf(sg, y.w, o[3]);
      }
    }
    if (last) {
      const int seg = q - q_first;
      float4* dst = reinterpret_cast<float4*>(a.part + ((((size_t)kq * a.segmax + seg) * GS + r) * SMAX) * W +
                                              (size_t)64 * tid);
#pragma unroll
      for (int m = 0; m < 16; ++m) dst[m] = make_float4(acc[4 * m], acc[4 * m + 1], acc[4 * m + 2], acc[4 * m + 3]);
    } else {
#pragma unroll
      for (int m = 0; m < 4; ++m) tmem_st16(taddr + 16 * m, acc + 16 * m);
      asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(TMEM_COLS));
  }
}

// out[t][col] = scale * sum of the run partials of col's slice, in run order.
__global__ void srht_acc_finalize(const float* __restrict__ part, const int32_t* __restrict__ qtab,
                                  const int32_t* __restrict__ slot_of, int maxl, int W, int64_t s, int64_t L,
                                  float scale, float* __restrict__ out, int64_t out_rs, int64_t out_cs) {
  const int GS = 32 / W;
  const int64_t total = s * L;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = e / L, col = e - t * L;
    const int64_t q = col >> 5;
    const int r = (int)((col & 31) / W), c = (int)(col % W);
    const int64_t slot = slot_of[t];
    float acc = 0.f;
    for (int m = 0; m < maxl; ++m) {
      const int ent = qtab[q * maxl + m];
      if (ent < 0) break;
      acc += part[(((size_t)ent * GS + r) * SMAX + slot) * W + c];
    }
    out[t * out_rs + col * out_cs] = acc * scale;
  }
}

// mask[jh][g] bit e = (row 4096 jh + g + 64 e < n and its sign is -1).
__global__ void srht_acc_masks(const int8_t* __restrict__ signs, int64_t n, int64_t jh_count,
                               unsigned long long* __restrict__ mask) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= jh_count * 64) return;
  const int64_t jh = i >> 6, g = i & 63;
  unsigned long long m = 0;
  for (int e = 0; e < 64; ++e) {
    const int64_t row = jh * ROWS + g + 64 * e;
    if (row < n && signs[row] < 0) m |= 1ull << e;
  }
  mask[i] = m;
}

}  // namespace

namespace {

template <int W>
void srht_acc_launch(rnla_ctx* ctx, const SrhtPlan& plan, const float* in, int64_t ld, int64_t L, float* out,
                     int64_t out_rs, int64_t out_cs, int64_t jh_count, int64_t qt) {
  using C = Cfg<W>;
  // Runs: KQ groups of GS CTAs (the slices of one 128-B line) split the Q * JH
  // line-tiles evenly, q-major.
  const int64_t nquads = qt / jh_count;
  const int kq = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)ctx->num_sms * (8 / W) / C::GS, qt));
  // qtab[q][m] = index (run k, segment of the run) of the m-th partial of line q, -1 padded.
  int segmax = 1;
  std::vector<std::vector<std::pair<int, int>>> lists((size_t)nquads);
  for (int k = 0; k < kq; ++k) {
    const int64_t s0 = (int64_t)k * qt / kq, s1 = (int64_t)(k + 1) * qt / kq;
    if (s1 <= s0) continue;
    const int64_t qa = s0 / jh_count, qb = (s1 - 1) / jh_count;
    segmax = std::max(segmax, (int)(qb - qa + 1));
    for (int64_t qq = qa; qq <= qb; ++qq) lists[(size_t)qq].emplace_back(k, (int)(qq - qa));
  }
  int maxl = 1;
  for (auto& l : lists) maxl = std::max(maxl, (int)l.size());
  std::vector<int32_t> qtab((size_t)nquads * maxl, -1);
  for (int64_t qq = 0; qq < nquads; ++qq)
    for (size_t m = 0; m < lists[(size_t)qq].size(); ++m)
      qtab[(size_t)qq * maxl + m] = lists[(size_t)qq][m].first * segmax + lists[(size_t)qq][m].second;
  DevBuf dq(sizeof(int32_t) * qtab.size(), ctx->stream);
  RNLA_CUDA(cudaMemcpyAsync(dq.p, qtab.data(), sizeof(int32_t) * qtab.size(), cudaMemcpyHostToDevice, ctx->stream));
  DevBuf part(sizeof(float) * (size_t)kq * segmax * C::GS * SMAX * W, ctx->stream);

  CUtensorMap amap;
  tma_map_rows_f32(&amap, in, plan.n, L, ld, W, 256);
  int jh_log = 0;
  while (((int64_t)1 << jh_log) < jh_count) ++jh_log;
  AccArgs args{plan.acc_mask.as<unsigned long long>(), plan.acc_samp.as<uint32_t>(), part.as<float>(), qt,
               (int)jh_count, jh_log, kq, segmax};
  ensure_dyn_smem((const void*)srht_acc_kernel<W>, C::SMEM_BYTES);
  srht_acc_kernel<W><<<C::GS * kq, C::NT, C::SMEM_BYTES, ctx->stream>>>(amap, args);
  RNLA_CUDA(cudaGetLastError());
  const float scale = (float)(1.0 / std::sqrt((double)plan.s));
  srht_acc_finalize<<<grid_for(ctx, plan.s * L, 256), 256, 0, ctx->stream>>>(
      part.as<float>(), dq.as<int32_t>(), plan.acc_slot.as<int32_t>(), maxl, W, plan.s, L, scale, out, out_rs,
      out_cs);
  RNLA_CUDA(cudaGetLastError());
  note_launch(ctx, 2);
  // qtab was staged by the pageable cudaMemcpyAsync before it returned; the
  // device buffers are freed stream-ordered.
}

}  // namespace

bool srht_acc_f32(rnla_ctx* ctx, const SrhtPlan& plan, const float* in, int64_t ld, int64_t L, float* out,
                  int64_t out_rs, int64_t out_cs) {
  if (std::getenv("RNLA_SRHT_NO_ACC") || plan.q < LO || plan.s > SMAX || L < 1 || !tma_encode_available()) return false;
  if ((reinterpret_cast<uintptr_t>(in) & 15) || ((ld * 4) % 16) || plan.n > (int64_t)INT32_MAX) return false;
  if (plan.n < 1 || ctx->num_sms < 4) return false;
  const int64_t jh_count = plan.big_n >> LO;
  const int64_t qt = (L + 31) / 32 * jh_count;
  if (qt > (int64_t)1 << 30) return false;
  if (!plan.acc_mask.p) {
    plan.acc_mask = DevBuf(sizeof(unsigned long long) * (size_t)jh_count * 64, ctx->stream);
    srht_acc_masks<<<(unsigned)((jh_count * 64 + 255) / 256), 256, 0, ctx->stream>>>(
        plan.signs.as<int8_t>(), plan.n, jh_count, plan.acc_mask.as<unsigned long long>());
    RNLA_CUDA(cudaGetLastError());
    note_launch(ctx);
    // Sample -> accumulator slot. Slot 8 tid + k is read by lane tid % 32 at
    // gather step k as two 16-B loads of physical tile row p; a quarter warp
    // (8 lanes) is one smem wavefront when its 8 rows have distinct p mod 8
    // (the 16-B bank group). Samples are bucketed by p mod 8 and
    // each (warp, quarter, k) group takes one per bucket while buckets last.
    std::vector<uint32_t> sp(SMAX, 0u);
    std::vector<int32_t> slot_of((size_t)plan.s, 0);
    {
      constexpr int GS8 = Cfg<8>::GS;
      std::vector<std::vector<int>> bucket(8);
      for (int64_t t = plan.s - 1; t >= 0; --t) {
        const int64_t tl = plan.host_idx[(size_t)t] & (ROWS - 1);
        bucket[(size_t)(swz<GS8>((int)tl) & 7)].push_back((int)t);
      }
      const int nt = Cfg<8>::NT, spt = Cfg<8>::SPT;
      for (int w = 0; w < nt / 32; ++w)
        for (int qq = 0; qq < 4; ++qq)
          for (int k = 0; k < spt; ++k) {
            bool used[8] = {false, false, false, false, false, false, false, false};
            int lanes[8], nl = 0;
            auto place = [&](int lane8, int t) {
              const int slot = spt * (32 * w + 8 * qq + lane8) + k;
              const int64_t ix = plan.host_idx[(size_t)t];
              sp[(size_t)slot] = (uint32_t)(ix & (ROWS - 1)) | ((uint32_t)(ix >> LO) << LO);
              slot_of[(size_t)t] = slot;
            };
            for (int b = 0; b < 8; ++b)
              if (!bucket[(size_t)b].empty()) {
                place(nl, bucket[(size_t)b].back());
                bucket[(size_t)b].pop_back();
                used[b] = true;
                ++nl;
              }
            for (int l = nl; l < 8; ++l) lanes[l - nl] = l;
            for (int l = 0; l < 8 - nl; ++l) {  // fill from the fullest bucket, else an idle row of a free class
              int best = -1;
              for (int b = 0; b < 8; ++b)
                if (!bucket[(size_t)b].empty() && (best < 0 || bucket[(size_t)b].size() > bucket[(size_t)best].size()))
                  best = b;
              if (best >= 0) {
                place(lanes[l], bucket[(size_t)best].back());
                bucket[(size_t)best].pop_back();
              } else {
                int fc = 0;
                while (fc < 7 && used[fc]) ++fc;
                used[fc] = true;
                const int slot = spt * (32 * w + 8 * qq + lanes[l]) + k;
                sp[(size_t)slot] = (uint32_t)swz<GS8>(fc);  // tile row of class fc (swz is an involution on it)
              }
            }
          }
    }
    plan.acc_slot = DevBuf(sizeof(int32_t) * (size_t)plan.s, ctx->stream);
    RNLA_CUDA(cudaMemcpyAsync(plan.acc_slot.p, slot_of.data(), sizeof(int32_t) * (size_t)plan.s,
                              cudaMemcpyHostToDevice, ctx->stream));
    plan.acc_samp = DevBuf(sizeof(uint32_t) * SMAX, ctx->stream);
    RNLA_CUDA(cudaMemcpyAsync(plan.acc_samp.p, sp.data(), sizeof(uint32_t) * SMAX, cudaMemcpyHostToDevice,
                              ctx->stream));
    RNLA_CUDA(cudaStreamSynchronize(ctx->stream));  // sp goes out of scope
  }
  // 8-column slices, one CTA per SM (4-column slices with two CTAs per SM
  // measured slower: 1.77 vs 1.575 ms on config 2)
  srht_acc_launch<8>(ctx, plan, in, ld, L, out, out_rs, out_cs, jh_count, qt);
  return true;
}

}  // namespace rnla
