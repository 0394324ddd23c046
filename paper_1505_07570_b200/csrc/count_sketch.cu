// count_sketch.cu -- CountSketch as a bandwidth-bound bucket gather-reduce.
//
// Reference: count_sketch_stream / count_sketch_hash,
// /root/reference/proj/src/sketch.cpp:16-26 and :83-97:
//     C = 0; for j = 0..n-1: (b, g) = hash(seed, j, s); C.col(b) += g * col(j)
// One "segment" is one column of the reference's column-major operand, which
// is one row of a row-major tall matrix.
//
// B200 design:
//  1. plan (cached per (n, s, seed, j0)): the counter-based hash is evaluated
//     on the device from the GLOBAL segment index; a stable radix sort groups
//     segment ids by bucket, keeping them ascending inside each bucket.
//  2. gather-reduce: one team of threads per bucket streams its segments in
//     ascending j order (each a contiguous L-element run, read exactly once,
//     evict-first) and accumulates them in registers, then writes the bucket
//     once. Summation order per bucket equals the reference's, so fp64 output
//     is bit-identical to the single-threaded reference loop, and no atomics
//     are needed. U segments are loaded ahead of the adds to keep enough
//     bytes in flight per SM for HBM3e.
#include <cub/cub.cuh>

#include "rnla_internal.h"
#include "util.cuh"

namespace rnla {

namespace {

__device__ __forceinline__ uint64_t d_splitmix64(uint64_t& state) {
  uint64_t z = (state += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

constexpr uint32_t kNegBit = 0x80000000u;

// keys[j] = bucket, vals[j] = j | (sign < 0 ? kNegBit : 0); counts[bucket]++.
__global__ void cs_hash_kernel(uint64_t seed, int64_t j0, int64_t n, uint64_t s, uint64_t s_mask, uint32_t* keys,
                               uint32_t* vals, uint32_t* counts) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    uint64_t state = seed ^ (0xa0761d6478bd642fULL + (uint64_t)(j0 + j) * 0xe7037ed1a0b428dbULL);
    const uint64_t h1 = d_splitmix64(state);
    const uint64_t h2 = d_splitmix64(state);
    const uint32_t b = (uint32_t)(s_mask ? (h1 & s_mask) : (h1 % s));
    keys[j] = b;
    vals[j] = (uint32_t)j | ((h2 & 1ULL) ? 0u : kNegBit);
    atomicAdd(&counts[b], 1u);
  }
}

template <class T>
__device__ __forceinline__ T ld_stream(const T* p) {
  return __ldcs(p);  // read-once data: evict-first in L1/L2
}

// One team of TEAM threads per bucket; blockDim.x == 128 (128 / TEAM buckets per CTA).
// Thread t of a team owns segment offsets col0 + t + i*TEAM, i < CPT.
template <class T, int TEAM, int CPT, int U>
__global__ void __launch_bounds__(128) cs_gather_kernel(const T* __restrict__ in, int64_t ld,
                                                        const T* __restrict__ extra, int64_t extra_stride, int64_t L,
                                                        int64_t Lo, const uint32_t* __restrict__ offsets,
                                                        const uint32_t* __restrict__ rows, int64_t b0, int64_t s,
                                                        T* __restrict__ out, int64_t ldo, int accumulate) {
  constexpr int kTeams = 128 / TEAM;
  const int team = threadIdx.x / TEAM;
  const int t = threadIdx.x % TEAM;
  const int64_t b = b0 + (int64_t)blockIdx.x * kTeams + team;  // buckets [b0, s) of this launch
  if (b >= s) return;
  const int64_t col0 = (int64_t)blockIdx.y * (TEAM * CPT);

  int64_t col[CPT];
  bool live[CPT], isx[CPT];
#pragma unroll
  for (int i = 0; i < CPT; ++i) {
    col[i] = col0 + t + (int64_t)i * TEAM;
    live[i] = col[i] < Lo;
    isx[i] = col[i] >= L;  // the appended `extra` element
  }
  T acc[CPT];
  T* orow = out + b * ldo;
#pragma unroll
  for (int i = 0; i < CPT; ++i) acc[i] = (accumulate && live[i]) ? orow[col[i]] : T(0);

  const uint32_t beg = __ldg(offsets + b), end = __ldg(offsets + b + 1);
  for (uint32_t k = beg; k < end; k += U) {
    uint32_t e[U];
    T v[U][CPT];
#pragma unroll
    for (int u = 0; u < U; ++u) e[u] = (k + u < end) ? __ldg(rows + k + u) : 0xffffffffu;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool ok = e[u] != 0xffffffffu;
      const int64_t r = (int64_t)(e[u] & ~kNegBit);
      const T* seg = in + r * ld;
#pragma unroll
      for (int i = 0; i < CPT; ++i) {
        v[u][i] = T(0);
        if (ok && live[i]) v[u][i] = isx[i] ? ld_stream(extra + r * extra_stride) : ld_stream(seg + col[i]);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (e[u] == 0xffffffffu) break;
      const bool neg = (e[u] & kNegBit) != 0;
#pragma unroll
      for (int i = 0; i < CPT; ++i) acc[i] += neg ? -v[u][i] : v[u][i];  // == C.col(b) += g * col(j)
    }
  }
#pragma unroll
  for (int i = 0; i < CPT; ++i)
    if (live[i]) orow[col[i]] = acc[i];
}

template <class T, int TEAM, int CPT>
void launch_gather(rnla_ctx* ctx, const T* in, int64_t ld, const T* extra, int64_t xs, int64_t L, int64_t Lo,
                   const CountSketchPlan& plan, T* out, int64_t ldo, bool acc, int64_t b0, int64_t b1) {
  constexpr int U = (CPT <= 2) ? 8 : (CPT <= 4 ? 6 : 4);
  constexpr int kTeams = 128 / TEAM;
  if (b1 <= b0) return;
  dim3 grid((unsigned)((b1 - b0 + kTeams - 1) / kTeams), (unsigned)((Lo + TEAM * CPT - 1) / (TEAM * CPT)));
  cs_gather_kernel<T, TEAM, CPT, U><<<grid, 128, 0, ctx->stream>>>(
      in, ld, extra, xs, L, Lo, plan.offsets.as<uint32_t>(), plan.rows.as<uint32_t>(), b0, b1, out, ldo, acc ? 1 : 0);
  RNLA_CUDA(cudaGetLastError());
  note_launch(ctx);
}

}  // namespace

const CountSketchPlan& count_sketch_plan(rnla_ctx* ctx, int64_t n, int64_t s, uint64_t seed, int64_t j0) {
  require(n < (int64_t)kNegBit, "count_sketch: more than 2^31-1 segments in one plan");
  require(s >= 1 && s <= (int64_t)0xffffffffLL, "count_sketch: s out of range");
  auto key = std::make_tuple(n, s, j0, seed);
  auto it = ctx->cs_plans.find(key);
  if (it != ctx->cs_plans.end()) return *it->second;

  auto plan = std::make_unique<CountSketchPlan>();
  plan->n = n; plan->s = s; plan->seed = seed; plan->j0 = j0;
  cudaStream_t st = ctx->stream;
  plan->offsets = DevBuf(sizeof(uint32_t) * (size_t)(s + 1), st);
  plan->rows = DevBuf(sizeof(uint32_t) * (size_t)std::max<int64_t>(n, 1), st);
  RNLA_CUDA(cudaMemsetAsync(plan->offsets.p, 0, sizeof(uint32_t) * (size_t)(s + 1), st));
  if (n > 0) {
    DevBuf keys(sizeof(uint32_t) * n, st), keys_out(sizeof(uint32_t) * n, st), vals(sizeof(uint32_t) * n, st);
    DevBuf counts(sizeof(uint32_t) * (size_t)(s + 1), st);
    RNLA_CUDA(cudaMemsetAsync(counts.p, 0, sizeof(uint32_t) * (size_t)(s + 1), st));
    const uint64_t mask = ((uint64_t)s & ((uint64_t)s - 1)) == 0 ? (uint64_t)s - 1 : 0;
    const int grid = (int)std::min<int64_t>((n + 255) / 256, (int64_t)ctx->num_sms * 8);
    // s == 1: mask 0 would mean "use modulo"; h % 1 == 0 either way.
    cs_hash_kernel<<<grid, 256, 0, st>>>(seed, j0, n, (uint64_t)s, mask, keys.as<uint32_t>(), vals.as<uint32_t>(),
                                         counts.as<uint32_t>());
    RNLA_CUDA(cudaGetLastError());
    note_launch(ctx);
    int bits = 1;
    while (bits < 32 && ((int64_t)1 << bits) < s) ++bits;
    size_t tmp_bytes = 0, scan_bytes = 0;
    RNLA_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys.as<uint32_t>(), keys_out.as<uint32_t>(),
                                              vals.as<uint32_t>(), plan->rows.as<uint32_t>(), (int)n, 0, bits, st));
    RNLA_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, counts.as<uint32_t>(),
                                            plan->offsets.as<uint32_t>(), (int)(s + 1), st));
    DevBuf tmp(std::max(tmp_bytes, scan_bytes), st);
    RNLA_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, keys.as<uint32_t>(), keys_out.as<uint32_t>(),
                                              vals.as<uint32_t>(), plan->rows.as<uint32_t>(), (int)n, 0, bits, st));
    RNLA_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, scan_bytes, counts.as<uint32_t>(), plan->offsets.as<uint32_t>(),
                                            (int)(s + 1), st));
    note_launch(ctx, 4);
  }
  auto& ref = *plan;
  ctx->cs_plans.emplace(key, std::move(plan));
  return ref;
}

template <class T>
void count_sketch_segments(rnla_ctx* ctx, const T* in, int64_t ld, const T* extra, int64_t extra_stride, int64_t n,
                           int64_t L, int64_t s, uint64_t seed, int64_t j0, T* out, int64_t ldo, bool accumulate,
                           int64_t b0, int64_t b1) {
  const int64_t Lo = L + (extra ? 1 : 0);
  if (b1 < 0 || b1 > s) b1 = s;
  if (b0 < 0) b0 = 0;
  if (b1 <= b0) return;
  if (n == 0 || Lo == 0) {
    if (!accumulate && Lo > 0) {
      RNLA_CUDA(cudaMemset2DAsync(out + b0 * ldo, sizeof(T) * ldo, 0, sizeof(T) * Lo, b1 - b0, ctx->stream));
    }
    return;
  }
  const CountSketchPlan& plan = count_sketch_plan(ctx, n, s, seed, j0);
#define RNLA_G(TEAM, CPT) \
  launch_gather<T, TEAM, CPT>(ctx, in, ld, extra, extra_stride, L, Lo, plan, out, ldo, accumulate, b0, b1)
  if (Lo <= 32) RNLA_G(32, 1);
  else if (Lo <= 64) RNLA_G(32, 2);
  else if (Lo <= 128) RNLA_G(32, 4);
  else if (Lo <= 256) RNLA_G(128, 2);
  else if (Lo <= 512) RNLA_G(128, 4);
  else if (Lo <= 640) RNLA_G(128, 5);
  else RNLA_G(128, 8);
#undef RNLA_G
}

void count_sketch_plan_release(rnla_ctx* ctx, int64_t n, int64_t s, uint64_t seed, int64_t j0) {
  ctx->cs_plans.erase(std::make_tuple(n, s, j0, seed));
}

template void count_sketch_segments<double>(rnla_ctx*, const double*, int64_t, const double*, int64_t, int64_t, int64_t,
                                            int64_t, uint64_t, int64_t, double*, int64_t, bool, int64_t, int64_t);
template void count_sketch_segments<float>(rnla_ctx*, const float*, int64_t, const float*, int64_t, int64_t, int64_t,
                                           int64_t, uint64_t, int64_t, float*, int64_t, bool, int64_t, int64_t);

}  // namespace rnla
