// srht.h -- SRHT operator plan (signs, sampled indices grouped by low bits).
#pragma once
#include "rnla_internal.h"

namespace rnla {

struct SrhtPlan {
  int64_t n = 0, s = 0, big_n = 0;
  uint64_t seed = 0;
  int q = 0, qlo = 0, qhi = 0;
  std::vector<int64_t> host_idx;   // sorted sampled indices (src/sketch.cpp:65)
  DevBuf signs;                    // int8[n]
  DevBuf grp_off, grp_t, grp_hi;   // samples grouped by idx & (2^qlo - 1)
  SrhtPlan(rnla_ctx* ctx, int64_t n, int64_t s, uint64_t seed);
};

// TMA-fed fp32 path (srht_tma.cu); false when the shape/alignment does not apply.
bool srht_tma_f32(rnla_ctx* ctx, const SrhtPlan& plan, const float* in, int64_t ld, int64_t L, float* out,
                  int64_t out_rs, int64_t out_cs);

// out_t[c] (t < s, c < L) at out[t*out_rs + c*out_cs]; segment j at in + j*ld.
template <class T>
void srht_segments(rnla_ctx* ctx, const SrhtPlan& plan, const T* in, int64_t ld, int64_t L, T* out, int64_t out_rs,
                   int64_t out_cs);

}  // namespace rnla
