// srht.h -- SRHT operator plan (signs, sampled indices grouped by low bits).
#pragma once
#include <cuda.h>

#include "rnla_internal.h"

namespace rnla {

struct SrhtPlan {
  int64_t n = 0, s = 0, big_n = 0;
  uint64_t seed = 0;
  int q = 0, qlo = 0, qhi = 0;
  std::vector<int64_t> host_idx;   // sorted sampled indices (src/sketch.cpp:65)
  DevBuf signs;                    // int8[n]
  DevBuf grp_off, grp_t, grp_hi;   // samples grouped by idx & (2^qlo - 1)
  int64_t block_off = 0;           // block plans: global index of the block's first row
  DevBuf out_sign;                 // block plans: (-1)^popcount(block_off & idx_t), fp64[s]
  // One-pass accumulating path (srht_acc.cu), built on first use: per-(tile,
  // row-group) sign bit masks and the packed (high, low) bits of each sample.
  mutable DevBuf acc_mask, acc_samp, acc_slot;  // one-pass SRHT: sign masks, slot -> sample, sample -> slot
  SrhtPlan(rnla_ctx* ctx, int64_t n, int64_t s, uint64_t seed);
  // Plan of one aligned block (2^b rows at block_off, `present` of them real)
  // of a global operator whose sampled indices are idx[0..s).
  SrhtPlan(rnla_ctx* ctx, const int8_t* block_signs, int64_t present, int64_t block, const int64_t* idx, int64_t s,
           int64_t block_off);

 private:
  void build(rnla_ctx* ctx, const int8_t* signs, const int64_t* idx);
};

// Scratch budget per launch pair of the two-pass transform (RNLA_SRHT_STRIP_MB, default 1024).
inline int64_t srht_strip_mb() {
  static const int64_t mb = std::getenv("RNLA_SRHT_STRIP_MB") ? std::max<long long>(1, std::atoll(std::getenv("RNLA_SRHT_STRIP_MB"))) : 1024;
  return mb;
}

// TMA-fed fp32 path (srht_tma.cu); false when the shape/alignment does not apply.
bool srht_tma_f32(rnla_ctx* ctx, const SrhtPlan& plan, const float* in, int64_t ld, int64_t L, float* out,
                  int64_t out_rs, int64_t out_cs);

// One-pass fp32 path with the sampled outputs accumulated in TMEM
// (srht_acc.cu); false when the shape/alignment does not apply.
bool srht_acc_f32(rnla_ctx* ctx, const SrhtPlan& plan, const float* in, int64_t ld, int64_t L, float* out,
                  int64_t out_rs, int64_t out_cs);

// TMA tensor map over a row-major fp32 matrix (rows x cols, row pitch ld
// elements), boxes of box_rows x box_cols (srht_tma.cu).
bool tma_encode_available();
void tma_map_rows_f32(CUtensorMap* m, const float* base, int64_t rows, int64_t cols, int64_t ld, uint32_t box_cols,
                      uint32_t box_rows);

// out_t[c] (t < s, c < L) at out[t*out_rs + c*out_cs]; segment j at in + j*ld.
template <class T>
void srht_segments(rnla_ctx* ctx, const SrhtPlan& plan, const T* in, int64_t ld, int64_t L, T* out, int64_t out_rs,
                   int64_t out_cs);

// Row-sharded S^T M: this rank's n_local rows start at global row row_off of
// n_total; the replicated s x L result is written to out.
template <class T>
void srht_rows_sharded(rnla_ctx* ctx, const T* in, int64_t ld, int64_t n_local, int64_t L, int64_t row_off,
                       int64_t n_total, int64_t s, uint64_t seed, T* out, int64_t out_rs, int64_t out_cs);

}  // namespace rnla
