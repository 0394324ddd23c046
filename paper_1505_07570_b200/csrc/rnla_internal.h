// rnla_internal.h -- shared internals of librnla_b200 (not part of the ABI).
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "rnla.h"

namespace rnla {

// Exceptions used inside the library; the C ABI layer maps them to status
// codes (they never cross the boundary).
struct InvalidArgument : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct NumericError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NcclError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// Mirror of the reference's require() (include/randnla/types.hpp:35-37).
// Overloads: a literal message costs nothing unless the check fails (no
// std::string temporary per call inside host loops).
inline void require(bool cond, const char* msg) {
  if (!cond) throw InvalidArgument(msg);
}
inline void require(bool cond, const std::string& msg) {
  if (!cond) throw InvalidArgument(msg);
}

#define RNLA_CUDA(expr)                                                                       \
  do {                                                                                        \
    cudaError_t e__ = (expr);                                                                 \
    if (e__ != cudaSuccess)                                                                   \
      throw ::rnla::CudaError(std::string(#expr) + ": " + cudaGetErrorString(e__) + " @" +   \
                              __FILE__ + ":" + std::to_string(__LINE__));                     \
  } while (0)

// Device buffer owned by RAII (stream-ordered allocator).
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaStream_t st = nullptr;
  DevBuf() = default;
  DevBuf(size_t b, cudaStream_t s) : bytes(b), st(s) {
    if (b) RNLA_CUDA(cudaMallocAsync(&p, b, s));
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), bytes(o.bytes), st(o.st) { o.p = nullptr; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    release();
    p = o.p; bytes = o.bytes; st = o.st; o.p = nullptr;
    return *this;
  }
  ~DevBuf() { release(); }
  void release() {
    if (p) cudaFreeAsync(p, st);
    p = nullptr;
  }
  template <class T> T* as() const { return static_cast<T*>(p); }
};

// Cached device-resident operator (hash permutation, Gaussian Omega, ...).
struct CountSketchPlan {
  int64_t n = 0, s = 0, j0 = 0;
  uint64_t seed = 0;
  DevBuf offsets;  // int64[s + 1]: first slot of each bucket
  DevBuf rows;     // uint32[n]: local row index | sign bit (bit 31 = negative)
};

struct SrhtPlan;

struct DenseOperator {  // G / sqrt(s) as the reference forms it, device fp64/fp32
  DevBuf data;
  int64_t rows = 0, cols = 0;
  int dtype = RNLA_F64;
  // int8 digit planes of the transposed operator for the Ozaki-split Gaussian
  // stage (ozaki.cu), built on first use
  mutable DevBuf oz_planes, oz_rscale;
  mutable int64_t oz_pitch = 0;
};
// fp64 Gaussian stage out (+)= Gs(k0 : k0 + kc, :)' in(k0 : k0 + kc, :) on the
// int8 tensor cores (ozaki.cu); false when the shape does not apply.
bool ozaki_applies(int64_t s, int64_t L);
bool ozaki_gemm_rowcol(rnla_ctx* ctx, int64_t m, int64_t n, int64_t k, const double* A, int64_t a_ld, const double* B,
                       int64_t b_ld, double* C, int64_t c_rs, int64_t c_cs);
bool ozaki_gaussian_chunk(rnla_ctx* ctx, const DenseOperator& g, const double* in, int64_t ld, int64_t n, int64_t L,
                          int64_t s, int64_t k0, int64_t kc, bool accumulate, double* out, int64_t out_rs,
                          int64_t out_cs);


}  // namespace rnla

namespace rnla {
// An instantiated CUDA graph of a whole call (e.g. the speculative
// prototype_ksvd pipeline) plus the persistent device buffers it writes.
struct CachedGraph {
  cudaGraphExec_t exec = nullptr;
  std::vector<void*> bufs;  // cudaMalloc'd, owned
  int64_t kernels = 0;      // kernel nodes (launch accounting per replay)
  std::vector<int64_t> meta;
  CachedGraph() = default;
  CachedGraph(const CachedGraph&) = delete;
  CachedGraph& operator=(const CachedGraph&) = delete;
  ~CachedGraph() {
    if (exec) cudaGraphExecDestroy(exec);
    for (void* p : bufs) cudaFree(p);
  }
};
}  // namespace rnla

struct rnla_ctx {
  int device = 0;
  int world = 1, rank = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t copy_stream = nullptr;
  cudaStream_t aux_stream = nullptr;
  cudaEvent_t caller_ev = nullptr;  // rnla_ctx_wait_stream  // concurrent compute (e.g. Gaussian stage under the count sketch)
  void* nccl = nullptr;      // ncclComm_t
  rnla_group* group = nullptr;  // in-process host-staged group (dist.cpp), else NCCL
  void* cusolver = nullptr;  // cusolverDnHandle_t
  void* cublas = nullptr;    // cublasHandle_t
  int num_sms = 148;
  int64_t launches = 0;
  std::mutex mu;
  std::map<std::tuple<int64_t, int64_t, int64_t, uint64_t>, std::unique_ptr<rnla::CountSketchPlan>> cs_plans;
  std::map<std::tuple<int64_t, int64_t, uint64_t, int>, std::unique_ptr<rnla::DenseOperator>> gauss_ops;
  std::map<std::tuple<int64_t, int64_t, uint64_t>, std::shared_ptr<rnla::SrhtPlan>> srht_plans;
  // Nystrom landmark draws sample_without_replacement(n, s, derive_seed(seed, 1)), keyed by (n, s, seed)
  std::map<std::tuple<int64_t, int64_t, uint64_t>, std::vector<int64_t>> landmark_sel;
  // Helper context on the same device (own high-priority stream and library
  // handles) for independent work run from a second host thread, e.g. eig(W)
  // under the Nystrom C'C Gram; created lazily by side_ctx().
  std::unique_ptr<rnla_ctx> side;
  // Captured call graphs keyed by their full argument signature (pointers
  // included); they reference cached operators, so they are dropped first
  // whenever the operator caches are.
  std::map<std::string, std::unique_ptr<rnla::CachedGraph>> graphs;
  bool capturing = false;  // a stream capture is open (trace_mark must not synchronize)
  // Pinned host staging (grown on demand, freed with the context): device
  // results streamed to the host while later blocks still compute.
  void* pinned = nullptr;
  size_t pinned_bytes = 0;
};

namespace rnla {

// Pinned host buffer of at least `bytes` owned by the context.
void* pinned_scratch(rnla_ctx* ctx, size_t bytes);

// ---- host operator generation (host_rng.cpp; libstdc++ like the reference) ----
uint64_t splitmix64(uint64_t& state);
uint64_t derive_seed(uint64_t seed, uint64_t stream);
void gaussian_matrix_host(uint64_t seed, int64_t rows, int64_t cols, double* out_colmajor);
std::vector<int64_t> sample_without_replacement_host(uint64_t seed, int64_t n, int64_t count);
std::vector<int64_t> sample_with_replacement_host(uint64_t seed, const double* w, int64_t n, int64_t count);
// The same draw with the prefix sums built incrementally (blocks of weights in
// row order, e.g. as they arrive from the device): extend() appends, draw()
// samples once all n weights are in.
struct WeightPrefix {
  std::vector<double> cum;
  double total = 0.0;
  void extend(const double* w, int64_t m);
  std::vector<int64_t> draw(uint64_t seed, int64_t count) const;
  // The part of the draw that does not depend on the weights: the engine's
  // canonical uniforms in draw order and their ascending order. Prepared while
  // the device still computes the scores, it leaves only the scaling by the
  // total and the searches for draw(const Prepared&).
  struct Prepared {
    std::vector<double> canon;
    std::vector<int64_t> order;
  };
  static Prepared prepare(uint64_t seed, int64_t count);
  std::vector<int64_t> draw(const Prepared& pr) const;
};
void srht_operator_host(uint64_t seed, int64_t n, int64_t s, int8_t* signs, int64_t* idx);
int64_t next_pow2(int64_t n);

// ---- device kernels (launchers; all enqueue on ctx->stream) ----
// Count sketch of segments: out[b*ldo + c] (+)= sum_{j: h(j0+j)=b, j asc} g * seg_j[c]
// where seg_j[c] = in[j*ld + c] for c < L and extra[j*extra_stride] for c == L.
template <class T>
void count_sketch_segments(rnla_ctx* ctx, const T* in, int64_t ld, const T* extra, int64_t extra_stride, int64_t n,
                           int64_t L, int64_t s, uint64_t seed, int64_t j0, T* out, int64_t ldo, bool accumulate,
                           int64_t b0 = 0, int64_t b1 = -1);
const CountSketchPlan& count_sketch_plan(rnla_ctx* ctx, int64_t n, int64_t s, uint64_t seed, int64_t j0);
// Drop a cached plan (one-shot plans, e.g. the chunks of count_sketch_stream).
void count_sketch_plan_release(rnla_ctx* ctx, int64_t n, int64_t s, uint64_t seed, int64_t j0);

// General strided GEMM: C[m x n] = alpha * A[m x k] * B[k x n] + beta * C, element
// (i, j) of X at X[i*rs + j*cs].
template <class T>
void gemm(rnla_ctx* ctx, int64_t m, int64_t n, int64_t k, T alpha, const T* A, int64_t a_rs, int64_t a_cs,
          const T* B, int64_t b_rs, int64_t b_cs, T beta, T* C, int64_t c_rs, int64_t c_cs, int max_splits = 64);

// Phase tracing (RNLA_TRACE=1): synchronizes the context stream and prints the
// wall time since the previous mark of this thread to stderr. No-op otherwise.
void trace_mark(rnla_ctx* ctx, const char* label);
// The lazily created helper context of ctx (see rnla_ctx::side); world 1, no group.
rnla_ctx* side_ctx(rnla_ctx* ctx);

// Temporarily route ctx launches to another stream (RAII).
struct StreamScope {
  rnla_ctx* ctx;
  cudaStream_t saved;
  StreamScope(rnla_ctx* c, cudaStream_t s);
  ~StreamScope();
};

// fp32 GEMM on tcgen05 with the BF16x3 split (gemm_tc.cu); RNLA_DISABLE_TCGEN05
// selects the SIMT fp32 kernel instead (A/B comparison only).
bool tc_gemm_enabled();
void gemm_f32_tc(rnla_ctx* ctx, int64_t m, int64_t n, int64_t k, float alpha, const float* A, int64_t a_rs,
                 int64_t a_cs, const float* B, int64_t b_rs, int64_t b_cs, float beta, float* C, int64_t c_rs,
                 int64_t c_cs);
// Row sums of squares of C = alpha A B (B upper triangular) per N tile, C not
// stored: rownorm[t * m + i], t < the returned tile count (gemm_tc.cu).
int gemm_f32_tc_tri_b_rownorm(rnla_ctx* ctx, int64_t m, int64_t n, int64_t k, float alpha, const float* A,
                              int64_t a_rs, int64_t a_cs, const float* B, int64_t b_rs, int64_t b_cs, double* rownorm);
// gemm_f32_tc with B upper triangular (zero blocks below the diagonal skipped).
void gemm_f32_tc_tri_b(rnla_ctx* ctx, int64_t m, int64_t n, int64_t k, float alpha, const float* A, int64_t a_rs,
                       int64_t a_cs, const float* B, int64_t b_rs, int64_t b_cs, float beta, float* C, int64_t c_rs,
                       int64_t c_cs);

// Same on tcgen05 with double-float (~fp64) accumulation across 256-row chunks, fp64 output.
void gemm_f32_tc_f64acc(rnla_ctx* ctx, int64_t m, int64_t n, int64_t k, double alpha, const float* A, int64_t a_rs,
                        int64_t a_cs, const float* B, int64_t b_rs, int64_t b_cs, double beta, double* C,
                        int64_t c_rs, int64_t c_cs);

// Gram-type fp32 products with fp64-grade accumulation: tcgen05 double-float
// when enabled, else the DMMA widening kernel below.
// C = A B (fp64, DMMA) with structure: flags bit 0 C symmetric (upper tiles,
// mirrored), bit 1 B upper triangular, bit 2 A lower triangular -- the zero
// k-blocks are skipped. False when the K-major cp.async kernel does not apply.
bool gemm_f64_structured(rnla_ctx* ctx, int64_t m, int64_t n, int64_t k, const double* A, int64_t a_rs, int64_t a_cs,
                         const double* B, int64_t b_rs, int64_t b_cs, double* C, int64_t c_rs, int64_t c_cs,
                         int flags);
void gemm_f32_in_f64(rnla_ctx* ctx, int64_t m, int64_t n, int64_t k, double alpha, const float* A, int64_t a_rs,
                     int64_t a_cs, const float* B, int64_t b_rs, int64_t b_cs, double beta, double* C, int64_t c_rs,
                     int64_t c_cs);
inline void gemm_f32_f64acc(rnla_ctx* ctx, int64_t m, int64_t n, int64_t k, double alpha, const float* A,
                            int64_t a_rs, int64_t a_cs, const float* B, int64_t b_rs, int64_t b_cs, double beta,
                            double* C, int64_t c_rs, int64_t c_cs) {
  if (tc_gemm_enabled())
    gemm_f32_tc_f64acc(ctx, m, n, k, alpha, A, a_rs, a_cs, B, b_rs, b_cs, beta, C, c_rs, c_cs);
  else
    gemm_f32_in_f64(ctx, m, n, k, alpha, A, a_rs, a_cs, B, b_rs, b_cs, beta, C, c_rs, c_cs);
}

// fp32 operands, exact widening to fp64, DMMA fp64 accumulation (Gram-type products).
void gemm_f32_in_f64(rnla_ctx* ctx, int64_t m, int64_t n, int64_t k, double alpha, const float* A, int64_t a_rs,
                     int64_t a_cs, const float* B, int64_t b_rs, int64_t b_cs, double beta, double* C, int64_t c_rs,
                     int64_t c_cs);

// Device copy between strided 2-D layouts (also casts f64<->f32 via the typed overloads).
template <class T>
void copy2d(rnla_ctx* ctx, int64_t rows, int64_t cols, const T* src, int64_t s_rs, int64_t s_cs, T* dst, int64_t d_rs,
            int64_t d_cs);
template <class T>
void scale_inplace(rnla_ctx* ctx, T* p, int64_t count, double divisor);

inline void note_launch(rnla_ctx* ctx, int64_t k = 1) { ctx->launches += k; }

// Row-sharded context: more than one rank, or any NCCL context (a world-1
// NCCL context runs the sharded code paths and their collectives over a
// one-rank communicator, so the NCCL transport is exercised on one GPU).
inline bool is_sharded(const rnla_ctx* c) { return c->world > 1 || c->nccl != nullptr; }

}  // namespace rnla
