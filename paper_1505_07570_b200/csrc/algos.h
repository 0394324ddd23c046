// algos.h -- internal building blocks shared by the api_*.cpp entry points.
#pragma once
#include "marshal.h"
#include "srht.h"

namespace rnla {

struct SvdDev {  // condensed_svd result on the device (column-major fp64)
  DevBuf U, V;   // m x rank, n x rank (allocated for min(m, n) columns)
  std::vector<double> s;
  int64_t rank = 0, m = 0, n = 0;
};

const DenseOperator& gaussian_operator(rnla_ctx* ctx, int64_t n, int64_t s, uint64_t seed, int dtype);
std::shared_ptr<SrhtPlan> srht_plan(rnla_ctx* ctx, int64_t n, int64_t s, uint64_t seed);

void thin_qr_dev(rnla_ctx* ctx, int64_t m, int64_t n, double* W, double* R);
SvdDev condensed_svd_dev(rnla_ctx* ctx, int64_t m, int64_t n, const double* A, int64_t a_rs, int64_t a_cs);
void store_block(rnla_ctx* ctx, const double* src, int64_t rows, int64_t cols, int64_t ld, OutMat& o);
DevMat f64_colmajor(rnla_ctx* ctx, const rnla_mat* a);

// out (r x n, col-major) = diag(s) * V^T for V n x r col-major.
void scale_rows_dev(rnla_ctx* ctx, int64_t r, int64_t n, const double* V, const double* s, double* out);
// out (n x r, col-major) = V * diag(d).
void scale_cols_dev(rnla_ctx* ctx, int64_t n, int64_t r, const double* V, const double* d, double* out);
double sum_squares_dev(rnla_ctx* ctx, const double* p, int64_t count);
// out[e] uniform in [-1, 1) from a counter hash of (seed, e): deterministic start blocks.
void hash_uniform_dev(rnla_ctx* ctx, int64_t count, uint64_t seed, double* out);
// out[j] = |YZ(:, j) - theta[j] VZ(:, j)|^2 for n x k col-major YZ, VZ (theta on the device).
void ritz_residual_dev(rnla_ctx* ctx, int64_t n, int64_t k, const double* YZ, const double* VZ, const double* theta,
                       double* out);

// Top-k eigenpairs of the symmetric n x n fp64 matrix A (device, col-major) by
// block subspace iteration with Rayleigh-Ritz: lam (host, k, descending) and
// V (device, n x k, matching columns). Returns false (outputs untouched) when
// the problem is too small for a block of 2k or it did not converge; callers
// then use the direct solver (api_linalg.cpp).
bool eig_top_subspace(rnla_ctx* ctx, int64_t n, const double* A, int64_t k, double* lam, double* V,
                      bool values_only = false);

// g = A'(beta*b - A w) and *rr = |beta*b - A w|^2 in one pass over the
// row-major A (n x d, row stride ld; d <= 1024), fp64 accumulation; g and rr
// are device pointers (lsr.cu).
bool normal_gemv_supported(int64_t d);
template <class T>
void normal_gemv(rnla_ctx* ctx, int64_t n, int64_t d, const T* A, int64_t ld, const T* b, int64_t b_stride,
                 double beta, const double* w, double* g, double* rr);

// Row sketch of a row-major tall M (n rows of length L, row stride ld) into
// out (element (t, c) at out[t*o_rs + c*o_cs]); api_sketch.cpp.
template <class T>
void sketch_rows_dev(rnla_ctx* ctx, const T* M, int64_t ld, const T* extra, int64_t xs, int64_t n, int64_t L,
                     const rnla_sketch_spec* spec, int64_t row_offset, T* out, int64_t o_rs, int64_t o_cs);

}  // namespace rnla
