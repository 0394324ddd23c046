// linalg.cuh -- small dense factorizations on the device (linalg.cu).
#pragma once
#include "rnla_internal.h"

namespace rnla {

// fix_column_signs (src/core.cpp:15-33) on column-major-or-strided M (rows x cols):
// flips column j of M, and column j (pair_cols) or row j of P (p_len entries).
void fix_column_signs(rnla_ctx* ctx, int64_t rows, int64_t cols, double* M, int64_t m_rs, int64_t m_cs, double* P,
                      int64_t p_rs, int64_t p_cs, int64_t p_len, bool pair_cols);

void fix_column_signs_f32(rnla_ctx* ctx, int64_t rows, int64_t cols, float* M, int64_t m_rs, int64_t m_cs);
// The same rule for a row-sharded M (this rank's consecutive row block): the
// first entry over the global row order decides (one allgather of per-rank
// lead signs); P (replicated) is flipped like fix_column_signs does.
template <class T>
void fix_column_signs_sharded(rnla_ctx* ctx, int64_t rows, int64_t cols, T* M, int64_t m_rs, int64_t m_cs, double* P,
                              int64_t p_rs, int64_t p_cs, int64_t p_len, bool pair_cols);
// Flip columns of the upper-triangular Rinv so that Y * Rinv satisfies the sign
// rule on its first row (Y row 0 at Y[p * y_cs]); false when a sign is not
// decidable from row 0 (then fix the product with fix_column_signs).
template <class T>
bool presign_upper_inverse(rnla_ctx* ctx, int64_t cols, const T* Y, int64_t y_cs, double* Rinv);

// Householder thin QR of column-major A (m x n, ld m), in place: A <- Q;
// R (n x n, upper, exact zeros below) written with strides (r_rs, r_cs).
void qr_householder(rnla_ctx* ctx, int64_t m, int64_t n, double* A, double* R, int64_t r_rs, int64_t r_cs);

// Thin SVD: U m x r (col-major, ld m), S[r] descending, V n x r (col-major, ld n), r = min(m, n).
void svd_thin(rnla_ctx* ctx, int64_t m, int64_t n, const double* A, int64_t a_rs, int64_t a_cs, double* U, double* S,
              double* V);

// In-place upper Cholesky G = R'R of column-major G (n x n); false if not positive definite.
bool cholesky_upper(rnla_ctx* ctx, int64_t n, double* G);
// One CholeskyQR pass on the m x n col-major Y in place (Y := Y R^-1, R'R = Y'Y);
// false (Y untouched) on a Cholesky breakdown.
bool cholqr_inplace(rnla_ctx* ctx, int64_t m, int64_t n, double* Y);
// min |R_ii| > thresh * max |R_ii| and all finite (CholeskyQR breakdown test).
bool diag_ratio_ok(rnla_ctx* ctx, int64_t n, const double* R, double thresh);

// One-CTA Cholesky (G = R'R, upper) + R^-1 for n <= kSmallCholMax, all on the
// device: status (device int) bit 1 = breakdown, 2 = diag ratio below thresh,
// 4 = row-0 sign probe undecidable; with y0 the columns of Rinv are negated
// so that row 0 of Y Rinv is non-negative. Rinv32 (nullable) gets an fp32 copy.
// n <= 152: the factor, the blocked inverse and their scratch fit 227 KB of
// shared memory.
constexpr int64_t kSmallCholMax = 152;
// Same contract for any n on cuSOLVER potrf + cuBLAS trsm (G is overwritten by
// R), with no host round trip. Rinv32 (nullable) gets an fp32 copy.
template <class T>
void chol_inv_async(rnla_ctx* ctx, int64_t n, double* G, double* Rinv, float* Rinv32, const T* y0, int64_t y_cs,
                    double thresh, int* status);
template <class T>
void small_chol_inv(rnla_ctx* ctx, int64_t n, const double* G, double* Rinv, float* Rinv32, const T* y0, int64_t y_cs,
                    double thresh, int* status);
// Rinv = R^-1 for upper-triangular column-major R (entries below the diagonal ignored).
void upper_inverse(rnla_ctx* ctx, int64_t n, const double* R, double* Rinv);

// Symmetric eigen-decomposition of column-major A (n x n): A <- eigenvectors, W ascending.
void eig_sym(rnla_ctx* ctx, int64_t n, double* A, double* W);
// The same (syevd: W ascending, eigenvectors in A) without the host round
// trip: syevd's info lands in *info.
void eig_sym_async(rnla_ctx* ctx, int64_t n, double* A, double* W, int* info);
// One-CTA Jacobi (jacobi.cuh) for b <= 32 without a host round trip: lam
// descending, Z the matching eigenvectors; *status = 0 on convergence (sweeps
// in bits 8+), 1 otherwise. False when b is out of range.
// One-CTA tridiagonal eigensolver for 32 < n <= 128 (descending, Z may alias
// H); false when n is out of range. *status = 1: fall back (clustered spectrum).
bool eig_tri_async(rnla_ctx* ctx, int64_t n, const double* H, double* lam, double* Z, int* status);
bool eig_small_jacobi_async(rnla_ctx* ctx, int64_t b, const double* H, double* lam, double* Z, int* status);
// Symmetric b x b H (b <= 256) by cuSOLVER syevj: lam[b] descending and Z
// (b x b, column-major) the matching orthonormal eigenvectors; H is not
// modified. False when b is out of range (the caller falls back to eig_sym).
bool eig_sym_small_desc(rnla_ctx* ctx, int64_t b, const double* H, double* lam, double* Z);
// The k largest eigenpairs only (syevdx, index range): W[0..k) ascending, their
// eigenvectors in the first k columns of A. Returns the number found.
int64_t eig_sym_top(rnla_ctx* ctx, int64_t n, double* A, int64_t k, double* W);

}  // namespace rnla
