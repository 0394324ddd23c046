// api_linalg.cpp -- core.hpp (thin_qr, condensed/truncated SVD, pinv),
// randsvd.hpp (prototype_ksvd + power iterations) and the column-selection
// sketches behind the C ABI.
//
// Reference: /root/reference/proj/src/core.cpp:15-88, src/randsvd.cpp:88-110,
// src/sketch.cpp:125-167. Small factorizations run on the device in fp64
// (linalg.cu); the passes over A are the GEMM kernels of gemm.cu.
#include <cmath>
#include <cstdio>
#include <limits>
#include <numeric>

#include "algos.h"
#include "dist.h"
#include "linalg.cuh"
#include "marshal.h"
#include "rbf.cuh"

namespace rnla {

// ---------------------------------------------------------------------------
// small dense building blocks on fp64 column-major device buffers
// ---------------------------------------------------------------------------

// thin_qr semantics (src/core.cpp:37-46): Q (m x n) overwrites W, R n x n.
void thin_qr_dev(rnla_ctx* ctx, int64_t m, int64_t n, double* W, double* R) {
  qr_householder(ctx, m, n, W, R, 1, n);
  fix_column_signs(ctx, m, n, W, 1, m, R, 1, n, n, /*pair_cols=*/false);
}

// condensed_svd semantics (src/core.cpp:48-64) of A (m x n, strided fp64).
SvdDev condensed_svd_dev(rnla_ctx* ctx, int64_t m, int64_t n, const double* A, int64_t a_rs, int64_t a_cs) {
  SvdDev f;
  const int64_t r = std::min(m, n);
  f.U = DevBuf(sizeof(double) * std::max<int64_t>(m * r, 1), ctx->stream);
  f.V = DevBuf(sizeof(double) * std::max<int64_t>(n * r, 1), ctx->stream);
  DevBuf sv(sizeof(double) * std::max<int64_t>(r, 1), ctx->stream);
  if (r == 0) throw InvalidArgument("condensed_svd: zero matrix has rank 0");
  if (m >= 2 * n) {
    // Tall: A = Q R (Householder), R = Ur S V', U = Q Ur.
    DevBuf q(sizeof(double) * m * n, ctx->stream), rr(sizeof(double) * n * n, ctx->stream),
        ur(sizeof(double) * n * n, ctx->stream);
    copy2d<double>(ctx, m, n, A, a_rs, a_cs, q.as<double>(), 1, m);
    qr_householder(ctx, m, n, q.as<double>(), rr.as<double>(), 1, n);
    svd_thin(ctx, n, n, rr.as<double>(), 1, n, ur.as<double>(), sv.as<double>(), f.V.as<double>());
    gemm<double>(ctx, m, n, n, 1.0, q.as<double>(), 1, m, ur.as<double>(), 1, n, 0.0, f.U.as<double>(), 1, m);
  } else if (n >= 2 * m) {
    // Wide: A' = Q R, R = Ur S V' => A = V S (Q Ur)'.
    DevBuf q(sizeof(double) * n * m, ctx->stream), rr(sizeof(double) * m * m, ctx->stream),
        ur(sizeof(double) * m * m, ctx->stream);
    copy2d<double>(ctx, n, m, A, a_cs, a_rs, q.as<double>(), 1, n);
    qr_householder(ctx, n, m, q.as<double>(), rr.as<double>(), 1, m);
    svd_thin(ctx, m, m, rr.as<double>(), 1, m, ur.as<double>(), sv.as<double>(), f.U.as<double>());
    gemm<double>(ctx, n, m, m, 1.0, q.as<double>(), 1, n, ur.as<double>(), 1, m, 0.0, f.V.as<double>(), 1, n);
  } else {
    svd_thin(ctx, m, n, A, a_rs, a_cs, f.U.as<double>(), sv.as<double>(), f.V.as<double>());
  }
  f.s.resize((size_t)r);
  RNLA_CUDA(cudaMemcpyAsync(f.s.data(), sv.p, sizeof(double) * r, cudaMemcpyDeviceToHost, ctx->stream));
  RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
  const double sigma1 = f.s[0];
  if (!(sigma1 > 0.0)) throw InvalidArgument("condensed_svd: zero matrix has rank 0");
  const double thresh = (double)std::max(m, n) * std::numeric_limits<double>::epsilon() * sigma1;
  int64_t rho = 0;
  while (rho < r && f.s[(size_t)rho] > thresh) ++rho;
  f.rank = rho;
  f.m = m;
  f.n = n;
  f.s.resize((size_t)rho);
  fix_column_signs(ctx, m, rho, f.U.as<double>(), 1, m, f.V.as<double>(), 1, n, n, /*pair_cols=*/true);
  return f;
}

// Top-k of condensed_svd for a short-wide B (s x n, s <= n, column-major fp64),
// as truncated_svd(B, k) uses it in prototype_ksvd (src/randsvd.cpp:100-101):
// eig(B B') = (Ubar, sigma^2), V = B' Ubar / sigma, then the reference's sign
// rule on Ubar (paired with V). The Gram squares the condition number, so it
// is used only when sigma_k >= 1e-3 sigma_1 (relative error of sigma_i is
// ~eps (sigma_1/sigma_i)^2 <= 1e-10 there); otherwise QR + SVD.
SvdDev topk_svd_wide(rnla_ctx* ctx, int64_t s, int64_t n, const double* B, int64_t k) {
  if (s > 512 || k < 1 || std::getenv("RNLA_SVD_NO_GRAM")) return condensed_svd_dev(ctx, s, n, B, 1, s);
  DevBuf G(sizeof(double) * s * s, ctx->stream), lam(sizeof(double) * s, ctx->stream);
  gemm<double>(ctx, s, s, n, 1.0, B, 1, s, B, s, 1, 0.0, G.as<double>(), 1, s);
  std::vector<double> h((size_t)s);
  DevBuf Zd(sizeof(double) * s * s, ctx->stream);
  if (s <= 160 && eig_sym_small_desc(ctx, s, G.as<double>(), lam.as<double>(), Zd.as<double>())) {
    // one-CTA Jacobi / tridiagonal solver; back to the ascending layout used below
    copy2d<double>(ctx, s, s, Zd.as<double>() + (s - 1) * s, 1, -s, G.as<double>(), 1, s);
    RNLA_CUDA(cudaMemcpyAsync(h.data(), lam.p, sizeof(double) * s, cudaMemcpyDeviceToHost, ctx->stream));
    RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
    std::reverse(h.begin(), h.end());
  } else {
    eig_sym(ctx, s, G.as<double>(), lam.as<double>());
    RNLA_CUDA(cudaMemcpyAsync(h.data(), lam.p, sizeof(double) * s, cudaMemcpyDeviceToHost, ctx->stream));
    RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  const double l1 = h[(size_t)s - 1], lk = h[(size_t)(s - k)];
  if (!(l1 > 0.0) || !(lk > 1e-6 * l1)) return condensed_svd_dev(ctx, s, n, B, 1, s);
  SvdDev f;
  f.m = s;
  f.n = n;
  f.rank = k;
  f.s.resize((size_t)k);
  std::vector<double> inv((size_t)k);
  for (int64_t i = 0; i < k; ++i) {
    f.s[(size_t)i] = std::sqrt(h[(size_t)(s - 1 - i)]);
    inv[(size_t)i] = 1.0 / f.s[(size_t)i];
  }
  f.U = DevBuf(sizeof(double) * s * k, ctx->stream);
  f.V = DevBuf(sizeof(double) * n * k, ctx->stream);
  // Ubar = eigenvectors in descending order
  copy2d<double>(ctx, s, k, G.as<double>() + (s - 1) * s, 1, -s, f.U.as<double>(), 1, s);
  DevBuf dinv(sizeof(double) * k, ctx->stream), Us(sizeof(double) * s * k, ctx->stream);
  RNLA_CUDA(cudaMemcpyAsync(dinv.p, inv.data(), sizeof(double) * k, cudaMemcpyHostToDevice, ctx->stream));
  scale_cols_dev(ctx, s, k, f.U.as<double>(), dinv.as<double>(), Us.as<double>());
  gemm<double>(ctx, n, k, s, 1.0, B, s, 1, Us.as<double>(), 1, s, 0.0, f.V.as<double>(), 1, n);  // V = B' Ubar / sigma
  fix_column_signs(ctx, s, k, f.U.as<double>(), 1, s, f.V.as<double>(), 1, n, n, /*pair_cols=*/true);
  RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
  return f;
}

// Write a column-major fp64 device block (rows x cols, ld) into an output operand.
void store_block(rnla_ctx* ctx, const double* src, int64_t rows, int64_t cols, int64_t ld, OutMat& o) {
  if (o.dev.dtype == RNLA_F64)
    copy2d<double>(ctx, rows, cols, src, 1, ld, o.dev.as<double>(), o.dev.rs, o.dev.cs);
  else
    copy2d_cast<double, float>(ctx, rows, cols, src, 1, ld, o.dev.as<float>(), o.dev.rs, o.dev.cs);
}

// fp64 column-major working copy of any operand.
DevMat f64_colmajor(rnla_ctx* ctx, const rnla_mat* a) {
  DevMat d = to_device(ctx, a);
  if (d.dtype == RNLA_F64 && d.colmajor()) return d;
  return dense_copy(ctx, d, false, RNLA_F64);
}

// ---------------------------------------------------------------------------
// prototype_ksvd (src/randsvd.cpp:88-110) + power iterations
// ---------------------------------------------------------------------------
template <class T>
struct KsvdWork {
  // orth(Y) = thin_qr(Y).Q semantics (src/core.cpp:37-46). Tall-skinny Y is
  // orthonormalized by CholeskyQR2 (Gram -> Cholesky -> Y R^-1, twice; the
  // Gram of fp64 data on DMMA, of fp32 data on tcgen05), then the reference's
  // sign rule is applied, which makes Q unique: any stable orthonormalization
  // of the same range gives the same Q up to rounding (SURVEY A.6 measured
  // Householder vs CholeskyQR2 top-20 sigma within 1e-15). A Cholesky
  // breakdown (numerically rank-deficient Y) falls back to Householder.
  //
  // Row-sharded Y (`sharded`: this rank's consecutive row block, SURVEY
  // §8(e)): the Gram is allreduced (every rank then factors the identical
  // matrix and takes the same branch), the breakdown fallback is TSQR
  // (local Householder, allgather of the R factors, QR of the stack), and the
  // sign rule is decided on the global row order.
  static void orth(rnla_ctx* ctx, int64_t rows, int64_t cols, T* Y, bool sharded) {
    if (sharded) {
      if (cholqr2(ctx, rows, cols, Y, true)) return;
      tsqr(ctx, rows, cols, Y);
      return;
    }
    if (rows >= 4 * cols && cholqr2_fast(ctx, rows, cols, Y)) return;
    householder(ctx, rows, cols, Y);
  }

  // Intermediate orthonormalization of the power iteration (only
  // span(Q) matters there, not its sign convention or last-bit
  // orthonormality): ONE CholeskyQR pass, |Q'Q - I| ~ kappa(Y)^2 u (config 3:
  // kappa <= 19 per step, SURVEY hard part 7), with the full orth as the
  // breakdown fallback. The final Q before B = Q'A always takes the full orth.
  static void orth_light(rnla_ctx* ctx, int64_t rows, int64_t cols, T* Y, bool sharded) {
    if (sharded || rows < 4 * cols) return orth(ctx, rows, cols, Y, sharded);
    constexpr bool f64 = std::is_same<T, double>::value;
    DevBuf G(sizeof(double) * cols * cols, ctx->stream), Rinv(sizeof(double) * cols * cols, ctx->stream);
    DevBuf st(sizeof(int), ctx->stream), tmp(sizeof(T) * rows * cols, ctx->stream), Rt;
    if constexpr (!f64) Rt = DevBuf(sizeof(float) * cols * cols, ctx->stream);
    float* rt = f64 ? nullptr : Rt.as<float>();
    RNLA_CUDA(cudaMemsetAsync(st.p, 0, sizeof(int), ctx->stream));
    gram(ctx, rows, cols, Y, G.as<double>());
    const double thresh = f64 ? 1e-5 : 1e-2;
    if (cols <= kSmallCholMax)
      small_chol_inv<T>(ctx, cols, G.as<double>(), Rinv.as<double>(), rt, nullptr, rows, thresh, st.as<int>());
    else
      chol_inv_async<T>(ctx, cols, G.as<double>(), Rinv.as<double>(), rt, nullptr, rows, thresh, st.as<int>());
    if constexpr (f64)
      gemm<double>(ctx, rows, cols, cols, 1.0, Y, 1, rows, Rinv.as<double>(), 1, cols, 0.0, tmp.as<double>(), 1, rows);
    else
      gemm<float>(ctx, rows, cols, cols, 1.f, Y, 1, rows, rt, 1, cols, 0.f, tmp.as<float>(), 1, rows);
    int hs = 0;
    RNLA_CUDA(cudaMemcpyAsync(&hs, st.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
    if (hs & 3) return orth(ctx, rows, cols, Y, sharded);  // breakdown: Y untouched
    RNLA_CUDA(cudaMemcpyAsync(Y, tmp.p, sizeof(T) * rows * cols, cudaMemcpyDeviceToDevice, ctx->stream));
  }

  // G = Y'Y (fp64) of a column-major rows x cols Y.
  static void gram(rnla_ctx* ctx, int64_t rows, int64_t cols, const T* Y, double* G) {
    if constexpr (std::is_same<T, double>::value) {
      gemm<double>(ctx, cols, cols, rows, 1.0, Y, rows, 1, Y, 1, rows, 0.0, G, 1, cols);
    } else {
      DevBuf Gf(sizeof(float) * cols * cols, ctx->stream);
      gemm<float>(ctx, cols, cols, rows, 1.f, Y, rows, 1, Y, 1, rows, 0.f, Gf.as<float>(), 1, cols);
      copy2d_cast<float, double>(ctx, cols, cols, Gf.as<float>(), 1, cols, G, 1, cols);
    }
  }

  // CholeskyQR2 with both small factorizations on the device (small_chol_inv)
  // and one host round trip: pass 1 writes Q1 = Y R1^-1 to a scratch buffer,
  // pass 2 factors Q1'Q1 with the sign rule folded into R2^-1, and only when
  // both passes factored cleanly is Y overwritten by Q1 R2^-1. Otherwise Y is
  // untouched and the caller falls back to Householder.
  static bool cholqr2_fast(rnla_ctx* ctx, int64_t rows, int64_t cols, T* Y) {
    constexpr bool f64 = std::is_same<T, double>::value;
    const double thresh = f64 ? 1e-5 : 1e-2;
    DevBuf G(sizeof(double) * cols * cols, ctx->stream), Rinv(sizeof(double) * cols * cols, ctx->stream);
    DevBuf st(2 * sizeof(int), ctx->stream), tmp(sizeof(T) * rows * cols, ctx->stream), Rt;
    if constexpr (!f64) Rt = DevBuf(sizeof(float) * cols * cols, ctx->stream);
    float* rt = f64 ? nullptr : Rt.as<float>();
    auto apply = [&](const T* X, T* out) {  // out = X Rinv
      if constexpr (f64)
        gemm<double>(ctx, rows, cols, cols, 1.0, X, 1, rows, Rinv.as<double>(), 1, cols, 0.0, out, 1, rows);
      else
        gemm<float>(ctx, rows, cols, cols, 1.f, X, 1, rows, rt, 1, cols, 0.f, out, 1, rows);
    };
    // one-CTA factorization for narrow blocks, cuSOLVER potrf + trsm above
    auto factor = [&](const T* y0, int* status) {
      if (cols <= kSmallCholMax)
        small_chol_inv<T>(ctx, cols, G.as<double>(), Rinv.as<double>(), rt, y0, rows, thresh, status);
      else
        chol_inv_async<T>(ctx, cols, G.as<double>(), Rinv.as<double>(), rt, y0, rows, thresh, status);
    };
    RNLA_CUDA(cudaMemsetAsync(st.p, 0, 2 * sizeof(int), ctx->stream));
    gram(ctx, rows, cols, Y, G.as<double>());
    trace_mark(ctx, "cholqr2: gram 1");
    factor(nullptr, st.as<int>());
    trace_mark(ctx, "cholqr2: chol+inv 1");
    apply(Y, tmp.as<T>());
    trace_mark(ctx, "cholqr2: Y R^-1");
    gram(ctx, rows, cols, tmp.as<T>(), G.as<double>());
    trace_mark(ctx, "cholqr2: gram 2");
    factor(tmp.as<T>(), st.as<int>() + 1);
    int hs[2] = {0, 0};
    RNLA_CUDA(cudaMemcpyAsync(hs, st.p, sizeof hs, cudaMemcpyDeviceToHost, ctx->stream));
    RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
    trace_mark(ctx, "cholqr2: chol+inv 2");
    if ((hs[0] & 3) || (hs[1] & 3)) return false;
    apply(tmp.as<T>(), Y);
    trace_mark(ctx, "cholqr2: Q1 R2^-1");
    if (hs[1] & 4) sign_fix(ctx, rows, cols, Y);
    return true;
  }

  // Host-round-trip-free variants for the speculative pipeline of
  // prototype_ksvd_async: every factorization writes its status word to its
  // own slot and the caller reads all of them once at the end (a breakdown
  // there reruns the call on the checked path above).
  static void factor_async(rnla_ctx* ctx, int64_t rows, int64_t cols, double* G, double* Rinv, float* rt, const T* y0,
                           int* status) {
    constexpr bool f64 = std::is_same<T, double>::value;
    const double thresh = f64 ? 1e-5 : 1e-2;
    if (cols <= kSmallCholMax)
      small_chol_inv<T>(ctx, cols, G, Rinv, rt, y0, rows, thresh, status);
    else
      chol_inv_async<T>(ctx, cols, G, Rinv, rt, y0, rows, thresh, status);
  }
  static void apply_rinv(rnla_ctx* ctx, int64_t rows, int64_t cols, const T* X, const double* Rinv, const float* rt,
                         T* out) {
    if constexpr (std::is_same<T, double>::value)
      gemm<double>(ctx, rows, cols, cols, 1.0, X, 1, rows, Rinv, 1, cols, 0.0, out, 1, rows);
    else
      gemm<float>(ctx, rows, cols, cols, 1.f, X, 1, rows, rt, 1, cols, 0.f, out, 1, rows);
  }
  // one CholeskyQR pass (orth_light semantics): y <- Y R^-1, the result lands in
  // `spare` and the two pointers swap
  static void orth1_async(rnla_ctx* ctx, int64_t rows, int64_t cols, T*& y, T*& spare, int* status) {
    DevBuf G(sizeof(double) * cols * cols, ctx->stream), Rinv(sizeof(double) * cols * cols, ctx->stream), Rt;
    if constexpr (!std::is_same<T, double>::value) Rt = DevBuf(sizeof(float) * cols * cols, ctx->stream);
    gram(ctx, rows, cols, y, G.as<double>());
    factor_async(ctx, rows, cols, G.as<double>(), Rinv.as<double>(), Rt.as<float>(), nullptr, status);
    apply_rinv(ctx, rows, cols, y, Rinv.as<double>(), Rt.as<float>(), spare);
    std::swap(y, spare);
  }
  // CholeskyQR2 with the reference's sign rule folded into R2^-1 (orth
  // semantics): y <- Q in place, `spare` is scratch. status[0], status[1]: the
  // two factorizations (bit 4 of status[1]: sign undecidable from row 0).
  static void orth2_async(rnla_ctx* ctx, int64_t rows, int64_t cols, T* y, T* spare, int* status) {
    DevBuf G(sizeof(double) * cols * cols, ctx->stream), Rinv(sizeof(double) * cols * cols, ctx->stream), Rt;
    if constexpr (!std::is_same<T, double>::value) Rt = DevBuf(sizeof(float) * cols * cols, ctx->stream);
    gram(ctx, rows, cols, y, G.as<double>());
    factor_async(ctx, rows, cols, G.as<double>(), Rinv.as<double>(), Rt.as<float>(), nullptr, status);
    apply_rinv(ctx, rows, cols, y, Rinv.as<double>(), Rt.as<float>(), spare);
    gram(ctx, rows, cols, spare, G.as<double>());
    factor_async(ctx, rows, cols, G.as<double>(), Rinv.as<double>(), Rt.as<float>(), spare, status + 1);
    apply_rinv(ctx, rows, cols, spare, Rinv.as<double>(), Rt.as<float>(), y);
  }

  static void tsqr(rnla_ctx* ctx, int64_t rows, int64_t cols, T* Y) {
    const int W = ctx->world;
    DevBuf w(sizeof(double) * rows * cols, ctx->stream), r(sizeof(double) * cols * cols, ctx->stream),
        all(sizeof(double) * W * cols * cols, ctx->stream), stack(sizeof(double) * W * cols * cols, ctx->stream),
        rr(sizeof(double) * cols * cols, ctx->stream), qw(sizeof(double) * rows * cols, ctx->stream);
    if constexpr (std::is_same<T, double>::value)
      RNLA_CUDA(cudaMemcpyAsync(w.p, Y, sizeof(double) * rows * cols, cudaMemcpyDeviceToDevice, ctx->stream));
    else
      copy2d_cast<float, double>(ctx, rows, cols, Y, 1, rows, w.as<double>(), 1, rows);
    thin_qr_dev(ctx, rows, cols, w.as<double>(), r.as<double>());
    allgather_blocks(ctx, r.p, all.p, (size_t)(cols * cols), RNLA_F64);
    for (int q = 0; q < W; ++q)  // stacked (W cols) x cols, rank blocks in order
      copy2d<double>(ctx, cols, cols, all.as<double>() + (int64_t)q * cols * cols, 1, cols,
                     stack.as<double>() + (int64_t)q * cols, 1, (int64_t)W * cols);
    thin_qr_dev(ctx, (int64_t)W * cols, cols, stack.as<double>(), rr.as<double>());
    gemm<double>(ctx, rows, cols, cols, 1.0, w.as<double>(), 1, rows, stack.as<double>() + (int64_t)ctx->rank * cols, 1,
                 (int64_t)W * cols, 0.0, qw.as<double>(), 1, rows);
    if constexpr (std::is_same<T, double>::value)
      RNLA_CUDA(cudaMemcpyAsync(Y, qw.p, sizeof(double) * rows * cols, cudaMemcpyDeviceToDevice, ctx->stream));
    else
      copy2d_cast<double, float>(ctx, rows, cols, qw.as<double>(), 1, rows, Y, 1, rows);
    fix_column_signs_sharded<T>(ctx, rows, cols, Y, 1, rows, nullptr, 0, 0, 0, false);
  }

  // Y is overwritten only after both passes factored cleanly: pass 0 writes
  // Q1 to a scratch buffer and pass 1 reads it, so a breakdown in either pass
  // leaves the original Y for the TSQR / Householder fallback.
  static bool cholqr2(rnla_ctx* ctx, int64_t rows, int64_t cols, T* Y, bool sharded) {
    DevBuf G(sizeof(double) * cols * cols, ctx->stream), Rinv(sizeof(double) * cols * cols, ctx->stream);
    DevBuf tmp(sizeof(T) * rows * cols, ctx->stream), q1(sizeof(T) * rows * cols, ctx->stream), Rt;
    if constexpr (!std::is_same<T, double>::value) Rt = DevBuf(sizeof(T) * cols * cols, ctx->stream);
    bool signed_ok = false;
    for (int pass = 0; pass < 2; ++pass) {
      const T* X = pass == 0 ? Y : q1.as<T>();
      T* out = pass == 0 ? q1.as<T>() : tmp.as<T>();
      if constexpr (std::is_same<T, double>::value) {
        gemm<double>(ctx, cols, cols, rows, 1.0, X, rows, 1, X, 1, rows, 0.0, G.as<double>(), 1, cols);
      } else {
        DevBuf Gf(sizeof(float) * cols * cols, ctx->stream);
        gemm<float>(ctx, cols, cols, rows, 1.f, X, rows, 1, X, 1, rows, 0.f, Gf.as<float>(), 1, cols);
        copy2d_cast<float, double>(ctx, cols, cols, Gf.as<float>(), 1, cols, G.as<double>(), 1, cols);
      }
      if (sharded) allreduce_sum(ctx, G.p, (size_t)(cols * cols), RNLA_F64);
      if (!cholesky_upper(ctx, cols, G.as<double>())) return false;
      if (!diag_ratio_ok(ctx, cols, G.as<double>(), std::is_same<T, double>::value ? 1e-5 : 1e-2)) return false;
      upper_inverse(ctx, cols, G.as<double>(), Rinv.as<double>());
      // sign rule folded into the last R^-1: no extra pass over Q
      if (pass == 1 && !sharded) signed_ok = presign_upper_inverse<T>(ctx, cols, X, rows, Rinv.as<double>());
      if constexpr (std::is_same<T, double>::value) {
        gemm<double>(ctx, rows, cols, cols, 1.0, X, 1, rows, Rinv.as<double>(), 1, cols, 0.0, out, 1, rows);
      } else {
        copy2d_cast<double, float>(ctx, cols, cols, Rinv.as<double>(), 1, cols, Rt.as<float>(), 1, cols);
        gemm<float>(ctx, rows, cols, cols, 1.f, X, 1, rows, Rt.as<float>(), 1, cols, 0.f, out, 1, rows);
      }
    }
    RNLA_CUDA(cudaMemcpyAsync(Y, tmp.p, sizeof(T) * rows * cols, cudaMemcpyDeviceToDevice, ctx->stream));
    if (sharded)
      fix_column_signs_sharded<T>(ctx, rows, cols, Y, 1, rows, nullptr, 0, 0, 0, false);
    else if (!signed_ok)
      sign_fix(ctx, rows, cols, Y);
    return true;
  }

  static void sign_fix(rnla_ctx* ctx, int64_t rows, int64_t cols, T* Y) {
    if constexpr (std::is_same<T, double>::value) {
      fix_column_signs(ctx, rows, cols, Y, 1, rows, nullptr, 0, 0, 0, true);
    } else {
      fix_column_signs_f32(ctx, rows, cols, Y, 1, rows);
    }
  }

  static void householder(rnla_ctx* ctx, int64_t rows, int64_t cols, T* Y) {
    DevBuf w(sizeof(double) * rows * cols, ctx->stream), r(sizeof(double) * cols * cols, ctx->stream);
    if constexpr (std::is_same<T, double>::value) {
      RNLA_CUDA(cudaMemcpyAsync(w.p, Y, sizeof(double) * rows * cols, cudaMemcpyDeviceToDevice, ctx->stream));
      thin_qr_dev(ctx, rows, cols, w.as<double>(), r.as<double>());
      RNLA_CUDA(cudaMemcpyAsync(Y, w.p, sizeof(double) * rows * cols, cudaMemcpyDeviceToDevice, ctx->stream));
    } else {
      copy2d_cast<float, double>(ctx, rows, cols, Y, 1, rows, w.as<double>(), 1, rows);
      thin_qr_dev(ctx, rows, cols, w.as<double>(), r.as<double>());
      copy2d_cast<double, float>(ctx, rows, cols, w.as<double>(), 1, rows, Y, 1, rows);
    }
  }
};

// Block subspace iteration with Rayleigh-Ritz for the top-k eigenpairs of a
// symmetric A (the Nystrom approx_eig subproblem M = T'(C'C)T, SURVEY §8(a)
// row 20; the reference takes them from a full BDCSVD, src/spsd.cpp:257-265).
// Block b = max(2k, k + 32) (k + 32 for values only): the top-k Ritz pairs converge at the rate
// lam_{b+1} / lam_k per iteration (config 4: 0.065), and a cluster straddling
// k (config 4: lam_64 / lam_65 = 1.0036) is resolved by the Rayleigh-Ritz step
// inside the block rather than by the iteration. An iteration is one n x n x b
// DMMA GEMM and one CholeskyQR pass; a Rayleigh-Ritz checkpoint (b x b eig,
// ~2 ms of cuSOLVER latency at b = 128) runs after two iterations and then
// after as many more as the Ritz values predict the residual needs. Converged
// when every top-k residual |A v - theta v| <= 1e-12 theta_1.
// values_only: the caller needs the eigenvalues alone; they converge with the
// square of the residual (|theta - lam| <= r^2 / gap), so a residual of
// 1e-9 theta_1 already gives fp64-level values, and the first Rayleigh-Ritz
// checkpoint is placed where the config-4 rate (0.065 per iteration) reaches it.
bool eig_top_subspace(rnla_ctx* ctx, int64_t n, const double* A, int64_t k, double* lam, double* V,
                      bool values_only) {
  // Block: 2k for eigenvectors (faster rate lam_{b+1} / lam_k); k + 32 for
  // values only, where the cheaper b x b Rayleigh-Ritz wins (config 4, k = 64:
  // b = 80 / 96 / 112 / 128 -> 10.6 / 10.6 / 11.9 / 12.2 ms, 5 iterations each).
  const int64_t b = values_only ? k + 32 : std::max<int64_t>(2 * k, k + 32);
  if (k < 1 || 2 * b > n || std::getenv("RNLA_EIG_DIRECT")) return false;
  constexpr int kMaxIt = 80;
  const double kTol = values_only ? 1e-9 : 1e-12;
  DevBuf Q(sizeof(double) * n * b, ctx->stream), Y(sizeof(double) * n * b, ctx->stream),
      H(sizeof(double) * b * b, ctx->stream), Hs(sizeof(double) * b * b, ctx->stream),
      th(sizeof(double) * b, ctx->stream), Zk(sizeof(double) * b * k, ctx->stream),
      YZ(sizeof(double) * n * k, ctx->stream), VZ(sizeof(double) * n * k, ctx->stream),
      thd(sizeof(double) * k, ctx->stream), res(sizeof(double) * k, ctx->stream);
  hash_uniform_dev(ctx, n * b, 0x6a09e667f3bcc909ull, Y.as<double>());
  std::vector<double> ht((size_t)b), hr((size_t)k), td((size_t)k);
  int next_rr = values_only ? 5 : 2, rr_count = 0;
  // Between checkpoints the CholeskyQR passes run without host round trips
  // (one-CTA Cholesky + inverse, status words read at the next checkpoint);
  // a breakdown there abandons this route (the caller falls back).
  const bool async_qr = b <= kSmallCholMax && !std::getenv("RNLA_EIG_SYNC_QR");
  DevBuf Gq(sizeof(double) * b * b, ctx->stream), Rq(sizeof(double) * b * b, ctx->stream),
      qst(sizeof(int) * (kMaxIt + 1), ctx->stream);
  if (async_qr) RNLA_CUDA(cudaMemsetAsync(qst.p, 0, sizeof(int) * (kMaxIt + 1), ctx->stream));
  int nq = 0;
  for (int it = 0; it < kMaxIt; ++it) {
    // Q = orth(Y) (CholeskyQR2 + Householder fallback at checkpoints, one
    // CholeskyQR pass in between); Y = A Q
    const bool rr = it == next_rr;
    if (!rr && async_qr) {
      gemm<double>(ctx, b, b, n, 1.0, Y.as<double>(), n, 1, Y.as<double>(), 1, n, 0.0, Gq.as<double>(), 1, b);
      small_chol_inv<double>(ctx, b, Gq.as<double>(), Rq.as<double>(), nullptr, nullptr, n, 0.0,
                             qst.as<int>() + nq++);
      gemm<double>(ctx, n, b, b, 1.0, Y.as<double>(), 1, n, Rq.as<double>(), 1, b, 0.0, Q.as<double>(), 1, n);
    } else {
      RNLA_CUDA(cudaMemcpyAsync(Q.p, Y.p, sizeof(double) * n * b, cudaMemcpyDeviceToDevice, ctx->stream));
      if (rr || !cholqr_inplace(ctx, n, b, Q.as<double>())) {
        RNLA_CUDA(cudaMemcpyAsync(Q.p, Y.p, sizeof(double) * n * b, cudaMemcpyDeviceToDevice, ctx->stream));
        KsvdWork<double>::orth(ctx, n, b, Q.as<double>(), false);
      }
    }
    if (rr && nq > 0) {  // the passes since the last checkpoint factored cleanly?
      std::vector<int> hq((size_t)nq);
      RNLA_CUDA(cudaMemcpyAsync(hq.data(), qst.p, sizeof(int) * nq, cudaMemcpyDeviceToHost, ctx->stream));
      RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
      for (int v : hq)
        if (v & 1) return false;
    }
    gemm<double>(ctx, n, b, n, 1.0, A, 1, n, Q.as<double>(), 1, n, 0.0, Y.as<double>(), 1, n);
    trace_mark(ctx, rr ? "eig_top_subspace: orth + A Q (RR step)" : "eig_top_subspace: cholqr + A Q");
    if (!rr) continue;
    ++rr_count;
    // Rayleigh-Ritz: H = Q'AQ = (Z, theta); top-k Ritz vectors Q Z_k, images Y Z_k
    gemm<double>(ctx, b, b, n, 1.0, Q.as<double>(), n, 1, Y.as<double>(), 1, n, 0.0, H.as<double>(), 1, b);
    symmetrize(ctx, b, H.as<double>(), Hs.as<double>());
    trace_mark(ctx, "eig_top_subspace: H = Q'AQ");
    const double* zfull = H.as<double>();  // all b Ritz vectors (column order irrelevant)
    if (eig_sym_small_desc(ctx, b, Hs.as<double>(), th.as<double>(), H.as<double>())) {  // descending
      RNLA_CUDA(cudaMemcpyAsync(ht.data(), th.p, sizeof(double) * b, cudaMemcpyDeviceToHost, ctx->stream));
      RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
      std::reverse(ht.begin(), ht.end());  // ascending, as below
      copy2d<double>(ctx, b, k, H.as<double>(), 1, b, Zk.as<double>(), 1, b);
    } else {
      zfull = Hs.as<double>();
      eig_sym(ctx, b, Hs.as<double>(), th.as<double>());  // ascending
      RNLA_CUDA(cudaMemcpyAsync(ht.data(), th.p, sizeof(double) * b, cudaMemcpyDeviceToHost, ctx->stream));
      RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
      copy2d<double>(ctx, b, k, Hs.as<double>() + (b - 1) * b, 1, -b, Zk.as<double>(), 1, b);
    }
    trace_mark(ctx, "eig_top_subspace: eig(H)");
    for (int64_t t = 0; t < k; ++t) td[(size_t)t] = ht[(size_t)(b - 1 - t)];
    gemm<double>(ctx, n, k, b, 1.0, Q.as<double>(), 1, n, Zk.as<double>(), 1, b, 0.0, VZ.as<double>(), 1, n);
    gemm<double>(ctx, n, k, b, 1.0, Y.as<double>(), 1, n, Zk.as<double>(), 1, b, 0.0, YZ.as<double>(), 1, n);
    RNLA_CUDA(cudaMemcpyAsync(thd.p, td.data(), sizeof(double) * k, cudaMemcpyHostToDevice, ctx->stream));
    ritz_residual_dev(ctx, n, k, YZ.as<double>(), VZ.as<double>(), thd.as<double>(), res.as<double>());
    RNLA_CUDA(cudaMemcpyAsync(hr.data(), res.p, sizeof(double) * k, cudaMemcpyDeviceToHost, ctx->stream));
    RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
    const double top = std::abs(td[0]);
    if (!(top > 0.0)) return false;
    double worst = 0.0;
    for (int64_t t = 0; t < k; ++t) worst = std::max(worst, std::sqrt(hr[(size_t)t]) / top);
    if (worst <= kTol) {
      std::copy(td.begin(), td.end(), lam);
      RNLA_CUDA(cudaMemcpyAsync(V, VZ.p, sizeof(double) * n * k, cudaMemcpyDeviceToDevice, ctx->stream));
      RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
      char label[96];
      std::snprintf(label, sizeof label, "eig_top_subspace: %d iterations, %d Rayleigh-Ritz", it, rr_count);
      trace_mark(ctx, label);
      return true;
    }
    // continue from the Ritz basis: Y <- Y Z spans the same space with its
    // columns along the current eigenvector estimates, so the next
    // Rayleigh-Ritz matrix starts nearly diagonal (few Jacobi sweeps)
    gemm<double>(ctx, n, b, b, 1.0, Y.as<double>(), 1, n, zfull, 1, b, 0.0, Q.as<double>(), 1, n);
    std::swap(Q, Y);
    // iterations to the tolerance at the rate theta_b / theta_k (the Ritz
    // values under-estimate lam_b, so cap the rate from below and re-check)
    const double rate = std::min(0.9, std::max(0.02, std::abs(ht[0]) / std::abs(td[(size_t)k - 1])));
    const double need = std::log(kTol / worst) / std::log(rate);
    next_rr = it + std::max(1, std::min(20, (int)std::ceil(need)));
  }
  return false;
}

// Gram-route core SVD from the eigenpairs of B B' (s x s), lam/Z descending
// (desc = 1, Jacobi) or ascending (desc = 0, syevd): for the k leading pairs
// sigma_i = sqrt(lam_i), Ubar(:, i) = z_i and Us(:, i) = z_i / sigma_i.
// *status = 1 when the route does not apply (lam_1 <= 0 or lam_k <= 1e-6 lam_1,
// topk_svd_wide's rule).
static __global__ void gram_svd_post_kernel(int64_t s, int64_t k, int desc, const double* __restrict__ lam,
                                     const double* __restrict__ Z, double* sigma, double* Ubar, double* Us,
                                     int* status) {
  const double l1 = desc ? lam[0] : lam[s - 1], lk = desc ? lam[k - 1] : lam[s - k];
  if (blockIdx.x == 0 && threadIdx.x == 0) *status = (l1 > 0.0 && lk > 1e-6 * l1) ? 0 : 1;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < s * k; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % s, j = e / s, jj = desc ? j : s - 1 - j;
    const double sg = sqrt(fmax(lam[jj], 0.0)), z = Z[i + jj * s];
    Ubar[e] = z;
    Us[e] = z / sg;
    if (i == 0) sigma[j] = sg;
  }
}

// prototype_ksvd with power iterations as one speculative device pipeline:
// no host round trip until the end. The orthonormalizations run as in the
// checked path (one CholeskyQR pass in the power steps, CholeskyQR2 + sign rule
// for the final Q) and the core SVD takes the Gram route (topk_svd_wide), but
// their breakdown tests -- Cholesky failure, diagonal ratio, an undecidable
// sign, the Gram-route condition, eigensolver convergence -- only write status
// words, read once together with sigma. Any flag returns false and the caller
// reruns the checked path, so results are identical to it whenever it
// returns true. Config 0 had six host round trips per call.
//
// With the one-CTA Jacobi core (s <= 32) the whole pipeline is captured once
// per argument signature into a CUDA graph (cached in the context) and
// replayed: ~35 launches and their stream-ordered allocations become one
// graph launch. U, V, sigma and the status words land in buffers the graph
// owns; the per-call work outside it is two copies into the outputs and one
// device-to-host read.
struct KsvdAsyncOut {
  double *U64, *Vd, *sig;
  int* st;
  int slots = 0, eig_slot = 0, desc = 1;
};

template <class T>
void prototype_ksvd_async_body(rnla_ctx* ctx, const T* Ap, int64_t a_rs, int64_t a_cs, int64_t m, int64_t n,
                               int64_t kk, int64_t s, const T* omega, int32_t q, KsvdAsyncOut& o) {
  constexpr bool f64 = std::is_same<T, double>::value;
  RNLA_CUDA(cudaMemsetAsync(o.st, 0, sizeof(int) * (2 * q + 4), ctx->stream));
  int slot = 0;
  DevBuf Y0(sizeof(T) * m * s, ctx->stream), Y1(sizeof(T) * m * s, ctx->stream);
  DevBuf Z0(sizeof(T) * n * s, ctx->stream), Z1(sizeof(T) * n * s, ctx->stream);
  T *y = Y0.as<T>(), *ys = Y1.as<T>(), *z = Z0.as<T>(), *zs = Z1.as<T>();
  gemm<T>(ctx, m, s, n, T(1), Ap, a_rs, a_cs, omega, 1, n, T(0), y, 1, m);
  trace_mark(ctx, "ksvd (async): Y = A S");
  for (int32_t it = 0; it < q; ++it) {
    KsvdWork<T>::orth1_async(ctx, m, s, y, ys, o.st + slot++);
    gemm<T>(ctx, n, s, m, T(1), Ap, a_cs, a_rs, y, 1, m, T(0), z, 1, n);
    KsvdWork<T>::orth1_async(ctx, n, s, z, zs, o.st + slot++);
    gemm<T>(ctx, m, s, n, T(1), Ap, a_rs, a_cs, z, 1, n, T(0), y, 1, m);
  }
  trace_mark(ctx, "ksvd (async): power iterations");
  KsvdWork<T>::orth2_async(ctx, m, s, y, ys, o.st + slot);
  slot += 2;
  trace_mark(ctx, "ksvd (async): orth(Y)");
  // B' = A'Q, stored as B (s x n, column-major)
  DevBuf B(sizeof(T) * s * n, ctx->stream), B64;
  gemm<T>(ctx, n, s, m, T(1), Ap, a_cs, a_rs, y, 1, m, T(0), B.as<T>(), s, 1);
  const double* Bp;
  if constexpr (f64) {
    Bp = B.as<double>();
  } else {
    B64 = DevBuf(sizeof(double) * s * n, ctx->stream);
    copy2d_cast<float, double>(ctx, s, n, B.as<float>(), 1, s, B64.as<double>(), 1, s);
    Bp = B64.as<double>();
  }
  trace_mark(ctx, "ksvd (async): B = Q' A");
  DevBuf G(sizeof(double) * s * s, ctx->stream), lam(sizeof(double) * s, ctx->stream),
      Zd(sizeof(double) * s * s, ctx->stream);
  gemm<double>(ctx, s, s, n, 1.0, Bp, 1, s, Bp, s, 1, 0.0, G.as<double>(), 1, s);
  o.eig_slot = slot++;
  o.desc = 1;
  if (!eig_small_jacobi_async(ctx, s, G.as<double>(), lam.as<double>(), Zd.as<double>(), o.st + o.eig_slot) &&
      !eig_tri_async(ctx, s, G.as<double>(), lam.as<double>(), Zd.as<double>(), o.st + o.eig_slot)) {
    o.desc = 0;
    RNLA_CUDA(cudaMemcpyAsync(Zd.p, G.p, sizeof(double) * s * s, cudaMemcpyDeviceToDevice, ctx->stream));
    eig_sym_async(ctx, s, Zd.as<double>(), lam.as<double>(), o.st + o.eig_slot);
  }
  DevBuf Ub(sizeof(double) * s * kk, ctx->stream), Us(sizeof(double) * s * kk, ctx->stream);
  gram_svd_post_kernel<<<1, 256, 0, ctx->stream>>>(s, kk, o.desc, lam.as<double>(), Zd.as<double>(), o.sig,
                                                   Ub.as<double>(), Us.as<double>(), o.st + slot++);
  RNLA_CUDA(cudaGetLastError());
  note_launch(ctx);
  gemm<double>(ctx, n, kk, s, 1.0, Bp, s, 1, Us.as<double>(), 1, s, 0.0, o.Vd, 1, n);  // V = B' Ubar / sigma
  fix_column_signs(ctx, s, kk, Ub.as<double>(), 1, s, o.Vd, 1, n, n, /*pair_cols=*/true);
  trace_mark(ctx, "ksvd (async): small SVD");
  if constexpr (f64) {
    gemm<double>(ctx, m, kk, s, 1.0, y, 1, m, Ub.as<double>(), 1, s, 0.0, o.U64, 1, m);
  } else {
    DevBuf uf(sizeof(float) * s * kk, ctx->stream), Uf(sizeof(float) * m * kk, ctx->stream);
    copy2d_cast<double, float>(ctx, s, kk, Ub.as<double>(), 1, s, uf.as<float>(), 1, s);
    gemm<float>(ctx, m, kk, s, 1.f, y, 1, m, uf.as<float>(), 1, s, 0.f, Uf.as<float>(), 1, m);
    copy2d_cast<float, double>(ctx, m, kk, Uf.as<float>(), 1, m, o.U64, 1, m);
  }
  o.slots = slot;
}

template <class T>
bool prototype_ksvd_async(rnla_ctx* ctx, const T* Ap, int64_t a_rs, int64_t a_cs, int64_t m, int64_t n, int64_t k,
                          int64_t s, uint64_t seed, int32_t q, bool a_stable, OutMat& uo, OutMat& vo, double* sv_out,
                          int64_t* rank_out, int32_t* passes_out) {
  constexpr bool f64 = std::is_same<T, double>::value;
  if (m < 4 * s || n < 4 * s || s > 512 || q > 16 || std::getenv("RNLA_KSVD_SYNC")) return false;
  const int64_t kk = std::min(k, s);
  const T* omega = gaussian_operator(ctx, n, s, seed, f64 ? RNLA_F64 : RNLA_F32).data.template as<T>();
  KsvdAsyncOut o{};
  CachedGraph* cg = nullptr;
  std::unique_ptr<CachedGraph> own;
  // graphs only for the caller's own device pointer (a host input is staged
  // through a fresh device buffer whose address is not stable across calls)
  const bool use_graph = a_stable && s <= 32 && !std::getenv("RNLA_NO_GRAPH");
  if (use_graph) {
    char key[256];
    std::snprintf(key, sizeof key, "ksvd:%d:%p:%lld:%lld:%lld:%lld:%lld:%lld:%p:%d", f64 ? 64 : 32, (const void*)Ap,
                  (long long)a_rs, (long long)a_cs, (long long)m, (long long)n, (long long)kk, (long long)s,
                  (const void*)omega, (int)q);
    auto it = ctx->graphs.find(key);
    if (it != ctx->graphs.end()) {
      cg = it->second.get();
    } else {
      if (ctx->graphs.size() >= 32) {  // bounded cache: drop all (stream-ordered with this call)
        RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
        ctx->graphs.clear();
      }
      own.reset(new CachedGraph());
      for (size_t bytes : {sizeof(double) * m * kk, sizeof(double) * n * kk, sizeof(double) * kk, sizeof(int) * 64}) {
        void* p = nullptr;
        RNLA_CUDA(cudaMalloc(&p, std::max<size_t>(bytes, 16)));
        own->bufs.push_back(p);
      }
      KsvdAsyncOut oc{static_cast<double*>(own->bufs[0]), static_cast<double*>(own->bufs[1]),
                      static_cast<double*>(own->bufs[2]), static_cast<int*>(own->bufs[3])};
      const int64_t launches0 = ctx->launches;
      cudaGraph_t graph = nullptr;
      RNLA_CUDA(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
      ctx->capturing = true;
      try {
        prototype_ksvd_async_body<T>(ctx, Ap, a_rs, a_cs, m, n, kk, s, omega, q, oc);
      } catch (...) {
        ctx->capturing = false;
        cudaStreamEndCapture(ctx->stream, &graph);
        if (graph) cudaGraphDestroy(graph);
        throw;
      }
      ctx->capturing = false;
      RNLA_CUDA(cudaStreamEndCapture(ctx->stream, &graph));
      ctx->launches = launches0;
      const cudaError_t ie = cudaGraphInstantiate(&own->exec, graph, 0);
      size_t nn = 0;
      cudaGraphGetNodes(graph, nullptr, &nn);
      std::vector<cudaGraphNode_t> nodes(nn);
      if (nn) cudaGraphGetNodes(graph, nodes.data(), &nn);
      for (auto nd : nodes) {
        cudaGraphNodeType ty;
        if (cudaGraphNodeGetType(nd, &ty) == cudaSuccess && ty == cudaGraphNodeTypeKernel) ++own->kernels;
      }
      cudaGraphDestroy(graph);
      RNLA_CUDA(ie);
      own->meta = {oc.slots, oc.eig_slot, oc.desc};
      cg = own.get();
      ctx->graphs.emplace(key, std::move(own));
    }
    o = KsvdAsyncOut{static_cast<double*>(cg->bufs[0]), static_cast<double*>(cg->bufs[1]),
                     static_cast<double*>(cg->bufs[2]), static_cast<int*>(cg->bufs[3]), (int)cg->meta[0],
                     (int)cg->meta[1], (int)cg->meta[2]};
    RNLA_CUDA(cudaGraphLaunch(cg->exec, ctx->stream));
    note_launch(ctx, cg->kernels);
  }
  DevBuf U64, Vd, sig, st;
  if (!cg) {
    U64 = DevBuf(sizeof(double) * m * kk, ctx->stream);
    Vd = DevBuf(sizeof(double) * n * kk, ctx->stream);
    sig = DevBuf(sizeof(double) * kk, ctx->stream);
    st = DevBuf(sizeof(int) * 64, ctx->stream);
    o = KsvdAsyncOut{U64.as<double>(), Vd.as<double>(), sig.as<double>(), st.as<int>()};
    prototype_ksvd_async_body<T>(ctx, Ap, a_rs, a_cs, m, n, kk, s, omega, q, o);
  }
  store_block(ctx, o.U64, m, kk, m, uo);
  store_block(ctx, o.Vd, n, kk, n, vo);
  std::vector<int> hs((size_t)o.slots);
  std::vector<double> hsig((size_t)kk);
  RNLA_CUDA(cudaMemcpyAsync(hs.data(), o.st, sizeof(int) * o.slots, cudaMemcpyDeviceToHost, ctx->stream));
  RNLA_CUDA(cudaMemcpyAsync(hsig.data(), o.sig, sizeof(double) * kk, cudaMemcpyDeviceToHost, ctx->stream));
  RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
  trace_mark(ctx, "ksvd (async): U = Q Ubar, stores, status");
  for (int i = 0; i < o.slots; ++i) {
    const int v = (i == o.eig_slot && o.desc) ? (hs[(size_t)i] & 255) : hs[(size_t)i];
    if (v != 0) {
      if (std::getenv("RNLA_TRACE")) std::fprintf(stderr, "[rnla] ksvd (async): status slot %d = %d, checked path\n", i, v);
      return false;
    }
  }
  for (int64_t i = 0; i < kk; ++i) sv_out[i] = hsig[(size_t)i];
  *rank_out = kk;
  *passes_out = 2 + 2 * q;
  return true;
}

template <class T>
void prototype_ksvd_impl(rnla_ctx* ctx, const rnla_mat* a, int64_t k, int64_t s, uint64_t seed,
                         const rnla_sketch_spec* spec, int32_t q, const rnla_mat* u_out, double* sv_out,
                         const rnla_mat* v_out, int64_t* rank_out, int32_t* passes_out, double* error_fro) {
  const int64_t m = a->rows, n = a->cols;
  DevMat A = to_device(ctx, a);
  const T* Ap = A.as<T>();
  OutMat uo(ctx, u_out, m, k, "prototype_ksvd: U", false), vo(ctx, v_out, n, k, "prototype_ksvd: V", false);
  rnla_sketch_spec local{};
  if (spec) local = *spec;
  else { local.kind = RNLA_SKETCH_GAUSSIAN; local.seed = seed; }
  local.s = s;
  // Row-sharded A: U comes back as this rank's rows,
  // sigma and V replicated.
  const bool sharded = is_sharded(ctx);
  require(!sharded || local.kind == RNLA_SKETCH_GAUSSIAN,
          "prototype_ksvd: row-sharded contexts support the Gaussian test matrix");
  require(!sharded || m >= s, "prototype_ksvd: every row shard needs at least s rows");
  if (!sharded && local.kind == RNLA_SKETCH_GAUSSIAN && !error_fro &&
      prototype_ksvd_async<T>(ctx, Ap, A.rs, A.cs, m, n, k, s, local.seed, q, a->on_device != 0, uo, vo, sv_out,
                              rank_out, passes_out)) {
    uo.finish(ctx);
    vo.finish(ctx);
    return;
  }
  int passes = 0;
  // pass 1: Y = A S (m x s, column-major)
  DevBuf Y(sizeof(T) * m * s, ctx->stream);
  ++passes;
  if (local.kind == RNLA_SKETCH_GAUSSIAN) {
    const DenseOperator& g = gaussian_operator(ctx, n, s, local.seed, std::is_same<T, double>::value ? RNLA_F64 : RNLA_F32);
    gemm<T>(ctx, m, s, n, T(1), Ap, A.rs, A.cs, g.data.as<T>(), 1, n, T(0), Y.as<T>(), 1, m);
  } else {
    rnla_mat ym{Y.p, m, s, 1, m, a->dtype, 1};
    rnla_mat am{A.p, m, n, A.rs, A.cs, a->dtype, 1};
    int64_t cols = 0;
    const rnla_status st = rnla_apply_sketch(ctx, &am, &local, &ym, &cols);
    if (st != RNLA_OK) throw InvalidArgument(rnla_last_error());
    require(cols == s, "prototype_ksvd: sketch returned a different width");
  }
  trace_mark(ctx, "ksvd: Y = A S");
  const int dt = std::is_same<T, double>::value ? RNLA_F64 : RNLA_F32;
  DevBuf Z(sizeof(T) * n * s, ctx->stream);
  for (int32_t it = 0; it < q; ++it) {
    KsvdWork<T>::orth_light(ctx, m, s, Y.as<T>(), sharded);
    trace_mark(ctx, "ksvd: orth(Y)");
    // Z = orth(A' Q): n x s (a sum over row shards)
    gemm<T>(ctx, n, s, m, T(1), Ap, A.cs, A.rs, Y.as<T>(), 1, m, T(0), Z.as<T>(), 1, n);
    if (sharded) allreduce_sum(ctx, Z.p, (size_t)(n * s), dt);
    ++passes;
    trace_mark(ctx, "ksvd: Z = A' Q");
    KsvdWork<T>::orth_light(ctx, n, s, Z.as<T>(), false);
    trace_mark(ctx, "ksvd: orth(Z)");
    // Y = A Z
    gemm<T>(ctx, m, s, n, T(1), Ap, A.rs, A.cs, Z.as<T>(), 1, n, T(0), Y.as<T>(), 1, m);
    ++passes;
    trace_mark(ctx, "ksvd: Y = A Z");
  }
  KsvdWork<T>::orth(ctx, m, s, Y.as<T>(), sharded);  // Q = thin_qr(C).Q
  trace_mark(ctx, "ksvd: orth(Y)");
  // pass 2: B = Q' A (s x n), column-major
  // computed as B' = A' Q (the streaming orientation of the A' Q power step),
  // written transposed: element (i, j) of B' lands at B[j + i*s].
  DevBuf B(sizeof(T) * s * n, ctx->stream);
  gemm<T>(ctx, n, s, m, T(1), Ap, A.cs, A.rs, Y.as<T>(), 1, m, T(0), B.as<T>(), s, 1);
  if (sharded) allreduce_sum(ctx, B.p, (size_t)(n * s), dt);
  ++passes;
  DevBuf B64;
  const double* Bp;
  if constexpr (std::is_same<T, double>::value) {
    Bp = B.as<double>();
  } else {
    B64 = DevBuf(sizeof(double) * s * n, ctx->stream);
    copy2d_cast<float, double>(ctx, s, n, B.as<float>(), 1, s, B64.as<double>(), 1, s);
    Bp = B64.as<double>();
  }
  trace_mark(ctx, "ksvd: B = Q' A");
  const int64_t kk = std::min(k, std::min(s, n));
  SvdDev small = topk_svd_wide(ctx, s, n, Bp, kk);
  trace_mark(ctx, "ksvd: small SVD");
  const int64_t rk = std::min(kk, small.rank);
  // U = Q Ubar (m x rk)
  DevBuf U64(sizeof(double) * m * std::max<int64_t>(rk, 1), ctx->stream);
  if constexpr (std::is_same<T, double>::value) {
    gemm<double>(ctx, m, rk, s, 1.0, Y.as<double>(), 1, m, small.U.as<double>(), 1, s, 0.0, U64.as<double>(), 1, m);
  } else {
    DevBuf uf(sizeof(float) * s * std::max<int64_t>(rk, 1), ctx->stream), Uf(sizeof(float) * m * std::max<int64_t>(rk, 1), ctx->stream);
    copy2d_cast<double, float>(ctx, s, rk, small.U.as<double>(), 1, s, uf.as<float>(), 1, s);
    gemm<float>(ctx, m, rk, s, 1.f, Y.as<float>(), 1, m, uf.as<float>(), 1, s, 0.f, Uf.as<float>(), 1, m);
    copy2d_cast<float, double>(ctx, m, rk, Uf.as<float>(), 1, m, U64.as<double>(), 1, m);
  }
  store_block(ctx, U64.as<double>(), m, rk, m, uo);
  store_block(ctx, small.V.as<double>(), n, rk, n, vo);
  trace_mark(ctx, "ksvd: U = Q Ubar, stores");
  for (int64_t i = 0; i < rk; ++i) sv_out[i] = small.s[(size_t)i];
  *rank_out = rk;
  *passes_out = passes;
  if (error_fro) {
    // |A - U S V'|_F computed block-wise as a residual (no cancellation).
    DevBuf svd(sizeof(double) * std::max<int64_t>(rk, 1), ctx->stream);
    RNLA_CUDA(cudaMemcpyAsync(svd.p, sv_out, sizeof(double) * rk, cudaMemcpyHostToDevice, ctx->stream));
    DevBuf SVt(sizeof(double) * std::max<int64_t>(rk * n, 1), ctx->stream);  // diag(S) V' : rk x n col-major
    scale_rows_dev(ctx, rk, n, small.V.as<double>(), svd.as<double>(), SVt.as<double>());
    const int64_t blk = std::max<int64_t>(1, std::min<int64_t>(m, ((int64_t)1 << 27) / std::max<int64_t>(n, 1)));
    DevBuf R(sizeof(double) * blk * n, ctx->stream);
    double total = 0.0;
    for (int64_t r0 = 0; r0 < m; r0 += blk) {
      const int64_t rows = std::min(blk, m - r0);
      if constexpr (std::is_same<T, double>::value)
        copy2d<double>(ctx, rows, n, Ap + r0 * A.rs, A.rs, A.cs, R.as<double>(), 1, rows);
      else
        copy2d_cast<float, double>(ctx, rows, n, Ap + r0 * A.rs, A.rs, A.cs, R.as<double>(), 1, rows);
      gemm<double>(ctx, rows, n, rk, -1.0, U64.as<double>() + r0, 1, m, SVt.as<double>(), 1, rk, 1.0, R.as<double>(),
                   1, rows);
      total += sum_squares_dev(ctx, R.as<double>(), rows * n);
    }
    if (sharded) total = allreduce_scalar(ctx, total);
    *error_fro = std::sqrt(total);
  }
  uo.finish(ctx);
  vo.finish(ctx);
}

// ---------------------------------------------------------------------------
// faster_ksvd (src/randsvd.cpp:112-160), fp64 working precision
// ---------------------------------------------------------------------------
const DenseOperator& gaussian_operator(rnla_ctx* ctx, int64_t n, int64_t s, uint64_t seed, int dtype);

// ||A - U diag(s) V'||_F, row blocks of A (column-major fp64 A, U m x r, V n x r).
static double residual_fro_f64(rnla_ctx* ctx, const double* A, int64_t m, int64_t n, const double* U,
                               const std::vector<double>& s, const double* V) {
  const int64_t r = (int64_t)s.size();
  DevBuf sd(sizeof(double) * std::max<int64_t>(r, 1), ctx->stream), SVt(sizeof(double) * std::max<int64_t>(r * n, 1),
                                                                        ctx->stream);
  RNLA_CUDA(cudaMemcpyAsync(sd.p, s.data(), sizeof(double) * r, cudaMemcpyHostToDevice, ctx->stream));
  scale_rows_dev(ctx, r, n, V, sd.as<double>(), SVt.as<double>());
  DevBuf R(sizeof(double) * m * n, ctx->stream);
  RNLA_CUDA(cudaMemcpyAsync(R.p, A, sizeof(double) * m * n, cudaMemcpyDeviceToDevice, ctx->stream));
  gemm<double>(ctx, m, n, r, -1.0, U, 1, m, SVt.as<double>(), 1, r, 1.0, R.as<double>(), 1, m);
  const double t = sum_squares_dev(ctx, R.as<double>(), m * n);
  RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
  return std::sqrt(t);
}

void faster_ksvd_impl(rnla_ctx* ctx, const rnla_mat* a, int64_t k, int64_t s, int64_t p_cs, int64_t p, uint64_t seed,
                      const rnla_mat* u_out, double* sv_out, const rnla_mat* v_out, int64_t* rank_out,
                      int32_t* passes_out, double* error_fro) {
  const int64_t m = a->rows, n = a->cols;
  OutMat uo(ctx, u_out, m, k, "faster_ksvd: U", false), vo(ctx, v_out, n, k, "faster_ksvd: V", false);
  DevMat A = f64_colmajor(ctx, a);
  const double* Ap = A.as<double>();
  // pass 1: C = A S (count sketch of the columns, seed derive_seed(seed, 1)) -> m x s column-major
  DevBuf C(sizeof(double) * m * s, ctx->stream);
  count_sketch_segments<double>(ctx, Ap, A.cs, nullptr, 1, n, m, s, derive_seed(seed, 1), 0, C.as<double>(), m,
                                false);
  // pass 2: joint row sketch of [A, C] (count p_cs -> Gaussian p), rows keyed by their index
  const int64_t w = n + s;
  DevBuf AC(sizeof(double) * m * w, ctx->stream);
  copy2d<double>(ctx, m, n, Ap, 1, A.cs, AC.as<double>(), w, 1);
  copy2d<double>(ctx, m, s, C.as<double>(), 1, m, AC.as<double>() + n, w, 1);
  DevBuf sk(sizeof(double) * p * w, ctx->stream);
  {
    rnla_sketch_spec sp{};
    sp.kind = RNLA_SKETCH_COMBINED;
    sp.s = p_cs;
    sp.seed = derive_seed(seed, 2);
    sp.stage2_kind = RNLA_SKETCH_GAUSSIAN;
    sp.stage2_s = p;
    sp.stage2_seed = derive_seed(seed, 3);
    sketch_rows_dev<double>(ctx, AC.as<double>(), w, nullptr, 1, m, w, &sp, 0, sk.as<double>(), w, 1);
  }
  // L = sk[:, :n] (p x n), D = sk[:, n:] (p x s); thin_qr(D)
  DevBuf D(sizeof(double) * p * s, ctx->stream), Rd(sizeof(double) * s * s, ctx->stream);
  copy2d<double>(ctx, p, s, sk.as<double>() + n, w, 1, D.as<double>(), 1, p);
  thin_qr_dev(ctx, p, s, D.as<double>(), Rd.as<double>());
  // small = truncated_svd(Q_D' L, k)
  DevBuf QtL(sizeof(double) * s * n, ctx->stream);
  gemm<double>(ctx, s, n, p, 1.0, D.as<double>(), p, 1, sk.as<double>(), w, 1, 0.0, QtL.as<double>(), 1, s);
  SvdDev small = condensed_svd_dev(ctx, s, n, QtL.as<double>(), 1, s);
  const int64_t k1 = std::min(k, small.rank);
  // back = C pinv(R_D) (Ubar Sigma): m x k1
  DevBuf pinv(sizeof(double) * s * s, ctx->stream);
  {
    DevBuf Ur(sizeof(double) * s * s, ctx->stream), Vr(sizeof(double) * s * s, ctx->stream),
        Sr(sizeof(double) * s, ctx->stream), inv(sizeof(double) * s, ctx->stream), Vs(sizeof(double) * s * s,
                                                                                         ctx->stream);
    svd_thin(ctx, s, s, Rd.as<double>(), 1, s, Ur.as<double>(), Sr.as<double>(), Vr.as<double>());
    std::vector<double> hs((size_t)s), hinv((size_t)s, 0.0);
    RNLA_CUDA(cudaMemcpyAsync(hs.data(), Sr.p, sizeof(double) * s, cudaMemcpyDeviceToHost, ctx->stream));
    RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
    for (int64_t i = 0; i < s; ++i)
      if (hs[0] > 0.0 && hs[(size_t)i] > 1e-12 * hs[0]) hinv[(size_t)i] = 1.0 / hs[(size_t)i];
    RNLA_CUDA(cudaMemcpyAsync(inv.p, hinv.data(), sizeof(double) * s, cudaMemcpyHostToDevice, ctx->stream));
    scale_cols_dev(ctx, s, s, Vr.as<double>(), inv.as<double>(), Vs.as<double>());
    gemm<double>(ctx, s, s, s, 1.0, Vs.as<double>(), 1, s, Ur.as<double>(), s, 1, 0.0, pinv.as<double>(), 1, s);
  }
  DevBuf sd(sizeof(double) * std::max<int64_t>(k1, 1), ctx->stream), US(sizeof(double) * s * std::max<int64_t>(k1, 1),
                                                                         ctx->stream),
      T(sizeof(double) * s * std::max<int64_t>(k1, 1), ctx->stream),
      back(sizeof(double) * m * std::max<int64_t>(k1, 1), ctx->stream);
  RNLA_CUDA(cudaMemcpyAsync(sd.p, small.s.data(), sizeof(double) * k1, cudaMemcpyHostToDevice, ctx->stream));
  scale_cols_dev(ctx, s, k1, small.U.as<double>(), sd.as<double>(), US.as<double>());
  gemm<double>(ctx, s, k1, s, 1.0, pinv.as<double>(), 1, s, US.as<double>(), 1, s, 0.0, T.as<double>(), 1, s);
  gemm<double>(ctx, m, k1, s, 1.0, C.as<double>(), 1, m, T.as<double>(), 1, s, 0.0, back.as<double>(), 1, m);
  SvdDev fin = condensed_svd_dev(ctx, m, k1, back.as<double>(), 1, m);
  const int64_t r = fin.rank;
  DevBuf Vout(sizeof(double) * n * std::max<int64_t>(r, 1), ctx->stream);
  gemm<double>(ctx, n, r, k1, 1.0, small.V.as<double>(), 1, n, fin.V.as<double>(), 1, k1, 0.0, Vout.as<double>(), 1,
               n);
  store_block(ctx, fin.U.as<double>(), m, r, m, uo);
  store_block(ctx, Vout.as<double>(), n, r, n, vo);
  for (int64_t i = 0; i < r; ++i) sv_out[i] = fin.s[(size_t)i];
  *rank_out = r;
  *passes_out = 2;
  if (error_fro) *error_fro = residual_fro_f64(ctx, Ap, m, n, fin.U.as<double>(), fin.s, Vout.as<double>());
  uo.finish(ctx);
  vo.finish(ctx);
}

}  // namespace rnla

using namespace rnla;

extern "C" {

rnla_status rnla_faster_ksvd(rnla_ctx* ctx, const rnla_mat* a, int64_t k, int64_t s, int64_t p_cs, int64_t p,
                             uint64_t seed, rnla_mat* u, double* sv, rnla_mat* v, int64_t* rank, int32_t* passes,
                             double* error_fro) {
  return guard([&] {
    enter(ctx);
    check_mat(a, "faster_ksvd: a");
    require(k >= 1 && k < s && s < p && p < p_cs, "faster_ksvd: need k < s < p < p_cs");
    require(ctx->world == 1, "faster_ksvd: row-sharded contexts are not supported");
    require(sv && rank && passes, "faster_ksvd: null output");
    faster_ksvd_impl(ctx, a, k, s, p_cs, p, seed, u, sv, v, rank, passes, error_fro);
  });
}

rnla_status rnla_thin_qr(rnla_ctx* ctx, const rnla_mat* a, rnla_mat* q, rnla_mat* r) {
  return guard([&] {
    enter(ctx);
    check_mat(a, "thin_qr: a");
    require(a->rows >= a->cols, "thin_qr: rows < cols");
    const int64_t m = a->rows, n = a->cols;
    OutMat qo(ctx, q, m, n, "thin_qr: Q", false), ro(ctx, r, n, n, "thin_qr: R", false);
    DevMat w = dense_copy(ctx, to_device(ctx, a), false, RNLA_F64);
    DevBuf rr(sizeof(double) * std::max<int64_t>(n * n, 1), ctx->stream);
    if (n > 0) thin_qr_dev(ctx, m, n, w.as<double>(), rr.as<double>());
    store_block(ctx, w.as<double>(), m, n, m, qo);
    store_block(ctx, rr.as<double>(), n, n, n, ro);
    qo.finish(ctx);
    ro.finish(ctx);
  });
}

rnla_status rnla_condensed_svd(rnla_ctx* ctx, const rnla_mat* a, rnla_mat* u, double* sv, rnla_mat* v,
                               int64_t* rank) {
  return guard([&] {
    enter(ctx);
    check_mat(a, "condensed_svd: a");
    require(sv && rank, "condensed_svd: null output");
    const int64_t m = a->rows, n = a->cols, r = std::min(m, n);
    OutMat uo(ctx, u, m, r, "condensed_svd: U", false), vo(ctx, v, n, r, "condensed_svd: V", false);
    DevMat w = f64_colmajor(ctx, a);
    SvdDev f = condensed_svd_dev(ctx, m, n, w.as<double>(), w.rs, w.cs);
    store_block(ctx, f.U.as<double>(), m, f.rank, m, uo);
    store_block(ctx, f.V.as<double>(), n, f.rank, n, vo);
    for (int64_t i = 0; i < f.rank; ++i) sv[i] = f.s[(size_t)i];
    *rank = f.rank;
    uo.finish(ctx);
    vo.finish(ctx);
  });
}

rnla_status rnla_truncated_svd(rnla_ctx* ctx, const rnla_mat* a, int64_t k, rnla_mat* u, double* sv, rnla_mat* v,
                               int64_t* rank) {
  return guard([&] {
    enter(ctx);
    check_mat(a, "truncated_svd: a");
    require(k >= 1 && k <= std::min(a->rows, a->cols), "truncated_svd: k out of range");
    require(sv && rank, "truncated_svd: null output");
    const int64_t m = a->rows, n = a->cols;
    OutMat uo(ctx, u, m, k, "truncated_svd: U", false), vo(ctx, v, n, k, "truncated_svd: V", false);
    DevMat w = f64_colmajor(ctx, a);
    SvdDev f = condensed_svd_dev(ctx, m, n, w.as<double>(), w.rs, w.cs);
    const int64_t rk = std::min(k, f.rank);
    store_block(ctx, f.U.as<double>(), m, rk, m, uo);
    store_block(ctx, f.V.as<double>(), n, rk, n, vo);
    for (int64_t i = 0; i < rk; ++i) sv[i] = f.s[(size_t)i];
    *rank = rk;
    uo.finish(ctx);
    vo.finish(ctx);
  });
}

rnla_status rnla_pseudo_inverse(rnla_ctx* ctx, const rnla_mat* a, double tol, rnla_mat* p) {
  return guard([&] {
    enter(ctx);
    check_mat(a, "pseudo_inverse: a");
    const int64_t m = a->rows, n = a->cols, r = std::min(m, n);
    OutMat po(ctx, p, n, m, "pseudo_inverse: P", false);
    DevBuf out(sizeof(double) * std::max<int64_t>(n * m, 1), ctx->stream);
    RNLA_CUDA(cudaMemsetAsync(out.p, 0, sizeof(double) * std::max<int64_t>(n * m, 1), ctx->stream));
    if (r > 0) {
      DevMat w = f64_colmajor(ctx, a);
      DevBuf U(sizeof(double) * m * r, ctx->stream), V(sizeof(double) * n * r, ctx->stream),
          S(sizeof(double) * r, ctx->stream);
      svd_thin(ctx, m, n, w.as<double>(), w.rs, w.cs, U.as<double>(), S.as<double>(), V.as<double>());
      std::vector<double> hs((size_t)r);
      RNLA_CUDA(cudaMemcpyAsync(hs.data(), S.p, sizeof(double) * r, cudaMemcpyDeviceToHost, ctx->stream));
      RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
      if (hs[0] > 0.0) {  // zero matrix -> zero of transposed shape (src/core.cpp:81)
        const double cut = tol * hs[0];
        std::vector<double> inv((size_t)r, 0.0);
        for (int64_t i = 0; i < r; ++i)
          if (hs[(size_t)i] > cut) inv[(size_t)i] = 1.0 / hs[(size_t)i];
        DevBuf dinv(sizeof(double) * r, ctx->stream), Vs(sizeof(double) * n * r, ctx->stream);
        RNLA_CUDA(cudaMemcpyAsync(dinv.p, inv.data(), sizeof(double) * r, cudaMemcpyHostToDevice, ctx->stream));
        scale_cols_dev(ctx, n, r, V.as<double>(), dinv.as<double>(), Vs.as<double>());  // V diag(inv)
        gemm<double>(ctx, n, m, r, 1.0, Vs.as<double>(), 1, n, U.as<double>(), m, 1, 0.0, out.as<double>(), 1, n);
        RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
      }
    }
    store_block(ctx, out.as<double>(), n, m, n, po);
    po.finish(ctx);
  });
}

rnla_status rnla_prototype_ksvd(rnla_ctx* ctx, const rnla_mat* a, int64_t k, int64_t s, uint64_t seed,
                                const rnla_sketch_spec* spec, int32_t power_iters, rnla_mat* u, double* sv,
                                rnla_mat* v, int64_t* rank, int32_t* passes, double* error_fro) {
  return guard([&] {
    enter(ctx);
    check_mat(a, "prototype_ksvd: a");
    require(k >= 1 && k <= s && s <= std::min(a->rows, a->cols), "prototype_ksvd: need k <= s <= min(m, n)");
    require(power_iters >= 0, "prototype_ksvd: power_iters < 0");
    require(sv && rank && passes, "prototype_ksvd: null output");
    if (a->dtype == RNLA_F64)
      prototype_ksvd_impl<double>(ctx, a, k, s, seed, spec, power_iters, u, sv, v, rank, passes, error_fro);
    else
      prototype_ksvd_impl<float>(ctx, a, k, s, seed, spec, power_iters, u, sv, v, rank, passes, error_fro);
  });
}

// ---- column selection (src/sketch.cpp:125-167) ----

rnla_status rnla_uniform_sample_columns(rnla_ctx* ctx, const rnla_mat* a, int64_t s, uint64_t seed, rnla_mat* c,
                                        int64_t* indices) {
  return guard([&] {
    enter(ctx);
    check_mat(a, "uniform_sample_columns: a");
    require(s >= 1 && s <= a->cols, "uniform_sample_columns: s > n");
    require(indices != nullptr, "uniform_sample_columns: null indices");
    std::vector<int64_t> idx = sample_without_replacement_host(seed, a->cols, s);
    std::copy(idx.begin(), idx.end(), indices);
    OutMat o(ctx, c, a->rows, s, "uniform_sample_columns: C", false);
    require(o.dev.dtype == a->dtype, "uniform_sample_columns: dtype mismatch");
    DevMat A = to_device(ctx, a);
    DevBuf di(sizeof(int64_t) * s, ctx->stream);
    RNLA_CUDA(cudaMemcpyAsync(di.p, idx.data(), sizeof(int64_t) * s, cudaMemcpyHostToDevice, ctx->stream));
    if (a->dtype == RNLA_F64)
      gather_columns<double>(ctx, a->rows, s, A.as<double>(), A.rs, A.cs, di.as<int64_t>(), nullptr,
                             o.dev.as<double>(), o.dev.rs, o.dev.cs);
    else
      gather_columns<float>(ctx, a->rows, s, A.as<float>(), A.rs, A.cs, di.as<int64_t>(), nullptr, o.dev.as<float>(),
                            o.dev.rs, o.dev.cs);
    o.finish(ctx);
  });
}

static std::vector<double> leverage_scores_host(rnla_ctx* ctx, const rnla_mat* a, int64_t k) {
  const int64_t m = a->rows, n = a->cols;
  DevMat w = f64_colmajor(ctx, a);
  SvdDev f = condensed_svd_dev(ctx, m, n, w.as<double>(), w.rs, w.cs);
  const int64_t rk = k > 0 ? std::min(k, f.rank) : f.rank;
  DevBuf sc(sizeof(double) * std::max<int64_t>(n, 1), ctx->stream);
  row_sqnorms<double>(ctx, n, rk, f.V.as<double>(), 1, n, sc.as<double>());
  std::vector<double> out((size_t)n);
  RNLA_CUDA(cudaMemcpyAsync(out.data(), sc.p, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
  RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
  return out;
}

rnla_status rnla_leverage_scores(rnla_ctx* ctx, const rnla_mat* a, int64_t k, double* scores) {
  return guard([&] {
    enter(ctx);
    check_mat(a, "leverage_scores: a");
    require(scores != nullptr, "leverage_scores: null output");
    if (k > 0) require(k <= std::min(a->rows, a->cols), "truncated_svd: k out of range");
    auto v = leverage_scores_host(ctx, a, k);
    std::copy(v.begin(), v.end(), scores);
  });
}

rnla_status rnla_leverage_sample_columns(rnla_ctx* ctx, const rnla_mat* a, int64_t s, uint64_t seed, int64_t k,
                                         int scale, rnla_mat* c, int64_t* indices, double* weights,
                                         int64_t* count_out) {
  return guard([&] {
    enter(ctx);
    check_mat(a, "leverage_sample_columns: a");
    require(s >= 1, "leverage_sample_columns: s < 1");
    require(indices && count_out, "leverage_sample_columns: null output");
    if (k > 0) require(k <= std::min(a->rows, a->cols), "truncated_svd: k out of range");
    std::vector<double> scores = leverage_scores_host(ctx, a, k);
    double rho = 0.0;
    for (double x : scores) rho += x;
    std::vector<int64_t> draws = sample_with_replacement_host(seed, scores.data(), a->cols, s);
    std::sort(draws.begin(), draws.end());
    draws.erase(std::unique(draws.begin(), draws.end()), draws.end());
    const int64_t cnt = (int64_t)draws.size();
    std::vector<double> w((size_t)cnt);
    for (int64_t t = 0; t < cnt; ++t)
      w[(size_t)t] = std::sqrt(rho / (static_cast<double>(s) * scores[(size_t)draws[(size_t)t]]));
    std::copy(draws.begin(), draws.end(), indices);
    if (weights && scale) std::copy(w.begin(), w.end(), weights);
    *count_out = cnt;
    check_mat(c, "leverage_sample_columns: C");
    require(c->rows == a->rows && c->cols >= cnt, "leverage_sample_columns: C too small");
    rnla_mat cv = *c;
    cv.cols = cnt;
    OutMat o(ctx, &cv, a->rows, cnt, "leverage_sample_columns: C", false);
    DevMat A = to_device(ctx, a);
    DevBuf di(sizeof(int64_t) * std::max<int64_t>(cnt, 1), ctx->stream), dw(sizeof(double) * std::max<int64_t>(cnt, 1),
                                                                             ctx->stream);
    RNLA_CUDA(cudaMemcpyAsync(di.p, draws.data(), sizeof(int64_t) * cnt, cudaMemcpyHostToDevice, ctx->stream));
    RNLA_CUDA(cudaMemcpyAsync(dw.p, w.data(), sizeof(double) * cnt, cudaMemcpyHostToDevice, ctx->stream));
    const double* sp = scale ? dw.as<double>() : nullptr;
    if (a->dtype == RNLA_F64)
      gather_columns<double>(ctx, a->rows, cnt, A.as<double>(), A.rs, A.cs, di.as<int64_t>(), sp, o.dev.as<double>(),
                             o.dev.rs, o.dev.cs);
    else
      gather_columns<float>(ctx, a->rows, cnt, A.as<float>(), A.rs, A.cs, di.as<int64_t>(), sp, o.dev.as<float>(),
                            o.dev.rs, o.dev.cs);
    o.finish(ctx);
  });
}

// Row leverage of a tall M through CholeskyQR: G = M'M (fp64 accumulate),
// R = chol(G), l_i = ||m_i R^-1||^2 = ||Q_i,:||^2 (basis invariance, paper
// Fact 6; tests/test_facts.cpp:86-97); then the reference's weighted draw +
// sort + unique (src/spsd.cpp:150-154).
namespace {
// out[i] = sum_t part[t * rows + i], t ascending
__global__ void sum_tiles_kernel(int64_t rows, int nt, const double* __restrict__ part, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows; i += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int t = 0; t < nt; ++t) acc += part[(int64_t)t * rows + i];
    out[i] = acc;
  }
}
}  // namespace

rnla_status rnla_leverage_sample_rows(rnla_ctx* ctx, const rnla_mat* m, int64_t p, uint64_t seed, double* scores,
                                      int64_t* indices, int64_t* count_out) {
  return guard([&] {
    enter(ctx);
    check_mat(m, "leverage_sample_rows: m");
    require(scores != nullptr, "leverage_sample_rows: null scores");
    require(indices == nullptr || (p >= 1 && count_out), "sample_with_replacement: count < 1");
    // Row-sharded M: scores are this rank's rows, the
    // indices are global, drawn from the allgathered score vector (replicated).
    const int64_t n = m->rows, d = m->cols;
    int64_t n_total = n;
    const int64_t r_off = global_row_offset(ctx, n, &n_total);
    require(n_total >= d && d >= 1, "thin_qr: rows < cols");
    trace_mark(ctx, "leverage_rows: enter");
    DevMat M = to_device(ctx, m);
    DevBuf G(sizeof(double) * d * d, ctx->stream), Rinv(sizeof(double) * d * d, ctx->stream);
    if (n == 0)
      RNLA_CUDA(cudaMemsetAsync(G.p, 0, sizeof(double) * d * d, ctx->stream));
    else if (M.dtype == RNLA_F64)
      gemm<double>(ctx, d, d, n, 1.0, M.as<double>(), M.cs, M.rs, M.as<double>(), M.rs, M.cs, 0.0, G.as<double>(), 1,
                   d);
    else
      gemm_f32_f64acc(ctx, d, d, n, 1.0, M.as<float>(), M.cs, M.rs, M.as<float>(), M.rs, M.cs, 0.0, G.as<double>(), 1,
                      d);
    trace_mark(ctx, "leverage_rows: gram");
    if (is_sharded(ctx)) allreduce_sum(ctx, G.p, (size_t)(d * d), RNLA_F64);
    if (!cholesky_upper(ctx, d, G.as<double>()))
      throw NumericError("leverage_sample_rows: M'M is not positive definite (rank-deficient M)");
    upper_inverse(ctx, d, G.as<double>(), Rinv.as<double>());
    trace_mark(ctx, "leverage_rows: chol+inverse");
    DevBuf sc(sizeof(double) * n, ctx->stream);
    const int64_t blk = std::max<int64_t>(1, std::min<int64_t>(n, ((int64_t)1 << 26) / d));
    DevBuf T(sizeof(double) * blk * d, ctx->stream);
    DevBuf Rf;
    if (M.dtype != RNLA_F64) {
      Rf = DevBuf(sizeof(float) * d * d, ctx->stream);
      copy2d_cast<double, float>(ctx, d, d, Rinv.as<double>(), 1, d, Rf.as<float>(), 1, d);
    }
    // One GPU: each block's scores go to pinned host memory as soon as they
    // are computed, and the host extends the sequential fp64 prefix sums of
    // the draw (src/rng.cpp:42-65) while the device computes the next blocks.
    const bool stream_draw = indices != nullptr && ctx->world == 1 && n > 0;
    double* hs = stream_draw ? static_cast<double*>(pinned_scratch(ctx, sizeof(double) * n)) : nullptr;
    const int64_t nblk = (n + blk - 1) / blk;
    std::vector<cudaEvent_t> ev;
    WeightPrefix prefix;
    int64_t done = 0;  // blocks folded into prefix
    auto fold = [&](int64_t upto) {  // also moves the block into the caller's scores
      for (; done < upto; ++done) {
        const int64_t r0 = done * blk, rows = std::min(blk, n - r0);
        RNLA_CUDA(cudaEventSynchronize(ev[(size_t)done]));
        prefix.extend(hs + r0, rows);
        std::copy(hs + r0, hs + r0 + rows, scores + r0);
      }
    };
    WeightPrefix::Prepared prepared;
    if (stream_draw) {
      prepared = WeightPrefix::prepare(seed, p);  // host work under the Gram / Cholesky already queued
      ev.resize((size_t)nblk);
      for (auto& e : ev) RNLA_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      prefix.cum.reserve((size_t)n);
    }
    try {
      for (int64_t bi = 0; bi < nblk; ++bi) {
        const int64_t r0 = bi * blk, rows = std::min(blk, n - r0);
        if (M.dtype == RNLA_F64) {
          gemm<double>(ctx, rows, d, d, 1.0, M.as<double>() + r0 * M.rs, M.rs, M.cs, Rinv.as<double>(), 1, d, 0.0,
                       T.as<double>(), d, 1);
          row_sqnorms<double>(ctx, rows, d, T.as<double>(), d, 1, sc.as<double>() + r0);
        } else {
          // R^-1 is upper triangular: column tile j needs k < its last column only.
          // The GEMM epilogue sums the squares of each N tile of a row (M R^-1 is
          // never stored); the tiles are added in order.
          if (tc_gemm_enabled()) {
            const int nt = gemm_f32_tc_tri_b_rownorm(ctx, rows, d, d, 1.f, M.as<float>() + r0 * M.rs, M.rs, M.cs,
                                                     Rf.as<float>(), 1, d, T.as<double>());
            sum_tiles_kernel<<<grid_for(ctx, rows, 256), 256, 0, ctx->stream>>>(rows, nt, T.as<double>(),
                                                                              sc.as<double>() + r0);
            RNLA_CUDA(cudaGetLastError());
            note_launch(ctx);
          } else {
            gemm<float>(ctx, rows, d, d, 1.f, M.as<float>() + r0 * M.rs, M.rs, M.cs, Rf.as<float>(), 1, d, 0.f,
                        T.as<float>(), d, 1);
            row_sqnorms<float>(ctx, rows, d, T.as<float>(), d, 1, sc.as<double>() + r0);
          }
        }
        if (stream_draw) {
          RNLA_CUDA(cudaMemcpyAsync(hs + r0, sc.as<double>() + r0, sizeof(double) * rows, cudaMemcpyDeviceToHost,
                                    ctx->stream));
          RNLA_CUDA(cudaEventRecord(ev[(size_t)bi], ctx->stream));
          fold(bi);  // blocks before this one, while the device works on it
        }
      }
      if (stream_draw) fold(nblk);
    } catch (...) {
      cudaStreamSynchronize(ctx->stream);
      for (auto& e : ev) cudaEventDestroy(e);
      throw;
    }
    for (auto& e : ev) RNLA_CUDA(cudaEventDestroy(e));
    trace_mark(ctx, "leverage_rows: scores");
    if (!stream_draw) {
      if (n > 0) RNLA_CUDA(cudaMemcpyAsync(scores, sc.p, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
      RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
    }
    trace_mark(ctx, "leverage_rows: d2h");
    if (indices) {
      std::vector<int64_t> draws;
      if (stream_draw) {
        draws = prefix.draw(prepared);
      } else {
        std::vector<double> all_scores;
        const double* w = scores;
        if (is_sharded(ctx)) {
          DevBuf g(sizeof(double) * n_total, ctx->stream);
          RNLA_CUDA(cudaMemsetAsync(g.p, 0, sizeof(double) * n_total, ctx->stream));
          if (n > 0)
            RNLA_CUDA(cudaMemcpyAsync(g.as<double>() + r_off, sc.p, sizeof(double) * n, cudaMemcpyDeviceToDevice,
                                      ctx->stream));
          allreduce_sum(ctx, g.p, (size_t)n_total, RNLA_F64);
          all_scores.resize((size_t)n_total);
          RNLA_CUDA(cudaMemcpyAsync(all_scores.data(), g.p, sizeof(double) * n_total, cudaMemcpyDeviceToHost,
                                    ctx->stream));
          RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
          w = all_scores.data();
        }
        draws = sample_with_replacement_host(seed, w, n_total, p);
      }
      std::sort(draws.begin(), draws.end());
      draws.erase(std::unique(draws.begin(), draws.end()), draws.end());
      std::copy(draws.begin(), draws.end(), indices);
      trace_mark(ctx, "leverage_rows: d2h + host draw");
      *count_out = (int64_t)draws.size();
    }
  });
}

rnla_status rnla_apply_sketch(rnla_ctx* ctx, const rnla_mat* a, const rnla_sketch_spec* spec, rnla_mat* c,
                              int64_t* cols_out) {
  return guard([&] {
    enter(ctx);
    require(spec != nullptr, "null SketchSpec");
    rnla_status st = RNLA_OK;
    int64_t cols = spec->kind == RNLA_SKETCH_COMBINED ? spec->stage2_s : spec->s;
    switch (spec->kind) {
      case RNLA_SKETCH_GAUSSIAN: st = rnla_gaussian_sketch(ctx, a, spec->s, spec->seed, c); break;
      case RNLA_SKETCH_SRHT: st = rnla_srht_sketch(ctx, a, spec->s, spec->seed, c); break;
      case RNLA_SKETCH_COUNT: st = rnla_count_sketch(ctx, a, spec->s, spec->seed, c); break;
      case RNLA_SKETCH_COMBINED: st = rnla_combined_sketch(ctx, a, spec, c); break;
      case RNLA_SKETCH_UNIFORM_COLUMNS: {
        std::vector<int64_t> idx((size_t)std::max<int64_t>(spec->s, 1));
        st = rnla_uniform_sample_columns(ctx, a, spec->s, spec->seed, c, idx.data());
        break;
      }
      case RNLA_SKETCH_LEVERAGE_COLUMNS: {
        std::vector<int64_t> idx((size_t)std::max<int64_t>(spec->s, 1));
        std::vector<double> w((size_t)std::max<int64_t>(spec->s, 1));
        st = rnla_leverage_sample_columns(ctx, a, spec->s, spec->seed, spec->leverage_rank, spec->scale_columns, c,
                                          idx.data(), w.data(), &cols);
        break;
      }
      case RNLA_SKETCH_LANDMARK_COLUMNS:
        throw InvalidArgument("apply_sketch: landmark selection (k-means) is outside the B200 core");
      default:
        throw InvalidArgument("apply_sketch: unknown kind");
    }
    if (st != RNLA_OK) {
      const std::string msg = rnla_last_error();
      if (st == RNLA_EINVAL) throw InvalidArgument(msg);
      if (st == RNLA_ENUMERIC) throw NumericError(msg);
      throw CudaError(msg);
    }
    if (cols_out) *cols_out = cols;
  });
}

}  // extern "C"
