// api_spsd.cpp -- rbf_kernel, KernelView-backed nystrom, approx_eig and the
// fused Nystrom + top-k eigen route behind the C ABI.
//
// Reference: /root/reference/proj/src/spsd.cpp:33-72 (rbf_kernel, KernelView),
// :181-222 (nystrom), :257-265 (approx_eig).
#include <cmath>
#include <exception>
#include <limits>
#include <thread>

#include "algos.h"
#include "dist.h"
#include "linalg.cuh"
#include "rbf.cuh"

namespace rnla {

namespace {

// Selected landmarks (src/spsd.cpp:189-191) for the kernel columns C = K[:, S]
// of X (this rank's n_local x d rows of the global n points; fp64 output
// when T = double, else fp32). The landmark points are gathered by their
// owners and replicated (an allreduce of the zero-padded s x d block).
struct Landmarks {
  std::vector<int64_t> sel;  // global indices, ascending
  DevBuf dsel;               // local row of each landmark, -1 if another rank owns it
  DevBuf sq;                 // squared norms of this rank's rows
  DevMat Xs;                 // landmark points (s x d), replicated
  DevBuf sqS;                // their squared norms (same FMA chain: bitwise equal to sq[sel])
  int64_t r_off = 0;
};

template <class T>
Landmarks landmarks(rnla_ctx* ctx, const DevMat& X, int64_t s, uint64_t seed, int64_t n_global, int64_t r_off) {
  Landmarks L;
  const int64_t n = X.rows, d = X.cols;
  {  // the landmark draw is an operator: cached per (n, s, seed) like the other random operators
    auto key = std::make_tuple(n_global, s, seed);
    auto it = ctx->landmark_sel.find(key);
    if (it == ctx->landmark_sel.end())
      it = ctx->landmark_sel.emplace(key, sample_without_replacement_host(derive_seed(seed, 1), n_global, s)).first;
    L.sel = it->second;
  }
  L.r_off = r_off;
  std::vector<int64_t> loc(L.sel);
  for (auto& v : loc) v = (v >= r_off && v < r_off + n) ? v - r_off : -1;
  L.dsel = DevBuf(sizeof(int64_t) * s, ctx->stream);
  RNLA_CUDA(cudaMemcpyAsync(L.dsel.p, loc.data(), sizeof(int64_t) * s, cudaMemcpyHostToDevice, ctx->stream));
  L.sq = DevBuf(sizeof(T) * std::max<int64_t>(n, 1), ctx->stream);
  sq_norms<T>(ctx, n, d, X.as<T>(), X.rs, X.cs, nullptr, L.sq.as<T>());
  L.Xs = alloc_dense(ctx, s, d, true, X.dtype);
  gather_rows<T>(ctx, s, d, X.as<T>(), X.rs, X.cs, L.dsel.as<int64_t>(), L.Xs.as<T>(), L.Xs.rs, L.Xs.cs);
  if (is_sharded(ctx)) allreduce_sum(ctx, L.Xs.p, (size_t)(s * d), X.dtype);
  L.sqS = DevBuf(sizeof(T) * s, ctx->stream);
  sq_norms<T>(ctx, s, d, L.Xs.as<T>(), L.Xs.rs, L.Xs.cs, nullptr, L.sqS.as<T>());
  RNLA_CUDA(cudaStreamSynchronize(ctx->stream));  // `loc` leaves scope
  return L;
}

// Rows [r0, r0 + rows) of this rank's block of C = K[:, S].
template <class T>
void kernel_columns(rnla_ctx* ctx, const DevMat& X, const Landmarks& L, int64_t r0, int64_t rows, double sigma,
                    T* C, int64_t c_rs, int64_t c_cs) {
  const int64_t s = (int64_t)L.sel.size(), d = X.cols;
  // diag_of[t] = the landmark's own row inside this block (forced to exactly 1).
  DevBuf diag(sizeof(int64_t) * s, ctx->stream);
  std::vector<int64_t> h(L.sel);
  for (auto& v : h) v -= L.r_off + r0;
  RNLA_CUDA(cudaMemcpyAsync(diag.p, h.data(), sizeof(int64_t) * s, cudaMemcpyHostToDevice, ctx->stream));
  rbf_block<T>(ctx, rows, s, d, X.as<T>() + r0 * X.rs, X.rs, X.cs, L.Xs.as<T>(), L.Xs.rs, L.Xs.cs, nullptr,
               L.sq.as<T>() + r0, L.sqS.as<T>(), sigma, diag.as<int64_t>(), C, c_rs, c_cs);
  RNLA_CUDA(cudaStreamSynchronize(ctx->stream));  // `h` leaves scope
}

struct EigW {
  DevBuf U;  // s x kept (col-major), eigenvectors of the top `kept` eigenvalues, descending
  std::vector<double> lam;
  int64_t kept = 0;
};

// eig(0.5 (W + W')) ascending, walk from the top with the floor
// eps * lam_max * n (src/spsd.cpp:193-207).
EigW nystrom_core(rnla_ctx* ctx, const double* W, int64_t s, int64_t n, int64_t kk) {
  DevBuf ws(sizeof(double) * s * s, ctx->stream), lam(sizeof(double) * s, ctx->stream);
  symmetrize(ctx, s, W, ws.as<double>());
  eig_sym(ctx, s, ws.as<double>(), lam.as<double>());
  std::vector<double> h((size_t)s);
  RNLA_CUDA(cudaMemcpyAsync(h.data(), lam.p, sizeof(double) * s, cudaMemcpyDeviceToHost, ctx->stream));
  RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
  const double lam_max = h[(size_t)s - 1];
  if (!(lam_max > 0.0)) throw NumericError("nystrom: kernel block has no positive spectrum");
  const double floor = std::numeric_limits<double>::epsilon() * lam_max * static_cast<double>(n);
  int64_t kept = 0;
  while (kept < kk && h[(size_t)(s - 1 - kept)] > floor) ++kept;
  if (kept == 0) throw NumericError("nystrom: no retained eigenvalues");
  EigW e;
  e.kept = kept;
  e.U = DevBuf(sizeof(double) * s * kept, ctx->stream);
  // columns s-1, s-2, ... of the ascending eigenvector matrix
  copy2d<double>(ctx, s, kept, ws.as<double>() + (s - 1) * s, 1, -s, e.U.as<double>(), 1, s);
  e.lam.resize((size_t)kept);
  for (int64_t t = 0; t < kept; ++t) e.lam[(size_t)t] = h[(size_t)(s - 1 - t)];
  RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
  return e;
}

// T = U_k diag(lam^-1/2) (s x kept, col-major fp64)
DevBuf whitened(rnla_ctx* ctx, const EigW& e, int64_t s) {
  std::vector<double> inv((size_t)e.kept);
  for (int64_t t = 0; t < e.kept; ++t) inv[(size_t)t] = 1.0 / std::sqrt(e.lam[(size_t)t]);
  DevBuf dinv(sizeof(double) * e.kept, ctx->stream), T(sizeof(double) * s * e.kept, ctx->stream);
  RNLA_CUDA(cudaMemcpyAsync(dinv.p, inv.data(), sizeof(double) * e.kept, cudaMemcpyHostToDevice, ctx->stream));
  scale_cols_dev(ctx, s, e.kept, e.U.as<double>(), dinv.as<double>(), T.as<double>());
  RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
  return T;
}

// The reference's generic nystrom(SpsdSource) body (src/spsd.cpp:181-217)
// given C = K[:, S] on the device (n x s col-major, ld n, compute dtype T) and
// the landmarks' rows dsel inside C: W = rows S of C, eig(0.5 (W + W')),
// eigenvalue floor, L = C U_k Lambda_k^-1/2.
template <class T>
void nystrom_from_columns(rnla_ctx* ctx, const T* C, const int64_t* dsel, int64_t n, int64_t s, int64_t kk,
                          const rnla_mat* l_out, int64_t* kept_out) {
  DevBuf W(sizeof(double) * s * s, ctx->stream);
  if constexpr (std::is_same<T, double>::value) {
    gather_rows<double>(ctx, s, s, C, 1, n, dsel, W.as<double>(), 1, s);
  } else {
    DevBuf Wf(sizeof(float) * s * s, ctx->stream);
    gather_rows<float>(ctx, s, s, C, 1, n, dsel, Wf.as<float>(), 1, s);
    copy2d_cast<float, double>(ctx, s, s, Wf.as<float>(), 1, s, W.as<double>(), 1, s);
    RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  EigW e = nystrom_core(ctx, W.as<double>(), s, n, kk);
  DevBuf Tm = whitened(ctx, e, s);
  if (l_out) {
    OutMat lo(ctx, l_out, n, kk, "nystrom: L", false);
    if constexpr (std::is_same<T, double>::value) {
      gemm<double>(ctx, n, e.kept, s, 1.0, C, 1, n, Tm.as<double>(), 1, s, 0.0, lo.dev.as<double>(), lo.dev.rs,
                   lo.dev.cs);
    } else {
      DevBuf Tf(sizeof(float) * s * e.kept, ctx->stream);
      copy2d_cast<double, float>(ctx, s, e.kept, Tm.as<double>(), 1, s, Tf.as<float>(), 1, s);
      gemm<float>(ctx, n, e.kept, s, 1.f, C, 1, n, Tf.as<float>(), 1, s, 0.f, lo.dev.as<float>(), lo.dev.rs,
                  lo.dev.cs);
    }
    lo.finish(ctx);
  }
  *kept_out = e.kept;
  RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
}

static int64_t nystrom_k(int64_t target_k, int64_t s) {
  return target_k > 0 ? target_k : (int64_t)std::ceil(0.8 * static_cast<double>(s));
}

template <class T>
void nystrom_impl(rnla_ctx* ctx, const rnla_mat* x, double sigma, int64_t s, uint64_t seed, int64_t target_k,
                  const rnla_mat* l_out, int64_t* selected, int64_t* kept_out, int64_t* entries) {
  DevMat X = to_device(ctx, x);
  const int64_t n = X.rows;
  const int64_t kk = nystrom_k(target_k, s);
  require(kk >= 1 && kk <= s && s <= n, "nystrom: need k <= s <= n");
  require(ctx->world == 1, "nystrom: row-sharded contexts use nystrom_eig");
  Landmarks L = landmarks<T>(ctx, X, s, seed, n, 0);
  // C = K[:, S] (n x s, col-major, compute dtype) from the KernelView
  DevBuf C(sizeof(T) * n * s, ctx->stream);
  kernel_columns<T>(ctx, X, L, 0, n, sigma, C.as<T>(), 1, n);
  nystrom_from_columns<T>(ctx, C.as<T>(), L.dsel.as<int64_t>(), n, s, kk, l_out, kept_out);
  std::copy(L.sel.begin(), L.sel.end(), selected);
  if (entries) *entries = n * s;
}

// nystrom(const DenseMatrix& K, ...) (src/spsd.cpp:224-228): DenseSpsdSource
// columns K[:, S] gathered on the device.
template <class T>
void nystrom_dense_impl(rnla_ctx* ctx, const rnla_mat* k, int64_t s, uint64_t seed, int64_t target_k,
                        const rnla_mat* l_out, int64_t* selected, int64_t* kept_out) {
  require(k->rows == k->cols, "nystrom: K not square");
  const int64_t n = k->rows, kk = nystrom_k(target_k, s);
  require(kk >= 1 && kk <= s && s <= n, "nystrom: need k <= s <= n");
  DevMat K = to_device(ctx, k);
  const std::vector<int64_t> sel = sample_without_replacement_host(derive_seed(seed, 1), n, s);
  DevBuf dsel(sizeof(int64_t) * s, ctx->stream);
  RNLA_CUDA(cudaMemcpyAsync(dsel.p, sel.data(), sizeof(int64_t) * s, cudaMemcpyHostToDevice, ctx->stream));
  DevBuf C(sizeof(T) * n * s, ctx->stream);
  gather_columns<T>(ctx, n, s, K.as<T>(), K.rs, K.cs, dsel.as<int64_t>(), nullptr, C.as<T>(), 1, n);
  nystrom_from_columns<T>(ctx, C.as<T>(), dsel.as<int64_t>(), n, s, kk, l_out, kept_out);
  std::copy(sel.begin(), sel.end(), selected);
}

// nystrom(const SpsdSource&, ...) for a caller-provided source: C = K[:, S]
// already evaluated by the caller (the landmarks drawn as the reference does).
template <class T>
void nystrom_columns_impl(rnla_ctx* ctx, const rnla_mat* c, const int64_t* selected, int64_t target_k,
                          const rnla_mat* l_out, int64_t* kept_out) {
  const int64_t n = c->rows, s = c->cols, kk = nystrom_k(target_k, s);
  require(kk >= 1 && kk <= s && s <= n, "nystrom: need k <= s <= n");
  for (int64_t t = 0; t < s; ++t)
    require(selected[t] >= 0 && selected[t] < n && (t == 0 || selected[t] > selected[t - 1]),
            "nystrom: selected indices must be strictly increasing and < n");
  DevMat C = as_colmajor(ctx, to_device(ctx, c));
  DevMat Cd = C.cs == n ? std::move(C) : dense_copy(ctx, C, false, C.dtype);
  DevBuf dsel(sizeof(int64_t) * s, ctx->stream);
  RNLA_CUDA(cudaMemcpyAsync(dsel.p, selected, sizeof(int64_t) * s, cudaMemcpyHostToDevice, ctx->stream));
  nystrom_from_columns<T>(ctx, Cd.as<T>(), dsel.as<int64_t>(), n, s, kk, l_out, kept_out);
}

// nystrom + approx_eig(L, k) through the Gram route:
// L'L = T' (C'C) T with T = U_k Lambda^-1/2; eig(L'L) = (V, sigma^2);
// U_L = L V / sigma = C (T V / sigma). C is formed block by block and never
// stored; C'C accumulates in fp64 (DMMA) across row blocks.
template <class T>
void nystrom_eig_impl(rnla_ctx* ctx, const rnla_mat* x, double sigma, int64_t s, uint64_t seed, int64_t target_k,
                      int64_t k, const rnla_mat* u_out, double* lam_out, int64_t* selected, int64_t* kept_out) {
  DevMat X = to_device(ctx, x);
  const int64_t n_local = X.rows;
  int64_t n = n_local;
  const int64_t r_off = global_row_offset(ctx, n_local, &n);
  const int64_t kk = target_k > 0 ? target_k : (int64_t)std::ceil(0.8 * static_cast<double>(s));
  require(kk >= 1 && kk <= s && s <= n, "nystrom: need k <= s <= n");
  trace_mark(ctx, "nystrom_eig: enter");
  Landmarks L = landmarks<T>(ctx, X, s, seed, n, r_off);
  trace_mark(ctx, "nystrom_eig: landmarks");
  const int64_t blk = std::max<int64_t>(1, std::min<int64_t>(n_local, 16384));
  DevBuf Cb(sizeof(T) * blk * s, ctx->stream);
  DevBuf G(sizeof(double) * s * s, ctx->stream), W(sizeof(double) * s * s, ctx->stream);
  // fp32 points: the exact int8-digit Gram on the tensor cores (gram_i8.cu);
  // W and C'C then describe the same quantized kernel matrix.
  const bool i8 = std::is_same<T, float>::value && gram_i8_available();
  // W = K[S, S]: its rows are the landmark rows of C (recomputed directly).
  // digit planes of C (3 bytes per entry) in row blocks of at most ~2 GB
  const int64_t rows_blk =
      i8 ? std::max<int64_t>(1, std::min<int64_t>(
               n_local, std::max<int64_t>(65536, (int64_t)(2e9 / (3.0 * (double)s)) / 64 * 64)))
         : 1;
  const int64_t pitch = i8 ? digit_pitch(rows_blk) : 0;
  DevBuf planes(i8 ? 3 * (size_t)s * (size_t)pitch : 0, ctx->stream);
  // tensor-core kernel columns (d <= 64, C in one block of digit planes);
  // otherwise W and C both come from the sequential-FMA kernel
  const bool tc_rbf = i8 && rows_blk >= n_local && rbf_tc_available(X.cols);
  // SMs left to the eig(W) / Cholesky route that runs on the helper stream
  // while the tensor-core kernels below stream C (their kernels are
  // latency-bound cuSOLVER launches that would otherwise wait for whole SMs)
  int reserve_sms = 0;
  auto c_digits = [&](int64_t r0, int64_t rows) {  // digit planes of rows [r0, r0 + rows) of C
    DevBuf diag(sizeof(int64_t) * s, ctx->stream);
    std::vector<int64_t> h(L.sel);
    for (auto& v : h) v -= L.r_off + r0;
    RNLA_CUDA(cudaMemcpyAsync(diag.p, h.data(), sizeof(int64_t) * s, cudaMemcpyHostToDevice, ctx->stream));
    if (tc_rbf)
      rbf_tc_digits(ctx, rows, s, X.cols, X.as<float>() + r0 * X.rs, X.rs, X.cs, L.Xs.as<float>(), L.Xs.rs, L.Xs.cs,
                    L.sq.as<float>() + r0, L.sqS.as<float>(), sigma, diag.as<int64_t>(), planes.as<int8_t>(), pitch,
                    s * pitch, reserve_sms);
    else
      rbf_digits(ctx, rows, s, X.cols, X.as<float>() + r0 * X.rs, X.rs, X.cs, L.Xs.as<float>(), L.Xs.rs, L.Xs.cs,
                 L.sq.as<float>() + r0, L.sqS.as<float>(), sigma, diag.as<int64_t>(), planes.as<int8_t>(), pitch,
                 s * pitch, nullptr, 0);
    RNLA_CUDA(cudaStreamSynchronize(ctx->stream));  // `h` leaves scope
  };
  if (tc_rbf) {
    // W = K[S, S] from the same tensor-core kernel on the landmark points: an
    // MMA output element depends only on its row and column operands, so these
    // digits equal the landmark rows of C's digits bit for bit (checked with
    // RNLA_CHECK_W_DIGITS=1). W is ready before C, so the Cholesky route below
    // overlaps the kernel columns and the Gram.
    const int64_t pw = digit_pitch(s);
    DevBuf wplanes(3 * (size_t)s * (size_t)pw, ctx->stream), ident(sizeof(int64_t) * s, ctx->stream);
    std::vector<int64_t> id((size_t)s);
    for (int64_t i = 0; i < s; ++i) id[(size_t)i] = i;
    RNLA_CUDA(cudaMemcpyAsync(ident.p, id.data(), sizeof(int64_t) * s, cudaMemcpyHostToDevice, ctx->stream));
    rbf_tc_digits(ctx, s, s, X.cols, L.Xs.as<float>(), L.Xs.rs, L.Xs.cs, L.Xs.as<float>(), L.Xs.rs, L.Xs.cs,
                  L.sqS.as<float>(), L.sqS.as<float>(), sigma, ident.as<int64_t>(), wplanes.as<int8_t>(), pw, s * pw);
    w_from_digits(ctx, s, ident.as<int64_t>(), wplanes.as<int8_t>(), pw, s * pw, W.as<double>());
    RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
  } else if (i8) {
    DevBuf ident(sizeof(int64_t) * s, ctx->stream);
    std::vector<int64_t> id((size_t)s);
    for (int64_t i = 0; i < s; ++i) id[(size_t)i] = i;
    RNLA_CUDA(cudaMemcpyAsync(ident.p, id.data(), sizeof(int64_t) * s, cudaMemcpyHostToDevice, ctx->stream));
    rbf_digits(ctx, s, s, X.cols, L.Xs.as<float>(), L.Xs.rs, L.Xs.cs, L.Xs.as<float>(), L.Xs.rs, L.Xs.cs,
               L.sqS.as<float>(), L.sqS.as<float>(), sigma, ident.as<int64_t>(), nullptr, 0, 0, W.as<double>(), s);
    RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
  } else {
    DevBuf Wt(sizeof(T) * s * s, ctx->stream), ident(sizeof(int64_t) * s, ctx->stream);
    std::vector<int64_t> id((size_t)s);
    for (int64_t i = 0; i < s; ++i) id[(size_t)i] = i;
    RNLA_CUDA(cudaMemcpyAsync(ident.p, id.data(), sizeof(int64_t) * s, cudaMemcpyHostToDevice, ctx->stream));
    rbf_block<T>(ctx, s, s, X.cols, L.Xs.as<T>(), L.Xs.rs, L.Xs.cs, L.Xs.as<T>(), L.Xs.rs, L.Xs.cs, nullptr,
                 L.sqS.as<T>(), L.sqS.as<T>(), sigma, ident.as<int64_t>(), Wt.as<T>(), 1, s);
    if constexpr (std::is_same<T, double>::value)
      RNLA_CUDA(cudaMemcpyAsync(W.p, Wt.p, sizeof(double) * s * s, cudaMemcpyDeviceToDevice, ctx->stream));
    else
      copy2d_cast<float, double>(ctx, s, s, Wt.as<float>(), 1, s, W.as<double>(), 1, s);
    RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  trace_mark(ctx, "nystrom_eig: W");
  // Full-rank route. When target_k >= s and every eigenvalue of W clears the
  // floor, the reference keeps all of them: L = C U Lambda^-1/2 = C W^-1/2,
  // and approx_eig(L) depends on L only through L L' = C W^-1 C'. With the
  // Cholesky factor W = R'R, L' = C R^-1 has the same L L', hence the same
  // singular values and left singular vectors, so eig(W) (a 28 ms cuSOLVER
  // tridiagonalization at s = 2048) becomes potrf + one triangular inverse.
  // The floor test is conservative: lam_min(W) >= 1 / |R^-1|_F^2 and
  // lam_max(W) <= |W|_F, with a 4x margin (config 4: lam_min / floor = 6.8e3).
  // Otherwise the eigendecomposition route below runs.
  DevBuf Tm;  // s x kp: L = C Tm
  int64_t kp = 0;
  bool cholesky_T = false;  // Tm = R^-1 from the Cholesky route (upper triangular)
  auto cholesky_route = [&](rnla_ctx* c) {
    DevBuf Ws(sizeof(double) * s * s, c->stream), R(sizeof(double) * s * s, c->stream),
        Ri(sizeof(double) * s * s, c->stream);
    symmetrize(c, s, W.as<double>(), Ws.as<double>());
    RNLA_CUDA(cudaMemcpyAsync(R.p, Ws.p, sizeof(double) * s * s, cudaMemcpyDeviceToDevice, c->stream));
    if (!cholesky_upper(c, s, R.as<double>())) return false;
    upper_inverse(c, s, R.as<double>(), Ri.as<double>());
    const double inv_fro2 = sum_squares_dev(c, Ri.as<double>(), s * s);
    const double w_fro = std::sqrt(sum_squares_dev(c, Ws.as<double>(), s * s));
    const double floor_ub = std::numeric_limits<double>::epsilon() * w_fro * static_cast<double>(n);
    if (!(std::isfinite(inv_fro2) && inv_fro2 > 0.0 && 1.0 / inv_fro2 > 4.0 * floor_ub)) return false;
    RNLA_CUDA(cudaStreamSynchronize(c->stream));
    Tm = std::move(Ri);
    kp = s;
    cholesky_T = true;
    return true;
  };
  const bool try_cholesky = kk >= s && !std::getenv("RNLA_NYSTROM_EIGW");
  // The Cholesky route, and eig(W) when it does not apply (cuSOLVER syevd,
  // latency-bound), run on the helper context from a second host thread
  // while this thread accumulates C'C (DMMA-bound), their kernels dispatched
  // from the high-priority stream.
  EigW e;
  bool need_eig = false;
  std::exception_ptr eig_err;
  const bool overlap = !std::getenv("RNLA_NYSTROM_SERIAL");
  rnla_ctx* side = overlap ? side_ctx(ctx) : nullptr;
  if (!overlap && try_cholesky) cholesky_route(ctx);
  if (!overlap) need_eig = kp == 0;
  std::thread eig_thread;
  if (overlap)
    eig_thread = std::thread([&] {
      try {
        RNLA_CUDA(cudaSetDevice(side->device));
        if (!(try_cholesky && cholesky_route(side))) {
          need_eig = true;
          e = nystrom_core(side, W.as<double>(), s, n, kk);
        }
      } catch (...) {
        eig_err = std::current_exception();
      }
    });
  struct Joiner {
    std::thread& t;
    ~Joiner() {
      if (t.joinable()) t.join();
    }
  } joiner{eig_thread};
  RNLA_CUDA(cudaMemsetAsync(G.p, 0, sizeof(double) * s * s, ctx->stream));
  // Measured on config 4 once the Gram ran on the int8 tensor cores and the
  // kernel columns on tcgen05 (8 / 16 / 24 / 32 / 40 / 44 / 48 / 56 SMs: 9.47 /
  // 9.23 / 8.65 / 8.56 / 8.43 / 8.44 / 8.48 / 8.69 ms): the faster the tensor-core
  // stages, the more of the latency-bound Cholesky route is exposed, so it gets
  // about a quarter of the SMs (r01, fp64 DMMA Gram: 16 was best).
  reserve_sms = overlap ? std::max(1, (ctx->num_sms * 40 + 74) / 148) : 0;
  if (tc_rbf) {
    c_digits(0, n_local);
    if (std::getenv("RNLA_CHECK_W_DIGITS")) {  // W's digits == the landmark rows of C's digits?
      DevBuf W2(sizeof(double) * s * s, ctx->stream);
      w_from_digits(ctx, s, L.dsel.as<int64_t>(), planes.as<int8_t>(), pitch, s * pitch, W2.as<double>());
      std::vector<double> a((size_t)(s * s)), b((size_t)(s * s));
      RNLA_CUDA(cudaMemcpyAsync(a.data(), W.p, sizeof(double) * s * s, cudaMemcpyDeviceToHost, ctx->stream));
      RNLA_CUDA(cudaMemcpyAsync(b.data(), W2.p, sizeof(double) * s * s, cudaMemcpyDeviceToHost, ctx->stream));
      RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
      std::vector<int64_t> loc(L.sel);
      int64_t bad = 0, checked = 0;
      for (int64_t t = 0; t < s; ++t) {
        if (loc[(size_t)t] < L.r_off || loc[(size_t)t] >= L.r_off + n_local) continue;
        for (int64_t j = 0; j < s; ++j, ++checked) bad += a[(size_t)(t + j * s)] != b[(size_t)(t + j * s)];
      }
      std::fprintf(stderr, "[rnla] W digits vs C landmark-row digits: %lld of %lld differ\n", (long long)bad,
                   (long long)checked);
    }
    gram_i8(ctx, planes.as<int8_t>(), n_local, s, pitch, G.as<double>(), false, reserve_sms);
  } else if (i8) {
    for (int64_t r0 = 0; r0 < n_local; r0 += rows_blk) {
      const int64_t rows = std::min(rows_blk, n_local - r0);
      c_digits(r0, rows);
      gram_i8(ctx, planes.as<int8_t>(), rows, s, pitch, G.as<double>(), r0 > 0, reserve_sms);  // synchronizes
    }
  }
  for (int64_t r0 = 0; r0 < (i8 ? 0 : n_local); r0 += blk) {
    const int64_t rows = std::min(blk, n_local - r0);
    kernel_columns<T>(ctx, X, L, r0, rows, sigma, Cb.as<T>(), 1, rows);
    if constexpr (std::is_same<T, double>::value)
      gemm<double>(ctx, s, s, rows, 1.0, Cb.as<double>(), rows, 1, Cb.as<double>(), 1, rows, 1.0, G.as<double>(), 1,
                   s);
    else
      // exact fp32 products + fp64 accumulation (DMMA): at the reference's
      // eigenvalue floor (eps * lam_max * n, src/spsd.cpp:202-205) W^+ keeps
      // eigenvalues down to ~1e-11 lam_max, which amplifies Gram errors beyond
      // what tensor-core fp32 accumulation allows (measured 5.7e-3 / 2.1 top-64
      // error with BF16x3 / BF16x6 + double-float chunks vs 3.6e-7 here).
      gemm_f32_in_f64(ctx, s, s, rows, 1.0, Cb.as<float>(), rows, 1, Cb.as<float>(), 1, rows, 1.0, G.as<double>(), 1,
                      s);
  }
  if (is_sharded(ctx)) allreduce_sum(ctx, G.p, (size_t)(s * s), RNLA_F64);  // C'C over row shards
  trace_mark(ctx, "nystrom_eig: C'C gram");
  if (overlap) {
    eig_thread.join();
    if (eig_err) std::rethrow_exception(eig_err);
    ctx->launches += side->launches;
    side->launches = 0;
  } else if (need_eig) {
    e = nystrom_core(ctx, W.as<double>(), s, n, kk);
  }
  trace_mark(ctx, kp > 0 ? "nystrom_eig: Cholesky route (overlapped)" : "nystrom_eig: eig(W)");
  if (need_eig) {
    Tm = whitened(ctx, e, s);
    kp = e.kept;
  }
  require(k >= 1 && k <= kp, "approx_eig: k exceeds rank(L)");
  // M = T' G T (kp x kp), symmetric
  DevBuf GT(sizeof(double) * s * kp, ctx->stream), M(sizeof(double) * kp * kp, ctx->stream),
      Ms(sizeof(double) * kp * kp, ctx->stream), ev(sizeof(double) * kp, ctx->stream);
  // Cholesky route: T = R^-1 is upper triangular, so G T skips k > column and
  // M = T'(G T) (symmetric) skips k > row; G is read through its symmetry as
  // K-major. Otherwise plain GEMMs.
  const bool tri = kp == s && cholesky_T;
  // Cholesky route on one GPU: both products on the int8 tensor cores with
  // exact digit products (ozaki.cu: each row of G / T' and column of T / G T
  // scaled by its own power of two, 46-bit digits), 0.83 -> see DESIGN §3.5
  const bool oz = tri && !std::getenv("RNLA_NYSTROM_DMMA_M") &&
                  ozaki_gemm_rowcol(ctx, s, s, s, G.as<double>(), s, Tm.as<double>(), s, GT.as<double>(), 1, s) &&
                  ozaki_gemm_rowcol(ctx, s, s, s, Tm.as<double>(), s, GT.as<double>(), s, M.as<double>(), 1, kp);
  if (!oz && !(tri && gemm_f64_structured(ctx, s, kp, s, G.as<double>(), s, 1, Tm.as<double>(), 1, s, GT.as<double>(), 1, s,
                                   2) &&
        gemm_f64_structured(ctx, kp, kp, s, Tm.as<double>(), s, 1, GT.as<double>(), 1, s, M.as<double>(), 1, kp,
                            1 | 4))) {
    gemm<double>(ctx, s, kp, s, 1.0, G.as<double>(), 1, s, Tm.as<double>(), 1, s, 0.0, GT.as<double>(), 1, s);
    gemm<double>(ctx, kp, kp, s, 1.0, Tm.as<double>(), s, 1, GT.as<double>(), 1, s, 0.0, M.as<double>(), 1, kp);
  }
  symmetrize(ctx, kp, M.as<double>(), Ms.as<double>());
  trace_mark(ctx, "nystrom_eig: M = T'GT");
  // Only the top k eigenpairs are needed: block subspace iteration (a few
  // n x n x 2k GEMMs) when k is well below kp, else syevdx on an index range,
  // else the full syevd.
  std::vector<double> top((size_t)k);
  DevBuf Vk(sizeof(double) * kp * k, ctx->stream);  // descending eigenvectors
  if (!eig_top_subspace(ctx, kp, Ms.as<double>(), k, top.data(), Vk.as<double>(), u_out == nullptr)) {
    const double* vtop = nullptr;  // eigenvector of the largest eigenvalue; the next ones at stride -kp
    if (2 * k <= kp && !std::getenv("RNLA_EIG_FULL")) {
      const int64_t found = eig_sym_top(ctx, kp, Ms.as<double>(), k, ev.as<double>());
      if (found != k) throw NumericError("approx_eig: partial eigensolver returned fewer pairs");
      std::vector<double> h((size_t)k);
      RNLA_CUDA(cudaMemcpyAsync(h.data(), ev.p, sizeof(double) * k, cudaMemcpyDeviceToHost, ctx->stream));
      RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
      for (int64_t t = 0; t < k; ++t) top[(size_t)t] = h[(size_t)(k - 1 - t)];
      vtop = Ms.as<double>() + (k - 1) * kp;
    } else {
      eig_sym(ctx, kp, Ms.as<double>(), ev.as<double>());
      std::vector<double> h((size_t)kp);
      RNLA_CUDA(cudaMemcpyAsync(h.data(), ev.p, sizeof(double) * kp, cudaMemcpyDeviceToHost, ctx->stream));
      RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
      for (int64_t t = 0; t < k; ++t) top[(size_t)t] = h[(size_t)(kp - 1 - t)];
      vtop = Ms.as<double>() + (kp - 1) * kp;
    }
    copy2d<double>(ctx, kp, k, vtop, 1, -kp, Vk.as<double>(), 1, kp);
  }
  for (int64_t t = 0; t < k; ++t) lam_out[t] = top[(size_t)t];
  trace_mark(ctx, "nystrom_eig: top-k eig(M)");
  if (u_out) {
    // P = T V_k diag(1/sigma) (s x k), U = C P, sign-fixed like condensed_svd's U.
    DevBuf P(sizeof(double) * s * k, ctx->stream), isg(sizeof(double) * k, ctx->stream),
        Vs(sizeof(double) * kp * k, ctx->stream);
    std::vector<double> inv((size_t)k);
    for (int64_t t = 0; t < k; ++t) inv[(size_t)t] = 1.0 / std::sqrt(top[(size_t)t]);
    RNLA_CUDA(cudaMemcpyAsync(isg.p, inv.data(), sizeof(double) * k, cudaMemcpyHostToDevice, ctx->stream));
    scale_cols_dev(ctx, kp, k, Vk.as<double>(), isg.as<double>(), Vs.as<double>());
    gemm<double>(ctx, s, k, kp, 1.0, Tm.as<double>(), 1, s, Vs.as<double>(), 1, kp, 0.0, P.as<double>(), 1, s);
    OutMat uo(ctx, u_out, n_local, k, "nystrom_eig: U", false);
    DevBuf U64(sizeof(double) * n_local * k, ctx->stream);
    DevBuf Pt;
    if constexpr (!std::is_same<T, double>::value) {
      Pt = DevBuf(sizeof(float) * s * k, ctx->stream);
      copy2d_cast<double, float>(ctx, s, k, P.as<double>(), 1, s, Pt.as<float>(), 1, s);
    }
    for (int64_t r0 = 0; r0 < n_local; r0 += blk) {
      const int64_t rows = std::min(blk, n_local - r0);
      kernel_columns<T>(ctx, X, L, r0, rows, sigma, Cb.as<T>(), 1, rows);
      if constexpr (std::is_same<T, double>::value) {
        gemm<double>(ctx, rows, k, s, 1.0, Cb.as<double>(), 1, rows, P.as<double>(), 1, s, 0.0,
                     U64.as<double>() + r0, 1, n_local);
      } else {
        DevBuf Ub(sizeof(float) * rows * k, ctx->stream);
        gemm<float>(ctx, rows, k, s, 1.f, Cb.as<float>(), 1, rows, Pt.as<float>(), 1, s, 0.f, Ub.as<float>(), 1,
                    rows);
        copy2d_cast<float, double>(ctx, rows, k, Ub.as<float>(), 1, rows, U64.as<double>() + r0, 1, n_local);
      }
    }
    fix_column_signs_sharded<double>(ctx, n_local, k, U64.as<double>(), 1, n_local, nullptr, 0, 0, 0, true);
    store_block(ctx, U64.as<double>(), n_local, k, n_local, uo);
    uo.finish(ctx);
    trace_mark(ctx, "nystrom_eig: U lift");
  }
  std::copy(L.sel.begin(), L.sel.end(), selected);
  *kept_out = kp;
  RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
}

// spsd_faster (src/spsd.cpp:131-168) on a KernelView (x = points) or a dense
// SPSD K (dense_k): C = K[:, S] -> Q = thin_qr(C).Q; secondary rows P drawn
// from the row leverage of Q (union S); Z = pinv(Q_P) K[P, P] pinv(Q_P)'.
// The factorizations run in fp64 on the device; the draws on the host.
template <class T>
void spsd_faster_impl(rnla_ctx* ctx, const rnla_mat* x, bool dense_k, double sigma, int64_t s, int64_t p,
                      uint64_t seed, const rnla_mat* q_out, const rnla_mat* z_out, int64_t* selected,
                      int64_t* secondary, int64_t* n_secondary, int32_t* flagged) {
  DevMat X = to_device(ctx, x);
  const int64_t n = X.rows;
  if (dense_k) require(X.rows == X.cols, "spsd_faster: K not square");
  require(s >= 1 && s <= p && p <= n, "spsd_faster: need s <= p <= n");
  // primary columns C = K[:, S], fp64 column-major n x s
  DevBuf C64(sizeof(double) * n * s, ctx->stream), Ct(sizeof(T) * n * s, ctx->stream);
  std::vector<int64_t> S;
  if (!dense_k) {
    Landmarks L = landmarks<T>(ctx, X, s, seed, n, 0);  // S from derive_seed(seed, 1) (src/spsd.cpp:136-137)
    S = L.sel;
    kernel_columns<T>(ctx, X, L, 0, n, sigma, Ct.as<T>(), 1, n);
  } else {
    S = sample_without_replacement_host(derive_seed(seed, 1), n, s);
    DevBuf dS(sizeof(int64_t) * s, ctx->stream);
    RNLA_CUDA(cudaMemcpyAsync(dS.p, S.data(), sizeof(int64_t) * s, cudaMemcpyHostToDevice, ctx->stream));
    gather_columns<T>(ctx, n, s, X.as<T>(), X.rs, X.cs, dS.as<int64_t>(), nullptr, Ct.as<T>(), 1, n);
    RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  if constexpr (std::is_same<T, double>::value)
    RNLA_CUDA(cudaMemcpyAsync(C64.p, Ct.p, sizeof(double) * n * s, cudaMemcpyDeviceToDevice, ctx->stream));
  else
    copy2d_cast<float, double>(ctx, n, s, Ct.as<float>(), 1, n, C64.as<double>(), 1, n);
  DevBuf R(sizeof(double) * s * s, ctx->stream);
  thin_qr_dev(ctx, n, s, C64.as<double>(), R.as<double>());  // C64 <- Q
  // secondary selection P (src/spsd.cpp:142-156)
  std::vector<int64_t> P;
  if (p == n) {
    P.resize((size_t)n);
    for (int64_t i = 0; i < n; ++i) P[(size_t)i] = i;
  } else {
    DevBuf lev(sizeof(double) * n, ctx->stream);
    row_sqnorms<double>(ctx, n, s, C64.as<double>(), 1, n, lev.as<double>());
    std::vector<double> h((size_t)n);
    RNLA_CUDA(cudaMemcpyAsync(h.data(), lev.p, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
    RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
    P = sample_with_replacement_host(derive_seed(seed, 2), h.data(), n, p);
    P.insert(P.end(), S.begin(), S.end());  // sorted_union(p_idx, selected)
    std::sort(P.begin(), P.end());
    P.erase(std::unique(P.begin(), P.end()), P.end());
  }
  const int64_t np = (int64_t)P.size();
  DevBuf dP(sizeof(int64_t) * np, ctx->stream);
  RNLA_CUDA(cudaMemcpyAsync(dP.p, P.data(), sizeof(int64_t) * np, cudaMemcpyHostToDevice, ctx->stream));
  // q_sub = Q[P, :] (np x s) and K_sub = K[P, P] (np x np), fp64 column-major
  DevBuf qsub(sizeof(double) * np * s, ctx->stream), K64(sizeof(double) * np * np, ctx->stream),
      Kt(sizeof(T) * np * np, ctx->stream);
  gather_rows<double>(ctx, np, s, C64.as<double>(), 1, n, dP.as<int64_t>(), qsub.as<double>(), 1, np);
  if (!dense_k) {
    DevMat XP = alloc_dense(ctx, np, X.cols, true, X.dtype);
    gather_rows<T>(ctx, np, X.cols, X.as<T>(), X.rs, X.cs, dP.as<int64_t>(), XP.as<T>(), XP.rs, XP.cs);
    DevBuf sqP(sizeof(T) * np, ctx->stream), ident(sizeof(int64_t) * np, ctx->stream);
    sq_norms<T>(ctx, np, X.cols, XP.as<T>(), XP.rs, XP.cs, nullptr, sqP.as<T>());
    std::vector<int64_t> id((size_t)np);
    for (int64_t i = 0; i < np; ++i) id[(size_t)i] = i;
    RNLA_CUDA(cudaMemcpyAsync(ident.p, id.data(), sizeof(int64_t) * np, cudaMemcpyHostToDevice, ctx->stream));
    rbf_block<T>(ctx, np, np, X.cols, XP.as<T>(), XP.rs, XP.cs, XP.as<T>(), XP.rs, XP.cs, nullptr, sqP.as<T>(),
                 sqP.as<T>(), sigma, ident.as<int64_t>(), Kt.as<T>(), 1, np);
    RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
  } else {
    DevBuf rowsP(sizeof(T) * np * n, ctx->stream);
    gather_rows<T>(ctx, np, n, X.as<T>(), X.rs, X.cs, dP.as<int64_t>(), rowsP.as<T>(), 1, np);
    gather_columns<T>(ctx, np, np, rowsP.as<T>(), 1, np, dP.as<int64_t>(), nullptr, Kt.as<T>(), 1, np);
  }
  if constexpr (std::is_same<T, double>::value)
    RNLA_CUDA(cudaMemcpyAsync(K64.p, Kt.p, sizeof(double) * np * np, cudaMemcpyDeviceToDevice, ctx->stream));
  else
    copy2d_cast<float, double>(ctx, np, np, Kt.as<float>(), 1, np, K64.as<double>(), 1, np);
  // rank probe (threshold 1e-10) and pinv(q_sub) (tol 1e-12) from one SVD
  DevBuf Us(sizeof(double) * np * s, ctx->stream), Sv(sizeof(double) * s, ctx->stream),
      Vs(sizeof(double) * s * s, ctx->stream), inv(sizeof(double) * s, ctx->stream),
      Vi(sizeof(double) * s * s, ctx->stream), pinv(sizeof(double) * s * np, ctx->stream),
      PK(sizeof(double) * s * np, ctx->stream), Z(sizeof(double) * s * s, ctx->stream),
      Zs(sizeof(double) * s * s, ctx->stream);
  svd_thin(ctx, np, s, qsub.as<double>(), 1, np, Us.as<double>(), Sv.as<double>(), Vs.as<double>());
  std::vector<double> hs((size_t)s), hinv((size_t)s, 0.0);
  RNLA_CUDA(cudaMemcpyAsync(hs.data(), Sv.p, sizeof(double) * s, cudaMemcpyDeviceToHost, ctx->stream));
  RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
  int64_t rank = 0;
  for (int64_t i = 0; i < s; ++i) {
    if (hs[0] > 0.0 && hs[(size_t)i] > 1e-10 * hs[0]) ++rank;
    if (hs[0] > 0.0 && hs[(size_t)i] > 1e-12 * hs[0]) hinv[(size_t)i] = 1.0 / hs[(size_t)i];
  }
  *flagged = rank < s ? 1 : 0;
  RNLA_CUDA(cudaMemcpyAsync(inv.p, hinv.data(), sizeof(double) * s, cudaMemcpyHostToDevice, ctx->stream));
  scale_cols_dev(ctx, s, s, Vs.as<double>(), inv.as<double>(), Vi.as<double>());
  gemm<double>(ctx, s, np, s, 1.0, Vi.as<double>(), 1, s, Us.as<double>(), np, 1, 0.0, pinv.as<double>(), 1, s);
  gemm<double>(ctx, s, np, np, 1.0, pinv.as<double>(), 1, s, K64.as<double>(), 1, np, 0.0, PK.as<double>(), 1, s);
  gemm<double>(ctx, s, s, np, 1.0, PK.as<double>(), 1, s, pinv.as<double>(), s, 1, 0.0, Z.as<double>(), 1, s);
  symmetrize(ctx, s, Z.as<double>(), Zs.as<double>());
  OutMat qo(ctx, q_out, n, s, "spsd_faster: Q", false), zo(ctx, z_out, s, s, "spsd_faster: Z", false);
  store_block(ctx, C64.as<double>(), n, s, n, qo);
  store_block(ctx, Zs.as<double>(), s, s, s, zo);
  qo.finish(ctx);
  zo.finish(ctx);
  std::copy(S.begin(), S.end(), selected);
  std::copy(P.begin(), P.end(), secondary);
  *n_secondary = np;
  RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
}

// pinv (tol 1e-12 sigma_1, src/core.cpp:78-88) of a column-major fp64 rows x cols
// block into out (cols x rows), and its numerical rank at 1e-10 (the reference's
// ColPivHouseholderQR threshold) -- one thin SVD of the tall orientation.
int64_t pinv_rank_dev(rnla_ctx* ctx, int64_t rows, int64_t cols, const double* A, double* out) {
  const bool wide = rows < cols;
  const int64_t m = wide ? cols : rows, n = wide ? rows : cols;  // SVD of the m x n tall view
  DevBuf U(sizeof(double) * m * n, ctx->stream), S(sizeof(double) * n, ctx->stream), V(sizeof(double) * n * n, ctx->stream),
      inv(sizeof(double) * n, ctx->stream), Vi(sizeof(double) * n * n, ctx->stream);
  if (!wide) svd_thin(ctx, m, n, A, 1, rows, U.as<double>(), S.as<double>(), V.as<double>());
  else svd_thin(ctx, m, n, A, rows, 1, U.as<double>(), S.as<double>(), V.as<double>());
  std::vector<double> hs((size_t)n), hinv((size_t)n, 0.0);
  RNLA_CUDA(cudaMemcpyAsync(hs.data(), S.p, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
  RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
  int64_t rank = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (hs[0] > 0.0 && hs[(size_t)i] > 1e-10 * hs[0]) ++rank;
    if (hs[0] > 0.0 && hs[(size_t)i] > 1e-12 * hs[0]) hinv[(size_t)i] = 1.0 / hs[(size_t)i];
  }
  RNLA_CUDA(cudaMemcpyAsync(inv.p, hinv.data(), sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
  scale_cols_dev(ctx, n, n, V.as<double>(), inv.as<double>(), Vi.as<double>());
  // tall: pinv = V S^+ U' (n x m);  wide (A' = U S V'): pinv(A) = U S^+ V' (m x n)
  if (!wide)
    gemm<double>(ctx, n, m, n, 1.0, Vi.as<double>(), 1, n, U.as<double>(), m, 1, 0.0, out, 1, n);
  else
    gemm<double>(ctx, m, n, n, 1.0, U.as<double>(), 1, m, Vi.as<double>(), n, 1, 0.0, out, 1, m);
  RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
  return rank;
}

// cur_faster_kernel (src/cur.cpp:47-104, 188-212): the implicit RBF cross
// kernel K*_ij = kappa(xtest_i, xtrain_j), uniform primary and secondary draws
// (derive_seed(seed, 1..4)), U = pinv(C[P_C, :]) K*[P_C, P_R] pinv(R[:, P_R]).
// Visits m c + r n + |P_C| |P_R| entries.
template <class T>
void cur_faster_kernel_impl(rnla_ctx* ctx, const rnla_mat* xt, const rnla_mat* xr, double sigma, int64_t c, int64_t r,
                            uint64_t seed, const rnla_mat* c_out, const rnla_mat* u_out, const rnla_mat* r_out,
                            int64_t* col_idx, int64_t* row_idx, int64_t* sec_rows, int64_t* n_sec_rows,
                            int64_t* sec_cols, int64_t* n_sec_cols, int64_t* entries, int32_t* flagged) {
  DevMat Xt = to_device(ctx, xt), Xr = to_device(ctx, xr);
  const int64_t m = Xt.rows, n = Xr.rows, d = Xt.cols;
  require(c >= 1 && c <= n, "cur: c out of [1, n]");
  require(r >= 1 && r <= m, "cur: r out of [1, m]");
  const int64_t p_c = std::min<int64_t>(2 * (c + r), m), p_r = std::min<int64_t>(2 * (c + r), n);
  const std::vector<int64_t> SC = sample_without_replacement_host(derive_seed(seed, 1), n, c);
  const std::vector<int64_t> SR = sample_without_replacement_host(derive_seed(seed, 2), m, r);
  std::vector<int64_t> PC = sample_without_replacement_host(derive_seed(seed, 3), m, p_c);
  std::vector<int64_t> PR = sample_without_replacement_host(derive_seed(seed, 4), n, p_r);
  auto unite = [](std::vector<int64_t> a, const std::vector<int64_t>& b) {
    a.insert(a.end(), b.begin(), b.end());
    std::sort(a.begin(), a.end());
    a.erase(std::unique(a.begin(), a.end()), a.end());
    return a;
  };
  PC = unite(PC, SR);
  PR = unite(PR, SC);
  const int64_t npc = (int64_t)PC.size(), npr = (int64_t)PR.size();
  auto upload = [&](const std::vector<int64_t>& v) {
    DevBuf b(sizeof(int64_t) * std::max<size_t>(v.size(), 1), ctx->stream);
    RNLA_CUDA(cudaMemcpyAsync(b.p, v.data(), sizeof(int64_t) * v.size(), cudaMemcpyHostToDevice, ctx->stream));
    return b;
  };
  DevBuf dSC = upload(SC), dSR = upload(SR), dPC = upload(PC), dPR = upload(PR);
  // squared norms: all test rows, all train rows (the cached norms of CrossKernel)
  DevBuf sqt(sizeof(T) * m, ctx->stream), sqr(sizeof(T) * n, ctx->stream);
  sq_norms<T>(ctx, m, d, Xt.as<T>(), Xt.rs, Xt.cs, nullptr, sqt.as<T>());
  sq_norms<T>(ctx, n, d, Xr.as<T>(), Xr.rs, Xr.cs, nullptr, sqr.as<T>());
  auto gather_sq = [&](const DevBuf& sq, const DevBuf& idx, int64_t cnt) {
    DevBuf g(sizeof(T) * cnt, ctx->stream);
    gather_columns<T>(ctx, 1, cnt, sq.as<T>(), 1, 1, idx.as<int64_t>(), nullptr, g.as<T>(), 1, 1);
    return g;
  };
  DevBuf sqSC = gather_sq(sqr, dSC, c), sqPR = gather_sq(sqr, dPR, npr), sqSR = gather_sq(sqt, dSR, r),
         sqPC = gather_sq(sqt, dPC, npc);
  auto to64 = [&](const DevBuf& src, int64_t cnt) {
    DevBuf o(sizeof(double) * cnt, ctx->stream);
    if constexpr (std::is_same<T, double>::value)
      RNLA_CUDA(cudaMemcpyAsync(o.p, src.p, sizeof(double) * cnt, cudaMemcpyDeviceToDevice, ctx->stream));
    else
      copy2d_cast<float, double>(ctx, cnt, 1, src.as<float>(), 1, cnt, o.as<double>(), 1, cnt);
    return o;
  };
  // C = K*[:, S_C] (m x c), R = K*[S_R, :] (r x n), block = K*[P_C, P_R]; column-major
  DevBuf Ct(sizeof(T) * m * c, ctx->stream), Rt(sizeof(T) * r * n, ctx->stream), Bt(sizeof(T) * npc * npr, ctx->stream);
  rbf_block<T>(ctx, m, c, d, Xt.as<T>(), Xt.rs, Xt.cs, Xr.as<T>(), Xr.rs, Xr.cs, dSC.as<int64_t>(), sqt.as<T>(),
               sqSC.as<T>(), sigma, nullptr, Ct.as<T>(), 1, m);
  {
    DevMat XS = alloc_dense(ctx, r, d, true, Xt.dtype);
    gather_rows<T>(ctx, r, d, Xt.as<T>(), Xt.rs, Xt.cs, dSR.as<int64_t>(), XS.as<T>(), XS.rs, XS.cs);
    rbf_block<T>(ctx, r, n, d, XS.as<T>(), XS.rs, XS.cs, Xr.as<T>(), Xr.rs, Xr.cs, nullptr, sqSR.as<T>(), sqr.as<T>(),
                 sigma, nullptr, Rt.as<T>(), 1, r);
    DevMat XP = alloc_dense(ctx, npc, d, true, Xt.dtype);
    gather_rows<T>(ctx, npc, d, Xt.as<T>(), Xt.rs, Xt.cs, dPC.as<int64_t>(), XP.as<T>(), XP.rs, XP.cs);
    rbf_block<T>(ctx, npc, npr, d, XP.as<T>(), XP.rs, XP.cs, Xr.as<T>(), Xr.rs, Xr.cs, dPR.as<int64_t>(),
                 sqPC.as<T>(), sqPR.as<T>(), sigma, nullptr, Bt.as<T>(), 1, npc);
    RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  DevBuf C64 = to64(Ct, m * c), R64 = to64(Rt, r * n), B64 = to64(Bt, npc * npr);
  // c_sub = C[P_C, :] (npc x c), r_sub = R[:, P_R] (r x npr)
  DevBuf csub(sizeof(double) * npc * c, ctx->stream), rsub(sizeof(double) * r * npr, ctx->stream),
      pc(sizeof(double) * c * npc, ctx->stream), pr(sizeof(double) * npr * r, ctx->stream),
      t1(sizeof(double) * c * npr, ctx->stream), U(sizeof(double) * c * r, ctx->stream);
  gather_rows<double>(ctx, npc, c, C64.as<double>(), 1, m, dPC.as<int64_t>(), csub.as<double>(), 1, npc);
  gather_columns<double>(ctx, r, npr, R64.as<double>(), 1, r, dPR.as<int64_t>(), nullptr, rsub.as<double>(), 1, r);
  const int64_t rank_c = pinv_rank_dev(ctx, npc, c, csub.as<double>(), pc.as<double>());
  const int64_t rank_r = pinv_rank_dev(ctx, r, npr, rsub.as<double>(), pr.as<double>());
  *flagged = (rank_c < std::min(npc, c) || rank_r < std::min(r, npr)) ? 1 : 0;
  gemm<double>(ctx, c, npr, npc, 1.0, pc.as<double>(), 1, c, B64.as<double>(), 1, npc, 0.0, t1.as<double>(), 1, c);
  gemm<double>(ctx, c, r, npr, 1.0, t1.as<double>(), 1, c, pr.as<double>(), 1, npr, 0.0, U.as<double>(), 1, c);
  OutMat co(ctx, c_out, m, c, "cur: C", false), uo(ctx, u_out, c, r, "cur: U", false), ro(ctx, r_out, r, n, "cur: R", false);
  store_block(ctx, C64.as<double>(), m, c, m, co);
  store_block(ctx, U.as<double>(), c, r, c, uo);
  store_block(ctx, R64.as<double>(), r, n, r, ro);
  co.finish(ctx);
  uo.finish(ctx);
  ro.finish(ctx);
  std::copy(SC.begin(), SC.end(), col_idx);
  std::copy(SR.begin(), SR.end(), row_idx);
  std::copy(PC.begin(), PC.end(), sec_rows);
  std::copy(PR.begin(), PR.end(), sec_cols);
  *n_sec_rows = npc;
  *n_sec_cols = npr;
  if (entries) *entries = m * c + r * n + npc * npr;
  RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
}

}  // namespace

}  // namespace rnla

using namespace rnla;

extern "C" {

rnla_status rnla_rbf_kernel(rnla_ctx* ctx, const rnla_mat* x1, const rnla_mat* x2, double sigma, rnla_mat* k) {
  return guard([&] {
    enter(ctx);
    require(sigma > 0.0, "rbf_kernel: sigma <= 0");
    check_mat(x1, "rbf_kernel: x1");
    check_mat(x2, "rbf_kernel: x2");
    require(x1->cols == x2->cols, "rbf_kernel: dimension mismatch");
    require(x1->dtype == x2->dtype, "rbf_kernel: dtype mismatch");
    const int64_t n1 = x1->rows, n2 = x2->rows, d = x1->cols;
    OutMat o(ctx, k, n1, n2, "rbf_kernel: K", false);
    require(o.dev.dtype == x1->dtype, "rbf_kernel: output dtype mismatch");
    DevMat a = to_device(ctx, x1), b = to_device(ctx, x2);
    if (x1->dtype == RNLA_F64) {
      DevBuf s1(sizeof(double) * std::max<int64_t>(n1, 1), ctx->stream), s2(sizeof(double) * std::max<int64_t>(n2, 1),
                                                                              ctx->stream);
      sq_norms<double>(ctx, n1, d, a.as<double>(), a.rs, a.cs, nullptr, s1.as<double>());
      sq_norms<double>(ctx, n2, d, b.as<double>(), b.rs, b.cs, nullptr, s2.as<double>());
      rbf_block<double>(ctx, n1, n2, d, a.as<double>(), a.rs, a.cs, b.as<double>(), b.rs, b.cs, nullptr,
                        s1.as<double>(), s2.as<double>(), sigma, nullptr, o.dev.as<double>(), o.dev.rs, o.dev.cs);
    } else {
      DevBuf s1(sizeof(float) * std::max<int64_t>(n1, 1), ctx->stream), s2(sizeof(float) * std::max<int64_t>(n2, 1),
                                                                             ctx->stream);
      sq_norms<float>(ctx, n1, d, a.as<float>(), a.rs, a.cs, nullptr, s1.as<float>());
      sq_norms<float>(ctx, n2, d, b.as<float>(), b.rs, b.cs, nullptr, s2.as<float>());
      rbf_block<float>(ctx, n1, n2, d, a.as<float>(), a.rs, a.cs, b.as<float>(), b.rs, b.cs, nullptr, s1.as<float>(),
                       s2.as<float>(), sigma, nullptr, o.dev.as<float>(), o.dev.rs, o.dev.cs);
    }
    o.finish(ctx);
  });
}

rnla_status rnla_nystrom(rnla_ctx* ctx, const rnla_mat* x, double sigma, int64_t s, uint64_t seed, int64_t target_k,
                         rnla_mat* l, int64_t* selected, int64_t* kept, int64_t* entries) {
  return guard([&] {
    enter(ctx);
    require(sigma > 0.0, "KernelView: sigma <= 0");
    check_mat(x, "nystrom: x");
    require(selected && kept, "nystrom: null output");
    if (x->dtype == RNLA_F64) nystrom_impl<double>(ctx, x, sigma, s, seed, target_k, l, selected, kept, entries);
    else nystrom_impl<float>(ctx, x, sigma, s, seed, target_k, l, selected, kept, entries);
  });
}

rnla_status rnla_nystrom_dense(rnla_ctx* ctx, const rnla_mat* k, int64_t s, uint64_t seed, int64_t target_k,
                               rnla_mat* l, int64_t* selected, int64_t* kept) {
  return guard([&] {
    enter(ctx);
    check_mat(k, "nystrom: K");
    require(selected && kept, "nystrom: null output");
    require(ctx->world == 1, "nystrom: row-sharded contexts use nystrom_eig");
    if (k->dtype == RNLA_F64) nystrom_dense_impl<double>(ctx, k, s, seed, target_k, l, selected, kept);
    else nystrom_dense_impl<float>(ctx, k, s, seed, target_k, l, selected, kept);
  });
}

rnla_status rnla_nystrom_columns(rnla_ctx* ctx, const rnla_mat* c, const int64_t* selected, int64_t target_k,
                                 rnla_mat* l, int64_t* kept) {
  return guard([&] {
    enter(ctx);
    check_mat(c, "nystrom: C");
    require(selected && kept, "nystrom: null argument");
    require(ctx->world == 1, "nystrom: row-sharded contexts use nystrom_eig");
    if (c->dtype == RNLA_F64) nystrom_columns_impl<double>(ctx, c, selected, target_k, l, kept);
    else nystrom_columns_impl<float>(ctx, c, selected, target_k, l, kept);
  });
}

rnla_status rnla_approx_eig(rnla_ctx* ctx, const rnla_mat* l, int64_t k, rnla_mat* u, double* lam) {
  return guard([&] {
    enter(ctx);
    check_mat(l, "approx_eig: l");
    require(k >= 1 && k <= l->cols, "approx_eig: k > cols(L)");
    require(lam != nullptr, "approx_eig: null output");
    const int64_t m = l->rows, n = l->cols;
    DevMat w = f64_colmajor(ctx, l);
    SvdDev f = condensed_svd_dev(ctx, m, n, w.as<double>(), w.rs, w.cs);
    if (k > f.rank) throw InvalidArgument("approx_eig: k exceeds rank(L)");
    OutMat uo(ctx, u, m, k, "approx_eig: U", false);
    store_block(ctx, f.U.as<double>(), m, k, m, uo);
    for (int64_t i = 0; i < k; ++i) lam[i] = f.s[(size_t)i] * f.s[(size_t)i];
    uo.finish(ctx);
  });
}

rnla_status rnla_nystrom_eig(rnla_ctx* ctx, const rnla_mat* x, double sigma, int64_t s, uint64_t seed,
                             int64_t target_k, int64_t k, rnla_mat* u, double* lam, int64_t* selected,
                             int64_t* kept) {
  return guard([&] {
    enter(ctx);
    require(sigma > 0.0, "KernelView: sigma <= 0");
    check_mat(x, "nystrom_eig: x");
    require(lam && selected && kept, "nystrom_eig: null output");
    require(k >= 1, "approx_eig: k > cols(L)");
    if (x->dtype == RNLA_F64) nystrom_eig_impl<double>(ctx, x, sigma, s, seed, target_k, k, u, lam, selected, kept);
    else nystrom_eig_impl<float>(ctx, x, sigma, s, seed, target_k, k, u, lam, selected, kept);
  });
}

rnla_status rnla_spsd_faster(rnla_ctx* ctx, const rnla_mat* x, double sigma, int64_t s, int64_t p, uint64_t seed,
                             rnla_mat* q, rnla_mat* z, int64_t* selected, int64_t* secondary, int64_t* n_secondary,
                             int32_t* flagged) {
  return guard([&] {
    enter(ctx);
    require(sigma > 0.0, "KernelView: sigma <= 0");
    check_mat(x, "spsd_faster: x");
    require(ctx->world == 1, "spsd_faster: row-sharded contexts are not supported");
    require(selected && secondary && n_secondary && flagged, "spsd_faster: null output");
    if (x->dtype == RNLA_F64)
      spsd_faster_impl<double>(ctx, x, false, sigma, s, p, seed, q, z, selected, secondary, n_secondary, flagged);
    else
      spsd_faster_impl<float>(ctx, x, false, sigma, s, p, seed, q, z, selected, secondary, n_secondary, flagged);
  });
}

rnla_status rnla_spsd_faster_dense(rnla_ctx* ctx, const rnla_mat* k, int64_t s, int64_t p, uint64_t seed, rnla_mat* q,
                                   rnla_mat* z, int64_t* selected, int64_t* secondary, int64_t* n_secondary,
                                   int32_t* flagged) {
  return guard([&] {
    enter(ctx);
    check_mat(k, "spsd_faster: k");
    require(ctx->world == 1, "spsd_faster: row-sharded contexts are not supported");
    require(selected && secondary && n_secondary && flagged, "spsd_faster: null output");
    if (k->dtype == RNLA_F64)
      spsd_faster_impl<double>(ctx, k, true, 1.0, s, p, seed, q, z, selected, secondary, n_secondary, flagged);
    else
      spsd_faster_impl<float>(ctx, k, true, 1.0, s, p, seed, q, z, selected, secondary, n_secondary, flagged);
  });
}

rnla_status rnla_cur_faster_kernel(rnla_ctx* ctx, const rnla_mat* xtest, const rnla_mat* xtrain, double sigma,
                                   int64_t c, int64_t r, uint64_t seed, rnla_mat* cmat, rnla_mat* umat, rnla_mat* rmat,
                                   int64_t* col_idx, int64_t* row_idx, int64_t* sec_rows, int64_t* n_sec_rows,
                                   int64_t* sec_cols, int64_t* n_sec_cols, int64_t* entries, int32_t* flagged) {
  return guard([&] {
    enter(ctx);
    require(sigma > 0.0, "cur_faster_kernel: sigma <= 0");
    check_mat(xtest, "cur_faster_kernel: xtest");
    check_mat(xtrain, "cur_faster_kernel: xtrain");
    require(xtest->cols == xtrain->cols, "cur_faster_kernel: dimension mismatch");
    require(xtest->dtype == xtrain->dtype, "cur_faster_kernel: dtype mismatch");
    require(ctx->world == 1, "cur_faster_kernel: row-sharded contexts are not supported");
    require(col_idx && row_idx && sec_rows && n_sec_rows && sec_cols && n_sec_cols && flagged,
            "cur_faster_kernel: null output");
    if (xtest->dtype == RNLA_F64)
      cur_faster_kernel_impl<double>(ctx, xtest, xtrain, sigma, c, r, seed, cmat, umat, rmat, col_idx, row_idx,
                                     sec_rows, n_sec_rows, sec_cols, n_sec_cols, entries, flagged);
    else
      cur_faster_kernel_impl<float>(ctx, xtest, xtrain, sigma, c, r, seed, cmat, umat, rmat, col_idx, row_idx,
                                    sec_rows, n_sec_rows, sec_cols, n_sec_cols, entries, flagged);
  });
}

}  // extern "C"
