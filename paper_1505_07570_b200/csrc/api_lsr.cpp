// api_lsr.cpp -- sketch-and-precondition least squares behind the C ABI.
//
// Reference: lsr_preconditioned, /root/reference/proj/src/regression.cpp:94-198
// (include/randnla/regression.hpp:20-56). The sketch of [A, b] is the
// library's row sketch (CountSketch by default, bit-exact in fp64), the QR of
// Y = S'A is cuSOLVER Householder with the reference's sign rule, and every
// iteration is ONE fused pass over A (lsr.cu normal_gemv: A'(b - A T z)).
// The d-vector work (triangular solves with R_Y, z updates, norms) runs on
// the host in fp64 exactly as the reference writes it; A never leaves HBM.
// Row-sharded A: the pass partials g and |r|^2 are allreduced.
#include <cmath>
#include <limits>

#include "algos.h"
#include "dist.h"
#include "linalg.cuh"
#include "marshal.h"

namespace rnla {

namespace {

using HVec = std::vector<double>;

// R (d x d upper, column-major host) triangular solves: R v = u, R' v = u.
HVec solve_upper(const HVec& R, int64_t d, const HVec& u) {
  HVec v(u);
  for (int64_t i = d - 1; i >= 0; --i) {
    double s = v[(size_t)i];
    for (int64_t j = i + 1; j < d; ++j) s -= R[(size_t)(i + j * d)] * v[(size_t)j];
    v[(size_t)i] = s / R[(size_t)(i + i * d)];
  }
  return v;
}
HVec solve_upper_t(const HVec& R, int64_t d, const HVec& u) {
  HVec v(u);
  for (int64_t i = 0; i < d; ++i) {
    double s = v[(size_t)i];
    for (int64_t j = 0; j < i; ++j) s -= R[(size_t)(j + i * d)] * v[(size_t)j];
    v[(size_t)i] = s / R[(size_t)(i + i * d)];
  }
  return v;
}
double norm2(const HVec& v) {
  double s = 0.0;
  for (double x : v) s += x * x;
  return std::sqrt(s);
}
double dot(const HVec& a, const HVec& b) {
  double s = 0.0;
  for (size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
  return s;
}

template <class T>
struct Pass {
  rnla_ctx* ctx;
  const DevMat& A;
  const T* b;
  int64_t b_stride, n, d;
  DevBuf w, g, rr;
  Pass(rnla_ctx* c, const DevMat& a, const T* b_, int64_t bs)
      : ctx(c), A(a), b(b_), b_stride(bs), n(a.rows), d(a.cols), w(sizeof(double) * a.cols, c->stream),
        g(sizeof(double) * a.cols, c->stream), rr(sizeof(double), c->stream) {}
  // returns A'(beta b - A x) (summed over shards); *res2 = |beta b - A x|^2
  HVec operator()(double beta, const HVec& x, double* res2 = nullptr) {
    RNLA_CUDA(cudaMemcpyAsync(w.p, x.data(), sizeof(double) * d, cudaMemcpyHostToDevice, ctx->stream));
    normal_gemv<T>(ctx, n, d, A.as<T>(), A.rs, b, b_stride, beta, w.as<double>(), g.as<double>(), rr.as<double>());
    if (is_sharded(ctx)) {
      allreduce_sum(ctx, g.p, (size_t)d, RNLA_F64);
      allreduce_sum(ctx, rr.p, 1, RNLA_F64);
    }
    HVec out((size_t)d);
    double r2 = 0.0;
    RNLA_CUDA(cudaMemcpyAsync(out.data(), g.p, sizeof(double) * d, cudaMemcpyDeviceToHost, ctx->stream));
    RNLA_CUDA(cudaMemcpyAsync(&r2, rr.p, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
    if (res2) *res2 = r2;
    return out;
  }
};

template <class T>
void lsr_preconditioned_impl(rnla_ctx* ctx, const rnla_mat* a, const rnla_mat* b, double eps, uint64_t seed,
                             int64_t sketch_size, int32_t use_cg, int32_t kind, double* x_out, double* objective,
                             int32_t* iterations, double* kappa) {
  const int64_t n = a->rows, d = a->cols;
  int64_t total = n;
  const int64_t off = global_row_offset(ctx, n, &total);
  require(total >= d, "lsr_preconditioned: n < d");
  int64_t s = sketch_size;
  if (s == 0) s = std::min(d * d, 20 * d);
  s = std::min(s, total);
  require(s >= d, "lsr_preconditioned: sketch size < d");
  DevMat A = as_rowmajor(ctx, to_device(ctx, a));
  DevMat B = to_device(ctx, b);
  const int dt = a->dtype;

  // Sketch [A, b] (s x (d+1)); R_Y singular: resample once with a derived seed.
  DevMat sk = alloc_dense(ctx, s, d + 1, true, dt);
  DevBuf Y(sizeof(double) * s * d, ctx->stream), R(sizeof(double) * d * d, ctx->stream),
      sb(sizeof(double) * s, ctx->stream);
  HVec Rh((size_t)(d * d));
  uint64_t draw_seed = seed;
  for (int attempt = 0;; ++attempt) {
    rnla_sketch_spec spec{};
    spec.kind = kind;
    spec.s = s;
    spec.seed = draw_seed;
    if (kind == RNLA_SKETCH_COUNT) {
      sketch_rows_dev<T>(ctx, A.as<T>(), A.rs, B.as<T>(), B.rs, n, d, &spec, off, sk.as<T>(), d + 1, 1);
    } else {
      // dense sketches take the stacked [A, b]
      DevMat st = alloc_dense(ctx, n, d + 1, true, dt);
      copy2d<T>(ctx, n, d, A.as<T>(), A.rs, 1, st.as<T>(), d + 1, 1);
      copy2d<T>(ctx, n, 1, B.as<T>(), B.rs, 1, st.as<T>() + d, d + 1, 1);
      sketch_rows_dev<T>(ctx, st.as<T>(), d + 1, nullptr, 1, n, d + 1, &spec, off, sk.as<T>(), d + 1, 1);
    }
    if (dt == RNLA_F64) {
      copy2d<double>(ctx, s, d, sk.as<double>(), d + 1, 1, Y.as<double>(), 1, s);
      copy2d<double>(ctx, s, 1, sk.as<double>() + d, d + 1, 1, sb.as<double>(), 1, s);
    } else {
      copy2d_cast<float, double>(ctx, s, d, sk.as<float>(), d + 1, 1, Y.as<double>(), 1, s);
      copy2d_cast<float, double>(ctx, s, 1, sk.as<float>() + d, d + 1, 1, sb.as<double>(), 1, s);
    }
    thin_qr_dev(ctx, s, d, Y.as<double>(), R.as<double>());
    RNLA_CUDA(cudaMemcpyAsync(Rh.data(), R.p, sizeof(double) * d * d, cudaMemcpyDeviceToHost, ctx->stream));
    RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
    double dmin = std::numeric_limits<double>::infinity(), dmax = 0.0;
    for (int64_t i = 0; i < d; ++i) {
      const double v = std::fabs(Rh[(size_t)(i + i * d)]);
      dmin = std::min(dmin, v);
      dmax = std::max(dmax, v);
    }
    if (dmax > 0.0 && dmin > 1e-12 * dmax) break;
    if (attempt >= 1) throw NumericError("lsr_preconditioned: sketched matrix singular");
    draw_seed = derive_seed(seed, 0x5e5a);
  }
  // z0 = Q_Y' S'b
  HVec z((size_t)d);
  {
    DevBuf zd(sizeof(double) * d, ctx->stream);
    gemm<double>(ctx, d, 1, s, 1.0, Y.as<double>(), s, 1, sb.as<double>(), 1, s, 0.0, zd.as<double>(), 1, d);
    RNLA_CUDA(cudaMemcpyAsync(z.data(), zd.p, sizeof(double) * d, cudaMemcpyDeviceToHost, ctx->stream));
    RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  Pass<T> pass(ctx, A, B.as<T>(), B.rs);
  auto apply_t = [&](const HVec& v) { return solve_upper(Rh, d, v); };
  auto apply_tt = [&](const HVec& v) { return solve_upper_t(Rh, d, v); };
  const int budget = (int)std::ceil(10.0 * std::log10(1.0 / eps));
  const HVec zero((size_t)d, 0.0);
  const double grad_scale = norm2(apply_tt(pass(1.0, zero)));  // |T' A' b|
  const double grad_tol = std::max(1e-15 * grad_scale, 1e-300);
  int it = 0;
  if (!use_cg) {
    // gradient descent with unit step (regression.cpp:151-167)
    double prev = std::numeric_limits<double>::infinity();
    for (; it < budget; ++it) {
      const HVec grad = apply_tt(pass(1.0, apply_t(z)));
      for (int64_t i = 0; i < d; ++i) z[(size_t)i] += grad[(size_t)i];
      const double gn = norm2(grad);
      if (gn <= grad_tol || gn >= 0.9 * prev) {
        ++it;
        break;
      }
      prev = gn;
    }
  } else {
    // CG on the normal equations of (AT) z = b (regression.cpp:168-183)
    HVec r = apply_tt(pass(1.0, apply_t(z)));
    HVec p = r;
    double rs = dot(r, r);
    for (; it < budget && std::sqrt(rs) > grad_tol; ++it) {
      HVec ap = apply_tt(pass(0.0, apply_t(p)));  // = -T'A'A T p
      for (auto& v : ap) v = -v;
      const double alpha = rs / dot(p, ap);
      for (int64_t i = 0; i < d; ++i) {
        z[(size_t)i] += alpha * p[(size_t)i];
        r[(size_t)i] -= alpha * ap[(size_t)i];
      }
      const double rs_new = dot(r, r);
      for (int64_t i = 0; i < d; ++i) p[(size_t)i] = r[(size_t)i] + (rs_new / rs) * p[(size_t)i];
      rs = rs_new;
    }
  }
  const HVec x = apply_t(z);
  std::copy(x.begin(), x.end(), x_out);
  *iterations = it;
  if (objective) {
    double r2 = 0.0;
    pass(1.0, x, &r2);
    *objective = r2;
  }
  if (kappa) {
    // kappa(A T) (diagnostic): singular values of A T from eig(T' (A'A) T);
    // A T is well conditioned (kappa <= ~2), so the Gram route is accurate.
    DevBuf G(sizeof(double) * d * d, ctx->stream), Tm(sizeof(double) * d * d, ctx->stream),
        GT(sizeof(double) * d * d, ctx->stream), M(sizeof(double) * d * d, ctx->stream),
        ev(sizeof(double) * d, ctx->stream);
    if (dt == RNLA_F64)
      gemm<double>(ctx, d, d, n, 1.0, A.as<double>(), 1, A.rs, A.as<double>(), A.rs, 1, 0.0, G.as<double>(), 1, d);
    else  // exact products + fp64 accumulation: T'GT amplifies Gram errors by |T|^2
      gemm_f32_in_f64(ctx, d, d, n, 1.0, A.as<float>(), 1, A.rs, A.as<float>(), A.rs, 1, 0.0, G.as<double>(), 1, d);
    if (is_sharded(ctx)) allreduce_sum(ctx, G.p, (size_t)(d * d), RNLA_F64);
    upper_inverse(ctx, d, R.as<double>(), Tm.as<double>());
    gemm<double>(ctx, d, d, d, 1.0, G.as<double>(), 1, d, Tm.as<double>(), 1, d, 0.0, GT.as<double>(), 1, d);
    gemm<double>(ctx, d, d, d, 1.0, Tm.as<double>(), d, 1, GT.as<double>(), 1, d, 0.0, M.as<double>(), 1, d);
    eig_sym(ctx, d, M.as<double>(), ev.as<double>());
    HVec h((size_t)d);
    RNLA_CUDA(cudaMemcpyAsync(h.data(), ev.p, sizeof(double) * d, cudaMemcpyDeviceToHost, ctx->stream));
    RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
    *kappa = h[0] > 0.0 ? std::sqrt(h[(size_t)d - 1] / h[0]) : std::numeric_limits<double>::infinity();
  }
}

// lsr_cg (src/regression.cpp:38-66): CG on A'A x = A'b; every iteration's
// A'(A p) is one fused pass (beta = 0 gives -A'A p).
template <class T>
void lsr_cg_impl(rnla_ctx* ctx, const rnla_mat* a, const rnla_mat* b, double tol, int32_t maxit, double* x_out,
                 double* objective, int32_t* iterations, int32_t* converged) {
  const int64_t n = a->rows, d = a->cols;
  int64_t total = n;
  global_row_offset(ctx, n, &total);
  require(total >= d, "lsr_cg: n < d");
  DevMat A = as_rowmajor(ctx, to_device(ctx, a));
  DevMat B = to_device(ctx, b);
  Pass<T> pass(ctx, A, B.as<T>(), B.rs);
  HVec x((size_t)d, 0.0);
  HVec r = pass(1.0, x);  // A'b
  const double target = tol * norm2(r);
  HVec p = r;
  double rs = dot(r, r);
  int it = 0;
  bool conv = std::sqrt(rs) <= target;
  while (it < maxit && std::sqrt(rs) > target) {
    HVec ap = pass(0.0, p);
    for (auto& v : ap) v = -v;
    const double alpha = rs / dot(p, ap);
    for (int64_t i = 0; i < d; ++i) {
      x[(size_t)i] += alpha * p[(size_t)i];
      r[(size_t)i] -= alpha * ap[(size_t)i];
    }
    const double rs_new = dot(r, r);
    for (int64_t i = 0; i < d; ++i) p[(size_t)i] = r[(size_t)i] + (rs_new / rs) * p[(size_t)i];
    rs = rs_new;
    ++it;
    conv = std::sqrt(rs) <= target;
  }
  std::copy(x.begin(), x.end(), x_out);
  *iterations = it;
  if (converged) *converged = conv ? 1 : 0;
  if (objective) {
    double r2 = 0.0;
    pass(1.0, x, &r2);
    *objective = r2;
  }
}

}  // namespace

}  // namespace rnla

using namespace rnla;

extern "C" rnla_status rnla_lsr_cg(rnla_ctx* ctx, const rnla_mat* a, const rnla_mat* b, double tol, int32_t maxit,
                                   double* x, double* objective, int32_t* iterations, int32_t* converged) {
  return guard([&] {
    enter(ctx);
    check_mat(a, "lsr_cg: a");
    check_mat(b, "lsr_cg: b");
    require(a->rows == b->rows && b->cols == 1, "lsr_cg: dimension mismatch");
    require(a->dtype == b->dtype, "lsr_cg: a and b dtypes differ");
    require(x != nullptr && iterations != nullptr, "lsr_cg: null output");
    require(normal_gemv_supported(a->cols), "lsr_cg: d above 1024 is not supported");
    if (a->dtype == RNLA_F64) lsr_cg_impl<double>(ctx, a, b, tol, maxit, x, objective, iterations, converged);
    else lsr_cg_impl<float>(ctx, a, b, tol, maxit, x, objective, iterations, converged);
  });
}

using namespace rnla;

extern "C" rnla_status rnla_lsr_preconditioned(rnla_ctx* ctx, const rnla_mat* a, const rnla_mat* b, double eps,
                                               uint64_t seed, int64_t sketch_size, int32_t use_cg,
                                               int32_t sketch_kind, double* x, double* objective,
                                               int32_t* iterations, double* kappa_estimate) {
  return guard([&] {
    enter(ctx);
    check_mat(a, "lsr_preconditioned: a");
    check_mat(b, "lsr_preconditioned: b");
    require(a->rows == b->rows && b->cols == 1, "lsr_preconditioned: dimension mismatch");
    require(eps > 0.0 && eps < 1.0, "lsr_preconditioned: eps out of (0,1)");
    require(sketch_size >= 0, "lsr_preconditioned: sketch size < d");
    require(a->dtype == b->dtype, "lsr_preconditioned: a and b dtypes differ");
    require(x != nullptr && iterations != nullptr, "lsr_preconditioned: null output");
    require(sketch_kind == RNLA_SKETCH_COUNT || sketch_kind == RNLA_SKETCH_GAUSSIAN || sketch_kind == RNLA_SKETCH_SRHT,
            "lsr_preconditioned: sketch kind must be count, gaussian or srht");
    require(normal_gemv_supported(a->cols), "lsr_preconditioned: d above 1024 is not supported");
    if (a->dtype == RNLA_F64)
      lsr_preconditioned_impl<double>(ctx, a, b, eps, seed, sketch_size, use_cg, sketch_kind, x, objective,
                                      iterations, kappa_estimate);
    else
      lsr_preconditioned_impl<float>(ctx, a, b, eps, seed, sketch_size, use_cg, sketch_kind, x, objective,
                                     iterations, kappa_estimate);
  });
}
