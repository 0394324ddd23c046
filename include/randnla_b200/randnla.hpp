// randnla.hpp -- header-only C++ facade over the C ABI (include/rnla.h).
//
// Mirrors the reference's C++ hot-path API (/root/reference/proj/include/
// randnla/{rng,sketch,core,randsvd,regression,spsd}.hpp): same function names,
// argument order and meaning, value-returning results, and the same
// exception types (std::invalid_argument for require() failures,
// std::runtime_error for numerical failures). A reference caller switches by
// including this header instead of the reference headers and linking
// librnla_b200.so; see INTEGRATION.md.
//
// Matrices: randnla_b200::DenseMatrix is a column-major double matrix with
// the Eigen::MatrixXd accessors the reference code uses (rows(), cols(),
// data(), operator()(i, j)). Define RANDNLA_B200_USE_EIGEN before including
// to make DenseMatrix = Eigen::MatrixXd and Vector = Eigen::VectorXd instead.
#pragma once

#include <cmath>
#include <cstdint>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "rnla.h"

#ifdef RANDNLA_B200_USE_EIGEN
#include <Eigen/Dense>
#endif

namespace randnla_b200 {

using Index = std::int64_t;

#ifdef RANDNLA_B200_USE_EIGEN
using DenseMatrix = Eigen::MatrixXd;
using Vector = Eigen::VectorXd;
#else
class DenseMatrix {
 public:
  DenseMatrix() = default;
  DenseMatrix(Index r, Index c) : r_(r), c_(c), v_(static_cast<size_t>(r * c), 0.0) {}
  Index rows() const { return r_; }
  Index cols() const { return c_; }
  double* data() { return v_.data(); }
  const double* data() const { return v_.data(); }
  double& operator()(Index i, Index j) { return v_[static_cast<size_t>(i + j * r_)]; }
  double operator()(Index i, Index j) const { return v_[static_cast<size_t>(i + j * r_)]; }
  static DenseMatrix Zero(Index r, Index c) { return DenseMatrix(r, c); }
  void conservativeResizeCols(Index c) {
    v_.resize(static_cast<size_t>(r_ * c));
    c_ = c;
  }

 private:
  Index r_ = 0, c_ = 0;
  std::vector<double> v_;
};
class Vector {
 public:
  Vector() = default;
  explicit Vector(Index n) : v_(static_cast<size_t>(n), 0.0) {}
  Index size() const { return static_cast<Index>(v_.size()); }
  double* data() { return v_.data(); }
  const double* data() const { return v_.data(); }
  double& operator()(Index i) { return v_[static_cast<size_t>(i)]; }
  double operator()(Index i) const { return v_[static_cast<size_t>(i)]; }
  void resize(Index n) { v_.resize(static_cast<size_t>(n)); }

 private:
  std::vector<double> v_;
};
#endif

struct SvdFactors {
  DenseMatrix U;
  Vector singular_values;
  DenseMatrix V;
  Index rank() const { return singular_values.size(); }
};
struct QrFactors {
  DenseMatrix Q;
  DenseMatrix R;
};

namespace detail {
inline void check(rnla_status st) {
  if (st == RNLA_OK) return;
  const std::string msg = rnla_last_error();
  if (st == RNLA_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}
inline rnla_mat view(const DenseMatrix& m) {
  return rnla_mat{const_cast<double*>(m.data()), m.rows(), m.cols(), 1, m.rows() > 0 ? m.rows() : 1, RNLA_F64, 0};
}
inline rnla_mat view(const Vector& v) {
  return rnla_mat{const_cast<double*>(v.data()), v.size(), 1, 1, v.size() > 0 ? v.size() : 1, RNLA_F64, 0};
}
// One context per thread (the reference is reentrant; so is the ABI per context).
inline rnla_ctx* ctx() {
  struct Holder {
    rnla_ctx* c = nullptr;
    ~Holder() { rnla_ctx_destroy(c); }
  };
  thread_local Holder h;
  if (!h.c) check(rnla_ctx_create(0, &h.c));
  return h.c;
}
}  // namespace detail

// ---------------- rng.hpp ----------------
inline std::uint64_t splitmix64(std::uint64_t& state) { return rnla_splitmix64(&state); }
inline std::uint64_t derive_seed(std::uint64_t seed, std::uint64_t stream) { return rnla_derive_seed(seed, stream); }
inline std::vector<Index> sample_without_replacement(Index n, Index count, std::uint64_t seed) {
  std::vector<Index> out(static_cast<size_t>(count));
  detail::check(rnla_sample_without_replacement(seed, n, count, out.data()));
  return out;
}

// ---------------- sketch.hpp ----------------
enum class SketchKind { kGaussian, kSrht, kCountSketch, kUniformColumns, kLeverageColumns, kLandmarkColumns, kCombined };

struct SketchSpec {
  SketchKind kind = SketchKind::kGaussian;
  Index s = 1;
  std::uint64_t seed = 0;
  std::shared_ptr<const SketchSpec> stage2;
  bool scale_columns = false;
  std::optional<Index> leverage_rank;

  static SketchSpec gaussian(Index s, std::uint64_t seed) { return {SketchKind::kGaussian, s, seed, nullptr, false, {}}; }
  static SketchSpec srht(Index s, std::uint64_t seed) { return {SketchKind::kSrht, s, seed, nullptr, false, {}}; }
  static SketchSpec count_sketch(Index s, std::uint64_t seed) {
    return {SketchKind::kCountSketch, s, seed, nullptr, false, {}};
  }
  static SketchSpec uniform_columns(Index s, std::uint64_t seed) {
    return {SketchKind::kUniformColumns, s, seed, nullptr, false, {}};
  }
  static SketchSpec combined(Index s_cs, SketchSpec dense_stage, std::uint64_t seed) {
    SketchSpec sp;
    sp.kind = SketchKind::kCombined;
    sp.s = s_cs;
    sp.seed = seed;
    sp.stage2 = std::make_shared<const SketchSpec>(std::move(dense_stage));
    return sp;
  }
  rnla_sketch_spec to_c() const {
    rnla_sketch_spec c{};
    c.kind = static_cast<int32_t>(kind);
    c.s = s;
    c.seed = seed;
    if (stage2) {
      c.stage2_kind = static_cast<int32_t>(stage2->kind);
      c.stage2_s = stage2->s;
      c.stage2_seed = stage2->seed;
    }
    c.scale_columns = scale_columns ? 1 : 0;
    c.leverage_rank = leverage_rank ? *leverage_rank : 0;
    return c;
  }
};

inline DenseMatrix gaussian_sketch(const DenseMatrix& a, Index s, std::uint64_t seed) {
  if (s < 1) throw std::invalid_argument("gaussian_sketch: s < 1");
  DenseMatrix c(a.rows(), s);
  rnla_mat am = detail::view(a), cm = detail::view(c);
  detail::check(rnla_gaussian_sketch(detail::ctx(), &am, s, seed, &cm));
  return c;
}
inline DenseMatrix srht_sketch(const DenseMatrix& a, Index s, std::uint64_t seed) {
  DenseMatrix c(a.rows(), s);
  rnla_mat am = detail::view(a), cm = detail::view(c);
  detail::check(rnla_srht_sketch(detail::ctx(), &am, s, seed, &cm));
  return c;
}
inline DenseMatrix count_sketch(const DenseMatrix& a, Index s, std::uint64_t seed) {
  if (s < 1) throw std::invalid_argument("count_sketch: s < 1");
  DenseMatrix c(a.rows(), s);
  rnla_mat am = detail::view(a), cm = detail::view(c);
  detail::check(rnla_count_sketch(detail::ctx(), &am, s, seed, &cm));
  return c;
}
inline DenseMatrix combined_sketch(const DenseMatrix& a, const SketchSpec& spec) {
  if (spec.kind != SketchKind::kCombined || !spec.stage2)
    throw std::invalid_argument("combined_sketch: spec is not a combined sketch");
  DenseMatrix c(a.rows(), spec.stage2->s);
  rnla_mat am = detail::view(a), cm = detail::view(c);
  rnla_sketch_spec cs = spec.to_c();
  detail::check(rnla_combined_sketch(detail::ctx(), &am, &cs, &cm));
  return c;
}
inline DenseMatrix apply_sketch(const DenseMatrix& a, const SketchSpec& spec) {
  rnla_sketch_spec cs = spec.to_c();
  const Index width = spec.kind == SketchKind::kCombined ? (spec.stage2 ? spec.stage2->s : 0) : spec.s;
  DenseMatrix c(a.rows(), width);
  rnla_mat am = detail::view(a), cm = detail::view(c);
  Index cols = width;
  detail::check(rnla_apply_sketch(detail::ctx(), &am, &cs, &cm, &cols));
#ifndef RANDNLA_B200_USE_EIGEN
  if (cols < width) c.conservativeResizeCols(cols);
#else
  if (cols < width) c.conservativeResize(Eigen::NoChange, cols);
#endif
  return c;
}

// ---------------- core.hpp ----------------
inline QrFactors thin_qr(const DenseMatrix& a) {
  if (a.rows() < a.cols()) throw std::invalid_argument("thin_qr: rows < cols");
  QrFactors f{DenseMatrix(a.rows(), a.cols()), DenseMatrix(a.cols(), a.cols())};
  rnla_mat am = detail::view(a), qm = detail::view(f.Q), rm = detail::view(f.R);
  detail::check(rnla_thin_qr(detail::ctx(), &am, &qm, &rm));
  return f;
}

inline SvdFactors truncated_svd(const DenseMatrix& a, Index k) {
  if (k < 1 || k > std::min(a.rows(), a.cols())) throw std::invalid_argument("truncated_svd: k out of range");
  DenseMatrix u(a.rows(), k), v(a.cols(), k);
  std::vector<double> sv(static_cast<size_t>(k));
  Index rank = 0;
  rnla_mat am = detail::view(a), um = detail::view(u), vm = detail::view(v);
  detail::check(rnla_truncated_svd(detail::ctx(), &am, k, &um, sv.data(), &vm, &rank));
  SvdFactors f;
  f.U = DenseMatrix(a.rows(), rank);
  f.V = DenseMatrix(a.cols(), rank);
  f.singular_values = Vector(rank);
  for (Index j = 0; j < rank; ++j) {
    f.singular_values(j) = sv[static_cast<size_t>(j)];
    for (Index i = 0; i < a.rows(); ++i) f.U(i, j) = u(i, j);
    for (Index i = 0; i < a.cols(); ++i) f.V(i, j) = v(i, j);
  }
  return f;
}

inline SvdFactors condensed_svd(const DenseMatrix& a) {
  const Index r = std::min(a.rows(), a.cols());
  DenseMatrix u(a.rows(), r), v(a.cols(), r);
  std::vector<double> sv(static_cast<size_t>(std::max<Index>(r, 1)));
  Index rank = 0;
  rnla_mat am = detail::view(a), um = detail::view(u), vm = detail::view(v);
  detail::check(rnla_condensed_svd(detail::ctx(), &am, &um, sv.data(), &vm, &rank));
  SvdFactors f;
  f.U = DenseMatrix(a.rows(), rank);
  f.V = DenseMatrix(a.cols(), rank);
  f.singular_values = Vector(rank);
  for (Index j = 0; j < rank; ++j) {
    f.singular_values(j) = sv[static_cast<size_t>(j)];
    for (Index i = 0; i < a.rows(); ++i) f.U(i, j) = u(i, j);
    for (Index i = 0; i < a.cols(); ++i) f.V(i, j) = v(i, j);
  }
  return f;
}

inline DenseMatrix pseudo_inverse(const DenseMatrix& a, double tol = 1e-12) {
  DenseMatrix p(a.cols(), a.rows());
  rnla_mat am = detail::view(a), pm = detail::view(p);
  detail::check(rnla_pseudo_inverse(detail::ctx(), &am, tol, &pm));
  return p;
}

// ---------------- randsvd.hpp ----------------
struct KsvdResult {
  SvdFactors factors;
  int passes_over_a = 0;
  std::optional<double> error_fro;
};
struct KsvdOptions {
  bool evaluate_error = false;
};

inline KsvdResult prototype_ksvd(const DenseMatrix& a, Index k, Index s, std::uint64_t seed,
                                 const SketchSpec* spec = nullptr, const KsvdOptions& opts = {},
                                 int power_iters = 0) {
  DenseMatrix u(a.rows(), k), v(a.cols(), k);
  std::vector<double> sv(static_cast<size_t>(k));
  Index rank = 0;
  int32_t passes = 0;
  double err = 0.0;
  rnla_mat am = detail::view(a), um = detail::view(u), vm = detail::view(v);
  rnla_sketch_spec cs{};
  if (spec) cs = spec->to_c();
  detail::check(rnla_prototype_ksvd(detail::ctx(), &am, k, s, seed, spec ? &cs : nullptr, power_iters, &um, sv.data(),
                                    &vm, &rank, &passes, opts.evaluate_error ? &err : nullptr));
  KsvdResult r;
  r.factors.U = DenseMatrix(a.rows(), rank);
  r.factors.V = DenseMatrix(a.cols(), rank);
  r.factors.singular_values = Vector(rank);
  for (Index j = 0; j < rank; ++j) {
    r.factors.singular_values(j) = sv[static_cast<size_t>(j)];
    for (Index i = 0; i < a.rows(); ++i) r.factors.U(i, j) = u(i, j);
    for (Index i = 0; i < a.cols(); ++i) r.factors.V(i, j) = v(i, j);
  }
  r.passes_over_a = passes;
  if (opts.evaluate_error) r.error_fro = err;
  return r;
}

// randsvd.hpp:38-41: two passes, k < s < p < p_cs.
inline KsvdResult faster_ksvd(const DenseMatrix& a, Index k, Index s, Index p_cs, Index p, std::uint64_t seed,
                              const KsvdOptions& opts = {}) {
  DenseMatrix u(a.rows(), k), v(a.cols(), k);
  std::vector<double> sv(static_cast<size_t>(k));
  Index rank = 0;
  int32_t passes = 0;
  double err = 0.0;
  rnla_mat am = detail::view(a), um = detail::view(u), vm = detail::view(v);
  detail::check(rnla_faster_ksvd(detail::ctx(), &am, k, s, p_cs, p, seed, &um, sv.data(), &vm, &rank, &passes,
                                 opts.evaluate_error ? &err : nullptr));
  KsvdResult r;
  r.factors.U = DenseMatrix(a.rows(), rank);
  r.factors.V = DenseMatrix(a.cols(), rank);
  r.factors.singular_values = Vector(rank);
  for (Index j = 0; j < rank; ++j) {
    r.factors.singular_values(j) = sv[static_cast<size_t>(j)];
    for (Index i = 0; i < a.rows(); ++i) r.factors.U(i, j) = u(i, j);
    for (Index i = 0; i < a.cols(); ++i) r.factors.V(i, j) = v(i, j);
  }
  r.passes_over_a = passes;
  if (opts.evaluate_error) r.error_fro = err;
  return r;
}

// ---------------- regression.hpp ----------------
struct LsrSolution {
  Vector x;
  double objective = 0.0;
  int iterations = 0;
  std::optional<double> kappa_estimate;
  bool converged = true;
  bool flagged = false;
};

inline LsrSolution lsr_sketched(const DenseMatrix& a, const Vector& b, const SketchSpec& spec) {
  LsrSolution sol;
  sol.x = Vector(a.cols());
  int32_t flagged = 0;
  rnla_mat am = detail::view(a), bm = detail::view(b);
  rnla_sketch_spec cs = spec.to_c();
  detail::check(rnla_lsr_sketched(detail::ctx(), &am, &bm, &cs, sol.x.data(), &sol.objective, &flagged));
  sol.flagged = flagged != 0;
  return sol;
}

// regression.hpp:20-27: x = A^+ b (objective on the host).
inline LsrSolution lsr_exact(const DenseMatrix& a, const Vector& b) {
  if (a.rows() < a.cols()) throw std::invalid_argument("lsr_exact: n < d");
  if (a.rows() != b.size()) throw std::invalid_argument("lsr_exact: dimension mismatch");
  const DenseMatrix p = pseudo_inverse(a);
  LsrSolution sol;
  sol.x = Vector(a.cols());
  for (Index j = 0; j < a.cols(); ++j) {
    double s = 0.0;
    for (Index i = 0; i < a.rows(); ++i) s += p(j, i) * b(i);
    sol.x(j) = s;
  }
  for (Index i = 0; i < a.rows(); ++i) {
    double r = -b(i);
    for (Index j = 0; j < a.cols(); ++j) r += a(i, j) * sol.x(j);
    sol.objective += r * r;
  }
  return sol;
}

inline LsrSolution lsr_cg(const DenseMatrix& a, const Vector& b, double tol, int maxit) {
  if (a.rows() < a.cols()) throw std::invalid_argument("lsr_cg: n < d");
  LsrSolution sol;
  sol.x = Vector(a.cols());
  int32_t it = 0, conv = 0;
  rnla_mat am = detail::view(a), bm = detail::view(b);
  detail::check(rnla_lsr_cg(detail::ctx(), &am, &bm, tol, maxit, sol.x.data(), &sol.objective, &it, &conv));
  sol.iterations = it;
  sol.converged = conv != 0;
  return sol;
}

struct PreconditionedOptions {
  Index sketch_size = 0;  // 0: min(d^2, 20 d) capped at n
  bool use_cg = false;    // default: gradient descent with unit step
  SketchKind sketch_kind = SketchKind::kCountSketch;
};

// regression.hpp:44-56 (src/regression.cpp:94-198).
inline LsrSolution lsr_preconditioned(const DenseMatrix& a, const Vector& b, double eps, std::uint64_t seed,
                                      const PreconditionedOptions& opts = {}) {
  LsrSolution sol;
  sol.x = Vector(a.cols());
  int32_t it = 0;
  double kappa = 0.0;
  rnla_mat am = detail::view(a), bm = detail::view(b);
  detail::check(rnla_lsr_preconditioned(detail::ctx(), &am, &bm, eps, seed, opts.sketch_size, opts.use_cg ? 1 : 0,
                                        static_cast<int32_t>(opts.sketch_kind), sol.x.data(), &sol.objective, &it,
                                        &kappa));
  sol.iterations = it;
  sol.kappa_estimate = kappa;
  return sol;
}

// ---------------- spsd.hpp ----------------
struct KernelSpec {
  double sigma = 1.0;
};
struct NystromFactor {
  DenseMatrix L;
  std::vector<Index> selected;
};

inline DenseMatrix rbf_kernel(const DenseMatrix& x1, const DenseMatrix& x2, double sigma) {
  DenseMatrix k(x1.rows(), x2.rows());
  rnla_mat a = detail::view(x1), b = detail::view(x2), km = detail::view(k);
  detail::check(rnla_rbf_kernel(detail::ctx(), &a, &b, sigma, &km));
  return k;
}

// nystrom(KernelView(data, {sigma}), s, seed, target_k).
inline NystromFactor nystrom(const DenseMatrix& data, const KernelSpec& spec, Index s, std::uint64_t seed,
                             Index target_k = 0) {
  const Index kk = target_k > 0 ? target_k : static_cast<Index>(std::ceil(0.8 * static_cast<double>(s)));
  DenseMatrix l(data.rows(), kk);
  NystromFactor f;
  f.selected.resize(static_cast<size_t>(s));
  Index kept = 0, entries = 0;
  rnla_mat xm = detail::view(data), lm = detail::view(l);
  detail::check(rnla_nystrom(detail::ctx(), &xm, spec.sigma, s, seed, target_k, &lm, f.selected.data(), &kept, &entries));
  f.L = DenseMatrix(data.rows(), kept);
  for (Index j = 0; j < kept; ++j)
    for (Index i = 0; i < data.rows(); ++i) f.L(i, j) = l(i, j);
  return f;
}

// spsd.hpp:86-94, 109-115 (src/spsd.cpp:131-168).
struct SpsdSketch {
  DenseMatrix Q, Z;
  std::vector<Index> selected, secondary;
  bool flagged = false;
};

namespace detail {
inline SpsdSketch spsd_faster_call(const DenseMatrix& x, const KernelSpec* spec, Index s, Index p,
                                   std::uint64_t seed) {
  const Index n = x.rows();
  SpsdSketch out;
  out.Q = DenseMatrix(n, s);
  out.Z = DenseMatrix(s, s);
  out.selected.resize(static_cast<size_t>(s));
  std::vector<Index> sec(static_cast<size_t>(std::max<Index>(1, std::min(n, p + s))));
  Index nsec = 0;
  int32_t flagged = 0;
  rnla_mat xm = view(x), qm = view(out.Q), zm = view(out.Z);
  if (spec)
    check(rnla_spsd_faster(ctx(), &xm, spec->sigma, s, p, seed, &qm, &zm, out.selected.data(), sec.data(), &nsec,
                           &flagged));
  else
    check(rnla_spsd_faster_dense(ctx(), &xm, s, p, seed, &qm, &zm, out.selected.data(), sec.data(), &nsec,
                                 &flagged));
  sec.resize(static_cast<size_t>(nsec));
  out.secondary = sec;
  out.flagged = flagged != 0;
  return out;
}
}  // namespace detail

// ---------------- cur.hpp (kernel-lazy faster CUR) ----------------
struct CurFactors {
  DenseMatrix C, U, R;
  std::vector<Index> col_indices, row_indices, secondary_rows, secondary_cols;
  long entries_visited = 0;
  bool flagged = false;
};

// cur.hpp:44-52 (src/cur.cpp:188-212).
inline CurFactors cur_faster_kernel(const DenseMatrix& xtest, const DenseMatrix& xtrain, double sigma, Index c,
                                    Index r, std::uint64_t seed) {
  const Index m = xtest.rows(), n = xtrain.rows(), p = 2 * (c + r);
  CurFactors f;
  f.C = DenseMatrix(m, c);
  f.U = DenseMatrix(c, r);
  f.R = DenseMatrix(r, n);
  f.col_indices.resize(static_cast<size_t>(std::max<Index>(c, 0)));
  f.row_indices.resize(static_cast<size_t>(std::max<Index>(r, 0)));
  std::vector<Index> sr(static_cast<size_t>(std::max<Index>(1, std::min(m, p + r)))),
      sc(static_cast<size_t>(std::max<Index>(1, std::min(n, p + c))));
  Index nsr = 0, nsc = 0, ent = 0;
  int32_t flagged = 0;
  rnla_mat a = detail::view(xtest), b = detail::view(xtrain), cm = detail::view(f.C), um = detail::view(f.U),
           rm = detail::view(f.R);
  detail::check(rnla_cur_faster_kernel(detail::ctx(), &a, &b, sigma, c, r, seed, &cm, &um, &rm, f.col_indices.data(),
                                       f.row_indices.data(), sr.data(), &nsr, sc.data(), &nsc, &ent, &flagged));
  sr.resize(static_cast<size_t>(nsr));
  sc.resize(static_cast<size_t>(nsc));
  f.secondary_rows = sr;
  f.secondary_cols = sc;
  f.entries_visited = static_cast<long>(ent);
  f.flagged = flagged != 0;
  return f;
}

// KernelView over `data` with `spec` (the reference's spsd_faster(const KernelView&, ...)).
inline SpsdSketch spsd_faster(const DenseMatrix& data, const KernelSpec& spec, Index s, Index p, std::uint64_t seed) {
  return detail::spsd_faster_call(data, &spec, s, p, seed);
}
// Dense SPSD K (the reference's spsd_faster(const DenseMatrix&, ...)).
inline SpsdSketch spsd_faster(const DenseMatrix& k, Index s, Index p, std::uint64_t seed) {
  return detail::spsd_faster_call(k, nullptr, s, p, seed);
}

}  // namespace randnla_b200
