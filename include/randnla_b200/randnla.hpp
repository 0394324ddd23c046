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

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <functional>
#include <memory>
#include <numeric>
#include <optional>
#include <random>
#include <stdexcept>
#include <string>
#include <utility>
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
  // U diag(sigma) V' (types.hpp:18-27)
  DenseMatrix reconstruct() const {
    DenseMatrix out = DenseMatrix::Zero(U.rows(), V.rows());
    for (Index j = 0; j < V.rows(); ++j)
      for (Index t = 0; t < rank(); ++t) {
        const double w = singular_values(t) * V(j, t);
        for (Index i = 0; i < U.rows(); ++i) out(i, j) += U(i, t) * w;
      }
    return out;
  }
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
// The operator draws run on the host through libstdc++, exactly like the
// reference (include/randnla/rng.hpp:13-40, src/rng.cpp:8-65), so a caller's
// own Rng stream stays in step with the reference's.
inline std::uint64_t splitmix64(std::uint64_t& state) { return rnla_splitmix64(&state); }
inline std::uint64_t derive_seed(std::uint64_t seed, std::uint64_t stream) { return rnla_derive_seed(seed, stream); }

using Rng = std::mt19937_64;
inline Rng make_rng(std::uint64_t seed) { return Rng(seed); }

// Column-major fill with a fresh normal_distribution per call (the cached
// polar spare does not carry over between calls).
inline DenseMatrix gaussian_matrix(Index rows, Index cols, Rng& rng) {
  std::normal_distribution<double> nd(0.0, 1.0);
  DenseMatrix g(rows, cols);
  for (Index j = 0; j < cols; ++j)
    for (Index i = 0; i < rows; ++i) g(i, j) = nd(rng);
  return g;
}

inline Vector gaussian_unit_vector(Index dim, Rng& rng) {
  std::normal_distribution<double> nd(0.0, 1.0);
  Vector v(dim);
  double ss = 0.0;
  while (true) {
    ss = 0.0;
    for (Index i = 0; i < dim; ++i) {
      v(i) = nd(rng);
      ss += v(i) * v(i);
    }
    if (ss != 0.0) break;
  }
  const double r = std::sqrt(ss);
  for (Index i = 0; i < dim; ++i) v(i) /= r;
  return v;
}

// Partial Fisher-Yates over iota(n) with a fresh uniform_int_distribution
// per step, truncated to `count` and sorted.
inline std::vector<Index> sample_without_replacement(Index n, Index count, Rng& rng) {
  if (count < 0 || count > n) throw std::invalid_argument("sample_without_replacement: count > n");
  std::vector<Index> pool(static_cast<size_t>(n));
  std::iota(pool.begin(), pool.end(), Index{0});
  for (Index i = 0; i < count; ++i) {
    std::uniform_int_distribution<Index> pick(i, n - 1);
    const Index j = pick(rng);
    std::swap(pool[static_cast<size_t>(i)], pool[static_cast<size_t>(j)]);
  }
  pool.resize(static_cast<size_t>(count));
  std::sort(pool.begin(), pool.end());
  return pool;
}

// Sequential fp64 prefix sums, uniform_real(0, total), upper_bound, clamp.
inline std::vector<Index> sample_with_replacement(const Vector& weights, Index count, Rng& rng) {
  if (count < 1) throw std::invalid_argument("sample_with_replacement: count < 1");
  const Index n = weights.size();
  std::vector<double> prefix(static_cast<size_t>(n));
  double total = 0.0;
  for (Index i = 0; i < n; ++i) {
    if (!(weights(i) >= 0.0)) throw std::invalid_argument("sample_with_replacement: negative weight");
    total += weights(i);
    prefix[static_cast<size_t>(i)] = total;
  }
  if (!(total > 0.0)) throw std::invalid_argument("sample_with_replacement: all weights zero");
  std::uniform_real_distribution<double> u(0.0, total);
  std::vector<Index> out(static_cast<size_t>(count));
  for (auto& o : out) {
    const double x = u(rng);
    const Index j = static_cast<Index>(std::upper_bound(prefix.begin(), prefix.end(), x) - prefix.begin());
    o = std::min(j, n - 1);
  }
  return out;
}

// Seed-taking conveniences (make_rng(seed) then the draw), through the C ABI.
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

// sketch.hpp:55-59
struct ColumnSelection {
  std::vector<Index> indices;
  std::optional<Vector> weights;
};

// sketch.hpp:70 -- in-place unnormalized FWHT of a length-2^q buffer (on the device).
inline void fwht_inplace(double* data, Index n) {
  rnla_mat x{data, n, 1, 1, n > 0 ? n : 1, RNLA_F64, 0};
  detail::check(rnla_fwht(detail::ctx(), &x));
}

// sketch.hpp:75-76 -- one pass over the columns the callback delivers,
// called exactly once per j in order; chunks of columns are accumulated on
// the device (bit-identical to the reference's sequential loop).
inline DenseMatrix count_sketch_stream(Index m, Index n, Index s, std::uint64_t seed,
                                       const std::function<Vector(Index)>& column) {
  if (s < 1) throw std::invalid_argument("count_sketch: s < 1");
  rnla_count_stream* st = nullptr;
  detail::check(rnla_count_stream_begin(detail::ctx(), m, n, s, seed, RNLA_F64, &st));
  const Index chunk = std::max<Index>(1, std::min<Index>(n, std::max<Index>(1, (Index(1) << 24) / std::max<Index>(m, 1))));
  std::vector<double> buf(static_cast<size_t>(std::max<Index>(m, 1) * chunk));
  try {
    for (Index j0 = 0; j0 < n; j0 += chunk) {
      const Index k = std::min(chunk, n - j0);
      for (Index t = 0; t < k; ++t) {
        const Vector v = column(j0 + t);
        if (v.size() != m) throw std::invalid_argument("count_sketch_stream: column length differs from m");
        std::copy(v.data(), v.data() + m, buf.data() + static_cast<size_t>(t * m));
      }
      rnla_mat cm{buf.data(), m, k, 1, m > 0 ? m : 1, RNLA_F64, 0};
      detail::check(rnla_count_stream_push(st, &cm));
    }
  } catch (...) {
    rnla_count_stream_abort(st);
    throw;
  }
  DenseMatrix c(m, s);
  rnla_mat om = detail::view(c);
  detail::check(rnla_count_stream_end(st, &om));
  return c;
}

// sketch.hpp:81-82 -- the implied n x s operator (host, for tests at small n).
inline DenseMatrix count_sketch_operator(Index n, Index s, std::uint64_t seed) {
  std::vector<std::int64_t> b(static_cast<size_t>(n));
  std::vector<std::int8_t> g(static_cast<size_t>(n));
  detail::check(rnla_count_sketch_hashes(seed, 0, n, s, b.data(), g.data()));
  DenseMatrix op = DenseMatrix::Zero(n, s);
  for (Index j = 0; j < n; ++j) op(j, b[static_cast<size_t>(j)]) = g[static_cast<size_t>(j)];
  return op;
}

// sketch.hpp:89-90
inline std::pair<DenseMatrix, ColumnSelection> uniform_sample_columns(const DenseMatrix& a, Index s,
                                                                      std::uint64_t seed) {
  if (s < 1 || s > a.cols()) throw std::invalid_argument("uniform_sample_columns: s > n");
  DenseMatrix c(a.rows(), s);
  ColumnSelection sel;
  sel.indices.resize(static_cast<size_t>(s));
  rnla_mat am = detail::view(a), cm = detail::view(c);
  detail::check(rnla_uniform_sample_columns(detail::ctx(), &am, s, seed, &cm, sel.indices.data()));
  return {std::move(c), std::move(sel)};
}

// sketch.hpp:95
inline Vector leverage_scores(const DenseMatrix& a, std::optional<Index> k = {}) {
  Vector out(a.cols());
  rnla_mat am = detail::view(a);
  detail::check(rnla_leverage_scores(detail::ctx(), &am, k ? *k : 0, out.data()));
  return out;
}

// sketch.hpp:98-100
inline std::pair<DenseMatrix, ColumnSelection> leverage_sample_columns(const DenseMatrix& a, Index s,
                                                                       std::uint64_t seed,
                                                                       std::optional<Index> k = {},
                                                                       bool scale = false) {
  if (s < 1) throw std::invalid_argument("leverage_sample_columns: s < 1");
  DenseMatrix c(a.rows(), s);
  std::vector<Index> idx(static_cast<size_t>(s));
  std::vector<double> w(static_cast<size_t>(s));
  Index cnt = 0;
  rnla_mat am = detail::view(a), cm = detail::view(c);
  detail::check(rnla_leverage_sample_columns(detail::ctx(), &am, s, seed, k ? *k : 0, scale ? 1 : 0, &cm,
                                             idx.data(), w.data(), &cnt));
  ColumnSelection sel;
  sel.indices.assign(idx.begin(), idx.begin() + cnt);
  if (scale) {
    Vector wv(cnt);
    for (Index t = 0; t < cnt; ++t) wv(t) = w[static_cast<size_t>(t)];
    sel.weights = std::move(wv);
  }
  DenseMatrix out(a.rows(), cnt);
  for (Index j = 0; j < cnt; ++j)
    for (Index i = 0; i < a.rows(); ++i) out(i, j) = c(i, j);
  return {std::move(out), std::move(sel)};
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

// spsd.hpp:26-47 -- lazily evaluated RBF kernel over one dataset. Blocks
// are evaluated on the device (the same FMA chain for dots and squared
// norms, so K_ii = 1 and K = K' bitwise); every evaluated entry is counted.
class KernelView {
 public:
  KernelView(DenseMatrix data, KernelSpec spec) : data_(std::move(data)), spec_(spec) {
    if (!(spec_.sigma > 0.0)) throw std::invalid_argument("KernelView: sigma <= 0");
    for (Index j = 0; j < data_.cols(); ++j)
      for (Index i = 0; i < data_.rows(); ++i)
        if (!std::isfinite(data_(i, j))) throw std::invalid_argument("KernelView data: non-finite entries");
    sq_.resize(static_cast<size_t>(data_.rows()));
    for (Index i = 0; i < data_.rows(); ++i) {
      double t = 0.0;
      for (Index c = 0; c < data_.cols(); ++c) t += data_(i, c) * data_(i, c);
      sq_[static_cast<size_t>(i)] = t;
    }
  }
  KernelView(const KernelView& o) : data_(o.data_), spec_(o.spec_), sq_(o.sq_), counter_(o.counter_.load()) {}

  Index n() const { return data_.rows(); }
  // One entry on the host (src/spsd.cpp:58-64).
  double entry(Index i, Index j) const {
    counter_.fetch_add(1, std::memory_order_relaxed);
    double dot = 0.0;
    for (Index c = 0; c < data_.cols(); ++c) dot += data_(i, c) * data_(j, c);
    const double inv = 1.0 / (spec_.sigma * spec_.sigma);
    return std::exp((dot - 0.5 * (sq_[static_cast<size_t>(i)] + sq_[static_cast<size_t>(j)])) * inv);
  }
  DenseMatrix columns(const std::vector<Index>& cols) const {
    std::vector<Index> all(static_cast<size_t>(n()));
    std::iota(all.begin(), all.end(), Index{0});
    return block(all, cols);
  }
  DenseMatrix block(const std::vector<Index>& rows, const std::vector<Index>& cols) const {
    const DenseMatrix x1 = pick(rows), x2 = pick(cols);
    DenseMatrix out(static_cast<Index>(rows.size()), static_cast<Index>(cols.size()));
    if (!rows.empty() && !cols.empty()) {
      rnla_mat a = detail::view(x1), b = detail::view(x2), k = detail::view(out);
      detail::check(rnla_rbf_kernel(detail::ctx(), &a, &b, spec_.sigma, &k));
    }
    counter_.fetch_add(static_cast<long>(rows.size() * cols.size()), std::memory_order_relaxed);
    return out;
  }
  long entries_evaluated() const { return counter_.load(); }
  const DenseMatrix& data() const { return data_; }
  const KernelSpec& spec() const { return spec_; }
  void add_evaluated(long k) const { counter_.fetch_add(k, std::memory_order_relaxed); }

 private:
  DenseMatrix pick(const std::vector<Index>& idx) const {
    DenseMatrix out(static_cast<Index>(idx.size()), data_.cols());
    for (size_t t = 0; t < idx.size(); ++t) {
      if (idx[t] < 0 || idx[t] >= n()) throw std::invalid_argument("KernelView: index out of range");
      for (Index c = 0; c < data_.cols(); ++c) out(static_cast<Index>(t), c) = data_(idx[t], c);
    }
    return out;
  }
  DenseMatrix data_;
  KernelSpec spec_;
  std::vector<double> sq_;
  mutable std::atomic<long> counter_{0};
};

// spsd.hpp:51-84 -- column / block access to an SPSD matrix.
class SpsdSource {
 public:
  virtual ~SpsdSource() = default;
  virtual Index n() const = 0;
  virtual DenseMatrix columns(const std::vector<Index>& cols) const = 0;
  virtual DenseMatrix block(const std::vector<Index>& rows, const std::vector<Index>& cols) const = 0;
  virtual DenseMatrix full() const = 0;
};

class DenseSpsdSource final : public SpsdSource {
 public:
  explicit DenseSpsdSource(const DenseMatrix& k) : k_(k) {}
  Index n() const override { return k_.cols(); }
  DenseMatrix columns(const std::vector<Index>& cols) const override {
    DenseMatrix out(k_.rows(), static_cast<Index>(cols.size()));
    for (size_t t = 0; t < cols.size(); ++t)
      for (Index i = 0; i < k_.rows(); ++i) out(i, static_cast<Index>(t)) = k_(i, cols[t]);
    return out;
  }
  DenseMatrix block(const std::vector<Index>& rows, const std::vector<Index>& cols) const override {
    DenseMatrix out(static_cast<Index>(rows.size()), static_cast<Index>(cols.size()));
    for (size_t i = 0; i < rows.size(); ++i)
      for (size_t j = 0; j < cols.size(); ++j) out(static_cast<Index>(i), static_cast<Index>(j)) = k_(rows[i], cols[j]);
    return out;
  }
  DenseMatrix full() const override { return k_; }
  const DenseMatrix& matrix() const { return k_; }

 private:
  const DenseMatrix& k_;
};

class KernelSpsdSource final : public SpsdSource {
 public:
  explicit KernelSpsdSource(const KernelView& view) : view_(view) {}
  Index n() const override { return view_.n(); }
  DenseMatrix columns(const std::vector<Index>& cols) const override { return view_.columns(cols); }
  DenseMatrix block(const std::vector<Index>& rows, const std::vector<Index>& cols) const override {
    return view_.block(rows, cols);
  }
  DenseMatrix full() const override {
    std::vector<Index> all(static_cast<size_t>(view_.n()));
    std::iota(all.begin(), all.end(), Index{0});
    return view_.block(all, all);
  }
  const KernelView& view() const { return view_; }

 private:
  const KernelView& view_;
};

namespace detail {
inline Index nystrom_k(Index target_k, Index s) {
  return target_k > 0 ? target_k : static_cast<Index>(std::ceil(0.8 * static_cast<double>(s)));
}
inline NystromFactor nystrom_finish(const DenseMatrix& l, Index kept, std::vector<Index> selected) {
  NystromFactor f;
  f.L = DenseMatrix(l.rows(), kept);
  for (Index j = 0; j < kept; ++j)
    for (Index i = 0; i < l.rows(); ++i) f.L(i, j) = l(i, j);
  f.selected = std::move(selected);
  return f;
}
}  // namespace detail

// spsd.hpp:121-122 -- kernel columns evaluated on the device, counted.
inline NystromFactor nystrom(const KernelView& k, Index s, std::uint64_t seed, Index target_k = 0) {
  const Index n = k.n(), kk = detail::nystrom_k(target_k, s);
  if (!(kk >= 1 && kk <= s && s <= n)) throw std::invalid_argument("nystrom: need k <= s <= n");
  DenseMatrix l(n, kk);
  std::vector<Index> sel(static_cast<size_t>(s));
  Index kept = 0, entries = 0;
  rnla_mat xm = detail::view(k.data()), lm = detail::view(l);
  detail::check(rnla_nystrom(detail::ctx(), &xm, k.spec().sigma, s, seed, target_k, &lm, sel.data(), &kept, &entries));
  k.add_evaluated(static_cast<long>(entries));
  return detail::nystrom_finish(l, kept, std::move(sel));
}

// spsd.hpp:123-124 -- dense SPSD K.
inline NystromFactor nystrom(const DenseMatrix& k, Index s, std::uint64_t seed, Index target_k = 0) {
  if (k.rows() != k.cols()) throw std::invalid_argument("nystrom: K not square");
  const Index n = k.rows(), kk = detail::nystrom_k(target_k, s);
  if (!(kk >= 1 && kk <= s && s <= n)) throw std::invalid_argument("nystrom: need k <= s <= n");
  DenseMatrix l(n, kk);
  std::vector<Index> sel(static_cast<size_t>(s));
  Index kept = 0;
  rnla_mat km = detail::view(k), lm = detail::view(l);
  detail::check(rnla_nystrom_dense(detail::ctx(), &km, s, seed, target_k, &lm, sel.data(), &kept));
  return detail::nystrom_finish(l, kept, std::move(sel));
}

// spsd.hpp:119-120 -- any source: landmarks drawn as the reference does
// (src/spsd.cpp:189-191), columns from the source, the rest on the device.
inline NystromFactor nystrom(const SpsdSource& k, Index s, std::uint64_t seed, Index target_k = 0) {
  if (auto* kv = dynamic_cast<const KernelSpsdSource*>(&k)) return nystrom(kv->view(), s, seed, target_k);
  if (auto* ds = dynamic_cast<const DenseSpsdSource*>(&k)) return nystrom(ds->matrix(), s, seed, target_k);
  const Index n = k.n(), kk = detail::nystrom_k(target_k, s);
  if (!(kk >= 1 && kk <= s && s <= n)) throw std::invalid_argument("nystrom: need k <= s <= n");
  Rng rng = make_rng(derive_seed(seed, 1));
  std::vector<Index> sel = sample_without_replacement(n, s, rng);
  const DenseMatrix c = k.columns(sel);
  DenseMatrix l(n, kk);
  Index kept = 0;
  rnla_mat cm = detail::view(c), lm = detail::view(l);
  detail::check(rnla_nystrom_columns(detail::ctx(), &cm, sel.data(), target_k, &lm, &kept));
  return detail::nystrom_finish(l, kept, std::move(sel));
}

// Convenience: nystrom(KernelView(data, spec), s, seed, target_k).
inline NystromFactor nystrom(const DenseMatrix& data, const KernelSpec& spec, Index s, std::uint64_t seed,
                             Index target_k = 0) {
  return nystrom(KernelView(data, spec), s, seed, target_k);
}

// spsd.hpp:135 -- top-k eigenpairs of L L' from the SVD of L.
inline std::pair<DenseMatrix, Vector> approx_eig(const DenseMatrix& l, Index k) {
  if (k < 1 || k > l.cols()) throw std::invalid_argument("approx_eig: k > cols(L)");
  DenseMatrix u(l.rows(), k);
  Vector lam(k);
  rnla_mat lm = detail::view(l), um = detail::view(u);
  detail::check(rnla_approx_eig(detail::ctx(), &lm, k, &um, lam.data()));
  return {std::move(u), std::move(lam)};
}

// spsd.hpp:86-94, 109-115 (src/spsd.cpp:131-168).
struct SpsdSketch {
  DenseMatrix Q, Z;
  std::vector<Index> selected, secondary;
  bool flagged = false;
  // Q Z Q' (spsd.hpp:93)
  DenseMatrix reconstruct() const {
    const Index n = Q.rows(), s = Q.cols();
    DenseMatrix qz = DenseMatrix::Zero(n, s), out = DenseMatrix::Zero(n, n);
    for (Index j = 0; j < s; ++j)
      for (Index t = 0; t < s; ++t)
        for (Index i = 0; i < n; ++i) qz(i, j) += Q(i, t) * Z(t, j);
    for (Index j = 0; j < n; ++j)
      for (Index t = 0; t < s; ++t)
        for (Index i = 0; i < n; ++i) out(i, j) += qz(i, t) * Q(j, t);
    return out;
  }
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
// spsd.hpp:113-115 -- KernelView (entries counted: n s + |P|^2) and the two
// concrete sources; other SpsdSource implementations are not supported here.
inline SpsdSketch spsd_faster(const KernelView& k, Index s, Index p, std::uint64_t seed) {
  SpsdSketch out = detail::spsd_faster_call(k.data(), &k.spec(), s, p, seed);
  const long np = static_cast<long>(out.secondary.size());
  k.add_evaluated(static_cast<long>(k.n()) * static_cast<long>(s) + np * np);
  return out;
}
inline SpsdSketch spsd_faster(const SpsdSource& k, Index s, Index p, std::uint64_t seed) {
  if (auto* kv = dynamic_cast<const KernelSpsdSource*>(&k)) return spsd_faster(kv->view(), s, p, seed);
  if (auto* ds = dynamic_cast<const DenseSpsdSource*>(&k)) return spsd_faster(ds->matrix(), s, p, seed);
  throw std::invalid_argument("spsd_faster: only KernelView and dense sources are supported by the B200 core");
}

}  // namespace randnla_b200
