// test_acceptance.cpp -- the reference's hot-path acceptance criteria 3, 5,
// 6 and 10 (/root/reference/proj/src/acceptance.cpp:127-146, 185-248,
// 321-356; 50 seeds each, the same thresholds), plus the reference API
// surface that only the facade exposes (Rng& draws, KernelView with its
// entry counter, every nystrom overload, approx_eig, leverage / uniform
// column selection, count_sketch_stream, fwht_inplace), all written exactly
// as a reference caller would write them against include/randnla/*.hpp.
// Built and run by tests/test_cpp_facade.py.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "randnla_b200/randnla.hpp"

using namespace randnla_b200;

static int g_checks = 0;
#define CHECK(cond)                                                                \
  do {                                                                             \
    ++g_checks;                                                                    \
    if (!(cond)) {                                                                 \
      std::fprintf(stderr, "CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond); \
      std::exit(1);                                                                \
    }                                                                              \
  } while (0)

constexpr int kSeeds = 50;

// ---- small host helpers (Eigen expressions in the reference) ----
static DenseMatrix matmul(const DenseMatrix& a, const DenseMatrix& b) {
  DenseMatrix c = DenseMatrix::Zero(a.rows(), b.cols());
  for (Index j = 0; j < b.cols(); ++j)
    for (Index k = 0; k < a.cols(); ++k) {
      const double w = b(k, j);
      for (Index i = 0; i < a.rows(); ++i) c(i, j) += a(i, k) * w;
    }
  return c;
}
static DenseMatrix transpose(const DenseMatrix& a) {
  DenseMatrix t(a.cols(), a.rows());
  for (Index j = 0; j < a.cols(); ++j)
    for (Index i = 0; i < a.rows(); ++i) t(j, i) = a(i, j);
  return t;
}
static DenseMatrix sub(const DenseMatrix& a, const DenseMatrix& b) {
  DenseMatrix c(a.rows(), a.cols());
  for (Index j = 0; j < a.cols(); ++j)
    for (Index i = 0; i < a.rows(); ++i) c(i, j) = a(i, j) - b(i, j);
  return c;
}
static double sqnorm(const DenseMatrix& a) {
  double s = 0;
  for (Index j = 0; j < a.cols(); ++j)
    for (Index i = 0; i < a.rows(); ++i) s += a(i, j) * a(i, j);
  return s;
}
static double norm(const DenseMatrix& a) { return std::sqrt(sqnorm(a)); }
static Vector col0(const DenseMatrix& a) {
  Vector v(a.rows());
  for (Index i = 0; i < a.rows(); ++i) v(i) = a(i, 0);
  return v;
}

// acceptance.cpp:26-41
static DenseMatrix random_gaussian(Index rows, Index cols, std::uint64_t seed) {
  Rng rng = make_rng(seed);
  return gaussian_matrix(rows, cols, rng);
}
static DenseMatrix power_law_matrix(Index n, double exponent, std::uint64_t seed) {
  Rng rng = make_rng(seed);
  const DenseMatrix u = thin_qr(gaussian_matrix(n, n, rng)).Q;
  const DenseMatrix v = thin_qr(gaussian_matrix(n, n, rng)).Q;
  DenseMatrix us = u;
  for (Index j = 0; j < n; ++j) {
    const double sv = std::pow(static_cast<double>(j + 1), -exponent);
    for (Index i = 0; i < n; ++i) us(i, j) *= sv;
  }
  return matmul(us, transpose(v));
}
static DenseMatrix llt(const DenseMatrix& l) { return matmul(l, transpose(l)); }

static void criterion3(std::uint64_t seed) {  // sketched LSR (acceptance.cpp:127-146)
  const Index n = 2000, d = 10;
  const DenseMatrix a = random_gaussian(n, d, derive_seed(seed, 10));
  Rng rng = make_rng(derive_seed(seed, 11));
  const Vector x_star = col0(gaussian_matrix(d, 1, rng));
  const Vector noise = col0(gaussian_matrix(n, 1, rng));
  Vector b(n);
  for (Index i = 0; i < n; ++i) {
    double t = noise(i);
    double ax = 0.0;
    for (Index j = 0; j < d; ++j) ax += a(i, j) * x_star(j);
    b(i) = ax + t;
  }
  const double exact = lsr_exact(a, b).objective;
  int hits = 0;
  for (int t = 0; t < kSeeds; ++t) {
    const SketchSpec spec = SketchSpec::count_sketch(500, derive_seed(seed, 20 + t));
    if (lsr_sketched(a, b, spec).objective / exact <= 1.21) ++hits;
  }
  std::printf("criterion 3 (sketched-lsr): ratio<=1.21 in %d/50 (need >=45)\n", hits);
  CHECK(hits >= 45);
}

static void criterion5(std::uint64_t seed) {  // prototype k-SVD (acceptance.cpp:185-221)
  const Index n = 200, k = 10, s = 50;
  const DenseMatrix a = power_law_matrix(n, 2.0, derive_seed(seed, 10));
  const double opt2 = sqnorm(sub(a, truncated_svd(a, k).reconstruct()));
  Rng rng = make_rng(derive_seed(seed, 11));
  const DenseMatrix g1 = gaussian_matrix(n, k, rng);
  const DenseMatrix g2 = gaussian_matrix(k, n, rng);
  const DenseMatrix low = matmul(g1, g2);
  double ratio_sum = 0.0;
  int recovered = 0;
  bool passes_ok = true;
  KsvdOptions opts;
  opts.evaluate_error = true;
  for (int t = 0; t < kSeeds; ++t) {
    const std::uint64_t trial = derive_seed(seed, 20 + t);
    const KsvdResult r = prototype_ksvd(a, k, s, trial, nullptr, opts);
    ratio_sum += (*r.error_fro * *r.error_fro) / opt2;
    passes_ok = passes_ok && r.passes_over_a == 2;
    const KsvdResult rl = prototype_ksvd(low, k, s, trial, nullptr, opts);
    if (*rl.error_fro / norm(low) <= 1e-8) ++recovered;
    passes_ok = passes_ok && rl.passes_over_a == 2;
  }
  const double mean_ratio = ratio_sum / kSeeds;
  std::printf("criterion 5 (prototype-ksvd): mean ratio=%.4g, exact recovery %d/50, passes=2 %s\n", mean_ratio,
              recovered, passes_ok ? "yes" : "NO");
  CHECK(mean_ratio <= 1.2 && recovered >= 48 && passes_ok);
}

static void criterion6(std::uint64_t seed) {  // faster k-SVD (acceptance.cpp:223-248)
  const Index n = 500, k = 10, s = 4 * k, p = 4 * s, p_cs = 4 * p;
  const DenseMatrix a = power_law_matrix(n, 2.0, derive_seed(seed, 10));
  const double opt2 = sqnorm(sub(a, truncated_svd(a, k).reconstruct()));
  int hits = 0;
  bool passes_ok = true;
  KsvdOptions opts;
  opts.evaluate_error = true;
  for (int t = 0; t < kSeeds; ++t) {
    const KsvdResult r = faster_ksvd(a, k, s, p_cs, p, derive_seed(seed, 20 + t), opts);
    if ((*r.error_fro * *r.error_fro) / opt2 <= 1.95) ++hits;
    passes_ok = passes_ok && r.passes_over_a == 2;
  }
  std::printf("criterion 6 (faster-ksvd): ratio<=1.95 in %d/50, passes=2 %s\n", hits, passes_ok ? "yes" : "NO");
  CHECK(hits >= 40 && passes_ok);
}

static void criterion10(std::uint64_t seed) {  // Nystrom (acceptance.cpp:321-356)
  const DenseMatrix f = random_gaussian(200, 5, derive_seed(seed, 10));
  const DenseMatrix low = matmul(f, transpose(f));
  double worst = 0.0;
  for (int t = 0; t < kSeeds; ++t) {
    const NystromFactor nf = nystrom(low, 10, derive_seed(seed, 20 + t));
    worst = std::max(worst, norm(sub(low, llt(nf.L))) / norm(low));
  }
  const Index n = 400, s = 20;
  const DenseMatrix x = random_gaussian(n, 5, derive_seed(seed, 11));
  const double sigma = 2.0;
  const DenseMatrix kernel = rbf_kernel(x, x, sigma);
  double nys_sum = 0.0, fast_sum = 0.0;
  for (int t = 0; t < kSeeds; ++t) {
    const std::uint64_t trial = derive_seed(seed, 100 + t);
    const NystromFactor nf = nystrom(kernel, s, trial);
    nys_sum += norm(sub(kernel, llt(nf.L)));
    const SpsdSketch sk = spsd_faster(kernel, s, 4 * s, trial);
    fast_sum += norm(sub(kernel, sk.reconstruct()));
  }
  std::printf("criterion 10 (nystrom): rank-5 recovery worst=%.3g, mean err nystrom=%.4g vs faster=%.4g\n", worst,
              nys_sum / kSeeds, fast_sum / kSeeds);
  CHECK(worst <= 1e-6 && nys_sum >= fast_sum);
}

int main() {
  const std::uint64_t seed = 42;  // tests/acceptance_main.cpp: run_acceptance(seed = 42)
  {  // Rng& draws are the reference's libstdc++ streams (= the seed-taking C ABI)
    Rng rng = make_rng(7);
    const DenseMatrix g = gaussian_matrix(9, 5, rng);
    DenseMatrix h(9, 5);
    rnla_gaussian_matrix(7, 9, 5, h.data());
    for (Index j = 0; j < 5; ++j)
      for (Index i = 0; i < 9; ++i) CHECK(g(i, j) == h(i, j));
    Rng r2 = make_rng(11);
    CHECK(sample_without_replacement(1000, 37, r2) == sample_without_replacement(Index{1000}, Index{37},
                                                                                std::uint64_t{11}));
    Vector w(50);
    for (Index i = 0; i < 50; ++i) w(i) = 1.0 + (i % 7);
    Rng r3 = make_rng(13);
    const std::vector<Index> draws = sample_with_replacement(w, 64, r3);
    std::vector<Index> abi(64);
    rnla_sample_with_replacement(13, w.data(), 50, 64, abi.data());
    CHECK(draws == abi);
    Rng r4 = make_rng(3);
    const Vector u = gaussian_unit_vector(12, r4);
    double nn = 0;
    for (Index i = 0; i < 12; ++i) nn += u(i) * u(i);
    CHECK(std::abs(nn - 1.0) <= 1e-15);
  }
  {  // fwht_inplace known answers (test_sketch.cpp:19-35): H2 basis, H H = N I
    double e[8] = {1, 0, 0, 0, 0, 0, 0, 0};
    fwht_inplace(e, 8);
    for (double v : e) CHECK(v == 1.0);
    std::vector<double> x(1 << 14);
    for (size_t i = 0; i < x.size(); ++i) x[i] = std::sin(0.37 * static_cast<double>(i)) + 0.25;
    std::vector<double> y = x;
    fwht_inplace(y.data(), static_cast<Index>(y.size()));
    fwht_inplace(y.data(), static_cast<Index>(y.size()));
    for (size_t i = 0; i < x.size(); ++i) CHECK(std::abs(y[i] / static_cast<double>(x.size()) - x[i]) <= 1e-12);
    double h[4] = {1, 2, 3, 4};
    fwht_inplace(h, 4);
    CHECK(h[0] == 10 && h[1] == -2 && h[2] == -4 && h[3] == 0);
  }
  {  // count_sketch_stream == count_sketch, bitwise (sketch.hpp:73-78); the operator materializes it
    const DenseMatrix a = random_gaussian(13, 5000, 3);
    const DenseMatrix direct = count_sketch(a, 64, 99);
    const DenseMatrix streamed = count_sketch_stream(13, 5000, 64, 99, [&a](Index j) {
      Vector v(13);
      for (Index i = 0; i < 13; ++i) v(i) = a(i, j);
      return v;
    });
    for (Index j = 0; j < 64; ++j)
      for (Index i = 0; i < 13; ++i) CHECK(direct(i, j) == streamed(i, j));
    const DenseMatrix op = count_sketch_operator(5000, 64, 99);
    CHECK(norm(sub(matmul(a, op), direct)) <= 1e-13 * norm(a));
    for (Index j = 0; j < 5000; ++j) {
      int nz = 0;
      for (Index b = 0; b < 64; ++b) nz += op(j, b) != 0.0;
      CHECK(nz == 1);
    }
  }
  {  // uniform / leverage column selection (test_sketch.cpp:111-133)
    const DenseMatrix a = matmul(random_gaussian(30, 4, 1), random_gaussian(4, 200, 2));
    const auto [cu, su] = uniform_sample_columns(a, 20, 5);
    CHECK(cu.cols() == 20 && su.indices.size() == 20 && std::is_sorted(su.indices.begin(), su.indices.end()));
    for (Index t = 0; t < 20; ++t)
      for (Index i = 0; i < 30; ++i) CHECK(cu(i, t) == a(i, su.indices[static_cast<size_t>(t)]));
    const Vector lev = leverage_scores(a);
    double sum = 0;
    for (Index j = 0; j < 200; ++j) sum += lev(j);
    CHECK(std::abs(sum - 4.0) <= 1e-9);  // sums to rank(A)
    const Vector levk = leverage_scores(a, 2);
    sum = 0;
    for (Index j = 0; j < 200; ++j) sum += levk(j);
    CHECK(std::abs(sum - 2.0) <= 1e-9);
    const auto [cl, sl] = leverage_sample_columns(a, 40, 6, std::nullopt, true);
    CHECK(sl.weights.has_value() && static_cast<Index>(sl.indices.size()) == cl.cols());
    CHECK(std::adjacent_find(sl.indices.begin(), sl.indices.end()) == sl.indices.end());
    for (size_t t = 0; t < sl.indices.size(); ++t) {
      const double w = std::sqrt(4.0 / (40.0 * lev(sl.indices[t])));
      CHECK(std::abs((*sl.weights)(static_cast<Index>(t)) - w) <= 1e-9 * w);
    }
  }
  {  // KernelView: entries, counted evaluations, the three nystrom overloads agree
    const DenseMatrix x = random_gaussian(150, 4, 8);
    KernelView view(x, KernelSpec{1.7});
    CHECK(view.entries_evaluated() == 0);
    const double e01 = view.entry(0, 1);
    CHECK(view.entries_evaluated() == 1);
    const DenseMatrix k = rbf_kernel(x, x, 1.7);
    CHECK(std::abs(e01 - k(0, 1)) <= 1e-14);
    const DenseMatrix cols = view.columns({2, 5, 9});
    CHECK(view.entries_evaluated() == 1 + 150 * 3);
    CHECK(cols(2, 0) == 1.0 && cols(5, 1) == 1.0 && cols(9, 2) == 1.0);
    const NystromFactor nk = nystrom(view, 20, 31);
    CHECK(view.entries_evaluated() == 1 + 150 * 3 + 150 * 20);  // n s entries (the rows of C give W)
    const NystromFactor nd = nystrom(k, 20, 31);
    const NystromFactor ns = nystrom(KernelSpsdSource(view), 20, 31);
    const NystromFactor ng = nystrom(static_cast<const SpsdSource&>(DenseSpsdSource(k)), 20, 31);
    CHECK(nk.selected == nd.selected && nk.selected == ns.selected && nk.selected == ng.selected);
    CHECK(nk.L.cols() == 16 && nd.L.cols() == nk.L.cols());
    CHECK(norm(sub(llt(nk.L), llt(nd.L))) <= 1e-10 * norm(llt(nd.L)));
    // approx_eig: eigenpairs of L L' (test_spsd.cpp:133-142)
    const auto [u, lam] = approx_eig(nd.L, 5);
    const DenseMatrix lu = matmul(llt(nd.L), u);
    for (Index t = 0; t < 5; ++t) {
      double r = 0;
      for (Index i = 0; i < 150; ++i) r += std::pow(lu(i, t) - lam(t) * u(i, t), 2);
      CHECK(std::sqrt(r) <= 1e-8 * lam(0));
    }
    const SpsdSketch sk = spsd_faster(view, 10, 40, 6);
    CHECK(sk.Q.cols() == 10);
  }
  criterion3(seed);
  criterion5(seed);
  criterion6(seed);
  criterion10(seed);
  std::printf("acceptance ok: %d checks\n", g_checks);
  return 0;
}
