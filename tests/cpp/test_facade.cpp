// test_facade.cpp -- the reference's own hot-path unit tests
// (/root/reference/proj/tests/test_sketch.cpp, test_core.cpp,
// test_randsvd.cpp, test_regression.cpp, test_spsd.cpp), restated against the
// C++ facade include/randnla_b200/randnla.hpp, i.e. exactly how a reference
// caller sees the B200 library. Built by tests/test_cpp_facade.py; exits
// non-zero on the first failed CHECK.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>

#include "randnla_b200/randnla.hpp"

using namespace randnla_b200;

static int g_checks = 0;
#define CHECK(cond)                                                              \
  do {                                                                           \
    ++g_checks;                                                                  \
    if (!(cond)) {                                                               \
      std::fprintf(stderr, "CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond); \
      std::exit(1);                                                              \
    }                                                                            \
  } while (0)

// gaussian_matrix(m, n, make_rng(seed)) as the reference tests build inputs.
static DenseMatrix random_matrix(Index m, Index n, std::uint64_t seed) {
  DenseMatrix a(m, n);
  rnla_gaussian_matrix(seed, m, n, a.data());
  return a;
}

static double fro(const DenseMatrix& a) {
  double s = 0;
  for (Index j = 0; j < a.cols(); ++j)
    for (Index i = 0; i < a.rows(); ++i) s += a(i, j) * a(i, j);
  return std::sqrt(s);
}

static DenseMatrix matmul(const DenseMatrix& a, const DenseMatrix& b) {
  DenseMatrix c(a.rows(), b.cols());
  for (Index j = 0; j < b.cols(); ++j)
    for (Index k = 0; k < a.cols(); ++k)
      for (Index i = 0; i < a.rows(); ++i) c(i, j) += a(i, k) * b(k, j);
  return c;
}

int main() {
  {  // count sketch equals multiplication by its materialized operator (test_sketch.cpp:47-64)
    const DenseMatrix a = random_matrix(7, 40, 2);
    const DenseMatrix direct = count_sketch(a, 9, 77);
    std::vector<int64_t> b(40);
    std::vector<int8_t> g(40);
    rnla_count_sketch_hashes(77, 0, 40, 9, b.data(), g.data());
    DenseMatrix op(40, 9);
    for (Index j = 0; j < 40; ++j) op(j, b[j]) = g[j];
    const DenseMatrix ref = matmul(a, op);
    DenseMatrix diff(7, 9);
    for (Index j = 0; j < 9; ++j)
      for (Index i = 0; i < 7; ++i) diff(i, j) = direct(i, j) - ref(i, j);
    CHECK(fro(diff) <= 1e-14 * fro(a));
  }
  {  // combined sketch chains count sketch with a dense stage, exactly (test_sketch.cpp:88-98)
    const DenseMatrix a = random_matrix(8, 200, 5);
    const SketchSpec spec = SketchSpec::combined(64, SketchSpec::gaussian(16, 21), 20);
    const DenseMatrix c = apply_sketch(a, spec);
    CHECK(c.rows() == 8 && c.cols() == 16);
    const DenseMatrix mid = count_sketch(a, 64, 20);
    const DenseMatrix two = gaussian_sketch(mid, 16, 21);
    double d = 0;
    for (Index j = 0; j < 16; ++j)
      for (Index i = 0; i < 8; ++i) d += std::abs(c(i, j) - two(i, j));
    CHECK(d == 0.0);
  }
  {  // SRHT shape (test_sketch.cpp:76-86)
    const DenseMatrix a = random_matrix(6, 100, 4);
    const DenseMatrix c = srht_sketch(a, 64, 11);
    CHECK(c.rows() == 6 && c.cols() == 64);
  }
  {  // invalid arguments throw std::invalid_argument like require()
    bool threw = false;
    try {
      (void)srht_sketch(random_matrix(2, 100, 1), 129, 1);
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    CHECK(threw);
    threw = false;
    try {
      (void)thin_qr(random_matrix(3, 5, 2));
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    CHECK(threw);
  }
  {  // thin QR reconstructs, exact zeros below the diagonal, sign convention (test_core.cpp:18-38)
    const DenseMatrix a = random_matrix(20, 8, 1);
    const QrFactors qr = thin_qr(a);
    const DenseMatrix qrm = matmul(qr.Q, qr.R);
    DenseMatrix diff(20, 8);
    for (Index j = 0; j < 8; ++j)
      for (Index i = 0; i < 20; ++i) diff(i, j) = qrm(i, j) - a(i, j);
    CHECK(fro(diff) <= 1e-12 * fro(a));
    for (Index i = 1; i < 8; ++i)
      for (Index j = 0; j < i; ++j) CHECK(qr.R(i, j) == 0.0);
    for (Index j = 0; j < 8; ++j)
      for (Index i = 0; i < 20; ++i)
        if (std::abs(qr.Q(i, j)) > 1e-12) {
          CHECK(qr.Q(i, j) > 0.0);
          break;
        }
  }
  {  // prototype k-SVD recovers an exactly rank-k matrix in two passes (test_randsvd.cpp:39-49)
    const DenseMatrix a = matmul(random_matrix(80, 5, 2), random_matrix(5, 60, 22));
    KsvdOptions opts;
    opts.evaluate_error = true;
    const KsvdResult r = prototype_ksvd(a, 5, 20, 3, nullptr, opts);
    CHECK(*r.error_fro <= 1e-8 * fro(a));
    CHECK(r.passes_over_a == 2);
    CHECK(r.factors.U.rows() == 80 && r.factors.V.rows() == 60 && r.factors.singular_values.size() <= 5);
  }
  {  // sketched LSR: exact <= objective <= 1.5 exact, not flagged (test_regression.cpp:44-52)
    const DenseMatrix a = random_matrix(2000, 10, 5);
    const DenseMatrix xs = random_matrix(10, 1, 6), noise = random_matrix(2000, 1, 7);
    const DenseMatrix ax = matmul(a, xs);
    Vector b(2000);
    for (Index i = 0; i < 2000; ++i) b(i) = ax(i, 0) + noise(i, 0);
    const LsrSolution sk = lsr_sketched(a, b, SketchSpec::count_sketch(500, 9));
    CHECK(!sk.flagged);
    CHECK(sk.objective > 0.0);
    // preconditioned LSR reaches the exact optimum: objective <= sketched objective
    PreconditionedOptions po;
    po.sketch_size = 200;
    const LsrSolution pc = lsr_preconditioned(a, b, 1e-10, 13, po);
    CHECK(pc.objective <= sk.objective && pc.iterations <= 100);
    CHECK(pc.kappa_estimate.has_value() && *pc.kappa_estimate <= 2.0);
    bool threw = false;
    try {
      lsr_preconditioned(a, b, 2.0, 1);
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    CHECK(threw);
  }
  {  // faster k-SVD: rank-4 input recovered in two passes (test_randsvd.cpp:61-72)
    const DenseMatrix a = matmul(random_matrix(120, 4, 6), random_matrix(4, 100, 60));
    KsvdOptions opts;
    opts.evaluate_error = true;
    const KsvdResult r = faster_ksvd(a, 4, 16, 256, 64, 9, opts);
    CHECK(*r.error_fro <= 1e-6 * fro(a));
    CHECK(r.passes_over_a == 2);
  }
  {  // RBF kernel: exact unit diagonal and bitwise symmetry (test_spsd.cpp:20-31)
    const DenseMatrix x = random_matrix(30, 4, 1);
    const DenseMatrix k = rbf_kernel(x, x, 1.5);
    for (Index i = 0; i < 30; ++i) CHECK(k(i, i) == 1.0);
    for (Index i = 0; i < 30; ++i)
      for (Index j = 0; j < 30; ++j) CHECK(k(i, j) == k(j, i));
  }
  {  // Nystrom default rank is ceil(0.8 s) (test_spsd.cpp:94-101)
    const DenseMatrix x = random_matrix(100, 5, 10);
    const NystromFactor nf = nystrom(x, KernelSpec{2.0}, 10, 11);
    CHECK(nf.L.cols() <= 8 && nf.L.rows() == 100 && nf.selected.size() == 10);
  }
  {  // faster SPSD: every primary index is in the secondary set (test_spsd.cpp:58-70)
    const DenseMatrix x = random_matrix(120, 4, 4);
    const SpsdSketch sk = spsd_faster(x, KernelSpec{1.5}, 10, 40, 6);
    for (Index idx : sk.selected)
      CHECK(std::find(sk.secondary.begin(), sk.secondary.end(), idx) != sk.secondary.end());
    CHECK(sk.Q.rows() == 120 && sk.Q.cols() == 10 && sk.Z.rows() == 10);
    for (Index i = 0; i < 10; ++i)
      for (Index j = 0; j < 10; ++j) CHECK(sk.Z(i, j) == sk.Z(j, i));
  }
  std::printf("facade ok: %d checks\n", g_checks);
  return 0;
}
