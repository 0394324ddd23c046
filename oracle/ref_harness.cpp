// TEST INFRASTRUCTURE ONLY -- runs the reference's OWN operator and sketch
// code (/root/reference/proj/src/rng.cpp and src/sketch.cpp, compiled
// unmodified against oracle/ref_shim/Eigen/Dense by `make -C oracle ref`) on
// small deterministic inputs and prints tests/golden/ref_fixtures.json. The
// fixtures pin the oracle (tests/test_oracle_golden.py) and the GPU path
// (tests/test_gpu_ref_fixtures.py) to reference-run outputs.
#include <cstdio>
#include <string>
#include <vector>

#include "randnla/rng.hpp"
#include "randnla/sketch.hpp"

using namespace randnla;

static void put(const char* key, const DenseMatrix& m, bool last = false) {
  std::printf("  \"%s\": {\"rows\": %ld, \"cols\": %ld, \"colmajor\": [", key, (long)m.rows(), (long)m.cols());
  for (Index j = 0; j < m.cols(); ++j)
    for (Index i = 0; i < m.rows(); ++i)
      std::printf("%s%.17g", (i == 0 && j == 0) ? "" : ", ", m(i, j));
  std::printf("]}%s\n", last ? "" : ",");
}
static void put_idx(const char* key, const std::vector<Index>& v, bool last = false) {
  std::printf("  \"%s\": [", key);
  for (size_t i = 0; i < v.size(); ++i) std::printf("%s%ld", i ? ", " : "", (long)v[i]);
  std::printf("]%s\n", last ? "" : ",");
}

int main() {
  std::printf("{\n  \"source\": \"/root/reference/proj/src/rng.cpp + src/sketch.cpp compiled unmodified "
              "(oracle/ref_shim Eigen stand-in, g++ -ffp-contract=off)\",\n");
  // ---- rng.cpp: draws on one engine, in the reference's call order
  {
    Rng rng = make_rng(42);
    put("gaussian_matrix_seed42_7x3", gaussian_matrix(7, 3, rng));
    put("gaussian_matrix_seed42_then_5x2", gaussian_matrix(5, 2, rng));  // fresh distribution: spare dropped
    put("gaussian_unit_vector_seed42_then_6", gaussian_unit_vector(6, rng));
    put_idx("sample_without_replacement_seed42_then_1000_17", sample_without_replacement(1000, 17, rng));
  }
  {
    Rng rng = make_rng(7);
    Vector w(40);
    for (Index i = 0; i < 40; ++i) w(i) = 0.5 + (double)((i * 37) % 11);
    put_idx("sample_with_replacement_seed7_w40_25", sample_with_replacement(w, 25, rng));
  }
  // ---- sketch.cpp on a deterministic input A (6 x 300) = gaussian_matrix(6, 300, make_rng(5))
  Rng in = make_rng(5);
  const DenseMatrix a = gaussian_matrix(6, 300, in);
  put("A_6x300", a);
  put("count_sketch_s32_seed11", count_sketch(a, 32, 11));
  put("count_sketch_s7_seed3", count_sketch(a, 7, 3));
  put("count_sketch_operator_n40_s9_seed77", count_sketch_operator(40, 9, 77));
  put("srht_sketch_s64_seed13", srht_sketch(a, 64, 13));
  put("srht_sketch_s512_seed2", srht_sketch(a, 512, 2));  // N = 512: every output
  put("gaussian_sketch_s20_seed17", gaussian_sketch(a, 20, 17));
  put("combined_count64_gauss16", combined_sketch(a, SketchSpec::combined(64, SketchSpec::gaussian(16, 21), 20)));
  put("combined_count64_srht16", combined_sketch(a, SketchSpec::combined(64, SketchSpec::srht(16, 23), 20)));
  {
    const auto [c, sel] = uniform_sample_columns(a, 25, 31);
    put_idx("uniform_sample_columns_s25_seed31_indices", sel.indices);
    put("uniform_sample_columns_s25_seed31", c);
  }
  {
    std::vector<double> x(64);
    for (int i = 0; i < 64; ++i) x[(size_t)i] = std::sin(0.1 * i) + 0.01 * i;
    fwht_inplace(x.data(), 64);
    DenseMatrix m(64, 1);
    for (int i = 0; i < 64; ++i) m(i, 0) = x[(size_t)i];
    put("fwht_sin64", m, true);
  }
  std::printf("}\n");
  return 0;
}
