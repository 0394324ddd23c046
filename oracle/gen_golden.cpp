// gen_golden.cpp -- TEST INFRASTRUCTURE ONLY (fixture generator).
//
// Produces tests/golden/libstdcxx_streams.json from the REAL GCC libstdc++
// <random> (the third-party library that defines every random operator of
// the reference; see include/randnla/rng.hpp:26-28 and src/rng.cpp:8-65).
// The reference itself cannot be compiled here (Eigen3 is absent),
// so these vectors are drawn by calling libstdc++ exactly the way the
// reference's call sites do (fresh distribution objects where the reference
// builds them, same draw order). They pin the plain-C restatement in
// oracle/rnla_oracle.c and the product's host operator generation.
//
// Build + run: make -C oracle golden   (writes ../tests/golden/libstdcxx_streams.json)
#include <algorithm>
#include <cinttypes>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <numeric>
#include <random>
#include <string>
#include <vector>

using u64 = std::uint64_t;
using i64 = long;  // Eigen::Index == std::ptrdiff_t == long on LP64

static std::string arr_u64(const std::vector<u64>& v) {
  std::string s = "[";
  for (size_t i = 0; i < v.size(); ++i) {
    char b[32];
    std::snprintf(b, sizeof b, "%s\"%" PRIu64 "\"", i ? "," : "", v[i]);
    s += b;
  }
  return s + "]";
}
static std::string arr_i64(const std::vector<i64>& v) {
  std::string s = "[";
  for (size_t i = 0; i < v.size(); ++i) {
    char b[32];
    std::snprintf(b, sizeof b, "%s%ld", i ? "," : "", v[i]);
    s += b;
  }
  return s + "]";
}
static std::string arr_f64(const std::vector<double>& v) {  // exact: hex floats
  std::string s = "[";
  for (size_t i = 0; i < v.size(); ++i) {
    char b[48];
    std::snprintf(b, sizeof b, "%s\"%a\"", i ? "," : "", v[i]);
    s += b;
  }
  return s + "]";
}

static u64 splitmix64(u64& state) {
  u64 z = (state += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
static u64 derive_seed(u64 seed, u64 stream) {
  u64 s = seed ^ (0x6a09e667f3bcc909ULL + stream * 0x9e3779b97f4a7c15ULL);
  return splitmix64(s);
}

// Column-major gaussian fill with a fresh normal_distribution (src/rng.cpp:8-14).
static std::vector<double> gaussian(i64 rows, i64 cols, std::mt19937_64& rng) {
  std::normal_distribution<double> normal(0.0, 1.0);
  std::vector<double> g(static_cast<size_t>(rows * cols));
  for (i64 j = 0; j < cols; ++j)
    for (i64 i = 0; i < rows; ++i) g[static_cast<size_t>(j * rows + i)] = normal(rng);
  return g;
}

// Partial Fisher-Yates + sort (src/rng.cpp:27-40).
static std::vector<i64> swor(i64 n, i64 count, std::mt19937_64& rng) {
  std::vector<i64> idx(static_cast<size_t>(n));
  std::iota(idx.begin(), idx.end(), i64{0});
  for (i64 i = 0; i < count; ++i) {
    std::uniform_int_distribution<i64> pick(i, n - 1);
    std::swap(idx[static_cast<size_t>(i)], idx[static_cast<size_t>(pick(rng))]);
  }
  idx.resize(static_cast<size_t>(count));
  std::sort(idx.begin(), idx.end());
  return idx;
}

// Weighted draws (src/rng.cpp:42-65), in draw order.
static std::vector<i64> swr(const std::vector<double>& w, i64 count, std::mt19937_64& rng) {
  const i64 n = static_cast<i64>(w.size());
  std::vector<double> cum(w.size());
  double total = 0.0;
  for (i64 i = 0; i < n; ++i) {
    total += w[static_cast<size_t>(i)];
    cum[static_cast<size_t>(i)] = total;
  }
  std::uniform_real_distribution<double> unif(0.0, total);
  std::vector<i64> out(static_cast<size_t>(count));
  for (i64 i = 0; i < count; ++i) {
    const double u = unif(rng);
    i64 j = static_cast<i64>(std::upper_bound(cum.begin(), cum.end(), u) - cum.begin());
    if (j >= n) j = n - 1;
    out[static_cast<size_t>(i)] = j;
  }
  return out;
}

int main() {
  std::printf("{\n");
  std::printf("  \"generator\": \"oracle/gen_golden.cpp against GCC %d.%d libstdc++ <random>\",\n", __GNUC__,
              __GNUC_MINOR__);
  // Standard known answer ([rand.predef]).
  {
    std::mt19937_64 g;
    g.discard(9999);
    std::printf("  \"mt64_default_10000th\": \"%" PRIu64 "\",\n", g());
  }
  // Raw engine streams.
  std::printf("  \"mt64\": [\n");
  const u64 seeds[] = {0ULL, 1ULL, 42ULL, 5489ULL, 0xdeadbeefcafef00dULL};
  for (size_t k = 0; k < 5; ++k) {
    std::mt19937_64 g(seeds[k]);
    std::vector<u64> v;
    for (int i = 0; i < 700; ++i) v.push_back(g());  // crosses two twists
    std::vector<u64> head(v.begin(), v.begin() + 8), tail(v.end() - 4, v.end());
    std::printf("    {\"seed\": \"%" PRIu64 "\", \"head\": %s, \"tail700\": %s}%s\n", seeds[k], arr_u64(head).c_str(),
                arr_u64(tail).c_str(), k + 1 < 5 ? "," : "");
  }
  std::printf("  ],\n");
  // generate_canonical.
  {
    std::mt19937_64 g(7);
    std::vector<double> v;
    for (int i = 0; i < 16; ++i) v.push_back(std::generate_canonical<double, 53>(g));
    std::printf("  \"canonical_seed7\": %s,\n", arr_f64(v).c_str());
  }
  // uniform_int_distribution<long>(a, b), one fresh object per draw like src/rng.cpp:33.
  {
    std::mt19937_64 g(3);
    std::vector<i64> v;
    const i64 ranges[][2] = {{0, 1}, {0, 2}, {5, 9}, {0, 1048575}, {17, 131071}, {0, 6}, {0, 0},
                             {0, 4611686018427387903L}, {0, 3000000000L}, {-5, 5}};
    for (int rep = 0; rep < 4; ++rep)
      for (auto& r : ranges) {
        std::uniform_int_distribution<i64> d(r[0], r[1]);
        v.push_back(d(g));
      }
    std::printf("  \"uniform_int_seed3\": %s,\n", arr_i64(v).c_str());
  }
  // uniform_int_distribution<int>(0,1) coins (src/sketch.cpp:62-64).
  {
    std::mt19937_64 g(11);
    std::uniform_int_distribution<int> coin(0, 1);
    std::vector<i64> v;
    for (int i = 0; i < 64; ++i) v.push_back(coin(g));
    std::printf("  \"coin_seed11\": %s,\n", arr_i64(v).c_str());
  }
  // gaussian_matrix: two consecutive calls on one engine (odd count loses the spare).
  {
    std::mt19937_64 g(1);
    auto a = gaussian(5, 7, g);  // 35 draws: odd
    auto b = gaussian(3, 2, g);
    std::printf("  \"gaussian_seed1_5x7\": %s,\n", arr_f64(a).c_str());
    std::printf("  \"gaussian_seed1_then_3x2\": %s,\n", arr_f64(b).c_str());
    std::mt19937_64 g2(derive_seed(42, 200));
    auto c = gaussian(2048, 30, g2);
    std::vector<double> c_head(c.begin(), c.begin() + 8), c_tail(c.end() - 8, c.end());
    double sum = 0.0;
    for (double x : c) sum += x;
    std::printf("  \"gaussian_cfg0_2048x30\": {\"seed\": \"%" PRIu64 "\", \"head\": %s, \"tail\": %s, \"sum\": \"%a\"},\n",
                derive_seed(42, 200), arr_f64(c_head).c_str(), arr_f64(c_tail).c_str(), sum);
  }
  // sample_without_replacement.
  {
    std::printf("  \"swor\": [\n");
    const i64 cases[][3] = {{30, 10, 99}, {128, 64, 11}, {1000, 1000, 5}, {131072, 2048, 0}, {50, 0, 1}};
    for (int k = 0; k < 5; ++k) {
      u64 seed = static_cast<u64>(cases[k][2]);
      if (k == 3) seed = derive_seed(derive_seed(42, 204), 1);
      std::mt19937_64 g(seed);
      auto v = swor(cases[k][0], cases[k][1], g);
      if (v.size() > 64) {
        std::vector<i64> h(v.begin(), v.begin() + 32), t(v.end() - 32, v.end());
        long long s = 0;
        for (auto x : v) s += x;
        std::printf("    {\"n\": %ld, \"count\": %ld, \"seed\": \"%" PRIu64 "\", \"head\": %s, \"tail\": %s, \"sum\": %lld}%s\n",
                    cases[k][0], cases[k][1], seed, arr_i64(h).c_str(), arr_i64(t).c_str(), s, k + 1 < 5 ? "," : "");
      } else {
        std::printf("    {\"n\": %ld, \"count\": %ld, \"seed\": \"%" PRIu64 "\", \"idx\": %s}%s\n", cases[k][0],
                    cases[k][1], seed, arr_i64(v).c_str(), k + 1 < 5 ? "," : "");
      }
    }
    std::printf("  ],\n");
  }
  // SRHT operator: n coins then swor(N, s) on the same engine (src/sketch.cpp:61-65).
  {
    std::printf("  \"srht\": [\n");
    const i64 cases[][3] = {{100, 64, 11}, {80, 32, 55}, {1024, 16, 9000}};
    for (int k = 0; k < 3; ++k) {
      const i64 n = cases[k][0], s = cases[k][1];
      std::mt19937_64 g(static_cast<u64>(cases[k][2]));
      std::uniform_int_distribution<int> coin(0, 1);
      std::vector<i64> signs;
      for (i64 j = 0; j < n; ++j) signs.push_back(coin(g) ? 1 : -1);
      i64 big = 1;
      while (big < n) big *= 2;
      auto idx = swor(big, s, g);
      std::printf("    {\"n\": %ld, \"s\": %ld, \"seed\": \"%ld\", \"signs\": %s, \"idx\": %s}%s\n", n, s, cases[k][2],
                  arr_i64(signs).c_str(), arr_i64(idx).c_str(), k + 1 < 3 ? "," : "");
    }
    std::printf("  ],\n");
  }
  // sample_with_replacement.
  {
    std::vector<double> w = {0.2, 0.8, 0.0, 1.5, 0.25, 3.0, 1e-9, 0.7};
    std::mt19937_64 g(derive_seed(9, 2));
    auto v = swr(w, 40, g);
    std::printf("  \"swr\": {\"weights\": %s, \"seed\": \"%" PRIu64 "\", \"draws\": %s},\n", arr_f64(w).c_str(),
                derive_seed(9, 2), arr_i64(v).c_str());
  }
  // splitmix64 / derive_seed / count_sketch_hash (integer formulas of rng.hpp:13-24, sketch.cpp:16-26).
  {
    std::vector<u64> ds;
    for (u64 st : {0ULL, 1ULL, 2ULL, 3ULL, 100ULL, 101ULL, 200ULL, 201ULL, 202ULL, 203ULL, 204ULL})
      ds.push_back(derive_seed(42, st));
    std::printf("  \"derive_seed_42\": %s,\n", arr_u64(ds).c_str());
    std::vector<i64> buckets, signs;
    const u64 seed = derive_seed(42, 201);
    for (i64 j : {0L, 1L, 2L, 3L, 1000L, 4194303L, 4194304L - 2}) {
      u64 state = seed ^ (0xa0761d6478bd642fULL + static_cast<u64>(j) * 0xe7037ed1a0b428dbULL);
      const u64 h1 = splitmix64(state), h2 = splitmix64(state);
      buckets.push_back(static_cast<i64>(h1 % 8192ULL));
      signs.push_back((h2 & 1ULL) ? 1 : -1);
    }
    std::printf("  \"count_hash_cfg1\": {\"seed\": \"%" PRIu64 "\", \"s\": 8192, \"j\": [0,1,2,3,1000,4194303,4194302], "
                "\"bucket\": %s, \"sign\": %s}\n", seed, arr_i64(buckets).c_str(), arr_i64(signs).c_str());
  }
  std::printf("}\n");
  return 0;
}
