// host_rng.cpp -- operator generation on the host, through libstdc++ <random>
// exactly as the reference draws it (mt19937_64 + normal /
// uniform distributions are sequential and rejection-based, so Omega, SRHT
// signs/indices and sampled indices are drawn here and uploaded; only the
// counter-based CountSketch hash is evaluated on the device).
//
// Reference call sites (under /root/reference/proj):
//   include/randnla/rng.hpp:13-28, src/rng.cpp:8-65, src/sketch.cpp:57-65.
#include <algorithm>
#include <numeric>
#include <random>
#include <thread>

#include "rnla_internal.h"

namespace rnla {

uint64_t splitmix64(uint64_t& state) {
  uint64_t z = (state += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

uint64_t derive_seed(uint64_t seed, uint64_t stream) {
  uint64_t s = seed ^ (0x6a09e667f3bcc909ULL + stream * 0x9e3779b97f4a7c15ULL);
  return splitmix64(s);
}

int64_t next_pow2(int64_t n) {
  int64_t p = 1;
  while (p < n) p *= 2;
  return p;
}

// One fresh normal_distribution per call, column-major fill (src/rng.cpp:8-14).
void gaussian_matrix_host(uint64_t seed, int64_t rows, int64_t cols, double* out) {
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> normal(0.0, 1.0);
  for (int64_t j = 0; j < cols; ++j)
    for (int64_t i = 0; i < rows; ++i) out[j * rows + i] = normal(rng);
}

static std::vector<int64_t> swor(std::mt19937_64& rng, int64_t n, int64_t count) {
  require(count >= 0 && count <= n, "sample_without_replacement: count > n");
  std::vector<long> idx(static_cast<size_t>(n));
  std::iota(idx.begin(), idx.end(), 0L);
  for (int64_t i = 0; i < count; ++i) {
    std::uniform_int_distribution<long> pick(i, n - 1);  // fresh per step (src/rng.cpp:33-35)
    std::swap(idx[static_cast<size_t>(i)], idx[static_cast<size_t>(pick(rng))]);
  }
  idx.resize(static_cast<size_t>(count));
  std::sort(idx.begin(), idx.end());
  return std::vector<int64_t>(idx.begin(), idx.end());
}

std::vector<int64_t> sample_without_replacement_host(uint64_t seed, int64_t n, int64_t count) {
  std::mt19937_64 rng(seed);
  return swor(rng, n, count);
}

void WeightPrefix::extend(const double* w, int64_t m) {
  // one sequential fp64 add per weight (the reference's rounding order) into
  // pre-sized storage; the sign test is folded into one flag
  const size_t base = cum.size();
  cum.resize(base + static_cast<size_t>(m));
  double* c = cum.data() + base;
  double t = total;
  bool neg = false;
  for (int64_t i = 0; i < m; ++i) {
    neg |= !(w[i] >= 0.0);
    t += w[i];
    c[i] = t;
  }
  if (neg) {
    cum.resize(base);
    require(false, "sample_with_replacement: negative weight");
  }
  total = t;
}

WeightPrefix::Prepared WeightPrefix::prepare(uint64_t seed, int64_t count) {
  require(count >= 1, "sample_with_replacement: count < 1");
  Prepared pr;
  std::mt19937_64 rng(seed);
  pr.canon.resize(static_cast<size_t>(count));
  // libstdc++'s uniform_real_distribution(a, b)(g) is generate_canonical<double, 53>(g) * (b - a) + a
  // (bits/random.h), one engine word per draw; the scaling happens in draw()
  for (int64_t i = 0; i < count; ++i) pr.canon[static_cast<size_t>(i)] = std::generate_canonical<double, 53>(rng);
  pr.order.resize(static_cast<size_t>(count));
  for (int64_t i = 0; i < count; ++i) pr.order[static_cast<size_t>(i)] = i;
  // ascending canonical value = non-decreasing u (the scaling is monotone)
  std::stable_sort(pr.order.begin(), pr.order.end(), [&](int64_t a, int64_t b) {
    return pr.canon[static_cast<size_t>(a)] < pr.canon[static_cast<size_t>(b)];
  });
  return pr;
}

std::vector<int64_t> WeightPrefix::draw(uint64_t seed, int64_t count) const { return draw(prepare(seed, count)); }

std::vector<int64_t> WeightPrefix::draw(const Prepared& pr) const {
  const int64_t count = (int64_t)pr.canon.size();
  require(count >= 1, "sample_with_replacement: count < 1");
  require(total > 0.0, "sample_with_replacement: all weights zero");
  const int64_t n = (int64_t)cum.size();
  std::vector<double> u(static_cast<size_t>(count));
  for (int64_t i = 0; i < count; ++i) u[static_cast<size_t>(i)] = pr.canon[static_cast<size_t>(i)] * (total - 0.0) + 0.0;
  // upper_bound(cum, u_i) for every draw, visiting the draws in ascending u
  // order: from the previous position a galloping search brackets the next
  // one and a binary search inside the bracket finishes (about log2(n / count)
  // probes near the last hit per draw, instead of count cold binary searches
  // over an n-element array or one linear sweep over all of it). cum is
  // non-decreasing, so these are exactly the upper_bound positions.
  const std::vector<int64_t>& order = pr.order;
  std::vector<int64_t> out(static_cast<size_t>(count));
  const double* c = cum.data();
  // The sorted draws are cut into contiguous ranges searched by separate host
  // threads (each range starts from its own binary search): at n = 2^20 the
  // probes into the 8 MB prefix array are cache misses, ~1 ms on one thread.
  auto search = [&](int64_t r0, int64_t r1) {
    if (r0 >= r1) return;
    const double u0 = u[static_cast<size_t>(order[static_cast<size_t>(r0)])];
    int64_t j = std::upper_bound(c, c + n, u0) - c;
    for (int64_t r = r0; r < r1; ++r) {
      const int64_t i = order[static_cast<size_t>(r)];
      const double ui = u[static_cast<size_t>(i)];
      if (j < n && c[j] <= ui) {
        int64_t lo = j, step = 1;  // invariant: c[lo] <= ui
        while (lo + step < n && c[lo + step] <= ui) {
          lo += step;
          step *= 2;
        }
        int64_t hi = std::min(n, lo + step);  // c[hi] > ui or hi == n
        while (hi - lo > 1) {
          const int64_t mid = lo + (hi - lo) / 2;
          if (c[mid] <= ui) lo = mid;
          else hi = mid;
        }
        j = hi;
      }
      out[static_cast<size_t>(i)] = j >= n ? n - 1 : j;
    }
  };
  const int nth = (count >= 1024 && n >= (int64_t)1 << 16)
                      ? (int)std::max<unsigned>(1u, std::min<unsigned>(8u, std::thread::hardware_concurrency()))
                      : 1;
  std::vector<std::thread> th;
  for (int t = 1; t < nth; ++t) th.emplace_back(search, count * t / nth, count * (t + 1) / nth);
  search(0, count / nth);
  for (auto& x : th) x.join();
  return out;
}

// Sequential fp64 prefix sums (the reference's std::partial_sum order), one
// engine, uniform_real_distribution(0, total), upper_bound, clamp
// (src/rng.cpp:42-65).
std::vector<int64_t> sample_with_replacement_host(uint64_t seed, const double* w, int64_t n, int64_t count) {
  require(count >= 1, "sample_with_replacement: count < 1");
  WeightPrefix p;
  p.cum.reserve(static_cast<size_t>(n));
  p.extend(w, n);
  return p.draw(seed, count);
}

// Signs first, then the index sample, from one engine (src/sketch.cpp:61-65).
void srht_operator_host(uint64_t seed, int64_t n, int64_t s, int8_t* signs, int64_t* idx) {
  const int64_t big_n = next_pow2(n);
  require(s >= 1 && s <= big_n, "srht_sketch: s > padded dimension");
  std::mt19937_64 rng(seed);
  std::uniform_int_distribution<int> coin(0, 1);
  for (int64_t j = 0; j < n; ++j) signs[j] = coin(rng) ? 1 : -1;
  std::vector<int64_t> v = swor(rng, big_n, s);
  std::copy(v.begin(), v.end(), idx);
}

}  // namespace rnla
