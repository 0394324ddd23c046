// TEST INFRASTRUCTURE ONLY -- link stubs for the reference symbols that
// src/sketch.cpp references but the fixture harness never calls (the SVD and
// k-means back ends need the real Eigen). Calling one is a harness bug.
#include <stdexcept>

#include "randnla/core.hpp"
#include "randnla/kmeans.hpp"

namespace randnla {
SvdFactors condensed_svd(const DenseMatrix&) { throw std::logic_error("ref harness: condensed_svd not built"); }
SvdFactors truncated_svd(const DenseMatrix&, Index) { throw std::logic_error("ref harness: truncated_svd not built"); }
KmeansResult kmeans_once(const DenseMatrix&, Index, int, std::uint64_t) {
  throw std::logic_error("ref harness: kmeans_once not built");
}
}  // namespace randnla
