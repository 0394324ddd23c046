// util.cuh -- declarations of the helper launchers in util.cu / linalg.cu.
#pragma once
#include "rnla_internal.h"

namespace rnla {

int grid_for(rnla_ctx* ctx, int64_t work, int per_block);

// Raise (never lower) a kernel's dynamic shared-memory limit on the current
// device. The attribute is process-wide, so contexts launching the same kernel
// from several host threads must not shrink it under each other.
void ensure_dyn_smem(const void* kernel, size_t bytes);

template <class S, class D>
void copy2d_cast(rnla_ctx* ctx, int64_t rows, int64_t cols, const S* src, int64_t s_rs, int64_t s_cs, D* dst,
                 int64_t d_rs, int64_t d_cs);

// sum_i (a_i . x - b_i)^2 in fp64 (x on the device, fp64).
template <class T>
double residual_sq(rnla_ctx* ctx, int64_t n, int64_t d, const T* A, int64_t a_rs, int64_t a_cs, const T* b,
                   int64_t b_rs, const double* x_dev);

}  // namespace rnla
