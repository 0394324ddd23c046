// rbf.cuh -- RBF kernel blocks and gathers (rbf.cu).
#pragma once
#include "rnla_internal.h"

namespace rnla {

// out[i] = |X_r|^2 with r = rows ? rows[i] : i (sequential FMA chain).
template <class T>
void sq_norms(rnla_ctx* ctx, int64_t n, int64_t d, const T* X, int64_t rs, int64_t cs, const int64_t* rows, T* out);

// K(i, j) = exp((x_i . y_{sel(j)} - (sqx_i + sqy_j)/2) / sigma^2); entries with
// diag_of[j] == i are exactly 1 (the same point).
template <class T>
void rbf_block(rnla_ctx* ctx, int64_t n1, int64_t n2, int64_t d, const T* X, int64_t x_rs, int64_t x_cs, const T* Y,
               int64_t y_rs, int64_t y_cs, const int64_t* ysel, const T* sqx, const T* sqy, double sigma,
               const int64_t* diag_of, T* K, int64_t k_rs, int64_t k_cs);

// C(:, t) = A(:, idx[t]) * (scale ? scale[t] : 1).
template <class T>
void gather_columns(rnla_ctx* ctx, int64_t rows, int64_t cnt, const T* A, int64_t a_rs, int64_t a_cs,
                    const int64_t* idx, const double* scale, T* C, int64_t c_rs, int64_t c_cs);

// out[i] = sum_c M(i, c)^2 (fp64).
template <class T>
void row_sqnorms(rnla_ctx* ctx, int64_t n, int64_t d, const T* M, int64_t rs, int64_t cs, double* out);

}  // namespace rnla

namespace rnla {
// out(i, c) = A(idx[i], c) for i < cnt, c < cols (0 where idx[i] < 0).
template <class T>
void gather_rows(rnla_ctx* ctx, int64_t cnt, int64_t cols, const T* A, int64_t a_rs, int64_t a_cs, const int64_t* idx,
                 T* out, int64_t o_rs, int64_t o_cs);
// out = 0.5 * (W + W') for column-major n x n fp64 W (src/spsd.cpp:195-196).
void symmetrize(rnla_ctx* ctx, int64_t n, const double* W, double* out);
}  // namespace rnla

namespace rnla {
// Exact int8-digit Gram route for fp32 RBF kernel columns (gram_i8.cu).
bool gram_i8_available();
int64_t digit_pitch(int64_t n);
// Digits of K(i, j) (x rows vs y rows, diag_of forcing exact ones) into three
// int8 planes (planes + d * plane_stride + j * pitch + i), or the exact
// dequantized fp64 values into w (w[i + j * ldw]) when planes == nullptr.
void rbf_digits(rnla_ctx* ctx, int64_t n1, int64_t n2, int64_t d, const float* X, int64_t x_rs, int64_t x_cs,
                const float* Y, int64_t y_rs, int64_t y_cs, const float* sqx, const float* sqy, double sigma,
                const int64_t* diag_of, int8_t* planes, int64_t pitch, int64_t plane_stride, double* w, int64_t ldw);
// G (s x s col-major fp64; += when accumulate) = exact Gram of the digit
// planes of an n x s matrix (plane d of column p at planes + d s pitch + p pitch).
// reserve_sms SMs are left free (for concurrent work on another stream).
void gram_i8(rnla_ctx* ctx, const int8_t* planes, int64_t n, int64_t s, int64_t pitch, double* G, bool accumulate,
             int reserve_sms = 0);
// The digit planes of K(X, X_S) from a tcgen05 3xTF32 X X_S' (d <= 64) with the
// RBF epilogue in registers (rows i < n of the block; diag_of[j] == i -> 1).
bool rbf_tc_available(int64_t d);
void rbf_tc_digits(rnla_ctx* ctx, int64_t n, int64_t s, int64_t d, const float* X, int64_t x_rs, int64_t x_cs,
                   const float* Xs, int64_t s_rs, int64_t s_cs, const float* sqx, const float* sqy, double sigma,
                   const int64_t* diag_of, int8_t* planes, int64_t pitch, int64_t plane_stride,
                   int reserve_sms = 0);
// W[a, b] = dequantized digits at (row dsel[a], column b), 0 where dsel[a] < 0.
void w_from_digits(rnla_ctx* ctx, int64_t s, const int64_t* dsel, const int8_t* planes, int64_t pitch,
                   int64_t plane_stride, double* W);
}  // namespace rnla
