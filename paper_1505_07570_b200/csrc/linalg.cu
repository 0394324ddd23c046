#include <cstring>
// linalg.cu -- the small dense factorizations on the device.
//
// The reference does all of them with Eigen on the host
// (src/core.cpp:15-88: HouseholderQR, BDCSVD; src/spsd.cpp:195:
// SelfAdjointEigenSolver). Here they run on the GPU in fp64 through cuSOLVER
// (acceptable for the small s x s / c x c factorizations), plus
// the reference's sign convention (fix_column_signs, src/core.cpp:15-33) as a
// kernel. Inputs of the fp32 paths are promoted to fp64 for these steps.
#include <cublas_v2.h>
#include <cusolverDn.h>

#include "dist.h"
#include "linalg.cuh"
#include "util.cuh"

namespace rnla {

namespace {

void cusolver_check(cusolverStatus_t s, const char* what) {
  if (s != CUSOLVER_STATUS_SUCCESS) throw CudaError(std::string(what) + ": cuSOLVER status " + std::to_string((int)s));
}

cusolverDnHandle_t solver(rnla_ctx* ctx) { return static_cast<cusolverDnHandle_t>(ctx->cusolver); }

void check_info(rnla_ctx* ctx, const DevBuf& info, const char* what) {
  int h = 0;
  RNLA_CUDA(cudaMemcpyAsync(&h, info.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
  if (h != 0) throw NumericError(std::string(what) + ": info = " + std::to_string(h));
}

// One CTA per column: the first entry with |m| > tol decides the sign
// (src/core.cpp:15-33); flips the column of M and column/row j of P.
template <class T>
__global__ void flip_cols_kernel(int64_t rows, int64_t cols, T* M, int64_t m_rs, int64_t m_cs,
                                 const int* __restrict__ flip) {
  const int64_t total = rows * cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = (m_rs == 1) ? e % rows : e / cols, j = (m_rs == 1) ? e / rows : e % cols;
    if (flip[j]) M[i * m_rs + j * m_cs] = -M[i * m_rs + j * m_cs];
  }
}

template <class T>
__global__ void fix_signs_kernel(int64_t rows, int64_t cols, const T* M, int64_t m_rs, int64_t m_cs, T* P,
                                 int64_t p_rs, int64_t p_cs, int64_t p_len, int pair_cols, double tol, int* flip) {
  const int64_t j = blockIdx.x;
  if (j >= cols) return;
  __shared__ int64_t first;
  if (threadIdx.x == 0) first = INT64_MAX;
  __syncthreads();
  int64_t mine = INT64_MAX;
  for (int64_t i = threadIdx.x; i < rows; i += blockDim.x)
    if (fabs((double)M[i * m_rs + j * m_cs]) > tol) { mine = i; break; }
  if (mine != INT64_MAX) atomicMin((unsigned long long*)&first, (unsigned long long)mine);
  __syncthreads();
  if (first == INT64_MAX) return;
  const T lead = M[first * m_rs + j * m_cs];
  __syncthreads();
  if (!(lead < T(0))) return;
  if (threadIdx.x == 0) flip[j] = 1;  // the column of M is negated by flip_cols_kernel
  if (P)
    for (int64_t i = threadIdx.x; i < p_len; i += blockDim.x) {
      T* q = pair_cols ? &P[i * p_rs + j * p_cs] : &P[j * p_rs + i * p_cs];
      *q = -*q;
    }
}

__global__ void upper_copy_kernel(int64_t n, const double* __restrict__ A, int64_t lda, double* R, int64_t r_rs,
                                  int64_t r_cs) {
  const int64_t total = n * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % n, j = e / n;
    R[i * r_rs + j * r_cs] = i <= j ? A[i + j * lda] : 0.0;  // exact zeros below the diagonal
  }
}

}  // namespace

void fix_column_signs(rnla_ctx* ctx, int64_t rows, int64_t cols, double* M, int64_t m_rs, int64_t m_cs, double* P,
                      int64_t p_rs, int64_t p_cs, int64_t p_len, bool pair_cols) {
  if (cols == 0) return;
  DevBuf flip(sizeof(int) * cols, ctx->stream);
  RNLA_CUDA(cudaMemsetAsync(flip.p, 0, sizeof(int) * cols, ctx->stream));
  fix_signs_kernel<double><<<(unsigned)cols, 256, 0, ctx->stream>>>(rows, cols, M, m_rs, m_cs, P, p_rs, p_cs, p_len,
                                                                    pair_cols ? 1 : 0, 1e-12, flip.as<int>());
  RNLA_CUDA(cudaGetLastError());
  flip_cols_kernel<double><<<grid_for(ctx, rows * cols, 256), 256, 0, ctx->stream>>>(rows, cols, M, m_rs, m_cs,
                                                                                      flip.as<int>());
  RNLA_CUDA(cudaGetLastError());
  note_launch(ctx, 2);
}

namespace {
// *status |= bit when *flag is set
__global__ void or_flag_kernel(const int* flag, int bit, int* status) {
  if (*flag) *status |= bit;
}

// q0_j = sum_p Y(0, p) Rinv(p, j) in fp64; negate column j of Rinv when
// q0_j < 0 so that Q = Y Rinv comes out with the reference's sign rule
// (first entry with |q| > 1e-12 non-negative, src/core.cpp:15-33). Entries
// too close to zero to decide reliably raise *ambiguous.
template <class T>
__global__ void presign_kernel(int64_t cols, const T* __restrict__ Y, int64_t y_cs, double* Rinv, int* ambiguous) {
  for (int64_t j = threadIdx.x; j < cols; j += blockDim.x) {
    double q0 = 0.0;
    for (int64_t p = 0; p <= j; ++p) q0 += (double)Y[p * y_cs] * Rinv[p + j * cols];
    if (fabs(q0) < 1e-6) {
      atomicOr(ambiguous, 1);
    } else if (q0 < 0.0) {
      for (int64_t p = 0; p <= j; ++p) Rinv[p + j * cols] = -Rinv[p + j * cols];
    }
  }
}
}  // namespace

template <class T>
bool presign_upper_inverse(rnla_ctx* ctx, int64_t cols, const T* Y, int64_t y_cs, double* Rinv) {
  DevBuf flag(sizeof(int), ctx->stream);
  RNLA_CUDA(cudaMemsetAsync(flag.p, 0, sizeof(int), ctx->stream));
  presign_kernel<T><<<1, 256, 0, ctx->stream>>>(cols, Y, y_cs, Rinv, flag.as<int>());
  RNLA_CUDA(cudaGetLastError());
  note_launch(ctx);
  int h = 0;
  RNLA_CUDA(cudaMemcpyAsync(&h, flag.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
  return h == 0;
}
template bool presign_upper_inverse<double>(rnla_ctx*, int64_t, const double*, int64_t, double*);
template bool presign_upper_inverse<float>(rnla_ctx*, int64_t, const float*, int64_t, double*);

namespace {
// sign[j] = sign of the first entry of column j with |m| > tol (0: none).
template <class T>
__global__ void lead_sign_kernel(int64_t rows, int64_t cols, const T* M, int64_t m_rs, int64_t m_cs, double tol,
                                 double* sign) {
  const int64_t j = blockIdx.x;
  if (j >= cols) return;
  __shared__ unsigned long long first;
  if (threadIdx.x == 0) first = ~0ull;
  __syncthreads();
  for (int64_t i = threadIdx.x; i < rows; i += blockDim.x)
    if (fabs((double)M[i * m_rs + j * m_cs]) > tol) {
      atomicMin(&first, (unsigned long long)i);
      break;
    }
  __syncthreads();
  if (threadIdx.x == 0) sign[j] = first == ~0ull ? 0.0 : (M[(int64_t)first * m_rs + j * m_cs] < T(0) ? -1.0 : 1.0);
}

__global__ void flip_paired_kernel(int64_t cols, const int* __restrict__ flip, double* P, int64_t p_rs, int64_t p_cs,
                                   int64_t p_len, int pair_cols) {
  const int64_t total = cols * p_len;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / p_len, i = e % p_len;
    if (!flip[j]) continue;
    double* q = pair_cols ? &P[i * p_rs + j * p_cs] : &P[j * p_rs + i * p_cs];
    *q = -*q;
  }
}
}  // namespace

template <class T>
void fix_column_signs_sharded(rnla_ctx* ctx, int64_t rows, int64_t cols, T* M, int64_t m_rs, int64_t m_cs, double* P,
                              int64_t p_rs, int64_t p_cs, int64_t p_len, bool pair_cols) {
  if (cols == 0) return;
  const int W = std::max(1, ctx->world);
  DevBuf sign(sizeof(double) * cols, ctx->stream), all(sizeof(double) * cols * W, ctx->stream);
  lead_sign_kernel<T><<<(unsigned)cols, 256, 0, ctx->stream>>>(rows, cols, M, m_rs, m_cs, 1e-12, sign.as<double>());
  RNLA_CUDA(cudaGetLastError());
  note_launch(ctx);
  allgather_blocks(ctx, sign.p, all.p, (size_t)cols, RNLA_F64);
  std::vector<double> h((size_t)(cols * W));
  RNLA_CUDA(cudaMemcpyAsync(h.data(), all.p, sizeof(double) * cols * W, cudaMemcpyDeviceToHost, ctx->stream));
  RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
  std::vector<int> flip((size_t)cols, 0);
  for (int64_t j = 0; j < cols; ++j)
    for (int r = 0; r < W; ++r) {  // ranks hold consecutive row blocks: the first decisive rank wins
      const double sgn = h[(size_t)(r * cols + j)];
      if (sgn != 0.0) {
        flip[(size_t)j] = sgn < 0.0;
        break;
      }
    }
  DevBuf fl(sizeof(int) * cols, ctx->stream);
  RNLA_CUDA(cudaMemcpyAsync(fl.p, flip.data(), sizeof(int) * cols, cudaMemcpyHostToDevice, ctx->stream));
  if (rows > 0) {
    flip_cols_kernel<T><<<grid_for(ctx, rows * cols, 256), 256, 0, ctx->stream>>>(rows, cols, M, m_rs, m_cs,
                                                                                  fl.as<int>());
    RNLA_CUDA(cudaGetLastError());
    note_launch(ctx);
  }
  if (P && p_len > 0) {
    flip_paired_kernel<<<grid_for(ctx, cols * p_len, 256), 256, 0, ctx->stream>>>(cols, fl.as<int>(), P, p_rs, p_cs,
                                                                                   p_len, pair_cols ? 1 : 0);
    RNLA_CUDA(cudaGetLastError());
    note_launch(ctx);
  }
  RNLA_CUDA(cudaStreamSynchronize(ctx->stream));  // `flip` host vector lifetime
}
template void fix_column_signs_sharded<double>(rnla_ctx*, int64_t, int64_t, double*, int64_t, int64_t, double*, int64_t,
                                               int64_t, int64_t, bool);
template void fix_column_signs_sharded<float>(rnla_ctx*, int64_t, int64_t, float*, int64_t, int64_t, double*, int64_t,
                                              int64_t, int64_t, bool);

void fix_column_signs_f32(rnla_ctx* ctx, int64_t rows, int64_t cols, float* M, int64_t m_rs, int64_t m_cs) {
  if (cols == 0) return;
  DevBuf flip(sizeof(int) * cols, ctx->stream);
  RNLA_CUDA(cudaMemsetAsync(flip.p, 0, sizeof(int) * cols, ctx->stream));
  fix_signs_kernel<float><<<(unsigned)cols, 256, 0, ctx->stream>>>(rows, cols, M, m_rs, m_cs, nullptr, 0, 0, 0, 1,
                                                                   1e-12, flip.as<int>());
  RNLA_CUDA(cudaGetLastError());
  flip_cols_kernel<float><<<grid_for(ctx, rows * cols, 256), 256, 0, ctx->stream>>>(rows, cols, M, m_rs, m_cs,
                                                                                     flip.as<int>());
  RNLA_CUDA(cudaGetLastError());
  note_launch(ctx, 2);
}

void qr_householder(rnla_ctx* ctx, int64_t m, int64_t n, double* A, double* R, int64_t r_rs, int64_t r_cs) {
  require(m >= n, "thin_qr: rows < cols");
  if (n == 0) return;
  cusolverDnHandle_t h = solver(ctx);
  int lwork = 0, lwork2 = 0;
  DevBuf tau(sizeof(double) * n, ctx->stream), info(sizeof(int), ctx->stream);
  cusolver_check(cusolverDnDgeqrf_bufferSize(h, (int)m, (int)n, A, (int)m, &lwork), "geqrf_bufferSize");
  cusolver_check(cusolverDnDorgqr_bufferSize(h, (int)m, (int)n, (int)n, A, (int)m, tau.as<double>(), &lwork2),
                 "orgqr_bufferSize");
  DevBuf work(sizeof(double) * std::max(lwork, lwork2), ctx->stream);
  cusolver_check(cusolverDnDgeqrf(h, (int)m, (int)n, A, (int)m, tau.as<double>(), work.as<double>(), lwork,
                                  info.as<int>()),
                 "geqrf");
  note_launch(ctx);
  upper_copy_kernel<<<grid_for(ctx, n * n, 256), 256, 0, ctx->stream>>>(n, A, m, R, r_rs, r_cs);
  RNLA_CUDA(cudaGetLastError());
  note_launch(ctx);
  cusolver_check(cusolverDnDorgqr(h, (int)m, (int)n, (int)n, A, (int)m, tau.as<double>(), work.as<double>(),
                                  std::max(lwork, lwork2), info.as<int>()),
                 "orgqr");
  note_launch(ctx);
  check_info(ctx, info, "thin_qr");
}

void svd_thin(rnla_ctx* ctx, int64_t m, int64_t n, const double* A, int64_t a_rs, int64_t a_cs, double* U, double* S,
              double* V) {
  // U: m x r col-major (ld m), S[r], V: n x r col-major (ld n), r = min(m, n).
  const bool tall = m >= n;
  const int64_t M = tall ? m : n, N = tall ? n : m;  // factor the tall orientation
  DevBuf work_a(sizeof(double) * M * N, ctx->stream);
  double* W = work_a.as<double>();
  if (tall) copy2d<double>(ctx, m, n, A, a_rs, a_cs, W, 1, M);
  else copy2d<double>(ctx, n, m, A, a_cs, a_rs, W, 1, M);  // W = A^T
  DevBuf u(sizeof(double) * M * N, ctx->stream), vt(sizeof(double) * N * N, ctx->stream);
  DevBuf info(sizeof(int), ctx->stream);
  cusolverDnHandle_t h = solver(ctx);
  int lwork = 0;
  cusolver_check(cusolverDnDgesvd_bufferSize(h, (int)M, (int)N, &lwork), "gesvd_bufferSize");
  DevBuf work(sizeof(double) * lwork, ctx->stream), rwork(sizeof(double) * N, ctx->stream);
  cusolver_check(cusolverDnDgesvd(h, 'S', 'S', (int)M, (int)N, W, (int)M, S, u.as<double>(), (int)M, vt.as<double>(),
                                  (int)N, work.as<double>(), lwork, rwork.as<double>(), info.as<int>()),
                 "gesvd");
  note_launch(ctx);
  check_info(ctx, info, "condensed_svd");
  // Tall: U = u (m x n), V = vt^T. Wide: A^T = u S vt => A = vt^T S u^T: U = vt^T, V = u.
  if (tall) {
    copy2d<double>(ctx, m, N, u.as<double>(), 1, M, U, 1, m);
    copy2d<double>(ctx, n, N, vt.as<double>(), N, 1, V, 1, n);  // V(i,j) = vt(j,i)
  } else {
    copy2d<double>(ctx, m, N, vt.as<double>(), N, 1, U, 1, m);
    copy2d<double>(ctx, n, N, u.as<double>(), 1, M, V, 1, n);
  }
}

bool cholesky_upper(rnla_ctx* ctx, int64_t n, double* G) {
  cusolverDnHandle_t h = solver(ctx);
  int lwork = 0;
  DevBuf info(sizeof(int), ctx->stream);
  cusolver_check(cusolverDnDpotrf_bufferSize(h, CUBLAS_FILL_MODE_UPPER, (int)n, G, (int)n, &lwork),
                 "potrf_bufferSize");
  DevBuf work(sizeof(double) * std::max(lwork, 1), ctx->stream);
  cusolver_check(cusolverDnDpotrf(h, CUBLAS_FILL_MODE_UPPER, (int)n, G, (int)n, work.as<double>(), lwork,
                                  info.as<int>()),
                 "potrf");
  note_launch(ctx);
  int hinfo = 0;
  RNLA_CUDA(cudaMemcpyAsync(&hinfo, info.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
  return hinfo == 0;
}

bool cholqr_inplace(rnla_ctx* ctx, int64_t m, int64_t n, double* Y) {
  DevBuf G(sizeof(double) * n * n, ctx->stream);
  gemm<double>(ctx, n, n, m, 1.0, Y, m, 1, Y, 1, m, 0.0, G.as<double>(), 1, n);
  if (!cholesky_upper(ctx, n, G.as<double>())) return false;
  const double one = 1.0;
  if (cublasDtrsm(static_cast<cublasHandle_t>(ctx->cublas), CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N,
                  CUBLAS_DIAG_NON_UNIT, (int)m, (int)n, &one, G.as<double>(), (int)n, Y, (int)m) !=
      CUBLAS_STATUS_SUCCESS)
    throw CudaError("cublasDtrsm failed");
  note_launch(ctx);
  return true;
}

bool diag_ratio_ok(rnla_ctx* ctx, int64_t n, const double* R, double thresh) {
  std::vector<double> d((size_t)n);
  RNLA_CUDA(cudaMemcpy2DAsync(d.data(), sizeof(double), R, sizeof(double) * (n + 1), sizeof(double), n,
                              cudaMemcpyDeviceToHost, ctx->stream));
  RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
  double lo = INFINITY, hi = 0.0;
  for (double v : d) {
    if (!std::isfinite(v)) return false;
    lo = std::min(lo, std::fabs(v));
    hi = std::max(hi, std::fabs(v));
  }
  return n == 0 || (hi > 0.0 && lo > thresh * hi);
}

namespace {
__global__ void identity_kernel(int64_t n, double* M) {
  const int64_t total = n * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x)
    M[e] = (e % n == e / n) ? 1.0 : 0.0;
}
}  // namespace

namespace {
constexpr int TB = 128, TS = 32, TLD = TB + 1;
// X = R^-1 of the bs x bs (bs <= 128) diagonal block b of the upper triangular
// R (column-major, ld): four 32 x 32 diagonal sub-blocks inverted by one warp
// each (lane = column, back substitution), then the off-diagonal sub-blocks
// by block distance, X_IJ = -X_II sum_{K = I+1..J} R_IK X_KJ. One CTA per
// diagonal block, all blocks in one launch.
__global__ void __launch_bounds__(256) tri_block_inv_kernel(int64_t n, const double* __restrict__ R, int64_t ld,
                                                            double* __restrict__ X, int64_t ldx) {
  extern __shared__ double ts[];  // R(i, j) at ts[i * TLD + j] (i <= j); X(i, j) at ts[j * TLD + i] (i < j)
  double* xd = ts + TB * TLD;     // X(i, i)
  double* tmp = xd + TB;          // [3][TS][TS]
  const int64_t b0 = (int64_t)blockIdx.x * TB;
  const int bs = (int)min((int64_t)TB, n - b0);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double* Rb = R + b0 + b0 * ld;
  for (int e = tid; e < bs * bs; e += blockDim.x) {
    const int i = e % bs, j = e / bs;
    if (i <= j) ts[i * TLD + j] = Rb[i + (int64_t)j * ld];
  }
  __syncthreads();
  const int nsb = (bs + TS - 1) / TS;
  if (warp < nsb) {
    const int c0 = warp * TS, w = min(TS, bs - c0), col = c0 + lane;
    if (lane < w) {
      double xs[TS];
#pragma unroll
      for (int t = 0; t < TS; ++t) xs[t] = 0.0;
#pragma unroll
      for (int t = TS - 1; t >= 0; --t) {
        const int i = c0 + t;
        if (t < w && i <= col) {
          double v = i == col ? 1.0 : 0.0;
#pragma unroll
          for (int u = t + 1; u < TS; ++u)
            if (u < w && c0 + u <= col) v -= ts[i * TLD + c0 + u] * xs[u];
          xs[t] = v / ts[i * TLD + i];
        }
      }
#pragma unroll
      for (int t = 0; t < TS; ++t) {
        const int i = c0 + t;
        if (t < w && i < col) ts[col * TLD + i] = xs[t];
        if (t < w && i == col) xd[col] = xs[t];
      }
    }
  }
  __syncthreads();
  auto xget = [&](int i, int j) -> double { return i == j ? xd[i] : ts[j * TLD + i]; };
  for (int dist = 1; dist < nsb; ++dist) {
    const int npairs = nsb - dist;
    for (int e = tid; e < npairs * TS * TS; e += blockDim.x) {
      const int pr = e / (TS * TS), r = (e / TS) % TS, c = e % TS;
      const int row = pr * TS + r, col = (pr + dist) * TS + c;
      double v = 0.0;
      if (row < bs && col < bs)
        for (int p = (pr + 1) * TS; p <= col; ++p) v += ts[row * TLD + p] * xget(p, col);
      tmp[e] = v;
    }
    __syncthreads();
    for (int e = tid; e < npairs * TS * TS; e += blockDim.x) {
      const int pr = e / (TS * TS), r = (e / TS) % TS, c = e % TS;
      const int row = pr * TS + r, col = (pr + dist) * TS + c;
      if (row < bs && col < bs) {
        double v = 0.0;
        for (int q = r; q < TS && pr * TS + q < bs; ++q) v += xget(row, pr * TS + q) * tmp[(pr * TS + q) * TS + c];
        ts[col * TLD + row] = -v;
      }
    }
    __syncthreads();
  }
  double* Xb = X + b0 + b0 * ldx;
  for (int e = tid; e < bs * bs; e += blockDim.x) {
    const int i = e % bs, j = e / bs;
    Xb[i + (int64_t)j * ldx] = i < j ? ts[j * TLD + i] : (i == j ? xd[i] : 0.0);
  }
}
}  // namespace

void upper_inverse(rnla_ctx* ctx, int64_t n, const double* R, double* Rinv) {
  if (n >= 2 * TB && !std::getenv("RNLA_TRSM_INVERSE")) {
    // Blocked: the 128 x 128 diagonal-block inverses in one launch, then the
    // pairwise merges X_IJ = -X_II (R_IJ X_JJ) for block sizes 128, 256, ...
    // (DMMA GEMMs). cuBLAS trsm against the identity took 1.3 ms at n = 2048.
    RNLA_CUDA(cudaMemsetAsync(Rinv, 0, sizeof(double) * (size_t)(n * n), ctx->stream));
    const size_t smem = sizeof(double) * ((size_t)TB * TLD + TB + 3 * TS * TS);
    ensure_dyn_smem((const void*)tri_block_inv_kernel, smem);
    tri_block_inv_kernel<<<(unsigned)((n + TB - 1) / TB), 256, smem, ctx->stream>>>(n, R, n, Rinv, n);
    RNLA_CUDA(cudaGetLastError());
    note_launch(ctx);
    // Transposed forms keep both GEMMs on the K-major-A DMMA kernel:
    //   U = X_JJ' R_IJ' (bj x bi, row-major), X_IJ' = -U X_II' (written transposed).
    DevBuf U(sizeof(double) * (size_t)(n * (n / 2 + TB)), ctx->stream);
    for (int64_t b = TB; b < n; b *= 2) {
      for (int64_t i0 = 0; i0 + b < n; i0 += 2 * b) {
        const int64_t j0 = i0 + b, bi = b, bj = std::min<int64_t>(b, n - j0);
        gemm<double>(ctx, bj, bi, bj, 1.0, Rinv + j0 + j0 * n, n, 1, R + i0 + j0 * n, n, 1, 0.0, U.as<double>(), bi,
                     1);
        gemm<double>(ctx, bj, bi, bi, -1.0, U.as<double>(), bi, 1, Rinv + i0 + i0 * n, n, 1, 0.0,
                     Rinv + i0 + j0 * n, n, 1);
      }
    }
    RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
    return;
  }
  // Rinv = R^-1 by a triangular solve against the identity (built on the device:
  // an n^2 host upload cost ~3 ms at n = 1024). cuSOLVER trtri measured slower
  // here (leverage rows 29.8 vs 25.3 ms at n = 1024).
  identity_kernel<<<grid_for(ctx, n * n, 256), 256, 0, ctx->stream>>>(n, Rinv);
  RNLA_CUDA(cudaGetLastError());
  note_launch(ctx);
  const double one = 1.0;
  if (cublasDtrsm(static_cast<cublasHandle_t>(ctx->cublas), CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N,
                  CUBLAS_DIAG_NON_UNIT, (int)n, (int)n, &one, R, (int)n, Rinv, (int)n) != CUBLAS_STATUS_SUCCESS)
    throw CudaError("cublasDtrsm failed");
  note_launch(ctx);
  RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
}

void eig_sym(rnla_ctx* ctx, int64_t n, double* A, double* W) {
  cusolverDnHandle_t h = solver(ctx);
  int lwork = 0;
  DevBuf info(sizeof(int), ctx->stream);
  cusolver_check(cusolverDnDsyevd_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, (int)n, A, (int)n, W,
                                             &lwork),
                 "syevd_bufferSize");
  DevBuf work(sizeof(double) * lwork, ctx->stream);
  cusolver_check(cusolverDnDsyevd(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, (int)n, A, (int)n, W,
                                  work.as<double>(), lwork, info.as<int>()),
                 "syevd");
  note_launch(ctx);
  check_info(ctx, info, "eig");
}

void eig_sym_async(rnla_ctx* ctx, int64_t n, double* A, double* W, int* info) {
  cusolverDnHandle_t h = solver(ctx);
  int lwork = 0;
  cusolver_check(cusolverDnDsyevd_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, (int)n, A, (int)n, W,
                                             &lwork),
                 "syevd_bufferSize");
  DevBuf work(sizeof(double) * lwork, ctx->stream);
  cusolver_check(cusolverDnDsyevd(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, (int)n, A, (int)n, W,
                                  work.as<double>(), lwork, info),
                 "syevd");
  note_launch(ctx);
}

int64_t eig_sym_top(rnla_ctx* ctx, int64_t n, double* A, int64_t k, double* W) {
  cusolverDnHandle_t h = solver(ctx);
  int lwork = 0, found = 0;
  DevBuf info(sizeof(int), ctx->stream);
  const int il = (int)(n - k + 1), iu = (int)n;
  cusolver_check(cusolverDnDsyevdx_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, CUSOLVER_EIG_RANGE_I,
                                              CUBLAS_FILL_MODE_LOWER, (int)n, A, (int)n, 0.0, 0.0, il, iu, &found, W,
                                              &lwork),
                 "syevdx_bufferSize");
  DevBuf work(sizeof(double) * lwork, ctx->stream);
  cusolver_check(cusolverDnDsyevdx(h, CUSOLVER_EIG_MODE_VECTOR, CUSOLVER_EIG_RANGE_I, CUBLAS_FILL_MODE_LOWER, (int)n,
                                   A, (int)n, 0.0, 0.0, il, iu, &found, W, work.as<double>(), lwork, info.as<int>()),
                 "syevdx");
  note_launch(ctx);
  check_info(ctx, info, "eig");
  return found;
}

// ---------------------------------------------------------------------------
// One-CTA Cholesky + triangular inverse for the CholeskyQR2 passes of
// tall-skinny orthonormalization (n <= kSmallCholMax): no cuSOLVER call and no
// host round trip per pass (the potrf info read, the diagonal-ratio check and
// the sign probe each synchronized the stream before).
// ---------------------------------------------------------------------------
namespace {

constexpr int kSmallCholThreads = 1024;

// G (n x n, column-major, upper triangle read) = R'R; Rinv = R^-1 (column-major,
// exact zeros below the diagonal), optionally also as fp32. status bits:
// 1 = not positive definite / non-finite, 2 = min|r_ii| <= thresh * max|r_ii|,
// 4 = sign of a column of Q = Y Rinv undecidable from row 0 (|q0| < 1e-6).
// With y0 set, columns of Rinv are negated so that row 0 of Y Rinv is >= 0
// (the reference's sign rule, src/core.cpp:15-33).
template <class T>
__global__ void __launch_bounds__(kSmallCholThreads) small_chol_inv_kernel(int n, const double* __restrict__ G,
                                                                          double* __restrict__ Rinv, float* Rinv32,
                                                                          const T* __restrict__ y0, int64_t y_cs,
                                                                          double thresh, int* status) {
  extern __shared__ double sm[];  // R / X: [n][n + 1], element (i, j) at i * (n + 1) + j
  __shared__ double dmin, dmax;
  const int ld = n + 1, tid = threadIdx.x, nt = blockDim.x;
  for (int e = tid; e < n * n; e += nt) {
    const int i = e % n, j = e / n;
    sm[i * ld + j] = i <= j ? G[e] : 0.0;
  }
  __syncthreads();
  // right-looking upper Cholesky in the square-root-free form: step k updates
  // the trailing upper triangle with row k unscaled, A(i, j) -= A(k, i) A(k, j) / A(k, k),
  // so one barrier per step suffices; rows are scaled by 1/sqrt(A(k, k)) at the end.
  // The trailing matrix lives in registers: thread (tx, ty) of the 32 x 32 grid
  // owns the elements (ty + 32 ii, tx + 32 jj), ii <= jj < 5 (n <= 160), and each
  // step only publishes row k through a double-buffered shared row. Same
  // operations in the same order, so the factor is bitwise unchanged. Measured
  // (clock64 per phase, n = 150): the factorization loop 0.9 -> 0.55 us per step,
  // kernel 214 -> 157 us; what remains per step is the dependent fp64 chain
  // pivot -> 1/d -> a_ki -> FMA -> publish (~1000 cycles), not instruction issue.
  // (A blocked variant -- warp 0 factoring 16-row panels, all threads applying
  // the rank-16 updates -- measured slower: 0.37 vs 0.24 ms at n = 150.)
  static_assert(kSmallCholMax <= 160 && kSmallCholThreads == 1024, "register tiling of the Cholesky step");
  constexpr int NB = 5;
  const int tx = tid & 31, ty = tid >> 5, nty = nt >> 5;
  auto ridx = [](int ii, int jj) { return ii * NB - ii * (ii - 1) / 2 + (jj - ii); };
  // Out-of-range elements (i >= n or j >= n) hold zeros and the shared row is
  // zero beyond n, so their updates are no-ops; the lower halves of the diagonal
  // blocks (tx < ty) are updated like their mirror images and never published.
  // That leaves one warp-uniform test per step (is this warp's row of the pivot
  // block below the pivot?) and no per-element predicates.
  double a[NB * (NB + 1) / 2];
#pragma unroll
  for (int ii = 0; ii < NB; ++ii)
#pragma unroll
    for (int jj = ii; jj < NB; ++jj) {
      const int i = ty + 32 * ii, j = tx + 32 * jj;
      a[ridx(ii, jj)] = (n > 32 && i <= j && j < n) ? sm[i * ld + j] : 0.0;
    }
  constexpr int RB = 32 * NB;             // padded row length
  double* rowbuf = sm + (size_t)n * ld;  // 2 x RB doubles in the (still unused) inverse scratch
  if (n > 32) {
    for (int e = tid; e < 2 * RB; e += nt) rowbuf[e] = 0.0;
    __syncthreads();
  }
  bool isbad = false;
  if (n <= 32) {
    // one index block: the shared-memory form is shorter (25 vs 20 us at n = 30)
    for (int k = 0; k < n; ++k) {
      const double d = sm[k * ld + k];
      if (!(d > 0.0) || !isfinite(d)) {
        isbad = true;
        break;  // uniform: every thread read the same d
      }
      const double inv = 1.0 / d;
      for (int i = k + 1 + ty; i < n; i += nty) {
        const double aki = sm[k * ld + i] * inv;
        for (int j = i + tx; j < n; j += 32) sm[i * ld + j] -= aki * sm[k * ld + j];
      }
      __syncthreads();
    }
  }
#pragma unroll
  for (int kb = 0; kb < NB; ++kb) {
    if (n <= 32 || 32 * kb >= n || isbad) break;  // uniform
    for (int kk = 0; kk < 32; ++kk) {
      const int k = 32 * kb + kk;
      if (k >= n) break;  // uniform
      double* rb = rowbuf + (k & 1) * RB;
      if (ty == kk) {  // the owners of row k publish it (columns k .. n - 1)
#pragma unroll
        for (int jj = kb; jj < NB; ++jj) {
          const int j = tx + 32 * jj;
          if (j >= k && j < n) rb[j] = a[ridx(kb, jj)];
        }
      }
      __syncthreads();
      const double d = rb[k];
      if (!(d > 0.0) || !isfinite(d)) {
        isbad = true;
        break;  // uniform: every thread read the same d
      }
      const double inv = 1.0 / d;
      double rj[NB];
#pragma unroll
      for (int jj = kb; jj < NB; ++jj) rj[jj] = rb[tx + 32 * jj];
      if (ty > kk) {  // rows of the pivot block below the pivot (warp-uniform)
        const double aki = rb[ty + 32 * kb] * inv;
#pragma unroll
        for (int jj = kb; jj < NB; ++jj) a[ridx(kb, jj)] -= aki * rj[jj];
      }
#pragma unroll
      for (int ii = kb + 1; ii < NB; ++ii) {  // the blocks below are always active
        const double aki = rb[ty + 32 * ii] * inv;
#pragma unroll
        for (int jj = ii; jj < NB; ++jj) a[ridx(ii, jj)] -= aki * rj[jj];
      }
    }
  }
  __syncthreads();
  if (isbad) {
    if (tid == 0) *status = 1;
    return;
  }
  if (n > 32) {
#pragma unroll
    for (int ii = 0; ii < NB; ++ii)
#pragma unroll
      for (int jj = ii; jj < NB; ++jj) {
        const int i = ty + 32 * ii, j = tx + 32 * jj;
        if (i <= j && j < n) sm[i * ld + j] = a[ridx(ii, jj)];
      }
  }
  __syncthreads();
  for (int k = ty; k < n; k += nty) {
    const double dk = sqrt(sm[k * ld + k]), r = 1.0 / dk;
    for (int j = k + 1 + tx; j < n; j += 32) sm[k * ld + j] *= r;
    __syncwarp();
    if (tx == 0) sm[k * ld + k] = dk;
  }
  __syncthreads();
  if (tid == 0) {
    double lo = INFINITY, hi = 0.0;
    for (int k = 0; k < n; ++k) {
      lo = fmin(lo, fabs(sm[k * ld + k]));
      hi = fmax(hi, fabs(sm[k * ld + k]));
    }
    dmin = lo;
    dmax = hi;
  }
  __syncthreads();
  int st = (dmax > 0.0 && dmin > thresh * dmax) ? 0 : 2;
  // Blocked upper triangular inverse X = R^-1 with 16 x 16 blocks and a few
  // dozen barriers (a column-by-column inverse needed two per column):
  //  A: warp I inverts diagonal block R_II into Xd[I] (lane c: column c);
  //  B: block diagonal d = 1 .. nb-1: T_I = sum_{P=I+1..J} R_IP X_PJ, then
  //     X_IJ = -X_II T_I (J = I + d). Off-diagonal X blocks are kept transposed
  //     in the (zero) lower triangle of sm; at the end X moves to the upper one.
  constexpr int BS = 16;
  const int nb = (n + BS - 1) / BS;
  double* Xd = sm + (size_t)n * ld;              // [nb][BS][BS]
  double* Tb = Xd + (size_t)nb * BS * BS;         // [nb][BS][BS]
  double* tmp = Tb + (size_t)nb * BS * BS;        // n scratch doubles (sign probe)
  const int lane = tid & 31, wid = tid >> 5;
  if (wid < nb && lane < BS) {
    const int I0 = wid * BS, bs = min(BS, n - I0), c = lane;
    double x[BS];
#pragma unroll
    for (int r = 0; r < BS; ++r) x[r] = 0.0;
    if (c < bs) {
      x[0] = 0.0;
#pragma unroll
      for (int r = BS - 1; r >= 0; --r) {
        if (r == c) {
          x[r] = 1.0 / sm[(I0 + r) * ld + I0 + r];
        } else if (r < c) {
          double acc = 0.0;
#pragma unroll
          for (int p = r + 1; p < BS; ++p)
            if (p <= c) acc += sm[(I0 + r) * ld + I0 + p] * x[p];
          x[r] = -acc / sm[(I0 + r) * ld + I0 + r];
        }
      }
    }
#pragma unroll
    for (int r = 0; r < BS; ++r) Xd[(wid * BS + r) * BS + c] = (c < bs && r <= c) ? x[r] : 0.0;
  }
  __syncthreads();
  auto getx = [&](int p, int q) -> double {  // X(p, q), p <= q, blocks below the diagonal of q already formed
    const int bp = p / BS, bq = q / BS;
    return bp == bq ? Xd[(bp * BS + p % BS) * BS + q % BS] : sm[q * ld + p];
  };
  for (int d = 1; d < nb; ++d) {
    const int cnt = (nb - d) * BS * BS;
    for (int e = tid; e < cnt; e += nt) {
      const int I = e / (BS * BS), r = (e / BS) % BS, c = e % BS, J = I + d;
      const int row = I * BS + r, col = J * BS + c;
      // four independent partial sums: the dependent fp64 FMA chain (up to 16 d
      // terms) was the cost of this sweep, not the operation count. X(p, col) of
      // the blocks between I and J sits transposed in the lower triangle
      // (contiguous in p), the last block in Xd.
      double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;
      if (row < n && col < n) {
        const double* rr = sm + row * ld;
        const double* xc = sm + col * ld;
        for (int p = (I + 1) * BS; p < J * BS; p += 4) {
          acc0 += rr[p] * xc[p];
          acc1 += rr[p + 1] * xc[p + 1];
          acc2 += rr[p + 2] * xc[p + 2];
          acc3 += rr[p + 3] * xc[p + 3];
        }
        const double* xd = Xd + (size_t)J * BS * BS + c;
        for (int t = 0; t <= c; ++t) {
          const double v = rr[J * BS + t] * xd[t * BS];
          if ((t & 3) == 0) acc0 += v;
          else if ((t & 3) == 1) acc1 += v;
          else if ((t & 3) == 2) acc2 += v;
          else acc3 += v;
        }
      }
      Tb[e] = (acc0 + acc1) + (acc2 + acc3);
    }
    __syncthreads();
    for (int e = tid; e < cnt; e += nt) {
      const int I = e / (BS * BS), r = (e / BS) % BS, c = e % BS, J = I + d;
      const int row = I * BS + r, col = J * BS + c;
      if (row < n && col < n) {
        double acc = 0.0;
        for (int q = r; q < BS; ++q) acc += Xd[(I * BS + r) * BS + q] * Tb[(I * BS + q) * BS + c];
        sm[col * ld + row] = -acc;  // X(row, col), stored transposed
      }
    }
    __syncthreads();
  }
  for (int e = tid; e < n * n; e += nt) {
    const int i = e / n, j = e % n;
    if (i <= j) sm[i * ld + j] = getx(i, j);
  }
  __syncthreads();
  if (y0) {
    for (int j = tid; j < n; j += nt) {
      double q0 = 0.0;
      for (int p = 0; p <= j; ++p) q0 += (double)y0[p * y_cs] * sm[p * ld + j];
      tmp[j] = q0;
    }
    __syncthreads();
    for (int e = tid; e < n * n; e += nt) {
      const int i = e / n, j = e % n;
      if (i <= j && tmp[j] < 0.0) sm[i * ld + j] = -sm[i * ld + j];
    }
    if (tid == 0)
      for (int j = 0; j < n; ++j)
        if (fabs(tmp[j]) < 1e-6) st |= 4;
    __syncthreads();
  }
  for (int e = tid; e < n * n; e += nt) {
    const int i = e % n, j = e / n;
    const double v = i <= j ? sm[i * ld + j] : 0.0;
    Rinv[e] = v;
    if (Rinv32) Rinv32[e] = (float)v;
  }
  if (tid == 0) *status = st;
}

}  // namespace

template <class T>
void small_chol_inv(rnla_ctx* ctx, int64_t n, const double* G, double* Rinv, float* Rinv32, const T* y0, int64_t y_cs,
                    double thresh, int* status) {
  require(n >= 1 && n <= kSmallCholMax, "small_chol_inv: n out of range");
  const size_t nb = (size_t)((n + 15) / 16);
  const size_t smem = sizeof(double) * ((size_t)n * (n + 1) + 2 * nb * 256 + n);
  ensure_dyn_smem((const void*)small_chol_inv_kernel<T>, smem);
  small_chol_inv_kernel<T><<<1, kSmallCholThreads, smem, ctx->stream>>>((int)n, G, Rinv, Rinv32, y0, y_cs, thresh,
                                                                        status);
  RNLA_CUDA(cudaGetLastError());
  note_launch(ctx);
}
template void small_chol_inv<double>(rnla_ctx*, int64_t, const double*, double*, float*, const double*, int64_t,
                                     double, int*);
template void small_chol_inv<float>(rnla_ctx*, int64_t, const double*, double*, float*, const float*, int64_t, double,
                                    int*);

// ---------------------------------------------------------------------------
// The same CholeskyQR2 factorization step for wider blocks (n > kSmallCholMax)
// on cuSOLVER/cuBLAS, without host round trips: potrf's info, the diagonal
// ratio and the sign probe all land in a device status word.
// ---------------------------------------------------------------------------
namespace {
// status |= 1 (potrf info != 0 or a non-finite diagonal), |= 2 (min |r_ii| <= thresh * max |r_ii|)
__global__ void chol_status_kernel(int64_t n, const double* __restrict__ R, const int* __restrict__ info,
                                   double thresh, int* status) {
  __shared__ double lo_s[32], hi_s[32];
  __shared__ int bad_s;
  if (threadIdx.x == 0) bad_s = 0;
  __syncthreads();
  double lo = INFINITY, hi = 0.0;
  int bad = 0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double v = fabs(R[i * (n + 1)]);
    if (!isfinite(v)) bad = 1;
    lo = fmin(lo, v);
    hi = fmax(hi, v);
  }
  for (int o = 16; o > 0; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if (bad) atomicOr(&bad_s, 1);
  if ((threadIdx.x & 31) == 0) {
    lo_s[threadIdx.x >> 5] = lo;
    hi_s[threadIdx.x >> 5] = hi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      lo = fmin(lo, lo_s[w]);
      hi = fmax(hi, hi_s[w]);
    }
    int st = 0;
    if (*info != 0 || bad_s) st |= 1;
    else if (!(hi > 0.0 && lo > thresh * hi)) st |= 2;
    *status |= st;
  }
}
}  // namespace

template <class T>
void chol_inv_async(rnla_ctx* ctx, int64_t n, double* G, double* Rinv, float* Rinv32, const T* y0, int64_t y_cs,
                    double thresh, int* status) {
  cusolverDnHandle_t h = solver(ctx);
  int lwork = 0;
  cusolver_check(cusolverDnDpotrf_bufferSize(h, CUBLAS_FILL_MODE_UPPER, (int)n, G, (int)n, &lwork),
                 "potrf_bufferSize");
  DevBuf work(sizeof(double) * std::max(lwork, 1), ctx->stream), info(sizeof(int), ctx->stream);
  cusolver_check(cusolverDnDpotrf(h, CUBLAS_FILL_MODE_UPPER, (int)n, G, (int)n, work.as<double>(), lwork,
                                  info.as<int>()),
                 "potrf");
  chol_status_kernel<<<1, 256, 0, ctx->stream>>>(n, G, info.as<int>(), thresh, status);
  RNLA_CUDA(cudaGetLastError());
  identity_kernel<<<grid_for(ctx, n * n, 256), 256, 0, ctx->stream>>>(n, Rinv);
  RNLA_CUDA(cudaGetLastError());
  const double one = 1.0;
  if (cublasDtrsm(static_cast<cublasHandle_t>(ctx->cublas), CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N,
                  CUBLAS_DIAG_NON_UNIT, (int)n, (int)n, &one, G, (int)n, Rinv, (int)n) != CUBLAS_STATUS_SUCCESS)
    throw CudaError("cublasDtrsm failed");
  note_launch(ctx, 4);
  if (y0) {
    DevBuf amb(sizeof(int), ctx->stream);
    RNLA_CUDA(cudaMemsetAsync(amb.p, 0, sizeof(int), ctx->stream));
    presign_kernel<T><<<1, 256, 0, ctx->stream>>>(n, y0, y_cs, Rinv, amb.as<int>());
    RNLA_CUDA(cudaGetLastError());
    or_flag_kernel<<<1, 1, 0, ctx->stream>>>(amb.as<int>(), 4, status);
    RNLA_CUDA(cudaGetLastError());
    note_launch(ctx, 2);
  }
  if (Rinv32) {
    copy2d_cast<double, float>(ctx, n, n, Rinv, 1, n, Rinv32, 1, n);
  }
}
template void chol_inv_async<double>(rnla_ctx*, int64_t, double*, double*, float*, const double*, int64_t, double,
                                     int*);
template void chol_inv_async<float>(rnla_ctx*, int64_t, double*, double*, float*, const float*, int64_t, double,
                                    int*);

}  // namespace rnla

// ---------------------------------------------------------------------------
// Small symmetric eigenproblems: the s x s core Gram of prototype_ksvd's
// truncated SVD (s = 30 at config 0) and the b x b Rayleigh-Ritz matrices of
// the block subspace iteration (b = 96 at config 4).
//
// n <= kJacobiMax: one CTA, two-sided cyclic Jacobi in parallel (round-robin)
// order, A and V resident in shared memory. Round r rotates the n/2 disjoint
// pairs of the tournament schedule; warp w owns pairs w, w + nwarps, ...:
//   phase 1 (columns): the warp reads a_pp, a_qq, a_pq of its own pairs
//     (columns p, q are touched by no other warp in this phase), forms the
//     rotation and applies A <- A J, V <- V J to columns p, q;
//   barrier; phase 2 (rows): A <- J'A on rows p, q, a_pq = a_qp = 0; barrier.
// Two barriers per round. A pair is rotated when |a_pq| > 1e-15 sqrt(|a_pp a_qq|)
// (relative criterion: small eigenvalues of an SPD matrix keep their relative
// accuracy); the sweep loop stops after a sweep without rotations.
// Replaces cuSOLVER syevjBatched (n <= 32: 154 us for the config-0 30 x 30
// core) and syevj (config 4, b = 96).
#include "jacobi.cuh"
#include "syev_tri.cuh"

namespace rnla {
namespace {
// measured (tools/jacobi_bench.cu): n = 30 128 us vs 154 us for cuSOLVER
// syevjBatched; n = 96 1.02 ms standalone vs 1.67 ms for syevj, but the config-4
// Rayleigh-Ritz matrix (clustered eigenvalues) takes 9 sweeps (2.05 ms; config 4
// 11.1 vs 10.6 ms), so above 32 cuSOLVER stays
constexpr int kJacobiMax = 32;
}  // namespace

bool eig_small_jacobi_async(rnla_ctx* ctx, int64_t b, const double* H, double* lam, double* Z, int* status) {
  if (b < 1 || b > kJacobiMax || std::getenv("RNLA_EIG_CUSOLVER")) return false;
  const size_t smem = jacobi_smem_bytes((int)b);
  if (b <= 32) {
    ensure_dyn_smem((const void*)jacobi_eig_kernel<512>, smem);
    jacobi_eig_kernel<512><<<1, 512, smem, ctx->stream>>>((int)b, H, lam, Z, status);
  } else {
    ensure_dyn_smem((const void*)jacobi_eig_kernel<1024>, smem);
    jacobi_eig_kernel<1024><<<1, 1024, smem, ctx->stream>>>((int)b, H, lam, Z, status);
  }
  RNLA_CUDA(cudaGetLastError());
  note_launch(ctx);
  return true;
}

// 32 < n <= kTriMax: one-CTA tridiagonal eigensolver (syev_tri.cuh), descending
// lam / Z (Z may alias H); *status = 1 when the caller must fall back.
// Measured (tools/tri_check.py): n = 96 0.58-0.87 ms (random .. graded spectrum)
// vs 1.7 ms for syevj; n = 150 1.3-2.1 ms vs ~1.5 ms for syevd, so cuSOLVER
// keeps n > kTriUse.
constexpr int kTriUse = 128;
bool eig_tri_async(rnla_ctx* ctx, int64_t n, const double* H, double* lam, double* Z, int* status) {
  if (n < 3 || n > kTriUse || std::getenv("RNLA_EIG_CUSOLVER")) return false;
  DevBuf hv(sizeof(double) * n * n, ctx->stream);
  const size_t smem = tri_smem_bytes((int)n);
  ensure_dyn_smem((const void*)syev_tri_kernel, smem);
  syev_tri_kernel<<<1, kTriThreads, smem, ctx->stream>>>((int)n, H, lam, Z, hv.as<double>(), status, 1, nullptr);
  RNLA_CUDA(cudaGetLastError());
  note_launch(ctx);
  return true;
}

bool eig_sym_small_desc(rnla_ctx* ctx, int64_t b, const double* H, double* lam, double* Z) {
  if (b < 1 || b > 256) return false;
  DevBuf st(sizeof(int), ctx->stream);
  if (b > kJacobiMax && eig_tri_async(ctx, b, H, lam, Z, st.as<int>())) {
    int hs = 0;
    RNLA_CUDA(cudaMemcpyAsync(&hs, st.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
    if (hs == 0) return true;
    if (std::getenv("RNLA_TRACE")) std::fprintf(stderr, "[rnla] tridiagonal eig n=%lld: fallback\n", (long long)b);
  }
  if (eig_small_jacobi_async(ctx, b, H, lam, Z, st.as<int>())) {
    int hs = 0;
    RNLA_CUDA(cudaMemcpyAsync(&hs, st.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
    if (hs & 255) throw NumericError("eig (Jacobi): no convergence in 40 sweeps");
    if (std::getenv("RNLA_TRACE")) std::fprintf(stderr, "[rnla] jacobi n=%lld sweeps=%d\n", (long long)b, hs >> 8);
    return true;
  }
  cusolverDnHandle_t h = solver(ctx);
  syevjInfo_t params;
  if (cusolverDnCreateSyevjInfo(&params) != CUSOLVER_STATUS_SUCCESS) throw CudaError("cusolverDnCreateSyevjInfo");
  cusolverDnXsyevjSetTolerance(params, 1e-14);
  cusolverDnXsyevjSetMaxSweeps(params, 30);
  DevBuf A(sizeof(double) * b * b, ctx->stream), w(sizeof(double) * b, ctx->stream), info(sizeof(int), ctx->stream);
  RNLA_CUDA(cudaMemcpyAsync(A.p, H, sizeof(double) * b * b, cudaMemcpyDeviceToDevice, ctx->stream));
  int lwork = 0;
  if (b <= 32) {  // one-kernel batched Jacobi (n <= 32)
    cusolver_check(cusolverDnDsyevjBatched_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, (int)b,
                                                      A.as<double>(), (int)b, w.as<double>(), &lwork, params, 1),
                   "syevjBatched_bufferSize");
    DevBuf work(sizeof(double) * std::max(lwork, 1), ctx->stream);
    cusolver_check(cusolverDnDsyevjBatched(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, (int)b, A.as<double>(),
                                           (int)b, w.as<double>(), work.as<double>(), lwork, info.as<int>(), params, 1),
                   "syevjBatched");
  } else {
    cusolver_check(cusolverDnDsyevj_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, (int)b,
                                               A.as<double>(), (int)b, w.as<double>(), &lwork, params),
                   "syevj_bufferSize");
    DevBuf work(sizeof(double) * std::max(lwork, 1), ctx->stream);
    cusolver_check(cusolverDnDsyevj(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, (int)b, A.as<double>(),
                                    (int)b, w.as<double>(), work.as<double>(), lwork, info.as<int>(), params),
                   "syevj");
  }
  note_launch(ctx);
  copy2d<double>(ctx, b, b, A.as<double>() + (b - 1) * b, 1, -b, Z, 1, b);  // descending columns
  copy2d<double>(ctx, b, 1, w.as<double>() + (b - 1), -1, 1, lam, 1, b);
  RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
  cusolverDnDestroySyevjInfo(params);
  check_info(ctx, info, "eig (syevj)");
  return true;
}

}  // namespace rnla
