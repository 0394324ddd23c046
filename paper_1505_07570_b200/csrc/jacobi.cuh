// jacobi.cuh -- one-CTA parallel two-sided Jacobi eigensolver for small
// symmetric fp64 matrices (see linalg.cu: eig_sym_small_desc). Device code
// only, so tools/jacobi_bench.cu can time it standalone.
//
// A and V stay in shared memory. Round r of a sweep rotates the m/2 disjoint
// pairs (p, q) of a round-robin tournament on m = n rounded up to even
// indices (a pair with the dummy index n is skipped). Warp w owns pairs
// w, w + NW, ... (at most PPW per warp) in both phases of the round:
//   phase 1: read a_pp, a_qq, a_pq (columns p, q belong to this warp alone in
//     this phase), form the rotation J, apply A <- A J and V <- V J to columns
//     p, q; barrier;
//   phase 2: A <- J'A on rows p, q with a_pq = a_qp = 0; barrier.
// The rotation stays in the warp's registers between the phases. The round's
// critical path is the rotation: t = tan(phi) is seeded in fp32 on values
// scaled by a power of two, refined by one fp64 Newton step, and
// c = 1 / sqrt(1 + t^2) by an fp32 seed and two fp64 Newton steps -- no fp64
// division or square root. A pair is rotated when a_pq^2 > 1e-30 |a_pp a_qq|
// (relative criterion; small eigenvalues of an SPD matrix keep their relative
// accuracy); the sweep loop ends after a sweep without rotations.
#pragma once
#include <cstdint>

#ifndef RNLA_JACOBI_PROF
#define RNLA_JACOBI_PROF 0
#endif


namespace rnla {
namespace {

// 2^-e(x) with e(x) the binary exponent of x > 0 (x * 2^-e in [1, 2))
__device__ __forceinline__ double jacobi_pow2_inv(double x) {
  const long long bits = __double_as_longlong(x);
  int e = (int)((bits >> 52) & 0x7ff);
  e = e < 1 ? 1 : (e > 2045 ? 2045 : e);
  return __longlong_as_double((long long)(2046 - e) << 52);  // exponent field 2046 - e: 2^(1023 - e)
}

// Rotation (c, s) annihilating a_pq of the 2 x 2 block [app apq; apq aqq].
__device__ __forceinline__ void jacobi_rotation(double app, double aqq, double apq, double& c, double& s) {
  const double d = aqq - app, e = 2.0 * apq;
  const double sc = jacobi_pow2_inv(fmax(fabs(d), fabs(e)));
  const float df = (float)(d * sc), ef = (float)(e * sc);
  // t = sgn(d) e / (|d| + hypot(d, e)), the smaller root of e t^2 + 2 d t - e = 0
  const float h2 = fmaf(df, df, ef * ef);
  float tf = __fdividef(ef, fabsf(df) + h2 * rsqrtf(h2));
  if (df < 0.f) tf = -tf;
  double t = tf;
  const double g = fma(fma(e, t, 2.0 * d), t, -e) * sc, gp = 2.0 * fma(e, t, d) * sc;
  t -= g * (double)__frcp_rn((float)gp);
  const double u = fma(t, t, 1.0);
  c = (double)rsqrtf((float)u);
  c *= fma(-0.5 * u, c * c, 1.5);
  c *= fma(-0.5 * u, c * c, 1.5);
  s = t * c;
}

template <int NT>
__global__ void __launch_bounds__(NT) jacobi_eig_kernel(int n, const double* __restrict__ H, double* __restrict__ lam,
                                                        double* __restrict__ Z, int* __restrict__ status,
                                                        long long* prof = nullptr) {
  constexpr int NW = NT / 32;
  constexpr int PPW = 2;  // pairs per warp: n <= 2 * 2 * NW
  extern __shared__ double jsm[];
  const int ld = n + 1;
  const int m = n + (n & 1), np = m / 2, nr = m > 1 ? m - 1 : 0;
  double* A = jsm;                                            // [n][n + 1], A[i * ld + j] = a_ij
  double* V = jsm + (size_t)n * ld;                           // [n][n + 1], column j = eigenvector j
  uint8_t* P = reinterpret_cast<uint8_t*>(V + (size_t)n * ld);  // [nr][np] pair tables
  uint8_t* Q = P + nr * np;
  __shared__ int rotated[2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#if RNLA_JACOBI_PROF
  long long pt[5] = {0, 0, 0, 0, 0}, c0 = 0, c1;
#endif
  for (int e = tid; e < n * n; e += NT) {
    const int i = e % n, j = e / n;  // column-major H, lower triangle
    A[i * ld + j] = i >= j ? H[i + (int64_t)j * n] : H[j + (int64_t)i * n];
    V[i * ld + j] = i == j ? 1.0 : 0.0;
  }
  for (int e = tid; e < nr * np; e += NT) {
    const int r = e / np, pi = e % np;
    int p = pi == 0 ? m - 1 : (r + pi) % (m - 1);
    int q = pi == 0 ? r : (r - pi + (m - 1)) % (m - 1);
    P[e] = (uint8_t)min(p, q);
    Q[e] = (uint8_t)max(p, q);
  }
  if (tid < 2) rotated[tid] = 0;
  __shared__ double amax_s;
  if (tid == 0) {
    double mx = 0.0;
    for (int i = 0; i < n; ++i) mx = fmax(mx, fabs(A[i * ld + i]));
    amax_s = mx;
  }
  __syncthreads();
  // absolute floor: entries below 1e-17 max|a_ii| are left alone (eigenvalues
  // then carry ~1e-17 ||A|| absolute error, far below what the callers need:
  // sigma_k >= 1e-3 sigma_1 in topk_svd_wide, Ritz values relative to theta_1)
  const double afloor = 1e-17 * amax_s;
  int sweep = 0, conv = m <= 1;
  for (; sweep < 40 && !conv; ++sweep) {
    const int flag = sweep & 1;
    // A sweep that starts with no pair above the rotation threshold rotates
    // nothing (the matrix never changes), so it is recognized up front instead
    // of being walked through round by round; same result, same sweep count.
    {
      int need = 0;
      for (int e = tid; e < n * n; e += NT) {
        const int p = e / n, q = e - p * n;
        if (p != q) {  // both triangles: the rounds read A(p, q) in the tournament's order
          const double apq = A[p * ld + q];
          need |= fabs(apq) > afloor && apq * apq > 1e-30 * fabs(A[p * ld + p] * A[q * ld + q]);
        }
      }
      if (!__syncthreads_or(need)) {
        conv = 1;
        break;
      }
    }
    for (int r = 0; r < nr; ++r) {
#if RNLA_JACOBI_PROF
      c0 = clock64();
#endif
      double cs[PPW], sn[PPW];
      int pp[PPW], qq[PPW];
#pragma unroll
      for (int j = 0; j < PPW; ++j) {
        const int pi = warp + j * NW;
        cs[j] = 0.0;
        sn[j] = 0.0;
        pp[j] = 0;
        qq[j] = n;
        if (pi < np) {
          pp[j] = P[r * np + pi];
          qq[j] = Q[r * np + pi];
        }
        const int p = pp[j], q = qq[j];
        if (q < n) {
          const double app = A[p * ld + p], aqq = A[q * ld + q], apq = A[p * ld + q];
          if (fabs(apq) > afloor && apq * apq > 1e-30 * fabs(app * aqq)) jacobi_rotation(app, aqq, apq, cs[j], sn[j]);
        }
      }
      __syncwarp();
#if RNLA_JACOBI_PROF
      c1 = clock64(); pt[4] += c1 - c0; c0 = c1;
#endif
#pragma unroll
      for (int j = 0; j < PPW; ++j) {
        const double c = cs[j], s = sn[j];
        if (c == 0.0) continue;
        const int p = pp[j], q = qq[j];
        for (int l = lane; l < n; l += 32) {
          const double x = A[l * ld + p], y = A[l * ld + q];
          A[l * ld + p] = c * x - s * y;
          A[l * ld + q] = s * x + c * y;
          const double vx = V[l * ld + p], vy = V[l * ld + q];
          V[l * ld + p] = c * vx - s * vy;
          V[l * ld + q] = s * vx + c * vy;
        }
        if (lane == 0) rotated[flag] = 1;
      }
#if RNLA_JACOBI_PROF
      c1 = clock64(); pt[0] += c1 - c0; c0 = c1;
#endif
      __syncthreads();
#if RNLA_JACOBI_PROF
      c1 = clock64(); pt[1] += c1 - c0; c0 = c1;
#endif
#pragma unroll
      for (int j = 0; j < PPW; ++j) {
        const double c = cs[j], s = sn[j];
        if (c == 0.0) continue;
        const int p = pp[j], q = qq[j];
        for (int l = lane; l < n; l += 32) {
          const double x = A[p * ld + l], y = A[q * ld + l];
          A[p * ld + l] = l == q ? 0.0 : c * x - s * y;
          A[q * ld + l] = l == p ? 0.0 : s * x + c * y;
        }
      }
#if RNLA_JACOBI_PROF
      c1 = clock64(); pt[2] += c1 - c0; c0 = c1;
#endif
      __syncthreads();
#if RNLA_JACOBI_PROF
      c1 = clock64(); pt[3] += c1 - c0;
#endif
    }
    if (!rotated[flag]) {
      conv = 1;
      break;
    }
    if (tid == 0) rotated[flag ^ 1] = 0;
    __syncthreads();
  }
  // descending order: rank of each eigenvalue (ties by index)
  for (int i = tid; i < n; i += NT) {
    const double li = A[i * ld + i];
    int rank = 0;
    for (int j = 0; j < n; ++j) {
      const double lj = A[j * ld + j];
      rank += (lj > li || (lj == li && j < i)) ? 1 : 0;
    }
    lam[rank] = li;
    for (int l = 0; l < n; ++l) Z[l + (int64_t)rank * n] = V[l * ld + i];
  }
  if (tid == 0 && status) *status = conv ? (sweep + 1) << 8 : 1;  // bits 8+: sweeps taken
#if RNLA_JACOBI_PROF
  if (tid == 0 && prof)
    for (int i = 0; i < 5; ++i) prof[i] = pt[i];
#else
  (void)prof;
#endif
}

// dynamic shared memory of jacobi_eig_kernel for n
inline size_t jacobi_smem_bytes(int n) {
  const int m = n + (n & 1);
  return sizeof(double) * 2 * (size_t)n * (n + 1) + 2 * (size_t)(m > 1 ? m - 1 : 0) * (m / 2);
}

}  // namespace
}  // namespace rnla
