// gemm_skinny.cu -- fp64 DMMA GEMM for narrow outputs (n <= 32): the passes
// of the config-0 randomized SVD, Y = A Omega, Z = A'Q, Y = A Z and B' = A'Q
// with s = 30 (src/randsvd.cpp:94-99 plus the power iterations of SURVEY A.6).
//
// Each element of A is used n <= 32 times, so a pass is DMMA-bound
// (7.5 flop/B against a ~5.7 flop/B ridge at 37 TF fp64): the kernel streams
// A once through a cp.async ring with the whole 32-wide B strip of the stage
// next to it. A may be K-major (row-major A in A Omega) or M-major (A' of a
// row-major A in A'Q) -- both land in shared memory exactly as they lie in
// global memory (16-B cp.async copies, zero fill at the edges) and the DMMA
// fragments are read from either layout without a transpose. B is K-major
// (a column-major K x n strip).
//
// CTA tile 128 x 32, 8 warps of 32 x 16 (4 x 2 DMMA.8x8x4 tiles), k-step 16,
// 4-stage ring (~100 KB, two CTAs per SM). Split-K partials go to a workspace
// reduced in a fixed order, so results are run-to-run deterministic; within a
// split every output element sums k in increasing order.
#include "rnla_internal.h"
#include "util.cuh"

namespace rnla {

namespace {

constexpr int SBM = 128, SBN = 32, SBK = 16, SNT = 256;
constexpr int LDK = SBK + 4;   // K-major rows (doubles): fragment reads conflict-free
constexpr int LDM = SBM + 4;   // M-major k rows (doubles): 132 = 4 mod 16, conflict-free
constexpr int A_STAGE_KM = SBM * LDK, A_STAGE_MM = SBK * LDM, B_STAGE = SBN * LDK;

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp16(void* smem, const void* gmem, int bytes) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(bytes) : "memory");
}

template <bool A_KM>
__device__ __forceinline__ void load_stage(double* As, double* Bs, const double* __restrict__ A, int64_t lda,
                                           const double* __restrict__ B, int64_t ldb, int64_t m, int64_t n, int64_t m0,
                                           int64_t k0, int64_t kend, int tid) {
  if (A_KM) {  // A(i, p) = A[i * lda + p]: 128 rows x 8 copies of 2 doubles
#pragma unroll
    for (int c = tid; c < SBM * (SBK / 2); c += SNT) {
      const int r = c >> 3, kc = (c & 7) * 2;
      const int64_t gi = m0 + r, gk = k0 + kc;
      int bytes = 0;
      const double* src = A;
      if (gi < m && gk < kend) {
        bytes = kend - gk >= 2 ? 16 : 8;
        src = A + gi * lda + gk;
      }
      cp16(As + r * LDK + kc, src, bytes);
    }
  } else {  // A(i, p) = A[p * lda + i]: 16 k rows x 64 copies
#pragma unroll
    for (int c = tid; c < SBK * (SBM / 2); c += SNT) {
      const int kr = c >> 6, ic = (c & 63) * 2;
      const int64_t gi = m0 + ic, gk = k0 + kr;
      int bytes = 0;
      const double* src = A;
      if (gk < kend && gi < m) {
        bytes = m - gi >= 2 ? 16 : 8;
        src = A + gk * lda + gi;
      }
      cp16(As + kr * LDM + ic, src, bytes);
    }
  }
  // B(p, j) = B[j * ldb + p]: 32 columns x 8 copies
  {
    const int c = tid;  // SBN * SBK / 2 == SNT
    const int j = c >> 3, kc = (c & 7) * 2;
    const int64_t gk = k0 + kc;
    int bytes = 0;
    const double* src = B;
    if (j < n && gk < kend) {
      bytes = kend - gk >= 2 ? 16 : 8;
      src = B + (int64_t)j * ldb + gk;
    }
    cp16(Bs + j * LDK + kc, src, bytes);
  }
}

// grid (ceil(m / 128), 1, splits). ws: [splits][m][n] partials (or C directly
// when splits == 1: C(i, j) = alpha acc + beta C(i, j)).
template <bool A_KM, int SSTAGES, int MINB>
__global__ void __launch_bounds__(SNT, MINB) gemm_skinny_dmma(int64_t m, int64_t n, int64_t kdim, int64_t kchunk,
                                                          const double* __restrict__ A, int64_t lda,
                                                          const double* __restrict__ B, int64_t ldb, double alpha,
                                                          double beta, double* C, int64_t c_rs, int64_t c_cs,
                                                          double* ws) {
  constexpr int A_STAGE = A_KM ? A_STAGE_KM : A_STAGE_MM;
  extern __shared__ __align__(16) double ssm[];
  double* As = ssm;                              // [SSTAGES][A_STAGE]
  double* Bs = ssm + (size_t)SSTAGES * A_STAGE;  // [SSTAGES][B_STAGE]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 1, wn = warp & 1;  // 4 x 2 warps of 32 x 16
  const int g = lane >> 2, t = lane & 3;
  const int64_t m0 = (int64_t)blockIdx.x * SBM;
  const int64_t kbeg = (int64_t)blockIdx.z * kchunk;
  const int64_t kend = min(kdim, kbeg + kchunk);
  const int nsteps = kend > kbeg ? (int)((kend - kbeg + SBK - 1) / SBK) : 0;

  double acc[4][2][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

#pragma unroll
  for (int s = 0; s < SSTAGES - 1; ++s) {
    if (s < nsteps)
      load_stage<A_KM>(As + (size_t)s * A_STAGE, Bs + (size_t)s * B_STAGE, A, lda, B, ldb, m, n, m0,
                       kbeg + (int64_t)s * SBK, kend, tid);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  }
  for (int it = 0; it < nsteps; ++it) {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(SSTAGES - 2) : "memory");
    __syncthreads();
    const int nx = it + SSTAGES - 1;
    if (nx < nsteps)
      load_stage<A_KM>(As + (size_t)(nx % SSTAGES) * A_STAGE, Bs + (size_t)(nx % SSTAGES) * B_STAGE, A, lda, B, ldb, m,
                       n, m0, kbeg + (int64_t)nx * SBK, kend, tid);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    const double* as = As + (size_t)(it % SSTAGES) * A_STAGE;
    const double* bs = Bs + (size_t)(it % SSTAGES) * B_STAGE + (wn * 16 + g) * LDK + t;
#pragma unroll
    for (int kk = 0; kk < SBK; kk += 4) {
      double af[4], bf[2];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) {
        const int r = wm * 32 + mi * 8 + g;
        af[mi] = A_KM ? as[r * LDK + kk + t] : as[(kk + t) * LDM + r];
      }
#pragma unroll
      for (int ni = 0; ni < 2; ++ni) bf[ni] = bs[ni * 8 * LDK + kk];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 2; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni]);
    }
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");

#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 2; ++ni)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t i = m0 + wm * 32 + mi * 8 + g;
        const int64_t j = wn * 16 + ni * 8 + 2 * t + h;
        if (i < m && j < n) {
          if (ws) {
            ws[((int64_t)blockIdx.z * m + i) * n + j] = acc[mi][ni][h];
          } else {
            double* cp = C + i * c_rs + j * c_cs;
            *cp = beta == 0.0 ? alpha * acc[mi][ni][h] : alpha * acc[mi][ni][h] + beta * *cp;
          }
        }
      }
}

// many splits (the s x s Grams: K = 8192 rows in 64 splits): one warp per
// element, lanes take splits z = lane, lane + 32, ... and a fixed xor tree adds them
__global__ void skinny_reduce_warp(int64_t m, int64_t n, int splits, const double* __restrict__ ws, double alpha,
                                   double beta, double* C, int64_t c_rs, int64_t c_cs) {
  const int64_t total = m * n;
  const int lane = threadIdx.x & 31;
  for (int64_t e = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; e < total;
       e += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    double sum = 0.0;
    for (int z = lane; z < splits; z += 32) sum += ws[(int64_t)z * total + e];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (lane == 0) {
      const int64_t i = e / n, j = e % n;
      double* cp = C + i * c_rs + j * c_cs;
      *cp = beta == 0.0 ? alpha * sum : alpha * sum + beta * *cp;
    }
  }
}

__global__ void skinny_reduce(int64_t m, int64_t n, int splits, const double* __restrict__ ws, double alpha,
                              double beta, double* C, int64_t c_rs, int64_t c_cs) {
  const int64_t total = m * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    double sum = ws[e];
    for (int z = 1; z < splits; ++z) sum += ws[(int64_t)z * total + e];
    const int64_t i = e / n, j = e % n;
    double* cp = C + i * c_rs + j * c_cs;
    *cp = beta == 0.0 ? alpha * sum : alpha * sum + beta * *cp;
  }
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace

// C[m x n] = alpha A B + beta C for n <= 32 (see the file comment). Returns
// false when the layout does not fit (the caller uses the generic kernels).
bool gemm_skinny_f64(rnla_ctx* ctx, int64_t m, int64_t n, int64_t k, double alpha, const double* A, int64_t a_rs,
                     int64_t a_cs, const double* B, int64_t b_rs, int64_t b_cs, double beta, double* C, int64_t c_rs,
                     int64_t c_cs, int max_splits) {
  if (n < 1 || n > SBN || m < 1 || k < 1 || std::getenv("RNLA_DMMA_GENERIC")) return false;
  if (!aligned16(A) || !aligned16(B) || b_rs != 1 || (b_cs % 2) != 0 || b_cs < k) return false;
  bool a_km;
  if (a_cs == 1 && (a_rs % 2) == 0 && a_rs >= k) a_km = true;
  else if (a_rs == 1 && (a_cs % 2) == 0 && a_cs >= m) a_km = false;
  else return false;
  const int64_t tiles = (m + SBM - 1) / SBM;
  // as many K splits as keep every CTA in the first wave (two per SM), >= 8
  // k-steps each. (Wave-filling split counts -- 9 / 17 splits for the
  // config-0 passes -- measured no faster per pass and cost more reduction.)
  const int64_t slots = 2 * (int64_t)ctx->num_sms;
  int64_t splits = std::max<int64_t>(1, std::min<int64_t>(slots / tiles, k / (8 * SBK)));
  splits = std::min<int64_t>(splits, std::max(1, max_splits));
  int64_t kchunk = ((k + splits - 1) / splits + SBK - 1) / SBK * SBK;
  splits = std::max<int64_t>(1, (k + kchunk - 1) / kchunk);
  DevBuf ws;
  if (splits > 1) ws = DevBuf(sizeof(double) * (size_t)(splits * m * n), ctx->stream);
  constexpr int stages = 4;
  const size_t smem = sizeof(double) * (size_t)stages * ((a_km ? A_STAGE_KM : A_STAGE_MM) + B_STAGE);
  dim3 grid((unsigned)tiles, 1, (unsigned)splits);
  const int64_t lda = a_km ? a_rs : a_cs;
  double* wsp = splits > 1 ? ws.as<double>() : nullptr;
#define RNLA_SKINNY_LAUNCH(KM, ST, MB)                                                                              \
  do {                                                                                                              \
    ensure_dyn_smem((const void*)gemm_skinny_dmma<KM, ST, MB>, smem);                                                \
    gemm_skinny_dmma<KM, ST, MB><<<grid, SNT, smem, ctx->stream>>>(m, n, k, kchunk, A, lda, B, b_cs, alpha, beta, C, \
                                                                   c_rs, c_cs, wsp);                                \
  } while (0)
  if (a_km) RNLA_SKINNY_LAUNCH(true, 4, 2);
  else RNLA_SKINNY_LAUNCH(false, 4, 2);
#undef RNLA_SKINNY_LAUNCH
  RNLA_CUDA(cudaGetLastError());
  note_launch(ctx);
  if (splits > 1) {
    if (splits >= 8 && m * n <= 16384) {
      const int blocks = (int)std::min<int64_t>((m * n * 32 + 255) / 256, (int64_t)ctx->num_sms * 16);
      skinny_reduce_warp<<<blocks, 256, 0, ctx->stream>>>(m, n, (int)splits, wsp, alpha, beta, C, c_rs, c_cs);
    } else {
      const int blocks = (int)std::min<int64_t>((m * n + 255) / 256, (int64_t)ctx->num_sms * 8);
      skinny_reduce<<<blocks, 256, 0, ctx->stream>>>(m, n, (int)splits, wsp, alpha, beta, C, c_rs, c_cs);
    }
    RNLA_CUDA(cudaGetLastError());
    note_launch(ctx);
  }
  return true;
}

}  // namespace rnla
