// gemm_dmma.cu -- fp64-accumulating DMMA GEMM for K-major operands, fed by a
// multi-stage cp.async pipeline.
//
// C[m x n] = alpha * A * B + beta * C with A(i, p) = A[i * lda + p] (K-major)
// and B(p, j) = B[j * ldb + p] (K-major) or B[p * ldb + j] (N-major: the
// config-1 Gaussian stage Omega' * S'[A, b]). K-major x K-major covers the Gram C'C of a column-major block,
// the Nystrom C'C of config 4 (src/spsd.cpp:193-215 via the Gram route), Q'A
// of a row-major A, ...). TI = double, or float widened exactly to fp64 when a
// fragment is read (products of fp32 values are exact in fp64).
//
// Tiling: 256 threads = 4 x 2 warps of 32 x 32 (4 x 4 DMMA.8x8x4 tiles each),
// CTA tile 128 x 64, k-step 16, STAGES-deep cp.async ring (16-B copies with
// zero fill at the m/n/k edges), two CTAs per SM. The generic kernel in
// gemm.cu (64 x 64 tiles, register-staged double buffer) measured ~24 TF on
// the config-1 stage and ~21 TF on the config-4 Gram.
//
// Per output element the k-sum runs in increasing k in DMMA k4 steps from a
// zero accumulator within each split, exactly like the generic kernel, so the
// two kernels agree bitwise for the same split boundaries.
#include "rnla_internal.h"
#include "util.cuh"

namespace rnla {

namespace {

constexpr int BM = 128, BN = 64, BK = 16, PAD = 4, NT = 256;
// cp.async ring depth: 3 stages of fp64 (92 KB) or 4 of fp32 (61 KB) keep two CTAs per SM.
template <class TI>
constexpr int stages() { return sizeof(TI) == 8 ? 3 : 4; }
constexpr int LDS_K = BK + PAD;  // smem row length (elements): rows stay 16-B aligned, fragment reads conflict-free

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// One stage: rows [r0, r0 + R) of a K-major operand (row stride ld), k in
// [k0, k0 + BK) clipped to [.., kend), into S[R][LDS_K].
template <class TI, int R>
__device__ __forceinline__ void load_stage(TI* S, const TI* __restrict__ G, int64_t ld, int64_t rows, int64_t r0,
                                           int64_t k0, int64_t kend, int tid) {
  constexpr int EPC = 16 / sizeof(TI);  // elements per 16-B copy
  constexpr int CPR = BK / EPC;         // copies per row
  constexpr int TOTAL = R * CPR;
#pragma unroll
  for (int c = tid; c < TOTAL; c += NT) {
    const int r = c / CPR, kc = (c % CPR) * EPC;
    const int64_t gr = r0 + r, gk = k0 + kc;
    int bytes = 0;
    const TI* src = G;
    if (gr < rows && gk < kend) {
      bytes = (int)((kend - gk < EPC ? kend - gk : (int64_t)EPC) * (int64_t)sizeof(TI));
      src = G + gr * ld + gk;
    }
    cp_async16(S + r * LDS_K + kc, src, bytes);
  }
}

// One stage of an N-major operand B(p, j) = G[p * ld + j]: k rows [k0, k0 + BK)
// clipped to kend, columns [n0, n0 + BN) clipped to ncols, into S[BK][LDS_N].
// Row length of an N-major stage (elements): k rows stay 16-B aligned and the
// four k rows of a fragment read land in distinct banks (fp64: 68, fp32: 72).
template <class TI>
constexpr int lds_n() { return sizeof(TI) == 8 ? BN + 4 : BN + 8; }
template <class TI>
__device__ __forceinline__ void load_stage_kn(TI* S, const TI* __restrict__ G, int64_t ld, int64_t ncols, int64_t n0,
                                              int64_t k0, int64_t kend, int tid) {
  constexpr int EPC = 16 / sizeof(TI);
  constexpr int CPR = BN / EPC;
  constexpr int TOTAL = BK * CPR;
  constexpr int LDS_N = lds_n<TI>();
#pragma unroll
  for (int c = tid; c < TOTAL; c += NT) {
    const int kr = c / CPR, nc = (c % CPR) * EPC;
    const int64_t gk = k0 + kr, gj = n0 + nc;
    int bytes = 0;
    const TI* src = G;
    if (gk < kend && gj < ncols) {
      bytes = (int)((ncols - gj < EPC ? ncols - gj : (int64_t)EPC) * (int64_t)sizeof(TI));
      src = G + gk * ld + gj;
    }
    cp_async16(S + kr * LDS_N + nc, src, bytes);
  }
}

template <class TI, bool B_KM>
__global__ void __launch_bounds__(NT, 2) gemm_dmma_kk(int64_t m, int64_t n, int64_t kdim, int64_t kchunk, double alpha,
                                                     const TI* __restrict__ A, int64_t lda, const TI* __restrict__ B,
                                                     int64_t ldb, double beta, double* C, int64_t c_rs, int64_t c_cs,
                                                     double* ws, int sym_upper) {
  constexpr int MI = 4, NI = 4, STAGES = stages<TI>();
  const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;
  // sym_upper bit 0 (symmetric C): skip tiles strictly below the diagonal; the
  // caller mirrors the lower 64 x 64 tiles afterwards. Bit 1: B upper triangular
  // (k < n0 + BN only); bit 2: A lower triangular (k < m0 + BM only).
  if ((sym_upper & 1) && n0 + BN <= m0) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  TI* As = reinterpret_cast<TI*>(smem_raw);     // [STAGES][BM][LDS_K]
  TI* Bs = As + (size_t)STAGES * BM * LDS_K;    // [STAGES][BN][LDS_K] (K-major B) or [STAGES][BK][LDS_N]
  constexpr int LDS_N = lds_n<TI>();
  constexpr int BSTAGE = B_KM ? BN * LDS_K : BK * LDS_N;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 1, wn = warp & 1;
  const int g = lane >> 2, t = lane & 3;
  const int64_t kbeg = (int64_t)blockIdx.z * kchunk;
  int64_t kend = min(kdim, kbeg + kchunk);
  if (sym_upper & 2) kend = min(kend, n0 + BN);
  if (sym_upper & 4) kend = min(kend, m0 + BM);
  const int nsteps = kend > kbeg ? (int)((kend - kbeg + BK - 1) / BK) : 0;

  double acc[MI][NI][2];
#pragma unroll
  for (int a = 0; a < MI; ++a)
#pragma unroll
    for (int b = 0; b < NI; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nsteps) {
      load_stage<TI, BM>(As + (size_t)s * BM * LDS_K, A, lda, m, m0, kbeg + (int64_t)s * BK, kend, tid);
      if constexpr (B_KM) load_stage<TI, BN>(Bs + (size_t)s * BSTAGE, B, ldb, n, n0, kbeg + (int64_t)s * BK, kend, tid);
      else load_stage_kn<TI>(Bs + (size_t)s * BSTAGE, B, ldb, n, n0, kbeg + (int64_t)s * BK, kend, tid);
    }
    cp_commit();
  }
  for (int it = 0; it < nsteps; ++it) {
    cp_wait<STAGES - 2>();
    __syncthreads();  // stage `it` landed for everyone; stage it-1 fully read
    const int nx = it + STAGES - 1;
    if (nx < nsteps) {
      const int sl = nx % STAGES;
      load_stage<TI, BM>(As + (size_t)sl * BM * LDS_K, A, lda, m, m0, kbeg + (int64_t)nx * BK, kend, tid);
      if constexpr (B_KM) load_stage<TI, BN>(Bs + (size_t)sl * BSTAGE, B, ldb, n, n0, kbeg + (int64_t)nx * BK, kend, tid);
      else load_stage_kn<TI>(Bs + (size_t)sl * BSTAGE, B, ldb, n, n0, kbeg + (int64_t)nx * BK, kend, tid);
    }
    cp_commit();
    const TI* as = As + (size_t)(it % STAGES) * BM * LDS_K + (wm * 32 + g) * LDS_K + t;
    const TI* bs = B_KM ? Bs + (size_t)(it % STAGES) * BSTAGE + (wn * 32 + g) * LDS_K + t
                        : Bs + (size_t)(it % STAGES) * BSTAGE + t * LDS_N + wn * 32 + g;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[MI], bf[NI];
#pragma unroll
      for (int mi = 0; mi < MI; ++mi) af[mi] = (double)as[mi * 8 * LDS_K + kk];
#pragma unroll
      for (int ni = 0; ni < NI; ++ni) bf[ni] = (double)(B_KM ? bs[ni * 8 * LDS_K + kk] : bs[kk * LDS_N + ni * 8]);
#pragma unroll
      for (int mi = 0; mi < MI; ++mi)
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni]);
    }
  }
  cp_wait<0>();

#pragma unroll
  for (int mi = 0; mi < MI; ++mi)
#pragma unroll
    for (int ni = 0; ni < NI; ++ni)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t i = m0 + wm * 32 + mi * 8 + g;
        const int64_t j = n0 + wn * 32 + ni * 8 + 2 * t + h;
        if (i < m && j < n) {
          if (ws) {
            ws[(int64_t)blockIdx.z * m * n + i * n + j] = acc[mi][ni][h];
          } else {
            double* cp = C + i * c_rs + j * c_cs;
            *cp = beta == 0.0 ? alpha * acc[mi][ni][h] : alpha * acc[mi][ni][h] + beta * *cp;
          }
        }
      }
}

template <class TI, bool B_KM>
constexpr size_t smem_bytes() {
  return (size_t)stages<TI>() * (BM * LDS_K + (B_KM ? BN * LDS_K : BK * lds_n<TI>())) * sizeof(TI);
}

}  // namespace

// 1: K-major B, 2: N-major B, 0: not applicable (A must be K-major; 16-B aligned rows).
template <class TI>
int dmma_kk_applicable(const TI* A, int64_t a_rs, int64_t a_cs, const TI* B, int64_t b_rs, int64_t b_cs) {
  if (std::getenv("RNLA_DMMA_GENERIC")) return 0;
  const auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (a_cs != 1 || !al(A) || !al(B) || (a_rs * (int64_t)sizeof(TI)) % 16 != 0) return 0;
  if (b_rs == 1 && (b_cs * (int64_t)sizeof(TI)) % 16 == 0) return 1;
  if (b_cs == 1 && (b_rs * (int64_t)sizeof(TI)) % 16 == 0) return 2;
  return 0;
}

template <class TI>
void dmma_kk_launch(rnla_ctx* ctx, int layout, int64_t m, int64_t n, int64_t k, int64_t kchunk, int64_t splits,
                    double alpha, const TI* A, int64_t lda, const TI* B, int64_t ldb, double beta, double* C,
                    int64_t c_rs, int64_t c_cs, double* ws, int sym) {
  dim3 grid((unsigned)((n + BN - 1) / BN), (unsigned)((m + BM - 1) / BM), (unsigned)splits);
  if (layout == 1) {
    constexpr size_t smem = smem_bytes<TI, true>();
    ensure_dyn_smem((const void*)gemm_dmma_kk<TI, true>, smem);
    gemm_dmma_kk<TI, true><<<grid, NT, smem, ctx->stream>>>(m, n, k, kchunk, alpha, A, lda, B, ldb, beta, C, c_rs,
                                                            c_cs, ws, sym);
  } else {
    constexpr size_t smem = smem_bytes<TI, false>();
    ensure_dyn_smem((const void*)gemm_dmma_kk<TI, false>, smem);
    gemm_dmma_kk<TI, false><<<grid, NT, smem, ctx->stream>>>(m, n, k, kchunk, alpha, A, lda, B, ldb, beta, C, c_rs,
                                                             c_cs, ws, sym);
  }
  RNLA_CUDA(cudaGetLastError());
  note_launch(ctx);
}

int dmma_kk_tiles(int64_t m, int64_t n, int sym) {
  const int64_t tm = (m + BM - 1) / BM, tn = (n + BN - 1) / BN;
  if (!(sym & 1)) return (int)(tm * tn);
  int64_t live = 0;
  for (int64_t a = 0; a < tm; ++a)
    for (int64_t b = 0; b < tn; ++b)
      if (b * BN + BN > a * BM) ++live;
  return (int)live;
}

int dmma_kk_per_sm() { return 2; }

template int dmma_kk_applicable<double>(const double*, int64_t, int64_t, const double*, int64_t, int64_t);
template int dmma_kk_applicable<float>(const float*, int64_t, int64_t, const float*, int64_t, int64_t);
template void dmma_kk_launch<double>(rnla_ctx*, int, int64_t, int64_t, int64_t, int64_t, int64_t, double,
                                     const double*, int64_t, const double*, int64_t, double, double*, int64_t, int64_t,
                                     double*, int);
template void dmma_kk_launch<float>(rnla_ctx*, int, int64_t, int64_t, int64_t, int64_t, int64_t, double, const float*,
                                    int64_t, const float*, int64_t, double, double*, int64_t, int64_t, double*, int);

}  // namespace rnla
