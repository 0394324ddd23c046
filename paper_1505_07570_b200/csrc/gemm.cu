// gemm.cu -- strided GEMMs for the sketch projections.
//
//  fp64: DMMA tensor-core path (mma.sync.m8n8k4.f64 lowers to DMMA.8x8x4 on
//        sm_100a; tcgen05 has no f64 kind). Reference GEMM sites:
//        gaussian_sketch A*(G/sqrt(s)) src/sketch.cpp:41, Q'*A
//        src/randsvd.cpp:99, L = C*U*Lambda^-1/2 src/spsd.cpp:215.
//  fp32: tiled SIMT FFMA path (exact fp32 products/sums; the tcgen05 BF16x3
//        path of DESIGN.md §3.3 replaces it for the large fp32 configs).
//
// C[m x n] = alpha * A[m x k] * B[k x n] + beta * C, with element (i, j) of X
// at X[i*rs + j*cs]. Split-K writes per-split partials to a workspace and a
// fixed-order reduction finishes them, so results are run-to-run
// deterministic (the reference's determinism tests compare bitwise,
// tests/test_sketch.cpp:170-182).
#include "rnla_internal.h"
#include "util.cuh"

namespace rnla {

namespace {

constexpr int BM = 64, BN = 64, BK = 16, PAD = 4, THREADS = 128;

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <class T, class TS = T>
struct TileLoader {
  // 1024 elements per BM x BK (or BK x BN) tile, 8 per thread; stored to smem as TS.
  T regs[8];
  __device__ __forceinline__ void load_a(const T* A, int64_t rs, int64_t cs, int64_t m, int64_t kdim, int64_t m0,
                                         int64_t k0, int tid) {
    const bool mcontig = (rs == 1 && cs != 1);
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const int idx = tid + THREADS * r;
      const int i = mcontig ? idx % BM : idx / BK;
      const int p = mcontig ? idx / BM : idx % BK;
      const int64_t gi = m0 + i, gp = k0 + p;
      regs[r] = (gi < m && gp < kdim) ? A[gi * rs + gp * cs] : T(0);
    }
  }
  __device__ __forceinline__ void store_a(TS (*As)[BK + PAD], int64_t rs, int64_t cs, int tid) {
    const bool mcontig = (rs == 1 && cs != 1);
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const int idx = tid + THREADS * r;
      const int i = mcontig ? idx % BM : idx / BK;
      const int p = mcontig ? idx / BM : idx % BK;
      As[i][p] = (TS)regs[r];
    }
  }
  // B element (p, j) at B[p*rs + j*cs]; smem holds Bs[j][p]. NB = tile width (64 or 32).
  template <int NB = BN>
  __device__ __forceinline__ void load_b(const T* B, int64_t rs, int64_t cs, int64_t kdim, int64_t n, int64_t k0,
                                         int64_t n0, int tid) {
    const bool kcontig = (rs == 1 && cs != 1);
#pragma unroll
    for (int r = 0; r < NB * BK / THREADS; ++r) {
      const int idx = tid + THREADS * r;
      const int j = kcontig ? idx / BK : idx % NB;
      const int p = kcontig ? idx % BK : idx / NB;
      const int64_t gj = n0 + j, gp = k0 + p;
      regs[r] = (gj < n && gp < kdim) ? B[gp * rs + gj * cs] : T(0);
    }
  }
  template <int NB = BN>
  __device__ __forceinline__ void store_b(TS (*Bs)[BK + PAD], int64_t rs, int64_t cs, int tid) {
    const bool kcontig = (rs == 1 && cs != 1);
#pragma unroll
    for (int r = 0; r < NB * BK / THREADS; ++r) {
      const int idx = tid + THREADS * r;
      const int j = kcontig ? idx / BK : idx % NB;
      const int p = kcontig ? idx % BK : idx / NB;
      Bs[j][p] = (TS)regs[r];
    }
  }
};

// grid: (ceil(n/BN), ceil(m/BM), splits). Writes alpha*acc + beta*C when
// ws == nullptr, else the raw partial to ws[z*m*n + i*n + j]. TI = input
// element type (float inputs are widened exactly to fp64 on the way to smem).
// NB = 64: 2 x 2 warps of 32 x 32; NB = 32 (narrow outputs such as the
// s = 30 sketches of config 0): 4 x 1 warps of 16 x 32, so no half-empty tiles.
// MINB = resident CTAs per SM the register allocation must allow: 3 for the
// fp64-input 64-wide tile (244 -> 168 registers, no spills), 4 for the
// fp32-input Gram tile, which then covers a 2048^2 symmetric Gram (528 tiles)
// in one wave of 592 slots instead of two of 444.
#ifndef RNLA_DMMA_F32_MINB
#define RNLA_DMMA_F32_MINB 4
#endif
template <class TI, int NB = BN, int MINB = 1>
__global__ void __launch_bounds__(THREADS, MINB) gemm_f64_dmma(int64_t m, int64_t n, int64_t kdim, int64_t kchunk,
                                                         double alpha, const TI* __restrict__ A, int64_t a_rs,
                                                         int64_t a_cs, const TI* __restrict__ B, int64_t b_rs,
                                                         int64_t b_cs, double beta, double* C, int64_t c_rs,
                                                         int64_t c_cs, double* ws, int sym_upper) {
  constexpr int WN = NB == 64 ? 2 : 1, MI = NB == 64 ? 4 : 2, NI = 4;
  // sym_upper: C is symmetric (A = B'); tiles strictly below the diagonal are
  // skipped and mirrored afterwards (half the Gram flops).
  if (sym_upper && blockIdx.y > blockIdx.x) return;
  __shared__ __align__(16) double As[2][BM][BK + PAD];
  __shared__ __align__(16) double Bs[2][NB][BK + PAD];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / WN, wn = warp % WN;
  const int g = lane >> 2, t = lane & 3;
  const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * NB;
  const int64_t kbeg = (int64_t)blockIdx.z * kchunk;
  const int64_t kend = min(kdim, kbeg + kchunk);

  double acc[MI][NI][2];
#pragma unroll
  for (int a = 0; a < MI; ++a)
#pragma unroll
    for (int b = 0; b < NI; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

  TileLoader<TI, double> la, lb;
  int buf = 0;
  if (kbeg < kend) {
    la.load_a(A, a_rs, a_cs, m, kend, m0, kbeg, tid);
    lb.template load_b<NB>(B, b_rs, b_cs, kend, n, kbeg, n0, tid);
    la.store_a(As[0], a_rs, a_cs, tid);
    lb.template store_b<NB>(Bs[0], b_rs, b_cs, tid);
  }
  __syncthreads();
  for (int64_t k0 = kbeg; k0 < kend; k0 += BK) {
    const bool more = k0 + BK < kend;
    if (more) {
      la.load_a(A, a_rs, a_cs, m, kend, m0, k0 + BK, tid);
      lb.template load_b<NB>(B, b_rs, b_cs, kend, n, k0 + BK, n0, tid);
    }
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[MI], bf[NI];
#pragma unroll
      for (int mi = 0; mi < MI; ++mi) af[mi] = As[buf][wm * (MI * 8) + mi * 8 + g][kk + t];
#pragma unroll
      for (int ni = 0; ni < NI; ++ni) bf[ni] = Bs[buf][wn * (NI * 8) + ni * 8 + g][kk + t];
#pragma unroll
      for (int mi = 0; mi < MI; ++mi)
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni]);
    }
    if (more) {
      la.store_a(As[buf ^ 1], a_rs, a_cs, tid);
      lb.template store_b<NB>(Bs[buf ^ 1], b_rs, b_cs, tid);
    }
    __syncthreads();
    buf ^= 1;
  }

#pragma unroll
  for (int mi = 0; mi < MI; ++mi)
#pragma unroll
    for (int ni = 0; ni < NI; ++ni)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t i = m0 + wm * (MI * 8) + mi * 8 + g;
        const int64_t j = n0 + wn * (NI * 8) + ni * 8 + 2 * t + h;
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

// fp32 SIMT: 128 threads, each a 4 x 8 micro-tile (rows ty+16a, cols tx+8b)
// of the 64 x 64 CTA tile; products and sums in fp32 FFMA.
__global__ void __launch_bounds__(THREADS) gemm_f32_simt(int64_t m, int64_t n, int64_t kdim, int64_t kchunk,
                                                         float alpha, const float* __restrict__ A, int64_t a_rs,
                                                         int64_t a_cs, const float* __restrict__ B, int64_t b_rs,
                                                         int64_t b_cs, float beta, float* C, int64_t c_rs,
                                                         int64_t c_cs, float* ws) {
  __shared__ __align__(16) float As[2][BM][BK + PAD];
  __shared__ __align__(16) float Bs[2][BN][BK + PAD];
  const int tid = threadIdx.x;
  const int ty = tid / 8, tx = tid % 8;  // 16 x 8 threads
  const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;
  const int64_t kbeg = (int64_t)blockIdx.z * kchunk;
  const int64_t kend = min(kdim, kbeg + kchunk);
  float acc[4][8];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 8; ++b) acc[a][b] = 0.f;
  TileLoader<float> la, lb;
  int buf = 0;
  if (kbeg < kend) {
    la.load_a(A, a_rs, a_cs, m, kend, m0, kbeg, tid);
    lb.load_b(B, b_rs, b_cs, kend, n, kbeg, n0, tid);
    la.store_a(As[0], a_rs, a_cs, tid);
    lb.store_b(Bs[0], b_rs, b_cs, tid);
  }
  __syncthreads();
  for (int64_t k0 = kbeg; k0 < kend; k0 += BK) {
    const bool more = k0 + BK < kend;
    if (more) {
      la.load_a(A, a_rs, a_cs, m, kend, m0, k0 + BK, tid);
      lb.load_b(B, b_rs, b_cs, kend, n, k0 + BK, n0, tid);
    }
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float av[4], bv[8];
#pragma unroll
      for (int a = 0; a < 4; ++a) av[a] = As[buf][ty + 16 * a][kk];
#pragma unroll
      for (int b = 0; b < 8; ++b) bv[b] = Bs[buf][tx + 8 * b][kk];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 8; ++b) acc[a][b] = fmaf(av[a], bv[b], acc[a][b]);
    }
    if (more) {
      la.store_a(As[buf ^ 1], a_rs, a_cs, tid);
      lb.store_b(Bs[buf ^ 1], b_rs, b_cs, tid);
    }
    __syncthreads();
    buf ^= 1;
  }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      const int64_t i = m0 + ty + 16 * a, j = n0 + tx + 8 * b;
      if (i < m && j < n) {
        if (ws) {
          ws[(int64_t)blockIdx.z * m * n + i * n + j] = acc[a][b];
        } else {
          float* cp = C + i * c_rs + j * c_cs;
          *cp = beta == 0.f ? alpha * acc[a][b] : alpha * acc[a][b] + beta * *cp;
        }
      }
    }
}

// C(i, j) = C(j, i) for the tiles a symmetric launch skipped (tile(i) > tile(j)).
__global__ void mirror_lower_tiles(int64_t n, double* C, int64_t c_rs, int64_t c_cs) {
  const int64_t total = n * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / n, j = e % n;
    if (i / BM > j / BN) C[i * c_rs + j * c_cs] = C[j * c_rs + i * c_cs];
  }
}

template <class T>
__global__ void splitk_reduce(int64_t m, int64_t n, int splits, const T* __restrict__ ws, T alpha, T beta, T* C,
                              int64_t c_rs, int64_t c_cs) {
  const int64_t total = m * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    T sum = ws[e];
    for (int z = 1; z < splits; ++z) sum += ws[(int64_t)z * total + e];
    const int64_t i = e / n, j = e % n;
    T* cp = C + i * c_rs + j * c_cs;
    *cp = beta == T(0) ? alpha * sum : alpha * sum + beta * *cp;
  }
}

}  // namespace

// gemm_dmma.cu: the cp.async-pipelined DMMA kernel for K-major A and B.
template <class TI>
int dmma_kk_applicable(const TI* A, int64_t a_rs, int64_t a_cs, const TI* B, int64_t b_rs, int64_t b_cs);
template <class TI>
void dmma_kk_launch(rnla_ctx* ctx, int layout, int64_t m, int64_t n, int64_t k, int64_t kchunk, int64_t splits,
                    double alpha, const TI* A, int64_t lda, const TI* B, int64_t ldb, double beta, double* C,
                    int64_t c_rs, int64_t c_cs, double* ws, int sym);
int dmma_kk_tiles(int64_t m, int64_t n, int sym);
int dmma_kk_per_sm();
template <class TI>
static bool try_dmma_kk(rnla_ctx* ctx, int64_t m, int64_t n, int64_t k, double alpha, const TI* A, int64_t a_rs,
                        int64_t a_cs, const TI* B, int64_t b_rs, int64_t b_cs, double beta, double* C, int64_t c_rs,
                        int64_t c_cs, int max_splits, int sym);

// gemm_skinny.cu: fp64 DMMA kernel for n <= 32 outputs.
bool gemm_skinny_f64(rnla_ctx* ctx, int64_t m, int64_t n, int64_t k, double alpha, const double* A, int64_t a_rs,
                     int64_t a_cs, const double* B, int64_t b_rs, int64_t b_cs, double beta, double* C, int64_t c_rs,
                     int64_t c_cs, int max_splits);

template <class T>
void gemm(rnla_ctx* ctx, int64_t m, int64_t n, int64_t k, T alpha, const T* A, int64_t a_rs, int64_t a_cs,
          const T* B, int64_t b_rs, int64_t b_cs, T beta, T* C, int64_t c_rs, int64_t c_cs, int max_splits) {
  if (m == 0 || n == 0) return;
  if constexpr (std::is_same<T, float>::value) {
    if (tc_gemm_enabled()) {  // fp32: tcgen05 BF16x3 (gemm_tc.cu)
      gemm_f32_tc(ctx, m, n, k, alpha, A, a_rs, a_cs, B, b_rs, b_cs, beta, C, c_rs, c_cs);
      return;
    }
  }
  if constexpr (std::is_same<T, double>::value) {
    if (n <= 32 && gemm_skinny_f64(ctx, m, n, k, alpha, A, a_rs, a_cs, B, b_rs, b_cs, beta, C, c_rs, c_cs, max_splits))
      return;
    if (m >= 64 && n >= 64 &&
        try_dmma_kk<double>(ctx, m, n, k, alpha, A, a_rs, a_cs, B, b_rs, b_cs, beta, C, c_rs, c_cs, max_splits, 0))
      return;
  }
  // narrow outputs (n mod 64 in 1..32) use 32-wide tiles for the fp64 kernel
  const int nb = (std::is_same<T, double>::value && ((n % 64) != 0) && ((n % 64) <= 32)) ? 32 : BN;
  const int64_t tiles = ((m + BM - 1) / BM) * ((n + nb - 1) / nb);
  // Split K until there are ~4 CTAs per SM, keeping >= 256 k per split.
  int64_t splits = 1;
  const int64_t want = (int64_t)ctx->num_sms * 4;
  if (tiles < want && k >= 512) {
    splits = std::min<int64_t>((want + tiles - 1) / tiles, k / 256);
    splits = std::max<int64_t>(splits, 1);
    splits = std::min<int64_t>(splits, std::max(1, max_splits));
  }
  int64_t kchunk = (k + splits - 1) / splits;
  kchunk = (kchunk + BK - 1) / BK * BK;
  splits = std::max<int64_t>(1, (k + kchunk - 1) / kchunk);
  if (k == 0) splits = 1, kchunk = BK;
  DevBuf ws;
  T* wsp = nullptr;
  if (splits > 1) {
    ws = DevBuf(sizeof(T) * (size_t)(splits * m * n), ctx->stream);
    wsp = ws.as<T>();
  }
  dim3 grid((unsigned)((n + nb - 1) / nb), (unsigned)((m + BM - 1) / BM), (unsigned)splits);
  if constexpr (std::is_same<T, double>::value) {
    if (nb == 32)
      gemm_f64_dmma<double, 32, 1><<<grid, THREADS, 0, ctx->stream>>>(m, n, k, kchunk, alpha, A, a_rs, a_cs, B, b_rs,
                                                                   b_cs, beta, C, c_rs, c_cs, wsp, 0);
    else
      gemm_f64_dmma<double, 64, 3><<<grid, THREADS, 0, ctx->stream>>>(m, n, k, kchunk, alpha, A, a_rs, a_cs, B, b_rs, b_cs,
                                                               beta, C, c_rs, c_cs, wsp, 0);
  } else {
    gemm_f32_simt<<<grid, THREADS, 0, ctx->stream>>>(m, n, k, kchunk, alpha, A, a_rs, a_cs, B, b_rs, b_cs, beta, C,
                                                    c_rs, c_cs, wsp);
  }
  RNLA_CUDA(cudaGetLastError());
  note_launch(ctx);
  if (splits > 1) {
    const int blocks = (int)std::min<int64_t>((m * n + 255) / 256, (int64_t)ctx->num_sms * 8);
    splitk_reduce<T><<<blocks, 256, 0, ctx->stream>>>(m, n, (int)splits, wsp, alpha, beta, C, c_rs, c_cs);
    RNLA_CUDA(cudaGetLastError());
    note_launch(ctx);
  }
}

// Smallest split-K count whose CTAs keep >= 85 % of the last wave of `slots`
// busy (else the best one), with >= 256 k per split.
static int64_t wave_splits(int64_t active, int64_t slots, int64_t k, int64_t cap) {
  if (active <= 0 || slots <= 0 || k < 512) return 1;
  int64_t best = 1;
  double best_eff = 0.0;
  for (int64_t s = 1; s <= std::max<int64_t>(1, std::min<int64_t>(cap, k / 256)); ++s) {
    const int64_t ctas = active * s;
    const double eff = (double)ctas / (double)(((ctas + slots - 1) / slots) * slots);
    if (eff >= 0.85) return s;
    if (eff > best_eff + 1e-9) best_eff = eff, best = s;
  }
  return best;
}

// Split-K sized on the K-major DMMA kernel's tiles, fixed-order reduce, and
// the lower-tile mirror for symmetric products. False when the layout does not
// apply (the caller falls back to the generic kernel).
template <class TI>
static bool try_dmma_kk(rnla_ctx* ctx, int64_t m, int64_t n, int64_t k, double alpha, const TI* A, int64_t a_rs,
                        int64_t a_cs, const TI* B, int64_t b_rs, int64_t b_cs, double beta, double* C, int64_t c_rs,
                        int64_t c_cs, int max_splits, int sym) {
  const int layout = dmma_kk_applicable<TI>(A, a_rs, a_cs, B, b_rs, b_cs);
  if (!layout) return false;
  const int64_t active = dmma_kk_tiles(m, n, sym);
  int64_t splits = wave_splits(active, (int64_t)dmma_kk_per_sm() * ctx->num_sms, k, std::max(1, max_splits));
  int64_t kchunk = ((k + splits - 1) / splits + BK - 1) / BK * BK;
  if (k == 0) kchunk = BK;
  splits = std::max<int64_t>(1, (k + kchunk - 1) / kchunk);
  DevBuf ws;
  double* wsp = nullptr;
  if (splits > 1) {
    ws = DevBuf(sizeof(double) * (size_t)(splits * m * n), ctx->stream);
    wsp = ws.as<double>();
  }
  dmma_kk_launch<TI>(ctx, layout, m, n, k, kchunk, splits, alpha, A, a_rs, B, layout == 1 ? b_cs : b_rs, beta, C,
                     c_rs, c_cs, wsp, sym);
  if (splits > 1) {
    const int blocks = (int)std::min<int64_t>((m * n + 255) / 256, (int64_t)ctx->num_sms * 8);
    splitk_reduce<double><<<blocks, 256, 0, ctx->stream>>>(m, n, (int)splits, wsp, alpha, beta, C, c_rs, c_cs);
    RNLA_CUDA(cudaGetLastError());
    note_launch(ctx);
  }
  if (sym & 1) {
    mirror_lower_tiles<<<grid_for(ctx, m * n, 256), 256, 0, ctx->stream>>>(m, C, c_rs, c_cs);
    RNLA_CUDA(cudaGetLastError());
    note_launch(ctx);
  }
  return true;
}

bool gemm_f64_structured(rnla_ctx* ctx, int64_t m, int64_t n, int64_t k, const double* A, int64_t a_rs, int64_t a_cs,
                         const double* B, int64_t b_rs, int64_t b_cs, double* C, int64_t c_rs, int64_t c_cs,
                         int flags) {
  if (m == 0 || n == 0) return true;
  if ((flags & 1) && m != n) return false;
  return try_dmma_kk<double>(ctx, m, n, k, 1.0, A, a_rs, a_cs, B, b_rs, b_cs, 0.0, C, c_rs, c_cs, 64, flags);
}

void gemm_f32_in_f64(rnla_ctx* ctx, int64_t m, int64_t n, int64_t k, double alpha, const float* A, int64_t a_rs,
                     int64_t a_cs, const float* B, int64_t b_rs, int64_t b_cs, double beta, double* C, int64_t c_rs,
                     int64_t c_cs) {
  if (m == 0 || n == 0) return;
  // Gram products (B = A') are symmetric: compute the upper tiles only.
  const int sym = (A == B && m == n && a_rs == b_cs && a_cs == b_rs) ? 1 : 0;
  if (try_dmma_kk<float>(ctx, m, n, k, alpha, A, a_rs, a_cs, B, b_rs, b_cs, beta, C, c_rs, c_cs, 64, sym)) return;
  const int64_t tm = (m + BM - 1) / BM, tn = (n + BN - 1) / BN;
  const int64_t active = sym ? tm * (tm + 1) / 2 : tm * tn;
  static const int per_sm = [] {
    int b = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, gemm_f64_dmma<float, 64, RNLA_DMMA_F32_MINB>, THREADS, 0) !=
            cudaSuccess ||
        b < 1)
      b = 1;
    return b;
  }();
  int64_t splits = wave_splits(active, (int64_t)per_sm * ctx->num_sms, k, 64);
  int64_t kchunk = ((k + splits - 1) / splits + BK - 1) / BK * BK;
  if (k == 0) kchunk = BK;
  splits = std::max<int64_t>(1, (k + kchunk - 1) / kchunk);
  DevBuf ws;
  double* wsp = nullptr;
  if (splits > 1) {
    ws = DevBuf(sizeof(double) * (size_t)(splits * m * n), ctx->stream);
    wsp = ws.as<double>();
  }
  dim3 grid((unsigned)((n + BN - 1) / BN), (unsigned)((m + BM - 1) / BM), (unsigned)splits);
  gemm_f64_dmma<float, 64, RNLA_DMMA_F32_MINB><<<grid, THREADS, 0, ctx->stream>>>(m, n, k, kchunk, alpha, A, a_rs, a_cs, B, b_rs, b_cs, beta,
                                                          C, c_rs, c_cs, wsp, sym);
  RNLA_CUDA(cudaGetLastError());
  note_launch(ctx);
  if (splits > 1) {
    const int blocks = (int)std::min<int64_t>((m * n + 255) / 256, (int64_t)ctx->num_sms * 8);
    splitk_reduce<double><<<blocks, 256, 0, ctx->stream>>>(m, n, (int)splits, wsp, alpha, beta, C, c_rs, c_cs);
    RNLA_CUDA(cudaGetLastError());
    note_launch(ctx);
  }
  if (sym) {
    mirror_lower_tiles<<<grid_for(ctx, m * n, 256), 256, 0, ctx->stream>>>(m, C, c_rs, c_cs);
    RNLA_CUDA(cudaGetLastError());
    note_launch(ctx);
  }
}

template void gemm<double>(rnla_ctx*, int64_t, int64_t, int64_t, double, const double*, int64_t, int64_t,
                           const double*, int64_t, int64_t, double, double*, int64_t, int64_t, int);
template void gemm<float>(rnla_ctx*, int64_t, int64_t, int64_t, float, const float*, int64_t, int64_t, const float*,
                          int64_t, int64_t, float, float*, int64_t, int64_t, int);

}  // namespace rnla
