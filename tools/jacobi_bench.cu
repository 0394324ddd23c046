// Standalone timing of the one-CTA Jacobi eigensolver (jacobi.cuh):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -DRNLA_JACOBI_PROF=1 -I paper_1505_07570_b200/csrc tools/jacobi_bench.cu
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include "jacobi.cuh"

int main() {
  for (int n : {30, 96}) {
    std::vector<double> B((size_t)n * 300), H((size_t)n * n);
    srand(1);
    for (auto& x : B) x = (rand() / (double)RAND_MAX - 0.5);
    for (int i = 0; i < n; ++i)
      for (int k = 0; k < 300; ++k) B[i * 300 + k] *= exp(-i / 5.0);
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        double a = 0;
        for (int k = 0; k < 300; ++k) a += B[i * 300 + k] * B[j * 300 + k];
        H[i + j * n] = a;
      }
    double *dH, *dl, *dZ;
    int* ds;
    long long* dp;
    cudaMalloc(&dH, 8 * n * n); cudaMalloc(&dl, 8 * n); cudaMalloc(&dZ, 8 * n * n); cudaMalloc(&ds, 4);
    cudaMalloc(&dp, 64);
    cudaMemcpy(dH, H.data(), 8 * n * n, cudaMemcpyHostToDevice);
    const size_t smem = rnla::jacobi_smem_bytes(n);
    auto run = [&]() {
      if (n <= 32) {
        cudaFuncSetAttribute(rnla::jacobi_eig_kernel<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        rnla::jacobi_eig_kernel<512><<<1, 512, smem>>>(n, dH, dl, dZ, ds, dp);
      } else {
        cudaFuncSetAttribute(rnla::jacobi_eig_kernel<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        rnla::jacobi_eig_kernel<1024><<<1, 1024, smem>>>(n, dH, dl, dZ, ds, dp);
      }
    };
    run();
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int i = 0; i < 10; ++i) run();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    int st; long long pr[5];
    cudaMemcpy(&st, ds, 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(pr, dp, 40, cudaMemcpyDeviceToHost);
    std::vector<double> lam(n), Z((size_t)n * n);
    cudaMemcpy(lam.data(), dl, 8 * n, cudaMemcpyDeviceToHost);
    cudaMemcpy(Z.data(), dZ, 8 * n * n, cudaMemcpyDeviceToHost);
    double res = 0;
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i) {
        double a = 0;
        for (int k = 0; k < n; ++k) a += H[i + k * n] * Z[k + j * n];
        res = fmax(res, fabs(a - lam[j] * Z[i + j * n]));
      }
    const int sweeps = st >> 8, rounds = sweeps * (n + (n & 1) - 1);
    printf("n=%d  %.1f us/call  sweeps=%d status=%d  resid/lam1=%.2e  cycles/round: rot %.0f colupd %.0f sync1 %.0f phase2 %.0f sync2 %.0f  err=%s\n",
           n, ms * 100, sweeps, st & 255, res / lam[0], pr[4] / (double)rounds, pr[0] / (double)rounds, pr[1] / (double)rounds,
           pr[2] / (double)rounds, pr[3] / (double)rounds, cudaGetErrorString(cudaGetLastError()));
  }
}
