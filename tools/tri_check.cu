// Standalone harness for syev_tri_kernel (tools/tri_check.py drives it via ctypes).
#include <cuda_runtime.h>
#include <cstdio>
#include "../paper_1505_07570_b200/csrc/syev_tri.cuh"

extern "C" int tri_eig(int n, const double* Hh, double* lamh, double* Zh, int desc, int reps, float* ms, long long* profh) {
  long long* prof;
  cudaMalloc(&prof, sizeof(long long) * 8);
  double *H, *lam, *Z, *hv;
  int* st;
  cudaMalloc(&H, sizeof(double) * n * n);
  cudaMalloc(&Z, sizeof(double) * n * n);
  cudaMalloc(&hv, sizeof(double) * n * n);
  cudaMalloc(&lam, sizeof(double) * n);
  cudaMalloc(&st, sizeof(int));
  cudaMemcpy(H, Hh, sizeof(double) * n * n, cudaMemcpyHostToDevice);
  const size_t smem = rnla::tri_smem_bytes(n);
  cudaFuncSetAttribute(rnla::syev_tri_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  rnla::syev_tri_kernel<<<1, rnla::kTriThreads, smem>>>(n, H, lam, Z, hv, st, desc, prof);
  cudaEventRecord(a);
  for (int r = 0; r < reps; ++r) rnla::syev_tri_kernel<<<1, rnla::kTriThreads, smem>>>(n, H, lam, Z, hv, st, desc);
  cudaEventRecord(b);
  cudaError_t err = cudaDeviceSynchronize();
  if (err != cudaSuccess) {
    std::fprintf(stderr, "tri_eig: %s\n", cudaGetErrorString(err));
    return -1;
  }
  cudaEventElapsedTime(ms, a, b);
  if (reps > 0) *ms /= reps;
  int hs = 0;
  cudaMemcpy(&hs, st, sizeof(int), cudaMemcpyDeviceToHost);
  cudaMemcpy(lamh, lam, sizeof(double) * n, cudaMemcpyDeviceToHost);
  cudaMemcpy(Zh, Z, sizeof(double) * n * n, cudaMemcpyDeviceToHost);
  cudaMemcpy(profh, prof, sizeof(long long) * 6, cudaMemcpyDeviceToHost);
  cudaFree(prof);
  cudaFree(H); cudaFree(Z); cudaFree(hv); cudaFree(lam); cudaFree(st);
  return hs;
}
