// green.cpp -- SM-partitioned streams (CUDA green contexts) for running an
// HBM-bound kernel and a DMMA-bound kernel side by side on one GPU.
//
// The combined CountSketch -> Gaussian sketch of BASELINE config 1 is a
// bandwidth-bound gather followed by a DMMA GEMM. Launched on ordinary
// streams they cannot overlap: the gather's CTAs occupy every SM's register
// file. A green context pins the gather to most SMs and the GEMM chunks to the
// rest, so the Gaussian stage of finished bucket chunks runs under the gather
// (api_sketch.cpp combined_gaussian_pipelined). The driver entry points are
// fetched at run time (no -lcuda), and every failure falls back to the
// ordinary streams.
#include <cuda.h>

#include <cstdlib>

#include "rnla_internal.h"

namespace rnla {

namespace {

template <class F>
F entry(const char* name) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
    return nullptr;
  return reinterpret_cast<F>(p);
}

}  // namespace

GreenSplit::~GreenSplit() {
  using DestroyStream = CUresult (*)(CUstream);
  using DestroyGreen = CUresult (*)(CUgreenCtx);
  static auto ds = entry<DestroyStream>("cuStreamDestroy");
  static auto dg = entry<DestroyGreen>("cuGreenCtxDestroy");
  for (auto s : {gather[0], gather[1], gemm})
    if (s && ds) ds(reinterpret_cast<CUstream>(s));
  for (auto g : {ctx_gather, ctx_gemm})
    if (g && dg) dg(reinterpret_cast<CUgreenCtx>(g));
}

// Split the device's SMs into a GEMM group of about `gemm_sms` SMs and the
// remainder for the gather; two gather streams and one GEMM stream.
std::unique_ptr<GreenSplit> make_green_split(int device, int gemm_sms) {
  using GetDev = CUresult (*)(CUdevice*, int);
  using GetRes = CUresult (*)(CUdevice, CUdevResource*, CUdevResourceType);
  using Split = CUresult (*)(CUdevResource*, unsigned int*, const CUdevResource*, CUdevResource*, unsigned int,
                             unsigned int);
  using GenDesc = CUresult (*)(CUdevResourceDesc*, CUdevResource*, unsigned int);
  using Create = CUresult (*)(CUgreenCtx*, CUdevResourceDesc, CUdevice, unsigned int);
  using StreamCreate = CUresult (*)(CUstream*, CUgreenCtx, unsigned int, int);
  static auto get_dev = entry<GetDev>("cuDeviceGet");
  static auto get_res = entry<GetRes>("cuDeviceGetDevResource");
  static auto split = entry<Split>("cuDevSmResourceSplitByCount");
  static auto gen = entry<GenDesc>("cuDevResourceGenerateDesc");
  static auto create = entry<Create>("cuGreenCtxCreate");
  static auto screate = entry<StreamCreate>("cuGreenCtxStreamCreate");
  if (!get_dev || !get_res || !split || !gen || !create || !screate) return nullptr;
  CUdevice dev;
  if (get_dev(&dev, device) != CUDA_SUCCESS) return nullptr;
  CUdevResource all{}, groups[1]{}, rest{};
  if (get_res(dev, &all, CU_DEV_RESOURCE_TYPE_SM) != CUDA_SUCCESS) return nullptr;
  unsigned int n = 1;
  if (split(groups, &n, &all, &rest, 0, (unsigned)gemm_sms) != CUDA_SUCCESS || n != 1) return nullptr;
  if (rest.type != CU_DEV_RESOURCE_TYPE_SM || rest.sm.smCount == 0) return nullptr;
  auto g = std::make_unique<GreenSplit>();
  CUdevResourceDesc da, db;
  if (gen(&da, &rest, 1) != CUDA_SUCCESS || gen(&db, groups, 1) != CUDA_SUCCESS) return nullptr;
  CUgreenCtx ca, cb;
  if (create(&ca, da, dev, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS) return nullptr;
  g->ctx_gather = ca;
  if (create(&cb, db, dev, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS) return nullptr;
  g->ctx_gemm = cb;
  CUstream s0, s1, s2;
  if (screate(&s0, ca, CU_STREAM_NON_BLOCKING, 0) != CUDA_SUCCESS) return nullptr;
  g->gather[0] = reinterpret_cast<cudaStream_t>(s0);
  if (screate(&s1, ca, CU_STREAM_NON_BLOCKING, 0) != CUDA_SUCCESS) return nullptr;
  g->gather[1] = reinterpret_cast<cudaStream_t>(s1);
  if (screate(&s2, cb, CU_STREAM_NON_BLOCKING, 0) != CUDA_SUCCESS) return nullptr;
  g->gemm = reinterpret_cast<cudaStream_t>(s2);
  g->gather_sms = (int)rest.sm.smCount;
  g->gemm_sms = (int)groups[0].sm.smCount;
  return g;
}

}  // namespace rnla
