// dist.cpp -- NCCL plumbing for row-sharded contexts: one
// process per GPU, collectives on the context's stream.
#include <nccl.h>

#include "dist.h"

namespace rnla {

static void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw NcclError(std::string(what) + ": " + ncclGetErrorString(r));
}

void allreduce_sum(rnla_ctx* ctx, void* buf, size_t count, int dtype) {
  if (ctx->world <= 1 || count == 0) return;
  nccl_check(ncclAllReduce(buf, buf, count, dtype == RNLA_F64 ? ncclFloat64 : ncclFloat32, ncclSum,
                           static_cast<ncclComm_t>(ctx->nccl), ctx->stream),
             "ncclAllReduce");
}

void reduce_to(rnla_ctx* ctx, void* buf, size_t count, int dtype, int root) {
  if (ctx->world <= 1 || count == 0) return;
  nccl_check(ncclReduce(buf, buf, count, dtype == RNLA_F64 ? ncclFloat64 : ncclFloat32, ncclSum, root,
                        static_cast<ncclComm_t>(ctx->nccl), ctx->stream),
             "ncclReduce");
}

int64_t global_row_offset(rnla_ctx* ctx, int64_t local_rows, int64_t* total_rows) {
  if (ctx->world <= 1) {
    if (total_rows) *total_rows = local_rows;
    return 0;
  }
  DevBuf buf(sizeof(int64_t) * ctx->world, ctx->stream);
  DevBuf mine(sizeof(int64_t), ctx->stream);
  RNLA_CUDA(cudaMemcpyAsync(mine.p, &local_rows, sizeof(int64_t), cudaMemcpyHostToDevice, ctx->stream));
  nccl_check(ncclAllGather(mine.p, buf.p, 1, ncclInt64, static_cast<ncclComm_t>(ctx->nccl), ctx->stream),
             "ncclAllGather");
  std::vector<int64_t> counts(ctx->world);
  RNLA_CUDA(cudaMemcpyAsync(counts.data(), buf.p, sizeof(int64_t) * ctx->world, cudaMemcpyDeviceToHost, ctx->stream));
  RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
  int64_t off = 0, tot = 0;
  for (int r = 0; r < ctx->world; ++r) {
    if (r < ctx->rank) off += counts[r];
    tot += counts[r];
  }
  if (total_rows) *total_rows = tot;
  return off;
}

double allreduce_scalar(rnla_ctx* ctx, double v) {
  if (ctx->world <= 1) return v;
  DevBuf b(sizeof(double), ctx->stream);
  RNLA_CUDA(cudaMemcpyAsync(b.p, &v, sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  allreduce_sum(ctx, b.p, 1, RNLA_F64);
  RNLA_CUDA(cudaMemcpyAsync(&v, b.p, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
  return v;
}

}  // namespace rnla
