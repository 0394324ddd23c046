// dist.cpp -- NCCL plumbing for row-sharded contexts: one
// process per GPU, collectives on the context's stream.
#include <nccl.h>

#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <cstring>

#include "dist.h"

// In-process shard group (rnla_group_create): ranks are host threads, each with
// its own context; a collective syncs the rank's stream, stages its buffer in
// host memory, meets the others at a barrier and sums the staged buffers in
// rank order (identical bits on every rank), then copies the result back.
struct rnla_group {
  int world = 1;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t generation = 0;
  bool broken = false;
  std::vector<std::vector<char>> slots;
};

namespace rnla {

static void group_barrier(rnla_group* g) {
  static const double timeout_s = std::getenv("RNLA_GROUP_TIMEOUT_S") ? std::atof(std::getenv("RNLA_GROUP_TIMEOUT_S"))
                                                                      : 300.0;
  std::unique_lock<std::mutex> lk(g->mu);
  if (g->broken) throw NcclError("shard group: another rank failed");
  const uint64_t gen = g->generation;
  if (++g->arrived == g->world) {
    g->arrived = 0;
    ++g->generation;
    g->cv.notify_all();
    return;
  }
  const bool ok = g->cv.wait_for(lk, std::chrono::duration<double>(timeout_s),
                                 [&] { return g->generation != gen || g->broken; });
  if (!ok || g->broken) {
    g->broken = true;
    g->cv.notify_all();
    throw NcclError("shard group: collective timed out or another rank failed");
  }
}

static size_t dtype_size(int dtype) { return dtype == RNLA_F32 ? 4 : 8; }

template <class T>
static void sum_slots(rnla_group* g, size_t count, T* out) {
  const T* first = reinterpret_cast<const T*>(g->slots[0].data());
  std::memcpy(out, first, sizeof(T) * count);
  for (int r = 1; r < g->world; ++r) {
    const T* x = reinterpret_cast<const T*>(g->slots[(size_t)r].data());
    for (size_t i = 0; i < count; ++i) out[i] += x[i];
  }
}

// dtype: RNLA_F64, RNLA_F32, or -1 for int64.
static void group_reduce(rnla_ctx* ctx, void* buf, size_t count, int dtype, int root) {
  rnla_group* g = ctx->group;
  const size_t bytes = count * (dtype == -1 ? 8 : dtype_size(dtype));
  std::vector<char>& mine = g->slots[(size_t)ctx->rank];
  mine.resize(bytes);
  RNLA_CUDA(cudaMemcpyAsync(mine.data(), buf, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
  group_barrier(g);
  std::vector<char> out;
  if (root < 0 || root == ctx->rank) {
    out.resize(bytes);
    if (dtype == RNLA_F64) sum_slots<double>(g, count, reinterpret_cast<double*>(out.data()));
    else if (dtype == RNLA_F32) sum_slots<float>(g, count, reinterpret_cast<float*>(out.data()));
    else sum_slots<int64_t>(g, count, reinterpret_cast<int64_t*>(out.data()));
  }
  group_barrier(g);  // every rank has read the slots
  if (!out.empty()) {
    RNLA_CUDA(cudaMemcpyAsync(buf, out.data(), bytes, cudaMemcpyHostToDevice, ctx->stream));
    RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
  }
}

void group_mark_broken(rnla_group* g) {
  std::lock_guard<std::mutex> lk(g->mu);
  g->broken = true;
  g->cv.notify_all();
}

void group_destroy(rnla_group* g) { delete g; }
int group_world(const rnla_group* g) { return g->world; }

rnla_group* group_create(int world) {
  auto* g = new rnla_group();
  g->world = world;
  g->slots.resize((size_t)world);
  return g;
}

static void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw NcclError(std::string(what) + ": " + ncclGetErrorString(r));
}

void allreduce_sum(rnla_ctx* ctx, void* buf, size_t count, int dtype) {
  if (!is_sharded(ctx) || count == 0) return;
  if (ctx->group) return group_reduce(ctx, buf, count, dtype, -1);
  nccl_check(ncclAllReduce(buf, buf, count, dtype == RNLA_F64 ? ncclFloat64 : ncclFloat32, ncclSum,
                           static_cast<ncclComm_t>(ctx->nccl), ctx->stream),
             "ncclAllReduce");
}

void reduce_to(rnla_ctx* ctx, void* buf, size_t count, int dtype, int root) {
  if (!is_sharded(ctx) || count == 0) return;
  if (ctx->group) return group_reduce(ctx, buf, count, dtype, root);
  nccl_check(ncclReduce(buf, buf, count, dtype == RNLA_F64 ? ncclFloat64 : ncclFloat32, ncclSum, root,
                        static_cast<ncclComm_t>(ctx->nccl), ctx->stream),
             "ncclReduce");
}

int64_t global_row_offset(rnla_ctx* ctx, int64_t local_rows, int64_t* total_rows) {
  if (!is_sharded(ctx)) {
    if (total_rows) *total_rows = local_rows;
    return 0;
  }
  DevBuf buf(sizeof(int64_t) * ctx->world, ctx->stream);
  std::vector<int64_t> counts(ctx->world, 0);
  if (ctx->group) {
    counts[(size_t)ctx->rank] = local_rows;
    RNLA_CUDA(cudaMemcpyAsync(buf.p, counts.data(), sizeof(int64_t) * ctx->world, cudaMemcpyHostToDevice, ctx->stream));
    group_reduce(ctx, buf.p, (size_t)ctx->world, -1, -1);
  } else {
    DevBuf mine(sizeof(int64_t), ctx->stream);
    RNLA_CUDA(cudaMemcpyAsync(mine.p, &local_rows, sizeof(int64_t), cudaMemcpyHostToDevice, ctx->stream));
    nccl_check(ncclAllGather(mine.p, buf.p, 1, ncclInt64, static_cast<ncclComm_t>(ctx->nccl), ctx->stream),
               "ncclAllGather");
  }
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
  if (!is_sharded(ctx)) return v;
  DevBuf b(sizeof(double), ctx->stream);
  RNLA_CUDA(cudaMemcpyAsync(b.p, &v, sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  allreduce_sum(ctx, b.p, 1, RNLA_F64);
  RNLA_CUDA(cudaMemcpyAsync(&v, b.p, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
  return v;
}

void allgather_blocks(rnla_ctx* ctx, const void* mine, void* all, size_t count, int dtype) {
  const size_t es = dtype == -1 ? 8 : dtype_size(dtype);
  RNLA_CUDA(cudaMemsetAsync(all, 0, es * count * (size_t)ctx->world, ctx->stream));
  RNLA_CUDA(cudaMemcpyAsync(static_cast<char*>(all) + es * count * (size_t)ctx->rank, mine, es * count,
                            cudaMemcpyDeviceToDevice, ctx->stream));
  if (!is_sharded(ctx)) return;
  if (ctx->group) return group_reduce(ctx, all, count * (size_t)ctx->world, dtype, -1);
  nccl_check(ncclAllGather(mine, all, count,
                           dtype == RNLA_F32 ? ncclFloat32 : (dtype == RNLA_F64 ? ncclFloat64 : ncclInt64),
                           static_cast<ncclComm_t>(ctx->nccl), ctx->stream),
             "ncclAllGather");
}

}  // namespace rnla
