// api_core.cpp -- context lifecycle, error reporting, operand marshalling and
// the host-only entry points (seeds, hashes, libstdc++ operator draws).
#include <cublas_v2.h>
#include <cusolverDn.h>
#include <nccl.h>

#include <chrono>
#include <cstdlib>
#include <new>

#include "dist.h"
#include "marshal.h"

namespace rnla {

static thread_local std::string g_last_error;
static thread_local rnla_ctx* g_cur_ctx = nullptr;  // context of the entry point running on this thread

// A device/transport failure on one rank of an in-process shard group would
// leave the other ranks waiting in their next collective: mark the group
// broken so they fail fast instead (argument and numerical errors are
// replicated decisions, raised on every rank alike).
static void break_group_on_failure() {
  if (g_cur_ctx && g_cur_ctx->group && g_cur_ctx->world > 1) group_mark_broken(g_cur_ctx->group);
}

void set_error(const std::string& msg) { g_last_error = msg; }

rnla_status guard(const std::function<void()>& f) {
  g_cur_ctx = nullptr;
  try {
    f();
    return RNLA_OK;
  } catch (...) {
    // Drop a non-sticky CUDA error left by the failed call so the next
    // launch check on this thread does not report it again.
    (void)cudaGetLastError();
    try {
      throw;
    } catch (const InvalidArgument& e) {
    set_error(e.what());
    return RNLA_EINVAL;
  } catch (const NumericError& e) {
    set_error(e.what());
    return RNLA_ENUMERIC;
  } catch (const CudaError& e) {
    set_error(e.what());
    break_group_on_failure();
    return RNLA_ECUDA;
  } catch (const NcclError& e) {
    set_error(e.what());
    break_group_on_failure();
    return RNLA_ENCCL;
  } catch (const std::bad_alloc& e) {
    set_error("out of host memory");
    break_group_on_failure();
    return RNLA_ENOMEM;
  } catch (const std::exception& e) {
    set_error(e.what());
    break_group_on_failure();
    return RNLA_ECUDA;
  }
  }
}

void trace_mark(rnla_ctx* ctx, const char* label) {
  static const bool on = std::getenv("RNLA_TRACE") != nullptr;
  if (!on || ctx->capturing) return;
  static thread_local std::chrono::steady_clock::time_point last = std::chrono::steady_clock::now();
  cudaStreamSynchronize(ctx->stream);
  const auto now = std::chrono::steady_clock::now();
  std::fprintf(stderr, "[rnla trace] %-40s %9.3f ms\n", label,
               std::chrono::duration<double, std::milli>(now - last).count());
  last = now;
}

StreamScope::StreamScope(rnla_ctx* c, cudaStream_t s) : ctx(c), saved(c->stream) {
  ctx->stream = s;
  if (ctx->cusolver) cusolverDnSetStream(static_cast<cusolverDnHandle_t>(ctx->cusolver), s);
  if (ctx->cublas) cublasSetStream(static_cast<cublasHandle_t>(ctx->cublas), s);
}

StreamScope::~StreamScope() {
  ctx->stream = saved;
  if (ctx->cusolver) cusolverDnSetStream(static_cast<cusolverDnHandle_t>(ctx->cusolver), saved);
  if (ctx->cublas) cublasSetStream(static_cast<cublasHandle_t>(ctx->cublas), saved);
}

void enter(rnla_ctx* ctx) {
  require(ctx != nullptr, "null rnla_ctx");
  g_cur_ctx = ctx;
  RNLA_CUDA(cudaSetDevice(ctx->device));
}

void check_mat(const rnla_mat* m, const char* name) {
  require(m != nullptr, std::string(name) + ": null matrix");
  require(m->rows >= 0 && m->cols >= 0, std::string(name) + ": negative shape");
  require(m->dtype == RNLA_F64 || m->dtype == RNLA_F32, std::string(name) + ": unknown dtype");
  require(m->data != nullptr || m->rows == 0 || m->cols == 0, std::string(name) + ": null data");
  require(m->row_stride >= 0 && m->col_stride >= 0, std::string(name) + ": negative stride");
  require((m->row_stride > 0 || m->rows <= 1) && (m->col_stride > 0 || m->cols <= 1),
          std::string(name) + ": zero stride along an extent > 1");
}

static bool dense_col(const rnla_mat* m) { return m->row_stride == 1 && (m->col_stride >= m->rows || m->cols <= 1); }
static bool dense_row(const rnla_mat* m) { return m->col_stride == 1 && (m->row_stride >= m->cols || m->rows <= 1); }

DevMat alloc_dense(rnla_ctx* ctx, int64_t rows, int64_t cols, bool rowmajor, int dtype) {
  DevMat d;
  d.own = DevBuf(esize(dtype) * (size_t)std::max<int64_t>(rows * cols, 1), ctx->stream);
  d.p = d.own.p;
  d.rows = rows; d.cols = cols; d.dtype = dtype;
  d.rs = rowmajor ? cols : 1;
  d.cs = rowmajor ? 1 : rows;
  if (d.rs == 0) d.rs = 1;
  if (d.cs == 0) d.cs = 1;
  return d;
}

DevMat to_device(rnla_ctx* ctx, const rnla_mat* m) {
  check_mat(m, "matrix");
  DevMat d;
  d.rows = m->rows; d.cols = m->cols; d.dtype = m->dtype;
  if (m->on_device) {
    d.p = m->data; d.rs = m->row_stride; d.cs = m->col_stride;
    return d;
  }
  const size_t es = esize(m->dtype);
  if (m->rows == 0 || m->cols == 0) return alloc_dense(ctx, m->rows, m->cols, false, m->dtype);
  if (dense_row(m) && !dense_col(m)) {
    d = alloc_dense(ctx, m->rows, m->cols, true, m->dtype);
    const int64_t pitch = m->rows <= 1 ? m->cols : m->row_stride;
    RNLA_CUDA(cudaMemcpy2DAsync(d.p, es * m->cols, m->data, es * pitch, es * m->cols, m->rows,
                                cudaMemcpyHostToDevice, ctx->stream));
  } else if (dense_col(m)) {
    d = alloc_dense(ctx, m->rows, m->cols, false, m->dtype);
    const int64_t pitch = m->cols <= 1 ? m->rows : m->col_stride;
    RNLA_CUDA(cudaMemcpy2DAsync(d.p, es * m->rows, m->data, es * pitch, es * m->rows, m->cols,
                                cudaMemcpyHostToDevice, ctx->stream));
  } else {  // arbitrary host strides: gather on the host first
    d = alloc_dense(ctx, m->rows, m->cols, false, m->dtype);
    std::vector<char> tmp(es * (size_t)(m->rows * m->cols));
    const char* src = static_cast<const char*>(m->data);
    for (int64_t j = 0; j < m->cols; ++j)
      for (int64_t i = 0; i < m->rows; ++i)
        std::memcpy(&tmp[es * (size_t)(i + j * m->rows)], src + es * (size_t)(i * m->row_stride + j * m->col_stride),
                    es);
    RNLA_CUDA(cudaMemcpyAsync(d.p, tmp.data(), tmp.size(), cudaMemcpyHostToDevice, ctx->stream));
    RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  return d;
}

DevMat dense_copy(rnla_ctx* ctx, const DevMat& src, bool rowmajor, int dtype) {
  DevMat d = alloc_dense(ctx, src.rows, src.cols, rowmajor, dtype);
  if (src.dtype == RNLA_F64 && dtype == RNLA_F64)
    copy2d<double>(ctx, src.rows, src.cols, src.as<double>(), src.rs, src.cs, d.as<double>(), d.rs, d.cs);
  else if (src.dtype == RNLA_F32 && dtype == RNLA_F32)
    copy2d<float>(ctx, src.rows, src.cols, src.as<float>(), src.rs, src.cs, d.as<float>(), d.rs, d.cs);
  else if (src.dtype == RNLA_F64)
    copy2d_cast<double, float>(ctx, src.rows, src.cols, src.as<double>(), src.rs, src.cs, d.as<float>(), d.rs, d.cs);
  else
    copy2d_cast<float, double>(ctx, src.rows, src.cols, src.as<float>(), src.rs, src.cs, d.as<double>(), d.rs, d.cs);
  return d;
}

DevMat as_rowmajor(rnla_ctx* ctx, DevMat&& src) {
  if (src.rowmajor()) return std::move(src);
  return dense_copy(ctx, src, true, src.dtype);
}

DevMat as_colmajor(rnla_ctx* ctx, DevMat&& src) {
  if (src.colmajor()) return std::move(src);
  return dense_copy(ctx, src, false, src.dtype);
}

OutMat::OutMat(rnla_ctx* ctx, const rnla_mat* m, int64_t rows, int64_t cols, const char* name, bool prefer_rowmajor) {
  check_mat(m, name);
  require(m->rows == rows && m->cols == cols, std::string(name) + ": expected " + std::to_string(rows) + " x " +
                                                   std::to_string(cols) + ", got " + std::to_string(m->rows) + " x " +
                                                   std::to_string(m->cols));
  dst = m;
  if (m->on_device) {
    dev.p = m->data; dev.rows = rows; dev.cols = cols; dev.rs = m->row_stride; dev.cs = m->col_stride;
    dev.dtype = m->dtype;
    return;
  }
  staged = true;
  const bool rowmajor = dense_row(m) && !dense_col(m) ? true : (dense_col(m) ? false : prefer_rowmajor);
  dev = alloc_dense(ctx, rows, cols, rowmajor, m->dtype);
}

void OutMat::finish(rnla_ctx* ctx) {
  if (!staged || dev.rows == 0 || dev.cols == 0) {
    RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
    return;
  }
  const size_t es = esize(dst->dtype);
  if (dense_row(dst) && dev.rowmajor()) {
    const int64_t pitch = dst->rows <= 1 ? dst->cols : dst->row_stride;
    RNLA_CUDA(cudaMemcpy2DAsync(dst->data, es * pitch, dev.p, es * dev.cols, es * dev.cols, dev.rows,
                                cudaMemcpyDeviceToHost, ctx->stream));
  } else if (dense_col(dst) && dev.colmajor()) {
    const int64_t pitch = dst->cols <= 1 ? dst->rows : dst->col_stride;
    RNLA_CUDA(cudaMemcpy2DAsync(dst->data, es * pitch, dev.p, es * dev.rows, es * dev.rows, dev.cols,
                                cudaMemcpyDeviceToHost, ctx->stream));
  } else {
    std::vector<char> tmp(es * (size_t)(dev.rows * dev.cols));
    RNLA_CUDA(cudaMemcpyAsync(tmp.data(), dev.p, tmp.size(), cudaMemcpyDeviceToHost, ctx->stream));
    RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
    char* out = static_cast<char*>(dst->data);
    for (int64_t j = 0; j < dev.cols; ++j)
      for (int64_t i = 0; i < dev.rows; ++i)
        std::memcpy(out + es * (size_t)(i * dst->row_stride + j * dst->col_stride),
                    &tmp[es * (size_t)(i * dev.rs + j * dev.cs)], es);
  }
  RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
}

}  // namespace rnla

using namespace rnla;

extern "C" {

int rnla_abi_version(void) { return RNLA_ABI_VERSION; }

const char* rnla_last_error(void) { return g_last_error.c_str(); }

static void ctx_init(rnla_ctx* c, int device) {
  int count = 0;
  RNLA_CUDA(cudaGetDeviceCount(&count));
  require(device >= 0 && device < count, "rnla_ctx_create: no CUDA device " + std::to_string(device));
  c->device = device;
  RNLA_CUDA(cudaSetDevice(device));
  RNLA_CUDA(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));
  RNLA_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  RNLA_CUDA(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
  int prio_lo = 0, prio_hi = 0;
  RNLA_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
  // Higher priority: its CTAs are dispatched first when the streaming kernel frees SM slots.
  RNLA_CUDA(cudaStreamCreateWithPriority(&c->aux_stream, cudaStreamNonBlocking, prio_hi));
  cudaMemPool_t pool;
  RNLA_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
  uint64_t thresh = UINT64_MAX;  // keep freed blocks for reuse across calls
  RNLA_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thresh));
  cusolverDnHandle_t h;
  if (cusolverDnCreate(&h) != CUSOLVER_STATUS_SUCCESS) throw CudaError("cusolverDnCreate failed");
  cusolverDnSetStream(h, c->stream);
  c->cusolver = h;
  cublasHandle_t b;
  if (cublasCreate(&b) != CUBLAS_STATUS_SUCCESS) throw CudaError("cublasCreate failed");
  cublasSetStream(b, c->stream);
  c->cublas = b;
}

static void ctx_release(rnla_ctx* ctx) {
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  if (ctx->side) {
    ctx_release(ctx->side.get());
    ctx->side.reset();
  }
  ctx->graphs.clear();
  ctx->cs_plans.clear();
  ctx->gauss_ops.clear();
  ctx->srht_plans.clear();
  cudaStreamSynchronize(ctx->stream);
  if (ctx->nccl) ncclCommDestroy(static_cast<ncclComm_t>(ctx->nccl));
  if (ctx->cusolver) cusolverDnDestroy(static_cast<cusolverDnHandle_t>(ctx->cusolver));
  if (ctx->cublas) cublasDestroy(static_cast<cublasHandle_t>(ctx->cublas));
  ctx->nccl = ctx->cusolver = ctx->cublas = nullptr;
  if (ctx->pinned) cudaFreeHost(ctx->pinned);
  ctx->pinned = nullptr;
  ctx->pinned_bytes = 0;
  if (ctx->caller_ev) cudaEventDestroy(ctx->caller_ev);
  cudaStreamDestroy(ctx->copy_stream);
  cudaStreamDestroy(ctx->aux_stream);
  cudaStreamDestroy(ctx->stream);
}

}  // extern "C"

namespace rnla {
void* pinned_scratch(rnla_ctx* ctx, size_t bytes) {
  if (bytes > ctx->pinned_bytes) {
    RNLA_CUDA(cudaStreamSynchronize(ctx->stream));  // the old buffer may still be a copy target
    if (ctx->pinned) RNLA_CUDA(cudaFreeHost(ctx->pinned));
    ctx->pinned = nullptr;
    ctx->pinned_bytes = 0;
    RNLA_CUDA(cudaHostAlloc(&ctx->pinned, bytes, cudaHostAllocDefault));
    ctx->pinned_bytes = bytes;
  }
  return ctx->pinned;
}

rnla_ctx* side_ctx(rnla_ctx* ctx) {
  std::lock_guard<std::mutex> lk(ctx->mu);
  if (!ctx->side) {
    auto c = std::make_unique<rnla_ctx>();
    ctx_init(c.get(), ctx->device);
    // the main stream of the helper is the high-priority one
    std::swap(c->stream, c->aux_stream);
    cusolverDnSetStream(static_cast<cusolverDnHandle_t>(c->cusolver), c->stream);
    cublasSetStream(static_cast<cublasHandle_t>(c->cublas), c->stream);
    ctx->side = std::move(c);
  }
  return ctx->side.get();
}
}  // namespace rnla

extern "C" {

rnla_status rnla_ctx_create(int device, rnla_ctx** out) {
  return guard([&] {
    require(out != nullptr, "rnla_ctx_create: null out");
    auto c = std::make_unique<rnla_ctx>();
    ctx_init(c.get(), device);
    *out = c.release();
  });
}

rnla_status rnla_group_create(int world, rnla_group** out) {
  return guard([&] {
    require(out != nullptr && world >= 1, "rnla_group_create: bad argument");
    *out = group_create(world);
  });
}

void rnla_group_destroy(rnla_group* group) { group_destroy(group); }

rnla_status rnla_ctx_create_grouped(int device, rnla_group* group, int rank, rnla_ctx** out) {
  return guard([&] {
    require(out != nullptr && group != nullptr, "rnla_ctx_create_grouped: null argument");
    const int world = group_world(group);
    require(rank >= 0 && rank < world, "rnla_ctx_create_grouped: bad rank");
    auto c = std::make_unique<rnla_ctx>();
    ctx_init(c.get(), device);
    c->world = world;
    c->rank = rank;
    c->group = group;
    *out = c.release();
  });
}

rnla_status rnla_nccl_unique_id(void* out128) {
  return guard([&] {
    require(out128 != nullptr, "rnla_nccl_unique_id: null out");
    ncclUniqueId id;
    ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) throw NcclError(std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
    std::memcpy(out128, &id, sizeof(id));
  });
}

rnla_status rnla_ctx_create_dist(int device, int world, int rank, const void* nccl_unique_id, rnla_ctx** out) {
  return guard([&] {
    require(out != nullptr && nccl_unique_id != nullptr, "rnla_ctx_create_dist: null argument");
    require(world >= 1 && rank >= 0 && rank < world, "rnla_ctx_create_dist: bad rank/world");
    auto c = std::make_unique<rnla_ctx>();
    ctx_init(c.get(), device);
    c->world = world;
    c->rank = rank;
    {  // world 1 too: a one-rank communicator runs the sharded paths over NCCL
      ncclUniqueId id;
      std::memcpy(&id, nccl_unique_id, sizeof(id));
      ncclComm_t comm;
      ncclResult_t r = ncclCommInitRank(&comm, world, id, rank);
      if (r != ncclSuccess) throw NcclError(std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
      c->nccl = comm;
    }
    *out = c.release();
  });
}

void rnla_ctx_destroy(rnla_ctx* ctx) {
  if (!ctx) return;
  ctx_release(ctx);
  delete ctx;
}

rnla_status rnla_ctx_synchronize(rnla_ctx* ctx) {
  return guard([&] {
    enter(ctx);
    RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

rnla_status rnla_ctx_wait_stream(rnla_ctx* ctx, void* stream) {
  return guard([&] {
    enter(ctx);
    if (!ctx->caller_ev) RNLA_CUDA(cudaEventCreateWithFlags(&ctx->caller_ev, cudaEventDisableTiming));
    RNLA_CUDA(cudaEventRecord(ctx->caller_ev, static_cast<cudaStream_t>(stream)));
    RNLA_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->caller_ev, 0));
  });
}

void* rnla_ctx_stream(rnla_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

int64_t rnla_ctx_launch_count(rnla_ctx* ctx) { return ctx ? ctx->launches : 0; }

void rnla_ctx_clear_cache(rnla_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  ctx->graphs.clear();
  ctx->cs_plans.clear();
  ctx->gauss_ops.clear();
  ctx->srht_plans.clear();
  ctx->landmark_sel.clear();
  cudaStreamSynchronize(ctx->stream);
}

void rnla_shard_rows(int64_t n, int world, int rank, int64_t* begin, int64_t* end) {
  if (world < 1) world = 1;
  const int64_t base = n / world, rem = n % world;
  const int64_t b = rank * base + std::min<int64_t>(rank, rem);
  *begin = b;
  *end = b + base + (rank < rem ? 1 : 0);
}

uint64_t rnla_splitmix64(uint64_t* state) { return splitmix64(*state); }

uint64_t rnla_derive_seed(uint64_t seed, uint64_t stream) { return derive_seed(seed, stream); }

rnla_status rnla_count_sketch_hashes(uint64_t seed, int64_t j0, int64_t n, int64_t s, int64_t* buckets,
                                     int8_t* signs) {
  return guard([&] {
    require(s >= 1, "count_sketch: s < 1");
    require(n >= 0 && (n == 0 || (buckets && signs)), "count_sketch_hashes: null output");
    for (int64_t j = 0; j < n; ++j) {
      uint64_t state = seed ^ (0xa0761d6478bd642fULL + (uint64_t)(j0 + j) * 0xe7037ed1a0b428dbULL);
      const uint64_t h1 = splitmix64(state), h2 = splitmix64(state);
      buckets[j] = (int64_t)(h1 % (uint64_t)s);
      signs[j] = (h2 & 1ULL) ? 1 : -1;
    }
  });
}

rnla_status rnla_gaussian_matrix(uint64_t seed, int64_t rows, int64_t cols, double* out) {
  return guard([&] {
    require(rows >= 0 && cols >= 0 && (rows * cols == 0 || out), "gaussian_matrix: bad arguments");
    gaussian_matrix_host(seed, rows, cols, out);
  });
}

rnla_status rnla_sample_without_replacement(uint64_t seed, int64_t n, int64_t count, int64_t* out) {
  return guard([&] {
    auto v = sample_without_replacement_host(seed, n, count);
    require(count == 0 || out, "sample_without_replacement: null output");
    std::copy(v.begin(), v.end(), out);
  });
}

rnla_status rnla_sample_with_replacement(uint64_t seed, const double* weights, int64_t n, int64_t count,
                                         int64_t* out) {
  return guard([&] {
    require(weights && out, "sample_with_replacement: null argument");
    auto v = sample_with_replacement_host(seed, weights, n, count);
    std::copy(v.begin(), v.end(), out);
  });
}

rnla_status rnla_srht_operator(uint64_t seed, int64_t n, int64_t s, int8_t* signs, int64_t* idx) {
  return guard([&] {
    require(signs && idx, "srht_operator: null output");
    srht_operator_host(seed, n, s, signs, idx);
  });
}

}  // extern "C"
