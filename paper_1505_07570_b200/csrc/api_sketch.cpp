// api_sketch.cpp -- sketch operators and sketched least squares behind the C ABI.
//
// Reference semantics (/root/reference/proj):
//   gaussian_sketch     src/sketch.cpp:36-42     C = A * (G / sqrt(s)), G = gaussian_matrix(n, s)
//   srht_sketch         src/sketch.cpp:57-81
//   count_sketch        src/sketch.cpp:83-97
//   combined_sketch     src/sketch.cpp:108-123
//   apply_sketch        src/sketch.cpp:177-197
//   sketch_rows         src/regression.cpp:17-19 (S^T M = apply_sketch(M^T)^T)
//   lsr_sketched        src/regression.cpp:68-92
// A column sketch C = A*S of a column-major m x n A treats the n columns as
// contiguous segments of length m; a row sketch S^T M of a row-major n x d M
// treats its rows as segments of length d. Both run the same kernels.
#include <cublas_v2.h>

#include <cmath>

#include "dist.h"
#include "linalg.cuh"
#include "marshal.h"
#include "srht.h"
#include "algos.h"

namespace rnla {

// G / sqrt(s) for gaussian_matrix(n, s) from make_rng(seed), column-major n x s,
// device-resident and cached. fp32 operators are the fp64 values rounded once.
const DenseOperator& gaussian_operator(rnla_ctx* ctx, int64_t n, int64_t s, uint64_t seed, int dtype) {
  auto key = std::make_tuple(n, s, seed, dtype);
  auto it = ctx->gauss_ops.find(key);
  if (it != ctx->gauss_ops.end()) return *it->second;
  std::vector<double> g((size_t)(n * s));
  gaussian_matrix_host(seed, n, s, g.data());
  auto op = std::make_unique<DenseOperator>();
  op->rows = n; op->cols = s; op->dtype = dtype;
  DevBuf d64(sizeof(double) * g.size(), ctx->stream);
  RNLA_CUDA(cudaMemcpyAsync(d64.p, g.data(), sizeof(double) * g.size(), cudaMemcpyHostToDevice, ctx->stream));
  scale_inplace<double>(ctx, d64.as<double>(), n * s, std::sqrt(static_cast<double>(s)));  // g / sqrt(s)
  if (dtype == RNLA_F64) {
    op->data = std::move(d64);
  } else {
    op->data = DevBuf(sizeof(float) * g.size(), ctx->stream);
    copy2d_cast<double, float>(ctx, n * s, 1, d64.as<double>(), 1, 1, op->data.as<float>(), 1, 1);
  }
  RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
  auto& ref = *op;
  ctx->gauss_ops.emplace(key, std::move(op));
  return ref;
}

std::shared_ptr<SrhtPlan> srht_plan(rnla_ctx* ctx, int64_t n, int64_t s, uint64_t seed) {
  auto key = std::make_tuple(n, s, seed);
  auto it = ctx->srht_plans.find(key);
  if (it != ctx->srht_plans.end()) return it->second;
  auto p = std::make_shared<SrhtPlan>(ctx, n, s, seed);
  ctx->srht_plans.emplace(key, p);
  return p;
}

// ---- segment-form operators: n segments of length L (segment j at in + j*ld)
// to s segments (segment t at out + t*out_rs, element c at + c*out_cs). ----

// The Gaussian stage out(t, c) = sum_j Gs(j, t) in(j, c) (A = Gs^T, Gs col-major
// n x s) is accumulated over canonical K-chunks of kGaussKC segments in
// chunk order, one GEMM launch per chunk. The standalone call and the
// pipelined combined sketch (which runs chunk c while the count sketch
// produces chunk c+1) therefore produce bit-identical results, keeping
// combined == gaussian(count) exact (tests/test_sketch.cpp:88-98).
// Canonical K-chunk: the whole K on one GPU (measured: splitting the
// Gaussian stage under the count sketch does not overlap, the gather kernel
// holds the register file), s / world on a row-sharded job so each rank
// multiplies the chunks it owns after a per-chunk ncclReduce.
// One GPU, K >= 2 kOneGpuKC: chunks of kOneGpuKC, so the pipelined combined
// sketch can multiply chunk c while the gather produces chunk c + 1 (measured
// on config 1 with split-K per chunk: 3.29 -> 3.24 ms per step at 2048, 3.34 ms
// at 4096; without split-K: 3.17 ms at 2048, 3.16 ms at 1024).
static constexpr int64_t kOneGpuKC = 1024;
// whole: the fp64 stage runs on the int8 tensor cores (ozaki.cu). There it
// takes one launch over the whole K after the count sketch: the digit GEMM
// does not share SMs with the gather (its CTAs need most of an SM's shared
// memory and registers), and at 4.5 POPS the exposed stage is short
// (config 1: 0.57 ms of DMMA -> ~0.13 ms).
static int64_t gauss_kc_for(const rnla_ctx* ctx, int64_t k, bool whole) {
  const int64_t w = std::max(1, ctx->world);
  if (w == 1 && whole && k <= 16384) return std::max<int64_t>(16, k);
  if (w == 1 && k >= 2 * kOneGpuKC) return kOneGpuKC;
  return std::max<int64_t>(16, (k + w - 1) / w);
}

// the Gaussian stage of T-typed data with s outputs and L segments takes the Ozaki path
template <class T>
static bool gauss_whole(int64_t s, int64_t L) {
  return std::is_same<T, double>::value && ozaki_applies(s, L);
}

// Row pitch (elements) rounded up to 16 bytes.
template <class T>
static int64_t aligned_ld(int64_t L) {
  const int64_t e = 16 / (int64_t)sizeof(T);
  return (L + e - 1) / e * e;
}

template <class T>
void gaussian_chunk(rnla_ctx* ctx, const DenseOperator& g, const T* in, int64_t ld, int64_t n, int64_t L, int64_t s,
                    int64_t k0, bool first, T* out, int64_t out_rs, int64_t out_cs) {
  const int64_t kc = std::min(gauss_kc_for(ctx, n, gauss_whole<T>(s, L)), n - k0);
  // Chunked stages run each chunk without split-K (one CTA per output tile):
  // under the gather that interferes least (config 1: 3.24 -> 3.16 ms). The
  // standalone and the combined stage chunk identically, so the composition
  // stays bitwise.
  const int max_splits = gauss_kc_for(ctx, n, gauss_whole<T>(s, L)) < n ? 1 : 64;
  // fp64: the exact int8 digit split on the tensor cores (ozaki.cu), the same
  // for the standalone and the combined stage
  if constexpr (std::is_same<T, double>::value)
    if (ozaki_gaussian_chunk(ctx, g, in, ld, n, L, s, k0, kc, !first, out, out_rs, out_cs)) return;
  gemm<T>(ctx, s, L, kc, T(1), g.data.as<T>() + k0, n, 1, in + k0 * ld, ld, 1, first ? T(0) : T(1), out, out_rs,
          out_cs, max_splits);
}

template <class T>
void gaussian_segments(rnla_ctx* ctx, const T* in, int64_t ld, int64_t n, int64_t L, int64_t s, uint64_t seed, T* out,
                       int64_t out_rs, int64_t out_cs) {
  const DenseOperator& g = gaussian_operator(ctx, n, s, seed, std::is_same<T, double>::value ? RNLA_F64 : RNLA_F32);
  // fp64 segments whose rows are not 16-B aligned are first copied to padded
  // rows, so every large Gaussian stage runs the cp.async DMMA kernel and a
  // standalone call agrees bitwise with the combined sketch's stage
  // (tests/test_sketch.cpp:88-98).
  DevBuf padded;
  if (std::is_same<T, double>::value && (ld * (int64_t)sizeof(T)) % 16 != 0 && n > 0 && L >= 64 && s >= 64) {
    const int64_t ld2 = aligned_ld<T>(L);
    padded = DevBuf(sizeof(T) * (size_t)(n * ld2), ctx->stream);
    copy2d<T>(ctx, n, L, in, ld, 1, padded.as<T>(), ld2, 1);
    in = padded.as<T>();
    ld = ld2;
  }
  if (n == 0) {  // empty sum
    DevBuf z(sizeof(T) * (size_t)std::max<int64_t>(s * L, 1), ctx->stream);
    RNLA_CUDA(cudaMemsetAsync(z.p, 0, sizeof(T) * (size_t)(s * L), ctx->stream));
    copy2d<T>(ctx, s, L, z.as<T>(), L, 1, out, out_rs, out_cs);
    return;
  }
  const int64_t kc = gauss_kc_for(ctx, n, gauss_whole<T>(s, L));
  for (int64_t k0 = 0; k0 < n; k0 += kc) gaussian_chunk<T>(ctx, g, in, ld, n, L, s, k0, k0 == 0, out, out_rs, out_cs);
}

// Combined count -> Gaussian row sketch with the Gaussian stage pipelined
// under the count sketch: bucket chunk c is gathered on the main stream while
// the aux stream (higher priority) multiplies chunk c-1 on the DMMA units.
// Row-sharded contexts reduce each finished chunk onto an owner rank
// (c % world, ncclReduce), the owner multiplies it, and one allreduce of the
// s2 x Lo result finishes (SURVEY §7 hard part 10).
template <class T>
void combined_gaussian_pipelined(rnla_ctx* ctx, const T* M, int64_t ld, const T* extra, int64_t xs, int64_t n,
                                 int64_t L, const rnla_sketch_spec* spec, int64_t row_offset, T* out, int64_t o_rs,
                                 int64_t o_cs) {
  const int dt = std::is_same<T, double>::value ? RNLA_F64 : RNLA_F32;
  const int64_t Lo = L + (extra ? 1 : 0), s = spec->s, s2 = spec->stage2_s;
  const DenseOperator& g = gaussian_operator(ctx, s, s2, spec->stage2_seed, dt);
  if (n > 0) count_sketch_plan(ctx, n, s, spec->seed, row_offset);
  const int64_t ldm = aligned_ld<T>(Lo);
  DevBuf mid(sizeof(T) * (size_t)(s * ldm), ctx->stream);
  DevBuf acc(sizeof(T) * (size_t)(s2 * Lo), ctx->stream);
  const int64_t KC = gauss_kc_for(ctx, s, gauss_whole<T>(s2, Lo));
  const int64_t chunks = (s + KC - 1) / KC;
  std::vector<cudaEvent_t> ev((size_t)chunks + 2);
  for (auto& e : ev) RNLA_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  cudaEvent_t start = ev[(size_t)chunks], done = ev[(size_t)chunks + 1];
  RNLA_CUDA(cudaEventRecord(start, ctx->stream));
  cudaStream_t gemm_st = ctx->aux_stream;
  cudaStream_t gather_st[2] = {ctx->stream, ctx->copy_stream};
  RNLA_CUDA(cudaStreamWaitEvent(gemm_st, start, 0));
  RNLA_CUDA(cudaStreamWaitEvent(gather_st[0], start, 0));
  RNLA_CUDA(cudaStreamWaitEvent(gather_st[1], start, 0));
  bool first = true;
  // Gather chunks alternate between two streams so one chunk's last partial
  // wave overlaps the next chunk instead of draining the GPU.
  try {
    for (int64_t c = 0; c < chunks; ++c) {
      const int64_t b0 = c * KC, b1 = std::min(s, b0 + KC);
      {
        StreamScope on_gather(ctx, gather_st[c & 1]);
        count_sketch_segments<T>(ctx, M, ld, extra, xs, n, L, s, spec->seed, row_offset, mid.as<T>(), ldm, false, b0,
                                 b1);
        RNLA_CUDA(cudaEventRecord(ev[(size_t)c], ctx->stream));
      }
    }
    for (int64_t c = 0; c < chunks; ++c) {
      const int64_t b0 = c * KC, b1 = std::min(s, b0 + KC);
      RNLA_CUDA(cudaStreamWaitEvent(gemm_st, ev[(size_t)c], 0));
      StreamScope on_aux(ctx, gemm_st);
      const int owner = (int)(c % ctx->world);
      if (is_sharded(ctx)) reduce_to(ctx, mid.as<T>() + b0 * ldm, (size_t)((b1 - b0) * ldm), dt, owner);
      if (owner == ctx->rank) {
        gaussian_chunk<T>(ctx, g, mid.as<T>(), ldm, s, Lo, s2, b0, first, acc.as<T>(), Lo, 1);
        first = false;
      }
    }
    if (first) RNLA_CUDA(cudaMemsetAsync(acc.p, 0, sizeof(T) * (size_t)(s2 * Lo), gemm_st));
    RNLA_CUDA(cudaEventRecord(done, gemm_st));
    RNLA_CUDA(cudaStreamWaitEvent(ctx->stream, done, 0));
    // the gather streams' last chunks are covered by the GEMM dependencies
  } catch (...) {
    cudaStreamSynchronize(gemm_st);
    cudaStreamSynchronize(gather_st[0]);
    cudaStreamSynchronize(gather_st[1]);
    cudaStreamSynchronize(ctx->aux_stream);
    for (auto& e : ev) cudaEventDestroy(e);
    throw;
  }
  for (auto& e : ev) cudaEventDestroy(e);  // destruction is deferred until the events complete
  if (is_sharded(ctx)) allreduce_sum(ctx, acc.p, (size_t)(s2 * Lo), dt);
  copy2d<T>(ctx, s2, Lo, acc.as<T>(), Lo, 1, out, o_rs, o_cs);
}

template <class T>
void dense_stage(rnla_ctx* ctx, int kind, const T* in, int64_t ld, int64_t n, int64_t L, int64_t s, uint64_t seed,
                 T* out, int64_t out_rs, int64_t out_cs) {
  if (kind == RNLA_SKETCH_GAUSSIAN) {
    gaussian_segments<T>(ctx, in, ld, n, L, s, seed, out, out_rs, out_cs);
  } else if (kind == RNLA_SKETCH_SRHT) {
    auto plan = srht_plan(ctx, n, s, seed);
    srht_segments<T>(ctx, *plan, in, ld, L, out, out_rs, out_cs);
  } else {
    throw InvalidArgument("combined_sketch: stage2 must be gaussian or srht");
  }
}

static int64_t final_size(const rnla_sketch_spec* spec) {
  return spec->kind == RNLA_SKETCH_COMBINED ? spec->stage2_s : spec->s;
}

static void check_spec(const rnla_sketch_spec* spec) {
  require(spec != nullptr, "null SketchSpec");
  require(spec->s >= 1, "sketch: s < 1");
  if (spec->kind == RNLA_SKETCH_COMBINED) {
    require(spec->stage2_kind == RNLA_SKETCH_GAUSSIAN || spec->stage2_kind == RNLA_SKETCH_SRHT,
            "combined_sketch: stage2 must be gaussian or srht");
    require(spec->stage2_s >= 1, "sketch: s < 1");
    require(spec->stage2_s <= spec->s, "combined_sketch: s > s_cs");
  }
}

// Row sketch of a row-major tall M (segments = rows, length L (+1 with extra))
// into out (s_final x Lo, element (t, c) at out[t*o_rs + c*o_cs]).
template <class T>
void sketch_rows_dev(rnla_ctx* ctx, const T* M, int64_t ld, const T* extra, int64_t xs, int64_t n, int64_t L,
                     const rnla_sketch_spec* spec, int64_t row_offset, T* out, int64_t o_rs, int64_t o_cs) {
  const int64_t Lo = L + (extra ? 1 : 0);
  const int kind = spec->kind;
  const bool sharded = is_sharded(ctx);
  const bool chunked = spec->kind == RNLA_SKETCH_COMBINED &&
                       gauss_kc_for(ctx, spec->s, gauss_whole<T>(spec->stage2_s, Lo)) < spec->s;
  if (kind == RNLA_SKETCH_COMBINED && spec->stage2_kind == RNLA_SKETCH_GAUSSIAN &&
      (sharded || chunked)) {
    combined_gaussian_pipelined<T>(ctx, M, ld, extra, xs, n, L, spec, row_offset, out, o_rs, o_cs);
    return;
  }
  if (kind == RNLA_SKETCH_COUNT || kind == RNLA_SKETCH_COMBINED) {
    const int64_t s = spec->s;
    const bool direct = kind == RNLA_SKETCH_COUNT && o_cs == 1;
    DevBuf mid;
    T* mp = out;
    int64_t m_rs = o_rs;
    if (!direct) {
      // rows padded to 16 B so the Gaussian stage reads them with cp.async (gemm_dmma.cu)
      m_rs = aligned_ld<T>(Lo);
      mid = DevBuf(sizeof(T) * (size_t)(s * m_rs), ctx->stream);
      mp = mid.as<T>();
    }
    count_sketch_segments<T>(ctx, M, ld, extra, xs, n, L, s, spec->seed, row_offset, mp, m_rs, false);
    if (sharded) allreduce_sum(ctx, mp, (size_t)(s * m_rs), std::is_same<T, double>::value ? RNLA_F64 : RNLA_F32);
    if (kind == RNLA_SKETCH_COUNT) {
      if (!direct) copy2d<T>(ctx, s, Lo, mp, m_rs, 1, out, o_rs, o_cs);
      return;
    }
    dense_stage<T>(ctx, spec->stage2_kind, mp, m_rs, s, Lo, spec->stage2_s, spec->stage2_seed, out, o_rs, o_cs);
    return;
  }
  if (kind == RNLA_SKETCH_SRHT && sharded) {
    require(extra == nullptr, "sketch_rows: an appended column is supported for count and combined sketches");
    int64_t n_total = n;
    const int64_t off = global_row_offset(ctx, n, &n_total);
    require(off == row_offset, "sketch_rows: row_offset differs from the shard layout (rnla_shard_rows order)");
    srht_rows_sharded<T>(ctx, M, ld, n, L, off, n_total, spec->s, spec->seed, out, o_rs, o_cs);
    return;
  }
  require(!sharded && row_offset == 0,
          "sketch_rows: row sharding is supported for count, combined (count-first) and SRHT sketches");
  require(extra == nullptr, "sketch_rows: an appended column is supported for count and combined sketches");
  if (kind == RNLA_SKETCH_GAUSSIAN || kind == RNLA_SKETCH_SRHT) {
    dense_stage<T>(ctx, kind, M, ld, n, L, spec->s, spec->seed, out, o_rs, o_cs);
    return;
  }
  throw InvalidArgument("sketch_rows: unsupported sketch kind for a row sketch");
}

// Host-resident tall M streamed through the device in row chunks: H2D of
// chunk i+1 overlaps the count sketch of chunk i; chunks accumulate in row
// order so the per-bucket order (and fp64 bits) match the single-pass loop.
template <class T>
void count_rows_streamed(rnla_ctx* ctx, const rnla_mat* m, const rnla_mat* extra, int64_t s, uint64_t seed,
                         int64_t row_offset, T* out, int64_t ldo) {
  const int64_t n = m->rows, L = m->cols;
  const int64_t row_bytes = (int64_t)sizeof(T) * (L + (extra ? 1 : 0));
  int64_t chunk = std::max<int64_t>(1, ((int64_t)256 << 20) / std::max<int64_t>(row_bytes, 1));
  if (const char* env = std::getenv("RNLA_STREAM_CHUNK_ROWS")) chunk = std::max<int64_t>(1, std::atoll(env));
  chunk = std::min(chunk, n);
  DevBuf buf[2] = {DevBuf(sizeof(T) * (size_t)(chunk * L), ctx->stream),
                   DevBuf(sizeof(T) * (size_t)(chunk * L), ctx->stream)};
  DevBuf xbuf[2];
  if (extra) {
    xbuf[0] = DevBuf(sizeof(T) * (size_t)chunk, ctx->stream);
    xbuf[1] = DevBuf(sizeof(T) * (size_t)chunk, ctx->stream);
  }
  cudaEvent_t copied[2], consumed[2];
  for (int i = 0; i < 2; ++i) {
    RNLA_CUDA(cudaEventCreateWithFlags(&copied[i], cudaEventDisableTiming));
    RNLA_CUDA(cudaEventCreateWithFlags(&consumed[i], cudaEventDisableTiming));
    RNLA_CUDA(cudaEventRecord(consumed[i], ctx->stream));
  }
  RNLA_CUDA(cudaStreamSynchronize(ctx->stream));  // buffers allocated before the copy stream uses them
  const char* base = static_cast<const char*>(m->data);
  const char* xbase = extra ? static_cast<const char*>(extra->data) : nullptr;
  int64_t chunk_idx = 0;
  try {
    for (int64_t r0 = 0; r0 < n; r0 += chunk, ++chunk_idx) {
      const int64_t rows = std::min(chunk, n - r0);
      const int b = (int)(chunk_idx & 1);
      RNLA_CUDA(cudaStreamWaitEvent(ctx->copy_stream, consumed[b], 0));
      RNLA_CUDA(cudaMemcpy2DAsync(buf[b].p, sizeof(T) * L, base + sizeof(T) * (size_t)(r0 * m->row_stride),
                                  sizeof(T) * m->row_stride, sizeof(T) * L, rows, cudaMemcpyHostToDevice,
                                  ctx->copy_stream));
      if (extra)
        RNLA_CUDA(cudaMemcpy2DAsync(xbuf[b].p, sizeof(T), xbase + sizeof(T) * (size_t)(r0 * extra->row_stride),
                                    sizeof(T) * extra->row_stride, sizeof(T), rows, cudaMemcpyHostToDevice,
                                    ctx->copy_stream));
      RNLA_CUDA(cudaEventRecord(copied[b], ctx->copy_stream));
      RNLA_CUDA(cudaStreamWaitEvent(ctx->stream, copied[b], 0));
      count_sketch_segments<T>(ctx, buf[b].as<T>(), L, extra ? xbuf[b].as<T>() : nullptr, 1, rows, L, s, seed,
                               row_offset + r0, out, ldo, r0 > 0);
      RNLA_CUDA(cudaEventRecord(consumed[b], ctx->stream));
    }
  } catch (...) {
    cudaStreamSynchronize(ctx->copy_stream);
    cudaStreamSynchronize(ctx->stream);
    for (int i = 0; i < 2; ++i) { cudaEventDestroy(copied[i]); cudaEventDestroy(consumed[i]); }
    throw;
  }
  RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
  for (int i = 0; i < 2; ++i) { cudaEventDestroy(copied[i]); cudaEventDestroy(consumed[i]); }
}

template <class T>
void sketch_rows_entry(rnla_ctx* ctx, const rnla_mat* m, const rnla_mat* extra, const rnla_sketch_spec* spec,
                       int64_t row_offset, const rnla_mat* out) {
  const int64_t n = m->rows, L = m->cols, Lo = L + (extra ? 1 : 0);
  OutMat o(ctx, out, final_size(spec), Lo, "sketch_rows output", true);
  require(o.dev.dtype == m->dtype, "sketch_rows: output dtype differs from input dtype");
  const bool host_rowmajor = !m->on_device && m->col_stride == 1 && (!extra || !extra->on_device);
  if (host_rowmajor && (spec->kind == RNLA_SKETCH_COUNT || spec->kind == RNLA_SKETCH_COMBINED) && n > 0) {
    const int64_t s = spec->s;
    DevBuf mid(sizeof(T) * (size_t)(s * Lo), ctx->stream);
    count_rows_streamed<T>(ctx, m, extra, s, spec->seed, row_offset, mid.as<T>(), Lo);
    if (is_sharded(ctx)) allreduce_sum(ctx, mid.p, (size_t)(s * Lo), m->dtype);
    if (spec->kind == RNLA_SKETCH_COUNT)
      copy2d<T>(ctx, s, Lo, mid.as<T>(), Lo, 1, o.dev.as<T>(), o.dev.rs, o.dev.cs);
    else
      dense_stage<T>(ctx, spec->stage2_kind, mid.as<T>(), Lo, s, Lo, spec->stage2_s, spec->stage2_seed,
                     o.dev.as<T>(), o.dev.rs, o.dev.cs);
    o.finish(ctx);
    return;
  }
  DevMat dm = as_rowmajor(ctx, to_device(ctx, m));
  DevMat dx;
  const T* xp = nullptr;
  int64_t xs = 1;
  if (extra) {
    dx = to_device(ctx, extra);
    xp = dx.as<T>();
    xs = dx.rs;
  }
  sketch_rows_dev<T>(ctx, dm.as<T>(), dm.rs, xp, xs, n, L, spec, row_offset, o.dev.as<T>(), o.dev.rs, o.dev.cs);
  o.finish(ctx);
}

// Column sketch C = A * S of an m x n A: segments are the columns of A.
template <class T>
void apply_columns(rnla_ctx* ctx, const rnla_mat* a, const rnla_sketch_spec* spec, const rnla_mat* c) {
  const int64_t m = a->rows, n = a->cols;
  OutMat o(ctx, c, m, final_size(spec), "sketch output", false);
  require(o.dev.dtype == a->dtype, "sketch: output dtype differs from input dtype");
  DevMat da = as_colmajor(ctx, to_device(ctx, a));  // columns contiguous
  // Output segment t = column t of C: element (t, c) at C[c*rs + t*cs].
  const int kind = spec->kind;
  if (kind == RNLA_SKETCH_COUNT || kind == RNLA_SKETCH_COMBINED) {
    const int64_t s = spec->s;
    const bool direct = kind == RNLA_SKETCH_COUNT && o.dev.rs == 1;
    DevBuf mid;
    T* mp = o.dev.as<T>();
    int64_t ldm = o.dev.cs;
    if (!direct) {
      mid = DevBuf(sizeof(T) * (size_t)(s * m), ctx->stream);
      mp = mid.as<T>();
      ldm = m;
    }
    count_sketch_segments<T>(ctx, da.as<T>(), da.cs, nullptr, 1, n, m, s, spec->seed, 0, mp, ldm, false);
    if (kind == RNLA_SKETCH_COUNT) {
      if (!direct) copy2d<T>(ctx, s, m, mp, m, 1, o.dev.as<T>(), o.dev.cs, o.dev.rs);
    } else {
      dense_stage<T>(ctx, spec->stage2_kind, mp, ldm, s, m, spec->stage2_s, spec->stage2_seed, o.dev.as<T>(),
                     o.dev.cs, o.dev.rs);
    }
  } else if (kind == RNLA_SKETCH_GAUSSIAN || kind == RNLA_SKETCH_SRHT) {
    dense_stage<T>(ctx, kind, da.as<T>(), da.cs, n, m, spec->s, spec->seed, o.dev.as<T>(), o.dev.cs, o.dev.rs);
  } else {
    throw InvalidArgument("apply_sketch: unsupported kind for this entry point");
  }
  o.finish(ctx);
}

template void sketch_rows_dev<double>(rnla_ctx*, const double*, int64_t, const double*, int64_t, int64_t, int64_t,
                                      const rnla_sketch_spec*, int64_t, double*, int64_t, int64_t);

}  // namespace rnla

using namespace rnla;

static rnla_sketch_spec simple_spec(int kind, int64_t s, uint64_t seed) {
  rnla_sketch_spec sp{};
  sp.kind = kind; sp.s = s; sp.seed = seed;
  return sp;
}

extern "C" {

int64_t rnla_sketch_output_cols(const rnla_sketch_spec* spec, int64_t n) {
  if (!spec) return -1;
  (void)n;
  return spec->kind == RNLA_SKETCH_COMBINED ? spec->stage2_s : spec->s;
}

rnla_status rnla_gaussian_sketch(rnla_ctx* ctx, const rnla_mat* a, int64_t s, uint64_t seed, rnla_mat* c) {
  return guard([&] {
    enter(ctx);
    require(s >= 1, "gaussian_sketch: s < 1");
    check_mat(a, "gaussian_sketch: a");
    rnla_sketch_spec sp = simple_spec(RNLA_SKETCH_GAUSSIAN, s, seed);
    if (a->dtype == RNLA_F64) apply_columns<double>(ctx, a, &sp, c);
    else apply_columns<float>(ctx, a, &sp, c);
  });
}

rnla_status rnla_srht_sketch(rnla_ctx* ctx, const rnla_mat* a, int64_t s, uint64_t seed, rnla_mat* c) {
  return guard([&] {
    enter(ctx);
    check_mat(a, "srht_sketch: a");
    require(s >= 1 && s <= next_pow2(a->cols), "srht_sketch: s > padded dimension");
    rnla_sketch_spec sp = simple_spec(RNLA_SKETCH_SRHT, s, seed);
    if (a->dtype == RNLA_F64) apply_columns<double>(ctx, a, &sp, c);
    else apply_columns<float>(ctx, a, &sp, c);
  });
}

rnla_status rnla_count_sketch(rnla_ctx* ctx, const rnla_mat* a, int64_t s, uint64_t seed, rnla_mat* c) {
  return guard([&] {
    enter(ctx);
    require(s >= 1, "count_sketch: s < 1");
    check_mat(a, "count_sketch: a");
    rnla_sketch_spec sp = simple_spec(RNLA_SKETCH_COUNT, s, seed);
    if (a->dtype == RNLA_F64) apply_columns<double>(ctx, a, &sp, c);
    else apply_columns<float>(ctx, a, &sp, c);
  });
}

rnla_status rnla_combined_sketch(rnla_ctx* ctx, const rnla_mat* a, const rnla_sketch_spec* spec, rnla_mat* c) {
  return guard([&] {
    enter(ctx);
    require(spec != nullptr && spec->kind == RNLA_SKETCH_COMBINED,
            "combined_sketch: spec is not a combined sketch");
    check_spec(spec);
    check_mat(a, "combined_sketch: a");
    if (a->dtype == RNLA_F64) apply_columns<double>(ctx, a, spec, c);
    else apply_columns<float>(ctx, a, spec, c);
  });
}

rnla_status rnla_sketch_rows(rnla_ctx* ctx, const rnla_mat* m, const rnla_mat* extra, const rnla_sketch_spec* spec,
                             int64_t row_offset, rnla_mat* out) {
  return guard([&] {
    enter(ctx);
    check_spec(spec);
    check_mat(m, "sketch_rows: m");
    if (extra) {
      check_mat(extra, "sketch_rows: extra");
      require(extra->rows == m->rows && extra->cols == 1, "sketch_rows: extra must be n x 1");
      require(extra->dtype == m->dtype, "sketch_rows: extra dtype differs");
    }
    require(row_offset >= 0, "sketch_rows: negative row offset");
    if (m->dtype == RNLA_F64) sketch_rows_entry<double>(ctx, m, extra, spec, row_offset, out);
    else sketch_rows_entry<float>(ctx, m, extra, spec, row_offset, out);
  });
}

}  // extern "C"

// ---- lsr_sketched (src/regression.cpp:68-92) ----
namespace rnla {

// Solve min ||a_sk x - b_sk|| for a column-major s x d a_sk (device, fp64):
// Householder QR, rank test on the singular values of R with the reference's
// 1e-10 threshold (numerical_rank, src/regression.cpp:21-25), then R^-1 Q' b
// (full rank) or pinv(R) Q' b with the 1e-12 pseudo_inverse cut (flagged).
static void solve_sketched(rnla_ctx* ctx, int64_t s, int64_t d, double* a_sk, const double* b_sk, double* x_dev,
                           int32_t* flagged) {
  if (s < d) {
    // The final sketch has fewer rows than d (a combined spec with stage2.s < d
    // passes the reference's spec.s >= d check, src/regression.cpp:73): rank <= s < d,
    // so the reference takes its flagged pinv(a_sk) b_sk route (:84-89).
    *flagged = 1;
    DevBuf u(sizeof(double) * s * s, ctx->stream), v(sizeof(double) * d * s, ctx->stream),
        sv(sizeof(double) * std::max<int64_t>(s, 1), ctx->stream), w(sizeof(double) * std::max<int64_t>(s, 1), ctx->stream);
    if (s == 0) {
      RNLA_CUDA(cudaMemsetAsync(x_dev, 0, sizeof(double) * d, ctx->stream));
      return;
    }
    svd_thin(ctx, s, d, a_sk, 1, s, u.as<double>(), sv.as<double>(), v.as<double>());  // a_sk = U S V'
    gemm<double>(ctx, s, 1, s, 1.0, u.as<double>(), s, 1, b_sk, 1, 1, 0.0, w.as<double>(), 1, 1);  // U' b
    std::vector<double> hs(s), hw(s);
    RNLA_CUDA(cudaMemcpyAsync(hs.data(), sv.p, sizeof(double) * s, cudaMemcpyDeviceToHost, ctx->stream));
    RNLA_CUDA(cudaMemcpyAsync(hw.data(), w.p, sizeof(double) * s, cudaMemcpyDeviceToHost, ctx->stream));
    RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
    for (int64_t i = 0; i < s; ++i) hw[i] = hs[i] > 1e-12 * hs[0] ? hw[i] / hs[i] : 0.0;
    RNLA_CUDA(cudaMemcpyAsync(w.p, hw.data(), sizeof(double) * s, cudaMemcpyHostToDevice, ctx->stream));
    gemm<double>(ctx, d, 1, s, 1.0, v.as<double>(), 1, d, w.as<double>(), 1, 1, 0.0, x_dev, 1, 1);  // V (S^-1 U' b)
    RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
    return;
  }
  DevBuf r(sizeof(double) * d * d, ctx->stream);
  qr_householder(ctx, s, d, a_sk, r.as<double>(), 1, d);  // a_sk <- Q (s x d), r col-major
  DevBuf qtb(sizeof(double) * d, ctx->stream);
  gemm<double>(ctx, d, 1, s, 1.0, a_sk, s, 1, b_sk, 1, 1, 0.0, qtb.as<double>(), 1, 1);  // Q' b
  DevBuf u(sizeof(double) * d * d, ctx->stream), v(sizeof(double) * d * d, ctx->stream), sv(sizeof(double) * d,
                                                                                             ctx->stream);
  svd_thin(ctx, d, d, r.as<double>(), 1, d, u.as<double>(), sv.as<double>(), v.as<double>());
  std::vector<double> hs(d);
  RNLA_CUDA(cudaMemcpyAsync(hs.data(), sv.p, sizeof(double) * d, cudaMemcpyDeviceToHost, ctx->stream));
  RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
  int64_t rank = 0;
  for (int64_t i = 0; i < d; ++i) rank += hs[i] > 1e-10 * hs[0];
  if (d > 0 && rank == d) {
    *flagged = 0;
    RNLA_CUDA(cudaMemcpyAsync(x_dev, qtb.p, sizeof(double) * d, cudaMemcpyDeviceToDevice, ctx->stream));
    const double one = 1.0;
    cublasStatus_t st = cublasDtrsm(static_cast<cublasHandle_t>(ctx->cublas), CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_UPPER,
                                    CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, (int)d, 1, &one, r.as<double>(), (int)d, x_dev,
                                    (int)d);
    if (st != CUBLAS_STATUS_SUCCESS) throw CudaError("cublasDtrsm failed");
    note_launch(ctx);
  } else {
    *flagged = 1;
    // x = V diag(1/sv_i for sv_i > 1e-12 sv_1) U' (Q' b)
    std::vector<double> inv(d, 0.0);
    for (int64_t i = 0; i < d; ++i)
      if (hs[i] > 1e-12 * hs[0]) inv[i] = 1.0 / hs[i];
    DevBuf utb(sizeof(double) * d, ctx->stream), dinv(sizeof(double) * d, ctx->stream);
    gemm<double>(ctx, d, 1, d, 1.0, u.as<double>(), d, 1, qtb.as<double>(), 1, 1, 0.0, utb.as<double>(), 1, 1);
    std::vector<double> h_utb(d);
    RNLA_CUDA(cudaMemcpyAsync(h_utb.data(), utb.p, sizeof(double) * d, cudaMemcpyDeviceToHost, ctx->stream));
    RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
    for (int64_t i = 0; i < d; ++i) h_utb[i] *= inv[i];
    RNLA_CUDA(cudaMemcpyAsync(utb.p, h_utb.data(), sizeof(double) * d, cudaMemcpyHostToDevice, ctx->stream));
    gemm<double>(ctx, d, 1, d, 1.0, v.as<double>(), 1, d, utb.as<double>(), 1, 1, 0.0, x_dev, 1, 1);
    RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
  }
}

template <class T>
void lsr_sketched_impl(rnla_ctx* ctx, const rnla_mat* a, const rnla_mat* b, const rnla_sketch_spec* spec, double* x,
                       double* objective, int32_t* flagged) {
  const int64_t n = a->rows, d = a->cols;
  const int64_t sf = final_size(spec);
  int64_t total = n;
  const int64_t off = global_row_offset(ctx, n, &total);
  // Sketch [A, b] jointly (one pass), s_final x (d+1), row-major.
  DevMat sk = alloc_dense(ctx, sf, d + 1, true, a->dtype);
  rnla_mat skm{sk.p, sf, d + 1, d + 1, 1, a->dtype, 1};
  const rnla_status st = rnla_sketch_rows(ctx, a, b, spec, off, &skm);
  if (st != RNLA_OK) {
    const std::string msg = rnla_last_error();
    if (st == RNLA_EINVAL) throw InvalidArgument(msg);
    throw CudaError(msg);
  }
  // a_sk (col-major fp64 s x d) and b_sk.
  DevMat ask = alloc_dense(ctx, sf, d, false, RNLA_F64);
  DevBuf bsk(sizeof(double) * sf, ctx->stream);
  if (a->dtype == RNLA_F64) {
    copy2d<double>(ctx, sf, d, sk.as<double>(), d + 1, 1, ask.as<double>(), 1, sf);
    copy2d<double>(ctx, sf, 1, sk.as<double>() + d, d + 1, 1, bsk.as<double>(), 1, sf);
  } else {
    copy2d_cast<float, double>(ctx, sf, d, sk.as<float>(), d + 1, 1, ask.as<double>(), 1, sf);
    copy2d_cast<float, double>(ctx, sf, 1, sk.as<float>() + d, d + 1, 1, bsk.as<double>(), 1, sf);
  }
  DevBuf xd(sizeof(double) * std::max<int64_t>(d, 1), ctx->stream);
  solve_sketched(ctx, sf, d, ask.as<double>(), bsk.as<double>(), xd.as<double>(), flagged);
  RNLA_CUDA(cudaMemcpyAsync(x, xd.p, sizeof(double) * d, cudaMemcpyDeviceToHost, ctx->stream));
  // objective = ||A x - b||^2: one more streaming pass over A (device-resident A only).
  if (objective) {
    DevMat da = to_device(ctx, a);
    DevMat db = to_device(ctx, b);
    double local = residual_sq<T>(ctx, n, d, da.as<T>(), da.rs, da.cs, db.as<T>(), db.rs, xd.as<double>());
    *objective = allreduce_scalar(ctx, local);
  }
  RNLA_CUDA(cudaStreamSynchronize(ctx->stream));
}

}  // namespace rnla

extern "C" rnla_status rnla_lsr_sketched(rnla_ctx* ctx, const rnla_mat* a, const rnla_mat* b,
                                         const rnla_sketch_spec* spec, double* x, double* objective,
                                         int32_t* flagged) {
  return guard([&] {
    enter(ctx);
    check_mat(a, "lsr_sketched: a");
    check_mat(b, "lsr_sketched: b");
    check_spec(spec);
    require(a->rows == b->rows && b->cols == 1, "lsr_sketched: dimension mismatch");
    require(spec->s >= a->cols, "lsr_sketched: s < d");
    require(a->dtype == b->dtype, "lsr_sketched: a and b dtypes differ");
    require(x != nullptr && flagged != nullptr, "lsr_sketched: null output");
    if (a->dtype == RNLA_F64) lsr_sketched_impl<double>(ctx, a, b, spec, x, objective, flagged);
    else lsr_sketched_impl<float>(ctx, a, b, spec, x, objective, flagged);
  });
}
