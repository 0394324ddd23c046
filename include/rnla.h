/*
 * rnla.h -- C ABI of the B200-native randomized sketch / rSVD / Nystrom core.
 *
 * This is the drop-in boundary for the hot path of the reference `randnla`
 * library (arXiv 1505.07570; the headers under /root/reference/proj/include/randnla).
 * Every entry point below names the reference function it replaces. The
 * reference passes Eigen::MatrixXd (column-major fp64) by const reference and
 * returns fresh matrices by value; here the caller describes its buffers with
 * rnla_mat (pointer + shape + strides + dtype + host/device) and owns every
 * output buffer (sizes are known from the arguments; returned ranks come back
 * through out-parameters).
 *
 * Conventions
 *  - Element (i, j) of an rnla_mat lives at data[i*row_stride + j*col_stride]
 *    (in elements). Eigen/Fortran column-major: row_stride = 1,
 *    col_stride = ld. C row-major: row_stride = ld, col_stride = 1. A
 *    row-major n x d buffer is the column-major d x n transpose the
 *    reference sketches inside sketch_rows (src/regression.cpp:17-19).
 *  - dtype RNLA_F64 reproduces the reference's double precision; RNLA_F32 is
 *    the fp32 path of BASELINE configs 2-4 (the reference has none).
 *  - on_device = 1: data is a CUDA device pointer on the context's device;
 *    on_device = 0: host memory (pinned host memory streams fastest), the
 *    library moves it across PCIe inside the call.
 *  - No entry point throws. Failures return a status; rnla_last_error()
 *    returns the thread-local message. RNLA_EINVAL corresponds to the
 *    reference's std::invalid_argument from require() (types.hpp:35-37),
 *    RNLA_ENUMERIC to std::runtime_error (e.g. src/spsd.cpp:200-207).
 *    "Flagged" fallbacks are reported through an int out-parameter, as the
 *    reference's LsrSolution::flagged (regression.hpp:17).
 *  - Ordering: every call runs on the context's own stream and returns only
 *    when its outputs are complete (host-synchronous results). Device INPUTS
 *    written asynchronously by the caller (another stream, e.g. torch's
 *    current stream) must be ordered first: either synchronize that stream or
 *    call rnla_ctx_wait_stream(ctx, stream) before the call.
 *  - Strides must be non-negative (a zero stride is allowed only along an
 *    extent of 1); anything else returns RNLA_EINVAL.
 *  - There is no CPU fallback: compute entry points need a CUDA device and
 *    return RNLA_ECUDA without one. Host-only helpers (seeds, hashes and the
 *    libstdc++ operator draws) run anywhere.
 */
#ifndef RNLA_H_
#define RNLA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RNLA_ABI_VERSION 1

typedef enum {
  RNLA_OK = 0,
  RNLA_EINVAL = 1,   /* std::invalid_argument in the reference */
  RNLA_ENUMERIC = 2, /* std::runtime_error in the reference */
  RNLA_ECUDA = 3,
  RNLA_ENCCL = 4,
  RNLA_ENOMEM = 5
} rnla_status;

typedef enum { RNLA_F64 = 0, RNLA_F32 = 1 } rnla_dtype;

typedef struct {
  void* data;
  int64_t rows, cols;
  int64_t row_stride, col_stride; /* in elements */
  int32_t dtype;                  /* rnla_dtype */
  int32_t on_device;              /* 1 = CUDA device pointer, 0 = host */
} rnla_mat;

/* SketchKind, include/randnla/sketch.hpp:14-22 (same order). */
typedef enum {
  RNLA_SKETCH_GAUSSIAN = 0,
  RNLA_SKETCH_SRHT = 1,
  RNLA_SKETCH_COUNT = 2,
  RNLA_SKETCH_UNIFORM_COLUMNS = 3,
  RNLA_SKETCH_LEVERAGE_COLUMNS = 4,
  RNLA_SKETCH_LANDMARK_COLUMNS = 5, /* out of scope: returns RNLA_EINVAL */
  RNLA_SKETCH_COMBINED = 6
} rnla_sketch_kind;

/* SketchSpec, include/randnla/sketch.hpp:25-54. stage2_* is the dense stage
 * of a combined sketch (stage2 != nullptr there); leverage_rank <= 0 means
 * std::nullopt. */
typedef struct {
  int32_t kind;
  int64_t s;
  uint64_t seed;
  int32_t stage2_kind;
  int64_t stage2_s;
  uint64_t stage2_seed;
  int32_t scale_columns;
  int64_t leverage_rank;
} rnla_sketch_spec;

typedef struct rnla_ctx rnla_ctx;

/* ---- library / context ------------------------------------------------ */
int rnla_abi_version(void);
const char* rnla_last_error(void);
/* Context on one CUDA device: stream, workspace, cuSOLVER handle and the
 * operator cache (hash permutations, Gaussian Omega keyed by (n, s, seed)). */
rnla_status rnla_ctx_create(int device, rnla_ctx** out);
/* Row-sharded context: rank `rank` of `world` processes, one GPU each, joined
 * through NCCL with a 128-byte ncclUniqueId produced by rnla_nccl_unique_id on
 * rank 0 and broadcast by the caller. world = 1 creates a one-rank
 * communicator: the row-sharded code paths and their NCCL collectives run on
 * a single GPU (results equal a plain context's to rounding). */
rnla_status rnla_ctx_create_dist(int device, int world, int rank, const void* nccl_unique_id, rnla_ctx** out);
rnla_status rnla_nccl_unique_id(void* out128);
/* In-process shard group: `world` contexts driven by `world` host threads of
 * one process (any devices, including several ranks on one GPU). Collectives
 * are staged through pinned host memory and summed in rank order, so results
 * are bitwise identical on every rank and independent of the device count;
 * no kernel ever waits on another rank's kernel. Same shard semantics as
 * rnla_ctx_create_dist. The group must outlive its contexts. */
typedef struct rnla_group rnla_group;
rnla_status rnla_group_create(int world, rnla_group** out);
void rnla_group_destroy(rnla_group* group);
rnla_status rnla_ctx_create_grouped(int device, rnla_group* group, int rank, rnla_ctx** out);
void rnla_ctx_destroy(rnla_ctx* ctx);
rnla_status rnla_ctx_synchronize(rnla_ctx* ctx);
/* Make the context's stream wait for all work enqueued so far on the caller's
 * `stream` (a cudaStream_t on the context's device; NULL = the legacy default
 * stream) without blocking the host: event record + cudaStreamWaitEvent. */
rnla_status rnla_ctx_wait_stream(rnla_ctx* ctx, void* stream);
/* The context's CUDA stream (a cudaStream_t), for callers that time with events. */
void* rnla_ctx_stream(rnla_ctx* ctx);
/* Kernel launches issued by this context since creation (instrumentation). */
int64_t rnla_ctx_launch_count(rnla_ctx* ctx);
/* Release cached operators and workspace. */
void rnla_ctx_clear_cache(rnla_ctx* ctx);
/* Contiguous row block [begin, end) of rank `rank` out of `world` for n rows
 * (host-only; the shard layout every distributed entry point uses). */
void rnla_shard_rows(int64_t n, int world, int rank, int64_t* begin, int64_t* end);

/* ---- seeds, hashes, operator draws (host, libstdc++) -------------------- */
/* include/randnla/rng.hpp:13-18 (returns the output, advances *state). */
uint64_t rnla_splitmix64(uint64_t* state);
/* include/randnla/rng.hpp:21-24 */
uint64_t rnla_derive_seed(uint64_t seed, uint64_t stream);
/* src/sketch.cpp:16-26 for j in [j0, j0+n): buckets[i], signs[i] (+1/-1). */
rnla_status rnla_count_sketch_hashes(uint64_t seed, int64_t j0, int64_t n, int64_t s, int64_t* buckets,
                                     int8_t* signs);
/* src/rng.cpp:8-14 on make_rng(seed): column-major rows x cols fill. */
rnla_status rnla_gaussian_matrix(uint64_t seed, int64_t rows, int64_t cols, double* out_colmajor);
/* src/rng.cpp:27-40 on make_rng(seed); out[count], sorted ascending. */
rnla_status rnla_sample_without_replacement(uint64_t seed, int64_t n, int64_t count, int64_t* out);
/* src/rng.cpp:42-65 on make_rng(seed); out[count] in draw order. */
rnla_status rnla_sample_with_replacement(uint64_t seed, const double* weights, int64_t n, int64_t count,
                                         int64_t* out);
/* src/sketch.cpp:57-65: signs[n] then idx[s] (sorted) from one engine. */
rnla_status rnla_srht_operator(uint64_t seed, int64_t n, int64_t s, int8_t* signs, int64_t* idx);

/* ---- sketch operators: C = A * S (reference semantics) ------------------ */
/* gaussian_sketch, include/randnla/sketch.hpp:62 (src/sketch.cpp:36-42). */
rnla_status rnla_gaussian_sketch(rnla_ctx* ctx, const rnla_mat* a, int64_t s, uint64_t seed, rnla_mat* c);
/* srht_sketch, sketch.hpp:67 (src/sketch.cpp:57-81). */
rnla_status rnla_srht_sketch(rnla_ctx* ctx, const rnla_mat* a, int64_t s, uint64_t seed, rnla_mat* c);
/* count_sketch, sketch.hpp:78 (src/sketch.cpp:94-97). Bit-exact with the
 * reference's single-pass j-ascending accumulation for fp64. */
rnla_status rnla_count_sketch(rnla_ctx* ctx, const rnla_mat* a, int64_t s, uint64_t seed, rnla_mat* c);
/* combined_sketch, sketch.hpp:86 (src/sketch.cpp:108-123). */
rnla_status rnla_combined_sketch(rnla_ctx* ctx, const rnla_mat* a, const rnla_sketch_spec* spec, rnla_mat* c);
/* apply_sketch, sketch.hpp:107 (src/sketch.cpp:177-197). c must have
 * a->rows rows and rnla_sketch_output_cols(spec, a->cols) columns; for the
 * leverage kind the effective column count comes back in *cols_out. */
rnla_status rnla_apply_sketch(rnla_ctx* ctx, const rnla_mat* a, const rnla_sketch_spec* spec, rnla_mat* c,
                              int64_t* cols_out);
int64_t rnla_sketch_output_cols(const rnla_sketch_spec* spec, int64_t n);
/* S^T M for a tall M (n x d): sketch_rows of src/regression.cpp:17-19
 * (= apply_sketch(M^T)^T) without the transpose copies. out is s_final x d.
 * `extra` (nullable, n x 1) appends one column, i.e. sketches [M, extra] as
 * lsr_sketched's stacked matrix (src/regression.cpp:76-78); out is then
 * s_final x (d+1). row_offset is the global index of M's first row (row
 * sharding); rows are hashed / signed by their global index. */
rnla_status rnla_sketch_rows(rnla_ctx* ctx, const rnla_mat* m, const rnla_mat* extra, const rnla_sketch_spec* spec,
                             int64_t row_offset, rnla_mat* out);
/* count_sketch_stream, sketch.hpp:75-76 (src/sketch.cpp:83-92): a single
 * pass over n columns of length m delivered in order by the caller. begin
 * opens a device-resident m x s accumulator; push appends the next chunk of
 * columns (an m x k matrix holding columns j .. j+k-1, host or device; the
 * call returns once the chunk buffer may be reused); end writes C (m x s)
 * and frees the stream (also on error); abort frees it without a result.
 * fp64 results are bit-identical to the reference's sequential loop. */
typedef struct rnla_count_stream rnla_count_stream;
rnla_status rnla_count_stream_begin(rnla_ctx* ctx, int64_t m, int64_t n, int64_t s, uint64_t seed, int32_t dtype,
                                    rnla_count_stream** out);
rnla_status rnla_count_stream_push(rnla_count_stream* stream, const rnla_mat* columns);
rnla_status rnla_count_stream_end(rnla_count_stream* stream, rnla_mat* c);
void rnla_count_stream_abort(rnla_count_stream* stream);
/* fwht_inplace, sketch.hpp:70 (src/sketch.cpp:44-55) applied to every
 * column of x in place (column length a power of two); same butterflies in
 * the same stage order as the reference loop (bit-identical). */
rnla_status rnla_fwht(rnla_ctx* ctx, rnla_mat* x);
/* uniform_sample_columns, sketch.hpp:89-90: indices[s] + gathered c. */
rnla_status rnla_uniform_sample_columns(rnla_ctx* ctx, const rnla_mat* a, int64_t s, uint64_t seed, rnla_mat* c,
                                        int64_t* indices);
/* leverage_scores, sketch.hpp:95 (src/sketch.cpp:138-141): scores[a->cols];
 * k <= 0 means std::nullopt. */
rnla_status rnla_leverage_scores(rnla_ctx* ctx, const rnla_mat* a, int64_t k, double* scores);
/* leverage_sample_columns, sketch.hpp:98-100. indices / weights sized s;
 * *count_out = effective (deduplicated) count; weights may be NULL when
 * scale == 0. c has a->rows rows and >= s columns. */
rnla_status rnla_leverage_sample_columns(rnla_ctx* ctx, const rnla_mat* a, int64_t s, uint64_t seed, int64_t k,
                                         int scale, rnla_mat* c, int64_t* indices, double* weights,
                                         int64_t* count_out);
/* Row leverage of a tall M from its orthonormal basis (the
 * `Q.rowwise().squaredNorm()` pattern of src/spsd.cpp:150): scores[n] =
 * ||Q_i,:||^2 with Q = thin_qr(M).Q, computed as ||m_i R^-1||^2
 * (CholeskyQR); then p draws with replacement from make_rng(seed), sorted and
 * deduplicated into indices (*count_out entries). indices may be NULL. */
rnla_status rnla_leverage_sample_rows(rnla_ctx* ctx, const rnla_mat* m, int64_t p, uint64_t seed, double* scores,
                                      int64_t* indices, int64_t* count_out);

/* ---- core linear algebra (include/randnla/core.hpp) --------------------- */
/* thin_qr, core.hpp:12 (src/core.cpp:37-46): q is m x n, r is n x n. */
rnla_status rnla_thin_qr(rnla_ctx* ctx, const rnla_mat* a, rnla_mat* q, rnla_mat* r);
/* condensed_svd, core.hpp:17 (src/core.cpp:48-64). u m x min(m,n), sv
 * [min(m,n)], v n x min(m,n); the first *rank columns are valid. */
rnla_status rnla_condensed_svd(rnla_ctx* ctx, const rnla_mat* a, rnla_mat* u, double* sv, rnla_mat* v,
                               int64_t* rank);
/* truncated_svd, core.hpp:20 (src/core.cpp:66-76). u m x k, v n x k. */
rnla_status rnla_truncated_svd(rnla_ctx* ctx, const rnla_mat* a, int64_t k, rnla_mat* u, double* sv, rnla_mat* v,
                               int64_t* rank);
/* pseudo_inverse, core.hpp:25 (src/core.cpp:78-88). p is n x m. */
rnla_status rnla_pseudo_inverse(rnla_ctx* ctx, const rnla_mat* a, double tol, rnla_mat* p);

/* ---- randomized k-SVD (include/randnla/randsvd.hpp) ---------------------- */
/* prototype_ksvd, randsvd.hpp:29-32 (src/randsvd.cpp:88-110), plus
 * power_iters q >= 0 (BASELINE configs 0/3; q = 0 is
 * exactly the reference). spec may be NULL (Gaussian). u m x k, sv[k],
 * v n x k; *rank = number of valid columns; *passes = passes over A
 * (2 + 2q); error_fro (nullable) = ||A - U S V'||_F (KsvdOptions). */
rnla_status rnla_prototype_ksvd(rnla_ctx* ctx, const rnla_mat* a, int64_t k, int64_t s, uint64_t seed,
                                const rnla_sketch_spec* spec, int32_t power_iters, rnla_mat* u, double* sv,
                                rnla_mat* v, int64_t* rank, int32_t* passes, double* error_fro);
/* faster_ksvd, randsvd.hpp:38-41 (src/randsvd.cpp:112-160): column count
 * sketch C = A S (s), joint row sketch of [A, C] (count p_cs -> Gaussian p),
 * QR of D, rank-k SVD of Q_D' L, back-substitution and a final small SVD.
 * Exactly two passes over A. Requires k < s < p < p_cs. u m x k, sv[k], v n x k. */
rnla_status rnla_faster_ksvd(rnla_ctx* ctx, const rnla_mat* a, int64_t k, int64_t s, int64_t p_cs, int64_t p,
                             uint64_t seed, rnla_mat* u, double* sv, rnla_mat* v, int64_t* rank, int32_t* passes,
                             double* error_fro);

/* ---- regression (include/randnla/regression.hpp) ------------------------ */
/* lsr_sketched, regression.hpp:31-32 (src/regression.cpp:68-92). x[d];
 * objective = ||Ax - b||^2; *flagged = 1 when the pseudo-inverse fallback
 * ran. a is n x d, b is n x 1. */
rnla_status rnla_lsr_sketched(rnla_ctx* ctx, const rnla_mat* a, const rnla_mat* b, const rnla_sketch_spec* spec,
                              double* x, double* objective, int32_t* flagged);
/* lsr_preconditioned, regression.hpp:44-56 with PreconditionedOptions
 * {sketch_size (0: min(d^2, 20d) capped at n), use_cg, sketch_kind (COUNT,
 * GAUSSIAN or SRHT)} (src/regression.cpp:94-198). x[d], *iterations; the
 * objective |Ax - b|^2 and kappa(A R_Y^-1) are skipped when their pointers
 * are NULL. Each iteration is one fused pass over A: A'(b - A T z). d <= 1024.
 * RNLA_ENUMERIC when the sketched matrix is singular twice. */
/* lsr_cg, regression.hpp:24-27 (src/regression.cpp:38-66): CG on the normal
 * equations, converged when |A'(Ax - b)| <= tol |A'b|; each iteration is one
 * fused pass over A. x[d]; objective (nullable) = |Ax - b|^2; *converged
 * (nullable). d <= 1024. */
rnla_status rnla_lsr_cg(rnla_ctx* ctx, const rnla_mat* a, const rnla_mat* b, double tol, int32_t maxit, double* x,
                        double* objective, int32_t* iterations, int32_t* converged);
rnla_status rnla_lsr_preconditioned(rnla_ctx* ctx, const rnla_mat* a, const rnla_mat* b, double eps, uint64_t seed,
                                    int64_t sketch_size, int32_t use_cg, int32_t sketch_kind, double* x,
                                    double* objective, int32_t* iterations, double* kappa_estimate);

/* ---- SPSD / kernels (include/randnla/spsd.hpp) -------------------------- */
/* rbf_kernel, spsd.hpp:19-20 (src/spsd.cpp:33-47). Rows are points. */
rnla_status rnla_rbf_kernel(rnla_ctx* ctx, const rnla_mat* x1, const rnla_mat* x2, double sigma, rnla_mat* k);
/* nystrom(KernelView, s, seed, target_k), spsd.hpp:119-124 (src/spsd.cpp:181-222)
 * with KernelView(data = x, sigma). l (nullable) is n x target_k (or
 * ceil(0.8 s)); selected[s]; *kept = valid columns of l;
 * *entries = kernel entries evaluated (KernelView::entries_evaluated). */
rnla_status rnla_nystrom(rnla_ctx* ctx, const rnla_mat* x, double sigma, int64_t s, uint64_t seed, int64_t target_k,
                         rnla_mat* l, int64_t* selected, int64_t* kept, int64_t* entries);
/* nystrom(const DenseMatrix& K, s, seed, target_k), spsd.hpp:123-124
 * (src/spsd.cpp:224-228, DenseSpsdSource): K n x n; l (nullable) n x
 * target_k (or ceil(0.8 s)); selected[s]; *kept as rnla_nystrom. */
rnla_status rnla_nystrom_dense(rnla_ctx* ctx, const rnla_mat* k, int64_t s, uint64_t seed, int64_t target_k,
                               rnla_mat* l, int64_t* selected, int64_t* kept);
/* nystrom(const SpsdSource&, ...), spsd.hpp:119-120 (src/spsd.cpp:181-217)
 * for any caller-side source: c = K[:, selected] (n x s) already evaluated,
 * selected[s] strictly increasing (the reference draws them with
 * sample_without_replacement(n, s, make_rng(derive_seed(seed, 1)))). */
rnla_status rnla_nystrom_columns(rnla_ctx* ctx, const rnla_mat* c, const int64_t* selected, int64_t target_k,
                                 rnla_mat* l, int64_t* kept);
/* approx_eig, spsd.hpp:135 (src/spsd.cpp:257-265): u n x k, lam[k]. */
rnla_status rnla_approx_eig(rnla_ctx* ctx, const rnla_mat* l, int64_t k, rnla_mat* u, double* lam);
/* nystrom followed by approx_eig(L, k) without materializing C or L (Gram
 * route). u (nullable) n x k, lam[k], selected[s]. */
rnla_status rnla_nystrom_eig(rnla_ctx* ctx, const rnla_mat* x, double sigma, int64_t s, uint64_t seed,
                             int64_t target_k, int64_t k, rnla_mat* u, double* lam, int64_t* selected,
                             int64_t* kept);
/* spsd_faster on a KernelView of the points x (n x d), spsd.hpp:113-115
 * (src/spsd.cpp:131-168): S = landmarks (derive_seed(seed, 1)), Q = thin_qr(K[:, S]).Q
 * (n x s), secondary rows P = leverage draws of Q's rows (derive_seed(seed, 2);
 * all rows when p == n) united with S, Z = pinv(Q_P) K[P, P] pinv(Q_P)' (s x s,
 * symmetrized). selected[s]; secondary needs room for min(n, p + s) indices,
 * *n_secondary = |P|; *flagged = 1 when Q_P is rank deficient (threshold 1e-10).
 * Kernel entries evaluated: n*s + |P|^2. */
rnla_status rnla_spsd_faster(rnla_ctx* ctx, const rnla_mat* x, double sigma, int64_t s, int64_t p, uint64_t seed,
                             rnla_mat* q, rnla_mat* z, int64_t* selected, int64_t* secondary, int64_t* n_secondary,
                             int32_t* flagged);
/* cur_faster_kernel, cur.hpp:44-52 (src/cur.cpp:47-104, 188-212): CUR of the
 * implicit RBF cross kernel K*_ij = kappa(xtest_i, xtrain_j) (m x n) with
 * uniform primary (c columns, r rows) and secondary (p = 2(c + r)) draws:
 * C (m x c), U (c x r), R (r x n); col_idx[c], row_idx[r]; the secondary
 * rows / cols (room for min(m, p + r) / min(n, p + c)) with their counts;
 * *entries (nullable) = m c + r n + |P_C| |P_R|; *flagged when C[P_C,:] or
 * R[:,P_R] is rank deficient (threshold 1e-10). */
rnla_status rnla_cur_faster_kernel(rnla_ctx* ctx, const rnla_mat* xtest, const rnla_mat* xtrain, double sigma,
                                   int64_t c, int64_t r, uint64_t seed, rnla_mat* cmat, rnla_mat* umat, rnla_mat* rmat,
                                   int64_t* col_idx, int64_t* row_idx, int64_t* sec_rows, int64_t* n_sec_rows,
                                   int64_t* sec_cols, int64_t* n_sec_cols, int64_t* entries, int32_t* flagged);
/* The same on a dense SPSD K (n x n), spsd.hpp:111-112. */
rnla_status rnla_spsd_faster_dense(rnla_ctx* ctx, const rnla_mat* k, int64_t s, int64_t p, uint64_t seed, rnla_mat* q,
                                   rnla_mat* z, int64_t* selected, int64_t* secondary, int64_t* n_secondary,
                                   int32_t* flagged);

#ifdef __cplusplus
}
#endif
#endif /* RNLA_H_ */
