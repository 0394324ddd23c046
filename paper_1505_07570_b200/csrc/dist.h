// dist.h -- collectives for row-sharded contexts (no-ops when world == 1).
#pragma once
#include "rnla_internal.h"

namespace rnla {

// In-place sum over ranks of a device buffer (NCCL, on ctx->stream).
void allreduce_sum(rnla_ctx* ctx, void* buf, size_t count, int dtype);
// In-place sum over ranks onto `root` (NCCL, on ctx->stream).
void reduce_to(rnla_ctx* ctx, void* buf, size_t count, int dtype, int root);
// Global index of this rank's first row given every rank's local row count.
int64_t global_row_offset(rnla_ctx* ctx, int64_t local_rows, int64_t* total_rows);
double allreduce_scalar(rnla_ctx* ctx, double v);
// Every rank's `count`-element block, concatenated in rank order into `all`
// (world * count elements; a zero-padded allreduce).
void allgather_blocks(rnla_ctx* ctx, const void* mine, void* all, size_t count, int dtype);
rnla_group* group_create(int world);
void group_destroy(rnla_group* g);
void group_mark_broken(rnla_group* g);
int group_world(const rnla_group* g);

}  // namespace rnla
