// Row-shard group collective (collective.cu): NCCL or the in-process peer group.
#pragma once
#include "context.cuh"

namespace mvsk_b200 {

// true when this context is one shard of a group (NCCL or in-process)
bool is_sharded(const mvsk_gpu_ctx* ctx);
// in-place fp64 sum over the group, on ctx->stream; no-op for a lone context
void allreduce_sum(mvsk_gpu_ctx* ctx, double* buf, size_t cnt);

LocalGroup* group_new(int nranks);
void group_join(LocalGroup* g, mvsk_gpu_ctx* ctx, int rank);
void group_leave(mvsk_gpu_ctx* ctx);
int group_live(const LocalGroup* g);
void group_delete(LocalGroup* g);

}  // namespace mvsk_b200
