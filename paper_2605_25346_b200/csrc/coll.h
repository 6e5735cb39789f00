// Internal (not ABI): the collectives a sharded entry point uses (coll.cu).
#pragma once

#include <cstddef>
#include <cstdint>

struct reach_ctx;

namespace rbh {
// Contiguous [b, e) slice of [begin, end) for this ctx's rank (sizes differ by at most one).
void coll_shard(const reach_ctx* ctx, long long begin, long long end, long long& b, long long& e);
int coll_allreduce(reach_ctx* ctx, void* buf, size_t count, int dtype, int op);
int coll_allgather(reach_ctx* ctx, const void* send, void* recv, size_t count, int dtype);
// The split-hull combination: order keys (min / max), part-0 NaN flags, box-diverged flags,
// box count and failure key -- all integer reductions, exact and order independent.
int coll_hull(reach_ctx* ctx, unsigned long long* klo, unsigned long long* khi, int* nan0, int count2, int* div,
              int hp1, int* nboxes, unsigned long long* key);
// Releases the built-in communicator (reach_ctx_destroy).
void coll_release(reach_ctx* ctx);
}  // namespace rbh
