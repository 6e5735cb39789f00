// Multi-GPU collectives of the library (include/reach_b200.h, "Multi-GPU"):
// user callbacks (reach_ctx_set_collectives) or the built-in NCCL communicator
// (reach_ctx_init_nccl; NCCL is dlopen-ed, so there is no link dependency).
// The sharded entry points use coll_shard / coll_hull / coll_allgather.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>

#include "coll.h"
#include "ctx.cuh"

using namespace rbh;

namespace {

struct NcclApi {
  bool ok = false;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*errorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    // prefer an already-loaded NCCL (e.g. the one torch brought in), else the system library
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    api.getUniqueId = reinterpret_cast<decltype(api.getUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    api.commInitRank = reinterpret_cast<decltype(api.commInitRank)>(dlsym(h, "ncclCommInitRank"));
    api.commDestroy = reinterpret_cast<decltype(api.commDestroy)>(dlsym(h, "ncclCommDestroy"));
    api.allReduce = reinterpret_cast<decltype(api.allReduce)>(dlsym(h, "ncclAllReduce"));
    api.allGather = reinterpret_cast<decltype(api.allGather)>(dlsym(h, "ncclAllGather"));
    api.errorString = reinterpret_cast<decltype(api.errorString)>(dlsym(h, "ncclGetErrorString"));
    api.ok = api.getUniqueId && api.commInitRank && api.commDestroy && api.allReduce && api.allGather;
  });
  return api;
}

ncclDataType_t nccl_type(int dt) {
  return dt == REACH_DT_U64 ? ncclUint64 : dt == REACH_DT_I32 ? ncclInt32 : ncclFloat64;
}

size_t dt_bytes(int dt) { return dt == REACH_DT_I32 ? 4 : 8; }

int nccl_allreduce(void* user, void* buf, size_t count, int32_t dtype, int32_t op, void* stream) {
  const auto& api = nccl();
  ncclResult_t r = api.allReduce(buf, buf, count, nccl_type(dtype), op == REACH_OP_MIN ? ncclMin : ncclMax,
                                 static_cast<ncclComm_t>(user), static_cast<cudaStream_t>(stream));
  return r == ncclSuccess ? REACH_OK : REACH_E_CUDA;
}

int nccl_allgather(void* user, const void* send, void* recv, size_t count, int32_t dtype, void* stream) {
  const auto& api = nccl();
  ncclResult_t r = api.allGather(send, recv, count, nccl_type(dtype), static_cast<ncclComm_t>(user),
                                 static_cast<cudaStream_t>(stream));
  return r == ncclSuccess ? REACH_OK : REACH_E_CUDA;
}

}  // namespace

namespace rbh {

void coll_shard(const reach_ctx* ctx, long long begin, long long end, long long& b, long long& e) {
  if (!ctx->has_coll || ctx->coll.world <= 1) {
    b = begin;
    e = end;
    return;
  }
  const long long total = end - begin, world = ctx->coll.world, rank = ctx->coll.rank;
  const long long base = total / world, rem = total % world;
  b = begin + rank * base + std::min(rank, rem);
  e = b + base + (rank < rem ? 1 : 0);
}

int coll_allreduce(reach_ctx* ctx, void* buf, size_t count, int dtype, int op) {
  if (!ctx->has_coll || ctx->coll.world <= 1 || count == 0) return REACH_OK;
  const int rc = ctx->coll.allreduce(ctx->coll.user, buf, count, dtype, op, ctx->stream);
  return rc ? fail(ctx, REACH_E_CUDA, "collective all-reduce failed") : REACH_OK;
}

int coll_allgather(reach_ctx* ctx, const void* send, void* recv, size_t count, int dtype) {
  if (!ctx->has_coll || ctx->coll.world <= 1) {
    if (recv != send && count) RB_CUDA(cudaMemcpyAsync(recv, send, count * dt_bytes(dtype), cudaMemcpyDefault, ctx->stream));
    return REACH_OK;
  }
  const int rc = ctx->coll.allgather(ctx->coll.user, send, recv, count, dtype, ctx->stream);
  return rc ? fail(ctx, REACH_E_CUDA, "collective all-gather failed") : REACH_OK;
}

int coll_hull(reach_ctx* ctx, unsigned long long* klo, unsigned long long* khi, int* nan0, int count2, int* div,
              int hp1, int* nboxes, unsigned long long* key) {
  if (!ctx->has_coll || ctx->coll.world <= 1) return REACH_OK;
  int rc = coll_allreduce(ctx, klo, count2 / 2, REACH_DT_U64, REACH_OP_MIN);
  if (!rc) rc = coll_allreduce(ctx, khi, count2 / 2, REACH_DT_U64, REACH_OP_MAX);
  if (!rc) rc = coll_allreduce(ctx, nan0, count2, REACH_DT_I32, REACH_OP_MAX);
  if (!rc) rc = coll_allreduce(ctx, div, hp1, REACH_DT_I32, REACH_OP_MAX);
  if (!rc) rc = coll_allreduce(ctx, nboxes, 1, REACH_DT_I32, REACH_OP_MIN);
  if (!rc) rc = coll_allreduce(ctx, key, 1, REACH_DT_U64, REACH_OP_MIN);
  return rc;
}

void coll_release(reach_ctx* ctx) {
  if (ctx->nccl_comm && nccl().ok) nccl().commDestroy(static_cast<ncclComm_t>(ctx->nccl_comm));
  ctx->nccl_comm = nullptr;
  ctx->has_coll = false;
}

}  // namespace rbh

extern "C" {

int reach_nccl_unique_id(uint8_t out_id[128]) {
  if (!out_id) return REACH_E_INVALID_ARGUMENT;
  const auto& api = nccl();
  if (!api.ok) return REACH_E_UNSUPPORTED;
  ncclUniqueId id;
  if (api.getUniqueId(&id) != ncclSuccess) return REACH_E_CUDA;
  std::memcpy(out_id, id.internal, 128);
  return REACH_OK;
}

int reach_ctx_init_nccl(reach_ctx* ctx, const uint8_t unique_id[128], int32_t world, int32_t rank) {
  rbh::DeviceGuard device_guard_(ctx);
  if (!ctx || !unique_id || world < 1 || rank < 0 || rank >= world) return REACH_E_INVALID_ARGUMENT;
  const auto& api = nccl();
  if (!api.ok) return fail(ctx, REACH_E_UNSUPPORTED, "NCCL (libnccl.so.2) not loadable");
  coll_release(ctx);
  ncclUniqueId id;
  std::memcpy(id.internal, unique_id, 128);
  ncclComm_t comm = nullptr;
  ncclResult_t r = api.commInitRank(&comm, world, id, rank);
  if (r != ncclSuccess)
    return fail(ctx, REACH_E_CUDA, std::string("ncclCommInitRank: ") + (api.errorString ? api.errorString(r) : "error"));
  ctx->nccl_comm = comm;
  ctx->coll = reach_collectives{rank, world, nccl_allreduce, nccl_allgather, comm};
  ctx->has_coll = true;
  return REACH_OK;
}

int reach_ctx_set_collectives(reach_ctx* ctx, const reach_collectives* coll) {
  if (!ctx) return REACH_E_INVALID_ARGUMENT;
  coll_release(ctx);
  if (!coll) return REACH_OK;
  if (coll->world < 1 || coll->rank < 0 || coll->rank >= coll->world || !coll->allreduce || !coll->allgather)
    return fail(ctx, REACH_E_INVALID_ARGUMENT, "reach_collectives: bad rank / world / callbacks");
  ctx->coll = *coll;
  ctx->has_coll = true;
  return REACH_OK;
}

int reach_ctx_memcpy(reach_ctx* ctx, void* dst, const void* src, size_t bytes) {
  rbh::DeviceGuard device_guard_(ctx);
  if (!ctx || (!dst && bytes) || (!src && bytes)) return REACH_E_INVALID_ARGUMENT;
  if (!bytes) return REACH_OK;
  RB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, ctx->stream));
  RB_CUDA(cudaStreamSynchronize(ctx->stream));
  return REACH_OK;
}

}  // extern "C"
