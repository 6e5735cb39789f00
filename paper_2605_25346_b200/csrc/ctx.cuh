// Host-side internals shared by the library's translation units (reach_capi.cu:
// DT / MPC entry points, ct_capi.cu: continuous-time closed loop).  Not part of
// the ABI: include/reach_b200.h exposes these types as opaque handles.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include "../../include/reach_b200.h"
#include "dt_kernel.cuh"
#include "tcw_types.cuh"

struct reach_ctx {
  int device = 0;
  cudaStream_t own = nullptr;
  cudaStream_t stream = nullptr;
  std::string err;
  int64_t launches = 0;
  int num_sms = 0;
  int max_smem = 0;
  // growable device workspace for host-pointer calls
  void* ws = nullptr;
  size_t ws_bytes = 0;
  // plan-problem staging buffer (goal, weights, constraints) for the MPC kernels
  void* pbuf = nullptr;
  size_t pbuf_bytes = 0;
  // pinned host staging (MPC candidate populations, scores), grown on demand
  void* hpin = nullptr;
  size_t hpin_bytes = 0;
  // per-CTA symbolic-state buffers of the wide kernel family
  void* wws = nullptr;
  size_t wws_bytes = 0;
  unsigned long long* wphase = nullptr;
  cudaStream_t aux = nullptr;  // second stream: plan_eval's rollouts run beside its tube kernel
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  void* ctd_ws = nullptr;  // Dual CT working sets (ctl_reach_loss gradient), one per persistent CTA
  size_t ctd_bytes = 0;  // wide-kernel phase counters (RB_WIDE_PHASE=1)
  // multi-GPU collectives (coll.cu): user callbacks or the built-in NCCL communicator
  reach_collectives coll{};
  bool has_coll = false;
  void* nccl_comm = nullptr;
  // kernel timing
  bool timing = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_used, ev_free;
};

struct reach_net {
  rb::DevNet dev{};
  double* blob = nullptr;
  int L = 0;
  int cpl = 0;  // hidden units per lane of the kernel family (0 = unsupported width)
  int hp = 0;   // padded hidden width 32 * cpl
  std::vector<int> dims, acts;
  std::vector<double> params;  // host copy in net_params order (neural.hpp:133-140)
  // tensor-core mode (tc_capi.cu, built on first use): Ozaki split planes of W_l^T,
  // their TMA tensor maps, row scale exponents and L1 norms, in one device allocation
  mutable void* oz_mem = nullptr;
  mutable rb::OzNet oz{};
};

namespace rbh {

inline int fail(reach_ctx* ctx, int code, const std::string& msg) {
  if (ctx) ctx->err = msg;
  return code;
}

inline int cuda_fail(reach_ctx* ctx, cudaError_t e, const char* where) {
  return fail(ctx, e == cudaErrorMemoryAllocation ? REACH_E_OOM : REACH_E_CUDA,
              std::string(where) + ": " + cudaGetErrorString(e));
}

#define RB_CUDA(call)                                   \
  do {                                                  \
    cudaError_t e_ = (call);                            \
    if (e_ != cudaSuccess) return cuda_fail(ctx, e_, #call); \
  } while (0)

// Every entry point runs on its context's device and leaves the caller's current
// device as it found it (contexts on different GPUs may alternate in one thread).
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(const reach_ctx* c) {
    if (!c) return;
    int cur = -1;
    if (cudaGetDevice(&cur) == cudaSuccess && cur != c->device) {
      cudaSetDevice(c->device);
      prev = cur;
    }
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
  DeviceGuard(const DeviceGuard&) = delete;
  DeviceGuard& operator=(const DeviceGuard&) = delete;
};

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

inline int ensure_ws(reach_ctx* ctx, size_t bytes) {
  if (bytes <= ctx->ws_bytes) return REACH_OK;
  if (ctx->ws) {
    cudaStreamSynchronize(ctx->stream);
    cudaFree(ctx->ws);
    ctx->ws = nullptr;
    ctx->ws_bytes = 0;
  }
  RB_CUDA(cudaMalloc(&ctx->ws, bytes));
  ctx->ws_bytes = bytes;
  return REACH_OK;
}

inline int ensure_pinned(reach_ctx* ctx, size_t bytes) {
  if (bytes <= ctx->hpin_bytes) return REACH_OK;
  if (ctx->hpin) {
    cudaStreamSynchronize(ctx->stream);
    cudaFreeHost(ctx->hpin);
    ctx->hpin = nullptr;
    ctx->hpin_bytes = 0;
  }
  RB_CUDA(cudaMallocHost(&ctx->hpin, bytes));
  ctx->hpin_bytes = bytes;
  return REACH_OK;
}

inline int timed_begin(reach_ctx* ctx, cudaEvent_t* stop) {
  *stop = nullptr;
  if (!ctx->timing) return REACH_OK;
  std::pair<cudaEvent_t, cudaEvent_t> p;
  if (!ctx->ev_free.empty()) {
    p = ctx->ev_free.back();
    ctx->ev_free.pop_back();
  } else {
    RB_CUDA(cudaEventCreate(&p.first));
    RB_CUDA(cudaEventCreate(&p.second));
  }
  RB_CUDA(cudaEventRecord(p.first, ctx->stream));
  ctx->ev_used.push_back(p);
  *stop = p.second;
  return REACH_OK;
}

inline int timed_end(reach_ctx* ctx, cudaEvent_t stop) {
  if (stop) RB_CUDA(cudaEventRecord(stop, ctx->stream));
  return REACH_OK;
}

}  // namespace rbh
