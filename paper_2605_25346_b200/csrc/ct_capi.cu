// C ABI of the continuous-time closed loop (include/reach_b200.h):
// reach_cl_batch (cl_reach per initial box, closed_loop.hpp:76-182) and
// reach_cl_split_hull (reach_with_splitting(cl_reach), refine.hpp:121-160).
//
// Per control interval: ct_ctl_kernel (controller certification + stacking)
// then ct_flow_kernel (k_atomic flowpipe steps); the symbolic state of every
// sub-box stays in device memory across the 2 * ctl_steps launches.  No CPU
// fallback: an unsupported plant or shape is an error.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "ct_kernel.cuh"
#include "ctx.cuh"

using namespace rbh;

namespace {

__global__ void ct_hull_init_kernel(unsigned long long* klo, unsigned long long* khi, int* nan0, int* div, int count,
                                    int T, int* nboxes, unsigned long long* key) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < count) {
    klo[t] = ~0ull;
    khi[t] = 0ull;
    nan0[2 * t] = 0;
    nan0[2 * t + 1] = 0;
  }
  if (t < T) div[t] = 0;
  if (t == 0) {
    *nboxes = INT_MAX;
    *key = static_cast<unsigned long long>(INT64_MAX);
  }
}

__global__ void ct_hull_finalize_kernel(const unsigned long long* klo, const unsigned long long* khi, const int* nan0,
                                        int count, double* lo, double* hi) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= count) return;
  lo[t] = nan0[2 * t] ? __longlong_as_double(0x7ff8000000000000ll) : rb::from_order_key(klo[t]);
  hi[t] = nan0[2 * t + 1] ? __longlong_as_double(0x7ff8000000000000ll) : rb::from_order_key(khi[t]);
}

// ClosedLoopSpec::validate (closed_loop.hpp:30-43) + the device family's limits.
int validate_cl(reach_ctx* ctx, const reach_net* ctl, const reach_cl_spec* s) {
  const reach_flowpipe_params& f = s->fp;
  if (!(f.h > 0) || f.steps <= 0 || f.order < 1 || f.order > 2 || !(f.eps_init > 0) || !(f.enlargement > 1.0) ||
      f.refine_rounds < 0 || f.max_enlargements < 0 || f.window < 0)
    return fail(ctx, REACH_E_INVALID_ARGUMENT, "FlowpipeParams: invalid configuration");
  if (s->n <= 0 || s->l <= 0 || s->ctl_steps <= 0 || s->k_atomic <= 0)
    return fail(ctx, REACH_E_INVALID_ARGUMENT, "ClosedLoopSpec: invalid dimensions");
  if (s->plant != REACH_PLANT_QUADROTOR) return fail(ctx, REACH_E_UNSUPPORTED, "cl_reach: unknown plant");
  if (s->n != rb::ct::NX || s->n + s->l != rb::ct::NA)
    return fail(ctx, REACH_E_INVALID_ARGUMENT, "ClosedLoopSpec: dynamics must act on the augmented (x,u) state");
  if (ctl->dims[ctl->L] != s->l) return fail(ctx, REACH_E_INVALID_ARGUMENT, "ClosedLoopSpec: controller output dim mismatch");
  if (s->ref_dim < 0 || (s->ref_dim > 0 && !s->y_ref))
    return fail(ctx, REACH_E_INVALID_ARGUMENT, "ClosedLoopSpec: reference sequence length mismatch");
  if (ctl->dims[0] != s->n + s->ref_dim)
    return fail(ctx, REACH_E_INVALID_ARGUMENT, "ClosedLoopSpec: controller input dim mismatch");
  if (f.window > 4) return fail(ctx, REACH_E_UNSUPPORTED, "cl_reach: window > 4 exceeds the 96-column TM rows");
  for (int t = 0; t + 1 < ctl->L; ++t)
    if (ctl->dims[t + 1] > rb::ct::kMaxCtlW) return fail(ctx, REACH_E_UNSUPPORTED, "cl_reach: controller layer wider than 128");
  if (ctl->dims[0] > rb::ct::kMaxCtlW) return fail(ctx, REACH_E_UNSUPPORTED, "cl_reach: controller input wider than 128");
  return REACH_OK;
}


int setup_params(reach_ctx* ctx, const reach_net* ctl, const reach_cl_spec* s, long long B, rb::ct::CTParams& P) {
  P.B = static_cast<int>(B);
  P.n = s->n;
  P.l = s->l;
  P.K = s->k_atomic;
  P.window = s->fp.window;
  P.order = s->fp.order;
  P.refine = s->fp.refine_rounds;
  P.maxe = s->fp.max_enlargements;
  P.intervalize = s->intervalize_boundary;
  P.ref_dim = s->ref_dim;
  P.ctl_steps = s->ctl_steps;
  P.h = s->fp.h;
  P.eps = s->fp.eps_init;
  P.enl = s->fp.enlargement;
  for (int i = 0; i < 8; ++i) P.prm[i] = s->plant_params[i];
  // quadrotor_ode's constants, computed as the reference does (systems.hpp:48-63)
  const double mass = s->plant_params[0], grav = s->plant_params[1], jx = s->plant_params[2],
               jy = s->plant_params[3], jz = s->plant_params[4];
  P.kc[0] = 1.0 / mass;
  P.kc[1] = grav;
  P.kc[2] = (jy - jz) / jx;
  P.kc[3] = 1.0 / jx;
  P.kc[4] = (jz - jx) / jy;
  P.kc[5] = 1.0 / jy;
  P.kc[6] = (jx - jy) / jz;
  P.kc[7] = 1.0 / jz;
  P.ctl = ctl->dev;
  P.T = 1 + s->ctl_steps * s->k_atomic;
  (void)ctx;
  return REACH_OK;
}

int launch_cl(reach_ctx* ctx, rb::ct::CTParams& P) {
  const size_t flow_smem = rb::ct::SPW * sizeof(rb::ct::FlowSmem);  // SPW sub-boxes per warp
  const size_t ctl_smem = sizeof(rb::ct::CtlSmem) * rb::ct::kCtlWarps;
  RB_CUDA(cudaFuncSetAttribute(rb::ct::ct_flow_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(flow_smem)));
  RB_CUDA(cudaFuncSetAttribute(rb::ct::ct_ctl_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(ctl_smem)));
  cudaEvent_t stop;
  int rc = timed_begin(ctx, &stop);
  if (rc) return rc;
  const int ctl_grid = (P.B + rb::ct::kCtlWarps - 1) / rb::ct::kCtlWarps;
  for (int ci = 0; ci < P.ctl_steps; ++ci) {
    P.ci = ci;
    rb::ct::ct_ctl_kernel<<<ctl_grid, 32 * rb::ct::kCtlWarps, ctl_smem, ctx->stream>>>(P);
    RB_CUDA(cudaGetLastError());
    rb::ct::ct_flow_kernel<<<(P.B + rb::ct::SPW - 1) / rb::ct::SPW, 32, flow_smem, ctx->stream>>>(P);
    RB_CUDA(cudaGetLastError());
  }
  rc = timed_end(ctx, stop);
  if (rc) return rc;
  ctx->launches += 2 * P.ctl_steps;
  return REACH_OK;
}

// Workspace carve-up: state (c, M, meta) + y_ref + caller-side staging.
struct Carve {
  size_t off = 0;
  size_t take(size_t bytes) {
    size_t o = off;
    off = align_up(off + bytes, 256);
    return o;
  }
};

}  // namespace

extern "C" {

int reach_cl_batch(reach_ctx* ctx, const reach_net* ctl, const reach_cl_spec* s, int32_t batch, const double* x0_lo,
                   const double* x0_hi, const reach_tube_out* out, int32_t flags) {
  if (!ctx || !ctl || !s || !out) return REACH_E_INVALID_ARGUMENT;
  if (batch < 0) return fail(ctx, REACH_E_INVALID_ARGUMENT, "cl_reach: negative batch");
  int rc = validate_cl(ctx, ctl, s);
  if (rc) return rc;
  if (batch == 0) return REACH_OK;
  const bool dev = (flags & REACH_FLAG_DEVICE_PTRS) != 0;
  if (!dev) {  // build_linear_tm rejects diverged X0 (taylor_model.hpp:55)
    for (size_t i = 0; i < static_cast<size_t>(batch) * s->n; ++i)
      if (!std::isfinite(x0_lo[i]) || !std::isfinite(x0_hi[i]))
        return fail(ctx, REACH_E_INVALID_ARGUMENT, "build_linear_tm: diverged box");
  }
  RB_CUDA(cudaSetDevice(ctx->device));
  rb::ct::CTParams P{};
  setup_params(ctx, ctl, s, batch, P);
  const size_t B = batch, n = s->n, NA = rb::ct::NA, T = P.T;
  const size_t box_bytes = B * T * NA * 8, i_bytes = B * 4, x_bytes = B * n * 8;
  Carve cv;
  const size_t o_c = cv.take(B * NA * 8), o_M = cv.take(B * NA * rb::ct::NZP * 8), o_meta = cv.take(B * 16),
               o_y = cv.take(std::max<size_t>(static_cast<size_t>(s->ctl_steps) * s->ref_dim * 8, 8));
  size_t o_xl = 0, o_xh = 0, o_ol = 0, o_oh = 0, o_nb = 0, o_fs = 0, o_st = 0;
  if (!dev) {
    o_xl = cv.take(x_bytes);
    o_xh = cv.take(x_bytes);
    o_ol = cv.take(box_bytes);
    o_oh = cv.take(box_bytes);
    o_nb = cv.take(i_bytes);
    o_fs = cv.take(i_bytes);
    o_st = cv.take(i_bytes);
  }
  rc = ensure_ws(ctx, cv.off);
  if (rc) return rc;
  char* w = static_cast<char*>(ctx->ws);
  P.st_c = reinterpret_cast<double*>(w + o_c);
  P.st_M = reinterpret_cast<double*>(w + o_M);
  P.st_meta = reinterpret_cast<int*>(w + o_meta);
  P.y_ref = reinterpret_cast<double*>(w + o_y);
  if (s->ref_dim > 0)
    RB_CUDA(cudaMemcpyAsync(const_cast<double*>(P.y_ref), s->y_ref, static_cast<size_t>(s->ctl_steps) * s->ref_dim * 8,
                            cudaMemcpyHostToDevice, ctx->stream));
  if (dev) {
    P.x0_lo = x0_lo;
    P.x0_hi = x0_hi;
    P.out_lo = out->lo;
    P.out_hi = out->hi;
    P.n_boxes = out->n_boxes;
    P.failed_step = out->failed_step;
    P.status = out->status;
  } else {
    P.x0_lo = reinterpret_cast<double*>(w + o_xl);
    P.x0_hi = reinterpret_cast<double*>(w + o_xh);
    P.out_lo = reinterpret_cast<double*>(w + o_ol);
    P.out_hi = reinterpret_cast<double*>(w + o_oh);
    P.n_boxes = reinterpret_cast<int*>(w + o_nb);
    P.failed_step = reinterpret_cast<int*>(w + o_fs);
    P.status = reinterpret_cast<int*>(w + o_st);
    RB_CUDA(cudaMemcpyAsync(const_cast<double*>(P.x0_lo), x0_lo, x_bytes, cudaMemcpyHostToDevice, ctx->stream));
    RB_CUDA(cudaMemcpyAsync(const_cast<double*>(P.x0_hi), x0_hi, x_bytes, cudaMemcpyHostToDevice, ctx->stream));
  }
  rc = launch_cl(ctx, P);
  if (rc) return rc;
  if (!dev) {
    std::vector<int32_t> nb(B);
    RB_CUDA(cudaMemcpyAsync(nb.data(), P.n_boxes, i_bytes, cudaMemcpyDeviceToHost, ctx->stream));
    RB_CUDA(cudaMemcpyAsync(out->failed_step, P.failed_step, i_bytes, cudaMemcpyDeviceToHost, ctx->stream));
    RB_CUDA(cudaMemcpyAsync(out->status, P.status, i_bytes, cudaMemcpyDeviceToHost, ctx->stream));
    RB_CUDA(cudaStreamSynchronize(ctx->stream));
    std::memcpy(out->n_boxes, nb.data(), i_bytes);
    bool all_full = true;
    for (size_t i = 0; i < B; ++i) all_full &= (nb[i] == static_cast<int32_t>(T));
    if (all_full) {
      RB_CUDA(cudaMemcpyAsync(out->lo, P.out_lo, box_bytes, cudaMemcpyDeviceToHost, ctx->stream));
      RB_CUDA(cudaMemcpyAsync(out->hi, P.out_hi, box_bytes, cudaMemcpyDeviceToHost, ctx->stream));
    } else {
      for (size_t i = 0; i < B; ++i) {
        const size_t o = i * T * NA, cnt = static_cast<size_t>(nb[i]) * NA * 8;
        if (!cnt) continue;
        RB_CUDA(cudaMemcpyAsync(out->lo + o, P.out_lo + o, cnt, cudaMemcpyDeviceToHost, ctx->stream));
        RB_CUDA(cudaMemcpyAsync(out->hi + o, P.out_hi + o, cnt, cudaMemcpyDeviceToHost, ctx->stream));
      }
    }
    RB_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  return REACH_OK;
}

int reach_cl_split_hull(reach_ctx* ctx, const reach_net* ctl, const reach_cl_spec* s, const reach_cl_split_args* a,
                        const reach_hull_out* out, int32_t flags) {
  if (!ctx || !ctl || !s || !a || !out) return REACH_E_INVALID_ARGUMENT;
  int rc = validate_cl(ctx, ctl, s);
  if (rc) return rc;
  const int n = s->n;
  if (n > rb::kMaxSplitDims) return fail(ctx, REACH_E_UNSUPPORTED, "too many split dimensions");
  long long total = 1;
  for (int d = 0; d < n; ++d) {
    if (a->counts[d] < 1) return fail(ctx, REACH_E_INVALID_ARGUMENT, "SplitPlan: counts must be >= 1");
    total *= a->counts[d];
    if (total > (1ll << 20)) return fail(ctx, REACH_E_INVALID_ARGUMENT, "SplitPlan: total part count overflow");
    if (!std::isfinite(a->x0_lo[d]) || !std::isfinite(a->x0_hi[d]))
      return fail(ctx, REACH_E_INVALID_ARGUMENT, "build_linear_tm: diverged box");
  }
  const long long begin = a->part_begin, end = a->part_end <= 0 ? total : a->part_end;
  if (begin < 0 || begin >= end || end > total) return fail(ctx, REACH_E_INVALID_ARGUMENT, "bad part range");
  RB_CUDA(cudaSetDevice(ctx->device));
  const bool dev = (flags & REACH_FLAG_DEVICE_PTRS) != 0;
  rb::ct::CTParams P{};
  setup_params(ctx, ctl, s, end - begin, P);
  P.split = 1;
  P.part_begin = begin;
  for (int d = 0; d < n; ++d) {
    P.sx_lo[d] = a->x0_lo[d];
    P.sx_hi[d] = a->x0_hi[d];
    P.counts[d] = a->counts[d];
  }
  const size_t B = end - begin, NA = rb::ct::NA, T = P.T, cnt = T * NA;
  Carve cv;
  const size_t o_c = cv.take(B * NA * 8), o_M = cv.take(B * NA * rb::ct::NZP * 8), o_meta = cv.take(B * 16),
               o_y = cv.take(std::max<size_t>(static_cast<size_t>(s->ctl_steps) * s->ref_dim * 8, 8)),
               o_kl = cv.take(cnt * 8), o_kh = cv.take(cnt * 8), o_nan = cv.take(cnt * 8), o_div = cv.take(T * 4),
               o_nb = cv.take(4), o_key = cv.take(8), o_lo = cv.take(cnt * 8), o_hi = cv.take(cnt * 8);
  rc = ensure_ws(ctx, cv.off);
  if (rc) return rc;
  char* w = static_cast<char*>(ctx->ws);
  P.st_c = reinterpret_cast<double*>(w + o_c);
  P.st_M = reinterpret_cast<double*>(w + o_M);
  P.st_meta = reinterpret_cast<int*>(w + o_meta);
  P.y_ref = reinterpret_cast<double*>(w + o_y);
  P.hull_lo = reinterpret_cast<unsigned long long*>(w + o_kl);
  P.hull_hi = reinterpret_cast<unsigned long long*>(w + o_kh);
  P.hull_nan0 = reinterpret_cast<int*>(w + o_nan);
  P.hull_div = reinterpret_cast<int*>(w + o_div);
  P.hull_nboxes = reinterpret_cast<int*>(w + o_nb);
  P.hull_fail_key = reinterpret_cast<unsigned long long*>(w + o_key);
  if (s->ref_dim > 0)
    RB_CUDA(cudaMemcpyAsync(const_cast<double*>(P.y_ref), s->y_ref, static_cast<size_t>(s->ctl_steps) * s->ref_dim * 8,
                            cudaMemcpyHostToDevice, ctx->stream));
  const int icount = static_cast<int>(cnt), tpb = 256;
  ct_hull_init_kernel<<<std::max((std::max(icount, static_cast<int>(T)) + tpb - 1) / tpb, 1), tpb, 0, ctx->stream>>>(
      P.hull_lo, P.hull_hi, P.hull_nan0, P.hull_div, icount, static_cast<int>(T), P.hull_nboxes, P.hull_fail_key);
  RB_CUDA(cudaGetLastError());
  rc = launch_cl(ctx, P);
  if (rc) return rc;
  double* dlo = dev ? out->lo : reinterpret_cast<double*>(w + o_lo);
  double* dhi = dev ? out->hi : reinterpret_cast<double*>(w + o_hi);
  ct_hull_finalize_kernel<<<(icount + tpb - 1) / tpb, tpb, 0, ctx->stream>>>(P.hull_lo, P.hull_hi, P.hull_nan0, icount,
                                                                             dlo, dhi);
  RB_CUDA(cudaGetLastError());
  ctx->launches += 2;
  if (dev) {
    RB_CUDA(cudaMemcpyAsync(out->box_diverged, P.hull_div, T * 4, cudaMemcpyDeviceToDevice, ctx->stream));
    RB_CUDA(cudaMemcpyAsync(out->n_boxes, P.hull_nboxes, 4, cudaMemcpyDeviceToDevice, ctx->stream));
    RB_CUDA(cudaMemcpyAsync(out->fail_key, P.hull_fail_key, 8, cudaMemcpyDeviceToDevice, ctx->stream));
  } else {
    RB_CUDA(cudaMemcpyAsync(out->lo, dlo, cnt * 8, cudaMemcpyDeviceToHost, ctx->stream));
    RB_CUDA(cudaMemcpyAsync(out->hi, dhi, cnt * 8, cudaMemcpyDeviceToHost, ctx->stream));
    RB_CUDA(cudaMemcpyAsync(out->box_diverged, P.hull_div, T * 4, cudaMemcpyDeviceToHost, ctx->stream));
    RB_CUDA(cudaMemcpyAsync(out->n_boxes, P.hull_nboxes, 4, cudaMemcpyDeviceToHost, ctx->stream));
    RB_CUDA(cudaMemcpyAsync(out->fail_key, P.hull_fail_key, 8, cudaMemcpyDeviceToHost, ctx->stream));
    RB_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  return REACH_OK;
}

}  // extern "C"
