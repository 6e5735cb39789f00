// C ABI of the B200 reachability library (include/reach_b200.h).
//
// Host side: context (device, stream, workspaces), immutable network upload
// (weights laid out once for the kernels: W row-major and W^T, 16-byte padded
// rows, one blob), argument validation with the reference's error behaviour,
// and the launches.  No CPU fallback: every entry point runs the CUDA kernels
// or returns an error.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <functional>
#include <cmath>
#include <limits>
#include <memory>
#include <climits>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "cem_kernel.cuh"
#include "coll.h"
#include "tc_capi.h"
#include "../../include/reach_b200.h"
#include "diag.cuh"
#include "dual_kernel.cuh"
#include "ct_dual.cuh"
#include "dt_kernel.cuh"
#include "plan.cuh"
#include "wide_kernel.cuh"

namespace rb {  // wide_inst.cu, one object per rows-per-thread value
cudaError_t wide_call_rd1(int rc, const DTParams* P, size_t smem, int grid, int* occ, cudaStream_t s);
cudaError_t wide_call_rd2(int rc, const DTParams* P, size_t smem, int grid, int* occ, cudaStream_t s);
cudaError_t wide_call_rd4(int rc, const DTParams* P, size_t smem, int grid, int* occ, cudaStream_t s);
cudaError_t wide_call_rd9(int rc, const DTParams* P, size_t smem, int grid, int* occ, cudaStream_t s);
}  // namespace rb
namespace rbh {  // REACH_PREC_FUSED builds (dt_fused.cu)
cudaError_t wide_call_fused_rd1(int rc, const void* P, size_t smem, int grid, int* occ, cudaStream_t s);
cudaError_t wide_call_fused_rd2(int rc, const void* P, size_t smem, int grid, int* occ, cudaStream_t s);
cudaError_t wide_call_fused_rd4(int rc, const void* P, size_t smem, int grid, int* occ, cudaStream_t s);
cudaError_t wide_call_fused_rd9(int rc, const void* P, size_t smem, int grid, int* occ, cudaStream_t s);
cudaError_t launch_dt_fused(const void* P, int no, int cpl, unsigned grid, unsigned threads, size_t smem,
                            cudaStream_t s);
size_t fused_params_size();
}  // namespace rbh
namespace rb {
}  // namespace rb

#include <atomic>
#include <random>
#include <thread>

#include "ctx.cuh"

using namespace rbh;

namespace {

// Launch geometry and shared-memory carve-up of the DT horizon kernel.
struct DTLayout {
  int spc = 0, no = 0, cpl = 0;
  size_t smem = 0;
  bool wide = false;  // dt_wide_kernel<rd, rc>, grid CTAs persistent over the batch
  int rd = 0, rc = 0, grid = 0;
  bool tcw = false;   // dt_tcw_kernel (REACH_PREC_TC), grid CTAs persistent over the batch
  bool fused = false; // REACH_PREC_FUSED: the same kernel from the RB_FUSED build (dt_fused.cu)
  rb::TcwParams tx{};
};

// Two 48 KB bulk-copy stages (double buffering with 48-row chunks of a 128-wide layer): fewer, larger
// chunks than the earlier 6 x 16 KB ring cut the per-chunk acquire / release / row-count overhead
// (C4 sweep 116.7 -> 104.1 ms; measured sweep in profiles/r01_c4_summary.md).
constexpr int kStageDoublesDefault = 6144;
constexpr int kNStageDefault = 2;
// host-pointer DT calls whose device workspace is at most this large stage through pinned memory (one
// copy in, one copy out)
constexpr size_t kSmallCallBytes = 1u << 20;

// Weight-stream ring geometry; RB_NSTAGE / RB_STAGE_DOUBLES override it for tuning runs.
int env_int(const char* name, int dflt, int lo, int hi) {
  const char* v = std::getenv(name);
  if (!v) return dflt;
  int x = std::atoi(v);
  return (x < lo || x > hi) ? dflt : x;
}

int cpl_for(int maxh) { return maxh <= 32 ? 1 : maxh <= 64 ? 2 : maxh <= 96 ? 3 : maxh <= 128 ? 4 : maxh <= 256 ? 8 : 0; }

// Layout of the horizon kernel for the one-step network `net` (open loop) or
// the dynamics `net` + controller `ctl` (closed loop, l = ctl output dim).
int plan_warp(reach_ctx* ctx, const reach_net* net, int n, int m, int window, rb::DTParams& P, DTLayout& lay,
              const reach_net* ctl) {
  const int L = net->L;
  const int l = ctl ? ctl->dims[ctl->L] : 0;
  const int cap = window > 0 ? window : 1;
  const int rows_max = std::max(n, l);
  const int no = rows_max <= 2 ? 2 : rows_max <= 4 ? 4 : rows_max <= 6 ? 6 : rows_max <= 8 ? 8 : 0;
  if (no == 0) return fail(ctx, REACH_E_UNSUPPORTED, "state dim > 8 not in this kernel family");
  if (net->cpl == 0 || (ctl && ctl->cpl == 0))
    return fail(ctx, REACH_E_UNSUPPORTED, "hidden width > 256 not in this kernel family");
  if (ctl && ctl->cpl != net->cpl)
    return fail(ctx, REACH_E_UNSUPPORTED, "controller and dynamics hidden widths in different kernel families");
  const int hp = net->hp;
  const int n_i = n + l;  // rows of the certified input TM
  const int wmax = n + l;  // widest generator block
  const int nzs = n + (cap + 2) * wmax;  // G0 + queue (<= cap + 2 blocks before a fold)
  if (n + (cap + 1) * wmax > 64) return fail(ctx, REACH_E_UNSUPPORTED, "generator matrix wider than 64 columns");
  if (n * n_i > 64 || n + wmax > 32) return fail(ctx, REACH_E_UNSUPPORTED, "state/control dims too large");
  const int nop = (no + 1) & ~1;
  const int Lmax = std::max(L, ctl ? ctl->L : 0);
  auto ev = [](int x) { return (x + 1) & ~1; };
  int off = 0;
  P.o_stA = off;
  off += ev(n * nzs);
  P.o_c = off;
  off += ev(n);
  P.o_pre = off;
  off += (Lmax - 1) * 2 * hp;
  P.o_LT = off;  // also the IBP input buffer (2 hp) and the fold scratch
  const int fold_scr = n * (n + wmax) + 2 * n * wmax + n;
  off += ev(std::max({nop * std::max(hp, n_i + m), 2 * std::max(hp, n_i), fold_scr}));
  bool tanh_any = false;
  for (int i = 0; i + 1 < L; ++i) tanh_any |= net->acts[i] == REACH_ACT_TANH;
  if (ctl)
    for (int i = 0; i + 1 < ctl->L; ++i) tanh_any |= ctl->acts[i] == REACH_ACT_TANH;
  P.has_tanh = tanh_any ? 1 : 0;
  P.o_R = off;
  if (tanh_any) off += 3 * hp;
  P.o_bf0 = off;
  if (m > 0) off += std::max(hp, ev(n));
  P.o_idx = off;  // per hidden layer two unit bitmasks (active, unstable) + the active-unit list
  off += ev(((Lmax - 1) * 2 * (hp / 32) * 4 + (Lmax - 1) * hp + 7) / 8);
  P.o_wid = off;  // generator block widths
  off += ev((cap + 4 + 1) / 2);
  P.o_aug = off;
  P.ldag = nzs;
  if (ctl) off += ev(n_i * nzs);
  P.o_cag = off;
  if (ctl) off += ev(n_i);
  P.warp_doubles = ev(off);
  P.nzs = nzs;
  P.hp = hp;
  int boff = 0;
  for (int i = 0; i < L; ++i) {
    P.bias_s_off[i] = boff;
    boff += (i + 1 < L) ? hp : ev(net->dims[i + 1]);
  }
  if (ctl)
    for (int i = 0; i < ctl->L; ++i) {
      P.bias_s_off_ctl[i] = boff;
      boff += (i + 1 < ctl->L) ? hp : ev(ctl->dims[i + 1]);
    }
  P.bias_doubles = ev(boff);
  const int kNStage = env_int("RB_NSTAGE", kNStageDefault, 2, 8);
  // Stage size: RB_STAGE_DOUBLES, else the largest stage (<= kStageDoublesDefault) that keeps
  // kSampleWarps sample warps resident -- residency beats chunk size on this latency-bound kernel
  // (C4 fused: 8 warps x 48 KB stages 74.8 ms, 12 warps x 21 KB stages 69.1 ms, tools/warp_sweep.sh);
  // fewer warps only when one row of the widest streamed matrix no longer fits a stage.
  int kStageDoubles = env_int("RB_STAGE_DOUBLES", 0, 512, 8192) & ~1;
  if (kStageDoubles == 0) {
    int maxld = 0;
    auto scan = [&](const reach_net* nt) {
      for (int i = 0; i < nt->dev.L; ++i) maxld = std::max({maxld, nt->dev.ldw[i], i + 1 < nt->dev.L ? nt->dev.ldt[i] : 0});
    };
    scan(net);
    if (ctl) scan(ctl);
    const long long base = rb::kHeaderBytes + static_cast<long long>(P.bias_doubles) * 8;
    const long long per = static_cast<long long>(P.warp_doubles) * 8;
    for (int spc_t = rb::kSampleWarps; spc_t >= 1; --spc_t) {
      const long long avail = (static_cast<long long>(ctx->max_smem) - base - spc_t * per) / (kNStage * 8ll);
      kStageDoubles = static_cast<int>(std::min<long long>(kStageDoublesDefault, std::max<long long>(avail, 0))) & ~1;
      if (kStageDoubles >= maxld) break;
    }
    if (kStageDoubles < 512) kStageDoubles = std::max(512, maxld + (maxld & 1));
  }
  P.stage_doubles = kStageDoubles;
  P.nstage = kNStage;
  // weight-stream chunk table of one DT step (consumption order of the kernel), absolute addresses
  int nc = 0;
  auto add_matrix = [&](const double* base, long long moff, int rows, int ld) -> bool {
    if (ld > kStageDoubles) return false;
    const int rpc = std::max(1, kStageDoubles / ld);
    for (int r0 = 0; r0 < rows; r0 += rpc) {
      if (nc >= rb::kMaxChunks) return false;
      const int nr = std::min(rpc, rows - r0);
      P.ch_off[nc] = reinterpret_cast<long long>(base + moff + static_cast<long long>(r0) * ld);
      P.ch_bytes[nc] = static_cast<unsigned>(nr) * ld * 8u;
      ++nc;
    }
    return true;
  };
  auto add_net = [&](const reach_net* nt) -> bool {
    const rb::DevNet& d = nt->dev;
    bool ok = true;
    for (int i = 0; i + 1 < d.L; ++i) ok = ok && add_matrix(nt->blob, d.wt_off[i], d.dims[i], d.ldt[i]);
    for (int i = d.L - 1; i >= 0; --i) ok = ok && add_matrix(nt->blob, d.w_off[i], d.dims[i + 1], d.ldw[i]);
    return ok;
  };
  bool ok = true;
  if (ctl) ok = add_net(ctl);
  ok = ok && add_net(net);
  if (!ok) return fail(ctx, REACH_E_UNSUPPORTED, "network too large for the weight stream");
  P.n_chunks_step = nc;
  P.l = l;
  if (ctl) P.ctl = ctl->dev;
  const size_t fixed =
      rb::kHeaderBytes + static_cast<size_t>(kNStage) * kStageDoubles * 8 + static_cast<size_t>(P.bias_doubles) * 8;
  const size_t per = static_cast<size_t>(P.warp_doubles) * 8;
  int spc = static_cast<int>((static_cast<size_t>(ctx->max_smem) - fixed) / per);
  spc = std::min(spc, rb::kSampleWarps);
  if (spc < 1) return fail(ctx, REACH_E_UNSUPPORTED, "per-sample working set exceeds shared memory");
  lay.spc = spc;
  lay.no = no;
  lay.cpl = net->cpl;
  lay.smem = fixed + per * spc;
  // tuning knob: pad the allocation to force fewer CTAs per SM (RB_MIN_SMEM_KB)
  lay.smem = std::max<size_t>(lay.smem, static_cast<size_t>(env_int("RB_MIN_SMEM_KB", 0, 0, 227)) * 1024);
  return REACH_OK;
}

int wide_rows_pick(int rows) { return rows <= 8 ? 1 : rows <= 16 ? 2 : rows <= 32 ? 4 : rows <= 72 ? 9 : 0; }

cudaError_t wide_dispatch(const rb::DTParams* P, const DTLayout& lay, int* occ, cudaStream_t s) {
  if (lay.fused) {
    switch (lay.rd) {
      case 1: return rbh::wide_call_fused_rd1(lay.rc, P, lay.smem, lay.grid, occ, s);
      case 2: return rbh::wide_call_fused_rd2(lay.rc, P, lay.smem, lay.grid, occ, s);
      case 4: return rbh::wide_call_fused_rd4(lay.rc, P, lay.smem, lay.grid, occ, s);
      case 9: return rbh::wide_call_fused_rd9(lay.rc, P, lay.smem, lay.grid, occ, s);
      default: return cudaErrorInvalidValue;
    }
  }
  switch (lay.rd) {
    case 1: return rb::wide_call_rd1(lay.rc, P, lay.smem, lay.grid, occ, s);
    case 2: return rb::wide_call_rd2(lay.rc, P, lay.smem, lay.grid, occ, s);
    case 4: return rb::wide_call_rd4(lay.rc, P, lay.smem, lay.grid, occ, s);
    case 9: return rb::wide_call_rd9(lay.rc, P, lay.smem, lay.grid, occ, s);
    default: return cudaErrorInvalidValue;
  }
}

// Layout of the wide (CTA-per-sample) family: Lambda^T, the cp.async ring, the
// relaxations and small per-sample vectors in shared memory; two symbolic-state
// buffers per CTA in global memory.
int plan_wide(reach_ctx* ctx, const reach_net* net, int n, int m, int window, long long B, rb::DTParams& P,
              DTLayout& lay, const reach_net* ctl) {
  const int l = ctl ? ctl->dims[ctl->L] : 0;
  const int cap = window > 0 ? window : 1;
  const int n_i = n + l;
  const int rd = wide_rows_pick(n), rc = l == 0 ? 0 : l <= 8 ? 1 : l <= 24 ? 3 : -1;
  if (rd == 0 || rc < 0 || n > 128)
    return fail(ctx, REACH_E_UNSUPPORTED, "state/control dims outside the wide kernel family (n <= 72, l <= 24)");
  int hw = n_i;
  auto widths = [&](const reach_net* nt) {
    for (int i = 0; i + 1 < nt->L; ++i) hw = std::max(hw, nt->dims[i + 1]);
  };
  widths(net);
  if (ctl) widths(ctl);
  if (hw > rb::kWideSW) return fail(ctx, REACH_E_UNSUPPORTED, "layer width > 256 not in the wide kernel family");
  const int lmax = std::max(net->L, ctl ? ctl->L : 0);
  auto ev = [](long long x) { return (x + 1) & ~1ll; };
  const int nop = std::max(8 * rd, 8 * rc) | 1;
  long long off = static_cast<long long>(nop) * hw;
  P.w_o_stage = static_cast<int>(ev(off));
  off = P.w_o_stage + rb::kWideNS * rb::kWideRS * rb::kWideSW;
  P.w_o_relax = static_cast<int>(off);
  off += static_cast<long long>(std::max(lmax - 1, 1)) * hw * 4;
  P.w_o_bf0 = static_cast<int>(off);
  const int wmax = n + l;
  const long long fold_need = static_cast<long long>(n) * (n + 2 * wmax) + 4 * n;
  if (fold_need > P.w_o_bf0) return fail(ctx, REACH_E_UNSUPPORTED, "fold scratch exceeds shared memory");
  off += hw;
  P.w_o_misc = static_cast<int>(off);
  const int nomax = std::max(n, l);
  off += n + n_i + 2 * n + 3 * nomax + std::max(l, 1) + n + 32;
  P.w_o_int = static_cast<int>(ev(off));
  // the ring mbarriers (8 x 8 B) after the int region (48 ints + the active-unit lists)
  const size_t ints = 48 * 4 + static_cast<size_t>(std::max(lmax - 1, 1)) * 256;
  P.w_o_bar = P.w_o_int + static_cast<int>((ints + 15) / 16 * 2);
  const size_t bytes = static_cast<size_t>(P.w_o_bar) * 8 + 8 * 8;
  if (bytes > static_cast<size_t>(ctx->max_smem))
    return fail(ctx, REACH_E_UNSUPPORTED, "wide kernel working set exceeds shared memory");
  P.w_nop = nop;
  P.w_hw = hw;
  P.w_rows = n + l;
  P.w_lds = static_cast<int>(ev(n + static_cast<long long>(cap + 2) * wmax));
  P.wws_stride = ev(2ll * P.w_rows * P.w_lds);
  P.l = l;
  if (ctl) P.ctl = ctl->dev;
  lay.wide = true;
  lay.rd = rd;
  lay.rc = rc;
  lay.smem = bytes;
  int occ = 0;
  cudaError_t e = wide_dispatch(nullptr, lay, &occ, nullptr);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "wide kernel setup");
  if (occ < 1) return fail(ctx, REACH_E_UNSUPPORTED, "wide kernel does not fit on an SM");
  lay.grid = static_cast<int>(std::min<long long>(B, static_cast<long long>(occ) * ctx->num_sms));
  const size_t need = static_cast<size_t>(lay.grid) * P.wws_stride * 8;
  if (need > ctx->wws_bytes) {
    if (ctx->wws) {
      cudaStreamSynchronize(ctx->stream);
      cudaFree(ctx->wws);
      ctx->wws = nullptr;
      ctx->wws_bytes = 0;
    }
    RB_CUDA(cudaMalloc(&ctx->wws, need));
    ctx->wws_bytes = need;
  }
  P.wws = static_cast<double*>(ctx->wws);
  if (env_int("RB_WIDE_PHASE", 0, 0, 1)) {
    if (!ctx->wphase) {
      RB_CUDA(cudaMalloc(&ctx->wphase, 16 * sizeof(unsigned long long)));
      RB_CUDA(cudaMemset(ctx->wphase, 0, 16 * sizeof(unsigned long long)));
    }
    P.w_phase = ctx->wphase;
  }
  return REACH_OK;
}

// Kernel family choice: the warp-per-sample kernel when the sample fits a
// warp's shared-memory slice, else the wide CTA-per-sample kernel
// (RB_FORCE_WIDE=1 forces the wide family, for parity runs of both).
int plan_dt(reach_ctx* ctx, const reach_net* net, int n, int m, int window, long long B, rb::DTParams& P,
            DTLayout& lay, const reach_net* ctl = nullptr, int prec = REACH_PREC_EXACT) {
  // a network without a hidden layer has no Lambda.W contraction for the tensor cores (only the prepended
  // [A | I] layer): the tensor-core mode is then the exact mode
  if (prec == REACH_PREC_TC && net->L < 2 && (!ctl || ctl->L < 2)) prec = REACH_PREC_EXACT;
  if (prec == REACH_PREC_TC) {
    const int rc = plan_wide(ctx, net, n, m, window, B, P, lay, ctl);
    if (rc) return rc;
    const int rt = rbh::plan_tcw(ctx, net, ctl, n, B, P, lay.smem, lay.grid, lay.tx);
    if (rt) return rt;
    lay.tcw = true;
    return REACH_OK;
  }
  if (prec != REACH_PREC_EXACT && prec != REACH_PREC_FUSED)
    return fail(ctx, REACH_E_INVALID_ARGUMENT, "unknown precision mode");
  static_assert(sizeof(rb::DTParams) > 0, "");
  if (prec == REACH_PREC_FUSED && rbh::fused_params_size() != sizeof(rb::DTParams))
    return fail(ctx, REACH_E_CUDA, "fused build out of step with the exact build (DTParams layout)");
  const bool fused = prec == REACH_PREC_FUSED;
  if (!env_int("RB_FORCE_WIDE", 0, 0, 1)) {
    lay.fused = fused;
    const int rc = plan_warp(ctx, net, n, m, window, P, lay, ctl);
    if (rc != REACH_E_UNSUPPORTED) return rc;
    const std::string why = ctx->err;
    P = rb::DTParams{};
    lay = DTLayout{};
    lay.fused = fused;
    const int rw = plan_wide(ctx, net, n, m, window, B, P, lay, ctl);
    if (rw == REACH_E_UNSUPPORTED) ctx->err = why + "; " + ctx->err;
    return rw;
  }
  lay.fused = fused;
  return plan_wide(ctx, net, n, m, window, B, P, lay, ctl);
}

template <int NO, int CPL>
cudaError_t launch_dt_t(const rb::DTParams& P, const DTLayout& lay, long long B, cudaStream_t s) {
  auto k = rb::dt_horizon_kernel<NO, CPL>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(lay.smem));
  if (e != cudaSuccess) return e;
  const long long grid = (B + lay.spc - 1) / lay.spc;
  k<<<static_cast<unsigned>(grid), 32 * lay.spc, lay.smem, s>>>(P);
  return cudaGetLastError();
}

template <int NO>
cudaError_t launch_dt_no(const rb::DTParams& P, const DTLayout& lay, long long B, cudaStream_t s) {
  switch (lay.cpl) {
    case 1: return launch_dt_t<NO, 1>(P, lay, B, s);
    case 2: return launch_dt_t<NO, 2>(P, lay, B, s);
    case 3: return launch_dt_t<NO, 3>(P, lay, B, s);
    case 4: return launch_dt_t<NO, 4>(P, lay, B, s);
    default: return launch_dt_t<NO, 8>(P, lay, B, s);
  }
}

cudaError_t launch_dt(const rb::DTParams& P, const DTLayout& lay, long long B, cudaStream_t s) {
  if (lay.tcw) return rbh::tcw_launch(P, lay.tx, lay.smem, lay.grid, s);
  if (lay.wide) return wide_dispatch(&P, lay, nullptr, s);
  if (lay.fused)
    return rbh::launch_dt_fused(&P, lay.no, lay.cpl, static_cast<unsigned>((B + lay.spc - 1) / lay.spc),
                                32u * lay.spc, lay.smem, s);
  switch (lay.no) {
    case 2: return launch_dt_no<2>(P, lay, B, s);
    case 4: return launch_dt_no<4>(P, lay, B, s);
    case 6: return launch_dt_no<6>(P, lay, B, s);
    default: return launch_dt_no<8>(P, lay, B, s);
  }
}

// Validation mirroring DTSystem::validate (dt_reach.hpp:23-28) and MLPNet::validate (neural.hpp:49-56).
int validate_system(reach_ctx* ctx, const reach_net* net, int n, int m) {
  if (n <= 0 || m < 0) return fail(ctx, REACH_E_INVALID_ARGUMENT, "DTSystem: invalid dimensions");
  if (net->dims[0] != n + m || net->dims[net->L] != n)
    return fail(ctx, REACH_E_INVALID_ARGUMENT, "DTSystem: one-step map shape mismatch");
  return REACH_OK;
}

}  // namespace

extern "C" {

int reach_abi_version(void) { return REACH_B200_ABI_VERSION; }

const char* reach_tube_status_string(int32_t status) {
  switch (status) {
    case REACH_TUBE_OK: return "";
    case REACH_TUBE_NONFINITE_PREACT: return "relax_activation: non-finite preactivation";
    case REACH_TUBE_DIVERGED_CERT: return "diverged certification";
    case REACH_TUBE_DIVERGED_BOX: return "diverged box";
    case REACH_TUBE_CTL_FAILED: return "controller certification failed: relax_activation: non-finite preactivation";
    case REACH_TUBE_CTL_DIVERGED: return "controller certification diverged";
    case REACH_TUBE_REMAINDER: return "remainder not contractive after max enlargements (reduce h)";
    case REACH_TUBE_PICARD_NONFINITE: return "poly_picard: non-finite coefficients";
    case REACH_TUBE_TME_INV: return "tme_inv: range contains zero";
    default: return "error";
  }
}

int reach_ctx_create(int32_t device, reach_ctx** out) {
  if (!out) return REACH_E_INVALID_ARGUMENT;
  *out = nullptr;
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count <= 0) return REACH_E_NO_DEVICE;
  if (device < 0 || device >= count) return REACH_E_INVALID_ARGUMENT;
  reach_ctx* ctx = new reach_ctx();
  ctx->device = device;
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->own, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&ctx->max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  if (e != cudaSuccess) {
    delete ctx;
    return REACH_E_CUDA;
  }
  ctx->stream = ctx->own;
  *out = ctx;
  return REACH_OK;
}

int reach_ctx_destroy(reach_ctx* ctx) {
  rbh::DeviceGuard device_guard_(ctx);
  if (!ctx) return REACH_OK;
  cudaSetDevice(ctx->device);
  rbh::coll_release(ctx);
  if (ctx->ws) cudaFree(ctx->ws);
  if (ctx->pbuf) cudaFree(ctx->pbuf);
  if (ctx->wws) cudaFree(ctx->wws);
  if (ctx->wphase) cudaFree(ctx->wphase);
  if (ctx->ctd_ws) cudaFree(ctx->ctd_ws);
  if (ctx->aux) {
    cudaStreamSynchronize(ctx->aux);
    cudaStreamDestroy(ctx->aux);
    cudaEventDestroy(ctx->ev_fork);
    cudaEventDestroy(ctx->ev_join);
  }
  if (ctx->hpin) cudaFreeHost(ctx->hpin);
  for (auto& p : ctx->ev_used) { cudaEventDestroy(p.first); cudaEventDestroy(p.second); }
  for (auto& p : ctx->ev_free) { cudaEventDestroy(p.first); cudaEventDestroy(p.second); }
  if (ctx->own) cudaStreamDestroy(ctx->own);
  delete ctx;
  return REACH_OK;
}

int reach_ctx_set_stream(reach_ctx* ctx, void* s) {
  rbh::DeviceGuard device_guard_(ctx);
  if (!ctx) return REACH_E_INVALID_ARGUMENT;
  ctx->stream = s ? static_cast<cudaStream_t>(s) : ctx->own;
  return REACH_OK;
}

int reach_ctx_synchronize(reach_ctx* ctx) {
  rbh::DeviceGuard device_guard_(ctx);
  if (!ctx) return REACH_E_INVALID_ARGUMENT;
  RB_CUDA(cudaStreamSynchronize(ctx->stream));
  return REACH_OK;
}

int reach_ctx_enable_kernel_timing(reach_ctx* ctx, int32_t on) {
  rbh::DeviceGuard device_guard_(ctx);
  if (!ctx) return REACH_E_INVALID_ARGUMENT;
  ctx->timing = on != 0;
  return REACH_OK;
}

int reach_ctx_kernel_time(reach_ctx* ctx, double* total_ms, int64_t* launches) {
  rbh::DeviceGuard device_guard_(ctx);
  if (!ctx || !total_ms || !launches) return REACH_E_INVALID_ARGUMENT;
  RB_CUDA(cudaSetDevice(ctx->device));
  RB_CUDA(cudaStreamSynchronize(ctx->stream));
  double tot = 0.0;
  for (auto& p : ctx->ev_used) {
    float ms = 0.f;
    RB_CUDA(cudaEventElapsedTime(&ms, p.first, p.second));
    tot += ms;
    ctx->ev_free.push_back(p);
  }
  *total_ms = tot;
  *launches = static_cast<int64_t>(ctx->ev_used.size());
  ctx->ev_used.clear();
  return REACH_OK;
}

int reach_measure_fp64_peak(reach_ctx* ctx, double* tflops_fma, double* tflops_muladd) {
  rbh::DeviceGuard device_guard_(ctx);
  if (!ctx || !tflops_fma || !tflops_muladd) return REACH_E_INVALID_ARGUMENT;
  RB_CUDA(cudaSetDevice(ctx->device));
  double* dout = nullptr;
  RB_CUDA(cudaMalloc(&dout, 8));
  cudaEvent_t a, b;
  RB_CUDA(cudaEventCreate(&a));
  RB_CUDA(cudaEventCreate(&b));
  const int blocks = ctx->num_sms * 8, threads = 256, iters = 4096;
  const double work = static_cast<double>(blocks) * threads * iters * 16;  // instructions
  double best_fma = 0, best_ma = 0;
  for (int rep = 0; rep < 6; ++rep) {
    float ms = 0;
    RB_CUDA(cudaEventRecord(a, ctx->stream));
    rb::fp64_fma_peak_kernel<<<blocks, threads, 0, ctx->stream>>>(dout, iters, 0.999999, 1e-7);
    RB_CUDA(cudaEventRecord(b, ctx->stream));
    RB_CUDA(cudaEventSynchronize(b));
    RB_CUDA(cudaEventElapsedTime(&ms, a, b));
    if (rep > 0) best_fma = std::max(best_fma, 2.0 * work / (ms * 1e-3) / 1e12);
    RB_CUDA(cudaEventRecord(a, ctx->stream));
    rb::fp64_muladd_peak_kernel<<<blocks, threads, 0, ctx->stream>>>(dout, iters, 0.999999, 1e-7);
    RB_CUDA(cudaEventRecord(b, ctx->stream));
    RB_CUDA(cudaEventSynchronize(b));
    RB_CUDA(cudaEventElapsedTime(&ms, a, b));
    if (rep > 0) best_ma = std::max(best_ma, 2.0 * work / (ms * 1e-3) / 1e12);
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(dout);
  *tflops_fma = best_fma;
  *tflops_muladd = best_ma;
  return REACH_OK;
}

int reach_debug_phase_cycles(reach_ctx* ctx, uint64_t* out, int32_t count) {
  rbh::DeviceGuard device_guard_(ctx);
  if (!ctx || !out || count <= 0) return REACH_E_INVALID_ARGUMENT;
  if (ctx->wphase) {  // wide family, runtime-enabled counters
    RB_CUDA(cudaSetDevice(ctx->device));
    RB_CUDA(cudaStreamSynchronize(ctx->stream));
    unsigned long long tmp[16] = {0};
    RB_CUDA(cudaMemcpy(tmp, ctx->wphase, sizeof(tmp), cudaMemcpyDeviceToHost));
    for (int i = 0; i < count && i < 16; ++i) out[i] = tmp[i];
    RB_CUDA(cudaMemset(ctx->wphase, 0, sizeof(tmp)));
    return REACH_OK;
  }
#ifdef RB_PHASE_TIMING
  RB_CUDA(cudaSetDevice(ctx->device));
  RB_CUDA(cudaStreamSynchronize(ctx->stream));
  unsigned long long tmp[16] = {0};
  RB_CUDA(cudaMemcpyFromSymbol(tmp, rb::g_phase_cycles, sizeof(tmp)));
  for (int i = 0; i < count && i < 16; ++i) out[i] = tmp[i];
  unsigned long long zero[16] = {0};
  RB_CUDA(cudaMemcpyToSymbol(rb::g_phase_cycles, zero, sizeof(zero)));
  return REACH_OK;
#else
  return fail(ctx, REACH_E_UNSUPPORTED, "library built without RB_PHASE_TIMING");
#endif
}

const char* reach_ctx_last_error(const reach_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int64_t reach_ctx_launch_count(const reach_ctx* ctx) { return ctx ? ctx->launches : 0; }

int reach_net_upload(reach_ctx* ctx, const reach_net_desc* d, reach_net** out) {
  rbh::DeviceGuard device_guard_(ctx);
  if (!ctx || !d || !out) return REACH_E_INVALID_ARGUMENT;
  *out = nullptr;
  if (d->n_layers < 1) return fail(ctx, REACH_E_INVALID_ARGUMENT, "MLPNet: empty");
  if (d->n_layers > rb::kMaxLayers) return fail(ctx, REACH_E_UNSUPPORTED, "too many layers");
  for (int l = 0; l < d->n_layers; ++l) {
    if (d->dims[l] <= 0 || d->dims[l + 1] <= 0) return fail(ctx, REACH_E_INVALID_ARGUMENT, "MLPNet: empty layer");
    if (d->acts[l] < 0 || d->acts[l] > 2) return fail(ctx, REACH_E_INVALID_ARGUMENT, "unknown activation");
  }
  if (d->acts[d->n_layers - 1] != REACH_ACT_IDENTITY)
    return fail(ctx, REACH_E_INVALID_ARGUMENT, "MLPNet: final activation must be identity");
  RB_CUDA(cudaSetDevice(ctx->device));
  reach_net* net = new reach_net();
  net->L = d->n_layers;
  net->dims.assign(d->dims, d->dims + d->n_layers + 1);
  net->acts.assign(d->acts, d->acts + d->n_layers);
  {
    size_t np = 0;
    for (int l = 0; l < d->n_layers; ++l) np += static_cast<size_t>(d->dims[l + 1]) * (d->dims[l] + 1);
    net->params.assign(d->params, d->params + np);
  }
  // host blob, laid out for the kernels: per layer W (rows x ldw) and W^T
  // (cols x ldt), zero-padded so that hidden layers span the padded width
  // hp = 32 * cpl (no per-column guards in the kernels), biases padded to 32.
  int maxh = 0;
  for (int l = 0; l + 1 < d->n_layers; ++l) maxh = std::max(maxh, d->dims[l + 1]);
  net->cpl = cpl_for(maxh);
  net->hp = 32 * std::max(net->cpl, 1);
  const int hp = net->hp;
  const int L = d->n_layers;
  std::vector<double> blob;
  auto ev = [](int x) { return (x + 1) & ~1; };
  auto r32 = [](int x) { return (x + 31) / 32 * 32; };
  size_t src = 0;
  rb::DevNet& dn = net->dev;
  dn.L = L;
  for (int l = 0; l <= L; ++l) dn.dims[l] = d->dims[l];
  for (int l = 0; l < L; ++l) {
    const int rows = d->dims[l + 1], cols = d->dims[l];
    dn.acts[l] = d->acts[l];
    dn.ldw[l] = (l >= 1) ? std::max(r32(cols), hp) : ev(cols);
    dn.ldt[l] = (l + 1 < L) ? std::max(r32(rows), hp) : ev(rows);
    const double* w = d->params + src;
    const double* b = w + static_cast<size_t>(rows) * cols;
    src += static_cast<size_t>(rows) * cols + rows;
    dn.w_off[l] = static_cast<long long>(blob.size());
    blob.resize(blob.size() + static_cast<size_t>(rows) * dn.ldw[l], 0.0);
    for (int i = 0; i < rows; ++i)
      for (int j = 0; j < cols; ++j) blob[dn.w_off[l] + static_cast<size_t>(i) * dn.ldw[l] + j] = w[static_cast<size_t>(i) * cols + j];
    dn.wt_off[l] = static_cast<long long>(blob.size());
    blob.resize(blob.size() + static_cast<size_t>(cols) * dn.ldt[l], 0.0);
    for (int i = 0; i < rows; ++i)
      for (int j = 0; j < cols; ++j) blob[dn.wt_off[l] + static_cast<size_t>(j) * dn.ldt[l] + i] = w[static_cast<size_t>(i) * cols + j];
    dn.b_off[l] = static_cast<long long>(blob.size());
    blob.resize(blob.size() + std::max(r32(rows), hp), 0.0);
    for (int i = 0; i < rows; ++i) blob[dn.b_off[l] + i] = b[i];
  }
  cudaError_t e = cudaMalloc(&net->blob, blob.size() * sizeof(double));
  if (e == cudaSuccess) e = cudaMemcpy(net->blob, blob.data(), blob.size() * sizeof(double), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    if (net->blob) cudaFree(net->blob);
    delete net;
    return cuda_fail(ctx, e, "reach_net_upload");
  }
  dn.blob = net->blob;
  *out = net;
  return REACH_OK;
}

int reach_net_free(reach_ctx* ctx, reach_net* net) {
  rbh::DeviceGuard device_guard_(ctx);
  if (!net) return REACH_OK;
  if (ctx) cudaSetDevice(ctx->device);
  if (net->blob) cudaFree(net->blob);
  rbh::free_oz(net);
  delete net;
  return REACH_OK;
}

}  // extern "C"

namespace {
int run_dt_batch(reach_ctx* ctx, const reach_net* net, const reach_net* ctl, const reach_dt_args* a,
                 const reach_tube_out* out, int32_t flags) {
  int rc = 0;
  if (a->batch == 0) return REACH_OK;
  RB_CUDA(cudaSetDevice(ctx->device));
  rb::DTParams P{};
  DTLayout lay;
  rc = plan_dt(ctx, net, a->n, a->m, a->window, a->batch, P, lay, ctl, flags & REACH_FLAG_PREC_MASK);
  if (rc) return rc;
  P.net = net->dev;
  P.B = a->batch;
  P.H = a->horizon;
  P.n = a->n;
  P.m = a->m;
  P.window = a->window;
  P.rebuild = a->rebuild_from_box;
  P.actions_shared = a->actions_shared;
  const size_t B = static_cast<size_t>(a->batch), H = static_cast<size_t>(a->horizon), n = a->n, m = a->m;
  const size_t x_bytes = B * n * 8, act_bytes = (a->actions_shared ? 1 : B) * H * m * 8;
  const size_t box_bytes = B * (H + 1) * n * 8, i_bytes = B * 4;
  const bool dev = (flags & REACH_FLAG_DEVICE_PTRS) != 0;
  bool small = false;
  size_t o_out = 0, out_end = 0;
  if (dev) {
    P.x0_lo = a->x0_lo;
    P.x0_hi = a->x0_hi;
    P.actions = a->actions;
    P.out_lo = out->lo;
    P.out_hi = out->hi;
    P.n_boxes = out->n_boxes;
    P.failed_step = out->failed_step;
    P.status = out->status;
  } else {
    size_t off = 0;
    auto take = [&](size_t bytes) {
      size_t o = off;
      off = align_up(off + bytes, 256);
      return o;
    };
    size_t o_xl = take(x_bytes), o_xh = take(x_bytes), o_a = take(std::max<size_t>(act_bytes, 8));
    size_t o_ol = take(box_bytes), o_oh = take(box_bytes), o_nb = take(i_bytes), o_fs = take(i_bytes),
           o_st = take(i_bytes);
    rc = ensure_ws(ctx, off);
    if (rc) return rc;
    char* w = static_cast<char*>(ctx->ws);
    P.x0_lo = reinterpret_cast<double*>(w + o_xl);
    P.x0_hi = reinterpret_cast<double*>(w + o_xh);
    P.actions = reinterpret_cast<double*>(w + o_a);
    P.out_lo = reinterpret_cast<double*>(w + o_ol);
    P.out_hi = reinterpret_cast<double*>(w + o_oh);
    P.n_boxes = reinterpret_cast<int*>(w + o_nb);
    P.failed_step = reinterpret_cast<int*>(w + o_fs);
    P.status = reinterpret_cast<int*>(w + o_st);
    // small calls (the batch-1 latency case): every input in ONE copy and every output in ONE copy through
    // the context's pinned staging, laid out as the device workspace
    small = off <= kSmallCallBytes;
    if (small) {
      rc = ensure_pinned(ctx, off);
      if (rc) return rc;
      char* h = static_cast<char*>(ctx->hpin);
      std::memcpy(h + o_xl, a->x0_lo, x_bytes);
      std::memcpy(h + o_xh, a->x0_hi, x_bytes);
      if (act_bytes) std::memcpy(h + o_a, a->actions, act_bytes);
      RB_CUDA(cudaMemcpyAsync(w, h, o_ol, cudaMemcpyHostToDevice, ctx->stream));
      o_out = o_ol;
      out_end = off;
    } else {
      RB_CUDA(cudaMemcpyAsync(const_cast<double*>(P.x0_lo), a->x0_lo, x_bytes, cudaMemcpyHostToDevice, ctx->stream));
      RB_CUDA(cudaMemcpyAsync(const_cast<double*>(P.x0_hi), a->x0_hi, x_bytes, cudaMemcpyHostToDevice, ctx->stream));
      if (act_bytes)
        RB_CUDA(cudaMemcpyAsync(const_cast<double*>(P.actions), a->actions, act_bytes, cudaMemcpyHostToDevice, ctx->stream));
    }
  }
  cudaEvent_t stop;
  rc = timed_begin(ctx, &stop);
  if (rc) return rc;
  RB_CUDA(launch_dt(P, lay, a->batch, ctx->stream));
  rc = timed_end(ctx, stop);
  if (rc) return rc;
  ctx->launches += 1;
  if (!dev && small) {
    // one read-back of the whole output region; boxes beyond n_boxes stay untouched in the caller's buffer
    const char* h = static_cast<const char*>(ctx->hpin);
    RB_CUDA(cudaMemcpyAsync(static_cast<char*>(ctx->hpin) + o_out, static_cast<const char*>(ctx->ws) + o_out,
                            out_end - o_out, cudaMemcpyDeviceToHost, ctx->stream));
    RB_CUDA(cudaStreamSynchronize(ctx->stream));
    const char* base = static_cast<const char*>(ctx->ws);
    auto host = [&](const void* dptr) { return h + (static_cast<const char*>(dptr) - base); };
    std::memcpy(out->n_boxes, host(P.n_boxes), i_bytes);
    std::memcpy(out->failed_step, host(P.failed_step), i_bytes);
    std::memcpy(out->status, host(P.status), i_bytes);
    const double* hl = reinterpret_cast<const double*>(host(P.out_lo));
    const double* hh = reinterpret_cast<const double*>(host(P.out_hi));
    for (size_t i = 0; i < B; ++i) {
      const size_t o = i * (H + 1) * n, cnt = static_cast<size_t>(out->n_boxes[i]) * n * 8;
      if (!cnt) continue;
      std::memcpy(out->lo + o, hl + o, cnt);
      std::memcpy(out->hi + o, hh + o, cnt);
    }
  } else if (!dev) {
    // boxes beyond n_boxes are untouched in the caller's buffer: copy only the
    // tube prefix per sample after reading n_boxes
    std::vector<int32_t> nb(B);
    RB_CUDA(cudaMemcpyAsync(nb.data(), P.n_boxes, i_bytes, cudaMemcpyDeviceToHost, ctx->stream));
    RB_CUDA(cudaMemcpyAsync(out->failed_step, P.failed_step, i_bytes, cudaMemcpyDeviceToHost, ctx->stream));
    RB_CUDA(cudaMemcpyAsync(out->status, P.status, i_bytes, cudaMemcpyDeviceToHost, ctx->stream));
    RB_CUDA(cudaStreamSynchronize(ctx->stream));
    std::memcpy(out->n_boxes, nb.data(), i_bytes);
    bool all_full = true;
    for (size_t i = 0; i < B; ++i) all_full &= (nb[i] == static_cast<int32_t>(H + 1));
    if (all_full) {
      RB_CUDA(cudaMemcpyAsync(out->lo, P.out_lo, box_bytes, cudaMemcpyDeviceToHost, ctx->stream));
      RB_CUDA(cudaMemcpyAsync(out->hi, P.out_hi, box_bytes, cudaMemcpyDeviceToHost, ctx->stream));
    } else {
      for (size_t i = 0; i < B; ++i) {
        const size_t o = i * (H + 1) * n, cnt = static_cast<size_t>(nb[i]) * n * 8;
        if (!cnt) continue;
        RB_CUDA(cudaMemcpyAsync(out->lo + o, P.out_lo + o, cnt, cudaMemcpyDeviceToHost, ctx->stream));
        RB_CUDA(cudaMemcpyAsync(out->hi + o, P.out_hi + o, cnt, cudaMemcpyDeviceToHost, ctx->stream));
      }
    }
    RB_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  return REACH_OK;
}

}  // namespace

extern "C" {

int reach_dt_batch(reach_ctx* ctx, const reach_net* net, const reach_dt_args* a, const reach_tube_out* out,
                   int32_t flags) {
  rbh::DeviceGuard device_guard_(ctx);
  if (!ctx || !net || !a || !out) return REACH_E_INVALID_ARGUMENT;
  if (flags & REACH_FLAG_OUTWARD_ROUNDING)
    return fail(ctx, REACH_E_UNSUPPORTED, "outward rounding (g_outward_rounding) is not supported by the device kernels");
  if (a->batch < 0 || a->horizon < 0) return fail(ctx, REACH_E_INVALID_ARGUMENT, "dt_reach_batch: negative size");
  int rc = validate_system(ctx, net, a->n, a->m);
  if (rc) return rc;
  return run_dt_batch(ctx, net, nullptr, a, out, flags);
}

int reach_dtcl_batch(reach_ctx* ctx, const reach_net* dyn, const reach_net* ctl, const reach_dt_args* a,
                     const reach_tube_out* out, int32_t flags) {
  rbh::DeviceGuard device_guard_(ctx);
  if (!ctx || !dyn || !ctl || !a || !out) return REACH_E_INVALID_ARGUMENT;
  if (flags & REACH_FLAG_OUTWARD_ROUNDING)
    return fail(ctx, REACH_E_UNSUPPORTED, "outward rounding (g_outward_rounding) is not supported by the device kernels");
  if (a->batch < 0 || a->horizon < 0) return fail(ctx, REACH_E_INVALID_ARGUMENT, "dt closed loop: negative size");
  if (a->m != 0) return fail(ctx, REACH_E_INVALID_ARGUMENT, "dt closed loop: actions come from the controller (m = 0)");
  const int l = ctl->dims[ctl->L];
  if (a->n <= 0 || ctl->dims[0] != a->n)
    return fail(ctx, REACH_E_INVALID_ARGUMENT, "ClosedLoopSpec: controller input dim mismatch");
  if (dyn->dims[0] != a->n + l || dyn->dims[dyn->L] != a->n)
    return fail(ctx, REACH_E_INVALID_ARGUMENT, "ClosedLoopSpec: dynamics must act on the augmented (x,u) state");
  return run_dt_batch(ctx, dyn, ctl, a, out, flags);
}

}  // extern "C"

namespace {
__global__ void hull_init_kernel(unsigned long long* klo, unsigned long long* khi, int* nan0, int* div, int count,
                                 int hp1, int* nboxes, unsigned long long* key) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < count) {
    klo[t] = ~0ull;
    khi[t] = 0ull;
    nan0[2 * t] = 0;
    nan0[2 * t + 1] = 0;
  }
  if (t < hp1) div[t] = 0;
  if (t == 0) {
    *nboxes = INT_MAX;
    *key = static_cast<unsigned long long>(INT64_MAX);
  }
}
}  // namespace

extern "C" {

int reach_split_hull(reach_ctx* ctx, const reach_net* net, const reach_split_args* a, const reach_hull_out* out,
                     int32_t flags) {
  rbh::DeviceGuard device_guard_(ctx);
  if (!ctx || !net || !a || !out) return REACH_E_INVALID_ARGUMENT;
  if (flags & REACH_FLAG_OUTWARD_ROUNDING)
    return fail(ctx, REACH_E_UNSUPPORTED, "outward rounding (g_outward_rounding) is not supported by the device kernels");
  int rc = validate_system(ctx, net, a->n, a->m);
  if (rc) return rc;
  if (a->horizon < 0) return fail(ctx, REACH_E_INVALID_ARGUMENT, "reach_with_splitting: negative horizon");
  if (a->n > rb::kMaxSplitDims) return fail(ctx, REACH_E_UNSUPPORTED, "too many split dimensions");
  long long total = 1;
  for (int d = 0; d < a->n; ++d) {
    if (a->counts[d] < 1) return fail(ctx, REACH_E_INVALID_ARGUMENT, "SplitPlan: counts must be >= 1");
    total *= a->counts[d];
    if (total > (1ll << 20)) return fail(ctx, REACH_E_INVALID_ARGUMENT, "SplitPlan: total part count overflow");
  }
  const long long begin0 = a->part_begin, end0 = a->part_end <= 0 ? total : a->part_end;
  if (begin0 < 0 || begin0 >= end0 || end0 > total) return fail(ctx, REACH_E_INVALID_ARGUMENT, "bad part range");
  // multi-GPU: this rank's contiguous slice of the parts; the hull is all-reduced below
  long long begin, end;
  rbh::coll_shard(ctx, begin0, end0, begin, end);
  RB_CUDA(cudaSetDevice(ctx->device));
  rb::DTParams P{};
  DTLayout lay;
  rc = plan_dt(ctx, net, a->n, a->m, a->window, std::max(end - begin, 1ll), P, lay, nullptr,
               flags & REACH_FLAG_PREC_MASK);
  if (rc) return rc;
  const bool dev = (flags & REACH_FLAG_DEVICE_PTRS) != 0;
  const int n = a->n, H = a->horizon, m = a->m;
  P.net = net->dev;
  P.B = static_cast<int>(end - begin);
  P.H = H;
  P.n = n;
  P.m = m;
  P.window = a->window;
  P.rebuild = a->rebuild_from_box;
  P.split = 1;
  P.part_begin = begin;
  P.actions_shared = 1;
  const size_t cnt = static_cast<size_t>(H + 1) * n;
  // the X0 box and the plan are host-side plan parameters; they travel in the
  // kernel's parameter block (no device round trip)
  for (int d = 0; d < n; ++d) {
    P.sx_lo[d] = a->x0_lo[d];
    P.sx_hi[d] = a->x0_hi[d];
    P.counts[d] = a->counts[d];
  }
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align_up(off + bytes, 256);
    return o;
  };
  const size_t o_kl = take(cnt * 8), o_kh = take(cnt * 8), o_nan = take(cnt * 8), o_div = take((H + 1) * 4),
               o_nb = take(4), o_key = take(8), o_act = take(std::max<size_t>(static_cast<size_t>(H) * m * 8, 8)),
               o_lo = take(cnt * 8), o_hi = take(cnt * 8);
  rc = ensure_ws(ctx, off);
  if (rc) return rc;
  char* w = static_cast<char*>(ctx->ws);
  P.hull_lo = reinterpret_cast<unsigned long long*>(w + o_kl);
  P.hull_hi = reinterpret_cast<unsigned long long*>(w + o_kh);
  P.hull_nan0 = reinterpret_cast<int*>(w + o_nan);
  P.hull_div = reinterpret_cast<int*>(w + o_div);
  P.hull_nboxes = reinterpret_cast<int*>(w + o_nb);
  P.hull_fail_key = reinterpret_cast<unsigned long long*>(w + o_key);
  if (dev) {
    P.actions = a->actions;
  } else {
    P.actions = reinterpret_cast<double*>(w + o_act);
    if (H * m)
      RB_CUDA(cudaMemcpyAsync(const_cast<double*>(P.actions), a->actions, static_cast<size_t>(H) * m * 8,
                              cudaMemcpyHostToDevice, ctx->stream));
  }
  const int icount = static_cast<int>(cnt);
  const int tpb = 256;
  const int blocks = std::max((std::max(icount, H + 1) + tpb - 1) / tpb, 1);
  hull_init_kernel<<<blocks, tpb, 0, ctx->stream>>>(P.hull_lo, P.hull_hi, P.hull_nan0, P.hull_div, icount, H + 1,
                                                     P.hull_nboxes, P.hull_fail_key);
  RB_CUDA(cudaGetLastError());
  if (P.B > 0) {
    cudaEvent_t stop;
    rc = timed_begin(ctx, &stop);
    if (rc) return rc;
    RB_CUDA(launch_dt(P, lay, P.B, ctx->stream));
    rc = timed_end(ctx, stop);
    if (rc) return rc;
  }
  rc = rbh::coll_hull(ctx, P.hull_lo, P.hull_hi, P.hull_nan0, 2 * icount, P.hull_div, H + 1, P.hull_nboxes,
                      P.hull_fail_key);
  if (rc) return rc;
  double* dlo = dev ? out->lo : reinterpret_cast<double*>(w + o_lo);
  double* dhi = dev ? out->hi : reinterpret_cast<double*>(w + o_hi);
  rb::hull_finalize_kernel<<<(icount + tpb - 1) / tpb, tpb, 0, ctx->stream>>>(P.hull_lo, P.hull_hi, P.hull_nan0,
                                                                              icount, dlo, dhi);
  RB_CUDA(cudaGetLastError());
  ctx->launches += 3;
  if (dev) {
    RB_CUDA(cudaMemcpyAsync(out->box_diverged, P.hull_div, (H + 1) * 4, cudaMemcpyDeviceToDevice, ctx->stream));
    RB_CUDA(cudaMemcpyAsync(out->n_boxes, P.hull_nboxes, 4, cudaMemcpyDeviceToDevice, ctx->stream));
    RB_CUDA(cudaMemcpyAsync(out->fail_key, P.hull_fail_key, 8, cudaMemcpyDeviceToDevice, ctx->stream));
  } else {
    RB_CUDA(cudaMemcpyAsync(out->lo, dlo, cnt * 8, cudaMemcpyDeviceToHost, ctx->stream));
    RB_CUDA(cudaMemcpyAsync(out->hi, dhi, cnt * 8, cudaMemcpyDeviceToHost, ctx->stream));
    RB_CUDA(cudaMemcpyAsync(out->box_diverged, P.hull_div, (H + 1) * 4, cudaMemcpyDeviceToHost, ctx->stream));
    RB_CUDA(cudaMemcpyAsync(out->n_boxes, P.hull_nboxes, 4, cudaMemcpyDeviceToHost, ctx->stream));
    RB_CUDA(cudaMemcpyAsync(out->fail_key, P.hull_fail_key, 8, cudaMemcpyDeviceToHost, ctx->stream));
    RB_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  return REACH_OK;
}


}  // extern "C"

// ---------------------------------------------------------------------------
// Reachability-aware MPC (mpc.hpp).
namespace {

// PlanProblem::validate + Constraint::validate (mpc.hpp:88-142).
int validate_problem(reach_ctx* ctx, const reach_net* net, const reach_plan_problem* p) {
  int rc = validate_system(ctx, net, p->n, p->m);
  if (rc) return rc;
  if (p->horizon < 1) return fail(ctx, REACH_E_INVALID_ARGUMENT, "PlanProblem: horizon < 1");
  if (!p->x_goal || !p->q_weights || (p->m > 0 && !p->r_weights))
    return fail(ctx, REACH_E_INVALID_ARGUMENT, "PlanProblem: cost dimension mismatch");
  if (p->m > 0 && (!p->u_lo || !p->u_hi))
    return fail(ctx, REACH_E_INVALID_ARGUMENT, "PlanProblem: action box dimension mismatch");
  for (int j = 0; j < p->m; ++j)
    if (!(p->u_lo[j] <= p->u_hi[j]) || !std::isfinite(p->u_lo[j]) || !std::isfinite(p->u_hi[j]))
      return fail(ctx, REACH_E_INVALID_ARGUMENT, "PlanProblem: action box must be bounded");
  if (p->eps < 0.0 || p->penalty < 0.0) return fail(ctx, REACH_E_INVALID_ARGUMENT, "PlanProblem: negative weight");
  if (p->n_constraints < 0 || p->n_constraints > rb::kMaxConstraints)
    return fail(ctx, REACH_E_UNSUPPORTED, "too many constraints");
  for (int c = 0; c < p->n_constraints; ++c) {
    const reach_constraint& k = p->constraints[c];
    for (int j = 0; j < k.n_dims; ++j)
      if (k.dims[j] < 0 || k.dims[j] >= p->n) return fail(ctx, REACH_E_INVALID_ARGUMENT, "Constraint: dim out of range");
    switch (k.type) {
      case REACH_CON_HALFSPACE_AVOID:
        if (!k.a) return fail(ctx, REACH_E_INVALID_ARGUMENT, "Constraint: halfspace size");
        break;
      case REACH_CON_SPHERE_AVOID:
        if (!k.center || k.radius < 0.0) return fail(ctx, REACH_E_INVALID_ARGUMENT, "Constraint: sphere parameters");
        break;
      case REACH_CON_BOX_STAY_IN:
        if (!k.lo || !k.hi) return fail(ctx, REACH_E_INVALID_ARGUMENT, "Constraint: stay-in box size");
        break;
      case REACH_CON_MAX_VOLUME:
        if (k.vmax < 0.0) return fail(ctx, REACH_E_INVALID_ARGUMENT, "Constraint: volume budget");
        break;
      default:
        return fail(ctx, REACH_E_INVALID_ARGUMENT, "Constraint: unknown type");
    }
  }
  return REACH_OK;
}

// Device-side copy of the problem's small arrays (goal, weights, constraints).
struct PlanBuffers {
  std::vector<int> ib;
  std::vector<double> db;
  rb::PlanParams P{};
};

void pack_problem(const reach_plan_problem* p, PlanBuffers& pb) {
  auto put = [&](const double* v, int k) {
    const int o = static_cast<int>(pb.db.size());
    for (int j = 0; j < k; ++j) pb.db.push_back(v ? v[j] : 0.0);
    return o;
  };
  const int og = put(p->x_goal, p->n), oq = put(p->q_weights, p->n), orr = put(p->r_weights, p->m);
  pb.P.n_con = p->n_constraints;
  for (int c = 0; c < p->n_constraints; ++c) {
    const reach_constraint& k = p->constraints[c];
    rb::DevConstraint& d = pb.P.con[c];
    d.type = k.type;
    d.k = k.n_dims > 0 ? k.n_dims : p->n;
    d.dims_off = static_cast<int>(pb.ib.size());
    for (int j = 0; j < d.k; ++j) pb.ib.push_back(k.n_dims > 0 ? k.dims[j] : j);
    d.a_off = put(k.a, k.type == REACH_CON_HALFSPACE_AVOID ? d.k : 0);
    d.c_off = put(k.center, k.type == REACH_CON_SPHERE_AVOID ? d.k : 0);
    d.lo_off = put(k.lo, k.type == REACH_CON_BOX_STAY_IN ? d.k : 0);
    d.hi_off = put(k.hi, k.type == REACH_CON_BOX_STAY_IN ? d.k : 0);
    d.b = k.b;
    d.radius = k.radius;
    d.vmax = k.vmax;
  }
  if (pb.ib.empty()) pb.ib.push_back(0);
  pb.P.penalty = p->penalty;
  pb.P.diverged_margin = p->diverged_margin;
  pb.P.x_goal = reinterpret_cast<const double*>(static_cast<intptr_t>(og));  // offsets, rebased after upload
  pb.P.q_w = reinterpret_cast<const double*>(static_cast<intptr_t>(oq));
  pb.P.r_w = reinterpret_cast<const double*>(static_cast<intptr_t>(orr));
}

// plan_eval for `batch` candidates with everything already on the device.
int plan_eval_device(reach_ctx* ctx, const reach_net* net, const reach_plan_problem* p, const double* d_x0, int batch,
                     const double* d_actions, double* d_obj, int* d_div, double* d_tlo, double* d_thi, int* d_nb,
                     int* d_fs, int* d_st) {
  rb::DTParams P{};
  DTLayout lay;
  int rc = plan_dt(ctx, net, p->n, p->m, p->window, batch, P, lay);
  if (rc) return rc;
  P.net = net->dev;
  P.B = batch;
  P.H = p->horizon;
  P.n = p->n;
  P.m = p->m;
  P.window = p->window;
  P.rebuild = p->rebuild_from_box;
  P.x0_lo = d_x0;
  P.x0_hi = d_x0;
  P.x0_center = 1;
  P.x0_eps = p->eps;
  P.actions = d_actions;
  P.out_lo = d_tlo;
  P.out_hi = d_thi;
  P.n_boxes = d_nb;
  P.failed_step = d_fs;
  P.status = d_st;
  // objective kernel: problem arrays staged after the tube in the plan workspace
  PlanBuffers pb;
  pack_problem(p, pb);
  const size_t need = align_up(pb.db.size() * 8 + 8, 256) + pb.ib.size() * 4;
  if (need > ctx->pbuf_bytes) {
    RB_CUDA(cudaStreamSynchronize(ctx->stream));
    if (ctx->pbuf) cudaFree(ctx->pbuf);
    ctx->pbuf = nullptr;
    RB_CUDA(cudaMalloc(&ctx->pbuf, need));
    ctx->pbuf_bytes = need;
  }
  double* d_db = static_cast<double*>(ctx->pbuf);
  int* d_ib = reinterpret_cast<int*>(static_cast<char*>(ctx->pbuf) + align_up(pb.db.size() * 8 + 8, 256));
  RB_CUDA(cudaMemcpyAsync(d_db, pb.db.data(), pb.db.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
  RB_CUDA(cudaMemcpyAsync(d_ib, pb.ib.data(), pb.ib.size() * 4, cudaMemcpyHostToDevice, ctx->stream));
  rb::PlanParams Q = pb.P;
  Q.net = net->dev;
  Q.B = batch;
  Q.H = p->horizon;
  Q.n = p->n;
  Q.m = p->m;
  Q.x0 = d_x0;
  Q.actions = d_actions;
  Q.x_goal = d_db + reinterpret_cast<intptr_t>(pb.P.x_goal);
  Q.q_w = d_db + reinterpret_cast<intptr_t>(pb.P.q_w);
  Q.r_w = d_db + reinterpret_cast<intptr_t>(pb.P.r_w);
  Q.ibuf = d_ib;
  Q.dbuf = d_db;
  Q.tube_lo = d_tlo;
  Q.tube_hi = d_thi;
  Q.n_boxes = d_nb;
  Q.status = d_st;
  Q.objective = d_obj;
  Q.diverged = d_div;
  int vec = 0;
  for (int l = 0; l <= net->L; ++l) vec = std::max(vec, net->dims[l]);
  vec = (vec + 1) & ~1;
  int wmax = 0;
  for (int l = 0; l < net->L; ++l) wmax = std::max(wmax, net->dims[l] * net->dims[l + 1]);
  wmax = (wmax + 1) & ~1;
  // every layer resident in shared memory when it fits with >= 8 candidate warps (one persistent CTA per
  // SM): the nominal rollouts + stage costs do not read the tube, so they run on a second stream
  // concurrently with the tube kernel (filling the SMs its last wave leaves idle); the penalty pass joins
  // after both (plan_objective = rollout terms, then the constraint terms, in the reference's order).
  {
    int wtot = 0;
    int maxrows = 0;
    for (int l = 0; l < net->L; ++l) {
      wtot += net->dims[l] * net->dims[l + 1];
      maxrows = std::max(maxrows, net->dims[l + 1]);
    }
    wtot = (wtot + 1) & ~1;
    const long long room = static_cast<long long>(ctx->max_smem) - static_cast<long long>(wtot) * 8;
    const int warps = room > 0 ? static_cast<int>(std::min<long long>(rb::kPlanMaxWarps, room / (2ll * vec * 8))) : 0;
    if (warps >= 8 && maxrows <= 4096) {
      if (!ctx->aux) {
        RB_CUDA(cudaStreamCreateWithFlags(&ctx->aux, cudaStreamNonBlocking));
        RB_CUDA(cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming));
        RB_CUDA(cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming));
      }
      const size_t rsmem = (static_cast<size_t>(wtot) + static_cast<size_t>(warps) * 2 * vec) * 8;
      RB_CUDA(cudaFuncSetAttribute(rb::plan_rollout_resident_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(rsmem)));
      const int grid = static_cast<int>(std::min<long long>((batch + warps - 1) / warps, ctx->num_sms));
      RB_CUDA(cudaEventRecord(ctx->ev_fork, ctx->stream));
      RB_CUDA(cudaStreamWaitEvent(ctx->aux, ctx->ev_fork, 0));
      rb::plan_rollout_resident_kernel<<<grid, 32 * warps, rsmem, ctx->aux>>>(Q, vec, wtot);
      RB_CUDA(cudaGetLastError());
      RB_CUDA(cudaEventRecord(ctx->ev_join, ctx->aux));
  cudaEvent_t stop;
    rc = timed_begin(ctx, &stop);
    if (rc) return rc;
    RB_CUDA(launch_dt(P, lay, batch, ctx->stream));
    rc = timed_end(ctx, stop);
    if (rc) return rc;
      RB_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ev_join, 0));
      rb::plan_penalty_kernel<<<(batch + 255) / 256, 256, 0, ctx->stream>>>(Q);
      RB_CUDA(cudaGetLastError());
      ctx->launches += 3;
      return REACH_OK;
    }
  }
  cudaEvent_t stop;
  rc = timed_begin(ctx, &stop);
  if (rc) return rc;
  RB_CUDA(launch_dt(P, lay, batch, ctx->stream));
  rc = timed_end(ctx, stop);
  if (rc) return rc;
  const size_t smem = (static_cast<size_t>(wmax) + static_cast<size_t>(rb::kPlanWarps) * 2 * vec) * 8;
  if (smem > static_cast<size_t>(ctx->max_smem))
    return fail(ctx, REACH_E_UNSUPPORTED, "plan_eval: layer too large for the staged rollout");
  RB_CUDA(cudaFuncSetAttribute(rb::plan_objective_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(smem)));
  rb::plan_objective_kernel<<<(batch + rb::kPlanWarps - 1) / rb::kPlanWarps, 32 * rb::kPlanWarps, smem,
                              ctx->stream>>>(Q, vec, wmax);
  RB_CUDA(cudaGetLastError());
  ctx->launches += 2;
  return REACH_OK;
}

// Host-pointer plan_eval: stages inputs / outputs through the ctx workspace.
int plan_eval_host(reach_ctx* ctx, const reach_net* net, const reach_plan_problem* p, const double* x0, int batch,
                   const double* actions, double* objective, int32_t* diverged, const reach_tube_out* tubes) {
  const size_t B = batch, H = p->horizon, n = p->n, m = p->m;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align_up(off + std::max<size_t>(bytes, 8), 256);
    return o;
  };
  const size_t box = B * (H + 1) * n * 8;
  const size_t o_x0 = take(n * 8), o_a = take(B * H * m * 8), o_obj = take(B * 8), o_div = take(B * 4),
               o_lo = take(box), o_hi = take(box), o_nb = take(B * 4), o_fs = take(B * 4), o_st = take(B * 4);
  int rc = ensure_ws(ctx, off);
  if (rc) return rc;
  char* w = static_cast<char*>(ctx->ws);
  auto D = [&](size_t o) { return reinterpret_cast<double*>(w + o); };
  auto I = [&](size_t o) { return reinterpret_cast<int*>(w + o); };
  RB_CUDA(cudaMemcpyAsync(D(o_x0), x0, n * 8, cudaMemcpyHostToDevice, ctx->stream));
  if (m) RB_CUDA(cudaMemcpyAsync(D(o_a), actions, B * H * m * 8, cudaMemcpyHostToDevice, ctx->stream));
  rc = plan_eval_device(ctx, net, p, D(o_x0), batch, D(o_a), D(o_obj), I(o_div), D(o_lo), D(o_hi), I(o_nb), I(o_fs),
                        I(o_st));
  if (rc) return rc;
  RB_CUDA(cudaMemcpyAsync(objective, D(o_obj), B * 8, cudaMemcpyDeviceToHost, ctx->stream));
  RB_CUDA(cudaMemcpyAsync(diverged, I(o_div), B * 4, cudaMemcpyDeviceToHost, ctx->stream));
  if (tubes) {
    RB_CUDA(cudaMemcpyAsync(tubes->lo, D(o_lo), box, cudaMemcpyDeviceToHost, ctx->stream));
    RB_CUDA(cudaMemcpyAsync(tubes->hi, D(o_hi), box, cudaMemcpyDeviceToHost, ctx->stream));
    RB_CUDA(cudaMemcpyAsync(tubes->n_boxes, I(o_nb), B * 4, cudaMemcpyDeviceToHost, ctx->stream));
    RB_CUDA(cudaMemcpyAsync(tubes->failed_step, I(o_fs), B * 4, cudaMemcpyDeviceToHost, ctx->stream));
    RB_CUDA(cudaMemcpyAsync(tubes->status, I(o_st), B * 4, cudaMemcpyDeviceToHost, ctx->stream));
  }
  RB_CUDA(cudaStreamSynchronize(ctx->stream));
  return REACH_OK;
}

// plan_eval of a CEM population with multi-GPU collectives: this rank evaluates its contiguous slice,
// one all-gather per output array (padded to ceil(pop / world) per rank) assembles every rank's
// scores in candidate order, so all ranks run the identical sort / refit (mpc.hpp:300-333).
int plan_eval_sharded(reach_ctx* ctx, const reach_net* net, const reach_plan_problem* p, const double* x0, int pop,
                      const double* actions, double* objective, int32_t* diverged) {
  if (!ctx->has_coll || ctx->coll.world <= 1)
    return plan_eval_host(ctx, net, p, x0, pop, actions, objective, diverged, nullptr);
  const int world = ctx->coll.world;
  long long b, e;
  rbh::coll_shard(ctx, 0, pop, b, e);
  const size_t width = (static_cast<size_t>(pop) + world - 1) / world, B = static_cast<size_t>(e - b);
  const size_t H = p->horizon, n = p->n, m = p->m, box = std::max<size_t>(B, 1) * (H + 1) * n * 8;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align_up(off + std::max<size_t>(bytes, 8), 256);
    return o;
  };
  const size_t o_x0 = take(n * 8), o_a = take(B * H * m * 8), o_obj = take(width * 8), o_div = take(width * 4),
               o_go = take(world * width * 8), o_gd = take(world * width * 4), o_lo = take(box), o_hi = take(box),
               o_nb = take(B * 4), o_fs = take(B * 4), o_st = take(B * 4);
  int rc = ensure_ws(ctx, off);
  if (rc) return rc;
  char* w = static_cast<char*>(ctx->ws);
  auto D = [&](size_t o) { return reinterpret_cast<double*>(w + o); };
  auto I = [&](size_t o) { return reinterpret_cast<int*>(w + o); };
  RB_CUDA(cudaMemsetAsync(w + o_obj, 0, width * 8, ctx->stream));
  RB_CUDA(cudaMemsetAsync(w + o_div, 0, width * 4, ctx->stream));
  if (B > 0) {
    RB_CUDA(cudaMemcpyAsync(D(o_x0), x0, n * 8, cudaMemcpyHostToDevice, ctx->stream));
    if (m) RB_CUDA(cudaMemcpyAsync(D(o_a), actions + b * H * m, B * H * m * 8, cudaMemcpyHostToDevice, ctx->stream));
    rc = plan_eval_device(ctx, net, p, D(o_x0), static_cast<int>(B), D(o_a), D(o_obj), I(o_div), D(o_lo), D(o_hi),
                          I(o_nb), I(o_fs), I(o_st));
    if (rc) return rc;
  }
  rc = rbh::coll_allgather(ctx, D(o_obj), D(o_go), width, REACH_DT_F64);
  if (!rc) rc = rbh::coll_allgather(ctx, I(o_div), I(o_gd), width, REACH_DT_I32);
  if (rc) return rc;
  std::vector<double> go(world * width);
  std::vector<int32_t> gd(world * width);
  RB_CUDA(cudaMemcpyAsync(go.data(), D(o_go), go.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
  RB_CUDA(cudaMemcpyAsync(gd.data(), I(o_gd), gd.size() * 4, cudaMemcpyDeviceToHost, ctx->stream));
  RB_CUDA(cudaStreamSynchronize(ctx->stream));
  for (int r = 0; r < world; ++r) {
    const long long total = pop, base = total / world, rem = total % world;
    const long long rb0 = r * base + std::min<long long>(r, rem), cnt = base + (r < rem ? 1 : 0);
    for (long long k = 0; k < cnt; ++k) {
      objective[rb0 + k] = go[r * width + k];
      diverged[rb0 + k] = gd[r * width + k];
    }
  }
  return REACH_OK;
}

// grad_forward (refine.hpp:186-207) of plan_objective over the flat action
// sequence: one Dual pass per direction, all directions in one launch
// (dual_kernel.cuh).  `value` receives the primal objective (equal in every
// pass); returns REACH_OK, or REACH_E_CUDA family errors; non-finite
// derivatives are reported through `finite`.
int plan_grad_device(reach_ctx* ctx, const reach_net* net, const reach_plan_problem* p, const double* x0,
                     const double* actions, double* grad, double* value, bool* finite) {
  namespace rd = rb::dual;
  const int H = p->horizon, n = p->n, m = p->m, dim = H * m;
  int maxw = 0;
  for (int l = 0; l <= net->L; ++l) maxw = std::max(maxw, net->dims[l]);
  const int cap = p->window > 0 ? p->window : 1;
  if (n > rd::kN || m > rd::kM || maxw > rd::kW || net->L > rd::kL || H > rd::kH || n * (cap + 2) > rd::kZ ||
      n * (cap + 2) + n > rd::kW || cap + 2 > rd::kQ)
    return fail(ctx, REACH_E_UNSUPPORTED, "plan gradient: shape outside the Dual kernel family");
  PlanBuffers pb;
  pack_problem(p, pb);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align_up(off + std::max<size_t>(bytes, 8), 256);
    return o;
  };
  const size_t o_db = take(pb.db.size() * 8), o_ib = take(pb.ib.size() * 4), o_x0 = take(n * 8),
               o_a = take(static_cast<size_t>(dim) * 8), o_g = take(static_cast<size_t>(dim) * 8),
               o_v = take(static_cast<size_t>(dim) * 8);
  int rc = ensure_ws(ctx, off);
  if (rc) return rc;
  char* w = static_cast<char*>(ctx->ws);
  auto Dp = [&](size_t o) { return reinterpret_cast<double*>(w + o); };
  RB_CUDA(cudaMemcpyAsync(Dp(o_db), pb.db.data(), pb.db.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
  RB_CUDA(cudaMemcpyAsync(w + o_ib, pb.ib.data(), pb.ib.size() * 4, cudaMemcpyHostToDevice, ctx->stream));
  RB_CUDA(cudaMemcpyAsync(Dp(o_x0), x0, n * 8, cudaMemcpyHostToDevice, ctx->stream));
  RB_CUDA(cudaMemcpyAsync(Dp(o_a), actions, static_cast<size_t>(dim) * 8, cudaMemcpyHostToDevice, ctx->stream));
  rd::GradArgs G{};
  G.P = pb.P;
  G.P.net = net->dev;
  G.P.H = H;
  G.P.n = n;
  G.P.m = m;
  G.P.x0 = Dp(o_x0);
  G.P.dbuf = Dp(o_db);
  G.P.ibuf = reinterpret_cast<const int*>(w + o_ib);
  G.P.x_goal = Dp(o_db) + reinterpret_cast<intptr_t>(pb.P.x_goal);
  G.P.q_w = Dp(o_db) + reinterpret_cast<intptr_t>(pb.P.q_w);
  G.P.r_w = Dp(o_db) + reinterpret_cast<intptr_t>(pb.P.r_w);
  G.window = p->window;
  G.rebuild = p->rebuild_from_box;
  G.eps = p->eps;
  G.base = Dp(o_a);
  G.grad = Dp(o_g);
  G.value = Dp(o_v);
  cudaEvent_t stop;
  rc = timed_begin(ctx, &stop);
  if (rc) return rc;
  RB_CUDA(cudaFuncSetAttribute(rd::plan_grad_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(sizeof(rd::Work))));
  rd::plan_grad_kernel<<<dim, rd::kThreads, sizeof(rd::Work), ctx->stream>>>(G);
  RB_CUDA(cudaGetLastError());
  rc = timed_end(ctx, stop);
  if (rc) return rc;
  ctx->launches += 1;
  std::vector<double> vals(dim);
  RB_CUDA(cudaMemcpyAsync(grad, Dp(o_g), static_cast<size_t>(dim) * 8, cudaMemcpyDeviceToHost, ctx->stream));
  RB_CUDA(cudaMemcpyAsync(vals.data(), Dp(o_v), static_cast<size_t>(dim) * 8, cudaMemcpyDeviceToHost, ctx->stream));
  RB_CUDA(cudaStreamSynchronize(ctx->stream));
  *value = vals[0];
  *finite = true;
  for (int j = 0; j < dim; ++j)
    if (!std::isfinite(vals[j]) || !std::isfinite(grad[j])) *finite = false;
  return REACH_OK;
}

}  // namespace

// CEM state (plan_cem, mpc.hpp:258-335): the reference's Rng (rng.hpp:13-52)
// -- std::mt19937_64, 53-bit uniforms, cached Box-Muller -- drawn sequentially.
struct reach_cem {
  int h = 0, m = 0;
  std::vector<double> u_lo, u_hi;
  reach_sampler_config cfg{};
  std::mt19937_64 gen;
  bool has_spare = false;
  double spare = 0.0;
  std::vector<double> mean, stdv, best;
  double best_obj = std::numeric_limits<double>::infinity();
  bool any_finite = false;
  int n_elite = 1, it = 0;
  std::vector<std::vector<double>> cands;
  std::vector<double> history;

  double uniform01() { return static_cast<double>(gen() >> 11) * 0x1.0p-53; }
  double normal() {
    if (has_spare) {
      has_spare = false;
      return spare;
    }
    double u1 = uniform01(), u2 = uniform01();
    while (u1 <= 0.0) u1 = uniform01();
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double a = 6.28318530717958647692 * u2;
    spare = r * std::sin(a);
    has_spare = true;
    return r * std::cos(a);
  }
  void clip(std::vector<double>& flat) const {
    for (size_t k = 0; k < flat.size(); ++k) {
      const size_t j = k % static_cast<size_t>(m);
      flat[k] = std::clamp(flat[k], u_lo[j], u_hi[j]);
    }
  }
};

extern "C" {

int reach_plan_eval_batch(reach_ctx* ctx, const reach_net* net, const reach_plan_problem* prob, const double* x0,
                          int32_t batch, const double* actions, double* objective, int32_t* diverged,
                          const reach_tube_out* tubes, int32_t flags) {
  rbh::DeviceGuard device_guard_(ctx);
  if (!ctx || !net || !prob || !x0 || !objective || !diverged || batch < 0) return REACH_E_INVALID_ARGUMENT;
  if (flags & REACH_FLAG_OUTWARD_ROUNDING)
    return fail(ctx, REACH_E_UNSUPPORTED, "outward rounding (g_outward_rounding) is not supported by the device kernels");
  int rc = validate_problem(ctx, net, prob);
  if (rc) return rc;
  if (batch == 0) return REACH_OK;
  RB_CUDA(cudaSetDevice(ctx->device));
  if (flags & REACH_FLAG_DEVICE_PTRS) {
    const size_t B = batch, H = prob->horizon, n = prob->n;
    double *tlo = tubes ? tubes->lo : nullptr, *thi = tubes ? tubes->hi : nullptr;
    int *nb = tubes ? tubes->n_boxes : nullptr, *fs = tubes ? tubes->failed_step : nullptr,
        *st = tubes ? tubes->status : nullptr;
    if (!tubes) {  // scratch tube in the workspace
      size_t off = 0;
      auto take = [&](size_t bytes) {
        size_t o = off;
        off = align_up(off + bytes, 256);
        return o;
      };
      const size_t box = B * (H + 1) * n * 8;
      const size_t o_lo = take(box), o_hi = take(box), o_nb = take(B * 4), o_fs = take(B * 4), o_st = take(B * 4);
      rc = ensure_ws(ctx, off);
      if (rc) return rc;
      char* w = static_cast<char*>(ctx->ws);
      tlo = reinterpret_cast<double*>(w + o_lo);
      thi = reinterpret_cast<double*>(w + o_hi);
      nb = reinterpret_cast<int*>(w + o_nb);
      fs = reinterpret_cast<int*>(w + o_fs);
      st = reinterpret_cast<int*>(w + o_st);
    }
    return plan_eval_device(ctx, net, prob, x0, batch, actions, objective, diverged, tlo, thi, nb, fs, st);
  }
  return plan_eval_host(ctx, net, prob, x0, batch, actions, objective, diverged, tubes);
}

namespace {
int reach_cem_create_impl(const reach_plan_problem* prob, const reach_sampler_config* cfg, reach_cem** out,
                          bool allow_refine);
}

int reach_cem_create(const reach_plan_problem* prob, const reach_sampler_config* cfg, reach_cem** out) {
  return reach_cem_create_impl(prob, cfg, out, false);
}

}  // extern "C"

namespace {
int reach_cem_create_impl(const reach_plan_problem* prob, const reach_sampler_config* cfg, reach_cem** out,
                          bool allow_refine) {
  if (!prob || !cfg || !out) return REACH_E_INVALID_ARGUMENT;
  *out = nullptr;
  // SamplerConfig::validate (mpc.hpp:228-233)
  if (cfg->population < 2 || cfg->elite_frac <= 0.0 || cfg->elite_frac > 1.0 || cfg->iterations < 1 ||
      cfg->init_std <= 0.0 || cfg->smoothing < 0.0 || cfg->smoothing >= 1.0 || cfg->refine_iters < 0)
    return REACH_E_INVALID_ARGUMENT;
  // the piecewise CEM API leaves the refinement to its driver (reach_plan_objective_grad)
  if (cfg->refine_iters > 0 && !allow_refine) return REACH_E_UNSUPPORTED;
  if (prob->m < 1 || prob->horizon < 1) return REACH_E_INVALID_ARGUMENT;
  reach_cem* c = new reach_cem();
  c->h = prob->horizon;
  c->m = prob->m;
  c->u_lo.assign(prob->u_lo, prob->u_lo + prob->m);
  c->u_hi.assign(prob->u_hi, prob->u_hi + prob->m);
  c->cfg = *cfg;
  c->gen.seed(cfg->seed);
  const size_t dim = static_cast<size_t>(c->h) * c->m;
  c->mean.assign(dim, 0.0);
  c->stdv.assign(dim, cfg->init_std);
  for (int t = 0; t < c->h; ++t)
    for (int j = 0; j < c->m; ++j) c->mean[static_cast<size_t>(t) * c->m + j] = 0.5 * (c->u_lo[j] + c->u_hi[j]);
  c->best = c->mean;
  c->clip(c->best);
  c->n_elite = std::max(1, static_cast<int>(cfg->population * cfg->elite_frac));
  c->cands.assign(static_cast<size_t>(cfg->population), std::vector<double>(dim));
  *out = c;
  return REACH_OK;
}
}  // namespace

extern "C" {

int reach_cem_destroy(reach_cem* cem) {
  delete cem;
  return REACH_OK;
}

int reach_cem_sample(reach_cem* c, double* candidates) {
  if (!c || !candidates) return REACH_E_INVALID_ARGUMENT;
  if (c->it >= c->cfg.iterations) return REACH_E_INVALID_ARGUMENT;
  const size_t dim = c->mean.size();
  for (int k = 0; k < c->cfg.population; ++k) {  // mpc.hpp:290-299, sequential stream
    std::vector<double>& u = c->cands[static_cast<size_t>(k)];
    if (c->it > 0 && k == 0) {
      u = c->best;
    } else {
      for (size_t q = 0; q < dim; ++q) u[q] = c->mean[q] + c->stdv[q] * c->normal();
      c->clip(u);
    }
    std::copy(u.begin(), u.end(), candidates + static_cast<size_t>(k) * dim);
  }
  return REACH_OK;
}

int reach_cem_update(reach_cem* c, const double* scores, const int32_t* ok) {
  if (!c || !scores || !ok) return REACH_E_INVALID_ARGUMENT;
  const int pop = c->cfg.population;
  std::vector<int> order(static_cast<size_t>(pop));
  for (int k = 0; k < pop; ++k) order[static_cast<size_t>(k)] = k;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return scores[a] < scores[b]; });
  const int top = order.front();
  if (scores[top] < c->best_obj) {
    c->best_obj = scores[top];
    c->best = c->cands[static_cast<size_t>(top)];
  }
  for (int e = 0; e < c->n_elite; ++e)
    if (ok[order[static_cast<size_t>(e)]]) c->any_finite = true;
  c->history.push_back(c->best_obj);
  const double sm = c->cfg.smoothing;
  for (size_t k = 0; k < c->mean.size(); ++k) {  // mpc.hpp:320-333
    double em = 0.0, ev = 0.0;
    for (int e = 0; e < c->n_elite; ++e) em += c->cands[static_cast<size_t>(order[static_cast<size_t>(e)])][k];
    em /= c->n_elite;
    for (int e = 0; e < c->n_elite; ++e) {
      const double d = c->cands[static_cast<size_t>(order[static_cast<size_t>(e)])][k] - em;
      ev += d * d;
    }
    const double es = std::sqrt(ev / c->n_elite);
    c->mean[k] = sm * c->mean[k] + (1.0 - sm) * em;
    c->stdv[k] = std::max(1e-6, sm * c->stdv[k] + (1.0 - sm) * es);
  }
  ++c->it;
  return REACH_OK;
}

int reach_cem_result(const reach_cem* c, double* best_actions, double* best_objective, int32_t* best_effort,
                     double* best_history) {
  if (!c) return REACH_E_INVALID_ARGUMENT;
  if (best_actions) std::copy(c->best.begin(), c->best.end(), best_actions);
  if (best_objective) *best_objective = c->best_obj;
  if (best_effort) *best_effort = c->any_finite ? 0 : 1;
  if (best_history) std::copy(c->history.begin(), c->history.end(), best_history);
  return REACH_OK;
}

// gradient_refine (refine.hpp:347-398) of plan_objective from best_actions (the CEM's top candidate,
// objective best_obj): forward-dual gradients on the device, batched Armijo trials; best_actions is
// replaced when the refined objective is lower (mpc.hpp:337-361).
static int plan_refine_impl(reach_ctx* ctx, const reach_net* net, const reach_plan_problem* prob, const double* x0,
                            int iters, double best_obj, double* best_actions, int32_t* refined) {
  int rc = REACH_OK;
  {
    const size_t d = static_cast<size_t>(prob->horizon) * prob->m;
    std::vector<double> lo(d), hi(d), x(best_actions, best_actions + d), g(d), xn(d);
    for (size_t k = 0; k < d; ++k) {
      lo[k] = prob->u_lo[k % prob->m];
      hi[k] = prob->u_hi[k % prob->m];
    }
    auto project = [&](std::vector<double>& v) {
      for (size_t k = 0; k < d; ++k) v[k] = std::clamp(v[k], lo[k], hi[k]);
    };
    auto f = [&](const std::vector<double>& v, double& out) {
      int32_t dv2 = 0;
      return plan_eval_host(ctx, net, prob, x0, 1, v.data(), &out, &dv2, nullptr);
    };
    project(x);
    double fx = 0.0;
    rc = f(x, fx);
    if (rc) return rc;
    if (!std::isfinite(fx)) return fail(ctx, REACH_E_NONFINITE, "gradient_refine: initial objective non-finite");
    int accepted_steps = 0;
    std::vector<double> cands, fvals;
    std::vector<int32_t> cdiv;
    for (int it = 0; it < iters; ++it) {
      // grad_forward's primal pass (refine.hpp:190-193) re-evaluates f(x) = fx, finite by construction
      // (checked above or accepted below): evaluation is deterministic, so it is not repeated here
      double v = 0.0;
      bool fin = true;
      rc = plan_grad_device(ctx, net, prob, x0, x.data(), g.data(), &v, &fin);
      if (rc) return rc;
      if (!fin) return fail(ctx, REACH_E_NONFINITE, "grad_forward: non-finite derivative");
      double gnorm2 = 0.0;
      for (size_t k = 0; k < d; ++k) gnorm2 += g[k] * g[k];
      if (gnorm2 == 0.0) break;
      // Armijo backtracking (RefineParams: step0 1, shrink 0.5, armijo 1e-4, 30 backtracks).  The trial
      // points do not depend on earlier trials' objectives, so every trial up to the first one that does not
      // move is evaluated in ONE batch on the device and the first accepted trial is taken in order --
      // the same point the reference's sequential loop accepts.
      cands.clear();
      std::vector<double> moved_v;
      double t = 1.0;
      for (int bt = 0; bt < 30; ++bt, t *= 0.5) {
        for (size_t k = 0; k < d; ++k) xn[k] = x[k] - t * g[k];
        project(xn);
        double moved = 0.0;
        for (size_t k = 0; k < d; ++k) moved += g[k] * (x[k] - xn[k]);
        if (moved <= 0.0) break;
        cands.insert(cands.end(), xn.begin(), xn.end());
        moved_v.push_back(moved);
      }
      const int nt = static_cast<int>(moved_v.size());
      bool accepted = false;
      if (nt > 0) {
        fvals.assign(nt, 0.0);
        cdiv.assign(nt, 0);
        rc = plan_eval_host(ctx, net, prob, x0, nt, cands.data(), fvals.data(), cdiv.data(), nullptr);
        if (rc) return rc;
        for (int q = 0; q < nt; ++q) {
          const double fn = fvals[q];
          if (std::isfinite(fn) && fn <= fx - 1e-4 * moved_v[q]) {
            std::copy(cands.begin() + static_cast<size_t>(q) * d, cands.begin() + static_cast<size_t>(q + 1) * d,
                      x.begin());
            fx = fn;
            accepted = true;
            ++accepted_steps;
            break;
          }
        }
      }
      if (!accepted) break;
    }
    if (fx < best_obj) {
      std::copy(x.begin(), x.end(), best_actions);
      if (refined) *refined = accepted_steps > 0 ? 1 : 0;
    }
  }
  return REACH_OK;
}

int reach_plan_cem_ex(reach_ctx* ctx, const reach_net* net, const reach_plan_problem* prob,
                      const reach_sampler_config* cfg, const double* x0, double* best_actions, double* objective,
                      double* best_history, int32_t* best_effort, int32_t* refined, const reach_tube_out* final_tube) {
  rbh::DeviceGuard device_guard_(ctx);
  if (!ctx || !net || !prob || !cfg || !x0 || !best_actions || !objective) return REACH_E_INVALID_ARGUMENT;
  int rc = validate_problem(ctx, net, prob);
  if (rc) return rc;
  reach_cem* c = nullptr;
  rc = reach_cem_create_impl(prob, cfg, &c, /*allow_refine=*/true);
  if (rc) return fail(ctx, rc, "SamplerConfig: invalid configuration");
  std::unique_ptr<reach_cem> guard(c);
  const size_t dim = c->mean.size(), pop = cfg->population;
  const int iters = cfg->iterations;
  // The normal stream does not depend on mean/std, so it is drawn ahead on a
  // worker thread (same sequential order as mpc.hpp:290-299) while the device
  // evaluates the previous population.
  const size_t per_it0 = pop * dim, per_it = (pop - 1) * dim;
  // the whole normal stream of the replan in pinned host memory: uploaded per iteration, async
  const size_t z_count = per_it0 + static_cast<size_t>(iters - 1) * per_it;
  rc = ensure_pinned(ctx, z_count * sizeof(double));
  if (rc) return rc;
  double* z = static_cast<double*>(ctx->hpin);
  std::atomic<int> ready{0};
  // Rng::normal (rng.hpp:24-37) split in two: the uniform pairs (u1, u2; u1 redrawn while <= 0) are
  // drawn in stream order on the worker, then the Box-Muller transforms -- the same libm calls per
  // pair, independent of each other -- run on a few host threads; value k of the stream is bit for
  // bit what the sequential generator returns (cos first, sin cached as the spare).
  std::thread gen([&] {
    const unsigned nth = std::max(1u, std::min(8u, std::thread::hardware_concurrency()));
    std::vector<double> u1s, u2s;
    size_t o = 0;
    for (int it = 0; it < iters; ++it) {
      const size_t cnt = it == 0 ? per_it0 : per_it;
      size_t q = 0;
      if (cnt > 0 && c->has_spare) {
        z[o] = c->spare;
        c->has_spare = false;
        q = 1;
      }
      const size_t np = (cnt - q + 1) / 2;
      u1s.resize(np);
      u2s.resize(np);
      for (size_t p = 0; p < np; ++p) {
        double u1 = c->uniform01(), u2 = c->uniform01();
        while (u1 <= 0.0) u1 = c->uniform01();
        u1s[p] = u1;
        u2s[p] = u2;
      }
      double* zz = z + o + q;
      const size_t left = cnt - q;
      auto work = [&](size_t p0, size_t p1) {
        for (size_t p = p0; p < p1; ++p) {
          const double r = std::sqrt(-2.0 * std::log(u1s[p]));
          const double a = 6.28318530717958647692 * u2s[p];
          zz[2 * p] = r * std::cos(a);
          if (2 * p + 1 < left) zz[2 * p + 1] = r * std::sin(a);
        }
      };
      if (np < 4096 || nth == 1) {
        work(0, np);
      } else {
        std::vector<std::thread> pool;
        const size_t per = (np + nth - 1) / nth;
        for (unsigned t = 1; t < nth; ++t) {
          const size_t p0 = std::min(np, t * per), p1 = std::min(np, (t + 1) * per);
          if (p0 < p1) pool.emplace_back(work, p0, p1);
        }
        work(0, std::min(np, per));
        for (auto& th : pool) th.join();
      }
      if ((left & 1u) && np > 0) {  // the last pair's sine is the next draw (Rng's cached spare)
        const size_t p = np - 1;
        c->spare = std::sqrt(-2.0 * std::log(u1s[p])) * std::sin(6.28318530717958647692 * u2s[p]);
        c->has_spare = true;
      }
      o += cnt;
      ready.store(it + 1, std::memory_order_release);
    }
  });
  struct Joiner {
    std::thread& t;
    ~Joiner() {
      if (t.joinable()) t.join();
    }
  } joiner{gen};
  // The sampler runs on the device (cem_kernel.cuh): the population, its scores and the CEM state stay
  // in HBM across the iterations; the host only uploads each iteration's normals (async, pinned) and
  // reads the result once.
  const int H = prob->horizon, n = prob->n, m = prob->m;
  const int world = (ctx->has_coll && ctx->coll.world > 1) ? ctx->coll.world : 1;
  long long sb, se;
  rbh::coll_shard(ctx, 0, static_cast<long long>(pop), sb, se);
  const size_t width = (pop + world - 1) / world, nloc = static_cast<size_t>(se - sb);
  const size_t box = std::max<size_t>(nloc, 1) * (H + 1) * n * 8;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align_up(off + std::max<size_t>(bytes, 8), 256);
    return o;
  };
  const size_t o_x0 = take(n * 8), o_z = take(pop * dim * 8), o_c = take(pop * dim * 8), o_s = take(pop * 8),
               o_d = take(pop * 4), o_ls = take(width * 8), o_ld = take(width * 4), o_gs = take(world * width * 8),
               o_gd = take(world * width * 4), o_mean = take(dim * 8), o_std = take(dim * 8), o_best = take(dim * 8),
               o_bo = take(8), o_any = take(4), o_hist = take(iters * 8), o_lo = take(m * 8), o_hi = take(m * 8),
               o_tlo = take(box), o_thi = take(box), o_nb = take(width * 4), o_fs = take(width * 4),
               o_st = take(width * 4);
  rc = ensure_ws(ctx, off);
  if (rc) return rc;
  char* w = static_cast<char*>(ctx->ws);
  auto D = [&](size_t o) { return reinterpret_cast<double*>(w + o); };
  auto I = [&](size_t o) { return reinterpret_cast<int*>(w + o); };
  rb::cem::CemDev S{};
  S.cand = D(o_c);
  S.z = D(o_z);
  S.score = D(o_s);
  S.div = I(o_d);
  S.mean = D(o_mean);
  S.stdv = D(o_std);
  S.best = D(o_best);
  S.best_obj = D(o_bo);
  S.any_finite = I(o_any);
  S.hist = D(o_hist);
  S.lo = D(o_lo);
  S.hi = D(o_hi);
  S.pop = static_cast<int>(pop);
  S.dim = static_cast<int>(dim);
  S.m = m;
  S.n_elite = c->n_elite;
  S.smoothing = cfg->smoothing;
  RB_CUDA(cudaMemcpyAsync(D(o_x0), x0, n * 8, cudaMemcpyHostToDevice, ctx->stream));
  RB_CUDA(cudaMemcpyAsync(D(o_lo), prob->u_lo, m * 8, cudaMemcpyHostToDevice, ctx->stream));
  RB_CUDA(cudaMemcpyAsync(D(o_hi), prob->u_hi, m * 8, cudaMemcpyHostToDevice, ctx->stream));
  rb::cem::cem_init_kernel<<<1, 256, 0, ctx->stream>>>(S, cfg->init_std);
  RB_CUDA(cudaGetLastError());
  int p2 = 1;
  while (p2 < static_cast<int>(pop)) p2 <<= 1;
  const size_t usmem = static_cast<size_t>(p2) * (8 + 4);
  if (usmem > static_cast<size_t>(ctx->max_smem)) return fail(ctx, REACH_E_UNSUPPORTED, "CEM population too large");
  RB_CUDA(cudaFuncSetAttribute(rb::cem::cem_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(usmem)));
  const int gen_blocks = static_cast<int>(std::min<size_t>((pop * dim + 255) / 256, 4 * ctx->num_sms));
  size_t zo = 0;
  for (int it = 0; it < iters; ++it) {
    while (ready.load(std::memory_order_acquire) <= it) std::this_thread::yield();
    const size_t cnt = it == 0 ? per_it0 : per_it;
    RB_CUDA(cudaMemcpyAsync(D(o_z), z + zo, cnt * 8, cudaMemcpyHostToDevice, ctx->stream));
    zo += cnt;
    rb::cem::cem_generate_kernel<<<gen_blocks, 256, 0, ctx->stream>>>(S, it);
    RB_CUDA(cudaGetLastError());
    if (world == 1) {
      rc = plan_eval_device(ctx, net, prob, D(o_x0), static_cast<int>(pop), S.cand, D(o_s), I(o_d), D(o_tlo),
                            D(o_thi), I(o_nb), I(o_fs), I(o_st));
      if (rc) return rc;
    } else {
      RB_CUDA(cudaMemsetAsync(w + o_ls, 0, width * 8, ctx->stream));
      RB_CUDA(cudaMemsetAsync(w + o_ld, 0, width * 4, ctx->stream));
      if (nloc > 0) {
        rc = plan_eval_device(ctx, net, prob, D(o_x0), static_cast<int>(nloc), S.cand + sb * dim, D(o_ls), I(o_ld),
                              D(o_tlo), D(o_thi), I(o_nb), I(o_fs), I(o_st));
        if (rc) return rc;
      }
      rc = rbh::coll_allgather(ctx, D(o_ls), D(o_gs), width, REACH_DT_F64);
      if (!rc) rc = rbh::coll_allgather(ctx, I(o_ld), I(o_gd), width, REACH_DT_I32);
      if (rc) return rc;
      rb::cem::cem_unpad_kernel<<<std::max<int>(1, static_cast<int>((pop + 255) / 256)), 256, 0, ctx->stream>>>(
          D(o_gs), I(o_gd), world, static_cast<int>(width), static_cast<int>(pop), D(o_s), I(o_d));
      RB_CUDA(cudaGetLastError());
    }
    rb::cem::cem_update_kernel<<<1, 1024, usmem, ctx->stream>>>(S, it, p2);
    RB_CUDA(cudaGetLastError());
    ctx->launches += 2;
  }
  // the one read-back of the replan
  double best_obj = 0.0;
  int32_t any = 0;
  RB_CUDA(cudaMemcpyAsync(best_actions, S.best, dim * 8, cudaMemcpyDeviceToHost, ctx->stream));
  RB_CUDA(cudaMemcpyAsync(&best_obj, S.best_obj, 8, cudaMemcpyDeviceToHost, ctx->stream));
  RB_CUDA(cudaMemcpyAsync(&any, S.any_finite, 4, cudaMemcpyDeviceToHost, ctx->stream));
  if (best_history) RB_CUDA(cudaMemcpyAsync(best_history, S.hist, iters * 8, cudaMemcpyDeviceToHost, ctx->stream));
  RB_CUDA(cudaStreamSynchronize(ctx->stream));
  const int32_t be = any ? 0 : 1;
  if (best_effort) *best_effort = be;
  if (refined) *refined = 0;
  // gradient refinement of the top candidate (mpc.hpp:337-361):
  // gradient_refine (refine.hpp:347-398) with forward-dual gradients on the device
  if (cfg->refine_iters > 0 && std::isfinite(best_obj)) {
    rc = plan_refine_impl(ctx, net, prob, x0, cfg->refine_iters, best_obj, best_actions, refined);
    if (rc) return rc;
  }
  // final evaluation of the chosen plan (mpc.hpp:363-367)
  int32_t dv = 0;
  rc = plan_eval_host(ctx, net, prob, x0, 1, best_actions, objective, &dv, final_tube);
  return rc;
}

int reach_plan_cem(reach_ctx* ctx, const reach_net* net, const reach_plan_problem* prob,
                   const reach_sampler_config* cfg, const double* x0, double* best_actions, double* objective,
                   double* best_history, int32_t* best_effort, const reach_tube_out* final_tube) {
  rbh::DeviceGuard device_guard_(ctx);
  return reach_plan_cem_ex(ctx, net, prob, cfg, x0, best_actions, objective, best_history, best_effort, nullptr,
                           final_tube);
}

int reach_plan_objective_grad(reach_ctx* ctx, const reach_net* net, const reach_plan_problem* prob, const double* x0,
                              const double* actions, double* grad, double* objective) {
  rbh::DeviceGuard device_guard_(ctx);
  if (!ctx || !net || !prob || !x0 || !actions || !grad) return REACH_E_INVALID_ARGUMENT;
  int rc = validate_problem(ctx, net, prob);
  if (rc) return rc;
  double v = 0.0;
  bool fin = true;
  rc = plan_grad_device(ctx, net, prob, x0, actions, grad, &v, &fin);
  if (rc) return rc;
  if (objective) *objective = v;
  if (!fin) return fail(ctx, REACH_E_NONFINITE, "grad_forward: non-finite derivative");
  return REACH_OK;
}

}  // extern "C"

namespace {
// grad_tube_volume with X0 = box_from_center(center, radius) given directly (refine.hpp:283, the CLI's
// refine objective uses box_from_center(c, eps)); a supplies the shapes, actions and DTReachParams.
int grad_tube_volume_cr(reach_ctx* ctx, const reach_net* net, const reach_dt_args* a, const double* center,
                        const double* radius, int32_t target, int32_t method, double* grad, int32_t* subgradient,
                        double* volume, long long begin = 0, long long end = -1) {
  namespace rd = rb::dual;
  const int n = a->n, m = a->m, H = a->horizon;
  rd::VolArgs V{};
  V.poff[0] = 0;
  for (int l = 0; l < net->L; ++l)
    V.poff[l + 1] = V.poff[l] + static_cast<long long>(net->dims[l + 1]) * net->dims[l] + net->dims[l + 1];
  const long long full = target == REACH_GRAD_X0_CENTER ? n
                         : target == REACH_GRAD_ACTIONS ? static_cast<long long>(H) * m
                                                        : V.poff[net->L];
  if (end < 0) end = full;
  if (begin < 0 || begin > end || end > full)
    return fail(ctx, REACH_E_INVALID_ARGUMENT, "grad_tube_volume: parameter range out of bounds");
  const long long dim = end - begin;  // this call's slice of the parameters
  V.p0 = begin;
  const bool fd = method == REACH_GRAD_FINITE_DIFFERENCE;
  const long long passes = fd ? 2 * dim + 1 : dim;
  if (passes > (1ll << 30)) return fail(ctx, REACH_E_UNSUPPORTED, "grad_tube_volume: too many parameters");
  if (subgradient) *subgradient = 0;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align_up(off + std::max<size_t>(bytes, 8), 256);
    return o;
  };
  const long long np = std::max<long long>(passes, 1);
  const size_t o_c = take(n * 8), o_r = take(n * 8), o_a = take(static_cast<size_t>(H) * m * 8),
               o_v = take(static_cast<size_t>(np) * 8), o_t = take(static_cast<size_t>(np) * 8), o_s = take(4);
  int rc = ensure_ws(ctx, off);
  if (rc) return rc;
  char* w = static_cast<char*>(ctx->ws);
  auto Dp = [&](size_t o) { return reinterpret_cast<double*>(w + o); };
  RB_CUDA(cudaMemcpyAsync(Dp(o_c), center, n * 8, cudaMemcpyHostToDevice, ctx->stream));
  RB_CUDA(cudaMemcpyAsync(Dp(o_r), radius, n * 8, cudaMemcpyHostToDevice, ctx->stream));
  if (H * m > 0)
    RB_CUDA(cudaMemcpyAsync(Dp(o_a), a->actions, static_cast<size_t>(H) * m * 8, cudaMemcpyHostToDevice, ctx->stream));
  RB_CUDA(cudaMemsetAsync(w + o_s, 0, 4, ctx->stream));
  V.net = net->dev;
  V.n = n;
  V.m = m;
  V.H = H;
  V.window = a->window;
  V.rebuild = a->rebuild_from_box;
  V.center = Dp(o_c);
  V.radius = Dp(o_r);
  V.actions = Dp(o_a);
  V.target = target;
  V.dim = static_cast<int>(dim);
  V.fd = fd ? 1 : 0;
  V.rel_step = 1e-5;
  V.value = Dp(o_v);
  V.tangent = Dp(o_t);
  V.sub = reinterpret_cast<int*>(w + o_s);
  // grad_forward with no parameters still runs its primal pass: launch one unseeded pass
  const long long launch = passes > 0 ? passes : 1;
  if (passes == 0) V.fd = 1;  // dim 0: pass 0 == 2 * dim is the unperturbed pass
  RB_CUDA(cudaFuncSetAttribute(rd::tube_volume_grad_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(sizeof(rd::Work))));
  cudaEvent_t stop;
  rc = timed_begin(ctx, &stop);
  if (rc) return rc;
  rd::tube_volume_grad_kernel<<<static_cast<unsigned>(launch), rd::kThreads, sizeof(rd::Work), ctx->stream>>>(V);
  RB_CUDA(cudaGetLastError());
  rc = timed_end(ctx, stop);
  if (rc) return rc;
  ctx->launches += 1;
  std::vector<double> val(launch), tan(launch);
  int32_t sub = 0;
  RB_CUDA(cudaMemcpyAsync(val.data(), Dp(o_v), launch * 8, cudaMemcpyDeviceToHost, ctx->stream));
  RB_CUDA(cudaMemcpyAsync(tan.data(), Dp(o_t), launch * 8, cudaMemcpyDeviceToHost, ctx->stream));
  RB_CUDA(cudaMemcpyAsync(&sub, w + o_s, 4, cudaMemcpyDeviceToHost, ctx->stream));
  RB_CUDA(cudaStreamSynchronize(ctx->stream));
  const double f0 = (fd || passes == 0) ? val[launch - 1] : val[0];  // primal values are identical across passes
  if (volume) *volume = f0;
  if (!std::isfinite(f0))
    return fail(ctx, REACH_E_NONFINITE, fd ? "grad_fd: objective non-finite" : "grad_forward: objective non-finite");
  for (long long j = 0; j < dim; ++j) {
    if (!fd) {
      if (!std::isfinite(val[j]) || !std::isfinite(tan[j]))
        return fail(ctx, REACH_E_NONFINITE, "grad_forward: non-finite derivative");
      grad[j] = tan[j];
    } else {
      const double fp = val[2 * j], fm = val[2 * j + 1];
      if (!std::isfinite(fp) || !std::isfinite(fm))
        return fail(ctx, REACH_E_NONFINITE, "grad_fd: objective non-finite near x");
      double xj;  // the parameter value, for h (refine.hpp:222)
      const long long pj = begin + j;
      if (target == REACH_GRAD_X0_CENTER) {
        xj = center[pj];
      } else if (target == REACH_GRAD_ACTIONS) {
        xj = a->actions[pj];
      } else {
        xj = net->params[static_cast<size_t>(pj)];  // net_params order == the upload's flat order
      }
      const double h = 1e-5 * std::max(1.0, std::abs(xj));
      grad[j] = (fp - fm) / (2.0 * h);
    }
  }
  if (subgradient) *subgradient = sub ? 1 : 0;
  return REACH_OK;
}
}  // namespace

extern "C" {

int reach_grad_tube_volume(reach_ctx* ctx, const reach_net* net, const reach_dt_args* a, int32_t target,
                           int32_t method, double* grad, int32_t* subgradient, double* volume) {
  rbh::DeviceGuard device_guard_(ctx);
  return reach_grad_tube_volume_range(ctx, net, a, target, method, 0, -1, grad, subgradient, volume);
}

int reach_grad_tube_volume_range(reach_ctx* ctx, const reach_net* net, const reach_dt_args* a, int32_t target,
                                 int32_t method, int64_t param_begin, int64_t param_end, double* grad,
                                 int32_t* subgradient, double* volume) {
  rbh::DeviceGuard device_guard_(ctx);
  namespace rd = rb::dual;
  if (!ctx || !net || !a || !grad) return REACH_E_INVALID_ARGUMENT;
  if (a->batch != 1) return fail(ctx, REACH_E_INVALID_ARGUMENT, "grad_tube_volume: batch must be 1");
  if (a->horizon < 0) return fail(ctx, REACH_E_INVALID_ARGUMENT, "dt_reach: negative horizon");
  if (target < REACH_GRAD_X0_CENTER || target > REACH_GRAD_WEIGHTS || method < REACH_GRAD_FORWARD_DUAL ||
      method > REACH_GRAD_FINITE_DIFFERENCE)
    return fail(ctx, REACH_E_INVALID_ARGUMENT, "grad_tube_volume: unknown target / method");
  int rc = validate_system(ctx, net, a->n, a->m);
  if (rc) return rc;
  const int n = a->n, m = a->m, H = a->horizon;
  if (!a->x0_lo || !a->x0_hi || (H * m > 0 && !a->actions))
    return fail(ctx, REACH_E_INVALID_ARGUMENT, "grad_tube_volume: missing input");
  int maxw = 0;
  for (int l = 0; l <= net->L; ++l) maxw = std::max(maxw, net->dims[l]);
  const int cap = a->window > 0 ? a->window : 1;
  if (n > rd::kN || m > rd::kM || maxw > rd::kW || net->L > rd::kL || H > rd::kH || n * (cap + 2) > rd::kZ ||
      n * (cap + 2) + n > rd::kW || cap + 2 > rd::kQ)
    return fail(ctx, REACH_E_UNSUPPORTED, "grad_tube_volume: shape outside the Dual kernel family");
  // box_center / box_radius (interval.hpp:270-281), box_from_center's radius check (interval.hpp:229)
  std::vector<double> center(n), radius(n);
  for (int i = 0; i < n; ++i) {
    center[i] = (a->x0_lo[i] + a->x0_hi[i]) * 0.5;
    radius[i] = (a->x0_hi[i] - a->x0_lo[i]) * 0.5;
    if (radius[i] < 0.0) return fail(ctx, REACH_E_INVALID_ARGUMENT, "box_from_center: negative radius");
  }
  return grad_tube_volume_cr(ctx, net, a, center.data(), radius.data(), target, method, grad, subgradient, volume,
                             param_begin, param_end);
}

// mpc_run (mpc.hpp:425-495): receding-horizon execution around plan_cem.
// Planning, the simulator (the uploaded model's forward when sim == NULL, the
// CLI's choice, reach_cli.cpp:445-449) and the constraint margins run on the
// device; the loop, the disturbance stream (std::mt19937_64(cfg.seed), 53-bit
// uniforms) and the log bookkeeping are the reference's host logic.
int reach_mpc_run(reach_ctx* ctx, const reach_net* net, const reach_plan_problem* prob,
                  const reach_sampler_config* sampler, const reach_mpc_config* cfg, reach_sim_fn sim, void* sim_user,
                  const double* x0, int32_t* success, int32_t* violated, int32_t* steps_used, double* final_state,
                  const reach_mpc_log* log, int32_t* log_rows) {
  rbh::DeviceGuard device_guard_(ctx);
  if (!ctx || !net || !prob || !sampler || !cfg || !x0) return REACH_E_INVALID_ARGUMENT;
  int rc = validate_problem(ctx, net, prob);
  if (rc) return rc;
  if (cfg->replan_period < 1 || cfg->replan_period > prob->horizon || cfg->total_steps < 1 ||
      cfg->dist_action < 0.0 || cfg->dist_state < 0.0 || cfg->goal_radius <= 0.0)
    return fail(ctx, REACH_E_INVALID_ARGUMENT, "MPCConfig: invalid configuration");
  const int n = prob->n, m = prob->m, H = prob->horizon;
  for (int j = 0; j < cfg->n_goal_dims; ++j)
    if (!cfg->goal_dims || cfg->goal_dims[j] < 0 || cfg->goal_dims[j] >= n)
      return fail(ctx, REACH_E_INVALID_ARGUMENT, "MPCConfig: goal dim out of range");
  if (!sim && (net->dims[0] != n + m || net->dims[net->L] != n))
    return fail(ctx, REACH_E_INVALID_ARGUMENT, "mpc_run: the model simulator needs the one-step map");
  // device buffers of this run (own allocation: plan_cem may grow the context workspace)
  PlanBuffers pb;
  pack_problem(prob, pb);
  int maxw = 0;
  for (int l = 0; l <= net->L; ++l) maxw = std::max(maxw, net->dims[l]);
  const size_t nb_boxes = static_cast<size_t>(H) + 1;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align_up(off + std::max<size_t>(bytes, 8), 256);
    return o;
  };
  const size_t o_db = take(pb.db.size() * 8), o_ib = take(pb.ib.size() * 4), o_xu = take((n + m) * 8),
               o_x = take(n * 8), o_lo = take(nb_boxes * n * 8), o_hi = take(nb_boxes * n * 8),
               o_mg = take(nb_boxes * 8);
  char* dev = nullptr;
  RB_CUDA(cudaMalloc(&dev, off));
  struct Free {
    char* p;
    ~Free() { cudaFree(p); }
  } free_guard{dev};
  auto Dp = [&](size_t o) { return reinterpret_cast<double*>(dev + o); };
  RB_CUDA(cudaMemcpyAsync(Dp(o_db), pb.db.data(), pb.db.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
  RB_CUDA(cudaMemcpyAsync(dev + o_ib, pb.ib.data(), pb.ib.size() * 4, cudaMemcpyHostToDevice, ctx->stream));
  rb::PlanParams MP = pb.P;
  MP.n = n;
  MP.dbuf = Dp(o_db);
  MP.ibuf = reinterpret_cast<const int*>(dev + o_ib);
  // margins of K boxes on the device (plan_step_margin, mpc.hpp:211-215)
  auto margins = [&](const double* lo, const double* hi, int K, double* out) -> int {
    RB_CUDA(cudaMemcpyAsync(Dp(o_lo), lo, static_cast<size_t>(K) * n * 8, cudaMemcpyHostToDevice, ctx->stream));
    RB_CUDA(cudaMemcpyAsync(Dp(o_hi), hi, static_cast<size_t>(K) * n * 8, cudaMemcpyHostToDevice, ctx->stream));
    rb::box_margin_kernel<<<(K + 127) / 128, 128, 0, ctx->stream>>>(MP, Dp(o_lo), Dp(o_hi), K, Dp(o_mg));
    RB_CUDA(cudaGetLastError());
    ctx->launches += 1;
    RB_CUDA(cudaMemcpyAsync(out, Dp(o_mg), static_cast<size_t>(K) * 8, cudaMemcpyDeviceToHost, ctx->stream));
    RB_CUDA(cudaStreamSynchronize(ctx->stream));
    return REACH_OK;
  };
  auto state_ok = [&](const std::vector<double>& s, bool& ok) -> int {  // box_from_center(s, 0.0)
    std::vector<double> lo(s), hi(s);
    for (int d = 0; d < n; ++d) {
      lo[d] = s[d] - 0.0;
      hi[d] = s[d] + 0.0;
    }
    double g = 0.0;
    int e = margins(lo.data(), hi.data(), 1, &g);
    ok = g >= 0.0;
    return e;
  };
  auto goal_reached = [&](const std::vector<double>& s) {
    double d2 = 0.0;
    const int k = cfg->n_goal_dims > 0 ? cfg->n_goal_dims : n;
    for (int j = 0; j < k; ++j) {
      const int d = cfg->n_goal_dims > 0 ? cfg->goal_dims[j] : j;
      const double diff = s[d] - prob->x_goal[d];
      d2 += diff * diff;
    }
    return std::sqrt(d2) <= cfg->goal_radius;
  };
  auto sim_step = [&](const std::vector<double>& x, const std::vector<double>& u, std::vector<double>& xn) -> int {
    if (sim) {
      if (sim(sim_user, x.data(), u.data(), xn.data()) != 0)
        return fail(ctx, REACH_E_INVALID_ARGUMENT, "mpc_run: sim_step failed");
      return REACH_OK;
    }
    std::vector<double> xu(x);
    xu.insert(xu.end(), u.begin(), u.end());
    RB_CUDA(cudaMemcpyAsync(Dp(o_xu), xu.data(), xu.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
    rb::model_step_kernel<<<1, 256, 2 * maxw * sizeof(double), ctx->stream>>>(net->dev, Dp(o_xu), Dp(o_x), maxw);
    RB_CUDA(cudaGetLastError());
    ctx->launches += 1;
    RB_CUDA(cudaMemcpyAsync(xn.data(), Dp(o_x), n * 8, cudaMemcpyDeviceToHost, ctx->stream));
    RB_CUDA(cudaStreamSynchronize(ctx->stream));
    return REACH_OK;
  };
  std::mt19937_64 rng(cfg->seed);
  auto uniform = [&](double lo, double hi) {  // Rng::uniform (rng.hpp:22)
    return lo + (hi - lo) * (static_cast<double>(rng() >> 11) * 0x1.0p-53);
  };
  std::vector<double> x(x0, x0 + n), xn(n), u(m), best(static_cast<size_t>(H) * m), hist(sampler->iterations);
  std::vector<double> tlo(nb_boxes * n), thi(nb_boxes * n);
  int32_t tnb = 0, tfs = -1, tst = 0;
  reach_tube_out tube{tlo.data(), thi.data(), &tnb, &tfs, &tst};
  bool viol = false, ok = true;
  int rows = 0;
  auto finish = [&](int used, bool succ) {
    if (success) *success = succ ? 1 : 0;
    if (violated) *violated = viol ? 1 : 0;
    if (steps_used) *steps_used = used;
    if (final_state) std::copy(x.begin(), x.end(), final_state);
    if (log_rows) *log_rows = rows;
    return REACH_OK;
  };
  if ((rc = state_ok(x, ok))) return rc;
  if (!ok) viol = true;
  int step = 0;
  reach_sampler_config plan_cfg = *sampler;
  while (step < cfg->total_steps && !goal_reached(x)) {
    plan_cfg.seed = sampler->seed ^ (0x9e3779b97f4a7c15ull * static_cast<uint64_t>(step + 1));
    double pobj = 0.0;
    int32_t be = 0, rf = 0;
    rc = reach_plan_cem_ex(ctx, net, prob, &plan_cfg, x.data(), best.data(), &pobj, hist.data(), &be, &rf, &tube);
    if (rc) return rc;
    // tube_volume of the plan's tube (tube.hpp:40-46) and the per-step planned margins
    double tvol = std::numeric_limits<double>::infinity();
    if (tst == REACH_TUBE_OK) {
      tvol = 0.0;
      for (int k = 0; k < tnb; ++k) {
        double v = 0.0;
        for (int d = 0; d < n; ++d) v += thi[static_cast<size_t>(k) * n + d] - tlo[static_cast<size_t>(k) * n + d];
        tvol += v;
      }
    }
    std::vector<double> gm(std::max(tnb, 1));
    if (tnb > 0 && (rc = margins(tlo.data(), thi.data(), tnb, gm.data()))) return rc;
    for (int k = 0; k < cfg->replan_period && step < cfg->total_steps; ++k, ++step) {
      for (int j = 0; j < m; ++j) {
        double v = best[static_cast<size_t>(k) * m + j];
        v += uniform(-cfg->dist_action, cfg->dist_action);
        u[j] = std::clamp(v, prob->u_lo[j], prob->u_hi[j]);
      }
      if (log && rows < cfg->total_steps) {
        if (log->step) log->step[rows] = step;
        if (log->state) std::copy(x.begin(), x.end(), log->state + static_cast<size_t>(rows) * n);
        if (log->action) std::copy(u.begin(), u.end(), log->action + static_cast<size_t>(rows) * m);
        if (log->objective) log->objective[rows] = pobj;
        if (log->tube_volume) log->tube_volume[rows] = tvol;
        if (log->g_margin) log->g_margin[rows] = (k + 1 < tnb) ? gm[k + 1] : -std::numeric_limits<double>::infinity();
      }
      ++rows;
      if ((rc = sim_step(x, u, xn))) return rc;
      x = xn;
      for (auto& v : x) {
        if (!std::isfinite(v)) return finish(step + 1, false);  // simulator divergence: failure with log
        v += uniform(-cfg->dist_state, cfg->dist_state);
      }
      if ((rc = state_ok(x, ok))) return rc;
      if (!ok) viol = true;
      if (goal_reached(x)) {
        ++step;
        break;
      }
    }
  }
  return finish(step, goal_reached(x) && !viol);
}

// gradient_refine (refine.hpp:354-398) of tube_volume(dt_reach(box_from_center(c, r), actions)) over
// the X0 centre or the action sequence -- the reference CLI's `refine` (reach_cli.cpp:293-341).  Forward-dual
// gradients from tube_volume_grad_kernel; the Armijo trial points of one iteration are evaluated in one
// dt_reach batch on the device and the first accepted one is taken in order.
int reach_refine_tube_volume(reach_ctx* ctx, const reach_net* net, const reach_dt_args* a, const double* center,
                             const double* radius, int32_t target, const double* lo, const double* hi,
                             int32_t iters, double* x, double* initial_objective, double* objective,
                             int32_t* progressed, int32_t* subgradient, int32_t* accepted_steps) {
  rbh::DeviceGuard device_guard_(ctx);
  if (!ctx || !net || !a || !center || !radius || !lo || !hi || !x) return REACH_E_INVALID_ARGUMENT;
  if (target != REACH_GRAD_X0_CENTER && target != REACH_GRAD_ACTIONS)
    return fail(ctx, REACH_E_INVALID_ARGUMENT, "refine: target must be the X0 centre or the actions");
  if (iters < 0) return fail(ctx, REACH_E_INVALID_ARGUMENT, "RefineParams: invalid configuration");
  int rc = validate_system(ctx, net, a->n, a->m);
  if (rc) return rc;
  const int n = a->n, m = a->m, H = a->horizon;
  if (H < 0 || (H * m > 0 && !a->actions)) return fail(ctx, REACH_E_INVALID_ARGUMENT, "refine: missing actions");
  for (int i = 0; i < n; ++i)
    if (radius[i] < 0.0) return fail(ctx, REACH_E_INVALID_ARGUMENT, "box_from_center: negative radius");
  const size_t d = target == REACH_GRAD_X0_CENTER ? n : static_cast<size_t>(H) * m;
  for (size_t j = 0; j < d; ++j)
    if (!(lo[j] <= hi[j])) return fail(ctx, REACH_E_INVALID_ARGUMENT, "gradient_refine: empty bound box");
  std::vector<double> xv(x, x + d), g(d), xn(d);
  auto project = [&](std::vector<double>& v) {
    for (size_t j = 0; j < d; ++j) v[j] = std::clamp(v[j], lo[j], hi[j]);
  };
  // f of K points (rows of pts): one dt_reach batch, tube_volume per tube (tube.hpp:40-46)
  const size_t boxes = static_cast<size_t>(H) + 1;
  auto f_batch = [&](const std::vector<double>& pts, int K, std::vector<double>& fv) -> int {
    std::vector<double> x0lo(static_cast<size_t>(K) * n), x0hi(x0lo.size()),
        acts(static_cast<size_t>(K) * H * m), olo(static_cast<size_t>(K) * boxes * n), ohi(olo.size());
    std::vector<int32_t> nb(K), fs(K), st(K);
    for (int k = 0; k < K; ++k) {
      const double* p = pts.data() + static_cast<size_t>(k) * d;
      for (int i = 0; i < n; ++i) {
        const double c = target == REACH_GRAD_X0_CENTER ? p[i] : center[i];
        x0lo[static_cast<size_t>(k) * n + i] = c - radius[i];
        x0hi[static_cast<size_t>(k) * n + i] = c + radius[i];
      }
      for (size_t q = 0; q < static_cast<size_t>(H) * m; ++q)
        acts[static_cast<size_t>(k) * H * m + q] = target == REACH_GRAD_ACTIONS ? p[q] : a->actions[q];
    }
    reach_dt_args b = *a;
    b.batch = K;
    b.x0_lo = x0lo.data();
    b.x0_hi = x0hi.data();
    b.actions = acts.empty() ? nullptr : acts.data();
    b.actions_shared = 0;
    reach_tube_out o{olo.data(), ohi.data(), nb.data(), fs.data(), st.data()};
    int e = run_dt_batch(ctx, net, nullptr, &b, &o, 0);
    if (e) return e;
    fv.assign(K, std::numeric_limits<double>::infinity());
    for (int k = 0; k < K; ++k) {
      if (st[k] != REACH_TUBE_OK) continue;
      double acc = 0.0;
      for (int t = 0; t < nb[k]; ++t) {
        double v = 0.0;
        for (int i = 0; i < n; ++i) {
          const size_t q = (static_cast<size_t>(k) * boxes + t) * n + i;
          v += ohi[q] - olo[q];
        }
        acc += v;
      }
      fv[k] = acc;
    }
    return REACH_OK;
  };
  project(xv);
  std::vector<double> fv;
  if ((rc = f_batch(xv, 1, fv))) return rc;
  double fx = fv[0];
  if (!std::isfinite(fx)) return fail(ctx, REACH_E_NONFINITE, "gradient_refine: initial objective non-finite");
  if (initial_objective) *initial_objective = fx;
  int acc_steps = 0;
  bool sub_any = false;
  std::vector<double> cands, moved_v, cvec(center, center + n);
  for (int it = 0; it < iters; ++it) {
    reach_dt_args ga = *a;
    ga.batch = 1;
    if (target == REACH_GRAD_ACTIONS) ga.actions = xv.data();
    int32_t sub = 0;
    double vol = 0.0;
    rc = grad_tube_volume_cr(ctx, net, &ga, target == REACH_GRAD_X0_CENTER ? xv.data() : cvec.data(), radius, target,
                             REACH_GRAD_FORWARD_DUAL, g.data(), &sub, &vol);
    if (rc) return rc;
    sub_any = sub_any || sub != 0;
    double gnorm2 = 0.0;
    for (size_t j = 0; j < d; ++j) gnorm2 += g[j] * g[j];
    if (gnorm2 == 0.0) break;
    cands.clear();
    moved_v.clear();
    double t = 1.0;
    for (int bt = 0; bt < 30; ++bt, t *= 0.5) {
      for (size_t j = 0; j < d; ++j) xn[j] = xv[j] - t * g[j];
      project(xn);
      double moved = 0.0;
      for (size_t j = 0; j < d; ++j) moved += g[j] * (xv[j] - xn[j]);
      if (moved <= 0.0) break;
      cands.insert(cands.end(), xn.begin(), xn.end());
      moved_v.push_back(moved);
    }
    bool accepted = false;
    if (!moved_v.empty()) {
      if ((rc = f_batch(cands, static_cast<int>(moved_v.size()), fv))) return rc;
      for (size_t q = 0; q < moved_v.size(); ++q)
        if (std::isfinite(fv[q]) && fv[q] <= fx - 1e-4 * moved_v[q]) {
          std::copy(cands.begin() + q * d, cands.begin() + (q + 1) * d, xv.begin());
          fx = fv[q];
          accepted = true;
          ++acc_steps;
          break;
        }
    }
    if (!accepted) break;
  }
  std::copy(xv.begin(), xv.end(), x);
  if (objective) *objective = fx;
  if (progressed) *progressed = acc_steps > 0 ? 1 : 0;
  if (subgradient) *subgradient = sub_any ? 1 : 0;
  if (accepted_steps) *accepted_steps = acc_steps;
  return REACH_OK;
}

// reach_loss (training.hpp:99-126) of a batch of M episodes and, optionally, its gradient over the
// network parameters (grad_forward, refine.hpp:186-207, in net_params order).
int reach_reach_loss(reach_ctx* ctx, const reach_net* net, const reach_dt_args* a, int32_t episodes,
                     double eps, double cap, double* loss, double* grad, int32_t* diverged_count) {
  rbh::DeviceGuard device_guard_(ctx);
  namespace rd = rb::dual;
  if (!ctx || !net || !a || !loss) return REACH_E_INVALID_ARGUMENT;
  if (episodes < 1 || a->horizon < 1) return fail(ctx, REACH_E_INVALID_ARGUMENT, "reach_loss: bad batch/horizon");
  int rc = validate_system(ctx, net, a->n, a->m);
  if (rc) return rc;
  const int n = a->n, m = a->m, H = a->horizon, M = episodes;
  if (!a->x0_lo || (m > 0 && !a->actions)) return fail(ctx, REACH_E_INVALID_ARGUMENT, "reach_loss: missing input");
  if (eps < 0.0) return fail(ctx, REACH_E_INVALID_ARGUMENT, "box_from_center: negative radius");
  int maxw = 0;
  for (int l = 0; l <= net->L; ++l) maxw = std::max(maxw, net->dims[l]);
  const int cap_q = a->window > 0 ? a->window : 1;
  if (n > rd::kN || m > rd::kM || maxw > rd::kW || net->L > rd::kL || H > rd::kH || n * (cap_q + 2) > rd::kZ ||
      n * (cap_q + 2) + n > rd::kW || cap_q + 2 > rd::kQ || M > 65535)
    return fail(ctx, REACH_E_UNSUPPORTED, "reach_loss: shape outside the Dual kernel family");
  rd::LossArgs L{};
  L.poff[0] = 0;
  for (int l = 0; l < net->L; ++l)
    L.poff[l + 1] = L.poff[l] + static_cast<long long>(net->dims[l + 1]) * net->dims[l] + net->dims[l + 1];
  const long long P = grad ? L.poff[net->L] : 1;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align_up(off + std::max<size_t>(bytes, 8), 256);
    return o;
  };
  const size_t o_x = take(static_cast<size_t>(M) * n * 8), o_a = take(static_cast<size_t>(M) * H * m * 8),
               o_v = take(static_cast<size_t>(P) * M * 8), o_d = take(static_cast<size_t>(P) * M * 8),
               o_div = take(static_cast<size_t>(M) * 4);
  rc = ensure_ws(ctx, off);
  if (rc) return rc;
  char* w = static_cast<char*>(ctx->ws);
  auto Dp = [&](size_t o) { return reinterpret_cast<double*>(w + o); };
  RB_CUDA(cudaMemcpyAsync(Dp(o_x), a->x0_lo, static_cast<size_t>(M) * n * 8, cudaMemcpyHostToDevice, ctx->stream));
  if (m > 0)
    RB_CUDA(cudaMemcpyAsync(Dp(o_a), a->actions, static_cast<size_t>(M) * H * m * 8, cudaMemcpyHostToDevice,
                            ctx->stream));
  L.net = net->dev;
  L.n = n;
  L.m = m;
  L.H = H;
  L.window = a->window;
  L.rebuild = a->rebuild_from_box;
  L.M = M;
  L.x0 = Dp(o_x);
  L.actions = Dp(o_a);
  L.eps = eps;
  L.cap = cap;
  L.seeded = grad ? 1 : 0;
  L.term_v = Dp(o_v);
  L.term_d = Dp(o_d);
  L.diverged = reinterpret_cast<int*>(w + o_div);
  RB_CUDA(cudaFuncSetAttribute(rd::reach_loss_grad_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(sizeof(rd::Work))));
  cudaEvent_t stop;
  rc = timed_begin(ctx, &stop);
  if (rc) return rc;
  rd::reach_loss_grad_kernel<<<dim3(static_cast<unsigned>(P), static_cast<unsigned>(M)), rd::kThreads,
                               sizeof(rd::Work), ctx->stream>>>(L);
  RB_CUDA(cudaGetLastError());
  rc = timed_end(ctx, stop);
  if (rc) return rc;
  ctx->launches += 1;
  std::vector<double> tv(static_cast<size_t>(P) * M), td(tv.size());
  std::vector<int32_t> dv(M);
  RB_CUDA(cudaMemcpyAsync(tv.data(), Dp(o_v), tv.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
  RB_CUDA(cudaMemcpyAsync(td.data(), Dp(o_d), td.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
  RB_CUDA(cudaMemcpyAsync(dv.data(), w + o_div, static_cast<size_t>(M) * 4, cudaMemcpyDeviceToHost, ctx->stream));
  RB_CUDA(cudaStreamSynchronize(ctx->stream));
  // acc += term per episode, then acc / S(M) (scalar.hpp:22-28: (a.d*b.v - a.v*b.d) / (b.v*b.v))
  const double Md = static_cast<double>(M);
  for (long long p = 0; p < P; ++p) {
    double av = 0.0, ad = 0.0;
    for (int e = 0; e < M; ++e) {
      av = av + tv[static_cast<size_t>(p) * M + e];
      ad = ad + td[static_cast<size_t>(p) * M + e];
    }
    if (p == 0) *loss = av / Md;
    if (grad) grad[p] = (ad * Md - av * 0.0) / (Md * Md);
  }
  if (diverged_count) {
    int c = 0;
    for (int e = 0; e < M; ++e) c += dv[e];
    *diverged_count = c;
  }
  return REACH_OK;
}

// pred_loss (training.hpp:60-83) of a batch and, optionally, its grad_forward over net_params.
int reach_pred_loss(reach_ctx* ctx, const reach_net* net, const reach_episode_set* b, int32_t t_h,
                    const double* weights, double* loss, double* grad) {
  rbh::DeviceGuard device_guard_(ctx);
  namespace rd = rb::dual;
  if (!ctx || !net || !b || !loss) return REACH_E_INVALID_ARGUMENT;
  if (b->episodes < 1 || t_h < 1 || !weights)
    return fail(ctx, REACH_E_INVALID_ARGUMENT, "pred_loss: bad batch/horizon/weights");
  if (b->length < t_h) return fail(ctx, REACH_E_INVALID_ARGUMENT, "pred_loss: episode shorter than T_h");
  const int n = b->n, m = b->m, M = b->episodes, T = t_h, Ls = b->length;
  if (n < 1 || m < 0 || !b->states || (m > 0 && !b->actions))
    return fail(ctx, REACH_E_INVALID_ARGUMENT, "pred_loss: missing episode data");
  if (net->dims[0] != n + m || net->dims[net->L] != n)
    return fail(ctx, REACH_E_INVALID_ARGUMENT, "pred_loss: model shape does not match the episodes");
  int maxw = 0;
  for (int l = 0; l <= net->L; ++l) maxw = std::max(maxw, net->dims[l]);
  if (maxw > rd::kPredW || M > 65535) return fail(ctx, REACH_E_UNSUPPORTED, "pred_loss: shape outside the kernel");
  rd::PredArgs A{};
  A.poff[0] = 0;
  for (int l = 0; l < net->L; ++l)
    A.poff[l + 1] = A.poff[l] + static_cast<long long>(net->dims[l + 1]) * net->dims[l] + net->dims[l + 1];
  const long long P = grad ? A.poff[net->L] : 1;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align_up(off + std::max<size_t>(bytes, 8), 256);
    return o;
  };
  const size_t ns = static_cast<size_t>(M) * (Ls + 1) * n, na = static_cast<size_t>(M) * Ls * m,
               nt = static_cast<size_t>(P) * M * T;
  const size_t o_s = take(ns * 8), o_a = take(na * 8), o_w = take(static_cast<size_t>(T) * 8), o_v = take(nt * 8),
               o_d = take(nt * 8);
  int rc = ensure_ws(ctx, off);
  if (rc) return rc;
  char* w = static_cast<char*>(ctx->ws);
  auto Dp = [&](size_t o) { return reinterpret_cast<double*>(w + o); };
  RB_CUDA(cudaMemcpyAsync(Dp(o_s), b->states, ns * 8, cudaMemcpyHostToDevice, ctx->stream));
  if (na) RB_CUDA(cudaMemcpyAsync(Dp(o_a), b->actions, na * 8, cudaMemcpyHostToDevice, ctx->stream));
  RB_CUDA(cudaMemcpyAsync(Dp(o_w), weights, static_cast<size_t>(T) * 8, cudaMemcpyHostToDevice, ctx->stream));
  A.net = net->dev;
  A.n = n;
  A.m = m;
  A.T = T;
  A.M = M;
  A.seeded = grad ? 1 : 0;
  A.states = Dp(o_s);
  A.actions = Dp(o_a);
  A.ls = Ls;
  A.weights = Dp(o_w);
  A.term_v = Dp(o_v);
  A.term_d = Dp(o_d);
  cudaEvent_t stop;
  rc = timed_begin(ctx, &stop);
  if (rc) return rc;
  rd::pred_loss_grad_kernel<<<dim3(static_cast<unsigned>(P), static_cast<unsigned>(M)), rd::kPredThreads, 0,
                              ctx->stream>>>(A);
  RB_CUDA(cudaGetLastError());
  rc = timed_end(ctx, stop);
  if (rc) return rc;
  ctx->launches += 1;
  std::vector<double> tv(nt), td(nt);
  RB_CUDA(cudaMemcpyAsync(tv.data(), Dp(o_v), nt * 8, cudaMemcpyDeviceToHost, ctx->stream));
  RB_CUDA(cudaMemcpyAsync(td.data(), Dp(o_d), nt * 8, cudaMemcpyDeviceToHost, ctx->stream));
  RB_CUDA(cudaStreamSynchronize(ctx->stream));
  // acc += term in (episode, step) order, then acc / S(M * T_h) (Dual division, scalar.hpp:22-28)
  const double q = static_cast<double>(M) * T;
  for (long long p = 0; p < P; ++p) {
    double av = 0.0, ad = 0.0;
    const size_t base = static_cast<size_t>(p) * M * T;
    for (size_t k = 0; k < static_cast<size_t>(M) * T; ++k) {
      av = av + tv[base + k];
      ad = ad + td[base + k];
    }
    if (p == 0) *loss = av / q;
    if (grad) grad[p] = (ad * q - av * 0.0) / (q * q);
  }
  return REACH_OK;
}

// track_loss (training.hpp:134-178) with the quadrotor plant and, optionally, its grad_forward.
int reach_track_loss(reach_ctx* ctx, const reach_net* ctl, int32_t plant, const double* plant_params,
                     const reach_episode_set* b, int32_t t_t, const double* weights, double gamma, double delta,
                     int32_t rk4_substeps, double cap, double* loss, double* grad, int32_t* blowup_count) {
  rbh::DeviceGuard device_guard_(ctx);
  namespace rd = rb::dual;
  if (!ctx || !ctl || !b || !loss || !plant_params) return REACH_E_INVALID_ARGUMENT;
  if (b->episodes < 1 || t_t < 1 || !weights || delta <= 0.0 || rk4_substeps < 1)
    return fail(ctx, REACH_E_INVALID_ARGUMENT, "track_loss: bad configuration");
  if (b->length < t_t) return fail(ctx, REACH_E_INVALID_ARGUMENT, "track_loss: episode shorter than T_t");
  if (plant != REACH_PLANT_QUADROTOR) return fail(ctx, REACH_E_UNSUPPORTED, "track_loss: unknown plant");
  const int n = b->n, l = b->m, r = b->y_ref ? b->ref_dim : 0, M = b->episodes, T = t_t, Ls = b->length;
  if (n != 12 || l < 4 || !b->states || !b->actions)
    return fail(ctx, REACH_E_INVALID_ARGUMENT, "track_loss: quadrotor episodes need n = 12, >= 4 controls");
  if (ctl->dims[0] != n + r || ctl->dims[ctl->L] != l)
    return fail(ctx, REACH_E_INVALID_ARGUMENT, "track_loss: controller shape does not match the episodes");
  int maxw = 0;
  for (int q = 0; q <= ctl->L; ++q) maxw = std::max(maxw, ctl->dims[q]);
  if (maxw > rd::kPredW || l > 8 || M > 65535) return fail(ctx, REACH_E_UNSUPPORTED, "track_loss: shape outside the kernel");
  rd::TrackArgs A{};
  A.poff[0] = 0;
  for (int q = 0; q < ctl->L; ++q)
    A.poff[q + 1] = A.poff[q] + static_cast<long long>(ctl->dims[q + 1]) * ctl->dims[q] + ctl->dims[q + 1];
  const long long P = grad ? A.poff[ctl->L] : 1;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align_up(off + std::max<size_t>(bytes, 8), 256);
    return o;
  };
  const size_t ns = static_cast<size_t>(M) * (Ls + 1) * n, na = static_cast<size_t>(M) * Ls * l,
               nr = static_cast<size_t>(M) * Ls * r, ne = static_cast<size_t>(P) * M;
  const size_t o_s = take(ns * 8), o_a = take(na * 8), o_r = take(nr * 8), o_w = take(static_cast<size_t>(T) * 8),
               o_v = take(ne * 8), o_d = take(ne * 8), o_b = take(static_cast<size_t>(M) * 4);
  int rc = ensure_ws(ctx, off);
  if (rc) return rc;
  char* w = static_cast<char*>(ctx->ws);
  auto Dp = [&](size_t o) { return reinterpret_cast<double*>(w + o); };
  RB_CUDA(cudaMemcpyAsync(Dp(o_s), b->states, ns * 8, cudaMemcpyHostToDevice, ctx->stream));
  RB_CUDA(cudaMemcpyAsync(Dp(o_a), b->actions, na * 8, cudaMemcpyHostToDevice, ctx->stream));
  if (nr) RB_CUDA(cudaMemcpyAsync(Dp(o_r), b->y_ref, nr * 8, cudaMemcpyHostToDevice, ctx->stream));
  RB_CUDA(cudaMemcpyAsync(Dp(o_w), weights, static_cast<size_t>(T) * 8, cudaMemcpyHostToDevice, ctx->stream));
  A.net = ctl->dev;
  A.n = n;
  A.l = l;
  A.r = r;
  A.T = T;
  A.M = M;
  A.seeded = grad ? 1 : 0;
  A.rk4 = rk4_substeps;
  for (int i = 0; i < 5; ++i) A.prm[i] = plant_params[i];
  A.gamma = gamma;
  A.delta = delta;
  A.cap = cap;
  A.states = Dp(o_s);
  A.actions = Dp(o_a);
  A.y_ref = nr ? Dp(o_r) : nullptr;
  A.ls = Ls;
  A.weights = Dp(o_w);
  A.ep_v = Dp(o_v);
  A.ep_d = Dp(o_d);
  A.blown = reinterpret_cast<int*>(w + o_b);
  cudaEvent_t stop;
  rc = timed_begin(ctx, &stop);
  if (rc) return rc;
  rd::track_loss_grad_kernel<<<dim3(static_cast<unsigned>(P), static_cast<unsigned>(M)), rd::kPredThreads, 0,
                               ctx->stream>>>(A);
  RB_CUDA(cudaGetLastError());
  rc = timed_end(ctx, stop);
  if (rc) return rc;
  ctx->launches += 1;
  std::vector<double> tv(ne), td(ne);
  std::vector<int32_t> bl(M);
  RB_CUDA(cudaMemcpyAsync(tv.data(), Dp(o_v), ne * 8, cudaMemcpyDeviceToHost, ctx->stream));
  RB_CUDA(cudaMemcpyAsync(td.data(), Dp(o_d), ne * 8, cudaMemcpyDeviceToHost, ctx->stream));
  RB_CUDA(cudaMemcpyAsync(bl.data(), w + o_b, static_cast<size_t>(M) * 4, cudaMemcpyDeviceToHost, ctx->stream));
  RB_CUDA(cudaStreamSynchronize(ctx->stream));
  const double q = static_cast<double>(M) * T;  // acc / S(M' T_t)
  for (long long p = 0; p < P; ++p) {
    double av = 0.0, ad = 0.0;
    for (int e = 0; e < M; ++e) {
      av = av + tv[static_cast<size_t>(p) * M + e];
      ad = ad + td[static_cast<size_t>(p) * M + e];
    }
    if (p == 0) *loss = av / q;
    if (grad) grad[p] = (ad * q - av * 0.0) / (q * q);
  }
  if (blowup_count) {
    int c = 0;
    for (int e = 0; e < M; ++e) c += bl[e];
    *blowup_count = c;
  }
  return REACH_OK;
}

// ctl_reach_loss (training.hpp:183-213) with the quadrotor plant: value and, optionally, its grad_forward
// over the controller's parameters -- one Dual cl_reach per (parameter, episode) (ct_dual.cuh).
int reach_ctl_reach_loss(reach_ctx* ctx, const reach_net* ctl, const reach_cl_spec* sp, int32_t episodes,
                         const double* x0s, const double* y_refs, double eps, double cap, double* loss, double* grad,
                         int32_t* diverged_count) {
  rbh::DeviceGuard device_guard_(ctx);
  namespace cd = rb::ctd;
  if (!ctx || !ctl || !sp || !x0s || !loss) return REACH_E_INVALID_ARGUMENT;
  if (episodes < 1 || sp->ctl_steps < 1) return fail(ctx, REACH_E_INVALID_ARGUMENT, "ctl_reach_loss: bad batch/horizon");
  if (sp->plant != REACH_PLANT_QUADROTOR || sp->n != 12 || sp->l != 4)
    return fail(ctx, REACH_E_UNSUPPORTED, "ctl_reach_loss: the quadrotor plant (n = 12, l = 4) only");
  if (eps < 0.0) return fail(ctx, REACH_E_INVALID_ARGUMENT, "box_from_center: negative radius");
  const int n = sp->n, l = sp->l, na = n + l, M = episodes, r = sp->ref_dim;
  if (ctl->dims[0] != n + r || ctl->dims[ctl->L] != l)
    return fail(ctx, REACH_E_INVALID_ARGUMENT, "ClosedLoopSpec: controller input dim mismatch");
  if (r > 0 && !y_refs) return fail(ctx, REACH_E_INVALID_ARGUMENT, "ctl_reach_loss: missing reference sequences");
  if (sp->k_atomic < 1 || !(sp->fp.h > 0.0) || sp->fp.order < 1)
    return fail(ctx, REACH_E_INVALID_ARGUMENT, "ClosedLoopSpec: invalid flowpipe parameters");
  const int cap_q = sp->fp.window > 0 ? sp->fp.window : 1;
  int maxw = 0;
  for (int q = 1; q < ctl->L; ++q) maxw = std::max(maxw, ctl->dims[q]);
  if (na > cd::MR || n + (cap_q + 1) * na > cd::MZ || maxw > cd::CW || l > cd::CO || M > 65535 ||
      n + (cap_q + 1) * na + n > cd::CA)
    return fail(ctx, REACH_E_UNSUPPORTED, "ctl_reach_loss: shape outside the Dual CT kernel");
  cd::CtlLossArgs A{};
  A.poff[0] = 0;
  for (int q = 0; q < ctl->L; ++q)
    A.poff[q + 1] = A.poff[q] + static_cast<long long>(ctl->dims[q + 1]) * ctl->dims[q] + ctl->dims[q + 1];
  const long long P = grad ? A.poff[ctl->L] : 1;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align_up(off + std::max<size_t>(bytes, 8), 256);
    return o;
  };
  const size_t nyr = static_cast<size_t>(M) * sp->ctl_steps * std::max(r, 0);
  const size_t o_x = take(static_cast<size_t>(M) * n * 8), o_y = take(nyr * 8),
               o_v = take(static_cast<size_t>(P) * M * 8), o_d = take(static_cast<size_t>(P) * M * 8),
               o_dv = take(static_cast<size_t>(M) * 4);
  int rc = ensure_ws(ctx, off);
  if (rc) return rc;
  char* w = static_cast<char*>(ctx->ws);
  auto Dp = [&](size_t o) { return reinterpret_cast<double*>(w + o); };
  RB_CUDA(cudaMemcpyAsync(Dp(o_x), x0s, static_cast<size_t>(M) * n * 8, cudaMemcpyHostToDevice, ctx->stream));
  if (nyr) RB_CUDA(cudaMemcpyAsync(Dp(o_y), y_refs, nyr * 8, cudaMemcpyHostToDevice, ctx->stream));
  A.net = ctl->dev;
  A.n = n;
  A.l = l;
  A.rdim = r;
  A.ctl_steps = sp->ctl_steps;
  A.k_atomic = sp->k_atomic;
  A.intervalize = sp->intervalize_boundary;
  A.M = M;
  A.seeded = grad ? 1 : 0;
  for (int i = 0; i < 5; ++i) A.prm[i] = sp->plant_params[i];
  A.F = cd::FlowCfg{sp->fp.h, sp->fp.eps_init, sp->fp.enlargement, sp->fp.order, sp->fp.refine_rounds,
                    sp->fp.max_enlargements, sp->fp.window};
  A.eps = eps;
  A.cap = cap;
  A.x0 = Dp(o_x);
  A.yref = nyr ? Dp(o_y) : nullptr;
  A.term_v = Dp(o_v);
  A.term_d = Dp(o_d);
  A.diverged = reinterpret_cast<int*>(w + o_dv);
  const size_t smem = sizeof(cd::Work);
  // RB_CTD_SLOTS_PER_SM > 0: the working sets in global memory, that many persistent passes per SM
  const int slots_per_sm = env_int("RB_CTD_SLOTS_PER_SM", 12, 0, 64);
  cudaEvent_t stop;
  if (slots_per_sm > 0) {
    const long long total = P * M;
    const int grid = static_cast<int>(std::min<long long>(total, static_cast<long long>(slots_per_sm) * ctx->num_sms));
    const size_t need = static_cast<size_t>(grid) * sizeof(cd::Work);
    if (need > ctx->ctd_bytes) {
      if (ctx->ctd_ws) {
        cudaStreamSynchronize(ctx->stream);
        cudaFree(ctx->ctd_ws);
        ctx->ctd_ws = nullptr;
        ctx->ctd_bytes = 0;
      }
      RB_CUDA(cudaMalloc(&ctx->ctd_ws, need));
      ctx->ctd_bytes = need;
    }
    rc = timed_begin(ctx, &stop);
    if (rc) return rc;
    cd::ctl_reach_loss_grad_kernel_g<<<grid, 32, 0, ctx->stream>>>(A, static_cast<cd::Work*>(ctx->ctd_ws), total);
    RB_CUDA(cudaGetLastError());
  } else {
    if (smem > static_cast<size_t>(ctx->max_smem))
      return fail(ctx, REACH_E_UNSUPPORTED, "ctl_reach_loss: Dual working set exceeds shared memory");
    RB_CUDA(cudaFuncSetAttribute(cd::ctl_reach_loss_grad_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem)));
    rc = timed_begin(ctx, &stop);
    if (rc) return rc;
    cd::ctl_reach_loss_grad_kernel<<<dim3(static_cast<unsigned>(P), static_cast<unsigned>(M)), 32, smem,
                                     ctx->stream>>>(A);
    RB_CUDA(cudaGetLastError());
  }
  rc = timed_end(ctx, stop);
  if (rc) return rc;
  ctx->launches += 1;
  std::vector<double> tv(static_cast<size_t>(P) * M), td(tv.size());
  std::vector<int32_t> dv(M);
  RB_CUDA(cudaMemcpyAsync(tv.data(), Dp(o_v), tv.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
  RB_CUDA(cudaMemcpyAsync(td.data(), Dp(o_d), td.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
  RB_CUDA(cudaMemcpyAsync(dv.data(), w + o_dv, static_cast<size_t>(M) * 4, cudaMemcpyDeviceToHost, ctx->stream));
  RB_CUDA(cudaStreamSynchronize(ctx->stream));
  const double Md = static_cast<double>(M);  // acc / S(batch.size())
  for (long long p = 0; p < P; ++p) {
    double av = 0.0, ad = 0.0;
    for (int e = 0; e < M; ++e) {
      av = av + tv[static_cast<size_t>(p) * M + e];
      ad = ad + td[static_cast<size_t>(p) * M + e];
    }
    if (p == 0) *loss = av / Md;
    if (grad) grad[p] = (ad * Md - av * 0.0) / (Md * Md);
  }
  if (diverged_count) {
    int c = 0;
    for (int e = 0; e < M; ++e) c += dv[e];
    *diverged_count = c;
  }
  return REACH_OK;
}

// train_dt_dyn (training.hpp:333-382) with every loss and gradient on the device.
int reach_train_dt_dyn(reach_ctx* ctx, const reach_net_desc* init, const reach_train_config* cfg,
                       const reach_episode_set* ds, double* params_out, reach_train_log_row* log) {
  rbh::DeviceGuard device_guard_(ctx);
  if (!ctx || !init || !cfg || !ds || !params_out) return REACH_E_INVALID_ARGUMENT;
  const reach_train_config& c = *cfg;
  if (c.horizon_max < 1 || c.eps0 < c.eps_final || c.eps_final < 0.0 || c.lambda < 0.0 || c.gamma < 0.0 ||
      c.iters < 1 || c.batch < 1 || c.lr <= 0.0 || c.reach_cap <= 0.0)
    return fail(ctx, REACH_E_INVALID_ARGUMENT, "TrainConfig: invalid configuration");
  if (ds->episodes < 1) return fail(ctx, REACH_E_INVALID_ARGUMENT, "train_dt_dyn: empty dataset");
  if (ds->length < c.horizon_max) return fail(ctx, REACH_E_INVALID_ARGUMENT, "train_dt_dyn: episode shorter than T_h^max");
  const int n = ds->n, m = ds->m, L = init->n_layers, E = ds->episodes, Ls = ds->length;
  size_t np = 0;
  for (int l = 0; l < L; ++l) np += static_cast<size_t>(init->dims[l + 1]) * (init->dims[l] + 1);
  std::vector<double> params(init->params, init->params + np);
  std::vector<int32_t> dims(init->dims, init->dims + L + 1), acts(init->acts, init->acts + L);
  // Adam (training.hpp:239-260)
  const double beta1 = 0.9, beta2 = 0.999, aeps = 1e-8;
  std::vector<double> am(np, 0.0), av(np, 0.0);
  int at = 0;
  std::mt19937_64 gen(c.seed);  // Rng(cfg.seed) (rng.hpp:13-15); sample_batch draws uniform_int
  constexpr double kE = 2.718281828459045235360287471352662498;  // std::numbers::e
  std::vector<double> bs(static_cast<size_t>(c.batch) * (c.horizon_max + 1) * n),
      ba(static_cast<size_t>(c.batch) * c.horizon_max * std::max(m, 0)), x0s(static_cast<size_t>(c.batch) * n);
  std::vector<double> gp(np), gr(np), g(np);
  for (int s = 0; s < c.iters; ++s) {
    int t_h = c.horizon_max;
    double eps = c.eps_final;
    if (c.curriculum) {  // horizon_schedule / eps_schedule (training.hpp:219-236)
      if (c.iters <= 1) {
        t_h = c.horizon_max;
        eps = c.eps_final;
      } else {
        const double u = std::log(1.0 + static_cast<double>(s) * (kE - 1.0) / (c.iters - 1));
        t_h = std::min(std::max(1, static_cast<int>(std::llround(c.horizon_max * u))), c.horizon_max);
        eps = c.eps_final + (c.eps0 - c.eps_final) * (1.0 - static_cast<double>(s) / (c.iters - 1));
      }
    }
    // detail::sample_batch (training.hpp:305-314): the first t_h steps of each drawn episode
    const int Tm = c.horizon_max;
    for (int b = 0; b < c.batch; ++b) {
      const int e = static_cast<int>(gen() % static_cast<uint64_t>(E));
      std::memcpy(bs.data() + static_cast<size_t>(b) * (Tm + 1) * n, ds->states + static_cast<size_t>(e) * (Ls + 1) * n,
                  sizeof(double) * (Tm + 1) * n);
      if (m > 0)
        std::memcpy(ba.data() + static_cast<size_t>(b) * Tm * m, ds->actions + static_cast<size_t>(e) * Ls * m,
                    sizeof(double) * Tm * m);
      std::memcpy(x0s.data() + static_cast<size_t>(b) * n, ds->states + static_cast<size_t>(e) * (Ls + 1) * n,
                  sizeof(double) * n);
    }
    std::vector<double> wts(static_cast<size_t>(t_h));  // horizon_weights (training.hpp:48-53)
    for (int t = 0; t < t_h; ++t) wts[static_cast<size_t>(t)] = 1.0 + static_cast<double>(t + 1) / t_h;
    reach_net_desc d{L, dims.data(), acts.data(), params.data()};
    reach_net* cur = nullptr;
    int rc = reach_net_upload(ctx, &d, &cur);
    if (rc) return rc;
    std::unique_ptr<reach_net, std::function<void(reach_net*)>> guard(cur, [ctx](reach_net* p) { reach_net_free(ctx, p); });
    reach_episode_set bset{c.batch, Tm, n, m, bs.data(), ba.data()};
    double lp = 0.0, lr_ = 0.0;
    int div = 0;
    rc = reach_pred_loss(ctx, cur, &bset, t_h, wts.data(), &lp, gp.data());
    if (rc) return rc;
    if (c.lambda > 0.0) {
      reach_dt_args a{};
      a.batch = c.batch;
      a.horizon = t_h;
      a.n = n;
      a.m = m;
      a.window = c.window;
      a.rebuild_from_box = c.rebuild_from_box;
      std::vector<double> acts_th(static_cast<size_t>(c.batch) * t_h * std::max(m, 0));
      for (int b = 0; b < c.batch && m > 0; ++b)
        std::memcpy(acts_th.data() + static_cast<size_t>(b) * t_h * m, ba.data() + static_cast<size_t>(b) * Tm * m,
                    sizeof(double) * t_h * m);
      a.x0_lo = x0s.data();
      a.x0_hi = x0s.data();
      a.actions = m > 0 ? acts_th.data() : nullptr;
      rc = reach_reach_loss(ctx, cur, &a, c.batch, eps, c.reach_cap, &lr_, gr.data(), &div);
      if (rc) return rc;
    }
    const double lt = lp + c.lambda * lr_;
    if (log) log[s] = reach_train_log_row{s, t_h, eps, lp, lr_, lt, div};
    if (!std::isfinite(lt)) {
      char msg[256];
      std::snprintf(msg, sizeof msg, "train_dt_dyn: non-finite loss at iter %d", s);
      return fail(ctx, REACH_E_NONFINITE, msg);
    }
    // grad_forward of pred_loss + S(lambda) reach_loss: per direction the Dual sum of the two parts
    for (size_t j = 0; j < np; ++j) {
      double dv = gp[j];
      if (c.lambda > 0.0) {
        const double rv = lr_, rdv = gr[j];
        if (!std::isfinite(rv) || !std::isfinite(rdv))
          return fail(ctx, REACH_E_NONFINITE, "grad_forward: non-finite derivative");
        dv = dv + (0.0 * rv + c.lambda * rdv);  // dmul(S(lambda), r).d, then dadd
      }
      if (!std::isfinite(dv)) return fail(ctx, REACH_E_NONFINITE, "grad_forward: non-finite derivative");
      g[j] = dv;
    }
    ++at;  // Adam::step
    const double bc1 = 1.0 - std::pow(beta1, at), bc2 = 1.0 - std::pow(beta2, at);
    for (size_t j = 0; j < np; ++j) {
      am[j] = beta1 * am[j] + (1.0 - beta1) * g[j];
      av[j] = beta2 * av[j] + (1.0 - beta2) * g[j] * g[j];
      params[j] -= c.lr * (am[j] / bc1) / (std::sqrt(av[j] / bc2) + aeps);
    }
  }
  std::memcpy(params_out, params.data(), sizeof(double) * np);
  return REACH_OK;
}

// train_ct_ctl (training.hpp:389-442) with the quadrotor plant: L = track_loss + lambda ctl_reach_loss, the
// same curriculum / minibatch stream / Adam as train_dt_dyn; every loss and gradient on the device.
int reach_train_ct_ctl(reach_ctx* ctx, const reach_net_desc* init, const reach_train_config* cfg,
                       const reach_episode_set* ds, const reach_cl_spec* base, double delta, int32_t rk4_substeps,
                       double* params_out, reach_train_log_row* log) {
  rbh::DeviceGuard device_guard_(ctx);
  if (!ctx || !init || !cfg || !ds || !base || !params_out) return REACH_E_INVALID_ARGUMENT;
  const reach_train_config& c = *cfg;
  if (c.horizon_max < 1 || c.eps0 < c.eps_final || c.eps_final < 0.0 || c.lambda < 0.0 || c.gamma < 0.0 ||
      c.iters < 1 || c.batch < 1 || c.lr <= 0.0 || c.reach_cap <= 0.0)
    return fail(ctx, REACH_E_INVALID_ARGUMENT, "TrainConfig: invalid configuration");
  if (ds->episodes < 1) return fail(ctx, REACH_E_INVALID_ARGUMENT, "train_ct_ctl: empty dataset");
  if (ds->length < c.horizon_max) return fail(ctx, REACH_E_INVALID_ARGUMENT, "train_ct_ctl: episode shorter than T_h^max");
  const int n = ds->n, l = ds->m, L = init->n_layers, E = ds->episodes, Ls = ds->length;
  const int r = ds->y_ref ? ds->ref_dim : 0;
  size_t np = 0;
  for (int q = 0; q < L; ++q) np += static_cast<size_t>(init->dims[q + 1]) * (init->dims[q] + 1);
  std::vector<double> params(init->params, init->params + np);
  std::vector<int32_t> dims(init->dims, init->dims + L + 1), acts(init->acts, init->acts + L);
  const double beta1 = 0.9, beta2 = 0.999, aeps = 1e-8;
  std::vector<double> am(np, 0.0), av(np, 0.0);
  int at = 0;
  std::mt19937_64 gen(c.seed);
  constexpr double kE = 2.718281828459045235360287471352662498;
  const int Tm = c.horizon_max;
  std::vector<double> bs(static_cast<size_t>(c.batch) * (Tm + 1) * n), ba(static_cast<size_t>(c.batch) * Tm * l),
      br(static_cast<size_t>(c.batch) * Tm * std::max(r, 1)), x0s(static_cast<size_t>(c.batch) * n);
  std::vector<double> gt(np), gr(np), g(np);
  for (int s = 0; s < c.iters; ++s) {
    int t_h = c.horizon_max;
    double eps = c.eps_final;
    if (c.curriculum && c.iters > 1) {
      const double u = std::log(1.0 + static_cast<double>(s) * (kE - 1.0) / (c.iters - 1));
      t_h = std::min(std::max(1, static_cast<int>(std::llround(c.horizon_max * u))), c.horizon_max);
      eps = c.eps_final + (c.eps0 - c.eps_final) * (1.0 - static_cast<double>(s) / (c.iters - 1));
    }
    for (int b = 0; b < c.batch; ++b) {
      const int e = static_cast<int>(gen() % static_cast<uint64_t>(E));
      std::memcpy(bs.data() + static_cast<size_t>(b) * (Tm + 1) * n, ds->states + static_cast<size_t>(e) * (Ls + 1) * n,
                  sizeof(double) * (Tm + 1) * n);
      std::memcpy(ba.data() + static_cast<size_t>(b) * Tm * l, ds->actions + static_cast<size_t>(e) * Ls * l,
                  sizeof(double) * Tm * l);
      if (r > 0)
        std::memcpy(br.data() + static_cast<size_t>(b) * Tm * r, ds->y_ref + static_cast<size_t>(e) * Ls * r,
                    sizeof(double) * Tm * r);
      std::memcpy(x0s.data() + static_cast<size_t>(b) * n, ds->states + static_cast<size_t>(e) * (Ls + 1) * n,
                  sizeof(double) * n);
    }
    std::vector<double> wts(static_cast<size_t>(t_h));
    for (int t = 0; t < t_h; ++t) wts[static_cast<size_t>(t)] = 1.0 + static_cast<double>(t + 1) / t_h;
    reach_net_desc d{L, dims.data(), acts.data(), params.data()};
    reach_net* cur = nullptr;
    int rc = reach_net_upload(ctx, &d, &cur);
    if (rc) return rc;
    std::unique_ptr<reach_net, std::function<void(reach_net*)>> guard(cur, [ctx](reach_net* p) { reach_net_free(ctx, p); });
    reach_episode_set bset{c.batch, Tm, n, l, bs.data(), ba.data(), r, r > 0 ? br.data() : nullptr};
    double ltr = 0.0, lr_ = 0.0;
    int div = 0;
    rc = reach_track_loss(ctx, cur, base->plant, base->plant_params, &bset, t_h, wts.data(), c.gamma, delta,
                          rk4_substeps, 1e6, &ltr, gt.data(), nullptr);
    if (rc) return rc;
    if (c.lambda > 0.0) {
      reach_cl_spec sp = *base;
      sp.n = n;
      sp.l = l;
      sp.ctl_steps = t_h;
      sp.ref_dim = r;
      sp.y_ref = nullptr;
      sp.fp.h = delta / base->k_atomic;
      std::vector<double> yr(static_cast<size_t>(c.batch) * t_h * std::max(r, 1));
      for (int b = 0; b < c.batch && r > 0; ++b)
        std::memcpy(yr.data() + static_cast<size_t>(b) * t_h * r, br.data() + static_cast<size_t>(b) * Tm * r,
                    sizeof(double) * t_h * r);
      rc = reach_ctl_reach_loss(ctx, cur, &sp, c.batch, x0s.data(), r > 0 ? yr.data() : nullptr, eps, c.reach_cap,
                                &lr_, gr.data(), &div);
      if (rc) return rc;
    }
    const double lt = ltr + c.lambda * lr_;
    if (log) log[s] = reach_train_log_row{s, t_h, eps, ltr, lr_, lt, div};
    if (!std::isfinite(lt)) {
      char msg[256];
      std::snprintf(msg, sizeof msg, "train_ct_ctl: non-finite loss at iter %d", s);
      return fail(ctx, REACH_E_NONFINITE, msg);
    }
    for (size_t j = 0; j < np; ++j) {
      double dv = gt[j];
      if (c.lambda > 0.0) dv = dv + (0.0 * lr_ + c.lambda * gr[j]);
      if (!std::isfinite(dv)) return fail(ctx, REACH_E_NONFINITE, "grad_forward: non-finite derivative");
      g[j] = dv;
    }
    ++at;
    const double bc1 = 1.0 - std::pow(beta1, at), bc2 = 1.0 - std::pow(beta2, at);
    for (size_t j = 0; j < np; ++j) {
      am[j] = beta1 * am[j] + (1.0 - beta1) * g[j];
      av[j] = beta2 * av[j] + (1.0 - beta2) * g[j] * g[j];
      params[j] -= c.lr * (am[j] / bc1) / (std::sqrt(av[j] / bc2) + aeps);
    }
  }
  std::memcpy(params_out, params.data(), sizeof(double) * np);
  return REACH_OK;
}

// The refinement step of plan_cem alone (mpc.hpp:337-361), for drivers that run the CEM loop in pieces.
int reach_plan_refine(reach_ctx* ctx, const reach_net* net, const reach_plan_problem* prob, const double* x0,
                      int32_t refine_iters, double best_objective, double* best_actions, int32_t* refined) {
  rbh::DeviceGuard device_guard_(ctx);
  if (!ctx || !net || !prob || !x0 || !best_actions) return REACH_E_INVALID_ARGUMENT;
  if (refine_iters < 0) return fail(ctx, REACH_E_INVALID_ARGUMENT, "SamplerConfig: invalid configuration");
  int rc = validate_problem(ctx, net, prob);
  if (rc) return rc;
  if (refined) *refined = 0;
  if (refine_iters == 0 || !std::isfinite(best_objective)) return REACH_OK;
  return plan_refine_impl(ctx, net, prob, x0, refine_iters, best_objective, best_actions, refined);
}

// dt_interval_baseline (dt_reach.hpp:129-149) for a batch: the naive interval tube of the same map.
int reach_dt_interval_baseline_batch(reach_ctx* ctx, const reach_net* net, const reach_dt_args* a,
                                     const reach_tube_out* out) {
  rbh::DeviceGuard device_guard_(ctx);
  if (!ctx || !net || !a || !out) return REACH_E_INVALID_ARGUMENT;
  if (a->batch < 0 || a->horizon < 0) return fail(ctx, REACH_E_INVALID_ARGUMENT, "dt_reach_batch: negative size");
  int rc = validate_system(ctx, net, a->n, a->m);
  if (rc) return rc;
  if (a->batch == 0) return REACH_OK;
  const size_t B = a->batch, H = a->horizon, n = a->n, m = a->m;
  int maxw = 0;
  for (int l = 0; l <= net->L; ++l) maxw = std::max(maxw, net->dims[l]);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align_up(off + std::max<size_t>(bytes, 8), 256);
    return o;
  };
  const size_t act_bytes = (a->actions_shared ? 1 : B) * H * m * 8, box_bytes = B * (H + 1) * n * 8;
  const size_t o_xl = take(B * n * 8), o_xh = take(B * n * 8), o_a = take(act_bytes), o_ol = take(box_bytes),
               o_oh = take(box_bytes), o_nb = take(B * 4), o_fs = take(B * 4), o_st = take(B * 4);
  rc = ensure_ws(ctx, off);
  if (rc) return rc;
  char* w = static_cast<char*>(ctx->ws);
  auto Dp = [&](size_t o) { return reinterpret_cast<double*>(w + o); };
  RB_CUDA(cudaMemcpyAsync(Dp(o_xl), a->x0_lo, B * n * 8, cudaMemcpyHostToDevice, ctx->stream));
  RB_CUDA(cudaMemcpyAsync(Dp(o_xh), a->x0_hi, B * n * 8, cudaMemcpyHostToDevice, ctx->stream));
  if (act_bytes) RB_CUDA(cudaMemcpyAsync(Dp(o_a), a->actions, act_bytes, cudaMemcpyHostToDevice, ctx->stream));
  rb::IBLArgs A{};
  A.net = net->dev;
  A.B = static_cast<int>(B);
  A.H = static_cast<int>(H);
  A.n = static_cast<int>(n);
  A.m = static_cast<int>(m);
  A.maxw = maxw;
  A.x0_lo = Dp(o_xl);
  A.x0_hi = Dp(o_xh);
  A.actions = Dp(o_a);
  A.actions_shared = a->actions_shared;
  A.out_lo = Dp(o_ol);
  A.out_hi = Dp(o_oh);
  A.n_boxes = reinterpret_cast<int*>(w + o_nb);
  A.failed_step = reinterpret_cast<int*>(w + o_fs);
  A.status = reinterpret_cast<int*>(w + o_st);
  const size_t smem = static_cast<size_t>(rb::kIblWarps) * 5 * maxw * sizeof(double);
  RB_CUDA(cudaFuncSetAttribute(rb::interval_baseline_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(smem)));
  cudaEvent_t stop;
  rc = timed_begin(ctx, &stop);
  if (rc) return rc;
  rb::interval_baseline_kernel<<<static_cast<unsigned>((B + rb::kIblWarps - 1) / rb::kIblWarps),
                                 rb::kIblWarps * 32, smem, ctx->stream>>>(A);
  RB_CUDA(cudaGetLastError());
  rc = timed_end(ctx, stop);
  if (rc) return rc;
  ctx->launches += 1;
  RB_CUDA(cudaMemcpyAsync(out->lo, Dp(o_ol), box_bytes, cudaMemcpyDeviceToHost, ctx->stream));
  RB_CUDA(cudaMemcpyAsync(out->hi, Dp(o_oh), box_bytes, cudaMemcpyDeviceToHost, ctx->stream));
  RB_CUDA(cudaMemcpyAsync(out->n_boxes, w + o_nb, B * 4, cudaMemcpyDeviceToHost, ctx->stream));
  RB_CUDA(cudaMemcpyAsync(out->failed_step, w + o_fs, B * 4, cudaMemcpyDeviceToHost, ctx->stream));
  RB_CUDA(cudaMemcpyAsync(out->status, w + o_st, B * 4, cudaMemcpyDeviceToHost, ctx->stream));
  RB_CUDA(cudaStreamSynchronize(ctx->stream));
  return REACH_OK;
}

}  // extern "C"
