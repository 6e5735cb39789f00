// C ABI of the B200 reachability library (include/reach_b200.h).
//
// Host side: context (device, stream, workspaces), immutable network upload
// (weights laid out once for the kernels: W row-major and W^T, 16-byte padded
// rows, one blob), argument validation with the reference's error behaviour,
// and the launches.  No CPU fallback: every entry point runs the CUDA kernels
// or returns an error.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/reach_b200.h"
#include "diag.cuh"
#include "dt_kernel.cuh"

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
};

namespace {

int fail(reach_ctx* ctx, int code, const std::string& msg) {
  if (ctx) ctx->err = msg;
  return code;
}

int cuda_fail(reach_ctx* ctx, cudaError_t e, const char* where) {
  return fail(ctx, e == cudaErrorMemoryAllocation ? REACH_E_OOM : REACH_E_CUDA,
              std::string(where) + ": " + cudaGetErrorString(e));
}

#define RB_CUDA(call)                                   \
  do {                                                  \
    cudaError_t e_ = (call);                            \
    if (e_ != cudaSuccess) return cuda_fail(ctx, e_, #call); \
  } while (0)

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

int ensure_ws(reach_ctx* ctx, size_t bytes) {
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

int timed_begin(reach_ctx* ctx, cudaEvent_t* stop) {
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

int timed_end(reach_ctx* ctx, cudaEvent_t stop) {
  if (stop) RB_CUDA(cudaEventRecord(stop, ctx->stream));
  return REACH_OK;
}

// Launch geometry and shared-memory carve-up of the DT horizon kernel.
struct DTLayout {
  int spc = 0, no = 0, cpl = 0;
  size_t smem = 0;
};

constexpr int kStageDoublesDefault = 2048;  // 16 KB bulk-copy stages
constexpr int kNStageDefault = 6;

// Weight-stream ring geometry; RB_NSTAGE / RB_STAGE_DOUBLES override it for tuning runs.
int env_int(const char* name, int dflt, int lo, int hi) {
  const char* v = std::getenv(name);
  if (!v) return dflt;
  int x = std::atoi(v);
  return (x < lo || x > hi) ? dflt : x;
}

int cpl_for(int maxh) { return maxh <= 32 ? 1 : maxh <= 64 ? 2 : maxh <= 96 ? 3 : maxh <= 128 ? 4 : maxh <= 256 ? 8 : 0; }

int plan_dt(reach_ctx* ctx, const reach_net* net, int n, int m, int window, rb::DTParams& P, DTLayout& lay) {
  const int L = net->L;
  const int cap = window > 0 ? window : 1;
  const int no = n <= 2 ? 2 : n <= 4 ? 4 : n <= 6 ? 6 : n <= 8 ? 8 : 0;
  if (no == 0) return fail(ctx, REACH_E_UNSUPPORTED, "state dim > 8 not in this kernel family");
  if (net->cpl == 0) return fail(ctx, REACH_E_UNSUPPORTED, "hidden width > 256 not in this kernel family");
  const int hp = net->hp;
  const int nzs = n * (cap + 2);
  if (nzs > 64) return fail(ctx, REACH_E_UNSUPPORTED, "n * (window + 2) > 64 not in this kernel family");
  const int nop = (no + 1) & ~1;
  auto ev = [](int x) { return (x + 1) & ~1; };
  int off = 0;
  P.o_stA = off;
  off += ev(n * nzs);
  P.o_c = off;
  off += ev(n);
  P.o_pre = off;
  off += (L - 1) * 2 * hp;
  P.o_LT = off;  // also the IBP input buffer (2 hp) and the fold scratch (4 n^2 + n)
  off += ev(std::max({nop * std::max(hp, n + m), 2 * hp, 4 * n * n + n}));
  bool tanh_any = false;
  for (int l = 0; l + 1 < L; ++l) tanh_any |= net->acts[l] == REACH_ACT_TANH;
  P.has_tanh = tanh_any ? 1 : 0;
  P.o_R = off;
  if (tanh_any) off += 3 * hp;
  P.o_bf0 = off;
  if (m > 0) off += std::max(hp, ev(n));
  P.o_idx = off;  // per hidden layer two unit bitmasks (active, unstable) + the active-unit list
  off += ev(((L - 1) * 2 * (hp / 32) * 4 + (L - 1) * hp + 7) / 8);
  P.warp_doubles = ev(off);
  P.nzs = nzs;
  P.hp = hp;
  int boff = 0;
  for (int l = 0; l < L; ++l) {
    P.bias_s_off[l] = boff;
    boff += (l + 1 < L) ? hp : ev(net->dims[l + 1]);
  }
  P.bias_doubles = ev(boff);
  const int kStageDoubles = env_int("RB_STAGE_DOUBLES", kStageDoublesDefault, 512, 8192) & ~1;
  const int kNStage = env_int("RB_NSTAGE", kNStageDefault, 2, 8);
  P.stage_doubles = kStageDoubles;
  P.nstage = kNStage;
  // weight-stream chunk table of one DT step (consumption order of the kernel)
  const rb::DevNet& d = net->dev;
  int nc = 0;
  auto add_matrix = [&](long long moff, int rows, int ld) -> bool {
    if (ld > kStageDoubles) return false;
    const int rpc = std::max(1, kStageDoubles / ld);
    for (int r0 = 0; r0 < rows; r0 += rpc) {
      if (nc >= rb::kMaxChunks) return false;
      const int nr = std::min(rpc, rows - r0);
      P.ch_off[nc] = moff + static_cast<long long>(r0) * ld;
      P.ch_bytes[nc] = static_cast<unsigned>(nr) * ld * 8u;
      ++nc;
    }
    return true;
  };
  bool ok = true;
  for (int l = 0; l + 1 < L; ++l) ok = ok && add_matrix(d.wt_off[l], d.dims[l], d.ldt[l]);
  for (int l = L - 1; l >= 0; --l) ok = ok && add_matrix(d.w_off[l], d.dims[l + 1], d.ldw[l]);
  if (!ok) return fail(ctx, REACH_E_UNSUPPORTED, "network too large for the weight stream");
  P.n_chunks_step = nc;
  const size_t fixed = rb::kHeaderBytes + static_cast<size_t>(kNStage) * kStageDoubles * 8 + static_cast<size_t>(P.bias_doubles) * 8;
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
  if (!ctx) return REACH_OK;
  cudaSetDevice(ctx->device);
  if (ctx->ws) cudaFree(ctx->ws);
  for (auto& p : ctx->ev_used) { cudaEventDestroy(p.first); cudaEventDestroy(p.second); }
  for (auto& p : ctx->ev_free) { cudaEventDestroy(p.first); cudaEventDestroy(p.second); }
  if (ctx->own) cudaStreamDestroy(ctx->own);
  delete ctx;
  return REACH_OK;
}

int reach_ctx_set_stream(reach_ctx* ctx, void* s) {
  if (!ctx) return REACH_E_INVALID_ARGUMENT;
  ctx->stream = s ? static_cast<cudaStream_t>(s) : ctx->own;
  return REACH_OK;
}

int reach_ctx_synchronize(reach_ctx* ctx) {
  if (!ctx) return REACH_E_INVALID_ARGUMENT;
  RB_CUDA(cudaStreamSynchronize(ctx->stream));
  return REACH_OK;
}

int reach_ctx_enable_kernel_timing(reach_ctx* ctx, int32_t on) {
  if (!ctx) return REACH_E_INVALID_ARGUMENT;
  ctx->timing = on != 0;
  return REACH_OK;
}

int reach_ctx_kernel_time(reach_ctx* ctx, double* total_ms, int64_t* launches) {
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
  if (!ctx || !out || count <= 0) return REACH_E_INVALID_ARGUMENT;
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
  if (!net) return REACH_OK;
  if (ctx) cudaSetDevice(ctx->device);
  if (net->blob) cudaFree(net->blob);
  delete net;
  return REACH_OK;
}

int reach_dt_batch(reach_ctx* ctx, const reach_net* net, const reach_dt_args* a, const reach_tube_out* out,
                   int32_t flags) {
  if (!ctx || !net || !a || !out) return REACH_E_INVALID_ARGUMENT;
  if (a->batch < 0 || a->horizon < 0) return fail(ctx, REACH_E_INVALID_ARGUMENT, "dt_reach_batch: negative size");
  int rc = validate_system(ctx, net, a->n, a->m);
  if (rc) return rc;
  if (a->batch == 0) return REACH_OK;
  RB_CUDA(cudaSetDevice(ctx->device));
  rb::DTParams P{};
  DTLayout lay;
  rc = plan_dt(ctx, net, a->n, a->m, a->window, P, lay);
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
    RB_CUDA(cudaMemcpyAsync(const_cast<double*>(P.x0_lo), a->x0_lo, x_bytes, cudaMemcpyHostToDevice, ctx->stream));
    RB_CUDA(cudaMemcpyAsync(const_cast<double*>(P.x0_hi), a->x0_hi, x_bytes, cudaMemcpyHostToDevice, ctx->stream));
    if (act_bytes)
      RB_CUDA(cudaMemcpyAsync(const_cast<double*>(P.actions), a->actions, act_bytes, cudaMemcpyHostToDevice, ctx->stream));
  }
  cudaEvent_t stop;
  rc = timed_begin(ctx, &stop);
  if (rc) return rc;
  RB_CUDA(launch_dt(P, lay, a->batch, ctx->stream));
  rc = timed_end(ctx, stop);
  if (rc) return rc;
  ctx->launches += 1;
  if (!dev) {
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

int reach_split_hull(reach_ctx* ctx, const reach_net* net, const reach_split_args* a, const reach_hull_out* out,
                     int32_t flags) {
  if (!ctx || !net || !a || !out) return REACH_E_INVALID_ARGUMENT;
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
  const long long begin = a->part_begin, end = a->part_end <= 0 ? total : a->part_end;
  if (begin < 0 || begin >= end || end > total) return fail(ctx, REACH_E_INVALID_ARGUMENT, "bad part range");
  RB_CUDA(cudaSetDevice(ctx->device));
  rb::DTParams P{};
  DTLayout lay;
  rc = plan_dt(ctx, net, a->n, a->m, a->window, P, lay);
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
  cudaEvent_t stop;
  rc = timed_begin(ctx, &stop);
  if (rc) return rc;
  RB_CUDA(launch_dt(P, lay, P.B, ctx->stream));
  rc = timed_end(ctx, stop);
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
