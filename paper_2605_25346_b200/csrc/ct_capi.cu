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
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "coll.h"
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

// ---------------------------------------------------------------------------
// Field programs (ct_kernel.cuh: slots P0.., T0..3, V0..9, C0..3).  Each is the
// reference's expression tree for the field body, operand order included.
using rb::ct::TOp;
struct Program {
  std::vector<TOp> ops;
  double kc[rb::ct::kMaxKc] = {};
};
using rb::ct::C_;
using rb::ct::P_;
using rb::ct::T_;
using rb::ct::V_;

// quadrotor_ode (systems.hpp:24-64) with the input rows u: the augmented rows
// P12..15 (make_augmented_field, fields.hpp:96-107: cl_reach) or held
// constants (quadrotor_field, fields.hpp:20-32,51-56: ct_reach); the entries
// are RB_CT_QUAD_OPS (ct_kernel.cuh), which the scalar-only replay compiles.
Program quad_program(const double* prm, const double* u_held) {
  using namespace rb::ct;
  Program p;
  const double mass = prm[0], grav = prm[1], jx = prm[2], jy = prm[3], jz = prm[4];
  p.kc[0] = 1.0 / mass;  // the reference's constants (systems.hpp:48-63)
  p.kc[1] = grav;
  p.kc[2] = (jy - jz) / jx;
  p.kc[3] = 1.0 / jx;
  p.kc[4] = (jz - jx) / jy;
  p.kc[5] = 1.0 / jy;
  p.kc[6] = (jx - jy) / jz;
  p.kc[7] = 1.0 / jz;
  auto U = [&](int k) { return u_held ? C_(k) : P_(12 + k); };
  auto& o = p.ops;
  if (u_held)
    for (int k = 0; k < 4; ++k) {
      p.kc[8 + k] = u_held[k];
      o.push_back({OP_CONST, C_(k), 0, static_cast<unsigned char>(8 + k)});
    }
#define RB_CT_TOP(c, d, a, b) TOp{c, static_cast<unsigned char>(d), static_cast<unsigned char>(a), static_cast<unsigned char>(b)},
  o.insert(o.end(), {RB_CT_QUAD_OPS(RB_CT_TOP, U(0), U(1), U(2), U(3))});
#undef RB_CT_TOP
  if (!u_held)
    for (int i = 12; i < 16; ++i) o.push_back({OP_CONS0, static_cast<unsigned char>(i), 0, 0});  // udot = 0
  o.push_back({OP_END, 0, 0, 0});
  return p;
}

// rotation_ode (systems.hpp:162-167): dx0 = x1 * (-w), dx1 = x0 * w.  Both
// rows read each other, so the scaled rows are materialized before consuming.
Program rotation_program(double w) {
  using namespace rb::ct;
  Program p;
  p.kc[0] = -w;
  p.kc[1] = w;
  p.ops = {{OP_SCALE, V_(0), P_(1), 0}, {OP_SCALE, V_(1), P_(0), 1}, {OP_COPY, T_(0), V_(0), 0},
           {OP_COPY, T_(1), V_(1), 0},  {OP_CONS, 0, T_(0), 0},      {OP_CONS, 1, T_(1), 0},
           {OP_END, 0, 0, 0}};
  return p;
}

// diag_linear_ode (systems.hpp:154-159): dx_i = x_i * lambda_i.
Program diag_program(const double* lam, int n) {
  using namespace rb::ct;
  Program p;
  for (int i = 0; i < n; ++i) {
    p.kc[i] = lam[i];
    p.ops.push_back({OP_SCALE, V_(0), P_(i), static_cast<unsigned char>(i)});
    p.ops.push_back({OP_CONS, static_cast<unsigned char>(i), V_(0), 0});
  }
  p.ops.push_back({OP_END, 0, 0, 0});
  return p;
}

// zero_field (fields.hpp:87-92): dx.assign(n, x[0] * 0.0).
Program zero_program(int n) {
  using namespace rb::ct;
  Program p;
  p.kc[0] = 0.0;
  p.ops = {{OP_SCALE, V_(0), P_(0), 0}, {OP_COPY, T_(0), V_(0), 0}};
  for (int i = 0; i < n; ++i) p.ops.push_back({OP_CONS, static_cast<unsigned char>(i), T_(0), 0});
  p.ops.push_back({OP_END, 0, 0, 0});
  return p;
}

// The program store: every field program's op sequence (they depend on the
// field kind and n only; per-call constants travel in CTParams::kc), uploaded
// to the constant bank of each device once.
struct ProgramStore {
  std::vector<TOp> ops;
  std::map<std::pair<int, int>, int> offset;  // (kind, n) -> first op
  std::mutex mu;
  std::vector<char> uploaded = std::vector<char>(256, 0);
  bool too_long = false;  // a program exceeds the flow kernel's replay cache (FlowSmem::fc)
};
constexpr int kKindQuadAug = 100;
ProgramStore& program_store() {
  static ProgramStore* s = [] {
    auto* st = new ProgramStore();
    const double prm[5] = {1.0, 1.0, 1.0, 1.0, 1.0}, u[4] = {0.0, 0.0, 0.0, 0.0}, lam[16] = {};
    auto add = [&](int kind, int n, const Program& p) {
      st->offset[{kind, n}] = static_cast<int>(st->ops.size());
      st->ops.insert(st->ops.end(), p.ops.begin(), p.ops.end());
      if (p.ops.size() > static_cast<size_t>(rb::ct::kFieldCache) + 1) st->too_long = true;  // + OP_END
    };
    add(kKindQuadAug, 16, quad_program(prm, nullptr));
    add(REACH_FIELD_QUADROTOR, 12, quad_program(prm, u));
    add(REACH_FIELD_ROTATION, 2, rotation_program(1.0));
    for (int n = 1; n <= 16; ++n) {
      add(REACH_FIELD_DIAG_LINEAR, n, diag_program(lam, n));
      add(REACH_FIELD_ZERO, n, zero_program(n));
    }
    return st;
  }();
  return *s;
}

int ensure_programs(reach_ctx* ctx) {
  ProgramStore& st = program_store();
  std::lock_guard<std::mutex> g(st.mu);
  if (ctx->device < 0 || ctx->device >= static_cast<int>(st.uploaded.size())) return REACH_E_INVALID_ARGUMENT;
  if (st.uploaded[ctx->device]) return REACH_OK;
  if (st.ops.size() > static_cast<size_t>(rb::ct::kProgCap)) return fail(ctx, REACH_E_UNSUPPORTED, "program store full");
  if (st.too_long) return fail(ctx, REACH_E_UNSUPPORTED, "field program longer than the flow kernel's replay cache");
  RB_CUDA(cudaMemcpyToSymbol(rb::ct::kProgs, st.ops.data(), st.ops.size() * sizeof(TOp)));
  st.uploaded[ctx->device] = 1;
  return REACH_OK;
}

// Selects a stored program and loads the call's constants; derives the Picard
// bz row of every state row: a row whose derivative is a copy of P_j (and which
// the program never reads) has bz = S_j, one whose derivative is 0 the zero row.
void load_program(const Program& p, int kind, int na, rb::ct::CTParams& P) {
  using namespace rb::ct;
  P.prog = program_store().offset.at({kind, na});
  P.fast_prog = kind == kKindQuadAug ? 1 : kind == REACH_FIELD_QUADROTOR ? 2 : 0;  // the compiled programs
  for (int i = 0; i < kMaxKc; ++i) P.kc[i] = p.kc[i];
  bool read[16] = {};
  for (const TOp& op : p.ops) {
    if (op.code == OP_CONS0 || op.code == OP_END || op.code == OP_CONST || op.code == OP_SUBK) continue;
    if (op.code != OP_CONS) {
      if (op.a < NA) read[op.a] = true;
      if ((op.code == OP_MUL || op.code == OP_MUL2 || op.code == OP_ADD || op.code == OP_SUB) && op.b < NA)
        read[op.b] = true;
    }
  }
  for (int i = 0; i < 16; ++i) P.bzsrc[i] = -1;
  for (const TOp& op : p.ops) {
    if (op.code == OP_CONS0) P.bzsrc[op.dst] = -2;
    if (op.code == OP_CONS && op.a < NA && !read[op.dst]) P.bzsrc[op.dst] = static_cast<signed char>(op.a);
  }
  // the compiled quadrotor programs assume QuadLayout's rows; the interpreter serves anything else
  if (P.fast_prog) {
    const bool held = P.fast_prog == 2;
    const int nrow = held ? NX : NA;
    bool match = na == nrow;
    for (int i = 0; i < nrow && match; ++i) {
      const int want = i < 3 ? i + 3 : i < 12 ? -1 : -2;
      match = P.bzsrc[i] == want;
    }
    if (!match) P.fast_prog = 0;
  }
  // RB_CT_INTERPRET=1 runs every program through the interpreter (tests compare the two implementations)
  if (const char* v = std::getenv("RB_CT_INTERPRET"))
    if (v[0] == '1') P.fast_prog = 0;
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
  P.na = rb::ct::NA;
  P.bw = rb::ct::NA;
  P.square = 0;
  P.ct = 0;
  load_program(quad_program(s->plant_params, nullptr), kKindQuadAug, P.na, P);
  P.ctl = ctl->dev;
  P.T = 1 + s->ctl_steps * s->k_atomic;
  (void)ctx;
  return REACH_OK;
}

// Dynamic shared memory of the flow kernel: the fixed part + S, the zero row,
// the own Picard bz rows and the temporaries; the compact layout (cl_reach
// under the compiled quadrotor program) has a shorter header, 76-column rows
// and no zero row (ct_kernel.cuh, kCompactHdr).
bool flow_compact(const rb::ct::CTParams& P) { return !P.square && P.fast_prog == 1 && P.side != nullptr; }
size_t flow_smem_bytes(const rb::ct::CTParams& P) {
  int npb = 0;
  for (int i = 0; i < P.na; ++i) npb += (P.bzsrc[i] == -1);
  if (flow_compact(P))
    return rb::ct::kCompactHdr + static_cast<size_t>(P.na + npb + 2 * rb::ct::NTF) * rb::ct::kRowC * 8;
  return sizeof(rb::ct::FlowSmem) + static_cast<size_t>(P.na + 1 + npb + 2 * rb::ct::NTF) * rb::ct::NZP * 8;
}

int launch_cl(reach_ctx* ctx, rb::ct::CTParams& P) {
  int prc = ensure_programs(ctx);
  if (prc) return prc;
  const size_t flow_smem = flow_smem_bytes(P);
  int cw = P.ctl.dims[0];  // widest controller layer (and input): the 64-wide buffers fit 12 warps per SM
  for (int t = 1; t < P.ctl.L; ++t) cw = std::max(cw, P.ctl.dims[t]);
  const bool narrow = cw <= 64;
  auto* ctlk = narrow ? rb::ct::ct_ctl_kernel<64> : rb::ct::ct_ctl_kernel<rb::ct::kMaxCtlW>;
  const size_t ctl_smem = rb::ct::kCtlWarps * (narrow ? rb::ct::ctl_warp_bytes<64>(P.ctl.L)
                                                      : rb::ct::ctl_warp_bytes<rb::ct::kMaxCtlW>(P.ctl.L));
  const bool cmp = flow_compact(P);
  auto* flow = cmp ? rb::ct::ct_flow_kernel<false, true> : rb::ct::ct_flow_kernel<false, false>;
  RB_CUDA(cudaFuncSetAttribute(flow, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(flow_smem)));
  RB_CUDA(cudaFuncSetAttribute(ctlk, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(ctl_smem)));
  cudaEvent_t stop;
  int rc = timed_begin(ctx, &stop);
  if (rc) return rc;
  const int ctl_grid = (P.B + rb::ct::kCtlWarps - 1) / rb::ct::kCtlWarps;
  for (int ci = 0; ci < P.ctl_steps; ++ci) {
    P.ci = ci;
    ctlk<<<ctl_grid, 32 * rb::ct::kCtlWarps, ctl_smem, ctx->stream>>>(P);
    RB_CUDA(cudaGetLastError());
    flow<<<P.B, 32, flow_smem, ctx->stream>>>(P);
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
  rbh::DeviceGuard device_guard_(ctx);
  if (!ctx || !ctl || !s || !out) return REACH_E_INVALID_ARGUMENT;
  if (flags & REACH_FLAG_OUTWARD_ROUNDING)
    return fail(ctx, REACH_E_UNSUPPORTED, "outward rounding (g_outward_rounding) is not supported by the device kernels");
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
               o_y = cv.take(std::max<size_t>(static_cast<size_t>(s->ctl_steps) * s->ref_dim * 8, 8)),
               o_side = cv.take(B * rb::ct::kSideBytes);
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
  P.side = reinterpret_cast<unsigned char*>(w + o_side);
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
  rbh::DeviceGuard device_guard_(ctx);
  if (!ctx || !ctl || !s || !a || !out) return REACH_E_INVALID_ARGUMENT;
  if (flags & REACH_FLAG_OUTWARD_ROUNDING)
    return fail(ctx, REACH_E_UNSUPPORTED, "outward rounding (g_outward_rounding) is not supported by the device kernels");
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
  const long long begin0 = a->part_begin, end0 = a->part_end <= 0 ? total : a->part_end;
  if (begin0 < 0 || begin0 >= end0 || end0 > total) return fail(ctx, REACH_E_INVALID_ARGUMENT, "bad part range");
  long long begin, end;  // multi-GPU: this rank's slice; the hull is all-reduced below
  rbh::coll_shard(ctx, begin0, end0, begin, end);
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
               o_side = cv.take(B * rb::ct::kSideBytes), o_kl = cv.take(cnt * 8), o_kh = cv.take(cnt * 8), o_nan = cv.take(cnt * 8), o_div = cv.take(T * 4),
               o_nb = cv.take(4), o_key = cv.take(8), o_lo = cv.take(cnt * 8), o_hi = cv.take(cnt * 8);
  rc = ensure_ws(ctx, cv.off);
  if (rc) return rc;
  char* w = static_cast<char*>(ctx->ws);
  P.st_c = reinterpret_cast<double*>(w + o_c);
  P.st_M = reinterpret_cast<double*>(w + o_M);
  P.st_meta = reinterpret_cast<int*>(w + o_meta);
  P.side = reinterpret_cast<unsigned char*>(w + o_side);
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
  if (P.B > 0) {
    rc = launch_cl(ctx, P);
    if (rc) return rc;
  }
  rc = rbh::coll_hull(ctx, P.hull_lo, P.hull_hi, P.hull_nan0, 2 * icount, P.hull_div, static_cast<int>(T),
                      P.hull_nboxes, P.hull_fail_key);
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

namespace {

// ct_reach's kernel parameters for a field (validation as FlowpipeParams::validate,
// flowpipe_ct.hpp:45-49, plus the device family's limits).
int ct_params(reach_ctx* ctx, const reach_field_desc* fd, const reach_flowpipe_params* fp, rb::ct::CTParams& P) {
  if (!(fp->h > 0) || fp->steps <= 0 || fp->order < 1 || fp->order > 2 || !(fp->eps_init > 0) ||
      !(fp->enlargement > 1.0) || fp->refine_rounds < 0 || fp->max_enlargements < 0 || fp->window < 0)
    return fail(ctx, REACH_E_INVALID_ARGUMENT, "FlowpipeParams: invalid configuration");
  const int n = fd->n;
  Program prog;
  switch (fd->kind) {
    case REACH_FIELD_ZERO: prog = zero_program(n); break;
    case REACH_FIELD_DIAG_LINEAR: prog = diag_program(fd->params, n); break;
    case REACH_FIELD_ROTATION:
      if (n != 2) return fail(ctx, REACH_E_INVALID_ARGUMENT, "rotation_field: n must be 2");
      prog = rotation_program(fd->params[0]);
      break;
    case REACH_FIELD_QUADROTOR:
      if (n != 12) return fail(ctx, REACH_E_INVALID_ARGUMENT, "quadrotor_field: n must be 12");
      prog = quad_program(fd->params, fd->params + 5);
      break;
    default: return fail(ctx, REACH_E_UNSUPPORTED, "ct_reach: unknown field");
  }
  if (n < 1 || n > 16 || n * (fp->window + 2) > rb::ct::NZP)
    return fail(ctx, REACH_E_UNSUPPORTED, "ct_reach: n <= 16 and n (window + 2) <= 80 on the device");
  P.n = n;
  P.na = n;
  P.bw = n;
  P.square = 1;
  P.ct = 1;
  P.ci = 0;
  P.ctl_steps = 1;
  P.K = fp->steps;
  P.T = 1 + fp->steps;
  P.window = fp->window;
  P.order = fp->order;
  P.refine = fp->refine_rounds;
  P.maxe = fp->max_enlargements;
  P.h = fp->h;
  P.eps = fp->eps_init;
  P.enl = fp->enlargement;
  load_program(prog, fd->kind, n, P);
  return ensure_programs(ctx);
}

int launch_ct(reach_ctx* ctx, const rb::ct::CTParams& P) {
  const size_t smem = flow_smem_bytes(P);
  RB_CUDA(cudaFuncSetAttribute(rb::ct::ct_flow_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(smem)));
  cudaEvent_t stop;
  int rc = timed_begin(ctx, &stop);
  if (rc) return rc;
  rb::ct::ct_flow_kernel<true, false><<<P.B, 32, smem, ctx->stream>>>(P);
  RB_CUDA(cudaGetLastError());
  rc = timed_end(ctx, stop);
  if (rc) return rc;
  ctx->launches += 1;
  return REACH_OK;
}

}  // namespace

extern "C" {

int reach_ct_batch(reach_ctx* ctx, const reach_field_desc* fd, const reach_flowpipe_params* fp, int32_t batch,
                   const double* x0_lo, const double* x0_hi, const reach_tube_out* out, int32_t flags) {
  rbh::DeviceGuard device_guard_(ctx);
  if (!ctx || !fd || !fp || !out) return REACH_E_INVALID_ARGUMENT;
  if (flags & REACH_FLAG_OUTWARD_ROUNDING)
    return fail(ctx, REACH_E_UNSUPPORTED, "outward rounding (g_outward_rounding) is not supported by the device kernels");
  if (batch < 0) return fail(ctx, REACH_E_INVALID_ARGUMENT, "ct_reach: negative batch");
  rb::ct::CTParams P{};
  int rc = ct_params(ctx, fd, fp, P);
  if (rc) return rc;
  const int n = fd->n;
  if (batch == 0) return REACH_OK;
  const bool dev = (flags & REACH_FLAG_DEVICE_PTRS) != 0;
  if (!dev)  // build_linear_tm / init_symbolic_state on a diverged X0
    for (size_t i = 0; i < static_cast<size_t>(batch) * n; ++i)
      if (!std::isfinite(x0_lo[i]) || !std::isfinite(x0_hi[i]))
        return fail(ctx, REACH_E_INVALID_ARGUMENT, "ct_reach: non-finite X0");
  RB_CUDA(cudaSetDevice(ctx->device));
  P.B = batch;
  const size_t B = batch, NA = rb::ct::NA, T = P.T;
  const size_t box_bytes = B * T * n * 8, i_bytes = B * 4, x_bytes = B * n * 8;
  Carve cv;
  const size_t o_c = cv.take(B * NA * 8), o_M = cv.take(B * NA * rb::ct::NZP * 8), o_meta = cv.take(B * 16);
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
  rc = launch_ct(ctx, P);
  if (rc) return rc;
  if (!dev) {
    std::vector<int32_t> nb(B);
    RB_CUDA(cudaMemcpyAsync(nb.data(), P.n_boxes, i_bytes, cudaMemcpyDeviceToHost, ctx->stream));
    RB_CUDA(cudaMemcpyAsync(out->failed_step, P.failed_step, i_bytes, cudaMemcpyDeviceToHost, ctx->stream));
    RB_CUDA(cudaMemcpyAsync(out->status, P.status, i_bytes, cudaMemcpyDeviceToHost, ctx->stream));
    RB_CUDA(cudaStreamSynchronize(ctx->stream));
    std::memcpy(out->n_boxes, nb.data(), i_bytes);
    for (size_t i = 0; i < B; ++i) {
      const size_t o = i * T * n, cnt = static_cast<size_t>(nb[i]) * n * 8;
      if (!cnt) continue;
      RB_CUDA(cudaMemcpyAsync(out->lo + o, P.out_lo + o, cnt, cudaMemcpyDeviceToHost, ctx->stream));
      RB_CUDA(cudaMemcpyAsync(out->hi + o, P.out_hi + o, cnt, cudaMemcpyDeviceToHost, ctx->stream));
    }
    RB_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  return REACH_OK;
}

int reach_ct_split_hull(reach_ctx* ctx, const reach_field_desc* fd, const reach_flowpipe_params* fp,
                        const reach_cl_split_args* a, const reach_hull_out* out, int32_t flags) {
  rbh::DeviceGuard device_guard_(ctx);
  if (!ctx || !fd || !fp || !a || !out) return REACH_E_INVALID_ARGUMENT;
  if (flags & REACH_FLAG_OUTWARD_ROUNDING)
    return fail(ctx, REACH_E_UNSUPPORTED, "outward rounding (g_outward_rounding) is not supported by the device kernels");
  rb::ct::CTParams P{};
  int rc = ct_params(ctx, fd, fp, P);
  if (rc) return rc;
  const int n = fd->n;
  long long total = 1;
  for (int d = 0; d < n; ++d) {
    if (a->counts[d] < 1) return fail(ctx, REACH_E_INVALID_ARGUMENT, "SplitPlan: counts must be >= 1");
    total *= a->counts[d];
    if (total > (1ll << 20)) return fail(ctx, REACH_E_INVALID_ARGUMENT, "SplitPlan: total part count overflow");
    if (!std::isfinite(a->x0_lo[d]) || !std::isfinite(a->x0_hi[d]))
      return fail(ctx, REACH_E_INVALID_ARGUMENT, "ct_reach: non-finite X0");
  }
  const long long begin0 = a->part_begin, end0 = a->part_end <= 0 ? total : a->part_end;
  if (begin0 < 0 || begin0 >= end0 || end0 > total) return fail(ctx, REACH_E_INVALID_ARGUMENT, "bad part range");
  long long begin, end;  // multi-GPU: this rank's slice; the hull is all-reduced below
  rbh::coll_shard(ctx, begin0, end0, begin, end);
  RB_CUDA(cudaSetDevice(ctx->device));
  const bool dev = (flags & REACH_FLAG_DEVICE_PTRS) != 0;
  P.B = static_cast<int>(end - begin);
  P.split = 1;
  P.part_begin = begin;
  for (int d = 0; d < n; ++d) {
    P.sx_lo[d] = a->x0_lo[d];
    P.sx_hi[d] = a->x0_hi[d];
    P.counts[d] = a->counts[d];
  }
  const size_t B = end - begin, NA = rb::ct::NA, T = P.T, cnt = T * n;
  Carve cv;
  const size_t o_c = cv.take(B * NA * 8), o_M = cv.take(B * NA * rb::ct::NZP * 8), o_meta = cv.take(B * 16),
               o_kl = cv.take(cnt * 8), o_kh = cv.take(cnt * 8), o_nan = cv.take(cnt * 8), o_div = cv.take(T * 4),
               o_nb = cv.take(4), o_key = cv.take(8), o_lo = cv.take(cnt * 8), o_hi = cv.take(cnt * 8);
  rc = ensure_ws(ctx, cv.off);
  if (rc) return rc;
  char* w = static_cast<char*>(ctx->ws);
  P.st_c = reinterpret_cast<double*>(w + o_c);
  P.st_M = reinterpret_cast<double*>(w + o_M);
  P.st_meta = reinterpret_cast<int*>(w + o_meta);
  P.hull_lo = reinterpret_cast<unsigned long long*>(w + o_kl);
  P.hull_hi = reinterpret_cast<unsigned long long*>(w + o_kh);
  P.hull_nan0 = reinterpret_cast<int*>(w + o_nan);
  P.hull_div = reinterpret_cast<int*>(w + o_div);
  P.hull_nboxes = reinterpret_cast<int*>(w + o_nb);
  P.hull_fail_key = reinterpret_cast<unsigned long long*>(w + o_key);
  const int icount = static_cast<int>(cnt), tpb = 256;
  ct_hull_init_kernel<<<std::max((std::max(icount, static_cast<int>(T)) + tpb - 1) / tpb, 1), tpb, 0, ctx->stream>>>(
      P.hull_lo, P.hull_hi, P.hull_nan0, P.hull_div, icount, static_cast<int>(T), P.hull_nboxes, P.hull_fail_key);
  RB_CUDA(cudaGetLastError());
  if (P.B > 0) {
    rc = launch_ct(ctx, P);
    if (rc) return rc;
  }
  rc = rbh::coll_hull(ctx, P.hull_lo, P.hull_hi, P.hull_nan0, 2 * icount, P.hull_div, static_cast<int>(T),
                      P.hull_nboxes, P.hull_fail_key);
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
