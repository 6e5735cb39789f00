// reach_b200.hpp -- header-only C++17 host API over the C ABI (reach_b200.h).
//
// Mirrors the reference's C++ API for the DT reachability path
// (/root/reference/proj/include/reach/): same names, argument meaning and
// error behaviour (std::invalid_argument on shape errors, per-sample
// failures as tube data), with every batch evaluated by the B200 kernels.
//
//   reference                                   here
//   MLPNet<double> / Layer / Act (neural.hpp)   reach_b200::MLPNet / Layer / Act
//   DTSystem, DTReachParams (dt_reach.hpp)      reach_b200::DTSystem, DTReachParams
//   IntervalBox<double> (interval.hpp)          reach_b200::Box
//   ReachTube<double> (tube.hpp)                reach_b200::ReachTube
//   dt_reach / dt_reach_batch                   reach_b200::dt_reach / dt_reach_batch
//   SplitPlan / reach_with_splitting(dt_reach)  reach_b200::SplitPlan / reach_with_splitting
//   QuadrotorParams (systems.hpp:16-20)         reach_b200::QuadrotorParams
//   FlowpipeParams (flowpipe_ct.hpp:35-50)      reach_b200::FlowpipeParams
//   ClosedLoopSpec / cl_reach (closed_loop.hpp) reach_b200::ClosedLoopSpec / cl_reach / cl_reach_batch
//   reach_with_splitting(cl_reach)              reach_b200::reach_with_splitting_cl
//   ct_reach + zero/diag_linear/rotation/       reach_b200::ct_reach / ct_reach_batch +
//   quadrotor_field (flowpipe_ct.hpp, fields.hpp)  AnalyticField::{zero, diag_linear, rotation, quadrotor}
//   Constraint / PlanProblem / SamplerConfig /  reach_b200::Constraint / PlanProblem / SamplerConfig /
//   PlanResult / plan_objective / plan_cem      PlanResult / plan_objective(_batch) / plan_cem
//   grad_forward(plan_objective) (refine.hpp)   reach_b200::plan_objective_grad
//   MPCConfig / MPCResult / mpc_run (mpc.hpp)   reach_b200::MPCConfig / MPCResult / mpc_run
//   reach_loss (+ grad_forward over params)     reach_b200::reach_loss / reach_loss_gradient
//   gradient_refine of the CLI refine objective reach_b200::refine_tube_volume
//   GradTarget / GradMethod / Gradient /        reach_b200::GradTarget / GradMethod / Gradient /
//   grad_tube_volume (refine.hpp:165-311)       grad_tube_volume
//
// For code that already holds the reference's own types, see
// reach_b200_reference.hpp (drop-in overloads taking reach:: types).
#pragma once

#include <array>
#include <cstdint>
#include <functional>
#include <limits>
#include <memory>
#include <stdexcept>
#include <list>
#include <string>
#include <unordered_map>
#include <vector>

#include "reach_b200.h"

namespace reach_b200 {

enum class Act { Relu = REACH_ACT_RELU, Tanh = REACH_ACT_TANH, Identity = REACH_ACT_IDENTITY };

struct Layer {
  int rows = 0, cols = 0;
  std::vector<double> w;  // row-major rows x cols
  std::vector<double> b;  // rows
  Act act = Act::Identity;
};

struct MLPNet {
  std::vector<Layer> layers;
  int input_dim() const { return layers.front().cols; }
  int output_dim() const { return layers.back().rows; }
  void validate() const {  // neural.hpp:49-56
    if (layers.empty()) throw std::invalid_argument("MLPNet: empty");
    for (size_t l = 0; l + 1 < layers.size(); ++l)
      if (layers[l + 1].cols != layers[l].rows) throw std::invalid_argument("MLPNet: layer shapes do not chain");
    if (layers.back().act != Act::Identity)
      throw std::invalid_argument("MLPNet: final activation must be identity");
  }
};

struct DTSystem {  // dt_reach.hpp:17-29
  MLPNet step;
  int n = 0, m = 0;
  void validate() const {
    step.validate();
    if (n <= 0 || m < 0) throw std::invalid_argument("DTSystem: invalid dimensions");
    if (step.input_dim() != n + m || step.output_dim() != n)
      throw std::invalid_argument("DTSystem: one-step map shape mismatch");
  }
};

struct DTReachParams {  // dt_reach.hpp:31-36
  int window = 4;
  bool rebuild_from_box = false;
};

struct Interval {
  double lo = 0.0, hi = 0.0;
};
using Box = std::vector<Interval>;

struct ReachTube {  // tube.hpp:12-35
  std::vector<Box> boxes;
  std::vector<double> t_lo, t_hi;
  bool diverged = false;
  int failed_step = -1;
  std::string failure_reason;
  int steps() const { return static_cast<int>(boxes.size()); }
};

struct SplitPlan {  // refine.hpp:25-78
  std::vector<int> counts;
};

class Error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

// One device + stream + uploaded networks (one per host thread).
class Context {
 public:
  explicit Context(int device = 0) {
    int rc = reach_ctx_create(device, &ctx_);
    if (rc != REACH_OK) throw Error("reach_ctx_create failed (no usable CUDA device)");
  }
  ~Context() {
    for (auto& c : nets_) reach_net_free(ctx_, c.handle);
    reach_ctx_destroy(ctx_);
  }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;

  reach_ctx* raw() const { return ctx_; }

  // Multi-GPU (one Context per GPU, one process or host thread each): after init_nccl, the batch
  // calls -- reach_with_splitting*, plan_cem -- shard over the ranks inside the library and every
  // rank returns the full single-GPU result (include/reach_b200.h, "Multi-GPU").
  static std::array<uint8_t, 128> nccl_unique_id() {
    std::array<uint8_t, 128> id{};
    if (reach_nccl_unique_id(id.data()) != REACH_OK) throw Error("reach_nccl_unique_id: NCCL not loadable");
    return id;
  }
  void init_nccl(const std::array<uint8_t, 128>& id, int world, int rank) {
    check(reach_ctx_init_nccl(ctx_, id.data(), world, rank), "reach_ctx_init_nccl");
  }
  void set_collectives(const reach_collectives& c) { check(reach_ctx_set_collectives(ctx_, &c), "set_collectives"); }
  void single_gpu() { check(reach_ctx_set_collectives(ctx_, nullptr), "set_collectives"); }

  void check(int rc, const char* what) const {
    if (rc == REACH_OK) return;
    std::string msg = std::string(what) + ": " + reach_ctx_last_error(ctx_);
    if (rc == REACH_E_INVALID_ARGUMENT) throw std::invalid_argument(msg);
    throw Error(msg);
  }

  // Uploads (once per distinct network value) and returns the device network.
  reach_net* upload(const MLPNet& net) {
    net.validate();
    std::vector<int32_t> dims{net.input_dim()}, acts;
    std::vector<double> params;
    for (const auto& L : net.layers) {
      dims.push_back(L.rows);
      acts.push_back(static_cast<int32_t>(L.act));
      params.insert(params.end(), L.w.begin(), L.w.end());
      params.insert(params.end(), L.b.begin(), L.b.end());
    }
    uint64_t key = 1469598103934665603ull;  // FNV-1a over the flattened value
    auto mix = [&key](const void* p, size_t bytes) {
      const unsigned char* c = static_cast<const unsigned char*>(p);
      for (size_t i = 0; i < bytes; ++i) key = (key ^ c[i]) * 1099511628211ull;
    };
    mix(dims.data(), dims.size() * sizeof(int32_t));
    mix(acts.data(), acts.size() * sizeof(int32_t));
    mix(params.data(), params.size() * sizeof(double));
    // hit only on an equal value (the hash is a bucket key, never the identity)
    for (auto it = nets_.begin(); it != nets_.end(); ++it) {
      if (it->key == key && it->dims == dims && it->acts == acts && it->params == params) {
        nets_.splice(nets_.begin(), nets_, it);  // most recently used first
        return it->handle;
      }
    }
    reach_net_desc d{static_cast<int32_t>(net.layers.size()), dims.data(), acts.data(), params.data()};
    reach_net* h = nullptr;
    check(reach_net_upload(ctx_, &d, &h), "reach_net_upload");
    nets_.push_front(Cached{key, std::move(dims), std::move(acts), std::move(params), h});
    while (nets_.size() > kMaxCachedNets) {  // bounded: weight-update loops upload a new value each step
      reach_net_free(ctx_, nets_.back().handle);
      nets_.pop_back();
    }
    return h;
  }

 private:
  struct Cached {
    uint64_t key;
    std::vector<int32_t> dims, acts;
    std::vector<double> params;
    reach_net* handle;
  };
  static constexpr size_t kMaxCachedNets = 32;
  reach_ctx* ctx_ = nullptr;
  std::list<Cached> nets_;
};

inline const char* failure_reason(int32_t status) { return reach_tube_status_string(status); }

// dt_reach_batch (dt_reach.hpp:108-125).
inline std::vector<ReachTube> dt_reach_batch(Context& ctx, const DTSystem& sys, const std::vector<Box>& x0s,
                                             const std::vector<std::vector<std::vector<double>>>& action_seqs,
                                             const DTReachParams& prm = {}) {
  sys.validate();
  if (x0s.size() != action_seqs.size()) throw std::invalid_argument("dt_reach_batch: batch size mismatch");
  std::vector<ReachTube> out(x0s.size());
  if (x0s.empty()) return out;
  const int B = static_cast<int>(x0s.size()), n = sys.n, m = sys.m;
  const int H = static_cast<int>(action_seqs.front().size());
  std::vector<double> lo(static_cast<size_t>(B) * n), hi(lo.size()), acts(static_cast<size_t>(B) * H * m);
  for (int b = 0; b < B; ++b) {
    if (static_cast<int>(x0s[b].size()) != n) throw std::invalid_argument("dt_reach: X0 dimension mismatch");
    if (static_cast<int>(action_seqs[b].size()) != H) throw std::invalid_argument("dt_reach_batch: ragged horizon");
    for (int d = 0; d < n; ++d) {
      lo[static_cast<size_t>(b) * n + d] = x0s[b][d].lo;
      hi[static_cast<size_t>(b) * n + d] = x0s[b][d].hi;
    }
    for (int k = 0; k < H; ++k) {
      if (static_cast<int>(action_seqs[b][k].size()) != m)
        throw std::invalid_argument("dt_reach: action dimension mismatch");
      for (int j = 0; j < m; ++j) acts[(static_cast<size_t>(b) * H + k) * m + j] = action_seqs[b][k][j];
    }
  }
  std::vector<double> olo(static_cast<size_t>(B) * (H + 1) * n), ohi(olo.size());
  std::vector<int32_t> nb(B), fs(B), st(B);
  reach_dt_args a{B, H, n, m, prm.window, prm.rebuild_from_box ? 1 : 0, lo.data(), hi.data(),
                  acts.empty() ? nullptr : acts.data(), 0};
  reach_tube_out o{olo.data(), ohi.data(), nb.data(), fs.data(), st.data()};
  ctx.check(reach_dt_batch(ctx.raw(), ctx.upload(sys.step), &a, &o, 0), "dt_reach_batch");
  for (int b = 0; b < B; ++b) {
    ReachTube& t = out[b];
    for (int k = 0; k < nb[b]; ++k) {
      Box box(n);
      for (int d = 0; d < n; ++d) {
        const size_t i = (static_cast<size_t>(b) * (H + 1) + k) * n + d;
        box[d] = {olo[i], ohi[i]};
      }
      t.boxes.push_back(std::move(box));
      t.t_lo.push_back(k);
      t.t_hi.push_back(k);
    }
    t.failed_step = fs[b];
    t.diverged = st[b] != REACH_TUBE_OK;
    t.failure_reason = st[b] != REACH_TUBE_OK ? failure_reason(st[b]) : "";
  }
  return out;
}

// dt_reach (dt_reach.hpp:40-104).
inline ReachTube dt_reach(Context& ctx, const DTSystem& sys, const Box& x0,
                          const std::vector<std::vector<double>>& actions, const DTReachParams& prm = {}) {
  return dt_reach_batch(ctx, sys, {x0}, {actions}, prm).front();
}

// reach_with_splitting(dt_reach engine, x0, plan) (refine.hpp:121-160); the
// sub-box grid, every sub-tube and the per-step hull stay on the device.
inline ReachTube reach_with_splitting(Context& ctx, const DTSystem& sys, const Box& x0, const SplitPlan& plan,
                                      const std::vector<std::vector<double>>& actions, const DTReachParams& prm = {}) {
  sys.validate();
  const int n = sys.n, m = sys.m, H = static_cast<int>(actions.size());
  if (static_cast<int>(x0.size()) != n || static_cast<int>(plan.counts.size()) != n)
    throw std::invalid_argument("SplitPlan: dimension mismatch");
  std::vector<double> lo(n), hi(n), acts(static_cast<size_t>(H) * m);
  for (int d = 0; d < n; ++d) {
    lo[d] = x0[d].lo;
    hi[d] = x0[d].hi;
  }
  for (int k = 0; k < H; ++k)
    for (int j = 0; j < m; ++j) acts[static_cast<size_t>(k) * m + j] = actions[k][j];
  std::vector<int32_t> counts(plan.counts.begin(), plan.counts.end());
  std::vector<double> olo(static_cast<size_t>(H + 1) * n), ohi(olo.size());
  std::vector<int32_t> div(H + 1);
  int32_t nb = 0;
  int64_t key = 0;
  reach_split_args a{n, m, H, prm.window, prm.rebuild_from_box ? 1 : 0, lo.data(), hi.data(), counts.data(),
                     acts.empty() ? nullptr : acts.data(), 0, 0};
  reach_hull_out o{olo.data(), ohi.data(), div.data(), &nb, &key};
  ctx.check(reach_split_hull(ctx.raw(), ctx.upload(sys.step), &a, &o, 0), "reach_with_splitting");
  ReachTube t;
  for (int k = 0; k < nb; ++k) {
    Box box(n);
    for (int d = 0; d < n; ++d) box[d] = {olo[static_cast<size_t>(k) * n + d], ohi[static_cast<size_t>(k) * n + d]};
    t.boxes.push_back(std::move(box));
    t.t_lo.push_back(k);
    t.t_hi.push_back(k);
    if (div[k]) t.diverged = true;
  }
  if (key != std::numeric_limits<int64_t>::max()) {
    t.diverged = true;
    t.failed_step = static_cast<int>(key >> 40);
    t.failure_reason = "sub-box " + std::to_string((key >> 8) & 0xffffffffLL) + ": " +
                       failure_reason(static_cast<int32_t>(key & 0xff));
  }
  return t;
}

// ---------------------------------------------------------------------------
// Continuous-time closed loop (closed_loop.hpp:16-182).  The dynamics are an
// analytic plant from systems.hpp evaluated on the device (VectorField's host
// closures cannot run there): quadrotor_ode augmented by udot = 0 rows.
struct QuadrotorParams {  // systems.hpp:16-20
  double mass = 1.0, gravity = 9.81, jx = 0.01, jy = 0.01, jz = 0.02;
};

struct FlowpipeParams {  // flowpipe_ct.hpp:35-50
  double h = 0.01;
  int steps = 100;
  int order = 2;
  double eps_init = 1e-4;
  int refine_rounds = 3;
  double enlargement = 2.0;
  int max_enlargements = 20;
  int window = 4;
};

struct ClosedLoopSpec {  // closed_loop.hpp:16-44 (dynamics = the quadrotor plant)
  QuadrotorParams plant;
  MLPNet controller;
  int n = 12, l = 4, ctl_steps = 1, k_atomic = 1;
  std::vector<std::vector<double>> y_ref;
  FlowpipeParams fp;
  bool intervalize_boundary = false;
};

namespace detail {
inline reach_cl_spec cl_c_spec(const ClosedLoopSpec& s, std::vector<double>& yr) {
  reach_cl_spec c{};
  c.plant = REACH_PLANT_QUADROTOR;
  c.plant_params[0] = s.plant.mass;
  c.plant_params[1] = s.plant.gravity;
  c.plant_params[2] = s.plant.jx;
  c.plant_params[3] = s.plant.jy;
  c.plant_params[4] = s.plant.jz;
  c.n = s.n;
  c.l = s.l;
  c.ctl_steps = s.ctl_steps;
  c.k_atomic = s.k_atomic;
  c.ref_dim = s.y_ref.empty() ? 0 : static_cast<int32_t>(s.y_ref.front().size());
  if (!s.y_ref.empty() && static_cast<int>(s.y_ref.size()) != s.ctl_steps)
    throw std::invalid_argument("ClosedLoopSpec: reference sequence length mismatch");
  yr.clear();
  for (const auto& v : s.y_ref) {
    if (static_cast<int>(v.size()) != c.ref_dim) throw std::invalid_argument("ClosedLoopSpec: ragged reference");
    yr.insert(yr.end(), v.begin(), v.end());
  }
  c.y_ref = yr.empty() ? nullptr : yr.data();
  c.fp = reach_flowpipe_params{s.fp.h, s.fp.steps, s.fp.order, s.fp.eps_init, s.fp.refine_rounds,
                               s.fp.enlargement, s.fp.max_enlargements, s.fp.window};
  c.intervalize_boundary = s.intervalize_boundary ? 1 : 0;
  return c;
}
inline void ct_times(ReachTube& t, int k, double h) {  // closed_loop.hpp:155, 172
  t.t_lo.push_back(k == 0 ? 0.0 : (k - 1) * h);
  t.t_hi.push_back(k == 0 ? 0.0 : k * h);
}
}  // namespace detail

// cl_reach (closed_loop.hpp:76-182) for a batch of initial boxes (n dims);
// tubes have up to 1 + ctl_steps * k_atomic boxes of n + l dims.
inline std::vector<ReachTube> cl_reach_batch(Context& ctx, const ClosedLoopSpec& spec, const std::vector<Box>& x0s) {
  std::vector<ReachTube> out(x0s.size());
  if (x0s.empty()) return out;
  std::vector<double> yr;
  reach_cl_spec c = detail::cl_c_spec(spec, yr);
  const int B = static_cast<int>(x0s.size()), n = spec.n, na = spec.n + spec.l;
  const int T = 1 + spec.ctl_steps * spec.k_atomic;
  std::vector<double> lo(static_cast<size_t>(B) * n), hi(lo.size());
  for (int b = 0; b < B; ++b) {
    if (static_cast<int>(x0s[b].size()) != n) throw std::invalid_argument("cl_reach: X0 dimension mismatch");
    for (int d = 0; d < n; ++d) {
      lo[static_cast<size_t>(b) * n + d] = x0s[b][d].lo;
      hi[static_cast<size_t>(b) * n + d] = x0s[b][d].hi;
    }
  }
  std::vector<double> olo(static_cast<size_t>(B) * T * na), ohi(olo.size());
  std::vector<int32_t> nb(B), fs(B), st(B);
  reach_tube_out o{olo.data(), ohi.data(), nb.data(), fs.data(), st.data()};
  ctx.check(reach_cl_batch(ctx.raw(), ctx.upload(spec.controller), &c, B, lo.data(), hi.data(), &o, 0), "cl_reach");
  for (int b = 0; b < B; ++b) {
    ReachTube& t = out[b];
    for (int k = 0; k < nb[b]; ++k) {
      Box box(na);
      for (int d = 0; d < na; ++d) {
        const size_t i = (static_cast<size_t>(b) * T + k) * na + d;
        box[d] = {olo[i], ohi[i]};
      }
      t.boxes.push_back(std::move(box));
      detail::ct_times(t, k, spec.fp.h);
    }
    t.failed_step = fs[b];
    t.diverged = st[b] != REACH_TUBE_OK;
    t.failure_reason = st[b] != REACH_TUBE_OK ? failure_reason(st[b]) : "";
  }
  return out;
}

inline ReachTube cl_reach(Context& ctx, const ClosedLoopSpec& spec, const Box& x0) {
  return cl_reach_batch(ctx, spec, {x0}).front();
}

// reach_with_splitting(cl_reach engine, x0, plan) (refine.hpp:121-160) on the device.
inline ReachTube reach_with_splitting_cl(Context& ctx, const ClosedLoopSpec& spec, const Box& x0,
                                         const SplitPlan& plan) {
  const int n = spec.n, na = spec.n + spec.l, T = 1 + spec.ctl_steps * spec.k_atomic;
  if (static_cast<int>(x0.size()) != n || static_cast<int>(plan.counts.size()) != n)
    throw std::invalid_argument("SplitPlan: dimension mismatch");
  std::vector<double> yr, lo(n), hi(n);
  reach_cl_spec c = detail::cl_c_spec(spec, yr);
  for (int d = 0; d < n; ++d) {
    lo[d] = x0[d].lo;
    hi[d] = x0[d].hi;
  }
  std::vector<int32_t> counts(plan.counts.begin(), plan.counts.end());
  std::vector<double> olo(static_cast<size_t>(T) * na), ohi(olo.size());
  std::vector<int32_t> div(T);
  int32_t nb = 0;
  int64_t key = 0;
  reach_cl_split_args a{lo.data(), hi.data(), counts.data(), 0, 0};
  reach_hull_out o{olo.data(), ohi.data(), div.data(), &nb, &key};
  ctx.check(reach_cl_split_hull(ctx.raw(), ctx.upload(spec.controller), &c, &a, &o, 0),
            "reach_with_splitting(cl_reach)");
  ReachTube t;
  for (int k = 0; k < nb; ++k) {
    Box box(na);
    for (int d = 0; d < na; ++d) box[d] = {olo[static_cast<size_t>(k) * na + d], ohi[static_cast<size_t>(k) * na + d]};
    t.boxes.push_back(std::move(box));
    detail::ct_times(t, k, spec.fp.h);
    if (div[k]) t.diverged = true;
  }
  if (key != std::numeric_limits<int64_t>::max()) {
    t.diverged = true;
    t.failed_step = static_cast<int>(key >> 40);
    t.failure_reason = "sub-box " + std::to_string((key >> 8) & 0xffffffffLL) + ": " +
                       failure_reason(static_cast<int32_t>(key & 0xff));
  }
  return t;
}

// ---------------------------------------------------------------------------
// Open-loop continuous-time flowpipes (ct_reach, flowpipe_ct.hpp:428-458) of the
// analytic fields of fields.hpp: a descriptor, since a VectorField's closures
// cannot run on the device.
struct AnalyticField {
  reach_field_desc d{};
  static AnalyticField zero(int n) { return make(REACH_FIELD_ZERO, n, {}); }
  static AnalyticField diag_linear(const std::vector<double>& lambda) {
    return make(REACH_FIELD_DIAG_LINEAR, static_cast<int>(lambda.size()), lambda);
  }
  static AnalyticField rotation(double w) { return make(REACH_FIELD_ROTATION, 2, {w}); }
  static AnalyticField quadrotor(const QuadrotorParams& p, const std::vector<double>& u) {
    if (u.size() != 4) throw std::invalid_argument("quadrotor_field: 4 inputs");
    return make(REACH_FIELD_QUADROTOR, 12, {p.mass, p.gravity, p.jx, p.jy, p.jz, u[0], u[1], u[2], u[3]});
  }
  int n() const { return d.n; }

 private:
  static AnalyticField make(int kind, int n, const std::vector<double>& prm) {
    if (prm.size() > 16) throw std::invalid_argument("AnalyticField: too many parameters");
    AnalyticField f;
    f.d.kind = kind;
    f.d.n = n;
    for (size_t i = 0; i < prm.size(); ++i) f.d.params[i] = prm[i];
    return f;
  }
};

inline std::vector<ReachTube> ct_reach_batch(Context& ctx, const AnalyticField& f, const std::vector<Box>& x0s,
                                             const FlowpipeParams& prm) {
  std::vector<ReachTube> out(x0s.size());
  if (x0s.empty()) return out;
  const int B = static_cast<int>(x0s.size()), n = f.n(), T = 1 + prm.steps;
  std::vector<double> lo(static_cast<size_t>(B) * n), hi(lo.size());
  for (int b = 0; b < B; ++b) {
    if (static_cast<int>(x0s[b].size()) != n) throw std::invalid_argument("ct_reach: X0 dimension mismatch");
    for (int d = 0; d < n; ++d) {
      lo[static_cast<size_t>(b) * n + d] = x0s[b][d].lo;
      hi[static_cast<size_t>(b) * n + d] = x0s[b][d].hi;
    }
  }
  reach_flowpipe_params fp{prm.h, prm.steps, prm.order, prm.eps_init, prm.refine_rounds,
                           prm.enlargement, prm.max_enlargements, prm.window};
  std::vector<double> olo(static_cast<size_t>(B) * T * n), ohi(olo.size());
  std::vector<int32_t> nb(B), fs(B), st(B);
  reach_tube_out o{olo.data(), ohi.data(), nb.data(), fs.data(), st.data()};
  ctx.check(reach_ct_batch(ctx.raw(), &f.d, &fp, B, lo.data(), hi.data(), &o, 0), "ct_reach");
  for (int b = 0; b < B; ++b) {
    ReachTube& t = out[b];
    for (int k = 0; k < nb[b]; ++k) {
      Box box(n);
      for (int d = 0; d < n; ++d) {
        const size_t i = (static_cast<size_t>(b) * T + k) * n + d;
        box[d] = {olo[i], ohi[i]};
      }
      t.boxes.push_back(std::move(box));
      detail::ct_times(t, k, prm.h);
    }
    t.failed_step = fs[b];
    t.diverged = st[b] != REACH_TUBE_OK;
    t.failure_reason = st[b] != REACH_TUBE_OK ? failure_reason(st[b]) : "";
  }
  return out;
}

inline ReachTube ct_reach(Context& ctx, const AnalyticField& f, const Box& x0, const FlowpipeParams& prm) {
  return ct_reach_batch(ctx, f, {x0}, prm).front();
}

// ---------------------------------------------------------------------------
// Reachability-aware MPC (mpc.hpp).

struct Constraint {  // mpc.hpp:25-112
  enum class Type { halfspace_avoid = REACH_CON_HALFSPACE_AVOID, sphere_avoid = REACH_CON_SPHERE_AVOID,
                    box_stay_in = REACH_CON_BOX_STAY_IN, max_volume = REACH_CON_MAX_VOLUME };
  Type type = Type::max_volume;
  std::vector<int> dims;  // empty = all state dims
  std::vector<double> a;
  double b = 0.0;
  std::vector<double> center;
  double radius = 0.0;
  std::vector<double> lo, hi;
  double vmax = 0.0;
};

struct PlanProblem {  // mpc.hpp:115-142
  DTSystem sys;
  std::vector<double> x_goal, q_weights, r_weights;
  std::vector<Constraint> constraints;
  double penalty = 100.0;
  double diverged_margin = 1e3;
  int horizon = 5;
  std::vector<double> u_lo, u_hi;
  double eps = 0.0;
  DTReachParams dt_prm;
};

struct SamplerConfig {  // mpc.hpp:220-234
  int population = 256;
  double elite_frac = 0.1;
  int iterations = 5;
  double init_std = 0.3;
  double smoothing = 0.5;
  int refine_iters = 5;
  uint64_t seed = 0;
};

struct PlanResult {  // mpc.hpp:236-243
  std::vector<std::vector<double>> actions;
  double objective = 0.0;
  ReachTube tube;
  std::vector<double> best_history;
  bool best_effort = false;
  bool refined = false;
};

namespace detail {

// The C ABI view of a PlanProblem; owns the flattened constraint arrays.
struct PlanC {
  reach_plan_problem p{};
  std::vector<reach_constraint> cons;
  std::vector<std::vector<int32_t>> dims;
  explicit PlanC(const PlanProblem& pr) {
    pr.sys.validate();
    for (const auto& c : pr.constraints) {
      dims.emplace_back(c.dims.begin(), c.dims.end());
      reach_constraint r{};
      r.type = static_cast<int32_t>(c.type);
      r.n_dims = static_cast<int32_t>(c.dims.size());
      r.dims = dims.back().empty() ? nullptr : dims.back().data();
      r.a = c.a.empty() ? nullptr : c.a.data();
      r.b = c.b;
      r.center = c.center.empty() ? nullptr : c.center.data();
      r.radius = c.radius;
      r.lo = c.lo.empty() ? nullptr : c.lo.data();
      r.hi = c.hi.empty() ? nullptr : c.hi.data();
      r.vmax = c.vmax;
      cons.push_back(r);
    }
    // sizes the ABI cannot see are checked here (PlanProblem::validate, mpc.hpp:129-141)
    const size_t n = static_cast<size_t>(pr.sys.n), m = static_cast<size_t>(pr.sys.m);
    if (pr.x_goal.size() != n || pr.q_weights.size() != n || pr.r_weights.size() != m)
      throw std::invalid_argument("PlanProblem: cost dimension mismatch");
    if (pr.u_lo.size() != m || pr.u_hi.size() != m)
      throw std::invalid_argument("PlanProblem: action box dimension mismatch");
    for (const auto& c : pr.constraints) {
      const size_t k = c.dims.empty() ? n : c.dims.size();
      const bool ok = c.type == Constraint::Type::halfspace_avoid ? c.a.size() == k
                      : c.type == Constraint::Type::sphere_avoid  ? c.center.size() == k
                      : c.type == Constraint::Type::box_stay_in   ? c.lo.size() == k && c.hi.size() == k
                                                                  : true;
      if (!ok) throw std::invalid_argument("Constraint: parameter size");
    }
    p.n = pr.sys.n;
    p.m = pr.sys.m;
    p.horizon = pr.horizon;
    p.window = pr.dt_prm.window;
    p.rebuild_from_box = pr.dt_prm.rebuild_from_box ? 1 : 0;
    p.x_goal = pr.x_goal.data();
    p.q_weights = pr.q_weights.data();
    p.r_weights = pr.r_weights.data();
    p.n_constraints = static_cast<int32_t>(cons.size());
    p.constraints = cons.empty() ? nullptr : cons.data();
    p.penalty = pr.penalty;
    p.diverged_margin = pr.diverged_margin;
    p.eps = pr.eps;
    p.u_lo = pr.u_lo.data();
    p.u_hi = pr.u_hi.data();
  }
};

inline std::vector<double> flatten_plan(const PlanProblem& pr, const std::vector<std::vector<double>>& acts) {
  if (static_cast<int>(acts.size()) != pr.horizon) throw std::invalid_argument("plan: horizon mismatch");
  std::vector<double> flat;
  flat.reserve(static_cast<size_t>(pr.horizon) * pr.sys.m);
  for (const auto& u : acts) {
    if (static_cast<int>(u.size()) != pr.sys.m) throw std::invalid_argument("plan: action dimension mismatch");
    flat.insert(flat.end(), u.begin(), u.end());
  }
  return flat;
}

}  // namespace detail

// plan_objective (mpc.hpp:204-208) of a batch of action sequences, evaluated
// together (plan_eval's objective and diverged flag per candidate).
inline std::vector<double> plan_objective_batch(Context& ctx, const PlanProblem& pr, const std::vector<double>& x0,
                                                const std::vector<std::vector<std::vector<double>>>& cands,
                                                std::vector<bool>* diverged = nullptr) {
  detail::PlanC pc(pr);
  if (static_cast<int>(x0.size()) != pr.sys.n) throw std::invalid_argument("plan_eval: x0 dimension mismatch");
  std::vector<double> flat;
  for (const auto& c : cands) {
    auto f = detail::flatten_plan(pr, c);
    flat.insert(flat.end(), f.begin(), f.end());
  }
  const int B = static_cast<int>(cands.size());
  std::vector<double> obj(B);
  std::vector<int32_t> div(B);
  if (B > 0)
    ctx.check(reach_plan_eval_batch(ctx.raw(), ctx.upload(pr.sys.step), &pc.p, x0.data(), B, flat.data(),
                                    obj.data(), div.data(), nullptr, 0),
              "plan_eval");
  if (diverged) diverged->assign(div.begin(), div.end());
  return obj;
}

inline double plan_objective(Context& ctx, const PlanProblem& pr, const std::vector<double>& x0,
                             const std::vector<std::vector<double>>& actions) {
  return plan_objective_batch(ctx, pr, x0, {actions}).front();
}

// grad_forward (refine.hpp:186-207) of plan_objective over the flat action
// sequence ([H][m], row-major): forward-dual directions evaluated on the device.
inline std::vector<double> plan_objective_grad(Context& ctx, const PlanProblem& pr, const std::vector<double>& x0,
                                               const std::vector<std::vector<double>>& actions,
                                               double* objective = nullptr) {
  detail::PlanC pc(pr);
  if (static_cast<int>(x0.size()) != pr.sys.n) throw std::invalid_argument("plan_eval: x0 dimension mismatch");
  auto flat = detail::flatten_plan(pr, actions);
  std::vector<double> g(flat.size());
  double obj = 0.0;
  ctx.check(reach_plan_objective_grad(ctx.raw(), ctx.upload(pr.sys.step), &pc.p, x0.data(), flat.data(), g.data(),
                                      &obj),
            "grad_forward");
  if (objective) *objective = obj;
  return g;
}

// plan_cem (mpc.hpp:258-368): CEM over device-evaluated populations, then the
// top candidate's gradient refinement (refine_iters > 0).
inline PlanResult plan_cem(Context& ctx, const PlanProblem& pr, const SamplerConfig& cfg,
                           const std::vector<double>& x0) {
  detail::PlanC pc(pr);
  if (static_cast<int>(x0.size()) != pr.sys.n) throw std::invalid_argument("plan_eval: x0 dimension mismatch");
  reach_sampler_config c{cfg.population, cfg.elite_frac, cfg.iterations, cfg.init_std, cfg.smoothing,
                         cfg.refine_iters, cfg.seed};
  const int H = pr.horizon, m = pr.sys.m, n = pr.sys.n;
  std::vector<double> best(static_cast<size_t>(H) * m), hist(cfg.iterations > 0 ? cfg.iterations : 1);
  double obj = 0.0;
  int32_t be = 0, rf = 0;
  std::vector<double> olo(static_cast<size_t>(H + 1) * n), ohi(olo.size());
  int32_t nb = 0, fs = -1, st = 0;
  reach_tube_out o{olo.data(), ohi.data(), &nb, &fs, &st};
  ctx.check(reach_plan_cem_ex(ctx.raw(), ctx.upload(pr.sys.step), &pc.p, &c, x0.data(), best.data(), &obj,
                              hist.data(), &be, &rf, &o),
            "plan_cem");
  PlanResult r;
  for (int t = 0; t < H; ++t) r.actions.emplace_back(best.begin() + t * m, best.begin() + (t + 1) * m);
  r.objective = obj;
  r.best_history.assign(hist.begin(), hist.begin() + cfg.iterations);
  r.best_effort = be != 0;
  r.refined = rf != 0;
  for (int k = 0; k < nb; ++k) {
    Box box(n);
    for (int d = 0; d < n; ++d) box[d] = {olo[static_cast<size_t>(k) * n + d], ohi[static_cast<size_t>(k) * n + d]};
    r.tube.boxes.push_back(std::move(box));
    r.tube.t_lo.push_back(k);
    r.tube.t_hi.push_back(k);
  }
  r.tube.failed_step = fs;
  r.tube.diverged = st != REACH_TUBE_OK;
  r.tube.failure_reason = st != REACH_TUBE_OK ? failure_reason(st) : "";
  return r;
}

// ---------------------------------------------------------------------------
// Receding-horizon MPC (mpc.hpp:373-495).

struct MPCConfig {  // mpc.hpp:373-387
  int replan_period = 3;
  int total_steps = 30;
  double dist_action = 0.0;
  double dist_state = 0.0;
  std::vector<int> goal_dims;
  double goal_radius = 0.1;
  uint64_t seed = 0;
};

struct MPCLogRow {  // mpc.hpp:389-396
  int step = 0;
  std::vector<double> state, action;
  double objective = 0.0, tube_volume = 0.0, g_margin = 0.0;
};

struct MPCResult {  // mpc.hpp:398-419
  bool success = false, violated = false;
  int steps_used = 0;
  std::vector<double> final_state;
  std::vector<MPCLogRow> log;
};

using SimStep = std::function<std::vector<double>(const std::vector<double>&, const std::vector<double>&)>;

// mpc_run: planning, margins and (sim empty) the model simulator on the device;
// a non-empty `sim` is the caller's true system, called on the host.
inline MPCResult mpc_run(Context& ctx, const PlanProblem& pr, const SamplerConfig& sampler, const MPCConfig& cfg,
                         const SimStep& sim, const std::vector<double>& x0) {
  detail::PlanC pc(pr);
  const int n = pr.sys.n, m = pr.sys.m, T = cfg.total_steps > 0 ? cfg.total_steps : 1;
  if (static_cast<int>(x0.size()) != n) throw std::invalid_argument("mpc_run: x0 dimension mismatch");
  reach_sampler_config sc{sampler.population, sampler.elite_frac, sampler.iterations, sampler.init_std,
                          sampler.smoothing, sampler.refine_iters, sampler.seed};
  std::vector<int32_t> gd(cfg.goal_dims.begin(), cfg.goal_dims.end());
  reach_mpc_config mc{cfg.replan_period, cfg.total_steps, cfg.dist_action, cfg.dist_state,
                      static_cast<int32_t>(gd.size()), gd.empty() ? nullptr : gd.data(), cfg.goal_radius, cfg.seed};
  std::vector<int32_t> st(T);
  std::vector<double> xs(static_cast<size_t>(T) * n), us(static_cast<size_t>(T) * (m > 0 ? m : 1)), ob(T), tv(T),
      gm(T);
  reach_mpc_log lg{st.data(), xs.data(), us.data(), ob.data(), tv.data(), gm.data()};
  struct Tramp {
    const SimStep* f;
    int n, m;
    static int call(void* user, const double* x, const double* u, double* xn) {
      auto* t = static_cast<Tramp*>(user);
      try {
        std::vector<double> out = (*t->f)(std::vector<double>(x, x + t->n), std::vector<double>(u, u + t->m));
        if (static_cast<int>(out.size()) != t->n) return 1;
        std::copy(out.begin(), out.end(), xn);
        return 0;
      } catch (...) {
        return 1;
      }
    }
  } tr{&sim, n, m};
  MPCResult r;
  r.final_state.assign(n, 0.0);
  int32_t succ = 0, viol = 0, used = 0, rows = 0;
  ctx.check(reach_mpc_run(ctx.raw(), ctx.upload(pr.sys.step), &pc.p, &sc, &mc, sim ? &Tramp::call : nullptr, &tr,
                          x0.data(), &succ, &viol, &used, r.final_state.data(), &lg, &rows),
            "mpc_run");
  r.success = succ != 0;
  r.violated = viol != 0;
  r.steps_used = used;
  for (int i = 0; i < rows; ++i) {
    MPCLogRow row;
    row.step = st[i];
    row.state.assign(xs.begin() + static_cast<size_t>(i) * n, xs.begin() + static_cast<size_t>(i + 1) * n);
    if (m > 0) row.action.assign(us.begin() + static_cast<size_t>(i) * m, us.begin() + static_cast<size_t>(i + 1) * m);
    row.objective = ob[i];
    row.tube_volume = tv[i];
    row.g_margin = gm[i];
    r.log.push_back(std::move(row));
  }
  return r;
}

// ---------------------------------------------------------------------------
// Tube-volume gradients (refine.hpp:165-311).

enum class GradTarget { x0_center = REACH_GRAD_X0_CENTER, actions = REACH_GRAD_ACTIONS, weights = REACH_GRAD_WEIGHTS };
enum class GradMethod { forward_dual = REACH_GRAD_FORWARD_DUAL, finite_difference = REACH_GRAD_FINITE_DIFFERENCE };

struct Gradient {  // refine.hpp:171-178
  std::vector<double> g;
  GradMethod method = GradMethod::forward_dual;
  bool subgradient = false;
};

// grad_tube_volume (refine.hpp:263-311): every pass on the device, one launch.
inline Gradient grad_tube_volume(Context& ctx, const DTSystem& sys, const Box& x0,
                                 const std::vector<std::vector<double>>& actions, GradTarget target,
                                 GradMethod method = GradMethod::forward_dual, const DTReachParams& prm = {}) {
  sys.validate();
  const int n = sys.n, m = sys.m, H = static_cast<int>(actions.size());
  if (static_cast<int>(x0.size()) != n) throw std::invalid_argument("dt_reach: X0 dimension mismatch");
  std::vector<double> lo(n), hi(n), acts;
  for (int d = 0; d < n; ++d) {
    lo[d] = x0[d].lo;
    hi[d] = x0[d].hi;
  }
  for (const auto& u : actions) {
    if (static_cast<int>(u.size()) != m) throw std::invalid_argument("dt_reach: action dimension mismatch");
    acts.insert(acts.end(), u.begin(), u.end());
  }
  size_t dim = 0;
  if (target == GradTarget::x0_center) dim = n;
  else if (target == GradTarget::actions) dim = acts.size();
  else
    for (const auto& L : sys.step.layers) dim += L.w.size() + L.b.size();
  Gradient out;
  out.method = method;
  out.g.assign(std::max<size_t>(dim, 1), 0.0);
  int32_t sub = 0;
  reach_dt_args a{1, H, n, m, prm.window, prm.rebuild_from_box ? 1 : 0, lo.data(), hi.data(),
                  acts.empty() ? nullptr : acts.data(), 0};
  ctx.check(reach_grad_tube_volume(ctx.raw(), ctx.upload(sys.step), &a, static_cast<int32_t>(target),
                                   static_cast<int32_t>(method), out.g.data(), &sub, nullptr),
            "grad_tube_volume");
  out.g.resize(dim);
  out.subgradient = sub != 0;
  return out;
}

// reach_loss (training.hpp:99-126) over episodes given by their start states [M][n] and first t_h
// actions [M][t_h][m]; grad != nullptr also returns its gradient over the model's parameters
// (net_params order), the training objective's grad_forward.
inline double reach_loss(Context& ctx, const MLPNet& model, const std::vector<std::vector<double>>& x0s,
                         const std::vector<std::vector<std::vector<double>>>& actions, double eps, double cap,
                         int* diverged_count = nullptr, const DTReachParams& prm = {},
                         std::vector<double>* grad = nullptr) {
  model.validate();
  const int M = static_cast<int>(x0s.size());
  if (M == 0 || actions.size() != x0s.size() || actions.front().empty())
    throw std::invalid_argument("reach_loss: bad batch/horizon");
  const int n = static_cast<int>(x0s.front().size()), t_h = static_cast<int>(actions.front().size());
  const int m = static_cast<int>(actions.front().front().size());
  std::vector<double> x(static_cast<size_t>(M) * n), a(static_cast<size_t>(M) * t_h * m);
  for (int e = 0; e < M; ++e) {
    if (static_cast<int>(x0s[e].size()) != n || static_cast<int>(actions[e].size()) != t_h)
      throw std::invalid_argument("reach_loss: ragged batch");
    std::copy(x0s[e].begin(), x0s[e].end(), x.begin() + static_cast<size_t>(e) * n);
    for (int t = 0; t < t_h; ++t) {
      if (static_cast<int>(actions[e][t].size()) != m) throw std::invalid_argument("reach_loss: action dims");
      std::copy(actions[e][t].begin(), actions[e][t].end(), a.begin() + (static_cast<size_t>(e) * t_h + t) * m);
    }
  }
  size_t np = 0;
  for (const auto& L : model.layers) np += L.w.size() + L.b.size();
  if (grad) grad->assign(np, 0.0);
  reach_dt_args args{M, t_h, n, m, prm.window, prm.rebuild_from_box ? 1 : 0, x.data(), x.data(),
                     a.empty() ? nullptr : a.data(), 0};
  double loss = 0.0;
  int32_t dc = 0;
  ctx.check(reach_reach_loss(ctx.raw(), ctx.upload(model), &args, M, eps, cap, &loss, grad ? grad->data() : nullptr,
                             &dc),
            "reach_loss");
  if (diverged_count) *diverged_count += dc;
  return loss;
}

struct RefineResult {  // refine.hpp:333-340
  std::vector<double> x;
  double initial_objective = 0.0, objective = 0.0;
  bool progressed = false, subgradient = false;
  int accepted_steps = 0;
};

// gradient_refine (refine.hpp:354-398) of tube_volume(dt_reach(box_from_center(c, radius), actions))
// over the X0 centre or the flat action sequence within [lo, hi] -- the reference CLI's `refine`.
inline RefineResult refine_tube_volume(Context& ctx, const DTSystem& sys, const std::vector<double>& center,
                                       const std::vector<double>& radius,
                                       const std::vector<std::vector<double>>& actions, GradTarget target,
                                       const std::vector<double>& x0, const std::vector<double>& lo,
                                       const std::vector<double>& hi, int iters = 20,
                                       const DTReachParams& prm = {}) {
  sys.validate();
  const int n = sys.n, m = sys.m, H = static_cast<int>(actions.size());
  std::vector<double> acts;
  for (const auto& u : actions) {
    if (static_cast<int>(u.size()) != m) throw std::invalid_argument("dt_reach: action dimension mismatch");
    acts.insert(acts.end(), u.begin(), u.end());
  }
  const size_t d = target == GradTarget::x0_center ? static_cast<size_t>(n) : acts.size();
  if (center.size() != static_cast<size_t>(n) || radius.size() != static_cast<size_t>(n) || x0.size() != d ||
      lo.size() != d || hi.size() != d)
    throw std::invalid_argument("gradient_refine: bound dimension mismatch");
  RefineResult r;
  r.x = x0;
  int32_t pr = 0, sb = 0, ac = 0;
  reach_dt_args a{1, H, n, m, prm.window, prm.rebuild_from_box ? 1 : 0, center.data(), center.data(),
                  acts.empty() ? nullptr : acts.data(), 0};
  ctx.check(reach_refine_tube_volume(ctx.raw(), ctx.upload(sys.step), &a, center.data(), radius.data(),
                                     static_cast<int32_t>(target), lo.data(), hi.data(), iters, r.x.data(),
                                     &r.initial_objective, &r.objective, &pr, &sb, &ac),
            "gradient_refine");
  r.progressed = pr != 0;
  r.subgradient = sb != 0;
  r.accepted_steps = ac;
  return r;
}

// dt_interval_baseline (dt_reach.hpp:129-149): the naive interval tube of the same map.
inline ReachTube dt_interval_baseline(Context& ctx, const DTSystem& sys, const Box& x0,
                                      const std::vector<std::vector<double>>& actions) {
  sys.validate();
  const int n = sys.n, m = sys.m, H = static_cast<int>(actions.size());
  if (static_cast<int>(x0.size()) != n) throw std::invalid_argument("dt_reach: X0 dimension mismatch");
  std::vector<double> lo(n), hi(n), acts;
  for (int d = 0; d < n; ++d) {
    lo[d] = x0[d].lo;
    hi[d] = x0[d].hi;
  }
  for (const auto& u : actions) {
    if (static_cast<int>(u.size()) != m) throw std::invalid_argument("dt_reach: action dimension mismatch");
    acts.insert(acts.end(), u.begin(), u.end());
  }
  std::vector<double> olo(static_cast<size_t>(H + 1) * n), ohi(olo.size());
  int32_t nb = 0, fs = -1, st = 0;
  reach_dt_args a{1, H, n, m, 0, 0, lo.data(), hi.data(), acts.empty() ? nullptr : acts.data(), 0};
  reach_tube_out o{olo.data(), ohi.data(), &nb, &fs, &st};
  ctx.check(reach_dt_interval_baseline_batch(ctx.raw(), ctx.upload(sys.step), &a, &o), "dt_interval_baseline");
  ReachTube t;
  for (int k = 0; k < nb; ++k) {
    Box box(n);
    for (int d = 0; d < n; ++d) box[d] = {olo[static_cast<size_t>(k) * n + d], ohi[static_cast<size_t>(k) * n + d]};
    t.boxes.push_back(std::move(box));
    t.t_lo.push_back(k);
    t.t_hi.push_back(k);
  }
  t.failed_step = fs;
  t.diverged = st != REACH_TUBE_OK;
  t.failure_reason = st != REACH_TUBE_OK ? failure_reason(st) : "";
  return t;
}

}  // namespace reach_b200
