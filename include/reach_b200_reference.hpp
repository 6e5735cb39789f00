// reach_b200_reference.hpp -- drop-in overloads for code that holds the
// reference's own types (include after the reference headers, with the
// reference's include/ on the include path):
//
//   #include "reach/dt_reach.hpp"
//   #include "reach/refine.hpp"
//   #include "reach_b200_reference.hpp"
//   reach_b200::Context gpu;
//   auto tubes = reach_b200::dt_reach_batch(gpu, sys, x0s, seqs, prm);   // same args as
//                                                                        // reach::dt_reach_batch
//
// Each overload converts the reference value types at the boundary and
// returns reference ReachTube<double> values (boxes, time stamps, diverged,
// failed_step, failure_reason exactly as the reference builds them,
// tube.hpp:23-34), computed by the B200 kernels.
#pragma once

#include <cmath>

#include "reach/closed_loop.hpp"
#include "reach/dt_reach.hpp"
#include "reach/mpc.hpp"
#include "reach/refine.hpp"
#include "reach/systems.hpp"
#include "reach/training.hpp"
#include "reach_b200.hpp"

namespace reach_b200 {

inline MLPNet from_reference(const reach::MLPNet<double>& net) {
  MLPNet out;
  for (const auto& L : net.layers) {
    Layer l;
    l.rows = L.w.rows;
    l.cols = L.w.cols;
    l.w = L.w.a;
    l.b = L.b;
    l.act = L.act == reach::Act::Relu ? Act::Relu : L.act == reach::Act::Tanh ? Act::Tanh : Act::Identity;
    out.layers.push_back(std::move(l));
  }
  return out;
}

inline DTSystem from_reference(const reach::DTSystem<double>& sys) {
  DTSystem s;
  s.step = from_reference(sys.step);
  s.n = sys.n;
  s.m = sys.m;
  return s;
}

inline Box from_reference(const reach::IntervalBox<double>& b) {
  Box out(b.size());
  for (int d = 0; d < b.size(); ++d) out[d] = {b[d].lo, b[d].hi};
  return out;
}

inline reach::ReachTube<double> to_reference(const ReachTube& t) {
  reach::ReachTube<double> out;
  for (size_t k = 0; k < t.boxes.size(); ++k) {
    reach::IntervalBox<double> b(static_cast<int>(t.boxes[k].size()));
    for (int d = 0; d < b.size(); ++d) b[d] = {t.boxes[k][d].lo, t.boxes[k][d].hi};
    b.check_divergence();
    out.push(b, t.t_lo[k], t.t_hi[k]);
  }
  if (t.failed_step >= 0 || t.diverged) out.mark_failed(t.failed_step, t.failure_reason);
  return out;
}

namespace detail {
// A caller that switched on the reference's outward rounding (reach::ScopedOutwardRounding,
// interval.hpp:19-25) gets an error, not round-to-nearest results (C ABI: REACH_FLAG_OUTWARD_ROUNDING).
inline void refuse_outward_rounding() {
  if (reach::g_outward_rounding)
    throw Error("outward rounding (g_outward_rounding) is not supported by the device kernels");
}
}  // namespace detail

// reach::dt_reach_batch (dt_reach.hpp:108-125)
inline std::vector<reach::ReachTube<double>> dt_reach_batch(
    Context& ctx, const reach::DTSystem<double>& sys, const std::vector<reach::IntervalBox<double>>& x0s,
    const std::vector<std::vector<reach::Vec<double>>>& action_seqs, const reach::DTReachParams& prm = {}) {
  detail::refuse_outward_rounding();
  std::vector<Box> boxes;
  boxes.reserve(x0s.size());
  for (const auto& b : x0s) boxes.push_back(from_reference(b));
  DTReachParams p{prm.window, prm.rebuild_from_box};
  auto tubes = dt_reach_batch(ctx, from_reference(sys), boxes, action_seqs, p);
  std::vector<reach::ReachTube<double>> out;
  out.reserve(tubes.size());
  for (const auto& t : tubes) out.push_back(to_reference(t));
  return out;
}

// reach::dt_reach (dt_reach.hpp:40-104)
inline reach::ReachTube<double> dt_reach(Context& ctx, const reach::DTSystem<double>& sys,
                                         const reach::IntervalBox<double>& x0,
                                         const std::vector<reach::Vec<double>>& actions,
                                         const reach::DTReachParams& prm = {}) {
  return dt_reach_batch(ctx, sys, {x0}, {actions}, prm).front();
}

// reach::reach_with_splitting with the dt_reach engine (refine.hpp:121-160)
inline reach::ReachTube<double> reach_with_splitting_dt(Context& ctx, const reach::DTSystem<double>& sys,
                                                        const reach::IntervalBox<double>& x0,
                                                        const reach::SplitPlan& plan,
                                                        const std::vector<reach::Vec<double>>& actions,
                                                        const reach::DTReachParams& prm = {}) {
  detail::refuse_outward_rounding();
  plan.validate(x0.size());
  SplitPlan p{plan.counts};
  DTReachParams q{prm.window, prm.rebuild_from_box};
  return to_reference(reach_with_splitting(ctx, from_reference(sys), from_reference(x0), p, actions, q));
}

// reach::cl_reach (closed_loop.hpp:76-182).  A ClosedLoopSpec's dynamics is a
// host closure the device cannot run, so the caller names the plant it was
// built from: spec.dynamics must be make_augmented_field(12, 4, quadrotor_ode
// with `plant`) (fields.hpp:96-128), which the shape check below enforces.
inline ClosedLoopSpec from_reference(const reach::ClosedLoopSpec<double>& spec, const reach::QuadrotorParams& plant) {
  spec.validate();
  if (spec.n != 12 || spec.l != 4 || spec.dynamics.n != 16)
    throw std::invalid_argument("cl_reach: the device plant is quadrotor_ode (n = 12, l = 4)");
  ClosedLoopSpec s;
  s.plant = {plant.mass, plant.gravity, plant.jx, plant.jy, plant.jz};
  s.controller = from_reference(spec.controller);
  s.n = spec.n;
  s.l = spec.l;
  s.ctl_steps = spec.ctl_steps;
  s.k_atomic = spec.k_atomic;
  s.y_ref = spec.y_ref;
  s.fp = {spec.fp.h, spec.fp.steps, spec.fp.order, spec.fp.eps_init, spec.fp.refine_rounds,
          spec.fp.enlargement, spec.fp.max_enlargements, spec.fp.window};
  s.intervalize_boundary = spec.intervalize_boundary;
  return s;
}

inline reach::ReachTube<double> cl_reach(Context& ctx, const reach::ClosedLoopSpec<double>& spec,
                                         const reach::QuadrotorParams& plant, const reach::IntervalBox<double>& x0) {
  detail::refuse_outward_rounding();
  return to_reference(cl_reach(ctx, from_reference(spec, plant), from_reference(x0)));
}

// reach::reach_with_splitting with the cl_reach engine (refine.hpp:121-160)
inline reach::ReachTube<double> reach_with_splitting_cl(Context& ctx, const reach::ClosedLoopSpec<double>& spec,
                                                        const reach::QuadrotorParams& plant,
                                                        const reach::IntervalBox<double>& x0,
                                                        const reach::SplitPlan& plan) {
  detail::refuse_outward_rounding();
  plan.validate(x0.size());
  return to_reference(reach_with_splitting_cl(ctx, from_reference(spec, plant), from_reference(x0), SplitPlan{plan.counts}));
}

// reach::ct_reach(field, x0, prm) (flowpipe_ct.hpp:428-458) for the analytic
// fields of fields.hpp, named by a descriptor (a VectorField's closures cannot
// run on the device): e.g. reach::rotation_field<double>(w) ->
// AnalyticField::rotation(w).
inline reach::ReachTube<double> ct_reach(Context& ctx, const AnalyticField& f, const reach::IntervalBox<double>& x0,
                                         const reach::FlowpipeParams& prm) {
  detail::refuse_outward_rounding();
  prm.validate();
  FlowpipeParams p{prm.h, prm.steps, prm.order, prm.eps_init, prm.refine_rounds, prm.enlargement,
                   prm.max_enlargements, prm.window};
  return to_reference(ct_reach(ctx, f, from_reference(x0), p));
}

// reach::plan_cem (mpc.hpp:258-368) on reference PlanProblem / SamplerConfig
// values; returns the reference PlanResult (plan, objective, final tube,
// history, best_effort, refined) computed on the device.
inline PlanProblem from_reference(const reach::PlanProblem& p) {
  PlanProblem q;
  q.sys = from_reference(p.sys);
  q.x_goal = p.x_goal;
  q.q_weights = p.q_weights;
  q.r_weights = p.r_weights;
  for (const auto& c : p.constraints) {
    Constraint k;
    k.type = static_cast<Constraint::Type>(static_cast<int>(c.type));
    k.dims = c.dims;
    k.a = c.a;
    k.b = c.b;
    k.center = c.center;
    k.radius = c.radius;
    k.lo = c.lo;
    k.hi = c.hi;
    k.vmax = c.vmax;
    q.constraints.push_back(std::move(k));
  }
  q.penalty = p.penalty;
  q.diverged_margin = p.diverged_margin;
  q.horizon = p.horizon;
  q.u_lo = p.u_lo;
  q.u_hi = p.u_hi;
  q.eps = p.eps;
  q.dt_prm = {p.dt_prm.window, p.dt_prm.rebuild_from_box};
  return q;
}

inline reach::PlanResult plan_cem(Context& ctx, const reach::PlanProblem& prob, const reach::SamplerConfig& cfg,
                                  const reach::Vec<double>& x0) {
  prob.validate();
  cfg.validate();
  SamplerConfig c{cfg.population, cfg.elite_frac, cfg.iterations, cfg.init_std, cfg.smoothing, cfg.refine_iters,
                  cfg.seed};
  PlanResult r = plan_cem(ctx, from_reference(prob), c, x0);
  reach::PlanResult out;
  out.actions = r.actions;
  out.objective = r.objective;
  out.tube = to_reference(r.tube);
  out.best_history = r.best_history;
  out.best_effort = r.best_effort;
  out.refined = r.refined;
  return out;
}

// reach::plan_objective (mpc.hpp:204-208) with S = double.
inline double plan_objective(Context& ctx, const reach::PlanProblem& prob, const reach::Vec<double>& x0,
                             const std::vector<reach::Vec<double>>& actions) {
  prob.validate();
  return plan_objective(ctx, from_reference(prob), x0, actions);
}

// reach::grad_tube_volume (refine.hpp:263-311) -> reach::Gradient, computed on the device.
inline reach::Gradient grad_tube_volume(Context& ctx, const reach::DTSystem<double>& sys,
                                        const reach::IntervalBox<double>& x0,
                                        const std::vector<reach::Vec<double>>& actions, reach::GradTarget target,
                                        reach::GradMethod method = reach::GradMethod::forward_dual,
                                        const reach::DTReachParams& prm = {}) {
  sys.validate();
  const GradTarget t = target == reach::GradTarget::x0_center ? GradTarget::x0_center
                       : target == reach::GradTarget::actions ? GradTarget::actions
                                                              : GradTarget::weights;
  const GradMethod me =
      method == reach::GradMethod::forward_dual ? GradMethod::forward_dual : GradMethod::finite_difference;
  Gradient g = grad_tube_volume(ctx, from_reference(sys), from_reference(x0), actions, t, me,
                                DTReachParams{prm.window, prm.rebuild_from_box});
  reach::Gradient out;
  out.g = g.g;
  out.method = method;
  out.subgradient = g.subgradient;
  return out;
}

// reach::mpc_run (mpc.hpp:425-495) -> reach::MPCResult.  sim_step is the
// reference's Sim argument (called on the host); planning runs on the device.
template <class Sim>
inline reach::MPCResult mpc_run(Context& ctx, const reach::PlanProblem& prob, const reach::SamplerConfig& sampler,
                                const reach::MPCConfig& cfg, Sim&& sim_step, const reach::Vec<double>& x0) {
  prob.validate();
  cfg.validate(prob.horizon);
  SamplerConfig s{sampler.population, sampler.elite_frac, sampler.iterations, sampler.init_std, sampler.smoothing,
                  sampler.refine_iters, sampler.seed};
  MPCConfig c{cfg.replan_period, cfg.total_steps, cfg.dist_action, cfg.dist_state, cfg.goal_dims, cfg.goal_radius,
              cfg.seed};
  SimStep f = [&](const std::vector<double>& x, const std::vector<double>& u) {
    return std::vector<double>(sim_step(reach::Vec<double>(x), reach::Vec<double>(u)));
  };
  MPCResult r = mpc_run(ctx, from_reference(prob), s, c, f, x0);
  reach::MPCResult out;
  out.success = r.success;
  out.violated = r.violated;
  out.steps_used = r.steps_used;
  out.final_state = r.final_state;
  for (const auto& row : r.log) {
    reach::MPCLogRow q;
    q.step = row.step;
    q.state = row.state;
    q.action = row.action;
    q.objective = row.objective;
    q.tube_volume = row.tube_volume;
    q.g_margin = row.g_margin;
    out.log.push_back(std::move(q));
  }
  return out;
}

// reach::reach_loss (training.hpp:99-126) on the device; reach_loss_gradient = grad_forward of it over
// net_params(model) (what train_dt_dyn differentiates), one launch over parameters x episodes.
namespace detail {
inline void episodes_to_arrays(const std::vector<reach::Episode>& batch, int t_h,
                               std::vector<std::vector<double>>& x0s,
                               std::vector<std::vector<std::vector<double>>>& acts) {
  if (batch.empty() || t_h < 1) throw std::invalid_argument("reach_loss: bad batch/horizon");
  for (const auto& ep : batch) {
    if (ep.length() < t_h) throw std::invalid_argument("reach_loss: episode shorter than T_h");
    x0s.push_back(ep.states.front());
    acts.emplace_back(ep.actions.begin(), ep.actions.begin() + t_h);
  }
}
}  // namespace detail

inline double reach_loss(Context& ctx, const reach::MLPNet<double>& model, const std::vector<reach::Episode>& batch,
                         double eps, int t_h, double cap, int* diverged_count = nullptr,
                         const reach::DTReachParams& prm = {}) {
  std::vector<std::vector<double>> x0s;
  std::vector<std::vector<std::vector<double>>> acts;
  detail::episodes_to_arrays(batch, t_h, x0s, acts);
  return reach_loss(ctx, from_reference(model), x0s, acts, eps, cap, diverged_count,
                    DTReachParams{prm.window, prm.rebuild_from_box});
}

inline reach::Gradient reach_loss_gradient(Context& ctx, const reach::MLPNet<double>& model,
                                           const std::vector<reach::Episode>& batch, double eps, int t_h,
                                           double cap, const reach::DTReachParams& prm = {}) {
  std::vector<std::vector<double>> x0s;
  std::vector<std::vector<std::vector<double>>> acts;
  detail::episodes_to_arrays(batch, t_h, x0s, acts);
  reach::Gradient g;
  reach_loss(ctx, from_reference(model), x0s, acts, eps, cap, nullptr, DTReachParams{prm.window, prm.rebuild_from_box},
             &g.g);
  g.method = reach::GradMethod::forward_dual;
  return g;
}

// ---- certified training (training.hpp) on the device ------------------------------------------------
namespace detail {
// Episodes of one length as a reach_episode_set (storage kept in `buf`).
struct EpisodeArrays {
  std::vector<double> states, actions, y_ref;
  reach_episode_set set{};
};
inline EpisodeArrays episode_arrays(const std::vector<reach::Episode>& batch) {
  EpisodeArrays a;
  if (batch.empty()) throw std::invalid_argument("empty episode batch");
  const int T = batch.front().length();
  const int n = static_cast<int>(batch.front().states.front().size());
  const int m = T > 0 ? static_cast<int>(batch.front().actions.front().size()) : 0;
  const int r = batch.front().y_ref.empty() ? 0 : static_cast<int>(batch.front().y_ref.front().size());
  for (const auto& ep : batch) {
    ep.validate();
    if (ep.length() != T) throw std::invalid_argument("episodes of one batch must share a length");
    for (const auto& x : ep.states) a.states.insert(a.states.end(), x.begin(), x.end());
    for (const auto& u : ep.actions) a.actions.insert(a.actions.end(), u.begin(), u.end());
    if (r > 0) {
      if (static_cast<int>(ep.y_ref.size()) != T) throw std::invalid_argument("Episode: reference length mismatch");
      for (const auto& y : ep.y_ref) a.y_ref.insert(a.y_ref.end(), y.begin(), y.end());
    }
  }
  a.set = reach_episode_set{static_cast<int32_t>(batch.size()), T, n, m, a.states.data(),
                            a.actions.empty() ? nullptr : a.actions.data(), r, r > 0 ? a.y_ref.data() : nullptr};
  return a;
}
inline reach_net_desc net_desc(const MLPNet& net, std::vector<int32_t>& dims, std::vector<int32_t>& acts,
                               std::vector<double>& params) {
  net.validate();
  dims.assign(1, net.input_dim());
  for (const auto& L : net.layers) {
    dims.push_back(L.rows);
    acts.push_back(static_cast<int32_t>(L.act));
    params.insert(params.end(), L.w.begin(), L.w.end());
    params.insert(params.end(), L.b.begin(), L.b.end());
  }
  return reach_net_desc{static_cast<int32_t>(net.layers.size()), dims.data(), acts.data(), params.data()};
}
inline reach_train_config train_config(const reach::TrainConfig& c) {
  return reach_train_config{c.horizon_max, c.eps0, c.eps_final, c.lambda, c.gamma, c.iters, c.batch, c.lr,
                            c.reach_cap, c.curriculum ? 1 : 0, c.seed, c.dt_prm.window,
                            c.dt_prm.rebuild_from_box ? 1 : 0};
}
inline reach::TrainLog train_log(const std::vector<reach_train_log_row>& rows) {
  reach::TrainLog log;
  for (const auto& r : rows) log.rows.push_back({r.iter, r.t_h, r.eps, r.l_pred, r.l_reach, r.l_total, r.diverged_count});
  return log;
}
inline reach_cl_spec quad_spec(const reach::QuadrotorParams& plant, int n, int l, int k_atomic, int ref_dim,
                               const reach::FlowpipeParams& fp) {
  reach_cl_spec sp{};
  sp.plant = REACH_PLANT_QUADROTOR;
  sp.plant_params[0] = plant.mass;
  sp.plant_params[1] = plant.gravity;
  sp.plant_params[2] = plant.jx;
  sp.plant_params[3] = plant.jy;
  sp.plant_params[4] = plant.jz;
  sp.n = n;
  sp.l = l;
  sp.ctl_steps = 1;
  sp.k_atomic = k_atomic;
  sp.ref_dim = ref_dim;
  sp.fp = reach_flowpipe_params{fp.h, fp.steps, fp.order, fp.eps_init, fp.refine_rounds, fp.enlargement,
                                fp.max_enlargements, fp.window};
  return sp;
}
}  // namespace detail

// reach::pred_loss (training.hpp:60-83) and its grad_forward over net_params.
inline double pred_loss(Context& ctx, const reach::MLPNet<double>& model, const std::vector<reach::Episode>& batch,
                        int t_h, const reach::Vec<double>& weights, reach::Gradient* grad = nullptr) {
  if (batch.empty() || t_h < 1 || static_cast<int>(weights.size()) != t_h)
    throw std::invalid_argument("pred_loss: bad batch/horizon/weights");
  auto a = detail::episode_arrays(batch);
  double loss = 0.0;
  if (grad) {
    grad->g.assign(static_cast<size_t>(model.param_count()), 0.0);
    grad->method = reach::GradMethod::forward_dual;
  }
  ctx.check(reach_pred_loss(ctx.raw(), ctx.upload(from_reference(model)), &a.set, t_h, weights.data(), &loss,
                            grad ? grad->g.data() : nullptr),
            "pred_loss");
  return loss;
}

// reach::track_loss (training.hpp:134-178) with the quadrotor plant, and its grad_forward.
inline double track_loss(Context& ctx, const reach::MLPNet<double>& controller, const reach::QuadrotorParams& plant,
                         const std::vector<reach::Episode>& batch, int t_t, const reach::Vec<double>& weights,
                         double gamma, double delta, int rk4_substeps = 4, double cap = 1e6,
                         int* blowup_count = nullptr, reach::Gradient* grad = nullptr) {
  auto a = detail::episode_arrays(batch);
  const double prm[5] = {plant.mass, plant.gravity, plant.jx, plant.jy, plant.jz};
  double loss = 0.0;
  int32_t bc = 0;
  if (grad) {
    grad->g.assign(static_cast<size_t>(controller.param_count()), 0.0);
    grad->method = reach::GradMethod::forward_dual;
  }
  ctx.check(reach_track_loss(ctx.raw(), ctx.upload(from_reference(controller)), REACH_PLANT_QUADROTOR, prm, &a.set,
                             t_t, weights.data(), gamma, delta, rk4_substeps, cap, &loss,
                             grad ? grad->g.data() : nullptr, &bc),
            "track_loss");
  if (blowup_count) *blowup_count += bc;
  return loss;
}

// grad_forward of reach::ctl_reach_loss over the controller's net_params (Dual cl_reach per parameter
// and episode on the device).  Every episode must carry its t_h references when the controller takes
// them (the reference's carry-over of an empty y_ref is resolved here).
inline reach::Gradient ctl_reach_loss_gradient(Context& ctx, const reach::MLPNet<double>& controller,
                                               const reach::QuadrotorParams& plant,
                                               const std::vector<reach::Episode>& batch, double eps, int t_h, int n,
                                               int l, double delta, int k_atomic, double cap,
                                               const reach::FlowpipeParams& fp_base = {},
                                               double* loss = nullptr, int* diverged_count = nullptr) {
  if (batch.empty() || t_h < 1) throw std::invalid_argument("ctl_reach_loss: bad batch/horizon");
  std::vector<double> x0s, yr;
  std::vector<reach::Vec<double>> cur;
  int r = 0;
  for (const auto& ep : batch) {
    x0s.insert(x0s.end(), ep.states.front().begin(), ep.states.front().end());
    if (!ep.y_ref.empty()) cur.assign(ep.y_ref.begin(), ep.y_ref.begin() + t_h);
    if (!cur.empty()) r = static_cast<int>(cur.front().size());
    for (const auto& y : cur) yr.insert(yr.end(), y.begin(), y.end());
  }
  if (r > 0 && yr.size() != batch.size() * static_cast<size_t>(t_h) * r)
    throw std::invalid_argument("freeze_trailing_inputs: dimension mismatch");
  reach::FlowpipeParams fp = fp_base;
  fp.h = delta / k_atomic;
  reach_cl_spec sp = detail::quad_spec(plant, n, l, k_atomic, r, fp);
  sp.ctl_steps = t_h;
  reach::Gradient g;
  g.g.assign(static_cast<size_t>(controller.param_count()), 0.0);
  double lv = 0.0;
  int32_t dc = 0;
  ctx.check(reach_ctl_reach_loss(ctx.raw(), ctx.upload(from_reference(controller)), &sp,
                                 static_cast<int32_t>(batch.size()), x0s.data(), r > 0 ? yr.data() : nullptr, eps, cap,
                                 &lv, g.g.data(), &dc),
            "ctl_reach_loss");
  if (loss) *loss = lv;
  if (diverged_count) *diverged_count = dc;
  return g;
}

// reach::train_dt_dyn (training.hpp:333-382): the reference's loop, every loss and gradient on the device.
inline reach::TrainResult train_dt_dyn(Context& ctx, const reach::MLPNet<double>& init, const reach::TrainConfig& cfg,
                                       const std::vector<reach::Episode>& dataset) {
  auto a = detail::episode_arrays(dataset);
  std::vector<int32_t> dims, acts;
  std::vector<double> params;
  const MLPNet net = from_reference(init);
  reach_net_desc d = detail::net_desc(net, dims, acts, params);
  reach_train_config c = detail::train_config(cfg);
  std::vector<double> out(params.size());
  std::vector<reach_train_log_row> rows(static_cast<size_t>(std::max(cfg.iters, 1)));
  const int rc = reach_train_dt_dyn(ctx.raw(), &d, &c, &a.set, out.data(), rows.data());
  if (rc == REACH_E_NONFINITE) throw std::runtime_error(reach_ctx_last_error(ctx.raw()));
  ctx.check(rc, "train_dt_dyn");
  return reach::TrainResult{reach::net_with_params<double>(init, out), detail::train_log(rows)};
}

// reach::train_ct_ctl (training.hpp:389-442) with the quadrotor plant.
inline reach::TrainResult train_ct_ctl(Context& ctx, const reach::MLPNet<double>& init, const reach::TrainConfig& cfg,
                                       const std::vector<reach::Episode>& dataset,
                                       const reach::QuadrotorParams& plant, int n, int l, double delta,
                                       int k_atomic = 1, int rk4_substeps = 4,
                                       const reach::FlowpipeParams& fp_base = {}) {
  auto a = detail::episode_arrays(dataset);
  std::vector<int32_t> dims, acts;
  std::vector<double> params;
  const MLPNet net = from_reference(init);
  reach_net_desc d = detail::net_desc(net, dims, acts, params);
  reach_train_config c = detail::train_config(cfg);
  reach_cl_spec sp = detail::quad_spec(plant, n, l, k_atomic, a.set.ref_dim, fp_base);
  std::vector<double> out(params.size());
  std::vector<reach_train_log_row> rows(static_cast<size_t>(std::max(cfg.iters, 1)));
  const int rc = reach_train_ct_ctl(ctx.raw(), &d, &c, &a.set, &sp, delta, rk4_substeps, out.data(), rows.data());
  if (rc == REACH_E_NONFINITE) throw std::runtime_error(reach_ctx_last_error(ctx.raw()));
  ctx.check(rc, "train_ct_ctl");
  return reach::TrainResult{reach::net_with_params<double>(init, out), detail::train_log(rows)};
}

// reach::dt_interval_baseline (dt_reach.hpp:129-149)
inline reach::ReachTube<double> dt_interval_baseline(Context& ctx, const reach::DTSystem<double>& sys,
                                                     const reach::IntervalBox<double>& x0,
                                                     const std::vector<reach::Vec<double>>& actions) {
  return to_reference(dt_interval_baseline(ctx, from_reference(sys), from_reference(x0), actions));
}

// reach::ctl_reach_loss (training.hpp:183-213) with the quadrotor plant (the reference takes the plant
// body as a template argument; the device runs quadrotor_ode with `plant`): every episode's closed loop
// on the device -- episodes sharing a reference sequence in one batch -- and the loss summed in episode
// order on the host.  As the reference, an episode without y_ref keeps the previous one's.
inline double ctl_reach_loss(Context& ctx, const reach::MLPNet<double>& controller,
                             const reach::QuadrotorParams& plant, const std::vector<reach::Episode>& batch,
                             double eps, int t_h, int n, int l, double delta, int k_atomic, double cap,
                             int* diverged_count = nullptr, const reach::FlowpipeParams& fp_base = {}) {
  if (batch.empty() || t_h < 1) throw std::invalid_argument("ctl_reach_loss: bad batch/horizon");
  ClosedLoopSpec spec;
  spec.plant = {plant.mass, plant.gravity, plant.jx, plant.jy, plant.jz};
  spec.controller = from_reference(controller);
  spec.n = n;
  spec.l = l;
  spec.ctl_steps = t_h;
  spec.k_atomic = k_atomic;
  spec.fp = {delta / k_atomic, fp_base.steps, fp_base.order, fp_base.eps_init, fp_base.refine_rounds,
             fp_base.enlargement, fp_base.max_enlargements, fp_base.window};
  std::vector<std::vector<std::vector<double>>> refs;  // per episode, after the carry-over
  std::vector<std::vector<double>> cur;
  for (const auto& ep : batch) {
    if (!ep.y_ref.empty()) cur.assign(ep.y_ref.begin(), ep.y_ref.begin() + t_h);
    refs.push_back(cur);
  }
  std::vector<double> terms(batch.size(), 0.0);
  std::vector<bool> done(batch.size(), false);
  int dc = 0;
  for (size_t e0 = 0; e0 < batch.size(); ++e0) {
    if (done[e0]) continue;
    std::vector<size_t> idx;
    std::vector<Box> x0s;
    for (size_t e = e0; e < batch.size(); ++e)
      if (!done[e] && refs[e] == refs[e0]) {
        idx.push_back(e);
        Box b(static_cast<size_t>(n));
        for (int d = 0; d < n; ++d) b[d] = {batch[e].states.front()[d] - eps, batch[e].states.front()[d] + eps};
        x0s.push_back(std::move(b));
        done[e] = true;
      }
    spec.y_ref = refs[e0];
    auto tubes = cl_reach_batch(ctx, spec, x0s);
    for (size_t q = 0; q < idx.size(); ++q) {
      const ReachTube& t = tubes[q];
      if (t.diverged) {
        terms[idx[q]] = cap;
        ++dc;
      } else {
        double v = 0.0;  // predicted_volume (training.hpp:89-93)
        for (size_t k = 1; k < t.boxes.size(); ++k) {
          double w = 0.0;
          bool fin = true;
          for (const auto& iv : t.boxes[k]) {
            fin = fin && std::isfinite(iv.lo) && std::isfinite(iv.hi);
            w += iv.hi - iv.lo;
          }
          v += fin ? w : std::numeric_limits<double>::infinity();
        }
        terms[idx[q]] = std::log(1.0 + v);
      }
    }
  }
  double acc = 0.0;
  for (double v : terms) acc += v;
  if (diverged_count) *diverged_count += dc;
  return acc / static_cast<double>(batch.size());
}

}  // namespace reach_b200
