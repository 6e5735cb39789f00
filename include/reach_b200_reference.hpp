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

// reach::dt_reach_batch (dt_reach.hpp:108-125)
inline std::vector<reach::ReachTube<double>> dt_reach_batch(
    Context& ctx, const reach::DTSystem<double>& sys, const std::vector<reach::IntervalBox<double>>& x0s,
    const std::vector<std::vector<reach::Vec<double>>>& action_seqs, const reach::DTReachParams& prm = {}) {
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
  return to_reference(cl_reach(ctx, from_reference(spec, plant), from_reference(x0)));
}

// reach::reach_with_splitting with the cl_reach engine (refine.hpp:121-160)
inline reach::ReachTube<double> reach_with_splitting_cl(Context& ctx, const reach::ClosedLoopSpec<double>& spec,
                                                        const reach::QuadrotorParams& plant,
                                                        const reach::IntervalBox<double>& x0,
                                                        const reach::SplitPlan& plan) {
  plan.validate(x0.size());
  return to_reference(reach_with_splitting_cl(ctx, from_reference(spec, plant), from_reference(x0), SplitPlan{plan.counts}));
}

// reach::ct_reach(field, x0, prm) (flowpipe_ct.hpp:428-458) for the analytic
// fields of fields.hpp, named by a descriptor (a VectorField's closures cannot
// run on the device): e.g. reach::rotation_field<double>(w) ->
// AnalyticField::rotation(w).
inline reach::ReachTube<double> ct_reach(Context& ctx, const AnalyticField& f, const reach::IntervalBox<double>& x0,
                                         const reach::FlowpipeParams& prm) {
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
