// TEST INFRASTRUCTURE ONLY -- never linked into the product library.
//
// C-ABI driver around the UNMODIFIED reference headers
// (/root/reference/proj/include/reach/, compiled by include path, nothing
// copied).  Built by oracle/Makefile into oracle/_ref/libreach_ref.so, which
// the tests use as the ground truth and bench.py's `--impl reference` /
// cpu_baseline legs time on the host cores.  Only tests/, __graft_entry__.smoke()
// and bench.py's CPU legs may load it.
//
// Every call below is a reference entry point; the glue only converts the
// flat C structs of include/reach_b200.h to/from reference types.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include "reach/closed_loop.hpp"
#include "reach/dt_reach.hpp"
#include "reach/fields.hpp"
#include "reach/mpc.hpp"
#include "reach/training.hpp"
#include "reach/neural.hpp"
#include "reach/parallel.hpp"
#include "reach/refine.hpp"

#include "reach_b200.h"

using namespace reach;

namespace {

MLPNet<double> net_from_desc(const reach_net_desc* d) {
  MLPNet<double> net;
  size_t k = 0;
  for (int l = 0; l < d->n_layers; ++l) {
    Layer<double> layer;
    int rows = d->dims[l + 1], cols = d->dims[l];
    layer.w = Mat<double>(rows, cols);
    for (int i = 0; i < rows * cols; ++i) layer.w.a[static_cast<size_t>(i)] = d->params[k++];
    layer.b.resize(static_cast<size_t>(rows));
    for (int i = 0; i < rows; ++i) layer.b[static_cast<size_t>(i)] = d->params[k++];
    layer.act = d->acts[l] == REACH_ACT_RELU   ? Act::Relu
                : d->acts[l] == REACH_ACT_TANH ? Act::Tanh
                                               : Act::Identity;
    net.layers.push_back(std::move(layer));
  }
  return net;
}

int32_t status_of(const ReachTube<double>& t) {
  if (!t.diverged && t.failed_step < 0) return REACH_TUBE_OK;
  if (t.failure_reason == "relax_activation: non-finite preactivation") return REACH_TUBE_NONFINITE_PREACT;
  if (t.failure_reason == "diverged certification") return REACH_TUBE_DIVERGED_CERT;
  if (t.failure_reason == "diverged box") return REACH_TUBE_DIVERGED_BOX;
  return REACH_TUBE_OTHER;
}

Box box_at(const double* lo, const double* hi, int n) {
  Box b(n);
  for (int d = 0; d < n; ++d) b[d] = {lo[d], hi[d]};
  return b;
}

std::vector<Vec<double>> actions_at(const double* a, int horizon, int m) {
  std::vector<Vec<double>> out(static_cast<size_t>(horizon), Vec<double>(static_cast<size_t>(m)));
  for (int k = 0; k < horizon; ++k)
    for (int j = 0; j < m; ++j) out[static_cast<size_t>(k)][static_cast<size_t>(j)] = a[k * m + j];
  return out;
}

DTSystem<double> make_sys(const reach_net_desc* desc, int n, int m) {
  DTSystem<double> sys;
  sys.step = net_from_desc(desc);
  sys.n = n;
  sys.m = m;
  return sys;
}

}  // namespace

extern "C" {

// dt_reach (dt_reach.hpp:41) per sample inside the reference parallel_for
// (parallel.hpp:17) with an explicit thread count (0 = hardware threads),
// per-element exception isolation as dt_reach_batch (dt_reach.hpp:116-123).
int ref_dt_batch(const reach_net_desc* desc, const reach_dt_args* a, const reach_tube_out* out,
                 int32_t threads) {
  try {
    DTSystem<double> sys = make_sys(desc, a->n, a->m);
    DTReachParams prm;
    prm.window = a->window;
    prm.rebuild_from_box = a->rebuild_from_box != 0;
    const int H = a->horizon, n = a->n, m = a->m;
    parallel_for(
        a->batch,
        [&](int b) {
          ReachTube<double> tube;
          try {
            const double* act = a->actions_shared ? a->actions : a->actions + static_cast<size_t>(b) * H * m;
            tube = dt_reach(sys, box_at(a->x0_lo + static_cast<size_t>(b) * n, a->x0_hi + static_cast<size_t>(b) * n, n),
                            actions_at(act, H, m), prm);
          } catch (const std::exception& e) {
            tube.mark_failed(0, e.what());
          }
          out->n_boxes[b] = tube.steps();
          out->failed_step[b] = tube.failed_step;
          out->status[b] = status_of(tube);
          for (int k = 0; k < tube.steps(); ++k)
            for (int d = 0; d < n; ++d) {
              size_t o = (static_cast<size_t>(b) * (H + 1) + k) * n + d;
              out->lo[o] = tube.boxes[static_cast<size_t>(k)][d].lo;
              out->hi[o] = tube.boxes[static_cast<size_t>(k)][d].hi;
            }
        },
        threads);
  } catch (const std::exception&) {
    return REACH_E_INVALID_ARGUMENT;
  }
  return REACH_OK;
}

// reach_with_splitting(dt_reach, x0, plan) (refine.hpp:121-160) restricted to
// parts [begin, end): it always reassembles the reference pieces -- split_box,
// dt_reach per part in parallel_for, box_hull in ascending index order, the
// failure key -- because the reference driver itself has no part range (a
// bounded CPU sample / one shard needs one).  The driver verbatim is
// ref_reach_with_splitting below; tests/test_oracle.py checks the two agree on
// full plans.
int ref_split_hull(const reach_net_desc* desc, const reach_split_args* a, const reach_hull_out* out,
                   int32_t threads) {
  try {
    DTSystem<double> sys = make_sys(desc, a->n, a->m);
    DTReachParams prm;
    prm.window = a->window;
    prm.rebuild_from_box = a->rebuild_from_box != 0;
    const int H = a->horizon, n = a->n;
    auto actions = actions_at(a->actions, H, a->m);
    Box x0 = box_at(a->x0_lo, a->x0_hi, n);
    SplitPlan plan;
    plan.counts.assign(a->counts, a->counts + n);
    const long long total = plan.total_parts();
    long long begin = a->part_begin, end = a->part_end <= 0 ? total : a->part_end;
    if (begin < 0 || begin >= end || end > total) return REACH_E_INVALID_ARGUMENT;

    auto engine = [&](const Box& b) { return dt_reach(sys, b, actions, prm); };
    auto parts = split_box(x0, plan);
    const int count = static_cast<int>(end - begin);
    std::vector<ReachTube<double>> subs(static_cast<size_t>(count));
    parallel_for(
        count,
        [&](int i) {
          try {
            subs[static_cast<size_t>(i)] = engine(parts[static_cast<size_t>(begin + i)]);
          } catch (const std::exception& e) {
            subs[static_cast<size_t>(i)].mark_failed(0, e.what());
          }
        },
        threads);
    // identical reduction to refine.hpp:133-158
    int steps = subs.front().steps();
    int64_t key = std::numeric_limits<int64_t>::max();
    for (int i = 0; i < count; ++i) {
      const auto& s = subs[static_cast<size_t>(i)];
      steps = std::min(steps, s.steps());
      if (s.diverged) {
        int fs = s.failed_step >= 0 ? s.failed_step : s.steps();
        int64_t k = (static_cast<int64_t>(fs) << 40) | (static_cast<int64_t>(begin + i) << 8) |
                    static_cast<int64_t>(status_of(s) & 0xff);
        key = std::min(key, k);
      }
    }
    for (int k = 0; k < steps; ++k) {
      Box b = subs.front().boxes[static_cast<size_t>(k)];
      for (int i = 1; i < count; ++i) b = box_hull(b, subs[static_cast<size_t>(i)].boxes[static_cast<size_t>(k)]);
      for (int d = 0; d < n; ++d) {
        out->lo[static_cast<size_t>(k) * n + d] = b[d].lo;
        out->hi[static_cast<size_t>(k) * n + d] = b[d].hi;
      }
      out->box_diverged[k] = b.diverged ? 1 : 0;
    }
    out->n_boxes[0] = steps;
    out->fail_key[0] = key;
  } catch (const std::exception&) {
    return REACH_E_INVALID_ARGUMENT;
  }
  return REACH_OK;
}

// The reference driver itself, for the `--impl reference` arm on full plans.
int ref_reach_with_splitting(const reach_net_desc* desc, const reach_split_args* a, double* lo, double* hi,
                             int32_t* n_boxes, int32_t* failed_step) {
  try {
    DTSystem<double> sys = make_sys(desc, a->n, a->m);
    DTReachParams prm;
    prm.window = a->window;
    prm.rebuild_from_box = a->rebuild_from_box != 0;
    auto actions = actions_at(a->actions, a->horizon, a->m);
    SplitPlan plan;
    plan.counts.assign(a->counts, a->counts + a->n);
    auto hull = reach_with_splitting([&](const Box& b) { return dt_reach(sys, b, actions, prm); },
                                     box_at(a->x0_lo, a->x0_hi, a->n), plan);
    for (int k = 0; k < hull.steps(); ++k)
      for (int d = 0; d < a->n; ++d) {
        lo[static_cast<size_t>(k) * a->n + d] = hull.boxes[static_cast<size_t>(k)][d].lo;
        hi[static_cast<size_t>(k) * a->n + d] = hull.boxes[static_cast<size_t>(k)][d].hi;
      }
    *n_boxes = hull.steps();
    *failed_step = hull.failed_step;
  } catch (const std::exception&) {
    return REACH_E_INVALID_ARGUMENT;
  }
  return REACH_OK;
}

// reach::grad_tube_volume (refine.hpp:263-311); REACH_E_INVALID_ARGUMENT where it throws.
int ref_grad_tube_volume(const reach_net_desc* desc, const reach_dt_args* a, int32_t target, int32_t method,
                         double* grad, int32_t* subgradient) {
  try {
    DTSystem<double> sys = make_sys(desc, a->n, a->m);
    DTReachParams prm;
    prm.window = a->window;
    prm.rebuild_from_box = a->rebuild_from_box != 0;
    const GradTarget t = target == 0 ? GradTarget::x0_center : target == 1 ? GradTarget::actions : GradTarget::weights;
    const GradMethod me = method == 0 ? GradMethod::forward_dual : GradMethod::finite_difference;
    Gradient g = grad_tube_volume(sys, box_at(a->x0_lo, a->x0_hi, a->n), actions_at(a->actions, a->horizon, a->m), t,
                                  me, prm);
    std::copy(g.g.begin(), g.g.end(), grad);
    if (subgradient) *subgradient = g.subgradient ? 1 : 0;
  } catch (const std::exception&) {
    return REACH_E_INVALID_ARGUMENT;
  }
  return REACH_OK;
}

int ref_hardware_threads(void) { return hardware_threads(); }

}  // extern "C"

namespace {

// DT closed loop: the reference has no driver for it; this
// composes reference functions only, mirroring cl_reach's stacking
// (closed_loop.hpp:118-153) on a DT one-step network: u = ctl_crown(x_tm, ctl)
// (neural.hpp:418), [x; u] over the shared variables with the control remainder
// as a fresh block (no fold on the stacked state), certify_tm_input(dyn, .),
// then dt_reach's re-seed / fold_overflow / symbolic_box (dt_reach.hpp:69-100).
ReachTube<double> dt_closed_loop(const MLPNet<double>& dyn, const MLPNet<double>& ctl, int n, const Box& x0, int H,
                                 int window, bool rebuild) {
  const int l = ctl.output_dim();
  ReachTube<double> tube;
  tube.push(x0, 0.0, 0.0);
  SymbolicState<double> sym = init_symbolic_state(x0, window);
  for (int k = 0; k < H; ++k) {
    LinearTM<double> x_tm = symbolic_seed(sym);
    LinearTM<double> u_tm;
    try {
      u_tm = ctl_crown(x_tm, ctl, Vec<double>{});
    } catch (const std::exception& e) {
      tube.mark_failed(k, std::string("controller certification failed: ") + e.what());
      return tube;
    }
    if (!u_tm.remainder.finite() || u_tm.remainder.diverged) {
      tube.mark_failed(k, "controller certification diverged");
      return tube;
    }
    const int nz = x_tm.nz(), p0 = sym.g0.cols;
    SymbolicState<double> aug;
    aug.window = window;
    aug.c = Vec<double>(static_cast<size_t>(n + l));
    aug.g0 = Mat<double>(n + l, p0);
    Mat<double> fresh(n + l, n + l);
    for (int d = 0; d < n; ++d) {
      aug.c[static_cast<size_t>(d)] = x_tm.c[static_cast<size_t>(d)] + x_tm.remainder[d].mid();
      for (int j = 0; j < p0; ++j) aug.g0(d, j) = x_tm.A(d, j);
      fresh(d, d) = x_tm.remainder[d].rad();
    }
    for (int d = 0; d < l; ++d) {
      aug.c[static_cast<size_t>(n + d)] = u_tm.c[static_cast<size_t>(d)] + u_tm.remainder[d].mid();
      for (int j = 0; j < p0; ++j) aug.g0(n + d, j) = u_tm.A(d, j);
      fresh(n + d, n + d) = u_tm.remainder[d].rad();
    }
    int off = p0;
    for (const auto& q : sym.queue) {
      Mat<double> nq(n + l, q.cols);
      for (int j = 0; j < q.cols; ++j) {
        for (int d = 0; d < n; ++d) nq(d, j) = x_tm.A(d, off + j);
        for (int d = 0; d < l; ++d) nq(n + d, j) = u_tm.A(d, off + j);
      }
      aug.queue.push_back(std::move(nq));
      off += q.cols;
    }
    (void)nz;
    aug.queue.push_back(std::move(fresh));
    LinearTM<double> xu = symbolic_seed(aug);
    LinearTM<double> out;
    try {
      out = certify_tm_input(dyn, xu);
    } catch (const std::exception& e) {
      tube.mark_failed(k, e.what());
      return tube;
    }
    if (!out.remainder.finite() || out.remainder.diverged) {
      tube.mark_failed(k, "diverged certification");
      return tube;
    }
    SymbolicState<double> next;
    next.window = window;
    next.c = Vec<double>(static_cast<size_t>(n));
    next.g0 = Mat<double>(n, p0);
    for (int i = 0; i < n; ++i) {
      next.c[static_cast<size_t>(i)] = out.c[static_cast<size_t>(i)] + out.remainder[i].mid();
      for (int j = 0; j < p0; ++j) next.g0(i, j) = out.A(i, j);
    }
    off = p0;
    for (const auto& q : aug.queue) {
      Mat<double> nq(n, q.cols);
      for (int i = 0; i < n; ++i)
        for (int j = 0; j < q.cols; ++j) nq(i, j) = out.A(i, off + j);
      next.queue.push_back(std::move(nq));
      off += q.cols;
    }
    Mat<double> fr(n, n);
    for (int i = 0; i < n; ++i) fr(i, i) = out.remainder[i].rad();
    next.queue.push_back(std::move(fr));
    fold_overflow(next);
    sym = std::move(next);
    Box box = symbolic_box(sym);
    const double t = static_cast<double>(k + 1);
    tube.push(box, t, t);
    if (box.diverged) {
      tube.mark_failed(k, "diverged box");
      return tube;
    }
    if (rebuild) sym = init_symbolic_state(box, window);
  }
  return tube;
}

int32_t cl_status_of(const ReachTube<double>& t) {
  if (t.failure_reason == "controller certification failed: relax_activation: non-finite preactivation")
    return REACH_TUBE_CTL_FAILED;
  if (t.failure_reason == "controller certification diverged") return REACH_TUBE_CTL_DIVERGED;
  return status_of(t);
}

}  // namespace

extern "C" {

int ref_dtcl_batch(const reach_net_desc* dyn_desc, const reach_net_desc* ctl_desc, const reach_dt_args* a,
                   const reach_tube_out* out, int32_t threads) {
  try {
    MLPNet<double> dyn = net_from_desc(dyn_desc), ctl = net_from_desc(ctl_desc);
    const int H = a->horizon, n = a->n;
    parallel_for(
        a->batch,
        [&](int b) {
          ReachTube<double> tube;
          try {
            tube = dt_closed_loop(dyn, ctl, n,
                                  box_at(a->x0_lo + static_cast<size_t>(b) * n, a->x0_hi + static_cast<size_t>(b) * n, n),
                                  H, a->window, a->rebuild_from_box != 0);
          } catch (const std::exception& e) {
            tube.mark_failed(0, e.what());
          }
          out->n_boxes[b] = tube.steps();
          out->failed_step[b] = tube.failed_step;
          out->status[b] = cl_status_of(tube);
          for (int k = 0; k < tube.steps(); ++k)
            for (int d = 0; d < n; ++d) {
              size_t o = (static_cast<size_t>(b) * (H + 1) + k) * n + d;
              out->lo[o] = tube.boxes[static_cast<size_t>(k)][d].lo;
              out->hi[o] = tube.boxes[static_cast<size_t>(k)][d].hi;
            }
        },
        threads);
  } catch (const std::exception&) {
    return REACH_E_INVALID_ARGUMENT;
  }
  return REACH_OK;
}

}  // extern "C"

namespace {

PlanProblem problem_from(const reach_net_desc* desc, const reach_plan_problem* p) {
  PlanProblem prob;
  prob.sys = make_sys(desc, p->n, p->m);
  prob.x_goal.assign(p->x_goal, p->x_goal + p->n);
  prob.q_weights.assign(p->q_weights, p->q_weights + p->n);
  prob.r_weights.assign(p->r_weights, p->r_weights + p->m);
  for (int c = 0; c < p->n_constraints; ++c) {
    const reach_constraint& k = p->constraints[c];
    Constraint con;
    con.type = static_cast<Constraint::Type>(k.type);
    con.dims.assign(k.dims, k.dims + k.n_dims);
    const int kk = k.n_dims > 0 ? k.n_dims : p->n;
    if (k.a) con.a.assign(k.a, k.a + kk);
    con.b = k.b;
    if (k.center) con.center.assign(k.center, k.center + kk);
    con.radius = k.radius;
    if (k.lo) con.lo.assign(k.lo, k.lo + kk);
    if (k.hi) con.hi.assign(k.hi, k.hi + kk);
    con.vmax = k.vmax;
    prob.constraints.push_back(con);
  }
  prob.penalty = p->penalty;
  prob.diverged_margin = p->diverged_margin;
  prob.horizon = p->horizon;
  prob.u_lo.assign(p->u_lo, p->u_lo + p->m);
  prob.u_hi.assign(p->u_hi, p->u_hi + p->m);
  prob.eps = p->eps;
  prob.dt_prm.window = p->window;
  prob.dt_prm.rebuild_from_box = p->rebuild_from_box != 0;
  return prob;
}

}  // namespace

extern "C" {

// plan_eval (mpc.hpp:158-202) per candidate inside the reference parallel_for.
int ref_plan_eval_batch(const reach_net_desc* desc, const reach_plan_problem* p, const double* x0, int32_t batch,
                        const double* actions, double* objective, int32_t* diverged, int32_t threads) {
  try {
    PlanProblem prob = problem_from(desc, p);
    prob.validate();
    Vec<double> x(x0, x0 + p->n);
    const int H = p->horizon, m = p->m;
    parallel_for(
        batch,
        [&](int b) {
          auto ev = plan_eval(prob, x, actions_at(actions + static_cast<size_t>(b) * H * m, H, m));
          objective[b] = ev.objective;
          diverged[b] = ev.diverged ? 1 : 0;
        },
        threads);
  } catch (const std::exception&) {
    return REACH_E_INVALID_ARGUMENT;
  }
  return REACH_OK;
}

// grad_forward (refine.hpp:186-207) of plan_objective (mpc.hpp:204-208) -- the
// gradient plan_cem's refinement takes (mpc.hpp:339-346).  Returns 1 where the
// reference throws (non-finite objective or derivative).
int ref_plan_objective_grad(const reach_net_desc* desc, const reach_plan_problem* p, const double* x0,
                            const double* actions, double* grad) {
  try {
    PlanProblem prob = problem_from(desc, p);
    const int h = p->horizon, m = p->m;
    Vec<double> x(x0, x0 + p->n);
    auto objective = [&](const auto& q) {
      using S = typename std::decay_t<decltype(q)>::value_type;
      std::vector<Vec<S>> acts(static_cast<size_t>(h));
      for (int t = 0; t < h; ++t)
        acts[static_cast<size_t>(t)] =
            Vec<S>(q.begin() + static_cast<long>(t) * m, q.begin() + static_cast<long>(t + 1) * m);
      return plan_objective(prob, x, acts);
    };
    Vec<double> flat(actions, actions + static_cast<size_t>(h) * m);
    Gradient g = grad_forward(objective, flat);
    for (size_t j = 0; j < g.g.size(); ++j) grad[j] = g.g[j];
  } catch (const std::exception&) {
    return 1;
  }
  return REACH_OK;
}

// plan_cem (mpc.hpp:258-368), the reference driver itself (its own parallel_for).
int ref_plan_cem_ex(const reach_net_desc* desc, const reach_plan_problem* p, const reach_sampler_config* c,
                    const double* x0, double* best_actions, double* objective, double* best_history,
                    int32_t* best_effort, int32_t* refined);
int ref_plan_cem(const reach_net_desc* desc, const reach_plan_problem* p, const reach_sampler_config* c,
                 const double* x0, double* best_actions, double* objective, double* best_history,
                 int32_t* best_effort) {
  int32_t refined = 0;
  return ref_plan_cem_ex(desc, p, c, x0, best_actions, objective, best_history, best_effort, &refined);
}

int ref_plan_cem_ex(const reach_net_desc* desc, const reach_plan_problem* p, const reach_sampler_config* c,
                    const double* x0, double* best_actions, double* objective, double* best_history,
                    int32_t* best_effort, int32_t* refined) {
  try {
    PlanProblem prob = problem_from(desc, p);
    SamplerConfig cfg;
    cfg.population = c->population;
    cfg.elite_frac = c->elite_frac;
    cfg.iterations = c->iterations;
    cfg.init_std = c->init_std;
    cfg.smoothing = c->smoothing;
    cfg.refine_iters = c->refine_iters;
    cfg.seed = c->seed;
    auto res = plan_cem(prob, cfg, Vec<double>(x0, x0 + p->n));
    for (int t = 0; t < p->horizon; ++t)
      for (int j = 0; j < p->m; ++j) best_actions[t * p->m + j] = res.actions[static_cast<size_t>(t)][static_cast<size_t>(j)];
    *objective = res.objective;
    for (size_t i = 0; i < res.best_history.size(); ++i) best_history[i] = res.best_history[i];
    *best_effort = res.best_effort ? 1 : 0;
    *refined = res.refined ? 1 : 0;
  } catch (const std::exception&) {
    return REACH_E_INVALID_ARGUMENT;
  }
  return REACH_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Continuous-time closed loop (cl_reach, closed_loop.hpp:76-182) with the
// quadrotor plant augmented by udot = 0 rows (make_augmented_field,
// fields.hpp:96-128 -- exactly the CLI's `make_augmented("quadrotor")`,
// reach_cli.cpp:125-131), and reach_with_splitting over it (refine.hpp:121-160).
namespace {

ClosedLoopSpec<double> cl_spec_from(const reach_net_desc* ctl_desc, const reach_cl_spec* sp) {
  if (sp->plant != REACH_PLANT_QUADROTOR) throw std::invalid_argument("unknown plant");
  QuadrotorParams prm;
  prm.mass = sp->plant_params[0];
  prm.gravity = sp->plant_params[1];
  prm.jx = sp->plant_params[2];
  prm.jy = sp->plant_params[3];
  prm.jz = sp->plant_params[4];
  ClosedLoopSpec<double> spec;
  spec.n = sp->n;
  spec.l = sp->l;
  spec.ctl_steps = sp->ctl_steps;
  spec.k_atomic = sp->k_atomic;
  spec.controller = net_from_desc(ctl_desc);
  auto plant = [prm](const auto& x, const auto& u, auto& dx) { quadrotor_ode(x, u, prm, dx); };
  spec.dynamics = make_augmented_field<double>(sp->n, sp->l, plant);
  for (int i = 0; sp->ref_dim > 0 && i < sp->ctl_steps; ++i)
    spec.y_ref.emplace_back(sp->y_ref + static_cast<size_t>(i) * sp->ref_dim,
                            sp->y_ref + static_cast<size_t>(i + 1) * sp->ref_dim);
  spec.fp.h = sp->fp.h;
  spec.fp.steps = sp->fp.steps;
  spec.fp.order = sp->fp.order;
  spec.fp.eps_init = sp->fp.eps_init;
  spec.fp.refine_rounds = sp->fp.refine_rounds;
  spec.fp.enlargement = sp->fp.enlargement;
  spec.fp.max_enlargements = sp->fp.max_enlargements;
  spec.fp.window = sp->fp.window;
  spec.intervalize_boundary = sp->intervalize_boundary != 0;
  return spec;
}

int32_t ct_status_of(const ReachTube<double>& t) {
  if (!t.diverged && t.failed_step < 0) return REACH_TUBE_OK;
  const std::string& r = t.failure_reason;
  if (r == "remainder not contractive after max enlargements (reduce h)") return REACH_TUBE_REMAINDER;
  if (r == "poly_picard: non-finite coefficients") return REACH_TUBE_PICARD_NONFINITE;
  if (r == "tme_inv: range contains zero") return REACH_TUBE_TME_INV;
  return cl_status_of(t);
}

void put_tube(const ReachTube<double>& t, int na, int T, double* lo, double* hi, int32_t* nb, int32_t* fs,
              int32_t* st) {
  for (int k = 0; k < t.steps() && k < T; ++k)
    for (int d = 0; d < na; ++d) {
      lo[static_cast<size_t>(k) * na + d] = t.boxes[static_cast<size_t>(k)][d].lo;
      hi[static_cast<size_t>(k) * na + d] = t.boxes[static_cast<size_t>(k)][d].hi;
    }
  *nb = t.steps();
  *fs = t.failed_step;
  *st = ct_status_of(t);
}

}  // namespace

extern "C" {

// cl_reach per initial box (parallel_for over the batch, like dt_reach_batch).
int ref_cl_batch(const reach_net_desc* ctl_desc, const reach_cl_spec* sp, int32_t batch, const double* x0_lo,
                 const double* x0_hi, const reach_tube_out* out, int32_t threads) {
  try {
    ClosedLoopSpec<double> spec = cl_spec_from(ctl_desc, sp);
    const int n = sp->n, na = sp->n + sp->l, T = 1 + sp->ctl_steps * sp->k_atomic;
    parallel_for(
        batch,
        [&](int b) {
          ReachTube<double> t;
          try {
            t = cl_reach(spec, box_at(x0_lo + static_cast<size_t>(b) * n, x0_hi + static_cast<size_t>(b) * n, n));
          } catch (const std::exception& e) {
            t = ReachTube<double>();
            t.mark_failed(0, e.what());
          }
          put_tube(t, na, T, out->lo + static_cast<size_t>(b) * T * na, out->hi + static_cast<size_t>(b) * T * na,
                   out->n_boxes + b, out->failed_step + b, out->status + b);
        },
        threads);
  } catch (const std::exception&) {
    return REACH_E_INVALID_ARGUMENT;
  }
  return REACH_OK;
}

// reach_with_splitting(cl_reach, x0, plan).  Full range and threads == 0: the
// reference driver verbatim; otherwise the same pieces on parts [begin, end).
int ref_cl_split_hull(const reach_net_desc* ctl_desc, const reach_cl_spec* sp, const reach_cl_split_args* a,
                      const reach_hull_out* out, int32_t threads) {
  try {
    ClosedLoopSpec<double> spec = cl_spec_from(ctl_desc, sp);
    const int n = sp->n, na = sp->n + sp->l;
    Box x0 = box_at(a->x0_lo, a->x0_hi, n);
    SplitPlan plan;
    plan.counts.assign(a->counts, a->counts + n);
    const long long total = plan.total_parts();
    long long begin = a->part_begin, end = a->part_end <= 0 ? total : a->part_end;
    if (begin < 0 || begin >= end || end > total) return REACH_E_INVALID_ARGUMENT;
    auto engine = [&](const Box& b) { return cl_reach(spec, b); };
    if (begin == 0 && end == total && threads == 0) {
      ReachTube<double> hull = reach_with_splitting(engine, x0, plan);
      for (int k = 0; k < hull.steps(); ++k) {
        for (int d = 0; d < na; ++d) {
          out->lo[static_cast<size_t>(k) * na + d] = hull.boxes[static_cast<size_t>(k)][d].lo;
          out->hi[static_cast<size_t>(k) * na + d] = hull.boxes[static_cast<size_t>(k)][d].hi;
        }
        out->box_diverged[k] = hull.boxes[static_cast<size_t>(k)].diverged ? 1 : 0;
      }
      out->n_boxes[0] = hull.steps();
      // the reference reports (failed_step, "sub-box i: reason"); rebuild the key
      int64_t key = std::numeric_limits<int64_t>::max();
      if (hull.diverged) {
        size_t colon = hull.failure_reason.find(':');
        long long part = std::stoll(hull.failure_reason.substr(7, colon - 7));
        ReachTube<double> t;
        t.mark_failed(hull.failed_step, hull.failure_reason.substr(colon + 2));
        key = (static_cast<int64_t>(hull.failed_step) << 40) | (static_cast<int64_t>(part) << 8) |
              static_cast<int64_t>(ct_status_of(t) & 0xff);
      }
      out->fail_key[0] = key;
      return REACH_OK;
    }
    auto parts = split_box(x0, plan);
    const int count = static_cast<int>(end - begin);
    std::vector<ReachTube<double>> subs(static_cast<size_t>(count));
    parallel_for(
        count,
        [&](int i) {
          try {
            subs[static_cast<size_t>(i)] = engine(parts[static_cast<size_t>(begin + i)]);
          } catch (const std::exception& e) {
            subs[static_cast<size_t>(i)].mark_failed(0, e.what());
          }
        },
        threads);
    int steps = subs.front().steps();
    int64_t key = std::numeric_limits<int64_t>::max();
    for (int i = 0; i < count; ++i) {
      const auto& s = subs[static_cast<size_t>(i)];
      steps = std::min(steps, s.steps());
      if (s.diverged) {
        int fs = s.failed_step >= 0 ? s.failed_step : s.steps();
        int64_t k = (static_cast<int64_t>(fs) << 40) | (static_cast<int64_t>(begin + i) << 8) |
                    static_cast<int64_t>(ct_status_of(s) & 0xff);
        key = std::min(key, k);
      }
    }
    for (int k = 0; k < steps; ++k) {
      Box b = subs.front().boxes[static_cast<size_t>(k)];
      for (int i = 1; i < count; ++i) b = box_hull(b, subs[static_cast<size_t>(i)].boxes[static_cast<size_t>(k)]);
      for (int d = 0; d < na; ++d) {
        out->lo[static_cast<size_t>(k) * na + d] = b[d].lo;
        out->hi[static_cast<size_t>(k) * na + d] = b[d].hi;
      }
      out->box_diverged[k] = b.diverged ? 1 : 0;
    }
    out->n_boxes[0] = steps;
    out->fail_key[0] = key;
  } catch (const std::exception&) {
    return REACH_E_INVALID_ARGUMENT;
  }
  return REACH_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// ct_reach (flowpipe_ct.hpp:428-458) with the analytic fields of fields.hpp.
namespace {
VectorField<double> field_from(const reach_field_desc* f) {
  switch (f->kind) {
    case REACH_FIELD_ZERO: return zero_field<double>(f->n);
    case REACH_FIELD_DIAG_LINEAR: return diag_linear_field<double>(std::vector<double>(f->params, f->params + f->n));
    case REACH_FIELD_ROTATION: return rotation_field<double>(f->params[0]);
    case REACH_FIELD_QUADROTOR: {
      QuadrotorParams prm;
      prm.mass = f->params[0];
      prm.gravity = f->params[1];
      prm.jx = f->params[2];
      prm.jy = f->params[3];
      prm.jz = f->params[4];
      return quadrotor_field<double>(prm, Vec<double>(f->params + 5, f->params + 9));
    }
  }
  throw std::invalid_argument("unknown field");
}
}  // namespace

extern "C" {
int ref_ct_batch(const reach_field_desc* fd, const reach_flowpipe_params* fp, int32_t batch, const double* x0_lo,
                 const double* x0_hi, const reach_tube_out* out, int32_t threads) {
  try {
    VectorField<double> f = field_from(fd);
    FlowpipeParams prm;
    prm.h = fp->h;
    prm.steps = fp->steps;
    prm.order = fp->order;
    prm.eps_init = fp->eps_init;
    prm.refine_rounds = fp->refine_rounds;
    prm.enlargement = fp->enlargement;
    prm.max_enlargements = fp->max_enlargements;
    prm.window = fp->window;
    const int n = fd->n, T = 1 + fp->steps;
    parallel_for(
        batch,
        [&](int b) {
          ReachTube<double> t;
          try {
            t = ct_reach(f, box_at(x0_lo + static_cast<size_t>(b) * n, x0_hi + static_cast<size_t>(b) * n, n), prm);
          } catch (const std::exception& e) {
            t = ReachTube<double>();
            t.mark_failed(0, e.what());
          }
          put_tube(t, n, T, out->lo + static_cast<size_t>(b) * T * n, out->hi + static_cast<size_t>(b) * T * n,
                   out->n_boxes + b, out->failed_step + b, out->status + b);
        },
        threads);
  } catch (const std::exception&) {
    return REACH_E_INVALID_ARGUMENT;
  }
  return REACH_OK;
}
}  // extern "C"

extern "C" {
// reach_with_splitting(ct_reach, x0, plan) -- the CLI's `split` path (reach_cli.cpp:200-211).
int ref_ct_split_hull(const reach_field_desc* fd, const reach_flowpipe_params* fp, const reach_cl_split_args* a,
                      const reach_hull_out* out, int32_t threads) {
  try {
    VectorField<double> f = field_from(fd);
    FlowpipeParams prm;
    prm.h = fp->h;
    prm.steps = fp->steps;
    prm.order = fp->order;
    prm.eps_init = fp->eps_init;
    prm.refine_rounds = fp->refine_rounds;
    prm.enlargement = fp->enlargement;
    prm.max_enlargements = fp->max_enlargements;
    prm.window = fp->window;
    const int n = fd->n;
    Box x0 = box_at(a->x0_lo, a->x0_hi, n);
    SplitPlan plan;
    plan.counts.assign(a->counts, a->counts + n);
    const long long total = plan.total_parts();
    long long begin = a->part_begin, end = a->part_end <= 0 ? total : a->part_end;
    if (begin < 0 || begin >= end || end > total) return REACH_E_INVALID_ARGUMENT;
    auto engine = [&](const Box& b) { return ct_reach(f, b, prm); };
    auto parts = split_box(x0, plan);
    const int count = static_cast<int>(end - begin);
    std::vector<ReachTube<double>> subs(static_cast<size_t>(count));
    parallel_for(
        count,
        [&](int i) {
          try {
            subs[static_cast<size_t>(i)] = engine(parts[static_cast<size_t>(begin + i)]);
          } catch (const std::exception& e) {
            subs[static_cast<size_t>(i)].mark_failed(0, e.what());
          }
        },
        threads);
    int steps = subs.front().steps();
    int64_t key = std::numeric_limits<int64_t>::max();
    for (int i = 0; i < count; ++i) {
      const auto& s = subs[static_cast<size_t>(i)];
      steps = std::min(steps, s.steps());
      if (s.diverged) {
        int fs = s.failed_step >= 0 ? s.failed_step : s.steps();
        int64_t k = (static_cast<int64_t>(fs) << 40) | (static_cast<int64_t>(begin + i) << 8) |
                    static_cast<int64_t>(ct_status_of(s) & 0xff);
        key = std::min(key, k);
      }
    }
    for (int k = 0; k < steps; ++k) {
      Box b = subs.front().boxes[static_cast<size_t>(k)];
      for (int i = 1; i < count; ++i) b = box_hull(b, subs[static_cast<size_t>(i)].boxes[static_cast<size_t>(k)]);
      for (int d = 0; d < n; ++d) {
        out->lo[static_cast<size_t>(k) * n + d] = b[d].lo;
        out->hi[static_cast<size_t>(k) * n + d] = b[d].hi;
      }
      out->box_diverged[k] = b.diverged ? 1 : 0;
    }
    out->n_boxes[0] = steps;
    out->fail_key[0] = key;
  } catch (const std::exception&) {
    return REACH_E_INVALID_ARGUMENT;
  }
  return REACH_OK;
}
}  // extern "C"

// reach::mpc_run (mpc.hpp:425-495) with the CLI's simulator (the model's own forward,
// reach_cli.cpp:445-449) and the CSV log (MPCResult::log_to_csv) written to csv[csv_cap].
extern "C" int ref_mpc_run(const reach_net_desc* desc, const reach_plan_problem* p, const reach_sampler_config* c,
                           const reach_mpc_config* mc, const double* x0, int32_t* success, int32_t* violated,
                           int32_t* steps_used, double* final_state, char* csv, int32_t csv_cap) {
  try {
    PlanProblem prob = problem_from(desc, p);
    SamplerConfig cfg;
    cfg.population = c->population;
    cfg.elite_frac = c->elite_frac;
    cfg.iterations = c->iterations;
    cfg.init_std = c->init_std;
    cfg.smoothing = c->smoothing;
    cfg.refine_iters = c->refine_iters;
    cfg.seed = c->seed;
    MPCConfig m;
    m.replan_period = mc->replan_period;
    m.total_steps = mc->total_steps;
    m.dist_action = mc->dist_action;
    m.dist_state = mc->dist_state;
    m.goal_dims.assign(mc->goal_dims, mc->goal_dims + mc->n_goal_dims);
    m.goal_radius = mc->goal_radius;
    m.seed = mc->seed;
    auto sim = [&](const Vec<double>& x, const Vec<double>& u) {
      Vec<double> in = x;
      in.insert(in.end(), u.begin(), u.end());
      return prob.sys.step.forward(in);
    };
    auto res = mpc_run(prob, cfg, m, sim, Vec<double>(x0, x0 + p->n));
    *success = res.success ? 1 : 0;
    *violated = res.violated ? 1 : 0;
    *steps_used = res.steps_used;
    std::copy(res.final_state.begin(), res.final_state.end(), final_state);
    const std::string s = res.log_to_csv();
    if (static_cast<int32_t>(s.size()) + 1 > csv_cap) return REACH_E_INVALID_ARGUMENT;
    std::memcpy(csv, s.c_str(), s.size() + 1);
  } catch (const std::exception&) {
    return REACH_E_INVALID_ARGUMENT;
  }
  return REACH_OK;
}

// The reference CLI's refine objective (reach_cli.cpp:293-341): gradient_refine of
// tube_volume(dt_reach(box_from_center(c, eps), acts)) over the centre (target 0) or the actions (1).
extern "C" int ref_refine_tube_volume(const reach_net_desc* desc, int32_t n, int32_t m, int32_t horizon,
                                      const double* center, double eps, const double* actions, int32_t target,
                                      const double* lo, const double* hi, int32_t iters, double* x,
                                      double* initial_objective, double* objective, int32_t* progressed,
                                      int32_t* subgradient, int32_t* accepted_steps) {
  try {
    DTSystem<double> sys = make_sys(desc, n, m);
    Vec<double> cen(center, center + n);
    auto f = [&](const auto& p) {
      using S = typename std::decay_t<decltype(p)>::value_type;
      DTSystem<S> s;
      s.step = net_cast<S>(sys.step);
      s.n = n;
      s.m = m;
      Vec<S> c = to_scalar<S>(cen);
      std::vector<Vec<S>> acts(static_cast<size_t>(horizon), Vec<S>(static_cast<size_t>(m), S(0.0)));
      for (int t = 0; t < horizon; ++t)
        for (int j = 0; j < m; ++j) acts[static_cast<size_t>(t)][static_cast<size_t>(j)] = S(actions[t * m + j]);
      if (target == 0) {
        c.assign(p.begin(), p.end());
      } else {
        for (int t = 0; t < horizon; ++t)
          acts[static_cast<size_t>(t)] =
              Vec<S>(p.begin() + static_cast<long>(t) * m, p.begin() + static_cast<long>(t + 1) * m);
      }
      return tube_volume(dt_reach(s, box_from_center(c, S(eps)), acts));
    };
    const size_t d = target == 0 ? static_cast<size_t>(n) : static_cast<size_t>(horizon) * m;
    RefineParams rp;
    rp.iters = iters;
    auto res = gradient_refine(f, Vec<double>(x, x + d), Vec<double>(lo, lo + d), Vec<double>(hi, hi + d), rp);
    std::copy(res.x.begin(), res.x.end(), x);
    *initial_objective = res.initial_objective;
    *objective = res.objective;
    *progressed = res.progressed ? 1 : 0;
    *subgradient = res.subgradient ? 1 : 0;
    *accepted_steps = res.accepted_steps;
  } catch (const std::invalid_argument&) {
    return REACH_E_INVALID_ARGUMENT;
  } catch (const std::exception&) {
    return REACH_E_NONFINITE;
  }
  return REACH_OK;
}

// reach::reach_loss (training.hpp:99-126) and its grad_forward over net_params (the training gradient).
extern "C" int ref_reach_loss(const reach_net_desc* desc, int32_t n, int32_t m, int32_t t_h, int32_t M,
                              const double* x0s, const double* actions, double eps, double cap, int32_t window,
                              int32_t rebuild, double* loss, double* grad, int32_t* diverged_count) {
  try {
    DTSystem<double> sys = make_sys(desc, n, m);
    std::vector<Episode> batch(static_cast<size_t>(M));
    for (int e = 0; e < M; ++e) {
      Episode& ep = batch[static_cast<size_t>(e)];
      for (int t = 0; t <= t_h; ++t) ep.states.push_back(Vec<double>(x0s + static_cast<size_t>(e) * n,
                                                                   x0s + static_cast<size_t>(e + 1) * n));
      for (int t = 0; t < t_h; ++t) {
        const double* u = actions + (static_cast<size_t>(e) * t_h + t) * m;
        ep.actions.push_back(Vec<double>(u, u + m));
      }
    }
    DTReachParams prm;
    prm.window = window;
    prm.rebuild_from_box = rebuild != 0;
    int dc = 0;
    *loss = reach_loss(sys.step, batch, eps, t_h, cap, &dc, prm);
    if (diverged_count) *diverged_count = dc;
    if (grad) {
      auto f = [&](const auto& p) {
        using S = typename std::decay_t<decltype(p)>::value_type;
        return reach_loss(net_with_params<S>(sys.step, p), batch, eps, t_h, cap, nullptr, prm);
      };
      Gradient g = grad_forward(f, net_params(sys.step));
      std::copy(g.g.begin(), g.g.end(), grad);
    }
  } catch (const std::invalid_argument&) {
    return REACH_E_INVALID_ARGUMENT;
  } catch (const std::exception&) {
    return REACH_E_NONFINITE;
  }
  return REACH_OK;
}

// reach::dt_interval_baseline (dt_reach.hpp:129-149) per sample; same layout as ref_dt_batch.
extern "C" int ref_dt_interval_baseline_batch(const reach_net_desc* desc, const reach_dt_args* a,
                                              const reach_tube_out* out) {
  try {
    DTSystem<double> sys = make_sys(desc, a->n, a->m);
    const int H = a->horizon, n = a->n, m = a->m;
    for (int b = 0; b < a->batch; ++b) {
      const double* act = a->actions_shared ? a->actions : a->actions + static_cast<size_t>(b) * H * m;
      ReachTube<double> tube = dt_interval_baseline(
          sys, box_at(a->x0_lo + static_cast<size_t>(b) * n, a->x0_hi + static_cast<size_t>(b) * n, n),
          actions_at(act, H, m));
      out->n_boxes[b] = tube.steps();
      out->failed_step[b] = tube.failed_step;
      out->status[b] = status_of(tube);
      for (int k = 0; k < tube.steps(); ++k)
        for (int d = 0; d < n; ++d) {
          size_t o = (static_cast<size_t>(b) * (H + 1) + k) * n + d;
          out->lo[o] = tube.boxes[static_cast<size_t>(k)][d].lo;
          out->hi[o] = tube.boxes[static_cast<size_t>(k)][d].hi;
        }
    }
  } catch (const std::exception&) {
    return REACH_E_INVALID_ARGUMENT;
  }
  return REACH_OK;
}

// reach::ctl_reach_loss (training.hpp:183-213) with the quadrotor plant of `sp` and FlowpipeParams
// sp->fp as fp_base; episodes: start states x0s [M][n], optional y_ref [M][t_h][ref_dim] (has_yref[e]).
extern "C" int ref_ctl_reach_loss(const reach_net_desc* ctl_desc, const reach_cl_spec* sp, int32_t M,
                                  const double* x0s, const double* yrefs, const int32_t* has_yref, int32_t ref_dim,
                                  double eps, int32_t t_h, double delta, double cap, double* loss,
                                  int32_t* diverged_count) {
  try {
    ClosedLoopSpec<double> base = cl_spec_from(ctl_desc, sp);
    QuadrotorParams prm;
    prm.mass = sp->plant_params[0];
    prm.gravity = sp->plant_params[1];
    prm.jx = sp->plant_params[2];
    prm.jy = sp->plant_params[3];
    prm.jz = sp->plant_params[4];
    auto plant = [prm](const auto& x, const auto& u, auto& dx) { quadrotor_ode(x, u, prm, dx); };
    std::vector<Episode> batch(static_cast<size_t>(M));
    for (int e = 0; e < M; ++e) {
      Episode& ep = batch[static_cast<size_t>(e)];
      Vec<double> s(x0s + static_cast<size_t>(e) * sp->n, x0s + static_cast<size_t>(e + 1) * sp->n);
      ep.states.assign(static_cast<size_t>(t_h) + 1, s);
      ep.actions.assign(static_cast<size_t>(t_h), Vec<double>(static_cast<size_t>(sp->l), 0.0));
      if (has_yref && has_yref[e])
        for (int t = 0; t < t_h; ++t) {
          const double* r = yrefs + (static_cast<size_t>(e) * t_h + t) * ref_dim;
          ep.y_ref.emplace_back(r, r + ref_dim);
        }
    }
    int dc = 0;
    *loss = ctl_reach_loss(base.controller, plant, batch, eps, t_h, sp->n, sp->l, delta, sp->k_atomic, cap, &dc,
                           base.fp);
    if (diverged_count) *diverged_count = dc;
  } catch (const std::invalid_argument&) {
    return REACH_E_INVALID_ARGUMENT;
  } catch (const std::exception&) {
    return REACH_E_NONFINITE;
  }
  return REACH_OK;
}

// ---------------------------------------------------------------------------
// Certified training (training.hpp): pred_loss with its grad_forward, and the train_dt_dyn loop,
// on reach_episode_set data (uniform episode length).
static std::vector<Episode> episodes_from(const reach_episode_set* s) {
  std::vector<Episode> out(static_cast<size_t>(s->episodes));
  for (int e = 0; e < s->episodes; ++e) {
    Episode& ep = out[static_cast<size_t>(e)];
    for (int t = 0; t <= s->length; ++t) {
      const double* x = s->states + (static_cast<size_t>(e) * (s->length + 1) + t) * s->n;
      ep.states.push_back(Vec<double>(x, x + s->n));
    }
    for (int t = 0; t < s->length; ++t) {
      const double* u = s->actions + (static_cast<size_t>(e) * s->length + t) * s->m;
      ep.actions.push_back(Vec<double>(u, u + s->m));
    }
  }
  return out;
}

extern "C" int ref_pred_loss(const reach_net_desc* desc, const reach_episode_set* b, int32_t t_h,
                             const double* weights, double* loss, double* grad) {
  try {
    MLPNet<double> net = net_from_desc(desc);
    auto batch = episodes_from(b);
    Vec<double> w(weights, weights + t_h);
    *loss = pred_loss(net, batch, t_h, w);
    if (grad) {
      auto f = [&](const auto& p) {
        using S = typename std::decay_t<decltype(p)>::value_type;
        return pred_loss(net_with_params<S>(net, p), batch, t_h, w);
      };
      Gradient g = grad_forward(f, net_params(net));
      std::copy(g.g.begin(), g.g.end(), grad);
    }
  } catch (const std::invalid_argument&) {
    return REACH_E_INVALID_ARGUMENT;
  } catch (const std::exception&) {
    return REACH_E_NONFINITE;
  }
  return REACH_OK;
}

extern "C" int ref_train_dt_dyn(const reach_net_desc* init, const reach_train_config* c, const reach_episode_set* ds,
                                double* params_out, reach_train_log_row* log, int32_t* log_rows) {
  TrainConfig cfg;
  cfg.horizon_max = c->horizon_max;
  cfg.eps0 = c->eps0;
  cfg.eps_final = c->eps_final;
  cfg.lambda = c->lambda;
  cfg.gamma = c->gamma;
  cfg.iters = c->iters;
  cfg.batch = c->batch;
  cfg.lr = c->lr;
  cfg.reach_cap = c->reach_cap;
  cfg.curriculum = c->curriculum != 0;
  cfg.seed = c->seed;
  cfg.dt_prm.window = c->window;
  cfg.dt_prm.rebuild_from_box = c->rebuild_from_box != 0;
  try {
    MLPNet<double> net = net_from_desc(init);
    TrainResult r = train_dt_dyn(net, cfg, episodes_from(ds));
    Vec<double> p = net_params(r.net);
    std::copy(p.begin(), p.end(), params_out);
    for (size_t i = 0; i < r.log.rows.size(); ++i) {
      const auto& row = r.log.rows[i];
      log[i] = reach_train_log_row{row.iter, row.t_h, row.eps, row.l_pred, row.l_reach, row.l_total,
                                   row.diverged_count};
    }
    *log_rows = static_cast<int32_t>(r.log.rows.size());
  } catch (const std::invalid_argument&) {
    return REACH_E_INVALID_ARGUMENT;
  } catch (const std::exception&) {
    return REACH_E_NONFINITE;
  }
  return REACH_OK;
}

// reach::track_loss (training.hpp:134-178) with the quadrotor plant and its grad_forward over the
// controller's net_params.
extern "C" int ref_track_loss(const reach_net_desc* ctl_desc, const double* qp, const reach_episode_set* b,
                              int32_t t_t, const double* weights, double gamma, double delta, int32_t rk4,
                              double cap, double* loss, double* grad, int32_t* blowups) {
  try {
    MLPNet<double> ctl = net_from_desc(ctl_desc);
    QuadrotorParams prm;
    prm.mass = qp[0];
    prm.gravity = qp[1];
    prm.jx = qp[2];
    prm.jy = qp[3];
    prm.jz = qp[4];
    auto batch = episodes_from(b);
    if (b->ref_dim > 0 && b->y_ref)
      for (int e = 0; e < b->episodes; ++e)
        for (int t = 0; t < b->length; ++t) {
          const double* y = b->y_ref + (static_cast<size_t>(e) * b->length + t) * b->ref_dim;
          batch[static_cast<size_t>(e)].y_ref.push_back(Vec<double>(y, y + b->ref_dim));
        }
    Vec<double> w(weights, weights + t_t);
    auto plant = [&](const auto& x, const auto& u, auto& dx) { quadrotor_ode(x, u, prm, dx); };
    int bc = 0;
    *loss = track_loss(ctl, plant, batch, t_t, w, gamma, delta, rk4, cap, &bc);
    if (blowups) *blowups = bc;
    if (grad) {
      auto f = [&](const auto& p) {
        using S = typename std::decay_t<decltype(p)>::value_type;
        return track_loss(net_with_params<S>(ctl, p), plant, batch, t_t, w, gamma, delta, rk4, cap);
      };
      Gradient g = grad_forward(f, net_params(ctl));
      std::copy(g.g.begin(), g.g.end(), grad);
    }
  } catch (const std::invalid_argument&) {
    return REACH_E_INVALID_ARGUMENT;
  } catch (const std::exception&) {
    return REACH_E_NONFINITE;
  }
  return REACH_OK;
}

// reach::ctl_reach_loss with its grad_forward over the controller's net_params (training.hpp:183-213,
// refine.hpp:186-207); episodes as ref_ctl_reach_loss.
extern "C" int ref_ctl_reach_loss_grad(const reach_net_desc* ctl_desc, const reach_cl_spec* sp, int32_t M,
                                       const double* x0s, const double* yrefs, const int32_t* has_yref,
                                       int32_t ref_dim, double eps, int32_t t_h, double delta, double cap,
                                       double* loss, double* grad, int32_t* diverged_count) {
  try {
    ClosedLoopSpec<double> base = cl_spec_from(ctl_desc, sp);
    QuadrotorParams prm;
    prm.mass = sp->plant_params[0];
    prm.gravity = sp->plant_params[1];
    prm.jx = sp->plant_params[2];
    prm.jy = sp->plant_params[3];
    prm.jz = sp->plant_params[4];
    auto plant = [prm](const auto& x, const auto& u, auto& dx) { quadrotor_ode(x, u, prm, dx); };
    std::vector<Episode> batch(static_cast<size_t>(M));
    for (int e = 0; e < M; ++e) {
      Episode& ep = batch[static_cast<size_t>(e)];
      Vec<double> s(x0s + static_cast<size_t>(e) * sp->n, x0s + static_cast<size_t>(e + 1) * sp->n);
      ep.states.assign(static_cast<size_t>(t_h) + 1, s);
      ep.actions.assign(static_cast<size_t>(t_h), Vec<double>(static_cast<size_t>(sp->l), 0.0));
      if (has_yref && has_yref[e])
        for (int t = 0; t < t_h; ++t) {
          const double* r = yrefs + (static_cast<size_t>(e) * t_h + t) * ref_dim;
          ep.y_ref.emplace_back(r, r + ref_dim);
        }
    }
    int dc = 0;
    *loss = ctl_reach_loss(base.controller, plant, batch, eps, t_h, sp->n, sp->l, delta, sp->k_atomic, cap, &dc,
                           base.fp);
    if (diverged_count) *diverged_count = dc;
    auto f = [&](const auto& p) {
      using S = typename std::decay_t<decltype(p)>::value_type;
      return ctl_reach_loss(net_with_params<S>(base.controller, p), plant, batch, eps, t_h, sp->n, sp->l, delta,
                            sp->k_atomic, cap, nullptr, base.fp);
    };
    Gradient g = grad_forward(f, net_params(base.controller));
    std::copy(g.g.begin(), g.g.end(), grad);
  } catch (const std::invalid_argument&) {
    return REACH_E_INVALID_ARGUMENT;
  } catch (const std::exception&) {
    return REACH_E_NONFINITE;
  }
  return REACH_OK;
}

// reach::train_ct_ctl (training.hpp:389-442) with the quadrotor plant.
extern "C" int ref_train_ct_ctl(const reach_net_desc* init, const reach_train_config* c, const reach_episode_set* ds,
                                const reach_cl_spec* sp, double delta, int32_t rk4, double* params_out,
                                reach_train_log_row* log, int32_t* log_rows) {
  TrainConfig cfg;
  cfg.horizon_max = c->horizon_max;
  cfg.eps0 = c->eps0;
  cfg.eps_final = c->eps_final;
  cfg.lambda = c->lambda;
  cfg.gamma = c->gamma;
  cfg.iters = c->iters;
  cfg.batch = c->batch;
  cfg.lr = c->lr;
  cfg.reach_cap = c->reach_cap;
  cfg.curriculum = c->curriculum != 0;
  cfg.seed = c->seed;
  try {
    MLPNet<double> net = net_from_desc(init);
    QuadrotorParams prm;
    prm.mass = sp->plant_params[0];
    prm.gravity = sp->plant_params[1];
    prm.jx = sp->plant_params[2];
    prm.jy = sp->plant_params[3];
    prm.jz = sp->plant_params[4];
    auto plant = [prm](const auto& x, const auto& u, auto& dx) { quadrotor_ode(x, u, prm, dx); };
    auto data = episodes_from(ds);
    if (ds->ref_dim > 0 && ds->y_ref)
      for (int e = 0; e < ds->episodes; ++e)
        for (int t = 0; t < ds->length; ++t) {
          const double* y = ds->y_ref + (static_cast<size_t>(e) * ds->length + t) * ds->ref_dim;
          data[static_cast<size_t>(e)].y_ref.push_back(Vec<double>(y, y + ds->ref_dim));
        }
    FlowpipeParams fp;
    fp.order = sp->fp.order;
    fp.eps_init = sp->fp.eps_init;
    fp.refine_rounds = sp->fp.refine_rounds;
    fp.enlargement = sp->fp.enlargement;
    fp.max_enlargements = sp->fp.max_enlargements;
    fp.window = sp->fp.window;
    TrainResult r = train_ct_ctl(net, cfg, data, plant, sp->n, sp->l, delta, sp->k_atomic, rk4, fp);
    Vec<double> p = net_params(r.net);
    std::copy(p.begin(), p.end(), params_out);
    for (size_t i = 0; i < r.log.rows.size(); ++i) {
      const auto& row = r.log.rows[i];
      log[i] = reach_train_log_row{row.iter, row.t_h, row.eps, row.l_pred, row.l_reach, row.l_total,
                                   row.diverged_count};
    }
    *log_rows = static_cast<int32_t>(r.log.rows.size());
  } catch (const std::invalid_argument&) {
    return REACH_E_INVALID_ARGUMENT;
  } catch (const std::exception&) {
    return REACH_E_NONFINITE;
  }
  return REACH_OK;
}
