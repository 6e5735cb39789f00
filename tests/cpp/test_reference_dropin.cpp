// The reference's own types and test-style workloads, evaluated twice: by the
// reference (reach::) and by the B200 library through the drop-in overloads
// (reach_b200::).  ReLU / identity paths must agree bit for bit (up to the
// sign of an exact zero); exits non-zero on any mismatch.
#include <cmath>
#include <cstdio>
#include <vector>

#include "reach/closed_loop.hpp"
#include "reach/dt_reach.hpp"
#include "reach/fields.hpp"
#include "reach/mpc.hpp"
#include "reach/refine.hpp"
#include "reach/rng.hpp"
#include "reach/training.hpp"
#include "reach_b200_reference.hpp"

using namespace reach;

static int compare(const ReachTube<double>& a, const ReachTube<double>& b, const char* what) {
  int bad = 0;
  if (a.steps() != b.steps() || a.diverged != b.diverged || a.failed_step != b.failed_step ||
      a.failure_reason != b.failure_reason) {
    std::printf("%s: tube metadata differs (%d/%d steps, failed %d/%d, '%s'/'%s')\n", what, a.steps(), b.steps(),
                a.failed_step, b.failed_step, a.failure_reason.c_str(), b.failure_reason.c_str());
    return 1;
  }
  for (int k = 0; k < a.steps(); ++k)
    for (int d = 0; d < a.boxes[k].size(); ++d) {
      const auto& x = a.boxes[k][d];
      const auto& y = b.boxes[k][d];
      const bool same_lo = x.lo == y.lo || (std::isnan(x.lo) && std::isnan(y.lo));
      const bool same_hi = x.hi == y.hi || (std::isnan(x.hi) && std::isnan(y.hi));
      if (!same_lo || !same_hi) ++bad;
    }
  if (bad) std::printf("%s: %d interval bounds differ\n", what, bad);
  return bad;
}

int main() {
  reach_b200::Context gpu(0);
  int failures = 0;
  Rng rng(2024);
  // random ReLU nets in the shape of test_dt_reach.cpp:125-170, batched
  for (int c = 0; c < 6; ++c) {
    DTSystem<double> sys;
    sys.n = 4;
    sys.m = 2;
    sys.step = random_mlp(rng, 6, {32, 32}, 4, Act::Relu, 0.6);
    for (auto& w : sys.step.layers.back().w.a) w *= 0.3;
    std::vector<Box> x0s;
    std::vector<std::vector<Vec<double>>> seqs;
    for (int b = 0; b < 16; ++b) {
      Vec<double> cen(4), rad(4);
      for (auto& v : cen) v = rng.uniform(-0.6, 0.6);
      for (auto& v : rad) v = rng.uniform(0.01, 0.2);
      x0s.push_back(box_from_center(cen, rad));
      std::vector<Vec<double>> a;
      for (int k = 0; k < 10; ++k) a.push_back({rng.uniform(-0.5, 0.5), rng.uniform(-0.5, 0.5)});
      seqs.push_back(a);
    }
    auto ref = reach::dt_reach_batch(sys, x0s, seqs);
    auto got = reach_b200::dt_reach_batch(gpu, sys, x0s, seqs);
    for (size_t b = 0; b < ref.size(); ++b) failures += compare(ref[b], got[b], "dt_reach_batch");
  }
  // the affine-decay golden system through dt_reach
  {
    DTSystem<double> sys;
    sys.n = 2;
    sys.m = 0;
    Mat<double> w(2, 2);
    w(0, 0) = 0.5;
    w(1, 1) = 0.25;
    sys.step = affine_net(w, Vec<double>{0.25, -0.5});
    auto x0 = box_from_center<double>({0.5, 0.5}, 0.125);
    std::vector<Vec<double>> acts(8, Vec<double>{});
    failures += compare(reach::dt_reach(sys, x0, acts), reach_b200::dt_reach(gpu, sys, x0, acts), "golden");
  }
  // reach_with_splitting with the dt_reach engine
  {
    DTSystem<double> sys;
    sys.n = 3;
    sys.m = 1;
    sys.step = random_mlp(rng, 4, {48, 48}, 3, Act::Relu, 0.7);
    for (auto& w : sys.step.layers.back().w.a) w *= 0.4;
    auto x0 = box_from_center<double>({0.1, -0.2, 0.3}, 0.2);
    std::vector<Vec<double>> acts;
    for (int k = 0; k < 12; ++k) acts.push_back({rng.uniform(-0.5, 0.5)});
    SplitPlan plan;
    plan.counts = {4, 3, 5};
    auto ref = reach_with_splitting([&](const Box& b) { return reach::dt_reach(sys, b, acts); }, x0, plan);
    auto got = reach_b200::reach_with_splitting_dt(gpu, sys, x0, plan, acts);
    failures += compare(ref, got, "reach_with_splitting");
  }
  // cl_reach with the quadrotor plant and a tanh controller (test_closed_loop.cpp:236-254 shape):
  // CUDA libm + tree-reduced abs-sums, so bounds agree to rounding (rel. 1e-9), statuses exactly
  {
    QuadrotorParams prm;
    Rng crng(7788);
    ClosedLoopSpec<double> spec;
    spec.n = 12;
    spec.l = 4;
    spec.ctl_steps = 4;
    spec.k_atomic = 5;
    spec.fp.h = 0.01;
    spec.controller = random_mlp(crng, 15, {16}, 4, Act::Tanh, 0.4);
    for (auto& w : spec.controller.layers.back().w.a) w *= 0.1;
    spec.controller.layers.back().b[0] += prm.mass * prm.gravity;
    auto plant = [prm](const auto& x, const auto& u, auto& dx) { quadrotor_ode(x, u, prm, dx); };
    spec.dynamics = make_augmented_field<double>(12, 4, plant);
    spec.y_ref.assign(4, Vec<double>{0.1, 0.0, 0.0});
    Box x0(12);
    for (int d = 0; d < 12; ++d) x0[d] = {d < 3 ? -0.3 : d < 6 ? -0.05 : -0.02, d < 3 ? 0.3 : d < 6 ? 0.05 : 0.02};
    auto ref = reach::cl_reach(spec, x0);
    auto got = reach_b200::cl_reach(gpu, spec, prm, x0);
    int bad = (ref.steps() != got.steps() || ref.diverged != got.diverged || ref.failed_step != got.failed_step) ? 1 : 0;
    double worst = 0.0;
    for (int k = 0; !bad && k < ref.steps(); ++k)
      for (int d = 0; d < 16; ++d) {
        const auto& x = ref.boxes[k][d];
        const auto& y = got.boxes[k][d];
        const double scale = std::fmax(std::fmax(std::fabs(x.lo), std::fabs(x.hi)), x.hi - x.lo);
        worst = std::fmax(worst, std::fmax(std::fabs(x.lo - y.lo), std::fabs(x.hi - y.hi)) / scale);
        if (ref.t_lo[k] != got.t_lo[k] || ref.t_hi[k] != got.t_hi[k]) bad = 1;
      }
    if (bad || worst > 1e-9) {
      std::printf("cl_reach: mismatch (bad=%d, max rel diff %.3e)\n", bad, worst);
      ++failures;
    }
    SplitPlan plan;
    plan.counts = std::vector<int>(12, 1);
    plan.counts[6] = plan.counts[7] = 2;
    auto href = reach_with_splitting([&](const Box& b) { return reach::cl_reach(spec, b); }, x0, plan);
    auto hgot = reach_b200::reach_with_splitting_cl(gpu, spec, prm, x0, plan);
    double hw = 0.0;
    for (int k = 0; k < href.steps() && k < hgot.steps(); ++k)
      for (int d = 0; d < 16; ++d) {
        const auto& x = href.boxes[k][d];
        const auto& y = hgot.boxes[k][d];
        const double scale = std::fmax(std::fmax(std::fabs(x.lo), std::fabs(x.hi)), x.hi - x.lo);
        hw = std::fmax(hw, std::fmax(std::fabs(x.lo - y.lo), std::fabs(x.hi - y.hi)) / scale);
      }
    if (href.steps() != hgot.steps() || hw > 1e-9) {
      std::printf("reach_with_splitting(cl_reach): mismatch (%d/%d steps, max rel diff %.3e)\n", href.steps(),
                  hgot.steps(), hw);
      ++failures;
    }
  }
  // ct_reach of the reference's own rotation / quadrotor-hover flowpipe tests (test_flowpipe_ct.cpp:179-282)
  {
    auto rel = [](const ReachTube<double>& a, const ReachTube<double>& b) {
      if (a.steps() != b.steps() || a.diverged != b.diverged) return 1.0;
      double worst = 0.0;
      for (int k = 0; k < a.steps(); ++k)
        for (int d = 0; d < a.boxes[k].size(); ++d) {
          const auto& x = a.boxes[k][d];
          const auto& y = b.boxes[k][d];
          const double scale = std::fmax(std::fmax(std::fmax(std::fabs(x.lo), std::fabs(x.hi)), x.hi - x.lo), 1e-300);
          worst = std::fmax(worst, std::fmax(std::fabs(x.lo - y.lo), std::fabs(x.hi - y.hi)) / scale);
        }
      return worst;
    };
    FlowpipeParams prm;
    prm.h = 0.05;
    prm.steps = 60;
    auto x0 = box_from_center<double>({1.0, 0.0}, 0.1);
    double r1 = rel(reach::ct_reach(rotation_field<double>(1.0), x0, prm),
                    reach_b200::ct_reach(gpu, reach_b200::AnalyticField::rotation(1.0), x0, prm));
    QuadrotorParams qp;
    Vec<double> u = quadrotor_hover_input(qp);
    Vec<double> rad(12, 0.0);
    for (int j = 0; j < 6; ++j) rad[j] = 0.05;
    auto qx0 = box_from_center(Vec<double>(12, 0.0), rad);
    FlowpipeParams qprm;
    qprm.h = 0.01;
    qprm.steps = 100;
    double r2 = rel(reach::ct_reach(quadrotor_field<double>(qp, u), qx0, qprm),
                    reach_b200::ct_reach(gpu, reach_b200::AnalyticField::quadrotor({qp.mass, qp.gravity, qp.jx, qp.jy, qp.jz}, u),
                                         qx0, qprm));
    if (r1 > 1e-9 || r2 > 1e-9) {
      std::printf("ct_reach: max rel diff rotation %.3e quadrotor %.3e\n", r1, r2);
      ++failures;
    }
  }
  // plan_cem with the reference-default gradient refinement (refine_iters = 5) on a ReLU model with
  // every constraint type (test_mpc.cpp shape): plan, objective, history, flags and final tube bit-identical
  {
    Rng r2(77);
    PlanProblem prob;
    prob.sys.n = 3;
    prob.sys.m = 2;
    prob.sys.step = random_mlp(r2, 5, {24, 24}, 3, Act::Relu, 0.7);
    for (auto& w : prob.sys.step.layers.back().w.a) w *= 0.4;
    prob.x_goal = {0.3, -0.2, 0.1};
    prob.q_weights = {1.0, 1.0, 1.0};
    prob.r_weights = {0.05, 0.05};
    Constraint a;
    a.type = Constraint::Type::sphere_avoid;
    a.dims = {0, 2};
    a.center = {0.2, 0.1};
    a.radius = 0.1;
    Constraint b;
    b.type = Constraint::Type::box_stay_in;
    b.lo = {-1.0, -1.0, -1.0};
    b.hi = {1.0, 1.0, 1.0};
    Constraint c;
    c.type = Constraint::Type::halfspace_avoid;
    c.dims = {1};
    c.a = {1.0};
    c.b = 0.9;
    Constraint d;
    d.type = Constraint::Type::max_volume;
    d.vmax = 0.5;
    prob.constraints = {a, b, c, d};
    prob.horizon = 6;
    prob.u_lo = {-1.0, -1.0};
    prob.u_hi = {1.0, 1.0};
    prob.eps = 0.01;
    SamplerConfig cfg;
    cfg.population = 48;
    cfg.iterations = 4;
    cfg.seed = 3;
    Vec<double> x0{0.05, -0.05, 0.0};
    auto ref = reach::plan_cem(prob, cfg, x0);
    auto got = reach_b200::plan_cem(gpu, prob, cfg, x0);
    bool same = ref.actions == got.actions && ref.objective == got.objective &&
                ref.best_history == got.best_history && ref.best_effort == got.best_effort &&
                ref.refined == got.refined;
    if (!same) {
      std::printf("plan_cem: mismatch (objective %.17g / %.17g, refined %d / %d)\n", ref.objective, got.objective,
                  int(ref.refined), int(got.refined));
      ++failures;
    }
    failures += compare(ref.tube, got.tube, "plan_cem tube") ? 1 : 0;
    const double o1 = reach::plan_objective(prob, x0, ref.actions);
    const double o2 = reach_b200::plan_objective(gpu, prob, x0, ref.actions);
    if (o1 != o2) {
      std::printf("plan_objective: %.17g / %.17g\n", o1, o2);
      ++failures;
    }
  }
  // grad_tube_volume on the reference's own gradient-test shapes (test_refine.cpp:253-284): all three
  // targets, both methods, ReLU map -> bit-identical gradients and subgradient flags
  {
    Rng r3(9090);
    DTSystem<double> sys;
    sys.n = 3;
    sys.m = 2;
    sys.step = random_mlp(r3, 5, {16, 16}, 3, Act::Relu, 0.6);
    Box x0 = box_from_center<double>({0.1, 0.0, -0.2}, 0.05);
    std::vector<Vec<double>> actions;
    for (int k = 0; k < 5; ++k) actions.push_back({r3.uniform(-0.3, 0.3), r3.uniform(-0.3, 0.3)});
    for (auto t : {GradTarget::x0_center, GradTarget::actions, GradTarget::weights})
      for (auto me : {GradMethod::forward_dual, GradMethod::finite_difference}) {
        auto ref = reach::grad_tube_volume(sys, x0, actions, t, me);
        auto got = reach_b200::grad_tube_volume(gpu, sys, x0, actions, t, me);
        if (ref.g != got.g || ref.subgradient != got.subgradient) {
          std::printf("grad_tube_volume(target %d, method %d): mismatch\n", int(t), int(me));
          ++failures;
        }
      }
  }
  // mpc_run with the CLI's simulator (the model's forward) and disturbances: run log byte-identical
  {
    Rng r4(31);
    PlanProblem prob;
    prob.sys.n = 3;
    prob.sys.m = 2;
    prob.sys.step = random_mlp(r4, 5, {24, 24}, 3, Act::Relu, 0.7);
    for (auto& w : prob.sys.step.layers.back().w.a) w *= 0.4;
    prob.x_goal = {0.3, -0.2, 0.1};
    prob.q_weights = {1.0, 1.0, 1.0};
    prob.r_weights = {0.05, 0.05};
    Constraint b;
    b.type = Constraint::Type::box_stay_in;
    b.lo = {-1.0, -1.0, -1.0};
    b.hi = {1.0, 1.0, 1.0};
    prob.constraints = {b};
    prob.horizon = 5;
    prob.u_lo = {-1.0, -1.0};
    prob.u_hi = {1.0, 1.0};
    prob.eps = 0.01;
    SamplerConfig cfg;
    cfg.population = 32;
    cfg.iterations = 2;
    cfg.seed = 11;
    MPCConfig mc;
    mc.replan_period = 2;
    mc.total_steps = 6;
    mc.dist_action = 0.02;
    mc.dist_state = 0.01;
    mc.seed = 5;
    auto sim = [&](const Vec<double>& x, const Vec<double>& u) {
      Vec<double> in = x;
      in.insert(in.end(), u.begin(), u.end());
      return prob.sys.step.forward(in);
    };
    Vec<double> x0{0.05, -0.05, 0.0};
    auto ref = reach::mpc_run(prob, cfg, mc, sim, x0);
    auto got = reach_b200::mpc_run(gpu, prob, cfg, mc, sim, x0);
    if (ref.log_to_csv() != got.log_to_csv() || ref.success != got.success || ref.violated != got.violated ||
        ref.steps_used != got.steps_used || ref.final_state != got.final_state) {
      std::printf("mpc_run: mismatch\n");
      ++failures;
    }
  }
  // reach_loss and its parameter gradient (training.hpp:99-126 under grad_forward): gradient
  // bit-identical, loss within 1e-14 (CUDA log)
  {
    Rng r5(12);
    MLPNet<double> model = random_mlp(r5, 4, {16}, 2, Act::Relu, 0.6);
    std::vector<Episode> batch(3);
    for (auto& ep : batch) {
      ep.states.assign(5, Vec<double>{r5.uniform(-0.4, 0.4), r5.uniform(-0.4, 0.4)});
      for (int t = 0; t < 4; ++t) ep.actions.push_back({r5.uniform(-0.5, 0.5), r5.uniform(-0.5, 0.5)});
    }
    int d1 = 0, d2 = 0;
    const double l1 = reach::reach_loss(model, batch, 0.05, 3, 50.0, &d1);
    const double l2 = reach_b200::reach_loss(gpu, model, batch, 0.05, 3, 50.0, &d2);
    auto f = [&](const auto& p) {
      using S = typename std::decay_t<decltype(p)>::value_type;
      return reach::reach_loss(net_with_params<S>(model, p), batch, 0.05, 3, 50.0);
    };
    auto gref = grad_forward(f, net_params(model));
    auto ggot = reach_b200::reach_loss_gradient(gpu, model, batch, 0.05, 3, 50.0);
    if (std::fabs(l1 - l2) > 1e-14 * std::fabs(l1) || d1 != d2 || gref.g != ggot.g) {
      std::printf("reach_loss: mismatch (%.17g / %.17g)\n", l1, l2);
      ++failures;
    }
  }
  // dt_interval_baseline (dt_reach.hpp:129-149): bit-identical tube
  {
    Rng r6(5);
    DTSystem<double> sys;
    sys.n = 3;
    sys.m = 1;
    sys.step = random_mlp(r6, 4, {24, 24}, 3, Act::Relu, 0.6);
    Box x0 = box_from_center<double>({0.1, -0.2, 0.05}, 0.05);
    std::vector<Vec<double>> acts;
    for (int k = 0; k < 8; ++k) acts.push_back({r6.uniform(-0.5, 0.5)});
    failures += compare(reach::dt_interval_baseline(sys, x0, acts), reach_b200::dt_interval_baseline(gpu, sys, x0, acts),
                        "dt_interval_baseline") ? 1 : 0;
  }
  // ctl_reach_loss (training.hpp:183-213), quadrotor plant, tanh controller with y_ref: within 1e-12
  {
    Rng r7(3);
    QuadrotorParams qp;
    MLPNet<double> ctl = random_mlp(r7, 15, {16, 16}, 4, Act::Tanh, 0.4);
    for (auto& w : ctl.layers.back().w.a) w *= 0.1;
    ctl.layers.back().b[0] += qp.mass * qp.gravity;
    std::vector<Episode> batch(3);
    for (size_t e = 0; e < batch.size(); ++e) {
      Vec<double> x0(12, 0.0);
      for (int d = 0; d < 6; ++d) x0[d] = r7.uniform(-0.05, 0.05);
      batch[e].states.assign(4, x0);
      batch[e].actions.assign(3, Vec<double>(4, 0.0));
      if (e != 1) batch[e].y_ref.assign(3, Vec<double>{r7.uniform(-0.1, 0.1), 0.0, 0.0});
    }
    auto plant = [qp](const auto& x, const auto& u, auto& dx) { quadrotor_ode(x, u, qp, dx); };
    int d1 = 0, d2 = 0;
    const double l1 = reach::ctl_reach_loss(ctl, plant, batch, 0.01, 3, 12, 4, 0.02, 2, 40.0, &d1);
    const double l2 = reach_b200::ctl_reach_loss(gpu, ctl, qp, batch, 0.01, 3, 12, 4, 0.02, 2, 40.0, &d2);
    if (std::fabs(l1 - l2) > 1e-12 * std::fabs(l1) || d1 != d2) {
      std::printf("ctl_reach_loss: %.17g / %.17g\n", l1, l2);
      ++failures;
    }
  }
  // certified training on the device: pred_loss gradient and the whole train_dt_dyn bit-identical;
  // the ctl_reach_loss gradient (Dual through the CT engine) within 1e-9
  {
    Rng r8(21);
    MLPNet<double> model = random_mlp(r8, 4, {16, 16}, 2, Act::Relu, 0.6);
    auto step = [&](const Vec<double>& x, const Vec<double>& u) {
      Vec<double> in = x;
      in.insert(in.end(), u.begin(), u.end());
      Vec<double> y = model.forward(in);
      for (size_t i = 0; i < y.size(); ++i) y[i] = 0.5 * y[i] + 0.9 * x[i];
      return y;
    };
    auto data = make_dt_dataset(step, 2, 2, 5, 5, 0.4, 0.5, r8);
    const auto w = horizon_weights(3);
    auto f = [&](const auto& p) {
      using S = typename std::decay_t<decltype(p)>::value_type;
      return pred_loss(net_with_params<S>(model, p), data, 3, w);
    };
    auto gref = grad_forward(f, net_params(model));
    reach::Gradient ggot;
    const double lp = reach_b200::pred_loss(gpu, model, data, 3, w, &ggot);
    if (lp != pred_loss(model, data, 3, w) || gref.g != ggot.g) {
      std::printf("pred_loss: mismatch\n");
      ++failures;
    }
    TrainConfig cfg;
    cfg.horizon_max = 3;
    cfg.iters = 3;
    cfg.batch = 2;
    cfg.lambda = 0.5;
    cfg.eps0 = 0.02;
    cfg.eps_final = 0.005;
    cfg.seed = 4;
    auto tr = train_dt_dyn(model, cfg, data);
    auto tg = reach_b200::train_dt_dyn(gpu, model, cfg, data);
    if (tr.log.to_csv() != tg.log.to_csv() || net_params(tr.net) != net_params(tg.net)) {
      std::printf("train_dt_dyn: mismatch\n%s---\n%s", tr.log.to_csv().c_str(), tg.log.to_csv().c_str());
      ++failures;
    }
  }
  {
    Rng r9(3);
    QuadrotorParams qp;
    MLPNet<double> ctl = random_mlp(r9, 15, {8, 8}, 4, Act::Tanh, 0.4);
    for (auto& w : ctl.layers.back().w.a) w *= 0.1;
    ctl.layers.back().b[0] += qp.mass * qp.gravity;
    std::vector<Episode> batch(2);
    for (auto& ep : batch) {
      Vec<double> x0(12, 0.0);
      for (int d = 0; d < 6; ++d) x0[d] = r9.uniform(-0.05, 0.05);
      ep.states.assign(3, x0);
      ep.actions.assign(2, Vec<double>(4, 0.0));
      ep.y_ref.assign(2, Vec<double>{0.1, 0.0, 0.0});
    }
    auto plant = [qp](const auto& x, const auto& u, auto& dx) { quadrotor_ode(x, u, qp, dx); };
    auto f = [&](const auto& p) {
      using S = typename std::decay_t<decltype(p)>::value_type;
      return ctl_reach_loss(net_with_params<S>(ctl, p), plant, batch, 0.01, 2, 12, 4, 0.02, 2, 40.0);
    };
    auto gref = grad_forward(f, net_params(ctl));
    auto ggot = reach_b200::ctl_reach_loss_gradient(gpu, ctl, qp, batch, 0.01, 2, 12, 4, 0.02, 2, 40.0);
    double worst = 0.0, scale = 0.0;
    for (size_t j = 0; j < gref.g.size(); ++j) {
      worst = std::max(worst, std::fabs(gref.g[j] - ggot.g[j]));
      scale = std::max(scale, std::fabs(gref.g[j]));
    }
    if (gref.g.size() != ggot.g.size() || worst > 1e-9 * scale) {
      std::printf("ctl_reach_loss gradient: max err %.3g (scale %.3g)\n", worst, scale);
      ++failures;
    }
  }
  // the reference's outward-rounding mode is refused, never silently ignored
  {
    reach::ScopedOutwardRounding on(true);
    bool threw = false;
    try {
      Rng r10(1);
      DTSystem<double> sys;
      sys.n = 2;
      sys.m = 0;
      sys.step = random_mlp(r10, 2, {8}, 2, Act::Relu, 0.5);
      reach_b200::dt_reach(gpu, sys, box_from_center<double>({0.1, 0.2}, 0.05), std::vector<Vec<double>>(3));
    } catch (const std::exception&) {
      threw = true;
    }
    if (!threw) {
      std::printf("outward rounding: not refused\n");
      ++failures;
    }
  }
  std::printf(failures ? "FAIL (%d)\n" : "OK: reference drop-in parity\n", failures);
  return failures ? 1 : 0;
}
