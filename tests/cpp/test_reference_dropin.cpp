// The reference's own types and test-style workloads, evaluated twice: by the
// reference (reach::) and by the B200 library through the drop-in overloads
// (reach_b200::).  ReLU / identity paths must agree bit for bit (up to the
// sign of an exact zero); exits non-zero on any mismatch.
#include <cmath>
#include <cstdio>
#include <vector>

#include "reach/dt_reach.hpp"
#include "reach/refine.hpp"
#include "reach/rng.hpp"
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
  std::printf(failures ? "FAIL (%d)\n" : "OK: reference drop-in parity\n", failures);
  return failures ? 1 : 0;
}
