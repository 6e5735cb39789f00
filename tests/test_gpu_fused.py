"""GPU: the fused fp64 precision mode (REACH_PREC_FUSED) -- the exact mode's kernels with every a*b+c
contracted into one DFMA.  Not bit-identical to the reference (one rounding where it rounds twice).

Parity bar (north_star, fp64 mode): final reachable-set bounds within rtol = 1e-5 of the oracle,
|dbound| <= rtol * max(|ref|, ref box width); statuses / failure steps identical.  Enclosure: >= 1e3
Monte-Carlo rollouts of the true map stay inside every box (1e-12 slack, as the reference's tests)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from cases import cases
from cl_cases import cl_cases
from oracle_bind import oracle_dt_batch, oracle_dtcl_batch, oracle_split_hull
from paper_2605_25346_b200.api import (DTReachParams, DTSystem, SplitPlan, dt_closed_loop_batch,
                                       dt_reach_batch_arrays, reach_split_hull, split_box)
from paper_2605_25346_b200.workloads import c4_partition_sweep, c5_closed_loop, residual_relu_dynamics
from test_gpu_tcw import rel_dev

RTOL = 1e-5


def hull_rel_dev(g, e):
    k = e.n_boxes
    assert g.n_boxes == k
    scale = np.maximum(np.maximum(np.abs(e.lo[:k]), np.abs(e.hi[:k])), e.hi[:k] - e.lo[:k])
    scale = np.maximum(scale, 1e-300)
    return max(float(np.max(np.abs(g.lo[:k] - e.lo[:k]) / scale)), float(np.max(np.abs(g.hi[:k] - e.hi[:k]) / scale)))


@pytest.mark.parametrize("case", cases(), ids=lambda c: c[0])
def test_fused_dt_matches_oracle(case):
    name, sys, lo, hi, acts, prm, tanh = case
    exp = oracle_dt_batch(sys, lo, hi, acts, prm)
    got = dt_reach_batch_arrays(sys, lo, hi, acts, prm, precision="fused")
    assert np.array_equal(got.status, exp.status) and np.array_equal(got.failed_step, exp.failed_step)
    dev = rel_dev(got, exp)
    print(name, "fused max rel dev", dev)
    assert dev <= RTOL


@pytest.mark.parametrize("case", cl_cases(), ids=lambda c: c[0])
def test_fused_closed_loop_matches_oracle(case):
    name, dyn, ctl, n, lo, hi, H, prm, tanh = case
    exp = oracle_dtcl_batch(dyn, ctl, n, lo, hi, H, prm)
    got = dt_closed_loop_batch(dyn, ctl, n, lo, hi, H, prm, precision="fused")
    assert np.array_equal(got.status, exp.status)
    assert rel_dev(got, exp) <= RTOL


def test_fused_c4_hull_full_size():
    """The bench's C4 sweep (65,536 sub-boxes x 30) in the fused mode: the hull within rtol of the exact
    mode's (itself bit-identical to the oracle, tests/test_gpu_dt.py), 48 strided sub-boxes against the
    oracle, and >= 1e3 rollouts per checked sub-box inside the hull."""
    w = c4_partition_sweep()
    x0 = (w.x0_lo, w.x0_hi)
    ex = reach_split_hull(w.sys, x0, w.plan, w.actions)
    fu = reach_split_hull(w.sys, x0, w.plan, w.actions, precision="fused")
    assert fu.fail_key == ex.fail_key
    dev = hull_rel_dev(fu, ex)
    print("C4 hull fused vs exact max rel dev", dev)
    assert dev <= RTOL
    lo, hi = split_box(w.x0_lo, w.x0_hi, w.plan)
    idx = np.arange(0, lo.shape[0], lo.shape[0] // 48)[:48]
    acts = np.zeros((len(idx), w.horizon, 0))
    got = dt_reach_batch_arrays(w.sys, lo[idx], hi[idx], acts, DTReachParams(), precision="fused")
    exp = oracle_dt_batch(w.sys, lo[idx], hi[idx], acts, DTReachParams())
    assert rel_dev(got, exp) <= RTOL
    rng = np.random.default_rng(17)
    for b in idx[:4]:
        x = rng.uniform(lo[b], hi[b], size=(1000, w.sys.n))
        x[:64] = np.where(rng.random((64, w.sys.n)) < 0.5, lo[b], hi[b])
        x = x.T
        for k in range(1, fu.n_boxes):
            x = w.sys.step.forward(x)
            assert (x.T >= fu.lo[k] - 1e-12).all() and (x.T <= fu.hi[k] + 1e-12).all()


def test_fused_split_hull_matches_oracle():
    rng = np.random.default_rng(31)
    net = residual_relu_dynamics(rng, 6, 0, [128, 128, 128], dt=0.1)
    sys = DTSystem(net, 6, 0)
    c = rng.uniform(-0.5, 0.5, size=6)
    plan = SplitPlan([2, 2, 1, 2, 1, 3])
    acts = np.zeros((12, 0))
    got = reach_split_hull(sys, (c - 0.004, c + 0.004), plan, acts, DTReachParams(), precision="fused")
    exp = oracle_split_hull(sys, c - 0.004, c + 0.004, plan, acts, DTReachParams())
    assert got.fail_key == exp.fail_key
    assert hull_rel_dev(got, exp) <= RTOL


def test_fused_c5_matches_oracle_and_encloses():
    w = c5_closed_loop(batch=4)
    got = dt_closed_loop_batch(w.dyn, w.ctl, w.n, w.x0_lo, w.x0_hi, w.horizon, precision="fused")
    exp = oracle_dtcl_batch(w.dyn, w.ctl, w.n, w.x0_lo, w.x0_hi, w.horizon)
    assert (got.status == 0).all()
    assert rel_dev(got, exp) <= RTOL
    rng = np.random.default_rng(3)
    x = rng.uniform(w.x0_lo[1], w.x0_hi[1], size=(1000, w.n)).T
    for k in range(1, got.n_boxes[1]):
        u = w.ctl.forward(x)
        x = w.dyn.forward(np.concatenate([x, u], axis=0))
        assert (x.T >= got.lo[1, k] - 1e-12).all() and (x.T <= got.hi[1, k] + 1e-12).all()
