"""GPU: the tensor-core precision mode (REACH_PREC_TC) of the wide DT engine -- CROWN contractions on
tcgen05.mma kind::i8 (Ozaki split, exact int32 accumulation, rigorous contraction-error bound).

Parity bar (north_star): final reachable-set bounds within rtol = 1e-5 of the fp64 oracle / reference,
|dbound| <= rtol * max(|ref|, ref box width); the measured deviation is ~1e-9.  Enclosure: >= 1e3
Monte-Carlo rollouts of the true closed loop stay inside every box (the bound inflation keeps the
result sound, so the reference tests' 1e-12 slack applies)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle_bind import oracle_dt_batch, oracle_dtcl_batch
from paper_2605_25346_b200.api import DTReachParams, DTSystem, dt_closed_loop_batch, dt_reach_batch_arrays
from paper_2605_25346_b200.workloads import c5_closed_loop, residual_relu_dynamics

RTOL = 1e-5


def rel_dev(got, exp):
    k = exp.n_boxes
    assert np.array_equal(got.n_boxes, k) and np.array_equal(got.status, exp.status)
    worst = 0.0
    for b in range(len(k)):
        e_lo, e_hi = exp.lo[b, :k[b]], exp.hi[b, :k[b]]
        g_lo, g_hi = got.lo[b, :k[b]], got.hi[b, :k[b]]
        scale = np.maximum(np.maximum(np.abs(e_lo), np.abs(e_hi)), e_hi - e_lo)
        scale = np.maximum(scale, 1e-300)
        worst = max(worst, float(np.max(np.abs(g_lo - e_lo) / scale)), float(np.max(np.abs(g_hi - e_hi) / scale)))
    return worst


def test_c5_tc_matches_oracle():
    w = c5_closed_loop(batch=3)
    got = dt_closed_loop_batch(w.dyn, w.ctl, w.n, w.x0_lo, w.x0_hi, w.horizon, precision="tc")
    exp = oracle_dtcl_batch(w.dyn, w.ctl, w.n, w.x0_lo, w.x0_hi, w.horizon)
    assert (exp.status == 0).all()
    dev = rel_dev(got, exp)
    print("C5 tc max rel dev", dev)
    assert dev <= RTOL


def test_c5_tc_enclosure_monte_carlo():
    w = c5_closed_loop(batch=2)
    t = dt_closed_loop_batch(w.dyn, w.ctl, w.n, w.x0_lo, w.x0_hi, w.horizon, precision="tc")
    rng = np.random.default_rng(7)
    for b in range(2):
        x = rng.uniform(w.x0_lo[b], w.x0_hi[b], size=(1000, w.n))
        x[:8] = np.where(rng.random((8, w.n)) < 0.5, w.x0_lo[b], w.x0_hi[b])  # corners
        x = x.T
        for k in range(1, t.n_boxes[b]):
            u = w.ctl.forward(x)
            x = w.dyn.forward(np.concatenate([x, u], axis=0))
            assert (x.T >= t.lo[b, k] - 1e-12).all() and (x.T <= t.hi[b, k] + 1e-12).all()


def test_dt_tc_small_matches_oracle():
    rng = np.random.default_rng(12)
    net = residual_relu_dynamics(rng, 6, 2, [128, 128, 128], dt=0.1)
    sys = DTSystem(net, 6, 2)
    B, H = 5, 12
    c = rng.uniform(-0.5, 0.5, size=(B, 6))
    acts = rng.uniform(-1, 1, size=(B, H, 2))
    got = dt_reach_batch_arrays(sys, c - 0.004, c + 0.004, acts, DTReachParams(), precision="tc")
    exp = oracle_dt_batch(sys, c - 0.004, c + 0.004, acts, DTReachParams())
    dev = rel_dev(got, exp)
    print("DT tc max rel dev", dev)
    assert dev <= RTOL
