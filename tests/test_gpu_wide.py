"""GPU parity of the wide (CTA-per-sample) kernel family.

RB_FORCE_WIDE=1 routes every DT / closed-loop / split / MPC call through the
wide family, so the whole small-shape parity suite doubles as its test; the
C5 shape (n = 72, l = 18, 3 x 256 nets) only fits the wide family.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from cases import cases
from cl_cases import cl_cases
from oracle_bind import assert_tubes_equal, oracle_dt_batch, oracle_dtcl_batch, oracle_split_hull
from paper_2605_25346_b200.api import (DTReachParams, DTSystem, SplitPlan, dt_closed_loop_batch,
                                       dt_reach_batch_arrays, reach_split_hull)
from paper_2605_25346_b200.workloads import c5_closed_loop, residual_relu_dynamics

TANH_RTOL = 1e-9


@pytest.fixture
def force_wide(monkeypatch):
    monkeypatch.setenv("RB_FORCE_WIDE", "1")


@pytest.mark.parametrize("case", cases(), ids=lambda c: c[0])
def test_wide_dt_matches_oracle(case, force_wide):
    name, sys, lo, hi, acts, prm, tanh = case
    exp = oracle_dt_batch(sys, lo, hi, acts, prm)
    got = dt_reach_batch_arrays(sys, lo, hi, acts, prm)
    assert_tubes_equal(got, exp, exact=not tanh, rtol=TANH_RTOL)


@pytest.mark.parametrize("case", cl_cases(), ids=lambda c: c[0])
def test_wide_closed_loop_matches_oracle(case, force_wide):
    name, dyn, ctl, n, lo, hi, H, prm, tanh = case
    exp = oracle_dtcl_batch(dyn, ctl, n, lo, hi, H, prm)
    got = dt_closed_loop_batch(dyn, ctl, n, lo, hi, H, prm)
    assert_tubes_equal(got, exp, exact=not tanh, rtol=TANH_RTOL)


def test_wide_split_hull_matches_oracle(force_wide):
    rng = np.random.default_rng(31)
    net = residual_relu_dynamics(rng, 6, 0, [128, 128, 128], dt=0.1)
    sys = DTSystem(net, 6, 0)
    c = rng.uniform(-0.5, 0.5, size=6)
    x0 = (c - 0.004, c + 0.004)
    plan = SplitPlan([2, 2, 1, 2, 1, 3])
    acts = np.zeros((12, 0))
    got = reach_split_hull(sys, x0, plan, acts, DTReachParams())
    exp = oracle_split_hull(sys, x0[0], x0[1], plan, acts, DTReachParams())
    assert np.array_equal(got.lo, exp.lo) and np.array_equal(got.hi, exp.hi)
    assert got.n_boxes == exp.n_boxes and got.fail_key == exp.fail_key


def test_c5_shape_matches_oracle():
    """C5: 72-D closed loop, 3x256 dynamics and controller, H = 20 (the wide family's target)."""
    w = c5_closed_loop(batch=3)
    got = dt_closed_loop_batch(w.dyn, w.ctl, w.n, w.x0_lo, w.x0_hi, w.horizon)
    exp = oracle_dtcl_batch(w.dyn, w.ctl, w.n, w.x0_lo, w.x0_hi, w.horizon)
    assert (exp.status == 0).all()
    assert_tubes_equal(got, exp, exact=True)


def test_c5_enclosure_monte_carlo():
    w = c5_closed_loop(batch=1)
    t = dt_closed_loop_batch(w.dyn, w.ctl, w.n, w.x0_lo, w.x0_hi, w.horizon)
    x = np.random.default_rng(5).uniform(w.x0_lo[0], w.x0_hi[0], size=(1000, w.n)).T
    for k in range(1, t.n_boxes[0]):
        u = w.ctl.forward(x)
        x = w.dyn.forward(np.concatenate([x, u], axis=0))
        assert (x.T >= t.lo[0, k] - 1e-12).all() and (x.T <= t.hi[0, k] + 1e-12).all()


@pytest.mark.parametrize("precision", ["exact", "tc"])
def test_c5_full_batch_strided(precision):
    """The bench's C5 workload at its full size (batch 1024): 32 strided samples against the oracle --
    bit for bit in the exact mode, within the north_star's rtol = 1e-5 in the tensor-core mode."""
    from test_gpu_tcw import rel_dev
    w = c5_closed_loop(batch=1024)
    got = dt_closed_loop_batch(w.dyn, w.ctl, w.n, w.x0_lo, w.x0_hi, w.horizon, precision=precision)
    idx = np.arange(0, 1024, 32)
    exp = oracle_dtcl_batch(w.dyn, w.ctl, w.n, w.x0_lo[idx], w.x0_hi[idx], w.horizon)
    assert (exp.status == 0).all() and (got.status == 0).all()
    sub = type(got)(got.lo[idx], got.hi[idx], got.n_boxes[idx], got.failed_step[idx], got.status[idx])
    if precision == "exact":
        assert_tubes_equal(sub, exp, exact=True)
    else:
        assert rel_dev(sub, exp) <= 1e-5


def test_c5_enclosure_monte_carlo_boxes():
    """>= 1e3 exact rollouts (with the box vertices among them) on four C5 samples."""
    w = c5_closed_loop(batch=64)
    t = dt_closed_loop_batch(w.dyn, w.ctl, w.n, w.x0_lo, w.x0_hi, w.horizon)
    rng = np.random.default_rng(11)
    for b in (0, 21, 42, 63):
        x = rng.uniform(w.x0_lo[b], w.x0_hi[b], size=(1000, w.n))
        x[:64] = np.where(rng.random((64, w.n)) < 0.5, w.x0_lo[b], w.x0_hi[b])
        x = x.T
        for k in range(1, t.n_boxes[b]):
            u = w.ctl.forward(x)
            x = w.dyn.forward(np.concatenate([x, u], axis=0))
            assert (x.T >= t.lo[b, k] - 1e-12).all() and (x.T <= t.hi[b, k] + 1e-12).all()
