"""GPU parity for the DT closed loop through the C ABI vs the CPU oracle."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from cl_cases import cl_cases
from oracle_bind import assert_tubes_equal, oracle_dtcl_batch
from paper_2605_25346_b200.api import DTReachParams, dt_closed_loop_batch
from paper_2605_25346_b200.workloads import c1_closed_loop

TANH_RTOL = 1e-9


@pytest.mark.parametrize("case", cl_cases(), ids=lambda c: c[0])
def test_dtcl_matches_oracle(case):
    name, dyn, ctl, n, lo, hi, H, prm, tanh = case
    exp = oracle_dtcl_batch(dyn, ctl, n, lo, hi, H, prm)
    got = dt_closed_loop_batch(dyn, ctl, n, lo, hi, H, prm)
    assert_tubes_equal(got, exp, exact=not tanh, rtol=TANH_RTOL)


def test_dtcl_large_batch_rows_independent():
    w = c1_closed_loop(batch=2048)
    full = dt_closed_loop_batch(w.dyn, w.ctl, w.n, w.x0_lo, w.x0_hi, w.horizon)
    idx = np.array([0, 1, 777, 2047])
    exp = oracle_dtcl_batch(w.dyn, w.ctl, w.n, w.x0_lo[idx], w.x0_hi[idx], w.horizon)
    sub = type(full)(full.lo[idx], full.hi[idx], full.n_boxes[idx], full.failed_step[idx], full.status[idx])
    assert_tubes_equal(sub, exp, exact=True)


def test_dtcl_enclosure_monte_carlo():
    w = c1_closed_loop(batch=2)
    t = dt_closed_loop_batch(w.dyn, w.ctl, w.n, w.x0_lo, w.x0_hi, w.horizon)
    rng = np.random.default_rng(0)
    for b in range(2):
        x = rng.uniform(w.x0_lo[b], w.x0_hi[b], size=(256, w.n)).T  # [n][S]
        for k in range(1, t.n_boxes[b]):
            u = w.ctl.forward(x)
            x = w.dyn.forward(np.concatenate([x, u], axis=0))
            assert (x.T >= t.lo[b, k] - 1e-12).all() and (x.T <= t.hi[b, k] + 1e-12).all()
