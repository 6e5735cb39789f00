"""GPU: a seeded sweep of random DT systems through the tolerance modes (fused, tc) against the oracle --
widths, depths, action inputs, windows, rebuild_from_box and tanh layers beyond the fixed cases.
Bar: identical statuses / failed steps / box counts, bounds within rtol = 1e-5 (north_star)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle_bind import oracle_dt_batch
from paper_2605_25346_b200.api import Act, DTReachParams, DTSystem, dt_reach_batch_arrays
from paper_2605_25346_b200.workloads import random_mlp, residual_relu_dynamics
from test_gpu_tcw import rel_dev


def _system(seed):
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(2, 7))
    m = int(rng.integers(0, 3))
    depth = int(rng.integers(1, 4))
    hidden = [int(rng.choice([16, 32, 64, 96, 128])) for _ in range(depth)]
    if seed % 3 == 2:
        net = random_mlp(rng, n + m, hidden, n, Act.Tanh, 0.5)
        net.layers[-1].w *= 0.3
    else:
        net = residual_relu_dynamics(rng, n, m, hidden, dt=0.1)
    prm = DTReachParams(window=int(rng.choice([1, 2, 4])), rebuild_from_box=bool(seed % 5 == 4))
    B, H = 6, int(rng.integers(3, 12))
    c = rng.uniform(-0.5, 0.5, size=(B, n))
    r = rng.uniform(1e-3, 2e-2, size=(B, n))
    acts = rng.uniform(-0.5, 0.5, size=(B, H, m))
    return DTSystem(net, n, m), c - r, c + r, acts, prm


@pytest.mark.parametrize("precision", ["fused", "tc"])
@pytest.mark.parametrize("seed", range(12))
def test_random_systems_within_tolerance(seed, precision):
    sys, lo, hi, acts, prm = _system(seed)
    exp = oracle_dt_batch(sys, lo, hi, acts, prm)
    got = dt_reach_batch_arrays(sys, lo, hi, acts, prm, precision=precision)
    assert np.array_equal(got.status, exp.status) and np.array_equal(got.failed_step, exp.failed_step)
    dev = rel_dev(got, exp)
    assert dev <= 1e-5, dev


def _closed_loop(seed):
    rng = np.random.default_rng(2000 + seed)
    n = int(rng.integers(2, 6))
    l = int(rng.integers(1, 3))
    hidden = [int(rng.choice([16, 32, 64])) for _ in range(int(rng.integers(1, 3)))]
    dyn = residual_relu_dynamics(rng, n, l, hidden, dt=0.1)
    act = Act.Tanh if seed % 2 else Act.Relu
    ctl = random_mlp(rng, n, [int(rng.choice([16, 32]))], l, act, 0.5)
    ctl.layers[-1].w *= 0.3
    B, H = 4, int(rng.integers(3, 10))
    c = rng.uniform(-0.4, 0.4, size=(B, n))
    r = rng.uniform(1e-3, 1e-2, size=(B, n))
    return dyn, ctl, n, c - r, c + r, H, DTReachParams(window=int(rng.choice([1, 4])))


@pytest.mark.parametrize("precision", ["fused", "tc"])
@pytest.mark.parametrize("seed", range(6))
def test_random_closed_loops_within_tolerance(seed, precision):
    from oracle_bind import oracle_dtcl_batch
    from paper_2605_25346_b200.api import dt_closed_loop_batch
    dyn, ctl, n, lo, hi, H, prm = _closed_loop(seed)
    exp = oracle_dtcl_batch(dyn, ctl, n, lo, hi, H, prm)
    got = dt_closed_loop_batch(dyn, ctl, n, lo, hi, H, prm, precision=precision)
    assert np.array_equal(got.status, exp.status) and np.array_equal(got.failed_step, exp.failed_step)
    assert rel_dev(got, exp) <= 1e-5
