"""GPU parity for the continuous-time closed loop (cl_reach, closed_loop.hpp:76-182; SURVEY §8a
A14-A19) through the C ABI vs the CPU oracle (oracle/ct_oracle.c, itself pinned bit for bit to the
reference in tests/test_oracle_ct.py).

Tolerance: the kernels keep the reference's operation order inside every TMExpr operation but
reduce the abs-sums with warp trees and use CUDA's libm (sin / cos / tanh), so boxes agree to
rounding: |gpu - oracle| <= CT_RTOL * max(|oracle|, box width, 1e-300) with CT_RTOL = 1e-9
(north_star allows 1e-5 in fp64).  Status codes, failed steps and box counts must match exactly.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from ct_cases import ct_cases, ct_split_case
from oracle_bind import oracle_cl_batch, oracle_cl_split_hull
from paper_2605_25346_b200.api import cl_reach_batch_arrays, cl_split_hull, split_box
from paper_2605_25346_b200.workloads import c2_quadrotor

CT_RTOL = 1e-9


def _close(g, e, wlo, whi):
    width = np.abs(whi - wlo)
    scale = np.maximum(np.maximum(np.abs(e), width), 1e-300)
    both_nan = np.isnan(g) & np.isnan(e)
    err = np.where(both_nan, 0.0, np.abs(g - e) / scale)
    return float(np.max(err)) if err.size else 0.0


def assert_ct_close(got, exp, rtol=CT_RTOL):
    assert np.array_equal(got.status, exp.status), (got.status, exp.status)
    assert np.array_equal(got.failed_step, exp.failed_step), (got.failed_step, exp.failed_step)
    assert np.array_equal(got.n_boxes, exp.n_boxes), (got.n_boxes, exp.n_boxes)
    worst = 0.0
    for b in range(got.lo.shape[0]):
        k = int(exp.n_boxes[b])
        el, eh = exp.lo[b, :k], exp.hi[b, :k]
        worst = max(worst, _close(got.lo[b, :k], el, el, eh), _close(got.hi[b, :k], eh, el, eh))
    assert worst <= rtol, worst
    return worst


@pytest.mark.parametrize("case", ct_cases(), ids=lambda c: c[0])
def test_cl_matches_oracle(case):
    name, spec, lo, hi, expect_fail = case
    exp = oracle_cl_batch(spec, lo, hi)
    got = cl_reach_batch_arrays(spec, lo, hi)
    worst = assert_ct_close(got, exp)
    print(f"{name}: max rel diff {worst:.3e}")
    assert bool((got.status != 0).any()) == expect_fail


def test_cl_split_hull_matches_oracle():
    spec, lo, hi, plan = ct_split_case()
    exp = oracle_cl_split_hull(spec, lo, hi, plan)
    got = cl_split_hull(spec, (lo, hi), plan)
    assert got.n_boxes == exp.n_boxes and got.fail_key == exp.fail_key
    assert np.array_equal(got.box_diverged, exp.box_diverged)
    assert _close(got.lo, exp.lo, exp.lo, exp.hi) <= CT_RTOL
    assert _close(got.hi, exp.hi, exp.lo, exp.hi) <= CT_RTOL


@pytest.mark.parametrize("case", ct_cases(), ids=lambda c: c[0])
def test_compiled_program_matches_interpreter(case, monkeypatch):
    """The quadrotor field runs as compiled straight-line code (quad_full / quad_fast, ct_kernel.cuh);
    RB_CT_INTERPRET=1 routes the same program through the interpreter.  Both implement the same
    operation sequence: statuses, failed steps and box counts identical, boxes within 1e-11."""
    name, spec, lo, hi, _ = case
    got = cl_reach_batch_arrays(spec, lo, hi)
    monkeypatch.setenv("RB_CT_INTERPRET", "1")
    ref = cl_reach_batch_arrays(spec, lo, hi)
    monkeypatch.delenv("RB_CT_INTERPRET")
    worst = assert_ct_close(got, ref, rtol=1e-11)
    print(f"{name}: compiled vs interpreted max rel diff {worst:.3e}")


def test_cl_batch_rows_independent():
    """A sub-box's tube does not depend on the batch around it (bit-identical)."""
    w = c2_quadrotor()
    lo, hi = split_box(w.x0_lo, w.x0_hi, w.plan)
    idx = np.arange(0, 4096, 37)
    full = cl_reach_batch_arrays(w.spec, lo[idx], hi[idx])
    one = cl_reach_batch_arrays(w.spec, lo[idx[5:6]], hi[idx[5:6]])
    assert np.array_equal(full.lo[5], one.lo[0]) and np.array_equal(full.hi[5], one.hi[0])
    assert (full.status == 0).all()


def test_c2_full_sweep_hull_properties():
    """C2 at full size (rpy:4096): the device hull equals the min/max of the hulls of a partition of
    the part range (order-independent reduction), and a 16-part window matches the oracle."""
    w = c2_quadrotor()
    x0 = (w.x0_lo, w.x0_hi)
    full = cl_split_hull(w.spec, x0, w.plan)
    assert full.n_boxes == w.spec.steps() and full.fail_key == np.iinfo(np.int64).max
    parts = [cl_split_hull(w.spec, x0, w.plan, a, b) for a, b in ((0, 1000), (1000, 3000), (3000, 4096))]
    assert np.array_equal(full.lo, np.minimum.reduce([p.lo for p in parts]))
    assert np.array_equal(full.hi, np.maximum.reduce([p.hi for p in parts]))
    exp = oracle_cl_split_hull(w.spec, w.x0_lo, w.x0_hi, w.plan, 2040, 2056)
    got = cl_split_hull(w.spec, x0, w.plan, 2040, 2056)
    assert _close(got.lo, exp.lo, exp.lo, exp.hi) <= CT_RTOL and _close(got.hi, exp.hi, exp.lo, exp.hi) <= CT_RTOL


# --- Monte-Carlo enclosure (the reference's test_closed_loop.cpp:256-279 pattern) ---------------
def _quad_rhs(x, u, prm):
    mass, g, jx, jy, jz = prm
    vx, vy, vz = x[3], x[4], x[5]
    phi, th, psi = x[6], x[7], x[8]
    p, q, r = x[9], x[10], x[11]
    sphi, cphi, sth, cth, spsi, cpsi = np.sin(phi), np.cos(phi), np.sin(th), np.cos(th), np.sin(psi), np.cos(psi)
    a = u[0] / mass
    tth = sth / cth
    return np.stack([
        vx, vy, vz,
        a * (cphi * sth * cpsi + sphi * spsi), a * (cphi * sth * spsi - sphi * cpsi), a * cphi * cth - g,
        p + sphi * tth * q + cphi * tth * r, cphi * q - sphi * r, (sphi / cth) * q + (cphi / cth) * r,
        q * r * ((jy - jz) / jx) + u[1] / jx, p * r * ((jz - jx) / jy) + u[2] / jy, p * q * ((jx - jy) / jz) + u[3] / jz,
    ])


def simulate_zoh(spec, x):
    """Zero-order-hold closed loop (test_closed_loop.cpp:21-38) with fine RK4; x [12][S]."""
    prm = spec.plant_params.as_array()
    states = [x.copy()]
    sub = 40
    dt = spec.fp.h / sub
    for i in range(spec.ctl_steps):
        ref = np.asarray(spec.y_ref[i], np.float64)[:, None] * np.ones((1, x.shape[1]))
        u = spec.controller.forward(np.concatenate([x, ref], axis=0))
        for _ in range(spec.k_atomic):
            for _ in range(sub):
                k1 = _quad_rhs(x, u, prm)
                k2 = _quad_rhs(x + 0.5 * dt * k1, u, prm)
                k3 = _quad_rhs(x + 0.5 * dt * k2, u, prm)
                k4 = _quad_rhs(x + dt * k3, u, prm)
                x = x + dt / 6.0 * (k1 + 2 * k2 + 2 * k3 + k4)
            states.append(x.copy())
    return states


def test_cl_monte_carlo_enclosure():
    w = c2_quadrotor()
    lo, hi = split_box(w.x0_lo, w.x0_hi, w.plan)
    idx = np.array([0, 2047, 4095])
    t = cl_reach_batch_arrays(w.spec, lo[idx], hi[idx])
    assert (t.status == 0).all()
    rng = np.random.default_rng(5)
    for bi in range(len(idx)):
        # >= 1e3 rollouts per checked sub-box, the first 64 at box vertices
        x = rng.uniform(lo[idx[bi]], hi[idx[bi]], size=(1000, 12))
        x[:64] = np.where(rng.random((64, 12)) < 0.5, lo[idx[bi]], hi[idx[bi]])
        x = x.T
        states = simulate_zoh(w.spec, x)
        for k in range(1, len(states)):
            assert (states[k].T >= t.lo[bi, k, :12] - 1e-10).all(), k
            assert (states[k].T <= t.hi[bi, k, :12] + 1e-10).all(), k
