"""GPU parity for the open-loop continuous-time flowpipe (ct_reach, flowpipe_ct.hpp:428-458) through
the C ABI vs the CPU oracle (oracle/ct_oracle.c, pinned bit for bit to the reference in
tests/test_oracle_ct_open.py), plus the reference's own flowpipe test properties
(tests/test_flowpipe_ct.cpp:146-316).  Tolerance as tests/test_gpu_ct.py: CT_RTOL = 1e-9."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from ct_open_cases import ct_open_cases, ct_open_split_case
from oracle_bind import oracle_ct_batch, oracle_ct_split_hull
from paper_2605_25346_b200.api import (FlowpipeParams, ct_reach, ct_reach_batch_arrays, ct_split_hull, diag_linear_field,
                                       quadrotor_field, rotation_field, zero_field)
from test_gpu_ct import CT_RTOL, _close, _quad_rhs, assert_ct_close


@pytest.mark.parametrize("case", ct_open_cases(), ids=lambda c: c[0])
def test_ct_matches_oracle(case):
    name, f, lo, hi, prm, expect_fail = case
    exp = oracle_ct_batch(f, lo, hi, prm)
    got = ct_reach_batch_arrays(f, lo, hi, prm)
    worst = assert_ct_close(got, exp)
    print(f"{name}: max rel diff {worst:.3e}")
    assert bool((got.status != 0).any()) == expect_fail


@pytest.mark.parametrize("case", [c for c in ct_open_cases() if c[0].startswith("quad")], ids=lambda c: c[0])
def test_compiled_quadrotor_matches_interpreter(case, monkeypatch):
    """The held-input quadrotor field's compiled program (quad_full / quad_fast<HELD>) against the
    interpreter (RB_CT_INTERPRET=1) on the same inputs: codes identical, boxes within 1e-11."""
    name, f, lo, hi, prm, _ = case
    got = ct_reach_batch_arrays(f, lo, hi, prm)
    monkeypatch.setenv("RB_CT_INTERPRET", "1")
    ref = ct_reach_batch_arrays(f, lo, hi, prm)
    monkeypatch.delenv("RB_CT_INTERPRET")
    worst = assert_ct_close(got, ref, rtol=1e-11)
    print(f"{name}: compiled vs interpreted max rel diff {worst:.3e}")


def test_zero_field_keeps_x0():  # test_flowpipe_ct.cpp:146-160
    lo, hi = np.array([0.4, -0.45]), np.array([0.6, -0.05])
    t = ct_reach(zero_field(2), (lo, hi), FlowpipeParams(h=0.05, steps=10))
    assert t.steps() == 11 and not t.diverged
    assert np.allclose(t.lo, lo, rtol=1e-12) and np.allclose(t.hi, hi, rtol=1e-12)


def test_exp_decay_closed_form():  # :162-177
    t = ct_reach(diag_linear_field([-1.0]), (np.array([0.9]), np.array([1.1])), FlowpipeParams(h=0.01, steps=100))
    assert not t.diverged
    lo, hi = t.lo[-1, 0], t.hi[-1, 0]
    assert lo <= 0.9 * math.exp(-1.0) and hi >= 1.1 * math.exp(-1.0)
    assert hi - lo <= 1.2 * (1.1 * math.exp(-0.99) - 0.9 * math.exp(-1.0))


def test_rotation_soundness_and_wrapping():  # :179-234
    x0 = (np.array([0.9, -0.1]), np.array([1.1, 0.1]))
    t = ct_reach(rotation_field(1.0), x0, FlowpipeParams(h=0.05, steps=60))
    assert not t.diverged
    rng = np.random.default_rng(1029384756)
    x = rng.uniform(x0[0], x0[1], size=(200, 2))
    for k in range(1, t.steps()):
        tt = t.t_hi[k]
        xt = np.stack([x[:, 0] * np.cos(tt) - x[:, 1] * np.sin(tt), x[:, 0] * np.sin(tt) + x[:, 1] * np.cos(tt)], 1)
        assert (xt >= t.lo[k]).all() and (xt <= t.hi[k]).all()
    w = ct_reach(rotation_field(1.0), x0, FlowpipeParams(h=2 * math.pi / 100, steps=100))
    assert not w.diverged and (w.hi[-1, 0] - w.lo[-1, 0]) <= 1.5 * 0.2


def test_quadrotor_hover_monte_carlo():  # :252-282
    prm = FlowpipeParams(h=0.01, steps=100)
    r = np.array([0.05] * 6 + [0.0] * 6)
    t = ct_reach(quadrotor_field(), (-r, r), prm)
    assert not t.diverged and t.steps() == 101
    rng = np.random.default_rng(8675309)
    x = rng.uniform(-r, r, size=(50, 12)).T
    u = np.array([9.81, 0.0, 0.0, 0.0])[:, None] * np.ones((1, 50))
    prmq = [1.0, 9.81, 0.01, 0.01, 0.02]
    sub = 40
    dt = prm.h / sub
    for k in range(1, t.steps()):
        for _ in range(sub):
            k1 = _quad_rhs(x, u, prmq)
            k2 = _quad_rhs(x + 0.5 * dt * k1, u, prmq)
            k3 = _quad_rhs(x + 0.5 * dt * k2, u, prmq)
            k4 = _quad_rhs(x + dt * k3, u, prmq)
            x = x + dt / 6.0 * (k1 + 2 * k2 + 2 * k3 + k4)
        assert (x.T >= t.lo[k] - 1e-10).all() and (x.T <= t.hi[k] + 1e-10).all(), k


def test_batch_rows_independent():
    rng = np.random.default_rng(3)
    c = rng.uniform(-0.1, 0.1, size=(37, 12))
    r = np.array([0.02] * 6 + [0.01] * 6)
    f = quadrotor_field()
    prm = FlowpipeParams(h=0.01, steps=20)
    full = ct_reach_batch_arrays(f, c - r, c + r, prm)
    one = ct_reach_batch_arrays(f, (c - r)[17:18], (c + r)[17:18], prm)
    assert np.array_equal(full.lo[17], one.lo[0]) and np.array_equal(full.hi[17], one.hi[0])


def test_ct_split_hull_matches_oracle():
    f, lo, hi, plan, prm = ct_open_split_case()
    exp = oracle_ct_split_hull(f, lo, hi, plan, prm)
    got = ct_split_hull(f, (lo, hi), plan, prm)
    assert got.n_boxes == exp.n_boxes and got.fail_key == exp.fail_key
    assert _close(got.lo, exp.lo, exp.lo, exp.hi) <= CT_RTOL and _close(got.hi, exp.hi, exp.lo, exp.hi) <= CT_RTOL


def test_ct_error_behaviour():
    """FlowpipeParams::validate / shape errors raise ValueError (the reference's std::invalid_argument);
    shapes outside the device family raise ReachError (REACH_E_UNSUPPORTED), never a CPU fallback."""
    from paper_2605_25346_b200 import ReachError
    lo, hi = np.array([[0.9, -0.1]]), np.array([[1.1, 0.1]])
    with pytest.raises(ValueError):
        ct_reach_batch_arrays(rotation_field(1.0), lo, hi, FlowpipeParams(h=-0.1))
    with pytest.raises(ValueError):
        ct_reach_batch_arrays(rotation_field(1.0), lo[:, :1], hi[:, :1], FlowpipeParams())
    with pytest.raises(ValueError):
        ct_reach_batch_arrays(rotation_field(1.0), np.array([[np.inf, 0.0]]), hi, FlowpipeParams())
    with pytest.raises(ReachError):  # 12 x (window + 2) = 96 > 80 generator columns
        ct_reach_batch_arrays(quadrotor_field(), np.zeros((1, 12)), np.full((1, 12), 0.01), FlowpipeParams(window=6))


def test_cl_error_behaviour():
    from paper_2605_25346_b200 import ReachError
    from paper_2605_25346_b200.api import ClosedLoopSpec, cl_reach_batch_arrays
    from paper_2605_25346_b200.workloads import c2_quadrotor
    w = c2_quadrotor()
    lo, hi = w.x0_lo[None], w.x0_hi[None]
    bad = ClosedLoopSpec(controller=w.spec.controller, ctl_steps=2, k_atomic=2)  # 15-input controller, no y_ref
    with pytest.raises(ValueError):
        cl_reach_batch_arrays(bad, lo, hi)
    spec = ClosedLoopSpec(controller=w.spec.controller, ctl_steps=2, k_atomic=2, y_ref=w.spec.y_ref[:2],
                          fp=FlowpipeParams(window=5))
    with pytest.raises(ReachError):  # window 5: 12 + 5 x 16 generator columns exceed the device rows
        cl_reach_batch_arrays(spec, lo, hi)
    with pytest.raises(ValueError):
        cl_reach_batch_arrays(w.spec, lo[:, :6], hi[:, :6])


def test_ct_device_pointer_path_matches_host_path():
    """REACH_FLAG_DEVICE_PTRS: stream-ordered call on device buffers (no host copies inside)."""
    import ctypes as C

    import torch
    from paper_2605_25346_b200 import _abi as A
    from paper_2605_25346_b200.api import default_context
    f = quadrotor_field()
    prm = FlowpipeParams(h=0.01, steps=15)
    rng = np.random.default_rng(9)
    c = rng.uniform(-0.1, 0.1, size=(8, 12))
    lo, hi = c - 0.01, c + 0.01
    exp = ct_reach_batch_arrays(f, lo, hi, prm)
    ctx = default_context()
    dev = torch.device("cuda", 0)
    dlo, dhi = torch.tensor(lo, device=dev), torch.tensor(hi, device=dev)
    T = prm.steps + 1
    olo = torch.full((8, T, 12), float("nan"), dtype=torch.float64, device=dev)
    ohi = torch.full_like(olo, float("nan"))
    nb, fs, st = (torch.zeros(8, dtype=torch.int32, device=dev) for _ in range(3))
    to = A.TubeOut(A.dptr(olo.data_ptr()), A.dptr(ohi.data_ptr()), A.iptr(nb.data_ptr()), A.iptr(fs.data_ptr()),
                   A.iptr(st.data_ptr()))
    fd, fp = f.c_struct(), prm.c_struct()
    ctx.check(ctx._lib.reach_ct_batch(ctx.handle, C.byref(fd), C.byref(fp), 8, A.dptr(dlo.data_ptr()),
                                      A.dptr(dhi.data_ptr()), C.byref(to), A.REACH_FLAG_DEVICE_PTRS), "ct_reach")
    ctx.synchronize()
    assert np.array_equal(olo.cpu().numpy(), exp.lo) and np.array_equal(ohi.cpu().numpy(), exp.hi)
    assert np.array_equal(nb.cpu().numpy(), exp.n_boxes)
