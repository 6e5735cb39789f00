"""Continuous-time closed-loop cases (cl_reach, closed_loop.hpp:76-182)
shared by the CPU oracle tests and the GPU parity tests."""
import copy

import numpy as np

from paper_2605_25346_b200.api import Act, ClosedLoopSpec, FlowpipeParams, SplitPlan, split_box
from paper_2605_25346_b200.workloads import c2_quadrotor, quadrotor_controller, random_mlp


def _with(spec, **kw):
    s = copy.copy(spec)
    s.fp = copy.copy(spec.fp)
    for k, v in kw.items():
        if k.startswith("fp_"):
            setattr(s.fp, k[3:], v)
        else:
            setattr(s, k, v)
    if "ctl_steps" in kw and s.y_ref is not None:
        s.y_ref = np.tile(np.asarray(spec.y_ref)[0], (s.ctl_steps, 1))
    return s


def c2_parts(w, idx):
    lo, hi = split_box(w.x0_lo, w.x0_hi, w.plan)
    return lo[idx], hi[idx]


def ct_cases():
    """(name, spec, x0_lo [B][12], x0_hi, expect_failure)."""
    out = []
    w = c2_quadrotor()
    idx = np.array([0, 1, 273, 1500, 2048, 4095])
    lo, hi = c2_parts(w, idx)
    out.append(("c2_full", w.spec, lo[:3], hi[:3], False))
    short = _with(w.spec, ctl_steps=3)
    out.append(("c2_short", short, lo, hi, False))
    out.append(("intervalize", _with(short, intervalize_boundary=True), lo[:3], hi[:3], False))
    out.append(("order1", _with(short, fp_order=1), lo[:3], hi[:3], False))
    for wd in (0, 1, 2):
        out.append((f"window{wd}", _with(short, fp_window=wd), lo[:2], hi[:2], False))
    out.append(("refine0", _with(short, fp_refine_rounds=0), lo[:2], hi[:2], False))
    # controller without a reference input (ClosedLoopSpec::y_ref empty)
    rng = np.random.default_rng(77)
    ctl12 = random_mlp(rng, 12, [32, 32], 4, Act.Tanh, 0.4)
    ctl12.layers[-1].w *= 0.1
    ctl12.layers[-1].b[0] += 9.81
    out.append(("no_ref", ClosedLoopSpec(controller=ctl12, ctl_steps=3, k_atomic=4), lo[:3], hi[:3], False))
    # the reference's own quadrotor closed-loop test shape (test_closed_loop.cpp:236-254)
    rng = np.random.default_rng(7788)
    ctl16 = quadrotor_controller(rng, hidden=(16,))
    spec = ClosedLoopSpec(controller=ctl16, ctl_steps=4, k_atomic=5, y_ref=np.tile([0.1, 0.0, 0.0], (4, 1)),
                          fp=FlowpipeParams(h=0.01))
    x0 = np.array([0.3] * 3 + [0.05] * 3 + [0.02] * 6)
    out.append(("ref_test_shape", spec, (-x0)[None], x0[None], False))
    # a controller wider than 64 (the 128-wide certification buffers, ct_ctl_kernel<128>)
    rng = np.random.default_rng(4242)
    ctlw = quadrotor_controller(rng, hidden=(96, 80))
    out.append(("wide_ctl", _with(short, controller=ctlw), lo[:2], hi[:2], False))
    # failures: remainder never contractive; tme_inv on a cos(theta) range through 0; blow-up
    out.append(("remainder_fail", _with(short, fp_eps_init=1e-14, fp_max_enlargements=0), lo[:2], hi[:2], True))
    tl, th = lo[:2].copy(), hi[:2].copy()
    tl[:, 7], th[:, 7] = 1.50, 1.66
    out.append(("tme_inv", short, tl, th, True))
    out.append(("big_h", _with(w.spec, fp_h=0.25), lo[:2], hi[:2], True))
    return out


def ct_split_case():
    """A small rpy split of the C2 workload (reach_with_splitting(cl_reach), refine.hpp:121-160)."""
    w = c2_quadrotor()
    return _with(w.spec, ctl_steps=2), w.x0_lo, w.x0_hi, SplitPlan.rpy(12, 8)
