"""Open-loop continuous-time flowpipe cases (ct_reach, flowpipe_ct.hpp:428-458): the configurations of
the reference's own tests/test_flowpipe_ct.cpp:146-316 plus failure cases, shared by the CPU oracle
tests and the GPU parity tests."""
import math

import numpy as np

from paper_2605_25346_b200.api import (FlowpipeParams, QuadrotorParams, diag_linear_field, quadrotor_field,
                                       quadrotor_hover_input, rotation_field, zero_field)


def _box(center, rad):
    c = np.asarray(center, np.float64)
    r = np.broadcast_to(np.asarray(rad, np.float64), c.shape)
    return (c - r)[None], (c + r)[None]


def ct_open_cases():
    """(name, field, x0_lo [B][n], x0_hi, FlowpipeParams, expect_failure)."""
    out = []
    lo, hi = _box([0.5, -0.25], [0.1, 0.2])
    out.append(("zero_f", zero_field(2), lo, hi, FlowpipeParams(h=0.05, steps=10), False))           # :146-160
    out.append(("exp_decay", diag_linear_field([-1.0]), np.array([[0.9]]), np.array([[1.1]]),
                FlowpipeParams(h=0.01, steps=100), False))                                         # :162-177
    lo, hi = _box([1.0, 0.0], 0.1)
    out.append(("rotation", rotation_field(1.0), lo, hi, FlowpipeParams(h=0.05, steps=60), False))  # :179-198
    out.append(("wrapping", rotation_field(1.0), lo, hi, FlowpipeParams(h=2 * math.pi / 100, steps=100), False))
    lo5, hi5 = _box([1.0, 0.0], 0.05)
    out.append(("window0", rotation_field(1.0), lo5, hi5, FlowpipeParams(h=0.05, steps=40, window=0), False))
    out.append(("halving_coarse", rotation_field(1.0), lo, hi, FlowpipeParams(h=0.08, steps=25), False))
    out.append(("halving_fine", rotation_field(1.0), lo, hi, FlowpipeParams(h=0.04, steps=50), False))
    rad = [0.05] * 6 + [0.0] * 6
    qlo, qhi = _box([0.0] * 12, rad)
    out.append(("quad_hover", quadrotor_field(), qlo, qhi, FlowpipeParams(h=0.01, steps=100), False))  # :252-282
    rng = np.random.default_rng(11)
    c = rng.uniform(-0.1, 0.1, size=(3, 12))
    r = np.array([0.02] * 6 + [0.01] * 6)
    out.append(("quad_tilted", quadrotor_field(QuadrotorParams(), [10.5, 0.01, -0.02, 0.0]), c - r, c + r,
                FlowpipeParams(h=0.01, steps=40, window=2), False))
    lam = rng.uniform(-2.0, 0.5, size=5)
    c = rng.uniform(-1, 1, size=(4, 5))
    out.append(("diag5", diag_linear_field(lam), c - 0.05, c + 0.05, FlowpipeParams(h=0.02, steps=50, order=1), False))
    # failures: a stiff decay the Picard contraction cannot certify at this h; tme_inv at |theta| ~ pi/2
    out.append(("stiff_fail", diag_linear_field([-80.0]), np.array([[0.9]]), np.array([[1.1]]),
                FlowpipeParams(h=0.2, steps=5), True))
    tl, th = qlo.copy(), qhi.copy()
    tl[0, 7], th[0, 7] = 1.50, 1.66
    out.append(("quad_tme_inv", quadrotor_field(), tl, th, FlowpipeParams(h=0.01, steps=5), True))
    return out


def ct_open_split_case():
    """The CLI's `split --system quadrotor --split rpy:8` shape (reach_cli.cpp:200-211, 80-82)."""
    from paper_2605_25346_b200.api import SplitPlan
    r = np.array([0.05] * 6 + [0.02] * 6)
    return quadrotor_field(), -r, r.copy(), SplitPlan.rpy(12, 8), FlowpipeParams(h=0.01, steps=20)
