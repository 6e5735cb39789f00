"""DT closed-loop cases shared by CPU and GPU tests."""
import numpy as np

from paper_2605_25346_b200.api import Act, DTReachParams
from paper_2605_25346_b200.workloads import c1_closed_loop, random_mlp, residual_relu_dynamics


def cl_cases():
    out = []
    w = c1_closed_loop(batch=6)
    out.append(("c1_shape", w.dyn, w.ctl, w.n, w.x0_lo, w.x0_hi, w.horizon, DTReachParams(), False))
    rng = np.random.default_rng(3001)
    for s in range(2):
        dyn = random_mlp(rng, 6, [64, 64], 4, Act.Relu, 0.8)
        dyn.layers[-1].w *= 0.3
        ctl = random_mlp(rng, 4, [64, 64], 2, Act.Relu, 0.6)
        ctl.layers[-1].w *= 0.3
        c = rng.uniform(-0.5, 0.5, size=(5, 4))
        out.append((f"survey_probe_{s}", dyn, ctl, 4, c - 0.05, c + 0.05, 20, DTReachParams(), False))
    # window variants and a 3-D plant with a 1-D controller
    rng = np.random.default_rng(12)
    dyn = residual_relu_dynamics(rng, 3, 1, [32, 32], dt=0.1)
    ctl = random_mlp(rng, 3, [32], 1, Act.Relu, 0.5)
    c = rng.uniform(-0.5, 0.5, size=(4, 3))
    for wdw in (1, 2, 6):
        out.append((f"window_{wdw}", dyn, ctl, 3, c - 0.02, c + 0.02, 12, DTReachParams(window=wdw), False))
    out.append(("rebuild", dyn, ctl, 3, c - 0.02, c + 0.02, 12, DTReachParams(rebuild_from_box=True), False))
    # tanh controller
    ctl_t = random_mlp(rng, 3, [32, 32], 1, Act.Tanh, 0.5)
    out.append(("tanh_ctl", dyn, ctl_t, 3, c - 0.02, c + 0.02, 10, DTReachParams(), True))
    # explosive dynamics: failures of the dynamics certification / box
    dyn_x = random_mlp(rng, 4, [16], 3, Act.Relu, 3.0)
    dyn_x.layers[-1].w *= 20.0
    out.append(("explosive", dyn_x, ctl, 3, c - 0.2, c + 0.2, 120, DTReachParams(), False))
    return out
