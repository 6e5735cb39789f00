"""GPU: the ctl_reach_loss gradient (training.hpp:183-213) -- grad_forward's Dual passes of the quadrotor
closed loop (cl_reach, closed_loop.hpp:76-182) over the controller's parameters, on the device
(reach_ctl_reach_loss, ct_dual.cuh) -- against the reference's own grad_forward (oracle/_ref).

Bar: the loss within 1e-12 relative (the tubes agree to ~1e-15: tree-reduced abs-sums and CUDA's
sin / cos / tanh), the gradient within 1e-9 of its largest component, identical diverged counts."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle_bind import ref_available, ref_ctl_reach_loss
from paper_2605_25346_b200.api import Act, ClosedLoopSpec, Episode, FlowpipeParams, ctl_reach_loss

needs_ref = pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")
GRAD_RTOL = 1e-9


def _case(with_ref, seed=8, hidden=(8, 8), episodes=2, t_h=2):
    from paper_2605_25346_b200.workloads import quadrotor_controller, random_mlp
    rng = np.random.default_rng(seed)
    if with_ref:
        ctl = quadrotor_controller(rng, hidden)
    else:
        ctl = random_mlp(rng, 12, list(hidden), 4, Act.Tanh, 0.4)
        ctl.layers[-1].w *= 0.1
        ctl.layers[-1].b[0] += 9.81
    batch = []
    for _ in range(episodes):
        x0 = np.zeros(12)
        x0[:6] = rng.uniform(-0.05, 0.05, 6)
        yr = list(np.tile(rng.uniform(-0.1, 0.1, 3), (t_h, 1))) if with_ref else []
        batch.append(Episode([x0] * (t_h + 1), [np.zeros(4)] * t_h, yr))
    return ctl, batch


def _ref(ctl, batch, eps, t_h, delta, k_atomic, cap):
    spec = ClosedLoopSpec(ctl, ctl_steps=t_h, k_atomic=k_atomic, fp=FlowpipeParams(h=delta / k_atomic),
                          y_ref=np.asarray(batch[0].y_ref) if len(batch[0].y_ref) else None)
    return ref_ctl_reach_loss(spec, np.array([b.states[0] for b in batch]),
                              [None if not len(b.y_ref) else np.asarray(b.y_ref) for b in batch],
                              eps, t_h, delta, cap, with_grad=True)


@needs_ref
@pytest.mark.parametrize("with_ref", [False, True])
def test_ctl_reach_loss_gradient_matches_reference(with_ref):
    t_h, k_atomic, delta, eps, cap = 2, 2, 0.02, 0.01, 40.0
    ctl, batch = _case(with_ref, t_h=t_h)
    loss, g, dcount = ctl_reach_loss(ctl, batch, eps, t_h, delta, k_atomic, cap, with_grad=True)
    el, eg, ed = _ref(ctl, batch, eps, t_h, delta, k_atomic, cap)
    assert dcount == ed == 0
    assert abs(loss - el) <= 1e-12 * abs(el), (loss, el)
    scale = float(np.max(np.abs(eg)))
    err = float(np.max(np.abs(g - eg)))
    print("ctl_reach_loss grad max abs err", err, "scale", scale)
    assert err <= GRAD_RTOL * scale
    v, dv = ctl_reach_loss(ctl, batch, eps, t_h, delta, k_atomic, cap)
    assert abs(v - loss) <= 1e-12 * abs(loss) and dv == dcount


@needs_ref
def test_ctl_reach_loss_gradient_diverged_episode_is_capped():
    """An episode whose closed loop fails contributes the cap (zero tangent), as the reference."""
    t_h, k_atomic, delta, eps, cap = 2, 1, 0.5, 0.3, 40.0  # a step far too long: the remainder blows up
    ctl, batch = _case(False, seed=3, t_h=t_h)
    loss, g, dcount = ctl_reach_loss(ctl, batch, eps, t_h, delta, k_atomic, cap, with_grad=True)
    el, eg, ed = _ref(ctl, batch, eps, t_h, delta, k_atomic, cap)
    assert dcount == ed
    assert abs(loss - el) <= 1e-12 * abs(el)
    assert float(np.max(np.abs(g - eg))) <= GRAD_RTOL * max(float(np.max(np.abs(eg))), 1.0)
