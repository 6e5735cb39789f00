"""GPU: the certified-training regularizer reach_loss (training.hpp:99-126) and its gradient over the model
parameters (grad_forward of reach_loss over net_params, as train_dt_dyn takes it) against the reference
(oracle/_ref).  The gradient is bit-identical (the Dual tangent of log is a.d / a.v); the loss value goes
through CUDA's log, within 1e-14 relative of glibc's."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle_bind import ref_available, ref_reach_loss, same_bits
from paper_2605_25346_b200.api import Act, DTReachParams, Episode, affine_net, reach_loss
from paper_2605_25346_b200.workloads import random_mlp

needs_ref = pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")


def _batch(rng, M, n, m, T):
    eps = []
    for _ in range(M):
        states = [rng.uniform(-0.4, 0.4, n)] + [np.zeros(n)] * T
        eps.append(Episode(states, [rng.uniform(-0.5, 0.5, m) for _ in range(T)]))
    return eps


def _arrays(batch, t_h):
    x0 = np.array([np.asarray(e.states[0]) for e in batch])
    acts = np.array([np.asarray(e.actions[:t_h]) for e in batch])
    return x0, acts


@needs_ref
@pytest.mark.parametrize("shape", [(4, 2, [16], 6, 3), (3, 1, [24, 24], 4, 5)], ids=["small", "deep"])
def test_reach_loss_and_gradient_match_reference(shape):
    n, m, hidden, M, t_h = shape
    rng = np.random.default_rng(17)
    model = random_mlp(rng, n + m, hidden, n, Act.Relu, 0.6)
    model.layers[-1].w *= 0.5
    batch = _batch(rng, M, n, m, t_h + 2)
    x0, acts = _arrays(batch, t_h)
    el, eg, ed = ref_reach_loss(model, x0, acts, 0.05, 50.0, with_grad=True)
    loss, g, dcount = reach_loss(model, batch, 0.05, t_h, 50.0, with_grad=True)
    assert dcount == ed
    assert abs(loss - el) <= 1e-14 * abs(el)
    assert same_bits(g, eg)
    assert reach_loss(model, batch, 0.05, t_h, 50.0)[0] == loss


@needs_ref
def test_diverged_episodes_charge_the_cap():
    w = np.concatenate([np.eye(2) * 1e200, np.eye(2)], axis=1)
    model = affine_net(w, np.zeros(2))
    rng = np.random.default_rng(2)
    batch = _batch(rng, 3, 2, 2, 4)
    loss, dcount = reach_loss(model, batch, 0.1, 4, 7.0)
    x0, acts = _arrays(batch, 4)
    el, _, ed = ref_reach_loss(model, x0, acts, 0.1, 7.0)
    assert dcount == ed == 3 and loss == el == 7.0


def test_bad_batch_raises():
    model = affine_net(np.concatenate([np.eye(2), np.eye(2)], axis=1), np.zeros(2))
    with pytest.raises(ValueError):
        reach_loss(model, [], 0.1, 3, 1.0)
    ep = Episode([np.zeros(2)] * 3, [np.zeros(2)] * 2)
    with pytest.raises(ValueError):
        reach_loss(model, [ep], 0.1, 3, 1.0)


@needs_ref
@pytest.mark.parametrize("with_ref", [False, True])
def test_ctl_reach_loss_matches_reference(with_ref):
    """ctl_reach_loss (training.hpp:183-213) value: the quadrotor closed loop from each episode start on the
    device.  CT tubes agree to ~1e-15 relative (CUDA libm in the tanh controller), so the loss within 1e-12."""
    from oracle_bind import ref_ctl_reach_loss
    from paper_2605_25346_b200.api import ClosedLoopSpec, FlowpipeParams, ctl_reach_loss
    from paper_2605_25346_b200.workloads import quadrotor_controller, random_mlp
    rng = np.random.default_rng(8)
    if with_ref:
        ctl = quadrotor_controller(rng, (16, 16))
    else:
        ctl = random_mlp(rng, 12, [16, 16], 4, Act.Tanh, 0.4)
        ctl.layers[-1].w *= 0.1
        ctl.layers[-1].b[0] += 9.81
    t_h, k_atomic, delta, eps, cap = 3, 2, 0.02, 0.01, 40.0
    batch, yrefs, cur = [], [], None
    for e in range(4):
        x0 = np.zeros(12)
        x0[:6] = rng.uniform(-0.05, 0.05, 6)
        yr = None
        if with_ref and e != 2:  # episode 2 keeps episode 1's reference (the reference's carry-over)
            yr = np.tile(rng.uniform(-0.1, 0.1, 3), (t_h, 1))
        batch.append(Episode([x0] * (t_h + 1), [np.zeros(4)] * t_h, [] if yr is None else list(yr)))
        cur = yr if yr is not None else cur
        yrefs.append(cur)
    loss, dcount = ctl_reach_loss(ctl, batch, eps, t_h, delta, k_atomic, cap)
    spec = ClosedLoopSpec(ctl, ctl_steps=t_h, k_atomic=k_atomic, fp=FlowpipeParams(h=delta / k_atomic),
                          y_ref=yrefs[0])
    el, ed = ref_ctl_reach_loss(spec, np.array([b.states[0] for b in batch]),
                                [None if not len(b.y_ref) else np.asarray(b.y_ref) for b in batch],
                                eps, t_h, delta, cap)
    assert dcount == ed
    assert abs(loss - el) <= 1e-12 * abs(el), (loss, el)
