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
