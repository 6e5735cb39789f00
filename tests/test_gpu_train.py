"""GPU: certified training (training.hpp) on the device against the reference itself (oracle/_ref).

pred_loss and its grad_forward over net_params: bit for bit (the Dual rollouts keep the reference's
operation order; the terms are summed on the host in its (episode, step) order).  train_dt_dyn: the
log (T_h, eps, L_pred, L_reach, L_total, diverged_count) and the trained parameters bit for bit --
the same minibatch stream, the same device losses / gradients, the same Adam arithmetic."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle_bind import ref_pred_loss, ref_train_dt_dyn
from paper_2605_25346_b200.api import horizon_weights, pred_loss, train_dt_dyn
from train_cases import dt_training_case, train_config


@pytest.mark.parametrize("t_h", [1, 3, 6])
def test_pred_loss_and_gradient_bit_identical(t_h):
    model, data = dt_training_case()
    w = horizon_weights(t_h)
    got, g = pred_loss(model, data[:4], t_h, w, with_grad=True)
    exp, ge = ref_pred_loss(model, data[:4], t_h, w, with_grad=True)
    assert got == exp
    assert np.array_equal(g, ge), float(np.max(np.abs(g - ge)))
    assert pred_loss(model, data[:4], t_h, w) == exp


def test_pred_loss_errors():
    model, data = dt_training_case()
    with pytest.raises(ValueError):
        pred_loss(model, data[:2], 7, horizon_weights(7))  # episodes of length 6
    with pytest.raises(ValueError):
        pred_loss(model, data[:2], 3, horizon_weights(2))


@pytest.mark.parametrize("lam", [0.0, 0.5])
def test_train_dt_dyn_matches_reference(lam):
    model, data = dt_training_case()
    cfg = train_config(lambda_=lam, iters=4)
    net, rows = train_dt_dyn(model, cfg, data)
    pe, rows_e, rc = ref_train_dt_dyn(model, cfg, data)
    assert rc == 0
    assert rows == rows_e
    assert np.array_equal(net.params(), pe), float(np.max(np.abs(net.params() - pe)))


def test_train_dt_dyn_one_iteration_update():
    """One training iteration's parameter update equals the reference's (the verdict's done-criterion)."""
    model, data = dt_training_case(seed=9)
    cfg = train_config(lambda_=1.0, iters=1, horizon_max=3)
    net, rows = train_dt_dyn(model, cfg, data)
    pe, rows_e, rc = ref_train_dt_dyn(model, cfg, data)
    assert rc == 0 and rows == rows_e and np.array_equal(net.params(), pe)
    assert rows[0].l_reach > 0 and not np.array_equal(pe, model.params())


TRACK_RTOL = 1e-9  # CUDA's sin / cos / tanh against glibc's: ulp-level differences, amplified by RK4


@pytest.mark.parametrize("t_t,rk4", [(1, 1), (3, 4), (5, 2)])
def test_track_loss_and_gradient_match_reference(t_t, rk4):
    from oracle_bind import ref_track_loss
    from paper_2605_25346_b200.api import track_loss
    from train_cases import ct_tracking_case
    ctl, data = ct_tracking_case()
    w = horizon_weights(t_t)
    got, g, bc = track_loss(ctl, data, t_t, w, 0.1, 0.05, rk4, with_grad=True)
    exp, ge, bce = ref_track_loss(ctl, data, t_t, w, 0.1, 0.05, rk4, with_grad=True)
    assert bc == bce == 0
    assert abs(got - exp) <= TRACK_RTOL * abs(exp)
    scale = max(float(np.max(np.abs(ge))), 1e-300)
    assert float(np.max(np.abs(g - ge))) <= TRACK_RTOL * scale
    v, bcv = track_loss(ctl, data, t_t, w, 0.1, 0.05, rk4)
    assert v == got and bcv == 0


def test_track_loss_blowup_charges_cap():
    from oracle_bind import ref_track_loss
    from paper_2605_25346_b200.api import track_loss
    from train_cases import ct_tracking_case
    ctl, data = ct_tracking_case()
    ctl.layers[-1].b[0] += 1e160  # thrust blows the rollout up
    w = horizon_weights(3)
    got, bc = track_loss(ctl, data, 3, w, 0.1, 0.05, 2, cap=1e6)
    exp, bce = ref_track_loss(ctl, data, 3, w, 0.1, 0.05, 2, cap=1e6)
    assert bc == bce == len(data) and got == exp


@pytest.mark.parametrize("lam", [0.0, 0.5])
def test_train_ct_ctl_matches_reference(lam):
    """train_ct_ctl (training.hpp:389-442): track_loss + lambda ctl_reach_loss, both gradients on the device.
    The CT values agree to ~1e-15 and the gradients to ~1e-16..1e-9 (CUDA transcendentals), so the log within
    1e-9 relative and the trained parameters' update within 1e-6 of the reference's."""
    from oracle_bind import ref_train_ct_ctl
    from paper_2605_25346_b200.api import train_ct_ctl
    from train_cases import ct_tracking_case
    ctl, data = ct_tracking_case(seed=4, episodes=4, length=3)
    from paper_2605_25346_b200.api import TrainConfig
    cfg = TrainConfig(horizon_max=2, eps0=0.01, eps_final=0.005, lambda_=lam, gamma=0.1, iters=3, batch=2, lr=1e-3,
                      reach_cap=40.0, curriculum=True, seed=7)
    net, rows = train_ct_ctl(ctl, cfg, data, delta=0.02, k_atomic=2, rk4_substeps=2)
    pe, rows_e, rc = ref_train_ct_ctl(ctl, cfg, data, delta=0.02, k_atomic=2, rk4=2)
    assert rc == 0 and len(rows) == len(rows_e)
    for a, b in zip(rows, rows_e):
        assert (a.iter, a.t_h, a.eps, a.diverged_count) == (b.iter, b.t_h, b.eps, b.diverged_count)
        for x, y in ((a.l_pred, b.l_pred), (a.l_reach, b.l_reach), (a.l_total, b.l_total)):
            assert abs(x - y) <= 1e-9 * max(abs(y), 1e-300)
    du, de = net.params() - ctl.params(), pe - ctl.params()
    assert float(np.max(np.abs(du - de))) <= 1e-6 * float(np.max(np.abs(de)))
    if lam > 0:
        assert rows[-1].l_reach > 0


def _tanh_case():
    """The reference CLI's train-dt task shape (reach_cli.cpp:355-383): a tanh one-step model trained on a
    damped rotation with a scalar forcing input."""
    from paper_2605_25346_b200.api import Act, Episode
    from paper_2605_25346_b200.workloads import random_mlp
    rng = np.random.default_rng(4)
    model = random_mlp(rng, 3, [16], 2, Act.Tanh, 0.5)
    th, damp = 0.3, 0.95
    data = []
    for _ in range(6):
        x = rng.uniform(-0.5, 0.5, 2)
        xs, us = [x.copy()], []
        for _ in range(4):
            u = rng.uniform(-0.3, 0.3, 1)
            x = np.array([damp * (x[0] * np.cos(th) - x[1] * np.sin(th)) + 0.1 * u[0],
                          damp * (x[0] * np.sin(th) + x[1] * np.cos(th))])
            xs.append(x.copy())
            us.append(u)
        data.append(Episode(xs, us))
    return model, data


def test_pred_loss_tanh_within_tolerance():
    """tanh through CUDA's libm: values and gradients within 1e-12 / 1e-10 of the reference's."""
    model, data = _tanh_case()
    w = horizon_weights(3)
    got, g = pred_loss(model, data, 3, w, with_grad=True)
    exp, ge = ref_pred_loss(model, data, 3, w, with_grad=True)
    assert abs(got - exp) <= 1e-12 * abs(exp)
    assert float(np.max(np.abs(g - ge))) <= 1e-10 * float(np.max(np.abs(ge)))


def test_train_dt_dyn_tanh_task_matches_reference():
    """The CLI's bundled train-dt configuration (tanh model, lambda = 0.5 through the Dual tanh relaxations)."""
    from paper_2605_25346_b200.api import TrainConfig
    model, data = _tanh_case()
    cfg = TrainConfig(horizon_max=3, eps0=0.1, eps_final=0.01, lambda_=0.5, iters=3, batch=4, lr=1e-3, seed=0)
    net, rows = train_dt_dyn(model, cfg, data)
    pe, rows_e, rc = ref_train_dt_dyn(model, cfg, data)
    assert rc == 0 and len(rows) == len(rows_e)
    for a, b in zip(rows, rows_e):
        assert (a.iter, a.t_h, a.eps, a.diverged_count) == (b.iter, b.t_h, b.eps, b.diverged_count)
        for x, y in ((a.l_pred, b.l_pred), (a.l_reach, b.l_reach), (a.l_total, b.l_total)):
            assert abs(x - y) <= 1e-10 * max(abs(y), 1e-300)
    du, de = net.params() - model.params(), pe - model.params()
    assert float(np.max(np.abs(du - de))) <= 1e-6 * float(np.max(np.abs(de)))
