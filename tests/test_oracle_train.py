"""CPU: the reference's certified-training entry points through oracle/_ref (the ground truth of
tests/test_gpu_train.py) run, are deterministic, and behave as training.hpp documents."""
import numpy as np
import pytest

from oracle_bind import ref_available, ref_pred_loss, ref_train_dt_dyn
from paper_2605_25346_b200.api import horizon_weights
from train_cases import dt_training_case, train_config

needs_ref = pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")


@needs_ref
def test_ref_pred_loss_gradient_matches_finite_differences():
    model, data = dt_training_case()
    w = horizon_weights(3)
    loss, g = ref_pred_loss(model, data[:3], 3, w, with_grad=True)
    assert np.isfinite(loss) and loss > 0
    p = model.params()
    rng = np.random.default_rng(0)
    from paper_2605_25346_b200.api import net_with_params
    for j in rng.choice(p.size, 6, replace=False):
        h = 1e-6 * max(1.0, abs(p[j]))
        q = p.copy()
        q[j] += h
        fp = ref_pred_loss(net_with_params(model, q), data[:3], 3, w)
        q[j] -= 2 * h
        fm = ref_pred_loss(net_with_params(model, q), data[:3], 3, w)
        assert abs((fp - fm) / (2 * h) - g[j]) <= 1e-6 * max(1.0, abs(g[j]))


@needs_ref
def test_ref_train_dt_dyn_deterministic_and_logged():
    model, data = dt_training_case()
    cfg = train_config(iters=3)
    p1, rows1, rc1 = ref_train_dt_dyn(model, cfg, data)
    p2, rows2, rc2 = ref_train_dt_dyn(model, cfg, data)
    assert rc1 == 0 and rc2 == 0
    assert np.array_equal(p1, p2) and rows1 == rows2
    assert [r.iter for r in rows1] == [0, 1, 2]
    assert rows1[0].t_h == 1 and rows1[-1].t_h == cfg.horizon_max  # horizon_schedule anchors
    assert rows1[0].eps == cfg.eps0 and rows1[-1].eps == cfg.eps_final  # eps_schedule anchors
    assert not np.array_equal(p1, model.params())
