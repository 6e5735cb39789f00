"""CPU: the reference's forward-dual gradient of plan_objective (grad_forward, refine.hpp:186-207) as bound
from oracle/_ref, pinned against central finite differences of the reference's own plan_eval; and
plan_cem's refinement flag plumbing (refine_iters = 0 reproduces plan_cem exactly)."""
import dataclasses

import numpy as np
import pytest

from mpc_cases import integrator_problem, relu_problem, small_cem
from oracle_bind import ref_available, ref_plan_cem, ref_plan_cem_ex, ref_plan_eval_batch, ref_plan_objective_grad

pytestmark = pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")


@pytest.mark.parametrize("which", ["integrator", "relu"])
def test_reference_grad_matches_finite_differences(which):
    prob = integrator_problem() if which == "integrator" else relu_problem()
    rng = np.random.default_rng(4)
    x0 = rng.uniform(-0.2, 0.2, prob.sys.n)
    acts = rng.uniform(0.5 * prob.u_lo, 0.5 * prob.u_hi, size=(prob.horizon, prob.sys.m))
    g = ref_plan_objective_grad(prob, x0, acts)
    assert g is not None and np.all(np.isfinite(g))
    h = 1e-6
    flat = acts.reshape(-1)
    pert = np.repeat(flat[None, :], 2 * flat.size, axis=0)
    for i in range(flat.size):
        pert[2 * i, i] += h
        pert[2 * i + 1, i] -= h
    obj, _ = ref_plan_eval_batch(prob, x0, pert.reshape(-1, prob.horizon, prob.sys.m))
    fd = (obj[0::2] - obj[1::2]) / (2 * h)
    # piecewise-smooth objective (ReLU kinks, max/min in the penalties): most coordinates agree tightly
    close = np.abs(fd - g.reshape(-1)) <= 1e-4 * (1 + np.abs(fd))
    assert close.mean() >= 0.9, (fd, g.reshape(-1))


def test_refine_zero_matches_plan_cem():
    prob, cfg, x0 = small_cem()
    a = ref_plan_cem(prob, cfg, x0)
    b = ref_plan_cem_ex(prob, cfg, x0)
    assert np.array_equal(a[0], b[0]) and a[1] == b[1] and np.array_equal(a[2], b[2]) and not b[4]


def test_refinement_never_worsens_objective():
    prob, cfg, x0 = small_cem()
    base = ref_plan_cem_ex(prob, cfg, x0)
    ref5 = ref_plan_cem_ex(prob, dataclasses.replace(cfg, refine_iters=5), x0)
    assert ref5[1] <= base[1]
    assert np.array_equal(ref5[2], base[2])  # the CEM history is untouched by the refinement
