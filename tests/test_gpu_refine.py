"""GPU: forward-dual gradients of the MPC objective (grad_forward, refine.hpp:186-207, of plan_objective,
mpc.hpp:204-208) and plan_cem's top-candidate gradient refinement (mpc.hpp:337-361, gradient_refine
refine.hpp:347-398; refine_iters = 5 is the reference default), checked against the reference itself
(oracle/_ref).  ReLU / identity networks: bit-identical gradients, plans, objectives and histories."""
import dataclasses

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from mpc_cases import integrator_problem, relu_problem, small_cem
from oracle_bind import ref_available, ref_plan_cem_ex, ref_plan_objective_grad, same_bits
from paper_2605_25346_b200.mpc import plan_cem, plan_objective_grad
from paper_2605_25346_b200.workloads import c3_tpushing

needs_ref = pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")


def _grad_cases():
    rng = np.random.default_rng(21)
    out = []
    for name, prob in (("integrator", integrator_problem()), ("relu", relu_problem())):
        for k in range(3):
            acts = rng.uniform(prob.u_lo, prob.u_hi, size=(prob.horizon, prob.sys.m))
            out.append((f"{name}_{k}", prob, rng.uniform(-0.3, 0.3, prob.sys.n), acts))
    prob, cfg, x0 = c3_tpushing(population=64, horizon=20)
    out.append(("c3_tpushing", prob, x0, np.clip(rng.normal(0.0, 0.3, size=(20, 2)), -1, 1)))
    return out


@needs_ref
@pytest.mark.parametrize("case", _grad_cases(), ids=lambda c: c[0])
def test_plan_objective_grad_matches_reference(case):
    name, prob, x0, acts = case
    exp = ref_plan_objective_grad(prob, x0, acts)
    assert exp is not None
    got, obj = plan_objective_grad(prob, x0, acts)
    assert same_bits(got, exp), (name, np.max(np.abs(got - exp)))
    assert np.isfinite(obj)


@needs_ref
@pytest.mark.parametrize("which", ["relu", "integrator"])
def test_plan_cem_with_refinement_matches_reference(which):
    prob, cfg, x0 = small_cem()
    if which == "integrator":
        prob = integrator_problem()
        x0 = np.array([0.1, -0.1])
    cfg = dataclasses.replace(cfg, refine_iters=5)
    eb, eo, eh, ebe, erf = ref_plan_cem_ex(prob, cfg, x0)
    r = plan_cem(prob, cfg, x0)
    assert same_bits(r.actions, eb) and r.objective == eo and same_bits(r.best_history, eh)
    assert r.best_effort == ebe and r.refined == erf


@needs_ref
def test_plan_cem_refinement_c3_shape_matches_reference():
    """BASELINE configs[2] network and constraints at a 256-candidate population, refine_iters = 5."""
    prob, cfg, x0 = c3_tpushing(population=256, horizon=20, iterations=3)
    cfg = dataclasses.replace(cfg, refine_iters=5)
    eb, eo, eh, ebe, erf = ref_plan_cem_ex(prob, cfg, x0)
    r = plan_cem(prob, cfg, x0)
    assert same_bits(r.actions, eb) and r.objective == eo and same_bits(r.best_history, eh)
    assert r.best_effort == ebe and r.refined == erf


def test_refine_step_alone_equals_plan_cem_refinement():
    """reach_plan_refine (the step the sharded CEM runs after its all-gathered loop) reproduces plan_cem."""
    from paper_2605_25346_b200.mpc import plan_refine
    prob, cfg, x0 = small_cem()
    r0 = plan_cem(prob, cfg, x0)
    r5 = plan_cem(prob, dataclasses.replace(cfg, refine_iters=5), x0)
    acts, refined = plan_refine(prob, x0, r0.actions, r0.objective, 5)
    assert same_bits(acts, r5.actions) and refined == r5.refined


def test_sharded_plan_cem_with_refinement_one_rank():
    import os
    import socket
    import torch.distributed as dist
    from paper_2605_25346_b200.distributed import sharded_plan_cem
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        prob, cfg, x0 = small_cem()
        cfg = dataclasses.replace(cfg, refine_iters=5)
        best, obj, be, hist = sharded_plan_cem(prob, cfg, x0)
        r = plan_cem(prob, cfg, x0)
        assert same_bits(best, r.actions) and obj == r.objective and same_bits(hist, r.best_history)
    finally:
        dist.destroy_process_group()
