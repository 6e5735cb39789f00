"""GPU: mpc_run (mpc.hpp:425-495) around the device planner against the reference itself (oracle/_ref):
success / violated / steps_used / final state bit-identical and the run log (MPCResult::log_to_csv,
%.17g) byte-identical, with action and state disturbances, goal dims, gradient refinement on and off."""
import dataclasses

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from mpc_cases import integrator_problem, relu_problem
from oracle_bind import ref_available, ref_mpc_run, same_bits
from paper_2605_25346_b200.mpc import MPCConfig, SamplerConfig, mpc_run

needs_ref = pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")


def _runs():
    integ = integrator_problem(horizon=6)
    relu = relu_problem(horizon=6)
    return [
        ("integrator_disturbed", integ, SamplerConfig(population=32, iterations=2, refine_iters=0, seed=5),
         MPCConfig(replan_period=2, total_steps=9, dist_action=0.01, dist_state=0.005, goal_radius=0.05, seed=9),
         np.array([-0.4, 0.3])),
        ("integrator_refine_goal_dims", integ, SamplerConfig(population=24, iterations=2, refine_iters=5, seed=1),
         MPCConfig(replan_period=3, total_steps=12, dist_action=0.02, goal_dims=[0], goal_radius=0.1, seed=4),
         np.array([0.0, 0.0])),
        ("relu_refine", relu, SamplerConfig(population=48, iterations=3, refine_iters=5, seed=3),
         MPCConfig(replan_period=2, total_steps=8, dist_state=0.01, goal_radius=0.05, seed=2),
         np.array([0.05, -0.05, 0.0])),
    ]


@needs_ref
@pytest.mark.parametrize("run", _runs(), ids=lambda r: r[0])
def test_mpc_run_matches_reference(run):
    name, prob, sampler, cfg, x0 = run
    es, ev, eu, ef, ecsv = ref_mpc_run(prob, sampler, cfg, x0)
    r = mpc_run(prob, sampler, cfg, x0)
    assert (r.success, r.violated, r.steps_used) == (es, ev, eu)
    assert same_bits(r.final_state, ef)
    assert r.log_to_csv() == ecsv


@needs_ref
def test_host_simulator_callback():
    """A user simulator (the reference's Sim template argument): x + u reproduces the integrator model."""
    name, prob, sampler, cfg, x0 = _runs()[0]
    calls = []

    def sim(x, u):
        calls.append(1)
        return x + u

    es, ev, eu, ef, ecsv = ref_mpc_run(prob, sampler, cfg, x0)
    r = mpc_run(prob, sampler, cfg, x0, sim=sim)
    assert len(calls) == r.steps_used
    assert r.log_to_csv() == ecsv and same_bits(r.final_state, ef)


def test_simulator_divergence_ends_the_run():
    name, prob, sampler, cfg, x0 = _runs()[0]
    r = mpc_run(prob, sampler, cfg, x0, sim=lambda x, u: np.full_like(x, np.inf))
    assert r.steps_used == 1 and not r.success and len(r.log) == 1
    assert np.all(np.isinf(r.final_state))


def test_invalid_config_raises():
    name, prob, sampler, cfg, x0 = _runs()[0]
    with pytest.raises(ValueError):
        mpc_run(prob, sampler, dataclasses.replace(cfg, replan_period=prob.horizon + 1), x0)
    with pytest.raises(ValueError):
        mpc_run(prob, sampler, dataclasses.replace(cfg, goal_radius=0.0), x0)
