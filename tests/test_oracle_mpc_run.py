"""CPU: the reference's mpc_run (mpc.hpp:425-495) as bound from oracle/_ref -- checked against its own
test_mpc.cpp properties before it serves as the GPU tests' checker: the log has one row per executed step,
replans every replan_period steps, logged actions stay in U, and a disturbance-free run is reproducible."""
import dataclasses

import numpy as np
import pytest

from mpc_cases import integrator_problem
from oracle_bind import ref_available, ref_mpc_run
from paper_2605_25346_b200.mpc import MPCConfig, SamplerConfig

pytestmark = pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")


def _rows(csv):
    lines = csv.strip().split("\n")
    assert lines[0] == "step,objective,tube_volume,g_margin,state,action"
    return [l.split(",") for l in lines[1:]]


def test_reference_mpc_run_log_shape():
    prob = integrator_problem(horizon=6)
    prob.constraints = prob.constraints[:3]
    sampler = SamplerConfig(population=32, iterations=2, refine_iters=0, seed=5)
    cfg = MPCConfig(replan_period=2, total_steps=7, dist_action=0.01, dist_state=0.005, goal_radius=0.05, seed=9)
    succ, viol, used, fin, csv = ref_mpc_run(prob, sampler, cfg, np.array([-0.4, 0.3]))
    rows = _rows(csv)
    assert len(rows) == used and 1 <= used <= 7
    assert [int(r[0]) for r in rows] == list(range(used))
    objs = [r[1] for r in rows]
    for k in range(0, used, 2):  # one plan per replan_period rows
        assert len(set(objs[k:k + 2])) == 1
    for r in rows:
        u = [float(v) for v in r[5].split(";")]
        assert all(-0.5 <= v <= 0.5 for v in u)
    again = ref_mpc_run(prob, sampler, cfg, np.array([-0.4, 0.3]))
    assert again[4] == csv
