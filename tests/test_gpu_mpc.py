"""GPU: reachability-aware MPC (plan_eval / plan_cem) vs the CPU oracle and the reference."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from mpc_cases import plan_cases, small_cem
from oracle_bind import (oracle_dt_batch, oracle_plan_cem, oracle_plan_eval_batch, ref_available, ref_plan_cem,
                         same_bits, assert_tubes_equal)
from paper_2605_25346_b200.mpc import CEM, plan_cem, plan_eval_batch
from paper_2605_25346_b200.workloads import c3_tpushing


@pytest.mark.parametrize("case", plan_cases(), ids=lambda c: c[0])
def test_plan_eval_batch_matches_oracle(case):
    name, prob, x0, acts = case
    eo, ed = oracle_plan_eval_batch(prob, x0, acts)
    got = plan_eval_batch(prob, x0, acts, with_tubes=True)
    assert same_bits(got.objective, eo), np.max(np.abs(got.objective - eo))
    assert np.array_equal(got.diverged, ed)
    # the tubes are dt_reach from box_from_center(x0, eps)
    B = acts.shape[0]
    lo = np.repeat((x0 - prob.eps)[None], B, 0)
    hi = np.repeat((x0 + prob.eps)[None], B, 0)
    exp = oracle_dt_batch(prob.sys, lo, hi, acts, prob.dt_prm)
    assert_tubes_equal(got.tubes, exp, exact=True)


def test_plan_cem_matches_oracle():
    prob, cfg, x0 = small_cem()
    eb, eo, eh, ebe = oracle_plan_cem(prob, cfg, x0)
    r = plan_cem(prob, cfg, x0)
    assert same_bits(r.actions, eb) and r.objective == eo and same_bits(r.best_history, eh)
    assert r.best_effort == ebe


def test_cem_pieces_reproduce_plan_cem():
    prob, cfg, x0 = small_cem()
    r = plan_cem(prob, cfg, x0)
    cem = CEM(prob, cfg)
    for _ in range(cfg.iterations):
        cands = cem.sample()
        ev = plan_eval_batch(prob, x0, cands)
        cem.update(ev.objective, ~ev.diverged)
    best, obj, be, hist = cem.result()
    assert same_bits(best, r.actions) and same_bits(hist, r.best_history)


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")
def test_c3_full_replan_matches_reference():
    """BASELINE configs[2] at full size: 4096 candidates x H=20 x 5 CEM iterations."""
    prob, cfg, x0 = c3_tpushing()
    eb, eo, eh, ebe = ref_plan_cem(prob, cfg, x0)
    r = plan_cem(prob, cfg, x0)
    assert same_bits(r.actions, eb) and r.objective == eo and same_bits(r.best_history, eh)
    assert r.best_effort == ebe


def test_plan_cem_odd_draw_count_threaded_normals():
    from mpc_cases import odd_cem
    prob, cfg, x0 = odd_cem()
    eb, eo, eh, ebe = oracle_plan_cem(prob, cfg, x0)
    r = plan_cem(prob, cfg, x0)
    assert same_bits(r.actions, eb) and r.objective == eo and same_bits(r.best_history, eh)
    assert r.best_effort == ebe
    if ref_available():
        rb, ro, rh, rbe = ref_plan_cem(prob, cfg, x0)
        assert same_bits(r.actions, rb) and r.objective == ro
