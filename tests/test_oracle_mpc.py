"""CPU: the C restatement of plan_eval / plan_cem vs the reference (oracle/_ref)."""
import numpy as np
import pytest

from mpc_cases import plan_cases, small_cem
from oracle_bind import (oracle_plan_cem, oracle_plan_eval_batch, ref_available, ref_plan_cem, ref_plan_eval_batch,
                         same_bits)

needs_ref = pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built (needs /root/reference)")


@needs_ref
@pytest.mark.parametrize("case", plan_cases(), ids=lambda c: c[0])
def test_plan_eval_oracle_matches_reference(case):
    name, prob, x0, acts = case
    eo, ed = ref_plan_eval_batch(prob, x0, acts, threads=1)
    go, gd = oracle_plan_eval_batch(prob, x0, acts)
    assert same_bits(go, eo)
    assert np.array_equal(gd, ed)
    if name == "explosive":
        assert ed.all()


@needs_ref
def test_plan_cem_oracle_matches_reference():
    prob, cfg, x0 = small_cem()
    eb, eo, eh, ebe = ref_plan_cem(prob, cfg, x0)
    gb, go, gh, gbe = oracle_plan_cem(prob, cfg, x0)
    assert same_bits(gb, eb) and go == eo and same_bits(gh, eh) and gbe == ebe
    assert np.all(np.diff(eh) <= 0)  # best objective is monotone non-increasing
