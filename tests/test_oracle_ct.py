"""CPU: the C restatement of cl_reach (oracle/ct_oracle.c) pinned bit for bit to the
reference itself (oracle/_ref: cl_reach and reach_with_splitting compiled from the
unmodified reference headers)."""
import numpy as np
import pytest

from ct_cases import ct_cases, ct_split_case
from oracle_bind import (assert_tubes_equal, oracle_cl_batch, oracle_cl_split_hull, ref_available, ref_cl_batch,
                         ref_cl_split_hull, same_bits)

needs_ref = pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built (needs /root/reference)")


@needs_ref
@pytest.mark.parametrize("case", ct_cases(), ids=lambda c: c[0])
def test_cl_oracle_matches_reference(case):
    name, spec, lo, hi, expect_fail = case
    exp = ref_cl_batch(spec, lo, hi, threads=1)
    got = oracle_cl_batch(spec, lo, hi)
    assert_tubes_equal(got, exp, exact=True)
    assert bool((exp.status != 0).any()) == expect_fail, (name, exp.status, exp.failed_step)


@needs_ref
def test_cl_split_hull_matches_reference_driver():
    spec, lo, hi, plan = ct_split_case()
    exp = ref_cl_split_hull(spec, lo, hi, plan)  # reach_with_splitting verbatim
    got = oracle_cl_split_hull(spec, lo, hi, plan)
    assert got.n_boxes == exp.n_boxes == spec.steps()
    assert same_bits(got.lo, exp.lo) and same_bits(got.hi, exp.hi)
    assert got.fail_key == exp.fail_key
    # a sub-range equals the hull of the same parts through the reference pieces
    exp2 = ref_cl_split_hull(spec, lo, hi, plan, begin=2, end=7, threads=2)
    got2 = oracle_cl_split_hull(spec, lo, hi, plan, begin=2, end=7)
    assert same_bits(got2.lo, exp2.lo) and same_bits(got2.hi, exp2.hi)
