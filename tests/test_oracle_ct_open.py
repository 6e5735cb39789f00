"""CPU: the C restatement of ct_reach (oracle/ct_oracle.c) pinned bit for bit to the reference's
ct_reach with its own analytic fields (oracle/_ref), on the reference's flowpipe test configurations."""
import pytest

from ct_open_cases import ct_open_cases, ct_open_split_case
from oracle_bind import (assert_tubes_equal, oracle_ct_batch, oracle_ct_split_hull, ref_available, ref_ct_batch,
                         ref_ct_split_hull, same_bits)

needs_ref = pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built (needs /root/reference)")


@needs_ref
@pytest.mark.parametrize("case", ct_open_cases(), ids=lambda c: c[0])
def test_ct_oracle_matches_reference(case):
    name, f, lo, hi, prm, expect_fail = case
    exp = ref_ct_batch(f, lo, hi, prm, threads=1)
    got = oracle_ct_batch(f, lo, hi, prm)
    assert_tubes_equal(got, exp, exact=True)
    assert bool((exp.status != 0).any()) == expect_fail, (name, exp.status)


@needs_ref
def test_ct_split_hull_matches_reference():
    f, lo, hi, plan, prm = ct_open_split_case()
    exp = ref_ct_split_hull(f, lo, hi, plan, prm, threads=2)
    got = oracle_ct_split_hull(f, lo, hi, plan, prm)
    assert got.n_boxes == exp.n_boxes == prm.steps + 1 and got.fail_key == exp.fail_key
    assert same_bits(got.lo, exp.lo) and same_bits(got.hi, exp.hi)
