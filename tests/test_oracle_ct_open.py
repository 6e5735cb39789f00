"""CPU: the C restatement of ct_reach (oracle/ct_oracle.c) pinned bit for bit to the reference's
ct_reach with its own analytic fields (oracle/_ref), on the reference's flowpipe test configurations."""
import pytest

from ct_open_cases import ct_open_cases
from oracle_bind import assert_tubes_equal, oracle_ct_batch, ref_available, ref_ct_batch

needs_ref = pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built (needs /root/reference)")


@needs_ref
@pytest.mark.parametrize("case", ct_open_cases(), ids=lambda c: c[0])
def test_ct_oracle_matches_reference(case):
    name, f, lo, hi, prm, expect_fail = case
    exp = ref_ct_batch(f, lo, hi, prm, threads=1)
    got = oracle_ct_batch(f, lo, hi, prm)
    assert_tubes_equal(got, exp, exact=True)
    assert bool((exp.status != 0).any()) == expect_fail, (name, exp.status)
