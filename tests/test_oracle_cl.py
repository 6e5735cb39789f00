"""CPU: the C restatement of the DT closed loop vs the reference composition (oracle/_ref)."""
import numpy as np
import pytest

from cl_cases import cl_cases
from oracle_bind import assert_tubes_equal, oracle_dtcl_batch, ref_available, ref_dtcl_batch

needs_ref = pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built (needs /root/reference)")


@needs_ref
@pytest.mark.parametrize("case", cl_cases(), ids=lambda c: c[0])
def test_dtcl_oracle_matches_reference(case):
    name, dyn, ctl, n, lo, hi, H, prm, _ = case
    exp = ref_dtcl_batch(dyn, ctl, n, lo, hi, H, prm, threads=1)
    got = oracle_dtcl_batch(dyn, ctl, n, lo, hi, H, prm)
    assert_tubes_equal(got, exp, exact=True)
    if name == "explosive":
        assert (exp.status != 0).any()
