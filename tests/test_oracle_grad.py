"""CPU: the reference's grad_tube_volume (refine.hpp:263-311) as bound from oracle/_ref, pinned by its own
test_refine.cpp properties (exact zeros on constant-volume objectives, forward-dual vs central differences)
before it serves as the GPU tests' checker."""
import numpy as np
import pytest

from grad_cases import grad_cases, identity_case
from oracle_bind import ref_available, ref_grad_tube_volume

pytestmark = pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")


def test_reference_constant_volume_zero_gradients():
    sys, trans, x0 = identity_case()
    g, sub = ref_grad_tube_volume(sys, x0, [[]] * 4, 0, 0)
    assert np.all(g == 0.0) and not sub
    g, _ = ref_grad_tube_volume(trans, x0, [[0.1, -0.2]] * 3, 1, 0)
    assert g.shape == (6,) and np.all(g == 0.0)


@pytest.mark.parametrize("case", [c for c in grad_cases() if c[0] != "c4_shape"], ids=lambda c: c[0])
def test_reference_forward_matches_finite_differences(case):
    name, sys, x0, acts, prm, exact = case
    targets = (2,) if name == "relu_weights_small" else (0, 1) if sys.m else (0, 2)
    for t in targets:
        gf, _ = ref_grad_tube_volume(sys, x0, acts, t, 0, prm)
        gd, _ = ref_grad_tube_volume(sys, x0, acts, t, 1, prm)
        err = np.max(np.abs(gf - gd) / np.maximum(1e-3, np.abs(gd)))
        assert err <= 1e-3, (name, t, err)
