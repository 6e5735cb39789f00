"""GPU: grad_tube_volume (refine.hpp:263-311) on the device -- forward-dual passes (grad_forward) and central
differences (grad_fd), every parameter's pass(es) in one launch -- against the reference itself
(oracle/_ref).  ReLU / identity maps: bit-identical gradients and subgradient flags; tanh maps (CUDA libm vs
host libm tanh): relative 1e-9."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from grad_cases import diverging_case, grad_cases, identity_case
from oracle_bind import ref_available, ref_grad_tube_volume, same_bits
from paper_2605_25346_b200._native import NonFiniteError
from paper_2605_25346_b200.api import GradMethod, GradTarget, grad_tube_volume, tube_volume, dt_reach

needs_ref = pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")
TANH_RTOL = 1e-9


def _targets(sys, acts):
    t = [GradTarget.x0_center, GradTarget.weights]
    if sys.m and len(acts):
        t.append(GradTarget.actions)
    return t


@needs_ref
@pytest.mark.parametrize("method", [GradMethod.forward_dual, GradMethod.finite_difference])
@pytest.mark.parametrize("case", grad_cases(), ids=lambda c: c[0])
def test_grad_tube_volume_matches_reference(case, method):
    name, sys, x0, acts, prm, exact = case
    for target in _targets(sys, acts):
        if name == "c4_shape" and target == GradTarget.weights and method == GradMethod.finite_difference:
            continue  # 2 x 34k passes: covered by the forward-dual weights pass
        exp = ref_grad_tube_volume(sys, x0, acts, int(target), int(method), prm)
        assert exp is not None
        got = grad_tube_volume(sys, x0, acts, target, method, prm)
        assert got.g.shape == exp[0].shape
        if exact:
            assert same_bits(got.g, exp[0]), (name, target, np.max(np.abs(got.g - exp[0])))
            assert got.subgradient == exp[1]
        else:
            err = np.abs(got.g - exp[0])
            if method == GradMethod.forward_dual:
                assert np.all(err <= TANH_RTOL * np.maximum(np.abs(exp[0]), 1e-12)), (name, target)
            else:  # central differences turn last-ulp tanh differences into ~eps / (2h) = 1e-11 absolute
                assert np.all(err <= 1e-9 + 1e-6 * np.abs(exp[0])), (name, target, err.max())


def test_constant_volume_objectives_have_exact_zero_gradients():
    """test_refine.cpp:195-217 on the device."""
    sys, trans, x0 = identity_case()
    g = grad_tube_volume(sys, x0, [[]] * 4, GradTarget.x0_center)
    assert g.g.shape == (2,) and np.all(g.g == 0.0) and not g.subgradient
    gfd = grad_tube_volume(sys, x0, [[]] * 4, GradTarget.x0_center, GradMethod.finite_difference)
    assert np.all(np.abs(gfd.g) <= 1e-9)
    ga = grad_tube_volume(trans, x0, [[0.1, -0.2]] * 3, GradTarget.actions)
    assert ga.g.shape == (6,) and np.all(ga.g == 0.0)


def test_volume_is_the_tube_volume():
    name, sys, x0, acts, prm, _ = grad_cases()[2]
    g = grad_tube_volume(sys, x0, acts, GradTarget.x0_center, prm=prm)
    assert g.volume == tube_volume(dt_reach(sys, x0, acts, prm))


def test_diverged_tube_raises_like_grad_forward():
    sys, x0, acts = diverging_case()
    with pytest.raises(NonFiniteError, match="non-finite"):
        grad_tube_volume(sys, x0, acts, GradTarget.x0_center)
    with pytest.raises(NonFiniteError, match="non-finite"):
        grad_tube_volume(sys, x0, acts, GradTarget.weights, GradMethod.finite_difference)


def test_unit_gain_radius_closed_form_via_center():
    """1-D identity over H steps: the volume (H+1) * 2r does not depend on the centre (zero gradient) and
    the weight gradient of the single gain is the closed form d/dw sum_k 2r w^k at w = 1: 2r * H(H+1)/2."""
    from paper_2605_25346_b200.api import DTSystem, affine_net
    H, r = 6, 0.17
    sys = DTSystem(affine_net(np.eye(1), np.zeros(1)), 1, 0)
    x0 = (np.array([0.25 - r]), np.array([0.25 + r]))
    g = grad_tube_volume(sys, x0, [[]] * H, GradTarget.weights)
    assert g.g.shape == (2,)
    assert abs(g.g[0] - 2 * r * H * (H + 1) / 2) <= 1e-10 * abs(g.g[0])
    assert g.g[1] == 0.0


@needs_ref
@pytest.mark.parametrize("target", [GradTarget.x0_center, GradTarget.actions])
def test_refine_tube_volume_matches_reference(target):
    """The reference CLI's refine (gradient_refine of the tube volume, reach_cli.cpp:293-341)."""
    from oracle_bind import ref_refine_tube_volume
    from paper_2605_25346_b200.api import refine_tube_volume
    name, sys, x0, acts, prm, _ = grad_cases()[2]
    c = (x0[0] + x0[1]) * 0.5
    eps = 0.08
    start = c if target == GradTarget.x0_center else np.asarray(acts, np.float64).reshape(-1)
    lo, hi = start - 0.5, start + 0.5
    exp = ref_refine_tube_volume(sys, c, eps, acts, int(target), lo, hi, iters=6)
    got = refine_tube_volume(sys, c, eps, acts, target, lo, hi, iters=6)
    assert same_bits(got.x, exp[0])
    assert (got.initial_objective, got.objective, got.progressed, got.subgradient, got.accepted_steps) == exp[1:]
    assert got.objective <= got.initial_objective


@pytest.mark.parametrize("method", [GradMethod.forward_dual, GradMethod.finite_difference])
def test_parameter_slices_assemble_the_full_gradient(method):
    """reach_grad_tube_volume_range (the multi-GPU shard unit): slices concatenate to the full gradient."""
    name, sys, x0, acts, prm, _ = grad_cases()[2]
    full = grad_tube_volume(sys, x0, acts, GradTarget.weights, method, prm)
    dim = full.g.size
    cuts = [0, 7, dim // 2, dim - 3, dim]
    parts = [grad_tube_volume(sys, x0, acts, GradTarget.weights, method, prm, param_range=(b, e)).g
             for b, e in zip(cuts[:-1], cuts[1:])]
    assert same_bits(np.concatenate(parts), full.g)
    with pytest.raises(ValueError):
        grad_tube_volume(sys, x0, acts, GradTarget.weights, method, prm, param_range=(5, dim + 1))


def test_refine_zero_gradient_start_returns_input_unchanged():
    """test_refine.cpp:286-299 on the tube-volume objective: the identity map's volume does not depend on
    the centre, so the gradient is exactly zero and gradient_refine stops without moving."""
    from paper_2605_25346_b200.api import refine_tube_volume
    sys_, _, x0 = identity_case()
    c = np.array([0.4, -0.3])
    r = refine_tube_volume(sys_, c, 0.2, [[]] * 4, GradTarget.x0_center, c - 1.0, c + 1.0, iters=5)
    assert not r.progressed and r.accepted_steps == 0
    assert r.objective == r.initial_objective and same_bits(r.x, c)


def test_refine_stays_in_the_box_and_never_worsens():
    from paper_2605_25346_b200.api import refine_tube_volume
    name, sys_, x0, acts, prm, _ = grad_cases()[2]
    c = (x0[0] + x0[1]) * 0.5
    lo, hi = c - 0.05, c + 0.05
    r = refine_tube_volume(sys_, c, 0.08, acts, GradTarget.x0_center, lo, hi, iters=10)
    assert r.objective <= r.initial_objective
    assert np.all(r.x >= lo) and np.all(r.x <= hi)
