"""CPU: pin the C restatement (oracle/liboracle.so) against the reference
itself (oracle/_ref, the unmodified headers) and the reference's golden file."""
import numpy as np
import pytest

from cases import cases, golden_fixture
from oracle_bind import (assert_tubes_equal, oracle_dt_batch, oracle_split_hull, ref_available, ref_dt_batch,
                         ref_split_hull, ref_reach_with_splitting, same_bits)
from paper_2605_25346_b200 import _abi as A
from paper_2605_25346_b200.api import DTReachParams, DTSystem, SplitPlan, affine_net
from paper_2605_25346_b200.workloads import residual_relu_dynamics

needs_ref = pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built (needs /root/reference)")


def test_golden_affine_decay_oracle():
    sys, lo, hi, acts, exp_lo, exp_hi, fx = golden_fixture()
    t = oracle_dt_batch(sys, lo, hi, acts)
    assert t.n_boxes[0] == fx["horizon"] + 1 and t.status[0] == 0
    assert same_bits(t.lo[0], exp_lo) and same_bits(t.hi[0], exp_hi)
    # byte-identical CSV text (tube_to_csv %.17g, io.hpp:108-130)
    for k in range(fx["horizon"] + 1):
        for d in range(fx["n"]):
            assert ["%.17g" % t.lo[0, k, d], "%.17g" % t.hi[0, k, d]] == fx["expected_csv_text"][f"{k},{d}"]


@needs_ref
def test_golden_affine_decay_ref():
    sys, lo, hi, acts, exp_lo, exp_hi, fx = golden_fixture()
    t = ref_dt_batch(sys, lo, hi, acts)
    assert same_bits(t.lo[0], exp_lo) and same_bits(t.hi[0], exp_hi)


@needs_ref
@pytest.mark.parametrize("case", cases(), ids=lambda c: c[0])
def test_oracle_matches_reference_bitwise(case):
    name, sys, lo, hi, acts, prm, _ = case
    exp = ref_dt_batch(sys, lo, hi, acts, prm, threads=1)
    got = oracle_dt_batch(sys, lo, hi, acts, prm)
    assert_tubes_equal(got, exp, exact=True)


@needs_ref
def test_explosive_case_exercises_failures():
    case = [c for c in cases() if c[0] == "explosive"][0]
    _, sys, lo, hi, acts, prm, _ = case
    t = ref_dt_batch(sys, lo, hi, acts, prm)
    assert (t.status != 0).any(), "explosive case should fail some tubes"


@needs_ref
@pytest.mark.parametrize("window", [4, 1])
def test_split_hull_oracle_matches_reference(window):
    rng = np.random.default_rng(3)
    net = residual_relu_dynamics(rng, 4, 1, [32, 32], dt=0.1)
    sys = DTSystem(net, 4, 1)
    c = rng.uniform(-0.5, 0.5, 4)
    plan = SplitPlan([3, 2, 1, 4])
    acts = rng.uniform(-0.5, 0.5, size=(8, 1))
    prm = DTReachParams(window=window)
    for begin, end in ((0, 0), (5, 19)):
        exp = ref_split_hull(sys, c - 0.01, c + 0.01, plan, acts, prm, begin, end, threads=2)
        got = oracle_split_hull(sys, c - 0.01, c + 0.01, plan, acts, prm, begin, end)
        assert got.n_boxes == exp.n_boxes and got.fail_key == exp.fail_key
        k = exp.n_boxes
        assert same_bits(got.lo[:k], exp.lo[:k]) and same_bits(got.hi[:k], exp.hi[:k])


@needs_ref
def test_split_hull_full_range_equals_reference_driver():
    """ref_split_hull reassembles reach_with_splitting's pieces (it needs a part range); on a full plan it
    must equal the reference driver itself bit for bit (refine.hpp:121-160)."""
    rng = np.random.default_rng(31)
    net = residual_relu_dynamics(rng, 4, 1, [32, 32], dt=0.1)
    sys = DTSystem(net, 4, 1)
    c = rng.uniform(-0.5, 0.5, 4)
    plan = SplitPlan([3, 2, 2, 3])
    acts = rng.uniform(-0.5, 0.5, size=(10, 1))
    lo, hi, nb, fs = ref_reach_with_splitting(sys, c - 0.02, c + 0.02, plan, acts)
    got = ref_split_hull(sys, c - 0.02, c + 0.02, plan, acts, threads=2)
    assert got.n_boxes == nb and fs == -1 and A.decode_fail_key(got.fail_key) is None
    assert same_bits(got.lo[:nb], lo[:nb]) and same_bits(got.hi[:nb], hi[:nb])


@needs_ref
def test_split_hull_failures_key():
    # an explosive system: the hull's failure is the earliest (step, part)
    rng = np.random.default_rng(9)
    from paper_2605_25346_b200.workloads import random_mlp
    from paper_2605_25346_b200.api import Act
    net = random_mlp(rng, 2, [16], 2, Act.Relu, 3.0)
    net.layers[-1].w *= 20.0
    sys = DTSystem(net, 2, 0)
    plan = SplitPlan([3, 3])
    exp = ref_split_hull(sys, np.array([-1.0, -1.0]), np.array([1.0, 1.0]), plan, np.zeros((150, 0)), threads=1)
    got = oracle_split_hull(sys, np.array([-1.0, -1.0]), np.array([1.0, 1.0]), plan, np.zeros((150, 0)))
    assert got.fail_key == exp.fail_key and got.n_boxes == exp.n_boxes
    assert A.decode_fail_key(exp.fail_key) is not None
