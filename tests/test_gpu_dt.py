"""GPU parity: the CUDA DT path through the C ABI vs the CPU oracle.

Bar: bit-identical to the reference for ReLU/identity networks (same
operation order and roundings); tanh networks within rtol 1e-9 (CUDA libm
vs glibc tanh).  Plus Monte-Carlo enclosure, batch determinism and the
split-hull driver at full C4 size via size-independent properties.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from cases import cases, golden_fixture
from oracle_bind import assert_tubes_equal, oracle_dt_batch, oracle_split_hull, same_bits
from paper_2605_25346_b200 import _abi as A
from paper_2605_25346_b200.api import (DTReachParams, DTSystem, SplitPlan, dt_reach, dt_reach_batch,
                                       dt_reach_batch_arrays, reach_split_hull, reach_with_splitting, split_box)
from paper_2605_25346_b200.workloads import c4_partition_sweep, residual_relu_dynamics

TANH_RTOL = 1e-9


@pytest.mark.parametrize("case", cases(), ids=lambda c: c[0])
def test_dt_batch_matches_oracle(case):
    name, sys, lo, hi, acts, prm, tanh = case
    exp = oracle_dt_batch(sys, lo, hi, acts, prm)
    got = dt_reach_batch_arrays(sys, lo, hi, acts, prm)
    assert_tubes_equal(got, exp, exact=not tanh, rtol=TANH_RTOL)


def test_golden_affine_decay_through_api():
    sys, lo, hi, acts, exp_lo, exp_hi, fx = golden_fixture()
    tube = dt_reach(sys, (lo[0], hi[0]), [np.zeros(0)] * fx["horizon"])
    assert tube.steps() == fx["horizon"] + 1 and not tube.diverged and tube.failed_step == -1
    assert same_bits(tube.lo, exp_lo) and same_bits(tube.hi, exp_hi)
    for k in range(tube.steps()):
        for d in range(fx["n"]):
            assert ["%.17g" % tube.lo[k, d], "%.17g" % tube.hi[k, d]] == fx["expected_csv_text"][f"{k},{d}"]


def test_failure_semantics_match_reference():
    case = [c for c in cases() if c[0] == "explosive"][0]
    _, sys, lo, hi, acts, prm, _ = case
    got = dt_reach_batch_arrays(sys, lo, hi, acts, prm)
    assert set(np.unique(got.status)) >= {A.TUBE_NONFINITE_PREACT, A.TUBE_DIVERGED_BOX}
    tubes = got.tubes()
    for t, st, fs in zip(tubes, got.status, got.failed_step):
        # diverged certification keeps k+1 boxes, diverged box keeps k+2 (dt_reach.hpp:64-67,94-99)
        if st == A.TUBE_DIVERGED_BOX:
            assert t.steps() == fs + 2 and t.box_diverged(t.steps() - 1)
        elif st != A.TUBE_OK:
            assert t.steps() == fs + 1
        assert t.diverged == (st != A.TUBE_OK)


def test_batch_bit_identity_order_equivariance_isolation():
    case = [c for c in cases() if c[0] == "c3_shape"][0]
    _, sys, lo, hi, acts, prm, _ = case
    full = dt_reach_batch_arrays(sys, lo, hi, acts, prm)
    perm = np.arange(lo.shape[0])[::-1].copy()
    rev = dt_reach_batch_arrays(sys, lo[perm], hi[perm], acts[perm], prm)
    assert same_bits(full.lo[perm], rev.lo) and same_bits(full.hi[perm], rev.hi)
    for b in (0, 5, 23):
        one = dt_reach_batch_arrays(sys, lo[b:b + 1], hi[b:b + 1], acts[b:b + 1], prm)
        assert same_bits(one.lo[0], full.lo[b]) and same_bits(one.hi[0], full.hi[b])
    # list API == array API
    tubes = dt_reach_batch(sys, [(lo[b], hi[b]) for b in range(3)], [list(acts[b]) for b in range(3)], prm)
    for b in range(3):
        assert same_bits(tubes[b].lo, full.lo[b])


def _mc_violations(sys, lo, hi, acts, tube_lo, tube_hi, n_samples, rng, slack=1e-12):
    viol = 0
    for b in range(lo.shape[0]):
        x = rng.uniform(lo[b], hi[b], size=(n_samples, sys.n))
        for k in range(acts.shape[1]):
            u = np.broadcast_to(acts[b, k], (n_samples, sys.m))
            h = np.concatenate([x, u], axis=1).T
            for L in sys.step.layers:
                h = L.w @ h + L.b[:, None]
                if int(L.act) == 0:
                    h = np.where(h < 0, 0.0, h)
                elif int(L.act) == 1:
                    h = np.tanh(h)
            x = h.T
            viol += int(np.sum(x < tube_lo[b, k + 1] - slack) + np.sum(x > tube_hi[b, k + 1] + slack))
    return viol


@pytest.mark.parametrize("name", ["c4_shape", "c3_shape", "random_relu_0", "tanh_16"])
def test_monte_carlo_enclosure(name):
    case = [c for c in cases() if c[0] == name][0]
    _, sys, lo, hi, acts, prm, _ = case
    t = dt_reach_batch_arrays(sys, lo, hi, acts, prm)
    assert np.all(t.status == 0)
    assert _mc_violations(sys, lo, hi, acts, t.lo, t.hi, 1000, np.random.default_rng(1)) == 0


def test_device_pointer_path_matches_host_path():
    import torch
    case = [c for c in cases() if c[0] == "c3_shape"][0]
    _, sys, lo, hi, acts, prm, _ = case
    host = dt_reach_batch_arrays(sys, lo, hi, acts, prm)
    from paper_2605_25346_b200._native import default_context
    import ctypes as C
    ctx = default_context()
    dev = torch.device("cuda:0")
    B, H1, n = host.lo.shape
    tl, th = torch.tensor(lo, device=dev), torch.tensor(hi, device=dev)
    ta = torch.tensor(acts, device=dev)
    olo = torch.zeros((B, H1, n), dtype=torch.float64, device=dev)
    ohi = torch.zeros_like(olo)
    nb = torch.zeros(B, dtype=torch.int32, device=dev)
    fs = torch.zeros_like(nb)
    st = torch.zeros_like(nb)
    args = A.DTArgs(B, H1 - 1, sys.n, sys.m, prm.window, int(prm.rebuild_from_box), A.dptr(tl.data_ptr()),
                    A.dptr(th.data_ptr()), A.dptr(ta.data_ptr()), 0)
    out = A.TubeOut(A.dptr(olo.data_ptr()), A.dptr(ohi.data_ptr()), A.iptr(nb.data_ptr()), A.iptr(fs.data_ptr()),
                    A.iptr(st.data_ptr()))
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    try:
        net = ctx.upload(sys.step)
        ctx.check(ctx._lib.reach_dt_batch(ctx.handle, net, C.byref(args), C.byref(out), A.REACH_FLAG_DEVICE_PTRS),
                  "dt")
        torch.cuda.synchronize()
    finally:
        ctx.set_stream(None)
    assert same_bits(olo.cpu().numpy(), host.lo) and same_bits(ohi.cpu().numpy(), host.hi)
    assert np.array_equal(nb.cpu().numpy(), host.n_boxes)


@pytest.mark.parametrize("window", [4, 1])
def test_split_hull_matches_oracle(window):
    rng = np.random.default_rng(3)
    net = residual_relu_dynamics(rng, 4, 1, [32, 32], dt=0.1)
    sys = DTSystem(net, 4, 1)
    c = rng.uniform(-0.5, 0.5, 4)
    plan = SplitPlan([3, 2, 1, 4])
    acts = rng.uniform(-0.5, 0.5, size=(8, 1))
    prm = DTReachParams(window=window)
    for begin, end in ((0, 0), (5, 19)):
        exp = oracle_split_hull(sys, c - 0.01, c + 0.01, plan, acts, prm, begin, end)
        got = reach_split_hull(sys, (c - 0.01, c + 0.01), plan, acts, prm, begin, end)
        assert got.n_boxes == exp.n_boxes and got.fail_key == exp.fail_key
        k = exp.n_boxes
        assert same_bits(got.lo[:k], exp.lo[:k]) and same_bits(got.hi[:k], exp.hi[:k])


def test_split_hull_failure_key_matches_oracle():
    from paper_2605_25346_b200.workloads import random_mlp
    from paper_2605_25346_b200.api import Act
    rng = np.random.default_rng(9)
    net = random_mlp(rng, 2, [16], 2, Act.Relu, 3.0)
    net.layers[-1].w *= 20.0
    sys = DTSystem(net, 2, 0)
    plan = SplitPlan([3, 3])
    x0 = (np.array([-1.0, -1.0]), np.array([1.0, 1.0]))
    exp = oracle_split_hull(sys, x0[0], x0[1], plan, np.zeros((150, 0)))
    got = reach_split_hull(sys, x0, plan, np.zeros((150, 0)))
    assert got.fail_key == exp.fail_key and got.n_boxes == exp.n_boxes
    tube = reach_with_splitting(sys, x0, plan, np.zeros((150, 0)))
    assert tube.diverged and tube.failure_reason.startswith("sub-box ")


def test_c4_full_size_properties():
    """BASELINE configs[3] at full size (65,536 sub-boxes, H=30)."""
    w = c4_partition_sweep()
    total = w.plan.total_parts()
    assert total == 65536
    full = reach_split_hull(w.sys, (w.x0_lo, w.x0_hi), w.plan, w.actions)
    assert full.n_boxes == w.horizon + 1 and full.fail_key == A.FAIL_KEY_NONE
    # box 0 of the hull is X0 exactly (split_box covers X0 exactly)
    assert same_bits(full.lo[0], w.x0_lo) and same_bits(full.hi[0], w.x0_hi)
    # shard consistency: hull of halves == hull of the whole (min/max is order independent)
    a = reach_split_hull(w.sys, (w.x0_lo, w.x0_hi), w.plan, w.actions, part_begin=0, part_end=total // 2)
    b = reach_split_hull(w.sys, (w.x0_lo, w.x0_hi), w.plan, w.actions, part_begin=total // 2, part_end=total)
    assert same_bits(np.minimum(a.lo, b.lo), full.lo) and same_bits(np.maximum(a.hi, b.hi), full.hi)
    # exact parity vs the oracle on a strided sample of sub-boxes (each one a full dt_reach)
    lo, hi = split_box(w.x0_lo, w.x0_hi, w.plan)
    idx = np.linspace(0, total - 1, 48).astype(int)
    exp = oracle_dt_batch(w.sys, lo[idx], hi[idx], np.zeros((len(idx), w.horizon, 0)))
    got = dt_reach_batch_arrays(w.sys, lo[idx], hi[idx], np.zeros((len(idx), w.horizon, 0)))
    assert_tubes_equal(got, exp, exact=True)
    # the hull encloses every sampled sub-tube, and Monte-Carlo rollouts from X0
    assert np.all(full.lo[None] <= got.lo) and np.all(got.hi <= full.hi[None])
    rng = np.random.default_rng(4)
    x = rng.uniform(w.x0_lo, w.x0_hi, size=(4000, 6))
    for k in range(w.horizon):
        x = w.sys.step.forward(x.T).T
        assert np.all(x >= full.lo[k + 1] - 1e-12) and np.all(x <= full.hi[k + 1] + 1e-12)


def test_invalid_arguments_raise_value_error():
    case = [c for c in cases() if c[0] == "c3_shape"][0]
    _, sys, lo, hi, acts, prm, _ = case
    with pytest.raises(ValueError):
        dt_reach_batch_arrays(DTSystem(sys.step, 4, 3), lo[:, :4], hi[:, :4], acts, prm)
    with pytest.raises(ValueError):
        dt_reach_batch_arrays(sys, lo, hi, acts[:, :, :1], prm)


def test_outward_rounding_flag_is_refused():
    """REACH_FLAG_OUTWARD_ROUNDING (the reference's g_outward_rounding) is refused, never ignored."""
    import ctypes as C
    from paper_2605_25346_b200 import _abi as A
    from paper_2605_25346_b200.api import default_context
    rng = np.random.default_rng(2)
    net = residual_relu_dynamics(rng, 2, 0, [8], dt=0.1)
    sys = DTSystem(net, 2, 0)
    ctx = default_context()
    lo, hi = np.array([[0.0, 0.1]]), np.array([[0.1, 0.2]])
    H = 3
    out_lo, out_hi = np.zeros((1, H + 1, 2)), np.zeros((1, H + 1, 2))
    nb, fs, st = np.zeros(1, np.int32), np.zeros(1, np.int32), np.zeros(1, np.int32)
    args = A.DTArgs(1, H, 2, 0, 4, 0, A.dptr(lo), A.dptr(hi), A.dptr(np.zeros(1)), 0)
    to = A.TubeOut(A.dptr(out_lo), A.dptr(out_hi), A.iptr(nb), A.iptr(fs), A.iptr(st))
    rc = ctx._lib.reach_dt_batch(ctx.handle, ctx.upload(net), C.byref(args), C.byref(to), A.REACH_FLAG_OUTWARD_ROUNDING)
    assert rc == A.REACH_E_UNSUPPORTED
    assert "outward rounding" in ctx._lib.reach_ctx_last_error(ctx.handle).decode()


def test_net_cache_sees_in_place_weight_updates():
    """Context.upload's same-object fast path: an unchanged net reuses its device handle, an in-place
    weight update uploads the new value (and the results follow it), restoring it hits the cache again."""
    from paper_2605_25346_b200 import Context
    rng = np.random.default_rng(7)
    net = residual_relu_dynamics(rng, 4, 0, [64, 64], dt=0.1)
    sys_ = DTSystem(net, 4, 0)
    ctx = Context(0)
    h0 = ctx.upload(net).value
    assert ctx.upload(net).value == h0
    c = rng.uniform(-0.5, 0.5, size=(3, 4))
    lo, hi = c - 0.01, c + 0.01
    acts = np.zeros((3, 5, 0))
    before = dt_reach_batch_arrays(sys_, lo, hi, acts, DTReachParams(), ctx=ctx)
    net.layers[1].w[3, 5] += 0.25
    assert ctx.upload(net).value != h0
    after = dt_reach_batch_arrays(sys_, lo, hi, acts, DTReachParams(), ctx=ctx)
    assert_tubes_equal(after, oracle_dt_batch(sys_, lo, hi, acts, DTReachParams()), exact=True)
    assert not np.array_equal(after.lo, before.lo)
    net.layers[1].w[3, 5] -= 0.25
    assert ctx.upload(net).value == h0
