"""CPU, world_size 2 over gloo: the multi-GPU sharding logic (shard ranges,
hull all-reduce, sharded CEM with all-gathered scores) reproduces the
single-process results bit for bit.  Evaluation runs on the CPU oracle here;
on the GPU box the same code evaluates through the CUDA library over NCCL."""
import os
import socket

import numpy as np
import pytest

from paper_2605_25346_b200.distributed import combine_hulls, shard_range


def test_shard_range_covers_exactly():
    for total in (1, 7, 64, 65536, 4097):
        for world in (1, 2, 3, 8):
            spans = [shard_range(total, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            assert max(e - b for b, e in spans) - min(e - b for b, e in spans) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist
    from mpc_cases import small_cem
    from oracle_bind import oracle_plan_eval_batch, oracle_split_hull
    from paper_2605_25346_b200.api import DTReachParams, DTSystem, SplitPlan
    from paper_2605_25346_b200.distributed import sharded_cl_split_hull, sharded_plan_cem, sharded_split_hull
    from paper_2605_25346_b200.workloads import residual_relu_dynamics
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(3)
        net = residual_relu_dynamics(rng, 4, 1, [32, 32], dt=0.1)
        sys_ = DTSystem(net, 4, 1)
        c = rng.uniform(-0.5, 0.5, 4)
        plan = SplitPlan([3, 2, 1, 4])
        acts = rng.uniform(-0.5, 0.5, size=(8, 1))

        def ev_hull(s, x0, p, a, prm, b, e):
            return oracle_split_hull(s, x0[0], x0[1], p, a, prm, b, e)
        h = sharded_split_hull(sys_, (c - 0.01, c + 0.01), plan, acts, DTReachParams(), evaluate=ev_hull)
        # one part over two ranks: rank 1's slice is empty and contributes the reduction's identity
        h1 = sharded_split_hull(sys_, (c - 0.01, c + 0.01), SplitPlan([1, 1, 1, 1]), acts, DTReachParams(),
                                evaluate=ev_hull)

        prob, cfg, x0 = small_cem()

        def ev_plan(p, x, a):
            return oracle_plan_eval_batch(p, x, a)
        best, obj, be, hist = sharded_plan_cem(prob, cfg, x0, evaluate=ev_plan)

        from ct_cases import ct_split_case
        from oracle_bind import oracle_cl_split_hull
        spec, clo, chi, cplan = ct_split_case()
        ch = sharded_cl_split_hull(spec, (clo, chi), cplan,
                                   evaluate=lambda s_, x_, p_, b_, e_: oracle_cl_split_hull(s_, x_[0], x_[1], p_, b_, e_))
        # grad_tube_volume sharded over the parameters (the slices come from the reference here)
        from grad_cases import grad_cases
        from oracle_bind import ref_available, ref_grad_tube_volume
        from paper_2605_25346_b200.distributed import sharded_grad_tube_volume
        gsys = gx0 = gacts = None
        gw = None
        if ref_available():
            _, gsys, gx0, gacts, gprm, _ = grad_cases()[2]

            def ev_grad(s_, x_, a_, t_, m_, p_, b_, e_):
                g, sub = ref_grad_tube_volume(s_, x_, a_, int(t_), int(m_), p_)
                return g[b_:e_], sub
            gw = sharded_grad_tube_volume(gsys, gx0, gacts, 2, 0, gprm, evaluate=ev_grad).g
        q.put((rank, h.lo, h.hi, h.n_boxes, h.fail_key, best, obj, be, hist, ch.lo, ch.hi, ch.n_boxes, ch.fail_key,
               gw, h1.lo, h1.hi, h1.n_boxes, h1.fail_key))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_sharding_matches_single_process():
    import multiprocessing as mp
    from mpc_cases import small_cem
    from oracle_bind import oracle_plan_cem, oracle_split_hull, same_bits
    from paper_2605_25346_b200.api import DTReachParams, DTSystem, SplitPlan
    from paper_2605_25346_b200.workloads import residual_relu_dynamics
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # single-process references
    rng = np.random.default_rng(3)
    net = residual_relu_dynamics(rng, 4, 1, [32, 32], dt=0.1)
    sys_ = DTSystem(net, 4, 1)
    c = rng.uniform(-0.5, 0.5, 4)
    plan = SplitPlan([3, 2, 1, 4])
    acts = rng.uniform(-0.5, 0.5, size=(8, 1))
    full = oracle_split_hull(sys_, c - 0.01, c + 0.01, plan, acts, DTReachParams())
    prob, cfg, x0 = small_cem()
    eb, eo, eh, ebe = oracle_plan_cem(prob, cfg, x0)
    from ct_cases import ct_split_case
    from oracle_bind import oracle_cl_split_hull
    spec, clo, chi, cplan = ct_split_case()
    cfull = oracle_cl_split_hull(spec, clo, chi, cplan)
    from grad_cases import grad_cases
    from oracle_bind import ref_available, ref_grad_tube_volume
    gfull = None
    if ref_available():
        _, gsys, gx0, gacts, gprm, _ = grad_cases()[2]
        gfull = ref_grad_tube_volume(gsys, gx0, gacts, 2, 0, gprm)[0]
    one = oracle_split_hull(sys_, c - 0.01, c + 0.01, SplitPlan([1, 1, 1, 1]), acts, DTReachParams())
    for rank, lo, hi, nb, key, best, obj, be, hist, clo_r, chi_r, cnb, ckey, gw, lo1, hi1, nb1, key1 in outs:
        assert nb1 == one.n_boxes and key1 == one.fail_key
        assert same_bits(lo1[:nb1], one.lo[:nb1]) and same_bits(hi1[:nb1], one.hi[:nb1])
        if gfull is not None:  # weights gradient assembled from two ranks' parameter slices
            assert same_bits(gw, gfull)
        k = full.n_boxes
        assert nb == full.n_boxes and key == full.fail_key
        assert same_bits(lo[:k], full.lo[:k]) and same_bits(hi[:k], full.hi[:k])
        assert same_bits(best, eb) and obj == eo and same_bits(hist, eh) and be == ebe
        # C2's continuous-time hull sharded over two ranks: identical to the single-process hull
        assert cnb == cfull.n_boxes and ckey == cfull.fail_key
        assert same_bits(clo_r, cfull.lo) and same_bits(chi_r, cfull.hi)


def test_combine_hulls_matches_full_oracle():
    from oracle_bind import oracle_split_hull, same_bits
    from paper_2605_25346_b200.api import DTReachParams, DTSystem, SplitPlan
    from paper_2605_25346_b200.workloads import residual_relu_dynamics
    rng = np.random.default_rng(4)
    net = residual_relu_dynamics(rng, 3, 0, [16], dt=0.1)
    sys_ = DTSystem(net, 3, 0)
    c = rng.uniform(-0.5, 0.5, 3)
    plan = SplitPlan([4, 3, 2])
    acts = np.zeros((6, 0))
    full = oracle_split_hull(sys_, c - 0.02, c + 0.02, plan, acts)
    parts = [oracle_split_hull(sys_, c - 0.02, c + 0.02, plan, acts, DTReachParams(), b, e)
             for b, e in (shard_range(24, r, 3) for r in range(3))]
    lo, hi, div, nb, key = combine_hulls(parts)
    assert nb == full.n_boxes and key == full.fail_key
    assert same_bits(lo[:nb], full.lo[:nb]) and same_bits(hi[:nb], full.hi[:nb])
