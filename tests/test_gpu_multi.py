"""GPU: multi-GPU sharding inside the C ABI (reach_ctx_set_collectives / reach_ctx_init_nccl).
Two ranks share the one GPU of the test box (each its own ctx), combined over gloo through the
library's user-collectives hook; reach_split_hull, cl_split_hull and plan_cem then shard their batch
inside the library and every rank must return the single-GPU result bit for bit.  A one-rank NCCL
communicator checks the built-in NCCL path end to end."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problems():
    from ct_cases import ct_split_case
    from mpc_cases import odd_cem
    from paper_2605_25346_b200.api import DTSystem, SplitPlan
    from paper_2605_25346_b200.workloads import residual_relu_dynamics
    rng = np.random.default_rng(21)
    net = residual_relu_dynamics(rng, 6, 0, [64, 64], dt=0.1)
    sys_ = DTSystem(net, 6, 0)
    c = rng.uniform(-0.5, 0.5, 6)
    dt = (sys_, (c - 0.004, c + 0.004), SplitPlan([3, 2, 2, 1, 2, 3]), np.zeros((10, 0)))
    return dt, ct_split_case(), odd_cem()


def _run_all(ctx):
    from paper_2605_25346_b200.api import cl_split_hull, reach_split_hull
    from paper_2605_25346_b200.mpc import plan_cem
    (sys_, x0, plan, acts), (spec, clo, chi, cplan), (prob, cfg, px0) = _problems()
    h = reach_split_hull(sys_, x0, plan, acts, ctx=ctx)
    ch = cl_split_hull(spec, (clo, chi), cplan, ctx=ctx)
    r = plan_cem(prob, cfg, px0, ctx=ctx)
    return (h.lo, h.hi, h.n_boxes, h.fail_key, ch.lo, ch.hi, ch.n_boxes, ch.fail_key, r.actions, r.objective,
            r.best_history)


def _worker(rank, world, port, q):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, here)
    sys.path.insert(0, os.path.dirname(here))
    import torch.distributed as dist
    from paper_2605_25346_b200._native import Context
    from paper_2605_25346_b200.distributed import torch_collectives
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ctx = Context(0)
        torch_collectives(ctx)
        q.put((rank, _run_all(ctx)))
    finally:
        dist.destroy_process_group()


def _same(a, b):
    if isinstance(a, np.ndarray):
        return a.shape == b.shape and np.array_equal(a.view(np.uint8), b.view(np.uint8))
    return a == b


def test_two_ranks_shard_inside_the_library():
    import multiprocessing as mp
    from paper_2605_25346_b200._native import Context
    ref = _run_all(Context(0))
    mctx = mp.get_context("spawn")
    q = mctx.Queue()
    port = _port()
    procs = [mctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, got in outs:
        for g, e in zip(got, ref):
            assert _same(np.asarray(g), np.asarray(e)) if isinstance(e, np.ndarray) else g == e


def test_nccl_single_rank_matches():
    from paper_2605_25346_b200._native import Context, nccl_unique_id
    ref = _run_all(Context(0))
    ctx = Context(0)
    ctx.init_nccl(nccl_unique_id(), 1, 0)
    got = _run_all(ctx)
    for g, e in zip(got, ref):
        assert _same(np.asarray(g), np.asarray(e)) if isinstance(e, np.ndarray) else g == e
