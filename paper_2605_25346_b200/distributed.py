"""Multi-GPU sharding of the batch primitive (one process per GPU, torch.distributed).

The batch shards naturally: sub-boxes of a split plan or MPC
candidates are independent.  The only exchanges are
  * the per-step hull of reach_with_splitting (dt_reach or cl_reach engine):
    one all-reduce (min on lo, max on hi, min on the failure key / box count,
    max on the box-diverged flags);
  * CEM selection: one all-gather of each rank's (objective, ok) slice per
    iteration, after which every rank runs the identical stable sort / refit
    (every rank draws the same sampling stream, mpc.hpp:290-299).
With the NCCL backend these run on the GPU over NVLink; with gloo (tests) on
the CPU.  Evaluation is pluggable so the sharding logic is testable without a
GPU (tests pass the CPU oracle); the product path evaluates on the device.
"""
from __future__ import annotations

from typing import Callable, Optional, Tuple

import numpy as np

from . import _abi as A


def shard_range(total: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous [begin, end) slice of `total` items for `rank` (sizes differ by at most 1)."""
    base, rem = divmod(total, world)
    begin = rank * base + min(rank, rem)
    return begin, begin + base + (1 if rank < rem else 0)


def _dist():
    import torch.distributed as dist
    return dist


def _device_for(group) -> "object":
    import torch
    dist = _dist()
    backend = dist.get_backend(group)
    if backend == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def combine_hulls(partials):
    """Reference-order combination of partial hulls (list of HullResult, ascending part ranges)."""
    lo = partials[0].lo.copy()
    hi = partials[0].hi.copy()
    for p in partials[1:]:
        lo = np.where(p.lo < lo, p.lo, lo)  # std::min(a, b) = (b < a) ? b : a
        hi = np.where(hi < p.hi, p.hi, hi)
    nb = min(p.n_boxes for p in partials)
    key = min(p.fail_key for p in partials)
    div = np.max(np.stack([p.box_diverged for p in partials]), axis=0)
    return lo, hi, div, nb, key


def empty_hull(rows: int, n: int, h: float = 0.0):
    """The identity of the hull all-reduce: a rank with an empty part range contributes nothing
    (lo = +inf, hi = -inf, no failure, the largest box count)."""
    from .api import HullResult
    return HullResult(np.full((rows, n), np.inf), np.full((rows, n), -np.inf), np.zeros(rows, np.int32),
                      np.iinfo(np.int32).max, np.iinfo(np.int64).max, h)


def allreduce_hull(res, group=None):
    """All-reduces a rank's partial HullResult in place (NaN only survives from part 0, as the reference)."""
    import torch
    dist = _dist()
    dev = _device_for(group)
    nan0 = np.isnan(res.lo)
    nan0h = np.isnan(res.hi)
    lo = torch.tensor(np.where(nan0, np.inf, res.lo), device=dev)
    hi = torch.tensor(np.where(nan0h, -np.inf, res.hi), device=dev)
    meta = torch.tensor([res.n_boxes, res.fail_key], dtype=torch.int64, device=dev)
    div = torch.tensor(res.box_diverged.astype(np.int64), device=dev)
    dist.all_reduce(lo, op=dist.ReduceOp.MIN, group=group)
    dist.all_reduce(hi, op=dist.ReduceOp.MAX, group=group)
    dist.all_reduce(meta, op=dist.ReduceOp.MIN, group=group)
    dist.all_reduce(div, op=dist.ReduceOp.MAX, group=group)
    # the rank holding part 0 (rank 0) shares its NaN mask: reference NaN iff part 0's value is NaN
    rank = dist.get_rank(group)
    own = np.stack([nan0, nan0h]).astype(np.int64) if rank == 0 else np.zeros((2,) + res.lo.shape, np.int64)
    mask = torch.tensor(own, device=dev)
    dist.all_reduce(mask, op=dist.ReduceOp.MAX, group=group)
    m = mask.cpu().numpy().astype(bool)
    lo = torch.where(torch.tensor(m[0], device=dev), torch.full_like(lo, float("nan")), lo)
    hi = torch.where(torch.tensor(m[1], device=dev), torch.full_like(hi, float("nan")), hi)
    res.lo = lo.cpu().numpy()
    res.hi = hi.cpu().numpy()
    res.n_boxes = int(meta[0])
    res.fail_key = int(meta[1])
    res.box_diverged = div.cpu().numpy().astype(np.int32)
    return res


def sharded_split_hull(sys, x0, plan, actions, prm, group=None,
                       evaluate: Optional[Callable] = None, ctx=None):
    """reach_with_splitting over all ranks: each evaluates its contiguous part range, then one all-reduce."""
    dist = _dist()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    total = plan.total_parts()
    b, e = shard_range(total, rank, world)
    if evaluate is None:
        from .api import reach_split_hull

        def evaluate(sys_, x0_, plan_, acts_, prm_, begin, end):
            return reach_split_hull(sys_, x0_, plan_, acts_, prm_, part_begin=begin, part_end=end, ctx=ctx)
    if e <= b:  # more ranks than parts: this rank contributes the identity of the reduction
        res = empty_hull(len(actions) + 1, sys.n)
    else:
        res = evaluate(sys, x0, plan, actions, prm, b, e)
    return allreduce_hull(res, group)


def sharded_cl_split_hull(spec, x0, plan, group=None, evaluate: Optional[Callable] = None, ctx=None):
    """reach_with_splitting(cl_reach) over all ranks (C2): contiguous part ranges, one all-reduce."""
    dist = _dist()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    b, e = shard_range(plan.total_parts(), rank, world)
    if evaluate is None:
        from .api import cl_split_hull

        def evaluate(spec_, x0_, plan_, begin, end):
            return cl_split_hull(spec_, x0_, plan_, part_begin=begin, part_end=end, ctx=ctx)
    if e <= b:
        return allreduce_hull(empty_hull(spec.steps(), spec.n + spec.l, spec.fp.h), group)
    return allreduce_hull(evaluate(spec, x0, plan, b, e), group)


def sharded_plan_cem(prob, cfg, x0, group=None, evaluate: Optional[Callable] = None,
                     refine: Optional[Callable] = None, ctx=None):
    """plan_cem (mpc.hpp:258-368) over all ranks; returns (actions, objective, best_effort, history).

    Every rank draws the full population (same stream), evaluates its slice,
    and all-gathers (objective, ok) -- identical selection on every rank.  The top
    candidate's gradient refinement (refine_iters > 0) is deterministic, so every rank
    runs it on its own device (no collective) and all ranks keep the same plan."""
    import dataclasses

    import torch
    from .mpc import CEM, plan_eval_batch, plan_refine
    dist = _dist()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    dev = _device_for(group)
    if evaluate is None:
        def evaluate(prob_, x0_, acts_):
            r = plan_eval_batch(prob_, x0_, acts_, ctx=ctx)
            return r.objective, r.diverged
    cem = CEM(prob, dataclasses.replace(cfg, refine_iters=0))
    pop = cfg.population
    b, e = shard_range(pop, rank, world)
    sizes = [shard_range(pop, r, world) for r in range(world)]
    width = max(hi - lo for lo, hi in sizes)
    for _ in range(cfg.iterations):
        cands = cem.sample()
        obj, div = evaluate(prob, x0, cands[b:e])
        local = torch.zeros((width, 2), dtype=torch.float64, device=dev)
        local[: e - b, 0] = torch.as_tensor(obj, dtype=torch.float64)
        local[: e - b, 1] = torch.as_tensor((~np.asarray(div, bool)).astype(np.float64))
        gathered = [torch.zeros_like(local) for _ in range(world)]
        dist.all_gather(gathered, local, group=group)
        scores = np.concatenate([g[: hi - lo, 0].cpu().numpy() for g, (lo, hi) in zip(gathered, sizes)])
        ok = np.concatenate([g[: hi - lo, 1].cpu().numpy() for g, (lo, hi) in zip(gathered, sizes)]) > 0.5
        cem.update(scores, ok.astype(np.int32))
    best, best_obj, best_effort, hist = cem.result()
    if cfg.refine_iters > 0 and np.isfinite(best_obj):
        if refine is None:
            def refine(prob_, x0_, acts_, obj_, iters_):
                return plan_refine(prob_, x0_, acts_, obj_, iters_, ctx=ctx)[0]
        best = refine(prob, x0, best, best_obj, cfg.refine_iters)
    fin, _ = evaluate(prob, x0, best[None])
    return best, float(fin[0]), best_effort, hist


def sharded_grad_tube_volume(sys, x0, actions, target, method=0, prm=None, group=None,
                             evaluate: Optional[Callable] = None, ctx=None):
    """grad_tube_volume (refine.hpp:263-311) over all ranks: the parameters (one forward-dual pass, or two
    central-difference passes, each -- independent) are split into contiguous slices, each rank runs its
    slice's passes in one launch, one all-gather assembles the gradient; the subgradient flag is OR-ed.
    evaluate(sys, x0, actions, target, method, prm, begin, end) -> (g_slice, subgradient)."""
    import torch
    from .api import DTReachParams, GradMethod, GradTarget, Gradient, grad_tube_volume
    dist = _dist()
    prm = prm or DTReachParams()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    target = GradTarget(target)
    full = {GradTarget.x0_center: sys.n, GradTarget.actions: len(actions) * sys.m,
            GradTarget.weights: int(sys.step.params().size)}[target]
    b, e = shard_range(full, rank, world)
    if evaluate is None:
        def evaluate(s_, x_, a_, t_, m_, p_, b_, e_):
            g = grad_tube_volume(s_, x_, a_, t_, m_, p_, param_range=(b_, e_), ctx=ctx)
            return g.g, g.subgradient
    g_slice, sub = evaluate(sys, x0, actions, target, method, prm, b, e)
    dev = _device_for(group)
    width = max(shard_range(full, r, world)[1] - shard_range(full, r, world)[0] for r in range(world))
    buf = torch.zeros(width + 1, dtype=torch.float64, device=dev)
    buf[: e - b] = torch.from_numpy(np.ascontiguousarray(g_slice, dtype=np.float64))
    buf[width] = 1.0 if sub else 0.0
    outs = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(outs, buf, group=group)
    parts, any_sub = [], False
    for r, o in enumerate(outs):
        rb_, re_ = shard_range(full, r, world)
        parts.append(o[: re_ - rb_].cpu().numpy())
        any_sub = any_sub or bool(o[width].item() != 0.0)
    return Gradient(np.concatenate(parts) if parts else np.zeros(0), GradMethod(method), any_sub)


def torch_collectives(ctx, group=None):
    """Gives `ctx` the collectives of a torch.distributed group (gloo or NCCL process groups; the
    library's device buffers are staged through host tensors).  Afterwards reach_split_hull,
    cl_split_hull, ct_split_hull and plan_cem on `ctx` shard over the group inside the library
    (include/reach_b200.h, "Multi-GPU") -- the C-ABI counterpart of the sharded_* helpers above."""
    import torch
    dist = _dist()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    dev = _device_for(group)
    sign = np.uint64(1 << 63)

    def allreduce(a, op):
        u64 = a.dtype == np.uint64
        v = (a ^ sign).view(np.int64) if u64 else a  # order keys: flip the sign bit, compare as int64
        t = torch.from_numpy(np.ascontiguousarray(v)).to(dev)
        dist.all_reduce(t, op=dist.ReduceOp.MIN if op == "min" else dist.ReduceOp.MAX, group=group)
        r = t.cpu().numpy()
        return (r.view(np.uint64) ^ sign) if u64 else r

    def allgather(a):
        t = torch.from_numpy(np.ascontiguousarray(a)).to(dev)
        out = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(out, t, group=group)
        return np.concatenate([o.cpu().numpy() for o in out])

    ctx.set_collectives(rank, world, allreduce, allgather)
    return ctx


def nccl_collectives(ctx, group=None):
    """Gives `ctx` the library's built-in NCCL communicator over the ranks of `group` (the unique id
    travels by torch.distributed.broadcast_object_list)."""
    from ._native import nccl_unique_id
    dist = _dist()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    obj = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    ctx.init_nccl(obj[0], world, rank)
    return ctx
