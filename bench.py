#!/usr/bin/env python
"""Benchmark: certified reach-steps/s of the B200 DT reachability primitive.

Workload (default, BASELINE.json configs[3]): the initial-set partition sweep
-- 65,536 sub-boxes (8x8x8x8x4x4) of a 6-D system through a 3x128 ReLU
one-step map, horizon 30 -- i.e. reach_with_splitting(dt_reach) (refine.hpp:
121-160).  One "step" = one full sweep (65,536 sub-boxes x 30 DT steps) with
the per-step hull; a reach-step is one sub-box advanced one DT step.

  python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]

N > 1 (torchrun, one rank per GPU, NCCL): weak scaling -- the global plan is
N x 65,536 parts (first split count x N), each rank sweeps its own contiguous
65,536 parts, and the per-step hull is combined with one NCCL all-reduce
(min on lo / max on hi / min on the failure key), the path's only exchange.

Extra legs in the same JSON line (one per remaining BASELINE config):
ct_quadrotor (C2, continuous-time cl_reach sweep), c5_closed_loop (C5, 72-D DT
closed loop), c1_closed_loop (C1 latency at batch 1), mpc_replan (C3, ms per
replan) -- each with its CPU reference sample and parity note.

--impl reference: the reference's own CPU implementation (oracle/_ref, the
unmodified reference headers compiled -O2) on the host cores, each step a
bounded sample of the same sweep.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

METRIC = "certified reach-steps/sec (batch x horizon)"
UNIT = "reach-steps/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--cpu-sample-parts", type=int, default=0, help="parts per CPU sample (0 = auto)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-mpc", action="store_true", help="skip the C3 MPC replan leg")
    ap.add_argument("--no-grad", action="store_true", help="skip the grad_tube_volume leg")
    ap.add_argument("--no-ct", action="store_true", help="skip the C2 continuous-time closed-loop leg")
    ap.add_argument("--no-cl", action="store_true", help="skip the C5 / C1 DT closed-loop legs")
    ap.add_argument("--no-tc", action="store_true", help="skip the tensor-core precision-mode timings")
    ap.add_argument("--dist-dry-run", action="store_true", help="launcher logic check on CPU (gloo), no GPU work")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def _free_port() -> int:
    import socket
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return int(s.getsockname()[1])


def launch_command(argv, gpus: int, port: int):
    """The torchrun command that runs this script with one rank per GPU (the
    reference's fork-join parallel_for, parallel.hpp:17-37, becomes N processes)."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
            "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + list(argv)


def ensure_world(args, argv=None) -> int | None:
    """`--gpus N` without torchrun (WORLD_SIZE unset): re-exec under torch.distributed.run with N
    ranks and return its exit code.  Under torchrun the world size must equal --gpus.
    Returns None when the current process should run the benchmark itself."""
    env_world = os.environ.get("WORLD_SIZE")
    if env_world is None:
        if args.gpus <= 1:
            return None
        cmd = launch_command(sys.argv[1:] if argv is None else argv, args.gpus, _free_port())
        return subprocess.call(cmd)
    if int(env_world) != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={env_world} (torchrun "
                         f"--nproc-per-node must equal --gpus)")
    return None


def dist_dry_run(args):
    """--dist-dry-run: the N-rank launch / rendezvous / max-over-ranks path on CPU (gloo), no GPU
    work -- a logic check of the launcher, never a measurement."""
    import torch
    import torch.distributed as dist
    rank, world, _ = dist_env()
    if world > 1:
        dist.init_process_group("gloo")
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({"metric": METRIC, "dry_run": True, "n_gpus": world, "max_over_ranks": float(t[0]),
                          "config": {"parallelism": f"dp{world}"}}))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def algorithmic_flops_per_part(net_dims, n, m, H, window):
    """Algorithmic FP64 flops of one sub-box's H-step dt_reach:
    IBP (2 mul + 2 add per weight, hidden layers + prepend), the Lambda.W
    contractions (2 per MAC), the prepend Lambda.A and shift, relaxation
    chains (intercepts, scaling, shift: 7 per Lambda entry), and the fold
    solve (~6 n^3 when it runs).  I . W_out is excluded (a copy)."""
    L = len(net_dims) - 1
    cap = window if window > 0 else 1
    hidden = net_dims[1:L]
    total = 0
    nq = 0
    for k in range(H):
        nz = n * (1 + nq)
        f = 2 * n * nz + 2 * n  # prepend IBP
        f += 4 * n * net_dims[1] if L > 1 else 0  # layer 0 IBP (x columns)
        f += 2 * m * net_dims[1] if (L > 1 and m) else 0  # action fold
        for l in range(1, L - 1):
            f += 4 * net_dims[l] * net_dims[l + 1]
        # backward Lambda.W for l = L-2 .. 0
        for l in range(L - 2, -1, -1):
            cols = n if l == 0 else net_dims[l]
            f += 2 * n * net_dims[l + 1] * cols
        f += 7 * n * sum(hidden)  # relaxation chains
        f += 2 * n * n * nz + 2 * n * n  # prepend Lambda.A + shift
        nq += 1
        if nq > cap:
            f += 6 * n ** 3
            nq -= 1
        total += f
    return total


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def wait_first(self, timeout: float = 3.0):
        """Block until nvidia-smi has produced its first sample, so the sampling covers the timed region
        from its start (the tool takes a few hundred ms to come up; a short timed region could see none)."""
        t0 = time.time()
        while self.proc is not None and not self.lines and time.time() - t0 < timeout:
            time.sleep(0.01)

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], 0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def cpu_baseline(w, parts: int, threads: int = 0):
    """The reference itself (oracle/_ref) on `parts` sub-boxes of the sweep."""
    from oracle_bind import ref_available, ref_split_hull, ref_lib
    if not ref_available():
        return None
    lib = ref_lib()
    lib.ref_hardware_threads.restype = C.c_int
    cores = threads or int(lib.ref_hardware_threads())
    t0 = time.perf_counter()
    ref_split_hull(w.sys, w.x0_lo, w.x0_hi, w.plan, w.actions, begin=0, end=parts, threads=threads)
    dt = time.perf_counter() - t0
    return {"value": parts * w.horizon / dt, "unit": UNIT, "cores": cores, "kind": "reference",
            "sample": f"{parts} of {w.plan.total_parts()} sub-boxes x {w.horizon} steps through the reference "
                      f"reach_with_splitting pieces (oracle/_ref, g++ -O2), {dt:.2f} s"}


def auto_cpu_parts():
    cores = os.cpu_count() or 8
    # ~15 ms per sub-box-horizon per core (survey probe) -> aim at ~10-15 s
    return int(max(256, min(65536, cores * 800)))


def mpc_replan(args, ctx, world, rank, dev, barrier):
    """C3 T-pushing replan: 4096 candidates x H=20 x 5 CEM iterations + final plan_eval.
    N=1: the C++ host loop (reach_plan_cem); N>1: candidates sharded over the ranks with one
    NCCL all-gather of (objective, ok) per iteration.  Wall time of whole replans, max over ranks."""
    import torch
    from paper_2605_25346_b200.mpc import plan_cem
    from paper_2605_25346_b200.workloads import c3_tpushing
    prob, cfg, x0 = c3_tpushing()
    ctx.set_stream(None)

    def once():  # N > 1: the library shards the population (ctx collectives), same pipeline as N = 1
        r = plan_cem(prob, cfg, x0, ctx=ctx)
        return r.actions, r.objective

    reps = max(2, min(args.steps, 5))
    once()
    times = []
    for _ in range(reps):
        barrier()
        t0 = time.perf_counter()
        best, obj = once()
        times.append(time.perf_counter() - t0)
    t = float(np.mean(times))
    if world > 1:
        import torch.distributed as dist
        tt = torch.tensor([t], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = float(tt[0])
    steps = cfg.population * cfg.iterations * prob.horizon + prob.horizon
    out = {"workload": "c3_tpushing (BASELINE configs[2]): 4096 candidates x H=20 x 5 CEM iterations, "
                       "7->96x3->5 ReLU, eps=0.005, box-stay-in constraint, refine_iters=0",
           "ms_per_replan": 1e3 * t, "target_ms": 50.0, "replans_timed": reps,
           "reach_steps_per_s": steps / t, "objective": obj,
           "parity": "bit-identical plan/objective/history vs the reference plan_cem (tests/test_gpu_mpc.py)"}
    if world == 1:
        # the reference default refine_iters = 5: CEM + forward-dual gradient refinement of the top plan
        import dataclasses
        from paper_2605_25346_b200.mpc import plan_objective_grad
        cfg5 = dataclasses.replace(cfg, refine_iters=5)
        plan_cem(prob, cfg5, x0, ctx=ctx)
        tr = []
        for _ in range(reps):
            t0 = time.perf_counter()
            r5 = plan_cem(prob, cfg5, x0, ctx=ctx)
            tr.append(time.perf_counter() - t0)
        g_t = []
        for _ in range(5):
            t0 = time.perf_counter()
            plan_objective_grad(prob, x0, r5.actions, ctx=ctx)
            g_t.append(time.perf_counter() - t0)
        out["refine_iters_5"] = {"ms_per_replan": 1e3 * float(np.mean(tr)), "objective": r5.objective,
                                 "refined": r5.refined,
                                 "plan_objective_grad_ms": 1e3 * float(np.median(g_t)),
                                 "grad_directions": prob.horizon * prob.sys.m,
                                 "parity": "bit-identical plan / objective / refined flag vs the reference "
                                           "plan_cem with refinement (tests/test_gpu_refine.py)"}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            from oracle_bind import ref_available, ref_plan_cem, ref_lib
            if ref_available():
                t0 = time.perf_counter()
                ref_plan_cem(prob, cfg, x0)
                tc = time.perf_counter() - t0
                lib = ref_lib()
                lib.ref_hardware_threads.restype = C.c_int
                out["cpu_reference_ms_per_replan"] = 1e3 * tc
                out["cpu_reference_cores"] = int(lib.ref_hardware_threads())
        except Exception as ex:  # noqa: BLE001
            out["cpu_reference_error"] = str(ex)
    return out


def gradient_leg(args, ctx):
    """grad_tube_volume (refine.hpp:263-311) of the C4-shaped map (6->128x3->6 ReLU, H = 30, window 4):
    the weights target = 34,694 forward-dual passes in one launch.  CPU reference: the reference's
    grad_tube_volume on the 6-parameter x0_center target timed on one host core (grad_forward is
    serial), per pass, extrapolated to the weights target's pass count (said so in `cpu_reference`)."""
    from paper_2605_25346_b200.api import Act, DTSystem, GradTarget, grad_tube_volume
    from paper_2605_25346_b200.workloads import random_mlp
    rng = np.random.default_rng(1)
    net = random_mlp(rng, 6, [128, 128, 128], 6, Act.Relu, 0.9)
    net.layers[-1].w *= 0.5
    sys_ = DTSystem(net, 6, 0)
    x0 = (np.full(6, -0.05), np.full(6, 0.05))
    acts = [[]] * 30
    ctx.set_stream(None)
    ctx.enable_kernel_timing(True)
    grad_tube_volume(sys_, x0, acts, GradTarget.weights, ctx=ctx)
    ctx.kernel_time()
    t0 = time.perf_counter()
    g = grad_tube_volume(sys_, x0, acts, GradTarget.weights, ctx=ctx)
    wall = time.perf_counter() - t0
    km, _ = ctx.kernel_time()
    ctx.enable_kernel_timing(False)
    out = {"workload": "grad_tube_volume, weights target, 6->128x3->6 ReLU, H=30, window 4",
           "passes": int(g.g.size), "ms_per_gradient": 1e3 * wall, "kernel_ms": km,
           "passes_per_s": g.g.size / wall,
           "parity": "bit-identical to the reference grad_tube_volume (tests/test_gpu_grad.py)"}
    if not args.no_cpu_baseline:
        try:
            from oracle_bind import ref_available, ref_grad_tube_volume
            if ref_available():
                t0 = time.perf_counter()
                ref_grad_tube_volume(sys_, x0, acts, 0, 0)
                per_pass = (time.perf_counter() - t0) / 7.0  # 6 dual passes + the primal f0 pass
                out["cpu_reference"] = {"s_per_pass": per_pass, "cores": 1,
                                        "extrapolated_s_for_weights_target": per_pass * (g.g.size + 1),
                                        "sample": "x0_center target (7 passes) timed, per-pass cost extrapolated"}
        except Exception as ex:  # noqa: BLE001
            out["cpu_reference_error"] = str(ex)
    return out


def ct_flops_per_step(nz: int = 76, evals: float = 8.06) -> float:
    """Algorithmic FP64 work of one C2 flowpipe step, counted on the reference's own TMExpr
    operation sequence (taylor_model.hpp:245-445) for quadrotor_ode (systems.hpp:24-64):
    per field evaluation 23 products (10 flops per generator column + the 4 abs-sums of the
    operands' poly_range), 9 additions, 7 scalar products, 6 sin/cos and 3 reciprocals
    (total_range + scaling), 16 integrations and the Picard/replay/endpoint combinations;
    `evals` = measured field evaluations per step (2 Picard + remainder attempts + shrink
    replays + endpoint, oracle/ct_oracle.c counter on the C2 workload)."""
    mul = 14 * nz + 50
    add = 2 * nz + 4
    trig = 4 * nz + 20
    integ = nz + 10
    cons = 350 * nz / 76
    per_eval = 23 * mul + 9 * add + 7 * add + 6 * trig + 3 * trig + 16 * (integ + cons)
    return evals * per_eval + 3 * 16 * nz


def ct_sweep(args, ctx, world, rank, dev, barrier, stream):
    """C2 (BASELINE configs[1]): reach_with_splitting(cl_reach) of the quadrotor + 3x64 tanh
    controller, rpy:4096 sub-boxes x 50 flowpipe steps per GPU (weak scaling: x split N ways),
    one hull all-reduce for N > 1.  Device-resident hull output, CUDA events on the library's stream."""
    import torch
    import torch.distributed as dist
    from paper_2605_25346_b200 import _abi as A
    from paper_2605_25346_b200.api import SplitPlan, cl_split_hull
    from paper_2605_25346_b200.workloads import c2_quadrotor
    w = c2_quadrotor()
    spec = w.spec
    per_rank = w.plan.total_parts()
    counts = list(w.plan.counts)
    counts[0] *= world
    plan = SplitPlan(counts)
    begin, end = rank * per_rank, (rank + 1) * per_rank
    T, na = spec.steps(), spec.n + spec.l
    ctx.set_stream(stream.cuda_stream)
    d_lo = torch.empty(T * na, dtype=torch.float64, device=dev)
    d_hi = torch.empty(T * na, dtype=torch.float64, device=dev)
    d_div = torch.empty(T, dtype=torch.int32, device=dev)
    d_nb = torch.empty(1, dtype=torch.int32, device=dev)
    d_key = torch.empty(1, dtype=torch.int64, device=dev)
    cs, keep = spec.c_struct()
    cts = np.array(counts, dtype=np.int32)
    x0lo, x0hi = np.ascontiguousarray(w.x0_lo), np.ascontiguousarray(w.x0_hi)
    args_c = A.CLSplitArgs(A.dptr(x0lo), A.dptr(x0hi), A.iptr(cts), 0, 0)  # full plan; the library shards
    out_c = A.HullOut(A.dptr(d_lo.data_ptr()), A.dptr(d_hi.data_ptr()), A.iptr(d_div.data_ptr()),
                      A.iptr(d_nb.data_ptr()), A.lptr(d_key.data_ptr()))
    net = ctx.upload(spec.controller)

    def step():
        ctx.check(ctx._lib.reach_cl_split_hull(ctx.handle, net, C.byref(cs), C.byref(args_c), C.byref(out_c),
                                               A.REACH_FLAG_DEVICE_PTRS), "reach_cl_split_hull")

    for _ in range(max(args.warmup, 3)):
        step()
    barrier()
    reps = max(3, min(args.steps, 5))
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ctx.kernel_time()
    ms = []
    for _ in range(reps):
        ev0.record(stream)
        step()
        ev1.record(stream)
        ev1.synchronize()
        ms.append(ev0.elapsed_time(ev1))
    kern_ms, kern_n = ctx.kernel_time()
    t = float(np.mean(ms))
    if world > 1:
        tt = torch.tensor([t], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = float(tt[0])
    steps_total = per_rank * world * (T - 1)
    # end to end through the public API: host X0 / plan in, host hull out
    e2e = []
    for i in range(5):
        barrier()
        t0 = time.perf_counter()
        hres = cl_split_hull(spec, (w.x0_lo, w.x0_hi), plan, ctx=_host_ctx(ctx))
        if i >= 2:
            e2e.append(time.perf_counter() - t0)
    ctx.set_stream(stream.cuda_stream)
    te = float(np.mean(e2e))
    if world > 1:
        tt = torch.tensor([te], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        te = float(tt[0])
    fl = ct_flops_per_step()
    tf_fma, _ = ctx.fp64_peak()
    ach = fl * per_rank * (T - 1) / (t / 1e3) / 1e12
    out = {"workload": "c2_quadrotor (BASELINE configs[1]): reach_with_splitting(cl_reach), 12-D quadrotor_ode + "
                       "15->64x3->4 tanh controller, rpy:4096 sub-boxes per GPU, 10 control x 5 flowpipe steps, "
                       "h=0.01, order 2, window 4",
           "sub_boxes_per_gpu": per_rank, "ms_per_sweep": t, "reach_steps_per_s": steps_total / (t / 1e3),
           "launches_per_sweep": 2 * spec.ctl_steps + 2,
           "e2e": {"value": steps_total / te, "unit": UNIT, "h2d_bytes_per_step": 2 * 12 * 8 + 12 * 4 + 3 * 8 * spec.ctl_steps,
                   "d2h_bytes_per_step": 2 * T * 16 * 8 + T * 4 + 12},
           "roofline": {"bound": "fp64", "achieved": ach, "peak": tf_fma, "unit": "TFLOP/s", "frac": ach / tf_fma,
                        "flops_per_reach_step": fl,
                        "note": "algorithmic flops of the reference's TMExpr op sequence (bench.ct_flops_per_step); "
                                "the kernel is instruction-fetch/latency-bound and its replays skip most of that work "
                                "(profiles/r02_c2_summary.md)"}}
    if rank == 0 and world == 1:
        try:
            from oracle_bind import oracle_cl_split_hull, ref_available, ref_cl_split_hull, ref_lib
            g = cl_split_hull(spec, (w.x0_lo, w.x0_hi), plan, 2040, 2056, ctx=_host_ctx(ctx))
            e = oracle_cl_split_hull(spec, w.x0_lo, w.x0_hi, plan, 2040, 2056)
            scale = np.maximum(np.maximum(np.abs(e.lo), np.abs(e.hi - e.lo)), 1e-300)
            rel = float(max(np.max(np.abs(g.lo - e.lo) / scale), np.max(np.abs(g.hi - e.hi) / scale)))
            out["parity"] = {"parts": 16, "max_rel_diff_vs_oracle": rel, "tolerance": 1e-9,
                             "ok": bool(rel <= 1e-9 and g.n_boxes == e.n_boxes)}
            if ref_available() and not args.no_cpu_baseline:
                lib = ref_lib()
                lib.ref_hardware_threads.restype = C.c_int
                cores = int(lib.ref_hardware_threads())
                parts = int(min(per_rank, max(64, cores * 24)))
                t0 = time.perf_counter()
                ref_cl_split_hull(spec, w.x0_lo, w.x0_hi, plan, 0, parts, threads=0)
                dt = time.perf_counter() - t0
                out["cpu_baseline"] = {"value": parts * (T - 1) / dt, "unit": UNIT, "cores": cores,
                                       "kind": "reference",
                                       "sample": f"{parts} of {per_rank} sub-boxes x {T - 1} steps through the "
                                                 f"reference cl_reach / reach_with_splitting pieces (oracle/_ref), "
                                                 f"{dt:.2f} s"}
        except Exception as ex:  # noqa: BLE001
            out["check_error"] = str(ex)
    ctx.set_stream(stream.cuda_stream)
    return out


TC_INT8_PEAK_TOPS = 4500.0  # B200 dense int8 tensor-core peak (nominal; tools/mma_rate.py measures 8185 MAC/clk/SM)


def tc_int8_macs_per_step(nets):
    """int8 MACs the tensor-core mode (dt_tcw_kernel) issues per reach-step: for each certified net (dims,
    output rows) ceil(n_o / 24) passes, each with ceil(dims[l] / 128) M tiles x ceil(dims[l+1] / 32) K
    steps x 39 Ozaki slice pairs per contraction l = L-2 .. 0, every MMA 128 x 24 x 32."""
    total = 0
    for dims in nets:
        L = len(dims) - 1
        thirds = -(-dims[-1] // 24)
        per = sum(-(-dims[l] // 128) * -(-dims[l + 1] // 32) for l in range(L - 1))
        total += thirds * per * 39 * 128 * 24 * 32
    return total


def c5_flops_per_step():
    """SURVEY §8d formula for C5 (72-D, 3x256 ReLU dynamics + controller): controller
    certification over nz = 5n + 2l = 396 generators, dynamics certification over the stacked
    486, fold solve 6 n^3."""
    def cert(n_i, n_o, hidden, nz):
        w = [hidden[0] * n_i] + [hidden[i] * hidden[i - 1] for i in range(1, len(hidden))]
        return 2 * n_o * sum(w) + 2 * n_o * n_i * nz + 4 * (n_i * (nz + n_i) + sum(w)) + 6 * n_o * sum(hidden)
    return cert(72, 18, [256] * 3, 396) + cert(90, 72, [256] * 3, 486) + 6 * 72 ** 3


def closed_loop_legs(args, ctx, world, rank, dev, barrier, stream):
    """C5 (BASELINE configs[4]): 72-D DT closed loop, 1024 initial boxes x 20 steps per GPU (weak
    scaling, no collective: independent samples).  C1 (configs[0]): the 4-D DT closed loop at
    batch 1 -- a latency figure, timed on rank 0 only."""
    import torch
    import torch.distributed as dist
    from paper_2605_25346_b200.api import dt_closed_loop_batch
    from paper_2605_25346_b200.workloads import c1_closed_loop, c5_closed_loop
    ctx.set_stream(None)
    out = {}
    w = c5_closed_loop()
    B = w.x0_lo.shape[0]
    for _ in range(2):
        r = dt_closed_loop_batch(w.dyn, w.ctl, w.n, w.x0_lo, w.x0_hi, w.horizon, ctx=ctx)
    barrier()
    ctx.enable_kernel_timing(True)
    ctx.kernel_time()
    reps = 2
    for _ in range(reps):
        r = dt_closed_loop_batch(w.dyn, w.ctl, w.n, w.x0_lo, w.x0_hi, w.horizon, ctx=ctx)
    kern_ms, kern_n = ctx.kernel_time()
    ctx.enable_kernel_timing(False)
    t = kern_ms / reps
    if world > 1:
        tt = torch.tensor([t], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = float(tt[0])
    tf_fma, tf_ma = ctx.fp64_peak()
    fl = c5_flops_per_step()
    ach = fl * B * w.horizon / (t / 1e3) / 1e12
    c5 = {"workload": "c5_closed_loop (BASELINE configs[4]): 72-D DT closed loop, 90->256x3->72 ReLU dynamics + "
                      "72->256x3->18 ReLU controller, 1024 boxes x H=20 per GPU, window 4",
          "ms_per_batch": t, "reach_steps_per_s": B * world * w.horizon / (t / 1e3),
          "ok": int((r.status == 0).sum()), "kernel": "rb::dt_wide_kernel<9,3>",
          "roofline": {"bound": "fp64", "achieved": ach, "peak": tf_fma, "unit": "TFLOP/s", "frac": ach / tf_fma,
                       "flops_per_reach_step": fl, "exact_mode_ceiling_tflops": tf_ma},
          "parity": "bit-identical to the oracle / reference composition (tests/test_gpu_wide.py)"}
    # the tolerance modes of the same batch (kernel time) and an in-bench parity spot check: 8 strided
    # samples against the oracle -- exact bit for bit, fused / tc within rtol = 1e-5
    modes = {}
    outs = {"exact": r}
    for prec in ("fused", "tc"):
        if prec == "tc" and args.no_tc:
            continue
        try:
            dt_closed_loop_batch(w.dyn, w.ctl, w.n, w.x0_lo, w.x0_hi, w.horizon, ctx=ctx, precision=prec)
            barrier()
            ctx.enable_kernel_timing(True)
            ctx.kernel_time()
            rp = dt_closed_loop_batch(w.dyn, w.ctl, w.n, w.x0_lo, w.x0_hi, w.horizon, ctx=ctx, precision=prec)
            ms, nl = ctx.kernel_time()
            ctx.enable_kernel_timing(False)
            outs[prec] = rp
            modes[prec] = {"ms_per_batch": ms, "reach_steps_per_s": B * w.horizon / (ms / 1e3),
                           "ok": int((rp.status == 0).sum()),
                           "kernel": "rbf::dt_wide_kernel<9,3>" if prec == "fused" else "rb::dt_tcw_kernel"}
            if prec == "fused":
                a = fl * B * w.horizon / (ms / 1e3) / 1e12
                modes[prec]["tflops"] = a
                modes[prec]["frac_dfma_peak"] = a / tf_fma
            else:
                tops = 2.0 * tc_int8_macs_per_step([[int(x) for x in w.dyn.dims()], [int(x) for x in w.ctl.dims()]]) \
                    * B * w.horizon / (ms / 1e3) / 1e12
                modes[prec]["int8_tops"] = tops
                modes[prec]["frac_int8_dense_peak"] = tops / TC_INT8_PEAK_TOPS
                modes[prec]["peak_source"] = "B200 dense int8 nominal 4.5 POPS; ncu tensor pipe 3.2 % (profiles)"
        except Exception as ex:  # noqa: BLE001
            modes[prec] = {"error": str(ex)}
    c5["modes"] = modes
    if rank == 0:
        try:
            from oracle_bind import oracle_dtcl_batch, same_bits
            idx = np.arange(0, B, max(B // 8, 1))[:8]
            e = oracle_dtcl_batch(w.dyn, w.ctl, w.n, w.x0_lo[idx], w.x0_hi[idx], w.horizon)
            chk = {"samples": int(len(idx)), "rtol": 1e-5}
            for prec, rr in outs.items():
                k = e.n_boxes
                glo, ghi = rr.lo[idx], rr.hi[idx]
                if prec == "exact":
                    chk["exact_bit_exact"] = bool(np.array_equal(rr.n_boxes[idx], k) and
                                                  all(same_bits(glo[i, :k[i]], e.lo[i, :k[i]]) and
                                                      same_bits(ghi[i, :k[i]], e.hi[i, :k[i]]) for i in range(len(idx))))
                else:
                    dev_ = 0.0
                    for i in range(len(idx)):
                        el, eh = e.lo[i, :k[i]], e.hi[i, :k[i]]
                        sc = np.maximum(np.maximum(np.abs(el), np.abs(eh)), eh - el)
                        dev_ = max(dev_, float(np.max(np.abs(glo[i, :k[i]] - el) / sc)),
                                   float(np.max(np.abs(ghi[i, :k[i]] - eh) / sc)))
                    chk[f"{prec}_max_rel_dev"] = dev_
            c5["parity_check"] = chk
        except Exception as ex:  # noqa: BLE001
            c5["parity_check"] = {"error": str(ex)}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            from oracle_bind import ref_available, ref_dtcl_batch, ref_lib
            if ref_available():
                lib = ref_lib()
                lib.ref_hardware_threads.restype = C.c_int
                cores = int(lib.ref_hardware_threads())
                k = int(min(B, max(16, cores * 2)))
                t0 = time.perf_counter()
                ref_dtcl_batch(w.dyn, w.ctl, w.n, w.x0_lo[:k], w.x0_hi[:k], w.horizon, threads=0)
                dt = time.perf_counter() - t0
                c5["cpu_baseline"] = {"value": k * w.horizon / dt, "unit": UNIT, "cores": cores, "kind": "reference",
                                      "sample": f"{k} of {B} boxes x {w.horizon} steps through the reference "
                                                f"composition (oracle/_ref), {dt:.2f} s"}
        except Exception as ex:  # noqa: BLE001
            c5["check_error"] = str(ex)
    out["c5_closed_loop"] = c5
    if rank == 0:
        w1 = c1_closed_loop(batch=1)
        lat_by = {}
        for prec in ("fused", "exact"):
            for _ in range(3):
                dt_closed_loop_batch(w1.dyn, w1.ctl, w1.n, w1.x0_lo, w1.x0_hi, w1.horizon, ctx=ctx, precision=prec)
            lat = []
            for _ in range(10):
                t0 = time.perf_counter()
                dt_closed_loop_batch(w1.dyn, w1.ctl, w1.n, w1.x0_lo, w1.x0_hi, w1.horizon, ctx=ctx, precision=prec)
                lat.append(time.perf_counter() - t0)
            lat_by[prec] = 1e3 * float(np.median(lat))
        c1 = {"workload": "c1_closed_loop (BASELINE configs[0]): 4-D DT closed loop, 6->64x2->4 ReLU dynamics + "
                          "4->64x2->2 ReLU controller, one box, H=20",
              "latency_ms_end_to_end": lat_by["fused"], "precision": "fused",
              "latency_ms_end_to_end_exact": lat_by["exact"],
              "note": "batch 1 is latency-bound (SURVEY §8d): host call incl. copies, median of 10"}
        if not args.no_cpu_baseline:
            try:
                from oracle_bind import ref_available, ref_dtcl_batch
                if ref_available():
                    ts = []
                    for _ in range(5):
                        t0 = time.perf_counter()
                        ref_dtcl_batch(w1.dyn, w1.ctl, w1.n, w1.x0_lo, w1.x0_hi, w1.horizon, threads=1)
                        ts.append(time.perf_counter() - t0)
                    c1["cpu_reference_latency_ms"] = 1e3 * float(np.median(ts))
            except Exception as ex:  # noqa: BLE001
                c1["check_error"] = str(ex)
        out["c1_closed_loop"] = c1
    ctx.set_stream(stream.cuda_stream)
    return out


def _host_ctx(ctx):
    ctx.set_stream(None)
    return ctx


def run_reference(args):
    from paper_2605_25346_b200.workloads import c4_partition_sweep
    rank, world, _ = dist_env()
    if rank != 0:
        return
    w = c4_partition_sweep()
    parts = args.cpu_sample_parts or max(128, auto_cpu_parts() // 8)
    times = []
    cb = None
    for i in range(args.warmup + args.steps):
        r = cpu_baseline(w, parts)
        if r is None:
            print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libreach_ref.so not built"}))
            return
        if i >= args.warmup:
            times.append(parts * w.horizon / r["value"])
            cb = r
    ms = 1e3 * float(np.mean(times))
    value = parts * w.horizon / (ms / 1e3)
    cb["value"] = value
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "c4_partition_sweep (BASELINE configs[3]) bounded CPU sample",
                       "sub_boxes_per_step": parts, "horizon": w.horizon, "state_dim": 6,
                       "net": "6->128x3->6 ReLU", "plan": "8x8x8x8x4x4"},
            "impl": "reference", "cpu_baseline": cb,
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def main():
    args = parse()
    if args.impl == "reference" and os.environ.get("WORLD_SIZE") is None:
        return run_reference(args)  # rank 0's work only: no ranks to launch
    rc = ensure_world(args)
    if rc is not None:
        sys.exit(rc)
    if args.dist_dry_run:
        return dist_dry_run(args)
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist
    from paper_2605_25346_b200 import _abi as A
    from paper_2605_25346_b200._native import Context
    from paper_2605_25346_b200.api import SplitPlan, reach_split_hull
    from paper_2605_25346_b200.workloads import c4_partition_sweep

    rank, world, local = dist_env()
    # RB_BENCH_SHARE_GPU=1 (logic check of the N > 1 path on a 1-GPU box, never a measurement):
    # ranks share the visible GPUs and reduce over gloo
    share = os.environ.get("RB_BENCH_SHARE_GPU") == "1"
    if world > torch.cuda.device_count() and not share:
        raise SystemExit(f"bench.py: {world} ranks but {torch.cuda.device_count()} visible GPU(s); "
                         "set RB_BENCH_SHARE_GPU=1 for a shared-GPU logic check (gloo)")
    if share:
        local = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    w = c4_partition_sweep()
    per_rank = w.plan.total_parts()
    counts = list(w.plan.counts)
    counts[0] *= world
    plan = SplitPlan(counts)
    begin, end = rank * per_rank, (rank + 1) * per_rank
    H, n, m = w.horizon, w.sys.n, w.sys.m

    ctx = Context(local)
    if world > 1:
        # the library shards every batch call over the ranks and combines on its stream (NCCL over
        # NVLink; gloo staging only for the shared-GPU logic check)
        from paper_2605_25346_b200.distributed import nccl_collectives, torch_collectives
        (torch_collectives if share else nccl_collectives)(ctx)
    stream = torch.cuda.Stream(dev)  # the library launches here; torch work joins it below
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    netdims = [int(x) for x in w.sys.step.dims()]
    flops_part = algorithmic_flops_per_part(netdims, n, m, H, 4)

    # device-resident outputs; the X0 box / plan are kernel parameters
    cnt = (H + 1) * n
    d_lo = torch.empty(cnt, dtype=torch.float64, device=dev)
    d_hi = torch.empty(cnt, dtype=torch.float64, device=dev)
    d_div = torch.empty(H + 1, dtype=torch.int32, device=dev)
    d_nb = torch.empty(1, dtype=torch.int32, device=dev)
    d_key = torch.empty(1, dtype=torch.int64, device=dev)
    d_act = torch.zeros(max(H * m, 1), dtype=torch.float64, device=dev)
    x0lo = np.ascontiguousarray(w.x0_lo)
    x0hi = np.ascontiguousarray(w.x0_hi)
    cts = np.array(counts, dtype=np.int32)
    # the full global plan on every rank: the library takes this rank's contiguous slice of the parts
    args_c = A.SplitArgs(n, m, H, 4, 0, A.dptr(x0lo), A.dptr(x0hi), A.iptr(cts), A.dptr(d_act.data_ptr()), 0, 0)
    out_c = A.HullOut(A.dptr(d_lo.data_ptr()), A.dptr(d_hi.data_ptr()), A.iptr(d_div.data_ptr()),
                      A.iptr(d_nb.data_ptr()), A.lptr(d_key.data_ptr()))
    net = ctx.upload(w.sys.step)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2

    # headline precision: REACH_PREC_FUSED (fp64, DFMA contractions; parity within the north_star's fp64
    # tolerance, checked below); the bit-exact and tensor-core modes are timed beside it
    def device_step(prec=A.REACH_PREC_FUSED):
        ctx.check(ctx._lib.reach_split_hull(ctx.handle, net, C.byref(args_c), C.byref(out_c),
                                            A.REACH_FLAG_DEVICE_PTRS | prec), "reach_split_hull")

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    for _ in range(args.warmup):
        device_step()
    barrier()

    # ---- timed region (device events per step, L2 flushed between steps)
    ctx.enable_kernel_timing(True)
    ctx.kernel_time()
    launches0 = ctx.launch_count
    clocks = ClockSampler(local)
    clocks.start()
    clocks.wait_first()
    step_ms = []
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    barrier()
    for _ in range(args.steps):
        flush.zero_()
        ev0.record(stream)
        device_step()
        ev1.record(stream)
        ev1.synchronize()
        step_ms.append(ev0.elapsed_time(ev1))
    barrier()
    clk = clocks.stop()
    kern_ms, kern_n = ctx.kernel_time()
    launches = ctx.launch_count - launches0
    ctx.enable_kernel_timing(False)
    t_local = float(np.sum(step_ms))
    if world > 1:
        t = torch.tensor([t_local, kern_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_max, kern_max = float(t[0]), float(t[1])
    else:
        t_max, kern_max = t_local, kern_ms
    reach_steps = per_rank * world * H
    value = reach_steps * args.steps / (t_max / 1e3)

    # ---- end to end through the public API (host X0/plan/actions in, host hull out)
    from paper_2605_25346_b200.api import DTReachParams
    ctx.set_stream(None)
    e2e_t = []
    for i in range(args.warmup + args.steps):
        barrier()
        t0 = time.perf_counter()
        res = reach_split_hull(w.sys, (w.x0_lo, w.x0_hi), plan, w.actions, DTReachParams(), ctx=ctx,
                               precision="fused")
        dt_ = time.perf_counter() - t0
        if i >= args.warmup:
            e2e_t.append(dt_)
    e2e_local = float(np.sum(e2e_t))
    if world > 1:
        t = torch.tensor([e2e_local], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_local = float(t[0])
    e2e_value = reach_steps * args.steps / e2e_local
    h2d = 2 * n * 8 + n * 4 + H * m * 8
    d2h = 2 * (H + 1) * n * 8 + (H + 1) * 4 + 4 + 8

    # ---- roofline of the dominant kernel (dt_horizon_kernel), FP64 pipe
    tf_fma, tf_ma = ctx.fp64_peak()
    ach = flops_part * per_rank / (kern_max / max(kern_n, 1) / 1e3) / 1e12
    roof = {"bound": "fp64", "achieved": ach, "peak": tf_fma, "unit": "TFLOP/s", "frac": ach / tf_fma,
            "traffic": None, "kernel": "rbf::dt_horizon_kernel<6,4> (REACH_PREC_FUSED build)",
            "flops_per_launch": flops_part * per_rank,
            "flops_note": "dense-equivalent algorithmic flops (SURVEY §8d); ReLU-sparsity skipping executes fewer "
                          "(executed_tflops: ncu's executed DFMA/DMUL/DADD thread-op count of this kernel per "
                          "launch, profiles/c4_dram_traffic.json, over the live kernel time)",
            "peak_source": "measured on this box by reach_measure_fp64_peak (DFMA chains, 2 flops/instr)",
            "kernel_ms_per_launch": kern_max / max(kern_n, 1)}
    prof = os.path.join(ROOT, "profiles", "c4_dram_traffic.json")
    if os.path.exists(prof):
        try:
            tr = json.load(open(prof))
            roof["traffic"] = tr.get("fused", {}).get("dram_bytes_per_launch")
            roof["traffic_source"] = tr.get("fused", {}).get("source")
            xf = tr.get("fused", {}).get("executed_fp64_flops_per_launch")
            if xf:
                roof["executed_tflops"] = xf / (roof["kernel_ms_per_launch"] / 1e3) / 1e12
        except Exception:
            pass

    # ---- the other precision modes of the same sweep (kernel time, L2 flushed; N = 1 rank's share)
    def mode_time(prec, reps):
        device_step(prec)
        barrier()
        ctx.enable_kernel_timing(True)
        ctx.kernel_time()
        for _ in range(reps):
            flush.zero_()
            device_step(prec)
        barrier()
        ms, nl = ctx.kernel_time()
        ctx.enable_kernel_timing(False)
        if world > 1:
            t = torch.tensor([ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t[0])
        per = ms / max(nl, 1)
        return per, flops_part * per_rank / (per / 1e3) / 1e12

    ex_ms, ex_tf = mode_time(A.REACH_PREC_EXACT, args.steps)
    modes = {"fused": {"kernel_ms": kern_max / max(kern_n, 1), "reach_steps_per_s": reach_steps / (kern_max / max(kern_n, 1) / 1e3),
                       "tflops": ach, "frac_dfma_peak": ach / tf_fma},
             "exact": {"kernel_ms": ex_ms, "reach_steps_per_s": reach_steps / (ex_ms / 1e3), "tflops": ex_tf,
                       "frac_dfma_peak": ex_tf / tf_fma, "exact_mode_ceiling_tflops": tf_ma,
                       "frac_of_exact_mode_ceiling": ex_tf / tf_ma if tf_ma else None,
                       "kernel": "rb::dt_horizon_kernel<6,4>", "parity": "bit-identical to the oracle / reference"}}
    if not args.no_tc:
        try:
            tc_ms, tc_tf = mode_time(A.REACH_PREC_TC, 1)
            tops = 2.0 * tc_int8_macs_per_step([netdims]) * per_rank * H / (tc_ms / 1e3) / 1e12
            modes["tc"] = {"kernel_ms": tc_ms, "reach_steps_per_s": reach_steps / (tc_ms / 1e3), "tflops_fp64_equiv": tc_tf,
                           "int8_tops": tops, "frac_int8_dense_peak": tops / TC_INT8_PEAK_TOPS,
                           "peak_source": "B200 dense int8 nominal 4.5 POPS",
                           "kernel": "rb::dt_tcw_kernel (CTA per sub-box, tcgen05.mma kind::i8 Ozaki contractions)"}
        except Exception as ex:  # noqa: BLE001
            modes["tc"] = {"error": str(ex)}

    # ---- parity spot checks vs the oracle (first 64 parts of this rank): the headline (fused) mode within
    # rtol = 1e-5 (north_star, fp64), the exact mode bit for bit; the full-size fused hull against the
    # exact mode's hull (itself bit-identical to the oracle) within the same rtol
    parity = None
    if rank == 0:
        try:
            from oracle_bind import oracle_split_hull, same_bits
            solo = ctx if world == 1 else Context(local)  # rank-0-only call: a context without collectives

            def hull_dev(g, e):
                k = e.n_boxes
                sc = np.maximum(np.maximum(np.abs(e.lo[:k]), np.abs(e.hi[:k])), e.hi[:k] - e.lo[:k])
                sc = np.maximum(sc, 1e-300)
                return float(max(np.max(np.abs(g.lo[:k] - e.lo[:k]) / sc), np.max(np.abs(g.hi[:k] - e.hi[:k]) / sc)))

            e = oracle_split_hull(w.sys, w.x0_lo, w.x0_hi, plan, w.actions, begin=0, end=64)
            gf = reach_split_hull(w.sys, (w.x0_lo, w.x0_hi), plan, w.actions, part_begin=0, part_end=64, ctx=solo,
                                  precision="fused")
            ge = reach_split_hull(w.sys, (w.x0_lo, w.x0_hi), plan, w.actions, part_begin=0, part_end=64, ctx=solo)
            full_f = reach_split_hull(w.sys, (w.x0_lo, w.x0_hi), plan, w.actions, part_begin=begin, part_end=end,
                                      ctx=solo, precision="fused")
            full_e = reach_split_hull(w.sys, (w.x0_lo, w.x0_hi), plan, w.actions, part_begin=begin, part_end=end,
                                      ctx=solo)
            dev64, devfull = hull_dev(gf, e), hull_dev(full_f, full_e)
            parity = {"parts": 64, "rtol": 1e-5, "fused_max_rel_dev_vs_oracle": dev64,
                      "fused_full_hull_max_rel_dev_vs_exact": devfull,
                      "ok": bool(dev64 <= 1e-5 and devfull <= 1e-5 and gf.n_boxes == e.n_boxes
                                 and full_f.fail_key == full_e.fail_key),
                      "exact_bit_exact": bool(same_bits(ge.lo, e.lo) and same_bits(ge.hi, e.hi)
                                              and ge.n_boxes == e.n_boxes)}
            if "tc" in modes and "error" not in modes["tc"]:
                gt = reach_split_hull(w.sys, (w.x0_lo, w.x0_hi), plan, w.actions, part_begin=0, part_end=64,
                                      ctx=solo, precision="tc")
                modes["tc"]["max_rel_dev_vs_oracle"] = hull_dev(gt, e)
        except Exception as ex:  # the checker is optional at bench time
            parity = {"error": str(ex)}

    cb = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cb = cpu_baseline(w, args.cpu_sample_parts or auto_cpu_parts())

    # ---- C2: the continuous-time quadrotor closed loop (BASELINE configs[1])
    ct = None if args.no_ct else ct_sweep(args, ctx, world, rank, dev, barrier, stream)
    # ---- C5 / C1: the DT closed loop at 72-D (throughput) and 4-D batch 1 (latency)
    cl = {} if args.no_cl else closed_loop_legs(args, ctx, world, rank, dev, barrier, stream)

    # ---- the metric's second half: ms per reachability-aware MPC replan (BASELINE configs[2])
    mpc = None if args.no_mpc else mpc_replan(args, ctx, world, rank, dev, barrier)
    # ---- section 8(f) rank 1: forward-dual gradients through the DT engine (N = 1 only)
    grad = None if (args.no_grad or world > 1) else gradient_leg(args, ctx)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": t_max / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": "c4_partition_sweep (BASELINE configs[3])", "sub_boxes_per_gpu": per_rank,
                           "sub_boxes_total": per_rank * world, "plan": "x".join(map(str, counts)),
                           "horizon": H, "state_dim": n, "net": "6->128x3->6 ReLU (residual synthetic)",
                           "window": 4, "l2": "flushed between timed steps (256 MB write)",
                           "parallelism": f"dp{world}"},
                "precision": "fused (REACH_PREC_FUSED: fp64, DFMA contractions; exact and tc modes in 'modes')",
                "modes": modes, "roofline": roof, "cpu_baseline": cb,
                "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
                "gpu_launches": launches, "clocks": clk, "parity": parity, "ct_quadrotor": ct, **cl, "mpc_replan": mpc,
                "gradients": grad,
                "bit_exact_vs_reference": "exact mode: identical operation order and roundings (tests/test_gpu_dt.py); "
                                          "fused mode within rtol 1e-5 (tests/test_gpu_fused.py)"}
        print(json.dumps(line))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
