"""Runs C3 replans (plan_cem through the C ABI) -- for ncu launch lists; prints the wall time per replan
and the device kernel time per replan (ctx kernel timing: the launches this library makes)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_25346_b200._native import default_context  # noqa: E402
from paper_2605_25346_b200.mpc import plan_cem  # noqa: E402
from paper_2605_25346_b200.workloads import c3_tpushing  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
prob, cfg, x0 = c3_tpushing()
ctx = default_context()
plan_cem(prob, cfg, x0, ctx=ctx)
ctx.enable_kernel_timing(True)
for _ in range(reps):
    ctx.kernel_time()
    n0 = ctx.launch_count
    t0 = time.perf_counter()
    r = plan_cem(prob, cfg, x0, ctx=ctx)
    wall = time.perf_counter() - t0
    ms, n = ctx.kernel_time()
    print(f"replan wall {wall * 1e3:.2f} ms  device (timed launches) {ms:.2f} ms in {n} timed calls, "
          f"{ctx.launch_count - n0} library launches, objective {r.objective:.6f}")
