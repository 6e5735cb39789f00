"""Kernel time of the C4 sweep and the C5 closed loop in each precision mode (ctx kernel timing)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_25346_b200.api import default_context, dt_closed_loop_batch, reach_split_hull  # noqa: E402
from paper_2605_25346_b200.workloads import c4_partition_sweep, c5_closed_loop  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "c4"
modes = sys.argv[2].split(",") if len(sys.argv) > 2 else ["exact", "fused"]
ctx = default_context()
if which == "c4":
    w = c4_partition_sweep()
    run = lambda p: reach_split_hull(w.sys, (w.x0_lo, w.x0_hi), w.plan, w.actions, ctx=ctx, precision=p)  # noqa: E731
    steps = 65536 * 30
else:
    w = c5_closed_loop(batch=1024)
    run = lambda p: dt_closed_loop_batch(w.dyn, w.ctl, w.n, w.x0_lo, w.x0_hi, w.horizon, ctx=ctx, precision=p)  # noqa: E731
    steps = 1024 * 20
for p in modes:
    run(p)
    ctx.enable_kernel_timing(True)
    best = 1e30
    for _ in range(3):
        ctx.kernel_time()
        run(p)
        ms, n = ctx.kernel_time()
        best = min(best, ms)
    ctx.enable_kernel_timing(False)
    print(f"{which} {p:6s} kernel {best:8.2f} ms  {steps / (best * 1e-3):.4g} reach-steps/s")
