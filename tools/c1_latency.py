import sys, time, os
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2605_25346_b200.api import dt_closed_loop_batch, default_context
from paper_2605_25346_b200.workloads import c1_closed_loop
w = c1_closed_loop(batch=1)
ctx = default_context()
for _ in range(3): dt_closed_loop_batch(w.dyn, w.ctl, w.n, w.x0_lo, w.x0_hi, w.horizon, ctx=ctx)
ctx.enable_kernel_timing(True); ctx.kernel_time()
lat = []
for _ in range(10):
    t0 = time.perf_counter(); dt_closed_loop_batch(w.dyn, w.ctl, w.n, w.x0_lo, w.x0_hi, w.horizon, ctx=ctx); lat.append(time.perf_counter() - t0)
ms, n = ctx.kernel_time()
print(os.environ.get("RB_FORCE_WIDE", "0"), "e2e ms", 1e3 * np.median(lat), "kernel ms", ms / n)
