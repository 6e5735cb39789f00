"""C1 (4-D DT closed loop, batch 1, H = 20) latency through the public API: end to end (host call incl.
copies) and the one kernel launch, per precision mode.  usage: python tools/c1_latency.py [exact,fused]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2605_25346_b200.api import default_context, dt_closed_loop_batch  # noqa: E402
from paper_2605_25346_b200.workloads import c1_closed_loop  # noqa: E402

modes = sys.argv[1].split(",") if len(sys.argv) > 1 else ["exact"]
w = c1_closed_loop(batch=1)
ctx = default_context()
for prec in modes:
    for _ in range(3):
        dt_closed_loop_batch(w.dyn, w.ctl, w.n, w.x0_lo, w.x0_hi, w.horizon, ctx=ctx, precision=prec)
    ctx.enable_kernel_timing(True)
    ctx.kernel_time()
    lat = []
    for _ in range(10):
        t0 = time.perf_counter()
        dt_closed_loop_batch(w.dyn, w.ctl, w.n, w.x0_lo, w.x0_hi, w.horizon, ctx=ctx, precision=prec)
        lat.append(time.perf_counter() - t0)
    ms, n = ctx.kernel_time()
    ctx.enable_kernel_timing(False)
    print(f"{prec} RB_FORCE_WIDE={os.environ.get('RB_FORCE_WIDE', '0')} e2e ms {1e3 * np.median(lat):.3f} "
          f"kernel ms {ms / max(n, 1):.3f}")
