"""Times the C2 quadrotor closed-loop sweep (rpy:4096 sub-boxes x 50 flowpipe steps) on the device."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_25346_b200.api import cl_split_hull, default_context  # noqa: E402
from paper_2605_25346_b200.workloads import c2_quadrotor  # noqa: E402

parts = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
w = c2_quadrotor(parts=parts)
ctx = default_context()
x0 = (w.x0_lo, w.x0_hi)
h = cl_split_hull(w.spec, x0, w.plan, ctx=ctx)
ctx.enable_kernel_timing(True)
steps = parts * w.spec.ctl_steps * w.spec.k_atomic
for _ in range(reps):
    ctx.kernel_time()
    t0 = time.perf_counter()
    h = cl_split_hull(w.spec, x0, w.plan, ctx=ctx)
    wall = time.perf_counter() - t0
    ms, n = ctx.kernel_time()
    print(f"parts={parts} kernels {ms:.2f} ms ({n} timed regions) wall {wall*1e3:.1f} ms  "
          f"reach-steps/s {steps / (ms * 1e-3):.4g}  n_boxes {h.n_boxes} fail_key {h.fail_key}")
print("final hull width sum", float((h.hi[-1] - h.lo[-1]).sum()))
