"""Times the C5 72-D closed loop (batch 1024 by default) through the C ABI with kernel timing."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_25346_b200.api import dt_closed_loop_batch, default_context  # noqa: E402
from paper_2605_25346_b200.workloads import c5_closed_loop  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
prec = sys.argv[3] if len(sys.argv) > 3 else "exact"
w = c5_closed_loop(batch=B)
ctx = default_context()
dt_closed_loop_batch(w.dyn, w.ctl, w.n, w.x0_lo, w.x0_hi, w.horizon, ctx=ctx, precision=prec)
ctx.enable_kernel_timing(True)
for _ in range(reps):
    ctx.kernel_time()
    t0 = time.perf_counter()
    r = dt_closed_loop_batch(w.dyn, w.ctl, w.n, w.x0_lo, w.x0_hi, w.horizon, ctx=ctx, precision=prec)
    wall = time.perf_counter() - t0
    ms, n = ctx.kernel_time()
    print(f"{prec} B={B} kernel {ms:.2f} ms ({n} launches) wall {wall*1e3:.1f} ms  "
          f"reach-steps/s {B * w.horizon / (ms * 1e-3):.4g}  status_ok {(r.status == 0).sum()}/{B}")

if os.environ.get("RB_WIDE_PHASE") == "1":
    names = ["setup", "ctl pre-IBP", "ctl hid-IBP", "ctl chains", "ctl GEMM", "ctl pre-GEMM",
             "dyn pre-IBP", "dyn hid-IBP", "dyn chains", "dyn GEMM", "dyn pre-GEMM", "reseed", "fold other", "box",
             "fold elim", "fold backsub"]
    ctx.phase_cycles()
    dt_closed_loop_batch(w.dyn, w.ctl, w.n, w.x0_lo, w.x0_hi, w.horizon, ctx=ctx, precision=prec)
    cyc = ctx.phase_cycles()
    tot = sum(cyc[:16])
    for nm, c in zip(names, cyc):
        print(f"{nm:14s} {c / tot * 100:6.2f}%  {c / (B * w.horizon):10.0f} cycles/reach-step")
