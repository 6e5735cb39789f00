"""One short C5 launch (B samples x H steps) for ncu captures of the closed-loop kernels."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_25346_b200.api import dt_closed_loop_batch  # noqa: E402
from paper_2605_25346_b200.workloads import c5_closed_loop  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 148
H = int(sys.argv[2]) if len(sys.argv) > 2 else 4
prec = sys.argv[3] if len(sys.argv) > 3 else "tc"
w = c5_closed_loop(batch=B)
for _ in range(2):
    dt_closed_loop_batch(w.dyn, w.ctl, w.n, w.x0_lo, w.x0_hi, H, precision=prec)
