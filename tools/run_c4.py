"""Runs the C4 sweep (optionally a part prefix) twice through the C ABI -- for ncu captures."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_25346_b200.api import reach_split_hull  # noqa: E402
from paper_2605_25346_b200.workloads import c4_partition_sweep  # noqa: E402

parts = int(sys.argv[1]) if len(sys.argv) > 1 else 0
prec = sys.argv[2] if len(sys.argv) > 2 else "exact"
w = c4_partition_sweep()
for _ in range(2):
    r = reach_split_hull(w.sys, (w.x0_lo, w.x0_hi), w.plan, w.actions, part_end=parts, precision=prec)
print("n_boxes", r.n_boxes, "hull[-1]", r.lo[-1][:2], r.hi[-1][:2])
