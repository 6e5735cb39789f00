"""Dumps the C2 sweep's hull (and a small cl_batch tube) to an .npz, for bit-identity checks between library builds
(REACH_B200_LIB selects the build)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_25346_b200.api import cl_split_hull, default_context  # noqa: E402
from paper_2605_25346_b200.workloads import c2_quadrotor  # noqa: E402

out = sys.argv[1]
parts = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
w = c2_quadrotor(parts=parts)
h = cl_split_hull(w.spec, (w.x0_lo, w.x0_hi), w.plan, ctx=default_context())
np.savez(out, lo=h.lo, hi=h.hi, n_boxes=h.n_boxes, fail_key=h.fail_key)
print("saved", out, float((h.hi[-1] - h.lo[-1]).sum()))
