"""Diagnostics of the tensor-core precision mode vs the oracle: per-step deviation, widening."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from oracle_bind import oracle_dtcl_batch  # noqa: E402
from paper_2605_25346_b200.api import dt_closed_loop_batch  # noqa: E402
from paper_2605_25346_b200.workloads import c5_closed_loop  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
H = int(sys.argv[2]) if len(sys.argv) > 2 else 20
w = c5_closed_loop(batch=B)
got = dt_closed_loop_batch(w.dyn, w.ctl, w.n, w.x0_lo, w.x0_hi, H, precision="tc")
ex = dt_closed_loop_batch(w.dyn, w.ctl, w.n, w.x0_lo, w.x0_hi, H)
for k in range(H + 1):
    e_lo, e_hi, g_lo, g_hi = ex.lo[0, k], ex.hi[0, k], got.lo[0, k], got.hi[0, k]
    wid = e_hi - e_lo
    dlo, dhi = g_lo - e_lo, g_hi - e_hi
    widen = (g_hi - g_lo) - wid
    scale = np.maximum(np.maximum(np.abs(e_lo), np.abs(e_hi)), wid)
    rel = max(np.max(np.abs(dlo) / scale), np.max(np.abs(dhi) / scale))
    print(f"k={k:2d} width {np.mean(wid):.3e}  max|dlo| {np.max(np.abs(dlo)):.3e} max|dhi| {np.max(np.abs(dhi)):.3e} "
          f"mean widen {np.mean(widen):.3e} min widen {np.min(widen):.3e} center shift {np.max(np.abs((dlo+dhi)/2)):.3e} rel {rel:.2e}")
