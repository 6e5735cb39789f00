"""Per-phase cycle breakdown of the DT kernel on the C4 sweep (profiling build).

usage: REACH_B200_LIB=paper_2605_25346_b200/libreach_b200_phase.so python tools/phase_profile.py [parts]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("REACH_B200_LIB", os.path.join(ROOT, "paper_2605_25346_b200", "libreach_b200_phase.so"))

from paper_2605_25346_b200._native import Context  # noqa: E402
from paper_2605_25346_b200.api import reach_split_hull  # noqa: E402
from paper_2605_25346_b200.workloads import c4_partition_sweep  # noqa: E402

NAMES = ["prepend", "ibp", "bwd_init", "chains", "gemm", "gemm_l0", "tail", "fold", "box", "drain"]


def main():
    parts = int(sys.argv[1]) if len(sys.argv) > 1 else 0
    w = c4_partition_sweep()
    ctx = Context(0)
    reach_split_hull(w.sys, (w.x0_lo, w.x0_hi), w.plan, w.actions, part_end=parts, ctx=ctx)
    ctx.phase_cycles()
    t0 = time.perf_counter()
    reach_split_hull(w.sys, (w.x0_lo, w.x0_hi), w.plan, w.actions, part_end=parts, ctx=ctx)
    dt = time.perf_counter() - t0
    cyc = ctx.phase_cycles()
    if cyc is None:
        print(f"wall {dt*1e3:.1f} ms (product build, no phase counters)")
        return
    wait = cyc[10]
    cyc = cyc[:10]
    tot = sum(cyc)
    if tot == 0:
        print(f"wall {dt*1e3:.1f} ms; the horizon kernel carries no phase marks in this build (they went away when "
              "certify_tm_input became a device function; use the ncu source view, profiles/r02_c4_summary.md)")
        return
    print(f"wall {dt*1e3:.1f} ms; warp-cycles {tot:.3e}")
    for nm, c in zip(NAMES, cyc):
        print(f"  {nm:9s} {100*c/tot:5.1f}%  {c/ (w.plan.total_parts() if not parts else parts) / w.horizon:9.0f} cyc/sample-step")
    print(f"  (of which waiting for weight chunks: {100*wait/tot:5.1f}%)")


if __name__ == "__main__":
    main()
