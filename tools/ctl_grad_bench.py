"""Times the ctl_reach_loss gradient at the C2 controller size (15 -> 3x64 tanh -> 4, 9,668 parameters):
episodes x (t_h control intervals x k_atomic flowpipe steps), every Dual pass on the device; and the
reference's grad_forward on one host core for a one-episode, t_h = 1 sample (per-pass cost extrapolated)."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_2605_25346_b200.api import Episode, ctl_reach_loss, default_context  # noqa: E402
from paper_2605_25346_b200.workloads import quadrotor_controller  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 4
t_h = int(sys.argv[2]) if len(sys.argv) > 2 else 10
k_atomic, delta, eps, cap = 5, 0.05, 0.01, 40.0
rng = np.random.default_rng(2)
ctl = quadrotor_controller(rng, (64, 64, 64))
batch = []
for _ in range(M):
    x0 = np.zeros(12)
    x0[:6] = rng.uniform(-0.05, 0.05, 6)
    batch.append(Episode([x0] * (t_h + 1), [np.zeros(4)] * t_h, list(np.tile([0.1, 0.0, 0.0], (t_h, 1)))))
ctx = default_context()
ctl_reach_loss(ctl, batch[:1], eps, 1, delta / t_h, k_atomic, cap, with_grad=True, ctx=ctx)
t0 = time.perf_counter()
loss, g, dc = ctl_reach_loss(ctl, batch, eps, t_h, delta * t_h / t_h, k_atomic, cap, with_grad=True, ctx=ctx)
dt = time.perf_counter() - t0
P = g.size
print(f"device: {P} params x {M} episodes x {t_h * k_atomic} steps: {dt:.3f} s ({P * M / dt:.0f} passes/s), "
      f"loss {loss:.6f}, diverged {dc}")
if len(sys.argv) > 3:
    from oracle_bind import ref_ctl_reach_loss
    from paper_2605_25346_b200.api import ClosedLoopSpec, FlowpipeParams
    spec = ClosedLoopSpec(ctl, ctl_steps=1, k_atomic=k_atomic, fp=FlowpipeParams(h=delta / k_atomic),
                          y_ref=np.asarray(batch[0].y_ref[:1]))
    t0 = time.perf_counter()
    ref_ctl_reach_loss(spec, np.array([batch[0].states[0]]), [np.asarray(batch[0].y_ref[:1])], eps, 1, delta, cap,
                       with_grad=True)
    rt = time.perf_counter() - t0
    print(f"reference (1 core): 1 episode x 1 interval ({k_atomic} steps), {P} passes: {rt:.2f} s -> "
          f"{rt / P * t_h:.4f} s per pass of {t_h * k_atomic} steps; extrapolated {rt * t_h * M:.0f} s")
