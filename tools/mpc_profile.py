"""Breakdown of one C3 replan: host sampling / update vs device plan_eval."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_2605_25346_b200._native import default_context  # noqa: E402
from paper_2605_25346_b200.mpc import CEM, plan_cem, plan_eval_batch  # noqa: E402
from paper_2605_25346_b200.workloads import c3_tpushing  # noqa: E402

prob, cfg, x0 = c3_tpushing()
ctx = default_context()
plan_cem(prob, cfg, x0)
t0 = time.perf_counter()
plan_cem(prob, cfg, x0)
print(f"plan_cem total {1e3*(time.perf_counter()-t0):.1f} ms")
cem = CEM(prob, cfg)
ts = te = tu = 0.0
ctx.enable_kernel_timing(True)
ctx.kernel_time()
for it in range(cfg.iterations):
    a = time.perf_counter()
    c = cem.sample()
    b = time.perf_counter()
    r = plan_eval_batch(prob, x0, c)
    d = time.perf_counter()
    cem.update(r.objective, ~r.diverged)
    e = time.perf_counter()
    ts += b - a
    te += d - b
    tu += e - d
km, kn = ctx.kernel_time()
print(f"sample {1e3*ts:.1f} ms  plan_eval {1e3*te:.1f} ms (dt kernel {km:.1f} ms over {kn})  update {1e3*tu:.1f} ms")

# plan_cem with the reference-default gradient refinement of the top candidate (refine_iters = 5)
import dataclasses  # noqa: E402

from paper_2605_25346_b200.mpc import plan_objective_grad  # noqa: E402

cfg5 = dataclasses.replace(cfg, refine_iters=5)
r0 = plan_cem(prob, cfg, x0)
plan_cem(prob, cfg5, x0)
t0 = time.perf_counter()
r5 = plan_cem(prob, cfg5, x0)
print(f"plan_cem refine_iters=5 total {1e3*(time.perf_counter()-t0):.1f} ms  objective {r0.objective:.6g} -> "
      f"{r5.objective:.6g} refined={r5.refined}")
g, f = plan_objective_grad(prob, x0, r0.actions)
t0 = time.perf_counter()
for _ in range(10):
    plan_objective_grad(prob, x0, r0.actions)
print(f"plan_objective_grad (40 directions) {1e2*(time.perf_counter()-t0):.2f} ms per call, |g| {np.linalg.norm(g):.4g}")
