"""grad_tube_volume timings on the device vs the reference (oracle/_ref, one host thread per call)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

from grad_cases import _box  # noqa: E402
from oracle_bind import ref_available, ref_grad_tube_volume  # noqa: E402
from paper_2605_25346_b200.api import Act, DTReachParams, DTSystem, GradMethod, GradTarget, grad_tube_volume  # noqa: E402
from paper_2605_25346_b200._native import default_context  # noqa: E402
from paper_2605_25346_b200.workloads import random_mlp  # noqa: E402

rng = np.random.default_rng(1)
net = random_mlp(rng, 6, [128, 128, 128], 6, Act.Relu, 0.9)
net.layers[-1].w *= 0.5
sysm = DTSystem(net, 6, 0)
H = int(os.environ.get("H", "30"))
x0 = _box(np.zeros(6), 0.05)
acts = [[]] * H
ctx = default_context()
ctx.enable_kernel_timing(True)
for target in (GradTarget.x0_center, GradTarget.weights):
    grad_tube_volume(sysm, x0, acts, target)
    ctx.kernel_time()
    t0 = time.perf_counter()
    g = grad_tube_volume(sysm, x0, acts, target)
    wall = time.perf_counter() - t0
    km, kn = ctx.kernel_time()
    line = f"{target.name}: {g.g.size} passes, H={H}: kernel {km:.2f} ms, call {1e3 * wall:.2f} ms"
    if ref_available() and target == GradTarget.x0_center:
        t0 = time.perf_counter()
        ref_grad_tube_volume(sysm, x0, acts, int(target), 0)
        line += f"; reference {1e3 * (time.perf_counter() - t0):.1f} ms (1 thread)"
    print(line, flush=True)
