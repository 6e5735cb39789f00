"""Seeded synthetic workloads of the BASELINE.json configs.

Plain `random_mlp` nets make tubes collapse or explode over the horizon, so the
DT dynamics are near-identity residual ReLU maps: the first n+m hidden units
of every layer carry (x, u) through relu(v + K) with K = 10 (stably active, so
CROWN is exact on them); the remaining units are random features of (x, u);
the output layer is x' = a x + dt Bu u + dt Bf features with the K offset
cancelled in the biases.  Deterministic for a given seed (numpy PCG64).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List

import numpy as np

from .api import Act, DTSystem, Layer, MLPNet, SplitPlan

MASTER_SEED = 20261017
K_OFFSET = 10.0


def residual_relu_dynamics(rng: np.random.Generator, n: int, m: int, hidden: List[int], dt: float,
                           a: float = 0.95, mix: float = 0.3) -> MLPNet:
    p = n + m
    assert all(h >= p for h in hidden)
    layers = []
    prev = p
    prev_feat = 0
    for li, h in enumerate(hidden):
        F = h - p
        w = np.zeros((h, prev))
        b = np.zeros(h)
        # pass-through of (x, u): first layer adds K, deeper layers keep it
        for i in range(p):
            w[i, i] = 1.0
        if li == 0:
            b[:p] = K_OFFSET
            w[p:, :p] = rng.normal(0.0, 1.0 / np.sqrt(p), size=(F, p))
            b[p:] = rng.normal(0.0, 1.0, size=F)
        else:
            wx = rng.normal(0.0, 1.0 / np.sqrt(p), size=(F, p))
            w[p:, :p] = wx
            b[p:] = rng.normal(0.0, 1.0, size=F) - wx.sum(axis=1) * K_OFFSET  # cancel the K offset
            if prev_feat > 0:
                w[p:, p:prev] = rng.normal(0.0, mix / np.sqrt(prev_feat), size=(F, prev_feat))
        layers.append(Layer(w, b, Act.Relu))
        prev, prev_feat = h, F
    # output layer: x' = a x + dt Bu u + dt Bf f   (inputs carry +K on the first p units)
    w = np.zeros((n, prev))
    b = np.zeros(n)
    w[:, :n] = a * np.eye(n)
    if m > 0:
        bu = dt * rng.normal(0.0, 1.0, size=(n, m))
        w[:, n:p] = bu
    if prev_feat > 0:
        w[:, p:prev] = dt * rng.normal(0.0, 1.0 / np.sqrt(prev_feat), size=(n, prev_feat))
    b[:] = -w[:, :p].sum(axis=1) * K_OFFSET
    layers.append(Layer(w, b, Act.Identity))
    return MLPNet(layers)


def random_mlp(rng: np.random.Generator, in_dim: int, hidden: List[int], out_dim: int, act: Act = Act.Relu,
               scale: float = 1.0) -> MLPNet:
    """Shape of random_mlp (neural.hpp:97-115) on a numpy stream."""
    dims = [in_dim] + list(hidden) + [out_dim]
    layers = []
    for l in range(len(dims) - 1):
        std = scale / np.sqrt(dims[l])
        w = rng.normal(0.0, 1.0, size=(dims[l + 1], dims[l])) * std
        b = rng.normal(0.0, 1.0, size=dims[l + 1]) * 0.05 * scale
        layers.append(Layer(w, b, Act.Identity if l + 2 == len(dims) else act))
    return MLPNet(layers)


@dataclass
class SplitWorkload:
    sys: DTSystem
    x0_lo: np.ndarray
    x0_hi: np.ndarray
    plan: SplitPlan
    actions: np.ndarray  # [H][m]
    horizon: int


def c4_partition_sweep(seed: int = MASTER_SEED, counts=(8, 8, 8, 8, 4, 4), horizon: int = 30) -> SplitWorkload:
    """BASELINE configs[3]: 65,536 sub-boxes of a 6D system, 3x128 ReLU, H = 30 (SURVEY §8 shape sheet C4)."""
    rng = np.random.default_rng(seed + 4)
    n = 6
    net = residual_relu_dynamics(rng, n, 0, [128, 128, 128], dt=0.1)
    c0 = rng.uniform(-0.5, 0.5, size=n)
    return SplitWorkload(DTSystem(net, n, 0), c0 - 0.004, c0 + 0.004, SplitPlan(list(counts)),
                         np.zeros((horizon, 0)), horizon)


@dataclass
class BatchWorkload:
    sys: DTSystem
    x0_lo: np.ndarray  # [B][n]
    x0_hi: np.ndarray
    actions: np.ndarray  # [B][H][m]


def c3_mpc_candidates(seed: int = MASTER_SEED, batch: int = 4096, horizon: int = 20) -> BatchWorkload:
    """BASELINE configs[2] tube leg: 4096 CEM candidates x H=20, 7->96x3->5 ReLU, eps 0.005, U=[-1,1]^2."""
    rng = np.random.default_rng(seed + 3)
    n, m = 5, 2
    net = residual_relu_dynamics(rng, n, m, [96, 96, 96], dt=0.1)
    x0 = np.zeros((batch, n))
    acts = np.clip(rng.normal(0.0, 0.3, size=(batch, horizon, m)), -1.0, 1.0)
    return BatchWorkload(DTSystem(net, n, m), x0 - 0.005, x0 + 0.005, acts)


def small_batch(seed: int, n: int, m: int, hidden: List[int], batch: int, horizon: int, eps: float = 0.01,
                act: Act = Act.Relu, residual: bool = True) -> BatchWorkload:
    """Small seeded batch for parity tests."""
    rng = np.random.default_rng(seed)
    if residual and act == Act.Relu:
        net = residual_relu_dynamics(rng, n, m, hidden, dt=0.1)
    else:
        net = random_mlp(rng, n + m, hidden, n, act, 0.6)
        for L in net.layers[-1:]:
            L.w *= 0.3
    c = rng.uniform(-0.5, 0.5, size=(batch, n))
    r = rng.uniform(0.2 * eps, eps, size=(batch, n))
    acts = rng.uniform(-0.5, 0.5, size=(batch, horizon, m))
    return BatchWorkload(DTSystem(net, n, m), c - r, c + r, acts)


def c3_tpushing(seed: int = MASTER_SEED, population: int = 4096, horizon: int = 20, iterations: int = 5):
    """BASELINE configs[2]: T-pushing reachability-aware MPC -- 7->96x3->5 ReLU
    learned dynamics (n=5 object/pusher state, m=2 push action), H=20, planning
    radius eps=0.005 around x0=0, U=[-1,1]^2, one box-stay-in constraint on the
    object position, CEM with 4096 candidates x 5 iterations, no gradient refine
    (SURVEY.md §8 shape sheet C3 / §8d)."""
    from .mpc import Constraint, PlanProblem, SamplerConfig
    rng = np.random.default_rng(seed + 3)
    n, m = 5, 2
    net = residual_relu_dynamics(rng, n, m, [96, 96, 96], dt=0.1)
    prob = PlanProblem(
        sys=DTSystem(net, n, m),
        x_goal=np.array([0.4, 0.25, 0.0, 0.0, 0.0]),
        q_weights=np.array([1.0, 1.0, 0.1, 0.1, 0.1]),
        r_weights=np.array([0.01, 0.01]),
        constraints=[Constraint(type=Constraint.BOX_STAY_IN, dims=[0, 1], lo=np.array([-0.3, -0.3]),
                                hi=np.array([0.45, 0.3]))],
        penalty=100.0, diverged_margin=1e3, horizon=horizon,
        u_lo=np.array([-1.0, -1.0]), u_hi=np.array([1.0, 1.0]), eps=0.005)
    cfg = SamplerConfig(population=population, elite_frac=0.1, iterations=iterations, init_std=0.3, smoothing=0.5,
                        refine_iters=0, seed=seed)
    return prob, cfg, np.zeros(n)


@dataclass
class ClosedLoopWorkload:
    dyn: MLPNet
    ctl: MLPNet
    n: int
    x0_lo: np.ndarray  # [B][n]
    x0_hi: np.ndarray
    horizon: int


def c1_closed_loop(seed: int = MASTER_SEED, batch: int = 1, horizon: int = 20) -> ClosedLoopWorkload:
    """BASELINE configs[0]: DT closed loop, 4-D NN dynamics (6->64->64->4 ReLU) + 2x64 ReLU
    controller (4->64->64->2), one initial box, H=20 (SURVEY §8 shape sheet C1 / §8d)."""
    rng = np.random.default_rng(seed + 1)
    n, l = 4, 2
    dyn = residual_relu_dynamics(rng, n, l, [64, 64], dt=0.1)
    ctl = random_mlp(rng, n, [64, 64], l, Act.Relu, 0.6)
    ctl.layers[-1].w *= 0.3
    c = rng.uniform(-0.5, 0.5, size=(batch, n))
    return ClosedLoopWorkload(dyn, ctl, n, c - 0.05, c + 0.05, horizon)


def c5_closed_loop(seed: int = MASTER_SEED, batch: int = 1024, horizon: int = 20) -> ClosedLoopWorkload:
    """BASELINE configs[4]: 72-D closed loop (SURVEY §8 shape sheet C5): residual 3x256 ReLU
    dynamics 90->256->256->256->72 (dt 0.02) and a 3x256 ReLU controller 72->...->18
    (random_mlp scale 0.2, output x0.1); X0 = c0 +- 1e-3 with c0 ~ U(-0.2, 0.2)^72, H = 20.

    The survey's C1 controller recipe (scale 0.6, output x0.3) makes the 3x256 loop's certified
    width grow 1.7e26x over 20 steps (vacuous bounds); scale 0.2 / x0.1 grows 21x."""
    rng = np.random.default_rng(seed + 5)
    n, l = 72, 18
    dyn = residual_relu_dynamics(rng, n, l, [256, 256, 256], dt=0.02)
    ctl = random_mlp(rng, n, [256, 256, 256], l, Act.Relu, 0.2)
    ctl.layers[-1].w *= 0.1
    c = rng.uniform(-0.2, 0.2, size=(batch, n))
    return ClosedLoopWorkload(dyn, ctl, n, c - 1e-3, c + 1e-3, horizon)


@dataclass
class CTWorkload:
    spec: "ClosedLoopSpec"
    x0_lo: np.ndarray  # [n]
    x0_hi: np.ndarray
    plan: SplitPlan


def quadrotor_controller(rng: np.random.Generator, hidden=(64, 64, 64), scale: float = 0.4, out_scale: float = 0.1,
                         mass: float = 1.0, gravity: float = 9.81) -> MLPNet:
    """Velocity-command tanh controller of test_closed_loop.cpp:236-241 with the C2 widths:
    random_mlp(15 -> hidden -> 4, Tanh, scale), output layer x out_scale, thrust bias + m g."""
    ctl = random_mlp(rng, 15, list(hidden), 4, Act.Tanh, scale)
    ctl.layers[-1].w *= out_scale
    ctl.layers[-1].b[0] += mass * gravity
    return ctl


def c2_quadrotor(seed: int = MASTER_SEED, parts: int = 4096, ctl_steps: int = 10, k_atomic: int = 5,
                 hidden=(64, 64, 64)) -> CTWorkload:
    """BASELINE configs[1]: 12-D quadrotor (quadrotor_ode) under a 3x64 tanh NN controller (15 -> 4,
    y_ref = (0.1, 0, 0)), order-2 Taylor-model flowpipe, h = 0.01, 10 control intervals x 5 atomic
    steps = 50 steps; X0 = +-0.05 on dims 0-5, +-0.02 on dims 6-11, split rpy:parts."""
    from .api import ClosedLoopSpec, FlowpipeParams
    rng = np.random.default_rng(seed + 2)
    ctl = quadrotor_controller(rng, hidden)
    spec = ClosedLoopSpec(controller=ctl, n=12, l=4, ctl_steps=ctl_steps, k_atomic=k_atomic,
                          y_ref=np.tile([0.1, 0.0, 0.0], (ctl_steps, 1)), fp=FlowpipeParams(h=0.01, order=2))
    r = np.array([0.05] * 6 + [0.02] * 6)
    return CTWorkload(spec, -r, r.copy(), SplitPlan.rpy(12, parts))
