"""Seeded DT parity cases shared by the CPU oracle tests and the GPU tests.

Each case is (name, DTSystem, x0_lo [B][n], x0_hi [B][n], actions [B][H][m],
DTReachParams, tanh?) -- tanh cases are bit-exact between the two CPU
checkers (same libm) and within tolerance on the GPU (CUDA's tanh).
"""
from __future__ import annotations

import json
import os

import numpy as np

from paper_2605_25346_b200.api import Act, DTReachParams, DTSystem, Layer, MLPNet, affine_net
from paper_2605_25346_b200.workloads import random_mlp, residual_relu_dynamics

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "affine_decay.json")


def golden_fixture():
    fx = json.load(open(GOLDEN))
    layers = [Layer(np.array(L["w"], np.float64), np.array(L["b"], np.float64),
                    {"relu": Act.Relu, "tanh": Act.Tanh, "identity": Act.Identity}[L["act"]]) for L in fx["layers"]]
    sys = DTSystem(MLPNet(layers), fx["n"], fx["m"])
    c = np.array(fx["x0_center"])
    lo = (c - fx["eps"])[None, :]
    hi = (c + fx["eps"])[None, :]
    exp_lo = np.array([[float.fromhex(v) for v in row] for row in fx["expected_lo_hex"]])
    exp_hi = np.array([[float.fromhex(v) for v in row] for row in fx["expected_hi_hex"]])
    acts = np.zeros((1, fx["horizon"], 0))
    return sys, lo, hi, acts, exp_lo, exp_hi, fx


def _rand_boxes(rng, B, n, cmax, rmin, rmax):
    c = rng.uniform(-cmax, cmax, size=(B, n))
    r = rng.uniform(rmin, rmax, size=(B, n))
    return c - r, c + r


def cases():
    out = []
    # golden affine decay
    sys, lo, hi, acts, _, _, _ = golden_fixture()
    out.append(("golden_affine", sys, lo, hi, acts, DTReachParams(), False))
    # identity map (test_dt_reach.cpp:52-68)
    n = 3
    sys = DTSystem(affine_net(np.eye(n), np.zeros(n)), n, 0)
    lo, hi = np.array([[0.2, -0.1, 0.4]]) - 0.3, np.array([[0.2, -0.1, 0.4]]) + 0.3
    out.append(("identity", sys, lo, hi, np.zeros((1, 7, 0)), DTReachParams(), False))
    # affine rotation with an action (test_dt_reach.cpp:70-105)
    th = 0.3
    M = 0.9 * np.array([[np.cos(th), -np.sin(th)], [np.sin(th), np.cos(th)]])
    W = np.concatenate([M, np.array([[0.1], [-0.2]])], axis=1)
    sys = DTSystem(affine_net(W, np.array([0.05, 0.0])), 2, 1)
    rng = np.random.default_rng(42)
    acts = rng.uniform(-1, 1, size=(1, 10, 1))
    out.append(("affine_action", sys, np.array([[0.8, -0.7]]), np.array([[1.2, -0.3]]), acts, DTReachParams(), False))
    # zero radius (test_dt_reach.cpp:107-123)
    sys = DTSystem(affine_net(np.array([[0.5, 0.3], [-0.2, 0.8]]), np.array([0.1, -0.1])), 2, 0)
    out.append(("zero_radius", sys, np.array([[0.7, 0.2]]), np.array([[0.7, 0.2]]), np.zeros((1, 6, 0)),
                DTReachParams(), False))
    # random ReLU 2x32 nets, n=4, m=2 (test_dt_reach.cpp:125-170 shapes)
    rng = np.random.default_rng(2024)
    for c in range(3):
        net = random_mlp(rng, 6, [32, 32], 4, Act.Relu, 0.6)
        net.layers[-1].w *= 0.3
        lo, hi = _rand_boxes(rng, 12, 4, 0.6, 0.01, 0.2)
        acts = rng.uniform(-0.5, 0.5, size=(12, 10, 2))
        out.append((f"random_relu_{c}", DTSystem(net, 4, 2), lo, hi, acts, DTReachParams(), False))
    # tanh net (test_dt_reach.cpp:202-250 shapes)
    rng = np.random.default_rng(77)
    net = random_mlp(rng, 4, [16], 3, Act.Tanh, 0.5)
    lo, hi = _rand_boxes(rng, 9, 3, 0.5, 0.01, 0.15)
    acts = rng.uniform(-0.3, 0.3, size=(9, 6, 1))
    out.append(("tanh_16", DTSystem(net, 3, 1), lo, hi, acts, DTReachParams(), True))
    # residual ReLU dynamics of the C4 and C3 shapes
    rng = np.random.default_rng(7)
    net = residual_relu_dynamics(rng, 6, 0, [128, 128, 128], dt=0.1)
    lo, hi = _rand_boxes(rng, 24, 6, 0.5, 5e-4, 4e-3)
    out.append(("c4_shape", DTSystem(net, 6, 0), lo, hi, np.zeros((24, 30, 0)), DTReachParams(), False))
    rng = np.random.default_rng(8)
    net = residual_relu_dynamics(rng, 5, 2, [96, 96, 96], dt=0.1)
    lo = np.full((24, 5), -0.005)
    hi = np.full((24, 5), 0.005)
    acts = np.clip(rng.normal(0, 0.3, size=(24, 20, 2)), -1, 1)
    out.append(("c3_shape", DTSystem(net, 5, 2), lo, hi, acts, DTReachParams(), False))
    # window / ablation variants on a 4D ReLU net
    rng = np.random.default_rng(11)
    net = random_mlp(rng, 5, [48, 48], 4, Act.Relu, 0.7)
    net.layers[-1].w *= 0.4
    lo, hi = _rand_boxes(rng, 8, 4, 0.5, 0.01, 0.1)
    acts = rng.uniform(-0.5, 0.5, size=(8, 12, 1))
    for w in (0, 1, 2, 6):
        out.append((f"window_{w}", DTSystem(net, 4, 1), lo, hi, acts, DTReachParams(window=w), False))
    out.append(("rebuild_from_box", DTSystem(net, 4, 1), lo, hi, acts, DTReachParams(rebuild_from_box=True), False))
    # explosive dynamics: diverged box / certification / non-finite preactivation
    rng = np.random.default_rng(5)
    net = random_mlp(rng, 3, [32, 32], 3, Act.Relu, 3.0)
    net.layers[-1].w *= 20.0
    lo, hi = _rand_boxes(rng, 16, 3, 1.0, 0.05, 0.5)
    out.append(("explosive", DTSystem(net, 3, 0), lo, hi, np.zeros((16, 110, 0)), DTReachParams(), False))
    # wide hidden (256) and n = 8
    rng = np.random.default_rng(13)
    net = residual_relu_dynamics(rng, 8, 0, [256, 200], dt=0.05)
    lo, hi = _rand_boxes(rng, 10, 8, 0.3, 1e-3, 5e-3)
    out.append(("wide_n8", DTSystem(net, 8, 0), lo, hi, np.zeros((10, 12, 0)), DTReachParams(window=2), False))
    # a hidden unit whose preactivation is exactly [0, 0] on a point box (W x + b = 1 - 0.5 - 0.5):
    # relax_activation makes it stably ACTIVE (lo >= 0 branch first), so its Lambda column survives
    rng = np.random.default_rng(19)
    W0 = np.concatenate([np.array([[1.0, -1.0]]), rng.normal(0, 0.5, size=(4, 2))])
    b0 = np.concatenate([[-0.5], rng.normal(0, 0.3, size=4)])
    W1 = rng.normal(0, 0.5, size=(5, 5))
    b1 = rng.normal(0, 0.3, size=5)
    W2 = rng.normal(0, 0.3, size=(2, 5))
    b2 = rng.normal(0, 0.1, size=2)
    net = MLPNet([Layer(W0, b0, Act.Relu), Layer(W1, b1, Act.Relu), Layer(W2, b2, Act.Identity)])
    out.append(("zero_preact_point", DTSystem(net, 2, 0), np.array([[1.0, 0.5]]), np.array([[1.0, 0.5]]),
                np.zeros((1, 3, 0)), DTReachParams(), False))
    # n = 1, one hidden layer of 20
    rng = np.random.default_rng(17)
    net = random_mlp(rng, 2, [20], 1, Act.Relu, 0.8)
    lo, hi = _rand_boxes(rng, 5, 1, 0.5, 0.01, 0.2)
    acts = rng.uniform(-1, 1, size=(5, 9, 1))
    out.append(("n1_m1", DTSystem(net, 1, 1), lo, hi, acts, DTReachParams(), False))
    return out
