"""Seeded grad_tube_volume cases (refine.hpp:263-311) shared by CPU and GPU tests: the shapes of
test_refine.cpp:195-284 plus a C4-shaped ReLU map."""
import numpy as np

from paper_2605_25346_b200.api import Act, DTReachParams, DTSystem, affine_net
from paper_2605_25346_b200.workloads import random_mlp


def _box(c, r):
    c = np.asarray(c, np.float64)
    return (c - r, c + r)


def grad_cases():
    """(name, sys, x0, actions, prm, exact) -- exact: ReLU / identity (bit-identical to the reference)."""
    rng = np.random.default_rng(9090)
    out = []
    sys = DTSystem(random_mlp(rng, 2, [8], 2, Act.Relu, 0.6), 2, 0)
    out.append(("relu_weights_small", sys, _box([0.3, -0.2], 0.05), [[]] * 3, DTReachParams(), True))
    sys = DTSystem(random_mlp(rng, 5, [10], 3, Act.Tanh, 0.5), 3, 2)
    acts = [rng.uniform(-0.3, 0.3, 2) for _ in range(4)]
    out.append(("tanh_actions_center", sys, _box([0.1, 0.0, -0.2], 0.05), acts, DTReachParams(), False))
    net = random_mlp(rng, 6, [32, 32], 4, Act.Relu, 0.6)
    net.layers[-1].w *= 0.3
    sys = DTSystem(net, 4, 2)
    acts = [rng.uniform(-0.5, 0.5, 2) for _ in range(10)]
    out.append(("relu_4d_window4", sys, _box(rng.uniform(-0.4, 0.4, 4), 0.08), acts, DTReachParams(4, False), True))
    out.append(("relu_4d_window2", sys, _box(rng.uniform(-0.4, 0.4, 4), 0.08), acts, DTReachParams(2, False), True))
    out.append(("relu_4d_rebuild", sys, _box(rng.uniform(-0.4, 0.4, 4), 0.08), acts, DTReachParams(4, True), True))
    net = random_mlp(rng, 6, [128, 128, 128], 6, Act.Relu, 0.9)
    net.layers[-1].w *= 0.5
    sys = DTSystem(net, 6, 0)
    out.append(("c4_shape", sys, _box(np.zeros(6), 0.05), [[]] * 4, DTReachParams(), True))
    return out


def identity_case():
    """test_refine.cpp:195-217: identity map and pure-translation action channel."""
    sys = DTSystem(affine_net(np.eye(2), np.zeros(2)), 2, 0)
    w = np.zeros((2, 4))
    w[0, 0] = w[1, 1] = w[0, 2] = w[1, 3] = 1.0
    trans = DTSystem(affine_net(w, np.zeros(2)), 2, 2)
    return sys, trans, _box([0.4, -0.3], 0.2)


def diverging_case():
    """A map that blows up: the tube diverges, tube_volume = +inf, grad_forward throws."""
    sys = DTSystem(affine_net(np.eye(2) * 1e200, np.zeros(2)), 2, 0)
    return sys, _box([0.5, 0.5], 0.1), [[]] * 4
