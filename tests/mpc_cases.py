"""Seeded MPC cases (problems of mpc.hpp shape) shared by CPU and GPU tests."""
import numpy as np

from paper_2605_25346_b200.api import DTSystem, affine_net
from paper_2605_25346_b200.mpc import Constraint, PlanProblem, SamplerConfig
from paper_2605_25346_b200.workloads import c3_tpushing, random_mlp


def integrator_problem(n=2, horizon=6, u_max=0.5):
    """x' = x + u (test_mpc.cpp:17-42) with every constraint type."""
    w = np.concatenate([np.eye(n), np.eye(n)], axis=1)
    sys = DTSystem(affine_net(w, np.zeros(n)), n, n)
    cons = [
        Constraint(type=Constraint.HALFSPACE_AVOID, a=np.array([1.0, 0.5]), b=0.8),
        Constraint(type=Constraint.SPHERE_AVOID, center=np.array([0.3, -0.2]), radius=0.15),
        Constraint(type=Constraint.BOX_STAY_IN, dims=[1], lo=np.array([-0.6]), hi=np.array([0.6])),
        Constraint(type=Constraint.MAX_VOLUME, vmax=0.05),
    ]
    return PlanProblem(sys, np.array([0.7, 0.1]), np.ones(n), np.full(n, 0.01), cons, horizon=horizon,
                       u_lo=np.full(n, -u_max), u_hi=np.full(n, u_max), eps=0.02)


def relu_problem(seed=5, horizon=8):
    rng = np.random.default_rng(seed)
    net = random_mlp(rng, 5, [24, 24], 3, scale=0.7)
    net.layers[-1].w *= 0.4
    sys = DTSystem(net, 3, 2)
    cons = [Constraint(type=Constraint.SPHERE_AVOID, dims=[0, 2], center=np.array([0.2, 0.1]), radius=0.1),
            Constraint(type=Constraint.BOX_STAY_IN, lo=np.full(3, -1.0), hi=np.full(3, 1.0))]
    return PlanProblem(sys, np.array([0.3, -0.2, 0.1]), np.ones(3), np.full(2, 0.05), cons, horizon=horizon,
                       u_lo=np.full(2, -1.0), u_hi=np.full(2, 1.0), eps=0.01)


def explosive_problem(horizon=12):
    """A one-step map that diverges: penalties fall back to diverged_margin (test_mpc.cpp:367-397)."""
    w = np.concatenate([np.eye(2) * 1e30, np.eye(2)], axis=1)
    sys = DTSystem(affine_net(w, np.zeros(2)), 2, 2)
    cons = [Constraint(type=Constraint.MAX_VOLUME, vmax=1.0)]
    return PlanProblem(sys, np.zeros(2), np.ones(2), np.full(2, 0.01), cons, horizon=horizon,
                       u_lo=np.full(2, -1.0), u_hi=np.full(2, 1.0), eps=0.1)


def plan_cases():
    rng = np.random.default_rng(11)
    out = []
    for name, prob in (("integrator", integrator_problem()), ("relu", relu_problem()),
                       ("explosive", explosive_problem())):
        acts = rng.uniform(prob.u_lo, prob.u_hi, size=(16, prob.horizon, prob.sys.m))
        out.append((name, prob, rng.uniform(-0.3, 0.3, prob.sys.n), acts))
    prob, cfg, x0 = c3_tpushing(population=64, horizon=20)
    acts = np.clip(rng.normal(0.0, 0.4, size=(24, 20, 2)), -1, 1)
    out.append(("c3_tpushing", prob, x0, acts))
    return out


def small_cem():
    prob = relu_problem(horizon=6)
    return prob, SamplerConfig(population=48, elite_frac=0.1, iterations=4, init_std=0.3, smoothing=0.5,
                               refine_iters=0, seed=3), np.array([0.05, -0.05, 0.0])


def odd_cem():
    """An odd draw count per iteration (1201 candidates x H=7 x m=1 = 8407 normals, then 8400 >= the 4096-pair
    threshold of the threaded Box-Muller transform): the cached spare normal carries over between
    iterations (rng.hpp:24-37), and the multi-threaded transform branch runs."""
    rng = np.random.default_rng(17)
    net = random_mlp(rng, 4, [24, 24], 3, scale=0.7)
    net.layers[-1].w *= 0.4
    sys = DTSystem(net, 3, 1)
    cons = [Constraint(type=Constraint.BOX_STAY_IN, lo=np.full(3, -1.0), hi=np.full(3, 1.0))]
    prob = PlanProblem(sys, np.array([0.2, -0.1, 0.05]), np.ones(3), np.full(1, 0.05), cons, horizon=7,
                       u_lo=np.full(1, -1.0), u_hi=np.full(1, 1.0), eps=0.01)
    return prob, SamplerConfig(population=1201, elite_frac=0.05, iterations=3, init_std=0.4, smoothing=0.3,
                               refine_iters=0, seed=9), np.array([0.02, 0.0, -0.03])
