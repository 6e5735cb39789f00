"""Seeded certified-training cases (training.hpp) shared by the CPU reference tests and the GPU tests:
a small residual ReLU dynamics model and random-action rollouts of a perturbed 'true' system."""
import numpy as np

from paper_2605_25346_b200.api import Episode, TrainConfig
from paper_2605_25346_b200.workloads import residual_relu_dynamics


def dt_training_case(seed=5, n=4, m=2, hidden=(32, 32), episodes=6, length=6):
    rng = np.random.default_rng(seed)
    model = residual_relu_dynamics(rng, n, m, list(hidden), dt=0.1)
    true = residual_relu_dynamics(rng, n, m, list(hidden), dt=0.1)  # the data-generating system
    data = []
    for _ in range(episodes):
        x = rng.uniform(-0.5, 0.5, n)
        xs, us = [x.copy()], []
        for _ in range(length):
            u = rng.uniform(-0.5, 0.5, m)
            x = true.forward(np.concatenate([x, u])[:, None])[:, 0]
            xs.append(x.copy())
            us.append(u)
        data.append(Episode(xs, us))
    return model, data


def train_config(lambda_=0.5, iters=4, horizon_max=4, batch=3, seed=11):
    return TrainConfig(horizon_max=horizon_max, eps0=0.02, eps_final=0.005, lambda_=lambda_, iters=iters,
                       batch=batch, lr=1e-3, reach_cap=20.0, curriculum=True, seed=seed)


def ct_tracking_case(seed=7, episodes=4, length=5, delta=0.05, with_ref=True):
    """Quadrotor tracking data: closed-loop rollouts of a perturbed controller (RK4 with fine steps) and
    a freshly initialised controller to train (the C2 controller family, 15 -> 3x16 tanh -> 4)."""
    from paper_2605_25346_b200.workloads import quadrotor_controller
    rng = np.random.default_rng(seed)
    ctl = quadrotor_controller(rng, (16, 16, 16))
    teacher = quadrotor_controller(rng, (16, 16, 16))
    data = []
    prm = [1.0, 9.81, 0.01, 0.01, 0.02]

    def rhs(x, u):
        m, g, jx, jy, jz = prm
        phi, th, psi, p, q, r = x[6], x[7], x[8], x[9], x[10], x[11]
        sphi, cphi, sth, cth, spsi, cpsi = np.sin(phi), np.cos(phi), np.sin(th), np.cos(th), np.sin(psi), np.cos(psi)
        a = u[0] / m
        return np.array([x[3], x[4], x[5], a * (cphi * sth * cpsi + sphi * spsi), a * (cphi * sth * spsi - sphi * cpsi),
                         a * cphi * cth - g, p + sphi * sth / cth * q + cphi * sth / cth * r, cphi * q - sphi * r,
                         sphi / cth * q + cphi / cth * r, q * r * (jy - jz) / jx + u[1] / jx,
                         p * r * (jz - jx) / jy + u[2] / jy, p * q * (jx - jy) / jz + u[3] / jz])

    for _ in range(episodes):
        x = np.concatenate([rng.uniform(-0.05, 0.05, 6), rng.uniform(-0.02, 0.02, 6)])
        ref = np.tile([0.1, 0.0, 0.0], (length, 1)) + rng.uniform(-0.02, 0.02, (length, 3))
        xs, us = [x.copy()], []
        for t in range(length):
            u = teacher.forward(np.concatenate([x, ref[t]])[:, None])[:, 0]
            h = delta / 8
            for _ in range(8):
                k1 = rhs(x, u)
                k2 = rhs(x + 0.5 * h * k1, u)
                k3 = rhs(x + 0.5 * h * k2, u)
                k4 = rhs(x + h * k3, u)
                x = x + h / 6 * (k1 + 2 * k2 + 2 * k3 + k4)
            xs.append(x.copy())
            us.append(u)
        data.append(Episode(xs, us, [list(rr) for rr in ref] if with_ref else ()))
    return ctl, data
