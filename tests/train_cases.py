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
