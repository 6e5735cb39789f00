"""Command-line surface of the reference (tools/reach_cli.cpp) on the device engines.

    python -m paper_2605_25346_b200.cli reach-dt --net net.json --x0-center 0.5,0.5 --eps 0.125 --steps 8 --out o

Same subcommands, flags, self-contained JSON config, buffered outputs (tube.csv / tube.json /
manifest.json, run_log.csv / result.json, refine.json), manifest rerun and exit codes as the reference
(reach_cli.cpp:36-40): 0 success, 2 configuration error, 3 dimension error (no output), 4 step failure,
5 divergence (artifacts written, flagged in the tube).  Every reachable set comes from the CUDA library;
systems, baselines or modes the device library does not carry (the swarm / arm plants, the interval
baselines, outward rounding, training, bench) are configuration errors, never a CPU fallback.
"""
from __future__ import annotations

import argparse
import os
import sys
from typing import List, Tuple

import numpy as np

from . import formats as F
from .api import (DTSystem, FlowpipeParams, dt_interval_baseline, ClosedLoopSpec, GradTarget, QuadrotorParams, SplitPlan, box_from_center,
                  cl_reach, ct_reach, ct_reach_with_splitting, diag_linear_field, dt_reach, quadrotor_field,
                  quadrotor_hover_input, reach_with_splitting, refine_tube_volume, rotation_field)

EXIT_OK, EXIT_CONFIG, EXIT_DIMENSION, EXIT_STEP, EXIT_DIVERGENCE = 0, 2, 3, 4, 5


class ConfigError(RuntimeError):
    pass


class DimensionError(RuntimeError):
    pass


class Outputs:
    """Buffered outputs: nothing touches the filesystem until the run may emit artifacts."""

    def __init__(self):
        self.files: List[Tuple[str, str]] = []

    def add(self, name: str, content: str):
        self.files.append((name, content))

    def write_all(self, out_dir: str):
        os.makedirs(out_dir, exist_ok=True)
        for name, content in self.files:
            F.write_text_file(os.path.join(out_dir, name), content)


def parse_list(s: str) -> List[float]:
    out = []
    for tok in s.split(","):
        if tok == "":
            raise ValueError('empty entry in list "' + s + '"')
        out.append(float(tok))
    return out


def make_split_plan(spec: str, n_dims: int) -> SplitPlan:
    if spec.startswith("rpy:"):
        return SplitPlan.rpy(n_dims, int(spec[4:]))
    plan = SplitPlan.parse(spec)
    plan.validate(n_dims)
    return plan


def make_field(name: str):
    """System registry (reach_cli.cpp:96-117) restricted to the fields compiled into the device library."""
    if name == "quadrotor":
        prm = QuadrotorParams()
        return quadrotor_field(prm, quadrotor_hover_input(prm)), 12
    if name == "rotation":
        return rotation_field(1.0), 2
    if name == "decay":
        return diag_linear_field([-1.0]), 1
    if name in ("swarm", "arm"):
        raise ConfigError('system "' + name + '" is not compiled into the device library (known on the device: '
                          "quadrotor, rotation, decay)")
    raise ConfigError('unknown system "' + name + '" (known: quadrotor, swarm, arm, rotation, decay)')


def _unsupported_modes(cfg: dict, dt: bool = False):
    if cfg.get("baseline", "") == "interval" and not dt:
        raise ConfigError("the continuous-time interval baseline (baseline.hpp) is not part of the device build")
    if cfg.get("sound_rounding", False):
        raise ConfigError("outward rounding is not supported by the device kernels")


def emit_tube(out: Outputs, tube, with_time: bool):
    out.add("tube.csv", F.tube_to_csv(tube, with_time))
    out.add("tube.json", F.json_dump(F.tube_to_json(tube)) + "\n")


def finish(command: str, cfg: dict, out_dir: str, out: Outputs, diverged: bool, reason: str) -> int:
    m = F.Manifest(command, cfg, int(cfg.get("seed", 0)), os.cpu_count() or 1)
    out.add("manifest.json", F.json_dump(m.to_json()) + "\n")
    out.write_all(out_dir)
    if diverged:
        print("divergence: " + (reason or "enclosure diverged"), file=sys.stderr)
        return EXIT_DIVERGENCE
    return EXIT_OK


# ---------------------------------------------------------------------------
def cmd_reach_ct(cfg: dict, out_dir: str, command: str) -> int:
    field, n = make_field(cfg["system"])
    center = [float(v) for v in cfg["x0_center"]]
    if len(center) != n:
        raise DimensionError(f'x0 has {len(center)} dims, system "{cfg["system"]}" has {n}')
    fp = FlowpipeParams(h=float(cfg.get("h", 0.01)), steps=int(cfg.get("steps", 100)), order=int(cfg.get("order", 2)))
    fp.validate()
    x0 = box_from_center(center, float(cfg.get("eps", 0.0)))
    _unsupported_modes(cfg)
    split = cfg.get("split", "")
    tube = ct_reach(field, x0, fp) if not split else ct_reach_with_splitting(field, x0, make_split_plan(split, n), fp)
    out = Outputs()
    emit_tube(out, tube, True)
    return finish(command, cfg, out_dir, out, tube.diverged, tube.failure_reason)


def _dt_system(cfg: dict):
    net = F.net_from_json(cfg["net"])
    center = [float(v) for v in cfg["x0_center"]]
    n = len(center)
    m = net.input_dim() - n
    if m < 0 or net.output_dim() != n:
        raise DimensionError(f"one-step map is {net.input_dim()} -> {net.output_dim()}, x0 has {n} dims")
    sys_ = DTSystem(net, n, m)
    sys_.validate()
    return sys_, center


def cmd_reach_dt(cfg: dict, out_dir: str) -> int:
    sys_, center = _dt_system(cfg)
    n, m = sys_.n, sys_.m
    if "actions" in cfg:
        actions = [[float(v) for v in a] for a in cfg["actions"]]
        for a in actions:
            if len(a) != m:
                raise DimensionError(f"action row has {len(a)} dims, map expects {m}")
    else:
        actions = [[0.0] * m for _ in range(int(cfg.get("steps", 10)))]
    x0 = box_from_center(center, float(cfg.get("eps", 0.0)))
    _unsupported_modes(cfg, dt=True)
    baseline = cfg.get("baseline", "") == "interval"
    split = cfg.get("split", "")
    if baseline and split:
        raise ConfigError("--baseline interval with --split: the split engine is dt_reach on the device")
    precision = cfg.get("precision", "exact")  # device precision mode (not a reference option)
    if baseline:
        tube = dt_interval_baseline(sys_, x0, actions)
    elif split:
        tube = reach_with_splitting(sys_, x0, make_split_plan(split, n), actions, precision=precision)
    else:
        tube = dt_reach(sys_, x0, actions, precision=precision)
    out = Outputs()
    emit_tube(out, tube, False)
    return finish("reach-dt", cfg, out_dir, out, tube.diverged, tube.failure_reason)


def cmd_reach_cl(cfg: dict, out_dir: str) -> int:
    name = cfg["system"]
    if name != "quadrotor":
        if name in ("arm", "swarm", "integrator2"):
            raise ConfigError('closed-loop system "' + name + '" is not compiled into the device library '
                              "(on the device: quadrotor)")
        raise ConfigError('unknown closed-loop system "' + name + '" (known: quadrotor, arm, swarm, integrator2)')
    n, l = 12, 4
    controller = F.net_from_json(cfg["net"])
    center = [float(v) for v in cfg["x0_center"]]
    if len(center) != n:
        raise DimensionError(f"x0 has {len(center)} dims, plant has {n}")
    if controller.input_dim() != n or controller.output_dim() != l:
        raise DimensionError(f"controller is {controller.input_dim()} -> {controller.output_dim()}, plant needs "
                             f"{n} -> {l}")
    ctl_steps, k_atomic = int(cfg.get("steps", 5)), int(cfg.get("k_atomic", 1))
    fp = FlowpipeParams(h=float(cfg.get("h", 0.01)), order=int(cfg.get("order", 2)), steps=ctl_steps * k_atomic)
    spec = ClosedLoopSpec(controller, n=n, l=l, ctl_steps=ctl_steps, k_atomic=k_atomic, fp=fp)
    spec.validate()
    x0 = box_from_center(center, float(cfg.get("eps", 0.0)))
    _unsupported_modes(cfg)
    tube = cl_reach(spec, x0)
    out = Outputs()
    emit_tube(out, tube, True)
    return finish("reach-cl", cfg, out_dir, out, tube.diverged, tube.failure_reason)


def cmd_refine(cfg: dict, out_dir: str) -> int:
    sys_, center = _dt_system(cfg)
    horizon, eps = int(cfg.get("steps", 10)), float(cfg.get("eps", 0.0))
    bound, target = float(cfg.get("bound", 0.5)), cfg.get("target", "center")
    if target not in ("center", "actions"):
        raise ConfigError('refine target must be "center" or "actions"')
    actions = [[0.0] * sys_.m for _ in range(horizon)]
    x = np.array(center if target == "center" else [0.0] * (horizon * sys_.m), np.float64)
    t = GradTarget.x0_center if target == "center" else GradTarget.actions
    res = refine_tube_volume(sys_, center, eps, actions, t, x - bound, x + bound, int(cfg.get("grad_iters", 20)), x)
    out = Outputs()
    rj = {"target": target, "initial_objective": res.initial_objective, "objective": res.objective,
          "progressed": res.progressed, "subgradient": res.subgradient, "accepted_steps": res.accepted_steps,
          "x": list(map(float, res.x))}
    out.add("refine.json", F.json_dump(rj) + "\n")
    return finish("refine", cfg, out_dir, out, False, "")


def cmd_mpc(cfg: dict, out_dir: str) -> int:
    from .mpc import mpc_run
    prob, sampler, mpc = F.scenario_from_json(cfg["scenario"])
    x0 = [float(v) for v in cfg["x0_center"]]
    if len(x0) != prob.sys.n:
        raise DimensionError(f"x0 has {len(x0)} dims, model has {prob.sys.n}")
    if "seed" in cfg:
        mpc.seed = int(cfg["seed"])
        sampler.seed = int(cfg["seed"])
    res = mpc_run(prob, sampler, mpc, np.array(x0))  # sim = the model's forward on the device
    out = Outputs()
    out.add("run_log.csv", res.log_to_csv())
    rj = {"success": res.success, "violated": res.violated, "steps_used": res.steps_used,
          "final_state": list(map(float, res.final_state))}
    out.add("result.json", F.json_dump(rj) + "\n")
    return finish("mpc", cfg, out_dir, out, False, "")


def run_command(command: str, cfg: dict, out_dir: str) -> int:
    if command in ("reach-ct", "split"):
        return cmd_reach_ct(cfg, out_dir, command)
    if command == "reach-dt":
        return cmd_reach_dt(cfg, out_dir)
    if command == "reach-cl":
        return cmd_reach_cl(cfg, out_dir)
    if command == "refine":
        return cmd_refine(cfg, out_dir)
    if command == "mpc":
        return cmd_mpc(cfg, out_dir)
    if command in ("train-dt", "train-ctl", "bench"):
        raise ConfigError(f"{command} (training / the CPU bench) is not part of the device build")
    raise ValueError("unknown command in manifest: " + command)


def run_guarded(command: str, cfg: dict, out_dir: str) -> int:
    try:
        return run_command(command, cfg, out_dir)
    except ConfigError as e:
        print("config error: " + str(e), file=sys.stderr)
        return EXIT_CONFIG
    except DimensionError as e:
        print("dimension error: " + str(e), file=sys.stderr)
        return EXIT_DIMENSION
    except (KeyError, TypeError) as e:  # missing / mistyped config entries (nlohmann::json::exception)
        print("config error: " + str(e), file=sys.stderr)
        return EXIT_CONFIG
    except ValueError as e:  # engine-level validation failures are dimension/shape errors by contract
        print("dimension error: " + str(e), file=sys.stderr)
        return EXIT_DIMENSION
    except Exception as e:  # noqa: BLE001
        print("step failure: " + str(e), file=sys.stderr)
        return EXIT_STEP


class _Parser(argparse.ArgumentParser):
    def error(self, message):  # CLI11 parse errors exit with the config code
        print(message, file=sys.stderr)
        raise SystemExit(EXIT_CONFIG)


def main(argv=None) -> int:
    p = _Parser(prog="reach_cli", description="certified reachability toolkit (B200)")
    sub = p.add_subparsers(dest="command", required=True, parser_class=_Parser)

    def common_reach(c, ct):
        c.add_argument("--x0-center", required=True)
        c.add_argument("--eps", type=float, default=0.0)
        c.add_argument("--steps", type=int, default=10)
        if ct:
            c.add_argument("--h", type=float, default=0.01)
            c.add_argument("--order", type=int, default=2)
        c.add_argument("--split", default="")
        c.add_argument("--seed", type=int)
        c.add_argument("--sound-rounding", action="store_true")
        c.add_argument("--out", default="out")

    for name in ("reach-ct", "split"):
        c = sub.add_parser(name)
        c.add_argument("--system", required=True)
        c.add_argument("--baseline", default="")
        common_reach(c, True)
    c = sub.add_parser("reach-dt")
    c.add_argument("--net", required=True)
    c.add_argument("--actions", default="")
    c.add_argument("--baseline", default="")
    c.add_argument("--precision", default="exact", choices=["exact", "fused", "tc"],
                   help="device precision mode: exact (the reference bit for bit), fused (fp64 DFMA), tc (tensor cores)")
    common_reach(c, False)
    c = sub.add_parser("reach-cl")
    c.add_argument("--system", required=True)
    c.add_argument("--net", required=True)
    c.add_argument("--k-atomic", type=int, default=1)
    common_reach(c, True)
    c = sub.add_parser("refine")
    c.add_argument("--net", required=True)
    c.add_argument("--x0-center", required=True)
    c.add_argument("--eps", type=float, default=0.0)
    c.add_argument("--steps", type=int, default=10)
    c.add_argument("--grad-iters", type=int, default=20)
    c.add_argument("--bound", type=float, default=0.5)
    c.add_argument("--target", default="center")
    c.add_argument("--seed", type=int)
    c.add_argument("--out", default="out")
    for name in ("train-dt", "train-ctl"):
        c = sub.add_parser(name)
        for flag in ("--iters", "--batch", "--horizon", "--hidden", "--seed"):
            c.add_argument(flag, type=int)
        for flag in ("--lambda", "--lr", "--eps0", "--eps-final"):
            c.add_argument(flag, type=float)
        c.add_argument("--out", default="out")
    c = sub.add_parser("mpc")
    c.add_argument("--scenario", required=True)
    c.add_argument("--x0-center", required=True)
    c.add_argument("--seed", type=int)
    c.add_argument("--out", default="out")
    c = sub.add_parser("bench")
    c.add_argument("--h", type=float, default=0.01)
    c.add_argument("--steps", type=int, default=10)
    c.add_argument("--out", default="out")
    c = sub.add_parser("rerun")
    c.add_argument("--manifest", required=True)
    c.add_argument("--out", default="out")
    a = p.parse_args(argv)
    name = a.command
    try:
        if name == "rerun":
            m = F.Manifest.from_json(F.read_json_file(a.manifest))
            return run_guarded(m.command, m.config, a.out)
        cfg: dict = {}
        if getattr(a, "seed", None) is not None:
            cfg["seed"] = a.seed
        if name in ("reach-ct", "split", "reach-dt", "reach-cl"):
            cfg["x0_center"] = parse_list(a.x0_center)
            cfg["eps"] = a.eps
            cfg["steps"] = a.steps
            if a.split:
                cfg["split"] = a.split
            if a.sound_rounding:
                cfg["sound_rounding"] = True
            if getattr(a, "baseline", ""):
                cfg["baseline"] = a.baseline
        if name in ("reach-ct", "split", "reach-cl"):
            cfg["system"] = a.system
            cfg["h"] = a.h
            cfg["order"] = a.order
        if name == "split" and not a.split:
            raise ValueError("split requires --split")
        if name in ("reach-dt", "reach-cl", "refine"):
            cfg["net"] = F.read_json_file(a.net)
            if getattr(a, "precision", "exact") != "exact":
                cfg["precision"] = a.precision  # recorded in the manifest only when not the default
        if name == "reach-dt" and a.actions:
            cfg["actions"] = F.read_json_file(a.actions)
        if name == "reach-cl":
            cfg["k_atomic"] = a.k_atomic
        if name == "refine":
            cfg.update({"x0_center": parse_list(a.x0_center), "eps": a.eps, "steps": a.steps,
                        "grad_iters": a.grad_iters, "bound": a.bound, "target": a.target})
        if name == "mpc":
            cfg["scenario"] = F.read_json_file(a.scenario)
            cfg["x0_center"] = parse_list(a.x0_center)
        if name == "bench":
            cfg.update({"h": a.h, "steps": a.steps})
        if name in ("train-dt", "train-ctl"):
            cfg["iters"] = a.iters
        return run_guarded(name, cfg, a.out)
    except Exception as e:  # noqa: BLE001  (building the config: unreadable files, bad lists)
        print("config error: " + str(e), file=sys.stderr)
        return EXIT_CONFIG


if __name__ == "__main__":
    sys.exit(main())
