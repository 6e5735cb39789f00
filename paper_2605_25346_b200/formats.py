"""Serialization formats of the reference (io.hpp, mpc.hpp:500-613), byte-compatible:

    fmt_g17                      io.hpp:23-27     printf("%.17g")
    net_to_json / net_from_json  io.hpp:32-63
    tube_to_json / tube_from_json io.hpp:68-104
    tube_to_csv / tube_from_csv  io.hpp:109-160   (DT: no time-window columns)
    Manifest                     io.hpp:165-195
    json_dump                    nlohmann::json::dump(2): sorted keys, 2-space indent,
                                 shortest round-trip doubles, non-finite -> null
    scenario_to_json / _from_json mpc.hpp:500-613

Host-side text I/O only; nothing here computes a reachable set.
"""
from __future__ import annotations

import json
import math
import os
from dataclasses import dataclass, field
from typing import Any, Optional

import numpy as np

from .api import Act, Layer, MLPNet, ReachTube

VERSION = "reach-0.1.0"
_ACT_NAME = {Act.Relu: "relu", Act.Tanh: "tanh", Act.Identity: "identity"}


def fmt_g17(v: float) -> str:
    return "%.17g" % v


def _plain(o: Any) -> Any:
    """JSON-ready copy: numpy -> Python, non-finite doubles -> None (nlohmann writes null)."""
    if isinstance(o, dict):
        return {str(k): _plain(v) for k, v in o.items()}
    if isinstance(o, (list, tuple)):
        return [_plain(v) for v in o]
    if isinstance(o, np.ndarray):
        return [_plain(v) for v in o.tolist()]
    if isinstance(o, (bool, np.bool_)):
        return bool(o)
    if isinstance(o, (int, np.integer)):
        return int(o)
    if isinstance(o, (float, np.floating)):
        f = float(o)
        return f if math.isfinite(f) else None
    return o


def json_dump(o: Any) -> str:
    """nlohmann::json::dump(2): std::map key order, 2-space indent, shortest round-trip doubles."""
    return json.dumps(_plain(o), indent=2, sort_keys=True, ensure_ascii=False)


# ---------------------------------------------------------------------------
def act_name(a: Act) -> str:
    return _ACT_NAME[Act(a)]


def act_from_name(s: str) -> Act:
    for k, v in _ACT_NAME.items():
        if v == s:
            return k
    raise ValueError("unknown activation: " + str(s))


def net_to_json(net: MLPNet) -> dict:
    return {"layers": [{"act": act_name(L.act), "w": [list(map(float, row)) for row in np.asarray(L.w)],
                        "b": list(map(float, np.asarray(L.b)))} for L in net.layers]}


def net_from_json(j: dict) -> MLPNet:
    layers = []
    for lj in j["layers"]:
        rows = lj["w"]
        r = len(rows)
        c = len(rows[0]) if r else 0
        if any(len(row) != c for row in rows):
            raise ValueError("net_from_json: ragged weight matrix")
        w = np.array(rows, dtype=np.float64).reshape(r, c)
        b = np.array(lj["b"], dtype=np.float64)
        layers.append(Layer(w, b, act_from_name(lj["act"])))
    net = MLPNet(layers)
    net.validate()
    return net


# ---------------------------------------------------------------------------
def tube_to_json(t: ReachTube) -> dict:
    return {"boxes": [{"lo": list(map(float, t.lo[k])), "hi": list(map(float, t.hi[k]))} for k in range(t.steps())],
            "t_lo": list(map(float, t.t_lo)), "t_hi": list(map(float, t.t_hi)), "diverged": bool(t.diverged),
            "failed_step": int(t.failed_step), "failure_reason": t.failure_reason}


def tube_from_json(j: dict) -> ReachTube:
    boxes = j["boxes"]
    if len(boxes) != len(j["t_lo"]) or len(boxes) != len(j["t_hi"]):
        raise ValueError("tube_from_json: length mismatch")
    num = lambda v: math.nan if v is None else float(v)  # noqa: E731  (null = a non-finite bound)
    n = len(boxes[0]["lo"]) if boxes else 0
    lo = np.array([[num(v) for v in b["lo"]] for b in boxes], dtype=np.float64).reshape(len(boxes), n)
    hi = np.array([[num(v) for v in b["hi"]] for b in boxes], dtype=np.float64).reshape(len(boxes), n)
    return ReachTube(lo, hi, np.array(j["t_lo"], np.float64), np.array(j["t_hi"], np.float64), bool(j["diverged"]),
                     int(j["failed_step"]), str(j["failure_reason"]))


def tube_to_csv(t: ReachTube, with_time_window: bool = True) -> str:
    out = ["step,t_lo,t_hi,dim,lo,hi\n" if with_time_window else "step,dim,lo,hi\n"]
    for k in range(t.steps()):
        for d in range(t.lo.shape[1]):
            row = str(k)
            if with_time_window:
                row += "," + fmt_g17(t.t_lo[k]) + "," + fmt_g17(t.t_hi[k])
            out.append(row + "," + str(d) + "," + fmt_g17(t.lo[k, d]) + "," + fmt_g17(t.hi[k, d]) + "\n")
    return "".join(out)


def tube_from_csv(csv: str) -> ReachTube:
    lines = csv.split("\n")
    if not lines or lines[0] == "" and len(lines) == 1:
        raise ValueError("tube_from_csv: empty input")
    header = lines[0]
    with_time = header == "step,t_lo,t_hi,dim,lo,hi"
    if not with_time and header != "step,dim,lo,hi":
        raise ValueError('tube_from_csv: unknown header "' + header + '"')
    boxes, t_lo, t_hi = [], [], []
    for line in lines[1:]:
        if not line:
            continue
        tok = line.split(",")
        need = 6 if with_time else 4
        if len(tok) < need:
            raise ValueError("tube_from_csv: short row")
        step = int(tok[0])
        tl = th = float(step)
        i = 1
        if with_time:
            tl, th = float(tok[1]), float(tok[2])
            i = 3
        dim, lo, hi = int(tok[i]), float(tok[i + 1]), float(tok[i + 2])
        if step == len(boxes):
            boxes.append([])
            t_lo.append(tl)
            t_hi.append(th)
        if step != len(boxes) - 1 or dim != len(boxes[-1]):
            raise ValueError("tube_from_csv: rows out of order")
        boxes[-1].append((lo, hi))
    n = len(boxes[0]) if boxes else 0
    lo = np.array([[p[0] for p in b] for b in boxes], np.float64).reshape(len(boxes), n)
    hi = np.array([[p[1] for p in b] for b in boxes], np.float64).reshape(len(boxes), n)
    return ReachTube(lo, hi, np.array(t_lo), np.array(t_hi))


# ---------------------------------------------------------------------------
@dataclass
class Manifest:  # io.hpp:165-195
    command: str = ""
    config: dict = field(default_factory=dict)
    seed: int = 0
    threads: int = 1
    version: str = VERSION

    def to_json(self) -> dict:
        return {"version": self.version, "command": self.command, "config": self.config, "seed": int(self.seed),
                "threads": int(self.threads)}

    @staticmethod
    def from_json(j: dict) -> "Manifest":
        return Manifest(j["command"], j["config"], int(j["seed"]), int(j["threads"]), j["version"])


def write_text_file(path: str, content: str) -> None:
    with open(path, "w", newline="") as f:
        f.write(content)


def read_text_file(path: str) -> str:
    with open(path, newline="") as f:
        return f.read()


def write_json_file(path: str, j: Any) -> None:
    write_text_file(path, json_dump(j) + "\n")


def read_json_file(path: str) -> Any:
    return json.loads(read_text_file(path))


# ---------------------------------------------------------------------------
# Scenarios (mpc.hpp:500-613).
_CON_NAME = {0: "halfspace-avoid", 1: "sphere-avoid", 2: "box-stay-in", 3: "max-volume"}


def constraint_to_json(c) -> dict:
    t = int(c.type)
    if t == 0:
        j = {"type": _CON_NAME[t], "a": list(map(float, c.a)), "b": float(c.b)}
    elif t == 1:
        j = {"type": _CON_NAME[t], "center": list(map(float, c.center)), "radius": float(c.radius)}
    elif t == 2:
        j = {"type": _CON_NAME[t], "lo": list(map(float, c.lo)), "hi": list(map(float, c.hi))}
    else:
        j = {"type": _CON_NAME[t], "vmax": float(c.vmax)}
    j["dims"] = [int(d) for d in (c.dims or [])]
    return j


def constraint_from_json(j: dict):
    from .mpc import Constraint
    t = j["type"]
    names = {v: k for k, v in _CON_NAME.items()}
    if t not in names:
        raise ValueError("unknown constraint type: " + str(t))
    c = Constraint(type=names[t], dims=[int(d) for d in j["dims"]])
    if t == "halfspace-avoid":
        c.a, c.b = np.array(j["a"], np.float64), float(j["b"])
    elif t == "sphere-avoid":
        c.center, c.radius = np.array(j["center"], np.float64), float(j["radius"])
    elif t == "box-stay-in":
        c.lo, c.hi = np.array(j["lo"], np.float64), np.array(j["hi"], np.float64)
    else:
        c.vmax = float(j["vmax"])
    return c


def scenario_to_json(prob, sampler, mpc) -> dict:
    return {"model": net_to_json(prob.sys.step), "n": prob.sys.n, "m": prob.sys.m,
            "x_goal": list(map(float, prob.x_goal)), "q_weights": list(map(float, prob.q_weights)),
            "r_weights": list(map(float, prob.r_weights)),
            "constraints": [constraint_to_json(c) for c in prob.constraints], "penalty": float(prob.penalty),
            "horizon": int(prob.horizon), "u_lo": list(map(float, prob.u_lo)), "u_hi": list(map(float, prob.u_hi)),
            "eps": float(prob.eps),
            "sampler": {"population": sampler.population, "elite_frac": float(sampler.elite_frac),
                        "iterations": sampler.iterations, "init_std": float(sampler.init_std),
                        "smoothing": float(sampler.smoothing), "refine_iters": sampler.refine_iters,
                        "seed": int(sampler.seed)},
            "mpc": {"replan_period": mpc.replan_period, "total_steps": mpc.total_steps,
                    "dist_action": float(mpc.dist_action), "dist_state": float(mpc.dist_state),
                    "goal_dims": list(mpc.goal_dims), "goal_radius": float(mpc.goal_radius), "seed": int(mpc.seed)}}


def scenario_from_json(j: dict):
    """-> (PlanProblem, SamplerConfig, MPCConfig), validated as the reference does (mpc.hpp:588-611)."""
    from .api import DTSystem
    from .mpc import MPCConfig, PlanProblem, SamplerConfig
    sys = DTSystem(net_from_json(j["model"]), int(j["n"]), int(j["m"]))
    prob = PlanProblem(sys, np.array(j["x_goal"], np.float64), np.array(j["q_weights"], np.float64),
                       np.array(j["r_weights"], np.float64), [constraint_from_json(c) for c in j["constraints"]],
                       horizon=int(j["horizon"]), u_lo=np.array(j["u_lo"], np.float64),
                       u_hi=np.array(j["u_hi"], np.float64), eps=float(j["eps"]))
    prob.penalty = float(j["penalty"])
    s = j["sampler"]
    sampler = SamplerConfig(int(s["population"]), float(s["elite_frac"]), int(s["iterations"]), float(s["init_std"]),
                            float(s["smoothing"]), int(s["refine_iters"]), int(s["seed"]))
    mj = j["mpc"]
    mpc = MPCConfig(int(mj["replan_period"]), int(mj["total_steps"]), float(mj["dist_action"]),
                    float(mj["dist_state"]), [int(d) for d in mj["goal_dims"]], float(mj["goal_radius"]),
                    int(mj["seed"]))
    prob.validate()
    if (sampler.population < 2 or not (0.0 < sampler.elite_frac <= 1.0) or sampler.iterations < 1
            or sampler.init_std <= 0.0 or not (0.0 <= sampler.smoothing < 1.0) or sampler.refine_iters < 0):
        raise ValueError("SamplerConfig: invalid configuration")
    if (mpc.replan_period < 1 or mpc.replan_period > prob.horizon or mpc.total_steps < 1 or mpc.dist_action < 0.0
            or mpc.dist_state < 0.0 or mpc.goal_radius <= 0.0):
        raise ValueError("MPCConfig: invalid configuration")
    return prob, sampler, mpc
