"""Reachability-aware MPC host API (mirrors mpc.hpp).

    Constraint (mpc.hpp:26-110), PlanProblem (115-142), SamplerConfig (220-234),
    plan_eval (158-202), plan_cem (258-368), with every candidate population
    evaluated on the device (C ABI reach_plan_eval_batch / reach_plan_cem_ex),
    and the top candidate's gradient refinement (refine_iters > 0, the
    reference default; gradient_refine, refine.hpp:347-398) driven by
    forward-dual gradients computed on the device (plan_objective_grad,
    grad_forward refine.hpp:186-207); MPCConfig / mpc_run (373-495), the
    receding-horizon loop around the device planner.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _abi as A
from ._native import Context, default_context
from .api import DTReachParams, DTSystem, TubeBatch


@dataclass
class Constraint:
    type: int = A.CON_MAX_VOLUME
    dims: List[int] = field(default_factory=list)
    a: Optional[np.ndarray] = None
    b: float = 0.0
    center: Optional[np.ndarray] = None
    radius: float = 0.0
    lo: Optional[np.ndarray] = None
    hi: Optional[np.ndarray] = None
    vmax: float = 0.0

    HALFSPACE_AVOID, SPHERE_AVOID, BOX_STAY_IN, MAX_VOLUME = 0, 1, 2, 3

    def validate(self, n: int):
        """Constraint::validate (mpc.hpp:89-111)."""
        for d in self.dims:
            if d < 0 or d >= n:
                raise ValueError("Constraint: dim out of range")
        k = len(self.dims) if self.dims else n
        size = lambda v: 0 if v is None else np.asarray(v).size  # noqa: E731
        if self.type == self.HALFSPACE_AVOID and size(self.a) != k:
            raise ValueError("Constraint: halfspace size")
        if self.type == self.SPHERE_AVOID and (size(self.center) != k or self.radius < 0.0):
            raise ValueError("Constraint: sphere parameters")
        if self.type == self.BOX_STAY_IN and (size(self.lo) != k or size(self.hi) != k):
            raise ValueError("Constraint: stay-in box size")
        if self.type == self.MAX_VOLUME and self.vmax < 0.0:
            raise ValueError("Constraint: volume budget")


@dataclass
class PlanProblem:
    sys: DTSystem
    x_goal: np.ndarray
    q_weights: np.ndarray
    r_weights: np.ndarray
    constraints: List[Constraint] = field(default_factory=list)
    penalty: float = 100.0
    diverged_margin: float = 1e3
    horizon: int = 5
    u_lo: Optional[np.ndarray] = None
    u_hi: Optional[np.ndarray] = None
    eps: float = 0.0
    dt_prm: DTReachParams = field(default_factory=DTReachParams)

    def validate(self):
        """PlanProblem::validate (mpc.hpp:129-141)."""
        self.sys.validate()
        n, m = self.sys.n, self.sys.m
        if self.horizon < 1:
            raise ValueError("PlanProblem: horizon < 1")
        sz = lambda v: 0 if v is None else np.asarray(v).size  # noqa: E731
        if sz(self.x_goal) != n or sz(self.q_weights) != n or sz(self.r_weights) != m:
            raise ValueError("PlanProblem: cost dimension mismatch")
        if sz(self.u_lo) != m or sz(self.u_hi) != m:
            raise ValueError("PlanProblem: action box dimension mismatch")
        for lo, hi in zip(np.asarray(self.u_lo if m else [], float), np.asarray(self.u_hi if m else [], float)):
            if not (lo <= hi) or not np.isfinite(lo) or not np.isfinite(hi):
                raise ValueError("PlanProblem: action box must be bounded")
        if self.eps < 0.0 or self.penalty < 0.0:
            raise ValueError("PlanProblem: negative weight")
        for c in self.constraints:
            c.validate(n)

    def c_struct(self):
        """(reach_plan_problem, keepalive)."""
        keep = []

        def arr(x, dt=np.float64):
            if x is None:
                return None
            a = np.ascontiguousarray(np.asarray(x, dtype=dt))
            keep.append(a)
            return a

        cons = (A.ConstraintC * max(1, len(self.constraints)))()
        for i, c in enumerate(self.constraints):
            dims = arr(c.dims, np.int32) if c.dims else None
            cons[i] = A.ConstraintC(int(c.type), len(c.dims), A.iptr(dims), A.dptr(arr(c.a)), float(c.b),
                                    A.dptr(arr(c.center)), float(c.radius), A.dptr(arr(c.lo)), A.dptr(arr(c.hi)),
                                    float(c.vmax))
        keep.append(cons)
        p = A.PlanProblemC(self.sys.n, self.sys.m, self.horizon, self.dt_prm.window, int(self.dt_prm.rebuild_from_box),
                           A.dptr(arr(self.x_goal)), A.dptr(arr(self.q_weights)),
                           A.dptr(arr(self.r_weights if self.sys.m else np.zeros(1))),
                           len(self.constraints), cons, float(self.penalty), float(self.diverged_margin),
                           float(self.eps), A.dptr(arr(self.u_lo if self.sys.m else np.zeros(1))),
                           A.dptr(arr(self.u_hi if self.sys.m else np.zeros(1))))
        return p, keep


@dataclass
class SamplerConfig:
    population: int = 256
    elite_frac: float = 0.1
    iterations: int = 5
    init_std: float = 0.3
    smoothing: float = 0.5
    refine_iters: int = 5
    seed: int = 0

    def c_struct(self):
        return A.SamplerConfigC(self.population, self.elite_frac, self.iterations, self.init_std, self.smoothing,
                                self.refine_iters, self.seed)


@dataclass
class PlanBatch:
    objective: np.ndarray
    diverged: np.ndarray
    tubes: Optional[TubeBatch] = None


def plan_eval_batch(prob: PlanProblem, x0, actions: np.ndarray, with_tubes: bool = False,
                    ctx: Optional[Context] = None) -> PlanBatch:
    """plan_eval (mpc.hpp:158-202) for actions [B][H][m] from one x0."""
    prob.sys.validate()
    ctx = ctx or default_context()
    x0 = np.ascontiguousarray(x0, dtype=np.float64)
    acts = np.ascontiguousarray(actions, dtype=np.float64)
    B = acts.shape[0]
    if acts.shape[1:] != (prob.horizon, prob.sys.m):
        raise ValueError("plan_eval: action count != horizon")
    obj = np.zeros(B)
    div = np.zeros(B, np.int32)
    tubes = None
    to_p = None
    if with_tubes:
        H, n = prob.horizon, prob.sys.n
        tubes = TubeBatch(np.full((B, H + 1, n), np.nan), np.full((B, H + 1, n), np.nan), np.zeros(B, np.int32),
                          np.zeros(B, np.int32), np.zeros(B, np.int32))
        to = A.TubeOut(A.dptr(tubes.lo), A.dptr(tubes.hi), A.iptr(tubes.n_boxes), A.iptr(tubes.failed_step),
                       A.iptr(tubes.status))
        to_p = C.byref(to)
    p, keep = prob.c_struct()
    net = ctx.upload(prob.sys.step)
    ctx.check(ctx._lib.reach_plan_eval_batch(ctx.handle, net, C.byref(p), A.dptr(x0), B, A.dptr(acts), A.dptr(obj),
                                             A.iptr(div), to_p, 0), "plan_eval")
    return PlanBatch(obj, div.astype(bool), tubes)


def plan_eval(prob: PlanProblem, x0, actions, ctx: Optional[Context] = None):
    r = plan_eval_batch(prob, x0, np.asarray(actions, np.float64)[None], with_tubes=True, ctx=ctx)
    return r.objective[0], r.diverged[0], r.tubes.tube(0)


@dataclass
class PlanResult:
    actions: np.ndarray       # [H][m]
    objective: float
    best_history: np.ndarray  # [iterations]
    best_effort: bool
    tube: object = None
    refined: bool = False  # gradient refinement made progress (mpc.hpp:241)


def plan_objective_grad(prob: PlanProblem, x0, actions, ctx: Optional[Context] = None):
    """grad_forward (refine.hpp:186-207) of plan_objective over the flat action sequence
    [H][m] -> (gradient [H][m], objective); one reach::Dual pass per direction on the device."""
    prob.sys.validate()
    ctx = ctx or default_context()
    x0 = np.ascontiguousarray(x0, dtype=np.float64)
    acts = np.ascontiguousarray(np.asarray(actions, np.float64).reshape(prob.horizon, prob.sys.m))
    g = np.zeros_like(acts)
    obj = np.zeros(1)
    p, keep = prob.c_struct()
    net = ctx.upload(prob.sys.step)
    ctx.check(ctx._lib.reach_plan_objective_grad(ctx.handle, net, C.byref(p), A.dptr(x0), A.dptr(acts), A.dptr(g),
                                                 A.dptr(obj)), "grad_forward")
    return g, float(obj[0])


def plan_refine(prob: PlanProblem, x0, actions, best_objective: float, refine_iters: int = 5,
                ctx: Optional[Context] = None):
    """plan_cem's refinement step (mpc.hpp:337-361) alone -> (actions, refined): gradient_refine of the
    plan objective from `actions` (objective best_objective) with forward-dual gradients on the device."""
    prob.sys.validate()
    ctx = ctx or default_context()
    x0 = np.ascontiguousarray(x0, dtype=np.float64)
    acts = np.ascontiguousarray(np.asarray(actions, np.float64).reshape(prob.horizon, prob.sys.m)).copy()
    rf = np.zeros(1, np.int32)
    p, keep = prob.c_struct()
    net = ctx.upload(prob.sys.step)
    ctx.check(ctx._lib.reach_plan_refine(ctx.handle, net, C.byref(p), A.dptr(x0), int(refine_iters),
                                         float(best_objective), A.dptr(acts), A.iptr(rf)), "plan_refine")
    return acts, bool(rf[0])


def plan_cem(prob: PlanProblem, cfg: SamplerConfig, x0, ctx: Optional[Context] = None) -> PlanResult:
    """plan_cem (mpc.hpp:258-368), including the top-candidate gradient refinement."""
    prob.sys.validate()
    ctx = ctx or default_context()
    x0 = np.ascontiguousarray(x0, dtype=np.float64)
    H, m, n = prob.horizon, prob.sys.m, prob.sys.n
    best = np.zeros((H, m))
    obj = np.zeros(1)
    hist = np.zeros(cfg.iterations)
    be = np.zeros(1, np.int32)
    tb = TubeBatch(np.full((1, H + 1, n), np.nan), np.full((1, H + 1, n), np.nan), np.zeros(1, np.int32),
                   np.zeros(1, np.int32), np.zeros(1, np.int32))
    to = A.TubeOut(A.dptr(tb.lo), A.dptr(tb.hi), A.iptr(tb.n_boxes), A.iptr(tb.failed_step), A.iptr(tb.status))
    p, keep = prob.c_struct()
    c = cfg.c_struct()
    net = ctx.upload(prob.sys.step)
    refined = np.zeros(1, np.int32)
    ctx.check(ctx._lib.reach_plan_cem_ex(ctx.handle, net, C.byref(p), C.byref(c), A.dptr(x0), A.dptr(best),
                                         A.dptr(obj), A.dptr(hist), A.iptr(be), A.iptr(refined), C.byref(to)),
              "plan_cem")
    return PlanResult(best, float(obj[0]), hist, bool(be[0]), tb.tube(0), bool(refined[0]))


class CEM:
    """plan_cem's loop in pieces (sample -> evaluate a shard -> gather -> update)
    for multi-GPU drivers; identical sampling stream on every rank."""

    def __init__(self, prob: PlanProblem, cfg: SamplerConfig):
        from ._native import lib
        self._lib = lib()
        self.prob, self.cfg = prob, cfg
        self._p, self._keep = prob.c_struct()
        self._c = cfg.c_struct()
        h = C.c_void_p()
        rc = self._lib.reach_cem_create(C.byref(self._p), C.byref(self._c), C.byref(h))
        if rc != 0:
            raise ValueError(f"reach_cem_create failed ({rc})")
        self.h = h

    def sample(self) -> np.ndarray:
        out = np.zeros((self.cfg.population, self.prob.horizon, self.prob.sys.m))
        assert self._lib.reach_cem_sample(self.h, A.dptr(out)) == 0
        return out

    def update(self, scores: np.ndarray, ok: np.ndarray):
        s = np.ascontiguousarray(scores, np.float64)
        o = np.ascontiguousarray(ok, np.int32)
        assert self._lib.reach_cem_update(self.h, A.dptr(s), A.iptr(o)) == 0

    def result(self):
        best = np.zeros((self.prob.horizon, self.prob.sys.m))
        obj = np.zeros(1)
        be = np.zeros(1, np.int32)
        hist = np.zeros(self.cfg.iterations)
        assert self._lib.reach_cem_result(self.h, A.dptr(best), A.dptr(obj), A.iptr(be), A.dptr(hist)) == 0
        return best, float(obj[0]), bool(be[0]), hist

    def __del__(self):
        try:
            self._lib.reach_cem_destroy(self.h)
        except Exception:
            pass


# ---------------------------------------------------------------------------
@dataclass
class MPCConfig:  # mpc.hpp:373-387
    replan_period: int = 3
    total_steps: int = 30
    dist_action: float = 0.0
    dist_state: float = 0.0
    goal_dims: List[int] = field(default_factory=list)
    goal_radius: float = 0.1
    seed: int = 0


@dataclass
class MPCLogRow:  # mpc.hpp:389-396
    step: int
    state: np.ndarray
    action: np.ndarray
    objective: float
    tube_volume: float
    g_margin: float


def _g17(v: float) -> str:
    """fmt_g17 (io.hpp:23-27): printf("%.17g")."""
    return "%.17g" % v


@dataclass
class MPCResult:  # mpc.hpp:398-419
    success: bool
    violated: bool
    steps_used: int
    final_state: np.ndarray
    log: List[MPCLogRow]

    def log_to_csv(self) -> str:
        out = "step,objective,tube_volume,g_margin,state,action\n"
        for r in self.log:
            out += (f"{r.step},{_g17(r.objective)},{_g17(r.tube_volume)},{_g17(r.g_margin)},"
                    + ";".join(_g17(v) for v in r.state) + "," + ";".join(_g17(v) for v in r.action) + "\n")
        return out


def mpc_run(prob: PlanProblem, sampler: SamplerConfig, cfg: MPCConfig, x0, sim=None,
            ctx: Optional[Context] = None) -> MPCResult:
    """mpc_run (mpc.hpp:425-495).  sim(x, u) -> x_next is the true simulator; None = the planning model's
    forward on the device (the reference CLI's simulator, reach_cli.cpp:445-449)."""
    prob.sys.validate()
    ctx = ctx or default_context()
    n, m = prob.sys.n, prob.sys.m
    x0 = np.ascontiguousarray(x0, dtype=np.float64)
    if x0.shape != (n,):
        raise ValueError("mpc_run: x0 dimension mismatch")
    T = int(cfg.total_steps)
    rows = max(T, 1)
    lg_step = np.zeros(rows, np.int32)
    lg_state = np.zeros((rows, n))
    lg_action = np.zeros((rows, max(m, 1)))
    lg_obj, lg_vol, lg_mar = np.zeros(rows), np.zeros(rows), np.zeros(rows)
    log = A.MPCLogC(A.iptr(lg_step), A.dptr(lg_state), A.dptr(lg_action), A.dptr(lg_obj), A.dptr(lg_vol),
                    A.dptr(lg_mar))
    gd = np.ascontiguousarray(cfg.goal_dims, dtype=np.int32) if cfg.goal_dims else np.zeros(1, np.int32)
    mc = A.MPCConfigC(cfg.replan_period, cfg.total_steps, cfg.dist_action, cfg.dist_state, len(cfg.goal_dims),
                      A.iptr(gd), cfg.goal_radius, cfg.seed)
    err = []
    if sim is None:
        cb = A.SIM_FN()
    else:
        def _cb(user, xp, up, outp):
            try:
                xs = np.ctypeslib.as_array(xp, shape=(n,)).copy()
                us = np.ctypeslib.as_array(up, shape=(m,)).copy() if m else np.zeros(0)
                out = np.asarray(sim(xs, us), dtype=np.float64).reshape(n)
                np.ctypeslib.as_array(outp, shape=(n,))[:] = out
                return 0
            except Exception as e:  # surfaced after the call
                err.append(e)
                return 1
        cb = A.SIM_FN(_cb)
    succ, viol, used, nrows = (np.zeros(1, np.int32) for _ in range(4))
    fin = np.zeros(n)
    p, keep = prob.c_struct()
    sc = sampler.c_struct()
    net = ctx.upload(prob.sys.step)
    rc = ctx._lib.reach_mpc_run(ctx.handle, net, C.byref(p), C.byref(sc), C.byref(mc), cb, None, A.dptr(x0),
                                A.iptr(succ), A.iptr(viol), A.iptr(used), A.dptr(fin), C.byref(log), A.iptr(nrows))
    if err:
        raise err[0]
    ctx.check(rc, "mpc_run")
    k = int(nrows[0])
    rows_out = [MPCLogRow(int(lg_step[i]), lg_state[i].copy(), lg_action[i, :m].copy(), float(lg_obj[i]),
                          float(lg_vol[i]), float(lg_mar[i])) for i in range(k)]
    return MPCResult(bool(succ[0]), bool(viol[0]), int(used[0]), fin, rows_out)
