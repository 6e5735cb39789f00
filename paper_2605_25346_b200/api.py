"""Reference-facing host API (mirrors /root/reference/proj/include/reach/).

Same names, argument meaning and error behaviour as the reference's C++
templates for the DT reachability path:

    MLPNet / Layer / Act            neural.hpp:18-88
    affine_net                      neural.hpp:90-95
    DTSystem, DTReachParams         dt_reach.hpp:17-36
    dt_reach, dt_reach_batch        dt_reach.hpp:40-125
    SplitPlan, split_box            refine.hpp:25-115
    reach_with_splitting            refine.hpp:121-160  (engine = dt_reach)
    ReachTube, tube_volume          tube.hpp:12-46
    box_from_center, box_volume_proxy  interval.hpp:224-258
    QuadrotorParams                 systems.hpp:16-20
    FlowpipeParams                  flowpipe_ct.hpp:35-50
    ClosedLoopSpec, cl_reach        closed_loop.hpp:16-182  (plant = quadrotor_ode, fields.hpp:96-128)
    zero_field, diag_linear_field,  fields.hpp:51-92 (the analytic VectorFields the device runs)
    rotation_field, quadrotor_field
    ct_reach                        flowpipe_ct.hpp:428-458
    GradTarget, GradMethod,         refine.hpp:165-311 (forward-dual passes on the device)
    Gradient, grad_tube_volume

Every compute call runs the CUDA kernels through the C ABI
(include/reach_b200.h); there is no CPU path.  Shape errors raise
ValueError where the reference throws std::invalid_argument.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import enum
import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _abi as A
from ._native import Context, default_context


class Act(enum.IntEnum):
    Relu = A.ACT_RELU
    Tanh = A.ACT_TANH
    Identity = A.ACT_IDENTITY


@dataclass
class Layer:
    w: np.ndarray  # out x in
    b: np.ndarray
    act: Act = Act.Identity


@dataclass(eq=False)
class MLPNet:
    layers: List[Layer] = field(default_factory=list)

    def input_dim(self) -> int:
        return int(self.layers[0].w.shape[1])

    def output_dim(self) -> int:
        return int(self.layers[-1].w.shape[0])

    def validate(self):
        """MLPNet::validate (neural.hpp:49-56)."""
        if not self.layers:
            raise ValueError("MLPNet: empty")
        for l in range(len(self.layers) - 1):
            if self.layers[l + 1].w.shape[1] != self.layers[l].w.shape[0]:
                raise ValueError("MLPNet: layer shapes do not chain")
        if self.layers[-1].act != Act.Identity:
            raise ValueError("MLPNet: final activation must be identity")

    def forward(self, x: np.ndarray) -> np.ndarray:
        """MLPNet::forward (neural.hpp:58-76) -- host-side rollout for checks; x is [in] or [in][S]."""
        h = np.asarray(x, dtype=np.float64)
        for L in self.layers:
            h = L.w @ h + (L.b[:, None] if h.ndim == 2 else L.b)
            if L.act == Act.Relu:
                h = np.where(h < 0.0, 0.0, h)
            elif L.act == Act.Tanh:
                h = np.tanh(h)
        return h

    def params(self) -> np.ndarray:
        """net_params order (neural.hpp:133-140): per layer W row-major then b."""
        return np.concatenate([np.concatenate([L.w.ravel(), L.b.ravel()]) for L in self.layers]).astype(np.float64)

    def dims(self) -> np.ndarray:
        return np.array([self.layers[0].w.shape[1]] + [L.w.shape[0] for L in self.layers], dtype=np.int32)

    def acts(self) -> np.ndarray:
        return np.array([int(L.act) for L in self.layers], dtype=np.int32)

    def desc(self):
        """(reach_net_desc, keepalive) for the C ABI."""
        self.validate()
        dims, acts, params = self.dims(), self.acts(), np.ascontiguousarray(self.params())
        d = A.NetDesc(len(self.layers), A.iptr(dims), A.iptr(acts), A.dptr(params))
        return d, (dims, acts, params)


def affine_net(m: np.ndarray, d: np.ndarray) -> MLPNet:
    return MLPNet([Layer(np.asarray(m, np.float64), np.asarray(d, np.float64), Act.Identity)])


@dataclass
class DTSystem:
    step: MLPNet
    n: int
    m: int = 0

    def validate(self):
        """DTSystem::validate (dt_reach.hpp:23-28)."""
        self.step.validate()
        if self.n <= 0 or self.m < 0:
            raise ValueError("DTSystem: invalid dimensions")
        if self.step.input_dim() != self.n + self.m or self.step.output_dim() != self.n:
            raise ValueError("DTSystem: one-step map shape mismatch")


@dataclass
class DTReachParams:
    window: int = 4
    rebuild_from_box: bool = False


@dataclass
class ReachTube:
    """ReachTube<double> (tube.hpp:12-35); box k = (lo[k], hi[k])."""
    lo: np.ndarray
    hi: np.ndarray
    t_lo: np.ndarray
    t_hi: np.ndarray
    diverged: bool = False
    failed_step: int = -1
    failure_reason: str = ""

    def steps(self) -> int:
        return int(self.lo.shape[0])

    def box_diverged(self, k: int) -> bool:
        """IntervalBox::diverged after check_divergence (interval.hpp:215-218)."""
        return not (np.all(np.isfinite(self.lo[k])) and np.all(np.isfinite(self.hi[k])))


def box_volume_proxy(lo: np.ndarray, hi: np.ndarray) -> float:
    """interval.hpp:252-258: width sum, +inf for a non-finite box."""
    if not (np.all(np.isfinite(lo)) and np.all(np.isfinite(hi))):
        return math.inf
    acc = 0.0
    for a, b in zip(lo, hi):
        acc += b - a
    return acc


def tube_volume(t: ReachTube) -> float:
    """tube.hpp:40-46."""
    if t.diverged:
        return math.inf
    acc = 0.0
    for k in range(t.steps()):
        acc += box_volume_proxy(t.lo[k], t.hi[k])
    return acc


def box_from_center(center, radius):
    """interval.hpp:224-240 -> (lo, hi)."""
    c = np.asarray(center, dtype=np.float64)
    r = np.broadcast_to(np.asarray(radius, dtype=np.float64), c.shape)
    if np.any(r < 0.0):
        raise ValueError("box_from_center: negative radius")
    return c - r, c + r


# ---------------------------------------------------------------------------
@dataclass
class TubeBatch:
    """Batch output of dt_reach_batch / cl_reach in array form (the device layout)."""
    lo: np.ndarray  # [B][H+1][n]
    hi: np.ndarray
    n_boxes: np.ndarray
    failed_step: np.ndarray
    status: np.ndarray
    h: float = 0.0  # > 0: continuous-time tube, box k >= 1 covers [(k-1)h, kh] (closed_loop.hpp:172)

    def tube(self, b: int) -> ReachTube:
        k = int(self.n_boxes[b])
        st = int(self.status[b])
        t_lo, t_hi = _tube_times(k, self.h)
        return ReachTube(self.lo[b, :k].copy(), self.hi[b, :k].copy(), t_lo, t_hi, diverged=st != A.TUBE_OK,
                         failed_step=int(self.failed_step[b]), failure_reason=A.TUBE_REASON.get(st, "error"))

    def tubes(self) -> List[ReachTube]:
        return [self.tube(b) for b in range(self.lo.shape[0])]


def _tube_times(k: int, h: float):
    if h <= 0.0:
        t = np.arange(k, dtype=np.float64)
        return t, t.copy()
    j = np.arange(k, dtype=np.float64)
    return np.where(j > 0, (j - 1) * h, 0.0), j * h


def _actions_array(seqs, B, H, m) -> np.ndarray:
    a = np.zeros((B, H, m), dtype=np.float64)
    for b, seq in enumerate(seqs):
        if len(seq) != H:
            raise ValueError("dt_reach_batch: ragged action sequences")
        for k, u in enumerate(seq):
            u = np.asarray(u, dtype=np.float64).ravel()
            if u.size != m:
                raise ValueError("dt_reach: action dimension mismatch")
            a[b, k] = u
    return a


def dt_reach_batch_arrays(sys: DTSystem, x0_lo: np.ndarray, x0_hi: np.ndarray, actions: np.ndarray,
                          prm: DTReachParams = DTReachParams(), ctx: Optional[Context] = None,
                          actions_shared: bool = False, precision: str = "exact") -> TubeBatch:
    """dt_reach_batch (dt_reach.hpp:108-125) on arrays: x0 [B][n], actions [B][H][m] (or [H][m] shared).
    precision "tc": the CROWN contractions on the int8 tensor cores (A.REACH_PREC_TC)."""
    pflag = A.prec_flag(precision)
    sys.validate()
    ctx = ctx or default_context()
    x0_lo = np.ascontiguousarray(x0_lo, dtype=np.float64)
    x0_hi = np.ascontiguousarray(x0_hi, dtype=np.float64)
    B = x0_lo.shape[0]
    if x0_lo.shape != (B, sys.n) or x0_hi.shape != (B, sys.n):
        raise ValueError("dt_reach: X0 dimension mismatch")
    actions = np.ascontiguousarray(actions, dtype=np.float64)
    H = actions.shape[0] if actions_shared else actions.shape[1]
    if actions.shape[-1] != sys.m and not (sys.m == 0 and actions.size == 0):
        raise ValueError("dt_reach: action dimension mismatch")
    out = TubeBatch(np.full((B, H + 1, sys.n), np.nan), np.full((B, H + 1, sys.n), np.nan),
                    np.zeros(B, np.int32), np.zeros(B, np.int32), np.zeros(B, np.int32))
    args = A.DTArgs(B, H, sys.n, sys.m, prm.window, int(prm.rebuild_from_box), A.dptr(x0_lo), A.dptr(x0_hi),
                    A.dptr(actions if actions.size else np.zeros(1)), int(actions_shared))
    to = A.TubeOut(A.dptr(out.lo), A.dptr(out.hi), A.iptr(out.n_boxes), A.iptr(out.failed_step),
                   A.iptr(out.status))
    net = ctx.upload(sys.step)
    ctx.check(ctx._lib.reach_dt_batch(ctx.handle, net, C.byref(args), C.byref(to), pflag), "dt_reach_batch")
    return out


def dt_interval_baseline_batch_arrays(sys: DTSystem, x0_lo: np.ndarray, x0_hi: np.ndarray, actions: np.ndarray,
                                      ctx: Optional[Context] = None, actions_shared: bool = False) -> TubeBatch:
    """dt_interval_baseline (dt_reach.hpp:129-149) on arrays, one tube per row: the naive interval tube."""
    sys.validate()
    ctx = ctx or default_context()
    x0_lo = np.ascontiguousarray(x0_lo, dtype=np.float64)
    x0_hi = np.ascontiguousarray(x0_hi, dtype=np.float64)
    B = x0_lo.shape[0]
    if x0_lo.shape != (B, sys.n) or x0_hi.shape != (B, sys.n):
        raise ValueError("dt_reach: X0 dimension mismatch")
    actions = np.ascontiguousarray(actions, dtype=np.float64)
    H = actions.shape[0] if actions_shared else actions.shape[1]
    if actions.shape[-1] != sys.m and not (sys.m == 0 and actions.size == 0):
        raise ValueError("dt_reach: action dimension mismatch")
    out = TubeBatch(np.full((B, H + 1, sys.n), np.nan), np.full((B, H + 1, sys.n), np.nan),
                    np.zeros(B, np.int32), np.zeros(B, np.int32), np.zeros(B, np.int32))
    args = A.DTArgs(B, H, sys.n, sys.m, 0, 0, A.dptr(x0_lo), A.dptr(x0_hi),
                    A.dptr(actions if actions.size else np.zeros(1)), int(actions_shared))
    to = A.TubeOut(A.dptr(out.lo), A.dptr(out.hi), A.iptr(out.n_boxes), A.iptr(out.failed_step),
                   A.iptr(out.status))
    net = ctx.upload(sys.step)
    ctx.check(ctx._lib.reach_dt_interval_baseline_batch(ctx.handle, net, C.byref(args), C.byref(to)),
              "dt_interval_baseline")
    return out


def dt_interval_baseline(sys: DTSystem, x0, actions: Sequence, ctx: Optional[Context] = None) -> ReachTube:
    """dt_interval_baseline (dt_reach.hpp:129-149): x0 = (lo, hi)."""
    H = len(actions)
    acts = _actions_array([actions], 1, H, sys.m)
    lo = np.asarray(x0[0], np.float64).reshape(1, -1)
    hi = np.asarray(x0[1], np.float64).reshape(1, -1)
    return dt_interval_baseline_batch_arrays(sys, lo, hi, acts, ctx).tube(0)


def dt_reach_batch(sys: DTSystem, x0s: Sequence, action_seqs: Sequence, prm: DTReachParams = DTReachParams(),
                   ctx: Optional[Context] = None, precision: str = "exact") -> List[ReachTube]:
    """dt_reach_batch (dt_reach.hpp:108-125): x0s = [(lo, hi), ...], action_seqs = [[u_0..u_{H-1}], ...]."""
    if len(x0s) != len(action_seqs):
        raise ValueError("dt_reach_batch: batch size mismatch")
    if not x0s:
        return []
    B = len(x0s)
    lo = np.array([np.asarray(b[0], np.float64) for b in x0s])
    hi = np.array([np.asarray(b[1], np.float64) for b in x0s])
    H = len(action_seqs[0])
    acts = _actions_array(action_seqs, B, H, sys.m)
    return dt_reach_batch_arrays(sys, lo, hi, acts, prm, ctx, precision=precision).tubes()


def dt_reach(sys: DTSystem, x0, actions: Sequence, prm: DTReachParams = DTReachParams(),
             ctx: Optional[Context] = None, precision: str = "exact") -> ReachTube:
    """dt_reach (dt_reach.hpp:40-104): x0 = (lo, hi)."""
    return dt_reach_batch(sys, [x0], [actions], prm, ctx, precision)[0]


# ---------------------------------------------------------------------------
class GradTarget(enum.IntEnum):  # refine.hpp:240
    x0_center = 0
    actions = 1
    weights = 2


class GradMethod(enum.IntEnum):  # refine.hpp:165
    forward_dual = 0
    finite_difference = 1


@dataclass
class Gradient:  # refine.hpp:171-178
    g: np.ndarray
    method: GradMethod = GradMethod.forward_dual
    subgradient: bool = False
    volume: float = 0.0  # the primal tube volume the gradient was taken at


def grad_tube_volume(sys: DTSystem, x0, actions: Sequence, target: GradTarget,
                     method: GradMethod = GradMethod.forward_dual, prm: DTReachParams = DTReachParams(),
                     ctx: Optional[Context] = None, param_range: Optional[tuple] = None) -> Gradient:
    """grad_tube_volume (refine.hpp:263-311): d tube_volume(dt_reach(...)) / d target, x0 = (lo, hi).
    Parameter layouts: x0_center [n]; actions [H*m] step-major; weights in net_params order
    (neural.hpp:133-140).  Every pass (one per parameter, two per parameter for finite differences)
    runs on the device in one launch.  Raises ValueError where the reference throws."""
    sys.validate()
    ctx = ctx or default_context()
    lo = np.ascontiguousarray(x0[0], dtype=np.float64).reshape(-1)
    hi = np.ascontiguousarray(x0[1], dtype=np.float64).reshape(-1)
    if lo.size != sys.n or hi.size != sys.n:
        raise ValueError("dt_reach: X0 dimension mismatch")
    H = len(actions)
    acts = _actions_array([actions], 1, H, sys.m).reshape(-1)
    target, method = GradTarget(target), GradMethod(method)
    full = {GradTarget.x0_center: sys.n, GradTarget.actions: H * sys.m,
            GradTarget.weights: int(sys.step.params().size)}[target]
    begin, end = (0, full) if param_range is None else (int(param_range[0]), int(param_range[1]))
    dim = max(end - begin, 0)
    g = np.zeros(max(dim, 1))
    sub = np.zeros(1, np.int32)
    vol = np.zeros(1)
    args = A.DTArgs(1, H, sys.n, sys.m, prm.window, int(prm.rebuild_from_box), A.dptr(lo), A.dptr(hi),
                    A.dptr(acts if acts.size else np.zeros(1)), 0)
    net = ctx.upload(sys.step)
    ctx.check(ctx._lib.reach_grad_tube_volume_range(ctx.handle, net, C.byref(args), int(target), int(method),
                                                    begin, end, A.dptr(g), A.iptr(sub), A.dptr(vol)),
              "grad_tube_volume")
    return Gradient(g[:dim].copy(), method, bool(sub[0]), float(vol[0]))


@dataclass
class RefineResult:  # refine.hpp:333-340
    x: np.ndarray
    initial_objective: float
    objective: float
    progressed: bool
    subgradient: bool
    accepted_steps: int


def refine_tube_volume(sys: DTSystem, center, radius, actions: Sequence, target: GradTarget, lo, hi,
                       iters: int = 20, x=None, prm: DTReachParams = DTReachParams(),
                       ctx: Optional[Context] = None) -> RefineResult:
    """gradient_refine (refine.hpp:354-398) of tube_volume(dt_reach(box_from_center(c, radius), actions)) over
    the X0 centre or the flat action sequence within [lo, hi] (the reference CLI's `refine`,
    reach_cli.cpp:293-341).  x = the start point (default: the centre / the actions)."""
    sys.validate()
    ctx = ctx or default_context()
    target = GradTarget(target)
    if target == GradTarget.weights:
        raise ValueError("refine: target must be the X0 centre or the actions")
    c = np.ascontiguousarray(center, dtype=np.float64).reshape(-1)
    r = np.ascontiguousarray(np.broadcast_to(np.asarray(radius, np.float64), c.shape))
    if c.size != sys.n:
        raise ValueError("dt_reach: X0 dimension mismatch")
    H = len(actions)
    acts = _actions_array([actions], 1, H, sys.m).reshape(-1)
    d = sys.n if target == GradTarget.x0_center else H * sys.m
    xv = np.ascontiguousarray(c if x is None and target == GradTarget.x0_center else
                              (acts if x is None else x), dtype=np.float64).reshape(-1).copy()
    lo = np.ascontiguousarray(lo, dtype=np.float64).reshape(-1)
    hi = np.ascontiguousarray(hi, dtype=np.float64).reshape(-1)
    if xv.size != d or lo.size != d or hi.size != d:
        raise ValueError("gradient_refine: bound dimension mismatch")
    f0, f1 = np.zeros(1), np.zeros(1)
    pr, sb, ac = (np.zeros(1, np.int32) for _ in range(3))
    args = A.DTArgs(1, H, sys.n, sys.m, prm.window, int(prm.rebuild_from_box), A.dptr(c), A.dptr(c),
                    A.dptr(acts if acts.size else np.zeros(1)), 0)
    net = ctx.upload(sys.step)
    ctx.check(ctx._lib.reach_refine_tube_volume(ctx.handle, net, C.byref(args), A.dptr(c), A.dptr(r), int(target),
                                                A.dptr(lo), A.dptr(hi), int(iters), A.dptr(xv if d else np.zeros(1)),
                                                A.dptr(f0), A.dptr(f1), A.iptr(pr), A.iptr(sb), A.iptr(ac)),
              "gradient_refine")
    return RefineResult(xv[:d], float(f0[0]), float(f1[0]), bool(pr[0]), bool(sb[0]), int(ac[0]))


@dataclass
class Episode:  # training.hpp:28-45
    states: Sequence   # [T+1][n]
    actions: Sequence  # [T][m]
    y_ref: Sequence = ()

    def length(self) -> int:
        return len(self.actions)


def _loss_inputs(model: MLPNet, batch: Sequence[Episode], t_h: int):
    if not batch or t_h < 1:
        raise ValueError("reach_loss: bad batch/horizon")
    n = len(batch[0].states[0])
    m = len(batch[0].actions[0])
    x0 = np.zeros((len(batch), n))
    acts = np.zeros((len(batch), t_h, m))
    for e, ep in enumerate(batch):
        if ep.length() < t_h:
            raise ValueError("reach_loss: episode shorter than T_h")
        x0[e] = np.asarray(ep.states[0], np.float64)
        acts[e] = np.asarray(ep.actions[:t_h], np.float64).reshape(t_h, m)
    return DTSystem(model, n, m), x0, acts


def reach_loss(model: MLPNet, batch: Sequence[Episode], eps: float, t_h: int, cap: float,
               prm: DTReachParams = DTReachParams(), with_grad: bool = False, ctx: Optional[Context] = None):
    """reach_loss (training.hpp:99-126) on the device -> (loss, diverged_count), or with_grad ->
    (loss, gradient over net_params (neural.hpp:133-140), diverged_count): grad_forward's Dual passes,
    one CTA per (parameter, episode), one launch."""
    sys_, x0, acts = _loss_inputs(model, batch, t_h)
    sys_.validate()
    ctx = ctx or default_context()
    M = x0.shape[0]
    loss = np.zeros(1)
    dc = np.zeros(1, np.int32)
    g = np.zeros(model.params().size) if with_grad else None
    args = A.DTArgs(M, t_h, sys_.n, sys_.m, prm.window, int(prm.rebuild_from_box), A.dptr(x0), A.dptr(x0),
                    A.dptr(acts if acts.size else np.zeros(1)), 0)
    net = ctx.upload(model)
    ctx.check(ctx._lib.reach_reach_loss(ctx.handle, net, C.byref(args), M, float(eps), float(cap), A.dptr(loss),
                                        A.dptr(g) if with_grad else None, A.iptr(dc)), "reach_loss")
    return (float(loss[0]), g, int(dc[0])) if with_grad else (float(loss[0]), int(dc[0]))


def net_with_params(shape: MLPNet, params) -> MLPNet:
    """net_with_params (neural.hpp:142-152): the shape's layers with values from a net_params vector."""
    params = np.asarray(params, np.float64)
    layers, k = [], 0
    for L in shape.layers:
        r, c = L.w.shape
        w = params[k:k + r * c].reshape(r, c).copy()
        k += r * c
        b = params[k:k + r].copy()
        k += r
        layers.append(Layer(w, b, L.act))
    if k != params.size:
        raise ValueError("net_with_params: size mismatch")
    return MLPNet(layers)


def horizon_weights(t_h: int) -> np.ndarray:
    """horizon_weights (training.hpp:48-53)."""
    return np.array([1.0 + (t + 1) / t_h for t in range(t_h)], np.float64)


def _episode_set(batch: Sequence[Episode]):
    """(EpisodeSetC, keepalive) of episodes of one length (states [E][T+1][n], actions [E][T][m])."""
    if not batch:
        raise ValueError("empty episode batch")
    T = batch[0].length()
    if any(ep.length() != T for ep in batch):
        raise ValueError("episodes of one batch must share a length")
    n, m = len(batch[0].states[0]), len(batch[0].actions[0]) if T else 0
    st = np.ascontiguousarray(np.array([np.asarray(ep.states, np.float64).reshape(T + 1, n) for ep in batch]))
    ac = np.ascontiguousarray(np.array([np.asarray(ep.actions, np.float64).reshape(T, m) for ep in batch]))
    r = len(batch[0].y_ref[0]) if len(batch[0].y_ref) else 0
    if r and any(len(ep.y_ref) != T for ep in batch):
        raise ValueError("Episode: reference length mismatch")
    yr = np.ascontiguousarray(np.array([np.asarray(ep.y_ref, np.float64).reshape(T, r) for ep in batch])) if r \
        else np.zeros(1)
    es = A.EpisodeSetC(len(batch), T, n, m, A.dptr(st), A.dptr(ac if ac.size else np.zeros(1)), r,
                       A.dptr(yr) if r else None)
    return es, (st, ac, yr)


def pred_loss(model: MLPNet, batch: Sequence[Episode], t_h: int, weights, with_grad: bool = False,
              ctx: Optional[Context] = None):
    """pred_loss (training.hpp:60-83) on the device -> loss, or with_grad -> (loss, gradient over net_params):
    grad_forward's Dual rollouts, one CTA per (parameter, episode), one launch."""
    weights = np.ascontiguousarray(weights, np.float64)
    if not batch or t_h < 1 or weights.size != t_h:
        raise ValueError("pred_loss: bad batch/horizon/weights")
    ctx = ctx or default_context()
    es, keep = _episode_set(batch)
    loss = np.zeros(1)
    g = np.zeros(model.params().size) if with_grad else None
    net = ctx.upload(model)
    ctx.check(ctx._lib.reach_pred_loss(ctx.handle, net, C.byref(es), int(t_h), A.dptr(weights), A.dptr(loss),
                                       A.dptr(g) if with_grad else None), "pred_loss")
    return (float(loss[0]), g) if with_grad else float(loss[0])


def track_loss(controller: MLPNet, batch: Sequence[Episode], t_t: int, weights, gamma: float, delta: float,
               rk4_substeps: int = 4, cap: float = 1e6, plant=None, with_grad: bool = False,
               ctx: Optional[Context] = None):
    """track_loss (training.hpp:134-178) with the quadrotor plant (systems.hpp:22-64) on the device ->
    (loss, blowup_count), or with_grad -> (loss, gradient over the controller's net_params, blowup_count)."""
    weights = np.ascontiguousarray(weights, np.float64)
    if not batch or t_t < 1 or weights.size != t_t or delta <= 0.0 or rk4_substeps < 1:
        raise ValueError("track_loss: bad configuration")
    ctx = ctx or default_context()
    es, keep = _episode_set(batch)
    qp = np.ascontiguousarray((plant or QuadrotorParams()).as_array(), np.float64)
    loss = np.zeros(1)
    bc = np.zeros(1, np.int32)
    g = np.zeros(controller.params().size) if with_grad else None
    net = ctx.upload(controller)
    ctx.check(ctx._lib.reach_track_loss(ctx.handle, net, A.PLANT_QUADROTOR, A.dptr(qp), C.byref(es), int(t_t),
                                        A.dptr(weights), float(gamma), float(delta), int(rk4_substeps), float(cap),
                                        A.dptr(loss), A.dptr(g) if with_grad else None, A.iptr(bc)), "track_loss")
    return (float(loss[0]), g, int(bc[0])) if with_grad else (float(loss[0]), int(bc[0]))


@dataclass
class TrainConfig:  # training.hpp:262-282
    horizon_max: int = 4
    eps0: float = 0.1
    eps_final: float = 0.01
    lambda_: float = 0.0
    gamma: float = 0.1
    iters: int = 50
    batch: int = 4
    lr: float = 1e-3
    reach_cap: float = 20.0
    curriculum: bool = True
    seed: int = 0
    dt_prm: DTReachParams = field(default_factory=DTReachParams)

    def c(self):
        return A.TrainConfigC(self.horizon_max, self.eps0, self.eps_final, self.lambda_, self.gamma, self.iters,
                              self.batch, self.lr, self.reach_cap, int(self.curriculum), self.seed,
                              self.dt_prm.window, int(self.dt_prm.rebuild_from_box))


@dataclass
class TrainLogRow:  # training.hpp:284-292
    iter: int
    t_h: int
    eps: float
    l_pred: float
    l_reach: float
    l_total: float
    diverged_count: int


def train_log_csv(rows: Sequence[TrainLogRow]) -> str:
    """TrainLog::to_csv (training.hpp:297-305)."""
    from .formats import fmt_g17
    out = "iter,T_h,eps,L_pred,L_reach,L_total,diverged_count\n"
    for r in rows:
        out += (f"{r.iter},{r.t_h},{fmt_g17(r.eps)},{fmt_g17(r.l_pred)},{fmt_g17(r.l_reach)},"
                f"{fmt_g17(r.l_total)},{r.diverged_count}\n")
    return out


def train_dt_dyn(init: MLPNet, cfg: TrainConfig, dataset: Sequence[Episode], ctx: Optional[Context] = None):
    """train_dt_dyn (training.hpp:333-382) -> (trained MLPNet, [TrainLogRow]): the host loop (curriculum,
    the reference's minibatch stream, Adam) of the C ABI with every loss and gradient on the device."""
    ctx = ctx or default_context()
    es, keep = _episode_set(dataset)
    d, keep2 = init.desc()
    out = np.zeros(init.params().size)
    log = (A.TrainLogRowC * max(cfg.iters, 1))()
    cc = cfg.c()
    rc = ctx._lib.reach_train_dt_dyn(ctx.handle, C.byref(d), C.byref(cc), C.byref(es), A.dptr(out), log)
    rows = [TrainLogRow(r.iter, r.t_h, r.eps, r.l_pred, r.l_reach, r.l_total, r.diverged_count)
            for r in list(log)[:cfg.iters]]
    ctx.check(rc, "train_dt_dyn")
    return net_with_params(init, out), rows


# ---------------------------------------------------------------------------
class SplitPlan:
    """SplitPlan (refine.hpp:25-78)."""
    kMaxParts = 1 << 20

    def __init__(self, counts):
        self.counts = [int(c) for c in counts]

    @staticmethod
    def all_one(n_dims: int) -> "SplitPlan":
        return SplitPlan([1] * n_dims)

    @staticmethod
    def parse(s: str) -> "SplitPlan":
        toks = s.split("x")
        if any(t == "" for t in toks):
            raise ValueError(f'SplitPlan: empty count in "{s}"')
        return SplitPlan([int(t) for t in toks])

    @staticmethod
    def rpy(n_dims: int, parts: int) -> "SplitPlan":
        if n_dims < 9:
            raise ValueError("SplitPlan::rpy: needs at least 9 dimensions")
        k = int(round(parts ** (1.0 / 3.0)))
        if k < 1 or k * k * k != parts:
            raise ValueError("SplitPlan::rpy: parts must be a perfect cube")
        p = SplitPlan.all_one(n_dims)
        p.counts[6] = p.counts[7] = p.counts[8] = k
        return p

    def total_parts(self) -> int:
        t = 1
        for c in self.counts:
            if c < 1:
                raise ValueError("SplitPlan: counts must be >= 1")
            t *= c
            if t > self.kMaxParts:
                raise ValueError("SplitPlan: total part count overflow")
        return t

    def validate(self, n_dims: int):
        if len(self.counts) != n_dims:
            raise ValueError("SplitPlan: dimension mismatch")
        self.total_parts()


def split_box(x0_lo, x0_hi, plan: SplitPlan):
    """split_box (refine.hpp:83-115): [P][n] lo/hi, last dimension fastest."""
    x0_lo = np.asarray(x0_lo, np.float64)
    x0_hi = np.asarray(x0_hi, np.float64)
    n = x0_lo.size
    plan.validate(n)
    edges = []
    for d in range(n):
        k = plan.counts[d]
        e = [x0_lo[d] + (x0_hi[d] - x0_lo[d]) * (float(i) / k) for i in range(k + 1)]
        e[0], e[k] = x0_lo[d], x0_hi[d]
        edges.append(np.array(e))
    grids = np.meshgrid(*[np.arange(c) for c in plan.counts], indexing="ij")
    idx = np.stack([g.ravel() for g in grids], axis=1)
    lo = np.stack([edges[d][idx[:, d]] for d in range(n)], axis=1)
    hi = np.stack([edges[d][idx[:, d] + 1] for d in range(n)], axis=1)
    return lo, hi


@dataclass
class HullResult:
    """Partial or full hull of reach_with_splitting over a part range."""
    lo: np.ndarray  # [H+1][n]
    hi: np.ndarray
    box_diverged: np.ndarray
    n_boxes: int
    fail_key: int
    h: float = 0.0  # > 0: continuous-time hull (cl_reach engine)

    def tube(self) -> ReachTube:
        k = self.n_boxes
        t_lo, t_hi = _tube_times(k, self.h)
        tube = ReachTube(self.lo[:k].copy(), self.hi[:k].copy(), t_lo, t_hi)
        f = A.decode_fail_key(self.fail_key)
        tube.diverged = bool(np.any(self.box_diverged[:k])) or f is not None
        if f is not None:
            step, part, st = f
            tube.failed_step = int(step)
            tube.failure_reason = f"sub-box {part}: {A.TUBE_REASON.get(st, 'error')}"
        return tube


def reach_split_hull(sys: DTSystem, x0, plan: SplitPlan, actions, prm: DTReachParams = DTReachParams(),
                     part_begin: int = 0, part_end: int = 0, ctx: Optional[Context] = None,
                     precision: str = "exact") -> HullResult:
    """Hull over sub-boxes [part_begin, part_end) of reach_with_splitting (C ABI reach_split_hull)."""
    pflag = A.prec_flag(precision)
    sys.validate()
    ctx = ctx or default_context()
    lo0 = np.ascontiguousarray(x0[0], dtype=np.float64)
    hi0 = np.ascontiguousarray(x0[1], dtype=np.float64)
    plan.validate(sys.n)
    acts = np.ascontiguousarray(np.asarray(actions, dtype=np.float64).reshape(-1, sys.m) if sys.m else np.zeros((0, 0)))
    H = acts.shape[0] if sys.m else len(actions)
    counts = np.array(plan.counts, dtype=np.int32)
    out = HullResult(np.full((H + 1, sys.n), np.nan), np.full((H + 1, sys.n), np.nan), np.zeros(H + 1, np.int32), 0, 0)
    nb = np.zeros(1, np.int32)
    key = np.zeros(1, np.int64)
    args = A.SplitArgs(sys.n, sys.m, H, prm.window, int(prm.rebuild_from_box), A.dptr(lo0), A.dptr(hi0),
                       A.iptr(counts), A.dptr(acts if acts.size else np.zeros(1)), int(part_begin), int(part_end))
    ho = A.HullOut(A.dptr(out.lo), A.dptr(out.hi), A.iptr(out.box_diverged), A.iptr(nb), A.lptr(key))
    net = ctx.upload(sys.step)
    ctx.check(ctx._lib.reach_split_hull(ctx.handle, net, C.byref(args), C.byref(ho), pflag), "reach_with_splitting")
    out.n_boxes = int(nb[0])
    out.fail_key = int(key[0])
    return out


def reach_with_splitting(sys: DTSystem, x0, plan: SplitPlan, actions, prm: DTReachParams = DTReachParams(),
                         ctx: Optional[Context] = None, precision: str = "exact") -> ReachTube:
    """reach_with_splitting(dt_reach engine, x0, plan) (refine.hpp:121-160)."""
    return reach_split_hull(sys, x0, plan, actions, prm, ctx=ctx, precision=precision).tube()


# ---------------------------------------------------------------------------
def dt_closed_loop_batch(dyn: MLPNet, ctl: MLPNet, n: int, x0_lo: np.ndarray, x0_hi: np.ndarray, horizon: int,
                         prm: DTReachParams = DTReachParams(), ctx: Optional[Context] = None,
                         precision: str = "exact") -> TubeBatch:
    """DT closed loop: per step u = ctl_crown(x_tm, ctl) (neural.hpp:418),
    [x; u] stacked as cl_reach does (closed_loop.hpp:118-153), certify_tm_input(dyn, .), then
    dt_reach's re-seed / fold / box.  dyn: (n + l) -> n, ctl: n -> l.  precision "tc": the CROWN
    contractions on the int8 tensor cores (A.REACH_PREC_TC)."""
    pflag = A.prec_flag(precision)
    dyn.validate()
    ctl.validate()
    l = ctl.output_dim()
    if ctl.input_dim() != n:
        raise ValueError("ClosedLoopSpec: controller input dim mismatch")
    if dyn.input_dim() != n + l or dyn.output_dim() != n:
        raise ValueError("ClosedLoopSpec: dynamics must act on the augmented (x,u) state")
    ctx = ctx or default_context()
    x0_lo = np.ascontiguousarray(x0_lo, np.float64)
    x0_hi = np.ascontiguousarray(x0_hi, np.float64)
    B = x0_lo.shape[0]
    out = TubeBatch(np.full((B, horizon + 1, n), np.nan), np.full((B, horizon + 1, n), np.nan),
                    np.zeros(B, np.int32), np.zeros(B, np.int32), np.zeros(B, np.int32))
    args = A.DTArgs(B, horizon, n, 0, prm.window, int(prm.rebuild_from_box), A.dptr(x0_lo), A.dptr(x0_hi),
                    A.dptr(np.zeros(1)), 0)
    to = A.TubeOut(A.dptr(out.lo), A.dptr(out.hi), A.iptr(out.n_boxes), A.iptr(out.failed_step),
                   A.iptr(out.status))
    hd, hc = ctx.upload(dyn), ctx.upload(ctl)
    ctx.check(ctx._lib.reach_dtcl_batch(ctx.handle, hd, hc, C.byref(args), C.byref(to), pflag), "dt closed loop")
    return out


# ---------------------------------------------------------------------------
# Continuous-time closed loop (closed_loop.hpp:16-182) with an analytic plant.
@dataclass
class QuadrotorParams:
    """QuadrotorParams (systems.hpp:16-20)."""
    mass: float = 1.0
    gravity: float = 9.81
    jx: float = 0.01
    jy: float = 0.01
    jz: float = 0.02

    def as_array(self):
        return [self.mass, self.gravity, self.jx, self.jy, self.jz]


@dataclass
class FlowpipeParams:
    """FlowpipeParams (flowpipe_ct.hpp:35-50)."""
    h: float = 0.01
    steps: int = 100
    order: int = 2
    eps_init: float = 1e-4
    refine_rounds: int = 3
    enlargement: float = 2.0
    max_enlargements: int = 20
    window: int = 4

    def validate(self):
        if (self.h <= 0 or self.steps <= 0 or self.order < 1 or self.order > 2 or self.eps_init <= 0
                or self.enlargement <= 1.0 or self.refine_rounds < 0 or self.max_enlargements < 0 or self.window < 0):
            raise ValueError("FlowpipeParams: invalid configuration")

    def c_struct(self):
        return A.FlowpipeParamsC(self.h, self.steps, self.order, self.eps_init, self.refine_rounds, self.enlargement,
                                 self.max_enlargements, self.window)


@dataclass(eq=False)
class ClosedLoopSpec:
    """ClosedLoopSpec<double> (closed_loop.hpp:16-44).  The dynamics are an analytic plant
    augmented with udot = 0 rows (make_augmented_field, fields.hpp:96-128); only
    quadrotor_ode (systems.hpp:22-64, n = 12, l = 4) runs on the device."""
    controller: MLPNet
    n: int = 12
    l: int = 4
    ctl_steps: int = 1
    k_atomic: int = 1
    y_ref: Optional[np.ndarray] = None  # [ctl_steps][ref_dim]
    fp: FlowpipeParams = field(default_factory=FlowpipeParams)
    intervalize_boundary: bool = False
    plant: str = "quadrotor"
    plant_params: QuadrotorParams = field(default_factory=QuadrotorParams)

    def steps(self) -> int:
        return 1 + self.ctl_steps * self.k_atomic

    def validate(self):
        """ClosedLoopSpec::validate (closed_loop.hpp:30-43)."""
        self.fp.validate()
        if self.n <= 0 or self.l <= 0 or self.ctl_steps <= 0 or self.k_atomic <= 0:
            raise ValueError("ClosedLoopSpec: invalid dimensions")
        if self.plant != "quadrotor" or self.n != 12 or self.l != 4:
            raise ValueError("ClosedLoopSpec: dynamics must act on the augmented (x,u) state")
        self.controller.validate()
        if self.controller.output_dim() != self.l:
            raise ValueError("ClosedLoopSpec: controller output dim mismatch")
        yr = self._yref()
        ref_dim = 0 if yr is None else yr.shape[1]
        if self.controller.input_dim() != self.n + ref_dim:
            raise ValueError("ClosedLoopSpec: controller input dim mismatch")
        if yr is not None and yr.shape[0] != self.ctl_steps:
            raise ValueError("ClosedLoopSpec: reference sequence length mismatch")

    def _yref(self):
        if self.y_ref is None or len(self.y_ref) == 0:
            return None
        return np.ascontiguousarray(np.asarray(self.y_ref, np.float64).reshape(len(self.y_ref), -1))

    def c_struct(self):
        """(reach_cl_spec, keepalive)."""
        yr = self._yref()
        prm = (C.c_double * 8)(*(self.plant_params.as_array() + [0.0] * 3))
        s = A.CLSpecC(A.PLANT_QUADROTOR, prm, self.n, self.l, self.ctl_steps, self.k_atomic,
                      0 if yr is None else yr.shape[1], A.dptr(yr), self.fp.c_struct(), int(self.intervalize_boundary))
        return s, (yr, prm)


def train_ct_ctl(init: MLPNet, cfg: "TrainConfig", dataset: Sequence[Episode], delta: float, k_atomic: int = 1,
                 rk4_substeps: int = 4, fp_base: Optional[FlowpipeParams] = None,
                 plant: Optional[QuadrotorParams] = None, ctx: Optional[Context] = None):
    """train_ct_ctl (training.hpp:389-442) with the quadrotor plant -> (trained controller, [TrainLogRow]):
    L = track_loss + lambda ctl_reach_loss; the host loop of the C ABI (curriculum, the reference's
    minibatch stream, Adam) with every loss and gradient on the device."""
    ctx = ctx or default_context()
    es, keep = _episode_set(dataset)
    r = len(dataset[0].y_ref[0]) if len(dataset[0].y_ref) else 0
    base = ClosedLoopSpec(init, n=12, l=4, ctl_steps=1, k_atomic=k_atomic,
                          y_ref=np.zeros((1, r)) if r else None, fp=dataclasses.replace(fp_base or FlowpipeParams()),
                          plant_params=plant or QuadrotorParams())
    cs, keep2 = base.c_struct()
    d, keep3 = init.desc()
    out = np.zeros(init.params().size)
    log = (A.TrainLogRowC * max(cfg.iters, 1))()
    cc = cfg.c()
    rc = ctx._lib.reach_train_ct_ctl(ctx.handle, C.byref(d), C.byref(cc), C.byref(es), C.byref(cs), float(delta),
                                     int(rk4_substeps), A.dptr(out), log)
    rows = [TrainLogRow(q.iter, q.t_h, q.eps, q.l_pred, q.l_reach, q.l_total, q.diverged_count)
            for q in list(log)[:cfg.iters]]
    ctx.check(rc, "train_ct_ctl")
    return net_with_params(init, out), rows


def cl_reach_batch_arrays(spec: ClosedLoopSpec, x0_lo: np.ndarray, x0_hi: np.ndarray,
                          ctx: Optional[Context] = None) -> TubeBatch:
    """cl_reach (closed_loop.hpp:76-182) for a batch of initial boxes x0 [B][n]; boxes have n + l dims."""
    spec.validate()
    ctx = ctx or default_context()
    x0_lo = np.ascontiguousarray(x0_lo, dtype=np.float64)
    x0_hi = np.ascontiguousarray(x0_hi, dtype=np.float64)
    B = x0_lo.shape[0]
    if x0_lo.shape != (B, spec.n) or x0_hi.shape != (B, spec.n):
        raise ValueError("cl_reach: X0 dimension mismatch")
    T, na = spec.steps(), spec.n + spec.l
    out = TubeBatch(np.full((B, T, na), np.nan), np.full((B, T, na), np.nan), np.zeros(B, np.int32),
                    np.zeros(B, np.int32), np.zeros(B, np.int32), h=spec.fp.h)
    cs, keep = spec.c_struct()
    to = A.TubeOut(A.dptr(out.lo), A.dptr(out.hi), A.iptr(out.n_boxes), A.iptr(out.failed_step),
                   A.iptr(out.status))
    net = ctx.upload(spec.controller)
    ctx.check(ctx._lib.reach_cl_batch(ctx.handle, net, C.byref(cs), B, A.dptr(x0_lo), A.dptr(x0_hi), C.byref(to), 0),
              "cl_reach")
    return out


def cl_reach(spec: ClosedLoopSpec, x0, ctx: Optional[Context] = None) -> ReachTube:
    """cl_reach (closed_loop.hpp:76-77): x0 = (lo, hi)."""
    lo = np.asarray(x0[0], np.float64).reshape(1, -1)
    hi = np.asarray(x0[1], np.float64).reshape(1, -1)
    return cl_reach_batch_arrays(spec, lo, hi, ctx).tube(0)


def cl_split_hull(spec: ClosedLoopSpec, x0, plan: SplitPlan, part_begin: int = 0, part_end: int = 0,
                  ctx: Optional[Context] = None) -> HullResult:
    """Hull over sub-boxes [part_begin, part_end) of reach_with_splitting(cl_reach) (C ABI reach_cl_split_hull)."""
    spec.validate()
    ctx = ctx or default_context()
    lo0 = np.ascontiguousarray(x0[0], dtype=np.float64)
    hi0 = np.ascontiguousarray(x0[1], dtype=np.float64)
    plan.validate(spec.n)
    counts = np.array(plan.counts, dtype=np.int32)
    T, na = spec.steps(), spec.n + spec.l
    out = HullResult(np.full((T, na), np.nan), np.full((T, na), np.nan), np.zeros(T, np.int32), 0, 0, h=spec.fp.h)
    nb = np.zeros(1, np.int32)
    key = np.zeros(1, np.int64)
    cs, keep = spec.c_struct()
    args = A.CLSplitArgs(A.dptr(lo0), A.dptr(hi0), A.iptr(counts), int(part_begin), int(part_end))
    ho = A.HullOut(A.dptr(out.lo), A.dptr(out.hi), A.iptr(out.box_diverged), A.iptr(nb), A.lptr(key))
    net = ctx.upload(spec.controller)
    ctx.check(ctx._lib.reach_cl_split_hull(ctx.handle, net, C.byref(cs), C.byref(args), C.byref(ho), 0),
              "reach_with_splitting(cl_reach)")
    out.n_boxes = int(nb[0])
    out.fail_key = int(key[0])
    return out


def cl_reach_with_splitting(spec: ClosedLoopSpec, x0, plan: SplitPlan, ctx: Optional[Context] = None) -> ReachTube:
    """reach_with_splitting(cl_reach engine, x0, plan) (refine.hpp:121-160)."""
    return cl_split_hull(spec, x0, plan, ctx=ctx).tube()


# ---------------------------------------------------------------------------
# Open-loop continuous-time flowpipes (ct_reach, flowpipe_ct.hpp:428-458) of the
# analytic VectorFields of fields.hpp.  A field here is a descriptor, not a
# closure: the device evaluates it as a Taylor-model field program.
@dataclass
class AnalyticField:
    kind: int
    n: int
    params: List[float] = field(default_factory=list)

    def c_struct(self):
        p = (C.c_double * 16)(*(list(self.params) + [0.0] * (16 - len(self.params))))
        return A.FieldDescC(self.kind, self.n, p)


def zero_field(n: int) -> AnalyticField:
    """zero_field (fields.hpp:87-92)."""
    return AnalyticField(A.FIELD_ZERO, n)


def diag_linear_field(lam) -> AnalyticField:
    """diag_linear_field (fields.hpp:72-78): xdot_i = lambda_i x_i."""
    lam = [float(v) for v in lam]
    return AnalyticField(A.FIELD_DIAG_LINEAR, len(lam), lam)


def rotation_field(w: float) -> AnalyticField:
    """rotation_field (fields.hpp:80-85): x' = -w y, y' = w x."""
    return AnalyticField(A.FIELD_ROTATION, 2, [float(w)])


def quadrotor_hover_input(prm: QuadrotorParams = None):
    """quadrotor_hover_input (systems.hpp:66-68)."""
    prm = prm or QuadrotorParams()
    return [prm.mass * prm.gravity, 0.0, 0.0, 0.0]


def quadrotor_field(prm: QuadrotorParams = None, u=None) -> AnalyticField:
    """quadrotor_field (fields.hpp:51-56) with the held input u (4)."""
    prm = prm or QuadrotorParams()
    u = list(u) if u is not None else quadrotor_hover_input(prm)
    return AnalyticField(A.FIELD_QUADROTOR, 12, prm.as_array() + [float(v) for v in u])


def ct_reach_batch_arrays(f: AnalyticField, x0_lo: np.ndarray, x0_hi: np.ndarray, prm: FlowpipeParams = None,
                          ctx: Optional[Context] = None) -> TubeBatch:
    """ct_reach (flowpipe_ct.hpp:428-458) for a batch of initial boxes x0 [B][n]."""
    prm = prm or FlowpipeParams()
    prm.validate()
    ctx = ctx or default_context()
    x0_lo = np.ascontiguousarray(x0_lo, dtype=np.float64)
    x0_hi = np.ascontiguousarray(x0_hi, dtype=np.float64)
    B = x0_lo.shape[0]
    if x0_lo.shape != (B, f.n) or x0_hi.shape != (B, f.n):
        raise ValueError("ct_reach: X0 dimension mismatch")
    T = 1 + prm.steps
    out = TubeBatch(np.full((B, T, f.n), np.nan), np.full((B, T, f.n), np.nan), np.zeros(B, np.int32),
                    np.zeros(B, np.int32), np.zeros(B, np.int32), h=prm.h)
    fd = f.c_struct()
    fp = prm.c_struct()
    to = A.TubeOut(A.dptr(out.lo), A.dptr(out.hi), A.iptr(out.n_boxes), A.iptr(out.failed_step),
                   A.iptr(out.status))
    ctx.check(ctx._lib.reach_ct_batch(ctx.handle, C.byref(fd), C.byref(fp), B, A.dptr(x0_lo), A.dptr(x0_hi),
                                      C.byref(to), 0), "ct_reach")
    return out


def ct_reach(f: AnalyticField, x0, prm: FlowpipeParams = None, ctx: Optional[Context] = None) -> ReachTube:
    """ct_reach (flowpipe_ct.hpp:428-430): x0 = (lo, hi)."""
    lo = np.asarray(x0[0], np.float64).reshape(1, -1)
    hi = np.asarray(x0[1], np.float64).reshape(1, -1)
    return ct_reach_batch_arrays(f, lo, hi, prm, ctx).tube(0)


def ct_split_hull(f: AnalyticField, x0, plan: SplitPlan, prm: FlowpipeParams = None, part_begin: int = 0,
                  part_end: int = 0, ctx: Optional[Context] = None) -> HullResult:
    """Hull over sub-boxes [part_begin, part_end) of reach_with_splitting(ct_reach) (C ABI reach_ct_split_hull;
    the CLI's `split` / `reach-ct --split`, reach_cli.cpp:200-211)."""
    prm = prm or FlowpipeParams()
    prm.validate()
    ctx = ctx or default_context()
    lo0 = np.ascontiguousarray(x0[0], dtype=np.float64)
    hi0 = np.ascontiguousarray(x0[1], dtype=np.float64)
    plan.validate(f.n)
    counts = np.array(plan.counts, dtype=np.int32)
    T = 1 + prm.steps
    out = HullResult(np.full((T, f.n), np.nan), np.full((T, f.n), np.nan), np.zeros(T, np.int32), 0, 0, h=prm.h)
    nb = np.zeros(1, np.int32)
    key = np.zeros(1, np.int64)
    fd = f.c_struct()
    fp = prm.c_struct()
    args = A.CLSplitArgs(A.dptr(lo0), A.dptr(hi0), A.iptr(counts), int(part_begin), int(part_end))
    ho = A.HullOut(A.dptr(out.lo), A.dptr(out.hi), A.iptr(out.box_diverged), A.iptr(nb), A.lptr(key))
    ctx.check(ctx._lib.reach_ct_split_hull(ctx.handle, C.byref(fd), C.byref(fp), C.byref(args), C.byref(ho), 0),
              "reach_with_splitting(ct_reach)")
    out.n_boxes = int(nb[0])
    out.fail_key = int(key[0])
    return out


def ct_reach_with_splitting(f: AnalyticField, x0, plan: SplitPlan, prm: FlowpipeParams = None,
                            ctx: Optional[Context] = None) -> ReachTube:
    """reach_with_splitting(ct_reach engine, x0, plan) (refine.hpp:121-160)."""
    return ct_split_hull(f, x0, plan, prm, ctx=ctx).tube()


def _predicted_volume(lo: np.ndarray, hi: np.ndarray) -> float:
    """predicted_volume (training.hpp:86-93): box volume proxies of boxes 1.. (the input box excluded)."""
    v = 0.0
    for k in range(1, lo.shape[0]):
        v += box_volume_proxy(lo[k], hi[k])
    return v


def ctl_reach_loss(controller: MLPNet, batch: Sequence[Episode], eps: float, t_h: int, delta: float,
                   k_atomic: int, cap: float, fp_base: Optional[FlowpipeParams] = None,
                   plant: Optional[QuadrotorParams] = None, n: int = 12, l: int = 4,
                   ctx: Optional[Context] = None, with_grad: bool = False):
    """ctl_reach_loss (training.hpp:183-213) with the quadrotor plant: cl_reach from the eps-ball around
    each episode start, every tube on the device (episodes sharing a reference sequence in one batch)
    -> (loss, diverged_count); with_grad -> (loss, grad_forward over the controller's net_params,
    diverged_count): one Dual cl_reach per (parameter, episode) in one launch (reach_ctl_reach_loss).
    As the reference, an episode without y_ref keeps the previous episode's reference sequence."""
    if not batch or t_h < 1:
        raise ValueError("ctl_reach_loss: bad batch/horizon")
    fp = dataclasses.replace(fp_base or FlowpipeParams())
    fp.h = delta / k_atomic
    yrefs, cur = [], None
    for ep in batch:
        if len(ep.y_ref):
            cur = np.ascontiguousarray(np.asarray(ep.y_ref[:t_h], np.float64).reshape(t_h, -1))
        yrefs.append(cur)
    if with_grad:
        ctx = ctx or default_context()
        rd = 0 if yrefs[0] is None else yrefs[0].shape[1]
        if rd and any(y is None for y in yrefs):
            raise ValueError("freeze_trailing_inputs: dimension mismatch")
        spec = ClosedLoopSpec(controller, n=n, l=l, ctl_steps=t_h, k_atomic=k_atomic,
                              y_ref=yrefs[0] if rd else None, fp=dataclasses.replace(fp),
                              plant_params=plant or QuadrotorParams())
        cs, keep = spec.c_struct()
        x0 = np.ascontiguousarray([np.asarray(ep.states[0], np.float64) for ep in batch])
        yr = np.ascontiguousarray(np.array(yrefs, np.float64)) if rd else np.zeros(1)
        loss = np.zeros(1)
        g = np.zeros(controller.params().size)
        dc = np.zeros(1, np.int32)
        net = ctx.upload(controller)
        ctx.check(ctx._lib.reach_ctl_reach_loss(ctx.handle, net, C.byref(cs), len(batch), A.dptr(x0),
                                                A.dptr(yr) if rd else None, float(eps), float(cap), A.dptr(loss),
                                                A.dptr(g), A.iptr(dc)), "ctl_reach_loss")
        return float(loss[0]), g, int(dc[0])
    groups = {}
    for e, yr in enumerate(yrefs):
        groups.setdefault(None if yr is None else yr.tobytes(), []).append(e)
    terms = [0.0] * len(batch)
    diverged = [False] * len(batch)
    for key, idx in groups.items():
        yr = yrefs[idx[0]]
        spec = ClosedLoopSpec(controller, n=n, l=l, ctl_steps=t_h, k_atomic=k_atomic, y_ref=yr,
                              fp=dataclasses.replace(fp), plant_params=plant or QuadrotorParams())
        x0 = np.array([np.asarray(batch[e].states[0], np.float64) for e in idx])
        tb = cl_reach_batch_arrays(spec, x0 - eps, x0 + eps, ctx)
        for r, e in enumerate(idx):
            t = tb.tube(r)
            if t.diverged:
                diverged[e] = True
                terms[e] = cap
            else:
                terms[e] = math.log(1.0 + _predicted_volume(t.lo, t.hi))
    acc = 0.0
    for v in terms:
        acc += v
    return acc / float(len(batch)), int(sum(diverged))
