"""Test-side bindings of the CPU checkers (oracle/): the C restatement
(oracle/liboracle.so) and the reference itself (oracle/_ref/libreach_ref.so).

Only tests, __graft_entry__.smoke() and bench.py's CPU legs import this.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_2605_25346_b200 import _abi as A
from paper_2605_25346_b200.api import DTReachParams, DTSystem, HullResult, SplitPlan, TubeBatch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "liboracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libreach_ref.so")


def _build_oracle():
    if not os.path.exists(ORACLE_SO):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "liboracle.so"], check=True,
                       stdout=subprocess.DEVNULL)


def _load(path, prefix):
    lib = C.CDLL(path)
    f = getattr(lib, prefix + "dt_batch")
    f.argtypes = [C.POINTER(A.NetDesc), C.POINTER(A.DTArgs), C.POINTER(A.TubeOut)] + ([C.c_int32] if prefix == "ref_" else [])
    f.restype = C.c_int
    g = getattr(lib, prefix + "split_hull")
    g.argtypes = [C.POINTER(A.NetDesc), C.POINTER(A.SplitArgs), C.POINTER(A.HullOut)] + ([C.c_int32] if prefix == "ref_" else [])
    g.restype = C.c_int
    return lib


_cache = {}


def oracle_lib():
    if "orc" not in _cache:
        _build_oracle()
        _cache["orc"] = _load(ORACLE_SO, "orc_")
    return _cache["orc"]


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref_lib():
    if "ref" not in _cache:
        _cache["ref"] = _load(REF_SO, "ref_")
    return _cache["ref"]


def _dt(lib, prefix, sys: DTSystem, x0_lo, x0_hi, actions, prm: DTReachParams, shared=False, threads=None):
    x0_lo = np.ascontiguousarray(x0_lo, np.float64)
    x0_hi = np.ascontiguousarray(x0_hi, np.float64)
    B = x0_lo.shape[0]
    actions = np.ascontiguousarray(actions, np.float64)
    H = actions.shape[0] if shared else actions.shape[1]
    out = TubeBatch(np.full((B, H + 1, sys.n), np.nan), np.full((B, H + 1, sys.n), np.nan),
                    np.zeros(B, np.int32), np.zeros(B, np.int32), np.zeros(B, np.int32))
    desc, keep = sys.step.desc()
    args = A.DTArgs(B, H, sys.n, sys.m, prm.window, int(prm.rebuild_from_box), A.dptr(x0_lo), A.dptr(x0_hi),
                    A.dptr(actions if actions.size else np.zeros(1)), int(shared))
    to = A.TubeOut(A.dptr(out.lo), A.dptr(out.hi), A.iptr(out.n_boxes), A.iptr(out.failed_step), A.iptr(out.status))
    fn = getattr(lib, prefix + "dt_batch")
    rc = fn(C.byref(desc), C.byref(args), C.byref(to), *([threads or 0] if prefix == "ref_" else []))
    assert rc == 0, rc
    return out


def oracle_dt_batch(sys, x0_lo, x0_hi, actions, prm=DTReachParams(), shared=False):
    return _dt(oracle_lib(), "orc_", sys, x0_lo, x0_hi, actions, prm, shared)


def ref_dt_batch(sys, x0_lo, x0_hi, actions, prm=DTReachParams(), shared=False, threads=0):
    return _dt(ref_lib(), "ref_", sys, x0_lo, x0_hi, actions, prm, shared, threads)


def _hull(lib, prefix, sys, x0_lo, x0_hi, plan: SplitPlan, actions, prm, begin=0, end=0, threads=None):
    acts = np.ascontiguousarray(np.asarray(actions, np.float64).reshape(-1, sys.m) if sys.m else np.zeros((0, 0)))
    H = acts.shape[0] if sys.m else len(actions)
    lo0 = np.ascontiguousarray(x0_lo, np.float64)
    hi0 = np.ascontiguousarray(x0_hi, np.float64)
    counts = np.array(plan.counts, np.int32)
    out = HullResult(np.full((H + 1, sys.n), np.nan), np.full((H + 1, sys.n), np.nan), np.zeros(H + 1, np.int32), 0, 0)
    nb = np.zeros(1, np.int32)
    key = np.zeros(1, np.int64)
    desc, keep = sys.step.desc()
    args = A.SplitArgs(sys.n, sys.m, H, prm.window, int(prm.rebuild_from_box), A.dptr(lo0), A.dptr(hi0),
                       A.iptr(counts), A.dptr(acts if acts.size else np.zeros(1)), int(begin), int(end))
    ho = A.HullOut(A.dptr(out.lo), A.dptr(out.hi), A.iptr(out.box_diverged), A.iptr(nb), A.lptr(key))
    fn = getattr(lib, prefix + "split_hull")
    rc = fn(C.byref(desc), C.byref(args), C.byref(ho), *([threads or 0] if prefix == "ref_" else []))
    assert rc == 0, rc
    out.n_boxes = int(nb[0])
    out.fail_key = int(key[0])
    return out


def oracle_split_hull(sys, x0_lo, x0_hi, plan, actions, prm=DTReachParams(), begin=0, end=0):
    return _hull(oracle_lib(), "orc_", sys, x0_lo, x0_hi, plan, actions, prm, begin, end)


def ref_split_hull(sys, x0_lo, x0_hi, plan, actions, prm=DTReachParams(), begin=0, end=0, threads=0):
    return _hull(ref_lib(), "ref_", sys, x0_lo, x0_hi, plan, actions, prm, begin, end, threads)


def ref_reach_with_splitting(sys, x0_lo, x0_hi, plan: SplitPlan, actions, prm=DTReachParams()):
    """The reference's reach_with_splitting(dt_reach) driver verbatim (refine.hpp:121-160), full plan."""
    acts = np.ascontiguousarray(np.asarray(actions, np.float64).reshape(-1, sys.m) if sys.m else np.zeros((0, 0)))
    H = acts.shape[0] if sys.m else len(actions)
    lo0 = np.ascontiguousarray(x0_lo, np.float64)
    hi0 = np.ascontiguousarray(x0_hi, np.float64)
    counts = np.array(plan.counts, np.int32)
    lo = np.full((H + 1, sys.n), np.nan)
    hi = np.full((H + 1, sys.n), np.nan)
    nb = np.zeros(1, np.int32)
    fs = np.zeros(1, np.int32)
    desc, keep = sys.step.desc()
    args = A.SplitArgs(sys.n, sys.m, H, prm.window, int(prm.rebuild_from_box), A.dptr(lo0), A.dptr(hi0),
                       A.iptr(counts), A.dptr(acts if acts.size else np.zeros(1)), 0, 0)
    f = ref_lib().ref_reach_with_splitting
    f.argtypes = [C.POINTER(A.NetDesc), C.POINTER(A.SplitArgs), C.POINTER(C.c_double), C.POINTER(C.c_double),
                  C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
    f.restype = C.c_int
    rc = f(C.byref(desc), C.byref(args), A.dptr(lo), A.dptr(hi), A.iptr(nb), A.iptr(fs))
    assert rc == 0, rc
    return lo, hi, int(nb[0]), int(fs[0])


def same_bits(a: np.ndarray, b: np.ndarray) -> bool:
    """Bitwise equality up to the sign of zero (NaN == NaN)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if a.shape != b.shape:
        return False
    eq = (a == b) | (np.isnan(a) & np.isnan(b))
    return bool(np.all(eq))


def assert_tubes_equal(got: TubeBatch, exp: TubeBatch, exact=True, rtol=1e-12):
    assert np.array_equal(got.n_boxes, exp.n_boxes), (got.n_boxes, exp.n_boxes)
    assert np.array_equal(got.status, exp.status), (got.status, exp.status)
    assert np.array_equal(got.failed_step, exp.failed_step)
    for b in range(got.lo.shape[0]):
        k = int(exp.n_boxes[b])
        for arr_g, arr_e in ((got.lo, exp.lo), (got.hi, exp.hi)):
            g, e = arr_g[b, :k], arr_e[b, :k]
            if exact:
                assert same_bits(g, e), (b, np.max(np.abs(g - e)))
            else:
                fin = np.isfinite(e)
                scale = np.maximum(np.abs(e[fin]), 1e-300)
                assert np.all(np.abs(g[fin] - e[fin]) <= rtol * np.maximum(scale, 1.0)), b


# --- MPC -------------------------------------------------------------------
def _mpc_fn(lib, name, argtypes):
    f = getattr(lib, name)
    f.argtypes = argtypes
    f.restype = C.c_int
    return f


def _plan_eval(lib, prefix, prob, x0, actions, threads=None):
    dp, ip = C.POINTER(C.c_double), C.POINTER(C.c_int32)
    args = [C.POINTER(A.NetDesc), C.POINTER(A.PlanProblemC), dp, C.c_int32, dp, dp, ip]
    if prefix == "ref_":
        args.append(C.c_int32)
    f = _mpc_fn(lib, prefix + "plan_eval_batch", args)
    x0 = np.ascontiguousarray(x0, np.float64)
    acts = np.ascontiguousarray(actions, np.float64)
    B = acts.shape[0]
    obj = np.zeros(B)
    div = np.zeros(B, np.int32)
    desc, keep = prob.sys.step.desc()
    p, keep2 = prob.c_struct()
    extra = [threads or 0] if prefix == "ref_" else []
    rc = f(C.byref(desc), C.byref(p), A.dptr(x0), B, A.dptr(acts), A.dptr(obj), A.iptr(div), *extra)
    assert rc == 0, rc
    return obj, div.astype(bool)


def oracle_plan_eval_batch(prob, x0, actions):
    return _plan_eval(oracle_lib(), "orc_", prob, x0, actions)


def ref_plan_eval_batch(prob, x0, actions, threads=0):
    return _plan_eval(ref_lib(), "ref_", prob, x0, actions, threads)


def _plan_cem(lib, prefix, prob, cfg, x0):
    dp, ip = C.POINTER(C.c_double), C.POINTER(C.c_int32)
    f = _mpc_fn(lib, prefix + "plan_cem", [C.POINTER(A.NetDesc), C.POINTER(A.PlanProblemC),
                                           C.POINTER(A.SamplerConfigC), dp, dp, dp, dp, ip])
    x0 = np.ascontiguousarray(x0, np.float64)
    best = np.zeros((prob.horizon, prob.sys.m))
    obj = np.zeros(1)
    hist = np.zeros(cfg.iterations)
    be = np.zeros(1, np.int32)
    desc, keep = prob.sys.step.desc()
    p, keep2 = prob.c_struct()
    c = cfg.c_struct()
    rc = f(C.byref(desc), C.byref(p), C.byref(c), A.dptr(x0), A.dptr(best), A.dptr(obj), A.dptr(hist), A.iptr(be))
    assert rc == 0, rc
    return best, float(obj[0]), hist, bool(be[0])


def oracle_plan_cem(prob, cfg, x0):
    return _plan_cem(oracle_lib(), "orc_", prob, cfg, x0)


def ref_plan_cem(prob, cfg, x0):
    return _plan_cem(ref_lib(), "ref_", prob, cfg, x0)


# --- DT closed loop (A11) ---------------------------------------------------
def _dtcl(lib, prefix, dyn, ctl, n, x0_lo, x0_hi, horizon, prm, threads=None):
    args_t = [C.POINTER(A.NetDesc), C.POINTER(A.NetDesc), C.POINTER(A.DTArgs), C.POINTER(A.TubeOut)]
    if prefix == "ref_":
        args_t.append(C.c_int32)
    f = _mpc_fn(lib, prefix + "dtcl_batch", args_t)
    x0_lo = np.ascontiguousarray(x0_lo, np.float64)
    x0_hi = np.ascontiguousarray(x0_hi, np.float64)
    B = x0_lo.shape[0]
    out = TubeBatch(np.full((B, horizon + 1, n), np.nan), np.full((B, horizon + 1, n), np.nan),
                    np.zeros(B, np.int32), np.zeros(B, np.int32), np.zeros(B, np.int32))
    dd, k1 = dyn.desc()
    cd, k2 = ctl.desc()
    args = A.DTArgs(B, horizon, n, 0, prm.window, int(prm.rebuild_from_box), A.dptr(x0_lo), A.dptr(x0_hi),
                    A.dptr(np.zeros(1)), 0)
    to = A.TubeOut(A.dptr(out.lo), A.dptr(out.hi), A.iptr(out.n_boxes), A.iptr(out.failed_step), A.iptr(out.status))
    extra = [threads or 0] if prefix == "ref_" else []
    assert f(C.byref(dd), C.byref(cd), C.byref(args), C.byref(to), *extra) == 0
    return out


def oracle_dtcl_batch(dyn, ctl, n, x0_lo, x0_hi, horizon, prm=DTReachParams()):
    return _dtcl(oracle_lib(), "orc_", dyn, ctl, n, x0_lo, x0_hi, horizon, prm)


def ref_dtcl_batch(dyn, ctl, n, x0_lo, x0_hi, horizon, prm=DTReachParams(), threads=0):
    return _dtcl(ref_lib(), "ref_", dyn, ctl, n, x0_lo, x0_hi, horizon, prm, threads)


# --- continuous-time closed loop (cl_reach) ----------------------------------
def _cl(lib, prefix, spec, x0_lo, x0_hi, threads=None):
    from paper_2605_25346_b200.api import TubeBatch as TB
    args_t = [C.POINTER(A.NetDesc), C.POINTER(A.CLSpecC), C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_double),
              C.POINTER(A.TubeOut)]
    if prefix == "ref_":
        args_t.append(C.c_int32)
    f = _mpc_fn(lib, prefix + "cl_batch", args_t)
    x0_lo = np.ascontiguousarray(x0_lo, np.float64)
    x0_hi = np.ascontiguousarray(x0_hi, np.float64)
    B = x0_lo.shape[0]
    T, na = spec.steps(), spec.n + spec.l
    out = TB(np.full((B, T, na), np.nan), np.full((B, T, na), np.nan), np.zeros(B, np.int32),
             np.zeros(B, np.int32), np.zeros(B, np.int32), h=spec.fp.h)
    cd, k1 = spec.controller.desc()
    cs, k2 = spec.c_struct()
    to = A.TubeOut(A.dptr(out.lo), A.dptr(out.hi), A.iptr(out.n_boxes), A.iptr(out.failed_step), A.iptr(out.status))
    extra = [threads or 0] if prefix == "ref_" else []
    rc = f(C.byref(cd), C.byref(cs), B, A.dptr(x0_lo), A.dptr(x0_hi), C.byref(to), *extra)
    assert rc == 0, rc
    return out


def oracle_cl_batch(spec, x0_lo, x0_hi):
    return _cl(oracle_lib(), "orc_", spec, x0_lo, x0_hi)


def ref_cl_batch(spec, x0_lo, x0_hi, threads=0):
    return _cl(ref_lib(), "ref_", spec, x0_lo, x0_hi, threads)


def _cl_hull(lib, prefix, spec, x0_lo, x0_hi, plan, begin=0, end=0, threads=None):
    args_t = [C.POINTER(A.NetDesc), C.POINTER(A.CLSpecC), C.POINTER(A.CLSplitArgs), C.POINTER(A.HullOut)]
    if prefix == "ref_":
        args_t.append(C.c_int32)
    f = _mpc_fn(lib, prefix + "cl_split_hull", args_t)
    T, na = spec.steps(), spec.n + spec.l
    lo0 = np.ascontiguousarray(x0_lo, np.float64)
    hi0 = np.ascontiguousarray(x0_hi, np.float64)
    counts = np.array(plan.counts, np.int32)
    out = HullResult(np.full((T, na), np.nan), np.full((T, na), np.nan), np.zeros(T, np.int32), 0, 0, h=spec.fp.h)
    nb = np.zeros(1, np.int32)
    key = np.zeros(1, np.int64)
    cd, k1 = spec.controller.desc()
    cs, k2 = spec.c_struct()
    args = A.CLSplitArgs(A.dptr(lo0), A.dptr(hi0), A.iptr(counts), int(begin), int(end))
    ho = A.HullOut(A.dptr(out.lo), A.dptr(out.hi), A.iptr(out.box_diverged), A.iptr(nb), A.lptr(key))
    extra = [threads if threads is not None else 0] if prefix == "ref_" else []
    rc = f(C.byref(cd), C.byref(cs), C.byref(args), C.byref(ho), *extra)
    assert rc == 0, rc
    out.n_boxes = int(nb[0])
    out.fail_key = int(key[0])
    return out


def oracle_cl_split_hull(spec, x0_lo, x0_hi, plan, begin=0, end=0):
    return _cl_hull(oracle_lib(), "orc_", spec, x0_lo, x0_hi, plan, begin, end)


def ref_cl_split_hull(spec, x0_lo, x0_hi, plan, begin=0, end=0, threads=0):
    return _cl_hull(ref_lib(), "ref_", spec, x0_lo, x0_hi, plan, begin, end, threads)


# --- open-loop continuous-time flowpipe (ct_reach) ---------------------------
def _ct(lib, prefix, f, x0_lo, x0_hi, prm, threads=None):
    from paper_2605_25346_b200.api import TubeBatch as TB
    args_t = [C.POINTER(A.FieldDescC), C.POINTER(A.FlowpipeParamsC), C.c_int32, C.POINTER(C.c_double),
              C.POINTER(C.c_double), C.POINTER(A.TubeOut)]
    if prefix == "ref_":
        args_t.append(C.c_int32)
    fn = _mpc_fn(lib, prefix + "ct_batch", args_t)
    x0_lo = np.ascontiguousarray(x0_lo, np.float64)
    x0_hi = np.ascontiguousarray(x0_hi, np.float64)
    B = x0_lo.shape[0]
    T = 1 + prm.steps
    out = TB(np.full((B, T, f.n), np.nan), np.full((B, T, f.n), np.nan), np.zeros(B, np.int32),
             np.zeros(B, np.int32), np.zeros(B, np.int32), h=prm.h)
    fd = f.c_struct()
    fp = prm.c_struct()
    to = A.TubeOut(A.dptr(out.lo), A.dptr(out.hi), A.iptr(out.n_boxes), A.iptr(out.failed_step), A.iptr(out.status))
    extra = [threads or 0] if prefix == "ref_" else []
    rc = fn(C.byref(fd), C.byref(fp), B, A.dptr(x0_lo), A.dptr(x0_hi), C.byref(to), *extra)
    assert rc == 0, rc
    return out


def oracle_ct_batch(f, x0_lo, x0_hi, prm):
    return _ct(oracle_lib(), "orc_", f, x0_lo, x0_hi, prm)


def ref_ct_batch(f, x0_lo, x0_hi, prm, threads=0):
    return _ct(ref_lib(), "ref_", f, x0_lo, x0_hi, prm, threads)


def _ct_hull(lib, prefix, f, x0_lo, x0_hi, plan, prm, begin=0, end=0, threads=None):
    args_t = [C.POINTER(A.FieldDescC), C.POINTER(A.FlowpipeParamsC), C.POINTER(A.CLSplitArgs), C.POINTER(A.HullOut)]
    if prefix == "ref_":
        args_t.append(C.c_int32)
    fn = _mpc_fn(lib, prefix + "ct_split_hull", args_t)
    T = 1 + prm.steps
    lo0 = np.ascontiguousarray(x0_lo, np.float64)
    hi0 = np.ascontiguousarray(x0_hi, np.float64)
    counts = np.array(plan.counts, np.int32)
    out = HullResult(np.full((T, f.n), np.nan), np.full((T, f.n), np.nan), np.zeros(T, np.int32), 0, 0, h=prm.h)
    nb = np.zeros(1, np.int32)
    key = np.zeros(1, np.int64)
    fd = f.c_struct()
    fp = prm.c_struct()
    args = A.CLSplitArgs(A.dptr(lo0), A.dptr(hi0), A.iptr(counts), int(begin), int(end))
    ho = A.HullOut(A.dptr(out.lo), A.dptr(out.hi), A.iptr(out.box_diverged), A.iptr(nb), A.lptr(key))
    extra = [threads if threads is not None else 0] if prefix == "ref_" else []
    rc = fn(C.byref(fd), C.byref(fp), C.byref(args), C.byref(ho), *extra)
    assert rc == 0, rc
    out.n_boxes = int(nb[0])
    out.fail_key = int(key[0])
    return out


def oracle_ct_split_hull(f, x0_lo, x0_hi, plan, prm, begin=0, end=0):
    return _ct_hull(oracle_lib(), "orc_", f, x0_lo, x0_hi, plan, prm, begin, end)


def ref_ct_split_hull(f, x0_lo, x0_hi, plan, prm, begin=0, end=0, threads=0):
    return _ct_hull(ref_lib(), "ref_", f, x0_lo, x0_hi, plan, prm, begin, end, threads)



# --- forward-dual gradients of the MPC objective (grad_forward) ---------------
def ref_plan_objective_grad(prob, x0, actions):
    """The reference's grad_forward of plan_objective; None where it throws."""
    dp = C.POINTER(C.c_double)
    f = _mpc_fn(ref_lib(), "ref_plan_objective_grad", [C.POINTER(A.NetDesc), C.POINTER(A.PlanProblemC), dp, dp, dp])
    x0 = np.ascontiguousarray(x0, np.float64)
    acts = np.ascontiguousarray(np.asarray(actions, np.float64).reshape(prob.horizon, prob.sys.m))
    g = np.zeros_like(acts)
    desc, keep = prob.sys.step.desc()
    p, keep2 = prob.c_struct()
    rc = f(C.byref(desc), C.byref(p), A.dptr(x0), A.dptr(acts), A.dptr(g))
    return None if rc else g


def ref_plan_cem_ex(prob, cfg, x0):
    dp, ip = C.POINTER(C.c_double), C.POINTER(C.c_int32)
    f = _mpc_fn(ref_lib(), "ref_plan_cem_ex", [C.POINTER(A.NetDesc), C.POINTER(A.PlanProblemC),
                                               C.POINTER(A.SamplerConfigC), dp, dp, dp, dp, ip, ip])
    x0 = np.ascontiguousarray(x0, np.float64)
    best = np.zeros((prob.horizon, prob.sys.m))
    obj = np.zeros(1)
    hist = np.zeros(cfg.iterations)
    be = np.zeros(1, np.int32)
    rf = np.zeros(1, np.int32)
    desc, keep = prob.sys.step.desc()
    p, keep2 = prob.c_struct()
    c = cfg.c_struct()
    rc = f(C.byref(desc), C.byref(p), C.byref(c), A.dptr(x0), A.dptr(best), A.dptr(obj), A.dptr(hist), A.iptr(be),
           A.iptr(rf))
    assert rc == 0, rc
    return best, float(obj[0]), hist, bool(be[0]), bool(rf[0])


def ref_grad_tube_volume(sys, x0, actions, target, method=0, prm=DTReachParams()):
    """The reference's grad_tube_volume -> (g, subgradient), or None where it throws."""
    dp, ip = C.POINTER(C.c_double), C.POINTER(C.c_int32)
    f = _mpc_fn(ref_lib(), "ref_grad_tube_volume", [C.POINTER(A.NetDesc), C.POINTER(A.DTArgs), C.c_int32, C.c_int32,
                                                   dp, ip])
    lo = np.ascontiguousarray(x0[0], np.float64)
    hi = np.ascontiguousarray(x0[1], np.float64)
    H = len(actions)
    acts = np.ascontiguousarray(np.asarray(actions, np.float64).reshape(H * sys.m)) if H * sys.m else np.zeros(1)
    dim = {0: sys.n, 1: H * sys.m, 2: sys.step.params().size}[int(target)]
    g = np.zeros(max(dim, 1))
    sub = np.zeros(1, np.int32)
    desc, keep = sys.step.desc()
    args = A.DTArgs(1, H, sys.n, sys.m, prm.window, int(prm.rebuild_from_box), A.dptr(lo), A.dptr(hi), A.dptr(acts), 0)
    rc = f(C.byref(desc), C.byref(args), int(target), int(method), A.dptr(g), A.iptr(sub))
    return None if rc else (g[:dim], bool(sub[0]))


def ref_mpc_run(prob, sampler, cfg, x0):
    """The reference's mpc_run with the model as simulator -> (success, violated, steps_used, final_state, csv)."""
    dp, ip = C.POINTER(C.c_double), C.POINTER(C.c_int32)
    f = _mpc_fn(ref_lib(), "ref_mpc_run", [C.POINTER(A.NetDesc), C.POINTER(A.PlanProblemC),
                                           C.POINTER(A.SamplerConfigC), C.POINTER(A.MPCConfigC), dp, ip, ip, ip, dp,
                                           C.c_char_p, C.c_int32])
    x0 = np.ascontiguousarray(x0, np.float64)
    succ, viol, used = (np.zeros(1, np.int32) for _ in range(3))
    fin = np.zeros(prob.sys.n)
    buf = C.create_string_buffer(1 << 20)
    gd = np.ascontiguousarray(cfg.goal_dims, dtype=np.int32) if cfg.goal_dims else np.zeros(1, np.int32)
    mc = A.MPCConfigC(cfg.replan_period, cfg.total_steps, cfg.dist_action, cfg.dist_state, len(cfg.goal_dims),
                      A.iptr(gd), cfg.goal_radius, cfg.seed)
    desc, keep = prob.sys.step.desc()
    p, keep2 = prob.c_struct()
    sc = sampler.c_struct()
    rc = f(C.byref(desc), C.byref(p), C.byref(sc), C.byref(mc), A.dptr(x0), A.iptr(succ), A.iptr(viol), A.iptr(used),
           A.dptr(fin), buf, len(buf))
    assert rc == 0, rc
    return bool(succ[0]), bool(viol[0]), int(used[0]), fin, buf.value.decode()


def ref_refine_tube_volume(sys, center, eps, actions, target, lo, hi, iters=20, x=None):
    """The reference's gradient_refine of the CLI refine objective -> RefineResult-like tuple, or None."""
    dp, ip = C.POINTER(C.c_double), C.POINTER(C.c_int32)
    f = _mpc_fn(ref_lib(), "ref_refine_tube_volume", [C.POINTER(A.NetDesc), C.c_int32, C.c_int32, C.c_int32, dp,
                                                     C.c_double, dp, C.c_int32, dp, dp, C.c_int32, dp, dp, dp, ip,
                                                     ip, ip])
    c = np.ascontiguousarray(center, np.float64)
    H = len(actions)
    acts = np.ascontiguousarray(np.asarray(actions, np.float64).reshape(H * sys.m)) if H * sys.m else np.zeros(1)
    d = sys.n if int(target) == 0 else H * sys.m
    xv = np.ascontiguousarray(c if x is None and int(target) == 0 else (acts[:d] if x is None else x),
                              np.float64).copy()
    lo = np.ascontiguousarray(lo, np.float64)
    hi = np.ascontiguousarray(hi, np.float64)
    f0, f1 = np.zeros(1), np.zeros(1)
    pr, sb, ac = (np.zeros(1, np.int32) for _ in range(3))
    desc, keep = sys.step.desc()
    rc = f(C.byref(desc), sys.n, sys.m, H, A.dptr(c), float(eps), A.dptr(acts), int(target), A.dptr(lo), A.dptr(hi),
           int(iters), A.dptr(xv), A.dptr(f0), A.dptr(f1), A.iptr(pr), A.iptr(sb), A.iptr(ac))
    if rc:
        return None
    return xv, float(f0[0]), float(f1[0]), bool(pr[0]), bool(sb[0]), int(ac[0])


def ref_reach_loss(model, x0s, actions, eps, cap, prm=DTReachParams(), with_grad=False):
    """The reference's reach_loss (+ grad_forward over net_params) -> (loss, grad or None, diverged_count)."""
    dp, ip = C.POINTER(C.c_double), C.POINTER(C.c_int32)
    f = _mpc_fn(ref_lib(), "ref_reach_loss", [C.POINTER(A.NetDesc), C.c_int32, C.c_int32, C.c_int32, C.c_int32, dp,
                                             dp, C.c_double, C.c_double, C.c_int32, C.c_int32, dp, dp, ip])
    x0s = np.ascontiguousarray(x0s, np.float64)
    acts = np.ascontiguousarray(actions, np.float64)
    M, n = x0s.shape
    t_h, m = acts.shape[1], acts.shape[2]
    loss = np.zeros(1)
    dc = np.zeros(1, np.int32)
    g = np.zeros(model.params().size) if with_grad else None
    desc, keep = model.desc()
    rc = f(C.byref(desc), n, m, t_h, M, A.dptr(x0s), A.dptr(acts if acts.size else np.zeros(1)), float(eps),
           float(cap), prm.window, int(prm.rebuild_from_box), A.dptr(loss), A.dptr(g) if with_grad else None,
           A.iptr(dc))
    assert rc == 0, rc
    return float(loss[0]), g, int(dc[0])


def ref_dt_interval_baseline_batch(sys, x0_lo, x0_hi, actions):
    f = _mpc_fn(ref_lib(), "ref_dt_interval_baseline_batch", [C.POINTER(A.NetDesc), C.POINTER(A.DTArgs),
                                                              C.POINTER(A.TubeOut)])
    x0_lo = np.ascontiguousarray(x0_lo, np.float64)
    x0_hi = np.ascontiguousarray(x0_hi, np.float64)
    acts = np.ascontiguousarray(actions, np.float64)
    B, H = x0_lo.shape[0], acts.shape[1]
    out = TubeBatch(np.full((B, H + 1, sys.n), np.nan), np.full((B, H + 1, sys.n), np.nan),
                    np.zeros(B, np.int32), np.zeros(B, np.int32), np.zeros(B, np.int32))
    desc, keep = sys.step.desc()
    args = A.DTArgs(B, H, sys.n, sys.m, 0, 0, A.dptr(x0_lo), A.dptr(x0_hi), A.dptr(acts if acts.size else np.zeros(1)),
                    0)
    to = A.TubeOut(A.dptr(out.lo), A.dptr(out.hi), A.iptr(out.n_boxes), A.iptr(out.failed_step), A.iptr(out.status))
    assert f(C.byref(desc), C.byref(args), C.byref(to)) == 0
    return out


def ref_ctl_reach_loss(spec, x0s, yrefs, eps, t_h, delta, cap, with_grad=False):
    """The reference's ctl_reach_loss (quadrotor plant, fp_base = spec.fp) -> (loss, diverged_count), or
    with_grad -> (loss, grad_forward over the controller's net_params, diverged_count)."""
    dp, ip = C.POINTER(C.c_double), C.POINTER(C.c_int32)
    name = "ref_ctl_reach_loss_grad" if with_grad else "ref_ctl_reach_loss"
    f = _mpc_fn(ref_lib(), name, [C.POINTER(A.NetDesc), C.POINTER(A.CLSpecC), C.c_int32, dp, dp, ip,
                                  C.c_int32, C.c_double, C.c_int32, C.c_double, C.c_double, dp]
                + ([dp] if with_grad else []) + [ip])
    x0s = np.ascontiguousarray(x0s, np.float64)
    M = x0s.shape[0]
    has = np.array([0 if y is None else 1 for y in yrefs], np.int32)
    rd = max([np.asarray(y).shape[-1] for y in yrefs if y is not None] or [1])
    yr = np.zeros((M, t_h, rd))
    for e, y in enumerate(yrefs):
        if y is not None:
            yr[e] = np.asarray(y, np.float64).reshape(t_h, rd)
    loss = np.zeros(1)
    dc = np.zeros(1, np.int32)
    desc, keep = spec.controller.desc()
    cs, keep2 = spec.c_struct()
    g = np.zeros(spec.controller.params().size) if with_grad else None
    rc = f(C.byref(desc), C.byref(cs), M, A.dptr(x0s), A.dptr(yr), A.iptr(has), rd, float(eps), t_h, float(delta),
           float(cap), A.dptr(loss), *([A.dptr(g)] if with_grad else []), A.iptr(dc))
    assert rc == 0, rc
    return (float(loss[0]), g, int(dc[0])) if with_grad else (float(loss[0]), int(dc[0]))


# --- certified training (training.hpp) through the reference itself -------------------------------
def ref_pred_loss(model, batch, t_h, weights, with_grad=False):
    from paper_2605_25346_b200.api import _episode_set
    es, keep = _episode_set(batch)
    d, keep2 = model.desc()
    w = np.ascontiguousarray(weights, np.float64)
    loss = np.zeros(1)
    g = np.zeros(model.params().size) if with_grad else None
    f = ref_lib().ref_pred_loss
    f.argtypes = [C.POINTER(A.NetDesc), C.POINTER(A.EpisodeSetC), C.c_int32, C.POINTER(C.c_double),
                  C.POINTER(C.c_double), C.POINTER(C.c_double)]
    f.restype = C.c_int
    rc = f(C.byref(d), C.byref(es), int(t_h), A.dptr(w), A.dptr(loss), A.dptr(g) if with_grad else None)
    assert rc == 0, rc
    return (float(loss[0]), g) if with_grad else float(loss[0])


def ref_train_dt_dyn(init, cfg, dataset):
    """(trained net_params, [TrainLogRow], rc) of the reference's train_dt_dyn."""
    from paper_2605_25346_b200.api import TrainLogRow, _episode_set
    es, keep = _episode_set(dataset)
    d, keep2 = init.desc()
    out = np.zeros(init.params().size)
    log = (A.TrainLogRowC * max(cfg.iters, 1))()
    nrows = np.zeros(1, np.int32)
    f = ref_lib().ref_train_dt_dyn
    f.argtypes = [C.POINTER(A.NetDesc), C.POINTER(A.TrainConfigC), C.POINTER(A.EpisodeSetC), C.POINTER(C.c_double),
                  C.POINTER(A.TrainLogRowC), C.POINTER(C.c_int32)]
    f.restype = C.c_int
    cc = cfg.c()
    rc = f(C.byref(d), C.byref(cc), C.byref(es), A.dptr(out), log, A.iptr(nrows))
    rows = [TrainLogRow(r.iter, r.t_h, r.eps, r.l_pred, r.l_reach, r.l_total, r.diverged_count)
            for r in list(log)[:int(nrows[0])]]
    return out, rows, rc


def ref_track_loss(controller, batch, t_t, weights, gamma, delta, rk4=4, cap=1e6, plant=None, with_grad=False):
    from paper_2605_25346_b200.api import QuadrotorParams, _episode_set
    es, keep = _episode_set(batch)
    d, keep2 = controller.desc()
    qp = np.ascontiguousarray((plant or QuadrotorParams()).as_array(), np.float64)
    w = np.ascontiguousarray(weights, np.float64)
    loss = np.zeros(1)
    bc = np.zeros(1, np.int32)
    g = np.zeros(controller.params().size) if with_grad else None
    dp = C.POINTER(C.c_double)
    f = ref_lib().ref_track_loss
    f.argtypes = [C.POINTER(A.NetDesc), dp, C.POINTER(A.EpisodeSetC), C.c_int32, dp, C.c_double, C.c_double,
                  C.c_int32, C.c_double, dp, dp, C.POINTER(C.c_int32)]
    f.restype = C.c_int
    rc = f(C.byref(d), A.dptr(qp), C.byref(es), int(t_t), A.dptr(w), float(gamma), float(delta), int(rk4), float(cap),
           A.dptr(loss), A.dptr(g) if with_grad else None, A.iptr(bc))
    assert rc == 0, rc
    return (float(loss[0]), g, int(bc[0])) if with_grad else (float(loss[0]), int(bc[0]))


def ref_train_ct_ctl(init, cfg, dataset, delta, k_atomic=1, rk4=4, fp_base=None):
    """(trained net_params, [TrainLogRow], rc) of the reference's train_ct_ctl with the quadrotor plant."""
    import dataclasses as _dc
    from paper_2605_25346_b200.api import ClosedLoopSpec, FlowpipeParams, TrainLogRow, _episode_set
    es, keep = _episode_set(dataset)
    r = len(dataset[0].y_ref[0]) if len(dataset[0].y_ref) else 0
    base = ClosedLoopSpec(init, ctl_steps=1, k_atomic=k_atomic, y_ref=np.zeros((1, r)) if r else None,
                          fp=_dc.replace(fp_base or FlowpipeParams()))
    cs, keep2 = base.c_struct()
    d, keep3 = init.desc()
    out = np.zeros(init.params().size)
    log = (A.TrainLogRowC * max(cfg.iters, 1))()
    nrows = np.zeros(1, np.int32)
    f = ref_lib().ref_train_ct_ctl
    f.argtypes = [C.POINTER(A.NetDesc), C.POINTER(A.TrainConfigC), C.POINTER(A.EpisodeSetC), C.POINTER(A.CLSpecC),
                  C.c_double, C.c_int32, C.POINTER(C.c_double), C.POINTER(A.TrainLogRowC), C.POINTER(C.c_int32)]
    f.restype = C.c_int
    cc = cfg.c()
    rc = f(C.byref(d), C.byref(cc), C.byref(es), C.byref(cs), float(delta), int(rk4), A.dptr(out), log, A.iptr(nrows))
    rows = [TrainLogRow(q.iter, q.t_h, q.eps, q.l_pred, q.l_reach, q.l_total, q.diverged_count)
            for q in list(log)[:int(nrows[0])]]
    return out, rows, rc
