"""ctypes mirror of include/reach_b200.h (the C ABI).

Struct layouts here must match the header field for field; tests/test_abi.py
checks the exported symbols against the header declarations.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

REACH_OK = 0
REACH_E_INVALID_ARGUMENT = 1
REACH_E_CUDA = 2
REACH_E_UNSUPPORTED = 3
REACH_E_NO_DEVICE = 4
REACH_E_OOM = 5
REACH_E_NONFINITE = 6

REACH_FLAG_DEVICE_PTRS = 1
REACH_FLAG_OUTWARD_ROUNDING = 0x10  # the reference's g_outward_rounding: refused (REACH_E_UNSUPPORTED)
REACH_FLAG_PREC_MASK = 0xF00
REACH_PREC_EXACT = 0x000
REACH_PREC_TC = 0x100
REACH_PREC_FUSED = 0x200
PRECISIONS = {"exact": REACH_PREC_EXACT, "tc": REACH_PREC_TC, "fused": REACH_PREC_FUSED}


def prec_flag(precision: str) -> int:
    """Flags bits of a precision mode: "exact" (the reference's arithmetic, bit for bit), "fused" (the
    same kernels with every a*b+c a DFMA; fp64 tolerance mode) or "tc" (CROWN contractions on the
    int8 tensor cores, Ozaki split, rigorous error bound)."""
    try:
        return PRECISIONS[precision]
    except KeyError:
        raise ValueError(f"unknown precision mode {precision!r} (exact | fused | tc)") from None

ACT_RELU, ACT_TANH, ACT_IDENTITY = 0, 1, 2

# reach_tube_status -> reference failure_reason strings (tube.hpp:30-34)
TUBE_OK = 0
TUBE_NONFINITE_PREACT = 1
TUBE_DIVERGED_CERT = 2
TUBE_DIVERGED_BOX = 3
TUBE_CTL_FAILED = 4
TUBE_CTL_DIVERGED = 5
TUBE_REMAINDER = 6
TUBE_PICARD_NONFINITE = 7
TUBE_TME_INV = 8
TUBE_OTHER = 99
TUBE_REASON = {
    TUBE_OK: "",
    TUBE_NONFINITE_PREACT: "relax_activation: non-finite preactivation",
    TUBE_DIVERGED_CERT: "diverged certification",
    TUBE_DIVERGED_BOX: "diverged box",
    TUBE_CTL_FAILED: "controller certification failed: relax_activation: non-finite preactivation",
    TUBE_CTL_DIVERGED: "controller certification diverged",
    TUBE_REMAINDER: "remainder not contractive after max enlargements (reduce h)",
    TUBE_PICARD_NONFINITE: "poly_picard: non-finite coefficients",
    TUBE_TME_INV: "tme_inv: range contains zero",
    TUBE_OTHER: "error",
}

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)
_lp = C.POINTER(C.c_int64)


class NetDesc(C.Structure):
    _fields_ = [("n_layers", C.c_int32), ("dims", _ip), ("acts", _ip), ("params", _dp)]


class DTArgs(C.Structure):
    _fields_ = [
        ("batch", C.c_int32), ("horizon", C.c_int32), ("n", C.c_int32), ("m", C.c_int32),
        ("window", C.c_int32), ("rebuild_from_box", C.c_int32),
        ("x0_lo", _dp), ("x0_hi", _dp), ("actions", _dp), ("actions_shared", C.c_int32),
    ]


class TubeOut(C.Structure):
    _fields_ = [("lo", _dp), ("hi", _dp), ("n_boxes", _ip), ("failed_step", _ip), ("status", _ip)]


class SplitArgs(C.Structure):
    _fields_ = [
        ("n", C.c_int32), ("m", C.c_int32), ("horizon", C.c_int32), ("window", C.c_int32),
        ("rebuild_from_box", C.c_int32),
        ("x0_lo", _dp), ("x0_hi", _dp), ("counts", _ip), ("actions", _dp),
        ("part_begin", C.c_int64), ("part_end", C.c_int64),
    ]


class HullOut(C.Structure):
    _fields_ = [("lo", _dp), ("hi", _dp), ("box_diverged", _ip), ("n_boxes", _ip), ("fail_key", _lp)]


def dptr(a) -> "C._Pointer":
    """Pointer to a C-contiguous float64 numpy array, or a raw device address (int)."""
    if a is None:
        return C.cast(None, _dp)
    if isinstance(a, int):
        return C.cast(C.c_void_p(a), _dp)
    assert a.dtype == np.float64 and a.flags.c_contiguous, (a.dtype, a.flags)
    return a.ctypes.data_as(_dp)


def iptr(a):
    if a is None:
        return C.cast(None, _ip)
    if isinstance(a, int):
        return C.cast(C.c_void_p(a), _ip)
    assert a.dtype == np.int32 and a.flags.c_contiguous
    return a.ctypes.data_as(_ip)


def lptr(a):
    if isinstance(a, int):
        return C.cast(C.c_void_p(a), _lp)
    assert a.dtype == np.int64 and a.flags.c_contiguous
    return a.ctypes.data_as(_lp)


FAIL_KEY_NONE = np.iinfo(np.int64).max


def decode_fail_key(key: int):
    """(div_step, part, status) of a hull fail key, or None."""
    key = int(key)
    if key == FAIL_KEY_NONE:
        return None
    return key >> 40, (key >> 8) & ((1 << 32) - 1), key & 0xFF


# --- MPC (mpc.hpp) -----------------------------------------------------------
CON_HALFSPACE_AVOID, CON_SPHERE_AVOID, CON_BOX_STAY_IN, CON_MAX_VOLUME = 0, 1, 2, 3


class ConstraintC(C.Structure):
    _fields_ = [
        ("type", C.c_int32), ("n_dims", C.c_int32), ("dims", _ip), ("a", _dp), ("b", C.c_double),
        ("center", _dp), ("radius", C.c_double), ("lo", _dp), ("hi", _dp), ("vmax", C.c_double),
    ]


class PlanProblemC(C.Structure):
    _fields_ = [
        ("n", C.c_int32), ("m", C.c_int32), ("horizon", C.c_int32), ("window", C.c_int32),
        ("rebuild_from_box", C.c_int32),
        ("x_goal", _dp), ("q_weights", _dp), ("r_weights", _dp),
        ("n_constraints", C.c_int32), ("constraints", C.POINTER(ConstraintC)),
        ("penalty", C.c_double), ("diverged_margin", C.c_double), ("eps", C.c_double),
        ("u_lo", _dp), ("u_hi", _dp),
    ]


class SamplerConfigC(C.Structure):
    _fields_ = [
        ("population", C.c_int32), ("elite_frac", C.c_double), ("iterations", C.c_int32),
        ("init_std", C.c_double), ("smoothing", C.c_double), ("refine_iters", C.c_int32), ("seed", C.c_uint64),
    ]


class MPCConfigC(C.Structure):
    _fields_ = [
        ("replan_period", C.c_int32), ("total_steps", C.c_int32), ("dist_action", C.c_double),
        ("dist_state", C.c_double), ("n_goal_dims", C.c_int32), ("goal_dims", _ip), ("goal_radius", C.c_double),
        ("seed", C.c_uint64),
    ]


class MPCLogC(C.Structure):
    _fields_ = [("step", _ip), ("state", _dp), ("action", _dp), ("objective", _dp), ("tube_volume", _dp),
                ("g_margin", _dp)]


SIM_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, _dp, _dp, _dp)


# --- continuous-time closed loop (closed_loop.hpp) -----------------------------
PLANT_QUADROTOR = 0


class FlowpipeParamsC(C.Structure):
    _fields_ = [
        ("h", C.c_double), ("steps", C.c_int32), ("order", C.c_int32), ("eps_init", C.c_double),
        ("refine_rounds", C.c_int32), ("enlargement", C.c_double), ("max_enlargements", C.c_int32),
        ("window", C.c_int32),
    ]


class CLSpecC(C.Structure):
    _fields_ = [
        ("plant", C.c_int32), ("plant_params", C.c_double * 8), ("n", C.c_int32), ("l", C.c_int32),
        ("ctl_steps", C.c_int32), ("k_atomic", C.c_int32), ("ref_dim", C.c_int32), ("y_ref", _dp),
        ("fp", FlowpipeParamsC), ("intervalize_boundary", C.c_int32),
    ]


class CLSplitArgs(C.Structure):
    _fields_ = [("x0_lo", _dp), ("x0_hi", _dp), ("counts", _ip), ("part_begin", C.c_int64), ("part_end", C.c_int64)]


FIELD_ZERO, FIELD_DIAG_LINEAR, FIELD_ROTATION, FIELD_QUADROTOR = 0, 1, 2, 3


class FieldDescC(C.Structure):
    _fields_ = [("kind", C.c_int32), ("n", C.c_int32), ("params", C.c_double * 16)]


# ---- multi-GPU collectives (include/reach_b200.h, "Multi-GPU")
REACH_DT_U64, REACH_DT_I32, REACH_DT_F64 = 0, 1, 2
REACH_OP_MIN, REACH_OP_MAX = 0, 1
ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_int32, C.c_int32, C.c_void_p)
ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_int32, C.c_void_p)


class Collectives(C.Structure):
    _fields_ = [("rank", C.c_int32), ("world", C.c_int32), ("allreduce", ALLREDUCE_FN), ("allgather", ALLGATHER_FN),
                ("user", C.c_void_p)]


# --- certified training (training.hpp) --------------------------------------------------------
class EpisodeSetC(C.Structure):
    _fields_ = [("episodes", C.c_int32), ("length", C.c_int32), ("n", C.c_int32), ("m", C.c_int32),
                ("states", _dp), ("actions", _dp), ("ref_dim", C.c_int32), ("y_ref", _dp)]


class TrainConfigC(C.Structure):
    _fields_ = [("horizon_max", C.c_int32), ("eps0", C.c_double), ("eps_final", C.c_double),
                ("lambda_", C.c_double), ("gamma", C.c_double), ("iters", C.c_int32), ("batch", C.c_int32),
                ("lr", C.c_double), ("reach_cap", C.c_double), ("curriculum", C.c_int32), ("seed", C.c_uint64),
                ("window", C.c_int32), ("rebuild_from_box", C.c_int32)]


class TrainLogRowC(C.Structure):
    _fields_ = [("iter", C.c_int32), ("t_h", C.c_int32), ("eps", C.c_double), ("l_pred", C.c_double),
                ("l_reach", C.c_double), ("l_total", C.c_double), ("diverged_count", C.c_int32)]
