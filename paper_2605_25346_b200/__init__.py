"""B200-native batched reachability primitive (DiffReach DT path).

Public API mirrors the reference's C++ (see api.py); compute runs only in
the in-tree CUDA library libreach_b200.so via the C ABI in include/reach_b200.h.
"""
from .api import (  # noqa: F401
    Act, Layer, MLPNet, affine_net, DTSystem, DTReachParams, ReachTube, TubeBatch, HullResult,
    SplitPlan, split_box, dt_reach, dt_reach_batch, dt_reach_batch_arrays, reach_split_hull,
    reach_with_splitting, tube_volume, box_volume_proxy, box_from_center, dt_closed_loop_batch,
    QuadrotorParams, FlowpipeParams, ClosedLoopSpec, cl_reach, cl_reach_batch_arrays, cl_split_hull,
    cl_reach_with_splitting, AnalyticField, zero_field, diag_linear_field, rotation_field, quadrotor_field,
    quadrotor_hover_input, ct_reach, ct_reach_batch_arrays, ct_split_hull, ct_reach_with_splitting,
    GradTarget, GradMethod, Gradient, grad_tube_volume, RefineResult, refine_tube_volume, Episode, reach_loss, ctl_reach_loss,
)
from ._native import Context, default_context, ReachError, NativeMissing, NonFiniteError, LIB_PATH  # noqa: F401
