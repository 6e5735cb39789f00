"""CPU: the C-ABI library loads and exports every symbol include/*.h declares;
host-side validation and plan logic (no compute calls without a GPU)."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

from paper_2605_25346_b200 import _abi as A
from paper_2605_25346_b200 import LIB_PATH
from paper_2605_25346_b200.api import DTSystem, SplitPlan, affine_net, split_box

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "reach_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?(?:int|int64_t|char)\s*\*?\s*(reach_\w+)\s*\(", src, flags=re.M)))


def test_header_declares_entry_points():
    names = declared_functions()
    for f in ("reach_ctx_create", "reach_net_upload", "reach_dt_batch", "reach_split_hull", "reach_abi_version"):
        assert f in names


@pytest.mark.skipif(not os.path.exists(LIB_PATH), reason="libreach_b200.so not built")
def test_library_exports_every_declared_symbol():
    out = subprocess.run(["nm", "-D", "--defined-only", LIB_PATH], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r" T (\w+)", out))
    missing = [f for f in declared_functions() if f not in exported]
    assert not missing, missing


@pytest.mark.skipif(not os.path.exists(LIB_PATH), reason="libreach_b200.so not built")
def test_library_loads_and_reports_abi_without_gpu():
    lib = C.CDLL(LIB_PATH)
    assert lib.reach_abi_version() == 1
    lib.reach_tube_status_string.restype = C.c_char_p
    assert lib.reach_tube_status_string(3) == b"diverged box"
    assert lib.reach_tube_status_string(1) == b"relax_activation: non-finite preactivation"
    # context creation must fail cleanly (not crash) when no device is visible
    import torch
    if not torch.cuda.is_available():
        h = C.c_void_p()
        lib.reach_ctx_create.argtypes = [C.c_int32, C.POINTER(C.c_void_p)]
        assert lib.reach_ctx_create(0, C.byref(h)) == A.REACH_E_NO_DEVICE


def test_struct_layouts():
    # field offsets of the ctypes mirror follow the C layout of the header
    assert C.sizeof(A.NetDesc) == 32
    assert A.DTArgs.x0_lo.offset == 24 and A.DTArgs.actions_shared.offset == 48
    assert A.SplitArgs.part_begin.offset == 56 and C.sizeof(A.SplitArgs) == 72
    assert C.sizeof(A.HullOut) == 40


def test_dt_system_validation_mirrors_reference():
    sys = DTSystem(affine_net(np.eye(2), np.zeros(2)), 3, 0)
    with pytest.raises(ValueError, match="shape mismatch"):
        sys.validate()
    with pytest.raises(ValueError, match="invalid dimensions"):
        DTSystem(affine_net(np.eye(2), np.zeros(2)), 0, 0).validate()


def test_split_plan_and_split_box():
    assert SplitPlan.parse("8x8x4").counts == [8, 8, 4]
    with pytest.raises(ValueError):
        SplitPlan.parse("8xx4")
    with pytest.raises(ValueError):
        SplitPlan([1 << 11, 1 << 10]).total_parts()
    p = SplitPlan.rpy(12, 4096)
    assert p.counts[6:9] == [16, 16, 16] and p.total_parts() == 4096
    lo, hi = split_box(np.array([0.0, -1.0]), np.array([1.0, 1.0]), SplitPlan([3, 2]))
    assert lo.shape == (6, 2)
    # last dim fastest, exact shared edges, exact outer endpoints
    assert hi[0, 1] == lo[1, 1] and lo[0, 0] == 0.0 and hi[-1, 0] == 1.0 and hi[-1, 1] == 1.0
    assert lo[2, 0] == hi[0, 0]


def test_fail_key_codec():
    key = (7 << 40) | (12345 << 8) | 3
    assert A.decode_fail_key(key) == (7, 12345, 3)
    assert A.decode_fail_key(A.FAIL_KEY_NONE) is None
