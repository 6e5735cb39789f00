"""tcgen05.mma kind::i8 issue/throughput probe (reach_debug_mma_rate).
mode 0: one thread in a divergent branch; 1: converged warp, elect.sync in the asm; 2: one thread,
loop-invariant operands."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_25346_b200 import default_context  # noqa: E402

ctx = default_context()
f = ctx._lib.reach_debug_mma_rate
f.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_double)]
f.restype = C.c_int
for mode in (0, 1, 2):
    for N in (8, 24, 64, 128, 256):
        v = C.c_double()
        ctx.check(f(ctx.handle, 4096, N, (mode << 8) | 1, C.byref(v)), "mma_rate")
        print(f"mode {mode} N={N:3d} {v.value:7.1f} cycles/MMA  -> {128 * N * 32 / v.value:8.0f} MAC/cycle")
