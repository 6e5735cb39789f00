"""GPU: the reference's own C++ types and workloads through the drop-in
overloads of include/reach_b200_reference.hpp (tests/cpp), bit-compared with
the reference's dt_reach / reach_with_splitting in the same binary."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

BIN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "test_reference_dropin")


@pytest.mark.skipif(not os.path.exists(BIN), reason="tests/cpp/test_reference_dropin not built (needs /root/reference)")
def test_reference_types_dropin_bit_exact():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "OK: reference drop-in parity" in r.stdout
