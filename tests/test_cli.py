"""CPU: the CLI's exit-code classes that need no device (test_cli.cpp:51-72) and the formats
(io.hpp: %.17g CSV round trip, tube / net JSON, nlohmann-style dump)."""
import math
import os

import numpy as np

from cli_util import golden_net, run_cli
from paper_2605_25346_b200 import formats as F
from paper_2605_25346_b200.api import Act, Layer, MLPNet, ReachTube


def test_dimension_mismatch_exits_3_and_writes_nothing(tmp_path):
    out = str(tmp_path / "dim")
    net = golden_net(str(tmp_path))
    assert run_cli(["reach-dt", "--net", net, "--x0-center", "0.5,0.5,0.5", "--out", out], str(tmp_path)) == 3
    assert run_cli(["reach-ct", "--system", "rotation", "--x0-center", "1,0,0", "--out", out], str(tmp_path)) == 3
    assert not os.path.exists(out)


def test_config_errors_exit_2(tmp_path):
    out = str(tmp_path / "cfg")
    cwd = str(tmp_path)
    assert run_cli(["reach-dt", "--net", "no_such_file.json", "--x0-center", "0,0", "--out", out], cwd) == 2
    assert run_cli(["reach-ct", "--system", "no-such-system", "--x0-center", "0", "--out", out], cwd) == 2
    assert run_cli(["reach-ct", "--x0-center", "1,0", "--out", out], cwd) == 2  # missing --system
    assert run_cli(["split", "--system", "rotation", "--x0-center", "1,0", "--out", out], cwd) == 2  # no --split
    assert run_cli(["reach-ct", "--system", "swarm", "--x0-center", "0", "--out", out], cwd) == 2  # not on device
    assert not os.path.exists(out)


def test_tube_csv_and_json_round_trip():
    lo = np.array([[0.1, -1e-300], [1.0 / 3.0, -2.5e17]])
    hi = np.array([[0.2, 5e-324], [2.0 / 3.0, math.inf]])
    t = ReachTube(lo, hi, np.array([0.0, 0.0]), np.array([0.0, 0.01]), True, 1, "diverged box")
    for wt in (True, False):
        back = F.tube_from_csv(F.tube_to_csv(t, wt))
        assert np.array_equal(back.lo, lo) and np.array_equal(back.hi, hi)
    j = F.tube_from_json(F.tube_to_json(t))
    assert np.array_equal(j.lo, lo) and j.diverged and j.failed_step == 1 and j.failure_reason == "diverged box"
    assert "null" in F.json_dump(F.tube_to_json(t))  # nlohmann writes non-finite doubles as null
    assert F.fmt_g17(0.1) == "0.10000000000000001" and F.fmt_g17(-0.0) == "-0"


def test_net_json_round_trip_and_dump_format():
    net = MLPNet([Layer(np.array([[0.5, 0.0], [0.0, 0.25]]), np.array([0.25, -0.5]), Act.Identity)])
    d = F.net_to_json(net)
    back = F.net_from_json(d)
    assert np.array_equal(back.layers[0].w, net.layers[0].w) and back.layers[0].act == Act.Identity
    s = F.json_dump(d)
    # nlohmann::json::dump(2) layout: sorted keys, 2-space indent, doubles keep ".0"
    assert s.splitlines()[:4] == ["{", '  "layers": [', "    {", '      "act": "identity",']
    assert '"b": [\n        0.25,\n        -0.5\n      ],' in s and "0.0" in s


def test_net_json_matches_reference_file_bytes():
    """nlohmann dump(2) of the reference's own data/affine_decay_net.json (skipped where it is absent)."""
    import json
    import pytest
    p = "/root/reference/proj/data/affine_decay_net.json"
    if not os.path.exists(p):
        pytest.skip("reference data not present")
    t = open(p).read()
    assert F.json_dump(F.net_to_json(F.net_from_json(json.loads(t)))) + "\n" == t
