"""GPU: dt_interval_baseline (dt_reach.hpp:129-149) on the device against the reference (oracle/_ref):
bit-identical tubes for ReLU / identity maps (incl. the diverged-box failure), wider than the certified
dt_reach tube, and the CLI's `reach-dt --baseline interval`."""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from cases import cases
from cli_util import golden_net, read, run_cli
from oracle_bind import assert_tubes_equal, ref_available, ref_dt_interval_baseline_batch
from paper_2605_25346_b200 import formats as F
from paper_2605_25346_b200.api import (DTSystem, affine_net, dt_interval_baseline_batch_arrays, dt_reach_batch_arrays,
                                       tube_volume)

needs_ref = pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")


@needs_ref
@pytest.mark.parametrize("case", [c for c in cases() if "tanh" not in c[0]][:6], ids=lambda c: c[0])
def test_interval_baseline_matches_reference(case):
    name, sys_, lo, hi, acts, prm, _ = case
    exp = ref_dt_interval_baseline_batch(sys_, lo, hi, acts)
    got = dt_interval_baseline_batch_arrays(sys_, lo, hi, acts)
    assert_tubes_equal(got, exp, exact=True)


@needs_ref
def test_interval_baseline_diverged_box_failure():
    sys_ = DTSystem(affine_net(np.eye(2) * 1e200, np.zeros(2)), 2, 0)
    lo, hi = np.full((3, 2), -0.1), np.full((3, 2), 0.1)
    acts = np.zeros((3, 6, 0))
    exp = ref_dt_interval_baseline_batch(sys_, lo, hi, acts)
    got = dt_interval_baseline_batch_arrays(sys_, lo, hi, acts)
    assert np.all(got.status == 3) and np.array_equal(got.failed_step, exp.failed_step)
    assert_tubes_equal(got, exp, exact=True)


def test_baseline_is_wider_than_the_certified_tube():
    name, sys_, lo, hi, acts, prm, _ = [c for c in cases() if "tanh" not in c[0]][0]
    b = dt_interval_baseline_batch_arrays(sys_, lo, hi, acts).tubes()
    c = dt_reach_batch_arrays(sys_, lo, hi, acts, prm).tubes()
    for tb, tc in zip(b, c):
        if not tb.diverged and not tc.diverged:
            assert tube_volume(tc) <= tube_volume(tb)


def test_cli_reach_dt_interval_baseline(tmp_path):
    out = str(tmp_path / "bl")
    net = golden_net(str(tmp_path))
    assert run_cli(["reach-dt", "--net", net, "--x0-center", "0.5,0.5", "--eps", "0.125", "--steps", "8",
                    "--baseline", "interval", "--out", out], str(tmp_path)) == 0
    t = F.tube_from_csv(read(os.path.join(out, "tube.csv")))
    assert t.steps() == 9
    manifest = json.loads(read(os.path.join(out, "manifest.json")))
    assert manifest["config"]["baseline"] == "interval"
