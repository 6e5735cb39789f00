"""GPU: the CLI end to end on the device engines (test_cli.cpp): the bundled affine example reproduces the
reference's golden CSV byte for byte, manifest reruns are byte-identical, divergence exits 5 with the
flagged tube written, splitting tightens the hull, the mpc subcommand reaches its goal, and `refine`
equals the reference's gradient_refine."""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from cli_util import golden_csv, golden_net, read, run_cli
from oracle_bind import ref_available, ref_refine_tube_volume
from paper_2605_25346_b200 import formats as F
from paper_2605_25346_b200.api import DTSystem, affine_net, tube_volume
from paper_2605_25346_b200.mpc import Constraint, MPCConfig, PlanProblem, SamplerConfig


def test_golden_csv_byte_for_byte(tmp_path):
    out = str(tmp_path / "g")
    net = golden_net(str(tmp_path))
    assert run_cli(["reach-dt", "--net", net, "--x0-center", "0.5,0.5", "--eps", "0.125", "--steps", "8", "--out",
                    out], str(tmp_path)) == 0
    assert read(os.path.join(out, "tube.csv")) == golden_csv()


@pytest.mark.parametrize("kind", ["ct_split", "dt"])
def test_rerun_from_manifest_is_byte_identical(tmp_path, kind):
    a, b = str(tmp_path / "a"), str(tmp_path / "b")
    if kind == "ct_split":
        args = ["reach-ct", "--system", "rotation", "--x0-center", "1,0", "--eps", "0.05", "--h", "0.05", "--steps",
                "12", "--split", "2x2", "--seed", "5", "--out", a]
    else:
        args = ["reach-dt", "--net", golden_net(str(tmp_path)), "--x0-center", "0.5,0.5", "--eps", "0.125", "--steps",
                "8", "--out", a]
    assert run_cli(args, str(tmp_path)) == 0
    assert run_cli(["rerun", "--manifest", os.path.join(a, "manifest.json"), "--out", b], str(tmp_path)) == 0
    for f in ("tube.csv", "tube.json", "manifest.json"):
        assert read(os.path.join(a, f)) == read(os.path.join(b, f))


def test_divergence_exits_5_and_writes_flagged_tube(tmp_path):
    out = str(tmp_path / "div")
    assert run_cli(["reach-ct", "--system", "decay", "--x0-center", "1", "--eps", "0.01", "--h", "5.0", "--steps",
                    "60", "--out", out], str(tmp_path)) == 5
    t = F.tube_from_json(json.loads(read(os.path.join(out, "tube.json"))))
    assert t.diverged


def test_split_tightens_the_hull(tmp_path):
    plain, split = str(tmp_path / "p"), str(tmp_path / "s")
    base = ["reach-ct", "--system", "rotation", "--x0-center", "1,0", "--eps", "0.1", "--h", "0.05", "--steps", "20"]
    assert run_cli(base + ["--out", plain], str(tmp_path)) == 0
    assert run_cli(base + ["--split", "3x3", "--out", split], str(tmp_path)) == 0
    tp = F.tube_from_json(json.loads(read(os.path.join(plain, "tube.json"))))
    ts = F.tube_from_json(json.loads(read(os.path.join(split, "tube.json"))))
    assert tp.steps() == ts.steps() and tube_volume(ts) <= tube_volume(tp)
    assert np.all(ts.lo[-1] >= tp.lo[-1] - 1e-12) and np.all(ts.hi[-1] <= tp.hi[-1] + 1e-12)


def test_mpc_subcommand_reaches_goal_and_reruns(tmp_path):
    """test_cli.cpp:144-193: scenario written through the serializer, consumed by the CLI."""
    w = np.zeros((2, 4))
    w[0, 0] = w[1, 1] = w[0, 2] = w[1, 3] = 1.0
    prob = PlanProblem(DTSystem(affine_net(w, np.zeros(2)), 2, 2), np.array([0.8, 0.5]), np.ones(2),
                       np.full(2, 0.01), [Constraint(type=Constraint.BOX_STAY_IN, lo=np.full(2, -2.0),
                                                     hi=np.full(2, 2.0))],
                       horizon=5, u_lo=np.full(2, -0.3), u_hi=np.full(2, 0.3), eps=0.02)
    sc = SamplerConfig(population=64, iterations=3, seed=11)
    mc = MPCConfig(total_steps=20, goal_radius=0.1, seed=11)
    scen = str(tmp_path / "scenario.json")
    F.write_json_file(scen, F.scenario_to_json(prob, sc, mc))
    out, out2 = str(tmp_path / "mpc"), str(tmp_path / "mpc2")
    assert run_cli(["mpc", "--scenario", scen, "--x0-center", "0,0", "--out", out], str(tmp_path)) == 0
    res = json.loads(read(os.path.join(out, "result.json")))
    assert res["success"] is True and res["violated"] is False
    log = read(os.path.join(out, "run_log.csv"))
    assert log.count("\n") == res["steps_used"] + 1
    assert run_cli(["rerun", "--manifest", os.path.join(out, "manifest.json"), "--out", out2], str(tmp_path)) == 0
    for f in ("run_log.csv", "result.json"):
        assert read(os.path.join(out, f)) == read(os.path.join(out2, f))


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")
def test_refine_subcommand_matches_reference(tmp_path):
    from paper_2605_25346_b200.workloads import random_mlp
    from paper_2605_25346_b200.api import Act
    rng = np.random.default_rng(3)
    net = random_mlp(rng, 4, [16, 16], 2, Act.Relu, 0.6)
    p = str(tmp_path / "net.json")
    F.write_json_file(p, F.net_to_json(net))
    out = str(tmp_path / "rf")
    for target in ("center", "actions"):
        assert run_cli(["refine", "--net", p, "--x0-center", "0.1,-0.2", "--eps", "0.05", "--steps", "6",
                        "--grad-iters", "5", "--target", target, "--out", out], str(tmp_path)) == 0
        rj = json.loads(read(os.path.join(out, "refine.json")))
        sys_ = DTSystem(net, 2, 2)
        c = np.array([0.1, -0.2])
        acts = [[0.0, 0.0]] * 6
        x = c if target == "center" else np.zeros(12)
        exp = ref_refine_tube_volume(sys_, c, 0.05, acts, 0 if target == "center" else 1, x - 0.5, x + 0.5, 5, x)
        assert rj["x"] == list(exp[0]) and rj["objective"] == exp[2] and rj["accepted_steps"] == exp[5]


@pytest.mark.parametrize("precision", ["fused", "tc"])
def test_reach_dt_precision_modes(tmp_path, precision):
    """reach-dt --precision fused|tc: the golden example within rtol 1e-5 of the exact tube; the manifest
    records the mode, and a rerun reproduces it byte for byte."""
    a, b = str(tmp_path / "a"), str(tmp_path / "b")
    args = ["reach-dt", "--net", golden_net(str(tmp_path)), "--x0-center", "0.5,0.5", "--eps", "0.125", "--steps", "8",
            "--precision", precision, "--out", a]
    assert run_cli(args, str(tmp_path)) == 0
    got = np.array([[float(v) for v in line.split(",")] for line in read(os.path.join(a, "tube.csv")).splitlines()[1:]])
    exp = np.array([[float(v) for v in line.split(",")] for line in golden_csv().splitlines()[1:]])
    assert got.shape == exp.shape
    assert float(np.max(np.abs(got - exp))) <= 1e-5 * float(np.max(np.abs(exp)))
    assert json.loads(read(os.path.join(a, "manifest.json")))["config"]["precision"] == precision
    assert run_cli(["rerun", "--manifest", os.path.join(a, "manifest.json"), "--out", b], str(tmp_path)) == 0
    assert read(os.path.join(a, "tube.csv")) == read(os.path.join(b, "tube.csv"))
