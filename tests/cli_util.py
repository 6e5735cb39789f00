"""Helpers for the CLI tests: run `python -m paper_2605_25346_b200.cli` in a subprocess, golden files."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden", "affine_decay.json")


def run_cli(args, cwd):
    env = dict(os.environ)
    env["PYTHONPATH"] = ROOT + os.pathsep + env.get("PYTHONPATH", "")
    r = subprocess.run([sys.executable, "-m", "paper_2605_25346_b200.cli"] + args, cwd=cwd, env=env,
                       capture_output=True, text=True, timeout=600)
    return r.returncode


def golden_net(tmp):
    """The reference's data/affine_decay_net.json (re-encoded in the fixture) written to tmp."""
    d = json.load(open(GOLDEN))
    p = os.path.join(tmp, "affine_decay_net.json")
    with open(p, "w") as f:
        json.dump({"layers": d["layers"]}, f)
    return p


def golden_csv():
    """data/affine_decay_golden.csv byte for byte (tube_to_csv(tube, false) of the reference)."""
    e = json.load(open(GOLDEN))["expected_csv_text"]
    keys = sorted(e, key=lambda k: (int(k.split(",")[0]), int(k.split(",")[1])))
    return "step,dim,lo,hi\n" + "".join(f"{k},{e[k][0]},{e[k][1]}\n" for k in keys)


def read(path):
    with open(path, newline="") as f:
        return f.read()
