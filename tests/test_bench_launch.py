"""CPU: bench.py's multi-rank launcher.  `--gpus N` without torchrun re-execs itself under
torch.distributed.run with N ranks (gloo in the dry run); under torchrun the world size must
equal --gpus.  The dry run exercises the launch, rendezvous and max-over-ranks reduction
without GPU work."""
import json
import os
import subprocess
import sys
import types

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench():
    sys.path.insert(0, ROOT)
    import bench
    return bench


def test_launch_command_shape():
    b = _bench()
    cmd = b.launch_command(["--gpus", "4", "--steps", "2"], 4, 29511)
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--master-addr=127.0.0.1" in cmd and "--master-port=29511" in cmd
    assert cmd[-4:] == ["--gpus", "4", "--steps", "2"]
    assert cmd[-5].endswith("bench.py")


def test_world_must_match_gpus(monkeypatch):
    b = _bench()
    monkeypatch.setenv("WORLD_SIZE", "2")
    with pytest.raises(SystemExit):
        b.ensure_world(types.SimpleNamespace(gpus=4))
    assert b.ensure_world(types.SimpleNamespace(gpus=2)) is None
    monkeypatch.delenv("WORLD_SIZE")
    assert b.ensure_world(types.SimpleNamespace(gpus=1)) is None


def test_self_launch_two_ranks_gloo():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["MASTER_ADDR"] = "127.0.0.1"
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dist-dry-run"],
                       capture_output=True, text=True, timeout=240, env=env, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout
    rec = json.loads(lines[0])
    assert rec["n_gpus"] == 2 and rec["config"]["parallelism"] == "dp2"
    assert rec["max_over_ranks"] == 2.0
