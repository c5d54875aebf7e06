"""bench.py --gpus N starts N ranks itself (torch.distributed.run on
127.0.0.1) and every rank sees the world: checked on CPU with the gloo dry
run (the driver's torchrun launch sets WORLD_SIZE and skips the relaunch)."""

import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_gpus2_launches_two_ranks():
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--gpus", "2", "--dry-run"],
                         capture_output=True, text=True, timeout=300, cwd=REPO)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2
    assert [r[0] for r in line["ranks"]] == [0, 1]
    # contiguous row shards covering the database
    assert line["ranks"][0][2] == 0 and line["ranks"][0][3] == line["ranks"][1][2]
    assert line["ranks"][1][3] == 1_000_000


def test_bench_world_mismatch_is_an_error():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--gpus", "2", "--dry-run"],
                         capture_output=True, text=True, timeout=300, cwd=REPO, env=env)
    assert out.returncode != 0
