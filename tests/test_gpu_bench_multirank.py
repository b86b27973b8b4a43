"""bench.py at --gpus 2 on a one-GPU box (MPSF_BENCH_ONE_GPU=1: both ranks on cuda:0 over
gloo): the self-launch, the sharded weak-scaling headline, the strong-scaling config-5 extra
and the sharded config-3 storm (dense slots + sparse exchange of the page-sized tables), each
checked against the C oracle on the whole batch by rank 0."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_two_ranks_parity():
    env = dict(os.environ, MPSF_BENCH_ONE_GPU="1")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3", "--warmup", "3",
                        "--entries", "300000", "--storm-n", "3000000", "--no-remap", "--no-e2e"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=1500)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    line = lines[0]
    assert line["n_gpus"] == 2
    assert line["parity"].startswith("bit-exact"), line["parity"]
    assert line["extra"]["strong_c5"]["parity"].startswith("bit-exact"), line["extra"]["strong_c5"]
    assert line["extra"]["storm_c3"]["parity"].startswith("bit-exact"), line["extra"]["storm_c3"]
    assert line["extra"]["storm_c3"]["dedup_count_exact"]
