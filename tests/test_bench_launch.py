"""bench.py's launcher: ``--gpus N`` without a torchrun environment re-executes the script
under torch.distributed.run with N ranks on 127.0.0.1 (the driver's own launch form), and a
rank count that disagrees with ``--gpus`` is refused instead of silently reporting 1 GPU."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_gpus_n_self_launches_n_ranks():
    env = dict(os.environ, MPSF_BENCH_LAUNCH_PROBE="1")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "3", "--n", "1000"], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert sorted(x["rank"] for x in lines) == [0, 1, 2], r.stdout
    assert all(x["world_size"] == 3 and x["master_addr"] == "127.0.0.1" for x in lines)
    assert sorted(x["local_rank"] for x in lines) == [0, 1, 2]


def test_gpus_mismatch_with_world_size_is_refused():
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "4", "--no-storm"], cwd=ROOT,
                       env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode != 0
    assert "--gpus 4 but WORLD_SIZE=2" in (r.stderr + r.stdout)
