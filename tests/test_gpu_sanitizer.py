"""compute-sanitizer over every kernel family at small sizes (tools/sanitize_target.py): the
fault-path passes (row-table and global-table variants, dense and claimed-slot layouts, the
general path, the sharded phase API and the sparse exchange), the batched translation, the
fold (both paths), the KV pool restore and the remaps.  memcheck (out-of-bounds / misaligned accesses),
racecheck (shared-memory hazards between threads of a CTA: the per-warp queues, the block-local
minima, the staged tables) and synccheck (barrier / __syncwarp misuse) must report 0 errors."""

import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.parametrize("tool,part", [("memcheck", "all"), ("synccheck", "all"),
                                       ("racecheck", "fault"), ("racecheck", "sharded"),
                                       ("racecheck", "translate"), ("racecheck", "fold"),
                                       ("memcheck", "fold_radix"), ("racecheck", "fold_radix"),
                                       ("racecheck", "remap")])
def test_compute_sanitizer_clean(tool, part):
    cmd = [SAN, "--tool", tool, "--error-exitcode", "3", "--print-limit", "20"]
    if tool == "racecheck":
        cmd += ["--racecheck-report", "all"]
    r = subprocess.run(cmd + [sys.executable, os.path.join(ROOT, "tools", "sanitize_target.py"), part], cwd=ROOT,
                       capture_output=True, text=True, timeout=1800)
    out = r.stdout + r.stderr
    if r.returncode == 86 and "closed on this pool" in out:
        # the GPU pool's compute-sanitizer wrapper refuses to run (exit 86); the clean runs of the
        # current kernels are recorded in profiles/r02/gpu_tests_sanitizer*.txt
        pytest.skip("compute-sanitizer closed on this GPU pool: " + out.strip().splitlines()[-1][:200])
    assert r.returncode == 0, out[-4000:]
    assert "sanitize target ok" in out, out[-4000:]
    if tool == "racecheck":
        assert "RACECHECK SUMMARY: 0 hazards displayed (0 errors, 0 warnings)" in out, out[-4000:]
    else:
        assert "ERROR SUMMARY: 0 errors" in out, out[-4000:]
