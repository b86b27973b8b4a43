"""The reference's six bundled scenarios (harness.BUNDLED) with the batch drop-in installed
produce byte-identical verdicts and artifacts -- per-scenario DES traces, containment matrix,
recovery and sync sweeps, the reachability audit -- to the unmodified reference (SURVEY.md
§8(b), machine.py:188-191, pipeline.py:160-183).  CPU: the drop-in runs on the C-oracle engine
(tests/scenario_parity.py); the device engine is tests/test_gpu_shim_scenarios.py."""

import json
import os
import subprocess
import sys

import pytest

from tests import refharness as H

pytestmark = pytest.mark.skipif(not H.reference_available(), reason="reference not present")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_parity(engine):
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([ROOT, H.REF_SRC]))
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "scenario_parity.py"), engine], cwd=ROOT,
                       env=env, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def check(rep):
    assert len(rep["scenarios"]) == 6, rep
    for name, s in rep["scenarios"].items():
        assert s["passed"] and s["verdicts_identical"] and not s["artifacts_differing"], (name, s)
        assert s["artifacts"] > 0
    assert rep["shim_calls"] > 1000 and rep["remap_maps"] > 100, rep


def test_bundled_scenarios_identical_with_batch_bottom_half():
    check(run_parity("oracle"))
