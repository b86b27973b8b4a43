"""The drop-in ``service_bottom_half`` on the GPU under the reference's own test suite: every
reference test (``pkg/tests``, 169) must pass with ``mpssim.pipeline.service_bottom_half``
replaced by the batch path running on cuda:0 (``shim.install(FaultEngine(0))``, called at
``machine.py:188-191``; reference semantics ``pipeline.py:160-183``).  On the GPU box the
reference is the pip install under ``baseline/_ref`` (``tools/install_reference.sh``)."""

import os
import subprocess
import sys

import pytest

from tests import refharness as H

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not H.reference_available() or not os.path.isdir(H.REF_TESTS),
                                 reason="reference (baseline/_ref) not installed")]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_suite_passes_with_gpu_bottom_half():
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([ROOT, H.REF_SRC]), MPSF_SHIM_ENGINE="gpu")
    r = subprocess.run([sys.executable, "-m", "pytest", H.REF_TESTS, "-q", "-p", "no:cacheprovider",
                        "-p", "tests.shim_plugin"], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=1500)
    tail = r.stdout[-3000:]
    assert r.returncode == 0, tail + r.stderr[-2000:]
    assert "169 passed" in tail, tail
    calls = int(tail.split("SHIM_CALLS=")[1].split()[0])
    assert calls > 100, tail
    assert int(tail.split("REMAP_MAPS=")[1].split()[0]) > 10, tail     # vmm_map remap tables checked
