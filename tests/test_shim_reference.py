"""The drop-in ``service_bottom_half`` (shim.py) under the reference's own 169-test suite:
every reference test must still pass with the batch path doing the bottom half."""

import os
import subprocess
import sys

import pytest

from tests import refharness as H

pytestmark = pytest.mark.skipif(not H.reference_available(), reason="reference not present")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_suite_passes_with_batch_bottom_half():
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([ROOT, H.REF_SRC]))
    tests_dir = H.REF_TESTS
    r = subprocess.run([sys.executable, "-m", "pytest", tests_dir, "-q", "-p", "no:cacheprovider",
                        "-p", "tests.shim_plugin"], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=900)
    tail = r.stdout[-3000:]
    assert r.returncode == 0, tail
    assert "169 passed" in tail, tail
    calls = int(tail.split("SHIM_CALLS=")[1].split()[0])
    assert calls > 100, tail
    assert int(tail.split("REMAP_MAPS=")[1].split()[0]) > 10, tail     # vmm_map remap tables checked
