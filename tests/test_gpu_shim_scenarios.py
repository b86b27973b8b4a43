"""The reference's six bundled scenarios with the drop-in on the GPU (``FaultEngine(0)`` behind
``service_bottom_half`` and ``vmm_map``): byte-identical verdicts and artifacts (DES traces,
matrices, sweeps, audit) to the unmodified reference.  On the GPU box the reference is the
install under ``baseline/_ref`` (tools/install_reference.sh)."""

import pytest

from tests import refharness as H
from tests.test_shim_scenarios import check, run_parity

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not H.reference_available(), reason="reference not installed")]


def test_bundled_scenarios_identical_with_gpu_bottom_half():
    check(run_parity("gpu"))
