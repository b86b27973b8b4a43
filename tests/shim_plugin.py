"""pytest plugin: run the REFERENCE's own test suite with ``mpssim.pipeline.service_bottom_half``
replaced by the batch drop-in (``paper_2605_26461_b200.shim``).  The engine behind it is the
C oracle by default (CPU container); with ``MPSF_SHIM_ENGINE=gpu`` it is the device path
(``FaultEngine(0)``, libmpsf.so on cuda:0) -- the drop-in as a user would install it."""

import os

import numpy as np

CALLS = {"n": 0, "records": 0}


class OracleEngine:
    def upload_world(self, flat):
        self.flat = flat

    def remap(self, va_base, phys, gran_log2):
        from oracle import seq_oracle as so
        return so.remap_table(va_base, phys, gran_log2)

    def process(self, entries, params):
        from oracle import c_oracle as co
        from oracle import seq_oracle as so
        CALLS["n"] += 1
        CALLS["records"] += len(entries)
        return co.process_batch(self.flat, entries, so.Params(
            isolation=params.isolation, benign_us=params.benign_us, m1_us=params.m1_us,
            m2_us=params.m2_us, m3_us=params.m3_us))


class CountingEngine:
    """The device engine, counting the batches it processes."""

    def __init__(self):
        from paper_2605_26461_b200.engine import FaultEngine
        self.eng = FaultEngine(0)

    def upload_world(self, flat):
        self.eng.upload_world(flat)

    def remap(self, va_base, phys, gran_log2):
        return self.eng.remap(va_base, phys, gran_log2)

    def process(self, entries, params):
        CALLS["n"] += 1
        CALLS["records"] += len(entries)
        return self.eng.process(entries, params)


def pytest_configure(config):
    from paper_2605_26461_b200 import shim
    shim.install(CountingEngine() if os.environ.get("MPSF_SHIM_ENGINE") == "gpu" else OracleEngine())


def pytest_sessionfinish(session, exitstatus):
    from paper_2605_26461_b200.shim import REMAP_CHECKS
    print(f"\nSHIM_CALLS={CALLS['n']} SHIM_RECORDS={CALLS['records']} "
          f"REMAP_MAPS={REMAP_CHECKS['maps']} REMAP_PAGES={REMAP_CHECKS['pages']}")
