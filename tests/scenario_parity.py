"""Every bundled reference scenario (``mpssim.harness.BUNDLED``: table3, table4, fig3, fig6, fig8,
the reachability audit) run twice -- as the reference ships it, then with the batch drop-in
installed (``shim.install``: ``service_bottom_half`` at machine.py:188-191 and ``vmm_map`` at
memory.py:269-283 replaced) -- and every verdict and artifact (the per-scenario DES traces,
matrices, sweep tables) compared byte for byte.  SURVEY.md §8(b): "DES timing and traces stay
byte-identical".

    python tests/scenario_parity.py oracle|gpu     # prints one JSON line

Run as a subprocess by tests/test_shim_scenarios.py (C-oracle engine, CPU) and
tests/test_gpu_shim_scenarios.py (the device engine, ``-m gpu``); needs the reference importable
(``PYTHONPATH`` with its ``src``).
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run_all(harness):
    out = {}
    for name in harness.BUNDLED:
        r = harness.run_scenario_text(harness.load_bundled(name))
        out[name] = (r.passed, dict(r.verdicts), dict(r.artifacts))
    return out


def main():
    engine_kind = sys.argv[1] if len(sys.argv) > 1 else "oracle"
    from mpssim import harness
    from paper_2605_26461_b200 import shim
    from tests import shim_plugin as sp

    want = run_all(harness)
    engine = sp.CountingEngine() if engine_kind == "gpu" else sp.OracleEngine()
    undo = shim.install(engine)
    try:
        got = run_all(harness)
    finally:
        undo()
    report = {}
    for name, (wp, wv, wa) in want.items():
        gp, gv, ga = got[name]
        diff = sorted(k for k in set(wa) | set(ga) if wa.get(k) != ga.get(k))
        report[name] = {"passed": gp, "verdicts_identical": gv == wv, "artifacts": len(wa),
                        "artifact_bytes": sum(len(v) for v in wa.values()), "artifacts_differing": diff}
    print(json.dumps({"engine": engine_kind, "scenarios": report, "shim_calls": sp.CALLS["n"],
                      "shim_records": sp.CALLS["records"], "remap_maps": shim.REMAP_CHECKS["maps"]}))


if __name__ == "__main__":
    main()
