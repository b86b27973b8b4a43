"""Pin the sequential oracle against the reference package itself.

On every random batch the reference can process (it raises ``UnknownTsg`` / ``KeyError``
on the batches SURVEY.md Appendix A [P2] describes), the oracle must reproduce the
reference's labels, isolation outcomes, benign completions, fatal-report count, fault-log
scenarios and per-client fates exactly.  Batches with duplicate dedup keys are excluded
from the mechanism/benign comparison (the build coalesces them by rule C2, the reference
does not), exactly as in the [P11]/[P12]/[P15] method.

Skips when the reference is not importable (the GPU box).
"""

import random

import numpy as np
import pytest

from paper_2605_26461_b200 import constants as K
from paper_2605_26461_b200.world import export_reference_world

from oracle import seq_oracle as so
from tests import refharness as H

pytestmark = pytest.mark.skipif(not H.reference_available(), reason="reference not present")


def _compare(flat, entries, ref, res):
    names = flat.channel_names
    drained_scen = [K.SCENARIOS[int(res.out["scenario"][i])].sid
                    for i in range(len(entries)) if int(entries["kind"][i]) < 8]
    assert drained_scen == ref["scenarios"]
    assert [K.OUTCOME_NAMES[o] for _, o in res.labels] == ref["labels"]
    iso = [(K.SCENARIOS[s].sid, K.MECH_NAMES[m], flat.client_names[c])
           for _, s, m, c in res.isolation_outcomes]
    assert iso == ref["isolation"]
    ben = [(names[int(entries["channel"][i])], int(entries["va"][i]), ok)
           for i, ok in res.benign_events]
    assert ben == ref["benign"]
    assert len(res.fatal_reports) == ref["fatal_reports"]
    for c, pid in enumerate(flat.client_names):
        v = res.verdict[c]
        got = ("running" if v["state"] == K.ST_RUNNING else "terminated",
               K.REASON_NAMES[int(v["reason"])], K.notifier_name(int(v["notifier"])))
        assert got == ref["clients"][pid], pid


def _has_dup_keys(res):
    return bool(np.any(res.out["verdict"] & K.V_DUP))


def _run(seed, n_batches, lat_random):
    rnd = random.Random(seed)
    ok = crashed = skipped_dup = 0
    for _ in range(n_batches):
        spec = H.random_small_world_spec(rnd)
        params_kw = {}
        if lat_random:
            params_kw = dict(m1_latency_us=rnd.choice((131, 226, 300)),
                             m2_latency_us=rnd.choice((2780, 226, 100)),
                             m3_latency_us=rnd.choice((1700, 226, 0)),
                             benign_service_us=226)
        w = H.build_reference_world(spec, params_kw)
        flat = export_reference_world(w)
        iso = rnd.random() < 0.6
        entries = H.random_batch(rnd, flat, rnd.randint(1, 12))
        p = so.Params(isolation=iso,
                      benign_us=w.params.benign_service_us, m1_us=w.params.m1_latency_us,
                      m2_us=w.params.m2_latency_us, m3_us=w.params.m3_latency_us)
        res = so.process_batch(flat, entries, p)
        if _has_dup_keys(res):
            skipped_dup += 1
            continue
        try:
            ref = H.run_reference_batch(w, flat, entries, isolation=iso)
        except Exception as exc:  # reference crash: UnknownTsg / KeyError
            assert type(exc).__name__ in ("UnknownTsg", "KeyError"), repr(exc)
            crashed += 1
            continue
        _compare(flat, entries, ref, res)
        ok += 1
    return ok, crashed, skipped_dup


def test_oracle_equals_reference_default_latencies():
    ok, crashed, _ = _run(11, 700, lat_random=False)
    assert ok > 200 and crashed > 20


def test_oracle_equals_reference_random_latencies():
    ok, crashed, _ = _run(12, 700, lat_random=True)
    assert ok > 200 and crashed > 20


def test_classify_equals_reference_classify_on_synthetic_world():
    """Per-entry attribution + classification vs faults.classify (direct, gates bypassed)."""
    H.import_reference()
    from mpssim import faults
    from mpssim.execmodel import EngineClass
    from mpssim.memory import AccessType, FaultSeed
    from paper_2605_26461_b200 import synth

    w = H.build_reference_world(H.synthetic_spec(4, 16, 1))
    flat = export_reference_world(w)
    mine, _ = synth.build_synthetic_world(4, 16, 1)
    for f in ("ranges", "page_state", "client_off", "clients", "channels"):
        assert np.array_equal(getattr(flat, f), getattr(mine, f)), f
    trace = synth.generate_trace(mine, synth.TraceSpec(n=3000, seed=5))
    for e in trace:
        c = int(e["channel"]) // 3
        pid = flat.client_names[c]
        seed = FaultSeed(va=int(e["va"]), access=AccessType(H.ACCESSES[int(e["access"])]),
                         engine=EngineClass(H.ENGINES[int(e["engine"])]))
        want = faults.classify(seed, w.mem, pid).sid
        rng = w.mem.range_at(pid, int(e["va"]))
        ridx, s = so.classify(flat, c, int(e["va"]), int(e["engine"]), int(e["access"]))
        assert K.SCENARIOS[s].sid == want
        assert (rng.rid if rng else None) == (int(flat.ranges["rid"][ridx]) if ridx >= 0 else None)
