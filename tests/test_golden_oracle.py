"""The oracle against every golden fixture the reference produced.

These are the known answers the parity chain is anchored on: the GPU path is compared
with the oracle (tests/test_gpu_parity.py) *and* with these same fixtures."""

import numpy as np

from paper_2605_26461_b200 import constants as K
from paper_2605_26461_b200 import synth

from oracle import seq_oracle as so
from tests import golden_io as G
from tests.observe import observables


def test_synthetic_world_matches_reference_build():
    z = G.classify_c1()
    w, _ = synth.build_synthetic_world(4, 16, 1)
    assert np.array_equal(w.ranges, z["ranges"])
    assert np.array_equal(w.page_state, z["page_state"])
    trace = synth.generate_trace(w, synth.TraceSpec(n=100_000, seed=1))[:20_000]
    assert np.array_equal(trace, z["entries"]), "trace generator drifted"


def test_oracle_classify_matches_reference_golden():
    z = G.classify_c1()
    w, _ = synth.build_synthetic_world(4, 16, 1)
    e = z["entries"]
    for i in range(0, len(e), 7):
        ridx, s = so.classify(w, int(e["channel"][i]) // 3, int(e["va"][i]),
                              int(e["engine"][i]), int(e["access"][i]))
        assert s == z["scenario"][i]
        assert (int(w.ranges["rid"][ridx]) if ridx >= 0 else K.NO_RID) == z["rid"][i]


def test_oracle_matches_reference_batches():
    n = 0
    for flat, entries, p, expect in G.batches():
        res = so.process_batch(flat, entries, so.Params(**p))
        assert observables(flat, entries, res.out, res.verdict) == G.as_tuples(expect)
        n += 1
    assert n == 400


def test_oracle_matches_reference_truth_table():
    for row, flat, entries in G.truth_table():
        res = so.process_batch(flat, entries, so.Params(isolation=row["isolation"]))
        obs = observables(flat, entries, res.out, res.verdict)
        ex = row["expect"]
        assert obs["clients"] == {k: tuple(v) for k, v in ex["clients"].items()}, row["trigger"]
        assert [m for _, m, _ in obs["isolation"]] == ex["mechanisms"], row["trigger"]
        assert obs["fatal_reports"] == ex["fatal_reports"], row["trigger"]
        assert obs["scenarios"] == ex["scenarios"], row["trigger"]


def test_oracle_remap_matches_reference_vmm_map():
    for case in G.load_json("remap.json"):
        for name, m in case["maps"].items():
            t = so.remap_table(m["base"], m["phys"], 12)
            assert len(t) == m["npages"]
            assert list(t["va"]) == [m["base"] + i * 4096 for i in range(m["npages"])]
            assert list(t["phys"]) == m["phys"]
        kv = case["maps"]["kv"]
        for rid, blocks in case["folded"].items():
            assert case["restored"][rid] == blocks
            t = so.remap_blocks(kv["base"], kv["phys"], blocks)
            assert list(t["phys"]) == [kv["phys"][b] for b in blocks]
