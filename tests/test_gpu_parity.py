"""Parity of the sm_100a path (through the C ABI) with the oracle and the reference's
golden fixtures.  Bit-exact: every output is integer."""

import random

import numpy as np
import pytest

from paper_2605_26461_b200 import constants as K
from paper_2605_26461_b200 import synth
from paper_2605_26461_b200.engine import BatchParams, DeviceBuffers, FaultEngine
from paper_2605_26461_b200.errors import EntryError, KindMismatch, NoChannelAttribution
from paper_2605_26461_b200.world import ENTRY_DTYPE

from oracle import seq_oracle as so
from tests import golden_io as G
from tests import randworld as RW
from tests.observe import observables

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def eng():
    e = FaultEngine(0)
    yield e
    e.close()


def bp(p: so.Params) -> BatchParams:
    return BatchParams(isolation=p.isolation, benign_us=p.benign_us, m1_us=p.m1_us,
                       m2_us=p.m2_us, m3_us=p.m3_us)


def assert_same(got, want, ctx=""):
    assert np.array_equal(got.out, want.out), (ctx, _first_diff(got.out, want.out))
    assert np.array_equal(got.verdict, want.verdict), (ctx, got.verdict, want.verdict)
    assert np.array_equal(got.counts, want.counts), ctx
    assert np.array_equal(got.dedup_keys, want.dedup_keys), ctx
    assert np.array_equal(got.dedup_idx, want.dedup_idx), ctx
    assert np.array_equal(got.cancel, want.cancel), ctx


def _first_diff(a, b):
    bad = np.nonzero(a != b)[0]
    return (int(bad[0]), a[bad[0]], b[bad[0]]) if len(bad) else None


def run_both(eng, w, entries, p):
    eng.upload_world(w)
    got = eng.process(entries, bp(p))
    want = so.process_batch(w, entries, p)
    return got, want


def run_device(eng, w, entries, p, layout="auto"):
    """The device-resident form (mpsf_process on device buffers, no host chunking); ``layout``
    forces the dedup-slot layout: "dense" one slot per (page, group) whatever the world size,
    "sparse" the large-world layout (claimed page slots + hash for other groups, no per-page
    first-eligible keys, so a client released before the drain takes the general path)."""
    import torch
    if layout is True or layout is False:
        layout = "dense" if layout else "auto"
    eng.set_dedup_layout(layout)
    eng.upload_world(w)
    try:
        n = len(entries)
        raw = entries.view(np.uint8).copy() if n else np.zeros(16, np.uint8)
        d_in = torch.from_numpy(raw).cuda()
        bufs = DeviceBuffers(n, w.n_clients)
        return eng.process_resident(d_in, n, bp(p), bufs)
    finally:
        eng.set_dedup_layout("auto")


# -- golden fixtures from the reference ---------------------------------------------------

def test_classify_golden_c1(eng):
    z = G.classify_c1()
    w, _ = synth.build_synthetic_world(4, 16, 1)
    eng.upload_world(w)
    res = eng.process(z["entries"], BatchParams())
    assert np.array_equal(res.out["scenario"], z["scenario"])
    assert np.array_equal(res.out["rid"], z["rid"])


@pytest.fixture
def layout_eng(eng, request):
    """The engine with the dedup-slot layout of the test's ``layout`` parameter."""
    eng.set_dedup_layout(request.param)
    yield eng
    eng.set_dedup_layout("auto")


@pytest.mark.parametrize("layout_eng", ["auto", "sparse"], indirect=True)
def test_reference_batches_golden(layout_eng):
    eng = layout_eng
    n = 0
    for flat, entries, p, expect in G.batches():
        eng.upload_world(flat)
        res = eng.process(entries, BatchParams(**p))
        assert observables(flat, entries, res.out, res.verdict) == G.as_tuples(expect), n
        n += 1
    assert n == 400


@pytest.mark.parametrize("layout_eng", ["auto", "sparse"], indirect=True)
def test_truth_table_golden(layout_eng):
    eng = layout_eng
    for row, flat, entries in G.truth_table():
        eng.upload_world(flat)
        res = eng.process(entries, BatchParams(isolation=row["isolation"]))
        obs = observables(flat, entries, res.out, res.verdict)
        ex = row["expect"]
        assert obs["clients"] == {k: tuple(v) for k, v in ex["clients"].items()}, row["trigger"]
        assert [m for _, m, _ in obs["isolation"]] == ex["mechanisms"], row["trigger"]
        assert obs["fatal_reports"] == ex["fatal_reports"], row["trigger"]


def test_remap_golden(eng):
    for case in G.load_json("remap.json"):
        for m in case["maps"].values():
            t = eng.remap(m["base"], np.array(m["phys"], np.uint64), 12)
            assert list(t["va"]) == [m["base"] + i * 4096 for i in range(m["npages"])]
            assert list(t["phys"]) == m["phys"]
        kv = case["maps"]["kv"]
        for rid, blocks in case["folded"].items():
            t = eng.remap_blocks(kv["base"], np.array(kv["phys"], np.uint64), blocks)
            assert np.array_equal(t, so.remap_blocks(kv["base"], kv["phys"], blocks))


# -- oracle parity on the build-defined batch semantics ---------------------------------------

@pytest.mark.parametrize("seed", range(6))
def test_random_batches_vs_oracle(eng, seed):
    rnd = random.Random(1000 + seed)
    for it in range(150):
        w = RW.random_world(rnd, dead_p=0.15 if seed % 2 else 0.0)
        p = RW.random_params(rnd)
        entries = RW.random_batch(rnd, w, rnd.randint(1, 64))
        got, want = run_both(eng, w, entries, p)
        assert_same(got, want, (seed, it))


@pytest.mark.parametrize("seed", range(4))
@pytest.mark.parametrize("dense", ["auto", "dense", "sparse"])
def test_random_batches_device_form_vs_oracle(eng, seed, dense):
    rnd = random.Random(5000 + seed)
    for it in range(80):
        w = RW.random_world(rnd, dead_p=0.15 if seed % 2 else 0.0)
        p = RW.random_params(rnd)
        entries = RW.random_batch(rnd, w, rnd.randint(1, 300))
        got = run_device(eng, w, entries, p, dense)
        want = so.process_batch(w, entries, p)
        assert_same(got, want, (seed, it, dense))


@pytest.mark.parametrize("dense", ["auto", "dense", "sparse"])
def test_large_random_batch_device_form_vs_oracle(eng, dense):
    rnd = random.Random(91)
    for it in range(4):
        w = RW.random_world(rnd, max_mps=6, max_sa=3)
        p = RW.random_params(rnd)
        entries = RW.random_batch(rnd, w, 30_000, parse_p=0.001, trap_p=0.0005, pool=12)
        got = run_device(eng, w, entries, p, dense)
        want = so.process_batch(w, entries, p)
        assert_same(got, want, (it, dense))


def test_config2b_and_storm_device_form_vs_oracle(eng):
    w, trace = synth.make_config("c2b", n=100_000)
    assert_same(run_device(eng, w, trace, so.Params(isolation=True)),
                so.process_batch(w, trace, so.Params(isolation=True)), "c2b")
    w, _ = synth.build_synthetic_world(6, 64, 3)
    trace = synth.generate_storm(w, 80_000, 8_000, 3)
    for iso in (True, False):
        assert_same(run_device(eng, w, trace, so.Params(isolation=iso)),
                    so.process_batch(w, trace, so.Params(isolation=iso)), ("storm", iso))


def test_large_random_batch_vs_oracle(eng):
    rnd = random.Random(77)
    for it in range(6):
        w = RW.random_world(rnd, max_mps=6, max_sa=3)
        p = RW.random_params(rnd)
        entries = RW.random_batch(rnd, w, 20_000, parse_p=0.001, trap_p=0.0005, pool=12)
        got, want = run_both(eng, w, entries, p)
        assert_same(got, want, it)


@pytest.mark.parametrize("iso", [True, False])
def test_config1_full_vs_oracle(eng, iso):
    w, trace = synth.make_config("c1")
    p = so.Params(isolation=iso)
    got, want = run_both(eng, w, trace, p)
    assert_same(got, want)
    assert got.counts.sum() == len(trace)


def test_config2b_slice_vs_oracle(eng):
    w, trace = synth.make_config("c2b", n=60_000)
    got, want = run_both(eng, w, trace, so.Params(isolation=True))
    assert_same(got, want)


def test_storm_slice_vs_oracle(eng):
    w, _ = synth.build_synthetic_world(6, 64, 3)
    trace = synth.generate_storm(w, 50_000, 5_000, 3)
    got, want = run_both(eng, w, trace, so.Params(isolation=True))
    assert_same(got, want)


# -- size-independent properties at full size ---------------------------------------------------

def test_storm_1e7_properties(eng):
    w, _ = synth.build_synthetic_world(48, 1024, 3)
    n, u = 10_000_000, 1_000_000
    trace = synth.generate_storm(w, n, u, 3)
    eng.upload_world(w)
    res = eng.process(trace, BatchParams(isolation=True))
    v = res.out["verdict"]
    assert len(res.dedup_keys) == u                     # every (client, page) pair has one key
    assert int(((v & K.V_DUP) != 0).sum()) == n - u
    assert len(np.unique(res.dedup_keys)) == u
    assert np.all(np.diff(res.dedup_idx.astype(np.int64)) > 0)
    assert np.all(np.diff(res.cancel.astype(np.int64)) > 0)
    assert res.counts.sum() == n
    # the representative of each key is its first occurrence
    key_of = ((trace["channel"].astype(np.uint64) // 3) << np.uint64(48))
    first = np.unique(res.dedup_idx)
    assert np.all((v[first] & K.V_DUP) == 0)
    # determinism: a second run is identical
    res2 = eng.process(trace, BatchParams(isolation=True))
    assert np.array_equal(res.out, res2.out) and np.array_equal(res.cancel, res2.cancel)
    del key_of


def test_device_resident_matches_host_form(eng):
    import torch
    w, trace = synth.make_config("c2a", n=200_000)
    eng.upload_world(w)
    host = eng.process(trace, BatchParams())
    d_in = torch.from_numpy(trace.view(np.uint8)).cuda()
    bufs = DeviceBuffers(len(trace), w.n_clients)
    dev = eng.process_resident(d_in, len(trace), BatchParams(), bufs)
    assert_same(dev, host)


@pytest.mark.parametrize("pinned", [True, False])
def test_pipelined_host_batches_vs_oracle(eng, pinned):
    """mpsf_submit_host / mpsf_collect_host: two slots in flight, batches of different sizes and
    worlds-compatible parameters; every batch equals its oracle result."""
    from paper_2605_26461_b200.engine import alloc_host_outputs
    w, trace = synth.make_config("c2b", n=300_000)
    eng.upload_world(w)
    cuts = [(0, 120_000), (120_000, 130_000), (130_000, 300_000), (5_000, 250_000)]
    params = [so.Params(isolation=True), so.Params(isolation=False), so.Params(isolation=True),
              so.Params(isolation=True, m2_us=100)]
    pending = {}
    for k, ((lo, hi), p) in enumerate(zip(cuts, params)):
        slot = k % 2
        if slot in pending:
            got = eng.collect(slot)
            want = pending.pop(slot)
            assert_same(got, want, ("slot", slot))
        part = trace[lo:hi]
        bufs = alloc_host_outputs(len(part), w.n_clients, pinned=pinned)
        eng.submit(part, bp(p), bufs, slot)
        pending[slot] = so.process_batch(w, part, p)
    for slot, want in pending.items():
        assert_same(eng.collect(slot), want, ("slot", slot))


# -- edge cases ------------------------------------------------------------------------------

def test_empty_and_invalid_batches(eng):
    w, _ = synth.build_synthetic_world(2, 4, 1)
    eng.upload_world(w)
    empty = np.zeros(0, ENTRY_DTYPE)
    res = eng.process(empty, BatchParams())
    assert len(res.out) == 0 and len(res.cancel) == 0
    assert np.all(res.verdict["state"] == K.ST_RUNNING)
    invalid = np.zeros(100, ENTRY_DTYPE)      # valid bit clear everywhere
    res = eng.process(invalid, BatchParams())
    assert np.all(res.out["scenario"] == 0xFF) and res.counts.sum() == 0


def test_entry_errors_map_to_reference_exceptions(eng):
    w, _ = synth.build_synthetic_world(2, 4, 1)
    eng.upload_world(w)
    e = np.zeros(3, ENTRY_DTYPE)
    e[:] = (0x100000, 0, 0, 0, 0, 1)
    e[1]["channel"] = 999
    with pytest.raises(NoChannelAttribution):
        eng.process(e, BatchParams())
    e[1]["channel"] = 1                        # CE channel, SM engine
    with pytest.raises(EntryError):
        eng.process(e, BatchParams())
    e[1]["engine"] = 1
    e[1]["va"] = 1 << 60
    with pytest.raises(EntryError):
        eng.process(e, BatchParams())
    bad = w.ranges.copy()
    bad[[0, 1]] = bad[[1, 0]]
    w2 = type(w)(w.clients, w.channels, bad, w.client_off, w.page_state)
    with pytest.raises(KindMismatch):
        eng.upload_world(w2)


@pytest.mark.parametrize("gran", [12, 16, 21])
def test_remap_granularities_vs_oracle(eng, gran):
    rng = np.random.default_rng(gran)
    npages = 5000 + gran
    phys = (rng.integers(1, 1 << 40, npages)).astype(np.uint64)
    got = eng.remap(0x7F00_0000_0000, phys, gran)
    want = so.remap_table(0x7F00_0000_0000, phys, gran)
    assert np.array_equal(got, want)


def test_maximum_batch_size_properties(eng):
    """A batch of exactly MAX_GIDX = 2^29 entries (the largest the global index / drain key
    encoding allows), device-resident: size-independent properties of the storm (exactly
    `u` representatives, every other entry a duplicate, ordered lists, counts summing to n),
    and one entry more is refused with MPSF_E_TOO_LARGE before any work."""
    import torch
    from paper_2605_26461_b200.errors import SimError
    n, u = 1 << 29, 10_000_000
    w, _ = synth.build_synthetic_world(48, 8192, 3)
    d_in = synth.generate_storm(w, n, u, 3, device="cuda")
    eng.upload_world(w)
    bufs = DeviceBuffers(n, w.n_clients)
    p = BatchParams(isolation=True)
    for _ in range(4):
        eng.process_device(d_in, n, p, bufs)
        try:
            s = eng.summary()
            break
        except Exception as exc:   # hash overflow: the table grew, run again
            assert type(exc).__name__ == "HashOverflow"
    assert int(s.n_dedup) == u
    out = bufs.out[:8 * n].view(torch.int64)
    verdict = (out >> 40) & 0xFF
    assert int(((verdict & K.V_DUP) != 0).sum()) == n - u
    didx = bufs.didx[:4 * u].view(torch.int32).to(torch.int64)
    assert bool((didx[1:] > didx[:-1]).all())
    nc = int(s.n_cancel)
    if nc > 1:
        ca = bufs.cancel[:4 * nc].view(torch.int32).to(torch.int64)
        assert bool((ca[1:] > ca[:-1]).all())
    counts = bufs.counts[:8 * K.N_SCENARIOS * w.n_clients].view(torch.int64)
    assert int(counts.sum()) == n
    with pytest.raises(SimError):
        eng.process_device(d_in, n + 1, p, bufs)
    del d_in, bufs, out, verdict, didx
    torch.cuda.empty_cache()


def test_wild_page_hash_overflow_retries_exactly(eng):
    """More distinct wild-page keys than the first hash sizing expects: the batch reports
    MPSF_E_OVERFLOW, the tables grow and the rerun is exact (host form, asynchronous form and
    device form)."""
    from oracle import c_oracle as co
    from paper_2605_26461_b200.engine import alloc_host_outputs
    w, _ = synth.build_synthetic_world(4, 16, 1)
    n = 300_000
    e = np.zeros(n, ENTRY_DTYPE)
    e["va"] = (np.uint64(1) << np.uint64(34)) + (np.arange(n, dtype=np.uint64) << np.uint64(12))   # no range
    e["channel"] = (np.arange(n) % w.n_clients) * 3          # SM channels
    e["engine"] = K.ENG_SM
    e["access"] = K.ACC_READ
    e["flags"] = K.ENTRY_FLAG_VALID
    p = so.Params(isolation=True)
    want = co.process_batch(w, e, p)
    fresh = FaultEngine(0)                                   # fresh context: first sizing from n
    try:
        fresh.upload_world(w)
        assert_same(fresh.process(e, bp(p)), want, "host")
        fresh2 = FaultEngine(0)
        try:
            fresh2.upload_world(w)
            bufs = alloc_host_outputs(n, w.n_clients, pinned=True)
            fresh2.submit(e, bp(p), bufs, 0)
            assert_same(fresh2.collect(0), want, "async")
        finally:
            fresh2.close()
    finally:
        fresh.close()
    assert_same(run_device(eng, w, e, p), want, "device")


# -- batched top half (mpsf_classify): the reference's per-record classify + range_at ------------

def test_batched_classify_golden_c1(eng):
    """mpsf_classify on the 20k-entry config-1 trace equals faults.classify / range_at as the
    reference computed them (tests/golden/classify_c1.npz, made by the reference itself)."""
    z = G.classify_c1()
    w, _ = synth.build_synthetic_world(4, 16, 1)
    eng.upload_world(w)
    sid, rid = eng.classify(z["entries"])
    assert np.array_equal(sid, z["scenario"])
    assert np.array_equal(rid, z["rid"])


@pytest.mark.parametrize("seed", range(3))
def test_batched_classify_vs_process(eng, seed):
    """The top half alone equals the scenario / rid fields mpsf_process writes, on random worlds
    with parse-time, trap, invalid and wild entries (and a world beyond the fixed layout)."""
    rnd = random.Random(700 + seed)
    for it in range(40):
        w = RW.random_world(rnd, max_mps=6, max_sa=3)
        entries = RW.random_batch(rnd, w, rnd.randint(1, 400))
        eng.upload_world(w)
        sid, rid = eng.classify(entries, base_index=it)
        full = eng.process(entries, BatchParams())
        assert np.array_equal(sid, full.out["scenario"]), (seed, it)
        assert np.array_equal(rid, full.out["rid"]), (seed, it)
    w, trace = synth.build_synthetic_world(80, 4, 5)[0], None
    trace = synth.generate_trace(w, synth.TraceSpec(n=5000, seed=seed, parse_frac=0.01, trap_frac=0.001))
    eng.upload_world(w)
    sid, rid = eng.classify(trace)
    full = eng.process(trace, BatchParams())
    assert np.array_equal(sid, full.out["scenario"]) and np.array_equal(rid, full.out["rid"])


def test_batched_classify_errors(eng):
    w, _ = synth.build_synthetic_world(2, 4, 1)
    eng.upload_world(w)
    e = np.zeros(3, ENTRY_DTYPE)
    e[:] = (0x100000, 0, 0, 0, 0, 1)
    e[2]["channel"] = 999
    with pytest.raises(NoChannelAttribution):
        eng.classify(e)
