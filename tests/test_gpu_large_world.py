"""Parity of the large-world layout on the config-3 world itself (48 clients x 32 ranges x
8192 pages = 12.6 M page slots, so the device picks one claimed dedup slot per page, sends
every further dedup group of a page through the wild-page hash table and keeps no per-page
first-eligible keys).  Mixed traces of 1.2 M entries -- storm duplicates, every scenario
class, wild and guard pages, several dedup groups on one page, parse-time records and SM
traps at fixed positions, clients dead or with a destroyed CE TSG at batch start -- are
compared on all six outputs against the C restatement of the sequential drain
(oracle/mpsf_oracle.c, pinned to the reference by tests/test_c_oracle.py).  Reference
semantics: pipeline.py:160-183 with SURVEY.md Appendix C rules C2/C3."""

import numpy as np
import pytest

from paper_2605_26461_b200 import constants as K
from paper_2605_26461_b200 import synth
from paper_2605_26461_b200.engine import BatchParams, DeviceBuffers, FaultEngine

from oracle import c_oracle as co
from oracle import seq_oracle as so

pytestmark = pytest.mark.gpu

N = 1_200_000
MPS, SA = 44, 4          # clients 0..43 MPS, 44..47 standalone


@pytest.fixture(scope="module")
def world():
    w, _ = synth.build_synthetic_world(MPS, 8192, 3, n_standalone=SA)
    assert w.n_pages > 3_400_000          # over the dense-slot limit: the claimed-slot layout
    return w


@pytest.fixture(scope="module")
def eng():
    e = FaultEngine(0)
    yield e
    e.close()


def with_dead(w, dead=(5, 45), ce_dead=(7,)):
    """The same world with some clients terminated / a CE TSG destroyed before the batch."""
    cl = w.clients.copy()
    for c in dead:
        cl["flags"][c] = 0
    for c in ce_dead:
        cl["flags"][c] |= K.CF_CE_TSG_DEAD
    return type(w)(cl, w.channels, w.ranges, w.client_off, w.page_state, w.world_flags)


def run(eng, w, trace, p, layout):
    import torch
    eng.set_dedup_layout(layout)
    try:
        eng.upload_world(w)
        d_in = torch.from_numpy(trace.view(np.uint8).copy()).cuda()
        bufs = DeviceBuffers(len(trace), w.n_clients)
        return eng.process_resident(d_in, len(trace), BatchParams(
            isolation=p.isolation, benign_us=p.benign_us, m1_us=p.m1_us, m2_us=p.m2_us, m3_us=p.m3_us), bufs)
    finally:
        eng.set_dedup_layout("auto")


def same(got, want, ctx):
    for f in ("out", "verdict", "counts", "dedup_keys", "dedup_idx", "cancel"):
        a, b = getattr(got, f), getattr(want, f)
        if not np.array_equal(a, b):
            bad = np.nonzero(a != b)[0] if a.shape == b.shape else None
            raise AssertionError(f"{ctx}: {f} differs (len {len(a)} vs {len(b)}; first {bad[:3] if bad is not None else '-'})")


CASES = {
    # a parse-time record of an MPS client inside the drain (GR teardown mid-batch: C3 epochs
    # for every MPS client), a standalone trap (released before the drain), dead clients
    "parse_mid": dict(specials=((0.4, K.KIND_PARSE_FIRST + 2, 11), (0.6, K.KIND_TRAP_FIRST + 1, 46)),
                      params=so.Params(isolation=True)),
    # an MPS trap: every MPS client released before the drain (epoch-1 keys only)
    "mps_trap": dict(specials=((0.3, K.KIND_TRAP_FIRST, 3),), params=so.Params(isolation=True)),
    # no release at all, isolation on, M2 faster than a benign completion (general stage 2)
    "m2_fast": dict(specials=(), params=so.Params(isolation=True, m2_us=100)),
    # isolation off: every non-serviceable record is a fatal report
    "iso_off": dict(specials=((0.5, K.KIND_PARSE_FIRST, 44),), params=so.Params(isolation=False)),
}


@pytest.mark.parametrize("layout", ["auto", "dense"])
@pytest.mark.parametrize("case", sorted(CASES))
def test_c3_world_mixed_trace_vs_c_oracle(eng, world, case, layout):
    cfg = CASES[case]
    w = with_dead(world)
    trace = synth.generate_mixed_storm(w, N, seed=31 + len(case), specials=cfg["specials"])
    got = run(eng, w, trace, cfg["params"], layout)
    want = co.process_batch(w, trace, cfg["params"], threads=8)
    same(got, want, (case, layout))
    assert len(got.dedup_keys) > 100_000 and got.counts.sum() == N


def test_c3_world_several_groups_per_page_use_the_hash(eng, world):
    """The trace really puts several dedup groups on one page (the claimed-slot layout's
    hash fallback runs) and the dedup set holds keys of the same page in different groups."""
    trace = synth.generate_mixed_storm(world, 300_000, seed=7)
    got = run(eng, world, trace, so.Params(isolation=True), "auto")
    want = co.process_batch(world, trace, so.Params(isolation=True), threads=8)
    same(got, want, "groups")
    k = got.dedup_keys
    page_of = (k & np.uint64((1 << 41) - 1)) | ((k >> np.uint64(48)) << np.uint64(41))
    _, cnt = np.unique(page_of, return_counts=True)
    assert (cnt > 1).sum() > 1000
    assert eng.summary().hash_used > 1000
