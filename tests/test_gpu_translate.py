"""Batched translation on the GPU (mpsf_translate) against the oracle's
restatement of MemoryModel.resolve_va (pinned against the reference in
tests/test_translate_oracle.py): hit bytes, the misses as fault entries in order, the
populating prefetches.  Bit-exact."""

import random

import numpy as np
import pytest

from paper_2605_26461_b200 import constants as K
from paper_2605_26461_b200 import synth
from paper_2605_26461_b200.engine import BatchParams, FaultEngine
from paper_2605_26461_b200.errors import EntryError, NoChannelAttribution
from paper_2605_26461_b200.world import ENTRY_DTYPE

from oracle import seq_oracle as so
from tests import randworld as RW

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def eng():
    e = FaultEngine(0)
    yield e
    e.close()


def check(eng, w, acc, want):
    eng.upload_world(w)
    hit, faults, fi, pi = eng.translate(acc)
    assert np.array_equal(hit, want.hit)
    assert np.array_equal(fi, want.fault_idx)
    assert np.array_equal(pi, want.pop_idx)
    assert np.array_equal(faults, acc[want.fault_idx])          # the misses' seeds, in order


@pytest.mark.parametrize("cfg", [(4, 16, 1), (48, 16, 2), (6, 1024, 3)])
def test_translate_synthetic_vs_oracle(eng, cfg):
    w, _ = synth.build_synthetic_world(*cfg)
    acc = synth.generate_access_stream(w, 200_000, seed=cfg[2])
    want = so.translate_batch_np(w, acc)
    check(eng, w, acc, want)
    assert 0 < len(want.fault_idx) < len(acc) and len(want.pop_idx) > 0


def test_translate_random_worlds_vs_sequential_oracle(eng):
    rnd = random.Random(31)
    for it in range(60):
        w = RW.random_world(rnd, dead_p=0.1)
        e = RW.random_batch(rnd, w, rnd.randint(1, 400), parse_p=0.0, trap_p=0.0)
        e["access"] = np.where(np.array([rnd.random() < 0.3 for _ in range(len(e))]), K.ACC_PREFETCH, e["access"])
        check(eng, w, e, so.translate_batch(w, e))


def test_translate_large_stream_properties(eng):
    """10^7 accesses: hits + misses = valid entries, the fault entries feed mpsf_process."""
    w, _ = synth.build_synthetic_world(48, 16, 2)
    acc = synth.generate_access_stream(w, 10_000_000, seed=7)
    eng.upload_world(w)
    hit, faults, fi, pi = eng.translate(acc)
    assert int((hit == 1).sum()) + len(fi) == len(acc)
    assert np.all(np.diff(fi.astype(np.int64)) > 0) and np.all(np.diff(pi.astype(np.int64)) > 0)
    assert np.all(acc["access"][pi] == K.ACC_PREFETCH)
    want = so.translate_batch_np(w, acc)
    assert np.array_equal(hit, want.hit) and np.array_equal(fi, want.fault_idx) and np.array_equal(pi, want.pop_idx)
    res = eng.process(faults, BatchParams(isolation=True))     # the misses are a valid fault batch
    assert res.counts.sum() == len(faults)


def test_translate_errors_and_empty(eng):
    w, _ = synth.build_synthetic_world(2, 4, 1)
    eng.upload_world(w)
    hit, faults, fi, pi = eng.translate(np.zeros(0, ENTRY_DTYPE))
    assert len(hit) == 0 and len(fi) == 0
    e = np.zeros(3, ENTRY_DTYPE)
    e[:] = (0x100000, 0, 0, 0, 0, 1)
    e[1]["channel"] = 999
    with pytest.raises(NoChannelAttribution):
        eng.translate(e)
    e[1]["channel"] = 0
    e[1]["engine"] = 1                                            # SM channel, CE engine
    with pytest.raises(EntryError) as ei:
        eng.translate(e)
    assert ei.value.index == 1
    e[1]["engine"] = 0
    e[1]["kind"] = 8                                              # a trap record is not an access
    with pytest.raises(EntryError):
        eng.translate(e)


@pytest.mark.parametrize("nshards", [2, 3])
def test_sharded_translation_vs_whole_stream(nshards):
    """The two-phase API (mpsf_translate_prefetch, exchange stage 4, mpsf_translate_finish)
    over contiguous shards, one context each, the first-PREFETCH tables MIN-combined:
    concatenated results equal the whole-stream oracle bit for bit."""
    import torch
    from paper_2605_26461_b200.parallel import GpuTranslateShard, LocalTranslateGroup
    rnd = random.Random(60 + nshards)
    for it in range(6):
        w, _ = synth.build_synthetic_world(rnd.choice((6, 48)), rnd.choice((16, 64)), 1 + it % 3)
        acc = synth.generate_access_stream(w, rnd.randint(1000, 300_000), seed=it, prefetch=rnd.choice((0.1, 0.4)))
        n = len(acc)
        cut = [n * r // nshards for r in range(nshards + 1)]
        engs, ads = [], []
        for r in range(nshards):
            e = FaultEngine(0)
            e.upload_world(w)
            sh = acc[cut[r]:cut[r + 1]]
            d = torch.from_numpy(sh.view(np.uint8).copy()).cuda() if len(sh) else torch.empty(16, dtype=torch.uint8,
                                                                                                device="cuda")
            ads.append(GpuTranslateShard(e, d, len(sh), cut[r]))
            engs.append(e)
        parts = LocalTranslateGroup(ads).translate()
        for e in engs:
            e.close()
        want = so.translate_batch_np(w, acc)
        assert np.array_equal(np.concatenate([p["hit"] for p in parts]), want.hit), it
        assert np.array_equal(np.concatenate([p["fault_idx"] for p in parts]), want.fault_idx), it
        assert np.array_equal(np.concatenate([p["pop_idx"] for p in parts]), want.pop_idx), it


def test_translate_phase_misuse(eng):
    """mpsf_translate_finish must follow mpsf_translate_prefetch of the same batch size."""
    import torch
    from paper_2605_26461_b200.errors import SimError
    from paper_2605_26461_b200.parallel import GpuTranslateShard
    w, _ = synth.build_synthetic_world(4, 16, 1)
    eng.upload_world(w)
    acc = synth.generate_access_stream(w, 1000, seed=3)
    d = torch.from_numpy(acc.view(np.uint8).copy()).cuda()
    sh = GpuTranslateShard(eng, d, 1000, 0)
    sh.prefetch()
    sh.n = 999                                                   # a different batch than the prefetch's
    with pytest.raises(SimError):
        sh.finish()
