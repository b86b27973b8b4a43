"""Sharded GPU path (the phase entry points of libmpsf.so + the exchanges of
parallel.py), several shards on one device: concatenated shard outputs must equal the
single-context GPU result and the oracle bit for bit."""

import random

import numpy as np
import pytest
import torch

from paper_2605_26461_b200 import synth
from paper_2605_26461_b200.engine import BatchParams, DeviceBuffers, FaultEngine
from paper_2605_26461_b200.parallel import GpuShard, LocalShardGroup
from paper_2605_26461_b200.world import ENTRY_DTYPE

from oracle import c_oracle as co
from oracle import seq_oracle as so
from tests import randworld as RW

pytestmark = pytest.mark.gpu


def run_sharded(w, entries, bp, nshards):
    n = len(entries)
    cut = [n * r // nshards for r in range(nshards + 1)]
    ads, params, engs = [], [], []
    for r in range(nshards):
        e = FaultEngine(0)
        e.set_dense_dedup(True)
        e.upload_world(w)
        shard = entries[cut[r]:cut[r + 1]]
        d_in = torch.from_numpy(shard.view(np.uint8).copy()).cuda() if len(shard) else \
            torch.empty(16, dtype=torch.uint8, device="cuda")
        bufs = DeviceBuffers(max(len(shard), 1), w.n_clients)
        ads.append(GpuShard(e, d_in, len(shard), bufs))
        p = BatchParams(**{**bp.__dict__, "base_index": cut[r]})
        params.append(p)
        engs.append(e)
    res = LocalShardGroup(ads).process(params)
    for e in engs:
        e.close()
    return res


def check(w, entries, bp, res):
    want = co.process_batch(w, entries, so.Params(isolation=bp.isolation, benign_us=bp.benign_us,
                                                   m1_us=bp.m1_us, m2_us=bp.m2_us, m3_us=bp.m3_us))
    assert np.array_equal(np.concatenate([r.out for r in res]), want.out)
    for r in res:
        assert np.array_equal(r.verdict, want.verdict)
        assert np.array_equal(r.counts, want.counts)
    assert np.array_equal(np.concatenate([r.dedup_keys for r in res]), want.dedup_keys)
    assert np.array_equal(np.concatenate([r.dedup_idx for r in res]), want.dedup_idx)
    assert np.array_equal(np.concatenate([r.cancel for r in res]), want.cancel)


@pytest.mark.parametrize("nshards", [2, 3])
def test_sharded_random_batches(nshards):
    rnd = random.Random(500 + nshards)
    for it in range(40):
        w = RW.random_world(rnd, dead_p=0.1 if it % 2 else 0.0)
        p = RW.random_params(rnd)
        entries = RW.random_batch(rnd, w, rnd.randint(8, 400), pool=3)
        bp = BatchParams(isolation=p.isolation, benign_us=p.benign_us, m1_us=p.m1_us, m2_us=p.m2_us, m3_us=p.m3_us)
        check(w, entries, bp, run_sharded(w, entries, bp, nshards))


def test_sharded_config2b_slice():
    w, trace = synth.make_config("c2b", n=300_000)
    bp = BatchParams(isolation=True)
    check(w, trace, bp, run_sharded(w, trace, bp, 4))


def test_sharded_storm_slice():
    w, _ = synth.build_synthetic_world(8, 256, 3)
    trace = synth.generate_storm(w, 200_000, 20_000, 3)
    bp = BatchParams(isolation=True)
    check(w, trace, bp, run_sharded(w, trace, bp, 2))


@pytest.mark.parametrize("nshards", [2, 3])
def test_sharded_wild_hash_overflow_reruns(nshards):
    """Distinct wild-page keys beyond the first hash sizing, split over shards: the merge of
    the other shards' keys overflows the tables, every shard reruns the batch with grown
    tables, and the result is exact."""
    w, _ = synth.build_synthetic_world(4, 16, 1)
    n = 240_000
    e = np.zeros(n, ENTRY_DTYPE)
    e["va"] = (np.uint64(1) << np.uint64(34)) + (np.arange(n, dtype=np.uint64) << np.uint64(12))
    e["channel"] = (np.arange(n) % w.n_clients) * 3
    e["flags"] = 1
    bp = BatchParams(isolation=True)
    check(w, e, bp, run_sharded(w, e, bp, nshards))


def test_sparse_export_merge_equals_min():
    """mpsf_sparse_export / mpsf_sparse_merge: compaction of the non-empty words and the MIN
    merge of another rank's pairs equal an elementwise unsigned MIN of the two buffers."""
    import torch
    from paper_2605_26461_b200.engine import FaultEngine
    from paper_2605_26461_b200.parallel import GpuShard
    eng = FaultEngine(0)
    rng = np.random.default_rng(5)
    n = 3_000_001
    a = np.full(n, 0xFFFFFFFF, np.uint32)
    b = a.copy()
    ia, ib = rng.choice(n, 200_000, replace=False), rng.choice(n, 150_000, replace=False)
    a[ia] = rng.integers(0, 1 << 31, len(ia))
    b[ib] = rng.integers(0, 1 << 32, len(ib), dtype=np.uint64).astype(np.uint32) & 0xFFFFFFFE
    ta = torch.from_numpy(a.view(np.int32).copy()).cuda()
    tb = torch.from_numpy(b.view(np.int32).copy()).cuda()

    class _Sh(GpuShard):
        def __init__(self, e):
            self.eng, self.lib, self.ctx = e, e.lib, e.ctx
            import ctypes as C
            self.sp = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    sh = _Sh(eng)
    idx, val = sh.sparse_export(tb)
    got_i = idx.cpu().numpy().astype(np.int64)
    order = np.argsort(got_i)
    assert np.array_equal(got_i[order], np.sort(ib))
    assert np.array_equal(val.cpu().numpy().view(np.uint32)[order], b[np.sort(ib)])
    sh.sparse_merge(ta, idx, val)
    torch.cuda.synchronize()
    assert np.array_equal(ta.cpu().numpy().view(np.uint32), np.minimum(a, b))
    eng.close()
