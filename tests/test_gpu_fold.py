"""Snapshot delta fold on the GPU (mpsf_fold) against the oracle's
``fold_snapshots`` (pinned against the reference ``StandbyInstance.fold`` in
tests/test_fold_oracle.py), and the fold chained into the live-KV remap
(``complete_wake``, recovery.py:310-363).  Bit-exact."""

import numpy as np
import pytest

from paper_2605_26461_b200.engine import FaultEngine
from paper_2605_26461_b200.errors import EntryError

from oracle import seq_oracle as so

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def eng():
    e = FaultEngine(0)
    yield e
    e.close()


def snapshots(rng, n_req, n_snap, max_blk=4, max_tok=8, liveness=0.1):
    req = rng.integers(0, n_req, n_snap, dtype=np.uint32)
    req[rng.random(n_snap) < liveness] = so.NO_REQ
    seq = np.arange(1, n_snap + 1, dtype=np.uint64) * 3
    nblk = rng.integers(0, max_blk + 1, n_snap, dtype=np.uint32)
    ntok = rng.integers(0, max_tok + 1, n_snap, dtype=np.uint32)
    prog = rng.integers(0, 1 << 20, n_snap, dtype=np.uint32)
    done = (rng.random(n_snap) < 0.05).astype(np.uint8)
    blocks = rng.integers(0, 1 << 24, int(nblk.sum()), dtype=np.uint32)
    tokens = rng.integers(0, 50000, int(ntok.sum()), dtype=np.uint32)
    return req, seq, nblk, ntok, prog, done, blocks, tokens


def check(got, want):
    assert np.array_equal(got.order, want.order)
    assert np.array_equal(got.blk_off, want.blk_off)
    assert np.array_equal(got.blocks, want.blocks)
    assert np.array_equal(got.tok_off, want.tok_off)
    assert np.array_equal(got.tokens, want.tokens)
    assert np.array_equal(got.progress, want.progress)
    assert np.array_equal(got.done, want.done)
    assert got.last_seq == want.last_seq


@pytest.mark.parametrize("n_req,n_snap", [(1, 1), (1, 50), (7, 300), (200, 5000), (5000, 20000),
                                          (100_000, 200_000),
                                          # tile edges (8192 snapshots per tile), one request over
                                          # many tiles, a three-pass radix sort (2^19 ranks)
                                          (1000, 8191), (1000, 8192), (1000, 8193), (3, 16385), (1, 100_000),
                                          (400_000, 600_000)])
def test_fold_vs_oracle(eng, n_req, n_snap):
    rng = np.random.default_rng(n_req * 7 + n_snap)
    a = snapshots(rng, n_req, n_snap)
    check(eng.fold(*a, n_req_ids=n_req), so.fold_snapshots(*a))


def test_fold_edge_cases(eng):
    rng = np.random.default_rng(5)
    # empty
    a = snapshots(rng, 3, 0)
    check(eng.fold(*a), so.fold_snapshots(*a))
    # liveness only: nothing folded, seq still advances
    a = snapshots(rng, 3, 40, liveness=1.0)
    check(eng.fold(*a, n_req_ids=3), so.fold_snapshots(*a))
    # empty deltas everywhere
    a = snapshots(rng, 9, 500, max_blk=0, max_tok=0)
    check(eng.fold(*a, n_req_ids=9), so.fold_snapshots(*a))
    # one request with long deltas (warp copy loops > 32)
    a = snapshots(rng, 1, 64, max_blk=300, max_tok=1000)
    check(eng.fold(*a, n_req_ids=1), so.fold_snapshots(*a))
    # sparse ids: a large id space, few requests
    a = list(snapshots(rng, 5, 1000))
    ids = np.array([3, 77, 1 << 20, 9, 123456], np.uint32)
    live = a[0] != so.NO_REQ
    a[0] = a[0].copy()
    a[0][live] = ids[a[0][live]]
    check(eng.fold(*a, n_req_ids=(1 << 20) + 1), so.fold_snapshots(*a))


def test_fold_bad_request_id(eng):
    rng = np.random.default_rng(9)
    a = list(snapshots(rng, 10, 100, liveness=0.0))
    a[0] = a[0].copy()
    a[0][37] = 10
    a[0][80] = 11
    with pytest.raises(EntryError) as ei:
        eng.fold(*a, n_req_ids=10)
    assert ei.value.index == 37


def test_fold_then_remap_blocks(eng):
    """complete_wake: the folded block table of every live request remapped onto the
    standby's physical pages -- the fold output feeds mpsf_remap_blocks directly."""
    rng = np.random.default_rng(11)
    npages = 1 << 16
    phys = rng.integers(1, 1 << 40, npages, dtype=np.uint64)
    a = list(snapshots(rng, 300, 4000))
    a[6] = rng.integers(0, npages, len(a[6]), dtype=np.uint32)
    got = eng.fold(*a, n_req_ids=300)
    want = so.fold_snapshots(*a)
    check(got, want)
    va = 0x7F00_0000_0000
    t = eng.remap_blocks(va, phys, got.blocks)
    assert np.array_equal(t, so.remap_blocks(va, phys, want.blocks))


def test_fold_delta_overrun_rejected(eng):
    """Delta lengths that reach past the payload arrays are an argument error, not a read past
    the buffer."""
    from paper_2605_26461_b200.errors import SimError
    rng = np.random.default_rng(13)
    a = list(snapshots(rng, 4, 50, liveness=0.0))
    a[6] = a[6][:-3]                      # three block ids short
    with pytest.raises(SimError):
        eng.fold(*a, n_req_ids=4)


@pytest.mark.parametrize("total,n", [(0, 0), (1, 0), (1, 1), (64, 10), (1000, 5000), (1 << 20, 300_000),
                                     (8191, 3000), (8192, 8192), (8193, 100), (3 * 8192 + 5, 20_000)])
def test_kv_reserve_vs_oracle(eng, total, n):
    rng = np.random.default_rng(total + n)
    ids = rng.integers(0, total + 50, n, dtype=np.uint32) if n else np.zeros(0, np.uint32)
    reserved, free = eng.kv_reserve(total, ids)
    want_r, want_f = so.kv_reserve(total, ids) if total <= 5000 else _kv_reserve_np(total, ids)
    assert np.array_equal(reserved, want_r)
    assert np.array_equal(free, want_f)


def _kv_reserve_np(total, ids):
    r = np.zeros(total, np.uint8)
    ids = ids[ids < total]
    r[ids] = 1
    return r, np.nonzero(r == 0)[0].astype(np.uint32)


def test_fold_then_kv_reserve(eng):
    """complete_wake: every folded request's blocks reserved in the standby's pool."""
    rng = np.random.default_rng(17)
    a = list(snapshots(rng, 50, 2000))
    total = 4096
    a[6] = rng.integers(0, total, len(a[6]), dtype=np.uint32)
    got = eng.fold(*a, n_req_ids=50)
    reserved, free = eng.kv_reserve(total, got.blocks)
    want = so.fold_snapshots(*a)
    want_r, want_f = so.kv_reserve(total, want.blocks)
    assert np.array_equal(reserved, want_r) and np.array_equal(free, want_f)


def test_fold_id_space_limit(eng):
    from paper_2605_26461_b200.errors import SimError
    rng = np.random.default_rng(1)
    a = snapshots(rng, 4, 10, liveness=0.0)
    with pytest.raises(SimError):
        eng.fold(*a, n_req_ids=(1 << 30) + 1)


@pytest.mark.parametrize("nshards", [2, 4])
def test_sharded_fold_merge_on_gpu(eng, nshards):
    """The sharded fold's two GPU steps on one device: each contiguous range folded, the
    per-range folds (as one snapshot per request) concatenated and folded again == the whole
    stream's fold (parallel.ShardedFold does the same with an all-gather between them)."""
    rng = np.random.default_rng(40 + nshards)
    a = snapshots(rng, 500, 20_000)
    n = len(a[0])
    cut = [n * r // nshards for r in range(nshards + 1)]
    parts = []
    for lo, hi in zip(cut[:-1], cut[1:]):
        bo = int(a[2][:lo].sum()), int(a[2][:hi].sum())
        to = int(a[3][:lo].sum()), int(a[3][:hi].sum())
        sub = (a[0][lo:hi], a[1][lo:hi], a[2][lo:hi], a[3][lo:hi], a[4][lo:hi], a[5][lo:hi],
               a[6][bo[0]:bo[1]], a[7][to[0]:to[1]])
        parts.append(so.fold_as_snapshots(eng.fold(*sub, n_req_ids=500)))
    merged = tuple(np.concatenate([p[j] for p in parts]) for j in range(8))
    got = eng.fold(*merged, n_req_ids=500)
    want = so.fold_snapshots(*a)
    for f in ("order", "blk_off", "blocks", "tok_off", "tokens", "progress", "done"):
        assert np.array_equal(getattr(got, f), getattr(want, f)), f


def test_fold_radix_path_forced():
    """The radix path (id spaces above 2^17) forced at every size of this suite: the same
    parity cases in a subprocess with MPSF_FOLD_RADIX=1, so both fold paths stay bit-exact."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, MPSF_FOLD_RADIX="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", os.path.abspath(__file__),
                        "-k", "not radix_path_forced"], cwd=root, env=env, capture_output=True, text=True)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert " passed" in r.stdout
