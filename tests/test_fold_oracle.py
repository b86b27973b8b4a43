"""Pin the snapshot-fold oracle (``seq_oracle.fold_snapshots``) against the reference's own
``StandbyInstance.fold`` (recovery.py:83-92) on random consumed-snapshot sequences.  Skips when
the reference is not importable (the GPU box)."""

import random

import numpy as np
import pytest

from oracle import seq_oracle as so
from tests import refharness as H

pytestmark = pytest.mark.skipif(not H.reference_available(), reason="reference not present")


def random_snapshots(rnd, n_req, n_snap):
    snaps = []
    for i in range(n_snap):
        r = rnd.randrange(n_req) if rnd.random() > 0.1 else None
        snaps.append(dict(req=r, seq=i + 1, blocks=[rnd.randrange(1 << 20) for _ in range(rnd.randrange(0, 5))],
                          tokens=[rnd.randrange(50000) for _ in range(rnd.randrange(0, 9))],
                          progress=rnd.randrange(1000), done=rnd.random() < 0.1))
    return snaps


def to_arrays(snaps):
    req = np.array([so.NO_REQ if s["req"] is None else s["req"] for s in snaps], np.uint32)
    seq = np.array([s["seq"] for s in snaps], np.uint64)
    nblk = np.array([len(s["blocks"]) for s in snaps], np.uint32)
    ntok = np.array([len(s["tokens"]) for s in snaps], np.uint32)
    prog = np.array([s["progress"] for s in snaps], np.uint32)
    done = np.array([s["done"] for s in snaps], np.uint8)
    blocks = np.array([b for s in snaps for b in s["blocks"]], np.uint32)
    tokens = np.array([t for s in snaps for t in s["tokens"]], np.uint32)
    return req, seq, nblk, ntok, prog, done, blocks, tokens


@pytest.mark.parametrize("seed", range(4))
def test_fold_oracle_matches_standby_fold(seed):
    H.import_reference()
    from mpssim.recovery import ForwardSnapshot, StandbyInstance
    rnd = random.Random(70 + seed)
    for it in range(40):
        snaps = random_snapshots(rnd, rnd.randint(1, 12), rnd.randint(0, 80))
        st = StandbyInstance("p", 1, 2)
        for s in snaps:
            st.fold(ForwardSnapshot(request_id="" if s["req"] is None else f"r{s['req']}", seq=s["seq"],
                                    kv_block_ids_delta=list(s["blocks"]), token_delta=list(s["tokens"]),
                                    progress=s["progress"], done=s["done"]))
        got = so.fold_snapshots(*to_arrays(snaps))
        assert [f"r{r}" for r in got.order] == list(st.folded)
        for k, rid in enumerate(st.folded):
            f = st.folded[rid]
            b0, b1 = int(got.blk_off[k]), int(got.blk_off[k + 1])
            t0, t1 = int(got.tok_off[k]), int(got.tok_off[k + 1])
            assert got.blocks[b0:b1].tolist() == f.block_ids
            assert got.tokens[t0:t1].tolist() == f.tokens
            assert int(got.progress[k]) == f.progress and bool(got.done[k]) == f.done
        assert got.last_seq == st.last_consumed_seq


def _same(a, b):
    for f in ("order", "blk_off", "blocks", "tok_off", "tokens", "progress", "done"):
        x, y = getattr(a, f), getattr(b, f)
        assert x.dtype == y.dtype and np.array_equal(x, y), f
    assert a.last_seq == b.last_seq


@pytest.mark.parametrize("seed", range(3))
def test_fold_np_matches_loop(seed):
    rnd = random.Random(900 + seed)
    for it in range(30):
        snaps = random_snapshots(rnd, rnd.randint(1, 40), rnd.randint(0, 300))
        a = to_arrays(snaps)
        _same(so.fold_snapshots_np(*a), so.fold_snapshots(*a))


@pytest.mark.parametrize("seed", range(3))
def test_kv_reserve_oracle_matches_block_pool(seed):
    """``seq_oracle.kv_reserve`` against the reference ``BlockPool.reserve`` + pops."""
    H.import_reference()
    from mpssim.workload import BlockPool
    rnd = random.Random(300 + seed)
    for it in range(30):
        total = rnd.randint(0, 300)
        ids = [rnd.randrange(total + 20) for _ in range(rnd.randint(0, 2 * total + 1))]
        pool = BlockPool(total)
        pool.reserve(ids)
        pops = [pool.allocate() for _ in range(pool.free_count)]
        reserved, free = so.kv_reserve(total, ids)
        assert free.tolist() == pops
        assert reserved.tolist() == [1 if b in set(ids) else 0 for b in range(total)]


@pytest.mark.parametrize("seed", range(3))
def test_fold_composes_over_contiguous_ranges(seed):
    """fold(A ++ B ++ ...) == fold(snapshots(fold(A)) ++ snapshots(fold(B)) ++ ...): the merge
    step of the sharded fold (parallel.ShardedFold)."""
    rnd = random.Random(1200 + seed)
    for it in range(30):
        snaps = random_snapshots(rnd, rnd.randint(1, 20), rnd.randint(0, 200))
        a = to_arrays(snaps)
        n = len(a[0])
        k = rnd.randint(1, 4)
        cuts = sorted([0, n] + [rnd.randint(0, n) for _ in range(k - 1)])
        parts = []
        for lo, hi in zip(cuts[:-1], cuts[1:]):
            bo = int(a[2][:lo].sum()), int(a[2][:hi].sum())
            to = int(a[3][:lo].sum()), int(a[3][:hi].sum())
            sub = (a[0][lo:hi], a[1][lo:hi], a[2][lo:hi], a[3][lo:hi], a[4][lo:hi], a[5][lo:hi],
                   a[6][bo[0]:bo[1]], a[7][to[0]:to[1]])
            parts.append(so.fold_as_snapshots(so.fold_snapshots_np(*sub)))
        merged = tuple(np.concatenate([p[j] for p in parts]) if parts else np.zeros(0) for j in range(8))
        got = so.fold_snapshots_np(*merged)
        want = so.fold_snapshots_np(*a)
        for f in ("order", "blk_off", "blocks", "tok_off", "tokens", "progress", "done"):
            assert np.array_equal(getattr(got, f), getattr(want, f)), (seed, it, f)
