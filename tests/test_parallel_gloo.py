"""Sharded (multi-rank) fault path on CPU: world_size-2 gloo runs of
``parallel.ShardedFaultPath`` driving the phase-by-phase CPU mirror of the kernels
(``oracle/c9_oracle.py``) must equal the sequential oracle on the whole batch, bit for bit
(SURVEY.md Appendix C, C8).  The GPU adapter (``parallel.GpuShard``) runs the same
orchestration over NCCL."""

import os
import random
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2605_26461_b200 import constants as K
from paper_2605_26461_b200.engine import BatchParams
from paper_2605_26461_b200.parallel import ShardedFaultPath

from oracle import c9_oracle as c9
from oracle import seq_oracle as so
from tests import randworld as RW


def oparams(p: BatchParams) -> so.Params:
    return so.Params(isolation=p.isolation, benign_us=p.benign_us, m1_us=p.m1_us, m2_us=p.m2_us, m3_us=p.m3_us)


class C9Shard:
    """CPU adapter with the same surface as parallel.GpuShard."""

    def __init__(self, w, entries, base):
        self.e = c9.C9Engine(w)
        self.entries, self.base = entries, base

    def scan(self, p):
        self.e.scan(self.entries, oparams(p), self.base)

    def exchange(self, stage):
        return [(torch.from_numpy(a.view(np.int64 if a.dtype == np.uint64 else np.int32)), op)
                for a, op in self.e.exchange_buffers(stage)]

    def hash_export(self, which):
        k, v = self.e.hash_export(which)
        return torch.from_numpy(k.view(np.int64).copy()), torch.from_numpy(v.view(np.int32).copy())

    def hash_merge(self, which, ks, vs):
        self.e.hash_merge(which, ks.numpy().view(np.uint64), vs.numpy().view(np.uint32))

    def resolve(self, p):
        self.verdict = self.e.resolve(oparams(p))

    def general(self, p, stage):
        self.e.general(oparams(p), stage)

    def resolve2(self, p):
        self.e.resolve2(oparams(p))

    def finalize(self, p):
        self.out, self.dk, self.di, self.ca, self.counts = self.e.finalize(self.entries, oparams(p))

    def counts_tensor(self):
        return torch.from_numpy(self.e.counts.view(np.int64))

    def sparse_export(self, t):
        """CPU stand-in of mpsf_sparse_export: the non-empty words as (index, value)."""
        idx = torch.nonzero(t != -1).flatten()
        return idx.to(torch.int32), t[idx].clone()

    def sparse_merge(self, t, idx, val):
        flip = -(1 << 31)
        cur = (t ^ flip).clone()
        cur.scatter_reduce_(0, idx.long(), val ^ flip, reduce="amin")
        t.copy_(cur ^ flip)

    def status(self):
        return 0, -1

    def result(self):
        return dict(out=self.out, dk=self.dk, di=self.di, ca=self.ca, verdict=self.verdict,
                    counts=self.e.counts.reshape(-1, K.N_SCENARIOS).copy())


def make_case(seed):
    rnd = random.Random(seed)
    w = RW.random_world(rnd, max_mps=4, max_sa=2, dead_p=0.1 if seed % 3 == 0 else 0.0)
    p = RW.random_params(rnd)
    entries = RW.random_batch(rnd, w, rnd.randint(2, 90), pool=3)
    bp = BatchParams(isolation=p.isolation, benign_us=p.benign_us, m1_us=p.m1_us, m2_us=p.m2_us, m3_us=p.m3_us)
    return w, entries, bp


def check_against_oracle(w, entries, bp, parts):
    want = so.process_batch(w, entries, oparams(bp))
    out = np.concatenate([r["out"] for r in parts])
    assert np.array_equal(out, want.out)
    for r in parts:
        assert np.array_equal(r["verdict"], want.verdict)
        assert np.array_equal(r["counts"], want.counts)
    assert np.array_equal(np.concatenate([r["dk"] for r in parts]), want.dedup_keys)
    assert np.array_equal(np.concatenate([r["di"] for r in parts]), want.dedup_idx)
    assert np.array_equal(np.concatenate([r["ca"] for r in parts]), want.cancel)


class _NoDist:
    """Single-shard run: the exchanges become identities."""


def test_c9_mirror_single_shard_equals_sequential_oracle(monkeypatch):
    import paper_2605_26461_b200.parallel as par
    monkeypatch.setattr(par, "allreduce_min_unsigned", lambda t, g=None: None)
    monkeypatch.setattr(par, "allreduce_sum", lambda t, g=None: None)
    monkeypatch.setattr(par, "allgather_ragged", lambda k, v, g=None: (k, v))
    for seed in range(250):
        w, entries, bp = make_case(seed)
        res = ShardedFaultPath(C9Shard(w, entries, 0)).process(bp)
        check_against_oracle(w, entries, bp, [res])


def _worker(rank, ws, port, seeds, outdir, sparse="auto"):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["MPSF_SPARSE_X"] = sparse
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    import pickle
    results = {}
    for seed in seeds:
        w, entries, bp = make_case(seed)
        n = len(entries)
        cut = [n * r // ws for r in range(ws + 1)]
        shard = entries[cut[rank]:cut[rank + 1]]
        res = ShardedFaultPath(C9Shard(w, shard, cut[rank])).process(bp)
        results[seed] = res
    with open(os.path.join(outdir, f"r{rank}.pkl"), "wb") as f:
        pickle.dump(results, f)
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("ws,sparse", [(2, "auto"), (3, "auto"), (2, "always")])
def test_sharded_gloo_equals_sequential_oracle(ws, sparse):
    """Dense all-reduce of every exchange buffer, and (``always``) the sparse form of the
    page-sized ones: compacted (index, value) pairs all-gathered and MIN-merged."""
    import pickle
    seeds = list(range(1000, 1060))
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_worker, args=(ws, _free_port(), seeds, d, sparse), nprocs=ws, start_method="fork")
        per_rank = [pickle.load(open(os.path.join(d, f"r{r}.pkl"), "rb")) for r in range(ws)]
    for seed in seeds:
        w, entries, bp = make_case(seed)
        check_against_oracle(w, entries, bp, [per_rank[r][seed] for r in range(ws)])


class _BadShard(C9Shard):
    """A shard whose batch reports an entry error (what GpuShard.status() returns after the
    device flagged a bad entry in this rank's range)."""

    def __init__(self, w, entries, base, err):
        super().__init__(w, entries, base)
        self.err = err

    def status(self):
        return self.err


def _err_worker(rank, ws, port, errs, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    from paper_2605_26461_b200.errors import SimError
    w, entries, bp = make_case(1003)
    cut = [len(entries) * r // ws for r in range(ws + 1)]
    shard = _BadShard(w, entries[cut[rank]:cut[rank + 1]], cut[rank], errs[rank])
    got = None
    try:
        ShardedFaultPath(shard).process(bp)
    except SimError as exc:
        got = (type(exc).__name__, getattr(exc, "index", None), str(exc))
    with open(os.path.join(outdir, f"e{rank}.txt"), "w") as f:
        f.write(repr(got))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("errs,want", [
    # one rank has a bad entry: every rank raises it (nobody waits in a collective)
    ([(0, -1), (-3, 17), (0, -1)], ("NoChannelAttribution", 17)),
    # two kinds on two ranks: the highest-priority code, the smallest index of any bad entry
    ([(-6, 5), (-4, 40), (0, -1)], ("EntryError", 5)),
])
def test_sharded_entry_error_raises_on_every_rank(errs, want):
    ws = len(errs)
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_err_worker, args=(ws, _free_port(), errs, d), nprocs=ws, start_method="fork")
        got = [eval(open(os.path.join(d, f"e{r}.txt")).read()) for r in range(ws)]
    for g in got:
        assert g is not None and g[0] == want[0], got
        assert str(want[1]) in g[2], got
    if want[0] == "EntryError":
        assert all(g[1] == want[1] and "-4" in g[2] for g in got), got    # E_BAD_ENTRY outranks E_VA


# -- sharded batched translation (one MIN exchange of the first-PREFETCH page table) ----------

class OracleTranslateShard:
    """CPU adapter with the surface of parallel.GpuTranslateShard (the oracle's two phases)."""

    def __init__(self, w, acc, base):
        self.w, self.acc, self.base = w, acc, base

    def prefetch(self):
        self.pf = so.translate_prefetch_np(self.w, self.acc, self.base)

    def exchange(self, stage):
        assert stage == 4
        return [(torch.from_numpy(self.pf), "min")]

    def finish(self):
        r = so.translate_finish_np(self.w, self.acc, self.base, self.pf)
        return dict(hit=r.hit, fault_idx=r.fault_idx, pop_idx=r.pop_idx)


def translate_case(seed):
    from paper_2605_26461_b200 import synth
    rnd = random.Random(seed)
    w, _ = synth.build_synthetic_world(rnd.choice((4, 6)), rnd.choice((16, 64)), 1 + seed % 3)
    acc = synth.generate_access_stream(w, rnd.randint(1, 3000), seed=seed, prefetch=rnd.choice((0.1, 0.4)))
    return w, acc


def _translate_worker(rank, ws, port, seeds, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    import pickle
    from paper_2605_26461_b200.parallel import ShardedTranslate
    results = {}
    for seed in seeds:
        w, acc = translate_case(seed)
        n = len(acc)
        cut = [n * r // ws for r in range(ws + 1)]
        results[seed] = ShardedTranslate(OracleTranslateShard(w, acc[cut[rank]:cut[rank + 1]], cut[rank])).translate()
    with open(os.path.join(outdir, f"t{rank}.pkl"), "wb") as f:
        pickle.dump(results, f)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("ws", [2, 3])
def test_sharded_translation_gloo_equals_whole_stream(ws):
    """Concatenated per-rank hits / misses / populations == the whole stream translated at once
    (and that equals the access-by-access oracle, tests/test_translate_oracle.py)."""
    import pickle
    seeds = list(range(200, 230))
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_translate_worker, args=(ws, _free_port(), seeds, d), nprocs=ws, start_method="fork")
        per_rank = [pickle.load(open(os.path.join(d, f"t{r}.pkl"), "rb")) for r in range(ws)]
    for seed in seeds:
        w, acc = translate_case(seed)
        want = so.translate_batch(w, acc)
        parts = [per_rank[r][seed] for r in range(ws)]
        assert np.array_equal(np.concatenate([p["hit"] for p in parts]), want.hit), seed
        assert np.array_equal(np.concatenate([p["fault_idx"] for p in parts]), want.fault_idx), seed
        assert np.array_equal(np.concatenate([p["pop_idx"] for p in parts]), want.pop_idx), seed


# -- sharded snapshot fold (all-gather of the per-rank folds, then one merge fold) -------------

def fold_case(seed):
    rnd = np.random.default_rng(seed)
    S = int(rnd.integers(0, 400))
    R = int(rnd.integers(1, 30))
    req = rnd.integers(0, R, S, dtype=np.uint32)
    req[rnd.random(S) < 0.1] = so.NO_REQ
    seq = np.arange(1, S + 1, dtype=np.uint64)
    nblk = rnd.integers(0, 4, S, dtype=np.uint32)
    ntok = rnd.integers(0, 6, S, dtype=np.uint32)
    prog = rnd.integers(0, 1000, S, dtype=np.uint32)
    done = (rnd.random(S) < 0.1).astype(np.uint8)
    blocks = rnd.integers(0, 1 << 20, int(nblk.sum()), dtype=np.uint32)
    tokens = rnd.integers(0, 50000, int(ntok.sum()), dtype=np.uint32)
    return (req, seq, nblk, ntok, prog, done, blocks, tokens), R


def shard_of(a, lo, hi):
    bo = int(a[2][:lo].sum()), int(a[2][:hi].sum())
    to = int(a[3][:lo].sum()), int(a[3][:hi].sum())
    return (a[0][lo:hi], a[1][lo:hi], a[2][lo:hi], a[3][lo:hi], a[4][lo:hi], a[5][lo:hi],
            a[6][bo[0]:bo[1]], a[7][to[0]:to[1]])


def _fold_worker(rank, ws, port, seeds, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    import pickle
    from paper_2605_26461_b200.parallel import ShardedFold
    sf = ShardedFold(lambda *a: so.fold_snapshots_np(*a[:8]))
    results = {}
    for seed in seeds:
        a, R = fold_case(seed)
        n = len(a[0])
        cut = [n * r // ws for r in range(ws + 1)]
        f = sf.fold(*shard_of(a, cut[rank], cut[rank + 1]), R)
        results[seed] = {k: getattr(f, k) for k in ("order", "blk_off", "blocks", "tok_off", "tokens", "progress",
                                                    "done", "last_seq")}
    with open(os.path.join(outdir, f"f{rank}.pkl"), "wb") as fh:
        pickle.dump(results, fh)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("ws", [2, 3])
def test_sharded_fold_gloo_equals_whole_stream(ws):
    import pickle
    seeds = list(range(300, 340))
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_fold_worker, args=(ws, _free_port(), seeds, d), nprocs=ws, start_method="fork")
        per_rank = [pickle.load(open(os.path.join(d, f"f{r}.pkl"), "rb")) for r in range(ws)]
    for seed in seeds:
        a, R = fold_case(seed)
        want = so.fold_snapshots(*a)
        for r in range(ws):
            got = per_rank[r][seed]
            for k in ("order", "blk_off", "blocks", "tok_off", "tokens", "progress", "done"):
                assert np.array_equal(got[k], getattr(want, k)), (seed, r, k)
            assert got["last_seq"] == want.last_seq, seed
