"""The multi-rank fault path end to end on one GPU: two processes, gloo collectives on CUDA
tensors (NCCL refuses two ranks on one device), each rank a FaultEngine driving its shard
through parallel.ShardedFaultPath / GpuShard -- the code the NCCL runs use.  Concatenated
per-rank results equal the C oracle on the whole batch, including a batch whose wild-page
keys overflow the hash tables in the cross-rank merge."""

import os
import socket
import tempfile

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _case(which):
    from paper_2605_26461_b200 import synth
    from paper_2605_26461_b200.world import ENTRY_DTYPE
    if which == "c2b":
        return synth.make_config("c2b", n=200_000)
    w, _ = synth.build_synthetic_world(4, 16, 1)
    n = 200_000
    e = np.zeros(n, ENTRY_DTYPE)
    e["va"] = (np.uint64(1) << np.uint64(34)) + (np.arange(n, dtype=np.uint64) << np.uint64(12))
    e["channel"] = (np.arange(n) % w.n_clients) * 3
    e["flags"] = 1
    return w, e


def _worker(rank, ws, port, outdir):
    import pickle
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    torch.cuda.set_device(0)
    from paper_2605_26461_b200.engine import BatchParams, DeviceBuffers, FaultEngine
    from paper_2605_26461_b200.parallel import GpuShard, ShardedFaultPath
    out = {}
    for which in ("c2b", "wild"):
        w, e = _case(which)
        n = len(e)
        cut = [n * r // ws for r in range(ws + 1)]
        sh = e[cut[rank]:cut[rank + 1]]
        eng = FaultEngine(0)
        eng.set_dense_dedup(True)
        eng.upload_world(w)
        d_in = torch.from_numpy(sh.view(np.uint8).copy()).cuda()
        bufs = DeviceBuffers(len(sh), w.n_clients)
        res = ShardedFaultPath(GpuShard(eng, d_in, len(sh), bufs)).process(
            BatchParams(isolation=True, base_index=cut[rank]))
        out[which] = {f: getattr(res, f) for f in ("out", "verdict", "counts", "dedup_keys", "dedup_idx", "cancel")}
        eng.close()
    with open(os.path.join(outdir, f"r{rank}.pkl"), "wb") as f:
        pickle.dump(out, f)
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_on_one_gpu_equal_oracle():
    import pickle
    import torch.multiprocessing as mp
    from oracle import c_oracle as co
    from oracle import seq_oracle as so
    ws = 2
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_worker, args=(ws, _free_port(), d), nprocs=ws, start_method="spawn")
        parts = [pickle.load(open(os.path.join(d, f"r{r}.pkl"), "rb")) for r in range(ws)]
    for which in ("c2b", "wild"):
        w, e = _case(which)
        want = co.process_batch(w, e, so.Params(isolation=True))
        assert np.array_equal(np.concatenate([p[which]["out"] for p in parts]), want.out), which
        for p in parts:
            assert np.array_equal(p[which]["verdict"], want.verdict), which
            assert np.array_equal(p[which]["counts"], want.counts), which
        for f, g in (("dedup_keys", "dedup_keys"), ("dedup_idx", "dedup_idx"), ("cancel", "cancel")):
            assert np.array_equal(np.concatenate([p[which][f] for p in parts]), getattr(want, g)), (which, f)


def _worker_tf(rank, ws, port, outdir):
    """Sharded translation (one MIN exchange) and sharded fold (all-gather + merge fold) with
    the GPU adapters, gloo collectives on CUDA tensors."""
    import pickle
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    torch.cuda.set_device(0)
    from paper_2605_26461_b200 import synth
    from paper_2605_26461_b200.engine import FaultEngine
    from paper_2605_26461_b200.parallel import GpuTranslateShard, ShardedFold, ShardedTranslate
    eng = FaultEngine(0)
    w, _ = synth.build_synthetic_world(6, 64, 2)
    eng.upload_world(w)
    acc = synth.generate_access_stream(w, 300_000, seed=9, prefetch=0.3)
    n = len(acc)
    cut = [n * r // ws for r in range(ws + 1)]
    sh = acc[cut[rank]:cut[rank + 1]]
    d = torch.from_numpy(sh.view(np.uint8).copy()).cuda()
    tr = ShardedTranslate(GpuTranslateShard(eng, d, len(sh), cut[rank])).translate()
    from tests.test_gpu_fold import snapshots
    a = snapshots(np.random.default_rng(77), 300, 40_000)
    m = len(a[0])
    c2 = [m * r // ws for r in range(ws + 1)]
    lo, hi = c2[rank], c2[rank + 1]
    bo = int(a[2][:lo].sum()), int(a[2][:hi].sum())
    to = int(a[3][:lo].sum()), int(a[3][:hi].sum())
    sub = (a[0][lo:hi], a[1][lo:hi], a[2][lo:hi], a[3][lo:hi], a[4][lo:hi], a[5][lo:hi],
           a[6][bo[0]:bo[1]], a[7][to[0]:to[1]])
    fo = ShardedFold(lambda *x: eng.fold(*x[:8], n_req_ids=x[8]), device="cuda").fold(*sub, 300)
    with open(os.path.join(outdir, f"t{rank}.pkl"), "wb") as f:
        pickle.dump({"tr": tr, "fold": {k: getattr(fo, k) for k in ("order", "blk_off", "blocks", "tok_off",
                                                                   "tokens", "progress", "done", "last_seq")}}, f)
    eng.close()
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_translation_and_fold():
    import pickle
    import torch.multiprocessing as mp
    from oracle import seq_oracle as so
    from paper_2605_26461_b200 import synth
    from tests.test_gpu_fold import snapshots
    ws = 2
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_worker_tf, args=(ws, _free_port(), d), nprocs=ws, start_method="spawn")
        parts = [pickle.load(open(os.path.join(d, f"t{r}.pkl"), "rb")) for r in range(ws)]
    w, _ = synth.build_synthetic_world(6, 64, 2)
    acc = synth.generate_access_stream(w, 300_000, seed=9, prefetch=0.3)
    want = so.translate_batch_np(w, acc)
    assert np.array_equal(np.concatenate([p["tr"]["hit"] for p in parts]), want.hit)
    assert np.array_equal(np.concatenate([p["tr"]["fault_idx"] for p in parts]), want.fault_idx)
    assert np.array_equal(np.concatenate([p["tr"]["pop_idx"] for p in parts]), want.pop_idx)
    a = snapshots(np.random.default_rng(77), 300, 40_000)
    wf = so.fold_snapshots_np(*a)
    for p in parts:
        for k in ("order", "blk_off", "blocks", "tok_off", "tokens", "progress", "done"):
            assert np.array_equal(p["fold"][k], getattr(wf, k)), k
        assert p["fold"]["last_seq"] == wf.last_seq
