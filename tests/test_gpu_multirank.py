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
