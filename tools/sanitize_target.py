"""Small invocation of every kernel family of libmpsf.so, for compute-sanitizer
(tests/test_gpu_sanitizer.py): the fault path on a config-2b slice (row-table passes, dense and
claimed-slot layouts, isolation on / off, device and host forms, a general-path batch), a
world beyond the fixed layout (global-table passes), the sharded phase API with the sparse
exchange, the batched translation, the snapshot fold, the KV pool restore and both remaps.
Every result is checked against the oracle, so a sanitizer run is also a parity run."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from oracle import seq_oracle as so
    from paper_2605_26461_b200 import synth
    from paper_2605_26461_b200.engine import BatchParams, DeviceBuffers, FaultEngine
    from paper_2605_26461_b200.parallel import GpuShard, LocalShardGroup
    only = sys.argv[1] if len(sys.argv) > 1 else "all"
    if only == "fold_radix":   # the fold's radix path (id spaces above 2^17) at the same small size
        os.environ["MPSF_FOLD_RADIX"] = "1"
        only = "fold"
    eng = FaultEngine(0)

    def check(got, want, what):
        for f in ("out", "verdict", "counts", "dedup_keys", "dedup_idx", "cancel"):
            assert np.array_equal(getattr(got, f), getattr(want, f)), (what, f)

    if only in ("all", "fault"):
        w, trace = synth.make_config("c2b", n=6000)
        for layout in ("auto", "sparse"):
            eng.set_dedup_layout(layout)
            eng.upload_world(w)
            for iso in (True, False):
                p = so.Params(isolation=iso)
                want = so.process_batch(w, trace, p)
                check(eng.process(trace, BatchParams(isolation=iso)), want, (layout, iso, "host"))
                d_in = torch.from_numpy(trace.view(np.uint8).copy()).cuda()
                bufs = DeviceBuffers(len(trace), w.n_clients)
                check(eng.process_resident(d_in, len(trace), BatchParams(isolation=iso), bufs), want, (layout, iso))
            # a batch that takes the general (release-aware) path: m2 faster than a benign completion
            p = so.Params(isolation=True, m2_us=100)
            check(eng.process(trace, BatchParams(isolation=True, m2_us=100)), so.process_batch(w, trace, p), "general")
        eng.set_dedup_layout("auto")
        # beyond the fixed shared-memory layout: 80 clients -> the global-table passes
        wb, _ = synth.build_synthetic_world(80, 4, 5)
        tb = synth.generate_trace(wb, synth.TraceSpec(n=4000, seed=9, parse_frac=0.01, trap_frac=0.001))
        eng.upload_world(wb)
        check(eng.process(tb, BatchParams()), so.process_batch(wb, tb, so.Params()), "global tables")
    if only in ("all", "sharded"):
        w, trace = synth.make_config("c2b", n=4000)
        cut = [0, 1500, 4000]
        ads, ps, engs = [], [], []
        for r in range(2):
            e = FaultEngine(0)
            e.set_dense_dedup(True)
            e.upload_world(w)
            sh = trace[cut[r]:cut[r + 1]]
            d = torch.from_numpy(sh.view(np.uint8).copy()).cuda()
            b = DeviceBuffers(len(sh), w.n_clients)
            ads.append(GpuShard(e, d, len(sh), b))
            ps.append(BatchParams(base_index=cut[r]))
            engs.append(e)
        res = LocalShardGroup(ads).process(ps)
        want = so.process_batch(w, trace, so.Params())
        assert np.array_equal(np.concatenate([r.out for r in res]), want.out)
        idx, val = ads[0].sparse_export(ads[0].exchange(1)[2][0])
        ads[1].sparse_merge(ads[1].exchange(1)[2][0], idx, val)
        torch.cuda.synchronize()
    if only in ("all", "translate"):
        w, _ = synth.make_config("c2b", n=10)
        eng.upload_world(w)
        acc = synth.generate_access_stream(w, 5000, seed=4)
        hit, faults, fi, pi = eng.translate(acc)
        want = so.translate_batch_np(w, acc)
        assert np.array_equal(hit, want.hit) and np.array_equal(fi, want.fault_idx)
    if only in ("all", "fold"):
        rng = np.random.default_rng(2)
        S = 3000
        req = rng.integers(0, 50, S, dtype=np.uint32)
        req[rng.random(S) < 0.1] = so.NO_REQ
        nblk = rng.integers(0, 3, S, dtype=np.uint32)
        ntok = rng.integers(0, 4, S, dtype=np.uint32)
        snap = (req, np.arange(1, S + 1, dtype=np.uint64), nblk, ntok, rng.integers(0, 99, S, dtype=np.uint32),
                (rng.random(S) < 0.05).astype(np.uint8), rng.integers(0, 1000, int(nblk.sum()), dtype=np.uint32),
                rng.integers(0, 9000, int(ntok.sum()), dtype=np.uint32))
        f = eng.fold(*snap, n_req_ids=50)
        g = so.fold_snapshots(*snap)
        assert np.array_equal(f.blocks, g.blocks) and np.array_equal(f.tokens, g.tokens)
        r, fr = eng.kv_reserve(1024, f.blocks)
        wr, wf = so.kv_reserve(1024, g.blocks)
        assert np.array_equal(r, wr) and np.array_equal(fr, wf)
    if only in ("all", "remap"):
        phys = np.arange(514, 514 + 5000, dtype=np.uint64)
        for gran in (12, 16, 21):
            assert np.array_equal(eng.remap(0x7F0000000000, phys, gran), so.remap_table(0x7F0000000000, phys, gran))
        blocks = np.array([3, 17, 0, 4999, 17], np.uint32)
        assert np.array_equal(eng.remap_blocks(0x7F0000000000, phys, blocks), so.remap_blocks(0x7F0000000000, phys, blocks))
    torch.cuda.synchronize()
    print("sanitize target ok:", only)


if __name__ == "__main__":
    main()
