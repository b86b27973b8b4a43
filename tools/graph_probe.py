"""Probe: the device-resident fault path captured in a CUDA graph (small batches are
launch-bound): replay time vs direct enqueue, and bit-exact outputs."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2605_26461_b200 import synth
from paper_2605_26461_b200.engine import BatchParams, DeviceBuffers, FaultEngine

for wl, n in (("c1", 100_000), ("c1", 10_000), ("c2b", 1_000_000)):
    w, trace = synth.make_config(wl, n=n)
    eng = FaultEngine(0)
    eng.upload_world(w)
    d_in = torch.from_numpy(trace.view(np.uint8)).cuda()
    bufs = DeviceBuffers(n, w.n_clients)
    p = BatchParams(isolation=True)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            eng.process_device(d_in, n, p, bufs, stream=s)
        eng.summary()
        ref = bufs.out[:8 * n].clone()
    torch.cuda.synchronize()

    def t_direct(reps=200):
        with torch.cuda.stream(s):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            for _ in range(reps):
                eng.process_device(d_in, n, p, bufs, stream=s)
            b.record(s)
        b.synchronize()
        return a.elapsed_time(b) / reps * 1e3

    g = torch.cuda.CUDAGraph()
    try:
        with torch.cuda.graph(g, stream=s):
            eng.process_device(d_in, n, p, bufs, stream=s)
        ok_cap = True
    except Exception as exc:
        print(wl, n, "capture failed:", repr(exc)[:300])
        ok_cap = False
    if ok_cap:
        bufs.out.zero_()
        g.replay()
        torch.cuda.synchronize()
        same = torch.equal(bufs.out[:8 * n], ref)

        def t_graph(reps=200):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            with torch.cuda.stream(s):
                for _ in range(reps):
                    g.replay()
            b.record(s)
            b.synchronize()
            return a.elapsed_time(b) / reps * 1e3
        print(wl, n, f"direct {t_direct():.1f} us/batch, graph {t_graph():.1f} us/batch, same={same}", flush=True)
    eng.close()
