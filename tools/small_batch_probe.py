"""Per-kernel device time of small device-resident batches (launch / prologue-bound sizes)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2605_26461_b200 import synth
from paper_2605_26461_b200.engine import BatchParams, DeviceBuffers, FaultEngine

for wl, n in (("c1", 1_000), ("c1", 100_000), ("c2b", 100_000)):
    w, trace = synth.make_config(wl, n=n)
    eng = FaultEngine(0)
    eng.upload_world(w)
    d_in = torch.from_numpy(trace.view(np.uint8)).cuda()
    bufs = DeviceBuffers(n, w.n_clients)
    p = BatchParams(isolation=True)
    for _ in range(5):
        eng.process_device(d_in, n, p, bufs)
    eng.summary()
    eng.set_profiling(True)
    for _ in range(50):
        eng.process_device(d_in, n, p, bufs)
    prof = eng.profile()
    eng.set_profiling(False)
    print(wl, n, {k: round(v[1] / max(v[0], 1) * 1e3, 1) for k, v in sorted(prof.items())}, flush=True)
    eng.close()
