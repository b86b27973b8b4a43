"""e2e probe (experiment tool): per-batch time of the asynchronous host form over streams of
increasing length (pipeline fill / drain amortisation), c2b batches, pinned host buffers."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2605_26461_b200 import synth  # noqa: E402
from paper_2605_26461_b200.engine import BatchParams, FaultEngine, alloc_host_outputs  # noqa: E402

w, trace = synth.make_config("c2b")
n = len(trace)
eng = FaultEngine(0)
eng.upload_world(w)
pinned = torch.from_numpy(trace.view(np.uint8)).pin_memory().numpy().view(trace.dtype)
params = BatchParams(isolation=True)
NS = int(os.environ.get("NS", 3))
hb = [alloc_host_outputs(n, w.n_clients, pinned=True) for _ in range(NS)]


def stream(nb):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(nb):
        if k >= NS:
            eng.collect(k % NS)
        eng.submit(pinned, params, hb[k % NS], k % NS)
    for k in range(max(0, nb - NS), nb):
        eng.collect(k % NS)
    return (time.perf_counter() - t0) / nb


stream(2 * NS)
for nb in (6, 12, 24, 48):
    print(nb, "batches:", round(min(stream(nb), stream(nb)) * 1e3, 3), "ms per batch", flush=True)
