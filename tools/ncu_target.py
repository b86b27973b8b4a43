"""Small driver for ncu captures: runs the fault path on one workload a few times.
    python tools/ncu_target.py c2b|c3 [reps]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2605_26461_b200 import synth
    from paper_2605_26461_b200.engine import BatchParams, DeviceBuffers, FaultEngine
    wl = sys.argv[1] if len(sys.argv) > 1 else "c2b"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    eng = FaultEngine(0)
    if wl == "c3":
        n = int(os.environ.get("STORM_N", 100_000_000))
        w, _ = synth.build_synthetic_world(48, 8192, 3)
        d_in = synth.generate_storm(w, n, n // 10, 3, device="cuda")
    else:
        w, trace = synth.make_config(wl)
        n = len(trace)
        d_in = torch.from_numpy(trace.view(np.uint8)).cuda()
    eng.upload_world(w)
    bufs = DeviceBuffers(n, w.n_clients)
    for _ in range(reps):
        eng.process_resident(d_in, n, BatchParams(isolation=True), bufs)
    torch.cuda.synchronize()
    print("done", wl, n)


if __name__ == "__main__":
    main()
