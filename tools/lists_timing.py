"""Experiment tool: per-block start/end of k_lists (built with -DMPSF_ABLATE=8704 = 8192|512)."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ["MPSF_LIB"] = os.path.join(ROOT, "build", "ablate", "libmpsf_8704.so")
sys.path.insert(0, ROOT)
import torch
from paper_2605_26461_b200 import synth
from paper_2605_26461_b200.engine import BatchParams, DeviceBuffers, FaultEngine
w, trace = synth.make_config("c2b")
n = len(trace)
d_in = torch.from_numpy(trace.view(np.uint8)).cuda()
eng = FaultEngine(0); eng.upload_world(w)
bufs = DeviceBuffers(n, w.n_clients)
for _ in range(3):
    eng.process_device(d_in, n, BatchParams(isolation=True), bufs)
torch.cuda.synchronize()
nseg = -(-(-(-n // 64)) // 256)
t = bufs.cancel[:8 * 4 * nseg].cpu().numpy().view(np.uint64).reshape(-1, 4)[:nseg]
t0 = t[:, 0].min()
st, en = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3
order = np.argsort(-(en - st))
for b in order[:12]:
    print(f"block {b:4d} sm {t[b,2]:4d} start {st[b]:8.2f} end {en[b]:8.2f} dur {en[b]-st[b]:8.2f} us")
print("median dur", np.median(en - st), "max end", en.max(), "starts spread", st.max())
dd = bufs.dedup_idx if hasattr(bufs, "dedup_idx") else None
res = eng.process(trace, BatchParams(isolation=True))
seg = np.asarray(res.dedup_idx, np.int64) // (64 * 256)
cnt = np.bincount(seg, minlength=nseg)
print("reps per segment: first 8", cnt[:8].tolist(), "max", cnt.max(), "median", int(np.median(cnt)), "total", cnt.sum())
