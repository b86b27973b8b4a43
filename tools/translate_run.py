"""Run the bench's translation workload (for ncu launch lists): python tools/translate_run.py [reps]"""
import os
import sys
from types import SimpleNamespace

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2605_26461_b200 import synth  # noqa: E402
from paper_2605_26461_b200.engine import FaultEngine  # noqa: E402

eng = FaultEngine(0)
w, _ = synth.build_synthetic_world(48, 16, 2)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
r = bench.bench_translate(SimpleNamespace(steps=int(sys.argv[1]) if len(sys.argv) > 1 else 5, n=None), eng, 6461.2,
                          flush, w)
print(r)
eng.set_profiling(True)
bench.bench_translate(SimpleNamespace(steps=20, n=None), eng, 6461.2, flush, w)
prof = eng.profile()
print({k: round(v[1] / max(v[0], 1) * 1e3, 2) for k, v in sorted(prof.items())}, "us per call")
