"""Run the bench's fold workload (timing + oracle check), then a profiled pass with the per-kernel
times recorded by the ABI: python tools/fold_run.py [steps]"""
import os
import sys
from types import SimpleNamespace

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2605_26461_b200.engine import FaultEngine  # noqa: E402

eng = FaultEngine(0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
r = bench.bench_fold(SimpleNamespace(steps=int(sys.argv[1]) if len(sys.argv) > 1 else 20), eng, 6448.4, flush)
print({k: v for k, v in r.items() if k != "cpu_baseline"})
eng.set_profiling(True)
bench.bench_fold(SimpleNamespace(steps=20), eng, 6448.4, flush)
prof = eng.profile()
print({k: round(v[1] / max(v[0], 1) * 1e3, 2) for k, v in sorted(prof.items())}, "us per call")
