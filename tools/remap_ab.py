"""A/B timing of the remap across library builds: python tools/remap_ab.py lib1.so lib2.so ..."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 1 and sys.argv[1] == "one":
    os.environ["MPSF_LIB"] = sys.argv[2]
    sys.path.insert(0, ROOT)
    from types import SimpleNamespace
    import torch
    import bench
    from paper_2605_26461_b200.engine import FaultEngine
    eng = FaultEngine(0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    r = bench.bench_remap(SimpleNamespace(steps=50), eng, 6461.2, flush)
    print({k: (round(v["kernel_ms"] * 1e3, 2), round(v["ms_per_step"] * 1e3, 2), v["check"]) for k, v in r.items()
           if isinstance(v, dict)})
else:
    for lib in sys.argv[1:]:
        out = subprocess.run([sys.executable, __file__, "one", lib], capture_output=True, text=True)
        print(os.path.basename(lib), (out.stdout.strip().splitlines() or [out.stderr[-300:]])[-1], flush=True)
