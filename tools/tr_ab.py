"""A/B timing of mpsf_translate across library builds (experiment tool):
    python tools/tr_ab.py lib1.so lib2.so ..."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

if len(sys.argv) > 1 and sys.argv[1] == "one":
    os.environ["MPSF_LIB"] = sys.argv[2]
    sys.path.insert(0, ROOT)
    from types import SimpleNamespace
    import numpy as np
    import torch
    import bench
    from paper_2605_26461_b200 import synth
    from paper_2605_26461_b200.engine import FaultEngine
    eng = FaultEngine(0)
    w, _ = synth.build_synthetic_world(48, 16, 2)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    r = bench.bench_translate(SimpleNamespace(steps=50, n=None), eng, 6461.2, flush, w)
    # per-kernel times from the ABI's profiled pass (events after every launch)
    acc = synth.generate_access_stream(w, 10_000_000, seed=11)
    d_acc = torch.from_numpy(acc.view(np.uint8)).cuda()
    n = 10_000_000
    bufs = [torch.empty(k * n, dtype=torch.uint8, device="cuda") for k in (1, 16, 4, 4)]
    eng.set_profiling(True)
    for _ in range(20):
        flush.zero_()
        eng.translate_device(d_acc, n, *bufs)
    torch.cuda.synchronize()
    prof = eng.profile()
    eng.set_profiling(False)
    print(round(r["ms_per_step"] * 1e3, 1), "us", r["bit_exact_vs_oracle"],
          {k: round(v[1] / max(v[0], 1) * 1e3, 1) for k, v in sorted(prof.items())})
else:
    for lib in sys.argv[1:]:
        out = subprocess.run([sys.executable, __file__, "one", lib], capture_output=True, text=True)
        print(os.path.basename(lib), (out.stdout.strip().splitlines() or [out.stderr[-300:]])[-1], flush=True)
