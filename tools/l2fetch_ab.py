"""A/B of the device's maximum L2 fetch granularity (cudaLimitMaxL2FetchGranularity) over the
bench paths: python tools/l2fetch_ab.py [0 32 64 128 ...]  ("-" = leave the default).

Each setting runs in its own process: the limit is set on the primary context (the one torch and
libmpsf share) before bench.main() runs with its oracle checks off, and the step times of the
headline step, the c3 storm, the remap, the fold and the translation are printed side by side.
The random 4-byte probes of the passes (page state, dedup slot) and the remap's strided 8-byte
reads each pull a whole fetch unit from DRAM, so a smaller unit may trade DRAM bytes for nothing."""
import io
import json
import os
import subprocess
import sys
from contextlib import redirect_stdout

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

if len(sys.argv) > 1 and sys.argv[1] == "one":
    sys.path.insert(0, ROOT)
    import torch
    torch.cuda.init()
    torch.empty(1, device="cuda")
    from cuda.bindings import runtime as rt
    if sys.argv[2] != "-":
        err, = rt.cudaDeviceSetLimit(rt.cudaLimit.cudaLimitMaxL2FetchGranularity, int(sys.argv[2]))
        assert err == rt.cudaError_t.cudaSuccess, err
    err, got = rt.cudaDeviceGetLimit(rt.cudaLimit.cudaLimitMaxL2FetchGranularity)
    import bench
    sys.argv = ["bench.py", "--no-e2e", "--no-check", "--no-ref-path", "--steps", "20"]
    buf = io.StringIO()
    with redirect_stdout(buf):
        bench.main()
    line = json.loads([x for x in buf.getvalue().splitlines() if x.startswith("{")][-1])
    ex = line.get("extra", {})
    out = {"limit": int(got), "c2b_ms": round(line["ms_per_step"], 4),
           "k_scan_ms": line.get("kernels", {}).get("k_scan", {}).get("ms"),
           "k_finalize_ms": line.get("kernels", {}).get("k_finalize", {}).get("ms")}
    for k, v in ex.items():
        if isinstance(v, dict):
            if "ms_per_step" in v:
                out[k + "_ms"] = round(v["ms_per_step"], 4)
            for g, r in v.items():
                if isinstance(r, dict) and "kernel_ms" in r:
                    out[f"{k}.{g}_kernel_us"] = round(r["kernel_ms"] * 1e3, 2)
    print(json.dumps(out))
else:
    for lim in (sys.argv[1:] or ["-", "32", "64", "128"]):
        r = subprocess.run([sys.executable, __file__, "one", lim], capture_output=True, text=True, cwd=ROOT)
        print(lim, (r.stdout.strip().splitlines() or [r.stderr[-600:]])[-1], flush=True)
