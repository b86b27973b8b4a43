"""Experiment tool: time k_scan / k_finalize of libmpsf variants built with -DMPSF_ABLATE=<mask>.

    python tools/ablate.py build 0 1 2 ...      # here: builds build/ablate/libmpsf_<mask>.so
    python tools/ablate.py run [wl] 0 1 2 ...   # on the GPU box: kernel times per variant

Variant outputs are NOT the fault path's results (switched-off work); only timings are read.
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "build", "ablate")


def build(masks, extra=()):
    import glob
    os.makedirs(OUT, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(ROOT, "paper_2605_26461_b200", "csrc", "*.cu")) +
                  glob.glob(os.path.join(ROOT, "paper_2605_26461_b200", "csrc", "*.cpp")))
    procs = []
    for m in masks:
        lib = os.path.join(OUT, f"libmpsf_{m}.so")
        cmd = ["nvcc", "-O3", "-lineinfo", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a",
               "-Xcompiler", "-fPIC,-O3", "-I", os.path.join(ROOT, "include"), f"-DMPSF_ABLATE={m}",
               *extra, "-shared", "-o", lib, *srcs]
        procs.append(subprocess.Popen(cmd))
    for p in procs:
        assert p.wait() == 0


def one(wl, lib, reps):
    os.environ["MPSF_LIB"] = lib
    sys.path.insert(0, ROOT)
    import numpy as np
    import torch
    from paper_2605_26461_b200 import synth
    from paper_2605_26461_b200.engine import BatchParams, DeviceBuffers, FaultEngine
    cache = f"/tmp/ablate_{wl}.npy"
    if wl == "c3":
        w, _ = synth.build_synthetic_world(48, 8192, 3)
        n = 100_000_000
        d_in = synth.generate_storm(w, n, n // 10, 3, device="cuda")
    else:
        w, _ = synth.build_synthetic_world(48, 16, 2)
        if os.path.exists(cache):
            trace = np.load(cache)
        else:
            _, trace = synth.make_config(wl)
            np.save(cache, trace)
        n = len(trace)
        d_in = torch.from_numpy(trace.view(np.uint8)).cuda()
    eng = FaultEngine(0)
    eng.upload_world(w)
    bufs = DeviceBuffers(n, w.n_clients)
    p = BatchParams(isolation=True)
    for _ in range(3):
        eng.process_device(d_in, n, p, bufs)
        eng.lib.mpsf_get_summary(eng.ctx, None) if False else None
    torch.cuda.synchronize()
    eng.set_profiling(True)
    for _ in range(reps):
        eng.process_device(d_in, n, p, bufs)
    prof = eng.profile()
    res = {k: round(v[1] / max(v[0], 1), 4) for k, v in prof.items()}
    if "k_batch" in res:
        import ctypes
        ts = (ctypes.c_uint64 * 8)()
        eng.lib.mpsf_debug_phase_times(ctypes.cast(ts, ctypes.c_void_p))
        names = ["clear", "scan", "resolve", "finalize", "lists"]
        res["phases_us"] = {names[k]: round((ts[k + 1] - ts[k]) / 1e3, 1) for k in range(5)}
    return res


def main():
    if sys.argv[1] == "build":
        build(sys.argv[2:])
        return
    if sys.argv[1] == "one":
        print(json.dumps(one(sys.argv[2], sys.argv[3], int(sys.argv[4]))))
        return
    wl = sys.argv[2]
    for m in sys.argv[3:]:
        lib = os.path.join(OUT, f"libmpsf_{m}.so") if m != "prod" else os.path.join(
            ROOT, "paper_2605_26461_b200", "libmpsf.so")
        r = subprocess.run([sys.executable, __file__, "one", wl, lib, "10"], capture_output=True, text=True)
        line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-500:]
        print(f"{wl} mask={m}: {line}", flush=True)


if __name__ == "__main__":
    main()
