"""Experiment tool: A/B timing of libmpsf.so variants built with extra -D defines.

    python tools/variants.py build name=-DFOO,-DBAR name2= ...   # here: build/var/libmpsf_<name>.so
    python tools/variants.py run c2b,c3 name name2 ...            # on the GPU box

Per variant and workload: the device-resident step time (CUDA events, L2 flushed between steps,
median of 15) and the per-kernel times of a separate profiled pass; the outputs of every variant
are compared with the first one's (a variant that changes results is flagged)."""
import glob
import hashlib
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "build", "var")


def build(specs):
    os.makedirs(OUT, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(ROOT, "paper_2605_26461_b200", "csrc", "*.cu")) +
                  glob.glob(os.path.join(ROOT, "paper_2605_26461_b200", "csrc", "*.cpp")))
    procs = []
    for spec in specs:
        name, _, defs = spec.partition("=")
        lib = os.path.join(OUT, f"libmpsf_{name}.so")
        cmd = ["nvcc", "-O3", "-lineinfo", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a",
               "-Xcompiler", "-fPIC,-O3", "-I", os.path.join(ROOT, "include"),
               *[d for d in defs.split(",") if d], "-shared", "-o", lib, *srcs]
        procs.append(subprocess.Popen(cmd))
    for p in procs:
        assert p.wait() == 0


def one(wl, lib):
    os.environ["MPSF_LIB"] = lib
    sys.path.insert(0, ROOT)
    import numpy as np
    import statistics
    import torch
    from paper_2605_26461_b200 import synth
    from paper_2605_26461_b200.engine import BatchParams, DeviceBuffers, FaultEngine
    if wl == "c3":
        w, _ = synth.build_synthetic_world(48, 8192, 3)
        n = int(os.environ.get("STORM_N", 100_000_000))
        d_in = synth.generate_storm(w, n, n // 10, 3, device="cuda")
    else:
        cache = f"/tmp/var_{wl}.npy"
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
        res = eng.process_resident(d_in, n, p, bufs)
    h = hashlib.sha1()
    for f in ("out", "verdict", "counts", "dedup_keys", "dedup_idx", "cancel"):
        h.update(np.ascontiguousarray(getattr(res, f)).tobytes())
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ts = []
    for _ in range(15):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        eng.process_device(d_in, n, p, bufs)
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    eng.set_profiling(True)
    for _ in range(5):
        flush.zero_()
        eng.process_device(d_in, n, p, bufs)
    prof = eng.profile()
    return {"step_ms": round(statistics.median(ts), 4), "digest": h.hexdigest()[:12],
            **{k: round(v[1] / max(v[0], 1), 4) for k, v in sorted(prof.items())}}


def main():
    if sys.argv[1] == "build":
        build(sys.argv[2:])
        return
    if sys.argv[1] == "one":
        print(json.dumps(one(sys.argv[2], sys.argv[3])))
        return
    for wl in sys.argv[2].split(","):
        ref = None
        for name in sys.argv[3:]:
            lib = os.path.join(OUT, f"libmpsf_{name}.so") if name != "prod" else os.path.join(
                ROOT, "paper_2605_26461_b200", "libmpsf.so")
            r = subprocess.run([sys.executable, __file__, "one", wl, lib], capture_output=True, text=True)
            line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-800:]
            try:
                d = json.loads(line)
                ref = ref or d["digest"]
                if d["digest"] != ref:
                    d["RESULTS_DIFFER"] = True
                line = json.dumps(d)
            except Exception:
                pass
            print(f"{wl} {name}: {line}", flush=True)


if __name__ == "__main__":
    main()
