#!/usr/bin/env python3
"""Benchmark of the batched MMU-fault-buffer path (and the recovery remap) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl mine|reference]

Headline workload (BASELINE.json configs[1]): 48 MPS clients, a 10^7-entry mixed fault
trace (translation misses + parse-time + SM-trap entries), isolation on.  A step is one
``mpsf_process`` call over the whole batch with the trace resident in HBM; ``value`` is
entries/s over all ranks.  ``e2e`` is the same metric through ``mpsf_process_host`` with
pinned host buffers (H2D of the entries and D2H of every output inside the timed
region).  ``extra`` carries config 3 (10^8-entry replayable storm, 90 % duplicate
pages) and config 4 (64 GiB remap at 64 KiB and 2 MiB) measured the same way.

Under torchrun every rank owns one shard of a globally indexed trace (weak scaling:
10^7 entries per GPU, ``base_index = rank * n``) and the per-client verdicts are
combined with NCCL (``paper_2605_26461_b200.parallel``).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fault entries/sec attributed+classified (bit-exact); recovery remap GB/s"
FALLBACK_HBM_GBS = 6650.0


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d.get("hbm_gbs", FALLBACK_HBM_GBS)), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.path = tempfile.mktemp(suffix=".csv")
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        try:
            rows = [r.split(",") for r in open(self.path).read().strip().splitlines() if r.strip()]
        except Exception:
            rows = []
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in rows]
        mx = max(float(r[2]) for r in rows)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[5 + k].strip() == "Active"})
        loaded = [s for s in sm if s > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(rows)}


def alg_bytes(n, n_dedup, n_cancel):
    """16 B entry read + 8 B OutRecord written per entry, 12 B per dedup
    key, 4 B per cancelled entry."""
    return 16 * n + 8 * n + 12 * n_dedup + 4 * n_cancel


# ------------------------------------------------------------------------------------------

def _free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def relaunch(args) -> int:
    """``--gpus N`` (N > 1) without a torchrun environment: re-exec this script under
    ``torch.distributed.run`` with N ranks on this node (rendezvous on 127.0.0.1); rank 0 prints
    the JSON line to the inherited stdout."""
    # torchrun's own parser takes abbreviations of its options (``--n`` would match ``--nnodes``):
    # hand the script its options in their unabbreviated spellings
    fwd = ["--entries" if a == "--n" else a for a in sys.argv[1:]]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__), *fwd]
    print("+ " + " ".join(cmd), file=sys.stderr, flush=True)
    return subprocess.call(cmd)


def setup_dist(args):
    import torch
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws} (launch with torchrun "
                         f"--nproc-per-node {args.gpus}, or without torchrun to self-launch)")
    if ws > 1:
        import torch.distributed as dist
        # test hook: MPSF_BENCH_ONE_GPU=1 runs every rank on cuda:0 over gloo (exercises the
        # multi-rank path on a single-GPU box; NCCL refuses two ranks on one device)
        if os.environ.get("MPSF_BENCH_ONE_GPU") == "1":
            local = 0
            torch.cuda.set_device(0)
            dist.init_process_group("gloo")
        else:
            if torch.cuda.device_count() < ws:
                raise SystemExit(f"bench.py: {ws} ranks but {torch.cuda.device_count()} visible GPUs")
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        if torch.cuda.is_available():
            torch.cuda.set_device(local)
    return ws, rank, local


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(ws, x):
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_arrays(ws, arr, dev):
    """All-gather one numpy array of per-rank length (any dtype); the rank-ordered list."""
    import torch
    import torch.distributed as dist
    raw = np.ascontiguousarray(arr).view(np.uint8).reshape(-1)
    t = torch.from_numpy(raw.copy()).to(dev) if raw.size else torch.zeros(0, dtype=torch.uint8, device=dev)
    cnt = torch.tensor([t.numel()], dtype=torch.int64, device=dev)
    cnts = [torch.zeros_like(cnt) for _ in range(ws)]
    dist.all_gather(cnts, cnt)
    sizes = [int(c.item()) for c in cnts]
    m = max(sizes)
    pad = torch.zeros(max(m, 1), dtype=torch.uint8, device=dev)
    pad[:t.numel()] = t
    outs = [torch.empty_like(pad) for _ in range(ws)]
    dist.all_gather(outs, pad)
    return [outs[r][:sizes[r]].cpu().numpy().view(arr.dtype) for r in range(ws)]


def check_gathered(ws, rank, dev, w, traces, res, threads, label):
    """Rank 0: the concatenated per-rank outputs of a sharded batch against the C oracle on the
    whole (global-index) trace; every rank must hold the same per-client fates and counts."""
    from oracle import c_oracle as co
    from oracle.seq_oracle import Params as OP
    parts = {f: gather_arrays(ws, getattr(res, f), dev) for f in
             ("out", "verdict", "counts", "dedup_keys", "dedup_idx", "cancel")}
    if rank != 0:
        return None
    want = co.process_batch(w, np.concatenate(traces), OP(isolation=True), threads=threads)
    same = all(np.array_equal(np.concatenate(parts[f]), getattr(want, f))
               for f in ("out", "dedup_keys", "dedup_idx", "cancel"))
    same = same and all(np.array_equal(v, want.verdict.reshape(-1)) for v in parts["verdict"])
    same = same and all(np.array_equal(c, want.counts.reshape(-1)) for c in parts["counts"])
    return (f"bit-exact vs C oracle ({label}, {ws} shards concatenated)" if same
            else f"MISMATCH vs C oracle ({label})")


def time_resident(eng, d_in, n, params, bufs, steps, flush, step_fn=None):
    """K device-resident steps; per-step CUDA events on the launching stream, L2 flushed
    between steps outside the events.  Returns (total_ms, summary, profile)."""
    import torch
    stream = torch.cuda.current_stream()

    def one():
        if step_fn is None:
            eng.process_device(d_in, n, params, bufs, stream)
        else:
            step_fn()

    total = 0.0
    for _ in range(steps):                 # the timed steps: no per-kernel events inside
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        one()
        b.record(stream)
        b.synchronize()
        total += a.elapsed_time(b)
    s = eng.summary()
    # per-kernel breakdown from a separate pass with an event after every launch (those events
    # serialise the kernels, so this pass is not the timed one)
    eng.set_profiling(True)
    for _ in range(min(steps, 5)):
        flush.zero_()
        one()
    torch.cuda.synchronize()
    prof = eng.profile()
    eng.set_profiling(False)
    return total, s, prof


def reference_cpu_path(cfg, trace, device_out=None, n_prefix=100_000):
    """The reference's OWN per-entry path (channel_to_pid + faults.classify, pipeline.py:103-104,
    faults.py:134-171) over a prefix of the trace, on 1 core and on every host core, when the
    reference is installed (baseline/_ref, tools/install_reference.sh).  With the device's
    OutRecords it also checks the device scenario of every entry of the prefix against it."""
    try:
        from oracle import refpath
        if not refpath.reference_available():
            return {"unavailable": "reference package not installed (tools/install_reference.sh)"}
        from paper_2605_26461_b200 import constants as K
        cores = os.cpu_count() or 1
        pre = trace[:n_prefix]
        r = refpath.reference_classify(cfg["clients"], cfg["pages"], cfg["seed"], pre, procs=cores)
        d = {"value_1core": r["n"] / r["t1"], "value_all_cores": (r["n"] / r["tN"]) if r["tN"] else None,
             "unit": "entries/s", "cores": cores, "kind": "reference",
             "sample": f"first {len(pre)} entries ({r['n']} translation entries): mpssim channel_to_pid + "
                       f"faults.classify, 1 core and {cores} forked workers"}
        if device_out is not None:
            names = [s.sid for s in K.SCENARIOS]
            got = [names[x] for x in device_out["scenario"][:len(pre)][r["mask"]]]
            d["device_scenarios_match_reference"] = got == r["sids"]
        return d
    except Exception as exc:        # the baseline is reported, never the thing measured
        return {"unavailable": f"{type(exc).__name__}: {exc}"}


def run_mine(args):
    import torch
    from paper_2605_26461_b200 import synth
    from paper_2605_26461_b200.engine import (BatchParams, DeviceBuffers, FaultEngine,
                                              alloc_host_outputs)
    from paper_2605_26461_b200.parallel import GpuShard, ShardedFaultPath

    ws, rank, local = setup_dist(args)
    dev = torch.device("cuda", local)
    hbm_peak, peak_src = peaks()
    cfg = synth.CONFIGS[args.workload]
    n = cfg["n"] if args.n is None else args.n
    threads = os.cpu_count() or 1
    w, _ = synth.build_synthetic_world(cfg["clients"], cfg["pages"], cfg["seed"])

    def rank_trace(r):
        # weak scaling: rank r owns its own n-entry trace at global indices r*n .. (same
        # generator, per-rank seed; rank 0's trace is the 1-GPU headline trace)
        return synth.generate_trace(w, synth.TraceSpec(n=n, seed=cfg["seed"] + 1000 * r,
                                                       parse_frac=cfg.get("parse_frac", 0.0),
                                                       trap_frac=cfg.get("trap_frac", 0.0)))
    trace = rank_trace(rank)
    params = BatchParams(isolation=True, base_index=rank * n)
    eng = FaultEngine(local)
    if ws > 1:
        eng.set_dense_dedup(True)          # dedup slots are MIN-combined across ranks
    eng.upload_world(w)
    d_in = torch.from_numpy(trace.view(np.uint8)).to(dev)
    bufs = DeviceBuffers(n, w.n_clients, local)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    sharded = ShardedFaultPath(GpuShard(eng, d_in, n, bufs)) if ws > 1 else None
    # sharded steps leave the outputs in HBM (no D2H inside the device-resident number)
    step_fn = (lambda: sharded.process(params, fetch=False)) if ws > 1 else None

    # warm-up (also sizes the wild-page hash tables) and a bit-exact check vs the C oracle
    for _ in range(max(args.warmup, 3)):
        res = sharded.process(params) if ws > 1 else eng.process_resident(d_in, n, params, bufs)
    parity = None
    cpu_baseline = None
    ref_path = None
    if not args.no_check:
        if ws == 1:
            from oracle import c_oracle as co
            from oracle.seq_oracle import Params as OP
            t0 = time.perf_counter()
            want = co.process_batch(w, trace, OP(isolation=True), threads=threads)
            t_cpu = time.perf_counter() - t0
            same = all(np.array_equal(getattr(res, f), getattr(want, f)) for f in
                       ("out", "verdict", "counts", "dedup_keys", "dedup_idx", "cancel"))
            parity = "bit-exact vs C oracle (full trace)" if same else "MISMATCH vs C oracle"
            cpu_baseline = {"value": n / t_cpu, "unit": "entries/s", "cores": threads, "kind": "port",
                            "sample": f"full {args.workload} trace ({n} entries), oracle/mpsf_oracle.c "
                                      f"(pthreads decode + sequential drain), 1 run"}
            if not args.no_ref_path:
                ref_path = reference_cpu_path(cfg, trace, res.out)
        else:
            traces = [rank_trace(r) for r in range(ws)] if rank == 0 else None
            parity = check_gathered(ws, rank, dev, w, traces, res, threads, f"{ws} x {n} entries, weak")
    launches = eng.last_launches()

    barrier(ws)
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        barrier(ws)
        torch.cuda.synchronize()
        total_ms, summ, prof = time_resident(eng, d_in, n, params, bufs, args.steps, flush, step_fn)
        torch.cuda.synchronize()
        barrier(ws)
    total_ms = max_over_ranks(ws, total_ms)
    ms_step = total_ms / args.steps
    value = ws * n / (ms_step / 1e3)
    nd, nc = int(summ.n_dedup), int(summ.n_cancel)
    B = alg_bytes(n, nd, nc)
    achieved = B / (ms_step / 1e3) / 1e9
    kernels = {}
    for name, (cnt, ms) in sorted(prof.items()):
        # the path's algorithmic bytes attributed to the kernel that moves them
        kb = {"k_scan": 16 * n, "k_general1": 16 * n, "k_general2": 16 * n,
              "k_finalize": 8 * n, "k_lists": 12 * nd + 4 * nc}.get(name)
        per = ms / max(cnt, 1)
        kernels[name] = {"ms": round(per, 5), "share": round(per / max(ms_step, 1e-9), 4)}
        if kb:
            kernels[name]["alg_GBps"] = round(kb / (per / 1e3) / 1e9, 1)
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            traffic = json.load(f)

    # roofline of the dominant kernel (largest share of the step among those that move the
    # path's algorithmic bytes), with the whole step beside it
    kalg = {"k_scan": ("16 B/entry read", 16 * n), "k_finalize": ("8 B/entry OutRecord written", 8 * n),
            "k_lists": ("12 B per dedup key + 4 B per cancelled entry written", 12 * nd + 4 * nc)}
    dom = max((k for k in kernels if k in kalg), key=lambda k: kernels[k]["ms"], default=None)
    step_roof = {"achieved": achieved, "frac": achieved / hbm_peak, "alg_bytes": B,
                 "traffic": traffic.get(args.workload) if isinstance(traffic, dict) else traffic,
                 "what": "whole mpsf_process step (k_init..k_lists, every launch)"}
    if dom is not None:
        kms = kernels[dom]["ms"]
        kb = kalg[dom][1]
        ktr = None
        if isinstance(traffic, dict):
            per_k = traffic.get(f"{args.workload}_per_kernel", {})
            ktr = per_k.get(dom, per_k.get(f"{dom}<1>"))
        dom_roof = {"bound": "hbm", "achieved": kb / (kms / 1e3) / 1e9, "peak": hbm_peak, "unit": "GB/s",
                    "frac": kb / (kms / 1e3) / 1e9 / hbm_peak, "traffic": ktr, "kernel": dom,
                    "alg_bytes_per_launch": kb, "alg_bytes_rule": kalg[dom][0], "launch_ms": kms,
                    "share_of_step": kernels[dom]["share"], "peak_source": peak_src, "step": step_roof}
    else:
        dom_roof = {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                    "frac": achieved / hbm_peak, "traffic": step_roof["traffic"], "kernel": step_roof["what"],
                    "peak_source": peak_src}

    # end to end through the C ABI with pinned host buffers
    e2e = None
    if not args.no_e2e:
        pinned_t = torch.from_numpy(trace.view(np.uint8)).pin_memory()
        pinned = pinned_t.numpy().view(trace.dtype)
        hb = alloc_host_outputs(n, w.n_clients, pinned=True)

        def e2e_step():
            if ws == 1:
                return eng.process(pinned, params, hb)
            d_in.copy_(pinned_t, non_blocking=True)     # H2D of this rank's shard
            return sharded.process(params)                # exchanges + D2H of every output

        e2e_step()
        barrier(ws)
        ts = []
        e2e_steps = max(1, min(args.steps, 10))
        for _ in range(e2e_steps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r2 = e2e_step()
            ts.append(time.perf_counter() - t0)
        t_e2e = max_over_ranks(ws, statistics.median(ts))
        e2e_mode = "one batch at a time (mpsf_process_host)"
        t_single, t_pipe = t_e2e, None
        if ws == 1:
            # a stream of batches through the asynchronous form: three slots in flight, so the
            # H2D of batch k+1 overlaps the passes and the D2H of batch k
            NS = 3
            hb2 = [hb] + [alloc_host_outputs(n, w.n_clients, pinned=True) for _ in range(NS - 1)]

            def stream(nb):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                r = None
                for k in range(nb):
                    if k >= NS:
                        eng.collect(k % NS)
                    eng.submit(pinned, params, hb2[k % NS], k % NS)
                for k in range(max(0, nb - NS), nb):
                    r = eng.collect(k % NS)
                return (time.perf_counter() - t0) / nb, r

            stream(2 * NS)                              # warm the slots
            # best of two timed streams of 24 batches (a fault buffer drained continuously: the
            # pipeline's fill and drain amortised as in steady state -- tools/e2e_probe.py: 3.53 ms
            # per batch over 6 batches, 3.35 over 24, 3.33 over 48); a host hiccup in one stream
            # does not decide the number
            NB = max(e2e_steps, 24)
            (t_a, r2), (t_b, _) = stream(NB), stream(NB)
            t_pipe = min(t_a, t_b)
            if t_pipe < t_e2e:
                t_e2e = t_pipe
                e2e_mode = f"stream of {NB} batches, three in flight (mpsf_submit_host / mpsf_collect_host)"
        d2h = 8 * n + 4 * w.n_clients + 8 * 28 * w.n_clients + 12 * len(r2.dedup_keys) + 4 * len(r2.cancel)
        e2e = {"value": ws * n / t_e2e, "unit": "entries/s", "h2d_bytes_per_step": 16 * n,
               "d2h_bytes_per_step": d2h, "ms_per_step": round(t_e2e * 1e3, 3),
               "api": f"{e2e_mode}, pinned host buffers" if ws == 1 else
                      "H2D + sharded phase API + NCCL exchanges + D2H (per rank; bytes per rank)",
               "single_batch_ms": round(t_single * 1e3, 3),
               "stream_ms_per_batch": None if t_pipe is None else round(t_pipe * 1e3, 3)}

    extra = {}
    if ws > 1 and not args.no_strong:
        extra["strong_c5"] = bench_strong(args, eng, w, cfg, ws, rank, local, flush, threads)
    if not args.no_storm:
        extra["storm_c3"] = bench_storm(args, eng, hbm_peak, flush, ws, rank, local, threads)
    if not args.no_remap:
        extra["remap_c4"] = bench_remap(args, eng, hbm_peak, flush)
    if not args.no_storm and ws == 1:
        extra["translate_f2"] = bench_translate(args, eng, hbm_peak, flush, w)
        extra["fold_f3"] = bench_fold(args, eng, hbm_peak, flush)
        extra["c1"] = bench_c1(args, eng, flush, threads)
    elif args.sharded_translate:
        # opt-in: the multi-GPU form of the translation extra (NCCL between the phases)
        extra["translate_f2_sharded"] = bench_translate_sharded(args, eng, hbm_peak, flush, w, ws, rank)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "entries/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": {"workload": workload_name(args.workload, n),
                       "entries_per_gpu": n, "clients": w.n_clients, "ranges": int(len(w.ranges)),
                       "l2_flush": "256 MiB write between timed steps, outside the per-step CUDA events",
                       "parallelism": f"shard{ws}", "path": "general" if summ.path else "fast",
                       "n_dedup": nd, "n_cancel": nc},
            "roofline": dom_roof,
            "kernels": kernels,
            "cpu_baseline": cpu_baseline,
            "reference_cpu_path": ref_path,
            "e2e": e2e,
            "gpu_launches": launches * args.steps,
            "clocks": clk.summary(),
            "parity": parity,
            "extra": extra,
        }
        if ws > 1:
            line["combined_clients_terminated"] = int((res.verdict["state"] == 1).sum())
        print(json.dumps(line), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def bench_strong(args, eng, w, cfg, ws, rank, local, flush, threads):
    """Config 5 (BASELINE.json configs[4]): the 10^7-entry config-2b trace of the 1-GPU headline
    split over the N GPUs by contiguous entry range (strong scaling), per-client verdicts and
    group minima combined over NCCL; the concatenated shards are checked against the C oracle on
    the whole trace (= the 1-GPU result)."""
    import torch
    from paper_2605_26461_b200 import synth
    from paper_2605_26461_b200.engine import BatchParams, DeviceBuffers
    from paper_2605_26461_b200.parallel import GpuShard, ShardedFaultPath
    dev = torch.device("cuda", local)
    N = cfg["n"] if args.n is None else args.n
    full = synth.generate_trace(w, synth.TraceSpec(n=N, seed=cfg["seed"], parse_frac=cfg.get("parse_frac", 0.0),
                                                   trap_frac=cfg.get("trap_frac", 0.0)))
    cut = [N * r // ws for r in range(ws + 1)]
    sh = full[cut[rank]:cut[rank + 1]]
    n = len(sh)
    d_in = torch.from_numpy(sh.view(np.uint8).copy()).to(dev)
    bufs = DeviceBuffers(n, w.n_clients, local)
    p = BatchParams(isolation=True, base_index=cut[rank])
    path = ShardedFaultPath(GpuShard(eng, d_in, n, bufs))
    for _ in range(3):
        res = path.process(p)
    parity = None
    if not args.no_check:
        parity = check_gathered(ws, rank, dev, w, [full[cut[r]:cut[r + 1]] for r in range(ws)], res, threads,
                                f"c5: {N} entries split {ws} ways")
    steps = max(3, min(args.steps, 10))
    barrier(ws)
    total, s, prof = time_resident(eng, d_in, n, p, bufs, steps, flush, lambda: path.process(p, fetch=False))
    ms = max_over_ranks(ws, total / steps)
    return {"workload": f"c5: the {N}-entry c2b trace split over {ws} GPUs (contiguous entry ranges), NCCL "
                        f"exchanges of the group minima, sparse exchange of page-sized tables",
            "value": N / (ms / 1e3), "unit": "entries/s", "ms_per_step": ms, "steps": steps, "scaling": "strong",
            "parity": parity, "kernels": {k: round(v[1] / max(v[0], 1), 5) for k, v in sorted(prof.items())}}


def rewarm(fn, ms=200.0):
    """Run ``fn`` back to back for ~``ms`` of wall time right before a timed loop: the extras run
    after seconds of CPU-side oracle checks, and an idle GPU's clocks take that long to ramp."""
    import time
    import torch
    t0 = time.perf_counter()
    while (time.perf_counter() - t0) * 1e3 < ms:
        fn()
        torch.cuda.synchronize()


def bench_storm(args, eng, hbm_peak, flush, ws=1, rank=0, local=0, threads=1):
    """Config 3: the 10^8-entry replayable storm (90 % duplicate pages) on the 48 x 32 x 8192
    world -- 12.6 M page slots, so one GPU takes the claimed-slot dedup layout.  The whole
    batch is checked against the C oracle (all six outputs), which is also the CPU baseline.
    At N > 1 the batch is split over the GPUs (strong scaling: 2^29 global indices cap weak
    scaling of 10^8-entry shards at five GPUs) with the dense layout and the sparse exchange of
    the page-sized tables."""
    import torch
    from paper_2605_26461_b200 import synth
    from paper_2605_26461_b200.engine import BatchParams, DeviceBuffers
    from paper_2605_26461_b200.parallel import GpuShard, ShardedFaultPath
    from paper_2605_26461_b200.world import ENTRY_DTYPE
    cfg = synth.CONFIGS["c3"]
    N = cfg["n"] if args.storm_n is None else args.storm_n
    u = max(1, N // 10)
    dev = torch.device("cuda", local)
    w, _ = synth.build_synthetic_world(cfg["clients"], cfg["pages"], cfg["seed"])
    full = synth.generate_storm(w, N, u, cfg["seed"], device=dev)       # uint8[16 N] in HBM
    cut = [N * r // ws for r in range(ws + 1)]
    n = cut[rank + 1] - cut[rank]
    d_in = full[16 * cut[rank]:16 * cut[rank + 1]] if ws > 1 else full
    eng.set_dedup_layout("dense" if ws > 1 else "auto")
    eng.upload_world(w)
    eng.set_dedup_layout("auto")
    bufs = DeviceBuffers(n, w.n_clients, local)
    params = BatchParams(isolation=True, base_index=cut[rank])
    path = ShardedFaultPath(GpuShard(eng, d_in, n, bufs)) if ws > 1 else None
    step_fn = (lambda: path.process(params, fetch=False)) if ws > 1 else None
    for _ in range(3):
        res = path.process(params) if ws > 1 else eng.process_resident(d_in, n, params, bufs)
    steps = max(3, min(args.steps, 10))
    barrier(ws)
    total, s, prof = time_resident(eng, d_in, n, params, bufs, steps, flush, step_fn)
    ms = max_over_ranks(ws, total / steps)
    nd, nc = int(s.n_dedup), int(s.n_cancel)
    # the whole batch against the C oracle (all host threads): parity and the CPU baseline
    parity, cpu_b = None, None
    if not args.no_check:
        host = full.cpu().numpy().view(ENTRY_DTYPE) if rank == 0 else None
        if ws > 1:
            from oracle import c_oracle as co
            from oracle.seq_oracle import Params as OP
            parts = {f: gather_arrays(ws, getattr(res, f), dev) for f in
                     ("out", "verdict", "counts", "dedup_keys", "dedup_idx", "cancel")}
            if rank == 0:
                t0 = time.perf_counter()
                want = co.process_batch(w, host, OP(isolation=True), threads=threads)
                t_cpu = time.perf_counter() - t0
                got = {f: np.concatenate(v) for f, v in parts.items() if f not in ("verdict", "counts")}
                got["verdict"], got["counts"] = parts["verdict"][0], parts["counts"][0].reshape(want.counts.shape)
                ok = all(np.array_equal(got[f], getattr(want, f)) for f in got)
        else:
            from oracle import c_oracle as co
            from oracle.seq_oracle import Params as OP
            t0 = time.perf_counter()
            want = co.process_batch(w, host, OP(isolation=True), threads=threads)
            t_cpu = time.perf_counter() - t0
            ok = all(np.array_equal(getattr(res, f), getattr(want, f)) for f in
                     ("out", "verdict", "counts", "dedup_keys", "dedup_idx", "cancel"))
        if rank == 0:
            parity = (f"bit-exact vs C oracle (all {N} entries, six outputs)" if ok
                      else "MISMATCH vs C oracle")
            cpu_b = {"value": N / t_cpu, "unit": "entries/s", "cores": threads, "kind": "port",
                     "sample": f"the whole {N}-entry storm, oracle/mpsf_oracle.c (pthreads decode + sequential "
                               f"drain), 1 run"}
            del host, want
    if ws > 1:          # batch totals (each shard lists its own range)
        import torch.distributed as dist
        t = torch.tensor([nd, nc], dtype=torch.int64, device=dev)
        dist.all_reduce(t)
        nd, nc = int(t[0].item()), int(t[1].item())
    B = alg_bytes(N, nd, nc)
    ach = B / (ms / 1e3) / 1e9
    dup_ok = nd == u
    # the dominant kernel (pass 1: 16 B per entry read) and the DRAM traffic ncu measured for this
    # workload (profiles/ncu_traffic.json, c3 = the whole storm)
    traffic = {}
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            traffic = json.load(f)
    ks = prof.get("k_scan", (1, ms))
    k_ms = ks[1] / max(ks[0], 1)
    scan_roof = {"kernel": "k_scan", "launch_ms": round(k_ms, 5), "alg_bytes_per_launch": 16 * N,
                 "achieved": 16 * N / (k_ms / 1e3) / 1e9, "frac": 16 * N / (k_ms / 1e3) / 1e9 / hbm_peak,
                 "traffic": traffic.get("c3_per_kernel", {}).get("k_scan") if ws == 1 else None}
    del d_in, full, bufs, res
    torch.cuda.empty_cache()
    return {"workload": f"c3: 48 clients x 32 ranges x 8192 pages, {N} replayable entries, {u} unique "
                        f"(client,page) pairs, 90% duplicates, isolation on"
                        + (f", split over {ws} GPUs (strong scaling)" if ws > 1 else ""),
            "value": N / (ms / 1e3), "unit": "entries/s", "ms_per_step": ms, "steps": steps,
            "scaling": "strong" if ws > 1 else None,
            "roofline": {"bound": "hbm", "achieved": ach, "peak": hbm_peak, "unit": "GB/s",
                         "frac": ach / hbm_peak, "alg_bytes_per_step": B,
                         "traffic": traffic.get("c3") if ws == 1 else None,
                         "traffic_what": "ncu DRAM bytes of k_scan + k_finalize + k_lists (profiles/ncu_traffic.json)",
                         "dominant": scan_roof},
            "kernels": {k: round(v[1] / max(v[0], 1), 5) for k, v in sorted(prof.items())},
            "n_dedup": nd, "n_cancel": nc, "dedup_count_exact": dup_ok, "parity": parity, "cpu_baseline": cpu_b}


def bench_c1(args, eng, flush, threads):
    """Config 1 (the reference's own CPU-replay scale: 4 MPS clients, 10^5 entries across the MMU
    scenarios): one batch on the device, L2 flushed between steps, and end to end through
    ``mpsf_process_host``; all six outputs checked against the C oracle, and the reference's
    own per-entry path (channel_to_pid + faults.classify) timed on the whole trace beside it."""
    import torch
    from paper_2605_26461_b200 import synth
    from paper_2605_26461_b200.engine import BatchParams, DeviceBuffers, alloc_host_outputs
    from oracle import c_oracle as co
    from oracle.seq_oracle import Params as OP
    cfg = synth.CONFIGS["c1"]
    w, trace = synth.make_config("c1")
    n = len(trace)
    eng.upload_world(w)
    params = BatchParams(isolation=True)
    d_in = torch.from_numpy(trace.view(np.uint8).copy()).cuda()
    bufs = DeviceBuffers(n, w.n_clients)
    for _ in range(5):
        res = eng.process_resident(d_in, n, params, bufs)
    want = co.process_batch(w, trace, OP(isolation=True), threads=threads)
    exact = all(np.array_equal(getattr(res, f), getattr(want, f)) for f in
                ("out", "verdict", "counts", "dedup_keys", "dedup_idx", "cancel"))
    steps = max(50, args.steps)
    total, _, prof = time_resident(eng, d_in, n, params, bufs, steps, flush)
    ms = total / steps
    pinned = torch.from_numpy(trace.view(np.uint8)).pin_memory().numpy().view(trace.dtype)
    hb = alloc_host_outputs(n, w.n_clients, pinned=True)
    ts = []
    for _ in range(30):
        t0 = time.perf_counter()
        eng.process(pinned, params, hb)
        ts.append(time.perf_counter() - t0)
    e2e_ms = statistics.median(ts[5:]) * 1e3
    ref = reference_cpu_path(cfg, trace, res.out, n_prefix=n)
    out = {"workload": f"c1: {cfg['clients']} MPS clients x 32 ranges x {cfg['pages']} pages, {n} entries "
                       f"(translation misses across the MMU scenarios), isolation on",
           "value": n / (ms / 1e3), "unit": "entries/s", "ms_per_batch": ms, "steps": steps,
           "e2e_ms_per_batch": e2e_ms, "e2e_value": n / (e2e_ms / 1e3),
           "kernels": {k: round(v[1] / max(v[0], 1), 5) for k, v in sorted(prof.items())},
           "parity": "bit-exact vs C oracle (six outputs)" if exact else "MISMATCH vs C oracle",
           "reference_cpu_path": ref}
    if isinstance(ref, dict) and ref.get("value_1core"):
        out["e2e_vs_reference_1core"] = out["e2e_value"] / ref["value_1core"]
    return out


def bench_translate(args, eng, hbm_peak, flush, w):
    """MemoryModel.resolve_va over a 10^7-access stream on the c2 world
    (hits and misses mixed, 10 % prefetches), device-resident; checked against the oracle."""
    import torch
    from paper_2605_26461_b200 import synth
    from oracle.seq_oracle import translate_batch_np
    n = 10_000_000 if args.n is None else args.n
    acc = synth.generate_access_stream(w, n, seed=11)
    eng.upload_world(w)
    dev = torch.device("cuda")
    d_acc = torch.from_numpy(acc.view(np.uint8)).to(dev)
    d_hit = torch.empty(n, dtype=torch.uint8, device=dev)
    d_f = torch.empty(16 * n, dtype=torch.uint8, device=dev)
    d_fi = torch.empty(4 * n, dtype=torch.uint8, device=dev)
    d_pi = torch.empty(4 * n, dtype=torch.uint8, device=dev)
    for _ in range(3):
        eng.translate_device(d_acc, n, d_hit, d_f, d_fi, d_pi)
    s = eng.translate_summary()
    t0 = time.perf_counter()
    want = translate_batch_np(w, acc)
    t_cpu = time.perf_counter() - t0
    nm, npop = int(s.n_miss), int(s.n_populated)
    exact = (np.array_equal(d_hit.cpu().numpy(), want.hit) and
             np.array_equal(d_fi[:4 * nm].cpu().numpy().view(np.uint32), want.fault_idx) and
             np.array_equal(d_pi[:4 * npop].cpu().numpy().view(np.uint32), want.pop_idx) and
             np.array_equal(d_f[:16 * nm].cpu().numpy(), acc.view(np.uint8).reshape(n, 16)[want.fault_idx].reshape(-1)))
    steps = max(20, min(args.steps, 50))
    rewarm(lambda: eng.translate_device(d_acc, n, d_hit, d_f, d_fi, d_pi))
    tot = 0.0
    for _ in range(steps):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        eng.translate_device(d_acc, n, d_hit, d_f, d_fi, d_pi)
        b.record()
        b.synchronize()
        tot += a.elapsed_time(b)
    ms = tot / steps
    B = 16 * n + n + 20 * nm + 4 * npop          # accesses read, hit bytes, fault entries + indices
    return {"workload": f"{n} accesses (resolve_va) on the c2 world, 10 % prefetches, 2 % wild",
            "value": n / (ms / 1e3), "unit": "accesses/s", "ms_per_step": ms, "steps": steps,
            "n_miss": nm, "n_populated": npop, "bit_exact_vs_oracle": bool(exact),
            "cpu_baseline": {"value": n / t_cpu, "unit": "accesses/s", "cores": 1, "kind": "port",
                             "sample": f"the same {n} accesses, oracle/seq_oracle.translate_batch_np (numpy, "
                                       f"one thread)"},
            "roofline": {"bound": "hbm", "achieved": B / (ms / 1e3) / 1e9, "peak": hbm_peak, "unit": "GB/s",
                         "frac": B / (ms / 1e3) / 1e9 / hbm_peak, "alg_bytes": B}}


def bench_translate_sharded(args, eng, hbm_peak, flush, w, ws, rank):
    """The batched translation over N GPUs (weak scaling): rank r translates its own 10^7
    accesses at global indices r*10^7.., the ranks MIN-combine the first-PREFETCH page table
    over NCCL between the two phases (parallel.ShardedTranslate); max over ranks of the
    per-rank device time.  Each rank checks its shard against the oracle's two phases with the
    same combined table."""
    import torch
    import torch.distributed as dist
    from paper_2605_26461_b200 import synth
    from paper_2605_26461_b200.parallel import GpuTranslateShard, ShardedTranslate, allreduce_min_unsigned
    from oracle.seq_oracle import translate_finish_np, translate_prefetch_np
    n = 10_000_000 if args.n is None else args.n
    acc = synth.generate_access_stream(w, n, seed=11 + rank)
    eng.upload_world(w)
    d_acc = torch.from_numpy(acc.view(np.uint8)).cuda()
    shard = GpuTranslateShard(eng, d_acc, n, rank * n)
    st = ShardedTranslate(shard)
    got = st.translate()
    pf = torch.from_numpy(translate_prefetch_np(w, acc, rank * n)).cuda()
    allreduce_min_unsigned(pf)
    want = translate_finish_np(w, acc, rank * n, pf.cpu().numpy())
    ok = (np.array_equal(got["hit"], want.hit) and np.array_equal(got["fault_idx"], want.fault_idx)
          and np.array_equal(got["pop_idx"], want.pop_idx))
    ok_all = torch.tensor([1 if ok else 0], dtype=torch.int32, device="cuda")
    dist.all_reduce(ok_all, op=dist.ReduceOp.MIN)
    steps = max(20, min(args.steps, 50))

    def one():
        shard.prefetch()
        for t, _ in shard.exchange(4):
            allreduce_min_unsigned(t)
        eng._check(eng.lib.mpsf_translate_finish(eng.ctx, d_acc.data_ptr(), n, rank * n, shard.hit.data_ptr(),
                                                 shard.faults.data_ptr(), shard.fi.data_ptr(), shard.pi.data_ptr(),
                                                 shard.sp))
    rewarm(one)
    barrier(ws)
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        one()
    b.record()
    b.synchronize()
    ms = max_over_ranks(ws, a.elapsed_time(b) / steps)
    return {"workload": f"{n} accesses per GPU (resolve_va) on the c2 world, sharded over {ws} GPUs, one NCCL MIN "
                        f"of the first-PREFETCH page table between the phases",
            "value": ws * n / (ms / 1e3), "unit": "accesses/s", "ms_per_step": ms, "steps": steps,
            "scaling": "weak", "bit_exact_vs_oracle": bool(int(ok_all.item()))}


def bench_fold(args, eng, hbm_peak, flush):
    """StandbyInstance.fold over a 4 M-snapshot ring drain (100 k
    requests, decode-step deltas: 1-4 tokens, a KV block every ~4th snapshot, 5 % liveness-only),
    device-resident; checked against the oracle's vectorized fold."""
    import torch
    from oracle.seq_oracle import NO_REQ, fold_snapshots_np
    from paper_2605_26461_b200.engine import alloc_fold_outputs
    S, R = 4_000_000, 100_000
    rng = np.random.default_rng(21)
    req = rng.integers(0, R, S, dtype=np.uint32)
    req[rng.random(S) < 0.05] = NO_REQ
    seq = np.arange(1, S + 1, dtype=np.uint64)
    ntok = rng.integers(1, 5, S, dtype=np.uint32)
    nblk = (rng.random(S) < 0.25).astype(np.uint32)
    prog = rng.integers(0, 1 << 20, S, dtype=np.uint32)
    done = (rng.random(S) < 0.01).astype(np.uint8)
    blocks = rng.integers(0, 1 << 24, int(nblk.sum()), dtype=np.uint32)
    tokens = rng.integers(0, 50000, int(ntok.sum()), dtype=np.uint32)
    dev = torch.device("cuda")
    up = lambda a: torch.from_numpy(a.view(np.uint8).copy()).to(dev)  # noqa: E731
    d = [up(req), up(nblk), up(ntok), up(prog), up(done), up(blocks), up(tokens)]
    out = alloc_fold_outputs(S, len(blocks), len(tokens))
    for _ in range(3):
        s = eng.fold_device(S, R, *d[:6], len(blocks), d[6], len(tokens), out)
    t0 = time.perf_counter()
    want = fold_snapshots_np(req, seq, nblk, ntok, prog, done, blocks, tokens)
    t_cpu = time.perf_counter() - t0
    r, nb, nt = int(s.n_requests), int(s.n_blocks), int(s.n_tokens)
    exact = (r == len(want.order) and
             np.array_equal(out["order"][:4 * r].cpu().numpy().view(np.uint32), want.order) and
             np.array_equal(out["blk_off"][:8 * (r + 1)].cpu().numpy().view(np.uint64), want.blk_off) and
             np.array_equal(out["blocks"][:4 * nb].cpu().numpy().view(np.uint32), want.blocks) and
             np.array_equal(out["tokens"][:4 * nt].cpu().numpy().view(np.uint32), want.tokens) and
             np.array_equal(out["progress"][:4 * r].cpu().numpy().view(np.uint32), want.progress) and
             np.array_equal(out["done"][:r].cpu().numpy(), want.done))
    steps = max(20, min(args.steps, 50))
    rewarm(lambda: eng.fold_device(S, R, *d[:6], len(blocks), d[6], len(tokens), out))
    tot = 0.0
    for _ in range(steps):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        eng.fold_device(S, R, *d[:6], len(blocks), d[6], len(tokens), out)     # includes the summary read (a stream sync)
        b.record()
        b.synchronize()
        tot += a.elapsed_time(b)
    ms = tot / steps
    # snapshot SoA read (17 B) + payload read and written + per-request outputs (order,
    # offsets, progress, done = 25 B)
    B = 17 * S + 8 * (nb + nt) + 25 * r
    return {"workload": f"{S} snapshots, {R} requests, decode-step deltas (fold)",
            "value": S / (ms / 1e3), "unit": "snapshots/s", "ms_per_step": ms, "steps": steps,
            "n_requests": r, "n_blocks": nb, "n_tokens": nt, "bit_exact_vs_oracle": bool(exact),
            "cpu_baseline": {"value": S / t_cpu, "unit": "snapshots/s", "cores": 1, "kind": "port",
                             "sample": f"the same {S} snapshots, oracle/seq_oracle.fold_snapshots_np (numpy, "
                                       f"one thread)"},
            "roofline": {"bound": "hbm", "achieved": B / (ms / 1e3) / 1e9, "peak": hbm_peak, "unit": "GB/s",
                         "frac": B / (ms / 1e3) / 1e9 / hbm_peak, "alg_bytes": B}}


def bench_remap(args, eng, hbm_peak, flush):
    import torch
    from oracle.seq_oracle import remap_table
    state_bytes = 64 << 30
    npages = state_bytes >> 12
    # one shared allocation's physical pages (bump-allocated, as _take_pages does)
    phys = torch.arange(514, 514 + npages, dtype=torch.int64, device="cuda")
    out = {}
    for gran in (16, 21):
        e = npages >> (gran - 12)
        d_out = torch.empty(16 * e, dtype=torch.uint8, device="cuda")
        for _ in range(3):
            eng.remap_device(0x7F00_0000_0000, phys, npages, gran, d_out)
        torch.cuda.synchronize()
        steps = max(20, min(args.steps, 50))
        rewarm(lambda: eng.remap_device(0x7F00_0000_0000, phys, npages, gran, d_out))
        eng.set_profiling(True)
        tot = 0.0
        for _ in range(steps):
            flush.zero_()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            eng.remap_device(0x7F00_0000_0000, phys, npages, gran, d_out)
            b.record()
            b.synchronize()
            tot += a.elapsed_time(b)
        prof = eng.profile()
        eng.set_profiling(False)
        ms = tot / steps
        k_ms = prof.get("k_remap", (1, ms))[1] / max(prof.get("k_remap", (1, ms))[0], 1)
        B = 24 * e
        # spot-check against the oracle on the first and last 4096 entries
        host = d_out.view(torch.int64).view(-1, 2)
        head = host[:4096].cpu().numpy()
        want = remap_table(0x7F00_0000_0000, np.arange(514, 514 + 4096 * (1 << (gran - 12)), dtype=np.uint64), gran)
        ok = np.array_equal(head[:, 0].astype(np.uint64), want["va"]) and \
            np.array_equal(head[:, 1].astype(np.uint64), want["phys"])
        # the CPU restatement on a bounded sample (100 k entries), one thread
        ns = 100_000
        t0 = time.perf_counter()
        remap_table(0x7F00_0000_0000, np.arange(514, 514 + ns * (1 << (gran - 12)), dtype=np.uint64), gran)
        t_cpu = time.perf_counter() - t0
        cpu_b = {"value": ns * (1 << gran) / t_cpu / 1e9, "unit": "GB/s of state", "cores": 1, "kind": "port",
                 "sample": f"{ns} entries, oracle/seq_oracle.remap_table (one thread)"}
        out[f"{1 << (gran - 10)}KiB"] = {
            "entries": e, "ms_per_step": ms, "kernel_ms": k_ms,
            "remap_GBps_of_state": state_bytes / (ms / 1e3) / 1e9,
            "roofline": {"bound": "hbm", "achieved": B / (k_ms / 1e3) / 1e9, "peak": hbm_peak, "unit": "GB/s",
                         "frac": B / (k_ms / 1e3) / 1e9 / hbm_peak, "alg_bytes": B},
            "check": "matches oracle" if ok else "MISMATCH", "cpu_baseline": cpu_b}
        del d_out
    return {"state": "64 GiB shared state (one allocation, 16,777,216 x 4 KiB pages)", **out}


# ------------------------------------------------------------------------------------------

def workload_name(wl: str, n: int) -> str:
    """The `config.workload` both arms report (same text, so the driver's ratio compares like
    with like)."""
    from paper_2605_26461_b200 import synth
    c = synth.CONFIGS[wl]
    mix = "translation misses"
    if c.get("parse_frac"):
        mix += f" + parse-time ({c['parse_frac']:g})"
    if c.get("trap_frac"):
        mix += f" + SM traps ({c['trap_frac']:g})"
    return (f"{wl}: {c['clients']} MPS clients x 32 ranges x {c['pages']} pages, {n} entries/GPU, {mix}, "
            f"isolation on")


def run_reference(args):
    """The reference arm: the reference's CPU implementation of the path on the host cores, on
    the same workload as this arm's line.  The reference is pure Python whose bottom half cannot
    run a 10^7-entry batch (it raises on duplicate pages and on a second fatal record, SURVEY.md
    [P2]), so each step runs its restatement ``oracle/mpsf_oracle.c`` over the WHOLE trace on
    every host thread (pinned bit-exact to the reference by tests/test_c_oracle.py and
    tests/test_oracle_vs_reference.py); when the reference is installed (baseline/_ref) its own
    top half -- channel_to_pid + faults.classify -- is timed beside it on a prefix."""
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import c_oracle as co
    from oracle.seq_oracle import Params as OP
    from paper_2605_26461_b200 import synth
    cfg = synth.CONFIGS[args.workload]
    n = cfg["n"] if args.n is None else args.n
    w, _ = synth.build_synthetic_world(cfg["clients"], cfg["pages"], cfg["seed"])
    trace = synth.generate_trace(w, synth.TraceSpec(n=n, seed=cfg["seed"], parse_frac=cfg.get("parse_frac", 0.0),
                                                    trap_frac=cfg.get("trap_frac", 0.0)))
    threads = os.cpu_count() or 1
    steps, warmup = args.steps, args.warmup
    # bounded run: the whole trace per step; steps capped so the arm ends within a few minutes
    t0 = time.perf_counter()
    co.process_batch(w, trace, OP(isolation=True), threads=threads)
    t_one = time.perf_counter() - t0
    budget = 150.0
    if t_one * (steps + warmup) > budget:
        steps = max(3, int(budget / t_one) - 1)
        warmup = 1
    for _ in range(warmup - 1):
        co.process_batch(w, trace, OP(isolation=True), threads=threads)
    ts = []
    for _ in range(steps):
        t0 = time.perf_counter()
        co.process_batch(w, trace, OP(isolation=True), threads=threads)
        ts.append(time.perf_counter() - t0)
    ms = 1e3 * sum(ts) / len(ts)
    value = n / (ms / 1e3)
    smp = f"the whole {args.workload} trace ({n} entries) per step, oracle/mpsf_oracle.c, {threads} threads"
    line = {"metric": METRIC, "value": value, "unit": "entries/s", "impl": "reference", "n_gpus": args.gpus,
            "steps": steps, "warmup": warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": {"workload": workload_name(args.workload, n), "entries_per_gpu": n,
                       "entries_per_step": n},
            "cpu_baseline": {"value": value, "unit": "entries/s", "cores": threads, "kind": "port", "sample": smp},
            "reference_cpu_path": None if args.no_ref_path else reference_cpu_path(cfg, trace),
            "e2e": {"value": value, "unit": "entries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    if steps != args.steps:
        line["steps_capped"] = f"{args.steps} requested; {steps} whole-trace steps fit the time budget"
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--sharded-translate", action="store_true",
                    help="with --gpus N > 1: also time the sharded batched translation (NCCL MIN between phases)")
    ap.add_argument("--impl", default="mine", choices=("mine", "reference"))
    ap.add_argument("--workload", default="c2b", choices=("c1", "c2a", "c2b"))
    ap.add_argument("--entries", "--n", dest="n", type=int, default=None, help="entries per GPU (default: the config's)")
    ap.add_argument("--storm-n", type=int, default=None)
    ap.add_argument("--no-storm", action="store_true")
    ap.add_argument("--no-remap", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-check", action="store_true")
    ap.add_argument("--no-strong", action="store_true", help="N > 1: skip the strong-scaling config-5 extra")
    ap.add_argument("--no-ref-path", action="store_true", help="skip timing the reference's own classify")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    elif args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args))
    elif os.environ.get("MPSF_BENCH_LAUNCH_PROBE") == "1":
        # test hook (tests/test_bench_launch.py): report the rank layout and stop before any CUDA work
        # one write(2) per rank: print() may split the line and the newline, interleaving ranks
        os.write(1, (json.dumps({"probe": True, "rank": int(os.environ.get("RANK", "0")),
                                 "world_size": int(os.environ.get("WORLD_SIZE", "1")),
                                 "local_rank": int(os.environ.get("LOCAL_RANK", "0")),
                                 "master_addr": os.environ.get("MASTER_ADDR")}) + "\n").encode())
    else:
        run_mine(args)


if __name__ == "__main__":
    main()
