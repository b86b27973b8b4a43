"""Generate the golden fixtures under tests/golden/ by running the REFERENCE package.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

Writes:
  classify_c1.npz   -- config-1 world + 20k-entry trace prefix, reference
                       ``faults.classify`` scenario and ``range_at`` rid per entry
  batches.json      -- random multi-record batches the reference processes without
                       raising, with its labels / isolation outcomes / benign
                       completions / fatal reports / client fates
  truth_table.json  -- single-trigger fates ([P9]) through ``faults.inject``
  remap.json        -- ``deploy_pair`` standby mappings (``vmm_map``) and the folded
                       KV block ids after a crash -> failover -> wake cycle
The fixtures are committed; the GPU box reads them, never the reference.
"""

from __future__ import annotations

import json
import os
import random
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from paper_2605_26461_b200 import constants as K  # noqa: E402
from paper_2605_26461_b200 import synth  # noqa: E402
from paper_2605_26461_b200.world import (entries_to_list, export_reference_world,  # noqa: E402
                                         flat_to_dict)
from tests import refharness as H  # noqa: E402
from tests.observe import normalise_reference  # noqa: E402


def make_classify():
    H.import_reference()
    from mpssim import faults
    from mpssim.execmodel import EngineClass
    from mpssim.memory import AccessType, FaultSeed

    w = H.build_reference_world(H.synthetic_spec(4, 16, 1))
    flat = export_reference_world(w)
    mine, _ = synth.build_synthetic_world(4, 16, 1)
    assert np.array_equal(flat.ranges, mine.ranges)
    assert np.array_equal(flat.page_state, mine.page_state)
    trace = synth.generate_trace(mine, synth.TraceSpec(n=100_000, seed=1))[:20_000]
    scen = np.zeros(len(trace), np.uint8)
    rid = np.zeros(len(trace), np.uint32)
    for i, e in enumerate(trace):
        pid = flat.client_names[int(e["channel"]) // 3]
        seed = FaultSeed(va=int(e["va"]), access=AccessType(H.ACCESSES[int(e["access"])]),
                         engine=EngineClass(H.ENGINES[int(e["engine"])]))
        scen[i] = K.SID_TO_ID[faults.classify(seed, w.mem, pid).sid]
        r = w.mem.range_at(pid, int(e["va"]))
        rid[i] = r.rid if r is not None else K.NO_RID
    np.savez_compressed(os.path.join(HERE, "classify_c1.npz"), entries=trace, scenario=scen,
                        rid=rid, ranges=flat.ranges, page_state=flat.page_state)
    print("classify_c1: all scenarios seen:", sorted(set(scen.tolist())))


def make_batches(n_target=400, seed=2026):
    from oracle import seq_oracle as so
    rnd = random.Random(seed)
    out, crashes = [], 0
    while len(out) < n_target:
        spec = H.random_small_world_spec(rnd)
        lat = {}
        if rnd.random() < 0.5:
            lat = dict(m1_latency_us=rnd.choice((131, 226, 300)),
                       m2_latency_us=rnd.choice((2780, 226, 100)),
                       m3_latency_us=rnd.choice((1700, 226, 0)))
        w = H.build_reference_world(spec, lat)
        flat = export_reference_world(w)
        iso = rnd.random() < 0.6
        entries = H.random_batch(rnd, flat, rnd.randint(1, 16))
        p = so.Params(isolation=iso, benign_us=w.params.benign_service_us,
                      m1_us=w.params.m1_latency_us, m2_us=w.params.m2_latency_us,
                      m3_us=w.params.m3_latency_us)
        res = so.process_batch(flat, entries, p)
        if np.any(res.out["verdict"] & K.V_DUP):
            continue
        try:
            ref = H.run_reference_batch(w, flat, entries, isolation=iso)
        except Exception:
            crashes += 1
            continue
        out.append(dict(world=flat_to_dict(flat), entries=entries_to_list(entries),
                        params=dict(isolation=iso, benign_us=p.benign_us, m1_us=p.m1_us,
                                    m2_us=p.m2_us, m3_us=p.m3_us),
                        expect=normalise_reference(ref)))
    with open(os.path.join(HERE, "batches.json"), "w") as f:
        json.dump(out, f, separators=(",", ":"))
    print(f"batches: {len(out)} processable, {crashes} reference crashes skipped")


def _pending_entry(w, flat, pid):
    """The faulting command faults.inject just enqueued, as a packed entry."""
    for eng in (0, 1, 2):
        ch = w.gpu.channels[f"{pid}.{H.ENGINES[eng]}"]
        if ch.pushbuffer:
            cmd = ch.pushbuffer[-1]
            chan = flat.channel_names.index(ch.id)
            if cmd.kind == "exception":
                code = ("EXC_2", "EXC_4", "EXC_5", "EXC_6", "EXC_7").index(cmd.args["code"])
                return (0, chan, eng, 0, 8 + code, 1)
            if cmd.kind == "parse_fault":
                from mpssim import faults
                return (0, chan, eng, 0, 1 + faults.PARSE_TIME_ORDER.index(cmd.args["category"]), 1)
            acc = {"access": cmd.args.get("access"), "copy": cmd.args.get("access", "write"),
                   "sem_wait": "read"}[cmd.kind]
            return (int(cmd.args["va"]), chan, eng, H.ACCESSES.index(acc), 0, 1)
    raise RuntimeError("no pending command")


def make_truth_table():
    H.import_reference()
    from mpssim import faults, machine
    from mpssim.kernel import SimParams

    rows = []
    triggers = (faults.MMU_TRIGGER_ORDER + ["benign.demand_paging.sm", "benign.page_fault.ce",
                                            "benign.page_fault.pbdma", "benign.invalid_prefetch.sm"]
                + faults.SM_TRIGGER_ORDER + faults.PARSE_TIME_ORDER)
    for trig in triggers:
        for iso in (False, True):
            for faulter in ("mps", "standalone"):
                w = machine.build_world(SimParams(per_process_overhead_pages=0))
                w.gpu.create_mps_session(w)
                a = machine.create_client(w, "mps-client")
                b = machine.create_client(w, "mps-client")
                s = machine.create_client(w, "standalone")
                who = a if faulter == "mps" else s
                w.uvm.isolation_enabled = iso
                faults.inject(w, who.pid, trig, privileged=trig.startswith("parse."))
                flat = export_reference_world(w)
                entry = _pending_entry(w, flat, who.pid)
                w.run_until_quiescent()
                rows.append(dict(
                    trigger=trig, isolation=iso, faulter=faulter, world=flat_to_dict(flat),
                    entries=[list(entry)],
                    expect=dict(
                        clients={p: (c.state.value, c.terminate_reason or "-", c.error_notifier or "-")
                                 for p, c in w.gpu.clients.items()},
                        mechanisms=[o.mechanism for o in w.uvm.isolation_outcomes],
                        fatal_reports=len(w.rmgsp.fatal_reports),
                        scenarios=[r.scenario for r in w.uvm.fault_log])))
    with open(os.path.join(HERE, "truth_table.json"), "w") as f:
        json.dump(rows, f, separators=(",", ":"))
    print(f"truth_table: {len(rows)} rows")


def make_remap():
    H.import_reference()
    from mpssim import faults, machine, recovery
    from mpssim.kernel import SimParams
    from mpssim.workload import RequestSpec, WorkloadSpec

    cases = []
    for (wp, kvb, n, crash_k) in ((64, 32, 4, 21), (32, 64, 16, 20), (128, 48, 1, 9)):
        w = machine.build_world(SimParams())
        w.gpu.create_mps_session(w)
        inj = machine.create_client(w, "mps-client")
        machine.attach_injector(w, inj, WorkloadSpec(kind="injector"))
        spec = WorkloadSpec(kind="serving", weight_pages=wp, kv_blocks=kvb)
        active, standby = recovery.deploy_pair(w, spec, n, service="svc")
        pair = w.pairs["svc"]
        maps = {}
        for rng in w.mem.ranges.values():
            if rng.owner_pid == standby and rng.backing_handle in (pair.weights_handle, pair.kv_handle):
                alloc = w.mem.allocations[rng.backing_handle]
                assert all(p.backing == ("alloc", rng.backing_handle) for p in rng.pages)
                maps["weights" if rng.backing_handle == pair.weights_handle else "kv"] = dict(
                    base=rng.base, npages=len(rng.pages), phys=list(alloc.pages))
        machine.schedule_request(w, "svc", RequestSpec("r1", 0, 6, 40))
        machine.schedule_request(w, "svc", RequestSpec("r2", 0, 6, 40))
        engine = w.gpu.clients[active].workload
        engine.watchers.append({"rid": "r1", "progress": crash_k,
                                "action": lambda world: faults.inject(world, inj.pid,
                                                                      "sm.exc4.illegal_instruction")})
        restored = {}
        orig_wake = recovery.complete_wake

        def spy_wake(world, pid):
            orig_wake(world, pid)      # block tables restored at recovery.py:343
            eng = world.gpu.clients[pid].workload
            restored.update({rid: list(t) for rid, t in eng.block_tables.items()})

        recovery.complete_wake = spy_wake
        try:
            w.run_until_quiescent()
        finally:
            recovery.complete_wake = orig_wake
        inst = w.standby_instances[standby]
        folded = {rid: list(f.block_ids) for rid, f in inst.folded.items()}
        cases.append(dict(weight_pages=wp, kv_blocks=kvb, n=n, crash_k=crash_k, maps=maps,
                          folded=folded, restored=restored))
    with open(os.path.join(HERE, "remap.json"), "w") as f:
        json.dump(cases, f, separators=(",", ":"))
    print(f"remap: {len(cases)} cases", [c["folded"] for c in cases])


if __name__ == "__main__":
    make_classify()
    make_batches()
    make_truth_table()
    make_remap()
