"""Drive the *reference* package (mpssim) on a batch, for differential tests and for
``tests/golden/make_golden.py``.  Needs ``/root/reference`` (or ``$MPSSIM_REF``); the
GPU box does not have it, so everything here is used only from CPU tests that skip
when it is absent, and from the golden-fixture generator.

Batch protocol (the [P11]/[P12]/[P15] method of SURVEY.md Appendix C): raise every
translation / parse-time entry in trace order through the reference's own top half
(``pipeline.raise_mmu_fault`` / ``raise_parse_time_fault``), then every SM trap
(``raise_sm_trap``), then one ``service_bottom_half`` and ``run_until_quiescent``.
"""

from __future__ import annotations

import os
import random
import sys

import numpy as np

# where the reference (and its tests) are: $MPSSIM_REF, /root/reference/pkg/src, or the
# baseline/_ref install that travels to the GPU box (oracle/refpath.py)
from oracle.refpath import REF_SRC, REF_TESTS, import_reference, reference_available  # noqa: E402,F401


ENGINES = ("sm", "ce", "pbdma")
ACCESSES = ("read", "write", "prefetch")


def build_reference_world(spec, params_kw=None):
    """spec: list of (mode, [range recipes]).  Recipes: ('device', pages),
    ('managed', pages), ('managed_ro_cpu', pages), ('managed_ro_gpu', pages),
    ('vmm_ro', pages), ('zombie', pages), ('pinned', pages), ('mixed_ro', pages, mask)."""
    import_reference()
    from mpssim import machine
    from mpssim.kernel import PAGE_SIZE, SimParams
    from mpssim.memory import Protection

    kw = dict(per_process_overhead_pages=0, gpu_pages=1 << 26)
    kw.update(params_kw or {})
    w = machine.build_world(SimParams(**kw))
    if any(m == "mps" for m, _ in spec):
        w.gpu.create_mps_session(w)
    mem = w.mem
    for mode, recipes in spec:
        cl = machine.create_client(w, "mps-client" if mode == "mps" else "standalone")
        pid = cl.pid
        for rec in recipes:
            kind, pages = rec[0], rec[1]
            size = pages * PAGE_SIZE
            if kind == "device":
                mem.alloc_device(w, pid, size)
            elif kind == "managed":
                mem.alloc_managed(w, pid, size)
            elif kind == "managed_ro_cpu":
                r = mem.alloc_managed(w, pid, size)
                mem.set_access(w, r, Protection.READ_ONLY)
            elif kind == "managed_ro_gpu":
                r = mem.alloc_managed(w, pid, size)
                for i in range(pages):
                    mem.populate_page(w, r, i)
                mem.set_access(w, r, Protection.READ_ONLY)
            elif kind == "vmm_ro":
                _, r = mem.vmm_create_map(w, pid, size)
                mem.set_access(w, r, Protection.READ_ONLY)
            elif kind == "zombie":
                r = mem.alloc_managed(w, pid, size)
                mem.make_zombie(w, r)
            elif kind == "pinned":
                r = mem.alloc_managed(w, pid, size)
                mem.pin_non_migratable(w, r)
            elif kind == "mixed_ro":
                r = mem.alloc_managed(w, pid, size)
                for i in np.nonzero(rec[2])[0]:
                    mem.populate_page(w, r, int(i))
                mem.set_access(w, r, Protection.READ_ONLY)
            else:
                raise ValueError(kind)
    return w


def synthetic_spec(n_clients, pages, seed, n_standalone=0, ranges_per_kind=4):
    """The same recipe as paper_2605_26461_b200.synth.build_synthetic_world."""
    from paper_2605_26461_b200.synth import RANGE_KINDS, mixed_mask
    rng = np.random.Generator(np.random.PCG64(seed))
    spec = []
    for mode in ["mps"] * n_clients + ["standalone"] * n_standalone:
        recipes = []
        for kind in RANGE_KINDS:
            for _ in range(ranges_per_kind):
                if kind == "mixed_ro":
                    recipes.append((kind, pages, mixed_mask(rng, pages)))
                else:
                    recipes.append((kind, pages))
        spec.append((mode, recipes))
    return spec


def run_reference_batch(w, flat, entries, isolation=True):
    """Returns a dict of reference observables, or raises the reference's exception."""
    import_reference()
    from mpssim import faults, pipeline
    from mpssim.execmodel import EngineClass
    from mpssim.memory import AccessType, FaultSeed

    w.uvm.isolation_enabled = isolation
    benign_log = []
    orig = pipeline.finish_benign_service

    def spy(world, ev):
        ch = world.gpu.channels.get(ev.args["channel"])
        dropped = ch is None or ch.state.value == "torn-down"
        benign_log.append((ev.args["channel"], ev.args["va"], not dropped))
        return orig(world, ev)

    pipeline.finish_benign_service = spy
    try:
        traps = []
        for e in entries:
            ch = flat.channel_names[int(e["channel"])]
            kind = int(e["kind"])
            if kind == 0:
                seed = FaultSeed(va=int(e["va"]), access=AccessType(ACCESSES[int(e["access"])]),
                                 engine=EngineClass(ENGINES[int(e["engine"])]), channel_id=ch)
                pipeline.raise_mmu_fault(w, seed)
            elif 1 <= kind <= 5:
                pipeline.raise_parse_time_fault(w, ch, faults.PARSE_TIME_ORDER[kind - 1])
            else:
                traps.append(e)
        for e in traps:
            ch = flat.channel_names[int(e["channel"])]
            code = ("EXC_2", "EXC_4", "EXC_5", "EXC_6", "EXC_7")[int(e["kind"]) - 8]
            pipeline.raise_sm_trap(w, code, 0, w.gpu.channels[ch].owner_pid)
        labels = pipeline.service_bottom_half(w)
        w.run_until_quiescent()
    finally:
        pipeline.finish_benign_service = orig
    clients = {}
    for pid, cl in w.gpu.clients.items():
        clients[pid] = (cl.state.value, cl.terminate_reason or "-", cl.error_notifier or "-")
    return dict(
        labels=labels,
        isolation=[(o.scenario, o.mechanism, o.terminated_pid) for o in w.uvm.isolation_outcomes],
        benign=benign_log,
        clients=clients,
        fatal_reports=len(w.rmgsp.fatal_reports),
        scenarios=[r.scenario for r in w.uvm.fault_log],
    )


def random_small_world_spec(rnd: random.Random):
    """[P11]-style worlds: 1-3 MPS clients + 0-2 standalone, small ranges of every kind."""
    spec = []
    n_mps = rnd.randint(1, 3)
    n_sa = rnd.randint(0, 2)
    for mode in ["mps"] * n_mps + ["standalone"] * n_sa:
        recipes = [("device", rnd.randint(1, 2)), ("managed", rnd.randint(1, 2)),
                   ("managed_ro_cpu", 2), ("managed_ro_gpu", 1), ("vmm_ro", 2),
                   ("zombie", 1), ("pinned", 1)]
        if rnd.random() < 0.5:
            m = np.array([rnd.random() < 0.5 for _ in range(3)])
            recipes.append(("mixed_ro", 3, m))
        rnd.shuffle(recipes)
        spec.append((mode, recipes))
    return spec


def random_batch(rnd: random.Random, flat, n, parse_p=0.12, trap_p=0.05):
    from paper_2605_26461_b200 import constants as K
    from paper_2605_26461_b200.world import ENTRY_DTYPE

    out = np.zeros(n, ENTRY_DTYPE)
    r = flat.ranges
    for i in range(n):
        c = rnd.randrange(flat.n_clients)
        lo, hi = int(flat.client_off[c]), int(flat.client_off[c + 1])
        u = rnd.random()
        if u < parse_p:
            out[i] = (0, 3 * c, 0, 0, 1 + rnd.randrange(5), 1)
            continue
        if u < parse_p + trap_p:
            out[i] = (0, 3 * c, 0, 0, 8 + rnd.randrange(5), 1)
            continue
        eng = rnd.choice((0, 0, 1, 2))
        acc = rnd.choice((0, 1, 1, 2) if rnd.random() < 0.9 else (2,))
        v = rnd.random()
        if v < 0.08 or hi == lo:
            va = rnd.choice((0xDEAD_0000, 0xBEEF_0123, (1 << 32) + rnd.randrange(1 << 20)))
        else:
            k = rnd.randrange(lo, hi)
            base, end = int(r["base"][k]), int(r["end"][k])
            va = base + rnd.randrange(end - base + K.PAGE_SIZE)
        out[i] = (va, 3 * c + eng, eng, acc, 0, 1)
    return out
