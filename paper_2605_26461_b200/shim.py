"""Drop-in for the reference's bottom half.

``service_bottom_half_gpu(world)`` has the signature and return value of
``mpssim.pipeline.service_bottom_half`` (``pkg/src/mpssim/pipeline.py:160-183``).  It drains
both fault buffers exactly as the reference does (pipeline.py:164), snapshots the world into
flat tables (``world.export_reference_world``), packs the drained ``FaultRecord``s into
16-byte entries and processes the whole batch with one ``mpsf_process_host`` call.  The
verdicts are then applied in drain order through the reference's own handlers, so traces,
event scheduling and state mutations stay the simulator's:

* labels ("fatal" / "serviced" / "isolated") come from the device (pure function of the
  scenario and ``uvm.isolation_enabled``, pipeline.py:168-182);
* isolated records go through ``intercept_and_isolate`` (pipeline.py:270-304) and the
  mechanism it picks must equal the device's (checked, raises on disagreement);
* fatal reports (``_report_fatal``, pipeline.py:224-232) are skipped when the device
  cancelled them -- a second teardown of a destroyed TSG, where the reference raises
  ``UnknownTsg`` (batch rule C4);
* benign records schedule ``benign_done`` (pipeline.py:186-190); the reference's own
  ``finish_benign_service`` drops completions on torn-down channels, which is the device's
  cancel flag (C5);
* duplicate replayable records (rule C2) are coalesced: they get their label and a
  ``bh_service`` trace line but no action (the reference would re-isolate them with M2 and
  crash from the third one on, SURVEY.md [P2-A2]).

Install with ``install(engine)``, which patches ``mpssim.pipeline.service_bottom_half``
(the DES looks it up at call time, ``machine.py:188-191``).
"""

from __future__ import annotations

import numpy as np

from . import constants as K
from .world import ENTRY_DTYPE, export_reference_world

_ENG = ("sm", "ce", "pbdma")
_ACC = ("read", "write", "prefetch")
_PARSE = ("parse.mmu_structural", "parse.channel_state", "parse.privilege", "parse.aperture",
          "parse.ecc_poison")

_default_engine = None


def default_engine():
    global _default_engine
    if _default_engine is None:
        from .engine import FaultEngine
        _default_engine = FaultEngine(0)
    return _default_engine


def pack_records(records, flat) -> np.ndarray:
    """FaultRecords (drain order) -> packed entries.  Parse-time records carry their
    category in ``kind`` (faults.py:289-292); translation records their FaultSeed."""
    chan = {name: i for i, name in enumerate(flat.channel_names)}
    out = np.zeros(len(records), ENTRY_DTYPE)
    for i, rec in enumerate(records):
        ch = chan[rec.channel_id]
        if rec.fatality_stage == "parse-time":
            eng = int(flat.channels["engine"][ch])
            out[i] = (0, ch, eng, 0, 1 + _PARSE.index(rec.scenario), K.ENTRY_FLAG_VALID)
        else:
            s = rec.seed
            out[i] = (s.va, ch, _ENG.index(s.engine.value), _ACC.index(s.access.value), 0, K.ENTRY_FLAG_VALID)
    return out


def _same_world(a, b) -> bool:
    return (b is not None and a.world_flags == b.world_flags and
            all(np.array_equal(getattr(a, f), getattr(b, f))
                for f in ("clients", "channels", "ranges", "client_off", "page_state")))


def upload_if_changed(eng, flat) -> None:
    """``mpsf_upload_world`` only when the flat snapshot differs from the engine's last one
    (the reference mutates its world between drains -- isolations create / convert ranges,
    teardowns release clients -- but most drains see the same tables)."""
    if not _same_world(flat, getattr(eng, "_shim_world", None)):
        eng.upload_world(flat)
        eng._shim_world = flat


class ShimMismatch(RuntimeError):
    """The device verdict disagrees with what the reference's own handler did."""


def service_bottom_half_gpu(world, engine=None) -> list:
    from mpssim import pipeline as P   # the drop-in runs inside the reference simulator

    from .engine import BatchParams
    uvm = world.uvm
    records = uvm.replayable_buf.drain() + uvm.nonreplayable_buf.drain()
    if not records:
        return []
    eng = engine if engine is not None else default_engine()
    flat = export_reference_world(world)
    entries = pack_records(records, flat)
    upload_if_changed(eng, flat)
    res = eng.process(entries, BatchParams.from_sim_params(world.params, uvm.isolation_enabled))
    out = res.out
    labels = []
    for i, rec in enumerate(records):
        sid = int(out["scenario"][i])
        if K.SCENARIOS[sid].sid != rec.scenario:
            raise ShimMismatch(f"record {i}: device classified {K.SCENARIOS[sid].sid}, "
                               f"raise-time scenario was {rec.scenario} (world changed since raise)")
        v = int(out["verdict"][i])
        outcome, mech = v & 3, (v >> 2) & 3
        dup, cancelled = bool(v & K.V_DUP), bool(v & K.V_CANCELLED)
        world.trace.emit(world.clock.now, "uvm", "bh_service", scenario=rec.scenario, channel=rec.channel_id)
        label = K.OUTCOME_NAMES[outcome]
        labels.append(label)
        if dup:
            continue
        if rec.fatality_stage == "parse-time":
            world.trace.emit(world.clock.now, "uvm", "parse_fatal", scenario=rec.scenario)
            if not cancelled:
                P._report_fatal(world, rec)
        elif outcome == K.OUT_SERVICED:
            P._begin_benign_service(world, rec)
        elif outcome == K.OUT_ISOLATED:
            o = P.intercept_and_isolate(world, rec)
            if o.mechanism != K.MECH_NAMES[mech]:
                raise ShimMismatch(f"record {i}: device mechanism {K.MECH_NAMES[mech]}, reference {o.mechanism}")
        elif not cancelled:
            P._report_fatal(world, rec)
    return labels


REMAP_CHECKS = {"maps": 0, "pages": 0}


def vmm_map_with_remap(orig, engine):
    """``MemoryModel.vmm_map`` (memory.py:269-283) that also builds the mapping's remap table on
    the device: entry i = (range base + i * 4 KiB, alloc.pages[i]) -- the page-granular state the
    reference's PageRecs alias (one PageRec per physical page of the allocation).  The table is
    checked against the reference's own allocation on every call (deploy_pair maps weights and
    KV this way, recovery.py:175-184) and kept as ``world.remap_tables[rid]``."""
    def vmm_map(self, world, pid, handle):
        rng = orig(self, world, pid, handle)
        eng = engine if engine is not None else default_engine()
        phys = np.asarray(self.allocations[handle].pages, dtype=np.uint64)
        table = eng.remap(rng.base, phys, K.PAGE_SHIFT)
        if not (np.array_equal(table["phys"], phys) and np.array_equal(
                table["va"], np.uint64(rng.base) + (np.arange(len(phys), dtype=np.uint64) << np.uint64(K.PAGE_SHIFT)))):
            raise ShimMismatch(f"remap table of rid {rng.rid} differs from the allocation's pages")
        if not hasattr(world, "remap_tables"):
            world.remap_tables = {}
        world.remap_tables[rng.rid] = table
        REMAP_CHECKS["maps"] += 1
        REMAP_CHECKS["pages"] += len(phys)
        return rng
    return vmm_map


def install(engine=None, remap: bool = True):
    """Patch ``mpssim.pipeline.service_bottom_half`` with the batch path (and, with ``remap``,
    ``MemoryModel.vmm_map`` with the device remap); returns an undo."""
    from mpssim import memory as M
    from mpssim import pipeline as P
    orig = P.service_bottom_half
    orig_map = M.MemoryModel.vmm_map

    def patched(world):
        return service_bottom_half_gpu(world, engine)

    P.service_bottom_half = patched
    if remap:
        M.MemoryModel.vmm_map = vmm_map_with_remap(orig_map, engine)

    def undo():
        P.service_bottom_half = orig
        M.MemoryModel.vmm_map = orig_map
    return undo
