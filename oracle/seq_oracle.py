"""Sequential CPU oracle for the batched fault path -- TEST INFRASTRUCTURE ONLY.

This module is the *checker*.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import it; the
product path (``paper_2605_26461_b200``) never does.

It restates, one record at a time and in the reference's own order, what
``mpssim`` does with a batch of fault-buffer entries:

* top half, per entry (``pipeline.raise_mmu_fault``, pipeline.py:96-129): channel ->
  client (pipeline.py:103), ``faults.classify`` (faults.py:134-171) with the reference's
  *linear* ``range_at`` scan (memory.py:233-237), buffer choice by the classified
  ``replayable`` flag (pipeline.py:116-123); parse-time records go to the replayable
  buffer (pipeline.py:132-148);
* SM traps run RC recovery at raise time, before the drain (pipeline.py:151-155);
* bottom half (``service_bottom_half``, pipeline.py:160-183): drain replayable then
  non-replayable, label each record, report fatal -> ``rc_recovery`` (pipeline.py:235-265,
  ``teardown_tsg`` execmodel.py:345-374, ``terminate_client`` pipeline.py:329-365),
  benign -> schedule ``benign_done`` (pipeline.py:186-190), isolation ->
  ``intercept_and_isolate`` on the *evolving* range state (pipeline.py:270-304);
* the event loop in (time, seq) order (kernel.py:206-265): ``finish_benign_service``
  drops completions on torn-down channels (pipeline.py:198-200), ``finish_isolation``
  terminates a still-running raiser (pipeline.py:307-324).

Where the reference is undefined (it raises ``UnknownTsg``/``KeyError``, SURVEY.md
Appendix A [P2], [P6]) the build's batch rules apply:
C0 snapshot classification, C1 drain order, C2 dedup of replayable translation
records by (client, engine, page, scenario) with the first in drain order acting,
C4 a fatal record whose TSG is already destroyed is *cancelled*, C5/C6 dropped
benign completions are *cancelled*.  On every batch the reference can process this
oracle reproduces it exactly (``tests/test_oracle_vs_reference.py``).
"""

from __future__ import annotations

import heapq
from dataclasses import dataclass, field

import numpy as np

from paper_2605_26461_b200 import constants as K
from paper_2605_26461_b200.world import OUT_DTYPE, VERDICT_DTYPE, FlatWorld


class OracleError(Exception):
    """Input the reference would reject (maps onto mpssim.errors in the shim)."""

    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


@dataclass
class Params:
    isolation: bool = True
    benign_us: int = 226           # SimParams defaults, kernel.py:34-37
    m1_us: int = 131
    m2_us: int = 2780
    m3_us: int = 1700

    def latency(self, mech: int) -> int:
        return (0, self.m1_us, self.m2_us, self.m3_us)[mech]


@dataclass
class BatchResult:
    out: np.ndarray
    verdict: np.ndarray
    counts: np.ndarray
    dedup_keys: np.ndarray
    dedup_idx: np.ndarray
    cancel: np.ndarray
    isolation_outcomes: list = field(default_factory=list)  # (idx, scenario, mech, client) drain order
    benign_events: list = field(default_factory=list)       # (idx, serviced) event order
    labels: list = field(default_factory=list)              # (idx, outcome) drain order
    fatal_reports: list = field(default_factory=list)       # idx of applied fatal reports


def dedup_key(client: int, engine: int, page: int, scen: int) -> int:
    """C2 packed key: client<<48 | engine<<46 | scenario<<41 | page."""
    return (client << 48) | (engine << 46) | (scen << 41) | page


# -- classification (faults.py:134-171) --------------------------------------------

def range_at(w: FlatWorld, client: int, va: int) -> int:
    """Linear scan, as ``MemoryModel.range_at`` (memory.py:233-237); -1 if none."""
    lo, hi = int(w.client_off[client]), int(w.client_off[client + 1])
    r = w.ranges
    for i in range(lo, hi):
        if int(r["base"][i]) <= va < int(r["end"][i]):
            return i
    return -1


def page_state_at(w: FlatWorld, ridx: int, va: int) -> int:
    r = w.ranges[ridx]
    return int(w.page_state[int(r["page_off"]) + ((va - int(r["base"])) >> K.PAGE_SHIFT)])


def classify(w: FlatWorld, client: int, va: int, engine: int, access: int):
    """Returns (range index or -1, scenario id).  Priority order of faults.py:145-171."""
    ridx = range_at(w, client, va)
    if access == K.ACC_PREFETCH:
        return ridx, K.S_PREFETCH                       # faults.py:145-146 (any engine)
    if ridx < 0:
        return ridx, K.S_OOB[engine]                    # 147-148
    r = w.ranges[ridx]
    if int(r["lifecycle"]) == K.LC_ZOMBIE:
        return ridx, K.S_ZOMBIE[engine]                 # 149-150
    st = page_state_at(w, ridx, va)
    res, ro = st & 0x3, bool(st & K.PS_RO)
    if not int(r["migratable"]) and res == K.RES_CPU:
        return ridx, K.S_NONMIG[engine]                 # 151-153
    if access == K.ACC_WRITE and ro:                    # 154-161
        if engine == K.ENG_SM:
            if int(r["kind"]) == K.RK_EXTERNAL:
                return ridx, K.S_AM_VMM_SM
            if res == K.RES_GPU:
                return ridx, K.S_AM_GPU_SM
            return ridx, K.S_AM_CPU_SM
        return ridx, K.S_AM[engine]
    if int(r["kind"]) == K.RK_MANAGED and res in (K.RES_UNPOP, K.RES_CPU):   # 162-168
        return ridx, K.S_DEMAND_SM if engine == K.ENG_SM else K.S_BENIGN[engine]
    return ridx, K.S_OOB[engine]                        # 169-171 (would-hit fallthrough)


# -- the batch -------------------------------------------------------------------------

ERR_BAD_CHANNEL = -3
ERR_BAD_ENTRY = -4
ERR_ENGINE_MISMATCH = -5
ERR_VA_RANGE = -6


def decode(w: FlatWorld, entries: np.ndarray):
    """Per-entry decode + attribution + classification (snapshot, rule C0)."""
    n = len(entries)
    recs = []
    nch = len(w.channels)
    for i in range(n):
        e = entries[i]
        if not (int(e["flags"]) & K.ENTRY_FLAG_VALID):
            recs.append(None)
            continue
        ch = int(e["channel"])
        if ch >= nch or int(w.channels["client"][ch]) >= w.n_clients:
            raise OracleError(ERR_BAD_CHANNEL, f"entry {i}: channel {ch} has no client")
        c = int(w.channels["client"][ch])
        ceng = int(w.channels["engine"][ch])
        kind, eng, acc, va = int(e["kind"]), int(e["engine"]), int(e["access"]), int(e["va"])
        if kind == K.KIND_TRANSLATION:
            if eng > 2 or acc > 2:
                raise OracleError(ERR_BAD_ENTRY, f"entry {i}: bad engine/access")
            if eng != ceng:
                raise OracleError(ERR_ENGINE_MISMATCH, f"entry {i}: engine != channel engine")
            if va >= (1 << 53):
                raise OracleError(ERR_VA_RANGE, f"entry {i}: va >= 2^53")
            ridx, s = classify(w, c, va, eng, acc)
            recs.append(dict(i=i, c=c, ceng=ceng, eng=eng, va=va, kind=0, s=s, ridx=ridx,
                             rep=K.SCENARIOS[s].replayable))
        else:
            s = K.scenario_of_kind(kind)
            if s is None:
                raise OracleError(ERR_BAD_ENTRY, f"entry {i}: bad kind {kind}")
            trap = kind >= K.KIND_TRAP_FIRST
            recs.append(dict(i=i, c=c, ceng=ceng, eng=ceng, va=va, kind=kind, s=s, ridx=-1,
                             rep=not trap and True, trap=trap))
    return recs


class _State:
    """The slice of GpuModel / MemoryModel state the drain mutates."""

    def __init__(self, w: FlatWorld):
        C = w.n_clients
        self.w = w
        self.mode = [int(m) for m in w.clients["mode"]]
        self.alive = [bool(int(f) & K.CF_ALIVE) for f in w.clients["flags"]]
        self.state = [K.ST_RUNNING if a else K.ST_TERMINATED for a in self.alive]
        self.reason = [K.RS_NONE if a else K.RS_UNCHANGED for a in self.alive]
        self.notifier = [K.NOTIFIER_NONE if a else K.NOTIFIER_UNCHANGED for a in self.alive]
        mps = [c for c in range(C) if self.mode[c] == K.MODE_MPS]
        self.session = mps                          # MpsSession.client_pids (never pruned)
        self.gr_alive = bool(mps) and not (w.world_flags & K.WF_GR_DEAD)
        self.ce_alive = [self.mode[c] == K.MODE_MPS and self.alive[c]
                         and not (int(w.clients["flags"][c]) & K.CF_CE_TSG_DEAD) for c in range(C)]
        self.sa_alive = [self.mode[c] == K.MODE_STANDALONE and self.alive[c] for c in range(C)]
        # channel torn-down flags [client][engine]
        self.torn = [[not self.alive[c]] * 3 for c in range(C)]
        for c in range(C):
            if self.mode[c] == K.MODE_MPS and self.alive[c]:
                if not self.ce_alive[c]:
                    self.torn[c][K.ENG_CE] = True
                if not self.gr_alive:
                    self.torn[c][K.ENG_SM] = self.torn[c][K.ENG_PBDMA] = True
        # current VA ranges per client: list of [base, end, kind]; dead clients released
        self.ranges = []
        r = w.ranges
        for c in range(C):
            lo, hi = int(w.client_off[c]), int(w.client_off[c + 1])
            self.ranges.append([[int(r["base"][i]), int(r["end"][i]), int(r["kind"][i])]
                                for i in range(lo, hi)] if self.alive[c] else [])

    # TSG identity: ("gr",) | ("ce", c) | ("sa", c)
    def tsg_of(self, c: int, ch_engine: int):
        if self.mode[c] == K.MODE_STANDALONE:
            return ("sa", c)
        if ch_engine == K.ENG_CE:
            return ("ce", c)
        return ("gr",)

    def tsg_alive(self, t) -> bool:
        if t[0] == "gr":
            return self.gr_alive
        if t[0] == "ce":
            return self.ce_alive[t[1]]
        return self.sa_alive[t[1]]

    def rc_recovery(self, t, error: int) -> None:
        """pipeline.py:235-265 + execmodel.py:345-374 on a live TSG."""
        if t[0] == "gr":
            for c in self.session:                  # notifies every session pid (pipeline.py:255-256)
                self.notifier[c] = error
            for c in self.session:
                self.torn[c][K.ENG_SM] = self.torn[c][K.ENG_PBDMA] = True
            self.gr_alive = False
            for c in self.session:
                if self.state[c] == K.ST_RUNNING:
                    self.terminate(c, K.RS_FAULT_PROPAGATION)
        elif t[0] == "ce":
            c = t[1]
            self.notifier[c] = error
            self.torn[c][K.ENG_CE] = True
            self.ce_alive[c] = False                # context survives: owner keeps running
        else:
            c = t[1]
            self.notifier[c] = error
            self.torn[c] = [True, True, True]
            self.sa_alive[c] = False
            if self.state[c] == K.ST_RUNNING:
                self.terminate(c, K.RS_FAULT_PROPAGATION)

    def terminate(self, c: int, reason: int) -> None:
        """pipeline.py:329-365: channels, private TSGs, VA ranges."""
        self.state[c] = K.ST_TERMINATED
        self.reason[c] = reason
        self.torn[c] = [True, True, True]
        if self.mode[c] == K.MODE_MPS:
            self.ce_alive[c] = False
        else:
            self.sa_alive[c] = False
        self.ranges[c] = []

    def range_at(self, c: int, va: int):
        for rg in self.ranges[c]:
            if rg[0] <= va < rg[1]:
                return rg
        return None


def process_batch(w: FlatWorld, entries: np.ndarray, params: Params | None = None,
                  base_index: int = 0) -> BatchResult:
    params = params or Params()
    n = len(entries)
    C = w.n_clients
    if w.world_flags & K.WF_GR_DEAD and any(
            int(w.clients["mode"][c]) == K.MODE_MPS and int(w.clients["flags"][c]) & K.CF_ALIVE
            for c in range(C)):
        raise OracleError(-7, "GR TSG destroyed while an MPS client is alive")
    recs = decode(w, entries)
    out = np.zeros(n, OUT_DTYPE)
    out["rid"] = K.NO_RID
    out["scenario"] = 0xFF
    out["client"] = 0xFFFF
    counts = np.zeros((C, K.N_SCENARIOS), np.uint64)
    verdict_bits = np.zeros(n, np.uint8)
    cancelled = np.zeros(n, bool)

    for r in recs:
        if r is None:
            continue
        i = r["i"]
        out["scenario"][i] = r["s"]
        out["client"][i] = r["c"]
        if r["ridx"] >= 0:
            out["rid"][i] = int(w.ranges["rid"][r["ridx"]])
        counts[r["c"], r["s"]] += 1
        if r["rep"]:
            verdict_bits[i] |= K.V_REPLAYABLE

    # C2 dedup over replayable translation records, first in index order acts
    rep_of = {}
    dup_rep = {}
    dedup_keys, dedup_idx = [], []
    for r in recs:
        if r is None or r["kind"] != 0 or not r["rep"]:
            continue
        key = dedup_key(r["c"], r["eng"], r["va"] >> K.PAGE_SHIFT, r["s"])
        if key in rep_of:
            dup_rep[r["i"]] = rep_of[key]
            verdict_bits[r["i"]] |= K.V_DUP
        else:
            rep_of[key] = r["i"]
            dedup_keys.append(key)
            dedup_idx.append(base_index + r["i"])

    st = _State(w)
    res = BatchResult(out, None, counts, np.array(dedup_keys, np.uint64),
                      np.array(dedup_idx, np.uint32), None)

    # SM traps at raise time, in trace order (pipeline.py:151-155, 244-249)
    for r in recs:
        if r is None or not r.get("trap"):
            continue
        c = r["c"]
        t = ("gr",) if st.mode[c] == K.MODE_MPS else ("sa", c)
        if not st.tsg_alive(t):
            cancelled[r["i"]] = True                 # reference: UnknownTsg
            continue
        st.rc_recovery(t, r["s"])

    # C1 drain order: replayable buffer then non-replayable, each in arrival order
    drained = [r for r in recs if r is not None and not r.get("trap") and r["rep"]]
    drained += [r for r in recs if r is not None and not r.get("trap") and not r["rep"]]
    events = []
    seq = 0
    for r in drained:
        i, c, s = r["i"], r["c"], r["s"]
        info = K.SCENARIOS[s]
        parse = info.stage == "parse-time"
        if parse:
            label = K.OUT_FATAL
        elif info.serviceable:
            label = K.OUT_SERVICED
        elif params.isolation:
            label = K.OUT_ISOLATED
        else:
            label = K.OUT_FATAL
        verdict_bits[i] |= label
        res.labels.append((i, label))
        if i in dup_rep:
            continue                                 # coalesced: no separate action
        if label == K.OUT_FATAL:
            t = st.tsg_of(c, r["ceng"])
            if not st.tsg_alive(t):
                cancelled[i] = True                  # reference: UnknownTsg
                continue
            res.fatal_reports.append(i)
            st.rc_recovery(t, s)
        elif label == K.OUT_SERVICED:
            heapq.heappush(events, (params.benign_us, seq, "benign", i, c, r["ceng"]))
            seq += 1
        else:
            rg = st.range_at(c, r["va"])            # post-mutation state (pipeline.py:283)
            if rg is None:
                mech = K.MECH_M1
                pb = r["va"] - (r["va"] % K.PAGE_SIZE)
                st.ranges[c].append([pb, pb + K.PAGE_SIZE, K.RK_MANAGED])
            elif rg[2] == K.RK_MANAGED:
                mech = K.MECH_M2
            else:
                mech = K.MECH_M3
                rg[2] = K.RK_MANAGED
            verdict_bits[i] |= mech << 2
            res.isolation_outcomes.append((i, s, mech, c))
            heapq.heappush(events, (params.latency(mech), seq, "iso", i, c, r["ceng"]))
            seq += 1

    while events:
        _t, _s, kind, i, c, ceng = heapq.heappop(events)
        if kind == "benign":
            dropped = st.torn[c][ceng]
            cancelled[i] = dropped
            res.benign_events.append((i, not dropped))
        else:
            if st.state[c] == K.ST_RUNNING:
                st.terminate(c, K.RS_ISOLATION)

    for i, rep in dup_rep.items():
        cancelled[i] = cancelled[rep]
    verdict_bits[cancelled] |= K.V_CANCELLED
    out["verdict"] = verdict_bits
    res.cancel = (np.nonzero(cancelled)[0] + base_index).astype(np.uint32)
    verdict = np.zeros(C, VERDICT_DTYPE)
    verdict["state"] = st.state
    verdict["reason"] = st.reason
    verdict["notifier"] = st.notifier
    res.verdict = verdict
    return res


# -- recovery remap (memory.py:269-283, recovery.py:156-212, 342-344) ---------------------

def remap_table(va_base: int, phys_pages, gran_log2: int) -> np.ndarray:
    """Remap table of one shared allocation mapped at ``va_base``: ``vmm_map`` gives page i
    of the standby's range (VA ``base + i*4096``) the backing ``alloc.pages[i]``.  At
    granularity G one entry covers G/4096 pages: ``(base + k*G) -> pages[k*G/4096]``."""
    from paper_2605_26461_b200.world import REMAP_DTYPE
    phys = np.asarray(phys_pages, np.uint64)
    step = 1 << (gran_log2 - K.PAGE_SHIFT)
    e = -(-len(phys) // step)
    out = np.zeros(e, REMAP_DTYPE)
    for k in range(e):
        out[k] = (va_base + (k << gran_log2), int(phys[k * step]))
    return out


def remap_blocks(va_base: int, phys_pages, block_ids) -> np.ndarray:
    """Live-KV remap from folded block ids (recovery.py:343-344): KV block b is KV page b."""
    from paper_2605_26461_b200.world import REMAP_DTYPE
    phys = np.asarray(phys_pages, np.uint64)
    out = np.zeros(len(block_ids), REMAP_DTYPE)
    for j, b in enumerate(block_ids):
        out[j] = (va_base + (int(b) << K.PAGE_SHIFT), int(phys[int(b)]))
    return out


def kv_reserve(total_blocks: int, block_ids):
    """``BlockPool(total).reserve(block_ids)`` (workload.py:77-80): the reserved mask over the
    pool's ids and the free ids in pop order (the heap pops smallest first)."""
    taken = set(int(b) for b in block_ids)
    reserved = np.array([1 if b in taken else 0 for b in range(total_blocks)], np.uint8)
    free = np.array([b for b in range(total_blocks) if b not in taken], np.uint32)
    return reserved, free


# -- batched translation (the step before the fault path) ---------------

@dataclass
class TranslateResult:
    hit: np.ndarray          # uint8[n]: 1 Hit, 0 Miss, 0xFF skipped (valid flag clear)
    fault_idx: np.ndarray    # uint32[]: the misses, in access order (their seeds become fault entries)
    pop_idx: np.ndarray      # uint32[]: prefetches that populated a page (populate_page), in order


def translate_batch(w: FlatWorld, entries: np.ndarray, base_index: int = 0) -> TranslateResult:
    """``MemoryModel.resolve_va`` (memory.py:339-364) over an access stream, one access at a
    time in stream order, on the batch-start page tables plus the only mutation translation
    itself makes: a PREFETCH into a managed range populates its page (``populate_page``,
    memory.py:368-380: residency -> GPU, protection unchanged), so later accesses to that
    page see it GPU-resident.  Entries are the 16-byte fault-entry format with kind 0 (the
    would-be seed: va, access, engine, channel); the same entry errors as ``decode``."""
    n = len(entries)
    hit = np.full(n, 0xFF, np.uint8)
    faults, pops = [], []
    populated = set()                  # (ridx, page) made GPU-resident in this batch
    nch = len(w.channels)
    r = w.ranges
    for i in range(n):
        e = entries[i]
        if not (int(e["flags"]) & K.ENTRY_FLAG_VALID):
            continue
        ch = int(e["channel"])
        if ch >= nch or int(w.channels["client"][ch]) >= w.n_clients:
            raise OracleError(ERR_BAD_CHANNEL, f"entry {i}: channel {ch} has no client")
        c, ceng = int(w.channels["client"][ch]), int(w.channels["engine"][ch])
        kind, eng, acc, va = int(e["kind"]), int(e["engine"]), int(e["access"]), int(e["va"])
        if kind != K.KIND_TRANSLATION or eng > 2 or acc > 2:
            raise OracleError(ERR_BAD_ENTRY, f"entry {i}: not a translation access")
        if eng != ceng:
            raise OracleError(ERR_ENGINE_MISMATCH, f"entry {i}: engine != channel engine")
        if va >= (1 << 53):
            raise OracleError(ERR_VA_RANGE, f"entry {i}: va >= 2^53")
        ridx = range_at(w, c, va)
        ok = False
        if acc == K.ACC_PREFETCH:                                  # memory.py:344-349
            if ridx >= 0 and int(r["kind"][ridx]) == K.RK_MANAGED:
                page = (va - int(r["base"][ridx])) >> K.PAGE_SHIFT
                res = page_state_at(w, ridx, va) & 0x3
                if res != K.RES_GPU and (ridx, page) not in populated:
                    populated.add((ridx, page))
                    pops.append(base_index + i)
                ok = True
        elif ridx >= 0 and int(r["lifecycle"][ridx]) != K.LC_ZOMBIE:   # 350-353
            page = (va - int(r["base"][ridx])) >> K.PAGE_SHIFT
            st = page_state_at(w, ridx, va)
            res, ro = st & 0x3, bool(st & K.PS_RO)
            if (ridx, page) in populated:
                res = K.RES_GPU
            if not (not int(r["migratable"][ridx]) and res == K.RES_CPU) and \
                    not (acc == K.ACC_WRITE and ro) and res == K.RES_GPU:   # 355-361
                ok = True
        hit[i] = 1 if ok else 0
        if not ok:
            faults.append(base_index + i)
    return TranslateResult(hit, np.array(faults, np.uint32), np.array(pops, np.uint32))


def _translate_attr(w: FlatWorld, entries: np.ndarray):
    valid = (entries["flags"] & K.ENTRY_FLAG_VALID) != 0
    ch = entries["channel"].astype(np.int64)
    client = w.channels["client"][ch].astype(np.uint64)
    va = entries["va"].astype(np.uint64)
    acc = entries["access"].astype(np.int64)
    r = w.ranges
    keys = (r["client"].astype(np.uint64) << np.uint64(40)) | (r["base"] >> np.uint64(12))
    page = va >> np.uint64(12)
    pos = np.searchsorted(keys, (client << np.uint64(40)) | page, side="right").astype(np.int64) - 1
    p = np.where(pos >= 0, pos, 0)
    has = (pos >= 0) & (r["client"][p] == client) & (page < (r["end"][p] >> np.uint64(12)))
    slot = (r["page_off"][p].astype(np.int64) + (page - (r["base"][p] >> np.uint64(12))).astype(np.int64))
    slot = np.where(has, slot, 0)
    managed = has & (r["kind"][p] == K.RK_MANAGED)
    return valid, acc, p, has, slot, managed


def translate_prefetch_np(w: FlatWorld, entries: np.ndarray, base_index: int = 0) -> np.ndarray:
    """Phase 1 of ``translate_batch_np`` for a shard at global index ``base_index``: the first
    PREFETCH index per managed page slot (global indices; int64 max where none).  Shards of a
    stream combine these with an elementwise MIN."""
    valid, acc, _, _, slot, managed = _translate_attr(w, entries)
    pf_first = np.full(len(w.page_state) + 1, np.iinfo(np.int64).max, np.int64)
    sel = valid & (acc == K.ACC_PREFETCH) & managed
    idx = np.arange(len(entries), dtype=np.int64) + base_index
    np.minimum.at(pf_first, slot[sel], idx[sel])
    return pf_first


def translate_finish_np(w: FlatWorld, entries: np.ndarray, base_index: int, pf_first: np.ndarray) -> TranslateResult:
    """Phase 2: hit / miss of the shard's accesses given the (combined) first-prefetch table."""
    n = len(entries)
    valid, acc, p, has, slot, managed = _translate_attr(w, entries)
    r = w.ranges
    st = np.where(has, w.page_state[slot], 0).astype(np.int64)
    res, ro = st & 3, (st & K.PS_RO) != 0
    pref = acc == K.ACC_PREFETCH
    idx = np.arange(n, dtype=np.int64) + base_index
    populated_before = has & (pf_first[slot] < idx)
    res_eff = np.where(populated_before, K.RES_GPU, res)
    live = has & (r["lifecycle"][p] == K.LC_LIVE)
    nonmig = (r["migratable"][p] == 0) & (res_eff == K.RES_CPU)
    am = (acc == K.ACC_WRITE) & ro
    ok = np.where(pref, managed, live & ~nonmig & ~am & (res_eff == K.RES_GPU))
    hit = np.where(valid, ok.astype(np.uint8), np.uint8(0xFF)).astype(np.uint8)
    pop = valid & pref & managed & (pf_first[slot] == idx) & (res != K.RES_GPU)
    return TranslateResult(hit, (np.nonzero(valid & ~ok)[0] + base_index).astype(np.uint32),
                           (np.nonzero(pop)[0] + base_index).astype(np.uint32))


def translate_batch_np(w: FlatWorld, entries: np.ndarray, base_index: int = 0) -> TranslateResult:
    """The same result as ``translate_batch`` for large streams (numpy, no per-entry loop):
    the only in-batch dependency is "was this page populated by an earlier prefetch", i.e. the
    first prefetch index per (range, page).  Assumes well-formed entries (no error checks)."""
    return translate_finish_np(w, entries, base_index, translate_prefetch_np(w, entries, base_index))


# -- snapshot delta fold (the step after the remap) ----------------------

@dataclass
class FoldResult:
    order: np.ndarray        # uint32[R']: request ids in first-appearance order (dict order)
    blk_off: np.ndarray      # uint64[R'+1]: CSR offsets into blocks
    blocks: np.ndarray       # uint32[]: each request's KV block ids, deltas concatenated in seq order
    tok_off: np.ndarray      # uint64[R'+1]
    tokens: np.ndarray       # uint32[]
    progress: np.ndarray     # uint32[R']: the last snapshot's progress
    done: np.ndarray         # uint8[R']: any snapshot done
    last_seq: int            # last consumed sequence number


NO_REQ = 0xFFFFFFFF


def fold_snapshots(req, seq, nblk, ntok, progress, done, blocks, tokens) -> FoldResult:
    """``StandbyInstance.fold`` (recovery.py:83-92) over consumed snapshots in order: per
    request (dict insertion order = first appearance) the block-id and token deltas are
    appended, progress is the last snapshot's, done is sticky; a snapshot without a request id
    (``NO_REQ``) only advances ``last_consumed_seq``.  Snapshot i's deltas are
    ``blocks[sum(nblk[:i]) : sum(nblk[:i+1])]`` (same for tokens)."""
    folded = {}
    bo = to = 0
    last = 0
    for i in range(len(req)):
        b = blocks[bo:bo + int(nblk[i])]
        t = tokens[to:to + int(ntok[i])]
        bo += int(nblk[i])
        to += int(ntok[i])
        last = int(seq[i])
        r = int(req[i])
        if r == NO_REQ:
            continue
        e = folded.setdefault(r, [[], [], 0, False])
        e[0].extend(int(x) for x in b)
        e[1].extend(int(x) for x in t)
        e[2] = int(progress[i])
        e[3] = e[3] or bool(done[i])
    order = np.array(list(folded), np.uint32)
    bl = [folded[r][0] for r in folded]
    tl = [folded[r][1] for r in folded]
    return FoldResult(order, np.concatenate([[0], np.cumsum([len(x) for x in bl])]).astype(np.uint64),
                      np.array([x for l in bl for x in l], np.uint32),
                      np.concatenate([[0], np.cumsum([len(x) for x in tl])]).astype(np.uint64),
                      np.array([x for l in tl for x in l], np.uint32),
                      np.array([folded[r][2] for r in folded], np.uint32),
                      np.array([folded[r][3] for r in folded], np.uint8), last)


def _seg_gather(src, starts, lens):
    """Concatenate src[starts[k] : starts[k]+lens[k]] over k (vectorized)."""
    lens = np.asarray(lens, np.int64)
    tot = int(lens.sum())
    if tot == 0:
        return np.zeros(0, src.dtype)
    excl = np.cumsum(lens) - lens
    return src[np.repeat(np.asarray(starts, np.int64) - excl, lens) + np.arange(tot)]


def fold_snapshots_np(req, seq, nblk, ntok, progress, done, blocks, tokens) -> FoldResult:
    """Vectorized ``fold_snapshots`` for large batches (the same result; checked against the
    loop form in tests/test_fold_oracle.py): requests ranked by first appearance, snapshots
    stably grouped by rank, deltas gathered by segment."""
    req = np.asarray(req, np.uint32)
    nblk = np.asarray(nblk, np.int64)
    ntok = np.asarray(ntok, np.int64)
    blocks = np.asarray(blocks, np.uint32)
    tokens = np.asarray(tokens, np.uint32)
    idx = np.nonzero(req != NO_REQ)[0]
    r = req[idx]
    uniq, first = np.unique(r, return_index=True)
    pos = np.argsort(first, kind="stable")
    order = uniq[pos].astype(np.uint32)
    rank_u = np.empty(len(uniq), np.int64)
    rank_u[pos] = np.arange(len(uniq))
    rk = rank_u[np.searchsorted(uniq, r)]
    o = np.argsort(rk, kind="stable")
    perm, rks = idx[o], rk[o]
    bstart = np.cumsum(nblk) - nblk
    tstart = np.cumsum(ntok) - ntok
    R = len(order)
    bc = np.bincount(rks, weights=nblk[perm], minlength=R).astype(np.int64) if R else np.zeros(0, np.int64)
    tc = np.bincount(rks, weights=ntok[perm], minlength=R).astype(np.int64) if R else np.zeros(0, np.int64)
    ends = np.cumsum(np.bincount(rks, minlength=R)) - 1 if R else np.zeros(0, np.int64)
    dn = np.bincount(rks, weights=np.asarray(done)[perm] != 0, minlength=R) if R else np.zeros(0)
    return FoldResult(order, np.concatenate([[0], np.cumsum(bc)]).astype(np.uint64),
                      _seg_gather(blocks, bstart[perm], nblk[perm]).astype(np.uint32),
                      np.concatenate([[0], np.cumsum(tc)]).astype(np.uint64),
                      _seg_gather(tokens, tstart[perm], ntok[perm]).astype(np.uint32),
                      np.asarray(progress, np.uint32)[perm[ends]] if R else np.zeros(0, np.uint32),
                      (dn > 0).astype(np.uint8), int(seq[-1]) if len(req) else 0)


def fold_as_snapshots(f: FoldResult):
    """A fold result as one snapshot per folded request (first-appearance order), so that folds
    of contiguous ranges of a stream compose: fold(A ++ B) == fold(snaps(fold(A)) ++
    snaps(fold(B))) -- the merge step of a sharded fold."""
    r = len(f.order)
    nblk = np.diff(f.blk_off).astype(np.uint32) if r else np.zeros(0, np.uint32)
    ntok = np.diff(f.tok_off).astype(np.uint32) if r else np.zeros(0, np.uint32)
    return (np.asarray(f.order, np.uint32), np.zeros(r, np.uint64), nblk, ntok, np.asarray(f.progress, np.uint32),
            np.asarray(f.done, np.uint8), np.asarray(f.blocks, np.uint32), np.asarray(f.tokens, np.uint32))
