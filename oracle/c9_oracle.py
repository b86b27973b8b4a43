"""Phase-by-phase CPU mirror of the GPU kernels -- TEST INFRASTRUCTURE ONLY.

Implements the parallel recipe C9 of SURVEY.md Appendix C exactly the way
``paper_2605_26461_b200/csrc/fault_kernels.cu`` evaluates it (scan -> exchange ->
resolve -> general -> finalize), with the same exchange buffers and hash merge as the C
ABI's phase entry points, so ``paper_2605_26461_b200.parallel.ShardedFaultPath`` can be
driven over gloo on CPU (``tests/test_parallel_gloo.py``) and compared bit for bit with the
sequential oracle (``seq_oracle``), which is itself pinned against the reference.
"""

from __future__ import annotations

import numpy as np

from paper_2605_26461_b200 import constants as K
from paper_2605_26461_b200.world import OUT_DTYPE, VERDICT_DTYPE, FlatWorld

from .seq_oracle import Params, dedup_key

E32 = 0xFFFFFFFF
E64 = 0xFFFFFFFFFFFFFFFF
REL_NONE = (1 << 63) - 1
REL_PRE = -1


def _nr_key(c, epoch, page):
    return (c << 42) | (epoch << 41) | page


def _classify(eng, acc, at, w):
    """faults.classify on the kernel's attribution record."""
    if acc == 2:
        return 15
    oob = 0 if eng == 0 else 2 + 4 * eng
    if not at["in_range"]:
        return oob
    if at["lifecycle"] == 1:
        return 4 + 4 * eng
    st = at["st"]
    res, ro = st & 3, bool(st & 4)
    if not at["migr"] and res == 1:
        return 5 + 4 * eng
    if acc == 1 and ro:
        if eng == 0:
            return 3 if at["kind"] == 1 else (2 if res == 2 else 1)
        return 3 + 4 * eng
    if at["kind"] == 0 and res <= 1:
        return 14 if eng == 0 else 15 + eng
    return oob


class C9Engine:
    """Same phase API as ``engine.FaultEngine`` (scan/resolve/general/finalize + exchange)."""

    def __init__(self, w: FlatWorld):
        self.w = w
        self.C = w.n_clients
        self.R = len(w.ranges)
        self.P = w.n_pages

    # -- decode (kernel: decode + attribute) ------------------------------------------
    def _attr(self, c, va):
        w = self.w
        lo, hi = int(w.client_off[c]), int(w.client_off[c + 1])
        r = w.ranges
        k = None
        for i in range(lo, hi):
            if int(r["base"][i]) <= va:
                k = i
        at = dict(ridx=-1, in_range=False, guard=False, slot=0, st=0, kind=0, lifecycle=0, migr=1, rid=K.NO_RID)
        if k is not None:
            base, end = int(r["base"][k]), int(r["end"][k])
            if va < end:
                slot = int(r["page_off"][k]) + ((va - base) >> 12)
                ust = int(r["state"][k])
                at.update(ridx=k, in_range=True, slot=slot, kind=int(r["kind"][k]), lifecycle=int(r["lifecycle"][k]),
                          migr=int(r["migratable"][k]), rid=int(r["rid"][k]),
                          st=ust if ust != 0xFF else int(w.page_state[slot]))
            elif va < end + 4096:
                at.update(ridx=k, guard=True, slot=int(r["page_off"][k]) + ((end - base) >> 12))
        return at

    def _decode(self, e):
        if not (int(e["flags"]) & 1):
            return None
        w = self.w
        ch = int(e["channel"])
        c = int(w.channels["client"][ch])
        rec = dict(c=c, ceng=int(w.channels["engine"][ch]), eng=int(e["engine"]), kind=int(e["kind"]),
                   va=int(e["va"]), sa=int(w.clients["mode"][c]) == 1, group=0,
                   at=dict(ridx=-1, in_range=False, guard=False, rid=K.NO_RID))
        acc = int(e["access"])
        if rec["kind"] == 0:
            at = self._attr(c, rec["va"])
            rec["at"] = at
            s = _classify(rec["eng"], acc, at, w)
            rec["s"] = s
            rec["repl"] = K.SCENARIOS[s].replayable
            if rec["eng"] == 0 and acc != 2:
                rec["group"] = 1 if (acc == 1 and _classify(0, 1, at, w) != _classify(0, 0, at, w)) else 0
            else:
                rec["group"] = 2 if rec["eng"] == 0 else 2 + rec["eng"]
        elif rec["kind"] <= 5:
            rec["s"], rec["repl"] = 23 + rec["kind"] - 1, True
        else:
            rec["s"], rec["repl"] = 18 + rec["kind"] - 8, False
        return rec

    # -- phase 1 ------------------------------------------------------------------------
    def scan(self, entries, params: Params, base_index: int):
        C, R, P = self.C, self.R, self.P
        self.base = base_index
        self.u64 = np.full(3 * C + 2, E64, np.uint64)       # ft_ce | ft_sa | trap_sa | ft_gr | trap_mps
        self.u32 = np.full(2 * R + 3 * C, E32, np.uint32)   # nr0 | ext | iso1 | iso2 | iso3
        self.giso = np.full(3 * C, E32, np.uint32)
        self.dd = np.full(P * 5, E32, np.uint32)
        self.nr1 = np.full(max(P, 1), E32, np.uint32)
        self.hdd, self.hnr = {}, {}
        self.counts = np.zeros(C * K.N_SCENARIOS, np.uint64)
        self.recs = [self._decode(e) for e in entries]
        iso = params.isolation

        def mn(arr, i, v):
            if v < int(arr[i]):
                arr[i] = v

        for i, r in enumerate(self.recs):
            if r is None:
                continue
            g = base_index + i
            c, s = r["c"], r["s"]
            self.counts[c * K.N_SCENARIOS + s] += 1
            if K.S_TRAP_FIRST <= s < K.S_PARSE_FIRST:
                t = (g << 8) | s
                if r["sa"]:
                    mn(self.u64, 2 * C + c, t)
                else:
                    mn(self.u64, 3 * C + 1, t)
                continue
            ok = (0 if r["repl"] else 0x80000000) | g
            serv = 14 <= s <= 17
            at = r["at"]
            if s >= 23 or (not serv and not iso):
                t = (ok << 8) | s
                if r["sa"]:
                    mn(self.u64, C + c, t)
                elif r["ceng"] == 1:
                    mn(self.u64, c, t)
                else:
                    mn(self.u64, 3 * C, t)
            elif not serv:
                if not at["in_range"]:
                    mn(self.u32, 2 * R + c, ok)
                    if at["guard"]:
                        mn(self.u32, at["ridx"], ok)
                    else:
                        key = _nr_key(c, 0, r["va"] >> 12)
                        self.hnr[key] = min(self.hnr.get(key, E32), ok)
                elif at["kind"] == 0:
                    mn(self.u32, 2 * R + C + c, ok)
                else:
                    mn(self.u32, 2 * R + 2 * C + c, ok)
                    mn(self.u32, R + at["ridx"], ok)
            if r["kind"] == 0 and r["repl"]:
                if at["in_range"] or at["guard"]:
                    mn(self.dd, at["slot"] * 5 + r["group"], (g << 3) | r["group"])
                else:
                    key = dedup_key(c, r["eng"], r["va"] >> 12, s)
                    self.hdd[key] = min(self.hdd.get(key, E32), g)

    # -- exchange --------------------------------------------------------------------------
    def exchange_buffers(self, stage):
        if stage == 1:
            return [(self.u64, "min"), (self.u32, "min"), (self.dd, "min")]
        if stage == 2:
            return [(self.giso, "min"), (self.nr1, "min")]
        return [(self.giso, "min")]

    def hash_export(self, which):
        h = self.hdd if which == 0 else self.hnr
        keys = np.array(list(h.keys()), np.uint64)
        vals = np.array([h[k] for k in h.keys()], np.uint32)
        return keys, vals

    def hash_merge(self, which, keys, vals):
        h = self.hdd if which == 0 else self.hnr
        for k, v in zip(keys.tolist(), vals.tolist()):
            if k != E64:
                h[k] = min(h.get(k, E32), v)

    # -- resolve ---------------------------------------------------------------------------
    def resolve(self, params: Params):
        w, C, R = self.w, self.C, self.R
        u64, u32 = self.u64, self.u32
        has_mps = bool(np.any(w.clients["mode"] == K.MODE_MPS))
        gr_alive0 = has_mps and not (w.world_flags & K.WF_GR_DEAD)
        trap_mps, ft_gr = int(u64[3 * C + 1]), int(u64[3 * C])
        trapped_mps = gr_alive0 and trap_mps != E64
        gr_applied = gr_alive0 and not trapped_mps and ft_gr != E64
        gr_rel = REL_PRE if (not gr_alive0 or trapped_mps) else ((ft_gr >> 8) if gr_applied else REL_NONE)
        self.G = dict(ft_gr_ok=(ft_gr >> 8) if gr_applied else E32,
                      trap_mps_idx=(trap_mps >> 8) if trapped_mps else E32, gr_alive0=gr_alive0)
        self.cs = []
        verdict = np.zeros(C, VERDICT_DTYPE)
        general = False
        for c in range(C):
            sa = int(w.clients["mode"][c]) == 1
            fl = int(w.clients["flags"][c])
            alive0 = bool(fl & 1)
            ce_alive0 = (not sa) and alive0 and not (fl & 2)
            tsa, fsa, fce = int(u64[2 * C + c]), int(u64[C + c]), int(u64[c])
            trapped = (alive0 and tsa != E64) if sa else trapped_mps
            sa_applied = sa and alive0 and not trapped and fsa != E64
            if not alive0:
                rel = REL_PRE
            elif sa:
                rel = REL_PRE if trapped else ((fsa >> 8) if sa_applied else REL_NONE)
            else:
                rel = gr_rel
            ce_applied = ce_alive0 and fce != E64 and not (rel < (fce >> 8))
            i1, i2, i3 = int(u32[2 * R + c]), int(u32[2 * R + C + c]), int(u32[2 * R + 2 * C + c])
            elig = min(i1, i2, i3) != E32
            kill_all, tie = self._kill(params, i1, i2, i3, False)
            self.cs.append(dict(rel=rel, ft_ce_ok=E32 if fce == E64 else fce >> 8,
                                ft_sa_ok=E32 if fsa == E64 else fsa >> 8,
                                trap_sa_idx=E32 if tsa == E64 else tsa >> 8, kill_tie=tie, kill_all=kill_all,
                                alive0=alive0, sa=sa, ce_alive0=ce_alive0,
                                ce_torn=(not sa) and ((not ce_alive0) or ce_applied), trapped=trapped))
            if alive0:
                if trapped:
                    v = (1, 2, (tsa if sa else trap_mps) & 0xFF)
                elif not sa and gr_applied:
                    v = (1, 2, ft_gr & 0xFF)
                elif sa_applied:
                    v = (1, 2, fsa & 0xFF)
                elif elig:
                    v = (1, 1, (fce & 0xFF) if ce_applied else 0xFF)
                elif ce_applied:
                    v = (0, 0, fce & 0xFF)
                else:
                    v = (0, 0, 0xFF)
            else:
                n = (trap_mps & 0xFF) if (not sa and trapped_mps) else \
                    ((ft_gr & 0xFF) if (not sa and gr_applied) else 0xFE)
                v = (1, 3, n)
            verdict[c] = (v[0], v[1], v[2], 0)
            if params.isolation and elig and (rel != REL_NONE or params.m2_us <= params.benign_us):
                general = True
        self.general_path = general
        self.verdict = verdict
        return verdict

    @staticmethod
    def _kill(params, m1, m2, m3, use_m2):
        kill_all, tie = False, E32
        for m, (lat, v) in enumerate(((params.m1_us, m1), (params.m2_us, m2), (params.m3_us, m3))):
            if m == 1 and not use_m2:
                continue
            if v == E32:
                continue
            if lat < params.benign_us:
                kill_all = True
            elif lat == params.benign_us and v < tie:
                tie = v
        return kill_all, tie

    def _rep(self, r):
        at = r["at"]
        if at["in_range"] or at["guard"]:
            cur = int(self.dd[at["slot"] * 5 + r["group"]])
            if cur != E32:
                return cur >> 3
        return self.hdd.get(dedup_key(r["c"], r["eng"], r["va"] >> 12, r["s"]), E32)

    def _nr(self, r, epoch1):
        at = r["at"]
        if epoch1:
            if at["in_range"] or at["guard"]:
                return int(self.nr1[at["slot"]])
            return self.hnr.get(_nr_key(r["c"], 1, r["va"] >> 12), E32)
        if at["guard"]:
            return int(self.u32[at["ridx"]])
        return self.hnr.get(_nr_key(r["c"], 0, r["va"] >> 12), E32)

    # -- general path ----------------------------------------------------------------------
    def general(self, params: Params, stage: int):
        if not self.general_path:
            return
        R = self.R
        for i, r in enumerate(self.recs):
            if r is None or r["kind"] != 0 or 14 <= r["s"] <= 17:
                continue
            g = self.base + i
            rel = self.cs[r["c"]]["rel"]
            ok = (0 if r["repl"] else 0x80000000) | g
            if rel == REL_NONE and params.m2_us > params.benign_us:
                continue
            if r["repl"] and self._rep(r) != g:
                continue
            epoch1 = rel < ok
            at = r["at"]
            no_range = (not at["in_range"]) or epoch1
            base = 3 * r["c"]
            if stage == 1:
                if no_range:
                    self.giso[base] = min(int(self.giso[base]), ok)
                    if epoch1:
                        if at["in_range"] or at["guard"]:
                            self.nr1[at["slot"]] = min(int(self.nr1[at["slot"]]), ok)
                        else:
                            key = _nr_key(r["c"], 1, r["va"] >> 12)
                            self.hnr[key] = min(self.hnr.get(key, E32), ok)
                elif at["kind"] == 0:
                    self.giso[base + 1] = min(int(self.giso[base + 1]), ok)
                else:
                    ext = int(self.u32[R + at["ridx"]])
                    if ok == ext and ext < rel:
                        self.giso[base + 2] = min(int(self.giso[base + 2]), ok)
                    else:
                        self.giso[base + 1] = min(int(self.giso[base + 1]), ok)
            else:
                if no_range and self._nr(r, epoch1) != ok:
                    self.giso[base + 1] = min(int(self.giso[base + 1]), ok)

    def resolve2(self, params: Params):
        if not self.general_path:
            return
        R, C = self.R, self.C
        for c in range(self.C):
            cs = self.cs[c]
            if cs["rel"] == REL_NONE and params.m2_us > params.benign_us:
                continue
            g0, g1, g2 = (int(x) for x in self.giso[3 * c:3 * c + 3])
            if cs["rel"] == REL_NONE:
                g0, g2 = int(self.u32[2 * R + c]), int(self.u32[2 * R + 2 * C + c])
            cs["kill_all"], cs["kill_tie"] = self._kill(params, g0, g1, g2, True)

    # -- phase 2 -------------------------------------------------------------------------------
    def finalize(self, entries, params: Params):
        n = len(entries)
        R = self.R
        out = np.zeros(n, OUT_DTYPE)
        out["rid"] = K.NO_RID
        out["scenario"] = 0xFF
        out["client"] = 0xFFFF
        cancel, dkeys, didx = [], [], []
        G = self.G
        for i, r in enumerate(self.recs):
            if r is None:
                continue
            g = self.base + i
            cs = self.cs[r["c"]]
            out["scenario"][i] = r["s"]
            out["client"][i] = r["c"]
            if r["at"]["in_range"]:
                out["rid"][i] = r["at"]["rid"]
            s = r["s"]
            if K.S_TRAP_FIRST <= s < K.S_PARSE_FIRST:
                if not cs["sa"]:
                    canc = not (G["gr_alive0"] and g == G["trap_mps_idx"])
                else:
                    canc = not (cs["alive0"] and g == cs["trap_sa_idx"])
                out["verdict"][i] = 0x10 if canc else 0
                if canc:
                    cancel.append(g)
                continue
            parse, serv = s >= 23, 14 <= s <= 17
            outcome = 3 if parse else (1 if serv else (2 if params.isolation else 3))
            ok = (0 if r["repl"] else 0x80000000) | g
            rep_ok, dup = ok, False
            if r["kind"] == 0 and r["repl"]:
                ri = self._rep(r)
                dup = ri != g
                rep_ok = ri
                if not dup:
                    dkeys.append(dedup_key(r["c"], r["eng"], r["va"] >> 12, s))
                    didx.append(g)
            mech, canc = 0, False
            if outcome == 3:
                if cs["sa"]:
                    applied = cs["alive0"] and not cs["trapped"] and rep_ok == cs["ft_sa_ok"]
                elif r["ceng"] == 1:
                    applied = cs["ce_alive0"] and rep_ok == cs["ft_ce_ok"] and not (cs["rel"] < rep_ok)
                else:
                    applied = rep_ok == G["ft_gr_ok"]
                canc = not applied
            elif outcome == 1:
                canc = cs["rel"] != REL_NONE or (r["ceng"] == 1 and cs["ce_torn"]) or cs["kill_all"] or \
                    rep_ok > cs["kill_tie"]
            elif not dup:
                epoch1 = cs["rel"] < ok
                at = r["at"]
                if (not at["in_range"]) or epoch1:
                    mech = 1 if self._nr(r, epoch1) == ok else 2
                elif at["kind"] == 0:
                    mech = 2
                else:
                    mech = 3 if int(self.u32[R + at["ridx"]]) == ok else 2
            out["verdict"][i] = outcome | (mech << 2) | (0x10 if canc else 0) | (0x20 if dup else 0) | \
                (0x40 if r["repl"] else 0)
            if canc:
                cancel.append(g)
        return (out, np.array(dkeys, np.uint64), np.array(didx, np.uint32), np.array(cancel, np.uint32),
                self.counts.reshape(self.C, K.N_SCENARIOS))
