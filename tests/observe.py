"""Turn a packed batch result (OutRecord[] + ClientVerdict[]) into the reference's own
observables, so GPU results, oracle results and reference runs compare in one vocabulary:

* ``labels``        -- ``service_bottom_half``'s return list (pipeline.py:160-183), drain order
* ``isolation``     -- ``uvm.isolation_outcomes`` as (scenario, mechanism, pid) (pipeline.py:299-301)
* ``benign``        -- ``finish_benign_service`` calls as (channel, va, serviced) in event order
* ``fatal_reports`` -- ``len(rmgsp.fatal_reports)`` (pipeline.py:231)
* ``clients``       -- (state, reason, notifier) per pid, what ``client_final`` records (machine.py:203-217)
* ``scenarios``     -- ``uvm.fault_log`` scenarios in raise order
"""

from __future__ import annotations

import numpy as np

from paper_2605_26461_b200 import constants as K


def drain_order(entries, out) -> list:
    valid = (entries["flags"] & K.ENTRY_FLAG_VALID) != 0
    notrap = entries["kind"] < K.KIND_TRAP_FIRST
    rep = (out["verdict"] & K.V_REPLAYABLE) != 0
    idx = np.arange(len(entries))
    first = idx[valid & notrap & rep]
    second = idx[valid & notrap & ~rep]
    return list(first) + list(second)


def observables(flat, entries, out, verdict) -> dict:
    order = drain_order(entries, out)
    v = out["verdict"]
    labels, iso, benign, fatal = [], [], [], 0
    for i in order:
        o = int(v[i]) & 3
        labels.append(K.OUTCOME_NAMES[o])
        dup = bool(v[i] & K.V_DUP)
        canc = bool(v[i] & K.V_CANCELLED)
        if dup:
            continue
        s = int(out["scenario"][i])
        if o == K.OUT_ISOLATED:
            iso.append((K.SCENARIOS[s].sid, K.MECH_NAMES[(int(v[i]) >> 2) & 3],
                        flat.client_names[int(out["client"][i])]))
        elif o == K.OUT_SERVICED:
            benign.append((flat.channel_names[int(entries["channel"][i])],
                           int(entries["va"][i]), not canc))
        elif o == K.OUT_FATAL and not canc:
            fatal += 1
    clients = {}
    for c, pid in enumerate(flat.client_names):
        vc = verdict[c]
        clients[pid] = ("running" if vc["state"] == K.ST_RUNNING else "terminated",
                        K.REASON_NAMES[int(vc["reason"])] or "?",
                        "?" if int(vc["notifier"]) == K.NOTIFIER_UNCHANGED
                        else K.notifier_name(int(vc["notifier"])))
    scen = [K.SCENARIOS[int(out["scenario"][i])].sid for i in range(len(entries))
            if entries["flags"][i] & K.ENTRY_FLAG_VALID and entries["kind"][i] < K.KIND_TRAP_FIRST]
    return dict(labels=labels, isolation=iso, benign=benign, fatal_reports=fatal,
                clients=clients, scenarios=scen)


def normalise_reference(ref: dict) -> dict:
    """JSON round-trip friendly form of refharness.run_reference_batch output."""
    return dict(labels=list(ref["labels"]),
                isolation=[tuple(x) for x in ref["isolation"]],
                benign=[tuple(x) for x in ref["benign"]],
                fatal_reports=int(ref["fatal_reports"]),
                clients={k: tuple(v) for k, v in ref["clients"].items()},
                scenarios=list(ref["scenarios"]))
