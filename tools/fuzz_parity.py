"""Differential fuzzing of the fault path against the C oracle (experiment tool, GPU box):
random worlds (dead clients, GR-dead worlds), random batch parameters (isolation on / off,
latency ties), random batches (duplicates, same-page cross-engine records, parse-time records,
traps, wild pages, invalid entries), every dedup layout (auto / dense / sparse) and both the
device-resident and the host form, all six outputs compared bit for bit.

    python tools/fuzz_parity.py [seconds] [seed base]   # prints one JSON summary line
"""
import json
import os
import random
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from oracle import c_oracle as co  # noqa: E402
from paper_2605_26461_b200.engine import FaultEngine  # noqa: E402
from tests import randworld as RW  # noqa: E402
from tests.test_gpu_parity import bp, run_device  # noqa: E402

FIELDS = ("out", "verdict", "counts", "dedup_keys", "dedup_idx", "cancel")


def main():
    budget = float(sys.argv[1]) if len(sys.argv) > 1 else 300.0
    sbase = int(sys.argv[2]) if len(sys.argv) > 2 else 900_000
    eng = FaultEngine(0)
    t0 = time.time()
    stats = {"batches": 0, "entries": 0, "mismatches": 0, "by_layout": {}, "by_form": {}, "isolation_on": 0,
             "max_batch": 0}
    bad = []
    seed = 0
    while time.time() - t0 < budget:
        rnd = random.Random(sbase + seed)
        seed += 1
        w = RW.random_world(rnd, max_mps=rnd.choice((2, 4, 6)), max_sa=rnd.choice((1, 2, 3)),
                            dead_p=rnd.choice((0.0, 0.0, 0.15, 0.3)))
        p = RW.random_params(rnd)
        n = rnd.randint(1, 300) if rnd.random() < 0.85 else rnd.randint(1000, 40_000)
        entries = RW.random_batch(rnd, w, n, parse_p=rnd.choice((0.05, 0.01, 0.001)),
                                  trap_p=rnd.choice((0.02, 0.005, 0.0005)), wild_p=rnd.choice((0.1, 0.3)),
                                  pool=rnd.choice((2, 4, 12)))
        want = co.process_batch(w, entries, p)
        layout = rnd.choice(("auto", "dense", "sparse"))
        form = "device" if rnd.random() < 0.7 else "host"
        if form == "device":
            got = run_device(eng, w, entries, p, layout)
        else:
            eng.set_dedup_layout(layout)
            eng.upload_world(w)
            got = eng.process(entries, bp(p))
            eng.set_dedup_layout("auto")
        ok = all(np.array_equal(getattr(got, f), getattr(want, f)) for f in FIELDS)
        stats["batches"] += 1
        stats["entries"] += n
        stats["max_batch"] = max(stats["max_batch"], n)
        stats["isolation_on"] += int(p.isolation)
        stats["by_layout"][layout] = stats["by_layout"].get(layout, 0) + 1
        stats["by_form"][form] = stats["by_form"].get(form, 0) + 1
        if not ok:
            stats["mismatches"] += 1
            if len(bad) < 5:
                bad.append({"seed": sbase + seed - 1, "layout": layout, "form": form, "n": n,
                            "fields": [f for f in FIELDS if not np.array_equal(getattr(got, f), getattr(want, f))]})
    stats["seconds"] = round(time.time() - t0, 1)
    stats["first_mismatches"] = bad
    print(json.dumps(stats))


if __name__ == "__main__":
    main()
