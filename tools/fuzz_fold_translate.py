"""Differential fuzzing of the snapshot fold + KV-pool restore and of the batched translation
against their oracles (experiment tool, GPU box): random request-id spaces (1 .. 2^20, sparse
ids), liveness-only fractions, skewed request popularity (one hot request over many tiles),
zero / long deltas, sizes across tile edges; random worlds and access streams for
``resolve_va``.

    python tools/fuzz_fold_translate.py [seconds]    # prints one JSON summary line
"""
import json
import os
import random
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from oracle import seq_oracle as so  # noqa: E402
from paper_2605_26461_b200.engine import FaultEngine  # noqa: E402
from tests import randworld as RW  # noqa: E402


def fold_case(rng, rnd):
    S = rnd.choice((rnd.randint(0, 300), rnd.randint(300, 20_000), rnd.randint(20_000, 400_000),
                    8192 * rnd.randint(1, 6) + rnd.randint(-2, 2)))
    S = max(S, 0)
    R = rnd.choice((1, 7, 300, 5000, 100_000, 1 << 20))
    if rnd.random() < 0.3:                     # skew: a few hot requests
        req = (rng.zipf(1.3, S) % R).astype(np.uint32)
    else:
        req = rng.integers(0, R, S, dtype=np.uint32)
    req[rng.random(S) < rnd.choice((0.0, 0.05, 0.5, 1.0))] = so.NO_REQ
    maxb, maxt = rnd.choice(((0, 0), (1, 4), (4, 8), (40, 200)))
    nblk = rng.integers(0, maxb + 1, S, dtype=np.uint32)
    ntok = rng.integers(0, maxt + 1, S, dtype=np.uint32)
    seq = np.arange(1, S + 1, dtype=np.uint64)
    prog = rng.integers(0, 1 << 20, S, dtype=np.uint32)
    done = (rng.random(S) < 0.05).astype(np.uint8)
    blocks = rng.integers(0, 1 << 16, int(nblk.sum()), dtype=np.uint32)
    tokens = rng.integers(0, 50000, int(ntok.sum()), dtype=np.uint32)
    return (req, seq, nblk, ntok, prog, done, blocks, tokens), R


def main():
    budget = float(sys.argv[1]) if len(sys.argv) > 1 else 300.0
    sbase = int(sys.argv[2]) if len(sys.argv) > 2 else 700_000
    eng = FaultEngine(0)
    t0 = time.time()
    st = {"fold_cases": 0, "fold_snapshots": 0, "fold_mismatches": 0, "kv_cases": 0, "kv_mismatches": 0,
          "tr_cases": 0, "tr_accesses": 0, "tr_mismatches": 0}
    bad = []
    k = 0
    while time.time() - t0 < budget:
        rnd = random.Random(sbase + k)
        rng = np.random.default_rng(sbase + k)
        k += 1
        if k % 3:
            snap, R = fold_case(rng, rnd)
            got = eng.fold(*snap, n_req_ids=R)
            want = so.fold_snapshots_np(*snap)
            ok = all(np.array_equal(getattr(got, f), getattr(want, f))
                     for f in ("order", "blk_off", "blocks", "tok_off", "tokens", "progress", "done"))
            ok = ok and got.last_seq == want.last_seq
            st["fold_cases"] += 1
            st["fold_snapshots"] += len(snap[0])
            if not ok:
                st["fold_mismatches"] += 1
                bad.append(("fold", 700_000 + k - 1))
            total = rnd.choice((1, 64, 4096, 8193, 1 << 16))
            r, fr = eng.kv_reserve(total, got.blocks % (total + 3))
            wr, wf = so.kv_reserve(total, want.blocks % (total + 3))
            st["kv_cases"] += 1
            if not (np.array_equal(r, wr) and np.array_equal(fr, wf)):
                st["kv_mismatches"] += 1
                bad.append(("kv", 700_000 + k - 1))
        else:
            w = RW.random_world(rnd, max_mps=rnd.choice((2, 4)), max_sa=rnd.choice((1, 2)))
            n = rnd.randint(1, 2000) if (rnd.random() < 0.5 or len(w.ranges) == 0) else rnd.randint(2000, 50_000)
            acc = RW.random_batch(rnd, w, n, parse_p=0.0, trap_p=0.0, wild_p=rnd.choice((0.0, 0.1, 0.3)),
                                  pool=rnd.choice((2, 4, 12)))
            eng.upload_world(w)
            hit, faults, fi, pi = eng.translate(acc)
            # the per-access restatement on small streams and range-less worlds, numpy otherwise
            want = so.translate_batch(w, acc) if (n <= 2000 or len(w.ranges) == 0) else so.translate_batch_np(w, acc)
            ok = (np.array_equal(hit, want.hit) and np.array_equal(fi, want.fault_idx) and
                  np.array_equal(pi, want.pop_idx) and np.array_equal(faults, acc[want.fault_idx]))
            st["tr_cases"] += 1
            st["tr_accesses"] += n
            if not ok:
                st["tr_mismatches"] += 1
                bad.append(("translate", 700_000 + k - 1))
    st["seconds"] = round(time.time() - t0, 1)
    st["first_mismatches"] = bad[:5]
    print(json.dumps(st))


if __name__ == "__main__":
    main()
