"""Random worlds and batches built without the reference (usable on the GPU box).

Batches are drawn from a small pool of pages per client so duplicates, same-page
cross-engine records, released clients (parse-time / trap entries) and every C3/C4/C5
corner of SURVEY.md Appendix C occur often.
"""

from __future__ import annotations

import random

import numpy as np

from paper_2605_26461_b200 import constants as K
from paper_2605_26461_b200.synth import _make_range
from paper_2605_26461_b200.world import ENTRY_DTYPE, WorldBuilder

KINDS = ("device", "managed", "managed_ro_cpu", "managed_ro_gpu", "vmm_ro", "zombie", "pinned", "mixed_ro")


def random_world(rnd: random.Random, max_mps=4, max_sa=2, dead_p=0.0):
    b = WorldBuilder()
    nrng = np.random.Generator(np.random.PCG64(rnd.randrange(1 << 30)))
    n_mps = rnd.randint(0, max_mps)
    n_sa = rnd.randint(0 if n_mps else 1, max_sa)
    for mode in [K.MODE_MPS] * n_mps + [K.MODE_STANDALONE] * n_sa:
        c = b.add_client(mode)
        for _ in range(rnd.randint(0, 6)):
            kind = rnd.choice(KINDS)
            pages = rnd.randint(1, 3)
            _make_range(b, c, kind, pages * K.PAGE_SIZE, pages, nrng)
    if dead_p:
        for c in range(len(b.modes)):
            if rnd.random() < dead_p:
                b.flags[c] = 0
            elif b.modes[c] == K.MODE_MPS and rnd.random() < dead_p:
                b.flags[c] |= K.CF_CE_TSG_DEAD
        mps = [c for c in range(len(b.modes)) if b.modes[c] == K.MODE_MPS]
        if mps and all(not (b.flags[c] & K.CF_ALIVE) for c in mps) and rnd.random() < 0.5:
            b.world_flags |= K.WF_GR_DEAD
    return b.flatten()


def random_batch(rnd: random.Random, w, n, parse_p=0.05, trap_p=0.02, wild_p=0.1, pool=4):
    out = np.zeros(n, ENTRY_DTYPE)
    r = w.ranges
    C = w.n_clients
    # a small per-client page pool so records collide
    pools = []
    for c in range(C):
        lo, hi = int(w.client_off[c]), int(w.client_off[c + 1])
        vas = []
        for _ in range(pool):
            if hi > lo and rnd.random() > wild_p:
                k = rnd.randrange(lo, hi)
                base, end = int(r["base"][k]), int(r["end"][k])
                vas.append(base + rnd.randrange(0, end - base + K.PAGE_SIZE, K.PAGE_SIZE))
            else:
                vas.append(rnd.choice((0xDEAD_0000, (1 << 32) + rnd.randrange(64) * K.PAGE_SIZE)))
        pools.append(vas)
    for i in range(n):
        c = rnd.randrange(C)
        u = rnd.random()
        valid = 0 if rnd.random() < 0.01 else 1
        if u < parse_p:
            eng = rnd.randrange(3)
            out[i] = (0, 3 * c + eng, eng, 0, 1 + rnd.randrange(5), valid)
        elif u < parse_p + trap_p:
            eng = rnd.randrange(3)
            out[i] = (0, 3 * c + eng, eng, 0, 8 + rnd.randrange(5), valid)
        else:
            eng = rnd.choice((0, 0, 1, 2))
            acc = rnd.choice((0, 1, 1, 2))
            va = rnd.choice(pools[c]) + rnd.randrange(K.PAGE_SIZE)
            out[i] = (va, 3 * c + eng, eng, acc, 0, valid)
    return out


def random_params(rnd: random.Random):
    from oracle.seq_oracle import Params
    lat = rnd.random() < 0.5
    return Params(isolation=rnd.random() < 0.65, benign_us=226,
                  m1_us=rnd.choice((131, 226, 300)) if lat else 131,
                  m2_us=rnd.choice((2780, 226, 100)) if lat else 2780,
                  m3_us=rnd.choice((1700, 226, 0)) if lat else 1700)
