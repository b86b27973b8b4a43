"""Pin the batched-translation oracle (``seq_oracle.translate_batch``) against the reference's
own ``MemoryModel.resolve_va`` run access by access (memory.py:339-364), including the prefetch
population side effect.  Skips when the reference is not importable (the GPU box)."""

import random

import numpy as np
import pytest

from paper_2605_26461_b200 import constants as K
from paper_2605_26461_b200.world import ENTRY_DTYPE, export_reference_world

from oracle import seq_oracle as so
from tests import refharness as H

pytestmark = pytest.mark.skipif(not H.reference_available(), reason="reference not present")


def random_accesses(rnd, w, flat, n):
    """Accesses aimed at the world's ranges, their guard pages and wild VAs, with repeats of
    the same page so in-batch prefetch population matters."""
    from mpssim.execmodel import EngineClass  # noqa: F401
    r = flat.ranges
    pool = []
    for _ in range(max(4, n // 3)):
        if rnd.random() < 0.1 or len(r) == 0:
            ch = rnd.randrange(len(flat.channels))
            pool.append((ch, rnd.randrange(1 << 32, 1 << 33) & ~0xFFF))
        else:
            k = rnd.randrange(len(r))
            c = int(r["client"][k])
            chans = [i for i in range(len(flat.channels)) if int(flat.channels["client"][i]) == c]
            npg = (int(r["end"][k]) - int(r["base"][k])) >> 12
            pool.append((rnd.choice(chans), int(r["base"][k]) + (rnd.randrange(npg + 1) << 12)))
    e = np.zeros(n, ENTRY_DTYPE)
    for i in range(n):
        ch, page_va = rnd.choice(pool)
        e[i]["va"] = page_va + rnd.randrange(4096)
        e[i]["channel"] = ch
        e[i]["engine"] = int(flat.channels["engine"][ch])
        e[i]["access"] = rnd.choices((0, 1, 2), (0.4, 0.35, 0.25))[0]
        e[i]["kind"] = 0
        e[i]["flags"] = K.ENTRY_FLAG_VALID if rnd.random() > 0.02 else 0
    return e


def reference_translate(w, flat, entries):
    from mpssim.execmodel import EngineClass
    from mpssim.memory import AccessType, Hit
    hit, faults, pops = [], [], []
    for i, e in enumerate(entries):
        if not (int(e["flags"]) & K.ENTRY_FLAG_VALID):
            hit.append(0xFF)
            continue
        ch = flat.channel_names[int(e["channel"])]
        pid = w.gpu.channels[ch].owner_pid
        va = int(e["va"])
        rng = w.mem.range_at(pid, va)
        rec = rng.pages[rng.page_index(va)] if rng is not None else None
        before = rec.residency if rec is not None else None
        res = w.mem.resolve_va(w, pid, va, AccessType(H.ACCESSES[int(e["access"])]),
                               EngineClass(H.ENGINES[int(e["engine"])]), channel_id=ch)
        ok = isinstance(res, Hit)
        hit.append(1 if ok else 0)
        if not ok:
            faults.append(i)
        if rec is not None and rec.residency != before:      # populate_page ran (memory.py:368-380)
            pops.append(i)
    return np.array(hit, np.uint8), np.array(faults, np.uint32), np.array(pops, np.uint32)


@pytest.mark.parametrize("seed", range(3))
def test_translate_oracle_matches_resolve_va(seed):
    H.import_reference()
    rnd = random.Random(900 + seed)
    for it in range(25):
        spec = H.random_small_world_spec(rnd)
        w = H.build_reference_world(spec)
        flat = export_reference_world(w)
        entries = random_accesses(rnd, w, flat, rnd.randint(1, 120))
        got = so.translate_batch(flat, entries)
        hit, faults, pops = reference_translate(w, flat, entries)
        assert np.array_equal(got.hit, hit), (seed, it)
        assert np.array_equal(got.fault_idx, faults), (seed, it)
        assert np.array_equal(got.pop_idx, pops), (seed, it)


def test_vectorized_translate_oracle_matches_sequential():
    """The numpy form used at large sizes equals the access-by-access restatement (no
    reference needed: runs on the synthetic worlds)."""
    from paper_2605_26461_b200 import synth
    rnd = random.Random(5)
    for cfg in ((4, 16, 1), (6, 64, 3)):
        w, _ = synth.build_synthetic_world(*cfg)
        for it in range(4):
            e = synth.generate_access_stream(w, 4000, seed=rnd.randrange(1 << 30))
            a = so.translate_batch(w, e)
            b = so.translate_batch_np(w, e)
            assert np.array_equal(a.hit, b.hit) and np.array_equal(a.fault_idx, b.fault_idx)
            assert np.array_equal(a.pop_idx, b.pop_idx)
