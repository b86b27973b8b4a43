"""Synthetic worlds and fault traces for the BASELINE.json configs.

World recipe (per client, in creation order): 4 ranges of each of 8 kinds, P pages each --
device, managed-unpopulated, managed-RO-cpu, managed-RO-gpu, VMM-RO, managed-zombie,
managed-pinned, managed-mixed-RO (random half of the pages populated, then read-only).
Built through :class:`world.WorldBuilder`, whose calls restate the reference
allocation APIs (``pkg/src/mpssim/memory.py:241-335``); ``tests/golden/make_golden.py``
builds the same recipe through the reference itself and the flat tables must match.

Trace recipe: numpy ``Generator(PCG64(seed))``; client uniform, target range uniform
in the client, ``va = base + U[0, length + 4096)`` (the +4096 lands on the guard page),
2 % wild VAs in ``[2^32, 2^33)``, engine SM/CE/PBDMA = .60/.25/.15, access
read/write/prefetch = .45/.50/.05, and entries that would *hit* under
``MemoryModel.resolve_va`` (``memory.py:339-364``) are rejected so every entry is a
plausible MMU miss.  This module only synthesises inputs; it is not the fault path.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import constants as K
from .world import ENTRY_DTYPE, FlatWorld, WorldBuilder

RANGE_KINDS = ("device", "managed", "managed_ro_cpu", "managed_ro_gpu", "vmm_ro",
               "zombie", "pinned", "mixed_ro")


def build_synthetic_world(n_clients: int, pages_per_range: int, seed: int,
                          n_standalone: int = 0, ranges_per_kind: int = 4):
    """Returns (FlatWorld, WorldBuilder).  Clients 0..n_clients-1 are MPS clients,
    followed by ``n_standalone`` standalone clients."""
    b = WorldBuilder()
    rng = np.random.Generator(np.random.PCG64(seed))
    P = pages_per_range
    size = P * K.PAGE_SIZE
    modes = [K.MODE_MPS] * n_clients + [K.MODE_STANDALONE] * n_standalone
    for mode in modes:
        c = b.add_client(mode)
        for kind in RANGE_KINDS:
            for _ in range(ranges_per_kind):
                _make_range(b, c, kind, size, P, rng)
    return b.flatten(), b


def _make_range(b: WorldBuilder, c: int, kind: str, size: int, P: int, rng):
    if kind == "device":
        return b.alloc_device(c, size)
    if kind == "managed":
        return b.alloc_managed(c, size)
    if kind == "managed_ro_cpu":
        r = b.alloc_managed(c, size)
        b.set_access(r, True)
        return r
    if kind == "managed_ro_gpu":
        r = b.alloc_managed(c, size)
        b.populate_pages(r, np.arange(P))
        b.set_access(r, True)
        return r
    if kind == "vmm_ro":
        _, r = b.vmm_create_map(c, size)
        b.set_access(r, True)
        return r
    if kind == "zombie":
        r = b.alloc_managed(c, size)
        b.make_zombie(r)
        return r
    if kind == "pinned":
        r = b.alloc_managed(c, size)
        b.pin_non_migratable(r)
        return r
    if kind == "mixed_ro":
        r = b.alloc_managed(c, size)
        mask = mixed_mask(rng, P)
        b.populate_pages(r, np.nonzero(mask)[0])
        b.set_access(r, True)
        return r
    raise ValueError(kind)


def mixed_mask(rng, P: int) -> np.ndarray:
    """Which pages of a managed-mixed-RO range get populated (one draw per range)."""
    return rng.random(P) < 0.5


# -- vectorised attribution used only to reject would-hit draws ------------------------

class _Lookup:
    def __init__(self, w: FlatWorld):
        r = w.ranges
        self.w = w
        self.keys = (r["client"].astype(np.uint64) << np.uint64(40)) | (r["base"] >> np.uint64(12))
        self.end_pages = r["end"] >> np.uint64(12)

    def attribute(self, client: np.ndarray, va: np.ndarray) -> np.ndarray:
        """Index into w.ranges of the range containing va for client, or -1."""
        page = va >> np.uint64(12)
        key = (client.astype(np.uint64) << np.uint64(40)) | page
        pos = np.searchsorted(self.keys, key, side="right").astype(np.int64) - 1
        ok = pos >= 0
        p = np.where(ok, pos, 0)
        r = self.w.ranges
        ok &= (r["client"][p] == client) & (page < self.end_pages[p]) & (va < np.uint64(1) << np.uint64(52))
        return np.where(ok, pos, -1)

    def page_state(self, ridx: np.ndarray, va: np.ndarray) -> np.ndarray:
        r = self.w.ranges
        p = np.where(ridx >= 0, ridx, 0)
        idx = r["page_off"][p].astype(np.int64) + ((va - r["base"][p]) >> np.uint64(12)).astype(np.int64)
        idx = np.where(ridx >= 0, idx, 0)
        return self.w.page_state[idx]


def would_hit(lk: _Lookup, client, va, engine, access) -> np.ndarray:
    """Side-effect-free restatement of ``MemoryModel.resolve_va``'s Hit outcome
    (``memory.py:339-364``)."""
    ridx = lk.attribute(client, va)
    r = lk.w.ranges
    p = np.where(ridx >= 0, ridx, 0)
    has = ridx >= 0
    kind = r["kind"][p]
    st = lk.page_state(ridx, va)
    res = st & 0x3
    ro = (st & K.PS_RO) != 0
    pref = access == K.ACC_PREFETCH
    hit_pref = has & (kind == K.RK_MANAGED)
    live = has & (r["lifecycle"][p] == K.LC_LIVE)
    nonmig = (r["migratable"][p] == 0) & (res == K.RES_CPU)
    am = (access == K.ACC_WRITE) & ro
    hit_other = live & ~nonmig & ~am & (res == K.RES_GPU)
    return np.where(pref, hit_pref, hit_other)


@dataclass
class TraceSpec:
    n: int
    seed: int
    wild_frac: float = 0.02
    parse_frac: float = 0.0
    trap_frac: float = 0.0


ENGINE_P = (0.60, 0.25, 0.15)
ACCESS_P = (0.45, 0.50, 0.05)


def _draw(lk: _Lookup, rng, m: int, wild_frac: float):
    w = lk.w
    C = w.n_clients
    nr = np.diff(w.client_off.astype(np.int64))
    client = rng.integers(0, C, m).astype(np.uint32)
    k = (rng.random(m) * nr[client]).astype(np.int64)
    ridx = w.client_off[client].astype(np.int64) + k
    base = w.ranges["base"][ridx]
    length = w.ranges["end"][ridx] - base
    off = (rng.random(m) * (length + K.PAGE_SIZE).astype(np.float64)).astype(np.uint64)
    va = base + off
    wild = rng.random(m) < wild_frac
    va = np.where(wild, rng.integers(1 << 32, 1 << 33, m).astype(np.uint64), va)
    engine = rng.choice(3, m, p=ENGINE_P).astype(np.uint8)
    access = rng.choice(3, m, p=ACCESS_P).astype(np.uint8)
    return client, va, engine, access


def generate_trace(w: FlatWorld, spec: TraceSpec) -> np.ndarray:
    """Config 1 / 2a / 2b traces: translation misses, plus optional parse-time and
    SM-trap entries (variant 2b)."""
    rng = np.random.Generator(np.random.PCG64(spec.seed))
    lk = _Lookup(w)
    parts, have = [], 0
    while have < spec.n:
        m = max(1024, int((spec.n - have) * 1.3))
        client, va, engine, access = _draw(lk, rng, m, spec.wild_frac)
        keep = ~would_hit(lk, client, va, engine, access)
        parts.append((client[keep], va[keep], engine[keep], access[keep]))
        have += int(keep.sum())
    client, va, engine, access = (np.concatenate([p[i] for p in parts])[:spec.n] for i in range(4))
    out = np.zeros(spec.n, ENTRY_DTYPE)
    out["va"] = va
    out["channel"] = client * 3 + engine
    out["engine"] = engine
    out["access"] = access
    out["kind"] = K.KIND_TRANSLATION
    out["flags"] = K.ENTRY_FLAG_VALID
    if spec.parse_frac or spec.trap_frac:
        u = rng.random(spec.n)
        parse = u < spec.parse_frac
        trap = (u >= spec.parse_frac) & (u < spec.parse_frac + spec.trap_frac)
        cat = rng.integers(0, 5, spec.n).astype(np.uint8)
        special = parse | trap
        out["kind"] = np.where(parse, K.KIND_PARSE_FIRST + cat,
                               np.where(trap, K.KIND_TRAP_FIRST + cat, out["kind"]))
        out["engine"] = np.where(special, K.ENG_SM, out["engine"])
        out["channel"] = np.where(special, client * 3 + K.ENG_SM, out["channel"])
        out["access"] = np.where(special, 0, out["access"])
        out["va"] = np.where(special, 0, out["va"])
    return out


def generate_access_stream(w: FlatWorld, n: int, seed: int, wild_frac: float = 0.02,
                           prefetch: float = 0.10) -> np.ndarray:
    """An access stream for the batched translation (``MemoryModel.resolve_va``,
    memory.py:339-364): the trace recipe without the would-hit rejection, so hits and misses
    mix, with ``prefetch`` of the accesses PREFETCHes (they populate managed pages for the
    accesses after them)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    lk = _Lookup(w)
    client, va, engine, _ = _draw(lk, rng, n, wild_frac)
    u = rng.random(n)
    access = np.where(u < prefetch, K.ACC_PREFETCH, np.where(u < prefetch + (1 - prefetch) * 0.47, K.ACC_WRITE,
                                                            K.ACC_READ)).astype(np.uint8)
    out = np.zeros(n, ENTRY_DTYPE)
    out["va"] = va
    out["channel"] = client * 3 + engine
    out["engine"] = engine
    out["access"] = access
    out["kind"] = K.KIND_TRANSLATION
    out["flags"] = K.ENTRY_FLAG_VALID
    return out


def generate_storm(w: FlatWorld, n: int, unique: int, seed: int,
                   wild_frac: float = 0.02, device=None):
    """Config 3: ``unique`` distinct (client, page) pairs, each with one fixed
    replayable (engine, access) -- SM, or PREFETCH from any engine -- emitted once,
    then ``n - unique`` resamples of the same pairs (in-page offset re-drawn),
    shuffled.  Exactly ``1 - unique/n`` of the entries are page duplicates."""
    rng = np.random.Generator(np.random.PCG64(seed))
    lk = _Lookup(w)
    r = w.ranges
    # distinct in-world pages (every range's pages plus its guard page) ...
    npg = ((r["end"] - r["base"]) >> np.uint64(12)).astype(np.int64) + 1
    starts = np.cumsum(npg) - npg
    n_wild = int(round(unique * wild_frac))
    n_world = unique - n_wild
    if n_world > int(npg.sum()):
        raise ValueError("world has fewer pages than the requested unique pairs")
    slots = rng.choice(int(npg.sum()), n_world, replace=False)
    ridx = np.searchsorted(starts, slots, side="right") - 1
    client = r["client"][ridx].astype(np.uint32)
    page_va = r["base"][ridx] + ((slots - starts[ridx]).astype(np.uint64) << np.uint64(12))
    # ... plus distinct wild pages in [2^32, 2^33)
    wild_page = rng.choice(1 << 20, n_wild, replace=False).astype(np.uint64)
    client = np.concatenate([client, rng.integers(0, w.n_clients, n_wild).astype(np.uint32)])
    page_va = np.concatenate([page_va, (np.uint64(1) << np.uint64(32)) + (wild_page << np.uint64(12))])
    va = page_va | rng.integers(0, 4096, unique).astype(np.uint64)
    # one fixed replayable miss per pair: SM, or PREFETCH from any engine
    engine = rng.choice(3, unique, p=ENGINE_P).astype(np.uint8)
    access = rng.choice(3, unique, p=ACCESS_P).astype(np.uint8)
    todo = np.arange(unique)
    for rnd in range(17):
        c_, v_, e_, a_ = client[todo], va[todo], engine[todo], access[todo]
        bad = would_hit(lk, c_, v_, e_, a_) | ((e_ != K.ENG_SM) & (a_ != K.ACC_PREFETCH))
        todo = todo[bad]
        nb = len(todo)
        if nb == 0:
            break
        if rnd < 16:
            engine[todo] = rng.choice(3, nb, p=ENGINE_P).astype(np.uint8)
            access[todo] = rng.choice(3, nb, p=ACCESS_P).astype(np.uint8)
        else:
            # pages where only a rare combination misses: healthy external pages miss
            # only on PREFETCH; every managed page misses on an SM write
            ridx = lk.attribute(client[todo], va[todo])
            managed = (ridx >= 0) & (r["kind"][np.where(ridx >= 0, ridx, 0)] == K.RK_MANAGED)
            access[todo] = np.where(managed, K.ACC_WRITE, K.ACC_PREFETCH)
            engine[todo] = np.where(managed, K.ENG_SM, engine[todo])
    if np.any(would_hit(lk, client, va, engine, access)):
        raise RuntimeError("could not draw a replayable miss for every storm page")
    if device is not None:
        return _expand_storm_torch(client, va, engine, access, n, seed, device)
    pick = np.concatenate([np.arange(unique, dtype=np.int64),
                           rng.integers(0, unique, n - unique)])
    va_all = va[pick]
    resampled = np.arange(n) >= unique
    va_all = np.where(resampled,
                      (va_all & ~np.uint64(0xFFF)) | rng.integers(0, 4096, n).astype(np.uint64),
                      va_all)
    perm = rng.permutation(n)
    pick, va_all = pick[perm], va_all[perm]
    out = np.zeros(n, ENTRY_DTYPE)
    out["va"] = va_all
    out["engine"] = engine[pick]
    out["access"] = access[pick]
    out["channel"] = client[pick] * 3 + engine[pick]
    out["kind"] = K.KIND_TRANSLATION
    out["flags"] = K.ENTRY_FLAG_VALID
    return out


def _expand_storm_torch(client, va, engine, access, n, seed, device):
    """Same expansion as the numpy path (each pair once + uniform resamples with a fresh
    in-page offset, shuffled) done with torch's Philox generator on the GPU, so a 10^8-entry
    trace is produced in HBM in well under a second.  Returns a uint8 tensor of n*16 bytes."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    u = len(va)
    t_va = torch.from_numpy(va.view(np.int64)).to(device)
    w1 = (client.astype(np.int64) * 3 + engine) | (engine.astype(np.int64) << 32) | \
         (access.astype(np.int64) << 40) | (np.int64(K.KIND_TRANSLATION) << 48) | \
         (np.int64(K.ENTRY_FLAG_VALID) << 56)
    t_w1 = torch.from_numpy(w1).to(device)
    pick = torch.cat([torch.arange(u, device=device),
                      torch.randint(0, u, (n - u,), device=device, generator=g)])
    off = torch.randint(0, 4096, (n,), device=device, generator=g)
    perm = torch.randperm(n, device=device, generator=g)
    pick = pick[perm]
    resampled = perm >= u
    v = t_va[pick]
    v = torch.where(resampled, (v & ~0xFFF) | off, v)
    out = torch.empty((n, 2), dtype=torch.int64, device=device)
    out[:, 0] = v
    out[:, 1] = t_w1[pick]
    return out.view(torch.uint8).reshape(-1)


def generate_mixed_storm(w: FlatWorld, n: int, seed: int, cross_frac: float = 0.1,
                         specials: tuple = ()) -> np.ndarray:
    """A large-world parity trace: half a config-3 storm (replayable duplicates), the config-2
    recipe (every scenario class, wild pages, guard pages), and ``cross_frac`` of entries that
    hit a storm page again from the same client with another (engine, access) -- SM read/write
    and PREFETCH from every engine -- so one page carries several dedup groups (in the
    claimed-slot layout the later groups go through the hash table).  ``specials`` =
    ((position in [0, 1), kind, client), ...) places parse-time (kind 1..5) or SM-trap (8..12)
    entries at fixed positions of the shuffled trace.  Synthetic worlds only (channel =
    3 * client + engine)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    n_storm = n // 2
    n_cross = int(n * cross_frac)
    n_tr = n - n_storm - n_cross
    storm = generate_storm(w, n_storm, max(1, n_storm // 10), seed)
    tr = generate_trace(w, TraceSpec(n=n_tr, seed=seed + 1))
    src = storm[rng.integers(0, n_storm, n_cross)]
    combos = np.array([(K.ENG_SM, K.ACC_READ), (K.ENG_SM, K.ACC_WRITE), (K.ENG_SM, K.ACC_PREFETCH),
                       (K.ENG_CE, K.ACC_PREFETCH), (K.ENG_PBDMA, K.ACC_PREFETCH), (K.ENG_CE, K.ACC_WRITE)],
                      np.uint8)
    pick = combos[rng.integers(0, len(combos), n_cross)]
    cross = np.zeros(n_cross, ENTRY_DTYPE)
    client = src["channel"] // 3
    cross["va"] = (src["va"] & ~np.uint64(0xFFF)) | rng.integers(0, 4096, n_cross).astype(np.uint64)
    cross["engine"] = pick[:, 0]
    cross["access"] = pick[:, 1]
    cross["channel"] = client * 3 + pick[:, 0]
    cross["kind"] = K.KIND_TRANSLATION
    cross["flags"] = K.ENTRY_FLAG_VALID
    out = np.concatenate([storm, tr, cross])[rng.permutation(n)]
    for pos, kind, c in specials:
        i = min(n - 1, int(pos * n))
        out[i] = (0, 3 * c + K.ENG_SM, K.ENG_SM, K.ACC_READ, kind, K.ENTRY_FLAG_VALID)
    return out


# -- config table (BASELINE.json "configs") -------------------------------------------

CONFIGS = {
    # name: (clients, pages/range, world seed, trace kwargs)
    "c1": dict(clients=4, pages=16, n=100_000, seed=1),
    "c2a": dict(clients=48, pages=16, n=10_000_000, seed=2),
    "c2b": dict(clients=48, pages=16, n=10_000_000, seed=2, parse_frac=1e-4, trap_frac=1e-5),
    "c3": dict(clients=48, pages=8192, n=100_000_000, seed=3, unique=10_000_000),
}


def make_config(name: str, n: int | None = None, unique: int | None = None):
    cfg = CONFIGS[name]
    w, _ = build_synthetic_world(cfg["clients"], cfg["pages"], cfg["seed"])
    n = cfg["n"] if n is None else n
    if name == "c3":
        u = cfg["unique"] if unique is None else unique
        u = min(u, n)
        return w, generate_storm(w, n, u, cfg["seed"])
    return w, generate_trace(w, TraceSpec(n=n, seed=cfg["seed"],
                                          parse_frac=cfg.get("parse_frac", 0.0),
                                          trap_frac=cfg.get("trap_frac", 0.0)))
