"""Flat, device-uploadable snapshot of the reference's memory + execution model.

The reference keeps its world as Python objects: ``VaRange`` with a list of
``PageRec`` (``pkg/src/mpssim/memory.py:76-101``), clients/channels/TSGs in
``GpuModel`` (``pkg/src/mpssim/execmodel.py:127-204``).  The batch path needs
that state as flat tables it can put in HBM once and read from every entry:

* ``ranges``      -- one 32-byte ``RangeEntry`` per live ``VaRange``, sorted by
                     (client, base): the interval table searched by binary search
                     (replaces the linear ``MemoryModel.range_at`` scan, memory.py:233-237)
* ``client_off``  -- CSR offsets of each client's slice of ``ranges``
* ``page_state``  -- one byte per 4 KiB page (residency bits 0-1, read-only bit 2),
                     ``npages + 1`` slots per range (the trailing slot is the range's
                     guard page, memory.py:214-219, used as a dedup/NR slot only)
* ``channels``    -- channel index -> (client, engine); the reference's
                     ``UvmHandler.channel_to_pid`` (pipeline.py:73,89-91)
* ``clients``     -- MPS vs standalone (execmodel.py:164-188) + liveness flags

Two producers exist: :class:`WorldBuilder`, a from-scratch restatement of the
reference's allocation APIs used for synthetic configs (no reference import),
and :func:`export_reference_world`, which reads a live reference ``World``
(duck-typed; used by the DES drop-in shim).
``tests/test_oracle_vs_reference.py::test_classify_equals_reference_classify_on_synthetic_world`` checks the two
give identical tables for the same recipe.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import constants as K

ENTRY_DTYPE = np.dtype([("va", "<u8"), ("channel", "<u4"), ("engine", "u1"),
                        ("access", "u1"), ("kind", "u1"), ("flags", "u1")])
RANGE_DTYPE = np.dtype([("base", "<u8"), ("end", "<u8"), ("client", "<u4"),
                        ("page_off", "<u4"), ("kind", "u1"), ("lifecycle", "u1"),
                        ("migratable", "u1"), ("state", "u1"), ("rid", "<u4")])
CHANNEL_DTYPE = np.dtype([("client", "<u4"), ("engine", "u1"), ("pad", "u1", (3,))])
CLIENT_DTYPE = np.dtype([("mode", "u1"), ("flags", "u1"), ("pad", "<u2")])
OUT_DTYPE = np.dtype([("rid", "<u4"), ("scenario", "u1"), ("verdict", "u1"),
                      ("client", "<u2")])
VERDICT_DTYPE = np.dtype([("state", "u1"), ("reason", "u1"), ("notifier", "u1"),
                          ("flags", "u1")])
REMAP_DTYPE = np.dtype([("va", "<u8"), ("phys", "<u8")])

assert ENTRY_DTYPE.itemsize == 16 and RANGE_DTYPE.itemsize == 32
assert CHANNEL_DTYPE.itemsize == 8 and CLIENT_DTYPE.itemsize == 4
assert OUT_DTYPE.itemsize == 8 and VERDICT_DTYPE.itemsize == 4 and REMAP_DTYPE.itemsize == 16

NO_CLIENT = 0xFFFFFFFF


def page_state_byte(residency: int, read_only: bool) -> int:
    return residency | (K.PS_RO if read_only else 0)


@dataclass
class FlatWorld:
    clients: np.ndarray                  # CLIENT_DTYPE[C]
    channels: np.ndarray                 # CHANNEL_DTYPE[nch]
    ranges: np.ndarray                   # RANGE_DTYPE[R], sorted by (client, base)
    client_off: np.ndarray               # uint32[C+1]
    page_state: np.ndarray               # uint8[P]
    world_flags: int = 0
    client_names: list = field(default_factory=list)    # reference pids, e.g. "c1"
    channel_names: list = field(default_factory=list)   # reference channel ids, e.g. "c1.sm"

    @property
    def n_clients(self) -> int:
        return len(self.clients)

    @property
    def n_pages(self) -> int:
        return len(self.page_state)

    def channel_index(self, client: int, engine: int) -> int:
        """Channel index of (client, engine); synthetic worlds use 3*client+engine."""
        hits = np.nonzero((self.channels["client"] == client)
                          & (self.channels["engine"] == engine))[0]
        if len(hits) == 0:
            raise KeyError((client, engine))
        return int(hits[0])

    def validate(self) -> None:
        """Host-side restatement of the upload checks in ``mpsf_upload_world``."""
        C = self.n_clients
        r = self.ranges
        assert len(self.client_off) == C + 1
        assert self.client_off[0] == 0 and self.client_off[-1] == len(r)
        for c in range(C):
            lo, hi = int(self.client_off[c]), int(self.client_off[c + 1])
            seg = r[lo:hi]
            assert np.all(seg["client"] == c)
            assert np.all(seg["base"] < seg["end"])
            assert np.all(seg["base"][1:] >= seg["end"][:-1]), "overlapping ranges"


class _Range:
    __slots__ = ("rid", "client", "base", "length", "kind", "lifecycle",
                 "migratable", "pages", "backing_handle", "semaphore_pool")

    def __init__(self, rid, client, base, length, kind, pages, backing_handle=None):
        self.rid = rid
        self.client = client
        self.base = base
        self.length = length
        self.kind = kind
        self.lifecycle = K.LC_LIVE
        self.migratable = True
        self.pages = pages               # uint8 page-state array
        self.backing_handle = backing_handle
        self.semaphore_pool = False

    @property
    def end(self) -> int:
        return self.base + self.length

    @property
    def npages(self) -> int:
        return self.length >> K.PAGE_SHIFT


class WorldBuilder:
    """Restatement of the reference's world-construction APIs, enough to build
    the synthetic configs without importing the reference.

    Mirrors: client/channel wiring (``execmodel.py:164-204``; channel ids
    ``f"{pid}.{engine}"`` at 191), VA placement with a one-page guard
    (``memory.py:214-219``), rid numbering (``memory.py:221-231``), physical page
    bump allocation with the dummy pool taking pages 1..513 first
    (``memory.py:135-153``), and the page-state effects of ``set_access``
    (295-303), ``populate_page`` (368-380), ``make_zombie`` (305-314),
    ``pin_non_migratable`` (316-326), ``create_managed_at`` (395-404) and
    ``convert_external_to_managed`` (406-426).
    """

    def __init__(self):
        self.modes: list[int] = []
        self.names: list[str] = []
        self.flags: list[int] = []
        self.world_flags = 0
        self.ranges: dict[int, _Range] = {}
        self._va_cursor: dict[int, int] = {}
        self._next_rid = 1
        self._next_page = 1 + 1 + K.DUMMY_CHUNK_PAGES   # dummy 4K page + 2M chunk
        self._next_handle = 1
        self.allocations: dict[int, list[int]] = {}     # handle -> physical pages

    # -- clients ---------------------------------------------------------------
    def add_client(self, mode: int) -> int:
        c = len(self.modes)
        self.modes.append(mode)
        self.names.append(f"c{c + 1}")
        self.flags.append(K.CF_ALIVE)
        return c

    # -- physical pages ------------------------------------------------------------
    def _take_pages(self, count: int) -> list[int]:
        pages = list(range(self._next_page, self._next_page + count))
        self._next_page += count
        return pages

    def vmm_create(self, size: int) -> int:
        npages = -(-size // K.PAGE_SIZE)
        h = self._next_handle
        self._next_handle += 1
        self.allocations[h] = self._take_pages(npages)
        return h

    # -- VA ranges -------------------------------------------------------------------
    def _place(self, client: int, length: int) -> int:
        base = self._va_cursor.get(client, K.VA_CURSOR_START)
        self._va_cursor[client] = base + length + K.PAGE_SIZE
        return base

    def _add(self, client, length, kind, pages, base=None, backing_handle=None) -> _Range:
        if base is None:
            base = self._place(client, length)
        rng = _Range(self._next_rid, client, base, length, kind, pages, backing_handle)
        self._next_rid += 1
        self.ranges[rng.rid] = rng
        return rng

    def alloc_device(self, client: int, size: int) -> _Range:
        h = self.vmm_create(size)
        n = len(self.allocations[h])
        pages = np.full(n, page_state_byte(K.RES_GPU, False), np.uint8)
        return self._add(client, n * K.PAGE_SIZE, K.RK_EXTERNAL, pages, backing_handle=h)

    def alloc_managed(self, client: int, size: int) -> _Range:
        n = -(-size // K.PAGE_SIZE)
        pages = np.zeros(n, np.uint8)
        return self._add(client, n * K.PAGE_SIZE, K.RK_MANAGED, pages)

    def vmm_map(self, client: int, handle: int) -> _Range:
        n = len(self.allocations[handle])
        pages = np.full(n, page_state_byte(K.RES_GPU, False), np.uint8)
        return self._add(client, n * K.PAGE_SIZE, K.RK_EXTERNAL, pages, backing_handle=handle)

    def vmm_create_map(self, client: int, size: int):
        h = self.vmm_create(size)
        return h, self.vmm_map(client, h)

    def set_access(self, rng: _Range, read_only: bool) -> None:
        res = rng.pages & 0x3
        if rng.kind == K.RK_MANAGED:
            res = np.where(res == K.RES_UNPOP, K.RES_CPU, res).astype(np.uint8)
        rng.pages = (res | (K.PS_RO if read_only else 0)).astype(np.uint8)

    def populate_page(self, rng: _Range, idx: int) -> None:
        st = int(rng.pages[idx])
        if st & 0x3 == K.RES_GPU:
            return
        # a non-GPU page has no backing chunk here, so one is allocated (memory.py:374-376)
        self._take_pages(1)
        rng.pages[idx] = (st & K.PS_RO) | K.RES_GPU

    def populate_pages(self, rng: _Range, idx) -> None:
        """Vectorised ``populate_page`` over several page indices."""
        idx = np.asarray(idx, np.int64)
        st = rng.pages[idx]
        todo = idx[(st & 0x3) != K.RES_GPU]
        self._take_pages(0)
        self._next_page += len(todo)
        rng.pages[todo] = (rng.pages[todo] & K.PS_RO) | K.RES_GPU

    def make_zombie(self, rng: _Range) -> None:
        assert rng.kind == K.RK_MANAGED
        rng.lifecycle = K.LC_ZOMBIE

    def pin_non_migratable(self, rng: _Range) -> None:
        assert rng.kind == K.RK_MANAGED
        rng.migratable = False
        rng.pages = ((rng.pages & K.PS_RO) | K.RES_CPU).astype(np.uint8)

    def create_managed_at(self, client: int, base: int) -> _Range:
        return self._add(client, K.PAGE_SIZE, K.RK_MANAGED, np.zeros(1, np.uint8), base=base)

    def convert_external_to_managed(self, rng: _Range) -> _Range:
        assert rng.kind == K.RK_EXTERNAL
        del self.ranges[rng.rid]
        pages = np.full(rng.npages, page_state_byte(K.RES_GPU, False), np.uint8)
        return self._add(rng.client, rng.length, K.RK_MANAGED, pages, base=rng.base)

    # -- export -----------------------------------------------------------------------
    def flatten(self) -> FlatWorld:
        return _flatten(self.modes, self.flags, self.names, self.world_flags,
                        [(r.rid, r.client, r.base, r.length, r.kind, r.lifecycle,
                          r.migratable, r.pages) for r in self.ranges.values()])


def _flatten(modes, flags, names, world_flags, rows) -> FlatWorld:
    C = len(modes)
    clients = np.zeros(C, CLIENT_DTYPE)
    clients["mode"] = modes
    clients["flags"] = flags
    channels = np.zeros(3 * C, CHANNEL_DTYPE)
    channels["client"] = np.repeat(np.arange(C, dtype=np.uint32), 3)
    channels["engine"] = np.tile(np.arange(3, dtype=np.uint8), C)
    channel_names = [f"{names[c]}.{K.ENGINE_NAMES[e]}" for c in range(C) for e in range(3)]

    rows = sorted(rows, key=lambda t: (t[1], t[2]))
    R = len(rows)
    ranges = np.zeros(R, RANGE_DTYPE)
    total = sum(len(t[7]) + 1 for t in rows)
    page_state = np.zeros(total, np.uint8)
    off = 0
    for i, (rid, client, base, length, kind, lifecycle, migratable, pages) in enumerate(rows):
        n = len(pages)
        assert n * K.PAGE_SIZE == length
        page_state[off:off + n] = pages
        uniform = n > 0 and np.all(pages == pages[0])
        ranges[i] = (base, base + length, client, off, kind, lifecycle,
                     1 if migratable else 0,
                     int(pages[0]) if uniform else K.PAGE_STATE_PER_PAGE, rid)
        off += n + 1
    client_off = np.zeros(C + 1, np.uint32)
    if R:
        counts = np.bincount(ranges["client"].astype(np.int64), minlength=C)
        client_off[1:] = np.cumsum(counts)
    w = FlatWorld(clients, channels, ranges, client_off, page_state, world_flags,
                  list(names), channel_names)
    w.validate()
    return w


# -- export from a live reference World (duck-typed; no reference import) -----------

_RES = {"unpopulated": K.RES_UNPOP, "cpu": K.RES_CPU, "gpu": K.RES_GPU}


def export_reference_world(world) -> FlatWorld:
    """Snapshot a reference ``World`` (``machine.build_world``) into flat tables.

    Reads ``world.gpu.clients`` / ``channels`` / ``tsgs`` / ``mps_session`` and
    ``world.mem.ranges`` exactly as the reference's own lookups do
    (``pipeline.py:103``, ``memory.py:233-237``, ``pipeline.py:244-258``).
    Channel table order is client order x engine (sm, ce, pbdma).
    """
    gpu = world.gpu
    pids = sorted(gpu.clients, key=lambda p: int(p[1:]) if p[1:].isdigit() else p)
    index = {p: i for i, p in enumerate(pids)}
    modes, flags = [], []
    session = gpu.mps_session
    for p in pids:
        cl = gpu.clients[p]
        mps = cl.mode == "mps-client"
        modes.append(K.MODE_MPS if mps else K.MODE_STANDALONE)
        f = K.CF_ALIVE if cl.state.value == "running" else 0
        if mps:
            ce = gpu.channels[cl.channel_ids[_engine_key(cl, "ce")]]
            tsg = gpu.tsgs.get(ce.tsg_id)
            if tsg is None or tsg.state.value == "destroyed":
                f |= K.CF_CE_TSG_DEAD
        flags.append(f)
    wflags = 0
    if session is not None:
        gr = gpu.tsgs.get(session.gr_tsg)
        if gr is None or gr.state.value == "destroyed":
            wflags |= K.WF_GR_DEAD
    rows = []
    for rng in world.mem.ranges.values():
        if rng.owner_pid not in index:
            continue
        pages = np.array([_RES[p.residency.value] | (K.PS_RO if p.protection.value == "read-only" else 0)
                          for p in rng.pages], np.uint8)
        rows.append((rng.rid, index[rng.owner_pid], rng.base, rng.length,
                     K.RK_MANAGED if rng.kind.value == "managed" else K.RK_EXTERNAL,
                     K.LC_ZOMBIE if rng.lifecycle.value == "zombie" else K.LC_LIVE,
                     bool(rng.migratable), pages))
    return _flatten(modes, flags, pids, wflags, rows)


def _engine_key(client, name):
    for k in client.channel_ids:
        if getattr(k, "value", k) == name:
            return k
    raise KeyError(name)


# -- (de)serialisation for golden fixtures ----------------------------------------------

def flat_to_dict(w: FlatWorld) -> dict:
    return dict(
        clients=[[int(x["mode"]), int(x["flags"])] for x in w.clients],
        channels=[[int(x["client"]), int(x["engine"])] for x in w.channels],
        ranges=[[int(x[f]) for f in RANGE_DTYPE.names] for x in w.ranges],
        client_off=[int(x) for x in w.client_off],
        page_state=w.page_state.tobytes().hex(),
        world_flags=int(w.world_flags),
        client_names=list(w.client_names),
        channel_names=list(w.channel_names),
    )


def flat_from_dict(d: dict) -> FlatWorld:
    clients = np.zeros(len(d["clients"]), CLIENT_DTYPE)
    for i, (m, f) in enumerate(d["clients"]):
        clients[i]["mode"], clients[i]["flags"] = m, f
    channels = np.zeros(len(d["channels"]), CHANNEL_DTYPE)
    for i, (c, e) in enumerate(d["channels"]):
        channels[i]["client"], channels[i]["engine"] = c, e
    ranges = np.zeros(len(d["ranges"]), RANGE_DTYPE)
    for i, row in enumerate(d["ranges"]):
        ranges[i] = tuple(row)
    return FlatWorld(clients, channels, ranges, np.array(d["client_off"], np.uint32),
                     np.frombuffer(bytes.fromhex(d["page_state"]), np.uint8).copy(),
                     d["world_flags"], list(d["client_names"]), list(d["channel_names"]))


def entries_to_list(e: np.ndarray) -> list:
    return [[int(x[f]) for f in ENTRY_DTYPE.names] for x in e]


def entries_from_list(rows: list) -> np.ndarray:
    out = np.zeros(len(rows), ENTRY_DTYPE)
    for i, r in enumerate(rows):
        out[i] = tuple(r)
    return out
