"""Trace and fault-buffer formats.

* ``render_trace`` -- the reference's ``Trace`` line format (``t=.. who=.. kind=.. k=v``,
  ``Trace.render_record``, kernel.py:127-132) for a processed batch: the top-half lines per
  entry (``fault_raised``, ``shadow_copy``; pipeline.py:113-143) and the bottom-half lines
  the batch verdicts produce (``bh_service``, ``parse_fatal``, ``tlb_invalidate``,
  ``fatal_report``, ``isolate_begin``; pipeline.py:160-183, 224-230, 296-298), rendered by
  ``mpsf_render_trace`` in libmpsf.so on all host threads.  Lines parse with the
  reference's ``parse_trace_line`` (kernel.py:140-148).
* ``write_dump`` / ``read_dump`` -- a binary fault-buffer dump: a 64-byte header, the
  16-byte entries exactly as ``mpsf_process`` takes them (read back zero-copy with
  ``np.memmap``), optional per-entry raise times, and the channel / client names the
  renderer needs, so a recorded buffer replays and renders without the simulator.
"""

from __future__ import annotations

import ctypes as C
import struct
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib
from .world import ENTRY_DTYPE, OUT_DTYPE

RENDER_TOP = 1
RENDER_DRAIN = 2

DUMP_MAGIC = b"MPSFBUF1"
DUMP_VERSION = 1
_HDR = struct.Struct("<8sIIQQIIIIQ8x")       # 64 bytes
assert _HDR.size == 64
F_ISOLATION, F_TRAISE = 1, 2


def _names(lst):
    arr = (C.c_char_p * max(len(lst), 1))()
    for i, s in enumerate(lst):
        arr[i] = s.encode()
    return arr


def render_trace(entries: np.ndarray, out: np.ndarray, channel_names, client_names, t_drain: int = 0,
                 t_raise: Optional[np.ndarray] = None, parts: int = RENDER_TOP | RENDER_DRAIN,
                 m_us=(131, 2780, 1700), threads: int = 0) -> str:
    """Trace text (``Trace.render()`` format, one ``\\n``-terminated line per record) of a
    batch and its OutRecords; see ``include/mpsf.h`` ``mpsf_render_trace``."""
    lib = _lib.load()
    entries = np.ascontiguousarray(entries, dtype=ENTRY_DTYPE)
    out = np.ascontiguousarray(out, dtype=OUT_DTYPE)
    n = len(entries)
    if len(out) != n:
        raise ValueError("entries and out records differ in length")
    ch, cl = _names(channel_names), _names(client_names)
    tr = None
    if t_raise is not None:
        tr = np.ascontiguousarray(t_raise, dtype=np.uint64)
        if len(tr) != n:
            raise ValueError("t_raise length")
    p = _lib.RenderParams(t_drain=t_drain, t_raise=tr.ctypes.data if tr is not None else None,
                          m1_us=m_us[0], m2_us=m_us[1], m3_us=m_us[2], parts=parts,
                          channel_names=C.cast(ch, C.POINTER(C.c_char_p)), n_channels=len(channel_names),
                          n_clients=len(client_names), client_names=C.cast(cl, C.POINTER(C.c_char_p)),
                          threads=threads)
    cap = 320 * n + 4096
    e_ptr = entries.ctypes.data if n else None
    o_ptr = out.ctypes.data if n else None
    while True:
        buf = np.empty(cap, np.uint8)
        got = lib.mpsf_render_trace(e_ptr, o_ptr, n, C.byref(p), buf.ctypes.data, cap)
        if got < 0:
            from .errors import raise_for
            raise_for(int(got), lib.mpsf_strerror(int(got)).decode())
        if got <= cap:
            return buf[:got].tobytes().decode()
        cap = got


@dataclass
class Dump:
    entries: np.ndarray                  # ENTRY_DTYPE[n] (memmap)
    channel_names: list = field(default_factory=list)
    client_names: list = field(default_factory=list)
    isolation: bool = True
    base_index: int = 0
    t_drain: int = 0
    t_raise: Optional[np.ndarray] = None


def write_dump(path: str, entries: np.ndarray, channel_names=(), client_names=(), isolation: bool = True,
               base_index: int = 0, t_drain: int = 0, t_raise: Optional[np.ndarray] = None) -> None:
    entries = np.ascontiguousarray(entries, dtype=ENTRY_DTYPE)
    n = len(entries)
    names = b"".join(struct.pack("<H", len(s.encode())) + s.encode() for s in list(channel_names) + list(client_names))
    flags = (F_ISOLATION if isolation else 0) | (F_TRAISE if t_raise is not None else 0)
    with open(path, "wb") as f:
        f.write(_HDR.pack(DUMP_MAGIC, DUMP_VERSION, ENTRY_DTYPE.itemsize, n, base_index, flags,
                          len(channel_names), len(client_names), len(names), t_drain))
        f.write(entries.tobytes())
        if t_raise is not None:
            tr = np.ascontiguousarray(t_raise, dtype="<u8")
            if len(tr) != n:
                raise ValueError("t_raise length")
            f.write(tr.tobytes())
        f.write(names)


def read_dump(path: str) -> Dump:
    with open(path, "rb") as f:
        hdr = f.read(_HDR.size)
    if len(hdr) < _HDR.size:
        raise ValueError(f"{path}: truncated header")
    magic, ver, esz, n, base, flags, nch, ncl, nb, t_drain = _HDR.unpack(hdr)
    if magic != DUMP_MAGIC or ver != DUMP_VERSION or esz != ENTRY_DTYPE.itemsize:
        raise ValueError(f"{path}: not an mpsf fault-buffer dump (magic {magic!r}, version {ver})")
    off = _HDR.size
    entries = (np.memmap(path, dtype=ENTRY_DTYPE, mode="r", offset=off, shape=(n,)) if n
               else np.zeros(0, ENTRY_DTYPE))
    off += n * esz
    t_raise = None
    if flags & F_TRAISE:
        t_raise = np.memmap(path, dtype="<u8", mode="r", offset=off, shape=(n,)) if n else np.zeros(0, np.uint64)
        off += 8 * n
    with open(path, "rb") as f:
        f.seek(off)
        raw = f.read(nb)
    if len(raw) != nb:
        raise ValueError(f"{path}: truncated name table")
    names, pos = [], 0
    for _ in range(nch + ncl):
        (ln,) = struct.unpack_from("<H", raw, pos)
        names.append(raw[pos + 2:pos + 2 + ln].decode())
        pos += 2 + ln
    return Dump(entries, names[:nch], names[nch:], bool(flags & F_ISOLATION), base, t_drain, t_raise)
