"""Host side of the batched fault path: owns one ``mpsf_ctx`` (device world tables +
scratch) and drives libmpsf.so.  Device memory is allocated as torch tensors (torch is
the plumbing: allocator + streams); the compute is the sm_100a kernels behind the C ABI.

Two call forms, matching ``include/mpsf.h``:

* :meth:`FaultEngine.process_device` -- entries already in HBM, async on a stream (the
  device-resident throughput the bench reports as ``value``);
* :meth:`FaultEngine.process` -- numpy host buffers in, numpy results out, every copy
  included (``mpsf_process_host``; the bench's ``e2e``).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib
from . import constants as K
from .errors import HashOverflow, raise_for
from .world import (ENTRY_DTYPE, OUT_DTYPE, REMAP_DTYPE, VERDICT_DTYPE, FlatWorld)


@dataclass
class BatchParams:
    """``uvm.isolation_enabled`` plus the ``SimParams`` latencies (kernel.py:34-37)."""

    isolation: bool = True
    benign_us: int = 226
    m1_us: int = 131
    m2_us: int = 2780
    m3_us: int = 1700
    base_index: int = 0

    @classmethod
    def from_sim_params(cls, params, isolation: bool) -> "BatchParams":
        return cls(isolation=isolation, benign_us=params.benign_service_us,
                   m1_us=params.m1_latency_us, m2_us=params.m2_latency_us,
                   m3_us=params.m3_latency_us)

    def to_c(self) -> _lib.Params:
        return _lib.Params(K.PF_ISOLATION if self.isolation else 0, self.benign_us, self.m1_us,
                           self.m2_us, self.m3_us, 0, self.base_index)


@dataclass
class BatchResult:
    out: np.ndarray          # OUT_DTYPE[n]
    verdict: np.ndarray      # VERDICT_DTYPE[C]
    counts: np.ndarray       # uint64[C, 28]
    dedup_keys: np.ndarray   # uint64[U]
    dedup_idx: np.ndarray    # uint32[U]
    cancel: np.ndarray       # uint32[C]
    path: int = 0


class DeviceBuffers:
    """Output buffers in HBM for batches of up to ``n`` entries."""

    def __init__(self, n: int, n_clients: int, device: int = 0):
        import torch
        dev = torch.device("cuda", device)
        self.n = n
        self.out = torch.empty(max(8 * n, 8), dtype=torch.uint8, device=dev)
        self.verdict = torch.empty(max(4 * n_clients, 4), dtype=torch.uint8, device=dev)
        self.counts = torch.empty(max(8 * K.N_SCENARIOS * n_clients, 8), dtype=torch.uint8, device=dev)
        self.dkeys = torch.empty(max(8 * n, 8), dtype=torch.uint8, device=dev)
        self.didx = torch.empty(max(4 * n, 4), dtype=torch.uint8, device=dev)
        self.cancel = torch.empty(max(4 * n, 4), dtype=torch.uint8, device=dev)

    def fetch(self, n: int, n_clients: int, n_dedup: int, n_cancel: int, path: int = 0) -> BatchResult:
        out = self.out[:8 * n].cpu().numpy().view(OUT_DTYPE)
        verdict = self.verdict[:4 * n_clients].cpu().numpy().view(VERDICT_DTYPE)
        counts = self.counts[:8 * K.N_SCENARIOS * n_clients].cpu().numpy().view(np.uint64)
        counts = counts.reshape(n_clients, K.N_SCENARIOS)
        dk = self.dkeys[:8 * n_dedup].cpu().numpy().view(np.uint64)
        di = self.didx[:4 * n_dedup].cpu().numpy().view(np.uint32)
        ca = self.cancel[:4 * n_cancel].cpu().numpy().view(np.uint32)
        return BatchResult(out, verdict, counts, dk, di, ca, path)


class FaultEngine:
    """One device context of the fault path (``mpsf_ctx``)."""

    def __init__(self, device: int = 0):
        self.lib = _lib.load()
        self.device = device
        h = C.c_void_p()
        rc = self.lib.mpsf_create(C.byref(h), device)
        self._check(rc)
        self.ctx = h
        self.world: Optional[FlatWorld] = None

    def close(self) -> None:
        if getattr(self, "ctx", None):
            self.lib.mpsf_destroy(self.ctx)
            self.ctx = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc: int, index: int = -1) -> None:
        if rc:
            raise_for(rc, self.lib.mpsf_strerror(rc).decode(), index)

    # -- world ---------------------------------------------------------------------------
    def set_dense_dedup(self, on: bool = True) -> None:
        """One dedup slot per (page, group) regardless of world size.  Call before upload."""
        self.set_dedup_layout("dense" if on else "auto")

    def set_dedup_layout(self, layout: str = "auto") -> None:
        """Dedup-slot layout of the next upload: "dense" (one slot per (page, group)),
        "sparse" (one claimed slot per page, other groups through the hash table, no per-page
        first-eligible keys -- what worlds over ~3.3 M pages get), or "auto" (by size)."""
        mode = {"auto": 0, "dense": 1, "sparse": -1}[layout]
        self._check(self.lib.mpsf_set_dense_dedup(self.ctx, mode))

    def upload_world(self, w: FlatWorld) -> None:
        """``mpsf_upload_world``: the interval table, page states, channels, clients."""
        r = np.ascontiguousarray(w.ranges)
        ps = np.ascontiguousarray(w.page_state)
        ch = np.ascontiguousarray(w.channels)
        cl = np.ascontiguousarray(w.clients)
        rc = self.lib.mpsf_upload_world(self.ctx, r.ctypes.data, len(r), ps.ctypes.data, len(ps),
                                        ch.ctypes.data, len(ch), cl.ctypes.data, len(cl),
                                        int(w.world_flags))
        self._check(rc)
        self.world = w

    # -- device-resident form ---------------------------------------------------------------
    def process_device(self, d_entries, n: int, params: BatchParams, bufs: DeviceBuffers,
                       stream=None) -> None:
        """Enqueue one batch on ``stream`` (torch stream or None = current)."""
        import torch
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        p = params.to_c()
        rc = self.lib.mpsf_process(self.ctx, d_entries.data_ptr(), n, C.byref(p),
                                   bufs.out.data_ptr(), bufs.verdict.data_ptr(),
                                   bufs.counts.data_ptr(), bufs.dkeys.data_ptr(),
                                   bufs.didx.data_ptr(), bufs.cancel.data_ptr(),
                                   C.c_void_p(stream.cuda_stream))
        self._check(rc)

    def summary(self) -> _lib.Summary:
        s = _lib.Summary()
        self._check(self.lib.mpsf_get_summary(self.ctx, C.byref(s)))
        if s.status:
            raise_for(s.status, self.lib.mpsf_strerror(s.status).decode(), int(s.error_index))
        return s

    def process_resident(self, d_entries, n: int, params: BatchParams,
                         bufs: DeviceBuffers) -> BatchResult:
        """Device-resident call with the overflow retry, results fetched to numpy."""
        for _ in range(4):
            self.process_device(d_entries, n, params, bufs)
            try:
                s = self.summary()
            except HashOverflow:
                continue
            return bufs.fetch(n, self.world.n_clients, int(s.n_dedup), int(s.n_cancel), int(s.path))
        raise HashOverflow("wild-page hash table kept overflowing")

    def last_launches(self) -> int:
        return int(self.lib.mpsf_last_launches(self.ctx))

    def set_profiling(self, on: bool) -> None:
        self._check(self.lib.mpsf_set_profiling(self.ctx, 1 if on else 0))

    def profile(self) -> dict:
        """{kernel name: (launches, total ms)} since profiling was enabled (waits)."""
        arr = (_lib.KernelTime * 32)()
        k = self.lib.mpsf_get_profile(self.ctx, C.cast(arr, C.c_void_p), 32)
        if k < 0:
            self._check(k)
        return {arr[i].name.decode(): (int(arr[i].launches), float(arr[i].total_ms)) for i in range(k)}

    # -- host-buffer form (end to end) ---------------------------------------------------------
    def process(self, entries: np.ndarray, params: BatchParams, out_bufs: Optional[dict] = None) -> BatchResult:
        """``mpsf_process_host``: host entries in, host results out (H2D + D2H inside)."""
        entries = np.ascontiguousarray(entries, dtype=ENTRY_DTYPE)
        n = len(entries)
        Cn = self.world.n_clients
        if out_bufs is None:
            out_bufs = alloc_host_outputs(n, Cn)
        p = params.to_c()
        s = _lib.Summary()
        rc = self.lib.mpsf_process_host(self.ctx, entries.ctypes.data, n, C.byref(p),
                                        out_bufs["out"].ctypes.data, out_bufs["verdict"].ctypes.data,
                                        out_bufs["counts"].ctypes.data, out_bufs["dkeys"].ctypes.data,
                                        out_bufs["didx"].ctypes.data, out_bufs["cancel"].ctypes.data,
                                        C.byref(s))
        self._check(rc)
        if s.status:
            raise_for(s.status, self.lib.mpsf_strerror(s.status).decode(), int(s.error_index))
        return BatchResult(out_bufs["out"][:n], out_bufs["verdict"][:Cn],
                           out_bufs["counts"][:Cn], out_bufs["dkeys"][:s.n_dedup],
                           out_bufs["didx"][:s.n_dedup], out_bufs["cancel"][:s.n_cancel], int(s.path))

    # -- batched top half (faults.classify + range_at per entry) ------------------------------
    def classify(self, entries: np.ndarray, base_index: int = 0):
        """``mpsf_classify``: (scenario id u8[n] -- 0xFF skipped --, rid u32[n] -- 0xFFFFFFFF
        none) of every entry, as ``raise_mmu_fault`` classifies it (pipeline.py:103-104)."""
        import torch
        entries = np.ascontiguousarray(entries, dtype=ENTRY_DTYPE)
        n = len(entries)
        dev = torch.device("cuda", self.device)
        d_in = torch.from_numpy(entries.view(np.uint8).copy() if n else np.zeros(16, np.uint8)).to(dev)
        d_s = torch.empty(max(n, 2), dtype=torch.uint8, device=dev)
        d_r = torch.empty(max(4 * n, 8), dtype=torch.uint8, device=dev)
        stream = torch.cuda.current_stream(self.device)
        self._check(self.lib.mpsf_classify(self.ctx, d_in.data_ptr(), n, base_index, d_s.data_ptr(), d_r.data_ptr(),
                                           C.c_void_p(stream.cuda_stream)))
        self.summary()
        return d_s[:n].cpu().numpy(), d_r[:4 * n].cpu().numpy().view(np.uint32)

    # -- batched translation (resolve_va over an access stream) -------------------------------
    def translate_device(self, d_acc, n: int, d_hit, d_faults, d_fault_idx, d_pop_idx, base_index: int = 0,
                         stream=None) -> None:
        """``mpsf_translate`` on device buffers (torch tensors); see :meth:`translate_summary`."""
        import torch
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        rc = self.lib.mpsf_translate(self.ctx, d_acc.data_ptr(), n, base_index, d_hit.data_ptr(),
                                     d_faults.data_ptr(), d_fault_idx.data_ptr(), d_pop_idx.data_ptr(),
                                     C.c_void_p(stream.cuda_stream))
        self._check(rc)

    def translate_summary(self) -> _lib.TranslateSummary:
        s = _lib.TranslateSummary()
        self._check(self.lib.mpsf_get_translate_summary(self.ctx, C.byref(s)))
        if s.status:
            raise_for(s.status, self.lib.mpsf_strerror(s.status).decode(), int(s.error_index))
        return s

    def translate(self, accesses: np.ndarray, base_index: int = 0):
        """Host form: returns (hit u8[n], fault entries in order, their indices, populating
        prefetch indices) -- the outputs of ``MemoryModel.resolve_va`` per access."""
        import torch
        accesses = np.ascontiguousarray(accesses, dtype=ENTRY_DTYPE)
        n = len(accesses)
        dev = torch.device("cuda", self.device)
        raw = accesses.view(np.uint8) if n else np.zeros(16, np.uint8)
        d_acc = torch.from_numpy(raw.copy()).to(dev)
        d_hit = torch.empty(max(n, 1), dtype=torch.uint8, device=dev)
        d_faults = torch.empty(max(16 * n, 16), dtype=torch.uint8, device=dev)
        d_fi = torch.empty(max(4 * n, 4), dtype=torch.uint8, device=dev)
        d_pi = torch.empty(max(4 * n, 4), dtype=torch.uint8, device=dev)
        self.translate_device(d_acc, n, d_hit, d_faults, d_fi, d_pi, base_index)
        s = self.translate_summary()
        nm, npop = int(s.n_miss), int(s.n_populated)
        hit = d_hit[:n].cpu().numpy()
        faults = d_faults[:16 * nm].cpu().numpy().view(ENTRY_DTYPE)
        fi = d_fi[:4 * nm].cpu().numpy().view(np.uint32)
        pi = d_pi[:4 * npop].cpu().numpy().view(np.uint32)
        return hit, faults, fi, pi

    # -- asynchronous host-buffer form (two slots, pipelined batches) -------------------------
    def submit(self, entries: np.ndarray, params: BatchParams, out_bufs: dict, slot: int) -> None:
        """``mpsf_submit_host``: enqueue one batch into slot 0/1 and return.  ``entries`` and
        ``out_bufs`` (``alloc_host_outputs``; pinned for device-written lists) must stay alive
        until :meth:`collect`."""
        entries = np.ascontiguousarray(entries, dtype=ENTRY_DTYPE)
        p = params.to_c()
        rc = self.lib.mpsf_submit_host(self.ctx, slot, entries.ctypes.data, len(entries), C.byref(p),
                                       out_bufs["out"].ctypes.data, out_bufs["verdict"].ctypes.data,
                                       out_bufs["counts"].ctypes.data, out_bufs["dkeys"].ctypes.data,
                                       out_bufs["didx"].ctypes.data, out_bufs["cancel"].ctypes.data)
        self._check(rc)
        if not hasattr(self, "_inflight"):
            self._inflight = {}
        self._inflight[slot] = (entries, out_bufs, len(entries))

    def collect(self, slot: int) -> BatchResult:
        """``mpsf_collect_host``: wait for slot ``slot`` and return its results."""
        entries, out_bufs, n = self._inflight.pop(slot)
        s = _lib.Summary()
        self._check(self.lib.mpsf_collect_host(self.ctx, slot, C.byref(s)))
        if s.status:
            raise_for(s.status, self.lib.mpsf_strerror(s.status).decode(), int(s.error_index))
        Cn = self.world.n_clients
        del entries
        return BatchResult(out_bufs["out"][:n], out_bufs["verdict"][:Cn], out_bufs["counts"][:Cn],
                           out_bufs["dkeys"][:s.n_dedup], out_bufs["didx"][:s.n_dedup],
                           out_bufs["cancel"][:s.n_cancel], int(s.path))

    # -- recovery remap -------------------------------------------------------------------------
    def remap_device(self, va_base: int, d_phys, npages4k: int, gran_log2: int, d_out, stream=None) -> None:
        import torch
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        self._check(self.lib.mpsf_remap(self.ctx, va_base, d_phys.data_ptr(), npages4k, gran_log2,
                                        d_out.data_ptr(), C.c_void_p(stream.cuda_stream)))

    def remap(self, va_base: int, phys_pages: np.ndarray, gran_log2: int = 12) -> np.ndarray:
        """``vmm_map``-equivalent remap table of one shared allocation (numpy in/out)."""
        import torch
        phys = np.ascontiguousarray(phys_pages, dtype=np.uint64)
        step = 1 << (gran_log2 - K.PAGE_SHIFT)
        e = -(-len(phys) // step)
        d_phys = torch.from_numpy(phys.view(np.int64)).to(f"cuda:{self.device}")
        d_out = torch.empty(max(16 * e, 16), dtype=torch.uint8, device=f"cuda:{self.device}")
        self.remap_device(va_base, d_phys, len(phys), gran_log2, d_out)
        torch.cuda.synchronize(self.device)
        return d_out[:16 * e].cpu().numpy().view(REMAP_DTYPE)

    def remap_blocks(self, va_base: int, phys_pages: np.ndarray, block_ids) -> np.ndarray:
        import torch
        phys = np.ascontiguousarray(phys_pages, dtype=np.uint64)
        blocks = np.ascontiguousarray(block_ids, dtype=np.uint32)
        d_phys = torch.from_numpy(phys.view(np.int64)).to(f"cuda:{self.device}")
        d_b = torch.from_numpy(blocks.view(np.int32)).to(f"cuda:{self.device}")
        d_out = torch.empty(max(16 * len(blocks), 16), dtype=torch.uint8, device=f"cuda:{self.device}")
        stream = torch.cuda.current_stream(self.device)
        self._check(self.lib.mpsf_remap_blocks(self.ctx, va_base, d_phys.data_ptr(), len(phys),
                                               d_b.data_ptr(), len(blocks), d_out.data_ptr(),
                                               C.c_void_p(stream.cuda_stream)))
        return d_out[:16 * len(blocks)].cpu().numpy().view(REMAP_DTYPE)

    # -- snapshot delta fold (StandbyInstance.fold, recovery.py:83-92) -------------------------
    def fold_device(self, n_snap: int, n_req_ids: int, d_req, d_nblk, d_ntok, d_progress, d_done, d_blocks,
                    n_blocks: int, d_tokens, n_tokens: int, out: dict, stream=None) -> _lib.FoldSummary:
        """``mpsf_fold`` on device tensors; ``out`` holds ``alloc_fold_outputs`` tensors."""
        import torch
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        s = _lib.FoldSummary()
        rc = self.lib.mpsf_fold(self.ctx, n_snap, n_req_ids, d_req.data_ptr(), d_nblk.data_ptr(),
                                d_ntok.data_ptr(), d_progress.data_ptr(), d_done.data_ptr(), d_blocks.data_ptr(),
                                n_blocks, d_tokens.data_ptr(), n_tokens, out["order"].data_ptr(), out["blk_off"].data_ptr(),
                                out["blocks"].data_ptr(), out["tok_off"].data_ptr(), out["tokens"].data_ptr(),
                                out["progress"].data_ptr(), out["done"].data_ptr(), C.byref(s),
                                C.c_void_p(stream.cuda_stream))
        if rc:
            raise_for(rc, self.lib.mpsf_strerror(rc).decode(), int(s.error_index))
        return s

    def fold(self, req, seq, nblk, ntok, progress, done, blocks, tokens, n_req_ids: int | None = None) -> "Folded":
        """Host form: the fold of ``len(req)`` consumed snapshots (SoA, consume order; request id
        0xFFFFFFFF = liveness-only).  Returns :class:`Folded` (requests in first-appearance
        order, CSR deltas, last progress, sticky done, last consumed seq)."""
        import torch
        dev = torch.device("cuda", self.device)
        req = np.ascontiguousarray(req, dtype=np.uint32)
        S = len(req)
        if n_req_ids is None:
            live = req[req != 0xFFFFFFFF]
            n_req_ids = int(live.max()) + 1 if len(live) else 1

        def up(a, dt):
            a = np.ascontiguousarray(a, dtype=dt)
            return torch.from_numpy(a.view(np.uint8).copy() if len(a) else np.zeros(4, np.uint8)).to(dev)
        d = [up(req, np.uint32), up(nblk, np.uint32), up(ntok, np.uint32), up(progress, np.uint32),
             up(done, np.uint8), up(blocks, np.uint32), up(tokens, np.uint32)]
        out = alloc_fold_outputs(S, len(blocks), len(tokens), self.device)
        s = self.fold_device(S, n_req_ids, *d[:6], len(blocks), d[6], len(tokens), out)
        r, nb, nt = int(s.n_requests), int(s.n_blocks), int(s.n_tokens)
        u32 = lambda t, k: t[:4 * k].cpu().numpy().view(np.uint32)  # noqa: E731
        u64 = lambda t, k: t[:8 * k].cpu().numpy().view(np.uint64)  # noqa: E731
        return Folded(order=u32(out["order"], r), blk_off=u64(out["blk_off"], r + 1) if r else np.zeros(1, np.uint64),
                      blocks=u32(out["blocks"], nb), tok_off=u64(out["tok_off"], r + 1) if r else np.zeros(1, np.uint64),
                      tokens=u32(out["tokens"], nt), progress=u32(out["progress"], r),
                      done=out["done"][:r].cpu().numpy().copy(), last_seq=int(seq[-1]) if S else 0)

    def kv_reserve_device(self, total_blocks: int, d_blocks, n: int, d_reserved, d_free, stream=None) -> int:
        """``mpsf_kv_reserve`` on device tensors; returns the number of free ids."""
        import torch
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        nf = C.c_uint64(0)
        self._check(self.lib.mpsf_kv_reserve(self.ctx, total_blocks, d_blocks.data_ptr() if n else None, n,
                                             d_reserved.data_ptr(), d_free.data_ptr(), C.byref(nf),
                                             C.c_void_p(stream.cuda_stream)))
        return int(nf.value)

    def kv_reserve(self, total_blocks: int, block_ids):
        """``BlockPool(total_blocks).reserve(block_ids)``: (reserved mask u8[total], free ids
        ascending -- the pool's pop order)."""
        import torch
        dev = torch.device("cuda", self.device)
        ids = np.ascontiguousarray(block_ids, dtype=np.uint32)
        d_b = torch.from_numpy(ids.view(np.uint8).copy() if len(ids) else np.zeros(4, np.uint8)).to(dev)
        d_r = torch.empty(max(total_blocks, 1), dtype=torch.uint8, device=dev)
        d_f = torch.empty(max(4 * total_blocks, 4), dtype=torch.uint8, device=dev)
        nf = self.kv_reserve_device(total_blocks, d_b, len(ids), d_r, d_f)
        return d_r[:total_blocks].cpu().numpy(), d_f[:4 * nf].cpu().numpy().view(np.uint32)


@dataclass
class Folded:
    """Result of :meth:`FaultEngine.fold` -- ``StandbyInstance`` state after ``fold``: the
    ``folded`` dict as CSR (rows in insertion order) plus ``last_consumed_seq``."""
    order: np.ndarray
    blk_off: np.ndarray
    blocks: np.ndarray
    tok_off: np.ndarray
    tokens: np.ndarray
    progress: np.ndarray
    done: np.ndarray
    last_seq: int


def alloc_fold_outputs(n_snap: int, n_blocks: int, n_tokens: int, device: int = 0) -> dict:
    """Device output tensors (raw bytes) for ``FaultEngine.fold_device``."""
    import torch
    dev = torch.device("cuda", device)
    b = lambda n: torch.empty(max(n, 8), dtype=torch.uint8, device=dev)  # noqa: E731
    return dict(order=b(4 * n_snap), blk_off=b(8 * (n_snap + 1)), blocks=b(4 * n_blocks),
                tok_off=b(8 * (n_snap + 1)), tokens=b(4 * n_tokens), progress=b(4 * n_snap), done=b(n_snap))


def alloc_host_outputs(n: int, n_clients: int, pinned: bool = False) -> dict:
    """Host result buffers for ``FaultEngine.process`` (optionally page-locked)."""
    def buf(count, dtype):
        if pinned:
            import torch
            t = torch.empty(max(count * np.dtype(dtype).itemsize, 1), dtype=torch.uint8).pin_memory()
            return t.numpy().view(dtype)[:count]
        return np.empty(count, dtype)
    return dict(out=buf(n, OUT_DTYPE), verdict=buf(n_clients, VERDICT_DTYPE),
                counts=buf(n_clients * K.N_SCENARIOS, np.uint64).reshape(n_clients, K.N_SCENARIOS),
                dkeys=buf(n, np.uint64), didx=buf(n, np.uint32), cancel=buf(n, np.uint32))
