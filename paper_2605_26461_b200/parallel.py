"""Sharded multi-GPU fault path: one process per GPU, torch.distributed.

A batch is split into contiguous entry ranges; rank r processes entries with global indices
``base_r .. base_r + n_r`` (``BatchParams.base_index``) against a replicated world.  Every
cross-entry dependency of the batch rules is a first-in-group minimum over the drain key,
a sum, or a max of flags, so the shards only need:

1. after pass 1 (``mpsf_scan``): all-reduce MIN of the dense group minima (fatal TSG
   teardowns, traps, first isolation per external range / guard page / client) and of the
   dedup slots, plus a sparse merge (all-gather + atomic-min insert) of the two wild-page
   hash tables.  Page-sized tables (dedup slots, first-eligible page keys) go dense only
   while small; beyond ``SPARSE_MIN_BYTES`` each rank compacts its non-empty words to
   (index, value) pairs, the ranks all-gather them and MIN-merge (SURVEY.md §8(e) round 1b:
   O(keys) bytes, not O(pages) -- 252 MB of dedup slots per batch on the config-3 world);
2. with isolation on, after the release-aware stage (``mpsf_general`` 1): MIN of the exact
   per-client mechanism minima and of the epoch-1 first-isolation slots, sparse NR merge;
   after stage 2 (only when m2 <= benign): MIN of the per-client M2 minima;
3. after ``mpsf_finalize``: SUM of the per-(client, scenario) counts.

Per-client fates come out identical on every rank; each rank's OutRecords, cancel list and
dedup set cover its own index range, so concatenating them in rank order reproduces the
single-GPU result bit for bit.  Collectives go through NCCL over NVLink on GPUs and gloo in
the CPU tests; unsigned MIN is done on signed views with the sign bit flipped.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import _lib
from .engine import BatchParams, DeviceBuffers, FaultEngine
from .errors import E_BAD_ENTRY, E_MISMATCH, E_NO_CHANNEL, E_OVERFLOW, E_VA, raise_for

# 4-byte MIN buffers larger than this are exchanged as compacted (index, value) pairs
# (MPSF_SPARSE_X=always|never overrides, for tests)
SPARSE_MIN_BYTES = 4 << 20

# entry errors in the priority mpsf_get_summary reports them (the device ORs the error bits of
# every bad entry and reports the highest-priority code with the smallest offending index)
_ERR_PRIO = {E_NO_CHANNEL: 4, E_BAD_ENTRY: 3, E_MISMATCH: 2, E_VA: 1}
_PRIO_ERR = {v: k for k, v in _ERR_PRIO.items()}
_ERR_MSG = {E_NO_CHANNEL: "fault entry channel has no client attribution",
            E_BAD_ENTRY: "malformed fault entry (engine/access/kind)",
            E_MISMATCH: "fault entry engine differs from its channel's engine",
            E_VA: "fault VA >= 2^53"}


def use_sparse(t) -> bool:
    mode = os.environ.get("MPSF_SPARSE_X", "auto")
    if mode == "always":
        return t.element_size() == 4
    if mode == "never":
        return False
    return t.element_size() == 4 and t.numel() * 4 > SPARSE_MIN_BYTES


def _dist():
    import torch.distributed as dist
    return dist


def allreduce_min_unsigned(t, group=None):
    """MIN over ranks of an unsigned array held in a signed (int32/int64) view, in place."""
    import torch
    dist = _dist()
    flip = torch.tensor(-(1 << 31) if t.dtype == torch.int32 else -(1 << 63), dtype=t.dtype, device=t.device)
    t.bitwise_xor_(flip)
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    t.bitwise_xor_(flip)


def allreduce_sum(t, group=None):
    dist = _dist()
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)


def allgather_ragged(keys, vals, group=None):
    """All-gather two aligned 1-D tensors of per-rank length; returns the concatenation."""
    import torch
    dist = _dist()
    ws = dist.get_world_size(group)
    cnt = torch.tensor([keys.numel()], dtype=torch.int64, device=keys.device)
    cnts = [torch.zeros_like(cnt) for _ in range(ws)]
    dist.all_gather(cnts, cnt, group=group)
    m = int(max(int(c.item()) for c in cnts))
    if m == 0:
        return keys[:0], vals[:0]
    kp = torch.full((m,), -1, dtype=keys.dtype, device=keys.device)
    vp = torch.full((m,), -1, dtype=vals.dtype, device=vals.device)
    kp[:keys.numel()] = keys
    vp[:vals.numel()] = vals
    ka = [torch.empty_like(kp) for _ in range(ws)]
    va = [torch.empty_like(vp) for _ in range(ws)]
    dist.all_gather(ka, kp, group=group)
    dist.all_gather(va, vp, group=group)
    ks = torch.cat([ka[r][:int(cnts[r].item())] for r in range(ws)])
    vs = torch.cat([va[r][:int(cnts[r].item())] for r in range(ws)])
    return ks, vs


class ShardedFaultPath:
    """Drives one shard through the phase API and the cross-rank exchanges."""

    def __init__(self, adapter, group=None):
        self.a = adapter
        self.group = group

    def _combine(self, stage):
        for t, op in self.a.exchange(stage):
            if op == "min" and use_sparse(t):
                idx, val = self.a.sparse_export(t)
                gi, gv = allgather_ragged(idx, val, self.group)
                self.a.sparse_merge(t, gi, gv)
            elif op == "min":
                allreduce_min_unsigned(t, self.group)
            else:
                allreduce_sum(t, self.group)

    def _merge_hash(self, which):
        keys, vals = self.a.hash_export(which)
        ks, vs = allgather_ragged(keys, vals, self.group)
        self.a.hash_merge(which, ks, vs)

    def _agree(self, status: int, error_index: int):
        """Every rank's batch status -> the one the whole batch has: the highest-priority entry
        error of any rank with the smallest global offending index (what one GPU reports), else
        overflow if any rank overflowed, else ok.  One MAX and one MIN all-reduce."""
        import torch
        dev = self.a.counts_tensor().device
        flags = torch.tensor([1 if status == E_OVERFLOW else 0, _ERR_PRIO.get(status, 0)], dtype=torch.int64,
                             device=dev)
        idx = torch.tensor([error_index if status in _ERR_PRIO else (1 << 62)], dtype=torch.int64, device=dev)
        if _dist().is_initialized():
            _dist().all_reduce(flags, op=_dist().ReduceOp.MAX, group=self.group)
        prio = int(flags[1].item())
        if prio:
            if _dist().is_initialized():     # the smallest bad entry of any kind on any rank
                _dist().all_reduce(idx, op=_dist().ReduceOp.MIN, group=self.group)
            return _PRIO_ERR[prio], int(idx.item())
        return (E_OVERFLOW if int(flags[0].item()) else 0), -1

    def process(self, params: BatchParams, max_attempts: int = 6, fetch: bool = True):
        """One sharded batch.  A wild-page hash table that fills up on any rank -- in its own
        inserts or in the merge of the other ranks' keys -- makes every rank run the batch
        again (the full tables have grown).  An entry error on any rank raises the same
        exception on every rank (no rank is left waiting in a collective).  ``fetch=False``
        leaves this shard's outputs in device memory (returns None)."""
        from .errors import HashOverflow
        for _ in range(max_attempts):
            self._once(params)
            status, eidx = self._agree(*self.a.status())
            if status == E_OVERFLOW:
                continue
            if status:
                raise_for(status, _ERR_MSG[status], eidx)
            return self.a.result() if fetch else None
        raise HashOverflow("wild-page hash tables kept overflowing")

    def _once(self, params: BatchParams):
        a = self.a
        a.scan(params)
        self._combine(1)
        self._merge_hash(0)
        self._merge_hash(1)
        a.resolve(params)
        if params.isolation:
            a.general(params, 1)
            self._combine(2)
            self._merge_hash(1)
            if params.m2_us <= params.benign_us:
                a.general(params, 2)
                self._combine(3)
            a.resolve2(params)
        a.finalize(params)
        allreduce_sum(a.counts_tensor(), self.group)


class LocalShardGroup:
    """The same phase sequence and exchanges as :class:`ShardedFaultPath`, but over several
    shards held by one process (e.g. several contexts on one device): the reductions are
    elementwise across the shards' buffers instead of collectives."""

    def __init__(self, adapters):
        self.ads = adapters

    def _combine(self, stage):
        import torch
        groups = list(zip(*[a.exchange(stage) for a in self.ads]))
        for bufs in groups:
            ts = [t for t, _ in bufs]
            op = bufs[0][1]
            if op == "min":
                flip = -(1 << 31) if ts[0].dtype == torch.int32 else -(1 << 63)
                acc = ts[0] ^ flip
                for t in ts[1:]:
                    acc = torch.minimum(acc, (t.to(acc.device)) ^ flip)
                acc = acc ^ flip
            else:
                acc = sum(t.to(ts[0].device) for t in ts)
            for t in ts:
                t.copy_(acc.to(t.device))

    def _merge_hash(self, which):
        import torch
        ex = [a.hash_export(which) for a in self.ads]
        ks = torch.cat([k.to(ex[0][0].device) for k, _ in ex])
        vs = torch.cat([v.to(ex[0][1].device) for _, v in ex])
        for a in self.ads:
            a.hash_merge(which, ks, vs)

    def process(self, params_list, max_attempts: int = 6):
        from .errors import HashOverflow
        for _ in range(max_attempts):
            self._once(params_list)
            st = [a.status() for a in self.ads]
            errs = [(_ERR_PRIO[c], i) for c, i in st if c in _ERR_PRIO]
            if errs:
                code = _PRIO_ERR[max(p for p, _ in errs)]
                raise_for(code, _ERR_MSG[code], min(i for _, i in errs))
            if any(c == E_OVERFLOW for c, _ in st):
                continue
            return [a.result() for a in self.ads]
        raise HashOverflow("wild-page hash tables kept overflowing")

    def _once(self, params_list):
        for a, p in zip(self.ads, params_list):
            a.scan(p)
        self._combine(1)
        self._merge_hash(0)
        self._merge_hash(1)
        p0 = params_list[0]
        for a, p in zip(self.ads, params_list):
            a.resolve(p)
        if p0.isolation:
            for a, p in zip(self.ads, params_list):
                a.general(p, 1)
            self._combine(2)
            self._merge_hash(1)
            if p0.m2_us <= p0.benign_us:
                for a, p in zip(self.ads, params_list):
                    a.general(p, 2)
                self._combine(3)
            for a, p in zip(self.ads, params_list):
                a.resolve2(p)
        for a, p in zip(self.ads, params_list):
            a.finalize(p)
        import torch
        tot = sum(a.counts_tensor().clone() for a in self.ads)
        for a in self.ads:
            a.counts_tensor().copy_(tot)


class _CAI:
    """Zero-copy torch view of device memory owned by libmpsf.so (CUDA array interface)."""

    def __init__(self, ptr, count, typestr):
        self.__cuda_array_interface__ = {"shape": (int(count),), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3}


def device_view(ptr, count, elem_bytes):
    import torch
    if not ptr or not count:
        return torch.empty(0, dtype=torch.int64 if elem_bytes == 8 else torch.int32, device="cuda")
    return torch.as_tensor(_CAI(ptr, count, "<i8" if elem_bytes == 8 else "<i4"), device="cuda")


class GpuShard:
    """Adapter: the GPU phase entry points of libmpsf.so for one rank's shard."""

    def __init__(self, eng: FaultEngine, d_in, n: int, bufs: DeviceBuffers):
        import torch
        self.eng, self.d_in, self.n, self.bufs = eng, d_in, n, bufs
        self.lib, self.ctx = eng.lib, eng.ctx
        self.stream = torch.cuda.current_stream()
        self.sp = C.c_void_p(self.stream.cuda_stream)
        cap = 1 << 20
        self.hk = torch.empty(cap, dtype=torch.int64, device="cuda")
        self.hv = torch.empty(cap, dtype=torch.int32, device="cuda")

    def _p(self, params):
        self.cp = params.to_c()
        return C.byref(self.cp)

    def scan(self, params):
        self.eng._check(self.lib.mpsf_scan(self.ctx, self.d_in.data_ptr(), self.n, self._p(params),
                                           self.bufs.counts.data_ptr(), self.sp))

    def exchange(self, stage):
        arr = (_lib.XBuf * 4)()
        k = self.lib.mpsf_exchange_buffers(self.ctx, stage, C.cast(arr, C.c_void_p), 4)
        self.eng._check(min(k, 0))
        return [(device_view(arr[i].ptr, arr[i].count, arr[i].elem_bytes), "min" if arr[i].op == 0 else "sum")
                for i in range(k)]

    def hash_export(self, which):
        while True:
            k = self.lib.mpsf_hash_export(self.ctx, which, self.hk.data_ptr(), self.hv.data_ptr(),
                                          self.hk.numel(), self.sp)
            if k >= 0:
                return self.hk[:k], self.hv[:k]
            import torch
            self.hk = torch.empty(self.hk.numel() * 4, dtype=torch.int64, device="cuda")
            self.hv = torch.empty(self.hv.numel() * 4, dtype=torch.int32, device="cuda")

    def hash_merge(self, which, keys, vals):
        keys, vals = keys.contiguous(), vals.contiguous()
        self.eng._check(self.lib.mpsf_hash_merge(self.ctx, which, keys.data_ptr(), vals.data_ptr(),
                                                 keys.numel(), self.sp))

    def sparse_export(self, t):
        """Non-empty words of a 4-byte MIN exchange buffer as (index, value) int32 tensors."""
        import torch
        cap = max(1 << 16, t.numel() // 8)
        while True:
            idx = torch.empty(cap, dtype=torch.int32, device=t.device)
            val = torch.empty(cap, dtype=torch.int32, device=t.device)
            k = self.lib.mpsf_sparse_export(self.ctx, t.data_ptr(), t.numel(), idx.data_ptr(), val.data_ptr(),
                                            cap, self.sp)
            if k >= 0:
                return idx[:k], val[:k]
            if k != E_OVERFLOW:
                self.eng._check(int(k))
            cap = t.numel()

    def sparse_merge(self, t, idx, val):
        idx, val = idx.contiguous(), val.contiguous()
        self.eng._check(self.lib.mpsf_sparse_merge(self.ctx, t.data_ptr(), t.numel(), idx.data_ptr(),
                                                   val.data_ptr(), idx.numel(), self.sp))

    def resolve(self, params):
        self.eng._check(self.lib.mpsf_resolve(self.ctx, self._p(params), self.bufs.verdict.data_ptr(),
                                              self.bufs.counts.data_ptr(), self.sp))

    def general(self, params, stage):
        self.eng._check(self.lib.mpsf_general(self.ctx, self.d_in.data_ptr(), self.n, self._p(params), stage,
                                              self.sp))

    def resolve2(self, params):
        self.eng._check(self.lib.mpsf_resolve2(self.ctx, self._p(params), self.sp))

    def finalize(self, params):
        b = self.bufs
        self.eng._check(self.lib.mpsf_finalize(self.ctx, self.d_in.data_ptr(), self.n, self._p(params),
                                               b.out.data_ptr(), b.dkeys.data_ptr(), b.didx.data_ptr(),
                                               b.cancel.data_ptr(), self.sp))

    def counts_tensor(self):
        from . import constants as K
        return self.bufs.counts[:8 * K.N_SCENARIOS * self.eng.world.n_clients].view(__import__("torch").int64)

    def status(self):
        """(status, global index of the first bad entry) of this shard's batch, not raised."""
        s = _lib.Summary()
        self.eng._check(self.lib.mpsf_get_summary(self.ctx, C.byref(s)))
        self._summary = s
        return int(s.status), int(s.error_index)

    def result(self):
        """The shard's results (after :meth:`status` reported the batch ok)."""
        s = self._summary
        return self.bufs.fetch(self.n, self.eng.world.n_clients, int(s.n_dedup), int(s.n_cancel), int(s.path))


# -- sharded batched translation (MemoryModel.resolve_va over a stream) --

class ShardedTranslate:
    """One rank's contiguous range of an access stream.  The only cross-access dependency of
    ``resolve_va`` over a stream is "did an earlier PREFETCH populate this page", so after
    phase 1 the ranks MIN-combine the first-PREFETCH page table (global indices) and each rank
    classifies its range; the concatenated per-rank results equal the single-GPU result."""

    def __init__(self, adapter, group=None):
        self.a = adapter
        self.group = group

    def translate(self):
        self.a.prefetch()
        for t, op in self.a.exchange(4):
            allreduce_min_unsigned(t, self.group)
        return self.a.finish()


class LocalTranslateGroup:
    """The same over several shards held by one process (elementwise MIN across buffers)."""

    def __init__(self, adapters):
        self.ads = adapters

    def translate(self):
        import torch
        for a in self.ads:
            a.prefetch()
        tabs = [a.exchange(4)[0][0] for a in self.ads]
        flip = -(1 << 31)
        acc = tabs[0] ^ flip
        for t in tabs[1:]:
            acc = torch.minimum(acc, t.to(acc.device) ^ flip)
        acc = acc ^ flip
        for t in tabs:
            t.copy_(acc.to(t.device))
        return [a.finish() for a in self.ads]


class GpuTranslateShard:
    """Adapter: ``mpsf_translate_prefetch`` / exchange stage 4 / ``mpsf_translate_finish`` for
    one shard (accesses ``d_acc[0:n]`` at global index ``base``)."""

    def __init__(self, eng: FaultEngine, d_acc, n: int, base: int):
        import torch
        self.eng, self.d_acc, self.n, self.base = eng, d_acc, n, base
        self.lib, self.ctx = eng.lib, eng.ctx
        self.sp = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        dev = d_acc.device
        self.hit = torch.empty(max(n, 1), dtype=torch.uint8, device=dev)
        self.faults = torch.empty(max(16 * n, 16), dtype=torch.uint8, device=dev)
        self.fi = torch.empty(max(4 * n, 4), dtype=torch.uint8, device=dev)
        self.pi = torch.empty(max(4 * n, 4), dtype=torch.uint8, device=dev)

    def prefetch(self):
        self.eng._check(self.lib.mpsf_translate_prefetch(self.ctx, self.d_acc.data_ptr(), self.n, self.base, self.sp))

    def exchange(self, stage):
        arr = (_lib.XBuf * 4)()
        k = self.lib.mpsf_exchange_buffers(self.ctx, stage, C.cast(arr, C.c_void_p), 4)
        self.eng._check(min(k, 0))
        return [(device_view(arr[i].ptr, arr[i].count, arr[i].elem_bytes), "min") for i in range(k)]

    def finish(self):
        self.eng._check(self.lib.mpsf_translate_finish(self.ctx, self.d_acc.data_ptr(), self.n, self.base,
                                                       self.hit.data_ptr(), self.faults.data_ptr(),
                                                       self.fi.data_ptr(), self.pi.data_ptr(), self.sp))
        s = self.eng.translate_summary()
        nm, npop = int(s.n_miss), int(s.n_populated)
        return dict(hit=self.hit[:self.n].cpu().numpy(), fault_idx=self.fi[:4 * nm].cpu().numpy().view(np.uint32),
                    pop_idx=self.pi[:4 * npop].cpu().numpy().view(np.uint32))


# -- sharded snapshot fold (StandbyInstance.fold over a consumed stream) --

def allgather_cat(t, group=None):
    """All-gather a 1-D tensor of per-rank length; returns the concatenation in rank order."""
    import torch
    dist = _dist()
    ws = dist.get_world_size(group)
    cnt = torch.tensor([t.numel()], dtype=torch.int64, device=t.device)
    cnts = [torch.zeros_like(cnt) for _ in range(ws)]
    dist.all_gather(cnts, cnt, group=group)
    sizes = [int(c.item()) for c in cnts]
    m = max(sizes)
    if m == 0:
        return t[:0]
    pad = torch.zeros(m, dtype=t.dtype, device=t.device)
    pad[:t.numel()] = t
    out = [torch.empty_like(pad) for _ in range(ws)]
    dist.all_gather(out, pad, group=group)
    return torch.cat([out[r][:sizes[r]] for r in range(ws)])


class ShardedFold:
    """Each rank folds a contiguous range of the consumed snapshot stream; the folds compose
    (fold(A ++ B) == fold(snapshots(fold(A)) ++ snapshots(fold(B))), one snapshot per folded
    request), so the ranks all-gather their folds as snapshots and fold once more.  Every
    rank ends with the whole stream's fold.  ``fold_fn(req, seq, nblk, ntok, progress, done,
    blocks, tokens, n_req_ids)`` returns an object with order / blk_off / blocks / tok_off /
    tokens / progress / done / last_seq (``FaultEngine.fold`` on GPUs, the oracle on CPU)."""

    def __init__(self, fold_fn, device=None, group=None):
        if device is None:      # the process group's own device (NCCL needs CUDA tensors)
            device = "cuda" if _dist().get_backend(group) == "nccl" else "cpu"
        self.fold_fn, self.device, self.group = fold_fn, device, group

    def fold(self, req, seq, nblk, ntok, progress, done, blocks, tokens, n_req_ids):
        import torch
        local = self.fold_fn(req, seq, nblk, ntok, progress, done, blocks, tokens, n_req_ids)
        r = len(local.order)
        cols = [np.asarray(local.order, np.uint32),
                (np.diff(local.blk_off) if r else np.zeros(0)).astype(np.uint32),
                (np.diff(local.tok_off) if r else np.zeros(0)).astype(np.uint32),
                np.asarray(local.progress, np.uint32), np.asarray(local.done, np.uint8).astype(np.uint32),
                np.asarray(local.blocks, np.uint32), np.asarray(local.tokens, np.uint32)]
        # int64 carriers (gloo and NCCL both gather them; values are < 2^32)
        g = [allgather_cat(torch.from_numpy(c.astype(np.int64)).to(self.device), self.group).cpu().numpy()
             for c in cols]
        # last_consumed_seq = the seq of the last consumed snapshot of the whole stream: the
        # last one of the highest rank that consumed any (recovery.py:83-92 advances it for every
        # snapshot, monotone or not)
        ws = _dist().get_world_size(self.group)
        mine = torch.tensor([_dist().get_rank(self.group) if len(req) else -1, int(local.last_seq) if len(req) else 0],
                            dtype=torch.int64, device=self.device)
        allp = [torch.zeros_like(mine) for _ in range(ws)]
        _dist().all_gather(allp, mine, group=self.group)
        owners = [(int(p[0].item()), int(p[1].item())) for p in allp if int(p[0].item()) >= 0]
        last_seq = max(owners)[1] if owners else 0
        m = len(g[0])
        merged = self.fold_fn(g[0].astype(np.uint32), np.zeros(m, np.uint64), g[1].astype(np.uint32),
                              g[2].astype(np.uint32), g[3].astype(np.uint32), g[4].astype(np.uint8),
                              g[5].astype(np.uint32), g[6].astype(np.uint32), n_req_ids)
        merged.last_seq = last_seq
        return merged
