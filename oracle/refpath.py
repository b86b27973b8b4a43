"""TEST INFRASTRUCTURE ONLY: locate and drive the reference package (``mpssim``) itself.

Used by the differential tests (via ``tests/refharness.py``) and by ``bench.py``'s reference
leg to time the reference's OWN per-entry path -- ``UvmHandler.channel_to_pid``
(pipeline.py:73,103) + ``faults.classify`` (faults.py:134-171, with ``MemoryModel.range_at``
memory.py:233-237) -- on the host cores (SURVEY.md §8(d) CPU baseline), and to check the
device's per-entry scenario / rid against it.  The product never imports this module.

Where the reference is looked for, in order: ``$MPSSIM_REF``; ``/root/reference/pkg/src`` (the
build container); ``baseline/_ref`` (the pip install ``tools/install_reference.sh`` makes,
which travels to the GPU box).  Its test suite: ``$MPSSIM_REF_TESTS``, the ``tests`` directory
beside the source tree, or ``baseline/_ref_tests``.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _find_src():
    env = os.environ.get("MPSSIM_REF")
    for cand in ([env] if env else []) + ["/root/reference/pkg/src", os.path.join(ROOT, "baseline", "_ref")]:
        if cand and os.path.isdir(os.path.join(cand, "mpssim")):
            return cand
    return env or "/root/reference/pkg/src"


def _find_tests(src):
    env = os.environ.get("MPSSIM_REF_TESTS")
    for cand in ([env] if env else []) + [os.path.join(os.path.dirname(src), "tests"),
                                          os.path.join(ROOT, "baseline", "_ref_tests")]:
        if cand and os.path.isdir(cand) and any(f.startswith("test_") for f in os.listdir(cand)):
            return cand
    return env or os.path.join(os.path.dirname(src), "tests")


REF_SRC = _find_src()
REF_TESTS = _find_tests(REF_SRC)


def reference_available() -> bool:
    return os.path.isdir(os.path.join(REF_SRC, "mpssim"))


def import_reference():
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import mpssim  # noqa: F401
    from mpssim import faults, machine, pipeline  # noqa: F401
    return mpssim


# -- the reference's own top-half classification, timed ------------------------------------

_W = None        # (reference World, seeds, pids) inherited by forked workers
ENGINES = ("sm", "ce", "pbdma")
ACCESSES = ("read", "write", "prefetch")


def _classify_slice(bounds):
    from mpssim import faults
    w, seeds, _ = _W
    lo, hi = bounds
    uvm, mem = w.uvm, w.mem
    t0 = time.perf_counter()
    out = []
    for s in seeds[lo:hi]:
        pid = uvm.channel_to_pid[s.channel_id]          # pipeline.py:103
        out.append(faults.classify(s, mem, pid).sid)     # pipeline.py:104
    return time.perf_counter() - t0, out


def reference_classify(n_clients: int, pages: int, world_seed: int, entries: np.ndarray, procs: int = 1):
    """Build the synthetic world through the reference's own allocation APIs
    (``tests/refharness.build_reference_world`` recipe), then run its per-entry
    ``channel_to_pid`` + ``classify`` over the translation entries of ``entries``, on one core
    and on ``procs`` forked workers.  Returns dict(n, t1, tN, sids, mask)."""
    global _W
    import multiprocessing as mp
    import_reference()
    from mpssim.execmodel import EngineClass
    from mpssim.memory import AccessType, FaultSeed
    from tests import refharness as H

    flat_names = [f"c{c + 1}.{e}" for c in range(n_clients) for e in ENGINES]
    w = H.build_reference_world(H.synthetic_spec(n_clients, pages, world_seed))
    mask = entries["kind"] == 0
    tr = entries[mask]
    seeds = [FaultSeed(va=int(e["va"]), access=AccessType(ACCESSES[int(e["access"])]),
                       engine=EngineClass(ENGINES[int(e["engine"])]), channel_id=flat_names[int(e["channel"])])
             for e in tr]
    _W = (w, seeds, flat_names)
    t1, sids = _classify_slice((0, len(seeds)))
    tN = None
    if procs > 1:
        cuts = [len(seeds) * k // procs for k in range(procs + 1)]
        ctx = mp.get_context("fork")
        t0 = time.perf_counter()
        with ctx.Pool(procs) as pool:
            parts = pool.map(_classify_slice, list(zip(cuts[:-1], cuts[1:])))
        tN = time.perf_counter() - t0
        assert sum((p[1] for p in parts), []) == sids
    _W = None
    return dict(n=len(seeds), t1=t1, tN=tN, sids=sids, mask=mask)
