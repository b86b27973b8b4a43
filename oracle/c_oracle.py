"""ctypes wrapper of oracle/libmpsf_oracle.so -- TEST INFRASTRUCTURE ONLY (checker and
CPU baseline).  Same results as seq_oracle.process_batch, ~1000x faster; built by
``__graft_entry__.build()`` / ``make -C oracle``."""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_2605_26461_b200 import constants as K
from paper_2605_26461_b200.world import OUT_DTYPE, VERDICT_DTYPE, FlatWorld

from .seq_oracle import BatchResult, OracleError, Params

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "libmpsf_oracle.so")
_lib = None


def build() -> str:
    root = os.path.dirname(HERE)
    subprocess.run(["gcc", "-O3", "-march=x86-64-v3", "-fPIC", "-shared", "-pthread", "-I",
                    os.path.join(root, "include"), "-o", LIB, os.path.join(HERE, "mpsf_oracle.c")],
                   check=True)
    return LIB


def load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(os.path.join(HERE, "mpsf_oracle.c")):
            build()
        lib = C.CDLL(LIB)
        vp = C.c_void_p
        lib.oracle_process.restype = C.c_int
        lib.oracle_process.argtypes = [vp, C.c_uint32, vp, C.c_uint64, vp, C.c_uint32, vp, C.c_uint32,
                                       C.c_uint32, vp, C.c_uint64, vp, C.c_int, vp, vp, vp, vp, vp,
                                       vp, vp, vp, vp]
        _lib = lib
    return _lib


class _P(C.Structure):
    _fields_ = [("flags", C.c_uint32), ("benign_us", C.c_uint32), ("m1_us", C.c_uint32),
                ("m2_us", C.c_uint32), ("m3_us", C.c_uint32), ("reserved", C.c_uint32),
                ("base_index", C.c_uint64)]


def process_batch(w: FlatWorld, entries: np.ndarray, params: Params | None = None,
                  base_index: int = 0, threads: int = 1) -> BatchResult:
    params = params or Params()
    lib = load()
    n = len(entries)
    Cn = w.n_clients
    entries = np.ascontiguousarray(entries)
    r = np.ascontiguousarray(w.ranges)
    ps = np.ascontiguousarray(w.page_state)
    ch = np.ascontiguousarray(w.channels)
    cl = np.ascontiguousarray(w.clients)
    out = np.empty(max(n, 1), OUT_DTYPE)
    verdict = np.empty(max(Cn, 1), VERDICT_DTYPE)
    counts = np.zeros((max(Cn, 1), K.N_SCENARIOS), np.uint64)
    dk = np.empty(max(n, 1), np.uint64)
    di = np.empty(max(n, 1), np.uint32)
    ca = np.empty(max(n, 1), np.uint32)
    nd = C.c_uint64()
    nc = C.c_uint64()
    ei = C.c_uint64()
    p = _P(K.PF_ISOLATION if params.isolation else 0, params.benign_us, params.m1_us,
           params.m2_us, params.m3_us, 0, base_index)
    rc = lib.oracle_process(r.ctypes.data, len(r), ps.ctypes.data, len(ps), ch.ctypes.data, len(ch),
                            cl.ctypes.data, len(cl), int(w.world_flags), entries.ctypes.data, n,
                            C.addressof(p), threads, out.ctypes.data, verdict.ctypes.data,
                            counts.ctypes.data, dk.ctypes.data, di.ctypes.data, C.addressof(nd),
                            ca.ctypes.data, C.addressof(nc), C.addressof(ei))
    if rc:
        raise OracleError(rc, f"oracle error {rc} at entry {ei.value}")
    return BatchResult(out[:n], verdict[:Cn], counts[:Cn], dk[:nd.value], di[:nd.value], ca[:nc.value])
