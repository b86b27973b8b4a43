"""ctypes binding of libmpsf.so (include/mpsf.h).  Fails loudly: there is no CPU path."""

from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MPSF_LIB", os.path.join(_HERE, "libmpsf.so"))


class FaultEntry(C.Structure):
    _fields_ = [("va", C.c_uint64), ("channel", C.c_uint32), ("engine", C.c_uint8),
                ("access", C.c_uint8), ("kind", C.c_uint8), ("flags", C.c_uint8)]


class RangeEntry(C.Structure):
    _fields_ = [("base", C.c_uint64), ("end", C.c_uint64), ("client", C.c_uint32),
                ("page_off", C.c_uint32), ("kind", C.c_uint8), ("lifecycle", C.c_uint8),
                ("migratable", C.c_uint8), ("state", C.c_uint8), ("rid", C.c_uint32)]


class ChannelEntry(C.Structure):
    _fields_ = [("client", C.c_uint32), ("engine", C.c_uint8), ("pad", C.c_uint8 * 3)]


class ClientEntry(C.Structure):
    _fields_ = [("mode", C.c_uint8), ("flags", C.c_uint8), ("pad", C.c_uint16)]


class OutRecord(C.Structure):
    _fields_ = [("rid", C.c_uint32), ("scenario", C.c_uint8), ("verdict", C.c_uint8),
                ("client", C.c_uint16)]


class ClientVerdict(C.Structure):
    _fields_ = [("state", C.c_uint8), ("reason", C.c_uint8), ("notifier", C.c_uint8),
                ("flags", C.c_uint8)]


class RemapEntry(C.Structure):
    _fields_ = [("va", C.c_uint64), ("phys", C.c_uint64)]


class Params(C.Structure):
    _fields_ = [("flags", C.c_uint32), ("benign_us", C.c_uint32), ("m1_us", C.c_uint32),
                ("m2_us", C.c_uint32), ("m3_us", C.c_uint32), ("reserved", C.c_uint32),
                ("base_index", C.c_uint64)]


class Summary(C.Structure):
    _fields_ = [("status", C.c_int32), ("path", C.c_uint32), ("n_dedup", C.c_uint64),
                ("n_cancel", C.c_uint64), ("error_index", C.c_uint64), ("hash_used", C.c_uint64)]


class FoldSummary(C.Structure):
    _fields_ = [("status", C.c_int32), ("pad", C.c_uint32), ("n_requests", C.c_uint64),
                ("n_blocks", C.c_uint64), ("n_tokens", C.c_uint64), ("error_index", C.c_uint64)]


class RenderParams(C.Structure):
    _fields_ = [("t_drain", C.c_uint64), ("t_raise", C.c_void_p), ("m1_us", C.c_uint32), ("m2_us", C.c_uint32),
                ("m3_us", C.c_uint32), ("parts", C.c_uint32), ("channel_names", C.POINTER(C.c_char_p)),
                ("n_channels", C.c_uint32), ("n_clients", C.c_uint32), ("client_names", C.POINTER(C.c_char_p)),
                ("threads", C.c_uint32), ("pad", C.c_uint32)]


class TranslateSummary(C.Structure):
    _fields_ = [("status", C.c_int32), ("pad", C.c_uint32), ("n_miss", C.c_uint64),
                ("n_populated", C.c_uint64), ("error_index", C.c_uint64)]


SIGNATURES = {
    "mpsf_version": (C.c_int, []),
    "mpsf_strerror": (C.c_char_p, [C.c_int]),
    "mpsf_create": (C.c_int, [C.POINTER(C.c_void_p), C.c_int]),
    "mpsf_destroy": (None, [C.c_void_p]),
    "mpsf_upload_world": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint64,
                                    C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint32, C.c_uint32]),
    "mpsf_process": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.POINTER(Params), C.c_void_p,
                               C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                               C.c_void_p]),
    "mpsf_get_summary": (C.c_int, [C.c_void_p, C.POINTER(Summary)]),
    "mpsf_process_host": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.POINTER(Params),
                                    C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                    C.c_void_p, C.POINTER(Summary)]),
    "mpsf_submit_host": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_uint64, C.POINTER(Params), C.c_void_p,
                                   C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "mpsf_collect_host": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(Summary)]),
    "mpsf_translate": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p, C.c_void_p,
                                 C.c_void_p, C.c_void_p, C.c_void_p]),
    "mpsf_translate_prefetch": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p]),
    "mpsf_translate_finish": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p, C.c_void_p,
                                        C.c_void_p, C.c_void_p, C.c_void_p]),
    "mpsf_get_translate_summary": (C.c_int, [C.c_void_p, C.POINTER(TranslateSummary)]),
    "mpsf_remap": (C.c_int, [C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64, C.c_uint32,
                             C.c_void_p, C.c_void_p]),
    "mpsf_fold": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint32] + [C.c_void_p] * 6 + [C.c_uint64, C.c_void_p]
                  + [C.c_uint64] + [C.c_void_p] * 7 + [C.POINTER(FoldSummary), C.c_void_p]),
    "mpsf_kv_reserve": (C.c_int, [C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p,
                                  C.POINTER(C.c_uint64), C.c_void_p]),
    "mpsf_render_trace": (C.c_int64, [C.c_void_p, C.c_void_p, C.c_uint64, C.POINTER(RenderParams), C.c_void_p,
                                      C.c_uint64]),
    "mpsf_remap_blocks": (C.c_int, [C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64, C.c_void_p,
                                    C.c_uint64, C.c_void_p, C.c_void_p]),
    "mpsf_last_launches": (C.c_int, [C.c_void_p]),
    "mpsf_set_profiling": (C.c_int, [C.c_void_p, C.c_int]),
    "mpsf_get_profile": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int]),
    "mpsf_set_dense_dedup": (C.c_int, [C.c_void_p, C.c_int]),
    "mpsf_scan": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.POINTER(Params), C.c_void_p, C.c_void_p]),
    "mpsf_resolve": (C.c_int, [C.c_void_p, C.POINTER(Params), C.c_void_p, C.c_void_p, C.c_void_p]),
    "mpsf_general": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.POINTER(Params), C.c_int, C.c_void_p]),
    "mpsf_resolve2": (C.c_int, [C.c_void_p, C.POINTER(Params), C.c_void_p]),
    "mpsf_finalize": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.POINTER(Params), C.c_void_p,
                                C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "mpsf_exchange_buffers": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_int]),
    "mpsf_hash_export": (C.c_int64, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p]),
    "mpsf_hash_merge": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p]),
    "mpsf_classify": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p, C.c_void_p,
                                C.c_void_p]),
    "mpsf_sparse_export": (C.c_int64, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_uint64,
                                       C.c_void_p]),
    "mpsf_sparse_merge": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_uint64,
                                    C.c_void_p]),
}


class XBuf(C.Structure):
    _fields_ = [("ptr", C.c_void_p), ("count", C.c_uint64), ("elem_bytes", C.c_uint32), ("op", C.c_uint32)]


class KernelTime(C.Structure):
    _fields_ = [("name", C.c_char * 32), ("launches", C.c_uint64), ("total_ms", C.c_double)]

_lib = None


def load() -> C.CDLL:
    """Load libmpsf.so and bind every exported symbol.  Raises if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libmpsf.so not built at {LIB_PATH}: run `python -c 'import __graft_entry__ as g; "
                          f"g.build()'` (there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def sizes_match_numpy() -> bool:
    from .world import (CHANNEL_DTYPE, CLIENT_DTYPE, ENTRY_DTYPE, OUT_DTYPE, RANGE_DTYPE,
                        REMAP_DTYPE, VERDICT_DTYPE)
    return all(C.sizeof(s) == d.itemsize for s, d in (
        (FaultEntry, ENTRY_DTYPE), (RangeEntry, RANGE_DTYPE), (ChannelEntry, CHANNEL_DTYPE),
        (ClientEntry, CLIENT_DTYPE), (OutRecord, OUT_DTYPE), (ClientVerdict, VERDICT_DTYPE),
        (RemapEntry, REMAP_DTYPE)))
