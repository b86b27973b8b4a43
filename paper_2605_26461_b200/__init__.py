"""B200-native batched MMU-fault-buffer processing and recovery remap for the
fault-resilient MPS design of arxiv/paper_2605_26461 (reference package ``mpssim``).

The compute path lives in ``libmpsf.so`` (sm_100a CUDA behind the C ABI declared in
``include/mpsf.h``); this package is the Python host side that mirrors the
reference's operator names (see ``engine.py`` and ``shim.py``).
"""

from . import constants  # noqa: F401

__all__ = ["constants"]
