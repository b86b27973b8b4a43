"""Status codes of libmpsf.so mapped onto the reference's exception types.

The reference raises ``NoChannelAttribution`` for a fault record without channel
identity (``pkg/src/mpssim/errors.py:59-60``; ``pipeline.py:278-279``), ``KindMismatch``
for range-kind violations (``errors.py:36-37``) and ``SimError`` as the base
(``errors.py:4-5``).  When the reference package is importable (drop-in use inside the
simulator) its own classes are raised, so ``except mpssim.errors.X`` keeps working;
otherwise same-named local classes are used.
"""

from __future__ import annotations

try:  # drop-in: raise the reference's own exception types
    from mpssim.errors import KindMismatch, NoChannelAttribution, SimError  # type: ignore
except Exception:  # pragma: no cover - the GPU box has no reference install
    class SimError(Exception):
        """Base class for all simulator errors (mirrors mpssim.errors.SimError)."""

    class NoChannelAttribution(SimError):
        """A fault record that must carry a channel identity does not."""

    class KindMismatch(SimError):
        """Operation applied to a VA range of the wrong kind."""


class DeviceError(SimError):
    """CUDA failure or invalid use of the device path."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"mpsf error {code}: {msg}")
        self.code = code


class EntryError(SimError):
    """Malformed fault-buffer entry (bad engine/access/kind, engine mismatch, VA >= 2^53)."""

    def __init__(self, code: int, msg: str, index: int):
        super().__init__(f"mpsf error {code}: {msg} (entry {index})")
        self.code = code
        self.index = index


class HashOverflow(SimError):
    pass


E_CUDA, E_ARG, E_NO_CHANNEL, E_BAD_ENTRY, E_MISMATCH, E_VA, E_WORLD, E_OVERFLOW, E_NO_WORLD, E_TOO_LARGE = \
    -1, -2, -3, -4, -5, -6, -7, -8, -9, -10


def raise_for(code: int, msg: str, index: int = -1) -> None:
    if code == 0:
        return
    if code == E_NO_CHANNEL:
        raise NoChannelAttribution(f"{msg} (entry {index})")
    if code in (E_BAD_ENTRY, E_MISMATCH, E_VA):
        raise EntryError(code, msg, index)
    if code == E_WORLD:
        raise KindMismatch(msg)
    if code == E_OVERFLOW:
        raise HashOverflow(msg)
    raise DeviceError(code, msg)
