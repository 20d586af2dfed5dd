"""Error types, mirroring the reference's conventions
(``lf/diagnostics.py:8-9`` ``LoopforgeError``; ``:208-209``
``ExecutionError``; ``lf/interp.py:51-74`` raises ``ExecutionError`` for
missing arrays, shape and dtype mismatches).

The C-ABI returns integer codes (``include/lfb_volume.h``); the Python layer
maps each to one of these classes with the library's message.
"""

from __future__ import annotations


class LoopforgeError(Exception):
    """Base class for all errors of this package (same name as the
    reference's base class so ``except LoopforgeError`` keeps working)."""


class ExecutionError(LoopforgeError):
    """Bad arguments to a kernel execution: missing array, shape or dtype
    mismatch, invalid sizes (``lf/interp.py:60-72``)."""


class KernelLaunchError(ExecutionError):
    """The CUDA launch itself failed (``LFB_ERR_LAUNCH`` / ``LFB_ERR_CUDA``)."""


class NativeLibraryMissing(LoopforgeError):
    """The CUDA C-ABI library is not built or cannot be loaded. There is no
    CPU fallback: build it with ``__graft_entry__.build()``."""
