"""ctypes binding of the C oracle (``oracle/volterm_oracle.c``) — TEST
INFRASTRUCTURE ONLY (see ``oracle/volterm.py`` for the usage rule).

Arrays are in the element-batched (Fortran) layout of the C-ABI; the
``to_element_batched`` / ``from_element_batched`` helpers here are an
independent numpy restatement of that layout (they do not use the
product's conversion code, so the checker stays independent of the thing
checked).
"""

from __future__ import annotations

import ctypes
import os
import pathlib
import subprocess

import numpy as np

_HERE = pathlib.Path(__file__).resolve().parent
_LIB_PATH = _HERE / "build" / "liboracle.so"
_lib = None

_dp = ctypes.POINTER(ctypes.c_double)


def build() -> pathlib.Path:
    """Compile the C oracle (``make -C oracle``)."""
    subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            build()
        L = ctypes.CDLL(str(_LIB_PATH))
        L.oracle_volume_f64.restype = ctypes.c_int
        L.oracle_volume_f64.argtypes = [
            ctypes.c_int, ctypes.c_int64, ctypes.c_double, ctypes.c_double,
            ctypes.c_double, _dp, _dp, _dp, _dp, _dp, ctypes.c_int,
            ctypes.c_int]
        L.oracle_max_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def max_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return lib().oracle_max_threads()


def to_element_batched(state, dtype=np.float64):
    """(q, g, Jinv, D) of a FieldState in the C-ABI layout:
    q [Ne,8,k,j,i], g [Ne,dir,a,k,j,i], Jinv [Ne,k,j,i], D [n,i]."""
    q = np.ascontiguousarray(state.q.transpose(4, 3, 2, 1, 0), dtype=dtype)
    g = np.ascontiguousarray(state.g.transpose(5, 4, 3, 2, 1, 0), dtype=dtype)
    j = np.ascontiguousarray(state.Jinv.transpose(3, 2, 1, 0), dtype=dtype)
    d = np.ascontiguousarray(state.D.T, dtype=dtype)
    return q, g, j, d


def from_element_batched(x: np.ndarray) -> np.ndarray:
    """[Ne,8,k,j,i] -> logical [i,j,k,8,Ne] (a view)."""
    return x.transpose(4, 3, 2, 1, 0)


def volume_f64_eb(nq: int, q, g, jinv, D, constants, out=None,
                  accumulate: bool = False, nthreads: int = 0) -> np.ndarray:
    """Run the C oracle on element-batched fp64 arrays."""
    for a in (q, g, jinv, D):
        assert a.dtype == np.float64 and a.flags.c_contiguous
    ne = q.shape[0]
    if out is None:
        out = np.zeros_like(q)
    rc = lib().oracle_volume_f64(
        nq, ne, float(constants.p0), float(constants.R),
        float(constants.gamma), q.ctypes.data_as(_dp), out.ctypes.data_as(_dp),
        D.ctypes.data_as(_dp), g.ctypes.data_as(_dp),
        jinv.ctypes.data_as(_dp), int(bool(accumulate)), int(nthreads))
    if rc != 0:
        raise RuntimeError(f"oracle_volume_f64 failed with code {rc}")
    return out


def volume_term_f64_c(state, c=None, nthreads: int = 0) -> np.ndarray:
    """fp64 increment in the logical [Nq,Nq,Nq,8,Ne] layout."""
    c = c or state.constants
    q, g, j, d = to_element_batched(state)
    out = volume_f64_eb(state.q.shape[0], q, g, j, d, c, nthreads=nthreads)
    return np.ascontiguousarray(from_element_batched(out))
