"""sm_100a backend for the reference's emitted device kernels
(``include/lfb_emitted.h``, ``csrc/emitted.cu``).

loopforge writes its optimised kernels as device-dialect text
(``emit_source``, ``lf/codegen.py:443-460``; ``loopforge build --emit``) and
executes them only through its interpreter. ``EmittedKernel`` compiles such a
text unchanged with NVRTC for sm_100a (a CUDA prelude for the dialect
macros) and runs it on a ``DeviceFieldState`` with the emitted launch
geometry — so the reference's own level-k kernels run natively on B200,
next to this package's hand-written ones (``tools/emitted_ladder.py``, the
paper's Table 1 structure).

The volume corpus' kernel ABI is ``(int Ne, float p0, float Rgas, float gam,
q, rhsq, D, g, Jinv)`` (``lf/codegen.py:361-373``), fp32. Levels >= 2 declare
``q``/``rhsq`` as ``vec4f*`` over the interleaved layout
``[e][field/4][k][j][i][field%4]`` (``lf/bench/recipes.py:46-47``); level 1
uses the element-batched layout of this package.
"""

from __future__ import annotations

import ctypes
import pathlib
import re
import threading

import torch

from . import _native
from .diagnostics import ExecutionError, NativeLibraryMissing

LIB_PATH = pathlib.Path(__file__).resolve().parent / "_lib" / "liblfb_emitted.so"
EXPORTED_SYMBOLS = ("lfb_emitted_compile", "lfb_emitted_cubin", "lfb_emitted_launch_volume",
                    "lfb_emitted_destroy")

_lock = threading.Lock()
_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise NativeLibraryMissing(f"{LIB_PATH} is not built; run __graft_entry__.build()")
            L = ctypes.CDLL(str(LIB_PATH))
            vp, i, i64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64
            L.lfb_emitted_compile.restype = i
            L.lfb_emitted_compile.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p,
                                              ctypes.POINTER(vp), ctypes.c_char_p,
                                              ctypes.c_size_t]
            L.lfb_emitted_cubin.restype = i64
            L.lfb_emitted_cubin.argtypes = [vp, ctypes.POINTER(vp)]
            L.lfb_emitted_launch_volume.restype = i
            L.lfb_emitted_launch_volume.argtypes = [vp, i64, i, i, i, ctypes.c_float,
                                                    ctypes.c_float, ctypes.c_float, vp, vp,
                                                    vp, vp, vp, vp]
            L.lfb_emitted_destroy.restype = i
            L.lfb_emitted_destroy.argtypes = [vp]
            _lib = L
    return _lib


_LAUNCH = re.compile(r"//\s*launch:\s*groups\s*=\s*(\w+),\s*lanes per group\s*=\s*(\d+)\s*x\s*(\d+)")
_KNAME = re.compile(r"//\s*kernel:\s*(\w+)")
_SIG = re.compile(r"KERNEL\s+void\s+(\w+)\s*\(([^)]*)\)")


class EmittedKernel:
    """One emitted kernel text, compiled for sm_100a (no GPU needed to
    compile; the cubin is loaded on the first launch)."""

    def __init__(self, source: str, arch: str = "sm_100a"):
        m = _SIG.search(source)
        if not m:
            raise ExecutionError("no 'KERNEL void name(...)' signature in the emitted text")
        self.name = m.group(1)
        params = [p.strip() for p in m.group(2).split(",")]
        self.vec4 = {}
        for p in params:
            pm = re.search(r"(\w+)\s*\*\s*(?:restrict\s+)?(\w+)$", p)
            if pm:
                self.vec4[pm.group(2)] = pm.group(1) == "vec4f"
        want = ["q", "rhsq", "D", "g", "Jinv"]
        if sorted(self.vec4) != sorted(want):
            raise ExecutionError(f"kernel {self.name!r} does not have the volume-corpus ABI "
                                 f"(arrays {sorted(self.vec4)})")
        lm = _LAUNCH.search(source)
        if not lm or lm.group(1) != "Ne":
            raise ExecutionError("no '// launch: groups = Ne, lanes per group = A x B' line")
        self.lanes = (int(lm.group(2)), int(lm.group(3)))
        self.source = source
        log = ctypes.create_string_buffer(1 << 16)
        h = ctypes.c_void_p()
        rc = lib().lfb_emitted_compile(source.encode(), self.name.encode(), arch.encode(),
                                       ctypes.byref(h), log, len(log))
        self.log = log.value.decode(errors="replace")
        if rc != _native.LFB_OK:
            raise ExecutionError(f"NVRTC rejected kernel {self.name!r}: {self.log.strip()}")
        self._h = h

    @classmethod
    def from_file(cls, path, arch: str = "sm_100a") -> "EmittedKernel":
        return cls(pathlib.Path(path).read_text(), arch)

    @property
    def cubin_size(self) -> int:
        return int(lib().lfb_emitted_cubin(self._h, None))

    @property
    def interleaved(self) -> bool:
        """q / rhsq as vec4f over [e][field/4][k][j][i][field%4]."""
        return self.vec4["q"]

    # -- layout of q / rhsq ------------------------------------------------
    @staticmethod
    def to_interleaved(t: torch.Tensor) -> torch.Tensor:
        """(Ne, 8, Nq, Nq, Nq) element-batched -> (Ne, 2, Nq, Nq, Nq, 4)."""
        ne, f, a, b, c = t.shape
        return t.view(ne, f // 4, 4, a, b, c).permute(0, 1, 3, 4, 5, 2).contiguous()

    @staticmethod
    def from_interleaved(t: torch.Tensor) -> torch.Tensor:
        ne, fo, a, b, c, fi = t.shape
        return t.permute(0, 1, 5, 2, 3, 4).reshape(ne, fo * fi, a, b, c)

    def bind(self, ds) -> dict:
        """Device arrays in this kernel's layouts (fp32), from a DeviceFieldState."""
        if ds.dtype != torch.float32:
            raise ExecutionError("emitted kernels are float32 (lf/interp.py:71-72)")
        nq = ds.nq
        if self.lanes != (nq, nq):
            raise ExecutionError(f"kernel lanes {self.lanes} do not match Nq={nq}")
        q, r = ds.q, ds.rhsq
        if self.interleaved:
            q, r = self.to_interleaved(q), self.to_interleaved(r)
        return {"q": q, "rhsq": r, "D": ds.D, "g": ds.g, "Jinv": ds.Jinv, "ne": ds.ne,
                "constants": ds.constants}

    def launch(self, bound: dict, stream=None) -> None:
        c = bound["constants"]
        s = stream or torch.cuda.current_stream(bound["q"].device)
        rc = lib().lfb_emitted_launch_volume(
            self._h, bound["ne"], self.lanes[0], self.lanes[1], bound["ne"], c.p0, c.R,
            c.gamma, bound["q"].data_ptr(), bound["rhsq"].data_ptr(), bound["D"].data_ptr(),
            bound["g"].data_ptr(), bound["Jinv"].data_ptr(), s.cuda_stream)
        _native.check(rc, f"emitted kernel {self.name}")

    def unbind(self, bound: dict, ds) -> None:
        """Copy the kernel's rhsq back into ``ds.rhsq`` (element-batched)."""
        if self.interleaved:
            ds.rhsq.copy_(self.from_interleaved(bound["rhsq"]))

    def __call__(self, ds, stream=None) -> None:
        """``ds.rhsq += v`` by the emitted kernel (interpret_state semantics)."""
        b = self.bind(ds)
        self.launch(b, stream)
        self.unbind(b, ds)

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and _lib is not None:
            _lib.lfb_emitted_destroy(self._h)
        self._h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass
