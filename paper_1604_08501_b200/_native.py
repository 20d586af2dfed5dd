"""ctypes binding of the C-ABI library ``_lib/liblfb_volume.so``
(declared in ``include/lfb_volume.h``).

ctypes (not a torch extension) keeps the boundary a plain C ABI: the same
symbols a cgo / JNI / N-API binding would use. The
library is built in-tree by ``__graft_entry__.build()``; if it is missing,
every call raises ``NativeLibraryMissing`` — there is no fallback path.
"""

from __future__ import annotations

import ctypes
import pathlib
import threading

from .diagnostics import ExecutionError, KernelLaunchError, NativeLibraryMissing

LIB_PATH = pathlib.Path(__file__).resolve().parent / "_lib" / "liblfb_volume.so"
#: test-only build of the same sources plus the tc kernel's barrier-deletion
#: mutants (tests/test_mutants.py); the package never loads it by itself
MUTANT_LIB_PATH = LIB_PATH.with_name("liblfb_volume_mutants.so")

LFB_OK = 0
LFB_ERR_BAD_NQ = 1
LFB_ERR_BAD_NE = 2
LFB_ERR_NULL = 3
LFB_ERR_MISALIGNED = 4
LFB_ERR_LAUNCH = 5
LFB_ERR_CUDA = 6
LFB_ERR_BAD_CONSTANTS = 7
LFB_ERR_BAD_VARIANT = 8
LFB_ERR_ALLOC = 9

VARIANT_AUTO = 0
VARIANT_BASIC = 1
VARIANT_FUSED = 2
VARIANT_TC = 3
VARIANT_LINES = 4
VARIANT_COL = 5
VARIANT_LT = 6
VARIANT_LTU = 7
VARIANT_LO = 8
VARIANTS = {"auto": VARIANT_AUTO, "basic": VARIANT_BASIC, "fused": VARIANT_FUSED,
            "tc": VARIANT_TC, "lines": VARIANT_LINES, "col": VARIANT_COL, "lt": VARIANT_LT,
            "ltu": VARIANT_LTU, "lo": VARIANT_LO}

MAX_NQ = 16

#: every symbol include/lfb_volume.h declares (tests check the exports)
EXPORTED_SYMBOLS = (
    "lfb_volume_rhs_f64", "lfb_volume_rhs_f32",
    "lfb_volume_rhs_variant_f64", "lfb_volume_rhs_variant_f32",
    "lfb_variant_available", "lfb_variant_name", "lfb_resolve_variant",
    "lfb_error_string", "lfb_version",
    "lfb_field_state_to_element_batched", "lfb_element_batched_to_field_state",
    "lfb_make_inputs_device",
    "lfb_pipeline_create", "lfb_pipeline_destroy", "lfb_pipeline_info",
    "lfb_volume_host",
)

HOST_INCREMENT = 0
HOST_ACCUMULATE = 1

_lock = threading.Lock()
_lib = None

_i, _i64, _vp = ctypes.c_int, ctypes.c_int64, ctypes.c_void_p
_d, _f = ctypes.c_double, ctypes.c_float


def _declare(L) -> None:
    for name, scal in (("f64", _d), ("f32", _f)):
        fn = getattr(L, f"lfb_volume_rhs_{name}")
        fn.restype = _i
        fn.argtypes = [_i, _i64, scal, scal, scal, _vp, _vp, _vp, _vp, _vp, _vp]
        fn = getattr(L, f"lfb_volume_rhs_variant_{name}")
        fn.restype = _i
        fn.argtypes = [_i, _i, _i64, scal, scal, scal, _vp, _vp, _vp, _vp, _vp, _vp]
    L.lfb_variant_available.restype = _i
    L.lfb_variant_available.argtypes = [_i, _i, _i]
    L.lfb_resolve_variant.restype = _i
    L.lfb_resolve_variant.argtypes = [_i, _i]
    L.lfb_variant_name.restype = ctypes.c_char_p
    L.lfb_variant_name.argtypes = [_i]
    L.lfb_error_string.restype = ctypes.c_char_p
    L.lfb_error_string.argtypes = [_i]
    L.lfb_version.restype = _i
    L.lfb_version.argtypes = []
    for name in ("lfb_field_state_to_element_batched",
                 "lfb_element_batched_to_field_state"):
        fn = getattr(L, name)
        fn.restype = _i
        fn.argtypes = [_i, _i, _i, ctypes.POINTER(ctypes.c_int64), _i64, _vp, _vp, _vp]
    L.lfb_pipeline_create.restype = _i
    L.lfb_pipeline_create.argtypes = [_i, _i64, _i, _i, _i, ctypes.POINTER(_vp)]
    L.lfb_pipeline_destroy.restype = _i
    L.lfb_pipeline_destroy.argtypes = [_vp]
    L.lfb_pipeline_info.restype = _i
    L.lfb_pipeline_info.argtypes = [_vp, ctypes.POINTER(_i64), ctypes.POINTER(_i64)]
    L.lfb_volume_host.restype = _i
    L.lfb_volume_host.argtypes = [_vp, _i, _i64, _d, _d, _d, _vp, _vp, _vp, _vp, _vp, _vp]
    L.lfb_make_inputs_device.restype = _i
    L.lfb_make_inputs_device.argtypes = [_i, _i64, _i64, ctypes.c_uint64, _i, _d, _d,
                                         _vp, _vp, _vp, _vp, _vp]


_lib_path = LIB_PATH


def use_library(path) -> None:
    """Bind a different build of the C-ABI library (the mutant test library)
    instead of LIB_PATH; must precede the first call into the library."""
    global _lib_path
    with _lock:
        if _lib is not None:
            raise ExecutionError("the native library is already loaded")
        _lib_path = pathlib.Path(path)


def lib():
    """The loaded library (raises NativeLibraryMissing if absent)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not _lib_path.exists():
                raise NativeLibraryMissing(
                    f"{_lib_path} is not built; run __graft_entry__.build()")
            try:
                L = ctypes.CDLL(str(_lib_path))
            except OSError as exc:  # pragma: no cover - environment specific
                raise NativeLibraryMissing(str(exc)) from exc
            _declare(L)
            _lib = L
    return _lib


def error_string(code: int) -> str:
    return lib().lfb_error_string(code).decode()


def check(code: int, what: str = "lfb call") -> None:
    """Map a C-ABI return code to the reference-style exception."""
    if code == LFB_OK:
        return
    msg = f"{what}: {error_string(code)} (code {code})"
    if code in (LFB_ERR_LAUNCH, LFB_ERR_CUDA, LFB_ERR_ALLOC):
        raise KernelLaunchError(msg)
    raise ExecutionError(msg)


def variant_id(variant) -> int:
    if isinstance(variant, str):
        try:
            return VARIANTS[variant]
        except KeyError:
            raise ExecutionError(f"unknown kernel variant {variant!r}") from None
    return int(variant)


def resolve_variant(dtype_bytes: int, nq: int) -> str:
    L = lib()
    return L.lfb_variant_name(L.lfb_resolve_variant(dtype_bytes, nq)).decode()


def variant_available(variant, dtype_bytes: int, nq: int) -> bool:
    return bool(lib().lfb_variant_available(variant_id(variant), dtype_bytes, nq))


def volume_rhs_ptr(dtype_bytes: int, variant, nq: int, ne: int, p0: float,
                   R: float, gam: float, q: int, rhsq: int, D: int, g: int,
                   jinv: int, stream: int) -> None:
    """Raw C-ABI call on device pointers (ints). Raises on a non-zero code."""
    L = lib()
    fn = L.lfb_volume_rhs_variant_f64 if dtype_bytes == 8 else L.lfb_volume_rhs_variant_f32
    rc = fn(variant_id(variant), int(nq), int(ne), p0, R, gam, q, rhsq, D, g,
            jinv, stream)
    check(rc, "lfb_volume_rhs")


def reverse_axes_ptr(to_batched: bool, in_bytes: int, out_bytes: int, dims, ne: int,
                     src: int, dst: int, stream: int) -> None:
    """FieldState (C-order, element last) <-> element-batched conversion on
    device pointers, with a fused f32/f64 cast."""
    L = lib()
    arr = (ctypes.c_int64 * len(dims))(*[int(d) for d in dims])
    fn = (L.lfb_field_state_to_element_batched if to_batched
          else L.lfb_element_batched_to_field_state)
    check(fn(in_bytes, out_bytes, len(dims), arr, int(ne), src, dst, stream),
          "layout conversion")


def make_inputs_ptr(nq: int, ne: int, e_offset: int, seed: int, dtype_bytes: int,
                    p0: float, R: float, q: int, rhsq: int, g: int, jinv: int,
                    stream: int) -> None:
    check(lib().lfb_make_inputs_device(int(nq), int(ne), int(e_offset), int(seed),
                                       int(dtype_bytes), float(p0), float(R), q, rhsq,
                                       g, jinv, stream), "lfb_make_inputs_device")


class HostPipeline:
    """Owner of one native host-buffer pipeline (``lfb_pipeline_create``):
    device staging for 3 chunks of ``chunk`` elements and 3 streams. ``run``
    evaluates the volume term over arrays in the reference's HOST layout
    (C-order numpy, element axis last) — see include/lfb_volume.h."""

    def __init__(self, nq: int, chunk: int, host_bytes: int, compute_bytes: int,
                 device: int = -1):
        L = lib()
        h = _vp()
        check(L.lfb_pipeline_create(int(nq), int(chunk), int(host_bytes),
                                    int(compute_bytes), int(device), ctypes.byref(h)),
              "lfb_pipeline_create")
        self._h = h
        self._run_lock = threading.Lock()  # one pipeline serves one call at a time
        self.nq, self.chunk = int(nq), int(chunk)
        self.host_bytes, self.compute_bytes = int(host_bytes), int(compute_bytes)

    @property
    def device_bytes(self) -> int:
        n = _i64()
        check(lib().lfb_pipeline_info(self._h, None, ctypes.byref(n)), "lfb_pipeline_info")
        return int(n.value)

    def run(self, mode: int, ne: int, p0: float, R: float, gam: float, q: int, D: int,
            g: int, jinv: int, out: int, stream: int = 0) -> None:
        """Host pointers (ints). Synchronous: the result is in ``out`` on return."""
        with self._run_lock:
            if self._h is None:
                raise ExecutionError("pipeline is closed")
            check(lib().lfb_volume_host(self._h, int(mode), int(ne), float(p0), float(R),
                                        float(gam), q, D, g, jinv, out, stream),
                  "lfb_volume_host")

    def close(self) -> None:
        lock = getattr(self, "_run_lock", None)
        if lock is not None:
            lock.acquire()
        try:
            if getattr(self, "_h", None) is not None and _lib is not None:
                _lib.lfb_pipeline_destroy(self._h)
            self._h = None
        finally:
            if lock is not None:
                lock.release()

    def __del__(self):  # pragma: no cover - GC timing
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass
