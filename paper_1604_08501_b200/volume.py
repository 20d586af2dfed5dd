"""Host-side mirror of the reference's volume-term entry points, backed by
the sm_100a CUDA kernel behind the C-ABI (``include/lfb_volume.h``).

Reference entry points kept signature-compatible (``lf/`` =
``pkg/src/loopforge/``):

* ``reference_volume_term(state, c=None)`` — ``lf/bench/reference.py:36-70``:
  the rhsq increment, fp64 accumulation, float32 result, rhsq untouched;
* ``interpret_state(kernels, state, nq, ne)`` — ``lf/bench/driver.py:54-69``:
  in place ``rhsq += v`` at float32 (the fused level-8 kernel's semantics),
  returns ``(state.rhsq, envs)``;
* ``max_rel_error`` — ``lf/bench/driver.py:72-91`` (the parity metric).

New, B200-first entry points:

* ``volume_term(state, c=None, *, dtype=float64)`` — increment at the chosen
  precision (fp64 default);
* ``volume_rhs_(state, c=None, *, dtype=None)`` — in-place update;
* ``DeviceFieldState`` + ``volume_rhs_device`` — the device-resident hot
  path: element-batched tensors in HBM, one stream-ordered C-ABI call.

Every compute call goes through the CUDA library; if it is missing the call
raises ``NativeLibraryMissing`` (no CPU fallback exists in this package).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from .diagnostics import ExecutionError
from .inputs import FieldState, PhysicalConstants

_TORCH_DTYPES = {np.dtype(np.float32): torch.float32,
                 np.dtype(np.float64): torch.float64}


def _torch_dtype(dtype) -> torch.dtype:
    if isinstance(dtype, torch.dtype):
        if dtype not in (torch.float32, torch.float64):
            raise ExecutionError(f"unsupported dtype {dtype}")
        return dtype
    try:
        return _TORCH_DTYPES[np.dtype(dtype)]
    except (KeyError, TypeError):
        raise ExecutionError(f"unsupported dtype {dtype!r}") from None


def _device(device) -> torch.device:
    if device is None:
        if not torch.cuda.is_available():
            raise ExecutionError("no CUDA device available (this package has "
                                 "no CPU path)")
        return torch.device("cuda", torch.cuda.current_device())
    dev = torch.device(device)
    if dev.type != "cuda":
        raise ExecutionError(f"device must be a CUDA device, got {dev}")
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    return dev


def state_arrays(state) -> dict:
    """The five arrays of a FieldState — this package's mirror or the
    reference's own ``loopforge.bench.FieldState`` (``lf/bench/inputs.py:
    52-74``), which has ``arrays()`` and ``constants`` but none of the
    mirror's conveniences (``nq``, ``ne``, ``astype``): entry points use only
    what both define."""
    if hasattr(state, "arrays"):
        return state.arrays()
    return {n: getattr(state, n, None) for n in ("q", "rhsq", "D", "g", "Jinv")}


def state_constants(state) -> PhysicalConstants:
    c = getattr(state, "constants", None)
    return PhysicalConstants() if c is None else c


def validate_state(state: FieldState, nq: int | None = None,
                   ne: int | None = None, dtype=None) -> tuple[int, int]:
    """Shape/dtype checks with the reference's error behaviour
    (``lf/interp.py:51-74``: ``ExecutionError`` naming the array).
    Returns ``(Nq, Ne)`` read from the arrays, never from attributes only
    this package's FieldState mirror has."""
    arrays = state_arrays(state)
    for name in ("q", "rhsq", "D", "g", "Jinv"):
        if arrays.get(name) is None:
            raise ExecutionError(f"missing array argument {name!r}")
    q = arrays["q"]
    if q.ndim != 5 or q.shape[3] != 8:
        raise ExecutionError(f"array 'q' has shape {q.shape}, expected "
                             f"(Nq, Nq, Nq, 8, Ne)")
    nq_ = int(q.shape[0]) if nq is None else int(nq)
    ne_ = int(q.shape[4]) if ne is None else int(ne)
    want = {"q": (nq_, nq_, nq_, 8, ne_), "rhsq": (nq_, nq_, nq_, 8, ne_),
            "D": (nq_, nq_), "g": (nq_, nq_, nq_, 3, 3, ne_),
            "Jinv": (nq_, nq_, nq_, ne_)}
    for name, shape in want.items():
        if tuple(arrays[name].shape) != shape:
            raise ExecutionError(f"array {name!r} has shape "
                                 f"{tuple(arrays[name].shape)}, kernel expects "
                                 f"{shape}")
        if dtype is not None and arrays[name].dtype != np.dtype(dtype):
            raise ExecutionError(f"array {name!r} must be "
                                 f"{np.dtype(dtype).name}")
        if arrays[name].dtype not in (np.float32, np.float64):
            raise ExecutionError(f"array {name!r} must be float32 or float64")
    if not 1 <= nq_ <= _native.MAX_NQ:
        raise ExecutionError(f"Nq={nq_} outside [1, {_native.MAX_NQ}]")
    return nq_, ne_


@dataclass
class DeviceFieldState:
    """A FieldState resident in HBM in the element-batched layout of the
    C-ABI (the Fortran declarations' layout, ``volume.f90:14-18``):

    q, rhsq ``(Ne, 8, Nq, Nq, Nq)`` = [e][field][k][j][i];
    g ``(Ne, 3, 3, Nq, Nq, Nq)`` = [e][dir][a][k][j][i];
    Jinv ``(Ne, Nq, Nq, Nq)`` = [e][k][j][i]; D ``(Nq, Nq)`` = [n][i].
    """

    q: torch.Tensor
    rhsq: torch.Tensor
    D: torch.Tensor
    g: torch.Tensor
    Jinv: torch.Tensor
    constants: PhysicalConstants

    @property
    def nq(self) -> int:
        return int(self.q.shape[2])

    @property
    def ne(self) -> int:
        return int(self.q.shape[0])

    @property
    def dtype(self) -> torch.dtype:
        return self.q.dtype

    @property
    def device(self) -> torch.device:
        return self.q.device

    @classmethod
    def from_field_state(cls, state: FieldState, dtype=torch.float64,
                         device=None, stream=None) -> "DeviceFieldState":
        """Upload the reference's C-order arrays ([i,j,k,b,e], element
        fastest) as they are and convert them on the device (native
        layout kernel, cast fused) to the element-batched layout."""
        nq, ne = validate_state(state)
        arrays = state_arrays(state)
        dev = _device(device)
        dt = _torch_dtype(dtype)
        out_bytes = 8 if dt == torch.float64 else 4
        with torch.cuda.device(dev):
            s = stream or torch.cuda.current_stream(dev)

            def up(a: np.ndarray, batched_shape):
                src = torch.from_numpy(np.ascontiguousarray(a)).to(dev, non_blocking=False)
                out = torch.empty(batched_shape, dtype=dt, device=dev)
                dims = a.shape[:-1]
                _native.reverse_axes_ptr(True, src.element_size(), out_bytes, dims,
                                         a.shape[-1], src.data_ptr(), out.data_ptr(),
                                         s.cuda_stream)
                if src.is_cuda:  # staging buffer stays valid until the kernel ran
                    src.record_stream(s)
                return out

            ds = cls(q=up(arrays["q"], (ne, 8, nq, nq, nq)),
                     rhsq=up(arrays["rhsq"], (ne, 8, nq, nq, nq)),
                     D=up(arrays["D"], (nq, nq)),
                     g=up(arrays["g"], (ne, 3, 3, nq, nq, nq)),
                     Jinv=up(arrays["Jinv"], (ne, nq, nq, nq)),
                     constants=state_constants(state))
        return ds

    @classmethod
    def generate(cls, nq: int, ne: int, seed: int = 1, dtype=torch.float64,
                 device=None, e_offset: int = 0,
                 constants: PhysicalConstants | None = None,
                 stream=None) -> "DeviceFieldState":
        """Synthetic state generated on the device (make_inputs
        distributions, counter-based RNG; element e holds global element
        e + e_offset, so shards of a multi-GPU run reproduce one global
        state). D is the reference's differentiation_matrix."""
        from .inputs import differentiation_matrix
        c = constants or PhysicalConstants()
        ds = cls.empty(nq, ne, dtype=dtype, device=device, constants=c)
        with torch.cuda.device(ds.device):
            s = stream or torch.cuda.current_stream(ds.device)
            ds.D.copy_(torch.from_numpy(differentiation_matrix(nq).T.copy()))
            _native.make_inputs_ptr(nq, ne, e_offset, seed, ds.q.element_size(),
                                    c.p0, c.R, ds.q.data_ptr(), ds.rhsq.data_ptr(),
                                    ds.g.data_ptr(), ds.Jinv.data_ptr(), s.cuda_stream)
        return ds

    def to_field_state(self, dtype=None) -> FieldState:
        """Download into the reference's logical layout (native kernel)."""
        arrays = [self.to_logical(t, dtype) for t in (self.q, self.rhsq)]
        D = self.to_logical(self.D, dtype)
        g = self.to_logical(self.g, dtype)
        J = self.to_logical(self.Jinv, dtype)
        return FieldState(arrays[0], arrays[1], D, g, J, self.constants)

    @classmethod
    def empty(cls, nq: int, ne: int, dtype=torch.float64, device=None,
              constants: PhysicalConstants | None = None) -> "DeviceFieldState":
        dev = _device(device)
        dt = _torch_dtype(dtype)
        z = dict(dtype=dt, device=dev)
        return cls(q=torch.empty((ne, 8, nq, nq, nq), **z),
                   rhsq=torch.zeros((ne, 8, nq, nq, nq), **z),
                   D=torch.empty((nq, nq), **z),
                   g=torch.empty((ne, 3, 3, nq, nq, nq), **z),
                   Jinv=torch.empty((ne, nq, nq, nq), **z),
                   constants=constants or PhysicalConstants())

    def shard(self, start: int, stop: int) -> "DeviceFieldState":
        """Contiguous element range [start, stop) as views (no copy): in the
        element-batched layout each shard is one slab of every array."""
        return DeviceFieldState(self.q[start:stop], self.rhsq[start:stop],
                                self.D, self.g[start:stop],
                                self.Jinv[start:stop], self.constants)

    @staticmethod
    def to_logical(x: torch.Tensor, dtype=None) -> np.ndarray:
        """Element-batched [Ne][...] tensor -> numpy C-order [..., Ne]
        (the reference's layout), converted on the device by the native
        layout kernel (optionally cast to ``dtype``)."""
        dt = x.dtype if dtype is None else _torch_dtype(dtype)
        ne = int(x.shape[0])
        dims = tuple(int(d) for d in reversed(x.shape[1:]))
        out = torch.empty(dims + (ne,), dtype=dt, device=x.device)
        if x.numel():
            with torch.cuda.device(x.device):
                _native.reverse_axes_ptr(False, x.element_size(), out.element_size(),
                                         dims, ne, x.data_ptr(), out.data_ptr(),
                                         torch.cuda.current_stream(x.device).cuda_stream)
        return out.cpu().numpy()

    def rhsq_logical(self) -> np.ndarray:
        return self.to_logical(self.rhsq)


def volume_rhs_device(ds: DeviceFieldState, *, variant="auto",
                      stream: torch.cuda.Stream | None = None,
                      constants: PhysicalConstants | None = None) -> None:
    """The hot path: ``ds.rhsq += v`` on the device, one C-ABI call,
    asynchronous on ``stream`` (default: torch's current stream)."""
    tensors = (ds.q, ds.rhsq, ds.D, ds.g, ds.Jinv)
    dt = ds.q.dtype
    nq, ne = ds.nq, ds.ne
    shapes = ((ne, 8, nq, nq, nq), (ne, 8, nq, nq, nq), (nq, nq),
              (ne, 3, 3, nq, nq, nq), (ne, nq, nq, nq))
    for name, t, shape in zip(("q", "rhsq", "D", "g", "Jinv"), tensors, shapes):
        if tuple(t.shape) != shape:
            raise ExecutionError(f"array {name!r} has shape {tuple(t.shape)}, "
                                 f"kernel expects {shape}")
        if t.dtype != dt:
            raise ExecutionError(f"array {name!r} must be {dt}")
        if t.device.type != "cuda" or t.device != ds.q.device:
            raise ExecutionError(f"array {name!r} must be on {ds.q.device}")
        if not t.is_contiguous():
            raise ExecutionError(f"array {name!r} must be contiguous")
    if dt not in (torch.float32, torch.float64):
        raise ExecutionError(f"unsupported dtype {dt}")
    c = constants or ds.constants
    if stream is None:
        stream = torch.cuda.current_stream(ds.q.device)
    with torch.cuda.device(ds.q.device):
        _native.volume_rhs_ptr(
            8 if dt == torch.float64 else 4, variant, nq, ne,
            float(c.p0), float(c.R), float(c.gamma),
            ds.q.data_ptr(), ds.rhsq.data_ptr(), ds.D.data_ptr(),
            ds.g.data_ptr(), ds.Jinv.data_ptr(), stream.cuda_stream)


def volume_term(state: FieldState, c: PhysicalConstants | None = None, *,
                dtype=np.float64, device=None, variant="auto") -> np.ndarray:
    """The rhsq increment v at ``dtype`` (state.rhsq unchanged), logical
    layout ``[Nq, Nq, Nq, 8, Ne]``."""
    validate_state(state)
    ds = DeviceFieldState.from_field_state(state, dtype=dtype, device=device)
    ds.rhsq.zero_()
    volume_rhs_device(ds, variant=variant, constants=c or state_constants(state))
    return ds.rhsq_logical()


#: device staging budget of one pipeline slot (3 slots per pipeline)
PIPELINE_SLOT_BYTES = 320 << 20
_PIPELINES: dict = {}


def pipeline_chunk(nq: int, ne: int, host_bytes: int, compute_bytes: int,
                   slot_bytes: int = PIPELINE_SLOT_BYTES) -> int:
    """Elements per pipeline chunk: the largest power of two whose staging
    (26 values per point in host and compute dtype) fits ``slot_bytes``, at
    least 1, at most ``ne``. Nq=8 f32->f64: 2048 elements (8 KB copy rows,
    the fastest of 1024..16384 in profiles/r01_e2e_chunks.txt)."""
    per_elem = 26 * nq ** 3 * (host_bytes + compute_bytes)
    fit = max(1, slot_bytes // per_elem)
    return max(1, min(int(ne), 1 << (fit.bit_length() - 1)))


def host_pipeline(nq: int, ne: int, host_bytes: int, compute_bytes: int,
                  device=None, chunk: int | None = None) -> "_native.HostPipeline":
    """A cached native host-buffer pipeline for (device, Nq, dtypes, chunk)."""
    dev = _device(device)
    chunk = chunk or pipeline_chunk(nq, ne, host_bytes, compute_bytes)
    key = (dev.index, nq, host_bytes, compute_bytes, chunk)
    p = _PIPELINES.get(key)
    if p is None:
        if len(_PIPELINES) >= 4:  # bound the cached staging
            _PIPELINES.pop(next(iter(_PIPELINES))).close()
        p = _PIPELINES[key] = _native.HostPipeline(nq, chunk, host_bytes, compute_bytes,
                                                   dev.index)
    return p


def volume_host(state: FieldState, c: PhysicalConstants | None = None, *,
                accumulate: bool = False, compute_dtype=np.float64, out=None,
                device=None, chunk: int | None = None, stream=None) -> np.ndarray:
    """The volume term over HOST arrays in the reference's layout, through
    the native pipeline (``lfb_volume_host``): chunked 2-D copies, on-device
    layout conversion, the sm_100a kernel, copies back — all overlapped.
    ``accumulate=False``: returns the increment v (``reference_volume_term``
    semantics, rhsq untouched); ``True``: ``state.rhsq += v`` in place.
    Every array must share one dtype (f32 or f64); ``out`` (increment mode)
    may be a preallocated C-order array of that dtype, e.g. page-locked."""
    nq, ne = validate_state(state)
    arrays = state_arrays(state)
    hdt = arrays["q"].dtype
    for name in ("q", "rhsq", "D", "g", "Jinv"):
        a = arrays[name]
        if a.dtype != hdt:
            raise ExecutionError(f"array {name!r} must be {hdt.name} (one dtype "
                                 f"for the host pipeline)")
        if not a.flags.c_contiguous:
            raise ExecutionError(f"array {name!r} must be C-contiguous")
    cb = np.dtype(compute_dtype).itemsize
    if cb not in (4, 8):
        raise ExecutionError(f"unsupported compute dtype {compute_dtype!r}")
    c = c or state_constants(state)
    q = arrays["q"]
    if accumulate:
        target = arrays["rhsq"]
    else:
        target = np.empty(q.shape, hdt) if out is None else out
        if target.shape != q.shape or target.dtype != hdt or \
                not target.flags.c_contiguous:
            raise ExecutionError("out must be a C-contiguous array shaped like q")
    if ne == 0:
        if not accumulate:
            target[...] = 0
        return target
    p = host_pipeline(nq, ne, hdt.itemsize, cb, device, chunk)
    dev = _device(device)
    s = stream or torch.cuda.current_stream(dev)
    p.run(_native.HOST_ACCUMULATE if accumulate else _native.HOST_INCREMENT, ne,
          c.p0, c.R, c.gamma, q.ctypes.data, arrays["D"].ctypes.data,
          arrays["g"].ctypes.data, arrays["Jinv"].ctypes.data, target.ctypes.data,
          s.cuda_stream)
    return target


def reference_volume_term(state: FieldState,
                          c: PhysicalConstants | None = None) -> np.ndarray:
    """Drop-in for ``lf/bench/reference.py:36-70``: fp64 accumulation on
    the GPU, float32 result, rhsq untouched. f32 states (what ``make_inputs``
    builds) take the native host pipeline (``volume_host``)."""
    validate_state(state)
    if all(a.dtype == np.float32 and a.flags.c_contiguous
           for a in state_arrays(state).values()):
        return volume_host(state, c, compute_dtype=np.float64)
    return volume_term(state, c, dtype=np.float64).astype(np.float32)


def volume_rhs_(state: FieldState, c: PhysicalConstants | None = None, *,
                dtype=None, device=None, variant="auto") -> np.ndarray:
    """In place ``state.rhsq += v`` (``volume.f90:53-60`` semantics),
    computed at ``dtype`` (default: the dtype of ``state.rhsq``). Uniform-
    dtype states with the AUTO variant take the native host pipeline."""
    validate_state(state)
    arrays = state_arrays(state)
    rhsq = arrays["rhsq"]
    dt = rhsq.dtype if dtype is None else np.dtype(dtype)
    if variant == "auto" and all(a.dtype == rhsq.dtype and a.flags.c_contiguous
                                 for a in arrays.values()):
        volume_host(state, c, accumulate=True, compute_dtype=dt, device=device)
        return rhsq
    ds = DeviceFieldState.from_field_state(state, dtype=dt, device=device)
    volume_rhs_device(ds, variant=variant, constants=c or state_constants(state))
    rhsq[...] = ds.rhsq_logical().astype(rhsq.dtype, copy=False)
    return rhsq


def interpret_state(kernels, state: FieldState, nq: int, ne: int,
                    collect_counts: bool = False):
    """Drop-in for ``lf/bench/driver.py:54-69`` with the level-8 fused
    kernel: float32 arrays required (``lf/interp.py:71-72``), rhsq updated
    in place, returns ``(state.rhsq, envs)`` (``envs`` is empty: there is
    no interpreter environment). ``kernels`` is accepted for signature
    compatibility and ignored — the CUDA kernel IS the fused kernel."""
    validate_state(state, nq, ne, dtype=np.float32)
    return volume_rhs_(state, dtype=np.float32), []


def max_rel_error(got: np.ndarray, want: np.ndarray) -> float:
    """Per-field max-norm relative error, worst over fields
    (``lf/bench/driver.py:72-91``)."""
    got64 = np.asarray(got, np.float64)
    want64 = np.asarray(want, np.float64)
    worst = 0.0
    for b in range(want64.shape[3]):
        w = want64[:, :, :, b]
        d = np.abs(got64[:, :, :, b] - w)
        scale = float(np.max(np.abs(w))) if w.size else 0.0
        if scale == 0.0:
            worst = max(worst, float(np.max(d)) if d.size else 0.0)
        else:
            worst = max(worst, float(np.max(d)) / scale)
    return worst
