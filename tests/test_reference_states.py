"""States built by the UNMODIFIED reference (``loopforge.bench.make_inputs``,
``lf/bench/inputs.py:52-112``) through every public entry point.

The reference's ``FieldState`` has ``arrays()`` and ``constants`` but none of
this package's mirror conveniences (``nq``, ``ne``, ``astype``), so these
tests catch any entry point that reads a mirror-only attribute. The CPU
tests run the host-side logic with a mock device: the native layout
converter is replaced by a numpy axis reversal and the native pipeline by
a recorder, so argument semantics (shapes, pointers, constants, modes) are
checked without a GPU. The ``-m gpu`` tests run the real kernels and compare
with the reference's own ``reference_volume_term`` output.
"""

from __future__ import annotations

import contextlib
import ctypes
import types

import numpy as np
import pytest
import torch

from paper_1604_08501_b200 import (BenchmarkConfig, DeviceFieldState, ExecutionError,
                                   max_rel_error, validate_state)
from paper_1604_08501_b200 import _native, volume as V

from refpkg import loopforge_bench

LB = loopforge_bench()
needs_ref = pytest.mark.skipif(LB is None, reason="reference package not installed")


def ref_state(nq, ne, seed=1, constants=None):
    c = None if constants is None else LB.PhysicalConstants(*constants)
    return LB.make_inputs(LB.BenchmarkConfig(nq=nq, ne=ne, seed=seed), c)


@needs_ref
def test_reference_state_lacks_mirror_attributes():
    st = ref_state(3, 2)
    assert type(st).__module__.startswith("loopforge")
    assert not hasattr(st, "nq") and not hasattr(st, "ne") and not hasattr(st, "astype")


@needs_ref
@pytest.mark.parametrize("nq,ne", [(1, 1), (3, 2), (4, 5), (8, 1)])
def test_validate_state_reads_shapes_from_arrays(nq, ne):
    assert validate_state(ref_state(nq, ne)) == (nq, ne)
    assert validate_state(ref_state(nq, ne), nq, ne, dtype=np.float32) == (nq, ne)
    with pytest.raises(ExecutionError, match="'q'"):
        validate_state(ref_state(nq, ne), nq + 1, ne)
    with pytest.raises(ExecutionError, match="float64"):
        validate_state(ref_state(nq, ne), dtype=np.float64)


@needs_ref
def test_reference_inputs_equal_mirror_inputs():
    from paper_1604_08501_b200 import make_inputs
    a, b = ref_state(5, 3, seed=7), make_inputs(BenchmarkConfig(nq=5, ne=3, seed=7))
    for n in ("q", "rhsq", "D", "g", "Jinv"):
        assert np.array_equal(a.arrays()[n], b.arrays()[n]), n


# ---------------------------------------------------------------- mock device

def _np_view(ptr: int, nbytes: int, count: int) -> np.ndarray:
    dt = np.float64 if nbytes == 8 else np.float32
    buf = (ctypes.c_char * (count * nbytes)).from_address(ptr)
    return np.frombuffer(buf, dtype=dt, count=count)


def _mock_reverse_axes(to_batched, in_bytes, out_bytes, dims, ne, src, dst, stream):
    """numpy stand-in for lfb_field_state_to_element_batched / back: both are
    a full reversal of the axes (include/lfb_volume.h), with a cast."""
    dims = tuple(int(d) for d in dims)
    n = int(np.prod(dims, dtype=np.int64)) * int(ne)
    x = _np_view(src, in_bytes, n)
    shape = dims + (ne,) if to_batched else (ne,) + tuple(reversed(dims))
    y = np.transpose(x.reshape(shape))
    _np_view(dst, out_bytes, n)[...] = y.reshape(-1)


@pytest.fixture
def mock_device(monkeypatch):
    cpu = torch.device("cpu")
    monkeypatch.setattr(V, "_device", lambda device=None: cpu)
    monkeypatch.setattr(torch.cuda, "device", lambda d: contextlib.nullcontext())
    monkeypatch.setattr(torch.cuda, "current_stream",
                        lambda d=None: types.SimpleNamespace(cuda_stream=0))
    monkeypatch.setattr(_native, "reverse_axes_ptr", _mock_reverse_axes)
    calls = []

    class FakePipeline:
        chunk = 1

        def run(self, mode, ne, p0, R, gam, q, D, g, jinv, out, stream=0):
            calls.append(dict(mode=mode, ne=ne, p0=p0, R=R, gam=gam, q=q, D=D, g=g,
                              jinv=jinv, out=out))

    monkeypatch.setattr(V, "host_pipeline", lambda *a, **k: FakePipeline())
    return calls


@needs_ref
@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_from_field_state_accepts_reference_state(mock_device, dtype):
    st = ref_state(4, 3, seed=2, constants=(9.0e4, 280.0, 1.3))
    ds = DeviceFieldState.from_field_state(st, dtype=dtype)
    npdt = np.float64 if dtype == torch.float64 else np.float32
    assert (ds.nq, ds.ne) == (4, 3) and ds.dtype == dtype
    assert np.array_equal(ds.q.numpy(), np.transpose(st.q).astype(npdt))
    assert np.array_equal(ds.g.numpy(), np.transpose(st.g).astype(npdt))
    assert np.array_equal(ds.Jinv.numpy(), np.transpose(st.Jinv).astype(npdt))
    assert np.array_equal(ds.D.numpy(), st.D.T.astype(npdt))
    assert ds.constants.p0 == 9.0e4 and ds.constants.gamma == 1.3
    # and back to the reference layout
    assert np.array_equal(DeviceFieldState.to_logical(ds.q), st.q.astype(npdt))


@needs_ref
def test_volume_host_binds_reference_arrays(mock_device):
    st = ref_state(3, 4, seed=5, constants=(1.1e5, 290.0, 1.5))
    out = V.volume_host(st, compute_dtype=np.float64)
    (call,) = mock_device
    assert call["mode"] == _native.HOST_INCREMENT and call["ne"] == 4
    assert (call["p0"], call["R"], call["gam"]) == (1.1e5, 290.0, 1.5)
    assert call["q"] == st.q.ctypes.data and call["D"] == st.D.ctypes.data
    assert call["g"] == st.g.ctypes.data and call["jinv"] == st.Jinv.ctypes.data
    assert call["out"] == out.ctypes.data and out.shape == st.q.shape
    mock_device.clear()
    assert V.volume_host(st, accumulate=True) is st.rhsq
    assert mock_device[0]["mode"] == _native.HOST_ACCUMULATE
    assert mock_device[0]["out"] == st.rhsq.ctypes.data
    # validation paths raise the reference's exception type
    st.g = st.g.astype(np.float64)
    with pytest.raises(ExecutionError, match="one dtype"):
        V.volume_host(st)


@needs_ref
def test_public_entry_points_accept_reference_state(mock_device, monkeypatch):
    """reference_volume_term / volume_rhs_ / interpret_state route f32
    reference states to the host pipeline; volume_term and a forced variant
    go through from_field_state + the device call (recorded here)."""
    launched = []
    monkeypatch.setattr(V, "volume_rhs_device",
                        lambda ds, variant="auto", stream=None, constants=None:
                        launched.append((ds.nq, ds.ne, variant, constants)))
    st = ref_state(2, 3)
    V.reference_volume_term(st)
    assert mock_device[-1]["mode"] == _native.HOST_INCREMENT
    assert V.volume_rhs_(st) is st.rhsq
    assert mock_device[-1]["mode"] == _native.HOST_ACCUMULATE
    rhsq, envs = V.interpret_state([], st, 2, 3)
    assert rhsq is st.rhsq and envs == []
    with pytest.raises(ExecutionError):
        V.interpret_state([], st, 3, 3)
    v = V.volume_term(st, dtype=np.float64)
    assert v.shape == st.q.shape and launched[-1][:3] == (2, 3, "auto")
    assert launched[-1][3] is st.constants
    V.volume_rhs_(st, variant="tc")
    assert launched[-1][:3] == (2, 3, "tc")
    # non-f32 reference-shaped state: the device route of reference_volume_term
    st64 = ref_state(2, 3)
    for n in ("q", "rhsq", "D", "g", "Jinv"):
        setattr(st64, n, getattr(st64, n).astype(np.float64))
    V.reference_volume_term(st64)
    assert launched[-1][:2] == (2, 3)
    f64 = ref_state(2, 3)
    f64.q = f64.q.astype(np.float64)
    with pytest.raises(ExecutionError, match="float32"):
        V.interpret_state([], f64, 2, 3)


# ---------------------------------------------------------------------- GPU

@needs_ref
@pytest.mark.gpu
@pytest.mark.parametrize("nq,ne,seed", [(4, 512, 1), (8, 9, 3), (5, 7, 2), (11, 2, 4)])
def test_reference_states_on_gpu_match_reference_output(cuda_device, nq, ne, seed):
    """The reference's own make_inputs state through every public entry
    point on the GPU, against the reference's own reference_volume_term
    (f32, fp64 accumulation; one f32 rounding ulp apart at most)."""
    from paper_1604_08501_b200 import (interpret_state, reference_volume_term,
                                       volume_rhs_, volume_term)
    st = ref_state(nq, ne, seed)
    want = LB.reference_volume_term(st)
    got = reference_volume_term(st)
    np.testing.assert_array_max_ulp(got, want, maxulp=1)
    assert np.all(st.rhsq == 0)
    for variant in ("auto", "col", "basic"):
        if not _native.variant_available(variant, 8, nq):
            continue
        assert max_rel_error(volume_term(st, dtype=np.float64, variant=variant),
                             want) <= 1e-7, variant
    ds = DeviceFieldState.from_field_state(st, dtype=torch.float64)
    assert (ds.nq, ds.ne) == (nq, ne)
    st2 = ref_state(nq, ne, seed)
    volume_rhs_(st2, variant="auto")
    assert max_rel_error(st2.rhsq, want) <= 1e-5
    st3 = ref_state(nq, ne, seed)
    rhsq, _ = interpret_state(None, st3, nq, ne)
    assert rhsq is st3.rhsq and max_rel_error(rhsq, want) <= 1e-5
