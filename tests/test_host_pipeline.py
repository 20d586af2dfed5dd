"""The native host-buffer pipeline (``lfb_volume_host``): the reference's
entry points over HOST arrays in the reference's C-order layout —
``reference_volume_term`` (``lf/bench/reference.py:36-70``, INCREMENT) and
``rhsq += v`` (``lf/bench/driver.py:54-69``, ACCUMULATE) — chunked over
elements, 2-D copies, on-device layout conversion, overlapped streams.

CPU tests cover the argument validation that happens before any CUDA call;
``-m gpu`` tests check every chunking (one chunk, many, ragged last chunk,
chunk = 1) against the oracle."""

from __future__ import annotations

import ctypes

import numpy as np
import pytest

from oracle import volterm as O
from paper_1604_08501_b200 import (BenchmarkConfig, ExecutionError, FieldState, make_inputs,
                                   max_rel_error, reference_volume_term, volume_rhs_)
from paper_1604_08501_b200 import _native
from paper_1604_08501_b200.volume import pipeline_chunk, volume_host

TOL64 = 1e-12
TOL32 = 1e-5


# ---------------------------------------------------------------- CPU only --

def test_create_validation_codes_before_any_cuda_call():
    L = _native.lib()
    h = ctypes.c_void_p()
    assert L.lfb_pipeline_create(8, 16, 4, 8, -1, None) == _native.LFB_ERR_NULL
    assert L.lfb_pipeline_create(0, 16, 4, 8, -1, ctypes.byref(h)) == _native.LFB_ERR_BAD_NQ
    assert L.lfb_pipeline_create(17, 16, 4, 8, -1, ctypes.byref(h)) == _native.LFB_ERR_BAD_NQ
    assert L.lfb_pipeline_create(8, 0, 4, 8, -1, ctypes.byref(h)) == _native.LFB_ERR_BAD_NE
    assert L.lfb_pipeline_create(8, 16, 2, 8, -1, ctypes.byref(h)) == \
        _native.LFB_ERR_BAD_VARIANT
    assert h.value is None


def test_run_validation_codes():
    L = _native.lib()
    p = 4096
    assert L.lfb_volume_host(None, 0, 1, 1e5, 287.0, 1.4, p, p, p, p, p, None) == \
        _native.LFB_ERR_NULL
    assert L.lfb_pipeline_destroy(None) == 0
    assert L.lfb_pipeline_info(None, None, None) == _native.LFB_ERR_NULL


def test_default_chunking():
    # Nq=8, f32 host / f64 compute: 2048 elements per 320 MiB slot
    assert pipeline_chunk(8, 32768, 4, 8) == 2048
    assert pipeline_chunk(8, 100, 4, 8) == 100
    assert pipeline_chunk(16, 10 ** 6, 8, 8) >= 1


# ---------------------------------------------------------------- GPU -------

@pytest.mark.gpu
@pytest.mark.parametrize("nq,ne,chunk", [(8, 37, 37), (8, 37, 10), (8, 37, 1), (4, 1000, 333),
                                         (5, 41, 7), (2, 130, 64), (12, 7, 3), (3, 50, 16)])
def test_increment_matches_oracle_all_chunkings(cuda_device, nq, ne, chunk):
    st = make_inputs(BenchmarkConfig(nq=nq, ne=ne, seed=nq + ne))
    rhsq0 = st.rhsq.copy()
    want = O.volume_term_f64_batched(st)
    got = volume_host(st, compute_dtype=np.float64, chunk=chunk)
    assert got.dtype == np.float32 and got.shape == want.shape
    assert np.array_equal(st.rhsq, rhsq0)  # increment mode leaves rhsq alone
    # f64 compute, f32 result: the reference's own cast bounds the error
    assert max_rel_error(got, want) <= 1e-7
    got32 = volume_host(st, compute_dtype=np.float32, chunk=chunk)
    assert max_rel_error(got32, want) <= TOL32


@pytest.mark.gpu
def test_reference_volume_term_is_bit_compatible_with_fixtures(cuda_device, golden,
                                                               golden_meta):
    for nq, ne, seed in golden_meta["full"]:
        st = make_inputs(BenchmarkConfig(nq=nq, ne=ne, seed=seed))
        got = reference_volume_term(st)  # routes through the host pipeline
        np.testing.assert_array_max_ulp(got, golden[f"ref_{nq}_{ne}_{seed}"], maxulp=1)


@pytest.mark.gpu
@pytest.mark.parametrize("dtype,tol", [(np.float64, TOL64), (np.float32, TOL32)])
def test_accumulate_mode_and_f64_host_arrays(cuda_device, dtype, tol):
    st = make_inputs(BenchmarkConfig(nq=6, ne=29, seed=3)).astype(dtype)
    st.rhsq[...] = np.random.default_rng(1).uniform(-1e3, 1e3, st.rhsq.shape)
    base = st.rhsq.astype(np.float64)
    want = base + O.volume_term_f64_batched(st)
    out = volume_host(st, accumulate=True, compute_dtype=dtype, chunk=8)
    assert out is st.rhsq
    assert max_rel_error(st.rhsq, want) <= tol
    # the public in-place entry point takes the same path
    st2 = make_inputs(BenchmarkConfig(nq=6, ne=29, seed=3)).astype(dtype)
    st2.rhsq[...] = base
    volume_rhs_(st2)
    assert max_rel_error(st2.rhsq, want) <= tol


@pytest.mark.gpu
def test_full_config2_increment_pinned(cuda_device):
    """BASELINE config 2 through the e2e path (pinned buffers, default
    chunking = 16 chunks over 3 streams), checked on a sampled subset of
    elements against the oracle and in full for finiteness."""
    import torch
    st = make_inputs(BenchmarkConfig(nq=8, ne=32768, seed=1))
    out = torch.empty(st.q.shape, dtype=torch.float32).pin_memory().numpy()
    volume_host(st, out=out)
    assert np.isfinite(out).all()
    idx = np.random.default_rng(0).choice(32768, 96, replace=False)
    c = np.ascontiguousarray
    sub = FieldState(c(st.q[..., idx]), c(st.rhsq[..., idx]), st.D, c(st.g[..., idx]),
                     c(st.Jinv[..., idx]), st.constants)
    assert max_rel_error(out[..., idx], O.volume_term_f64_batched(sub)) <= 1e-7


@pytest.mark.gpu
def test_mixed_dtypes_rejected(cuda_device):
    st = make_inputs(BenchmarkConfig(nq=2, ne=2, seed=1))
    st.g = st.g.astype(np.float64)
    with pytest.raises(ExecutionError, match="one dtype"):
        volume_host(st)
    # the public drop-in still works (device path)
    want = O.volume_term_f64_batched(st)
    assert max_rel_error(reference_volume_term(st), want) <= 1e-7
