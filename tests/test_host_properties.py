"""Property tests (hypothesis) of the host-side logic that needs no GPU:
argument validation with the reference's error behaviour
(``lf/interp.py:51-74``), element sharding, host-pipeline chunking, the
logical<->element-batched layout map, and the emitted-text parser."""

from __future__ import annotations

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from paper_1604_08501_b200 import (BenchmarkConfig, ExecutionError, FieldState,
                                   make_inputs, validate_state)
from paper_1604_08501_b200.distributed import shard_range
from paper_1604_08501_b200.volume import pipeline_chunk


@settings(max_examples=200, deadline=None)
@given(ne=st.integers(0, 10 ** 7), world=st.integers(1, 64))
def test_shards_tile_the_element_range(ne, world):
    spans = [shard_range(ne, r, world) for r in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == ne
    assert all(a <= b for a, b in spans)
    assert all(s[1] == t[0] for s, t in zip(spans, spans[1:]))
    sizes = [b - a for a, b in spans]
    assert max(sizes) - min(sizes) <= 1


@settings(max_examples=200, deadline=None)
@given(nq=st.integers(1, 16), ne=st.integers(1, 10 ** 6),
       hb=st.sampled_from([4, 8]), cb=st.sampled_from([4, 8]),
       slot=st.integers(1 << 10, 1 << 32))
def test_pipeline_chunk_is_a_power_of_two_that_fits(nq, ne, hb, cb, slot):
    c = pipeline_chunk(nq, ne, hb, cb, slot)
    assert 1 <= c <= ne
    per_elem = 26 * nq ** 3 * (hb + cb)
    if c < ne:
        assert c & (c - 1) == 0           # power of two
        assert c == 1 or c * per_elem <= slot


@settings(max_examples=60, deadline=None)
@given(nq=st.integers(1, 5), ne=st.integers(1, 4))
def test_element_batched_layout_is_the_full_axis_reversal(nq, ne):
    """The C-ABI layout [e][field][k][j][i] is the reversal of the
    reference's C-order (i, j, k, field, e) — the map DeviceFieldState and
    the native layout kernels implement (lf/bench/data/volume.f90:14-18)."""
    st_ = make_inputs(BenchmarkConfig(nq=nq, ne=ne, seed=nq * 7 + ne))
    eb = np.ascontiguousarray(st_.q.transpose(4, 3, 2, 1, 0))
    for e in range(ne):
        for b in range(8):
            for k in range(nq):
                for j in range(nq):
                    for i in range(nq):
                        assert eb[e, b, k, j, i] == st_.q[i, j, k, b, e]
    flat = eb.reshape(-1)
    i, j, k, b, e = (nq - 1, 0, nq // 2, 5, ne - 1)
    assert flat[(((e * 8 + b) * nq + k) * nq + j) * nq + i] == st_.q[i, j, k, b, e]


@settings(max_examples=100, deadline=None)
@given(nq=st.integers(1, 6), ne=st.integers(1, 3),
       which=st.sampled_from(["q", "rhsq", "D", "g", "Jinv"]),
       fault=st.sampled_from(["shape", "dtype", "missing"]))
def test_validation_rejects_like_the_interpreter(nq, ne, which, fault):
    st_ = make_inputs(BenchmarkConfig(nq=nq, ne=ne, seed=1))
    arrays = st_.arrays()
    a = arrays[which]
    if fault == "shape":
        arrays[which] = np.zeros(a.shape[:-1] + (a.shape[-1] + 1,), a.dtype)
    elif fault == "dtype":
        arrays[which] = a.astype(np.int32)
    else:
        arrays[which] = None
    bad = FieldState(arrays["q"], arrays["rhsq"], arrays["D"], arrays["g"], arrays["Jinv"],
                     st_.constants)
    with pytest.raises(ExecutionError):
        validate_state(bad)


def test_validation_accepts_every_reference_state():
    for nq in range(1, 9):
        st_ = make_inputs(BenchmarkConfig(nq=nq, ne=2, seed=nq))
        assert validate_state(st_) == (nq, 2)


@settings(max_examples=50, deadline=None)
@given(junk=st.text(max_size=200))
def test_emitted_parser_rejects_non_kernels(junk):
    from paper_1604_08501_b200.emitted import EmittedKernel
    if "KERNEL" in junk:
        return
    with pytest.raises(ExecutionError):
        EmittedKernel(junk)
