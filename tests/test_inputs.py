"""The reference-interface mirror of the input API
(pkg/tests/test_bench.py:29-72 behaviours)."""

from __future__ import annotations

import numpy as np
import pytest

from paper_1604_08501_b200 import (BenchmarkConfig, PhysicalConstants,
                                   differentiation_matrix, make_inputs)


def test_deterministic():
    cfg = BenchmarkConfig(nq=3, ne=2, seed=9)
    a, b = make_inputs(cfg), make_inputs(cfg)
    for name in ("q", "rhsq", "D", "g", "Jinv"):
        np.testing.assert_array_equal(a.arrays()[name], b.arrays()[name])


def test_invalid_config_rejected():
    with pytest.raises(ValueError):
        BenchmarkConfig(nq=2, ne=0)
    with pytest.raises(ValueError):
        BenchmarkConfig(nq=0, ne=1)
    with pytest.raises(ValueError):
        BenchmarkConfig(nq=2, ne=1, level=9)


def test_state_invariants():
    st = make_inputs(BenchmarkConfig(nq=4, ne=3, seed=2))
    assert (st.q[:, :, :, 0] > 0).all()
    assert (st.Jinv > 0).all()
    assert (st.q[:, :, :, 4] > 0).all()
    c = st.constants
    p = c.p0 * (c.R * st.q[:, :, :, 4].astype(np.float64) / c.p0) ** c.gamma
    assert 0.5 * c.p0 < p.min() < p.max() < 2 * c.p0


def test_constants_relations():
    c = PhysicalConstants()
    assert c.R == pytest.approx(c.cp - c.cv)
    assert c.gamma == pytest.approx(c.cp / c.cv)
    with pytest.raises(ValueError):
        PhysicalConstants(gamma=0.9)


@pytest.mark.parametrize("nq", [2, 3, 5, 8, 12, 16])
def test_differentiation_matrix_rows_sum_to_zero_exactly(nq):
    d = differentiation_matrix(nq)
    for i in range(nq):
        acc = np.float32(0.0)
        for n in range(nq):
            if n != i:
                acc = np.float32(acc + d[i, n])
        assert np.float32(acc + d[i, i]) == np.float32(0.0)
    assert float(np.abs(d.sum(axis=1)).max()) < 1e-6


def test_state_copy_and_astype():
    st = make_inputs(BenchmarkConfig(nq=2, ne=2, seed=1))
    c = st.copy()
    c.q[0, 0, 0, 0, 0] = 7.0
    assert st.q[0, 0, 0, 0, 0] != 7.0
    s64 = st.astype(np.float64)
    assert s64.q.dtype == np.float64
    np.testing.assert_array_equal(s64.q.astype(np.float32), st.q)
    assert (st.nq, st.ne) == (2, 2)
