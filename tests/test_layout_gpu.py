"""Native layout conversion (FieldState C-order <-> element-batched) and
device-side input generation."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import coracle, volterm as O
from paper_1604_08501_b200 import (BenchmarkConfig, DeviceFieldState, make_inputs,
                                   max_rel_error, volume_rhs_device)
from paper_1604_08501_b200 import _native
from paper_1604_08501_b200.distributed import shard_range

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("nq,ne", [(1, 5), (2, 3), (3, 33), (8, 7), (12, 2)])
@pytest.mark.parametrize("out_dtype", [torch.float32, torch.float64])
def test_from_field_state_matches_numpy_transpose(cuda_device, nq, ne, out_dtype):
    st = make_inputs(BenchmarkConfig(nq=nq, ne=ne, seed=3))
    ds = DeviceFieldState.from_field_state(st, dtype=out_dtype)
    q, g, j, d = coracle.to_element_batched(st)  # independent numpy layout
    np_dt = np.float32 if out_dtype == torch.float32 else np.float64
    for got, want in ((ds.q, q), (ds.g, g), (ds.Jinv, j), (ds.D, d)):
        np.testing.assert_array_equal(got.cpu().numpy(), want.astype(np_dt))


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_round_trip_is_exact(cuda_device, dtype):
    st = make_inputs(BenchmarkConfig(nq=5, ne=19, seed=4)).astype(dtype)
    st.rhsq[...] = np.random.default_rng(1).normal(size=st.rhsq.shape)
    ds = DeviceFieldState.from_field_state(st, dtype=dtype)
    back = ds.to_field_state()
    for name in ("q", "rhsq", "D", "g", "Jinv"):
        np.testing.assert_array_equal(back.arrays()[name], st.arrays()[name])


def test_layout_validation_codes(cuda_device):
    x = torch.zeros(8, device=cuda_device, dtype=torch.float64)
    with pytest.raises(Exception, match="Nq|dims"):
        _native.reverse_axes_ptr(True, 8, 8, (), 1, x.data_ptr(), x.data_ptr(), 0)
    with pytest.raises(Exception, match="aligned"):
        _native.reverse_axes_ptr(True, 8, 8, (2,), 2, x.data_ptr() + 4, x.data_ptr(), 0)


def test_device_inputs_distributions_and_invariants(cuda_device):
    ds = DeviceFieldState.generate(8, 2000, seed=5)
    q = ds.q.cpu().numpy()
    assert (ds.rhsq == 0).all()
    rho, U, th, tr = q[:, 0], q[:, 1:4], q[:, 4], q[:, 5:8]
    assert 0.5 <= rho.min() and rho.max() < 1.5 and abs(rho.mean() - 1.0) < 0.01
    assert -0.1 <= U.min() and U.max() < 0.1 and abs(U.mean()) < 0.002
    p0R = 1.0e5 / 287.0
    assert 0.9 * p0R * (1 - 1e-7) <= th.min() and th.max() < 1.1 * p0R * (1 + 1e-7)
    assert 0.0 <= tr.min() and tr.max() < 1.0 and abs(tr.mean() - 0.5) < 0.01
    g = ds.g.cpu().numpy()
    assert -1.0 <= g.min() and g.max() < 1.0 and abs(g.mean()) < 0.01
    J = ds.Jinv.cpu().numpy()
    assert 0.5 <= J.min() and J.max() < 2.0
    # values are f32-representable, like the reference's f32 arrays
    np.testing.assert_array_equal(q, q.astype(np.float32).astype(np.float64))
    np.testing.assert_array_equal(ds.D.cpu().numpy().T,
                                  make_inputs(BenchmarkConfig(8, 1)).D.astype(np.float64))


def test_device_inputs_shards_reproduce_the_whole_state(cuda_device):
    whole = DeviceFieldState.generate(4, 101, seed=9, dtype=torch.float32)
    for r in range(3):
        a, b = shard_range(101, r, 3)
        part = DeviceFieldState.generate(4, b - a, seed=9, dtype=torch.float32, e_offset=a)
        assert torch.equal(part.q, whole.q[a:b])
        assert torch.equal(part.g, whole.g[a:b])
        assert torch.equal(part.Jinv, whole.Jinv[a:b])
    other = DeviceFieldState.generate(4, 101, seed=10, dtype=torch.float32)
    assert not torch.equal(other.q, whole.q)


def test_parity_on_device_generated_state_sampled_elements(cuda_device):
    """Config-3-style check: device-generated inputs, parity on sampled
    elements against the oracle (elements are independent)."""
    ds = DeviceFieldState.generate(8, 4096, seed=2)
    volume_rhs_device(ds)
    torch.cuda.synchronize()
    idx = torch.tensor(sorted(np.random.default_rng(0).choice(4096, 64, replace=False)),
                       device=cuda_device)
    sub = DeviceFieldState(ds.q[idx].contiguous(), torch.zeros_like(ds.rhsq[idx]),
                           ds.D, ds.g[idx].contiguous(), ds.Jinv[idx].contiguous(),
                           ds.constants)
    st = sub.to_field_state()
    want = O.volume_term_f64_batched(st)
    got = DeviceFieldState.to_logical(ds.rhsq[idx].contiguous())
    assert max_rel_error(got, want) <= 1e-12
