"""Parity of the CUDA volume kernel (through the C-ABI) with the pinned
oracle. Tolerances (per-field max-norm relative error,
lf/bench/driver.py:72-91): fp64 <= 1e-12, fp32 <= 1e-5
(pkg/tests/test_acceptance.py:42)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import coracle, volterm as O
from paper_1604_08501_b200 import (BenchmarkConfig, DeviceFieldState,
                                   ExecutionError, interpret_state,
                                   make_inputs, max_rel_error,
                                   reference_volume_term, volume_rhs_,
                                   volume_rhs_device, volume_term)
from paper_1604_08501_b200 import _native

pytestmark = pytest.mark.gpu

TOL64 = 1e-12
TOL32 = 1e-5

SMALL = [(1, 3, 1), (2, 1, 42), (2, 5, 2), (2, 130, 3), (3, 2, 3), (3, 33, 4), (4, 5, 3),
         (4, 37, 5), (4, 8, 2),
         (4, 17, 6), (5, 3, 4), (6, 7, 7), (7, 2, 8), (8, 3, 1), (8, 13, 9),
         (9, 2, 2), (10, 2, 3), (11, 1, 4), (12, 3, 5), (13, 1, 6), (16, 2, 7)]


def _variants(nbytes, nq):
    return [v for v in ("basic", "fused", "tc", "lines", "col", "lt", "ltu", "lo")
            if _native.variant_available(v, nbytes, nq)]


@pytest.mark.parametrize("nq,ne,seed", SMALL)
def test_fp64_parity_all_variants(cuda_device, nq, ne, seed):
    st = make_inputs(BenchmarkConfig(nq=nq, ne=ne, seed=seed))
    want = O.volume_term_f64_batched(st)
    for v in _variants(8, nq) + ["auto"]:
        got = volume_term(st, dtype=np.float64, device=cuda_device, variant=v)
        err = max_rel_error(got, want)
        assert err <= TOL64, (v, err)


@pytest.mark.parametrize("nq,ne,seed", SMALL)
def test_fp32_parity_all_variants(cuda_device, nq, ne, seed):
    st = make_inputs(BenchmarkConfig(nq=nq, ne=ne, seed=seed))
    want = O.volume_term_f64_batched(st)
    for v in _variants(4, nq) + ["auto"]:
        got = volume_term(st, dtype=np.float32, device=cuda_device, variant=v)
        assert got.dtype == np.float32
        err = max_rel_error(got, want)
        assert err <= TOL32, (v, err)


def test_reference_fixtures(cuda_device, golden, golden_meta):
    """Every reference-generated f32 output (tests/golden/make_golden.py)."""
    for nq, ne, seed in golden_meta["full"]:
        st = make_inputs(BenchmarkConfig(nq=nq, ne=ne, seed=seed))
        got = reference_volume_term(st)
        want = golden[f"ref_{nq}_{ne}_{seed}"]
        assert got.dtype == np.float32 and got.shape == want.shape
        # f64 on both sides, cast to f32: equal up to a rounding-boundary ulp
        np.testing.assert_array_max_ulp(got, want, maxulp=1)
        assert max_rel_error(got, want) <= 1e-7


def test_reference_golden_vector(cuda_device, golden, golden_meta):
    cfg = golden_meta["volterm_nq2_ne1_seed42_config"]
    st = make_inputs(BenchmarkConfig(nq=cfg["nq"], ne=cfg["ne"], seed=cfg["seed"]))
    got = volume_term(st, dtype=np.float64)
    want32 = golden["volterm_nq2_ne1_seed42"].reshape(got.shape)
    np.testing.assert_array_max_ulp(got.astype(np.float32), want32, maxulp=1)
    assert max_rel_error(got, O.volume_term_f64(st)) <= TOL64


def test_interpret_state_adapter_matches_reference_interpreter(cuda_device, golden,
                                                               golden_meta):
    """The reference's fused level-8 kernel executed by its interpreter
    (f32) vs ours through the interpret_state-compatible adapter."""
    for nq, ne, seed in golden_meta["interp8"]:
        st = make_inputs(BenchmarkConfig(nq=nq, ne=ne, seed=seed))
        want_oracle = O.volume_term_f64(st)
        got, envs = interpret_state(None, st, nq, ne)
        assert got is st.rhsq and envs == []
        assert max_rel_error(got, golden[f"interp8_{nq}_{ne}_{seed}"]) <= TOL32
        assert max_rel_error(got, want_oracle) <= TOL32


def test_interpret_state_rejects_f64_like_reference(cuda_device):
    st = make_inputs(BenchmarkConfig(nq=2, ne=1, seed=1)).astype(np.float64)
    with pytest.raises(ExecutionError, match="float32"):
        interpret_state(None, st, 2, 1)
    st32 = make_inputs(BenchmarkConfig(nq=2, ne=1, seed=1))
    with pytest.raises(ExecutionError, match="shape"):
        interpret_state(None, st32, 2, 3)


@pytest.mark.parametrize("dtype,tol", [(np.float64, TOL64), (np.float32, TOL32)])
def test_in_place_accumulate_semantics(cuda_device, dtype, tol):
    st = make_inputs(BenchmarkConfig(nq=4, ne=9, seed=11)).astype(dtype)
    rng = np.random.default_rng(0)
    st.rhsq[...] = rng.uniform(-1e4, 1e4, st.rhsq.shape).astype(dtype)
    rhsq0 = st.rhsq.astype(np.float64).copy()
    v = O.volume_term_f64_batched(st)
    out = volume_rhs_(st)
    assert out is st.rhsq
    assert max_rel_error(st.rhsq, rhsq0 + v) <= tol


def test_zero_D_gives_exact_zero(cuda_device):
    for dtype in (np.float64, np.float32):
        st = make_inputs(BenchmarkConfig(nq=3, ne=4, seed=5))
        st.D[:] = 0.0
        for v in _variants(np.dtype(dtype).itemsize, 3):
            assert np.all(volume_term(st, dtype=dtype, variant=v) == 0.0)


def test_telescoping_constant_fields(cuda_device):
    st = make_inputs(BenchmarkConfig(nq=4, ne=2, seed=6))
    st.q[:] = st.q[0, 0, 0, :, 0][None, None, None, :, None]
    st.g[:] = st.g[0, 0, 0, :, :, 0][None, None, None, :, :, None]
    for v in _variants(8, 4):
        out = volume_term(st, dtype=np.float64, variant=v)
        assert np.abs(out).max() / st.constants.p0 < 1e-6


def test_custom_constants(cuda_device):
    from paper_1604_08501_b200 import PhysicalConstants
    c = PhysicalConstants(p0=9.0e4, R=300.0, gamma=1.3)
    st = make_inputs(BenchmarkConfig(nq=5, ne=3, seed=2), constants=c)
    want = O.volume_term_f64_batched(st)
    assert max_rel_error(volume_term(st, dtype=np.float64), want) <= TOL64
    # explicit c overrides the state's constants, like the reference
    other = PhysicalConstants(p0=1.1e5, R=280.0, gamma=1.45)
    want2 = O.volume_term_f64_batched(st, other)
    assert max_rel_error(volume_term(st, other, dtype=np.float64), want2) <= TOL64


def test_repeated_launches_accumulate_linearly(cuda_device):
    st = make_inputs(BenchmarkConfig(nq=8, ne=37, seed=3))
    ds = DeviceFieldState.from_field_state(st, dtype=torch.float64)
    volume_rhs_device(ds)
    one = ds.rhsq.clone()
    for _ in range(3):
        volume_rhs_device(ds)
    torch.cuda.synchronize()
    rel = (ds.rhsq - 4 * one).abs().max() / one.abs().max()
    assert float(rel) <= 1e-14


def test_sharded_launches_equal_whole_launch_bitwise(cuda_device):
    """Element sharding (the multi-GPU decomposition) is bit-exact."""
    st = make_inputs(BenchmarkConfig(nq=8, ne=50, seed=4))
    whole = DeviceFieldState.from_field_state(st, dtype=torch.float64)
    volume_rhs_device(whole)
    parts = DeviceFieldState.from_field_state(st, dtype=torch.float64)
    from paper_1604_08501_b200.distributed import shard_range
    for r in range(3):
        a, b = shard_range(50, r, 3)
        volume_rhs_device(parts.shard(a, b))
    torch.cuda.synchronize()
    assert torch.equal(whole.rhsq, parts.rhsq)


def test_device_api_validation(cuda_device):
    st = make_inputs(BenchmarkConfig(nq=4, ne=3, seed=1))
    ds = DeviceFieldState.from_field_state(st, dtype=torch.float64)
    bad = DeviceFieldState(ds.q, ds.rhsq, ds.D, ds.g[:, :2].contiguous(), ds.Jinv,
                           ds.constants)
    with pytest.raises(ExecutionError, match="'g'"):
        volume_rhs_device(bad)
    bad = DeviceFieldState(ds.q, ds.rhsq.float(), ds.D, ds.g, ds.Jinv, ds.constants)
    with pytest.raises(ExecutionError, match="'rhsq'"):
        volume_rhs_device(bad)
    with pytest.raises(ExecutionError):
        volume_rhs_device(ds, variant="nope")


def test_misaligned_pointer_is_rejected(cuda_device):
    st = make_inputs(BenchmarkConfig(nq=2, ne=2, seed=1))
    ds = DeviceFieldState.from_field_state(st, dtype=torch.float64)
    with pytest.raises(ExecutionError, match="aligned"):
        _native.volume_rhs_ptr(8, "auto", 2, 2, 1e5, 287.0, 1.4,
                               ds.q.data_ptr() + 4, ds.rhsq.data_ptr(),
                               ds.D.data_ptr(), ds.g.data_ptr(),
                               ds.Jinv.data_ptr(), 0)


@pytest.mark.parametrize("dtype,tol", [(torch.float64, TOL64), (torch.float32, TOL32)])
def test_full_size_config2_against_c_oracle(cuda_device, dtype, tol):
    """BASELINE config 2 (Nq=8, Ne=32768) in full against the C oracle;
    every element is checked."""
    st = make_inputs(BenchmarkConfig(nq=8, ne=32768, seed=1))
    ds = DeviceFieldState.from_field_state(st, dtype=dtype)
    volume_rhs_device(ds)
    got = ds.rhsq.to(torch.float64).cpu().numpy()
    q, g, j, d = coracle.to_element_batched(st)
    want = coracle.volume_f64_eb(8, q, g, j, d, st.constants)
    err = max_rel_error(coracle.from_element_batched(got),
                        coracle.from_element_batched(want))
    assert err <= tol, err


@pytest.mark.parametrize("nq", [8, 7, 2])
def test_tc_needs_16_byte_alignment_and_auto_falls_back(cuda_device, nq):
    """The TMA/DMMA kernel moves 16-byte pairs; AUTO must still accept any
    8-byte aligned arrays (it then takes the column kernel)."""
    if not _native.variant_available("tc", 8, 8):
        pytest.skip("no tc kernel")
    st = make_inputs(BenchmarkConfig(nq=nq, ne=9, seed=12))
    want = O.volume_term_f64_batched(st)
    ds = DeviceFieldState.from_field_state(st, dtype=torch.float64)
    # shift every array by one double inside a bigger buffer
    def shifted(t):
        buf = torch.zeros(t.numel() + 1, dtype=t.dtype, device=t.device)
        v = buf[1:].view(t.shape)
        v.copy_(t)
        return v
    sh = DeviceFieldState(shifted(ds.q), shifted(ds.rhsq), ds.D, shifted(ds.g),
                          shifted(ds.Jinv), ds.constants)
    with pytest.raises(ExecutionError, match="aligned"):
        volume_rhs_device(sh, variant="tc")
    volume_rhs_device(sh, variant="auto")
    torch.cuda.synchronize()
    got = DeviceFieldState.to_logical(sh.rhsq)
    assert max_rel_error(got, want) <= TOL64


@pytest.mark.parametrize("nq,ne", [(4, 8 * 300 + 3), (2, 64 * 20 + 17), (5, 201), (6, 302),
                                   (7, 151), (9, 333), (12, 160), (13, 40)])
@pytest.mark.parametrize("dtype,tol", [(torch.float64, TOL64), (torch.float32, TOL32)])
def test_packed_tc_groups_and_tail_against_c_oracle(cuda_device, nq, ne, dtype, tol):
    """Nq = 4 / 2 run as packed virtual Nq=8 elements (blockdiag D), Nq =
    5..7 as zero-padded ones (odd Nq: unaligned g slabs via 16-byte
    superset copies), plus a fused/basic tail; Nq >= 9 through the line-GEMM
    kernel; every element against the C oracle."""
    st = make_inputs(BenchmarkConfig(nq=nq, ne=ne, seed=8))
    ds = DeviceFieldState.from_field_state(st, dtype=dtype)
    volume_rhs_device(ds, variant="tc" if nq <= 8 else "lines")
    got = ds.rhsq.to(torch.float64).cpu().numpy()
    q, g, j, d = coracle.to_element_batched(st)
    want = coracle.volume_f64_eb(nq, q, g, j, d, st.constants)
    err = max_rel_error(coracle.from_element_batched(got), coracle.from_element_batched(want))
    assert err <= tol, err


@pytest.mark.parametrize("dtype,tol", [(torch.float64, TOL64), (torch.float32, TOL32)])
def test_config3_full_size_properties(cuda_device, dtype, tol):
    """BASELINE config 3/4 size (Nq=8, Ne=262144; 36.5 GB at fp64) on one
    GPU through size-independent properties: the whole launch equals the
    4-way element-sharded launches bit for bit (the multi-GPU decomposition),
    a second launch doubles the increment (linearity), and 128 sampled
    elements match the C oracle."""
    from paper_1604_08501_b200.distributed import shard_range
    nq, ne = 8, 262144
    ds = DeviceFieldState.generate(nq, ne, seed=5, dtype=dtype)
    volume_rhs_device(ds)
    whole = ds.rhsq.clone()
    ds.rhsq.zero_()
    for r in range(4):
        a, b = shard_range(ne, r, 4)
        volume_rhs_device(ds.shard(a, b))
    torch.cuda.synchronize()
    assert torch.equal(whole, ds.rhsq)
    volume_rhs_device(ds)
    torch.cuda.synchronize()
    lin = float(((ds.rhsq - 2 * whole).abs().max() / whole.abs().max()))
    assert lin <= (1e-14 if dtype == torch.float64 else 1e-6), lin
    idx = torch.randperm(ne, generator=torch.Generator().manual_seed(0))[:128].sort().values
    cpu = lambda t: t[idx.to(t.device)].to(torch.float64).cpu().numpy()
    q, g, j, d = cpu(ds.q), cpu(ds.g), cpu(ds.Jinv), ds.D.to(torch.float64).cpu().numpy()
    want = coracle.volume_f64_eb(nq, q, g, j, d, ds.constants)
    got = cpu(whole)
    err = max_rel_error(coracle.from_element_batched(got), coracle.from_element_batched(want))
    assert err <= tol, err
    del ds, whole
    torch.cuda.empty_cache()


@pytest.mark.parametrize("nq,ne", [(8, 40), (4, 24), (2, 70), (7, 6), (5, 9), (6, 5), (9, 3),
                                   (12, 2), (3, 11), (16, 1)])
def test_arbitrary_differentiation_matrix(cuda_device, nq, ne):
    """D is an input (lf/codegen.py:361-373), not necessarily the corpus'
    (n-i)/Nq matrix: a dense random D (not exactly representable in TF32,
    so the fp32 tensor-core path needs all three split products) through
    every variant, fp64 <= 1e-12 and fp32 <= 1e-5."""
    st = make_inputs(BenchmarkConfig(nq=nq, ne=ne, seed=nq + 100))
    rng = np.random.default_rng(nq)
    st.D[...] = rng.uniform(-1.0, 1.0, st.D.shape).astype(st.D.dtype)
    want = O.volume_term_f64_batched(st)
    for v in _variants(8, nq) + ["auto"]:
        assert max_rel_error(volume_term(st, dtype=np.float64, variant=v), want) <= TOL64, v
    for v in _variants(4, nq) + ["auto"]:
        assert max_rel_error(volume_term(st, dtype=np.float32, variant=v), want) <= TOL32, v


@pytest.mark.parametrize("nq,ne", [(9, 600), (12, 450), (14, 320), (16, 300)])
def test_tc16_fp32_many_elements_against_c_oracle(cuda_device, nq, ne):
    """The 16x16-plane TF32 kernel (fp32 storage, Nq 9..16) on enough
    elements that every CTA runs several persistent iterations."""
    st = make_inputs(BenchmarkConfig(nq=nq, ne=ne, seed=nq + 3))
    ds = DeviceFieldState.from_field_state(st, dtype=torch.float32)
    volume_rhs_device(ds, variant="tc")
    got = ds.rhsq.to(torch.float64).cpu().numpy()
    q, g, j, d = coracle.to_element_batched(st)
    want = coracle.volume_f64_eb(nq, q, g, j, d, st.constants)
    err = max_rel_error(coracle.from_element_batched(got), coracle.from_element_batched(want))
    assert err <= TOL32, err


@pytest.mark.parametrize("nq,ne", [(9, 701), (10, 650), (11, 613), (12, 597)])
def test_line_tile_kernels_many_elements_against_c_oracle(cuda_device, nq, ne):
    """The line-tile kernels (lt fp64 / fp32, ltu fp32 on tcgen05) and the
    line-owner kernel (lo) over more
    elements than resident CTAs, so every CTA runs several persistent
    iterations and the stage pipelines wrap across elements; odd Ne puts the
    last element of odd Nq through the column kernel."""
    st = make_inputs(BenchmarkConfig(nq=nq, ne=ne, seed=nq + 11))
    q, g, j, d = coracle.to_element_batched(st)
    want = coracle.from_element_batched(coracle.volume_f64_eb(nq, q, g, j, d, st.constants))
    for dtype, nbytes, tol in ((torch.float64, 8, TOL64), (torch.float32, 4, TOL32)):
        for v in [x for x in ("lt", "ltu", "lo") if _native.variant_available(x, nbytes, nq)]:
            ds = DeviceFieldState.from_field_state(st, dtype=dtype)
            volume_rhs_device(ds, variant=v)
            got = ds.rhsq.to(torch.float64).cpu().numpy()
            err = max_rel_error(coracle.from_element_batched(got), want)
            assert err <= tol, (v, dtype, err)


@pytest.mark.parametrize("nq,ne", [(5, 1301), (6, 977), (7, 611), (9, 523), (10, 409), (13, 151)])
def test_padded_column_and_lines_kernels_many_elements(cuda_device, nq, ne):
    """The per-plane tc schedule (paired / reordered stage reads at Nq 6, 7),
    the column kernel's Nq-parity line layouts, and the lines kernel's tail
    outputs, one-line tiles and permuted contraction order — over more
    elements than resident CTAs, against the C oracle."""
    st = make_inputs(BenchmarkConfig(nq=nq, ne=ne, seed=nq + 23))
    q, g, j, d = coracle.to_element_batched(st)
    want = coracle.from_element_batched(coracle.volume_f64_eb(nq, q, g, j, d, st.constants))
    for dtype, nbytes, tol in ((torch.float64, 8, TOL64), (torch.float32, 4, TOL32)):
        for v in [x for x in ("tc", "col", "lines") if _native.variant_available(x, nbytes, nq)]:
            ds = DeviceFieldState.from_field_state(st, dtype=dtype)
            volume_rhs_device(ds, variant=v)
            got = ds.rhsq.to(torch.float64).cpu().numpy()
            err = max_rel_error(coracle.from_element_batched(got), want)
            assert err <= tol, (v, dtype, err)


@pytest.mark.parametrize("nq", [9, 10, 11, 12])
def test_large_nq_variants_accumulate_dense_D_custom_constants(cuda_device, nq):
    """Every Nq 9..12 kernel (lines, col, lt, ltu, lo, tc) accumulates into a
    non-zero rhsq (rhsq += v) with a dense random D (no structure for a
    transposed or mis-indexed D row to hide behind) and non-default
    constants, against the oracle."""
    from paper_1604_08501_b200 import PhysicalConstants
    c = PhysicalConstants(p0=9.5e4, R=290.0, gamma=1.35)
    base = make_inputs(BenchmarkConfig(nq=nq, ne=7, seed=nq + 40), constants=c)
    rng = np.random.default_rng(nq)
    base.D[...] = rng.uniform(-1.0, 1.0, base.D.shape).astype(base.D.dtype)
    base.rhsq[...] = rng.uniform(-50.0, 50.0, base.rhsq.shape).astype(base.rhsq.dtype)
    want = base.rhsq.astype(np.float64) + O.volume_term_f64_batched(base)
    for dtype, tol in ((np.float64, TOL64), (np.float32, TOL32)):
        for v in _variants(np.dtype(dtype).itemsize, nq):
            st = make_inputs(BenchmarkConfig(nq=nq, ne=7, seed=nq + 40), constants=c)
            st.D[...] = base.D
            st.rhsq[...] = base.rhsq
            st = st.astype(dtype)
            volume_rhs_(st, variant=v)
            assert max_rel_error(st.rhsq, want) <= tol, (v, dtype)
