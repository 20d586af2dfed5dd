"""B200 counterparts of the reference's driver entry points
(``paper_1604_08501_b200/driver.py`` vs ``lf/bench/driver.py:94-178``):
equivalence_error / full_check / run_benchmark over the reference's emitted
level kernels (compiled for sm_100a) and the native variants."""

from __future__ import annotations

import pytest

from paper_1604_08501_b200 import BenchmarkConfig, ExecutionError
from paper_1604_08501_b200 import driver


def test_corpus_covers_every_level_the_reference_can_emit():
    idx = driver.corpus_index()
    for nq in (2, 4, 8):
        for lv in range(1, 9):
            assert f"level{lv}_nq{nq}.cl" in idx
    with pytest.raises(ExecutionError, match="cannot emit"):
        driver.emitted_level(4, 7)
    with pytest.raises(ExecutionError, match="no emitted kernel"):
        driver.emitted_level(5, 8)


@pytest.mark.gpu
def test_equivalence_error_emitted_and_native(cuda_device):
    cfg = BenchmarkConfig(nq=4, ne=24, level=8, seed=3)
    k = driver.emitted_level(4, 8)
    assert driver.equivalence_error([k], cfg) <= 1e-5
    assert driver.equivalence_error(["auto"], cfg) <= 1e-5
    assert driver.equivalence_error(["col"], cfg) <= 1e-5


@pytest.mark.gpu
def test_full_check_grid(cuda_device):
    rows = list(driver.full_check([1, 7, 8], [2, 4], [5], [1, 2]))
    assert len(rows) == 3 * 2 * 1 * 2
    for cfg, err, ok in rows:
        if cfg.level == 7:
            assert err is None and not ok
        else:
            assert ok, (cfg, err)


@pytest.mark.gpu
def test_run_benchmark_report(cuda_device):
    rep = driver.run_benchmark(BenchmarkConfig(nq=4, ne=2048, level=8), steps=3)
    assert rep.emitted_ms > 0 and rep.native_f32_ms > 0 and rep.native_f64_ms > 0
    assert rep.equivalence_error is not None and rep.equivalence_error <= 1e-5
    assert "KERNEL void fused_r_s" in rep.source
    assert "level=8" in rep.row_text()
