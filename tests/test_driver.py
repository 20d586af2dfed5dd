"""B200 counterparts of the reference's driver entry points
(``paper_1604_08501_b200/driver.py`` vs ``lf/bench/driver.py:94-178``):
equivalence_error / full_check / run_benchmark over the reference's emitted
level kernels (compiled for sm_100a) and the native variants."""

from __future__ import annotations

import pytest

from oracle import volterm as O
from paper_1604_08501_b200 import BenchmarkConfig, ExecutionError
from paper_1604_08501_b200 import driver

#: the independent CPU reference of every GPU check here: the pinned oracle
#: (``lf/bench/driver.py:98`` uses the reference's numpy oracle the same way)
ORACLE = O.reference_volume_term


def test_corpus_covers_every_level_the_reference_can_emit():
    idx = driver.corpus_index()
    for nq in (2, 3, 4, 8):
        for lv in range(1, 9):
            assert f"level{lv}_nq{nq}.cl" in idx
    with pytest.raises(ExecutionError, match="cannot emit"):
        driver.emitted_level(4, 7)
    with pytest.raises(ExecutionError, match="no emitted kernel"):
        driver.emitted_level(5, 8)


def test_equivalence_error_never_uses_the_product_as_want(monkeypatch):
    """Without an independent reference the driver refuses instead of
    comparing the GPU path with itself."""
    import importlib
    real = importlib.import_module

    def no_loopforge(name, *a, **k):
        if name.startswith("loopforge"):
            raise ImportError(name)
        return real(name, *a, **k)

    monkeypatch.setattr(driver.importlib, "import_module", no_loopforge)
    monkeypatch.setattr(driver, "REFERENCE_INSTALL", driver.REFERENCE_INSTALL / "absent")
    with pytest.raises(ExecutionError, match="independent CPU reference"):
        driver.independent_reference()


@pytest.mark.gpu
def test_equivalence_error_emitted_and_native(cuda_device):
    cfg = BenchmarkConfig(nq=4, ne=24, level=8, seed=3)
    k = driver.emitted_level(4, 8)
    assert driver.equivalence_error([k], cfg, reference=ORACLE) <= 1e-5
    assert driver.equivalence_error(["auto"], cfg, reference=ORACLE) <= 1e-5
    assert driver.equivalence_error(["col"], cfg, reference=ORACLE) <= 1e-5


@pytest.mark.gpu
def test_criterion1_grid_against_oracle(cuda_device):
    """The reference's acceptance criterion 1 (``pkg/tests/test_acceptance.py:
    65-83``): Nq {2,3,4} x Ne {1,2,5} x seeds {1,2,3} x levels 1..8, every
    level's emitted kernel compiled for sm_100a and run on the GPU, against
    the pinned CPU oracle at the reference's tolerance 1e-5 (``:42``).
    Level 7 is the one level the reference's own emitter rejects
    (``VecAccessMisaligned``), so it has no text to run."""
    rows = list(driver.full_check(range(1, 9), [2, 3, 4], [1, 2, 5], [1, 2, 3],
                                  reference=ORACLE))
    assert len(rows) == 8 * 3 * 3 * 3
    for cfg, err, ok in rows:
        if cfg.level == 7:
            assert err is None and not ok
        else:
            assert ok, (cfg, err)


@pytest.mark.gpu
def test_full_check_default_reference_is_the_unmodified_reference(cuda_device):
    try:
        ref = driver.independent_reference()
    except ExecutionError:
        pytest.skip("reference not installed in baseline/_ref")
    assert ref.__module__.startswith("loopforge")
    rows = list(driver.full_check([8], [3], [2], [1]))
    assert rows and all(ok for _, _, ok in rows)


@pytest.mark.gpu
def test_run_benchmark_report(cuda_device):
    rep = driver.run_benchmark(BenchmarkConfig(nq=4, ne=2048, level=8), steps=3,
                               reference=ORACLE)
    assert rep.emitted_ms > 0 and rep.native_f32_ms > 0 and rep.native_f64_ms > 0
    assert rep.equivalence_error is not None and rep.equivalence_error <= 1e-5
    assert "KERNEL void fused_r_s" in rep.source
    assert "level=8" in rep.row_text()
