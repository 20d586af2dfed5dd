"""B200 counterparts of the reference's benchmark-driver entry points
(``lf/bench/driver.py``): the callers on the far side of the volume-term
path.

* ``equivalence_error(kernels, cfg)`` — ``lf/bench/driver.py:94-100``: run a
  kernel pipeline on ``cfg``'s inputs (in place, ``rhsq += v``, float32 —
  the interpreter's contract, ``lf/interp.py:71-72``) and return the
  per-field max-norm relative error against an INDEPENDENT CPU reference
  (``want``, as ``lf/bench/driver.py:98`` uses the reference's numpy
  oracle): by default the unmodified reference's own
  ``loopforge.bench.reference_volume_term`` (``baseline/_ref``), or any
  callable passed as ``reference=`` (the tests pass the pinned oracle).
  Never this package's own GPU path, so common-mode errors cannot pass.
  The reference interprets its kernel IR; here a "kernel" is either one of
  the reference's emitted kernels compiled for sm_100a (``EmittedKernel``)
  or a native variant name (``"auto"``, ``"tc"``, ``"col"``, ...), both run
  on the GPU.
* ``full_check(levels, nqs, nes, seeds, tolerance=1e-5)`` —
  ``lf/bench/driver.py:165-178``: the equivalence grid over the reference's
  optimisation levels, with each level's emitted kernel from the corpus
  (``paper_1604_08501_b200/corpus``); yields ``(cfg, err, ok)``.
* ``run_benchmark(cfg)`` — ``lf/bench/driver.py:142-162``: for
  ``cfg.level``, the emitted kernel's and this package's kernel's measured
  time on the GPU (CUDA events) in place of the reference's static cost
  report, plus the equivalence error and the emitted source.
"""

from __future__ import annotations

import importlib
import json
import pathlib
import sys
from dataclasses import dataclass

import torch

from .diagnostics import ExecutionError
from .emitted import CORPUS, EmittedKernel
from .inputs import BenchmarkConfig, make_inputs
from .volume import DeviceFieldState, max_rel_error, volume_rhs_device

#: where ``pip install --target`` puts the unmodified reference
REFERENCE_INSTALL = pathlib.Path(__file__).resolve().parents[1] / "baseline" / "_ref"


def independent_reference():
    """The unmodified reference's ``reference_volume_term``
    (``lf/bench/reference.py:36-70``): importable ``loopforge``, else the
    ``baseline/_ref`` install. Raises ExecutionError when neither exists —
    there is no silent substitute."""
    try:
        return importlib.import_module("loopforge.bench").reference_volume_term
    except ImportError:
        pass
    if (REFERENCE_INSTALL / "loopforge").is_dir():
        sys.path.append(str(REFERENCE_INSTALL))
        try:
            return importlib.import_module("loopforge.bench").reference_volume_term
        except ImportError:
            pass
    raise ExecutionError("equivalence_error needs an independent CPU reference: pass "
                         "reference=<callable(state) -> increment> or install the "
                         "reference into baseline/_ref")


def corpus_index() -> dict:
    return json.loads((CORPUS / "index.json").read_text())


def emitted_level(nq: int, level: int) -> EmittedKernel:
    """The reference's emitted kernel for (Nq, level), compiled for sm_100a
    (``build_level`` + ``emit_source``, ``lf/bench/driver.py:49-51``)."""
    name = f"level{level}_nq{nq}.cl"
    meta = corpus_index().get(name)
    if meta is None:
        raise ExecutionError(f"no emitted kernel for Nq={nq} level {level} in the corpus")
    if "unemittable" in meta:
        raise ExecutionError(f"the reference cannot emit level {level}: {meta['unemittable']}")
    return EmittedKernel.from_file(CORPUS / name)


def _run(kernels, ds: DeviceFieldState) -> None:
    for k in kernels:
        if isinstance(k, EmittedKernel):
            k(ds)
        elif isinstance(k, str):
            volume_rhs_device(ds, variant=k)
        else:
            raise ExecutionError(f"not a kernel: {k!r}")


def equivalence_error(kernels, cfg: BenchmarkConfig, device=None,
                      reference=None) -> float:
    """Max relative error of the kernel pipeline (on the GPU, f32, in place)
    against the independent CPU ``reference(state)`` on cfg's inputs."""
    state = make_inputs(cfg)
    want = (reference or independent_reference())(state)
    ds = DeviceFieldState.from_field_state(state, dtype=torch.float32, device=device)
    _run(list(kernels), ds)
    got = ds.rhsq_logical()
    return max_rel_error(got - state.rhsq, want)


def full_check(levels, nqs, nes, seeds, tolerance: float = 1e-5, reference=None):
    """Equivalence suite over the grid; yields ``(cfg, err, ok)``; levels the
    reference cannot emit yield ``err = None, ok = False``."""
    reference = reference or independent_reference()
    for nq in nqs:
        for level in levels:
            try:
                k = emitted_level(nq, level)
            except ExecutionError:
                for ne in nes:
                    for seed in seeds:
                        yield BenchmarkConfig(nq=nq, ne=ne, level=level, seed=seed), None, False
                continue
            for ne in nes:
                for seed in seeds:
                    cfg = BenchmarkConfig(nq=nq, ne=ne, level=level, seed=seed)
                    err = equivalence_error([k], cfg, reference=reference)
                    yield cfg, err, err <= tolerance
            k.close()


@dataclass(frozen=True)
class BenchReport:
    """``lf/bench/driver.py:103-139`` with measured GPU times in place of the
    static cost model."""

    level: int
    nq: int
    ne: int
    emitted_ms: float        # the reference's level kernel, sm_100a, f32
    native_f32_ms: float     # this package's AUTO kernel, f32
    native_f64_ms: float     # this package's AUTO kernel, f64
    equivalence_error: float | None
    source: str

    def row_text(self) -> str:
        pts = self.nq ** 3 * self.ne
        parts = [f"level={self.level}", f"Nq={self.nq}", f"Ne={self.ne}",
                 f"emitted_ms={self.emitted_ms:.4f}",
                 f"emitted_GDOF/s={pts / self.emitted_ms / 1e6:.2f}",
                 f"native_f32_ms={self.native_f32_ms:.4f}",
                 f"native_f64_ms={self.native_f64_ms:.4f}"]
        if self.equivalence_error is not None:
            parts.append(f"equiv_rel_err={self.equivalence_error:.3e}")
        return "  ".join(parts)

    def row_csv(self) -> str:
        err = "" if self.equivalence_error is None else f"{self.equivalence_error:.6e}"
        pts = self.nq ** 3 * self.ne
        return (f"{self.level},{self.nq},{self.ne},{self.emitted_ms:.6f},"
                f"{pts / self.emitted_ms / 1e6:.4f},{self.native_f32_ms:.6f},"
                f"{self.native_f64_ms:.6f},{err}")

    @staticmethod
    def csv_header() -> str:
        return ("level,nq,ne,emitted_ms,emitted_gdofs,native_f32_ms,native_f64_ms,"
                "equiv_rel_err")


def _time(fn, steps: int) -> float:
    fn()
    s = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(s)
    for _ in range(steps):
        fn()
    b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / steps


def run_benchmark(cfg: BenchmarkConfig, check: bool | None = None,
                  steps: int = 10, reference=None) -> BenchReport:
    """Time cfg.level's emitted kernel and this package's kernels on the GPU
    on device-generated inputs of cfg's shape; optionally verify (always when
    Nq <= 4 unless disabled, like the reference)."""
    k = emitted_level(cfg.nq, cfg.level)
    ds32 = DeviceFieldState.generate(cfg.nq, cfg.ne, seed=cfg.seed, dtype=torch.float32)
    b = k.bind(ds32)
    emitted_ms = _time(lambda: k.launch(b), steps)
    native32 = _time(lambda: volume_rhs_device(ds32), steps)
    ds64 = DeviceFieldState.generate(cfg.nq, cfg.ne, seed=cfg.seed, dtype=torch.float64)
    native64 = _time(lambda: volume_rhs_device(ds64), steps)
    del b, ds32, ds64
    if check is None:
        check = cfg.nq <= 4
    err = equivalence_error([k], cfg, reference=reference) if check else None
    src = k.source
    k.close()
    return BenchReport(level=cfg.level, nq=cfg.nq, ne=cfg.ne, emitted_ms=emitted_ms,
                       native_f32_ms=native32, native_f64_ms=native64,
                       equivalence_error=err, source=src)


__all__ = ["independent_reference", "corpus_index", "emitted_level", "equivalence_error", "full_check",
           "run_benchmark", "BenchReport"]
