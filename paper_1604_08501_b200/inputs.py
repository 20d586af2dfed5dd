"""Benchmark state for the DG volume term: constants, configurations,
deterministic inputs.

Mirrors the reference's public input API so callers switch by import path
only:

* ``PhysicalConstants``   — ``lf/bench/inputs.py:17-35``
* ``BenchmarkConfig``     — ``lf/bench/inputs.py:38-49``
* ``FieldState``          — ``lf/bench/inputs.py:52-74``
* ``differentiation_matrix`` — ``lf/bench/inputs.py:77-89``
* ``make_inputs``         — ``lf/bench/inputs.py:92-112`` (same RNG stream,
  same draw order, so the arrays are bit-identical to the reference's)

(``lf/`` = ``pkg/src/loopforge/`` of the reference.)

Logical shapes and axis meanings are unchanged: ``q``/``rhsq`` are
``[Nq, Nq, Nq, 8, Ne]`` (i, j, k, field, element), ``g`` is
``[Nq, Nq, Nq, 3, 3, Ne]`` (i, j, k, a, dir, element), ``Jinv`` is
``[Nq, Nq, Nq, Ne]`` and ``D`` is ``[Nq, Nq]`` with ``D[i, n] = D(i, n)``.
The arrays may be float32 (the reference's dtype) or float64.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

F32 = np.float32

#: field names in storage order (PAPER.md eq. set 2C)
FIELDS = ("rho", "U1", "U2", "U3", "Theta", "Q1", "Q2", "Q3")


@dataclass(frozen=True)
class PhysicalConstants:
    """Dry-air defaults (``lf/bench/inputs.py:17-35``)."""

    p0: float = 1.0e5
    R: float = 287.0
    gamma: float = 1.4

    def __post_init__(self):
        if not (self.p0 > 0 and self.R > 0 and self.gamma > 1):
            raise ValueError("need p0 > 0, R > 0, gamma > 1")

    @property
    def cv(self) -> float:
        return self.R / (self.gamma - 1.0)

    @property
    def cp(self) -> float:
        return self.gamma * self.cv


@dataclass(frozen=True)
class BenchmarkConfig:
    """One benchmark configuration (``lf/bench/inputs.py:38-49``)."""

    nq: int
    ne: int
    level: int = 8
    seed: int = 1

    def __post_init__(self):
        if self.nq < 1 or self.ne < 1:
            raise ValueError("Nq and Ne must be at least 1")
        if not 1 <= self.level <= 8:
            raise ValueError("level must be in 1..8")

    @property
    def points(self) -> int:
        return self.nq ** 3 * self.ne


@dataclass
class FieldState:
    """The 8 prognostic fields with the differentiation matrix and metric
    terms (``lf/bench/inputs.py:52-74``).

    q and rhsq are [Nq, Nq, Nq, 8, Ne]; D is [Nq, Nq] with exact zero row
    sums; g is [Nq, Nq, Nq, 3, 3, Ne]; Jinv is [Nq, Nq, Nq, Ne].
    """

    q: np.ndarray
    rhsq: np.ndarray
    D: np.ndarray
    g: np.ndarray
    Jinv: np.ndarray
    constants: PhysicalConstants = field(default_factory=PhysicalConstants)

    def arrays(self) -> dict[str, np.ndarray]:
        return {"q": self.q, "rhsq": self.rhsq, "D": self.D, "g": self.g,
                "Jinv": self.Jinv}

    def copy(self) -> "FieldState":
        return FieldState(self.q.copy(), self.rhsq.copy(), self.D.copy(),
                          self.g.copy(), self.Jinv.copy(), self.constants)

    def astype(self, dtype) -> "FieldState":
        """Copy of the state with every array cast to ``dtype`` (the fp64
        runs upcast the reference's f32 inputs; the cast is exact)."""
        return FieldState(*(a.astype(dtype) for a in
                            (self.q, self.rhsq, self.D, self.g, self.Jinv)),
                          self.constants)

    @property
    def nq(self) -> int:
        return int(self.q.shape[0])

    @property
    def ne(self) -> int:
        return int(self.q.shape[4])


def differentiation_matrix(nq: int) -> np.ndarray:
    """Analytic differentiation-like matrix with exact zero row sums in f32:
    ``D[i][n] = (n - i)/Nq`` off the diagonal, diagonal = minus the f32 sum
    of the row (``lf/bench/inputs.py:77-89``)."""
    d = np.zeros((nq, nq), F32)
    n_idx = np.arange(nq)
    for i in range(nq):
        off = (n_idx - i).astype(F32) / F32(nq)
        acc = F32(0.0)
        for n in range(nq):
            if n != i:
                d[i, n] = off[n]
                acc = F32(acc + off[n])
        d[i, i] = -acc
    return d


def make_inputs(cfg: BenchmarkConfig,
                constants: PhysicalConstants | None = None) -> FieldState:
    """Deterministic pseudo-random state (``lf/bench/inputs.py:92-112``).

    The draws happen in the reference's order from ``default_rng(seed)``:
    rho ~ U(0.5, 1.5); U1..3 ~ U(-0.1, 0.1); Theta = (p0/R)·U(0.9, 1.1);
    Q1..3 ~ U(0, 1); g ~ U(-1, 1); Jinv ~ U(0.5, 2); rhsq = 0.  Every array
    is float32, exactly as the reference produces it.
    """
    c = constants or PhysicalConstants()
    rng = np.random.default_rng(cfg.seed)
    nq, ne = cfg.nq, cfg.ne
    q = np.empty((nq, nq, nq, 8, ne), F32)
    q[:, :, :, 0] = rng.uniform(0.5, 1.5, (nq, nq, nq, ne))
    q[:, :, :, 1:4] = rng.uniform(-0.1, 0.1, (nq, nq, nq, 3, ne))
    q[:, :, :, 4] = (c.p0 / c.R) * rng.uniform(0.9, 1.1, (nq, nq, nq, ne))
    q[:, :, :, 5:8] = rng.uniform(0.0, 1.0, (nq, nq, nq, 3, ne))
    g = rng.uniform(-1.0, 1.0, (nq, nq, nq, 3, 3, ne)).astype(F32)
    jinv = rng.uniform(0.5, 2.0, (nq, nq, nq, ne)).astype(F32)
    return FieldState(
        q=q,
        rhsq=np.zeros((nq, nq, nq, 8, ne), F32),
        D=differentiation_matrix(nq),
        g=g,
        Jinv=jinv,
        constants=c,
    )
