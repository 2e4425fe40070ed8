"""Seeded synthetic pencil generators shared by the oracle tests, the GPU tests and bench.py.

This module holds NO arithmetic of the method (no reflectors, no solves, no
reduction). It only draws the inputs (A, B) that both sides consume, following
BASELINE.json `configs` and SURVEY.md §8(d) "Generator spec":

  rng = numpy.random.Generator(numpy.random.PCG64(seed)); element [i, j] of the
  C-order draw is matrix entry (i, j); arrays are returned in Fortran
  (column-major) order, which is the layout of the C-ABI (include/ht.h).

Workload recipes (the paper's Test Suite 1 shape, plus
the BASELINE.json variants):
  cfg1  n=256,   seed 0: A ~ N(0,1); B = R of QR(N(0,1))
  cfg2  n=2048,  seed 1: A ~ N(0,1); B = triu(N(0,1)) + sqrt(n) I
  cfg3  n=8192,  seed 2: A ~ U(-1,1); B = R of QR(U(-1,1))
  cfg4  n=8192,  seed 3: A ~ N(0,1); B = triu(N(0,1)), diag(B)[k] = 10^(-8k/n),
                          then round(0.1 n) random diagonal positions set to 0
                          (reading R-Z17)
  cfg5  n=16384, seed 4: as cfg2
  saddle  (Test Suite 4): A = [[X, Y], [Y^T, 0]], B = diag(I_{3n/4}, 0)
  general A, B ~ N(0,1), B not triangular (QZ step-1 front end)

The generators also accept any n so that tests can draw the same distributions
at sizes the oracle finishes in seconds.
"""
from __future__ import annotations

import numpy as np

CONFIGS = {
    1: dict(n=256, nb=32, seed=0, kind="qrnormal"),
    2: dict(n=2048, nb=64, seed=1, kind="shifted"),
    3: dict(n=8192, nb=128, seed=2, kind="qruniform"),
    4: dict(n=8192, nb=128, seed=3, kind="singular"),
    5: dict(n=16384, nb=256, seed=4, kind="shifted"),
}


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def pencil(kind: str, n: int, seed: int):
    """Return (A, B) as Fortran-ordered float64 arrays for the named recipe."""
    rng = _rng(seed)
    if kind == "qrnormal":
        A = rng.standard_normal((n, n))
        G = rng.standard_normal((n, n))
        B = np.triu(np.linalg.qr(G, mode="r"))
    elif kind == "qruniform":
        A = rng.uniform(-1.0, 1.0, (n, n))
        G = rng.uniform(-1.0, 1.0, (n, n))
        B = np.triu(np.linalg.qr(G, mode="r"))
    elif kind == "shifted":
        A = rng.standard_normal((n, n))
        B = np.triu(rng.standard_normal((n, n)))
        B[np.diag_indices(n)] += np.sqrt(n)
    elif kind == "singular":
        A = rng.standard_normal((n, n))
        B = np.triu(rng.standard_normal((n, n)))
        k = np.arange(n, dtype=np.float64)
        B[np.diag_indices(n)] = 10.0 ** (-8.0 * k / n)
        if n > 0:
            nz = int(round(0.1 * n))
            idx = rng.choice(n, nz, replace=False)
            B[idx, idx] = 0.0
    elif kind == "saddle":
        # Test Suite 4: A = [[X, Y], [Y^T, 0]], B = diag(I, 0) with X
        # symmetric positive definite of 3/4 the dimension and Y random full-rank; X = G^T G + n I
        # (SPEC S:612's documented construction of "random SPD").  n must be divisible by 4.
        if n % 4:
            raise ValueError("saddle pencils need n divisible by 4")
        m1 = 3 * n // 4
        G = rng.standard_normal((m1, m1))
        X = G.T @ G + n * np.eye(m1)
        Y = rng.standard_normal((m1, n - m1))
        A = np.zeros((n, n))
        A[:m1, :m1] = X
        A[:m1, m1:] = Y
        A[m1:, :m1] = Y.T
        B = np.zeros((n, n))
        B[np.arange(m1), np.arange(m1)] = 1.0
    elif kind == "general":
        # a general (not triangular) B: the QZ step-1 front end (HT_FLAG_GENERAL_B)
        A = rng.standard_normal((n, n))
        B = rng.standard_normal((n, n))
    elif kind == "ht":
        # already in Hessenberg-triangular form: the degenerate case where
        # every reflector is the identity (SURVEY §8(c) special cases)
        A = np.triu(rng.standard_normal((n, n)), -1)
        B = np.triu(rng.standard_normal((n, n)))
        B[np.diag_indices(n)] += np.sqrt(max(n, 1))
    else:
        raise ValueError(f"unknown pencil kind {kind!r}")
    return np.asfortranarray(A, dtype=np.float64), np.asfortranarray(B, dtype=np.float64)


def config_pencil(cfg: int, n: int | None = None):
    """(A, B, nb) for BASELINE.json config `cfg`; `n` overrides the size (same recipe)."""
    c = CONFIGS[cfg]
    nn = c["n"] if n is None else n
    A, B = pencil(c["kind"], nn, c["seed"])
    return A, B, c["nb"]
