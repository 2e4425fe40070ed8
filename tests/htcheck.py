"""Verification metrics (test infrastructure; numpy only, no method arithmetic).

They restate the properties the paper fixes for the result (PAPER.md P:38,
Theorem 1) and the north-star tolerances.
"""
from __future__ import annotations

import ctypes
import glob
import os

import numpy as np

U = 2.0 ** -53
EPS_NS = 2.2e-16  # north star's unit in 20*n*2.2e-16


def fro(M):
    return float(np.linalg.norm(M, "fro"))


def backward_errors(A0, B0, H, T, Q, Z):
    """(resA, resB, orthQ, orthZ) as in the north star tolerance list."""
    n = A0.shape[0]
    I = np.eye(n)
    nA = max(fro(A0), 1e-300)
    nB = max(fro(B0), 1e-300)
    resA = fro(Q.T @ A0 @ Z - H) / nA
    resB = fro(Q.T @ B0 @ Z - T) / nB
    oq = fro(Q.T @ Q - I)
    oz = fro(Z.T @ Z - I)
    return resA, resB, oq, oz


def structure_ok(H, T):
    """Exact zeros below the sub-diagonal of H and below the diagonal of T."""
    return bool(np.all(np.tril(H, -2) == 0.0) and np.all(np.tril(T, -1) == 0.0))


def abs_diff(X, Y, nrm):
    return fro(np.abs(X) - np.abs(Y)) / max(nrm, 1e-300)


def tol_ns(n):
    return 20.0 * n * EPS_NS


def dgghrd():
    """LAPACK DGGHRD from scipy's bundled OpenBLAS (a library routine used as
    an independent pin of the oracle), or None if the symbol is absent."""
    import scipy
    base = os.path.join(os.path.dirname(scipy.__file__), "..", "scipy.libs")
    for path in glob.glob(os.path.join(base, "libscipy_openblas*.so*")):
        lib = ctypes.CDLL(path)
        for sym in ("scipy_dgghrd_", "dgghrd_"):
            if hasattr(lib, sym):
                f = getattr(lib, sym)
                f.restype = None

                def run(A, B, f=f):
                    n = A.shape[0]
                    H = np.array(A, order="F", dtype=np.float64, copy=True)
                    T = np.array(B, order="F", dtype=np.float64, copy=True)
                    Q = np.zeros((n, n), order="F")
                    Z = np.zeros((n, n), order="F")
                    c = ctypes.c_char
                    i = ctypes.c_int
                    info = i(0)
                    P = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
                    f(ctypes.byref(c(b"I")), ctypes.byref(c(b"I")), ctypes.byref(i(n)),
                      ctypes.byref(i(1)), ctypes.byref(i(n)), P(H), ctypes.byref(i(n)),
                      P(T), ctypes.byref(i(n)), P(Q), ctypes.byref(i(n)), P(Z),
                      ctypes.byref(i(n)), ctypes.byref(info), ctypes.c_size_t(1), ctypes.c_size_t(1))
                    assert info.value == 0
                    return H, T, Q, Z
                return run
    return None
