"""Oracle package -- TEST INFRASTRUCTURE ONLY.

Python (ctypes) front end to oracle/ht_oracle.c, the plain CPU reference for the
Hessenberg-triangular reduction.  Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / `--impl reference` leg
may import this package.  The product path (paper_1710_08538_b200) never
imports it and shares no code with it.

Parity status:
  house      pinned: closed forms (S:124-126 worked examples, reflector identity)
  givens     pinned: closed form
  ht_G       pinned: LAPACK DGGHRD (library routine) up to signs; brute-force
             definition checks (structure, orthogonality, backward error, det)
  ht_0       pinned: Oracle-G up to signs; paper identities
  ht_T       pinned: Oracle-G / DGGHRD up to signs; paper identities
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ht_oracle.c")
_LIB = os.path.join(_HERE, "libht_oracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (-O2 -fopenmp); returns the .so path."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        d, i64, u64 = ctypes.c_double, ctypes.c_int64, ctypes.c_uint64
        P = ctypes.POINTER(ctypes.c_double)
        lib.orc_house.restype = d
        lib.orc_house.argtypes = [i64, P]
        lib.orc_givens.restype = None
        lib.orc_givens.argtypes = [d, d, P, P, P]
        lib.orc_rho.restype = d
        lib.orc_rho.argtypes = [u64, i64, i64, ctypes.c_uint32]
        for name in ("orc_ht_G", "orc_ht_0"):
            f = getattr(lib, name)
            f.restype = ctypes.c_int
            f.argtypes = [i64, P, P, P, P]
        lib.orc_ht_T.restype = ctypes.c_int
        lib.orc_ht_T.argtypes = [i64, P, P, P, P, u64, i64, ctypes.POINTER(i64)]
        lib.orc_num_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _prep(A, B):
    A = np.array(A, dtype=np.float64, order="F", copy=True)
    B = np.array(B, dtype=np.float64, order="F", copy=True)
    n = A.shape[0]
    assert A.shape == (n, n) and B.shape == (n, n)
    Q = np.zeros((n, n), order="F")
    Z = np.zeros((n, n), order="F")
    return n, A, B, Q, Z


def house(x):
    """(v, beta, alpha): (I - beta v v^T) x = alpha e1, v[0] = 1 (dlarfg convention)."""
    w = np.array(x, dtype=np.float64, copy=True)
    beta = _load().orc_house(len(w), _ptr(w))
    alpha = w[0]
    v = w.copy()
    if len(v):
        v[0] = 1.0
    if beta == 0.0 and len(v):
        v[1:] = 0.0
    return v, beta, alpha


def givens(f, g):
    c, s, r = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    _load().orc_givens(f, g, ctypes.byref(c), ctypes.byref(s), ctypes.byref(r))
    return c.value, s.value, r.value


def rho(seed, col, row, ctr=0):
    return _load().orc_rho(seed, col, row, ctr)


def ht_G(A, B):
    """Oracle-G (Moler-Stewart Givens). Returns H, T, Q, Z."""
    n, A, B, Q, Z = _prep(A, B)
    rc = _load().orc_ht_G(n, _ptr(A), _ptr(B), _ptr(Q), _ptr(Z))
    if rc:
        raise RuntimeError(f"orc_ht_G rc={rc}")
    return A, B, Q, Z


def ht_0(A, B):
    """Oracle-0 (Algorithm 2 verbatim, dense LU solve; small n). Returns H, T, Q, Z."""
    n, A, B, Q, Z = _prep(A, B)
    rc = _load().orc_ht_0(n, _ptr(A), _ptr(B), _ptr(Q), _ptr(Z))
    if rc:
        raise RuntimeError(f"orc_ht_0 rc={rc} (exactly singular trailing B)")
    return A, B, Q, Z


def ht_T(A, B, seed: int = 0, jmax: int | None = None, stats: dict | None = None):
    """Oracle-T (O(n^3) unblocked Householder HT reduction). Returns H, T, Q, Z."""
    n, A, B, Q, Z = _prep(A, B)
    nd = ctypes.c_int64(0)
    jm = n if jmax is None else int(jmax)
    rc = _load().orc_ht_T(n, _ptr(A), _ptr(B), _ptr(Q), _ptr(Z), seed, jm, ctypes.byref(nd))
    if rc:
        raise RuntimeError(f"orc_ht_T rc={rc}")
    if stats is not None:
        stats["desingularizations"] = nd.value
    return A, B, Q, Z


def num_threads() -> int:
    return int(_load().orc_num_threads())


def flops_T(n: int, jmax: int | None = None) -> float:
    """Executed-flop model of Oracle-T, 39 m^2 + 40 n m per column."""
    jm = n - 2 if jmax is None else min(jmax, n - 2)
    tot = 0.0
    for j in range(max(jm, 0)):
        m = n - j - 1
        tot += 39.0 * m * m + 40.0 * n * m
    return tot
