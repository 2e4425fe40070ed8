#!/usr/bin/env python
"""Write full-size oracle samples for the GPU parity gate at BASELINE.json sizes.

TEST INFRASTRUCTURE.  Calls only `oracle/` (and the seeded input generator
ht_inputs.py); nothing here comes from the CUDA path.  For config `cfg` it runs
the oracle once on the full pencil (cfg 3/5: Oracle-T, the primary oracle of
SURVEY §8(c); cfg 4: Oracle-G, the parity reference for singular B)
and stores |H| and |T| at a fixed, seeded set of positions plus the SHA-256 of
the inputs, so that tests/test_gpu.py can gate the n = 8192 GPU result entry by
entry without re-running a ~1 h host computation.  Signs are free (uniqueness up
to D1 H D2), hence absolute values.

    python scripts/make_fullsize_golden.py --config 3     # -> tests/golden/fullsize_cfg3_T.npz
"""
from __future__ import annotations

import argparse
import hashlib
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import ht_inputs  # noqa: E402
import oracle  # noqa: E402


def sha256(M) -> str:
    return hashlib.sha256(np.asfortranarray(M, dtype=np.float64).tobytes(order="F")).hexdigest()


def sample_positions(n: int, seed: int = 12345, nrand: int = 32768):
    """Positions (rows, cols) sampled inside the Hessenberg pattern of H and the triangle of T.
    Independent of any result: diagonals, a few full rows, and uniform random entries."""
    rng = np.random.Generator(np.random.PCG64(seed))
    full_rows = sorted({0, 1, n // 3, n // 2, (2 * n) // 3, n - 2, n - 1})
    # H: i <= j + 1
    hr, hc = [], []
    for d in (-1, 0, 1):
        j = np.arange(max(0, -d), n - max(0, d))
        hr.append(j + d)
        hc.append(j)
    for i in full_rows:
        c = np.arange(max(0, i - 1), n)
        hr.append(np.full(c.size, i))
        hc.append(c)
    i = rng.integers(0, n, nrand)
    j = rng.integers(0, n, nrand)
    keep = i <= j + 1
    hr.append(i[keep]); hc.append(j[keep])
    # T: i <= j
    tr, tc = [], []
    for d in (0, 1):
        j = np.arange(d, n)
        tr.append(j - d)
        tc.append(j)
    for i0 in full_rows:
        c = np.arange(i0, n)
        tr.append(np.full(c.size, i0))
        tc.append(c)
    i = rng.integers(0, n, nrand)
    j = rng.integers(0, n, nrand)
    keep = i <= j
    tr.append(i[keep]); tc.append(j[keep])
    cat = lambda xs: np.concatenate(xs).astype(np.int64)
    return cat(hr), cat(hc), cat(tr), cat(tc)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, required=True)
    ap.add_argument("--n", type=int, default=0)
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    cfg = args.config
    A, B, nb = ht_inputs.config_pencil(cfg, n=args.n or None)
    n = A.shape[0]
    which = "G" if cfg == 4 else "T"
    t0 = time.time()
    if which == "T":
        H, T, _, _ = oracle.ht_T(A, B)
    else:
        H, T, _, _ = oracle.ht_G(A, B)
    el = time.time() - t0
    hr, hc, tr, tc = sample_positions(n)
    out = args.out or os.path.join(ROOT, "tests", "golden", f"fullsize_cfg{cfg}_{which}.npz")
    np.savez_compressed(
        out, n=n, config=cfg, oracle=which, sha_A=sha256(A), sha_B=sha256(B),
        fro_A=np.linalg.norm(A), fro_B=np.linalg.norm(B),
        h_rows=hr, h_cols=hc, h_abs=np.abs(H[hr, hc]), t_rows=tr, t_cols=tc, t_abs=np.abs(T[tr, tc]),
        seconds=el, threads=oracle.num_threads() if which == "T" else 1,
        note=f"Oracle-{which} (oracle/ht_oracle.c) on config_pencil({cfg}) n={n}; "
             f"written by scripts/make_fullsize_golden.py")
    print(f"cfg{cfg} n={n} Oracle-{which}: {el:.0f} s -> {out} ({hr.size} H, {tr.size} T samples)")


if __name__ == "__main__":
    main()
