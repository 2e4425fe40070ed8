"""Pins of the CPU oracle (oracle/ht_oracle.c) against what the paper and the
mathematics fix -- no GPU needed.  Each test names the passage it checks.

A plausible mistake anywhere in an oracle (a dropped rank-1 term, a wrong sign,
a transposed operand, a missed rotation on Q) breaks either the backward-error
identity H = Q^T A Z (Theorem 1), the exact structure (Alg. 2 "Set ... <- 0"),
or the agreement with an independent reduction (LAPACK DGGHRD, Oracle-G),
which by the uniqueness argument of DESIGN.md (implicit-Q) must hold up to
diagonal +-1 scaling for nonsingular B.
"""
import json
import os

import numpy as np
import pytest

import ht_inputs
import htcheck as C
import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")
KINDS_NONSING = ["qrnormal", "shifted", "qruniform"]


# --- house ---------------------------------------------------------
def test_house_golden_examples():
    with open(os.path.join(GOLD, "house_examples.json")) as f:
        cases = json.load(f)["cases"]
    for c in cases:
        v, beta, alpha = oracle.house(c["x"])
        assert np.allclose(v, c["v"], rtol=0, atol=1e-15)
        assert beta == pytest.approx(c["beta"], abs=1e-15)
        assert alpha == pytest.approx(c["alpha"], abs=1e-15)


@pytest.mark.parametrize("m", [2, 3, 17, 100])
def test_house_reflects_onto_e1(m):
    rng = np.random.default_rng(m)
    x = rng.standard_normal(m)
    v, beta, alpha = oracle.house(x)
    H = np.eye(m) - beta * np.outer(v, v)
    hx = H @ x
    assert abs(alpha) == pytest.approx(np.linalg.norm(x), rel=1e-15)
    assert np.sign(alpha) == -np.sign(x[0])
    assert np.max(np.abs(hx[1:])) <= 4 * m * C.U * np.linalg.norm(x)   # S:121 bound
    assert abs(hx[0] - alpha) <= 4 * m * C.U * abs(alpha)
    assert np.linalg.norm(H.T @ H - np.eye(m)) <= 10 * m * C.U        # orthogonal
    assert 1.0 <= beta <= 2.0


def test_givens_closed_form():
    c, s, r = oracle.givens(3.0, 4.0)
    assert (c, s, r) == pytest.approx((0.6, 0.8, 5.0), abs=1e-15)
    assert oracle.givens(2.0, 0.0) == (1.0, 0.0, 2.0)


def test_opposite_reflector_identity():
    """(B H) e1 = +- e1 / ||B^{-1} e1||  (sec. 2.2), house from the oracle,
    x = B^{-1} e1 from numpy's solver (a library routine)."""
    for kind in KINDS_NONSING:
        A, B = ht_inputs.pencil(kind, 60, 3)
        x = np.linalg.solve(B, np.eye(60)[:, 0])
        v, beta, _ = oracle.house(x)
        BH = B - np.outer(B @ v, beta * v)
        c1 = BH[:, 0]
        assert abs(abs(c1[0]) - 1.0 / np.linalg.norm(x)) <= 1e-14 * abs(c1[0])
        assert np.max(np.abs(c1[1:])) <= 60 * C.U * C.fro(B)


def test_rho_generator_is_normal_and_deterministic():
    r = np.array([oracle.rho(5, j, i) for j in range(40) for i in range(100)])
    assert abs(r.mean()) < 0.06 and abs(r.std() - 1.0) < 0.05
    assert oracle.rho(5, 3, 4) == oracle.rho(5, 3, 4)
    assert oracle.rho(5, 3, 4) != oracle.rho(5, 4, 3)


# --- whole-reduction properties ---------------------------------------------
def _check_props(A, B, H, T, Q, Z):
    n = A.shape[0]
    assert C.structure_ok(H, T)
    ra, rb, oq, oz = C.backward_errors(A, B, H, T, Q, Z)
    tol = C.tol_ns(n)
    assert ra <= tol and rb <= tol and oq <= tol and oz <= tol, (ra, rb, oq, oz)
    # Q e1 = Z e1 = e1 (transforms act on rows/cols >= 2)
    if n:
        assert Q[0, 0] == 1.0 and np.all(Q[1:, 0] == 0) and np.all(Q[0, 1:] == 0)
        assert Z[0, 0] == 1.0 and np.all(Z[1:, 0] == 0) and np.all(Z[0, 1:] == 0)


ORACLES = {"T": oracle.ht_T, "0": oracle.ht_0, "G": oracle.ht_G}


@pytest.mark.parametrize("name", ["T", "0", "G"])
@pytest.mark.parametrize("kind", KINDS_NONSING + ["singular"])
@pytest.mark.parametrize("n", [3, 4, 7, 8, 33, 96])
def test_structure_backward_error_orthogonality(name, kind, n):
    if name == "0" and kind == "singular":
        pytest.skip("Oracle-0's dense LU solve needs nonsingular B")
    A, B = ht_inputs.pencil(kind, n, 11 + n)
    _check_props(A, B, *ORACLES[name](A, B))


@pytest.mark.parametrize("kind", KINDS_NONSING + ["singular"])
@pytest.mark.parametrize("n", [3, 5, 8, 40, 150])
def test_oracle_G_matches_lapack_dgghrd(kind, n):
    """Library pin: LAPACK DGGHRD is the Moler-Stewart algorithm."""
    run = C.dgghrd()
    if run is None:
        pytest.skip("scipy OpenBLAS does not export dgghrd")
    A, B = ht_inputs.pencil(kind, n, 100 + n)
    H, T, _, _ = oracle.ht_G(A, B)
    H2, T2, _, _ = run(A, B)
    assert C.abs_diff(H, H2, C.fro(A)) <= 1e-12
    assert C.abs_diff(T, T2, C.fro(B)) <= 1e-12


@pytest.mark.parametrize("kind", KINDS_NONSING)
@pytest.mark.parametrize("n", [3, 4, 6, 8, 40, 150])
def test_householder_oracles_match_givens(kind, n):
    """Uniqueness up to diagonal +-1 (implicit-Q with Qe1 = Ze1 = e1, nonsingular B):
    Oracle-T and Oracle-0 (Algorithm 2) must reproduce |H|, |T| of Oracle-G."""
    A, B = ht_inputs.pencil(kind, n, 200 + n)
    Hg, Tg, _, _ = oracle.ht_G(A, B)
    for name in ("T", "0"):
        H, T, _, _ = ORACLES[name](A, B)
        assert C.abs_diff(H, Hg, C.fro(A)) <= 1e-12, name
        assert C.abs_diff(T, Tg, C.fro(B)) <= 1e-12, name


@pytest.mark.parametrize("n", [3, 5, 8])
def test_tiny_n_brute_force_agreement_up_to_signs(n):
    """North star: on n <= 8 the Householder oracle agrees with the Givens
    reduction up to diagonal +-1 scaling -- checked as H_T = D1 H_G D2 with
    D1 = diag(sign), D2 = diag(sign) recovered from Q, Z."""
    A, B = ht_inputs.pencil("qrnormal", n, 300 + n)
    H, T, Q, Z = oracle.ht_T(A, B)
    Hg, Tg, Qg, Zg = oracle.ht_G(A, B)
    d1 = np.sign(np.sum(Q * Qg, axis=0))
    d2 = np.sign(np.sum(Z * Zg, axis=0))
    assert np.allclose(Q, Qg * d1, atol=1e-12)
    assert np.allclose(Z, Zg * d2, atol=1e-12)
    assert np.allclose(H, d1[:, None] * Hg * d2[None, :], atol=1e-12 * C.fro(A))
    assert np.allclose(T, d1[:, None] * Tg * d2[None, :], atol=1e-12 * C.fro(B))


@pytest.mark.parametrize("name", ["T", "0", "G"])
@pytest.mark.parametrize("n", [4, 8, 16])
def test_det_pencil_equivalence(name, n):
    """det(A - lam B) det(Q) det(Z) = det(H - lam T) at seeded lam."""
    A, B = ht_inputs.pencil("shifted", n, 400 + n)
    H, T, Q, Z = ORACLES[name](A, B)
    sq, sz = np.linalg.det(Q), np.linalg.det(Z)
    for lam in np.random.default_rng(n).uniform(-3, 3, 5):
        d0 = np.linalg.det(A - lam * B) * sq * sz
        d1 = np.linalg.det(H - lam * T)
        assert abs(d0 - d1) <= 1e-8 * abs(d0)


@pytest.mark.parametrize("name", ["T", "0", "G"])
def test_degenerate_sizes(name):
    for n in (0, 1, 2):
        A, B = ht_inputs.pencil("shifted", n, 1)
        H, T, Q, Z = ORACLES[name](A, B)
        assert np.array_equal(H, A) and np.array_equal(T, B)
        assert np.array_equal(Q, np.eye(n)) and np.array_equal(Z, np.eye(n))


@pytest.mark.parametrize("name", ["T", "0", "G"])
def test_already_ht_form_is_fixed_point(name):
    """Input already in HT form: every reflector tail is zero, so beta = gamma = 0
    (dlarfg convention) and the output equals the input bitwise."""
    A, B = ht_inputs.pencil("ht", 20, 5)
    H, T, Q, Z = ORACLES[name](A, B)
    assert np.array_equal(H, A) and np.array_equal(T, B)
    assert np.array_equal(Q, np.eye(20)) and np.array_equal(Z, np.eye(20))


def test_oracle_T_singular_is_backward_stable_and_desingularises():
    """Config-4 shape (Remark 1): Oracle-T desingularises zero pivots and
    stays backward stable; its HT form may differ from Givens (non-unique for singular
    B), so it is not the cfg-4 parity reference."""
    A, B = ht_inputs.pencil("singular", 120, 9)
    st = {}
    H, T, Q, Z = oracle.ht_T(A, B, seed=1, stats=st)
    _check_props(A, B, H, T, Q, Z)
    assert st["desingularizations"] >= 1


def test_config_shapes_small():
    for cfg in (1, 2, 3, 4, 5):
        A, B, nb = ht_inputs.config_pencil(cfg, n=48)
        assert np.array_equal(B, np.triu(B))
        if cfg == 4:
            assert np.sum(np.diag(B) == 0) == round(0.1 * 48)
        H, T, Q, Z = oracle.ht_G(A, B)
        _check_props(A, B, H, T, Q, Z)


def test_config1_full_size_T_vs_G():
    """BASELINE config 1 (n = 256) at full size: Oracle-T vs Oracle-G up to signs."""
    A, B, _ = ht_inputs.config_pencil(1)
    H, T, Q, Z = oracle.ht_T(A, B)
    _check_props(A, B, H, T, Q, Z)
    Hg, Tg, _, _ = oracle.ht_G(A, B)
    assert C.abs_diff(H, Hg, C.fro(A)) <= 1e-11
    assert C.abs_diff(T, Tg, C.fro(B)) <= 1e-11
