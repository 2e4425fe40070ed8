"""GPU parity tests: the CUDA path (through the C ABI) against the CPU oracle.

Tolerances are the north star's (BASELINE.json):
  ||Q^T A Z - H||_F/||A||_F, ||Q^T B Z - T||_F/||B||_F, ||Q^T Q - I||_F, ||Z^T Z - I||_F <= 20 n 2.2e-16
  || |H| - |H_oracle| ||_F <= 1e-9 ||A||_F  and the same for T   (unique up to signs)
Structure is checked bitwise (exact zeros).  Config-4 (singular B) parity is
against Oracle-G (the HT form of a singular pencil is not unique).
"""
import functools
import json
import os

import numpy as np
import pytest

import ht_inputs
import htcheck as C
import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1710_08538_b200 as ht  # noqa: E402
from paper_1710_08538_b200.model import model_flops  # noqa: E402

PARITY = 1e-9
# cfg 4 (singular B) vs Oracle-G: the HT form of a singular pencil is not unique (SURVEY
# F7, reading R-F7): O(u) changes of the window transforms (tests/test_blocked_mirror.py)
# or of the desingularisation draws (test_config4_form_depends_on_rho below) move it by
# O(0.1).  Measured GPU distance to Oracle-G: 0.089-0.106 (gpurun_out/parity_cfg4_*.json,
# profiles/r02_parity.md).  The hard gates are structure, backward error, orthogonality;
# this bound only catches regressions.
CFG4_G_GATE = 0.25
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


def record(name, payload):
    """Measured parity numbers go to gpurun_out/parity_<name>.json (copied under profiles/)."""
    d = os.path.join(ROOT, "gpurun_out")
    os.makedirs(d, exist_ok=True)
    with open(os.path.join(d, f"parity_{name}.json"), "w") as f:
        json.dump(payload, f, indent=1)


@functools.lru_cache(maxsize=None)
def oracle_T_cached(cfg, n):
    A, B, _ = ht_inputs.config_pencil(cfg, n=n)
    return oracle.ht_T(A, B)[:2]


@functools.lru_cache(maxsize=None)
def oracle_G_cached(cfg, n):
    A, B, _ = ht_inputs.config_pencil(cfg, n=n)
    return oracle.ht_G(A, B)[:2]


def to_dev(M):
    return torch.from_numpy(np.ascontiguousarray(np.asarray(M, dtype=np.float64).T)).cuda()


def from_dev(t):
    return np.asfortranarray(t.cpu().numpy().T)


def gpu_reduce(A, B, nb=0, wantq=True, wantz=True, **kw):
    n = A.shape[0]
    dA, dB = to_dev(A), to_dev(B)
    dQ = torch.empty((n, n), dtype=torch.float64, device="cuda") if wantq else None
    dZ = torch.empty((n, n), dtype=torch.float64, device="cuda") if wantz else None
    rep = ht.reduce_device(dA, dB, dQ, dZ, nb=nb, **kw)
    torch.cuda.synchronize()
    out = [from_dev(dA), from_dev(dB), from_dev(dQ) if wantq else None, from_dev(dZ) if wantz else None]
    return (*out, rep)


def check_props(A, B, H, T, Q, Z, tolmul=1.0):
    n = A.shape[0]
    assert C.structure_ok(H, T)
    ra, rb, oq, oz = C.backward_errors(A, B, H, T, Q, Z)
    tol = C.tol_ns(n) * tolmul
    assert ra <= tol and rb <= tol and oq <= tol and oz <= tol, (ra, rb, oq, oz, tol)
    return ra, rb, oq, oz


def check_parity(A, B, H, T, Hr, Tr):
    dh = C.abs_diff(H, Hr, C.fro(A))
    dt = C.abs_diff(T, Tr, C.fro(B))
    assert dh <= PARITY and dt <= PARITY, (dh, dt)
    return dh, dt


@pytest.mark.parametrize("kind", ["qrnormal", "shifted", "qruniform"])
@pytest.mark.parametrize("n,nb", [(3, 1), (4, 2), (5, 8), (8, 3), (17, 4), (40, 5), (64, 8), (100, 16),
                                  (130, 32), (161, 13)])
def test_small_sweep_vs_oracle_T(kind, n, nb):
    A, B = ht_inputs.pencil(kind, n, 1000 + n + nb)
    H, T, Q, Z, rep = gpu_reduce(A, B, nb=nb)
    check_props(A, B, H, T, Q, Z)
    Hr, Tr, _, _ = oracle.ht_T(A, B)
    check_parity(A, B, H, T, Hr, Tr)
    assert rep["ir_failed_columns"] == 0


def test_config1_full_size():
    A, B, nb = ht_inputs.config_pencil(1)
    H, T, Q, Z, rep = gpu_reduce(A, B, nb=nb)
    check_props(A, B, H, T, Q, Z)
    Hr, Tr, _, _ = oracle.ht_T(A, B)
    check_parity(A, B, H, T, Hr, Tr)
    assert rep["ir_failed_columns"] == 0


@pytest.mark.parametrize("cfg,n", [(3, 600), (5, 700), (2, 520)])
def test_config_shapes_multi_panel(cfg, n):
    """Config recipes at sizes the oracle finishes in seconds: several panels,
    staircase windows with Remark-4 ragged first windows, and the tail rule."""
    A, B, nb = ht_inputs.config_pencil(cfg, n=n)
    nb = min(nb, 64)
    H, T, Q, Z, rep = gpu_reduce(A, B, nb=nb)
    check_props(A, B, H, T, Q, Z)
    Hr, Tr, _, _ = oracle.ht_T(A, B)
    check_parity(A, B, H, T, Hr, Tr)


@pytest.mark.parametrize("cfg,n,nb", [(5, 900, 160), (5, 1100, 256)])
def test_windows_taller_than_256_rows(cfg, n, nb):
    """nb > 128: staircase windows of 2nb > 256 rows take the 512-thread factorization,
    512-column chain rings and single-buffered band/Qhat staging (cfg5 uses nb = 256)."""
    A, B, _ = ht_inputs.config_pencil(cfg, n=n)
    H, T, Q, Z, rep = gpu_reduce(A, B, nb=nb)
    check_props(A, B, H, T, Q, Z)
    Hr, Tr, _, _ = oracle.ht_T(A, B)
    check_parity(A, B, H, T, Hr, Tr)


@pytest.mark.parametrize("cfg,n,fails", [(3, 1300, ()), (3, 1300, (200, 201, 777)), (2, 600, ()),
                                         (1, 700, (300,)), (5, 900, ())])
def test_headline_nb128_vs_oracle_T(cfg, n, fails):
    """The headline launch configuration nb = 128 (cfg 3): 256 x 128 staircase windows take
    the FactorSmem<256,32,1> factorization, the cap-256 / h-64 chain rings, the pipelined
    R1/R2 and R3/L2 windows (k >= 64) and the double-buffered <= 256-row band staging.
    Forced IR failures add premature absorptions with 64 <= k < 128 and k < 64 (batched
    path).  B is nonsingular, so the HT form is unique up to signs: gate at 1e-9."""
    A, B, _ = ht_inputs.config_pencil(cfg, n=n)
    H, T, Q, Z, rep = gpu_reduce(A, B, nb=128, force_ir_fail=fails)
    check_props(A, B, H, T, Q, Z)
    Hr, Tr = oracle_T_cached(cfg, n)
    dh, dt = check_parity(A, B, H, T, Hr, Tr)
    assert rep["premature_absorptions"] == len(fails)
    record(f"nb128_cfg{cfg}_n{n}_f{len(fails)}", {"cfg": cfg, "n": n, "nb": 128, "forced_fails": list(fails),
                                                  "absH_vs_oracleT": dh, "absT_vs_oracleT": dt})


@pytest.mark.parametrize("cfg,n,fails", [(3, 1300, ()), (3, 1300, (500, 901)), (5, 900, ())])
def test_solve_paths_agree(cfg, n, fails):
    """The panel's solves on 256-row blocks / 4-CTA clusters (default when the diagonal blocks
    are safe) and on 128-row blocks / 2-CTA clusters (HT_FLAG_SOLVE128) are the same recurrence
    blocked differently: both match Oracle-T, and each other to rounding."""
    A, B, _ = ht_inputs.config_pencil(cfg, n=n)
    nb = ht_inputs.CONFIGS[cfg]["nb"] if n > 1000 else 128
    r4 = gpu_reduce(A, B, nb=nb, force_ir_fail=fails)
    r2 = gpu_reduce(A, B, nb=nb, force_ir_fail=fails, flags=ht.HT_FLAG_SOLVE128)
    Hr, Tr = oracle_T_cached(cfg, n)
    for H, T, Q, Z, _ in (r4, r2):
        check_props(A, B, H, T, Q, Z)
        check_parity(A, B, H, T, Hr, Tr)
    for x, y, nrm in zip(r4[:4], r2[:4], (C.fro(A), C.fro(B), 1.0, 1.0)):
        assert np.max(np.abs(np.abs(x) - np.abs(y))) <= 1e-11 * nrm


def test_flop_accounting_within_15pct_of_model():
    """SURVEY §8(c) pin: instrumented executed flops (per-launch formulas, the paper's
    interposition convention P:2161-2162) within +-15% of the App. A model -- catches
    missing or duplicated work.  Full size is checked in test_full_size_config_properties."""
    for cfg, n, nb in ((3, 1300, 128), (2, 1000, 64), (5, 1100, 256)):
        A, B, _ = ht_inputs.config_pencil(cfg, n=n)
        *_, rep = gpu_reduce(A, B, nb=nb)
        ratio = rep["flops"] / model_flops(n, nb)
        assert 0.85 <= ratio <= 1.15, (cfg, n, nb, ratio)


def test_report_times_are_consistent():
    """ht_report timing fields (include/ht.h): the union of the chain-apply launch intervals
    (t_chain_busy) is positive, no longer than their sum (t_chain; they overlap on concurrent
    streams) and no longer than the reduction; the critical-stream spans fit in the reduction."""
    A, B, _ = ht_inputs.config_pencil(3, n=1300)
    *_, rep = gpu_reduce(A, B, nb=128)
    eps = 1e-4
    assert rep["chain_launches"] > 0 and rep["flops_chain"] > 0
    assert 0.0 < rep["t_chain_busy"] <= rep["t_chain"] + eps
    assert rep["t_chain_busy"] <= rep["seconds"] + eps
    assert rep["t_panel"] + rep["t_absorb_right"] + rep["t_absorb_left"] <= rep["seconds"] + eps
    assert rep["t_factor_exposed"] <= rep["t_factor"] + eps


@pytest.mark.parametrize("sa,sb", [(1e200, 1.0), (1.0, 1e-200), (1e-200, 1e200), (1e300, 1e300)])
def test_extreme_scaling_is_invariant(sa, sb):
    """Any finite pencil is accepted (include/ht.h "Range"): entries near 1e+-200 would
    overflow or underflow squared norms; the library scales by exact powers of two and
    undoes it on H, T.  The HT form of (sa A, sb B) is (sa H, sb T) with the same Q, Z."""
    A, B = ht_inputs.pencil("qruniform", 300, 8)
    H, T, Q, Z, _ = gpu_reduce(A, B, nb=32)
    As, Bs = A * sa, B * sb
    Hs, Ts, Qs, Zs, rep = gpu_reduce(As, Bs, nb=32)
    assert np.all(np.isfinite(Hs)) and np.all(np.isfinite(Ts))
    check_props(A, B, Hs / sa, Ts / sb, Qs, Zs)  # (numpy's own products would overflow at 1e300)
    assert C.abs_diff(Hs / sa, H, C.fro(A)) <= PARITY and C.abs_diff(Ts / sb, T, C.fro(B)) <= PARITY
    assert (rep["scale_a"] != 1.0) == (sa != 1.0) and (rep["scale_b"] != 1.0) == (sb != 1.0)


@pytest.mark.parametrize("n,nb", [(120, 16), (300, 32), (700, 64), (700, 128)])
def test_config4_singular(n, nb):
    """Config 4 (singular, graded B): the HT form of a singular pencil is not unique
    (tests/test_blocked_mirror.py::test_singular_ht_form_is_not_unique shows O(u)
    perturbations of the window transforms move it by >> 1e-9), so the hard gate is
    structure + backward error + orthogonality; |H|,|T| vs Oracle-G are reported."""
    A, B, _ = ht_inputs.config_pencil(4, n=n)
    H, T, Q, Z, rep = gpu_reduce(A, B, nb=nb)
    check_props(A, B, H, T, Q, Z)
    assert rep["desingularizations"] > 0
    Hg, Tg = oracle_G_cached(4, n)
    dh = C.abs_diff(H, Hg, C.fro(A))
    dt = C.abs_diff(T, Tg, C.fro(B))
    record(f"cfg4_n{n}_nb{nb}", {"cfg": 4, "n": n, "nb": nb, "absH_vs_oracleG": dh, "absT_vs_oracleG": dt,
                                 "ir_failed_columns": rep["ir_failed_columns"],
                                 "premature_absorptions": rep["premature_absorptions"],
                                 "desingularizations": rep["desingularizations"],
                                 "solve_rescales": rep["solve_rescales"]})
    assert dh <= CFG4_G_GATE and dt <= CFG4_G_GATE, (dh, dt)


def test_config4_form_depends_on_rho():
    """Evidence for reading R-F7 on the product path itself: two seeds of the
    desingularisation draws rho (perturbations of B of size 2u||B||_F) give two
    backward-stable HT forms of the same singular pencil that differ by >> 1e-9."""
    A, B, _ = ht_inputs.config_pencil(4, n=300)
    H0, T0, Q0, Z0, _ = gpu_reduce(A, B, nb=32, seed=0)
    H1, T1, Q1, Z1, _ = gpu_reduce(A, B, nb=32, seed=1)
    check_props(A, B, H0, T0, Q0, Z0)
    check_props(A, B, H1, T1, Q1, Z1)
    d = C.abs_diff(H0, H1, C.fro(A))
    record("cfg4_rho_seed", {"n": 300, "nb": 32, "absH_seed0_vs_seed1": d,
                             "absT_seed0_vs_seed1": C.abs_diff(T0, T1, C.fro(B))})
    assert d > 1e-9, d


def test_staircase_step_wider_than_pending_reflectors():
    """Reading R-step: a premature absorption with k < min(32, nb) pending reflectors uses
    windows of 2*32 x k rows stepping by 32.  Forced IR failures one, two and three
    columns into panels (nb = 64) make k = 1, 2, 3; B is nonsingular, so the HT form is
    unique up to signs and must match the oracle like any other blocking."""
    A, B = ht_inputs.pencil("shifted", 400, 31)
    H, T, Q, Z, rep = gpu_reduce(A, B, nb=64, force_ir_fail=(1, 3, 7, 100, 170))
    assert rep["premature_absorptions"] >= 4
    check_props(A, B, H, T, Q, Z)
    Hr, Tr, _, _ = oracle.ht_T(A, B)
    check_parity(A, B, H, T, Hr, Tr)


def test_streams_and_pipelining_match_one_stream_bitwise(monkeypatch):
    """The absorption runs on five streams with cross-phase pipelining (R1/R2, R3/L2;
    readings R-commute and R-win).  Every element must receive the same transforms in the
    same order as on one stream (HT_SERIAL=1), so the outputs are bitwise identical;
    forced IR failures add premature absorptions (batched, small-k path) to the run."""
    A, B, _ = ht_inputs.config_pencil(3, n=1100)
    out = []
    for serial in (False, True):
        if serial:
            monkeypatch.setenv("HT_SERIAL", "1")
        out.append(gpu_reduce(A, B, nb=128, force_ir_fail=(300, 301))[:4])
    for M1, M2 in zip(*out):
        assert np.array_equal(M1, M2)


@pytest.mark.parametrize("knob", ["HT_NO_WAVE", "HT_L2PERSIST", "HT_SWEEP_RES_MB"])
def test_scheduling_switches_are_bitwise_neutral(monkeypatch, knob):
    """The wavefront factorization of the R1/L1 staircase chains (window i's panel b starts once
    (i-1, b) and (i, b-1) are stored), the (opt-in) L2-persisting panel workspace and the fused
    sweep's evict-first cache hints (HT_SWEEP_RES_MB=-1: none) change only WHEN and WHERE work
    runs, not its arithmetic: the outputs equal the window-by-window / plain-cache run bit for
    bit (premature absorptions included)."""
    A, B, _ = ht_inputs.config_pencil(3, n=1100)
    out = []
    for off in (False, True):
        if off:
            monkeypatch.setenv(knob, "-1" if knob == "HT_SWEEP_RES_MB" else "1")
        out.append(gpu_reduce(A, B, nb=128, force_ir_fail=(300, 301))[:4])
    for M1, M2 in zip(*out):
        assert np.array_equal(M1, M2)


def test_row_split_and_cluster_solves_agree(monkeypatch):
    """trsv4r (the four 64-row slices of a 256-row block on four independent CTAs, default) and
    trsv4 (column slices on a 4-CTA cluster combined by DSMEM, HT_TRSV4_CLUSTER=1) solve the same
    recurrence with different summation orders: both match Oracle-T and each other to rounding."""
    cfg, n = 3, 1300
    A, B, _ = ht_inputs.config_pencil(cfg, n=n)
    r1 = gpu_reduce(A, B, nb=128, force_ir_fail=(500,))
    monkeypatch.setenv("HT_TRSV4_CLUSTER", "1")
    r2 = gpu_reduce(A, B, nb=128, force_ir_fail=(500,))
    Hr, Tr = oracle_T_cached(cfg, n)
    for H, T, Q, Z, _ in (r1, r2):
        check_props(A, B, H, T, Q, Z)
        check_parity(A, B, H, T, Hr, Tr)
    for x, y, nrm in zip(r1[:4], r2[:4], (C.fro(A), C.fro(B), 1.0, 1.0)):
        assert np.max(np.abs(np.abs(x) - np.abs(y))) <= 1e-11 * nrm


def test_chain_apply_measurement_hook():
    """ht_bench_chain_apply (bench.py's standalone roofline) runs the product kernel."""
    sec, fl = ht.ht_bench_chain_apply(1024, 128, 6, False, 2)
    assert sec > 0 and fl == 2.0 * 1024 * 128 * 128 * 6
    sec, fl = ht.ht_bench_chain_apply(512, 96, 4, True, 1)
    assert sec > 0 and fl == 2.0 * 512 * 96 * 96 * 4


def test_forced_ir_failures_premature_absorption():
    """IR-failure fallback (Algorithm 1): forced failures make
    the panel stop early (k < nb) and restart at the failed column."""
    A, B = ht_inputs.pencil("qrnormal", 200, 77)
    H, T, Q, Z, rep = gpu_reduce(A, B, nb=16, force_ir_fail=(5, 6, 40, 41, 42, 130))
    assert rep["premature_absorptions"] >= 4
    check_props(A, B, H, T, Q, Z)
    Hr, Tr, _, _ = oracle.ht_T(A, B)
    check_parity(A, B, H, T, Hr, Tr)


def test_no_q_no_z():
    A, B = ht_inputs.pencil("shifted", 90, 3)
    H1, T1, Q, Z, _ = gpu_reduce(A, B, nb=8)
    H2, T2, _, _, _ = gpu_reduce(A, B, nb=8, wantq=False, wantz=False)
    assert np.array_equal(H1, H2) and np.array_equal(T1, T2)


def test_degenerate_sizes_and_ht_input():
    for n in (0, 1, 2):
        A, B = ht_inputs.pencil("shifted", n, 1)
        if n == 0:
            continue
        H, T, Q, Z, _ = gpu_reduce(A, B)
        assert np.array_equal(H, A) and np.array_equal(T, B)
        assert np.array_equal(Q, np.eye(n)) and np.array_equal(Z, np.eye(n))
    A, B = ht_inputs.pencil("ht", 70, 5)
    H, T, Q, Z, _ = gpu_reduce(A, B, nb=16)
    assert np.array_equal(H, A) and np.array_equal(T, B)
    assert np.array_equal(Q, np.eye(70)) and np.array_equal(Z, np.eye(70))


def test_error_codes_on_device():
    A, B = ht_inputs.pencil("shifted", 16, 2)
    Bbad = B.copy()
    Bbad[5, 2] = 1.0
    with pytest.raises(ht.HTError) as e:
        gpu_reduce(A, Bbad)
    assert e.value.code == -3
    Abad = A.copy()
    Abad[3, 3] = np.nan
    with pytest.raises(ht.HTError) as e:
        gpu_reduce(Abad, B)
    assert e.value.code == 1


def test_host_entry_point_matches_device():
    A, B = ht_inputs.pencil("qrnormal", 77, 9)
    H, T, Q, Z = ht.ht_reduce(A, B, nb=8)
    H2, T2, Q2, Z2, _ = gpu_reduce(A, B, nb=8)
    assert np.array_equal(H, H2) and np.array_equal(T, T2)
    assert np.array_equal(Q, Q2) and np.array_equal(Z, Z2)


def test_host_entry_point_out_of_place_pinned():
    """ht_reduce_host: A, B untouched, outputs (pageable or pinned) bitwise equal to the
    in-place ht_reduce; the device staging is reused across calls and sizes."""
    A, B = ht_inputs.pencil("qruniform", 130, 5)
    A0, B0 = A.copy(), B.copy()
    ref = ht.ht_reduce(A, B, nb=16)
    assert np.array_equal(A, A0) and np.array_equal(B, B0)
    lib = ht.load_library()
    Hi, Ti = np.asfortranarray(A.copy()), np.asfortranarray(B.copy())
    Qi, Zi = np.empty((130, 130), order="F"), np.empty((130, 130), order="F")
    assert lib.ht_reduce(130, Hi.ctypes.data, Ti.ctypes.data, Qi.ctypes.data, Zi.ctypes.data, 1, 1, 16) == 0
    for x, y in zip(ref, (Hi, Ti, Qi, Zi)):
        assert np.array_equal(x, y)
    Ap, Bp = ht.pinned_empty(130), ht.pinned_empty(130)
    Ap[:], Bp[:] = A, B
    outs = tuple(ht.pinned_empty(130) for _ in range(4))
    got = ht.ht_reduce(Ap, Bp, nb=16, out=outs)
    assert all(g is o for g, o in zip(got, outs))
    for x, y in zip(ref, got):
        assert np.array_equal(x, y)
    assert np.array_equal(Ap, A0) and np.array_equal(Bp, B0)
    small = ht.ht_reduce(A[:40, :40], np.triu(B[:40, :40]), nb=8)  # smaller n after a larger one
    assert small[0].shape == (40, 40)


@pytest.mark.parametrize("pad", [1, 2, 3])
def test_leading_dimensions(pad):
    """ld = n + pad (odd pads take the 8-byte fallbacks of the bulk-copy and vector-load paths):
    the same pencil gives the same H, T, Q, Z as ld = n, element by element; NaN guard regions
    around every matrix and in its padding stay untouched (a write-bounds check standing in for
    compute-sanitizer memcheck, which this GPU pool does not run)."""
    A, B = ht_inputs.pencil("qruniform", 600, 12)
    ref = gpu_reduce(A, B, nb=128)
    n = A.shape[0]
    G = 3  # guard columns of M (rows of the tensor) before and after the matrix
    def padded(M):
        buf = torch.full((n + 2 * G, n + pad), float("nan"), dtype=torch.float64, device="cuda")
        t = buf[G:G + n, :n]
        if M is not None:
            t.copy_(torch.from_numpy(np.ascontiguousarray(M.T)))
        return buf, t
    (bA, tA), (bB, tB), (bQ, tQ), (bZ, tZ) = padded(A), padded(B), padded(None), padded(None)
    ht.reduce_device(tA, tB, tQ, tZ, nb=128)
    torch.cuda.synchronize()
    for x, t in zip(ref[:4], (tA, tB, tQ, tZ)):
        got = t.cpu().numpy().T
        assert np.allclose(got, x, rtol=0, atol=1e-13 * max(1.0, np.abs(x).max())), np.abs(got - x).max()
    for b in (bA, bB, bQ, bZ):  # padding and guard regions were never written (out-of-bounds check)
        assert torch.isnan(b[G:G + n, n:]).all()
        assert torch.isnan(b[:G]).all() and torch.isnan(b[G + n:]).all()


def test_deterministic():
    A, B = ht_inputs.pencil("qruniform", 300, 4)
    r1 = gpu_reduce(A, B, nb=32)
    r2 = gpu_reduce(A, B, nb=32)
    for x, y in zip(r1[:4], r2[:4]):
        assert np.array_equal(x, y)


@pytest.mark.slow
def test_config2_full_size_vs_oracle():
    A, B, nb = ht_inputs.config_pencil(2)
    H, T, Q, Z, rep = gpu_reduce(A, B, nb=nb)
    check_props(A, B, H, T, Q, Z)
    Hr, Tr, _, _ = oracle.ht_T(A, B)
    check_parity(A, B, H, T, Hr, Tr)


def test_repeated_calls_on_the_default_stream_are_identical():
    """Inputs refreshed by copies queued on torch's (legacy default) stream right before each
    call: the library must order itself after them (ht_options.stream NULL = default stream)."""
    A, B = ht_inputs.pencil("qruniform", 700, 21)
    dA, dB = to_dev(A), to_dev(B)
    A0, B0 = dA.clone(), dB.clone()
    dQ, dZ = torch.empty_like(dA), torch.empty_like(dA)
    outs = []
    for _ in range(3):
        dA.copy_(A0)
        dB.copy_(B0)
        ht.reduce_device(dA, dB, dQ, dZ, nb=64)
        torch.cuda.synchronize()
        outs.append([from_dev(t) for t in (dA, dB, dQ, dZ)])
    for o in outs[1:]:
        for x, y in zip(outs[0], o):
            assert np.array_equal(x, y)


def _device_backward_errors(A, B, dA, dB, dQ, dZ):
    """North-star residuals at full size, computed on the device (torch fp64 = cuBLAS DGEMM;
    test infrastructure).  Tensors hold column-major matrices as t = M^T, so M1^T M2 M3 of the
    matrices is computed as (t3^T t2^T t1)... on the transposed tensors."""
    tA = torch.from_numpy(np.ascontiguousarray(A.T)).cuda()
    tB = torch.from_numpy(np.ascontiguousarray(B.T)).cuda()
    n = A.shape[0]
    # M = Q^T X Z  <=>  M^T = Z^T X^T Q = dZ @ tX @ dQ^T  (tensors hold the transposes)
    def qtxz(tX):
        return dZ @ tX @ dQ.T
    fro = lambda t: float(torch.linalg.norm(t))
    I = torch.eye(n, dtype=torch.float64, device="cuda")
    ra = fro(qtxz(tA) - dA) / fro(tA)
    rb = fro(qtxz(tB) - dB) / fro(tB)
    oq = fro(dQ @ dQ.T - I)
    oz = fro(dZ @ dZ.T - I)
    # exact structure: H(i, j) = 0 for i > j + 1 and T(i, j) = 0 for i > j (t[j, i] = M[i, j])
    Ht, Tt = dA, dB
    lowH = torch.triu(Ht, diagonal=2)  # entries t[j, i] with i >= j + 2
    lowT = torch.triu(Tt, diagonal=1)
    struct = bool((lowH == 0).all()) and bool((lowT == 0).all())
    return ra, rb, oq, oz, struct


def _golden_gate(A, B, dA, dB, cfg):
    """Entry-wise |H|, |T| against the full-size oracle samples written by
    scripts/make_fullsize_golden.py (Oracle-T for cfg 3/5, Oracle-G for cfg 4), keyed by the
    SHA-256 of the inputs.  Returns (max |d| / ||.||_F, sampled-Frobenius estimate / ||.||_F)
    for H and T, or None if no sample file exists for this config."""
    import hashlib
    path = [os.path.join(GOLD, f"fullsize_cfg{cfg}_{w}.npz") for w in ("T", "G")]
    path = [p for p in path if os.path.exists(p)]
    if not path:
        return None
    g = np.load(path[0])
    sha = lambda M: hashlib.sha256(np.asfortranarray(M).tobytes(order="F")).hexdigest()
    # A (plain draws) must be bitwise the same; B = R of numpy's QR (LAPACK/OpenBLAS) may differ
    # in the last bits between the box that wrote the samples and this one (CPU-specific kernels):
    # then it must agree in ||B||_F to 1e-13 -- a u-level input perturbation, which moves |H|, |T|
    # of a pencil with nonsingular B by ~1e-12, far inside the 1e-9 gate
    assert str(g["sha_A"]) == sha(A), "golden samples are for other inputs"
    b_exact = str(g["sha_B"]) == sha(B)
    if not b_exact:
        assert abs(np.linalg.norm(B) - float(g["fro_B"])) <= 1e-13 * float(g["fro_B"]), "B differs beyond rounding"
    n = A.shape[0]
    out = {}
    for name, t, rows, cols, ref, nrm, region in (
            ("H", dA, g["h_rows"], g["h_cols"], g["h_abs"], float(g["fro_A"]), n * (n + 1) / 2 + n - 1),
            ("T", dB, g["t_rows"], g["t_cols"], g["t_abs"], float(g["fro_B"]), n * (n + 1) / 2)):
        # tensors hold M^T: M[i, j] = t[j, i]
        got = t[torch.from_numpy(cols).cuda(), torch.from_numpy(rows).cuda()].abs().cpu().numpy()
        d = got - ref
        out[name] = (float(np.max(np.abs(d))) / nrm, float(np.sqrt(region / d.size) * np.linalg.norm(d)) / nrm)
    out["oracle"] = str(g["oracle"])
    out["b_sha_match"] = b_exact
    return out


@pytest.mark.slow
@pytest.mark.parametrize("cfg", [3, 4, 5])
def test_full_size_config_properties(cfg):
    """BASELINE.json configs at full size, in the launch configuration bench.py times:
    exact structure, backward errors and orthogonality (north-star tolerances) computed on
    the device; executed flops within +-15% of the App. A model; and |H|, |T| entry by entry
    against the full-size oracle samples of tests/golden/ (Oracle-T for cfg 3, Oracle-G for
    cfg 4) at the north-star 1e-9 -- both as the max entry-wise difference and as the
    sampled estimate of || |H| - |H_oracle| ||_F, relative to ||A||_F (||B||_F for T)."""
    A, B, nb = ht_inputs.config_pencil(cfg)
    n = A.shape[0]
    dA, dB = to_dev(A), to_dev(B)
    dQ, dZ = torch.empty_like(dA), torch.empty_like(dA)
    rep = ht.reduce_device(dA, dB, dQ, dZ, nb=nb)
    torch.cuda.synchronize()
    ra, rb, oq, oz, struct = _device_backward_errors(A, B, dA, dB, dQ, dZ)
    tol = C.tol_ns(n)
    print(f"cfg{cfg} n={n}: resA {ra:.2e} resB {rb:.2e} orthQ {oq:.2e} orthZ {oz:.2e} (tol {tol:.2e}), "
          f"IR extra {rep['ir_extra_columns']} failed {rep['ir_failed_columns']} desing {rep['desingularizations']}")
    assert struct
    assert ra <= tol and rb <= tol and oq <= tol and oz <= tol, (ra, rb, oq, oz, tol)
    if cfg != 4:
        assert rep["ir_failed_columns"] == 0
    ratio = rep["flops"] / model_flops(n, nb)
    assert 0.85 <= ratio <= 1.15, ratio
    gate = _golden_gate(A, B, dA, dB, cfg)
    if gate is not None:
        record(f"fullsize_cfg{cfg}", {"cfg": cfg, "n": n, "nb": nb, "oracle": gate["oracle"],
                                      "absH_max_rel": gate["H"][0], "absH_fro_est_rel": gate["H"][1],
                                      "absT_max_rel": gate["T"][0], "absT_fro_est_rel": gate["T"][1],
                                      "b_sha_match": gate["b_sha_match"], "flops_exec_over_model": ratio,
                                      "backward": {"resA": ra, "resB": rb, "orthQ": oq, "orthZ": oz}})
        lim = PARITY if cfg != 4 else CFG4_G_GATE
        assert max(list(gate["H"]) + list(gate["T"])) <= lim, gate
    elif cfg == 3:
        pytest.fail("tests/golden/fullsize_cfg3_T.npz missing (scripts/make_fullsize_golden.py --config 3)")
    # Q e1 = Z e1 = e1 (every transform acts on rows/columns >= 2)
    e1 = torch.zeros(n, dtype=torch.float64, device="cuda")
    e1[0] = 1.0
    assert torch.equal(dQ[0], e1) and torch.equal(dZ[0], e1)


# ---------------- front ends ------------------------------------------
def test_general_b_front_end_vs_oracle():
    """QZ step 1 (HT_FLAG_GENERAL_B): a general B is first reduced by a Householder
    QR (staircase panels) with A <- Q0^T A.  The result is the HT form of (Q0^T A, R); QR is
    unique up to row signs of R and the HT form up to D1 H D2 (8(c)), so |H|, |T| must match
    Oracle-T run on numpy's QR of B (a library routine) to 1e-9; backward errors are measured
    against the ORIGINAL pencil with the returned Q, Z."""
    for n, nb in ((300, 32), (520, 64)):
        A, B = ht_inputs.pencil("general", n, 5 + n)
        H, T, Q, Z, rep = gpu_reduce(A, B, nb=nb, flags=ht.HT_FLAG_GENERAL_B)
        check_props(A, B, H, T, Q, Z)
        Q0, R = np.linalg.qr(B)
        Hr, Tr, _, _ = oracle.ht_T(Q0.T @ A, np.triu(R))
        check_parity(A, B, H, T, Hr, Tr)
        assert rep["t_front"] > 0 and rep["deflated_columns"] == 0


def test_general_b_required_flag():
    A, B = ht_inputs.pencil("general", 40, 1)
    with pytest.raises(ht.HTError) as e:
        gpu_reduce(A, B)
    assert e.value.code == -3


@pytest.mark.parametrize("n,nb", [(200, 16), (400, 32)])
def test_saddle_point_preprocessing(n, nb):
    """Sec. 3.5.1 preprocessing on Test Suite 4 pencils: B = diag(I, 0) has n/4
    zero columns; with HT_FLAG_DEFLATE_ZERO_COLUMNS they are moved first, A's first n/4 columns
    are QR-reduced and only the trailing pencil is reduced.  Gates: structure, backward error and
    orthogonality of the whole result (the form of a singular pencil is not unique, R-F7), the
    deflated count, T's first n/4 columns exactly 0, and the paper's qualitative pin (Table 4
    P:2314-2321): with preprocessing far fewer columns need IR and none fails."""
    A, B = ht_inputs.pencil("saddle", n, 13)
    l = n // 4
    H, T, Q, Z, rep = gpu_reduce(A, B, nb=nb, flags=ht.HT_FLAG_DEFLATE_ZERO_COLUMNS)
    check_props(A, B, H, T, Q, Z)
    assert rep["deflated_columns"] == l
    assert np.all(T[:, :l] == 0.0)
    H0, T0, Q0, Z0, rep0 = gpu_reduce(A, B, nb=nb)
    check_props(A, B, H0, T0, Q0, Z0)
    record(f"saddle_n{n}", {"n": n, "nb": nb, "with_preprocessing": {k: rep[k] for k in (
        "ir_extra_columns", "ir_failed_columns", "ir_steps_total", "premature_absorptions", "deflated_columns")},
        "without": {k: rep0[k] for k in ("ir_extra_columns", "ir_failed_columns", "ir_steps_total",
                                         "premature_absorptions")}})
    # measured (gpurun_out/parity_saddle_n*.json): n = 200: 77 -> 15 columns with extra IR
    # (38% -> 7.5%; the paper's 27-38% -> < 1% at n >= 1000 used its own B22 re-triangularisation)
    assert rep["ir_failed_columns"] == 0
    assert rep["ir_extra_columns"] <= 0.1 * n
    assert rep0["ir_extra_columns"] >= 3 * max(rep["ir_extra_columns"], 1)
