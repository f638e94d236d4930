"""Pins of the float64 oracle against things other than itself (`-m "not gpu"`).

Each test names what fixes the expected value: a number printed in the paper (tests/golden/),
a closed form, an exact identity of the mathematics, brute force on tiny inputs, or an
extended-precision (mpmath) recomputation. Labels T1..T16 follow SURVEY.md §8(c).
"""
import math

import mpmath
import numpy as np
import pytest

import oracle
from synth import configs as S


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-300))


def rand_sys(m, p, q, rho=0.95, seed=7, zero_D=False):
    wl = S.make_random_mimo(m, p, q, L=8, batch=1, N=0, rho=rho, seed=seed, zero_D=zero_D)
    return wl.Abar[0], wl.Bbar[0], wl.C[0], wl.D[0]


def rand_u(batch, L, p, seed=11):
    return np.random.default_rng(seed).standard_normal((batch, L, p))


# ---------------------------------------------------------------- T1: paper's d_1, d_100
def test_T1_hippo_discretisation_matches_paper(golden_hippo):
    """d_1 = 0.999000499750125, d_100 = 0.9507437210436478 (m=100, Delta=5e-4)."""
    m, dl = int(golden_hippo["m"]), golden_hippo["delta"]
    Abar, _ = S.trapezoid(S.hippo(m), None, dl)
    d = np.diag(Abar)
    assert abs(d[0] - golden_hippo["d1"]) < 1e-12
    assert abs(d[-1] - golden_hippo["d100"]) < 1e-12
    # lower triangular (Eq. 9) -> eigenvalues are the diagonal, |d| < 1
    assert np.all(np.triu(Abar, 1) == 0.0)
    assert np.all(np.abs(d) < 1.0)
    # 0-based indices would not reproduce the paper (R9)
    A0, _ = S.trapezoid(S.hippo(m, base=0), None, dl)
    assert abs(np.diag(A0)[0] - golden_hippo["d1"]) > 1e-4


# ---------------------------------------------------------------- T2: (Abar^(2^15))_11 and N=14
def test_T2_power_2_15_matches_paper_and_mpmath(golden_hippo):
    m, dl = int(golden_hippo["m"]), golden_hippo["delta"]
    Abar, _ = S.trapezoid(S.hippo(m), None, dl)
    P = oracle.powers(Abar, 15)
    v = P[15][0, 0]
    # the paper's printed value (6 significant digits, reading R8: printed 5.87548 vs exact 5.875397)
    assert abs(v / golden_hippo["d1_pow_2_15"] - 1.0) < 2e-5
    # exact: d_1 = (1 - Delta)/(1 + Delta) for lambda = -2 (closed form of Eq. 10 on the diagonal)
    mpmath.mp.dps = 50
    d1 = (1 - mpmath.mpf("0.0005")) / (1 + mpmath.mpf("0.0005"))
    exact = float(d1 ** (2 ** 15))
    # 15 fp64 squarings amplify the initial rounding of d_1 by 2^15 (~4e-12 relative)
    assert abs(v / exact - 1.0) < 5e-11


def test_T2_stage_count_N14_under_eigenvalue_criterion(golden_hippo):
    """Abar^(2^15) negligible -> 15 products apply H_14 of degree 32767."""
    m, dl = int(golden_hippo["m"]), golden_hippo["delta"]
    Abar, _ = S.trapezoid(S.hippo(m), None, dl)
    P = oracle.powers(Abar, 16)
    # the paper's argument: the largest eigenvalue power d_1^(2^(N+1)) falls below ~1e-14
    N = next(n for n in range(16) if np.max(np.abs(np.diag(P[n + 1]))) < 1e-14)
    assert N == int(golden_hippo["N"])
    assert 2 ** (N + 1) - 1 == int(golden_hippo["degree"])
    assert N + 1 == int(golden_hippo["stages"])


# ---------------------------------------------------------------- T3: triangular closed form
def test_T3_triangular_powers_diagonal_closed_form():
    """diag(Abar^(2^k)) = d_i^(2^k) for lower-triangular Abar; upper part stays exactly 0."""
    m, dl = 32, 2e-3
    Abar, _ = S.trapezoid(S.hippo(m), None, dl)
    P = oracle.powers(Abar, 12)
    mpmath.mp.dps = 40
    lam = [-(n + 1) for n in range(1, m + 1)]            # diag of Eq. 9, 1-based
    for k in (0, 1, 5, 12):
        assert np.all(np.triu(P[k], 1) == 0.0)
        for i in (0, m // 2, m - 1):
            d = (1 + mpmath.mpf(dl) / 2 * lam[i]) / (1 - mpmath.mpf(dl) / 2 * lam[i])
            exact = float(d ** (2 ** k))
            assert abs(P[k][i, i] - exact) <= 1e-10 * abs(exact) + 1e-300


# ---------------------------------------------------------------- T4: powers vs 40-digit squaring
def test_T4_powers_accuracy_vs_mpmath():
    """PAPER.md:274-275 ("powers computed with accuracy ~1e-14"): fp64 squaring of the fp64 Abar
    against the same squaring carried out in 40-digit arithmetic."""
    m, dl, K = 12, 5e-4, 15
    Abar, _ = S.trapezoid(S.hippo(m), None, dl)
    P = oracle.powers(Abar, K)
    mpmath.mp.dps = 40
    X = mpmath.matrix([[mpmath.mpf(float(Abar[i, j])) for j in range(m)] for i in range(m)])
    for k in range(1, K + 1):
        X = X * X
        if k in (4, 10, 15):
            ref = np.array([[float(X[i, j]) for j in range(m)] for i in range(m)])
            scale = np.max(np.abs(ref))
            assert np.max(np.abs(P[k] - ref)) <= 1e-12 * max(scale, 1.0)


# ---------------------------------------------------------------- T5: cascade == recurrence if 2^(N+1) >= L
@pytest.mark.parametrize("m,p,q,L,N", [(6, 2, 3, 200, 7), (16, 1, 1, 4096, 11), (5, 3, 2, 64, 5)])
def test_T5_cascade_equals_recurrence_when_exact(m, p, q, L, N):
    Ab, Bb, C, D = rand_sys(m, p, q)
    u = rand_u(2, L, p)
    y_rec = oracle.recurrence(Ab, Bb, C, D, u)
    y_cas = oracle.cascade(oracle.powers(Ab, N), Bb, C, D, u, N)
    assert 2 ** (N + 1) >= L
    assert rel(y_cas, y_rec) < 1e-12


def test_T5_E1_config_exact():
    wl = S.make_E1(L=4096)
    u = wl.u_all()[0]
    y_rec = oracle.recurrence(wl.Abar[0], wl.Bbar[0], wl.C[0], wl.D[0], u)
    y_cas = oracle.cascade(oracle.powers(wl.Abar[0], 11), wl.Bbar[0], wl.C[0], wl.D[0], u, 11)
    assert rel(y_cas, y_rec) < 1e-12


# ---------------------------------------------------------------- T6: exact truncation residual
def test_T6_truncation_residual_identity():
    """y_rec - y_casc = C Abar^(2^(N+1)) x_{l - 2^(N+1)} for l >= 2^(N+1), 0 before."""
    m, p, q, L, N = 6, 2, 3, 200, 4
    Ab, Bb, C, D = rand_sys(m, p, q, rho=0.97)
    u = rand_u(2, L, p)
    y_rec, x = oracle.recurrence(Ab, Bb, C, D, u, return_states=True)
    y_cas = oracle.cascade(oracle.powers(Ab, N), Bb, C, D, u, N)
    T = 2 ** (N + 1)
    Apow = np.linalg.matrix_power(Ab, T)              # independent of oracle.powers
    expect = np.zeros_like(y_rec)
    expect[:, T:, :] = x[:, :L - T, :] @ (C @ Apow).T
    assert np.max(np.abs((y_rec - y_cas) - expect)) < 1e-12 * np.max(np.abs(y_rec))
    assert np.max(np.abs(y_rec[:, :T] - y_cas[:, :T])) < 1e-13 * np.max(np.abs(y_rec))
    assert np.max(np.abs(expect)) > 1e-6                # the dropped term is really there


# ---------------------------------------------------------------- T7: scalar closed forms
def test_T7_scalar_impulse_spec_example():
    """a=0.5, Bbar=C=1, D=0, S=2 stages, impulse -> (1, .5, .25, .125, 0, 0), exactly."""
    A, B, C, D = np.array([[0.5]]), np.array([[1.0]]), np.array([[1.0]]), np.array([[0.0]])
    u = np.zeros((1, 6, 1)); u[0, 0, 0] = 1.0
    y = oracle.cascade(oracle.powers(A, 1), B, C, D, u, 1)[0, :, 0]
    assert list(y) == [1.0, 0.5, 0.25, 0.125, 0.0, 0.0]


@pytest.mark.parametrize("a,N", [(0.9, 3), (-0.7, 2), (0.99, 6)])
def test_T7_scalar_step_response_closed_form(a, N):
    """Constant input: v_l = b (1 - a^min(l+1, 2^(N+1))) / (1 - a) (geometric series, truncated)."""
    b, c, d, L = 0.3, 1.7, -0.4, 300
    u = np.ones((1, L, 1))
    y = oracle.cascade(oracle.powers(np.array([[a]]), N), np.array([[b]]), np.array([[c]]),
                       np.array([[d]]), u, N)[0, :, 0]
    l = np.arange(L)
    expect = c * b * (1 - a ** np.minimum(l + 1, 2 ** (N + 1))) / (1 - a) + d
    assert np.max(np.abs(y - expect)) < 1e-13 * np.max(np.abs(expect))


def test_spec_recurrence_scalar_example():
    """a=0.5, Bbar=C=D=1, u=(1,1) -> x=(1,1.5), y=(2,2.5)."""
    one = np.array([[1.0]])
    y, x = oracle.recurrence(np.array([[0.5]]), one, one, one, np.ones((1, 2, 1)), return_states=True)
    assert list(y[0, :, 0]) == [2.0, 2.5] and list(x[0, :, 0]) == [1.0, 1.5]


# ---------------------------------------------------------------- T8: frequency domain / Lemma 1
def test_T8_scalar_transfer_truncation():
    """a=0.5, S=2: H(1)=2, H_1(1)=1.875, error 0.125 = gamma^4/(1-gamma) (Lemma 1 attained)."""
    A, B, C, D = np.array([[0.5]]), np.array([[1.0]]), np.array([[1.0]]), np.array([[0.0]])
    H = oracle.transfer(A, B, C, D, 1.0)[0, 0]
    HN = oracle.transfer_N(oracle.powers(A, 1), B, C, D, 1.0, 1)[0, 0]
    assert abs(H - 2.0) < 1e-15 and abs(HN - 1.875) < 1e-15
    assert abs(oracle.lemma1_bound(A, B, C, 1) - 0.125) < 1e-15
    assert abs(oracle.transfer(A, B, C, D, -1.0)[0, 0] - 2.0 / 3.0) < 1e-15


def test_T8_exact_frequency_residual_and_lemma1():
    """H - H_N = C W^(2^(N+1)) (I - W)^-1 Bbar, W = z^-1 Abar (exact); ||H - H_N|| <= Lemma 1 bound."""
    m, p, q, N = 6, 2, 3, 3
    Ab, Bb, C, D = rand_sys(m, p, q, rho=0.9)
    P = oracle.powers(Ab, N)
    for th in np.linspace(0.0, 2 * np.pi, 17)[:-1]:
        z = np.exp(1j * th)
        W = Ab / z
        resid = C @ np.linalg.matrix_power(W, 2 ** (N + 1)) @ np.linalg.solve(np.eye(m) - W, Bb)
        diff = oracle.transfer(Ab, Bb, C, D, z) - oracle.transfer_N(P, Bb, C, D, z, N)
        assert np.max(np.abs(diff - resid)) < 1e-12
    # Lemma 1 where its premise gamma < 1 holds
    g = np.random.default_rng(5)
    for _ in range(20):
        G = g.standard_normal((m, m))
        A9 = 0.9 * G / np.linalg.norm(G, 2)
        Bq, Cq = g.standard_normal((m, p)), g.standard_normal((q, m))
        P9 = oracle.powers(A9, N)
        bound = oracle.lemma1_bound(A9, Bq, Cq, N)
        err = max(np.linalg.norm(oracle.transfer(A9, Bq, Cq, np.zeros((q, p)), np.exp(1j * t))
                                 - oracle.transfer_N(P9, Bq, Cq, np.zeros((q, p)), np.exp(1j * t), N), 2)
                  for t in np.linspace(0, 2 * np.pi, 65)[:-1])
        assert err <= bound * (1 + 1e-12)


# ---------------------------------------------------------------- T9: matrix step response
def test_T9_matrix_step_response():
    """Constant u: v_l = (I-Abar)^-1 (I - Abar^min(l+1, 2^(N+1))) Bbar u (finite geometric sum)."""
    m, p, q, N, L = 5, 2, 2, 3, 40
    Ab, Bb, C, D = rand_sys(m, p, q, rho=0.8)
    u0 = np.array([0.7, -1.3])
    u = np.tile(u0, (1, L, 1))
    y = oracle.cascade(oracle.powers(Ab, N), Bb, C, D, u, N)[0]
    for l in (0, 1, 7, 15, 16, 39):
        n = min(l + 1, 2 ** (N + 1))
        v = np.linalg.solve(np.eye(m) - Ab, (np.eye(m) - np.linalg.matrix_power(Ab, n)) @ Bb @ u0)
        assert np.max(np.abs(y[l] - (C @ v + D @ u0))) < 1e-13


# ---------------------------------------------------------------- T10: impulse, stage count exact
@pytest.mark.parametrize("N", [0, 1, 3, 5])
def test_T10_impulse_response_and_exact_zero_tail(N):
    m, p, q, L = 6, 2, 3, 150
    Ab, Bb, C, D = rand_sys(m, p, q, rho=0.97)
    for j in range(p):
        u = np.zeros((1, L, p)); u[0, 0, j] = 1.0
        y = oracle.cascade(oracle.powers(Ab, N), Bb, C, D, u, N)[0]
        T = 2 ** (N + 1)
        for l in range(min(T, L)):
            h = C @ np.linalg.matrix_power(Ab, l) @ Bb[:, j] + (D[:, j] if l == 0 else 0.0)
            assert np.max(np.abs(y[l] - h)) < 1e-14
        assert np.all(y[T:] == 0.0)                      # exactly zero beyond the degree
        assert np.max(np.abs(y[T - 1])) > 0.0            # the last tap is present


# ---------------------------------------------------------------- T11: brute-force block Toeplitz
def _matmul_py(A, B):
    return [[sum(A[i][k] * B[k][j] for k in range(len(B))) for j in range(len(B[0]))] for i in range(len(A))]


@pytest.mark.parametrize("m,p,q,L,N", [(3, 2, 2, 20, 2), (4, 1, 3, 24, 1), (2, 2, 1, 17, 3)])
def test_T11_brute_force_toeplitz(m, p, q, L, N):
    """Dense block-Toeplitz map with blocks C Abar^(i-j) Bbar, 0 <= i-j < 2^(N+1), D on the diagonal
    (Eq. 8 truncated to the degree of H_N), written with explicit Python loops."""
    Ab, Bb, C, D = rand_sys(m, p, q, rho=0.9, seed=3)
    u = rand_u(1, L, p, seed=4)
    Al, Bl, Cl, Dl = Ab.tolist(), Bb.tolist(), C.tolist(), D.tolist()
    Apow = [[[1.0 if i == j else 0.0 for j in range(m)] for i in range(m)]]
    for _ in range(L):
        Apow.append(_matmul_py(Apow[-1], Al))
    y = [[0.0] * q for _ in range(L)]
    for i in range(L):
        for jt in range(i + 1):
            n = i - jt
            if n >= 2 ** (N + 1):
                continue
            blk = _matmul_py(_matmul_py(Cl, Apow[n]), Bl)
            for a in range(q):
                for b in range(p):
                    y[i][a] += blk[a][b] * u[0, jt, b]
        for a in range(q):
            for b in range(p):
                y[i][a] += Dl[a][b] * u[0, i, b]
    y_cas = oracle.cascade(oracle.powers(Ab, N), Bb, C, D, u, N)[0]
    assert rel(y_cas, np.array(y)) < 1e-12


# ---------------------------------------------------------------- T12: recurrence == kernel convolution
def test_T12_recurrence_equals_materialised_convolution():
    m, p, q, L = 7, 2, 3, 128
    Ab, Bb, C, D = rand_sys(m, p, q, rho=0.93)
    u = rand_u(3, L, p)
    y_rec = oracle.recurrence(Ab, Bb, C, D, u)
    y_conv = oracle.convolution(oracle.kernel_taps(Ab, Bb, C, L), D, u)
    assert rel(y_conv, y_rec) < 1e-12
    # and the truncated convolution equals the cascade (same operator H_N)
    N = 3
    y_tr = oracle.convolution(oracle.kernel_taps(Ab, Bb, C, 2 ** (N + 1)), D, u)
    assert rel(oracle.cascade(oracle.powers(Ab, N), Bb, C, D, u, N), y_tr) < 1e-12


# ---------------------------------------------------------------- T13: invariants
def test_T13_causality_linearity_shift():
    m, p, q, L, N = 6, 2, 3, 120, 4
    Ab, Bb, C, D = rand_sys(m, p, q)
    P = oracle.powers(Ab, N)
    u, w = rand_u(1, L, p, 1), rand_u(1, L, p, 2)
    y = oracle.cascade(P, Bb, C, D, u, N)
    # causality: zeroing inputs after j does not change y_0..y_j (exact)
    j = 50
    u2 = u.copy(); u2[:, j + 1:] = 0.0
    assert np.array_equal(oracle.cascade(P, Bb, C, D, u2, N)[:, :j + 1], y[:, :j + 1])
    # linearity
    a, b = 0.3, -1.7
    lhs = oracle.cascade(P, Bb, C, D, a * u + b * w, N)
    rhs = a * y + b * oracle.cascade(P, Bb, C, D, w, N)
    assert rel(lhs, rhs) < 1e-13
    # time-shift equivariance: shift u right by s -> y shifts right by s, leading zeros
    s = 13
    us = np.zeros_like(u); us[:, s:] = u[:, :L - s]
    ys = oracle.cascade(P, Bb, C, D, us, N)
    assert np.all(ys[:, :s] == 0.0)
    assert rel(ys[:, s:], y[:, :L - s]) < 1e-13


# ---------------------------------------------------------------- T14: window property
def test_T14_window_equals_global():
    m, p, q, L, N = 6, 2, 3, 400, 4
    Ab, Bb, C, D = rand_sys(m, p, q)
    P = oracle.powers(Ab, N)
    u = rand_u(2, L, p)
    y = oracle.cascade(P, Bb, C, D, u, N)
    for l0, W in ((0, 10), (5, 40), (100, 37), (363, 37)):
        lo = oracle.window_start(l0, N)
        yw = oracle.cascade_window(P, Bb, C, D, u[:, lo:l0 + W], N, l0, lo)
        assert rel(yw, y[:, l0:l0 + W]) < 1e-14


# ---------------------------------------------------------------- T16: effective stages
def test_T16_effective_stages():
    assert oracle.effective_stages(1, 5) == 0
    for L in range(2, 300):
        for N in range(0, 10):
            assert oracle.effective_stages(L, N) == min(N + 1, int(math.floor(math.log2(L - 1))) + 1)


# ---------------------------------------------------------------- input-construction pins (SPEC examples)
def test_hippo_small_cases():
    """Eq. 9: m=1 -> [[-2]]; m=2 -> [[-2, 0], [-sqrt(15), -3]]."""
    assert np.array_equal(S.hippo(1), np.array([[-2.0]]))
    assert np.allclose(S.hippo(2), np.array([[-2.0, 0.0], [-math.sqrt(15.0), -3.0]]), rtol=0, atol=1e-15)
    A = S.hippo(9)
    s = np.sqrt(2 * np.arange(1, 10) + 1.0)
    assert np.allclose(np.tril(A, -1), -np.tril(np.outer(s, s), -1), rtol=0, atol=1e-14)


def test_trapezoid_special_cases():
    """A=0 -> Abar=I, Bbar=Delta B; scalar A=-2, B=1 -> Bbar = Delta/(1+Delta)."""
    Ab, Bb = S.trapezoid(np.zeros((3, 3)), np.ones((3, 1)), 0.25)
    assert np.array_equal(Ab, np.eye(3)) and np.allclose(Bb, 0.25)
    Ab, Bb = S.trapezoid(np.array([[-2.0]]), np.array([[1.0]]), 0.5e-3)
    assert abs(Bb[0, 0] - 0.5e-3 / 1.0005) < 1e-18
    assert abs(Ab[0, 0] - 0.9995 / 1.0005) < 1e-16
