"""Pins for the CPU oracle (oracle/ssa_oracle.c) against what the paper and the
mathematics fix -- NOT against the oracle itself.  Runs without a GPU.

Each pin is chosen so that a plausible slip (dropped term, wrong sign or index,
transposed operand, wrong divisor) fails at least one of them:
  * golden worked examples (tests/golden/spec_examples.json, each cited),
  * unit-vector selection (X e_j is column j of the Hankel matrix, sliced from F),
  * adjoint identity, Hankel structure, linearity,
  * LAPACK SVD and Theorem 1 eigenvalues on tiny inputs (library special case),
  * closed forms (constant, exponential, sinusoid, cos(πn), polynomial ranks),
  * invariants: Σσ² = ‖X‖_F² = Σ c_k f_k², orthonormality, window symmetry,
    full-rank reconstruction identity, averaging a Hankel matrix returns its series.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
import parity
import ssa_inputs

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def _expr(s):
    return eval(s, {"sqrt": math.sqrt})


# ----------------------------------------------------------------------------- golden
@pytest.mark.parametrize("case", GOLD["trajectory"])
def test_golden_trajectory(case):
    X = oracle.trajectory(np.array(case["f"], float), case["L"])
    assert np.array_equal(X, np.array(case["X"], float)), case["cite"]


@pytest.mark.parametrize("case", GOLD["matvec"])
def test_golden_matvec(case):
    y = oracle.matvec(np.array(case["f"], float), case["L"], np.array(case["x"], float), case["transpose"])
    assert np.array_equal(y, np.array(case["y"], float)), case["cite"]


@pytest.mark.parametrize("case", GOLD["diag_average"])
def test_golden_diag_average(case):
    g = oracle.diag_average(np.array(case["Y"], float))
    assert np.array_equal(g, np.array(case["g"], float)), case["cite"]


@pytest.mark.parametrize("case", GOLD["hankelize_rank1"])
def test_golden_hankelize(case):
    g = oracle.hankelize_rank1(case["sigma"], np.array(case["u"], float), np.array(case["v"], float))
    assert np.array_equal(g, np.array(case["g"], float)), case["cite"]


@pytest.mark.parametrize("case", GOLD["sigma"])
def test_golden_sigma(case):
    f = np.array(case["f"], float)
    s, U, V, _ = oracle.svd(f, case["L"])
    if "sigma1_expr" in case:
        assert abs(s[0] - _expr(case["sigma1_expr"])) <= 1e-14 * s[0], case["cite"]
    else:
        want = [_expr(e) for e in case["sigma_expr"]]
        assert np.allclose(s[: len(want)], want, rtol=1e-13, atol=0), case["cite"]


# ----------------------------------------------------------------------------- matvec
def test_trajectory_is_hankel_and_sliced_from_series():
    rng = np.random.default_rng(11)
    for N in (3, 7, 20):
        f = rng.standard_normal(N)
        for L in range(2, N):
            X = oracle.trajectory(f, L)
            K = N - L + 1
            assert X.shape == (L, K)
            for j in range(K):        # column j is the lagged vector X_{j+1} = (f_{j+1..j+L})
                assert np.array_equal(X[:, j], f[j:j + L])
            assert np.array_equal(X[1:, :-1], X[:-1, 1:])   # constant antidiagonals


def test_matvec_unit_vectors_select_columns_and_rows():
    rng = np.random.default_rng(12)
    N = 23
    f = rng.standard_normal(N)
    for L in (2, 5, 12, 22):
        K = N - L + 1
        for j in range(K):
            e = np.zeros(K); e[j] = 1.0
            assert np.array_equal(oracle.matvec(f, L, e), f[j:j + L])
        for i in range(L):
            e = np.zeros(L); e[i] = 1.0
            assert np.array_equal(oracle.matvec(f, L, e, True), f[i:i + K])


def test_matvec_adjoint_and_linearity():
    rng = np.random.default_rng(13)
    for N, L in [(64, 17), (65, 40), (128, 64), (9, 8)]:
        K = N - L + 1
        f = rng.standard_normal(N)
        v = rng.standard_normal(K); u = rng.standard_normal(L); w = rng.standard_normal(K)
        lhs = np.dot(oracle.matvec(f, L, v), u)
        rhs = np.dot(v, oracle.matvec(f, L, u, True))
        assert abs(lhs - rhs) <= 1e-12 * (abs(lhs) + 1)
        a, b = 0.7, -1.3
        y1 = oracle.matvec(f, L, a * v + b * w)
        y2 = a * oracle.matvec(f, L, v) + b * oracle.matvec(f, L, w)
        assert np.allclose(y1, y2, rtol=0, atol=1e-12 * np.abs(y2).max())


# ----------------------------------------------------------------------------- averaging
def test_diag_average_of_trajectory_returns_series():
    """A Hankel matrix is fixed by diagonal averaging: H(X(F)) = F."""
    rng = np.random.default_rng(14)
    for N in (3, 4, 11, 30):
        f = rng.standard_normal(N)
        for L in range(2, N):
            g = oracle.diag_average(oracle.trajectory(f, L))
            assert np.allclose(g, f, rtol=0, atol=1e-14 * np.abs(f).max())


def test_diag_average_divisors_three_cases():
    """All-ones L x K matrix -> all ones (divisors are exactly the antidiagonal counts)
    and single entry (j,l) lands at g_{j+l-1} / c_{j+l-1}."""
    for L, K in [(3, 7), (7, 3), (5, 5), (2, 9)]:
        assert np.array_equal(oracle.diag_average(np.ones((L, K))), np.ones(L + K - 1))
        for j in range(L):
            for l in range(K):
                Y = np.zeros((L, K)); Y[j, l] = 6.0
                g = oracle.diag_average(Y)
                k = j + l  # 0-based antidiagonal index
                cnt = min(k + 1, L, K, L + K - 1 - k)
                want = np.zeros(L + K - 1); want[k] = 6.0 / cnt
                assert np.allclose(g, want, rtol=1e-15, atol=0)


def test_diag_average_transpose_symmetry():
    rng = np.random.default_rng(15)
    Y = rng.standard_normal((6, 11))
    assert np.allclose(oracle.diag_average(Y), oracle.diag_average(Y.T), rtol=1e-15, atol=1e-15)


def test_hankelize_rank1_matches_explicit_averaging():
    rng = np.random.default_rng(16)
    for L, K in [(7, 11), (11, 7), (1, 5), (5, 1), (32, 33)]:
        u = rng.standard_normal(L); v = rng.standard_normal(K); s = 2.5
        g1 = oracle.hankelize_rank1(s, u, v)
        g2 = oracle.diag_average(s * np.outer(u, v))
        assert np.allclose(g1, g2, rtol=1e-14, atol=1e-14)


# ----------------------------------------------------------------------------- SVD
@pytest.mark.parametrize("N", [3, 5, 8, 13, 24, 40])
def test_svd_matches_lapack_and_theorem1_all_windows(N):
    rng = np.random.default_rng(100 + N)
    f = rng.standard_normal(N)
    for L in range(2, N):
        X = oracle.trajectory(f, L)
        s, U, V, sweeps = oracle.svd(f, L)
        assert sweeps > 0, "Jacobi did not converge"
        s_ref = np.linalg.svd(X, compute_uv=False)
        assert np.allclose(s, s_ref, rtol=1e-13, atol=1e-14 * s_ref[0])
        # Theorem 1: sigma_i^2 = eigenvalues of X X^T
        ev = np.sort(np.linalg.eigvalsh(X @ X.T))[::-1][: len(s)]
        assert np.allclose(s ** 2, ev, rtol=1e-12, atol=1e-12 * ev[0])
        n = min(L, N - L + 1)
        assert np.allclose(U @ U.T, np.eye(n), atol=1e-13)
        assert np.allclose(V @ V.T, np.eye(n), atol=1e-13)
        R = X - (U.T * s) @ V            # X = U Sigma V^T (DESIGN R3)
        assert np.linalg.norm(R) <= 1e-13 * np.linalg.norm(X)
        assert np.all(np.diff(s) <= 0)


def test_svd_vectors_match_lapack_up_to_sign():
    rng = np.random.default_rng(17)
    f = rng.standard_normal(31)
    for L in (4, 16, 28):
        X = oracle.trajectory(f, L)
        s, U, V, _ = oracle.svd(f, L)
        Ul, sl, Vtl = np.linalg.svd(X, full_matrices=False)
        for i in range(len(s)):
            assert parity.sine_angle(Ul[:, i], U[i]) < 1e-11
            assert parity.sine_angle(Vtl[i], V[i]) < 1e-11


def test_svd_sign_canonical():
    rng = np.random.default_rng(18)
    f = rng.standard_normal(50)
    s, U, V, _ = oracle.svd(f, 20)
    for i in range(len(s)):
        j = int(np.argmax(np.abs(U[i])))
        assert U[i][j] > 0


def test_svd_frobenius_identity_and_window_symmetry():
    """Σσ² = ‖X‖_F² = Σ_k c_k f_k² and σ(L) = σ(K) (X_K = X_Lᵀ)."""
    rng = np.random.default_rng(19)
    N = 61
    f = rng.standard_normal(N)
    for L in (2, 10, 30, 31, 45):
        K = N - L + 1
        s, _, _, _ = oracle.svd(f, L)
        c = np.array([min(k, L, K, N - k + 1) for k in range(1, N + 1)], float)
        w = float(np.sum(c * f * f))
        assert abs(np.sum(s ** 2) - w) <= 1e-13 * w
        s2, _, _, _ = oracle.svd(f, K)
        assert np.allclose(s, s2, rtol=1e-12, atol=1e-13 * s[0])


def test_closed_form_constant_and_exponential():
    N = 40
    for L in (2, 13, 20, 33):
        K = N - L + 1
        s, U, V, _ = oracle.svd(np.full(N, -3.0), L)
        assert abs(s[0] - 3.0 * math.sqrt(L * K)) <= 1e-14 * s[0]
        assert s[1] <= 1e-13 * s[0]
        assert np.allclose(np.abs(U[0]), 1 / math.sqrt(L), atol=1e-14)
        # exponential a r^n (n = 1..N): rank 1, σ₁ = |a| ‖(r¹..r^L)‖ ‖(r⁰..r^{K−1})‖
        a, r = 0.5, 1.03
        n = np.arange(1, N + 1, dtype=float)
        s, U, V, _ = oracle.svd(a * r ** n, L)
        want = abs(a) * np.linalg.norm(r ** np.arange(1, L + 1)) * np.linalg.norm(r ** np.arange(0, K))
        assert abs(s[0] - want) <= 1e-13 * want
        assert s[1] <= 1e-13 * s[0]


def test_closed_form_sinusoid_rank2_equal_pair():
    """A sin(2πn/P + φ), P | L and P | K: σ₁ = σ₂ = A √(LK) / 2, rank 2."""
    A, P, phi = 1.7, 6, 0.3
    L, K = 24, 30
    N = L + K - 1
    n = np.arange(1, N + 1, dtype=float)
    s, _, _, _ = oracle.svd(A * np.sin(2 * np.pi * n / P + phi), L)
    want = A * math.sqrt(L * K) / 2
    assert abs(s[0] - want) <= 1e-13 * want and abs(s[1] - want) <= 1e-13 * want
    assert s[2] <= 1e-12 * s[0]


@pytest.mark.parametrize("deg", [0, 1, 2, 3])
def test_closed_form_polynomial_rank(deg):
    N, L = 50, 20
    n = np.arange(1, N + 1, dtype=float) / N
    f = sum((0.5 + j) * n ** j for j in range(deg + 1))
    s, _, _, _ = oracle.svd(f, L)
    assert s[deg] > 1e-8 * s[0]
    assert s[deg + 1] <= 1e-12 * s[0]


def test_closed_form_alternating_and_damped():
    N, L = 41, 17
    n = np.arange(1, N + 1, dtype=float)
    s, _, _, _ = oracle.svd(np.cos(np.pi * n), L)       # rank 1
    assert s[1] <= 1e-13 * s[0]
    s, _, _, _ = oracle.svd(np.exp(-0.02 * n) * np.sin(2 * np.pi * n / 9.3), L)   # rank 2
    assert s[1] > 1e-3 * s[0] and s[2] <= 1e-12 * s[0]


def test_full_reconstruction_identity_and_finite_rank():
    """Σ over all elementary reconstructions = F (PAPER.md:117-121 + averaging fixes Hankel),
    and a rank-2 series is reconstructed exactly from 2 triples."""
    rng = np.random.default_rng(20)
    for N, L in [(12, 5), (25, 13), (30, 22)]:
        f = rng.standard_normal(N)
        s, U, V, G = oracle.reconstruct(f, L)
        assert np.allclose(G.sum(axis=0), f, rtol=0, atol=1e-12 * np.abs(f).max())
    n = np.arange(1, 81, dtype=float)
    f = 2.0 * np.sin(2 * np.pi * n / 7.3 + 0.4)
    s, U, V, G = oracle.reconstruct(f, 30, 2)
    assert np.allclose(G.sum(axis=0), f, rtol=0, atol=1e-12)


def test_grouped_reconstruction_pins():
    """oracle.grouped (explicit X_I) against what the paper fixes:
    one group of all min(L,K) triples returns F (X = sum X_i, and the
    averaging of a Hankel matrix is the identity); a one-triple group equals the rank-1
    on-the-fly averaging (a different code path); the groups of a partition sum to the
    all-in-one group (linearity of the averaging); the two leading
    triples of a pure sinusoid (rank 2) reconstruct it exactly; a dropped triple (-1)
    contributes nothing."""
    rng = np.random.default_rng(31)
    N, L = 29, 12
    f = rng.standard_normal(N)
    s, U, V, _ = oracle.svd(f, L)
    r = len(s)
    allg = oracle.grouped(s, U, V, [0] * r, 1)
    assert np.allclose(allg[0], f, rtol=0, atol=1e-12 * np.abs(f).max())
    groups = [i % 3 for i in range(r)]
    G3 = oracle.grouped(s, U, V, groups, 3)
    assert np.allclose(G3.sum(axis=0), allg[0], rtol=0, atol=1e-12 * np.abs(f).max())
    g1 = oracle.grouped(s, U, V, [-1, 0] + [-1] * (r - 2), 1)
    assert np.allclose(g1[0], oracle.hankelize_rank1(s[1], U[1], V[1]), rtol=0, atol=1e-14 * np.abs(g1).max())
    n = np.arange(1, 61, dtype=float)
    sin = 1.3 * np.sin(2 * np.pi * n / 8.5 + 0.2)
    s, U, V, _ = oracle.svd(sin + 0.0, 25, 4)
    g = oracle.grouped(s, U, V, [0, 0, -1, -1], 1)
    assert np.allclose(g[0], sin, rtol=0, atol=1e-12)


def test_hmatrix_oracle_pins():
    """oracle.hmatrix (Eq. (g)) against what the paper fixes: 0 <= g <= 1;
    the rewritten form 1 - sum (U^T X)^2 / sum |X|^2 (a different formula)
    agrees; a pure sinusoid (rank 2) with I = {1,2} gives g = 0 everywhere (every window's
    lagged vectors lie in the same 2-D space); I = all L triples gives g = 0; the paper's
    change-point series (Eq. (hseries)) shows the block structure of its H-matrix figure
    (PAPER.md:1049-1066): small inside the homogeneous parts, large across the change."""
    f = ssa_inputs.change_point_series(160, 80, 3)
    B, T, L = 40, 40, 20
    G = oracle.hmatrix(f, B, T, L, [1, 2])
    assert G.min() >= 0.0 and G.max() <= 1.0
    # rewritten formula at a few entries
    for i, j in [(0, 0), (5, 100), (120, 7), (60, 60)]:
        _, U, _, _ = oracle.svd(f[i:i + B], L, 2)
        X = oracle.trajectory(f[j:j + T], L)
        g2 = 1.0 - np.sum((U[:2] @ X) ** 2) / np.sum(X * X)
        assert abs(g2 - G[i, j]) <= 1e-12
    n = np.arange(1, 161, dtype=float)
    sin = np.sin(2 * np.pi * n / 10 + 0.3)
    assert np.abs(oracle.hmatrix(sin, B, T, L, [1, 2])).max() <= 1e-12
    rng = np.random.default_rng(4)
    g = rng.standard_normal(60)
    assert np.abs(oracle.hmatrix(g, 30, 25, 10, list(range(1, 11)))).max() <= 1e-12
    nb = 80 - B + 1  # base windows inside the first regime: i + B <= Q
    inside = G[:nb, :nb].mean()
    across = G[:nb, 80:].mean()
    assert inside < 1e-3 and across > 20 * inside


def test_bootstrap_oracle_pins():
    """oracle.bootstrap: with no noise every replicate is the rank-5
    series itself (a finite-rank series is reconstructed exactly from its d triples,
    PAPER.md:117-121), so mean = F, var = 0, mse = 0; with noise, var >= 0 and the
    identity mse = bias^2 + (R-1)/R var holds (definitions of the three estimates)."""
    N, L, d, R = 120, 60, 5, 6
    f = ssa_inputs.bootstrap_series(N)
    eps = ssa_inputs.bootstrap_noise(R, N)
    mean, var, mse, G = oracle.bootstrap(f, eps, 0.0, L, d)
    scale = np.abs(f).max()
    assert np.abs(mean - f).max() <= 1e-11 * scale
    assert var.max() <= 1e-20 * scale ** 2 and mse.max() <= 1e-20 * scale ** 2
    mean, var, mse, G = oracle.bootstrap(f, eps, 0.3, L, d)
    assert var.min() >= 0.0
    assert np.abs(mse - ((mean - f) ** 2 + (R - 1) / R * var)).max() <= 1e-12 * mse.max()
    # more noise, larger error of the estimate
    _, _, mse2, _ = oracle.bootstrap(f, eps, 0.6, L, d)
    assert mse2.mean() > mse.mean()


def test_cfg1_oracle_spectrum_structure():
    """cfg1 (BASELINE configs[0]): σ₁ dominated by the exponential trend, then the two
    sinusoid pairs, then noise (SURVEY Appendix A 'Spectrum structure')."""
    f = ssa_inputs.cfg1_series()
    s, U, V, sweeps = oracle.svd(f, 512, 11)
    assert sweeps > 0
    r = s / s[0]
    assert 0.29 < r[1] < 0.32 and 0.29 < r[2] < 0.32
    assert 0.07 < r[3] < 0.08 and 0.07 < r[4] < 0.08
    assert r[5] < 0.004
    X = oracle.trajectory(f, 512)
    s_ref = np.linalg.svd(X, compute_uv=False)[:11]
    assert np.allclose(s, s_ref, rtol=1e-12)


# ----------------------------------------------------------------------------- parity helper
def test_parity_helpers():
    s = np.array([10.0, 5.0, 4.9999, 4.99985, 1.0, 0.99995])
    cl = parity.clusters(s, 5)
    assert [c[0] for c in cl] == [[0], [1, 2, 3], [4]]
    assert cl[-1][1] is True          # index 4 straddles (gap to 5 < 1e-4 * 10)
    rng = np.random.default_rng(0)
    u = rng.standard_normal(100)
    assert parity.sine_angle(u, -u) < 1e-15
    w = rng.standard_normal(100); w -= np.dot(w, u) / np.dot(u, u) * u
    pert = u / np.linalg.norm(u) + 1e-9 * w / np.linalg.norm(w)
    assert abs(parity.sine_angle(u, pert) - 1e-9) < 1e-12
    Q = np.linalg.qr(rng.standard_normal((50, 3)))[0].T
    M = np.array([[0.6, 0.8, 0], [-0.8, 0.6, 0], [0, 0, -1.0]])
    assert parity.subspace_sine(Q, M @ Q) < 1e-14
