"""TEST INFRASTRUCTURE ONLY -- the CPU oracle for the fast Basic-SSA hot path.

Plain, slow, obviously-correct definitions (explicit Hankel entries, one-sided Jacobi
SVD, direct diagonal averaging) in ``ssa_oracle.c`` (fp64, -ffp-contract=off), loaded
through ctypes.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package; the product
package ``paper_0911_4498_b200`` never does, and the two share no code.

Each wrapper names the PAPER.md passage it follows; see the C file header.
Parity status: all functions pinned by tests/test_oracle.py (no "parity unpinned").
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ssa_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None
_lock = threading.Lock()

_dp = ctypes.POINTER(ctypes.c_double)


def build(force: bool = False) -> str:
    """Compile ssa_oracle.c with gcc (-O2, no FMA contraction) into oracle/liboracle.so."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
                               "-std=c99", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB_PATH)
            i64 = ctypes.c_int64
            lib.oracle_trajectory.argtypes = [_dp, i64, i64, _dp]
            lib.oracle_matvec.argtypes = [_dp, i64, i64, _dp, _dp, ctypes.c_int]
            lib.oracle_diag_average.argtypes = [_dp, i64, i64, _dp]
            lib.oracle_hankelize_rank1.argtypes = [ctypes.c_double, _dp, i64, _dp, i64, _dp]
            lib.oracle_svd_jacobi.argtypes = [_dp, i64, i64, i64, _dp, _dp, _dp]
            lib.oracle_svd_jacobi.restype = ctypes.c_int
            lib.oracle_svd_jacobi_capped.argtypes = [_dp, i64, i64, i64, _dp, _dp, _dp, ctypes.c_int]
            lib.oracle_svd_jacobi_capped.restype = ctypes.c_int
            _lib = lib
    return _lib


def _c(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _p(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def trajectory(f, L: int) -> np.ndarray:
    """Explicit L x K trajectory matrix, x_ij = f_{i+j-1} (sec 2.1)."""
    f = _c(f)
    N = f.shape[0]
    K = N - L + 1
    X = np.empty((L, K))
    _load().oracle_trajectory(_p(f), N, L, _p(X))
    return X


def matvec(f, L: int, x, transpose: bool = False) -> np.ndarray:
    """y = X x (x len K) or X^T x (x len L) over the explicit entries (Algs. 2-3 compute this)."""
    f = _c(f); x = _c(x)
    N = f.shape[0]
    K = N - L + 1
    y = np.empty(K if transpose else L)
    assert x.shape[0] == (L if transpose else K)
    _load().oracle_matvec(_p(f), N, L, _p(x), _p(y), 1 if transpose else 0)
    return y


def diag_average(Y) -> np.ndarray:
    """Diagonal averaging of an L x K matrix (sec 2.4)."""
    Y = _c(Y)
    L, K = Y.shape
    g = np.empty(L + K - 1)
    _load().oracle_diag_average(_p(Y), L, K, _p(g))
    return g


def hankelize_rank1(sigma: float, u, v) -> np.ndarray:
    """Diagonal averaging of sigma u v^T, entries formed on the fly (Eq. hankelization1)."""
    u = _c(u); v = _c(v)
    g = np.empty(u.shape[0] + v.shape[0] - 1)
    _load().oracle_hankelize_rank1(float(sigma), _p(u), u.shape[0], _p(v), v.shape[0], _p(g))
    return g


def grouped(sigma, U, V, groups, ngroups: int) -> np.ndarray:
    """Grouped reconstruction, Basic SSA steps 3-4 written out: for each group I the
    resultant matrix X_I = sum_{i in I} sigma_i u_i v_i^T (sec 2.3) is
    formed explicitly and diagonally averaged (sec 2.4).  Returns
    [ngroups][L + K - 1]; triples with group -1 are left out."""
    U = np.asarray(U, dtype=np.float64); V = np.asarray(V, dtype=np.float64)
    L, K = U.shape[1], V.shape[1]
    out = np.empty((ngroups, L + K - 1))
    for g in range(ngroups):
        X = np.zeros((L, K))
        for i, gi in enumerate(groups):
            if gi == g:
                X += float(sigma[i]) * np.outer(U[i], V[i])
        out[g] = diag_average(X)
    return out


def hmatrix(f, B: int, T: int, L: int, I) -> np.ndarray:
    """Heterogeneity matrix written out from PAPER.md:962-1040 (sec 6.2): base windows
    F_i = (f_i..f_{i+B-1}), i = 1..N-B+1, test windows F_j = (f_j..f_{j+T-1}),
    j = 1..N-T+1 (R21); for each base window the Jacobi SVD of its trajectory
    matrix gives the orthonormal U_r, r in I (1-based); for each test window its L-lagged
    vectors X_m are the columns of its explicit trajectory matrix, and
        g_ij = sum_m dist^2(X_m, span U_I) / sum_m |X_m|^2            (Eq. (g))
    with dist(X, span) = |X - U_I U_I^T X| (orthogonal projection)."""
    f = np.asarray(f, dtype=np.float64)
    N = f.shape[0]
    I = [int(r) for r in I]
    nb, nt = N - B + 1, N - T + 1
    Xs = [trajectory(f[j:j + T], L) for j in range(nt)]
    den = np.array([np.sum(X * X) for X in Xs])
    G = np.empty((nb, nt))
    for i in range(nb):
        _, U, _, _ = svd(f[i:i + B], L, max(I))
        P = U[[r - 1 for r in I]].T          # L x |I|, orthonormal columns
        for j in range(nt):
            R = Xs[j] - P @ (P.T @ Xs[j])     # residuals of the lagged vectors
            G[i, j] = np.sum(R * R) / den[j]
    return G


def bootstrap(f, eps, noise_sigma: float, L: int, d: int):
    """Bootstrap study of the rank-d reconstruction (sec 6.3) written out:
    for each replicate F' = F + noise_sigma eps_r, the Jacobi SVD of its trajectory matrix,
    the first d triples grouped and averaged (Basic SSA steps 3-4) into G_r; then per point
    the sample mean, the unbiased variance and the mean square error against F (plain
    loops over the replicates).  Returns (mean, var, mse, G)."""
    f = np.asarray(f, dtype=np.float64)
    R, N = eps.shape
    G = np.empty((R, N))
    for r in range(R):
        fp = f + noise_sigma * eps[r]
        s, U, V, _ = svd(fp, L, d)
        G[r] = grouped(s, U, V, [0] * d, 1)[0]
    mean = np.zeros(N)
    for r in range(R):
        mean += G[r]
    mean /= R
    var = np.zeros(N)
    mse = np.zeros(N)
    for r in range(R):
        var += (G[r] - mean) ** 2
        mse += (G[r] - f) ** 2
    var = var / (R - 1) if R > 1 else var
    return mean, var, mse / R, G


def svd(f, L: int, nsv: int | None = None):
    """Leading nsv singular triples of the trajectory matrix by one-sided Jacobi
    (sec 2.2, with X = U Sigma V^T, R3).
    Returns (sigma[nsv], U[nsv][L], V[nsv][K], sweeps)."""
    f = _c(f)
    N = f.shape[0]
    K = N - L + 1
    n = min(L, K)
    nsv = n if nsv is None else min(nsv, n)
    s = np.empty(nsv); U = np.empty((nsv, L)); V = np.empty((nsv, K))
    sweeps = _load().oracle_svd_jacobi(_p(f), N, L, nsv, _p(s), _p(U), _p(V))
    return s, U, V, sweeps


def svd_sweeps(f, L: int, nsv: int, max_sweeps: int):
    """The same Jacobi computation stopped after max_sweeps sweeps (bench.py's bounded
    CPU-baseline sample only; results are not converged triples)."""
    f = _c(f)
    N = f.shape[0]
    K = N - L + 1
    nsv = min(nsv, min(L, K))
    s = np.empty(nsv); U = np.empty((nsv, L)); V = np.empty((nsv, K))
    return _load().oracle_svd_jacobi_capped(_p(f), N, L, nsv, _p(s), _p(U), _p(V), int(max_sweeps))


def reconstruct(f, L: int, nsv: int | None = None):
    """Oracle decompose + reconstruct: triples by Jacobi, then each elementary series by
    direct averaging.  Returns (sigma, U, V, G[nsv][N])."""
    s, U, V, _ = svd(f, L, nsv)
    G = np.stack([hankelize_rank1(s[i], U[i], V[i]) for i in range(s.shape[0])]) if s.shape[0] else np.zeros((0, len(f)))
    return s, U, V, G
