"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the SSA method (no embedding, FFT, Lanczos,
SVD or averaging): it only draws the synthetic series / vectors that BASELINE.json's
``configs`` describe, so that the oracle side (``oracle/``) and the CUDA side
(``paper_0911_4498_b200``) can be fed byte-identical inputs.  Every item is drawn
from its own ``numpy.random.default_rng([cfg_seed, item])`` stream, so any subset
of a batch regenerates independently of the batch size and of the sharding over
ranks (SURVEY.md §8(d) "Synthetic inputs").

The paper's real workloads (HadCET daily temperature N=86867, Quebec births
N=5113; §7) are not in the container; these series with trend
+ periodic + noise structure and L ~ N/2 (§2.4, 859-860 §6.1)
stand in for them.  Index convention n = 1..N (reading R15).
"""
from __future__ import annotations

import numpy as np

__all__ = [
    "CONFIGS", "cfg1_series", "cfg2_series", "cfg2_batch", "cfg3_series",
    "cfg3_like_series", "cfg4_item", "cfg4_batch", "cfg5_problem", "change_point_series",
    "bootstrap_series", "bootstrap_noise", "cfg3_params",
]

# name -> (N, L, k, batch); K = N - L + 1.  BASELINE.json "configs" [0..4].
CONFIGS = {
    "cfg1": dict(N=1024, L=512, k=10, batch=1),
    "cfg2": dict(N=4096, L=2048, k=16, batch=4096),
    "cfg3": dict(N=1 << 20, L=1 << 19, k=32, batch=1),
    "cfg4": dict(N=8192, L=4096, k=0, batch=65536, products=64),
    "cfg5": dict(N=262144, L=131072, k=50, batch=256),
}


def _n(N: int) -> np.ndarray:
    return np.arange(1, N + 1, dtype=np.float64)


def cfg1_series(N: int = 1024) -> np.ndarray:
    """BASELINE.json configs[0]: f_n = 2 sin(2πn/12) + 0.5 cos(2πn/37) + exp(0.002 n) + N(0, 0.1²), seed 0."""
    n = _n(N)
    noise = np.random.default_rng(0).normal(0.0, 0.1, N)
    return 2.0 * np.sin(2 * np.pi * n / 12) + 0.5 * np.cos(2 * np.pi * n / 37) + np.exp(0.002 * n) + noise


def cfg2_series(i: int, N: int = 4096) -> np.ndarray:
    """BASELINE.json configs[1], series i.  Draw order: A(3)~U[0.5,2], P(3)~U[5,200],
    φ(3)~U[0,2π), a~U[0,1], b~U[-1e-3,1e-3], then ε~N(0,0.2²)^N."""
    rng = np.random.default_rng([1, i])
    A = rng.uniform(0.5, 2.0, 3)
    P = rng.uniform(5.0, 200.0, 3)
    phi = rng.uniform(0.0, 2 * np.pi, 3)
    a = rng.uniform(0.0, 1.0)
    b = rng.uniform(-1e-3, 1e-3)
    eps = rng.normal(0.0, 0.2, N)
    n = _n(N)
    f = a * np.exp(b * n) + eps
    for j in range(3):
        f = f + A[j] * np.sin(2 * np.pi * n / P[j] + phi[j])
    return f


def cfg2_batch(start: int, count: int, N: int = 4096) -> np.ndarray:
    """Series start..start+count-1 of configs[1] as a C-contiguous [count][N] fp64 array."""
    out = np.empty((count, N), dtype=np.float64)
    for r in range(count):
        out[r] = cfg2_series(start + r, N)
    return out


def cfg3_like_series(N: int, seed: int = 3) -> np.ndarray:
    """BASELINE.json configs[2] generator at any N: 8 sinusoids with periods 10^U[1,5],
    amplitudes U[0.1,1], phases U[0,2π) (reading R16), + 1e-12 n² + N(0,0.05²).
    Draw order: P(8), A(8), φ(8), then the noise."""
    rng = np.random.default_rng(seed)
    P = 10.0 ** rng.uniform(1.0, 5.0, 8)
    A = rng.uniform(0.1, 1.0, 8)
    phi = rng.uniform(0.0, 2 * np.pi, 8)
    eps = rng.normal(0.0, 0.05, N)
    n = _n(N)
    f = 1e-12 * n * n + eps
    for j in range(8):
        f = f + A[j] * np.sin(2 * np.pi * n / P[j] + phi[j])
    return f


def cfg3_series() -> np.ndarray:
    return cfg3_like_series(1 << 20, 3)


def cfg3_params(seed: int = 3):
    """The generator parameters (P[8], A[8], phi[8]) that cfg3_like_series(N, seed) draws
    first (same stream, same order), for the closed-form pin of the sinusoid pairs."""
    rng = np.random.default_rng(seed)
    P = 10.0 ** rng.uniform(1.0, 5.0, 8)
    A = rng.uniform(0.1, 1.0, 8)
    phi = rng.uniform(0.0, 2 * np.pi, 8)
    return P, A, phi


def cfg4_item(i: int, N: int = 8192, L: int = 4096):
    """BASELINE.json configs[3], series i: (f~N(0,1)^N, v~N(0,1)^K, u~N(0,1)^L) in that draw order."""
    K = N - L + 1
    rng = np.random.default_rng([4, i])
    f = rng.standard_normal(N)
    v = rng.standard_normal(K)
    u = rng.standard_normal(L)
    return f, v, u


def cfg4_batch(start: int, count: int, N: int = 8192, L: int = 4096):
    K = N - L + 1
    F = np.empty((count, N)); V = np.empty((count, K)); U = np.empty((count, L))
    for r in range(count):
        F[r], V[r], U[r] = cfg4_item(start + r, N, L)
    return F, V, U


def cfg5_problem(p: int, N: int = 262144, L: int = 131072, terms: int = 50):
    """BASELINE.json configs[4], problem p: for i = 1..terms draw g~N(0,I_L) then h~N(0,I_K);
    u_i = g/‖g‖, v_i = h/‖h‖ (unit random vectors), σ_i = 1/i.  Returns (sigma[terms], U[terms][L], V[terms][K])."""
    K = N - L + 1
    rng = np.random.default_rng([5, p])
    U = np.empty((terms, L)); V = np.empty((terms, K))
    for i in range(terms):
        g = rng.standard_normal(L)
        h = rng.standard_normal(K)
        U[i] = g / np.sqrt(np.dot(g, g))
        V[i] = h / np.sqrt(np.dot(h, h))
    sigma = 1.0 / np.arange(1, terms + 1, dtype=np.float64)
    return sigma, U, V


def change_point_series(N: int = 400, Q: int = 200, seed: int = 7) -> np.ndarray:
    """Eq. (hseries) of PAPER.md:1049-1056 (sec 6.2, H-matrix example): f_n = sin(2πn/10)
    + 0.01 ε_n for n < Q, sin(2πn/10.5) + 0.01 ε_n for n >= Q, n = 1..N, ε_n ~ N(0,1)
    white noise from default_rng(seed).  The paper's example: N = 400, Q = 200."""
    n = _n(N)
    rng = np.random.default_rng(seed)
    f = np.where(n < Q, np.sin(2 * np.pi * n / 10), np.sin(2 * np.pi * n / 10.5))
    return f + 0.01 * rng.standard_normal(N)


def bootstrap_series(N: int = 1000) -> np.ndarray:
    """The rank-5 series of the bootstrap study (sec 6.3) with the
    periods read in n (R17 / SURVEY.md §8(c) #17: as printed, (2π/13)(n/N) makes
    the series numerically rank 3): f_n = 10 e^{-5n/N} + sin(2πn/13) + 2.5 sin(2πn/37)."""
    n = _n(N)
    return 10.0 * np.exp(-5.0 * n / N) + np.sin(2 * np.pi * n / 13) + 2.5 * np.sin(2 * np.pi * n / 37)


def bootstrap_noise(R: int, N: int, seed: int = 6) -> np.ndarray:
    """White noise eps_r ~ N(0,1)^N of replicate r from default_rng([seed, r]) ([R][N])."""
    return np.stack([np.random.default_rng([seed, r]).standard_normal(N) for r in range(R)])
