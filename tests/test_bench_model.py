"""bench.py's algorithmic-byte model of the Lanczos kernel against a
direct step-by-step count of what Alg. 1 + one-pass FRO must move through HBM."""
import numpy as np

import bench


def direct_count(m, N, L, k):
    K = N - L + 1
    M = 1
    while M < N:
        M <<= 1
    H = M // 2
    spec = 16 * (H + 1)
    total = 8 * N + 8 * L                      # read series, write u_1
    for j in range(1, m + 2):                  # half-step A, j = 1..m+1
        total += spec + 2 * 8 * K * (j - 1) + 8 * K
    for j in range(1, m + 1):                  # half-step B, j = 1..m
        total += spec + 2 * 8 * L * j + 8 * L
    total += 8 * ((m + 1) * L + m * K)         # Ritz: read U_{m+1}, V_m once
    total += 8 * k * (L + K)                   # write U_k, V_k
    return total


def test_byte_model_matches_direct_count():
    for m, N, L, k in [(60, 1024, 512, 10), (100, 4096, 2048, 16), (3, 10, 4, 2), (172, 4096, 1000, 16)]:
        assert bench.lanczos_alg_bytes(np.array([m]), N, L, k) == direct_count(m, N, L, k)
    ms = np.array([60, 100, 136])
    assert bench.lanczos_alg_bytes(ms, 4096, 2048, 16) == sum(direct_count(int(x), 4096, 2048, 16) for x in ms)
