"""bench.py's algorithmic-byte models against direct step-by-step counts of
what Alg. 1 + reorthogonalization and the Ritz assembly must move through HBM."""
import numpy as np

import bench


def direct_count(m, N, L, reorth_rows):
    """Lanczos kernel bytes with reorth_rows(side, j) = basis rows read by the CGS of that
    half-step (0 when it skipped reorthogonalization)."""
    K = N - L + 1
    M = 1
    while M < N:
        M <<= 1
    H = M // 2
    spec = 16 * (H + 1)
    total = 8 * N + 8 * L                      # read series, write u_1
    ru = rv = 0
    for j in range(1, m + 2):                  # half-step A, j = 1..m+1 (v side)
        r = reorth_rows("v", j)
        rv += r
        total += spec + 8 * K * r + 8 * K
    for j in range(1, m + 1):                  # half-step B, j = 1..m (u side)
        r = reorth_rows("u", j)
        ru += r
        total += spec + 8 * L * r + 8 * L
    return total, ru, rv


def fro(side, j):
    return 2 * (j - 1) if side == "v" else 2 * j   # one CGS pass: dots + update reads


def test_lanczos_model_matches_direct_count_fro():
    for m, N, L in [(60, 1024, 512), (100, 4096, 2048), (3, 10, 4), (172, 4096, 1000)]:
        tot, ru, rv = direct_count(m, N, L, fro)
        assert ru == rv == bench.fro_rows(m)
        assert bench.lanczos_alg_bytes([m], [ru], [rv], N, L) == tot


def test_lanczos_model_matches_direct_count_pro_pattern():
    """PRO reorthogonalizes on a subset of half-steps (pairs of consecutive ones); the
    model only needs the row totals the kernel reports."""
    rng = np.random.default_rng(1)
    for m, N, L in [(90, 4096, 2048), (40, 1000, 300)]:
        hits = {("v", j): rng.random() < 0.3 for j in range(1, m + 2)}
        hits.update({("u", j): rng.random() < 0.3 for j in range(1, m + 1)})
        tot, ru, rv = direct_count(m, N, L, lambda s, j: fro(s, j) if hits[(s, j)] else 0)
        assert bench.lanczos_alg_bytes([m], [ru], [rv], N, L) == tot
    ms = np.array([60, 100, 136])
    rows = bench.fro_rows(ms)
    assert bench.lanczos_alg_bytes(ms, rows, rows, 4096, 2048) == sum(
        direct_count(int(x), 4096, 2048, fro)[0] for x in ms)


def test_ritz_model():
    for m, N, L, k in [(60, 1024, 512, 10), (100, 4096, 2048, 16)]:
        K = N - L + 1
        assert bench.ritz_alg_bytes([m], N, L, k) == 8 * ((m + 1) * L + m * K) + 8 * k * (L + K)
