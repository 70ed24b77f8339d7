"""GPU parity of the long-series path (M > 16384: four-step FFT through L2, grid-wide
Lanczos; BASELINE configs 3 and 5).  The same kernels are forced onto small problems
(force_long) so the full oracle (Jacobi SVD) can check them; at the real sizes the
products and Hankelizations are compared with the oracle's direct O(LK) sums."""
import numpy as np
import pytest

import oracle
import parity
import ssa_inputs

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_0911_4498_b200 as pkg
    return pkg


def cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def nrel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.parametrize("N,L,force", [(200, 77, True), (1000, 500, True), (4096, 1000, True), (32768, 16384, False),
                                       (40000, 9000, False), (600000, 100, False)])
def test_long_spectrum_and_matvec(P, N, L, force):
    rng = np.random.default_rng(N + L)
    K = N - L + 1
    B = 2
    F = rng.standard_normal((B, N)); x = rng.standard_normal((B, K)); u = rng.standard_normal((B, L))
    plan = P.Plan(N, L, 0, B, force_long=force)
    spec = plan.spectrum(cuda(F))
    S = spec.cpu().numpy()
    ref = np.fft.rfft(F, plan.M)   # library cross-check of the spectrum only
    assert np.abs(S[..., 0] + 1j * S[..., 1] - ref).max() <= 1e-12 * np.abs(ref).max()
    y = plan.matvec(spec, cuda(x)).cpu().numpy()
    z = plan.matvec(spec, cuda(u), transpose=True).cpu().numpy()
    for b in range(B):
        assert nrel(y[b], oracle.matvec(F[b], L, x[b])) <= 1e-12
        assert nrel(z[b], oracle.matvec(F[b], L, u[b], True)) <= 1e-12


@pytest.mark.parametrize("N,L,force", [(300, 100, True), (4096, 2048, True), (32768, 16384, False)])
def test_long_hankelize(P, N, L, force):
    rng = np.random.default_rng(3 * N + L)
    K = N - L + 1
    B, T = 2, 3
    s = rng.uniform(0.5, 2, (B, T)); U = rng.standard_normal((B, T, L)); V = rng.standard_normal((B, T, K))
    plan = P.Plan(N, L, 0, B, force_long=force)
    g = plan.hankelize(cuda(s), cuda(U), cuda(V)).cpu().numpy()
    for b in range(B):
        for i in range(T):
            assert nrel(g[b, i], oracle.hankelize_rank1(s[b, i], U[b, i], V[b, i])) <= 1e-12


def test_long_hankelize_many_batches(P):
    """150 terms > the 64-term batch: three batches alternating over the caller's stream
    and the plan's second stream (own buffers); every term against the oracle, and the
    same terms one problem at a time (single batch) bit for bit."""
    N, L = 1000, 400
    K = N - L + 1
    B, T = 30, 5
    rng = np.random.default_rng(77)
    s = rng.uniform(0.5, 2, (B, T)); U = rng.standard_normal((B, T, L)); V = rng.standard_normal((B, T, K))
    plan = P.Plan(N, L, 0, B, force_long=True)
    g = plan.hankelize(cuda(s), cuda(U), cuda(V)).cpu().numpy()
    for b in range(B):
        for i in range(T):
            assert nrel(g[b, i], oracle.hankelize_rank1(s[b, i], U[b, i], V[b, i])) <= 1e-12
    one = P.Plan(N, L, 0, 1, force_long=True)
    for b in (0, 13, 29):
        g1 = one.hankelize(cuda(s[b:b + 1]), cuda(U[b:b + 1]), cuda(V[b:b + 1])).cpu().numpy()
        assert np.array_equal(g1[0], g[b])


def test_cfg5_shape_two_batches_sampled(P):
    """BASELINE configs[4] shape, problems 0 and 1 (100 terms: two batches on two streams);
    the last term of each problem against the oracle's direct averaging."""
    c = ssa_inputs.CONFIGS["cfg5"]
    N, L = c["N"], c["L"]
    probs = [ssa_inputs.cfg5_problem(p, N, L, terms=50) for p in (0, 1)]
    sig = np.stack([q[0] for q in probs]); U = np.stack([q[1] for q in probs]); V = np.stack([q[2] for q in probs])
    plan = P.Plan(N, L, 0, 2)
    g = plan.hankelize(cuda(sig), cuda(U), cuda(V)).cpu().numpy()
    for p in (0, 1):
        ref = oracle.hankelize_rank1(sig[p, 49], U[p, 49], V[p, 49])
        assert nrel(g[p, 49], ref) <= 1e-10


def test_cfg5_shape_sampled_terms(P):
    """BASELINE configs[4] shape (N = 262144, L = 131072), problem 0, first 4 terms."""
    c = ssa_inputs.CONFIGS["cfg5"]
    N, L = c["N"], c["L"]
    sig, U, V = ssa_inputs.cfg5_problem(0, N, L, terms=4)
    plan = P.Plan(N, L, 0, 1)
    g = plan.hankelize(cuda(sig[None]), cuda(U[None]), cuda(V[None])).cpu().numpy()
    for i in (0, 3):
        ref = oracle.hankelize_rank1(sig[i], U[i], V[i])
        assert nrel(g[0, i], ref) <= 1e-10


@pytest.mark.parametrize("N,L", [(100003, 37001), (100003, 70001), (131072, 65536), (150001, 100000)])
def test_long_hankelize_radix16_columns(P, N, L):
    """H = 2^16 and 2^17 (N1 = 256): the register radix-16 x 16 column kernels
    (lg_col16_fwd / lg_col16_hank).  Ragged N (odd item stride: the scalar store path),
    L < K and L > K (inputs longer than H / 2 packed points: the non-padded columns), the
    H = 2^17 with L > K; two terms per problem, three problems, every term against
    the oracle's direct averaging (Alg. 4)."""
    K = N - L + 1
    B, T = 3, 2
    rng = np.random.default_rng(N + L)
    s = rng.uniform(0.5, 2, (B, T)); U = rng.standard_normal((B, T, L)); V = rng.standard_normal((B, T, K))
    plan = P.Plan(N, L, 0, B)
    g = plan.hankelize(cuda(s), cuda(U), cuda(V)).cpu().numpy()
    for b, i in ((0, 0), (1, 1), (2, 1)):
        assert nrel(g[b, i], oracle.hankelize_rank1(s[b, i], U[b, i], V[b, i])) <= 1e-12


@pytest.mark.parametrize("N,L,k", [(1024, 512, 10), (600, 250, 8), (4096, 2048, 16), (700, 520, 6)])
def test_long_decompose_vs_oracle(P, N, L, k):
    """The long-series Lanczos path forced onto sizes the Jacobi oracle can do."""
    if N == 1024:
        f = ssa_inputs.cfg1_series(N)
    elif N == 4096:
        f = ssa_inputs.cfg3_like_series(N)
    else:
        rng = np.random.default_rng(5)
        n = np.arange(1, N + 1)
        f = np.sin(2 * np.pi * n / 11.3) + 0.2 * rng.standard_normal(N)
    plan = P.Plan(N, L, k, 1, force_long=True)
    sigma, U, V, info = plan.decompose(cuda(f[None]))
    G = plan.reconstruct(sigma, U, V)
    torch.cuda.synchronize()
    inf = P.info_to_numpy(info)[0]
    assert inf["status"] == 0, inf
    s_ref, U_ref, V_ref, _ = oracle.svd(f, L, k + 1)
    G_ref = np.stack([oracle.hankelize_rank1(s_ref[i], U_ref[i], V_ref[i]) for i in range(k)])
    rep = parity.compare(s_ref, U_ref, V_ref, sigma.cpu().numpy()[0], U.cpu().numpy()[0], V.cpu().numpy()[0], k,
                         G_ref, G.cpu().numpy()[0], recon_scale=np.linalg.norm(f), f=f, L=L)
    assert rep.ok(), rep.failures


def test_decompose_h8192_routes_to_long_path(P):
    """N in (8192, 16384] (M = 16384): the batched decompose kernel would exceed one CTA's
    shared memory, so the plan takes the long path on its own; two series vs the oracle."""
    N, L, k = 9000, 300, 6
    F = np.stack([ssa_inputs.cfg3_like_series(N, seed) for seed in (11, 12)])
    plan = P.Plan(N, L, k, 2)
    assert plan.M == 16384
    sigma, U, V, info = plan.decompose(cuda(F))
    G = plan.reconstruct(sigma, U, V)
    torch.cuda.synchronize()
    for b in range(2):
        inf = P.info_to_numpy(info)[b]
        assert inf["status"] == 0, inf
        s_ref, U_ref, V_ref, _ = oracle.svd(F[b], L, k + 1)
        G_ref = np.stack([oracle.hankelize_rank1(s_ref[i], U_ref[i], V_ref[i]) for i in range(k)])
        rep = parity.compare(s_ref, U_ref, V_ref, sigma.cpu().numpy()[b], U.cpu().numpy()[b], V.cpu().numpy()[b], k,
                             G_ref, G.cpu().numpy()[b], recon_scale=np.linalg.norm(F[b]))
        assert rep.ok(), rep.failures


def test_cfg3_like_long_series_residuals(P):
    """N = 2^17 (cfg3 generator): the oracle cannot do the SVD, so check true residuals
    with its direct product, orthonormality and the Frobenius bound."""
    N, L, k = 1 << 17, 1 << 16, 16
    f = ssa_inputs.cfg3_like_series(N)
    plan = P.Plan(N, L, k, 1)
    sigma, U, V, info = plan.decompose(cuda(f[None]))
    torch.cuda.synchronize()
    inf = P.info_to_numpy(info)[0]
    assert inf["status"] == 0, inf
    s = sigma.cpu().numpy()[0]; Uh = U.cpu().numpy()[0]; Vh = V.cpu().numpy()[0]
    assert np.all(np.diff(s) <= 0)
    assert np.abs(Uh @ Uh.T - np.eye(k)).max() <= 1e-12
    assert np.abs(Vh @ Vh.T - np.eye(k)).max() <= 1e-12
    K = N - L + 1
    cnt = np.minimum.reduce([np.arange(1, N + 1), np.full(N, L), np.full(N, K), N - np.arange(N)])
    assert (s * s).sum() <= (f * f * cnt).sum() * (1 + 1e-12)
    for i in (0, 1, k - 1):
        r1 = np.linalg.norm(oracle.matvec(f, L, Vh[i]) - s[i] * Uh[i])
        r2 = np.linalg.norm(oracle.matvec(f, L, Uh[i], True) - s[i] * Vh[i])
        assert max(r1, r2) <= 1e-11 * s[0], (i, r1, r2)   # 10 tol sigma_1


@pytest.mark.parametrize("N,L,k", [(32768, 16384, 8), (1024, 512, 10)])
def test_decompose_only_enqueues(P, N, L, k):
    """include/ssa.h: ssa_decompose on device buffers only enqueues -- on the long path too
    (the Lanczos loop is one graph launch with device-side decisions, no host sync).  The
    stream is kept busy by a spin kernel first; the call must return while it still is."""
    import time
    f = ssa_inputs.cfg3_like_series(N, 7)
    plan = P.Plan(N, L, k, 1)
    x = cuda(f[None])
    s, U, V, info = plan.decompose(x)          # first call builds the graph (long path)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    torch.cuda._sleep(int(2e9))                # ~1 s of device time ahead of the decompose
    t0 = time.perf_counter()
    plan.decompose(x, s, U, V, info)
    t1 = time.perf_counter()
    busy = not stream.query()
    torch.cuda.synchronize()
    assert busy, "decompose waited for the device"
    assert t1 - t0 < 0.5
    inf = P.info_to_numpy(info)[0]
    assert inf["status"] == 0 and inf["converged"] == 1, inf
