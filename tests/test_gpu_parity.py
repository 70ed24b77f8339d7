"""GPU parity: the CUDA path through the C-ABI (paper_0911_4498_b200 -> libssa.so) against
the CPU oracle (oracle/), on the same seeded inputs.  Tolerances (BASELINE.json north_star,
DESIGN.md §Parity):
  * matvec: normwise ‖y − y°‖/‖y°‖ ≤ 1e-12
  * hankelization: normwise ≤ 1e-12 relative to ‖g°‖
  * σ: relative ≤ 1e-10; sine angles ≤ 1e-8 (well separated / non-straddling clusters);
    reconstructions ‖g − g°‖ ≤ 1e-9 ‖F‖ (per triple / per cluster).
"""
import json
import os

import numpy as np
import pytest

import oracle
import parity
import ssa_inputs

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


@pytest.fixture(scope="module")
def P():
    import paper_0911_4498_b200 as pkg
    assert torch.cuda.is_available()
    return pkg


def cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def nrel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


# ----------------------------------------------------------------------------- matvec
@pytest.mark.parametrize("case", GOLD["matvec"])
def test_matvec_golden(P, case):
    f = np.array(case["f"], float)
    plan = P.Plan(len(f), case["L"], 0, 1)
    spec = plan.spectrum(cuda(f[None]))
    y = plan.matvec(spec, cuda(np.array(case["x"], float)[None]), transpose=case["transpose"])
    assert np.allclose(y.cpu().numpy()[0], case["y"], rtol=0, atol=1e-13), case["cite"]


@pytest.mark.parametrize("N", [3, 4, 5, 7, 16, 17, 33, 64, 100])
def test_matvec_all_windows_vs_oracle(P, N):
    rng = np.random.default_rng(1000 + N)
    for L in range(2, N):
        K = N - L + 1
        B = 3
        F = rng.standard_normal((B, N))
        x = rng.standard_normal((B, K)); u = rng.standard_normal((B, L))
        plan = P.Plan(N, L, 0, B)
        spec = plan.spectrum(cuda(F))
        y = plan.matvec(spec, cuda(x)).cpu().numpy()
        z = plan.matvec(spec, cuda(u), transpose=True).cpu().numpy()
        for b in range(B):
            assert nrel(y[b], oracle.matvec(F[b], L, x[b])) <= 1e-12
            assert nrel(z[b], oracle.matvec(F[b], L, u[b], True)) <= 1e-12


def test_spectrum_matches_dft(P):
    rng = np.random.default_rng(5)
    for N in (5, 64, 1000, 4096):
        F = rng.standard_normal((2, N))
        plan = P.Plan(N, N // 2, 0, 2)
        spec = plan.spectrum(cuda(F)).cpu().numpy()
        S = spec[..., 0] + 1j * spec[..., 1]
        ref = np.fft.rfft(F, plan.M)   # library DFT, debugging cross-check only
        assert np.abs(S - ref).max() <= 1e-13 * np.abs(ref).max()


def test_matvec_cfg4_sample(P):
    """cfg4 shape (N=8192, L=4096), series 0..7 of the seeded generator."""
    c = ssa_inputs.CONFIGS["cfg4"]
    N, L = c["N"], c["L"]
    F, V, U = ssa_inputs.cfg4_batch(0, 8, N, L)
    plan = P.Plan(N, L, 0, 8)
    spec = plan.spectrum(cuda(F))
    y = plan.matvec(spec, cuda(V)).cpu().numpy()
    z = plan.matvec(spec, cuda(U), transpose=True).cpu().numpy()
    for b in range(8):
        assert nrel(y[b], oracle.matvec(F[b], L, V[b])) <= 1e-12
        assert nrel(z[b], oracle.matvec(F[b], L, U[b], True)) <= 1e-12


@pytest.mark.parametrize("N,L", [(8192, 4096), (7000, 3000), (5000, 4000), (4097, 2), (8192, 4095), (6001, 2999)])
def test_matvec_register_path_vs_oracle(P, N, L):
    """M = 8192 (H = 4096): the register-resident radix-16 correlation (fft_reg.cuh) when
    the input fits the zero-padded half (n_in <= 4097), the shared-memory path otherwise;
    ragged N, both directions, several series per launch."""
    rng = np.random.default_rng(N + L)
    K = N - L + 1
    B = 3
    F = rng.standard_normal((B, N)); v = rng.standard_normal((B, K)); u = rng.standard_normal((B, L))
    plan = P.Plan(N, L, 0, B)
    assert plan.M == 8192
    spec = plan.spectrum(cuda(F))
    y = plan.matvec(spec, cuda(v)).cpu().numpy()
    z = plan.matvec(spec, cuda(u), transpose=True).cpu().numpy()
    for b in range(B):
        assert nrel(y[b], oracle.matvec(F[b], L, v[b])) <= 1e-12
        assert nrel(z[b], oracle.matvec(F[b], L, u[b], True)) <= 1e-12


@pytest.mark.parametrize("N,L,nvec,force", [(8192, 4096, 5, False), (6001, 2999, 3, False), (4096, 2048, 4, False),
                                              (1000, 333, 7, False), (8192, 4095, 2, False), (4096, 1500, 3, True)])
def test_matvec_multi_vs_oracle(P, N, L, nvec, force):
    """ssa_matvec_multi: nvec vectors per series against that series' spectrum (item b of
    the launch -> series b / nvec), register path (M = 8192), shared-memory path, and the
    four-step path (force_long), both directions, against the oracle's explicit product."""
    rng = np.random.default_rng(N + 7 * nvec)
    K = N - L + 1
    B = 3
    F = rng.standard_normal((B, N)); v = rng.standard_normal((B, nvec, K)); u = rng.standard_normal((B, nvec, L))
    plan = P.Plan(N, L, 0, B, force_long=force)
    spec = plan.spectrum(cuda(F))
    y = plan.matvec_multi(spec, cuda(v)).cpu().numpy()
    z = plan.matvec_multi(spec, cuda(u), transpose=True).cpu().numpy()
    for b in range(B):
        for i in range(nvec):
            assert nrel(y[b, i], oracle.matvec(F[b], L, v[b, i])) <= 1e-12
            assert nrel(z[b, i], oracle.matvec(F[b], L, u[b, i], True)) <= 1e-12
    # one vector per series: identical bits to ssa_matvec
    y1 = plan.matvec(spec, cuda(v[:, 0])).cpu().numpy()
    assert np.array_equal(y1, plan.matvec_multi(spec, cuda(v[:, :1])).cpu().numpy()[:, 0])


def test_matvec_adjoint(P):
    rng = np.random.default_rng(6)
    N, L = 4096, 2048
    K = N - L + 1
    F = rng.standard_normal((4, N)); v = rng.standard_normal((4, K)); u = rng.standard_normal((4, L))
    plan = P.Plan(N, L, 0, 4)
    spec = plan.spectrum(cuda(F))
    Xv = plan.matvec(spec, cuda(v)).cpu().numpy()
    XTu = plan.matvec(spec, cuda(u), transpose=True).cpu().numpy()
    for b in range(4):
        lhs, rhs = np.dot(Xv[b], u[b]), np.dot(v[b], XTu[b])
        assert abs(lhs - rhs) <= 1e-12 * np.linalg.norm(Xv[b]) * np.linalg.norm(u[b])


# ----------------------------------------------------------------------------- hankelize
@pytest.mark.parametrize("case", GOLD["hankelize_rank1"])
def test_hankelize_golden(P, case):
    u = np.array(case["u"], float); v = np.array(case["v"], float)
    N = len(u) + len(v) - 1
    plan = P.Plan(N, len(u), 0, 1)
    g = plan.hankelize(cuda([[case["sigma"]]]), cuda(u[None, None]), cuda(v[None, None])).cpu().numpy()
    assert np.allclose(g[0, 0], case["g"], rtol=0, atol=1e-14), case["cite"]


@pytest.mark.parametrize("N,L", [(3, 2), (5, 3), (10, 3), (10, 8), (33, 17), (64, 5), (100, 90), (1000, 500),
                                 (4096, 2048), (8192, 3000), (16384, 8192)])
def test_hankelize_vs_oracle(P, N, L):
    rng = np.random.default_rng(N * 7 + L)
    K = N - L + 1
    B, T = 2, 3
    s = rng.uniform(0.5, 2, (B, T)); U = rng.standard_normal((B, T, L)); V = rng.standard_normal((B, T, K))
    plan = P.Plan(N, L, 0, B)
    g = plan.hankelize(cuda(s), cuda(U), cuda(V)).cpu().numpy()
    for b in range(B):
        for i in range(T):
            ref = oracle.hankelize_rank1(s[b, i], U[b, i], V[b, i])
            assert nrel(g[b, i], ref) <= 1e-12


# ----------------------------------------------------------------------------- decompose
def run_decompose(P, F, L, k, **kw):
    B, N = F.shape
    plan = P.Plan(N, L, k, B, **kw)
    sigma, U, V, info = plan.decompose(cuda(F))
    G = plan.reconstruct(sigma, U, V)
    torch.cuda.synchronize()
    return (sigma.cpu().numpy(), U.cpu().numpy(), V.cpu().numpy(), G.cpu().numpy(),
            P.info_to_numpy(info))


def check_against_oracle(f, L, k, s, U, V, G, sigma_tol=1e-10, recon_scale=None, residuals=True):
    s_ref, U_ref, V_ref, _ = oracle.svd(f, L, k + 1)
    G_ref = np.stack([oracle.hankelize_rank1(s_ref[i], U_ref[i], V_ref[i]) for i in range(k)])
    scale = np.linalg.norm(f) if recon_scale is None else recon_scale
    rep = parity.compare(s_ref, U_ref, V_ref, s, U, V, k, G_ref, G, recon_scale=scale, sigma_tol=sigma_tol,
                         f=f if residuals else None, L=L)
    assert rep.ok(), rep.failures
    return rep


def test_decompose_cfg1(P):
    c = ssa_inputs.CONFIGS["cfg1"]
    f = ssa_inputs.cfg1_series(c["N"])
    s, U, V, G, info = run_decompose(P, f[None], c["L"], c["k"])
    assert info[0]["status"] == 0 and info[0]["converged"] == 1, info
    assert info[0]["max_residual"] <= 1e-12
    rep = check_against_oracle(f, c["L"], c["k"], s[0], U[0], V[0], G[0])
    print("cfg1 worst:", rep.worst(), "steps", info[0]["steps"])


@pytest.mark.parametrize("reorth", [1, 2, 3])
@pytest.mark.parametrize("N,L,k", [(40, 20, 3), (41, 30, 5), (64, 10, 4), (100, 50, 8), (127, 64, 6),
                                   (300, 100, 10), (513, 256, 12), (2000, 1700, 16)])
def test_decompose_random_shapes(P, N, L, k, reorth):
    """All reorthogonalization modes (FRO: CGS + DGKS, CGS2; PRO) against the oracle;
    Ritz vectors orthonormal to working precision (FRO) / to the PRO level eps^(3/4)
    (R22)."""
    rng = np.random.default_rng(N + 13 * L)
    n = np.arange(1, N + 1)
    B = 3
    F = np.stack([np.sin(2 * np.pi * n / 9.7) + 0.5 * np.cos(2 * np.pi * n / 31) + 0.3 * rng.standard_normal(N)
                  for _ in range(B)])
    s, U, V, G, info = run_decompose(P, F, L, k, reorth=reorth)
    for b in range(B):
        assert info[b]["status"] == 0, info[b]
        check_against_oracle(F[b], L, k, s[b], U[b], V[b], G[b])
        otol = 1e-13 if reorth != 3 else 1e-12
        assert np.abs(U[b] @ U[b].T - np.eye(k)).max() <= otol
        assert np.abs(V[b] @ V[b].T - np.eye(k)).max() <= otol


def test_decompose_full_rank_small_exact(P):
    """k = min(L, K): the Krylov space is exhausted; all triples and Σ g_i = F."""
    rng = np.random.default_rng(21)
    for N, L in [(12, 5), (20, 10), (25, 20)]:
        f = rng.standard_normal(N)
        k = min(L, N - L + 1)
        s, U, V, G, info = run_decompose(P, f[None], L, k)
        assert info[0]["status"] == 0, info
        check_against_oracle(f, L, k, s[0], U[0], V[0], G[0])
        assert np.allclose(G[0].sum(axis=0), f, atol=1e-11 * np.abs(f).max())


def test_decompose_rank_deficient(P):
    """Exact sinusoid: rank 2, Lanczos breaks down; σ₃.. = 0 (restart path)."""
    N, L, k = 200, 100, 5
    n = np.arange(1, N + 1)
    f = 1.5 * np.sin(2 * np.pi * n / 10 + 0.3)
    s, U, V, G, info = run_decompose(P, f[None], L, k)
    assert info[0]["breakdown_step"] > 0 and info[0]["status"] == 0
    s_ref = oracle.svd(f, L, 3)[0]
    assert np.allclose(s[0, :2], s_ref[:2], rtol=1e-12)
    assert s[0, 2] <= 1e-10 * s[0, 0]
    assert np.allclose(G[0, 0] + G[0, 1], f, atol=1e-10)


def test_decompose_nonfinite_reported(P):
    f = np.random.default_rng(3).standard_normal((2, 64))
    f[1, 10] = np.nan
    s, U, V, G, info = run_decompose(P, f, 32, 3)
    assert info[0]["status"] == 0
    assert info[1]["status"] == 1  # SSA_ERR_INVALID_ARGUMENT


def test_invalid_arguments(P):
    with pytest.raises(P.SsaError):
        P.Plan(2, 1, 1, 1)
    with pytest.raises(P.SsaError):
        P.Plan(10, 10, 1, 1)
    with pytest.raises(P.SsaError):
        P.Plan(10, 5, 7, 1)   # k > min(L, K) = 5 -> 6? min(5,6)=5
    with pytest.raises(P.SsaError):
        P.Plan(10, 5, 1, 0)


def test_run_host_matches_device(P):
    c = ssa_inputs.CONFIGS["cfg1"]
    f = ssa_inputs.cfg1_series(c["N"])[None]
    plan = P.Plan(c["N"], c["L"], c["k"], 1)
    s, U, V, G, info = plan.run_host(f)
    sd, Ud, Vd, Gd, infod = run_decompose(P, f, c["L"], c["k"])
    assert np.array_equal(s, sd) and np.array_equal(G, Gd)


def test_decompose_chunked_matches_single_chunk(P, monkeypatch):
    """A plan whose workspace holds fewer series than the batch loops over chunks; every
    series keeps its global index (start vector), so the results equal one chunk's."""
    N, L, k, B = 400, 150, 6, 12
    F = np.stack([ssa_inputs.cfg2_series(i, N) for i in range(B)])
    s1, U1, V1, G1, i1 = run_decompose(P, F, L, k)
    monkeypatch.setenv("SSA_MAX_CHUNK", "5")
    s2, U2, V2, G2, i2 = run_decompose(P, F, L, k)
    assert np.array_equal(s1, s2) and np.array_equal(U1, U2) and np.array_equal(G1, G2)
    check_against_oracle(F[7], L, k, s2[7], U2[7], V2[7], G2[7])


@pytest.mark.parametrize("svd", ["tgk", "qr"])
def test_decompose_k_max_and_svd_options(P, svd):
    """k = 32 (the batched path's maximum) with both bidiagonal SVD methods (TGK twisted
    factorization + inverse iteration fallback; implicit-shift QR)."""
    rng = np.random.default_rng(32)
    N, L, k = 700, 300, 32
    n = np.arange(1, N + 1)
    f = (np.sin(2 * np.pi * n / 17) + 0.7 * np.sin(2 * np.pi * n / 45) + 0.02 * n ** 0.5
         + 0.4 * rng.standard_normal(N))
    s, U, V, G, info = run_decompose(P, f[None], L, k, svd=svd)
    assert info[0]["status"] == 0, info
    check_against_oracle(f, L, k, s[0], U[0], V[0], G[0])
    assert np.abs(U[0] @ U[0].T - np.eye(k)).max() <= 1e-13


def test_plans_of_different_sizes_interleaved(P):
    """Kernel shared-memory limits are per function, plans are not: a small plan created
    after a large one must not lower the limit the large plan's launches need."""
    c = ssa_inputs.CONFIGS["cfg1"]
    f = ssa_inputs.cfg1_series(c["N"])[None]
    big = P.Plan(c["N"], c["L"], c["k"], 1)
    s1 = big.decompose(cuda(f))[0].cpu().numpy()
    small = P.Plan(40, 20, 3, 1)
    small.decompose(cuda(np.sin(np.arange(1, 41) / 3.0)[None]))
    s2 = big.decompose(cuda(f))[0].cpu().numpy()
    torch.cuda.synchronize()
    assert np.array_equal(s1, s2)


@pytest.mark.parametrize("B", [512, 2100])
def test_run_host_pipelined_matches_device(P, B):
    """ssa_run_host splits batches >= 512 into slices (a partial last slice re-runs an
    overlap) on two compute streams, inputs on a copy stream, outputs on another; every
    output must equal the single-launch device path bit for bit (per-series arithmetic is
    independent and fixed-order)."""
    N, L, k = 300, 120, 4
    F = np.stack([ssa_inputs.cfg2_series(i, N) for i in range(B)])
    plan = P.Plan(N, L, k, B)
    s, U, V, G, info = plan.run_host(F)
    sd, Ud, Vd, Gd, infod = run_decompose(P, F, L, k)
    assert np.array_equal(s, sd) and np.array_equal(U, Ud) and np.array_equal(V, Vd) and np.array_equal(G, Gd)
    assert np.array_equal(info["steps"], infod["steps"])


# ----------------------------------------------------------------------------- cfg2 full size
def test_decompose_cfg2_full_batch_sampled(P):
    """BASELINE configs[1] at full size in bench.py's launch configuration (batch 4096,
    N=4096, L=2048, k=16): sampled series 0, 1234, 4095 against oracle results written by
    oracle/make_golden.py (Jacobi + direct averaging, CPU); all series: convergence,
    ordering and the Frobenius bound Σσ² ≤ ‖X‖_F²."""
    import glob
    c = ssa_inputs.CONFIGS["cfg2"]
    N, L, k, B = c["N"], c["L"], c["k"], c["batch"]
    F = ssa_inputs.cfg2_batch(0, B, N)
    s, U, V, G, info = run_decompose(P, F, L, k)
    assert np.all(info["status"] == 0), np.unique(info["status"], return_counts=True)
    assert np.all(info["max_residual"] <= 1e-12)
    assert np.all(np.diff(s, axis=1) <= 0)
    K = N - L + 1
    cnt = np.minimum.reduce([np.arange(1, N + 1), np.full(N, L), np.full(N, K), N - np.arange(N)])
    fro2 = (F * F * cnt).sum(axis=1)
    assert np.all((s * s).sum(axis=1) <= fro2 * (1 + 1e-12))
    files = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "oracle_cfg2_*.npz")))
    assert files, "run python -m oracle.make_golden"
    for p in files:
        d = np.load(p)
        i = int(d["series_index"])
        rep = parity.compare(d["sigma"], d["U"], d["V"], s[i], U[i], V[i], k, d["G"], G[i],
                             recon_scale=float(d["norm_f"]))
        assert rep.ok(), (i, rep.failures)
        print(f"cfg2 series {i}: steps {info[i]['steps']} worst {rep.worst()}")


# ----------------------------------------------------------------------------- grouping
@pytest.mark.parametrize("N,L,k,force", [(1024, 512, 10, False), (700, 520, 6, False), (4096, 2048, 16, False),
                                         (10000, 3000, 8, False), (1000, 400, 6, True)])
def test_reconstruct_grouped_vs_oracle(P, N, L, k, force):
    """Grouped reconstruction of seeded random triples against the
    oracle's explicit X_I + averaging: shared-memory accumulation of the group's product
    spectra (M <= 8192), the elementary-then-sum route (M = 16384, forced long path);
    groups with several triples, a singleton, an empty group and dropped triples."""
    rng = np.random.default_rng(N + 7 * k)
    K = N - L + 1
    B = 3
    s = np.sort(rng.uniform(0.1, 3, (B, k)))[:, ::-1].copy()
    U = rng.standard_normal((B, k, L)); V = rng.standard_normal((B, k, K))
    groups = np.array([(i % 3) if i < k - 1 else -1 for i in range(k)], dtype=np.int32)
    groups[0] = 3                     # singleton group 3
    ng = 5                            # group 4 empty
    plan = P.Plan(N, L, k, B, force_long=force)
    G = plan.reconstruct_grouped(cuda(s), cuda(U), cuda(V), groups, ngroups=ng).cpu().numpy()
    assert not G[:, 4].any()          # the empty group
    for b in range(B):
        ref = oracle.grouped(s[b], U[b], V[b], groups, 4)
        for g in range(4):
            assert nrel(G[b, g], ref[g]) <= 1e-12
    E = plan.reconstruct(cuda(s), cuda(U), cuda(V)).cpu().numpy()
    for b in range(B):
        for g in range(4):
            assert nrel(G[b, g], E[b][groups == g].sum(axis=0)) <= 1e-13


def test_reconstruct_grouped_signal_of_cfg1(P):
    """cfg1 series: the two sinusoid pairs and the trend grouped from the decomposition
    (triples 0 | 1,2 | 3,4) equal the oracle's grouping of its own Jacobi triples (the
    groups span whole clusters, so the result is unique); together with the residual
    group they sum to the series."""
    c = ssa_inputs.CONFIGS["cfg1"]
    N, L, k = c["N"], c["L"], c["k"]
    f = ssa_inputs.cfg1_series(N)
    plan = P.Plan(N, L, k, 1)
    sg, U, V, info = plan.decompose(cuda(f[None]))
    groups = np.array([0, 1, 1, 2, 2] + [3] * (k - 5), dtype=np.int32)
    G = plan.reconstruct_grouped(sg, U, V, groups).cpu().numpy()[0]
    s_o, U_o, V_o, _ = oracle.svd(f, L, k)
    ref = oracle.grouped(s_o, U_o, V_o, groups, 4)
    for g in range(3):
        assert np.linalg.norm(G[g] - ref[g]) <= 1e-9 * np.linalg.norm(f)
