"""GPU parity of the thick-restarted Lanczos bidiagonalization (restart_dim > 0;
PAPER.md:435-446 sec 3.3 "restarting schemes"; R23) against the CPU oracle
(explicit X + one-sided Jacobi + direct averaging), with the tolerances of
test_gpu_parity.py: sigma relative <= 1e-10, sine angles <= 1e-8, reconstructions
<= 1e-9 ||F||, true residuals <= 1e-11 sigma_1 through the oracle's explicit product,
Ritz vectors orthonormal.  Every case restarts at least once (info.reserved counts the
thick restarts), so the arrow-shaped projected matrix, the dense Jacobi SVD and the in-
place basis rotation are all exercised."""
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
    assert torch.cuda.is_available()
    return pkg


def cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def run(P, F, L, k, **kw):
    B, N = F.shape
    plan = P.Plan(N, L, k, B, **kw)
    sigma, U, V, info = plan.decompose(cuda(F))
    G = plan.reconstruct(sigma, U, V)
    torch.cuda.synchronize()
    return sigma.cpu().numpy(), U.cpu().numpy(), V.cpu().numpy(), G.cpu().numpy(), P.info_to_numpy(info)


def check(f, L, k, s, U, V, G):
    s_ref, U_ref, V_ref, _ = oracle.svd(f, L, k + 1)
    G_ref = np.stack([oracle.hankelize_rank1(s_ref[i], U_ref[i], V_ref[i]) for i in range(k)])
    rep = parity.compare(s_ref, U_ref, V_ref, s, U, V, k, G_ref, G, recon_scale=np.linalg.norm(f), f=f, L=L)
    assert rep.ok(), rep.failures
    return rep


def test_trl_cfg1(P):
    """BASELINE configs[0] (N = 1024, L = 512, k = 10) with a Krylov dimension of 28: the
    unrestarted run needs ~62 steps, so this restarts several times."""
    c = ssa_inputs.CONFIGS["cfg1"]
    f = ssa_inputs.cfg1_series(c["N"])
    s, U, V, G, info = run(P, f[None], c["L"], c["k"], restart_dim=28, restart_keep=14)
    i = info[0]
    assert i["status"] == 0 and i["converged"] == 1, i
    assert i["reserved"] >= 2, i  # thick restarts taken
    assert i["max_residual"] <= 1e-12
    rep = check(f, c["L"], c["k"], s[0], U[0], V[0], G[0])
    print("cfg1 TRL:", rep.worst(), "steps", i["steps"], "restarts", i["reserved"])


@pytest.mark.parametrize("dp", [(12, 4), (8, 2), (2.5, 1.25)])
@pytest.mark.parametrize("N,L,k", [(300, 100, 6), (513, 256, 8), (2000, 1700, 8), (1024, 512, 16)])
def test_trl_shapes(P, N, L, k, dp):
    """Several windows (L < K and L > K), Krylov dimensions d and keep counts p: d = k + 12,
    p = k + 4; d = k + 8, p = k + 2 (few new vectors per cycle); d = 2.5 k, p = 1.25 k (the
    model's ratio).  (With p = k and d = k + 4 the restarted iteration stalls on the
    clustered noise triples of a k = 16 problem: keep a few vectors beyond k.)"""
    if dp[0] < 3:
        d, p = int(dp[0] * k), int(dp[1] * k)
    else:
        d, p = k + int(dp[0]), k + int(dp[1])
    rng = np.random.default_rng(N + 7 * L + d)
    n = np.arange(1, N + 1)
    B = 2
    F = np.stack([np.sin(2 * np.pi * n / 9.7 + b) + 0.5 * np.cos(2 * np.pi * n / 31) + 0.3 * rng.standard_normal(N)
                  for b in range(B)])
    s, U, V, G, info = run(P, F, L, k, restart_dim=d, restart_keep=p)
    for b in range(B):
        assert info[b]["status"] == 0, info[b]
        assert info[b]["reserved"] >= 1 or info[b]["steps"] <= d, info[b]
        check(F[b], L, k, s[b], U[b], V[b], G[b])
        assert np.abs(U[b] @ U[b].T - np.eye(k)).max() <= 1e-13
        assert np.abs(V[b] @ V[b].T - np.eye(k)).max() <= 1e-13


def test_trl_cfg2_series_match_unrestarted(P):
    """cfg2 series (BASELINE configs[1] shape, k = 16) with d = 40, p = 20 (the numpy
    model's trl:40:20, tools/model_reorth.py): sigma, vectors and reconstructions agree
    with the unrestarted FRO run and with the oracle's stored cfg2 results."""
    import glob
    import os
    c = ssa_inputs.CONFIGS["cfg2"]
    N, L, k = c["N"], c["L"], c["k"]
    files = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "oracle_cfg2_*.npz")))
    assert files
    idx = [int(np.load(p)["series_index"]) for p in files]
    F = np.stack([ssa_inputs.cfg2_series(i, N) for i in idx])
    s, U, V, G, info = run(P, F, L, k, restart_dim=40, restart_keep=20)
    for j, p in enumerate(files):
        d = np.load(p)
        assert info[j]["status"] == 0 and info[j]["reserved"] >= 1, info[j]
        rep = parity.compare(d["sigma"], d["U"], d["V"], s[j], U[j], V[j], k, d["G"], G[j],
                             recon_scale=float(d["norm_f"]))
        assert rep.ok(), (idx[j], rep.failures)
        print(f"cfg2 series {idx[j]} TRL: steps {info[j]['steps']} restarts {info[j]['reserved']} worst {rep.worst()}")


def test_trl_rank_deficient_and_exact_pairs(P):
    """A rank-2 sinusoid whose period divides L and K (sigma_1 = sigma_2 = A sqrt(LK)/2
    exactly, SURVEY.md 8(c) closed forms): the Krylov space is exhausted before the first
    restart; breakdown restarts then fill the basis with the zero singular directions."""
    N, L, k = 239, 120, 4
    n = np.arange(1, N + 1)
    f = 2.0 * np.sin(2 * np.pi * n / 12 + 0.4)
    s, U, V, G, info = run(P, f[None], L, k, restart_dim=10, restart_keep=5)
    assert info[0]["status"] == 0, info[0]
    closed = 2.0 * np.sqrt(L * (N - L + 1)) / 2
    assert abs(s[0, 0] - closed) <= 1e-12 * closed and abs(s[0, 1] - closed) <= 1e-12 * closed
    assert s[0, 2] <= 1e-10 * closed
    assert np.allclose(G[0, 0] + G[0, 1], f, atol=1e-10 * np.abs(f).max())


def test_trl_not_converged_reports(P):
    """A total step cap below what the tolerance needs: NOT_CONVERGED with the best Ritz
    triples written, as the unrestarted path."""
    c = ssa_inputs.CONFIGS["cfg1"]
    f = ssa_inputs.cfg1_series(c["N"])
    s, U, V, G, info = run(P, f[None], c["L"], c["k"], restart_dim=20, restart_keep=12, max_steps=24)
    assert info[0]["status"] == 2 and info[0]["converged"] == 0, info[0]
    assert info[0]["steps"] == 24
    s_ref = oracle.svd(f, c["L"], 2)[0]
    assert abs(s[0, 0] - s_ref[0]) <= 1e-8 * s_ref[0]


def test_trl_invalid_options(P):
    for d, p in [(5, 0), (600, 0), (30, 9), (30, 29)]:
        with pytest.raises(P.SsaError):
            P.Plan(1024, 512, 10, 1, restart_dim=d, restart_keep=p)
