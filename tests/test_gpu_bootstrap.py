"""GPU parity of the bootstrap study (ssa_bootstrap)
against oracle.bootstrap (Jacobi SVD of each replicate, explicit grouping + averaging)."""
import numpy as np
import pytest

import oracle
import ssa_inputs

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_0911_4498_b200 as pkg
    return pkg


@pytest.mark.parametrize("N,L,R,noise", [(300, 150, 12, 0.5), (257, 100, 9, 0.2)])
def test_bootstrap_vs_oracle(P, N, L, R, noise):
    """Rank-5 series of the paper's study (periods in n, R17) with seeded noise;
    the 5 signal triples are well separated from the noise, so every replicate's rank-5
    reconstruction is unique; reconstructions, mean, variance and MSE against the oracle."""
    d = 5
    f = ssa_inputs.bootstrap_series(N)
    eps = ssa_inputs.bootstrap_noise(R, N)
    plan = P.Plan(N, L, d, R)
    G = torch.empty(R, N, dtype=torch.float64, device="cuda")
    mean, var, mse = plan.bootstrap(torch.from_numpy(f).cuda(), torch.from_numpy(eps).cuda(), noise, G=G)
    m0, v0, e0, G0 = oracle.bootstrap(f, eps, noise, L, d)
    scale = np.linalg.norm(f)
    for r in range(R):
        assert np.linalg.norm(G.cpu().numpy()[r] - G0[r]) <= 1e-9 * scale
    assert np.abs(mean.cpu().numpy() - m0).max() <= 1e-9 * np.abs(f).max()
    assert np.abs(var.cpu().numpy() - v0).max() <= 1e-8 * v0.max()
    assert np.abs(mse.cpu().numpy() - e0).max() <= 1e-8 * e0.max()


def test_bootstrap_noise_free_is_exact(P):
    """noise_sigma = 0: every replicate is F (rank 5), so mean = F, var = mse = 0 (closed form)."""
    N, L, R = 200, 100, 4
    f = ssa_inputs.bootstrap_series(N)
    eps = ssa_inputs.bootstrap_noise(R, N)
    plan = P.Plan(N, L, 5, R)
    mean, var, mse = plan.bootstrap(torch.from_numpy(f).cuda(), torch.from_numpy(eps).cuda(), 0.0)
    assert np.abs(mean.cpu().numpy() - f).max() <= 1e-10 * np.abs(f).max()
    assert var.cpu().numpy().max() <= 1e-18 * np.abs(f).max() ** 2


def test_bootstrap_single_replicate(P):
    """R = 1: the variance is defined as 0, the MSE is the squared error of the one replicate."""
    N, L = 150, 60
    f = ssa_inputs.bootstrap_series(N)
    eps = ssa_inputs.bootstrap_noise(1, N)
    plan = P.Plan(N, L, 5, 1)
    G = torch.empty(1, N, dtype=torch.float64, device="cuda")
    mean, var, mse = plan.bootstrap(torch.from_numpy(f).cuda(), torch.from_numpy(eps).cuda(), 0.3, G=G)
    g = G.cpu().numpy()[0]
    assert np.array_equal(mean.cpu().numpy(), g)
    assert not var.cpu().numpy().any()
    assert np.allclose(mse.cpu().numpy(), (g - f) ** 2, rtol=1e-15, atol=0)
