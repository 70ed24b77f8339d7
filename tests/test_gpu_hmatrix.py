"""GPU parity of the heterogeneity matrix (ssa_hmatrix; SURVEY.md §8(f)
#3) against oracle.hmatrix (explicit trajectory matrices, Jacobi SVDs, Eq. (g))."""
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


def test_hmatrix_paper_example(P):
    """The paper's example: Eq. (hseries) with N = 400, Q = 200, B = T = 100, L = 50,
    I = {1, 2}.  I covers the sinusoid pair, so the subspaces (and
    g) are unique even though the two singular values are close."""
    f = ssa_inputs.change_point_series(400, 200, 7)
    G, info = P.hmatrix(torch.from_numpy(f).cuda(), 100, 100, 50, [1, 2])
    G = G.cpu().numpy()
    assert (P.info_to_numpy(info)["status"] == 0).all()
    ref = oracle.hmatrix(f, 100, 100, 50, [1, 2])
    assert np.abs(G - ref).max() <= 1e-9
    assert G[:101, :101].mean() < 0.01 and G[:101, 200:].mean() > 0.1


@pytest.mark.parametrize("N,B,T,L,I", [(300, 80, 60, 30, [1, 2, 3]), (257, 64, 90, 21, [1, 2, 3])])
def test_hmatrix_shapes(P, N, B, T, L, I):
    """B != T, T > B, ragged sizes; an exponential trend + sinusoid (rank 3: the trend
    triple and the sinusoid pair, I covers both clusters)."""
    rng = np.random.default_rng(N)
    n = np.arange(1, N + 1, dtype=float)
    f = np.exp(0.005 * n) + np.sin(2 * np.pi * n / 12) + 0.01 * rng.standard_normal(N)
    G, info = P.hmatrix(torch.from_numpy(f).cuda(), B, T, L, I)
    ref = oracle.hmatrix(f, B, T, L, I)
    assert np.abs(G.cpu().numpy() - ref).max() <= 1e-9


def test_hmatrix_invalid_arguments(P):
    f = torch.zeros(100, dtype=torch.float64, device="cuda")
    for B, T, L, I in [(20, 20, 20, [1]), (20, 10, 12, [1]), (20, 20, 10, [0]), (20, 20, 10, [1, 1]),
                       (120, 20, 10, [1])]:
        with pytest.raises(P.SsaError):
            P.hmatrix(f, B, T, L, I)


@pytest.mark.parametrize("B,T,L", [(120, 120, 30), (60, 25, 25), (41, 120, 40)])
def test_hmatrix_edge_shapes(P, B, T, L):
    """Edge shapes: one base and one test window (B = T = N), single-lag test windows
    (T = L: K2 = 1), the smallest base window (B = L + 1: K_B = 2)."""
    N = 120
    rng = np.random.default_rng(B + T + L)
    n = np.arange(1, N + 1, dtype=float)
    f = np.sin(2 * np.pi * n / 9.0) + 0.5 * np.cos(2 * np.pi * n / 23.0) + 0.05 * rng.standard_normal(N)
    I = [1] if B - L + 1 < 3 else [1, 2]
    G, info = P.hmatrix(torch.from_numpy(f).cuda(), B, T, L, I)
    ref = oracle.hmatrix(f, B, T, L, I)
    assert G.shape == ref.shape
    assert np.abs(G.cpu().numpy() - ref).max() <= 1e-9


def test_hmatrix_plan_reuse_matches_one_shot(P):
    """A plan executed on two different series gives exactly the one-shot results."""
    f1 = ssa_inputs.change_point_series(300, 150, 1)
    f2 = ssa_inputs.change_point_series(300, 100, 2)
    hm = P.HMatrix(300, 70, 60, 30, [1, 2])
    for f in (f1, f2):
        x = torch.from_numpy(f).cuda()
        G, _ = hm(x)
        G1, _ = P.hmatrix(x, 70, 60, 30, [1, 2])
        assert torch.equal(G, G1)
    hm.close()
