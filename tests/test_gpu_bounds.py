"""Out-of-bounds writes into caller buffers, and writes to inputs (include/ssa.h: "inputs are
read-only", every output has exactly the shape written next to it).  compute-sanitizer is
closed on this pool (profiles/r02/sanitizer_memcheck_closed.txt), so each output buffer of
the C-ABI calls is a view into the middle of a larger allocation whose guard zones are
filled with a sentinel; after the call (and a device synchronize) the guard zones must be
bit-identical, and so must every input.  Ragged shapes (odd K, N not a power of two,
L > K), both FFT paths (register / shared-memory / four-step), batched and long-series
decompose, thick restart, reconstruct, hankelize, matvec and matvec_multi."""
import numpy as np
import pytest

import ssa_inputs

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

GUARD = 4096          # doubles of guard zone on each side
SENT = 1.2345678e300  # sentinel value of the guard zones


@pytest.fixture(scope="module")
def P():
    import paper_0911_4498_b200 as pkg
    assert torch.cuda.is_available()
    return pkg


class Guarded:
    """A float64 (or uint8) CUDA buffer of `shape` with sentinel guard zones around it."""

    def __init__(self, shape, dtype=torch.float64):
        n = int(np.prod(shape))
        self.dtype = dtype
        if dtype == torch.float64:
            self.big = torch.full((n + 2 * GUARD,), SENT, dtype=dtype, device="cuda")
        else:
            self.big = torch.full((n + 2 * GUARD,), 0xA5, dtype=dtype, device="cuda")
        self.n = n
        self.t = self.big[GUARD:GUARD + n].view(*shape)

    def check(self, name):
        torch.cuda.synchronize()
        lo = self.big[:GUARD].cpu().numpy()
        hi = self.big[GUARD + self.n:].cpu().numpy()
        ref = SENT if self.dtype == torch.float64 else 0xA5
        assert np.all(lo == ref), f"{name}: write below the buffer"
        assert np.all(hi == ref), f"{name}: write past the end of the buffer"


def _series(B, N, seed):
    rng = np.random.default_rng(seed)
    n = np.arange(1, N + 1)
    f = np.sin(2 * np.pi * n / 17.0)[None, :] + 0.5 * np.cos(2 * np.pi * n / 5.3)[None, :] \
        + 0.1 * rng.standard_normal((B, N))
    return torch.from_numpy(f).cuda()


@pytest.mark.parametrize("N,L,k,B,opts", [
    (1000, 333, 6, 3, {}),                          # ragged, shared-memory FFT path
    (1024, 700, 5, 2, {}),                          # L > K (transposed)
    (4096, 2048, 16, 5, {}),                        # cfg2 shape
    (8000, 4001, 8, 2, {}),                         # M = 8192, odd K
    (3000, 1400, 8, 2, {"force_long": True}),       # four-step long path, batch served serially
    (2000, 900, 6, 3, {"restart_dim": 24, "restart_keep": 12}),  # thick restart
])
def test_decompose_reconstruct_stay_in_bounds(P, N, L, k, B, opts):
    K = N - L + 1
    f = _series(B, N, N + L)
    f0 = f.clone()
    plan = P.Plan(N, L, k, B, **opts)
    sig, U, V = Guarded((B, k)), Guarded((B, k, L)), Guarded((B, k, K))
    info = Guarded((B, P.INFO_DTYPE.itemsize), dtype=torch.uint8)
    plan.decompose(f, sig.t, U.t, V.t, info.t)
    for g, name in ((sig, "sigma"), (U, "U"), (V, "V"), (info, "info")):
        g.check(name)
    assert torch.equal(f, f0), "decompose wrote to its input series"
    inf = P.info_to_numpy(info.t)
    assert np.all(inf["status"] == 0), inf
    s0, U0, V0 = sig.t.clone(), U.t.clone(), V.t.clone()
    G = Guarded((B, k, N))
    plan.reconstruct(sig.t, U.t, V.t, out=G.t)
    G.check("reconstruct out")
    assert torch.equal(sig.t, s0) and torch.equal(U.t, U0) and torch.equal(V.t, V0), "reconstruct wrote to inputs"
    assert torch.isfinite(G.t).all()


@pytest.mark.parametrize("N,L,force", [(8192, 4096, False), (8192, 4095, False), (6001, 2999, False),
                                       (1000, 333, False), (4097, 2, False), (5000, 2500, True)])
def test_spectrum_matvec_stay_in_bounds(P, N, L, force):
    K = N - L + 1
    B, nv = 3, 4
    rng = np.random.default_rng(N * 7 + L)
    f = torch.from_numpy(rng.standard_normal((B, N))).cuda()
    plan = P.Plan(N, L, 0, B, force_long=force)
    S = Guarded((B, plan.M // 2 + 1, 2))
    plan.spectrum(f, out=S.t)
    S.check("spectrum out")
    spec0 = S.t.clone()
    for transpose, n_in, n_out in ((False, K, L), (True, L, K)):
        x = torch.from_numpy(rng.standard_normal((B, n_in))).cuda()
        x0 = x.clone()
        y = Guarded((B, n_out))
        plan.matvec(S.t, x, transpose=transpose, out=y.t)
        y.check("matvec out")
        xm = torch.from_numpy(rng.standard_normal((B, nv, n_in))).cuda()
        ym = Guarded((B, nv, n_out))
        plan.matvec_multi(S.t, xm, transpose=transpose, out=ym.t)
        ym.check("matvec_multi out")
        assert torch.equal(x, x0)
    assert torch.equal(S.t, spec0), "matvec wrote to the spectrum"


@pytest.mark.parametrize("N,L,nt,B", [(1000, 400, 5, 3), (4096, 2048, 16, 2), (7777, 3000, 3, 2),
                                      (262144, 131072, 3, 2)])
def test_hankelize_stays_in_bounds(P, N, L, nt, B):
    K = N - L + 1
    g = torch.Generator(device="cuda").manual_seed(N)
    U = torch.randn(B, nt, L, dtype=torch.float64, device="cuda", generator=g)
    V = torch.randn(B, nt, K, dtype=torch.float64, device="cuda", generator=g)
    s = torch.rand(B, nt, dtype=torch.float64, device="cuda", generator=g)
    U0, V0, s0 = U.clone(), V.clone(), s.clone()
    plan = P.Plan(N, L, 0, B)
    G = Guarded((B, nt, N))
    plan.hankelize(s, U, V, out=G.t)
    G.check("hankelize out")
    assert torch.equal(U, U0) and torch.equal(V, V0) and torch.equal(s, s0)
    assert torch.isfinite(G.t).all()


def test_cfg1_series_stays_in_bounds(P):
    """The BASELINE cfg1 series through decompose + reconstruct (smoke's workload)."""
    c = ssa_inputs.CONFIGS["cfg1"]
    N, L, k = c["N"], c["L"], c["k"]
    f = torch.from_numpy(ssa_inputs.cfg1_series(N)[None, :].copy()).cuda()
    plan = P.Plan(N, L, k, 1)
    sig, U, V = Guarded((1, k)), Guarded((1, k, L)), Guarded((1, k, N - L + 1))
    plan.decompose(f, sig.t, U.t, V.t)
    G = Guarded((1, k, N))
    plan.reconstruct(sig.t, U.t, V.t, out=G.t)
    for g_, name in ((sig, "sigma"), (U, "U"), (V, "V"), (G, "reconstruct")):
        g_.check(name)
