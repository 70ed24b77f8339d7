"""One small cfg4 matvec batch and one cfg5 hankelization batch, for ncu captures."""
import sys, torch
sys.path.insert(0, '.')
import paper_0911_4498_b200 as P
which = sys.argv[1:] or ["cfg4", "cfg5"]
if "cfg4" in which:
    N, L, B = 8192, 4096, 4096
    K = N - L + 1
    g = torch.Generator(device="cuda").manual_seed(4)
    F = torch.randn(B, N, dtype=torch.float64, device="cuda", generator=g)
    v = torch.randn(B, K, dtype=torch.float64, device="cuda", generator=g)
    plan = P.Plan(N, L, 0, B)
    spec = plan.spectrum(F)
    y = plan.matvec(spec, v)
    torch.cuda.synchronize()
    print("cfg4 ok")
if "cfg4m" in which:   # ssa_matvec_multi: 2048 series x 32 vectors (one bench chunk)
    N, L, B, nv = 8192, 4096, 2048, 32
    K = N - L + 1
    g = torch.Generator(device="cuda").manual_seed(4)
    F = torch.randn(B, N, dtype=torch.float64, device="cuda", generator=g)
    v = torch.randn(B, nv, K, dtype=torch.float64, device="cuda", generator=g)
    plan = P.Plan(N, L, 0, B)
    spec = plan.spectrum(F)
    y = plan.matvec_multi(spec, v)
    y = plan.matvec_multi(spec, v, out=y)
    torch.cuda.synchronize()
    print("cfg4m ok")
if "cfg3mv" in which:  # one long-series product (N = 2^20): the four-step kernels of the Lanczos loop
    N, L = 1 << 20, 1 << 19
    g = torch.Generator(device="cuda").manual_seed(3)
    F = torch.randn(1, N, dtype=torch.float64, device="cuda", generator=g)
    v = torch.randn(1, N - L + 1, dtype=torch.float64, device="cuda", generator=g)
    plan = P.Plan(N, L, 0, 1)
    spec = plan.spectrum(F)
    for _ in range(3):
        y = plan.matvec(spec, v)
    torch.cuda.synchronize()
    print("cfg3mv ok")
if "cfg5" in which:
    N, L, Bc, T = 262144, 131072, 2, 50
    K = N - L + 1
    g = torch.Generator(device="cuda").manual_seed(5)
    U = torch.randn(Bc, T, L, dtype=torch.float64, device="cuda", generator=g); U /= U.norm(dim=2, keepdim=True)
    V = torch.randn(Bc, T, K, dtype=torch.float64, device="cuda", generator=g); V /= V.norm(dim=2, keepdim=True)
    sig = (1.0 / torch.arange(1, T + 1, dtype=torch.float64, device="cuda")).repeat(Bc, 1).contiguous()
    plan = P.Plan(N, L, 0, Bc)
    out = plan.hankelize(sig, U, V)
    torch.cuda.synchronize()
    print("cfg5 ok")
