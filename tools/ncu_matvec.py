import sys, torch
sys.path.insert(0, '.')
import paper_0911_4498_b200 as P
N, L, B = 8192, 4096, int(sys.argv[1]) if len(sys.argv) > 1 else 4096
K = N - L + 1
g = torch.Generator(device="cuda").manual_seed(4)
F = torch.randn(B, N, dtype=torch.float64, device="cuda", generator=g)
v = torch.randn(B, K, dtype=torch.float64, device="cuda", generator=g)
plan = P.Plan(N, L, 0, B)
spec = plan.spectrum(F)
y = plan.matvec(spec, v)
torch.cuda.synchronize()
print("ok")
