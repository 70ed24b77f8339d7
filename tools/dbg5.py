"""Determinism of the FFT kernels under full occupancy."""
import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_0911_4498_b200 as P
N, L, B = 4096, 2048, 8192
K = N - L + 1
g = torch.Generator(device="cuda").manual_seed(0)
F = torch.randn(B, N, dtype=torch.float64, device="cuda", generator=g)
x = torch.randn(B, L, dtype=torch.float64, device="cuda", generator=g)
plan = P.Plan(N, L, 0, B)
spec0 = plan.spectrum(F).clone()
y0 = plan.matvec(spec0, x, transpose=True).clone()
bad_s = bad_y = 0
for r in range(10):
    s = plan.spectrum(F)
    y = plan.matvec(spec0, x, transpose=True)
    torch.cuda.synchronize()
    bad_s += int((s != spec0).any(dim=(1, 2)).sum()); bad_y += int((y != y0).any(dim=1).sum())
print("spectrum nondeterministic rows:", bad_s, "matvec:", bad_y)
