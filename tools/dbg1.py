import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_0911_4498_b200 as P
try:
    P.Plan(16384, 8192, 0, 2)
except Exception as e: print("ERR", e)
# rank deficient debug
N, L, k = 200, 100, 5
n = np.arange(1, N + 1); f = 1.5*np.sin(2*np.pi*n/10+0.3)
plan = P.Plan(N, L, k, 1)
s,U,V,info = plan.decompose(torch.from_numpy(f[None].copy()).cuda())
print(s.cpu().numpy(), P.info_to_numpy(info))
import oracle
print(oracle.svd(f, L, 6)[0])
