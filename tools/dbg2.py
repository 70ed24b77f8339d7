import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_0911_4498_b200 as P, ssa_inputs
c = ssa_inputs.CONFIGS["cfg2"]; N, L, k, B = c["N"], c["L"], c["k"], 4096
F = ssa_inputs.cfg2_batch(0, B, N)
plan = P.Plan(N, L, k, B)
s, U, V, info = plan.decompose(torch.from_numpy(F).cuda()); torch.cuda.synchronize()
s = s.cpu().numpy(); inf = P.info_to_numpy(info)
K = N - L + 1
cnt = np.minimum.reduce([np.arange(1, N + 1), np.full(N, L), np.full(N, K), N - np.arange(N)])
fro2 = (F * F * cnt).sum(axis=1)
bad = np.where((s * s).sum(axis=1) > fro2 * (1 + 1e-12))[0]
print("bad", bad[:20], len(bad))
for b in bad[:3]:
    print(b, s[b], fro2[b], (s[b]**2).sum(), inf[b])
np.save("gpurun_out/bad_idx.npy", bad)
# check orthonormality of U for a few series
Uc = U.cpu().numpy()
for b in list(bad[:3]) + [0, 1]:
    G = Uc[b] @ Uc[b].T
    print("orthU", b, np.abs(G - np.eye(k)).max())
