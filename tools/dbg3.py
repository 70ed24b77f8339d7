import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_0911_4498_b200 as P, ssa_inputs, oracle
c = ssa_inputs.CONFIGS["cfg2"]; N, L, k = c["N"], c["L"], c["k"]
B = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
F = ssa_inputs.cfg2_batch(0, B, N)
plan = P.Plan(N, L, k, B, check_every=int(sys.argv[2]) if len(sys.argv) > 2 else 4)
s, U, V, info = plan.decompose(torch.from_numpy(F).cuda()); torch.cuda.synchronize()
s = s.cpu().numpy(); inf = P.info_to_numpy(info); U = U.cpu().numpy(); V = V.cpu().numpy()
print("reorth_extra hist", np.bincount(np.minimum(inf["reorth_extra"], 10)))
K = N - L + 1
cnt = np.minimum.reduce([np.arange(1, N + 1), np.full(N, L), np.full(N, K), N - np.arange(N)])
fro2 = (F * F * cnt).sum(axis=1)
bad = np.where((s * s).sum(axis=1) > fro2 * (1 + 1e-12))[0]
print("bad", len(bad), bad[:10], "extra of bad", inf["reorth_extra"][bad[:10]], "steps", inf["steps"][bad[:10]])
for b in list(bad[:2]) + [0]:
    res = [np.linalg.norm(oracle.matvec(F[b], L, V[b, i]) - s[b, i] * U[b, i]) / s[b, 0] for i in range(k)]
    res2 = [np.linalg.norm(oracle.matvec(F[b], L, U[b, i], True) - s[b, i] * V[b, i]) / s[b, 0] for i in range(k)]
    print(b, "true res max", max(res), max(res2))
