import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_0911_4498_b200 as P, ssa_inputs, oracle
c = ssa_inputs.CONFIGS["cfg2"]; N, L, k = c["N"], c["L"], c["k"]
B = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
F = ssa_inputs.cfg2_batch(0, B, N)
Ft = torch.from_numpy(F).cuda()
res = {}
for meth in ("tgk", "qr"):
    plan = P.Plan(N, L, k, B, svd=meth)
    s, U, V, info = plan.decompose(Ft); torch.cuda.synchronize()
    s, U, V, info = plan.decompose(Ft, s, U, V, info); torch.cuda.synchronize()
    res[meth] = (s.cpu().numpy(), U.cpu().numpy(), V.cpu().numpy(), P.info_to_numpy(info), plan.phase_ms())
    plan.close()
for meth in res:
    s, U, V, inf, ph = res[meth]
    print(meth, "phase", {kk: round(v, 2) for kk, v in ph.items()}, "status", np.unique(inf["status"], return_counts=True), "maxres", inf["max_residual"].max())
s1, U1, V1, _, _ = res["tgk"]; s2, U2, V2, _, _ = res["qr"]
print("sigma max rel diff tgk vs qr:", np.max(np.abs(s1 - s2) / s2))
orth = max(np.abs(U1[b] @ U1[b].T - np.eye(k)).max() for b in range(0, B, max(1, B // 64)))
print("tgk U orthonormality:", orth)
for b in (0, 1):
    rr = max(np.linalg.norm(oracle.matvec(F[b], L, V1[b, i]) - s1[b, i] * U1[b, i]) for i in range(k)) / s1[b, 0]
    print("series", b, "tgk true residual", rr)
