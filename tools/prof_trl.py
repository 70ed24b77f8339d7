"""Phase profile of the thick-restart kernel on cfg2 (batch argv[1], default 1024; d, p argv[2:4])."""
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import paper_0911_4498_b200 as P, ssa_inputs
B = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
d = int(sys.argv[2]) if len(sys.argv) > 2 else 40
p = int(sys.argv[3]) if len(sys.argv) > 3 else 20
c = ssa_inputs.CONFIGS["cfg2"]
F = torch.from_numpy(ssa_inputs.cfg2_batch(0, B, c["N"])).cuda()
plan = P.Plan(c["N"], c["L"], c["k"], B, profile=True, reorth=1, restart_dim=d, restart_keep=p)
s, U, V, info = plan.decompose(F); torch.cuda.synchronize()
t0 = time.time(); plan.decompose(F, s, U, V, info); torch.cuda.synchronize(); dt = time.time() - t0
pr = plan.profile()
names = {"fft": "fft", "reorth": "cgs", "check": "jacobi", "n_checks": "n_checks", "svd_fused": "restart", "other": "other"}
tot = sum(v for kk, v in pr.items() if kk in ("fft", "reorth", "check", "svd_fused", "other"))
print("TRL d=%d p=%d decompose %.1f ms for %d series" % (d, p, dt * 1e3, B))
for kk, v in pr.items():
    if kk in names:
        print(f"  {names[kk]:10s} {v:16d}  " + (f"{100*v/tot:5.1f}%" if kk != "n_checks" else f"({v/B:.1f} per series)"))
inf = P.info_to_numpy(info)
print("steps mean", inf["steps"].mean(), "thick restarts mean", inf["reserved"].mean(), "status",
      np.unique(inf["status"], return_counts=True))
