"""Phase profile of the decompose kernels on cfg2 (batch argv[1], default 1024;
reorth mode argv[2], default 1)."""
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import paper_0911_4498_b200 as P, ssa_inputs
B = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
R = int(sys.argv[2]) if len(sys.argv) > 2 else 1
CE = int(sys.argv[3]) if len(sys.argv) > 3 else 4
c = ssa_inputs.CONFIGS["cfg2"]
F = torch.from_numpy(ssa_inputs.cfg2_batch(0, B, c["N"])).cuda()
plan = P.Plan(c["N"], c["L"], c["k"], B, profile=True, reorth=R, check_every=CE)
s, U, V, info = plan.decompose(F); torch.cuda.synchronize()
t0 = time.time(); plan.decompose(F, s, U, V, info); torch.cuda.synchronize(); dt = time.time() - t0
pr = plan.profile(); tot = sum(v for k, v in pr.items() if k in ("fft", "reorth", "check", "svd_fused", "other"))
print("check_every=%d reorth=%d decompose %.1f ms for %d series; phase ms:" % (CE, R, dt * 1e3, B), plan.phase_ms())
for k, v in pr.items():
    print(f"  {k:14s} {v:16d}  {100*v/tot:5.1f}%" if k != "n_checks" else f"  {k:14s} {v:16d}  ({v/B:.1f} per series)")
inf = P.info_to_numpy(info)
print("steps mean", inf["steps"].mean(), "status", np.unique(inf["status"], return_counts=True), "maxres", inf["max_residual"].max(),
      "reorth_extra mean", inf["reorth_extra"].mean(), "max", inf["reorth_extra"].max())
