"""Phase profile of the decompose kernel on cfg1 (one N = 1024 series, k = 10)."""
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import paper_0911_4498_b200 as P, ssa_inputs
f = ssa_inputs.cfg1_series(1024)
plan = P.Plan(1024, 512, 10, 1, profile=True)
x = torch.from_numpy(f[None].copy()).cuda()
s, U, V, info = plan.decompose(x); torch.cuda.synchronize()
for _ in range(3):
    t0 = time.time(); plan.decompose(x, s, U, V, info); torch.cuda.synchronize(); dt = time.time() - t0
print("decompose %.3f ms" % (dt * 1e3), plan.phase_ms())
pr = plan.profile(); tot = sum(v for k, v in pr.items() if k in ("fft", "reorth", "check", "svd_fused", "other"))
for k, v in pr.items():
    print(f"  {k:14s} {v:16d}  {100*v/tot:5.1f}%" if k != "n_checks" else f"  {k:14s} {v:16d}")
print("steps", P.info_to_numpy(info)[0]["steps"])
