"""One decompose + reconstruct of cfg2-shaped series for ncu captures
(batch argv[1], default 1024; reorth mode argv[2], default 1)."""
import sys, torch
sys.path.insert(0, '.')
import paper_0911_4498_b200 as P, ssa_inputs
B = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
R = int(sys.argv[2]) if len(sys.argv) > 2 else 1
c = ssa_inputs.CONFIGS["cfg2"]
F = torch.from_numpy(ssa_inputs.cfg2_batch(0, B, c["N"])).cuda()
plan = P.Plan(c["N"], c["L"], c["k"], B, reorth=R)
s, U, V, info = plan.decompose(F)
G = plan.reconstruct(s, U, V)
torch.cuda.synchronize()
print("ok", P.info_to_numpy(info)["steps"].mean())
