import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_0911_4498_b200 as P, ssa_inputs
c = ssa_inputs.CONFIGS["cfg2"]; N, L, k = 1024, 512, 8
B = int(sys.argv[1]) if len(sys.argv) > 1 else 2
F = np.stack([ssa_inputs.cfg2_series(i, N) for i in range(B)])
plan = P.Plan(N, L, k, B, max_steps=40)
s, U, V, info = plan.decompose(torch.from_numpy(F).cuda()); torch.cuda.synchronize()
print(s.cpu().numpy()[:, :4], P.info_to_numpy(info)["reorth_extra"])
