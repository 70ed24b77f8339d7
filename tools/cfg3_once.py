"""One cfg3 decompose (N = 2^20, L = 2^19, k = 32) for ncu launch lists."""
import sys, torch
sys.path.insert(0, '.')
import paper_0911_4498_b200 as P, ssa_inputs
f = ssa_inputs.cfg3_series()
plan = P.Plan(1 << 20, 1 << 19, 32, 1, reorth=int(sys.argv[1]) if len(sys.argv) > 1 else 1)
x = torch.from_numpy(f[None].copy()).cuda()
s, U, V, info = plan.decompose(x)
torch.cuda.synchronize()
print("ok", P.info_to_numpy(info)[0])
