"""Race hunt: same batch with 148 vs 296 Lanczos CTAs; first step where alpha/beta differ."""
import os, sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_0911_4498_b200 as P, ssa_inputs
N, L, k, B = 4096, 2048, 16, 2048
F = torch.from_numpy(ssa_inputs.cfg2_batch(0, B, N)).cuda()
out = {}
for slots in ("148", "148b", "296", "296b"):
    os.environ["SSA_LANCZOS_SLOTS"] = slots[:3]
    plan = P.Plan(N, L, k, B)
    s, U, V, info = plan.decompose(F); torch.cuda.synchronize()
    out[slots] = plan.bidiagonals() + (P.info_to_numpy(info),)
    plan.close()
a1, b1, s1, i1 = out["148"]; a2, b2, s2, i2 = out["296"]
a3, b3, s3, i3 = out["296b"]
a4, b4, s4, i4 = out["148b"]
print("repeat 148 vs 148b differing:", sum(1 for b in range(B) if s1[b] != s4[b] or np.any(a1[b, 1:s1[b]+2] != a4[b, 1:s1[b]+2])))
print("repeat 296 vs 296b differing:", sum(1 for b in range(B) if s2[b] != s3[b] or np.any(a2[b, 1:s2[b]+2] != a3[b, 1:s2[b]+2])))
diff = [b for b in range(B) if s1[b] != s2[b] or np.any(a1[b, 1:s1[b]+2] != a2[b, 1:s1[b]+2]) or np.any(b1[b, 1:s1[b]+2] != b2[b, 1:s1[b]+2])]
diff = np.array(diff, dtype=int)
print("differing series:", len(diff), diff[:20])
for b in diff[:8]:
    m = min(s1[b], s2[b])
    da = np.where(a1[b, 1:m+1] != a2[b, 1:m+1])[0]
    db = np.where(b1[b, 2:m+2] != b2[b, 2:m+2])[0]
    ja = da[0] + 1 if len(da) else -1; jb = db[0] + 2 if len(db) else -1
    print(f"series {b}: steps {s1[b]} vs {s2[b]}; first alpha diff j={ja}, first beta diff j={jb};",
          f"extra {i1['reorth_extra'][b]} vs {i2['reorth_extra'][b]}",
          "rel diff at ja:", (abs(a1[b, ja] - a2[b, ja]) / a1[b, ja]) if ja > 0 else None)
