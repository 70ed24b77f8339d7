"""cfg3 (N = 2^20, L = 2^19, k = 32) decompose + reconstruct timing, PRO and FRO, for quick
iteration on the long-series path (bench.py's decompose_cfg3 line is the reported one)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, '.')
import paper_0911_4498_b200 as P  # noqa: E402
import ssa_inputs  # noqa: E402

f = ssa_inputs.cfg3_series()
x = torch.from_numpy(f[None].copy()).cuda()
for reorth in (3, 1):
    plan = P.Plan(1 << 20, 1 << 19, 32, 1, reorth=reorth)
    s, U, V, info = plan.decompose(x)
    G = plan.reconstruct(s, U, V)
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        t0 = time.perf_counter()
        plan.decompose(x, s, U, V, info)
        t1 = time.perf_counter()
        plan.reconstruct(s, U, V, out=G)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    inf = P.info_to_numpy(info)[0]
    print(f"reorth={reorth} ms={min(ts):.2f} host_enqueue_ms={1e3 * (t1 - t0):.2f} steps={inf['steps']} "
          f"rsteps={inf['reorth_steps']} rows=({inf['rows_u']},{inf['rows_v']}) status={inf['status']} "
          f"conv={inf['converged']} res={inf['max_residual']:.2e} extra={inf['reorth_extra']} "
          f"launches={plan.launches}", flush=True)
    print("  sigma[:4]", s[0, :4].cpu().numpy(), "sigma[31]", float(s[0, 31]))
    plan.close()
