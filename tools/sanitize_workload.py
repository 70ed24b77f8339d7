"""Small workloads for compute-sanitizer (memcheck / racecheck / synccheck / initcheck).

  python tools/sanitize_workload.py cfg1|cfg2b8|cfg4b64|long4096|hank|hmatrix|bootstrap

Each one exercises a different set of kernels of libssa.so at a size the sanitizer
finishes in seconds to minutes (it serializes every launch and instruments every
shared/global access).  Exit code 0 iff every call returned SSA_OK and the decompose
status words are OK."""
from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import ssa_inputs  # noqa: E402
import paper_0911_4498_b200 as P  # noqa: E402


def dec(N, L, k, F, **kw):
    plan = P.Plan(N, L, k, F.shape[0], **kw)
    x = torch.from_numpy(np.ascontiguousarray(F)).cuda()
    s, U, V, info = plan.decompose(x)
    G = plan.reconstruct(s, U, V)
    torch.cuda.synchronize()
    inf = P.info_to_numpy(info)
    assert (inf["status"] == 0).all(), inf
    plan.close()
    return G


def main(which: str) -> int:
    torch.cuda.set_device(0)
    if which == "cfg1":
        c = ssa_inputs.CONFIGS["cfg1"]
        dec(c["N"], c["L"], c["k"], ssa_inputs.cfg1_series(c["N"])[None])
    elif which == "cfg2b8":
        c = ssa_inputs.CONFIGS["cfg2"]
        dec(c["N"], c["L"], c["k"], ssa_inputs.cfg2_batch(0, 8, c["N"]))
    elif which == "cfg4b64":
        N, L, B = 8192, 4096, 64
        K = N - L + 1
        g = torch.Generator(device="cuda").manual_seed(4)
        F = torch.randn(B, N, dtype=torch.float64, device="cuda", generator=g)
        v = torch.randn(B, K, dtype=torch.float64, device="cuda", generator=g)
        u = torch.randn(B, L, dtype=torch.float64, device="cuda", generator=g)
        plan = P.Plan(N, L, 0, B)
        spec = plan.spectrum(F)
        plan.matvec(spec, v)
        plan.matvec(spec, u, transpose=True)
        torch.cuda.synchronize()
    elif which == "long4096":
        N, L, k = 4096, 2048, 16
        dec(N, L, k, ssa_inputs.cfg3_like_series(N)[None], force_long=True)
    elif which == "hank":
        # batched hankelization (M <= 16384 smem path) and the four-step path (N = 2^17)
        for N, L, T in ((4096, 2048, 4), (1 << 17, 1 << 16, 2)):
            K = N - L + 1
            g = torch.Generator(device="cuda").manual_seed(5)
            U = torch.randn(2, T, L, dtype=torch.float64, device="cuda", generator=g)
            V = torch.randn(2, T, K, dtype=torch.float64, device="cuda", generator=g)
            s = torch.ones(2, T, dtype=torch.float64, device="cuda")
            plan = P.Plan(N, L, 0, 2)
            plan.hankelize(s, U, V)
            torch.cuda.synchronize()
            plan.close()
    elif which == "hmatrix":
        N = 400
        f = torch.from_numpy(ssa_inputs.change_point_series(N, 200, 7)).cuda()
        G, info = P.hmatrix(f, 100, 100, 50, [1, 2])
        torch.cuda.synchronize()
    elif which == "bootstrap":
        N, L, d, R = 1000, 500, 5, 16
        f = torch.from_numpy(ssa_inputs.bootstrap_series(N)).cuda()
        eps = torch.from_numpy(ssa_inputs.bootstrap_noise(R, N)).cuda()
        plan = P.Plan(N, L, d, R)
        plan.bootstrap(f, eps, 5.0)
        torch.cuda.synchronize()
    else:
        print("unknown workload", which)
        return 2
    print(f"workload {which} ok")
    return 0


if __name__ == "__main__":
    sys.exit(main(sys.argv[1]))
