"""Write oracle-only expected values for full-size parity cases (test infrastructure).

Calls nothing but ``oracle`` (one-sided Jacobi SVD + direct averaging on CPU) and the
seeded generators of ``ssa_inputs``; never the CUDA path.  Output:
tests/golden/oracle_cfg2_<i>.npz with sigma (k+1 values, so the straddling rule can be
applied), U/V (k rows), G (k elementary reconstructions) and the Jacobi sweep count.

usage: python -m oracle.make_golden [series indices...]   (default 0 1234 4095)
"""
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import ssa_inputs  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def one(i: int):
    c = ssa_inputs.CONFIGS["cfg2"]
    f = ssa_inputs.cfg2_series(i, c["N"])
    t0 = time.time()
    s, U, V, sweeps = oracle.svd(f, c["L"], c["k"] + 1)
    k = c["k"]
    G = np.stack([oracle.hankelize_rank1(s[j], U[j], V[j]) for j in range(k)])
    path = os.path.join(OUT, f"oracle_cfg2_{i}.npz")
    np.savez_compressed(path, sigma=s, U=U[:k], V=V[:k], G=G, sweeps=sweeps, series_index=i,
                        norm_f=np.linalg.norm(f))
    return i, sweeps, time.time() - t0


if __name__ == "__main__":
    idx = [int(a) for a in sys.argv[1:]] or [0, 1234, 4095]
    with ThreadPoolExecutor(len(idx)) as ex:
        for i, sw, dt in ex.map(one, idx):
            print(f"series {i}: {sw} sweeps, {dt:.1f} s", flush=True)
