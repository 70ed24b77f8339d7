#!/usr/bin/env python
"""bench.py -- throughput of the fast Basic-SSA hot path on B200 (driver contract).

Default workload = BASELINE.json configs[1] ("cfg2"): a batch of 4096 independent fp64
series, N=4096, L=2048, k=16.  One step = the whole hot path over the batch (SURVEY.md
§8(a) rows a1-a10): spectra, GKL bidiagonalization with partial reorthogonalization (FFT
Hankel products; PRO, R22), convergence tests and the
bidiagonal SVD on device, Ritz assembly, and rank-1 Hankelization of all 16 triples of
every series (ssa_decompose + ssa_reconstruct through the C-ABI).  A secondary line runs
the same batch with full reorthogonalization (FRO, the round-1 default).

Metric: eigentriples/s (fp64) for the whole job; Hankel matvecs/s and roofline of the
dominant kernel (lanczos_kernel, HBM-bound) are reported beside it.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--batch B]

Multi-GPU (torchrun, one rank per GPU): the 4096 series are sharded by series over the
ranks (parallel.shard_range: 512 per GPU at 8), no data-path collective, strong scaling;
a weak-scaling line (4096 series per GPU) is reported beside it.  Timing is per step with
CUDA events, MAX over ranks; value = all triples / that time.  The cfg4 / cfg5 lines shard
their series / problems the same way; cfg1 / cfg3 (one series) run as replicas.

--impl reference times the CPU oracle (oracle/: one-sided Jacobi SVD + direct averaging)
as it stands on the host cores on a bounded sample of the same workload (rank 0 only).
"""
from __future__ import annotations

import argparse
import glob
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import ssa_inputs  # noqa: E402

METRIC = "SSA eigentriples/s and Hankel matvecs/s (fp64), % HBM/fp64 roofline, 1–8 B200"
UNIT = "eigentriples/s"
CFG = ssa_inputs.CONFIGS["cfg2"]


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=CFG["batch"], help="global batch, sharded over the GPUs (4096)")
    ap.add_argument("--no-fro", action="store_true", help="skip the FRO comparison line")
    ap.add_argument("--no-trl", action="store_true", help="skip the thick-restart line")
    ap.add_argument("--no-overshoot", action="store_true", help="skip the test-schedule overshoot probe")
    ap.add_argument("--no-weak", action="store_true", help="skip the weak-scaling line (N > 1)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-once", action="store_true", help="1 decompose, no timing (for ncu)")
    ap.add_argument("--no-micro", action="store_true", help="skip the cfg4 / cfg5 microbenchmarks")
    return ap.parse_args()


# ------------------------------------------------------------------------ model bytes
def _H(N: int) -> int:
    M = 1
    while M < N:
        M <<= 1
    return M // 2


def lanczos_alg_bytes(steps, rows_u, rows_v, N: int, L: int) -> float:
    """Algorithmic HBM bytes of lanczos_kernel for series that ran m = steps
    Lanczos steps and whose reorthogonalizations read rows_u / rows_v basis rows in total
    (ssa_series_info: every CGS pass reads its rows once for the dots and once for the
    update; FRO without DGKS passes gives rows_u = rows_v = m(m+1), PRO far fewer):
      every half-step reads the spectrum (16 (H+1)) and writes one basis vector;
      half-steps A, j = 1..m+1 (v side): 8 K each; half-steps B, j = 1..m (u side): 8 L each;
      reorthogonalization: 8 (rows_u L + rows_v K);  start: read the series, write u_1.
    The Ritz assembly is a separate kernel (ritz_alg_bytes)."""
    K = N - L + 1
    H = _H(N)
    m = np.asarray(steps, dtype=np.float64)
    ru = np.asarray(rows_u, dtype=np.float64)
    rv = np.asarray(rows_v, dtype=np.float64)
    half = (m + 1) * (16 * (H + 1) + 8 * K) + m * (16 * (H + 1) + 8 * L)
    return float(np.sum(half + 8 * (ru * L + rv * K) + 8 * N + 8 * L))


def fro_rows(steps):
    """Basis rows one-pass FRO reads: sum_{j=1}^{m+1} 2 (j-1) = sum_{j=1}^{m} 2 j = m (m+1) per side."""
    m = np.asarray(steps, dtype=np.float64)
    return m * (m + 1)


def ritz_alg_bytes(steps, N: int, L: int, k: int) -> float:
    """ritz_kernel: read U_{m+1} and V_m once, write U_k, V_k (Eq. 1)."""
    K = N - L + 1
    m = np.asarray(steps, dtype=np.float64)
    return float(np.sum(8 * ((m + 1) * L + m * K) + 8 * k * (L + K)))


def hankelize_alg_bytes(nterms: int, N: int, L: int) -> float:
    K = N - L + 1
    return float(nterms) * 8 * (L + K + N + 1)


def hankelize_flops(nterms: int, N: int) -> float:
    """Three real FFTs of length M + the spectrum product + sigma / c_t scaling."""
    M = 2 * _H(N)
    return float(nterms) * (3 * fft_flops(M) + 6 * (M // 2 + 1) + 2 * N)


# ------------------------------------------------------------------------ microbenchmarks
def fp64_peak():
    """Measured fp64 peak (TFLOP/s of DFMA, 2 flops each): the sustained figure (4 s of
    back-to-back DFMA launches, tools/peaks.cu, profiles/peaks_r02.json: 34.13 TF at
    1965 MHz, no power cap -- a DFMA loop draws ~590 W) is used for kernels timed inside a
    long step; the guide's nominal 37 TF if no measured file is present."""
    for name, key in (("peaks_r02.json", "dfma_tflops_sustained"), ("peaks_r01.json", "dfma_tflops")):
        try:
            with open(os.path.join(ROOT, "profiles", name)) as fh:
                return float(json.load(fh)[key]), f"profiles/{name} {key} (tools/peaks.cu, measured)"
        except Exception:
            pass
    return 37.0, "nominal fp64 (no measured file)"


def fft_flops(n: int) -> float:
    """Real FFT of length n: 2.5 n log2 n (benchFFT convention)."""
    import math
    return 2.5 * n * math.log2(n)


def _events_ms(fn, reps=1):
    import torch
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b)


class Ctx:
    """Rank / world and the MAX-over-ranks reduction of device times (multi-GPU timing rule)."""

    def __init__(self, rank: int, world: int):
        self.rank, self.world = rank, world

    def max_ms(self, ms: float) -> float:
        if self.world == 1:
            return ms
        import torch
        import torch.distributed as dist
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def barrier(self):
        if self.world > 1:
            import torch.distributed as dist
            dist.barrier()

    def shard(self, n: int):
        from paper_0911_4498_b200.parallel import shard_range
        return shard_range(n, self.rank, self.world)


def _timed(ctx, fn, reps):
    """best-of-reps device time of fn() (CUDA events, barrier before each), MAX over ranks."""
    best = float("inf")
    for _ in range(reps):
        ctx.barrier()
        best = min(best, _events_ms(fn))
    return ctx.max_ms(best)


def micro_matvec(P, peak, ctx):
    """BASELINE.json configs[3] (cfg4): 65,536 series N=8192, L=4096, i.i.d. N(0,1) series and
    vectors (drawn on the device, per-rank generator seeds); 64 products per series, 32 X v
    and 32 X^T u, over this rank's contiguous shard of the series.  The
    series run in chunks of 2048; per chunk two ssa_matvec_multi calls (32 vectors per
    series against its one spectrum: X v, then X^T u), the vectors read from HBM and the
    products written to HBM (the same drawn chunk of vectors stands in for every chunk:
    2 GB per operand, far above L2).  Algorithmic bytes per product 8(K+L) + 16(M/2+1)/32
    (the spectrum read once per call); flops 2 x 2.5 M log2 M + 6(M/2+1).  The bound is
    the larger of the two: fp64 (16 ns vs 10 ns of HBM per product).  The one-product-per-
    series launch (ssa_matvec, spectrum read per product) is timed beside it."""
    import torch
    c = ssa_inputs.CONFIGS["cfg4"]
    N, L, GB, T = c["N"], c["L"], c["batch"], c["products"]
    b0, b1 = ctx.shard(GB)
    B = b1 - b0
    K = N - L + 1
    nv = T // 2
    Bc = min(2048, B)
    g = torch.Generator(device="cuda").manual_seed(4 + 1000 * ctx.rank)
    spec = torch.empty(B, N // 2 + 1, 2, dtype=torch.float64, device="cuda")  # M = N (power of two)
    for c0 in range(0, B, 4096):      # spectra of every series of the shard (drawn in chunks)
        cb = min(4096, B - c0)
        pc = P.Plan(N, L, 0, cb)
        F = torch.randn(cb, N, dtype=torch.float64, device="cuda", generator=g)
        pc.spectrum(F, out=spec[c0:c0 + cb])
        pc.close()
        del F
    V = torch.randn(Bc, nv, K, dtype=torch.float64, device="cuda", generator=g)
    U = torch.randn(Bc, nv, L, dtype=torch.float64, device="cuda", generator=g)
    Y = torch.empty(Bc, nv, L, dtype=torch.float64, device="cuda")
    Z = torch.empty(Bc, nv, K, dtype=torch.float64, device="cuda")
    plan = P.Plan(N, L, 0, Bc)
    tail = B % Bc
    plan_t = P.Plan(N, L, 0, tail) if tail else None

    def run():
        for c0 in range(0, B, Bc):
            cb = min(Bc, B - c0)
            pl = plan if cb == Bc else plan_t
            sp = spec[c0:c0 + cb]
            pl.matvec_multi(sp, V[:cb], out=Y[:cb])
            pl.matvec_multi(sp, U[:cb], transpose=True, out=Z[:cb])
    run()
    ms = _timed(ctx, run, 3)
    nprod = T * GB
    M = plan.M
    byt = nprod * (8 * (K + L) + 16 * (M // 2 + 1) / nv)
    fl = nprod * (2 * fft_flops(M) + 6 * (M // 2 + 1))
    fpk, fsrc = fp64_peak()
    w = ctx.world
    # one product per series per launch (ssa_matvec): the spectrum is read for every product
    v1, u1 = V[:, 0].contiguous(), U[:, 0].contiguous()
    y1, z1 = Y[:, 0].contiguous(), Z[:, 0].contiguous()
    sp1 = spec[:Bc]

    def run1():
        for t in range(8):
            if t % 2 == 0:
                plan.matvec(sp1, v1, out=y1)
            else:
                plan.matvec(sp1, u1, transpose=True, out=z1)
    run1()
    ms1 = _timed(ctx, run1, 3)
    n1 = 8 * Bc
    out = {"value": nprod / (ms * 1e-3), "unit": "Hankel matvecs/s", "ms": ms, "products": nprod,
           "series_per_gpu": B, "scaling": "strong", "api": "ssa_matvec_multi (32 vectors per series and call)",
           "workload": "cfg4 (BASELINE.json configs[3]): 65536 series N=8192 L=4096, 32 X v + 32 X^T u products "
                       f"per series, series sharded over {w} GPU(s)",
           "roofline": {"bound": "fp64 (model flops: 2 x 2.5 M log2 M + 6(M/2+1) per product)",
                        "achieved": fl / (ms * 1e-3) / 1e12 / w, "peak": fpk, "unit": "TFLOP/s per GPU",
                        "frac": fl / (ms * 1e-3) / 1e12 / w / fpk, "peak_src": fsrc},
           "hbm_roofline": {"achieved": byt / (ms * 1e-3) / 1e9 / w, "peak": peak, "unit": "GB/s per GPU",
                            "frac": byt / (ms * 1e-3) / 1e9 / w / peak, "alg_bytes_per_product": byt / nprod},
           "single_vector": {"value": n1 / (ms1 * 1e-3), "unit": "Hankel matvecs/s", "api": "ssa_matvec",
                             "alg_bytes_per_product": 8 * (K + L) + 16 * (M // 2 + 1),
                             "hbm_frac": n1 * (8 * (K + L) + 16 * (M // 2 + 1)) / (ms1 * 1e-3) / 1e9 / peak}}
    for pl in (plan, plan_t):
        if pl is not None:
            pl.close()
    del spec, V, U, Y, Z
    torch.cuda.empty_cache()
    return out


def micro_hankelize(P, peak, ctx):
    """BASELINE.json configs[4] (cfg5): 256 problems N=262144, L=131072, 50 rank-1 terms each,
    sigma_i = 1/i, u_i, v_i Gaussian normalized (drawn on the device); every term
    Hankelized separately.  This rank's contiguous shard of the problems runs in launches of
    up to 32 problems (the same 32 drawn problems stand in for every chunk).  Algorithmic
    bytes per term 8(L+K+N); flops per term 3 x 2.5 N log2 N + 6(N/2+1) + 2N."""
    import torch
    c = ssa_inputs.CONFIGS["cfg5"]
    N, L, GB, T = c["N"], c["L"], c["batch"], c["k"]
    b0, b1 = ctx.shard(GB)
    B = b1 - b0
    K = N - L + 1
    Bc = min(32, B)
    g = torch.Generator(device="cuda").manual_seed(5 + 1000 * ctx.rank)
    U = torch.randn(Bc, T, L, dtype=torch.float64, device="cuda", generator=g)
    U /= U.norm(dim=2, keepdim=True)
    V = torch.randn(Bc, T, K, dtype=torch.float64, device="cuda", generator=g)
    V /= V.norm(dim=2, keepdim=True)
    sig = (1.0 / torch.arange(1, T + 1, dtype=torch.float64, device="cuda")).repeat(Bc, 1).contiguous()
    plan = P.Plan(N, L, 0, Bc)
    out = torch.empty(Bc, T, N, dtype=torch.float64, device="cuda")
    chunks = [(q, min(Bc, B - q)) for q in range(0, B, Bc)]
    tail = [q for q in chunks if q[1] != Bc]
    plan_t = P.Plan(N, L, 0, tail[0][1]) if tail else None

    def run():
        for _, n in chunks:
            if n == Bc:
                plan.hankelize(sig, U, V, out=out)
            else:
                plan_t.hankelize(sig[:n], U[:n], V[:n], out=out[:n])
    run()
    ms = _timed(ctx, run, 2)
    nt = GB * T
    byt = hankelize_alg_bytes(nt, N, L)
    flops = hankelize_flops(nt, N)
    fpk, fsrc = fp64_peak()
    w = ctx.world
    res = {"value": nt / (ms * 1e-3), "unit": "terms/s", "ms": ms, "terms": nt, "problems_per_gpu": B,
           "scaling": "strong",
           "workload": f"cfg5 (BASELINE.json configs[4]): 256 x 50 terms, N=262144 L=131072, problems sharded over {w} GPU(s)",
           "roofline": {"bound": "fp64 (model flops 3 x 2.5 N log2 N + 6(N/2+1) + 2N per term; "
                                 "SURVEY.md §8(d): 1.07 us/term fp64 vs 0.64 us HBM)",
                        "achieved": flops / (ms * 1e-3) / 1e12 / w, "peak": fpk, "unit": "TFLOP/s per GPU",
                        "frac": flops / (ms * 1e-3) / 1e12 / w / fpk, "peak_src": fsrc},
           "hbm_roofline": {"achieved": byt / (ms * 1e-3) / 1e9 / w, "peak": peak, "unit": "GB/s per GPU",
                            "frac": byt / (ms * 1e-3) / 1e9 / w / peak, "alg_bytes_per_term": byt / nt}}
    plan.close()
    if plan_t:
        plan_t.close()
    del U, V, out, sig
    torch.cuda.empty_cache()
    return res


def micro_hmatrix(P, ctx, N: int = 4000):
    """Heterogeneity matrix (ssa_hmatrix) in the paper's comparison
    setting: Eq. (hseries) series with Q = N/2, B = T = N/4, L = B/2,
    I = {1, 2}; N = 4000 here (3001 base-window decompositions, 6002 Hankel products of the
    whole series, a 3001 x 3001 matrix).  ssa_hmatrix_exec timed (plan and workspace
    created once, outside; the exec ends with the per-window status read-back).  One
    series: replicas only."""
    import torch
    Q, B = N // 2, N // 4
    T, L = B, B // 2
    f = torch.from_numpy(ssa_inputs.change_point_series(N, Q, 7)).cuda()
    hm = P.HMatrix(N, B, T, L, [1, 2])
    G, info = hm(f)
    torch.cuda.synchronize()
    ms = _timed(ctx, lambda: hm(f, out=G, info=info), 3)
    nb, nt = N - B + 1, N - T + 1
    inf = P.info_to_numpy(info)
    res = {"value": nb * nt / (ms * 1e-3), "unit": "H-matrix entries/s", "ms": ms, "replicas": ctx.world,
           "windows_decomposed_per_s": nb / (ms * 1e-3), "mean_steps": float(inf["steps"].mean()),
           "workload": f"H-matrix of Eq. (hseries), N={N} Q={Q} B=T={B} L={L} I={{1,2}} ({nb}x{nt})",
           "g_inside_mean": float(G[: Q - B + 1, : Q - T + 1].mean().item()),
           "g_across_mean": float(G[: Q - B + 1, Q:].mean().item())}
    hm.close()
    del f, G
    torch.cuda.empty_cache()
    return res


def micro_bootstrap(P, ctx, R: int = 1024):
    """Bootstrap study of the paper (sec 6.3): the
    rank-5 series (periods in n, R17), N = 1000, L = 500, noise sigma = 5, R
    replicates (seeded N(0,1) noise, drawn on the host and copied once): replicates,
    batched decompose (k = 5), grouped reconstruction, per-point mean/var/MSE.  Replicas."""
    import torch
    N, L, d, noise = 1000, 500, 5, 5.0
    f = torch.from_numpy(ssa_inputs.bootstrap_series(N)).cuda()
    eps = torch.from_numpy(ssa_inputs.bootstrap_noise(R, N)).cuda()
    plan = P.Plan(N, L, d, R)
    info = torch.zeros((R, P.INFO_DTYPE.itemsize), dtype=torch.uint8, device="cuda")
    plan.bootstrap(f, eps, noise, info=info)
    torch.cuda.synchronize()
    ms = _timed(ctx, lambda: plan.bootstrap(f, eps, noise, info=info), 3)
    inf = P.info_to_numpy(info)
    res = {"value": R / (ms * 1e-3), "unit": "replicates/s", "ms": ms, "replicates": R, "replicas": ctx.world,
           "eigentriples_per_s": R * d / (ms * 1e-3), "mean_steps": float(inf["steps"].mean()),
           "converged_fraction": float((inf["converged"] == 1).mean()),
           "workload": f"bootstrap of the rank-5 series, N={N} L={L} sigma={noise}, {R} replicates"}
    plan.close()
    del f, eps
    torch.cuda.empty_cache()
    return res


def micro_decompose_cfg1(P, ctx):
    """BASELINE.json configs[0] (cfg1): one fp64 series N=1024, L=512, k=10 (ssa_inputs
    cfg1_series, seed 0), decompose + reconstruct of all 10 components on one GPU.  A
    latency regime (~60 dependent Lanczos steps in one CTA): time, us per Lanczos step and
    triples/s are reported, no roofline.  Replicas only (§8(e))."""
    import torch
    c = ssa_inputs.CONFIGS["cfg1"]
    N, L, k = c["N"], c["L"], c["k"]
    x = torch.from_numpy(ssa_inputs.cfg1_series(N)[None].copy()).cuda()
    plan = P.Plan(N, L, k, 1)
    s_, U, V, info = plan.decompose(x)
    G = plan.reconstruct(s_, U, V)
    torch.cuda.synchronize()

    def run():
        plan.decompose(x, s_, U, V, info)
        plan.reconstruct(s_, U, V, out=G)
    ms = _timed(ctx, run, 5)
    inf = P.info_to_numpy(info)[0]
    m = int(inf["steps"])
    res = {"value": k / (ms * 1e-3), "unit": "eigentriples/s", "ms": ms, "steps": m, "us_per_step": 1e3 * ms / m,
           "reorth_steps": int(inf["reorth_steps"]), "replicas": ctx.world,
           "hankel_matvecs_per_s": 2 * m / (ms * 1e-3), "status": int(inf["status"]),
           "workload": "cfg1 (BASELINE.json configs[0]): one series N=1024 L=512 k=10, decompose + reconstruct",
           "regime": "latency (one CTA, dependent steps): no roofline"}
    plan.close()
    return res


def micro_decompose_cfg3(P, peak, ctx):
    """BASELINE.json configs[2] (cfg3): one long series N=2^20, L=2^19, k=32 (ssa_inputs
    cfg3_series, seed 3) on one GPU, "Lanczos with full reorthogonalization" as the config
    states (reorth = 1: CGS + DGKS against the whole basis every half-step): full decompose
    (four-step FFT products through L2, reorthogonalization, bidiagonal SVD, DMMA Ritz
    vectors) + reconstruct of the 32 triples.  The default PRO mode is timed beside it.
    Roofline: HBM, algorithmic bytes of the half-steps (lanczos_alg_bytes with the basis
    rows the run read) + Ritz + Hankelization.  Replicas only (§8(e))."""
    import torch
    c = ssa_inputs.CONFIGS["cfg3"]
    N, L, k = c["N"], c["L"], c["k"]
    x = torch.from_numpy(ssa_inputs.cfg3_series()[None].copy()).cuda()

    def one(reorth):
        plan = P.Plan(N, L, k, 1, reorth=reorth)
        s_, U, V, info = plan.decompose(x)
        G = plan.reconstruct(s_, U, V)
        torch.cuda.synchronize()

        def run():
            plan.decompose(x, s_, U, V, info)
            plan.reconstruct(s_, U, V, out=G)
        ms = _timed(ctx, run, 3)
        inf = P.info_to_numpy(info)[0]
        m = int(inf["steps"])
        ru, rv = int(inf["rows_u"]), int(inf["rows_v"])
        if ru == 0 and rv == 0:        # path without row accounting: one-pass FRO
            ru = rv = int(fro_rows(m))
        byt = (lanczos_alg_bytes([m], [ru], [rv], N, L) + ritz_alg_bytes([m], N, L, k) +
               hankelize_alg_bytes(k, N, L))
        plan.close()
        return ms, inf, m, ru, rv, byt

    ms, inf, m, ru, rv, byt = one(1)
    res = {"value": k / (ms * 1e-3), "unit": "eigentriples/s", "ms": ms, "steps": m, "replicas": ctx.world,
           "reorth": "FRO (CGS + DGKS every half-step, as BASELINE configs[2] states)",
           "hankel_matvecs_per_s": 2 * m / (ms * 1e-3), "status": int(inf["status"]),
           "converged": int(inf["converged"]), "max_residual": float(inf["max_residual"]),
           "reorth_steps": int(inf["reorth_steps"]), "basis_rows_read": [ru, rv],
           "workload": "cfg3 (BASELINE.json configs[2]): one series N=2^20 L=2^19 k=32, decompose + reconstruct",
           "roofline": {"bound": "hbm", "achieved": byt / (ms * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                        "frac": byt / (ms * 1e-3) / 1e9 / peak, "alg_bytes": byt}}
    ms2, inf2, m2, ru2, rv2, byt2 = one(3)
    res["pro"] = {"value": k / (ms2 * 1e-3), "ms": ms2, "steps": m2, "reorth_steps": int(inf2["reorth_steps"]),
                  "basis_rows_read": [ru2, rv2], "status": int(inf2["status"]),
                  "roofline_frac": byt2 / (ms2 * 1e-3) / 1e9 / peak}
    del x
    torch.cuda.empty_cache()
    return res


# ------------------------------------------------------------------------ clocks
class ClockSampler:
    """Samples SM clock and throttle reasons with NVML every 100 ms in a thread."""

    def __init__(self, dev: int):
        self.dev = dev
        self.samples = []
        self.reasons = set()
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(dev)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover
            self.err = str(e)

    def _run(self):
        nv = self.nv
        names = {
            "gpu_idle": getattr(nv, "nvmlClocksEventReasonGpuIdle", 0x1),
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "hw_power_brake_slowdown": getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for n, bit in names.items():
                    if r & bit and n != "gpu_idle":
                        self.reasons.add(n)
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": float(self.max_mhz),
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------------------ peaks
def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (driver-measured copy)"
    return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


def ncu_traffic(name: str, batch: int):
    """dram read+write bytes per launch of `name` from the committed ncu summary of the
    current round (profiles/ncu_r02_cfg2_summary*.json) for the same batch, else None."""
    for p in sorted(glob.glob(os.path.join(ROOT, "profiles", "ncu_r02*cfg2_summary*.json")), reverse=True):
        try:
            d = json.load(open(p))
            if name in d and d[name].get("dram_bytes_per_launch"):
                if d[name].get("batch") == batch:
                    return float(d[name]["dram_bytes_per_launch"]), os.path.basename(p)
        except Exception:
            pass
    return None, None


# ------------------------------------------------------------------------ oracle arm
def oracle_sample(cores: int, seconds_hint: float = 20.0):
    """Time the CPU oracle on a bounded sample of cfg2: each of `cores` threads runs ONE
    Jacobi sweep of a different cfg2 series (GIL released inside the C call) plus the k
    direct averagings; the full per-series time is extrapolated with the sweep count the
    oracle itself needed on cfg2 series (tests/golden/oracle_cfg2_*.npz, written by
    oracle/make_golden.py).  Returns (triples/s on `cores` cores, description)."""
    from concurrent.futures import ThreadPoolExecutor

    import oracle
    N, L, k = CFG["N"], CFG["L"], CFG["k"]
    K = N - L + 1
    sweeps = []
    for p in glob.glob(os.path.join(ROOT, "tests", "golden", "oracle_cfg2_*.npz")):
        sweeps.append(abs(int(np.load(p)["sweeps"])))
    s_full = float(np.mean(sweeps)) if sweeps else 12.0
    rng = np.random.default_rng(0)
    u = rng.standard_normal(L); u /= np.linalg.norm(u)
    v = rng.standard_normal(K); v /= np.linalg.norm(v)

    def work(i):
        f = ssa_inputs.cfg2_series(i, N)
        t0 = time.perf_counter()
        oracle.svd_sweeps(f, L, k, 1)
        t1 = time.perf_counter()
        for _ in range(k):
            oracle.hankelize_rank1(1.0, u, v)
        t2 = time.perf_counter()
        return t1 - t0, t2 - t1

    oracle.build()
    t0 = time.perf_counter()
    with ThreadPoolExecutor(cores) as ex:
        res = list(ex.map(work, range(cores)))
    wall = time.perf_counter() - t0
    per_series = float(np.mean([a * s_full + b for a, b in res]))
    rate = cores * k / per_series
    desc = (f"{cores} cfg2 series (one per core, threads): 1 Jacobi sweep each timed "
            f"({np.mean([a for a, _ in res]):.2f} s) x {s_full:.1f} sweeps the oracle needs on cfg2 "
            f"+ {k} direct averagings ({np.mean([b for _, b in res]):.2f} s); wall {wall:.1f} s")
    return rate, desc, wall


def run_reference(args, rank):
    if rank != 0:
        return 0
    cores = os.cpu_count() or 1
    times = []
    for _ in range(args.warmup if args.warmup < 1 else 1):
        pass
    vals = []
    descs = []
    for _ in range(max(1, args.steps)):
        rate, desc, wall = oracle_sample(cores)
        vals.append(rate)
        times.append(wall)
        descs.append(desc)
    value = float(np.median(vals))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * CFG["batch"] * CFG["k"] / value,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "cfg2: 4096 series N=4096 L=2048 k=16, decompose+reconstruct (CPU oracle)",
                   "N": CFG["N"], "L": CFG["L"], "k": CFG["k"], "batch_per_gpu": CFG["batch"]},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": descs[0]},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------ our arm
def run_cfg2(P, ctx, host, b0, reorth, steps, warmup, flush, clk=None, **plan_kw):
    """Time `steps` decompose + reconstruct steps of this rank's shard (host rows, global
    index b0 of row 0) with the given reorthogonalization; returns a dict of results."""
    import torch
    N, L, k = CFG["N"], CFG["L"], CFG["k"]
    K = N - L + 1
    B = host.shape[0]
    series = torch.from_numpy(host).cuda()
    plan = P.Plan(N, L, k, B, reorth=reorth, series_base=b0, **plan_kw)
    sigma = torch.empty((B, k), dtype=torch.float64, device="cuda")
    U = torch.empty((B, k, L), dtype=torch.float64, device="cuda")
    V = torch.empty((B, k, K), dtype=torch.float64, device="cuda")
    G = torch.empty((B, k, N), dtype=torch.float64, device="cuda")
    info = torch.zeros((B, P.INFO_DTYPE.itemsize), dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()

    def step():
        plan.decompose(series, sigma, U, V, info)
        plan.reconstruct(sigma, U, V, G)

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    ph = {n: [] for n in ("spectrum", "lanczos", "bidiag_svd", "ritz", "hankelize")}
    launches0 = plan.launches
    import contextlib
    with (clk if clk is not None else contextlib.nullcontext()):
        for i in range(steps):
            flush.zero_()                       # L2 flush between timed steps (untimed)
            ctx.barrier()
            torch.cuda.synchronize()
            ev0[i].record(stream)
            step()
            ev1[i].record(stream)
            torch.cuda.synchronize()
            for n, v in plan.phase_ms().items():
                ph[n].append(v)
    launches = (plan.launches - launches0) // steps
    step_ms = np.array([x.elapsed_time(y) for x, y in zip(ev0, ev1)])
    ms = ctx.max_ms(float(step_ms.sum())) / steps
    inf = P.info_to_numpy(info)
    out = dict(plan=plan, sigma=sigma, info=info, inf=inf, ms=ms, launches=launches,
               phase_ms={n: float(np.mean(v)) for n, v in ph.items()}, series=series, G=G, U=U, V=V)
    return out


def main():
    args = parse()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        return run_reference(args, rank)

    import torch
    import torch.distributed as dist

    import paper_0911_4498_b200 as P

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    ctx = Ctx(rank, world)
    N, L, k = CFG["N"], CFG["L"], CFG["k"]
    K = N - L + 1
    GB = args.batch
    # the configured batch (BASELINE configs[1]: 4096 series) sharded by series over the
    # ranks: rank r owns the contiguous block shard_range(GB, r, world),
    # generated from the series' own seeds and started from their global indices
    b0, b1 = ctx.shard(GB)
    B = b1 - b0
    host = ssa_inputs.cfg2_batch(b0, B, N)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    if args.profile_once:
        plan = P.Plan(N, L, k, B, series_base=b0)
        x = torch.from_numpy(host).cuda()
        s_, U_, V_, _ = plan.decompose(x)
        plan.reconstruct(s_, U_, V_)
        torch.cuda.synchronize()
        return 0

    clk = ClockSampler(local)
    r = run_cfg2(P, ctx, host, b0, 3, args.steps, max(3, args.warmup), flush, clk)
    ms_per_step = r["ms"]
    inf = r["inf"]
    gather = None
    if world > 1:
        # the only collective: after compute, all ranks gather sigma and
        # the per-series info over NCCL (timed apart from the compute steps)
        from paper_0911_4498_b200.parallel import gather_rows
        dist.barrier()
        torch.cuda.synchronize()
        g0 = time.perf_counter()
        all_sigma = gather_rows(r["sigma"], world)
        all_info = gather_rows(r["info"], world)
        torch.cuda.synchronize()
        gather = {"ms": 1e3 * (time.perf_counter() - g0), "rows": int(all_sigma.shape[0]),
                  "bytes": int(all_sigma.numel() * 8 + all_info.numel()), "backend": "nccl all_gather"}
        assert all_sigma.shape[0] == GB
    steps_m = inf["steps"].astype(np.int64)
    conv = float(np.mean(inf["converged"]))
    triples = GB * k
    value = triples / (ms_per_step * 1e-3)
    matvecs_local = float((2 * steps_m + 1).sum())
    matvecs = ctx.world * matvecs_local / (ms_per_step * 1e-3) if world == 1 else None
    if world > 1:
        t = torch.tensor([matvecs_local], dtype=torch.float64, device="cuda")
        dist.all_reduce(t)
        matvecs = float(t.item()) / (ms_per_step * 1e-3)

    # roofline of the dominant kernel (lanczos_kernel) from live CUDA events (rank 0's shard)
    peak, peak_src = measured_peaks()
    ph = r["phase_ms"]
    lan = ph["lanczos"]
    alg = lanczos_alg_bytes(steps_m, inf["rows_u"], inf["rows_v"], N, L)
    achieved = alg / (lan * 1e-3) / 1e9
    traffic, traffic_src = ncu_traffic("lanczos_kernel", B)
    ritz_b = ritz_alg_bytes(steps_m, N, L, k)
    hk = ph["hankelize"]
    hk_bw = hankelize_alg_bytes(B * k, N, L) / (hk * 1e-3) / 1e9
    hk_fl = hankelize_flops(B * k, N) / (hk * 1e-3) / 1e12
    fpk, fsrc = fp64_peak()
    fro_equiv = lanczos_alg_bytes(steps_m, fro_rows(steps_m), fro_rows(steps_m), N, L)

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "cfg2 (BASELINE.json configs[1]): 4096 fp64 series N=4096 L=2048 k=16 sharded by "
                               "series over the GPUs, decompose + reconstruct all 16 triples",
                   "N": N, "L": L, "k": k, "global_batch": GB, "batch_per_gpu": B,
                   "parallelism": f"series-sharded x{world} (shard_range; no data-path collective)",
                   "l2": "inputs (134 MB) > L2 and a 256 MiB L2 flush before every timed step",
                   "tol": 1e-12, "reorth": "PRO (Simon/Larsen omega recurrence, eta = eps^(3/4); DESIGN.md R22)"},
        "hankel_matvecs_per_s": matvecs,
        **({"gather": gather} if gather else {}),
        "lanczos_steps": {"min": int(steps_m.min()), "median": float(np.median(steps_m)),
                          "max": int(steps_m.max()), "mean": float(steps_m.mean())},
        "reorth": {"mode": "PRO", "reorth_halfsteps_mean": float(inf["reorth_steps"].mean()),
                   "halfsteps_mean": float((2 * steps_m + 1).mean()),
                   "lanczos_bytes_per_series": alg / B, "fro_equivalent_bytes_per_series": fro_equiv / B,
                   "bytes_vs_fro": alg / fro_equiv},
        "converged_fraction": conv,
        "max_residual": float(inf["max_residual"].max()),
        "phase_ms": ph,
        "roofline": {"kernel": "lanczos_kernel", "bound": "hbm", "achieved": achieved, "peak": peak,
                     "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                     "traffic_src": traffic_src, "peak_src": peak_src,
                     "alg_bytes_per_launch": alg},
        "ritz_roofline": {"kernel": "ritz_kernel", "bound": "hbm", "achieved": ritz_b / (ph["ritz"] * 1e-3) / 1e9,
                          "peak": peak, "unit": "GB/s", "frac": ritz_b / (ph["ritz"] * 1e-3) / 1e9 / peak,
                          "alg_bytes_per_launch": ritz_b},
        "hankelize_roofline": {"kernel": "hankelize_kernel", "bound": "fp64 (model flops, SURVEY.md §8(d))",
                               "achieved": hk_fl, "peak": fpk, "unit": "TFLOP/s", "frac": hk_fl / fpk,
                               "peak_src": fsrc, "hbm_achieved_gbs": hk_bw, "hbm_frac": hk_bw / peak},
        "gpu_launches": int(r["launches"]),
        "clocks": clk.summary(),
    }
    for key in ("plan",):
        r[key].close()
    del r
    torch.cuda.empty_cache()

    # FRO (reorth = 1, round-1 default) on the same shard: the bytes PRO saves, measured
    if not args.no_fro:
        rf = run_cfg2(P, ctx, host, b0, 1, 2, 1, flush)
        inff = rf["inf"]
        mf = inff["steps"].astype(np.int64)
        algf = lanczos_alg_bytes(mf, inff["rows_u"], inff["rows_v"], N, L)
        lanf = rf["phase_ms"]["lanczos"]
        line["fro"] = {"value": triples / (rf["ms"] * 1e-3), "ms_per_step": rf["ms"],
                       "lanczos_steps_mean": float(mf.mean()), "lanczos_bytes_per_series": algf / B,
                       "roofline": {"kernel": "lanczos_kernel", "achieved": algf / (lanf * 1e-3) / 1e9, "peak": peak,
                                    "unit": "GB/s", "frac": algf / (lanf * 1e-3) / 1e9 / peak}}
        rf["plan"].close()
        del rf
        torch.cuda.empty_cache()

    # thick restart: Krylov dimension d = 40, keep
    # p = 20 (the numpy model's trl:40:20, tools/model_reorth.py), FRO inside a cycle
    if not args.no_trl:
        d_trl, p_trl = 40, 20
        rt = run_cfg2(P, ctx, host, b0, 1, 2, 1, flush, restart_dim=d_trl, restart_keep=p_trl)
        inft = rt["inf"]
        mt = inft["steps"].astype(np.int64)
        thick = inft["reserved"].astype(np.int64)
        # CGS rows from the info counters + each restart's in-place rotation of both bases
        # (read d + 1 rows, write p (+1) rows per side)
        rot_b = float((thick * 8 * ((d_trl + 1 + p_trl) * L + (d_trl + 2 + p_trl) * K)).sum())
        algt = lanczos_alg_bytes(mt, inft["rows_u"], inft["rows_v"], N, L) + rot_b
        lant = rt["phase_ms"]["lanczos"]
        line["trl"] = {"value": triples / (rt["ms"] * 1e-3), "ms_per_step": rt["ms"], "restart_dim": d_trl,
                       "restart_keep": p_trl, "lanczos_steps_mean": float(mt.mean()),
                       "thick_restarts_mean": float(thick.mean()), "converged_fraction": float(inft["converged"].mean()),
                       "max_residual": float(inft["max_residual"].max()),
                       "lanczos_bytes_per_series": algt / B,
                       "basis_bytes_per_series": 8 * (d_trl + 1) * (L + K),
                       "basis_bytes_per_series_unrestarted": 8 * (max(256, 8 * k) + 1) * (L + K),
                       "roofline": {"kernel": "lanczos_trl_kernel", "achieved": algt / (lant * 1e-3) / 1e9,
                                    "peak": peak, "unit": "GB/s", "frac": algt / (lant * 1e-3) / 1e9 / peak}}
        rt["plan"].close()
        del rt
        torch.cuda.empty_cache()

    # overshoot of the convergence-test schedule: the first 256 series
    # of the shard with a test after every step vs the default schedule
    if not args.no_overshoot:
        n_o = min(256, B)
        x = torch.from_numpy(host[:n_o].copy()).cuda()
        ms_default = P.info_to_numpy(P.Plan(N, L, k, n_o, series_base=b0).decompose(x)[3])["steps"]
        os.environ["SSA_FIRST_CHECK"] = str(k)
        os.environ["SSA_CHECK_CAP"] = "1"
        try:
            ms_every = P.info_to_numpy(P.Plan(N, L, k, n_o, check_every=1, series_base=b0).decompose(x)[3])["steps"]
        finally:
            del os.environ["SSA_FIRST_CHECK"], os.environ["SSA_CHECK_CAP"]
        d = ms_default.astype(np.int64) - ms_every.astype(np.int64)
        line["overshoot"] = {"series": n_o, "mean_steps": float(d.mean()), "max_steps": int(d.max()),
                             "min_steps": int(d.min()), "note": "default schedule m minus m of a test after every step"}
        torch.cuda.empty_cache()

    # weak scaling (secondary): every rank its own 4096 series, global indices rank*4096 + i
    if world > 1 and not args.no_weak:
        hw = ssa_inputs.cfg2_batch(rank * CFG["batch"], CFG["batch"], N)
        rw = run_cfg2(P, ctx, hw, rank * CFG["batch"], 3, 2, 1, flush)
        line["weak_scaling"] = {"value": world * CFG["batch"] * k / (rw["ms"] * 1e-3), "unit": UNIT,
                                "ms_per_step": rw["ms"], "batch_per_gpu": CFG["batch"], "scaling": "weak"}
        rw["plan"].close()
        del rw, hw
        torch.cuda.empty_cache()

    # e2e through the public C call on host buffers (pinned), copies inside the timed region
    if not args.no_e2e:
        pin_series = torch.from_numpy(host).pin_memory()
        outs = [torch.empty(sh, dtype=torch.float64).pin_memory() for sh in
                [(B, k), (B, k, L), (B, k, K), (B, k, N)]]
        h_info = np.zeros(B, dtype=P.INFO_DTYPE)
        import ctypes
        lib = P.load_library()
        plan2 = P.Plan(N, L, k, B, series_base=b0)
        stream = torch.cuda.current_stream()

        def e2e_step():
            return lib.ssa_run_host(plan2._h, pin_series.data_ptr(), outs[0].data_ptr(), outs[1].data_ptr(),
                                    outs[2].data_ptr(), outs[3].data_ptr(), h_info.ctypes.data,
                                    ctypes.c_void_p(stream.cuda_stream))

        e2e_step()
        times = []
        for _ in range(max(1, min(3, args.steps))):
            flush.zero_()
            ctx.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            e2e_step()
            times.append(time.perf_counter() - t0)
        te = ctx.max_ms(1e3 * float(np.mean(times)))
        line["e2e"] = {"value": triples / (te * 1e-3), "unit": UNIT,
                       "h2d_bytes_per_step": int(B * N * 8),
                       "d2h_bytes_per_step": int(B * k * (1 + L + K + N) * 8 + B * P.INFO_DTYPE.itemsize),
                       "api": "ssa_run_host (pinned host buffers; H2D series, D2H sigma/U/V/recon/info), per GPU"}
        plan2.close()
        torch.cuda.empty_cache()

    if not args.no_micro:
        line["matvec_cfg4"] = micro_matvec(P, peak, ctx)
        line["hankelize_cfg5"] = micro_hankelize(P, peak, ctx)
        line["decompose_cfg3"] = micro_decompose_cfg3(P, peak, ctx)
        line["decompose_cfg1"] = micro_decompose_cfg1(P, ctx)
        line["hmatrix"] = micro_hmatrix(P, ctx)
        line["bootstrap"] = micro_bootstrap(P, ctx)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cores = os.cpu_count() or 1
        rate, desc, wall = oracle_sample(cores)
        line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc}
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(line), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
