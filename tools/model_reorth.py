"""Numpy model of the Lanczos bidiagonalization variants the paper names, on cfg2 series.

PAPER.md:373-386 (sec 3.2.1, no reorthogonalization), :388-400 (FRO), :402-411 (PRO),
:435-446 (restarting).  The question (VERDICT r01 "Next round" #7): how many basis bytes
does each variant read per series at the accuracy the parity tests demand, and how many
steps does the kernel's convergence-test schedule overshoot?

Variants (A = trajectory matrix, applied through FFT correlations, never formed):
  fro       CGS + DGKS against the whole basis every half-step (the shipped kernel)
  pro:<d>   partial reorthogonalization, Simon/Larsen omega recurrences (Larsen 1998);
            when max|omega| > d, CGS against the rows with |omega| > eta = d^(3/2)/...
            (Larsen's intervals, extended by eta) on this half-step and the next
  prof:<d>  as pro, but against the whole basis when triggered (Simon's PRO)
  trl:<D>:<p>  thick restart: Krylov dimension D, keep p Ritz triples (Baglama-Reichel
            augmentation / Wu-Simon thick restart), CGS + DGKS inside a cycle
Bytes: 8 B per basis element read or written (dots pass + update pass per CGS), plus the
restart GEMMs (read the D rows, write p rows per side).

Accuracy measured against LAPACK on the explicit X (2048 x 2049): sigma rel error,
sign-free sine angles of well-separated triples (gap >= 1e-4 sigma_1), true residuals
|Xv - s u|, |X^T u - s v| / sigma_1 and the orthogonality of the Ritz vectors.

  python tools/model_reorth.py [nseries] [variants...]
This is a design tool: it is not the oracle and not on the product path.
"""
from __future__ import annotations

import sys

import numpy as np

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import ssa_inputs  # noqa: E402

EPS = np.finfo(float).eps


class Op:
    def __init__(self, f, L):
        self.N = len(f); self.L = L; self.K = self.N - L + 1
        M = 1
        while M < self.N:
            M <<= 1
        self.M = M
        self.F = np.fft.rfft(f, M)
        self.nmv = 0

    def Xv(self, v):
        self.nmv += 1
        return np.fft.irfft(self.F * np.conj(np.fft.rfft(v, self.M)), self.M)[: self.L]

    def XTu(self, u):
        self.nmv += 1
        return np.fft.irfft(self.F * np.conj(np.fft.rfft(u, self.M)), self.M)[: self.K]


def cgs(r, B, rows=None):
    """CGS + DGKS of r against rows `rows` of B; returns r, coefficients, rows read."""
    if rows is None:
        rows = np.arange(B.shape[0])
    if len(rows) == 0:
        return r, np.zeros(0), 0
    Bs = B[rows]
    n0 = np.linalg.norm(r)
    h = Bs @ r
    r = r - Bs.T @ h
    read = 2 * len(rows)
    if np.linalg.norm(r) < n0 / np.sqrt(2):
        h2 = Bs @ r
        r = r - Bs.T @ h2
        h = h + h2
        read += 2 * len(rows)
    return r, h, read


def ritz_check(Bsm, alpha_next):
    P, w, Qt = np.linalg.svd(Bsm, full_matrices=False)
    res = alpha_next * np.abs(P[-1, :])
    return P, w, Qt.T, res


def schedule_kernel(k, ce=4, cap=12):
    """The shipped batched kernel's test schedule (ssa_lanczos.cu / ssa_api.cu)."""
    return dict(first=3 * k + 8, ce=ce, cap=cap, frac=0.7, stop=0.5)


def run(op, k, variant, tol=1e-12, m_max=400, seed=42, sched=None):
    """GKL (u_1 seeded) with the variant; convergence tested every step (records m_first,
    the first m with residual <= tol) and the kernel schedule (m_stop).  Returns dict."""
    L, K = op.L, op.K
    rng = np.random.default_rng(seed)
    kind = variant.split(":")[0]
    par = variant.split(":")[1:]
    D = int(par[0]) if kind == "trl" else m_max + 2
    pkeep = int(par[1]) if kind == "trl" else 0
    delta = float(par[0]) if kind in ("pro", "prof") else 0.0  # suffix ":nl": no local dot, plain beta_j / alpha_j
    eta = delta ** 1.5 if kind == "pro" else 0.0   # Larsen: eta = eps^(3/4) for delta = sqrt(eps)
    if kind == "pro" and len(par) > 1 and par[1] != "nl":
        eta = float(par[1])                        # pro:<delta>:<eta> selection threshold
    U = np.zeros((m_max + 2, L)); V = np.zeros((m_max + 2, K))
    nU = nV = 0
    Bsm = np.zeros((m_max + 2, m_max + 2))  # A V[:nV-1] = U[:nU] Bsm[:nU, :nV-1]
    p0 = rng.uniform(-1, 1, L)
    U[0] = p0 / np.linalg.norm(p0); nU = 1
    reads = 0; writes = L                      # basis elements read / written
    mu = np.zeros(m_max + 3); nu = np.zeros(m_max + 3)   # omega estimates of the newest u / v
    mu_old = np.zeros(m_max + 3); nu_old = np.zeros(m_max + 3)
    alpha = [0.0]; beta = [0.0, np.linalg.norm(p0)]
    force_u = force_v = None
    ntrig = 0
    anorm = 0.0
    m_first = None; m_stop = None; restarts = 0
    sc = sched or schedule_kernel(k)
    next_check = sc["first"]; prev = None
    out = {}
    m_total = 0
    while True:
        # ---- right step: r = A^T u_last - (coefficients vs V) ----
        j = nU  # 1-based index of u_last
        r = op.XTu(U[nU - 1])
        if kind in ("fro", "trl"):
            r, h, rd = cgs(r, V[:nV]); reads += rd * K   # A V = U Bsm: columns come from the left steps
        else:
            # local step of plain GKL: r -= beta_j v_{j-1}
            if nV > 0:
                hj = V[nV - 1] @ r if not variant.endswith(":nl") else beta[j]
                r = r - hj * V[nV - 1]
        a = np.linalg.norm(r)
        if kind in ("pro", "prof") and nV > 0:
            # omega recurrence for v_j vs v_1..v_{j-1} (Larsen 1998, update_nu)
            # alpha_j nu_{j,i} = alpha_i mu_{j,i} + beta_{i+1} mu_{j,i+1} - beta_j nu_{j-1,i}
            bj = beta[j]
            new = np.zeros(m_max + 3)
            for i in range(1, nV + 1):
                t = alpha[i] * mu[i] + beta[i + 1] * mu[i + 1] - bj * nu[i]
                d = EPS * (np.hypot(alpha[i], beta[i + 1]) + np.hypot(a, bj)) + EPS * anorm
                t = t + np.copysign(d, t)
                new[i] = t / a
            sel = None
            if np.max(np.abs(new[1:nV + 1])) > delta or force_v is not None:
                if kind == "prof":
                    sel = np.arange(nV)
                else:
                    idx = np.nonzero(np.abs(new[1:nV + 1]) > eta)[0] if force_v is None else force_v
                    sel = idx
                r, h, rd = cgs(r, V[:nV], sel); reads += rd * K; ntrig += 1
                a = np.linalg.norm(r)
                new[1:nV + 1][sel] = EPS
                force_v = None if force_v is not None else sel
            nu_old, nu = nu, new
        if nV > 0:
            pass
        alpha.append(a)
        anorm = max(anorm, a)
        V[nV] = r / a; nV += 1; writes += K
        if kind in ("pro", "prof"):
            nu[nV] = 1.0
        m = nV - 1  # B_m with alpha_{m+1} = a
        m_total += 1
        # ---- convergence test (every step for the model; the kernel's schedule) ----
        if m >= k:
            P, w, Q, res = ritz_check(Bsm[:nU, :nV - 1], a)
            rel = np.max(res[:k]) / w[0]
            if m_first is None and rel <= tol:
                m_first = m_total
            if m_stop is None and (kind != "fro" or m_total >= next_check):
                if rel <= sc["stop"] * tol:
                    m_stop = m_total
                elif kind == "fro":
                    step = sc["ce"]
                    if prev is not None and 0 < rel < prev[0]:
                        rate = np.log(rel / prev[0]) / (m_total - prev[1])
                        need = np.log(sc["stop"] * tol / rel) / rate
                        s2 = int(sc["frac"] * need)
                        if s2 > step:
                            step = min(s2, sc["cap"])
                    prev = (rel, m_total)
                    next_check = m_total + step
            done = (rel <= tol) if kind != "fro" else (m_stop is not None)
            if done or m_total >= m_max:
                out.update(P=P, w=w, Q=Q, nU=nU, nV=nV - 1, rel=rel)
                break
            if kind == "trl" and nV - 1 >= D:
                # thick restart: keep p Ritz triples; v_new is the residual direction
                p = pkeep
                Up = P[:, :p].T @ U[:nU]; Vp = Q[:, :p].T @ V[:nV - 1]
                reads += nU * L + (nV - 1) * K; writes += p * (L + K)
                vnew = V[nV - 1].copy()
                U[:] = 0; V[:] = 0; Bsm[:] = 0
                U[:p] = Up; V[:p] = Vp; V[p] = vnew
                Bsm[:p, :p] = np.diag(w[:p])
                # u_i^T A v_new = rho_i = a P[-1, i]: the left step's CGS recomputes them into Bsm
                nU = p; nV = p + 1
                restarts += 1
        # ---- left step: p = A v_last - coefficients vs U ----
        pv = op.Xv(V[nV - 1])
        if kind in ("fro", "trl"):
            pv, g, rd = cgs(pv, U[:nU]); reads += rd * L
            Bsm[:nU, nV - 1] += g
        else:
            gj = U[nU - 1] @ pv if not variant.endswith(":nl") else alpha[nV]
            pv = pv - gj * U[nU - 1]
            Bsm[nU - 1, nV - 1] += gj
        b = np.linalg.norm(pv)
        if kind in ("pro", "prof"):
            # beta_{j+1} mu_{j+1,i} = alpha_i nu_{j,i} + beta_i nu_{j,i-1} - alpha_j mu_{j,i}
            aj = alpha[nV]
            new = np.zeros(m_max + 3)
            for i in range(1, nU + 1):
                t = alpha[i] * nu[i] + beta[i] * nu[i - 1] - aj * mu[i]
                d = EPS * (np.hypot(alpha[i], beta[i]) + np.hypot(aj, b)) + EPS * anorm
                t = t + np.copysign(d, t)
                new[i] = t / b
            if np.max(np.abs(new[1:nU + 1])) > delta or force_u is not None:
                if kind == "prof":
                    sel = np.arange(nU)
                else:
                    sel = np.nonzero(np.abs(new[1:nU + 1]) > eta)[0] if force_u is None else force_u
                pv, g, rd = cgs(pv, U[:nU], sel); reads += rd * L; ntrig += 1
                b = np.linalg.norm(pv)
                new[1:nU + 1][sel] = EPS
                force_u = None if force_u is not None else sel
            mu_old, mu = mu, new
        beta.append(b)
        anorm = max(anorm, b)
        U[nU] = pv / b; nU += 1; writes += L
        Bsm[nU - 1, nV - 1] = b
        if kind in ("pro", "prof"):
            mu[nU] = 1.0
    P, w, Q = out["P"], out["w"], out["Q"]
    Uk = P[:, :k].T @ U[: out["nU"]]
    Vk = Q[:, :k].T @ V[: out["nV"]]
    reads += out["nU"] * L + out["nV"] * K  # Ritz assembly
    writes += k * (L + K)
    return dict(sigma=w[:k], U=Uk, V=Vk, m=m_total, m_first=m_first, m_stop=m_stop, restarts=restarts,
                bytes=8.0 * (reads + writes), matvecs=op.nmv, rel=out["rel"], ntrig=ntrig)


def explicit(f, L):
    N = len(f); K = N - L + 1
    idx = np.arange(L)[:, None] + np.arange(K)[None, :]
    return f[idx]


def accuracy(X, r, k, s_ref, U_ref, V_ref):
    s = r["sigma"]; U = r["U"]; V = r["V"]
    srel = np.max(np.abs(s - s_ref[:k]) / s_ref[:k])
    gap = DELTA = 1e-4 * s_ref[0]
    ang = 0.0
    for i in range(k):
        lo = s_ref[i - 1] - s_ref[i] if i > 0 else np.inf
        hi = s_ref[i] - s_ref[i + 1]
        if min(lo, hi) >= DELTA:
            for a, b in ((U_ref[:, i], U[i]), (V_ref[i], V[i])):
                b = b / np.linalg.norm(b)
                ang = max(ang, np.linalg.norm(b - (a @ b) * a))
    res = 0.0
    for i in range(k):
        res = max(res, np.linalg.norm(X @ V[i] - s[i] * U[i]), np.linalg.norm(X.T @ U[i] - s[i] * V[i]))
    orth = max(np.abs(U @ U.T - np.eye(k)).max(), np.abs(V @ V.T - np.eye(k)).max())
    return srel, ang, res / s_ref[0], orth


def main():
    ns = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    variants = sys.argv[2:] or ["fro", "prof:1.5e-8", "pro:1.5e-8", "prof:1e-10", "pro:1e-10", "prof:1.8e-12",
                                "pro:1.8e-12", "trl:48:24", "trl:64:32", "trl:40:20"]
    c = ssa_inputs.CONFIGS["cfg2"]
    N, L, k = c["N"], c["L"], c["k"]
    rows = {v: [] for v in variants}
    for i in range(ns):
        f = ssa_inputs.cfg2_series(i * 997, N)
        X = explicit(f, L)
        U_ref, s_ref, Vt = np.linalg.svd(X, full_matrices=False)
        for v in variants:
            op = Op(f, L)
            r = run(op, k, v)
            srel, ang, res, orth = accuracy(X, r, k, s_ref, U_ref, Vt)
            rows[v].append((r["m"], r["m_first"], r["m_stop"], r["bytes"], r["matvecs"], r["restarts"], srel, ang, res,
                            orth))
            print(f"series {i * 997:5d} {v:14s} m={r['m']:4d} m_first={r['m_first']} m_stop={r['m_stop']} "
                  f"MB={r['bytes'] / 1e6:7.1f} mv={r['matvecs']:4d} rs={r['restarts']:2d} trig={r['ntrig']:3d} "
                  f"srel={srel:.1e} ang={ang:.1e} res={res:.1e} orth={orth:.1e}", flush=True)
    print("\nsummary (mean over series)")
    base = np.mean([t[3] for t in rows["fro"]]) if "fro" in rows else None
    for v in variants:
        a = np.array([[np.nan if x is None else x for x in t] for t in rows[v]], dtype=float)
        mb = a[:, 3].mean() / 1e6
        print(f"{v:14s} m={a[:, 0].mean():6.1f} MB={mb:7.1f} ({'' if base is None else f'{a[:, 3].mean() / base:.2f}x fro'}) "
              f"matvecs={a[:, 4].mean():6.1f} worst srel={np.nanmax(a[:, 6]):.1e} ang={np.nanmax(a[:, 7]):.1e} "
              f"res={np.nanmax(a[:, 8]):.1e} orth={np.nanmax(a[:, 9]):.1e}")
        if v == "fro":
            print(f"   fro: kernel schedule stops at m={np.nanmean(a[:, 2]):.1f}, first m meeting tol "
                  f"{np.nanmean(a[:, 1]):.1f} (overshoot {np.nanmean(a[:, 2] - a[:, 1]):.1f} steps)")


if __name__ == "__main__":
    main()
