"""Cluster-aware parity comparator (SURVEY.md §8(c) "Parity rule").

Host-side test logic only.  Given oracle triples (σ°, U°, V°, G°) and candidate triples
(σ, U, V, G) it classifies the first k oracle triples into well-separated triples and
clusters using the gap rule δ = 1e-4·σ°₁, and measures
  * relative σ error,
  * sign-free sine angles ‖(I − ûûᵀ)u‖₂ (never acos / sqrt(1 − cos²), whose √ε floor
    would fail a 1e-8 target even for exact vectors — SURVEY.md §0 finding 6),
  * for a cluster C, the largest principal-angle sine between span(U_C) and span(U°_C),
  * reconstruction errors, per triple or summed over a cluster,
  * when the series is given: the TRUE residuals ‖Xv_i − σ_iu_i‖, ‖Xᵀu_i − σ_iv_i‖ of
    every triple (straddling clusters included, where the vectors themselves are not
    unique) through the oracle's explicit product, ≤ res_tol·σ°₁ (10·tol, SURVEY.md
    §8(c) "Lanczos internals"), and the orthonormality of the computed U, V.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

DELTA = 1e-4


def clusters(sig_ref: np.ndarray, k: int, delta: float = DELTA):
    """Split indices 0..k-1 into groups of consecutive non-separated values.
    sig_ref must hold at least k values; index k (if present) decides straddling.
    Returns list of (indices, straddles)."""
    s = np.asarray(sig_ref, dtype=np.float64)
    gap_tol = delta * s[0]
    groups = []
    cur = [0]
    for i in range(1, k):
        if s[i - 1] - s[i] >= gap_tol:
            groups.append(cur)
            cur = [i]
        else:
            cur.append(i)
    groups.append(cur)
    out = []
    for g in groups:
        last = g[-1]
        straddles = (last == k - 1) and (len(s) > k) and (s[k - 1] - s[k] < gap_tol)
        out.append((g, bool(straddles)))
    return out


def sine_angle(a: np.ndarray, b: np.ndarray) -> float:
    """Sign-free sine of the angle between unit-ish vectors: ‖b − (âᵀb)â‖ / ‖b‖."""
    a = a / np.linalg.norm(a)
    b = b / np.linalg.norm(b)
    r = b - np.dot(a, b) * a
    return float(np.linalg.norm(r))


def subspace_sine(A: np.ndarray, B: np.ndarray) -> float:
    """Largest principal-angle sine between span of rows of A and span of rows of B
    (both c × n, rows orthonormal): ‖(I − QₐQₐᵀ) Q_b‖₂."""
    Qa, _ = np.linalg.qr(np.asarray(A, dtype=np.float64).T)
    Qb, _ = np.linalg.qr(np.asarray(B, dtype=np.float64).T)
    R = Qb - Qa @ (Qa.T @ Qb)
    return float(np.linalg.norm(R, 2))


@dataclass
class ParityReport:
    sigma_rel: list = field(default_factory=list)        # (i, err, separated)
    u_angle: list = field(default_factory=list)          # (indices, sine)
    v_angle: list = field(default_factory=list)
    recon: list = field(default_factory=list)            # (indices, normwise err / scale)
    residual: list = field(default_factory=list)         # (i, max true residual / sigma_1)
    failures: list = field(default_factory=list)

    def ok(self) -> bool:
        return not self.failures

    def worst(self):
        def mx(lst, j):
            return max([t[j] for t in lst], default=0.0)
        return dict(sigma=mx(self.sigma_rel, 1), u=mx(self.u_angle, 1), v=mx(self.v_angle, 1), recon=mx(self.recon, 1),
                    residual=mx(self.residual, 1))


def true_residuals(f, L, sig, U, V, idx, matvec):
    """max(‖X v_i − σ_i u_i‖, ‖Xᵀ u_i − σ_i v_i‖) for i in idx; matvec(f, L, x, transpose)
    is the oracle's explicit-entry product (Eqs. (1)-(2), PAPER.md:323-328 define the
    residuals the Lanczos stop rule bounds)."""
    out = []
    for i in idx:
        r1 = np.linalg.norm(matvec(f, L, V[i]) - sig[i] * U[i])
        r2 = np.linalg.norm(matvec(f, L, U[i], True) - sig[i] * V[i])
        out.append(max(r1, r2))
    return out


def compare(sig_ref, U_ref, V_ref, sig, U, V, k, G_ref=None, G=None, recon_scale=None,
            sigma_tol=1e-10, angle_tol=1e-8, recon_tol=1e-9, delta=DELTA, f=None, L=None, res_tol=1e-11,
            orth_tol=1e-12) -> ParityReport:
    """Cluster-aware comparison of the first k triples.  sig_ref may hold k+1 values so
    the straddling rule can be applied.  recon_scale is ‖F‖₂ (default) — errors are
    normwise ‖g − g°‖₂ / recon_scale.  With the series f and window L, every triple's
    true residual (oracle product) must be ≤ res_tol·σ°₁ and U, V orthonormal ≤ orth_tol."""
    rep = ParityReport()
    sig_ref = np.asarray(sig_ref)
    if f is not None:
        import oracle
        res = true_residuals(f, L, sig, U, V, range(k), oracle.matvec)
        for i, r in enumerate(res):
            rep.residual.append((i, float(r / sig_ref[0])))
            if r > res_tol * sig_ref[0]:
                rep.failures.append(f"true residual of triple {i}: {r / sig_ref[0]:.3e} sigma_1 > {res_tol:g}")
        for name, Q in (("U", U[:k]), ("V", V[:k])):
            o = float(np.abs(Q @ Q.T - np.eye(k)).max())
            if o > orth_tol:
                rep.failures.append(f"{name} orthonormality {o:.3e} > {orth_tol:g}")
    for grp, straddles in clusters(sig_ref, k, delta):
        separated = len(grp) == 1 and not straddles
        for i in grp:
            err = abs(sig[i] - sig_ref[i]) / sig_ref[i] if sig_ref[i] > 0 else abs(sig[i])
            rep.sigma_rel.append((i, float(err), separated))
            if err > sigma_tol:
                rep.failures.append(f"sigma[{i}] rel err {err:.3e} > {sigma_tol:g} ({'separated' if separated else 'cluster'})")
        if straddles:
            continue
        if separated:
            i = grp[0]
            su = sine_angle(U_ref[i], U[i]); sv = sine_angle(V_ref[i], V[i])
        else:
            su = subspace_sine(U_ref[grp], U[grp]); sv = subspace_sine(V_ref[grp], V[grp])
        rep.u_angle.append((tuple(grp), su)); rep.v_angle.append((tuple(grp), sv))
        if su > angle_tol:
            rep.failures.append(f"u angle {grp}: {su:.3e} > {angle_tol:g}")
        if sv > angle_tol:
            rep.failures.append(f"v angle {grp}: {sv:.3e} > {angle_tol:g}")
        if G_ref is not None and G is not None:
            gr = np.sum(G_ref[grp], axis=0); gg = np.sum(G[grp], axis=0)
            e = float(np.linalg.norm(gg - gr) / recon_scale)
            rep.recon.append((tuple(grp), e))
            if e > recon_tol:
                rep.failures.append(f"recon {grp}: {e:.3e} > {recon_tol:g}")
    return rep
