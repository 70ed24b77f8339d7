// lanczos_trl.cuh -- thick-restarted Lanczos bidiagonalization (sec 3.3,
// "restarting schemes"; the Wu-Simon / Baglama-Reichel thick restart), SURVEY.md 8(f) #1.
// Included by ssa_lanczos.cu (it uses that file's correlation, CGS and ring helpers).
//
// The bases hold at most d + 1 vectors per side (d = a.trl_d, the Krylov dimension), so
// the basis storage, d + 1 rows instead of m_max + 1, and the reorthogonalization traffic
// per step are capped by d.  The projected matrix T (rows: U vectors, columns: V vectors)
// keeps A V = U T exactly and A^T U = V T^T + alpha v_next e_last^T (Eqs. (1)-(2),
// PAPER.md:323-328, the residual on the A^T side).  First cycle: T is the lower bidiagonal
// B_m of Alg. 1.  At a restart (the V basis is full), with T = P Omega Q^T:
//   U <- U P[:, :p],  V <- [V Q[:, :p], v_next],  T <- diag(omega_1..omega_p)
// (the kept Ritz triples and the residual direction); the next u half-step computes
// A v_next - sum_i rho_i u~_i by CGS against the kept u~_i, whose coefficients
// rho_i = alpha_next P_{last,i} become the arrow column of T; later steps append the usual
// bidiagonal (upper, after a restart).  The small SVD of T (not bidiagonal after a
// restart) is a one-sided Jacobi SVD in shared memory; the residual of triple i is
// alpha_next |P_{last,i}| as in the unrestarted test (R7).  Reorthogonalization
// inside a cycle is FRO (CGS + DGKS, or two passes for reorth = 2).
#pragma once

namespace ssa {

__device__ __forceinline__ int rr_player(int pos, int round, int n2) {
  return pos == 0 ? 0 : 1 + (pos - 1 + round) % (n2 - 1);
}

// One-sided (Hestenes) Jacobi SVD of T_c = T[0:nu][0:nc] (row-major, ldT) into W (column c
// of the rotated matrix at W + c ldw, ldw >= nu) and Qm (column c at Qm + c nc): T_c Q = W,
// sigma_c = |W_c|, P_c = W_c / sigma_c.  Round-robin pairs, one half-warp (16 lanes) per
// pair, so the 16 half-warps of the CTA rotate 16 pairs at once; sweeps until none
// rotates (|w_p . w_q| <= 1e-15 |w_p| |w_q|, the oracle's criterion).  ord[i] = column of
// the i-th largest sigma (ties by column index).
__device__ __forceinline__ double half_sum(double v) {  // sum over the 16 lanes of a half-warp
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ void trl_jacobi(const double* T, int ldT, int nu, int nc, double* W, int ldw, double* Qm, double* sig,
                           int* ord, int* redi) {
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const int hw = 2 * w + (lane >> 4), hl = lane & 15;  // half-warp index, lane in it
  constexpr int kHalfWarps = 2 * kWarps;
  for (int idx = tid; idx < nc * ldw; idx += blockDim.x) {
    const int c = idx / ldw, r = idx - c * ldw;
    W[idx] = (r < nu) ? T[r * ldT + c] : 0.0;
  }
  for (int idx = tid; idx < nc * nc; idx += blockDim.x) Qm[idx] = (idx / nc == idx % nc) ? 1.0 : 0.0;
  __syncthreads();
  const int n2 = nc + (nc & 1);
  for (int sweep = 0; sweep < 60 && n2 >= 2; ++sweep) {
    int rot = 0;
    for (int round = 0; round < n2 - 1; ++round) {
      for (int pb = 0; pb < n2 / 2; pb += kHalfWarps) {  // warp-uniform trip count
        const int pi = pb + hw;
        int p = rr_player(pi, round, n2), q = rr_player(n2 - 1 - pi, round, n2);
        const bool act = pi < n2 / 2 && p < nc && q < nc;  // both halves run the shuffles
        if (p > q) {
          const int t = p;
          p = q;
          q = t;
        }
        double* wp = W + (size_t)(act ? p : 0) * ldw;
        double* wq = W + (size_t)(act ? q : 0) * ldw;
        double a = 0.0, b = 0.0, c = 0.0;
        if (act)
          for (int r = hl; r < nu; r += 16) {
            const double x = wp[r], y = wq[r];
            a = fma(x, x, a);
            b = fma(y, y, b);
            c = fma(x, y, c);
          }
        a = half_sum(a);
        b = half_sum(b);
        c = half_sum(c);
        if (act && c != 0.0 && fabs(c) > 1e-15 * sqrt(a * b)) {
          const double zeta = (b - a) / (2.0 * c);
          const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(fma(zeta, zeta, 1.0)));
          const double cs = 1.0 / sqrt(fma(t, t, 1.0)), sn = cs * t;
          for (int r = hl; r < nu; r += 16) {
            const double x = wp[r], y = wq[r];
            wp[r] = cs * x - sn * y;
            wq[r] = fma(sn, x, cs * y);
          }
          double* qp = Qm + (size_t)p * nc;
          double* qq = Qm + (size_t)q * nc;
          for (int r = hl; r < nc; r += 16) {
            const double x = qp[r], y = qq[r];
            qp[r] = cs * x - sn * y;
            qq[r] = fma(sn, x, cs * y);
          }
          rot = 1;
        }
      }
      __syncthreads();
    }
    if (!block_or(rot, redi)) break;
  }
  for (int c = tid; c < nc; c += blockDim.x) {
    double ss = 0.0;
    for (int r = 0; r < nu; ++r) ss = fma(W[(size_t)c * ldw + r], W[(size_t)c * ldw + r], ss);
    sig[c] = sqrt(ss);
  }
  __syncthreads();
  for (int c = tid; c < nc; c += blockDim.x) {
    int rank = 0;
    for (int c2 = 0; c2 < nc; ++c2) rank += (sig[c2] > sig[c] || (sig[c2] == sig[c] && c2 < c)) ? 1 : 0;
    ord[rank] = c;
  }
  __syncthreads();
}

// In-place restart of one basis side: rows i < p become sum_r C(r, i) row_r over the nrows
// old rows (C(r, i) = Wc[ord[i] ldw + r] * scl[i]), and row p a copy of old row src (none
// for src < 0).  Each warp owns a column slab, in chunks of 32 / LPE elements: the LPE
// lanes of an element each keep 16 of its p <= 16 LPE outputs in registers while the old
// rows stream past (8 rows in flight), so a chunk is read completely before it is
// overwritten (only this warp touches it).
template <int LPE>
__device__ void trl_restart_side(double* basis, int ld, int nrows, int p, const double* Wc, int ldw, const int* ord,
                                 const double* scl, int src) {
  constexpr int EPW = 32 / LPE;  // elements per warp chunk
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int el = lane / LPE, sub = lane % LPE;  // element in the chunk, output subset
  const int slab = ld / kWarps;
  for (int e0 = 0; e0 < slab; e0 += EPW) {
    const int col = w * slab + e0 + el;
    const bool ok = e0 + el < slab;
    double acc[16];
#pragma unroll
    for (int t = 0; t < 16; ++t) acc[t] = 0.0;
    const double keep = (ok && src >= 0 && sub == 0) ? __ldcg(basis + (size_t)src * ld + col) : 0.0;
    for (int r0 = 0; r0 < nrows; r0 += 8) {
      double x[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) x[q] = (ok && r0 + q < nrows) ? __ldcg(basis + (size_t)(r0 + q) * ld + col) : 0.0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        if (r0 + q < nrows) {
#pragma unroll
          for (int t = 0; t < 16; ++t) {
            const int i = sub + LPE * t;
            if (i < p) acc[t] = fma(Wc[(size_t)ord[i] * ldw + r0 + q] * scl[i], x[q], acc[t]);
          }
        }
      }
    }
    __syncwarp();
    if (ok) {
#pragma unroll
      for (int t = 0; t < 16; ++t) {
        const int i = sub + LPE * t;
        if (i < p) basis[(size_t)i * ld + col] = acc[t];
      }
      if (src >= 0 && sub == 0) basis[(size_t)p * ld + col] = keep;
    }
  }
}

// restart of one side with LPE = ceil(p / 16) lanes per element
__device__ __noinline__ void trl_restart(double* basis, int ld, int nrows, int p, const double* Wc, int ldw,
                                         const int* ord, const double* scl, int src) {
  if (p <= 16) trl_restart_side<1>(basis, ld, nrows, p, Wc, ldw, ord, scl, src);
  else if (p <= 32) trl_restart_side<2>(basis, ld, nrows, p, Wc, ldw, ord, scl, src);
  else trl_restart_side<4>(basis, ld, nrows, p, Wc, ldw, ord, scl, src);
}

__global__ void __launch_bounds__(kThreads, 2) lanczos_trl_kernel(const DecomposeArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  LSmem sm = carve(smem_raw, a);
  const int tid = threadIdx.x, w = tid >> 5;
  const FftShape sh = make_shape(a.H);
  const int slab_max = (a.ldL > a.ldK ? a.ldL : a.ldK) / kWarps;
  double2* fbuf = reinterpret_cast<double2*>(sm.regionA);
  double* rings = reinterpret_cast<double*>(sm.regionA);
  double* part = rings + (size_t)kWarps * kStages * slab_max;
  const int pstride = a.m_max + 2;
  const int d = a.trl_d, ldT = a.m_max + 1;
  // Jacobi scratch in region A (used between half-steps only)
  const int ldw = d + 1;
  double* Wj = reinterpret_cast<double*>(sm.regionA);
  double* Qj = Wj + (size_t)(d + 1) * ldw;
  double* sg = Qj + (size_t)(d + 1) * (d + 1);
  int* ord = reinterpret_cast<int*>(sg + (d + 1));
  double* T = sm.T;
  double* scl = sm.nu;   // restart: 1 / sigma of the kept columns (m_max + 3 >= p entries)
  double* hacc = sm.mu;  // restart: the arrow column, accumulated by the next u-side CGS

  const TwSmem tw = load_tw2(a.tw, sm.tw, 2 * a.H);
  WarpRing rg;
  ring_init(rg, rings + (size_t)w * kStages * slab_max, sm.bars + w * kStages);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  const int L = a.L, K = a.K, k = a.k;
  const int mode = a.reorth_mode == 2 ? 2 : 1;

  while (true) {
    __syncthreads();
    if (tid == 0) sm.redi[4] = atomicAdd(a.counters + 0, 1);
    __syncthreads();
    const int bl = sm.redi[4];
    if (bl >= a.nb) break;
    const int b = a.b0 + bl;
    const double* f = a.series + (size_t)b * a.N;
    const double2* spec = a.spec + (size_t)bl * (a.H + 1);
    double* U = a.U + (size_t)bl * (a.m_max + 1) * a.ldL;
    double* V = a.V + (size_t)bl * (a.m_max + 1) * a.ldK;
    int* st = a.state + (size_t)bl * kStateInts;

    int bad = 0;
    for (int t = tid; t < a.N; t += blockDim.x) bad |= !isfinite(f[t]);
    if (block_or(bad, sm.redi)) {
      if (tid == 0)
        for (int q = 0; q < kStateInts; ++q) st[q] = (q == 5) ? 1 : 0;
      continue;
    }
    // Alg. 1 lines 1-2: u_1 = p_0 / |p_0| (the seeded start vector of lanczos_kernel)
    double ss = 0.0;
    for (int t = tid; t < a.ldL; t += blockDim.x) {
      const double v = (t < L) ? rng_uniform_pm1(a.seed, (uint64_t)(b + a.series_base), (uint64_t)t) : 0.0;
      sm.bufU[t] = v;
      ss += v * v;
    }
    for (int t = tid; t < a.ldK; t += blockDim.x) sm.bufV[t] = 0.0;
    for (int i = tid; i < ldT * ldT; i += blockDim.x) T[i] = 0.0;
    const double beta1 = sqrt(block_sum(ss, sm.red));
    normalize_store(sm.bufU, L, a.ldL, 1.0 / beta1, U);

    int nu = 1, nv = 0, mtot = 0, breakdown = 0, extra = 0, restarts = 0, thick = 0, checks = 0;
    int rows_u = 0, rows_v = 0, rsteps = 0;
    bool fresh = false;
    double runmax = 0.0, prev_res = -1.0;
    int prev_m = 0, next_check = a.first_check;
    const int ce = a.check_every > 0 ? a.check_every : 4;
    while (true) {
      // ---- half-step A: r = X^T u_nu - T[nu-1][nv-1] v_nv; CGS + DGKS against V ----
      const double cA = (nv > 0) ? T[(nu - 1) * ldT + nv - 1] : 0.0;
      correlate_cta(
          fbuf, sh, tw, spec, L, K, [&](int i) { return sm.bufU[i]; },
          [&](int t, double y) { sm.bufV[t] = y - cA * sm.bufV[t]; });
      __syncthreads();
      ss = 0.0;
      for (int t = tid; t < K; t += blockDim.x) ss = fma(sm.bufV[t], sm.bufV[t], ss);
      const double nr = sqrt(block_sum(ss, sm.red));
      double al = nr;
      if (nv > 0) {
        const int e0 = extra;
        al = reorth(sm.bufV, V, nv, a.ldK, nr, mode, sm, rg, part, pstride, extra);
        rows_v += 2 * nv * (1 + extra - e0);
        ++rsteps;
      }
      if (!(al > 1e-12 * runmax) || al == 0.0) {  // breakdown: restart vector (R11)
        if (!breakdown) breakdown = mtot + 1;
        const double q = (nv < K) ? restart_vector(sm.bufV, K, a.ldK, V, nv, a.seed, (uint64_t)(b + a.series_base),
                                                   ((uint64_t)(++restarts) << 40), sm, rg, part, pstride)
                                  : 0.0;
        ss = 0.0;
        for (int t = tid; t < K; t += blockDim.x) ss = fma(sm.bufV[t], sm.bufV[t], ss);
        const double nn = sqrt(block_sum(ss, sm.red));
        normalize_store(sm.bufV, K, a.ldK, (q > 1e-8 && nn > 0.0) ? 1.0 / nn : 0.0, V + (size_t)nv * a.ldK);
        al = 0.0;
      } else {
        normalize_store(sm.bufV, K, a.ldK, 1.0 / al, V + (size_t)nv * a.ldK);
      }
      if (tid == 0) T[(nu - 1) * ldT + nv] = al;
      runmax = fmax(runmax, al);
      ++nv;
      ++mtot;
      __syncthreads();
      // ---- convergence test / thick restart on T_c = T[0:nu][0:nc], alpha_next = al ----
      const int nc = nv - 1;
      const bool last = mtot >= a.m_cap, full = nc >= d;
      if (nc >= k && (mtot >= next_check || full || last)) {
        ++checks;
        trl_jacobi(T, ldT, nu, nc, Wj, ldw, Qj, sg, ord, sm.redi);
        double mr = 0.0;
        for (int i = 0; i < k; ++i) {
          const int c = ord[i];
          const double pl = (sg[c] > 0.0) ? Wj[(size_t)c * ldw + nu - 1] / sg[c] : 0.0;
          mr = fmax(mr, fabs(al * pl));
        }
        const double om0 = sg[ord[0]];
        const double rel = (om0 > 0.0) ? mr / om0 : 0.0;
        const bool conv = rel <= 0.5 * a.tol;
        // every warp has read sg / ord / W before the next correlation overwrites region A
        if (!(conv || last || full)) __syncthreads();
        if (conv || last) {
          // final: sigma and the Ritz coefficients P_k (nu rows), Q_k (nc rows) for ritz_kernel
          double* cP = a.coef + (size_t)bl * 2 * (a.m_max + 2) * k;
          double* cQ = cP + (size_t)(a.m_max + 2) * k;
          for (int idx = tid; idx < (a.m_max + 2) * k; idx += blockDim.x) {
            const int r = idx / k, i = idx - r * k;
            const int c = ord[i];
            const double inv = (sg[c] > 0.0) ? 1.0 / sg[c] : 0.0;
            cP[idx] = (r < nu) ? Wj[(size_t)c * ldw + r] * inv : 0.0;
            cQ[idx] = (r < nc) ? Qj[(size_t)c * nc + r] : 0.0;
          }
          if (tid < k) a.sigma[(size_t)b * k + tid] = sg[ord[tid]];
          if (tid == 0) {
            ssa_series_info inf;
            inf.steps = mtot;
            inf.converged = conv ? 1 : 0;
            inf.breakdown_step = breakdown;
            inf.reorth_extra = extra;
            inf.restarts = restarts;
            inf.rows_u = rows_u;
            inf.rows_v = rows_v;
            inf.reorth_steps = rsteps;
            inf.reserved = thick;
            inf.status = rel <= a.tol ? SSA_OK : SSA_ERR_NOT_CONVERGED;
            inf.max_residual = rel;
            inf.sigma1 = om0;
            a.info[b] = inf;
            st[0] = nc; st[1] = conv ? 1 : 0; st[2] = breakdown; st[3] = extra; st[4] = restarts; st[5] = 0;
            st[6] = checks; st[7] = 1; st[8] = rows_u; st[9] = rows_v; st[10] = rsteps; st[11] = nu;
          }
          break;
        }
        int step = ce;
        if (prev_res > 0.0 && rel < prev_res && rel > 0.0) {
          const double rate = log(rel / prev_res) / (double)(mtot - prev_m);
          const double need = log(0.5 * a.tol / rel) / rate;
          const int s2 = (int)(0.7 * need);
          if (s2 > step) step = s2 < a.check_cap ? s2 : a.check_cap;
        }
        prev_res = rel;
        prev_m = mtot;
        next_check = mtot + step;
        if (full) {
          // thick restart: keep p Ritz triples and the residual direction v_next
          const int p = min(a.trl_p, nc - 1);
          for (int i = tid; i < p; i += blockDim.x) scl[i] = (sg[ord[i]] > 0.0) ? 1.0 / sg[ord[i]] : 0.0;
          __syncthreads();
          trl_restart(U, a.ldL, nu, p, Wj, ldw, ord, scl, -1);
          __syncthreads();
          for (int i = tid; i < p; i += blockDim.x) scl[i] = 1.0;
          __syncthreads();
          trl_restart(V, a.ldK, nc, p, Qj, nc, ord, scl, nc);
          fence_proxy_async_global();  // the TMA rings read the new rows next
          __syncthreads();
          for (int i = tid; i < ldT * ldT; i += blockDim.x) {
            const int r = i / ldT, c = i - r * ldT;
            T[i] = (r == c && r < p) ? sg[ord[r]] : 0.0;
          }
          nu = p;
          nv = p + 1;
          fresh = true;
          ++thick;
          __syncthreads();
        }
      }
      // ---- half-step B: p = X v_nv - T[nu-1][nv-1] u_nu; after a restart no recurrence
      // term: the CGS coefficients against the kept u~_i are the arrow column rho ----
      const double cB = fresh ? 0.0 : T[(nu - 1) * ldT + nv - 1];
      correlate_cta(
          fbuf, sh, tw, spec, K, L, [&](int i) { return sm.bufV[i]; },
          [&](int t, double y) { sm.bufU[t] = y - cB * sm.bufU[t]; });
      __syncthreads();
      ss = 0.0;
      for (int t = tid; t < L; t += blockDim.x) ss = fma(sm.bufU[t], sm.bufU[t], ss);
      const double nrb = sqrt(block_sum(ss, sm.red));
      if (fresh)
        for (int i = tid; i < nu; i += blockDim.x) hacc[i] = 0.0;
      __syncthreads();
      const int e0 = extra;
      double be = reorth(sm.bufU, U, nu, a.ldL, nrb, mode, sm, rg, part, pstride, extra, fresh ? hacc : nullptr);
      rows_u += 2 * nu * (1 + extra - e0);
      ++rsteps;
      if (fresh) {
        for (int i = tid; i < nu; i += blockDim.x) T[i * ldT + nv - 1] = hacc[i];
        fresh = false;
      }
      if (!(be > 1e-12 * runmax) || be == 0.0) {
        if (!breakdown) breakdown = mtot;
        const double q = (nu < L) ? restart_vector(sm.bufU, L, a.ldL, U, nu, a.seed, (uint64_t)(b + a.series_base),
                                                   ((uint64_t)(++restarts) << 40), sm, rg, part, pstride)
                                  : 0.0;
        ss = 0.0;
        for (int t = tid; t < L; t += blockDim.x) ss = fma(sm.bufU[t], sm.bufU[t], ss);
        const double nn = sqrt(block_sum(ss, sm.red));
        normalize_store(sm.bufU, L, a.ldL, (q > 1e-8 && nn > 0.0) ? 1.0 / nn : 0.0, U + (size_t)nu * a.ldL);
        be = 0.0;
      } else {
        normalize_store(sm.bufU, L, a.ldL, 1.0 / be, U + (size_t)nu * a.ldL);
      }
      if (tid == 0) T[nu * ldT + nv - 1] = be;
      runmax = fmax(runmax, be);
      ++nu;
      __syncthreads();
    }
  }
}

}  // namespace ssa
