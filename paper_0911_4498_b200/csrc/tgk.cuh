// tgk.cuh -- CTA-parallel singular triples of the (m+1) x m lower bidiagonal B_m of
// Golub-Kahan-Lanczos bidiagonalization through its Golub-Kahan
// tridiagonal TGK: the cyclic matrix [[0, B],[B^T, 0]] of Theorem 1
// permuted to tridiagonal form, size n = 2m+1, zero diagonal, off-diagonal
// c = (alpha_1, beta_2, alpha_2, beta_3, ..., alpha_m, beta_{m+1}).  Its eigenvalues are
// +-omega_i and 0; the eigenvector of +omega_i interleaves (p_1, q_1, p_2, ..., q_m,
// p_{m+1}) / sqrt(2) with B q = omega p, B^T p = omega q.
//
//  tgk_topk_values  k largest eigenvalues by multisection on Sturm counts (negcount of
//                   the LDL^T pivots of TGK - x I), T threads per value, to full precision.
//  tgk_check        values + last eigenvector entry by a twisted factorization: the Ritz
//                   residual alpha_{m+1} |P_{m+1,i}| of Eq. (2) that
//                   decides when Lanczos stops (R7).
//  tgk_vectors      eigenvectors by inverse iteration with a partially pivoted tridiagonal
//                   LU (LAPACK dgttrf/dgttrs style), Gram-Schmidt inside clusters of close
//                   values (|gap| <= 1e-5 |T|), one thread per cluster.
#pragma once
#include <cuda_runtime.h>

namespace ssa {

// Number of eigenvalues of TGK that are < x.  c2[i] = (i-th off-diagonal)^2, i < n-1.
__device__ __forceinline__ int tgk_negcount(const double* c2, int n, double x, double pivmin) {
  double q = -x;
  int cnt = q < 0.0;
  for (int i = 1; i < n; ++i) {
    if (fabs(q) < pivmin) q = -pivmin;
    q = -x - c2[i - 1] / q;
    cnt += q < 0.0;
  }
  return cnt;
}

// Division-free Sturm count: number of eigenvalues of TGK below x, from the sign changes
// of the characteristic-polynomial sequence p_0 = 1, p_1 = -x, p_i = -x p_{i-1} -
// c_{i-1}^2 p_{i-2} (Wilkinson), on the matrix scaled by 1/|T| (c2n = c2 / |T|^2,
// xn = x / |T|) so |p_i| grows at most like the golden ratio per step; an exact
// power-of-two rescale every 16 steps keeps the pair away from under/overflow.  Only
// one FMA per step sits on the dependency chain (the ratio form q_i = p_i / p_{i-1}
// has a division there).  A zero p_i takes the sign opposite to p_{i-1}.
__device__ __forceinline__ int tgk_negcount_poly(const double* c2n, int n, double xn) {
  double p2 = 1.0, p1 = -xn;
  int cnt = p1 < 0.0;
  int i = 1;
  // blocks of 16 steps: the 16 squared off-diagonals are loaded first so that only the
  // FMA chain is sequential (the loads of a step-by-step loop sat on it), then the exact
  // power-of-two rescale at i = 16, 32, ...
  for (; i + 16 <= n; i += 16) {
    double cv[16];
#pragma unroll
    for (int t = 0; t < 16; ++t) cv[t] = c2n[i - 1 + t];
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      double p = fma(-xn, p1, -cv[t] * p2);
      if (p == 0.0) p = -copysign(0x1.0p-900, p1);
      cnt += (p < 0.0) != (p1 < 0.0);
      p2 = p1;
      p1 = p;
    }
    const double mx = fmax(fabs(p1), fabs(p2));
    if (mx < 0x1.0p-400) { p1 *= 0x1.0p+400; p2 *= 0x1.0p+400; }
    else if (mx > 0x1.0p+400) { p1 *= 0x1.0p-400; p2 *= 0x1.0p-400; }
  }
  for (; i < n; ++i) {  // fewer than 16 steps left: no rescale point among them
    double p = fma(-xn, p1, -c2n[i - 1] * p2);
    if (p == 0.0) p = -copysign(0x1.0p-900, p1);
    cnt += (p < 0.0) != (p1 < 0.0);
    p2 = p1;
    p1 = p;
  }
  return cnt;
}

struct TgkNorms {
  double gmax;    // Gershgorin bound >= |T|
  double pivmin;  // smallest pivot magnitude allowed in the Sturm recurrence
};

__device__ __forceinline__ TgkNorms tgk_norms(const double* c, const double* c2, int n) {
  double gmax = 0.0, cmax2 = 0.0;
  for (int i = 0; i < n; ++i) {
    double l = (i > 0) ? fabs(c[i - 1]) : 0.0, r = (i < n - 1) ? fabs(c[i]) : 0.0;
    gmax = fmax(gmax, l + r);
  }
  for (int i = 0; i < n - 1; ++i) cmax2 = fmax(cmax2, c2[i]);
  TgkNorms t;
  t.gmax = gmax;
  t.pivmin = 1e-290 * fmax(1.0, cmax2);
  return t;
}

// k largest eigenvalues of TGK into lam[0..k-1] (descending).  lohi: SMEM scratch 2k.
// max_rounds multisection rounds (each shrinks the bracket T+1 fold); stops early when
// every bracket is below 2 eps of its upper end.  All threads call; ends with a barrier.
// c2n: c2 / gmax^2 (shared memory).
__device__ inline void tgk_topk_values(const double* c2n, int n, int k, const TgkNorms& nrm, double* lohi, double* lam,
                                int max_rounds, int stride = 1) {
  // value j is the (j * stride + 1)-th largest eigenvalue (stride > 1: a sparse subset)
  // T threads per value: up to 32 with warp ballots; few values (the cheap convergence
  // test) get whole warps, up to 256 threads each, counted through shared memory, so
  // every round shrinks the bracket up to 257-fold
  const int tid = threadIdx.x, nthr = blockDim.x;
  int T = 32;
  while (T > 1 && k * T > nthr) T >>= 1;
  if (T == 32)
    while (T < 256 && k * T * 2 <= nthr) T *= 2;
  __shared__ int cnt_s[8];
  const int j = tid / T, t = tid - j * T;
  const bool act = j < k;
  if (act && t == 0) { lohi[2 * j] = 0.0; lohi[2 * j + 1] = nrm.gmax * (1.0 + 1e-15) + 1e-300; }
  if (T > 32 && tid < 8) cnt_s[tid] = 0;
  __syncthreads();
  for (int round = 0; round < max_rounds; ++round) {
    double lo = act ? lohi[2 * j] : 0.0, hi = act ? lohi[2 * j + 1] : 0.0;
    int open = act && (hi - lo > 4.440892098500626e-16 * hi) && (hi - lo > nrm.pivmin);
    if (!__syncthreads_or(open)) break;
    double x = lo + (hi - lo) * (double)(t + 1) / (double)(T + 1);
    bool pred = act && (n - tgk_negcount_poly(c2n, n, x / nrm.gmax) >= j * stride + 1);
    unsigned bits = __ballot_sync(0xffffffffu, pred);
    int ts;
    if (T > 32) {  // whole warps per value: popcounts summed in shared memory
      if ((tid & 31) == 0 && act) atomicAdd(&cnt_s[j], __popc(bits));
      __syncthreads();
      ts = act ? cnt_s[j] - 1 : -1;  // monotone predicate: true for t <= ts
    } else {
      int shift = (T >= 32) ? 0 : ((tid & 31) / T) * T;
      unsigned gb = (T >= 32) ? bits : ((bits >> shift) & ((1u << T) - 1u));
      ts = __popc(gb) - 1;
    }
    __syncthreads();
    if (act && t == 0) {
      double nlo = (ts >= 0) ? lo + (hi - lo) * (double)(ts + 1) / (double)(T + 1) : lo;
      double nhi = (ts < T - 1) ? lo + (hi - lo) * (double)(ts + 2) / (double)(T + 1) : hi;
      lohi[2 * j] = nlo;
      lohi[2 * j + 1] = nhi;
      if (T > 32) cnt_s[j] = 0;
    }
    __syncthreads();
  }
  if (tid < k) lam[tid] = 0.5 * (lohi[2 * tid] + lohi[2 * tid + 1]);
  __syncthreads();
}

// Reciprocal for the convergence test's pivots: hardware approximation + one Newton step
// (~1e-12 relative; the test only needs the residual to a few digits -- the reported
// residual comes from tgk_final, which divides correctly rounded).
__device__ __forceinline__ double rcp_check(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  const double e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

// Convergence test: omega[j], res[j] (SMEM) for j < k; scratch: >= 2 k n doubles (shared
// memory when it fits, else global; layout [i][j]).  Needs 2k <= blockDim.x.
// alpha_next = alpha_{m+1}.  All threads call; ends with a barrier.
// c2n: scratch of n-1 doubles (shared memory) for the normalized squares.
__device__ inline void tgk_check(const double* c, const double* c2, double* c2n, int m, int k, double alpha_next,
                                 double* omega, double* res, double* lohi, double* scratch, int stride = 1,
                                 int kg = 32, unsigned long long* tm = nullptr) {
  const long long t_start = clock64();
  // k values (the (j * stride + 1)-th largest, j < k) and their residuals; the twisted
  // factorizations run in groups of at most kg values (scratch: 2 n kg doubles)
  const int n = 2 * m + 1;
  const int tid = threadIdx.x;
  const TgkNorms nrm = tgk_norms(c, c2, n);
  const double pivmin = nrm.pivmin;
  {
    const double ig2 = (nrm.gmax > 0.0) ? 1.0 / (nrm.gmax * nrm.gmax) : 0.0;
    for (int i = tid; i < n - 1; i += blockDim.x) c2n[i] = c2[i] * ig2;
    __syncthreads();
  }
  tgk_topk_values(c2n, n, k, nrm, lohi, omega, 16, stride);
  const long long t_vals = clock64();
  // twisted factorization for lambda = omega_j, two lanes per value: the even lane runs
  // the forward pivots D+ (and later the entries above the twist), the odd lane the
  // backward pivots D- (and the entries below).  Twist r at the smallest
  // |gamma_r| = |D+_r + D-_r + lambda|; z_r = 1, z_i = -(c_i / D+_i) z_{i+1} above,
  // -(c_{i-1} / D-_i) z_{i-1} below; result |z_n| / |z|.  Pivots are divided through a
  // correctly rounded reciprocal (one multiply more, no full division on the chain).
  if (kg < 1) kg = 1;
  for (int j0 = 0; j0 < k; j0 += kg) {
  const int nvg = (k - j0) < kg ? (k - j0) : kg;
  const unsigned pmask = __ballot_sync(0xffffffffu, tid < 2 * nvg);  // lanes taking part, per warp
  if (tid < 2 * nvg) {
    const int jl = tid >> 1, j = j0 + jl, role = tid & 1;
    const double lam = omega[j];
    double* Dp = scratch;                      // Dp[i * nvg + jl]
    double* Dm = scratch + (size_t)n * nvg;    // Dm[i * nvg + jl]
    if (role == 0) {
      double q = -lam;
      Dp[jl] = q;
      for (int i = 1; i < n; ++i) {
        if (fabs(q) < pivmin) q = -pivmin;
        q = fma(-c2[i - 1], rcp_check(q), -lam);
        Dp[(size_t)i * nvg + jl] = q;
      }
    } else {
      double q = -lam;
      Dm[(size_t)(n - 1) * nvg + jl] = q;
      for (int i = n - 2; i >= 0; --i) {
        if (fabs(q) < pivmin) q = -pivmin;
        q = fma(-c2[i], rcp_check(q), -lam);
        Dm[(size_t)i * nvg + jl] = q;
      }
    }
    __syncwarp(pmask);
    // argmin |gamma| over the two halves, then combine (lowest index on ties)
    const int h0 = role ? n / 2 : 0, h1 = role ? n : n / 2;
    double gbest = 1e308;
    int r = -1;
    for (int i = h0; i < h1; ++i) {
      const double g = fabs(Dp[(size_t)i * nvg + jl] + Dm[(size_t)i * nvg + jl] + lam);
      if (g < gbest) { gbest = g; r = i; }
    }
    const double go = __shfl_xor_sync(pmask, gbest, 1);
    const int ro = __shfl_xor_sync(pmask, r, 1);
    if (go < gbest || (go == gbest && ro >= 0 && (r < 0 || ro < r))) { gbest = go; r = ro; }
    double nrm2 = 0.0, zn = 0.0;
    if (role == 0) {  // entries above the twist
      double z = 1.0;
      for (int i = r - 1; i >= 0; --i) {
        double d = Dp[(size_t)i * nvg + jl];
        if (fabs(d) < pivmin) d = -pivmin;
        z = -(c[i] * rcp_check(d)) * z;
        nrm2 = fma(z, z, nrm2);
      }
    } else {  // entries below the twist (and the twist itself)
      double z = 1.0;
      nrm2 = 1.0;
      for (int i = r + 1; i < n; ++i) {
        double d = Dm[(size_t)i * nvg + jl];
        if (fabs(d) < pivmin) d = -pivmin;
        z = -(c[i - 1] * rcp_check(d)) * z;
        nrm2 = fma(z, z, nrm2);
      }
      zn = z;  // z_n (1 when r = n - 1)
    }
    const double tot = nrm2 + __shfl_xor_sync(pmask, nrm2, 1);
    if (role == 1) res[j] = alpha_next * 1.4142135623730951 * fabs(zn) / sqrt(tot);
  }
  __syncthreads();
  }
  if (tm && threadIdx.x == 0) {  // profiling: cycles in the values / twisted parts
    tm[0] += (unsigned long long)(t_vals - t_start);
    tm[1] += (unsigned long long)(clock64() - t_vals);
  }
}

// Clusters of the k values (descending): maximal runs with lam[j-1] - lam[j] <=
// 1e-3 |T| (LAPACK dstein's ORTOL: outside a cluster independently computed vectors are
// orthogonal to O(eps |T| / gap) <= 2e-13).  cl[0..nc] = starts (cl[nc] = k),
// cl[kClCount] = nc.  Returns 1 if some gap inside a cluster is below 1e-11 |T| or a value is
// below 1e-11 |T| (near the eigenvalue 0 that TGK of odd order always has): such
// near-degenerate values need inverse iteration with orthogonalization (tgk_vectors).
// Thread 0 only.
__device__ inline int tgk_clusters(const double* lam, int k, double tnorm, int* cl) {
  const double ortol = 1e-3 * tnorm, degen = 1e-11 * tnorm;
  int nc = 0, bad = 0;
  for (int j = 0; j < k; ++j) {
    if (j == 0 || lam[j - 1] - lam[j] > ortol) cl[nc++] = j;
    else if (lam[j - 1] - lam[j] < degen) bad = 1;
    if (!(lam[j] > degen)) bad = 1;
  }
  cl[nc] = k;
  cl[kClCount] = nc;
  return bad;
}

// Modified Gram-Schmidt (twice) of the columns j0..j1-1 of C (rows x k; element (r, j) at
// C[r * rs + j * cs]); one warp, lanes over rows.
__device__ inline void warp_mgs_cols(double* C, int rows, int rs, int cs, int j0, int j1) {
  const int lane = threadIdx.x & 31;
  for (int j = j0; j < j1; ++j) {
    for (int pass = 0; pass < 2; ++pass)
      for (int q = j0; q < j; ++q) {
        double d = 0.0;
        for (int r = lane; r < rows; r += 32) d = fma(C[(size_t)r * rs + (size_t)j * cs], C[(size_t)r * rs + (size_t)q * cs], d);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
        for (int r = lane; r < rows; r += 32)
          C[(size_t)r * rs + (size_t)j * cs] = fma(-d, C[(size_t)r * rs + (size_t)q * cs], C[(size_t)r * rs + (size_t)j * cs]);
        __syncwarp();
      }
    double s2 = 0.0;
    for (int r = lane; r < rows; r += 32) s2 = fma(C[(size_t)r * rs + (size_t)j * cs], C[(size_t)r * rs + (size_t)j * cs], s2);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    const double inv = s2 > 0.0 ? 1.0 / sqrt(s2) : 0.0;
    for (int r = lane; r < rows; r += 32) C[(size_t)r * rs + (size_t)j * cs] *= inv;
    __syncwarp();
  }
}

// Final small SVD of B_m (north star (b); Thm 1):
// the k largest eigenvalues of TGK to full precision (multisection), each eigenvector by
// ONE twisted factorization (two lanes per value, as in tgk_check: the solution of
// (TGK - lam I) z = gamma_r e_r at the twist r of smallest |gamma_r|), split into
// p (even entries, rows of P_k: cP[r * k + j], r <= m) and q (odd entries, Q_k: cQ[r * k +
// j], r < m), each half normalized, then MGS inside clusters (tgk_clusters) so P_k and
// Q_k are orthonormal to working precision.  res[j] = alpha_{m+1} |P_{m+1,j}| (Eq. (2)).
// scratch: 2 n k doubles (pivots).  Returns 0 (nothing written) when tgk_clusters finds
// near-degenerate values.  All threads call; ends with a barrier.  Needs 2k <= blockDim.x.
__device__ inline int tgk_final(const double* c, const double* c2, double* c2n, int m, int k, double alpha_next,
                                double* lam, double* lohi, double* res, double* scratch, double* cP, double* cQ,
                                int* cl, int kg = 32, double* stage = nullptr) {
  const int n = 2 * m + 1;
  const int tid = threadIdx.x;
  const TgkNorms nrm = tgk_norms(c, c2, n);
  const double pivmin = nrm.pivmin;
  {
    const double ig2 = (nrm.gmax > 0.0) ? 1.0 / (nrm.gmax * nrm.gmax) : 0.0;
    for (int i = tid; i < n - 1; i += blockDim.x) c2n[i] = c2[i] * ig2;
    __syncthreads();
  }
  tgk_topk_values(c2n, n, k, nrm, lohi, lam, 60);
  __shared__ int s_bad;
  if (tid == 0) s_bad = tgk_clusters(lam, k, nrm.gmax, cl);
  __syncthreads();
  if (s_bad) return 0;
  if (kg < 1) kg = 1;
  for (int j0 = 0; j0 < k; j0 += kg) {
  const int nvg = (k - j0) < kg ? (k - j0) : kg;
  const unsigned pmask = __ballot_sync(0xffffffffu, tid < 2 * nvg);
  if (tid < 2 * nvg) {
    const int jl = tid >> 1, j = j0 + jl, role = tid & 1;
    const double lm = lam[j];
    double* Dp = scratch;                    // Dp[i * nvg + jl]
    double* Dm = scratch + (size_t)n * nvg;  // Dm[i * nvg + jl]
    if (role == 0) {
      double q = -lm;
      Dp[jl] = q;
      for (int i = 1; i < n; ++i) {
        if (fabs(q) < pivmin) q = -pivmin;
        q = fma(-c2[i - 1], __drcp_rn(q), -lm);
        Dp[(size_t)i * nvg + jl] = q;
      }
    } else {
      double q = -lm;
      Dm[(size_t)(n - 1) * nvg + jl] = q;
      for (int i = n - 2; i >= 0; --i) {
        if (fabs(q) < pivmin) q = -pivmin;
        q = fma(-c2[i], __drcp_rn(q), -lm);
        Dm[(size_t)i * nvg + jl] = q;
      }
    }
    __syncwarp(pmask);
    const int h0 = role ? n / 2 : 0, h1 = role ? n : n / 2;
    double gbest = 1e308;
    int r = -1;
#pragma unroll 4
    for (int i = h0; i < h1; ++i) {
      const double g = fabs(Dp[(size_t)i * nvg + jl] + Dm[(size_t)i * nvg + jl] + lm);
      if (g < gbest) { gbest = g; r = i; }
    }
    const double go = __shfl_xor_sync(pmask, gbest, 1);
    const int ro = __shfl_xor_sync(pmask, r, 1);
    if (go < gbest || (go == gbest && ro >= 0 && (r < 0 || ro < r))) { gbest = go; r = ro; }
    // z_r = 1; role 0 writes the entries above the twist, role 1 the twist and below;
    // even i -> p_{i/2}, odd i -> q_{(i-1)/2}
    double sp = 0.0, sq = 0.0;
    if (role == 0) {
      double z = 1.0;
      for (int i = r - 1; i >= 0; --i) {
        double d = Dp[(size_t)i * nvg + jl];
        if (fabs(d) < pivmin) d = -pivmin;
        z = -(c[i] * __drcp_rn(d)) * z;
        if (i & 1) { cQ[(size_t)(i >> 1) * k + j] = z; sq = fma(z, z, sq); }
        else { cP[(size_t)(i >> 1) * k + j] = z; sp = fma(z, z, sp); }
      }
    } else {
      double z = 1.0;
      if (r & 1) { cQ[(size_t)(r >> 1) * k + j] = z; sq = 1.0; }
      else { cP[(size_t)(r >> 1) * k + j] = z; sp = 1.0; }
      for (int i = r + 1; i < n; ++i) {
        double d = Dm[(size_t)i * nvg + jl];
        if (fabs(d) < pivmin) d = -pivmin;
        z = -(c[i - 1] * __drcp_rn(d)) * z;
        if (i & 1) { cQ[(size_t)(i >> 1) * k + j] = z; sq = fma(z, z, sq); }
        else { cP[(size_t)(i >> 1) * k + j] = z; sp = fma(z, z, sp); }
      }
    }
    sp += __shfl_xor_sync(pmask, sp, 1);
    sq += __shfl_xor_sync(pmask, sq, 1);
    const double ip = sp > 0.0 ? 1.0 / sqrt(sp) : 0.0, iq = sq > 0.0 ? 1.0 / sqrt(sq) : 0.0;
    __syncwarp(pmask);
    // normalize the halves (each lane its own entries)
    const int i0 = role ? r : 0, i1 = role ? n : r;
    for (int i = i0; i < i1; ++i) {
      if (i & 1) cQ[(size_t)(i >> 1) * k + j] *= iq;
      else cP[(size_t)(i >> 1) * k + j] *= ip;
    }
  }
  __syncthreads();
  }
  // orthonormalize inside clusters: one warp per cluster; with `stage` (shared memory,
  // (2m+1) k doubles, free now that the pivots are done) the columns are copied in, worked
  // on there and copied back
  {
    const int nc = cl[kClCount];
    bool any = false;
    for (int q = 0; q < nc; ++q) any |= (cl[q + 1] - cl[q] > 1);
    if (any) {
      // staged copies are column-major (lanes over rows read consecutive words)
      double* P = cP;
      double* Q = cQ;
      int prs = k, pcs = 1, qrs = k, qcs = 1;
      if (stage) {
        P = stage;
        Q = stage + (size_t)(m + 1) * k;
        prs = 1; pcs = m + 1; qrs = 1; qcs = m;
        for (int i = tid; i < (m + 1) * k; i += blockDim.x) P[(i % k) * (m + 1) + i / k] = cP[i];
        for (int i = tid; i < m * k; i += blockDim.x) Q[(i % k) * m + i / k] = cQ[i];
        __syncthreads();
      }
      const int w = tid >> 5, nw = blockDim.x >> 5;
      for (int q = w; q < nc; q += nw) {
        if (cl[q + 1] - cl[q] < 2) continue;
        warp_mgs_cols(P, m + 1, prs, pcs, cl[q], cl[q + 1]);
        warp_mgs_cols(Q, m, qrs, qcs, cl[q], cl[q + 1]);
      }
      __syncthreads();
      if (stage) {
        for (int i = tid; i < (m + 1) * k; i += blockDim.x) cP[i] = P[(i % k) * (m + 1) + i / k];
        for (int i = tid; i < m * k; i += blockDim.x) cQ[i] = Q[(i % k) * m + i / k];
      }
    }
  }
  __syncthreads();
  if (tid < k) res[tid] = alpha_next * fabs(cP[(size_t)m * k + tid]);
  __syncthreads();
  return 1;
}

// splitmix64-based uniform(-1,1) for inverse-iteration start vectors.
__device__ __forceinline__ double tgk_rand(unsigned long long key, unsigned long long i) {
  unsigned long long x = key + (i + 1) * 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  x ^= x >> 31;
  return 2.0 * ((double)(x >> 11) * 0x1.0p-53) - 1.0;
}

// Eigenvectors of TGK for lam[0..k-1] (descending, from tgk_topk_values).
// Z: global, column j at Z[i * k + j] (i < n).  W: global scratch >= 5 * n * k doubles
// (LU factors of each shifted matrix), ipv: global scratch >= n * k ints.  Clusters:
// maximal runs with lam[j-1] - lam[j] <= 1e-5 |T| (outside a cluster inverse iteration
// alone keeps |z_i^T z_j| ~ eps |T| / gap <= 2e-11); one thread per cluster runs the
// members in order, orthogonalizing each iterate against the earlier members (MGS, as
// LAPACK dstein).  2 inverse-iteration steps (3 inside clusters) from a seeded random
// start; the LU recurrences carry their running values in registers so the only memory
// traffic on the dependency chain is independent loads/stores.  All threads call; ends
// with a barrier.
__device__ inline void tgk_vectors(const double* c, int n, int k, const double* lam, const TgkNorms& nrm, double* Z,
                                   double* W, int* ipv, unsigned long long seed, int* cl_start) {
  const int tid = threadIdx.x;
  const double tnorm = nrm.gmax;
  const double ortol = 1e-3 * tnorm;  // LAPACK dstein ORTOL
  if (tid == 0) {
    int nc = 0;
    for (int j = 0; j < k; ++j)
      if (j == 0 || lam[j - 1] - lam[j] > ortol) cl_start[nc++] = j;
    cl_start[nc] = k;
    cl_start[33] = nc;
  }
  __syncthreads();
  const int nclus = cl_start[33];
  if (tid < nclus) {
    const int j0 = cl_start[tid], j1 = cl_start[tid + 1];
    const double eps = 2.220446049250313e-16;
    const double pert = eps * tnorm;
    for (int j = j0; j < j1; ++j) {
      // perturb members of a cluster apart (LAPACK dstein: separate equal shifts)
      double x = lam[j];
      if (j > j0 && fabs(x - lam[j - 1]) < 10.0 * pert) x = lam[j - 1] - 10.0 * pert;
      double* __restrict__ fl = W;                      // multipliers l_i
      double* __restrict__ rd = W + (size_t)1 * n * k;  // 1 / u_ii
      double* __restrict__ u1 = W + (size_t)2 * n * k;  // first superdiagonal of U
      double* __restrict__ u2 = W + (size_t)3 * n * k;  // second superdiagonal of U
      double* __restrict__ b = W + (size_t)4 * n * k;
#define IX(i) ((size_t)(i) * k + j)
      // dgttrf of T - x I (sub/super diagonal c, diagonal -x), running d_i, du_i in registers
      double di = -x, dui = (n > 1) ? c[0] : 0.0;
      for (int i = 0; i < n - 1; ++i) {
        const double li = c[i];
        const double dn = -x;
        const double dun = (i < n - 2) ? c[i + 1] : 0.0;
        if (fabs(di) >= fabs(li)) {
          const double piv = (fabs(di) < pert) ? copysign(pert, di == 0.0 ? 1.0 : di) : di;
          const double f = li / piv;
          fl[IX(i)] = f; rd[IX(i)] = 1.0 / piv; u1[IX(i)] = dui; u2[IX(i)] = 0.0; ipv[IX(i)] = 0;
          di = dn - f * dui;
          dui = dun;
        } else {
          const double f = di / li;
          fl[IX(i)] = f; rd[IX(i)] = 1.0 / li; u1[IX(i)] = dn; u2[IX(i)] = dun; ipv[IX(i)] = 1;
          di = dui - f * dn;
          dui = -f * dun;
        }
      }
      {
        const double piv = (fabs(di) < pert) ? copysign(pert, di == 0.0 ? 1.0 : di) : di;
        rd[IX(n - 1)] = 1.0 / piv;
      }
      for (int i = 0; i < n; ++i) b[IX(i)] = tgk_rand(seed * 0x2545F4914F6CDD1Dull + (unsigned long long)j, i);
      const int iters = (j1 - j0 > 1) ? 3 : 2;
      for (int it = 0; it < iters; ++it) {
        // forward: L (with row interchanges), running b_i in a register
        double bi = b[IX(0)];
        for (int i = 0; i < n - 1; ++i) {
          const double bn = b[IX(i + 1)];
          const double f = fl[IX(i)];
          if (ipv[IX(i)] == 0) { b[IX(i)] = bi; bi = bn - f * bi; }
          else { b[IX(i)] = bn; bi = bi - f * bn; }
        }
        b[IX(n - 1)] = bi;
        // backward: U with two superdiagonals, running b_{i+1}, b_{i+2} in registers
        double x1 = bi * rd[IX(n - 1)], x2 = 0.0, bmax = fabs(x1);
        b[IX(n - 1)] = x1;
        for (int i = n - 2; i >= 0; --i) {
          const double xi = (b[IX(i)] - u1[IX(i)] * x1 - u2[IX(i)] * x2) * rd[IX(i)];
          b[IX(i)] = xi;
          bmax = fmax(bmax, fabs(xi));
          x2 = x1;
          x1 = xi;
        }
        // orthogonalize against earlier members of the cluster (their Z columns)
        for (int p = j0; p < j; ++p) {
          double s = 0.0;
          for (int i = 0; i < n; ++i) s = fma(b[IX(i)], Z[(size_t)i * k + p], s);
          for (int i = 0; i < n; ++i) b[IX(i)] = fma(-s, Z[(size_t)i * k + p], b[IX(i)]);
          bmax = 0.0;
          for (int i = 0; i < n; ++i) bmax = fmax(bmax, fabs(b[IX(i)]));
        }
        const double sc = (bmax > 0.0) ? 1.0 / bmax : 1.0;
        double s2 = 0.0;
        for (int i = 0; i < n; ++i) { const double v = b[IX(i)] * sc; s2 = fma(v, v, s2); }
        const double inv = (s2 > 0.0) ? sc / sqrt(s2) : 0.0;
        for (int i = 0; i < n; ++i) b[IX(i)] *= inv;
      }
      for (int i = 0; i < n; ++i) Z[(size_t)i * k + j] = b[IX(i)];
#undef IX
    }
  }
  __syncthreads();
}

}  // namespace ssa
