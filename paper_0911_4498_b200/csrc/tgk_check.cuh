// tgk_check.cuh -- CTA-parallel convergence test of Golub-Kahan-Lanczos (R7).
//
// The k largest singular values omega_j of the (m+1) x m lower bidiagonal B_m
// are the k largest eigenvalues of its Golub-Kahan tridiagonal
// TGK (the cyclic form [[0, B],[B^T, 0]] of Theorem 1, permuted to
// tridiagonal): size n = 2m+1, zero diagonal, off-diagonal (alpha_1, beta_2, alpha_2,
// beta_3, ..., alpha_m, beta_{m+1}).  They are found by multisection on Sturm counts
// (negcount of the LDL^T pivots of TGK - x I), T threads per value.  For each omega_j
// the eigenvector of TGK is formed by a twisted factorization (twist at the smallest
// |gamma_r|); its last entry is P_{m+1,j} / sqrt(2), so by Eq. (2) the
// Ritz residual is alpha_{m+1} sqrt(2) |z_n| / |z|.  This only decides when to stop; the
// reported residual comes from the final QR SVD (bidiag_qr.cuh).
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

// c2: squared off-diagonals (SMEM, n-1 entries); c: off-diagonals (SMEM).  k <= 32.
// omega[j], res[j] written for j < k (SMEM).  scratch: global, >= k * n doubles.
// alpha_next = alpha_{m+1}.  All threads of the CTA must call; ends with a barrier.
__device__ void tgk_check(const double* c, const double* c2, int m, int k, double alpha_next, double* omega,
                          double* res, double* lohi, double* scratch) {
  const int n = 2 * m + 1;
  const int tid = threadIdx.x, nthr = blockDim.x;
  // group size: largest power of two with k * T <= nthr, T <= 32
  int T = 32;
  while (T > 1 && k * T > nthr) T >>= 1;
  // Gershgorin bound and pivmin (every thread computes the same values)
  double gmax = 0.0, cmax2 = 0.0;
  for (int i = 0; i < n; ++i) {
    double l = (i > 0) ? fabs(c[i - 1]) : 0.0, r = (i < n - 1) ? fabs(c[i]) : 0.0;
    gmax = fmax(gmax, l + r);
  }
  for (int i = 0; i < n - 1; ++i) cmax2 = fmax(cmax2, c2[i]);
  const double pivmin = 1e-290 * fmax(1.0, cmax2);
  const int j = tid / T, t = tid - j * T;
  const bool act = j < k;
  if (act && t == 0) { lohi[2 * j] = 0.0; lohi[2 * j + 1] = gmax * (1.0 + 1e-15) + 1e-300; }
  __syncthreads();
  for (int round = 0; round < 16; ++round) {
    double lo = act ? lohi[2 * j] : 0.0, hi = act ? lohi[2 * j + 1] : 0.0;
    double x = lo + (hi - lo) * (double)(t + 1) / (double)(T + 1);
    bool pred = act && (n - tgk_negcount(c2, n, x, pivmin) >= j + 1);
    unsigned bits = __ballot_sync(0xffffffffu, pred);
    int shift = (T >= 32) ? 0 : ((tid & 31) / T) * T;
    unsigned gb = (T >= 32) ? bits : ((bits >> shift) & ((1u << T) - 1u));
    int ts = __popc(gb) - 1;  // monotone predicate: true for t <= ts
    __syncthreads();
    if (act && t == 0) {
      double nlo = (ts >= 0) ? lo + (hi - lo) * (double)(ts + 1) / (double)(T + 1) : lo;
      double nhi = (ts < T - 1) ? lo + (hi - lo) * (double)(ts + 2) / (double)(T + 1) : hi;
      lohi[2 * j] = nlo;
      lohi[2 * j + 1] = nhi;
    }
    __syncthreads();
  }
  // twisted factorization for lambda = omega_j, one thread per value
  if (tid < k) {
    const double lam = 0.5 * (lohi[2 * tid] + lohi[2 * tid + 1]);
    omega[tid] = lam;
    double* D = scratch;  // D[i * k + tid]
    // forward pivots D+_i of TGK - lam I
    double q = -lam;
    D[tid] = q;
    for (int i = 1; i < n; ++i) {
      if (fabs(q) < pivmin) q = -pivmin;
      q = -lam - c2[i - 1] / q;
      D[(size_t)i * k + tid] = q;
    }
    // backward pivots D-_i, gamma_i = D+_i + D-_i + lam; twist r = argmin |gamma|
    double dm = -lam;
    int r = n - 1;
    double gbest = fabs(D[(size_t)(n - 1) * k + tid] + dm + lam);
    for (int i = n - 2; i >= 0; --i) {
      if (fabs(dm) < pivmin) dm = -pivmin;
      dm = -lam - c2[i] / dm;
      double g = fabs(D[(size_t)i * k + tid] + dm + lam);
      if (g < gbest) { gbest = g; r = i; }
    }
    // recompute D-_i for i > r into D (D+ is only needed for i < r)
    dm = -lam;
    for (int i = n - 1; i > r; --i) {
      if (i < n - 1) {
        if (fabs(dm) < pivmin) dm = -pivmin;
        dm = -lam - c2[i] / dm;
      }
      D[(size_t)i * k + tid] = dm;
    }
    // z_r = 1; up: z_i = -(c_i / D+_i) z_{i+1}; down: z_i = -(c_{i-1} / D-_i) z_{i-1}
    double nrm2 = 1.0, z = 1.0;
    for (int i = r - 1; i >= 0; --i) {
      double d = D[(size_t)i * k + tid];
      if (fabs(d) < pivmin) d = -pivmin;
      z = -(c[i] / d) * z;
      nrm2 = fma(z, z, nrm2);
    }
    z = 1.0;
    for (int i = r + 1; i < n; ++i) {
      double d = D[(size_t)i * k + tid];
      if (fabs(d) < pivmin) d = -pivmin;
      z = -(c[i - 1] / d) * z;
      nrm2 = fma(z, z, nrm2);
    }
    const double zn = (r == n - 1) ? 1.0 : z;
    res[tid] = alpha_next * 1.4142135623730951 * fabs(zn) / sqrt(nrm2);
  }
  __syncthreads();
}

}  // namespace ssa
