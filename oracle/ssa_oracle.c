/*
 * ssa_oracle.c -- TEST INFRASTRUCTURE ONLY.  Plain, slow, obviously-correct CPU
 * reference for the fast Basic-SSA hot path (Korobeynikov, arXiv:0911.4498).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * leg may load this library.  It shares no code, header, table or helper with the
 * CUDA path in paper_0911_4498_b200/ and neither side includes the other.
 *
 * Everything is IEEE binary64, round-to-nearest, compiled with -ffp-contract=off so
 * that no FMA contraction changes the plain left-to-right sums written below
 * (reading R18).  No FFT, no Lanczos: only the definitions.
 *
 *  - oracle_trajectory       : the L x K trajectory (Hankel) matrix x_ij = f_{i+j-1}
 *                              PAPER.md:84-94 (sec 2.1 Embedding).
 *  - oracle_matvec           : y = X x or y = X^T x by the definition of the
 *                              matrix-vector product over explicit entries f_{i+j-1}
 *                              (the operation Alg. 2/3 compute,
 *                              PAPER.md:680-729 sec 4.3).
 *  - oracle_svd_jacobi       : singular triples of X by one-sided (Hestenes) Jacobi
 *                              on the explicit matrix (SVD as defined
 *                              sec 2.2, standard X = U Sigma V^T; R3).
 *  - oracle_diag_average     : diagonal averaging of an arbitrary L x K matrix Y,
 *                              the three-case formula of PAPER.md:155-163 (sec 2.4).
 *  - oracle_hankelize_rank1  : the same three-case formula applied to Y = sigma u v^T
 *                              with y_jl formed on the fly
 *                              (Eq. hankelization1, sec 5).
 *
 * Parity status: every function above is pinned by -m "not gpu" tests in
 * tests/test_oracle.py (SPEC/paper examples, closed forms, invariants, brute force
 * and LAPACK on tiny inputs).  Nothing here is "parity unpinned".
 *
 * Conventions: arrays are C row-major.  Indices in comments are the paper's 1-based
 * ones; code is 0-based (f[0] = f_1).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* X[i*K + j] = f_{i+j+1} (0-based i, j), i < L, j < K, K = N - L + 1.  PAPER.md:84-94. */
void oracle_trajectory(const double* f, int64_t N, int64_t L, double* X) {
  int64_t K = N - L + 1;
  for (int64_t i = 0; i < L; ++i)
    for (int64_t j = 0; j < K; ++j) X[i * K + j] = f[i + j];
}

/* transpose == 0: y (len L) = X x (x len K): y_i = sum_j x_ij x_j.
 * transpose == 1: y (len K) = X^T x (x len L): y_j = sum_i x_ij x_i.
 * x_ij = f_{i+j-1} read straight from the series (no FFT).  PAPER.md:84-94, 680-729. */
void oracle_matvec(const double* f, int64_t N, int64_t L, const double* x, double* y, int transpose) {
  int64_t K = N - L + 1;
  if (!transpose) {
    for (int64_t i = 0; i < L; ++i) {
      double s = 0.0;
      for (int64_t j = 0; j < K; ++j) s += f[i + j] * x[j];
      y[i] = s;
    }
  } else {
    for (int64_t j = 0; j < K; ++j) {
      double s = 0.0;
      for (int64_t i = 0; i < L; ++i) s += f[i + j] * x[i];
      y[j] = s;
    }
  }
}

/* g (len N = L+K-1) = diagonal averaging of Y (L x K, row-major), PAPER.md:155-163:
 *   g_k = (1/k)       sum_{j=1}^{k}      y_{j,k-j+1},  1 <= k <= L
 *   g_k = (1/L)       sum_{j=1}^{L}      y_{j,k-j+1},  L <  k <  K
 *   g_k = (1/(N-k+1)) sum_{j=k-K+1}^{L}  y_{j,k-j+1},  K <= k <= N
 * The formula is printed for L <= K ("without loss of generality");
 * for L > K the same antidiagonal mean is taken over the entries that exist, i.e. the
 * sum runs over j = max(1, k-K+1) .. min(k, L) and the divisor is that entry count
 * (reading R14).  For L <= K this is exactly the three cases above. */
void oracle_diag_average(const double* Y, int64_t L, int64_t K, double* g) {
  int64_t N = L + K - 1;
  for (int64_t k = 1; k <= N; ++k) {
    int64_t jlo = (k - K + 1 > 1) ? k - K + 1 : 1;
    int64_t jhi = (k < L) ? k : L;
    double s = 0.0;
    for (int64_t j = jlo; j <= jhi; ++j) s += Y[(j - 1) * K + (k - j)];
    g[k - 1] = s / (double)(jhi - jlo + 1);
  }
}

/* Rank-1 case Y = sigma u v^T, PAPER.md:751-760 (Eq. hankelization1): y_jl = sigma u_j v_l
 * formed entry by entry (the explicit matrix would be 137 GB at cfg5). */
void oracle_hankelize_rank1(double sigma, const double* u, int64_t L, const double* v, int64_t K, double* g) {
  int64_t N = L + K - 1;
  for (int64_t k = 1; k <= N; ++k) {
    int64_t jlo = (k - K + 1 > 1) ? k - K + 1 : 1;
    int64_t jhi = (k < L) ? k : L;
    double s = 0.0;
    for (int64_t j = jlo; j <= jhi; ++j) s += sigma * u[j - 1] * v[k - j];
    g[k - 1] = s / (double)(jhi - jlo + 1);
  }
}

/* ---------------------------------------------------------------------------------
 * One-sided (Hestenes) Jacobi SVD of the explicit trajectory matrix.
 *
 * Let n = min(L,K), m = max(L,K).  A is the m x n matrix whose n columns are
 *   L <= K : the rows of X (A = X^T, columns of length K)
 *   L >  K : the columns of X (A = X, columns of length L)
 * Cyclic-by-rows sweeps over column pairs (p < q): a = |A_p|^2, b = |A_q|^2,
 * c = A_p . A_q; rotate iff |c| > tol * sqrt(a b) with tol = 1e-15, choosing the
 * rotation that makes the two columns orthogonal (Hestenes 1958; Golub & Van Loan
 * sec 8.6.3 "one-sided Jacobi").  The same rotations are accumulated into J (n x n,
 * starts at I).  Stop after a sweep without rotation (cap 60 sweeps).  Then
 * A = W J^T with W = A J having orthogonal columns, sigma_i = |W_i|.
 *   L <= K : X^T = W J^T -> X = J Sigma (W/Sigma)^T : u_i = J_i, v_i = W_i / sigma_i
 *   L >  K : X   = W J^T                            : u_i = W_i / sigma_i, v_i = J_i
 * Ordering: sigma descending, stable (ties keep column order).  Sign: each u_i is
 * flipped so that its largest-|.| entry (lowest index on ties) is positive, v_i with it
 * (reading R12).  Pairs where one column norm is below
 * tiny = (1e-300 + (eps * |X|_F)^2) are skipped: such columns are numerically zero and
 * rotating them only stirs rounding noise (their sigma is ~0 either way).
 *
 * Outputs: sigma[nsv] (nsv <= n), U[nsv][L], V[nsv][K] (row i = i-th vector).
 * Returns the number of sweeps used (negative if the cap was hit).
 * --------------------------------------------------------------------------------- */
int oracle_svd_jacobi_capped(const double* f, int64_t N, int64_t L, int64_t nsv,
                             double* sigma, double* U, double* V, int max_sweeps) {
  int64_t K = N - L + 1;
  int transposed = (L <= K);         /* A = X^T */
  int64_t n = transposed ? L : K;    /* number of columns of A */
  int64_t m = transposed ? K : L;    /* column length */
  /* columns stored contiguously: A[c*m + r] */
  double* A = (double*)malloc(sizeof(double) * (size_t)(n * m));
  double* J = (double*)malloc(sizeof(double) * (size_t)(n * n));
  if (!A || !J) { free(A); free(J); return -1000; }
  double fro2 = 0.0;
  for (int64_t c = 0; c < n; ++c)
    for (int64_t r = 0; r < m; ++r) {
      /* L <= K: column c of A = row c of X: A[c][r] = x_{c,r} = f[c + r]
         L >  K: column c of A = column c of X: A[c][r] = x_{r,c} = f[r + c] */
      double x = f[c + r];
      A[c * m + r] = x;
      fro2 += x * x;
    }
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) J[i * n + j] = (i == j) ? 1.0 : 0.0;   /* J[col][row] */

  const double tol = 1e-15;
  const double tiny = 1e-300 + (2.220446049250313e-16 * 2.220446049250313e-16) * fro2;
  int sweep, rotated = 1;
  for (sweep = 0; sweep < max_sweeps && rotated; ++sweep) {
    rotated = 0;
    for (int64_t p = 0; p < n - 1; ++p) {
      for (int64_t q = p + 1; q < n; ++q) {
        double* x = A + p * m;
        double* y = A + q * m;
        double a = 0.0, b = 0.0, c = 0.0;
        for (int64_t r = 0; r < m; ++r) {
          a += x[r] * x[r];
          b += y[r] * y[r];
          c += x[r] * y[r];
        }
        if (a < tiny || b < tiny) continue;
        if (!(fabs(c) > tol * sqrt(a * b))) continue;
        rotated = 1;
        /* x' = cs x - sn y, y' = sn x + cs y with x'.y' = 0:
           t = sn/cs solves t^2 + 2 zeta t - 1 = 0, zeta = (b - a) / (2c); smaller root. */
        double zeta = (b - a) / (2.0 * c);
        double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        double cs = 1.0 / sqrt(1.0 + t * t);
        double sn = cs * t;
        for (int64_t r = 0; r < m; ++r) {
          double xr = x[r], yr = y[r];
          x[r] = cs * xr - sn * yr;
          y[r] = sn * xr + cs * yr;
        }
        double* jp = J + p * n;
        double* jq = J + q * n;
        for (int64_t r = 0; r < n; ++r) {
          double xr = jp[r], yr = jq[r];
          jp[r] = cs * xr - sn * yr;
          jq[r] = sn * xr + cs * yr;
        }
      }
    }
  }
  int sweeps_used = rotated ? -sweep : sweep;

  /* sigma_c = |W_c|; stable selection sort by descending sigma */
  double* s = (double*)malloc(sizeof(double) * (size_t)n);
  int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  for (int64_t c = 0; c < n; ++c) {
    double ss = 0.0;
    for (int64_t r = 0; r < m; ++r) ss += A[c * m + r] * A[c * m + r];
    s[c] = sqrt(ss);
    order[c] = c;
  }
  for (int64_t i = 1; i < n; ++i) {          /* insertion sort: stable */
    int64_t oi = order[i];
    int64_t j = i - 1;
    while (j >= 0 && s[order[j]] < s[oi]) { order[j + 1] = order[j]; --j; }
    order[j + 1] = oi;
  }
  if (nsv > n) nsv = n;
  for (int64_t i = 0; i < nsv; ++i) {
    int64_t c = order[i];
    double sg = s[c];
    sigma[i] = sg;
    double* ui = U + i * L;
    double* vi = V + i * K;
    const double* w = A + c * m;
    const double* jc = J + c * n;
    if (transposed) {   /* u = J_c (len L = n), v = W_c / sigma (len K = m) */
      for (int64_t r = 0; r < L; ++r) ui[r] = jc[r];
      for (int64_t r = 0; r < K; ++r) vi[r] = (sg > 0.0) ? w[r] / sg : 0.0;
    } else {            /* u = W_c / sigma (len L = m), v = J_c (len K = n) */
      for (int64_t r = 0; r < L; ++r) ui[r] = (sg > 0.0) ? w[r] / sg : 0.0;
      for (int64_t r = 0; r < K; ++r) vi[r] = jc[r];
    }
    /* sign canonicalization: largest-|.| entry of u positive, lowest index on ties */
    int64_t imax = 0;
    for (int64_t r = 1; r < L; ++r)
      if (fabs(ui[r]) > fabs(ui[imax])) imax = r;
    if (ui[imax] < 0.0) {
      for (int64_t r = 0; r < L; ++r) ui[r] = -ui[r];
      for (int64_t r = 0; r < K; ++r) vi[r] = -vi[r];
    }
  }
  free(s); free(order); free(A); free(J);
  return sweeps_used;
}

/* The oracle proper: sweep until no rotation (cap 60).  The capped variant exists only so
 * bench.py can time a bounded sample (a fixed number of sweeps) of the same computation. */
int oracle_svd_jacobi(const double* f, int64_t N, int64_t L, int64_t nsv,
                      double* sigma, double* U, double* V) {
  return oracle_svd_jacobi_capped(f, N, L, nsv, sigma, U, V, 60);
}
