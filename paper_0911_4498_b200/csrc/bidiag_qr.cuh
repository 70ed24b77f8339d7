// bidiag_qr.cuh -- SVD of the (m+1) x m lower bidiagonal B_m of Golub-Kahan-Lanczos
// bidiagonalization (sec 3.1), done on device by one thread.
//
// Method: implicit-shift Golub-Kahan QR sweeps (the "QR method" PAPER.md:262-265 lists;
// Golub & Van Loan sec 8.6.2) after a first sweep of left rotations that turns the
// rectangular lower bidiagonal into an m x m upper bidiagonal (its last row becomes
// zero).  Zero diagonal entries (Lanczos restarts put alpha_j = 0 into B) are removed by
// rotation chasing before shifting.  Bookkeeping keeps B_orig = P_acc B_cur Q_acc^T:
//   * a left rotation (rows a, b):  row_a' = c row_a + s row_b, row_b' = -s row_a + c row_b,
//     and P_acc gets the same column operation;
//   * a right rotation (cols a, b): col_a' = c col_a + s col_b, col_b' = -s col_a + c col_b,
//     and Q_acc gets the same column operation.
// Optionally the last row w = e_{m+1}^T P_acc is tracked (O(1) per left rotation): with
// Eq. (2) the Ritz residual of triple i is alpha_{m+1} |w_i|
// (R7/R8).  Optionally every rotation is recorded (a, b, c, s) so that selected
// columns of P_acc / Q_acc can be formed afterwards by applying the rotations in reverse
// order to unit vectors (P_acc = G_1^T G_2^T ... so P_acc e_j = G_1^T(...(G_T^T e_j))).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace ssa {

struct RotRec {       // one recorded rotation, 3 doubles: packed (a,b), c, s
  double* base;       // records: base[3*idx + {0,1,2}]
  int cap;
  int n;
  __device__ __forceinline__ void push(int a, int b, double c, double s) {
    if (n < cap) {
      base[3 * n + 0] = __longlong_as_double(((long long)a << 32) | (unsigned)b);
      base[3 * n + 1] = c;
      base[3 * n + 2] = s;
    }
    ++n;
  }
};

__device__ __forceinline__ void givens(double y, double z, double& c, double& s, double& r) {
  if (z == 0.0) { c = 1.0; s = 0.0; r = y; return; }
  if (y == 0.0) { c = 0.0; s = 1.0; r = z; return; }
  double ay = fabs(y), az = fabs(z);
  double mx = fmax(ay, az), mn = fmin(ay, az);
  double q = mn / mx;
  double rr = mx * sqrt(fma(q, q, 1.0));
  c = y / rr;
  s = z / rr;
  r = rr;
}

// Returns the number of QR iterations (>= 0) or -1 if maxit was exceeded.
// Inputs: alpha[1..m], beta[2..m+1] (1-based as in Alg. 1).  Outputs: d[0..m-1] (signed
// singular values), w[0..m] if TRACK, records if REC.  e is scratch (m entries).
template <bool TRACK, bool REC>
__device__ int bidiag_qr(int m, const double* alpha, const double* beta, double* d, double* e, double* w,
                         RotRec* recL, RotRec* recR, int maxit) {
  for (int i = 0; i < m; ++i) { d[i] = alpha[i + 1]; e[i] = 0.0; }
  if (TRACK) {
    for (int i = 0; i <= m; ++i) w[i] = 0.0;
    w[m] = 1.0;
  }
  // lower (m+1) x m -> upper m x m (rows i, i+1)
  for (int i = 0; i < m; ++i) {
    double b = beta[i + 2];
    double c, s, r;
    givens(d[i], b, c, s, r);
    d[i] = r;
    if (i < m - 1) {
      double a1 = d[i + 1];
      e[i] = s * a1;
      d[i + 1] = c * a1;
    }
    if (TRACK) {
      double wa = w[i], wb = w[i + 1];
      w[i] = c * wa + s * wb;
      w[i + 1] = -s * wa + c * wb;
    }
    if (REC) recL->push(i, i + 1, c, s);
  }
  double normB = 0.0;
  for (int i = 0; i < m; ++i) normB = fmax(normB, fmax(fabs(d[i]), fabs(e[i])));
  if (normB == 0.0) return 0;
  const double eps = 2.220446049250313e-16;
  const double zthr = eps * normB;
  const double athr = 1e-3 * eps * normB;
  int hi = m - 1, iter = 0;
  while (hi > 0) {
    if (iter > maxit) return -1;
    if (fabs(e[hi - 1]) <= fmax(eps * (fabs(d[hi - 1]) + fabs(d[hi])), athr)) {
      e[hi - 1] = 0.0;
      --hi;
      continue;
    }
    int lo = hi - 1;
    while (lo > 0 && fabs(e[lo - 1]) > fmax(eps * (fabs(d[lo - 1]) + fabs(d[lo])), athr)) --lo;
    if (lo > 0) e[lo - 1] = 0.0;
    // zero diagonal entry inside the block: chase it out
    int z = -1;
    for (int i = lo; i <= hi; ++i)
      if (fabs(d[i]) <= zthr) { z = i; break; }
    if (z >= 0) {
      ++iter;
      d[z] = 0.0;
      if (z < hi) {
        // row z has only x = e[z] at column z+1; rotate rows (j, z), j = z+1..hi
        double x = e[z];
        e[z] = 0.0;
        for (int j = z + 1; j <= hi; ++j) {
          double c, s, r;
          givens(d[j], x, c, s, r);
          d[j] = r;
          if (j < hi) { x = -s * e[j]; e[j] = c * e[j]; }
          if (TRACK) {
            double wa = w[j], wb = w[z];
            w[j] = c * wa + s * wb;
            w[z] = -s * wa + c * wb;
          }
          if (REC) recL->push(j, z, c, s);
        }
      } else {
        // column hi has only x = e[hi-1] at row hi-1; rotate cols (j, hi), j = hi-1..lo
        double x = e[hi - 1];
        e[hi - 1] = 0.0;
        for (int j = hi - 1; j >= lo; --j) {
          double c, s, r;
          givens(d[j], x, c, s, r);
          d[j] = r;
          if (j > lo) { x = -s * e[j - 1]; e[j - 1] = c * e[j - 1]; }
          if (REC) recR->push(j, hi, c, s);
        }
      }
      continue;
    }
    // Wilkinson shift from the trailing 2x2 of B^T B of the block
    double dm1 = d[hi - 1], dh = d[hi], em1 = e[hi - 1];
    double em2 = (hi - 1 > lo) ? e[hi - 2] : 0.0;
    double t11 = dm1 * dm1 + em2 * em2;
    double t12 = dm1 * em1;
    double t22 = dh * dh + em1 * em1;
    double dl = 0.5 * (t11 - t22);
    double den = dl + copysign(sqrt(dl * dl + t12 * t12), dl);
    double mu = (den != 0.0) ? t22 - t12 * t12 / den : t22;
    double y = d[lo] * d[lo] - mu;
    double zz = d[lo] * e[lo];
    for (int i = lo; i < hi; ++i) {
      double c, s, r;
      // right rotation on columns (i, i+1)
      givens(y, zz, c, s, r);
      if (i > lo) e[i - 1] = r;
      double di = d[i], ei = e[i], di1 = d[i + 1];
      double ndi = c * di + s * ei;
      double nei = -s * di + c * ei;
      double bulge = s * di1;
      double ndi1 = c * di1;
      if (REC) recR->push(i, i + 1, c, s);
      // left rotation on rows (i, i+1) to remove the bulge at (i+1, i)
      givens(ndi, bulge, c, s, r);
      d[i] = r;
      double ne = c * nei + s * ndi1;
      double nd1 = -s * nei + c * ndi1;
      e[i] = ne;
      d[i + 1] = nd1;
      if (i < hi - 1) {
        double ei1 = e[i + 1];
        zz = s * ei1;
        e[i + 1] = c * ei1;
      }
      y = ne;
      if (TRACK) {
        double wa = w[i], wb = w[i + 1];
        w[i] = c * wa + s * wb;
        w[i + 1] = -s * wa + c * wb;
      }
      if (REC) recL->push(i, i + 1, c, s);
    }
    ++iter;
  }
  return iter;
}

// Select the k largest |d| (stable: lower index first on ties).  sel[0..k-1], om[0..k-1].
__device__ inline void select_topk(int m, const double* d, int k, int* sel, double* om) {
  int cnt = 0;
  for (int i = 0; i < m; ++i) {
    double v = fabs(d[i]);
    if (cnt < k) {
      int p = cnt++;
      while (p > 0 && om[p - 1] < v) { om[p] = om[p - 1]; sel[p] = sel[p - 1]; --p; }
      om[p] = v; sel[p] = i;
    } else if (v > om[k - 1]) {
      int p = k - 1;
      while (p > 0 && om[p - 1] < v) { om[p] = om[p - 1]; sel[p] = sel[p - 1]; --p; }
      om[p] = v; sel[p] = i;
    }
  }
  for (int i = cnt; i < k; ++i) { om[i] = 0.0; sel[i] = -1; }
}

// x <- G^T x for a recorded rotation on (a, b): x_a' = c x_a - s x_b, x_b' = s x_a + c x_b.
// Applied in reverse record order to a unit vector this forms a column of P_acc / Q_acc.
// (records were written earlier in the same kernel: plain loads, not the read-only path)
__device__ inline void apply_records_reverse(const double* base, int n, double* x, int stride) {
  for (int t = n - 1; t >= 0; --t) {
    long long ab = __double_as_longlong(base[3 * t]);
    int a = (int)(ab >> 32), b = (int)(ab & 0xffffffff);
    double c = base[3 * t + 1], s = base[3 * t + 2];
    double xa = x[a * stride], xb = x[b * stride];
    x[a * stride] = c * xa - s * xb;
    x[b * stride] = s * xa + c * xb;
  }
}

}  // namespace ssa
