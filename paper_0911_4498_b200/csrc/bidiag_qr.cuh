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
//
// Latency: one thread runs this, so the bulge chase keeps the values it just produced in
// registers (only the untouched d[i+1], e[i+1], w[i+1] are loaded, and those loads do
// not depend on the rotation chain); a rotation costs one reciprocal square root.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

namespace ssa {

// Rotation records: index pairs and (c, s) in separate arrays.
struct RotRec {
  int2* ab;       // [cap]
  double2* cs;    // [cap]
  int cap;
  int n;
};

__host__ __device__ __forceinline__ void rec_push(RotRec* __restrict__ r, int& n, int a, int b, double c, double s) {
  if (n < r->cap) {
    r->ab[n] = make_int2(a, b);
    r->cs[n] = make_double2(c, s);
  }
  ++n;
}

// Plane rotation [c s; -s c] with c y + s z = r, -s y + c z = 0.  One reciprocal square
// root instead of a hypot + two divisions.
__host__ __device__ __forceinline__ void givens(double y, double z, double& c, double& s, double& r) {
  if (z == 0.0) { c = 1.0; s = 0.0; r = y; return; }
  double t = fma(y, y, z * z);
#ifdef __CUDA_ARCH__
  double ri = rsqrt(t);
#else
  double ri = 1.0 / sqrt(t);
#endif
  c = y * ri;
  s = z * ri;
  r = t * ri;
}

// Returns the number of QR iterations (>= 0) or -1 if maxit was exceeded.
// Inputs: alpha[1..m], beta[2..m+1] (1-based as in Alg. 1).  Outputs: d[0..m-1] (signed
// singular values), w[0..m] if TRACK, records if REC (counts in recL->n / recR->n).
template <bool TRACK, bool REC>
__host__ __device__ int bidiag_qr(int m, const double* __restrict__ alpha, const double* __restrict__ beta,
                                  double* __restrict__ d, double* __restrict__ e, double* __restrict__ w,
                                  RotRec* recL, RotRec* recR, int maxit) {
  int nL = 0, nR = 0;
  // lower (m+1) x m -> upper m x m (rows i, i+1); carry the running diagonal value
  {
    double di = alpha[1], wi = 0.0;
    for (int i = 0; i < m; ++i) {
      const double b = beta[i + 2];
      const double a1 = (i < m - 1) ? alpha[i + 2] : 0.0;
      double c, s, r;
      givens(di, b, c, s, r);
      d[i] = r;
      e[i] = s * a1;
      di = c * a1;
      if (TRACK) {
        const double wb = (i == m - 1) ? 1.0 : 0.0;  // w starts as e_{m+1}^T
        w[i] = c * wi + s * wb;
        wi = -s * wi + c * wb;
      }
      if (REC) rec_push(recL, nL, i, i + 1, c, s);
    }
    if (TRACK) w[m] = wi;
    e[m - 1] = 0.0;
  }
  double normB = 0.0;
  for (int i = 0; i < m; ++i) normB = fmax(normB, fmax(fabs(d[i]), fabs(e[i])));
  int iter = 0;
  if (normB > 0.0) {
    const double eps = 2.220446049250313e-16;
    const double zthr = eps * normB;
    const double athr = 1e-3 * eps * normB;
    int hi = m - 1;
    while (hi > 0) {
      if (iter > maxit) { iter = -1; break; }
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
            if (REC) rec_push(recL, nL, j, z, c, s);
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
            if (REC) rec_push(recR, nR, j, hi, c, s);
          }
        }
        continue;
      }
      // Wilkinson shift from the trailing 2x2 of B^T B of the block
      const double dm1 = d[hi - 1], dh = d[hi], em1 = e[hi - 1];
      const double em2 = (hi - 1 > lo) ? e[hi - 2] : 0.0;
      const double t11 = dm1 * dm1 + em2 * em2;
      const double t12 = dm1 * em1;
      const double t22 = dh * dh + em1 * em1;
      const double dl = 0.5 * (t11 - t22);
      const double den = dl + copysign(sqrt(dl * dl + t12 * t12), dl);
      const double mu = (den != 0.0) ? t22 - t12 * t12 / den : t22;
      double di = d[lo], ei = e[lo];
      double y = di * di - mu;
      double zz = di * ei;
      double wi = TRACK ? w[lo] : 0.0;
      for (int i = lo; i < hi; ++i) {
        const double di1 = d[i + 1];                       // untouched so far
        const double ei1 = (i < hi - 1) ? e[i + 1] : 0.0;  // untouched so far
        const double wi1 = TRACK ? w[i + 1] : 0.0;
        double c, s, r;
        // right rotation on columns (i, i+1)
        givens(y, zz, c, s, r);
        if (i > lo) e[i - 1] = r;
        const double ndi = c * di + s * ei;
        const double nei = -s * di + c * ei;
        const double bulge = s * di1;
        const double ndi1 = c * di1;
        if (REC) rec_push(recR, nR, i, i + 1, c, s);
        // left rotation on rows (i, i+1) to remove the bulge at (i+1, i)
        givens(ndi, bulge, c, s, r);
        d[i] = r;
        const double ne = c * nei + s * ndi1;
        di = -s * nei + c * ndi1;
        e[i] = ne;
        zz = s * ei1;
        ei = c * ei1;
        y = ne;
        if (TRACK) {
          w[i] = c * wi + s * wi1;
          wi = -s * wi + c * wi1;
        }
        if (REC) rec_push(recL, nL, i, i + 1, c, s);
      }
      d[hi] = di;
      if (TRACK) w[hi] = wi;
      ++iter;
    }
  }
  if (REC) { recL->n = nL; recR->n = nR; }
  return iter;
}

// Select the k largest |d| (stable: lower index first on ties).  sel[0..k-1], om[0..k-1].
__host__ __device__ inline void select_topk(int m, const double* d, int k, int* sel, double* om) {
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

// x <- G^T x for each recorded rotation on (a, b), in reverse record order:
//   x_a' = c x_a - s x_b,  x_b' = s x_a + c x_b.
// Applied to a unit vector this forms a column of P_acc / Q_acc.  x has stride `stride`.
// Sweeps recorded as (i, i+1), i increasing, are replayed with i decreasing, so x_a of
// one record is x_b of the next: that value is carried in a register and only x_a of the
// next record is loaded (a load that does not depend on the rotation chain).
// (Records were written earlier in the same kernel: plain loads, not the read-only path.)
__host__ __device__ inline void apply_records_reverse(const int2* ab, const double2* cs, int n, double* x,
                                                      int stride) {
  int ci = -1;  // index whose current value lives in register cv
  double cv = 0.0;
  for (int t = n - 1; t >= 0; --t) {
    const int2 p = ab[t];
    const double2 r = cs[t];
    double xa, xb;
    if (p.x == ci) xa = cv; else xa = x[p.x * stride];
    if (p.y == ci) xb = cv; else xb = x[p.y * stride];
    if (ci >= 0 && ci != p.x && ci != p.y) x[ci * stride] = cv;  // flush the carried value
    const double na = r.x * xa - r.y * xb;
    const double nb = r.y * xa + r.x * xb;
    x[p.y * stride] = nb;
    ci = p.x;
    cv = na;
  }
  if (ci >= 0) x[ci * stride] = cv;
}

}  // namespace ssa
