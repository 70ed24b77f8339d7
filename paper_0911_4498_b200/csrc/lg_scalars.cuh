// lg_scalars.cuh -- device-side scalars of the long-series Lanczos loop (ssa_large_lanczos.cu)
// and the per-half-step decisions that run in the last CTA of a grid-wide kernel:
//   lg_pro_tail   after the correlation (ssa_large_fft.cu lg_col_inv): |r|, the PRO omega
//                 recurrences or FRO, the reorthogonalization decision
//   lg_take_coef  the Lanczos coefficient of a half-step (Alg. 1 lines 5 / 7) and the
//                 scale 1/coef that the next half-step's column FFT applies when it reads r
//                 (normalization fused into lg_col_fwd)
// Shared by the two translation units; no host code.
#pragma once
#include "device_common.cuh"

namespace ssa {

constexpr double kLgEps = 2.220446049250313e-16;
constexpr int kLgMaxGroups = 64;  // dots partial groups (ld <= 64 * 32 * 512)

// device scalars of the long-series run (one struct, plan memory)
struct LgScalars {
  double nr;        // |r| before reorthogonalization (correlation partials)
  double nrm;       // current |r|
  double runmax;    // running max of alpha, beta
  double res;       // last convergence estimate
  double prev_res;  // previous estimate (test schedule)
  double acur;      // alpha_j (coefficient of half-step B)
  double bcur;      // beta_j  (coefficient of half-step A)
  double nr_rs;     // restart vector norm before orthogonalization
  double inv_next;  // scale of r when the next column FFT reads it (1 / coefficient, 0: zero vector)
  int j;            // current step (1-based)
  int m;            // B_m: steps so far (set by lg_check)
  int halt;         // loop ends after half-step A of this step
  int do_ro;        // this half-step reorthogonalizes
  int again;        // DGKS second pass needed
  int force;        // PRO follow-up: bit 0 the next v half-step, bit 1 the next u half-step
  int restart;      // breakdown: restart vector pending
  int stop;         // space exhausted: zero vector, stop at the next test
  int breakdown;    // first breakdown step
  int restarts;     // restarts so far
  int extra;        // DGKS second passes
  int conv;         // converged
  int next_check, prev_m;
  int rows_u, rows_v, rsteps;
  unsigned int done_grp;                // last-group counter of lg_dots
  unsigned int done_upd;                // last-CTA counter of lg_update
  unsigned int done_inv;                // last-CTA counter of lg_col_inv (correlation tail)
  unsigned int grp_done[kLgMaxGroups];  // per-group counters of lg_dots
  unsigned long long seed, series;      // start / restart vectors of this call's series
};

// Normalization fused into the column FFT: x = r * (*inv) is also written to basis row
// (*jrow - 1) and to cur (the "current vector" the next correlation's recurrence term reads).
struct LgNorm {
  const double* inv;  // &sc->inv_next
  const int* jrow;    // &sc->j (row j - 1 of either side)
  double* basis;
  double* cur;
  int ld;
};

// The decision tail of a correlation (the last CTA of lg_col_inv).
struct LgProTail {
  LgScalars* sc;
  int side;  // 0: half-step A (v side), 1: half-step B (u side)
  double* ab;
  int w;
  double* om;
  int mode;
  double eta;
  cudaGraphConditionalHandle h_fix;  // IF node of the fix-ups (DGKS second pass, restart)
  int has_ro;                        // experiment: an IF node around the reorthogonalization pass
  cudaGraphConditionalHandle h_ro;
};

__device__ __forceinline__ int lg_nb(const LgScalars* sc, int side) { return side == 0 ? sc->j - 1 : sc->j; }

// fixed-order sum of n partials by one CTA (thread-strided, shuffle tree, warps in order)
__device__ inline double cta_sum(const double* a, int n, double* red) {
  double s = 0.0;
  // loads four at a time in flight, added in index order (same sum as one at a time)
  const int step = blockDim.x;
  int i = threadIdx.x;
  for (; i + 3 * step < n; i += 4 * step) {
    const double x0 = __ldcg(a + i), x1 = __ldcg(a + i + step), x2 = __ldcg(a + i + 2 * step),
                 x3 = __ldcg(a + i + 3 * step);
    s += x0;
    s += x1;
    s += x2;
    s += x3;
  }
  for (; i < n; i += step) s += __ldcg(a + i);
  s = warp_sum(s);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  double t = 0.0;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += red[i];
  return t;
}

// The Lanczos coefficient of a half-step: |r| (or 0 at breakdown -> restart pending), into
// ab (alpha_j: side 0, beta_{j+1}: side 1) and the current-coefficient slot; the scale the
// next column FFT applies to r (a restart overrides it after its orthogonalization).
__device__ inline void lg_take_coef(LgScalars* sc, int side, double nn, double* ab, int w) {
  const int j = sc->j;
  double c = nn;
  if (!(nn > 1e-12 * sc->runmax) || nn == 0.0) {
    if (!sc->breakdown) sc->breakdown = j;
    sc->restart = 1;
    c = 0.0;
  } else {
    sc->runmax = fmax(sc->runmax, nn);
  }
  sc->nrm = nn;
  sc->inv_next = (c > 0.0) ? 1.0 / c : 0.0;
  if (side == 0) { ab[j] = c; sc->acur = c; }
  else { ab[w + j + 1] = c; sc->bcur = c; }
}

// One CTA after the correlation of a half-step: |r| from the correlation partials, then
// the reorthogonalization decision -- FRO (mode 1 / 2): whenever the basis is not empty;
// PRO (mode 3): the omega recurrences of ssa_lanczos.cu (Larsen 1998 update_nu /
// update_mu) over om[side][1..nb], against eta, plus the forced follow-up half-step.
// Without reorthogonalization the coefficient is taken here (and the fix-up IF node opened
// on a breakdown); otherwise the gated reorthogonalization kernels run and the update's
// last CTA takes it.  All threads of the CTA call it.
__device__ inline void lg_pro_tail(const double* cpart, int ncol, const LgProTail& t, double* red) {
  LgScalars* sc = t.sc;
  const int side = t.side, w = t.w;
  const double nr = sqrt(cta_sum(cpart, ncol, red));
  const int j = sc->j, nb = lg_nb(sc, side);
  double* mu = t.om;            // u side, 1-based
  double* nu = t.om + (w + 1);  // v side
  const double* alpha = t.ab;
  const double* beta = t.ab + w;
  int do_ro = (nb > 0) && !sc->stop;
  if (t.mode == 3 && do_ro) {
    const double anorm = sc->runmax;
    double mx = 0.0;
    if (side == 0) {
      const double bj = sc->bcur, rj = hypot(nr, bj);
      for (int i = 1 + threadIdx.x; i <= nb; i += blockDim.x) {
        double x = fma(alpha[i], mu[i], fma(beta[i + 1], mu[i + 1], -bj * nu[i]));
        const double d = kLgEps * (hypot(alpha[i], beta[i + 1]) + rj) + kLgEps * anorm;
        x = (x + copysign(d, x)) / nr;
        nu[i] = x;
        mx = fmax(mx, fabs(x));
      }
    } else {
      const double aj = sc->acur, rj = hypot(aj, nr);
      for (int i = 1 + threadIdx.x; i <= nb; i += blockDim.x) {
        double x = fma(alpha[i], nu[i], fma(beta[i], nu[i - 1], -aj * mu[i]));
        const double d = kLgEps * (hypot(alpha[i], beta[i]) + rj) + kLgEps * anorm;
        x = (x + copysign(d, x)) / nr;
        mu[i] = x;
        mx = fmax(mx, fabs(x));
      }
    }
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    mx = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) mx = fmax(mx, red[i]);
    const int bit = 1 << side;
    const bool forced = (sc->force & bit) != 0;
    do_ro = (mx > t.eta) || forced || !(nr > 0.0);
    __syncthreads();
    if (do_ro) {
      double* o = side == 0 ? nu : mu;
      for (int i = 1 + threadIdx.x; i <= nb; i += blockDim.x) o[i] = kLgEps;
    }
    if (threadIdx.x == 0) sc->force = (do_ro && !forced) ? (sc->force | bit) : (sc->force & ~bit);
  }
  if (threadIdx.x != 0) return;
  if (side == 0) nu[j] = 1.0;
  else mu[j + 1] = 1.0;
  sc->nr = nr;
  sc->again = 0;
  sc->restart = 0;
  sc->do_ro = do_ro;
  if (do_ro) {
    sc->rsteps += 1;
    if (side == 0) sc->rows_v += 2 * nb;
    else sc->rows_u += 2 * nb;
  } else {
    lg_take_coef(sc, side, sc->stop ? 0.0 : nr, t.ab, w);
    if (sc->stop) sc->restart = 0;
    if (sc->restart) sc->restarts += 1;
    cudaGraphSetConditional(t.h_fix, sc->restart ? 1u : 0u);
  }
  if (t.has_ro) cudaGraphSetConditional(t.h_ro, do_ro ? 1u : 0u);
}

// Last-CTA election of a grid: every CTA calls it after its global writes; returns true in
// the one CTA that finished last (its reads then see every other CTA's writes).
__device__ __forceinline__ bool last_cta(unsigned int* counter, unsigned int total, int* flag) {
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) *flag = (atomicAdd(counter, 1u) == total - 1);
  __syncthreads();
  const bool l = *flag != 0;
  if (l) __threadfence();
  return l;
}

}  // namespace ssa
