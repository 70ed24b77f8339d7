// ssa_large_lanczos.cu -- Golub-Kahan-Lanczos bidiagonalization with reorthogonalization for a
// series too long for one CTA (BASELINE config 3: N = 2^20, L = 2^19, k = 32), one series at
// a time with the whole GPU on it (Alg. 1; FRO PAPER.md:388-393, PRO
// PAPER.md:402-411).
//
// The whole Lanczos loop is ONE CUDA graph launch: a WHILE conditional node whose body is
// one step (half-steps A and B) of grid-wide kernels, with IF conditional nodes around the
// work that only some steps need; every decision (reorthogonalize or not, a DGKS second
// pass, a breakdown restart, the convergence test, the stop) is taken on the device, so
// ssa_decompose only enqueues (no host synchronization, include/ssa.h conventions):
//   correlation  three-pass four-step FFT (ssa_large_fft.cu) with the recurrence term
//                fused in the epilogue: r = X^T u_j - beta_j v_{j-1} (or X v_j - alpha_j u_j),
//                plus per-CTA partial sums of squares;  x and the previous vector are the
//                plan's "current vector" buffers, so every launch has fixed arguments;
//   lg_pro       one CTA: |r|, the PRO omega recurrences (or FRO: always), the decision;
//                without reorthogonalization it also takes the Lanczos coefficient;
//   IF reorth    dots (h = B^T r, per-chunk partials, the last CTA sums them in a fixed
//                order), update (r -= B h, rows in reverse so the rows the dots read last
//                hit L2), finish (norm, DGKS decision); IF again: a second pass;
//   IF restart   breakdown (coefficient < 1e-12 running max): a fresh seeded vector
//                orthogonalized twice against the basis, coefficient 0 (R11);
//   normalize    the basis row and the current-vector buffer;
//   lg_check     after half-step A, on the device-side schedule: the residual test of
//                tgk.cuh on B_m, the next test step, the stop flag;
//   IF not stop  half-step B; lg_loop sets the WHILE condition.
// Every kernel is launched with programmatic dependent launch (launch_pdl / pdl_wait) where
// the graph allows it.  After the loop the bidiagonal SVD reuses bidiag_svd_tgk_kernel and
// the Ritz vectors come from lg_ritz (grid-wide, one pass over each basis) with sign
// canonicalization.
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <vector>

#include "device_common.cuh"
#include "tgk.cuh"

namespace ssa {

cudaError_t large_spectrum(const Plan& p, const double* series, double2* spec, int items, cudaStream_t s);
cudaError_t launch_bidiag_svd(const Plan& p, const DecomposeArgs& a, cudaStream_t s);
void large_geom(const Plan& p, int* N1, int* N2);

constexpr int kLgChunk = 2048;  // elements per CTA of the start / restart vector
constexpr double kLgEps = 2.220446049250313e-16;

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
  unsigned int done_ctas;  // last-CTA counter of lg_dots
  unsigned long long seed, series;  // start / restart vectors of this call's series
};

__device__ __forceinline__ double lg_rng(uint64_t seed, uint64_t series, uint64_t i) {
  // the same counter-based generator as the batched kernel (R6)
  uint64_t x = seed ^ (series * 0xD1B54A32D192ED03ull);
  x += (i + 1) * 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  x ^= x >> 31;
  return 2.0 * ((double)(x >> 11) * 0x1.0p-53) - 1.0;
}

// Start vector (Alg. 1 line 1): r = seeded uniform(-1, 1), partial sums of squares; with
// sc != null it is a breakdown restart: salt (restarts << 40) as the batched kernel.
__global__ void __launch_bounds__(kThreads) lg_start(double* r, int n, int ld, uint64_t seed, uint64_t series,
                                                     double* part, const LgScalars* sc) {
  pdl_wait();
  __shared__ double red[kWarps];
  const uint64_t salt = sc ? ((uint64_t)sc->restarts << 40) : 0;
  if (sc) {
    seed = sc->seed;
    series = sc->series;
  }
  double ss = 0.0;
  for (int t = blockIdx.x * kLgChunk + threadIdx.x; t < (blockIdx.x + 1) * kLgChunk && t < ld; t += blockDim.x) {
    const double v = (t < n) ? lg_rng(seed, series, salt + (uint64_t)t) : 0.0;
    r[t] = v;
    ss = fma(v, v, ss);
  }
  ss = warp_sum(ss);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < kWarps; ++i) s += red[i];
    part[blockIdx.x] = s;
  }
}

// Reorthogonalization kernels: each CTA owns a kRoChunk-element chunk of r, each thread
// kRoE elements of it in registers; the basis rows stream in groups of kRoG rows with all
// kRoG x kRoE loads of a group in flight per thread (HBM-bound: bytes in flight per SM
// set the rate).  512-element chunks: ~7 CTAs per SM at L = 2^19 (an even load).  The row
// count nb is the device-side step (side 0: V_{j-1}, side 1: U_j).
constexpr int kRoChunk = 512;
constexpr int kRoE = kRoChunk / kThreads;  // 2
constexpr int kRoG = 8;                    // rows per group (warp_sum8)

__device__ __forceinline__ int lg_nb(const LgScalars* sc, int side) { return side == 0 ? sc->j - 1 : sc->j; }

// dots: part[row][cta] = <basis[row][chunk], r[chunk]>, then the last CTA to finish sums the
// partials of every row in a fixed order into h[row] (deterministic).  Rows are read with
// L2 evict_last so lg_update (rows in reverse) finds the last ones.
__global__ void __launch_bounds__(kThreads) lg_dots(const double* __restrict__ basis, int ld, int side,
                                                    const double* __restrict__ r, double* part, int nchunk,
                                                    double* h, LgScalars* sc) {
  pdl_wait();
  const int nb = lg_nb(sc, side);
  extern __shared__ double red[];  // [nb][kWarps]
  __shared__ int last;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c0 = blockIdx.x * kRoChunk + threadIdx.x;
  const bool full = (blockIdx.x + 1) * kRoChunk <= ld;
  double v[kRoE];
#pragma unroll
  for (int e = 0; e < kRoE; ++e) v[e] = (c0 + e * kThreads < ld) ? r[c0 + e * kThreads] : 0.0;
  const uint64_t pol = policy_evict_last();
  for (int row0 = 0; row0 < nb; row0 += kRoG) {
    double b[kRoG][kRoE];
#pragma unroll
    for (int q = 0; q < kRoG; ++q)
#pragma unroll
      for (int e = 0; e < kRoE; ++e) {
        const int t = c0 + e * kThreads;
        double x = 0.0;
        if (row0 + q < nb && (full || t < ld)) {
          const double* ad = basis + (size_t)(row0 + q) * ld + t;
          asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(x) : "l"(ad), "l"(pol));
        }
        b[q][e] = x;
      }
    double d[kRoG];
#pragma unroll
    for (int q = 0; q < kRoG; ++q) {
      double acc = 0.0;
#pragma unroll
      for (int e = 0; e < kRoE; ++e) acc = fma(b[q][e], v[e], acc);
      d[q] = acc;
    }
    const double tot = warp_sum8(d, lane);
    const int q = (lane >> 2) & 7;
    if ((lane & 3) == 0 && row0 + q < nb) red[(row0 + q) * kWarps + w] = tot;
  }
  __syncthreads();
  for (int row = threadIdx.x; row < nb; row += kThreads) {
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < kWarps; ++i) s += red[row * kWarps + i];
    part[(size_t)row * nchunk + blockIdx.x] = s;
  }
  // last CTA: h[row] = sum over CTAs in index order (threadfence / counter pattern)
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = (atomicAdd(&sc->done_ctas, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int row = w; row < nb; row += kWarps) {
    double s = 0.0;
    for (int i = lane; i < nchunk; i += 32) s += __ldcg(part + (size_t)row * nchunk + i);
    s = warp_sum(s);
    if (lane == 0) h[row] = s;
  }
  if (threadIdx.x == 0) sc->done_ctas = 0;
}

// update: r -= sum_row h[row] basis[row] (rows in reverse: the rows lg_dots read last
// are still in L2), partial sums of squares; groups of kRoG rows, all loads in flight.
__global__ void __launch_bounds__(kThreads) lg_update(const double* __restrict__ basis, int ld, int side,
                                                      const double* __restrict__ h, double* r, double* part,
                                                      const LgScalars* sc) {
  pdl_wait();
  const int nb = lg_nb(sc, side);
  __shared__ double red[kWarps];
  extern __shared__ double hs[];  // nb coefficients
  for (int i = threadIdx.x; i < nb; i += blockDim.x) hs[i] = h[i];
  __syncthreads();
  const int c0 = blockIdx.x * kRoChunk + threadIdx.x;
  const bool full = (blockIdx.x + 1) * kRoChunk <= ld;
  double v[kRoE];
#pragma unroll
  for (int e = 0; e < kRoE; ++e) v[e] = (c0 + e * kThreads < ld) ? r[c0 + e * kThreads] : 0.0;
  int top = nb - 1;
  if (full) {
    for (; top >= kRoG - 1; top -= kRoG) {  // whole groups: no guards, all loads in flight
      double b[kRoG][kRoE];
#pragma unroll
      for (int q = 0; q < kRoG; ++q)
#pragma unroll
        for (int e = 0; e < kRoE; ++e) b[q][e] = __ldcs(basis + (size_t)(top - q) * ld + c0 + e * kThreads);
#pragma unroll
      for (int q = 0; q < kRoG; ++q) {
        const double hr = hs[top - q];
#pragma unroll
        for (int e = 0; e < kRoE; ++e) v[e] = fma(-hr, b[q][e], v[e]);
      }
    }
  }
  for (; top >= 0; --top) {
    const double hr = hs[top];
#pragma unroll
    for (int e = 0; e < kRoE; ++e)
      if (c0 + e * kThreads < ld) v[e] = fma(-hr, __ldcs(basis + (size_t)top * ld + c0 + e * kThreads), v[e]);
  }
  double ss = 0.0;
#pragma unroll
  for (int e = 0; e < kRoE; ++e)
    if (c0 + e * kThreads < ld) {
      r[c0 + e * kThreads] = v[e];
      ss = fma(v[e], v[e], ss);
    }
  ss = warp_sum(ss);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < kWarps; ++i) t += red[i];
    part[blockIdx.x] = t;
  }
}

// fixed-order sum of n partials by one CTA (thread-strided, shuffle tree, warps in order)
__device__ double cta_sum(const double* __restrict__ a, int n, double* red) {
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += a[i];
  s = warp_sum(s);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  double t = 0.0;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += red[i];
  return t;
}

// The Lanczos coefficient of a half-step: |r| (or 0 at breakdown -> restart pending), into
// ab (alpha_j: side 0, beta_{j+1}: side 1) and the current-coefficient slot.
__device__ void lg_take_coef(LgScalars* sc, int side, double nn, double* ab, int w) {
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
  if (side == 0) { ab[j] = c; sc->acur = c; }
  else { ab[w + j + 1] = c; sc->bcur = c; }
}

// One CTA after the correlation of a half-step: |r| from the correlation partials, then
// the reorthogonalization decision -- FRO (mode 1 / 2): whenever the basis is not empty;
// PRO (mode 3): the omega recurrences of ssa_lanczos.cu (Larsen 1998 update_nu /
// update_mu) over om[side][1..nb], against eta, plus the forced follow-up half-step.
// Without reorthogonalization the coefficient is taken here.  Sets the IF handle of the
// reorthogonalization body.
__global__ void __launch_bounds__(kThreads) lg_pro(const double* __restrict__ cpart, int ncol, int side, LgScalars* sc,
                                                   double* ab, int w, double* om, int mode, double eta,
                                                   cudaGraphConditionalHandle h_ro) {
  pdl_wait();
  __shared__ double red[kWarps];
  const double nr = sqrt(cta_sum(cpart, ncol, red));
  const int j = sc->j, nb = lg_nb(sc, side);
  double* mu = om;              // u side, 1-based
  double* nu = om + (w + 1);    // v side
  const double* alpha = ab;
  const double* beta = ab + w;
  int do_ro = (nb > 0) && !sc->stop;
  if (mode == 3 && do_ro) {
    const double anorm = sc->runmax;
    double mx = 0.0;
    if (side == 0) {
      const double bj = sc->bcur, rj = hypot(nr, bj);
      for (int i = 1 + threadIdx.x; i <= nb; i += blockDim.x) {
        double t = fma(alpha[i], mu[i], fma(beta[i + 1], mu[i + 1], -bj * nu[i]));
        const double d = kLgEps * (hypot(alpha[i], beta[i + 1]) + rj) + kLgEps * anorm;
        t = (t + copysign(d, t)) / nr;
        nu[i] = t;
        mx = fmax(mx, fabs(t));
      }
    } else {
      const double aj = sc->acur, rj = hypot(aj, nr);
      for (int i = 1 + threadIdx.x; i <= nb; i += blockDim.x) {
        double t = fma(alpha[i], nu[i], fma(beta[i], nu[i - 1], -aj * mu[i]));
        const double d = kLgEps * (hypot(alpha[i], beta[i]) + rj) + kLgEps * anorm;
        t = (t + copysign(d, t)) / nr;
        mu[i] = t;
        mx = fmax(mx, fabs(t));
      }
    }
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    mx = 0.0;
    for (int i = 0; i < kWarps; ++i) mx = fmax(mx, red[i]);
    const int bit = 1 << side;
    const bool forced = (sc->force & bit) != 0;
    do_ro = (mx > eta) || forced || !(nr > 0.0);
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
    lg_take_coef(sc, side, sc->stop ? 0.0 : nr, ab, w);
    if (sc->stop) sc->restart = 0;
  }
  cudaGraphSetConditional(h_ro, do_ro ? 1u : 0u);
}

// After a reorthogonalization pass (one CTA): |r| from the update partials; pass 0 decides
// the DGKS second pass (|r| < |r_before| / sqrt 2, or always for mode 2) and sets its IF
// handle; otherwise (or after pass 1) the coefficient.
__global__ void __launch_bounds__(kThreads) lg_finish(const double* __restrict__ part, int nch, int side, LgScalars* sc,
                                                      int pass, int mode, double* ab, int w,
                                                      cudaGraphConditionalHandle h_again) {
  pdl_wait();
  __shared__ double red[kWarps];
  const double nn = sqrt(cta_sum(part, nch, red));
  if (threadIdx.x != 0) return;
  int again = 0;
  if (pass == 0) {
    again = (mode == 2 || nn < 0.70710678118654752 * sc->nr) ? 1 : 0;
    if (again) {
      sc->extra += 1;
      const int nb = lg_nb(sc, side);
      if (side == 0) sc->rows_v += 2 * nb;
      else sc->rows_u += 2 * nb;
    }
  }
  sc->again = again;
  if (!again) lg_take_coef(sc, side, nn, ab, w);
  if (pass == 0) cudaGraphSetConditional(h_again, again ? 1u : 0u);
}

// After the coefficient of a half-step: sets the IF handle of the breakdown restart.
__global__ void lg_restart_gate(LgScalars* sc, cudaGraphConditionalHandle h_rs) {
  if (threadIdx.x != 0) return;
  const int rs = sc->restart;
  if (rs) sc->restarts += 1;
  cudaGraphSetConditional(h_rs, rs ? 1u : 0u);
}

// Restart vector after its two orthogonalization passes: q = |r| / |r_0|; a vector that
// lost almost everything (q <= 1e-8) means the space is exhausted: zero vector, stop.
// The coefficient stays 0 (R11); normalize then scales by 1 / |r|.
__global__ void __launch_bounds__(kThreads) lg_restart_norm(const double* __restrict__ part, int nch,
                                                            const double* __restrict__ spart, int nst, LgScalars* sc,
                                                            int side, double* om, int w) {
  pdl_wait();
  __shared__ double red[kWarps];
  const double nn = sqrt(cta_sum(part, nch, red));
  const double n0 = sqrt(cta_sum(spart, nst, red));
  // the restart vector is orthogonal to the basis: its PRO estimates drop to eps
  double* o = side == 0 ? om + (w + 1) : om;
  const int nb = lg_nb(sc, side);
  for (int i = 1 + threadIdx.x; i <= nb; i += blockDim.x) o[i] = kLgEps;
  if (threadIdx.x != 0) return;
  const bool ok = nn > 1e-8 * n0;
  sc->nr_rs = ok ? nn : 0.0;
  if (!ok) sc->stop = 1;
}

// v = r / coef into the basis row (side 0: V row j-1, coefficient alpha_j; side 1: U row j,
// beta_{j+1}) and the current-vector buffer; after a restart the scale is 1 / |r|.
// fixed_row >= 0: the start vector u_1 (row 0, beta_1).
__global__ void __launch_bounds__(kThreads) lg_normalize(const double* __restrict__ r, int n, int ld, int side,
                                                         int fixed_row, const LgScalars* sc, const double* ab, int w,
                                                         double* basis, double* cur) {
  pdl_wait();
  int row;
  double c;
  if (fixed_row >= 0) {
    row = fixed_row;
    c = ab[w + 1];
  } else {
    const int j = sc->j;
    row = side == 0 ? j - 1 : j;
    c = side == 0 ? ab[j] : ab[w + j + 1];
    if (sc->restart) c = sc->nr_rs;
  }
  const double inv = (c > 0.0) ? 1.0 / c : 0.0;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < ld) {
    const double v = (t < n) ? r[t] * inv : 0.0;
    basis[(size_t)row * ld + t] = v;
    cur[t] = v;
  }
}

// beta_1 = |p_0| from the start vector's partials (Alg. 1 line 2)
__global__ void __launch_bounds__(kThreads) lg_beta1(const double* __restrict__ part, int n, LgScalars* sc, double* ab,
                                                     int w) {
  pdl_wait();
  __shared__ double red[kWarps];
  const double b1 = sqrt(cta_sum(part, n, red));
  if (threadIdx.x != 0) return;
  ab[w + 1] = b1;
  sc->bcur = b1;
}

__global__ void lg_init(LgScalars* sc, double* om, int w, int first_check, uint64_t seed, uint64_t series) {
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < 2 * (w + 1)) om[i] = (i == 1) ? 1.0 : 0.0;  // mu_1 = 1 (u_1)
  if (i == 0) {
    LgScalars z = {};
    z.j = 1;
    z.next_check = first_check;
    z.prev_res = -1.0;
    z.seed = seed;
    z.series = series;
    *sc = z;
  }
}

// convergence test on B_m, m = j - 1 (tgk.cuh), on the device-side schedule (R7):
// first at 2k, then every check_every steps stretched up to 2 check_every when the residual
// decays geometrically; always at m_max and after the space was exhausted.  Sets halt and
// the IF handle of half-step B.
size_t lg_check_smem(int m_max) { return (size_t)(3 * (2 * m_max + 1) + 4 * kMaxK) * 8 + 64; }

__global__ void __launch_bounds__(kThreads) lg_check(const double* __restrict__ ab, int w, int k, int m_max,
                                                     int ce, double tol, double* scratch, LgScalars* sc,
                                                     cudaGraphConditionalHandle h_b) {
  pdl_wait();
  const int m = sc->j - 1;
  const bool due = m >= k && (m >= sc->next_check || m >= m_max || sc->stop);
  if (due) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double* c = reinterpret_cast<double*>(smem_raw);
    const int n = 2 * m + 1;
    double* c2 = c + n;
    double* c2n = c2 + n;
    double* om = c2n + n;
    double* res = om + kMaxK;
    double* lohi = res + kMaxK;
    for (int i = threadIdx.x; i < n - 1; i += blockDim.x) {
      double v = (i & 1) ? ab[w + (i >> 1) + 2] : ab[(i >> 1) + 1];
      c[i] = v;
      c2[i] = v * v;
    }
    __syncthreads();
    tgk_check(c, c2, c2n, m, k, ab[m + 1], om, res, lohi, scratch);
    if (threadIdx.x == 0) {
      double mr = 0.0;
      for (int i = 0; i < k; ++i) mr = fmax(mr, res[i]);
      const double rel = (om[0] > 0.0) ? mr / om[0] : 0.0;
      sc->res = rel;
      sc->conv = (rel <= 0.5 * tol) ? 1 : 0;
      int step = ce;
      if (sc->prev_res > 0.0 && rel < sc->prev_res && rel > 0.0) {
        const double rate = log(rel / sc->prev_res) / (double)(m - sc->prev_m);
        const double need = log(0.5 * tol / rel) / rate;
        const int s2 = (int)(0.7 * need);
        if (s2 > step) step = s2 < 2 * ce ? s2 : 2 * ce;
      }
      sc->prev_res = rel;
      sc->prev_m = m;
      sc->next_check = m + step;
    }
  }
  if (threadIdx.x != 0) return;
  sc->m = m;
  const int halt = (due && (sc->conv || sc->stop)) || m >= m_max;
  sc->halt = halt;
  cudaGraphSetConditional(h_b, halt ? 0u : 1u);
}

// end of a step: j advances unless the loop stops; the WHILE condition
__global__ void lg_loop(LgScalars* sc, cudaGraphConditionalHandle h_while) {
  if (threadIdx.x != 0) return;
  const int go = !sc->halt;
  if (go) sc->j += 1;
  cudaGraphSetConditional(h_while, go ? 1u : 0u);
}

// Ritz vectors: out[i][t] = sum_row coef[row][i] basis[row][t], one element per thread
// (U_k = U_{m+1} P_k, V_k = V_m Q_k, Eq. (1)), triples in blocks of
// kRitzK (blockIdx.y).  The coefficient rows are staged through a fixed shared-memory tile
// of kRitzRows rows (zero-padded to kRitzK per row, read as broadcast 16-byte loads), so
// the kernel's shared memory does not depend on the step count m.
constexpr int kRitzRows = 128;
constexpr int kRitzK = 32;

__global__ void __launch_bounds__(kThreads) lg_ritz(const double* __restrict__ basis, int ld, int add_rows,
                                                    const int* __restrict__ state, const double* __restrict__ coef,
                                                    int k, int n, double* out, double* amax, int* aidx) {
  pdl_wait();
  const int rows = state[0] + add_rows;  // U_{m+1} (add 1) or V_m (add 0); m from the device
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int i0 = blockIdx.y * kRitzK, ki = min(kRitzK, k - i0);
  __shared__ __align__(16) double cs[kRitzRows * kRitzK];
  double acc[kRitzK];
#pragma unroll
  for (int i = 0; i < kRitzK; ++i) acc[i] = 0.0;
  for (int r0 = 0; r0 < rows; r0 += kRitzRows) {
    const int nr = min(kRitzRows, rows - r0);
    __syncthreads();
    for (int e = threadIdx.x; e < nr * kRitzK; e += blockDim.x) {
      const int r = e / kRitzK, i = e - r * kRitzK;
      cs[e] = (i < ki) ? __ldg(coef + (size_t)(r0 + r) * k + i0 + i) : 0.0;
    }
    __syncthreads();
    if (t < n) {
      for (int row = 0; row < nr; ++row) {
        const double x = __ldcs(basis + (size_t)(r0 + row) * ld + t);
        const double2* cr = reinterpret_cast<const double2*>(cs + (size_t)row * kRitzK);
#pragma unroll
        for (int i = 0; i < kRitzK / 2; ++i) {
          const double2 c = cr[i];
          acc[2 * i] = fma(c.x, x, acc[2 * i]);
          acc[2 * i + 1] = fma(c.y, x, acc[2 * i + 1]);
        }
      }
    }
  }
  if (t < n) {
#pragma unroll
    for (int i = 0; i < kRitzK; ++i)
      if (i < ki) out[(size_t)(i0 + i) * n + t] = acc[i];
  }
  if (amax) {
    // per-CTA argmax |out_i| (lowest index on ties) for sign canonicalization
    __shared__ double sv[kWarps][kRitzK];
    __shared__ int si[kWarps][kRitzK];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
    for (int i = 0; i < kRitzK; ++i) {
      if (i >= ki) break;
      double v = (t < n) ? fabs(acc[i]) : -1.0;
      int ix = t;
      for (int o = 16; o > 0; o >>= 1) {
        double v2 = __shfl_xor_sync(0xffffffffu, v, o);
        int i2 = __shfl_xor_sync(0xffffffffu, ix, o);
        if (v2 > v || (v2 == v && i2 < ix)) { v = v2; ix = i2; }
      }
      if (lane == 0) { sv[w][i] = v; si[w][i] = ix; }
    }
    __syncthreads();
    if (threadIdx.x < ki) {
      double v = -1.0;
      int ix = 0x7fffffff;
      for (int q = 0; q < kWarps; ++q)
        if (sv[q][threadIdx.x] > v || (sv[q][threadIdx.x] == v && si[q][threadIdx.x] < ix)) {
          v = sv[q][threadIdx.x];
          ix = si[q][threadIdx.x];
        }
      amax[(size_t)blockIdx.x * k + i0 + threadIdx.x] = v;
      aidx[(size_t)blockIdx.x * k + i0 + threadIdx.x] = ix;
    }
  }
}

__global__ void lg_sign(const double* __restrict__ amax, const int* __restrict__ aidx, int nblk, int k,
                        const double* __restrict__ U, int L, double* sgn) {
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= k) return;
  double v = -1.0;
  int ix = 0x7fffffff;
  for (int b = 0; b < nblk; ++b) {
    const double v2 = amax[(size_t)b * k + i];
    const int i2 = aidx[(size_t)b * k + i];
    if (v2 > v || (v2 == v && i2 < ix)) { v = v2; ix = i2; }
  }
  sgn[i] = (ix < L && U[(size_t)i * L + ix] < 0.0) ? -1.0 : 1.0;
}

__global__ void lg_flip(double* X, int n, int k, const double* __restrict__ sgn) {
  pdl_wait();
  const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (size_t)n * k) return;
  const int i = (int)(idx / n);
  if (sgn[i] < 0.0) X[idx] = -X[idx];
}

__global__ void lg_finite(const double* __restrict__ f, int N, int* state) {
  pdl_wait();
  int bad = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) bad |= !isfinite(f[i]);
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(state + 5, 1);
}


cudaError_t large_lanczos_set_attributes(int m_max) {
  cudaError_t e = raise_smem_limit(lg_check, (int)lg_check_smem(m_max));
  if (e == cudaSuccess) e = raise_smem_limit(lg_dots, (size_t)(m_max + 2) * kWarps * 8);
  if (e == cudaSuccess) e = raise_smem_limit(lg_update, (size_t)(m_max + 2) * 8);
  return e;
}

__global__ void lg_state(const LgScalars* sc, int* state) {
  pdl_wait();
  if (threadIdx.x != 0) return;
  state[0] = sc->m;
  state[1] = sc->conv;
  state[2] = sc->breakdown;
  state[3] = sc->extra;
  state[4] = sc->restarts;
  state[6] = 0;
  state[8] = sc->rows_u;
  state[9] = sc->rows_v;
  state[10] = sc->rsteps;
}

// ---- graph construction (stream capture into conditional-node bodies) -----------------
static cudaError_t cond_handle(cudaStream_t s, cudaGraphConditionalHandle* h) {
  cudaStreamCaptureStatus st;
  cudaGraph_t g = nullptr;
  cudaError_t e = cudaStreamGetCaptureInfo(s, &st, nullptr, &g, nullptr, nullptr);
  if (e != cudaSuccess) return e;
  return cudaGraphConditionalHandleCreate(h, g, 0, cudaGraphCondAssignDefault);
}

// Appends an IF node on handle h at the capture position of s and captures its body with
// body(si) on stream si.
template <class F>
static cudaError_t cond_if(cudaStream_t s, cudaGraphConditionalHandle h, cudaStream_t si, F&& body) {
  cudaStreamCaptureStatus st;
  cudaGraph_t g = nullptr;
  const cudaGraphNode_t* deps = nullptr;
  size_t nd = 0;
  cudaError_t e = cudaStreamGetCaptureInfo(s, &st, nullptr, &g, &deps, &nd);
  if (e != cudaSuccess) return e;
  cudaGraphNodeParams prm = {};
  prm.type = cudaGraphNodeTypeConditional;
  prm.conditional.handle = h;
  prm.conditional.type = cudaGraphCondTypeIf;
  prm.conditional.size = 1;
  cudaGraphNode_t node;
  if ((e = cudaGraphAddNode(&node, g, deps, nd, &prm)) != cudaSuccess) return e;
  if ((e = cudaStreamUpdateCaptureDependencies(s, &node, 1, cudaStreamSetCaptureDependencies)) != cudaSuccess) return e;
  cudaGraph_t bg = prm.conditional.phGraph_out[0];
  if ((e = cudaStreamBeginCaptureToGraph(si, bg, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed)) != cudaSuccess)
    return e;
  const cudaError_t eb = body(si);
  cudaGraph_t out = nullptr;
  e = cudaStreamEndCapture(si, &out);
  return eb != cudaSuccess ? eb : e;
}

// The Lanczos loop as a graph: WHILE(step) with the IF bodies described at the top.
static cudaError_t build_lanczos_graph(Plan& p) {
  const int L = (int)p.L, K = (int)p.K, k = p.k;
  const int ldL = p.ldL, ldK = p.ldK;
  int N1, N2;
  large_geom(p, &N1, &N2);
  const int ncol = N2 / 8;  // partial sums written by lg_col_inv (one per 8-column CTA)
  const int w = p.m_max + 3;
  double* ab = p.d_ab;
  LgScalars* sc = reinterpret_cast<LgScalars*>(p.d_lgsc);
  double* part = p.d_lgpart;
  const size_t nchmax = (size_t)(std::max(ldL, ldK) + kRoChunk - 1) / kRoChunk;
  double* cpart = part + nchmax * (p.m_max + 2);
  double* spart = cpart + 1024;
  double* h = p.d_lgh;
  double* r = p.d_lgr;
  const int mode = p.opt.reorth;
  const double eta = p.opt.reorth_eta;
  const size_t dots_smem = (size_t)(p.m_max + 2) * kWarps * 8, upd_smem = (size_t)(p.m_max + 2) * 8;
  const int ce = p.opt.check_every > 0 ? p.opt.check_every : 4;
  cudaStream_t cs[4] = {};
  cudaError_t e = cudaSuccess;
  for (int i = 0; i < 4 && e == cudaSuccess; ++i) e = cudaStreamCreateWithFlags(&cs[i], cudaStreamNonBlocking);
  cudaGraph_t g0 = nullptr;
  if (e == cudaSuccess) e = cudaGraphCreate(&g0, 0);
  cudaGraphConditionalHandle hw;
  if (e == cudaSuccess) e = cudaGraphConditionalHandleCreate(&hw, g0, 1, cudaGraphCondAssignDefault);
  cudaGraphNodeParams wp = {};
  wp.type = cudaGraphNodeTypeConditional;
  wp.conditional.handle = hw;
  wp.conditional.type = cudaGraphCondTypeWhile;
  wp.conditional.size = 1;
  cudaGraphNode_t wnode;
  if (e == cudaSuccess) e = cudaGraphAddNode(&wnode, g0, nullptr, 0, &wp);

  // reorthogonalization pass against the side's basis (CGS: dots, then update)
  auto ro_pass = [&](cudaStream_t s, int side) {
    const double* basis = side == 0 ? p.d_V : p.d_U;
    const int ld = side == 0 ? ldK : ldL;
    const int nch = (ld + kRoChunk - 1) / kRoChunk;
    launch_pdl(lg_dots, dim3(nch), dim3(kThreads), dots_smem, s, basis, ld, side, r, part, nch, h, sc);
    launch_pdl(lg_update, dim3(nch), dim3(kThreads), upd_smem, s, basis, ld, side, h, r, part, sc);
    return nch;
  };
  // one half-step on stream s (nested bodies on s1, s2)
  auto half = [&](cudaStream_t s, int side, cudaStream_t s1, cudaStream_t s2) -> cudaError_t {
    const bool A = side == 0;
    double* cur = A ? p.d_vcur : p.d_ucur;
    double* basis = A ? p.d_V : p.d_U;
    const int n = A ? K : L, ld = A ? ldK : ldL, nch = (ld + kRoChunk - 1) / kRoChunk;
    cudaError_t err = large_correlate(p, p.d_spec, 0, A ? p.d_ucur : p.d_vcur, 0, A ? L : K, r, 0, n, ld,
                                      A ? p.d_vcur : p.d_ucur, 0,
                                      A ? &sc->bcur : &sc->acur, cpart, 1, s, nullptr);
    if (err != cudaSuccess) return err;
    cudaGraphConditionalHandle hro, hrs;
    if ((err = cond_handle(s, &hro)) != cudaSuccess) return err;
    launch_pdl(lg_pro, dim3(1), dim3(kThreads), 0, s, cpart, ncol, side, sc, ab, w, p.d_lgom, mode, eta, hro);
    err = cond_if(s, hro, s1, [&](cudaStream_t sb) -> cudaError_t {
      ro_pass(sb, side);
      cudaGraphConditionalHandle hag;
      cudaError_t e2 = cond_handle(sb, &hag);
      if (e2 != cudaSuccess) return e2;
      launch_pdl(lg_finish, dim3(1), dim3(kThreads), 0, sb, part, nch, side, sc, 0, mode, ab, w, hag);
      return cond_if(sb, hag, s2, [&](cudaStream_t sc2) -> cudaError_t {
        ro_pass(sc2, side);
        launch_pdl(lg_finish, dim3(1), dim3(kThreads), 0, sc2, part, nch, side, sc, 1, mode, ab, w, hag);
        return cudaGetLastError();
      });
    });
    if (err != cudaSuccess) return err;
    if ((err = cond_handle(s, &hrs)) != cudaSuccess) return err;
    lg_restart_gate<<<1, 32, 0, s>>>(sc, hrs);
    err = cond_if(s, hrs, s1, [&](cudaStream_t sb) -> cudaError_t {
      const int nst = (ld + kLgChunk - 1) / kLgChunk;
      launch_pdl(lg_start, dim3(nst), dim3(kThreads), 0, sb, r, n, ld, (uint64_t)0, (uint64_t)0, spart,
                 (const LgScalars*)sc);
      ro_pass(sb, side);
      ro_pass(sb, side);
      launch_pdl(lg_restart_norm, dim3(1), dim3(kThreads), 0, sb, part, nch, spart, nst, sc, side, p.d_lgom, w);
      return cudaGetLastError();
    });
    if (err != cudaSuccess) return err;
    launch_pdl(lg_normalize, dim3((ld + kThreads - 1) / kThreads), dim3(kThreads), 0, s, r, n, ld, side, -1,
               (const LgScalars*)sc, (const double*)ab, w, basis, cur);
    return cudaGetLastError();
  };

  cudaGraph_t body = wp.conditional.phGraph_out[0];
  if (e == cudaSuccess) e = cudaStreamBeginCaptureToGraph(cs[0], body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed);
  if (e == cudaSuccess) {
    cudaError_t eb = half(cs[0], 0, cs[1], cs[2]);
    cudaGraphConditionalHandle hb;
    if (eb == cudaSuccess) eb = cond_handle(cs[0], &hb);
    if (eb == cudaSuccess) {
      launch_pdl(lg_check, dim3(1), dim3(kThreads), lg_check_smem(p.m_max), cs[0], (const double*)ab, w, k, p.m_max,
                 ce, p.opt.tol, p.d_tgk, sc, hb);
      eb = cond_if(cs[0], hb, cs[1], [&](cudaStream_t sb) { return half(sb, 1, cs[2], cs[3]); });
    }
    if (eb == cudaSuccess) {
      lg_loop<<<1, 32, 0, cs[0]>>>(sc, hw);
      eb = cudaGetLastError();
    }
    cudaGraph_t out = nullptr;
    e = cudaStreamEndCapture(cs[0], &out);
    if (eb != cudaSuccess) e = eb;
  }
  if (e == cudaSuccess) e = cudaGraphInstantiate(&p.lg_exec, g0, 0);
  if (e == cudaSuccess) p.lg_graph = g0;
  else if (g0) cudaGraphDestroy(g0);
  for (int i = 0; i < 4; ++i)
    if (cs[i]) cudaStreamDestroy(cs[i]);
  return e;
}

cudaError_t large_graph_build(Plan& p) {
  if (p.lg_exec) return cudaSuccess;
  const bool nopdl = getenv("SSA_LG_NOPDL") != nullptr;  // diagnostics: build without PDL
  pdl_enabled() = !nopdl;
  cudaError_t e = build_lanczos_graph(p);
  p.lg_pdl = !nopdl;
  if (e != cudaSuccess && !nopdl) {
    // some drivers reject programmatic edges inside conditional bodies: rebuild without PDL
    cudaGetLastError();
    pdl_enabled() = false;
    e = build_lanczos_graph(p);
    p.lg_pdl = false;
  }
  pdl_enabled() = true;
  if (getenv("SSA_DEBUG")) fprintf(stderr, "[ssa] long-series loop graph: %s, PDL %s\n", cudaGetErrorString(e),
                                   p.lg_pdl ? "on" : "off");
  return e;
}

// One long series b of the call: decompose into sigma/U/V (+info).  Everything is enqueued
// on s (the loop is one graph launch); nothing waits for the device.
cudaError_t large_decompose_one(Plan& p, const DecomposeArgs& a0, int b, cudaStream_t s) {
  DecomposeArgs a = a0;
  a.b0 = b;
  a.nb = 1;
  const int L = (int)p.L, K = (int)p.K, N = (int)p.N, k = p.k;
  const int ldL = p.ldL, ldK = p.ldK;
  const int nchL = (ldL + kLgChunk - 1) / kLgChunk;
  double* U = p.d_U;
  double* V = p.d_V;
  const int w = p.m_max + 3;
  LgScalars* sc = reinterpret_cast<LgScalars*>(p.d_lgsc);
  double* part = p.d_lgpart;
  const size_t nchmax = (size_t)(std::max(ldL, ldK) + kRoChunk - 1) / kRoChunk;
  double* cpart = part + nchmax * (p.m_max + 2);
  double* spart = cpart + 1024;
  double* h = p.d_lgh;
  double* r = p.d_lgr;
  cudaError_t e;
  if ((e = large_graph_build(p))) return e;
  if ((e = cudaMemsetAsync(p.d_state, 0, kStateInts * sizeof(int), s))) return e;
  launch_pdl(lg_finite, dim3(64), dim3(kThreads), 0, s, a.series + (size_t)b * N, N, p.d_state);
  if ((e = large_spectrum(p, a.series + (size_t)b * N, p.d_spec, 1, s))) return e;
  const uint64_t series = (uint64_t)(b + a.series_base);
  const int first_check = (2 * k < p.m_max) ? 2 * k : k;
  launch_pdl(lg_init, dim3((2 * (w + 1) + kThreads - 1) / kThreads), dim3(kThreads), 0, s, sc, p.d_lgom, w, first_check,
             a.seed, series);
  if ((e = cudaMemsetAsync(p.d_ab, 0, 2 * (size_t)w * 8, s))) return e;
  if ((e = cudaMemsetAsync(p.d_vcur, 0, (size_t)ldK * 8, s))) return e;
  // Alg. 1 lines 1-2: beta_1 = |p0|, u_1 = p0 / beta_1 (row 0 of U and the current u)
  launch_pdl(lg_start, dim3(nchL), dim3(kThreads), 0, s, r, L, ldL, a.seed, series, spart, (const LgScalars*)nullptr);
  launch_pdl(lg_beta1, dim3(1), dim3(kThreads), 0, s, (const double*)spart, nchL, sc, p.d_ab, w);
  launch_pdl(lg_normalize, dim3((ldL + kThreads - 1) / kThreads), dim3(kThreads), 0, s, (const double*)r, L, ldL, 1, 0,
             (const LgScalars*)sc, (const double*)p.d_ab, w, U, p.d_ucur);
  if ((e = cudaGraphLaunch(p.lg_exec, s))) return e;
  launch_pdl(lg_state, dim3(1), dim3(32), 0, s, (const LgScalars*)sc, p.d_state);
  // ---- bidiagonal SVD (reuses the batched kernel with one series) ----
  if ((e = cudaMemsetAsync(p.d_counters, 0, 4 * sizeof(int), s))) return e;
  if ((e = launch_bidiag_svd(p, a, s))) return e;
  // ---- Ritz vectors + sign canonicalization ----
  const int mstride = p.m_max + 2;
  const double* cP = p.d_coef;
  const double* cQ = p.d_coef + (size_t)mstride * k;
  double* Uo = a.Uout + (size_t)b * k * L;
  double* Vo = a.Vout + (size_t)b * k * K;
  const int gU = (L + kThreads - 1) / kThreads, gV = (K + kThreads - 1) / kThreads;
  double* amax = p.d_lgpart;
  int* aidx = reinterpret_cast<int*>(p.d_lgpart + (size_t)gU * k);
  // the Ritz kernel reads the step count m from the state word the SVD kernel used
  const int kb = (k + kRitzK - 1) / kRitzK;
  launch_pdl(lg_ritz, dim3(gU, kb), dim3(kThreads), 0, s, (const double*)U, ldL, 1, (const int*)p.d_state, cP, k, L,
             Uo, amax, aidx);
  launch_pdl(lg_ritz, dim3(gV, kb), dim3(kThreads), 0, s, (const double*)V, ldK, 0, (const int*)p.d_state, cQ, k, K,
             Vo, (double*)nullptr, (int*)nullptr);
  launch_pdl(lg_sign, dim3((k + 31) / 32), dim3(32), 0, s, (const double*)amax, (const int*)aidx, gU, k, (const double*)Uo, L, h);
  launch_pdl(lg_flip, dim3((int)(((size_t)L * k + kThreads - 1) / kThreads)), dim3(kThreads), 0, s, Uo, L, k,
             (const double*)h);
  launch_pdl(lg_flip, dim3((int)(((size_t)K * k + kThreads - 1) / kThreads)), dim3(kThreads), 0, s, Vo, K, k,
             (const double*)h);
  return cudaGetLastError();
}

}  // namespace ssa
