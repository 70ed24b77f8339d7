// ssa_large_lanczos.cu -- Golub-Kahan-Lanczos bidiagonalization with reorthogonalization for a
// series too long for one CTA (BASELINE config 3: N = 2^20, L = 2^19, k = 32), one series at
// a time with the whole GPU on it (Alg. 1; FRO PAPER.md:388-393, PRO
// PAPER.md:402-411).
//
// The whole Lanczos loop is ONE CUDA graph launch: a WHILE conditional node whose body is
// one step (half-steps A and B) of grid-wide kernels; every decision (reorthogonalize or
// not, a DGKS second pass, a breakdown restart, the convergence test, the stop) is taken
// on the device, so ssa_decompose only enqueues (no host synchronization, include/ssa.h
// conventions).  A half-step:
//   correlation  three-pass four-step FFT (ssa_large_fft.cu).  The column FFT reads the
//                previous half-step's unnormalized vector r, scales it by 1/coefficient
//                and stores it to its basis row and "current vector" buffer (the
//                normalization of Alg. 1 lines 5 / 7); the epilogue subtracts the
//                recurrence term, r = X^T u_j - beta_j v_{j-1} (or X v_j - alpha_j u_j),
//                with per-CTA partial sums of squares, and its last CTA takes |r| and the
//                reorthogonalization decision: the PRO omega recurrences or FRO
//                (lg_pro_tail, lg_scalars.cuh); without reorthogonalization it also takes
//                the Lanczos coefficient.  Every launch has fixed arguments;
//   reorth       gated on the decision (a gated-off kernel returns at once; cheaper than
//                an IF node when the pass runs on most half-steps): dots (h = B^T r,
//                per-chunk partials summed in a fixed two-level order by the last CTAs),
//                update (r -= B h, rows in reverse so the rows the dots read last hit L2;
//                its last CTA takes the norm, the DGKS decision and the coefficient);
//   IF fix-up    rare: the DGKS second pass and / or a breakdown restart (coefficient
//                < 1e-12 running max: a fresh seeded vector orthogonalized twice against
//                the basis, coefficient 0, R11), its handle set by whichever
//                tail took the decision.
// After half-step A the convergence test lg_check (tgk.cuh residuals of B_m on the
// device-side schedule, the halt flag) runs on a parallel branch of the graph, concurrent
// with half-step B, which therefore runs once more than needed on the last step (its
// results unused); lg_loop (after both) advances j unless halted and sets the WHILE
// condition.
// Every kernel is launched with programmatic dependent launch (launch_pdl / pdl_wait) where
// the graph allows it.  After the loop the bidiagonal SVD reuses bidiag_svd_tgk_kernel and
// the Ritz vectors come from lg_ritz (grid-wide, one pass over each basis) with sign
// canonicalization.
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <type_traits>
#include <vector>

#include "device_common.cuh"
#include "tgk.cuh"
#include "lg_scalars.cuh"

namespace ssa {

cudaError_t trace_attach_fft(unsigned long long* p);
cudaError_t large_correlate_lanczos(const Plan& p, const double2* spec, const double* r, int n_in, const LgNorm& nrm,
                                    double* out, int n_out, int ld_out, const double* prev, const double* coef,
                                    double* part, const LgProTail& tail, cudaStream_t s,
                                    const double* dbasis = nullptr, int dld = 0, double* dpart = nullptr,
                                    double* dh = nullptr);
int large_fused_dots_rows(long long H);
cudaError_t large_spectrum(const Plan& p, const double* series, double2* spec, int items, cudaStream_t s);
cudaError_t launch_bidiag_svd(const Plan& p, const DecomposeArgs& a, cudaStream_t s);
void large_geom(const Plan& p, int* N1, int* N2);

constexpr int kLgChunk = 2048;  // elements per CTA of the start / restart vector

__device__ __forceinline__ double lg_rng(uint64_t seed, uint64_t series, uint64_t i) {
  // the same counter-based generator as the batched kernel (R6)
  uint64_t x = seed ^ (series * 0xD1B54A32D192ED03ull);
  x += (i + 1) * 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  x ^= x >> 31;
  return 2.0 * ((double)(x >> 11) * 0x1.0p-53) - 1.0;
}

// Device-side gates of the kernels of a half-step (no IF node around them): 0 the
// reorthogonalization pass (do_ro), 1 the DGKS second pass (again), 2 the breakdown
// restart (restart).  A gated-off launch returns at once.
__device__ __forceinline__ bool lg_open(const LgScalars* sc, int gate) {
  return gate == 0 ? sc->do_ro != 0 : gate == 1 ? sc->again != 0 : sc->restart != 0;
}

// Start vector (Alg. 1 line 1): r = seeded uniform(-1, 1), partial sums of squares; with
// sc != null it is a breakdown restart (gate 2): salt (restarts << 40) as the batched kernel.
__global__ void __launch_bounds__(kThreads) lg_start(double* r, int n, int ld, uint64_t seed, uint64_t series,
                                                     double* part, const LgScalars* sc) {
  pdl_wait(10);
  if (sc && !lg_open(sc, 2)) return;
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

// dots: part[row][cta] = <basis[row][chunk], r[chunk]>, then a two-level fixed-order sum
// (deterministic): the last CTA of each group of kDotGroup CTAs sums its group's partials
// of every row (one thread per row, all kDotGroup loads in flight) into gpart[row][group];
// the last group to finish sums the groups into h[row].  Rows are read with L2
// evict_last so lg_update (rows in reverse) finds the last ones.
constexpr int kDotGroup = 32;

__global__ void __launch_bounds__(kThreads) lg_dots(const double* __restrict__ basis, int ld, int side,
                                                    const double* __restrict__ r, double* part, double* gpart,
                                                    int nchunk, double* h, LgScalars* sc, int gate) {
  pdl_wait(6);
  if (!lg_open(sc, gate)) return;
  const int nb = lg_nb(sc, side);
  extern __shared__ double red[];  // [nb][kWarps]
  __shared__ int lastf;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c0 = blockIdx.x * kRoChunk + threadIdx.x;
  const bool full = (blockIdx.x + 1) * kRoChunk <= ld;
  double v[kRoE];
#pragma unroll
  for (int e = 0; e < kRoE; ++e) v[e] = (c0 + e * kThreads < ld) ? r[c0 + e * kThreads] : 0.0;
  const uint64_t pol = policy_evict_last();
  auto group = [&](int row0, auto guarded) {
    double b[kRoG][kRoE];
#pragma unroll
    for (int q = 0; q < kRoG; ++q)
#pragma unroll
      for (int e = 0; e < kRoE; ++e) {
        const int t = c0 + e * kThreads;
        double x = 0.0;
        if (!decltype(guarded)::value || (row0 + q < nb && (full || t < ld))) {
          const double* ad = basis + (size_t)(row0 + q) * ld + t;
          // not volatile: the compiler may issue all kRoG x kRoE loads before the FMAs
          asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(x) : "l"(ad), "l"(pol));
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
  };
  int row0 = 0;
  if (full)  // whole groups of a whole chunk: no guards, all 16 loads in flight
    for (; row0 + kRoG <= nb; row0 += kRoG) group(row0, std::false_type());
  for (; row0 < nb; row0 += kRoG) group(row0, std::true_type());
  __syncthreads();
  if (blockIdx.x == 0) trace_point_any(22);
  for (int row = threadIdx.x; row < nb; row += kThreads) {
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < kWarps; ++i) s += red[row * kWarps + i];
    part[(size_t)row * nchunk + blockIdx.x] = s;
  }
  // level 1: the last CTA of this group sums the group's partials, one thread per row
  const int g = blockIdx.x / kDotGroup, ng = (nchunk + kDotGroup - 1) / kDotGroup;
  const int g0 = g * kDotGroup, gn = min(kDotGroup, nchunk - g0);
  if (!last_cta(&sc->grp_done[g], (unsigned)gn, &lastf)) return;
  if (g == 0) trace_point_any(23);
  for (int row = threadIdx.x; row < nb; row += kThreads) {
    const double* pr = part + (size_t)row * nchunk + g0;
    double s = 0.0;
    for (int i0 = 0; i0 < gn; i0 += 16) {  // 16 loads in flight, summed in index order
      double x[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) x[i] = (i0 + i < gn) ? __ldcg(pr + i0 + i) : 0.0;
#pragma unroll
      for (int i = 0; i < 16; ++i) s += x[i];
    }
    gpart[(size_t)row * kLgMaxGroups + g] = s;
  }
  if (threadIdx.x == 0) sc->grp_done[g] = 0;
  // level 2: the last group sums the groups in index order
  if (!last_cta(&sc->done_grp, (unsigned)ng, &lastf)) return;
  trace_point_any(24);
  for (int row = threadIdx.x; row < nb; row += kThreads) {
    const double* pr = gpart + (size_t)row * kLgMaxGroups;
    double s = 0.0;
    for (int i0 = 0; i0 < ng; i0 += 16) {
      double x[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) x[i] = (i0 + i < ng) ? __ldcg(pr + i0 + i) : 0.0;
#pragma unroll
      for (int i = 0; i < 16; ++i) s += x[i];
    }
    h[row] = s;
  }
  if (threadIdx.x == 0) sc->done_grp = 0;
}

// update: r -= sum_row h[row] basis[row] (rows in reverse: the rows lg_dots read last
// are still in L2), partial sums of squares; groups of kRoG rows, all loads in flight.
// The last CTA then finishes the pass: |r| from the partials; pass 0 decides the DGKS
// second pass (|r| < |r_before| / sqrt 2, or always for mode 2) and sets its IF handle;
// otherwise (or after pass 1) it takes the Lanczos coefficient (lg_take_coef).
__global__ void __launch_bounds__(kThreads) lg_update(const double* __restrict__ basis, int ld, int side,
                                                      const double* __restrict__ h, double* r, double* part,
                                                      LgScalars* sc, int pass, int gate, int mode, double* ab,
                                                      int w, cudaGraphConditionalHandle h_fix) {
  pdl_wait(7);
  if (!lg_open(sc, gate)) return;
  const int nb = lg_nb(sc, side);
  __shared__ double red[kWarps];
  __shared__ int lastf;
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
  if (blockIdx.x == 0) trace_point_any(25);
  if (pass < 0) return;  // restart passes: lg_restart_norm finishes them
  if (!last_cta(&sc->done_upd, gridDim.x, &lastf)) return;
  trace_point_any(26);
  const double nn = sqrt(cta_sum(part, gridDim.x, red));
  if (threadIdx.x != 0) return;
  sc->done_upd = 0;
  int again = 0;
  if (pass == 0) {
    again = (mode == 2 || nn < 0.70710678118654752 * sc->nr) ? 1 : 0;
    if (again) {
      sc->extra += 1;
      if (side == 0) sc->rows_v += 2 * nb;
      else sc->rows_u += 2 * nb;
    }
  }
  sc->again = again;
  if (pass == 0) {
    // the fix-up IF node of this half-step: a DGKS second pass or a breakdown restart
    if (!again) lg_take_coef(sc, side, nn, ab, w);
    if (!again && sc->restart) sc->restarts += 1;
    cudaGraphSetConditional(h_fix, (again || sc->restart) ? 1u : 0u);
  } else {
    lg_take_coef(sc, side, nn, ab, w);  // inside the fix-up body: its restart kernels follow
    if (sc->restart) sc->restarts += 1;
  }
}

// Restart vector after its two orthogonalization passes: q = |r| / |r_0|; a vector that
// lost almost everything (q <= 1e-8) means the space is exhausted: zero vector, stop.
// The coefficient stays 0 (R11); normalize then scales by 1 / |r|.
__global__ void __launch_bounds__(kThreads) lg_restart_norm(const double* __restrict__ part, int nch,
                                                            const double* __restrict__ spart, int nst, LgScalars* sc,
                                                            int side, double* om, int w) {
  pdl_wait(11);
  if (!lg_open(sc, 2)) return;
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
  sc->inv_next = ok ? 1.0 / nn : 0.0;
  if (!ok) sc->stop = 1;
}

// beta_1 = |p_0| from the start vector's partials (Alg. 1 line 2)
__global__ void __launch_bounds__(kThreads) lg_beta1(const double* __restrict__ part, int n, LgScalars* sc, double* ab,
                                                     int w) {
  pdl_wait(16);
  __shared__ double red[kWarps];
  const double b1 = sqrt(cta_sum(part, n, red));
  if (threadIdx.x != 0) return;
  ab[w + 1] = b1;
  sc->bcur = b1;
  sc->inv_next = 1.0 / b1;  // u_1 = p_0 / beta_1, applied by the first column FFT
}

__global__ void lg_init(LgScalars* sc, double* om, int w, int first_check, uint64_t seed, uint64_t series) {
  pdl_wait(17);
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
// decays geometrically; always at m_max and after the space was exhausted.  Sets halt (read
// by lg_loop).  It runs concurrently with half-step B of the same step (a graph fork): B
// does not wait for the test, and its results are simply unused when the loop halts.
size_t lg_check_smem(int m_max) { return (size_t)(3 * (2 * m_max + 1) + 4 * kMaxK) * 8 + 64; }

__global__ void __launch_bounds__(kThreads) lg_check(const double* __restrict__ ab, int w, int k, int m_max,
                                                     int ce, double tol, double* scratch, LgScalars* sc) {
  pdl_wait(13);
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
}

// end of a step: j advances unless the loop stops; the WHILE condition
__global__ void lg_loop(LgScalars* sc, cudaGraphConditionalHandle h_while) {
  trace_point(14);
  if (threadIdx.x != 0) return;
  const int go = !sc->halt;
  if (go) sc->j += 1;
  cudaGraphSetConditional(h_while, go ? 1u : 0u);
}

// Ritz vectors: out[i][t] = sum_row coef[row][i] basis[row][t] (U_k = U_{m+1} P_k,
// V_k = V_m Q_k, Eq. (1)), triples in blocks of 32 (blockIdx.y).  A dense
// contraction of arithmetic intensity 2 * 32 / 8 = 8 flop per basis byte (above the fp64
// ridge), so it runs on the fp64 tensor cores: mma.sync m8n8k4 f64 (DMMA), M = triples,
// N = elements, K = basis rows.  Each warp owns 8 kRmNt consecutive elements and all 32
// triples (4 x kRmNt accumulator tiles); per k-step of 4 rows a lane loads its kRmNt basis
// values (row 4 ks + (lane & 3), element 8 j + (lane >> 2): 64-byte row segments) and reads
// its four A fragments from a shared tile of the coefficients stored in fragment order
// ([k-step][M tile][lane]: conflict-free), staged kRitzRows rows at a time (shared memory
// independent of m).
constexpr int kRitzRows = 128;
constexpr int kRitzK = 32;
constexpr int kRmNt = 4;                     // 8-element N tiles per warp
constexpr int kRmU = 4;                      // k-steps per load group (16 loads in flight)
constexpr int kRitzSpan = kWarps * 8 * kRmNt;  // elements per CTA (256)

__global__ void __launch_bounds__(kThreads, 2) lg_ritz(const double* __restrict__ basis, int ld, int add_rows,
                                                       const int* __restrict__ state, const double* __restrict__ coef,
                                                       int k, int n, double* out, double* amax, int* aidx) {
  pdl_wait(15);
  const int rows = state[0] + add_rows;  // U_{m+1} (add 1) or V_m (add 0); m from the device
  const int i0 = blockIdx.y * kRitzK, ki = min(kRitzK, k - i0);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
  const int tw0 = blockIdx.x * kRitzSpan + w * 8 * kRmNt;  // the warp's first element
  __shared__ __align__(16) double cf[kRitzRows / 4][4][32];  // [k-step][M tile][lane]
  double acc[4][kRmNt][2];
#pragma unroll
  for (int mt = 0; mt < 4; ++mt)
#pragma unroll
    for (int j = 0; j < kRmNt; ++j) acc[mt][j][0] = acc[mt][j][1] = 0.0;
  for (int r0 = 0; r0 < rows; r0 += kRitzRows) {
    const int nr = min(kRitzRows, rows - r0), nks = (nr + 3) >> 2;
    __syncthreads();
    for (int e = threadIdx.x; e < nks * 128; e += kThreads) {
      const int ks = e >> 7, mt = (e >> 5) & 3, l = e & 31;
      const int r = 4 * ks + (l & 3), i = 8 * mt + (l >> 2);
      cf[ks][mt][l] = (r < nr && i < ki) ? __ldg(coef + (size_t)(r0 + r) * k + i0 + i) : 0.0;
    }
    __syncthreads();
    // kRmU k-steps per group: all kRmU kRmNt basis loads issued, then the MMAs
    for (int ks0 = 0; ks0 < nks; ks0 += kRmU) {
      double b[kRmU][kRmNt];
#pragma unroll
      for (int u = 0; u < kRmU; ++u) {
        const int r = r0 + 4 * (ks0 + u) + q;
        const double* bp = basis + (size_t)r * ld + tw0 + g;
#pragma unroll
        for (int j = 0; j < kRmNt; ++j)
          b[u][j] = (ks0 + u < nks && r < rows && tw0 + 8 * j + g < n) ? ldg_stream(bp + 8 * j) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < kRmU; ++u) {
        const int ks = ks0 + u < nks ? ks0 + u : nks - 1;  // beyond nks: zero B, any A
        double a[4];
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) a[mt] = cf[ks][mt][lane];
#pragma unroll
        for (int mt = 0; mt < 4; ++mt)
#pragma unroll
          for (int j = 0; j < kRmNt; ++j) dmma_m8n8k4(acc[mt][j][0], acc[mt][j][1], a[mt], b[u][j]);
      }
    }
  }
  // D fragment: triple 8 mt + g, elements tw0 + 8 j + 2 q + {0, 1}
#pragma unroll
  for (int mt = 0; mt < 4; ++mt) {
    const int i = 8 * mt + g;
    if (i < ki) {
      double* o = out + (size_t)(i0 + i) * n;
#pragma unroll
      for (int j = 0; j < kRmNt; ++j) {
        const int t = tw0 + 8 * j + 2 * q;
        if (t + 1 < n && ((reinterpret_cast<uintptr_t>(o + t) & 15) == 0)) {
          *reinterpret_cast<double2*>(o + t) = make_double2(acc[mt][j][0], acc[mt][j][1]);
        } else {
          if (t < n) o[t] = acc[mt][j][0];
          if (t + 1 < n) o[t + 1] = acc[mt][j][1];
        }
      }
    }
  }
  if (amax) {
    // per-CTA argmax |out_i| (lowest index on ties) for sign canonicalization
    __shared__ double sv[kWarps][kRitzK];
    __shared__ int si[kWarps][kRitzK];
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) {
      double v = -1.0;
      int ix = 0x7fffffff;
#pragma unroll
      for (int j = 0; j < kRmNt; ++j)  // increasing t: ties keep the lower index
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int t = tw0 + 8 * j + 2 * q + c;
          const double av = (t < n) ? fabs(acc[mt][j][c]) : -1.0;
          if (av > v) { v = av; ix = t; }
        }
      for (int o = 1; o < 4; o <<= 1) {  // the four lanes of triple 8 mt + g
        const double v2 = __shfl_xor_sync(0xffffffffu, v, o);
        const int i2 = __shfl_xor_sync(0xffffffffu, ix, o);
        if (v2 > v || (v2 == v && i2 < ix)) { v = v2; ix = i2; }
      }
      if (q == 0) { sv[w][8 * mt + g] = v; si[w][8 * mt + g] = ix; }
    }
    __syncthreads();
    if (threadIdx.x < ki) {
      double v = -1.0;
      int ix = 0x7fffffff;
      for (int qq = 0; qq < kWarps; ++qq)
        if (sv[qq][threadIdx.x] > v || (sv[qq][threadIdx.x] == v && si[qq][threadIdx.x] < ix)) {
          v = sv[qq][threadIdx.x];
          ix = si[qq][threadIdx.x];
        }
      amax[(size_t)blockIdx.x * k + i0 + threadIdx.x] = v;
      aidx[(size_t)blockIdx.x * k + i0 + threadIdx.x] = ix;
    }
  }
}

// sign of each Ritz pair from the largest-|.| entry of u_i (lowest index on ties): one warp
// per triple over the per-CTA candidates of lg_ritz
__global__ void lg_sign(const double* __restrict__ amax, const int* __restrict__ aidx, int nblk, int k,
                        const double* __restrict__ U, int L, double* sgn) {
  pdl_wait(18);
  const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (i >= k) return;
  double v = -1.0;
  int ix = 0x7fffffff;
  for (int b = lane; b < nblk; b += 32) {
    const double v2 = amax[(size_t)b * k + i];
    const int i2 = aidx[(size_t)b * k + i];
    if (v2 > v || (v2 == v && i2 < ix)) { v = v2; ix = i2; }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double v2 = __shfl_xor_sync(0xffffffffu, v, o);
    const int i2 = __shfl_xor_sync(0xffffffffu, ix, o);
    if (v2 > v || (v2 == v && i2 < ix)) { v = v2; ix = i2; }
  }
  if (lane == 0) sgn[i] = (ix < L && U[(size_t)i * L + ix] < 0.0) ? -1.0 : 1.0;
}

__global__ void lg_flip(double* X, int n, int k, const double* __restrict__ sgn) {
  pdl_wait(19);
  const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (size_t)n * k) return;
  const int i = (int)(idx / n);
  if (sgn[i] < 0.0) X[idx] = -X[idx];
}

__global__ void lg_finite(const double* __restrict__ f, int N, int* state) {
  pdl_wait(20);
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
  pdl_wait(21);
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
  double* gpart = spart + 1024;
  double* h = p.d_lgh;
  double* r = p.d_lgr;
  const int mode = p.opt.reorth;
  const double eta = p.opt.reorth_eta;
  const size_t dots_smem = (size_t)(p.m_max + 2) * kWarps * 8, upd_smem = (size_t)(p.m_max + 2) * 8;
  const int ce = p.opt.check_every > 0 ? p.opt.check_every : 4;
  const int exp_bits = getenv("SSA_LG_EXP") ? atoi(getenv("SSA_LG_EXP")) : 0;  // graph-shape experiments
  // fused first-pass dots (FRO / CGS2 only: PRO skips passes), when the column kernel's
  // buffer holds the per-warp sums of every basis row (m_max + 1 rows)
  const bool fuse_dots = (mode == 1 || mode == 2) && !getenv("SSA_LG_NOFUSE") &&
                         p.m_max + 2 <= large_fused_dots_rows((long long)p.H);
  cudaStream_t cs[5] = {};
  cudaEvent_t ev[2] = {};
  cudaError_t e = cudaSuccess;
  for (int i = 0; i < 5 && e == cudaSuccess; ++i) e = cudaStreamCreateWithFlags(&cs[i], cudaStreamNonBlocking);
  for (int i = 0; i < 2 && e == cudaSuccess; ++i) e = cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming);
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

  // reorthogonalization pass against the side's basis (CGS: dots, then update; the last
  // CTA of the update finishes the pass, pass < 0: restart passes, no finish), gated on
  // the device (lg_open)
  auto ro_pass = [&](cudaStream_t s, int side, int pass, int gate, cudaGraphConditionalHandle hfx) {
    const double* basis = side == 0 ? p.d_V : p.d_U;
    const int ld = side == 0 ? ldK : ldL;
    const int nch = (ld + kRoChunk - 1) / kRoChunk;
    if (exp_bits & 1) {  // experiment: the dots pass without a programmatic dependency
      lg_dots<<<nch, kThreads, dots_smem, s>>>(basis, ld, side, (const double*)r, part, gpart, nch, h, sc, gate);
    } else {
      launch_pdl(lg_dots, dim3(nch), dim3(kThreads), dots_smem, s, basis, ld, side, (const double*)r, part, gpart, nch,
                 h, sc, gate);
    }
    launch_pdl(lg_update, dim3(nch), dim3(kThreads), upd_smem, s, basis, ld, side, (const double*)h, r, part, sc, pass,
               gate, mode, ab, w, hfx);
    return nch;
  };
  // one half-step on stream s (the fix-up body on s1): the column FFT first normalizes
  // the previous half-step's vector (r * inv_next -> basis row j - 1 and the current
  // vector of that side); the correlation's last CTA takes the reorthogonalization
  // decision (lg_pro_tail); the reorthogonalization pass runs gated on it; one IF node
  // holds the rare fix-ups (DGKS second pass, breakdown restart), its handle set by
  // whichever tail took the decision.
  auto half = [&](cudaStream_t s, int side, cudaStream_t s1, cudaStream_t s2) -> cudaError_t {
    const bool A = side == 0;
    const int n = A ? K : L, ld = A ? ldK : ldL, nch = (ld + kRoChunk - 1) / kRoChunk;
    cudaGraphConditionalHandle hfx;
    cudaError_t err = cond_handle(s, &hfx);
    if (err != cudaSuccess) return err;
    // input: the other side's vector (u_j for A, v_j for B), normalized on the fly
    LgNorm nrm{&sc->inv_next, &sc->j, A ? p.d_U : p.d_V, A ? p.d_ucur : p.d_vcur, A ? ldL : ldK};
    LgProTail tail{sc, side, ab, w, p.d_lgom, mode, eta, hfx, 0, 0};
    cudaGraphConditionalHandle hro = 0;
    if (exp_bits & 2) {
      if ((err = cond_handle(s, &hro)) != cudaSuccess) return err;
      tail.has_ro = 1;
      tail.h_ro = hro;
    }
    // FRO / CGS2 (every half-step reorthogonalizes): the first CGS pass's dots are fused
    // into the correlation's last kernel (lg_col_inv: each CTA's outputs against every
    // basis row, no grid-wide wait on r), so only the update kernel follows
    const bool fuse = fuse_dots && !(exp_bits & 2);
    err = large_correlate_lanczos(p, p.d_spec, r, A ? L : K, nrm, r, n, ld, A ? p.d_vcur : p.d_ucur,
                                  A ? &sc->bcur : &sc->acur, cpart, tail, s, fuse ? (A ? p.d_V : p.d_U) : nullptr,
                                  ld, part, h);
    if (err != cudaSuccess) return err;
    if (exp_bits & 2) {
      err = cond_if(s, hro, s2, [&](cudaStream_t sb) -> cudaError_t {
        ro_pass(sb, side, 0, 0, hfx);
        return cudaGetLastError();
      });
      if (err != cudaSuccess) return err;
    } else if (fuse) {
      launch_pdl(lg_update, dim3(nch), dim3(kThreads), upd_smem, s, (A ? (const double*)p.d_V : (const double*)p.d_U),
                 ld, side, (const double*)h, r, part, sc, 0, 0, mode, ab, w, hfx);
    } else {
      ro_pass(s, side, 0, 0, hfx);
    }
    return cond_if(s, hfx, s1, [&](cudaStream_t sb) -> cudaError_t {
      ro_pass(sb, side, 1, 1, hfx);  // DGKS second pass (gate: again)
      const int nst = (ld + kLgChunk - 1) / kLgChunk;
      launch_pdl(lg_start, dim3(nst), dim3(kThreads), 0, sb, r, n, ld, (uint64_t)0, (uint64_t)0, spart,
                 (const LgScalars*)sc);
      ro_pass(sb, side, -1, 2, hfx);  // restart vector, orthogonalized twice (gate: restart)
      ro_pass(sb, side, -1, 2, hfx);
      launch_pdl(lg_restart_norm, dim3(1), dim3(kThreads), 0, sb, (const double*)part, nch, (const double*)spart, nst,
                 sc, side, p.d_lgom, w);
      return cudaGetLastError();
    });
  };

  cudaGraph_t body = wp.conditional.phGraph_out[0];
  if (e == cudaSuccess) e = cudaStreamBeginCaptureToGraph(cs[0], body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed);
  if (e == cudaSuccess) {
    cudaError_t eb = half(cs[0], 0, cs[1], cs[2]);
    // fork: the convergence test on B_m (one CTA, cs[4]) runs beside half-step B (the rest
    // of the GPU); join before lg_loop
    if (eb == cudaSuccess) eb = cudaEventRecord(ev[0], cs[0]);
    if (eb == cudaSuccess) eb = cudaStreamWaitEvent(cs[4], ev[0], 0);
    if (eb == cudaSuccess) {
      lg_check<<<1, kThreads, lg_check_smem(p.m_max), cs[4]>>>((const double*)ab, w, k, p.m_max, ce, p.opt.tol,
                                                              p.d_tgk, sc);
      eb = cudaGetLastError();
    }
    if (eb == cudaSuccess) eb = cudaEventRecord(ev[1], cs[4]);
    if (eb == cudaSuccess) eb = half(cs[0], 1, cs[1], cs[2]);
    if (eb == cudaSuccess) eb = cudaStreamWaitEvent(cs[0], ev[1], 0);
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
  for (int i = 0; i < 5; ++i)
    if (cs[i]) cudaStreamDestroy(cs[i]);
  for (int i = 0; i < 2; ++i)
    if (ev[i]) cudaEventDestroy(ev[i]);
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

// SSA_TRACE diagnostics (trace_point in device_common.cuh): a device buffer of kTraceMax
// records, and a report on stderr of the time from each traced kernel's start to the next
// traced start, summed per kernel id (this synchronizes the stream: diagnostics only).
static unsigned long long* trace_buffer() {
  static unsigned long long* buf = nullptr;
  if (!getenv("SSA_TRACE")) return nullptr;
  if (!buf && cudaMalloc(&buf, (size_t)(2 * kTraceMax + 1) * 8) != cudaSuccess) buf = nullptr;
  return buf;
}

static void trace_report(unsigned long long* trace, cudaStream_t s) {
  static const char* names[32] = {"?", "lg_col_fwd", "lg_row_cta", "lg_row_warp", "lg_col_inv", "-", "lg_dots",
                                  "lg_update", "-", "-", "lg_start", "lg_restart_norm",
                                  "-", "lg_check", "lg_loop", "lg_ritz", "lg_beta1", "lg_init", "lg_sign",
                                  "lg_flip", "lg_finite", "lg_state", "dots_streamed", "dots_tail1", "dots_tail2",
                                  "upd_streamed", "upd_tail"};
  cudaStreamSynchronize(s);
  unsigned long long n = 0;
  cudaMemcpy(&n, trace, 8, cudaMemcpyDeviceToHost);
  n = std::min<unsigned long long>(n, kTraceMax);
  std::vector<unsigned long long> rec(2 * n);
  cudaMemcpy(rec.data(), trace + 1, 2 * n * 8, cudaMemcpyDeviceToHost);
  trace_attach(nullptr);
  trace_attach_fft(nullptr);
  std::vector<std::pair<unsigned long long, int>> ev(n);
  for (size_t i = 0; i < n; ++i) ev[i] = {rec[2 * i], (int)rec[2 * i + 1]};
  std::sort(ev.begin(), ev.end());
  double tot[32] = {0};
  int cnt[32] = {0};
  for (size_t i = 0; i + 1 < n; ++i) {
    const int id = ev[i].second & 31;
    tot[id] += 1e-3 * (double)(ev[i + 1].first - ev[i].first);
    cnt[id] += 1;
  }
  const double span = n > 1 ? 1e-3 * (double)(ev[n - 1].first - ev[0].first) : 0.0;
  if (getenv("SSA_TRACE_SEQ")) {  // the raw sequence of a window of records
    const size_t a0 = std::min<size_t>(n, (size_t)atoi(getenv("SSA_TRACE_SEQ")));
    for (size_t i = a0; i + 1 < n && i < a0 + 40; ++i)
      fprintf(stderr, "[ssa seq] %5zu %-16s %8.2f us\n", i, names[ev[i].second & 31],
              1e-3 * (double)(ev[i + 1].first - ev[i].first));
  }
  fprintf(stderr, "[ssa trace] %llu kernels, %.1f us from first to last start\n", n, span);
  for (int id = 0; id < 32; ++id)
    if (cnt[id])
      fprintf(stderr, "[ssa trace] %-16s %6d x %8.2f us = %9.1f us (%4.1f%%)\n", names[id], cnt[id], tot[id] / cnt[id],
              tot[id], 100.0 * tot[id] / span);
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
  unsigned long long* trace = nullptr;
  if ((trace = trace_buffer()) != nullptr) {
    if ((e = cudaMemsetAsync(trace, 0, 8, s))) return e;
    if ((e = trace_attach(trace)) || (e = trace_attach_fft(trace))) return e;
  }
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
  const int gU = (L + kRitzSpan - 1) / kRitzSpan, gV = (K + kRitzSpan - 1) / kRitzSpan;
  double* amax = p.d_lgpart;
  int* aidx = reinterpret_cast<int*>(p.d_lgpart + (size_t)gU * k);
  // the Ritz kernel reads the step count m from the state word the SVD kernel used
  const int kb = (k + kRitzK - 1) / kRitzK;
  launch_pdl(lg_ritz, dim3(gU, kb), dim3(kThreads), 0, s, (const double*)U, ldL, 1, (const int*)p.d_state, cP, k, L,
             Uo, amax, aidx);
  launch_pdl(lg_ritz, dim3(gV, kb), dim3(kThreads), 0, s, (const double*)V, ldK, 0, (const int*)p.d_state, cQ, k, K,
             Vo, (double*)nullptr, (int*)nullptr);
  launch_pdl(lg_sign, dim3((k + 7) / 8), dim3(256), 0, s, (const double*)amax, (const int*)aidx, gU, k, (const double*)Uo, L, h);
  launch_pdl(lg_flip, dim3((int)(((size_t)L * k + kThreads - 1) / kThreads)), dim3(kThreads), 0, s, Uo, L, k,
             (const double*)h);
  launch_pdl(lg_flip, dim3((int)(((size_t)K * k + kThreads - 1) / kThreads)), dim3(kThreads), 0, s, Vo, K, k,
             (const double*)h);
  if (trace) trace_report(trace, s);
  return cudaGetLastError();
}

}  // namespace ssa
