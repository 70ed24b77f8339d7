// ssa_large_lanczos.cu -- Golub-Kahan-Lanczos with full reorthogonalization for a series
// too long for one CTA (BASELINE config 3: N = 2^20, L = 2^19, k = 32), one series at a
// time with the whole GPU on it (Alg. 1, FRO PAPER.md:388-393).
//
// Each half-step is a short sequence of grid-wide kernels on the same stream, each launched
// with programmatic dependent launch (launch_pdl / pdl_wait, device_common.cuh):
//   correlation  three-pass four-step FFT (ssa_large_fft.cu) with the recurrence term
//                fused in the epilogue: r = X^T u_j - beta_j v_{j-1} (or X v_j - alpha_j u_j),
//                plus per-CTA partial sums of squares;
//   dots         h = B^T r: each CTA owns a 512-element chunk of r (registers), streams the
//                basis rows of that chunk in groups of 8 with all loads in flight; per-CTA
//                partials are then summed in a fixed order (deterministic);
//   update       r -= B h with the rows in reverse order (recently read rows hit L2);
//   finish       one CTA (lg_finish): norms, the DGKS decision for a second pass, breakdown,
//                alpha_j / beta_{j+1} in device memory; second-pass kernels read the flag
//                and return at once when it is not needed;
//   normalize    v = r / alpha into the basis row.
// Convergence (the residual test of tgk.cuh on B_m) is evaluated by a one-CTA kernel and
// read by the host every check interval; after it, the bidiagonal SVD reuses
// bidiag_svd_tgk_kernel and the Ritz vectors come from lg_ritz (grid-wide, one pass over
// each basis) with sign canonicalization.
#include <stdio.h>

#include <algorithm>
#include <vector>

#include "device_common.cuh"
#include "tgk.cuh"

namespace ssa {

cudaError_t large_correlate(const Plan& p, const double2* spec, size_t spec_stride, const double* x, size_t xs, int n_in,
                            double* out, size_t os, int n_out, int ld_out, const double* prev, size_t ps,
                            const double* coef, double* part, int items, cudaStream_t s);
cudaError_t large_spectrum(const Plan& p, const double* series, double2* spec, int items, cudaStream_t s);
cudaError_t launch_bidiag_svd(const Plan& p, const DecomposeArgs& a, cudaStream_t s);
void large_geom(const Plan& p, int* N1, int* N2);

constexpr int kLgChunk = 2048;  // elements per CTA of the start vector (lg_start)

// device scalars of the long-series run
struct LgScalars {
  double nr;        // |r| before reorth (from the correlation partials)
  double nrm;       // current |r|
  double runmax;    // running max of alpha, beta
  double res;       // last convergence estimate
  int again;        // DGKS second pass needed
  int stop;         // breakdown with an exhausted space: stop
  int breakdown;    // first breakdown step
  int extra;        // DGKS passes taken
  int conv;         // converged flag
  int pad;
};

__global__ void __launch_bounds__(kThreads) lg_start(double* r, int n, int ld, uint64_t seed, uint64_t series,
                                                     double* part) {
  pdl_wait();
  __shared__ double red[kWarps];
  double ss = 0.0;
  for (int t = blockIdx.x * kLgChunk + threadIdx.x; t < (blockIdx.x + 1) * kLgChunk && t < ld; t += blockDim.x) {
    // the same counter-based generator as the batched kernel (R6)
    uint64_t x = seed ^ (series * 0xD1B54A32D192ED03ull);
    x += ((uint64_t)t + 1) * 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    x ^= x >> 31;
    double v = (t < n) ? 2.0 * ((double)(x >> 11) * 0x1.0p-53) - 1.0 : 0.0;
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
// set the rate).  512-element chunks: ~7 CTAs per SM at L = 2^19 (an even load).
constexpr int kRoChunk = 512;
constexpr int kRoE = kRoChunk / kThreads;  // 2
constexpr int kRoG = 8;                    // rows per group (warp_sum8)

// dots: part[row][cta] = <basis[row][chunk], r[chunk]>; smem red[nb][warps] (dynamic).
// Rows are read with L2 evict_last so lg_update (rows in reverse) finds the last ones.
__global__ void __launch_bounds__(kThreads) lg_dots(const double* __restrict__ basis, int ld, int nb,
                                                    const double* __restrict__ r, double* part, int nchunk,
                                                    const LgScalars* sc, int pass) {
  pdl_wait();
  if (pass == 1 && !sc->again) return;
  if (sc->stop) return;
  extern __shared__ double red[];  // [nb][kWarps]
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
}

// h[row] = sum over CTAs (fixed order)
__global__ void lg_rows(const double* __restrict__ part, int nb, int nchunk, double* h, const LgScalars* sc, int pass) {
  pdl_wait();
  if (pass == 1 && !sc->again) return;
  if (sc->stop) return;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= nb) return;
  double s = 0.0;
  for (int i = lane; i < nchunk; i += 32) s += part[(size_t)w * nchunk + i];
  s = warp_sum(s);
  if (lane == 0) h[w] = s;
}

// update: r -= sum_row h[row] basis[row] (rows in reverse: the rows lg_dots read last
// are still in L2), partial sums of squares; groups of kRoG rows, all loads in flight.
__global__ void __launch_bounds__(kThreads) lg_update(const double* __restrict__ basis, int ld, int nb,
                                                      const double* __restrict__ h, double* r, double* part,
                                                      const LgScalars* sc, int pass) {
  pdl_wait();
  if (pass == 1 && !sc->again) return;
  if (sc->stop) return;
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

// Norm bookkeeping at the end of a reorthogonalization pass, one CTA (replaces the
// separate |r| / DGKS / coefficient kernels):
//   pass 0: nr = |r| before reorth from the correlation partials (cpart[ncol]); with a
//           reorth pass (nb > 0) |r| from the update partials (part[nch]) and the DGKS
//           decision (second pass if |r| < nr / sqrt 2, or always for mode 2);
//   pass 1: runs only after a second pass: |r| from its update partials;
// then, unless a second pass follows, the Lanczos coefficient |r| (or 0 at breakdown,
// DESIGN.md R11) into coef_out.  Partial sums in a fixed order (deterministic).
__global__ void lg_finish(const double* __restrict__ cpart, int ncol, const double* __restrict__ part, int nch, int nb,
                          LgScalars* sc, int pass, int mode, double* coef_out, int step) {
  pdl_wait();
  if (pass == 1 && !sc->again) return;
  if (sc->stop) {
    if (pass == 0 && threadIdx.x == 0) *coef_out = 0.0;
    return;
  }
  // one CTA: thread-strided partial sums, shuffle trees, warps added in index order
  __shared__ double r1[kWarps], r2[kWarps];
  double s1 = 0.0, s2 = 0.0;
  if (pass == 0)
    for (int i = threadIdx.x; i < ncol; i += blockDim.x) s1 += cpart[i];
  if (nb > 0)
    for (int i = threadIdx.x; i < nch; i += blockDim.x) s2 += part[i];
  s1 = warp_sum(s1);
  s2 = warp_sum(s2);
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if ((threadIdx.x & 31) == 0) { r1[w] = s1; r2[w] = s2; }
  __syncthreads();
  if (threadIdx.x != 0) return;
  s1 = 0.0;
  s2 = 0.0;
  for (int i = 0; i < nw; ++i) { s1 += r1[i]; s2 += r2[i]; }
  int again = 0;
  double nn;
  if (pass == 0) {
    const double nr = sqrt(s1);
    sc->nr = nr;
    nn = (nb > 0) ? sqrt(s2) : nr;
    if (nb > 0) {
      again = (mode == 2 || nn < 0.70710678118654752 * nr) ? 1 : 0;
      if (again) sc->extra += 1;
    }
  } else {
    nn = sqrt(s2);
  }
  sc->nrm = nn;
  sc->again = again;
  if (again) return;
  if (!(nn > 1e-12 * sc->runmax) || nn == 0.0) {
    if (!sc->breakdown) sc->breakdown = step;
    *coef_out = 0.0;
    sc->stop = 1;  // invariant subspace found: no restart on the long path (R11)
  } else {
    *coef_out = nn;
    if (step > 0) sc->runmax = fmax(sc->runmax, nn);  // beta_1 (start vector norm) excluded
  }
}


__global__ void __launch_bounds__(kThreads) lg_normalize(const double* __restrict__ r, int n, int ld,
                                                         const double* coef, double* dst) {
  pdl_wait();
  const double c = *coef;
  const double inv = (c > 0.0) ? 1.0 / c : 0.0;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < ld) dst[t] = (t < n) ? r[t] * inv : 0.0;
}

// convergence test on B_m (tgk.cuh); alpha/beta 1-based in ab (alpha) and ab + w (beta)
__global__ void __launch_bounds__(kThreads) lg_check(const double* __restrict__ ab, int w, int m, int k, double tol,
                                                     double* scratch, LgScalars* sc) {
  pdl_wait();
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
  }
}

// Ritz vectors: out[i][t] = sum_row coef[row][i] basis[row][t], one element per thread.
// The coefficient rows are staged through a fixed shared-memory tile of kRitzRows rows
// (zero-padded to kMaxK per row, read as broadcast 16-byte loads), so the kernel's shared
// memory does not depend on the step count m.
constexpr int kRitzRows = 128;

__global__ void __launch_bounds__(kThreads) lg_ritz(const double* __restrict__ basis, int ld, int rows,
                                                    const double* __restrict__ coef, int k, int n, double* out,
                                                    double* amax, int* aidx) {
  pdl_wait();
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  __shared__ __align__(16) double cs[kRitzRows * kMaxK];
  double acc[kMaxK];
#pragma unroll
  for (int i = 0; i < kMaxK; ++i) acc[i] = 0.0;
  for (int r0 = 0; r0 < rows; r0 += kRitzRows) {
    const int nr = min(kRitzRows, rows - r0);
    __syncthreads();
    for (int e = threadIdx.x; e < nr * kMaxK; e += blockDim.x) {
      const int r = e / kMaxK, i = e - r * kMaxK;
      cs[e] = (i < k) ? __ldg(coef + (size_t)(r0 + r) * k + i) : 0.0;
    }
    __syncthreads();
    if (t < n) {
      for (int row = 0; row < nr; ++row) {
        const double x = __ldcs(basis + (size_t)(r0 + row) * ld + t);
        const double2* cr = reinterpret_cast<const double2*>(cs + (size_t)row * kMaxK);
#pragma unroll
        for (int i = 0; i < kMaxK / 2; ++i) {
          const double2 c = cr[i];
          acc[2 * i] = fma(c.x, x, acc[2 * i]);
          acc[2 * i + 1] = fma(c.y, x, acc[2 * i + 1]);
        }
      }
    }
  }
  if (t < n) {
#pragma unroll
    for (int i = 0; i < kMaxK; ++i)
      if (i < k) out[(size_t)i * n + t] = acc[i];
  }
  if (amax) {
    // per-CTA argmax |out_i| (lowest index on ties) for sign canonicalization
    __shared__ double sv[kWarps][kMaxK];
    __shared__ int si[kWarps][kMaxK];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
    for (int i = 0; i < kMaxK; ++i) {
      if (i >= k) break;
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
    if (threadIdx.x < k) {
      double v = -1.0;
      int ix = 0x7fffffff;
      for (int q = 0; q < kWarps; ++q)
        if (sv[q][threadIdx.x] > v || (sv[q][threadIdx.x] == v && si[q][threadIdx.x] < ix)) {
          v = sv[q][threadIdx.x];
          ix = si[q][threadIdx.x];
        }
      amax[(size_t)blockIdx.x * k + threadIdx.x] = v;
      aidx[(size_t)blockIdx.x * k + threadIdx.x] = ix;
    }
  }
}

__global__ void lg_sign(const double* __restrict__ amax, const int* __restrict__ aidx, int nblk, int k,
                        const double* __restrict__ U, int L, double* sgn) {
  pdl_wait();
  const int i = threadIdx.x;
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

size_t lg_check_smem(int m_max) { return (size_t)(3 * (2 * m_max + 1) + 4 * kMaxK) * 8 + 64; }

cudaError_t large_lanczos_set_attributes(int m_max) {
  cudaError_t e = raise_smem_limit(lg_check, (int)lg_check_smem(m_max));
  if (e == cudaSuccess) e = raise_smem_limit(lg_dots, (size_t)(m_max + 2) * kWarps * 8);
  if (e == cudaSuccess) e = raise_smem_limit(lg_update, (size_t)(m_max + 2) * 8);
  return e;
}


__global__ void lg_finite(const double* __restrict__ f, int N, int* state) {
  pdl_wait();
  int bad = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) bad |= !isfinite(f[i]);
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(state + 5, 1);
}

__global__ void lg_state(const LgScalars* sc, int* state, int m) {
  pdl_wait();
  if (threadIdx.x != 0) return;
  state[0] = m;
  state[1] = sc->conv;
  state[2] = sc->breakdown;
  state[3] = sc->extra;
  state[4] = 0;
  state[6] = 0;
}

// One long series b of the call: decompose into sigma/U/V (+info).  Host-driven loop; the
// host reads the device scalars only at convergence tests.
cudaError_t large_decompose_one(Plan& p, const DecomposeArgs& a0, int b, cudaStream_t s) {
  DecomposeArgs a = a0;
  a.b0 = b;
  a.nb = 1;
  const int L = (int)p.L, K = (int)p.K, N = (int)p.N, k = p.k;
  const int ldL = p.ldL, ldK = p.ldK;
  const int nchL = (ldL + kLgChunk - 1) / kLgChunk;
  int N1, N2;
  large_geom(p, &N1, &N2);
  const int ncol = N2 / 8;  // partial sums written by lg_col_inv (one per 8-column CTA)
  double* U = p.d_U;
  double* V = p.d_V;
  const int w = p.m_max + 3;
  double* alpha = p.d_ab;
  double* beta = p.d_ab + w;
  LgScalars* sc = reinterpret_cast<LgScalars*>(p.d_lgsc);
  double* part = p.d_lgpart;
  double* h = p.d_lgh;
  double* r = p.d_lgr;
  cudaError_t e;
  if ((e = cudaMemsetAsync(p.d_state, 0, kStateInts * sizeof(int), s))) return e;
  launch_pdl(lg_finite, dim3(64), dim3(kThreads), 0, s, a.series + (size_t)b * N, N, p.d_state);
  if ((e = large_spectrum(p, a.series + (size_t)b * N, p.d_spec, 1, s))) return e;
  LgScalars z{};
  if ((e = cudaMemcpyAsync(sc, &z, sizeof(z), cudaMemcpyHostToDevice, s))) return e;
  if ((e = cudaMemsetAsync(p.d_ab, 0, 2 * (size_t)w * 8, s))) return e;
  // Alg. 1 lines 1-2: u_1 = p0 / |p0|
  // partial sums of the correlation / start vector go after the dots partials (the
  // reorth kernels overwrite `part`)
  double* cpart = part + (size_t)((std::max(ldL, ldK) + kRoChunk - 1) / kRoChunk) * (p.m_max + 2);
  launch_pdl(lg_start, dim3(nchL), dim3(kThreads), 0, s, r, L, ldL, a.seed, (uint64_t)(b + a.series_base), cpart);
  // beta_1 = |p0| into beta[1], then u_1 = p0 / beta_1
  launch_pdl(lg_finish, dim3(1), dim3(kThreads), 0, s, cpart, nchL, part, 0, 0, sc, 0, p.opt.reorth, beta + 1, 0);
  launch_pdl(lg_normalize, dim3((ldL + kThreads - 1) / kThreads), dim3(kThreads), 0, s, r, L, ldL, beta + 1, U);
  // reorth against nb basis rows (CGS + DGKS), then the coefficient into coef
  auto reorth = [&](const double* basis, int ld, int nb, double* coef, int step) {
    const int nch = (ld + kRoChunk - 1) / kRoChunk;
    for (int pass = 0; pass < 2; ++pass) {
      if (nb > 0) {
        launch_pdl(lg_dots, dim3(nch), dim3(kThreads), (size_t)nb * kWarps * 8, s, basis, ld, nb, r, part, nch, sc, pass);
        launch_pdl(lg_rows, dim3((nb * 32 + kThreads - 1) / kThreads), dim3(kThreads), 0, s, part, nb, nch, h, sc, pass);
        launch_pdl(lg_update, dim3(nch), dim3(kThreads), (size_t)nb * 8, s, basis, ld, nb, h, r, part, sc, pass);
      }
      launch_pdl(lg_finish, dim3(1), dim3(kThreads), 0, s, cpart, ncol, part, nch, nb, sc, pass, p.opt.reorth, coef, step);
      if (nb == 0) break;
    }
  };
  int m = 0;
  int next_check = (2 * k < p.m_max) ? 2 * k : k;
  const int ce = p.opt.check_every > 0 ? p.opt.check_every : 4;
  double prev_res = -1.0;
  int prev_m = 0;
  LgScalars hs{};
  for (int j = 1; j <= p.m_max + 1; ++j) {
    // ---- half-step A (Alg. 1 l.4-5): r = X^T u_j - beta_j v_{j-1}; FRO vs V_{j-1} ----
    if ((e = large_correlate(p, p.d_spec, 0, U + (size_t)(j - 1) * ldL, 0, L, r, 0, K, ldK,
                             (j > 1) ? V + (size_t)(j - 2) * ldK : nullptr, 0, beta + j, cpart, 1, s)))
      return e;
    reorth(V, ldK, j - 1, alpha + j, j);
    launch_pdl(lg_normalize, dim3((ldK + kThreads - 1) / kThreads), dim3(kThreads), 0, s, r, K, ldK, alpha + j, V + (size_t)(j - 1) * ldK);
    m = j - 1;
    const bool last = (m >= p.m_max);
    if (m >= k && (m >= next_check || last)) {
      launch_pdl(lg_check, dim3(1), dim3(kThreads), lg_check_smem(p.m_max), s, p.d_ab, w, m, k, p.opt.tol, p.d_tgk, sc);
      if ((e = cudaMemcpyAsync(&hs, sc, sizeof(hs), cudaMemcpyDeviceToHost, s))) return e;
      if ((e = cudaStreamSynchronize(s))) return e;
      if (hs.conv) break;
      int step = ce;
      if (prev_res > 0.0 && hs.res < prev_res && hs.res > 0.0) {
        double rate = log(hs.res / prev_res) / (double)(m - prev_m);
        double need = log(0.5 * p.opt.tol / hs.res) / rate;
        int s2 = (int)(0.7 * need);
        if (s2 > step) step = s2 < 2 * ce ? s2 : 2 * ce;
      }
      prev_res = hs.res;
      prev_m = m;
      next_check = m + step;
    }
    if (last) break;
    // ---- half-step B (Alg. 1 l.6-7): p = X v_j - alpha_j u_j; FRO vs U_j ----
    if ((e = large_correlate(p, p.d_spec, 0, V + (size_t)(j - 1) * ldK, 0, K, r, 0, L, ldL,
                             U + (size_t)(j - 1) * ldL, 0, alpha + j, cpart, 1, s)))
      return e;
    reorth(U, ldL, j, beta + j + 1, j);
    launch_pdl(lg_normalize, dim3((ldL + kThreads - 1) / kThreads), dim3(kThreads), 0, s, r, L, ldL, beta + j + 1, U + (size_t)j * ldL);
  }
  launch_pdl(lg_state, dim3(1), dim3(32), 0, s, sc, p.d_state, m);
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
  launch_pdl(lg_ritz, dim3(gU), dim3(kThreads), 0, s, U, ldL, m + 1, cP, k, L, Uo, amax, aidx);
  launch_pdl(lg_ritz, dim3(gV), dim3(kThreads), 0, s, V, ldK, m, cQ, k, K, Vo, nullptr, nullptr);
  launch_pdl(lg_sign, dim3(1), dim3(32), 0, s, amax, aidx, gU, k, Uo, L, h);
  launch_pdl(lg_flip, dim3((int)(((size_t)L * k + kThreads - 1) / kThreads)), dim3(kThreads), 0, s, Uo, L, k, h);
  launch_pdl(lg_flip, dim3((int)(((size_t)K * k + kThreads - 1) / kThreads)), dim3(kThreads), 0, s, Vo, K, k, h);
  return cudaGetLastError();
}

}  // namespace ssa
