// ssa_lanczos.cu -- persistent batched Golub-Kahan-Lanczos bidiagonalization with full
// reorthogonalization (Alg. 1; FRO PAPER.md:388-393), one CTA per
// series taken from a work queue.
//
// Per step j (all on chip except the Krylov basis, which lives in HBM):
//   A: r = X^T u_j - beta_j v_{j-1}      FFT correlation in shared memory (Alg. 3)
//      CGS against V_{j-1} (+ DGKS pass)  basis streamed by per-warp TMA bulk rings
//      alpha_j = |r|, v_j = r / alpha_j   written once to HBM
//      convergence test on B_{j-1} using alpha_j (tgk_check.cuh), on schedule
//   B: p = X v_j - alpha_j u_j           FFT correlation (Alg. 2)
//      CGS against U_j (+ DGKS pass); beta_{j+1} = |p|; u_{j+1} = p / beta_{j+1}
// Lucky breakdown (alpha or beta < 1e-12 running max) restarts with a seeded random
// vector orthogonal to the basis and a zero coefficient in B (R11).
// Output per series: the bases, alpha/beta and the step count m; the bidiagonal SVD and
// the Ritz assembly are separate kernels (ssa_svd.cu).
#include "device_common.cuh"
#include "tgk.cuh"

namespace ssa {

struct LSmem {
  unsigned char* regionA;  // union: FFT buffer | rings + partial dots | TGK arrays
  double* bufU;            // ldL
  double* bufV;            // ldK
  double* h;               // m_max + 2
  double* alpha;           // m_max + 3 (1-based)
  double* beta;            // m_max + 3 (1-based)
  double* mu;              // m_max + 3: PRO estimates of u_{j}^T u_i (1-based), R22
  double* nu;              // m_max + 3: PRO estimates of v_{j}^T v_i
  double* red;             // 32
  int* redi;               // 8 ints
  int* cl;                 // kClInts ints: cluster starts of the final SVD (tgk_clusters)
  double* chk;             // 4 k: omega, res, lohi(2k)
  double2* tw;             // two-level twiddle table for M (tw2_entries(M))
  uint64_t* bars;          // kWarps * kStages
  double* T;               // thick restart: the projected matrix, (m_max+1) x (m_max+1) row-major
};

// thick restart: doubles of the one-sided Jacobi scratch in region A (W, Q, sigma, order)
__host__ __device__ inline size_t trl_jacobi_doubles(int d) { return (size_t)2 * (d + 1) * (d + 1) + 2 * (d + 1); }

__host__ __device__ inline size_t lanczos_regionA_bytes(int H, int ldL, int ldK, int m_max, bool trl = false) {
  int slab_max = (ldL > ldK ? ldL : ldK) / kWarps;
  size_t fft = (size_t)fft_elems(H) * 16;
  size_t rings = (size_t)kWarps * kStages * slab_max * 8 + (size_t)kWarps * (m_max + 2) * 8;
  size_t tgk = (size_t)7 * (2 * m_max + 2) * 8;  // c, c^2, c^2/|T|^2 + the cheap test's pivots
  size_t r = fft;
  if (rings > r) r = rings;
  if (tgk > r) r = tgk;
  if (trl && trl_jacobi_doubles(m_max) * 8 > r) r = trl_jacobi_doubles(m_max) * 8;
  return align16(r);
}

size_t lanczos_smem_bytes(int H, int ldL, int ldK, int m_max, int k, bool trl) {
  size_t s = lanczos_regionA_bytes(H, ldL, ldK, m_max, trl);
  s += align16((size_t)ldL * 8) + align16((size_t)ldK * 8);
  s += 5 * align16((size_t)(m_max + 3) * 8);
  s += 32 * 8 + 8 * 4 + align16((size_t)kClInts * 4) + (size_t)4 * k * 8;
  s += (size_t)tw2_entries(2 * H) * 16;
  s += (size_t)kWarps * kStages * 8;
  if (trl) s += (size_t)(m_max + 1) * (m_max + 1) * 8;
  return align16(s) + 16;
}

__device__ inline LSmem carve(unsigned char* base, const DecomposeArgs& a) {
  LSmem s;
  size_t off = 0;
  s.regionA = base;
  off += lanczos_regionA_bytes(a.H, a.ldL, a.ldK, a.m_max, a.trl_d > 0);
  s.bufU = reinterpret_cast<double*>(base + off); off += align16((size_t)a.ldL * 8);
  s.bufV = reinterpret_cast<double*>(base + off); off += align16((size_t)a.ldK * 8);
  s.h = reinterpret_cast<double*>(base + off); off += align16((size_t)(a.m_max + 3) * 8);
  s.alpha = reinterpret_cast<double*>(base + off); off += align16((size_t)(a.m_max + 3) * 8);
  s.beta = reinterpret_cast<double*>(base + off); off += align16((size_t)(a.m_max + 3) * 8);
  s.mu = reinterpret_cast<double*>(base + off); off += align16((size_t)(a.m_max + 3) * 8);
  s.nu = reinterpret_cast<double*>(base + off); off += align16((size_t)(a.m_max + 3) * 8);
  s.red = reinterpret_cast<double*>(base + off); off += 32 * 8;
  s.redi = reinterpret_cast<int*>(base + off); off += 8 * 4;
  s.cl = reinterpret_cast<int*>(base + off); off += align16((size_t)kClInts * 4);
  s.chk = reinterpret_cast<double*>(base + off); off += (size_t)4 * a.k * 8;
  s.tw = reinterpret_cast<double2*>(base + off); off += (size_t)tw2_entries(2 * a.H) * 16;
  s.bars = reinterpret_cast<uint64_t*>(base + off); off += (size_t)kWarps * kStages * 8;
  s.T = (a.trl_d > 0) ? reinterpret_cast<double*>(base + off) : nullptr;
  return s;
}

// Values per group of twisted factorizations whose pivots (2 n doubles each) fit in
// region A after the three TGK arrays.
__device__ __forceinline__ int tgk_group(const DecomposeArgs& a, int n) {
  const long long avail = (long long)(lanczos_regionA_bytes(a.H, a.ldL, a.ldK, a.m_max) / 8) - 3LL * (2 * a.m_max + 2);
  long long kg = avail / (2LL * n);
  if (kg > a.k) kg = a.k;
  return kg < 1 ? 1 : (int)kg;
}

// Counter-based start / restart vectors (R6): splitmix64 of (seed, series, i).
__device__ __forceinline__ double rng_uniform_pm1(uint64_t seed, uint64_t series, uint64_t i) {
  uint64_t x = seed ^ (series * 0xD1B54A32D192ED03ull);
  x += (i + 1) * 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  x ^= x >> 31;
  return 2.0 * ((double)(x >> 11) * 0x1.0p-53) - 1.0;
}

// CGS pass(es) of r (SMEM, ld doubles, zero padding) against basis rows [0, nb).
// Returns the new norm; nrm_in is |r| before.  mode 1: DGKS (second pass iff the norm
// fell below 1/sqrt(2) of its value), mode 2: always two passes (PAPER.md:388-393,
// DESIGN.md R9).  Each warp owns a column slab of r and of the basis; the dot products
// are reduced across warps in a fixed order (deterministic).
// EPL elements of the warp's slab per lane live in registers (element lane + 32 t).
template <int EPL>
__device__ double reorth_t(double* r, const double* basis, int nb, int ld, double nrm_in, int mode, const LSmem& sm,
                           WarpRing& rg, double* part, int pstride, int& extra, double* hacc) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int slab = ld / kWarps;
  double* rw = r + w * slab;
  const double* bw = basis + (size_t)w * slab;
  double rv[EPL];
#pragma unroll
  for (int t = 0; t < EPL; ++t) {
    const int e = lane + 32 * t;
    rv[t] = (e < slab) ? rw[e] : 0.0;
  }
  double nrm = nrm_in;
  const uint64_t pol_last = policy_evict_last(), pol_first = policy_evict_first();
  for (int pass = 0; pass < 2 && nb > 0; ++pass) {
    fence_proxy_async_smem();
    __syncthreads();
    // pass 1: partial dots of this warp's slab with every basis row; the lines stay in L2
    // (evict_last) for pass 2
    if constexpr (EPL <= 4) {
      // small slabs (N <~ 2K): the rows are a few hundred bytes and L2-resident, and the
      // TMA ring is latency-bound on them; read groups of 8 rows with plain L2 loads (all
      // in flight) and reduce their 8 partial dots together (warp_sum8: 9 shuffles)
      for (int row0 = 0; row0 < nb; row0 += 8) {
        double x[8][EPL];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int t = 0; t < EPL; ++t) {
            const int e = lane + 32 * t;
            x[i][t] = (row0 + i < nb && e < slab) ? __ldcg(bw + (size_t)(row0 + i) * ld + e) : 0.0;
          }
        double d[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          double acc = 0.0;
#pragma unroll
          for (int t = 0; t < EPL; ++t) acc = fma(x[i][t], rv[t], acc);
          d[i] = acc;
        }
        const double tot = warp_sum8(d, lane);
        const int q = (lane >> 2) & 7;
        if ((lane & 3) == 0 && row0 + q < nb) part[w * pstride + row0 + q] = tot;
      }
    } else {
      stream_rows(bw, ld, nb, false, slab, rg, pol_last, [&](int row, const double* ch) {
        double s = 0.0;
#pragma unroll
        for (int t = 0; t < EPL; ++t) {
          const int e = lane + 32 * t;
          if (e < slab) s = fma(ch[e], rv[t], s);
        }
        s = warp_sum(s);
        if (lane == 0) part[w * pstride + row] = s;
      });
    }
    __syncthreads();
    for (int c = threadIdx.x; c < nb; c += blockDim.x) {
      double s = 0.0;
      for (int q = 0; q < kWarps; ++q) s += part[q * pstride + c];
      sm.h[c] = s;
      if (hacc) hacc[c] += s;  // thick restart: the coefficients are entries of T
    }
    __syncthreads();
    // pass 2: r -= V h, rows streamed in reverse so the most recently read rows (still
    // in L2) come first; read for the last time in this half-step (evict_first)
    if constexpr (EPL <= 4) {
      // rows in reverse, groups of 8 plain L2 loads in flight (as the dots pass)
      for (int top = nb - 1; top >= 0; top -= 8) {
        double x[8][EPL];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int t = 0; t < EPL; ++t) {
            const int e = lane + 32 * t;
            x[i][t] = (top - i >= 0 && e < slab) ? __ldcg(bw + (size_t)(top - i) * ld + e) : 0.0;
          }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const double hc = (top - i >= 0) ? sm.h[top - i] : 0.0;
#pragma unroll
          for (int t = 0; t < EPL; ++t) rv[t] = fma(-hc, x[i][t], rv[t]);
        }
      }
    } else {
      stream_rows(bw, ld, nb, true, slab, rg, pol_first, [&](int row, const double* ch) {
        const double hc = sm.h[row];
#pragma unroll
        for (int t = 0; t < EPL; ++t) {
          const int e = lane + 32 * t;
          if (e < slab) rv[t] = fma(-hc, ch[e], rv[t]);
        }
      });
    }
    double ss = 0.0;
#pragma unroll
    for (int t = 0; t < EPL; ++t) ss = fma(rv[t], rv[t], ss);
    double nn = sqrt(block_sum(ss, sm.red));
    bool again = (pass == 0) && (mode == 2 || nn < 0.70710678118654752 * nrm);
    nrm = nn;
    if (!again) break;
    ++extra;
  }
#pragma unroll
  for (int t = 0; t < EPL; ++t) {
    const int e = lane + 32 * t;
    if (e < slab) rw[e] = rv[t];
  }
  __syncthreads();
  return nrm;
}

// CGS pass(es) of r (SMEM, ld doubles, zero padding) against basis rows [0, nb).
// Returns the new norm; nrm_in is |r| before.  mode 1: DGKS (second pass iff the norm
// fell below 1/sqrt(2) of its value), mode 2: always two passes (PAPER.md:388-393,
// DESIGN.md R9).  Each warp owns a column slab of r (held in registers) and of the basis;
// the dot products are reduced across warps in a fixed order (deterministic).
__device__ double reorth(double* r, const double* basis, int nb, int ld, double nrm_in, int mode, const LSmem& sm,
                         WarpRing& rg, double* part, int pstride, int& extra, double* hacc = nullptr) {
  const int epl = (ld / kWarps + 31) / 32;
  if (epl <= 1) return reorth_t<1>(r, basis, nb, ld, nrm_in, mode, sm, rg, part, pstride, extra, hacc);
  if (epl <= 2) return reorth_t<2>(r, basis, nb, ld, nrm_in, mode, sm, rg, part, pstride, extra, hacc);
  if (epl <= 4) return reorth_t<4>(r, basis, nb, ld, nrm_in, mode, sm, rg, part, pstride, extra, hacc);
  if (epl <= 8) return reorth_t<8>(r, basis, nb, ld, nrm_in, mode, sm, rg, part, pstride, extra, hacc);
  if (epl <= 9) return reorth_t<9>(r, basis, nb, ld, nrm_in, mode, sm, rg, part, pstride, extra, hacc);
  if (epl <= 16) return reorth_t<16>(r, basis, nb, ld, nrm_in, mode, sm, rg, part, pstride, extra, hacc);
  if (epl <= 17) return reorth_t<17>(r, basis, nb, ld, nrm_in, mode, sm, rg, part, pstride, extra, hacc);
  return reorth_t<32>(r, basis, nb, ld, nrm_in, mode, sm, rg, part, pstride, extra, hacc);
}

// Write r * inv into basis row dst (plain coalesced stores), scale r in place.
__device__ __forceinline__ void normalize_store(double* r, int n, int ld, double inv, double* dst) {
  for (int t = threadIdx.x; t < ld; t += blockDim.x) {
    double v = (t < n) ? r[t] * inv : 0.0;
    r[t] = v;
    dst[t] = v;
  }
  fence_proxy_async_global();
  __syncthreads();
}

// Seeded random vector orthogonalized twice against the basis (restart at breakdown).
// Returns its norm after orthogonalization relative to before (0 if the space is full).
__device__ double restart_vector(double* r, int n, int ld, const double* basis, int nb, uint64_t seed,
                                 uint64_t series, uint64_t salt, const LSmem& sm, WarpRing& rg, double* part,
                                 int pstride) {
  double ss = 0.0;
  for (int t = threadIdx.x; t < ld; t += blockDim.x) {
    double v = (t < n) ? rng_uniform_pm1(seed, series, salt + t) : 0.0;
    r[t] = v;
    ss += v * v;
  }
  double nrm = sqrt(block_sum(ss, sm.red));
  int extra = 0;
  double nn = reorth(r, basis, nb, ld, nrm, 2, sm, rg, part, pstride, extra);
  return nn / nrm;
}

// ---- partial reorthogonalization (PRO; Simon 1984, Larsen 1998) ----
// The orthogonality levels omega of the newest Lanczos vector against the basis obey the
// recurrences obtained from Alg. 1 lines 4-7 by taking inner products:
//   v side:  alpha_j nu_{j,i}     = alpha_i mu_{j,i} + beta_{i+1} mu_{j,i+1} - beta_j nu_{j-1,i}
//   u side:  beta_{j+1} mu_{j+1,i} = alpha_i nu_{j,i} + beta_i nu_{j,i-1}    - alpha_j mu_{j,i}
// plus a rounding term eps (|B row i| + |B row j|) + eps |A| with the sign of the value
// (Larsen's update_nu / update_mu).  Updated in place (thread i owns index i; the other
// side's array is read only).  Returns max_i |omega_i| (block-uniform).
constexpr double kEps = 2.220446049250313e-16;

__device__ __forceinline__ double block_max(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s = fmax(s, red[i]);
  return s;
}

// nu_{j,i}, i = 1..j-1, for the new v_j (norm a_est before any reorthogonalization)
__device__ double pro_update_nu(const LSmem& sm, int j, double a_est, double bj, double anorm) {
  double mx = 0.0;
  const double rj = hypot(a_est, bj);
  for (int i = 1 + threadIdx.x; i <= j - 1; i += blockDim.x) {
    double t = fma(sm.alpha[i], sm.mu[i], fma(sm.beta[i + 1], sm.mu[i + 1], -bj * sm.nu[i]));
    const double d = kEps * (hypot(sm.alpha[i], sm.beta[i + 1]) + rj) + kEps * anorm;
    t = (t + copysign(d, t)) / a_est;
    sm.nu[i] = t;
    mx = fmax(mx, fabs(t));
  }
  return block_max(mx, sm.red);
}

// mu_{j+1,i}, i = 1..j, for the new u_{j+1} (norm b_est before any reorthogonalization)
__device__ double pro_update_mu(const LSmem& sm, int j, double b_est, double aj, double anorm) {
  double mx = 0.0;
  const double rj = hypot(aj, b_est);
  for (int i = 1 + threadIdx.x; i <= j; i += blockDim.x) {
    double t = fma(sm.alpha[i], sm.nu[i], fma(sm.beta[i], sm.nu[i - 1], -aj * sm.mu[i]));
    const double d = kEps * (hypot(sm.alpha[i], sm.beta[i]) + rj) + kEps * anorm;
    t = (t + copysign(d, t)) / b_est;
    sm.mu[i] = t;
    mx = fmax(mx, fabs(t));
  }
  return block_max(mx, sm.red);
}

// after a full reorthogonalization against rows 1..n the estimates drop to eps
__device__ __forceinline__ void pro_reset(double* om, int n) {
  for (int i = 1 + threadIdx.x; i <= n; i += blockDim.x) om[i] = kEps;
}

__global__ void __launch_bounds__(kThreads, 2) lanczos_kernel(const DecomposeArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  LSmem sm = carve(smem_raw, a);
  const int tid = threadIdx.x, w = tid >> 5;
  const FftShape sh = make_shape(a.H);
  const int slab_max = (a.ldL > a.ldK ? a.ldL : a.ldK) / kWarps;
  double2* fbuf = reinterpret_cast<double2*>(sm.regionA);
  double* rings = reinterpret_cast<double*>(sm.regionA);
  double* part = rings + (size_t)kWarps * kStages * slab_max;
  const int pstride = a.m_max + 2;
  double* tc = reinterpret_cast<double*>(sm.regionA);  // TGK off-diagonals (aliases the rings)
  double* tc2 = tc + (2 * a.m_max + 2);

  const TwSmem tw = load_tw2(a.tw, sm.tw, 2 * a.H);
  WarpRing rg;
  ring_init(rg, rings + (size_t)w * kStages * slab_max, sm.bars + w * kStages);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();

  const int L = a.L, K = a.K, k = a.k;
  unsigned long long pc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long t_mark = clock64();
  auto lap = [&](int slot) {
    long long t = clock64();
    pc[slot] += (unsigned long long)(t - t_mark);
    t_mark = t;
  };

  while (true) {
    __syncthreads();
    if (tid == 0) sm.redi[4] = atomicAdd(a.counters + 0, 1);
    __syncthreads();
    const int bl = sm.redi[4];  // series index within the chunk
    if (bl >= a.nb) break;
    const int b = a.b0 + bl;
    const double* f = a.series + (size_t)b * a.N;
    const double2* spec = a.spec + (size_t)bl * (a.H + 1);
    double* U = a.U + (size_t)bl * (a.m_max + 1) * a.ldL;
    double* V = a.V + (size_t)bl * (a.m_max + 1) * a.ldK;
    double* abg = a.ab + (size_t)bl * 2 * (a.m_max + 3);
    int* st = a.state + (size_t)bl * kStateInts;

    // ---- non-finite input -> INVALID_ARGUMENT ----
    int bad = 0;
    for (int t = tid; t < a.N; t += blockDim.x) bad |= !isfinite(f[t]);
    if (block_or(bad, sm.redi)) {
      if (tid == 0) {
        for (int q = 0; q < kStateInts; ++q) st[q] = (q == 5) ? 1 : 0;
      }
      continue;
    }

    // ---- Alg. 1 lines 1-2: p0 seeded, beta_1 = |p0|, u_1 = p0 / beta_1, v_0 = 0 ----
    double ss = 0.0;
    for (int t = tid; t < a.ldL; t += blockDim.x) {
      double v = (t < L) ? rng_uniform_pm1(a.seed, (uint64_t)(b + a.series_base), (uint64_t)t) : 0.0;
      sm.bufU[t] = v;
      ss += v * v;
    }
    for (int t = tid; t < a.ldK; t += blockDim.x) sm.bufV[t] = 0.0;
    double beta1 = sqrt(block_sum(ss, sm.red));
    if (tid == 0) { sm.beta[1] = beta1; sm.alpha[0] = 0.0; sm.beta[0] = 0.0; }
    normalize_store(sm.bufU, L, a.ldL, 1.0 / beta1, U);

    // PRO state: omega estimates (1-based; mu_1 = 1 for u_1), forced follow-up flags
    const bool pro = (a.reorth_mode == 3);
    for (int i = tid; i < a.m_max + 3; i += blockDim.x) {
      sm.mu[i] = (i == 1) ? 1.0 : 0.0;
      sm.nu[i] = 0.0;
    }
    bool force_v = false, force_u = false;
    int rows_u = 0, rows_v = 0, rsteps = 0;

    double runmax = 0.0, bcur = beta1;
    int m = 0, converged = 0, breakdown = 0, extra = 0, restarts = 0, checks = 0;
    int next_check = (a.first_check < a.m_max) ? a.first_check : k;
    double prev_res = -1.0;
    int prev_m = 0;
    const int ce = a.check_every > 0 ? a.check_every : 4;

    for (int j = 1; j <= a.m_max + 1; ++j) {
      // ---- half-step A (Alg. 1 l.4-5): r = X^T u_j - beta_j v_{j-1}; FRO vs V_{j-1} ----
      lap(7);
      const double bj = bcur;  // beta_j (register copy: sm.beta is written by thread 0 only)
      correlate_cta(
          fbuf, sh, tw, spec, L, K, [&](int i) { return sm.bufU[i]; },
          [&](int t, double y) { sm.bufV[t] = y - bj * sm.bufV[t]; });
      __syncthreads();
      ss = 0.0;
      for (int t = tid; t < K; t += blockDim.x) ss = fma(sm.bufV[t], sm.bufV[t], ss);
      double nr = sqrt(block_sum(ss, sm.red));
      lap(0);
      // FRO: every half-step; PRO: only when the estimated level exceeds eta, and on the
      // v half-step after one that did (Simon / Larsen), R22
      bool do_ro = !pro || force_v;
      if (pro && j >= 2 && nr > 0.0) do_ro = (pro_update_nu(sm, j, nr, bj, runmax) > a.pro_eta) || force_v;
      double al = nr;
      if (do_ro && j >= 2) {
        const int e0 = extra;
        al = reorth(sm.bufV, V, j - 1, a.ldK, nr, pro ? 1 : a.reorth_mode, sm, rg, part, pstride, extra);
        rows_v += 2 * (j - 1) * (1 + extra - e0);
        ++rsteps;
        if (pro) pro_reset(sm.nu, j - 1);
        force_v = pro && !force_v;
      } else {
        force_v = false;
      }
      if (!(al > 1e-12 * runmax) || al == 0.0) {
        if (!breakdown) breakdown = j;
        double q = (j - 1 < K) ? restart_vector(sm.bufV, K, a.ldK, V, j - 1, a.seed, (uint64_t)(b + a.series_base),
                                                ((uint64_t)(++restarts) << 40), sm, rg, part, pstride)
                               : 0.0;
        if (q > 1e-8) {
          ss = 0.0;
          for (int t = tid; t < K; t += blockDim.x) ss = fma(sm.bufV[t], sm.bufV[t], ss);
          double nn = sqrt(block_sum(ss, sm.red));
          normalize_store(sm.bufV, K, a.ldK, 1.0 / nn, V + (size_t)(j - 1) * a.ldK);
        } else {
          normalize_store(sm.bufV, K, a.ldK, 0.0, V + (size_t)(j - 1) * a.ldK);
        }
        al = 0.0;
        if (pro) pro_reset(sm.nu, j - 1);  // the restart vector is orthogonalized twice
      } else {
        normalize_store(sm.bufV, K, a.ldK, 1.0 / al, V + (size_t)(j - 1) * a.ldK);
      }
      if (tid == 0) {
        sm.alpha[j] = al;
        sm.nu[j] = 1.0;
      }
      runmax = fmax(runmax, al);
      m = j - 1;
      lap(1);

      // ---- convergence test on B_m with alpha_{m+1} = al (R7) ----
      const bool last = (m >= a.m_max);
      if (m >= k && (m >= next_check || last)) {
        // TGK off-diagonals (alpha_1, beta_2, ..., alpha_m, beta_{m+1}) into SMEM
        const int n = 2 * m + 1;
        __syncthreads();
        for (int i = tid; i < n - 1; i += blockDim.x) {
          double v = (i & 1) ? sm.beta[(i >> 1) + 2] : sm.alpha[(i >> 1) + 1];
          tc[i] = v;
          tc2[i] = v * v;
        }
        __syncthreads();
        double* om = sm.chk;
        double* res = om + k;
        double* lohi = res + k;
        // pivots of the twisted factorizations: shared memory when they fit in region A
        double* tc2n = tc2 + (2 * a.m_max + 2);
        // pivots of the twisted factorizations in shared memory (region A after the
        // three TGK arrays), in groups of kg values when all k do not fit
        double* dsc = tc2n + (2 * a.m_max + 2);
        const int kg = tgk_group(a, n);
        // cheap test first: omega_1 and the k-th (slowest-converging) triple only; the
        // full test of all k runs only when that one passes
        double rel;
        {
          const int nv = (k > 1) ? 2 : 1;
          tgk_check(tc, tc2, tc2n, m, nv, al, om, res, lohi, tc2n + (2 * a.m_max + 2), k - 1, 32, pc + 4);
          rel = (om[0] > 0.0) ? res[nv - 1] / om[0] : 0.0;
        }
        if (rel <= 0.5 * a.tol && k > 1) {
          tgk_check(tc, tc2, tc2n, m, k, al, om, res, lohi, dsc, 1, kg, pc + 4);
          double mr = 0.0;
          for (int i = 0; i < k; ++i) mr = fmax(mr, res[i]);
          rel = (om[0] > 0.0) ? mr / om[0] : 0.0;
        }
        ++checks;
        lap(2);
        // the estimate must be below tol/2 (the final QR residual is what gets reported)
        if (rel <= 0.5 * a.tol) { converged = 1; break; }
        // schedule the next test from the observed geometric decay of the residual
        int step = ce;
        if (prev_res > 0.0 && rel < prev_res && rel > 0.0) {
          double rate = log(rel / prev_res) / (double)(m - prev_m);
          double need = log(0.5 * a.tol / rel) / rate;
          int s2 = (int)(0.7 * need);
          if (s2 > step) step = s2 < a.check_cap ? s2 : a.check_cap;
        }
        prev_res = rel;
        prev_m = m;
        next_check = m + step;
      }
      if (last) break;

      // ---- half-step B (Alg. 1 l.6-7): p = X v_j - alpha_j u_j; FRO vs U_j ----
      lap(7);
      const double aj = al;
      correlate_cta(
          fbuf, sh, tw, spec, K, L, [&](int i) { return sm.bufV[i]; },
          [&](int t, double y) { sm.bufU[t] = y - aj * sm.bufU[t]; });
      __syncthreads();
      ss = 0.0;
      for (int t = tid; t < L; t += blockDim.x) ss = fma(sm.bufU[t], sm.bufU[t], ss);
      nr = sqrt(block_sum(ss, sm.red));
      lap(0);
      bool do_ro_u = !pro || force_u;
      if (pro && nr > 0.0) do_ro_u = (pro_update_mu(sm, j, nr, aj, runmax) > a.pro_eta) || force_u;
      double be = nr;
      if (do_ro_u) {
        const int e0 = extra;
        be = reorth(sm.bufU, U, j, a.ldL, nr, pro ? 1 : a.reorth_mode, sm, rg, part, pstride, extra);
        rows_u += 2 * j * (1 + extra - e0);
        ++rsteps;
        if (pro) pro_reset(sm.mu, j);
        force_u = pro && !force_u;
      } else {
        force_u = false;
      }
      if (!(be > 1e-12 * runmax) || be == 0.0) {
        if (!breakdown) breakdown = j;
        double q = (j < L) ? restart_vector(sm.bufU, L, a.ldL, U, j, a.seed, (uint64_t)(b + a.series_base),
                                            ((uint64_t)(++restarts) << 40), sm, rg, part, pstride)
                           : 0.0;
        if (q > 1e-8) {
          ss = 0.0;
          for (int t = tid; t < L; t += blockDim.x) ss = fma(sm.bufU[t], sm.bufU[t], ss);
          double nn = sqrt(block_sum(ss, sm.red));
          normalize_store(sm.bufU, L, a.ldL, 1.0 / nn, U + (size_t)j * a.ldL);
        } else {
          normalize_store(sm.bufU, L, a.ldL, 0.0, U + (size_t)j * a.ldL);
        }
        be = 0.0;
        if (pro) pro_reset(sm.mu, j);
      } else {
        normalize_store(sm.bufU, L, a.ldL, 1.0 / be, U + (size_t)j * a.ldL);
      }
      if (tid == 0) {
        sm.beta[j + 1] = be;
        sm.mu[j + 1] = 1.0;
      }
      bcur = be;
      runmax = fmax(runmax, be);
      lap(1);
    }
    lap(7);
    // ---- final bidiagonal SVD right here (north star (b), tgk_final): it overlaps the
    // other CTAs' basis streaming; near-degenerate cases are left to the SVD kernel ----
    int fused = 0;
    if (a.svd_method == 0) {
      const int n = 2 * m + 1;
      __syncthreads();
      for (int i = tid; i < n - 1; i += blockDim.x) {
        double v = (i & 1) ? sm.beta[(i >> 1) + 2] : sm.alpha[(i >> 1) + 1];
        tc[i] = v;
        tc2[i] = v * v;
      }
      __syncthreads();
      double* om = sm.chk;
      double* res = om + k;
      double* lohi = res + k;
      double* tc2n = tc2 + (2 * a.m_max + 2);
      double* dsc = tc2n + (2 * a.m_max + 2);
      const int kg = tgk_group(a, n);
      double* cP = a.coef + (size_t)bl * 2 * (a.m_max + 2) * k;
      double* cQ = cP + (size_t)(a.m_max + 2) * k;
      // the cluster Gram-Schmidt works on a shared-memory copy when (2m+1) k doubles fit
      const long long avail = (long long)(lanczos_regionA_bytes(a.H, a.ldL, a.ldK, a.m_max) / 8) - 3LL * (2 * a.m_max + 2);
      double* stage = ((long long)n * k <= avail) ? dsc : nullptr;
      fused = tgk_final(tc, tc2, tc2n, m, k, sm.alpha[m + 1], om, lohi, res, dsc, cP, cQ, sm.cl, kg, stage);
      if (fused) {
        if (tid < k) a.sigma[(size_t)b * k + tid] = om[tid];
        if (tid == 0) {
          double mr = 0.0;
          for (int i = 0; i < k; ++i) mr = fmax(mr, res[i]);
          const double fres = om[0] > 0.0 ? mr / om[0] : 0.0;
          ssa_series_info inf;
          inf.steps = m;
          inf.converged = converged;
          inf.breakdown_step = breakdown;
          inf.reorth_extra = extra;
          inf.restarts = restarts;
          inf.rows_u = rows_u;
          inf.rows_v = rows_v;
          inf.reorth_steps = rsteps;
          inf.reserved = 0;
          inf.status = fres <= a.tol ? SSA_OK : SSA_ERR_NOT_CONVERGED;
          inf.max_residual = fres;
          inf.sigma1 = om[0];
          a.info[b] = inf;
        }
      }
      lap(6);
    }
    // ---- publish B_m and the step count for the SVD kernel ----
    __syncthreads();
    for (int i = tid; i <= m + 2 && i < a.m_max + 3; i += blockDim.x) {
      abg[i] = sm.alpha[i];
      abg[a.m_max + 3 + i] = sm.beta[i];
    }
    if (tid == 0) {
      st[0] = m; st[1] = converged; st[2] = breakdown; st[3] = extra; st[4] = restarts; st[5] = 0; st[6] = checks;
      st[7] = fused; st[8] = rows_u; st[9] = rows_v; st[10] = rsteps; st[11] = 0;
      pc[3] += (unsigned long long)checks;  // profile slot 3: number of convergence tests
    }
  }
  if (a.prof && tid == 0)
    for (int i = 0; i < 8; ++i) atomicAdd(a.prof + i, pc[i]);
}

}  // namespace ssa

#include "lanczos_trl.cuh"

namespace ssa {

cudaError_t lanczos_set_attributes(size_t smem) {
  cudaError_t e = raise_smem_limit(lanczos_kernel, (int)smem);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(lanczos_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                             cudaSharedmemCarveoutMaxShared);
  if (e == cudaSuccess) e = raise_smem_limit(lanczos_trl_kernel, (int)smem);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(lanczos_trl_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                             cudaSharedmemCarveoutMaxShared);
  return e;
}

cudaError_t launch_lanczos(const Plan& p, const DecomposeArgs& a, cudaStream_t s) {
  int grid = p.lanczos_slots < a.nb ? p.lanczos_slots : a.nb;
  if (a.trl_d > 0)
    lanczos_trl_kernel<<<grid, kThreads, p.smem_lanczos, s>>>(a);
  else
    lanczos_kernel<<<grid, kThreads, p.smem_lanczos, s>>>(a);
  return cudaGetLastError();
}

}  // namespace ssa
