// ssa_svd.cu -- the small projected bidiagonal SVD (north star (b)) and the Ritz assembly.
//
//  bidiag_svd_tgk_kernel (default) one CTA per series: TGK multisection + inverse
//                     iteration (tgk.cuh).
//  bidiag_svd_kernel  (option) one warp per series (persistent): implicit-shift QR SVD of the
//                     (m+1) x m lower bidiagonal B_m by lane 0
//                     with every rotation recorded; then P_k, Q_k columns of the k largest
//                     singular values are formed by 2k lanes applying the records in
//                     reverse to unit vectors (bidiag_qr.cuh).  Writes sigma, the Ritz
//                     coefficients and the final residual alpha_{m+1} |P_{m+1,i}| (Eq. 2).
//  ritz_kernel        one CTA per series (persistent): U_k = U_{m+1} P_k, V_k = V_m Q_k
//                     (Eq. 1) streaming each basis once more through
//                     the per-warp TMA rings, then sign canonicalization (largest-|.| entry
//                     of u_i positive, R12).
#include "bidiag_qr.cuh"
#include "device_common.cuh"
#include "tgk.cuh"

namespace ssa {

constexpr int kSvdWarps = kSvdWarpsPerCta;

__global__ void __launch_bounds__(kSvdWarps * 32) bidiag_svd_kernel(const DecomposeArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wslot = blockIdx.x * kSvdWarps + warp;
  if (wslot >= a.svd_slots) return;  // scratch exists for svd_slots warps only
  const int mstride = a.m_max + 2;
  double* d = reinterpret_cast<double*>(smem_raw) + (size_t)warp * (3 * mstride + 2 * kMaxK);
  double* e = d + mstride;
  double* wv = e + mstride;
  double* om = wv + mstride;
  int* sel = reinterpret_cast<int*>(om + kMaxK);
  double* rbase = a.rot + (size_t)wslot * 6 * a.rot_cap;
  int2* abL = reinterpret_cast<int2*>(rbase);
  double2* csL = reinterpret_cast<double2*>(rbase + a.rot_cap);
  int2* abR = reinterpret_cast<int2*>(rbase + 3 * (size_t)a.rot_cap);
  double2* csR = reinterpret_cast<double2*>(rbase + 4 * (size_t)a.rot_cap);
  const int k = a.k, k2 = 2 * a.k;
  double* vec = a.vecs + (size_t)wslot * k2 * mstride;  // vec[row * 2k + t]
  unsigned long long cq = 0, ca = 0;
  while (true) {
    int bl = 0;
    if (lane == 0) bl = atomicAdd(a.counters + 1, 1);
    bl = __shfl_sync(0xffffffffu, bl, 0);
    if (bl >= a.nb) break;
    const int b = a.b0 + bl;
    const int* st = a.state + (size_t)bl * kStateInts;
    const int m = st[0];
    const double* alpha = a.ab + (size_t)bl * 2 * (a.m_max + 3);
    const double* beta = alpha + (a.m_max + 3);
    if (st[5]) {  // non-finite series
      if (lane < k) a.sigma[(size_t)b * k + lane] = __longlong_as_double(0x7ff8000000000000ll);
      if (lane == 0) {
        ssa_series_info inf = {};
        inf.status = SSA_ERR_INVALID_ARGUMENT;
        a.info[b] = inf;
      }
      continue;
    }
    if (st[7]) continue;  // the Lanczos kernel already did the final SVD (thick restart)
    long long t0 = clock64();
    int nL = 0, nR = 0, it = 0;
    double fres = 0.0;
    if (lane == 0) {
      RotRec rl{abL, csL, a.rot_cap, 0}, rr{abR, csR, a.rot_cap, 0};
      it = bidiag_qr<true, true>(m, alpha, beta, d, e, wv, &rl, &rr, 30 * m + 100);
      select_topk(m, d, k, sel, om);
      double mr = 0.0;
      for (int i = 0; i < k; ++i)
        if (sel[i] >= 0) mr = fmax(mr, alpha[m + 1] * fabs(wv[sel[i]]));
      fres = (om[0] > 0.0) ? mr / om[0] : 0.0;
      nL = rl.n;
      nR = rr.n;
      if (it < 0 || nL > a.rot_cap || nR > a.rot_cap) nL = -1;
    }
    __syncwarp();
    long long t1 = clock64();
    nL = __shfl_sync(0xffffffffu, nL, 0);
    nR = __shfl_sync(0xffffffffu, nR, 0);
    const bool ok = nL >= 0;
    // columns of P (length m+1) and Q (length m): one lane per column
    for (int t = lane; t < k2; t += 32) {
      const bool isP = t < k;
      const int i = isP ? t : t - k;
      const int len = isP ? m + 1 : m;
      for (int r = 0; r < len; ++r) vec[(size_t)r * k2 + t] = 0.0;
      const int si = sel[i];
      if (si >= 0 && ok) {
        vec[(size_t)si * k2 + t] = 1.0;
        if (isP) apply_records_reverse(abL, csL, nL, vec + t, k2);
        else apply_records_reverse(abR, csR, nR, vec + t, k2);
        if (!isP && d[si] < 0.0)
          for (int r = 0; r < len; ++r) vec[(size_t)r * k2 + t] = -vec[(size_t)r * k2 + t];
      }
    }
    __syncwarp();
    // Ritz coefficients [2][m_max+2][k]
    double* cP = a.coef + (size_t)bl * 2 * mstride * k;
    double* cQ = cP + (size_t)mstride * k;
    for (int idx = lane; idx < (m + 1) * k; idx += 32) {
      int r = idx / k, i = idx - r * k;
      cP[idx] = vec[(size_t)r * k2 + i];
      cQ[idx] = (r < m) ? vec[(size_t)r * k2 + k + i] : 0.0;
    }
    if (lane < k) a.sigma[(size_t)b * k + lane] = om[lane];
    if (lane == 0) {
      ssa_series_info inf;
      inf.steps = m;
      inf.converged = st[1];
      inf.breakdown_step = st[2];
      inf.reorth_extra = st[3];
      inf.restarts = st[4];
      inf.rows_u = st[8];
      inf.rows_v = st[9];
      inf.reorth_steps = st[10];
      inf.reserved = 0;
      inf.status = !ok ? SSA_ERR_INTERNAL : (fres <= a.tol ? SSA_OK : SSA_ERR_NOT_CONVERGED);
      inf.max_residual = fres;
      inf.sigma1 = om[0];
      a.info[b] = inf;
    }
    __syncwarp();
    long long t2 = clock64();
    cq += (unsigned long long)(t1 - t0);
    ca += (unsigned long long)(t2 - t1);
  }
  if (a.prof && lane == 0) {
    atomicAdd(a.prof + 7, cq + ca);  // slots 3-5 belong to the Lanczos kernel
  }
}

// Default final SVD: one CTA per series (persistent).  sigma = k largest eigenvalues of
// TGK(B_m) by multisection; P_k, Q_k from TGK eigenvectors by inverse iteration
// (tgk.cuh); residual alpha_{m+1} |P_{m+1,i}| (Eq. 2) reported in info.
__global__ void __launch_bounds__(kThreads) bidiag_svd_tgk_kernel(const DecomposeArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int tid = threadIdx.x;
  const int nmax = 2 * a.m_max + 1;
  double* c = reinterpret_cast<double*>(smem_raw);
  double* c2 = c + nmax;
  double* c2n = c2 + nmax;
  double* lohi = c2n + nmax;
  double* lam = lohi + 2 * kMaxK;
  double* red = lam + kMaxK;
  int* cl = reinterpret_cast<int*>(red + 2 * kMaxK);
  __shared__ int sb;
  const int k = a.k;
  double* Z = a.tgkw + a.tgkw_stride * blockIdx.x;
  double* W = Z + (size_t)nmax * k;
  int* ipv = reinterpret_cast<int*>(W + (size_t)5 * nmax * k);
  const int mstride = a.m_max + 2;
  long long tvals = 0, tvecs = 0;
  while (true) {
    __syncthreads();
    if (tid == 0) sb = atomicAdd(a.counters + 1, 1);
    __syncthreads();
    const int bl = sb;
    if (bl >= a.nb) break;
    const int b = a.b0 + bl;
    const int* st = a.state + (size_t)bl * kStateInts;
    const int m = st[0];
    const double* alpha = a.ab + (size_t)bl * 2 * (a.m_max + 3);
    const double* beta = alpha + (a.m_max + 3);
    if (st[5]) {  // non-finite series
      if (tid < k) a.sigma[(size_t)b * k + tid] = __longlong_as_double(0x7ff8000000000000ll);
      if (tid == 0) {
        ssa_series_info inf = {};
        inf.status = SSA_ERR_INVALID_ARGUMENT;
        a.info[b] = inf;
      }
      continue;
    }
    if (st[7]) continue;  // the Lanczos kernel already did the final SVD of this series
    const int n = 2 * m + 1;
    for (int i = tid; i < n - 1; i += blockDim.x) {
      double v = (i & 1) ? beta[(i >> 1) + 2] : alpha[(i >> 1) + 1];
      c[i] = v;
      c2[i] = v * v;
    }
    __syncthreads();
    const double anext = alpha[m + 1];
    double* cP = a.coef + (size_t)bl * 2 * mstride * k;
    double* cQ = cP + (size_t)mstride * k;
    long long ta = clock64();
    // twisted-factorization vectors (tgk.cuh); inverse iteration only for near-degenerate
    // values
    const int done = tgk_final(c, c2, c2n, m, k, anext, lam, lohi, red, Z, cP, cQ, cl);
    long long tb = clock64();
    tvals += tb - ta;
    if (!done) {
      const TgkNorms nrm = tgk_norms(c, c2, n);
      tgk_vectors(c, n, k, lam, nrm, Z, W, ipv, a.seed ^ ((unsigned long long)(b + a.series_base) << 20), cl);
      // split z = (p1, q1, p2, ..., q_m, p_{m+1}) into unit p (m+1) and q (m)
      if (tid < k) {
        const int j = tid;
        double sp = 0.0, sq = 0.0;
        for (int r = 0; r <= m; ++r) { double v = Z[(size_t)(2 * r) * k + j]; sp = fma(v, v, sp); }
        for (int r = 0; r < m; ++r) { double v = Z[(size_t)(2 * r + 1) * k + j]; sq = fma(v, v, sq); }
        const double ip = sp > 0.0 ? 1.0 / sqrt(sp) : 0.0, iq = sq > 0.0 ? 1.0 / sqrt(sq) : 0.0;
        red[j] = anext * fabs(Z[(size_t)(2 * m) * k + j]) * ip;
        red[kMaxK + j] = ip;
        lohi[j] = iq;
      }
      __syncthreads();
      for (int idx = tid; idx < (m + 1) * k; idx += blockDim.x) {
        const int r = idx / k, j = idx - r * k;
        cP[idx] = Z[(size_t)(2 * r) * k + j] * red[kMaxK + j];
        cQ[idx] = (r < m) ? Z[(size_t)(2 * r + 1) * k + j] * lohi[j] : 0.0;
      }
      __syncthreads();
      // inside a cluster the p- and q-halves of orthonormal TGK vectors are only orthogonal
      // to O(eps |T| / gap): re-orthonormalize each half (one warp per cluster)
      {
        const int w = tid >> 5, nw = blockDim.x >> 5;
        for (int q = w; q < cl[kClCount]; q += nw) {
          if (cl[q + 1] - cl[q] < 2) continue;
          warp_mgs_cols(cP, m + 1, k, 1, cl[q], cl[q + 1]);
          warp_mgs_cols(cQ, m, k, 1, cl[q], cl[q + 1]);
        }
      }
      __syncthreads();
      tvecs += clock64() - tb;
    }
    if (tid < k) a.sigma[(size_t)b * k + tid] = lam[tid];
    if (tid == 0) {
      double mr = 0.0;
      for (int j = 0; j < k; ++j) mr = fmax(mr, red[j]);
      const double fres = lam[0] > 0.0 ? mr / lam[0] : 0.0;
      ssa_series_info inf;
      inf.steps = m;
      inf.converged = st[1];
      inf.breakdown_step = st[2];
      inf.reorth_extra = st[3];
      inf.restarts = st[4];
      inf.rows_u = st[8];
      inf.rows_v = st[9];
      inf.reorth_steps = st[10];
      inf.reserved = 0;
      inf.status = fres <= a.tol ? SSA_OK : SSA_ERR_NOT_CONVERGED;
      inf.max_residual = fres;
      inf.sigma1 = lam[0];
      a.info[b] = inf;
    }
  }
  if (a.prof && tid == 0) {
    atomicAdd(a.prof + 7, (unsigned long long)(tvals + tvecs));  // slots 3-5 belong to the Lanczos kernel
  }
}

size_t tgk_svd_smem_bytes(int m_max) {
  return (size_t)(3 * (2 * m_max + 1) + 2 * kMaxK + kMaxK + 2 * kMaxK) * 8 + kClInts * 4 + 16;
}

// Ritz assembly U_k = U_{m+1} P_k, V_k = V_m Q_k (Eq. (1)): a dense
// contraction of the basis (rows) with the coefficient block (16 triples at a time) that
// reads every basis element once, on the fp64 tensor cores (mma.sync m8n8k4 f64: M =
// triples (two 8-row tiles), N = elements, K = basis rows).  Each CTA takes one series at
// a time from the work queue; for each side and 16-triple block, each warp owns 8 kRzNt
// consecutive elements of a 64 kRzNt-element window; per k-step of 4 rows a lane loads
// kRzNt basis values (row 4 ks + (lane & 3), elements 8 j + (lane >> 2)) and reads its two
// A fragments from the coefficient block, staged in fragment order ([k-step][tile][lane]).
constexpr int kRzNt = 8;                    // 8-element N tiles per warp
constexpr int kRzSpan = kWarps * 8 * kRzNt;  // elements per CTA window (512)
constexpr int kRzU = 2;                      // k-steps per load group (16 loads in flight)

size_t ritz_smem_bytes(int ldL, int ldK, int k, int m_max) {
  (void)ldL; (void)ldK; (void)k;
  size_t s = (size_t)((m_max + 2 + 3) / 4) * 64 * 8;
  s += (size_t)kWarps * kMaxK * (8 + 4) + kMaxK * 8;
  return align16(s) + 16;
}

__global__ void __launch_bounds__(kThreads, 2) ritz_kernel(const DecomposeArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  double* scoef = reinterpret_cast<double*>(smem_raw);                 // [k-steps][2][32]
  double* mxv = scoef + (size_t)((a.m_max + 2 + 3) / 4) * 64;           // [kWarps][kMaxK]
  double* sgn = mxv + kWarps * kMaxK;                                  // [kMaxK]
  int* mxi = reinterpret_cast<int*>(sgn + kMaxK);                      // [kWarps][kMaxK]
  __shared__ int sb;
  const int L = a.L, K = a.K, k = a.k;
  const int mstride = a.m_max + 2;
  unsigned long long t0 = clock64();
  while (true) {
    __syncthreads();
    if (tid == 0) sb = atomicAdd(a.counters + 2, 1);
    __syncthreads();
    const int bl = sb;
    if (bl >= a.nb) break;
    const int b = a.b0 + bl;
    const int* st = a.state + (size_t)bl * kStateInts;
    if (st[5]) continue;
    const int m = st[0];
    const double* cP = a.coef + (size_t)bl * 2 * mstride * k;
    for (int side = 0; side < 2; ++side) {
      const bool isU = side == 0;
      // U rows: m + 1 (B_m of Alg. 1), or st[11] after a thick restart (lanczos_trl.cuh)
      const int n = isU ? L : K, ld = isU ? a.ldL : a.ldK, rows = isU ? (st[11] > 0 ? st[11] : m + 1) : m;
      const double* basis = isU ? a.U + (size_t)bl * (a.m_max + 1) * a.ldL : a.V + (size_t)bl * (a.m_max + 1) * a.ldK;
      const double* coef = cP + (isU ? 0 : (size_t)mstride * k);
      double* out = (isU ? a.Uout : a.Vout) + (size_t)b * k * n;
      const int nks = (rows + 3) >> 2, g = lane >> 2, q = lane & 3;
      for (int i0 = 0; i0 < k; i0 += 16) {
        const int ki = (k - i0) < 16 ? (k - i0) : 16;
        __syncthreads();
        for (int idx = tid; idx < nks * 64; idx += blockDim.x) {
          const int ks = idx >> 6, mt = (idx >> 5) & 1, l = idx & 31;
          const int r = 4 * ks + (l & 3), i = 8 * mt + (l >> 2);
          scoef[idx] = (r < rows && i < ki) ? __ldg(coef + (size_t)r * k + i0 + i) : 0.0;
        }
        __syncthreads();
        // U side: running argmax |u_i| of this lane's triples 8 mt + g over its elements, in
        // increasing element order (sign canonicalization, R12)
        double bmax[2] = {-1.0, -1.0};
        int bidx[2] = {0x7fffffff, 0x7fffffff};
        for (int c0 = 0; c0 < n; c0 += kRzSpan) {
          const int tw0 = c0 + w * 8 * kRzNt;  // the warp's first element
          if (tw0 >= n) continue;               // no barrier below: idle warps may leave
          double acc[2][kRzNt][2];
#pragma unroll
          for (int mt = 0; mt < 2; ++mt)
#pragma unroll
            for (int jn = 0; jn < kRzNt; ++jn) acc[mt][jn][0] = acc[mt][jn][1] = 0.0;
          const double* bq = basis + (size_t)q * ld + tw0 + g;
          // kRzU k-steps per group: all kRzU kRzNt basis loads issued, then the MMAs
          for (int ks0 = 0; ks0 < nks; ks0 += kRzU) {
            double bv[kRzU][kRzNt];
#pragma unroll
            for (int u = 0; u < kRzU; ++u) {
              const int r = 4 * (ks0 + u) + q;
              const double* bp = bq + (size_t)(4 * (ks0 + u)) * ld;
#pragma unroll
              for (int jn = 0; jn < kRzNt; ++jn)
                bv[u][jn] = (r < rows && tw0 + 8 * jn + g < n) ? ldg_stream(bp + 8 * jn) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < kRzU; ++u) {
              const int ks = ks0 + u < nks ? ks0 + u : nks - 1;  // beyond nks: zero B, any A
              const double a0 = scoef[ks * 64 + lane], a1 = scoef[ks * 64 + 32 + lane];
#pragma unroll
              for (int jn = 0; jn < kRzNt; ++jn) {
                dmma_m8n8k4(acc[0][jn][0], acc[0][jn][1], a0, bv[u][jn]);
                dmma_m8n8k4(acc[1][jn][0], acc[1][jn][1], a1, bv[u][jn]);
              }
            }
          }
          if (isU) {
#pragma unroll
            for (int mt = 0; mt < 2; ++mt)
#pragma unroll
              for (int jn = 0; jn < kRzNt; ++jn)
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                  const int t = tw0 + 8 * jn + 2 * q + c;
                  const double av = fabs(acc[mt][jn][c]);
                  if (t < n && av > bmax[mt]) { bmax[mt] = av; bidx[mt] = t; }
                }
          }
          // D fragment: triple i0 + 8 mt + g, elements tw0 + 8 jn + 2 q + {0, 1}
#pragma unroll
          for (int mt = 0; mt < 2; ++mt) {
            const int i = 8 * mt + g;
            if (i < ki) {
              double* o = out + (size_t)(i0 + i) * n;
              const double sg = isU ? 1.0 : sgn[i0 + i];  // V side: sign of u_i known
#pragma unroll
              for (int jn = 0; jn < kRzNt; ++jn) {
                const int t = tw0 + 8 * jn + 2 * q;
                const double y0 = sg * acc[mt][jn][0], y1 = sg * acc[mt][jn][1];
                if (t + 1 < n && ((reinterpret_cast<uintptr_t>(o + t) & 15) == 0)) {
                  *reinterpret_cast<double2*>(o + t) = make_double2(y0, y1);
                } else {
                  if (t < n) o[t] = y0;
                  if (t + 1 < n) o[t + 1] = y1;
                }
              }
            }
          }
        }
        if (isU) {  // the four lanes of a triple, then one entry per warp
#pragma unroll
          for (int mt = 0; mt < 2; ++mt) {
            double v = bmax[mt];
            int ix = bidx[mt];
            for (int o = 1; o < 4; o <<= 1) {
              const double v2 = __shfl_xor_sync(0xffffffffu, v, o);
              const int i2 = __shfl_xor_sync(0xffffffffu, ix, o);
              if (v2 > v || (v2 == v && i2 < ix)) { v = v2; ix = i2; }
            }
            if (q == 0 && 8 * mt + g < ki) { mxv[w * kMaxK + i0 + 8 * mt + g] = v; mxi[w * kMaxK + i0 + 8 * mt + g] = ix; }
          }
        }
      }
      if (isU) {
        // sign canonicalization (R12): largest-|.| entry of each u_i (lowest
        // index on ties) from the per-warp candidates of the U contraction; the V side
        // that follows stores v_i with the sign applied
        __syncthreads();
        if (tid < k) {
          double v = -1.0;
          int ix = 0;
          for (int qq = 0; qq < kWarps; ++qq) {
            double v2 = mxv[qq * kMaxK + tid];
            int i2 = mxi[qq * kMaxK + tid];
            if (v2 > v || (v2 == v && i2 < ix)) { v = v2; ix = i2; }
          }
          const double* uo = a.Uout + ((size_t)b * k + tid) * L;
          sgn[tid] = (uo[ix] < 0.0) ? -1.0 : 1.0;
        }
        __syncthreads();
      }
    }
    for (int i = 0; i < k; ++i) {  // flip the u_i of negative sign (L2-resident rows)
      if (sgn[i] < 0.0) {
        double* uo = a.Uout + ((size_t)b * k + i) * L;
        for (int t = tid; t < L; t += blockDim.x) uo[t] = -uo[t];
      }
    }
  }
  if (a.prof && tid == 0) atomicAdd(a.prof + 7, (unsigned long long)(clock64() - t0));
}

static size_t svd_smem_bytes(int m_max) { return (size_t)kSvdWarps * ((3 * (m_max + 2) + 2 * kMaxK) * 8); }

cudaError_t svd_ritz_set_attributes(int m_max, size_t smem_ritz) {
  cudaError_t e;
  if ((e = raise_smem_limit(ritz_kernel, (int)smem_ritz))) return e;
  if ((e = raise_smem_limit(bidiag_svd_kernel, (int)svd_smem_bytes(m_max))))
    return e;
  if ((e = raise_smem_limit(bidiag_svd_tgk_kernel, (int)tgk_svd_smem_bytes(m_max))))
    return e;
  return cudaSuccess;
}

cudaError_t launch_bidiag_svd(const Plan& p, const DecomposeArgs& a, cudaStream_t s) {
  if (a.svd_method == 0) {
    int grid = p.tgk_slots < a.nb ? p.tgk_slots : a.nb;
    bidiag_svd_tgk_kernel<<<grid, kThreads, tgk_svd_smem_bytes(a.m_max), s>>>(a);
  } else {
    int grid = (a.svd_slots + kSvdWarps - 1) / kSvdWarps;
    bidiag_svd_kernel<<<grid, kSvdWarps * 32, svd_smem_bytes(a.m_max), s>>>(a);
  }
  return cudaGetLastError();
}

cudaError_t launch_ritz(const Plan& p, const DecomposeArgs& a, cudaStream_t s) {
  int grid = p.ritz_slots < a.nb ? p.ritz_slots : a.nb;
  ritz_kernel<<<grid, kThreads, p.smem_ritz, s>>>(a);
  return cudaGetLastError();
}

}  // namespace ssa
