// ssa_kernels.cu -- sm_100a kernels of the fast Basic-SSA hot path (arXiv:0911.4498).
//
//  spectrum_kernel   F^ = rfft(f, M)                     Alg. 2 l.1-2
//  matvec_kernel     y = X x / X^T x by FFT correlation  Alg. 2/3
//  hankelize_kernel  g = sigma irfft(rfft u rfft v) / c  sec 5, Alg. 4
//  lanczos_kernel    persistent per-series GKL + FRO + bidiagonal SVD + Ritz assembly
//                    Alg. 1, FRO PAPER.md:388-393, Eqs. (1)-(2) 323-328
//
// Correlation form (R1): with F^ = rfft(f, M) for any M >= N,
//   (X v)_i   = sum_j f_{i+j} v_j = irfft(F^ conj(rfft(v, M)))[i],  i < L
//   (X^T u)_j = sum_i f_{i+j} u_i = irfft(F^ conj(rfft(u, M)))[j],  j < K
// which is Alg. 2 / Alg. 3 (circulant embedding + backward identity) with the reversal
// folded into the conjugate and the output slice of Alg. 3 read as p'_L..p'_N.
#include <cuda_runtime.h>
#include <stdint.h>

#include "bidiag_qr.cuh"
#include "fft_smem.cuh"
#include "ssa_internal.h"

namespace ssa {

// ------------------------------------------------------------------ reductions
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic CTA sum: fixed shuffle tree, then warps summed in index order.
__device__ __forceinline__ double block_sum(double v, double* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  const int nw = blockDim.x >> 5;
  for (int i = 0; i < nw; ++i) s += red[i];
  return s;
}

__device__ __forceinline__ int block_or(int v, int* redi) {
  __syncthreads();
  if (threadIdx.x == 0) *redi = 0;
  __syncthreads();
  if (v) atomicOr(redi, 1);
  __syncthreads();
  return *redi;
}

// ------------------------------------------------------------------ FFT pair steps
// Forward real post-processing for the pair (p, H-p) from digit-reversed Z.
__device__ __forceinline__ void real_pair(const double2* buf, const FftShape& sh, const double2* __restrict__ T,
                                          int p, double2& Xp, double2& Xq, int& pr, int& qr) {
  const int H = sh.H;
  const int q = (H - p) & (H - 1);
  pr = rev_index(sh, p);
  qr = rev_index(sh, q);
  double2 Zp = buf[fpad(pr)], Zq = buf[fpad(qr)];
  double2 W = twiddle(T, p, H);
  double2 E = make_double2(0.5 * (Zp.x + Zq.x), 0.5 * (Zp.y - Zq.y));
  double2 D = make_double2(0.5 * (Zp.x - Zq.x), 0.5 * (Zp.y + Zq.y));
  double2 O = make_double2(D.y, -D.x);  // -i D
  double2 WO = cmul(W, O);
  Xp = cadd(E, WO);
  Xq = conjg(csub(E, WO));
}

// Inverse pre-processing: from half-spectrum values Y_p, Y_{H-p} produce Z'_p, Z'_{H-p}.
__device__ __forceinline__ void inv_pair(double2* buf, const double2* __restrict__ T, int H, int p, int pr, int qr,
                                         double2 Yp, double2 Yq) {
  double2 W = twiddle(T, p, H);
  double2 E = make_double2(0.5 * (Yp.x + Yq.x), 0.5 * (Yp.y - Yq.y));
  double2 D = make_double2(0.5 * (Yp.x - Yq.x), 0.5 * (Yp.y + Yq.y));
  double2 O = cmulc(D, W);
  buf[fpad(pr)] = make_double2(E.x - O.y, E.y + O.x);
  if (qr != pr) buf[fpad(qr)] = make_double2(E.x + O.y, O.x - E.y);
}

// Correlation spectrum step: Z (digit-reversed FFT of packed x) -> Z' whose inverse is
// the packed correlation y = irfft(F^ conj(X^)).
__device__ __forceinline__ void corr_pairs(double2* buf, const FftShape& sh, const double2* __restrict__ T,
                                           const double2* __restrict__ spec, int tid, int nthr) {
  const int H = sh.H;
  for (int p = tid; p <= (H >> 1); p += nthr) {
    double2 Xp, Xq;
    int pr, qr;
    real_pair(buf, sh, T, p, Xp, Xq, pr, qr);
    double2 Fp = __ldg(spec + p), Fq = __ldg(spec + (H - p));
    inv_pair(buf, T, H, p, pr, qr, cmulc(Fp, Xp), cmulc(Fq, Xq));
  }
}

// Full correlation in one CTA (all threads): y_t = sum_s f_{t+s} x_s, t < n_out.
template <class LoadX, class StoreY>
__device__ __forceinline__ void correlate_cta(double2* buf, const FftShape& sh, const double2* __restrict__ T,
                                              const double2* __restrict__ spec, int n_in, int n_out, LoadX loadx,
                                              StoreY storey) {
  const int H = sh.H, tid = threadIdx.x, nthr = blockDim.x;
  for (int n = tid; n < H; n += nthr) {
    int i0 = 2 * n;
    double a = (i0 < n_in) ? loadx(i0) : 0.0;
    double b = (i0 + 1 < n_in) ? loadx(i0 + 1) : 0.0;
    buf[fpad(n)] = make_double2(a, b);
  }
  __syncthreads();
  fft_forward(buf, sh, T, tid, nthr, CtaSync());
  corr_pairs(buf, sh, T, spec, tid, nthr);
  __syncthreads();
  fft_inverse(buf, sh, T, tid, nthr, CtaSync());
  const double invH = 1.0 / (double)H;
  for (int t = tid; t < n_out; t += nthr) {
    double2 z = buf[fpad(t >> 1)];
    storey(t, ((t & 1) ? z.y : z.x) * invH);
  }
}

// ------------------------------------------------------------------ spectrum / matvec
__global__ void __launch_bounds__(kThreads) spectrum_kernel(const double* __restrict__ series, int N, int H,
                                                            const double2* __restrict__ T, double2* __restrict__ spec) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* buf = reinterpret_cast<double2*>(smem_raw);
  const FftShape sh = make_shape(H);
  const int b = blockIdx.x;
  const double* f = series + (size_t)b * N;
  double2* out = spec + (size_t)b * (H + 1);
  for (int n = threadIdx.x; n < H; n += blockDim.x) {
    int i0 = 2 * n;
    double a = (i0 < N) ? f[i0] : 0.0;
    double c = (i0 + 1 < N) ? f[i0 + 1] : 0.0;
    buf[fpad(n)] = make_double2(a, c);
  }
  __syncthreads();
  fft_forward(buf, sh, T, threadIdx.x, blockDim.x, CtaSync());
  for (int p = threadIdx.x; p <= (H >> 1); p += blockDim.x) {
    double2 Xp, Xq;
    int pr, qr;
    real_pair(buf, sh, T, p, Xp, Xq, pr, qr);
    out[p] = Xp;
    out[H - p] = Xq;
  }
}

__global__ void __launch_bounds__(kThreads) matvec_kernel(const double2* __restrict__ spec, int H, int n_in, int n_out,
                                                          const double2* __restrict__ T, const double* __restrict__ x,
                                                          double* __restrict__ y) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* buf = reinterpret_cast<double2*>(smem_raw);
  const FftShape sh = make_shape(H);
  const int b = blockIdx.x;
  const double* xb = x + (size_t)b * n_in;
  double* yb = y + (size_t)b * n_out;
  correlate_cta(
      buf, sh, T, spec + (size_t)b * (H + 1), n_in, n_out, [&](int i) { return __ldg(xb + i); },
      [&](int t, double v) { yb[t] = v; });
}

// ------------------------------------------------------------------ hankelization
// g_t = sigma * (u' * v')_t / c_t, c_t = min(t, L, K, N-t+1), t = 1..N  (PAPER.md:751-785,
// Alg. 4 PAPER.md:807-824 with the weights read as division, R2).
// Two shared-memory buffers when they fit (H <= kMaxHankelSmemH); otherwise (BIG) the
// post-processed spectrum of u goes to a per-CTA global scratch row (L2-resident) and the
// grid is persistent over terms.
template <bool BIG>
__global__ void __launch_bounds__(kThreads) hankelize_kernel(const double* __restrict__ sigma,
                                                             const double* __restrict__ U,
                                                             const double* __restrict__ V, size_t nterm_total, int N,
                                                             int L, int K, int H, const double2* __restrict__ T,
                                                             double* __restrict__ out, double2* gscratch) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* bufB = reinterpret_cast<double2*>(smem_raw);
  double2* bufA = BIG ? nullptr : bufB + fpad_size(H);
  double2* Xu = BIG ? gscratch + (size_t)blockIdx.x * (H + 1) : nullptr;
  const FftShape sh = make_shape(H);
  const int mn = L < K ? L : K;
  for (size_t term = blockIdx.x; term < nterm_total; term += gridDim.x) {
    const double* u = U + term * L;
    const double* v = V + term * K;
    const double sg = __ldg(sigma + term);
    if (BIG) {
      __syncthreads();
      for (int n = threadIdx.x; n < H; n += blockDim.x) {
        int i0 = 2 * n;
        bufB[fpad(n)] = make_double2(i0 < L ? __ldg(u + i0) : 0.0, i0 + 1 < L ? __ldg(u + i0 + 1) : 0.0);
      }
      __syncthreads();
      fft_forward(bufB, sh, T, threadIdx.x, blockDim.x, CtaSync());
      for (int p = threadIdx.x; p <= (H >> 1); p += blockDim.x) {
        double2 Up, Uq;
        int pr, qr;
        real_pair(bufB, sh, T, p, Up, Uq, pr, qr);
        Xu[p] = Up;
        Xu[H - p] = Uq;
      }
      __syncthreads();
      for (int n = threadIdx.x; n < H; n += blockDim.x) {
        int i0 = 2 * n;
        bufB[fpad(n)] = make_double2(i0 < K ? __ldg(v + i0) : 0.0, i0 + 1 < K ? __ldg(v + i0 + 1) : 0.0);
      }
      __syncthreads();
      fft_forward(bufB, sh, T, threadIdx.x, blockDim.x, CtaSync());
      for (int p = threadIdx.x; p <= (H >> 1); p += blockDim.x) {
        double2 Vp, Vq;
        int pr, qr;
        real_pair(bufB, sh, T, p, Vp, Vq, pr, qr);
        inv_pair(bufB, T, H, p, pr, qr, cmul(Xu[p], Vp), cmul(Xu[H - p], Vq));
      }
    } else {
      __syncthreads();
      for (int n = threadIdx.x; n < H; n += blockDim.x) {
        int i0 = 2 * n;
        bufA[fpad(n)] = make_double2(i0 < L ? __ldg(u + i0) : 0.0, i0 + 1 < L ? __ldg(u + i0 + 1) : 0.0);
        bufB[fpad(n)] = make_double2(i0 < K ? __ldg(v + i0) : 0.0, i0 + 1 < K ? __ldg(v + i0 + 1) : 0.0);
      }
      __syncthreads();
      fft_forward(bufA, sh, T, threadIdx.x, blockDim.x, CtaSync());
      fft_forward(bufB, sh, T, threadIdx.x, blockDim.x, CtaSync());
      for (int p = threadIdx.x; p <= (H >> 1); p += blockDim.x) {
        double2 Up, Uq, Vp, Vq;
        int pr, qr;
        real_pair(bufA, sh, T, p, Up, Uq, pr, qr);
        real_pair(bufB, sh, T, p, Vp, Vq, pr, qr);
        inv_pair(bufB, T, H, p, pr, qr, cmul(Up, Vp), cmul(Uq, Vq));
      }
    }
    __syncthreads();
    fft_inverse(bufB, sh, T, threadIdx.x, blockDim.x, CtaSync());
    const double scale = sg / (double)H;
    double* g = out + term * N;
    for (int t = threadIdx.x; t < N; t += blockDim.x) {
      double2 z = bufB[fpad(t >> 1)];
      int k1 = t + 1;  // 1-based
      int c = k1;
      if (c > mn) c = mn;
      if (N - k1 + 1 < c) c = N - k1 + 1;
      g[t] = ((t & 1) ? z.y : z.x) * scale / (double)c;
    }
  }
}

// ------------------------------------------------------------------ TMA bulk streaming
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t a = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

// Per-warp ring of kStages chunks; one lane issues cp.async.bulk, all lanes consume.
struct WarpRing {
  double* buf;      // kStages * slab doubles
  uint64_t* bar;    // kStages barriers
  uint32_t cnt;     // chunks consumed so far (== issued at the end of each stream)
};

// Streams rows (q-th job = row q, or nb-1-q if reverse) of this warp's column slab
// [w*slab, (w+1)*slab) of a row-major basis (row stride ld doubles) through the ring;
// calls f(row, chunk) for each in order.
template <class F>
__device__ __forceinline__ void stream_rows(const double* base_w, int ld, int nb, bool reverse, int slab, WarpRing& rg,
                                            F f) {
  const int lane = threadIdx.x & 31;
  const uint32_t bytes = (uint32_t)slab * 8u;
  const uint32_t c0 = rg.cnt;
  auto row_of = [&](int q) { return reverse ? nb - 1 - q : q; };
  if (lane == 0) {
    int pre = nb < kStages ? nb : kStages;
    for (int q = 0; q < pre; ++q) {
      int st = (int)((c0 + q) % kStages);
      mbar_expect_tx(rg.bar + st, bytes);
      tma_load_1d(rg.buf + (size_t)st * slab, base_w + (size_t)row_of(q) * ld, bytes, rg.bar + st);
    }
  }
  for (int q = 0; q < nb; ++q) {
    const uint32_t c = c0 + q;
    const int st = (int)(c % kStages);
    mbar_wait(rg.bar + st, (c / kStages) & 1u);
    f(row_of(q), rg.buf + (size_t)st * slab);
    __syncwarp();
    if (lane == 0 && q + kStages < nb) {
      mbar_expect_tx(rg.bar + st, bytes);
      tma_load_1d(rg.buf + (size_t)st * slab, base_w + (size_t)row_of(q + kStages) * ld, bytes, rg.bar + st);
    }
  }
  rg.cnt = c0 + nb;
}

// ------------------------------------------------------------------ Lanczos kernel
struct LSmem {
  unsigned char* regionA;  // union: FFT buffer | rings + partial dots | QR work | P/Q vectors
  double* bufU;            // ldL
  double* bufV;            // ldK
  double* h;               // m_max + 2
  double* alpha;           // m_max + 3 (1-based)
  double* beta;            // m_max + 3 (1-based)
  double* red;             // 32
  int* redi;               // 8 ints
  double* om;              // 64: selected singular values (final)
  double* sgn;             // 64: sign flips
  double* mxv;             // kWarps * 32: per-warp max |u_i|
  int* sel;                // 64: selected indices
  int* mxi;                // kWarps * 32
  uint64_t* bars;          // kWarps * kStages
};
constexpr int kFinBytes = 64 * 8 * 2 + kWarps * 32 * 8 + 64 * 4 + kWarps * 32 * 4;

__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~(size_t)15; }

__host__ __device__ inline size_t regionA_bytes(int H, int ldL, int ldK, int m_max, int k) {
  int slab_max = (ldL > ldK ? ldL : ldK) / kWarps;
  size_t fft = (size_t)fpad_size(H) * 16;
  size_t rings = (size_t)kWarps * kStages * slab_max * 8 + (size_t)kWarps * (m_max + 2) * 8;
  size_t qr = (size_t)3 * (m_max + 2) * 8;                          // d, e, w
  size_t pq = (size_t)k * 2 * (m_max + 2) * 8;                        // P_k, Q_k columns
  size_t r = fft;
  if (rings > r) r = rings;
  if (qr > r) r = qr;
  if (pq + qr > r) r = pq + qr;
  return align16(r);
}

size_t lanczos_smem_bytes(int H, int ldL, int ldK, int m_max, int k) {
  size_t s = regionA_bytes(H, ldL, ldK, m_max, k);
  s += align16((size_t)ldL * 8) + align16((size_t)ldK * 8);
  s += 3 * align16((size_t)(m_max + 3) * 8);
  s += 32 * 8 + 8 * 4;
  s += kFinBytes;
  s += (size_t)kWarps * kStages * 8;
  return align16(s) + 16;
}

__device__ inline LSmem carve(unsigned char* base, const LanczosArgs& a) {
  LSmem s;
  size_t off = 0;
  s.regionA = base;
  off += regionA_bytes(a.H, a.ldL, a.ldK, a.m_max, a.k);
  s.bufU = reinterpret_cast<double*>(base + off); off += align16((size_t)a.ldL * 8);
  s.bufV = reinterpret_cast<double*>(base + off); off += align16((size_t)a.ldK * 8);
  s.h = reinterpret_cast<double*>(base + off); off += align16((size_t)(a.m_max + 3) * 8);
  s.alpha = reinterpret_cast<double*>(base + off); off += align16((size_t)(a.m_max + 3) * 8);
  s.beta = reinterpret_cast<double*>(base + off); off += align16((size_t)(a.m_max + 3) * 8);
  s.red = reinterpret_cast<double*>(base + off); off += 32 * 8;
  s.redi = reinterpret_cast<int*>(base + off); off += 8 * 4;
  s.om = reinterpret_cast<double*>(base + off); off += 64 * 8;
  s.sgn = reinterpret_cast<double*>(base + off); off += 64 * 8;
  s.mxv = reinterpret_cast<double*>(base + off); off += kWarps * 32 * 8;
  s.sel = reinterpret_cast<int*>(base + off); off += 64 * 4;
  s.mxi = reinterpret_cast<int*>(base + off); off += kWarps * 32 * 4;
  s.bars = reinterpret_cast<uint64_t*>(base + off);
  return s;
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

struct Reorth {
  // CGS pass(es) of r (SMEM, ld doubles, zero padding) against basis rows [0, nb).
  // Returns the new norm; nrm_in is |r| before.  mode 1: DGKS (second pass iff the norm
  // fell below 1/sqrt(2) of its value), mode 2: always two passes (PAPER.md:388-393,
  // DESIGN.md R9).
  __device__ static double run(double* r, const double* basis, int nb, int ld, double nrm_in, int mode,
                               const LSmem& sm, WarpRing& rg, double* part, int pstride, int& extra) {
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int slab = ld / kWarps;
    double* rw = r + w * slab;
    const double* bw = basis + (size_t)w * slab;
    double nrm = nrm_in;
    for (int pass = 0; pass < 2 && nb > 0; ++pass) {
      fence_proxy_async_smem();
      __syncthreads();
      // pass 1: partial dots of this warp's slab with every basis row
      stream_rows(bw, ld, nb, false, slab, rg, [&](int row, const double* ch) {
        double s = 0.0;
        for (int e = lane; e < slab; e += 32) s = fma(ch[e], rw[e], s);
        s = warp_sum(s);
        if (lane == 0) part[w * pstride + row] = s;
      });
      __syncthreads();
      for (int c = threadIdx.x; c < nb; c += blockDim.x) {
        double s = 0.0;
        for (int q = 0; q < kWarps; ++q) s += part[q * pstride + c];
        sm.h[c] = s;
      }
      __syncthreads();
      // pass 2: r -= V h, rows streamed in reverse so the most recently read rows (still
      // in L2) come first
      stream_rows(bw, ld, nb, true, slab, rg, [&](int row, const double* ch) {
        const double hc = sm.h[row];
        for (int e = lane; e < slab; e += 32) rw[e] = fma(-hc, ch[e], rw[e]);
      });
      double ss = 0.0;
      for (int e = lane; e < slab; e += 32) ss = fma(rw[e], rw[e], ss);
      double nn = sqrt(block_sum(ss, sm.red));
      bool again = (pass == 0) && (mode == 2 || nn < 0.70710678118654752 * nrm);
      nrm = nn;
      if (!again) break;
      ++extra;
    }
    return nrm;
  }
};

// Write normalized r into basis row `row` (plain coalesced stores), scale in place.
__device__ __forceinline__ void normalize_store(double* r, int n, int ld, double inv, double* dst) {
  for (int t = threadIdx.x; t < ld; t += blockDim.x) {
    double v = (t < n) ? r[t] * inv : 0.0;
    r[t] = v;
    dst[t] = v;
  }
  fence_proxy_async_global();
  __syncthreads();
}

// Fill r with a seeded random vector, orthogonalize twice against the basis, normalize.
// Used at a Lanczos breakdown (restart, R11).  Returns false if the norm
// after orthogonalization vanished (space exhausted).
__device__ bool restart_vector(double* r, int n, int ld, const double* basis, int nb, uint64_t seed, uint64_t series,
                               uint64_t salt, const LSmem& sm, WarpRing& rg, double* part, int pstride) {
  double ss = 0.0;
  for (int t = threadIdx.x; t < ld; t += blockDim.x) {
    double v = (t < n) ? rng_uniform_pm1(seed, series, salt + t) : 0.0;
    r[t] = v;
    ss += v * v;
  }
  double nrm = sqrt(block_sum(ss, sm.red));
  int extra = 0;
  double nn = Reorth::run(r, basis, nb, ld, nrm, 2, sm, rg, part, pstride, extra);
  return nn > 1e-10 * nrm;
}

__global__ void __launch_bounds__(kThreads, 2) lanczos_kernel(const LanczosArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  LSmem sm = carve(smem_raw, a);
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const FftShape sh = make_shape(a.H);
  const int slab_max = (a.ldL > a.ldK ? a.ldL : a.ldK) / kWarps;
  double2* fbuf = reinterpret_cast<double2*>(sm.regionA);
  double* rings = reinterpret_cast<double*>(sm.regionA);
  double* part = rings + (size_t)kWarps * kStages * slab_max;
  const int pstride = a.m_max + 2;
  // QR work arrays (aliases the rings; only used between streaming phases)
  double* qd = reinterpret_cast<double*>(sm.regionA);
  double* qe = qd + (a.m_max + 2);
  double* qw = qe + (a.m_max + 2);
  double* qom = sm.om;
  int* qsel = sm.sel;
  double* pvec = qw + (a.m_max + 2);          // k x (m_max+2)   (P columns, stride m_max+2)
  double* qvec = pvec + (size_t)a.k * (a.m_max + 2);

  WarpRing rg;
  rg.buf = rings + (size_t)w * kStages * slab_max;
  rg.bar = sm.bars + w * kStages;
  rg.cnt = 0;
  if (lane == 0)
    for (int s = 0; s < kStages; ++s) mbar_init(rg.bar + s, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();

  double* U = a.Ubase + a.slot_stride_U * blockIdx.x;
  double* V = a.Vbase + a.slot_stride_V * blockIdx.x;
  double* rotL = a.rot + a.slot_stride_rot * blockIdx.x;
  double* rotR = rotL + (size_t)3 * a.rot_cap;
  double* pq = a.pq + a.slot_stride_pq * blockIdx.x;
  const int L = a.L, K = a.K, k = a.k;

  while (true) {
    __syncthreads();
    if (tid == 0) sm.redi[4] = atomicAdd(a.counter, 1);
    __syncthreads();
    const int b = sm.redi[4];
    if (b >= a.batch) break;
    const double* f = a.series + (size_t)b * a.N;
    const double2* spec = a.spec + (size_t)b * (a.H + 1);

    // ---- non-finite input -> INVALID_ARGUMENT ----
    int bad = 0;
    for (int t = tid; t < a.N; t += blockDim.x) bad |= !isfinite(f[t]);
    if (block_or(bad, sm.redi)) {
      if (tid < k) a.sigma[(size_t)b * k + tid] = __longlong_as_double(0x7ff8000000000000ll);
      if (tid == 0) {
        ssa_series_info inf = {};
        inf.status = SSA_ERR_INVALID_ARGUMENT;
        a.info[b] = inf;
      }
      continue;
    }

    // ---- Alg. 1 lines 1-2: p0 seeded, beta_1 = |p0|, u_1 = p0 / beta_1, v_0 = 0 ----
    double ss = 0.0;
    for (int t = tid; t < a.ldL; t += blockDim.x) {
      double v = (t < L) ? rng_uniform_pm1(a.seed, (uint64_t)b, (uint64_t)t) : 0.0;
      sm.bufU[t] = v;
      ss += v * v;
    }
    for (int t = tid; t < a.ldK; t += blockDim.x) sm.bufV[t] = 0.0;
    double beta1 = sqrt(block_sum(ss, sm.red));
    if (tid == 0) { sm.beta[1] = beta1; sm.alpha[0] = 0.0; }
    normalize_store(sm.bufU, L, a.ldL, 1.0 / beta1, U);

    double runmax = 0.0;
    int m = 0, converged = 0, breakdown = 0, extra = 0, restarts = 0;
    int next_check = k;
    double prev_res = -1.0;
    int prev_m = 0;
    double max_res = 0.0;
    const int ce = a.check_every > 0 ? a.check_every : 4;

    for (int j = 1; j <= a.m_max + 1; ++j) {
      // ---- half-step A (Alg. 1 l.4-5): r = X^T u_j - beta_j v_{j-1}; FRO vs V_{j-1} ----
      const double bj = sm.beta[j];
      correlate_cta(
          fbuf, sh, a.tw, spec, L, K, [&](int i) { return sm.bufU[i]; },
          [&](int t, double y) { sm.bufV[t] = y - bj * sm.bufV[t]; });
      __syncthreads();
      ss = 0.0;
      for (int t = tid; t < K; t += blockDim.x) ss = fma(sm.bufV[t], sm.bufV[t], ss);
      double nr = sqrt(block_sum(ss, sm.red));
      double al = Reorth::run(sm.bufV, V, j - 1, a.ldK, nr, a.reorth_mode, sm, rg, part, pstride, extra);
      if (!(al > 1e-12 * runmax) || al == 0.0) {
        if (!breakdown) breakdown = j;
        bool ok = (j - 1 < K) && restart_vector(sm.bufV, K, a.ldK, V, j - 1, a.seed, (uint64_t)b,
                                                 ((uint64_t)(++restarts) << 40), sm, rg, part, pstride);
        if (ok) {
          ss = 0.0;
          for (int t = tid; t < K; t += blockDim.x) ss = fma(sm.bufV[t], sm.bufV[t], ss);
          double nn = sqrt(block_sum(ss, sm.red));
          normalize_store(sm.bufV, K, a.ldK, 1.0 / nn, V + (size_t)(j - 1) * a.ldK);
        } else {
          normalize_store(sm.bufV, K, a.ldK, 0.0, V + (size_t)(j - 1) * a.ldK);
        }
        al = 0.0;
      } else {
        normalize_store(sm.bufV, K, a.ldK, 1.0 / al, V + (size_t)(j - 1) * a.ldK);
      }
      if (tid == 0) sm.alpha[j] = al;
      runmax = fmax(runmax, al);
      m = j - 1;

      // ---- convergence test on B_m with alpha_{m+1} = al (R7) ----
      bool last = (m >= a.m_max);
      if (m >= k && (m >= next_check || last)) {
        __syncthreads();
        if (tid == 0) {
          int it = bidiag_qr<true, false>(m, sm.alpha, sm.beta, qd, qe, qw, nullptr, nullptr, 30 * m + 100);
          select_topk(m, qd, k, qsel, qom);
          double om1 = qom[0], mr = 0.0;
          for (int i = 0; i < k; ++i) {
            double res = (qsel[i] >= 0) ? al * fabs(qw[qsel[i]]) : 0.0;
            mr = fmax(mr, res);
          }
          double rel = (om1 > 0.0) ? mr / om1 : 0.0;
          sm.red[16] = rel;
          sm.redi[5] = (it >= 0) && (rel <= a.tol);
        }
        __syncthreads();
        double rel = sm.red[16];
        max_res = rel;
        if (sm.redi[5]) { converged = 1; break; }
        // schedule the next test from the observed geometric decay of the residual
        int step = ce;
        if (prev_res > 0.0 && rel < prev_res && rel > 0.0) {
          double rate = log(rel / prev_res) / (double)(m - prev_m);
          double need = log(a.tol / rel) / rate;
          int s2 = (int)(0.8 * need);
          if (s2 > step) step = s2 < 4 * ce ? s2 : 4 * ce;
        }
        prev_res = rel;
        prev_m = m;
        next_check = m + step;
      }
      if (last) break;

      // ---- half-step B (Alg. 1 l.6-7): p = X v_j - alpha_j u_j; FRO vs U_j ----
      const double aj = al;
      correlate_cta(
          fbuf, sh, a.tw, spec, K, L, [&](int i) { return sm.bufV[i]; },
          [&](int t, double y) { sm.bufU[t] = y - aj * sm.bufU[t]; });
      __syncthreads();
      ss = 0.0;
      for (int t = tid; t < L; t += blockDim.x) ss = fma(sm.bufU[t], sm.bufU[t], ss);
      nr = sqrt(block_sum(ss, sm.red));
      double be = Reorth::run(sm.bufU, U, j, a.ldL, nr, a.reorth_mode, sm, rg, part, pstride, extra);
      if (!(be > 1e-12 * runmax) || be == 0.0) {
        if (!breakdown) breakdown = j;
        bool ok = (j < L) && restart_vector(sm.bufU, L, a.ldL, U, j, a.seed, (uint64_t)b,
                                             ((uint64_t)(++restarts) << 40), sm, rg, part, pstride);
        if (ok) {
          ss = 0.0;
          for (int t = tid; t < L; t += blockDim.x) ss = fma(sm.bufU[t], sm.bufU[t], ss);
          double nn = sqrt(block_sum(ss, sm.red));
          normalize_store(sm.bufU, L, a.ldL, 1.0 / nn, U + (size_t)j * a.ldL);
        } else {
          normalize_store(sm.bufU, L, a.ldL, 0.0, U + (size_t)j * a.ldL);
        }
        be = 0.0;
      } else {
        normalize_store(sm.bufU, L, a.ldL, 1.0 / be, U + (size_t)j * a.ldL);
      }
      if (tid == 0) sm.beta[j + 1] = be;
      runmax = fmax(runmax, be);
    }

    // ---- final SVD of B_m with rotation records ----
    __syncthreads();
    if (tid == 0) {
      RotRec rl{rotL, a.rot_cap, 0}, rr{rotR, a.rot_cap, 0};
      int it = bidiag_qr<true, true>(m, sm.alpha, sm.beta, qd, qe, qw, &rl, &rr, 30 * m + 100);
      select_topk(m, qd, k, qsel, qom);
      double om1 = qom[0], mr = 0.0;
      for (int i = 0; i < k; ++i)
        if (qsel[i] >= 0) mr = fmax(mr, sm.alpha[m + 1] * fabs(qw[qsel[i]]));
      sm.red[17] = (om1 > 0.0) ? mr / om1 : 0.0;
      sm.redi[6] = rl.n;
      sm.redi[7] = rr.n;
      if (it < 0 || rl.n > a.rot_cap || rr.n > a.rot_cap) sm.redi[6] = -1;
    }
    __syncthreads();
    const int nL = sm.redi[6], nR = sm.redi[7];
    const double final_res = sm.red[17];
    const int ok_svd = nL >= 0;
    // P_k columns (length m+1) and Q_k columns (length m) from the records, one thread
    // per column; sign of d folded into Q (B = P diag(|d|) (Q diag(sign d))^T).
    const int pst = a.m_max + 2;
    if (tid < 2 * k) {
      const bool isP = tid < k;
      const int i = isP ? tid : tid - k;
      double* x = isP ? pvec + (size_t)i * pst : qvec + (size_t)i * pst;
      const int len = isP ? m + 1 : m;
      for (int t = 0; t < len; ++t) x[t] = 0.0;
      const int si = qsel[i];
      if (si >= 0 && ok_svd) {
        x[si] = 1.0;
        apply_records_reverse(isP ? rotL : rotR, isP ? nL : nR, x, 1);
        if (!isP && qd[si] < 0.0)
          for (int t = 0; t < len; ++t) x[t] = -x[t];
      }
    }
    __syncthreads();
    // stage coefficients in global scratch as [row][i] for broadcast loads in the GEMM
    for (int idx = tid; idx < (m + 1) * k; idx += blockDim.x) {
      int row = idx / k, i = idx - row * k;
      pq[idx] = pvec[(size_t)i * pst + row];
      pq[(size_t)(a.m_max + 2) * k + idx] = (row < m) ? qvec[(size_t)i * pst + row] : 0.0;
    }
    __syncthreads();

    // ---- Ritz assembly (Eq. 1): U_k = U_{m+1} P_k, V_k = V_m Q_k, streamed basis ----
    constexpr int KMAX = 32;
    double* mxv = sm.mxv;  // [kWarps][KMAX] max |u| per warp
    int* mxi = sm.mxi;
    for (int side = 0; side < 2; ++side) {
      const bool isU = side == 0;
      const int n = isU ? L : K, ld = isU ? a.ldL : a.ldK, rows = isU ? m + 1 : m;
      const double* basis = isU ? U : V;
      const double* coef = pq + (isU ? 0 : (size_t)(a.m_max + 2) * k);
      double* out = (isU ? a.Uout : a.Vout) + (size_t)b * k * n;
      const int slab = ld / kWarps;
      const double* bw = basis + (size_t)w * slab;
      double bestv[KMAX];
      int besti[KMAX];
      for (int i = 0; i < KMAX; ++i) { bestv[i] = -1.0; besti[i] = 0; }
      constexpr int E = 2;
      for (int e0 = 0; e0 < slab; e0 += 32 * E) {
        double acc[E][16];
        // k <= 16 handled per chunk of 16 outputs
        for (int i0 = 0; i0 < k; i0 += 16) {
          const int ki = (k - i0) < 16 ? (k - i0) : 16;
#pragma unroll
          for (int t = 0; t < E; ++t)
#pragma unroll
            for (int i = 0; i < 16; ++i) acc[t][i] = 0.0;
          fence_proxy_async_smem();
          __syncwarp();
          stream_rows(bw, ld, rows, false, slab, rg, [&](int row, const double* ch) {
            const double* cr = coef + (size_t)row * k + i0;
            double cf[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) cf[i] = (i < ki) ? cr[i] : 0.0;
#pragma unroll
            for (int t = 0; t < E; ++t) {
              int e = e0 + t * 32 + lane;
              double x = (e < slab) ? ch[e] : 0.0;
#pragma unroll
              for (int i = 0; i < 16; ++i) acc[t][i] = fma(cf[i], x, acc[t][i]);
            }
          });
#pragma unroll
          for (int t = 0; t < E; ++t) {
            int e = e0 + t * 32 + lane;
            int g = w * slab + e;
            if (e < slab && g < n) {
#pragma unroll
              for (int i = 0; i < 16; ++i)
                if (i < ki) {
                  out[(size_t)(i0 + i) * n + g] = acc[t][i];
                  if (isU && fabs(acc[t][i]) > bestv[i0 + i]) { bestv[i0 + i] = fabs(acc[t][i]); besti[i0 + i] = g; }
                }
            }
          }
        }
      }
      if (isU) {
        // argmax |u_i| (lowest index on ties): warp reduce then across warps
        for (int i = 0; i < k; ++i) {
          double v = bestv[i];
          int ix = besti[i];
          for (int o = 16; o > 0; o >>= 1) {
            double v2 = __shfl_xor_sync(0xffffffffu, v, o);
            int i2 = __shfl_xor_sync(0xffffffffu, ix, o);
            if (v2 > v || (v2 == v && i2 < ix)) { v = v2; ix = i2; }
          }
          if (lane == 0) { mxv[w * KMAX + i] = v; mxi[w * KMAX + i] = ix; }
        }
      }
    }
    __syncthreads();
    // sign canonicalization: flip (u_i, v_i) if the largest-|.| entry of u_i is negative
    if (tid < k) {
      double v = -1.0;
      int ix = 0;
      for (int q = 0; q < kWarps; ++q) {
        double v2 = mxv[q * KMAX + tid];
        int i2 = mxi[q * KMAX + tid];
        if (v2 > v || (v2 == v && i2 < ix)) { v = v2; ix = i2; }
      }
      double* uo = a.Uout + ((size_t)b * k + tid) * L;
      sm.sgn[tid] = (uo[ix] < 0.0) ? -1.0 : 1.0;
    }
    __syncthreads();
    for (int i = 0; i < k; ++i) {
      if (sm.sgn[i] < 0.0) {
        double* uo = a.Uout + ((size_t)b * k + i) * L;
        double* vo = a.Vout + ((size_t)b * k + i) * K;
        for (int t = tid; t < L; t += blockDim.x) uo[t] = -uo[t];
        for (int t = tid; t < K; t += blockDim.x) vo[t] = -vo[t];
      }
    }
    if (tid < k) a.sigma[(size_t)b * k + tid] = qom[tid];
    if (tid == 0) {
      ssa_series_info inf;
      inf.steps = m;
      inf.converged = converged;
      inf.breakdown_step = breakdown;
      inf.reorth_extra = extra;
      inf.status = !ok_svd ? SSA_ERR_INTERNAL : (converged ? SSA_OK : SSA_ERR_NOT_CONVERGED);
      inf.reserved = restarts;
      inf.max_residual = final_res;
      inf.sigma1 = qom[0];
      a.info[b] = inf;
      (void)max_res;
    }
  }
}

// ------------------------------------------------------------------ launchers
static size_t fft_smem(int H) { return (size_t)fpad_size(H) * 16; }

cudaError_t fft_set_attributes(int H, const char** which) {
  cudaError_t e;
  size_t s1 = fft_smem(H), s2 = 2 * fft_smem(H);
  *which = "spectrum_kernel";
  if ((e = cudaFuncSetAttribute(spectrum_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s1))) return e;
  *which = "matvec_kernel";
  if ((e = cudaFuncSetAttribute(matvec_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s1))) return e;
  *which = "hankelize_kernel<BIG>";
  if ((e = cudaFuncSetAttribute(hankelize_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s1))) return e;
  *which = "hankelize_kernel";
  if (H <= kMaxHankelSmemH)
    if ((e = cudaFuncSetAttribute(hankelize_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s2)))
      return e;
  return cudaSuccess;
}

cudaError_t lanczos_set_attributes(size_t smem) {
  return cudaFuncSetAttribute(lanczos_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

cudaError_t launch_spectrum(const Plan& p, const double* series, double2* spec, cudaStream_t s) {
  spectrum_kernel<<<(unsigned)p.batch, kThreads, fft_smem((int)p.H), s>>>(series, (int)p.N, (int)p.H, p.d_tw, spec);
  return cudaGetLastError();
}

cudaError_t launch_matvec(const Plan& p, const double2* spec, const double* x, double* y, int transpose,
                          cudaStream_t s) {
  int n_in = transpose ? (int)p.L : (int)p.K;
  int n_out = transpose ? (int)p.K : (int)p.L;
  matvec_kernel<<<(unsigned)p.batch, kThreads, fft_smem((int)p.H), s>>>(spec, (int)p.H, n_in, n_out, p.d_tw, x, y);
  return cudaGetLastError();
}

cudaError_t launch_hankelize(const Plan& p, const double* sigma, const double* U, const double* V, int nterms,
                             double* out, cudaStream_t s) {
  size_t total = (size_t)p.batch * nterms;
  if (p.H <= kMaxHankelSmemH) {
    hankelize_kernel<false><<<(unsigned)total, kThreads, 2 * fft_smem((int)p.H), s>>>(
        sigma, U, V, total, (int)p.N, (int)p.L, (int)p.K, (int)p.H, p.d_tw, out, nullptr);
  } else {
    size_t grid = total < (size_t)p.hank_slots ? total : (size_t)p.hank_slots;
    hankelize_kernel<true><<<(unsigned)grid, kThreads, fft_smem((int)p.H), s>>>(
        sigma, U, V, total, (int)p.N, (int)p.L, (int)p.K, (int)p.H, p.d_tw, out, p.d_hscratch);
  }
  return cudaGetLastError();
}

cudaError_t launch_lanczos(const Plan& p, const LanczosArgs& a, cudaStream_t s) {
  int grid = p.slots;
  lanczos_kernel<<<grid, kThreads, p.smem_lanczos, s>>>(a);
  return cudaGetLastError();
}

}  // namespace ssa
