// ssa_fft_kernels.cu -- FFT-based building blocks of the fast Basic-SSA hot path.
//
//  spectrum_kernel   F^ = rfft(f, M)                     Alg. 2 l.1-2
//  matvec_kernel     y = X x / X^T x by FFT correlation  Alg. 2/3
//  hankelize_kernel  g = sigma irfft(rfft u rfft v) / c  sec 5, Alg. 4
//
// Correlation form (R1): with F^ = rfft(f, M) for any M >= N,
//   (X v)_i   = sum_j f_{i+j} v_j = irfft(F^ conj(rfft(v, M)))[i],  i < L
//   (X^T u)_j = sum_i f_{i+j} u_i = irfft(F^ conj(rfft(u, M)))[j],  j < K
// which is Alg. 2 / Alg. 3 (circulant embedding + backward identity) with the reversal
// folded into the conjugate and the output slice of Alg. 3 read as p'_L..p'_N.
#include "device_common.cuh"
#include "fft_reg.cuh"

#include <stdlib.h>

#include <algorithm>

namespace ssa {

template <int LOGH>
__device__ __forceinline__ void spectrum_body(double2* buf, const TwSmem& tw, const double* __restrict__ f, int N,
                                              double2* __restrict__ out) {
  constexpr int H = 1 << LOGH;
  for (int n = threadIdx.x; n < H; n += blockDim.x) {
    int i0 = 2 * n;
    double a = (i0 < N) ? f[i0] : 0.0;
    double c = (i0 + 1 < N) ? f[i0 + 1] : 0.0;
    buf[fsw(n)] = make_double2(a, c);
  }
  __syncthreads();
  fft_run_t<LOGH, false>(buf, tw, threadIdx.x, blockDim.x, CtaSync());
  for (int p = threadIdx.x; p <= (H >> 1); p += blockDim.x) {
    double2 Xp, Xq;
    int pr, qr;
    real_pair<LOGH>(buf, tw, p, Xp, Xq, pr, qr);
    out[p] = Xp;
    out[H - p] = Xq;
  }
}

#define SSA_DISPATCH_LOGH(logH, CALL)                                                                   \
  switch (logH) {                                                                                       \
    case 1: CALL(1); break; case 2: CALL(2); break; case 3: CALL(3); break; case 4: CALL(4); break;     \
    case 5: CALL(5); break; case 6: CALL(6); break; case 7: CALL(7); break; case 8: CALL(8); break;     \
    case 9: CALL(9); break; case 10: CALL(10); break; case 11: CALL(11); break; case 12: CALL(12); break; \
    default: CALL(13); break;                                                                           \
  }

__global__ void __launch_bounds__(kThreads) spectrum_kernel(const double* __restrict__ series, int N, int H,
                                                            const double2* __restrict__ T, double2* __restrict__ spec) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double2* buf = reinterpret_cast<double2*>(smem_raw);
  const TwSmem tw = load_tw2(T, buf + fft_elems(H), 2 * H);
  const FftShape sh = make_shape(H);
  const int b = blockIdx.x;
  const double* f = series + (size_t)b * N;
  double2* out = spec + (size_t)b * (H + 1);
#define SSA_SPEC(L) spectrum_body<L>(buf, tw, f, N, out)
  SSA_DISPATCH_LOGH(sh.logH, SSA_SPEC)
#undef SSA_SPEC
}

__global__ void __launch_bounds__(kThreads) matvec_kernel(const double2* __restrict__ spec, size_t spec_stride, int nvec,
                                                          int H, int n_in, int n_out, const double2* __restrict__ T,
                                                          const double* __restrict__ x, double* __restrict__ y) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double2* buf = reinterpret_cast<double2*>(smem_raw);
  const TwSmem tw = load_tw2(T, buf + fft_elems(H), 2 * H);  // visible after correlate's first barrier
  const FftShape sh = make_shape(H);
  const int b = blockIdx.x;
  const double* xb = x + (size_t)b * n_in;
  double* yb = y + (size_t)b * n_out;
  correlate_cta(
      buf, sh, tw, spec + (size_t)(b / nvec) * spec_stride, n_in, n_out, [&](int i) { return __ldg(xb + i); },
      [&](int t, double v) { yb[t] = v; });
}

// H = 4096 (BASELINE config 4): register-resident radix-16 correlation (fft_reg.cuh).
// Persistent CTAs (2 per SM); the next item's x is copied into a shared-memory stage by
// cp.async and its spectrum pulled into L2 while the current item is transformed.
__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__global__ void __launch_bounds__(kThreads, 2) matvec4096_kernel(const double2* __restrict__ spec, size_t spec_stride,
                                                                 int nvec, int n_in, int n_out,
                                                                 const double2* __restrict__ T,
                                                                 const double* __restrict__ x, double* __restrict__ y,
                                                                 int nitems) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double2* buf = reinterpret_cast<double2*>(smem_raw);
  double2* t2 = buf + 4096;
  double* stage = reinterpret_cast<double*>(t2 + 256);
  const TwSmem tw = load_tw2(T, reinterpret_cast<double2*>(stage + kReg4096StageDoubles), 8192);
  auto fetch = [&](int item) {
    if (item < nitems) {
      const double* src = x + (size_t)item * n_in;
      for (int i = threadIdx.x; i < n_in; i += kThreads) cp_async8(stage + i, src + i);
      const double2* sp = spec + (size_t)(item / nvec) * spec_stride;
      for (int i = threadIdx.x; i < 513; i += kThreads) asm volatile("prefetch.global.L2 [%0];" ::"l"(sp + 8 * i));
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  fetch(blockIdx.x);
  __syncthreads();
  reg4096_tables(t2, tw);
  for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    double* yb = y + (size_t)item * n_out;
    correlate_reg4096(
        buf, t2, tw, stage, spec + (size_t)(item / nvec) * spec_stride, n_in, n_out, [&]() { fetch(item + gridDim.x); },
        [&](int t, double v) { yb[t] = v; });
  }
}

// g_t = sigma * (u' * v')_t / c_t, c_t = min(t, L, K, N-t+1), t = 1..N  (PAPER.md:751-785,
// Alg. 4 PAPER.md:807-824 with the weights read as division, R2).
// Two shared-memory buffers when they fit (H <= kMaxHankelSmemH); otherwise (BIG) the
// post-processed spectrum of u goes to a per-CTA global scratch row (L2-resident) and the
// grid is persistent over terms.
template <int LOGH, bool BIG>
__device__ __forceinline__ void hankelize_body(double2* bufA, double2* bufB, const TwSmem& tw,
                                               const double* __restrict__ sigma, const double* __restrict__ U,
                                               const double* __restrict__ V, size_t nterm_total, int N, int L, int K,
                                               double* __restrict__ out, double2* Xu) {
  constexpr int H = 1 << LOGH;
  const int mn = L < K ? L : K;
  for (size_t term = blockIdx.x; term < nterm_total; term += gridDim.x) {
    const double* u = U + term * L;
    const double* v = V + term * K;
    const double sg = __ldg(sigma + term);
    if (BIG) {
      __syncthreads();
      for (int n = threadIdx.x; n < H; n += blockDim.x) {
        int i0 = 2 * n;
        bufB[fsw(n)] = make_double2(i0 < L ? __ldg(u + i0) : 0.0, i0 + 1 < L ? __ldg(u + i0 + 1) : 0.0);
      }
      __syncthreads();
      fft_run_t<LOGH, false>(bufB, tw, threadIdx.x, blockDim.x, CtaSync());
      for (int p = threadIdx.x; p <= (H >> 1); p += blockDim.x) {
        double2 Up, Uq;
        int pr, qr;
        real_pair<LOGH>(bufB, tw, p, Up, Uq, pr, qr);
        Xu[p] = Up;
        Xu[H - p] = Uq;
      }
      __syncthreads();
      for (int n = threadIdx.x; n < H; n += blockDim.x) {
        int i0 = 2 * n;
        bufB[fsw(n)] = make_double2(i0 < K ? __ldg(v + i0) : 0.0, i0 + 1 < K ? __ldg(v + i0 + 1) : 0.0);
      }
      __syncthreads();
      fft_run_t<LOGH, false>(bufB, tw, threadIdx.x, blockDim.x, CtaSync());
      for (int p = threadIdx.x; p <= (H >> 1); p += blockDim.x) {
        double2 Vp, Vq;
        int pr, qr;
        const double2 W = real_pair<LOGH>(bufB, tw, p, Vp, Vq, pr, qr);
        inv_pair(bufB, W, pr, qr, cmul(Xu[p], Vp), cmul(Xu[H - p], Vq));
      }
    } else {
      __syncthreads();
      for (int n = threadIdx.x; n < H; n += blockDim.x) {
        int i0 = 2 * n;
        bufA[fsw(n)] = make_double2(i0 < L ? __ldg(u + i0) : 0.0, i0 + 1 < L ? __ldg(u + i0 + 1) : 0.0);
        bufB[fsw(n)] = make_double2(i0 < K ? __ldg(v + i0) : 0.0, i0 + 1 < K ? __ldg(v + i0 + 1) : 0.0);
      }
      __syncthreads();
      fft_run_t<LOGH, false>(bufA, tw, threadIdx.x, blockDim.x, CtaSync());
      fft_run_t<LOGH, false>(bufB, tw, threadIdx.x, blockDim.x, CtaSync());
      for (int p = threadIdx.x; p <= (H >> 1); p += blockDim.x) {
        double2 Up, Uq, Vp, Vq;
        int pr, qr;
        real_pair<LOGH>(bufA, tw, p, Up, Uq, pr, qr);
        const double2 W = real_pair<LOGH>(bufB, tw, p, Vp, Vq, pr, qr);
        inv_pair(bufB, W, pr, qr, cmul(Up, Vp), cmul(Uq, Vq));
      }
    }
    __syncthreads();
    fft_run_t<LOGH, true>(bufB, tw, threadIdx.x, blockDim.x, CtaSync());
    const double scale = sg / (double)H;
    double* g = out + term * N;
    for (int t = threadIdx.x; t < N; t += blockDim.x) {
      double2 z = bufB[fsw(t >> 1)];
      int k1 = t + 1;  // 1-based
      int c = k1;
      if (c > mn) c = mn;
      if (N - k1 + 1 < c) c = N - k1 + 1;
      g[t] = ((t & 1) ? z.y : z.x) * (scale * rcp_count_f64(c));
    }
  }
}

template <bool BIG>
__global__ void __launch_bounds__(kThreads) hankelize_kernel(const double* __restrict__ sigma,
                                                             const double* __restrict__ U,
                                                             const double* __restrict__ V, size_t nterm_total, int N,
                                                             int L, int K, int H, const double2* __restrict__ T,
                                                             double* __restrict__ out, double2* gscratch) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double2* bufB = reinterpret_cast<double2*>(smem_raw);
  double2* bufA = BIG ? nullptr : bufB + fft_elems(H);
  const TwSmem tw = load_tw2(T, bufB + (BIG ? 1 : 2) * fft_elems(H), 2 * H);
  double2* Xu = BIG ? gscratch + (size_t)blockIdx.x * (H + 1) : nullptr;
  const FftShape sh = make_shape(H);
#define SSA_HANK(LG) hankelize_body<LG, BIG>(bufA, bufB, tw, sigma, U, V, nterm_total, N, L, K, out, Xu)
  SSA_DISPATCH_LOGH(sh.logH, SSA_HANK)
#undef SSA_HANK
}

// Grouped reconstruction (PAPER.md:131-146 grouping, 148-167 averaging): for group I_g,
// g = sum_{i in I_g} hankelization(sigma_i u_i v_i^T) = irfft(sum_i sigma_i rfft(u_i) rfft(v_i)) / c
// (diagonal averaging is linear), so the packed product spectra of the group's triples
// are accumulated in shared memory and one inverse FFT per group is run.  One CTA per
// (series, group); three H-point buffers (H <= kMaxHankelSmemH).
template <int LOGH>
__device__ __forceinline__ void group_body(double2* bufA, double2* bufB, double2* acc, const TwSmem& tw,
                                           const double* __restrict__ sigma, const double* __restrict__ U,
                                           const double* __restrict__ V, const GroupList& gl, int b, int g, int N,
                                           int L, int K, double* __restrict__ out) {
  constexpr int H = 1 << LOGH;
  const int k = gl.k;
  const int mn = L < K ? L : K;
  const int i0 = gl.ptr[g], i1 = gl.ptr[g + 1];
  for (int n = threadIdx.x; n < H; n += blockDim.x) acc[fsw(n)] = make_double2(0.0, 0.0);
  for (int ii = i0; ii < i1; ++ii) {
    const int i = gl.idx[ii];
    const double* u = U + ((size_t)b * k + i) * L;
    const double* v = V + ((size_t)b * k + i) * K;
    const double sg = __ldg(sigma + (size_t)b * k + i);
    __syncthreads();
    for (int n = threadIdx.x; n < H; n += blockDim.x) {
      const int j0 = 2 * n;
      bufA[fsw(n)] = make_double2(j0 < L ? __ldg(u + j0) : 0.0, j0 + 1 < L ? __ldg(u + j0 + 1) : 0.0);
      bufB[fsw(n)] = make_double2(j0 < K ? __ldg(v + j0) : 0.0, j0 + 1 < K ? __ldg(v + j0 + 1) : 0.0);
    }
    __syncthreads();
    fft_run_t<LOGH, false>(bufA, tw, threadIdx.x, blockDim.x, CtaSync());
    fft_run_t<LOGH, false>(bufB, tw, threadIdx.x, blockDim.x, CtaSync());
    for (int p = threadIdx.x; p <= (H >> 1); p += blockDim.x) {
      double2 Up, Uq, Vp, Vq;
      int pr, qr;
      real_pair<LOGH>(bufA, tw, p, Up, Uq, pr, qr);
      const double2 W = real_pair<LOGH>(bufB, tw, p, Vp, Vq, pr, qr);
      // inv_pair of sigma * (U V) added into acc (inv_pair is linear in its inputs)
      const double2 Yp = cmul(Up, Vp), Yq = cmul(Uq, Vq);
      const double2 E = make_double2(0.5 * sg * (Yp.x + Yq.x), 0.5 * sg * (Yp.y - Yq.y));
      const double2 D = make_double2(0.5 * sg * (Yp.x - Yq.x), 0.5 * sg * (Yp.y + Yq.y));
      const double2 O = cmulc(D, W);
      acc[pr] = cadd(acc[pr], make_double2(E.x - O.y, E.y + O.x));
      if (qr != pr) acc[qr] = cadd(acc[qr], make_double2(E.x + O.y, O.x - E.y));
    }
  }
  __syncthreads();
  fft_run_t<LOGH, true>(acc, tw, threadIdx.x, blockDim.x, CtaSync());
  constexpr double invH = 1.0 / (double)H;
  double* o = out + ((size_t)b * gl.ngroups + g) * N;
  for (int t = threadIdx.x; t < N; t += blockDim.x) {
    const double2 z = acc[fsw(t >> 1)];
    const int k1 = t + 1;
    int c = k1;
    if (c > mn) c = mn;
    if (N - k1 + 1 < c) c = N - k1 + 1;
    o[t] = ((t & 1) ? z.y : z.x) * (invH * rcp_count_f64(c));
  }
}

__global__ void __launch_bounds__(kThreads) group_hankelize_kernel(const double* __restrict__ sigma,
                                                                   const double* __restrict__ U,
                                                                   const double* __restrict__ V, GroupList gl, int N,
                                                                   int L, int K, int H, const double2* __restrict__ T,
                                                                   double* __restrict__ out) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double2* bufA = reinterpret_cast<double2*>(smem_raw);
  double2* bufB = bufA + H;
  double2* acc = bufB + H;
  const TwSmem tw = load_tw2(T, acc + H, 2 * H);
  const FftShape sh = make_shape(H);
  const int b = blockIdx.x / gl.ngroups, g = blockIdx.x % gl.ngroups;
#define SSA_GRP(LG) group_body<LG>(bufA, bufB, acc, tw, sigma, U, V, gl, b, g, N, L, K, out)
  SSA_DISPATCH_LOGH(sh.logH, SSA_GRP)
#undef SSA_GRP
}

// out[b][g][t] = sum_{i in I_g} elem[b][i][t] (large path: elementary series first).
__global__ void group_sum_kernel(const double* __restrict__ elem, GroupList gl, int N, size_t total,
                                 double* __restrict__ out) {
  for (size_t x = (size_t)blockIdx.x * blockDim.x + threadIdx.x; x < total; x += (size_t)gridDim.x * blockDim.x) {
    const size_t t = x % N, bg = x / N;
    const int g = (int)(bg % gl.ngroups);
    const size_t b = bg / gl.ngroups;
    double s = 0.0;
    for (int ii = gl.ptr[g]; ii < gl.ptr[g + 1]; ++ii) s += elem[((size_t)b * gl.k + gl.idx[ii]) * N + t];
    out[x] = s;
  }
}

static size_t tw_smem(int H) { return (size_t)tw2_entries(2 * H) * 16; }
static size_t fft_smem(int H) { return (size_t)fft_elems(H) * 16 + tw_smem(H); }
static size_t reg4096_smem() { return (size_t)kReg4096SmemElems * 16 + kReg4096StageDoubles * 8 + tw_smem(4096); }
static size_t fft_smem2(int H) { return (size_t)2 * fft_elems(H) * 16 + tw_smem(H); }

cudaError_t fft_set_attributes(int H, const char** which) {
  cudaError_t e;
  size_t s1 = fft_smem(H), s2 = fft_smem2(H);
  *which = "spectrum_kernel";
  if ((e = raise_smem_limit(spectrum_kernel, (int)s1))) return e;
  *which = "matvec_kernel";
  if ((e = raise_smem_limit(matvec_kernel, (int)s1))) return e;
  *which = "matvec4096_kernel";
  if (H == 4096 && (e = raise_smem_limit(matvec4096_kernel, (int)reg4096_smem()))) return e;
  *which = "hankelize_kernel<BIG>";
  if ((e = raise_smem_limit(hankelize_kernel<true>, (int)s1))) return e;
  *which = "group_hankelize_kernel";
  if (H <= kMaxHankelSmemH &&
      (e = raise_smem_limit(group_hankelize_kernel, (size_t)3 * fft_elems(H) * 16 + tw_smem(H))))
    return e;
  *which = "hankelize_kernel";
  if (H <= kMaxHankelSmemH)
    if ((e = raise_smem_limit(hankelize_kernel<false>, (int)s2)))
      return e;
  // shared memory over L1: these kernels keep everything in shared memory, and e.g. three
  // 75 KB matvec CTAs per SM only fit with the maximum carveout
  *which = "carveout";
  const int carve = cudaSharedmemCarveoutMaxShared;
  if ((e = cudaFuncSetAttribute(spectrum_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, carve))) return e;
  if ((e = cudaFuncSetAttribute(matvec_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, carve))) return e;
  if ((e = cudaFuncSetAttribute(matvec4096_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, carve))) return e;
  if ((e = cudaFuncSetAttribute(hankelize_kernel<true>, cudaFuncAttributePreferredSharedMemoryCarveout, carve))) return e;
  if ((e = cudaFuncSetAttribute(hankelize_kernel<false>, cudaFuncAttributePreferredSharedMemoryCarveout, carve)))
    return e;
  return cudaSuccess;
}

cudaError_t launch_spectrum(const Plan& p, const double* series, double2* spec, int nseries, cudaStream_t s) {
  spectrum_kernel<<<(unsigned)nseries, kThreads, fft_smem((int)p.H), s>>>(series, (int)p.N, (int)p.H, p.d_twl, spec);
  return cudaGetLastError();
}

cudaError_t launch_matvec_strided(const Plan& p, const double2* spec, size_t spec_stride, const double* x, double* y,
                                  int transpose, cudaStream_t s, int nvec) {
  int n_in = transpose ? (int)p.L : (int)p.K;
  int n_out = transpose ? (int)p.K : (int)p.L;
  const int64_t items = p.batch * nvec;
  if (p.H == 4096 && n_in <= 4097 && !getenv("SSA_MATVEC_SMEM")) {
    const int grid = (int)std::min<int64_t>(items, 2 * (int64_t)p.sms);
    matvec4096_kernel<<<grid, kThreads, reg4096_smem(), s>>>(spec, spec_stride, nvec, n_in, n_out, p.d_twl, x, y,
                                                              (int)items);
    return cudaGetLastError();
  }
  matvec_kernel<<<(unsigned)items, kThreads, fft_smem((int)p.H), s>>>(spec, spec_stride, nvec, (int)p.H, n_in, n_out,
                                                                      p.d_twl, x, y);
  return cudaGetLastError();
}

cudaError_t launch_matvec(const Plan& p, const double2* spec, const double* x, double* y, int transpose,
                          cudaStream_t s, int nvec) {
  return launch_matvec_strided(p, spec, (size_t)p.H + 1, x, y, transpose, s, nvec);
}

cudaError_t launch_group_hankelize(const Plan& p, const double* sigma, const double* U, const double* V,
                                   const GroupList& gl, double* out, cudaStream_t s) {
  const size_t grid = (size_t)p.batch * gl.ngroups;
  group_hankelize_kernel<<<(unsigned)grid, kThreads, (size_t)3 * fft_elems((int)p.H) * 16 + tw_smem((int)p.H), s>>>(
      sigma, U, V, gl, (int)p.N, (int)p.L, (int)p.K, (int)p.H, p.d_twl, out);
  return cudaGetLastError();
}

cudaError_t launch_group_sum(const Plan& p, const double* elem, const GroupList& gl, double* out, cudaStream_t s) {
  const size_t total = (size_t)p.batch * gl.ngroups * p.N;
  const size_t grid = std::min<size_t>((total + kThreads - 1) / kThreads, (size_t)p.sms * 16);
  group_sum_kernel<<<(unsigned)grid, kThreads, 0, s>>>(elem, gl, (int)p.N, total, out);
  return cudaGetLastError();
}

cudaError_t launch_hankelize(const Plan& p, const double* sigma, const double* U, const double* V, int nterms,
                             double* out, cudaStream_t s) {
  size_t total = (size_t)p.batch * nterms;
  if (p.H <= kMaxHankelSmemH) {
    hankelize_kernel<false><<<(unsigned)total, kThreads, fft_smem2((int)p.H), s>>>(
        sigma, U, V, total, (int)p.N, (int)p.L, (int)p.K, (int)p.H, p.d_twl, out, nullptr);
  } else {
    size_t grid = total < (size_t)p.hank_slots ? total : (size_t)p.hank_slots;
    hankelize_kernel<true><<<(unsigned)grid, kThreads, fft_smem((int)p.H), s>>>(
        sigma, U, V, total, (int)p.N, (int)p.L, (int)p.K, (int)p.H, p.d_twl, out, p.d_hscratch);
  }
  return cudaGetLastError();
}

}  // namespace ssa
