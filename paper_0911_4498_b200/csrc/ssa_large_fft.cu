// ssa_large_fft.cu -- multi-CTA (four-step) real FFT correlation / hankelization for
// series too long for one CTA's shared memory (M > 16384: BASELINE configs 3 and 5).
//
// The H = M/2 packed complex points z_n = x_2n + i x_2n+1 are split H = N1 x N2,
// n = n2 + N2 n1, frequency k = k1 + N1 k2:
//   X_{k1+N1k2} = sum_{n2} W_N2^{n2 k2} [ W_H^{n2 k1} sum_{n1} z_{n2+N2n1} W_N1^{n1 k1} ]
// (the DFT of PAPER.md:473-509 evaluated by the Cooley-Tukey four-step split).
//   large_col_fwd   N1-point column FFTs (one warp per column, 8 columns per CTA, shared
//                   memory) + twiddle W_H^{n2 k1}; writes Y[n2 + N2 k1] (global, L2).
//   large_row_pair  rows k1 and N1-k1 together: N2-point row FFTs, the real-FFT split
//                   step on the pairs (p, H-p) -- spectrum output, correlation with a
//                   stored spectrum (Algs. 2/3) or the product of two
//                   spectra (Alg. 4) -- then inverse row FFTs and the
//                   conjugate twiddle.
//   large_col_inv   inverse N1-point column FFTs, unpacking y_2n + i y_2n+1 with an
//                   epilogue (correlation output / Hankelization weights 1/c_t).
// The work buffers are [items][H] complex in global memory; for one item they are
// 8 MB (cfg3) or 2 MB (cfg5), so the three passes run out of L2.
#include <stdlib.h>

#include <algorithm>

#include "device_common.cuh"

namespace ssa {

constexpr int kColW = 8;  // columns per CTA in the column passes (one warp each)

struct WarpSync {
  __device__ __forceinline__ void operator()() const { __syncwarp(); }
};

// rev_index for a sub-FFT shape
__device__ __forceinline__ int subrev(const FftShape& s, int k) { return rev_index(s, k); }

// exp(-2 pi i e / H) for any integer e, from the M-table T (M = 2H): index 2e mod M.
__device__ __forceinline__ double2 twH(const double2* __restrict__ T, long long e, int H) {
  long long t = (2 * e) % (2LL * H);
  return twiddle(T, (int)t, H);
}

// ---- pass 1: forward column FFTs on packed real input x (len n_in) -------------------
// grid (N2 / kColW, items); x item stride xs; Y item stride H.
__global__ void __launch_bounds__(kThreads) large_col_fwd(const double* __restrict__ x, size_t xs, int n_in, int H,
                                                          int N1, int N2, const double2* __restrict__ T4,
                                                          const double2* __restrict__ T1, double2* __restrict__ Y) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double2* buf = reinterpret_cast<double2*>(smem_raw);
  const int cs = N1 + 1;  // odd stride (16-byte units): interleaved column loads are conflict-free
  const TwSmem tw1 = load_tw2(T1, buf + kColW * cs, 2 * N1);
  const FftShape s1 = make_shape(N1);
  const int n2_0 = blockIdx.x * kColW;
  const double* xi = x + (size_t)blockIdx.y * xs;
  double2* Yi = Y + (size_t)blockIdx.y * H;
  for (int idx = threadIdx.x; idx < N1 * kColW; idx += blockDim.x) {
    const int c = idx & (kColW - 1), n1 = idx >> 3;
    const long long n = (long long)(n2_0 + c) + (long long)N2 * n1;
    const long long i0 = 2 * n;
    double a = (i0 < n_in) ? __ldg(xi + i0) : 0.0;
    double b = (i0 + 1 < n_in) ? __ldg(xi + i0 + 1) : 0.0;
    buf[c * cs + fsw(n1)] = make_double2(a, b);
  }
  __syncthreads();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  fft_forward(buf + w * cs, s1, tw1, lane, 32, WarpSync());
  __syncthreads();
  for (int idx = threadIdx.x; idx < N1 * kColW; idx += blockDim.x) {
    const int c = idx & (kColW - 1), k1 = idx >> 3;
    const int n2 = n2_0 + c;
    double2 v = buf[c * cs + fsw(subrev(s1, k1))];
    v = cmul(v, __ldg(T4 + (size_t)n2 + (size_t)N2 * k1));  // W_H^{n2 k1}, same index as Y
    Yi[(size_t)n2 + (size_t)N2 * k1] = v;
  }
}

// ---- pass 3: inverse column FFTs + epilogue ------------------------------------------
// Epilogue modes: 0 correlation (out[t] = y_t - coef * prev[t], t < n_out, zero-filled to
// ld_out; partial sum of squares per CTA into part[blockIdx]) ; 1 hankelization
// (out[t] = sigma * y_t / c_t, t < N).
struct ColInvArgs {
  int H, N1, N2, mode;
  int n_out, ld_out;           // correlation output length and padded row length
  size_t out_stride;           // item stride of out
  double* out;
  const double* prev;          // correlation: previous vector (may be null)
  size_t prev_stride;
  const double* coef;          // correlation: per-item coefficient (device scalar), null -> 0
  double* part;                // correlation: partial sums of squares [items][gridDim.x]
  const double* sigma;         // hankelization: per-item sigma
  int N, L, K;                 // hankelization: weights
};

__global__ void __launch_bounds__(kThreads) large_col_inv(const double2* __restrict__ Y, const double2* __restrict__ T1,
                                                          ColInvArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double2* buf = reinterpret_cast<double2*>(smem_raw);
  __shared__ double red[kWarps];
  const int H = a.H, N1 = a.N1, N2 = a.N2;
  const int cs = N1 + 1;  // odd stride (16-byte units): interleaved column loads are conflict-free
  const TwSmem tw1 = load_tw2(T1, buf + kColW * cs, 2 * N1);
  const FftShape s1 = make_shape(N1);
  const int n2_0 = blockIdx.x * kColW;
  const size_t item = blockIdx.y;
  const double2* Yi = Y + item * H;
  for (int idx = threadIdx.x; idx < N1 * kColW; idx += blockDim.x) {
    const int c = idx & (kColW - 1), k1 = idx >> 3;
    buf[c * cs + fsw(subrev(s1, k1))] = Yi[(size_t)(n2_0 + c) + (size_t)N2 * k1];
  }
  __syncthreads();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  fft_inverse(buf + w * cs, s1, tw1, lane, 32, WarpSync());
  __syncthreads();
  const double invH = 1.0 / (double)H;
  double ss = 0.0;
  const double cf = (a.mode == 0 && a.coef) ? a.coef[item] : 0.0;
  const double sg = (a.mode == 1) ? a.sigma[item] : 0.0;
  const int mn = a.L < a.K ? a.L : a.K;
  for (int idx = threadIdx.x; idx < N1 * kColW * 2; idx += blockDim.x) {
    // element t = 2n + h of the real output, n = n2 + N2 n1
    const int h = idx & 1, rest = idx >> 1;
    const int c = rest & (kColW - 1), n1 = rest >> 3;
    const long long n = (long long)(n2_0 + c) + (long long)N2 * n1;
    const long long t = 2 * n + h;
    const double2 z = buf[c * cs + fsw(n1)];
    const double y = (h ? z.y : z.x) * invH;
    if (a.mode == 0) {
      if (t < a.ld_out) {
        double v = 0.0;
        if (t < a.n_out) {
          v = y;
          if (a.prev) v -= cf * a.prev[item * a.prev_stride + t];
        }
        a.out[item * a.out_stride + t] = v;
        ss = fma(v, v, ss);
      }
    } else {
      if (t < a.N) {
        const long long k1 = t + 1;
        long long cnt = k1;
        if (cnt > mn) cnt = mn;
        if (a.N - k1 + 1 < cnt) cnt = a.N - k1 + 1;
        a.out[item * a.out_stride + t] = sg * y / (double)cnt;
      }
    }
  }
  if (a.mode == 0 && a.part) {
    ss = warp_sum(ss);
    if (lane == 0) red[w] = ss;
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = 0.0;
      for (int i = 0; i < kWarps; ++i) s += red[i];
      a.part[item * gridDim.x + blockIdx.x] = s;
    }
  }
}

// ---- pass 2: row pairs ----------------------------------------------------------------
// Row index r = blockIdx.x in [0, N1/2]: rows A = r and B = N1 - r (B == A for r = 0 and
// r = N1/2).  Modes: 0 spectrum (write F^[0..H] natural order), 1 correlation with F^,
// 2 product of the spectra of two buffers (Ya * Yb, result in Yb).
struct RowArgs {
  int H, N1, N2, mode;
  const double2* T4;    // W_H^{n2 k1} at [n2 + N2 k1]
  const double2* Tp;    // W_M^{A + N1 k2} at [A N2 + k2], A <= N1/2
  double2* Ya;          // buffer of the (first) vector, [items][H]
  double2* Yb;          // mode 2: second buffer
  const double2* spec;  // mode 1: F^ [items or 1][H+1]
  size_t spec_stride;   // 0 -> shared spectrum for all items
  double2* spec_out;    // mode 0: [items][H+1]
};

__device__ __forceinline__ int partner_k2(int A, int k2, int N2) {
  return (A == 0) ? ((N2 - k2) & (N2 - 1)) : (N2 - 1 - k2);
}

// Row pairs, CTA-wide FFTs (modes 0/1: one item at a time, 257..513 CTAs of 256 threads
// keep the GPU busier than warp-level rows would).
__global__ void __launch_bounds__(kThreads) large_row_pair_cta(const double2* __restrict__ T, const double2* __restrict__ T2,
                                                           RowArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int H = a.H, N1 = a.N1, N2 = a.N2;
  const int rs = fft_elems(N2);
  double2* bA = reinterpret_cast<double2*>(smem_raw);  // row A of Ya
  double2* bB = bA + rs;                                // row B of Ya
  double2* cA = bB + rs;                                // mode 2: row A of Yb
  double2* cB = cA + rs;                                // mode 2: row B of Yb
  const TwSmem tw2 = load_tw2(T2, cB + rs, 2 * N2);
  const FftShape s2 = make_shape(N2);
  const int A = blockIdx.x, B = (N1 - A) & (N1 - 1);
  const bool two = (A != B);
  const size_t item = blockIdx.y;
  double2* Ya = a.Ya + item * H;
  double2* Yb = (a.mode == 2) ? a.Yb + item * H : nullptr;
  for (int i = threadIdx.x; i < N2; i += blockDim.x) {
    bA[fsw(i)] = Ya[(size_t)A * N2 + i];
    if (two) bB[fsw(i)] = Ya[(size_t)B * N2 + i];
    if (a.mode == 2) {
      cA[fsw(i)] = Yb[(size_t)A * N2 + i];
      if (two) cB[fsw(i)] = Yb[(size_t)B * N2 + i];
    }
  }
  __syncthreads();
  fft_forward(bA, s2, tw2, threadIdx.x, blockDim.x, CtaSync());
  if (two) fft_forward(bB, s2, tw2, threadIdx.x, blockDim.x, CtaSync());
  if (a.mode == 2) {
    fft_forward(cA, s2, tw2, threadIdx.x, blockDim.x, CtaSync());
    if (two) fft_forward(cB, s2, tw2, threadIdx.x, blockDim.x, CtaSync());
  }
  // pairs (p, q = H - p): p = A + N1 k2 in row A, q in row B at partner_k2
  const int npairs = two ? N2 : ((A == 0) ? N2 / 2 + 1 : N2 / 2);
  double2* rowB = two ? bB : bA;
  double2* rowBc = two ? cB : cA;
  const double2* F = (a.mode == 1) ? a.spec + item * a.spec_stride : nullptr;
  double2* Fo = (a.mode == 0) ? a.spec_out + item * (size_t)(H + 1) : nullptr;
  for (int k2 = threadIdx.x; k2 < npairs; k2 += blockDim.x) {
    const int k2q = partner_k2(A, k2, N2);
    const int pr = fsw(rev_index(s2, k2)), qr = fsw(rev_index(s2, k2q));
    const long long p = (long long)A + (long long)N1 * k2;
    const long long q = (p == 0) ? H : H - p;
    const double2 W = __ldg(a.Tp + (size_t)A * N2 + k2);  // exp(-2 pi i p / M), p = A + N1 k2
    auto split = [&](double2 Zp, double2 Zq, double2& Xp, double2& Xq) {
      double2 E = make_double2(0.5 * (Zp.x + Zq.x), 0.5 * (Zp.y - Zq.y));
      double2 D = make_double2(0.5 * (Zp.x - Zq.x), 0.5 * (Zp.y + Zq.y));
      double2 O = make_double2(D.y, -D.x);
      double2 WO = cmul(W, O);
      Xp = cadd(E, WO);
      Xq = conjg(csub(E, WO));
    };
    double2 Xp, Xq;
    split(bA[pr], rowB[qr], Xp, Xq);
    const bool same = (!two) && (pr == qr);
    if (a.mode == 0) {
      Fo[p] = Xp;
      Fo[q] = Xq;
    } else {
      double2 Yp, Yq;
      if (a.mode == 1) {
        Yp = cmulc(__ldg(F + p), Xp);
        Yq = cmulc(__ldg(F + q), Xq);
      } else {
        double2 Vp, Vq;
        split(cA[pr], rowBc[qr], Vp, Vq);
        Yp = cmul(Xp, Vp);
        Yq = cmul(Xq, Vq);
      }
      double2 E = make_double2(0.5 * (Yp.x + Yq.x), 0.5 * (Yp.y - Yq.y));
      double2 D = make_double2(0.5 * (Yp.x - Yq.x), 0.5 * (Yp.y + Yq.y));
      double2 O = cmulc(D, W);
      double2* dA = (a.mode == 2) ? cA : bA;
      double2* dB = (a.mode == 2) ? rowBc : rowB;
      dA[pr] = make_double2(E.x - O.y, E.y + O.x);
      if (!same) dB[qr] = make_double2(E.x + O.y, O.x - E.y);
    }
  }
  if (a.mode == 0) return;
  __syncthreads();
  double2* oA = (a.mode == 2) ? cA : bA;
  double2* oB = (a.mode == 2) ? cB : bB;
  double2* Yo = (a.mode == 2) ? Yb : Ya;
  fft_inverse(oA, s2, tw2, threadIdx.x, blockDim.x, CtaSync());
  if (two) fft_inverse(oB, s2, tw2, threadIdx.x, blockDim.x, CtaSync());
  for (int n2 = threadIdx.x; n2 < N2; n2 += blockDim.x) {
    Yo[(size_t)A * N2 + n2] = cmulc(oA[fsw(n2)], __ldg(a.T4 + (size_t)N2 * A + n2));
    if (two) Yo[(size_t)B * N2 + n2] = cmulc(oB[fsw(n2)], __ldg(a.T4 + (size_t)N2 * B + n2));
  }
}

// Row pairs with warp-level FFTs: each CTA takes G = warps / R row pairs (R = rows per
// pair: 2, or 4 in mode 2; G from the launch: 1 when one item must fill the GPU), warp g R + j loads and transforms row j of pair g on its own
// (no CTA barrier inside the FFTs), the pair step runs on the 32 R threads of the pair,
// and warps 0 / 1 of the pair run the inverse transforms of rows A / B and write them
// back with the conjugate twiddle.
__global__ void __launch_bounds__(kThreads) large_row_pair(const double2* __restrict__ T, const double2* __restrict__ T2,
                                                           RowArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int H = a.H, N1 = a.N1, N2 = a.N2;
  const int nw = blockDim.x >> 5;                         // warps = R rows x G pairs
  double2* rows = reinterpret_cast<double2*>(smem_raw);  // nw rows of N2
  const TwSmem tw2 = load_tw2(T2, rows + (size_t)nw * N2, 2 * N2);
  const FftShape s2 = make_shape(N2);
  const int R = (a.mode == 2) ? 4 : 2, G = nw / R;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = w / R, j = w - g * R;
  const int A = blockIdx.x * G + g, B = (N1 - A) & (N1 - 1);
  const bool valid = A <= N1 / 2, two = (A != B);
  const size_t item = blockIdx.y;
  double2* Ya = a.Ya + item * H;
  double2* Yb = (a.mode == 2) ? a.Yb + item * H : nullptr;
  double2* rA = rows + (size_t)(g * R) * N2;  // row A of Ya, row B of Ya, row A of Yb, row B of Yb
  double2* rB = rA + N2;
  double2* cA = rA + 2 * N2;
  double2* cB = rA + 3 * N2;
  __syncthreads();  // twiddle table
  const bool mine = valid && (two || !(j & 1));
  if (mine) {
    const double2* src = ((j >> 1) ? Yb : Ya) + (size_t)((j & 1) ? B : A) * N2;
    double2* dst = rows + (size_t)w * N2;
    for (int i = lane; i < N2; i += 32) dst[fsw(i)] = src[i];
    __syncwarp();
    fft_forward(dst, s2, tw2, lane, 32, WarpSync());
  }
  __syncthreads();
  if (valid) {
    // pairs (p, q = H - p): p = A + N1 k2 in row A, q in row B at partner_k2
    const int npairs = two ? N2 : ((A == 0) ? N2 / 2 + 1 : N2 / 2);
    double2* rowB = two ? rB : rA;
    double2* rowBc = two ? cB : cA;
    const double2* F = (a.mode == 1) ? a.spec + item * a.spec_stride : nullptr;
    double2* Fo = (a.mode == 0) ? a.spec_out + item * (size_t)(H + 1) : nullptr;
    for (int k2 = j * 32 + lane; k2 < npairs; k2 += 32 * R) {
      const int k2q = partner_k2(A, k2, N2);
      const int pr = fsw(rev_index(s2, k2)), qr = fsw(rev_index(s2, k2q));
      const long long p = (long long)A + (long long)N1 * k2;
      const long long q = (p == 0) ? H : H - p;
      const double2 W = __ldg(a.Tp + (size_t)A * N2 + k2);  // exp(-2 pi i p / M), p = A + N1 k2
      auto split = [&](double2 Zp, double2 Zq, double2& Xp, double2& Xq) {
        double2 E = make_double2(0.5 * (Zp.x + Zq.x), 0.5 * (Zp.y - Zq.y));
        double2 D = make_double2(0.5 * (Zp.x - Zq.x), 0.5 * (Zp.y + Zq.y));
        double2 O = make_double2(D.y, -D.x);
        double2 WO = cmul(W, O);
        Xp = cadd(E, WO);
        Xq = conjg(csub(E, WO));
      };
      double2 Xp, Xq;
      split(rA[pr], rowB[qr], Xp, Xq);
      const bool same = (!two) && (pr == qr);
      if (a.mode == 0) {
        Fo[p] = Xp;
        Fo[q] = Xq;
      } else {
        double2 Yp, Yq;
        if (a.mode == 1) {
          Yp = cmulc(__ldg(F + p), Xp);
          Yq = cmulc(__ldg(F + q), Xq);
        } else {
          double2 Vp, Vq;
          split(cA[pr], rowBc[qr], Vp, Vq);
          Yp = cmul(Xp, Vp);
          Yq = cmul(Xq, Vq);
        }
        double2 E = make_double2(0.5 * (Yp.x + Yq.x), 0.5 * (Yp.y - Yq.y));
        double2 D = make_double2(0.5 * (Yp.x - Yq.x), 0.5 * (Yp.y + Yq.y));
        double2 O = cmulc(D, W);
        double2* dA = (a.mode == 2) ? cA : rA;
        double2* dB = (a.mode == 2) ? rowBc : rowB;
        dA[pr] = make_double2(E.x - O.y, E.y + O.x);
        if (!same) dB[qr] = make_double2(E.x + O.y, O.x - E.y);
      }
    }
  }
  if (a.mode == 0) return;
  __syncthreads();
  if (valid && j < 2 && (two || j == 0)) {
    double2* o = (a.mode == 2) ? (j ? cB : cA) : (j ? rB : rA);
    const int row = j ? B : A;
    double2* Yo = ((a.mode == 2) ? Yb : Ya) + (size_t)row * N2;
    fft_inverse(o, s2, tw2, lane, 32, WarpSync());
    const double2* t4 = a.T4 + (size_t)N2 * row;  // W_H^{n2 row}
    for (int n2 = lane; n2 < N2; n2 += 32) Yo[n2] = cmulc(o[fsw(n2)], __ldg(t4 + n2));
  }
}

size_t large_col_smem(int N1) { return ((size_t)kColW * (N1 + 1) + tw2_entries(2 * N1)) * 16; }
size_t large_row_smem(int N2, int warps) {  // one row per warp, then the table
  return ((size_t)warps * N2 + tw2_entries(2 * N2)) * 16;
}
size_t large_row_cta_smem(int N2) { return ((size_t)4 * N2 + tw2_entries(2 * N2)) * 16; }

cudaError_t large_set_attributes(int N1, int N2) {
  cudaError_t e;
  if ((e = raise_smem_limit(large_col_fwd, (int)large_col_smem(N1))))
    return e;
  if ((e = raise_smem_limit(large_col_inv, (int)large_col_smem(N1))))
    return e;
  if ((e = raise_smem_limit(large_row_pair_cta, (int)large_row_cta_smem(N2)))) return e;
  if ((e = raise_smem_limit(large_row_pair, (int)large_row_smem(N2, kWarps))))
    return e;
  return cudaSuccess;
}

// ---- host-side drivers ----------------------------------------------------------------
struct LargeGeom {
  int H, N1, N2;
};

void large_geom(const Plan& p, int* N1, int* N2) {
  int l = 0;
  while ((1LL << l) < p.H) ++l;
  *N1 = 1 << (l / 2);
  *N2 = (int)(p.H / *N1);
}

static LargeGeom geom(const Plan& p) {
  LargeGeom g;
  g.H = (int)p.H;
  int l = 0;
  while ((1 << l) < g.H) ++l;
  g.N1 = 1 << (l / 2);
  g.N2 = g.H / g.N1;
  return g;
}

cudaError_t large_spectrum(const Plan& p, const double* series, double2* spec, int items, cudaStream_t s) {
  const LargeGeom g = geom(p);
  double2* Y = p.d_lbuf;
  for (int i0 = 0; i0 < items; i0 += p.lbuf_items) {
    const int ni = std::min(items - i0, p.lbuf_items);
    large_col_fwd<<<dim3(g.N2 / kColW, ni), kThreads, large_col_smem(g.N1), s>>>(
        series + (size_t)i0 * p.N, (size_t)p.N, (int)p.N, g.H, g.N1, g.N2, p.d_tw4, p.d_tw1, Y);
    RowArgs ra{g.H, g.N1, g.N2, 0, p.d_tw4, p.d_twp, Y, nullptr, nullptr, 0, spec + (size_t)i0 * (g.H + 1)};
    large_row_pair_cta<<<dim3(g.N1 / 2 + 1, ni), kThreads, large_row_cta_smem(g.N2), s>>>(p.d_tw, p.d_tw2, ra);
  }
  return cudaGetLastError();
}

// y[item] = X x (transpose 0) or X^T x (1) for items sharing one spectrum stride.
cudaError_t large_correlate(const Plan& p, const double2* spec, size_t spec_stride, const double* x, size_t xs, int n_in,
                            double* out, size_t os, int n_out, int ld_out, const double* prev, size_t ps,
                            const double* coef, double* part, int items, cudaStream_t s) {
  const LargeGeom g = geom(p);
  double2* Y = p.d_lbuf;
  for (int i0 = 0; i0 < items; i0 += p.lbuf_items) {
    const int ni = std::min(items - i0, p.lbuf_items);
    large_col_fwd<<<dim3(g.N2 / kColW, ni), kThreads, large_col_smem(g.N1), s>>>(
        x + (size_t)i0 * xs, xs, n_in, g.H, g.N1, g.N2, p.d_tw4, p.d_tw1, Y);
    RowArgs ra{g.H, g.N1, g.N2, 1, p.d_tw4, p.d_twp, Y, nullptr, spec + (size_t)i0 * spec_stride, spec_stride, nullptr};
    large_row_pair_cta<<<dim3(g.N1 / 2 + 1, ni), kThreads, large_row_cta_smem(g.N2), s>>>(p.d_tw, p.d_tw2, ra);
    ColInvArgs ca{};
    ca.H = g.H; ca.N1 = g.N1; ca.N2 = g.N2; ca.mode = 0;
    ca.n_out = n_out; ca.ld_out = ld_out; ca.out_stride = os; ca.out = out + (size_t)i0 * os;
    ca.prev = prev ? prev + (size_t)i0 * ps : nullptr; ca.prev_stride = ps;
    ca.coef = coef ? coef + i0 : nullptr;
    ca.part = part ? part + (size_t)i0 * (g.N2 / kColW) : nullptr;
    large_col_inv<<<dim3(g.N2 / kColW, ni), kThreads, large_col_smem(g.N1), s>>>(Y, p.d_tw1, ca);
  }
  return cudaGetLastError();
}

cudaError_t large_hankelize(const Plan& p, const double* sigma, const double* U, const double* V, size_t nterm_total,
                            double* out, cudaStream_t s) {
  const LargeGeom g = geom(p);
  // terms per batch (two H-point buffers each): as many as the work buffers hold -- the
  // four-step kernels are latency-bound per CTA, so more terms in flight win over keeping
  // the buffers in L2 (measured: 8 terms 14.9 us/term, 16: 11.9, 32: 11.2 at cfg5)
  int per = std::max(1, p.lbuf_items / 2);
  if (const char* e = getenv("SSA_HANK_PER")) per = std::max(1, std::min(p.lbuf_items / 2, atoi(e)));
  double2* Ya = p.d_lbuf;
  double2* Yb = p.d_lbuf + (size_t)per * g.H;
  for (size_t t0 = 0; t0 < nterm_total; t0 += per) {
    const int ni = (int)std::min<size_t>(nterm_total - t0, per);
    large_col_fwd<<<dim3(g.N2 / kColW, ni), kThreads, large_col_smem(g.N1), s>>>(
        U + t0 * p.L, (size_t)p.L, (int)p.L, g.H, g.N1, g.N2, p.d_tw4, p.d_tw1, Ya);
    large_col_fwd<<<dim3(g.N2 / kColW, ni), kThreads, large_col_smem(g.N1), s>>>(
        V + t0 * p.K, (size_t)p.K, (int)p.K, g.H, g.N1, g.N2, p.d_tw4, p.d_tw1, Yb);
    RowArgs ra{g.H, g.N1, g.N2, 2, p.d_tw4, p.d_twp, Ya, Yb, nullptr, 0, nullptr};
    large_row_pair<<<dim3((g.N1 / 2 + 2) / 2, ni), kThreads, large_row_smem(g.N2, kWarps), s>>>(p.d_tw, p.d_tw2, ra);
    ColInvArgs ca{};
    ca.H = g.H; ca.N1 = g.N1; ca.N2 = g.N2; ca.mode = 1;
    ca.out_stride = (size_t)p.N; ca.out = out + t0 * p.N;
    ca.sigma = sigma + t0; ca.N = (int)p.N; ca.L = (int)p.L; ca.K = (int)p.K;
    large_col_inv<<<dim3(g.N2 / kColW, ni), kThreads, large_col_smem(g.N1), s>>>(Yb, p.d_tw1, ca);
  }
  return cudaGetLastError();
}

}  // namespace ssa
