// fft_smem.cuh -- fp64 FFT building blocks held entirely in shared memory (sm_100a).
//
// One CTA transforms one complex vector of H = M/2 = 2^logH points (H <= 8192) in place:
//   * forward: in-place decimation-in-frequency passes (radix 8, final radix 4/2),
//     natural order in -> mixed-radix digit-reversed order out;
//   * inverse: the exact inverse passes in reverse order with conjugate twiddles,
//     digit-reversed in -> natural order out, unnormalized (result x H).
// So forward -> pointwise work in digit-reversed positions -> inverse needs no
// permutation pass.  Real transforms of length M are packed into H complex points
// (z_n = x_2n + i x_2n+1) with the usual split post-/pre-processing (ssa_kernels.cu).
// This is the DFT of PAPER.md:473-509 (sec 4.1: unnormalized forward, 1/N inverse),
// evaluated as an FFT.  All index arithmetic is shifts/masks (H and radices are powers
// of two).
//
// Shared-memory layout: the XOR swizzle fsw below.
// Twiddles come from a global table T[t] = exp(-2 pi i t / M), t in [0, H), computed on
// the host in extended precision (ssa_api.cu); exp(-2 pi i t / M) for t in [H, M) is
// -T[t - H].
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace ssa {

// XOR swizzle of the 16-byte elements inside each 128-byte row (8 elements): element i
// lives at i ^ g(i >> 3), g = XOR of the 3-bit digits of the row index.  Conflict-free
// (one wavefront per 8 lanes) for unit-stride runs, the stride-8 accesses of the last
// radix-8/4/2 passes and the digit-reversed pair steps (stride H/8), where plain rows
// would be 8-way conflicted; no padding, so a buffer of H points is H * 16 bytes.
__host__ __device__ __forceinline__ int fsw(int i) {
  const int j = i >> 3;
  return i ^ ((j ^ (j >> 3) ^ (j >> 6) ^ (j >> 9) ^ (j >> 12)) & 7);
}
__host__ __device__ __forceinline__ int fft_elems(int H) { return H; }

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {  // a * conj(b)
  return make_double2(fma(a.x, b.x, a.y * b.y), fma(a.y, b.x, -a.x * b.y));
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 conjg(double2 a) { return make_double2(a.x, -a.y); }

// exp(-2 pi i t / M) for t in [0, M) from the half table (t < H direct, else negated).
__device__ __forceinline__ double2 twiddle(const double2* __restrict__ T, int t, int H) {
  if (t < H) return __ldg(T + t);
  double2 w = __ldg(T + (t - H));
  return make_double2(-w.x, -w.y);
}

// Twiddle accessors: exp(-2 pi i t / M) for t in [0, M).
//  TwGlobal: the half table T[t] = exp(-2 pi i t / M), t < H, in global memory.
//  TwSmem:   two-level table in shared memory, lo[j] = exp(-2 pi i j / M) (j < 64) and
//            hi[j] = exp(-2 pi i 64 j / M) (j < max(1, M/64)); one complex product per lookup
//            (error ~1 ulp more than a direct table) -- used by the real-FFT pair steps,
//            whose lanes read consecutive entries.  Followed by per-pass tables for the
//            radix-8 passes of the H = M/2 point FFT (tw_pass_entries): pass with block
//            size S = 2^logS needs W_S^{n1}, n1 < Q = S/8, as lo_p[n1 & 63] (x hi_p[n1 >> 6]
//            when Q > 64), so consecutive lanes (consecutive n1) read consecutive entries:
//            no bank conflicts (a single table indexed by n1 << shift would be 2..8-way
//            conflicted) and one complex product fewer for Q <= 64.
__host__ __device__ constexpr int tw_pass_count(int logS) {  // entries of one radix-8 pass
  return (logS - 3 > 6) ? 64 + (1 << (logS - 3 - 6)) : (1 << (logS - 3 > 0 ? logS - 3 : 0));
}
__host__ __device__ constexpr int tw_pass_offset(int logH, int logS) {  // passes before logS
  return (logS >= logH) ? 0 : tw_pass_count(logH) + tw_pass_offset(logH - 3, logS);
}
__host__ __device__ constexpr int tw_pass_entries(int logH) {  // all radix-8 passes
  return (logH < 3) ? 0 : tw_pass_count(logH) + tw_pass_entries(logH - 3);
}
struct TwGlobal {
  const double2* T;
  int H;
  __device__ __forceinline__ double2 operator()(int t) const { return twiddle(T, t, H); }
};
struct TwSmem {
  const double2* lo;
  const double2* hi;
  const double2* pass;  // per-pass tables of the H-point FFT (H = M/2)
  __device__ __forceinline__ double2 operator()(int t) const { return cmul(lo[t & 63], hi[t >> 6]); }
  // W_S^{n1} for the radix-8 pass with block size 2^logS of an FFT of 2^logH points
  __device__ __forceinline__ double2 pass_w(int logH, int logS, int n1) const {
    const double2* tp = pass + tw_pass_offset(logH, logS);
    if (logS - 3 > 6) return cmul(tp[n1 & 63], tp[64 + (n1 >> 6)]);
    return tp[n1];
  }
};
// entries of the two-level table for size M (lo then hi), then the pass tables of M/2
__host__ __device__ inline int tw2_base_entries(int M) { return 64 + (M / 64 > 1 ? M / 64 : 1); }
__host__ __device__ inline int tw2_entries(int M) {
  int l = 0;
  while ((1 << l) < M / 2) ++l;
  return tw2_base_entries(M) + tw_pass_entries(l);
}

// Shape: n8 radix-8 passes then one radix-2^lastb pass (lastb in {0,1,2}).
struct FftShape {
  int H, logH, n8, lastb;
};

__host__ __device__ inline FftShape make_shape(int H) {
  FftShape s;
  s.H = H;
  int l = 0;
  while ((1 << l) < H) ++l;
  s.logH = l;
  s.n8 = l / 3;
  s.lastb = l - 3 * s.n8;
  return s;
}

// Digit-reversed position of frequency k (forward output order).
__device__ __forceinline__ int rev_index(const FftShape& s, int k) {
  int pos = 0, lsz = s.logH;
#pragma unroll 5
  for (int p = 0; p < s.n8; ++p) {
    lsz -= 3;
    pos += (k & 7) << lsz;
    k >>= 3;
  }
  if (s.lastb) pos += (k & ((1 << s.lastb) - 1));  // final block size is 1
  return pos;
}

// ---- small DFT kernels (forward sign exp(-2 pi i / R)); INV selects exp(+...) ----
template <bool INV>
__device__ __forceinline__ void dft2(double2& a, double2& b) {
  double2 t = a;
  a = cadd(t, b);
  b = csub(t, b);
}

template <bool INV>
__device__ __forceinline__ double2 mul_mi(double2 a) {  // multiply by -i (forward) or +i (inverse)
  return INV ? make_double2(-a.y, a.x) : make_double2(a.y, -a.x);
}

template <bool INV>
__device__ __forceinline__ void dft4(double2& a0, double2& a1, double2& a2, double2& a3) {
  double2 s0 = cadd(a0, a2), d0 = csub(a0, a2);
  double2 s1 = cadd(a1, a3), d1 = mul_mi<INV>(csub(a1, a3));
  a0 = cadd(s0, s1);
  a2 = csub(s0, s1);
  a1 = cadd(d0, d1);
  a3 = csub(d0, d1);
}

template <bool INV>
__device__ __forceinline__ void dft8(double2* a) {
  const double r = 0.70710678118654752440084436210485;  // 1/sqrt(2)
  double2 e0 = a[0], e1 = a[2], e2 = a[4], e3 = a[6];
  double2 o0 = a[1], o1 = a[3], o2 = a[5], o3 = a[7];
  dft4<INV>(e0, e1, e2, e3);
  dft4<INV>(o0, o1, o2, o3);
  double2 t1, t2, t3;
  if (!INV) {
    t1 = make_double2(r * (o1.x + o1.y), r * (o1.y - o1.x));    // * (1 - i)/sqrt2
    t2 = make_double2(o2.y, -o2.x);                               // * -i
    t3 = make_double2(r * (o3.y - o3.x), -r * (o3.x + o3.y));   // * (-1 - i)/sqrt2
  } else {
    t1 = make_double2(r * (o1.x - o1.y), r * (o1.y + o1.x));    // * (1 + i)/sqrt2
    t2 = make_double2(-o2.y, o2.x);                               // * i
    t3 = make_double2(-r * (o3.x + o3.y), r * (o3.x - o3.y));   // * (-1 + i)/sqrt2
  }
  a[0] = cadd(e0, o0); a[4] = csub(e0, o0);
  a[1] = cadd(e1, t1); a[5] = csub(e1, t1);
  a[2] = cadd(e2, t2); a[6] = csub(e2, t2);
  a[3] = cadd(e3, t3); a[7] = csub(e3, t3);
}

// dft8 with a[4..7] == 0 (the zero-padded half of a real-FFT input): the first radix-2
// stage of each dft4 is the identity, 16 additions fewer.
template <bool INV>
__device__ __forceinline__ void dft8_lowhalf(double2* a) {
  const double r = 0.70710678118654752440084436210485;  // 1/sqrt(2)
  const double2 ea = a[0], eb = a[2], oa = a[1], ob = a[3];
  const double2 eb_i = mul_mi<INV>(eb), ob_i = mul_mi<INV>(ob);
  const double2 e0 = cadd(ea, eb), e1 = cadd(ea, eb_i), e2 = csub(ea, eb), e3 = csub(ea, eb_i);
  const double2 o0 = cadd(oa, ob), o1 = cadd(oa, ob_i), o2 = csub(oa, ob), o3 = csub(oa, ob_i);
  double2 t1, t2, t3;
  if (!INV) {
    t1 = make_double2(r * (o1.x + o1.y), r * (o1.y - o1.x));    // * (1 - i)/sqrt2
    t2 = make_double2(o2.y, -o2.x);                               // * -i
    t3 = make_double2(r * (o3.y - o3.x), -r * (o3.x + o3.y));   // * (-1 - i)/sqrt2
  } else {
    t1 = make_double2(r * (o1.x - o1.y), r * (o1.y + o1.x));    // * (1 + i)/sqrt2
    t2 = make_double2(-o2.y, o2.x);                               // * i
    t3 = make_double2(-r * (o3.x + o3.y), r * (o3.x - o3.y));   // * (-1 + i)/sqrt2
  }
  a[0] = cadd(e0, o0); a[4] = csub(e0, o0);
  a[1] = cadd(e1, t1); a[5] = csub(e1, t1);
  a[2] = cadd(e2, t2); a[6] = csub(e2, t2);
  a[3] = cadd(e3, t3); a[7] = csub(e3, t3);
}

template <int R, bool INV>
__device__ __forceinline__ void dftR(double2* a) {
  if constexpr (R == 8) dft8<INV>(a);
  else if constexpr (R == 4) dft4<INV>(a[0], a[1], a[2], a[3]);
  else dft2<INV>(a[0], a[1]);
}

// g(j) of the swizzle as a constant expression (for compile-time offsets)
__host__ __device__ constexpr int gsw(int j) { return (j ^ (j >> 3) ^ (j >> 6) ^ (j >> 9) ^ (j >> 12)) & 7; }

// One DIF pass (forward) or its inverse: block size S = 2^LOGS, radix R = 2^LR,
// Q = S / R.  Butterfly (b, n1):
//   forward: y[n1 + Q k2] = W_S^{n1 k2} * sum_{n2} x[n1 + Q n2] W_R^{n2 k2}
//   inverse: x[n1 + Q n2] = sum_{k2} W_R^{-n2 k2} W_S^{-n1 k2} y[n1 + Q k2]   (times R)
// Addresses: for Q >= 8 the rows of the R elements differ by q Q / 8 in bits the row
// of `base` leaves zero, so fsw(base + q Q) = (fsw(base) + q Q) ^ gsw(q Q / 8): one
// swizzle per butterfly plus a constant XOR per element.
template <int LOGH, int LOGS, int LR, bool INV, class TW>
__device__ __forceinline__ void fft_pass_t(double2* buf, const TW& tw, int tid, int nthr) {
  constexpr int R = 1 << LR, LOGQ = LOGS - LR, Q = 1 << LOGQ, H = 1 << LOGH;
  for (int bf = tid; bf < (H >> LR); bf += nthr) {
    const int b = bf >> LOGQ, n1 = bf & (Q - 1);
    const int base = (b << LOGS) + n1;
    int idx[R];
    if constexpr (Q >= 8) {
      const int pb = fsw(base);
#pragma unroll
      for (int q = 0; q < R; ++q) idx[q] = (pb + (q << LOGQ)) ^ gsw((q << LOGQ) >> 3);
    } else {
#pragma unroll
      for (int q = 0; q < R; ++q) idx[q] = fsw(base + (q << LOGQ));
    }
    double2 a[R];
#pragma unroll
    for (int q = 0; q < R; ++q) a[q] = buf[idx[q]];
    double2 w[R];
    if constexpr (Q > 1) {
      // w_q = W_S^{n1 q} = (W_S^{n1})^q: one per-pass table lookup, powers by products
      w[1] = tw.pass_w(LOGH, LOGS, n1);
      if constexpr (R >= 4) { w[2] = cmul(w[1], w[1]); w[3] = cmul(w[2], w[1]); }
      if constexpr (R == 8) {
        w[4] = cmul(w[2], w[2]); w[5] = cmul(w[4], w[1]); w[6] = cmul(w[4], w[2]); w[7] = cmul(w[4], w[3]);
      }
      if constexpr (INV) {
#pragma unroll
        for (int q = 1; q < R; ++q) a[q] = cmulc(a[q], w[q]);
      }
    }
    dftR<R, INV>(a);
    if constexpr (!INV && Q > 1) {
#pragma unroll
      for (int q = 1; q < R; ++q) a[q] = cmul(a[q], w[q]);
    }
#pragma unroll
    for (int q = 0; q < R; ++q) buf[idx[q]] = a[q];
  }
}

struct CtaSync {
  __device__ __forceinline__ void operator()() const { __syncthreads(); }
};

// Forward FFT of H points in place (natural -> digit-reversed).  Caller must have
// synchronized after writing buf; returns after a final barrier.
// Whole transform with a compile-time size (all index arithmetic folds to constants).
template <int LOGH, int P, bool INV, int PMIN = 0, class TW, class Sync>
__device__ __forceinline__ void fft_radix8_passes(double2* buf, const TW& T, int tid, int nthr, Sync sync) {
  // passes P..N8-1 forward (INV: N8-1..PMIN, called with P counting down from the top)
  if constexpr (P >= PMIN && P < LOGH / 3) {
    if constexpr (!INV) {
      fft_pass_t<LOGH, LOGH - 3 * P, 3, false>(buf, T, tid, nthr);
      sync();
      fft_radix8_passes<LOGH, P + 1, false, PMIN>(buf, T, tid, nthr, sync);
    } else {
      fft_pass_t<LOGH, LOGH - 3 * P, 3, true>(buf, T, tid, nthr);
      sync();
      fft_radix8_passes<LOGH, P - 1, true, PMIN>(buf, T, tid, nthr, sync);
    }
  }
}

template <int LOGH, bool INV, class TW, class Sync>
__device__ __forceinline__ void fft_run_t(double2* buf, const TW& T, int tid, int nthr, Sync sync) {
  constexpr int N8 = LOGH / 3, LB = LOGH - 3 * N8;
  if constexpr (!INV) {
    fft_radix8_passes<LOGH, 0, false>(buf, T, tid, nthr, sync);
    if constexpr (LB == 2) { fft_pass_t<LOGH, 2, 2, false>(buf, T, tid, nthr); sync(); }
    if constexpr (LB == 1) { fft_pass_t<LOGH, 1, 1, false>(buf, T, tid, nthr); sync(); }
  } else {
    if constexpr (LB == 2) { fft_pass_t<LOGH, 2, 2, true>(buf, T, tid, nthr); sync(); }
    if constexpr (LB == 1) { fft_pass_t<LOGH, 1, 1, true>(buf, T, tid, nthr); sync(); }
    fft_radix8_passes<LOGH, N8 - 1, true>(buf, T, tid, nthr, sync);
  }
}

// The same transform without its outermost radix-8 pass (block 2^LOGH): forward runs
// passes 1.. (the caller did pass 0 in registers, dif_pass0_store), inverse stops before
// pass 0 (the caller finishes it in registers, dif_pass0_inverse_load).  LOGH >= 3.
template <int LOGH, bool INV, class TW, class Sync>
__device__ __forceinline__ void fft_run_inner_t(double2* buf, const TW& T, int tid, int nthr, Sync sync) {
  constexpr int N8 = LOGH / 3, LB = LOGH - 3 * N8;
  if constexpr (!INV) {
    fft_radix8_passes<LOGH, 1, false>(buf, T, tid, nthr, sync);
    if constexpr (LB == 2) { fft_pass_t<LOGH, 2, 2, false>(buf, T, tid, nthr); sync(); }
    if constexpr (LB == 1) { fft_pass_t<LOGH, 1, 1, false>(buf, T, tid, nthr); sync(); }
  } else {
    if constexpr (LB == 2) { fft_pass_t<LOGH, 2, 2, true>(buf, T, tid, nthr); sync(); }
    if constexpr (LB == 1) { fft_pass_t<LOGH, 1, 1, true>(buf, T, tid, nthr); sync(); }
    fft_radix8_passes<LOGH, N8 - 1, true, 1>(buf, T, tid, nthr, sync);
  }
}

// Pass 0 (block 2^LOGH, radix 8, stride Q = 2^LOGH / 8) on values a thread already holds:
// v[e] = x[base + STRIDE e], e < 2^LOGH / STRIDE; the thread owns the butterflies
// n1 = base + STRIDE b (b < NB = Q / STRIDE) with inputs e = b + NB q.  Forward: the pass
// outputs y[n1 + Q k] are stored to buf (swizzled); the rest of the transform is
// fft_run_inner_t.
// lowhalf: inputs q >= 4 (the upper half of the block) are zero (zero padding of a real
// input), so the butterfly skips their additions.
template <int LOGH, int STRIDE, class TW>
__device__ __forceinline__ void dif_pass0_store(const double2* v, int base, double2* buf, const TW& tw,
                                                bool lowhalf = false) {
  constexpr int Q = 1 << (LOGH - 3), NB = Q / STRIDE;
  static_assert(NB >= 1, "pass 0 needs 8 values per butterfly");
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const int n1 = base + STRIDE * b;
    double2 a[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) a[q] = v[b + NB * q];
    if (lowhalf) dft8_lowhalf<false>(a);
    else dftR<8, false>(a);
    double2 w[8];
    w[1] = tw.pass_w(LOGH, LOGH, n1);
    w[2] = cmul(w[1], w[1]); w[3] = cmul(w[2], w[1]);
    w[4] = cmul(w[2], w[2]); w[5] = cmul(w[4], w[1]); w[6] = cmul(w[4], w[2]); w[7] = cmul(w[4], w[3]);
    buf[fsw(n1)] = a[0];
#pragma unroll
    for (int q = 1; q < 8; ++q) buf[fsw(n1 + Q * q)] = cmul(a[q], w[q]);
  }
}

// Inverse of pass 0 after fft_run_inner_t<LOGH, true>: loads y[n1 + Q k] from buf and
// returns v[e] = H-scaled x[base + STRIDE e] (same ownership as dif_pass0_store).
template <int LOGH, int STRIDE, class TW>
__device__ __forceinline__ void dif_pass0_inverse_load(double2* v, int base, const double2* buf, const TW& tw) {
  constexpr int Q = 1 << (LOGH - 3), NB = Q / STRIDE;
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const int n1 = base + STRIDE * b;
    double2 a[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) a[q] = buf[fsw(n1 + Q * q)];
    double2 w[8];
    w[1] = tw.pass_w(LOGH, LOGH, n1);
    w[2] = cmul(w[1], w[1]); w[3] = cmul(w[2], w[1]);
    w[4] = cmul(w[2], w[2]); w[5] = cmul(w[4], w[1]); w[6] = cmul(w[4], w[2]); w[7] = cmul(w[4], w[3]);
#pragma unroll
    for (int q = 1; q < 8; ++q) a[q] = cmulc(a[q], w[q]);
    dftR<8, true>(a);
#pragma unroll
    for (int q = 0; q < 8; ++q) v[b + NB * q] = a[q];
  }
}

template <bool INV, class TW, class Sync>
__device__ __forceinline__ void fft_run(double2* buf, int logH, const TW& T, int tid, int nthr, Sync sync) {
  switch (logH) {
    case 1: fft_run_t<1, INV>(buf, T, tid, nthr, sync); break;
    case 2: fft_run_t<2, INV>(buf, T, tid, nthr, sync); break;
    case 3: fft_run_t<3, INV>(buf, T, tid, nthr, sync); break;
    case 4: fft_run_t<4, INV>(buf, T, tid, nthr, sync); break;
    case 5: fft_run_t<5, INV>(buf, T, tid, nthr, sync); break;
    case 6: fft_run_t<6, INV>(buf, T, tid, nthr, sync); break;
    case 7: fft_run_t<7, INV>(buf, T, tid, nthr, sync); break;
    case 8: fft_run_t<8, INV>(buf, T, tid, nthr, sync); break;
    case 9: fft_run_t<9, INV>(buf, T, tid, nthr, sync); break;
    case 10: fft_run_t<10, INV>(buf, T, tid, nthr, sync); break;
    case 11: fft_run_t<11, INV>(buf, T, tid, nthr, sync); break;
    case 12: fft_run_t<12, INV>(buf, T, tid, nthr, sync); break;
    default: fft_run_t<13, INV>(buf, T, tid, nthr, sync); break;
  }
}

// Forward FFT of H points in place (natural -> digit-reversed).  Caller must have
// synchronized after writing buf; returns after a final barrier.
template <class TW, class Sync>
__device__ __forceinline__ void fft_forward(double2* buf, const FftShape& s, const TW& T, int tid, int nthr, Sync sync) {
  fft_run<false>(buf, s.logH, T, tid, nthr, sync);
}

// Inverse (unnormalized, x H) FFT in place (digit-reversed -> natural).
template <class TW, class Sync>
__device__ __forceinline__ void fft_inverse(double2* buf, const FftShape& s, const TW& T, int tid, int nthr, Sync sync) {
  fft_run<true>(buf, s.logH, T, tid, nthr, sync);
}

}  // namespace ssa
