// fft_reg.cuh -- register-resident radix-16 FFT correlation for H = M/2 = 4096 packed
// complex points (M = 8192 real: BASELINE config 4, N = 8192) on one CTA of 256 threads.
//
// Same products as correlate_t (device_common.cuh): y = irfft(F^ conj(rfft(x, M)))[0:n_out],
// the Hankel products X v / X^T u of Alg. 2 / Alg. 3 in correlation form (PAPER.md:680-729,
// DESIGN.md R1), but each thread keeps 16 points in registers through three radix-16
// decimation-in-frequency passes (4096 = 16^3), so per product there are five shared-
// memory exchanges instead of ten radix-8 passes:
//   pass 1 (block 4096, stride 256)  from the x stage in shared memory (filled by cp.async
//                                    during the previous item; thread t: points t + 256 q),
//                                    half the inputs are the zero padding
//   pass 2 (block 256, stride 16)    via shared memory
//   pass 3 (block 16, stride 1)      via shared memory; thread t takes block swap(t) so it
//                                    ends holding the frequencies r + 256 k, r = t
//   pair step                        thread t and its partner 256 - t hold the pairs
//                                    (p, H - p) of the real-FFT split; each thread owns the
//                                    pairs of its slots k < 8: reads the partner's value,
//                                    keeps Z'_p, writes Z'_q into the partner's slot (every
//                                    warp does the same work)
//   inverse passes 3, 2, 1           in reverse; pass 3 starts from registers, pass 1
//                                    writes the real outputs straight to global memory.
// Shared-memory layout: swz(i) = i ^ ((i >> 8) & 7) (16-byte elements) makes every access
// pattern above one wavefront per 8 lanes.
#pragma once
#include "fft_smem.cuh"

namespace ssa {

__device__ __forceinline__ int swz4096(int i) { return i ^ ((i >> 8) & 7); }

// y[k] = sum_q a[q] W16^{qk} (forward W16 = exp(-2 pi i / 16); INV: conjugate), natural
// order in and out.  HALF: a[8..15] are zero.
template <bool INV, bool HALF>
__device__ __forceinline__ void dft16(double2* a) {
  const double c1 = 0.92387953251128675613, s1 = 0.38268343236508977173;  // cos, sin(pi/8)
  const double r2 = 0.70710678118654752440;
  double2 b[4][4];  // b[q1][k1]
#pragma unroll
  for (int q1 = 0; q1 < 4; ++q1) {
    double2 x0 = a[q1], x1 = a[q1 + 4];
    if constexpr (HALF) {
      // dft4 of (x0, x1, 0, 0)
      const double2 ix1 = mul_mi<INV>(x1);
      b[q1][0] = cadd(x0, x1);
      b[q1][1] = cadd(x0, ix1);
      b[q1][2] = csub(x0, x1);
      b[q1][3] = csub(x0, ix1);
    } else {
      double2 x2 = a[q1 + 8], x3 = a[q1 + 12];
      dft4<INV>(x0, x1, x2, x3);
      b[q1][0] = x0; b[q1][1] = x1; b[q1][2] = x2; b[q1][3] = x3;
    }
  }
  // internal twiddles W16^{q1 k1}
  auto w1 = [&](double2 x) {  // * W16^1 (INV: conj)
    return INV ? make_double2(c1 * x.x - s1 * x.y, c1 * x.y + s1 * x.x) : make_double2(c1 * x.x + s1 * x.y, c1 * x.y - s1 * x.x);
  };
  auto w3 = [&](double2 x) {  // * W16^3: cos(3pi/8) = s1, sin(3pi/8) = c1
    return INV ? make_double2(s1 * x.x - c1 * x.y, s1 * x.y + c1 * x.x) : make_double2(s1 * x.x + c1 * x.y, s1 * x.y - c1 * x.x);
  };
  auto w2 = [&](double2 x) {  // * W16^2 = (1 - i)/sqrt2
    return INV ? make_double2(r2 * (x.x - x.y), r2 * (x.y + x.x)) : make_double2(r2 * (x.x + x.y), r2 * (x.y - x.x));
  };
  auto w6 = [&](double2 x) {  // * W16^6 = (-1 - i)/sqrt2
    return INV ? make_double2(-r2 * (x.x + x.y), r2 * (x.x - x.y)) : make_double2(r2 * (x.y - x.x), -r2 * (x.x + x.y));
  };
  b[1][1] = w1(b[1][1]);
  b[1][2] = w2(b[1][2]);
  b[1][3] = w3(b[1][3]);
  b[2][1] = w2(b[2][1]);
  b[2][2] = mul_mi<INV>(b[2][2]);
  b[2][3] = w6(b[2][3]);
  b[3][1] = w3(b[3][1]);
  b[3][2] = w6(b[3][2]);
  {
    const double2 t = w1(b[3][3]);  // W16^9 = -W16^1
    b[3][3] = make_double2(-t.x, -t.y);
  }
#pragma unroll
  for (int k1 = 0; k1 < 4; ++k1) {
    double2 x0 = b[0][k1], x1 = b[1][k1], x2 = b[2][k1], x3 = b[3][k1];
    dft4<INV>(x0, x1, x2, x3);
    a[k1] = x0; a[k1 + 4] = x1; a[k1 + 8] = x2; a[k1 + 12] = x3;
  }
}

// a[k] *= w1^k (CONJ: conj(w1)^k), k = 1..15, powers by a depth-4 product tree (each within
// a few ulp), applied as they are formed so only a few powers are live at a time.
template <bool CONJ>
__device__ __forceinline__ void twiddle16(double2* a, double2 w1) {
  auto mul = [&](double2 x, double2 w) { return CONJ ? cmulc(x, w) : cmul(x, w); };
  const double2 w2 = cmul(w1, w1), w4 = cmul(w2, w2), w8 = cmul(w4, w4);
  const double2 w3 = cmul(w2, w1);
  a[1] = mul(a[1], w1); a[2] = mul(a[2], w2); a[3] = mul(a[3], w3); a[4] = mul(a[4], w4); a[8] = mul(a[8], w8);
  a[9] = mul(a[9], cmul(w8, w1)); a[10] = mul(a[10], cmul(w8, w2)); a[11] = mul(a[11], cmul(w8, w3));
  a[12] = mul(a[12], cmul(w8, w4));
  const double2 w5 = cmul(w4, w1), w6 = cmul(w4, w2), w7 = cmul(w4, w3);
  a[5] = mul(a[5], w5); a[6] = mul(a[6], w6); a[7] = mul(a[7], w7);
  a[13] = mul(a[13], cmul(w8, w5)); a[14] = mul(a[14], cmul(w8, w6)); a[15] = mul(a[15], cmul(w8, w7));
}

// Shared memory: 4096 double2 buffer + 256 double2 table (pass-2 twiddles, [k][n1]).
constexpr int kReg4096SmemElems = 4096 + 256;
constexpr int kReg4096StageDoubles = 4112;  // x staging (n_in <= 4097), 16-byte multiple

// Builds the pass-2 table T2[k * 16 + n1] = W_256^{n1 k} from the M = 8192 two-level table
// (all threads; the caller's first barrier publishes it).
__device__ __forceinline__ void reg4096_tables(double2* t2, const TwSmem& tw) {
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    const int k = i >> 4, n1 = i & 15;
    t2[i] = tw((32 * n1 * k) & 8191);  // W_8192^{32 n1 k} = W_256^{n1 k}
  }
}

// y_t = sum_s f_{t+s} x_s, t < n_out, for H = 4096 (blockDim.x == 256).  n_in <= 4097 (the
// zero padding covers the upper half of the packed input, except packed point 2048 when
// n_in = 4097).  stage: x[0..n_in) in shared memory; spec: F^[0..4096] (global); tw: M = 8192
// two-level table (TwSmem); t2: pass-2 table (reg4096_tables, published by a barrier).
// after1() runs after the first barrier, when every thread has read `stage` (the caller
// refills it there for the next item).
template <class After1, class StoreY>
__device__ __forceinline__ void correlate_reg4096(double2* buf, const double2* t2, const TwSmem& tw,
                                                  const double* stage, const double2* __restrict__ spec, int n_in,
                                                  int n_out, After1 after1, StoreY storey) {
  constexpr int H = 4096;
  const int t = threadIdx.x;
  double2 a[16];
  // ---- forward pass 1 (block 4096, stride 256): packed points t + 256 q, q < 8 (+ q = 8 at t = 0)
  const double2* st2 = reinterpret_cast<const double2*>(stage);
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int i0 = 2 * (t + 256 * q);
    if (i0 + 1 < n_in) {
      a[q] = st2[t + 256 * q];
    } else {
      a[q].x = (i0 < n_in) ? stage[i0] : 0.0;
      a[q].y = 0.0;
    }
  }
  double2 extra = make_double2(0.0, 0.0);  // packed point 2048 = (x_4096, x_4097) at t = 0
  if (t == 0) {
    extra.x = (4096 < n_in) ? stage[4096] : 0.0;
    extra.y = (4097 < n_in) ? stage[4097] : 0.0;
  }
#pragma unroll
  for (int q = 8; q < 16; ++q) a[q] = make_double2(0.0, 0.0);
  dft16<false, true>(a);
  if (t == 0) {  // + extra * W16^{8k} = extra * (-1)^k
#pragma unroll
    for (int k = 0; k < 16; ++k) a[k] = (k & 1) ? csub(a[k], extra) : cadd(a[k], extra);
  }
  twiddle16<false>(a, tw(2 * t));  // W_4096^{t k}
#pragma unroll
  for (int k = 0; k < 16; ++k) buf[swz4096(t + 256 * k)] = a[k];
  __syncthreads();
  after1();
  // ---- pass 2 (block 256, stride 16): thread t = butterfly (b = t >> 4, n1 = t & 15)
  const int b2 = t >> 4, n1 = t & 15;
  const int base2 = (b2 << 8) + n1;
#pragma unroll
  for (int q = 0; q < 16; ++q) a[q] = buf[swz4096(base2 + 16 * q)];
  dft16<false, false>(a);
#pragma unroll
  for (int k = 1; k < 16; ++k) a[k] = cmul(a[k], t2[k * 16 + n1]);
#pragma unroll
  for (int k = 0; k < 16; ++k) buf[swz4096(base2 + 16 * k)] = a[k];
  __syncthreads();
  // ---- pass 3 (block 16): thread t takes block b = swap(t) -> frequencies t + 256 k
  const int b3 = ((t & 15) << 4) | (t >> 4);
#pragma unroll
  for (int q = 0; q < 16; ++q) a[q] = buf[swz4096(16 * b3 + q)];
  dft16<false, false>(a);
  // a[k] = Z_{t + 256 k}; publish them for the partner (own block: no hazard)
#pragma unroll
  for (int k = 0; k < 16; ++k) buf[swz4096(16 * b3 + k)] = a[k];
  __syncthreads();
  // ---- pair step: p = t + 256 k, q = H - p (mod H) lives at thread tp = (256 - t) & 255,
  // slot kp = 15 - k (t = 0: (16 - k) & 15).  Every thread owns the pairs of its k < 8 (and
  // thread 0 the self pair k = 8): it reads the partner's Z_q, keeps Z'_p and writes Z'_q
  // into the partner's slot (slots >= 8 are read and written by one thread only).
  {
    const int tp = (256 - t) & 255;
    const int bp = ((tp & 15) << 4) | (tp >> 4);
    auto pair = [&](int k, double2& zp, double2 Fp, double2 Fq) {
      const int kp = (t == 0) ? ((16 - k) & 15) : (15 - k);
      const int p = t + 256 * k;
      const double2 Zp = zp;
      const double2 Zq = buf[swz4096(16 * bp + kp)];
      const double2 W = tw(p);  // exp(-2 pi i p / M)
      // the two 1/2 factors of the split / merge are exact powers of two: folded into the
      // final 1/H scale (invH / 4), bit-identical results, 8 multiplications fewer per pair
      const double2 E = make_double2(Zp.x + Zq.x, Zp.y - Zq.y);
      const double2 D = make_double2(Zp.x - Zq.x, Zp.y + Zq.y);
      const double2 WO = cmul(W, make_double2(D.y, -D.x));
      const double2 Xp = cadd(E, WO), Xq = conjg(csub(E, WO));
      const double2 Yp = cmulc(Fp, Xp), Yq = cmulc(Fq, Xq);
      const double2 E2 = make_double2(Yp.x + Yq.x, Yp.y - Yq.y);
      const double2 D2 = make_double2(Yp.x - Yq.x, Yp.y + Yq.y);
      const double2 O2 = cmulc(D2, W);
      zp = make_double2(E2.x - O2.y, E2.y + O2.x);
      buf[swz4096(16 * bp + kp)] = make_double2(E2.x + O2.y, O2.x - E2.y);
    };
    // spectrum loads of four pairs at a time in flight (p = 0: F^_H is the partner)
#pragma unroll
    for (int k0 = 0; k0 < 8; k0 += 4) {
      double2 Fp[4], Fq[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int p = t + 256 * (k0 + j);
        Fp[j] = __ldg(spec + p);
        Fq[j] = __ldg(spec + (H - p));
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) pair(k0 + j, a[k0 + j], Fp[j], Fq[j]);
    }
    if (t == 0) pair(8, a[8], __ldg(spec + 2048), __ldg(spec + 2048));  // (2048, 2048)
  }
  __syncthreads();
#pragma unroll
  for (int k = 8; k < 16; ++k) a[k] = buf[swz4096(16 * b3 + k)];
  // ---- inverse pass 3 (registers), 2, 1
  dft16<true, false>(a);
#pragma unroll
  for (int k = 0; k < 16; ++k) buf[swz4096(16 * b3 + k)] = a[k];
  __syncthreads();
#pragma unroll
  for (int q = 0; q < 16; ++q) a[q] = buf[swz4096(base2 + 16 * q)];
#pragma unroll
  for (int k = 1; k < 16; ++k) a[k] = cmulc(a[k], t2[k * 16 + n1]);
  dft16<true, false>(a);
#pragma unroll
  for (int k = 0; k < 16; ++k) buf[swz4096(base2 + 16 * k)] = a[k];
  __syncthreads();
#pragma unroll
  for (int q = 0; q < 16; ++q) a[q] = buf[swz4096(t + 256 * q)];
  twiddle16<true>(a, tw(2 * t));
  dft16<true, false>(a);
  // a[n2] = 4 H * y packed at n = t + 256 n2 (the pair step's 1/4 deferred): real outputs 2n, 2n + 1
  constexpr double invH = 0.25 / (double)H;
#pragma unroll
  for (int n2 = 0; n2 < 16; ++n2) {
    const int i0 = 2 * (t + 256 * n2);
    if (i0 < n_out) storey(i0, a[n2].x * invH);
    if (i0 + 1 < n_out) storey(i0 + 1, a[n2].y * invH);
  }
}

}  // namespace ssa
