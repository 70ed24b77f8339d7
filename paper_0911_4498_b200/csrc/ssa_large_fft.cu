// ssa_large_fft.cu -- multi-CTA (four-step) real FFT correlation / hankelization for
// series too long for one CTA's shared memory (M > 16384: BASELINE configs 3 and 5).
//
// The H = M/2 packed complex points z_n = x_2n + i x_2n+1 are split H = N1 x N2,
// n = n2 + N2 n1, frequency k = k1 + N1 k2:
//   X_{k1+N1k2} = sum_{n2} W_N2^{n2 k2} [ W_H^{n2 k1} sum_{n1} z_{n2+N2n1} W_N1^{n1 k1} ]
// (the DFT of PAPER.md:473-509 evaluated by the Cooley-Tukey four-step split).
//   lg_col_fwd   N1-point column FFTs (one warp per column, 8 columns per CTA, shared
//                memory) + twiddle W_H^{n2 k1}; writes Y[n2 + N2 k1] (global, L2).  One
//                launch can transform two inputs (blockIdx.z: the u and v of a term).
//   lg_row_*     rows k1 and N1-k1 together: N2-point row FFTs, the real-FFT split step on
//                the pairs (p, H-p) -- spectrum output, correlation with a stored spectrum
//                (Algs. 2/3) or the product of two spectra (Alg. 4,
//                PAPER.md:807-824) -- then inverse row FFTs and the conjugate twiddle.
//   lg_col_inv   inverse N1-point column FFTs, unpacking y_2n + i y_2n+1 with an epilogue
//                (correlation output / Hankelization weights 1/c_t).
// Every shape is a compile-time constant (one switch on log2 H per launch), so the
// global loads of a thread are unrolled and all in flight together.  Twiddles come from
// small tables: W_H^e = TL[e mod 2^a] TH[e >> a] (a = ceil(log2 H / 2), global, L1-resident),
// W_M^{A + N1 k2} = W_M^A W_{2 N2}^{k2}; all tables are computed on the host in extended
// precision.  The work buffers are [items][H] complex in global memory; for one item they
// are 8 MB (cfg3) or 2 MB (cfg5), so the passes run out of L2.
#include <stdlib.h>

#include <algorithm>

#include "device_common.cuh"
#include "fft_reg.cuh"
#include "lg_scalars.cuh"

namespace ssa {

cudaError_t trace_attach_fft(unsigned long long* p) { return trace_attach(p); }

constexpr int kColW = 8;  // columns per CTA in the column passes

// Threads of a column-pass CTA: 256 (one warp per column) for the batched sizes; 512 (two
// warps per column, 8 rows per thread) for H >= 2^19, where one item's 128 CTAs are all the
// parallelism there is and the per-warp FFT chain sets the time (cfg3: one series, N = 2^20).
template <int LOGH>
__host__ __device__ constexpr int col_threads() { return LOGH >= 19 ? 512 : 256; }

// barrier of the threads of one column: a warp, or a named barrier over its two warps
template <int CT>
struct ColSync {
  int id;
  __device__ __forceinline__ void operator()() const {
    if constexpr (CT / kColW == 32) __syncwarp();
    else asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(CT / kColW) : "memory");
  }
};

struct WarpSync {
  __device__ __forceinline__ void operator()() const { __syncwarp(); }
};
// Named barriers over 64 / 128 threads (two / four warps); ids 1..15 (0 is __syncthreads).
struct NamedSync64 {
  int id;
  __device__ __forceinline__ void operator()() const { asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory"); }
};
struct NamedSync128 {
  int id;
  __device__ __forceinline__ void operator()() const { asm volatile("bar.sync %0, 128;" ::"r"(id) : "memory"); }
};

// Compile-time four-step geometry for H = 2^LOGH.
template <int LOGH>
struct Geo {
  static constexpr int H = 1 << LOGH;
  static constexpr int L1 = LOGH / 2, N1 = 1 << L1;  // column length
  static constexpr int L2 = LOGH - L1, N2 = 1 << L2;  // row length
  static constexpr int TA = (LOGH + 1) / 2;           // W_H two-level split
  static constexpr int NTL = 1 << TA, NTH = H >> TA;
  static constexpr int NTW = NTL + NTH;               // entries of the W_H table
};

int large_twh_entries(int logH) { return (1 << ((logH + 1) / 2)) + (1 << (logH - (logH + 1) / 2)); }

// W_H^e for any integer e >= 0 from the two-level table (global memory, L1-resident:
// 12-32 KB shared by every CTA of the SM).
template <int LOGH>
__device__ __forceinline__ double2 twH(const double2* __restrict__ th, long long e) {
  using G = Geo<LOGH>;
  const int t = (int)(e & (G::H - 1));
  return cmul(__ldg(th + (t & (G::NTL - 1))), __ldg(th + G::NTL + (t >> G::TA)));
}

// f(j, W_H^{e0 + d j}) for j = 0..n-1: one table lookup per 8 values, then products by
// W_H^d (chains of at most 7 products: each twiddle within a few ulp).
template <int LOGH, int NMAX, class F>
__device__ __forceinline__ void twiddle_seq(const double2* __restrict__ th, long long e0, long long d, int n, F f) {
  const double2 step = twH<LOGH>(th, d);
#pragma unroll
  for (int g = 0; g < NMAX; g += 8) {
    double2 w = twH<LOGH>(th, e0 + d * g);
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) {
      if (g + jj < NMAX && g + jj < n) {
        f(g + jj, w);
        if (jj < 7) w = cmul(w, step);
      }
    }
  }
}

// ---- pass 1: forward column FFTs on packed real input x (len n_in) -------------------
struct ColFwdIn {
  const double* x;  // [items][xs] real
  size_t xs;
  int n_in;
  double2* Y;       // [items][H]
  int vec;          // x 16-byte aligned: pairs (x_2n, x_2n+1) of aligned rows as one 16-byte load
  LgNorm nrm;       // long-series Lanczos: x is r, scaled by *nrm.inv on the fly and written to
                    // the basis row and the current vector (nrm.inv null: plain input)
};
struct ColFwdArgs {
  ColFwdIn in[2];   // blockIdx.z selects
  const int* gate;  // device flag: nonzero -> the launch does nothing (graph-driven loops)
};

template <int LOGH>
__global__ void __launch_bounds__(col_threads<LOGH>()) lg_col_fwd(ColFwdArgs args, const double2* __restrict__ T1,
                                                       const double2* __restrict__ TWH) {
  using G = Geo<LOGH>;
  constexpr int N1 = G::N1, N2 = G::N2, CS = N1 + 1;  // odd column stride (16-byte units)
  constexpr int CT = col_threads<LOGH>(), RS = CT / kColW;  // threads, row step of a thread
  constexpr int NE = (N1 * kColW + CT - 1) / CT;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double2* buf = reinterpret_cast<double2*>(smem_raw);
  const double2* th = TWH;
  const TwSmem tw1 = load_tw2(T1, buf + kColW * CS, 2 * N1);  // constant: before the wait
  pdl_wait(1);
  if (args.gate && *args.gate) return;
  const ColFwdIn a = blockIdx.z ? args.in[1] : args.in[0];
  const int n2_0 = blockIdx.x * kColW;
  const double* xi = a.x + (size_t)blockIdx.y * a.xs;
  double2* Yi = a.Y + (size_t)blockIdx.y * G::H;
  // 16-byte pair loads when this row starts 16-byte aligned (every row when the stride is
  // even; every other row of an odd stride, e.g. the v_i of length K = L + 1)
  const bool rvec = a.vec && ((reinterpret_cast<uintptr_t>(xi) & 15) == 0);
  // thread t: column c = t & 7 of the CTA, rows n1 = (t >> 3) + 32 j (idx = t + 256 j)
  const int cc = threadIdx.x & (kColW - 1), r0 = threadIdx.x >> 3;
  const int i00 = 2 * (n2_0 + cc + N2 * r0);  // packed point n = n2 + N2 n1 -> x_2n, x_2n+1
  double2 v[NE];
#pragma unroll
  for (int j = 0; j < NE; ++j) {
    const bool ok = threadIdx.x + j * CT < N1 * kColW;
    const int i0 = i00 + j * (2 * N2 * (RS));
    if (rvec && ok && i0 + 1 < a.n_in) {
      v[j] = __ldg(reinterpret_cast<const double2*>(xi + i0));
    } else {
      v[j].x = (ok && i0 < a.n_in) ? __ldg(xi + i0) : 0.0;
      v[j].y = (ok && i0 + 1 < a.n_in) ? __ldg(xi + i0 + 1) : 0.0;
    }
  }
  if (a.nrm.inv) {
    // Lanczos normalization of the previous half-step's vector (one item): every element of
    // x is read by exactly one thread of the grid, which scales it and stores it to the
    // basis row and the current vector (the padding of the basis row stays zero)
    const double inv = *a.nrm.inv;
    double* brow = a.nrm.basis + (size_t)(*a.nrm.jrow - 1) * a.nrm.ld;
#pragma unroll
    for (int j = 0; j < NE; ++j) {
      const bool ok = threadIdx.x + j * CT < N1 * kColW;
      const int i0 = i00 + j * (2 * N2 * (RS));
      v[j].x *= inv;
      v[j].y *= inv;
      if (rvec && ok && i0 + 1 < a.n_in) {
        *reinterpret_cast<double2*>(brow + i0) = v[j];
        *reinterpret_cast<double2*>(a.nrm.cur + i0) = v[j];
      } else {
        if (ok && i0 < a.n_in) { brow[i0] = v[j].x; a.nrm.cur[i0] = v[j].x; }
        if (ok && i0 + 1 < a.n_in) { brow[i0 + 1] = v[j].y; a.nrm.cur[i0 + 1] = v[j].y; }
      }
    }
    if (blockIdx.x == 0 && threadIdx.x < a.nrm.ld - a.n_in) brow[a.n_in + threadIdx.x] = 0.0;
  }
  // column of the FFT phase: warps [c * RS / 32, (c + 1) * RS / 32), thread ct of RS
  const int fc = threadIdx.x / RS, ct = threadIdx.x % RS;
  const ColSync<CT> csync{1 + fc};
  if constexpr (G::L1 >= 8) {
    // the thread holds rows r0 + 32 j of its column: the butterflies of the outermost
    // radix-8 pass, done in registers before the first shared-memory store
    __syncthreads();  // twiddle tables
    // the upper half of every column is zero padding when 2 (n2 + H/2) >= n_in (all
    // columns for n_in <= H: the u / v / Lanczos vectors are at most half of M)
    dif_pass0_store<G::L1, RS>(v, r0, buf + cc * CS, tw1, 2 * (n2_0 + cc) + G::H >= a.n_in);
    __syncthreads();
    fft_run_inner_t<G::L1, false>(buf + fc * CS, tw1, ct, RS, csync);
  } else {
#pragma unroll
    for (int j = 0; j < NE; ++j)
      if (threadIdx.x + j * CT < N1 * kColW) buf[cc * CS + fsw(r0 + (RS) * j)] = v[j];
    __syncthreads();
    fft_run_t<G::L1, false>(buf + fc * CS, tw1, ct, RS, csync);
  }
  __syncthreads();
  // element j: column c = t & 7, k1 = (t >> 3) + (256 / 8) j; twiddle W_H^{n2 k1}
  const int c = threadIdx.x & (kColW - 1), k0 = threadIdx.x >> 3;
  const int n2 = n2_0 + c;
  const int nval = (N1 * kColW - threadIdx.x + CT - 1) / CT;
  twiddle_seq<LOGH, NE>(th, (long long)n2 * k0, (long long)n2 * (RS), nval, [&](int j, double2 w) {
    const int k1 = k0 + (RS) * j;
    const double2 z = buf[c * CS + fsw(rev_t<G::L1>(k1))];
    Yi[(size_t)n2 + (size_t)N2 * k1] = cmul(z, w);
  });
}

// ---- pass 3: inverse column FFTs + epilogue ------------------------------------------
// Epilogue modes: 0 correlation (out[t] = y_t - coef * prev[t], t < n_out, zero-filled to
// ld_out; partial sum of squares per CTA into part[blockIdx]) ; 1 hankelization
// (out[t] = sigma * y_t / c_t, t < N).
struct ColInvArgs {
  int mode;
  int n_out, ld_out;           // correlation output length and padded row length
  size_t out_stride;           // item stride of out
  double* out;
  const double* prev;          // correlation: previous vector (may be null; read before the grid
                               // dependency wait: no kernel of this correlation may write it)
  size_t prev_stride;
  const double* coef;          // correlation: per-item coefficient (device scalar), null -> 0
  double* part;                // correlation: partial sums of squares [items][gridDim.x]
  const double* sigma;         // hankelization: per-item sigma
  int N, L, K;                 // hankelization: weights
  const double* rcpc;          // hankelization: 1/c for c = 1..min(L, K) (plan table)
  const int* gate;             // device flag: nonzero -> the launch does nothing
  int has_tail;                // long-series Lanczos (one item): the last CTA runs lg_pro_tail
  LgProTail tail;
  // fused first CGS pass (long-series Lanczos, FRO): partial dots of this CTA's outputs with
  // every basis row of the tail's side into dpart[row][cta]; the last CTA sums them into dh
  // (null: the separate lg_dots kernel does it)
  const double* dbasis;
  int dld;
  double* dpart;
  double* dh;
};

template <int LOGH>
__global__ void __launch_bounds__(col_threads<LOGH>(), (LOGH >= 19) ? 1 : 3) lg_col_inv(const double2* __restrict__ Y, const double2* __restrict__ T1,
                                                       ColInvArgs a) {
  using G = Geo<LOGH>;
  constexpr int N1 = G::N1, N2 = G::N2, CS = N1 + 1;
  constexpr int CT = col_threads<LOGH>(), RS = CT / kColW;  // threads, row step of a thread
  constexpr int NE = (N1 * kColW + CT - 1) / CT;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double2* buf = reinterpret_cast<double2*>(smem_raw);
  __shared__ double red[CT / 32];
  const int n2_0 = blockIdx.x * kColW;
  const size_t item = blockIdx.y;
  const double2* Yi = Y + item * G::H;
  // thread t: column c = t & 7, rows n1 = (t >> 3) + RS j (as in lg_col_fwd)
  const int cc = threadIdx.x & (kColW - 1), r0 = threadIdx.x >> 3;
  // inputs that the preceding kernels of this correlation do not write, before the grid
  // dependency wait: the tables and (correlation) the previous Lanczos vector of the
  // recurrence term, written by an earlier half-step
  const TwSmem tw1 = load_tw2(T1, buf + kColW * CS, 2 * N1);
  double2 pr[NE];
  if (a.mode == 0) {
    const double* pv = a.prev ? a.prev + item * a.prev_stride : nullptr;
#pragma unroll
    for (int j = 0; j < NE; ++j) {
      const int t = 2 * (n2_0 + cc + N2 * (r0 + RS * j));
      const bool ok = threadIdx.x + j * CT < N1 * kColW;
      pr[j].x = (pv && ok && t < a.n_out) ? __ldg(pv + t) : 0.0;
      pr[j].y = (pv && ok && t + 1 < a.n_out) ? __ldg(pv + t + 1) : 0.0;
    }
  }
  pdl_wait(4);
  if (a.gate && *a.gate) return;
  double2 v[NE];
#pragma unroll
  for (int j = 0; j < NE; ++j)
    if (threadIdx.x + j * CT < N1 * kColW) v[j] = Yi[n2_0 + cc + N2 * (r0 + RS * j)];
#pragma unroll
  for (int j = 0; j < NE; ++j)
    if (threadIdx.x + j * CT < N1 * kColW) buf[cc * CS + fsw(rev_t<G::L1>(r0 + RS * j))] = v[j];
  __syncthreads();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int fc = threadIdx.x / RS, ct = threadIdx.x % RS;  // column of the FFT phase (as lg_col_fwd)
  const ColSync<CT> csync{1 + fc};
  // z[j] = H x packed point at row r0 + 32 j of this thread's column
  double2 z[NE];
  if constexpr (G::L1 >= 8) {
    // outermost inverse pass in registers: its outputs are exactly this thread's rows
    fft_run_inner_t<G::L1, true>(buf + fc * CS, tw1, ct, RS, csync);
    __syncthreads();
    dif_pass0_inverse_load<G::L1, RS>(z, r0, buf + cc * CS, tw1);
  } else {
    fft_run_t<G::L1, true>(buf + fc * CS, tw1, ct, RS, csync);
    __syncthreads();
#pragma unroll
    for (int j = 0; j < NE; ++j)
      if (threadIdx.x + j * CT < N1 * kColW) z[j] = buf[cc * CS + fsw(r0 + RS * j)];
  }
  constexpr double invH = 1.0 / (double)G::H;
  double ss = 0.0;
  const double cf = (a.mode == 0 && a.coef) ? a.coef[item] : 0.0;
  const double sg = (a.mode == 1) ? a.sigma[item] : 0.0;
  const int mn = a.L < a.K ? a.L : a.K;
  // thread t handles the packed points n = n2 + N2 n1 of its column c, rows n1 = r0 + 32 j:
  // real outputs t = 2n (z.x) and 2n + 1 (z.y)
  const int n2 = n2_0 + cc;
  if (a.mode == 0) {
    double* o = a.out + item * a.out_stride;
    double2 yv[NE];  // this thread's outputs (kept for the fused dots)
#pragma unroll
    for (int j = 0; j < NE; ++j) {
      yv[j] = make_double2(0.0, 0.0);
      if (threadIdx.x + j * CT < N1 * kColW) {
        const int n1 = r0 + RS * j;
        const int t = 2 * (n2 + N2 * n1);
        if (t < a.ld_out) {
          const double y = (t < a.n_out) ? fma(-cf, pr[j].x, z[j].x * invH) : 0.0;
          o[t] = y;
          yv[j].x = y;
          ss = fma(y, y, ss);
        }
        if (t + 1 < a.ld_out) {
          const double y = (t + 1 < a.n_out) ? fma(-cf, pr[j].y, z[j].y * invH) : 0.0;
          o[t + 1] = y;
          yv[j].y = y;
          ss = fma(y, y, ss);
        }
      }
    }
    if (a.part) {
      ss = warp_sum(ss);
      if (lane == 0) red[w] = ss;
      __syncthreads();  // also: every thread is done with buf (reused below)
      if (threadIdx.x == 0) {
        double s = 0.0;
        for (int i = 0; i < CT / 32; ++i) s += red[i];
        a.part[item * gridDim.x + blockIdx.x] = s;
      }
      int nbd = 0;
      if (a.dbasis) {
        // fused first CGS pass: <basis row b, r> over this CTA's outputs (16-byte pairs
        // t, t + 1 of 8 columns: 128-byte row segments), two rows' loads in flight; per-warp
        // sums into buf [row][warp], then one fixed-order sum per row -> dpart[row][cta]
        nbd = lg_nb(a.tail.sc, a.tail.side);
        double* wred = reinterpret_cast<double*>(buf);
        // streaming (evict-first) loads: measured faster here than lg_dots' evict_last
        // (cfg3 59.9 vs 61.1 ms), although lg_update then finds fewer rows in L2
        for (int b0 = 0; b0 < nbd; b0 += 2) {
          double2 x[2][NE];
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const double* brow = a.dbasis + (size_t)(b0 + q) * a.dld;
#pragma unroll
            for (int j = 0; j < NE; ++j) {
              const int t = 2 * (n2 + N2 * (r0 + RS * j));
              x[q][j] = (b0 + q < nbd && threadIdx.x + j * CT < N1 * kColW && t < a.ld_out)
                            ? __ldcs(reinterpret_cast<const double2*>(brow + t))
                            : make_double2(0.0, 0.0);
            }
          }
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            double d = 0.0;
#pragma unroll
            for (int j = 0; j < NE; ++j) d = fma(x[q][j].x, yv[j].x, fma(x[q][j].y, yv[j].y, d));
            d = warp_sum(d);
            if (lane == 0 && b0 + q < nbd) wred[(b0 + q) * (CT / 32) + w] = d;
          }
        }
        __syncthreads();
        for (int row = threadIdx.x; row < nbd; row += CT) {
          double sd = 0.0;
          for (int i = 0; i < CT / 32; ++i) sd += wred[row * (CT / 32) + i];
          a.dpart[(size_t)row * gridDim.x + blockIdx.x] = sd;
        }
      }
      if (a.has_tail) {
        __shared__ int lastf;
        if (last_cta(&a.tail.sc->done_inv, gridDim.x, &lastf)) {
          lg_pro_tail(a.part, gridDim.x, a.tail, red);
          if (a.dbasis) {
            // h[row] = sum of the CTAs' partials in a fixed order: four threads per row,
            // thread s of the four adds partials s, s + 4, ... (all loads in flight), then
            // a fixed two-level shuffle tree; 128 rows per pass of the CTA
            const int sub = threadIdx.x & 3;
            for (int row0 = 0; row0 < nbd; row0 += CT / 4) {
              const int row = row0 + (threadIdx.x >> 2);
              double sd = 0.0;
              if (row < nbd) {
                const double* pr0 = a.dpart + (size_t)row * gridDim.x;
                for (int i = sub; i < (int)gridDim.x; i += 16) {
                  double x[4];
#pragma unroll
                  for (int u = 0; u < 4; ++u) x[u] = (i + 4 * u < (int)gridDim.x) ? __ldcg(pr0 + i + 4 * u) : 0.0;
#pragma unroll
                  for (int u = 0; u < 4; ++u) sd += x[u];
                }
              }
              sd += __shfl_xor_sync(0xffffffffu, sd, 1);
              sd += __shfl_xor_sync(0xffffffffu, sd, 2);
              if (sub == 0 && row < nbd) a.dh[row] = sd;
            }
          }
          if (threadIdx.x == 0) a.tail.sc->done_inv = 0;
        }
      }
    }
  } else {
    // g_t = sigma y_t / c_t, c_t = min(t + 1, min(L, K), N - t) (R2)
    double* o = a.out + item * a.out_stride;
    const double scale = sg * invH;
#pragma unroll
    for (int j = 0; j < NE; ++j) {
      if (threadIdx.x + j * CT < N1 * kColW) {
        const int n1 = r0 + RS * j;
        const int t = 2 * (n2 + N2 * n1);
        if (t < a.N) {
          const int c0 = min(min(t + 1, mn), a.N - t);
          o[t] = z[j].x * scale * __ldg(a.rcpc + c0 - 1);
          if (t + 1 < a.N) {
            const int c1 = min(min(t + 2, mn), a.N - t - 1);
            o[t + 1] = z[j].y * scale * __ldg(a.rcpc + c1 - 1);
          }
        }
      }
    }
  }
}

// ---- register radix-16 x 16 column passes for N1 = 256 (H = 2^16, 2^17: cfg5) --------
// The hankelization's column FFTs with one shared-memory exchange instead of three radix-8 /
// radix-4 passes (the column kernels above are bound by shared-memory wavefronts): a
// 256-point column is 16 x 16; thread (c, q) of the CTA's CW columns first holds rows
// q + 16 j of column c (a 16-point DFT in registers, dft16, then the internal twiddles
// W_256^{q k}), one transposing exchange through shared memory, then frequencies / rows
// q + 16 j (the second 16-point DFT).  Same layouts and results as lg_col_fwd / lg_col_inv
// (mode 1): Y[n2 + N2 k1] natural order, the DFT split of PAPER.md:473-509.
// CW columns per CTA (16 x CW threads): 16 (256 threads, 2 CTAs/SM) or 8 (128 threads, 4 CTAs/SM)
constexpr int kCS16 = 257;    // column stride in shared memory (16-byte units, odd)
static size_t col16_smem(int cw) { return ((size_t)cw * kCS16 + tw2_entries(512)) * 16; }

template <int LOGH, int CW>
__global__ void __launch_bounds__(16 * CW, 512 / (16 * CW)) lg_col16_fwd(ColFwdArgs args, const double2* __restrict__ T1,
                                                            const double2* __restrict__ TWH) {
  using G = Geo<LOGH>;
  static_assert(G::N1 == 256, "radix-16 x 16 columns");
  constexpr int N2 = G::N2;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double2* buf = reinterpret_cast<double2*>(smem_raw);
  const TwSmem tw1 = load_tw2(T1, buf + CW * kCS16, 512);  // W_512^t
  pdl_wait(1);
  if (args.gate && *args.gate) return;
  const ColFwdIn a = blockIdx.z ? args.in[1] : args.in[0];
  const int c = threadIdx.x & (CW - 1), q = threadIdx.x / CW;
  const int n2 = blockIdx.x * CW + c;
  const double* xi = a.x + (size_t)blockIdx.y * a.xs;
  double2* Yi = a.Y + (size_t)blockIdx.y * G::H;
  const bool rvec = a.vec && ((reinterpret_cast<uintptr_t>(xi) & 15) == 0);
  // rows n1 = q + 16 j >= 128 (j >= 8) are zero padding when 2 (n2 + H/2) >= n_in
  const bool half = 2 * n2 + G::H >= a.n_in;
  double2 v[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const int i0 = 2 * (n2 + N2 * (q + 16 * j));
    if (j >= 8 && half) {
      v[j] = make_double2(0.0, 0.0);
    } else if (rvec && i0 + 1 < a.n_in) {
      v[j] = __ldcs(reinterpret_cast<const double2*>(xi + i0));
    } else {
      v[j].x = (i0 < a.n_in) ? __ldcs(xi + i0) : 0.0;
      v[j].y = (i0 + 1 < a.n_in) ? __ldcs(xi + i0 + 1) : 0.0;
    }
  }
  __syncthreads();  // twiddle table
  if (half) dft16<false, true>(v);
  else dft16<false, false>(v);
  twiddle16<false>(v, tw1(2 * q));  // v[k] *= W_256^{q k}
  double2* col = buf + c * kCS16;
#pragma unroll
  for (int k = 0; k < 16; ++k) col[q * 16 + k] = v[k];
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = col[i * 16 + q];
  dft16<false, false>(v);  // v[j] = column spectrum at k1 = q + 16 j
  twiddle_seq<LOGH, 16>(TWH, (long long)n2 * q, (long long)n2 * 16, 16, [&](int j, double2 w) {
    Yi[(size_t)n2 + (size_t)N2 * (q + 16 * j)] = cmul(v[j], w);
  });
}

// Inverse columns + hankelization epilogue (lg_col_inv mode 1): g_t = sigma y_t / c_t.
template <int LOGH, int CW>
__global__ void __launch_bounds__(16 * CW, 512 / (16 * CW)) lg_col16_hank(const double2* __restrict__ Y,
                                                             const double2* __restrict__ T1, ColInvArgs a) {
  using G = Geo<LOGH>;
  static_assert(G::N1 == 256, "radix-16 x 16 columns");
  constexpr int N2 = G::N2;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double2* buf = reinterpret_cast<double2*>(smem_raw);
  const TwSmem tw1 = load_tw2(T1, buf + CW * kCS16, 512);
  pdl_wait(4);
  if (a.gate && *a.gate) return;
  const size_t item = blockIdx.y;
  const double2* Yi = Y + item * G::H;
  const int c = threadIdx.x & (CW - 1), q = threadIdx.x / CW;
  const int n2 = blockIdx.x * CW + c;
  double2 v[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) v[j] = __ldcs(Yi + (size_t)n2 + (size_t)N2 * (q + 16 * j));  // k1 = q + 16 j
  __syncthreads();  // twiddle table
  dft16<true, false>(v);
  twiddle16<true>(v, tw1(2 * q));  // v[n] *= W_256^{-q n}
  double2* col = buf + c * kCS16;
#pragma unroll
  for (int n = 0; n < 16; ++n) col[q * 16 + n] = v[n];
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = col[i * 16 + q];
  dft16<true, false>(v);  // v[j] = H x packed point n2 + N2 (q + 16 j)
  const double scale = a.sigma[item] * (1.0 / (double)G::H);
  const int mn = a.L < a.K ? a.L : a.K;
  double* o = a.out + item * a.out_stride;
  const bool ovec = (reinterpret_cast<uintptr_t>(o) & 15) == 0;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const int t = 2 * (n2 + N2 * (q + 16 * j));
    if (t < a.N) {
      const int c0 = min(min(t + 1, mn), a.N - t);
      const double g0 = v[j].x * scale * __ldg(a.rcpc + c0 - 1);
      if (t + 1 < a.N) {
        const int c1 = min(min(t + 2, mn), a.N - t - 1);
        const double g1 = v[j].y * scale * __ldg(a.rcpc + c1 - 1);
        if (ovec) {
          __stcs(reinterpret_cast<double2*>(o + t), make_double2(g0, g1));
        } else {
          __stcs(o + t, g0);
          __stcs(o + t + 1, g1);
        }
      } else {
        __stcs(o + t, g0);
      }
    }
  }
}

// ---- pass 2: row pairs ----------------------------------------------------------------
// Row A in [0, N1/2] with its partner B = N1 - A (B == A for A = 0 and A = N1/2).  Modes:
// 0 spectrum (write F^[0..H] natural order), 1 correlation with F^, 2 product of the
// spectra of two buffers (Ya * Yb, result in Yb).
struct RowArgs {
  int mode;
  double2* Ya;          // buffer of the (first) vector, [items][H]
  double2* Yb;          // mode 2: second buffer
  const double2* spec;  // mode 1: F^ [items or 1][H+1]
  size_t spec_stride;   // 0 -> shared spectrum for all items
  double2* spec_out;    // mode 0: [items][H+1]
  const int* gate;      // device flag: nonzero -> the launch does nothing
};

__device__ __forceinline__ int partner_k2(int A, int k2, int N2) {
  return (A == 0) ? ((N2 - k2) & (N2 - 1)) : (N2 - 1 - k2);
}

// The pair step for pairs k2 = k0, k0 + ks, ... of rows (rA, rB[, cA, cB]) already
// transformed (digit-reversed).  WA = W_M^A; W_M^p = WA W_{2 N2}^{k2} (tw2).
// Spectrum values of the pairs a thread takes in the pair step (k2 = k0 + ks i, i < NI),
// loaded ahead (mode 1; the stored spectrum does not depend on the preceding kernels, so
// the loads can be issued before the grid dependency wait and overlap its latency).
template <int LOGH, int NI>
struct RowSpecPre {
  double2 Fp[NI], Fq[NI];
  __device__ __forceinline__ void load(const RowArgs& a, size_t item, int A, bool two, int k0, int ks) {
    using G = Geo<LOGH>;
    constexpr int N1 = G::N1, N2 = G::N2, H = G::H;
    const int npairs = two ? N2 : ((A == 0) ? N2 / 2 + 1 : N2 / 2);
    const double2* F = a.spec + item * a.spec_stride;
#pragma unroll
    for (int i = 0; i < NI; ++i) {
      const int k2 = k0 + ks * i;
      const long long p = (long long)A + (long long)N1 * k2;
      const long long q = (p == 0) ? H : H - p;
      if (k2 < npairs) { Fp[i] = __ldg(F + p); Fq[i] = __ldg(F + q); }
    }
  }
};

// pre: NI > 0 -> the thread's pairs are k2 = k0 + ks i, i < NI (unrolled), mode 1 reads the
// spectrum from pre; NI = 0 -> runtime loop, spectrum loads in place.
template <int LOGH, int NI = 0>
__device__ __forceinline__ void row_pair_step(const RowArgs& a, size_t item, int A, bool two, double2 WA,
                                              const TwSmem& tw2, double2* rA, double2* rB, double2* cA, double2* cB,
                                              int k0, int ks, const RowSpecPre<LOGH, (NI > 0 ? NI : 1)>* pre = nullptr) {
  using G = Geo<LOGH>;
  constexpr int N1 = G::N1, N2 = G::N2, H = G::H;
  const int npairs = two ? N2 : ((A == 0) ? N2 / 2 + 1 : N2 / 2);
  double2* rowB = two ? rB : rA;
  double2* rowBc = two ? cB : cA;
  const double2* F = (a.mode == 1) ? a.spec + item * a.spec_stride : nullptr;
  double2* Fo = (a.mode == 0) ? a.spec_out + item * (size_t)(H + 1) : nullptr;
#pragma unroll
  for (int i = 0; i < (NI > 0 ? NI : 1 << 30); ++i) {
    const int k2 = k0 + ks * i;
    if (k2 >= npairs) break;
    const int k2q = partner_k2(A, k2, N2);
    const int pr = fsw(rev_t<G::L2>(k2)), qr = fsw(rev_t<G::L2>(k2q));
    const long long p = (long long)A + (long long)N1 * k2;
    const long long q = (p == 0) ? H : H - p;
    double2 Fp, Fq;
    if (a.mode == 1) {
      if constexpr (NI > 0) { Fp = pre->Fp[i]; Fq = pre->Fq[i]; }
      else { Fp = __ldg(F + p); Fq = __ldg(F + q); }
    }
    const double2 W = cmul(WA, tw2(k2));  // exp(-2 pi i p / M), p = A + N1 k2
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
        Yp = cmulc(Fp, Xp);
        Yq = cmulc(Fq, Xq);
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

// Row pairs, CTA-wide FFTs (one item at a time: 257..513 CTAs of 256 threads keep the
// GPU busier than warp-level rows would).  Smem: 4 rows, tw2, W_H table.
template <int LOGH>
__global__ void __launch_bounds__(kThreads) lg_row_cta(const double2* __restrict__ T2, const double2* __restrict__ TWH,
                                                       const double2* __restrict__ TWA, RowArgs a) {
  using G = Geo<LOGH>;
  constexpr int N1 = G::N1, N2 = G::N2;
  constexpr int NE = (N2 + kThreads - 1) / kThreads;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double2* bA = reinterpret_cast<double2*>(smem_raw);  // row A of Ya
  double2* bB = bA + N2;                                // row B of Ya
  double2* cA = bB + N2;                                // mode 2: row A of Yb
  double2* cB = cA + N2;                                // mode 2: row B of Yb
  const double2* th = TWH;
  const int A = blockIdx.x, B = (N1 - A) & (N1 - 1);
  const bool two = (A != B);
  const size_t item = blockIdx.y;
  // constant inputs first (tables, the stored spectrum of the pair step), then the wait
  // for the preceding kernel's output
  const TwSmem tw2 = load_tw2(T2, cB + N2, 2 * N2);
  const double2 WA = __ldg(TWA + A);
  RowSpecPre<LOGH, NE> pre;
  if (a.mode == 1) pre.load(a, item, A, two, threadIdx.x, kThreads);
  pdl_wait(2);
  if (a.gate && *a.gate) return;
  double2* Ya = a.Ya + item * G::H;
  double2* Yb = (a.mode == 2) ? a.Yb + item * G::H : nullptr;
  if constexpr (G::L2 >= 10) {
    if (a.mode != 2) {
      // rows A and B concurrently, 128 threads each (named barriers): every thread holds
      // the 8 points t + 128 e of its row, i.e. one butterfly of the outermost radix-8 pass,
      // done in registers straight from the load; the inverse ends the same way into the
      // twiddled store
      constexpr int NEH = N2 / 128;
      const int half = threadIdx.x >> 7, t = threadIdx.x & 127;
      const bool active = (half == 0) || two;
      double2* row = half ? bB : bA;
      const int rid = half ? B : A;
      double2 v[NEH];
      if (active) {
        const double2* src = Ya + (size_t)rid * N2;
#pragma unroll
        for (int e = 0; e < NEH; ++e) v[e] = src[t + 128 * e];
      }
      __syncthreads();  // twiddle tables
      const NamedSync128 sync{1 + half};
      if (active) {
        dif_pass0_store<G::L2, 128>(v, t, row, tw2);
        sync();
        fft_run_inner_t<G::L2, false>(row, tw2, t, 128, sync);
      }
      __syncthreads();
      row_pair_step<LOGH, NE>(a, item, A, two, WA, tw2, bA, bB, cA, cB, threadIdx.x, kThreads, &pre);
      if (a.mode == 0) return;
      __syncthreads();
      if (active) {
        fft_run_inner_t<G::L2, true>(row, tw2, t, 128, sync);
        dif_pass0_inverse_load<G::L2, 128>(v, t, row, tw2);
        double2* Yo = Ya + (size_t)rid * N2;
        twiddle_seq<LOGH, NEH>(th, (long long)rid * t, (long long)rid * 128, NEH, [&](int e, double2 w) {
          Yo[t + 128 * e] = cmulc(v[e], w);
        });
      }
      return;
    }
  }
  // all rows' loads in flight before the shared-memory stores
  double2 v[4][NE];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const double2* src = ((r >> 1) ? Yb : Ya) + (size_t)((r & 1) ? B : A) * N2;
    const bool use = (r >> 1) ? (a.mode == 2) : true;
    const bool use2 = (r & 1) ? two : true;
#pragma unroll
    for (int j = 0; j < NE; ++j) {
      const int i = threadIdx.x + j * kThreads;
      if (use && use2 && i < N2) v[r][j] = src[i];
    }
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    double2* dst = bA + r * N2;
    const bool use = ((r >> 1) ? (a.mode == 2) : true) && ((r & 1) ? two : true);
#pragma unroll
    for (int j = 0; j < NE; ++j) {
      const int i = threadIdx.x + j * kThreads;
      if (use && i < N2) dst[fsw(i)] = v[r][j];
    }
  }
  __syncthreads();
  fft_run_t<G::L2, false>(bA, tw2, threadIdx.x, blockDim.x, CtaSync());
  if (two) fft_run_t<G::L2, false>(bB, tw2, threadIdx.x, blockDim.x, CtaSync());
  if (a.mode == 2) {
    fft_run_t<G::L2, false>(cA, tw2, threadIdx.x, blockDim.x, CtaSync());
    if (two) fft_run_t<G::L2, false>(cB, tw2, threadIdx.x, blockDim.x, CtaSync());
  }
  row_pair_step<LOGH, NE>(a, item, A, two, WA, tw2, bA, bB, cA, cB, threadIdx.x, kThreads, &pre);
  if (a.mode == 0) return;
  __syncthreads();
  double2* oA = (a.mode == 2) ? cA : bA;
  double2* oB = (a.mode == 2) ? cB : bB;
  double2* Yo = (a.mode == 2) ? Yb : Ya;
  fft_run_t<G::L2, true>(oA, tw2, threadIdx.x, blockDim.x, CtaSync());
  if (two) fft_run_t<G::L2, true>(oB, tw2, threadIdx.x, blockDim.x, CtaSync());
  const int nval = (N2 - (int)threadIdx.x + kThreads - 1) / kThreads;
  twiddle_seq<LOGH, NE>(th, (long long)A * threadIdx.x, (long long)A * kThreads, nval, [&](int j, double2 w) {
    const int n2 = threadIdx.x + j * kThreads;
    Yo[(size_t)A * N2 + n2] = cmulc(oA[fsw(n2)], w);
  });
  if (two)
    twiddle_seq<LOGH, NE>(th, (long long)B * threadIdx.x, (long long)B * kThreads, nval, [&](int j, double2 w) {
      const int n2 = threadIdx.x + j * kThreads;
      Yo[(size_t)B * N2 + n2] = cmulc(oB[fsw(n2)], w);
    });
}

// Row pairs with warp-level FFTs: each CTA takes G = warps / R row pairs (R = rows per
// pair: 2, or 4 in mode 2); warp g R + j loads and transforms row j of pair g on its own
// (no CTA barrier inside the FFTs), the pair step runs on the 32 R threads of the pair,
// and warps 0 / 1 of the pair run the inverse transforms of rows A / B and write them
// back with the conjugate twiddle.  Smem: one row per warp, tw2, W_H table.
template <int LOGH>
__global__ void __launch_bounds__(kThreads) lg_row_warp(const double2* __restrict__ T2,
                                                        const double2* __restrict__ TWH,
                                                        const double2* __restrict__ TWA, RowArgs a) {
  pdl_wait(3);
  if (a.gate && *a.gate) return;
  using Gm = Geo<LOGH>;
  constexpr int N1 = Gm::N1, N2 = Gm::N2;
  constexpr int NE = (N2 + 31) / 32;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  constexpr int nw = kWarps;
  double2* rows = reinterpret_cast<double2*>(smem_raw);  // nw rows of N2
  const double2* th = TWH;
  const TwSmem tw2 = load_tw2(T2, rows + (size_t)nw * N2, 2 * N2);
  const int R = (a.mode == 2) ? 4 : 2, G = nw / R;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = w / R, j = w - g * R;
  const int A = blockIdx.x * G + g, B = (N1 - A) & (N1 - 1);
  const bool valid = A <= N1 / 2, two = (A != B);
  const size_t item = blockIdx.y;
  double2* Ya = a.Ya + item * Gm::H;
  double2* Yb = (a.mode == 2) ? a.Yb + item * Gm::H : nullptr;
  double2* rA = rows + (size_t)(g * R) * N2;  // row A of Ya, row B of Ya, row A of Yb, row B of Yb
  double2* rB = rA + N2;
  double2* cA = rA + 2 * N2;
  double2* cB = rA + 3 * N2;
  const bool mine = valid && (two || !(j & 1));
  double2 v[NE];
  if (mine) {
    const double2* src = ((j >> 1) ? Yb : Ya) + (size_t)((j & 1) ? B : A) * N2;
    const bool dead = (a.mode == 2) && !(j >> 1);  // product mode: Ya is not read again
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      const int i = lane + 32 * e;
      if (i < N2) v[e] = dead ? __ldcs(src + i) : src[i];
    }
  }
  __syncthreads();  // tables
  if (mine) {
    double2* dst = rows + (size_t)w * N2;
    if constexpr (Gm::L2 >= 8) {  // outermost radix-8 pass in registers (lane holds lane + 32 e)
      dif_pass0_store<Gm::L2, 32>(v, lane, dst, tw2);
      __syncwarp();
      fft_run_inner_t<Gm::L2, false>(dst, tw2, lane, 32, WarpSync());
    } else {
#pragma unroll
      for (int e = 0; e < NE; ++e) {
        const int i = lane + 32 * e;
        if (i < N2) dst[fsw(i)] = v[e];
      }
      __syncwarp();
      fft_run_t<Gm::L2, false>(dst, tw2, lane, 32, WarpSync());
    }
  }
  __syncthreads();
  if (valid) {
    const double2 WA = __ldg(TWA + A);
    row_pair_step<LOGH>(a, item, A, two, WA, tw2, rA, rB, cA, cB, j * 32 + lane, 32 * R);
  }
  if (a.mode == 0) return;
  __syncthreads();
  if (a.mode == 2) {
    // inverse of rows A (warps 0, 1 of the group) and B (warps 2, 3) of Yb, two warps per
    // row (named barrier per row): all four warps of the pair busy
    const int half = j >> 1;
    if (valid && (two || half == 0)) {
      double2* o = half ? cB : cA;
      const int row = half ? B : A;
      double2* Yo = Yb + (size_t)row * N2;
      const int tid64 = ((j & 1) << 5) | lane;
      const NamedSync64 sync{1 + 2 * g + half};
      constexpr int NE2 = (N2 + 63) / 64;
      const int nval = (N2 - tid64 + 63) / 64;
      if constexpr (Gm::L2 >= 9) {  // outermost inverse pass in registers: thread's n2 = tid64 + 64 e
        fft_run_inner_t<Gm::L2, true>(o, tw2, tid64, 64, sync);
        double2 x[NE2];
        dif_pass0_inverse_load<Gm::L2, 64>(x, tid64, o, tw2);
        twiddle_seq<LOGH, NE2>(th, (long long)row * tid64, (long long)row * 64, nval, [&](int e, double2 w) {
          Yo[tid64 + 64 * e] = cmulc(x[e], w);
        });
      } else {
        fft_run_t<Gm::L2, true>(o, tw2, tid64, 64, sync);
        twiddle_seq<LOGH, NE2>(th, (long long)row * tid64, (long long)row * 64, nval, [&](int e, double2 w) {
          const int n2 = tid64 + 64 * e;
          Yo[n2] = cmulc(o[fsw(n2)], w);
        });
      }
    }
  } else if (valid && j < 2 && (two || j == 0)) {
    double2* o = j ? rB : rA;
    const int row = j ? B : A;
    double2* Yo = Ya + (size_t)row * N2;
    fft_run_t<Gm::L2, true>(o, tw2, lane, 32, WarpSync());
    const int nval = (N2 - lane + 31) / 32;
    twiddle_seq<LOGH, NE>(th, (long long)row * lane, (long long)row * 32, nval, [&](int e, double2 w) {
      const int n2 = lane + 32 * e;
      Yo[n2] = cmulc(o[fsw(n2)], w);
    });
  }
}


// ---- shared-memory sizes, attributes, dispatch ------------------------------------------
static int ilog2(long long v) {
  int l = 0;
  while ((1LL << l) < v) ++l;
  return l;
}
static size_t col_smem(int logH) {
  const int N1 = 1 << (logH / 2);
  return ((size_t)kColW * (N1 + 1) + tw2_entries(2 * N1)) * 16;
}
static size_t row_cta_smem(int logH) {
  const int N2 = 1 << (logH - logH / 2);
  return ((size_t)4 * N2 + tw2_entries(2 * N2)) * 16;
}
static size_t row_warp_smem(int logH) {
  const int N2 = 1 << (logH - logH / 2);
  return ((size_t)kWarps * N2 + tw2_entries(2 * N2)) * 16;
}

#define SSA_LG_DISPATCH(logH, CALL)                                                               \
  switch (logH) {                                                                                 \
    case 6: CALL(6); break; case 7: CALL(7); break; case 8: CALL(8); break; case 9: CALL(9); break; \
    case 10: CALL(10); break; case 11: CALL(11); break; case 12: CALL(12); break;                 \
    case 13: CALL(13); break; case 14: CALL(14); break; case 15: CALL(15); break;                 \
    case 16: CALL(16); break; case 17: CALL(17); break; case 18: CALL(18); break;                 \
    case 19: CALL(19); break; default: CALL(20); break;                                           \
  }

cudaError_t large_set_attributes(int N1, int N2) {
  const int logH = ilog2((long long)N1 * N2);
  cudaError_t e = cudaSuccess;
#define SSA_LG_ATTR(LG)                                                                            \
  do {                                                                                             \
    if ((e = raise_smem_limit(lg_col_fwd<LG>, col_smem(LG)))) return e;                            \
    if ((e = raise_smem_limit(lg_col_inv<LG>, col_smem(LG)))) return e;                            \
    if ((e = raise_smem_limit(lg_row_cta<LG>, row_cta_smem(LG)))) return e;                        \
    if ((e = raise_smem_limit(lg_row_warp<LG>, row_warp_smem(LG)))) return e;                      \
  } while (0)
  SSA_LG_DISPATCH(logH, SSA_LG_ATTR)
#undef SSA_LG_ATTR
  if (logH == 16 || logH == 17) {
    if ((e = raise_smem_limit(lg_col16_fwd<16, 16>, col16_smem(16)))) return e;
    if ((e = raise_smem_limit(lg_col16_hank<16, 16>, col16_smem(16)))) return e;
    if ((e = raise_smem_limit(lg_col16_fwd<17, 16>, col16_smem(16)))) return e;
    if ((e = raise_smem_limit(lg_col16_hank<17, 16>, col16_smem(16)))) return e;
    if ((e = raise_smem_limit(lg_col16_fwd<16, 8>, col16_smem(8)))) return e;
    if ((e = raise_smem_limit(lg_col16_hank<16, 8>, col16_smem(8)))) return e;
    if ((e = raise_smem_limit(lg_col16_fwd<17, 8>, col16_smem(8)))) return e;
    if ((e = raise_smem_limit(lg_col16_hank<17, 8>, col16_smem(8)))) return e;
  }
  return e;
}

// ---- host-side drivers ----------------------------------------------------------------
// Basis rows the fused first CGS pass of lg_col_inv can hold per-warp sums for (its column
// buffer, reused after the inverse FFT): 0 if the transform's column kernel is too small.
int large_fused_dots_rows(long long H) {
  int logH = 0;
  while ((1ll << logH) < H) ++logH;
  const int l1 = logH / 2, ct = logH >= 19 ? 512 : 256;
  return (int)((size_t)kColW * ((1 << l1) + 1) * 16 / ((size_t)(ct / 32) * 8));
}

void large_geom(const Plan& p, int* N1, int* N2) {
  const int l = ilog2(p.H);
  *N1 = 1 << (l / 2);
  *N2 = (int)(p.H / *N1);
}

// x is 16-byte aligned (the kernel checks each row's start)
static int vec16(const double* x, size_t) { return (reinterpret_cast<uintptr_t>(x) & 15) == 0; }

static void col_fwd(const Plan& p, const ColFwdArgs& ca, int nz, int items, cudaStream_t s) {
  const int logH = ilog2(p.H);
  const int N2 = 1 << (logH - logH / 2);
  const dim3 grid(N2 / kColW, items, nz);
#define SSA_LG_CF(LG) launch_pdl(lg_col_fwd<LG>, dim3(grid), dim3(col_threads<LG>()), col_smem(LG), s, ca, p.d_tw1, p.d_tw4)
  SSA_LG_DISPATCH(logH, SSA_LG_CF)
#undef SSA_LG_CF
}
static void col_inv(const Plan& p, const double2* Y, const ColInvArgs& ca, int items, cudaStream_t s) {
  const int logH = ilog2(p.H);
  const int N2 = 1 << (logH - logH / 2);
  const dim3 grid(N2 / kColW, items);
#define SSA_LG_CI(LG) launch_pdl(lg_col_inv<LG>, dim3(grid), dim3(col_threads<LG>()), col_smem(LG), s, Y, p.d_tw1, ca)
  SSA_LG_DISPATCH(logH, SSA_LG_CI)
#undef SSA_LG_CI
}
static void rows(const Plan& p, const RowArgs& ra, int items, bool warp_rows, cudaStream_t s) {
  const int logH = ilog2(p.H);
  const int N1 = 1 << (logH / 2);
  if (warp_rows) {
    const int G = kWarps / (ra.mode == 2 ? 4 : 2);
    const dim3 grid((N1 / 2 + G) / G, items);
#define SSA_LG_RW(LG) launch_pdl(lg_row_warp<LG>, dim3(grid), dim3(kThreads), row_warp_smem(LG), s, p.d_tw2, p.d_tw4, p.d_twp, ra)
    SSA_LG_DISPATCH(logH, SSA_LG_RW)
#undef SSA_LG_RW
  } else {
    const dim3 grid(N1 / 2 + 1, items);
#define SSA_LG_RC(LG) launch_pdl(lg_row_cta<LG>, dim3(grid), dim3(kThreads), row_cta_smem(LG), s, p.d_tw2, p.d_tw4, p.d_twp, ra)
    SSA_LG_DISPATCH(logH, SSA_LG_RC)
#undef SSA_LG_RC
  }
}

cudaError_t large_spectrum(const Plan& p, const double* series, double2* spec, int items, cudaStream_t s) {
  double2* Y = p.d_lbuf;
  for (int i0 = 0; i0 < items; i0 += p.lbuf_items) {
    const int ni = std::min(items - i0, p.lbuf_items);
    ColFwdArgs ca{};
    ca.in[0] = ColFwdIn{series + (size_t)i0 * p.N, (size_t)p.N, (int)p.N, Y, vec16(series, p.N)};
    col_fwd(p, ca, 1, ni, s);
    RowArgs ra{0, Y, nullptr, nullptr, 0, spec + (size_t)i0 * (p.H + 1), nullptr};
    rows(p, ra, ni, false, s);
  }
  return cudaGetLastError();
}

// y[item] = X x (transpose 0) or X^T x (1) for items sharing one spectrum stride.
cudaError_t large_correlate(const Plan& p, const double2* spec, size_t spec_stride, const double* x, size_t xs, int n_in,
                            double* out, size_t os, int n_out, int ld_out, const double* prev, size_t ps,
                            const double* coef, double* part, int items, cudaStream_t s, const int* gate) {
  int N1, N2;
  large_geom(p, &N1, &N2);
  double2* Y = p.d_lbuf;
  for (int i0 = 0; i0 < items; i0 += p.lbuf_items) {
    const int ni = std::min(items - i0, p.lbuf_items);
    ColFwdArgs cf{};
    cf.in[0] = ColFwdIn{x + (size_t)i0 * xs, xs, n_in, Y, vec16(x, xs)};
    cf.gate = gate;
    col_fwd(p, cf, 1, ni, s);
    RowArgs ra{1, Y, nullptr, spec + (size_t)i0 * spec_stride, spec_stride, nullptr, gate};
    rows(p, ra, ni, ni >= 8, s);
    ColInvArgs ca{};
    ca.mode = 0;
    ca.n_out = n_out; ca.ld_out = ld_out; ca.out_stride = os; ca.out = out + (size_t)i0 * os;
    ca.prev = prev ? prev + (size_t)i0 * ps : nullptr; ca.prev_stride = ps;
    ca.coef = coef ? coef + i0 : nullptr;
    ca.part = part ? part + (size_t)i0 * (N2 / kColW) : nullptr;
    ca.gate = gate;
    col_inv(p, Y, ca, ni, s);
  }
  return cudaGetLastError();
}

// One Lanczos half-step correlation (one series): x = r * (*nrm.inv) (normalization of the
// previous half-step's vector fused into the column FFT, written to nrm.basis / nrm.cur),
// y = correlation - coef * prev into out, and the decision tail (lg_pro_tail) in the last
// CTA of the inverse column pass.
cudaError_t large_correlate_lanczos(const Plan& p, const double2* spec, const double* r, int n_in, const LgNorm& nrm,
                                    double* out, int n_out, int ld_out, const double* prev, const double* coef,
                                    double* part, const LgProTail& tail, cudaStream_t s, const double* dbasis,
                                    int dld, double* dpart, double* dh) {
  int N1, N2;
  large_geom(p, &N1, &N2);
  double2* Y = p.d_lbuf;
  ColFwdArgs cf{};
  cf.in[0] = ColFwdIn{r, 0, n_in, Y, vec16(r, 0), nrm};
  col_fwd(p, cf, 1, 1, s);
  RowArgs ra{1, Y, nullptr, spec, 0, nullptr, nullptr};
  rows(p, ra, 1, false, s);
  ColInvArgs ca{};
  ca.mode = 0;
  ca.n_out = n_out; ca.ld_out = ld_out; ca.out_stride = 0; ca.out = out;
  ca.prev = prev; ca.prev_stride = 0;
  ca.coef = coef;
  ca.part = part;
  ca.has_tail = 1;
  ca.tail = tail;
  ca.dbasis = dbasis;
  ca.dld = dld;
  ca.dpart = dpart;
  ca.dh = dh;
  col_inv(p, Y, ca, 1, s);
  return cudaGetLastError();
}

cudaError_t large_hankelize(Plan& p, const double* sigma, const double* U, const double* V, size_t nterm_total,
                            double* out, cudaStream_t s) {
  // Batches of `per` terms (two H-point buffers each) alternate between the caller's
  // stream and a second one with their own buffers, so one batch's launch tails overlap
  // the next batch's work.  SSA_HANK_PER overrides the batch size (tuning).
  const int cap = std::max(1, p.lbuf_items / 4);
  int per = std::max(1, std::min(cap, p.hank_per));
  // H <= 2^17: keep the two buffers of the batches in flight on both streams (2 x per x 32 H
  // bytes) near half of the 126 MB L2 (cfg5: 16 terms per batch measured best, 8-16 within 1 %)
  if (p.H <= (1 << 17)) per = std::max(1, std::min(per, std::max(8, (int)((64u << 20) / (32u * (unsigned)p.H)))));
  if (const char* e = getenv("SSA_HANK_PER")) per = std::max(1, std::min(cap, atoi(e)));
  const bool two = nterm_total > (size_t)per && p.lbuf_items >= 4;
  cudaError_t err;
  if (two && !p.lg_aux) {
    if ((err = cudaStreamCreateWithFlags(&p.lg_aux, cudaStreamNonBlocking))) return err;
    for (int i = 0; i < 2; ++i)
      if ((err = cudaEventCreateWithFlags(&p.lg_ev[i], cudaEventDisableTiming))) return err;
  }
  if (two) {
    if ((err = cudaEventRecord(p.lg_ev[0], s))) return err;
    if ((err = cudaStreamWaitEvent(p.lg_aux, p.lg_ev[0], 0))) return err;
  }
  size_t bi = 0;
  for (size_t t0 = 0; t0 < nterm_total; t0 += per, ++bi) {
    const int ni = (int)std::min<size_t>(nterm_total - t0, per);
    const int set = two ? (int)(bi & 1) : 0;
    cudaStream_t st = set ? p.lg_aux : s;
    double2* Ya = p.d_lbuf + (size_t)(2 * set) * per * p.H;
    double2* Yb = Ya + (size_t)per * p.H;
    ColFwdArgs cf{};
    cf.in[0] = ColFwdIn{U + t0 * p.L, (size_t)p.L, (int)p.L, Ya, vec16(U, p.L)};
    cf.in[1] = ColFwdIn{V + t0 * p.K, (size_t)p.K, (int)p.K, Yb, vec16(V, p.K)};
    const int logH = ilog2(p.H);
    const bool r16 = (logH == 16 || logH == 17) && !getenv("SSA_HANK_R8");
    const bool cw8 = getenv("SSA_COL16_CW16") == nullptr;  // 8 columns per CTA (128 threads, 4 CTAs/SM) measured 0.7 % faster than 16
    if (r16) {
      const int cw = cw8 ? 8 : 16;
      const dim3 grid((unsigned)(p.H >> 8) / cw, ni, 2);
      const dim3 blk(16 * cw);
      if (logH == 16 && !cw8) launch_pdl(lg_col16_fwd<16, 16>, grid, blk, col16_smem(16), st, cf, p.d_tw1, p.d_tw4);
      else if (logH == 16) launch_pdl(lg_col16_fwd<16, 8>, grid, blk, col16_smem(8), st, cf, p.d_tw1, p.d_tw4);
      else if (!cw8) launch_pdl(lg_col16_fwd<17, 16>, grid, blk, col16_smem(16), st, cf, p.d_tw1, p.d_tw4);
      else launch_pdl(lg_col16_fwd<17, 8>, grid, blk, col16_smem(8), st, cf, p.d_tw1, p.d_tw4);
    } else {
      col_fwd(p, cf, 2, ni, st);
    }
    RowArgs ra{2, Ya, Yb, nullptr, 0, nullptr, nullptr};
    rows(p, ra, ni, true, st);
    ColInvArgs ca{};
    ca.mode = 1;
    ca.out_stride = (size_t)p.N; ca.out = out + t0 * p.N;
    ca.sigma = sigma + t0; ca.N = (int)p.N; ca.L = (int)p.L; ca.K = (int)p.K; ca.rcpc = p.d_rcpc;
    if (r16) {
      const int cw = cw8 ? 8 : 16;
      const dim3 grid((unsigned)(p.H >> 8) / cw, ni);
      const dim3 blk(16 * cw);
      if (logH == 16 && !cw8) launch_pdl(lg_col16_hank<16, 16>, grid, blk, col16_smem(16), st, (const double2*)Yb, p.d_tw1, ca);
      else if (logH == 16) launch_pdl(lg_col16_hank<16, 8>, grid, blk, col16_smem(8), st, (const double2*)Yb, p.d_tw1, ca);
      else if (!cw8) launch_pdl(lg_col16_hank<17, 16>, grid, blk, col16_smem(16), st, (const double2*)Yb, p.d_tw1, ca);
      else launch_pdl(lg_col16_hank<17, 8>, grid, blk, col16_smem(8), st, (const double2*)Yb, p.d_tw1, ca);
    } else {
      col_inv(p, Yb, ca, ni, st);
    }
  }
  if (two) {
    if ((err = cudaEventRecord(p.lg_ev[1], p.lg_aux))) return err;
    if ((err = cudaStreamWaitEvent(s, p.lg_ev[1], 0))) return err;
  }
  return cudaGetLastError();
}

}  // namespace ssa
