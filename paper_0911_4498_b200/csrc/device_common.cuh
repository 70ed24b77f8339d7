// device_common.cuh -- reductions, TMA bulk-copy streaming and the FFT correlation /
// real-FFT pair steps shared by the kernels of libssa.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

#include "fft_smem.cuh"
#include "ssa_internal.h"

namespace ssa {

// ------------------------------------------------------------------ programmatic dependent launch
// Kernels of the host-driven sequences (long-series path) are launched with programmatic
// stream serialization: the next kernel is scheduled while the previous one drains, and
// waits at pdl_wait() (griddepcontrol.wait: the previous grid completed and its memory is
// visible) before touching anything the previous kernels wrote.  Every kernel launched
// with launch_pdl calls pdl_wait() first; without a programmatic dependency it returns
// at once.  (No early griddepcontrol.launch_dependents: dependents parked on the SMs
// during a grid's run slowed the long-series step down, 66.5 -> 70.4 ms at cfg3; the
// implicit trigger at completion still removes the launch gap.)
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Diagnostics (env SSA_TRACE, long-series path): thread 0 of CTA (0,0,0) of a traced kernel
// records (%globaltimer, kernel id) after its dependency wait, so start-to-start times per
// kernel id show where a graph's time goes (including conditional-node gaps).  One
// pointer per translation unit (no -rdc); null = off (one predicated load per CTA).
constexpr int kTraceMax = 1 << 18;
static __device__ unsigned long long* g_trace;
__device__ __forceinline__ void trace_point(int id) {
  if (threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0) {
    unsigned long long* tr = g_trace;
    if (tr != nullptr) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      const unsigned long long i = atomicAdd(tr, 1ull);
      if (i < (unsigned long long)kTraceMax) {
        tr[1 + 2 * i] = t;
        tr[2 + 2 * i] = (unsigned long long)id;
      }
    }
  }
}
// the same record from thread 0 of whichever CTA calls it (tail phases of a grid)
__device__ __forceinline__ void trace_point_any(int id) {
  if (threadIdx.x == 0) {
    unsigned long long* tr = g_trace;
    if (tr != nullptr) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      const unsigned long long i = atomicAdd(tr, 1ull);
      if (i < (unsigned long long)kTraceMax) {
        tr[1 + 2 * i] = t;
        tr[2 + 2 * i] = (unsigned long long)id;
      }
    }
  }
}
__device__ __forceinline__ void pdl_wait(int id) {
  pdl_wait();
  trace_point(id);
}
static inline cudaError_t trace_attach(unsigned long long* p) { return cudaMemcpyToSymbol(g_trace, &p, sizeof(p)); }

// PDL attribute switch (a graph build falls back to plain launches if the driver rejects
// programmatic edges inside conditional-node bodies)
inline bool& pdl_enabled() {
  static thread_local bool on = true;
  return on;
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// ------------------------------------------------------------------ reductions
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Sum of 8 values over the warp with 9 shuffles: lane l ends with the total of value
// (l >> 2) & 7 (fixed pairing order: deterministic).
__device__ __forceinline__ double warp_sum8(double* v, int lane) {
  const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const double send = b4 ? v[i] : v[i + 4];
    const double keep = b4 ? v[i + 4] : v[i];
    v[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const double send = b3 ? v[i] : v[i + 2];
    const double keep = b3 ? v[i + 2] : v[i];
    v[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  }
  {
    const double send = b2 ? v[0] : v[1];
    const double keep = b2 ? v[1] : v[0];
    v[0] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
  }
  v[0] += __shfl_xor_sync(0xffffffffu, v[0], 2);
  v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
  return v[0];
}

// Streaming (evict-first) fp64 load without `volatile`, so the compiler may hoist a group
// of them ahead of the arithmetic that consumes them.
__device__ __forceinline__ double ldg_stream(const double* p) {
  double x;
  asm("ld.global.cs.f64 %0, [%1];" : "=d"(x) : "l"(p));
  return x;
}

// fp64 tensor-core MMA (DMMA), D = A B + D with A 8x4 (row), B 4x8 (col), D 8x8: lane l
// holds A[l >> 2][l & 3], B[l & 3][l >> 2] and D[l >> 2][2 (l & 3) + {0, 1}] (the layout is
// checked on the device by tools/dmma_check.cu and by the Ritz parity tests).
__device__ __forceinline__ void dmma_m8n8k4(double& d0, double& d1, double a, double b) {
  // not volatile: the loads feeding later MMAs may be scheduled ahead of this one
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
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
// Digit-reversed position of frequency k for a compile-time size 2^LOGH (rev_index).
template <int LOGH>
__device__ __forceinline__ int rev_t(int k) {
  constexpr int N8 = LOGH / 3, LB = LOGH - 3 * N8;
  int pos = 0;
#pragma unroll
  for (int p = 0; p < N8; ++p) pos += ((k >> (3 * p)) & 7) << (LOGH - 3 * (p + 1));
  if constexpr (LB > 0) pos += (k >> (3 * N8)) & ((1 << LB) - 1);
  return pos;
}

// Forward real post-processing for the pair (p, H-p) from digit-reversed Z:
//   X_p = E + W^p O,  X_{H-p} = conj(E - W^p O),  E = (Z_p + conj Z_{H-p})/2,
//   O = -i (Z_p - conj Z_{H-p})/2,  W = exp(-2 pi i / M).  Returns W^p for inv_pair.
template <int LOGH, class TW>
__device__ __forceinline__ double2 real_pair(const double2* buf, const TW& tw, int p, double2& Xp, double2& Xq,
                                             int& pr, int& qr) {
  constexpr int H = 1 << LOGH;
  const int q = (H - p) & (H - 1);
  pr = fsw(rev_t<LOGH>(p));
  qr = fsw(rev_t<LOGH>(q));
  double2 Zp = buf[pr], Zq = buf[qr];
  double2 W = tw(p);
  double2 E = make_double2(0.5 * (Zp.x + Zq.x), 0.5 * (Zp.y - Zq.y));
  double2 D = make_double2(0.5 * (Zp.x - Zq.x), 0.5 * (Zp.y + Zq.y));
  double2 O = make_double2(D.y, -D.x);  // -i D
  double2 WO = cmul(W, O);
  Xp = cadd(E, WO);
  Xq = conjg(csub(E, WO));
  return W;
}

// Inverse pre-processing: from half-spectrum values Y_p, Y_{H-p} of a real sequence
// produce Z'_p = E + i O, Z'_{H-p} = conj(E) + i conj(O), E = (Y_p + conj Y_{H-p})/2,
// O = (Y_p - conj Y_{H-p}) conj(W^p) / 2, whose inverse FFT is y_2n + i y_2n+1.
// pr, qr: swizzled slots from real_pair.
__device__ __forceinline__ void inv_pair(double2* buf, double2 W, int pr, int qr, double2 Yp, double2 Yq) {
  double2 E = make_double2(0.5 * (Yp.x + Yq.x), 0.5 * (Yp.y - Yq.y));
  double2 D = make_double2(0.5 * (Yp.x - Yq.x), 0.5 * (Yp.y + Yq.y));
  double2 O = cmulc(D, W);
  buf[pr] = make_double2(E.x - O.y, E.y + O.x);
  if (qr != pr) buf[qr] = make_double2(E.x + O.y, O.x - E.y);
}

// Full correlation in one CTA (all threads): y_t = sum_s f_{t+s} x_s, t < n_out
// (the Hankel products of Alg. 2 / Alg. 3, in correlation form):
// packed forward FFT of x, pair step Z -> Z' whose inverse is the packed correlation
// y = irfft(F^ conj(X^)), inverse FFT.
template <int LOGH, class TW, class LoadX, class StoreY>
__device__ __forceinline__ void correlate_t(double2* buf, const TW& T, const double2* __restrict__ spec, int n_in,
                                            int n_out, LoadX loadx, StoreY storey) {
  constexpr int H = 1 << LOGH;
  const int tid = threadIdx.x, nthr = blockDim.x;
  // pull this thread's spectrum entries of the pair step towards L2 now (they are used
  // after the forward transform; from HBM their latency would stall that step)
  for (int p = tid; p <= (H >> 1); p += nthr) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(spec + p));
    asm volatile("prefetch.global.L2 [%0];" ::"l"(spec + (H - p)));
  }
  for (int n = tid; n < H; n += nthr) {
    int i0 = 2 * n;
    double a = (i0 < n_in) ? loadx(i0) : 0.0;
    double b = (i0 + 1 < n_in) ? loadx(i0 + 1) : 0.0;
    buf[fsw(n)] = make_double2(a, b);
  }
  __syncthreads();
  fft_run_t<LOGH, false>(buf, T, tid, nthr, CtaSync());
  for (int p = tid; p <= (H >> 1); p += nthr) {
    const double2 Fp = __ldg(spec + p), Fq = __ldg(spec + (H - p));
    double2 Xp, Xq;
    int pr, qr;
    const double2 W = real_pair<LOGH>(buf, T, p, Xp, Xq, pr, qr);
    inv_pair(buf, W, pr, qr, cmulc(Fp, Xp), cmulc(Fq, Xq));
  }
  __syncthreads();
  fft_run_t<LOGH, true>(buf, T, tid, nthr, CtaSync());
  const double invH = 1.0 / (double)H;
  for (int t = tid; t < n_out; t += nthr) {
    double2 z = buf[fsw(t >> 1)];
    storey(t, ((t & 1) ? z.y : z.x) * invH);
  }
}

// Runtime-size entry (H = 2^logH, 2 <= H <= 8192): one switch, then everything compiles
// to constant shifts and offsets.
template <class TW, class LoadX, class StoreY>
__device__ __forceinline__ void correlate_cta(double2* buf, const FftShape& sh, const TW& T,
                                              const double2* __restrict__ spec, int n_in, int n_out, LoadX loadx,
                                              StoreY storey) {
  switch (sh.logH) {
#define SSA_CORR(L) \
  case L: correlate_t<L>(buf, T, spec, n_in, n_out, loadx, storey); break;
    SSA_CORR(1) SSA_CORR(2) SSA_CORR(3) SSA_CORR(4) SSA_CORR(5) SSA_CORR(6) SSA_CORR(7)
    SSA_CORR(8) SSA_CORR(9) SSA_CORR(10) SSA_CORR(11) SSA_CORR(12)
    default: correlate_t<13>(buf, T, spec, n_in, n_out, loadx, storey); break;
#undef SSA_CORR
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
// Same with an L2 cache-eviction policy (createpolicy.*: evict_last keeps a row that is
// read again soon, evict_first drops one read for the last time).
__device__ __forceinline__ void tma_load_1d_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                                 uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

// Per-warp ring of kStages chunks; one lane issues cp.async.bulk, all lanes consume.
struct WarpRing {
  double* buf;    // kStages * slab doubles
  uint64_t* bar;  // kStages barriers
  uint32_t cnt;   // chunks consumed so far (== issued at the end of each stream)
};

template <int NST = kStages>
__device__ __forceinline__ void ring_init(WarpRing& rg, double* buf, uint64_t* bar) {
  rg.buf = buf;
  rg.bar = bar;
  rg.cnt = 0;
  if ((threadIdx.x & 31) == 0)
    for (int s = 0; s < NST; ++s) mbar_init(bar + s, 1);
}

// Streams rows (q-th job = row q, or nb-1-q if reverse) of this warp's column slab
// [w*slab, (w+1)*slab) of a row-major basis (row stride ld doubles) through the ring;
// calls f(row, chunk) for each in order.  All lanes of the warp must call it.
template <int NST = kStages, class F>
__device__ __forceinline__ void stream_rows(const double* base_w, int ld, int nb, bool reverse, int slab, WarpRing& rg,
                                            F f) {
  stream_rows<NST>(base_w, ld, nb, reverse, slab, rg, 0ull, f);
}
// Same with an L2 eviction policy for every load (0: none).
template <int NST = kStages, class F>
__device__ __forceinline__ void stream_rows(const double* base_w, int ld, int nb, bool reverse, int slab, WarpRing& rg,
                                            uint64_t policy, F f) {
  constexpr int kStages = NST;  // ring depth of this stream (the ring must have NST stages)
  const int lane = threadIdx.x & 31;
  const uint32_t bytes = (uint32_t)slab * 8u;
  const uint32_t c0 = rg.cnt;
  if (lane == 0) {
    int pre = nb < kStages ? nb : kStages;
    for (int q = 0; q < pre; ++q) {
      int st = (int)((c0 + q) % kStages);
      int row = reverse ? nb - 1 - q : q;
      mbar_expect_tx(rg.bar + st, bytes);
      if (policy) tma_load_1d_hint(rg.buf + (size_t)st * slab, base_w + (size_t)row * ld, bytes, rg.bar + st, policy);
      else tma_load_1d(rg.buf + (size_t)st * slab, base_w + (size_t)row * ld, bytes, rg.bar + st);
    }
  }
  // refills are issued by lane 0 under a predicate (no divergent branch per row)
  const uint64_t pol = policy ? policy : policy_evict_normal();
  for (int q = 0; q < nb; ++q) {
    const uint32_t c = c0 + q;
    const int st = (int)(c % kStages);
    mbar_wait(rg.bar + st, (c / kStages) & 1u);
    f(reverse ? nb - 1 - q : q, rg.buf + (size_t)st * slab);
    __syncwarp();
    const int qn = q + kStages;
    const int row = reverse ? nb - 1 - qn : qn;
    const uint32_t issue = (lane == 0 && qn < nb) ? 1u : 0u;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %0, 0;\n"
        "@p mbarrier.arrive.expect_tx.shared::cta.b64 _, [%1], %2;\n"
        "@p cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%3], [%4], %2, [%1], %5;\n"
        "}\n" ::"r"(issue),
        "r"(smem_u32(rg.bar + st)), "r"(bytes), "r"(smem_u32(rg.buf + (size_t)st * slab)),
        "l"(base_w + (size_t)(issue ? row : 0) * ld), "l"(pol)
        : "memory");
  }
  rg.cnt = c0 + nb;
}

__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~(size_t)15; }

// 1/c for an integer count c >= 1 (the antidiagonal counts of Alg. 4, R2) to
// within an ulp: float reciprocal, two Newton steps in fp64 -- no fp64 division (a long
// instruction sequence with a slow path) in the Hankelization epilogues.
__device__ __forceinline__ double rcp_count_f64(int c) {
  const double cd = (double)c;
  double r = (double)__frcp_rn((float)c);
  r = fma(r, fma(-cd, r, 1.0), r);
  r = fma(r, fma(-cd, r, 1.0), r);
  return r;
}

// Copy the two-level twiddle table of size M (global, lo then hi) into shared memory
// (all threads; caller synchronizes).
__device__ __forceinline__ TwSmem load_tw2(const double2* __restrict__ g, double2* sm, int M) {
  const int n = tw2_entries(M);
  for (int i = threadIdx.x; i < n; i += blockDim.x) sm[i] = __ldg(g + i);
  return TwSmem{sm, sm + 64, sm + tw2_base_entries(M)};
}

}  // namespace ssa
