// ssa_api.cu -- the extern "C" boundary of libssa.so (include/ssa.h).
// Host-side validation, workspace sizing, twiddle tables and kernel enqueueing only;
// every arithmetic step of the method runs in the kernels (ssa_fft_kernels.cu,
// ssa_lanczos.cu, ssa_svd.cu).
#include <cuda_runtime.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <vector>

#include "fft_smem.cuh"
#include "ssa_internal.h"

using ssa::Plan;

static thread_local char g_err[512] = "";

static ssa_status fail(ssa_status s, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return s;
}

static ssa_status cuda_fail(cudaError_t e, const char* what) {
  cudaGetLastError();
  return fail(SSA_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

#define CK(call, what)                                 \
  do {                                                 \
    cudaError_t e_ = (call);                           \
    if (e_ != cudaSuccess) return cuda_fail(e_, what); \
  } while (0)

struct ssa_plan_s {
  Plan p;
};

static int round_up(int x, int m) { return (x + m - 1) / m * m; }

namespace ssa {
cudaError_t raise_smem_limit(const void* func, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> limit;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  size_t& cur = limit[std::make_pair(dev, func)];
  if (bytes <= cur) return cudaSuccess;
  e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) cur = bytes;
  return e;
}
}  // namespace ssa
// Golub-Kahan QR on an m x m bidiagonal takes ~2 sweeps per value, i.e. about m^2
// rotations per side; 2 m^2 + 8 m + 1024 leaves room.  Overflow -> SSA_ERR_INTERNAL.
static int rot_cap(int m_max) { return 2 * m_max * m_max + 8 * m_max + 1024; }

extern "C" ssa_status ssa_options_default(ssa_options* opt) {
  if (!opt) return fail(SSA_ERR_INVALID_ARGUMENT, "opt is NULL");
  memset(opt, 0, sizeof(*opt));
  opt->tol = 1e-12;
  opt->max_steps = 0;
  opt->check_every = 4;
  opt->seed = 42;
  opt->reorth = 3;
  opt->reorth_eta = 1.8189894035458565e-12;  // eps^(3/4)
  return SSA_OK;
}

// exp(-2 pi i t / M) for t in [0, H), in extended precision then rounded once.
static std::vector<double2> make_twiddles(int64_t M) {
  int64_t H = M / 2;
  std::vector<double2> tw((size_t)H);
  for (int64_t t = 0; t < H; ++t) {
    long double ang = 2.0L * 3.14159265358979323846264338327950288L * (long double)t / (long double)M;
    tw[(size_t)t].x = (double)cosl(ang);
    tw[(size_t)t].y = (double)(-sinl(ang));
  }
  return tw;
}

// Two-level table for size M: lo[j] = exp(-2 pi i j / M), j < 64; hi[j] = exp(-2 pi i 64 j / M).
static std::vector<double2> make_twiddles2(int64_t M) {
  // two-level table lo[j] = W_M^j (j < 64), hi[j] = W_M^{64 j}, then the per-pass tables
  // of the M/2-point FFT (fft_smem.cuh TwSmem): pass with block size S = 2^logS gets
  // W_S^a (a < min(Q, 64)) and, when Q = S/8 > 64, W_S^{64 b} (b < Q/64)
  const long double pi2 = 2.0L * 3.14159265358979323846264338327950288L;
  auto w = [&](long double num, long double den) {
    const long double ang = pi2 * num / den;
    return make_double2((double)cosl(ang), (double)(-sinl(ang)));
  };
  const int nhi = (int)std::max<int64_t>(1, M / 64);
  std::vector<double2> tw;
  for (int j = 0; j < 64 + nhi; ++j) tw.push_back(w((j < 64) ? (long double)j : 64.0L * (long double)(j - 64), (long double)M));
  int logH = 0;
  while ((1LL << logH) < M / 2) ++logH;
  for (int logS = logH; logS >= 3; logS -= 3) {
    const int64_t Q = 1LL << (logS - 3), S = 1LL << logS;
    for (int64_t a = 0; a < std::min<int64_t>(Q, 64); ++a) tw.push_back(w((long double)a, (long double)S));
    if (Q > 64)
      for (int64_t b = 0; b < Q / 64; ++b) tw.push_back(w(64.0L * (long double)b, (long double)S));
  }
  if (tw.size() != (size_t)ssa::tw2_entries((int)M)) tw.clear();  // layout mismatch: caller fails
  return tw;
}

static void free_plan(Plan& p) {
  void* ptrs[] = {p.d_tw, p.d_twl, p.d_spec, p.d_U, p.d_V, p.d_ab, p.d_state, p.d_tgk, p.d_rot, p.d_vecs, p.d_coef,
                  p.d_info, p.d_counters, p.d_hscratch, p.d_prof, p.d_tgkw, p.d_tw1, p.d_tw2, p.d_tw4, p.d_twp, p.d_rcpc, p.d_lbuf,
                  p.d_lgsc, p.d_lgpart, p.d_lgh, p.d_lgr, p.d_series, p.d_sigma, p.d_Uout, p.d_Vout,
                  p.d_recon, p.d_elem, p.d_bs, p.d_lgom, p.d_ucur, p.d_vcur};
  if (p.lg_exec) cudaGraphExecDestroy(p.lg_exec);
  if (p.lg_graph) cudaGraphDestroy(p.lg_graph);
  for (void* q : ptrs)
    if (q) cudaFree(q);
  for (int i = 0; i < 2 * Plan::kPhases; ++i)
    if (p.ev[i]) cudaEventDestroy(p.ev[i]);
  for (int i = 0; i < 3; ++i)
    if (p.sub[i]) ssa_plan_destroy(reinterpret_cast<ssa_plan_t>(p.sub[i]));
  for (int i = 0; i < 4; ++i)
    if (p.hs[i]) cudaStreamDestroy(p.hs[i]);
  if (p.lg_aux) cudaStreamDestroy(p.lg_aux);
  for (int i = 0; i < 2; ++i)
    if (p.lg_ev[i]) cudaEventDestroy(p.lg_ev[i]);
  for (int i = 0; i < 2 * Plan::kMaxSlices + 2; ++i)
    if (p.hev[i]) cudaEventDestroy(p.hev[i]);
}

static ssa_status alloc(void** ptr, size_t bytes, const char* what) {
  if (bytes == 0) bytes = 16;
  cudaError_t e = cudaMalloc(ptr, bytes);
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    return fail(SSA_ERR_OUT_OF_MEMORY, "cudaMalloc(%zu bytes) for %s failed", bytes, what);
  }
  if (e != cudaSuccess) return cuda_fail(e, what);
  return SSA_OK;
}

// Bytes of per-series decompose storage (bases, spectrum, B, Ritz coefficients).
static size_t per_series_bytes(const Plan& p) {
  size_t s = (size_t)(p.m_max + 1) * (p.ldL + p.ldK) * 8;
  s += (size_t)(p.H + 1) * 16;
  s += (size_t)2 * (p.m_max + 3) * 8 + 8 * 4;
  s += (size_t)2 * (p.m_max + 2) * p.k * 8;
  return s;
}

// doubles per TGK-SVD CTA slot: Z (n k), LU factors (5 n k), pivots (n k ints)
static size_t tgkw_stride(const Plan& p) { return (size_t)(2 * p.m_max + 1) * p.k * 7; }

static ssa_status create_decompose_workspace(Plan& p, const cudaDeviceProp& prop) {
  ssa_status st;
  cudaError_t e;
  const int k = p.k;
  if (k > ssa::kMaxK) return fail(SSA_ERR_UNSUPPORTED, "k = %d > %d not supported by the batched decompose", k, ssa::kMaxK);
  p.smem_lanczos = ssa::lanczos_smem_bytes((int)p.H, p.ldL, p.ldK, p.m_max, k, p.opt.restart_dim > 0);
  p.smem_ritz = ssa::ritz_smem_bytes(p.ldL, p.ldK, k, p.m_max);
  if (p.smem_lanczos > (size_t)prop.sharedMemPerBlockOptin)
    return fail(SSA_ERR_UNSUPPORTED, "decompose needs %zu B shared memory > %zu", p.smem_lanczos,
                (size_t)prop.sharedMemPerBlockOptin);
  if ((e = ssa::lanczos_set_attributes(p.smem_lanczos)) != cudaSuccess) return cuda_fail(e, "lanczos attributes");
  if ((e = ssa::svd_ritz_set_attributes(p.m_max, p.smem_ritz)) != cudaSuccess) return cuda_fail(e, "svd/ritz attributes");
  int per_sm = (int)std::max<size_t>(1, std::min<size_t>(2, (size_t)prop.sharedMemPerMultiprocessor / (p.smem_lanczos + 1024)));
  // chunk: as many series as fit in ~60% of free memory (env SSA_MAX_CHUNK caps it)
  size_t fr = 0, tot = 0;
  CK(cudaMemGetInfo(&fr, &tot), "cudaMemGetInfo");
  size_t per = per_series_bytes(p);
  int64_t fit = (int64_t)((double)fr * 0.6 / (double)per);
  int64_t chunk = std::min<int64_t>(p.batch, std::max<int64_t>(1, fit));
  if (const char* env = getenv("SSA_MAX_CHUNK")) chunk = std::max<int64_t>(1, std::min<int64_t>(chunk, atoll(env)));
  p.chunk = (int)chunk;
  p.lanczos_slots = (int)std::min<int64_t>(chunk, (int64_t)p.sms * per_sm);
  if (const char* env = getenv("SSA_LANCZOS_SLOTS")) p.lanczos_slots = std::max(1, std::min(p.lanczos_slots, atoi(env)));
  p.svd_slots = (int)std::min<int64_t>(chunk, (int64_t)p.sms * ssa::kSvdWarpsPerCta);
  p.ritz_slots = (int)std::min<int64_t>(chunk, (int64_t)p.sms * 2);
  p.rot_cap = rot_cap(p.m_max);
  size_t C = (size_t)chunk;
  if ((st = alloc((void**)&p.d_U, C * (p.m_max + 1) * p.ldL * 8, "U bases")) != SSA_OK) return st;
  if ((st = alloc((void**)&p.d_V, C * (p.m_max + 1) * p.ldK * 8, "V bases")) != SSA_OK) return st;
  if ((st = alloc((void**)&p.d_spec, C * (p.H + 1) * 16, "spectra")) != SSA_OK) return st;
  if ((st = alloc((void**)&p.d_ab, C * 2 * (p.m_max + 3) * 8, "bidiagonals")) != SSA_OK) return st;
  if ((st = alloc((void**)&p.d_state, C * ssa::kStateInts * sizeof(int), "series state")) != SSA_OK) return st;
  if ((st = alloc((void**)&p.d_coef, C * 2 * (p.m_max + 2) * k * 8, "Ritz coefficients")) != SSA_OK) return st;
  if ((st = alloc((void**)&p.d_tgk, (size_t)p.lanczos_slots * 2 * k * (2 * p.m_max + 2) * 8, "TGK scratch")) != SSA_OK)
    return st;
  if (p.opt.reserved & 2) {  // bidiagonal SVD by QR with rotation records
    if ((st = alloc((void**)&p.d_rot, (size_t)p.svd_slots * 6 * p.rot_cap * 8, "rotation records")) != SSA_OK)
      return st;
    if ((st = alloc((void**)&p.d_vecs, (size_t)p.svd_slots * 2 * k * (p.m_max + 2) * 8, "P/Q columns")) != SSA_OK)
      return st;
  } else {  // TGK multisection + inverse iteration
    p.tgk_slots = (int)std::min<int64_t>(chunk, (int64_t)p.sms * 8);
    if ((st = alloc((void**)&p.d_tgkw, (size_t)p.tgk_slots * tgkw_stride(p) * 8, "TGK vectors")) != SSA_OK) return st;
  }
  if ((st = alloc((void**)&p.d_info, (size_t)p.batch * sizeof(ssa_series_info), "info")) != SSA_OK) return st;
  if ((st = alloc((void**)&p.d_counters, 16 * sizeof(int), "counters")) != SSA_OK) return st;
  if (p.opt.reserved & 1) {
    if ((st = alloc((void**)&p.d_prof, 8 * sizeof(unsigned long long), "profile counters")) != SSA_OK) return st;
    CK(cudaMemset(p.d_prof, 0, 8 * sizeof(unsigned long long)), "memset");
  }
  return SSA_OK;
}

// Long-series workspace: one series at a time, the whole GPU on it.
static ssa_status create_large_workspace(Plan& p) {
  ssa_status st;
  cudaError_t e;
  const int k = p.k;
  if (k > ssa::kMaxK) return fail(SSA_ERR_UNSUPPORTED, "k = %d > %d not supported", k, ssa::kMaxK);
  if ((e = ssa::large_lanczos_set_attributes(p.m_max)) != cudaSuccess) return cuda_fail(e, "large lanczos attributes");
  if ((e = ssa::svd_ritz_set_attributes(p.m_max, 48 * 1024)) != cudaSuccess) return cuda_fail(e, "svd attributes");
  p.chunk = 1;
  p.tgk_slots = 1;
  p.rot_cap = rot_cap(p.m_max);
  if ((st = alloc((void**)&p.d_U, (size_t)(p.m_max + 1) * p.ldL * 8, "U basis")) != SSA_OK) return st;
  if ((st = alloc((void**)&p.d_V, (size_t)(p.m_max + 1) * p.ldK * 8, "V basis")) != SSA_OK) return st;
  if ((st = alloc((void**)&p.d_spec, (size_t)(p.H + 1) * 16, "spectrum")) != SSA_OK) return st;
  if ((st = alloc((void**)&p.d_ab, (size_t)2 * (p.m_max + 3) * 8, "bidiagonal")) != SSA_OK) return st;
  if ((st = alloc((void**)&p.d_state, ssa::kStateInts * sizeof(int), "series state")) != SSA_OK) return st;
  if ((st = alloc((void**)&p.d_coef, (size_t)2 * (p.m_max + 2) * k * 8, "Ritz coefficients")) != SSA_OK) return st;
  if ((st = alloc((void**)&p.d_tgk, (size_t)2 * k * (2 * p.m_max + 2) * 8, "TGK scratch")) != SSA_OK) return st;
  if ((st = alloc((void**)&p.d_tgkw, tgkw_stride(p) * 8, "TGK vectors")) != SSA_OK) return st;
  if ((st = alloc((void**)&p.d_info, (size_t)p.batch * sizeof(ssa_series_info), "info")) != SSA_OK) return st;
  if ((st = alloc((void**)&p.d_counters, 16 * sizeof(int), "counters")) != SSA_OK) return st;
  const size_t nch = (size_t)(std::max(p.ldL, p.ldK) + 511) / 512;  // reorth chunks (kRoChunk)
  const size_t gU = (size_t)(p.L + 255) / 256;
  // dots partials [row][chunk], then 1024 correlation partials, 1024 start-vector partials
  // and the dots group sums [row][kLgMaxGroups] (ssa_large_lanczos.cu)
  const size_t npart = std::max(nch * (p.m_max + 2), gU * k * 2) + 2048 + (size_t)(p.m_max + 2) * 64 + 64;
  if (nch > 64 * 32) return fail(SSA_ERR_UNSUPPORTED, "long-series reorthogonalization supports ld <= %d", 64 * 32 * 512);
  if ((st = alloc((void**)&p.d_lgsc, 2048, "scalars")) != SSA_OK) return st;
  if ((st = alloc((void**)&p.d_lgpart, npart * 8, "partials")) != SSA_OK) return st;
  if ((st = alloc((void**)&p.d_lgh, (size_t)(p.m_max + 2 + 64) * 8, "reorth coefficients")) != SSA_OK) return st;
  if ((st = alloc((void**)&p.d_lgr, (size_t)std::max(p.ldL, p.ldK) * 8, "work vector")) != SSA_OK) return st;
  if ((st = alloc((void**)&p.d_lgom, (size_t)2 * (p.m_max + 4) * 8, "PRO estimates")) != SSA_OK) return st;
  if ((st = alloc((void**)&p.d_ucur, (size_t)p.ldL * 8, "current u")) != SSA_OK) return st;
  if ((st = alloc((void**)&p.d_vcur, (size_t)p.ldK * 8, "current v")) != SSA_OK) return st;
  return SSA_OK;
}

extern "C" ssa_status ssa_plan_create(int64_t N, int64_t L, int32_t k, int64_t batch, const ssa_options* opt,
                                      int device, ssa_plan_t* out) {
  if (!out) return fail(SSA_ERR_INVALID_ARGUMENT, "out is NULL");
  *out = nullptr;
  if (N < 3) return fail(SSA_ERR_INVALID_ARGUMENT, "N = %lld < 3 (PAPER.md:70 requires N > 2)", (long long)N);
  if (L < 2 || L > N - 1)
    return fail(SSA_ERR_INVALID_ARGUMENT, "L = %lld outside [2, N-1] (PAPER.md:71: 1 < L < N)", (long long)L);
  int64_t K = N - L + 1;
  if (k < 0 || k > std::min(L, K))
    return fail(SSA_ERR_INVALID_ARGUMENT, "k = %d outside [1, min(L,K) = %lld]", k, (long long)std::min(L, K));
  if (batch < 1) return fail(SSA_ERR_INVALID_ARGUMENT, "batch = %lld < 1", (long long)batch);
  if (batch > 0x7fffffff) return fail(SSA_ERR_INVALID_ARGUMENT, "batch = %lld too large", (long long)batch);
  ssa_options o;
  ssa_options_default(&o);
  if (opt) o = *opt;
  if (!(o.tol > 0.0) || o.reorth < 1 || o.reorth > 3 || o.check_every < 0 || o.max_steps < 0 || o.series_base < 0 ||
      (o.reorth == 3 && !(o.reorth_eta > 0.0 && o.reorth_eta <= 1e-6)) || o.restart_dim < 0 || o.restart_keep < 0)
    return fail(SSA_ERR_INVALID_ARGUMENT,
                "bad options (tol > 0, reorth in {1,2,3}, reorth_eta in (0, 1e-6] for reorth 3, check_every >= 0, "
                "max_steps >= 0, series_base >= 0, restart_dim >= 0, restart_keep >= 0)");

  if (o.restart_dim > 0) {
    // thick restart (R23): validated here, before any allocation
    const int64_t d = o.restart_dim, mn = std::min(L, K);
    if (k < 1 || d < (int64_t)k + 2 || d > mn - 1)
      return fail(SSA_ERR_INVALID_ARGUMENT, "restart_dim = %lld must lie in [k + 2, min(L, K) - 1] = [%d, %lld]",
                  (long long)d, k + 2, (long long)(mn - 1));
    if (o.restart_keep == 0) o.restart_keep = (int32_t)std::max<int64_t>(k, d / 2);
    if (o.restart_keep < k || o.restart_keep > d - 2 || o.restart_keep > 64)
      return fail(SSA_ERR_INVALID_ARGUMENT, "restart_keep = %d must lie in [k, min(restart_dim - 2, 64)] = [%d, %lld]",
                  o.restart_keep, k, (long long)std::min<int64_t>(d - 2, 64));
  }

  int64_t M = 1;
  while (M < N) M <<= 1;
  int64_t H = M / 2;
  if (H > ssa::kMaxLargeH)
    return fail(SSA_ERR_UNSUPPORTED, "N = %lld needs M = %lld > %d", (long long)N, (long long)M, 2 * ssa::kMaxLargeH);

  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
  if (prop.major < 10)
    return fail(SSA_ERR_UNSUPPORTED, "device %d is sm_%d%d; libssa is built for sm_100a only", device, prop.major,
                prop.minor);

  ssa_plan_s* ps = new ssa_plan_s();
  Plan& p = ps->p;
  p.device = device;
  p.N = N; p.L = L; p.K = K; p.M = M; p.H = H; p.k = k; p.batch = batch; p.opt = o;
  p.series_base = o.series_base;
  p.sms = prop.multiProcessorCount;
  int64_t mn = std::min(L, K);
  int64_t mm = o.max_steps > 0 ? o.max_steps : std::max<int64_t>(256, 8 * (int64_t)k);
  p.m_max = (int32_t)std::max<int64_t>(k, std::min(mm, mn));
  if (o.restart_dim > 0) {
    p.m_max = o.restart_dim;  // thick restart: the bases hold d + 1 vectors
    p.m_cap = o.max_steps > 0 ? o.max_steps : std::max(512, 16 * k);
  }
  p.ldL = round_up((int)L, 16);
  p.ldK = round_up((int)K, 16);

  ssa_status st = SSA_OK;
  for (int i = 0; i < 2 * Plan::kPhases; ++i) {
    e = cudaEventCreate(&p.ev[i]);
    if (e != cudaSuccess) { st = cuda_fail(e, "cudaEventCreate"); goto bad; }
  }
  {
    std::vector<double2> tw = make_twiddles(M), twl = make_twiddles2(M);
    if (twl.empty()) { st = fail(SSA_ERR_INTERNAL, "twiddle table layout mismatch"); goto bad; }
    if ((st = alloc((void**)&p.d_tw, tw.size() * sizeof(double2), "twiddles")) != SSA_OK) goto bad;
    if ((st = alloc((void**)&p.d_twl, twl.size() * sizeof(double2), "twiddles")) != SSA_OK) goto bad;
    e = cudaMemcpy(p.d_tw, tw.data(), tw.size() * sizeof(double2), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(p.d_twl, twl.data(), twl.size() * sizeof(double2), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) { st = cuda_fail(e, "twiddle upload"); goto bad; }
    const char* which = "";
    e = (H <= ssa::kMaxSmemH) ? ssa::fft_set_attributes((int)H, &which) : cudaSuccess;
    if (e != cudaSuccess) {
      st = fail(SSA_ERR_CUDA, "cudaFuncSetAttribute(%s, %zu B smem): %s", which, ssa::fft_bytes((int)H),
                cudaGetErrorString(e));
      cudaGetLastError();
      goto bad;
    }
  }
  // long path: M > 16384, forced (reserved & 4, tests), or a decompose whose batched
  // kernel would not fit one CTA's shared memory (e.g. H = 8192 with k > 0)
  if (H > ssa::kMaxSmemH || ((o.reserved & 4) && H >= 64) ||
      (k > 0 && H >= 64 &&
       ssa::lanczos_smem_bytes((int)H, p.ldL, p.ldK, p.m_max, k, o.restart_dim > 0) >
           (size_t)prop.sharedMemPerBlockOptin)) {
    p.large = true;
    if (o.restart_dim > 0) {
      st = fail(SSA_ERR_UNSUPPORTED, "thick restart (restart_dim > 0) runs on the batched path only (M <= 16384)");
      goto bad;
    }
    int N1, N2;
    ssa::large_geom(p, &N1, &N2);
    std::vector<double2> t1 = make_twiddles2(2 * (int64_t)N1), t2 = make_twiddles2(2 * (int64_t)N2);
    if (t1.empty() || t2.empty()) { st = fail(SSA_ERR_INTERNAL, "twiddle table layout mismatch"); goto bad; }
    if ((st = alloc((void**)&p.d_tw1, t1.size() * 16, "twiddles N1")) != SSA_OK) goto bad;
    if ((st = alloc((void**)&p.d_tw2, t2.size() * 16, "twiddles N2")) != SSA_OK) goto bad;
    e = cudaMemcpy(p.d_tw1, t1.data(), t1.size() * 16, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(p.d_tw2, t2.data(), t2.size() * 16, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
      // four-step twiddles as a two-level table W_H^e = TL[e mod 2^a] TH[e >> a]
      // (a = ceil(log2 H / 2)) and the pair-step row factors W_M^A, A <= N1/2
      // (extended precision on the host, like every other table)
      const long double pi2 = 2.0L * 3.14159265358979323846264338327950288L;
      int logH = 0;
      while ((1LL << logH) < H) ++logH;
      const int64_t ntl = 1LL << ((logH + 1) / 2), nth = H / ntl;
      std::vector<double2> t4, tp;
      for (int64_t j = 0; j < ntl + nth; ++j) {
        const long double e = (j < ntl) ? (long double)j : (long double)((j - ntl) * ntl);
        const long double ang = pi2 * e / (long double)H;
        t4.push_back(make_double2((double)cosl(ang), (double)(-sinl(ang))));
      }
      if ((int64_t)t4.size() != ssa::large_twh_entries(logH)) t4.clear();
      for (int64_t A = 0; A <= N1 / 2; ++A) {
        const long double ang = pi2 * (long double)A / (long double)M;
        tp.push_back(make_double2((double)cosl(ang), (double)(-sinl(ang))));
      }
      if (t4.empty()) { st = fail(SSA_ERR_INTERNAL, "four-step table layout mismatch"); goto bad; }
      if ((st = alloc((void**)&p.d_tw4, t4.size() * 16, "four-step twiddles")) != SSA_OK) goto bad;
      if ((st = alloc((void**)&p.d_twp, tp.size() * 16, "pair twiddles")) != SSA_OK) goto bad;
      e = cudaMemcpy(p.d_tw4, t4.data(), t4.size() * 16, cudaMemcpyHostToDevice);
      if (e == cudaSuccess) e = cudaMemcpy(p.d_twp, tp.data(), tp.size() * 16, cudaMemcpyHostToDevice);
    }
    if (e == cudaSuccess) e = ssa::large_set_attributes(N1, N2);
    if (e != cudaSuccess) { st = cuda_fail(e, "large FFT setup"); goto bad; }
    {
      // 1/c_t of the Hankelization weights: every count is in [1, min(L, K)]
      const int64_t mn = std::min<int64_t>(L, N - L + 1);
      std::vector<double> rc((size_t)mn);
      for (int64_t c = 1; c <= mn; ++c) rc[(size_t)c - 1] = 1.0 / (double)c;
      if ((st = alloc((void**)&p.d_rcpc, rc.size() * 8, "hankelization weights")) != SSA_OK) goto bad;
      if ((e = cudaMemcpy(p.d_rcpc, rc.data(), rc.size() * 8, cudaMemcpyHostToDevice))) {
        st = cuda_fail(e, "large FFT setup");
        goto bad;
      }
    }
    // work buffers: ~512 MB, at least 2 items (hankelization needs a pair)
    p.lbuf_items = (int)std::max<int64_t>(2, std::min<int64_t>(256, ((int64_t)512 << 20) / (H * 16)));
    if ((st = alloc((void**)&p.d_lbuf, (size_t)p.lbuf_items * H * 16, "large FFT buffers")) != SSA_OK) goto bad;
  } else if (H > ssa::kMaxHankelSmemH) {
    p.hank_slots = p.sms;
    if ((st = alloc((void**)&p.d_hscratch, (size_t)p.hank_slots * (H + 1) * 16, "hankelization scratch")) != SSA_OK)
      goto bad;
  }
  if (k > 0 && (st = (p.large ? create_large_workspace(p) : create_decompose_workspace(p, prop))) != SSA_OK) goto bad;
  *out = ps;
  return SSA_OK;
bad:
  free_plan(p);
  delete ps;
  return st;
}

extern "C" void ssa_plan_destroy(ssa_plan_t plan) {
  if (!plan) return;
  cudaSetDevice(plan->p.device);
  free_plan(plan->p);
  delete plan;
}

extern "C" int64_t ssa_plan_fft_size(ssa_plan_t plan) { return plan ? plan->p.M : -1; }
extern "C" int32_t ssa_plan_max_steps(ssa_plan_t plan) { return plan ? plan->p.m_max : -1; }
extern "C" int64_t ssa_plan_launch_count(ssa_plan_t plan) { return plan ? plan->p.launches : -1; }

static cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// events around one phase: ph in [0, kPhases)
struct PhaseTimer {
  Plan& p;
  int ph;
  cudaStream_t s;
  PhaseTimer(Plan& p_, int ph_, cudaStream_t s_) : p(p_), ph(ph_), s(s_) { cudaEventRecord(p.ev[2 * ph], s); }
  ~PhaseTimer() {
    cudaEventRecord(p.ev[2 * ph + 1], s);
    p.ev_used[ph] = true;
  }
};

extern "C" ssa_status ssa_spectrum(ssa_plan_t plan, const double* d_series, double* d_spec, void* stream) {
  if (!plan || !d_series || !d_spec) return fail(SSA_ERR_INVALID_ARGUMENT, "NULL argument");
  if (((uintptr_t)d_spec) & 15) return fail(SSA_ERR_INVALID_ARGUMENT, "d_spec must be 16-byte aligned");
  Plan& p = plan->p;
  CK(cudaSetDevice(p.device), "cudaSetDevice");
  PhaseTimer pt(p, 0, S(stream));
  if (p.large) {
    CK(ssa::large_spectrum(p, d_series, reinterpret_cast<double2*>(d_spec), (int)p.batch, S(stream)),
       "large spectrum");
  } else {
    CK(ssa::launch_spectrum(p, d_series, reinterpret_cast<double2*>(d_spec), (int)p.batch, S(stream)),
       "spectrum launch");
  }
  p.launches += 1;
  return SSA_OK;
}

extern "C" ssa_status ssa_matvec(ssa_plan_t plan, const double* d_spec, const double* d_x, double* d_y,
                                 int transpose, void* stream) {
  if (!plan || !d_spec || !d_x || !d_y) return fail(SSA_ERR_INVALID_ARGUMENT, "NULL argument");
  if (((uintptr_t)d_spec) & 15) return fail(SSA_ERR_INVALID_ARGUMENT, "d_spec must be 16-byte aligned");
  if (transpose != 0 && transpose != 1) return fail(SSA_ERR_INVALID_ARGUMENT, "transpose must be 0 or 1");
  Plan& p = plan->p;
  CK(cudaSetDevice(p.device), "cudaSetDevice");
  if (p.large) {
    const int n_in = transpose ? (int)p.L : (int)p.K, n_out = transpose ? (int)p.K : (int)p.L;
    CK(ssa::large_correlate(p, reinterpret_cast<const double2*>(d_spec), (size_t)(p.H + 1), d_x, (size_t)n_in, n_in,
                            d_y, (size_t)n_out, n_out, n_out, nullptr, 0, nullptr, nullptr, (int)p.batch, S(stream)),
       "large matvec");
  } else {
    CK(ssa::launch_matvec(p, reinterpret_cast<const double2*>(d_spec), d_x, d_y, transpose, S(stream)),
       "matvec launch");
  }
  p.launches += 1;
  return SSA_OK;
}

extern "C" ssa_status ssa_matvec_multi(ssa_plan_t plan, const double* d_spec, const double* d_x, double* d_y,
                                       int32_t nvec, int transpose, void* stream) {
  if (!plan || !d_spec || !d_x || !d_y) return fail(SSA_ERR_INVALID_ARGUMENT, "NULL argument");
  if (((uintptr_t)d_spec) & 15) return fail(SSA_ERR_INVALID_ARGUMENT, "d_spec must be 16-byte aligned");
  if (transpose != 0 && transpose != 1) return fail(SSA_ERR_INVALID_ARGUMENT, "transpose must be 0 or 1");
  Plan& p = plan->p;
  if (nvec < 1 || p.batch * (int64_t)nvec > INT32_MAX)
    return fail(SSA_ERR_INVALID_ARGUMENT, "nvec must be >= 1 and batch * nvec < 2^31");
  CK(cudaSetDevice(p.device), "cudaSetDevice");
  const int n_in = transpose ? (int)p.L : (int)p.K, n_out = transpose ? (int)p.K : (int)p.L;
  if (p.large) {
    // one four-step pass per series: its nvec vectors against its one spectrum
    for (int64_t b = 0; b < p.batch; ++b)
      CK(ssa::large_correlate(p, reinterpret_cast<const double2*>(d_spec) + (size_t)b * (p.H + 1), 0,
                              d_x + (size_t)b * nvec * n_in, (size_t)n_in, n_in, d_y + (size_t)b * nvec * n_out,
                              (size_t)n_out, n_out, n_out, nullptr, 0, nullptr, nullptr, nvec, S(stream)),
         "large matvec");
  } else {
    CK(ssa::launch_matvec(p, reinterpret_cast<const double2*>(d_spec), d_x, d_y, transpose, S(stream), nvec),
       "matvec launch");
  }
  p.launches += 1;
  return SSA_OK;
}

extern "C" ssa_status ssa_hankelize(ssa_plan_t plan, const double* d_sigma, const double* d_U, const double* d_V,
                                    int32_t nterms, double* d_out, void* stream) {
  if (!plan || !d_sigma || !d_U || !d_V || !d_out) return fail(SSA_ERR_INVALID_ARGUMENT, "NULL argument");
  if (nterms < 1) return fail(SSA_ERR_INVALID_ARGUMENT, "nterms = %d < 1", nterms);
  Plan& p = plan->p;
  if ((int64_t)p.batch * nterms > (int64_t)0x7fffffff) return fail(SSA_ERR_INVALID_ARGUMENT, "batch*nterms too large");
  CK(cudaSetDevice(p.device), "cudaSetDevice");
  PhaseTimer pt(p, 4, S(stream));
  if (p.large) {
    CK(ssa::large_hankelize(p, d_sigma, d_U, d_V, (size_t)p.batch * nterms, d_out, S(stream)), "large hankelize");
  } else {
    CK(ssa::launch_hankelize(p, d_sigma, d_U, d_V, nterms, d_out, S(stream)), "hankelize launch");
  }
  p.launches += 1;
  return SSA_OK;
}

extern "C" ssa_status ssa_decompose(ssa_plan_t plan, const double* d_series, double* d_sigma, double* d_U,
                                    double* d_V, ssa_series_info* d_info, void* stream) {
  if (!plan || !d_series || !d_sigma || !d_U || !d_V) return fail(SSA_ERR_INVALID_ARGUMENT, "NULL argument");
  Plan& p = plan->p;
  if (p.k < 1) return fail(SSA_ERR_INVALID_ARGUMENT, "plan was created with k = 0");
  CK(cudaSetDevice(p.device), "cudaSetDevice");
  cudaStream_t s = S(stream);
  ssa::DecomposeArgs a;
  a.N = (int)p.N; a.L = (int)p.L; a.K = (int)p.K; a.M = (int)p.M; a.H = (int)p.H; a.k = p.k;
  a.m_max = p.m_max; a.ldL = p.ldL; a.ldK = p.ldK;
  a.check_every = p.opt.check_every; a.reorth_mode = p.opt.reorth; a.pro_eta = p.opt.reorth_eta;
  {
    // first test after 3k + 8 steps (no cfg1/cfg2 series converged before ~3.5k), then
    // every check_every steps, stretched up to 3 check_every when the residual decays
    // geometrically (R7); SSA_FIRST_CHECK / SSA_CHECK_CAP override (tuning)
    const int ce = p.opt.check_every > 0 ? p.opt.check_every : 4;
    a.first_check = 3 * p.k + 8;
    a.check_cap = 3 * ce;
    if (const char* e = getenv("SSA_FIRST_CHECK")) a.first_check = std::max(p.k, atoi(e));
    if (const char* e = getenv("SSA_CHECK_CAP")) a.check_cap = std::max(ce, atoi(e));
  }
  a.trl_d = p.opt.restart_dim > 0 ? p.m_max : 0;
  a.trl_p = p.opt.restart_keep;
  a.m_cap = p.m_cap;
  a.tol = p.opt.tol; a.seed = p.opt.seed; a.series_base = p.series_base;
  a.series = d_series; a.spec = p.d_spec; a.tw = p.d_twl;
  a.U = p.d_U; a.V = p.d_V; a.ab = p.d_ab; a.state = p.d_state;
  a.tgk = p.d_tgk; a.tgk_stride = (size_t)2 * p.k * (2 * p.m_max + 2);
  a.rot = p.d_rot; a.rot_cap = p.rot_cap; a.svd_slots = p.svd_slots;
  a.svd_method = (p.opt.reserved & 2) ? 1 : 0; a.tgkw = p.d_tgkw; a.tgkw_stride = tgkw_stride(p); a.vecs = p.d_vecs; a.coef = p.d_coef;
  a.sigma = d_sigma; a.Uout = d_U; a.Vout = d_V;
  a.info = d_info ? d_info : p.d_info;
  a.counters = p.d_counters;
  a.prof = p.d_prof;
  if (p.large) {
    PhaseTimer pt(p, 1, s);
    for (int64_t b = 0; b < p.batch; ++b) CK(ssa::large_decompose_one(p, a, (int)b, s), "long-series decompose");
    return SSA_OK;
  }
  for (int64_t b0 = 0; b0 < p.batch; b0 += p.chunk) {
    a.b0 = (int)b0;
    a.nb = (int)std::min<int64_t>(p.chunk, p.batch - b0);
    CK(cudaMemsetAsync(p.d_counters, 0, 4 * sizeof(int), s), "counter reset");
    {
      PhaseTimer pt(p, 0, s);
      CK(ssa::launch_spectrum(p, d_series + b0 * p.N, p.d_spec, a.nb, s), "spectrum launch");
    }
    {
      PhaseTimer pt(p, 1, s);
      CK(ssa::launch_lanczos(p, a, s), "lanczos launch");
    }
    {
      PhaseTimer pt(p, 2, s);
      CK(ssa::launch_bidiag_svd(p, a, s), "bidiag svd launch");
    }
    {
      PhaseTimer pt(p, 3, s);
      CK(ssa::launch_ritz(p, a, s), "ritz launch");
    }
    p.launches += 4;
  }
  return SSA_OK;
}

extern "C" ssa_status ssa_reconstruct(ssa_plan_t plan, const double* d_sigma, const double* d_U, const double* d_V,
                                      double* d_out, void* stream) {
  if (!plan) return fail(SSA_ERR_INVALID_ARGUMENT, "NULL plan");
  if (plan->p.k < 1) return fail(SSA_ERR_INVALID_ARGUMENT, "plan was created with k = 0");
  return ssa_hankelize(plan, d_sigma, d_U, d_V, plan->p.k, d_out, stream);
}

extern "C" ssa_status ssa_reconstruct_grouped(ssa_plan_t plan, const double* d_sigma, const double* d_U,
                                              const double* d_V, const int32_t* groups, int32_t ngroups, double* d_out,
                                              void* stream) {
  if (!plan || !d_sigma || !d_U || !d_V || !d_out || !groups) return fail(SSA_ERR_INVALID_ARGUMENT, "NULL argument");
  Plan& p = plan->p;
  const int k = p.k;
  if (k < 1) return fail(SSA_ERR_INVALID_ARGUMENT, "plan was created with k = 0");
  if (ngroups < 1 || ngroups > k) return fail(SSA_ERR_INVALID_ARGUMENT, "ngroups = %d not in [1, k = %d]", ngroups, k);
  if ((int64_t)p.batch * ngroups > (int64_t)0x7fffffff) return fail(SSA_ERR_INVALID_ARGUMENT, "batch*ngroups too large");
  ssa::GroupList gl{};
  gl.k = k;
  gl.ngroups = ngroups;
  int cnt[ssa::kMaxK + 1] = {0};
  for (int i = 0; i < k; ++i) {
    if (groups[i] < -1 || groups[i] >= ngroups)
      return fail(SSA_ERR_INVALID_ARGUMENT, "groups[%d] = %d not in [-1, %d)", i, groups[i], ngroups);
    if (groups[i] >= 0) cnt[groups[i] + 1]++;
  }
  for (int g = 0; g < ngroups; ++g) gl.ptr[g + 1] = gl.ptr[g] + cnt[g + 1];
  int fill[ssa::kMaxK] = {0};
  for (int i = 0; i < k; ++i)  // triples in increasing index order inside each group
    if (groups[i] >= 0) gl.idx[gl.ptr[groups[i]] + fill[groups[i]]++] = i;
  CK(cudaSetDevice(p.device), "cudaSetDevice");
  PhaseTimer pt(p, 4, S(stream));
  if (!p.large && p.H <= ssa::kMaxHankelSmemH) {
    CK(ssa::launch_group_hankelize(p, d_sigma, d_U, d_V, gl, d_out, S(stream)), "grouped hankelize launch");
    p.launches += 1;
    return SSA_OK;
  }
  // long path / H = 8192: elementary series into plan scratch, then the group sums
  ssa_status st;
  if (!p.d_elem && (st = alloc((void**)&p.d_elem, (size_t)p.batch * k * p.N * 8, "elementary series")) != SSA_OK)
    return st;
  if ((st = ssa_hankelize(plan, d_sigma, d_U, d_V, k, p.d_elem, stream)) != SSA_OK) return st;
  CK(ssa::launch_group_sum(p, p.d_elem, gl, d_out, S(stream)), "group sum launch");
  p.launches += 1;
  return SSA_OK;
}

// ---- heterogeneity matrix: plan (sub-plans + workspace, allocated once) and exec --------
struct ssa_hplan_s {
  int64_t N = 0, B = 0, T = 0, L = 0, KB = 0, KF = 0, nwin = 0;
  int nI = 0, kI = 0, device = 0;
  ssa_plan_t pa = nullptr, p1 = nullptr, pc = nullptr;  // window decompose, spectrum, products
  double *win = nullptr, *sig = nullptr, *U = nullptr, *V = nullptr, *x = nullptr, *y = nullptr, *spec = nullptr,
         *den = nullptr;
  int32_t* d_idx = nullptr;
  ssa_series_info* info = nullptr;
};

extern "C" void ssa_hmatrix_plan_destroy(ssa_hplan_t h) {
  if (!h) return;
  for (void* q : {(void*)h->win, (void*)h->sig, (void*)h->U, (void*)h->V, (void*)h->x, (void*)h->y, (void*)h->spec,
                  (void*)h->d_idx, (void*)h->den, (void*)h->info})
    if (q) cudaFree(q);
  if (h->pa) ssa_plan_destroy(h->pa);
  if (h->pc) ssa_plan_destroy(h->pc);
  if (h->p1) ssa_plan_destroy(h->p1);
  delete h;
}

extern "C" ssa_status ssa_hmatrix_plan_create(int64_t N, int64_t B, int64_t T, int64_t L, const int32_t* I, int32_t nI,
                                              const ssa_options* opt, int device, ssa_hplan_t* out) {
  if (!out || !I) return fail(SSA_ERR_INVALID_ARGUMENT, "NULL argument");
  *out = nullptr;
  if (N < 3 || L < 2 || B <= L || B > N || T < L || T > N)
    return fail(SSA_ERR_INVALID_ARGUMENT, "need N >= 3, 2 <= L < B <= N, L <= T <= N (N=%lld B=%lld T=%lld L=%lld)",
                (long long)N, (long long)B, (long long)T, (long long)L);
  const int64_t KB = B - L + 1, kmax = std::min(L, KB);
  if (nI < 1 || nI > ssa::kMaxK) return fail(SSA_ERR_INVALID_ARGUMENT, "nI = %d not in [1, %d]", nI, ssa::kMaxK);
  int kI = 0;
  std::vector<int32_t> idx((size_t)nI);
  for (int r = 0; r < nI; ++r) {
    if (I[r] < 1 || I[r] > kmax) return fail(SSA_ERR_INVALID_ARGUMENT, "I[%d] = %d not in [1, %lld]", r, I[r], (long long)kmax);
    for (int q = 0; q < r; ++q)
      if (I[q] == I[r]) return fail(SSA_ERR_INVALID_ARGUMENT, "I[%d] = %d repeated", r, I[r]);
    idx[(size_t)r] = I[r] - 1;
    kI = std::max(kI, (int)I[r]);
  }
  if (kI > ssa::kMaxK) return fail(SSA_ERR_INVALID_ARGUMENT, "max(I) = %d > %d", kI, ssa::kMaxK);
  CK(cudaSetDevice(device), "cudaSetDevice");
  ssa_hplan_s* h = new ssa_hplan_s();
  h->N = N; h->B = B; h->T = T; h->L = L; h->KB = KB; h->KF = N - L + 1; h->nwin = N - B + 1;
  h->nI = nI; h->kI = kI; h->device = device;
  const int64_t nwin = h->nwin;
  ssa_status st = SSA_OK;
  do {
    if ((st = ssa_plan_create(B, L, kI, nwin, opt, device, &h->pa)) != SSA_OK) break;
    if ((st = ssa_plan_create(N, L, 0, 1, opt, device, &h->p1)) != SSA_OK) break;
    if ((st = ssa_plan_create(N, L, 0, nwin * nI, opt, device, &h->pc)) != SSA_OK) break;
    if ((st = alloc((void**)&h->win, (size_t)nwin * B * 8, "H-matrix windows")) != SSA_OK) break;
    if ((st = alloc((void**)&h->sig, (size_t)nwin * kI * 8, "H-matrix sigma")) != SSA_OK) break;
    if ((st = alloc((void**)&h->U, (size_t)nwin * kI * L * 8, "H-matrix U")) != SSA_OK) break;
    if ((st = alloc((void**)&h->V, (size_t)nwin * kI * KB * 8, "H-matrix V")) != SSA_OK) break;
    if ((st = alloc((void**)&h->info, (size_t)nwin * sizeof(ssa_series_info), "H-matrix info")) != SSA_OK) break;
    if ((st = alloc((void**)&h->spec, (size_t)(h->pc->p.H + 1) * 16, "H-matrix spectrum")) != SSA_OK) break;
    if ((st = alloc((void**)&h->d_idx, (size_t)nI * 4, "H-matrix index")) != SSA_OK) break;
    if ((st = alloc((void**)&h->x, (size_t)nwin * nI * L * 8, "H-matrix vectors")) != SSA_OK) break;
    if ((st = alloc((void**)&h->y, (size_t)nwin * nI * h->KF * 8, "H-matrix projections")) != SSA_OK) break;
    if ((st = alloc((void**)&h->den, (size_t)(N - T + 1) * 8, "H-matrix norms")) != SSA_OK) break;
    cudaError_t e = cudaMemcpy(h->d_idx, idx.data(), (size_t)nI * 4, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) { st = cuda_fail(e, "H2D index"); break; }
  } while (0);
  if (st != SSA_OK) { ssa_hmatrix_plan_destroy(h); return st; }
  *out = h;
  return SSA_OK;
}

extern "C" ssa_status ssa_hmatrix_exec(ssa_hplan_t h, const double* d_series, double* d_G, ssa_series_info* d_info,
                                       void* stream) {
  if (!h || !d_series || !d_G) return fail(SSA_ERR_INVALID_ARGUMENT, "NULL argument");
  CK(cudaSetDevice(h->device), "cudaSetDevice");
  cudaStream_t s = S(stream);
  const int64_t nwin = h->nwin;
  ssa_series_info* info = d_info ? d_info : h->info;
  ssa_status st;
  cudaError_t e;
  // 1. leading left singular vectors of every base window (batched decompose)
  if ((e = ssa::launch_hm_windows(d_series, nwin, h->B, h->win, s)) != cudaSuccess) return cuda_fail(e, "hm windows");
  if ((st = ssa_decompose(h->pa, h->win, h->sig, h->U, h->V, info, stream)) != SSA_OK) return st;
  // 2. spectrum of the whole series once; X_F^T U_r for every (window, r) through it
  if ((st = ssa_spectrum(h->p1, d_series, h->spec, stream)) != SSA_OK) return st;
  if ((e = ssa::launch_hm_gather(h->U, nwin, h->kI, h->L, h->d_idx, h->nI, h->x, s)) != cudaSuccess)
    return cuda_fail(e, "hm gather");
  const Plan& qc = h->pc->p;
  if (qc.large)
    e = ssa::large_correlate(qc, reinterpret_cast<const double2*>(h->spec), 0, h->x, (size_t)h->L, (int)h->L, h->y,
                             (size_t)h->KF, (int)h->KF, (int)h->KF, nullptr, 0, nullptr, nullptr, (int)(nwin * h->nI), s);
  else
    e = ssa::launch_matvec_strided(qc, reinterpret_cast<const double2*>(h->spec), 0, h->x, h->y, 1, s);
  if (e != cudaSuccess) return cuda_fail(e, "H-matrix projections");
  // 3. the matrix: windowed sums of the squared projections over the norms of the lags
  if ((e = ssa::launch_hm_matrix(d_series, h->N, h->T, h->L, h->y, nwin, h->nI, h->KF, h->den, d_G, s)) != cudaSuccess)
    return cuda_fail(e, "H-matrix kernel");
  // per-window outcome (the host reads it after the stream synchronizes)
  std::vector<ssa_series_info> hi((size_t)nwin);
  CK(cudaMemcpyAsync(hi.data(), info, (size_t)nwin * sizeof(ssa_series_info), cudaMemcpyDeviceToHost, s), "D2H info");
  CK(cudaStreamSynchronize(s), "stream sync");
  for (const auto& q : hi)
    if (q.status != SSA_OK) return fail((ssa_status)q.status, "a base window did not converge");
  return SSA_OK;
}

extern "C" ssa_status ssa_hmatrix(const double* d_series, int64_t N, int64_t B, int64_t T, int64_t L,
                                  const int32_t* I, int32_t nI, const ssa_options* opt, int device, double* d_G,
                                  ssa_series_info* d_info, void* stream) {
  if (!d_series || !d_G || !I) return fail(SSA_ERR_INVALID_ARGUMENT, "NULL argument");
  ssa_hplan_t h = nullptr;
  ssa_status st = ssa_hmatrix_plan_create(N, B, T, L, I, nI, opt, device, &h);
  if (st != SSA_OK) return st;
  st = ssa_hmatrix_exec(h, d_series, d_G, d_info, stream);
  ssa_hmatrix_plan_destroy(h);
  return st;
}

extern "C" ssa_status ssa_bootstrap(ssa_plan_t plan, const double* d_series, const double* d_eps, double noise_sigma,
                                    double* d_mean, double* d_var, double* d_mse, double* d_G,
                                    ssa_series_info* d_info, void* stream) {
  if (!plan || !d_series || !d_eps || !d_mean) return fail(SSA_ERR_INVALID_ARGUMENT, "NULL argument");
  Plan& p = plan->p;
  if (p.k < 1) return fail(SSA_ERR_INVALID_ARGUMENT, "plan was created with k = 0");
  if (!(noise_sigma >= 0.0)) return fail(SSA_ERR_INVALID_ARGUMENT, "noise_sigma must be >= 0");
  CK(cudaSetDevice(p.device), "cudaSetDevice");
  cudaStream_t s = S(stream);
  const size_t R = (size_t)p.batch, N = (size_t)p.N, k = (size_t)p.k;
  ssa_status st;
  // plan scratch: replicates, reconstructions, sigma, U, V (one allocation)
  const size_t nbs = 2 * R * N + R * k * (1 + (size_t)p.L + (size_t)p.K);
  if (!p.d_bs && (st = alloc((void**)&p.d_bs, nbs * 8, "bootstrap workspace")) != SSA_OK) return st;
  double* reps = p.d_bs;
  double* G = d_G ? d_G : p.d_bs + R * N;
  double* sg = p.d_bs + 2 * R * N;
  double* Ub = sg + R * k;
  double* Vb = Ub + R * k * p.L;
  CK(ssa::launch_bs_replicates(d_series, d_eps, noise_sigma, (int64_t)R, (int64_t)N, reps, s), "bootstrap replicates");
  p.launches += 1;
  if ((st = ssa_decompose(plan, reps, sg, Ub, Vb, d_info, stream)) != SSA_OK) return st;
  std::vector<int32_t> groups(k, 0);  // the first k = d triples in one group: the rank-d signal
  if ((st = ssa_reconstruct_grouped(plan, sg, Ub, Vb, groups.data(), 1, G, stream)) != SSA_OK)
    return st;
  CK(ssa::launch_bs_stats(G, d_series, (int64_t)R, (int64_t)N, d_mean, d_var, d_mse, s), "bootstrap statistics");
  p.launches += 1;
  return SSA_OK;
}

extern "C" ssa_status ssa_run_host(ssa_plan_t plan, const double* h_series, double* h_sigma, double* h_U,
                                   double* h_V, double* h_recon, ssa_series_info* h_info, void* stream) {
  if (!plan || !h_series) return fail(SSA_ERR_INVALID_ARGUMENT, "NULL argument");
  Plan& p = plan->p;
  if (p.k < 1) return fail(SSA_ERR_INVALID_ARGUMENT, "plan was created with k = 0");
  CK(cudaSetDevice(p.device), "cudaSetDevice");
  ssa_status st;
  size_t B = (size_t)p.batch, k = (size_t)p.k;
  if (!p.d_series) {
    if ((st = alloc((void**)&p.d_series, B * p.N * 8, "series staging")) != SSA_OK) return st;
    if ((st = alloc((void**)&p.d_sigma, B * k * 8, "sigma staging")) != SSA_OK) return st;
    if ((st = alloc((void**)&p.d_Uout, B * k * p.L * 8, "U staging")) != SSA_OK) return st;
    if ((st = alloc((void**)&p.d_Vout, B * k * p.K * 8, "V staging")) != SSA_OK) return st;
    if ((st = alloc((void**)&p.d_recon, B * k * p.N * 8, "recon staging")) != SSA_OK) return st;
  }
  cudaStream_t s = S(stream);
  // Pipelined path: the batch in slices; slice i is decomposed + reconstructed by sub-plan
  // i % 2 on compute stream i % 2 (so one slice's kernel tail overlaps the next slice's
  // start) while the copy stream brings finished slices back -- the device-to-host copy of
  // the outputs (32 x the input bytes at cfg2) hides behind the compute of later slices.
  int nsl = 1;
  if (!p.large && B >= 512) nsl = 4;
  if (!p.large && B >= 2048) nsl = 8;  // cfg2 (4096 series): e2e 254K (4 slices) -> 271K eigentriples/s
  if (const char* e = getenv("SSA_HOST_SLICES")) nsl = std::max(1, std::min(Plan::kMaxSlices, atoi(e)));
  if (nsl > 1 && (int64_t)B >= 2 * nsl) {
    const int64_t sb = ((int64_t)B + nsl - 1) / nsl;
    nsl = (int)(((int64_t)B + sb - 1) / sb);
    const int64_t tail = (int64_t)B - (int64_t)(nsl - 1) * sb;  // 1 <= tail <= sb
    if (p.sub_batch != sb || p.tail_batch != tail) {
      for (int i = 0; i < 3; ++i)
        if (p.sub[i]) { ssa_plan_destroy(reinterpret_cast<ssa_plan_t>(p.sub[i])); p.sub[i] = nullptr; }
      for (int i = 0; i < 3; ++i) {
        if (i == 2 && tail == sb) break;
        ssa_plan_t q = nullptr;
        if ((st = ssa_plan_create(p.N, p.L, p.k, i < 2 ? sb : tail, &p.opt, p.device, &q)) != SSA_OK) return st;
        p.sub[i] = q;
      }
      p.sub_batch = sb;
      p.tail_batch = tail;
    }
    for (int i = 0; i < 4; ++i)
      if (!p.hs[i]) CK(cudaStreamCreateWithFlags(&p.hs[i], cudaStreamNonBlocking), "cudaStreamCreate");
    for (int i = 0; i < 2 * Plan::kMaxSlices + 2; ++i)
      if (!p.hev[i]) CK(cudaEventCreateWithFlags(&p.hev[i], cudaEventDisableTiming), "cudaEventCreate");
    cudaEvent_t ev_in = p.hev[2 * Plan::kMaxSlices], ev_cp = p.hev[2 * Plan::kMaxSlices + 1];
    CK(cudaEventRecord(ev_in, s), "event record");
    for (int c = 0; c < 4; ++c) CK(cudaStreamWaitEvent(p.hs[c], ev_in, 0), "stream wait");
    // inputs slice by slice on their own copy stream (host-to-device engine): slice i's
    // compute waits only for its own series
    for (int i = 0; i < nsl; ++i) {
      const size_t b0 = (size_t)i * sb;
      const size_t nb = std::min<size_t>(sb, B - b0);
      CK(cudaMemcpyAsync(p.d_series + b0 * p.N, h_series + b0 * p.N, nb * p.N * 8, cudaMemcpyHostToDevice, p.hs[3]),
         "H2D series");
      CK(cudaEventRecord(p.hev[Plan::kMaxSlices + i], p.hs[3]), "event record");
    }
    for (int i = 0; i < nsl; ++i) {
      const size_t b0 = (size_t)i * sb;
      const size_t nb = std::min<size_t>(sb, B - b0);
      // full slices alternate between sub-plans 0 and 1; a shorter last slice has its own
      // tail-sized sub-plan, so no rows are read or written by two streams at once
      const int si = (nb == (size_t)sb) ? (i & 1) : 2;
      ssa_plan_t qp = reinterpret_cast<ssa_plan_t>(p.sub[si]);
      Plan& q = qp->p;
      cudaStream_t cs = p.hs[i & 1];
      CK(cudaStreamWaitEvent(cs, p.hev[Plan::kMaxSlices + i], 0), "stream wait");
      q.series_base = p.series_base + (int64_t)b0;  // same start vectors as the single-launch path
      if ((st = ssa_decompose(qp, p.d_series + b0 * p.N, p.d_sigma + b0 * k, p.d_Uout + b0 * k * p.L,
                              p.d_Vout + b0 * k * p.K, p.d_info + b0, cs)) != SSA_OK)
        return st;
      if ((st = ssa_reconstruct(qp, p.d_sigma + b0 * k, p.d_Uout + b0 * k * p.L, p.d_Vout + b0 * k * p.K,
                                p.d_recon + b0 * k * p.N, cs)) != SSA_OK)
        return st;
      p.launches += q.launches;  // launch accounting of the caller's plan
      q.launches = 0;
      CK(cudaEventRecord(p.hev[i], cs), "event record");
      cudaStream_t ct = p.hs[2];
      CK(cudaStreamWaitEvent(ct, p.hev[i], 0), "stream wait");
      if (h_sigma) CK(cudaMemcpyAsync(h_sigma + b0 * k, p.d_sigma + b0 * k, nb * k * 8, cudaMemcpyDeviceToHost, ct), "D2H sigma");
      if (h_U) CK(cudaMemcpyAsync(h_U + b0 * k * p.L, p.d_Uout + b0 * k * p.L, nb * k * p.L * 8, cudaMemcpyDeviceToHost, ct), "D2H U");
      if (h_V) CK(cudaMemcpyAsync(h_V + b0 * k * p.K, p.d_Vout + b0 * k * p.K, nb * k * p.K * 8, cudaMemcpyDeviceToHost, ct), "D2H V");
      if (h_recon)
        CK(cudaMemcpyAsync(h_recon + b0 * k * p.N, p.d_recon + b0 * k * p.N, nb * k * p.N * 8, cudaMemcpyDeviceToHost, ct),
           "D2H recon");
    }
    CK(cudaEventRecord(ev_cp, p.hs[2]), "event record");
    CK(cudaStreamWaitEvent(s, ev_cp, 0), "stream wait");
  } else {
    CK(cudaMemcpyAsync(p.d_series, h_series, B * p.N * 8, cudaMemcpyHostToDevice, s), "H2D series");
    if ((st = ssa_decompose(plan, p.d_series, p.d_sigma, p.d_Uout, p.d_Vout, p.d_info, stream)) != SSA_OK) return st;
    if ((st = ssa_reconstruct(plan, p.d_sigma, p.d_Uout, p.d_Vout, p.d_recon, stream)) != SSA_OK) return st;
    if (h_sigma) CK(cudaMemcpyAsync(h_sigma, p.d_sigma, B * k * 8, cudaMemcpyDeviceToHost, s), "D2H sigma");
    if (h_U) CK(cudaMemcpyAsync(h_U, p.d_Uout, B * k * p.L * 8, cudaMemcpyDeviceToHost, s), "D2H U");
    if (h_V) CK(cudaMemcpyAsync(h_V, p.d_Vout, B * k * p.K * 8, cudaMemcpyDeviceToHost, s), "D2H V");
    if (h_recon) CK(cudaMemcpyAsync(h_recon, p.d_recon, B * k * p.N * 8, cudaMemcpyDeviceToHost, s), "D2H recon");
  }
  std::vector<ssa_series_info> info(B);
  CK(cudaMemcpyAsync(info.data(), p.d_info, B * sizeof(ssa_series_info), cudaMemcpyDeviceToHost, s), "D2H info");
  CK(cudaStreamSynchronize(s), "stream sync");
  if (h_info) memcpy(h_info, info.data(), B * sizeof(ssa_series_info));
  ssa_status worst = SSA_OK;
  for (size_t b = 0; b < B; ++b) {
    if (info[b].status == SSA_ERR_INVALID_ARGUMENT) return fail(SSA_ERR_INVALID_ARGUMENT, "series %zu is not finite", b);
    if (info[b].status != SSA_OK) worst = (ssa_status)info[b].status;
  }
  if (worst != SSA_OK) return fail(worst, "some series did not converge");
  return SSA_OK;
}

extern "C" ssa_status ssa_plan_phase_ms(ssa_plan_t plan, double out_ms[5]) {
  if (!plan || !out_ms) return fail(SSA_ERR_INVALID_ARGUMENT, "NULL argument");
  Plan& p = plan->p;
  CK(cudaSetDevice(p.device), "cudaSetDevice");
  for (int i = 0; i < Plan::kPhases; ++i) {
    out_ms[i] = -1.0;
    if (!p.ev_used[i]) continue;
    CK(cudaEventSynchronize(p.ev[2 * i + 1]), "event sync");
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, p.ev[2 * i], p.ev[2 * i + 1]), "event elapsed");
    out_ms[i] = ms;
  }
  return SSA_OK;
}

extern "C" ssa_status ssa_plan_profile(ssa_plan_t plan, int64_t out[8]) {
  if (!plan || !out) return fail(SSA_ERR_INVALID_ARGUMENT, "NULL argument");
  Plan& p = plan->p;
  if (!p.d_prof) return fail(SSA_ERR_INVALID_ARGUMENT, "plan was not created with profiling (options.reserved & 1)");
  CK(cudaSetDevice(p.device), "cudaSetDevice");
  CK(cudaMemcpy(out, p.d_prof, 8 * sizeof(int64_t), cudaMemcpyDeviceToHost), "D2H profile");
  return SSA_OK;
}

extern "C" ssa_status ssa_plan_bidiagonals(ssa_plan_t plan, double* h_alpha, double* h_beta, int32_t* h_steps) {
  if (!plan || !h_alpha || !h_beta || !h_steps) return fail(SSA_ERR_INVALID_ARGUMENT, "NULL argument");
  Plan& p = plan->p;
  if (p.k < 1) return fail(SSA_ERR_INVALID_ARGUMENT, "plan was created with k = 0");
  CK(cudaSetDevice(p.device), "cudaSetDevice");
  CK(cudaDeviceSynchronize(), "sync");
  const int64_t nb = std::min<int64_t>(p.chunk, p.batch - (p.batch - 1) / p.chunk * p.chunk);
  const size_t w = (size_t)p.m_max + 3;
  std::vector<double> ab((size_t)nb * 2 * w);
  std::vector<int> st((size_t)nb * ssa::kStateInts);
  CK(cudaMemcpy(ab.data(), p.d_ab, ab.size() * 8, cudaMemcpyDeviceToHost), "D2H ab");
  CK(cudaMemcpy(st.data(), p.d_state, st.size() * 4, cudaMemcpyDeviceToHost), "D2H state");
  for (int64_t b = 0; b < nb; ++b) {
    memcpy(h_alpha + b * w, &ab[(size_t)b * 2 * w], w * 8);
    memcpy(h_beta + b * w, &ab[(size_t)b * 2 * w + w], w * 8);
    h_steps[b] = st[(size_t)b * ssa::kStateInts];
  }
  return SSA_OK;
}

extern "C" const char* ssa_status_string(ssa_status s) {
  switch (s) {
    case SSA_OK: return "SSA_OK";
    case SSA_ERR_INVALID_ARGUMENT: return "SSA_ERR_INVALID_ARGUMENT";
    case SSA_ERR_NOT_CONVERGED: return "SSA_ERR_NOT_CONVERGED";
    case SSA_ERR_OUT_OF_MEMORY: return "SSA_ERR_OUT_OF_MEMORY";
    case SSA_ERR_CUDA: return "SSA_ERR_CUDA";
    case SSA_ERR_INTERNAL: return "SSA_ERR_INTERNAL";
    case SSA_ERR_UNSUPPORTED: return "SSA_ERR_UNSUPPORTED";
  }
  return "SSA_ERR_UNKNOWN";
}

extern "C" const char* ssa_last_error(void) { return g_err; }
