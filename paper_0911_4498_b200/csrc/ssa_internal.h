// ssa_internal.h -- plan layout and launcher declarations shared by ssa_api.cu and the
// kernel translation units (library-internal; not part of the C-ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/ssa.h"

namespace ssa {

constexpr int kThreads = 256;          // threads per CTA for every kernel
constexpr int kWarps = kThreads / 32;  // warps per CTA
constexpr int kStages = 3;             // TMA ring depth per warp (basis streaming)
constexpr int kMaxSmemH = 8192;        // largest H = M/2 held in one CTA's shared memory
constexpr int kMaxHankelSmemH = 4096;  // largest H with both hankelization buffers in SMEM
constexpr int kMaxK = 128;             // largest k (2k <= kThreads: two lanes per value in tgk.cuh)
constexpr int kClCount = kMaxK + 1;    // tgk_clusters: index of the cluster count in cl[]
constexpr int kClInts = kMaxK + 2;     // ints of a cl[] array
constexpr int kStateInts = 12;         // per-series state words (DecomposeArgs::state)

inline size_t fft_bytes(int H) { return (size_t)H * 16; }

// Arguments of the three decompose kernels (lanczos -> bidiag SVD -> Ritz).  Per-series
// storage covers one chunk of nb series [b0, b0+nb) of the call.
struct DecomposeArgs {
  int N, L, K, M, H, k, m_max, ldL, ldK;
  int check_every, reorth_mode;  // reorth_mode 1/2: FRO (DGKS / always two passes), 3: PRO
  double pro_eta;                 // PRO threshold (ssa_options::reorth_eta)
  int first_check, check_cap;  // step of the first convergence test; longest stretch between tests
  int trl_d, trl_p;            // thick restart (ssa_options::restart_dim / restart_keep; 0: off)
  int m_cap;                   // thick restart: cap on the total Lanczos steps (m_max = trl_d)
  int b0, nb;
  double tol;
  uint64_t seed;
  int64_t series_base;   // global index of series 0 of the call (seeds are per global index)
  const double* series;  // caller [batch][N]
  const double2* spec;   // [nb][H+1]
  const double2* tw;     // two-level twiddle table for M
  double* U;             // [nb][m_max+1][ldL]  Krylov basis U_{m+1}
  double* V;             // [nb][m_max+1][ldK]  Krylov basis V_{m+1}
  double* ab;            // [nb][2][m_max+3]    alpha_j, beta_j (1-based)
  int* state;            // [nb][kStateInts]: m, converged, breakdown, reorth_extra, restarts, bad, checks,
                         // svd done, rows_u, rows_v, reorth_steps, -
  double* tgk;           // per Lanczos CTA slot: k * (2 m_max + 2) doubles
  size_t tgk_stride;
  double* rot;           // per SVD warp slot: 2 sides x rot_cap x 3 doubles
  int rot_cap;
  int svd_slots;         // warps with rotation / vector scratch (QR method)
  int svd_method;        // 0: TGK multisection + inverse iteration, 1: QR with records
  double* tgkw;          // per TGK-SVD CTA slot: Z (n k) + W (5 n k) + ipv (n k ints)
  size_t tgkw_stride;    // doubles
  double* vecs;          // per SVD warp slot: 2k x (m_max+2) doubles
  double* coef;          // [nb][2][m_max+2][k]: P_k rows then Q_k rows (signs folded)
  double* sigma;         // caller [batch][k]
  double* Uout;          // caller [batch][k][L]
  double* Vout;          // caller [batch][k][K]
  ssa_series_info* info; // [batch]
  int* counters;         // [4] work-queue heads (lanczos, svd, ritz)
  unsigned long long* prof;  // nullable, 8 counters
};

struct Plan {
  int device = 0;
  int64_t N = 0, L = 0, K = 0, M = 0, H = 0;
  int32_t k = 0;
  int64_t batch = 0;
  ssa_options opt{};
  int32_t m_max = 0;           // Krylov basis rows - 1 (thick restart: the Krylov dimension d)
  int32_t m_cap = 0;           // thick restart: cap on the total Lanczos steps
  int ldL = 0, ldK = 0;
  int sms = 0;
  int chunk = 0;               // series per decompose chunk (per-series storage)
  int lanczos_slots = 0;       // persistent CTAs of the Lanczos kernel
  int svd_slots = 0;           // warps of the SVD kernel
  int ritz_slots = 0;          // CTAs of the Ritz kernel
  int tgk_slots = 0;           // CTAs of the TGK SVD kernel
  double* d_tgkw = nullptr;
  // long-series (M > 2 kMaxSmemH) path: four-step FFT tables and buffers, Lanczos scratch
  bool large = false;
  double2* d_tw1 = nullptr;      // two-level table for the N1-point sub-FFTs (M = 2 N1)
  double2* d_tw2 = nullptr;      // two-level table for the N2-point sub-FFTs (M = 2 N2)
  double2* d_tw4 = nullptr;      // four-step twiddles: two-level W_H table (large_twh_entries)
  double2* d_twp = nullptr;      // pair-step row factors W_M^A, A <= N1/2
  double* d_rcpc = nullptr;      // 1/c for the antidiagonal counts c = 1..min(L, K) (hankelization)
  int hank_per = 64;             // terms per four-step hankelization batch
  cudaStream_t lg_aux = nullptr; // second stream: alternate hankelization batches overlap
  cudaEvent_t lg_ev[2] = {};     // fork / join events of lg_aux
  double2* d_lbuf = nullptr;     // [lbuf_items][H] complex work buffers
  int lbuf_items = 0;
  double* d_lgsc = nullptr;      // device scalars (LgScalars)
  double* d_lgpart = nullptr;    // partial sums
  double* d_lgh = nullptr;       // reorth coefficients
  double* d_lgr = nullptr;       // work vector
  double* d_lgom = nullptr;      // PRO omega estimates [2][m_max+4] (mu, nu)
  double* d_ucur = nullptr;      // current u_j / v_j of the long-series loop (fixed graph arguments)
  double* d_vcur = nullptr;
  cudaGraph_t lg_graph = nullptr;       // the long-series Lanczos loop (WHILE / IF graph)
  cudaGraphExec_t lg_exec = nullptr;
  bool lg_pdl = false;                  // the graph's kernels use programmatic dependent launch
  int rot_cap = 0;
  size_t smem_lanczos = 0, smem_ritz = 0;
  double2* d_tw = nullptr;     // twiddles exp(-2 pi i t / M), t < H (long-series path)
  double2* d_twl = nullptr;    // two-level twiddle table for M (tw2_entries(M))
  double2* d_spec = nullptr;   // [chunk][H+1]
  double* d_U = nullptr;
  double* d_V = nullptr;
  double* d_ab = nullptr;
  int* d_state = nullptr;
  double* d_tgk = nullptr;
  double* d_rot = nullptr;
  double* d_vecs = nullptr;
  double* d_coef = nullptr;
  ssa_series_info* d_info = nullptr;
  int* d_counters = nullptr;
  double2* d_hscratch = nullptr;  // BIG hankelization: per-CTA rfft(u) rows
  int hank_slots = 0;
  unsigned long long* d_prof = nullptr;  // profiling counters (options.reserved & 1)
  // host-API staging (allocated lazily by ssa_run_host)
  double* d_series = nullptr;
  double* d_sigma = nullptr;
  double* d_Uout = nullptr;
  double* d_Vout = nullptr;
  double* d_recon = nullptr;
  double* d_elem = nullptr;  // grouped reconstruction on the long path: elementary series
  double* d_bs = nullptr;    // bootstrap: replicates [batch][N] then reconstructions [batch][N]
  // host-API pipelining (ssa_run_host): two sub-plans of one slice each, alternating on two
  // compute streams, device-to-host copies of finished slices on a third stream
  void* sub[3] = {nullptr, nullptr, nullptr};  // ssa_plan_t: two full slices + the short tail slice
  int64_t sub_batch = 0, tail_batch = 0;
  int64_t series_base = 0;  // sub-plans: global index of their current slice's first series
  cudaStream_t hs[4] = {};  // compute x2, device-to-host, host-to-device
  static constexpr int kMaxSlices = 16;
  cudaEvent_t hev[2 * kMaxSlices + 2] = {};  // per slice: computed, inputs copied; + 2
  int64_t launches = 0;
  static constexpr int kPhases = 5;  // spectrum, lanczos, bidiag_svd, ritz, hankelize
  cudaEvent_t ev[2 * kPhases] = {};
  bool ev_used[kPhases] = {};
};

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) that never lowers the limit set by an
// earlier plan on the same device (the attribute is per function, plans are not): the
// limit becomes the maximum over all plans created so far.  Thread-safe (ssa_api.cu).
cudaError_t raise_smem_limit(const void* func, size_t bytes);
template <class F>
inline cudaError_t raise_smem_limit(F* func, size_t bytes) {
  return raise_smem_limit(reinterpret_cast<const void*>(func), bytes);
}

// launchers; return cudaGetLastError() after enqueue
cudaError_t launch_spectrum(const Plan& p, const double* series, double2* spec, int nseries, cudaStream_t s);
// nvec products per series: item b uses the spectrum of series b / nvec (x, y: [batch][nvec][n])
cudaError_t launch_matvec(const Plan& p, const double2* spec, const double* x, double* y, int transpose,
                          cudaStream_t s, int nvec = 1);
// spec_stride (double2 elements) between the series' spectra; 0: one spectrum for all
cudaError_t launch_matvec_strided(const Plan& p, const double2* spec, size_t spec_stride, const double* x, double* y,
                                  int transpose, cudaStream_t s, int nvec = 1);
// heterogeneity matrix helpers (ssa_hmatrix.cu)
cudaError_t launch_hm_windows(const double* f, int64_t nwin, int64_t B, double* win, cudaStream_t s);
cudaError_t launch_hm_gather(const double* U, int64_t nwin, int k, int64_t L, const int32_t* d_idx, int nI, double* x,
                             cudaStream_t s);
cudaError_t launch_hm_matrix(const double* f, int64_t N, int64_t T, int64_t L, const double* y, int64_t nwin, int nI,
                             int64_t KF, double* den, double* G, cudaStream_t s);
cudaError_t launch_bs_replicates(const double* f, const double* eps, double noise_sigma, int64_t R, int64_t N,
                                 double* out, cudaStream_t s);
cudaError_t launch_bs_stats(const double* G, const double* f, int64_t R, int64_t N, double* mean, double* var,
                            double* mse, cudaStream_t s);
cudaError_t launch_hankelize(const Plan& p, const double* sigma, const double* U, const double* V, int nterms,
                             double* out, cudaStream_t s);
cudaError_t fft_set_attributes(int H, const char** which);
// Grouping of the k triples (CSR by group, passed by value): triples idx[ptr[g] .. ptr[g+1])
struct GroupList {
  int k, ngroups;
  int ptr[kMaxK + 1];
  int idx[kMaxK];
};
cudaError_t launch_group_hankelize(const Plan& p, const double* sigma, const double* U, const double* V,
                                   const GroupList& gl, double* out, cudaStream_t s);
cudaError_t launch_group_sum(const Plan& p, const double* elem, const GroupList& gl, double* out, cudaStream_t s);

size_t lanczos_smem_bytes(int H, int ldL, int ldK, int m_max, int k, bool trl = false);
size_t ritz_smem_bytes(int ldL, int ldK, int k, int m_max);
cudaError_t lanczos_set_attributes(size_t smem);
cudaError_t svd_ritz_set_attributes(int m_max, size_t smem_ritz);
constexpr int kSvdWarpsPerCta = 8;
cudaError_t launch_lanczos(const Plan& p, const DecomposeArgs& a, cudaStream_t s);
cudaError_t launch_bidiag_svd(const Plan& p, const DecomposeArgs& a, cudaStream_t s);
cudaError_t launch_ritz(const Plan& p, const DecomposeArgs& a, cudaStream_t s);

// long-series path (ssa_large_fft.cu, ssa_large_lanczos.cu)
constexpr int kMaxLargeH = 1 << 20;  // N1, N2 <= 1024
void large_geom(const Plan& p, int* N1, int* N2);
int large_twh_entries(int logH);
cudaError_t large_set_attributes(int N1, int N2);
cudaError_t large_lanczos_set_attributes(int m_max);
cudaError_t large_spectrum(const Plan& p, const double* series, double2* spec, int items, cudaStream_t s);
cudaError_t large_correlate(const Plan& p, const double2* spec, size_t spec_stride, const double* x, size_t xs, int n_in,
                            double* out, size_t os, int n_out, int ld_out, const double* prev, size_t ps,
                            const double* coef, double* part, int items, cudaStream_t s,
                            const int* gate = nullptr);
cudaError_t large_hankelize(Plan& p, const double* sigma, const double* U, const double* V, size_t nterm_total,
                            double* out, cudaStream_t s);
cudaError_t large_decompose_one(Plan& p, const DecomposeArgs& a, int b, cudaStream_t s);

}  // namespace ssa
