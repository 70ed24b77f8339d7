// ssa_internal.h -- plan layout and launcher declarations shared by ssa_api.cu and
// ssa_kernels.cu (library-internal; not part of the C-ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/ssa.h"

namespace ssa {

constexpr int kThreads = 256;          // threads per CTA for every kernel
constexpr int kWarps = kThreads / 32;  // worker warps in the Lanczos kernel
constexpr int kStages = 3;             // TMA ring depth per warp (basis streaming)
constexpr int kMaxSmemH = 8192;        // largest H = M/2 held in one CTA's shared memory
constexpr int kMaxHankelSmemH = 4096;  // largest H with both hankelization buffers in SMEM

inline size_t fpad_bytes(int H) { return (size_t)(H + (H >> 3) + 1) * 16; }

struct LanczosArgs {
  int N, L, K, M, H, k, m_max, ldL, ldK;
  int check_every, reorth_mode, batch;
  double tol;
  uint64_t seed;
  const double* series;     // [batch][N]
  const double2* spec;      // [batch][H+1]
  const double2* tw;        // [H]
  double* Ubase;            // per slot: (m_max+1) x ldL
  double* Vbase;            // per slot: (m_max+1) x ldK
  size_t slot_stride_U, slot_stride_V;  // doubles
  double* rot;              // per slot rotation records
  size_t slot_stride_rot;   // doubles
  int rot_cap;              // records per side per slot
  double* pq;               // per slot: P_k ((m_max+1) x k) and Q_k (m_max x k)
  size_t slot_stride_pq;
  double* sigma;            // [batch][k]
  double* Uout;             // [batch][k][L]
  double* Vout;             // [batch][k][K]
  ssa_series_info* info;    // [batch] (never NULL: plan scratch if caller passed NULL)
  int* counter;             // work queue head
};

struct Plan {
  int device = 0;
  int64_t N = 0, L = 0, K = 0, M = 0, H = 0;
  int32_t k = 0;
  int64_t batch = 0;
  ssa_options opt{};
  int32_t m_max = 0;
  int ldL = 0, ldK = 0;
  int sms = 0;
  int slots = 0;           // persistent CTAs for decompose
  size_t smem_lanczos = 0;
  double2* d_tw = nullptr;       // twiddles exp(-2 pi i t / M), t < H
  double2* d_spec = nullptr;     // [batch][H+1] spectra owned by the plan (decompose)
  double* d_U = nullptr;         // bases
  double* d_V = nullptr;
  double* d_rot = nullptr;
  double* d_pq = nullptr;
  ssa_series_info* d_info = nullptr;
  int* d_counter = nullptr;
  double2* d_hscratch = nullptr;  // BIG hankelization: per-CTA rfft(u) rows
  int hank_slots = 0;
  // host-API staging (allocated lazily by ssa_run_host)
  double* d_series = nullptr;
  double* d_sigma = nullptr;
  double* d_Uout = nullptr;
  double* d_Vout = nullptr;
  double* d_recon = nullptr;
  int64_t launches = 0;
  cudaEvent_t ev[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};  // [start,end] x 3 phases
  bool ev_used[3] = {false, false, false};
};

// launchers (ssa_kernels.cu); return cudaGetLastError() after enqueue
cudaError_t launch_spectrum(const Plan& p, const double* series, double2* spec, cudaStream_t s);
cudaError_t launch_matvec(const Plan& p, const double2* spec, const double* x, double* y, int transpose,
                          cudaStream_t s);
cudaError_t launch_hankelize(const Plan& p, const double* sigma, const double* U, const double* V, int nterms,
                             double* out, cudaStream_t s);
cudaError_t launch_lanczos(const Plan& p, const LanczosArgs& a, cudaStream_t s);
size_t lanczos_smem_bytes(int H, int ldL, int ldK, int m_max, int k);
cudaError_t lanczos_set_attributes(size_t smem);
cudaError_t fft_set_attributes(int H, const char** which);

}  // namespace ssa
