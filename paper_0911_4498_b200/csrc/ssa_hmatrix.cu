// ssa_hmatrix.cu -- heterogeneity matrix (H-matrix) of a series for structural-change
// detection (sec 6.2), on the hot-path kernels:
//
//   g_ij = 1 - sum_{m=1}^{K2} sum_{r in I} (U_r^(i)T X_m^(j))^2 / sum_{m=1}^{K2} |X_m^(j)|^2
//
// for base windows F_i = (f_i .. f_{i+B-1}), i = 1..N-B+1 (their leading left singular
// vectors U_r^(i), r in I, by the batched ssa_decompose) and test windows
// F_j = (f_j .. f_{j+T-1}), j = 1..N-T+1, whose L-lagged vectors X_m^(j) are the columns
// j .. j+K2-1 (K2 = T-L+1) of the trajectory matrix X_F of the whole series (window L).
// So U_r^T X_m^(j) = (X_F^T U_r)_{j+m-1}: ONE Hankel product X_F^T u per (i, r) through
// the stored spectrum of F gives the projections for every test window (the fast-matvec
// reduction of this step the paper mentions), and g_ij needs only
// windowed sums of their squares.  Kernels here: window gather, vector gather, and the
// matrix itself (one CTA per base window i, the rows (X_F^T U_r) staged in shared memory).
#include "device_common.cuh"

namespace ssa {

// win[i][t] = f[i + t], i < nwin, t < B
__global__ void hm_windows_kernel(const double* __restrict__ f, int64_t nwin, int64_t B, double* __restrict__ win) {
  const size_t total = (size_t)nwin * B;
  for (size_t x = (size_t)blockIdx.x * blockDim.x + threadIdx.x; x < total; x += (size_t)gridDim.x * blockDim.x) {
    const size_t i = x / B, t = x - i * B;
    win[x] = f[i + t];
  }
}

// x[i * nI + r][l] = U[i][idx[r]][l]  (U: [nwin][k][L])
__global__ void hm_gather_kernel(const double* __restrict__ U, int64_t nwin, int k, int64_t L,
                                 const int32_t* __restrict__ idx, int nI, double* __restrict__ x) {
  const size_t total = (size_t)nwin * nI * L;
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
    const size_t row = e / L, l = e - row * L;
    const size_t i = row / nI;
    const int r = (int)(row - i * nI);
    x[e] = U[((size_t)i * k + idx[r]) * L + l];
  }
}

// den[j] = sum_{m<K2} |X_{j+m}|^2 = sum_{t<T} c_t f_{j+t}^2, c_t = min(t+1, L, K2, T-t) (the
// number of lagged vectors of test window j that contain f_{j+t}); fixed order.
__global__ void hm_den_kernel(const double* __restrict__ f, int64_t N, int64_t T, int64_t L, double* __restrict__ den) {
  const int64_t K2 = T - L + 1, nj = N - T + 1;
  const int64_t mn = (L < K2) ? L : K2;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < nj; j += (int64_t)gridDim.x * blockDim.x) {
    double d = 0.0;
    for (int64_t t = 0; t < T; ++t) {
      int64_t c = t + 1;
      if (c > mn) c = mn;
      if (T - t < c) c = T - t;
      const double v = f[j + t];
      d = fma((double)c * v, v, d);
    }
    den[j] = d;
  }
}

// G[i][j] = 1 - num_ij / den_j:
//   num_ij = sum_r sum_{s=j}^{j+K2-1} y[i nI + r][s]^2   (y = X_F^T U_r^(i), length KF = N-L+1)
//   den_j  = sum_{m<K2} |X_{j+m}|^2 = sum_{t<T} c_t f_{j+t}^2, c_t = min(t+1, L, K2, T-t)
// (den from hm_den_kernel).  One CTA per i; the nI rows of y squared in shared memory;
// every thread sums its test windows directly (fixed order, deterministic; no prefix-sum
// cancellation).
__global__ void __launch_bounds__(kThreads) hm_matrix_kernel(const double* __restrict__ den, int64_t N, int64_t T,
                                                             int64_t L, const double* y, int64_t nwin, int nI,
                                                             int64_t KF, double* __restrict__ G, int staged,
                                                             double* sq) {
  extern __shared__ double ys_smem[];  // [nI][KF] squared projections (staged), else sq (global)
  const int64_t i = blockIdx.x;
  const int64_t K2 = T - L + 1, nj = N - T + 1;
  double* ys = staged ? ys_smem : sq + (size_t)i * nI * KF;
  for (int64_t e = threadIdx.x; e < (int64_t)nI * KF; e += blockDim.x) {
    const double v = y[(size_t)i * nI * KF + e];
    ys[e] = v * v;
  }
  __syncthreads();
  for (int64_t j = threadIdx.x; j < nj; j += blockDim.x) {
    double num = 0.0;
    for (int r = 0; r < nI; ++r) {
      const double* yr = ys + (size_t)r * KF + j;
      for (int64_t m = 0; m < K2; ++m) num += yr[m];
    }
    const double d = den[j];
    G[(size_t)i * nj + j] = (d > 0.0) ? 1.0 - num / d : 0.0;
  }
}

static unsigned grid_for(size_t total) {
  size_t g = (total + kThreads - 1) / kThreads;
  return (unsigned)(g < 65536 ? (g > 0 ? g : 1) : 65536);
}

cudaError_t launch_hm_windows(const double* f, int64_t nwin, int64_t B, double* win, cudaStream_t s) {
  hm_windows_kernel<<<grid_for((size_t)nwin * B), kThreads, 0, s>>>(f, nwin, B, win);
  return cudaGetLastError();
}

cudaError_t launch_hm_gather(const double* U, int64_t nwin, int k, int64_t L, const int32_t* d_idx, int nI, double* x,
                             cudaStream_t s) {
  hm_gather_kernel<<<grid_for((size_t)nwin * nI * L), kThreads, 0, s>>>(U, nwin, k, L, d_idx, nI, x);
  return cudaGetLastError();
}

// The squared projections of one base window are staged in shared memory when they fit,
// else squared in place into `y` itself (each CTA owns its rows).
cudaError_t launch_hm_matrix(const double* f, int64_t N, int64_t T, int64_t L, const double* y, int64_t nwin, int nI,
                             int64_t KF, double* den, double* G, cudaStream_t s) {
  hm_den_kernel<<<grid_for((size_t)(N - T + 1)), kThreads, 0, s>>>(f, N, T, L, den);
  const size_t smem = (size_t)nI * KF * 8;
  const bool staged = smem <= (size_t)200 * 1024;
  if (staged) {
    cudaError_t e = raise_smem_limit(hm_matrix_kernel, smem);
    if (e != cudaSuccess) return e;
  }
  hm_matrix_kernel<<<(unsigned)nwin, kThreads, staged ? smem : 0, s>>>(den, N, T, L, y, nwin, nI, KF, G,
                                                                        staged ? 1 : 0, const_cast<double*>(y));
  return cudaGetLastError();
}

}  // namespace ssa

namespace ssa {

// ---- bootstrap study (sec 6.3) -------------------
// replicates F'_r = F + noise_sigma * eps_r  (eps: [R][N], the caller's seeded noise)
__global__ void bs_replicates_kernel(const double* __restrict__ f, const double* __restrict__ eps, double noise_sigma,
                                     int64_t R, int64_t N, double* __restrict__ out) {
  const size_t total = (size_t)R * N;
  for (size_t x = (size_t)blockIdx.x * blockDim.x + threadIdx.x; x < total; x += (size_t)gridDim.x * blockDim.x)
    out[x] = fma(noise_sigma, eps[x], f[x % N]);
}

// per point t over the R reconstructions G_r: mean, unbiased variance (two passes, fixed
// order) and the mean square error against the clean series F
__global__ void bs_stats_kernel(const double* __restrict__ G, const double* __restrict__ f, int64_t R, int64_t N,
                                double* __restrict__ mean, double* __restrict__ var, double* __restrict__ mse) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < N; t += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0, e2 = 0.0;
    const double ft = f[t];
    for (int64_t r = 0; r < R; ++r) {
      const double g = G[(size_t)r * N + t];
      s += g;
      e2 = fma(g - ft, g - ft, e2);
    }
    const double m = s / (double)R;
    double v = 0.0;
    for (int64_t r = 0; r < R; ++r) {
      const double d = G[(size_t)r * N + t] - m;
      v = fma(d, d, v);
    }
    mean[t] = m;
    if (var) var[t] = (R > 1) ? v / (double)(R - 1) : 0.0;
    if (mse) mse[t] = e2 / (double)R;
  }
}

cudaError_t launch_bs_replicates(const double* f, const double* eps, double noise_sigma, int64_t R, int64_t N,
                                 double* out, cudaStream_t s) {
  bs_replicates_kernel<<<grid_for((size_t)R * N), kThreads, 0, s>>>(f, eps, noise_sigma, R, N, out);
  return cudaGetLastError();
}

cudaError_t launch_bs_stats(const double* G, const double* f, int64_t R, int64_t N, double* mean, double* var,
                            double* mse, cudaStream_t s) {
  bs_stats_kernel<<<grid_for((size_t)N), kThreads, 0, s>>>(G, f, R, N, mean, var, mse);
  return cudaGetLastError();
}

}  // namespace ssa
