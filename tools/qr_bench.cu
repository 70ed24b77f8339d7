// Microbenchmark: cycles of bidiag_qr (one thread) and of the record application
// (one warp) on a Lanczos bidiagonal (tools/B_m110.bin: m, alpha[0..m+2], beta[0..m+2]).
#include <cstdio>
#include <vector>
#include "../paper_0911_4498_b200/csrc/bidiag_qr.cuh"
using namespace ssa;
__global__ void k_qr(int m, const double* al, const double* be, int2* abL, double2* csL, int2* abR, double2* csR,
                     int cap, double* vec, long long* out) {
  __shared__ double d[300], e[300], w[300];
  __shared__ int sel[32];
  __shared__ double om[32];
  __shared__ int nn[2];
  long long t0 = clock64();
  if (threadIdx.x == 0) {
    RotRec rl{abL, csL, cap, 0}, rr{abR, csR, cap, 0};
    int it = bidiag_qr<true, true>(m, al, be, d, e, w, &rl, &rr, 30 * m + 100);
    select_topk(m, d, 16, sel, om);
    nn[0] = rl.n; nn[1] = rr.n;
    out[2] = it;
  }
  __syncwarp();
  long long t1 = clock64();
  int t = threadIdx.x, k2 = 32;
  for (int r = 0; r <= m; ++r) vec[r * k2 + t] = 0.0;
  int i = t < 16 ? t : t - 16;
  vec[sel[i] * k2 + t] = 1.0;
  if (t < 16) apply_records_reverse(abL, csL, nn[0], vec + t, k2);
  else apply_records_reverse(abR, csR, nn[1], vec + t, k2);
  __syncwarp();
  long long t2 = clock64();
  if (t == 0) { out[0] = t1 - t0; out[1] = t2 - t1; out[3] = nn[0]; out[4] = nn[1]; }
}
int main() {
  FILE* f = fopen("tools/B_m110.bin", "rb");
  std::vector<double> buf(1 + 2 * 113);
  fread(buf.data(), 8, buf.size(), f); fclose(f);
  int m = (int)buf[0];
  double *dal, *dbe, *vec; int2 *abL, *abR; double2 *csL, *csR; long long* out;
  int cap = 2 * m * m + 8 * m + 1024;
  cudaMalloc(&dal, 8 * (m + 3)); cudaMalloc(&dbe, 8 * (m + 3));
  cudaMemcpy(dal, buf.data() + 1, 8 * (m + 3), cudaMemcpyHostToDevice);
  cudaMemcpy(dbe, buf.data() + 1 + m + 3, 8 * (m + 3), cudaMemcpyHostToDevice);
  cudaMalloc(&abL, 8 * cap); cudaMalloc(&abR, 8 * cap); cudaMalloc(&csL, 16 * cap); cudaMalloc(&csR, 16 * cap);
  cudaMalloc(&vec, 8 * 32 * (m + 2)); cudaMalloc(&out, 64);
  for (int rep = 0; rep < 3; ++rep) {
    k_qr<<<1, 32>>>(m, dal, dbe, abL, csL, abR, csR, cap, vec, out);
    long long h[5];
    cudaMemcpy(h, out, 40, cudaMemcpyDeviceToHost);
    printf("m=%d iters=%lld recL=%lld recR=%lld qr_cycles=%lld (%.1f/rot) apply_cycles=%lld (%.1f/rec) err=%s\n", m,
           h[2], h[3], h[4], h[0], (double)h[0] / (h[3] + h[4]), h[1], (double)h[1] / h[3],
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
