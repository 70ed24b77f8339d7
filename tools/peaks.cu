// Microbenchmarks for the roofline denominators the driver does not measure:
// fp64 DFMA / DADD pipe throughput, fp64 DMMA (mma.sync m8n8k4 f64) throughput,
// HBM fp64 streaming read and copy bandwidth, and L2-resident read bandwidth.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/peaks tools/peaks.cu
// Prints one JSON object on stdout.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

template <int CHAINS>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = fma(x[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += x[c];
  if (s == 12345.678) out[0] = s;
}

template <int CHAINS>
__global__ void dadd_kernel(double* out, int iters, double a) {
  double x[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = x[c] + a;
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += x[c];
  if (s == 12345.678) out[0] = s;
}

// m8n8k4 f64 mma: 8*8*4*2 = 512 flop per warp-instruction.
template <int CHAINS>
__global__ void dmma_kernel(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-6, b = 0.5;
  double c[CHAINS][2];
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) { c[k][0] = 0; c[k][1] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < CHAINS; ++k) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) s += c[k][0] + c[k][1];
  if (s == 12345.678) out[0] = s;
}

__global__ void read_kernel(const double2* __restrict__ in, size_t n, double* out) {
  double2 acc = make_double2(0, 0);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    double2 v = __ldcg(in + i);
    acc.x += v.x; acc.y += v.y;
  }
  if (acc.x + acc.y == 12345.678) out[0] = acc.x;
}

__global__ void copy_kernel(const double2* __restrict__ in, double2* __restrict__ o, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    o[i] = in[i];
}

int main() {
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, 0));
  int sms = p.multiProcessorCount;
  double* d_out;
  CK(cudaMalloc(&d_out, 64));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  float ms;
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"smem_optin\": %zu, \"l2_bytes\": %d", p.name, sms,
         (size_t)p.sharedMemPerBlockOptin, p.l2CacheSize);

  // DFMA
  {
    const int iters = 1 << 16, threads = 256, blocks = sms * 8;
    for (int w = 0; w < 2; ++w) dfma_kernel<8><<<blocks, threads>>>(d_out, iters, 0.999999, 1e-7);
    CK(cudaDeviceSynchronize());
    double best = 0;
    for (int r = 0; r < 5; ++r) {
      CK(cudaEventRecord(e0));
      dfma_kernel<8><<<blocks, threads>>>(d_out, iters, 0.999999, 1e-7);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      CK(cudaEventElapsedTime(&ms, e0, e1));
      double tf = 2.0 * 8 * (double)iters * threads * blocks / (ms * 1e-3) / 1e12;
      if (tf > best) best = tf;
    }
    printf(", \"dfma_tflops\": %.3f", best);
    // sustained: back-to-back launches for ~4 s (power / clock limits under a long load,
    // the regime of a kernel timed inside a long step); the shell samples the SM clock
    CK(cudaEventRecord(e0));
    int n = 0;
    for (;;) {
      for (int r = 0; r < 20; ++r) dfma_kernel<8><<<blocks, threads>>>(d_out, iters, 0.999999, 1e-7);
      n += 20;
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (ms > 4000.0f) break;
    }
    printf(", \"dfma_tflops_sustained\": %.3f", 2.0 * 8 * (double)iters * threads * blocks * n / (ms * 1e-3) / 1e12);
  }
  // DADD
  {
    const int iters = 1 << 16, threads = 256, blocks = sms * 8;
    dadd_kernel<8><<<blocks, threads>>>(d_out, iters, 1e-7);
    CK(cudaDeviceSynchronize());
    double best = 0;
    for (int r = 0; r < 5; ++r) {
      CK(cudaEventRecord(e0));
      dadd_kernel<8><<<blocks, threads>>>(d_out, iters, 1e-7);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      CK(cudaEventElapsedTime(&ms, e0, e1));
      double tops = 8.0 * (double)iters * threads * blocks / (ms * 1e-3) / 1e12;
      if (tops > best) best = tops;
    }
    printf(", \"dadd_tops\": %.3f", best);
  }
  // DMMA
  {
    const int iters = 1 << 14, threads = 256, blocks = sms * 8;
    dmma_kernel<4><<<blocks, threads>>>(d_out, iters);
    CK(cudaDeviceSynchronize());
    double best = 0;
    for (int r = 0; r < 5; ++r) {
      CK(cudaEventRecord(e0));
      dmma_kernel<4><<<blocks, threads>>>(d_out, iters);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      CK(cudaEventElapsedTime(&ms, e0, e1));
      double tf = 512.0 * 4 * (double)iters * (threads / 32) * blocks / (ms * 1e-3) / 1e12;
      if (tf > best) best = tf;
    }
    printf(", \"dmma_tflops\": %.3f", best);
  }
  // HBM read / copy (2 GiB each side), L2 read (32 MiB and 64 MiB)
  {
    size_t bytes = (size_t)2 << 30;
    size_t n = bytes / 16;
    double2 *a, *b;
    CK(cudaMalloc(&a, bytes));
    CK(cudaMalloc(&b, bytes));
    CK(cudaMemset(a, 0, bytes));
    CK(cudaMemset(b, 0, bytes));
    int blocks = sms * 8, threads = 512;
    double best_r = 0, best_c = 0;
    for (int r = 0; r < 6; ++r) {
      CK(cudaEventRecord(e0));
      read_kernel<<<blocks, threads>>>(a, n, d_out);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      CK(cudaEventElapsedTime(&ms, e0, e1));
      double gbs = bytes / (ms * 1e-3) / 1e9;
      if (r && gbs > best_r) best_r = gbs;
      CK(cudaEventRecord(e0));
      copy_kernel<<<blocks, threads>>>(a, b, n);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      CK(cudaEventElapsedTime(&ms, e0, e1));
      gbs = 2.0 * bytes / (ms * 1e-3) / 1e9;
      if (r && gbs > best_c) best_c = gbs;
    }
    printf(", \"hbm_read_gbs\": %.1f, \"hbm_copy_gbs\": %.1f", best_r, best_c);
    size_t l2sizes[3] = {(size_t)16 << 20, (size_t)32 << 20, (size_t)64 << 20};
    for (int s = 0; s < 3; ++s) {
      size_t ln = l2sizes[s] / 16;
      double best = 0;
      for (int r = 0; r < 8; ++r) {
        CK(cudaEventRecord(e0));
        for (int rep = 0; rep < 20; ++rep) read_kernel<<<blocks, threads>>>(a, ln, d_out);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        CK(cudaEventElapsedTime(&ms, e0, e1));
        double gbs = 20.0 * l2sizes[s] / (ms * 1e-3) / 1e9;
        if (r && gbs > best) best = gbs;
      }
      printf(", \"l2_read_gbs_%zuMiB\": %.1f", l2sizes[s] >> 20, best);
    }
    CK(cudaFree(a));
    CK(cudaFree(b));
  }
  printf("}\n");
  return 0;
}
