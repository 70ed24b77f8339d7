// dmma_check.cu -- fragment layout of mma.sync.aligned.m8n8k4.row.col.f64 on sm_100a
// (the fp64 tensor-core op lg_ritz uses): D = A B + C with A 8x4 (row), B 4x8 (col);
// lane l holds A[l>>2][l&3], B[l&3][l>>2], D[l>>2][2(l&3)+{0,1}].  Prints the max error vs
// the host product.  nvcc -gencode arch=compute_100a,code=sm_100a -o tools/dmma_check tools/dmma_check.cu
#include <cstdio>
#include <cmath>
__global__ void k(const double* A, const double* B, double* D) {
  const int l = threadIdx.x;
  double a = A[(l >> 2) * 4 + (l & 3)];
  double b = B[(l & 3) * 8 + (l >> 2)];
  double d0 = 0.0, d1 = 0.0;
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
  D[(l >> 2) * 8 + 2 * (l & 3)] = d0;
  D[(l >> 2) * 8 + 2 * (l & 3) + 1] = d1;
}
int main() {
  double hA[32], hB[32], hD[64], ref[64];
  for (int i = 0; i < 32; ++i) { hA[i] = 1.0 + i * 0.37; hB[i] = 2.0 - i * 0.11; }
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 8; ++j) {
      double s = 0;
      for (int q = 0; q < 4; ++q) s += hA[i * 4 + q] * hB[q * 8 + j];
      ref[i * 8 + j] = s;
    }
  double *A, *B, *D;
  cudaMalloc(&A, 256); cudaMalloc(&B, 256); cudaMalloc(&D, 512);
  cudaMemcpy(A, hA, 256, cudaMemcpyHostToDevice); cudaMemcpy(B, hB, 256, cudaMemcpyHostToDevice);
  k<<<1, 32>>>(A, B, D);
  cudaMemcpy(hD, D, 512, cudaMemcpyDeviceToHost);
  double e = 0;
  for (int i = 0; i < 64; ++i) e = fmax(e, fabs(hD[i] - ref[i]));
  printf("dmma m8n8k4 f64 max abs err %.3e (%s)\n", e, e < 1e-12 ? "layout ok" : "LAYOUT WRONG");
  return e < 1e-12 ? 0 : 1;
}
