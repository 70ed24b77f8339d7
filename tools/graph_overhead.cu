// graph_overhead.cu -- cost of the building blocks of the long-series Lanczos loop graph
// (ssa_large_lanczos.cu) on the device: a kernel launch on a stream with / without
// programmatic dependent launch (PDL), the same inside a captured WHILE-graph body, and an
// IF conditional node that is taken or skipped.  Empty 1-CTA kernels, so the numbers are
// pure launch / dependency overheads per node.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/graph_overhead tools/graph_overhead.cu
#include <cuda_runtime.h>
#include <stdio.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e_ = (x);                                                          \
    if (e_ != cudaSuccess) {                                                       \
      printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_));   \
      return 1;                                                                    \
    }                                                                              \
  } while (0)

__global__ void k_nop(int* c) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0 && c) atomicAdd(c, 1);
}
__global__ void k_set(cudaGraphConditionalHandle h, int v) {
  if (threadIdx.x == 0) cudaGraphSetConditional(h, v);
}
__global__ void k_loop(cudaGraphConditionalHandle h, int* it, int n) {
  if (threadIdx.x == 0) {
    int v = ++*it;
    cudaGraphSetConditional(h, v < n ? 1u : 0u);
  }
}

__global__ void k_gridsync(int n, int* c) {
  cg::grid_group g = cg::this_grid();
  for (int i = 0; i < n; ++i) g.sync();
  if (c && threadIdx.x == 0 && blockIdx.x == 0) *c = n;
}

static bool g_pdl = true;
static cudaError_t launch(cudaStream_t s, int* c) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(1);
  cfg.blockDim = dim3(128);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = g_pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k_nop, c);
}

// WHILE graph: body = nk kernels, then (optional) IF(taken) with 1 kernel, k_loop
static int build(cudaGraphExec_t* ex, int* it, int iters, int nk, int nif, int taken, cudaStream_t s1, cudaStream_t s2) {
  cudaGraph_t g;
  CK(cudaGraphCreate(&g, 0));
  cudaGraphConditionalHandle hw;
  CK(cudaGraphConditionalHandleCreate(&hw, g, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams wp = {};
  wp.type = cudaGraphNodeTypeConditional;
  wp.conditional.handle = hw;
  wp.conditional.type = cudaGraphCondTypeWhile;
  wp.conditional.size = 1;
  cudaGraphNode_t wn;
  CK(cudaGraphAddNode(&wn, g, nullptr, 0, &wp));
  cudaGraph_t body = wp.conditional.phGraph_out[0];
  CK(cudaStreamBeginCaptureToGraph(s1, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  for (int i = 0; i < nk; ++i) CK(launch(s1, nullptr));
  for (int q = 0; q < nif; ++q) {
    cudaStreamCaptureStatus st;
    cudaGraph_t cg;
    const cudaGraphNode_t* deps;
    size_t nd;
    CK(cudaStreamGetCaptureInfo(s1, &st, nullptr, &cg, nullptr, nullptr));
    cudaGraphConditionalHandle hi;
    CK(cudaGraphConditionalHandleCreate(&hi, cg, 0, cudaGraphCondAssignDefault));
    k_set<<<1, 32, 0, s1>>>(hi, taken);
    CK(cudaStreamGetCaptureInfo(s1, &st, nullptr, &cg, &deps, &nd));
    cudaGraphNodeParams ip = {};
    ip.type = cudaGraphNodeTypeConditional;
    ip.conditional.handle = hi;
    ip.conditional.type = cudaGraphCondTypeIf;
    ip.conditional.size = 1;
    cudaGraphNode_t in;
    CK(cudaGraphAddNode(&in, cg, deps, nd, &ip));
    CK(cudaStreamUpdateCaptureDependencies(s1, &in, 1, cudaStreamSetCaptureDependencies));
    cudaGraph_t ib = ip.conditional.phGraph_out[0];
    CK(cudaStreamBeginCaptureToGraph(s2, ib, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    CK(launch(s2, nullptr));
    cudaGraph_t o2;
    CK(cudaStreamEndCapture(s2, &o2));
    CK(launch(s1, nullptr));
  }
  k_loop<<<1, 32, 0, s1>>>(hw, it, iters);
  cudaGraph_t o;
  CK(cudaStreamEndCapture(s1, &o));
  cudaError_t e = cudaGraphInstantiate(ex, g, 0);
  if (e != cudaSuccess) {
    printf("instantiate failed (pdl=%d): %s\n", (int)g_pdl, cudaGetErrorString(e));
    cudaGetLastError();
    return 2;
  }
  return 0;
}

int main() {
  cudaStream_t s, s1, s2;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  int* it;
  CK(cudaMalloc(&it, 4));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  const int iters = 200, nk = 20;
  for (int pdl = 1; pdl >= 0; --pdl) {
    g_pdl = pdl;
    // plain stream launches
    for (int w = 0; w < 2; ++w) {
      CK(cudaEventRecord(a, s));
      for (int i = 0; i < iters * nk; ++i) CK(launch(s, nullptr));
      CK(cudaEventRecord(b, s));
      CK(cudaEventSynchronize(b));
    }
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    printf("stream  pdl=%d: %.2f us per kernel\n", pdl, 1e3 * ms / (iters * nk));
    const int cfgs[][3] = {{nk, 0, 0}, {nk, 4, 0}, {nk, 4, 1}};
    for (auto& c : cfgs) {
      cudaGraphExec_t ex;
      int r = build(&ex, it, iters, c[0], c[1], c[2], s1, s2);
      if (r) continue;
      for (int w = 0; w < 2; ++w) {
        CK(cudaMemsetAsync(it, 0, 4, s));
        CK(cudaEventRecord(a, s));
        CK(cudaGraphLaunch(ex, s));
        CK(cudaEventRecord(b, s));
        CK(cudaEventSynchronize(b));
      }
      CK(cudaEventElapsedTime(&ms, a, b));
      const int nker = c[0] + c[1] * (2 + c[2]) + 1;
      printf("graph   pdl=%d kernels=%d ifs=%d taken=%d: %.2f us per iteration (%.2f us per node)\n", pdl, nker,
             c[1], c[2], 1e3 * ms / iters, 1e3 * ms / iters / (nker + c[1]));
      CK(cudaGraphExecDestroy(ex));
    }
  }
  // grid-wide barrier of a cooperative persistent kernel (the alternative to a graph)
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  for (int per = 1; per <= 4; per *= 2) {
    int n = 2000;
    void* args[] = {&n, &it};
    float ms = 0;
    for (int w = 0; w < 2; ++w) {
      CK(cudaEventRecord(a, s));
      CK(cudaLaunchCooperativeKernel((void*)k_gridsync, dim3(sms * per), dim3(256), args, 0, s));
      CK(cudaEventRecord(b, s));
      CK(cudaEventSynchronize(b));
    }
    CK(cudaEventElapsedTime(&ms, a, b));
    printf("grid.sync %d CTAs x 256: %.2f us per barrier\n", sms * per, 1e3 * ms / n);
  }
  return 0;
}
