// cond_nested.cu -- can a kernel inside an IF body set the handle of a conditional node of
// the enclosing (parent) graph?  Prints the IF-node outcomes for both placements.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/cond_nested tools/cond_nested.cu
#include <cuda_runtime.h>
#include <stdio.h>

#define CK(x)                                                                    \
  do {                                                                           \
    cudaError_t e_ = (x);                                                        \
    if (e_ != cudaSuccess) {                                                     \
      printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      return 1;                                                                  \
    }                                                                            \
  } while (0)

__global__ void k_set(cudaGraphConditionalHandle h, unsigned v) {
  if (threadIdx.x == 0) cudaGraphSetConditional(h, v);
}
__global__ void k_mark(int* out, int i) {
  if (threadIdx.x == 0) out[i] += 1;
}

static cudaError_t add_if(cudaStream_t s, cudaGraphConditionalHandle h, cudaGraph_t* body) {
  cudaStreamCaptureStatus st;
  cudaGraph_t g;
  const cudaGraphNode_t* deps;
  size_t nd;
  cudaError_t e = cudaStreamGetCaptureInfo(s, &st, nullptr, &g, &deps, &nd);
  if (e) return e;
  cudaGraphNodeParams p = {};
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = h;
  p.conditional.type = cudaGraphCondTypeIf;
  p.conditional.size = 1;
  cudaGraphNode_t n;
  if ((e = cudaGraphAddNode(&n, g, deps, nd, &p))) return e;
  if ((e = cudaStreamUpdateCaptureDependencies(s, &n, 1, cudaStreamSetCaptureDependencies))) return e;
  *body = p.conditional.phGraph_out[0];
  return cudaSuccess;
}

int main() {
  cudaStream_t s0, s1, s2;
  CK(cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  int* out;
  CK(cudaMalloc(&out, 16));
  CK(cudaMemset(out, 0, 16));
  cudaGraph_t g;
  CK(cudaGraphCreate(&g, 0));
  CK(cudaStreamBeginCaptureToGraph(s0, g, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  cudaGraphConditionalHandle h1, h2;
  CK(cudaGraphConditionalHandleCreate(&h1, g, 0, cudaGraphCondAssignDefault));
  CK(cudaGraphConditionalHandleCreate(&h2, g, 0, cudaGraphCondAssignDefault));
  k_set<<<1, 32, 0, s0>>>(h1, 1);
  cudaGraph_t b1;
  CK(add_if(s0, h1, &b1));
  CK(cudaStreamBeginCaptureToGraph(s1, b1, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  k_mark<<<1, 32, 0, s1>>>(out, 0);
  k_set<<<1, 32, 0, s1>>>(h2, 1);  // parent's handle from inside the IF body
  cudaGraph_t o1;
  CK(cudaStreamEndCapture(s1, &o1));
  cudaGraph_t b2;
  CK(add_if(s0, h2, &b2));
  CK(cudaStreamBeginCaptureToGraph(s2, b2, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  k_mark<<<1, 32, 0, s2>>>(out, 1);
  cudaGraph_t o2;
  CK(cudaStreamEndCapture(s2, &o2));
  cudaGraph_t o;
  CK(cudaStreamEndCapture(s0, &o));
  cudaGraphExec_t ex;
  cudaError_t e = cudaGraphInstantiate(&ex, g, 0);
  printf("instantiate: %s\n", cudaGetErrorString(e));
  if (e) return 0;
  CK(cudaGraphLaunch(ex, s0));
  e = cudaStreamSynchronize(s0);
  printf("run: %s\n", cudaGetErrorString(e));
  int h[2] = {0, 0};
  cudaMemcpy(h, out, 8, cudaMemcpyDeviceToHost);
  printf("IF1 body ran %d, IF2 (handle set inside IF1 body) ran %d\n", h[0], h[1]);
  return 0;
}
