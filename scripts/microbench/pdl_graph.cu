// Does programmatic dependent launch survive stream capture into the body of a conditional WHILE node?
// Two kernels per trip, the second launched with programmaticStreamSerialization; prints timings with / without.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void k_a(int* buf, int n) {
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) buf[i] += 1;
}
__global__ void k_b(int* buf, int n, int* counter, cudaGraphConditionalHandle h, int trips, int use_cond) {
  asm volatile("griddepcontrol.launch_dependents;");
  __shared__ int s[32];
  s[threadIdx.x & 31] = threadIdx.x;   // prologue
  asm volatile("griddepcontrol.wait;" ::: "memory");
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) buf[i] += 2;
  if (i == 0) {
    int c = ++*counter;
    if (use_cond) cudaGraphSetConditional(h, c < trips ? 1u : 0u);
  }
}

template <class... A>
cudaError_t launch(bool pdl, void (*k)(A...), dim3 g, dim3 b, cudaStream_t s, A... a) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = g; cfg.blockDim = b; cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at; cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, a...);
}

int run(bool pdl) {
  const int n = 32 * 128, trips = 200;
  int *buf, *counter;
  CK(cudaMalloc(&buf, n * 4)); CK(cudaMalloc(&counter, 4));
  cudaStream_t s; CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaGraph_t g; cudaGraphExec_t ex; cudaGraphConditionalHandle h;
  CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  CK(cudaMemsetAsync(counter, 0, 4, s));
  cudaStreamCaptureStatus st; cudaGraph_t cg; const cudaGraphNode_t* deps; size_t nd;
  CK(cudaStreamGetCaptureInfo_v2(s, &st, nullptr, &cg, &deps, &nd));
  CK(cudaGraphConditionalHandleCreate(&h, cg, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams np = {}; np.type = cudaGraphNodeTypeConditional; np.conditional.handle = h;
  np.conditional.type = cudaGraphCondTypeWhile; np.conditional.size = 1;
  cudaGraphNode_t node; CK(cudaGraphAddNode(&node, cg, deps, nd, &np));
  cudaGraph_t body = np.conditional.phGraph_out[0];
  CK(cudaStreamUpdateCaptureDependencies(s, &node, 1, cudaStreamSetCaptureDependencies));
  CK(cudaStreamEndCapture(s, &g));
  CK(cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  CK(launch(false, k_a, dim3(32), dim3(128), s, buf, n));
  CK(launch(pdl, k_b, dim3(32), dim3(128), s, buf, n, counter, h, trips, 1));
  cudaGraph_t bo; CK(cudaStreamEndCapture(s, &bo));
  CK(cudaGraphInstantiate(&ex, g, 0));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  CK(cudaMemsetAsync(buf, 0, n * 4, s));
  for (int w = 0; w < 3; ++w) CK(cudaGraphLaunch(ex, s));
  CK(cudaMemsetAsync(buf, 0, n * 4, s));
  CK(cudaEventRecord(e0, s)); CK(cudaGraphLaunch(ex, s)); CK(cudaEventRecord(e1, s));
  CK(cudaStreamSynchronize(s));
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  int v, c; cudaMemcpy(&v, buf + 77, 4, cudaMemcpyDeviceToHost); cudaMemcpy(&c, counter, 4, cudaMemcpyDeviceToHost);
  printf("while-graph pdl=%d: %d trips in %.1f us = %.2f us per trip (2 kernels), buf=%d (expect %d)\n", pdl, c, ms * 1e3, ms * 1e3 / c, v, 3 * trips);
  // plain stream
  CK(cudaMemsetAsync(buf, 0, n * 4, s));
  CK(cudaEventRecord(e0, s));
  for (int t = 0; t < trips; ++t) {
    CK(launch(pdl, k_a, dim3(32), dim3(128), s, buf, n));
    CK(launch(pdl, k_b, dim3(32), dim3(128), s, buf, n, counter, h, trips, 0));
  }
  CK(cudaEventRecord(e1, s)); CK(cudaStreamSynchronize(s));
  cudaEventElapsedTime(&ms, e0, e1);
  cudaMemcpy(&v, buf + 77, 4, cudaMemcpyDeviceToHost);
  printf("stream      pdl=%d: %.2f us per trip, buf=%d (expect %d)\n", pdl, ms * 1e3 / trips, v, 3 * trips);
  return 0;
}
int main() { if (run(false)) return 1; if (run(true)) return 1; return 0; }
