// Device probe: (1) CUDA-graph conditional WHILE node driven from device code,
// (2) nested conditional, (3) FP64 DFMA throughput (the per-tet kernel's compute roof),
// (4) graph kernel-node chain latency.  Run: ./probe_device
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("ERR %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

__global__ void body_kernel(int* counter, cudaGraphConditionalHandle h, int limit) {
  if (threadIdx.x == 0) {
    int c = ++(*counter);
    cudaGraphSetConditional(h, c < limit ? 1 : 0);
  }
}
__global__ void inner_kernel(int* counter, cudaGraphConditionalHandle h) {
  if (threadIdx.x == 0) {
    int c = ++counter[1];
    cudaGraphSetConditional(h, (c % 3) != 0 ? 1 : 0);
  }
}
__global__ void noop_kernel(int* p) { if (threadIdx.x == 0 && p[0] < 0) p[0] = 0; }

__global__ void dfma_kernel(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double b = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
    a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
    a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

int main() {
  cudaStream_t s; CK(cudaStreamCreate(&s));
  int* d; CK(cudaMalloc(&d, 16)); CK(cudaMemset(d, 0, 16));
  // ---- (1)+(2): outer WHILE (limit 5) containing a kernel and an inner WHILE
  cudaGraph_t g; CK(cudaGraphCreate(&g, 0));
  cudaGraphConditionalHandle ho; CK(cudaGraphConditionalHandleCreate(&ho, g, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams cp = {}; cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = ho; cp.conditional.type = cudaGraphCondTypeWhile; cp.conditional.size = 1;
  cudaGraphNode_t node; CK(cudaGraphAddNode(&node, g, nullptr, 0, &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  cudaGraphConditionalHandle hi; CK(cudaGraphConditionalHandleCreate(&hi, body, 1, cudaGraphCondAssignDefault));
  CK(cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeGlobal));
  body_kernel<<<1, 32, 0, s>>>(d, ho, 5);
  CK(cudaStreamEndCapture(s, &body));
  // inner while appended after body_kernel node
  size_t nn = 0; CK(cudaGraphGetNodes(body, nullptr, &nn));
  cudaGraphNode_t bn[8]; CK(cudaGraphGetNodes(body, bn, &nn));
  cudaGraphNodeParams ci = {}; ci.type = cudaGraphNodeTypeConditional;
  ci.conditional.handle = hi; ci.conditional.type = cudaGraphCondTypeWhile; ci.conditional.size = 1;
  cudaGraphNode_t inode; CK(cudaGraphAddNode(&inode, body, bn, nn, &ci));
  cudaGraph_t ibody = ci.conditional.phGraph_out[0];
  CK(cudaStreamBeginCaptureToGraph(s, ibody, nullptr, nullptr, 0, cudaStreamCaptureModeGlobal));
  inner_kernel<<<1, 32, 0, s>>>(d, hi);
  CK(cudaStreamEndCapture(s, &ibody));
  cudaGraphExec_t ge; CK(cudaGraphInstantiate(&ge, g, 0));
  CK(cudaGraphLaunch(ge, s)); CK(cudaStreamSynchronize(s));
  int h[2]; CK(cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost));
  printf("conditional: outer=%d (expect 5) inner=%d (expect 15)\n", h[0], h[1]);

  // ---- (4) chain of 100 noop kernel nodes in a graph
  cudaGraph_t g2; CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal));
  for (int i = 0; i < 100; ++i) noop_kernel<<<148, 128, 0, s>>>(d);
  CK(cudaStreamEndCapture(s, &g2));
  cudaGraphExec_t ge2; CK(cudaGraphInstantiate(&ge2, g2, 0));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) CK(cudaGraphLaunch(ge2, s));
  cudaEventRecord(e0, s); for (int r = 0; r < 10; ++r) cudaGraphLaunch(ge2, s); cudaEventRecord(e1, s);
  CK(cudaStreamSynchronize(s)); float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("graph kernel-node chain: %.3f us per node\n", ms * 1000.0 / 1000.0);
  cudaEventRecord(e0, s); for (int r = 0; r < 1000; ++r) noop_kernel<<<148, 128, 0, s>>>(d); cudaEventRecord(e1, s);
  CK(cudaStreamSynchronize(s)); cudaEventElapsedTime(&ms, e0, e1);
  printf("stream launches: %.3f us per kernel\n", ms * 1000.0 / 1000.0);

  // ---- (3) DFMA throughput
  double* o; CK(cudaMalloc(&o, 148 * 8 * 256 * 8));
  int iters = 20000;
  dfma_kernel<<<148 * 8, 256, 0, s>>>(o, 100);
  cudaEventRecord(e0, s); dfma_kernel<<<148 * 8, 256, 0, s>>>(o, iters); cudaEventRecord(e1, s);
  CK(cudaStreamSynchronize(s)); cudaEventElapsedTime(&ms, e0, e1);
  double flops = 2.0 * 8 * iters * 148.0 * 8 * 256;
  printf("fp64 fma: %.2f TFLOP/s\n", flops / (ms * 1e-3) / 1e12);
  int dev; cudaGetDevice(&dev); cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  printf("device %s sms=%d l2=%d MB smem/block optin=%zu\n", p.name, p.multiProcessorCount, p.l2CacheSize >> 20, p.sharedMemPerBlockOptin);
  return 0;
}
