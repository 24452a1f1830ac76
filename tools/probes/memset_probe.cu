// Probe: cost of memset nodes vs tiny kernel nodes in a replayed CUDA graph
// (the Stage-1 iteration has ~9 cudaMemsetAsync nodes).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/memset_probe tools/probes/memset_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void tiny(float* x) { x[threadIdx.x] += 1.f; }

int main() {
  float* x;
  cudaMalloc(&x, 64 << 20);
  cudaStream_t s;
  cudaStreamCreate(&s);
  for (int kind = 0; kind < 3; ++kind) {
    for (int K : {1, 20}) {
      cudaGraph_t g;
      cudaGraphExec_t ge;
      cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
      for (int k = 0; k < K; ++k) {
        if (kind == 0) cudaMemsetAsync(x + k * 64, 0, 256, s);                 // small memset
        else if (kind == 1) cudaMemsetAsync(x, 0, 12 << 20, s);                // 12 MB memset
        else tiny<<<1, 32, 0, s>>>(x + k * 64);                                // tiny kernel
      }
      cudaStreamEndCapture(s, &g);
      cudaGraphInstantiate(&ge, g, 0);
      for (int i = 0; i < 10; ++i) cudaGraphLaunch(ge, s);
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0, s);
      for (int i = 0; i < 200; ++i) cudaGraphLaunch(ge, s);
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("%s K=%d: %.2f us per graph, %.2f us per node\n",
             kind == 0 ? "memset 256 B" : kind == 1 ? "memset 12 MB" : "tiny kernel", K,
             ms / 200 * 1000, ms / 200 * 1000 / K);
    }
  }
  return 0;
}
