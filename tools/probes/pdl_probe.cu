// Probe: cost of a dependent kernel boundary inside a replayed CUDA graph,
// with and without programmatic dependent launch (PDL).  Chain of K kernels,
// each waits on its predecessor (griddepcontrol.wait) and then does a small
// amount of work on 148 x 256 threads.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/pdl_probe tools/probes/pdl_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void step(float* x, int work) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  float v = x[blockIdx.x * blockDim.x + threadIdx.x];
  for (int i = 0; i < work; ++i) v = v * 0.999f + 1.0f;
  x[blockIdx.x * blockDim.x + threadIdx.x] = v;
  asm volatile("griddepcontrol.launch_dependents;");
}

int main() {
  float* x;
  cudaMalloc(&x, 148 * 256 * sizeof(float));
  cudaMemset(x, 0, 148 * 256 * sizeof(float));
  cudaStream_t s;
  cudaStreamCreate(&s);
  for (int work : {0, 2000}) {
    for (int pdl = 0; pdl < 2; ++pdl) {
      for (int K : {1, 40}) {
        cudaGraph_t g;
        cudaGraphExec_t ge;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
        for (int k = 0; k < K; ++k) {
          cudaLaunchConfig_t cfg = {};
          cfg.gridDim = dim3(148);
          cfg.blockDim = dim3(256);
          cfg.stream = s;
          cudaLaunchAttribute at[1];
          at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
          at[0].val.programmaticStreamSerializationAllowed = 1;
          cfg.attrs = at;
          cfg.numAttrs = pdl ? 1 : 0;
          cudaLaunchKernelEx(&cfg, step, x, work);
        }
        cudaStreamEndCapture(s, &g);
        if (cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) { printf("instantiate failed\n"); return 1; }
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
        printf("work=%d pdl=%d K=%d: %.2f us per graph, %.2f us per kernel (%s)\n", work, pdl, K,
               ms / 200 * 1000, ms / 200 * 1000 / K, cudaGetErrorString(cudaGetLastError()));
      }
    }
  }
  return 0;
}
