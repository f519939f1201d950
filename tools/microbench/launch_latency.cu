// Launch-to-launch latency of dependent tiny kernels on one stream (B200): plain stream launches,
// the same chain captured in a CUDA graph, and with programmatic dependent launch (PDL).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_tiny(double* p, int n) {
  // one small dependent step: read, modify, write (like a chain of small GEMM tiles)
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = p[i] * 1.0000001 + 1.0;
}

__global__ void k_tiny_pdl(double* p, int n) {
  cudaGridDependencySynchronize();
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = p[i] * 1.0000001 + 1.0;
  cudaTriggerProgrammaticLaunchCompletion();
}

int main() {
  double* p;
  cudaMalloc(&p, 1 << 20);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int N = 2000;
  for (int blocks : {1, 4, 64}) {
    float ms;
    for (int w = 0; w < 2; ++w) {
      cudaEventRecord(e0, s);
      for (int i = 0; i < N; ++i) k_tiny<<<blocks, 128, 0, s>>>(p, blocks * 128);
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
    }
    cudaEventElapsedTime(&ms, e0, e1);
    printf("blocks=%d stream launches: %.2f us/kernel\n", blocks, 1000.f * ms / N);
    // graph
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    for (int i = 0; i < N; ++i) k_tiny<<<blocks, 128, 0, s>>>(p, blocks * 128);
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    for (int w = 0; w < 2; ++w) {
      cudaEventRecord(e0, s);
      cudaGraphLaunch(ge, s);
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
    }
    cudaEventElapsedTime(&ms, e0, e1);
    printf("blocks=%d graph: %.2f us/kernel\n", blocks, 1000.f * ms / N);
    // PDL
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = blocks;
    cfg.blockDim = 128;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    for (int w = 0; w < 2; ++w) {
      cudaEventRecord(e0, s);
      for (int i = 0; i < N; ++i) cudaLaunchKernelEx(&cfg, k_tiny_pdl, p, blocks * 128);
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
    }
    cudaEventElapsedTime(&ms, e0, e1);
    printf("blocks=%d PDL stream: %.2f us/kernel\n", blocks, 1000.f * ms / N);
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    for (int i = 0; i < N; ++i) cudaLaunchKernelEx(&cfg, k_tiny_pdl, p, blocks * 128);
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    for (int w = 0; w < 2; ++w) {
      cudaEventRecord(e0, s);
      cudaGraphLaunch(ge, s);
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
    }
    cudaEventElapsedTime(&ms, e0, e1);
    printf("blocks=%d PDL graph: %.2f us/kernel\n", blocks, 1000.f * ms / N);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
