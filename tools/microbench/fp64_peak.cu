// FP64 peak microbenchmark for sm_100a: DMMA (mma.sync m8n8k4 f64) vs DFMA.
// Used to establish the FP64 roofline denominator (MEASURED_PEAKS.json has none).
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

template <int CHAINS>
__global__ void k_dmma(double* out, int iters, double a, double b) {
  double c[CHAINS][2];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) { c[i][0] = threadIdx.x * 1e-9; c[i][1] = i * 1e-9; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) dmma(c[i][0], c[i][1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template <int CHAINS>
__global__ void k_dfma(double* out, int iters, double a, double b) {
  double c[CHAINS];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) c[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) c[i] = fma(c[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

// fragment layout check: A 8x4 row-major, B 4x8 col-major, C 8x8
__global__ void k_layout(const double* A, const double* B, double* C) {
  int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  double a = A[g * 4 + t];          // A[m=g][k=t]
  double b = B[t + 4 * g];          // B[k=t][n=g] (col-major 4x8)
  double c0 = 0, c1 = 0;
  dmma(c0, c1, a, b);
  C[g * 8 + 2 * t] = c0;            // C[m=g][n=2t]
  C[g * 8 + 2 * t + 1] = c1;
}

int main() {
  int dev = 0; cudaDeviceProp pr; CK(cudaGetDeviceProperties(&pr, dev));
  printf("device %s SMs %d cc %d.%d\n", pr.name, pr.multiProcessorCount, pr.major, pr.minor);
  double* out; CK(cudaMalloc(&out, 1 << 20));
  // layout check
  double hA[32], hB[32], hC[64], ref[64];
  for (int i = 0; i < 32; ++i) { hA[i] = i + 1; hB[i] = (i * 7 % 11) - 5; }
  for (int m = 0; m < 8; ++m) for (int n = 0; n < 8; ++n) { double s = 0; for (int k = 0; k < 4; ++k) s += hA[m * 4 + k] * hB[k + 4 * n]; ref[m * 8 + n] = s; }
  double *dA, *dB, *dC; CK(cudaMalloc(&dA, 256)); CK(cudaMalloc(&dB, 256)); CK(cudaMalloc(&dC, 512));
  CK(cudaMemcpy(dA, hA, 256, cudaMemcpyHostToDevice)); CK(cudaMemcpy(dB, hB, 256, cudaMemcpyHostToDevice));
  k_layout<<<1, 32>>>(dA, dB, dC); CK(cudaMemcpy(hC, dC, 512, cudaMemcpyDeviceToHost));
  int bad = 0; for (int i = 0; i < 64; ++i) bad += hC[i] != ref[i];
  printf("layout check mismatches: %d\n", bad);

  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  int sms = pr.multiProcessorCount;
  for (int wpb : {4, 8, 16}) for (int bps : {1, 2}) {
    int iters = 4096; int blocks = sms * bps; int threads = 32 * wpb;
    k_dmma<8><<<blocks, threads>>>(out, 16, 1.0000001, 0.9999999);
    CK(cudaEventRecord(e0));
    k_dmma<8><<<blocks, threads>>>(out, iters, 1.0000001, 0.9999999);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    double flops = 2.0 * 256 * 8 * (double)iters * blocks * wpb;
    printf("DMMA m8n8k4 chains=8 warps/blk=%d blk/SM=%d: %.2f TFLOP/s (%.3f ms)\n", wpb, bps, flops / ms / 1e9, ms);
  }
  for (int wpb : {8, 16, 32}) for (int bps : {1, 2}) {
    int iters = 8192; int blocks = sms * bps; int threads = 32 * wpb;
    k_dfma<8><<<blocks, threads>>>(out, 16, 1.0000001, 1e-12);
    CK(cudaEventRecord(e0));
    k_dfma<8><<<blocks, threads>>>(out, iters, 1.0000001, 1e-12);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    double flops = 2.0 * 8 * (double)iters * blocks * threads;
    printf("DFMA chains=8 warps/blk=%d blk/SM=%d: %.2f TFLOP/s (%.3f ms)\n", wpb, bps, flops / ms / 1e9, ms);
  }
  // sustained DMMA for ~2 s to see power-capped clocks
  {
    int blocks = sms * 2, threads = 256, iters = 200000;
    CK(cudaEventRecord(e0));
    k_dmma<8><<<blocks, threads>>>(out, iters, 1.0000001, 0.9999999);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    double flops = 2.0 * 256 * 8 * (double)iters * blocks * 8;
    printf("DMMA sustained: %.2f TFLOP/s over %.1f ms\n", flops / ms / 1e9, ms);
  }
  return 0;
}
