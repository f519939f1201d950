// Dependent-chain latencies (cycles) of FP64 operations on one warp: DFMA, DMUL, rsqrt(double),
// sqrt(double), 1/x, LDS.64 + DFMA, shuffle of a double.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_lat(double* out, long long* cyc, double seed) {
  __shared__ double sm[64];
  const int lane = threadIdx.x;
  sm[lane] = seed + lane;
  sm[lane + 32] = seed - lane;
  __syncwarp();
  double x = seed + lane * 1e-3, y = 1.0000001;
  long long t0, t1;
  const int N = 256;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; ++i) x = fma(x, y, 1e-9);
  t1 = clock64();
  if (lane == 0) cyc[0] = (t1 - t0) / N;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; ++i) x = rsqrt(x + 1.0);
  t1 = clock64();
  if (lane == 0) cyc[1] = (t1 - t0) / N;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; ++i) x = sqrt(x + 1.0);
  t1 = clock64();
  if (lane == 0) cyc[2] = (t1 - t0) / N;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; ++i) x = 1.0 / (x + 1.0);
  t1 = clock64();
  if (lane == 0) cyc[3] = (t1 - t0) / N;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; ++i) x = fma(sm[(i + (x > 1e300)) & 63], x, 1e-9);
  t1 = clock64();
  if (lane == 0) cyc[4] = (t1 - t0) / N;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; ++i) x = __shfl_sync(0xffffffffu, x, (lane + 1) & 31) * y;
  t1 = clock64();
  if (lane == 0) cyc[5] = (t1 - t0) / N;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; ++i) x = x * y;
  t1 = clock64();
  if (lane == 0) cyc[6] = (t1 - t0) / N;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; ++i) { double r = __drcp_rn(x + 1.0); x = r; }
  t1 = clock64();
  if (lane == 0) cyc[7] = (t1 - t0) / N;
  out[lane] = x;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 32 * 8);
  cudaMallocManaged(&cyc, 16 * 8);
  for (int r = 0; r < 2; ++r) k_lat<<<1, 32>>>(out, cyc, 1.5);
  cudaDeviceSynchronize();
  printf("cycles per dependent op: DFMA %lld  rsqrt(d) %lld  sqrt(d) %lld  1/x %lld  LDS+DFMA %lld  SHFL+DMUL %lld  "
         "DMUL %lld  drcp_rn %lld\n", cyc[0], cyc[1], cyc[2], cyc[3], cyc[4], cyc[5], cyc[6], cyc[7]);
  return 0;
}
