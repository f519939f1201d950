// FP64 tensor-pipe peak microbenchmark (test/bench-only export): back-to-back independent
// DMMA.8x8x4 chains on every SM, timed with CUDA events.  MEASURED_PEAKS.json carries no FP64
// figure, so bench.py measures this denominator live on the same GPU.
#include "common.cuh"
#include "../../include/cggm_testing.h"

namespace cggm {
namespace {

__global__ void __launch_bounds__(256) k_dmma_peak(double* out, int iters) {
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    c[i][0] = threadIdx.x * 1e-9;
    c[i][1] = i * 1e-9;
  }
  const double a = 1.0000001, b = 0.9999999;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) ptx::dmma_8x8x4(c[i][0], c[i][1], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

}  // namespace
}  // namespace cggm

using namespace cggm;

extern "C" cggm_status cggm_test_fp64_peak(cggm_ctx* ctx_, double seconds, double* tflops, double* elapsed_ms) {
  if (!ctx_ || !tflops || !elapsed_ms || !(seconds > 0)) return CGGM_ERR_INVALID_ARG;
  Ctx* c = reinterpret_cast<Ctx*>(ctx_);  // cggm_ctx wraps Ctx as its only member
  double* out = nullptr;
  if (cudaMalloc(&out, 256 * 8) != cudaSuccess) return CGGM_ERR_OOM;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = c->num_sms * 2, threads = 256;
  // calibrate iterations for the requested duration
  int iters = 4096;
  float ms = 0.f;
  for (int rep = 0; rep < 6; ++rep) {
    cudaEventRecord(e0, c->stream);
    k_dmma_peak<<<blocks, threads, 0, c->stream>>>(out, iters);
    cudaEventRecord(e1, c->stream);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms >= 0.9 * seconds * 1e3) break;
    double scale = (seconds * 1e3) / (ms > 0.01 ? ms : 0.01);
    iters = (int)std::min<double>(2e9, iters * scale);
  }
  const double flops = 2.0 * 256.0 * 8.0 * (double)iters * blocks * (threads / 32);
  *tflops = flops / (ms * 1e-3) / 1e12;
  *elapsed_ms = ms;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  return cudaGetLastError() == cudaSuccess ? CGGM_OK : CGGM_ERR_CUDA;
}

// L2 -> SM read bandwidth (test/bench-only export): every SM streams 16-byte loads (4 in flight per
// thread) over a 24 MB buffer that stays in L2 after a warm-up pass, as the SpMM's gathers do; the denominator of the SpMM's L2
// roofline (its algorithmic HBM bytes are far below its gathered bytes: it is L2-bound).
namespace cggm {
namespace {
__global__ void __launch_bounds__(512) k_l2_read(const double2* __restrict__ buf, int64_t n16, int passes,
                                                 double* out) {
  // 4 independent 16-byte loads in flight per thread, contiguous per warp (512 B per load group)
  double s0 = 0.0, s1 = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * 4;
  for (int p = 0; p < passes; ++p) {
    for (int64_t i = ((int64_t)blockIdx.x * blockDim.x) * 4 + threadIdx.x; i + 3 * (int64_t)blockDim.x < n16;
         i += stride) {
      double2 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = __ldcg(buf + i + u * (int64_t)blockDim.x);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        s0 += v[u].x;
        s1 += v[u].y;
      }
    }
  }
  if (s0 + s1 == 1234.5678) out[0] = s0;
}
}  // namespace
}  // namespace cggm

extern "C" cggm_status cggm_test_l2_peak(cggm_ctx* ctx_, double seconds, double* gbs, double* elapsed_ms) {
  if (!ctx_ || !gbs || !elapsed_ms || !(seconds > 0)) return CGGM_ERR_INVALID_ARG;
  Ctx* c = reinterpret_cast<Ctx*>(ctx_);
  const int64_t bytes = 24ll << 20;   // 24 MB: resident in the 126 MB L2 (both partitions)
  void* buf = nullptr;
  double* out = nullptr;
  if (cudaMalloc(&buf, bytes) != cudaSuccess) return CGGM_ERR_OOM;
  if (cudaMalloc(&out, 64) != cudaSuccess) {
    cudaFree(buf);
    return CGGM_ERR_OOM;
  }
  cudaMemsetAsync(buf, 0, bytes, c->stream);
  const int64_t n16 = bytes / 16;
  const int blocks = c->num_sms * 4, threads = 512;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_l2_read<<<blocks, threads, 0, c->stream>>>(static_cast<const double2*>(buf), n16, 1, out);   // warm L2
  int passes = 4;
  float ms = 0.f;
  for (int rep = 0; rep < 6; ++rep) {
    cudaEventRecord(e0, c->stream);
    k_l2_read<<<blocks, threads, 0, c->stream>>>(static_cast<const double2*>(buf), n16, passes, out);
    cudaEventRecord(e1, c->stream);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms >= 0.9 * seconds * 1e3) break;
    const double scale = (seconds * 1e3) / (ms > 0.01 ? ms : 0.01);
    passes = (int)std::min<double>(1e6, passes * scale) + 1;
  }
  *gbs = (double)bytes * passes / (ms * 1e-3) / 1e9;
  *elapsed_ms = ms;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(buf);
  cudaFree(out);
  return cudaGetLastError() == cudaSuccess ? CGGM_OK : CGGM_ERR_CUDA;
}
