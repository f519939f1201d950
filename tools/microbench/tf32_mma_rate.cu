// Microbenchmark: back-to-back tcgen05.mma.kind::tf32 (cta_group::1, M=128, K=8) issue rate from one
// thread, shared-memory operands (SS: A and B K-major SWIZZLE_128B, or A MN-major 32B-atom) or A in
// TMEM (TS).  Prints cycles per MMA for N = 64 / 128 / 256.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tf32_mma_rate tf32_mma_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint64_t layout) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (layout << 61);
}
__host__ __device__ constexpr uint32_t idesc_tf32(bool a_mn, bool b_mn, int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

template <int N, int MODE>   // MODE 0: SS K/K, 1: SS A-MN/B-K, 2: TS (A in TMEM); +4: walk 12 distinct operand slices
__global__ void k(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  uint8_t* s = (uint8_t*)(((uintptr_t)sm + 1023) & ~uintptr_t(1023));
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) ((float*)s)[i] = 1.0f;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n");
  }
  asm volatile("fence.proxy.async.shared::cta;\n");
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tm = slot;
  if (threadIdx.x == 0) {
    constexpr int M3 = MODE & 3;
    constexpr bool WALK = MODE & 4;
    const uint32_t a = smem_u32(s), b = a + 32768;
    const uint32_t id = idesc_tf32(M3 == 1, false, 128, N);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      // WALK: consecutive MMAs read different 4 KB A slices (32 KB region) and 4 KB B slices (+32 KB)
      const uint32_t off = WALK ? (uint32_t)(i & 7) * 4096u : 0u;
      const uint64_t da = M3 == 1 ? sdesc(a + off, 4096, 512, 1) : sdesc(a + off, 16, 1024, 2);
      const uint64_t db = sdesc(b + (WALK ? (uint32_t)(i & 3) * 8192u : 0u), 16, 1024, 2);
      if (M3 == 2) {
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tm),
                     "r"(tm + 256u + (uint32_t)(i & 3) * 8u), "l"(db), "r"(id), "r"(1));
      } else {
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tm),
                     "l"(da), "l"(db), "r"(id), "r"(1));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&bar)));
    asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@!P1 bra W;\n}\n" ::"r"(smem_u32(&bar)));
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tm));
}

template <int N, int MODE>
void run(const char* name, int blocks) {
  long long* d;
  cudaMalloc(&d, 1024 * 8);
  cudaFuncSetAttribute(k<N, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const int iters = 4096;
  k<N, MODE><<<blocks, 128, 100 * 1024>>>(d, 16);
  k<N, MODE><<<blocks, 128, 100 * 1024>>>(d, iters);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[1024];
  cudaMemcpy(h, d, blocks * 8, cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int i = 0; i < blocks; ++i) mx = h[i] > mx ? h[i] : mx;
  printf("%-22s N=%3d blocks=%3d: %7.1f cycles/MMA  (%s)  -> %.0f tf32 MAC/clk/SM\n", name, N, blocks, mx / iters,
         cudaGetErrorString(e), 128.0 * N * 8 / (mx / iters));
  cudaFree(d);
}

int main() {
  run<64, 0>("SS K/K", 148);
  run<128, 0>("SS K/K", 148);
  run<256, 0>("SS K/K", 148);
  run<128, 1>("SS A-MN/B-K", 148);
  run<256, 1>("SS A-MN/B-K", 148);
  run<128, 2>("TS (A in TMEM)", 148);
  run<256, 2>("TS (A in TMEM)", 148);
  run<128, 4>("SS K/K walk", 148);
  run<256, 4>("SS K/K walk", 148);
  run<128, 5>("SS A-MN/B-K walk", 148);
  run<128, 6>("TS walk", 148);
  run<256, 6>("TS walk", 148);
  return 0;
}
