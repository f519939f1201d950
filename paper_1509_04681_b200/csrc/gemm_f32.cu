// FP32 variant of the GEMM engine (reading A18: fp32 inputs, fp32 accumulation).  FP64 DMMA has no
// fp32 counterpart short of TF32 (10-bit mantissa, too inexact for the 1e-4 contract), so the
// consumers are SIMT FFMA: CTA tile 128x128, 256 threads with an 8x8 register tile each, fed by the
// same TMA (SWIZZLE_128B) -> shared-memory ring with mbarrier full/empty pipeline, thread 0
// producing STAGES-1 k-tiles (32 floats) ahead.  Thread -> row maps are chosen per operand layout
// so that every ld.shared.v4 quarter-warp hits 8 distinct 16-byte chunks:
//   MN-inner operand: x = 4*tx + 64*h + i   (two 16-byte chunks of 4 consecutive x per k)
//   K-inner  operand: x = tx + 16*r         (one 16-byte chunk = 4 consecutive k per row)
// Same flags (triangular k-ranges, lower trapezoid / mirror), tile order and epilogue as gemm.cu.
#include "common.cuh"

namespace cggm {
namespace {

constexpr int FBK = 32;
constexpr int FSTAGES = 4;
constexpr int FBM = 128, FBN = 128;
constexpr int FNT = 256;
constexpr int F_OP_BYTES = FBM * FBK * 4;   // 16 KB
constexpr int F_STAGE = 2 * F_OP_BYTES;
constexpr int F_EPI_LD = FBM + 1;
constexpr int F_EPI_BYTES = FBN * F_EPI_LD * 4;
constexpr int F_MAIN = FSTAGES * F_STAGE;
constexpr int F_DATA = F_MAIN > F_EPI_BYTES ? F_MAIN : F_EPI_BYTES;
constexpr int F_SMEM = F_DATA + 1024 + 2 * FSTAGES * 8;
constexpr int GROUP_N = 8;

struct KParamsF {
  int M, N, K;
  int tilesM, tilesN;
  int flags;
  int a3d, b3d;
  EpilogueT<float> epi;
};

__device__ __forceinline__ void tile_coords_f(const KParamsF& P, int t, int& I, int& J) {
  if (P.flags & SYM_LOWER) {
    const long long tri = (long long)P.tilesN * (P.tilesN + 1) / 2;
    if (t < tri) {
      int i = (int)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
      while ((long long)(i + 1) * (i + 2) / 2 <= t) ++i;
      while ((long long)i * (i + 1) / 2 > t) --i;
      I = i;
      J = t - (int)((long long)i * (i + 1) / 2);
    } else {
      const int r = t - (int)tri;
      I = P.tilesN + r / P.tilesN;
      J = r % P.tilesN;
    }
    return;
  }
  const int per_group = GROUP_N * P.tilesM;
  const int gi = t / per_group;
  const int local = t - gi * per_group;
  const int nb0 = gi * GROUP_N;
  const int width = min(GROUP_N, P.tilesN - nb0);
  I = local / width;
  J = nb0 + local % width;
  if (P.flags & B_KLE_N) J = P.tilesN - 1 - J;
  if (P.flags & A_KLE_M) I = P.tilesM - 1 - I;
}

__device__ __forceinline__ void epi_apply_f(const EpilogueT<float>& E, int64_t r, int64_t c, float v) {
  if (E.out1) {
    float o = __fmul_rn((float)E.a1, v);
    if (E.in1a) o = __fadd_rn(o, __fmul_rn((float)E.b1, E.in1a[r + c * E.ld1a]));
    if (E.in1b) o = __fadd_rn(o, __fmul_rn((float)E.c1, E.in1b[r + c * E.ld1b]));
    E.out1[r + c * E.ld1] = o;
  }
  if (E.out2) {
    float o = __fmul_rn((float)E.a2, v);
    if (E.in2a) o = __fadd_rn(o, __fmul_rn((float)E.b2, E.in2a[r + c * E.ld2a]));
    if (E.in2b) o = __fadd_rn(o, __fmul_rn((float)E.c2, E.in2b[r + c * E.ld2b]));
    E.out2[r + c * E.ld2] = o;
  }
}

__device__ __forceinline__ void epi_mirror_f(const EpilogueT<float>& E, int64_t r, int64_t c, float v) {
  if (E.mir1) E.mir1[r + c * E.ld1] = __fmul_rn((float)E.a1, v);
  else epi_apply_f(E, r, c, v);
}

template <bool KINNER>
__device__ __forceinline__ int fx(int tx, int r) {
  return KINNER ? tx + 16 * r : 4 * tx + 64 * (r >> 2) + (r & 3);
}

__device__ __forceinline__ void lds_v4(float (&v)[4], uint32_t addr) {
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];\n" : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]) : "r"(addr));
}

// operand tile loads for one group of 4 k (k4 = 0..7 inside the 32-wide k tile) into v[k][8]
template <bool KINNER>
__device__ __forceinline__ void load_group(float (&v)[4][8], uint32_t base, int tx, int k4) {
  if (KINNER) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const int x = tx + 16 * r;
      const int chunk = k4 ^ (x & 7);
      float q[4];
      lds_v4(q, base + x * 128 + chunk * 16);
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) v[kk][r] = q[kk];
    }
  } else {
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      const int k = 4 * k4 + kk;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int x0 = 4 * tx + 64 * h;
        const int xb = x0 >> 5;
        const int chunk = ((x0 & 31) >> 2) ^ (k & 7);
        float q[4];
        lds_v4(q, base + xb * 4096 + k * 128 + chunk * 16);
#pragma unroll
        for (int i = 0; i < 4; ++i) v[kk][4 * h + i] = q[i];
      }
    }
  }
}

template <bool AK, bool BKI>
__global__ void __launch_bounds__(FNT, 1)
    gemm_ffma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const KParamsF P) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + F_DATA);
  uint64_t* empty = full + FSTAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int I, J;
  tile_coords_f(P, blockIdx.x, I, J);
  const int m0 = I * FBM, n0 = J * FBN;
  int kbeg = 0, kend = P.K;
  if (P.flags & A_KGE_M) kbeg = max(kbeg, m0);
  if (P.flags & B_KGE_N) kbeg = max(kbeg, n0);
  if (P.flags & A_KLE_M) kend = min(kend, m0 + FBM);
  if (P.flags & B_KLE_N) kend = min(kend, n0 + FBN);
  const int kt0 = kbeg / FBK;
  const int nkt = kend > kbeg ? (kend - kt0 * FBK + FBK - 1) / FBK : 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < FSTAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], FNT / 32);
    }
    ptx::fence_barrier_init();
  }
  __syncthreads();
  int a_boxes = 0, b_boxes = 0;
  if (!AK)
    for (int xb = 0; xb < FBM / 32; ++xb) a_boxes += (m0 + xb * 32 < P.M);
  if (!BKI)
    for (int xb = 0; xb < FBN / 32; ++xb) b_boxes += (n0 + xb * 32 < P.N);
  const uint32_t tx_bytes =
      ((AK || P.a3d) ? F_OP_BYTES : a_boxes * 4096) + ((BKI || P.b3d) ? F_OP_BYTES : b_boxes * 4096);
  auto issue = [&](int i) {
    const int s = i % FSTAGES;
    uint8_t* sa = smem + s * F_STAGE;
    uint8_t* sb = sa + F_OP_BYTES;
    ptx::mbar_arrive_expect_tx(&full[s], tx_bytes);
    const int k = (kt0 + i) * FBK;
    if (AK) ptx::tma_load_2d(sa, &tmA, &full[s], k, m0);
    else if (P.a3d) ptx::tma_load_3d(sa, &tmA, &full[s], 0, k, m0 / 32);
    else
      for (int xb = 0; xb < a_boxes; ++xb) ptx::tma_load_2d(sa + xb * 4096, &tmA, &full[s], m0 + xb * 32, k);
    if (BKI) ptx::tma_load_2d(sb, &tmB, &full[s], k, n0);
    else if (P.b3d) ptx::tma_load_3d(sb, &tmB, &full[s], 0, k, n0 / 32);
    else
      for (int xb = 0; xb < b_boxes; ++xb) ptx::tma_load_2d(sb + xb * 4096, &tmB, &full[s], n0 + xb * 32, k);
  };
  if (threadIdx.x == 0) {
    if (nkt > 0) {
      ptx::prefetch_tmap(&tmA);
      ptx::prefetch_tmap(&tmB);
    }
    for (int i = 0; i < FSTAGES - 1 && i < nkt; ++i) issue(i);
  }
  const int tm = threadIdx.x & 15, tn = threadIdx.x >> 4;
  float acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
  for (int it = 0; it < nkt; ++it) {
    const int s = it % FSTAGES;
    ptx::mbar_wait(&full[s], (it / FSTAGES) & 1);
    const uint32_t sa = ptx::smem_u32(smem + s * F_STAGE);
    const uint32_t sb = sa + F_OP_BYTES;
#pragma unroll 2
    for (int k4 = 0; k4 < FBK / 4; ++k4) {
      float a[4][8], b[4][8];
      load_group<AK>(a, sa, tm, k4);
      load_group<BKI>(b, sb, tn, k4);
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[kk][i], b[kk][j], acc[i][j]);
    }
    __syncwarp();
    ptx::fence_proxy_async();   // generic reads of the stage ordered before its TMA refill (gemm.cu)
    if (lane == 0) ptx::mbar_arrive(&empty[s]);
    if (threadIdx.x == 0) {
      const int jn = it + FSTAGES - 1;
      if (jn < nkt) {
        if (jn >= FSTAGES) ptx::mbar_wait(&empty[jn % FSTAGES], ((jn / FSTAGES) & 1) ^ 1);
        issue(jn);
      }
    }
  }
  (void)warp;
  __syncthreads();
  float* Cs = reinterpret_cast<float*>(smem);
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) Cs[fx<BKI>(tn, j) * F_EPI_LD + fx<AK>(tm, i)] = acc[i][j];
  __syncthreads();
  const bool diag = (P.flags & SYM_LOWER) && I == J;
  for (int idx = threadIdx.x; idx < FBM * FBN; idx += FNT) {
    const int ml = idx % FBM, nl = idx / FBM;
    const int m = m0 + ml, n = n0 + nl;
    if (m >= P.M || n >= P.N) continue;
    if (diag && m < n) continue;
    epi_apply_f(P.epi, m, n, Cs[nl * F_EPI_LD + ml]);
  }
  if (P.flags & SYM_MIRROR) {
    for (int idx = threadIdx.x; idx < FBM * FBN; idx += FNT) {
      const int nl = idx % FBN, ml = idx / FBN;
      const int m = m0 + ml, n = n0 + nl;
      if (m >= P.M || n >= P.N) continue;
      if (diag && m <= n) continue;
      epi_mirror_f(P.epi, n, m, Cs[nl * F_EPI_LD + ml]);
    }
  }
}

CUtensorMap make_map_f(Ctx* c, const float* ptr, int64_t ld, int64_t inner, int64_t outer, uint32_t box_inner,
                       uint32_t box_outer) {
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 4)};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = c->encode_tiled(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(ptr), dims, strides, box,
                               estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError{CGGM_ERR_CUDA, "cuTensorMapEncodeTiled (f32) failed (" + std::to_string((int)r) + ")"};
  return m;
}

CUtensorMap make_map_f_mn3d(Ctx* c, const float* ptr, int64_t ld, int64_t X, int64_t K) {
  CUtensorMap m;
  cuuint64_t dims[3] = {32, (cuuint64_t)K, (cuuint64_t)(X / 32)};
  cuuint64_t strides[2] = {(cuuint64_t)(ld * 4), 128};
  cuuint32_t box[3] = {32, FBK, FBM / 32};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = c->encode_tiled(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(ptr), dims, strides, box,
                               estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError{CGGM_ERR_CUDA, "cuTensorMapEncodeTiled (f32 3d) failed (" + std::to_string((int)r) + ")"};
  return m;
}

// ------------------------------------------------------------------ small-shape FP32 GEMM
// The FP32 counterpart of gemm.cu's gemm_small_async_kernel, with the same routing: K <= 256 with
// min(M, N) <= 128 (the bottom of the Cholesky recursion) and mid-size products whose 64-tile grid
// is smaller than the SM count with K <= small_kmax.  Latency-bound work: 32x32 CTA tiles (16x the
// CTAs of the 128x128 engines), 128 threads with a 2x4 FFMA register tile each (rows mi, mi+16;
// columns nj, nj+8, nj+16, nj+24), the whole k-range of a CTA streamed through a 4-stage cp.async
// ring of 16-byte chunks (no tensor-map fetch, no mbarrier prologue, no TMEM set-up).  Shared tiles
// keep each operand's global contiguity.  fp32 accumulation in k order, like the FFMA engine.
constexpr int SF_T = 32, SF_KC = 32, SF_LD = SF_T + 4, SF_STAGES = 4;
constexpr int SF_TILE = SF_T * SF_LD;                   // floats per operand tile
constexpr int SF_SMEM = SF_STAGES * 2 * SF_TILE * 4;   // 36 KB

struct KParamsSF {
  int M, N, K, flags;
  EpilogueT<float> epi;
};

template <bool TA, bool TB>
__global__ void __launch_bounds__(128) gemm_small_f32_kernel(const float* __restrict__ A, int64_t lda,
                                                              const float* __restrict__ B, int64_t ldb,
                                                              const KParamsSF P) {
  extern __shared__ __align__(16) float sf_smem[];
  const int m0 = blockIdx.y * SF_T, n0 = blockIdx.x * SF_T;
  if ((P.flags & SYM_LOWER) && m0 + SF_T - 1 < n0) return;   // tile strictly above the diagonal
  int kbeg = 0, kend = P.K;
  if (P.flags & A_KGE_M) kbeg = max(kbeg, m0);
  if (P.flags & B_KGE_N) kbeg = max(kbeg, n0);
  if (P.flags & A_KLE_M) kend = min(kend, m0 + SF_T);
  if (P.flags & B_KLE_N) kend = min(kend, n0 + SF_T);
  const int tid = threadIdx.x, mi = tid & 15, nj = tid >> 4;
  const int nchunks = kend > kbeg ? (kend - kbeg + SF_KC - 1) / SF_KC : 0;
  // chunk -> stage: A tile [k][m] (!TA, m contiguous) or [m][k] (TA); B tile [k][n] (TB) or [n][k];
  // elements past kend / M / N are zero-filled by the copy's byte count
  auto issue = [&](int chunk) {
    const int kc = kbeg + chunk * SF_KC;
    float* as = sf_smem + (chunk % SF_STAGES) * 2 * SF_TILE;
    float* bs = as + SF_TILE;
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int pidx = tid + 128 * u, row = pidx >> 3, c4 = 4 * (pidx & 7);
      {
        const int k = TA ? kc + c4 : kc + row, m = TA ? m0 + row : m0 + c4;
        int bytes;
        if (TA) bytes = (m < P.M) ? min(max(kend - k, 0), 4) * 4 : 0;
        else bytes = (k < kend) ? min(max(P.M - m, 0), 4) * 4 : 0;
        const float* src = bytes ? (TA ? A + k + (int64_t)m * lda : A + m + (int64_t)k * lda) : A;
        ptx::cp_async16(as + row * SF_LD + c4, src, bytes);
      }
      {
        const int k = TB ? kc + row : kc + c4, n = TB ? n0 + c4 : n0 + row;
        int bytes;
        if (TB) bytes = (k < kend) ? min(max(P.N - n, 0), 4) * 4 : 0;
        else bytes = (n < P.N) ? min(max(kend - k, 0), 4) * 4 : 0;
        const float* src = bytes ? (TB ? B + n + (int64_t)k * ldb : B + k + (int64_t)n * ldb) : B;
        ptx::cp_async16(bs + row * SF_LD + c4, src, bytes);
      }
    }
  };
#pragma unroll
  for (int s = 0; s < SF_STAGES - 1; ++s) {
    if (s < nchunks) issue(s);
    ptx::cp_async_commit();
  }
  float acc[2][4];
#pragma unroll
  for (int f = 0; f < 2; ++f)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[f][j] = 0.f;
  for (int i = 0; i < nchunks; ++i) {
    ptx::cp_async_wait<SF_STAGES - 2>();
    __syncthreads();   // chunk i landed for every thread; stage (i-1) % S is free
    if (i + SF_STAGES - 1 < nchunks) issue(i + SF_STAGES - 1);
    ptx::cp_async_commit();
    const float* as = sf_smem + (i % SF_STAGES) * 2 * SF_TILE;
    const float* bs = as + SF_TILE;
#pragma unroll 8
    for (int k = 0; k < SF_KC; ++k) {
      float a[2], b[4];
#pragma unroll
      for (int f = 0; f < 2; ++f) a[f] = TA ? as[(mi + 16 * f) * SF_LD + k] : as[k * SF_LD + mi + 16 * f];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = TB ? bs[k * SF_LD + nj + 8 * j] : bs[(nj + 8 * j) * SF_LD + k];
#pragma unroll
      for (int f = 0; f < 2; ++f)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[f][j] = fmaf(a[f], b[j], acc[f][j]);
    }
  }
  ptx::cp_async_wait<0>();
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int f = 0; f < 2; ++f) {
      const int m = m0 + mi + 16 * f, n = n0 + nj + 8 * j;
      if (m >= P.M || n >= P.N) continue;
      if ((P.flags & SYM_LOWER) && m < n) continue;
      epi_apply_f(P.epi, m, n, acc[f][j]);
      if ((P.flags & SYM_MIRROR) && (m > n || P.epi.mir1)) epi_mirror_f(P.epi, n, m, acc[f][j]);
    }
}

template <bool TA, bool TB>
void launch_small_f(Ctx* c, const float* A, int64_t lda, const float* B, int64_t ldb, const KParamsSF& P) {
  dim3 grid((unsigned)((P.N + SF_T - 1) / SF_T), (unsigned)((P.M + SF_T - 1) / SF_T));
  Prof pr(c, c->cur_tag);
  gemm_small_f32_kernel<TA, TB><<<grid, 128, SF_SMEM, c->stream>>>(A, lda, B, ldb, P);
  post_launch(c, "gemm_small_f32_kernel");
}

template <bool AK, bool BKI>
void launch_f(Ctx* c, const CUtensorMap& ma, const CUtensorMap& mb, const KParamsF& P, int grid) {
  CGGM_ONCE_PER_DEVICE({
    CGGM_CUDA_CHECK(cudaFuncSetAttribute(gemm_ffma_kernel<AK, BKI>, cudaFuncAttributeMaxDynamicSharedMemorySize, F_SMEM));
  });
  Prof pr(c, c->cur_tag);
  gemm_ffma_kernel<AK, BKI><<<grid, FNT, F_SMEM, c->stream>>>(ma, mb, P);
  post_launch(c, "gemm_ffma_kernel");
}

bool tma_ok_f(const float* p, int64_t ld) { return (reinterpret_cast<uintptr_t>(p) % 16 == 0) && (ld % 4 == 0); }

}  // namespace

void gemm(Ctx* c, bool transA, bool transB, int64_t M, int64_t N, int64_t K, const float* A, int64_t lda,
          const float* B, int64_t ldb, const EpilogueT<float>& epi, int flags) {
  if (M <= 0 || N <= 0) return;
  if (M > (1LL << 30) || N > (1LL << 30) || K > (1LL << 30))
    throw CudaError{CGGM_ERR_UNSUPPORTED, "gemm dimension too large"};
  if ((flags & SYM_LOWER) && (M < N || ((flags & SYM_MIRROR) && M != N)))
    throw CudaError{CGGM_ERR_SHAPE, "SYM_LOWER gemm needs M >= N (M == N with SYM_MIRROR)"};
  if (epi.mir1 && (!(flags & SYM_MIRROR) || (flags & (SYM_LOWER | SPLIT_K2)) || !epi.out1 || epi.out2 || epi.in1a ||
                   epi.in1b))
    throw CudaError{CGGM_ERR_UNSUPPORTED, "mir1: SYM_MIRROR without SYM_LOWER, plain out1 only"};
  if (!(flags & SYM_LOWER) && (flags & SYM_MIRROR) && !epi.mir1)
    throw CudaError{CGGM_ERR_UNSUPPORTED, "SYM_MIRROR without SYM_LOWER needs mir1"};
  {  // small shapes and mid-size products with a sub-wave 64-tile grid: the 32x32 cp.async kernel
    // (an output aliasing an operand -- an in-place B := B X^T with N <= 64 -- needs one CTA per
    // row panel, which only the 128-wide kernels guarantee)
    const bool aliased = epi.out1 == A || epi.out1 == B || (epi.out2 && (epi.out2 == A || epi.out2 == B));
    const int64_t tiles64 = ((M + 63) / 64) * ((N + 63) / 64);
    const bool small_shape = K <= 256 && (M <= 128 || N <= 128);
    const bool mid_shape = K <= c->small_kmax && tiles64 < c->num_sms;
    const bool aligned = tma_ok_f(A, lda) && tma_ok_f(B, ldb);
    if ((small_shape || mid_shape) && K > 0 && aligned && !aliased && !c->no_small_async && c->force_tile != 1 &&
        c->force_tile != 2) {
      KParamsSF S;
      S.M = (int)M; S.N = (int)N; S.K = (int)K; S.flags = flags; S.epi = epi;
      if (transA && transB) launch_small_f<true, true>(c, A, lda, B, ldb, S);
      else if (transA) launch_small_f<true, false>(c, A, lda, B, ldb, S);
      else if (transB) launch_small_f<false, true>(c, A, lda, B, ldb, S);
      else launch_small_f<false, false>(c, A, lda, B, ldb, S);
      return;
    }
  }
  static float* dummy = nullptr;
  if (K <= 0) {
    if (!dummy) CGGM_CUDA_CHECK(cudaMalloc(&dummy, 32 * 32 * 4));
    A = dummy; B = dummy; lda = 32; ldb = 32;
  }
  const int64_t Keff = K > 0 ? K : 1;
  const int64_t arows = transA ? Keff : M, acols = transA ? M : Keff;
  const int64_t brows = transB ? N : Keff, bcols = transB ? Keff : N;
  if (K > 0 && !tma_ok_f(A, lda)) {
    const int64_t ld = (arows + 3) & ~int64_t(3);
    float* pk = static_cast<float*>(ws_get(c, WS_PACK0 + 2 * c->lane, (size_t)ld * acols * 4));
    CGGM_CUDA_CHECK(cudaMemcpy2DAsync(pk, ld * 4, A, lda * 4, arows * 4, acols, cudaMemcpyDeviceToDevice, c->stream));
    A = pk; lda = ld;
  }
  if (K > 0 && !tma_ok_f(B, ldb)) {
    const int64_t ld = (brows + 3) & ~int64_t(3);
    float* pk = static_cast<float*>(ws_get(c, WS_PACK1 + 2 * c->lane, (size_t)ld * bcols * 4));
    CGGM_CUDA_CHECK(cudaMemcpy2DAsync(pk, ld * 4, B, ldb * 4, brows * 4, bcols, cudaMemcpyDeviceToDevice, c->stream));
    B = pk; ldb = ld;
  }
  KParamsF P;
  P.M = (int)M; P.N = (int)N; P.K = (int)(K > 0 ? K : 0);
  P.flags = flags;
  P.epi = epi;
  P.tilesM = (int)((M + FBM - 1) / FBM);
  P.tilesN = (int)((N + FBN - 1) / FBN);
  const int grid = (flags & SYM_LOWER) ? P.tilesN * (P.tilesN + 1) / 2 + (P.tilesM - P.tilesN) * P.tilesN
                                       : P.tilesM * P.tilesN;
  P.a3d = (!transA && M % 32 == 0 && !c->no_tma3d) ? 1 : 0;
  P.b3d = (transB && N % 32 == 0 && !c->no_tma3d) ? 1 : 0;
  CUtensorMap ma = transA ? make_map_f(c, A, lda, Keff, M, FBK, FBM)
                          : (P.a3d ? make_map_f_mn3d(c, A, lda, M, Keff) : make_map_f(c, A, lda, M, Keff, 32, FBK));
  CUtensorMap mb = transB ? (P.b3d ? make_map_f_mn3d(c, B, ldb, N, Keff) : make_map_f(c, B, ldb, N, Keff, 32, FBK))
                          : make_map_f(c, B, ldb, Keff, N, FBK, FBN);
  // 3xTF32 on the tensor cores (gemm_tf32.cu, the same operand maps), except products too small to
  // amortise its per-tile set-up (TMEM allocation, stage pipeline, drain): those keep the FFMA engine
  const bool small = (int64_t)P.tilesM * P.tilesN < c->tf32_min_tiles || K < c->tf32_min_k;
  if (c->f32_engine == 0 && !small) {
    gemm_tf32x3(c, transA, transB, M, N, K, A, lda, B, ldb, epi, flags, ma, mb, P.a3d, P.b3d);
    return;
  }
  const bool AK = transA, BKI = !transB;
  if (AK && BKI) launch_f<true, true>(c, ma, mb, P, grid);
  else if (AK && !BKI) launch_f<true, false>(c, ma, mb, P, grid);
  else if (!AK && BKI) launch_f<false, true>(c, ma, mb, P, grid);
  else launch_f<false, false>(c, ma, mb, P, grid);
}

}  // namespace cggm
