// FP32 variant of the GEMM engine on the 5th-generation tensor cores (reading A18: fp32 inputs,
// fp32 accumulation; north_star "an FP32 variant" of the dense contractions).
//
// TF32 alone (10-bit mantissa) is too inexact for the 1e-4 contract, so every product is the
// 3xTF32 split: x = hi(x) + lo(x), hi = rna_tf32(x), lo = rna_tf32(x - hi) (both exact tf32
// values, |lo| <= 2^-11 |x|), and
//     A B  ~  A_lo B_hi + A_hi B_lo + A_hi B_hi        (the dropped A_lo B_lo is ~2^-22 |A||B|)
// accumulated in one fp32 TMEM accumulator by tcgen05.mma.kind::tf32 (M = 128, N = 128, K = 8).
//
// CTA = 8 producer warps + 4 drain warps + 1 MMA warp (416 threads), one 128 x 128 output tile:
//  * producers (warps 0-7) stream k-tiles of 32: 16-byte global loads of the raw fp32 operands into
//    registers one k-tile ahead, split into hi / lo, and store both into the stage's shared-memory
//    buffers in the canonical layouts the UMMA descriptors name (K-major: SWIZZLE_128B, one 128-byte
//    row per m / n; MN-major: SWIZZLE_128B with 32-byte atoms -- the only MN-major layout of 32-bit
//    operands -- 128-byte rows along m / n, one row per k, 4 KB per 32-wide chunk), then
//    fence.proxy.async and arrive on the stage's full barrier;
//  * the MMA warp's lane 0 waits on the full barrier, issues 4 k-steps x 3 products and
//    tcgen05.commit's the stage's empty barrier (the slot is reusable when those MMAs completed);
//  * hi*hi accumulates in TMEM over chunks of CH k-tiles (two buffers), the corrections in a third
//    accumulator; the drain warps (tcgen05.ld/st 32x32b, warp w owns TMEM lanes 32(w%4).. = rows)
//    add each finished chunk into a running fp32 sum kept in TMEM (the tensor core's own accumulation
//    rounds toward zero), then the corrections, stage the tile in shared memory and run the engine's
//    common epilogue (alpha / beta / second output, lower trapezoid, mirrored symmetric writes).
// Same flags, tile order and epilogue contract as the FFMA kernel (gemm_f32.cu), which stays as the
// A/B alternative (CGGM_F32_ENGINE=ffma, cggm_test_set_f32_engine).
#include "common.cuh"

namespace cggm {
namespace {

constexpr int TBM = 128, TBN = 128, TBK = 32;
constexpr int T_OP = TBM * TBK * 4;          // 16 KB per operand half (hi or lo) or raw operand tile
constexpr int T_STAGE = 4 * T_OP;            // split stage: A_hi, A_lo, B_hi, B_lo
constexpr int T_RAW = 2 * T_OP;              // raw stage (TMA producer): A, B fp32 tiles
constexpr int T_EPI_LD = TBM + 1;
constexpr int T_PROD = 256;                  // producer / converter threads (warps 0-7)
constexpr int T_PER = TBM * TBK / 4 / T_PROD;   // float4 per operand per producer thread per k-tile (4)
constexpr int T_DRAIN = 128;                 // accumulator-drain / epilogue threads (warps 8-11)
constexpr int T_DW0 = T_PROD / 32;           // first drain warp
constexpr int T_MMA_WARP = T_DW0 + 4;        // the MMA-issuing warp (12)
constexpr int T_TMA_WARP = T_MMA_WARP + 1;   // the TMA-issuing warp (13, TMA producer only)
constexpr int T_GROUP_N = 8;
constexpr uint32_t T_TMEM_COLS = 512;   // X0 (cols 0-127), D2 (128-255), X1 (256-383), running sum S (384-511)
// Producer modes: LDG (registers, one k-tile ahead; 3 split stages) or TMA (raw fp32 tiles by TMA into
// a 3-deep ring -- the loads no longer wait on the converters' registers -- converted from shared
// memory into 2 split stages)
template <bool TMA> struct TCfg {
  static constexpr int NSPLIT = TMA ? 2 : 3;
  static constexpr int NRAW = TMA ? 3 : 1;                         // (1: unused by the LDG producer)
  static constexpr int DATA = NSPLIT * T_STAGE + (TMA ? NRAW * T_RAW : 0);   // LDG 192 KB, TMA 224 KB
  static constexpr int SMEM = DATA + 1024 + 256;
  static constexpr int NT = T_PROD + T_DRAIN + 32 + (TMA ? 32 : 0);
  static_assert(TBN * T_EPI_LD * 4 <= DATA, "epilogue tile must fit in the stage buffers");
};

struct KParamsT {
  int M, N, K;
  int tilesM, tilesN;
  int flags;
  const float* A;
  int64_t lda;
  const float* B;
  int64_t ldb;
  int chunk;      // k-tiles per drained partial sum (0: one TMEM accumulator over the whole k-range)
  int a3d, b3d;   // TMA producer: MN-inner operand as one 3-D box (extent a multiple of 32)
  int dbg;        // measurement aid (CGGM_TF32_DEBUG): bit 0 = hi*hi products only
  int cfrel;      // TS form: split stages released by the chunk commits (Ctx::tf32_cfrel)
  EpilogueT<float> epi;
};

__device__ __forceinline__ void tile_coords_t(const KParamsT& P, int t, int& I, int& J) {
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
  const int per_group = T_GROUP_N * P.tilesM;
  const int gi = t / per_group;
  const int local = t - gi * per_group;
  const int nb0 = gi * T_GROUP_N;
  const int width = min(T_GROUP_N, P.tilesN - nb0);
  I = local / width;
  J = nb0 + local % width;
  if (P.flags & B_KLE_N) J = P.tilesN - 1 - J;
  if (P.flags & A_KLE_M) I = P.tilesM - 1 - I;
}

__device__ __forceinline__ void epi_apply_t(const EpilogueT<float>& E, int64_t r, int64_t c, float v) {
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

__device__ __forceinline__ void epi_mirror_t(const EpilogueT<float>& E, int64_t r, int64_t c, float v) {
  if (E.mir1) E.mir1[r + c * E.ld1] = __fmul_rn((float)E.a1, v);
  else epi_apply_t(E, r, c, v);
}

// ---------------------------------------------------------------- tcgen05 / TMEM PTX
// round-to-nearest (ties away) to tf32 on the bit pattern: +half an ulp of the 10-bit mantissa, clear
// the 13 low bits (a mantissa carry moves into the exponent, as it should); two integer ops instead
// of the conversion unit's cvt.rna.tf32 (the split runs on every operand element of every k-tile)
__device__ __forceinline__ uint32_t rna_tf32(float x) { return (__float_as_uint(x) + 0x1000u) & 0xFFFFE000u; }
// lo of the split for an operand the tensor core reads (hi = rna_tf32(v), so v - hi is exact in
// fp32): + half a tf32 ulp without the mask -- kind::tf32 ignores the 13 low mantissa bits of a
// 32-bit operand (truncation, measured: tools/debug/tf32_trunc_probe.py), so the MMA multiplies
// rna_tf32(lo) and the split costs one integer op less per element
__device__ __forceinline__ uint32_t lo_tf32(float v, uint32_t hi) { return __float_as_uint(v - __uint_as_float(hi)) + 0x1000u; }

// shared-memory matrix descriptor (tcgen05): start >> 4 [0,14), LBO >> 4 [16,30), SBO >> 4 [32,46),
// version 1 [46,48), base offset 0, layout at [61,64): SWIZZLE_128B = 2 (K-major), SWIZZLE_128B with
// 32-byte atoms = 1 (the only MN-major layout of 32-bit operands)
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint64_t layout) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (layout << 61);
}

// instruction descriptor: D fp32 [4,6) = 1, A / B tf32 [7,10) / [10,13) = 2, A / B major [15] / [16]
// (0 K-major, 1 MN-major), N >> 3 at [17,23), M >> 4 at [24,29)
__host__ __device__ constexpr uint32_t idesc_tf32(bool a_mn, bool b_mn, int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                   ptx::smem_u32(bar))
               : "memory");
}

// one lane of the (converged) warp: true on exactly one lane
__device__ __forceinline__ bool elect_one() {
  uint32_t p = 0;
  asm volatile("{\n.reg .pred P;\nelect.sync _|P, 0xffffffff;\nselp.u32 %0, 1, 0, P;\n}\n" : "=r"(p));
  return p != 0;
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}

// two 32-column loads in flight, one wait: the "+r" operands keep every use of the loaded registers
// after the wait (the loads' outputs are only valid then)
__device__ __forceinline__ void tmem_ld32_nowait(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}

__device__ __forceinline__ void tmem_wait_ld64(uint32_t (&a)[32], uint32_t (&b)[32]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;\n"
               : "+r"(a[0]),"+r"(a[1]),"+r"(a[2]),"+r"(a[3]),"+r"(a[4]),"+r"(a[5]),"+r"(a[6]),"+r"(a[7]),"+r"(a[8]),"+r"(a[9]),"+r"(a[10]),"+r"(a[11]),"+r"(a[12]),"+r"(a[13]),"+r"(a[14]),"+r"(a[15]),"+r"(a[16]),"+r"(a[17]),"+r"(a[18]),"+r"(a[19]),"+r"(a[20]),"+r"(a[21]),"+r"(a[22]),"+r"(a[23]),"+r"(a[24]),"+r"(a[25]),"+r"(a[26]),"+r"(a[27]),"+r"(a[28]),"+r"(a[29]),"+r"(a[30]),"+r"(a[31]),
                 "+r"(b[0]),"+r"(b[1]),"+r"(b[2]),"+r"(b[3]),"+r"(b[4]),"+r"(b[5]),"+r"(b[6]),"+r"(b[7]),"+r"(b[8]),"+r"(b[9]),"+r"(b[10]),"+r"(b[11]),"+r"(b[12]),"+r"(b[13]),"+r"(b[14]),"+r"(b[15]),"+r"(b[16]),"+r"(b[17]),"+r"(b[18]),"+r"(b[19]),"+r"(b[20]),"+r"(b[21]),"+r"(b[22]),"+r"(b[23]),"+r"(b[24]),"+r"(b[25]),"+r"(b[26]),"+r"(b[27]),"+r"(b[28]),"+r"(b[29]),"+r"(b[30]),"+r"(b[31])
               :
               : "memory");
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};\n" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
      "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
      "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
}

// ---------------------------------------------------------------- producer: loads and the split
// Operand tile of 128 (m or n) x 32 (k), 1024 float4 = 4 per producer thread.
//  K-inner (element (x, k) at base[k + x ld]):  f -> row x = f >> 3, 16-byte chunk c = f & 7
//  MN-inner (element (x, k) at base[x + k ld]): f -> k = f >> 5, x = 4 (f & 31)
template <bool KIN>
__device__ __forceinline__ void load_tile(float4 (&r)[T_PER], const float* __restrict__ base, int64_t ld, int x0, int X,
                                          int k0, int K, int tid) {
#pragma unroll
  for (int i = 0; i < T_PER; ++i) {
    const int f = tid + T_PROD * i;
    int x, k;
    if (KIN) {
      x = x0 + (f >> 3);
      k = k0 + 4 * (f & 7);
    } else {
      k = k0 + (f >> 5);
      x = x0 + 4 * (f & 31);
    }
    const float* p = KIN ? base + (int64_t)x * ld + k : base + (int64_t)k * ld + x;
    const bool full = KIN ? (x < X && k + 3 < K) : (k < K && x + 3 < X);
    if (full) {
      r[i] = __ldg(reinterpret_cast<const float4*>(p));
    } else {
      float v[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const bool ok = KIN ? (x < X && k + e < K) : (k < K && x + e < X);
        v[e] = ok ? __ldg(p + e) : 0.f;
      }
      r[i] = make_float4(v[0], v[1], v[2], v[3]);
    }
  }
}

__device__ __forceinline__ void sts128(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}

template <bool KIN>
__device__ __forceinline__ void store_split(const float4 (&r)[T_PER], uint32_t hi, uint32_t lo, int tid) {
#pragma unroll
  for (int i = 0; i < T_PER; ++i) {
    const int f = tid + T_PROD * i;
    uint32_t off;
    if (KIN) {
      const int row = f >> 3, c = f & 7;
      off = row * 128 + ((c ^ (row & 7)) << 4);
    } else {
      // MN-major, 128-byte rows along m / n, 32-byte swizzle atoms: 32-byte unit u of row k sits at
      // u ^ (k & 3) (byte-address bits [5,7) ^= [7,9))
      const int k = f >> 5, mc = f & 31, c = mc & 7;
      off = (mc >> 3) * 4096 + k * 128 + (((((c >> 1) ^ (k & 3)) << 1) | (c & 1)) << 4);
    }
    const float v[4] = {r[i].x, r[i].y, r[i].z, r[i].w};
    uint32_t h[4], l[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      h[e] = rna_tf32(v[e]);
      l[e] = rna_tf32(v[e] - __uint_as_float(h[e]));
    }
    sts128(hi + off, h[0], h[1], h[2], h[3]);
    sts128(lo + off, l[0], l[1], l[2], l[3]);
  }
}

// raw tile in the TMA SWIZZLE_128B layout (16-byte atoms: chunk c of 128-byte row r at c ^ (r & 7))
// -> hi / lo in the UMMA layouts (K-major: the same positions; MN-major: 32-byte atoms)
template <bool KIN, int NTH = T_PROD>
__device__ __forceinline__ void convert_split(uint32_t raw, uint32_t hi, uint32_t lo, int tid) {
#pragma unroll
  for (int i = 0; i < TBM * TBK / 4 / NTH; ++i) {
    const int f = tid + NTH * i;
    uint32_t ro, so;
    if (KIN) {
      const int row = f >> 3, c = f & 7;
      ro = so = row * 128 + ((c ^ (row & 7)) << 4);
    } else {
      const int k = f >> 5, mc = f & 31, c = mc & 7;
      const uint32_t base = (mc >> 3) * 4096 + k * 128;
      ro = base + ((c ^ (k & 7)) << 4);
      so = base + (((((c >> 1) ^ (k & 3)) << 1) | (c & 1)) << 4);
    }
    float v[4];
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];\n" : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]) : "r"(raw + ro));
    uint32_t h[4], l[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      h[e] = rna_tf32(v[e]);
      l[e] = rna_tf32(v[e] - __uint_as_float(h[e]));
    }
    sts128(hi + so, h[0], h[1], h[2], h[3]);
    sts128(lo + so, l[0], l[1], l[2], l[3]);
  }
}

// raw B tile (TMA SWIZZLE_128B) -> registers, NTH threads, 16-byte chunks f = tid + NTH i; and the
// split of those registers into the UMMA layouts of hi / lo (the convert_split positions)
// one 16-byte chunk (i-th of this thread) of the raw B tile / of its hi / lo stores
template <bool KIN, int NTH>
__device__ __forceinline__ void raw_b_chunk(uint32_t raw, float (&v)[4], int tid, int i) {
  const int f = tid + NTH * i;
  uint32_t ro;
  if (KIN) {
    const int row = f >> 3, c = f & 7;
    ro = row * 128 + ((c ^ (row & 7)) << 4);
  } else {
    const int k = f >> 5, mc = f & 31, c = mc & 7;
    ro = (mc >> 3) * 4096 + k * 128 + ((c ^ (k & 7)) << 4);
  }
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];\n" : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]) : "r"(raw + ro));
}

template <bool KIN, int NTH>
__device__ __forceinline__ void store_b_chunk(const uint32_t (&h)[4], const uint32_t (&l)[4], uint32_t hi, uint32_t lo,
                                              int tid, int i) {
  const int f = tid + NTH * i;
  uint32_t so;
  if (KIN) {
    const int row = f >> 3, c = f & 7;
    so = row * 128 + ((c ^ (row & 7)) << 4);
  } else {
    const int k = f >> 5, mc = f & 31, c = mc & 7;
    so = (mc >> 3) * 4096 + k * 128 + (((((c >> 1) ^ (k & 3)) << 1) | (c & 1)) << 4);
  }
  sts128(hi + so, h[0], h[1], h[2], h[3]);
  sts128(lo + so, l[0], l[1], l[2], l[3]);
}

template <bool AK, bool BKI, bool TMA>
__global__ void __launch_bounds__(TCfg<TMA>::NT, 1)
    gemm_tf32x3_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                       const __grid_constant__ KParamsT P) {
  using C = TCfg<TMA>;
  constexpr int TSTAGES = C::NSPLIT;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::DATA);
  uint64_t* empty = full + 3;
  uint64_t* rfull = empty + 3;           // raw stage landed (TMA)
  uint64_t* rempty = rfull + 3;          // raw stage converted
  uint64_t* cfull = rempty + 3;          // chunk partial in X[b] complete
  uint64_t* cempty = cfull + 2;          // X[b] drained
  uint64_t* accf = cempty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accf + 1);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  int I, J;
  tile_coords_t(P, blockIdx.x, I, J);
  const int m0 = I * TBM, n0 = J * TBN;
  int kbeg = 0, kend = P.K;
  if (P.flags & A_KGE_M) kbeg = max(kbeg, m0);
  if (P.flags & B_KGE_N) kbeg = max(kbeg, n0);
  if (P.flags & A_KLE_M) kend = min(kend, m0 + TBM);
  if (P.flags & B_KLE_N) kend = min(kend, n0 + TBN);
  const int kt0 = kbeg / TBK;
  const int nkt = kend > kbeg ? (kend - kt0 * TBK + TBK - 1) / TBK : 0;
  const int CH = P.chunk;
  const bool drain = CH > 0;
  if (tid == 0) {
    for (int s = 0; s < TSTAGES; ++s) {
      ptx::mbar_init(&full[s], T_PROD);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&cfull[b], 1);
      ptx::mbar_init(&cempty[b], T_DRAIN);
    }
    for (int r = 0; r < C::NRAW; ++r) {
      ptx::mbar_init(&rfull[r], 1);
      ptx::mbar_init(&rempty[r], T_PROD);
    }
    ptx::mbar_init(accf, 1);
    ptx::fence_barrier_init();
  }
  if (warp == T_MMA_WARP) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(ptx::smem_u32(tmem_slot)),
                 "n"(T_TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t sbase = ptx::smem_u32(smem);

  if (warp == T_MMA_WARP) {
    // ---- MMA issue (one thread).  With draining, the hi*hi products of chunk c (CH k-tiles) go to
    // X[c & 1], which the drain warps add into a running fp32 sum (round-to-nearest) while the next
    // chunk fills the other buffer; the two corrections (~2^-11 of the result) accumulate in D2 over
    // the whole k-range.  The tensor core's accumulation rounds toward zero, so a long k-range in one
    // accumulator is biased by ~k/8 x 2^-24 relative (measured, tools/debug/tf32_acc_probe.py);
    // bounded chunks keep fp32-class accuracy.
    if (lane == 0 && nkt > 0) {
      constexpr uint32_t idesc = idesc_tf32(!AK, !BKI, TBM, TBN);
      for (int j = 0; j < nkt; ++j) {
        const int s = j % TSTAGES;
        const int c = drain ? j / CH : 0;
        const bool first = drain && (j % CH == 0);
        if (first && c >= 2) {
          ptx::mbar_wait(&cempty[c & 1], ((c >> 1) - 1) & 1);
          tc_fence_after();
        }
        ptx::mbar_wait(&full[s], (j / TSTAGES) & 1);
        tc_fence_after();
        const uint32_t st = sbase + s * T_STAGE;
        const uint32_t a_hi = st, a_lo = st + T_OP, b_hi = st + 2 * T_OP, b_lo = st + 3 * T_OP;
        const uint32_t X = tmem + ((c & 1) ? 256u : 0u);
#pragma unroll
        for (int kk = 0; kk < TBK / 8; ++kk) {
          // K-major: the k-step advances 32 bytes inside the 128-byte swizzled row (SBO = 8 rows = 1 KB);
          // MN-major: it advances two 4-row k groups (SBO = 512 B; LBO = 4 KB between 32-wide chunks)
          const uint32_t oa = kk * (AK ? 32 : 1024), ob = kk * (BKI ? 32 : 1024);
          const uint32_t la = AK ? 16 : 4096, lb = BKI ? 16 : 4096;
          const uint32_t sa = AK ? 1024 : 512, sb = BKI ? 1024 : 512;
          const uint64_t ya = AK ? 2 : 1, yb = BKI ? 2 : 1;
          const uint64_t dah = sdesc(a_hi + oa, la, sa, ya), dal = sdesc(a_lo + oa, la, sa, ya);
          const uint64_t dbh = sdesc(b_hi + ob, lb, sb, yb), dbl = sdesc(b_lo + ob, lb, sb, yb);
          if (P.dbg & 1) {
            umma_tf32(X, dah, dbh, idesc, (first && kk == 0) || (!drain && (j | kk) == 0) ? 0u : 1u);
          } else if (drain) {
            umma_tf32(tmem + 128u, dal, dbh, idesc, (j | kk) != 0);
            umma_tf32(tmem + 128u, dah, dbl, idesc, 1u);
            umma_tf32(X, dah, dbh, idesc, (first && kk == 0) ? 0u : 1u);
          } else {
            umma_tf32(tmem, dal, dbh, idesc, (j | kk) != 0);
            umma_tf32(tmem, dah, dbl, idesc, 1u);
            umma_tf32(tmem, dah, dbh, idesc, 1u);
          }
        }
        umma_commit(&empty[s]);   // the slot is free once these MMAs have read it
        if (drain && (j % CH == CH - 1 || j == nkt - 1)) umma_commit(&cfull[c & 1]);
      }
      umma_commit(accf);
    }
    __syncwarp();
  } else if (warp < T_DW0 && !TMA) {
    // ---- producers (warps 0-7): operand k-tiles, one ahead in registers
    const float* A = P.A;
    const float* B = P.B;
    float4 ra[T_PER], rb[T_PER];
    if (nkt > 0) {
      load_tile<AK>(ra, A, P.lda, m0, P.M, kt0 * TBK, P.K, tid);
      load_tile<BKI>(rb, B, P.ldb, n0, P.N, kt0 * TBK, P.K, tid);
    }
    for (int it = 0; it < nkt; ++it) {
      const int s = it % TSTAGES;
      float4 na[T_PER], nb[T_PER];
      if (it + 1 < nkt) {
        load_tile<AK>(na, A, P.lda, m0, P.M, (kt0 + it + 1) * TBK, P.K, tid);
        load_tile<BKI>(nb, B, P.ldb, n0, P.N, (kt0 + it + 1) * TBK, P.K, tid);
      }
      if (it >= TSTAGES) ptx::mbar_wait(&empty[s], ((it / TSTAGES) - 1) & 1);
      const uint32_t st = sbase + s * T_STAGE;
      store_split<AK>(ra, st, st + T_OP, tid);
      store_split<BKI>(rb, st + 2 * T_OP, st + 3 * T_OP, tid);
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      ptx::mbar_arrive(&full[s]);
      if (it + 1 < nkt) {
#pragma unroll
        for (int i = 0; i < T_PER; ++i) {
          ra[i] = na[i];
          rb[i] = nb[i];
        }
      }
    }
  } else if (warp < T_DW0) {
    // ---- converters (warps 0-7, TMA producer): raw fp32 stage (TMA SWIZZLE_128B, 16-byte atoms) ->
    // hi / lo in the UMMA layouts of the split stage
    const uint32_t rbase = sbase + TSTAGES * T_STAGE;
    for (int it = 0; it < nkt; ++it) {
      const int s = it % TSTAGES, rs = it % C::NRAW;
      ptx::mbar_wait(&rfull[rs], (it / C::NRAW) & 1);
      if (it >= TSTAGES) ptx::mbar_wait(&empty[s], ((it / TSTAGES) - 1) & 1);
      const uint32_t st = sbase + s * T_STAGE, rw = rbase + rs * T_RAW;
      convert_split<AK>(rw, st, st + T_OP, tid);
      convert_split<BKI>(rw + T_OP, st + 2 * T_OP, st + 3 * T_OP, tid);
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      ptx::mbar_arrive(&full[s]);
      ptx::mbar_arrive(&rempty[rs]);
    }
  } else if (TMA && warp == T_TMA_WARP) {
    // ---- TMA warp: raw k-tiles into the 3-deep ring (K-inner: one {32, 128} box; MN-inner: one 3-D
    // {32, 32, 4} box, or 32-wide 2-D boxes for a ragged extent; out-of-range k is zero-filled)
    if (lane == 0 && nkt > 0) {
      int a_boxes = 0, b_boxes = 0;
      if (!AK)
        for (int xb = 0; xb < TBM / 32; ++xb) a_boxes += (m0 + xb * 32 < P.M);
      if (!BKI)
        for (int xb = 0; xb < TBN / 32; ++xb) b_boxes += (n0 + xb * 32 < P.N);
      const uint32_t txb = ((AK || P.a3d) ? T_OP : a_boxes * 4096) + ((BKI || P.b3d) ? T_OP : b_boxes * 4096);
      ptx::prefetch_tmap(&tmA);
      ptx::prefetch_tmap(&tmB);
      uint8_t* rbase = smem + TSTAGES * T_STAGE;
      for (int j = 0; j < nkt; ++j) {
        const int rs = j % C::NRAW;
        if (j >= C::NRAW) ptx::mbar_wait(&rempty[rs], ((j / C::NRAW) - 1) & 1);
        uint8_t* sa = rbase + rs * T_RAW;
        uint8_t* sb = sa + T_OP;
        ptx::mbar_arrive_expect_tx(&rfull[rs], txb);
        const int k = (kt0 + j) * TBK;
        if (AK) ptx::tma_load_2d(sa, &tmA, &rfull[rs], k, m0);
        else if (P.a3d) ptx::tma_load_3d(sa, &tmA, &rfull[rs], 0, k, m0 / 32);
        else
          for (int xb = 0; xb < a_boxes; ++xb) ptx::tma_load_2d(sa + xb * 4096, &tmA, &rfull[rs], m0 + xb * 32, k);
        if (BKI) ptx::tma_load_2d(sb, &tmB, &rfull[rs], k, n0);
        else if (P.b3d) ptx::tma_load_3d(sb, &tmB, &rfull[rs], 0, k, n0 / 32);
        else
          for (int xb = 0; xb < b_boxes; ++xb) ptx::tma_load_2d(sb + xb * 4096, &tmB, &rfull[rs], n0 + xb * 32, k);
      }
    }
    __syncwarp();
  } else {
    // ---- drain warps 8-11 (warp w reads TMEM lanes 32 (w % 4)..: one accumulator row per thread):
    // the running fp32 sum S (TMEM cols 384-511) += each finished chunk, then + D2, then the epilogue
    const int dt = tid - T_PROD;
    const int row = (warp - T_DW0) * 32 + lane;
    const uint32_t lanebase = tmem + ((uint32_t)((warp - T_DW0) * 32) << 16);
    const int nch = nkt > 0 ? (drain ? (nkt + CH - 1) / CH : 1) : 0;
    for (int c = 0; c < nch; ++c) {
      if (drain) ptx::mbar_wait(&cfull[c & 1], (c >> 1) & 1);
      else ptx::mbar_wait(accf, 0);
      tc_fence_after();
      const uint32_t xa = lanebase + ((c & 1) ? 256u : 0u);
#pragma unroll 1
      for (int g = 0; g < TBN / 32; ++g) {
        uint32_t v[32], w[32];
        tmem_ld32(xa + 32u * g, v);
        if (c > 0) {
          tmem_ld32(lanebase + 384u + 32u * g, w);
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = __float_as_uint(__uint_as_float(w[j]) + __uint_as_float(v[j]));
        }
        tmem_st32(lanebase + 384u + 32u * g, v);
      }
      tc_fence_before();
      if (drain) ptx::mbar_arrive(&cempty[c & 1]);
    }
    if (nkt > 0 && drain) {
      ptx::mbar_wait(accf, 0);
      tc_fence_after();
    }
    float* Cs = reinterpret_cast<float*>(smem);   // stage buffers: every MMA has completed (accf)
#pragma unroll 1
    for (int g = 0; g < TBN / 32; ++g) {
      uint32_t v[32], w[32];
      if (nkt > 0) {
        tmem_ld32(lanebase + 384u + 32u * g, v);
        if (drain) {
          tmem_ld32(lanebase + 128u + 32u * g, w);
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = __float_as_uint(__uint_as_float(v[j]) + __uint_as_float(w[j]));
        }
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = 0u;
      }
#pragma unroll
      for (int j = 0; j < 32; ++j) Cs[(32 * g + j) * T_EPI_LD + row] = __uint_as_float(v[j]);
    }
    tc_fence_before();
    asm volatile("bar.sync 1, %0;\n" ::"n"(T_DRAIN) : "memory");
    const bool diag = (P.flags & SYM_LOWER) && I == J;
    for (int idx = dt; idx < TBM * TBN; idx += T_DRAIN) {
      const int mm = idx % TBM, nl = idx / TBM;
      const int m = m0 + mm, n = n0 + nl;
      if (m >= P.M || n >= P.N) continue;
      if (diag && m < n) continue;
      epi_apply_t(P.epi, m, n, Cs[nl * T_EPI_LD + mm]);
    }
    if (P.flags & SYM_MIRROR) {
      for (int idx = dt; idx < TBM * TBN; idx += T_DRAIN) {
        const int nl = idx % TBN, mm = idx / TBN;
        const int m = m0 + mm, n = n0 + nl;
        if (m >= P.M || n >= P.N) continue;
        if (diag && m <= n) continue;
        epi_mirror_t(P.epi, n, m, Cs[nl * T_EPI_LD + mm]);
      }
    }
  }
  __syncthreads();
  if (warp == T_MMA_WARP) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(T_TMEM_COLS) : "memory");
  }
}

// ---------------------------------------------------------------- TS form (A from TMEM)
// The converters write A's hi / lo tiles into TMEM (tcgen05.st, one accumulator row per thread) and
// only B's into shared memory; the MMA reads A from TMEM (tcgen05.mma ... [a_tmem], b_desc) -- the
// SS form's A operand reads (half of its 122 B/clk of shared-memory traffic) disappear.  TMEM: chunk
// accumulators X0, X1 (cols 0-255; hi*hi AND the corrections, chunks of TS_CH k-tiles drained into
// fp32 registers) and 4 A stages of 64 columns (hi 32 + lo 32) at 256..511.
// CGGM_TS_CONV8 = 1: eight converter warps (two per TMEM lane quarter, each taking half of the k-tile's
// 32 k) instead of four -- the four were the bound (ncu, 8192^3: tensor pipe 57.7% active, the MMA
// waiting on the split stages); 16 warps in four warpgroups then, registers rebalanced by setmaxnreg
// (converters 96, drain 232, MMA / TMA / two idle warps 40)
#ifndef CGGM_TS_CONV8
#define CGGM_TS_CONV8 1
#endif
constexpr int TS_CONV = CGGM_TS_CONV8 ? 256 : 128;   // converter threads (warps 0-3 (and 4-7): TMEM lane quarters)
constexpr int TS_KH = TS_CONV / 128;          // k-parts of a row (one per converter warp of a lane quarter)
#ifndef CGGM_TS_NS
#define CGGM_TS_NS 4
#endif
constexpr int TS_NS = CGGM_TS_NS;            // split stages (TMEM A, shared B)
constexpr int TS_NRAW = 7 - CGGM_TS_NS;      // raw TMA stages (the two rings share 224 KB of shared memory)
constexpr int TS_BSTAGE = 2 * T_OP;          // B hi + lo
constexpr int TS_BPER = TBN * TBK / 4 / TS_CONV;   // raw B 16-byte chunks per converter thread (8 / 4)
constexpr int TS_DATA = TS_NS * TS_BSTAGE + TS_NRAW * T_RAW;   // 128 + 96 KB
static_assert(TBN * T_EPI_LD * 4 <= TS_DATA, "epilogue tile must fit");
constexpr int TS_SMEM = TS_DATA + 1024 + 256;
constexpr int TS_NT = CGGM_TS_CONV8 ? 512 : TS_CONV + T_DRAIN + 64;  // + MMA warp, TMA warp (+ 2 idle: whole warpgroups)
constexpr int TS_DW0 = TS_CONV / 32, TS_MMA = TS_DW0 + 4, TS_TMAW = TS_MMA + 1;

__device__ __forceinline__ void umma_tf32_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t db, uint32_t idesc,
                                             uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(db), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void tmem_st32_nowait(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};\n" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
      "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
      "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}

// row m of the raw A tile (TMA SWIZZLE_128B layout) -> the KN k-values k0 .. k0 + KN - 1
template <bool AK, int KN = 32>
__device__ __forceinline__ void raw_a_row(uint32_t raw, int m, float (&v)[KN], int k0 = 0) {
  if (AK) {   // K-inner: row m = one 128-byte row, 16-byte chunk c at c ^ (m & 7)
#pragma unroll
    for (int c = 0; c < KN / 4; ++c) {
      const int cc = k0 / 4 + c;
      asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];\n"
                   : "=f"(v[4 * c]), "=f"(v[4 * c + 1]), "=f"(v[4 * c + 2]), "=f"(v[4 * c + 3])
                   : "r"(raw + m * 128 + ((cc ^ (m & 7)) << 4)));
    }
  } else {    // MN-inner: element (m, k) in chunk m / 32, row k, 16-byte chunk ((m % 32) / 4) ^ (k & 7)
    const uint32_t base = (m >> 5) * 4096 + (m & 3) * 4;
    const int mc = (m & 31) >> 2;
#pragma unroll
    for (int e = 0; e < KN; ++e) {
      const int k = k0 + e;
      asm volatile("ld.shared.f32 %0, [%1];\n" : "=f"(v[e]) : "r"(raw + base + k * 128 + ((mc ^ (k & 7)) << 4)));
    }
  }
}

__device__ __forceinline__ void tmem_st16_nowait(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n" ::"r"(
          taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}

template <bool AK, bool BKI>
__global__ void __launch_bounds__(TS_NT, 1)
    gemm_tf32x3_ts_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                          const __grid_constant__ KParamsT P) {
  CGGM_DASSERT(blockDim.x == TS_NT);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + TS_DATA);
  uint64_t* empty = full + TS_NS;
  uint64_t* rfull = empty + TS_NS;
  uint64_t* rempty = rfull + TS_NRAW;
  uint64_t* cfull = rempty + TS_NRAW;
  uint64_t* cempty = cfull + 2;
  uint64_t* accf = cempty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accf + 1);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  int I, J;
  tile_coords_t(P, blockIdx.x, I, J);
  const int m0 = I * TBM, n0 = J * TBN;
  int kbeg = 0, kend = P.K;
  if (P.flags & A_KGE_M) kbeg = max(kbeg, m0);
  if (P.flags & B_KGE_N) kbeg = max(kbeg, n0);
  if (P.flags & A_KLE_M) kend = min(kend, m0 + TBM);
  if (P.flags & B_KLE_N) kend = min(kend, n0 + TBN);
  const int kt0 = kbeg / TBK;
  const int nkt = kend > kbeg ? (kend - kt0 * TBK + TBK - 1) / TBK : 0;
  const int CH = P.chunk > 0 ? P.chunk : 1 << 30;
  // split stages released by the chunk commits (one commit per chunk instead of one per stage plus
  // one per chunk) when a chunk spans whole stage groups and the converters cannot fall two phases
  // behind on a chunk barrier: CH divides TS_NS and 2 CH >= TS_NS (CGGM_TF32_CFREL=1; measured neutral:
  // the skeleton 235-248 TF/s either way)
  const bool cf_rel = P.cfrel && CH <= TS_NS && TS_NS % CH == 0 && 2 * CH >= TS_NS;
  if (tid == 0) {
    for (int s = 0; s < TS_NS; ++s) {
      ptx::mbar_init(&full[s], TS_CONV);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int r = 0; r < TS_NRAW; ++r) {
      ptx::mbar_init(&rfull[r], 1);
      ptx::mbar_init(&rempty[r], TS_CONV);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&cfull[b], 1);
      ptx::mbar_init(&cempty[b], T_DRAIN);
    }
    ptx::mbar_init(accf, 1);
    ptx::fence_barrier_init();
  }
  if (warp == TS_MMA) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(ptx::smem_u32(tmem_slot)),
                 "n"(T_TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t sbase = ptx::smem_u32(smem);
  const uint32_t rbase = sbase + TS_NS * TS_BSTAGE;
  auto mma_role = [&]() {
    // the whole warp walks the loop (warp-uniform control flow: the descriptors stay in uniform
    // registers); one elected lane issues the MMAs and their commits
    if (nkt > 0) {
      constexpr uint32_t idesc = idesc_tf32(false, !BKI, TBM, TBN);
      const bool leader = elect_one();
      for (int j = 0; j < nkt; ++j) {
        const int s = j % TS_NS;
        const int c = j / CH;
        const bool first = (j % CH == 0);
        if (first && c >= 2) {
          ptx::mbar_wait(&cempty[c & 1], ((c >> 1) - 1) & 1);
          tc_fence_after();
        }
        ptx::mbar_wait(&full[s], (j / TS_NS) & 1);
        tc_fence_after();
        const uint32_t b_hi = sbase + s * TS_BSTAGE, b_lo = b_hi + T_OP;
        const uint32_t a_hi = tmem + 256u + (uint32_t)s * 64u, a_lo = a_hi + 32u;
        const uint32_t X = tmem + ((c & 1) ? 128u : 0u);
        if (leader) {
#pragma unroll
          for (int kk = 0; kk < TBK / 8; ++kk) {
            const uint32_t ob = kk * (BKI ? 32 : 1024);
            const uint32_t lb = BKI ? 16 : 4096, sb = BKI ? 1024 : 512;
            const uint64_t yb = BKI ? 2 : 1;
            const uint64_t dbh = sdesc(b_hi + ob, lb, sb, yb), dbl = sdesc(b_lo + ob, lb, sb, yb);
            umma_tf32_ts(X, a_lo + kk * 8u, dbh, idesc, (first && kk == 0) ? 0u : 1u);
            umma_tf32_ts(X, a_hi + kk * 8u, dbl, idesc, 1u);
            umma_tf32_ts(X, a_hi + kk * 8u, dbh, idesc, 1u);
          }
          if (!cf_rel) umma_commit(&empty[s]);
          if (j % CH == CH - 1 || j == nkt - 1) umma_commit(&cfull[c & 1]);
        }
        __syncwarp();
      }
      if (leader) umma_commit(accf);
    }
    __syncwarp();
  };
  auto tma_role = [&]() {
    if (lane == 0 && nkt > 0) {
      int a_boxes = 0, b_boxes = 0;
      if (!AK)
        for (int xb = 0; xb < TBM / 32; ++xb) a_boxes += (m0 + xb * 32 < P.M);
      if (!BKI)
        for (int xb = 0; xb < TBN / 32; ++xb) b_boxes += (n0 + xb * 32 < P.N);
      const uint32_t txb = ((AK || P.a3d) ? T_OP : a_boxes * 4096) + ((BKI || P.b3d) ? T_OP : b_boxes * 4096);
      ptx::prefetch_tmap(&tmA);
      ptx::prefetch_tmap(&tmB);
      uint8_t* rb = smem + TS_NS * TS_BSTAGE;
      for (int j = 0; j < nkt; ++j) {
        const int rs = j % TS_NRAW;
        if (j >= TS_NRAW) ptx::mbar_wait(&rempty[rs], ((j / TS_NRAW) - 1) & 1);
        uint8_t* sa = rb + rs * T_RAW;
        uint8_t* sbp = sa + T_OP;
        ptx::mbar_arrive_expect_tx(&rfull[rs], txb);
        const int k = (kt0 + j) * TBK;
        if (AK) ptx::tma_load_2d(sa, &tmA, &rfull[rs], k, m0);
        else if (P.a3d) ptx::tma_load_3d(sa, &tmA, &rfull[rs], 0, k, m0 / 32);
        else
          for (int xb = 0; xb < a_boxes; ++xb) ptx::tma_load_2d(sa + xb * 4096, &tmA, &rfull[rs], m0 + xb * 32, k);
        if (BKI) ptx::tma_load_2d(sbp, &tmB, &rfull[rs], k, n0);
        else if (P.b3d) ptx::tma_load_3d(sbp, &tmB, &rfull[rs], 0, k, n0 / 32);
        else
          for (int xb = 0; xb < b_boxes; ++xb) ptx::tma_load_2d(sbp + xb * 4096, &tmB, &rfull[rs], n0 + xb * 32, k);
      }
    }
    __syncwarp();
  };
  auto conv_role = [&]() {
    // ---- converters: A row (32 k) of this thread's TMEM lane -> hi / lo columns of the stage; B tile
    // -> hi / lo in shared memory, one 16-byte chunk at a time (issuing all raw loads of a k-tile
    // first and storing after the split measured no faster)
    const int lq = warp & 3, kh = warp >> 2;   // TMEM lane quarter, k-part of the rows
    const int m = lq * 32 + lane;
    const uint32_t lanebase = tmem + ((uint32_t)(lq * 32) << 16);
    // measurement aid (CGGM_TF32_DEBUG bit 1): hi = the fp32 bits unrounded, so lo = v - hi = 0 and
    // the MMA sees the raw operand (how the tensor core reads the 13 low bits)
    const uint32_t h_add = (P.dbg & 2) ? 0u : 0x1000u, h_mask = (P.dbg & 2) ? 0xFFFFFFFFu : 0xFFFFE000u;
    for (int it = 0; it < nkt; ++it) {
      const int s = it % TS_NS, rs = it % TS_NRAW;
      ptx::mbar_wait(&rfull[rs], (it / TS_NRAW) & 1);
      if (it >= TS_NS) {
        if (cf_rel) {   // the previous use of this stage lies in chunk cp: its completion frees the stage
          const int cp = (it - TS_NS) / CH;
          ptx::mbar_wait(&cfull[cp & 1], (cp >> 1) & 1);
        } else {
          ptx::mbar_wait(&empty[s], ((it / TS_NS) - 1) & 1);
        }
        tc_fence_after();
      }
      const uint32_t rw = rbase + rs * T_RAW;
      if (!(P.dbg & 4)) {   // (bit 2: measurement aid -- skip the split and the stores; garbage product)
      if (TS_KH == 1) {
        float v[32];
        raw_a_row<AK, 32>(rw, m, v);
        uint32_t h[32], l[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          h[e] = (__float_as_uint(v[e]) + h_add) & h_mask;
          l[e] = lo_tf32(v[e], h[e]);
        }
        const uint32_t ac = lanebase + 256u + (uint32_t)s * 64u;
        tmem_st32_nowait(ac, h);
        tmem_st32_nowait(ac + 32u, l);
      } else {   // this warp's 16 of the row's 32 k: hi at columns 16 kh .., lo at 32 + 16 kh ..
        float v[16];
        raw_a_row<AK, 16>(rw, m, v, 16 * kh);
        uint32_t h[16], l[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          h[e] = (__float_as_uint(v[e]) + h_add) & h_mask;
          l[e] = lo_tf32(v[e], h[e]);
        }
        const uint32_t ac = lanebase + 256u + (uint32_t)s * 64u + 16u * (uint32_t)kh;
        tmem_st16_nowait(ac, h);
        tmem_st16_nowait(ac + 32u, l);
      }
      const uint32_t st = sbase + s * TS_BSTAGE;
#pragma unroll
      for (int i = 0; i < TS_BPER; ++i) {
        float vb[4];
        uint32_t hb[4], lb[4];
        raw_b_chunk<BKI, TS_CONV>(rw + T_OP, vb, tid, i);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          hb[e] = (__float_as_uint(vb[e]) + h_add) & h_mask;
          lb[e] = lo_tf32(vb[e], hb[e]);
        }
        store_b_chunk<BKI, TS_CONV>(hb, lb, st, st + T_OP, tid, i);
      }
      }
      asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      tc_fence_before();
      ptx::mbar_arrive(&full[s]);
      ptx::mbar_arrive(&rempty[rs]);
    }
  };
  auto drain_role = [&]() {
    // ---- drain warps 4-7: chunk partials (TMEM X0 / X1) added into fp32 registers, then the epilogue
    const int dt = tid - TS_CONV;
    const int row = (warp - TS_DW0) * 32 + lane;
    const uint32_t lanebase = tmem + ((uint32_t)((warp - TS_DW0) * 32) << 16);
    float acc[TBN];
#pragma unroll
    for (int j = 0; j < TBN; ++j) acc[j] = 0.f;
    const int nch = nkt > 0 ? (nkt + CH - 1) / CH : 0;
    for (int c = 0; c < nch; ++c) {
      ptx::mbar_wait(&cfull[c & 1], (c >> 1) & 1);
      tc_fence_after();
      const uint32_t xa = lanebase + ((c & 1) ? 128u : 0u);
      if (!(P.dbg & 8)) {   // (bit 3: measurement aid -- no drain)
#pragma unroll
        for (int g = 0; g < TBN / 32; g += 2) {   // two loads per wait: half the exposed TMEM latency
          uint32_t v[32], w[32];
          tmem_ld32_nowait(xa + 32u * g, v);
          tmem_ld32_nowait(xa + 32u * (g + 1), w);
          tmem_wait_ld64(v, w);
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            acc[32 * g + j] += __uint_as_float(v[j]);
            acc[32 * (g + 1) + j] += __uint_as_float(w[j]);
          }
        }
      }
      tc_fence_before();
      ptx::mbar_arrive(&cempty[c & 1]);
    }
    if (nkt > 0) {
      ptx::mbar_wait(accf, 0);   // every MMA done: the shared stage buffers are free for the tile
      tc_fence_after();
    }
    float* Cs = reinterpret_cast<float*>(smem);
#pragma unroll
    for (int j = 0; j < TBN; ++j) Cs[j * T_EPI_LD + row] = acc[j];
    asm volatile("bar.sync 1, %0;\n" ::"n"(T_DRAIN) : "memory");
    const bool diag = (P.flags & SYM_LOWER) && I == J;
    for (int idx = dt; idx < TBM * TBN; idx += T_DRAIN) {
      const int mm = idx % TBM, nl = idx / TBM;
      const int mr = m0 + mm, n = n0 + nl;
      if (mr >= P.M || n >= P.N) continue;
      if (diag && mr < n) continue;
      epi_apply_t(P.epi, mr, n, Cs[nl * T_EPI_LD + mm]);
    }
    if (P.flags & SYM_MIRROR) {
      for (int idx = dt; idx < TBM * TBN; idx += T_DRAIN) {
        const int nl = idx % TBN, mm = idx / TBN;
        const int mr = m0 + mm, n = n0 + nl;
        if (mr >= P.M || n >= P.N) continue;
        if (diag && mr <= n) continue;
        epi_mirror_t(P.epi, n, mr, Cs[nl * T_EPI_LD + mm]);
      }
    }
  };
  if (CGGM_TS_CONV8) {
    // registers by warpgroup (each setmaxnreg executed by its whole warpgroup at one point, the role's
    // code dominated by it): converters 96, drain 232, MMA / TMA / two idle warps 40
    const int wg = warp >> 2;
    if (wg < 2) {
      asm volatile("setmaxnreg.dec.sync.aligned.u32 96;\n" ::: "memory");
      conv_role();
    } else if (wg == 2) {
      asm volatile("setmaxnreg.inc.sync.aligned.u32 232;\n" ::: "memory");
      drain_role();
    } else {
      asm volatile("setmaxnreg.dec.sync.aligned.u32 40;\n" ::: "memory");
      if (warp == TS_MMA) mma_role();
      else if (warp == TS_TMAW) tma_role();
    }
  } else if (warp == TS_MMA) {
    mma_role();
  } else if (warp == TS_TMAW) {
    tma_role();
  } else if (warp < TS_DW0) {
    conv_role();
  } else {
    drain_role();
  }
  __syncthreads();
  if (warp == TS_MMA) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(T_TMEM_COLS) : "memory");
  }
}

template <bool AK, bool BKI>
void launch_ts(Ctx* c, const CUtensorMap& ma, const CUtensorMap& mb, const KParamsT& P, int grid) {
  CGGM_ONCE_PER_DEVICE({
    CGGM_CUDA_CHECK(cudaFuncSetAttribute(gemm_tf32x3_ts_kernel<AK, BKI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         TS_SMEM));
  });
  Prof pr(c, c->cur_tag);
  gemm_tf32x3_ts_kernel<AK, BKI><<<grid, TS_NT, TS_SMEM, c->stream>>>(ma, mb, P);
  post_launch(c, "gemm_tf32x3_ts_kernel");
}

template <bool AK, bool BKI, bool TMA>
void launch_t(Ctx* c, const CUtensorMap& ma, const CUtensorMap& mb, const KParamsT& P, int grid) {
  using C = TCfg<TMA>;
  CGGM_ONCE_PER_DEVICE({
    CGGM_CUDA_CHECK(cudaFuncSetAttribute(gemm_tf32x3_kernel<AK, BKI, TMA>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         C::SMEM));
  });
  Prof pr(c, c->cur_tag);
  gemm_tf32x3_kernel<AK, BKI, TMA><<<grid, C::NT, C::SMEM, c->stream>>>(ma, mb, P);
  post_launch(c, "gemm_tf32x3_kernel");
}

}  // namespace

// Operands 16-byte aligned with ld % 4 == 0 (gemm_f32.cu packs others first) and their TMA maps (the
// FFMA engine's: K-inner {32, 128} boxes, MN-inner 3-D {32, 32, 4} or 2-D {32, 32}); same contract as
// gemm().
void gemm_tf32x3(Ctx* c, bool transA, bool transB, int64_t M, int64_t N, int64_t K, const float* A, int64_t lda,
                 const float* B, int64_t ldb, const EpilogueT<float>& epi, int flags, const CUtensorMap& ma,
                 const CUtensorMap& mb, int a3d, int b3d) {
  KParamsT P;
  P.M = (int)M; P.N = (int)N; P.K = (int)(K > 0 ? K : 0);
  P.flags = flags;
  P.A = A; P.lda = lda; P.B = B; P.ldb = ldb;
  P.chunk = c->tf32_chunk;
  P.dbg = c->tf32_dbg;
  P.cfrel = c->tf32_cfrel;
  P.a3d = a3d; P.b3d = b3d;
  P.epi = epi;
  P.tilesM = (int)((M + TBM - 1) / TBM);
  P.tilesN = (int)((N + TBN - 1) / TBN);
  const int grid = (flags & SYM_LOWER) ? P.tilesN * (P.tilesN + 1) / 2 + (P.tilesM - P.tilesN) * P.tilesN
                                       : P.tilesM * P.tilesN;
  const bool AK = transA, BKI = !transB, tma = c->tf32_producer == 0, ts = c->tf32_producer == 2;
  if (ts) P.chunk = c->tf32_ts_chunk;   // the TS form accumulates all three products per chunk: shorter chunks
#define CGGM_TF32_LAUNCH(a, b)                                     \
  if (ts) launch_ts<a, b>(c, ma, mb, P, grid);                     \
  else if (tma) launch_t<a, b, true>(c, ma, mb, P, grid);          \
  else launch_t<a, b, false>(c, ma, mb, P, grid);
  if (AK && BKI) { CGGM_TF32_LAUNCH(true, true) }
  else if (AK && !BKI) { CGGM_TF32_LAUNCH(true, false) }
  else if (!AK && BKI) { CGGM_TF32_LAUNCH(false, true) }
  else { CGGM_TF32_LAUNCH(false, false) }
#undef CGGM_TF32_LAUNCH
}

}  // namespace cggm
