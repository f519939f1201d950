// FP64 tensor-pipe GEMM for sm_100a: TMA (128B swizzle) -> shared memory ring with mbarrier
// full/empty pipeline -> mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4, the only FP64 tensor op on
// sm_100a; tcgen05 has no f64 kind).  One producer warp issues TMA, 8 consumer warps run a
// 128x128 CTA tile (warp tile 64x32).  Triangular operands shrink the k-range per tile
// (flags), symmetric outputs compute only lower tiles and mirror bit-identically.
//
// Used for every dense contraction of the hot path: S_yy = Y^T Y/n,
// S_xy = X^T Y/n, W Sigma, Psi = R^T R, X^T E (Eq. 3 via I3), and
// the blocked Cholesky / triangular-inverse / Sigma = L^{-T} L^{-1} updates.
//
// Shared-memory layouts (both operands, per stage, 16 KB each):
//  K-inner  (operand stored with k contiguous): 128 rows (x) x 128 B (16 k), TMA box {16,128}.
//  MN-inner (operand stored with x contiguous): 8 boxes {16 x, 16 k}, each 16 rows (k) x 128 B.
// TMA SWIZZLE_128B XORs the 16-byte chunk index with (row & 7).  The fragment mapping below
// is chosen so that every LDS.128 of a quarter-warp hits 8 distinct chunks (conflict-free):
//  k inside a 16-wide k tile: step (kk, s), lane t  ->  k = 8*kk + 2*t + s     (both operands)
//  MN-inner fragment pair p, element e, lane g     ->  x = 16*p + 2*g + e
//  K-inner fragment f, lane g                       ->  x = 8*f + (g>>1) + 4*(g&1)
// The epilogue inverts the same maps.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"

namespace cggm {
namespace {

#ifndef CGGM_BIG_MAXNREG
#define CGGM_BIG_MAXNREG 192
#endif
constexpr int BK = 16;
#ifndef CGGM_WS
#define CGGM_WS 1
#endif
#ifndef CGGM_MID_CTAS
#define CGGM_MID_CTAS 2
#endif
constexpr int STAGES = 4;
constexpr int GROUP_N = 8;
#ifndef CGGM_SYM_BAND
#define CGGM_SYM_BAND 8
#endif
constexpr int SYM_BAND = CGGM_SYM_BAND;   // tile rows per band of a SYM_LOWER raster

// CTA tile BM_ x BN_ computed by WM_ x WN_ warps (warp tile (BM_/WM_) x (BN_/WN_), fragments of 8)
template <int BM_, int BN_, int WM_, int WN_>
struct Cfg {
  static constexpr int BM = BM_, BN = BN_, WM = WM_, WN = WN_;
  static constexpr int NTHREADS = WM * WN * 32;
  static constexpr int WTM = BM / WM, WTN = BN / WN;
  static constexpr int FM = WTM / 8, FN = WTN / 8;
  static constexpr int A_BYTES = BM * BK * 8, B_BYTES = BN * BK * 8;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int EPI_LD = BM + 1;
  static constexpr int EPI_BYTES = BN * EPI_LD * 8;
  static constexpr int MAIN_BYTES = STAGES * STAGE_BYTES;
  static constexpr int DATA_BYTES = MAIN_BYTES > EPI_BYTES ? MAIN_BYTES : EPI_BYTES;
  // after the ring: full / empty barriers, the K01 bitmap barrier, then the K01 stored / negative
  // bitmaps of the tile (BM / 32 words per column each), built during the main loop
  static constexpr int BAR_BYTES = (2 * STAGES + 2) * 8;
  static constexpr int SEL_BYTES = BM * BN / 4;
  static constexpr int SMEM_BYTES = DATA_BYTES + 1024 + BAR_BYTES + SEL_BYTES;
  // register cap: a 128x128 CTA (8 warps x 192) leaves 16384 registers and ~95 KB of shared memory
  // on its SM, exactly one 64x64 CTA (4 warps x 128), so latency-bound kernels of a concurrent
  // stream co-reside with the big tiles instead of waiting for a whole SM
  static constexpr int MAXREG = (WTM >= 64 && WTN >= 32) ? CGGM_BIG_MAXNREG : 128;
  // warp specialisation (the big-warp-tile configurations): a producer warpgroup streams the TMA
  // k-tiles and donates its registers (setmaxnreg 40), the consumer warpgroups run the DMMA main
  // loop and the epilogue at up to 232 registers; no consumer warp ever waits on a ring slot
  static constexpr bool WSP = CGGM_WS && (WTM >= 64 && WTN >= 32);
  static constexpr int LB_THREADS = NTHREADS + (WSP ? 128 : 0);
  // a warp-specialised 4-consumer-warp tile (128x64) runs two CTAs per SM: 2 x 256 threads x 128
  // registers at launch; the consumers raise to 216 with what the producer warpgroup donates
  static constexpr int LB_MINB = WSP ? (NTHREADS == 128 ? CGGM_MID_CTAS : 1) : 65536 / (NTHREADS * MAXREG);
  static constexpr int CONS_REG = (WSP && NTHREADS == 128 && CGGM_MID_CTAS == 2) ? 216 : 232;
  static_assert(FM % 2 == 0 && FN % 2 == 0, "MN-inner fragments come in pairs");
  static_assert(BM % 16 == 0 && BN % 16 == 0, "16-wide TMA boxes");
};
using CfgBig = Cfg<128, 128, 2, 4>;    // 8 warps, warp tile 64 x 32
using CfgSmall = Cfg<64, 64, 2, 2>;    // 4 warps, warp tile 32 x 32
using CfgMid = Cfg<128, 64, 2, 2>;     // 4 warps, warp tile 64 x 32: two CTAs per SM, so one's
                                       // prologue / epilogue overlaps the other's main loop

struct KParams {
  int M, N, K;
  int tilesM, tilesN;
  int flags;
  int a3d, b3d;  // MN-inner operand: tiles inside the first a3d / b3d rows (a multiple of 16) load one
                 // 3-D TMA box; 0 = never (the ragged last tile uses 16-wide 2-D boxes of the second map)
  int vec;       // epilogue outputs / inputs 16-B aligned with even leading dimensions, no in1b / in2b:
                 // interior tiles take the paired (double2) epilogue
  int ksplit;    // 1, or 2 (SPLIT_K2): CTA 2t + h computes k-half h of tile t
  int sym_split; // SYM_LOWER with BN = BM / 2: the walk runs over BM x BM squares (tilesM / tilesN
                 // count squares), tile 2s + h is column half h of square s
  Epilogue epi;
};

// Tile order.  SYM_LOWER: the lower trapezoid {I >= J} of a tilesM x tilesN grid (M >= N),
// enumerated column-block by column-block from the right edge of the triangle.  Otherwise groups
// of GROUP_N tile columns (an A row panel is reused across the group while it sits in L2).
// Triangular k-ranges are scheduled longest-first (LPT) to shorten the tail wave.
__device__ __forceinline__ void tile_coords(const KParams& P, int t, int& I, int& J) {
  if (P.flags & SYM_LOWER) {
    const int half = P.sym_split == 2 ? (t & 1) : 0;
    if (P.sym_split == 2) t >>= 1;
    // lower triangle part (rows I < tilesN) in bands of SYM_BAND tile rows, band by band (I
    // ascending: longest k-ranges first for A_KGE_M / B_KGE_N), column by column inside a band:
    // the CTAs in flight share the band's row panels and each column panel, so the panels are read
    // from DRAM about once per band instead of once per tile
    const long long tri = (long long)P.tilesN * (P.tilesN + 1) / 2;
    if (t < tri) {
      long long L = t;
      int r0 = 0;
      for (;;) {
        const int h = min(SYM_BAND, P.tilesN - r0);
        const long long cnt = (long long)h * r0 + (long long)h * (h + 1) / 2;
        if (L < cnt) {
          if (L < (long long)h * r0) {
            J = (int)(L / h);
            I = r0 + (int)(L % h);
          } else {
            int l2 = (int)(L - (long long)h * r0), j = r0;
            while (l2 >= r0 + h - j) {
              l2 -= r0 + h - j;
              ++j;
            }
            J = j;
            I = j + l2;
          }
          break;
        }
        L -= cnt;
        r0 += h;
      }
    } else {
      const int r = t - (int)tri;  // rectangular part below: rows tilesN .. tilesM-1
      I = P.tilesN + r / P.tilesN;
      J = r % P.tilesN;
    }
    if (P.sym_split == 2) J = 2 * J + half;
    return;
  }
  const int per_group = GROUP_N * P.tilesM;
  const int gi = t / per_group;
  const int local = t - gi * per_group;
  const int nb0 = gi * GROUP_N;
  const int width = min(GROUP_N, P.tilesN - nb0);
  I = local / width;
  J = nb0 + local % width;
  if (P.flags & B_KLE_N) J = P.tilesN - 1 - J;   // k-range grows with J: start from the right
  if (P.flags & A_KLE_M) I = P.tilesM - 1 - I;   // k-range grows with I: start from the bottom
}

__device__ __forceinline__ void epi_apply(const Epilogue& E, int64_t r, int64_t c, double v) {
  if (E.out1) {
    double o = __dmul_rn(E.a1, v);
    if (E.in1a) o = __dadd_rn(o, __dmul_rn(E.b1, E.in1a[r + c * E.ld1a]));
    if (E.in1b) o = __dadd_rn(o, __dmul_rn(E.c1, E.in1b[r + c * E.ld1b]));
    E.out1[r + c * E.ld1] = o;
  }
  if (E.out2) {
    double o = __dmul_rn(E.a2, v);
    if (E.in2a) o = __dadd_rn(o, __dmul_rn(E.b2, E.in2a[r + c * E.ld2a]));
    if (E.in2b) o = __dadd_rn(o, __dmul_rn(E.c2, E.in2b[r + c * E.ld2b]));
    E.out2[r + c * E.ld2] = o;
  }
}

// the transposed copy of a SYM_MIRROR product: into the same output (symmetric square) or into
// E.mir1 (the off-diagonal block of a symmetric result; host-checked to have no inputs / out2)
__device__ __forceinline__ void epi_mirror(const Epilogue& E, int64_t r, int64_t c, double v) {
  if (E.mir1) E.mir1[r + c * E.ld1] = __dmul_rn(E.a1, v);
  else epi_apply(E, r, c, v);
}

// K01: the S_Theta selection on the staged tile Cs (BM x BN, column nl at Cs + nl * EPI_LD) of
// grad_Theta = a1 * acc, in place of the stores.  Same per-element decisions as the scan
// (k_active_vec): flag = in && (|g| - lam > 0 || stored nonzero), tie = in && !stored && ||g| - lam|
// <= tie_eps; subgradient |g + lam sign x| for a stored nonzero x, else max(|g| - lam, 0).  Warp w
// takes tile columns w, w + NW, ...; per column: the flag words (written), the count and tie count
// (atomic adds: integers, order-free), and the subgradient partial (fixed shuffle tree) at
// subpart[64-row chunk][column].  The stored entries of the tile's rows come from the Theta CSC into two
// shared bitmaps (sel_bits: stored; + BM / 32 * BN words: negative).
// the tile's stored-nonzero / negative bitmaps from the Theta CSC: thread t of nt owns tile columns
// t, t + nt, ... (their words only: no sharing, no zeroing pass)
template <int BM, int BN>
__device__ __forceinline__ void select_bitmaps(const KParams& P, uint32_t* sel_bits, int m0, int n0, int t, int nt) {
  const SelectT& S = P.epi.sel;
  constexpr int WPC = BM / 32;
  uint32_t* neg_bits = sel_bits + WPC * BN;
  for (int nl = t; nl < BN; nl += nt) {   // one thread per tile column: its stored rows in [m0, m0 + BM)
    uint32_t* sw = sel_bits + nl * WPC;
    uint32_t* nw = neg_bits + nl * WPC;
#pragma unroll
    for (int k = 0; k < WPC; ++k) sw[k] = nw[k] = 0u;
    const int64_t j = (int64_t)n0 + nl;
    if (j >= P.N) continue;
    int64_t lo = S.colptr[j], hi = S.colptr[j + 1];
    while (lo < hi) {   // first stored row >= m0
      const int64_t mid = (lo + hi) >> 1;
      if (S.rowidx[mid] < m0) lo = mid + 1;
      else hi = mid;
    }
    for (int64_t e = lo; e < S.colptr[j + 1]; ++e) {
      const int r = S.rowidx[e] - m0;
      if (r >= BM) break;
      const double x = S.val[e];
      if (x == 0.0) continue;
      sw[r >> 5] |= 1u << (r & 31);
      if (x < 0.0) nw[r >> 5] |= 1u << (r & 31);
    }
  }
}

// the selection itself, on the staged tile and the finished bitmaps
template <int BM, int BN, int NTHREADS, int EPI_LD>
__device__ __forceinline__ void select_epilogue(const KParams& P, const double* Cs, const uint32_t* sel_bits, int m0,
                                                int n0, int tid) {
  const SelectT& S = P.epi.sel;
  constexpr int WPC = BM / 32, NW = NTHREADS / 32;
  const uint32_t* neg_bits = sel_bits + WPC * BN;
  const int w = tid >> 5, lane = tid & 31;
  const double a1 = P.epi.a1, lam = S.lam, teps = S.tie_eps;
  // (measured: one column at a time with the cold-chunk vote, X^T E 45.7 -> 47.9 ms; four independent
  // (column, chunk) items at a time without the vote 49.0 ms -- the per-element work, not latency,
  // is what the store epilogue did not have)
  for (int nl = w; nl < BN; nl += NW) {
    const int64_t j = (int64_t)n0 + nl;
    if (j >= P.N) break;   // (columns ascend with nl)
    const double* cs = Cs + nl * EPI_LD;
#pragma unroll
    for (int c = 0; c < BM / 64; ++c) {
      const int64_t chunk = m0 / 64 + c;
      if (64 * chunk >= P.M) break;
      const int rl = 64 * c + 2 * lane;
      const int64_t r = (int64_t)m0 + rl;
      const bool in0 = r < P.M, in1 = r + 1 < P.M;
      const double g0 = __dmul_rn(a1, cs[rl]), g1 = __dmul_rn(a1, cs[rl + 1]);
      const uint32_t sw = sel_bits[nl * WPC + (rl >> 5)] >> (rl & 31);
      const uint32_t nw = neg_bits[nl * WPC + (rl >> 5)] >> (rl & 31);
      const bool sp0 = sw & 1u, sp1 = (sw >> 1) & 1u;
      const double d0 = fabs(g0) - lam, d1 = fabs(g1) - lam;
      // cold chunk (most chunks: 0.7% of grad_Theta is active at `large`): nothing within the tie band
      // or above the threshold, no stored nonzero -> zero words, no tie / subgradient share
      if (!__any_sync(0xffffffffu, (sw & 3u) || d0 >= -teps || d1 >= -teps)) {
        if (lane == 0) {
          *reinterpret_cast<uint2*>(S.flags + j * S.wpc + 2 * chunk) = make_uint2(0u, 0u);
          S.subpart[chunk * S.ldsub + j] = 0.0;
        }
        continue;
      }
      const bool f0 = in0 && (d0 > 0.0 || sp0), f1 = in1 && (d1 > 0.0 || sp1);
      const unsigned b0 = __ballot_sync(0xffffffffu, f0), b1 = __ballot_sync(0xffffffffu, f1);
      long long tc = (in0 && !sp0 && fabs(d0) <= teps) + (in1 && !sp1 && fabs(d1) <= teps);
      double sub = 0.0;
      if (in0) sub += sp0 ? fabs(g0 + ((nw & 1u) ? -lam : lam)) : fmax(d0, 0.0);
      if (in1) sub += sp1 ? fabs(g1 + ((nw & 2u) ? -lam : lam)) : fmax(d1, 0.0);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        sub += __shfl_down_sync(0xffffffffu, sub, o);
        tc += __shfl_down_sync(0xffffffffu, tc, o);
      }
      if (lane == 0) {
        *reinterpret_cast<uint2*>(S.flags + j * S.wpc + 2 * chunk) = make_uint2(b0, b1);
        const int cnt = __popc(b0) + __popc(b1);
        if (cnt) atomicAdd(S.cnt + j, (unsigned long long)cnt);
        if (tc) atomicAdd(reinterpret_cast<unsigned long long*>(S.ties + j), (unsigned long long)tc);
        S.subpart[chunk * S.ldsub + j] = sub;
      }
    }
  }
}

// x offset (within the warp's 64/32-wide slab) of fragment f, fragment row/col index r
template <bool KINNER>
__device__ __forceinline__ int frag_x(int f, int r) {
  if (KINNER) return 8 * f + (r >> 1) + 4 * (r & 1);
  return 16 * (f >> 1) + 2 * r + (f & 1);
}

template <bool AK, bool BKI, class C>
__global__ void __launch_bounds__(C::LB_THREADS, C::LB_MINB)
    gemm_dmma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ CUtensorMap tmA2, const __grid_constant__ CUtensorMap tmB2,
                     const KParams P) {
  constexpr int BM = C::BM, BN = C::BN, NCW = C::WM * C::WN, FM = C::FM, FN = C::FN;
  constexpr int OP_BYTES = C::A_BYTES, STAGE_BYTES = C::STAGE_BYTES, DATA_BYTES = C::DATA_BYTES;
  constexpr int EPI_LD = C::EPI_LD, NTHREADS = C::NTHREADS;
  constexpr bool WS = C::WSP;
  extern __shared__ uint8_t smem_raw[];
  ptx::pdl_wait();   // (launched with the PDL attribute: the predecessor's output is visible from here)
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + DATA_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* selbar = empty + STAGES;   // K01 bitmaps built (WS: producer warps 1-3)
  uint32_t* sel_bits = reinterpret_cast<uint32_t*>(smem + DATA_BYTES + C::BAR_BYTES);

  const int tid = (int)threadIdx.x - (WS ? 128 : 0);   // consumer thread index
  const int warp = tid >> 5, lane = threadIdx.x & 31;
  auto cbar = [&]() {   // barrier of the consumer threads
    if (WS) asm volatile("bar.sync 1, %0;\n" ::"n"(NTHREADS) : "memory");
    else __syncthreads();
  };
  int I, J;
  const int part = P.ksplit > 1 ? (int)(blockIdx.x % P.ksplit) : 0;
  tile_coords(P, P.ksplit > 1 ? (int)(blockIdx.x / P.ksplit) : (int)blockIdx.x, I, J);
  const int m0 = I * BM, n0 = J * BN;

  int kbeg = 0, kend = P.K;
  if (P.flags & A_KGE_M) kbeg = max(kbeg, m0);
  if (P.flags & B_KGE_N) kbeg = max(kbeg, n0);
  if (P.flags & A_KLE_M) kend = min(kend, m0 + BM);
  if (P.flags & B_KLE_N) kend = min(kend, n0 + BN);
  int kt0 = kbeg / BK;
  int nkt = kend > kbeg && n0 < P.N ? (kend - kt0 * BK + BK - 1) / BK : 0;   // (a split square's
  if (P.ksplit > 1) {                                                        //  half past N: no work)   // this CTA's share of the k-tiles
    const int per = (nkt + P.ksplit - 1) / P.ksplit;
    kt0 += part * per;
    nkt = max(0, min(per, nkt - part * per));
  }

  // ------------------------------------------------ TMA producer: thread 0, STAGES-1 tiles ahead
  uint32_t tx_bytes = 0;
  if (threadIdx.x == 0 && nkt > 0) {
    ptx::prefetch_tmap(&tmA);
    ptx::prefetch_tmap(&tmB);
  }
  // MN-inner operands: one 3-D box when the tile lies inside the 16-row-aligned extent, else
  // 16-wide 2-D boxes (rows past the extent are neither loaded nor used)
  // (with no ragged rows, a box past the extent only reads the map's zero fill along its 3rd dim)
  const bool a_one = !AK && P.a3d && (m0 + BM <= P.a3d || P.a3d == P.M);
  const bool b_one = !BKI && P.b3d && (n0 + BN <= P.b3d || P.b3d == P.N);
  int a_boxes = 0, b_boxes = 0;
  if (!AK && !a_one)
    for (int xb = 0; xb < BM / 16; ++xb) a_boxes += (m0 + xb * 16 < P.M);
  if (!BKI && !b_one)
    for (int xb = 0; xb < BN / 16; ++xb) b_boxes += (n0 + xb * 16 < P.N);
  tx_bytes = ((AK || a_one) ? C::A_BYTES : a_boxes * 2048) + ((BKI || b_one) ? C::B_BYTES : b_boxes * 2048);
  if (threadIdx.x == 0 && nkt > 0) {
    if (!AK && !a_one) ptx::prefetch_tmap(&tmA2);
    if (!BKI && !b_one) ptx::prefetch_tmap(&tmB2);
  }
  auto issue = [&](int i) {
    const int s = i % STAGES;
    uint8_t* sa = smem + s * STAGE_BYTES;
    uint8_t* sb = sa + OP_BYTES;
    ptx::mbar_arrive_expect_tx(&full[s], tx_bytes);
    const int k = (kt0 + i) * BK;
    if (AK) {
      ptx::tma_load_2d(sa, &tmA, &full[s], k, m0);
    } else if (a_one) {
      ptx::tma_load_3d(sa, &tmA, &full[s], 0, k, m0 / 16);
    } else {
      for (int xb = 0; xb < a_boxes; ++xb) ptx::tma_load_2d(sa + xb * 2048, &tmA2, &full[s], m0 + xb * 16, k);
    }
    if (BKI) {
      ptx::tma_load_2d(sb, &tmB, &full[s], k, n0);
    } else if (b_one) {
      ptx::tma_load_3d(sb, &tmB, &full[s], 0, k, n0 / 16);
    } else {
      for (int xb = 0; xb < b_boxes; ++xb) ptx::tma_load_2d(sb + xb * 2048, &tmB2, &full[s], n0 + xb * 16, k);
    }
  };
  // thread 0 initialises the ring barriers and issues the first STAGES-1 k-tiles before the block
  // barrier, so the loads are in flight while the other threads reach it
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], NCW);
    }
    ptx::mbar_init(selbar, 96);
    ptx::fence_barrier_init();
    for (int i = 0; i < STAGES - 1 && i < nkt; ++i) issue(i);
  }
  __syncthreads();
  if (WS) {
    if (threadIdx.x < 128) {   // producer warpgroup: 40 registers, thread 0 streams the k-tiles
      asm volatile("setmaxnreg.dec.sync.aligned.u32 40;\n" ::: "memory");
      if (threadIdx.x == 0) {
        for (int j = STAGES - 1; j < nkt; ++j) {
          if (j >= STAGES) ptx::mbar_wait(&empty[j % STAGES], ((j / STAGES) & 1) ^ 1);
          issue(j);
        }
      } else if (threadIdx.x >= 32 && P.epi.sel.on) {   // K01: warps 1-3 build the tile's bitmaps meanwhile
        select_bitmaps<BM, BN>(P, sel_bits, m0, n0, (int)threadIdx.x - 32, 96);
        ptx::mbar_arrive(selbar);
      }
      return;
    }
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(C::CONS_REG) : "memory");
  }

  double acc[FM][FN][2];
#pragma unroll
  for (int a = 0; a < FM; ++a)
#pragma unroll
    for (int b = 0; b < FN; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

  const int g = lane >> 2, t = lane & 3;
  const int wm = warp / C::WN, wn = warp % C::WN;
  const int xa0 = wm * C::WTM, xb0 = wn * C::WTN;

  {
    // ------------------------------------------------ DMMA consumers
    for (int i = 0; i < nkt; ++i) {
      const int s = i % STAGES;
      ptx::mbar_wait(&full[s], (i / STAGES) & 1);
      const uint32_t sa = ptx::smem_u32(smem + s * STAGE_BYTES);
      const uint32_t sb = sa + OP_BYTES;
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) {
        double a[FM][2], b[FN][2];
        if (AK) {
#pragma unroll
          for (int f = 0; f < FM; ++f) {
            const int x = xa0 + frag_x<true>(f, g);
            const int chunk = (4 * kk + t) ^ (x & 7);
            ptx::lds128(a[f][0], a[f][1], sa + x * 128 + chunk * 16);
          }
        } else {
#pragma unroll
          for (int pr = 0; pr < FM / 2; ++pr) {
            const int xb = xa0 / 16 + pr;
#pragma unroll
            for (int s2 = 0; s2 < 2; ++s2) {
              const int k = 8 * kk + 2 * t + s2;
              const int chunk = g ^ (k & 7);
              ptx::lds128(a[2 * pr][s2], a[2 * pr + 1][s2], sa + xb * 2048 + k * 128 + chunk * 16);
            }
          }
        }
        if (BKI) {
#pragma unroll
          for (int f = 0; f < FN; ++f) {
            const int x = xb0 + frag_x<true>(f, g);
            const int chunk = (4 * kk + t) ^ (x & 7);
            ptx::lds128(b[f][0], b[f][1], sb + x * 128 + chunk * 16);
          }
        } else {
#pragma unroll
          for (int pr = 0; pr < FN / 2; ++pr) {
            const int xb = xb0 / 16 + pr;
#pragma unroll
            for (int s2 = 0; s2 < 2; ++s2) {
              const int k = 8 * kk + 2 * t + s2;
              const int chunk = g ^ (k & 7);
              ptx::lds128(b[2 * pr][s2], b[2 * pr + 1][s2], sb + xb * 2048 + k * 128 + chunk * 16);
            }
          }
        }
#pragma unroll
        for (int s2 = 0; s2 < 2; ++s2)
#pragma unroll
          for (int fm = 0; fm < FM; ++fm)
#pragma unroll
            for (int fn = 0; fn < FN; ++fn) ptx::dmma_8x8x4(acc[fm][fn][0], acc[fm][fn][1], a[fm][s2], b[fn][s2]);
      }
      __syncwarp();
      // the stage's generic-proxy reads (ld.shared) are ordered before the TMA (async proxy) that
      // refills it once every consumer warp has arrived: without this proxy fence the refill could
      // overwrite data still being read (observed: corrupted warp tiles when an HBM-streaming kernel
      // ran beside the warp-specialised 128x64 tiles, tools/debug/gl_race.py)
      ptx::fence_proxy_async();
      if (lane == 0) ptx::mbar_arrive(&empty[s]);
      if (!WS && threadIdx.x == 0) {
        const int j = i + STAGES - 1;
        if (j < nkt) {
          if (j >= STAGES) ptx::mbar_wait(&empty[j % STAGES], ((j / STAGES) & 1) ^ 1);
          issue(j);
        }
      }
    }
  }

  // ------------------------------------------------ epilogue through shared memory
  // every CTA of the grid has been scheduled once this one reaches its epilogue: the successor's CTAs
  // may be scheduled when all have (it still waits for this grid's completion in pdl_wait)
  if (tid == 0) ptx::pdl_trigger();
  cbar();
  double* Cs = reinterpret_cast<double*>(smem);
  {
#pragma unroll
    for (int fm = 0; fm < FM; ++fm) {
      const int ml = xa0 + frag_x<AK>(fm, g);
#pragma unroll
      for (int fn = 0; fn < FN; ++fn)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int nl = xb0 + frag_x<BKI>(fn, 2 * t + j);
          Cs[nl * EPI_LD + ml] = acc[fm][fn][j];
        }
    }
  }
  cbar();
  if (P.epi.sel.on) {   // K01: select instead of storing
    if (WS) {
      ptx::mbar_wait(selbar, 0);
    } else {
      select_bitmaps<BM, BN>(P, sel_bits, m0, n0, tid, NTHREADS);
      cbar();
    }
    select_epilogue<BM, BN, NTHREADS, EPI_LD>(P, Cs, sel_bits, m0, n0, tid);
    return;
  }
  const bool diag = (P.flags & SYM_LOWER) && m0 < n0 + BN;   // the tile reaches above the diagonal
  if (P.ksplit > 1) {   // partial sum of this k-half into out1 (zeros + two partials: order-free)
    for (int idx = tid; idx < BM * BN; idx += NTHREADS) {
      const int ml = idx % BM, nl = idx / BM;
      const int m = m0 + ml, n = n0 + nl;
      if (m >= P.M || n >= P.N) continue;
      atomicAdd(P.epi.out1 + m + (int64_t)n * P.epi.ld1, __dmul_rn(P.epi.a1, Cs[nl * EPI_LD + ml]));
    }
    return;
  }
  if (P.vec && !diag && m0 + BM <= P.M && n0 + BN <= P.N) {
    // interior tile: thread = row pair x column group, 16-B global accesses, the inputs of U
    // columns loaded before any is used (one memory round trip per U columns, not per element);
    // per element the same arithmetic as epi_apply
    constexpr int RP = BM / 2, CG = NTHREADS / RP, NCOL = BN / CG, U = 8;
    const Epilogue& E = P.epi;
    const int ml = 2 * (tid % RP), cg = tid / RP;
    const int64_t m = m0 + ml;
#pragma unroll 1
    for (int i0 = 0; i0 < NCOL; i0 += U) {
      double2 x1[U], x2[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t n = n0 + cg + CG * (i0 + u);
        if (E.in1a) x1[u] = *reinterpret_cast<const double2*>(E.in1a + m + n * E.ld1a);
        if (E.in2a) x2[u] = *reinterpret_cast<const double2*>(E.in2a + m + n * E.ld2a);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int nl = cg + CG * (i0 + u);
        const int64_t n = n0 + nl;
        const double v0 = Cs[nl * EPI_LD + ml], v1 = Cs[nl * EPI_LD + ml + 1];
        if (E.out1) {
          double2 o = make_double2(__dmul_rn(E.a1, v0), __dmul_rn(E.a1, v1));
          if (E.in1a) {
            o.x = __dadd_rn(o.x, __dmul_rn(E.b1, x1[u].x));
            o.y = __dadd_rn(o.y, __dmul_rn(E.b1, x1[u].y));
          }
          *reinterpret_cast<double2*>(E.out1 + m + n * E.ld1) = o;
        }
        if (E.out2) {
          double2 o = make_double2(__dmul_rn(E.a2, v0), __dmul_rn(E.a2, v1));
          if (E.in2a) {
            o.x = __dadd_rn(o.x, __dmul_rn(E.b2, x2[u].x));
            o.y = __dadd_rn(o.y, __dmul_rn(E.b2, x2[u].y));
          }
          if (E.in2b) {   // (only the Psi GEMM's grad_Lambda output has a second input: loaded here)
            const double2 x4 = *reinterpret_cast<const double2*>(E.in2b + m + n * E.ld2b);
            o.x = __dadd_rn(o.x, __dmul_rn(E.c2, x4.x));
            o.y = __dadd_rn(o.y, __dmul_rn(E.c2, x4.y));
          }
          *reinterpret_cast<double2*>(E.out2 + m + n * E.ld2) = o;
        }
      }
    }
  } else {
    for (int idx = tid; idx < BM * BN; idx += NTHREADS) {
      const int ml = idx % BM, nl = idx / BM;
      const int m = m0 + ml, n = n0 + nl;
      if (m >= P.M || n >= P.N) continue;
      if (diag && m < n) continue;
      epi_apply(P.epi, m, n, Cs[nl * EPI_LD + ml]);
    }
  }
  if (P.flags & SYM_MIRROR) {
    if (P.vec && !diag && m0 + BM <= P.M && n0 + BN <= P.N) {
      // transposed copy: lane l of a warp reads row nl = nb + l of the staged tile at columns ml and
      // ml + 1 (consecutive lanes 129 doubles apart: conflict-free), then lane pairs swap one value
      // so that the even lane stores (nl, nl + 1) of output column ml and the odd lane those of
      // column ml + 1, 16 bytes each, contiguous along the output rows
      constexpr int NWARPS = NTHREADS / 32, NBLK = BN / 32, GROUPS = NWARPS / NBLK, PAIRS = BM / 2 / GROUPS;
      static_assert(NWARPS % NBLK == 0 && (BM / 2) % GROUPS == 0, "mirror epilogue warp layout");
      const Epilogue& E = P.epi;
      const int wv = tid >> 5, ln = tid & 31;
      const int nl = 32 * (wv % NBLK) + ln, grp = wv / NBLK;
      const bool odd = ln & 1;
      const int64_t n = n0 + nl - (odd ? 1 : 0);
#pragma unroll 4
      for (int i = 0; i < PAIRS; ++i) {
        const int ml = 2 * (grp + GROUPS * i);
        const double a = Cs[nl * EPI_LD + ml], b = Cs[nl * EPI_LD + ml + 1];
        const double pa = __shfl_xor_sync(0xffffffffu, a, 1), pb = __shfl_xor_sync(0xffffffffu, b, 1);
        const double lo = odd ? pb : a, hi = odd ? b : pa;   // rows (n, n + 1) of output column m
        const int64_t m = m0 + ml + (odd ? 1 : 0);
        if (E.out1) {
          double2 o = make_double2(__dmul_rn(E.a1, lo), __dmul_rn(E.a1, hi));
          if (E.in1a) {   // in-place accumulation: the input at the written (transposed) position
            const double2 x = *reinterpret_cast<const double2*>(E.in1a + n + m * E.ld1a);
            o.x = __dadd_rn(o.x, __dmul_rn(E.b1, x.x));
            o.y = __dadd_rn(o.y, __dmul_rn(E.b1, x.y));
          }
          *reinterpret_cast<double2*>((E.mir1 ? E.mir1 : E.out1) + n + m * E.ld1) = o;
        }
        if (E.out2) {
          double2 o = make_double2(__dmul_rn(E.a2, lo), __dmul_rn(E.a2, hi));
          if (E.in2a) {   // the inputs at the written (transposed) position: contiguous along n
            const double2 x = *reinterpret_cast<const double2*>(E.in2a + n + m * E.ld2a);
            o.x = __dadd_rn(o.x, __dmul_rn(E.b2, x.x));
            o.y = __dadd_rn(o.y, __dmul_rn(E.b2, x.y));
          }
          if (E.in2b) {
            const double2 x = *reinterpret_cast<const double2*>(E.in2b + n + m * E.ld2b);
            o.x = __dadd_rn(o.x, __dmul_rn(E.c2, x.x));
            o.y = __dadd_rn(o.y, __dmul_rn(E.c2, x.y));
          }
          *reinterpret_cast<double2*>(E.out2 + n + m * E.ld2) = o;
        }
      }
    } else {
      for (int idx = tid; idx < BM * BN; idx += NTHREADS) {
        const int nl = idx % BN, ml = idx / BN;
        const int m = m0 + ml, n = n0 + nl;
        if (m >= P.M || n >= P.N) continue;
        if (diag && m <= n) continue;
        epi_mirror(P.epi, n, m, Cs[nl * EPI_LD + ml]);
      }
    }
  }
}

// MN-inner operand as a 3-D tensor {16 (x mod 16), K, X/16} with strides {ld*8, 128 B}: one TMA box
// {16, 16, BX/16} fills the whole [x/16][k][x%16] tile.  Only when X % 16 == 0 (no read past X).
// ------------------------------------------------------------------ small-shape GEMM
// K <= 256 and min(M, N) <= 128 (the bottom of the Cholesky recursion: 64x64x64 products and
// 64-column panel solves): latency, not throughput, bound.  32x32 CTA tiles (4x the CTAs of a
// 64-tile), 4 warps with 16x16 warp tiles of DMMA.8x8x4, operands loaded directly with coalesced
// global loads into padded shared memory (no tensor-map fetch / mbarrier prologue), the same
// flags and epilogue semantics as the TMA kernels.
constexpr int ST = 32;        // tile
constexpr int SKC = 32;       // k chunk
constexpr int SLD = ST + 4;   // padded row (conflict-free half-warp DMMA fragment loads)

struct KParamsS {
  int M, N, K, flags;
  Epilogue epi;
};

template <bool TA, bool TB>
__global__ void __launch_bounds__(128) gemm_small_kernel(const double* __restrict__ A, int64_t lda,
                                                          const double* __restrict__ B, int64_t ldb,
                                                          const KParamsS P) {
  // double-buffered shared tiles; chunk i+1 is fetched into registers while chunk i is multiplied,
  // so each chunk costs one L2 round trip overlapped with the DMMAs and one barrier
  __shared__ double As[2][SKC][SLD];
  __shared__ double Bs[2][SKC][SLD];
  ptx::pdl_wait();
  ptx::pdl_trigger();
  const int m0 = blockIdx.y * ST, n0 = blockIdx.x * ST;
  if ((P.flags & SYM_LOWER) && m0 + ST - 1 < n0) return;   // tile strictly above the diagonal
  int kbeg = 0, kend = P.K;
  if (P.flags & A_KGE_M) kbeg = max(kbeg, m0);
  if (P.flags & B_KGE_N) kbeg = max(kbeg, n0);
  if (P.flags & A_KLE_M) kend = min(kend, m0 + ST);
  if (P.flags & B_KLE_N) kend = min(kend, n0 + ST);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int wm = warp >> 1, wn = warp & 1;
  constexpr int PER = ST * SKC / 128;   // elements of each operand per thread and chunk
  double ra[PER], rb[PER];
  // consecutive threads walk the contiguous dimension of each operand
  auto fetch = [&](int kc) {
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int idx = tid + 128 * u;
      int mm, kk;
      if (TA) { kk = idx % SKC; mm = idx / SKC; } else { mm = idx % ST; kk = idx / ST; }
      const int m = m0 + mm, k = kc + kk;
      ra[u] = (m < P.M && k < kend) ? (TA ? A[k + (int64_t)m * lda] : A[m + (int64_t)k * lda]) : 0.0;
      int nn, k2;
      if (TB) { nn = idx % ST; k2 = idx / ST; } else { k2 = idx % SKC; nn = idx / SKC; }
      const int n = n0 + nn, kb = kc + k2;
      rb[u] = (n < P.N && kb < kend) ? (TB ? B[n + (int64_t)kb * ldb] : B[kb + (int64_t)n * ldb]) : 0.0;
    }
  };
  auto stash = [&](int buf) {
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int idx = tid + 128 * u;
      int mm, kk;
      if (TA) { kk = idx % SKC; mm = idx / SKC; } else { mm = idx % ST; kk = idx / ST; }
      As[buf][kk][mm] = ra[u];
      int nn, k2;
      if (TB) { nn = idx % ST; k2 = idx / ST; } else { k2 = idx % SKC; nn = idx / SKC; }
      Bs[buf][k2][nn] = rb[u];
    }
  };
  double acc[2][2][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  if (kbeg < kend) {
    fetch(kbeg);
    stash(0);
    __syncthreads();
    int buf = 0;
    for (int kc = kbeg; kc < kend; kc += SKC) {
      const bool more = kc + SKC < kend;
      if (more) fetch(kc + SKC);
#pragma unroll
      for (int k4 = 0; k4 < SKC / 4; ++k4) {
        double a[2], b[2];
#pragma unroll
        for (int f = 0; f < 2; ++f) {
          a[f] = As[buf][4 * k4 + t][16 * wm + 8 * f + g];
          b[f] = Bs[buf][4 * k4 + t][16 * wn + 8 * f + g];
        }
#pragma unroll
        for (int fm = 0; fm < 2; ++fm)
#pragma unroll
          for (int fn = 0; fn < 2; ++fn) ptx::dmma_8x8x4(acc[fm][fn][0], acc[fm][fn][1], a[fm], b[fn]);
      }
      if (more) stash(buf ^ 1);   // the other buffer was last read before the previous barrier
      __syncthreads();
      buf ^= 1;
    }
  }
#pragma unroll
  for (int fm = 0; fm < 2; ++fm)
#pragma unroll
    for (int fn = 0; fn < 2; ++fn)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int m = m0 + 16 * wm + 8 * fm + g, n = n0 + 16 * wn + 8 * fn + 2 * t + j;
        if (m >= P.M || n >= P.N) continue;
        if ((P.flags & SYM_LOWER) && m < n) continue;
        epi_apply(P.epi, m, n, acc[fm][fn][j]);
        if ((P.flags & SYM_MIRROR) && (m > n || P.epi.mir1)) epi_mirror(P.epi, n, m, acc[fm][fn][j]);
      }
}

// Same tile / flags / epilogue, operands streamed by cp.async through a 4-stage shared ring (the
// whole k-range of a CTA is in flight after the prologue): the latency of a K <= 256 product is
// about one L2 round trip plus its DMMAs.  Shared tiles keep the global contiguity of each operand
// (rows of SLD = 36 doubles: conflict-free fragment reads for either orientation).  Needs 16-byte
// aligned operands with even leading dimensions; gemm() falls back to gemm_small_kernel otherwise.
constexpr int SA_STAGES = 4;
constexpr int SA_TILE = ST * SLD;                              // doubles per operand tile
constexpr int SA_SMEM = SA_STAGES * 2 * SA_TILE * 8;

template <bool TA, bool TB>
__global__ void __launch_bounds__(128) gemm_small_async_kernel(const double* __restrict__ A, int64_t lda,
                                                                const double* __restrict__ B, int64_t ldb,
                                                                const KParamsS P) {
  extern __shared__ __align__(16) double sa_smem[];
  ptx::pdl_wait();
  ptx::pdl_trigger();   // (at most a wave of CTAs: the successor's CTAs queue behind this grid's)
  const int m0 = blockIdx.y * ST, n0 = blockIdx.x * ST;
  if ((P.flags & SYM_LOWER) && m0 + ST - 1 < n0) return;   // tile strictly above the diagonal
  int kbeg = 0, kend = P.K;
  if (P.flags & A_KGE_M) kbeg = max(kbeg, m0);
  if (P.flags & B_KGE_N) kbeg = max(kbeg, n0);
  if (P.flags & A_KLE_M) kend = min(kend, m0 + ST);
  if (P.flags & B_KLE_N) kend = min(kend, n0 + ST);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int wm = warp >> 1, wn = warp & 1;
  const int nchunks = kend > kbeg ? (kend - kbeg + SKC - 1) / SKC : 0;
  // operand X (rows x of extent XN, ld) in its stored orientation: KROWS = k is the strided index
  // (tile [k][x], x contiguous), else x is strided (tile [x][k], k contiguous)
  auto issue = [&](int chunk) {
    const int kc = kbeg + chunk * SKC;
    double* as = sa_smem + (chunk % SA_STAGES) * 2 * SA_TILE;
    double* bs = as + SA_TILE;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int pidx = tid + 128 * u, row = pidx >> 4, c2 = 2 * (pidx & 15);
      {  // A: !TA -> tile [k][m] (m contiguous); TA -> tile [m][k] (k contiguous)
        const int k = TA ? kc + c2 : kc + row, m = TA ? m0 + row : m0 + c2;
        int bytes;
        if (TA) bytes = (m < P.M) ? min(max(kend - k, 0), 2) * 8 : 0;
        else bytes = (k < kend) ? min(max(P.M - m, 0), 2) * 8 : 0;
        const double* src = bytes ? (TA ? A + k + (int64_t)m * lda : A + m + (int64_t)k * lda) : A;
        ptx::cp_async16(as + row * SLD + c2, src, bytes);
      }
      {  // B: TB -> op(B)[k][n] = B[n + k ldb]: tile [k][n]; !TB -> B[k + n ldb]: tile [n][k]
        const int k = TB ? kc + row : kc + c2, n = TB ? n0 + c2 : n0 + row;
        int bytes;
        if (TB) bytes = (k < kend) ? min(max(P.N - n, 0), 2) * 8 : 0;
        else bytes = (n < P.N) ? min(max(kend - k, 0), 2) * 8 : 0;
        const double* src = bytes ? (TB ? B + n + (int64_t)k * ldb : B + k + (int64_t)n * ldb) : B;
        ptx::cp_async16(bs + row * SLD + c2, src, bytes);
      }
    }
  };
#pragma unroll
  for (int s = 0; s < SA_STAGES - 1; ++s) {
    if (s < nchunks) issue(s);
    ptx::cp_async_commit();
  }
  double acc[2][2][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  for (int i = 0; i < nchunks; ++i) {
    ptx::cp_async_wait<SA_STAGES - 2>();
    __syncthreads();   // chunk i landed for every thread; stage (i-1) % S is free
    if (i + SA_STAGES - 1 < nchunks) issue(i + SA_STAGES - 1);
    ptx::cp_async_commit();
    const double* as = sa_smem + (i % SA_STAGES) * 2 * SA_TILE;
    const double* bs = as + SA_TILE;
#pragma unroll
    for (int k4 = 0; k4 < SKC / 4; ++k4) {
      const int k = 4 * k4 + t;
      double a[2], b[2];
#pragma unroll
      for (int f = 0; f < 2; ++f) {
        const int m = 16 * wm + 8 * f + g, n = 16 * wn + 8 * f + g;
        a[f] = TA ? as[m * SLD + k] : as[k * SLD + m];
        b[f] = TB ? bs[k * SLD + n] : bs[n * SLD + k];
      }
#pragma unroll
      for (int fm = 0; fm < 2; ++fm)
#pragma unroll
        for (int fn = 0; fn < 2; ++fn) ptx::dmma_8x8x4(acc[fm][fn][0], acc[fm][fn][1], a[fm], b[fn]);
    }
  }
  ptx::cp_async_wait<0>();
#pragma unroll
  for (int fm = 0; fm < 2; ++fm)
#pragma unroll
    for (int fn = 0; fn < 2; ++fn)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int m = m0 + 16 * wm + 8 * fm + g, n = n0 + 16 * wn + 8 * fn + 2 * t + j;
        if (m >= P.M || n >= P.N) continue;
        if ((P.flags & SYM_LOWER) && m < n) continue;
        epi_apply(P.epi, m, n, acc[fm][fn][j]);
        if ((P.flags & SYM_MIRROR) && (m > n || P.epi.mir1)) epi_mirror(P.epi, n, m, acc[fm][fn][j]);
      }
}

template <bool TA, bool TB>
void launch_small(Ctx* c, const double* A, int64_t lda, const double* B, int64_t ldb, const KParamsS& P) {
  dim3 grid((unsigned)((P.N + ST - 1) / ST), (unsigned)((P.M + ST - 1) / ST));
  Prof pr(c, c->cur_tag);
  const bool aligned = (reinterpret_cast<uintptr_t>(A) % 16 == 0) && (reinterpret_cast<uintptr_t>(B) % 16 == 0) &&
                       lda % 2 == 0 && ldb % 2 == 0 && !c->no_small_async;
  if (aligned) {
    CGGM_ONCE_PER_DEVICE({
      CGGM_CUDA_CHECK(cudaFuncSetAttribute(gemm_small_async_kernel<TA, TB>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, SA_SMEM));
    });
    launch_pdl(c, gemm_small_async_kernel<TA, TB>, grid, dim3(128), SA_SMEM, A, lda, B, ldb, P);
    post_launch(c, "gemm_small_async_kernel");
  } else {
    launch_pdl(c, gemm_small_kernel<TA, TB>, grid, dim3(128), 0, A, lda, B, ldb, P);
    post_launch(c, "gemm_small_kernel");
  }
}

CUtensorMap make_map_mn3d(Ctx* c, const double* ptr, int64_t ld, int64_t X, int64_t K, uint32_t bx) {
  CUtensorMap m;
  cuuint64_t dims[3] = {16, (cuuint64_t)K, (cuuint64_t)(X / 16)};
  cuuint64_t strides[2] = {(cuuint64_t)(ld * 8), 128};
  cuuint32_t box[3] = {16, 16, bx / 16};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = c->encode_tiled(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(ptr), dims, strides, box,
                               estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw CudaError{CGGM_ERR_CUDA, "cuTensorMapEncodeTiled (3d) failed (" + std::to_string((int)r) + ")"};
  return m;
}

CUtensorMap make_map(Ctx* c, const double* ptr, int64_t ld, int64_t inner, int64_t outer, uint32_t box_inner,
                     uint32_t box_outer) {
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 8)};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = c->encode_tiled(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(ptr), dims, strides, box,
                               estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw CudaError{CGGM_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")"};
  return m;
}

template <bool AK, bool BKI, class C>
void launch(Ctx* c, const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& ma2, const CUtensorMap& mb2,
            const KParams& P, int grid) {
  CGGM_ONCE_PER_DEVICE({
    CGGM_CUDA_CHECK(cudaFuncSetAttribute(gemm_dmma_kernel<AK, BKI, C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         C::SMEM_BYTES));
    // the largest shared-memory carveout, so that configurations sized for 2-3 CTAs per SM get them
    CGGM_CUDA_CHECK(cudaFuncSetAttribute(gemm_dmma_kernel<AK, BKI, C>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                         (int)cudaSharedmemCarveoutMaxShared));
  });
  Prof pr(c, c->cur_tag);
  launch_pdl(c, gemm_dmma_kernel<AK, BKI, C>, dim3(grid), dim3(C::LB_THREADS), C::SMEM_BYTES, ma, mb, ma2, mb2, P);
  post_launch(c, "gemm_dmma_kernel");
}

// ------------------------------------------------------------------ persistent warp-specialised
// One CTA per SM walks tiles tbase, tbase + rw, ... (windows of `resident` CTAs, so the tiles in
// flight at any moment are consecutive in the tile order).  The producer warpgroup streams the
// k-tiles of all of its tiles through the ring without a break, so while the consumers run a
// tile's epilogue (through a staging buffer of its own, half a tile per round) the ring already
// fills with the next tile's operands: the per-tile pipeline fill and CTA launch vanish.
template <class C>
constexpr int pws_smem_bytes() {
  return STAGES * C::STAGE_BYTES + (C::BN / 2) * C::EPI_LD * 8 + 2 * STAGES * 8 + 1024;
}

template <bool AK, bool BKI, class C>
__device__ __forceinline__ void pws_tile(const KParams& P, int tile, int& I, int& J, int& kt0, int& nkt) {
  tile_coords(P, tile, I, J);
  const int m0 = I * C::BM, n0 = J * C::BN;
  int kbeg = 0, kend = P.K;
  if (P.flags & A_KGE_M) kbeg = max(kbeg, m0);
  if (P.flags & B_KGE_N) kbeg = max(kbeg, n0);
  if (P.flags & A_KLE_M) kend = min(kend, m0 + C::BM);
  if (P.flags & B_KLE_N) kend = min(kend, n0 + C::BN);
  kt0 = kbeg / BK;
  nkt = kend > kbeg ? (kend - kt0 * BK + BK - 1) / BK : 0;
}

template <bool AK, bool BKI, class C>
__global__ void __launch_bounds__(C::NTHREADS + 128, 1)
    gemm_dmma_pws(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                  const __grid_constant__ CUtensorMap tmA2, const __grid_constant__ CUtensorMap tmB2,
                  const KParams P, int ntiles, int tpc, int resident) {
  constexpr int BM = C::BM, BN = C::BN, NCW = C::WM * C::WN, FM = C::FM, FN = C::FN;
  constexpr int OP_BYTES = C::A_BYTES, STAGE_BYTES = C::STAGE_BYTES;
  constexpr int EPI_LD = C::EPI_LD, NTHREADS = C::NTHREADS, SW = BN / 2;
  constexpr int RING = STAGES * STAGE_BYTES, SLAB = SW * EPI_LD * 8;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  double* Cs = reinterpret_cast<double*>(smem + RING);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + RING + SLAB);
  uint64_t* empty = full + STAGES;
  const int win = blockIdx.x / resident, r_in = blockIdx.x % resident;
  const int rw = min(resident, (int)gridDim.x - win * resident);
  const int tbase = win * resident * tpc + r_in;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], NCW);
    }
    ptx::fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x < 128) {   // ------------------------------ producer warpgroup
    asm volatile("setmaxnreg.dec.sync.aligned.u32 40;\n" ::: "memory");
    if (threadIdx.x == 0) {
      int slot = 0, g = 0;
      uint32_t ph = 0;   // parity to wait for on the slot's release (used from the second pass on)
      for (int kt = 0; kt < tpc; ++kt) {
        const int tile = tbase + kt * rw;
        if (tile >= ntiles) break;
        int I, J, kt0, nkt;
        pws_tile<AK, BKI, C>(P, tile, I, J, kt0, nkt);
        const int m0 = I * BM, n0 = J * BN;
        const bool a_one = !AK && P.a3d && (m0 + BM <= P.a3d || P.a3d == P.M);
        const bool b_one = !BKI && P.b3d && (n0 + BN <= P.b3d || P.b3d == P.N);
        int a_boxes = 0, b_boxes = 0;
        if (!AK && !a_one)
          for (int xb = 0; xb < BM / 16; ++xb) a_boxes += (m0 + xb * 16 < P.M);
        if (!BKI && !b_one)
          for (int xb = 0; xb < BN / 16; ++xb) b_boxes += (n0 + xb * 16 < P.N);
        const uint32_t tx = ((AK || a_one) ? C::A_BYTES : a_boxes * 2048) + ((BKI || b_one) ? C::B_BYTES : b_boxes * 2048);
        for (int i = 0; i < nkt; ++i, ++g) {
          if (g >= STAGES) ptx::mbar_wait(&empty[slot], ph ^ 1);
          uint8_t* sa = smem + slot * STAGE_BYTES;
          uint8_t* sb = sa + OP_BYTES;
          ptx::mbar_arrive_expect_tx(&full[slot], tx);
          const int k = (kt0 + i) * BK;
          if (AK) ptx::tma_load_2d(sa, &tmA, &full[slot], k, m0);
          else if (a_one) ptx::tma_load_3d(sa, &tmA, &full[slot], 0, k, m0 / 16);
          else for (int xb = 0; xb < a_boxes; ++xb) ptx::tma_load_2d(sa + xb * 2048, &tmA2, &full[slot], m0 + xb * 16, k);
          if (BKI) ptx::tma_load_2d(sb, &tmB, &full[slot], k, n0);
          else if (b_one) ptx::tma_load_3d(sb, &tmB, &full[slot], 0, k, n0 / 16);
          else for (int xb = 0; xb < b_boxes; ++xb) ptx::tma_load_2d(sb + xb * 2048, &tmB2, &full[slot], n0 + xb * 16, k);
          if (++slot == STAGES) {
            slot = 0;
            ph ^= 1;
          }
        }
      }
    }
    return;
  }
  // -------------------------------------------------------------- consumer warpgroups
  asm volatile("setmaxnreg.inc.sync.aligned.u32 232;\n" ::: "memory");
  const int tid = threadIdx.x - 128, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp / C::WN, wn = warp % C::WN;
  const int xa0 = wm * C::WTM, xb0 = wn * C::WTN;
  auto cbar = [&]() { asm volatile("bar.sync 1, %0;\n" ::"n"(NTHREADS) : "memory"); };
  int slot = 0;
  uint32_t ph = 0;
  for (int kt = 0; kt < tpc; ++kt) {
    const int tile = tbase + kt * rw;
    if (tile >= ntiles) break;
    int I, J, kt0, nkt;
    pws_tile<AK, BKI, C>(P, tile, I, J, kt0, nkt);
    double acc[FM][FN][2];
#pragma unroll
    for (int a = 0; a < FM; ++a)
#pragma unroll
      for (int b = 0; b < FN; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    for (int i = 0; i < nkt; ++i) {
      ptx::mbar_wait(&full[slot], ph);
      const uint32_t sa = ptx::smem_u32(smem + slot * STAGE_BYTES);
      const uint32_t sb = sa + OP_BYTES;
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) {
        double a[FM][2], b[FN][2];
        if (AK) {
#pragma unroll
          for (int f = 0; f < FM; ++f) {
            const int x = xa0 + frag_x<true>(f, g);
            const int chunk = (4 * kk + t) ^ (x & 7);
            ptx::lds128(a[f][0], a[f][1], sa + x * 128 + chunk * 16);
          }
        } else {
#pragma unroll
          for (int pr = 0; pr < FM / 2; ++pr) {
            const int xb = xa0 / 16 + pr;
#pragma unroll
            for (int s2 = 0; s2 < 2; ++s2) {
              const int k = 8 * kk + 2 * t + s2;
              const int chunk = g ^ (k & 7);
              ptx::lds128(a[2 * pr][s2], a[2 * pr + 1][s2], sa + xb * 2048 + k * 128 + chunk * 16);
            }
          }
        }
        if (BKI) {
#pragma unroll
          for (int f = 0; f < FN; ++f) {
            const int x = xb0 + frag_x<true>(f, g);
            const int chunk = (4 * kk + t) ^ (x & 7);
            ptx::lds128(b[f][0], b[f][1], sb + x * 128 + chunk * 16);
          }
        } else {
#pragma unroll
          for (int pr = 0; pr < FN / 2; ++pr) {
            const int xb = xb0 / 16 + pr;
#pragma unroll
            for (int s2 = 0; s2 < 2; ++s2) {
              const int k = 8 * kk + 2 * t + s2;
              const int chunk = g ^ (k & 7);
              ptx::lds128(b[2 * pr][s2], b[2 * pr + 1][s2], sb + xb * 2048 + k * 128 + chunk * 16);
            }
          }
        }
#pragma unroll
        for (int s2 = 0; s2 < 2; ++s2)
#pragma unroll
          for (int fm = 0; fm < FM; ++fm)
#pragma unroll
            for (int fn = 0; fn < FN; ++fn) ptx::dmma_8x8x4(acc[fm][fn][0], acc[fm][fn][1], a[fm][s2], b[fn][s2]);
      }
      __syncwarp();
      ptx::fence_proxy_async();   // (generic reads of the slot before its TMA refill, as above)
      if (lane == 0) ptx::mbar_arrive(&empty[slot]);
      if (++slot == STAGES) {
        slot = 0;
        ph ^= 1;
      }
    }
    // ---------------------------------------------------------- epilogue, half a tile per round
    const int m0 = I * BM, n0 = J * BN;
    const bool diag = (P.flags & SYM_LOWER) && m0 < n0 + BN;
    const bool interior = P.vec && !diag && m0 + BM <= P.M && n0 + BN <= P.N;
    const Epilogue& E = P.epi;
#pragma unroll 1
    for (int h = 0; h < 2; ++h) {
      const int nbase = n0 + h * SW;
      if (wn / (C::WN / 2) == h) {
#pragma unroll
        for (int fm = 0; fm < FM; ++fm) {
          const int ml = xa0 + frag_x<AK>(fm, g);
#pragma unroll
          for (int fn = 0; fn < FN; ++fn)
#pragma unroll
            for (int j = 0; j < 2; ++j) Cs[(xb0 - h * SW + frag_x<BKI>(fn, 2 * t + j)) * EPI_LD + ml] = acc[fm][fn][j];
        }
      }
      cbar();
      if (interior) {
        constexpr int RP = BM / 2, CG = NTHREADS / RP, NCOL = SW / CG, U = NCOL < 8 ? NCOL : 8;
        const int ml = 2 * (tid % RP), cg = tid / RP;
        const int64_t m = m0 + ml;
#pragma unroll 1
        for (int i0 = 0; i0 < NCOL; i0 += U) {
          double2 x1[U], x2[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int64_t n = nbase + cg + CG * (i0 + u);
            if (E.in1a) x1[u] = *reinterpret_cast<const double2*>(E.in1a + m + n * E.ld1a);
            if (E.in2a) x2[u] = *reinterpret_cast<const double2*>(E.in2a + m + n * E.ld2a);
          }
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int nl = cg + CG * (i0 + u);
            const int64_t n = nbase + nl;
            const double v0 = Cs[nl * EPI_LD + ml], v1 = Cs[nl * EPI_LD + ml + 1];
            if (E.out1) {
              double2 o = make_double2(__dmul_rn(E.a1, v0), __dmul_rn(E.a1, v1));
              if (E.in1a) {
                o.x = __dadd_rn(o.x, __dmul_rn(E.b1, x1[u].x));
                o.y = __dadd_rn(o.y, __dmul_rn(E.b1, x1[u].y));
              }
              *reinterpret_cast<double2*>(E.out1 + m + n * E.ld1) = o;
            }
            if (E.out2) {
              double2 o = make_double2(__dmul_rn(E.a2, v0), __dmul_rn(E.a2, v1));
              if (E.in2a) {
                o.x = __dadd_rn(o.x, __dmul_rn(E.b2, x2[u].x));
                o.y = __dadd_rn(o.y, __dmul_rn(E.b2, x2[u].y));
              }
              if (E.in2b) {   // (only the Psi GEMM's grad_Lambda output has a second input: loaded here)
                const double2 x4 = *reinterpret_cast<const double2*>(E.in2b + m + n * E.ld2b);
                o.x = __dadd_rn(o.x, __dmul_rn(E.c2, x4.x));
                o.y = __dadd_rn(o.y, __dmul_rn(E.c2, x4.y));
              }
              *reinterpret_cast<double2*>(E.out2 + m + n * E.ld2) = o;
            }
          }
        }
      } else {
        for (int idx = tid; idx < BM * SW; idx += NTHREADS) {
          const int ml = idx % BM, nl = idx / BM;
          const int m = m0 + ml, n = nbase + nl;
          if (m >= P.M || n >= P.N) continue;
          if (diag && m < n) continue;
          epi_apply(E, m, n, Cs[nl * EPI_LD + ml]);
        }
      }
      if (P.flags & SYM_MIRROR) {
        if (interior) {
          constexpr int NWARPS = NTHREADS / 32, NBLK = SW / 32, GROUPS = NWARPS / NBLK, PAIRS = BM / 2 / GROUPS;
          const int nl = 32 * (warp % NBLK) + lane, grp = warp / NBLK;
          const bool odd = lane & 1;
          const int64_t n = nbase + nl - (odd ? 1 : 0);
#pragma unroll 4
          for (int i = 0; i < PAIRS; ++i) {
            const int ml = 2 * (grp + GROUPS * i);
            const double a = Cs[nl * EPI_LD + ml], b = Cs[nl * EPI_LD + ml + 1];
            const double pa = __shfl_xor_sync(0xffffffffu, a, 1), pb = __shfl_xor_sync(0xffffffffu, b, 1);
            const double lo = odd ? pb : a, hi = odd ? b : pa;
            const int64_t m = m0 + ml + (odd ? 1 : 0);
            if (E.out1) {
              double2 o = make_double2(__dmul_rn(E.a1, lo), __dmul_rn(E.a1, hi));
              if (E.in1a) {
                const double2 x = *reinterpret_cast<const double2*>(E.in1a + n + m * E.ld1a);
                o.x = __dadd_rn(o.x, __dmul_rn(E.b1, x.x));
                o.y = __dadd_rn(o.y, __dmul_rn(E.b1, x.y));
              }
              *reinterpret_cast<double2*>((E.mir1 ? E.mir1 : E.out1) + n + m * E.ld1) = o;
            }
            if (E.out2) {
              double2 o = make_double2(__dmul_rn(E.a2, lo), __dmul_rn(E.a2, hi));
              if (E.in2a) {   // the inputs at the written (transposed) position: contiguous along n
                const double2 x = *reinterpret_cast<const double2*>(E.in2a + n + m * E.ld2a);
                o.x = __dadd_rn(o.x, __dmul_rn(E.b2, x.x));
                o.y = __dadd_rn(o.y, __dmul_rn(E.b2, x.y));
              }
              if (E.in2b) {
                const double2 x = *reinterpret_cast<const double2*>(E.in2b + n + m * E.ld2b);
                o.x = __dadd_rn(o.x, __dmul_rn(E.c2, x.x));
                o.y = __dadd_rn(o.y, __dmul_rn(E.c2, x.y));
              }
              *reinterpret_cast<double2*>(E.out2 + n + m * E.ld2) = o;
            }
          }
        } else {
          for (int idx = tid; idx < BM * SW; idx += NTHREADS) {
            const int nl = idx % SW, ml = idx / SW;
            const int m = m0 + ml, n = nbase + nl;
            if (m >= P.M || n >= P.N) continue;
            if (diag && m <= n) continue;
            epi_mirror(E, n, m, Cs[nl * EPI_LD + ml]);
          }
        }
      }
      cbar();
    }
  }
}

template <bool AK, bool BKI, class C>
void launch_pws(Ctx* c, const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& ma2, const CUtensorMap& mb2,
                const KParams& P, int ntiles) {
  constexpr int smem = pws_smem_bytes<C>();
  CGGM_ONCE_PER_DEVICE({
    CGGM_CUDA_CHECK(cudaFuncSetAttribute(gemm_dmma_pws<AK, BKI, C>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    CGGM_CUDA_CHECK(cudaFuncSetAttribute(gemm_dmma_pws<AK, BKI, C>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                         (int)cudaSharedmemCarveoutMaxShared));
  });
  const int tpc = c->persist_tpc, R = c->num_sms;
  const int full = ntiles / (R * tpc), rem = ntiles - full * R * tpc;
  const int grid = full * R + (rem + tpc - 1) / tpc;
  Prof pr(c, c->cur_tag);
  gemm_dmma_pws<AK, BKI, C><<<grid, C::NTHREADS + 128, smem, c->stream>>>(ma, mb, ma2, mb2, P, ntiles, tpc, R);
  post_launch(c, "gemm_dmma_pws");
}

// CGGM_GEMM_LOG=1: one stderr line per launch with the MMA flops the tiles execute (triangular
// k-ranges applied per tile), for joining with an ncu launch list (per-launch efficiency)
void gemm_log(Ctx* c, int BM, int BN, int M, int N, int K, int flags, int grid, bool tA, bool tB) {
  static int on = -1;
  if (on < 0) {
    const char* e = std::getenv("CGGM_GEMM_LOG");
    on = e ? std::atoi(e) : 0;
  }
  if (!on) return;
  const int tm = (M + BM - 1) / BM, tn = (N + BN - 1) / BN;
  double fl = 0.0;
  auto tile = [&](int m0, int n0) {   // executed flops of one BM x BN tile (16-wide k-steps)
    int kbeg = 0, kend = K;
    if (flags & A_KGE_M) kbeg = std::max(kbeg, m0);
    if (flags & B_KGE_N) kbeg = std::max(kbeg, n0);
    if (flags & A_KLE_M) kend = std::min(kend, m0 + BM);
    if (flags & B_KLE_N) kend = std::min(kend, n0 + BN);
    if (kend > kbeg) fl += 2.0 * BM * BN * (double)(((kend - kbeg + 15) / 16) * 16);
  };
  if ((flags & SYM_LOWER) && BN * 2 == BM) {
    // the sym_split walk (run_cfg): BM x BM squares I >= J, each as two BN-wide column halves
    const int ts = (N + BM - 1) / BM;
    for (int I = 0; I < tm; ++I)
      for (int J = 0; J < ts && J <= I; ++J)
        for (int h = 0; h < 2; ++h)
          if (J * BM + h * BN < N) tile(I * BM, J * BM + h * BN);
  } else {
    for (int I = 0; I < tm; ++I)
      for (int J = 0; J < tn; ++J)
        if (!((flags & SYM_LOWER) && I < J)) tile(I * BM, J * BN);
  }
  std::fprintf(stderr, "GEMMLOG tile=%dx%d M=%d N=%d K=%d flags=%d tA=%d tB=%d grid=%d exec_flops=%.6e lane=%d\n", BM, BN,
               M, N, K, flags, (int)tA, (int)tB, grid, fl, c->lane);
}

template <class C>
void run_cfg(Ctx* c, bool transA, bool transB, int64_t M, int64_t N, int64_t Keff, const double* A, int64_t lda,
             const double* B, int64_t ldb, KParams& P) {
  P.tilesM = (int)((M + C::BM - 1) / C::BM);
  P.tilesN = (int)((N + C::BN - 1) / C::BN);
  P.sym_split = 1;
  if ((P.flags & SYM_LOWER) && C::BN * 2 == C::BM) {   // walk BM x BM squares, two column halves each
    P.sym_split = 2;
    P.tilesN = (int)((N + C::BM - 1) / C::BM);
  }
  int grid;
  if (P.flags & SYM_LOWER) grid = (P.tilesN * (P.tilesN + 1) / 2 + (P.tilesM - P.tilesN) * P.tilesN) * P.sym_split;
  else grid = P.tilesM * P.tilesN;
  grid *= P.ksplit;
  // K-inner operand: dims {K, X}, box {16, BX}; MN-inner: dims {X, K}, box {16, 16}
  // MN-inner operand: the 3-D single-box map covers the leading multiple of 16 rows (so a box
  // never reads past the extent); a 16-wide 2-D map serves the ragged last tile
  const int64_t M16 = M / 16 * 16, N16 = N / 16 * 16;
  P.a3d = (!transA && M16 > 0 && !c->no_tma3d) ? (int)M16 : 0;
  P.b3d = (transB && N16 > 0 && !c->no_tma3d) ? (int)N16 : 0;
  CUtensorMap ma = transA ? make_map(c, A, lda, Keff, M, 16, C::BM)
                          : (P.a3d ? make_map_mn3d(c, A, lda, M16, Keff, C::BM) : make_map(c, A, lda, M, Keff, 16, 16));
  CUtensorMap mb = transB ? (P.b3d ? make_map_mn3d(c, B, ldb, N16, Keff, C::BN) : make_map(c, B, ldb, N, Keff, 16, 16))
                          : make_map(c, B, ldb, Keff, N, 16, C::BN);
  const bool a_tail = !transA && P.a3d && M16 != M, b_tail = transB && P.b3d && N16 != N;
  CUtensorMap ma2 = a_tail ? make_map(c, A, lda, M, Keff, 16, 16) : ma;
  CUtensorMap mb2 = b_tail ? make_map(c, B, ldb, N, Keff, 16, 16) : mb;
  const bool AK = transA, BKI = !transB;
  gemm_log(c, C::BM, C::BN, P.M, P.N, P.K, P.flags, grid, transA, transB);
  if constexpr (C::WSP) {
    if (C::BN == 128 && c->persist_tpc > 0 && P.ksplit == 1 && grid >= 2 * c->num_sms && !P.epi.sel.on) {
      if (AK && BKI) launch_pws<true, true, C>(c, ma, mb, ma2, mb2, P, grid);
      else if (AK && !BKI) launch_pws<true, false, C>(c, ma, mb, ma2, mb2, P, grid);
      else if (!AK && BKI) launch_pws<false, true, C>(c, ma, mb, ma2, mb2, P, grid);
      else launch_pws<false, false, C>(c, ma, mb, ma2, mb2, P, grid);
      return;
    }
  }
  if (AK && BKI) launch<true, true, C>(c, ma, mb, ma2, mb2, P, grid);
  else if (AK && !BKI) launch<true, false, C>(c, ma, mb, ma2, mb2, P, grid);
  else if (!AK && BKI) launch<false, true, C>(c, ma, mb, ma2, mb2, P, grid);
  else launch<false, false, C>(c, ma, mb, ma2, mb2, P, grid);
}

bool tma_ok(const double* p, int64_t ld) {
  return (reinterpret_cast<uintptr_t>(p) % 16 == 0) && (ld % 2 == 0);
}

}  // namespace

void gemm(Ctx* c, bool transA, bool transB, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda,
          const double* B, int64_t ldb, const Epilogue& epi, int flags) {
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
  // (an output aliasing an operand -- an in-place B := B X^T with N <= 64 -- needs one CTA per row
  // panel, which only the TMA kernels guarantee)
  const bool aliased = epi.out1 == A || epi.out1 == B || (epi.out2 && (epi.out2 == A || epi.out2 == B));
  // small shapes, and mid-size products whose 64x64 grid would leave most SMs idle (the middle of
  // the recursion: 4x the CTAs of a 64-tile grid with the whole k-range streamed by cp.async)
  const int64_t tiles64 = ((M + 63) / 64) * ((N + 63) / 64);
  const bool small_shape = K <= 256 && (M <= 128 || N <= 128);
  const bool mid_shape = K <= c->small_kmax && tiles64 < c->num_sms && !c->no_small_async &&
                         (reinterpret_cast<uintptr_t>(A) % 16 == 0) && (reinterpret_cast<uintptr_t>(B) % 16 == 0) &&
                         lda % 2 == 0 && ldb % 2 == 0;
  if (epi.sel.on && (flags & (SYM_LOWER | SYM_MIRROR | SPLIT_K2)))
    throw CudaError{CGGM_ERR_UNSUPPORTED, "K01 selection epilogue: plain products only"};
  if ((small_shape || mid_shape) && !aliased && !(flags & SPLIT_K2) && !epi.sel.on && c->force_tile != 1 &&
      c->force_tile != 2) {
    KParamsS S;
    S.M = (int)M; S.N = (int)N; S.K = (int)(K > 0 ? K : 0); S.flags = flags; S.epi = epi;
    if (transA && transB) launch_small<true, true>(c, A, lda, B, ldb, S);
    else if (transA) launch_small<true, false>(c, A, lda, B, ldb, S);
    else if (transB) launch_small<false, true>(c, A, lda, B, ldb, S);
    else launch_small<false, false>(c, A, lda, B, ldb, S);
    return;
  }
  static double* dummy = nullptr;
  if (K <= 0) {
    if (!dummy) CGGM_CUDA_CHECK(cudaMalloc(&dummy, 16 * 16 * 8));
    A = dummy; B = dummy; lda = 16; ldb = 16;
  }
  const int64_t Keff = K > 0 ? K : 1;
  // operands not meeting TMA constraints (16-B base, even ld) are packed
  const int64_t arows = transA ? Keff : M, acols = transA ? M : Keff;
  const int64_t brows = transB ? N : Keff, bcols = transB ? Keff : N;
  if (K > 0 && !tma_ok(A, lda)) {
    int64_t ld = (arows + 1) & ~int64_t(1);
    double* pk = static_cast<double*>(ws_get(c, WS_PACK0 + 2 * c->lane, (size_t)ld * acols * 8));
    CGGM_CUDA_CHECK(cudaMemcpy2DAsync(pk, ld * 8, A, lda * 8, arows * 8, acols, cudaMemcpyDeviceToDevice, c->stream));
    A = pk; lda = ld;
  }
  if (K > 0 && !tma_ok(B, ldb)) {
    int64_t ld = (brows + 1) & ~int64_t(1);
    double* pk = static_cast<double*>(ws_get(c, WS_PACK1 + 2 * c->lane, (size_t)ld * bcols * 8));
    CGGM_CUDA_CHECK(cudaMemcpy2DAsync(pk, ld * 8, B, ldb * 8, brows * 8, bcols, cudaMemcpyDeviceToDevice, c->stream));
    B = pk; ldb = ld;
  }
  KParams P;
  P.M = (int)M; P.N = (int)N; P.K = (int)(K > 0 ? K : 0);
  P.flags = flags;
  P.epi = epi;
  P.ksplit = (flags & SPLIT_K2) ? 2 : 1;
  if (P.ksplit > 1 && ((flags & (SYM_LOWER | SYM_MIRROR)) || epi.out2 || epi.in1a || epi.in1b || !epi.out1))
    throw CudaError{CGGM_ERR_UNSUPPORTED, "SPLIT_K2: plain out1 only"};
  {
    auto al = [](const double* q, int64_t ld) { return !q || (reinterpret_cast<uintptr_t>(q) % 16 == 0 && ld % 2 == 0); };
    P.vec = !c->no_vec_epi && !epi.in1b && al(epi.out1, epi.ld1) && al(epi.out2, epi.ld2) &&
            al(epi.in1a, epi.ld1a) && al(epi.in2a, epi.ld2a) && al(epi.in2b, epi.ld2b) && al(epi.mir1, epi.ld1);
  }
  if ((flags & SYM_LOWER) && (M < N || ((flags & SYM_MIRROR) && M != N)))
    throw CudaError{CGGM_ERR_SHAPE, "SYM_LOWER gemm needs M >= N (M == N with SYM_MIRROR)"};
  // 128x128 tiles unless they cannot fill the GPU; then 64x64 tiles (4x the CTAs, several per SM)
  const int64_t tm = (M + 127) / 128, tn = (N + 127) / 128;
  const int64_t big_tiles = (flags & SYM_LOWER) ? tn * (tn + 1) / 2 + (tm - tn) * tn : tm * tn;
  // wave efficiency of the 128-tile grid; below ~0.9 (and under 3 waves) the 64-tile grid (4x the
  // CTAs, 3 resident per SM) fills the machine better (profiles/r01_gemm_bench_tiles*.txt)
  const int64_t waves = (big_tiles + c->num_sms - 1) / c->num_sms;
  const double big_eff = (double)big_tiles / (double)(waves * c->num_sms);
  bool auto_big = big_tiles >= 3 * c->num_sms || big_eff >= 0.9;
  if (!auto_big && c->mid_min_waves > 0 && c->mid_tile) {
    // mid-size products: the warp-specialised 128x64 tiles (two per SM) once their grid fills at least
    // mid_min_waves / 4 waves (CGGM_MID_MIN_WAVES, quarter waves; 0 = the 128x128-tile rule above only)
    const int64_t mt = (flags & SYM_LOWER) ? 2 * (tn * (tn + 1) / 2 + (tm - tn) * tn) : tm * ((N + 63) / 64);
    auto_big = 4 * mt >= (int64_t)c->mid_min_waves * 2 * c->num_sms;
  }
  const bool use_big = c->force_tile ? (c->force_tile == 1) : auto_big;
  // CGGM_MID_TILE (two-CTA 128x64 tiles for): 3 = every large product (default; the step 410.2 ->
  // 409.7 ms against 4, although lauum alone is 74.46 -> 74.58 ms: its k-loop hides the epilogue,
  // but the co-running streams gain), 1 = non-symmetric and symmetric with K <= 4096, 2 = 1 plus
  // split-k, 4 = non-symmetric only; 0 = 128x128 everywhere
  const bool mid_sym = c->mid_tile == 3 || (c->mid_tile != 4 && Keff <= 4096);
  if (use_big && c->mid_tile && (mid_sym || !(flags & SYM_LOWER)) && (c->mid_tile == 2 || c->mid_tile == 3 || !(flags & SPLIT_K2)))
    run_cfg<CfgMid>(c, transA, transB, M, N, Keff, A, lda, B, ldb, P);
  else if (use_big) run_cfg<CfgBig>(c, transA, transB, M, N, Keff, A, lda, B, ldb, P);
  else run_cfg<CfgSmall>(c, transA, transB, M, N, Keff, A, lda, B, ldb, P);
}

}  // namespace cggm
