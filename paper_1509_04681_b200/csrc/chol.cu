// Sigma = Lambda^{-1}, log|Lambda| and the Cholesky PD test (§2.3;
// P:287-288 for the line search), as a recursive blocked Cholesky whose work is almost
// entirely the FP64 DMMA GEMM of gemm.cu:
//
//  node(A, n) with A = [A11 .; A21 A22], n1 ~ n/2 (multiple of 64):
//    full_inverse (cggm_invert_logdet):          potrf only (cggm_objective):
//      node(A11) -> X11 = L11^{-1}                 node(A11) -> L11 (+ leaf inverses)
//      T  = A21 X11^T          (= L21)             A21 := A21 L11^{-T}   (recursive trsm)
//      A22 -= T T^T            (lower tiles)       A22 -= A21 A21^T
//      A21 := T X11            (= L21 L11^{-1})    node(A22)
//      node(A22) -> X22
//      X21 = -X22 A21          (= L^{-1} block)
//  then Sigma = X^T X (lauum, one symmetric GEMM, k >= max(m, n)).
// Flops: potrf q^3/3 + trtri q^3/3 + lauum q^3/3 (= potrf + potri).  Leaves (<= 64 columns)
// run an unblocked Cholesky + triangular inverse in shared memory (one CTA), record the
// first failing pivot (atomicMin) and 2 sum ln L_jj per leaf (deterministic final sum).
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <climits>
#include <cstdlib>
#include <initializer_list>
#include <vector>

#include "common.cuh"

namespace cggm {
namespace {

__device__ __forceinline__ double rsqrt_t(double x) { return rsqrt(x); }
__device__ __forceinline__ float rsqrt_t(float x) { return rsqrtf(x); }
__device__ __forceinline__ double fma_t(double a, double b, double c) { return fma(a, b, c); }
__device__ __forceinline__ float fma_t(float a, float b, float c) { return fmaf(a, b, c); }

constexpr int NB = 64;
#ifndef CGGM_LEAF_THREADS
#define CGGM_LEAF_THREADS 256
#endif
// (128 threads x <= 128 registers would fit beside a 128x128 GEMM CTA, but measured slower)
constexpr int LEAF_THREADS = CGGM_LEAF_THREADS;
template <typename T>
constexpr int leaf_smem_bytes() { return 2 * NB * (NB + 1) * (int)sizeof(T); }

// Leaf: Cholesky + triangular inverse of one nb x nb (nb <= 64) diagonal block in one CTA of 256
// threads, blocked by 8-column panels (rows/columns >= nb padded with the identity, so L and
// L^{-1} are block-diag(., I)).  32 block barriers in total:
//   potrf, per panel p (columns c0 = 8p .. c0+7):
//     warp 0 factors the panel in registers (lane l holds rows c0+l and c0+l+32): pivot by shuffle,
//       1/sqrt(d) once, column scale, rank-1 update of the remaining panel columns -- shuffles only;
//       the first failing pivot is recorded (reading A10);
//     all warps apply the rank-8 update to the trailing lower triangle (4x4 blocks per thread);
//   trtri, per block row p (rows r0 = 8p .. r0+7):  T = E_p - L_{p,<p} X_{<p} (all threads),
//     then X_p = L_pp^{-1} T by an 8-row forward substitution per column (64 threads).
// Shared memory: L and X, column-major [col][row] with a padded leading dimension.
template <typename T>
#ifndef CGGM_LEAF_MINB
#define CGGM_LEAF_MINB (512 / CGGM_LEAF_THREADS)
#endif
__global__ void __launch_bounds__(LEAF_THREADS, CGGM_LEAF_MINB) leaf_potrf_trtri(T* A, int64_t lda, int nb, T* X, int64_t ldx,
                                                                  int write_L, double* logdet_slot, int* fail_col,
                                                                  int col0) {
  extern __shared__ __align__(16) unsigned char leaf_raw[];
  T(*Ls)[NB + 1] = reinterpret_cast<T(*)[NB + 1]>(leaf_raw);                              // [col][row]
  T(*Xs)[NB + 1] = reinterpret_cast<T(*)[NB + 1]>(leaf_raw + NB * (NB + 1) * sizeof(T));  // [col][row]
  __shared__ T Tb[NB][9];   // T block of the inverse sweep: [col][row - r0]
  __shared__ T diag[NB], invd[NB];
  __shared__ int fail_sm;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  ptx::pdl_wait();
  ptx::pdl_trigger();   // (one CTA: the successor may be scheduled now; it waits for this grid to complete)
#ifdef CGGM_LEAF_TIMING
  long long lt_[8];
#define LT(i) do { if (t == 0) lt_[i] = clock64(); } while (0)
#else
#define LT(i) do { } while (0)
#endif
  LT(0);
  {  // the loads of a thread in flight 8 at a time
    constexpr int PER = NB * NB / LEAF_THREADS, HALF = PER / 2;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      T v[HALF];
#pragma unroll
      for (int u = 0; u < HALF; ++u) {
        const int idx = t + LEAF_THREADS * (u + h * HALF), i = idx & (NB - 1), j = idx >> 6;
        v[u] = (i < nb && j < nb && i >= j) ? A[i + (int64_t)j * lda] : T(0);
      }
#pragma unroll
      for (int u = 0; u < HALF; ++u) {
        const int idx = t + LEAF_THREADS * (u + h * HALF), i = idx & (NB - 1), j = idx >> 6;
        Ls[j][i] = (i < nb && j < nb) ? v[u] : ((i == j) ? T(1) : T(0));
        Xs[j][i] = T(0);
      }
    }
  }
  if (t == 0) fail_sm = INT_MAX;
  __syncthreads();
  LT(1);
  // ------------------------------------------------------------ Cholesky, 8-column panels
  for (int p = 0; p < NB / 8; ++p) {
    const int c0 = 8 * p;
    if (warp == 0) {
      // the 8x8 diagonal block is factored redundantly by every lane in registers (no shuffles on
      // the dependency chain), then each lane solves its own rows of the panel: v := v Ld^{-T}
      T Ld[8][8];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j <= i; ++j) Ld[i][j] = Ls[c0 + j][c0 + i];
      T inv[8];
      int bad = INT_MAX;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const T d = Ld[j][j];
        if ((!(d > T(0)) || !isfinite(d)) && bad == INT_MAX) bad = j;
        inv[j] = rsqrt_t(d);
        Ld[j][j] = d * inv[j];
#pragma unroll
        for (int i = j + 1; i < 8; ++i) Ld[i][j] *= inv[j];
#pragma unroll
        for (int k = j + 1; k < 8; ++k)
#pragma unroll
          for (int i = k; i < 8; ++i) Ld[i][k] = fma_t(-Ld[i][j], Ld[k][j], Ld[i][k]);
      }
#pragma unroll
      for (int s2 = 0; s2 < 2; ++s2) {
        const int row = c0 + 8 + lane + 32 * s2;
        if (row < NB) {
          T v[8];
#pragma unroll
          for (int jj = 0; jj < 8; ++jj) v[jj] = Ls[c0 + jj][row];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            v[j] *= inv[j];
#pragma unroll
            for (int i = j + 1; i < 8; ++i) v[i] = fma_t(-v[j], Ld[i][j], v[i]);
          }
#pragma unroll
          for (int jj = 0; jj < 8; ++jj) Ls[c0 + jj][row] = v[jj];
        }
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (lane == i) {
#pragma unroll
          for (int j = 0; j <= i; ++j) Ls[c0 + j][c0 + i] = Ld[i][j];
          diag[c0 + i] = Ld[i][i];
          invd[c0 + i] = inv[i];
        }
      if (lane == 0 && bad != INT_MAX) atomicMin(&fail_sm, c0 + bad);
    }
    __syncthreads();
    if (p == 0) LT(2);
    // rank-8 update of the trailing lower triangle (columns >= c0 + 8)
    for (int blk = t; blk < 256; blk += LEAF_THREADS) {   // 4x4 blocks (rb, cb) of the 64x64 tile
      const int rb = blk & 15, cb = blk >> 4;
      if (4 * cb >= c0 + 8 && rb >= cb) {
        T acc[4][4];
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
          for (int i = 0; i < 4; ++i) acc[k][i] = Ls[4 * cb + k][4 * rb + i];
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
          T li[4], lk[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            li[u] = Ls[c0 + jj][4 * rb + u];
            lk[u] = Ls[c0 + jj][4 * cb + u];
          }
#pragma unroll
          for (int k = 0; k < 4; ++k)
#pragma unroll
            for (int i = 0; i < 4; ++i) acc[k][i] = fma_t(-li[i], lk[k], acc[k][i]);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
          for (int i = 0; i < 4; ++i) Ls[4 * cb + k][4 * rb + i] = acc[k][i];
      }
    }
    __syncthreads();
  }
  LT(4);
  // ------------------------------------------------------------ X = L^{-1}, 8-row block sweep
  for (int p = 0; p < NB / 8; ++p) {
    const int r0 = 8 * p;
    for (int e = t; e < 8 * (r0 + 8); e += LEAF_THREADS) {
      const int rr = e & 7, c = e >> 3, r = r0 + rr;
      // four independent partial sums: the dot product is not one serial FMA chain
      T a0 = (r == c) ? T(1) : T(0), a1 = T(0), a2 = T(0), a3 = T(0);
      int m = c;
      for (; m + 3 < r0; m += 4) {
        a0 = fma_t(-Ls[m][r], Xs[c][m], a0);
        a1 = fma_t(-Ls[m + 1][r], Xs[c][m + 1], a1);
        a2 = fma_t(-Ls[m + 2][r], Xs[c][m + 2], a2);
        a3 = fma_t(-Ls[m + 3][r], Xs[c][m + 3], a3);
      }
      for (; m < r0; ++m) a0 = fma_t(-Ls[m][r], Xs[c][m], a0);
      Tb[c][rr] = (a0 + a1) + (a2 + a3);
    }
    __syncthreads();
    if (t < r0 + 8) {
      const int c = t;
      T xv[8];
#pragma unroll
      for (int rr = 0; rr < 8; ++rr) {
        T acc = Tb[c][rr];
#pragma unroll
        for (int ss = 0; ss < rr; ++ss) acc = fma_t(-Ls[r0 + ss][r0 + rr], xv[ss], acc);
        xv[rr] = acc * invd[r0 + rr];
        Xs[c][r0 + rr] = xv[rr];
      }
    }
    __syncthreads();
  }
  LT(5);
#pragma unroll 4
  for (int idx = t; idx < NB * NB; idx += LEAF_THREADS) {
    const int i = idx & (NB - 1), j = idx >> 6;
    if (i >= nb || j >= nb) continue;
    if (write_L) A[i + (int64_t)j * lda] = (i >= j) ? Ls[j][i] : T(0);
    X[i + (int64_t)j * ldx] = (i >= j) ? Xs[j][i] : T(0);
  }
  LT(6);
  if (t < 32) {  // 2 sum ln L_jj, fixed order
    double sacc = log((double)diag[t]) + log((double)diag[t + 32]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sacc += __shfl_down_sync(0xffffffffu, sacc, o);
    if (t == 0) {
      *logdet_slot = 2.0 * sacc;
      if (fail_sm != INT_MAX && fail_sm < nb) atomicMin(fail_col, col0 + fail_sm);
    }
  }
#ifdef CGGM_LEAF_TIMING
  LT(7);
  if (t == 0 && col0 == 0)
    printf("leaf clocks: load %lld panel0 %lld potrf %lld trtri %lld store %lld logdet %lld total %lld\n",
           lt_[1] - lt_[0], lt_[2] - lt_[1], lt_[4] - lt_[1], lt_[5] - lt_[4], lt_[6] - lt_[5], lt_[7] - lt_[6],
           lt_[7] - lt_[0]);
#endif
#undef LT
}

// ---------------------------------------------------------------------------------------------
// Full-inverse leaf by the same recursion as node() below, carried out inside one CTA in shared
// memory: node(64) = node(32), T = A21 X11^T, {A22 -= T T^T, A21 := T X11}, node(32),
// X21 = -X22 A21, down to 8x8 base blocks that one warp factors and inverts in registers.  The
// dependency chain is 8 base blocks (8 pivots each: rsqrt + two FP64 latencies) plus three levels
// of short products, instead of 64 shuffle-driven pivot steps and a 64-step inverse sweep
// (profiles: 50k -> ~18k cycles per 64-column leaf).
template <typename T>
struct LeafRec {
  T (*L)[NB + 1];   // [col][row]: the block being factored (A11 regions become T)
  T (*X)[NB + 1];   // [col][row]: L^{-1}
  T* diag;
  T* invd;
  int* fail_sm;
};

// 8x8 base block at offset s: warp 0 (every lane redundantly holds the block), lane c < 8 then
// computes column c of the inverse
template <typename T>
__device__ __forceinline__ void leaf_base8(const LeafRec<T>& R, int s) {
  const int lane = threadIdx.x & 31;
  if ((threadIdx.x >> 5) == 0) {
    T a[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j <= i; ++j) a[i][j] = R.L[s + j][s + i];
    T inv[8];
    int bad = -1;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const T d = a[j][j];
      if ((!(d > T(0)) || !isfinite(d)) && bad < 0) bad = j;
      inv[j] = rsqrt_t(d);
      a[j][j] = d * inv[j];
#pragma unroll
      for (int i = j + 1; i < 8; ++i) a[i][j] *= inv[j];
#pragma unroll
      for (int k = j + 1; k < 8; ++k)
#pragma unroll
        for (int i = k; i < 8; ++i) a[i][k] = fma_t(-a[i][j], a[k][j], a[i][k]);
    }
    if (lane < 8) {
      const int c = lane;
      T x[8];
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        T acc = T(0);
#pragma unroll
        for (int m = 0; m < r; ++m) acc = fma_t(-a[r][m], x[m], acc);
        x[r] = (r < c) ? T(0) : ((r == c) ? inv[r] : acc * inv[r]);
      }
#pragma unroll
      for (int r = 0; r < 8; ++r)
        if (r >= c) R.X[s + c][s + r] = x[r];
    }
    if (lane == 0) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        R.diag[s + j] = a[j][j];
        R.invd[s + j] = inv[j];
      }
      if (bad >= 0) atomicMin(R.fail_sm, s + bad);
    }
  }
  __syncthreads();
}

// One product phase on 8x8 DMMA fragments of an H x H output (fp64): warp w takes fragments
// w, w + 8, ...; a(i, m) and b(m, k) read the operands from shared memory, c0 / c1 the lane's two
// initial accumulators (C[g][2t], C[g][2t+1]), st writes them back.
template <int H, bool LOWER, class FA, class FB, class FC, class FS>
__device__ __forceinline__ void frag_phase(FA a, FB b, FC cinit, FS st) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  constexpr int NF = H / 8;
  for (int f = warp; f < NF * NF; f += LEAF_THREADS / 32) {
    const int fi = f % NF, fk = f / NF;
    if (LOWER && fi < fk) continue;
    const int i = fi * 8 + g, k0 = fk * 8 + 2 * t;
    double c0, c1;
    cinit(i, k0, c0, c1);
#pragma unroll
    for (int kk = 0; kk < H / 4; ++kk) ptx::dmma_8x8x4(c0, c1, a(i, 4 * kk + t), b(4 * kk + t, fk * 8 + g));
    st(i, k0, c0, c1);
  }
}

// the products of one recursion level: block [s, s + 2H), halves of width H.  X blocks hold zeros
// above their diagonal and the loads put zeros above A's, so every dot product runs over the full
// length H (no triangular bounds).
template <typename T, int H>
__device__ __forceinline__ void leaf_products_down(const LeafRec<T>& R, int s) {
  const int a = s + H;   // first row/col of the second half
  if constexpr (sizeof(T) == 8) {
    auto L = R.L;
    auto X = R.X;
    auto zero = [](int, int, double& c0, double& c1) { c0 = 0.0; c1 = 0.0; };
    // T = A21 X11^T  (T[i][k] = sum_m A21[i][m] X11[k][m]) -> over the A11 block (not read here)
    frag_phase<H, false>([&](int i, int m) { return (double)L[s + m][a + i]; },
                         [&](int m, int k) { return (double)X[s + m][s + k]; }, zero,
                         [&](int i, int k, double c0, double c1) {
                           L[s + k][s + i] = c0;
                           L[s + k + 1][s + i] = c1;
                         });
    __syncthreads();
    // A22 -= T T^T (lower fragments) and A21 := T X11 (A21[i][k] = sum_m T[i][m] X11[m][k])
    frag_phase<H, true>([&](int i, int k) { return -(double)L[s + k][s + i]; },
                        [&](int k, int j) { return (double)L[s + k][s + j]; },
                        [&](int i, int j, double& c0, double& c1) {
                          c0 = L[a + j][a + i];
                          c1 = L[a + j + 1][a + i];
                        },
                        [&](int i, int j, double c0, double c1) {
                          L[a + j][a + i] = c0;
                          L[a + j + 1][a + i] = c1;
                        });
    frag_phase<H, false>([&](int i, int m) { return (double)L[s + m][s + i]; },
                         [&](int m, int k) { return (double)X[s + k][s + m]; }, zero,
                         [&](int i, int k, double c0, double c1) {
                           L[s + k][a + i] = c0;
                           L[s + k + 1][a + i] = c1;
                         });
    __syncthreads();
  } else {
    T tv[(H * H + LEAF_THREADS - 1) / LEAF_THREADS];
#pragma unroll
    for (int u = 0; u * LEAF_THREADS < H * H; ++u) {
      const int idx = threadIdx.x + u * LEAF_THREADS;
      T acc = T(0);
      if (idx < H * H) {
        const int i = idx % H, k = idx / H;
#pragma unroll 8
        for (int m = 0; m < H; ++m) acc = fma_t(R.L[s + m][a + i], R.X[s + m][s + k], acc);
      }
      tv[u] = acc;
    }
#pragma unroll
    for (int u = 0; u * LEAF_THREADS < H * H; ++u) {
      const int idx = threadIdx.x + u * LEAF_THREADS;
      if (idx < H * H) R.L[s + idx / H][s + idx % H] = tv[u];
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < 2 * H * H; idx += LEAF_THREADS) {
      const int w = idx / (H * H), e = idx - w * H * H, i = e % H, j = e / H;
      if (w == 0) {
        if (i < j) continue;
        T acc = R.L[a + j][a + i];
#pragma unroll 8
        for (int k = 0; k < H; ++k) acc = fma_t(-R.L[s + k][s + i], R.L[s + k][s + j], acc);
        R.L[a + j][a + i] = acc;
      } else {
        T acc = T(0);
#pragma unroll 8
        for (int m = 0; m < H; ++m) acc = fma_t(R.L[s + m][s + i], R.X[s + j][s + m], acc);
        R.L[s + j][a + i] = acc;
      }
    }
    __syncthreads();
  }
}

// X21 = -X22 A21  (X21[i][k] = -sum_m X22[i][m] A21[m][k])
template <typename T, int H>
__device__ __forceinline__ void leaf_products_up(const LeafRec<T>& R, int s) {
  const int a = s + H;
  if constexpr (sizeof(T) == 8) {
    auto L = R.L;
    auto X = R.X;
    frag_phase<H, false>([&](int i, int m) { return -(double)X[a + m][a + i]; },
                         [&](int m, int k) { return (double)L[s + k][a + m]; },
                         [](int, int, double& c0, double& c1) { c0 = 0.0; c1 = 0.0; },
                         [&](int i, int k, double c0, double c1) {
                           X[s + k][a + i] = c0;
                           X[s + k + 1][a + i] = c1;
                         });
  } else {
    for (int idx = threadIdx.x; idx < H * H; idx += LEAF_THREADS) {
      const int i = idx % H, k = idx / H;
      T acc = T(0);
#pragma unroll 8
      for (int m = 0; m < H; ++m) acc = fma_t(-R.X[a + m][a + i], R.L[s + k][a + m], acc);
      R.X[s + k][a + i] = acc;
    }
  }
  __syncthreads();
}

template <typename T, int N>
struct LeafNode {
  __device__ __forceinline__ static void run(const LeafRec<T>& R, int s) {
    LeafNode<T, N / 2>::run(R, s);
    leaf_products_down<T, N / 2>(R, s);
    LeafNode<T, N / 2>::run(R, s + N / 2);
    leaf_products_up<T, N / 2>(R, s);
  }
};
template <typename T>
struct LeafNode<T, 8> {
  __device__ __forceinline__ static void run(const LeafRec<T>& R, int s) { leaf_base8<T>(R, s); }
};

template <typename T>
__global__ void __launch_bounds__(LEAF_THREADS, CGGM_LEAF_MINB) leaf_rec_inverse(const T* A, int64_t lda, int nb, T* Xo,
                                                                                  int64_t ldx, double* logdet_slot,
                                                                                  int* fail_col, int col0) {
  extern __shared__ __align__(16) unsigned char leaf_raw[];
  T(*Ls)[NB + 1] = reinterpret_cast<T(*)[NB + 1]>(leaf_raw);
  T(*Xs)[NB + 1] = reinterpret_cast<T(*)[NB + 1]>(leaf_raw + NB * (NB + 1) * sizeof(T));
  __shared__ T diag[NB], invd[NB];
  __shared__ int fail_sm;
  const int t = threadIdx.x;
  ptx::pdl_wait();
  ptx::pdl_trigger();   // (one CTA: the successor may be scheduled now; it waits for this grid to complete)
  {
    constexpr int PER = NB * NB / LEAF_THREADS, HALF = PER / 2;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      T v[HALF];
#pragma unroll
      for (int u = 0; u < HALF; ++u) {
        const int idx = t + LEAF_THREADS * (u + h * HALF), i = idx & (NB - 1), j = idx >> 6;
        v[u] = (i < nb && j < nb && i >= j) ? A[i + (int64_t)j * lda] : T(0);
      }
#pragma unroll
      for (int u = 0; u < HALF; ++u) {
        const int idx = t + LEAF_THREADS * (u + h * HALF), i = idx & (NB - 1), j = idx >> 6;
        Ls[j][i] = (i < nb && j < nb) ? v[u] : ((i == j) ? T(1) : T(0));
        Xs[j][i] = T(0);
      }
    }
  }
  if (t == 0) fail_sm = INT_MAX;
  __syncthreads();
#ifdef CGGM_LEAF_TIMING
  const long long c0 = clock64();
#endif
  LeafRec<T> R{Ls, Xs, diag, invd, &fail_sm};
  LeafNode<T, NB>::run(R, 0);
#ifdef CGGM_LEAF_TIMING
  if (t == 0 && col0 == 0) printf("leaf_rec clocks: recursion %lld\n", clock64() - c0);
#endif
#pragma unroll 4
  for (int idx = t; idx < NB * NB; idx += LEAF_THREADS) {
    const int i = idx & (NB - 1), j = idx >> 6;
    if (i >= nb || j >= nb) continue;
    Xo[i + (int64_t)j * ldx] = (i >= j) ? Xs[j][i] : T(0);
  }
  if (t < 32) {  // 2 sum ln L_jj, fixed order
    double sacc = log((double)diag[t]) + log((double)diag[t + 32]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sacc += __shfl_down_sync(0xffffffffu, sacc, o);
    if (t == 0) {
      *logdet_slot = 2.0 * sacc;
      if (fail_sm != INT_MAX && fail_sm < nb) atomicMin(fail_col, col0 + fail_sm);
    }
  }
}

// CGGM_SPLIT_PANEL = B > 0: nodes wider than 2B split off a leading panel of B columns instead of
// halving (a right-looking recursion with recursive panels: each level's latency-bound panel
// factorisation overlaps the previous level's deferred trailing update); 0 = halving everywhere
int split_panel() {
  static int v = [] {
    const char* e = std::getenv("CGGM_SPLIT_PANEL");
    return e ? std::max(0, std::atoi(e)) / 128 * 128 : 0;
  }();
  return v;
}

int split_point(int64_t n) {
  const int64_t gran = n > 4 * 128 ? 128 : NB;
  if (split_panel() > 0 && n > 2 * split_panel()) return split_panel();
  int64_t n1 = (n / 2) / gran * gran;
  if (n1 <= 0) n1 = gran;
  if (n1 >= n) n1 = n - NB;
  return (int)n1;
}

// Per-depth slices of the full-inverse temporaries: the T of a node at depth d lives in slice d,
// so deferred side-stream products of a parent never share memory with a running child.
void tmp_depth_sizes(int64_t n, int depth, std::vector<size_t>& mx) {
  if (n <= NB) return;
  const int64_t n1 = split_point(n), n2 = n - n1;
  if ((int)mx.size() <= depth) mx.resize(depth + 1, 0);
  mx[depth] = std::max(mx[depth], (size_t)(n2 + (n2 & 1)) * (size_t)n1);
  tmp_depth_sizes(n1, depth + 1, mx);
  tmp_depth_sizes(n2, depth + 1, mx);
}

std::vector<size_t> tmp_slices(int64_t n, size_t* total) {
  std::vector<size_t> mx, off;
  tmp_depth_sizes(n, 0, mx);
  size_t acc = 0;
  for (size_t v : mx) {
    off.push_back(acc);
    acc += (v + 31) / 32 * 32;
  }
  if (total) *total = acc;
  return off;
}

cudaEvent_t la_record(Ctx* c, cudaStream_t s) {
  if (c->la_next >= c->la_events.size()) {
    cudaEvent_t e;
    CGGM_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    c->la_events.push_back(e);
  }
  cudaEvent_t e = c->la_events[c->la_next++];
  CGGM_CUDA_CHECK(cudaEventRecord(e, s));
  return e;
}

// enqueue on stream s (after `wait`, if any) for the lifetime of this object
struct OnStream {
  Ctx* c;
  cudaStream_t prev;
  OnStream(Ctx* c_, cudaStream_t s, cudaEvent_t wait) : c(c_), prev(c_->stream) {
    if (wait) CGGM_CUDA_CHECK(cudaStreamWaitEvent(s, wait, 0));
    c->stream = s;
  }
  ~OnStream() { c->stream = prev; }
};

// potrf-only mode: diagonal subtrees up to this size keep their inverse (CGGM_BINV overrides)
int binv_size() {
  static int v = [] {
    const char* e = std::getenv("CGGM_BINV");
    return e ? std::atoi(e) : 4096;
  }();
  return v;
}
#define BINV binv_size()

template <typename T>
struct Rec {
  Ctx* c;
  bool full_inverse;
  T* leafinv;   // compact leaf inverses (potrf-only mode), leaf k at leafinv + k*NB*NB, ld NB
  double* logdet_slots;
  int* fail_col;
  T* tmp;       // full-inverse recursion temporaries: one slice per recursion depth (tmp_off)
  size_t tmp_elems;
  std::vector<size_t> tmp_off;
  // lookahead streams (null upd/bg: everything on the chain, c->stream)
  cudaStream_t upd, bg;
  T* xdiag;     // potrf-only: inverse of the diagonal block at col0 stored at xdiag + col0 (ld ldxd)
  int64_t ldxd;
  T* tmp2;      // potrf-only: out-of-place product buffer for B := B Xblock^T
  size_t tmp2_elems;
  // full-inverse mode with sig != null: Sigma = L^{-T} L^{-1} assembled block by block as the
  // recursion finishes the blocks of L^{-1} (sig_node), on stream sgs (c->stream when null)
  T* sig = nullptr;
  int64_t ldsig = 0;
  int64_t sig_min = 0;
  cudaStream_t sgs = nullptr;
};

// B := B Xb^T for the inverse Xb (n x n, lower) of one diagonal block, out of place through tmp2
template <typename T>
void apply_block_inverse(Rec<T>& R, ViewT<T> B, const T* xb, int64_t ldxb, int64_t n) {
  if (B.rows == 0) return;
  const int64_t ldt = B.rows + (B.rows & 1);
  if ((size_t)(ldt * n) > R.tmp2_elems) throw CudaError{CGGM_ERR_OOM, "block-inverse temp too small"};
  EpilogueT<T> e; e.out1 = R.tmp2; e.ld1 = ldt;
  gemm(R.c, false, true, B.rows, n, n, B.p, B.ld, xb, ldxb, e, B_KLE_N);
  copy2d(R.c, B, R.tmp2, ldt);
}

template <typename T>
void trsm_rec(Rec<T>& R, ViewT<T> B, ViewT<T> L, int64_t col0);

template <typename T>
void leaf(Rec<T>& R, ViewT<T> A, ViewT<T> X, int64_t col0) {
  const int nb = (int)A.rows;
  // gate (Ctx::gate_ev): recorded on the chain when the recursion reaches the first leaf at or past
  // column gate_cols -- another stream's work can be held back until the factorisation is that far
  if (R.c->gate_ev && !R.c->gate_done && col0 >= R.c->gate_cols && R.full_inverse && R.c->lane == 0) {
    CGGM_CUDA_CHECK(cudaEventRecord(R.c->gate_ev, R.c->stream));
    R.c->gate_done = true;
  }
  T* xp;
  int64_t ldx;
  if (R.full_inverse) {
    xp = X.p;
    ldx = X.ld;
  } else {
    xp = R.leafinv + (col0 / NB) * NB * NB;
    ldx = NB;
  }
  CGGM_ONCE_PER_DEVICE({
    CGGM_CUDA_CHECK(cudaFuncSetAttribute(leaf_potrf_trtri<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, leaf_smem_bytes<T>()));
  });
  Prof pr(R.c, TAG_CHOL_LEAF);
  if (R.full_inverse && !R.c->leaf_sweep) {
    CGGM_ONCE_PER_DEVICE({
      CGGM_CUDA_CHECK(cudaFuncSetAttribute(leaf_rec_inverse<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           leaf_smem_bytes<T>()));
    });
    launch_pdl(R.c, leaf_rec_inverse<T>, dim3(1), dim3(LEAF_THREADS), leaf_smem_bytes<T>(), (const T*)A.p, A.ld, nb,
               xp, ldx, R.logdet_slots + col0 / NB, R.fail_col, (int)col0);
    post_launch(R.c, "leaf_rec_inverse");
    return;
  }
  launch_pdl(R.c, leaf_potrf_trtri<T>, dim3(1), dim3(LEAF_THREADS), leaf_smem_bytes<T>(), A.p, A.ld, nb, xp, ldx,
             R.full_inverse ? 0 : 1, R.logdet_slots + col0 / NB, R.fail_col, (int)col0);
  post_launch(R.c, "leaf_potrf_trtri");
}

// ---------------------------------------------------------------- Sigma interleaved with the recursion
// For a node with X = L^{-1} of its diagonal block = [[X11, 0], [X21, X22]] (Sigma = Lambda^{-1}
// = L^{-T} L^{-1}), its block of X^T X is
//   S11 = X11^T X11 + X21^T X21,   S21 = X22^T X21 (S12 = S21^T),   S22 = X22^T X22.
// X11^T X11 and X22^T X22 are the children's own blocks (formed as soon as each child's inverse is
// final, recursively), so only S21 and the update S11 += X21^T X21 wait for X21, the node's last
// product: the lauum work of the lower levels runs inside the recursion, in the SMs its
// latency-bound stretches leave idle, instead of as one product after it.  Nodes below sig_min form
// their block in one symmetric product.  Same arithmetic per entry as the one-shot product up to
// the order of the k-sums (a block's sum is split at the child boundaries).
// the Sigma pieces go to the Sigma stream after everything enqueued so far on the chain (the blocks
// of L^{-1} they read); returns the chain stream to restore afterwards
template <typename T>
cudaStream_t sig_enqueue_begin(Rec<T>& R) {
  const cudaStream_t prev = R.c->stream;
  if (R.sgs) {
    CGGM_CUDA_CHECK(cudaStreamWaitEvent(R.sgs, la_record(R.c, prev), 0));
    R.c->stream = R.sgs;
  }
  return prev;
}

template <typename T>
void sig_block_product(Rec<T>& R, ViewT<T> X, int64_t col0) {   // S_node = X^T X (X lower triangular)
  const int64_t n = X.rows;
  const cudaStream_t prev = sig_enqueue_begin(R);
  {
    Phase ph(R.c, TAG_LAUUM);   // (the GEMMs record under this tag)
    EpilogueT<T> e; e.out1 = R.sig + col0 + col0 * R.ldsig; e.ld1 = R.ldsig;
    gemm(R.c, true, false, n, n, n, X.p, X.ld, X.p, X.ld, e, A_KGE_M | B_KGE_N | SYM_LOWER | SYM_MIRROR);
  }
  R.c->stream = prev;
}

template <typename T>
void sig_node_pieces(Rec<T>& R, ViewT<T> X11, ViewT<T> X21, ViewT<T> X22, int64_t col0) {
  const int64_t n1 = X11.rows, n2 = X22.rows;
  T* S11 = R.sig + col0 + col0 * R.ldsig;
  const cudaStream_t prev = sig_enqueue_begin(R);
  {
    Phase ph(R.c, TAG_LAUUM);   // (the GEMMs record under this tag)
    {  // S21 = X22^T X21 (X22 lower: op(A) = X22^T has k >= m), S12 = S21^T by the mirrored epilogue
      EpilogueT<T> e; e.out1 = S11 + n1; e.ld1 = R.ldsig; e.mir1 = S11 + n1 * R.ldsig;
      gemm(R.c, true, false, n2, n1, n2, X22.p, X22.ld, X21.p, X21.ld, e, A_KGE_M | SYM_MIRROR);
    }
    {  // S11 += X21^T X21 (after X11^T X11, enqueued earlier on this stream)
      EpilogueT<T> e; e.out1 = S11; e.ld1 = R.ldsig; e.in1a = S11; e.ld1a = R.ldsig; e.b1 = 1.0;
      gemm(R.c, true, false, n1, n1, n2, X21.p, X21.ld, X21.p, X21.ld, e, SYM_LOWER | SYM_MIRROR);
    }
  }
  R.c->stream = prev;
}

// A is (n + extra) x n: the square block being factored with `extra` appended rows below it
// (potrf-only mode).  Factoring the augmented [Lambda; W] leaves Z = W L^{-T} in the bottom rows
// (block Cholesky of [[Lambda, W^T], [W, .]]), so the objective's triangular solve is carried by
// the same recursive GEMMs with taller panels.
// pending: event of the parent's deferred update of this node's trailing block A[n1:, n1:]
// (full-inverse lookahead); waited on before this node's own trailing update
// sig (full-inverse mode with R.sig): this node owns its block of Sigma (see sig_node_pieces)
template <typename T>
void node(Rec<T>& R, ViewT<T> A, ViewT<T> X, int64_t col0, int depth = 0, cudaEvent_t pending = nullptr,
          bool sig = false) {
  const int64_t n = A.cols, extra = A.rows - A.cols;
  Ctx* c = R.c;
  if (sig && n < R.sig_min) {   // the whole block in one product once this subtree's inverse is final
    node(R, A, X, col0, depth, pending, false);
    sig_block_product(R, X, col0);
    return;
  }
  if (!R.full_inverse && R.xdiag && n <= BINV) {
    // potrf-only: factor this diagonal subtree in full-inverse mode, keeping its inverse for the
    // triangular solves of the panels to its right and of the appended rows below
    Rec<T> R2 = R;
    R2.full_inverse = true;
    R2.tmp_off = tmp_slices(n, nullptr);
    ViewT<T> Xb{R.xdiag + col0, R.ldxd, n, n};
    node(R2, A.sub(0, 0, n, n), Xb, col0, 0);
    if (extra > 0) apply_block_inverse(R, A.sub(n, 0, extra, n), Xb.p, Xb.ld, n);
    return;
  }
  if (n <= NB) {
    leaf(R, A.sub(0, 0, n, n), X, col0);
    if (extra > 0) {  // bottom rows: B := B Xleaf^T (N <= 64: one tile column, in place)
      const T* xl = R.leafinv + (col0 / NB) * NB * NB;
      EpilogueT<T> e; e.out1 = A.p + n; e.ld1 = A.ld;
      gemm(c, false, true, extra, n, n, A.p + n, A.ld, xl, NB, e, B_KLE_N);
    }
    return;
  }
  const int64_t n1 = split_point(n), n2 = n - n1;
  ViewT<T> A11 = A.sub(0, 0, n1, n1), A21 = A.sub(n1, 0, n2 + extra, n1), A22 = A.sub(n1, n1, n2 + extra, n2);
  if (R.full_inverse) {
    if (extra) throw CudaError{CGGM_ERR_UNSUPPORTED, "augmented rows need potrf-only mode"};
    ViewT<T> X11 = X.sub(0, 0, n1, n1), X21 = X.sub(n1, 0, n2, n1), X22 = X.sub(n1, n1, n2, n2);
    node(R, A11, X11, col0, depth + 1, nullptr, sig);
    if ((size_t)depth >= R.tmp_off.size()) throw CudaError{CGGM_ERR_OOM, "recursion temp too small"};
    ViewT<T> Tm{R.tmp + R.tmp_off[depth], n2 + (n2 & 1), n2, n1};
    if (R.tmp_off[depth] + (size_t)(Tm.ld * n1) > R.tmp_elems) throw CudaError{CGGM_ERR_OOM, "recursion temp too small"};
    {  // T = A21 X11^T  (L21)
      EpilogueT<T> e; e.out1 = Tm.p; e.ld1 = Tm.ld;
      gemm(c, false, true, n2, n1, n1, A21.p, A21.ld, X11.p, X11.ld, e, B_KLE_N);
    }
    // Lookahead: node(A22) first factors its own leading block A22[0:n21, 0:n21] and forms its panel
    // from A22[n21:, 0:n21]; only its trailing update needs A22[n21:, n21:].  So the chain updates
    // the leading block column of A22 and the rest of A22 -= T T^T (and A21 := T X11, needed only
    // by X21 below) run on low-priority side streams, filling the SMs the recursion leaves idle.
    if (pending) CGGM_CUDA_CHECK(cudaStreamWaitEvent(c->stream, pending, 0));  // A22 complete
    const int64_t n21 = n2 > NB ? split_point(n2) : n2, n22 = n2 - n21;
    const bool defer = R.upd && c->la_min > 0 && n22 >= c->la_min;
    cudaEvent_t ev_upd = nullptr, ev_a21 = nullptr;
    if (defer) {
      cudaEvent_t ev_t = la_record(c, c->stream);
      {  // A22[:, 0:n21] -= T T[0:n21]^T (lower trapezoid), on the chain
        EpilogueT<T> e; e.out1 = A22.p; e.ld1 = A22.ld; e.a1 = -1.0; e.in1a = A22.p; e.ld1a = A22.ld; e.b1 = 1.0;
        gemm(c, false, true, n2, n21, n1, Tm.p, Tm.ld, Tm.p, Tm.ld, e, SYM_LOWER);
      }
      {  // A22[n21:, n21:] -= T[n21:] T[n21:]^T (lower), deferred
        OnStream os(c, R.upd, ev_t);
        ViewT<T> C = A22.sub(n21, n21, n22, n22);
        EpilogueT<T> e; e.out1 = C.p; e.ld1 = C.ld; e.a1 = -1.0; e.in1a = C.p; e.ld1a = C.ld; e.b1 = 1.0;
        gemm(c, false, true, n22, n22, n1, Tm.p + n21, Tm.ld, Tm.p + n21, Tm.ld, e, SYM_LOWER);
        ev_upd = la_record(c, c->stream);
      }
      {  // A21 := T X11, deferred
        OnStream os(c, R.bg, ev_t);
        EpilogueT<T> e; e.out1 = A21.p; e.ld1 = A21.ld;
        gemm(c, false, false, n2, n1, n1, Tm.p, Tm.ld, X11.p, X11.ld, e, B_KGE_N);
        ev_a21 = la_record(c, c->stream);
      }
    } else {
      {  // A22 -= T T^T (lower)
        EpilogueT<T> e; e.out1 = A22.p; e.ld1 = A22.ld; e.a1 = -1.0; e.in1a = A22.p; e.ld1a = A22.ld; e.b1 = 1.0;
        gemm(c, false, true, n2, n2, n1, Tm.p, Tm.ld, Tm.p, Tm.ld, e, SYM_LOWER);
      }
      {  // A21 := T X11
        EpilogueT<T> e; e.out1 = A21.p; e.ld1 = A21.ld;
        gemm(c, false, false, n2, n1, n1, Tm.p, Tm.ld, X11.p, X11.ld, e, B_KGE_N);
      }
    }
    node(R, A22, X22, col0 + n1, depth + 1, ev_upd, sig);
    if (ev_a21) CGGM_CUDA_CHECK(cudaStreamWaitEvent(c->stream, ev_a21, 0));
    {  // X21 = -X22 A21
      EpilogueT<T> e; e.out1 = X21.p; e.ld1 = X21.ld; e.a1 = -1.0;
      gemm(c, false, false, n2, n1, n2, X22.p, X22.ld, A21.p, A21.ld, e, A_KLE_M);
    }
    if (sig) sig_node_pieces(R, X11, X21, X22, col0);
  } else {
    node(R, A11, X, col0, depth + 1);
    trsm_rec(R, A21, A11, col0);
    {  // A22 -= A21 A21^T over the lower trapezoid (square part + appended rows)
      EpilogueT<T> e; e.out1 = A22.p; e.ld1 = A22.ld; e.a1 = -1.0; e.in1a = A22.p; e.ld1a = A22.ld; e.b1 = 1.0;
      gemm(c, false, true, n2 + extra, n2, n1, A21.p, A21.ld, A21.p, A21.ld, e, SYM_LOWER);
    }
    node(R, A22, X, col0 + n1, depth + 1);
  }
}

// B (m x n) := B L^{-T}, L the factor of the diagonal block at col0.  Same split tree as node(),
// so the recursion reaches exactly the blocks whose inverses node() kept.
template <typename T>
void trsm_rec(Rec<T>& R, ViewT<T> B, ViewT<T> L, int64_t col0) {
  const int64_t n = L.rows;
  if (B.rows == 0) return;
  if (R.xdiag && n <= BINV) {
    apply_block_inverse(R, B, R.xdiag + col0, R.ldxd, n);
    return;
  }
  if (n <= NB) {
    // B := B Xleaf^T; N = n <= 64 fits one tile column, so each CTA reads only the rows it writes
    const T* xl = R.leafinv + (col0 / NB) * NB * NB;
    EpilogueT<T> e; e.out1 = B.p; e.ld1 = B.ld;
    gemm(R.c, false, true, B.rows, n, n, B.p, B.ld, xl, NB, e, B_KLE_N);
    return;
  }
  const int64_t n1 = split_point(n), n2 = n - n1;
  ViewT<T> B1 = B.sub(0, 0, B.rows, n1), B2 = B.sub(0, n1, B.rows, n2);
  trsm_rec(R, B1, L.sub(0, 0, n1, n1), col0);
  {  // B2 -= B1 L21^T
    ViewT<T> L21 = L.sub(n1, 0, n2, n1);
    EpilogueT<T> e; e.out1 = B2.p; e.ld1 = B2.ld; e.a1 = -1.0; e.in1a = B2.p; e.ld1a = B2.ld; e.b1 = 1.0;
    gemm(R.c, false, true, B.rows, n2, n1, B1.p, B1.ld, L21.p, L21.ld, e, 0);
  }
  trsm_rec(R, B2, L.sub(n1, n1, n2, n2), col0 + n1);
}

}  // namespace

int leaf_nb() { return NB; }

template <typename T>
void potrf_recursive(Ctx* c, ViewT<T> A, ViewT<T> Linv, bool full_inverse, T* leafinv, double* logdet_slots,
                     int* fail_col_dev, T* tmp, size_t tmp_elems, T* xdiag, int64_t ldxd, T* tmp2,
                     size_t tmp2_elems, T* sigma, int64_t ldsigma) {
  Rec<T> R{c, full_inverse, leafinv, logdet_slots, fail_col_dev, tmp, tmp_elems, {}, nullptr, nullptr,
           xdiag, ldxd, tmp2, tmp2_elems};
  if (full_inverse) R.tmp_off = tmp_slices(A.cols, nullptr);
  const bool sig = full_inverse && sigma != nullptr;
  if (sig) {
    if ((sizeof(T) == 8 ? c->sig_min : c->sig_min_f32) < 2 * NB)
      throw CudaError{CGGM_ERR_INVALID_ARG, "interleaved Sigma needs sig_min >= 128"};
    R.sig = sigma;
    R.ldsig = ldsigma;
    R.sig_min = sizeof(T) == 8 ? c->sig_min : c->sig_min_f32;
  }
  Phase ph(c, TAG_CHOL_GEMM);
  const int lane = c->lane;
  if (c->la_min <= 0) {
    node(R, A, Linv, 0, 0, nullptr, sig);
    return;
  }
  // lookahead: the recursion's critical chain on a high-priority stream, deferred products on two
  // lower-priority side streams; forked from and joined back into c->stream
  if (!c->la_chain[lane]) {
    const int b = 2 + 3 * lane;
    CGGM_CUDA_CHECK(cudaStreamCreateWithPriority(&c->la_chain[lane], cudaStreamNonBlocking, stream_priority(b)));
    CGGM_CUDA_CHECK(cudaStreamCreateWithPriority(&c->la_upd[lane], cudaStreamNonBlocking, stream_priority(b + 1)));
    CGGM_CUDA_CHECK(cudaStreamCreateWithPriority(&c->la_bg[lane], cudaStreamNonBlocking, stream_priority(b + 2)));
  }
  if (sig && !c->la_sig) CGGM_CUDA_CHECK(cudaStreamCreateWithPriority(&c->la_sig, cudaStreamNonBlocking, stream_priority(8)));
  c->la_next = 0;
  cudaStream_t s_in = c->stream, chain = c->la_chain[lane];
  R.upd = c->la_upd[lane];
  R.bg = c->la_bg[lane];
  R.sgs = sig ? c->la_sig : nullptr;
  cudaEvent_t ev_in = la_record(c, s_in);
  for (cudaStream_t st : std::initializer_list<cudaStream_t>{chain, R.upd, R.bg}) CGGM_CUDA_CHECK(cudaStreamWaitEvent(st, ev_in, 0));
  if (sig) CGGM_CUDA_CHECK(cudaStreamWaitEvent(R.sgs, ev_in, 0));
  {
    OnStream os(c, chain, nullptr);
    const auto t0 = std::chrono::steady_clock::now();
    node(R, A, Linv, 0, 0, nullptr, sig);
    if (std::getenv("CGGM_HOSTPROF"))
      std::fprintf(stderr, "potrf_recursive q=%lld full=%d host enqueue %.3f ms\n", (long long)A.cols, (int)full_inverse,
                   std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
  }
  for (cudaStream_t st : std::initializer_list<cudaStream_t>{chain, R.upd, R.bg}) CGGM_CUDA_CHECK(cudaStreamWaitEvent(s_in, la_record(c, st), 0));
  if (sig) CGGM_CUDA_CHECK(cudaStreamWaitEvent(s_in, la_record(c, R.sgs), 0));
}

size_t chol_tmp_elems(int64_t q) {
  size_t total = 0;
  tmp_slices(q, &total);
  return total + 64;
}

int block_inverse_size() { return BINV; }

template <typename T>
void lauum(Ctx* c, ViewT<T> Linv, ViewT<T> Sigma) {
  const int64_t q = Linv.rows;
  Phase ph(c, TAG_LAUUM);
  EpilogueT<T> e; e.out1 = Sigma.p; e.ld1 = Sigma.ld;
  gemm(c, true, false, q, q, q, Linv.p, Linv.ld, Linv.p, Linv.ld, e, A_KGE_M | B_KGE_N | SYM_LOWER | SYM_MIRROR);
}

template void potrf_recursive<double>(Ctx*, ViewT<double>, ViewT<double>, bool, double*, double*, int*, double*,
                                      size_t, double*, int64_t, double*, size_t, double*, int64_t);
template void potrf_recursive<float>(Ctx*, ViewT<float>, ViewT<float>, bool, float*, double*, int*, float*, size_t,
                                     float*, int64_t, float*, size_t, float*, int64_t);
template void lauum<double>(Ctx*, ViewT<double>, ViewT<double>);
template void lauum<float>(Ctx*, ViewT<float>, ViewT<float>);

}  // namespace cggm
