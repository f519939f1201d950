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
#include <climits>

#include "common.cuh"

namespace cggm {
namespace {

__device__ __forceinline__ double rsqrt_t(double x) { return rsqrt(x); }
__device__ __forceinline__ float rsqrt_t(float x) { return rsqrtf(x); }
__device__ __forceinline__ double fma_t(double a, double b, double c) { return fma(a, b, c); }
__device__ __forceinline__ float fma_t(float a, float b, float c) { return fmaf(a, b, c); }

constexpr int NB = 64;
constexpr int LEAF_THREADS = 256;
template <typename T>
constexpr int leaf_smem_bytes() { return 2 * NB * (NB + 1) * (int)sizeof(T); }

// Leaf: Cholesky + triangular inverse of one nb x nb (nb <= 64) diagonal block in one CTA.
// 256 threads; thread t owns the 4x4 register blocks rows 4*(t&15).., cols 4*(t>>4).. of both
// the factor (a) and the inverse (x); rows/columns >= nb are padded with the identity (so L and
// L^{-1} are block-diag(., I)).  One fused sweep, ONE __syncthreads per column j:
//   before the barrier  - the owners of column j (one half-warp) receive the pivot d by warp
//     shuffle, test it, form inv = 1/sqrt(d), scale column j and publish it; the owners of row j
//     of X publish that row (not yet divided by L_jj);
//   after the barrier   - every thread applies the rank-1 Cholesky update to its block of a and
//     the forward-substitution update X[i,:] -= L_ij * X[j,:] * inv to its block of x.
// Buffers are double-buffered by column parity so no second barrier is needed.  The pivot test
// !(d > 0) records the first failing column (reading A10); log L_jj is summed in a fixed order.
template <typename T>
__global__ void __launch_bounds__(LEAF_THREADS) leaf_potrf_trtri(T* A, int64_t lda, int nb, T* X,
                                                                  int64_t ldx, int write_L, double* logdet_slot,
                                                                  int* fail_col, int col0) {
  extern __shared__ __align__(16) unsigned char leaf_raw[];
  T* leaf_smem = reinterpret_cast<T*>(leaf_raw);
  T(*Ls)[NB + 1] = reinterpret_cast<T(*)[NB + 1]>(leaf_smem);                   // Ls[col][row]
  T(*Xs)[NB + 1] = reinterpret_cast<T(*)[NB + 1]>(leaf_smem + NB * (NB + 1));  // Xs[col][row]
  __shared__ T cbuf[2][NB + 1];  // column j of L (rows > j); [NB] = 1/L_jj
  __shared__ T rbuf[2][NB];      // row j of X before the division by L_jj
  __shared__ T diag[NB];
  __shared__ int fail_sm;
  const int t = threadIdx.x, rb = t & 15, cb = t >> 4, lane = t & 31;
  for (int idx = t; idx < NB * NB; idx += LEAF_THREADS) {
    const int i = idx & (NB - 1), j = idx >> 6;
    T v;
    if (i < nb && j < nb) v = (i >= j) ? A[i + (int64_t)j * lda] : T(0);
    else v = (i == j) ? T(1) : T(0);
    Ls[j][i] = v;
  }
  if (t == 0) fail_sm = INT_MAX;
  __syncthreads();
  T a[4][4], x[4][4];
#pragma unroll
  for (int ii = 0; ii < 4; ++ii)
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      a[ii][kk] = Ls[4 * cb + kk][4 * rb + ii];
      x[ii][kk] = (4 * rb + ii == 4 * cb + kk) ? T(1) : T(0);
    }
  const bool has_lower = (rb >= cb);
  for (int jb = 0; jb < 16; ++jb) {
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) {
      const int j = 4 * jb + jj;
      T* cv = cbuf[jj & 1];
      T* rv = rbuf[jj & 1];
      if (cb == jb) {  // column-j owners (a half-warp)
        const unsigned hmask = (lane & 16) ? 0xffff0000u : 0x0000ffffu;
        const T d = __shfl_sync(hmask, a[jj][jj], (lane & 16) | jb);
        const T inv = rsqrt_t(d);
        const T ljj = d * inv;
        if (rb == jb) {
          if (!(d > 0.0) || !isfinite(d)) atomicMin(&fail_sm, j);
          diag[j] = ljj;
          cv[NB] = inv;
          a[jj][jj] = ljj;
        }
#pragma unroll
        for (int ii = 0; ii < 4; ++ii) {
          const int i = 4 * rb + ii;
          if (i > j) {
            a[ii][jj] *= inv;
            cv[i] = a[ii][jj];
          }
        }
      }
      if (rb == jb) {  // row-j owners of X publish the undivided row (columns <= j)
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) rv[4 * cb + cc] = x[jj][cc];
      }
      __syncthreads();
      const T inv = cv[NB];
      if (rb == jb) {
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) x[jj][cc] *= inv;
      }
      if (4 * rb + 3 > j) {
        T li[4], lk[4], xr[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          li[u] = cv[4 * rb + u];
          lk[u] = cv[4 * cb + u];
          xr[u] = rv[4 * cb + u] * inv;
        }
#pragma unroll
        for (int ii = 0; ii < 4; ++ii)
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const int i = 4 * rb + ii, k = 4 * cb + kk;
            if (i > j) {
              if (has_lower && k > j && i >= k) a[ii][kk] = fma_t(-li[ii], lk[kk], a[ii][kk]);
              if (k <= j) x[ii][kk] = fma_t(-li[ii], xr[kk], x[ii][kk]);
            }
          }
      }
    }
  }
#pragma unroll
  for (int ii = 0; ii < 4; ++ii)
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      const int i = 4 * rb + ii, k = 4 * cb + kk;
      Ls[k][i] = (i >= k) ? a[ii][kk] : T(0);
      Xs[k][i] = x[ii][kk];
    }
  __syncthreads();
  for (int idx = t; idx < nb * nb; idx += LEAF_THREADS) {
    const int i = idx % nb, j = idx / nb;
    if (write_L) A[i + (int64_t)j * lda] = Ls[j][i];
    X[i + (int64_t)j * ldx] = Xs[j][i];
  }
  if (t < 32) {  // 2 sum ln L_jj, fixed order: lane-strided partials then a fixed shuffle tree
    double s = 0.0;
    for (int j = t; j < NB; j += 32) s += log((double)diag[j]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if (t == 0) {
      *logdet_slot = 2.0 * s;
      if (fail_sm != INT_MAX && fail_sm < nb) atomicMin(fail_col, col0 + fail_sm);
    }
  }
}

int split_point(int64_t n) {
  const int64_t gran = n > 4 * 128 ? 128 : NB;
  int64_t n1 = (n / 2) / gran * gran;
  if (n1 <= 0) n1 = gran;
  if (n1 >= n) n1 = n - NB;
  return (int)n1;
}

constexpr int BINV = 512;   // potrf-only mode: diagonal subtrees up to this size keep their inverse

template <typename T>
struct Rec {
  Ctx* c;
  bool full_inverse;
  T* leafinv;   // compact leaf inverses (potrf-only mode), leaf k at leafinv + k*NB*NB, ld NB
  double* logdet_slots;
  int* fail_col;
  T* tmp;       // full-inverse recursion temporaries
  size_t tmp_elems;
  T* xdiag;     // potrf-only: inverse of the diagonal block at col0 stored at xdiag + col0 (ld ldxd)
  int64_t ldxd;
  T* tmp2;      // potrf-only: out-of-place product buffer for B := B Xblock^T
  size_t tmp2_elems;
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
  T* xp;
  int64_t ldx;
  if (R.full_inverse) {
    xp = X.p;
    ldx = X.ld;
  } else {
    xp = R.leafinv + (col0 / NB) * NB * NB;
    ldx = NB;
  }
  static bool attr = false;
  if (!attr) {
    CGGM_CUDA_CHECK(cudaFuncSetAttribute(leaf_potrf_trtri<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, leaf_smem_bytes<T>()));
    attr = true;
  }
  Prof pr(R.c, TAG_CHOL_LEAF);
  leaf_potrf_trtri<T><<<1, LEAF_THREADS, leaf_smem_bytes<T>(), R.c->stream>>>(A.p, A.ld, nb, xp, ldx, R.full_inverse ? 0 : 1,
                                                        R.logdet_slots + col0 / NB, R.fail_col, (int)col0);
  post_launch(R.c, "leaf_potrf_trtri");
}

// A is (n + extra) x n: the square block being factored with `extra` appended rows below it
// (potrf-only mode).  Factoring the augmented [Lambda; W] leaves Z = W L^{-T} in the bottom rows
// (block Cholesky of [[Lambda, W^T], [W, .]]), so the objective's triangular solve is carried by
// the same recursive GEMMs with taller panels.
template <typename T>
void node(Rec<T>& R, ViewT<T> A, ViewT<T> X, int64_t col0) {
  const int64_t n = A.cols, extra = A.rows - A.cols;
  Ctx* c = R.c;
  if (!R.full_inverse && R.xdiag && n <= BINV) {
    // potrf-only: factor this diagonal subtree in full-inverse mode, keeping its inverse for the
    // triangular solves of the panels to its right and of the appended rows below
    Rec<T> R2 = R;
    R2.full_inverse = true;
    ViewT<T> Xb{R.xdiag + col0, R.ldxd, n, n};
    node(R2, A.sub(0, 0, n, n), Xb, col0);
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
    node(R, A11, X11, col0);
    ViewT<T> Tm{R.tmp, n2 + (n2 & 1), n2, n1};
    if ((size_t)(Tm.ld * n1) > R.tmp_elems) throw CudaError{CGGM_ERR_OOM, "recursion temp too small"};
    {  // T = A21 X11^T  (L21)
      EpilogueT<T> e; e.out1 = Tm.p; e.ld1 = Tm.ld;
      gemm(c, false, true, n2, n1, n1, A21.p, A21.ld, X11.p, X11.ld, e, B_KLE_N);
    }
    {  // A22 -= T T^T (lower)
      EpilogueT<T> e; e.out1 = A22.p; e.ld1 = A22.ld; e.a1 = -1.0; e.in1a = A22.p; e.ld1a = A22.ld; e.b1 = 1.0;
      gemm(c, false, true, n2, n2, n1, Tm.p, Tm.ld, Tm.p, Tm.ld, e, SYM_LOWER);
    }
    {  // A21 := T X11
      EpilogueT<T> e; e.out1 = A21.p; e.ld1 = A21.ld;
      gemm(c, false, false, n2, n1, n1, Tm.p, Tm.ld, X11.p, X11.ld, e, B_KGE_N);
    }
    node(R, A22, X22, col0 + n1);
    {  // X21 = -X22 A21
      EpilogueT<T> e; e.out1 = X21.p; e.ld1 = X21.ld; e.a1 = -1.0;
      gemm(c, false, false, n2, n1, n2, X22.p, X22.ld, A21.p, A21.ld, e, A_KLE_M);
    }
  } else {
    node(R, A11, X, col0);
    trsm_rec(R, A21, A11, col0);
    {  // A22 -= A21 A21^T over the lower trapezoid (square part + appended rows)
      EpilogueT<T> e; e.out1 = A22.p; e.ld1 = A22.ld; e.a1 = -1.0; e.in1a = A22.p; e.ld1a = A22.ld; e.b1 = 1.0;
      gemm(c, false, true, n2 + extra, n2, n1, A21.p, A21.ld, A21.p, A21.ld, e, SYM_LOWER);
    }
    node(R, A22, X, col0 + n1);
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
                     size_t tmp2_elems) {
  Rec<T> R{c, full_inverse, leafinv, logdet_slots, fail_col_dev, tmp, tmp_elems, xdiag, ldxd, tmp2, tmp2_elems};
  Phase ph(c, TAG_CHOL_GEMM);
  node(R, A, Linv, 0);
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
                                      size_t, double*, int64_t, double*, size_t);
template void potrf_recursive<float>(Ctx*, ViewT<float>, ViewT<float>, bool, float*, double*, int*, float*, size_t,
                                     float*, int64_t, float*, size_t);
template void lauum<double>(Ctx*, ViewT<double>, ViewT<double>);
template void lauum<float>(Ctx*, ViewT<float>, ViewT<float>);

}  // namespace cggm
