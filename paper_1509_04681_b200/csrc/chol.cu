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

constexpr int NB = 64;
constexpr int LEAF_THREADS = 256;
constexpr int LEAF_SMEM = 2 * NB * (NB + 1) * 8;

__global__ void __launch_bounds__(LEAF_THREADS) leaf_potrf_trtri(double* A, int64_t lda, int nb, double* X,
                                                                  int64_t ldx, int write_L, double* logdet_slot,
                                                                  int* fail_col, int col0) {
  extern __shared__ double leaf_smem[];
  double(*S)[NB + 1] = reinterpret_cast<double(*)[NB + 1]>(leaf_smem);             // S[col][row] -> L
  double(*Xs)[NB + 1] = reinterpret_cast<double(*)[NB + 1]>(leaf_smem + NB * (NB + 1));  // Xs[col][row] -> L^{-1}
  __shared__ int failed;
  const int tid = threadIdx.x;
  for (int idx = tid; idx < NB * NB; idx += LEAF_THREADS) {
    const int i = idx % NB, j = idx / NB;
    S[j][i] = (i < nb && j < nb && i >= j) ? A[i + (int64_t)j * lda] : 0.0;
    Xs[j][i] = (i == j) ? 1.0 : 0.0;
  }
  if (tid == 0) failed = -1;
  __syncthreads();
  // unblocked right-looking Cholesky (column j: pivot, scale, rank-1 trailing update)
  for (int j = 0; j < nb; ++j) {
    const double d = S[j][j];
    const bool bad = !(d > 0.0) || !isfinite(d);
    const double ljj = sqrt(d);
    const double inv = 1.0 / ljj;
    __syncthreads();
    if (tid == 0) {
      if (bad && failed < 0) failed = j;
      S[j][j] = ljj;
    }
    for (int i = j + 1 + tid; i < nb; i += LEAF_THREADS) S[j][i] *= inv;
    __syncthreads();
    const int rem = nb - j - 1;
    for (int idx = tid; idx < rem * rem; idx += LEAF_THREADS) {
      const int ii = idx % rem, kk = idx / rem;
      if (ii >= kk) S[j + 1 + kk][j + 1 + ii] -= S[j][j + 1 + ii] * S[j][j + 1 + kk];
    }
    __syncthreads();
  }
  // triangular inverse: forward substitution L X = I, column of L by column of L
  for (int j = 0; j < nb; ++j) {
    const double ljj = S[j][j];
    for (int c = tid; c <= j; c += LEAF_THREADS) Xs[c][j] /= ljj;
    __syncthreads();
    const int rem = nb - j - 1;
    for (int idx = tid; idx < rem * (j + 1); idx += LEAF_THREADS) {
      const int ii = idx % rem, c = idx / rem;
      Xs[c][j + 1 + ii] -= S[j][j + 1 + ii] * Xs[c][j];
    }
    __syncthreads();
  }
  for (int idx = tid; idx < nb * nb; idx += LEAF_THREADS) {
    const int i = idx % nb, j = idx / nb;
    if (write_L) A[i + (int64_t)j * lda] = (i >= j) ? S[j][i] : 0.0;
    X[i + (int64_t)j * ldx] = (i >= j) ? Xs[j][i] : 0.0;
  }
  if (tid == 0) {
    double s = 0.0;
    for (int j = 0; j < nb; ++j) s += log(S[j][j]);
    *logdet_slot = 2.0 * s;
    if (failed >= 0) atomicMin(fail_col, col0 + failed);
  }
}

int split_point(int64_t n) {
  const int64_t gran = n > 4 * 128 ? 128 : NB;
  int64_t n1 = (n / 2) / gran * gran;
  if (n1 <= 0) n1 = gran;
  if (n1 >= n) n1 = n - NB;
  return (int)n1;
}

struct Rec {
  Ctx* c;
  bool full_inverse;
  double* leafinv;   // compact leaf inverses (potrf-only mode), leaf k at leafinv + k*NB*NB, ld NB
  double* logdet_slots;
  int* fail_col;
  double* tmp;
  size_t tmp_elems;
};

void leaf(Rec& R, View A, View X, int64_t col0) {
  const int nb = (int)A.rows;
  double* xp;
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
    CGGM_CUDA_CHECK(cudaFuncSetAttribute(leaf_potrf_trtri, cudaFuncAttributeMaxDynamicSharedMemorySize, LEAF_SMEM));
    attr = true;
  }
  Prof pr(R.c, TAG_CHOL_LEAF);
  leaf_potrf_trtri<<<1, LEAF_THREADS, LEAF_SMEM, R.c->stream>>>(A.p, A.ld, nb, xp, ldx, R.full_inverse ? 0 : 1,
                                                        R.logdet_slots + col0 / NB, R.fail_col, (int)col0);
  post_launch(R.c, "leaf_potrf_trtri");
}

void node(Rec& R, View A, View X, int64_t col0) {
  const int64_t n = A.rows;
  if (n <= NB) {
    leaf(R, A, X, col0);
    return;
  }
  const int64_t n1 = split_point(n), n2 = n - n1;
  View A11 = A.sub(0, 0, n1, n1), A21 = A.sub(n1, 0, n2, n1), A22 = A.sub(n1, n1, n2, n2);
  Ctx* c = R.c;
  if (R.full_inverse) {
    View X11 = X.sub(0, 0, n1, n1), X21 = X.sub(n1, 0, n2, n1), X22 = X.sub(n1, n1, n2, n2);
    node(R, A11, X11, col0);
    View T{R.tmp, n2 + (n2 & 1), n2, n1};
    if ((size_t)(T.ld * n1) > R.tmp_elems) throw CudaError{CGGM_ERR_OOM, "recursion temp too small"};
    {  // T = A21 X11^T  (L21)
      Epilogue e; e.out1 = T.p; e.ld1 = T.ld;
      gemm(c, false, true, n2, n1, n1, A21.p, A21.ld, X11.p, X11.ld, e, B_KLE_N);
    }
    {  // A22 -= T T^T (lower)
      Epilogue e; e.out1 = A22.p; e.ld1 = A22.ld; e.a1 = -1.0; e.in1a = A22.p; e.ld1a = A22.ld; e.b1 = 1.0;
      gemm(c, false, true, n2, n2, n1, T.p, T.ld, T.p, T.ld, e, SYM_LOWER);
    }
    {  // A21 := T X11
      Epilogue e; e.out1 = A21.p; e.ld1 = A21.ld;
      gemm(c, false, false, n2, n1, n1, T.p, T.ld, X11.p, X11.ld, e, B_KGE_N);
    }
    node(R, A22, X22, col0 + n1);
    {  // X21 = -X22 A21
      Epilogue e; e.out1 = X21.p; e.ld1 = X21.ld; e.a1 = -1.0;
      gemm(c, false, false, n2, n1, n2, X22.p, X22.ld, A21.p, A21.ld, e, A_KLE_M);
    }
  } else {
    node(R, A11, X, col0);
    trsm_right_lt(c, A21, A11, R.leafinv, col0);
    {
      Epilogue e; e.out1 = A22.p; e.ld1 = A22.ld; e.a1 = -1.0; e.in1a = A22.p; e.ld1a = A22.ld; e.b1 = 1.0;
      gemm(c, false, true, n2, n2, n1, A21.p, A21.ld, A21.p, A21.ld, e, SYM_LOWER);
    }
    node(R, A22, X, col0 + n1);
  }
}

}  // namespace

int leaf_nb() { return NB; }

void potrf_recursive(Ctx* c, View A, View Linv, bool full_inverse, double* leafinv, double* logdet_slots,
                     int* fail_col_dev, double* tmp, size_t tmp_elems) {
  Rec R{c, full_inverse, leafinv, logdet_slots, fail_col_dev, tmp, tmp_elems};
  Phase ph(c, TAG_CHOL_GEMM);
  node(R, A, Linv, 0);
}

void trsm_right_lt(Ctx* c, View B, View L, const double* leafinv, int64_t col0) {
  const int64_t n = L.rows;
  if (B.rows == 0) return;
  if (n <= NB) {
    // B := B Xleaf^T; N = n <= 64 fits one tile column, so each CTA reads only the rows it writes
    const double* xl = leafinv + (col0 / NB) * NB * NB;
    Epilogue e; e.out1 = B.p; e.ld1 = B.ld;
    gemm(c, false, true, B.rows, n, n, B.p, B.ld, xl, NB, e, B_KLE_N);
    return;
  }
  const int64_t n1 = split_point(n), n2 = n - n1;
  View B1 = B.sub(0, 0, B.rows, n1), B2 = B.sub(0, n1, B.rows, n2);
  trsm_right_lt(c, B1, L.sub(0, 0, n1, n1), leafinv, col0);
  {  // B2 -= B1 L21^T
    View L21 = L.sub(n1, 0, n2, n1);
    Epilogue e; e.out1 = B2.p; e.ld1 = B2.ld; e.a1 = -1.0; e.in1a = B2.p; e.ld1a = B2.ld; e.b1 = 1.0;
    gemm(c, false, true, B.rows, n2, n1, B1.p, B1.ld, L21.p, L21.ld, e, 0);
  }
  trsm_right_lt(c, B2, L.sub(n1, n1, n2, n2), leafinv, col0 + n1);
}

void lauum(Ctx* c, View Linv, View Sigma) {
  const int64_t q = Linv.rows;
  Phase ph(c, TAG_LAUUM);
  Epilogue e; e.out1 = Sigma.p; e.ld1 = Sigma.ld;
  gemm(c, true, false, q, q, q, Linv.p, Linv.ld, Linv.p, Linv.ld, e, A_KGE_M | B_KGE_N | SYM_LOWER | SYM_MIRROR);
}

}  // namespace cggm
