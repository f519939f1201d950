// HBM-bound kernels of the hot path: CSC densify (K00), SpMM W = X Theta (K05),
// CSC structure / symmetry checks, the elementwise grad_Lambda = S_yy - Sigma - Psi (Eq. 3),
// and the deterministic per-column partial sums used by the objective (K08, Eq. 1).
// All reductions are two-level with a fixed order (per-column partials, then one CTA), so
// every scalar is bitwise reproducible run to run.
#include "common.cuh"
#include "kernels.cuh"

namespace cggm {

// ------------------------------------------------------------------ densify CSC -> dense
template <typename T>
__global__ void k_scatter_csc(const int64_t* colptr, const int32_t* rowidx, const T* val, int64_t ncols, T* D,
                              int64_t ldd) {
  const int64_t j = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x / 32);
  if (j >= ncols) return;
  const int lane = threadIdx.x & 31;
  for (int64_t t = colptr[j] + lane; t < colptr[j + 1]; t += 32) D[rowidx[t] + j * ldd] = val[t];
}

template <typename T>
void densify_csc(Ctx* c, const cggm_csc* A, ViewT<T> D) {
  CGGM_CUDA_CHECK(cudaMemset2DAsync(D.p, D.ld * sizeof(T), 0, D.rows * sizeof(T), D.cols, c->stream));
  if (A->ncols == 0 || A->nnz == 0) return;
  const int wpb = 8;
  const int64_t grid = (A->ncols + wpb - 1) / wpb;
  Prof pr(c, TAG_DENSIFY);
  k_scatter_csc<T><<<(unsigned)grid, wpb * 32, 0, c->stream>>>(A->colptr, A->rowidx, static_cast<const T*>(A->val),
                                                               A->ncols, D.p, D.ld);
  post_launch(c, "k_scatter_csc");
}

// ------------------------------------------------------------------ W = X Theta
// W[k, j] = sum_t Theta_{row_t j} X[k, row_t] (ascending t).  Grid (column j, 128-row block of the
// samples), row-block-major dispatch order: all columns of one row block run together, so that
// block's slice of X (128 x p doubles, 41 MB at p = 40000) stays resident in the 126 MB L2 and X
// is read from HBM about once.
constexpr int SPMM_ROWS = 128;
template <typename T>
__global__ void __launch_bounds__(SPMM_ROWS) k_spmm_x_theta(const T* __restrict__ X, int64_t ldx, int64_t n,
                                                            const int64_t* __restrict__ colptr,
                                                            const int32_t* __restrict__ rowidx,
                                                            const T* __restrict__ val, T* __restrict__ W,
                                                            int64_t ldw) {
  __shared__ int32_t rows[SPMM_ROWS];
  __shared__ T vals[SPMM_ROWS];
  const int64_t j = blockIdx.x;
  const int64_t k = (int64_t)blockIdx.y * SPMM_ROWS + threadIdx.x;
  const int64_t a = colptr[j], b = colptr[j + 1];
  T acc = T(0);
  for (int64_t t0 = a; t0 < b; t0 += SPMM_ROWS) {
    const int cnt = (int)((b - t0) < SPMM_ROWS ? (b - t0) : SPMM_ROWS);
    __syncthreads();
    if (threadIdx.x < cnt) {
      rows[threadIdx.x] = rowidx[t0 + threadIdx.x];
      vals[threadIdx.x] = val[t0 + threadIdx.x];
    }
    __syncthreads();
    if (k < n) {
      int e = 0;
      for (; e + 8 <= cnt; e += 8) {  // 8 independent gathers in flight
        T xv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) xv[u] = __ldg(X + k + (int64_t)rows[e + u] * ldx);
#pragma unroll
        for (int u = 0; u < 8; ++u) acc = fma(vals[e + u], xv[u], acc);
      }
      for (; e < cnt; ++e) acc = fma(vals[e], __ldg(X + k + (int64_t)rows[e] * ldx), acc);
    }
  }
  if (k < n) W[k + j * ldw] = acc;
}

template <typename T>
struct SpPair;
template <>
struct SpPair<double> {
  using V = double2;
};
template <>
struct SpPair<float> {
  using V = float2;
};

// Paired variant (16-byte aligned X and W, even leading dimensions): each thread owns two adjacent
// rows, so one 16-byte gather serves both and the per-gather address / issue work halves (the
// kernel is bound by L2 gather throughput and SM issue, not by HBM: X is read from HBM about once)
template <typename T>
__global__ void __launch_bounds__(SPMM_ROWS / 2) k_spmm_x_theta2(const T* __restrict__ X, int64_t ldx, int64_t n,
                                                                const int64_t* __restrict__ colptr,
                                                                const int32_t* __restrict__ rowidx,
                                                                const T* __restrict__ val, T* __restrict__ W,
                                                                int64_t ldw) {
  using V = typename SpPair<T>::V;
  constexpr int NT = SPMM_ROWS / 2;
  __shared__ int64_t offs[SPMM_ROWS];
  __shared__ T vals[SPMM_ROWS];
  const int64_t j = blockIdx.x;
  const int64_t k = (int64_t)blockIdx.y * SPMM_ROWS + 2 * threadIdx.x;
  const int64_t a = colptr[j], b = colptr[j + 1];
  T acc0 = T(0), acc1 = T(0);
  const bool full = k + 1 < n;
  for (int64_t t0 = a; t0 < b; t0 += SPMM_ROWS) {
    const int cnt = (int)((b - t0) < SPMM_ROWS ? (b - t0) : SPMM_ROWS);
    __syncthreads();
    for (int e = threadIdx.x; e < cnt; e += NT) {
      CGGM_DASSERT(rowidx[t0 + e] >= 0);
      offs[e] = (int64_t)rowidx[t0 + e] * ldx;
      vals[e] = val[t0 + e];
    }
    __syncthreads();
    if (full) {
      int e = 0;
      for (; e + 8 <= cnt; e += 8) {  // 8 independent 16-byte gathers in flight
        V xv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) xv[u] = __ldg(reinterpret_cast<const V*>(X + k + offs[e + u]));
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          acc0 = fma(vals[e + u], xv[u].x, acc0);
          acc1 = fma(vals[e + u], xv[u].y, acc1);
        }
      }
      for (; e < cnt; ++e) {
        const V xv = __ldg(reinterpret_cast<const V*>(X + k + offs[e]));
        acc0 = fma(vals[e], xv.x, acc0);
        acc1 = fma(vals[e], xv.y, acc1);
      }
    } else if (k < n) {
      for (int e = 0; e < cnt; ++e) acc0 = fma(vals[e], __ldg(X + k + offs[e]), acc0);
    }
  }
  if (full) {
    *reinterpret_cast<V*>(W + k + j * ldw) = V{acc0, acc1};
  } else if (k < n) {
    W[k + j * ldw] = acc0;
  }
}

template <typename T>
void spmm_x_theta(Ctx* c, const T* X, int64_t ldx, int64_t n, const cggm_csc* Theta, ViewT<T> W) {
  if (Theta->ncols == 0 || n == 0) return;
  Prof pr(c, TAG_SPMM);
  dim3 grid((unsigned)Theta->ncols, (unsigned)((n + SPMM_ROWS - 1) / SPMM_ROWS));
  const bool paired = reinterpret_cast<uintptr_t>(X) % (2 * sizeof(T)) == 0 && ldx % 2 == 0 &&
                      reinterpret_cast<uintptr_t>(W.p) % (2 * sizeof(T)) == 0 && W.ld % 2 == 0;
  if (paired) {
    k_spmm_x_theta2<T><<<grid, SPMM_ROWS / 2, 0, c->stream>>>(X, ldx, n, Theta->colptr, Theta->rowidx,
                                                              static_cast<const T*>(Theta->val), W.p, W.ld);
    post_launch(c, "k_spmm_x_theta2");
    return;
  }
  k_spmm_x_theta<T><<<grid, SPMM_ROWS, 0, c->stream>>>(X, ldx, n, Theta->colptr, Theta->rowidx,
                                                      static_cast<const T*>(Theta->val), W.p, W.ld);
  post_launch(c, "k_spmm_x_theta");
}

// R = s * Acc, E = Y + Acc (the split-k W Sigma: Acc holds the sum of the two k-halves)
template <typename T>
__global__ void k_r_e_from_acc(int64_t n, int64_t q, const T* __restrict__ acc, int64_t lda,
                               const T* __restrict__ Y, int64_t ldy, T* __restrict__ R, int64_t ldr,
                               T* __restrict__ E, int64_t lde, double s) {
  const int64_t j = blockIdx.y;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const T a = acc[i + j * lda];
    R[i + j * ldr] = (T)((double)a * s);
    if (E) E[i + j * lde] = Y[i + j * ldy] + a;
  }
}

template <typename T>
void r_e_from_acc(Ctx* c, int64_t n, int64_t q, const T* acc, int64_t lda, const T* Y, int64_t ldy, T* R, int64_t ldr,
                  T* E, int64_t lde, double s) {
  if (n == 0 || q == 0) return;
  Prof pr(c, TAG_WSIGMA);
  dim3 grid((unsigned)((n + 255) / 256 < 8 ? (n + 255) / 256 : 8), (unsigned)q);
  k_r_e_from_acc<T><<<grid, 256, 0, c->stream>>>(n, q, acc, lda, Y, ldy, R, ldr, E, lde, s);
  post_launch(c, "k_r_e_from_acc");
}
template void r_e_from_acc<double>(Ctx*, int64_t, int64_t, const double*, int64_t, const double*, int64_t, double*,
                                   int64_t, double*, int64_t, double);
template void r_e_from_acc<float>(Ctx*, int64_t, int64_t, const float*, int64_t, const float*, int64_t, float*,
                                  int64_t, float*, int64_t, double);

// S[j][i] = S[i][j] for i > j: 32 x 32 tiles of the lower triangle through shared memory, so both
// the read of the lower tile and the write of its transpose are coalesced
template <typename T>
__global__ void k_symmetrize(int64_t n, T* S, int64_t ld) {
  __shared__ T tile[32][33];
  const int64_t bi = blockIdx.x, bj = blockIdx.y;   // source tile: rows 32 bi.., cols 32 bj..
  if (bi < bj) return;
  const int tx = threadIdx.x, ty = threadIdx.y;      // 32 x 8 threads
  for (int r = ty; r < 32; r += 8) {
    const int64_t i = bi * 32 + tx, j = bj * 32 + r;
    tile[r][tx] = (i < n && j < n) ? S[i + j * ld] : T(0);
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const int64_t i = bj * 32 + tx, j = bi * 32 + r;   // destination (row i, col j) = source (j, i)
    if (i < n && j < n && j > i) S[i + j * ld] = tile[tx][r];
  }
}

template <typename T>
void symmetrize(Ctx* c, int64_t n, T* S, int64_t ld) {
  if (n <= 1) return;
  const unsigned nt = (unsigned)((n + 31) / 32);
  Prof pr(c, TAG_MISC);
  k_symmetrize<T><<<dim3(nt, nt), dim3(32, 8), 0, c->stream>>>(n, S, ld);
  post_launch(c, "k_symmetrize");
}
template void symmetrize<double>(Ctx*, int64_t, double*, int64_t);
template void symmetrize<float>(Ctx*, int64_t, float*, int64_t);

// slice [lo, hi) of the sum over `world` peer buffers, in rank order, written back to every buffer
constexpr int PEER_MAX = 8;
struct PeerPtrs {
  void* p[PEER_MAX];
};
template <typename T>
__global__ void k_peer_allreduce(PeerPtrs bufs, int world, int64_t lo, int64_t hi) {
  for (int64_t i = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < hi; i += (int64_t)gridDim.x * blockDim.x) {
    T s = static_cast<const T*>(bufs.p[0])[i];
    for (int k = 1; k < world; ++k) s += static_cast<const T*>(bufs.p[k])[i];
    for (int k = 0; k < world; ++k) static_cast<T*>(bufs.p[k])[i] = s;
  }
}

template <typename T>
void peer_allreduce(Ctx* c, int world, int rank, void* const* bufs, int64_t count) {
  if (world < 1 || world > PEER_MAX) throw CudaError{CGGM_ERR_INVALID_ARG, "peer all-reduce: 1..8 ranks"};
  const int64_t per = (count + world - 1) / world;
  const int64_t lo = std::min<int64_t>(count, (int64_t)rank * per), hi = std::min<int64_t>(count, lo + per);
  if (hi <= lo) return;
  PeerPtrs P{};
  for (int k = 0; k < world; ++k) P.p[k] = bufs[k];
  Prof pr(c, TAG_MISC);
  k_peer_allreduce<T><<<(unsigned)(2 * c->num_sms), 256, 0, c->stream>>>(P, world, lo, hi);
  post_launch(c, "k_peer_allreduce");
}
template void peer_allreduce<double>(Ctx*, int, int, void* const*, int64_t);
template void peer_allreduce<float>(Ctx*, int, int, void* const*, int64_t);

// ------------------------------------------------------------------ CSC checks
// flag bits: 1 = colptr not monotone / bad ends, 2 = row out of range or not strictly increasing,
//            4 = not symmetric (symmetric mode)
template <typename T>
__global__ void k_check_csc(const int64_t* colptr, const int32_t* rowidx, const T* val, int64_t nrows,
                            int64_t ncols, int64_t nnz, int symmetric, int* flag) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j == 0 && (colptr[0] != 0 || colptr[ncols] != nnz)) atomicOr(flag, 1);
  if (j >= ncols) return;
  const int64_t a = colptr[j], b = colptr[j + 1];
  if (a > b || a < 0 || b > nnz) {
    atomicOr(flag, 1);
    return;
  }
  int32_t prev = -1;
  for (int64_t t = a; t < b; ++t) {
    const int32_t r = rowidx[t];
    if (r <= prev || r < 0 || r >= nrows) {
      atomicOr(flag, 2);
      return;
    }
    prev = r;
    if (symmetric) {
      // find (j, r): row j in column r, by binary search
      int64_t lo = colptr[r], hi = colptr[r + 1] - 1;
      bool found = false;
      while (lo <= hi) {
        const int64_t mid = (lo + hi) >> 1;
        const int32_t rm = rowidx[mid];
        if (rm == j) {
          found = (val[mid] == val[t]);
          break;
        }
        if (rm < j) lo = mid + 1;
        else hi = mid - 1;
      }
      if (!found) atomicOr(flag, 4);
    }
  }
}

template <typename T>
void check_csc(Ctx* c, const cggm_csc* A, bool symmetric, int* flag_dev) {
  if (A->ncols == 0) return;
  const int64_t grid = (A->ncols + 255) / 256;
  Prof pr(c, c->cur_tag);
  k_check_csc<T><<<(unsigned)grid, 256, 0, c->stream>>>(A->colptr, A->rowidx, static_cast<const T*>(A->val),
                                                     A->nrows, A->ncols, A->nnz, symmetric ? 1 : 0, flag_dev);
  post_launch(c, "k_check_csc");
}

// ------------------------------------------------------------------ grad_Lambda elementwise
__device__ __forceinline__ double sub_rn(double a, double b) { return __dadd_rn(a, -b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fadd_rn(a, -b); }

template <typename T>
__global__ void __launch_bounds__(256) k_grad_lambda(int64_t q, const T* __restrict__ Syy, int64_t l1,
                                                     const T* __restrict__ Sg, int64_t l2, const T* __restrict__ Psi,
                                                     int64_t l3, T* __restrict__ G, int64_t l4) {
  const int64_t j = blockIdx.x;
  const T* a = Syy + j * l1;
  const T* b = Sg + j * l2;
  const T* c = Psi + j * l3;
  T* g = G + j * l4;
  for (int64_t i = threadIdx.x; i < q; i += 256) g[i] = sub_rn(sub_rn(a[i], b[i]), c[i]);
}

template <typename T>
void grad_lambda(Ctx* c, int64_t q, const T* Syy, int64_t l1, const T* Sigma, int64_t l2, const T* Psi, int64_t l3,
                 T* G, int64_t l4) {
  if (q == 0) return;
  Prof pr(c, c->cur_tag);
  k_grad_lambda<T><<<(unsigned)q, 256, 0, c->stream>>>(q, Syy, l1, Sigma, l2, Psi, l3, G, l4);
  post_launch(c, "k_grad_lambda");
}

template <typename T>
void copy2d(Ctx* c, ViewT<T> dst, const T* src, int64_t lds) {
  if (dst.rows == 0 || dst.cols == 0) return;
  CGGM_CUDA_CHECK(cudaMemcpy2DAsync(dst.p, dst.ld * sizeof(T), src, lds * sizeof(T), dst.rows * sizeof(T), dst.cols,
                                    cudaMemcpyDeviceToDevice, c->stream));
}

// ------------------------------------------------------------------ deterministic block reduce
template <int NT>
__device__ __forceinline__ double block_sum(double v, double* sh) {
  sh[threadIdx.x] = v;
  __syncthreads();
#pragma unroll
  for (int s = NT / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] = sh[threadIdx.x] + sh[threadIdx.x + s];
    __syncthreads();
  }
  const double r = sh[0];
  __syncthreads();
  return r;
}

// ------------------------------------------------------------------ objective column partials
// mode 0: part[j] = sum_k Y[k,j] * (Y Lambda)[k,j]   (<Y, Y Lambda>, tr(S_yy Lambda) * n)
// mode 1: part[j] = sum_k A[k,j] * B[k,j]           (<W, Y>)
// mode 2: part[j] = sum_k A[k,j]^2                  (||Z||_F^2)
template <typename T>
__global__ void __launch_bounds__(256) k_col_partials(int mode, int64_t n, const T* __restrict__ A, int64_t lda,
                                                      const T* __restrict__ B, int64_t ldb,
                                                      const int64_t* __restrict__ colptr,
                                                      const int32_t* __restrict__ rowidx, const T* __restrict__ val,
                                                      double* part) {
  __shared__ double sh[256];
  const int64_t j = blockIdx.x;
  T s = T(0);
  if (mode == 0) {
    const int64_t a = colptr[j], b = colptr[j + 1];
    for (int64_t k = threadIdx.x; k < n; k += 256) {
      T yl = T(0);
      for (int64_t t = a; t < b; ++t) yl = fma(__ldg(A + k + (int64_t)rowidx[t] * lda), val[t], yl);
      s = fma(__ldg(A + k + j * lda), yl, s);
    }
  } else if (mode == 1) {
    for (int64_t k = threadIdx.x; k < n; k += 256) s = fma(A[k + j * lda], B[k + j * ldb], s);
  } else {
    for (int64_t k = threadIdx.x; k < n; k += 256) {
      const T v = A[k + j * lda];
      s = fma(v, v, s);
    }
  }
  const double r = block_sum<256>((double)s, sh);
  if (threadIdx.x == 0) part[j] = r;
}

// per-column sum |val| of a CSC (diagonal skipped when skip_diag)
template <typename T>
__global__ void k_csc_abs_partials(const int64_t* colptr, const int32_t* rowidx, const T* val, int64_t ncols,
                                   int skip_diag, double* part) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= ncols) return;
  double s = 0.0;
  for (int64_t t = colptr[j]; t < colptr[j + 1]; ++t) {
    if (skip_diag && rowidx[t] == j) continue;
    s += fabs((double)val[t]);
  }
  part[j] = s;
}

// out[r] = sum_{i < len_r} arr_r[i], fixed order (one CTA per array)
__global__ void __launch_bounds__(256) k_sum_arrays(const double* const* arrs, const int64_t* lens, double* out) {
  __shared__ double sh[256];
  const double* a = arrs[blockIdx.x];
  const int64_t len = lens[blockIdx.x];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < len; i += 256) s += a[i];
  s = block_sum<256>(s, sh);
  if (threadIdx.x == 0) out[blockIdx.x] = s;
}

template <typename T>
void col_partials(Ctx* c, int mode, int64_t n, int64_t ncols, const T* A, int64_t lda, const T* B, int64_t ldb,
                  const cggm_csc* csc, double* part) {
  if (ncols == 0) return;
  Prof pr(c, c->cur_tag);
  k_col_partials<T><<<(unsigned)ncols, 256, 0, c->stream>>>(mode, n, A, lda, B, ldb, csc ? csc->colptr : nullptr,
                                                            csc ? csc->rowidx : nullptr,
                                                            csc ? static_cast<const T*>(csc->val) : nullptr, part);
  post_launch(c, "k_col_partials");
}

template <typename T>
void csc_abs_partials(Ctx* c, const cggm_csc* A, bool skip_diag, double* part) {
  if (A->ncols == 0) return;
  Prof pr(c, c->cur_tag);
  k_csc_abs_partials<T><<<(unsigned)((A->ncols + 255) / 256), 256, 0, c->stream>>>(
      A->colptr, A->rowidx, static_cast<const T*>(A->val), A->ncols, skip_diag ? 1 : 0, part);
  post_launch(c, "k_csc_abs_partials");
}

void sum_arrays(Ctx* c, int count, const double* const* arrs_dev, const int64_t* lens_dev, double* out_dev) {
  Prof pr(c, c->cur_tag);
  k_sum_arrays<<<count, 256, 0, c->stream>>>(arrs_dev, lens_dev, out_dev);
  post_launch(c, "k_sum_arrays");
}

// out = sum_{i < len} a[i], fixed order (one CTA)
__global__ void __launch_bounds__(256) k_sum_vec(const double* a, int64_t len, double* out) {
  __shared__ double sh[256];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < len; i += 256) s += a[i];
  s = block_sum<256>(s, sh);
  if (threadIdx.x == 0) *out = s;
}

__global__ void k_stamp(unsigned long long* p) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  *p = t;
}

void prof_stamp(Ctx* c, int idx) {
  k_stamp<<<1, 1, 0, c->stream>>>(c->ts_buf + idx);
}

void sum_arrays_1(Ctx* c, const double* a, int64_t len, double* out_dev) {
  Prof pr(c, c->cur_tag);
  k_sum_vec<<<1, 256, 0, c->stream>>>(a, len, out_dev);
  post_launch(c, "k_sum_vec");
}

__global__ void k_init_scalars(int* fail_col, int* flag) {
  *fail_col = INT_MAX;
  *flag = 0;
}

void init_scalars(Ctx* c, int* fail_col, int* flag) {
  Prof pr(c, c->cur_tag);
  k_init_scalars<<<1, 1, 0, c->stream>>>(fail_col, flag);
  post_launch(c, "k_init_scalars");
}

#define CGGM_INST(T)                                                                                      \
  template void densify_csc<T>(Ctx*, const cggm_csc*, ViewT<T>);                                         \
  template void spmm_x_theta<T>(Ctx*, const T*, int64_t, int64_t, const cggm_csc*, ViewT<T>);             \
  template void check_csc<T>(Ctx*, const cggm_csc*, bool, int*);                                         \
  template void grad_lambda<T>(Ctx*, int64_t, const T*, int64_t, const T*, int64_t, const T*, int64_t, T*, \
                               int64_t);                                                                 \
  template void copy2d<T>(Ctx*, ViewT<T>, const T*, int64_t);                                            \
  template void col_partials<T>(Ctx*, int, int64_t, int64_t, const T*, int64_t, const T*, int64_t,        \
                                const cggm_csc*, double*);                                               \
  template void csc_abs_partials<T>(Ctx*, const cggm_csc*, bool, double*);
CGGM_INST(double)
CGGM_INST(float)
#undef CGGM_INST

}  // namespace cggm
