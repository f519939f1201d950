// Coordinate-descent consumers of the hot path: the Lambda
// Newton-direction sweep of Eq. (6) with U = D Sigma, the direct Theta sweep of
// Eq. (7) with V = Theta Sigma, and the sparse bookkeeping of Algorithm 1
// (P:407-435): the line-search candidate Lambda + alpha D as a symmetric CSC, the new Theta as
// a CSC.  Coefficients per the appendix with reading A15.
//
// A coordinate sweep is sequential by definition (each update changes U / V, which the next
// update reads), so one CTA of 1024 threads walks the active list in order: per update three
// (Lambda) or one (Theta) length-q / length-p dot products as a block reduction, then the two /
// one row updates of U / V, each thread owning a stride of the vector.  Reduction order is fixed,
// so sweeps are bitwise reproducible.
#include <cooperative_groups.h>

#include "kernels.cuh"

namespace cggm {
namespace {

constexpr int CD_NT = 1024;
constexpr int CD_NW = CD_NT / 32;
constexpr int CD_UNR = 4;   // vector elements per thread whose loads are issued together

__device__ __forceinline__ double soft(double w, double r) {
  const double m = fabs(w) - r;
  return m > 0.0 ? copysign(m, w) : 0.0;
}

// value of A_ij in a CSC with sorted rows (0 if not stored)
__device__ __forceinline__ double csc_at(const int64_t* colptr, const int32_t* rowidx, const double* val, int i,
                                         int j) {
  int64_t lo = colptr[j], hi = colptr[j + 1];
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    const int r = rowidx[mid];
    if (r == i) return val[mid];
    if (r < i) lo = mid + 1;
    else hi = mid;
  }
  return 0.0;
}

// sum over the block of NV values per thread; result valid in every thread
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double (*red)[NV]) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < NV; ++k)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < NV; ++k) red[w][k] = v[k];
  __syncthreads();
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    double s = lane < CD_NW ? red[lane][k] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    v[k] = s;
  }
  __syncthreads();   // red reusable
}

// Per-entry constants of the Lambda sweep (they do not change during it): a, Lambda_ij, GradL_ij and
// the entry's lambda, computed for the whole list in parallel before the sequential walk.
__global__ void k_lambda_coefs(int64_t m, const double* __restrict__ S, int64_t lds, const double* __restrict__ P,
                               int64_t ldp, const double* __restrict__ G, int64_t ldg, const int64_t* colptr,
                               const int32_t* rowidx, const double* lval, const int32_t* Lr, const int32_t* Lc,
                               double lam, int penalize_diag, double4* coef) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < m; k += (int64_t)gridDim.x * blockDim.x) {
    const int i = Lr[k], j = Lc[k];
    const double Sii = S[i + (int64_t)i * lds], Sjj = S[j + (int64_t)j * lds], Sij = S[i + (int64_t)j * lds];
    const double Pii = P[i + (int64_t)i * ldp], Pjj = P[j + (int64_t)j * ldp], Pij = P[i + (int64_t)j * ldp];
    const double a = (i == j) ? Sii * Sii + 2.0 * Sii * Pii
                              : Sij * Sij + Sii * Sjj + Sii * Pjj + Sjj * Pii + 2.0 * Sij * Pij;
    coef[k] = make_double4(a, csc_at(colptr, rowidx, lval, i, j), G[i + (int64_t)j * ldg],
                           (i == j && !penalize_diag) ? 0.0 : lam);
  }
}

// One CTA: D (values on the active list, zeroed here) by `passes` sweeps from D = 0; U (q x q,
// row-major with row stride ldu, zero on entry) = D Sigma throughout.  Per update: the three dot
// products, ONE barrier, every thread sums the 32 warp partials in the same order and forms the
// same mu (no broadcast barrier), the two contiguous row updates, ONE barrier.  The next entry's
// indices and constants are loaded while the current one is processed.  Afterwards out[0] =
// tr(GradL^T D) (both triangles), out[1] = ||Lambda + D||_1 - ||Lambda||_1 weighted by the penalty
// rule, out[2] = ||Lambda||_1 (all entries, from the CSC).
__global__ void __launch_bounds__(CD_NT) k_lambda_cd(int q, const double* __restrict__ S, int64_t lds,
                                                     const double* __restrict__ P, int64_t ldp,
                                                     const double* __restrict__ G, int64_t ldg, const int64_t* colptr,
                                                     const int32_t* rowidx, const double* lval, const int32_t* Lr,
                                                     const int32_t* Lc, const double4* coef, int64_t m,
                                                     int penalize_diag, double lam, int passes, double* D, double* U,
                                                     int64_t ldu, double* out) {
  __shared__ double red[2][CD_NW][3];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t k = threadIdx.x; k < m; k += CD_NT) D[k] = 0.0;   // a fresh direction (U = 0 on entry)
  __syncthreads();
  int par = 0;
  for (int pass = 0; pass < passes; ++pass) {
    int ni = m > 0 ? Lr[0] : 0, nj = m > 0 ? Lc[0] : 0;
    double4 nc = m > 0 ? coef[0] : make_double4(0, 0, 0, 0);
    double nd = m > 0 ? D[0] : 0.0;
    for (int64_t k = 0; k < m; ++k) {
      const int i = ni, j = nj;
      const double4 cf = nc;
      const double dk = nd;
      if (k + 1 < m) {   // prefetch: the list and the constants are not modified by the sweep
        ni = Lr[k + 1];
        nj = Lc[k + 1];
        nc = coef[k + 1];
        nd = D[k + 1];
      }
      const double* Si = S + (int64_t)i * lds;   // row i of Sigma = column i (symmetric)
      const double* Pi = P + (int64_t)i * ldp;
      const double* Pj = P + (int64_t)j * ldp;
      // U is row-major (U[t][c] at t * ldu + c): its columns j, i are strided reads, while the two
      // row updates below -- the larger traffic -- are contiguous
      // all of a thread's loads in flight together (CD_UNR elements per batch), then the FMAs
      double v0 = 0.0, v1 = 0.0, v2 = 0.0;
      for (int t0 = threadIdx.x; t0 < q; t0 += CD_UNR * CD_NT) {
        double uj[CD_UNR], ui[CD_UNR], si[CD_UNR], pi[CD_UNR], pj[CD_UNR];
#pragma unroll
        for (int u = 0; u < CD_UNR; ++u) {
          const int t = t0 + u * CD_NT;
          const bool in = t < q;
          uj[u] = in ? U[(int64_t)t * ldu + j] : 0.0;
          ui[u] = in ? U[(int64_t)t * ldu + i] : 0.0;
          si[u] = in ? Si[t] : 0.0;
          pi[u] = in ? Pi[t] : 0.0;
          pj[u] = in ? Pj[t] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < CD_UNR; ++u) {
          v0 = fma(si[u], uj[u], v0);
          v1 = fma(pi[u], uj[u], v1);
          v2 = fma(pj[u], ui[u], v2);
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        v0 += __shfl_xor_sync(0xffffffffu, v0, o);
        v1 += __shfl_xor_sync(0xffffffffu, v1, o);
        v2 += __shfl_xor_sync(0xffffffffu, v2, o);
      }
      if (lane == 0) {
        red[par][w][0] = v0;
        red[par][w][1] = v1;
        red[par][w][2] = v2;
      }
      __syncthreads();
      // every warp reduces the 32 warp partials by the same shfl_down tree and takes lane 0's value:
      // bitwise the same b in every thread, so every thread forms the same mu without a broadcast
      double b = (red[par][lane][0] + red[par][lane][1]) + red[par][lane][2];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) b += __shfl_down_sync(0xffffffffu, b, o);
      b = __shfl_sync(0xffffffffu, b, 0);
      par ^= 1;   // the other buffer was last read before this barrier
      b += cf.z;
      const double a = cf.x, c = cf.y + dk;
      const double mu = (a > 0.0) ? -c + soft(c - b / a, cf.w / a) : 0.0;
      if (threadIdx.x == 0) D[k] = dk + mu;
      if (mu != 0.0) {
        const double* Sj = S + (int64_t)j * lds;
        double* Ur_i = U + (int64_t)i * ldu;
        double* Ur_j = U + (int64_t)j * ldu;
        for (int t0 = threadIdx.x; t0 < q; t0 += CD_UNR * CD_NT) {
          double a0[CD_UNR], a1[CD_UNR], s0[CD_UNR], s1[CD_UNR];
#pragma unroll
          for (int u = 0; u < CD_UNR; ++u) {
            const int t = t0 + u * CD_NT;
            const bool in = t < q;
            a0[u] = in ? Ur_i[t] : 0.0;
            s0[u] = in ? Sj[t] : 0.0;
            a1[u] = (in && i != j) ? Ur_j[t] : 0.0;
            s1[u] = (in && i != j) ? Si[t] : 0.0;
          }
#pragma unroll
          for (int u = 0; u < CD_UNR; ++u) {
            const int t = t0 + u * CD_NT;
            if (t < q) {
              if (i != j) {
                Ur_i[t] = a0[u] + mu * s0[u];
                Ur_j[t] = a1[u] + mu * s1[u];
              } else {
                Ur_i[t] = a0[u] + mu * s0[u];
              }
            }
          }
        }
      }
      __syncthreads();
    }
  }
  // line-search decrease measure and ||Lambda||_1, fixed-order block reduction
  __shared__ double red3[CD_NW][3];
  double v[3] = {0.0, 0.0, 0.0};
  for (int64_t k = threadIdx.x; k < m; k += CD_NT) {
    const int i = Lr[k], j = Lc[k];
    const double wgt = (i == j) ? 1.0 : 2.0;
    const double4 cf = coef[k];
    v[0] += wgt * cf.z * D[k];
    v[1] += wgt * cf.w * (fabs(cf.y + D[k]) - fabs(cf.y));
  }
  for (int j = threadIdx.x; j < q; j += CD_NT)
    for (int64_t t = colptr[j]; t < colptr[j + 1]; ++t) v[2] += fabs(lval[t]);
  block_sum<3>(v, red3);
  if (threadIdx.x == 0) {
    out[0] = v[0];
    out[1] = v[1];
    out[2] = v[2];
  }
}

// V = Theta Sigma (p x q, ldv, zeroed): one warp per output column t walks Theta's columns in
// order (distinct rows inside a column: no write conflicts), deterministic summation order.
__global__ void k_theta_sigma(int q, const int64_t* colptr, const int32_t* rowidx, const double* val,
                              const double* __restrict__ S, int64_t lds, double* V, int64_t ldv) {
  const int t = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (t >= q) return;
  double* Vt = V + (int64_t)t * ldv;
  for (int j = 0; j < q; ++j) {
    const int64_t a = colptr[j], b = colptr[j + 1];
    if (a == b) continue;
    const double s = S[j + (int64_t)t * lds];
    for (int64_t e = a + lane; e < b; e += 32) Vt[rowidx[e]] += val[e] * s;
    __syncwarp();
  }
}

// Column of S_xx holding row / column i: the full p x p matrix (xmap null), or the compact block of
// the active rows' columns (cggm_gram_rows: xmap[i] = position of row i among them; NEXT-2 on-demand
// (S_xx)_i = X^T X_i / n)
__device__ __forceinline__ int64_t xcol(const int32_t* __restrict__ xmap, int i) { return xmap ? xmap[i] : i; }

// Per-entry constants of the Theta sweep: a = 2 Sigma_jj (S_xx)_ii, 2 (S_xy)_ij, the current Theta_ij
// (gathered from the CSC into T, the sweep's state) -- before the sequential walk.
__global__ void k_theta_coefs(int64_t m, const double* __restrict__ S, int64_t lds, const double* __restrict__ Sxx,
                              int64_t ldx, const int32_t* __restrict__ xmap, const double* __restrict__ Sxy, int64_t ldxy, const int64_t* colptr,
                              const int32_t* rowidx, const double* tval, const int32_t* Tr, const int32_t* Tc,
                              double2* coef, double* T) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < m; k += (int64_t)gridDim.x * blockDim.x) {
    const int i = Tr[k], j = Tc[k];
    coef[k] = make_double2(2.0 * S[j + (int64_t)j * lds] * Sxx[i + xcol(xmap, i) * ldx], 2.0 * Sxy[i + (int64_t)j * ldxy]);
    T[k] = csc_at(colptr, rowidx, tval, i, j);
  }
}

// One CTA: Theta values on the active list (T: the gathered current values on entry, the new ones
// on exit); V = Theta Sigma maintained (column-major: the length-p dot reads a contiguous column,
// the length-q row update is strided -- p > q on the paper's problems).  Same one-barrier-per-step
// structure as the Lambda sweep.  out[0] = ||Theta_new||_1.
__global__ void __launch_bounds__(CD_NT) k_theta_cd(int p, int q, const double* __restrict__ S, int64_t lds,
                                                    const double* __restrict__ Sxx, int64_t ldx,
                                                    const int32_t* __restrict__ xmap, const int32_t* Tr,
                                                    const int32_t* Tc, const double2* coef, int64_t m, double lam,
                                                    int passes, double* T, double* V, int64_t ldv, double* out) {
  __shared__ double red[2][CD_NW];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int par = 0;
  for (int pass = 0; pass < passes; ++pass) {
    int ni = m > 0 ? Tr[0] : 0, nj = m > 0 ? Tc[0] : 0;
    double2 nc = m > 0 ? coef[0] : make_double2(0, 0);
    double nt = m > 0 ? T[0] : 0.0;
    for (int64_t k = 0; k < m; ++k) {
      const int i = ni, j = nj;
      const double2 cf = nc;
      const double c = nt;
      if (k + 1 < m) {
        ni = Tr[k + 1];
        nj = Tc[k + 1];
        nc = coef[k + 1];
        nt = T[k + 1];
      }
      const double* Xi = Sxx + xcol(xmap, i) * ldx;   // row i of S_xx = column i
      const double* Vj = V + (int64_t)j * ldv;
      double v = 0.0;
      for (int t0 = threadIdx.x; t0 < p; t0 += CD_UNR * CD_NT) {
        double xa[CD_UNR], va[CD_UNR];
#pragma unroll
        for (int u = 0; u < CD_UNR; ++u) {
          const int t = t0 + u * CD_NT;
          xa[u] = t < p ? Xi[t] : 0.0;
          va[u] = t < p ? Vj[t] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < CD_UNR; ++u) v = fma(xa[u], va[u], v);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) red[par][w] = v;
      __syncthreads();
      double dot = red[par][lane];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) dot += __shfl_down_sync(0xffffffffu, dot, o);
      dot = __shfl_sync(0xffffffffu, dot, 0);
      par ^= 1;
      const double a = cf.x, b = cf.y + 2.0 * dot;
      const double mu = (a > 0.0) ? -c + soft(c - b / a, lam / a) : 0.0;
      if (threadIdx.x == 0) T[k] = c + mu;
      if (mu != 0.0) {
        const double* Sj = S + (int64_t)j * lds;
        for (int t0 = threadIdx.x; t0 < q; t0 += CD_UNR * CD_NT) {
          double va[CD_UNR], sa[CD_UNR];
#pragma unroll
          for (int u = 0; u < CD_UNR; ++u) {
            const int t = t0 + u * CD_NT;
            va[u] = t < q ? V[i + (int64_t)t * ldv] : 0.0;
            sa[u] = t < q ? Sj[t] : 0.0;
          }
#pragma unroll
          for (int u = 0; u < CD_UNR; ++u) {
            const int t = t0 + u * CD_NT;
            if (t < q) V[i + (int64_t)t * ldv] = va[u] + mu * sa[u];
          }
        }
      }
      __syncthreads();
    }
  }
  __shared__ double red1[CD_NW][1];
  double vv[1] = {0.0};
  for (int64_t k = threadIdx.x; k < m; k += CD_NT) vv[0] += fabs(T[k]);
  block_sum<1>(vv, red1);
  if (threadIdx.x == 0) out[0] = vv[0];
}

// ---------------------------------------------------------------- column-batched cooperative sweeps
// The active lists are column-major, so consecutive updates share the column j.  With
// Z = D Psi (so that (Psi D Sigma)_ji = (Sigma D Psi)_ij = Sigma_i . Z_{:,j}) every dot product of
// the Lambda update reads only column j of U = D Sigma and of Z:
//     b = GradL_ij + (Sigma_i + Psi_i) . U_{:,j} + Sigma_i . Z_{:,j}
// and an update changes column j in two entries only (rows i and j).  So per column: CTA 0 walks
// the column's entries with U_{:,j}, Z_{:,j} in shared memory (O(1) column updates), then the whole
// grid applies the column's deferred row updates U[i, t] += mu Sigma[j, t], U[j, t] += mu Sigma[i, t]
// (and Z with Psi) to every other column t -- off the sequential chain, coalesced (U, Z row-major).
// Two grid barriers per non-empty column.  The Theta sweep is the same with V = Theta Sigma.
constexpr int CO_NT = 512;
constexpr int CO_NW = CO_NT / 32;
constexpr int CO_UNR = 8;

__device__ __forceinline__ double co_block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) red[w] = v;
  __syncthreads();
  double b = lane < CO_NW ? red[lane] : 0.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) b += __shfl_down_sync(0xffffffffu, b, o);
  b = __shfl_sync(0xffffffffu, b, 0);   // the same value in every thread
  __syncthreads();
  return b;
}

__global__ void __launch_bounds__(CO_NT) k_lambda_sweep_coop(int q, const double* __restrict__ S, int64_t lds,
                                                             const double* __restrict__ P, int64_t ldp,
                                                             const int32_t* Lr, const double4* coef, const int64_t* lp,
                                                             int passes, double* D, double* dmu, double* U, double* Z,
                                                             int64_t ldu, double* colbuf, int use_smem) {
  namespace cgx = cooperative_groups;
  cgx::grid_group grid = cgx::this_grid();
  extern __shared__ double co_sm[];
  __shared__ double red[CO_NW];
  double* Uj = use_smem ? co_sm : colbuf;
  double* Zj = Uj + q;
  const int64_t gtid = blockIdx.x * (int64_t)CO_NT + threadIdx.x, gsz = (int64_t)gridDim.x * CO_NT;
  for (int pass = 0; pass < passes; ++pass) {
    for (int j = 0; j < q; ++j) {
      const int64_t k0 = lp[j], k1 = lp[j + 1];
      if (k0 == k1) continue;
      if (blockIdx.x == 0) {
        for (int t = threadIdx.x; t < q; t += CO_NT) {
          Uj[t] = U[(int64_t)t * ldu + j];
          Zj[t] = Z[(int64_t)t * ldu + j];
        }
        __syncthreads();
        const double Sjj = S[j + (int64_t)j * lds], Pjj = P[j + (int64_t)j * ldp];
        for (int64_t k = k0; k < k1; ++k) {
          const int i = Lr[k];
          const double4 cf = coef[k];
          const double* Si = S + (int64_t)i * lds;
          const double* Pi = P + (int64_t)i * ldp;
          // CO_UNR elements per thread in flight at once (the columns come from DRAM / L2)
          double v = 0.0;
          for (int t0 = threadIdx.x; t0 < q; t0 += CO_UNR * CO_NT) {
            double sv[CO_UNR], pv[CO_UNR];
#pragma unroll
            for (int u = 0; u < CO_UNR; ++u) {
              const int t = t0 + u * CO_NT;
              sv[u] = t < q ? Si[t] : 0.0;
              pv[u] = t < q ? Pi[t] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < CO_UNR; ++u) {
              const int t = t0 + u * CO_NT;
              if (t < q) v = fma(sv[u] + pv[u], Uj[t], fma(sv[u], Zj[t], v));
            }
          }
          const double b = cf.z + co_block_sum(v, red);
          const double a = cf.x, c = cf.y + D[k];
          const double mu = (a > 0.0) ? -c + soft(c - b / a, cf.w / a) : 0.0;
          if (threadIdx.x == 0) {
            D[k] = c - cf.y + mu;
            dmu[k] = mu;
            Uj[i] += mu * Sjj;
            Zj[i] += mu * Pjj;
            if (i != j) {
              Uj[j] += mu * Si[j];
              Zj[j] += mu * Pi[j];
            }
          }
          __syncthreads();
        }
        for (int t = threadIdx.x; t < q; t += CO_NT) {
          U[(int64_t)t * ldu + j] = Uj[t];
          Z[(int64_t)t * ldu + j] = Zj[t];
        }
      }
      grid.sync();
      // the column's deferred row updates, t != j (column j is current in memory already):
      //   rows i_k != j: U[i_k, t] += mu_k Sigma[j, t], Z[i_k, t] += mu_k Psi[j, t]  -- parallel over (k, t)
      //   row j:         U[j, t] += sum_k mu_k Sigma[i_k, t] (Z with Psi)          -- parallel over t
      // (disjoint elements: no ordering between the two loops)
      {
        const int64_t nk = k1 - k0, work = nk * (int64_t)q;
        for (int64_t w = gtid; w < work; w += gsz) {
          const int64_t k = k0 + w / q;
          const int t = (int)(w - (k - k0) * q);
          const int i = Lr[k];
          const double mu = dmu[k];
          if (t == j || i == j || mu == 0.0) continue;
          U[(int64_t)i * ldu + t] += mu * S[t + (int64_t)j * lds];
          Z[(int64_t)i * ldu + t] += mu * P[t + (int64_t)j * ldp];
        }
        for (int64_t t = gtid; t < q; t += gsz) {
          if (t == j) continue;
          double ua = 0.0, za = 0.0;
          for (int64_t k = k0; k < k1; ++k) {
            const double mu = dmu[k];
            const int i = Lr[k];
            ua = fma(mu, S[t + (int64_t)i * lds], ua);
            za = fma(mu, P[t + (int64_t)i * ldp], za);
          }
          U[(int64_t)j * ldu + t] += ua;
          Z[(int64_t)j * ldu + t] += za;
        }
      }
      grid.sync();
    }
  }
}

// the Lambda sweep's scalars after the walk: out[0] = tr(GradL^T D), out[1] = the penalty change,
// out[2] = ||Lambda||_1
__global__ void __launch_bounds__(CD_NT) k_lambda_tail(int q, const int64_t* colptr, const double* lval,
                                                       const int32_t* Lr, const int32_t* Lc, const double4* coef,
                                                       int64_t m, const double* D, double* out) {
  __shared__ double red3[CD_NW][3];
  double v[3] = {0.0, 0.0, 0.0};
  for (int64_t k = threadIdx.x; k < m; k += CD_NT) {
    const double wgt = (Lr[k] == Lc[k]) ? 1.0 : 2.0;
    const double4 cf = coef[k];
    v[0] += wgt * cf.z * D[k];
    v[1] += wgt * cf.w * (fabs(cf.y + D[k]) - fabs(cf.y));
  }
  for (int j = threadIdx.x; j < q; j += CD_NT)
    for (int64_t t = colptr[j]; t < colptr[j + 1]; ++t) v[2] += fabs(lval[t]);
  block_sum<3>(v, red3);
  if (threadIdx.x == 0) {
    out[0] = v[0];
    out[1] = v[1];
    out[2] = v[2];
  }
}

__global__ void __launch_bounds__(CD_NT) k_theta_l1(const double* T, int64_t m, double* out) {
  __shared__ double red1[CD_NW][1];
  double v[1] = {0.0};
  for (int64_t k = threadIdx.x; k < m; k += CD_NT) v[0] += fabs(T[k]);
  block_sum<1>(v, red1);
  if (threadIdx.x == 0) out[0] = v[0];
}

// V = Theta Sigma, ROW-major (row stride ldv): one warp per output column t
__global__ void k_theta_sigma_rm(int q, const int64_t* colptr, const int32_t* rowidx, const double* val,
                                 const double* __restrict__ S, int64_t lds, double* V, int64_t ldv) {
  const int t = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (t >= q) return;
  for (int j = 0; j < q; ++j) {
    const int64_t a = colptr[j], b = colptr[j + 1];
    if (a == b) continue;
    const double s = S[j + (int64_t)t * lds];
    for (int64_t e = a + lane; e < b; e += 32) V[(int64_t)rowidx[e] * ldv + t] += val[e] * s;
    __syncwarp();
  }
}

__global__ void __launch_bounds__(CO_NT) k_theta_sweep_coop(int p, int q, const double* __restrict__ S, int64_t lds,
                                                            const double* __restrict__ Sxx, int64_t ldx,
                                                            const int32_t* __restrict__ xmap,
                                                            const int32_t* Tr, const double2* coef, const int64_t* lp,
                                                            double lam, int passes, double* T, double* dmu, double* V,
                                                            int64_t ldv, double* colbuf, int use_smem) {
  namespace cgx = cooperative_groups;
  cgx::grid_group grid = cgx::this_grid();
  extern __shared__ double co_sm[];
  __shared__ double red[CO_NW];
  double* Vj = use_smem ? co_sm : colbuf;
  const int64_t gtid = blockIdx.x * (int64_t)CO_NT + threadIdx.x, gsz = (int64_t)gridDim.x * CO_NT;
  for (int pass = 0; pass < passes; ++pass) {
    for (int j = 0; j < q; ++j) {
      const int64_t k0 = lp[j], k1 = lp[j + 1];
      if (k0 == k1) continue;
      if (blockIdx.x == 0) {
        for (int t = threadIdx.x; t < p; t += CO_NT) Vj[t] = V[(int64_t)t * ldv + j];
        __syncthreads();
        const double Sjj = S[j + (int64_t)j * lds];
        for (int64_t k = k0; k < k1; ++k) {
          const int i = Tr[k];
          const double2 cf = coef[k];
          const double* Xi = Sxx + xcol(xmap, i) * ldx;
          double v = 0.0;
          for (int t0 = threadIdx.x; t0 < p; t0 += CO_UNR * CO_NT) {
            double xv[CO_UNR];
#pragma unroll
            for (int u = 0; u < CO_UNR; ++u) {
              const int t = t0 + u * CO_NT;
              xv[u] = t < p ? Xi[t] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < CO_UNR; ++u) {
              const int t = t0 + u * CO_NT;
              if (t < p) v = fma(xv[u], Vj[t], v);
            }
          }
          const double b = cf.y + 2.0 * co_block_sum(v, red);
          const double a = cf.x, c = T[k];
          const double mu = (a > 0.0) ? -c + soft(c - b / a, lam / a) : 0.0;
          if (threadIdx.x == 0) {
            T[k] = c + mu;
            dmu[k] = mu;
            Vj[i] += mu * Sjj;
          }
          __syncthreads();
        }
        for (int t = threadIdx.x; t < p; t += CO_NT) V[(int64_t)t * ldv + j] = Vj[t];
      }
      grid.sync();
      {   // deferred row updates V[i_k, t] += mu_k Sigma[j, t], t != j: parallel over (k, t)
        const int64_t nk = k1 - k0, work = nk * (int64_t)q;
        for (int64_t w = gtid; w < work; w += gsz) {
          const int64_t k = k0 + w / q;
          const int t = (int)(w - (k - k0) * q);
          const double mu = dmu[k];
          if (t == j || mu == 0.0) continue;
          V[(int64_t)Tr[k] * ldv + t] += mu * S[t + (int64_t)j * lds];
        }
      }
      grid.sync();
    }
  }
}

// Lambda sweep, register/prefetch variant (q <= CO_QMAX): columns j of U and Z live in registers, the
// Sigma and Psi columns of the NEXT entry are fetched by cp.async while the current update runs.
constexpr int CO_LU = 12;
constexpr int CO_QMAX = CO_NT * CO_LU;

__global__ void __launch_bounds__(CO_NT) k_lambda_sweep_pf(int q, const double* __restrict__ S, int64_t lds,
                                                           const double* __restrict__ P, int64_t ldp,
                                                           const int32_t* Lr, const double4* coef, const int64_t* lp,
                                                           int passes, double* D, double* dmu, double* U, double* Z,
                                                           int64_t ldu) {
  namespace cgx = cooperative_groups;
  cgx::grid_group grid = cgx::this_grid();
  extern __shared__ double co_sm[];
  __shared__ double red[CO_NW];
  const int64_t qs = (q + 1) & ~1;
  double* sb[2] = {co_sm, co_sm + 2 * qs};   // [Sigma_i | Psi_i] per buffer
  const int64_t gtid = blockIdx.x * (int64_t)CO_NT + threadIdx.x, gsz = (int64_t)gridDim.x * CO_NT;
  const int x = threadIdx.x;
  auto fetch = [&](int i, int b) {
    const double* s1 = S + (int64_t)i * lds;
    const double* p1 = P + (int64_t)i * ldp;
    for (int c2 = x; 2 * c2 < q; c2 += CO_NT) {
      const int r = 2 * c2;
      const uint32_t by = (r + 1 < q) ? 16u : 8u;
      ptx::cp_async16(sb[b] + r, s1 + r, by);
      ptx::cp_async16(sb[b] + qs + r, p1 + r, by);
    }
    ptx::cp_async_commit();
  };
  for (int pass = 0; pass < passes; ++pass) {
    for (int j = 0; j < q; ++j) {
      const int64_t k0 = lp[j], k1 = lp[j + 1];
      if (k0 == k1) continue;
      if (blockIdx.x == 0) {
        double ur[CO_LU], zr[CO_LU];
#pragma unroll
        for (int u = 0; u < CO_LU; ++u) {
          const int t = x + u * CO_NT;
          ur[u] = t < q ? U[(int64_t)t * ldu + j] : 0.0;
          zr[u] = t < q ? Z[(int64_t)t * ldu + j] : 0.0;
        }
        const double Sjj = S[j + (int64_t)j * lds], Pjj = P[j + (int64_t)j * ldp];
        int cur = 0;
        fetch(Lr[k0], 0);
        for (int64_t k = k0; k < k1; ++k) {
          const int i = Lr[k];
          const double4 cf = coef[k];
          if (k + 1 < k1) {
            fetch(Lr[k + 1], cur ^ 1);
            ptx::cp_async_wait<1>();
          } else {
            ptx::cp_async_wait<0>();
          }
          __syncthreads();
          const double* Si = sb[cur];
          const double* Pi = sb[cur] + qs;
          double v = 0.0;
#pragma unroll
          for (int u = 0; u < CO_LU; ++u) {
            const int t = x + u * CO_NT;
            if (t < q) v = fma(Si[t] + Pi[t], ur[u], fma(Si[t], zr[u], v));
          }
          const double b = cf.z + co_block_sum(v, red);
          const double a = cf.x, c = cf.y + D[k];
          const double mu = (a > 0.0) ? -c + soft(c - b / a, cf.w / a) : 0.0;
          if (x == 0) {
            D[k] = c - cf.y + mu;
            dmu[k] = mu;
          }
          if (mu != 0.0) {
            const double sij = Si[j], pij = Pi[j];   // Sigma_ji, Psi_ji from the staged column i
            const int ui = i / CO_NT, uj = j / CO_NT;
            const bool own_i = x == (i % CO_NT), own_j = (i != j) && x == (j % CO_NT);
#pragma unroll
            for (int u = 0; u < CO_LU; ++u) {
              if (own_i && u == ui) {
                ur[u] += mu * Sjj;
                zr[u] += mu * Pjj;
              }
              if (own_j && u == uj) {
                ur[u] += mu * sij;
                zr[u] += mu * pij;
              }
            }
          }
          cur ^= 1;
        }
#pragma unroll
        for (int u = 0; u < CO_LU; ++u) {
          const int t = x + u * CO_NT;
          if (t < q) {
            U[(int64_t)t * ldu + j] = ur[u];
            Z[(int64_t)t * ldu + j] = zr[u];
          }
        }
      }
      grid.sync();
      {
        const int64_t nk = k1 - k0, work = nk * (int64_t)q;
        for (int64_t w = gtid; w < work; w += gsz) {
          const int64_t k = k0 + w / q;
          const int t = (int)(w - (k - k0) * q);
          const int i = Lr[k];
          const double mu = dmu[k];
          if (t == j || i == j || mu == 0.0) continue;
          U[(int64_t)i * ldu + t] += mu * S[t + (int64_t)j * lds];
          Z[(int64_t)i * ldu + t] += mu * P[t + (int64_t)j * ldp];
        }
        for (int64_t t = gtid; t < q; t += gsz) {
          if (t == j) continue;
          double ua = 0.0, za = 0.0;
          for (int64_t k = k0; k < k1; ++k) {
            const double mu = dmu[k];
            const int i = Lr[k];
            ua = fma(mu, S[t + (int64_t)i * lds], ua);
            za = fma(mu, P[t + (int64_t)i * ldp], za);
          }
          U[(int64_t)j * ldu + t] += ua;
          Z[(int64_t)j * ldu + t] += za;
        }
      }
      grid.sync();
    }
  }
}

// Theta sweep, register/prefetch variant (p <= CO_PMAX): column j of V lives in registers (thread
// x owns rows x, x + 512, ...), and the S_xx column of the NEXT entry is fetched by cp.async into
// the other half of a shared double buffer while the current dot product runs -- the sequential
// walk no longer waits on DRAM for each update's length-p column.
constexpr int CO_VU = 24;                 // register slots per thread: p <= 512 * 24
constexpr int CO_PMAX = CO_NT * CO_VU;

__global__ void __launch_bounds__(CO_NT) k_theta_sweep_pf(int p, int q, const double* __restrict__ S, int64_t lds,
                                                          const double* __restrict__ Sxx, int64_t ldx,
                                                          const int32_t* __restrict__ xmap,
                                                          const int32_t* Tr, const double2* coef, const int64_t* lp,
                                                          double lam, int passes, double* T, double* dmu, double* V,
                                                          int64_t ldv) {
  namespace cgx = cooperative_groups;
  cgx::grid_group grid = cgx::this_grid();
  extern __shared__ double co_sm[];
  __shared__ double red[CO_NW];
  const int64_t pst = (p + 1) & ~1;        // buffer stride (16-byte aligned halves)
  double* buf[2] = {co_sm, co_sm + pst};
  const int64_t gtid = blockIdx.x * (int64_t)CO_NT + threadIdx.x, gsz = (int64_t)gridDim.x * CO_NT;
  const int x = threadIdx.x;
  // S_xx column i -> shared buffer b, 16-byte cp.async chunks (ldx even, so columns are aligned)
  auto fetch = [&](int i, int b) {
    const double* src = Sxx + xcol(xmap, i) * ldx;
    for (int c2 = x; 2 * c2 < p; c2 += CO_NT) {
      const int r = 2 * c2;
      ptx::cp_async16(buf[b] + r, src + r, (r + 1 < p) ? 16u : 8u);
    }
    ptx::cp_async_commit();
  };
  for (int pass = 0; pass < passes; ++pass) {
    for (int j = 0; j < q; ++j) {
      const int64_t k0 = lp[j], k1 = lp[j + 1];
      if (k0 == k1) continue;
      if (blockIdx.x == 0) {
        double vr[CO_VU];
#pragma unroll
        for (int u = 0; u < CO_VU; ++u) {
          const int t = x + u * CO_NT;
          vr[u] = t < p ? V[(int64_t)t * ldv + j] : 0.0;
        }
        const double Sjj = S[j + (int64_t)j * lds];
        int cur = 0;
        fetch(Tr[k0], 0);
        for (int64_t k = k0; k < k1; ++k) {
          const int i = Tr[k];
          const double2 cf = coef[k];
          if (k + 1 < k1) {
            fetch(Tr[k + 1], cur ^ 1);
            ptx::cp_async_wait<1>();    // the current column has landed (the next may be in flight)
          } else {
            ptx::cp_async_wait<0>();
          }
          __syncthreads();
          const double* Xs = buf[cur];
          double v = 0.0;
#pragma unroll
          for (int u = 0; u < CO_VU; ++u) {
            const int t = x + u * CO_NT;
            if (t < p) v = fma(Xs[t], vr[u], v);
          }
          const double b = cf.y + 2.0 * co_block_sum(v, red);   // (its barriers also retire buf[cur])
          const double a = cf.x, c = T[k];
          const double mu = (a > 0.0) ? -c + soft(c - b / a, lam / a) : 0.0;
          if (x == 0) {
            T[k] = c + mu;
            dmu[k] = mu;
          }
          if (mu != 0.0 && x == (i % CO_NT)) {
            const int ui = i / CO_NT;
#pragma unroll
            for (int u = 0; u < CO_VU; ++u)
              if (u == ui) vr[u] += mu * Sjj;
          }
          cur ^= 1;
        }
#pragma unroll
        for (int u = 0; u < CO_VU; ++u) {
          const int t = x + u * CO_NT;
          if (t < p) V[(int64_t)t * ldv + j] = vr[u];
        }
      }
      grid.sync();
      {
        const int64_t nk = k1 - k0, work = nk * (int64_t)q;
        for (int64_t w = gtid; w < work; w += gsz) {
          const int64_t k = k0 + w / q;
          const int t = (int)(w - (k - k0) * q);
          const double mu = dmu[k];
          if (t == j || mu == 0.0) continue;
          V[(int64_t)Tr[k] * ldv + t] += mu * S[t + (int64_t)j * lds];
        }
      }
      grid.sync();
    }
  }
}

// ---------------------------------------------------------------- entry-blocked cooperative sweeps
// When the column vector no longer fits the register variants (q > CO_QMAX / p > CO_PMAX: large and
// sharded), the column walk above leaves every dot product -- two length-q rows of Sigma / Psi, or a
// length-p column of S_xx, straight from DRAM -- to the one CTA on the sequential chain (13.9 us per
// update at large).  Within column j an update of entry m changes the column vector in two places
// only, so the dot product of a later entry k' of the same column is its value against the vector
// as it stood at the start of a block of entries plus one coupling term per earlier entry of the
// block (Lambda sweep, u = U_{:,j}, z = Z_{:,j}, rows i_m of the block):
//   b_k' = b0_k' + sum_{m < k'} mu_m c_{k'm},
//   c_{k'm} = Sjj (Sigma + Psi)_{i_k' i_m} + Psi_jj Sigma_{i_k' i_m}
//           + [i_m != j] (Sigma_{i_m j} (Sigma + Psi)_{i_k' j} + Psi_{i_m j} Sigma_{i_k' j})
// (Theta sweep, v = V_{:,j}: c_{k'm} = 2 Sigma_jj (S_xx)_{i_k' i_m}).  Per block of BK_B entries:
// phase 1 -- the whole grid, one warp per (entry, 1024-element chunk) item, forms the b0 partials
// (the same bytes the chain used to read, now at the grid's bandwidth) and the coupling matrix
// C (row m = the coefficients of mu_m, gathered from row i_m and row j); phase 2 -- one warp of CTA 0
// runs the block's updates in list order with C in shared memory: per update one shuffle, the
// closed-form coordinate minimiser (the same expression as above), and one FMA per later entry.
// The column vector is then advanced by the block's changes, and after the column the deferred row
// updates run as in the column walk.  Same updates in the same order; the dot products are summed
// in a different (fixed) order, so results agree with the column walk to rounding and are bitwise
// reproducible run to run.
// CGGM_CD_TIMING=1 (measurement aid): CTA 0 accumulates %globaltimer deltas per phase -- 0 column
// load + panel-row recompute, 1 phase 1, 2 phase-2 staging, 3 phase-2 chain + barrier, 4 column end
__device__ unsigned long long g_cd_tim[8];
__device__ int g_cd_tim_on;
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
constexpr int BK_B = 128;              // entries per block
constexpr int BK_R = BK_B / 32;        // block entries per lane in phase 2
constexpr int BK_CH = 1280;            // dot-product elements per warp item (large: 128 x 17 items, one round of the grid's 2368 warps)
constexpr int BK_U = 8;                // loads in flight per lane and operand
constexpr size_t BK_SMEM = (size_t)BK_B * BK_B * 8 + (size_t)BK_B * (7 * 8 + 4) + (size_t)BK_B * 64;

template <bool LAM>
__global__ void __launch_bounds__(CO_NT, 1) k_sweep_blk(int q, int nlen, const double* __restrict__ S, int64_t lds,
                                                     const double* __restrict__ P, int64_t ldp,
                                                     const int32_t* __restrict__ xmap, const int32_t* __restrict__ Lr,
                                                     const double* __restrict__ coefv, const int64_t* __restrict__ lp,
                                                     double lam, int passes, double* X, double* dmu, double* U,
                                                     double* Z, int64_t ldu, double* ucol, double* part, double* Ct,
                                                     double* sj, int j0, int j1, double* Dd, int64_t ldd,
                                                     double* rpart) {
  namespace cgx = cooperative_groups;
  cgx::grid_group grid = cgx::this_grid();
  extern __shared__ double bk_sm[];
  double* sC = bk_sm;                         // [BK_B][BK_B]: row m = coefficients of mu_m
  double* sB = sC + BK_B * BK_B;              // b0 + the entry's constant
  double* sA = sB + BK_B;                     // 1 / a (0 when a <= 0: no update)
  double* sT = sA + BK_B;                     // the entry's threshold / a
  double* sY = sT + BK_B;                     // Lambda: Lambda_ij (+ D_ij below); Theta: current value
  double* sW = sY + BK_B;                     // Lambda: c = Lambda_ij + D_ij
  double* sSj = sW + BK_B;                    // Lambda: Sigma_{i j}, Psi_{i j} of the block's rows
  double* sPj = sSj + BK_B;
  int* sI = reinterpret_cast<int*>(sPj + BK_B);
  // the chain's per-entry operands packed 64 bytes apiece (three 16-byte loads from one address):
  // 1 / a, c, threshold / a, C[k][k + 1], and Lambda's column-j factors (the diagonal's already chosen)
  double* sK = reinterpret_cast<double*>(sI + BK_B);
  double* zcol = ucol + nlen;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t gtid = blockIdx.x * (int64_t)CO_NT + threadIdx.x, gsz = (int64_t)gridDim.x * CO_NT;
  const int gw = blockIdx.x * CO_NW + warp, nwarps = gridDim.x * CO_NW;
  const int nch = (nlen + BK_CH - 1) / BK_CH;
  const double4* coef4 = reinterpret_cast<const double4*>(coefv);
  const double2* coef2 = reinterpret_cast<const double2*>(coefv);
  const bool tim = g_cd_tim_on && blockIdx.x == 0 && threadIdx.x == 0;
  unsigned long long tacc[5] = {0, 0, 0, 0, 0}, tl = 0;
#define CD_TICK(slot)                 \
  if (tim) {                          \
    const unsigned long long tn = gtimer(); \
    tacc[slot] += tn - tl;            \
    tl = tn;                          \
  }
  for (int pass = 0; pass < passes; ++pass) {
    for (int j = j0; j < j1; ++j) {
      const int64_t k0 = lp[j], k1 = lp[j + 1];
      if (k0 == k1) continue;
      if (tim) tl = gtimer();
      for (int64_t t = gtid; t < nlen; t += gsz) {
        ucol[t] = __ldcg(U + t * ldu + j);
        if (LAM) zcol[t] = __ldcg(Z + t * ldu + j);
      }
      const double Sjj = S[j + (int64_t)j * lds];
      const double Pjj = LAM ? P[j + (int64_t)j * ldp] : 0.0;
      if (LAM && Dd && j > j0) {
        // panel mode: rows r in [j0, j) of column j -- the rows this panel's earlier columns rewrote
        // wholesale -- are formed from the current dense D: U[r, j] = D_{:,r} . Sigma_{:,j},
        // Z[r, j] = D_{:,r} . Psi_{:,j} (chunk partials by the grid, summed in chunk order)
        const int nr = j - j0;
        const double* Sj = S + (int64_t)j * lds;
        const double* Pj = P + (int64_t)j * ldp;
        for (int it = gw; it < nr * nch; it += nwarps) {
          const int rr = it / nch, ch = it - rr * nch;
          const int t0 = ch * BK_CH, t1 = min(nlen, t0 + BK_CH);
          const double* Dr = Dd + (int64_t)(j0 + rr) * ldd;
          double vu = 0.0, vz = 0.0;
          int tb = t0;
          for (; tb + 32 * BK_U <= t1; tb += 32 * BK_U) {
            double dv[BK_U], sv[BK_U], pv[BK_U];
#pragma unroll
            for (int u = 0; u < BK_U; ++u) dv[u] = __ldcg(Dr + tb + lane + 32 * u);
#pragma unroll
            for (int u = 0; u < BK_U; ++u) sv[u] = Sj[tb + lane + 32 * u];
#pragma unroll
            for (int u = 0; u < BK_U; ++u) pv[u] = Pj[tb + lane + 32 * u];
#pragma unroll
            for (int u = 0; u < BK_U; ++u) {
              vu = fma(dv[u], sv[u], vu);
              vz = fma(dv[u], pv[u], vz);
            }
          }
          if (tb < t1) {
            double dv[BK_U], sv[BK_U], pv[BK_U];
#pragma unroll
            for (int u = 0; u < BK_U; ++u) {
              const int t = tb + lane + 32 * u;
              const bool in = t < t1;
              dv[u] = in ? __ldcg(Dr + t) : 0.0;
              sv[u] = in ? Sj[t] : 0.0;
              pv[u] = in ? Pj[t] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < BK_U; ++u) {
              vu = fma(dv[u], sv[u], vu);
              vz = fma(dv[u], pv[u], vz);
            }
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            vu += __shfl_xor_sync(0xffffffffu, vu, o);
            vz += __shfl_xor_sync(0xffffffffu, vz, o);
          }
          if (lane == 0) {
            rpart[2 * (int64_t)it] = vu;
            rpart[2 * (int64_t)it + 1] = vz;
          }
        }
        grid.sync();
        for (int64_t rr = gtid; rr < nr; rr += gsz) {
          double su = 0.0, sz = 0.0;
          for (int ch = 0; ch < nch; ++ch) {
            su += __ldcg(rpart + 2 * (rr * nch + ch));
            sz += __ldcg(rpart + 2 * (rr * nch + ch) + 1);
          }
          ucol[j0 + rr] = su;
          zcol[j0 + rr] = sz;
        }
      }
      grid.sync();
      CD_TICK(0)
      for (int64_t kb = k0; kb < k1; kb += BK_B) {
        const int nb = (int)(k1 - kb < BK_B ? k1 - kb : BK_B);
        // ---- phase 1: b0 partials against the block-start vector, and the coupling rows
        const int nit = nb * (nch + 1);
        for (int it = gw; it < nit; it += nwarps) {
          const int kk = it / (nch + 1), ch = it - kk * (nch + 1);
          const int i = Lr[kb + kk];
          if (ch < nch) {
            const int t0 = ch * BK_CH, t1 = min(nlen, t0 + BK_CH);
            const double* Si = LAM ? S + (int64_t)i * lds : P + xcol(xmap, i) * ldp;
            const double* Pi = LAM ? P + (int64_t)i * ldp : nullptr;
            double v = 0.0;
            int tb = t0;
            // full 32 * BK_U-element steps without predicates, so that all of a step's loads are
            // issued before the first use (with per-load predicates the compiler issued them four
            // at a time, one DRAM round trip per group: phase 1 ran at 1.2 TB/s)
            for (; tb + 32 * BK_U <= t1; tb += 32 * BK_U) {
              double sv[BK_U], pv[BK_U], uv[BK_U], zv[BK_U];
#pragma unroll
              for (int u = 0; u < BK_U; ++u) sv[u] = Si[tb + lane + 32 * u];
              if (LAM) {
#pragma unroll
                for (int u = 0; u < BK_U; ++u) pv[u] = Pi[tb + lane + 32 * u];
              }
#pragma unroll
              for (int u = 0; u < BK_U; ++u) uv[u] = __ldcg(ucol + tb + lane + 32 * u);
              if (LAM) {
#pragma unroll
                for (int u = 0; u < BK_U; ++u) zv[u] = __ldcg(zcol + tb + lane + 32 * u);
              }
#pragma unroll
              for (int u = 0; u < BK_U; ++u) {
                if (LAM) v = fma(sv[u] + pv[u], uv[u], fma(sv[u], zv[u], v));
                else v = fma(sv[u], uv[u], v);
              }
            }
            if (tb < t1) {
              double sv[BK_U], pv[BK_U], uv[BK_U], zv[BK_U];
#pragma unroll
              for (int u = 0; u < BK_U; ++u) {
                const int t = tb + lane + 32 * u;
                const bool in = t < t1;
                sv[u] = in ? Si[t] : 0.0;
                uv[u] = in ? __ldcg(ucol + t) : 0.0;
                if (LAM) {
                  pv[u] = in ? Pi[t] : 0.0;
                  zv[u] = in ? __ldcg(zcol + t) : 0.0;
                }
              }
#pragma unroll
              for (int u = 0; u < BK_U; ++u) {
                if (LAM) v = fma(sv[u] + pv[u], uv[u], fma(sv[u], zv[u], v));
                else v = fma(sv[u], uv[u], v);
              }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (lane == 0) part[(int64_t)kk * nch + ch] = v;
          } else if (LAM) {
            const double* Sm = S + (int64_t)i * lds;
            const double* Pm = P + (int64_t)i * ldp;
            const double smj = Sm[j], pmj = Pm[j];
            if (lane == 0) {
              sj[kk] = smj;
              sj[BK_B + kk] = pmj;
            }
            for (int k2 = lane; k2 < nb; k2 += 32) {
              const int i2 = Lr[kb + k2];
              const double s = Sm[i2], pp = Pm[i2];
              double cv = fma(Sjj, s + pp, Pjj * s);
              if (i != j) {
                const double sk = S[(int64_t)j * lds + i2], pk = P[(int64_t)j * ldp + i2];
                cv += fma(smj, sk + pk, pmj * sk);
              }
              Ct[(int64_t)kk * BK_B + k2] = cv;
            }
          } else {
            const double* Xm = P + xcol(xmap, i) * ldp;
            for (int k2 = lane; k2 < nb; k2 += 32) Ct[(int64_t)kk * BK_B + k2] = 2.0 * Sjj * Xm[Lr[kb + k2]];
          }
        }
        grid.sync();
        CD_TICK(1)
        // ---- phase 2: the block's updates in list order (CTA 0)
        if (blockIdx.x == 0) {
          {
            // the coupling matrix, 16 bytes per load, eight loads in flight per thread
            const double2* Ct2 = reinterpret_cast<const double2*>(Ct);
            double2* sC2 = reinterpret_cast<double2*>(sC);
            const int n2 = nb * BK_B / 2;
            for (int e0 = threadIdx.x; e0 < n2; e0 += CO_NT * 8) {
              double2 cv[8];
              bool live[8];
#pragma unroll
              for (int u = 0; u < 8; ++u) {
                const int e = e0 + u * CO_NT;
                // update m touches only the later entries: pairs of columns <= m are never used
                live[u] = e < n2 && 2 * (e & (BK_B / 2 - 1)) + 1 > e / (BK_B / 2);
                cv[u] = live[u] ? __ldcg(Ct2 + e) : double2{0.0, 0.0};
              }
#pragma unroll
              for (int u = 0; u < 8; ++u) {
                const int e = e0 + u * CO_NT;
                if (live[u]) sC2[e] = cv[u];
              }
            }
          }
          for (int kk = threadIdx.x; kk < nb; kk += CO_NT) {
            const int64_t k = kb + kk;
            double s = 0.0;
#pragma unroll 8
            for (int ch = 0; ch < nch; ++ch) s += __ldcg(part + (int64_t)kk * nch + ch);
            if (LAM) {
              const double4 cf = coef4[k];
              sB[kk] = cf.z + s;
              sA[kk] = cf.x > 0.0 ? 1.0 / cf.x : 0.0;
              sT[kk] = cf.x > 0.0 ? cf.w / cf.x : 0.0;
              sY[kk] = cf.y;
              sW[kk] = cf.y + __ldcg(X + k);
              sI[kk] = Lr[k];
              sSj[kk] = __ldcg(sj + kk);
              sPj[kk] = __ldcg(sj + BK_B + kk);
              sK[8 * kk + 1] = sW[kk];
              sK[8 * kk + 4] = sI[kk] == j ? Sjj : sSj[kk];
              sK[8 * kk + 5] = sI[kk] == j ? Pjj : sPj[kk];
            } else {
              const double2 cf = coef2[k];
              sB[kk] = cf.y + 2.0 * s;
              sA[kk] = cf.x > 0.0 ? 1.0 / cf.x : 0.0;
              sT[kk] = cf.x > 0.0 ? lam / cf.x : 0.0;
              sY[kk] = __ldcg(X + k);
              sI[kk] = Lr[k];
              sK[8 * kk + 1] = sY[kk];
            }
            sK[8 * kk] = sA[kk];
            sK[8 * kk + 2] = sT[kk];
            sK[8 * kk + 3] = __ldcg(Ct + (int64_t)kk * BK_B + min(kk + 1, BK_B - 1));
          }
          __syncthreads();
          CD_TICK(2)
          if (warp == 0) {
            double corr[BK_R], mymu[BK_R];
#pragma unroll
            for (int r = 0; r < BK_R; ++r) {
              const int kk = lane + 32 * r;
              corr[r] = kk < nb ? sB[kk] : 0.0;
              mymu[r] = 0.0;
            }
            double uj = 0.0, zj = 0.0;
            // the step's shared-memory operands are fetched one step ahead, so the chain per update
            // is shuffle -> FMA -> soft threshold -> add -> FMA with no load on it
            // and b of the next update is formed by every lane as fma(mu, C[kk][kk + 1], corr[kk + 1]
            // before this update) -- the owner lane's own arithmetic -- with that corr value
            // broadcast while mu is still being computed: the shuffle is off the chain too
            const double2* sK2 = reinterpret_cast<const double2*>(sK);
            double ia_n = sK2[0].x, c_n = sK2[0].y, th_n = sK2[1].x, cx_n = sK2[1].y, cr_n[BK_R];
            double su_n = LAM ? sK2[2].x : 0.0, sp_n = LAM ? sK2[2].y : 0.0;
            double b_cur = __shfl_sync(0xffffffffu, corr[0], 0);
#pragma unroll
            for (int r2 = 0; r2 < BK_R; ++r2) cr_n[r2] = sC[lane + 32 * r2];
#pragma unroll
            for (int r = 0; r < BK_R; ++r) {
#pragma unroll 4
              for (int s = 0; s < 32; ++s) {
                const int kk = 32 * r + s;
                if (kk >= nb) break;
                const double ia = ia_n, c = c_n, th = th_n, su = su_n, sp = sp_n, cx = cx_n;
                double cr[BK_R];
#pragma unroll
                for (int r2 = 0; r2 < BK_R; ++r2) cr[r2] = cr_n[r2];
                {
                  const int kn = min(kk + 1, BK_B - 1);
                  const double2 k0v = sK2[4 * kn], k1v = sK2[4 * kn + 1];
                  ia_n = k0v.x;
                  c_n = k0v.y;
                  th_n = k1v.x;
                  cx_n = k1v.y;
#pragma unroll
                  for (int r2 = 0; r2 < BK_R; ++r2) cr_n[r2] = sC[kn * BK_B + lane + 32 * r2];
                  if (LAM) {
                    const double2 k2v = sK2[4 * kn + 2];
                    su_n = k2v.x;
                    sp_n = k2v.y;
                  }
                }
                const double b = b_cur;
                double nx = corr[r];
                if (r + 1 < BK_R && s == 31) nx = corr[r + 1 < BK_R ? r + 1 : r];
                const double pre = __shfl_sync(0xffffffffu, nx, (s + 1) & 31);
                // the coordinate minimiser -c + soft(c - b / a, w / a) with 1 / a and w / a formed
                // off the chain; a <= 0 (no update) is stored as 1 / a = w / a = 0, for which the
                // expression is -c + c = 0 exactly
                const double mu = -c + soft(fma(-b, ia, c), th);
                b_cur = fma(mu, cx, pre);
#pragma unroll
                for (int r2 = 0; r2 < BK_R; ++r2) corr[r2] = fma(mu, cr[r2], corr[r2]);
                if (lane == s) mymu[r] = mu;
                if (LAM) {
                  uj = fma(mu, su, uj);
                  zj = fma(mu, sp, zj);
                }
              }
            }
#pragma unroll
            for (int r = 0; r < BK_R; ++r) {
              const int kk = lane + 32 * r;
              if (kk < nb) {
                const int64_t k = kb + kk;
                const double mu = mymu[r];
                const int i = sI[kk];
                if (LAM) {
                  const double dn = sW[kk] - sY[kk] + mu;
                  __stcg(X + k, dn);
                  if (Dd) {
                    __stcg(Dd + i + (int64_t)j * ldd, dn);
                    __stcg(Dd + j + (int64_t)i * ldd, dn);
                  }
                  if (i != j) {
                    __stcg(ucol + i, __ldcg(ucol + i) + mu * Sjj);
                    __stcg(zcol + i, __ldcg(zcol + i) + mu * Pjj);
                  }
                } else {
                  __stcg(X + k, sY[kk] + mu);
                  __stcg(ucol + i, __ldcg(ucol + i) + mu * Sjj);
                }
                __stcg(dmu + k, mu);
              }
            }
            if (LAM && lane == 0) {
              __stcg(ucol + j, __ldcg(ucol + j) + uj);
              __stcg(zcol + j, __ldcg(zcol + j) + zj);
            }
          }
        }
        grid.sync();
        CD_TICK(3)
      }
      // ---- column end: write the column back, deferred row updates (disjoint elements)
      for (int64_t t = gtid; t < nlen; t += gsz) {
        __stcg(U + t * ldu + j, __ldcg(ucol + t));
        if (LAM) __stcg(Z + t * ldu + j, __ldcg(zcol + t));
      }
      {
        for (int64_t k = k0 + blockIdx.x; k < k1; k += gridDim.x) {
          const int i = Lr[k];
          const double mu = __ldcg(dmu + k);
          if ((LAM && i == j) || mu == 0.0) continue;
          // panel mode: only the panel's later columns (the rest of U is never read again before
          // its own panel product)
          const int tlo = (LAM && Dd) ? j + 1 : 0, thi = (LAM && Dd) ? j1 : q;
          for (int t = tlo + threadIdx.x; t < thi; t += CO_NT) {
            if (t == j) continue;
            double* u = U + (int64_t)i * ldu + t;
            __stcg(u, __ldcg(u) + mu * S[t + (int64_t)j * lds]);
            if (LAM) {
              double* z = Z + (int64_t)i * ldu + t;
              __stcg(z, __ldcg(z) + mu * P[t + (int64_t)j * ldp]);
            }
          }
        }
        if (LAM && !Dd) {
          // row j: U[j, t] += sum_k mu_k Sigma[i_k, t] -- 128 columns t per CTA, the k-range split over
          // the CTA's four thread groups (k = k0 + g mod 4), the group sums added in fixed order
          double* rj = bk_sm;   // 2 x 4 x 128 (phase 2's shared memory is free here)
          const int tl = threadIdx.x & 127, g = threadIdx.x >> 7;
          for (int64_t tb = (int64_t)blockIdx.x * 128; tb < q; tb += (int64_t)gridDim.x * 128) {
            const int64_t t = tb + tl;
            double ua = 0.0, za = 0.0;
            if (t < q) {
              for (int64_t k = k0 + g; k < k1; k += CO_NT / 128) {
                const double mu = __ldcg(dmu + k);
                const int i = Lr[k];
                ua = fma(mu, S[t + (int64_t)i * lds], ua);
                za = fma(mu, P[t + (int64_t)i * ldp], za);
              }
            }
            rj[g * 128 + tl] = ua;
            rj[512 + g * 128 + tl] = za;
            __syncthreads();
            if (g == 0 && t < q && t != j) {
              double su = rj[tl], sz = rj[512 + tl];
#pragma unroll
              for (int g2 = 1; g2 < CO_NT / 128; ++g2) {
                su += rj[g2 * 128 + tl];
                sz += rj[512 + g2 * 128 + tl];
              }
              double* u = U + (int64_t)j * ldu + t;
              double* z = Z + (int64_t)j * ldu + t;
              __stcg(u, __ldcg(u) + su);
              __stcg(z, __ldcg(z) + sz);
            }
            __syncthreads();
          }
        }
      }
      grid.sync();
      CD_TICK(4)
    }
  }
  if (tim)
    for (int x = 0; x < 5; ++x) g_cd_tim[x] += tacc[x];
#undef CD_TICK
}

// ---------------------------------------------------------------- sparse bookkeeping
// count list entries per column (cl) and mirrored entries per column (cm: entry (i, j), i < j,
// mirrors into column i)
__global__ void k_list_counts(int64_t m, const int32_t* r, const int32_t* cidx, int mirror, int* cl, int* cm) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < m; k += (int64_t)gridDim.x * blockDim.x) {
    const int i = r[k], j = cidx[k];
    atomicAdd(&cl[j], 1);
    if (mirror && i < j) atomicAdd(&cm[i], 1);
  }
}

// exclusive scans (one block): lp = scan(cl), cp = scan(cl + cm) with cp[n] = total; mb = cp + cl
__global__ void __launch_bounds__(1024) k_list_scan(int n, const int* cl, const int* cm, int64_t* lp, int64_t* cp,
                                                    int64_t* mb) {
  __shared__ int64_t carry_l, carry_c;
  __shared__ int64_t sl[1024], sc[1024];
  if (threadIdx.x == 0) carry_l = carry_c = 0;
  __syncthreads();
  for (int base = 0; base < n; base += 1024) {
    const int c = base + threadIdx.x;
    const int64_t a = c < n ? cl[c] : 0, b = c < n ? (int64_t)cl[c] + (cm ? cm[c] : 0) : 0;
    sl[threadIdx.x] = a;
    sc[threadIdx.x] = b;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {   // Hillis-Steele inclusive scan
      const int64_t xa = threadIdx.x >= o ? sl[threadIdx.x - o] : 0, xb = threadIdx.x >= o ? sc[threadIdx.x - o] : 0;
      __syncthreads();
      sl[threadIdx.x] += xa;
      sc[threadIdx.x] += xb;
      __syncthreads();
    }
    if (c < n) {
      lp[c] = carry_l + sl[threadIdx.x] - a;
      cp[c] = carry_c + sc[threadIdx.x] - b;
      if (mb) mb[c] = cp[c] + a;
    }
    __syncthreads();
    if (threadIdx.x == 1023) {
      carry_l += sl[1023];
      carry_c += sc[1023];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    lp[n] = carry_l;
    cp[n] = carry_c;
  }
}

// Lambda + alpha D as a symmetric CSC: list entries at their column-major rank, mirrored entries
// placed per column in ascending row order by k_mirror_place
__global__ void k_lambda_trial_scatter(int64_t m, const int32_t* Lr, const int32_t* Lc, const double* D, double alpha,
                                       const int64_t* colptr, const int32_t* rowidx, const double* lval,
                                       const int64_t* lp, const int64_t* cp, int32_t* orow, double* oval) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < m; k += (int64_t)gridDim.x * blockDim.x) {
    const int i = Lr[k], j = Lc[k];
    const double v = csc_at(colptr, rowidx, lval, i, j) + alpha * D[k];
    const int64_t pos = cp[j] + (k - lp[j]);
    orow[pos] = i;
    oval[pos] = v;
  }
}

// the mirrored entries: entry (i, j), i < j, goes to column i's mirrored segment [mb[i], cp[i+1]).
// One CTA walks the list's columns j in ascending order (rows are distinct within a column, so the
// column's entries are placed in parallel), so every segment is filled in ascending row order --
// sorted by construction, deterministic, no atomics and no per-segment sort (the insertion sort
// below was quadratic in the segment length: ~19 s for the 1.03e8-entry list at large).
__global__ void __launch_bounds__(1024) k_mirror_place(int n, const int32_t* __restrict__ Lr, const int64_t* lp,
                                                       const int64_t* cp, const int64_t* mb, int* mfill,
                                                       int32_t* orow, double* oval) {
  for (int j = 0; j < n; ++j) {
    const int64_t a = lp[j], b = lp[j + 1];
    for (int64_t k = a + threadIdx.x; k < b; k += blockDim.x) {
      const int i = Lr[k];
      if (i < j) {
        const int64_t mp = mb[i] + mfill[i];
        mfill[i] += 1;
        orow[mp] = j;
        oval[mp] = oval[cp[j] + (k - a)];
      }
    }
    __syncthreads();
  }
}

__global__ void k_copy_list(int64_t m, const int32_t* r, const double* v, int32_t* orow, double* oval) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < m; k += (int64_t)gridDim.x * blockDim.x) {
    orow[k] = r[k];
    oval[k] = v[k];
  }
}

int grid_for(int64_t m) { return (int)std::min<int64_t>(std::max<int64_t>((m + 255) / 256, 1), 148 * 16); }

}  // namespace

void lambda_cd(Ctx* c, int q, const double* S, int64_t lds, const double* P, int64_t ldp, const double* G, int64_t ldg,
               const cggm_csc* Lam, const int32_t* Lr, const int32_t* Lc, int64_t m, double lam, int penalize_diag,
               int passes, double* D, double* U, int64_t ldu, double* coef_ws, double* out) {
  Prof pr(c, TAG_MISC);
  double4* coef = reinterpret_cast<double4*>(coef_ws);
  const double* lv = static_cast<const double*>(Lam->val);
  if (m > 0)
    k_lambda_coefs<<<grid_for(m), 256, 0, c->stream>>>(m, S, lds, P, ldp, G, ldg, Lam->colptr, Lam->rowidx, lv, Lr, Lc,
                                                       lam, penalize_diag, coef);
  k_lambda_cd<<<1, CD_NT, 0, c->stream>>>(q, S, lds, P, ldp, G, ldg, Lam->colptr, Lam->rowidx, lv, Lr, Lc, coef, m,
                                          penalize_diag, lam, passes, D, U, ldu, out);
  c->launches += m > 0 ? 1 : 0;
  post_launch(c, "k_lambda_cd");
}

void theta_sigma(Ctx* c, int q, const cggm_csc* Th, const double* S, int64_t lds, double* V, int64_t ldv) {
  Prof pr(c, TAG_MISC);
  k_theta_sigma<<<(q + 7) / 8, 256, 0, c->stream>>>(q, Th->colptr, Th->rowidx, static_cast<const double*>(Th->val), S,
                                                    lds, V, ldv);
  post_launch(c, "k_theta_sigma");
}

void theta_cd(Ctx* c, int p, int q, const double* S, int64_t lds, const double* Sxx, int64_t ldx, const int32_t* xmap,
              const double* Sxy,
              int64_t ldxy, const cggm_csc* Th, const int32_t* Tr, const int32_t* Tc, int64_t m, double lam, int passes,
              double* T, double* V, int64_t ldv, double* coef_ws, double* out) {
  Prof pr(c, TAG_MISC);
  double2* coef = reinterpret_cast<double2*>(coef_ws);
  if (m > 0)
    k_theta_coefs<<<grid_for(m), 256, 0, c->stream>>>(m, S, lds, Sxx, ldx, xmap, Sxy, ldxy, Th->colptr, Th->rowidx,
                                                      static_cast<const double*>(Th->val), Tr, Tc, coef, T);
  k_theta_cd<<<1, CD_NT, 0, c->stream>>>(p, q, S, lds, Sxx, ldx, xmap, Tr, Tc, coef, m, lam, passes, T, V, ldv, out);
  c->launches += m > 0 ? 1 : 0;
  post_launch(c, "k_theta_cd");
}

namespace {
__global__ void k_row_flags(int64_t m, const int32_t* __restrict__ Tr, int32_t* flags) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < m; k += (int64_t)gridDim.x * blockDim.x)
    flags[Tr[k]] = 1;
}

// one block: exclusive scan of the flags in 1024-entry rounds (warp shuffles), ascending row order
__global__ void __launch_bounds__(1024) k_row_map_scan(int p, int32_t* xmap, int32_t* rows, long long* count) {
  __shared__ int wsum[32];
  __shared__ long long base;
  if (threadIdx.x == 0) base = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int i0 = 0; i0 < p; i0 += 1024) {
    const int i = i0 + threadIdx.x;
    const int f = (i < p && xmap[i]) ? 1 : 0;
    int x = f;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    if (w == 0) {
      int v = wsum[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
      }
      wsum[lane] = v;
    }
    __syncthreads();
    const long long pos = base + (w > 0 ? wsum[w - 1] : 0) + x - f;
    if (i < p) {
      xmap[i] = f ? (int32_t)pos : -1;
      if (f) rows[pos] = i;
    }
    __syncthreads();
    if (threadIdx.x == 0) base += wsum[31];
    __syncthreads();
  }
  if (threadIdx.x == 0) *count = base;
}

__global__ void k_gather_cols(int64_t n, int64_t k, const double* __restrict__ X, int64_t ldx,
                              const int32_t* __restrict__ rows, double* __restrict__ G, int64_t ldg) {
  const int64_t c = blockIdx.y;
  const double* src = X + (int64_t)rows[c] * ldx;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    G[i + c * ldg] = src[i];
}
}  // namespace

void row_map(Ctx* c, int p, const int32_t* T_row, int64_t m, int32_t* xmap, int32_t* rows, long long* count_dev) {
  Prof pr(c, TAG_MISC);
  CGGM_CUDA_CHECK(cudaMemsetAsync(xmap, 0, sizeof(int32_t) * (size_t)p, c->stream));
  if (m > 0) k_row_flags<<<grid_for(m), 256, 0, c->stream>>>(m, T_row, xmap);
  k_row_map_scan<<<1, 1024, 0, c->stream>>>(p, xmap, rows, count_dev);
  c->launches += m > 0 ? 1 : 0;
  post_launch(c, "k_row_map_scan");
}

void gather_cols(Ctx* c, int64_t n, int64_t k, const double* X, int64_t ldx, const int32_t* rows, double* G,
                 int64_t ldg) {
  if (n == 0 || k == 0) return;
  Prof pr(c, TAG_MISC);
  dim3 grid((unsigned)std::min<int64_t>((n + 255) / 256, 8), (unsigned)k);
  k_gather_cols<<<grid, 256, 0, c->stream>>>(n, k, X, ldx, rows, G, ldg);
  post_launch(c, "k_gather_cols");
}

// list column pointers lp (n+1) of a column-major list: counts + scan (cnt: n ints, scr: n+1 int64)
static void list_colptr(Ctx* c, int n, const int32_t* r, const int32_t* cidx, int64_t m, int* cnt, int64_t* scr,
                        int64_t* lp) {
  CGGM_CUDA_CHECK(cudaMemsetAsync(cnt, 0, sizeof(int) * (size_t)n, c->stream));
  k_list_counts<<<grid_for(m), 256, 0, c->stream>>>(m, r, cidx, 0, cnt, nullptr);
  k_list_scan<<<1, 1024, 0, c->stream>>>(n, cnt, nullptr, lp, scr, nullptr);
  c->launches += 2;
}

bool coop_ok(Ctx* c) {
  static int ok = -1;
  if (ok < 0) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrCooperativeLaunch, c->device);
    ok = v;
  }
  return ok && c->cd_coop;
}

// ws: cnt (q ints), scr (q+1 int64), lp (q+1 int64), dmu (m), colbuf (2q or p doubles)
void lambda_cd_coop(Ctx* c, int q, const double* S, int64_t lds, const double* P, int64_t ldp, const double* G,
                    int64_t ldg, const cggm_csc* Lam, const int32_t* Lr, const int32_t* Lc, int64_t m, double lam,
                    int penalize_diag, int passes, double* D, double* U, double* Z, int64_t ldu, double* coef_ws,
                    int* cnt, int64_t* scr, int64_t* lp, double* dmu, double* colbuf, double* out) {
  Prof pr(c, TAG_MISC);
  double4* coef = reinterpret_cast<double4*>(coef_ws);
  const double* lv = static_cast<const double*>(Lam->val);
  CGGM_CUDA_CHECK(cudaMemsetAsync(D, 0, sizeof(double) * (size_t)std::max<int64_t>(m, 1), c->stream));
  if (m > 0) {
    k_lambda_coefs<<<grid_for(m), 256, 0, c->stream>>>(m, S, lds, P, ldp, G, ldg, Lam->colptr, Lam->rowidx, lv, Lr, Lc,
                                                       lam, penalize_diag, coef);
    list_colptr(c, q, Lr, Lc, m, cnt, scr, lp);
    if (c->cd_block == 1 || (c->cd_block < 0 && q > CO_QMAX)) {
      const int nch = (q + BK_CH - 1) / BK_CH;
      double* part = static_cast<double*>(ws_get(c, WS_CD_BLK, ((size_t)BK_B * nch + BK_B * BK_B + 2 * BK_B) * 8));
      double* Ct = part + (size_t)BK_B * nch;
      double* sjw = Ct + BK_B * BK_B;
      CGGM_ONCE_PER_DEVICE({
        CGGM_CUDA_CHECK(cudaFuncSetAttribute(k_sweep_blk<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)BK_SMEM));
      });
      int grid = c->num_sms, nlen = q;
      const int32_t* xm = nullptr;
      double lamv = 0.0;
      const double* cfd = coef_ws;
      // panel (left-looking) mode, CGGM_CD_PANEL = w > 0 (default above the register limits): the
      // q x q workspace U holds the dense symmetric D instead of U = D Sigma; before the columns
      // J = [j0, j0 + w) are swept, their part of U^T and Z^T is formed from it by two DMMA products
      // (PU = Sigma_{J,:} D, PZ = Psi_{J,:} D, w x q, in the Z workspace), so the deferred row
      // updates touch only the panel's later columns instead of all q (see k_sweep_blk)
      const int w = c->cd_panel >= 0 ? c->cd_panel : (q > CO_QMAX ? 512 : 0);
      static const int timing = [] { const char* e = std::getenv("CGGM_CD_TIMING"); return e ? std::atoi(e) : 0; }();
      if (timing) {
        unsigned long long z[8] = {0};
        CGGM_CUDA_CHECK(cudaMemcpyToSymbolAsync(g_cd_tim, z, sizeof(z), 0, cudaMemcpyHostToDevice, c->stream));
        CGGM_CUDA_CHECK(cudaMemcpyToSymbolAsync(g_cd_tim_on, &timing, sizeof(int), 0, cudaMemcpyHostToDevice, c->stream));
        CGGM_CUDA_CHECK(cudaStreamSynchronize(c->stream));
      }
      if (w > 0 && w % 2 == 0 && (size_t)2 * w <= (size_t)ldu) {
        double* Dd = U;
        int64_t ldd = ldu;
        const int64_t ldw = w;
        double* PU = Z;
        double* PZ = Z + (size_t)ldw * q;
        double* rpart = static_cast<double*>(ws_get(c, WS_CD_PANEL, (size_t)2 * w * nch * 8));
        int one = 1;
        for (int pass = 0; pass < passes; ++pass) {
          for (int j0 = 0; j0 < q; j0 += w) {
            int j1 = std::min(q, j0 + w);
            if (pass == 0 && j0 == 0) {   // D = 0
              CGGM_CUDA_CHECK(cudaMemsetAsync(PU, 0, (size_t)2 * ldw * q * 8, c->stream));
            } else {
              Epilogue eu, ez;
              eu.out1 = PU; eu.ld1 = ldw;
              ez.out1 = PZ; ez.ld1 = ldw;
              gemm(c, true, false, j1 - j0, q, q, S + (int64_t)j0 * lds, lds, Dd, ldd, eu, 0);
              gemm(c, true, false, j1 - j0, q, q, P + (int64_t)j0 * ldp, ldp, Dd, ldd, ez, 0);
            }
            double* Uo = PU - j0;
            double* Zo = PZ - j0;
            int64_t ldp2 = ldw;
            void* args[] = {&q, &nlen, &S, &lds, &P, &ldp, &xm, &Lr, &cfd, &lp, &lamv, &one, &D, &dmu, &Uo, &Zo, &ldp2,
                            &colbuf, &part, &Ct, &sjw, &j0, &j1, &Dd, &ldd, &rpart};
            CGGM_CUDA_CHECK(cudaLaunchCooperativeKernel((const void*)k_sweep_blk<true>, dim3(grid), dim3(CO_NT), args,
                                                        BK_SMEM, c->stream));
            c->launches += 1;
          }
        }
      } else {
        int j0 = 0, j1 = q;
        double* Dn = nullptr;
        int64_t ldd = 0;
        void* args[] = {&q, &nlen, &S, &lds, &P, &ldp, &xm, &Lr, &cfd, &lp, &lamv, &passes, &D, &dmu, &U, &Z, &ldu,
                        &colbuf, &part, &Ct, &sjw, &j0, &j1, &Dn, &ldd, &Dn};
        CGGM_CUDA_CHECK(cudaLaunchCooperativeKernel((const void*)k_sweep_blk<true>, dim3(grid), dim3(CO_NT), args, BK_SMEM,
                                                    c->stream));
      }
      c->launches += 2;
      if (timing) {
        unsigned long long t[8];
        CGGM_CUDA_CHECK(cudaStreamSynchronize(c->stream));
        CGGM_CUDA_CHECK(cudaMemcpyFromSymbol(t, g_cd_tim, sizeof(t)));
        std::fprintf(stderr, "CDTIMING lambda m=%lld panel=%d ms: column_start=%.2f phase1=%.2f stage=%.2f chain=%.2f column_end=%.2f\n",
                     (long long)m, w, t[0] * 1e-6, t[1] * 1e-6, t[2] * 1e-6, t[3] * 1e-6, t[4] * 1e-6);
      }
      k_lambda_tail<<<1, CD_NT, 0, c->stream>>>(q, Lam->colptr, lv, Lr, Lc, coef, m, D, out);
      post_launch(c, "k_sweep_blk<lambda>");
      return;
    }
    const size_t smem_pf = (size_t)4 * ((q + 1) & ~1) * 8;
    if (q >= 2048 && q <= CO_QMAX && smem_pf <= 200 * 1024 && lds % 2 == 0 && ldp % 2 == 0 && c->cd_prefetch) {
      CGGM_ONCE_PER_DEVICE({
        CGGM_CUDA_CHECK(cudaFuncSetAttribute(k_lambda_sweep_pf, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      });
      int grid = c->num_sms;
      void* args[] = {&q, &S, &lds, &P, &ldp, &Lr, &coef, &lp, &passes, &D, &dmu, &U, &Z, &ldu};
      CGGM_CUDA_CHECK(cudaLaunchCooperativeKernel((const void*)k_lambda_sweep_pf, dim3(grid), dim3(CO_NT), args, smem_pf,
                                                  c->stream));
      c->launches += 2;
      k_lambda_tail<<<1, CD_NT, 0, c->stream>>>(q, Lam->colptr, lv, Lr, Lc, coef, m, D, out);
      post_launch(c, "k_lambda_sweep_pf");
      return;
    }
    const size_t smem = (size_t)2 * q * 8;
    const int use_smem = smem <= 200 * 1024 ? 1 : 0;
    CGGM_ONCE_PER_DEVICE({
      CGGM_CUDA_CHECK(cudaFuncSetAttribute(k_lambda_sweep_coop, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    });
    int grid = c->num_sms;
    void* args[] = {&q, &S, &lds, &P, &ldp, &Lr, &coef, &lp, &passes, &D, &dmu, &U, &Z, &ldu, &colbuf,
                    const_cast<int*>(&use_smem)};
    CGGM_CUDA_CHECK(cudaLaunchCooperativeKernel((const void*)k_lambda_sweep_coop, dim3(grid), dim3(CO_NT), args,
                                                use_smem ? smem : 0, c->stream));
    c->launches += 2;
  }
  k_lambda_tail<<<1, CD_NT, 0, c->stream>>>(q, Lam->colptr, lv, Lr, Lc, coef, m, D, out);
  post_launch(c, "k_lambda_sweep_coop");
}

void theta_cd_coop(Ctx* c, int p, int q, const double* S, int64_t lds, const double* Sxx, int64_t ldx,
                   const int32_t* xmap, const double* Sxy, int64_t ldxy, const cggm_csc* Th, const int32_t* Tr, const int32_t* Tc, int64_t m,
                   double lam, int passes, double* T, double* V, int64_t ldv, double* coef_ws, int* cnt, int64_t* scr,
                   int64_t* lp, double* dmu, double* colbuf, double* out) {
  Prof pr(c, TAG_MISC);
  double2* coef = reinterpret_cast<double2*>(coef_ws);
  // V = Theta Sigma, row-major
  k_theta_sigma_rm<<<(q + 7) / 8, 256, 0, c->stream>>>(q, Th->colptr, Th->rowidx, static_cast<const double*>(Th->val),
                                                       S, lds, V, ldv);
  if (m > 0) {
    k_theta_coefs<<<grid_for(m), 256, 0, c->stream>>>(m, S, lds, Sxx, ldx, xmap, Sxy, ldxy, Th->colptr, Th->rowidx,
                                                      static_cast<const double*>(Th->val), Tr, Tc, coef, T);
    list_colptr(c, q, Tr, Tc, m, cnt, scr, lp);
    int grid = c->num_sms;
    if (c->cd_block == 1 || (c->cd_block < 0 && p > CO_PMAX)) {
      const int nch = (p + BK_CH - 1) / BK_CH;
      double* part = static_cast<double*>(ws_get(c, WS_CD_BLK, ((size_t)BK_B * nch + BK_B * BK_B + 2 * BK_B) * 8));
      double* Ct = part + (size_t)BK_B * nch;
      double* sjw = Ct + BK_B * BK_B;
      CGGM_ONCE_PER_DEVICE({
        CGGM_CUDA_CHECK(cudaFuncSetAttribute(k_sweep_blk<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)BK_SMEM));
      });
      int nlen = p;
      const double* cfd = coef_ws;
      double* Zn = nullptr;
      int j0 = 0, j1 = q;
      int64_t ldd = 0;
      void* args[] = {&q, &nlen, &S, &lds, &Sxx, &ldx, &xmap, &Tr, &cfd, &lp, &lam, &passes, &T, &dmu, &V, &Zn, &ldv,
                      &colbuf, &part, &Ct, &sjw, &j0, &j1, &Zn, &ldd, &Zn};
      CGGM_CUDA_CHECK(cudaLaunchCooperativeKernel((const void*)k_sweep_blk<false>, dim3(grid), dim3(CO_NT), args, BK_SMEM,
                                                  c->stream));
      c->launches += 2;
      k_theta_l1<<<1, CD_NT, 0, c->stream>>>(T, m, out);
      post_launch(c, "k_sweep_blk<theta>");
      return;
    }
    const size_t smem_pf = (size_t)2 * ((p + 1) & ~1) * 8;
    if (p >= 2048 && p <= CO_PMAX && smem_pf <= 200 * 1024 && ldx % 2 == 0 && c->cd_prefetch) {
      CGGM_ONCE_PER_DEVICE({
        CGGM_CUDA_CHECK(cudaFuncSetAttribute(k_theta_sweep_pf, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      });
      void* args[] = {&p, &q, &S, &lds, &Sxx, &ldx, &xmap, &Tr, &coef, &lp, &lam, &passes, &T, &dmu, &V, &ldv};
      CGGM_CUDA_CHECK(cudaLaunchCooperativeKernel((const void*)k_theta_sweep_pf, dim3(grid), dim3(CO_NT), args, smem_pf,
                                                  c->stream));
      c->launches += 2;
      k_theta_l1<<<1, CD_NT, 0, c->stream>>>(T, m, out);
      post_launch(c, "k_theta_sweep_pf");
      return;
    }
    const size_t smem = (size_t)p * 8;
    const int use_smem = smem <= 200 * 1024 ? 1 : 0;
    CGGM_ONCE_PER_DEVICE({
      CGGM_CUDA_CHECK(cudaFuncSetAttribute(k_theta_sweep_coop, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    });
    void* args[] = {&p, &q, &S, &lds, &Sxx, &ldx, &xmap, &Tr, &coef, &lp, &lam, &passes, &T, &dmu, &V, &ldv, &colbuf,
                    const_cast<int*>(&use_smem)};
    CGGM_CUDA_CHECK(cudaLaunchCooperativeKernel((const void*)k_theta_sweep_coop, dim3(grid), dim3(CO_NT), args,
                                                use_smem ? smem : 0, c->stream));
    c->launches += 2;
  }
  {
    double* o = out;
    // ||Theta_new||_1 by the single-CTA tail of the Theta kernel family
    k_theta_l1<<<1, CD_NT, 0, c->stream>>>(T, m, o);
  }
  post_launch(c, "k_theta_sweep_coop");
}

// workspace: ints[2n] counts, int64[3(n+1)] scans
void list_to_csc(Ctx* c, int n, const int32_t* r, const int32_t* cidx, int64_t m, bool mirror, const cggm_csc* base,
                 const double* D, double alpha, const double* vals, int64_t* out_colptr, int32_t* out_row,
                 double* out_val, int* cnt_ws, int64_t* scan_ws) {
  int* cl = cnt_ws;
  int* cm = cnt_ws + n;
  int* mfill = cnt_ws + 2 * n;
  int64_t* lp = scan_ws;
  int64_t* mb = scan_ws + (n + 1);
  CGGM_CUDA_CHECK(cudaMemsetAsync(cnt_ws, 0, sizeof(int) * 3 * (size_t)n, c->stream));
  Prof pr(c, TAG_MISC);
  k_list_counts<<<grid_for(m), 256, 0, c->stream>>>(m, r, cidx, mirror ? 1 : 0, cl, cm);
  k_list_scan<<<1, 1024, 0, c->stream>>>(n, cl, mirror ? cm : nullptr, lp, out_colptr, mirror ? mb : nullptr);
  if (mirror) {
    k_lambda_trial_scatter<<<grid_for(m), 256, 0, c->stream>>>(m, r, cidx, D, alpha, base->colptr, base->rowidx,
                                                              static_cast<const double*>(base->val), lp, out_colptr, out_row,
                                                              out_val);
    k_mirror_place<<<1, 1024, 0, c->stream>>>(n, r, lp, out_colptr, mb, mfill, out_row, out_val);
  } else {
    k_copy_list<<<grid_for(m), 256, 0, c->stream>>>(m, r, vals, out_row, out_val);
  }
  c->launches += mirror ? 3 : 2;
  post_launch(c, "list_to_csc");
}

}  // namespace cggm
