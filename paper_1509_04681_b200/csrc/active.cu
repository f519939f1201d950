// Active sets S_Lambda, S_Theta (§2.2) and the minimum-norm-subgradient stopping
// statistic (§5.1), as ordered, deterministic stream compaction:
//   1. count pass: one CTA per column; the column's stored nonzeros are set in a shared-memory
//      bitmask (value test, reading A7), the dense gradient column is scanned coalesced, and the
//      CTA writes (count, tie count, subgradient partial) for the column;
//   2. one-CTA exclusive scan of the counts -> per-column offsets + totals (fixed-order sums);
//   3. write pass: the same flags, block prefix sums via warp ballots, (row, col) written at the
//      column's offset -> ascending column-major order, identical run to run.
// Lambda: only i <= j is listed (reading A6); the subgradient covers both triangles using the
// exact symmetry of grad_Lambda (weight 2 for i < j) plus an exact per-stored-entry correction
// |g + lam sign(x)| - max(|g| - lam, 0) for nonzero x.
#include "kernels.cuh"

namespace cggm {
namespace {

constexpr int NT = 256;

template <bool LAM>
__device__ __forceinline__ double lam_of(int64_t i, int64_t j, double lam, int penalize_diag) {
  return (LAM && i == j && !penalize_diag) ? 0.0 : lam;
}

template <bool LAM>
__device__ void build_bits(uint32_t* bits, int64_t nwords, const int64_t* colptr, const int32_t* rowidx,
                           const double* val, int64_t j, int64_t scan_rows) {
  for (int64_t w = threadIdx.x; w < nwords; w += NT) bits[w] = 0u;
  __syncthreads();
  for (int64_t t = colptr[j] + threadIdx.x; t < colptr[j + 1]; t += NT) {
    const int32_t r = rowidx[t];
    if (r < scan_rows && val[t] != 0.0) atomicOr(&bits[r >> 5], 1u << (r & 31));
  }
  __syncthreads();
}

template <bool LAM>
__global__ void __launch_bounds__(NT) k_active_count(int64_t nrows, const double* __restrict__ G, int64_t ldg,
                                                     const int64_t* colptr, const int32_t* rowidx, const double* val,
                                                     double lam, int penalize_diag, double tie_eps, long long* cnt,
                                                     long long* ties, double* sub) {
  extern __shared__ uint32_t bits[];
  __shared__ double shd[NT];
  __shared__ long long shc[NT], sht[NT];
  const int64_t j = blockIdx.x;
  const int64_t scan_rows = LAM ? j + 1 : nrows;
  const int64_t nwords = (scan_rows + 31) >> 5;
  build_bits<LAM>(bits, nwords, colptr, rowidx, val, j, scan_rows);
  long long c = 0, tc = 0;
  double s = 0.0;
  const double* gc = G + j * ldg;
  for (int64_t i = threadIdx.x; i < scan_rows; i += NT) {
    const double a = fabs(gc[i]);
    const double lm = lam_of<LAM>(i, j, lam, penalize_diag);
    const bool sup = (bits[i >> 5] >> (i & 31)) & 1u;
    c += (a > lm || sup) ? 1 : 0;
    tc += (!sup && fabs(a - lm) <= tie_eps) ? 1 : 0;
    const double w = (LAM && i < j) ? 2.0 : 1.0;
    s += w * fmax(a - lm, 0.0);
  }
  // exact correction for stored nonzeros (all rows of the column)
  for (int64_t t = colptr[j] + threadIdx.x; t < colptr[j + 1]; t += NT) {
    const double x = val[t];
    if (x == 0.0) continue;
    const int64_t i = rowidx[t];
    const double g = gc[i];
    const double lm = lam_of<LAM>(i, j, lam, penalize_diag);
    s += fabs(g + lm * (x > 0.0 ? 1.0 : -1.0)) - fmax(fabs(g) - lm, 0.0);
  }
  shd[threadIdx.x] = s;
  shc[threadIdx.x] = c;
  sht[threadIdx.x] = tc;
  __syncthreads();
  for (int st = NT / 2; st > 0; st >>= 1) {
    if (threadIdx.x < st) {
      shd[threadIdx.x] += shd[threadIdx.x + st];
      shc[threadIdx.x] += shc[threadIdx.x + st];
      sht[threadIdx.x] += sht[threadIdx.x + st];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    cnt[j] = shc[0];
    ties[j] = sht[0];
    sub[j] = shd[0];
  }
}

// single CTA: exclusive scan of cnt -> off, totals (fixed-order sums)
constexpr int SCAN_NT = 1024;
__global__ void __launch_bounds__(SCAN_NT) k_active_scan(int64_t ncols, const long long* cnt, const long long* ties,
                                                         const double* sub, long long* off, long long* tot_m,
                                                         long long* tot_ties, double* tot_sub) {
  __shared__ long long sc[SCAN_NT], st[SCAN_NT];
  __shared__ double sd[SCAN_NT];
  const int64_t per = (ncols + SCAN_NT - 1) / SCAN_NT;
  const int64_t b = threadIdx.x * per, e = min(ncols, b + per);
  long long c = 0, tsum = 0;
  double d = 0.0;
  for (int64_t i = b; i < e; ++i) {
    c += cnt[i];
    tsum += ties[i];
    d += sub[i];
  }
  sc[threadIdx.x] = c;
  st[threadIdx.x] = tsum;
  sd[threadIdx.x] = d;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long run = 0, tt = 0;
    double dd = 0.0;
    for (int k = 0; k < SCAN_NT; ++k) {
      const long long v = sc[k];
      sc[k] = run;
      run += v;
      tt += st[k];
      dd += sd[k];
    }
    *tot_m = run;
    *tot_ties = tt;
    *tot_sub = dd;
  }
  __syncthreads();
  long long run = sc[threadIdx.x];
  for (int64_t i = b; i < e; ++i) {
    off[i] = run;
    run += cnt[i];
  }
}

template <bool LAM>
__global__ void __launch_bounds__(NT) k_active_write(int64_t nrows, const double* __restrict__ G, int64_t ldg,
                                                     const int64_t* colptr, const int32_t* rowidx, const double* val,
                                                     double lam, int penalize_diag, const long long* off,
                                                     int32_t* out_row, int32_t* out_col, const long long* total,
                                                     long long cap) {
  if (*total > cap) return;  // capacity exceeded: write nothing (reported as CGGM_ERR_CAPACITY)
  extern __shared__ uint32_t bits[];
  __shared__ int warp_tot[NT / 32];
  __shared__ long long base_sh;
  const int64_t j = blockIdx.x;
  const int64_t scan_rows = LAM ? j + 1 : nrows;
  const int64_t nwords = (scan_rows + 31) >> 5;
  build_bits<LAM>(bits, nwords, colptr, rowidx, val, j, scan_rows);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double* gc = G + j * ldg;
  long long base = off[j];
  for (int64_t r0 = 0; r0 < scan_rows; r0 += NT) {
    const int64_t i = r0 + threadIdx.x;
    bool f = false;
    if (i < scan_rows) {
      const double a = fabs(gc[i]);
      const double lm = lam_of<LAM>(i, j, lam, penalize_diag);
      const bool sup = (bits[i >> 5] >> (i & 31)) & 1u;
      f = (a > lm) || sup;
    }
    const unsigned m = __ballot_sync(0xffffffffu, f);
    if (lane == 0) warp_tot[warp] = __popc(m);
    __syncthreads();
    int before = 0, total = 0;
    for (int w = 0; w < NT / 32; ++w) {
      if (w < warp) before += warp_tot[w];
      total += warp_tot[w];
    }
    if (f) {
      const long long pos = base + before + __popc(m & ((1u << lane) - 1u));
      out_row[pos] = (int32_t)i;
      out_col[pos] = (int32_t)j;
    }
    base += total;
    __syncthreads();
  }
  (void)base_sh;
}

size_t bits_bytes(int64_t rows) { return (size_t)((rows + 31) / 32) * 4; }

template <typename K>
void set_smem(K kernel, size_t bytes) {
  if (bytes > 48 * 1024)
    CGGM_CUDA_CHECK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
}

}  // namespace

void active_count(Ctx* c, int64_t p, int64_t q, const double* GradL, int64_t ldgl, const double* GradT, int64_t ldgt,
                  const cggm_csc* Lambda, const cggm_csc* Theta, double lam_L, double lam_T, int penalize_diag,
                  double tie_eps, ActTotals* T, long long* offL, long long* offT, long long* cntL, long long* cntT,
                  long long* tieL, long long* tieT, double* subL, double* subT) {
  if (q == 0) return;
  size_t bl = bits_bytes(q), bt = bits_bytes(p);
  set_smem(k_active_count<true>, bl);
  set_smem(k_active_count<false>, bt);
  { Prof pr(c, TAG_ACTIVE);
  k_active_count<true><<<(unsigned)q, NT, bl, c->stream>>>(q, GradL, ldgl, Lambda->colptr, Lambda->rowidx,
                                                          static_cast<const double*>(Lambda->val), lam_L,
                                                          penalize_diag, tie_eps, cntL, tieL, subL);
  post_launch(c, "k_active_count<L>"); }
  { Prof pr(c, TAG_ACTIVE);
  k_active_count<false><<<(unsigned)q, NT, bt, c->stream>>>(p, GradT, ldgt, Theta->colptr, Theta->rowidx,
                                                           static_cast<const double*>(Theta->val), lam_T, 1, tie_eps,
                                                           cntT, tieT, subT);
  post_launch(c, "k_active_count<T>"); }
  { Prof pr(c, TAG_ACTIVE);
  k_active_scan<<<1, SCAN_NT, 0, c->stream>>>(q, cntL, tieL, subL, offL, &T->m_L, &T->ties_L, &T->sub_L);
  post_launch(c, "k_active_scan<L>"); }
  { Prof pr(c, TAG_ACTIVE);
  k_active_scan<<<1, SCAN_NT, 0, c->stream>>>(q, cntT, tieT, subT, offT, &T->m_T, &T->ties_T, &T->sub_T);
  post_launch(c, "k_active_scan<T>"); }
}

void active_write(Ctx* c, int64_t p, int64_t q, const double* GradL, int64_t ldgl, const double* GradT, int64_t ldgt,
                  const cggm_csc* Lambda, const cggm_csc* Theta, double lam_L, double lam_T, int penalize_diag,
                  const long long* offL, const long long* offT, int32_t* L_row, int32_t* L_col, int32_t* T_row,
                  int32_t* T_col, const ActTotals* totals, long long capL, long long capT) {
  if (q == 0) return;
  size_t bl = bits_bytes(q), bt = bits_bytes(p);
  set_smem(k_active_write<true>, bl);
  set_smem(k_active_write<false>, bt);
  { Prof pr(c, TAG_ACTIVE);
  k_active_write<true><<<(unsigned)q, NT, bl, c->stream>>>(q, GradL, ldgl, Lambda->colptr, Lambda->rowidx,
                                                          static_cast<const double*>(Lambda->val), lam_L,
                                                          penalize_diag, offL, L_row, L_col, &totals->m_L, capL);
  post_launch(c, "k_active_write<L>"); }
  { Prof pr(c, TAG_ACTIVE);
  k_active_write<false><<<(unsigned)q, NT, bt, c->stream>>>(p, GradT, ldgt, Theta->colptr, Theta->rowidx,
                                                           static_cast<const double*>(Theta->val), lam_T, 1, offT,
                                                           T_row, T_col, &totals->m_T, capT);
  post_launch(c, "k_active_write<T>"); }
}

}  // namespace cggm
