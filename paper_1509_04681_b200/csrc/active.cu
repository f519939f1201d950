// Active sets S_Lambda, S_Theta (§2.2) and the minimum-norm-subgradient stopping
// statistic (§5.1) as a SINGLE-PASS ordered stream compaction:
// one CTA per column j (columns are dispatched in order), 8 warps each scanning a contiguous
// 32-aligned segment of the column with 4 loads in flight per lane:
//   1. the column's stored nonzeros are set in a shared-memory support bitmask (value test,
//      reading A7);
//   2. each 32-row chunk's flags (|g| > lam or support) are kept as one ballot word in shared
//      memory; tie count and subgradient partial accumulate in registers;
//   3. the column offset comes from a decoupled look-back over the preceding columns' published
//      (aggregate | inclusive prefix) states -- no second pass over the gradient;
//   4. each warp writes (row, col) for its set bits from the shared bitmask -> ascending
//      column-major order, identical run to run.
// A final one-CTA kernel sums the per-column tie counts and subgradient partials in fixed order.
// Lambda: only i <= j is listed (reading A6); the subgradient covers both triangles using the
// exact symmetry of grad_Lambda (weight 2 for i < j) plus an exact per-stored-entry correction
// |g + lam sign(x)| - max(|g| - lam, 0) for nonzero x.  HBM bytes per call: one read of the
// upper triangle of grad_Lambda and of grad_Theta, 8 bytes written per active entry.
#include "kernels.cuh"

namespace cggm {
namespace {

constexpr int NT = 256;
constexpr int NW = NT / 32;   // warp segments per column
constexpr int UNR = 4;        // 32-row chunks in flight per lane
constexpr unsigned long long ST_AGG = 1ull << 62, ST_INC = 2ull << 62, ST_VAL = (1ull << 62) - 1;

template <bool LAM, typename T>
__device__ __forceinline__ T lam_of(int64_t i, int64_t j, T lam, int penalize_diag) {
  return (LAM && i == j && !penalize_diag) ? T(0) : lam;
}

// contiguous, 32-aligned segment of warp w among NW for a column of `rows` rows
__device__ __forceinline__ void segment(int64_t rows, int w, int64_t& a, int64_t& b) {
  const int64_t chunks = (rows + 31) >> 5;
  const int64_t per = (chunks + NW - 1) / NW;
  a = min(rows, (int64_t)w * per * 32);
  b = min(rows, (int64_t)(w + 1) * per * 32);
}

__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <bool LAM, typename T>
__global__ void __launch_bounds__(NT) k_active_onepass(int64_t nrows, const T* __restrict__ G, int64_t ldg,
                                                       const int64_t* colptr, const int32_t* rowidx, const T* val,
                                                       T lam, int penalize_diag, T tie_eps,
                                                       unsigned long long* state, int32_t* out_row,
                                                       int32_t* out_col, long long cap, long long* ties_col,
                                                       double* sub_col, int64_t col0) {
  extern __shared__ uint32_t sm[];
  const int64_t j = col0 + blockIdx.x;   // G holds columns col0 .. (a chunk of the gradient)
  const int64_t scan_rows = LAM ? j + 1 : nrows;
  const int64_t nwords = (scan_rows + 31) >> 5;
  uint32_t* sup_bits = sm;
  uint32_t* flag_bits = sm + nwords;
  __shared__ int wcnt[NW];
  __shared__ double wsub[NW];
  __shared__ long long wtie[NW];
  __shared__ long long col_base;
  for (int64_t w = threadIdx.x; w < nwords; w += NT) sup_bits[w] = 0u;
  __syncthreads();
  for (int64_t t = colptr[j] + threadIdx.x; t < colptr[j + 1]; t += NT) {
    const int32_t r = rowidx[t];
    if (r < scan_rows && val[t] != T(0)) atomicOr(&sup_bits[r >> 5], 1u << (r & 31));
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int64_t a, b;
  segment(scan_rows, w, a, b);
  const T* gc = G + (j - col0) * ldg;
  int cnt = 0;
  long long tc = 0;
  double s = 0.0;
  const int ib = (int)b;
  const int jj = (int)j;
  for (int r0 = (int)a; r0 < ib; r0 += 32 * UNR) {
    T g[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int i = r0 + u * 32 + lane;
      g[u] = (i < ib) ? __ldcs(gc + i) : T(0);   // streamed once: evict-first
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int c0 = r0 + u * 32;
      if (c0 >= ib) break;   // warp-uniform
      const int i = c0 + lane;
      const bool in = i < ib;
      const unsigned supw = sup_bits[c0 >> 5];   // one broadcast word per 32-row chunk
      const bool sup = (supw >> lane) & 1u;
      const T lm = (LAM && i == jj && !penalize_diag) ? T(0) : lam;
      const T av = fabs(g[u]);
      const T d = av - lm;
      const bool f = in && (d > T(0) || sup);
      const unsigned m = __ballot_sync(0xffffffffu, f);
      if (lane == 0) flag_bits[c0 >> 5] = m;
      cnt += __popc(m);
      tc += (in && !sup && fabs(d) <= tie_eps) ? 1 : 0;
      if (in) s += (LAM && i < jj) ? 2.0 * (double)fmax(d, T(0)) : (double)fmax(d, T(0));
    }
  }
  for (int64_t t = colptr[j] + threadIdx.x; t < colptr[j + 1]; t += NT) {
    const T x = val[t];
    if (x == T(0)) continue;
    const int64_t i = rowidx[t];
    const T gv = gc[i];
    const T lm = lam_of<LAM>(i, j, lam, penalize_diag);
    s += (double)fabs(gv + lm * (x > T(0) ? T(1) : T(-1))) - (double)fmax(fabs(gv) - lm, T(0));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s += __shfl_down_sync(0xffffffffu, s, o);
    tc += __shfl_down_sync(0xffffffffu, tc, o);
  }
  if (lane == 0) {
    wcnt[w] = cnt;
    wsub[w] = s;
    wtie[w] = tc;
  }
  __syncthreads();
  if (w == 0) {
    long long total = 0, tt = 0;
    double ss = 0.0;
    for (int k = 0; k < NW; ++k) {
      total += wcnt[k];
      tt += wtie[k];
      ss += wsub[k];
    }
    if (lane == 0) {
      sub_col[j] = ss;
      ties_col[j] = tt;
      st_release(&state[j], (j == 0 ? ST_INC : ST_AGG) | (unsigned long long)total);
    }
    // decoupled look-back, one warp: lane l inspects predecessor j-1-l of the current window
    long long excl = 0;
    int64_t k0 = j - 1;
    while (k0 >= 0) {
      const int64_t k = k0 - lane;
      unsigned long long v = (k >= 0) ? ld_acquire(&state[k]) : ST_INC;   // before column 0: prefix 0
      while (__any_sync(0xffffffffu, (v & ~ST_VAL) == 0)) {
        if ((v & ~ST_VAL) == 0) v = ld_acquire(&state[k]);
      }
      const unsigned inc = __ballot_sync(0xffffffffu, (v & ~ST_VAL) == ST_INC);
      const int stop = inc ? __ffs(inc) - 1 : 31;          // nearest inclusive predecessor
      long long add = (lane <= stop && k >= 0) ? (long long)(v & ST_VAL) : 0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) add += __shfl_xor_sync(0xffffffffu, add, o);
      excl += add;
      if (inc) break;
      k0 -= 32;
    }
    if (lane == 0) {
      if (j > 0) st_release(&state[j], ST_INC | (unsigned long long)(excl + total));
      col_base = excl;
    }
  }
  __syncthreads();
  long long pos = col_base;
  for (int k = 0; k < w; ++k) pos += wcnt[k];
  const unsigned below = (1u << lane) - 1u;
  for (int64_t r0 = a; r0 < b; r0 += 32) {
    const unsigned m = flag_bits[r0 >> 5];
    if (m & (1u << lane)) {
      const long long p = pos + __popc(m & below);
      if (p < cap) {
        out_row[p] = (int32_t)(r0 + lane);
        out_col[p] = (int32_t)j;
      }
    }
    pos += __popc(m);
  }
}

// totals: m from the last column's inclusive state, ties / subgradient summed in fixed order
constexpr int TOT_NT = 1024;
__global__ void __launch_bounds__(TOT_NT) k_active_totals(int64_t ncols, const unsigned long long* state,
                                                          const long long* ties_col, const double* sub_col,
                                                          long long* tot_m, long long* tot_ties, double* tot_sub) {
  __shared__ long long st[TOT_NT];
  __shared__ double sd[TOT_NT];
  const int64_t per = (ncols + TOT_NT - 1) / TOT_NT;
  const int64_t b = threadIdx.x * per, e = min(ncols, b + per);
  long long t = 0;
  double d = 0.0;
  for (int64_t i = b; i < e; ++i) {
    t += ties_col[i];
    d += sub_col[i];
  }
  st[threadIdx.x] = t;
  sd[threadIdx.x] = d;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long tt = 0;
    double dd = 0.0;
    for (int k = 0; k < TOT_NT; ++k) {
      tt += st[k];
      dd += sd[k];
    }
    *tot_m = ncols > 0 ? (long long)(state[ncols - 1] & ST_VAL) : 0;
    *tot_ties = tt;
    *tot_sub = dd;
  }
}

size_t smem_bytes(int64_t rows) { return (size_t)((rows + 31) / 32) * 4 * 2; }

template <typename K>
void set_smem(K kernel, size_t bytes) {
  if (bytes > 40 * 1024)
    CGGM_CUDA_CHECK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes + 4096));
}

}  // namespace

ActWs active_ws(Ctx* c, int64_t q) {
  const size_t bytes = (size_t)q * 2 * (8 + 8 + 8) + sizeof(ActTotals) + 256;
  char* base = static_cast<char*>(ws_get(c, WS_ACT, bytes));
  ActWs w;
  w.stateL = reinterpret_cast<unsigned long long*>(base);
  w.stateT = w.stateL + q;
  w.tieL = reinterpret_cast<long long*>(w.stateT + q);
  w.tieT = w.tieL + q;
  w.subL = reinterpret_cast<double*>(w.tieT + q);
  w.subT = w.subL + q;
  w.tot = reinterpret_cast<ActTotals*>(w.subT + q);
  return w;
}

void active_begin(Ctx* c, int64_t q, const ActWs& ws) {
  if (q > 0) CGGM_CUDA_CHECK(cudaMemsetAsync(ws.stateL, 0, (size_t)q * 2 * 8, c->stream));
}

template <typename T>
void active_lambda(Ctx* c, int64_t q, const T* GradL, int64_t ldgl, const cggm_csc* Lambda, double lam_L,
                   int penalize_diag, double tie_eps, const ActWs& ws, int32_t* L_row, int32_t* L_col,
                   long long capL) {
  if (q == 0) return;
  const size_t bl = smem_bytes(q);
  set_smem(k_active_onepass<true, T>, bl);
  Prof pr(c, TAG_ACTIVE);
  k_active_onepass<true, T><<<(unsigned)q, NT, bl, c->stream>>>(
      q, GradL, ldgl, Lambda->colptr, Lambda->rowidx, static_cast<const T*>(Lambda->val), (T)lam_L, penalize_diag,
      (T)tie_eps, ws.stateL, L_row, L_col, capL, ws.tieL, ws.subL, 0);
  post_launch(c, "k_active_onepass<L>");
}

template <typename T>
void active_theta_chunk(Ctx* c, int64_t p, int64_t col0, int64_t ncols, const T* G, int64_t ldg,
                        const cggm_csc* Theta, double lam_T, double tie_eps, const ActWs& ws, int32_t* T_row,
                        int32_t* T_col, long long capT) {
  if (ncols == 0) return;
  const size_t bt = smem_bytes(p);
  set_smem(k_active_onepass<false, T>, bt);
  Prof pr(c, TAG_ACTIVE);
  k_active_onepass<false, T><<<(unsigned)ncols, NT, bt, c->stream>>>(
      p, G, ldg, Theta->colptr, Theta->rowidx, static_cast<const T*>(Theta->val), (T)lam_T, 1, (T)tie_eps,
      ws.stateT, T_row, T_col, capT, ws.tieT, ws.subT, col0);
  post_launch(c, "k_active_onepass<T>");
}

void active_end(Ctx* c, int64_t q, const ActWs& ws) {
  if (q == 0) return;
  {
    Prof pr(c, TAG_ACTIVE);
    k_active_totals<<<1, TOT_NT, 0, c->stream>>>(q, ws.stateL, ws.tieL, ws.subL, &ws.tot->m_L, &ws.tot->ties_L,
                                                 &ws.tot->sub_L);
    post_launch(c, "k_active_totals<L>");
  }
  {
    Prof pr(c, TAG_ACTIVE);
    k_active_totals<<<1, TOT_NT, 0, c->stream>>>(q, ws.stateT, ws.tieT, ws.subT, &ws.tot->m_T, &ws.tot->ties_T,
                                                 &ws.tot->sub_T);
    post_launch(c, "k_active_totals<T>");
  }
}

template <typename T>
void active_compact(Ctx* c, int64_t p, int64_t q, const T* GradL, int64_t ldgl, const T* GradT, int64_t ldgt,
                    const cggm_csc* Lambda, const cggm_csc* Theta, double lam_L, double lam_T, int penalize_diag,
                    double tie_eps, const ActWs& ws, int32_t* L_row, int32_t* L_col, int32_t* T_row, int32_t* T_col,
                    long long capL, long long capT) {
  if (q == 0) return;
  active_begin(c, q, ws);
  active_lambda<T>(c, q, GradL, ldgl, Lambda, lam_L, penalize_diag, tie_eps, ws, L_row, L_col, capL);
  active_theta_chunk<T>(c, p, 0, q, GradT, ldgt, Theta, lam_T, tie_eps, ws, T_row, T_col, capT);
  active_end(c, q, ws);
}

template void active_compact<double>(Ctx*, int64_t, int64_t, const double*, int64_t, const double*, int64_t,
                                     const cggm_csc*, const cggm_csc*, double, double, int, double, const ActWs&,
                                     int32_t*, int32_t*, int32_t*, int32_t*, long long, long long);
template void active_compact<float>(Ctx*, int64_t, int64_t, const float*, int64_t, const float*, int64_t,
                                    const cggm_csc*, const cggm_csc*, double, double, int, double, const ActWs&,
                                    int32_t*, int32_t*, int32_t*, int32_t*, long long, long long);
#define CGGM_INST(T)                                                                                          \
  template void active_lambda<T>(Ctx*, int64_t, const T*, int64_t, const cggm_csc*, double, int, double,      \
                                 const ActWs&, int32_t*, int32_t*, long long);                                 \
  template void active_theta_chunk<T>(Ctx*, int64_t, int64_t, int64_t, const T*, int64_t, const cggm_csc*,     \
                                      double, double, const ActWs&, int32_t*, int32_t*, long long);
CGGM_INST(double)
CGGM_INST(float)
#undef CGGM_INST

}  // namespace cggm
