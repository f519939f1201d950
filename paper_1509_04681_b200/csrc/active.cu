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

#ifndef CGGM_ACT_LAM_MINB
#define CGGM_ACT_LAM_MINB 6
#endif
constexpr int NT = 256;
constexpr int NW = NT / 32;   // warp segments per column
constexpr int UNR = 4;        // 32-row chunks in flight per lane
#ifndef CGGM_LF_UNR
#define CGGM_LF_UNR 4
#endif
#ifndef CGGM_LF_MINB
#define CGGM_LF_MINB 6
#endif
constexpr int LF_UNR = CGGM_LF_UNR;   // 64-row pair chunks in flight per lane (split Lambda flags pass)
// words of the Lambda flag bitmask before column j (column c: ceil((c + 1) / 64) chunks of 2 words)
__host__ __device__ inline long long tri_words_before_i(long long j) {
  const long long m = j / 64, r = j % 64;
  return 2 * (64 * m * (m + 1) / 2 + r * (m + 1));
}

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
    if (LAM && i > j) continue;   // lower entries: counted twice from their mirror (symmetric Lambda, gradient)
    const T gv = gc[i];
    const T lm = lam_of<LAM>(i, j, lam, penalize_diag);
    const double wt = (LAM && i < j) ? 2.0 : 1.0;
    s += wt * ((double)fabs(gv + lm * (x > T(0) ? T(1) : T(-1))) - (double)fmax(fabs(gv) - lm, T(0)));
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

// Vectorised variant (the path taken whenever the gradient columns are 16-byte aligned): each lane
// loads a PAIR of rows per 64-row chunk (LDG.128 for fp64), flags are kept as two ballot words per
// chunk (even rows, odd rows), and the per-element work is a handful of instructions -- the scalar
// kernel above is issue-bound at ~40% of HBM bandwidth.  Same outputs and order: ascending rows per
// column, the subgradient partials of each column summed in a fixed order.
template <typename T>
struct PairOf;
template <>
struct PairOf<double> {
  using V = double2;
};
template <>
struct PairOf<float> {
  using V = float2;
};

template <bool LAM, typename T>
__global__ void __launch_bounds__(NT, LAM ? CGGM_ACT_LAM_MINB : 4) k_active_vec(int64_t nrows, const T* __restrict__ G, int64_t ldg,
                                                   const int64_t* colptr, const int32_t* rowidx, const T* val,
                                                   T lam, int penalize_diag, T tie_eps,
                                                   unsigned long long* state, int32_t* out_row, int32_t* out_col,
                                                   long long cap, long long* ties_col, double* sub_col,
                                                   int64_t col0) {
  using V = typename PairOf<T>::V;
  extern __shared__ uint32_t sm[];
  const int64_t j = col0 + blockIdx.x;
  const int scan_rows = (int)(LAM ? j + 1 : nrows);
  const int nch = (scan_rows + 63) >> 6;   // 64-row chunks
  uint32_t* sup = sm;                      // [2c + h]: rows 64c + 32h .. +31 (bit = row & 31)
  uint32_t* flg = sm + 2 * nch;            // [2c + e]: bit l = row 64c + 2l + e
  __shared__ int wcnt[NW];
  __shared__ double wsub[NW];
  __shared__ long long wtie[NW];
  __shared__ long long col_base;
  for (int w = threadIdx.x; w < 2 * nch; w += NT) sup[w] = 0u;
  __syncthreads();
  for (int64_t t = colptr[j] + threadIdx.x; t < colptr[j + 1]; t += NT) {
    const int32_t r = rowidx[t];
    if (r < scan_rows && val[t] != T(0)) atomicOr(&sup[r >> 5], 1u << (r & 31));
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int per = (nch + NW - 1) / NW;
  const int ca = min(nch, w * per), cb = min(nch, (w + 1) * per);
  const T* gc = G + (j - col0) * ldg;
  const V* gv = reinterpret_cast<const V*>(gc);
  const int full_end = scan_rows >> 6;     // chunks [0, full_end) lie entirely inside the column
  const int jj = (int)j;
  const T lam_diag = (LAM && !penalize_diag) ? T(0) : lam;
  int cnt = 0;
  long long tc = 0;
  double s0 = 0.0, s1 = 0.0;   // two accumulators (even / odd rows): shorter dependency chains
  auto process = [&](int c, T x0, T x1) {
    const int r = 64 * c + 2 * lane;
    const bool in0 = r < scan_rows, in1 = r + 1 < scan_rows;
    const uint32_t sw = sup[2 * c + (lane >> 4)];
    const uint32_t sb = sw >> ((2 * lane) & 31);
    const T l0 = (LAM && r == jj) ? lam_diag : lam;
    const T l1 = (LAM && r + 1 == jj) ? lam_diag : lam;
    const T d0 = fabs(x0) - l0, d1 = fabs(x1) - l1;
    // cold chunk (the common case for Theta): no entry within tie_eps of its threshold or above it,
    // no stored nonzero -> no flag, tie or subgradient contribution; one vote instead of the rest
    const bool hot = (sb & 3u) || d0 >= -tie_eps || d1 >= -tie_eps;
    if (!__any_sync(0xffffffffu, hot)) {
      if (lane == 0) *reinterpret_cast<uint2*>(&flg[2 * c]) = make_uint2(0u, 0u);
      return;
    }
    const bool sp0 = sb & 1u, sp1 = (sb >> 1) & 1u;
    const bool f0 = in0 && (d0 > T(0) || sp0), f1 = in1 && (d1 > T(0) || sp1);
    const unsigned m0 = __ballot_sync(0xffffffffu, f0), m1 = __ballot_sync(0xffffffffu, f1);
    if (lane == 0) {
      flg[2 * c] = m0;
      flg[2 * c + 1] = m1;
    }
    cnt += __popc(m0) + __popc(m1);
    tc += (in0 && !sp0 && fabs(d0) <= tie_eps) + (in1 && !sp1 && fabs(d1) <= tie_eps);
    // LAM: rows i < j count twice (both triangles), the diagonal once
    const double w0 = (LAM && r < jj) ? 2.0 : 1.0, w1 = (LAM && r + 1 < jj) ? 2.0 : 1.0;
    if (in0 && d0 > T(0)) s0 += w0 * (double)d0;
    if (in1 && d1 > T(0)) s1 += w1 * (double)d1;
  };
  const int fe = min(cb, full_end);
  int c = ca;
  if (LAM) {   // (the triangle's short columns: pipelining costs more registers than it hides)
    for (; c + UNR <= fe; c += UNR) {
      V v[UNR];
#pragma unroll
      for (int u = 0; u < UNR; ++u) v[u] = __ldcs(gv + (int64_t)(c + u) * 32 + lane);
#pragma unroll
      for (int u = 0; u < UNR; ++u) process(c + u, v[u].x, v[u].y);
    }
  } else if (c + UNR <= fe) {
    // software-pipelined: the next group's loads are in flight while the current one is processed
    V cur[UNR], nxt[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) cur[u] = __ldcs(gv + (int64_t)(c + u) * 32 + lane);   // streamed once
    for (; c + UNR <= fe; c += UNR) {
      const bool more = c + 2 * UNR <= fe;
      if (more) {
#pragma unroll
        for (int u = 0; u < UNR; ++u) nxt[u] = __ldcs(gv + (int64_t)(c + UNR + u) * 32 + lane);
      }
#pragma unroll
      for (int u = 0; u < UNR; ++u) process(c + u, cur[u].x, cur[u].y);
      if (more) {
#pragma unroll
        for (int u = 0; u < UNR; ++u) cur[u] = nxt[u];
      }
    }
  }
  for (; c < cb; ++c) {   // remainder and the partial last chunk (element loads, bounds-checked)
    const int r = 64 * c + 2 * lane;
    const T x0 = r < scan_rows ? __ldcs(gc + r) : T(0);
    const T x1 = r + 1 < scan_rows ? __ldcs(gc + r + 1) : T(0);
    process(c, x0, x1);
  }
  double sacc = s0 + s1;
  for (int64_t t = colptr[j] + threadIdx.x; t < colptr[j + 1]; t += NT) {
    const T x = val[t];
    if (x == T(0)) continue;
    const int64_t i = rowidx[t];
    // Lambda: entries below the diagonal are counted twice from their mirror in the upper triangle
    // (Lambda and its gradient are exactly symmetric), so only rows <= j of the gradient are read
    if (LAM && i > j) continue;
    const T gi = gc[i];
    const T lm = lam_of<LAM>(i, j, lam, penalize_diag);
    const double wt = (LAM && i < j) ? 2.0 : 1.0;
    sacc += wt * ((double)fabs(gi + lm * (x > T(0) ? T(1) : T(-1))) - (double)fmax(fabs(gi) - lm, T(0)));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sacc += __shfl_down_sync(0xffffffffu, sacc, o);
    tc += __shfl_down_sync(0xffffffffu, tc, o);
  }
  if (lane == 0) {
    wcnt[w] = cnt;
    wsub[w] = sacc;
    wtie[w] = tc;
  }
  __syncthreads();
  __shared__ long long s_total, s_add[NW];
  __shared__ int s_stop;
  if (threadIdx.x == 0) {
    long long total = 0, tt = 0;
    double ss = 0.0;
    for (int k = 0; k < NW; ++k) {
      total += wcnt[k];
      tt += wtie[k];
      ss += wsub[k];
    }
    sub_col[j] = ss;
    ties_col[j] = tt;
    st_release(&state[j], (j == 0 ? ST_INC : ST_AGG) | (unsigned long long)total);
    s_total = total;
    s_stop = NT;
  }
  __syncthreads();
  // decoupled look-back with the whole block: thread t inspects predecessor k0 - t, so a window
  // spans NT columns (the predecessors still scanning are about one wave of CTAs back)
  long long excl = 0;
  for (int64_t k0 = j - 1; k0 >= 0; k0 -= NT) {
    const int64_t k = k0 - threadIdx.x;
    unsigned long long v = ST_INC;   // before column 0: prefix 0
    if (k >= 0) {
      v = ld_acquire(&state[k]);
      while ((v & ~ST_VAL) == 0) v = ld_acquire(&state[k]);
    }
    if ((v & ~ST_VAL) == ST_INC) atomicMin(&s_stop, (int)threadIdx.x);
    __syncthreads();
    const int stop = s_stop;   // nearest inclusive predecessor
    long long add = (threadIdx.x <= stop && k >= 0) ? (long long)(v & ST_VAL) : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) add += __shfl_xor_sync(0xffffffffu, add, o);
    if (lane == 0) s_add[w] = add;
    __syncthreads();
    for (int k2 = 0; k2 < NW; ++k2) excl += s_add[k2];
    if (stop < NT) break;
    __syncthreads();
  }
  if (threadIdx.x == 0 && j > 0) st_release(&state[j], ST_INC | (unsigned long long)(excl + s_total));
  long long pos = excl;
  for (int k = 0; k < w; ++k) pos += wcnt[k];
  const unsigned below = (1u << lane) - 1u;
  // 32 chunks per round: lane l reads chunk c0 + l's words, the warp walks the non-empty ones
  for (int c0 = ca; c0 < cb; c0 += 32) {
    unsigned w0 = 0u, w1 = 0u;
    if (c0 + lane < cb) {
      w0 = flg[2 * (c0 + lane)];
      w1 = flg[2 * (c0 + lane) + 1];
    }
    unsigned nz = __ballot_sync(0xffffffffu, (w0 | w1) != 0u);
    while (nz) {
      const int l = __ffs(nz) - 1;
      nz &= nz - 1u;
      const unsigned m0 = __shfl_sync(0xffffffffu, w0, l), m1 = __shfl_sync(0xffffffffu, w1, l);
      const long long base = pos + __popc(m0 & below) + __popc(m1 & below);
      const int r = 64 * (c0 + l) + 2 * lane;
      const bool s0 = (m0 >> lane) & 1u, s1 = (m1 >> lane) & 1u;
      if (s0 && base < cap) {
        out_row[base] = r;
        out_col[base] = (int32_t)j;
      }
      const long long p1 = base + s0;
      if (s1 && p1 < cap) {
        out_row[p1] = r + 1;
        out_col[p1] = (int32_t)j;
      }
      pos += __popc(m0) + __popc(m1);
    }
  }
}

// ---------------------------------------------------------------- split Lambda compaction
// The Lambda list is ~half the upper triangle at `large` (1.03e8 entries): its single-pass kernel
// spent a quarter of its time with seven warps parked at the barrier behind warp 0's look-back.
// Split instead: (1) the scan writes each column's flag words (2 per 64 rows) to a global bitmask
// (q^2/64 words, 25 MB at q = 20000) with its count / ties / subgradient partial -- no
// inter-column dependency at all; (2) one block scans the q counts into column bases; (3) the
// writer turns each column's words into (row, col) entries at its base.
template <typename T>
__device__ __forceinline__ void k_lam_flags_col(const T* __restrict__ G, int64_t ldg, const int64_t* colptr,
                                                const int32_t* rowidx, const T* val, T lam, int penalize_diag,
                                                T tie_eps, uint32_t* flags, unsigned long long* cnt_col,
                                                long long* ties_col, double* sub_col, int64_t j) {
  using V = typename PairOf<T>::V;
  extern __shared__ uint32_t sm[];
  const int scan_rows = (int)(j + 1);
  const int nch = (scan_rows + 63) >> 6;
  uint32_t* sup = sm;
  uint32_t* flg = flags + tri_words_before_i(j);
  __shared__ int wcnt[NW];
  __shared__ double wsub[NW];
  __shared__ long long wtie[NW];
  for (int w = threadIdx.x; w < 2 * nch; w += NT) sup[w] = 0u;
  __syncthreads();
  for (int64_t t = colptr[j] + threadIdx.x; t < colptr[j + 1]; t += NT) {
    const int32_t r = rowidx[t];
    if (r < scan_rows && val[t] != T(0)) atomicOr(&sup[r >> 5], 1u << (r & 31));
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int per = (nch + NW - 1) / NW;
  const int ca = min(nch, w * per), cb = min(nch, (w + 1) * per);
  const T* gc = G + j * ldg;
  const V* gv = reinterpret_cast<const V*>(gc);
  const int full_end = scan_rows >> 6;
  const int jj = (int)j;
  const T lam_diag = !penalize_diag ? T(0) : lam;
  int cnt = 0, tc = 0;
  double s_all = 0.0, s_diag = 0.0;   // rows i < j count twice (both triangles): 2 s_all - s_diag
  auto process = [&](int c, T x0, T x1) {
    const int r = 64 * c + 2 * lane;
    const bool in0 = r < scan_rows, in1 = r + 1 < scan_rows;
    const uint32_t sb = sup[2 * c + (lane >> 4)] >> ((2 * lane) & 31);
    const T l0 = (r == jj) ? lam_diag : lam;
    const T l1 = (r + 1 == jj) ? lam_diag : lam;
    const T d0 = fabs(x0) - l0, d1 = fabs(x1) - l1;
    const bool sp0 = sb & 1u, sp1 = (sb >> 1) & 1u;
    const bool f0 = in0 && (d0 > T(0) || sp0), f1 = in1 && (d1 > T(0) || sp1);
    const unsigned m0 = __ballot_sync(0xffffffffu, f0), m1 = __ballot_sync(0xffffffffu, f1);
    if (lane == 0) *reinterpret_cast<uint2*>(&flg[2 * c]) = make_uint2(m0, m1);
    cnt += __popc(m0) + __popc(m1);
    tc += (in0 && !sp0 && fabs(d0) <= tie_eps) + (in1 && !sp1 && fabs(d1) <= tie_eps);
    const double e0 = (in0 && d0 > T(0)) ? (double)d0 : 0.0, e1 = (in1 && d1 > T(0)) ? (double)d1 : 0.0;
    s_all += e0 + e1;
    if (r == jj) s_diag += e0;
    if (r + 1 == jj) s_diag += e1;
  };
  // chunks wholly above the diagonal (64 c + 63 < j): every row in range, off-diagonal weight --
  // the bulk of the triangle, with a third fewer instructions than the general chunk (the pass is
  // issue-bound, not DRAM-bound, with the general form)
  auto process_off = [&](int c, T x0, T x1) {
    const uint32_t sb = sup[2 * c + (lane >> 4)] >> ((2 * lane) & 31);
    const T d0 = fabs(x0) - lam, d1 = fabs(x1) - lam;
    const bool sp0 = sb & 1u, sp1 = sb & 2u;
    const unsigned m0 = __ballot_sync(0xffffffffu, d0 > T(0) || sp0);
    const unsigned m1 = __ballot_sync(0xffffffffu, d1 > T(0) || sp1);
    if (lane == 0) *reinterpret_cast<uint2*>(&flg[2 * c]) = make_uint2(m0, m1);
    cnt += __popc(m0) + __popc(m1);
    tc += (!sp0 && fabs(d0) <= tie_eps) + (!sp1 && fabs(d1) <= tie_eps);
    s_all += (double)fmax(d0, T(0)) + (double)fmax(d1, T(0));
  };
  const int oe = min(cb, jj >> 6);
  int c = ca;
  for (; c + LF_UNR <= oe; c += LF_UNR) {
    V v[LF_UNR];
#pragma unroll
    for (int u = 0; u < LF_UNR; ++u) v[u] = __ldcs(gv + (int64_t)(c + u) * 32 + lane);
#pragma unroll
    for (int u = 0; u < LF_UNR; ++u) process_off(c + u, v[u].x, v[u].y);
  }
  for (; c < oe; ++c) {
    const V v = __ldcs(gv + (int64_t)c * 32 + lane);
    process_off(c, v.x, v.y);
  }
  const int fe = min(cb, full_end);
  for (; c < fe; ++c) {
    const V v = __ldcs(gv + (int64_t)c * 32 + lane);
    process(c, v.x, v.y);
  }
  for (; c < cb; ++c) {
    const int r = 64 * c + 2 * lane;
    const T x0 = r < scan_rows ? __ldcs(gc + r) : T(0);
    const T x1 = r + 1 < scan_rows ? __ldcs(gc + r + 1) : T(0);
    process(c, x0, x1);
  }
  double sacc = 2.0 * s_all - s_diag;
  for (int64_t t = colptr[j] + threadIdx.x; t < colptr[j + 1]; t += NT) {
    const T x = val[t];
    if (x == T(0)) continue;
    const int64_t i = rowidx[t];
    if (i > j) continue;   // counted twice from the mirror (symmetric)
    const T gi = gc[i];
    const T lm = lam_of<true>(i, j, lam, penalize_diag);
    const double wt = i < j ? 2.0 : 1.0;
    sacc += wt * ((double)fabs(gi + lm * (x > T(0) ? T(1) : T(-1))) - (double)fmax(fabs(gi) - lm, T(0)));
  }
  long long tcl = tc;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sacc += __shfl_down_sync(0xffffffffu, sacc, o);
    tcl += __shfl_down_sync(0xffffffffu, tcl, o);
  }
  if (lane == 0) {
    wcnt[w] = cnt;
    wsub[w] = sacc;
    wtie[w] = tcl;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    long long total = 0, tt = 0;
    double ss = 0.0;
    for (int k = 0; k < NW; ++k) {
      total += wcnt[k];
      tt += wtie[k];
      ss += wsub[k];
    }
    cnt_col[j] = (unsigned long long)total;
    ties_col[j] = tt;
    sub_col[j] = ss;
  }
}

// CTA k takes columns k and q - 1 - k: every CTA scans q + 1 rows of the triangle
template <typename T>
__global__ void __launch_bounds__(NT, CGGM_LF_MINB) k_lam_flags(const T* __restrict__ G, int64_t ldg,
                                                                const int64_t* colptr, const int32_t* rowidx,
                                                                const T* val, T lam, int penalize_diag, T tie_eps,
                                                                uint32_t* flags, unsigned long long* cnt_col,
                                                                long long* ties_col, double* sub_col, int64_t q) {
  for (int side = 0; side < 2; ++side) {
    const int64_t j = side == 0 ? (int64_t)blockIdx.x : q - 1 - (int64_t)blockIdx.x;
    if (side == 1 && j <= (int64_t)blockIdx.x) break;
    k_lam_flags_col<T>(G, ldg, colptr, rowidx, val, lam, penalize_diag, tie_eps, flags, cnt_col, ties_col, sub_col, j);
    __syncthreads();
  }
}

// exclusive scan of the column counts (one block): thread t owns a contiguous run of columns,
// the 1024 run totals are scanned with warp shuffles; state[q - 1] gets the inclusive total in the
// look-back encoding k_active_totals reads
__global__ void __launch_bounds__(1024) k_lam_scan(int64_t q, unsigned long long* cnt_state, long long* base) {
  __shared__ long long wsum[32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t per = (q + 1023) / 1024;
  const int64_t c0 = min(q, (int64_t)threadIdx.x * per), c1 = min(q, c0 + per);
  long long run = 0;
  for (int64_t c = c0; c < c1; ++c) run += (long long)cnt_state[c];
  long long incl = run;   // inclusive scan over the block
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long x = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += x;
  }
  if (lane == 31) wsum[w] = incl;
  __syncthreads();
  if (w == 0) {
    long long v = wsum[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long x = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += x;
    }
    wsum[lane] = v;   // inclusive over warps
  }
  __syncthreads();
  long long pos = incl - run + (w > 0 ? wsum[w - 1] : 0);
  for (int64_t c = c0; c < c1; ++c) {
    const long long v = (long long)cnt_state[c];
    base[c] = pos;
    pos += v;
  }
  if (threadIdx.x == 1023 && q > 0) {
    base[q] = wsum[31];
    cnt_state[q - 1] = ST_INC | (unsigned long long)wsum[31];
  }
}

// (row, col) entries of column j from its nch chunks of flag words flg[2c], flg[2c + 1] at base[j]
__device__ __forceinline__ void write_col_words(const uint32_t* __restrict__ flg, int nch, const long long* base,
                                                int32_t* __restrict__ out_row, int32_t* __restrict__ out_col,
                                                long long cap, int64_t j) {
  __shared__ int wcnt[NW];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int per = (nch + NW - 1) / NW;
  const int ca = min(nch, w * per), cb = min(nch, (w + 1) * per);
  int cnt = 0;
  for (int c = ca + lane; c < cb; c += 32) {
    const uint2 m = *reinterpret_cast<const uint2*>(&flg[2 * c]);
    cnt += __popc(m.x) + __popc(m.y);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if (lane == 0) wcnt[w] = cnt;
  __syncthreads();
  long long pos = base[j];
  for (int k = 0; k < w; ++k) pos += wcnt[k];
  const unsigned below = (1u << lane) - 1u;
  // 32 chunks per round: lane l loads chunk c0 + l's words, the warp walks the non-empty ones
  for (int c0 = ca; c0 < cb; c0 += 32) {
    uint2 mine = make_uint2(0u, 0u);
    if (c0 + lane < cb) mine = *reinterpret_cast<const uint2*>(&flg[2 * (c0 + lane)]);
    unsigned nz = __ballot_sync(0xffffffffu, (mine.x | mine.y) != 0u);
    while (nz) {
      const int l = __ffs(nz) - 1;
      nz &= nz - 1u;
      const unsigned m0 = __shfl_sync(0xffffffffu, mine.x, l), m1 = __shfl_sync(0xffffffffu, mine.y, l);
      const long long b = pos + __popc(m0 & below) + __popc(m1 & below);
      const int r = 64 * (c0 + l) + 2 * lane;
      const bool s0 = (m0 >> lane) & 1u, s1 = (m1 >> lane) & 1u;
      if (s0 && b < cap) {
        out_row[b] = r;
        out_col[b] = (int32_t)j;
      }
      const long long p1 = b + s0;
      if (s1 && p1 < cap) {
        out_row[p1] = r + 1;
        out_col[p1] = (int32_t)j;
      }
      pos += __popc(m0) + __popc(m1);
    }
  }
}

__device__ __forceinline__ void k_lam_write_col(const uint32_t* __restrict__ flags, const long long* base,
                                                int32_t* __restrict__ out_row, int32_t* __restrict__ out_col,
                                                long long cap, int64_t j) {
  write_col_words(flags + tri_words_before_i(j), (int)((j + 1 + 63) >> 6), base, out_row, out_col, cap, j);
}

// K01: S_Theta entries of column j from the words the X^T E epilogue wrote (wpc per column)
__global__ void __launch_bounds__(NT) k_sel_write(const uint32_t* flags, int64_t wpc, int nch, const long long* base,
                                                  int32_t* out_row, int32_t* out_col, long long cap) {
  const int64_t j = blockIdx.x;
  write_col_words(flags + j * wpc, nch, base, out_row, out_col, cap, j);
}

// K01: per-column subgradient = the row tiles' partials summed in row order (fixed: reproducible)
__global__ void k_sel_sub(int64_t q, int64_t nrow, const double* __restrict__ subpart, int64_t ld,
                          double* __restrict__ sub_col) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= q) return;
  double acc = 0.0;
  for (int64_t r = 0; r < nrow; ++r) acc += subpart[r * ld + j];
  sub_col[j] = acc;
}

// (row, col) entries of columns k and q - 1 - k from their flag words at base[]
__global__ void __launch_bounds__(NT) k_lam_write(const uint32_t* flags, const long long* base, int32_t* out_row,
                                                  int32_t* out_col, long long cap, int64_t q) {
  for (int side = 0; side < 2; ++side) {
    const int64_t j = side == 0 ? (int64_t)blockIdx.x : q - 1 - (int64_t)blockIdx.x;
    if (side == 1 && j <= (int64_t)blockIdx.x) break;
    k_lam_write_col(flags, base, out_row, out_col, cap, j);
    __syncthreads();
  }
}

// totals: m from the last column's inclusive state, ties / subgradient summed in a fixed order
// (contiguous runs per thread, then a fixed shuffle tree): bitwise reproducible
constexpr int TOT_NT = 1024;
// block 0: the Lambda list, block 1: the Theta list
__global__ void __launch_bounds__(TOT_NT) k_active_totals(int64_t ncols, ActWs ws) {
  const bool th = blockIdx.x == 1;
  const unsigned long long* state = th ? ws.stateT : ws.stateL;
  const long long* ties_col = th ? ws.tieT : ws.tieL;
  const double* sub_col = th ? ws.subT : ws.subL;
  long long* tot_m = th ? &ws.tot->m_T : &ws.tot->m_L;
  long long* tot_ties = th ? &ws.tot->ties_T : &ws.tot->ties_L;
  double* tot_sub = th ? &ws.tot->sub_T : &ws.tot->sub_L;
  __shared__ long long st[32];
  __shared__ double sd[32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t per = (ncols + TOT_NT - 1) / TOT_NT;
  const int64_t b = threadIdx.x * per, e = min(ncols, b + per);
  long long t = 0;
  double d = 0.0;
  for (int64_t i = b; i < e; ++i) {
    t += ties_col[i];
    d += sub_col[i];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    t += __shfl_down_sync(0xffffffffu, t, o);
    d += __shfl_down_sync(0xffffffffu, d, o);
  }
  if (lane == 0) {
    st[w] = t;
    sd[w] = d;
  }
  __syncthreads();
  if (w == 0) {
    t = st[lane];
    d = sd[lane];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      t += __shfl_down_sync(0xffffffffu, t, o);
      d += __shfl_down_sync(0xffffffffu, d, o);
    }
    if (lane == 0) {
      *tot_m = ncols > 0 ? (long long)(state[ncols - 1] & ST_VAL) : 0;
      *tot_ties = t;
      *tot_sub = d;
    }
  }
}

size_t smem_bytes(int64_t rows) { return (size_t)((rows + 31) / 32) * 4 * 2; }
size_t smem_bytes_vec(int64_t rows) { return (size_t)((rows + 63) / 64) * 4 * 4; }

// the pair loads need 2*sizeof(T)-aligned columns
template <typename T>
bool vec_ok(const T* G, int64_t ldg, int no_vec) {
  return !no_vec && (reinterpret_cast<uintptr_t>(G) % (2 * sizeof(T)) == 0) && (ldg % 2 == 0);
}

template <typename K>
void set_smem(K kernel, size_t bytes) {
  if (bytes > 40 * 1024)
    CGGM_CUDA_CHECK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes + 4096));
}

}  // namespace

ActWs active_ws(Ctx* c, int64_t q) {
  const size_t fl_words = (size_t)tri_words_before_i(q) + 64;
  const size_t bytes = (size_t)q * 2 * (8 + 8 + 8) + sizeof(ActTotals) + 256 + (size_t)(q + 1) * 8 + fl_words * 4;
  char* base = static_cast<char*>(ws_get(c, WS_ACT, bytes));
  ActWs w;
  w.stateL = reinterpret_cast<unsigned long long*>(base);
  w.stateT = w.stateL + q;
  w.tieL = reinterpret_cast<long long*>(w.stateT + q);
  w.tieT = w.tieL + q;
  w.subL = reinterpret_cast<double*>(w.tieT + q);
  w.subT = w.subL + q;
  w.tot = reinterpret_cast<ActTotals*>(w.subT + q);
  char* after = reinterpret_cast<char*>(w.tot) + ((sizeof(ActTotals) + 255) / 256) * 256;
  w.baseL = reinterpret_cast<long long*>(after);
  w.flagsL = reinterpret_cast<uint32_t*>(w.baseL + (q + 1));
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
  Prof pr(c, TAG_ACTIVE);
  if (vec_ok(GradL, ldgl, c->no_active_vec) && !c->act_onepass) {   // split: flags -> scan -> write
    const size_t bf = (size_t)((q + 63) / 64) * 2 * 4;
    set_smem(k_lam_flags<T>, bf);
    const unsigned pairs = (unsigned)((q + 1) / 2);
    k_lam_flags<T><<<pairs, NT, bf, c->stream>>>(GradL, ldgl, Lambda->colptr, Lambda->rowidx,
                                                 static_cast<const T*>(Lambda->val), (T)lam_L, penalize_diag,
                                                 (T)tie_eps, ws.flagsL, ws.stateL, ws.tieL, ws.subL, q);
    k_lam_scan<<<1, 1024, 0, c->stream>>>(q, ws.stateL, ws.baseL);
    k_lam_write<<<pairs, NT, 0, c->stream>>>(ws.flagsL, ws.baseL, L_row, L_col, capL, q);
    c->launches += 2;
    post_launch(c, "k_lam_flags/scan/write");
    return;
  }
  if (vec_ok(GradL, ldgl, c->no_active_vec)) {
    const size_t bv = smem_bytes_vec(q);
    set_smem(k_active_vec<true, T>, bv);
    k_active_vec<true, T><<<(unsigned)q, NT, bv, c->stream>>>(
        q, GradL, ldgl, Lambda->colptr, Lambda->rowidx, static_cast<const T*>(Lambda->val), (T)lam_L, penalize_diag,
        (T)tie_eps, ws.stateL, L_row, L_col, capL, ws.tieL, ws.subL, 0);
    post_launch(c, "k_active_vec<L>");
    return;
  }
  const size_t bl = smem_bytes(q);
  set_smem(k_active_onepass<true, T>, bl);
  k_active_onepass<true, T><<<(unsigned)q, NT, bl, c->stream>>>(
      q, GradL, ldgl, Lambda->colptr, Lambda->rowidx, static_cast<const T*>(Lambda->val), (T)lam_L, penalize_diag,
      (T)tie_eps, ws.stateL, L_row, L_col, capL, ws.tieL, ws.subL, 0);
  post_launch(c, "k_active_onepass<L>");
}

// Lambda list for columns [col0, col0 + ncols) from a gradient block G whose column j - col0 holds
// rows 0..j of column j (the memory-bounded evaluation forms grad_Lambda block by block); chunks in
// ascending column order, chained by the same decoupled look-back as the whole-matrix kernel
template <typename T>
void active_lambda_chunk(Ctx* c, int64_t q, int64_t col0, int64_t ncols, const T* G, int64_t ldg,
                         const cggm_csc* Lambda, double lam_L, int penalize_diag, double tie_eps, const ActWs& ws,
                         int32_t* L_row, int32_t* L_col, long long capL) {
  if (ncols == 0) return;
  Prof pr(c, TAG_ACTIVE);
  if (vec_ok(G, ldg, c->no_active_vec)) {
    const size_t bv = smem_bytes_vec(q);
    set_smem(k_active_vec<true, T>, bv);
    k_active_vec<true, T><<<(unsigned)ncols, NT, bv, c->stream>>>(
        q, G, ldg, Lambda->colptr, Lambda->rowidx, static_cast<const T*>(Lambda->val), (T)lam_L, penalize_diag,
        (T)tie_eps, ws.stateL, L_row, L_col, capL, ws.tieL, ws.subL, col0);
    post_launch(c, "k_active_vec<L> chunk");
    return;
  }
  const size_t bl = smem_bytes(q);
  set_smem(k_active_onepass<true, T>, bl);
  k_active_onepass<true, T><<<(unsigned)ncols, NT, bl, c->stream>>>(
      q, G, ldg, Lambda->colptr, Lambda->rowidx, static_cast<const T*>(Lambda->val), (T)lam_L, penalize_diag,
      (T)tie_eps, ws.stateL, L_row, L_col, capL, ws.tieL, ws.subL, col0);
  post_launch(c, "k_active_onepass<L> chunk");
}

template <typename T>
void active_theta_chunk(Ctx* c, int64_t p, int64_t col0, int64_t ncols, const T* G, int64_t ldg,
                        const cggm_csc* Theta, double lam_T, double tie_eps, const ActWs& ws, int32_t* T_row,
                        int32_t* T_col, long long capT) {
  if (ncols == 0) return;
  Prof pr(c, TAG_ACTIVE);
  if (vec_ok(G, ldg, c->no_active_vec)) {
    const size_t bv = smem_bytes_vec(p);
    set_smem(k_active_vec<false, T>, bv);
    k_active_vec<false, T><<<(unsigned)ncols, NT, bv, c->stream>>>(
        p, G, ldg, Theta->colptr, Theta->rowidx, static_cast<const T*>(Theta->val), (T)lam_T, 1, (T)tie_eps,
        ws.stateT, T_row, T_col, capT, ws.tieT, ws.subT, col0);
    post_launch(c, "k_active_vec<T>");
    return;
  }
  const size_t bt = smem_bytes(p);
  set_smem(k_active_onepass<false, T>, bt);
  k_active_onepass<false, T><<<(unsigned)ncols, NT, bt, c->stream>>>(
      p, G, ldg, Theta->colptr, Theta->rowidx, static_cast<const T*>(Theta->val), (T)lam_T, 1, (T)tie_eps,
      ws.stateT, T_row, T_col, capT, ws.tieT, ws.subT, col0);
  post_launch(c, "k_active_onepass<T>");
}

SelWs sel_ws(Ctx* c, int64_t p, int64_t q) {
  SelWs w;
  w.nch = (p + 63) / 64;
  w.wpc = 2 * w.nch;
  const size_t fbytes = ((size_t)q * w.wpc * 4 + 255) / 256 * 256, bbytes = ((size_t)(q + 1) * 8 + 255) / 256 * 256;
  char* base = static_cast<char*>(ws_get(c, WS_SEL, fbytes + bbytes + (size_t)w.nch * q * 8));
  w.flags = reinterpret_cast<uint32_t*>(base);
  w.base = reinterpret_cast<long long*>(base + fbytes);
  w.subpart = reinterpret_cast<double*>(base + fbytes + bbytes);
  return w;
}

SelectT select_begin(Ctx* c, int64_t p, int64_t q, const ActWs& ws, const SelWs& sw, const cggm_csc* Theta,
                     double lam_T, double tie_eps) {
  // (ws.stateT is zeroed by active_begin)
  CGGM_CUDA_CHECK(cudaMemsetAsync(ws.tieT, 0, (size_t)q * 8, c->stream));
  CGGM_CUDA_CHECK(cudaMemsetAsync(sw.subpart, 0, (size_t)sw.nch * q * 8, c->stream));
  SelectT S;
  S.on = 1;
  S.lam = lam_T;
  S.tie_eps = tie_eps;
  S.colptr = Theta->colptr;
  S.rowidx = Theta->rowidx;
  S.val = static_cast<const double*>(Theta->val);
  S.flags = sw.flags;
  S.wpc = sw.wpc;
  S.cnt = ws.stateT;
  S.ties = ws.tieT;
  S.subpart = sw.subpart;
  S.ldsub = q;
  return S;
}

void select_end(Ctx* c, int64_t p, int64_t q, const ActWs& ws, const SelWs& sw, int32_t* T_row, int32_t* T_col,
                long long capT) {
  if (q == 0) return;
  Prof pr(c, TAG_ACTIVE);
  k_sel_sub<<<(unsigned)((q + 255) / 256), 256, 0, c->stream>>>(q, sw.nch, sw.subpart, q, ws.subT);
  k_lam_scan<<<1, 1024, 0, c->stream>>>(q, ws.stateT, sw.base);
  k_sel_write<<<(unsigned)q, NT, 0, c->stream>>>(sw.flags, sw.wpc, (int)sw.nch, sw.base, T_row, T_col, capT);
  c->launches += 2;
  post_launch(c, "k_sel_sub/scan/write");
}

void active_end(Ctx* c, int64_t q, const ActWs& ws) {
  if (q == 0) return;
  Prof pr(c, TAG_ACTIVE);
  k_active_totals<<<2, TOT_NT, 0, c->stream>>>(q, ws);
  post_launch(c, "k_active_totals");
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
  template void active_lambda_chunk<T>(Ctx*, int64_t, int64_t, int64_t, const T*, int64_t, const cggm_csc*,    \
                                       double, int, double, const ActWs&, int32_t*, int32_t*, long long);      \
  template void active_theta_chunk<T>(Ctx*, int64_t, int64_t, int64_t, const T*, int64_t, const cggm_csc*,     \
                                      double, double, const ActWs&, int32_t*, int32_t*, long long);
CGGM_INST(double)
CGGM_INST(float)
#undef CGGM_INST

}  // namespace cggm
