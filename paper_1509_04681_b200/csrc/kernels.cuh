// Launch wrappers shared between translation units (reductions, active sets).
#pragma once
#include <climits>

#include "common.cuh"

namespace cggm {

template <typename T>
void col_partials(Ctx* c, int mode, int64_t n, int64_t ncols, const T* A, int64_t lda, const T* B, int64_t ldb,
                  const cggm_csc* csc, double* part);
template <typename T>
void csc_abs_partials(Ctx* c, const cggm_csc* A, bool skip_diag, double* part);
void sum_arrays(Ctx* c, int count, const double* const* arrs_dev, const int64_t* lens_dev, double* out_dev);
void init_scalars(Ctx* c, int* fail_col, int* flag);
void sum_arrays_1(Ctx* c, const double* a, int64_t len, double* out_dev);

// Active sets (active.cu).  Device totals:
template <typename T>
void r_e_from_acc(Ctx* c, int64_t n, int64_t q, const T* acc, int64_t lda, const T* Y, int64_t ldy, T* R, int64_t ldr,
                  T* E, int64_t lde, double s);
template <typename T>
void symmetrize(Ctx* c, int64_t n, T* S, int64_t ld);
template <typename T>
void peer_allreduce(Ctx* c, int world, int rank, void* const* bufs, int64_t count);
struct ActTotals {
  long long m_L, m_T, ties_L, ties_T;
  double sub_L, sub_T;
};
// per-column look-back states and partials, in workspace slot WS_ACT
struct ActWs {
  unsigned long long *stateL, *stateT;
  long long *tieL, *tieT;
  double *subL, *subT;
  ActTotals* tot;
  uint32_t* flagsL;        // Lambda flag bitmask of the upper triangle (split compaction)
  long long* baseL;        // column bases of the Lambda list
};
ActWs active_ws(Ctx* c, int64_t q);
// Building blocks of the single-pass compaction (one stream, in this order): begin (reset the
// look-back states), the Lambda list, the Theta list in one or several column chunks in ascending
// column order (G = the chunk's gradient columns col0 .. col0+ncols-1), end (totals).
void active_begin(Ctx* c, int64_t q, const ActWs& ws);
template <typename T>
void active_lambda(Ctx* c, int64_t q, const T* GradL, int64_t ldgl, const cggm_csc* Lambda, double lam_L,
                   int penalize_diag, double tie_eps, const ActWs& ws, int32_t* L_row, int32_t* L_col,
                   long long capL);
template <typename T>
void active_lambda_chunk(Ctx* c, int64_t q, int64_t col0, int64_t ncols, const T* G, int64_t ldg,
                         const cggm_csc* Lambda, double lam_L, int penalize_diag, double tie_eps, const ActWs& ws,
                         int32_t* L_row, int32_t* L_col, long long capL);
template <typename T>
void active_theta_chunk(Ctx* c, int64_t p, int64_t col0, int64_t ncols, const T* G, int64_t ldg,
                        const cggm_csc* Theta, double lam_T, double tie_eps, const ActWs& ws, int32_t* T_row,
                        int32_t* T_col, long long capT);
void active_end(Ctx* c, int64_t q, const ActWs& ws);
// K01: S_Theta selected in the X^T E GEMM epilogue (FP64): select_begin zeroes the tie / subgradient
// partials and returns the epilogue's SelectT (counts into ws.stateT); after the GEMM, select_end
// reduces the subgradient partials, scans the counts and writes the list (then active_end as usual)
struct SelWs {
  uint32_t* flags;
  long long* base;
  double* subpart;
  int64_t nch, wpc;
};
SelWs sel_ws(Ctx* c, int64_t p, int64_t q);
SelectT select_begin(Ctx* c, int64_t p, int64_t q, const ActWs& ws, const SelWs& sw, const cggm_csc* Theta,
                     double lam_T, double tie_eps);
void select_end(Ctx* c, int64_t p, int64_t q, const ActWs& ws, const SelWs& sw, int32_t* T_row, int32_t* T_col,
                long long capT);
// Single-pass ordered compaction of both lists + totals (device).  Entries at positions >= cap are
// not written (the caller reports CGGM_ERR_CAPACITY from the totals).
template <typename T>
void active_compact(Ctx* c, int64_t p, int64_t q, const T* GradL, int64_t ldgl, const T* GradT, int64_t ldgt,
                    const cggm_csc* Lambda, const cggm_csc* Theta, double lam_L, double lam_T, int penalize_diag,
                    double tie_eps, const ActWs& ws, int32_t* L_row, int32_t* L_col, int32_t* T_row, int32_t* T_col,
                    long long capL, long long capT);

// Coordinate-descent consumers (cd.cu), fp64
void lambda_cd(Ctx* c, int q, const double* S, int64_t lds, const double* P, int64_t ldp, const double* G, int64_t ldg,
               const cggm_csc* Lam, const int32_t* Lr, const int32_t* Lc, int64_t m, double lam, int penalize_diag,
               int passes, double* D, double* U, int64_t ldu, double* coef_ws /* 4m doubles */, double* out);
void theta_sigma(Ctx* c, int q, const cggm_csc* Th, const double* S, int64_t lds, double* V, int64_t ldv);
void theta_cd(Ctx* c, int p, int q, const double* S, int64_t lds, const double* Sxx, int64_t ldx, const int32_t* xmap,
              const double* Sxy,
              int64_t ldxy, const cggm_csc* Th, const int32_t* Tr, const int32_t* Tc, int64_t m, double lam, int passes,
              double* T, double* V, int64_t ldv, double* coef_ws /* 2m doubles */, double* out);
bool coop_ok(Ctx* c);
// NEXT-2 on-demand S_xx columns: xmap[i] = position of row i among the distinct rows of the list
// T_row[0..m) in ascending order (-1 if absent), rows[0..count) those rows, *count_dev their number
void row_map(Ctx* c, int p, const int32_t* T_row, int64_t m, int32_t* xmap, int32_t* rows, long long* count_dev);
// G (n x k, ldg) = X[:, rows[0..k)]
void gather_cols(Ctx* c, int64_t n, int64_t k, const double* X, int64_t ldx, const int32_t* rows, double* G, int64_t ldg);
void lambda_cd_coop(Ctx* c, int q, const double* S, int64_t lds, const double* P, int64_t ldp, const double* G,
                    int64_t ldg, const cggm_csc* Lam, const int32_t* Lr, const int32_t* Lc, int64_t m, double lam,
                    int penalize_diag, int passes, double* D, double* U, double* Z, int64_t ldu, double* coef_ws,
                    int* cnt, int64_t* scr, int64_t* lp, double* dmu, double* colbuf, double* out);
void theta_cd_coop(Ctx* c, int p, int q, const double* S, int64_t lds, const double* Sxx, int64_t ldx,
                   const int32_t* xmap, const double* Sxy, int64_t ldxy, const cggm_csc* Th, const int32_t* Tr, const int32_t* Tc, int64_t m,
                   double lam, int passes, double* T, double* V, int64_t ldv, double* coef_ws, int* cnt, int64_t* scr,
                   int64_t* lp, double* dmu, double* colbuf, double* out);
// sorted list (column-major) -> CSC: mirror = symmetric Lambda + alpha D from the upper-triangle list
// (values base_ij + alpha D[k]); otherwise the list itself with `vals`.  cnt_ws: 3n ints, scan_ws:
// 2(n+1) int64.
void list_to_csc(Ctx* c, int n, const int32_t* r, const int32_t* cidx, int64_t m, bool mirror, const cggm_csc* base,
                 const double* D, double alpha, const double* vals, int64_t* out_colptr, int32_t* out_row,
                 double* out_val, int* cnt_ws, int64_t* scan_ws);

}  // namespace cggm
