/*
 * CGGM hot-path ORACLE, second form: plain C loops, fp64, no BLAS / LAPACK.
 *
 * TEST INFRASTRUCTURE ONLY (like oracle/cggm_oracle.py): only tests/ load it (through
 * oracle/c_oracle.py); the product library shares no code with it.  An independent restatement of
 * the same definitions as the numpy oracle -- textbook loop nests, OpenMP only over independent
 * output entries -- so that the two oracles pin each other (tests/test_oracle_c.py)
 * besides the closed forms, and so that the CPU cost of the plain definition can be timed per phase
 * (cggm_oracle_c_eval).
 *
 * Layout: dense matrices column-major with leading dimension = rows; sparse matrices CSC with
 * int64 column pointers, int32 sorted row indices, double values (Lambda stores both triangles).
 * P:L = /root/reference/PAPER.md line L; readings A* are DESIGN.md §2.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#define AT(M, ld, i, j) ((M)[(size_t)(i) + (size_t)(j) * (size_t)(ld)])

static double now_s(void) {
  struct timespec t;
  clock_gettime(CLOCK_MONOTONIC, &t);
  return (double)t.tv_sec + 1e-9 * (double)t.tv_nsec;
}

/* O2: S_yy = Y^T Y / n (upper, mirrored: A19), S_xy = X^T Y / n */
void cggm_oracle_c_covariances(int64_t n, int64_t p, int64_t q, const double* X, const double* Y, double* Syy,
                               double* Sxy) {
#pragma omp parallel for schedule(dynamic)
  for (int64_t j = 0; j < q; ++j) {
    for (int64_t i = 0; i <= j; ++i) {
      double s = 0.0;
      for (int64_t k = 0; k < n; ++k) s += AT(Y, n, k, i) * AT(Y, n, k, j);
      AT(Syy, q, i, j) = s / (double)n;
      AT(Syy, q, j, i) = s / (double)n;
    }
    if (Sxy)
      for (int64_t i = 0; i < p; ++i) {
        double s = 0.0;
        for (int64_t k = 0; k < n; ++k) s += AT(X, n, k, i) * AT(Y, n, k, j);
        AT(Sxy, p, i, j) = s / (double)n;
      }
  }
}

/* O3: unblocked Cholesky Lambda = L L^T column by column; PD iff every pivot
 * d_j = Lambda_jj - sum_k L_jk^2 > 0 and finite (A10).  L lower, column-major.  Returns the first
 * failing column or -1. */
static int64_t cholesky(int64_t q, const double* A, double* L) {
  memset(L, 0, sizeof(double) * (size_t)q * (size_t)q);
  for (int64_t j = 0; j < q; ++j) {
    double d = AT(A, q, j, j);
    for (int64_t k = 0; k < j; ++k) d -= AT(L, q, j, k) * AT(L, q, j, k);
    if (!(d > 0.0) || !isfinite(d)) return j;
    const double ljj = sqrt(d);
    AT(L, q, j, j) = ljj;
#pragma omp parallel for
    for (int64_t i = j + 1; i < q; ++i) {
      double s = AT(A, q, i, j);
      for (int64_t k = 0; k < j; ++k) s -= AT(L, q, i, k) * AT(L, q, j, k);
      AT(L, q, i, j) = s / ljj;
    }
  }
  return -1;
}

/* O3/O4: log|Lambda| = 2 sum ln L_jj; Sigma = L^{-T} L^{-1}: L^{-1} by forward
 * substitution on the identity, column by column, then Sigma_ij = sum_k Linv_ki Linv_kj (upper,
 * mirrored).  Sigma may be NULL (PD test and log-det only). */
void cggm_oracle_c_invert_logdet(int64_t q, const double* Lam, double* Sigma, double* logdet, int* is_pd,
                                 int64_t* fail_col) {
  double* L = (double*)malloc(sizeof(double) * (size_t)q * (size_t)q);
  const int64_t f = cholesky(q, Lam, L);
  *fail_col = f;
  *is_pd = f < 0;
  *logdet = NAN;
  if (f >= 0) {
    free(L);
    return;
  }
  double ld = 0.0;
  for (int64_t j = 0; j < q; ++j) ld += log(AT(L, q, j, j));
  *logdet = 2.0 * ld;
  if (Sigma) {
    double* Li = (double*)calloc((size_t)q * (size_t)q, sizeof(double));
#pragma omp parallel for schedule(dynamic)
    for (int64_t c = 0; c < q; ++c) {   /* column c of L^{-1}: L z = e_c, rows c.. */
      for (int64_t i = c; i < q; ++i) {
        double s = (i == c) ? 1.0 : 0.0;
        for (int64_t k = c; k < i; ++k) s -= AT(L, q, i, k) * AT(Li, q, k, c);
        AT(Li, q, i, c) = s / AT(L, q, i, i);
      }
    }
#pragma omp parallel for schedule(dynamic)
    for (int64_t j = 0; j < q; ++j)
      for (int64_t i = 0; i <= j; ++i) {
        double s = 0.0;
        for (int64_t k = j; k < q; ++k) s += AT(Li, q, k, i) * AT(Li, q, k, j);   /* Linv_ki = 0 for k < i */
        AT(Sigma, q, i, j) = s;
        AT(Sigma, q, j, i) = s;
      }
    free(Li);
  }
  free(L);
}

/* O5-O7: W = X Theta, R = W Sigma / sqrt(n) (A11), Psi = R^T R (upper, mirrored),
 * grad_Lambda = S_yy - Sigma - Psi, grad_Theta = 2 S_xy + (2 / sqrt n) X^T R  (Eq. 3, P:264-269;
 * S_xy by its definition X^T Y / n). */
void cggm_oracle_c_psi_grad(int64_t n, int64_t p, int64_t q, const double* X, const double* Y,
                            const int64_t* tcp, const int32_t* tri, const double* tval, const double* Sigma,
                            const double* Syy, double* Psi, double* GradL, double* GradT) {
  double* W = (double*)calloc((size_t)n * (size_t)q, sizeof(double));
  double* R = (double*)malloc(sizeof(double) * (size_t)n * (size_t)q);
  const double rs = 1.0 / sqrt((double)n);
#pragma omp parallel for
  for (int64_t j = 0; j < q; ++j)
    for (int64_t t = tcp[j]; t < tcp[j + 1]; ++t)
      for (int64_t k = 0; k < n; ++k) AT(W, n, k, j) += tval[t] * AT(X, n, k, tri[t]);
#pragma omp parallel for
  for (int64_t j = 0; j < q; ++j)
    for (int64_t k = 0; k < n; ++k) {
      double s = 0.0;
      for (int64_t c = 0; c < q; ++c) s += AT(W, n, k, c) * AT(Sigma, q, c, j);
      AT(R, n, k, j) = s * rs;
    }
#pragma omp parallel for schedule(dynamic)
  for (int64_t j = 0; j < q; ++j)
    for (int64_t i = 0; i <= j; ++i) {
      double s = 0.0;
      for (int64_t k = 0; k < n; ++k) s += AT(R, n, k, i) * AT(R, n, k, j);
      AT(Psi, q, i, j) = s;
      AT(Psi, q, j, i) = s;
    }
#pragma omp parallel for
  for (int64_t j = 0; j < q; ++j)
    for (int64_t i = 0; i < q; ++i) AT(GradL, q, i, j) = AT(Syy, q, i, j) - AT(Sigma, q, i, j) - AT(Psi, q, i, j);
#pragma omp parallel for
  for (int64_t j = 0; j < q; ++j)
    for (int64_t i = 0; i < p; ++i) {
      double sxy = 0.0, xr = 0.0;
      for (int64_t k = 0; k < n; ++k) {
        sxy += AT(X, n, k, i) * AT(Y, n, k, j);
        xr += AT(X, n, k, i) * AT(R, n, k, j);
      }
      AT(GradT, p, i, j) = 2.0 * (sxy / (double)n) + 2.0 * rs * xr;
    }
  free(W);
  free(R);
}

static double csc_value(const int64_t* cp, const int32_t* ri, const double* v, int64_t i, int64_t j) {
  for (int64_t t = cp[j]; t < cp[j + 1]; ++t)
    if (ri[t] == i) return v[t];
  return 0.0;
}

/* O8/O9: the active sets (A5 strict '>', A6 Lambda pairs i <= j once, column-major
 * order, A7 value test) with counts, tie counts, and ||grad^S||_1 (A9: both
 * triangles of Lambda, all of Theta; lambda_ii = 0 for an unpenalised diagonal).  The row / col
 * outputs may be NULL (counts only); otherwise they must hold m_L / m_T entries. */
void cggm_oracle_c_active_set(int64_t p, int64_t q, const double* GradL, const double* GradT, const int64_t* lcp,
                              const int32_t* lri, const double* lval, const int64_t* tcp, const int32_t* tri,
                              const double* tval, double lam_L, double lam_T, int penalize_diag, double tie_eps,
                              int64_t* m_L, int64_t* m_T, int64_t* ties_L, int64_t* ties_T, double* subgrad,
                              int32_t* L_row, int32_t* L_col, int32_t* T_row, int32_t* T_col) {
  int64_t mL = 0, mT = 0, tL = 0, tT = 0;
  double sub = 0.0;
  for (int64_t j = 0; j < q; ++j)
    for (int64_t i = 0; i < q; ++i) {
      const double g = AT(GradL, q, i, j), x = csc_value(lcp, lri, lval, i, j);
      const double lm = (i == j && !penalize_diag) ? 0.0 : lam_L;
      sub += (x != 0.0) ? fabs(g + lm * (x > 0.0 ? 1.0 : -1.0)) : fmax(fabs(g) - lm, 0.0);
      if (i > j) continue;
      if (fabs(g) > lm || x != 0.0) {
        if (L_row) {
          L_row[mL] = (int32_t)i;
          L_col[mL] = (int32_t)j;
        }
        ++mL;
      }
      if (x == 0.0 && fabs(fabs(g) - lm) <= tie_eps) ++tL;
    }
  for (int64_t j = 0; j < q; ++j)
    for (int64_t i = 0; i < p; ++i) {
      const double g = AT(GradT, p, i, j), x = csc_value(tcp, tri, tval, i, j);
      sub += (x != 0.0) ? fabs(g + lam_T * (x > 0.0 ? 1.0 : -1.0)) : fmax(fabs(g) - lam_T, 0.0);
      if (fabs(g) > lam_T || x != 0.0) {
        if (T_row) {
          T_row[mT] = (int32_t)i;
          T_col[mT] = (int32_t)j;
        }
        ++mT;
      }
      if (x == 0.0 && fabs(fabs(g) - lam_T) <= tie_eps) ++tT;
    }
  *m_L = mL;
  *m_T = mT;
  *ties_L = tL;
  *ties_T = tT;
  *subgrad = sub;
}

/* O10: f = -log|Lambda| + tr(S_yy Lambda) + 2 tr(S_xy^T Theta) + tr(Lambda^{-1} Theta^T S_xx Theta)
 *        + lam_L ||Lambda||_1 + lam_T ||Theta||_1   (Eq. 1; A3 / A4 for the penalty)
 * with tr(Lambda^{-1} Theta^T S_xx Theta) = ||L^{-1} W^T||_F^2 / n, W = X Theta (A14): the columns
 * of W^T solved against L by forward substitution.  Non-PD Lambda: f = +inf. */
void cggm_oracle_c_objective(int64_t n, int64_t p, int64_t q, const double* X, const double* Y, const int64_t* lcp,
                             const int32_t* lri, const double* lval, const int64_t* tcp, const int32_t* tri,
                             const double* tval, double lam_L, double lam_T, int penalize_diag, double* f,
                             double* logdet, int* is_pd) {
  double* Lam = (double*)calloc((size_t)q * (size_t)q, sizeof(double));
  for (int64_t j = 0; j < q; ++j)
    for (int64_t t = lcp[j]; t < lcp[j + 1]; ++t) AT(Lam, q, lri[t], j) = lval[t];
  double* L = (double*)malloc(sizeof(double) * (size_t)q * (size_t)q);
  const int64_t fc = cholesky(q, Lam, L);
  double pen = 0.0;
  for (int64_t j = 0; j < q; ++j)
    for (int64_t t = lcp[j]; t < lcp[j + 1]; ++t)
      if (!(lri[t] == j && !penalize_diag)) pen += lam_L * fabs(lval[t]);
  for (int64_t j = 0; j < q; ++j)
    for (int64_t t = tcp[j]; t < tcp[j + 1]; ++t) pen += lam_T * fabs(tval[t]);
  *is_pd = fc < 0;
  if (fc >= 0) {
    *f = INFINITY;
    *logdet = NAN;
    free(Lam);
    free(L);
    return;
  }
  double ld = 0.0;
  for (int64_t j = 0; j < q; ++j) ld += log(AT(L, q, j, j));
  ld *= 2.0;
  double tr_syy = 0.0, tr_sxy = 0.0, tr_m = 0.0;
  for (int64_t j = 0; j < q; ++j)
    for (int64_t t = lcp[j]; t < lcp[j + 1]; ++t) {
      double s = 0.0;
      for (int64_t k = 0; k < n; ++k) s += AT(Y, n, k, lri[t]) * AT(Y, n, k, j);
      tr_syy += lval[t] * s / (double)n;
    }
  for (int64_t j = 0; j < q; ++j)
    for (int64_t t = tcp[j]; t < tcp[j + 1]; ++t) {
      double s = 0.0;
      for (int64_t k = 0; k < n; ++k) s += AT(X, n, k, tri[t]) * AT(Y, n, k, j);
      tr_sxy += tval[t] * s / (double)n;
    }
#pragma omp parallel for reduction(+ : tr_m) schedule(dynamic)
  for (int64_t k = 0; k < n; ++k) {   /* row k of W: w_j = sum_t Theta_tj X_kt; solve L z = w^T */
    double* z = (double*)malloc(sizeof(double) * (size_t)q);
    for (int64_t j = 0; j < q; ++j) {
      double w = 0.0;
      for (int64_t t = tcp[j]; t < tcp[j + 1]; ++t) w += tval[t] * AT(X, n, k, tri[t]);
      z[j] = w;
    }
    for (int64_t i = 0; i < q; ++i) {
      double s = z[i];
      for (int64_t c = 0; c < i; ++c) s -= AT(L, q, i, c) * z[c];
      z[i] = s / AT(L, q, i, i);
    }
    double acc = 0.0;
    for (int64_t i = 0; i < q; ++i) acc += z[i] * z[i];
    tr_m += acc;
    free(z);
  }
  tr_m /= (double)n;
  *logdet = ld;
  *f = -ld + tr_syy + 2.0 * tr_sxy + tr_m + pen;
  free(Lam);
  free(L);
}

/* One evaluation of the hot path at (Lambda, Theta) in the plain-loop form, per-phase seconds in
 * secs[0..4] = {invert_logdet, psi_grad, active_set, objective, covariances} (the covariance
 * phase is the per-dataset setup).  Outputs as the calls above; f, logdet, statistic, list sizes
 * returned through the pointers. */
void cggm_oracle_c_eval(int64_t n, int64_t p, int64_t q, const double* X, const double* Y, const int64_t* lcp,
                        const int32_t* lri, const double* lval, const int64_t* tcp, const int32_t* tri,
                        const double* tval, double lam_L, double lam_T, int penalize_diag, double* f,
                        double* logdet, int64_t* m_L, int64_t* m_T, double* subgrad, double* secs) {
  const size_t qq = (size_t)q * (size_t)q;
  double* Syy = (double*)malloc(sizeof(double) * qq);
  double* Lam = (double*)calloc(qq, sizeof(double));
  double* Sig = (double*)malloc(sizeof(double) * qq);
  double* Psi = (double*)malloc(sizeof(double) * qq);
  double* GL = (double*)malloc(sizeof(double) * qq);
  double* GT = (double*)malloc(sizeof(double) * (size_t)p * (size_t)q);
  double t0 = now_s();
  cggm_oracle_c_covariances(n, 0, q, X, Y, Syy, NULL);
  secs[4] = now_s() - t0;
  for (int64_t j = 0; j < q; ++j)
    for (int64_t t = lcp[j]; t < lcp[j + 1]; ++t) AT(Lam, q, lri[t], j) = lval[t];
  int pd;
  int64_t fc, tl, tt;
  t0 = now_s();
  cggm_oracle_c_invert_logdet(q, Lam, Sig, logdet, &pd, &fc);
  secs[0] = now_s() - t0;
  t0 = now_s();
  if (pd) cggm_oracle_c_psi_grad(n, p, q, X, Y, tcp, tri, tval, Sig, Syy, Psi, GL, GT);
  secs[1] = now_s() - t0;
  t0 = now_s();
  if (pd)
    cggm_oracle_c_active_set(p, q, GL, GT, lcp, lri, lval, tcp, tri, tval, lam_L, lam_T, penalize_diag, 1e-9, m_L,
                             m_T, &tl, &tt, subgrad, NULL, NULL, NULL, NULL);
  secs[2] = now_s() - t0;
  t0 = now_s();
  double ld2;
  int pd2;
  cggm_oracle_c_objective(n, p, q, X, Y, lcp, lri, lval, tcp, tri, tval, lam_L, lam_T, penalize_diag, f, &ld2, &pd2);
  secs[3] = now_s() - t0;
  free(Syy);
  free(Lam);
  free(Sig);
  free(Psi);
  free(GL);
  free(GT);
}
