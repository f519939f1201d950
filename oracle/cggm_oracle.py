"""CGGM hot-path ORACLE — plain, slow, obviously-correct CPU fp64 definitions.

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
`cpu_baseline` / `--impl reference` legs may import or execute anything under `oracle/`.
The product path (`paper_1509_04681_b200`) never imports it and shares no code with it.

Every function follows a passage of PAPER.md (`/root/reference/PAPER.md`, cited as P:line)
or a reading listed in DESIGN.md §"Readings".  Library primitives used as single steps:
numpy matmul (matrix products that ARE the definition, e.g. S_yy = Y^T Y / n), sqrt/log.
The Cholesky factorisation, the triangular inverse and the triangular solve are written
out as the textbook column algorithms (no blocking, no reordering).

Pins (tests/test_oracle_pins.py, `-m "not gpu"`): P1 scalar worked example (SPEC S:151,
S:161), P2 (I,0) closed form, P3/P4/P5 chain closed forms (logdet, Sigma, PD boundary),
P6 SPEC logdet examples, P7 Sigma Lambda = I, P8 central finite differences, P9 Psi PSD and
explicit-S_xx route, P10 trace identities, P11 two gradient routes, P12 active-set examples,
P13 1x1 optimum and a hand-worked q = 3 ||grad^S||_1 (both triangles, unpenalised
diagonal), P14 convexity, P15 eigenvalue logdet / library inverse, P16 generating-point
identity I7, P17 shard partial sums, plus a density-based pin of g (multivariate normal
log-likelihood, reading A1).  Tie-band entries of the active sets are "parity unpinned" by
design (excluded from comparisons and counted).
"""
from __future__ import annotations

import math
import numpy as np

__all__ = [
    "covariances", "cholesky", "logdet_from_cholesky", "inverse_from_cholesky",
    "invert_logdet", "spmm_x_theta", "psi_grad", "grad_theta_residual_route",
    "active_set", "min_norm_subgradient", "objective", "forward_substitution",
]


def _mirror_upper(A: np.ndarray) -> np.ndarray:
    """Full symmetric matrix from the upper triangle (reading A19: both triangles bit-identical)."""
    U = np.triu(A)
    return np.asfortranarray(U + np.triu(A, 1).T)


# ---------------------------------------------------------------- O2: sample covariances
def covariances(X: np.ndarray, Y: np.ndarray, n_total: int | None = None):
    """S_yy = Y^T Y / n, S_xy = X^T Y / n  (§2.1).  `n_total` is the global
    sample count used in every 1/n (reading A21); with X, Y a row shard this is the shard's
    partial sum."""
    n = X.shape[0] if n_total is None else n_total
    Syy = _mirror_upper((Y.T @ Y) / n)
    Sxy = np.asfortranarray((X.T @ Y) / n)
    return Syy, Sxy


# ---------------------------------------------------------------- O3: Cholesky + logdet
def cholesky(A: np.ndarray):
    """Unblocked Cholesky A = L L^T, column by column (§2.3 "via Cholesky
    decomposition"; SPEC S:45-54 contract).  Reading A10: PD iff every pivot
    d_j = A_jj - sum_{k<j} L_jk^2 is > 0 (and finite); otherwise return the first failing
    column j.  Returns (L lower-triangular, is_pd, fail_col) with fail_col = -1 when PD."""
    q = A.shape[0]
    A = np.asarray(A, dtype=np.float64)
    L = np.zeros((q, q), dtype=np.float64)            # C order: rows contiguous
    for j in range(q):
        d = A[j, j] - np.dot(L[j, :j], L[j, :j])
        if not (d > 0.0) or not math.isfinite(d):
            return L, False, j
        ljj = math.sqrt(d)
        L[j, j] = ljj
        if j + 1 < q:
            L[j + 1:, j] = (A[j + 1:, j] - L[j + 1:, :j] @ L[j, :j]) / ljj
    return L, True, -1


def logdet_from_cholesky(L: np.ndarray) -> float:
    """log|Lambda| = 2 sum_j ln L_jj (natural log, reading A10)."""
    return float(2.0 * np.sum(np.log(np.diag(L))))


def forward_substitution(L: np.ndarray, B: np.ndarray) -> np.ndarray:
    """Solve L Z = B for lower-triangular L, row by row (textbook forward substitution)."""
    q = L.shape[0]
    Z = np.zeros((q, B.shape[1]), dtype=np.float64)
    for i in range(q):
        Z[i, :] = (B[i, :] - L[i, :i] @ Z[:i, :]) / L[i, i]
    return Z


def inverse_from_cholesky(L: np.ndarray) -> np.ndarray:
    """Sigma = Lambda^{-1} = L^{-T} L^{-1}.  L^{-1} by forward substitution on the
    identity (row i of L^{-1} is zero beyond column i), then the product, upper mirrored."""
    q = L.shape[0]
    Linv = np.zeros((q, q), dtype=np.float64)
    for i in range(q):
        rhs = np.zeros(i + 1)
        rhs[i] = 1.0
        Linv[i, :i + 1] = (rhs - L[i, :i] @ Linv[:i, :i + 1]) / L[i, i]
    return _mirror_upper(Linv.T @ Linv)


def invert_logdet(Lam: np.ndarray, want_sigma: bool = True):
    """cggm_invert_logdet: (Sigma or None, logdet, is_pd, fail_col)."""
    L, ok, fail = cholesky(Lam)
    if not ok:
        return None, float("nan"), False, fail
    ld = logdet_from_cholesky(L)
    return (inverse_from_cholesky(L) if want_sigma else None), ld, True, -1


# ---------------------------------------------------------------- O5: W = X Theta
def spmm_x_theta(X: np.ndarray, theta) -> np.ndarray:
    """W[:, j] += Theta_ij X[:, i] for each stored Theta_ij (R = X Theta Sigma)."""
    n = X.shape[0]
    W = np.zeros((n, theta.ncols), order="F")
    for j in range(theta.ncols):
        a, b = theta.colptr[j], theta.colptr[j + 1]
        for t in range(a, b):
            W[:, j] += theta.val[t] * X[:, theta.rowidx[t]]
    return W


# ---------------------------------------------------------------- O6/O7: R, Psi, gradients
def psi_grad(X, Y, theta, Sigma, Syy, Sxy=None, n_total=None):
    """R = X Theta Sigma / sqrt(n) (reading A11), Psi = R^T R,
    grad_Lambda = S_yy - Sigma - Psi and grad_Theta = 2 S_xy + 2 S_xx Theta Sigma (Eq. 3,
    P:264-269) with S_xx Theta Sigma = X^T R / sqrt(n) (S_xx never formed, north_star (1)).
    If Sxy is None it is formed here by its definition X^T Y / n."""
    n = X.shape[0] if n_total is None else n_total
    W = spmm_x_theta(X, theta)
    R = np.asfortranarray((W @ Sigma) / math.sqrt(n))
    Psi = _mirror_upper(R.T @ R)
    GradL = np.asfortranarray(Syy - Sigma - Psi)
    if Sxy is None:
        Sxy = np.asfortranarray((X.T @ Y) / n)
    GradT = np.asfortranarray(2.0 * Sxy + (2.0 / math.sqrt(n)) * (X.T @ R))
    return dict(W=W, R=R, Psi=Psi, GradL=GradL, GradT=GradT)


def grad_theta_residual_route(X, Y, W, Sigma, n_total=None):
    """Second route (identity I3): grad_Theta = (2/n) X^T (Y + W Sigma)."""
    n = X.shape[0] if n_total is None else n_total
    E = Y + W @ Sigma
    return np.asfortranarray((2.0 / n) * (X.T @ E)), E


# ---------------------------------------------------------------- O8: active sets
def _support_dense(csc, shape):
    """Value test of reading A7: stored entries with value != 0."""
    S = np.zeros(shape, dtype=bool)
    for j in range(csc.ncols):
        a, b = csc.colptr[j], csc.colptr[j + 1]
        rows = csc.rowidx[a:b]
        vals = csc.val[a:b]
        S[rows[vals != 0], j] = True
    return S


def active_set(GradL, GradT, lam_csc, theta_csc, lam_L, lam_T, penalize_diag=True, tie_eps=1e-9):
    """S_Lambda = {(i,j), i<=j : |grad_L,ij| > lam_L or Lambda_ij != 0},
    S_Theta = {(i,j) : |grad_T,ij| > lam_T or Theta_ij != 0}  (§2.2).
    Reading A5: strict '>'; A6: Lambda pairs reported once (i <= j), both lists in ascending
    column-major order; unpenalised diagonal means lambda_ii = 0.  Tie band: entries not
    forced by the support with ||grad| - lambda| <= tie_eps are flagged."""
    q = GradL.shape[0]
    p = GradT.shape[0]
    lamM = np.full((q, q), float(lam_L))
    if not penalize_diag:
        np.fill_diagonal(lamM, 0.0)
    suppL = _support_dense(lam_csc, (q, q))
    suppT = _support_dense(theta_csc, (p, q))
    aL = np.abs(GradL)
    aT = np.abs(GradT)
    actL = ((aL > lamM) | suppL) & np.triu(np.ones((q, q), dtype=bool))
    actT = (aT > lam_T) | suppT
    tieL = (~suppL) & (np.abs(aL - lamM) <= tie_eps) & np.triu(np.ones((q, q), dtype=bool))
    tieT = (~suppT) & (np.abs(aT - lam_T) <= tie_eps)
    cL, rL = np.nonzero(actL.T)   # column-major order: sorted by column then row
    cT, rT = np.nonzero(actT.T)
    return dict(L_row=rL.astype(np.int32), L_col=cL.astype(np.int32),
                T_row=rT.astype(np.int32), T_col=cT.astype(np.int32),
                m_L=int(rL.size), m_T=int(rT.size),
                ties_L=int(tieL.sum()), ties_T=int(tieT.sum()),
                tie_mask_L=tieL, tie_mask_T=tieT)


# ---------------------------------------------------------------- O9: stopping statistic
def min_norm_subgradient(GradL, GradT, lam_csc, theta_csc, lam_L, lam_T, penalize_diag=True):
    """||grad^S||_1 (§5.1; SPEC S:183 per-coordinate rule, reading A9): sum over
    all Lambda entries (both triangles) and all Theta entries of |g + lam sign(x)| if x != 0
    else max(|g| - lam, 0)."""
    q = GradL.shape[0]
    p = GradT.shape[0]
    Ld = lam_csc.to_dense()
    Td = theta_csc.to_dense()
    lamM = np.full((q, q), float(lam_L))
    if not penalize_diag:
        np.fill_diagonal(lamM, 0.0)
    lamT = np.full((p, q), float(lam_T))

    def part(G, Xv, lm):
        nz = Xv != 0
        return float(np.sum(np.where(nz, np.abs(G + lm * np.sign(Xv)), np.maximum(np.abs(G) - lm, 0.0))))

    return part(GradL, Ld, lamM) + part(GradT, Td, lamT)


# ---------------------------------------------------------------- O10: objective
def objective(X, Y, lam_csc, theta_csc, lam_L, lam_T, penalize_diag=True, n_total=None, W=None):
    """f = g + h (Eq. 1):
        g = -log|Lambda| + tr(S_yy Lambda) + 2 tr(S_xy^T Theta) + tr(Lambda^{-1} Theta^T S_xx Theta)
        h = lam_L ||Lambda||_1 + lam_T ||Theta||_1   (elementwise, reading A4; diagonal per A3)
    tr(S_yy Lambda) and tr(S_xy^T Theta) are sums over the stored entries with S entries by
    definition (1/n) y_i . y_j and (1/n) x_i . y_j; tr(Sigma Theta^T S_xx Theta) =
    ||L^{-1} W^T||_F^2 / n with W = X Theta (reading A14).  The Cholesky is the PD test of the
    line search: a non-PD Lambda gives f = g = +inf."""
    n = X.shape[0] if n_total is None else n_total
    q = lam_csc.nrows
    Lam = lam_csc.to_dense()
    L, ok, fail = cholesky(Lam)
    penL = 0.0
    for j in range(q):
        a, b = lam_csc.colptr[j], lam_csc.colptr[j + 1]
        for t in range(a, b):
            i = lam_csc.rowidx[t]
            if i == j and not penalize_diag:
                continue
            penL += abs(lam_csc.val[t])
    penL *= lam_L
    penT = lam_T * float(np.sum(np.abs(theta_csc.val)))
    if not ok:
        return dict(f=math.inf, g=math.inf, logdet=float("nan"), is_pd=False, fail_col=fail,
                    tr_syy_lam=float("nan"), tr_sxy_theta=float("nan"), tr_sigma_m=float("nan"),
                    pen_L=penL, pen_T=penT)
    logdet = logdet_from_cholesky(L)
    tr_syy_lam = 0.0
    for j in range(q):
        a, b = lam_csc.colptr[j], lam_csc.colptr[j + 1]
        rows = lam_csc.rowidx[a:b]
        s = (Y[:, rows] * Y[:, [j]]).sum(axis=0) / n
        tr_syy_lam += float(np.dot(s, lam_csc.val[a:b]))
    tr_sxy_theta = 0.0
    for j in range(theta_csc.ncols):
        a, b = theta_csc.colptr[j], theta_csc.colptr[j + 1]
        rows = theta_csc.rowidx[a:b]
        s = (X[:, rows] * Y[:, [j]]).sum(axis=0) / n
        tr_sxy_theta += float(np.dot(s, theta_csc.val[a:b]))
    if W is None:
        W = spmm_x_theta(X, theta_csc)
    Z = forward_substitution(L, np.ascontiguousarray(W.T))
    tr_sigma_m = float(np.sum(Z * Z)) / n
    g = -logdet + tr_syy_lam + 2.0 * tr_sxy_theta + tr_sigma_m
    return dict(f=g + penL + penT, g=g, logdet=logdet, is_pd=True, fail_col=-1,
                tr_syy_lam=tr_syy_lam, tr_sxy_theta=tr_sxy_theta, tr_sigma_m=tr_sigma_m,
                pen_L=penL, pen_T=penT)
