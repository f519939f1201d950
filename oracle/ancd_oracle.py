"""ORACLE for the coordinate-descent consumers of the hot path:
the Lambda Newton-direction sweep with its Armijo line search, the direct Theta sweep, and the
alternating outer loop (Algorithm 1, `alg:Fast-alg`).  Plain numpy fp64, one
coordinate at a time, in the paper's order and notation.

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU legs may
import it; the product path never does and shares no code with it.

Readings:
  A15  the appendix coefficients are garbled.  Derived here from the Hessian
       Sigma (x) (Sigma + 2 Psi) of Eq. (4) along the symmetric coordinate direction
       E = e_i e_j^T + e_j e_i^T (Delta stays symmetric):
         i != j: a_L = S_ij^2 + S_ii S_jj + S_ii P_jj + S_jj P_ii + 2 S_ij P_ij
         i == j: a_L = S_ii^2 + 2 S_ii P_ii
       b_L = (GradL)_ij + (Sigma D Sigma)_ij + (Psi D Sigma)_ij + (Psi D Sigma)_ji   (as printed)
       and for Theta, from g_Lambda(Theta) of Eq. (7): a_T = 2 Sigma_jj (S_xx)_ii (printed without
       the 2), b_T = 2 (S_xy)_ij + 2 (S_xx Theta Sigma)_ij (as printed).  With these the printed
       update  x <- x - c + S_{lam/a}(c - b/a)  is the exact minimiser along the coordinate
       (pinned by brute force, tests/test_oracle_ancd.py).
  A16  Armijo constants beta = 0.5, sigma = 1e-4, at most 30 backtracks; decrease measure
       delta = tr(GradL^T D) + lam_L (||Lambda + D||_1 - ||Lambda||_1).
  A23  one active-set selection per outer iteration, used by both steps; the Theta
       step uses Sigma of the updated Lambda (Eq. 7 "with Lambda fixed"); one pass
       over each active set per outer iteration; stop when
       ||grad^S||_1 < 0.01 (||Lambda||_1 + ||Theta||_1).
"""
from __future__ import annotations

import math

import numpy as np

from . import cggm_oracle as O

__all__ = ["soft_threshold", "lambda_cd_a", "lambda_newton_direction", "lambda_surrogate",
           "armijo_lambda", "theta_cd_a", "theta_cd_sweep", "theta_subproblem", "ancd_fit",
           "prox_grad_fit", "objective_dense"]


def soft_threshold(w: float, r: float) -> float:
    """S_r(w) = sign(w) max(|w| - r, 0) (appendix)."""
    return math.copysign(max(abs(w) - r, 0.0), w) if w != 0.0 else 0.0


# ---------------------------------------------------------------- NEXT-1: Lambda step
def lambda_cd_a(Sigma, Psi, i, j) -> float:
    """Second-order coefficient a_Lambda of coordinate (i, j) (reading A15)."""
    if i == j:
        return Sigma[i, i] ** 2 + 2.0 * Sigma[i, i] * Psi[i, i]
    return (Sigma[i, j] ** 2 + Sigma[i, i] * Sigma[j, j] + Sigma[i, i] * Psi[j, j] + Sigma[j, j] * Psi[i, i]
            + 2.0 * Sigma[i, j] * Psi[i, j])


def lambda_newton_direction(Sigma, Psi, GradL, Lam, rows, cols, lam_L, penalize_diag=True, passes=1,
                            Delta=None):
    """D_Lambda of Eq. (6): coordinate descent over S_Lambda (pairs i <= j, in the given
    order), `passes` sweeps (a single pass), maintaining U = Delta Sigma:
        b = GradL_ij + Sigma_i . U[:, j] + Psi_i . U[:, j] + Psi_j . U[:, i]
        c = Lambda_ij + Delta_ij
        mu = -c + S_{lam/a}(c - b/a);   Delta_ij = Delta_ji += mu
        U[i, :] += mu Sigma[j, :];  U[j, :] += mu Sigma[i, :]   (once when i == j)
    Returns (Delta dense symmetric, U, list of the entries' final Delta values)."""
    q = Sigma.shape[0]
    D = np.zeros((q, q)) if Delta is None else np.array(Delta, dtype=np.float64)
    U = D @ Sigma
    for _ in range(passes):
        for i, j in zip(rows, cols):
            i, j = int(i), int(j)
            a = lambda_cd_a(Sigma, Psi, i, j)
            b = GradL[i, j] + float(np.dot(Sigma[i, :], U[:, j])) + float(np.dot(Psi[i, :], U[:, j])) \
                + float(np.dot(Psi[j, :], U[:, i]))
            c = Lam[i, j] + D[i, j]
            lam = 0.0 if (i == j and not penalize_diag) else lam_L
            if not (a > 0.0):
                continue   # numerically degenerate coordinate: skipped
            mu = -c + soft_threshold(c - b / a, lam / a)
            if mu == 0.0:
                continue
            D[i, j] += mu
            if i != j:
                D[j, i] += mu
                U[i, :] += mu * Sigma[j, :]
                U[j, :] += mu * Sigma[i, :]
            else:
                U[i, :] += mu * Sigma[i, :]
    vals = np.array([D[int(i), int(j)] for i, j in zip(rows, cols)])
    return D, U, vals


def lambda_surrogate(D, GradL, Sigma, Psi, Lam, lam_L, penalize_diag=True) -> float:
    """gbar(D) + lam_L ||Lambda + D||_1 of Eq. (6): tr(GradL D) + 1/2 tr(D S D S) + tr(D S D P)
    (the Hessian of Eq. 4 as a quadratic form on symmetric D) + the elementwise penalty."""
    lamM = np.full(Lam.shape, float(lam_L))
    if not penalize_diag:
        np.fill_diagonal(lamM, 0.0)
    DS = D @ Sigma
    return float(np.sum(GradL * D) + 0.5 * np.trace(DS @ DS) + np.trace(DS @ D @ Psi)
                 + np.sum(lamM * np.abs(Lam + D)))


def _l1(M, lam, penalize_diag):
    lamM = np.full(M.shape, float(lam))
    if not penalize_diag and M.shape[0] == M.shape[1]:
        np.fill_diagonal(lamM, 0.0)
    return float(np.sum(lamM * np.abs(M)))


def objective_dense(X, Y, Lam, Theta, lam_L, lam_T, penalize_diag=True) -> float:
    """f of Eq. (1) for dense Lambda / Theta through the oracle's objective (O10); +inf if not PD."""
    from synth.cggm_inputs import csc_from_dense
    return O.objective(X, Y, csc_from_dense(Lam), csc_from_dense(Theta), lam_L, lam_T, penalize_diag)["f"]


def armijo_lambda(X, Y, Lam, Theta, D, GradL, lam_L, lam_T, penalize_diag=True, f0=None, beta=0.5, sigma=1e-4,
                  max_backtracks=30):
    """Line search of Algorithm 1 (Armijo's rule P:242, P:287-288 'sufficient decrease ...
    and positive definiteness'): the largest alpha in {1, beta, beta^2, ...} with Lambda + alpha D PD
    (Cholesky succeeds inside the objective) and f(Lambda + alpha D) <= f0 + sigma alpha delta."""
    if f0 is None:
        f0 = objective_dense(X, Y, Lam, Theta, lam_L, lam_T, penalize_diag)
    delta = float(np.sum(GradL * D)) + _l1(Lam + D, lam_L, penalize_diag) - _l1(Lam, lam_L, penalize_diag)
    alpha = 1.0
    for k in range(max_backtracks + 1):
        Lt = Lam + alpha * D
        ft = objective_dense(X, Y, Lt, Theta, lam_L, lam_T, penalize_diag)
        if math.isfinite(ft) and ft <= f0 + sigma * alpha * delta:
            return dict(alpha=alpha, Lam=Lt, f=ft, backtracks=k, delta=delta)
        alpha *= beta
    return dict(alpha=0.0, Lam=Lam, f=f0, backtracks=max_backtracks + 1, delta=delta)


# ---------------------------------------------------------------- NEXT-2: Theta step
def theta_cd_a(Sigma, Sxx, i, j) -> float:
    """a_Theta = 2 Sigma_jj (S_xx)_ii (reading A15)."""
    return 2.0 * Sigma[j, j] * Sxx[i, i]


def theta_cd_sweep(Sigma, Sxx, Sxy, Theta, rows, cols, lam_T, passes=1):
    """Eq. (7) by coordinate descent over S_Theta (given order), `passes` sweeps,
    maintaining V = Theta Sigma:
        b = 2 (S_xy)_ij + 2 (S_xx)_i . V[:, j];  c = Theta_ij
        mu = -c + S_{lam/a}(c - b/a);  Theta_ij += mu;  V[i, :] += mu Sigma[j, :]
    Returns (Theta dense, V)."""
    T = np.array(Theta, dtype=np.float64)
    V = T @ Sigma
    for _ in range(passes):
        for i, j in zip(rows, cols):
            i, j = int(i), int(j)
            a = theta_cd_a(Sigma, Sxx, i, j)
            if not (a > 0.0):
                continue   # constant input column (S_xx)_ii = 0
            b = 2.0 * Sxy[i, j] + 2.0 * float(np.dot(Sxx[i, :], V[:, j]))
            c = T[i, j]
            mu = -c + soft_threshold(c - b / a, lam_T / a)
            if mu == 0.0:
                continue
            T[i, j] += mu
            V[i, :] += mu * Sigma[j, :]
    return T, V


def theta_subproblem(Theta, Sigma, Sxx, Sxy, lam_T) -> float:
    """g_Lambda(Theta) + lam_T ||Theta||_1 of Eq. (7): 2 tr(S_xy^T Theta) + tr(Sigma Theta^T S_xx Theta)."""
    return float(2.0 * np.sum(Sxy * Theta) + np.trace(Sigma @ Theta.T @ Sxx @ Theta) + lam_T * np.sum(np.abs(Theta)))


# ---------------------------------------------------------------- Algorithm 1
def ancd_fit(X, Y, lam_L, lam_T, penalize_diag=True, max_iter=200, tol=0.01, passes=1):
    """Alternating Newton coordinate descent (Algorithm 1) with the readings A16/A23.
    Returns dict(Lam, Theta, iters, f, history=[(f, ||grad^S||_1, m_L, m_T, alpha)])."""
    from synth.cggm_inputs import csc_from_dense
    n, p = X.shape
    q = Y.shape[1]
    Syy, Sxy = O.covariances(X, Y)
    Sxx = X.T @ X / n
    Lam = np.eye(q)
    Theta = np.zeros((p, q))
    hist = []
    f = objective_dense(X, Y, Lam, Theta, lam_L, lam_T, penalize_diag)
    for t in range(max_iter):
        lc, tc = csc_from_dense(Lam), csc_from_dense(Theta)
        Sigma, _, ok, _ = O.invert_logdet(Lam)
        r = O.psi_grad(X, Y, tc, Sigma, Syy, Sxy)
        stat = O.min_norm_subgradient(r["GradL"], r["GradT"], lc, tc, lam_L, lam_T, penalize_diag)
        scale = float(np.sum(np.abs(Lam)) + np.sum(np.abs(Theta)))
        act = O.active_set(r["GradL"], r["GradT"], lc, tc, lam_L, lam_T, penalize_diag)
        if stat < tol * scale:
            hist.append((f, stat, len(act["L_row"]), len(act["T_row"]), None))
            break
        D, _, _ = lambda_newton_direction(Sigma, r["Psi"], r["GradL"], Lam, act["L_row"], act["L_col"], lam_L,
                                          penalize_diag, passes)
        ls = armijo_lambda(X, Y, Lam, Theta, D, r["GradL"], lam_L, lam_T, penalize_diag, f0=f)
        Lam = ls["Lam"]
        Sigma, _, _, _ = O.invert_logdet(Lam)
        Theta, _ = theta_cd_sweep(Sigma, Sxx, Sxy, Theta, act["T_row"], act["T_col"], lam_T, passes)
        f = objective_dense(X, Y, Lam, Theta, lam_L, lam_T, penalize_diag)
        hist.append((f, stat, len(act["L_row"]), len(act["T_row"]), ls["alpha"]))
    return dict(Lam=Lam, Theta=Theta, iters=len(hist), f=f, history=hist)


def prox_grad_fit(X, Y, lam_L, lam_T, penalize_diag=True, max_iter=20000, tol=1e-10):
    """Independent reference solver: plain proximal gradient on (Lambda, Theta)
    jointly with backtracking on the step, rejecting non-PD Lambda; gradients of Eq. (3) from
    dense Sigma, Psi, Gamma.  No code shared with the coordinate-descent path above."""
    n, p = X.shape
    q = Y.shape[1]
    Syy = Y.T @ Y / n
    Sxy = X.T @ Y / n
    Sxx = X.T @ X / n
    lamM = np.full((q, q), float(lam_L))
    if not penalize_diag:
        np.fill_diagonal(lamM, 0.0)

    def smooth(L, T):
        w = np.linalg.eigvalsh(L)
        if w.min() <= 0:
            return math.inf
        Sig = np.linalg.inv(L)
        return float(-np.sum(np.log(w)) + np.sum(Syy * L) + 2 * np.sum(Sxy * T) + np.trace(Sig @ T.T @ Sxx @ T))

    def grads(L, T):
        Sig = np.linalg.inv(L)
        Gam = Sxx @ T @ Sig
        Psi = Sig @ T.T @ Gam
        return Syy - Sig - Psi, 2 * Sxy + 2 * Gam

    def st(M, r):
        return np.sign(M) * np.maximum(np.abs(M) - r, 0.0)

    L, T = np.eye(q), np.zeros((p, q))
    step = 1.0
    F = smooth(L, T) + float(np.sum(lamM * np.abs(L))) + lam_T * float(np.sum(np.abs(T)))
    for it in range(max_iter):
        gL, gT = grads(L, T)
        gL = 0.5 * (gL + gL.T)
        g0 = smooth(L, T)
        while True:
            Ln = st(L - step * gL, step * lamM)
            Ln = 0.5 * (Ln + Ln.T)
            Tn = st(T - step * gT, step * lam_T)
            gn = smooth(Ln, Tn)
            dL, dT = Ln - L, Tn - T
            quad = g0 + np.sum(gL * dL) + np.sum(gT * dT) + (np.sum(dL * dL) + np.sum(dT * dT)) / (2 * step)
            if math.isfinite(gn) and gn <= quad + 1e-15 * abs(quad):
                break
            step *= 0.5
            if step < 1e-20:
                break
        Fn = gn + float(np.sum(lamM * np.abs(Ln))) + lam_T * float(np.sum(np.abs(Tn)))
        L, T = Ln, Tn
        done = abs(F - Fn) <= tol * max(1.0, abs(Fn)) and np.max(np.abs(dL)) + np.max(np.abs(dT)) < 1e-9
        F = Fn
        step *= 1.5
        if done:
            break
    return dict(Lam=L, Theta=T, f=F, iters=it + 1)
