"""Algorithm 1 — alternating Newton coordinate descent (`alg:Fast-alg`) — driven through
the C-ABI.  Every numeric step runs in libcggm's kernels (Sigma / log-det by the recursive
Cholesky, Psi / gradients / active sets, the Lambda direction sweep, the line-search candidates
and their objectives, the Theta sweep); this loop only sequences the calls and takes the Armijo
accept / reject decision on the returned scalars (readings A16, A23 in DESIGN.md §2):

  for t = 0, 1, ...:
      Sigma = Lambda^{-1}; Psi, grad_Lambda, grad_Theta; S_Lambda, S_Theta, ||grad^S||_1  (one selection)
      D = Newton direction of Eq. (6) over S_Lambda (one pass, U = D Sigma)
      stop if ||grad^S||_1 < tol (||Lambda||_1 + ||Theta||_1)
      alpha = max{beta^k : Lambda + beta^k D PD and f <= f + sigma beta^k delta}
      Lambda <- Lambda + alpha D;  Sigma = Lambda^{-1}
      Theta <- one coordinate pass of Eq. (7) over S_Theta (V = Theta Sigma)

Factor reuse: every Lambda the loop keeps is factored once, into L^{-1} (cggm_chol_inverse_dense, the
recursive factorisation in full-inverse mode) -- a line-search trial's factorisation is its PD test
and its objective (cggm_objective_given_inverse: tr(Sigma M) = ||W L^{-T}||^2 / n, no second
factorisation), the accepted trial's L^{-1} gives Sigma = L^{-T} L^{-1} for the Theta step AND the next
iteration (one symmetric product), and the objective after the Theta step reuses it too.
S_xx on demand (sxx="rows", the default; the paper's (S_xx)_i rows): only the columns
X^T X_i / n of the rows i on the Theta active list are formed (cggm_gram_rows), never the p x p matrix.
"""
from __future__ import annotations

import dataclasses
import math

import torch

from .api import CggmError, Context, DeviceCsc, colmajor_empty

__all__ = ["AncdResult", "ancd_fit", "identity_csc", "empty_csc"]


def identity_csc(q: int, device="cuda") -> DeviceCsc:
    return DeviceCsc(q, q, torch.arange(q + 1, dtype=torch.int64, device=device),
                     torch.arange(q, dtype=torch.int32, device=device), torch.ones(q, dtype=torch.float64, device=device))


def empty_csc(p: int, q: int, device="cuda") -> DeviceCsc:
    return DeviceCsc(p, q, torch.zeros(q + 1, dtype=torch.int64, device=device),
                     torch.empty(0, dtype=torch.int32, device=device), torch.empty(0, dtype=torch.float64, device=device))


def _own(c: DeviceCsc) -> DeviceCsc:
    return DeviceCsc(c.nrows, c.ncols, c.colptr.clone(), c.rowidx.clone(), c.val.clone())


@dataclasses.dataclass
class AncdResult:
    Lam: DeviceCsc
    Theta: DeviceCsc
    f: float
    iters: int
    converged: bool
    history: list


def ancd_fit(ctx: Context, X, Y, lam_L, lam_T, penalize_diag=True, max_iter=100, tol=0.01, passes=1, beta=0.5,
             sigma=1e-4, max_backtracks=30, Lam0: DeviceCsc | None = None, Theta0: DeviceCsc | None = None,
             callback=None, sxx: str = "rows") -> AncdResult:
    """Fit an l1-regularised CGGM (Eq. 1) on device-resident column-major X (n x p), Y (n x q).
    Returns the final (Lambda, Theta) as device CSCs, the objective and the per-iteration history
    (f, ||grad^S||_1, m_Lambda, m_Theta, alpha, per-phase seconds).  sxx: "rows" (on-demand S_xx
    columns of the active rows) or "dense" (the p x p S_xx once)."""
    import time
    n, p = X.shape
    q = Y.shape[1]
    dev = X.device
    Syy, Sxy = ctx.cggm_covariances(X, Y)
    Sxx = ctx.cggm_gram(X) if sxx == "dense" else None
    sxx_cache = {}
    Lam = _own(Lam0) if Lam0 is not None else identity_csc(q, dev)
    Theta = _own(Theta0) if Theta0 is not None else empty_csc(p, q, dev)
    bufs = dict(Psi=colmajor_empty(q, q, device=dev), GradL=colmajor_empty(q, q, device=dev),
                GradT=colmajor_empty(p, q, device=dev))
    Sigma = colmajor_empty(q, q, device=dev)
    caps = [max(4 * q, 1024), max(4 * q, 1024)]
    lists = {}

    def alloc_lists():
        for k, cap in (("L_row", caps[0]), ("L_col", caps[0]), ("T_row", caps[1]), ("T_col", caps[1])):
            lists[k] = torch.empty(cap, dtype=torch.int32, device=dev)

    def factor(L):
        """(L^{-1}, log|L|, is_pd) of a CSC Lambda: densify + the recursive factorisation."""
        D = ctx.cggm_densify(L)
        Linv, ld, pd, _ = ctx.cggm_chol_inverse_dense(D)
        del D
        return Linv, ld, pd

    def sigma_from(Linv):
        """Sigma = L^{-T} L^{-1}: one symmetric GEMM (k-range from the triangle) + mirror."""
        ctx.cggm_gemm(Sigma, Linv, Linv, transA=True, flags=_A_KGE_M | _SYM_LOWER | _SYM_MIRROR)
        return Sigma

    def objective(L, T, Linv, ld):
        return ctx.cggm_objective_given_inverse(X, Y, L, T, lam_L, lam_T, Linv, ld, penalize_diag=penalize_diag)["f"]

    alloc_lists()
    Linv, logdet, pd = factor(Lam)
    if not pd:
        raise CggmError(3, "initial Lambda is not positive definite")
    sigma_from(Linv)
    f = objective(Lam, Theta, Linv, logdet)
    l1T = float(Theta.val.abs().sum()) if Theta.nnz else 0.0
    hist = []
    converged = False
    trial_buf = None
    for t in range(max_iter):
        ph = {}
        t0 = time.perf_counter()
        spec = dict(lam_L=lam_L, lam_T=lam_T, penalize_diag=int(bool(penalize_diag)), **lists)
        while True:   # two-call pattern for the list capacities
            try:
                r = ctx.cggm_psi_grad(X, Y, Theta, Sigma, Syy=Syy, Sxy=Sxy, Lam=Lam, fused=spec, out=bufs)
                break
            except CggmError as e:
                if e.status != 6:
                    raise
                mL, mT = ctx.last_active_sizes if hasattr(ctx, "last_active_sizes") and ctx.last_active_sizes \
                    else (2 * caps[0], 2 * caps[1])
                caps[0], caps[1] = max(caps[0] * 2, mL + 1024), max(caps[1] * 2, mT + 1024)
                alloc_lists()
                spec.update(lists)
        act = r["active"]
        stat = act["subgrad_l1"]
        t1 = time.perf_counter()
        ph["psi_grad_active"] = t1 - t0
        D, delta, l1L = ctx.cggm_lambda_direction(Sigma, bufs["Psi"], bufs["GradL"], Lam, act["L_row"], act["L_col"],
                                                  lam_L, penalize_diag, passes)
        t2 = time.perf_counter()
        ph["lambda_sweep"] = t2 - t1
        if stat < tol * (l1L + l1T):
            hist.append(dict(f=f, stat=stat, m_L=act["m_L"], m_T=act["m_T"], alpha=None, seconds=ph))
            converged = True
            break
        alpha, accepted = 1.0, None
        for _ in range(max_backtracks + 1):
            trial_buf = ctx.cggm_lambda_step(Lam, act["L_row"], act["L_col"], D, alpha, out=trial_buf)
            Lt, ldt, pdt = factor(trial_buf)          # the PD test of the line search
            if pdt:
                ft = objective(trial_buf, Theta, Lt, ldt)
                if math.isfinite(ft) and ft <= f + sigma * alpha * delta:
                    accepted = (Lt, ldt)
                    break
            del Lt
            alpha *= beta
        t3 = time.perf_counter()
        ph["line_search"] = t3 - t2
        if accepted is not None:
            Lam = _own(trial_buf)
            Linv, logdet = accepted
            sigma_from(Linv)                         # the accepted trial's factor: no new factorisation
        else:
            alpha = 0.0
        t4 = time.perf_counter()
        if sxx == "dense":
            Theta, l1T = ctx.cggm_theta_cd(Sigma, Sxx, Sxy, Theta, act["T_row"], act["T_col"], lam_T, passes)
        else:
            cols, xmap = ctx.cggm_gram_rows(X, act["T_row"], cache=sxx_cache)
            t4b = time.perf_counter()
            ph["sxx_rows"] = t4b - t4
            Theta, l1T = ctx.cggm_theta_cd_rows(Sigma, cols, xmap, Sxy, Theta, act["T_row"], act["T_col"], lam_T,
                                                passes)
        Theta = _own(Theta)
        t5 = time.perf_counter()
        ph["theta_sweep"] = t5 - t4 - ph.get("sxx_rows", 0.0)
        f = objective(Lam, Theta, Linv, logdet)      # the same factor again (Lambda unchanged)
        ph["objective"] = time.perf_counter() - t5
        hist.append(dict(f=f, stat=stat, m_L=act["m_L"], m_T=act["m_T"], alpha=alpha, seconds=ph))
        if callback is not None:
            callback(t, hist[-1])
    return AncdResult(Lam=Lam, Theta=Theta, f=f, iters=len(hist), converged=converged, history=hist)


_A_KGE_M, _SYM_LOWER, _SYM_MIRROR = 2, 16, 32
