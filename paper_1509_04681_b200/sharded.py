"""Sample-sharded Newton-iteration evaluation over a torch.distributed process group
(north_star: "each GPU holds row blocks of X and Y, and NCCL allreduce ... combines the partial
X^T Y, X^T(X Theta) and R^T R sums.  The q x q Cholesky/inverse runs on one GPU and is then
broadcast").  SURVEY.md §8(e), CS3.

Every 1/n uses the GLOBAL sample count (reading A21), so each rank's partial sums add up to the
unsharded quantity: S_yy = sum_r Y_r^T Y_r / n, Psi = sum_r R_r^T R_r, grad_Theta = sum_r
(2/n) X_r^T E_r (residual route, identity I3), and the three trace terms of the objective.

The evaluator is written against a small backend interface so that the same host logic runs
with the CUDA backend (`CudaBackend`, libcggm via the binding; NCCL process group) and, in the
CPU tests only, with a test backend over the gloo process group.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

__all__ = ["shard_rows", "flat", "ShardedEvaluator", "CudaBackend"]


def shard_rows(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced row block [a, b) of rank `rank` (first n % world ranks get one more)."""
    base, extra = divmod(n, world)
    a = rank * base + min(rank, extra)
    b = a + base + (1 if rank < extra else 0)
    return a, b


def flat(t: torch.Tensor) -> torch.Tensor:
    """1-D alias of the whole storage behind a column-major (rows, cols) view (ld padding
    included), for collectives."""
    rows, cols = t.shape
    ld = t.stride(1) if cols > 1 else rows
    return torch.as_strided(t, (ld * (cols - 1) + rows,), (1,))


class CudaBackend:
    """libcggm through the Python binding (device tensors)."""

    def __init__(self, ctx):
        self.ctx = ctx

    def covariances_partial(self, X, Y, n_total):
        Syy, _ = self.ctx.cggm_covariances(X, Y, n_total=n_total, want_sxy=False)
        return Syy

    def invert_logdet(self, Lam):
        S, ld, pd, fc = self.ctx.cggm_invert_logdet(Lam)
        return S, ld, pd, fc

    def empty_sigma(self, q, like):
        from .api import colmajor_empty
        return colmajor_empty(q, q, device=like.device)

    def psi_grad_partial(self, X, Y, Theta, Sigma, n_total):
        r = self.ctx.cggm_psi_grad(X, Y, Theta, Sigma, n_total=n_total, want_gradL=False)
        return r["Psi"], r["GradT"]

    def grad_lambda(self, Syy, Sigma, Psi):
        return self.ctx.cggm_grad_lambda(Syy, Sigma, Psi)

    def active_set(self, GradL, GradT, Lam, Theta, lam_L, lam_T, penalize_diag, tie_eps):
        return self.ctx.cggm_active_set(GradL, GradT, Lam, Theta, lam_L, lam_T, penalize_diag, tie_eps)

    def objective_partial(self, X, Y, Lam, Theta, lam_L, lam_T, penalize_diag, n_total):
        return self.ctx.cggm_objective(X, Y, Lam, Theta, lam_L, lam_T, penalize_diag, n_total=n_total)


class ShardedEvaluator:
    """One Newton-iteration evaluation with the rows of X, Y split over the process group."""

    def __init__(self, backend, group=None, replicate_inverse: bool = False):
        self.b = backend
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.replicate_inverse = replicate_inverse

    def _allreduce(self, t):
        if self.world > 1:
            dist.all_reduce(flat(t), group=self.group)
        return t

    def setup(self, X_r, Y_r, n_total):
        """Per-dataset S_yy (excluded from the evaluation's timing)."""
        self.n_total = n_total
        self.Syy = self._allreduce(self.b.covariances_partial(X_r, Y_r, n_total))
        return self.Syy

    def evaluate(self, X_r, Y_r, Lam, Theta, lam_L, lam_T, penalize_diag=True, tie_eps=1e-9):
        n = self.n_total
        q = Lam.nrows
        # Sigma = Lambda^{-1}: rank 0 factors and broadcasts (or every rank, replicate_inverse)
        if self.world == 1 or self.replicate_inverse or self.rank == 0:
            Sigma, logdet, pd, fc = self.b.invert_logdet(Lam)
        else:
            Sigma, logdet, pd, fc = self.b.empty_sigma(q, Y_r), None, None, None
        if self.world > 1 and not self.replicate_inverse:
            dist.broadcast(flat(Sigma), src=0, group=self.group)
            meta = torch.tensor([logdet if logdet is not None else 0.0, float(bool(pd)), float(fc or 0)],
                                dtype=torch.float64, device=Sigma.device)
            dist.broadcast(meta, src=0, group=self.group)
            logdet, pd, fc = float(meta[0]), bool(meta[1] > 0.5), int(meta[2])
        Psi, GradT = self.b.psi_grad_partial(X_r, Y_r, Theta, Sigma, n)
        self._allreduce(Psi)
        self._allreduce(GradT)
        GradL = self.b.grad_lambda(self.Syy, Sigma, Psi)
        act = self.b.active_set(GradL, GradT, Lam, Theta, lam_L, lam_T, penalize_diag, tie_eps)
        ob = self.b.objective_partial(X_r, Y_r, Lam, Theta, lam_L, lam_T, penalize_diag, n)
        parts = torch.tensor([ob["tr_syy_lam"], ob["tr_sxy_theta"], ob["tr_sigma_m"]], dtype=torch.float64,
                             device=Psi.device)
        if self.world > 1:
            dist.all_reduce(parts, group=self.group)
        tr_syy, tr_sxy, tr_sm = (float(v) for v in parts.tolist())
        if ob["is_pd"]:
            g = -ob["logdet"] + tr_syy + 2.0 * tr_sxy + tr_sm
            f = g + ob["pen_L"] + ob["pen_T"]
        else:
            g = f = float("inf")
        return dict(Sigma=Sigma, logdet=logdet, is_pd=pd, fail_col=fc, Psi=Psi, GradL=GradL, GradT=GradT,
                    active=act, f=f, g=g, obj_logdet=ob["logdet"], tr_syy_lam=tr_syy, tr_sxy_theta=tr_sxy,
                    tr_sigma_m=tr_sm)
