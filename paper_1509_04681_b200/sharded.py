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

Split factorisations (world >= 2, the default): the line-search objective needs a Cholesky of its
own (a trial Lambda), independent of the inverse's.  Rank 1 keeps a full copy of X and Y
(gathered once in setup(); the data do not change across evaluations) and evaluates the
objective on all n rows while rank 0 computes Sigma = Lambda^{-1} -- the two O(q^3) chains run on
different GPUs instead of one after the other (with split_objective=False every rank factors the
trial Lambda for its partial traces, as in a plain data-parallel reading).
"""
from __future__ import annotations

import torch
import torch.distributed as dist

__all__ = ["shard_rows", "flat", "ShardedEvaluator", "CudaBackend", "CollectiveEvaluator"]


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

    def empty_matrix(self, rows, cols, like):
        from .api import colmajor_empty
        return colmajor_empty(rows, cols, device=like.device, dtype=like.dtype)

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

    def __init__(self, backend, group=None, replicate_inverse: bool = False, split_objective: bool = True):
        self.b = backend
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.replicate_inverse = replicate_inverse
        self.split = split_objective and self.world > 1 and not replicate_inverse
        self.obj_rank = 1 if self.split else None
        self.X_full = self.Y_full = None

    def _allreduce(self, t):
        if self.world > 1:
            dist.all_reduce(flat(t), group=self.group)
        return t

    def setup(self, X_r, Y_r, n_total):
        """Per-dataset S_yy (excluded from the evaluation's timing); with split factorisations the
        objective rank also assembles the full X, Y from the row blocks (point-to-point)."""
        self.n_total = n_total
        self.Syy = self._allreduce(self.b.covariances_partial(X_r, Y_r, n_total))
        if self.split:
            self._gather_full(X_r, Y_r)
        return self.Syy

    def _gather_full(self, X_r, Y_r):
        n = self.n_total
        p, q = X_r.shape[1], Y_r.shape[1]
        # gloo's point-to-point needs host memory (the CPU tests, or a gloo smoke run on a GPU)
        host = dist.get_backend(self.group) == "gloo"
        if self.rank == self.obj_rank:
            self.X_full = self.b.empty_matrix(n, p, X_r)
            self.Y_full = self.b.empty_matrix(n, q, Y_r)
            for r in range(self.world):
                a, b = shard_rows(n, self.world, r)
                for full, local in ((self.X_full, X_r), (self.Y_full, Y_r)):
                    if r == self.rank:
                        full[a:b].copy_(local)
                    else:
                        buf = torch.empty((b - a) * full.shape[1], dtype=full.dtype,
                                          device="cpu" if host else full.device)
                        dist.recv(buf, src=r, group=self.group)
                        full[a:b].copy_(buf.view(full.shape[1], b - a).t())
        else:
            for local in (X_r, Y_r):
                buf = local.t().contiguous().view(-1)
                dist.send(buf.cpu() if host else buf, dst=self.obj_rank, group=self.group)

    _OB_KEYS = ("f", "g", "logdet", "tr_syy_lam", "tr_sxy_theta", "tr_sigma_m", "pen_L", "pen_T", "is_pd", "fail_col")

    def _objective_split(self, Lam, Theta, lam_L, lam_T, penalize_diag, like):
        """The objective on all rows at the objective rank (concurrently with rank 0's inverse),
        its scalars broadcast to every rank."""
        vals = torch.zeros(len(self._OB_KEYS), dtype=torch.float64, device=like.device)
        if self.rank == self.obj_rank:
            ob = self.b.objective_partial(self.X_full, self.Y_full, Lam, Theta, lam_L, lam_T, penalize_diag,
                                          self.n_total)
            vals = torch.tensor([float(ob[k]) for k in self._OB_KEYS], dtype=torch.float64, device=like.device)
        dist.broadcast(vals, src=self.obj_rank, group=self.group)
        ob = {k: float(v) for k, v in zip(self._OB_KEYS, vals.tolist())}
        ob["is_pd"] = ob["is_pd"] > 0.5
        ob["fail_col"] = int(ob["fail_col"])
        return ob

    def evaluate(self, X_r, Y_r, Lam, Theta, lam_L, lam_T, penalize_diag=True, tie_eps=1e-9):
        n = self.n_total
        q = Lam.nrows
        # Sigma = Lambda^{-1}: rank 0 factors and broadcasts (or every rank, replicate_inverse)
        if self.world == 1 or self.replicate_inverse or self.rank == 0:
            Sigma, logdet, pd, fc = self.b.invert_logdet(Lam)
        else:
            Sigma, logdet, pd, fc = self.b.empty_sigma(q, Y_r), None, None, None
        if self.split:
            self._ob_split = self._objective_split(Lam, Theta, lam_L, lam_T, penalize_diag, Sigma)
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
        if self.split:
            # the objective rank evaluated the whole objective on all rows (see _objective_split)
            ob = self._ob_split
            parts = torch.tensor([ob["tr_syy_lam"], ob["tr_sxy_theta"], ob["tr_sigma_m"]], dtype=torch.float64)
        else:
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


class CollectiveEvaluator:
    """The same sample-sharded evaluation with the collectives inside libcggm: the ctx carries a
    communicator (`Context.comm_init` for NCCL, `Context.comm_init_torch` for a torch.distributed
    group) and the library calls are collective (include/cggm.h, "sample sharding"):
    cggm_invert_logdet (rank 0 factors, Sigma broadcast), cggm_psi_grad (Psi and grad_Theta
    all-reduced before grad_Lambda), cggm_objective (each rank's trial Cholesky on its rows, the
    three traces all-reduced).  The active sets are then formed identically on every rank."""

    def __init__(self, ctx):
        self.ctx = ctx
        self.rank, self.world = ctx.comm_info()

    def setup(self, X_r, Y_r, n_total):
        self.n_total = n_total
        self.Syy, _ = self.ctx.cggm_covariances(X_r, Y_r, n_total=n_total, want_sxy=False)
        return self.Syy

    def evaluate(self, X_r, Y_r, Lam, Theta, lam_L, lam_T, penalize_diag=True, tie_eps=1e-9):
        n = self.n_total
        Sigma, logdet, pd, fc = self.ctx.cggm_invert_logdet(Lam)
        r = self.ctx.cggm_psi_grad(X_r, Y_r, Theta, Sigma, Syy=self.Syy, n_total=n)
        act = self.ctx.cggm_active_set(r["GradL"], r["GradT"], Lam, Theta, lam_L, lam_T, penalize_diag, tie_eps)
        ob = self.ctx.cggm_objective(X_r, Y_r, Lam, Theta, lam_L, lam_T, penalize_diag, n_total=n)
        return dict(Sigma=Sigma, logdet=logdet, is_pd=pd, fail_col=fc, Psi=r["Psi"], GradL=r["GradL"],
                    GradT=r["GradT"], active=act, f=ob["f"], g=ob["g"], obj_logdet=ob["logdet"],
                    tr_syy_lam=ob["tr_syy_lam"], tr_sxy_theta=ob["tr_sxy_theta"], tr_sigma_m=ob["tr_sigma_m"])
