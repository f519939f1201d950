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

__all__ = ["shard_rows", "flat", "ShardedEvaluator", "CudaBackend", "CollectiveEvaluator", "DistributedInverse",
           "PeerAllReduce"]


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

    def psi_grad_partial(self, X, Y, Theta, Sigma, n_total, out=None):
        r = self.ctx.cggm_psi_grad(X, Y, Theta, Sigma, n_total=n_total, want_gradL=False, out=out)
        return r["Psi"], r["GradT"]

    def grad_lambda(self, Syy, Sigma, Psi):
        return self.ctx.cggm_grad_lambda(Syy, Sigma, Psi)

    # sample-sharded grad_Theta by column ranges (reduce-scatter, local compaction, list all-gather)
    def psi_residual_partial(self, X, Y, Theta, Sigma, n_total):
        return self.ctx.cggm_psi_residual(X, Y, Theta, Sigma, n_total=n_total)

    def grad_theta_block(self, X, E, c0, c1, n_total, out):
        """out (p x (c1 - c0)) = (2/n) X_r^T E_r[:, c0:c1], this shard's grad_Theta partial (I3)."""
        self.ctx.cggm_gemm(out, X, E[:, c0:c1], transA=True, alpha=2.0 / n_total)

    def active_lambda_only(self, GradL, Lam, lam_L, penalize_diag, tie_eps):
        """S_Lambda and the Lambda part of the statistic (the Theta side empty: a 1 x q zero gradient
        with an empty Theta and lam_T = 1 contributes no entry and 0)."""
        from .api import DeviceCsc, colmajor_empty
        q = GradL.shape[0]
        key = ("lam_only", q)
        if getattr(self, "_lam_only_key", None) != key:
            self._zero_gt = colmajor_empty(1, q, device=GradL.device, dtype=GradL.dtype, zero=True)
            self._empty_th = DeviceCsc(1, q, torch.zeros(q + 1, dtype=torch.int64, device=GradL.device),
                                       torch.zeros(0, dtype=torch.int32, device=GradL.device),
                                       torch.zeros(0, dtype=GradL.dtype, device=GradL.device))
            self._lam_only_key = key
        return self.ctx.cggm_active_set(GradL, self._zero_gt, Lam, self._empty_th, lam_L, 1.0, penalize_diag, tie_eps)

    def active_theta_block(self, G, Theta, c0, lam_T, tie_eps, T_row, T_col):
        return self.ctx.cggm_active_theta_block(G, Theta, c0, lam_T, tie_eps, T_row, T_col)

    def flat_zeros(self, count, like):
        return torch.zeros(count, dtype=like.dtype, device=like.device)

    def int_lists(self, cap, like):
        return (torch.empty(cap, dtype=torch.int32, device=like.device),
                torch.empty(cap, dtype=torch.int32, device=like.device))

    def active_set(self, GradL, GradT, Lam, Theta, lam_L, lam_T, penalize_diag, tie_eps):
        return self.ctx.cggm_active_set(GradL, GradT, Lam, Theta, lam_L, lam_T, penalize_diag, tie_eps)

    def objective_partial(self, X, Y, Lam, Theta, lam_L, lam_T, penalize_diag, n_total):
        return self.ctx.cggm_objective(X, Y, Lam, Theta, lam_L, lam_T, penalize_diag, n_total=n_total)

    def objective_given_inverse_partial(self, X, Y, Lam, Theta, lam_L, lam_T, penalize_diag, n_total, Linv, logdet):
        return self.ctx.cggm_objective_given_inverse(X, Y, Lam, Theta, lam_L, lam_T, Linv, logdet,
                                                     penalize_diag=penalize_diag, n_total=n_total)

    def _obj_ctx(self, group):
        """A second context on the device with a library-owned communicator over `group` (NCCL, or the
        torch group's own collectives for gloo): its cggm_objective / cggm_objective_given_inverse are
        collective -- the shards' trace partials are all-reduced and f assembled inside libcggm."""
        if getattr(self, "_octx", None) is None:
            from .api import Context
            c = Context(self.ctx.device, dtype="f64" if self.ctx.tdtype == torch.float64 else "f32")
            if dist.get_backend(group) == "nccl":
                c.comm_init(group)
            else:
                c.comm_init_torch(group)
            self._octx = c
        return self._octx

    def objective_sharded(self, X, Y, Lam, Theta, lam_L, lam_T, penalize_diag, n_total, group, Linv=None,
                          logdet=None):
        """The whole objective of the sharded data, assembled by the library's collective calls."""
        c = self._obj_ctx(group)
        if Linv is None:
            return c.cggm_objective(X, Y, Lam, Theta, lam_L, lam_T, penalize_diag, n_total=n_total)
        return c.cggm_objective_given_inverse(X, Y, Lam, Theta, lam_L, lam_T, Linv, logdet,
                                              penalize_diag=penalize_diag, n_total=n_total)

    # dense building blocks (DistributedInverse)
    def zeros(self, rows, cols):
        from .api import colmajor_empty
        return colmajor_empty(rows, cols, device=torch.device("cuda", self.ctx.device), dtype=self.ctx.tdtype, zero=True)

    def densify(self, Lam):
        return self.ctx.cggm_densify(Lam)

    def chol_inverse(self, D):
        return self.ctx.cggm_chol_inverse_dense(D)

    def gemm(self, C, A, B, transA=False, transB=False, alpha=1.0, beta=0.0, flags=0):
        return self.ctx.cggm_gemm(C, A, B, transA=transA, transB=transB, alpha=alpha, beta=beta, flags=flags)

    def symmetrize(self, S):
        return self.ctx.cggm_symmetrize(S)


class ShardedEvaluator:
    """One Newton-iteration evaluation with the rows of X, Y split over the process group.

    Sigma: rank 0 factors and broadcasts (default), every rank factors (replicate_inverse), or all
    ranks factor together (distributed_inverse, NEXT-3, block-cyclic with `block`-wide columns).
    Objective: on one rank with the gathered full data while Sigma is formed (split_objective),
    else each rank's partial traces are all-reduced (with distributed_inverse its trial
    factorisation is distributed too).  Psi / grad_Theta partials: NCCL all-reduce, or CUDA IPC peer
    memory (peer_allreduce, CudaBackend only)."""

    def __init__(self, backend, group=None, replicate_inverse: bool = False, split_objective: bool = True,
                 distributed_inverse: bool = False, block: int = 2048, peer_allreduce: bool = False,
                 grad_theta: str = "allreduce", rs_width: int = 256):
        self.b = backend
        # grad_Theta: "allreduce" = every rank holds the summed p x q gradient (north_star's all-reduce);
        # "reduce_scatter" = column ranges owned by the ranks, each column block's partials
        # reduce-scattered (rs_width columns per owner per round), compacted by the owner, the compact
        # S_Theta lists all-gathered (SURVEY.md §8(e) "Better"): no rank holds a p x q buffer
        if grad_theta not in ("allreduce", "reduce_scatter"):
            raise ValueError(f"grad_theta must be allreduce or reduce_scatter, not {grad_theta!r}")
        self.grad_theta = grad_theta
        self.rs_width = int(rs_width)
        self._rs = {}
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.replicate_inverse = replicate_inverse
        # NEXT-3: Sigma by the block-cyclic factorisation over all ranks (every rank ends with Sigma)
        self.dist_inv = DistributedInverse(backend, block=block, group=group) if (
            distributed_inverse and self.world > 1 and not replicate_inverse) else None
        self.split = split_objective and self.world > 1 and not replicate_inverse
        self.obj_rank = (self.world - 1 if self.dist_inv is not None else 1) if self.split else None
        self.X_full = self.Y_full = None
        # Psi / grad_Theta partials summed over CUDA IPC peer memory instead of NCCL (CudaBackend)
        self.peer = PeerAllReduce(backend.ctx, group) if (peer_allreduce and self.world > 1) else None
        self._peer_out = None
        # per-phase CUDA events on the current stream (bench: per-rank phase times, collective GB/s)
        self.timing = False
        self._marks = []

    def _mark(self, name):
        if self.timing:
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            self._marks.append((name, e))

    def phase_times(self):
        """{phase: ms} between consecutive marks of the last timed evaluate() (synchronises)."""
        torch.cuda.synchronize()
        out = {}
        for (_, a), (name, b) in zip(self._marks, self._marks[1:]):
            out[name] = out.get(name, 0.0) + a.elapsed_time(b)
        self._marks = []
        return out

    def _g(self, r):
        """Global rank of group rank r (torch's src / dst arguments are global ranks)."""
        return dist.get_global_rank(self.group, r) if self.group is not None else r

    def _allreduce(self, t):
        if self.world > 1:
            if self.peer is not None and hasattr(t, "_peer_index"):
                return self.peer.allreduce(t)
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
                        dist.recv(buf, src=self._g(r), group=self.group)
                        full[a:b].copy_(buf.view(full.shape[1], b - a).t())
        else:
            for local in (X_r, Y_r):
                buf = local.t().contiguous().view(-1)
                dist.send(buf.cpu() if host else buf, dst=self._g(self.obj_rank), group=self.group)

    _OB_KEYS = ("f", "g", "logdet", "tr_syy_lam", "tr_sxy_theta", "tr_sigma_m", "pen_L", "pen_T", "is_pd", "fail_col")

    def _objective_split(self, Lam, Theta, lam_L, lam_T, penalize_diag, like):
        """The objective on all rows at the objective rank (concurrently with rank 0's inverse),
        its scalars broadcast to every rank."""
        vals = torch.zeros(len(self._OB_KEYS), dtype=torch.float64, device=like.device)
        if self.rank == self.obj_rank:
            ob = self.b.objective_partial(self.X_full, self.Y_full, Lam, Theta, lam_L, lam_T, penalize_diag,
                                          self.n_total)
            vals = torch.tensor([float(ob[k]) for k in self._OB_KEYS], dtype=torch.float64, device=like.device)
        dist.broadcast(vals, src=self._g(self.obj_rank), group=self.group)
        ob = {k: float(v) for k, v in zip(self._OB_KEYS, vals.tolist())}
        ob["is_pd"] = ob["is_pd"] > 0.5
        ob["fail_col"] = int(ob["fail_col"])
        return ob

    def _reduce_scatter(self, flat_in, flat_out):
        """flat_out = block `rank` of the element-wise sum over ranks of flat_in (world equal blocks)."""
        if self.world == 1:
            flat_out.copy_(flat_in[:flat_out.numel()])
            return
        if dist.get_backend(self.group) == "nccl":
            dist.reduce_scatter_tensor(flat_out, flat_in, group=self.group)
        else:   # gloo has no reduce-scatter: all-reduce, keep this rank's block (same sums)
            h = flat_in.cpu()
            dist.all_reduce(h, group=self.group)
            k = flat_out.numel()
            flat_out.copy_(h[self.rank * k:(self.rank + 1) * k].to(flat_out.device))

    def _all_gather_lists(self, rows, cols, m):
        """Concatenation in rank order of every rank's first m entries (rank r owns an ascending column
        range, so the result is the global column-major list, identical on every rank)."""
        if self.world == 1:
            return rows[:m].clone(), cols[:m].clone()
        host = dist.get_backend(self.group) == "gloo"
        dev = rows.device
        cnt = torch.tensor([m], dtype=torch.int64, device="cpu" if host else dev)
        cnts = [torch.zeros_like(cnt) for _ in range(self.world)]
        dist.all_gather(cnts, cnt, group=self.group)
        cnts = [int(c.item()) for c in cnts]
        mx = max(max(cnts), 1)
        out = []
        for src in (rows, cols):
            loc = torch.zeros(mx, dtype=src.dtype, device="cpu" if host else dev)
            loc[:m].copy_(src[:m])
            parts = [torch.empty_like(loc) for _ in range(self.world)]
            dist.all_gather(parts, loc, group=self.group)
            out.append(torch.cat([pt[:c] for pt, c in zip(parts, cnts)]).to(dev))
        return out[0], out[1]

    def _grad_theta_reduce_scatter(self, X_r, E, Theta, lam_T, tie_eps, actL):
        """S_Theta without a stored p x q gradient: ranks own balanced column ranges; round t forms,
        for every owner r, the partial (2/n) X^T E[:, a_r + t w : a_r + (t + 1) w] into block r of a
        p x (world w) buffer, reduce-scatters it (block r, summed, to rank r) and the owner compacts
        its block (global column indices).  The compact lists are all-gathered at the end."""
        n = self.n_total
        p, q = X_r.shape[1], Theta.ncols
        G, me = self.world, self.rank
        ranges = [shard_rows(q, G, r) for r in range(G)]
        span = max(b - a for a, b in ranges)
        w = max(1, min(self.rs_width, span))
        ld = p + (p & 1)
        key = (p, q, G, w)
        if self._rs.get("key") != key:
            self._rs = {"key": key, "buf": self.b.flat_zeros(G * ld * w, E), "out": self.b.flat_zeros(ld * w, E)}
            self._rs["T_row"], self._rs["T_col"] = self.b.int_lists(max(4096, 2 * Theta.nnz // G + p), E)
        buf, outf = self._rs["buf"], self._rs["out"]

        def block(flat, r):   # p x w column-major view of block r (leading dimension ld)
            return torch.as_strided(flat, (p, w), (1, ld), r * ld * w)

        a_me, b_me = ranges[me]
        m_tot, ties, sub = 0, 0, 0.0
        for t in range((span + w - 1) // w):
            for r, (a, b) in enumerate(ranges):
                c0, c1 = a + t * w, min(b, a + (t + 1) * w)
                if c1 > c0:
                    self.b.grad_theta_block(X_r, E, c0, c1, n, block(buf, r)[:, :c1 - c0])
            self._reduce_scatter(buf, outf)
            c0, c1 = a_me + t * w, min(b_me, a_me + (t + 1) * w)
            if c1 <= c0:
                continue
            G_blk = block(outf, 0)[:, :c1 - c0]
            while True:
                T_row, T_col = self._rs["T_row"], self._rs["T_col"]
                try:
                    mb, tb, sb = self.b.active_theta_block(G_blk, Theta, c0, lam_T, tie_eps, T_row[m_tot:],
                                                           T_col[m_tot:])
                    break
                except Exception as exc:   # CGGM_ERR_CAPACITY: grow the lists, keep what is written
                    need = getattr(exc, "m", None)
                    if need is None:
                        raise
                    nr, nc = self.b.int_lists(2 * (m_tot + need) + 4096, E)
                    nr[:m_tot].copy_(T_row[:m_tot])
                    nc[:m_tot].copy_(T_col[:m_tot])
                    self._rs["T_row"], self._rs["T_col"] = nr, nc
            m_tot += mb
            ties += tb
            sub += sb
        T_row, T_col = self._all_gather_lists(self._rs["T_row"], self._rs["T_col"], m_tot)
        tot = torch.tensor([float(ties), sub], dtype=torch.float64)
        if G > 1:
            host = dist.get_backend(self.group) == "gloo"
            tot = tot if host else tot.to(E.device)
            dist.all_reduce(tot, group=self.group)
        ties_T, sub_T = float(tot[0]), float(tot[1])
        act = dict(actL)
        act.update(T_row=T_row, T_col=T_col, m_T=int(T_row.numel()), ties_T=int(round(ties_T)),
                   subgrad_l1=float(actL["subgrad_l1"]) + sub_T)
        return act

    def evaluate(self, X_r, Y_r, Lam, Theta, lam_L, lam_T, penalize_diag=True, tie_eps=1e-9):
        n = self.n_total
        q = Lam.nrows
        self._marks = []
        self._mark("start")
        # Sigma = Lambda^{-1}: rank 0 factors and broadcasts (or every rank, replicate_inverse; or
        # all ranks together, distributed_inverse)
        if self.dist_inv is not None:
            Sigma, logdet, pd, fc = self.dist_inv.invert(Lam)
            if Sigma is None:
                Sigma = self.b.empty_sigma(q, Y_r)
        elif self.world == 1 or self.replicate_inverse or self.rank == 0:
            Sigma, logdet, pd, fc = self.b.invert_logdet(Lam)
        else:
            Sigma, logdet, pd, fc = self.b.empty_sigma(q, Y_r), None, None, None
        self._mark("inverse")
        if self.split:
            self._ob_split = self._objective_split(Lam, Theta, lam_L, lam_T, penalize_diag, Sigma)
            self._mark("objective_split")
        if self.world > 1 and not self.replicate_inverse and self.dist_inv is None:
            dist.broadcast(flat(Sigma), src=self._g(0), group=self.group)
            meta = torch.tensor([logdet if logdet is not None else 0.0, float(bool(pd)), float(fc or 0)],
                                dtype=torch.float64, device=Sigma.device)
            dist.broadcast(meta, src=self._g(0), group=self.group)
            logdet, pd, fc = float(meta[0]), bool(meta[1] > 0.5), int(meta[2])
            self._mark("bcast_sigma")
        if self.grad_theta == "reduce_scatter":
            Psi, E = self.b.psi_residual_partial(X_r, Y_r, Theta, Sigma, n)
            self._mark("psi_residual")
            self._allreduce(Psi)
            self._mark("allreduce_psi")
            GradL = self.b.grad_lambda(self.Syy, Sigma, Psi)
            actL = self.b.active_lambda_only(GradL, Lam, lam_L, penalize_diag, tie_eps)
            self._mark("grad_lambda_active")
            act = self._grad_theta_reduce_scatter(X_r, E, Theta, lam_T, tie_eps, actL)
            self._mark("reduce_scatter_grad_theta")
            GradT = None
            return self._finish(Sigma, logdet, pd, fc, Psi, GradL, GradT, act, X_r, Y_r, Lam, Theta, lam_L, lam_T,
                                penalize_diag, n)
        if self.peer is not None:
            if self._peer_out is None:   # symmetric buffers, allocated once (same shapes every call)
                p = X_r.shape[1]
                self._peer_out = {"Psi": self.peer.empty(q, q, Sigma.dtype), "GradT": self.peer.empty(p, q, Sigma.dtype)}
            Psi, GradT = self.b.psi_grad_partial(X_r, Y_r, Theta, Sigma, n, out=self._peer_out)
        else:
            Psi, GradT = self.b.psi_grad_partial(X_r, Y_r, Theta, Sigma, n)
        self._mark("psi_grad_partial")
        self._allreduce(Psi)
        self._mark("allreduce_psi")
        self._allreduce(GradT)
        self._mark("allreduce_grad_theta")
        GradL = self.b.grad_lambda(self.Syy, Sigma, Psi)
        act = self.b.active_set(GradL, GradT, Lam, Theta, lam_L, lam_T, penalize_diag, tie_eps)
        self._mark("grad_lambda_active")
        return self._finish(Sigma, logdet, pd, fc, Psi, GradL, GradT, act, X_r, Y_r, Lam, Theta, lam_L, lam_T,
                            penalize_diag, n)

    def _finish(self, Sigma, logdet, pd, fc, Psi, GradL, GradT, act, X_r, Y_r, Lam, Theta, lam_L, lam_T,
                penalize_diag, n):
        """The line-search objective and the result.  f comes from libcggm in every mode: the split
        objective rank's cggm_objective on all rows (scalars broadcast); otherwise the library's
        collective cggm_objective / cggm_objective_given_inverse (trace partials all-reduced inside the
        library) through the backend's objective_sharded."""
        if self.split:
            # the objective rank evaluated the whole objective on all rows (see _objective_split)
            ob = self._ob_split
        elif self.dist_inv is not None:
            # the trial factorisation distributed too: L^{-1} gathered, the shards' traces combined by
            # the library's collective objective
            Linv, ld_t, pd_t, fc_t = self.dist_inv.invert(Lam, want_sigma=False, want_linv=True)
            if pd_t:
                ob = self.b.objective_sharded(X_r, Y_r, Lam, Theta, lam_L, lam_T, penalize_diag, n, self.group,
                                              Linv=Linv, logdet=ld_t)
            else:
                ob = dict(f=float("inf"), g=float("inf"), is_pd=False, fail_col=fc_t, logdet=float("nan"),
                          tr_syy_lam=float("nan"), tr_sxy_theta=float("nan"), tr_sigma_m=float("nan"))
        elif self.world > 1:
            ob = self.b.objective_sharded(X_r, Y_r, Lam, Theta, lam_L, lam_T, penalize_diag, n, self.group)
        else:
            ob = self.b.objective_partial(X_r, Y_r, Lam, Theta, lam_L, lam_T, penalize_diag, n)
        self._mark("objective")
        return dict(Sigma=Sigma, logdet=logdet, is_pd=pd, fail_col=fc, Psi=Psi, GradL=GradL, GradT=GradT,
                    active=act, f=ob["f"], g=ob["g"], obj_logdet=ob["logdet"], tr_syy_lam=ob["tr_syy_lam"],
                    tr_sxy_theta=ob["tr_sxy_theta"], tr_sigma_m=ob["tr_sigma_m"])


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

    def _reduce_scatter(self, flat_in, flat_out):
        """flat_out = block `rank` of the element-wise sum over ranks of flat_in (world equal blocks)."""
        if self.world == 1:
            flat_out.copy_(flat_in[:flat_out.numel()])
            return
        if dist.get_backend(self.group) == "nccl":
            dist.reduce_scatter_tensor(flat_out, flat_in, group=self.group)
        else:   # gloo has no reduce-scatter: all-reduce, keep this rank's block (same sums)
            h = flat_in.cpu()
            dist.all_reduce(h, group=self.group)
            k = flat_out.numel()
            flat_out.copy_(h[self.rank * k:(self.rank + 1) * k].to(flat_out.device))

    def _all_gather_lists(self, rows, cols, m):
        """Concatenation in rank order of every rank's first m entries (rank r owns an ascending column
        range, so the result is the global column-major list, identical on every rank)."""
        if self.world == 1:
            return rows[:m].clone(), cols[:m].clone()
        host = dist.get_backend(self.group) == "gloo"
        dev = rows.device
        cnt = torch.tensor([m], dtype=torch.int64, device="cpu" if host else dev)
        cnts = [torch.zeros_like(cnt) for _ in range(self.world)]
        dist.all_gather(cnts, cnt, group=self.group)
        cnts = [int(c.item()) for c in cnts]
        mx = max(max(cnts), 1)
        out = []
        for src in (rows, cols):
            loc = torch.zeros(mx, dtype=src.dtype, device="cpu" if host else dev)
            loc[:m].copy_(src[:m])
            parts = [torch.empty_like(loc) for _ in range(self.world)]
            dist.all_gather(parts, loc, group=self.group)
            out.append(torch.cat([pt[:c] for pt, c in zip(parts, cnts)]).to(dev))
        return out[0], out[1]

    def _grad_theta_reduce_scatter(self, X_r, E, Theta, lam_T, tie_eps, actL):
        """S_Theta without a stored p x q gradient: ranks own balanced column ranges; round t forms,
        for every owner r, the partial (2/n) X^T E[:, a_r + t w : a_r + (t + 1) w] into block r of a
        p x (world w) buffer, reduce-scatters it (block r, summed, to rank r) and the owner compacts
        its block (global column indices).  The compact lists are all-gathered at the end."""
        n = self.n_total
        p, q = X_r.shape[1], Theta.ncols
        G, me = self.world, self.rank
        ranges = [shard_rows(q, G, r) for r in range(G)]
        span = max(b - a for a, b in ranges)
        w = max(1, min(self.rs_width, span))
        ld = p + (p & 1)
        key = (p, q, G, w)
        if self._rs.get("key") != key:
            self._rs = {"key": key, "buf": self.b.flat_zeros(G * ld * w, E), "out": self.b.flat_zeros(ld * w, E)}
            self._rs["T_row"], self._rs["T_col"] = self.b.int_lists(max(4096, 2 * Theta.nnz // G + p), E)
        buf, outf = self._rs["buf"], self._rs["out"]

        def block(flat, r):   # p x w column-major view of block r (leading dimension ld)
            return torch.as_strided(flat, (p, w), (1, ld), r * ld * w)

        a_me, b_me = ranges[me]
        m_tot, ties, sub = 0, 0, 0.0
        for t in range((span + w - 1) // w):
            for r, (a, b) in enumerate(ranges):
                c0, c1 = a + t * w, min(b, a + (t + 1) * w)
                if c1 > c0:
                    self.b.grad_theta_block(X_r, E, c0, c1, n, block(buf, r)[:, :c1 - c0])
            self._reduce_scatter(buf, outf)
            c0, c1 = a_me + t * w, min(b_me, a_me + (t + 1) * w)
            if c1 <= c0:
                continue
            G_blk = block(outf, 0)[:, :c1 - c0]
            while True:
                T_row, T_col = self._rs["T_row"], self._rs["T_col"]
                try:
                    mb, tb, sb = self.b.active_theta_block(G_blk, Theta, c0, lam_T, tie_eps, T_row[m_tot:],
                                                           T_col[m_tot:])
                    break
                except Exception as exc:   # CGGM_ERR_CAPACITY: grow the lists, keep what is written
                    need = getattr(exc, "m", None)
                    if need is None:
                        raise
                    nr, nc = self.b.int_lists(2 * (m_tot + need) + 4096, E)
                    nr[:m_tot].copy_(T_row[:m_tot])
                    nc[:m_tot].copy_(T_col[:m_tot])
                    self._rs["T_row"], self._rs["T_col"] = nr, nc
            m_tot += mb
            ties += tb
            sub += sb
        T_row, T_col = self._all_gather_lists(self._rs["T_row"], self._rs["T_col"], m_tot)
        tot = torch.tensor([float(ties), sub], dtype=torch.float64)
        if G > 1:
            host = dist.get_backend(self.group) == "gloo"
            tot = tot if host else tot.to(E.device)
            dist.all_reduce(tot, group=self.group)
        ties_T, sub_T = float(tot[0]), float(tot[1])
        act = dict(actL)
        act.update(T_row=T_row, T_col=T_col, m_T=int(T_row.numel()), ties_T=int(round(ties_T)),
                   subgrad_l1=float(actL["subgrad_l1"]) + sub_T)
        return act

    def evaluate(self, X_r, Y_r, Lam, Theta, lam_L, lam_T, penalize_diag=True, tie_eps=1e-9):
        n = self.n_total
        Sigma, logdet, pd, fc = self.ctx.cggm_invert_logdet(Lam)
        r = self.ctx.cggm_psi_grad(X_r, Y_r, Theta, Sigma, Syy=self.Syy, n_total=n)
        act = self.ctx.cggm_active_set(r["GradL"], r["GradT"], Lam, Theta, lam_L, lam_T, penalize_diag, tie_eps)
        ob = self.ctx.cggm_objective(X_r, Y_r, Lam, Theta, lam_L, lam_T, penalize_diag, n_total=n)
        return dict(Sigma=Sigma, logdet=logdet, is_pd=pd, fail_col=fc, Psi=r["Psi"], GradL=r["GradL"],
                    GradT=r["GradT"], active=act, f=ob["f"], g=ob["g"], obj_logdet=ob["logdet"],
                    tr_syy_lam=ob["tr_syy_lam"], tr_sxy_theta=ob["tr_sxy_theta"], tr_sigma_m=ob["tr_sigma_m"])


# ------------------------------------------------------------------ NEXT-3: distributed inverse
class DistributedInverse:
    """Sigma = Lambda^{-1}, log|Lambda| and the PD test with the q^3 work split over the ranks of a
    process group (the paper parallelises these precomputations).

    Block-cyclic 1-D distribution of b-wide column blocks (block k on rank k mod G):
      1. right-looking blocked Cholesky: the owner of block k factors its diagonal block into
         X_kk = L_kk^{-1} (cggm_chol_inverse_dense: the recursive GEMM-rich factorisation), forms
         the panel L_{>k,k} = A_{>k,k} X_kk^T and broadcasts (X_kk, panel, log-det, PD flag); every
         rank applies the panel to the trailing block columns it owns (A_jj.. -= L_j,k L_jk^T);
      2. L^{-1} by owned column blocks: X_JJ = X_kk, then block forward substitution
         X_mJ = X_mm R_m, R_{>m} -= L_{>m,m} X_mJ over the panels every rank received in step 1;
      3. Sigma's lower column blocks Sigma_{>=J,J} = X_{>=J,>=J}^T X_{>=J,J} (the k-range starts at
         the row block: X is lower triangular), gathered and mirrored.
    Per rank (4/3) q^3 / G flop (+ the owners' b^3 diagonal blocks); exchanged: the panels (q^2/2),
    L^{-1} (q^2/2) and Sigma (q^2/2).  Every flop runs in the backend's kernels (libcggm for
    CudaBackend); the exchanges are torch.distributed broadcasts.

    backend: zeros(r, c), densify(Lam), chol_inverse(D) -> (X, logdet, is_pd, fail_col),
    gemm(C, A, B, transA, transB, alpha, beta, flags), symmetrize(S).
    """

    A_KLE_M, A_KGE_M, B_KLE_N, B_KGE_N = 1, 2, 4, 8

    def __init__(self, backend, block: int = 2048, group=None):
        self.b = backend
        self.block = int(block)
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.host = dist.is_initialized() and dist.get_backend(group) == "gloo"

    def _bcast(self, t, src):
        """Broadcast the (possibly strided) view t from group rank src into t on every rank."""
        if self.world == 1:
            return t
        gsrc = dist.get_global_rank(self.group, src) if self.group is not None else src
        buf = t.contiguous() if self.rank == src else torch.empty(t.shape, dtype=t.dtype, device=t.device)
        if self.host:
            h = buf.cpu()
            dist.broadcast(h, src=gsrc, group=self.group)
            buf = h.to(t.device)
        else:
            dist.broadcast(buf, src=gsrc, group=self.group)
        if self.rank != src:
            t.copy_(buf)
        return t

    def invert(self, Lam, want_sigma=True, want_linv=False):
        """(Sigma, logdet, is_pd, fail_col); want_linv: return the gathered L^{-1} instead of Sigma."""
        q = Lam.nrows
        b, G, me = self.block, self.world, self.rank
        blocks = [(k0, min(q, k0 + b)) for k0 in range(0, q, b)]
        K = len(blocks)
        owned = [k for k in range(K) if k % G == me]
        A = self.b.densify(Lam)                 # working copy; panels overwrite their block columns
        Xd = [None] * K
        logdet, fail = 0.0, -1
        scal = [None] * K

        def factor(k):   # owner of block k: X_kk, panel into A's block column, (log-det, PD, column)
            c0, c1 = blocks[k]
            bk = c1 - c0
            D = self.b.zeros(bk, bk)
            D.copy_(A[c0:c1, c0:c1])
            X_, ld_k, pd_k, fc_k = self.b.chol_inverse(D)
            Xd[k] = X_
            scal[k] = torch.tensor([ld_k, float(pd_k), float(fc_k)], dtype=torch.float64, device=X_.device)
            if c1 < q and pd_k:
                P = self.b.zeros(q - c1, bk)
                self.b.gemm(P, A[c1:, c0:c1], X_, transB=True, flags=self.B_KLE_N)   # L_{>k,k} = A_{>k,k} X_kk^T
                A[c1:, c0:c1].copy_(P)

        def update(j, k):   # block column j (owned) -= panel k's contribution
            c1 = blocks[k][1]
            d0, d1 = blocks[j]
            P = A[c1:, blocks[k][0]:c1]
            self.b.gemm(A[d0:, d0:d1], P[d0 - c1:], P[d0 - c1:d1 - c1], transB=True, alpha=-1.0, beta=1.0)

        if me == 0 % G:
            factor(0)
        for k, (c0, c1) in enumerate(blocks):
            o, bk = k % G, c1 - c0
            if me != o:
                Xd[k] = self.b.zeros(bk, bk)
                scal[k] = torch.zeros(3, dtype=torch.float64, device=Xd[k].device)
            self._bcast(scal[k], o)
            if scal[k][1] < 0.5:
                fail = c0 + int(scal[k][2])
                break
            logdet += float(scal[k][0])
            self._bcast(Xd[k], o)
            if c1 == q:
                continue
            self._bcast(A[c1:, c0:c1], o)
            # lookahead: the next block's owner applies this panel to that block and factors it
            # before its other trailing updates, so the next panel's broadcast is not held up
            if me == (k + 1) % G:
                update(k + 1, k)
                factor(k + 1)
            for j in owned:
                if j > k and not (j == k + 1 and me == (k + 1) % G):
                    update(j, k)
        if fail >= 0:
            return None, float("nan"), False, fail
        if not want_sigma and not want_linv:
            return None, logdet, True, -1
        # 2. L^{-1}, owned column blocks (X_JJ, then forward substitution over the panels)
        X = self.b.zeros(q, q)
        for J in owned:
            j0, j1 = blocks[J]
            X[j0:j1, j0:j1].copy_(Xd[J])
            if j1 == q:
                continue
            R = self.b.zeros(q - j1, j1 - j0)
            self.b.gemm(R, A[j1:, j0:j1], Xd[J], alpha=-1.0, flags=self.B_KGE_N)   # -L_{>J,J} X_JJ
            for m in range(J + 1, K):
                m0, m1 = blocks[m]
                Xm = X[m0:m1, j0:j1]
                self.b.gemm(Xm, Xd[m], R[m0 - j1:m1 - j1], flags=self.A_KLE_M)       # X_mJ = X_mm R_m
                if m1 < q:
                    self.b.gemm(R[m1 - j1:], A[m1:, m0:m1], Xm, alpha=-1.0, beta=1.0)
        for J, (j0, j1) in enumerate(blocks):
            self._bcast(X[j0:, j0:j1], J % G)
        if want_linv:
            return X, logdet, True, -1
        # 3. Sigma's lower column blocks, gathered, mirrored
        S = self.b.zeros(q, q)
        for J in owned:
            j0, j1 = blocks[J]
            self.b.gemm(S[j0:, j0:j1], X[j0:, j0:], X[j0:, j0:j1], transA=True, flags=self.A_KGE_M)
        for J, (j0, j1) in enumerate(blocks):
            self._bcast(S[j0:, j0:j1], J % G)
        self.b.symmetrize(S)
        return S, logdet, True, -1


# ------------------------------------------------------------------ all-reduce over peer memory
class PeerAllReduce:
    """Sum of same-shaped partials over the ranks of a node through CUDA IPC peer memory
    (cggm_peer_allreduce): every rank's partial lives in a symmetric buffer (a cggm_device_alloc
    allocation whose IPC handle every other rank opened), the GEMM writes into it directly, and
    rank r reduces slice r of all buffers in rank order into all buffers -- NVLink loads / stores
    between GPUs instead of an NCCL call, bit-identical on every rank.  Host barriers order the
    phases (no kernel waits on another rank's kernel)."""

    def __init__(self, ctx, group=None):
        import ctypes
        self.ctypes = ctypes
        self.ctx = ctx
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self._bufs = []   # (own pointer, ctypes pointer array, opened peer pointers)

    def empty(self, rows, cols, dtype=torch.float64):
        """A (rows, cols) column-major symmetric buffer (identical layout on every rank)."""
        ct = self.ctypes
        ld = rows + (rows & 1)
        nbytes = ld * max(cols, 1) * torch.empty(0, dtype=dtype).element_size()
        p = ct.c_void_p()
        self.ctx._check(self.ctx.lib.cggm_device_alloc(self.ctx.h, nbytes, ct.byref(p)))
        h = (ct.c_char * 64)()
        self.ctx._check(self.ctx.lib.cggm_ipc_get_handle(self.ctx.h, p, h))
        handles = [None] * self.world
        dist.all_gather_object(handles, bytes(h), group=self.group)
        ptrs, opened = [], []
        for k, hb in enumerate(handles):
            if k == self.rank:
                ptrs.append(p.value)
                continue
            q = ct.c_void_p()
            self.ctx._check(self.ctx.lib.cggm_ipc_open_handle(self.ctx.h, (ct.c_char * 64).from_buffer_copy(hb),
                                                              ct.byref(q)))
            ptrs.append(q.value)
            opened.append(q.value)
        arr = (ct.c_void_p * self.world)(*ptrs)
        count = ld * (max(cols, 1) - 1) + rows
        self._bufs.append((p.value, arr, opened, count))
        typestr = {torch.float64: "<f8", torch.float32: "<f4"}[dtype]
        es = torch.empty(0, dtype=dtype).element_size()

        class _Cai:
            __cuda_array_interface__ = {"shape": (rows, cols), "typestr": typestr, "data": (p.value, False),
                                        "version": 3, "strides": (es, ld * es)}
        t = torch.as_tensor(_Cai(), device=torch.device("cuda", self.ctx.device))
        t._peer_index = len(self._bufs) - 1
        return t

    def allreduce(self, t):
        own, arr, _, count = self._bufs[t._peer_index]
        torch.cuda.synchronize()
        dist.barrier(group=self.group)          # every partial is complete
        self.ctx._sync_stream()
        self.ctx._check(self.ctx.lib.cggm_peer_allreduce(self.ctx.h, self.world, self.rank, arr, count))
        torch.cuda.synchronize()
        dist.barrier(group=self.group)          # every slice is written everywhere
        return t

    def close(self):
        for own, _, opened, _ in self._bufs:
            for q in opened:
                self.ctx.lib.cggm_ipc_close_handle(self.ctx.h, self.ctypes.c_void_p(q))
        dist.barrier(group=self.group)
        for own, _, _, _ in self._bufs:
            self.ctx.lib.cggm_device_free(self.ctx.h, self.ctypes.c_void_p(own))
        self._bufs = []
