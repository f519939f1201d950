"""The sample-sharded evaluation (paper_1509_04681_b200/sharded.py) over a world-size-2 gloo
process group on CPU.  The per-rank compute is a test backend over the ORACLE (the product
path uses the CUDA backend with NCCL); what is tested here is the host logic: row partition,
global-n scaling (reading A21), which partials are all-reduced, the rank-0 inverse + broadcast,
and how the objective's partial traces combine.  Result must equal the unsharded oracle."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import cggm_oracle as O
from synth.cggm_inputs import Csc, csc_from_dense, make_problem


def col(a):
    return torch.from_numpy(np.asfortranarray(a))


class OracleBackend:
    def covariances_partial(self, X, Y, n_total):
        Syy, _ = O.covariances(X.numpy(), Y.numpy(), n_total=n_total)
        return col(Syy)

    def invert_logdet(self, Lam):
        S, ld, pd, fc = O.invert_logdet(Lam.to_dense())
        return col(S), ld, pd, fc

    def empty_sigma(self, q, like):
        return col(np.zeros((q, q)))

    def empty_matrix(self, rows, cols, like):
        return col(np.zeros((rows, cols)))

    def psi_grad_partial(self, X, Y, Theta, Sigma, n_total):
        Xn, Yn, S = X.numpy(), Y.numpy(), Sigma.numpy()
        W = O.spmm_x_theta(Xn, Theta)
        R = W @ S / math.sqrt(n_total)
        G, _ = O.grad_theta_residual_route(Xn, Yn, W, S, n_total=n_total)
        return col(R.T @ R), col(G)

    def grad_lambda(self, Syy, Sigma, Psi):
        return col(Syy.numpy() - Sigma.numpy() - Psi.numpy())

    def active_set(self, GradL, GradT, Lam, Theta, lam_L, lam_T, penalize_diag, tie_eps):
        return O.active_set(GradL.numpy(), GradT.numpy(), Lam, Theta, lam_L, lam_T, penalize_diag, tie_eps)

    def objective_partial(self, X, Y, Lam, Theta, lam_L, lam_T, penalize_diag, n_total):
        return O.objective(X.numpy(), Y.numpy(), Lam, Theta, lam_L, lam_T, penalize_diag, n_total=n_total)

    def _assemble(self, ob, group):
        """(test backend) the shards' trace partials all-reduced over gloo and f of Eq. 1 assembled --
        what the CUDA backend's collective cggm_objective does inside libcggm."""
        parts = torch.tensor([ob["tr_syy_lam"], ob["tr_sxy_theta"], ob["tr_sigma_m"]], dtype=torch.float64)
        dist.all_reduce(parts, group=group)
        ob = dict(ob)
        ob["tr_syy_lam"], ob["tr_sxy_theta"], ob["tr_sigma_m"] = (float(v) for v in parts.tolist())
        if ob["is_pd"]:
            ob["g"] = -ob["logdet"] + ob["tr_syy_lam"] + 2.0 * ob["tr_sxy_theta"] + ob["tr_sigma_m"]
            ob["f"] = ob["g"] + ob["pen_L"] + ob["pen_T"]
        return ob

    def objective_sharded(self, X, Y, Lam, Theta, lam_L, lam_T, penalize_diag, n_total, group, Linv=None,
                          logdet=None):
        if Linv is None:
            ob = self.objective_partial(X, Y, Lam, Theta, lam_L, lam_T, penalize_diag, n_total)
        else:
            ob = self.objective_given_inverse_partial(X, Y, Lam, Theta, lam_L, lam_T, penalize_diag, n_total, Linv,
                                                      logdet)
        return self._assemble(ob, group)

    # reduce-scatter grad_Theta path
    def psi_residual_partial(self, X, Y, Theta, Sigma, n_total):
        Xn, Yn, S = X.numpy(), Y.numpy(), Sigma.numpy()
        W = O.spmm_x_theta(Xn, Theta)
        R = W @ S / math.sqrt(n_total)
        _, E = O.grad_theta_residual_route(Xn, Yn, W, S, n_total=n_total)
        return col(R.T @ R), col(E)

    def grad_theta_block(self, X, E, c0, c1, n_total, out):
        out.copy_(torch.from_numpy((2.0 / n_total) * (X.numpy().T @ E.numpy()[:, c0:c1])))

    def active_lambda_only(self, GradL, Lam, lam_L, penalize_diag, tie_eps):
        q = GradL.shape[0]
        th = Csc(1, q, np.zeros(q + 1, dtype=np.int64), np.zeros(0, dtype=np.int32), np.zeros(0))
        a = O.active_set(GradL.numpy(), np.zeros((1, q)), Lam, th, lam_L, 1.0, penalize_diag, tie_eps)
        a["subgrad_l1"] = O.min_norm_subgradient(GradL.numpy(), np.zeros((1, q)), Lam, th, lam_L, 1.0, penalize_diag)
        return {k: (torch.from_numpy(v) if isinstance(v, np.ndarray) and v.ndim == 1 else v) for k, v in a.items()}

    def active_theta_block(self, G, Theta, c0, lam_T, tie_eps, T_row, T_col):
        p, nc = G.shape
        t = Theta.to_scipy()[:, c0:c0 + nc].tocsc()
        t.sort_indices()
        tb = Csc(p, nc, t.indptr.astype(np.int64), t.indices.astype(np.int32), t.data.copy())
        one = csc_from_dense(np.eye(nc))   # a zero-gradient identity Lambda block: no Theta influence
        a = O.active_set(np.zeros((nc, nc)), G.numpy(), one, tb, 0.0, lam_T, True, tie_eps)
        m = a["m_T"]
        if m > T_row.numel():   # the library's two-call pattern (CGGM_ERR_CAPACITY with the size)
            err = RuntimeError("capacity")
            err.m = m
            raise err
        T_row[:m].copy_(torch.from_numpy(a["T_row"]))
        T_col[:m].copy_(torch.from_numpy(a["T_col"] + c0))
        sub = O.min_norm_subgradient(np.zeros((nc, nc)), G.numpy(), one, tb, 0.0, lam_T)
        return m, a["ties_T"], sub

    def flat_zeros(self, count, like):
        return torch.zeros(count, dtype=torch.float64)

    def int_lists(self, cap, like):
        return torch.empty(cap, dtype=torch.int32), torch.empty(cap, dtype=torch.int32)


class OracleBackendBlocks(OracleBackend):
    """OracleBackend plus the dense building blocks the distributed inverse (NEXT-3) composes."""

    def __init__(self):
        from tests.test_distributed_inverse import OracleBlocks
        self._blk = OracleBlocks()

    def __getattr__(self, name):
        return getattr(self._blk, name)

    def objective_given_inverse_partial(self, X, Y, Lam, Theta, lam_L, lam_T, penalize_diag, n_total, Linv, logdet):
        """The shard's objective terms with tr(Sigma M) from the caller's (gathered) L^{-1}."""
        ob = dict(O.objective(X.numpy(), Y.numpy(), Lam, Theta, lam_L, lam_T, penalize_diag, n_total=n_total))
        Z = O.spmm_x_theta(X.numpy(), Theta) @ Linv.numpy().T
        ob["tr_sigma_m"] = float(np.sum(Z * Z)) / n_total
        ob["logdet"] = logdet
        return ob


def _worker(rank, world, port, name, k, q_out, split=True, distributed=False, grad_theta="allreduce", rs_width=7):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1509_04681_b200.sharded import ShardedEvaluator, shard_rows
        P = make_problem(name)
        _, lam, th = P.points[k]
        a, b = shard_rows(P.n, world, rank)
        X, Y = col(P.X[a:b]), col(P.Y[a:b])
        ev = ShardedEvaluator(OracleBackendBlocks() if distributed else OracleBackend(), split_objective=split,
                              distributed_inverse=distributed, block=16, grad_theta=grad_theta, rs_width=rs_width)
        ev.setup(X, Y, P.n)
        r = ev.evaluate(X, Y, lam, th, P.lam_L, P.lam_T, True)
        if rank == 0:
            a = r["active"]
            q_out.put({"Psi": r["Psi"].numpy().copy(), "GradL": r["GradL"].numpy().copy(),
                       "GradT": None if r["GradT"] is None else r["GradT"].numpy().copy(), "f": r["f"],
                       "logdet": r["logdet"], "m_L": a["m_L"], "m_T": a["m_T"],
                       "T_row": np.asarray(a["T_row"]).copy(), "T_col": np.asarray(a["T_col"]).copy(),
                       "L_row": np.asarray(a["L_row"]).copy(), "L_col": np.asarray(a["L_col"]).copy(),
                       "subgrad_l1": a.get("subgrad_l1")})
    finally:
        dist.destroy_process_group()


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("name,k,world,split,distributed", [("tiny", 1, 2, True, False), ("small", 1, 2, True, False),
                                                            ("tiny", 1, 2, False, False), ("tiny", 1, 3, True, False),
                                                            ("tiny", 1, 2, True, True), ("tiny", 1, 3, False, True)])
def test_sharded_matches_unsharded_oracle(name, k, world, split, distributed):
    """split: the objective rank evaluates the objective on the gathered full data while Sigma is
    formed (by rank 0, or by all ranks with the distributed inverse); otherwise every rank
    contributes partial traces of its own rows."""
    ctx = mp.get_context("spawn")
    qo = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, k, qo, split, distributed)) for r in range(world)]
    for p in procs:
        p.start()
    res = qo.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    P = make_problem(name)
    _, lam, th = P.points[k]
    Syy, Sxy = O.covariances(P.X, P.Y)
    S, ld, _, _ = O.invert_logdet(lam.to_dense())
    ref = O.psi_grad(P.X, P.Y, th, S, Syy, Sxy)
    ob = O.objective(P.X, P.Y, lam, th, P.lam_L, P.lam_T)
    a = O.active_set(ref["GradL"], ref["GradT"], lam, th, P.lam_L, P.lam_T)
    rel = lambda x, y: np.linalg.norm(x - y) / np.linalg.norm(y)
    assert rel(res["Psi"], ref["Psi"]) < 1e-12
    assert rel(res["GradL"], ref["GradL"]) < 1e-11
    if res["GradT"] is not None:
        assert rel(res["GradT"], ref["GradT"]) < 1e-11
    assert res["f"] == pytest.approx(ob["f"], rel=1e-12)
    assert res["logdet"] == pytest.approx(ld, rel=1e-14)
    if a["ties_L"] == 0 and a["ties_T"] == 0:
        assert (res["m_L"], res["m_T"]) == (a["m_L"], a["m_T"])


@pytest.mark.parametrize("name,k,world,split,rs_width", [("tiny", 1, 2, True, 7), ("tiny", 1, 3, False, 4),
                                                         ("small", 1, 2, True, 64), ("small", 0, 3, True, 1000)])
def test_sharded_reduce_scatter_grad_theta(name, k, world, split, rs_width):
    """grad_theta="reduce_scatter": the ranks own column ranges of grad_Theta, each round's partial
    column blocks are reduce-scattered (gloo: all-reduce + own block), compacted by the owner with
    global column indices and the compact S_Theta lists all-gathered -- no rank holds the p x q
    gradient.  Lists identical to the unsharded oracle's, statistic and f to rounding."""
    ctx = mp.get_context("spawn")
    qo = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, k, qo, split, False, "reduce_scatter", rs_width))
             for r in range(world)]
    for p in procs:
        p.start()
    res = qo.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    P = make_problem(name)
    _, lam, th = P.points[k]
    Syy, Sxy = O.covariances(P.X, P.Y)
    S, ld, _, _ = O.invert_logdet(lam.to_dense())
    ref = O.psi_grad(P.X, P.Y, th, S, Syy, Sxy)
    ob = O.objective(P.X, P.Y, lam, th, P.lam_L, P.lam_T)
    a = O.active_set(ref["GradL"], ref["GradT"], lam, th, P.lam_L, P.lam_T)
    sub = O.min_norm_subgradient(ref["GradL"], ref["GradT"], lam, th, P.lam_L, P.lam_T)
    assert res["GradT"] is None
    assert a["ties_L"] == 0 and a["ties_T"] == 0
    np.testing.assert_array_equal(res["T_row"], a["T_row"])
    np.testing.assert_array_equal(res["T_col"], a["T_col"])
    np.testing.assert_array_equal(res["L_row"], a["L_row"])
    np.testing.assert_array_equal(res["L_col"], a["L_col"])
    assert res["subgrad_l1"] == pytest.approx(sub, rel=1e-12)
    assert res["f"] == pytest.approx(ob["f"], rel=1e-12)


def test_shard_rows_partition():
    from paper_1509_04681_b200.sharded import shard_rows
    for n in (1, 7, 100, 1000, 4000):
        for w in (1, 2, 3, 4, 8):
            blocks = [shard_rows(n, w, r) for r in range(w)]
            assert blocks[0][0] == 0 and blocks[-1][1] == n
            assert all(blocks[i][1] == blocks[i + 1][0] for i in range(w - 1))
            sizes = [b - a for a, b in blocks]
            assert max(sizes) - min(sizes) <= 1


def test_flat_aliases_colmajor_storage():
    from paper_1509_04681_b200.sharded import flat
    base = torch.zeros(5, 8, dtype=torch.float64)   # cols=5, ld=8
    v = base.t()[:7, :5]                            # 7 x 5 column-major view, ld 8
    f = flat(v)
    f += 1.0
    assert torch.all(v == 1.0)
    assert f.numel() == 8 * 4 + 7
