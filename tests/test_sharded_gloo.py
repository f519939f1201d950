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
from synth.cggm_inputs import make_problem


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


def _worker(rank, world, port, name, k, q_out, split=True, distributed=False):
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
                              distributed_inverse=distributed, block=16)
        ev.setup(X, Y, P.n)
        r = ev.evaluate(X, Y, lam, th, P.lam_L, P.lam_T, True)
        if rank == 0:
            q_out.put({"Psi": r["Psi"].numpy().copy(), "GradL": r["GradL"].numpy().copy(),
                       "GradT": r["GradT"].numpy().copy(), "f": r["f"], "logdet": r["logdet"],
                       "m_L": r["active"]["m_L"], "m_T": r["active"]["m_T"]})
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
    assert rel(res["GradT"], ref["GradT"]) < 1e-11
    assert res["f"] == pytest.approx(ob["f"], rel=1e-12)
    assert res["logdet"] == pytest.approx(ld, rel=1e-14)
    if a["ties_L"] == 0 and a["ties_T"] == 0:
        assert (res["m_L"], res["m_T"]) == (a["m_L"], a["m_T"])


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
