"""NEXT-3: the block-cyclic distributed factorisation and inverse of Lambda
(paper_1509_04681_b200/sharded.py DistributedInverse) over gloo process groups of 1-3 ranks on
CPU.  The per-block compute is a test backend over the ORACLE's unblocked Cholesky and plain
products, so what is tested is the distributed algorithm itself: block ownership, the panel
broadcasts, the trailing updates, the forward substitution for L^{-1} over the gathered panels, the
triangular k-ranges it declares, Sigma's gather and mirror, and the PD failure column.  Sigma must
equal the unblocked oracle inverse, log|Lambda| its log-det, and a non-PD Lambda must report the
same first failing column as the unblocked Cholesky (reading A10)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import cggm_oracle as O
from synth.cggm_inputs import csc_from_triplets, make_problem


def colmajor_zeros(r, c):
    return torch.zeros((max(c, 1), max(r, 1)), dtype=torch.float64).t()[:r, :c]


class OracleBlocks:
    """Dense building blocks on CPU tensors; gemm honours the declared structural zeros by zeroing
    the skipped operand entries first, so a wrong flag shows up as a wrong result."""

    def zeros(self, r, c):
        return colmajor_zeros(r, c)

    def densify(self, lam):
        D = colmajor_zeros(lam.nrows, lam.ncols)
        D.copy_(torch.from_numpy(lam.to_dense()))
        return D

    def chol_inverse(self, D):
        L, pd, fc = O.cholesky(D.numpy().copy())
        X = colmajor_zeros(*D.shape)
        if pd:
            X.copy_(torch.from_numpy(O.forward_substitution(L, np.eye(L.shape[0]))))
            return X, O.logdet_from_cholesky(L), True, -1
        return X, float("nan"), False, fc

    def gemm(self, C, A, B, transA=False, transB=False, alpha=1.0, beta=0.0, flags=0):
        a = (A.t() if transA else A).clone()
        b = (B.t() if transB else B).clone()
        m, k = a.shape
        n = b.shape[1]
        ii = torch.arange(m).unsqueeze(1)
        kk = torch.arange(k).unsqueeze(0)
        if flags & 1:
            a[kk.expand(m, k) > ii.expand(m, k)] = 0.0
        if flags & 2:
            a[kk.expand(m, k) < ii.expand(m, k)] = 0.0
        kr = torch.arange(k).unsqueeze(1)
        nn = torch.arange(n).unsqueeze(0)
        if flags & 4:
            b[kr.expand(k, n) > nn.expand(k, n)] = 0.0
        if flags & 8:
            b[kr.expand(k, n) < nn.expand(k, n)] = 0.0
        C.copy_(alpha * (a @ b) + (beta * C if beta != 0.0 else 0.0))
        return C

    def symmetrize(self, S):
        lo = torch.tril(S, -1)
        S.copy_(torch.tril(S) + lo.t())
        return S


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, lam, block, q_out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1509_04681_b200.sharded import DistributedInverse
        S, ld, pd, fc = DistributedInverse(OracleBlocks(), block=block).invert(lam)
        q_out.put((rank, None if S is None else S.numpy().copy(), ld, pd, fc))
    finally:
        dist.destroy_process_group()


def run(world, lam, block):
    ctx = mp.get_context("spawn")
    qo = ctx.Queue()
    port = free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, lam, block, qo)) for r in range(world)]
    for p in ps:
        p.start()
    res = [qo.get(timeout=300) for _ in range(world)]
    for p in ps:
        p.join(timeout=300)
        assert p.exitcode == 0
    return sorted(res, key=lambda r: r[0])


def random_spd_csc(q, seed, dens=0.05):
    rng = np.random.default_rng(seed)
    B = np.where(rng.random((q, q)) < dens, rng.standard_normal((q, q)), 0.0)
    A = B @ B.T + q * 0.05 * np.eye(q)
    r, c = np.nonzero(A)
    return csc_from_triplets(q, q, r, c, A[r, c])


@pytest.mark.parametrize("world,q,block", [(1, 70, 16), (2, 70, 16), (3, 101, 16), (2, 64, 64), (3, 40, 64)])
def test_distributed_inverse_matches_oracle(world, q, block):
    lam = random_spd_csc(q, seed=q + world)
    res = run(world, lam, block)
    S_ref, ld_ref, pd_ref, _ = O.invert_logdet(lam.to_dense())
    assert pd_ref
    for _, S, ld, pd, fc in res:
        assert pd and fc == -1
        assert np.linalg.norm(S - S_ref) <= 1e-11 * np.linalg.norm(S_ref)
        assert np.array_equal(S, S.T)
        assert ld == pytest.approx(ld_ref, rel=1e-12)


def test_distributed_inverse_chain_closed_form():
    """The chain Lambda (pin P3/P4): log-det ln((1 - phi^{2q+2}) / (1 - phi^2)), Sigma closed form."""
    P = make_problem("tiny")
    lam = P.points[0][1] if P.points[0][0] == "truth" else P.points[1][1]
    q = lam.nrows
    phi = 0.5
    res = run(2, lam, 8)
    i = np.arange(1, q + 1)
    I, J = np.meshgrid(i, i, indexing="ij")
    lo, hi = np.minimum(I, J), np.maximum(I, J)
    S_cf = (phi ** (hi - lo) - phi ** (lo + hi)) * (1 - phi ** (2 * (q + 1 - hi))) / ((1 - phi ** 2) * (1 - phi ** (2 * (q + 1))))
    ld_cf = np.log((1 - phi ** (2 * q + 2)) / (1 - phi ** 2))
    for _, S, ld, pd, _ in res:
        if not np.allclose(lam.to_dense(), lam.to_dense().T) or abs(lam.to_dense()[0, 0] - 1.25) > 1e-12:
            pytest.skip("tiny's truth Lambda is not the chain")
        assert np.abs(S - S_cf).max() <= 1e-13
        assert ld == pytest.approx(ld_cf, rel=1e-13)


@pytest.mark.parametrize("world,fail_at", [(2, 37), (3, 5), (3, 60)])
def test_distributed_inverse_reports_first_failing_column(world, fail_at):
    """A Lambda whose leading (fail_at x fail_at) block is PD but the next pivot is not: the same
    first failing column as the unblocked Cholesky, on every rank."""
    q = 70
    lam0 = random_spd_csc(q, seed=7)
    A = lam0.to_dense()
    # make the pivot at fail_at negative: A_jj := sum_{k<j} L_jk^2 - 1
    L, _, _ = O.cholesky(A)
    A[fail_at, fail_at] = float(np.dot(L[fail_at, :fail_at], L[fail_at, :fail_at])) - 1.0
    r, c = np.nonzero(A)
    lam = csc_from_triplets(q, q, r, c, A[r, c])
    _, pd_ref, fc_ref = O.cholesky(A)
    assert not pd_ref and fc_ref == fail_at
    for _, S, ld, pd, fc in run(world, lam, 16):
        assert not pd and fc == fail_at and S is None
