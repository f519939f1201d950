"""NEXT-3 on the GPU: the dense building blocks behind the C-ABI (cggm_gemm with its structural
flags, cggm_chol_inverse_dense, cggm_symmetrize, cggm_densify) against plain products / the oracle,
and DistributedInverse with the CUDA backend on 1-3 ranks sharing cuda:0 over gloo (a functional
check of the distributed path; NCCL refuses several ranks on one device)."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import cggm_oracle as O  # noqa: E402
from synth.cggm_inputs import csc_from_triplets  # noqa: E402


def random_spd(q, seed, dens=0.05):
    rng = np.random.default_rng(seed)
    B = np.where(rng.random((q, q)) < dens, rng.standard_normal((q, q)), 0.0)
    return B @ B.T + q * 0.05 * np.eye(q)


def to_csc(A):
    r, c = np.nonzero(A)
    return csc_from_triplets(A.shape[0], A.shape[1], r, c, A[r, c])


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1509_04681_b200 import Context
    return Context(0)


def test_building_blocks(ctx):
    from paper_1509_04681_b200 import DeviceCsc, to_device_colmajor
    from paper_1509_04681_b200.api import colmajor_empty
    rng = np.random.default_rng(3)
    A = random_spd(300, 1)
    D = ctx.cggm_densify(DeviceCsc.from_host(to_csc(A)))
    assert np.array_equal(D.cpu().numpy(), A)
    L_ref, pd, _ = O.cholesky(A)
    X, ld, ok, fc = ctx.cggm_chol_inverse_dense(to_device_colmajor(A))
    Xr = O.forward_substitution(L_ref, np.eye(300))
    assert ok and fc == -1
    assert np.linalg.norm(np.tril(X.cpu().numpy()) - Xr) <= 1e-12 * np.linalg.norm(Xr)
    assert np.array_equal(np.triu(X.cpu().numpy(), 1), np.zeros((300, 300)))
    assert ld == pytest.approx(O.logdet_from_cholesky(L_ref), rel=1e-13)
    # gemm with a declared lower-triangular op(B) on an odd-offset (unaligned) operand view
    M, N, K = 97, 65, 65
    Ah = rng.standard_normal((M + 1, K))
    Bh = np.tril(rng.standard_normal((N, K)))
    Ad, Bd = to_device_colmajor(Ah), to_device_colmajor(Bh)
    C = colmajor_empty(M, N)
    C.copy_(torch.from_numpy(rng.standard_normal((M, N))))
    C0 = C.cpu().numpy().copy()
    ctx.cggm_gemm(C, Ad[1:], Bd, transB=True, alpha=-0.5, beta=2.0, flags=4)   # B_KLE_N: op(B) = B^T upper
    ref = -0.5 * Ah[1:] @ Bh.T + 2.0 * C0
    assert np.abs(C.cpu().numpy() - ref).max() <= 1e-12 * np.abs(ref).max()
    S = to_device_colmajor(np.tril(rng.standard_normal((130, 130))))
    ctx.cggm_symmetrize(S)
    Sh = S.cpu().numpy()
    assert np.array_equal(Sh, Sh.T)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, A, block, q_out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_1509_04681_b200 import Context, DeviceCsc
        from paper_1509_04681_b200.sharded import CudaBackend, DistributedInverse
        ctx = Context(0)
        S, ld, pd, fc = DistributedInverse(CudaBackend(ctx), block=block).invert(DeviceCsc.from_host(to_csc(A)))
        torch.cuda.synchronize()
        q_out.put((rank, None if S is None else S.cpu().numpy(), ld, pd, fc))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,q,block", [(1, 300, 64), (2, 500, 128), (3, 515, 128), (2, 1100, 256)])
def test_distributed_inverse_cuda(world, q, block):
    import torch.multiprocessing as mp
    A = random_spd(q, seed=q)
    ctx = mp.get_context("spawn")
    qo = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, A, block, qo)) for r in range(world)]
    for p in ps:
        p.start()
    res = [qo.get(timeout=600) for _ in range(world)]
    for p in ps:
        p.join(timeout=600)
        assert p.exitcode == 0
    S_ref, ld_ref, pd_ref, _ = O.invert_logdet(A)
    for _, S, ld, pd, fc in res:
        assert pd and fc == -1
        assert np.linalg.norm(S - S_ref) <= 1e-10 * np.linalg.norm(S_ref)
        assert np.array_equal(S, S.T)
        assert ld == pytest.approx(ld_ref, rel=1e-12)
    for r in res[1:]:
        assert np.array_equal(r[1], res[0][1])


def test_distributed_inverse_cuda_non_pd():
    import torch.multiprocessing as mp
    q, fail_at = 400, 211
    A = random_spd(q, seed=9)
    L, _, _ = O.cholesky(A)
    A[fail_at, fail_at] = float(np.dot(L[fail_at, :fail_at], L[fail_at, :fail_at])) - 1.0
    ctx = mp.get_context("spawn")
    qo = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, A, 64, qo)) for r in range(2)]
    for p in ps:
        p.start()
    res = [qo.get(timeout=600) for _ in range(2)]
    for p in ps:
        p.join(timeout=600)
        assert p.exitcode == 0
    for _, S, ld, pd, fc in res:
        assert not pd and fc == fail_at and S is None


def test_objective_given_inverse_matches_objective(ctx):
    """cggm_objective_given_inverse with L^{-1} and log|Lambda| from cggm_chol_inverse_dense equals
    cggm_objective (its own factorisation) and the oracle."""
    from paper_1509_04681_b200 import DeviceCsc, to_device_colmajor
    from synth.cggm_inputs import make_problem
    P = make_problem("small")
    _, lam, th = P.points[1]
    X, Y = to_device_colmajor(P.X), to_device_colmajor(P.Y)
    L, T = DeviceCsc.from_host(lam), DeviceCsc.from_host(th)
    a = ctx.cggm_objective(X, Y, L, T, P.lam_L, P.lam_T)
    D = ctx.cggm_densify(L)
    Linv, ld, pd, _ = ctx.cggm_chol_inverse_dense(D)
    assert pd
    b = ctx.cggm_objective_given_inverse(X, Y, L, T, P.lam_L, P.lam_T, Linv, ld)
    ref = O.objective(P.X, P.Y, lam, th, P.lam_L, P.lam_T)
    for k in ("f", "g", "tr_syy_lam", "tr_sxy_theta", "tr_sigma_m", "pen_L", "pen_T", "logdet"):
        assert b[k] == pytest.approx(a[k], rel=1e-12), k
        assert b[k] == pytest.approx(ref[k], rel=1e-10), k


def test_building_block_errors_and_non_pd(ctx):
    """Argument errors of the building blocks are reported before any launch; a non-PD block is not
    an error (is_pd = 0 and the first failing column, reading A10)."""
    from paper_1509_04681_b200 import to_device_colmajor
    from paper_1509_04681_b200.api import CggmError, colmajor_empty
    C = colmajor_empty(64, 64)
    with pytest.raises(CggmError) as e:
        ctx.cggm_gemm(C, C, C)                      # output aliases an operand
    assert e.value.status == 1
    with pytest.raises(CggmError) as e:
        ctx.cggm_gemm(C, C, C, flags=1 << 7)        # unknown flag
    assert e.value.status == 1
    A = random_spd(97, 4)
    L, _, _ = O.cholesky(A)
    A[50, 50] = float(np.dot(L[50, :50], L[50, :50])) - 1.0
    X, ld, pd, fc = ctx.cggm_chol_inverse_dense(to_device_colmajor(A))
    assert not pd and fc == 50
    odd = torch.zeros((97, 97), dtype=torch.float64, device="cuda").t()   # ld 97: odd
    with pytest.raises(CggmError) as e:
        ctx.cggm_chol_inverse_dense(odd)
    assert e.value.status == 1
