"""The sample-sharded evaluator with the CUDA backend (libcggm) on two ranks.  Only one GPU is
available to the test suite, so both ranks share cuda:0 over a gloo group: a functional check of
the multi-rank CUDA path (row shards, rank-0 inverse + broadcast, rank-1 objective on the
gathered data, all-reduced partials), not a performance measurement.  Results must match the
single-process evaluation and the oracle."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, split, q_out, distributed=False, grad_theta="allreduce", rs_width=256):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_1509_04681_b200 import Context, DeviceCsc, to_device_colmajor
        from paper_1509_04681_b200.sharded import CudaBackend, ShardedEvaluator, shard_rows
        from synth.cggm_inputs import make_problem
        P = make_problem(name)
        _, lam, th = P.points[1 if name in ("tiny", "small") else 0]
        a, b = shard_rows(P.n, world, rank)
        X, Y = to_device_colmajor(P.X[a:b]), to_device_colmajor(P.Y[a:b])
        ctx = Context(0)
        ev = ShardedEvaluator(CudaBackend(ctx), split_objective=split, distributed_inverse=distributed, block=128,
                              grad_theta=grad_theta, rs_width=rs_width)
        ev.setup(X, Y, P.n)
        r = ev.evaluate(X, Y, DeviceCsc.from_host(lam), DeviceCsc.from_host(th), P.lam_L, P.lam_T, True)
        torch.cuda.synchronize()
        if rank == 0:
            act = r["active"]
            q_out.put({"Psi": r["Psi"].cpu().numpy(), "GradL": r["GradL"].cpu().numpy(),
                       "GradT": None if r["GradT"] is None else r["GradT"].cpu().numpy(),
                       "Sigma": r["Sigma"].cpu().numpy(), "f": r["f"],
                       "logdet": r["logdet"], "m_L": act["m_L"], "m_T": act["m_T"],
                       "lists": {k: act[k].cpu().numpy() for k in ("L_row", "L_col", "T_row", "T_col")},
                       "subgrad_l1": act["subgrad_l1"]})
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,split,distributed", [("small", True, False), ("small", False, False), ("tiny", True, False),
                                                    ("small", True, True), ("small", False, True)])
def test_two_ranks_match_oracle(name, split, distributed):
    import torch.multiprocessing as mp
    from oracle import cggm_oracle as O
    from synth.cggm_inputs import make_problem
    ctx = mp.get_context("spawn")
    qo = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, split, qo, distributed)) for r in range(2)]
    for p in procs:
        p.start()
    res = qo.get(timeout=600)
    for p in procs:
        p.join(timeout=600)
        assert p.exitcode == 0
    P = make_problem(name)
    _, lam, th = P.points[1]
    Syy, Sxy = O.covariances(P.X, P.Y)
    S, ld, _, _ = O.invert_logdet(lam.to_dense())
    ref = O.psi_grad(P.X, P.Y, th, S, Syy, Sxy)
    ob = O.objective(P.X, P.Y, lam, th, P.lam_L, P.lam_T)
    a = O.active_set(ref["GradL"], ref["GradT"], lam, th, P.lam_L, P.lam_T)
    rel = lambda x, y: np.linalg.norm(x - y) / np.linalg.norm(y)  # noqa: E731
    assert rel(res["Sigma"], S) <= 1e-9
    assert rel(res["Psi"], ref["Psi"]) <= 1e-9
    assert rel(res["GradL"], ref["GradL"]) <= 1e-9
    assert rel(res["GradT"], ref["GradT"]) <= 1e-9
    assert res["f"] == pytest.approx(ob["f"], rel=1e-10)
    assert res["logdet"] == pytest.approx(ld, rel=1e-12)
    if a["ties_L"] == 0 and a["ties_T"] == 0:
        assert (res["m_L"], res["m_T"]) == (a["m_L"], a["m_T"])


def _worker_lib(rank, world, port, name, q_out):
    """Collectives inside libcggm (cggm_comm_init_external over this gloo group)."""
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_1509_04681_b200 import Context, DeviceCsc, to_device_colmajor
        from paper_1509_04681_b200.sharded import CollectiveEvaluator, shard_rows
        from synth.cggm_inputs import make_problem
        P = make_problem(name)
        _, lam, th = P.points[1]
        a, b = shard_rows(P.n, world, rank)
        X, Y = to_device_colmajor(P.X[a:b]), to_device_colmajor(P.Y[a:b])
        ctx = Context(0)
        ctx.comm_init_torch()
        assert ctx.comm_info() == (rank, world)
        ev = CollectiveEvaluator(ctx)
        Syy = ev.setup(X, Y, P.n)
        r = ev.evaluate(X, Y, DeviceCsc.from_host(lam), DeviceCsc.from_host(th), P.lam_L, P.lam_T, True)
        # the one-GPU composite must refuse a multi-rank communicator
        from paper_1509_04681_b200.api import CggmError
        try:
            ctx.cggm_newton_eval(X, Y, Syy, DeviceCsc.from_host(lam), DeviceCsc.from_host(th), P.lam_L, P.lam_T)
            refused = False
        except CggmError as e:
            refused = e.status == 10
        torch.cuda.synchronize()
        q_out.put({"rank": rank, "Psi": r["Psi"].cpu().numpy(), "GradL": r["GradL"].cpu().numpy(),
                   "GradT": r["GradT"].cpu().numpy(), "Sigma": r["Sigma"].cpu().numpy(), "Syy": Syy.cpu().numpy(),
                   "f": r["f"], "logdet": r["logdet"], "is_pd": r["is_pd"], "m_L": r["active"]["m_L"],
                   "m_T": r["active"]["m_T"], "refused": refused})
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_library_collectives_match_oracle(world):
    """Every rank of the library-internal collective path ends with the unsharded results."""
    import torch.multiprocessing as mp
    from oracle import cggm_oracle as O
    from synth.cggm_inputs import make_problem
    ctx = mp.get_context("spawn")
    qo = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_lib, args=(r, world, port, "small", qo)) for r in range(world)]
    for p in procs:
        p.start()
    res = [qo.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=600)
        assert p.exitcode == 0
    P = make_problem("small")
    _, lam, th = P.points[1]
    Syy, Sxy = O.covariances(P.X, P.Y)
    S, ld, _, _ = O.invert_logdet(lam.to_dense())
    ref = O.psi_grad(P.X, P.Y, th, S, Syy, Sxy)
    ob = O.objective(P.X, P.Y, lam, th, P.lam_L, P.lam_T)
    a = O.active_set(ref["GradL"], ref["GradT"], lam, th, P.lam_L, P.lam_T)
    rel = lambda x, y: np.linalg.norm(x - y) / np.linalg.norm(y)  # noqa: E731
    for r in res:
        assert r["refused"]
        assert r["is_pd"]
        assert rel(r["Syy"], Syy) <= 1e-12
        assert rel(r["Sigma"], S) <= 1e-9
        assert rel(r["Psi"], ref["Psi"]) <= 1e-9
        assert rel(r["GradL"], ref["GradL"]) <= 1e-9
        assert rel(r["GradT"], ref["GradT"]) <= 1e-9
        assert r["f"] == pytest.approx(ob["f"], rel=1e-10)
        assert r["logdet"] == pytest.approx(ld, rel=1e-12)
        if a["ties_L"] == 0 and a["ties_T"] == 0:
            assert (r["m_L"], r["m_T"]) == (a["m_L"], a["m_T"])
    # every rank holds bit-identical results (one all-reduce / broadcast result)
    for r in res[1:]:
        for k in ("Sigma", "Psi", "GradL", "GradT"):
            assert np.array_equal(r[k], res[0][k]), k


def test_nccl_comm_single_rank_is_identity():
    """cggm_comm_init (NCCL, loaded at run time) with one rank: the collective calls run their NCCL
    all-reduce / broadcast and return exactly the single-GPU results."""
    import torch.distributed as dist
    from paper_1509_04681_b200 import Context, DeviceCsc, to_device_colmajor
    from paper_1509_04681_b200.sharded import CollectiveEvaluator
    from synth.cggm_inputs import make_problem
    P = make_problem("small")
    _, lam, th = P.points[1]
    X, Y = to_device_colmajor(P.X), to_device_colmajor(P.Y)
    L, T = DeviceCsc.from_host(lam), DeviceCsc.from_host(th)
    plain = Context(0)
    ev0 = CollectiveEvaluator(plain)
    ev0.setup(X, Y, P.n)
    r0 = ev0.evaluate(X, Y, L, T, P.lam_L, P.lam_T)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        c = Context(0)
        c.comm_init()
        assert c.comm_info() == (0, 1)
        ev = CollectiveEvaluator(c)
        ev.setup(X, Y, P.n)
        r = ev.evaluate(X, Y, L, T, P.lam_L, P.lam_T)
        for k in ("Sigma", "Psi", "GradL", "GradT"):
            assert torch.equal(r[k], r0[k]), k
        assert r["f"] == r0["f"] and r["logdet"] == r0["logdet"]
        c.comm_destroy()
        assert c.comm_info() == (0, 1)
    finally:
        dist.destroy_process_group()


def _worker_stream(rank, world, port, q_out):
    """cggm_psi_grad with the streamed grad_Theta (GradT = NULL, fused active sets) under the library
    collectives: each column chunk is all-reduced before its scan (medium: q = 4000, two chunks)."""
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_1509_04681_b200 import Context, DeviceCsc, to_device_colmajor
        from paper_1509_04681_b200.sharded import shard_rows
        from synth.cggm_inputs import make_problem
        P = make_problem("medium")
        _, lam, th = P.points[0]
        a, b = shard_rows(P.n, world, rank)
        X, Y = to_device_colmajor(P.X[a:b]), to_device_colmajor(P.Y[a:b])
        ctx = Context(0)
        ctx.comm_init_torch()
        Syy, _ = ctx.cggm_covariances(X, Y, n_total=P.n, want_sxy=False)
        L, T = DeviceCsc.from_host(lam), DeviceCsc.from_host(th)
        Sigma, _, _, _ = ctx.cggm_invert_logdet(L)
        cap = 2_000_000
        spec = dict(lam_L=P.lam_L, lam_T=P.lam_T, penalize_diag=1,
                    **{k: torch.empty(cap, dtype=torch.int32, device="cuda") for k in ("L_row", "L_col", "T_row", "T_col")})
        r = ctx.cggm_psi_grad(X, Y, T, Sigma, Syy=Syy, n_total=P.n, want_gradT=False, Lam=L, fused=spec)
        act = r["active"]
        torch.cuda.synchronize()
        q_out.put({"rank": rank, "m_L": act["m_L"], "m_T": act["m_T"], "ties": (act["ties_L"], act["ties_T"]),
                   "sub": act["subgrad_l1"], "T_row": act["T_row"].cpu().numpy(), "T_col": act["T_col"].cpu().numpy(),
                   "GradL": r["GradL"].cpu().numpy()})
    finally:
        dist.destroy_process_group()


def test_library_collectives_streamed_grad_theta():
    import torch.multiprocessing as mp
    from oracle import cggm_oracle as O
    from synth.cggm_inputs import make_problem
    ctx = mp.get_context("spawn")
    qo = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_stream, args=(r, 2, port, qo)) for r in range(2)]
    for p in procs:
        p.start()
    res = [qo.get(timeout=900) for _ in range(2)]
    for p in procs:
        p.join(timeout=900)
        assert p.exitcode == 0
    P = make_problem("medium")
    _, lam, th = P.points[0]
    Syy, Sxy = O.covariances(P.X, P.Y)
    S, _, _, _ = O.invert_logdet(lam.to_dense())
    ref = O.psi_grad(P.X, P.Y, th, S, Syy, Sxy)
    a = O.active_set(ref["GradL"], ref["GradT"], lam, th, P.lam_L, P.lam_T)
    sub = O.min_norm_subgradient(ref["GradL"], ref["GradT"], lam, th, P.lam_L, P.lam_T)
    for r in res:
        assert np.linalg.norm(r["GradL"] - ref["GradL"]) <= 1e-9 * np.linalg.norm(ref["GradL"])
        assert r["sub"] == pytest.approx(sub, rel=1e-9)
        if a["ties_L"] == 0 and a["ties_T"] == 0:
            assert (r["m_L"], r["m_T"]) == (a["m_L"], a["m_T"])
            assert np.array_equal(r["T_row"], a["T_row"]) and np.array_equal(r["T_col"], a["T_col"])
    assert (res[0]["m_L"], res[0]["m_T"], res[0]["ties"]) == (res[1]["m_L"], res[1]["m_T"], res[1]["ties"])
    assert np.array_equal(res[0]["T_row"], res[1]["T_row"])


def _worker_peer(rank, world, port, q_out):
    """Psi / grad_Theta partials summed over CUDA IPC peer memory (cggm_peer_allreduce)."""
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_1509_04681_b200 import Context, DeviceCsc, to_device_colmajor
        from paper_1509_04681_b200.sharded import CudaBackend, PeerAllReduce, ShardedEvaluator, shard_rows
        from synth.cggm_inputs import make_problem
        ctx = Context(0)
        # the primitive: random symmetric buffers, sum = the sum of every rank's seeded values
        pr = PeerAllReduce(ctx)
        buf = pr.empty(37, 5)
        g = torch.Generator().manual_seed(rank)
        buf.copy_(torch.randn(37, 5, generator=g, dtype=torch.float64))
        pr.allreduce(buf)
        ref = sum(torch.randn(37, 5, generator=torch.Generator().manual_seed(k), dtype=torch.float64)
                  for k in range(world))
        prim_ok = bool(torch.allclose(buf.cpu(), ref, rtol=1e-14, atol=1e-14))
        P = make_problem("small")
        _, lam, th = P.points[1]
        a, b = shard_rows(P.n, world, rank)
        X, Y = to_device_colmajor(P.X[a:b]), to_device_colmajor(P.Y[a:b])
        ev = ShardedEvaluator(CudaBackend(ctx), split_objective=False, peer_allreduce=True)
        ev.setup(X, Y, P.n)
        r = ev.evaluate(X, Y, DeviceCsc.from_host(lam), DeviceCsc.from_host(th), P.lam_L, P.lam_T, True)
        torch.cuda.synchronize()
        q_out.put({"rank": rank, "prim_ok": prim_ok, "Psi": r["Psi"].cpu().numpy().copy(),
                   "GradT": r["GradT"].cpu().numpy().copy(), "GradL": r["GradL"].cpu().numpy().copy(),
                   "f": r["f"]})
        pr.close()
        ev.peer.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_peer_allreduce_matches_oracle(world):
    import torch.multiprocessing as mp
    from oracle import cggm_oracle as O
    from synth.cggm_inputs import make_problem
    ctx = mp.get_context("spawn")
    qo = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_peer, args=(r, world, port, qo)) for r in range(world)]
    for p in procs:
        p.start()
    res = [qo.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=600)
        assert p.exitcode == 0
    P = make_problem("small")
    _, lam, th = P.points[1]
    Syy, Sxy = O.covariances(P.X, P.Y)
    S, _, _, _ = O.invert_logdet(lam.to_dense())
    ref = O.psi_grad(P.X, P.Y, th, S, Syy, Sxy)
    ob = O.objective(P.X, P.Y, lam, th, P.lam_L, P.lam_T)
    rel = lambda x, y: np.linalg.norm(x - y) / np.linalg.norm(y)  # noqa: E731
    for r in res:
        assert r["prim_ok"]
        assert rel(r["Psi"], ref["Psi"]) <= 1e-9
        assert rel(r["GradT"], ref["GradT"]) <= 1e-9
        assert rel(r["GradL"], ref["GradL"]) <= 1e-9
        assert r["f"] == pytest.approx(ob["f"], rel=1e-10)
    for r in res[1:]:
        assert np.array_equal(r["Psi"], res[0]["Psi"]) and np.array_equal(r["GradT"], res[0]["GradT"])


@pytest.mark.parametrize("name,world,rs_width", [("small", 2, 128), ("small", 3, 100), ("medium", 2, 512),
                                                 ("medium", 3, 256)])
def test_reduce_scatter_grad_theta_matches_oracle(name, world, rs_width):
    """grad_theta="reduce_scatter" with the CUDA backend: column ranges of grad_Theta reduce-scattered
    round by round (cggm_psi_residual, cggm_gemm blocks, cggm_active_theta_block compaction with global
    column indices), compact S_Theta lists all-gathered -- no rank holds a p x q buffer.  Lists equal
    the oracle's exactly outside the tie band, statistic and f to rounding; ranks share
    cuda:0 over gloo (functional check)."""
    import torch.multiprocessing as mp
    from oracle import cggm_oracle as O
    from synth.cggm_inputs import make_problem
    ctx = mp.get_context("spawn")
    qo = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, True, qo, False, "reduce_scatter", rs_width))
             for r in range(world)]
    for p in procs:
        p.start()
    res = qo.get(timeout=900)
    for p in procs:
        p.join(timeout=900)
        assert p.exitcode == 0
    P = make_problem(name)
    _, lam, th = P.points[1 if name in ("tiny", "small") else 0]
    Syy, Sxy = O.covariances(P.X, P.Y)
    S, ld, _, _ = O.invert_logdet(lam.to_dense())
    ref = O.psi_grad(P.X, P.Y, th, S, Syy, Sxy)
    ob = O.objective(P.X, P.Y, lam, th, P.lam_L, P.lam_T)
    a = O.active_set(ref["GradL"], ref["GradT"], lam, th, P.lam_L, P.lam_T)
    sub = O.min_norm_subgradient(ref["GradL"], ref["GradT"], lam, th, P.lam_L, P.lam_T)
    assert res["GradT"] is None
    for rk, ck, tm in (("L_row", "L_col", a["tie_mask_L"]), ("T_row", "T_col", a["tie_mask_T"])):
        g = set(zip(res["lists"][rk].tolist(), res["lists"][ck].tolist()))
        o = set(zip(a[rk].tolist(), a[ck].tolist()))
        for (i, j) in g ^ o:
            assert tm[i, j], (rk, i, j)
        key = res["lists"][ck].astype(np.int64) * (1 << 31) + res["lists"][rk]
        assert np.all(np.diff(key) > 0)
    assert res["subgrad_l1"] == pytest.approx(sub, rel=1e-9)
    assert res["f"] == pytest.approx(ob["f"], rel=1e-10)
