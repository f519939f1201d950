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


def _worker(rank, world, port, name, split, q_out):
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
        ev = ShardedEvaluator(CudaBackend(ctx), split_objective=split)
        ev.setup(X, Y, P.n)
        r = ev.evaluate(X, Y, DeviceCsc.from_host(lam), DeviceCsc.from_host(th), P.lam_L, P.lam_T, True)
        torch.cuda.synchronize()
        if rank == 0:
            q_out.put({"Psi": r["Psi"].cpu().numpy(), "GradL": r["GradL"].cpu().numpy(),
                       "GradT": r["GradT"].cpu().numpy(), "Sigma": r["Sigma"].cpu().numpy(), "f": r["f"],
                       "logdet": r["logdet"], "m_L": r["active"]["m_L"], "m_T": r["active"]["m_T"]})
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,split", [("small", True), ("small", False), ("tiny", True)])
def test_two_ranks_match_oracle(name, split):
    import torch.multiprocessing as mp
    from oracle import cggm_oracle as O
    from synth.cggm_inputs import make_problem
    ctx = mp.get_context("spawn")
    qo = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, split, qo)) for r in range(2)]
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
