"""K01: S_Theta (readings A5-A7), its tie count and the min-norm subgradient's Theta part
 selected in the X^T E GEMM epilogue while each tile of grad_Theta = (2/n) X^T E is in shared
memory -- grad_Theta is never stored (cggm_psi_grad / cggm_newton_eval with GradT = NULL, FP64,
CGGM_K01=1; the default GradT = NULL path streams column chunks through the scan instead).

The epilogue takes the same per-element decisions on the same gradient values as the scan of a
stored gradient, so the lists, counts and tie counts must be bit-identical to the stored path (itself
checked against the oracle at edge shapes in test_gpu_active_edges.py) and to the oracle's lists
outside the tie band; only the subgradient's summation order differs.  Shapes straddle the 64-row
chunk and the 128 x 64 / 64 x 64 output tiles, with supports holding explicit zeros and both signs."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import cggm_oracle as O  # noqa: E402
from synth.cggm_inputs import csc_from_triplets, make_problem  # noqa: E402


@pytest.fixture(scope="module")
def ctx():
    """A context with K01 on (CGGM_K01=1; off by default: measured slower than the stored scan)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import os
    from paper_1509_04681_b200 import Context
    os.environ["CGGM_K01"] = "1"
    try:
        return Context(0)
    finally:
        os.environ.pop("CGGM_K01", None)


def _case(n, p, q, seed):
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n, p))
    Y = rng.standard_normal((n, q))
    S = rng.standard_normal((q, q)) / np.sqrt(q)
    Sigma = S @ S.T + np.eye(q)
    rows, cols, vals = [], [], []
    for j in range(q):
        k = int(rng.integers(0, min(p, 6) + 1))
        for i in sorted(rng.choice(p, size=k, replace=False).tolist()):
            rows.append(i)
            cols.append(j)
            u = rng.uniform(0.2, 1.0) * rng.choice([-1.0, 1.0])
            vals.append(0.0 if rng.uniform() < 0.15 else u)   # explicit stored zeros (reading A7)
    th = csc_from_triplets(p, q, rows, cols, vals)
    L = np.eye(q) * 2.0
    lam = csc_from_triplets(q, q, list(range(q)), list(range(q)), [2.0] * q)
    W = X @ th.to_dense()
    G = (2.0 / n) * X.T @ (Y + W @ Sigma)     # grad_Theta (identity I6)
    lam_T = float(np.quantile(np.abs(G), 0.6)) if G.size else 0.1
    return X, Y, Sigma, th, lam, L, G, lam_T


def _run(ctx, X, Y, Sigma, th, lam, lam_T, stored):
    from paper_1509_04681_b200 import DeviceCsc, to_device_colmajor
    n, p = X.shape
    q = Y.shape[1]
    Xd, Yd, Sd = to_device_colmajor(X), to_device_colmajor(Y), to_device_colmajor(Sigma)
    Syy = to_device_colmajor(Y.T @ Y / n)
    cap = 4 * p * q + 1024
    spec = dict(lam_L=1e9, lam_T=lam_T, penalize_diag=1, tie_eps=1e-9,
                L_row=torch.empty(4 * q * q + 64, dtype=torch.int32, device="cuda"),
                L_col=torch.empty(4 * q * q + 64, dtype=torch.int32, device="cuda"),
                T_row=torch.empty(cap, dtype=torch.int32, device="cuda"),
                T_col=torch.empty(cap, dtype=torch.int32, device="cuda"))
    r = ctx.cggm_psi_grad(Xd, Yd, DeviceCsc.from_host(th), Sd, Syy=Syy, Lam=DeviceCsc.from_host(lam), fused=spec,
                          want_gradT=stored)
    torch.cuda.synchronize()
    a = r["active"]
    m = int(a["m_T"])
    return dict(rows=a["T_row"][:m].cpu().numpy(), cols=a["T_col"][:m].cpu().numpy(), m=m, ties=int(a["ties_T"]),
                sub=float(a["subgrad_l1"]), m_L=int(a["m_L"]), GradT=r["GradT"])


SHAPES = [(8, 1, 1), (20, 63, 5), (40, 64, 65), (50, 129, 70), (64, 200, 130), (100, 1000, 257), (33, 300, 1)]


@pytest.mark.parametrize("n,p,q", SHAPES)
def test_epilogue_selection_matches_stored_scan_and_oracle(ctx, n, p, q):
    X, Y, Sigma, th, lam, L, G, lam_T = _case(n, p, q, seed=n * 7 + p + 3 * q)
    a = _run(ctx, X, Y, Sigma, th, lam, lam_T, stored=True)
    b = _run(ctx, X, Y, Sigma, th, lam, lam_T, stored=False)
    assert b["GradT"] is None
    np.testing.assert_array_equal(a["rows"], b["rows"])
    np.testing.assert_array_equal(a["cols"], b["cols"])
    assert (a["m"], a["ties"], a["m_L"]) == (b["m"], b["ties"], b["m_L"])
    assert b["sub"] == pytest.approx(a["sub"], rel=1e-13, abs=1e-300)
    # the plain definition (oracle): |g| > lam or a stored nonzero, column-major order; entries inside
    # the 1e-9 tie band may go either way
    Gd = a["GradT"].cpu().numpy()
    assert np.linalg.norm(Gd - G) <= 1e-12 * max(1.0, np.linalg.norm(G))
    Th = th.to_dense()
    want = (np.abs(G) > lam_T) | (Th != 0)
    tie = np.abs(np.abs(G) - lam_T) <= 1e-9
    got = np.zeros_like(want)
    got[b["rows"], b["cols"]] = True
    assert not np.any((got != want) & ~tie)
    key = b["cols"].astype(np.int64) * (1 << 31) + b["rows"]
    assert np.all(np.diff(key) > 0)


@pytest.mark.parametrize("name,k", [("tiny", 0), ("tiny", 1), ("small", 0), ("small", 1)])
def test_newton_evaluation_without_stored_grad_theta_vs_oracle(ctx, name, k):
    """The composite evaluation with GradT = NULL (K01) against the oracle's lists and statistic."""
    from paper_1509_04681_b200 import DeviceCsc, to_device_colmajor
    from paper_1509_04681_b200.api import newton_evaluation
    P = make_problem(name)
    label, lam, th = P.points[k]
    X, Y = to_device_colmajor(P.X), to_device_colmajor(P.Y)
    Lg, Tg = DeviceCsc.from_host(lam), DeviceCsc.from_host(th)
    Syy, _ = ctx.cggm_covariances(X, Y, want_sxy=False)
    bufs = {kk: torch.empty(2_000_000, dtype=torch.int32, device="cuda") for kk in ("L_row", "L_col", "T_row", "T_col")}
    r = newton_evaluation(ctx, X, Y, Syy, Lg, Tg, P.lam_L, P.lam_T, True, bufs, stream_grad_theta=True)
    assert r["GradT"] is None
    Syy_o, Sxy_o = O.covariances(P.X, P.Y)
    Sig_o, _, _, _ = O.invert_logdet(lam.to_dense())
    ro = O.psi_grad(P.X, P.Y, th, Sig_o, Syy_o, Sxy_o)
    ao = O.active_set(ro["GradL"], ro["GradT"], lam, th, P.lam_L, P.lam_T, True, 1e-9)
    sub = O.min_norm_subgradient(ro["GradL"], ro["GradT"], lam, th, P.lam_L, P.lam_T, True)
    tie = np.abs(np.abs(ro["GradT"]) - P.lam_T) <= 1e-9
    a = r["active"]
    m = int(a["m_T"])
    g = set(zip(a["T_row"][:m].cpu().numpy().tolist(), a["T_col"][:m].cpu().numpy().tolist()))
    o = set(zip(ao["T_row"].tolist(), ao["T_col"].tolist()))
    for (i, j) in g ^ o:
        assert tie[i, j]
    assert a["subgrad_l1"] == pytest.approx(sub, rel=1e-9)
