"""GPU parity of the coordinate-descent consumers (NEXT-1 / NEXT-2) with the oracle
(oracle/ancd_oracle.py) on the same seeded inputs and the same (GPU-selected) active lists:
the Lambda direction sweep, the line-search candidate CSC, the Theta sweep, and Algorithm 1's
iterates.  The sweeps are sequential in the same order on both sides; only the summation order of
the dot products differs, so the tolerances are near machine precision."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import ancd_oracle as A  # noqa: E402
from oracle import cggm_oracle as O  # noqa: E402
from synth.cggm_inputs import make_problem  # noqa: E402


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1509_04681_b200 import Context
    return Context(0)


_P = {}


def problem(name):
    if name not in _P:
        _P[name] = make_problem(name)
    return _P[name]


def _gpu_state(ctx, P, k):
    """Sigma, Psi, gradients and active lists of point k on the GPU (the lists both sides use)."""
    from paper_1509_04681_b200 import DeviceCsc, to_device_colmajor
    label, lam, th = P.points[k]
    X, Y = to_device_colmajor(P.X), to_device_colmajor(P.Y)
    Lg, Tg = DeviceCsc.from_host(lam), DeviceCsc.from_host(th)
    Syy, Sxy = ctx.cggm_covariances(X, Y)
    Sigma, _, _, _ = ctx.cggm_invert_logdet(Lg)
    cap = 2_000_000
    spec = dict(lam_L=P.lam_L, lam_T=P.lam_T, penalize_diag=1,
                **{k2: torch.empty(cap, dtype=torch.int32, device="cuda") for k2 in ("L_row", "L_col", "T_row", "T_col")})
    r = ctx.cggm_psi_grad(X, Y, Tg, Sigma, Syy=Syy, Sxy=Sxy, Lam=Lg, fused=spec)
    return dict(X=X, Y=Y, Lg=Lg, Tg=Tg, Syy=Syy, Sxy=Sxy, Sigma=Sigma, lam=lam, th=th, **r)


@pytest.mark.parametrize("name,k", [("tiny", 1), ("small", 1), ("small", 0)])
def test_lambda_direction_matches_oracle(ctx, name, k):
    P = problem(name)
    s = _gpu_state(ctx, P, k)
    act = s["active"]
    D, delta, l1 = ctx.cggm_lambda_direction(s["Sigma"], s["Psi"], s["GradL"], s["Lg"], act["L_row"], act["L_col"],
                                             P.lam_L, True, 1)
    Sig, Psi, G = (s[x].cpu().numpy() for x in ("Sigma", "Psi", "GradL"))
    rows, cols = act["L_row"].cpu().numpy(), act["L_col"].cpu().numpy()
    Lam = s["lam"].to_dense()
    Dref, _, vals = A.lambda_newton_direction(Sig, Psi, G, Lam, rows, cols, P.lam_L, True, 1)
    Dg = D.cpu().numpy()
    assert np.linalg.norm(Dg - vals) <= 1e-10 * max(np.linalg.norm(vals), 1e-300)
    # decrease measure and ||Lambda||_1
    d_ref = float(np.sum(G * Dref)) + P.lam_L * (np.abs(Lam + Dref).sum() - np.abs(Lam).sum())
    assert delta == pytest.approx(d_ref, rel=1e-9, abs=1e-12)
    assert l1 == pytest.approx(np.abs(Lam).sum(), rel=1e-13)


def test_lambda_step_csc(ctx):
    P = problem("small")
    s = _gpu_state(ctx, P, 1)
    act = s["active"]
    D, _, _ = ctx.cggm_lambda_direction(s["Sigma"], s["Psi"], s["GradL"], s["Lg"], act["L_row"], act["L_col"],
                                        P.lam_L, True, 1)
    for alpha in (1.0, 0.25):
        t = ctx.cggm_lambda_step(s["Lg"], act["L_row"], act["L_col"], D, alpha)
        cp, ri, v = t.colptr.cpu().numpy(), t.rowidx.cpu().numpy(), t.val.cpu().numpy()
        q = P.q
        dense = np.zeros((q, q))
        for j in range(q):
            seg = ri[cp[j]:cp[j + 1]]
            assert np.all(np.diff(seg) > 0), "rows not strictly increasing"
            dense[seg, j] = v[cp[j]:cp[j + 1]]
        rows, cols = act["L_row"].cpu().numpy(), act["L_col"].cpu().numpy()
        Dd = np.zeros((q, q))
        Dd[rows, cols] = D.cpu().numpy()
        Dd[cols, rows] = D.cpu().numpy()
        ref = s["lam"].to_dense() + alpha * Dd
        np.testing.assert_array_equal(dense, dense.T)
        assert np.abs(dense - ref).max() <= 1e-15 * np.abs(ref).max()
        assert t.nnz == 2 * len(rows) - int(np.sum(rows == cols))


@pytest.mark.parametrize("name,k", [("tiny", 1), ("small", 1)])
def test_theta_sweep_matches_oracle(ctx, name, k):
    P = problem(name)
    s = _gpu_state(ctx, P, k)
    act = s["active"]
    Sxx = ctx.cggm_gram(s["X"])
    Tn, l1 = ctx.cggm_theta_cd(s["Sigma"], Sxx, s["Sxy"], s["Tg"], act["T_row"], act["T_col"], P.lam_T, 1)
    rows, cols = act["T_row"].cpu().numpy(), act["T_col"].cpu().numpy()
    n = P.X.shape[0]
    Sig = s["Sigma"].cpu().numpy()
    Sxx_h = P.X.T @ P.X / n
    Sxy_h = P.X.T @ P.Y / n
    Tref, _ = A.theta_cd_sweep(Sig, Sxx_h, Sxy_h, s["th"].to_dense(), rows, cols, P.lam_T, 1)
    vals = Tref[rows, cols]
    got = Tn.val.cpu().numpy()
    assert np.linalg.norm(got - vals) <= 1e-9 * np.linalg.norm(vals)
    assert l1 == pytest.approx(np.abs(Tref).sum(), rel=1e-9)
    # CSC structure = the list
    cp = Tn.colptr.cpu().numpy()
    assert cp[-1] == len(rows) and np.array_equal(np.repeat(np.arange(P.q), np.diff(cp)), cols)


def test_algorithm1_iterates_match_oracle(ctx):
    """Three outer iterations of Algorithm 1 on `tiny`: objective after every iteration, the step
    sizes and the final iterates agree with the oracle's loop."""
    from paper_1509_04681_b200 import to_device_colmajor
    from paper_1509_04681_b200.solver import ancd_fit
    P = problem("tiny")
    X, Y = to_device_colmajor(P.X), to_device_colmajor(P.Y)
    g = ancd_fit(ctx, X, Y, P.lam_L, P.lam_T, max_iter=3, tol=0.0)
    o = A.ancd_fit(P.X, P.Y, P.lam_L, P.lam_T, max_iter=3, tol=0.0)
    assert len(g.history) == len(o["history"]) == 3
    for hg, ho in zip(g.history, o["history"]):
        assert hg["f"] == pytest.approx(ho[0], rel=1e-9)
        assert hg["alpha"] == ho[4]
        assert (hg["m_L"], hg["m_T"]) == (ho[2], ho[3])
    Lg = np.zeros((P.q, P.q))
    cp, ri, v = (t.cpu().numpy() for t in (g.Lam.colptr, g.Lam.rowidx, g.Lam.val))
    for j in range(P.q):
        Lg[ri[cp[j]:cp[j + 1]], j] = v[cp[j]:cp[j + 1]]
    np.testing.assert_allclose(Lg, o["Lam"], rtol=0, atol=1e-9)
    Tg = np.zeros((P.p, P.q))
    cp, ri, v = (t.cpu().numpy() for t in (g.Theta.colptr, g.Theta.rowidx, g.Theta.val))
    for j in range(P.q):
        Tg[ri[cp[j]:cp[j + 1]], j] = v[cp[j]:cp[j + 1]]
    np.testing.assert_allclose(Tg, o["Theta"], rtol=0, atol=1e-9)


def test_algorithm1_converges_with_paper_rule(ctx):
    """Algorithm 1 on `tiny` with the paper's stopping rule converges; the objective is
    non-increasing and matches the oracle's converged fit."""
    from paper_1509_04681_b200 import to_device_colmajor
    from paper_1509_04681_b200.solver import ancd_fit
    P = problem("tiny")
    X, Y = to_device_colmajor(P.X), to_device_colmajor(P.Y)
    g = ancd_fit(ctx, X, Y, P.lam_L, P.lam_T, max_iter=100, tol=0.01)
    assert g.converged
    fs = [h["f"] for h in g.history]
    assert all(b <= a + 1e-12 for a, b in zip(fs, fs[1:]))
    o = A.ancd_fit(P.X, P.Y, P.lam_L, P.lam_T, max_iter=100, tol=0.01)
    assert g.iters == o["iters"]
    assert g.f == pytest.approx(o["f"], rel=1e-9)


def test_algorithm1_small_tight_tolerance_matches_prox_grad(ctx):
    """At a tight tolerance the GPU fit reaches the optimum of Eq. (1) found by the independent
    joint proximal-gradient oracle (convexity)."""
    from paper_1509_04681_b200 import to_device_colmajor
    from paper_1509_04681_b200.solver import ancd_fit
    rng = np.random.default_rng(5)
    n, p, q = 80, 12, 8
    Xh = rng.standard_normal((n, p))
    B = np.where(rng.random((p, q)) < 0.3, rng.standard_normal((p, q)), 0.0)
    Yh = Xh @ B + rng.standard_normal((n, q))
    X, Y = to_device_colmajor(Xh), to_device_colmajor(Yh)
    g = ancd_fit(ctx, X, Y, 0.1, 0.1, max_iter=1000, tol=1e-8)
    ref = A.prox_grad_fit(Xh, Yh, 0.1, 0.1)
    assert g.converged
    assert g.f == pytest.approx(ref["f"], rel=1e-7)


def _medium_oracle_sweeps(s, P, penalize_diag):
    """The oracle's Lambda direction and Theta sweep on the GPU state's lists at `medium` (q = 4000,
    p = 10000: the register / cp.async prefetch sweep path, q, p >= 2048), computed once."""
    key = ("medium_oracle", penalize_diag)
    if key not in _P:
        act = s["active"]
        Sig, Psi, G = (s[x].cpu().numpy() for x in ("Sigma", "Psi", "GradL"))
        rows, cols = act["L_row"].cpu().numpy(), act["L_col"].cpu().numpy()
        Lam = s["lam"].to_dense()
        Dref, _, vals = A.lambda_newton_direction(Sig, Psi, G, Lam, rows, cols, P.lam_L, penalize_diag, 1)
        lamM = np.full(Lam.shape, P.lam_L)
        if not penalize_diag:
            np.fill_diagonal(lamM, 0.0)
        d_ref = float(np.sum(G * Dref)) + float(np.sum(lamM * (np.abs(Lam + Dref) - np.abs(Lam))))
        trows, tcols = act["T_row"].cpu().numpy(), act["T_col"].cpu().numpy()
        n = P.X.shape[0]
        Tref, _ = A.theta_cd_sweep(Sig, P.X.T @ P.X / n, P.X.T @ P.Y / n, s["th"].to_dense(), trows, tcols,
                                   P.lam_T, 1)
        _P[key] = (vals, d_ref, Tref[trows, tcols], float(np.abs(Tref).sum()))
    return _P[key]


@pytest.mark.parametrize("variant", [{"CGGM_CD_COOP": "0"}, {"CGGM_CD_PREFETCH": "0"}, {"CGGM_CD_BLOCK": "1"}, {}])
def test_sweep_variants_agree_medium(variant):
    """The single-CTA sweeps, the column-batched cooperative sweeps, their register / prefetch
    variants (taken at medium sizes, q, p >= 2048) and the entry-blocked sweeps give the same direction and Theta to summation-order
    rounding, and each matches the oracle's sweeps on the same lists."""
    import os
    from paper_1509_04681_b200 import Context
    P = problem("medium")
    for k_, v_ in variant.items():
        os.environ[k_] = v_
    try:
        c = Context(0)
    finally:
        for k_ in variant:
            os.environ.pop(k_, None)
    s = _gpu_state(c, P, 0)
    act = s["active"]
    D, delta, _ = c.cggm_lambda_direction(s["Sigma"], s["Psi"], s["GradL"], s["Lg"], act["L_row"], act["L_col"],
                                          P.lam_L, True, 1)
    Sxx = c.cggm_gram(s["X"])
    Tn, l1 = c.cggm_theta_cd(s["Sigma"], Sxx, s["Sxy"], s["Tg"], act["T_row"], act["T_col"], P.lam_T, 1)
    key = "medium_sweeps"
    if key not in _P:
        _P[key] = (D.cpu().numpy(), Tn.val.cpu().numpy(), delta, l1)
    D0, T0, d0, l0 = _P[key]
    assert np.linalg.norm(D.cpu().numpy() - D0) <= 1e-10 * np.linalg.norm(D0)
    assert np.linalg.norm(Tn.val.cpu().numpy() - T0) <= 1e-10 * np.linalg.norm(T0)
    assert delta == pytest.approx(d0, rel=1e-9) and l1 == pytest.approx(l0, rel=1e-10)
    vals, d_ref, tvals, tl1 = _medium_oracle_sweeps(s, P, True)
    assert np.linalg.norm(D.cpu().numpy() - vals) <= 1e-10 * np.linalg.norm(vals)
    assert delta == pytest.approx(d_ref, rel=1e-9)
    assert np.linalg.norm(Tn.val.cpu().numpy() - tvals) <= 1e-9 * np.linalg.norm(tvals)
    assert l1 == pytest.approx(tl1, rel=1e-9)


def test_lambda_direction_medium_unpenalised_matches_oracle(ctx):
    """penalize_diag = 0 on the q >= 2048 sweep path against the oracle (reading A3)."""
    P = problem("medium")
    s = _gpu_state(ctx, P, 0)
    act = s["active"]
    D, delta, _ = ctx.cggm_lambda_direction(s["Sigma"], s["Psi"], s["GradL"], s["Lg"], act["L_row"], act["L_col"],
                                            P.lam_L, False, 1)
    vals, d_ref, _, _ = _medium_oracle_sweeps(s, P, False)
    assert np.linalg.norm(D.cpu().numpy() - vals) <= 1e-10 * np.linalg.norm(vals)
    assert delta == pytest.approx(d_ref, rel=1e-9)


@pytest.mark.parametrize("name,k", [("small", 1), ("medium", 0)])
def test_gram_rows_and_theta_sweep_on_demand(ctx, name, k):
    """NEXT-2 on-demand S_xx: cggm_gram_rows forms only the columns X^T X_i / n of the
    rows on the Theta list -- xmap is exact (row -> position among the distinct rows, ascending;
    -1 elsewhere), the columns match the definition -- and the Theta sweep on them equals the oracle's
    sweep on the full S_xx."""
    P = problem(name)
    s = _gpu_state(ctx, P, k)
    act = s["active"]
    cols, xmap = ctx.cggm_gram_rows(s["X"], act["T_row"])
    rows = np.unique(act["T_row"].cpu().numpy())
    want = np.full(P.p, -1, dtype=np.int64)
    want[rows] = np.arange(rows.size)
    np.testing.assert_array_equal(xmap.cpu().numpy(), want)
    n = P.X.shape[0]
    ref = P.X.T @ P.X[:, rows] / n
    got = cols.cpu().numpy()
    assert got.shape == ref.shape
    assert np.linalg.norm(got - ref) <= 1e-13 * np.linalg.norm(ref)
    Tn, l1 = ctx.cggm_theta_cd_rows(s["Sigma"], cols, xmap, s["Sxy"], s["Tg"], act["T_row"], act["T_col"], P.lam_T, 1)
    trows, tcols = act["T_row"].cpu().numpy(), act["T_col"].cpu().numpy()
    Tref, _ = A.theta_cd_sweep(s["Sigma"].cpu().numpy(), P.X.T @ P.X / n, P.X.T @ P.Y / n, s["th"].to_dense(), trows,
                               tcols, P.lam_T, 1)
    vals = Tref[trows, tcols]
    assert np.linalg.norm(Tn.val.cpu().numpy() - vals) <= 1e-9 * np.linalg.norm(vals)
    assert l1 == pytest.approx(np.abs(Tref).sum(), rel=1e-9)


def test_algorithm1_on_demand_sxx_matches_dense(ctx):
    """Algorithm 1 with on-demand S_xx columns and factor reuse gives the same iterates as with the
    dense S_xx (same sweep kernel, S_xx entries from different GEMMs: rounding-level differences)."""
    from paper_1509_04681_b200 import to_device_colmajor
    from paper_1509_04681_b200.solver import ancd_fit
    P = problem("tiny")
    X, Y = to_device_colmajor(P.X), to_device_colmajor(P.Y)
    a = ancd_fit(ctx, X, Y, P.lam_L, P.lam_T, max_iter=5, tol=0.0, sxx="rows")
    b = ancd_fit(ctx, X, Y, P.lam_L, P.lam_T, max_iter=5, tol=0.0, sxx="dense")
    for ha, hb in zip(a.history, b.history):
        assert ha["f"] == pytest.approx(hb["f"], rel=1e-12)
        assert ha["alpha"] == hb["alpha"] and (ha["m_L"], ha["m_T"]) == (hb["m_L"], hb["m_T"])
