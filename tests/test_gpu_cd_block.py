"""The entry-blocked cooperative sweeps (csrc/cd.cu k_sweep_blk; the default when the column vector
exceeds the register variants, q > 6144 / p > 12288, forced here with CGGM_CD_BLOCK=1) against the
oracle's sequential sweeps (oracle/ancd_oracle.py; Eq. (6) / (7)): the Lambda
direction with both diagonal-penalty settings and over two passes (D carried between passes), the
Theta sweep on the full S_xx and on the on-demand columns, blocks of 128 entries with a
ragged last block (columns of the small / medium lists hold up to several hundred entries), bitwise
run-to-run reproducibility, and Algorithm 1's iterates on `tiny`.  The left-looking panel mode of the
Lambda sweep (CGGM_CD_PANEL = w: U^T, Z^T of w columns at a time formed from the dense D by two GEMMs,
the default at q > 6144) is forced at panel widths that give several panels and a ragged last one."""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import ancd_oracle as A  # noqa: E402
from synth.cggm_inputs import make_problem  # noqa: E402

_P = {}


def problem(name):
    if name not in _P:
        _P[name] = make_problem(name)
    return _P[name]


@pytest.fixture(scope="module")
def bctx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1509_04681_b200 import Context
    os.environ["CGGM_CD_BLOCK"] = "1"
    try:
        return Context(0)
    finally:
        os.environ.pop("CGGM_CD_BLOCK", None)


def _state(ctx, P, k):
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


def _max_col_entries(cols):
    return int(np.bincount(cols).max()) if cols.size else 0


@pytest.mark.parametrize("name,k,pen,passes", [("tiny", 1, True, 1), ("small", 1, True, 1), ("small", 0, False, 1),
                                               ("small", 1, True, 2), ("medium", 0, True, 1)])
def test_blocked_lambda_direction_matches_oracle(bctx, name, k, pen, passes):
    P = problem(name)
    s = _state(bctx, P, k)
    act = s["active"]
    rows, cols = act["L_row"].cpu().numpy(), act["L_col"].cpu().numpy()
    D, delta, l1 = bctx.cggm_lambda_direction(s["Sigma"], s["Psi"], s["GradL"], s["Lg"], act["L_row"], act["L_col"],
                                              P.lam_L, pen, passes)
    Sig, Psi, G = (s[x].cpu().numpy() for x in ("Sigma", "Psi", "GradL"))
    Lam = s["lam"].to_dense()
    Dref, _, vals = A.lambda_newton_direction(Sig, Psi, G, Lam, rows, cols, P.lam_L, pen, passes)
    Dg = D.cpu().numpy()
    assert np.linalg.norm(Dg - vals) <= 1e-10 * max(np.linalg.norm(vals), 1e-300)
    lamM = np.full(Lam.shape, P.lam_L)
    if not pen:
        np.fill_diagonal(lamM, 0.0)
    d_ref = float(np.sum(G * Dref)) + float(np.sum(lamM * (np.abs(Lam + Dref) - np.abs(Lam))))
    assert delta == pytest.approx(d_ref, rel=1e-9, abs=1e-12)
    if name != "tiny":
        assert _max_col_entries(cols) > 128, "the case must span several blocks in some column"
    # bitwise reproducible
    D2, delta2, _ = bctx.cggm_lambda_direction(s["Sigma"], s["Psi"], s["GradL"], s["Lg"], act["L_row"], act["L_col"],
                                               P.lam_L, pen, passes)
    assert np.array_equal(D2.cpu().numpy(), Dg) and delta2 == delta


@pytest.mark.parametrize("name,k", [("tiny", 1), ("small", 1), ("medium", 0)])
def test_blocked_theta_sweep_matches_oracle(bctx, name, k):
    P = problem(name)
    s = _state(bctx, P, k)
    act = s["active"]
    trows, tcols = act["T_row"].cpu().numpy(), act["T_col"].cpu().numpy()
    n = P.X.shape[0]
    Tref, _ = A.theta_cd_sweep(s["Sigma"].cpu().numpy(), P.X.T @ P.X / n, P.X.T @ P.Y / n, s["th"].to_dense(), trows,
                               tcols, P.lam_T, 1)
    vals = Tref[trows, tcols]
    Sxx = bctx.cggm_gram(s["X"])
    Tn, l1 = bctx.cggm_theta_cd(s["Sigma"], Sxx, s["Sxy"], s["Tg"], act["T_row"], act["T_col"], P.lam_T, 1)
    assert np.linalg.norm(Tn.val.cpu().numpy() - vals) <= 1e-9 * np.linalg.norm(vals)
    assert l1 == pytest.approx(np.abs(Tref).sum(), rel=1e-9)
    cols, xmap = bctx.cggm_gram_rows(s["X"], act["T_row"])
    Tr, l1r = bctx.cggm_theta_cd_rows(s["Sigma"], cols, xmap, s["Sxy"], s["Tg"], act["T_row"], act["T_col"],
                                      P.lam_T, 1)
    assert np.linalg.norm(Tr.val.cpu().numpy() - vals) <= 1e-9 * np.linalg.norm(vals)
    if name != "tiny":
        assert _max_col_entries(tcols) > 128
    Tn2, _ = bctx.cggm_theta_cd(s["Sigma"], Sxx, s["Sxy"], s["Tg"], act["T_row"], act["T_col"], P.lam_T, 1)
    assert np.array_equal(Tn2.val.cpu().numpy(), Tn.val.cpu().numpy())


def test_blocked_algorithm1_iterates_match_oracle(bctx):
    from paper_1509_04681_b200 import to_device_colmajor
    from paper_1509_04681_b200.solver import ancd_fit
    P = problem("tiny")
    X, Y = to_device_colmajor(P.X), to_device_colmajor(P.Y)
    g = ancd_fit(bctx, X, Y, P.lam_L, P.lam_T, max_iter=3, tol=0.0)
    o = A.ancd_fit(P.X, P.Y, P.lam_L, P.lam_T, max_iter=3, tol=0.0)
    for hg, ho in zip(g.history, o["history"]):
        assert hg["f"] == pytest.approx(ho[0], rel=1e-9)
        assert hg["alpha"] == ho[4]
        assert (hg["m_L"], hg["m_T"]) == (ho[2], ho[3])


_PCTX = {}


def panel_ctx(w):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if w not in _PCTX:
        from paper_1509_04681_b200 import Context
        os.environ["CGGM_CD_BLOCK"] = "1"
        os.environ["CGGM_CD_PANEL"] = str(w)
        try:
            _PCTX[w] = Context(0)
        finally:
            os.environ.pop("CGGM_CD_BLOCK", None)
            os.environ.pop("CGGM_CD_PANEL", None)
    return _PCTX[w]


@pytest.mark.parametrize("name,k,pen,passes,w", [("tiny", 1, True, 2, 8), ("small", 1, True, 1, 64),
                                                 ("small", 0, False, 2, 96), ("small", 1, True, 2, 200),
                                                 ("medium", 0, True, 1, 512)])
def test_panel_lambda_direction_matches_oracle(name, k, pen, passes, w):
    """Left-looking panel mode: same updates in the same order as the oracle's sweep; U's entries come
    from D Sigma formed per panel instead of incremental row updates, so the direction agrees with
    the oracle to rounding (and with the right-looking blocked sweep to 1e-12)."""
    ctx = panel_ctx(w)
    ref = panel_ctx(0)
    P = problem(name)
    s = _state(ctx, P, k)
    act = s["active"]
    rows, cols = act["L_row"].cpu().numpy(), act["L_col"].cpu().numpy()
    args = (s["Sigma"], s["Psi"], s["GradL"], s["Lg"], act["L_row"], act["L_col"], P.lam_L, pen, passes)
    D, delta, l1 = ctx.cggm_lambda_direction(*args)
    Dg = D.cpu().numpy().copy()
    Sig, Psi, G = (s[x].cpu().numpy() for x in ("Sigma", "Psi", "GradL"))
    Lam = s["lam"].to_dense()
    Dref, _, vals = A.lambda_newton_direction(Sig, Psi, G, Lam, rows, cols, P.lam_L, pen, passes)
    assert np.linalg.norm(Dg - vals) <= 1e-10 * max(np.linalg.norm(vals), 1e-300)
    lamM = np.full(Lam.shape, P.lam_L)
    if not pen:
        np.fill_diagonal(lamM, 0.0)
    d_ref = float(np.sum(G * Dref)) + float(np.sum(lamM * (np.abs(Lam + Dref) - np.abs(Lam))))
    assert delta == pytest.approx(d_ref, rel=1e-9, abs=1e-12)
    assert P.q > 2 * w, "several panels"
    Db, delta_b, _ = ref.cggm_lambda_direction(*args)
    Db = Db.cpu().numpy()
    assert np.linalg.norm(Dg - Db) <= 1e-12 * max(np.linalg.norm(Db), 1e-300)
    D2, delta2, _ = ctx.cggm_lambda_direction(*args)
    assert np.array_equal(D2.cpu().numpy(), Dg) and delta2 == delta
