"""penalize_diag = 0 (reading A3: the diagonal of Lambda unpenalised, lam_ii = 0; Eq. 1 P:222 with the
`\\iffalse`'d variant P:222-229) on every entry point whose kernels branch on it, against the oracle
on the same seeded inputs: cggm_active_set, the fused active sets of cggm_psi_grad, cggm_objective,
the composite cggm_newton_eval, the memory-bounded cggm_newton_eval_blocked and the Lambda direction
sweep cggm_lambda_direction.  Tolerances as in test_gpu_parity.py (north_star)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import ancd_oracle as A  # noqa: E402
from oracle import cggm_oracle as O  # noqa: E402
from synth.cggm_inputs import csc_from_triplets, make_problem  # noqa: E402

REL_F = 1e-9
REL_OBJ = 1e-10
TIE = 1e-9
CASES = [("tiny", 0), ("tiny", 1), ("small", 0), ("small", 1), ("medium", 0)]


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1509_04681_b200 import Context
    return Context(0)


_C = {}


def oracle_point(name, k):
    if (name, k) not in _C:
        P = make_problem(name)
        _, lam, th = P.points[k]
        Syy, Sxy = O.covariances(P.X, P.Y)
        Sig, ld, ok, _ = O.invert_logdet(lam.to_dense())
        r = O.psi_grad(P.X, P.Y, th, Sig, Syy, Sxy)
        a = O.active_set(r["GradL"], r["GradT"], lam, th, P.lam_L, P.lam_T, False, TIE)
        sub = O.min_norm_subgradient(r["GradL"], r["GradT"], lam, th, P.lam_L, P.lam_T, False)
        sub_pen = O.min_norm_subgradient(r["GradL"], r["GradT"], lam, th, P.lam_L, P.lam_T, True)
        ob = O.objective(P.X, P.Y, lam, th, P.lam_L, P.lam_T, False)
        ob_pen = O.objective(P.X, P.Y, lam, th, P.lam_L, P.lam_T, True)
        _C[(name, k)] = (P, lam, th, dict(Syy=Syy, Sigma=Sig, logdet=ld, active=a, sub=sub, sub_pen=sub_pen,
                                          obj=ob, obj_pen=ob_pen, **r))
    return _C[(name, k)]


def lists(cap):
    return {k: torch.empty(cap, dtype=torch.int32, device="cuda") for k in ("L_row", "L_col", "T_row", "T_col")}


def check_lists(got, ora):
    """Bit-exact outside the tie band, ascending column-major order."""
    for rk, ck, tm in (("L_row", "L_col", ora["tie_mask_L"]), ("T_row", "T_col", ora["tie_mask_T"])):
        gr, gc = got[rk].cpu().numpy().astype(np.int64), got[ck].cpu().numpy().astype(np.int64)
        g = set(zip(gr.tolist(), gc.tolist()))
        o = set(zip(ora[rk].tolist(), ora[ck].tolist()))
        for (i, j) in g ^ o:
            assert tm[i, j], (rk, i, j)
        assert np.all(np.diff(gc * (1 << 31) + gr) > 0)
    if ora["ties_L"] == 0 and ora["ties_T"] == 0:
        assert (got["m_L"], got["m_T"]) == (ora["m_L"], ora["m_T"])


@pytest.mark.parametrize("name,k", CASES)
def test_active_set_and_fused_unpenalised(ctx, name, k):
    from paper_1509_04681_b200 import DeviceCsc, to_device_colmajor
    P, lam, th, ref = oracle_point(name, k)
    X, Y = to_device_colmajor(P.X), to_device_colmajor(P.Y)
    Lg, Tg = DeviceCsc.from_host(lam), DeviceCsc.from_host(th)
    Syy, _ = ctx.cggm_covariances(X, Y, want_sxy=False)
    Sigma, _, _, _ = ctx.cggm_invert_logdet(Lg)
    sep = ctx.cggm_psi_grad(X, Y, Tg, Sigma, Syy=Syy)
    a = ctx.cggm_active_set(sep["GradL"], sep["GradT"], Lg, Tg, P.lam_L, P.lam_T, penalize_diag=False)
    check_lists(a, ref["active"])
    assert a["subgrad_l1"] == pytest.approx(ref["sub"], rel=1e-9)
    # the statistic differs from the penalised one (otherwise this test would not see the flag)
    assert abs(ref["sub"] - ref["sub_pen"]) > 1e-6 * ref["sub_pen"]
    cap = max(ref["active"]["m_L"], ref["active"]["m_T"]) + 4096
    spec = dict(lam_L=P.lam_L, lam_T=P.lam_T, penalize_diag=0, tie_eps=TIE, **lists(cap))
    fu = ctx.cggm_psi_grad(X, Y, Tg, Sigma, Syy=Syy, Lam=Lg, fused=spec)["active"]
    check_lists(fu, ref["active"])
    assert fu["subgrad_l1"] == pytest.approx(ref["sub"], rel=1e-9)
    assert fu["m_L"] == a["m_L"] and fu["m_T"] == a["m_T"]


@pytest.mark.parametrize("name,k", CASES)
def test_objective_unpenalised(ctx, name, k):
    from paper_1509_04681_b200 import DeviceCsc, to_device_colmajor
    P, lam, th, ref = oracle_point(name, k)
    X, Y = to_device_colmajor(P.X), to_device_colmajor(P.Y)
    ob = ctx.cggm_objective(X, Y, DeviceCsc.from_host(lam), DeviceCsc.from_host(th), P.lam_L, P.lam_T,
                            penalize_diag=False)
    ro = ref["obj"]
    assert ob["f"] == pytest.approx(ro["f"], rel=REL_OBJ)
    assert ob["pen_L"] == pytest.approx(ro["pen_L"], rel=1e-12)
    assert ro["pen_L"] < ref["obj_pen"]["pen_L"]


@pytest.mark.parametrize("name,k", CASES)
def test_composite_and_blocked_unpenalised(ctx, name, k):
    from paper_1509_04681_b200 import DeviceCsc, to_device_colmajor
    P, lam, th, ref = oracle_point(name, k)
    X, Y = to_device_colmajor(P.X), to_device_colmajor(P.Y)
    Lg, Tg = DeviceCsc.from_host(lam), DeviceCsc.from_host(th)
    Syy, _ = ctx.cggm_covariances(X, Y, want_sxy=False)
    cap = max(ref["active"]["m_L"], ref["active"]["m_T"]) + 4096
    c = ctx.cggm_newton_eval(X, Y, Syy, Lg, Tg, P.lam_L, P.lam_T, False, bufs=lists(cap))
    assert relf(c["Sigma"], ref["Sigma"]) <= REL_F and relf(c["GradL"], ref["GradL"]) <= REL_F
    check_lists(c["active"], ref["active"])
    assert c["active"]["subgrad_l1"] == pytest.approx(ref["sub"], rel=1e-9)
    assert c["objective"]["f"] == pytest.approx(ref["obj"]["f"], rel=REL_OBJ)
    block = {"tiny": 8, "small": 96, "medium": 1024}[name]
    b = ctx.cggm_newton_eval_blocked(X, Y, Lg, Tg, P.lam_L, P.lam_T, penalize_diag=False, block=block,
                                     bufs=lists(cap))
    check_lists(b["active"], ref["active"])
    assert b["active"]["subgrad_l1"] == pytest.approx(ref["sub"], rel=1e-9)
    assert b["objective"]["f"] == pytest.approx(ref["obj"]["f"], rel=REL_OBJ)


def test_active_set_zero_diagonal_support_unpenalised(ctx):
    """Lambda without stored diagonal (the diagonal decided by the gradient alone against lam_ii = 0)
    at `small` gradients, on the composite's fused path through cggm_psi_grad."""
    from paper_1509_04681_b200 import DeviceCsc, to_device_colmajor
    P, lam, th, ref = oracle_point("small", 1)
    d = lam.to_dense()
    np.fill_diagonal(d, 0.0)
    r_, c_ = np.nonzero(d)
    off = csc_from_triplets(P.q, P.q, r_, c_, d[r_, c_])
    GL = ref["GradL"].copy()
    GL[np.arange(0, P.q, 7), np.arange(0, P.q, 7)] = 0.0   # exact zeros stay out of S_Lambda
    a_ref = O.active_set(GL, ref["GradT"], off, th, P.lam_L, P.lam_T, False, TIE)
    got = ctx.cggm_active_set(to_device_colmajor(GL), to_device_colmajor(ref["GradT"]), DeviceCsc.from_host(off),
                              DeviceCsc.from_host(th), P.lam_L, P.lam_T, penalize_diag=False)
    check_lists(got, a_ref)
    diag = got["L_row"].cpu().numpy() == got["L_col"].cpu().numpy()
    assert int(diag.sum()) == P.q - len(range(0, P.q, 7))
    sub = O.min_norm_subgradient(GL, ref["GradT"], off, th, P.lam_L, P.lam_T, False)
    assert got["subgrad_l1"] == pytest.approx(sub, rel=1e-9)


@pytest.mark.parametrize("name,k", [("tiny", 1), ("small", 1), ("small", 0)])
def test_lambda_direction_unpenalised(ctx, name, k):
    from paper_1509_04681_b200 import DeviceCsc, to_device_colmajor
    P, lam, th, ref = oracle_point(name, k)
    X, Y = to_device_colmajor(P.X), to_device_colmajor(P.Y)
    Lg, Tg = DeviceCsc.from_host(lam), DeviceCsc.from_host(th)
    Syy, _ = ctx.cggm_covariances(X, Y, want_sxy=False)
    Sigma, _, _, _ = ctx.cggm_invert_logdet(Lg)
    cap = max(ref["active"]["m_L"], ref["active"]["m_T"]) + 4096
    spec = dict(lam_L=P.lam_L, lam_T=P.lam_T, penalize_diag=0, tie_eps=TIE, **lists(cap))
    r = ctx.cggm_psi_grad(X, Y, Tg, Sigma, Syy=Syy, Lam=Lg, fused=spec)
    act = r["active"]
    D, delta, l1 = ctx.cggm_lambda_direction(Sigma, r["Psi"], r["GradL"], Lg, act["L_row"], act["L_col"],
                                             P.lam_L, False, 1)
    Sig, Psi, G = (r_.cpu().numpy() for r_ in (Sigma, r["Psi"], r["GradL"]))
    rows, cols = act["L_row"].cpu().numpy(), act["L_col"].cpu().numpy()
    Lam = lam.to_dense()
    Dref, _, vals = A.lambda_newton_direction(Sig, Psi, G, Lam, rows, cols, P.lam_L, False, 1)
    assert np.linalg.norm(D.cpu().numpy() - vals) <= 1e-10 * np.linalg.norm(vals)
    lamM = np.full(Lam.shape, P.lam_L)
    np.fill_diagonal(lamM, 0.0)
    d_ref = float(np.sum(G * Dref)) + float(np.sum(lamM * (np.abs(Lam + Dref) - np.abs(Lam))))
    assert delta == pytest.approx(d_ref, rel=1e-9, abs=1e-12)
    # and it differs from the penalised direction on the same list
    _, _, vals_pen = A.lambda_newton_direction(Sig, Psi, G, Lam, rows, cols, P.lam_L, True, 1)
    assert np.linalg.norm(vals_pen - vals) > 1e-6 * np.linalg.norm(vals)


def relf(a, b):
    a = a.cpu().numpy() if torch.is_tensor(a) else a
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))
