"""NEXT-4: the memory-bounded evaluation (cggm_newton_eval_blocked: Sigma, Psi and the gradients
only as column blocks) against the dense composite evaluation and the oracle on the same seeded
inputs: identical active lists and counts (integers, bit-exact when no entry is in the tie band),
log-det, PD flag, subgradient statistic and objective to rounding.  Block widths that do and do not
divide q, and a non-PD Lambda."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import cggm_oracle as O  # noqa: E402
from synth.cggm_inputs import make_problem  # noqa: E402


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1509_04681_b200 import Context
    return Context(0)


def lists(cap):
    return {k: torch.empty(cap, dtype=torch.int32, device="cuda") for k in ("L_row", "L_col", "T_row", "T_col")}


@pytest.mark.parametrize("name,k,block", [("tiny", 1, 8), ("small", 1, 128), ("small", 0, 96), ("medium", 0, 1024),
                                          ("medium", 0, 0)])
def test_blocked_matches_dense_and_oracle(ctx, name, k, block):
    from paper_1509_04681_b200 import DeviceCsc, to_device_colmajor
    from paper_1509_04681_b200.api import newton_evaluation
    P = make_problem(name)
    _, lam, th = P.points[k]
    X, Y = to_device_colmajor(P.X), to_device_colmajor(P.Y)
    L, T = DeviceCsc.from_host(lam), DeviceCsc.from_host(th)
    cap = 3_000_000
    b = ctx.cggm_newton_eval_blocked(X, Y, L, T, P.lam_L, P.lam_T, block=block, bufs=lists(cap))
    Syy, _ = ctx.cggm_covariances(X, Y, want_sxy=False)
    d = newton_evaluation(ctx, X, Y, Syy, L, T, P.lam_L, P.lam_T, True, lists(cap))
    assert b["is_pd"] and d["is_pd"]
    assert b["logdet"] == pytest.approx(d["logdet"], rel=1e-13)
    ab, ad = b["active"], d["active"]
    ties = ab["ties_L"] + ab["ties_T"]
    assert (ab["ties_L"], ab["ties_T"]) == (ad["ties_L"], ad["ties_T"])
    if ties == 0:
        assert (ab["m_L"], ab["m_T"]) == (ad["m_L"], ad["m_T"])
        for key in ("L_row", "L_col", "T_row", "T_col"):
            assert torch.equal(ab[key], ad[key]), key
    assert ab["subgrad_l1"] == pytest.approx(ad["subgrad_l1"], rel=1e-9)
    ob, od = b["objective"], d["objective"]
    for key in ("f", "g", "tr_syy_lam", "tr_sxy_theta", "tr_sigma_m", "pen_L", "pen_T"):
        assert ob[key] == pytest.approx(od[key], rel=1e-11), key
    ref = O.objective(P.X, P.Y, lam, th, P.lam_L, P.lam_T)
    assert ob["f"] == pytest.approx(ref["f"], rel=1e-10)
    # the lists directly against the oracle's definition, bit-exact outside the tie band
    ora = _oracle_active(name, k)
    for rk, ck, tm in (("L_row", "L_col", ora["tie_mask_L"]), ("T_row", "T_col", ora["tie_mask_T"])):
        gr, gc = ab[rk].cpu().numpy().astype(np.int64), ab[ck].cpu().numpy().astype(np.int64)
        for (i, j) in set(zip(gr.tolist(), gc.tolist())) ^ set(zip(ora[rk].tolist(), ora[ck].tolist())):
            assert tm[i, j], (rk, i, j)
        assert np.all(np.diff(gc * (1 << 31) + gr) > 0)
    if ora["ties_L"] + ora["ties_T"] == 0:
        assert (ab["m_L"], ab["m_T"]) == (ora["m_L"], ora["m_T"])
    assert (ab["ties_L"], ab["ties_T"]) == (ora["ties_L"], ora["ties_T"])
    assert ab["subgrad_l1"] == pytest.approx(ora["sub"], rel=1e-9)


_ORA = {}


def _oracle_active(name, k):
    if (name, k) not in _ORA:
        P = make_problem(name)
        _, lam, th = P.points[k]
        Syy, Sxy = O.covariances(P.X, P.Y)
        Sig, _, _, _ = O.invert_logdet(lam.to_dense())
        r = O.psi_grad(P.X, P.Y, th, Sig, Syy, Sxy)
        a = O.active_set(r["GradL"], r["GradT"], lam, th, P.lam_L, P.lam_T)
        a["sub"] = O.min_norm_subgradient(r["GradL"], r["GradT"], lam, th, P.lam_L, P.lam_T)
        _ORA[(name, k)] = a
    return _ORA[(name, k)]


def test_blocked_non_pd(ctx):
    from paper_1509_04681_b200 import DeviceCsc, to_device_colmajor
    from synth.cggm_inputs import csc_from_triplets
    P = make_problem("small")
    _, lam, th = P.points[1]
    A = lam.to_dense()
    Lc, _, _ = O.cholesky(A)
    j = 137
    A[j, j] = float(np.dot(Lc[j, :j], Lc[j, :j])) - 1.0
    r, c = np.nonzero(A)
    bad = csc_from_triplets(A.shape[0], A.shape[1], r, c, A[r, c])
    X, Y = to_device_colmajor(P.X), to_device_colmajor(P.Y)
    out = ctx.cggm_newton_eval_blocked(X, Y, DeviceCsc.from_host(bad), DeviceCsc.from_host(th), P.lam_L, P.lam_T,
                                       block=128, bufs=lists(1_000_000))
    assert not out["is_pd"] and out["fail_col"] == j
    assert out["objective"]["f"] == float("inf")


def test_blocked_fp32_matches_dense_fp32():
    """The FP32 variant of the memory-bounded evaluation against the FP32 dense composite (same
    arithmetic type, reading A18): active counts and lists (outside the fp32 tie band), objective."""
    from paper_1509_04681_b200 import Context, DeviceCsc, to_device_colmajor
    from paper_1509_04681_b200.api import newton_evaluation
    c32 = Context(0, dtype="f32")
    P = make_problem("medium")
    _, lam, th = P.points[0]
    f32 = torch.float32
    X, Y = to_device_colmajor(P.X, dtype=f32), to_device_colmajor(P.Y, dtype=f32)
    L, T = DeviceCsc.from_host(lam, dtype=f32), DeviceCsc.from_host(th, dtype=f32)
    cap = 2_000_000
    b = c32.cggm_newton_eval_blocked(X, Y, L, T, P.lam_L, P.lam_T, tie_eps=1e-5, block=512, bufs=lists(cap))
    Syy, _ = c32.cggm_covariances(X, Y, want_sxy=False)
    d = newton_evaluation(c32, X, Y, Syy, L, T, P.lam_L, P.lam_T, True, lists(cap), tie_eps=1e-5)
    assert b["is_pd"] and d["is_pd"]
    ab, ad = b["active"], d["active"]
    if ab["ties_L"] + ab["ties_T"] + ad["ties_L"] + ad["ties_T"] == 0:
        assert (ab["m_L"], ab["m_T"]) == (ad["m_L"], ad["m_T"])
        assert torch.equal(ab["T_row"], ad["T_row"]) and torch.equal(ab["T_col"], ad["T_col"])
    assert abs(ab["m_L"] - ad["m_L"]) <= ab["ties_L"] + ad["ties_L"]
    assert b["objective"]["f"] == pytest.approx(d["objective"]["f"], rel=1e-5)
