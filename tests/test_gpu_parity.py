"""Parity of the CUDA path (through the C-ABI) with the CPU oracle on the same seeded inputs.

Tolerances (BASELINE.json north_star): Sigma, Psi, gradients rel-Frobenius <= 1e-9 (fp64);
objective rel <= 1e-10; active sets bit-exact outside the tie band ||grad| - lam| <= 1e-9;
is_pd exact.  Symmetric outputs must have bit-identical triangles (reading A19).
"""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import cggm_oracle as O  # noqa: E402
from synth.cggm_inputs import csc_from_dense, make_problem  # noqa: E402

REL_F = 1e-9
REL_OBJ = 1e-10
TIE = 1e-9


def relf(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1509_04681_b200 import Context
    return Context(0)


_CACHE = {}


def problem(name):
    if name not in _CACHE:
        _CACHE[name] = make_problem(name)
    return _CACHE[name]


def oracle_point(name, k):
    key = (name, k)
    if key not in _CACHE:
        P = problem(name)
        label, lam, th = P.points[k]
        Syy, Sxy = O.covariances(P.X, P.Y)
        Sig, ld, ok, fc = O.invert_logdet(lam.to_dense())
        r = O.psi_grad(P.X, P.Y, th, Sig, Syy, Sxy)
        a = O.active_set(r["GradL"], r["GradT"], lam, th, P.lam_L, P.lam_T, True, TIE)
        sub = O.min_norm_subgradient(r["GradL"], r["GradT"], lam, th, P.lam_L, P.lam_T, True)
        ob = O.objective(P.X, P.Y, lam, th, P.lam_L, P.lam_T, True)
        _CACHE[key] = dict(Syy=Syy, Sxy=Sxy, Sigma=Sig, logdet=ld, **r, active=a, sub=sub, obj=ob)
    return _CACHE[key]


def to_np(t):
    return t.detach().cpu().numpy()


def compare_active(gpu, ora, m_name, row_k, col_k, tie_mask):
    """Lists must agree exactly outside the tie band."""
    g = set(zip(to_np(gpu[row_k]).tolist(), to_np(gpu[col_k]).tolist()))
    o = set(zip(ora[row_k].tolist(), ora[col_k].tolist()))
    diff = g ^ o
    for (i, j) in diff:
        assert tie_mask[i, j], f"{m_name}: ({i},{j}) differs outside the tie band"
    # ordering: ascending column-major
    rows, cols = to_np(gpu[row_k]).astype(np.int64), to_np(gpu[col_k]).astype(np.int64)
    key = cols * (1 << 31) + rows
    assert np.all(np.diff(key) > 0)


CASES = [("tiny", 0), ("tiny", 1), ("small", 0), ("small", 1)]


@pytest.mark.parametrize("name,k", CASES)
def test_parity_point(ctx, name, k):
    from paper_1509_04681_b200 import DeviceCsc, to_device_colmajor
    P = problem(name)
    ref = oracle_point(name, k)
    label, lam, th = P.points[k]
    X, Y = to_device_colmajor(P.X), to_device_colmajor(P.Y)
    Lg, Tg = DeviceCsc.from_host(lam), DeviceCsc.from_host(th)
    Syy, Sxy = ctx.cggm_covariances(X, Y)
    assert relf(to_np(Syy), ref["Syy"]) <= 1e-13
    assert relf(to_np(Sxy), ref["Sxy"]) <= 1e-13
    np.testing.assert_array_equal(to_np(Syy), to_np(Syy).T)
    Sigma, logdet, pd, fc = ctx.cggm_invert_logdet(Lg)
    assert pd and fc == -1
    S = to_np(Sigma)
    np.testing.assert_array_equal(S, S.T)
    assert relf(S, ref["Sigma"]) <= REL_F
    assert logdet == pytest.approx(ref["logdet"], rel=1e-12, abs=1e-13)
    for route in ("residual", "sxy"):
        r = ctx.cggm_psi_grad(X, Y, Tg, Sigma, Syy=Syy, Sxy=(Sxy if route == "sxy" else None))
        Psi, GL, GT = to_np(r["Psi"]), to_np(r["GradL"]), to_np(r["GradT"])
        np.testing.assert_array_equal(Psi, Psi.T)
        np.testing.assert_array_equal(GL, GL.T)
        assert relf(Psi, ref["Psi"]) <= REL_F
        assert relf(GL, ref["GradL"]) <= REL_F
        assert relf(GT, ref["GradT"]) <= REL_F
    a = ctx.cggm_active_set(r["GradL"], r["GradT"], Lg, Tg, P.lam_L, P.lam_T, True, TIE)
    ora = ref["active"]
    compare_active(a, ora, "S_Lambda", "L_row", "L_col", ora["tie_mask_L"])
    compare_active(a, ora, "S_Theta", "T_row", "T_col", ora["tie_mask_T"])
    if ora["ties_L"] == 0 and ora["ties_T"] == 0:
        assert a["m_L"] == ora["m_L"] and a["m_T"] == ora["m_T"]
    assert a["subgrad_l1"] == pytest.approx(ref["sub"], rel=1e-9)
    ob = ctx.cggm_objective(X, Y, Lg, Tg, P.lam_L, P.lam_T, True)
    ro = ref["obj"]
    assert ob["is_pd"] and ob["fail_col"] == -1
    assert ob["f"] == pytest.approx(ro["f"], rel=REL_OBJ)
    assert ob["g"] == pytest.approx(ro["g"], rel=REL_OBJ, abs=1e-10)
    assert ob["logdet"] == pytest.approx(ro["logdet"], rel=1e-12, abs=1e-13)


def test_fused_active_matches_separate(ctx):
    from paper_1509_04681_b200 import DeviceCsc, to_device_colmajor
    P = problem("small")
    label, lam, th = P.points[1]
    X, Y = to_device_colmajor(P.X), to_device_colmajor(P.Y)
    Lg, Tg = DeviceCsc.from_host(lam), DeviceCsc.from_host(th)
    Syy, _ = ctx.cggm_covariances(X, Y, want_sxy=False)
    Sigma, _, _, _ = ctx.cggm_invert_logdet(Lg)
    sep = ctx.cggm_psi_grad(X, Y, Tg, Sigma, Syy=Syy)
    a = ctx.cggm_active_set(sep["GradL"], sep["GradT"], Lg, Tg, P.lam_L, P.lam_T)
    cap = 200000
    spec = dict(lam_L=P.lam_L, lam_T=P.lam_T, penalize_diag=1, tie_eps=TIE,
                L_row=torch.empty(cap, dtype=torch.int32, device="cuda"),
                L_col=torch.empty(cap, dtype=torch.int32, device="cuda"),
                T_row=torch.empty(cap, dtype=torch.int32, device="cuda"),
                T_col=torch.empty(cap, dtype=torch.int32, device="cuda"))
    fu = ctx.cggm_psi_grad(X, Y, Tg, Sigma, Syy=Syy, Lam=Lg, fused=spec)["active"]
    assert fu["m_L"] == a["m_L"] and fu["m_T"] == a["m_T"]
    assert torch.equal(fu["L_row"], a["L_row"]) and torch.equal(fu["T_col"], a["T_col"])
    assert fu["subgrad_l1"] == a["subgrad_l1"]


def test_capacity_two_call(ctx):
    from paper_1509_04681_b200 import DeviceCsc, to_device_colmajor
    from paper_1509_04681_b200.api import CggmError
    P = problem("tiny")
    label, lam, th = P.points[1]
    X, Y = to_device_colmajor(P.X), to_device_colmajor(P.Y)
    Lg, Tg = DeviceCsc.from_host(lam), DeviceCsc.from_host(th)
    Syy, _ = ctx.cggm_covariances(X, Y, want_sxy=False)
    Sigma, _, _, _ = ctx.cggm_invert_logdet(Lg)
    r = ctx.cggm_psi_grad(X, Y, Tg, Sigma, Syy=Syy)
    with pytest.raises(CggmError) as ei:
        ctx.cggm_active_set(r["GradL"], r["GradT"], Lg, Tg, P.lam_L, P.lam_T, cap_L=1, cap_T=1)
    assert ei.value.status == 6


def test_non_pd_lambda(ctx):
    from paper_1509_04681_b200 import DeviceCsc, to_device_colmajor
    P = problem("small")
    A = P.lam_star.to_dense()
    lmin = 1.25 - math.cos(math.pi / (P.q + 1))
    for t, expect_pd in [(1 - 1e-6, True), (1 + 1e-6, False)]:
        B = A - t * lmin * np.eye(P.q)
        _, ok, fc_o = O.cholesky(B)
        assert ok == expect_pd
        Bg = DeviceCsc.from_host(csc_from_dense(B))
        _, ld, pd, fc = ctx.cggm_invert_logdet(Bg, want_sigma=False)
        assert pd == expect_pd
        if not expect_pd:
            assert fc == fc_o
            ob = ctx.cggm_objective(to_device_colmajor(P.X), to_device_colmajor(P.Y), Bg,
                                    DeviceCsc.from_host(P.theta_star), P.lam_L, P.lam_T)
            assert not ob["is_pd"] and ob["f"] == math.inf and ob["fail_col"] == fc_o


def test_spec_logdet_examples(ctx):
    from paper_1509_04681_b200 import DeviceCsc
    for A, pd_ref, ld_ref in [(np.eye(5), True, 0.0), (2 * np.eye(3), True, 3 * math.log(2)),
                              (np.array([[1.0, 2.0], [2.0, 1.0]]), False, None)]:
        Sg, ld, pd, fc = ctx.cggm_invert_logdet(DeviceCsc.from_host(csc_from_dense(A)))
        assert pd == pd_ref
        if pd:
            assert ld == pytest.approx(ld_ref, abs=1e-15)
            assert np.allclose(to_np(Sg), np.linalg.inv(A), rtol=1e-15)
        else:
            assert fc == 1


@pytest.mark.parametrize("q", [700, 2500])
def test_chain_sigma_closed_form(ctx, q):
    """P3/P4 on the GPU directly: several recursion levels, ragged leaf."""
    from paper_1509_04681_b200 import DeviceCsc
    from tests.test_oracle_pins import chain_dense, chain_sigma_closed_form
    Sg, ld, pd, fc = ctx.cggm_invert_logdet(DeviceCsc.from_host(csc_from_dense(chain_dense(q))))
    assert pd
    assert ld == pytest.approx(math.log((1 - 0.5 ** (2 * q + 2)) / 0.75), rel=1e-12)
    S = to_np(Sg)
    assert relf(S, chain_sigma_closed_form(q)) <= 1e-12


def test_validation_errors(ctx):
    from paper_1509_04681_b200 import DeviceCsc
    from paper_1509_04681_b200.api import CggmError
    A = np.array([[2.0, 1.0], [0.5, 2.0]])   # not symmetric
    with pytest.raises(CggmError) as ei:
        ctx.cggm_invert_logdet(DeviceCsc.from_host(csc_from_dense(A)))
    assert ei.value.status == 3
    bad = DeviceCsc.from_host(csc_from_dense(np.eye(3)))
    bad.rowidx[1] = 7   # out of range
    with pytest.raises(CggmError) as ei:
        ctx.cggm_invert_logdet(bad)
    assert ei.value.status == 4


def test_launch_count_increases(ctx):
    from paper_1509_04681_b200 import DeviceCsc
    before = ctx.launch_count()
    ctx.cggm_invert_logdet(DeviceCsc.from_host(csc_from_dense(2 * np.eye(40))))
    assert ctx.launch_count() > before


@pytest.mark.slow
def test_parity_medium(ctx):
    test_parity_point(ctx, "medium", 0)


@pytest.mark.parametrize("name,k", [("small", 1), ("medium", 0)])
def test_composite_eval_matches_separate_calls(ctx, name, k):
    """cggm_newton_eval (objective overlapped on the auxiliary stream) gives bit-identical results
    to the separate calls, and matches the oracle."""
    from paper_1509_04681_b200 import DeviceCsc, to_device_colmajor
    from paper_1509_04681_b200.api import newton_evaluation
    P = problem(name)
    label, lam, th = P.points[k]
    X, Y = to_device_colmajor(P.X), to_device_colmajor(P.Y)
    Lg, Tg = DeviceCsc.from_host(lam), DeviceCsc.from_host(th)
    Syy, _ = ctx.cggm_covariances(X, Y, want_sxy=False)
    cap = 4_000_000

    def bufs():
        return {k2: torch.empty(cap, dtype=torch.int32, device="cuda") for k2 in ("L_row", "L_col", "T_row", "T_col")}

    a = newton_evaluation(ctx, X, Y, Syy, Lg, Tg, P.lam_L, P.lam_T, True, bufs(), composite=False)
    b = newton_evaluation(ctx, X, Y, Syy, Lg, Tg, P.lam_L, P.lam_T, True, bufs(), composite=True)
    for key in ("Sigma", "Psi", "GradL", "GradT"):
        assert torch.equal(a[key], b[key]), key
    assert a["logdet"] == b["logdet"] and a["objective"]["f"] == b["objective"]["f"]
    for key in ("L_row", "L_col", "T_row", "T_col"):
        assert torch.equal(a["active"][key], b["active"][key]), key
    assert a["active"]["subgrad_l1"] == b["active"]["subgrad_l1"]
    if name == "small":
        ref = oracle_point(name, k)
        assert relf(to_np(b["Sigma"]), ref["Sigma"]) <= REL_F
        assert b["objective"]["f"] == pytest.approx(ref["obj"]["f"], rel=REL_OBJ)


def test_streamed_grad_theta_matches_stored(ctx):
    """GradT = NULL: grad_Theta streamed in column chunks into the compaction (never stored) gives
    the same lists / statistic as the stored gradient."""
    from paper_1509_04681_b200 import DeviceCsc, to_device_colmajor
    from paper_1509_04681_b200.api import newton_evaluation
    P = problem("medium")   # q = 4000 > the 2048-column chunk: two chunks, look-back across them
    label, lam, th = P.points[0]
    X, Y = to_device_colmajor(P.X), to_device_colmajor(P.Y)
    Lg, Tg = DeviceCsc.from_host(lam), DeviceCsc.from_host(th)
    Syy, _ = ctx.cggm_covariances(X, Y, want_sxy=False)
    cap = 4_000_000

    def bufs():
        return {k2: torch.empty(cap, dtype=torch.int32, device="cuda") for k2 in ("L_row", "L_col", "T_row", "T_col")}

    a = newton_evaluation(ctx, X, Y, Syy, Lg, Tg, P.lam_L, P.lam_T, True, bufs())
    b = newton_evaluation(ctx, X, Y, Syy, Lg, Tg, P.lam_L, P.lam_T, True, bufs(), stream_grad_theta=True)
    assert b["GradT"] is None
    for key in ("L_row", "L_col", "T_row", "T_col"):
        assert torch.equal(a["active"][key], b["active"][key]), key
    for key in ("m_L", "m_T", "ties_L", "ties_T"):
        assert a["active"][key] == b["active"][key], key
    # the column-chunk streaming runs the stored path's scan kernel: bit-identical statistic
    assert a["active"]["subgrad_l1"] == b["active"]["subgrad_l1"]
    assert a["objective"]["f"] == b["objective"]["f"]
    # K01 (CGGM_K01=1): S_Theta selected in the X^T E epilogue -- the same per-element decisions on the
    # same gradient values, the subgradient summed in another order
    import os
    from paper_1509_04681_b200 import Context
    os.environ["CGGM_K01"] = "1"
    try:
        c1 = Context(0)
    finally:
        os.environ.pop("CGGM_K01", None)
    d = newton_evaluation(c1, X, Y, Syy, Lg, Tg, P.lam_L, P.lam_T, True, bufs(), stream_grad_theta=True)
    for key in ("L_row", "L_col", "T_row", "T_col"):
        assert torch.equal(a["active"][key], d["active"][key]), key
    for key in ("m_L", "m_T", "ties_L", "ties_T"):
        assert a["active"][key] == d["active"][key], key
    assert d["active"]["subgrad_l1"] == pytest.approx(a["active"]["subgrad_l1"], rel=1e-13)


def test_composite_graph_replay(ctx):
    """cggm_newton_eval runs eagerly on a new argument set, captures a CUDA graph on the second
    call and replays it afterwards: all three give bit-identical results; a replay sees new values
    written into the same buffers (the graph holds pointers, not data); new pointers re-capture."""
    from paper_1509_04681_b200 import DeviceCsc, to_device_colmajor
    from paper_1509_04681_b200.api import newton_evaluation
    P = problem("small")
    _, lam0, th0 = P.points[0]
    _, lam1, th1 = P.points[1]
    X, Y = to_device_colmajor(P.X), to_device_colmajor(P.Y)
    Syy, _ = ctx.cggm_covariances(X, Y, want_sxy=False)
    cap = 1_000_000
    bufs = {k2: torch.empty(cap, dtype=torch.int32, device="cuda") for k2 in ("L_row", "L_col", "T_row", "T_col")}
    Lg, Tg = DeviceCsc.from_host(lam0), DeviceCsc.from_host(th0)

    def snap(r):
        return ({k: r[k].clone() for k in ("Sigma", "Psi", "GradL", "GradT")}, r["objective"]["f"], r["logdet"],
                r["active"]["subgrad_l1"], int(r["active"]["m_L"]), int(r["active"]["m_T"]))

    l0 = ctx.launch_count()
    runs = [snap(newton_evaluation(ctx, X, Y, Syy, Lg, Tg, P.lam_L, P.lam_T, True, bufs)) for _ in range(4)]
    per_call = (ctx.launch_count() - l0) / 4
    assert per_call > 100   # replays still count their kernels
    for r in runs[1:]:
        for k in r[0]:
            assert torch.equal(r[0][k], runs[0][0][k]), k
        assert r[1:] == runs[0][1:]
    # same buffers, new values (Lambda* + 0.1 P has a superset pattern: use the same structure only
    # when it matches, else copy values of point 1 into a fresh CSC of its own)
    L1, T1 = DeviceCsc.from_host(lam1), DeviceCsc.from_host(th1)
    fresh = snap(newton_evaluation(ctx, X, Y, Syy, L1, T1, P.lam_L, P.lam_T, True, bufs, composite=False))
    if Tg.nnz == T1.nnz and torch.equal(Tg.rowidx, T1.rowidx) and torch.equal(Tg.colptr, T1.colptr):
        Tg.val.copy_(T1.val)
        rep = snap(newton_evaluation(ctx, X, Y, Syy, Lg, Tg, P.lam_L, P.lam_T, True, bufs))
        ref = snap(newton_evaluation(ctx, X, Y, Syy, Lg, Tg, P.lam_L, P.lam_T, True, bufs, composite=False))
        assert torch.equal(rep[0]["GradT"], ref[0]["GradT"]) and rep[1] == ref[1]
    # new pointers: eager, capture, replay again agree with the separate calls
    for _ in range(3):
        got = snap(newton_evaluation(ctx, X, Y, Syy, L1, T1, P.lam_L, P.lam_T, True, bufs))
        for k in got[0]:
            assert torch.equal(got[0][k], fresh[0][k]), k
        assert got[1:] == fresh[1:]


@pytest.mark.parametrize("name,k", [("small", 1), ("medium", 0)])
def test_active_vector_kernel_matches_scalar(ctx, name, k):
    """The paired-load compaction kernel (16-byte aligned gradients) and the scalar fallback
    (CGGM_NO_ACTIVE_VEC=1) give identical lists, counts and ties; the subgradient statistic agrees
    to summation-order rounding."""
    import os
    from paper_1509_04681_b200 import Context, DeviceCsc, to_device_colmajor
    P = problem(name)
    label, lam, th = P.points[k]
    ref = oracle_point(name, k)
    GL, GT = to_device_colmajor(ref["GradL"]), to_device_colmajor(ref["GradT"])
    Lg, Tg = DeviceCsc.from_host(lam), DeviceCsc.from_host(th)
    os.environ["CGGM_NO_ACTIVE_VEC"] = "1"
    try:
        cs = Context(0)
    finally:
        os.environ.pop("CGGM_NO_ACTIVE_VEC", None)
    a = ctx.cggm_active_set(GL, GT, Lg, Tg, P.lam_L, P.lam_T)
    b = cs.cggm_active_set(GL, GT, Lg, Tg, P.lam_L, P.lam_T)
    for key in ("m_L", "m_T", "ties_L", "ties_T"):
        assert a[key] == b[key], key
    for key in ("L_row", "L_col", "T_row", "T_col"):
        assert torch.equal(a[key], b[key]), key
    assert a["subgrad_l1"] == pytest.approx(b["subgrad_l1"], rel=1e-13)
    assert a["subgrad_l1"] == pytest.approx(ref["sub"], rel=1e-9)


@pytest.mark.parametrize("name,k", [("small", 1), ("medium", 0)])
def test_factor_reuse_evaluation(ctx, name, k):
    """CGGM_OPT_FACTOR_REUSE: the objective keeps its trial L^{-1} and the next evaluation's Sigma is
    its symmetric product (no factorisation).  Same Lambda on consecutive calls: Sigma, Psi, the
    gradients and the lists equal the plain evaluation's, log-det and the PD flag are the kept
    trial's, the objective matches the oracle (its trace now by a triangular GEMM)."""
    from paper_1509_04681_b200 import Context, DeviceCsc, _abi, to_device_colmajor
    from paper_1509_04681_b200.api import newton_evaluation
    P = problem(name)
    label, lam, th = P.points[k]
    X, Y = to_device_colmajor(P.X), to_device_colmajor(P.Y)
    Lg, Tg = DeviceCsc.from_host(lam), DeviceCsc.from_host(th)
    cap = 4_000_000

    def bufs():
        return {k2: torch.empty(cap, dtype=torch.int32, device="cuda") for k2 in ("L_row", "L_col", "T_row", "T_col")}

    c2 = Context(0)
    Syy, _ = c2.cggm_covariances(X, Y, want_sxy=False)
    plain = newton_evaluation(c2, X, Y, Syy, Lg, Tg, P.lam_L, P.lam_T, True, bufs())
    plain = {kk: (v.clone() if torch.is_tensor(v) else v) for kk, v in plain.items()}
    c2.set_option(_abi.CGGM_OPT_FACTOR_REUSE, 1)
    runs = [newton_evaluation(c2, X, Y, Syy, Lg, Tg, P.lam_L, P.lam_T, True, bufs()) for _ in range(3)]
    c2.set_option(_abi.CGGM_OPT_FACTOR_REUSE, 0)
    ref = oracle_point(name, k)
    for r in runs:   # the first call factors, the next two reuse the kept trial inverse
        for key in ("Sigma", "Psi", "GradL", "GradT"):
            assert relf(to_np(r[key]), to_np(plain[key])) <= 1e-13, key
        assert r["logdet"] == pytest.approx(plain["logdet"], rel=1e-13) and r["is_pd"] and r["fail_col"] == -1
        assert r["objective"]["f"] == pytest.approx(ref["obj"]["f"], rel=REL_OBJ)
        assert r["active"]["m_L"] == plain["active"]["m_L"] and r["active"]["m_T"] == plain["active"]["m_T"]
        assert relf(to_np(r["Sigma"]), ref["Sigma"]) <= REL_F


@pytest.mark.parametrize("name,k", [("small", 1), ("medium", 0)])
def test_host_buffer_evaluation_matches_device(ctx, name, k):
    """cggm_newton_eval_host (uploads from page-locked host memory overlapped with the factorisation,
    S_yy formed in the call) gives bit-identical results to cggm_newton_eval on device copies."""
    from paper_1509_04681_b200 import DeviceCsc, HostCsc, host_colmajor, to_device_colmajor
    from paper_1509_04681_b200.api import newton_evaluation
    P = problem(name)
    label, lam, th = P.points[k]
    X, Y = to_device_colmajor(P.X), to_device_colmajor(P.Y)
    Lg, Tg = DeviceCsc.from_host(lam), DeviceCsc.from_host(th)
    Syy, _ = ctx.cggm_covariances(X, Y, want_sxy=False)
    cap = 4_000_000

    def bufs():
        return {k2: torch.empty(cap, dtype=torch.int32, device="cuda") for k2 in ("L_row", "L_col", "T_row", "T_col")}

    a = newton_evaluation(ctx, X, Y, Syy, Lg, Tg, P.lam_L, P.lam_T, True, bufs())
    a = {kk: (v.clone() if torch.is_tensor(v) else v) for kk, v in a.items()}
    Xh, Yh = host_colmajor(P.X), host_colmajor(P.Y)
    b = ctx.cggm_newton_eval_host(Xh, Yh, HostCsc.from_host(lam), HostCsc.from_host(th), P.lam_L, P.lam_T, True,
                                  bufs=bufs())
    assert torch.equal(b["Syy"], Syy)
    for key in ("Sigma", "Psi", "GradL", "GradT"):
        assert torch.equal(a[key], b[key]), key
    assert a["objective"]["f"] == b["objective"]["f"] and a["logdet"] == b["logdet"]
    for key in ("L_row", "L_col", "T_row", "T_col"):
        assert torch.equal(a["active"][key], b["active"][key]), key


def test_host_buffer_graph_replay_sees_new_host_data(ctx):
    """cggm_newton_eval_host with the same arguments runs eagerly, then captures a CUDA graph, then
    replays it; the uploads stay outside the graph (external event waits), so a replay must see host
    data changed in place between calls: results equal a fresh device-path evaluation of the new
    data, bit for bit."""
    from paper_1509_04681_b200 import Context, DeviceCsc, HostCsc, host_colmajor, to_device_colmajor
    from paper_1509_04681_b200.api import newton_evaluation
    P = problem("small")
    label, lam, th = P.points[1]
    Xh, Yh = host_colmajor(P.X), host_colmajor(P.Y)
    Lh, Th = HostCsc.from_host(lam), HostCsc.from_host(th)
    cap = 400_000
    bufs = {k2: torch.empty(cap, dtype=torch.int32, device="cuda") for k2 in ("L_row", "L_col", "T_row", "T_col")}
    c = Context(0)
    outs = []
    for it in range(5):
        if it == 3:   # new data in the same pinned buffers: the replayed graph must upload it
            Yh.mul_(0.5)
            Xh.add_(0.25)
        r = c.cggm_newton_eval_host(Xh, Yh, Lh, Th, P.lam_L, P.lam_T, True, bufs=bufs)
        outs.append({k: (v.clone() if torch.is_tensor(v) else v) for k, v in r.items() if k != "active"}
                    | {"active": {k: (v.clone() if torch.is_tensor(v) else v) for k, v in r["active"].items()}})
    for key in ("Sigma", "Psi", "GradL", "GradT", "Syy"):
        assert torch.equal(outs[0][key], outs[1][key]) and torch.equal(outs[1][key], outs[2][key]), key
        assert torch.equal(outs[3][key], outs[4][key]), key
    # reference for the modified data through the device path on a fresh context
    d = Context(0)
    X, Y = to_device_colmajor(Xh.numpy()), to_device_colmajor(Yh.numpy())
    Syy, _ = d.cggm_covariances(X, Y, want_sxy=False)
    bufs2 = {k2: torch.empty(cap, dtype=torch.int32, device="cuda") for k2 in ("L_row", "L_col", "T_row", "T_col")}
    ref = newton_evaluation(d, X, Y, Syy, DeviceCsc.from_host(lam), DeviceCsc.from_host(th), P.lam_L, P.lam_T, True,
                            bufs2)
    assert torch.equal(outs[4]["Syy"], Syy)
    for key in ("Sigma", "Psi", "GradL", "GradT"):
        assert torch.equal(outs[4][key], ref[key]), key
    assert outs[4]["objective"]["f"] == ref["objective"]["f"]
    assert outs[4]["active"]["m_L"] == ref["active"]["m_L"] and outs[4]["active"]["m_T"] == ref["active"]["m_T"]
    assert not torch.equal(outs[4]["GradT"], outs[0]["GradT"])


def test_host_buffer_evaluation_streamed_grad_theta(ctx):
    """cggm_newton_eval_host with GradT = NULL (grad_Theta streamed into the compaction, never stored --
    the form the `sharded` size needs) gives the same lists, statistic and objective as the device-path
    streamed evaluation."""
    from paper_1509_04681_b200 import DeviceCsc, HostCsc, host_colmajor, to_device_colmajor
    from paper_1509_04681_b200.api import newton_evaluation
    P = problem("medium")
    label, lam, th = P.points[0]
    X, Y = to_device_colmajor(P.X), to_device_colmajor(P.Y)
    Syy, _ = ctx.cggm_covariances(X, Y, want_sxy=False)
    cap = 4_000_000

    def bufs():
        return {k2: torch.empty(cap, dtype=torch.int32, device="cuda") for k2 in ("L_row", "L_col", "T_row", "T_col")}

    a = newton_evaluation(ctx, X, Y, Syy, DeviceCsc.from_host(lam), DeviceCsc.from_host(th), P.lam_L, P.lam_T, True,
                          bufs(), stream_grad_theta=True)
    a = {kk: (v.clone() if torch.is_tensor(v) else v) for kk, v in a.items()}
    b = ctx.cggm_newton_eval_host(host_colmajor(P.X), host_colmajor(P.Y), HostCsc.from_host(lam), HostCsc.from_host(th),
                                  P.lam_L, P.lam_T, True, bufs=bufs(), stream_grad_theta=True)
    assert b["GradT"] is None
    for key in ("L_row", "L_col", "T_row", "T_col"):
        assert torch.equal(a["active"][key], b["active"][key]), key
    assert a["active"]["subgrad_l1"] == b["active"]["subgrad_l1"]
    assert a["objective"]["f"] == b["objective"]["f"]
