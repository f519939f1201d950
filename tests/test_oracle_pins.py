"""Pins of the ORACLE against what the paper and the mathematics fix (never against itself).

Each test names the pin id of DESIGN.md §"Oracle pins".
CPU only (`-m "not gpu"`), tiny/small sizes so the suite stays within a few minutes.
"""
import json
import math
import os

import numpy as np
import pytest
import scipy.stats

from oracle import cggm_oracle as O
from synth.cggm_inputs import Csc, csc_from_dense, make_problem

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def chain_dense(q, phi=0.5):
    A = np.diag(np.full(q, 1.0 + phi * phi))
    i = np.arange(q - 1)
    A[i, i + 1] = -phi
    A[i + 1, i] = -phi
    return A


def chain_sigma_closed_form(q, phi=0.5):
    """P4: Sigma_ij (1-based, i<=j) = (phi^{j-i} - phi^{i+j})(1 - phi^{2(q+1-j)}) /
    ((1-phi^2)(1-phi^{2(q+1)}))  (derived for the tridiagonal chain)."""
    S = np.empty((q, q))
    for i in range(1, q + 1):
        j = np.arange(i, q + 1)
        v = (phi ** (j - i) - phi ** (i + j)) * (1 - phi ** (2 * (q + 1 - j))) / ((1 - phi ** 2) * (1 - phi ** (2 * (q + 1))))
        S[i - 1, i - 1:] = v
        S[i - 1:, i - 1] = v
    return S


@pytest.fixture(scope="module")
def tiny():
    return make_problem("tiny")


@pytest.fixture(scope="module")
def small():
    return make_problem("small")


# ------------------------------------------------------------------ P1 worked example
def test_p1_scalar_worked_example():
    g = json.load(open(os.path.join(GOLDEN, "p1_scalar_example.json")))
    s3 = math.sqrt(3.0)
    X = np.array([[1.0], [-1.0]], order="F")
    Y = np.array([[(1 + s3) / 2], [(s3 - 1) / 2]], order="F")
    lam = Csc(1, 1, np.array([0, 1], dtype=np.int64), np.array([0], dtype=np.int32), np.array([g["Lambda"]]))
    th = Csc(1, 1, np.array([0, 1], dtype=np.int64), np.array([0], dtype=np.int32), np.array([g["Theta"]]))
    Syy, Sxy = O.covariances(X, Y)
    assert Syy[0, 0] == pytest.approx(g["S_yy"], rel=1e-15)
    assert Sxy[0, 0] == pytest.approx(g["S_xy"], rel=1e-15)
    Sig, ld, ok, fc = O.invert_logdet(lam.to_dense())
    assert ok and fc == -1
    assert Sig[0, 0] == pytest.approx(g["Sigma"], rel=1e-15)
    assert ld == pytest.approx(g["logdet"], rel=1e-15)
    r = O.psi_grad(X, Y, th, Sig, Syy, Sxy)
    assert r["Psi"][0, 0] == pytest.approx(g["Psi"], rel=1e-14)
    assert r["GradL"][0, 0] == pytest.approx(g["grad_L"], rel=1e-13)
    assert r["GradT"][0, 0] == pytest.approx(g["grad_T"], rel=1e-14)
    ob = O.objective(X, Y, lam, th, g["lam_L"], g["lam_T"])
    assert ob["g"] == pytest.approx(g["g"], rel=1e-14)
    assert ob["f"] == pytest.approx(g["f"], rel=1e-14)


# ------------------------------------------------------------------ P2 identity point
def test_p2_identity_point(tiny):
    P = tiny
    label, lam, th = P.points[0]
    assert label == "identity"
    Syy, Sxy = O.covariances(P.X, P.Y)
    Sig, ld, ok, _ = O.invert_logdet(lam.to_dense())
    assert ok and ld == 0.0
    np.testing.assert_array_equal(Sig, np.eye(P.q))
    r = O.psi_grad(P.X, P.Y, th, Sig, Syy, Sxy)
    assert np.all(r["Psi"] == 0.0)
    np.testing.assert_allclose(r["GradL"], Syy - np.eye(P.q), rtol=0, atol=0)
    np.testing.assert_allclose(r["GradT"], 2 * Sxy, rtol=0, atol=0)
    ob = O.objective(P.X, P.Y, lam, th, P.lam_L, P.lam_T, penalize_diag=True)
    tr = float(np.trace(Syy))
    assert ob["g"] == pytest.approx(tr, rel=1e-13)
    assert ob["f"] == pytest.approx(tr + P.q * P.lam_L, rel=1e-13)
    ob2 = O.objective(P.X, P.Y, lam, th, P.lam_L, P.lam_T, penalize_diag=False)
    assert ob2["f"] == pytest.approx(tr, rel=1e-13)


def test_p2_spec_penalty_example():
    """Lambda=I (q=2), Theta=0, lam_L=0.1: f = tr(S_yy)+0.2 (penalised diag)
    and f = tr(S_yy) (unpenalised)."""
    rng = np.random.default_rng(5)
    X = np.asfortranarray(rng.standard_normal((7, 3)))
    Y = np.asfortranarray(rng.standard_normal((7, 2)))
    lam = csc_from_dense(np.eye(2))
    th = Csc(3, 2, np.zeros(3, dtype=np.int64), np.zeros(0, dtype=np.int32), np.zeros(0))
    tr = float(np.sum(Y * Y) / 7)
    assert O.objective(X, Y, lam, th, 0.1, 0.3, True)["f"] == pytest.approx(tr + 0.2, rel=1e-14)
    assert O.objective(X, Y, lam, th, 0.1, 0.3, False)["f"] == pytest.approx(tr, rel=1e-14)


# ------------------------------------------------------------------ P3/P4/P5 chain closed forms
@pytest.mark.parametrize("q", [1, 2, 3, 30, 200])
def test_p3_p4_chain_logdet_and_sigma(q):
    A = chain_dense(q)
    Sig, ld, ok, _ = O.invert_logdet(A)
    assert ok
    phi = 0.5
    ld_cf = math.log((1 - phi ** (2 * q + 2)) / (1 - phi ** 2))
    assert ld == pytest.approx(ld_cf, rel=1e-13, abs=1e-15)
    S_cf = chain_sigma_closed_form(q)
    assert np.linalg.norm(Sig - S_cf) / np.linalg.norm(S_cf) < 1e-14


def test_p3_chain_logdet_limit():
    # det -> 4/3 for q >= 27 to double precision: ln(4/3)
    _, ld, ok, _ = O.invert_logdet(chain_dense(60), want_sigma=False)
    assert ok and ld == pytest.approx(0.28768207245178085, rel=1e-14)


@pytest.mark.parametrize("q", [30, 500])
def test_p5_chain_pd_boundary(q):
    lmin = 1.25 - math.cos(math.pi / (q + 1))   # eigenvalues 1.25 - cos(k pi/(q+1))
    A = chain_dense(q)
    _, ok, fc = O.cholesky(A - (1 - 1e-6) * lmin * np.eye(q))
    assert ok and fc == -1
    _, ok, fc = O.cholesky(A - (1 + 1e-6) * lmin * np.eye(q))
    assert not ok and 0 <= fc < q


# ------------------------------------------------------------------ P6 SPEC logdet examples
def test_p6_spec_logdet_examples():
    g = json.load(open(os.path.join(GOLDEN, "p6_logdet_examples.json")))
    for case in g["cases"]:
        A = np.array(case["A"], dtype=float)
        _, ld, ok, fc = O.invert_logdet(A, want_sigma=False)
        assert ok == case["is_pd"]
        if ok:
            assert ld == pytest.approx(case["logdet"], abs=1e-15)
        else:
            assert fc == case["fail_col"]


# ------------------------------------------------------------------ P7 Sigma Lambda = I
def test_p7_sigma_times_lambda(small):
    for _, lam, _ in small.points:
        A = lam.to_dense()
        Sig, _, ok, _ = O.invert_logdet(A)
        assert ok
        err = np.linalg.norm(Sig @ A - np.eye(small.q)) / math.sqrt(small.q)
        assert err < 1e-12


def test_p7_random_spd():
    rng = np.random.default_rng(3)
    M = rng.standard_normal((60, 60))
    A = M @ M.T + 60 * np.eye(60)
    Sig, _, ok, _ = O.invert_logdet(A)
    assert ok and np.linalg.norm(Sig @ A - np.eye(60)) / math.sqrt(60) < 1e-12


# ------------------------------------------------------------------ P8 finite differences
def _g(P, Ld, Td):
    return O.objective(P.X, P.Y, csc_from_dense(Ld), csc_from_dense(Td), 0.0, 0.0)["g"]


@pytest.mark.parametrize("point", [0, 1])
def test_p8_gradients_vs_central_differences(tiny, point):
    P = tiny
    _, lam, th = P.points[point]
    Ld, Td = lam.to_dense(), th.to_dense()
    Syy, Sxy = O.covariances(P.X, P.Y)
    Sig, _, _, _ = O.invert_logdet(Ld)
    r = O.psi_grad(P.X, P.Y, th, Sig, Syy, Sxy)
    rng = np.random.default_rng(11)
    h = 1e-5
    scale = max(np.abs(r["GradL"]).max(), np.abs(r["GradT"]).max())
    for _ in range(12):   # Lambda: perturb (i,j) and (j,i) together (reading A8)
        i, j = rng.integers(0, P.q, size=2)
        E = np.zeros_like(Ld)
        E[i, j] = E[j, i] = 1.0
        fd = (_g(P, Ld + h * E, Td) - _g(P, Ld - h * E, Td)) / (2 * h)
        an = r["GradL"][i, j] * (1.0 if i == j else 2.0)
        assert abs(fd - an) <= 1e-7 * scale, (i, j, fd, an)
    for _ in range(12):
        i, j = rng.integers(0, P.p), rng.integers(0, P.q)
        E = np.zeros_like(Td)
        E[i, j] = 1.0
        fd = (_g(P, Ld, Td + h * E) - _g(P, Ld, Td - h * E)) / (2 * h)
        assert abs(fd - r["GradT"][i, j]) <= 1e-7 * scale, (i, j, fd, r["GradT"][i, j])


# ------------------------------------------------------------------ P9 Psi symmetric PSD, explicit S_xx
def test_p9_psi_psd_and_explicit_sxx(tiny):
    P = tiny
    _, lam, th = P.points[1]
    Syy, Sxy = O.covariances(P.X, P.Y)
    Sig, _, _, _ = O.invert_logdet(lam.to_dense())
    r = O.psi_grad(P.X, P.Y, th, Sig, Syy, Sxy)
    Psi = r["Psi"]
    np.testing.assert_array_equal(Psi, Psi.T)
    ev = np.linalg.eigvalsh(Psi)
    assert ev[0] >= -1e-12 * np.abs(ev).max()
    assert np.linalg.eigvalsh(Syy)[0] >= -1e-12 * np.abs(Syy).max()
    Sxx = P.X.T @ P.X / P.n
    Td = th.to_dense()
    Psi2 = Sig @ Td.T @ Sxx @ Td @ Sig          # Psi = Sigma Theta^T S_xx Theta Sigma
    assert np.linalg.norm(Psi - Psi2) / np.linalg.norm(Psi2) < 1e-13


# ------------------------------------------------------------------ P10 trace identities
def test_p10_trace_identities(small):
    P = small
    for _, lam, th in P.points:
        Syy, Sxy = O.covariances(P.X, P.Y)
        Ld = lam.to_dense()
        Sig, _, _, _ = O.invert_logdet(Ld)
        r = O.psi_grad(P.X, P.Y, th, Sig, Syy, Sxy)
        ob = O.objective(P.X, P.Y, lam, th, 0.0, 0.0)
        # I2: tr(Sigma M) = <Lambda, Psi>
        assert ob["tr_sigma_m"] == pytest.approx(float(np.sum(Ld * r["Psi"])), rel=1e-12)
        # I5: 2 tr(S_xy^T Theta) = (2/n) <W, Y>
        assert 2 * ob["tr_sxy_theta"] == pytest.approx(2.0 / P.n * float(np.sum(r["W"] * P.Y)), rel=1e-12)
        # I4: trace block = ||E L||_F^2 / n, E = Y + W Sigma
        L, _, _ = O.cholesky(Ld)
        E = P.Y + r["W"] @ Sig
        blk = ob["tr_syy_lam"] + 2 * ob["tr_sxy_theta"] + ob["tr_sigma_m"]
        assert blk == pytest.approx(float(np.sum((E @ L) ** 2)) / P.n, rel=1e-10)


# ------------------------------------------------------------------ P11 two gradient routes
def test_p11_grad_theta_two_routes(small):
    P = small
    _, lam, th = P.points[1]
    Syy, Sxy = O.covariances(P.X, P.Y)
    Sig, _, _, _ = O.invert_logdet(lam.to_dense())
    r = O.psi_grad(P.X, P.Y, th, Sig, Syy, Sxy)
    g2, _ = O.grad_theta_residual_route(P.X, P.Y, r["W"], Sig)
    assert np.linalg.norm(g2 - r["GradT"]) / np.linalg.norm(r["GradT"]) < 1e-12


# ------------------------------------------------------------------ P12 active-set examples
def test_p12_active_large_lambda(tiny):
    P = tiny
    _, lam, th = P.points[0]
    Syy, Sxy = O.covariances(P.X, P.Y)
    r = O.psi_grad(P.X, P.Y, th, np.eye(P.q), Syy, Sxy)
    lamL = np.abs(Syy - np.diag(np.diag(Syy))).max() + 1e-3
    lamT = 2 * np.abs(Sxy).max() + 1e-3
    a = O.active_set(r["GradL"], r["GradT"], lam, th, lamL, lamT)
    np.testing.assert_array_equal(a["L_row"], np.arange(P.q))
    np.testing.assert_array_equal(a["L_col"], np.arange(P.q))
    assert a["m_T"] == 0


def test_p12_spec_q3_example():
    """S_yy = [[1,.9,0],[.9,1,0],[0,0,1]], Lambda=I, lam=0.5 -> (1,2) enters."""
    Syy = np.array([[1, .9, 0], [.9, 1, 0], [0, 0, 1.0]])
    GL = Syy - np.eye(3)                     # Sigma = I, Psi = 0 at (I, 0)
    GT = np.zeros((2, 3))
    lam = csc_from_dense(np.eye(3))
    th = Csc(2, 3, np.zeros(4, dtype=np.int64), np.zeros(0, dtype=np.int32), np.zeros(0))
    a = O.active_set(GL, GT, lam, th, 0.5, 0.5)
    pairs = list(zip(a["L_row"].tolist(), a["L_col"].tolist()))
    assert pairs == [(0, 0), (0, 1), (1, 1), (2, 2)]
    assert a["m_T"] == 0


def test_p12_nonzero_always_active(small):
    P = small
    _, lam, th = P.points[0]
    q, p = P.q, P.p
    a = O.active_set(np.zeros((q, q)), np.zeros((p, q)), lam, th, 1e9, 1e9)
    # exactly the stored upper-triangle entries of Lambda and all stored Theta entries
    Ld = lam.to_dense()
    c, r = np.nonzero(np.triu(Ld != 0).T)
    np.testing.assert_array_equal(a["L_row"], r)
    np.testing.assert_array_equal(a["L_col"], c)
    assert a["m_T"] == th.nnz


# ------------------------------------------------------------------ P13 1x1 optimum
def test_p13_one_by_one_optimum():
    s3 = math.sqrt(3.0)
    X = np.array([[1.0], [-1.0]], order="F")
    Y = np.array([[(1 + s3) / 2], [(s3 - 1) / 2]], order="F")   # S_yy = 1, S_xy = 0.5
    lamL, lamT = 1.0, 10.0
    lstar = 1.0 / (1.0 + lamL)                                 # argmin -log L + s L + lam L
    lam = csc_from_dense(np.array([[lstar]]))
    th = Csc(1, 1, np.array([0, 0], dtype=np.int64), np.zeros(0, dtype=np.int32), np.zeros(0))
    Syy, Sxy = O.covariances(X, Y)
    Sig, _, _, _ = O.invert_logdet(lam.to_dense())
    r = O.psi_grad(X, Y, th, Sig, Syy, Sxy)
    stat = O.min_norm_subgradient(r["GradL"], r["GradT"], lam, th, lamL, lamT)
    assert abs(stat) < 1e-12


def _p13_hand_example():
    """q = 3, p = 2 hand example for ||grad^S||_1 (SPEC S:183 per-coordinate rule,
    reading A9: both triangles of Lambda, all of Theta).  lam_L = 0.5, lam_T = 0.25."""
    Lam = np.array([[2.0, -0.4, 0.0],
                    [-0.4, 1.0, 0.0],
                    [0.0, 0.0, 1.5]])
    GL = np.array([[0.3, -0.2, 0.8],
                   [-0.2, 0.9, 0.1],
                   [0.8, 0.1, -0.6]])
    Th = np.array([[0.0, 1.0, 0.0],
                   [-0.5, 0.0, 0.0]])
    GT = np.array([[0.1, -0.3, 0.4],
                   [0.2, 0.7, -0.25]])
    return Lam, GL, Th, GT


def test_p13_min_norm_subgradient_hand_example():
    """Worked by hand, entry by entry (x != 0: |g + lam sign x|; x == 0: max(|g| - lam, 0)):
      Lambda, diagonal penalised:   (0,0) |0.3+0.5| = 0.8   (1,1) |0.9+0.5| = 1.4   (2,2) |-0.6+0.5| = 0.1
                                    (0,1),(1,0): x = -0.4 -> |-0.2-0.5| = 0.7 each  -> 1.4
                                    (0,2),(2,0): x = 0    -> 0.8-0.5 = 0.3 each     -> 0.6
                                    (1,2),(2,1): x = 0    -> max(0.1-0.5, 0) = 0    -> 0
                                    sum 4.3   (one triangle only would give 3.3)
      Lambda, diagonal unpenalised (lam_ii = 0): diagonal |0.3| + |0.9| + |-0.6| = 1.8, off-diagonal 2.0
                                    sum 3.8   (keeping lam_ii would give 4.3)
      Theta: (0,0) max(0.1-0.25,0)=0  (0,1) |-0.3+0.25| = 0.05  (0,2) 0.4-0.25 = 0.15
             (1,0) |0.2-0.25| = 0.05  (1,1) 0.7-0.25 = 0.45   (1,2) |-0.25|-0.25 = 0 (exact tie)
             sum 0.70
    Totals: 5.0 (penalised diagonal), 4.5 (unpenalised)."""
    Lam, GL, Th, GT = _p13_hand_example()
    lc, tc = csc_from_dense(Lam), csc_from_dense(Th)
    assert O.min_norm_subgradient(GL, GT, lc, tc, 0.5, 0.25, True) == pytest.approx(5.0, abs=1e-14)
    assert O.min_norm_subgradient(GL, GT, lc, tc, 0.5, 0.25, False) == pytest.approx(4.5, abs=1e-14)
    # the Theta part alone (Lambda = gradient-free identity with lam_L = 0 contributes 0)
    z = np.zeros((3, 3))
    assert O.min_norm_subgradient(z, GT, csc_from_dense(np.eye(3)), tc, 0.0, 0.25) == pytest.approx(0.70, abs=1e-14)


def test_p12_active_set_unpenalised_diagonal():
    """Reading A3 with penalize_diag = 0 (lam_ii = 0, strict '>'): every diagonal entry with
    a nonzero gradient enters S_Lambda, an exactly-zero diagonal gradient does not; off-diagonal
    entries still use lam_L.  Hand example, lam_L = 1.0: GL diagonal (0.3, 0, -0.6), (0,2) = 1.2,
    (0,1) = 0.9, (1,2) = -1.0 (a tie with lam: not active), Lambda = I except Lambda_01 = 0.1."""
    GL = np.array([[0.3, 0.9, 1.2],
                   [0.9, 0.0, -1.0],
                   [1.2, -1.0, -0.6]])
    Lam = np.eye(3)
    Lam[0, 1] = Lam[1, 0] = 0.1
    GT = np.array([[0.5, -2.0, 0.0]])
    th = csc_from_dense(np.array([[0.0, 0.0, 3.0]]))
    lc = csc_from_dense(Lam)
    a = O.active_set(GL, GT, lc, th, 1.0, 1.0, penalize_diag=True)
    # penalised: (0,0), (1,1), (2,2) forced by Lambda = I; (0,1) forced by Lambda_01; (0,2) |1.2| > 1
    assert list(zip(a["L_row"].tolist(), a["L_col"].tolist())) == [(0, 0), (0, 1), (1, 1), (0, 2), (2, 2)]
    # unpenalised with a zero diagonal in Lambda: only the gradient decides the diagonal
    Lam0 = Lam - np.diag(np.diag(Lam))
    a0 = O.active_set(GL, GT, csc_from_dense(Lam0), th, 1.0, 1.0, penalize_diag=False)
    assert list(zip(a0["L_row"].tolist(), a0["L_col"].tolist())) == [(0, 0), (0, 1), (0, 2), (2, 2)]
    a1 = O.active_set(GL, GT, csc_from_dense(Lam0), th, 1.0, 1.0, penalize_diag=True)
    assert list(zip(a1["L_row"].tolist(), a1["L_col"].tolist())) == [(0, 1), (0, 2)]
    # Theta: |-2| > 1 and the stored 3.0; the diagonal flag does not touch Theta
    assert list(zip(a0["T_row"].tolist(), a0["T_col"].tolist())) == [(0, 1), (0, 2)]
    # the tie (1,2) is flagged in the tie band, the exact-zero diagonal (1,1) only when lam_ii = 0
    assert a0["tie_mask_L"][1, 2] and a0["tie_mask_L"][1, 1] and not a1["tie_mask_L"][1, 1]


# ------------------------------------------------------------------ P14 convexity
def test_p14_convexity(tiny):
    P = tiny
    rng = np.random.default_rng(7)
    for _ in range(5):
        mats = []
        for _ in range(2):
            M = rng.standard_normal((P.q, P.q)) * 0.1
            La = M @ M.T + np.eye(P.q)
            Ta = rng.standard_normal((P.p, P.q)) * (rng.random((P.p, P.q)) < 0.1)
            mats.append((La, Ta))
        (La, Ta), (Lb, Tb) = mats
        f = lambda L_, T_: O.objective(P.X, P.Y, csc_from_dense(L_), csc_from_dense(T_), 0.3, 0.3)["f"]
        assert f((La + Lb) / 2, (Ta + Tb) / 2) <= 0.5 * (f(La, Ta) + f(Lb, Tb)) + 1e-9


# ------------------------------------------------------------------ P15 independent routines
def test_p15_logdet_vs_eigenvalues_and_library_inverse(small):
    for _, lam, _ in small.points:
        A = lam.to_dense()
        Sig, ld, ok, _ = O.invert_logdet(A)
        ev = np.linalg.eigvalsh(A)
        assert ld == pytest.approx(float(np.sum(np.log(ev))), rel=1e-12)
        Sinv = np.linalg.inv(A)
        assert np.linalg.norm(Sig - Sinv) / np.linalg.norm(Sinv) < 1e-13
        L, _, _ = O.cholesky(A)
        np.testing.assert_allclose(L, np.linalg.cholesky(A), rtol=0, atol=1e-14)


def test_p15_covariances_brute_force(tiny):
    P = tiny
    Syy, Sxy = O.covariances(P.X, P.Y)
    for (i, j) in [(0, 0), (3, 17), (29, 2)]:
        s = sum(P.Y[k, i] * P.Y[k, j] for k in range(P.n)) / P.n
        assert Syy[i, j] == pytest.approx(s, rel=1e-13)
    for (i, j) in [(0, 0), (39, 29), (5, 11)]:
        s = sum(P.X[k, i] * P.Y[k, j] for k in range(P.n)) / P.n
        assert Sxy[i, j] == pytest.approx(s, rel=1e-13, abs=1e-15)


# ------------------------------------------------------------------ density pin (reading A1)
def test_g_equals_scaled_gaussian_nll(tiny):
    """g = (2/n) sum_k -log N(y_k; -Sigma Theta^T x_k, Sigma) - q log(2 pi)  (reading A1 of
    PAPER.md:177-205 / SPEC S:152), via scipy's independent multivariate-normal logpdf."""
    P = tiny
    _, lam, th = P.points[1]
    Ld, Td = lam.to_dense(), th.to_dense()
    Sig = np.linalg.inv(Ld)
    mu = -(P.X @ Td @ Sig)
    nll = -sum(scipy.stats.multivariate_normal.logpdf(P.Y[k], mean=mu[k], cov=Sig) for k in range(P.n))
    g_density = 2.0 / P.n * nll - P.q * math.log(2 * math.pi)
    ob = O.objective(P.X, P.Y, lam, th, 0.0, 0.0)
    assert ob["g"] == pytest.approx(g_density, rel=1e-11)


# ------------------------------------------------------------------ P16 generating-point identity I7
@pytest.mark.parametrize("name", ["tiny", "small"])
def test_p16_generating_point_identity(name):
    P = make_problem(name)
    label, lam, th = [pt for pt in P.points if pt[0] == "truth"][0]
    Syy, Sxy = O.covariances(P.X, P.Y)
    Sig, _, _, _ = O.invert_logdet(lam.to_dense())
    r = O.psi_grad(P.X, P.Y, th, Sig, Syy, Sxy)
    D = P.Y - P.E_noise
    Psi_star = D.T @ D / P.n
    G_star = 2.0 / P.n * (P.X.T @ P.E_noise)
    rel = lambda a, b: np.linalg.norm(a - b) / np.linalg.norm(b)
    assert rel(r["Psi"], Psi_star) < 1e-12
    assert rel(r["GradT"], G_star) < 1e-10
    assert rel(r["GradL"], Syy - Sig - Psi_star) < 1e-10


# ------------------------------------------------------------------ P17 shard partial sums
@pytest.mark.parametrize("G", [2, 4, 8])
def test_p17_shard_partial_sums(small, G):
    P = small
    _, lam, th = P.points[1]
    Syy, Sxy = O.covariances(P.X, P.Y)
    Sig, _, _, _ = O.invert_logdet(lam.to_dense())
    r = O.psi_grad(P.X, P.Y, th, Sig, Syy, Sxy)
    bounds = np.linspace(0, P.n, G + 1).astype(int)
    Syy_s = np.zeros_like(Syy)
    Psi_s = np.zeros_like(Syy)
    GT_s = np.zeros_like(Sxy)
    for a, b in zip(bounds[:-1], bounds[1:]):
        Xr, Yr = np.asfortranarray(P.X[a:b]), np.asfortranarray(P.Y[a:b])
        s, _ = O.covariances(Xr, Yr, n_total=P.n)
        Syy_s += s
        Wr = O.spmm_x_theta(Xr, th)
        Rr = Wr @ Sig / math.sqrt(P.n)
        Psi_s += Rr.T @ Rr
        g, _ = O.grad_theta_residual_route(Xr, Yr, Wr, Sig, n_total=P.n)
        GT_s += g
    rel = lambda a, b: np.linalg.norm(a - b) / np.linalg.norm(b)
    assert rel(Syy_s, Syy) < 1e-13
    assert rel(Psi_s, r["Psi"]) < 1e-13
    assert rel(GT_s, r["GradT"]) < 1e-11


# ------------------------------------------------------------------ non-PD objective
def test_objective_non_pd_is_inf(tiny):
    P = tiny
    A = chain_dense(P.q) - 2.0 * np.eye(P.q)
    ob = O.objective(P.X, P.Y, csc_from_dense(A), P.points[1][2], 0.5, 0.5)
    assert ob["f"] == math.inf and not ob["is_pd"] and ob["fail_col"] == 0
