"""The two oracle forms pin each other (CPU, `-m "not gpu"`): the numpy oracle (oracle/cggm_oracle.py,
BLAS products as steps) against the plain-C loop form (oracle/c/cggm_oracle_c.c, no BLAS / LAPACK,
independent code), on the seeded configs and on the closed forms -- a dropped term, a sign, an index
or a transposed operand in either would have to be repeated in the other to pass.  Plus a per-phase
host timing of the plain definition at `small` (the oracle timed per phase)."""
import math

import numpy as np
import pytest

from oracle import c_oracle as C
from oracle import cggm_oracle as O
from synth.cggm_inputs import csc_from_dense, make_problem
from tests.test_oracle_pins import chain_dense, chain_sigma_closed_form


def relf(a, b):
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


def test_scalar_worked_example():
    """P1 (realised with n = 2): X = [1, -1], Y = [(1+sqrt3)/2, (sqrt3-1)/2],
    Lambda = [2], Theta = [1]: S_yy = 1, S_xy = 0.5, Sigma = 0.5, Psi = 0.25, grad_Lambda = 0.25,
    grad_Theta = 2, f(lam_L = lam_T = 1) = 5.806852819440055."""
    s3 = math.sqrt(3.0)
    X = np.array([[1.0], [-1.0]])
    Y = np.array([[(1 + s3) / 2], [(s3 - 1) / 2]])
    lam = csc_from_dense(np.array([[2.0]]))
    th = csc_from_dense(np.array([[1.0]]))
    ob = C.objective(X, Y, lam, th, 1.0, 1.0)
    assert ob["is_pd"]
    assert ob["f"] == pytest.approx(5.806852819440055, rel=1e-14)
    Syy, Sxy = C.covariances(X, Y)
    assert Syy[0, 0] == pytest.approx(1.0, rel=1e-15) and Sxy[0, 0] == pytest.approx(0.5, rel=1e-15)
    S, ld, pd, fc = C.invert_logdet(np.array([[2.0]]))
    assert pd and S[0, 0] == pytest.approx(0.5, rel=1e-15) and ld == pytest.approx(math.log(2.0), rel=1e-15)
    r = C.psi_grad(X, Y, th, S, Syy)
    assert r["Psi"][0, 0] == pytest.approx(0.25, rel=1e-14)
    assert r["GradL"][0, 0] == pytest.approx(0.25, rel=1e-14)
    assert r["GradT"][0, 0] == pytest.approx(2.0, rel=1e-14)


@pytest.mark.parametrize("q", [1, 2, 3, 30, 200])
def test_chain_closed_forms(q):
    """P3 / P4 (chain log-det and Sigma) and P5 (the PD boundary) on the C form."""
    S, ld, pd, fc = C.invert_logdet(chain_dense(q))
    assert pd and fc == -1
    assert ld == pytest.approx(math.log((1 - 0.5 ** (2 * q + 2)) / 0.75), rel=1e-13, abs=1e-15)
    assert relf(S, chain_sigma_closed_form(q)) <= 1e-13
    np.testing.assert_array_equal(S, S.T)
    lmin = 1.25 - math.cos(math.pi / (q + 1))
    assert C.invert_logdet(chain_dense(q) - (1 - 1e-6) * lmin * np.eye(q))[2]
    assert not C.invert_logdet(chain_dense(q) - (1 + 1e-6) * lmin * np.eye(q))[2]


@pytest.mark.parametrize("name,k", [("tiny", 0), ("tiny", 1), ("small", 0), ("small", 1)])
@pytest.mark.parametrize("penalize_diag", [True, False])
def test_numpy_and_c_oracles_agree(name, k, penalize_diag):
    P = make_problem(name)
    label, lam, th = P.points[k]
    Syy_n, Sxy_n = O.covariances(P.X, P.Y)
    Syy_c, Sxy_c = C.covariances(P.X, P.Y)
    assert relf(Syy_c, Syy_n) <= 1e-13 and relf(Sxy_c, Sxy_n) <= 1e-13
    Sig_n, ld_n, ok_n, _ = O.invert_logdet(lam.to_dense())
    Sig_c, ld_c, ok_c, _ = C.invert_logdet(lam.to_dense())
    assert ok_n and ok_c
    assert ld_c == pytest.approx(ld_n, rel=1e-12)
    assert relf(Sig_c, Sig_n) <= 1e-12
    rn = O.psi_grad(P.X, P.Y, th, Sig_n, Syy_n, Sxy_n)
    rc = C.psi_grad(P.X, P.Y, th, Sig_c, Syy_c)
    for key in ("Psi", "GradL", "GradT"):
        assert relf(rc[key], rn[key]) <= 1e-11, key
    an = O.active_set(rn["GradL"], rn["GradT"], lam, th, P.lam_L, P.lam_T, penalize_diag, 1e-9)
    ac = C.active_set(rn["GradL"], rn["GradT"], lam, th, P.lam_L, P.lam_T, penalize_diag, 1e-9)
    for key in ("L_row", "L_col", "T_row", "T_col"):   # the same gradients in: integer results identical
        np.testing.assert_array_equal(ac[key], an[key])
    assert (ac["ties_L"], ac["ties_T"]) == (an["ties_L"], an["ties_T"])
    sub_n = O.min_norm_subgradient(rn["GradL"], rn["GradT"], lam, th, P.lam_L, P.lam_T, penalize_diag)
    assert ac["subgrad_l1"] == pytest.approx(sub_n, rel=1e-12)
    on = O.objective(P.X, P.Y, lam, th, P.lam_L, P.lam_T, penalize_diag)
    oc = C.objective(P.X, P.Y, lam, th, P.lam_L, P.lam_T, penalize_diag)
    assert oc["f"] == pytest.approx(on["f"], rel=1e-12)
    assert oc["logdet"] == pytest.approx(ld_n, rel=1e-12)


def test_non_pd_objective_is_infinite():
    A = np.array([[1.0, 2.0], [2.0, 1.0]])   # P6: not PD
    lam = csc_from_dense(A)
    th = csc_from_dense(np.zeros((1, 2)))
    ob = C.objective(np.ones((3, 1)), np.ones((3, 2)), lam, th, 0.1, 0.1)
    assert not ob["is_pd"] and ob["f"] == math.inf
    assert C.invert_logdet(A)[3] == 1


def test_timed_evaluation_small():
    """The plain definition timed per phase on the host (one evaluation at `small`): positive phase
    times and the same f / list sizes / statistic as the numpy oracle."""
    P = make_problem("small")
    label, lam, th = P.points[0]
    r = C.timed_evaluation(P.X, P.Y, lam, th, P.lam_L, P.lam_T)
    assert all(v > 0 for v in r["seconds"].values())
    on = O.objective(P.X, P.Y, lam, th, P.lam_L, P.lam_T)
    assert r["f"] == pytest.approx(on["f"], rel=1e-12)
    Syy, Sxy = O.covariances(P.X, P.Y)
    Sig, _, _, _ = O.invert_logdet(lam.to_dense())
    rn = O.psi_grad(P.X, P.Y, th, Sig, Syy, Sxy)
    an = O.active_set(rn["GradL"], rn["GradT"], lam, th, P.lam_L, P.lam_T, True, 1e-9)
    assert (r["m_L"], r["m_T"]) == (an["m_L"], an["m_T"])
