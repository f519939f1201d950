"""Pins of the coordinate-descent oracle (oracle/ancd_oracle.py) against what the paper and the
mathematics fix, independent of the oracle's own formulas:

  P18  every Lambda coordinate update is the exact minimiser of the l1-regularised quadratic model
       of Eq. (6) along that symmetric coordinate (brute-force 1-D minimisation of the model
       evaluated from its definition with dense matrix products) -- pins a_L (both forms), b_L, c_L
  P19  U = Delta Sigma after a sweep (recomputed)
  P20  the model value never increases across a sweep
  P21  q = 1 scalar example: Lambda = [1], S_yy = [s], Theta = 0, lam = 0 -> Delta = 1 - s
  P22  every Theta coordinate update is the exact minimiser of Eq. (7) along that coordinate
  P23  repeated Theta sweeps reach the minimiser of Eq. (7) found by an independent proximal-gradient
       solve of the same quadratic lasso
  P24  Armijo: the accepted Lambda is PD and decreases f; Lambda = I, D = -2I backtracks below 1/2
  P25  Algorithm 1 meets its stopping rule and its objective matches an independent joint
       proximal-gradient solver of Eq. (1) to 1e-6 relative (convexity)
  P26  the quadratic model of Eq. (6) (lambda_surrogate) is the second-order Taylor expansion of the
       oracle's g (Eq. 1 / Eq. 4) by central first and second differences
"""
import math

import numpy as np
import pytest

from oracle import ancd_oracle as A
from oracle import cggm_oracle as O

pytestmark = pytest.mark.filterwarnings("ignore::RuntimeWarning")


def _instance(q, seed, p=None, n=40):
    rng = np.random.default_rng(seed)
    p = p or q + 2
    X = rng.standard_normal((n, p))
    Y = rng.standard_normal((n, q)) + 0.5 * X[:, :q]
    M = rng.standard_normal((q, q)) * 0.3
    Lam = M @ M.T + np.eye(q)
    Theta = np.where(rng.random((p, q)) < 0.3, rng.standard_normal((p, q)) * 0.3, 0.0)
    return X, Y, Lam, Theta


def _model_pieces(X, Y, Lam, Theta):
    n = X.shape[0]
    Sxx, Syy, Sxy = X.T @ X / n, Y.T @ Y / n, X.T @ Y / n
    Sigma = np.linalg.inv(Lam)
    Psi = Sigma @ Theta.T @ Sxx @ Theta @ Sigma
    GradL = Syy - Sigma - Psi
    return Sxx, Syy, Sxy, Sigma, Psi, GradL


def _brute_min_1d(fun, center, scale):
    """Minimise a convex 1-D function: coarse grid, then golden-section refinement."""
    xs = center + scale * np.linspace(-4, 4, 4001)
    vals = np.array([fun(x) for x in xs])
    k = int(np.argmin(vals))
    lo, hi = xs[max(k - 1, 0)], xs[min(k + 1, len(xs) - 1)]
    g = (math.sqrt(5) - 1) / 2
    for _ in range(200):
        c, d = hi - g * (hi - lo), lo + g * (hi - lo)
        if fun(c) < fun(d):
            hi = d
        else:
            lo = c
    return 0.5 * (lo + hi)


@pytest.mark.parametrize("penalize_diag", [True, False])
def test_p18_lambda_update_is_exact_coordinate_minimiser(penalize_diag):
    X, Y, Lam, Theta = _instance(5, 1)
    Sxx, Syy, Sxy, Sigma, Psi, GradL = _model_pieces(X, Y, Lam, Theta)
    rng = np.random.default_rng(2)
    D0 = rng.standard_normal((5, 5)) * 0.05
    D0 = D0 + D0.T
    lam = 0.07
    for (i, j) in [(0, 0), (1, 3), (2, 4), (4, 4), (0, 2)]:
        D, _, _ = A.lambda_newton_direction(Sigma, Psi, GradL, Lam, [i], [j], lam, penalize_diag, Delta=D0)
        mu = D[i, j] - D0[i, j]
        E = np.zeros((5, 5))
        E[i, j] = E[j, i] = 1.0

        def model(t):
            return A.lambda_surrogate(D0 + t * E, GradL, Sigma, Psi, Lam, lam, penalize_diag)

        mu_bf = _brute_min_1d(model, mu, 0.5)
        # (a flat minimum resolves to ~sqrt(eps) in the argument; the value test is the sharp one)
        assert abs(mu - mu_bf) <= 1e-6, (i, j, mu, mu_bf)
        m0 = model(mu)
        assert m0 <= model(mu_bf) + 1e-13 * abs(m0)
        for dl in (1e-6, 1e-4, 1e-2):
            assert m0 <= model(mu + dl) and m0 <= model(mu - dl)


def test_p19_p20_sweep_keeps_u_and_decreases_model():
    X, Y, Lam, Theta = _instance(7, 3)
    Sxx, Syy, Sxy, Sigma, Psi, GradL = _model_pieces(X, Y, Lam, Theta)
    rows, cols = np.triu_indices(7)
    order = np.lexsort((rows, cols))      # column-major, i <= j
    rows, cols = rows[order], cols[order]
    D = np.zeros((7, 7))
    prev = A.lambda_surrogate(D, GradL, Sigma, Psi, Lam, 0.05)
    for k in range(len(rows)):   # one coordinate at a time: the model never increases
        D, U, _ = A.lambda_newton_direction(Sigma, Psi, GradL, Lam, rows[k:k + 1], cols[k:k + 1], 0.05, Delta=D)
        cur = A.lambda_surrogate(D, GradL, Sigma, Psi, Lam, 0.05)
        assert cur <= prev + 1e-13
        prev = cur
    D2, U2, _ = A.lambda_newton_direction(Sigma, Psi, GradL, Lam, rows, cols, 0.05, passes=3)
    np.testing.assert_allclose(U2, D2 @ Sigma, atol=1e-12)
    np.testing.assert_array_equal(D2, D2.T)


@pytest.mark.parametrize("seed", [21, 22, 23])
def test_p26_lambda_surrogate_matches_g_by_finite_differences(seed):
    """The quadratic model of Eq. (6) is the second-order Taylor expansion of g of Eq. (1) (P:270-282,
    Eq. 4), checked against the oracle's g itself (O.objective with lam = 0) along random symmetric
    directions D, with Theta != 0 so that Psi matters:
      linear:    (g(L+tD) - g(L-tD)) / 2t            -> tr(GradL D)             (error O(t^2))
      quadratic: (g(L+tD) + g(L-tD) - 2 g(L)) / 2t^2 -> 1/2 tr(DSDS) + tr(DSDP)  (error O(t^2))
    The surrogate's quadratic part is read off lambda_surrogate at lam = 0 as
    (m(tD) + m(-tD)) / 2t^2 (exact for a quadratic).  A wrong Hessian term (a dropped Psi term, a
    factor 2, Sigma for Psi) changes the quadratic by O(1) relative and fails."""
    from synth.cggm_inputs import csc_from_dense
    X, Y, Lam, Theta = _instance(6, seed, p=8)
    Sxx, Syy, Sxy, Sigma, Psi, GradL = _model_pieces(X, Y, Lam, Theta)
    rng = np.random.default_rng(seed + 100)
    tc = csc_from_dense(Theta)

    def g(L):
        return O.objective(X, Y, csc_from_dense(L), tc, 0.0, 0.0)["g"]

    g0 = g(Lam)
    for _ in range(3):
        D = rng.standard_normal((6, 6))
        D = 0.5 * (D + D.T)
        t = 2e-4
        gp, gm = g(Lam + t * D), g(Lam - t * D)
        lin_fd = (gp - gm) / (2 * t)
        quad_fd = (gp + gm - 2 * g0) / (2 * t * t)
        mp = A.lambda_surrogate(t * D, GradL, Sigma, Psi, Lam, 0.0)
        mm = A.lambda_surrogate(-t * D, GradL, Sigma, Psi, Lam, 0.0)
        quad_model = (mp + mm) / (2 * t * t)
        lin_model = (mp - mm) / (2 * t)
        assert lin_model == pytest.approx(float(np.sum(GradL * D)), rel=1e-12)
        assert lin_fd == pytest.approx(lin_model, rel=1e-6)
        assert quad_fd == pytest.approx(quad_model, rel=1e-5)
        # and the Psi term is not negligible here (the check would not see a Psi mistake otherwise)
        DS = D @ Sigma
        assert abs(np.trace(DS @ D @ Psi)) > 0.05 * abs(quad_model)


@pytest.mark.parametrize("s", [0.3, 1.0, 2.5])
def test_p21_scalar_newton_step(s):
    D, _, _ = A.lambda_newton_direction(np.eye(1), np.zeros((1, 1)), np.array([[s - 1.0]]), np.eye(1), [0], [0], 0.0)
    assert D[0, 0] == pytest.approx(1.0 - s, abs=1e-15)


def test_p22_theta_update_is_exact_coordinate_minimiser():
    X, Y, Lam, Theta = _instance(4, 5, p=6)
    Sxx, Syy, Sxy, Sigma, Psi, GradL = _model_pieces(X, Y, Lam, Theta)
    lam = 0.05
    for (i, j) in [(0, 0), (5, 3), (2, 1), (3, 3)]:
        T, _ = A.theta_cd_sweep(Sigma, Sxx, Sxy, Theta, [i], [j], lam)
        mu = T[i, j] - Theta[i, j]
        E = np.zeros_like(Theta)
        E[i, j] = 1.0
        fun = lambda t: A.theta_subproblem(Theta + t * E, Sigma, Sxx, Sxy, lam)  # noqa: E731
        mu_bf = _brute_min_1d(fun, mu, 0.5)
        assert abs(mu - mu_bf) <= 1e-6, (i, j, mu, mu_bf)
        m0 = fun(mu)
        assert m0 <= fun(mu_bf) + 1e-13 * abs(m0)
        for dl in (1e-6, 1e-4, 1e-2):
            assert m0 <= fun(mu + dl) and m0 <= fun(mu - dl)


def test_p23_theta_sweeps_reach_quadratic_lasso_minimiser():
    X, Y, Lam, _ = _instance(4, 7, p=6)
    Sxx, Syy, Sxy, Sigma, Psi, GradL = _model_pieces(X, Y, Lam, np.zeros((6, 4)))
    lam = 0.03
    rows, cols = np.meshgrid(np.arange(6), np.arange(4), indexing="ij")
    rows, cols = rows.T.ravel(), cols.T.ravel()    # column-major
    T, _ = A.theta_cd_sweep(Sigma, Sxx, Sxy, np.zeros((6, 4)), rows, cols, lam, passes=400)
    # independent: proximal gradient on Eq. (7), step 1/L with L = 2 ||Sxx|| ||Sigma||
    Lc = 2 * np.linalg.norm(Sxx, 2) * np.linalg.norm(Sigma, 2)
    Z = np.zeros((6, 4))
    for _ in range(20000):
        G = 2 * Sxy + 2 * Sxx @ Z @ Sigma
        W = Z - G / Lc
        Z = np.sign(W) * np.maximum(np.abs(W) - lam / Lc, 0.0)
    np.testing.assert_allclose(T, Z, atol=1e-7)
    assert A.theta_subproblem(T, Sigma, Sxx, Sxy, lam) <= A.theta_subproblem(Z, Sigma, Sxx, Sxy, lam) + 1e-12


def test_p24_armijo_pd_and_decrease():
    X, Y, Lam, Theta = _instance(5, 9)
    Sxx, Syy, Sxy, Sigma, Psi, GradL = _model_pieces(X, Y, Lam, Theta)
    rows, cols = np.triu_indices(5)
    D, _, _ = A.lambda_newton_direction(Sigma, Psi, GradL, Lam, rows, cols, 0.05)
    f0 = A.objective_dense(X, Y, Lam, Theta, 0.05, 0.05)
    r = A.armijo_lambda(X, Y, Lam, Theta, D, GradL, 0.05, 0.05, f0=f0)
    assert r["alpha"] > 0 and r["f"] < f0
    assert np.linalg.eigvalsh(r["Lam"]).min() > 0
    # Lambda = I, D = -2I fails PD at alpha = 1 and 1/2; with S_yy = 2I (GradL = I, so D
    # is a descent direction) f(I - 2a I) = -3 ln(1 - 2a) + 6 (1 - 2a) is minimal at a = 1/4, where
    # the Armijo test holds: the first accepted step is exactly 1/4
    q = 3
    Xs, Ys = np.zeros((4, 1)), np.eye(4, q) * math.sqrt(8.0)
    r2 = A.armijo_lambda(Xs, Ys, np.eye(q), np.zeros((1, q)), -2.0 * np.eye(q), np.eye(q), 0.0, 0.0)
    assert r2["alpha"] == 0.25 and r2["backtracks"] == 2
    assert r2["f"] == pytest.approx(3 * math.log(2) + 3.0, rel=1e-14)


@pytest.mark.parametrize("seed,penalize_diag", [(11, True), (12, False), (13, True)])
def test_p25_ancd_matches_independent_prox_grad(seed, penalize_diag):
    rng = np.random.default_rng(seed)
    n, p, q = 60, 6, 4
    X = rng.standard_normal((n, p))
    B = np.where(rng.random((p, q)) < 0.4, rng.standard_normal((p, q)), 0.0)
    Y = X @ B + rng.standard_normal((n, q))
    lam_L, lam_T = 0.1, 0.15
    fit = A.ancd_fit(X, Y, lam_L, lam_T, penalize_diag, max_iter=500, tol=1e-7)
    ref = A.prox_grad_fit(X, Y, lam_L, lam_T, penalize_diag)
    assert fit["history"][-1][4] is None, "stopping rule not met"
    assert fit["f"] == pytest.approx(ref["f"], rel=1e-6)
    np.testing.assert_allclose(fit["Lam"], ref["Lam"], atol=2e-3)
    np.testing.assert_allclose(fit["Theta"], ref["Theta"], atol=2e-3)
    # objective non-increasing over the outer iterations (descent method)
    fs = [h[0] for h in fit["history"]]
    assert all(b <= a + 1e-12 for a, b in zip(fs, fs[1:]))


def test_paper_stopping_rule_on_tiny_config():
    """Algorithm 1 with the paper's rule (tol 0.01) on the `tiny` config terminates."""
    from synth.cggm_inputs import make_problem
    P = make_problem("tiny")
    fit = A.ancd_fit(P.X, P.Y, P.lam_L, P.lam_T, max_iter=100, tol=0.01)
    assert fit["history"][-1][4] is None and fit["iters"] < 100
