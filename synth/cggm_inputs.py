"""Seeded synthetic CGGM problems shared by the oracle (tests) and the CUDA path (bench/tests).

This module holds NONE of the hot path's arithmetic (no covariances, no Cholesky of the
evaluation point, no Psi/gradients/active sets/objective).  It only draws inputs:
X, Y, the generating parameters (Lambda*, Theta*), the evaluation points and the noise
matrix E_noise used by pin I7.  To draw Y from the CGGM it needs
Sigma* = Lambda*^{-1} applied to a block of vectors; it does that with library routines
(LAPACK banded Cholesky via scipy for the chain, a block conjugate-gradient on the sparse
Lambda* otherwise), never with code from `oracle/` or from the CUDA library.

Model (§2.1; reading A1 of DESIGN.md): rows of Y are
    y = -Sigma* Theta*^T x + eps,  eps ~ N(0, Sigma*),  Sigma* = Lambda*^{-1},
i.e. Y = -X Theta* Sigma* + E_noise (BASELINE.json configs: "Y = -X Theta* Sigma* + E").

Configs are BASELINE.json `configs[0..4]`; readings of unstated details (A17 of
SURVEY.md §8(c)) are listed in DESIGN.md §"Input recipe".  Draw order (numpy PCG64,
`default_rng(seed)`), fixed and documented so both sides see the same bytes:
  1. Theta*: for each column j ascending, `choice(p, k, replace=False)` sorted rows;
     then all signs `integers(0,2,nnz)` and magnitudes `uniform(0.5,1.0,nnz)`.
  2. Lambda* (random kind only): pair endpoints `integers(0,q,npairs)` twice, signs,
     magnitudes `uniform(0.2,0.4)`; self pairs dropped, duplicates keep the first draw;
     diagonal = 1 + row |sum|.  Chain kind: deterministic (diag 1.25, off-diag -0.5).
  3. X: `standard_normal((p, n))` transposed -> column-major n x p.
  4. Noise: Z = `standard_normal((ncols(C), n))`, E_noise^T = Lambda*^{-1} C Z with
     C C^T = Lambda* (C = one column per off-diagonal pair plus a diagonal remainder).
  5. Evaluation-point extras (small only): perturbation pairs and values, Theta noise.
"""
from __future__ import annotations

import dataclasses
import numpy as np
import scipy.linalg
import scipy.sparse as sp

__all__ = ["Csc", "Problem", "CONFIGS", "make_problem", "csc_from_triplets"]


@dataclasses.dataclass
class Csc:
    """Compressed sparse column matrix, int64 colptr, int32 row indices (sorted per column)."""
    nrows: int
    ncols: int
    colptr: np.ndarray  # int64, ncols+1
    rowidx: np.ndarray  # int32, nnz
    val: np.ndarray     # float64, nnz

    @property
    def nnz(self) -> int:
        return int(self.rowidx.shape[0])

    def to_scipy(self) -> sp.csc_matrix:
        return sp.csc_matrix((self.val, self.rowidx.astype(np.int64), self.colptr),
                             shape=(self.nrows, self.ncols))

    def to_dense(self) -> np.ndarray:
        d = np.zeros((self.nrows, self.ncols), order="F")
        for j in range(self.ncols):
            a, b = self.colptr[j], self.colptr[j + 1]
            d[self.rowidx[a:b], j] = self.val[a:b]
        return d

    def astype(self, dtype) -> "Csc":
        return Csc(self.nrows, self.ncols, self.colptr, self.rowidx, self.val.astype(dtype))


def csc_from_triplets(nrows, ncols, rows, cols, vals) -> Csc:
    """Build a CSC with rows sorted within each column (duplicates must not occur)."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    vals = np.asarray(vals, dtype=np.float64)
    order = np.lexsort((rows, cols))
    rows, cols, vals = rows[order], cols[order], vals[order]
    colptr = np.zeros(ncols + 1, dtype=np.int64)
    np.add.at(colptr, cols + 1, 1)
    colptr = np.cumsum(colptr)
    return Csc(nrows, ncols, colptr, rows.astype(np.int32), vals)


def csc_from_dense(d: np.ndarray) -> Csc:
    r, c = np.nonzero(d)
    return csc_from_triplets(d.shape[0], d.shape[1], r, c, d[r, c])


CONFIGS = {
    # BASELINE.json configs[0]
    "tiny": dict(n=100, p=40, q=30, lam_kind="chain", theta_k=3, lam=0.5),
    # configs[1]
    "small": dict(n=200, p=1000, q=500, lam_kind="chain", theta_k=5, lam=0.3),
    # configs[2]: "~4 off-diagonals per row" -> 2q pairs (reading A17)
    "medium": dict(n=500, p=10000, q=4000, lam_kind="random", pairs_per_row=2.0, theta_k=10, lam=0.2),
    # configs[3]: lambda unstated -> 0.2 (reading A17)
    "large": dict(n=1000, p=40000, q=20000, lam_kind="chain", theta_k=20, lam=0.2),
    # configs[4]: "~3 off-diagonals per row" -> 1.5q pairs (reading A17)
    "sharded": dict(n=4000, p=200000, q=40000, lam_kind="random", pairs_per_row=1.5, theta_k=25, lam=0.2),
    # NEXT-4 demonstration (not a BASELINE config): q beyond one GPU's dense capacity (the dense
    # evaluation's q x q matrices alone are 8 x 28.8 GB); `large`'s recipe with a sparser target
    "block": dict(n=1000, p=20000, q=60000, lam_kind="chain", theta_k=10, lam=1.0),
}


@dataclasses.dataclass
class Problem:
    name: str
    seed: int
    n: int
    p: int
    q: int
    X: np.ndarray          # n x p, column-major (Fortran order)
    Y: np.ndarray          # n x q, column-major
    lam_star: Csc          # q x q, both triangles stored
    theta_star: Csc        # p x q
    E_noise: np.ndarray    # n x q, column-major; Y = -X Theta* Sigma* + E_noise
    points: list           # [(label, Lambda Csc, Theta Csc)]
    lam_L: float
    lam_T: float
    lam_edges: list = dataclasses.field(default_factory=list)  # [(i, j, w)] i<j off-diagonal pairs of Lambda*


def _theta_star(rng, p, q, k) -> Csc:
    rows = np.empty((q, k), dtype=np.int64)
    for j in range(q):
        rows[j] = np.sort(rng.choice(p, size=k, replace=False))
    nnz = q * k
    signs = rng.integers(0, 2, size=nnz) * 2 - 1
    mags = rng.uniform(0.5, 1.0, size=nnz)
    colptr = np.arange(0, nnz + 1, k, dtype=np.int64)
    return Csc(p, q, colptr, rows.reshape(-1).astype(np.int32), signs * mags)


def _lambda_chain(q):
    """Tridiagonal chain: diag 1.25, off-diagonal -0.5 (BASELINE.json configs[0,1,3])."""
    edges = [(i, i + 1, -0.5) for i in range(q - 1)]
    diag = np.full(q, 1.25)
    return edges, diag


def _lambda_random(rng, q, pairs_per_row):
    """Random sparse SPD: pairs +-U(0.2,0.4), diag = 1 + row |sum| (configs[2,4])."""
    npairs = int(round(pairs_per_row * q))
    a = rng.integers(0, q, size=npairs)
    b = rng.integers(0, q, size=npairs)
    signs = rng.integers(0, 2, size=npairs) * 2 - 1
    mags = rng.uniform(0.2, 0.4, size=npairs)
    keep = a != b
    i = np.minimum(a, b)[keep]
    j = np.maximum(a, b)[keep]
    w = (signs * mags)[keep]
    key = i * q + j
    _, first = np.unique(key, return_index=True)
    first = np.sort(first)
    i, j, w = i[first], j[first], w[first]
    rowabs = np.zeros(q)
    np.add.at(rowabs, i, np.abs(w))
    np.add.at(rowabs, j, np.abs(w))
    diag = 1.0 + rowabs
    edges = list(zip(i.tolist(), j.tolist(), w.tolist()))
    return edges, diag


def _sym_csc(q, edges, diag) -> Csc:
    if edges:
        ei = np.array([e[0] for e in edges], dtype=np.int64)
        ej = np.array([e[1] for e in edges], dtype=np.int64)
        ew = np.array([e[2] for e in edges], dtype=np.float64)
    else:
        ei = ej = np.zeros(0, dtype=np.int64)
        ew = np.zeros(0)
    d = np.arange(q, dtype=np.int64)
    rows = np.concatenate([d, ei, ej])
    cols = np.concatenate([d, ej, ei])
    vals = np.concatenate([diag, ew, ew])
    return csc_from_triplets(q, q, rows, cols, vals)


def _noise_factor(q, edges, diag) -> sp.csc_matrix:
    """Sparse C with C C^T = Lambda*: one column per pair (sqrt|w|(e_i + sign(w) e_j)) plus
    sqrt of the diagonal remainder diag_i - sum_{pairs at i} |w| (> 0 for both kinds)."""
    m = len(edges)
    rem = np.array(diag, dtype=np.float64).copy()
    rows, cols, vals = [], [], []
    for c, (i, j, w) in enumerate(edges):
        s = np.sqrt(abs(w))
        rows += [i, j]
        cols += [c, c]
        vals += [s, np.sign(w) * s]
        rem[i] -= abs(w)
        rem[j] -= abs(w)
    assert np.all(rem > 0), "diagonal remainder must be positive"
    rows += list(range(q))
    cols += list(range(m, m + q))
    vals += list(np.sqrt(rem))
    return sp.csc_matrix((vals, (rows, cols)), shape=(q, m + q))


def _solve_lambda(kind, lam_csc: Csc, edges, diag, B):
    """Return Lambda^{-1} B (B is q x m) with library routines (generator only)."""
    q = lam_csc.nrows
    if kind == "chain":
        ab = np.zeros((2, q))
        ab[1, :] = diag
        for (i, j, w) in edges:
            ab[0, j] = w  # upper band storage: ab[0, j] = A[j-1, j]
        return scipy.linalg.solveh_banded(ab, B, lower=False)
    A = lam_csc.to_scipy().tocsr()
    # block conjugate gradient, per-column step sizes; Lambda* is diagonally dominant
    Xs = np.zeros_like(B)
    R = B.copy()
    P = R.copy()
    rs = np.einsum("ij,ij->j", R, R)
    bn = np.sqrt(np.maximum(rs, 1e-300))
    for _ in range(2000):
        AP = A @ P
        alpha = rs / np.maximum(np.einsum("ij,ij->j", P, AP), 1e-300)
        Xs += P * alpha
        R -= AP * alpha
        rs_new = np.einsum("ij,ij->j", R, R)
        if np.max(np.sqrt(rs_new) / bn) < 1e-15:
            break
        P = R + P * (rs_new / np.maximum(rs, 1e-300))
        rs = rs_new
    return Xs


def make_problem(name: str, seed: int = 0) -> Problem:
    cfg = CONFIGS[name]
    n, p, q, k = cfg["n"], cfg["p"], cfg["q"], cfg["theta_k"]
    rng = np.random.default_rng(seed)
    # 1. Theta*
    theta_star = _theta_star(rng, p, q, k)
    # 2. Lambda*
    if cfg["lam_kind"] == "chain":
        edges, diag = _lambda_chain(q)
    else:
        edges, diag = _lambda_random(rng, q, cfg["pairs_per_row"])
    lam_star = _sym_csc(q, edges, diag)
    # 3. X (column-major n x p)
    X = np.asfortranarray(rng.standard_normal((p, n)).T)
    # 4. noise and Y
    C = _noise_factor(q, edges, diag)
    Z = rng.standard_normal((C.shape[1], n))
    M_noise = np.asarray(C @ Z)                       # q x n, covariance Lambda*
    W_star_T = np.asarray((theta_star.to_scipy().T @ X.T))   # q x n  (= (X Theta*)^T)
    sol = _solve_lambda(cfg["lam_kind"], lam_star, edges, diag, np.hstack([M_noise, W_star_T]))
    E_noise = np.asfortranarray(sol[:, :n].T)
    Y = np.asfortranarray((sol[:, :n] - sol[:, n:]).T)
    # 5. evaluation points
    lam = cfg["lam"]
    points = []
    if name == "tiny":
        ident = _sym_csc(q, [], np.ones(q))
        empty = Csc(p, q, np.zeros(q + 1, dtype=np.int64), np.zeros(0, dtype=np.int32), np.zeros(0))
        points.append(("identity", ident, empty))
        points.append(("truth", lam_star, theta_star))
    elif name == "small":
        points.append(("truth", lam_star, theta_star))
        seen = set()
        pi, pj = [], []
        while len(pi) < q - 1:
            a, b = rng.integers(0, q, size=2)
            if a == b:
                continue
            a, b = (int(min(a, b)), int(max(a, b)))
            if (a, b) in seen:
                continue
            seen.add((a, b))
            pi.append(a)
            pj.append(b)
        pv = rng.standard_normal(q - 1)
        theta_noise = rng.normal(0.0, 0.05, size=theta_star.nnz)
        base = lam_star.to_dense()
        P = np.zeros((q, q))
        P[pi, pj] = pv
        P[pj, pi] = pv
        t = 0.1
        while True:
            cand = base + t * P
            try:
                np.linalg.cholesky(cand)
                break
            except np.linalg.LinAlgError:
                t *= 0.5
        lam_pert = csc_from_dense(np.asfortranarray(cand))
        theta_pert = Csc(p, q, theta_star.colptr, theta_star.rowidx, theta_star.val + theta_noise)
        points.append(("perturbed", lam_pert, theta_pert))
    else:
        points.append(("truth", lam_star, theta_star))
    return Problem(name, seed, n, p, q, X, Y, lam_star, theta_star, E_noise, points, lam, lam,
                   lam_edges=edges)
