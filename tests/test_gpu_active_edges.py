"""Active-set compaction at ragged / edge sizes, on every kernel path, against the oracle's plain
definition (oracle.cggm_oracle.active_set, §2.2 with readings A5-A7): the split Lambda
compaction (flag bitmask -> column scan -> writer, columns paired per CTA), the single-pass
look-back kernel (CGGM_ACT_ONEPASS=1) and the scalar fallback (CGGM_NO_ACTIVE_VEC=1).  Sizes
straddle the 64-row chunk, the 32-chunk writer rounds and the odd q of the column pairing; the
gradients are drawn so that about half of the entries are active, with supports that include
entries below the threshold and explicit zeros.  Lists and counts are integer results: bit-exact."""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import cggm_oracle as O  # noqa: E402
from synth.cggm_inputs import csc_from_triplets  # noqa: E402

VARIANTS = {"split": {}, "onepass": {"CGGM_ACT_ONEPASS": "1"}, "scalar": {"CGGM_NO_ACTIVE_VEC": "1"}}
_CTX = {}


def ctx_for(variant):
    if variant not in _CTX:
        if not torch.cuda.is_available():
            pytest.skip("no CUDA device")
        from paper_1509_04681_b200 import Context
        env = VARIANTS[variant]
        os.environ.update(env)
        try:
            _CTX[variant] = Context(0)
        finally:
            for k in env:
                os.environ.pop(k, None)
    return _CTX[variant]


def case(p, q, seed, drop_diag=False):
    rng = np.random.default_rng(seed)
    G = rng.standard_normal((q, q))
    GL = (G + G.T) / 2.0
    if drop_diag:   # unpenalised-diagonal case: exact zeros and tiny values on the diagonal
        d = np.arange(q)
        GL[d[::3], d[::3]] = 0.0
        GL[d[1::5], d[1::5]] = 1e-300
    GT = rng.standard_normal((p, q))
    # symmetric Lambda support: diagonal, random off-diagonal pairs (some with small gradients), and
    # one explicit stored zero (reading A7: value test)
    pairs = {(i, i) for i in range(q)}
    for _ in range(2 * q):
        i, j = rng.integers(0, q, 2)
        pairs.add((int(i), int(j)))
        pairs.add((int(j), int(i)))
    if drop_diag:   # the diagonal is then decided by the gradient alone (lam_ii = 0)
        pairs = {(i, j) for (i, j) in pairs if i != j} or {(0, 0)}
    rows, cols = zip(*sorted(pairs))
    vals = rng.uniform(0.1, 0.5, len(rows)) * rng.choice([-1.0, 1.0], len(rows))
    for k, (r, c) in enumerate(zip(rows, cols)):
        if r == c:
            vals[k] = 2.0 + q
    sym = {(r, c): v for r, c, v in zip(rows, cols, vals)}
    vals = np.array([sym[(min(r, c), max(r, c))] for r, c in zip(rows, cols)])
    if q > 2:   # an explicit zero off the diagonal, both triangles
        i0 = next(k for k, (r, c) in enumerate(zip(rows, cols)) if r != c)
        r0, c0 = rows[i0], cols[i0]
        vals = np.array([0.0 if (r, c) in ((r0, c0), (c0, r0)) else v for r, c, v in zip(rows, cols, vals)])
    lam = csc_from_triplets(q, q, rows, cols, vals)
    k = max(1, p // 50)
    trow, tcol = [], []
    for j in range(q):
        rr = rng.choice(p, size=min(k, p), replace=False)
        trow += list(rr)
        tcol += [j] * len(rr)
    th = csc_from_triplets(p, q, trow, tcol, rng.uniform(0.5, 1.0, len(trow)))
    return GL, GT, lam, th


@pytest.mark.parametrize("diag", ["penalised", "unpenalised", "unpenalised_nodiag"])
@pytest.mark.parametrize("variant", list(VARIANTS))
@pytest.mark.parametrize("p,q", [(1, 1), (3, 2), (64, 63), (65, 64), (130, 65), (200, 127), (129, 128),
                                 (2049, 129), (300, 257), (70, 1000), (4100, 33)])
def test_active_lists_edge_sizes(variant, p, q, diag):
    """penalize_diag = 0 (reading A3: lam_ii = 0) on every kernel path: with the diagonal stored in
    Lambda (forced active, the subgradient uses |g_ii|) and with it absent from the support (the
    diagonal then enters iff |g_ii| > 0, exact zeros do not, 1e-300 does)."""
    from paper_1509_04681_b200 import DeviceCsc, to_device_colmajor
    c = ctx_for(variant)
    pen = diag == "penalised"
    GL, GT, lam, th = case(p, q, seed=1000 * p + q, drop_diag=diag == "unpenalised_nodiag")
    lam_L, lam_T = 0.6, 1.2
    ref = O.active_set(GL, GT, lam, th, lam_L, lam_T, penalize_diag=pen)
    got = c.cggm_active_set(to_device_colmajor(GL), to_device_colmajor(GT), DeviceCsc.from_host(lam),
                            DeviceCsc.from_host(th), lam_L, lam_T, penalize_diag=pen)
    assert (got["m_L"], got["m_T"]) == (ref["m_L"], ref["m_T"])
    assert (got["ties_L"], got["ties_T"]) == (ref["ties_L"], ref["ties_T"])
    for key in ("L_row", "L_col", "T_row", "T_col"):
        assert np.array_equal(got[key].cpu().numpy(), ref[key]), key
    sub = O.min_norm_subgradient(GL, GT, lam, th, lam_L, lam_T, penalize_diag=pen)
    assert got["subgrad_l1"] == pytest.approx(sub, rel=1e-12, abs=1e-12)
