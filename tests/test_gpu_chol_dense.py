"""Recursive Cholesky / triangular inverse on dense SPD matrices (cggm_test_chol_dense) against the
oracle's textbook column Cholesky and forward substitution, at sizes that
cross every recursion level the large configs use (leaf 64, block-inverse subtrees, lookahead
deferral) with ragged edges."""
import ctypes

import numpy as np
import pytest
import torch

from oracle import cggm_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    from paper_1509_04681_b200 import Context
    return Context(0)


def _spd(q, seed):
    rng = np.random.default_rng(seed)
    M = rng.standard_normal((q, q)) / np.sqrt(q)
    return M @ M.T + np.eye(q)


def _run(ctx, A, full):
    from paper_1509_04681_b200 import colmajor_empty, to_device_colmajor
    q = A.shape[0]
    Ad = to_device_colmajor(A)
    Xd = colmajor_empty(q, q)
    ld, fc = ctypes.c_double(), ctypes.c_int64()
    ctx._sync_stream()
    st = ctx.lib.cggm_test_chol_dense(ctx.h, ctypes.c_void_p(Ad.data_ptr()), Ad.stride(1), q,
                                      ctypes.c_void_p(Xd.data_ptr()), Xd.stride(1), int(full),
                                      ctypes.byref(ld), ctypes.byref(fc))
    assert st == 0, ctx.lib.cggm_last_error(ctx.h)
    return Xd.cpu().numpy(), ld.value, fc.value


@pytest.mark.parametrize("q", [1, 37, 64, 65, 200, 513, 777, 1100, 2049])
def test_full_inverse_matches_oracle(ctx, q):
    A = _spd(q, q)
    L = O.cholesky(A)[0]
    Linv_ref = O.forward_substitution(L, np.eye(q))
    X, logdet, fc = _run(ctx, A, True)
    Xl = np.tril(X)
    err = np.linalg.norm(Xl - Linv_ref) / np.linalg.norm(Linv_ref)
    assert err <= 1e-12, err
    assert fc == -1
    assert abs(logdet - O.logdet_from_cholesky(L)) <= 1e-10 * max(1.0, abs(logdet))


@pytest.mark.parametrize("q", [300, 1500])
def test_potrf_only_logdet_and_pd(ctx, q):
    A = _spd(q, q + 1)
    L = O.cholesky(A)[0]
    _, logdet, fc = _run(ctx, A, False)
    assert fc == -1
    assert abs(logdet - O.logdet_from_cholesky(L)) <= 1e-10 * abs(logdet)


@pytest.mark.parametrize("q,bad", [(700, 650), (1100, 3), (2049, 2048)])
def test_first_failing_pivot(ctx, q, bad):
    """A made indefinite at column `bad` only: the first failing pivot is exactly `bad` (A10)."""
    A = _spd(q, 5)
    A[bad, bad] = -1.0
    for full in (True, False):
        _, _, fc = _run(ctx, A, full)
        assert fc == bad


def test_lookahead_option_same_result(ctx):
    """CGGM_OPT_LOOKAHEAD_MIN only changes the schedule (side streams), not the arithmetic: the
    inverse with lookahead off and on at a small threshold agrees to the last bits."""
    from paper_1509_04681_b200 import _abi
    q = 3000
    A = _spd(q, 11)
    ctx.set_option(_abi.CGGM_OPT_LOOKAHEAD_MIN, 0)
    try:
        X0, l0, _ = _run(ctx, A, True)
        ctx.set_option(_abi.CGGM_OPT_LOOKAHEAD_MIN, 128)
        X1, l1, _ = _run(ctx, A, True)
    finally:
        ctx.set_option(_abi.CGGM_OPT_LOOKAHEAD_MIN, 256)
    assert np.linalg.norm(np.tril(X0) - np.tril(X1)) <= 1e-15 * np.linalg.norm(np.tril(X0))
    assert abs(l0 - l1) <= 1e-13 * abs(l0)
    from paper_1509_04681_b200.api import CggmError
    with pytest.raises(CggmError):
        ctx.set_option(99, 1)
