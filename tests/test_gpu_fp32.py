"""FP32 variant (reading A18: inputs rounded to fp32 once, fp32 arithmetic/accumulation in every
kernel; outputs compared with the fp64 oracle on the fp64 inputs).

Tolerances: Sigma, Psi, gradients rel-Frobenius <= 1e-4 (north_star); objective relative error
<= 1e-6 (A18; measured <= 3e-7 on tiny/small/medium);
active sets exact outside a tie band ||g| - lam| <= 1e-4 * max|g| (the fp32 gradient error
scale, reading A5)."""
import ctypes

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import cggm_oracle as O  # noqa: E402
from synth.cggm_inputs import make_problem  # noqa: E402

A_KLE_M, A_KGE_M, B_KLE_N, B_KGE_N, SYM_LOWER, SYM_MIRROR = 1, 2, 4, 8, 16, 32


def relf(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / np.linalg.norm(b))


@pytest.fixture(scope="module")
def ctx32():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1509_04681_b200 import Context
    return Context(0, dtype="f32")


def run_f32(ctx, tA, tB, A, B, C0, alpha, beta, flags, M, N, K):
    from paper_1509_04681_b200.api import colmajor_empty, ld_of
    ts = []
    for a in (A, B, C0):
        t = colmajor_empty(a.shape[0], a.shape[1], dtype=torch.float32)
        t.copy_(torch.from_numpy(np.asfortranarray(a)).float())
        ts.append(t)
    dA, dB, dC = ts
    ctx._check(ctx.lib.cggm_test_gemm_f32(ctx.h, int(tA), int(tB), M, N, K, ctypes.c_void_p(dA.data_ptr()), ld_of(dA),
                                          ctypes.c_void_p(dB.data_ptr()), ld_of(dB), ctypes.c_void_p(dC.data_ptr()),
                                          ld_of(dC), alpha, beta, flags))
    torch.cuda.synchronize()
    return dC.double().cpu().numpy()


@pytest.mark.parametrize("tA", [False, True])
@pytest.mark.parametrize("tB", [False, True])
@pytest.mark.parametrize("M,N,K", [(1, 1, 1), (37, 45, 29), (300, 260, 171), (256, 64, 300), (513, 129, 1000)])
@pytest.mark.parametrize("mode", [1, 5])   # 3-D / 2-D TMA boxes for MN-inner operands
def test_ffma_gemm_variants(ctx32, tA, tB, M, N, K, mode):
    ctx32._check(ctx32.lib.cggm_test_set_tile(ctx32.h, mode))
    rng = np.random.default_rng(M + 3 * N + 7 * K)
    A = rng.standard_normal((K, M) if tA else (M, K)).astype(np.float32).astype(np.float64)
    B = rng.standard_normal((N, K) if tB else (K, N)).astype(np.float32).astype(np.float64)
    C0 = rng.standard_normal((M, N)).astype(np.float32).astype(np.float64)
    ref = 0.75 * ((A.T if tA else A) @ (B.T if tB else B)) - 0.5 * C0
    out = run_f32(ctx32, tA, tB, A, B, C0, 0.75, -0.5, 0, M, N, K)
    assert relf(out, ref) < 2e-6
    ctx32._check(ctx32.lib.cggm_test_set_tile(ctx32.h, 0))


@pytest.mark.parametrize("flags", [A_KLE_M, A_KGE_M, B_KLE_N, B_KGE_N])
def test_ffma_gemm_triangular(ctx32, flags):
    rng = np.random.default_rng(flags)
    n = 333
    A = rng.standard_normal((n, n)).astype(np.float32).astype(np.float64)
    B = rng.standard_normal((n, n)).astype(np.float32).astype(np.float64)
    A = np.tril(A) if flags & A_KLE_M else np.triu(A) if flags & A_KGE_M else A
    B = np.triu(B) if flags & B_KLE_N else np.tril(B) if flags & B_KGE_N else B
    out = run_f32(ctx32, False, False, A, B, np.zeros((n, n)), 1.0, 0.0, flags, n, n, n)
    assert relf(out, A @ B) < 2e-6


def test_ffma_gemm_sym_and_trapezoid(ctx32):
    rng = np.random.default_rng(3)
    q, K = 385, 300
    A = rng.standard_normal((K, q)).astype(np.float32).astype(np.float64)
    out = run_f32(ctx32, True, False, A, A, np.zeros((q, q)), 1.0, 0.0, SYM_LOWER | SYM_MIRROR, q, q, K)
    np.testing.assert_array_equal(out, out.T)
    assert relf(out, A.T @ A) < 2e-6
    N, extra = 300, 257
    Bm = rng.standard_normal((N + extra, K)).astype(np.float32).astype(np.float64)
    C0 = rng.standard_normal((N + extra, N)).astype(np.float32).astype(np.float64)
    out2 = run_f32(ctx32, False, True, Bm, Bm[:N].copy(), C0, -1.0, 1.0, SYM_LOWER, N + extra, N, K)
    mask = np.tril(np.ones((N + extra, N), dtype=bool))
    ref = C0 - Bm @ Bm[:N].T
    assert np.max(np.abs(out2[mask] - ref[mask])) < 1e-3
    np.testing.assert_array_equal(out2[~mask], C0[~mask].astype(np.float32))


_CACHE = {}


def oracle_point(name, k):
    if (name, k) not in _CACHE:
        P = make_problem(name)
        _, lam, th = P.points[k]
        Syy, Sxy = O.covariances(P.X, P.Y)
        Sig, ld, ok, _ = O.invert_logdet(lam.to_dense())
        r = O.psi_grad(P.X, P.Y, th, Sig, Syy, Sxy)
        ob = O.objective(P.X, P.Y, lam, th, P.lam_L, P.lam_T)
        _CACHE[(name, k)] = (P, dict(Syy=Syy, Sigma=Sig, logdet=ld, obj=ob, **r))
    return _CACHE[(name, k)]


@pytest.mark.parametrize("name,k", [("tiny", 1), ("small", 0), ("small", 1), ("medium", 0)])
def test_fp32_parity(ctx32, name, k):
    from paper_1509_04681_b200 import DeviceCsc, to_device_colmajor
    from paper_1509_04681_b200.api import newton_evaluation
    P, ref = oracle_point(name, k)
    _, lam, th = P.points[k]
    f32 = torch.float32
    X, Y = to_device_colmajor(P.X, dtype=f32), to_device_colmajor(P.Y, dtype=f32)
    Lg, Tg = DeviceCsc.from_host(lam, dtype=f32), DeviceCsc.from_host(th, dtype=f32)
    Syy, _ = ctx32.cggm_covariances(X, Y, want_sxy=False)
    assert relf(Syy.double().cpu().numpy(), ref["Syy"]) <= 1e-5
    cap = 4_000_000
    bufs = {key: torch.empty(cap, dtype=torch.int32, device="cuda") for key in ("L_row", "L_col", "T_row", "T_col")}
    tie = 1e-4 * max(float(np.abs(ref["GradL"]).max()), float(np.abs(ref["GradT"]).max()))
    r = newton_evaluation(ctx32, X, Y, Syy, Lg, Tg, P.lam_L, P.lam_T, True, bufs, tie_eps=tie)
    assert r["is_pd"]
    errs = {key: relf(r[key].double().cpu().numpy(), ref[key]) for key in ("Sigma", "Psi", "GradL", "GradT")}
    for key, e in errs.items():
        assert e <= 1e-4, (key, e)
    S = r["Sigma"].cpu().numpy()
    np.testing.assert_array_equal(S, S.T)
    assert r["logdet"] == pytest.approx(ref["logdet"], rel=1e-5, abs=1e-5)
    ob = r["objective"]
    assert ob["f"] == pytest.approx(ref["obj"]["f"], rel=1e-6)
    # active sets: exact outside the fp32 tie band
    a = O.active_set(ref["GradL"], ref["GradT"], lam, th, P.lam_L, P.lam_T, True, tie)
    for rk, ck, tm in (("L_row", "L_col", a["tie_mask_L"]), ("T_row", "T_col", a["tie_mask_T"])):
        g = set(zip(r["active"][rk].cpu().numpy().tolist(), r["active"][ck].cpu().numpy().tolist()))
        o = set(zip(a[rk].tolist(), a[ck].tolist()))
        for (i, j) in g ^ o:
            assert tm[i, j], (rk, i, j)
