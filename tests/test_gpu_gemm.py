"""FP64 DMMA GEMM engine vs a plain fp64 product (numpy), through the test-only export
cggm_test_gemm (include/cggm_testing.h).  Covers the four transposition variants, ragged
edges (several tiles + tails), triangular k-ranges and symmetric lower/mirror outputs."""
import ctypes

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

A_KLE_M, A_KGE_M, B_KLE_N, B_KGE_N, SYM_LOWER, SYM_MIRROR = 1, 2, 4, 8, 16, 32


@pytest.fixture(scope="module", params=[0, 1, "big", 2, 5, 6, "direct"],
                ids=["auto_small", "tile128", "tile128_square", "tile64", "tile128_2d", "tile64_2d", "auto_small_direct"])
def ctx(request):
    """auto_small: small shapes on the cp.async kernel; auto_small_direct: on the direct-load one;
    tile128: the two-CTA 128x64 tiles (the default, CGGM_MID_TILE=3) -- symmetric (SYM_LOWER) products
    walk 128x128 squares in two column halves with per-element diagonal masking; tile128_square:
    everything on 128x128 (CGGM_MID_TILE=0)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import os
    from paper_1509_04681_b200 import Context
    direct = request.param == "direct"
    os.environ["CGGM_NO_SMALL_ASYNC"] = "1" if direct else "0"
    if request.param == "big":
        os.environ["CGGM_MID_TILE"] = "0"
    try:
        c = Context(0)
    finally:
        os.environ.pop("CGGM_NO_SMALL_ASYNC", None)
        os.environ.pop("CGGM_MID_TILE", None)
    tile = {"direct": 0, "big": 1}.get(request.param, request.param)
    c._check(c.lib.cggm_test_set_tile(c.h, tile))
    return c


def dev(a, ld_pad=0):
    from paper_1509_04681_b200.api import colmajor_empty
    t = colmajor_empty(a.shape[0], a.shape[1])
    t.copy_(torch.from_numpy(np.asfortranarray(a)))
    return t


def run(ctx, tA, tB, A, B, C0, alpha, beta, flags, M, N, K):
    from paper_1509_04681_b200.api import ld_of
    dA, dB, dC = dev(A), dev(B), dev(C0)
    st = ctx.lib.cggm_test_gemm(ctx.h, int(tA), int(tB), M, N, K, ctypes.c_void_p(dA.data_ptr()), ld_of(dA),
                                ctypes.c_void_p(dB.data_ptr()), ld_of(dB), ctypes.c_void_p(dC.data_ptr()), ld_of(dC),
                                alpha, beta, flags)
    ctx._check(st)
    torch.cuda.synchronize()
    return dC.cpu().numpy()


@pytest.mark.parametrize("tA", [False, True])
@pytest.mark.parametrize("tB", [False, True])
@pytest.mark.parametrize("M,N,K", [(1, 1, 1), (37, 45, 29), (128, 128, 16), (300, 260, 171), (513, 129, 1000),
                                   (320, 208, 96), (256, 64, 300), (1064, 64, 64), (64, 1064, 200), (100, 90, 256)])
def test_gemm_variants(ctx, tA, tB, M, N, K):
    rng = np.random.default_rng(M * 7 + N * 3 + K)
    A = rng.standard_normal((K, M) if tA else (M, K))
    B = rng.standard_normal((N, K) if tB else (K, N))
    C0 = rng.standard_normal((M, N))
    ref = 0.75 * ((A.T if tA else A) @ (B.T if tB else B)) - 0.5 * C0
    out = run(ctx, tA, tB, A, B, C0, 0.75, -0.5, 0, M, N, K)
    assert np.linalg.norm(out - ref) / np.linalg.norm(ref) < 1e-14


def test_gemm_k_zero(ctx):
    C0 = np.ones((20, 30))
    out = run(ctx, False, False, np.zeros((20, 1)), np.zeros((1, 30)), C0, 1.0, 2.0, 0, 20, 30, 0)
    np.testing.assert_array_equal(out, 2.0 * C0)


@pytest.mark.parametrize("q,K", [(200, 57), (385, 300), (100, 40), (128, 256)])
def test_gemm_sym_lower_mirror(ctx, q, K):
    rng = np.random.default_rng(q)
    A = rng.standard_normal((K, q))
    ref = A.T @ A
    out = run(ctx, True, False, A, A, np.zeros((q, q)), 1.0, 0.0, SYM_LOWER | SYM_MIRROR, q, q, K)
    np.testing.assert_array_equal(out, out.T)            # bit-identical triangles
    assert np.linalg.norm(out - ref) / np.linalg.norm(ref) < 1e-14
    C0 = np.full((q, q), 7.0)
    out2 = run(ctx, False, True, A.T.copy(), A.T.copy(), C0, -1.0, 1.0, SYM_LOWER, q, q, K)
    low = np.tril(np.ones((q, q), dtype=bool))
    np.testing.assert_allclose(out2[low], (7.0 - ref)[low], rtol=1e-13, atol=1e-12)
    np.testing.assert_array_equal(out2[~low], 7.0)       # upper triangle untouched


@pytest.mark.parametrize("q", [385, 200])
def test_gemm_sym_lower_mirror_lauum_flags(ctx, q):
    """The step's largest launch in miniature: Sigma = X^T X with X lower triangular (L^{-1}), the
    lauum flags A_KGE_M | B_KGE_N (triangular k-ranges) on the symmetric lower / mirror walk, at ragged
    q where the last square's right column half falls past N (q = 385: 4 squares, the last with one
    valid column)."""
    rng = np.random.default_rng(7 * q)
    X = np.tril(rng.standard_normal((q, q)))
    ref = X.T @ X
    out = run(ctx, True, False, X, X, np.zeros((q, q)), 1.0, 0.0, SYM_LOWER | SYM_MIRROR | A_KGE_M | B_KGE_N, q, q, q)
    np.testing.assert_array_equal(out, out.T)
    assert np.linalg.norm(out - ref) / np.linalg.norm(ref) < 1e-14


@pytest.mark.parametrize("n2,n1", [(385, 256), (200, 128), (130, 300), (64, 40)])
def test_gemm_mirror_block(ctx, n2, n1):
    """The off-diagonal piece of the interleaved Sigma assembly: S21 = X22^T X21 (X22 lower
    triangular: A_KGE_M) into one block and its transpose into the mirror block (mir1), bit-identical;
    ragged and sub-tile shapes on every kernel family."""
    from paper_1509_04681_b200.api import ld_of
    rng = np.random.default_rng(n2 * 3 + n1)
    X22 = np.tril(rng.standard_normal((n2, n2)))
    X21 = rng.standard_normal((n2, n1))
    ref = X22.T @ X21
    q = n1 + n2
    S = torch.full((q, q), 5.0, dtype=torch.float64, device="cuda").t()   # column-major, ld = q
    ldS = ld_of(S)
    dA, dB = dev(X22), dev(X21)
    base = S.data_ptr()
    st = ctx.lib.cggm_test_gemm_mir(ctx.h, 1, 0, n2, n1, n2, ctypes.c_void_p(dA.data_ptr()), ld_of(dA),
                                    ctypes.c_void_p(dB.data_ptr()), ld_of(dB), ctypes.c_void_p(base + 8 * n1), ldS,
                                    ctypes.c_void_p(base + 8 * n1 * ldS), 1.0, A_KGE_M)
    ctx._check(st)
    torch.cuda.synchronize()
    out = S.cpu().numpy()
    blk, mir = out[n1:, :n1], out[:n1, n1:]
    np.testing.assert_array_equal(blk, mir.T)
    assert np.linalg.norm(blk - ref) / np.linalg.norm(ref) < 1e-14
    np.testing.assert_array_equal(out[:n1, :n1], 5.0)     # diagonal blocks untouched
    np.testing.assert_array_equal(out[n1:, n1:], 5.0)


@pytest.mark.parametrize("q,K", [(385, 300), (200, 57), (256, 513)])
def test_gemm_sym_mirror_accumulate(ctx, q, K):
    """S11 += X21^T X21 in place on a full symmetric S11 (SYM_LOWER | SYM_MIRROR with the output as
    its own input): both triangles updated, bit-identical."""
    rng = np.random.default_rng(q + K)
    A = rng.standard_normal((K, q))
    S0 = rng.standard_normal((q, q))
    S0 = S0 + S0.T
    ref = S0 + A.T @ A
    out = run(ctx, True, False, A, A, S0, 1.0, 1.0, SYM_LOWER | SYM_MIRROR, q, q, K)
    np.testing.assert_array_equal(out, out.T)
    assert np.linalg.norm(out - ref) / np.linalg.norm(ref) < 1e-14


@pytest.mark.parametrize("flags", [A_KLE_M, A_KGE_M, B_KLE_N, B_KGE_N, A_KGE_M | B_KGE_N])
def test_gemm_triangular_k_range(ctx, flags):
    """Triangular operands with exact zeros outside the triangle: the shortened k-range must
    give the full product."""
    rng = np.random.default_rng(flags)
    n = 333 if flags != A_KLE_M else 120
    A = rng.standard_normal((n, n))
    B = rng.standard_normal((n, n))
    # op(A)[m][k] zero for k > m (A_KLE_M) etc.; no transposes here
    if flags & A_KLE_M:
        A = np.tril(A)
    if flags & A_KGE_M:
        A = np.triu(A)
    if flags & B_KLE_N:
        B = np.triu(B)
    if flags & B_KGE_N:
        B = np.tril(B)
    ref = A @ B
    out = run(ctx, False, False, A, B, np.zeros((n, n)), 1.0, 0.0, flags, n, n, n)
    assert np.linalg.norm(out - ref) / np.linalg.norm(ref) < 1e-14


def test_gemm_odd_leading_dimension_packs(ctx):
    """ld odd / unaligned views are packed before TMA."""
    from paper_1509_04681_b200.api import ld_of
    rng = np.random.default_rng(9)
    M, N, K = 77, 65, 43
    A = rng.standard_normal((M, K))
    B = rng.standard_normal((K, N))
    base = torch.from_numpy(np.asfortranarray(np.vstack([A, np.zeros((2, K))]))).cuda()  # ld = M + 2 (odd)
    baseA = torch.zeros((K, M + 2), dtype=torch.float64, device="cuda")
    baseA.copy_(torch.from_numpy(np.vstack([A, np.zeros((2, K))]).T.copy()))
    dA = baseA.t()[1:M + 1]            # offset by one element: unaligned base, ld = M + 2 = 79
    baseA.t()[1:M + 1].copy_(torch.from_numpy(A))
    dB = dev(B)
    dC = dev(np.zeros((M, N)))
    st = ctx.lib.cggm_test_gemm(ctx.h, 0, 0, M, N, K, ctypes.c_void_p(dA.data_ptr()), ld_of(dA),
                                ctypes.c_void_p(dB.data_ptr()), ld_of(dB), ctypes.c_void_p(dC.data_ptr()), ld_of(dC),
                                1.0, 0.0, 0)
    ctx._check(st)
    out = dC.cpu().numpy()
    ref = A @ B
    assert np.linalg.norm(out - ref) / np.linalg.norm(ref) < 1e-14
    del base


def test_gemm_lower_trapezoid(ctx):
    """SYM_LOWER with M > N: lower triangle of the square part plus the full rows below
    (the Cholesky trailing update of the augmented [Lambda; W] factor)."""
    rng = np.random.default_rng(21)
    N, extra, K = 300, 257, 140
    M = N + extra
    A = rng.standard_normal((M, K))
    C0 = rng.standard_normal((M, N))
    out = run(ctx, False, True, A, A[:N].copy(), C0, -1.0, 1.0, SYM_LOWER, M, N, K)
    ref = C0 - A @ A[:N].T
    mask = np.tril(np.ones((M, N), dtype=bool))
    np.testing.assert_allclose(out[mask], ref[mask], rtol=1e-12, atol=1e-12)
    np.testing.assert_array_equal(out[~mask], C0[~mask])


@pytest.mark.parametrize("flags", [1, 2, 4, 8, 10])
def test_gemm_small_triangular(ctx, flags):
    """Small-shape path (K <= 256): triangular k-ranges on 32-wide tiles."""
    rng = np.random.default_rng(100 + flags)
    n = 120
    A = rng.standard_normal((n, n))
    B = rng.standard_normal((n, n))
    A = np.tril(A) if flags & 1 else np.triu(A) if flags & 2 else A
    B = np.triu(B) if flags & 4 else np.tril(B) if flags & 8 else B
    out = run(ctx, False, False, A, B, np.zeros((n, n)), 1.0, 0.0, flags, n, n, n)
    assert np.linalg.norm(out - A @ B) / np.linalg.norm(A @ B) < 1e-14


def test_gemm_small_trapezoid_inplace_update(ctx):
    """C -= A A^T over the lower trapezoid with C also the epilogue input (Cholesky update)."""
    rng = np.random.default_rng(77)
    N, extra, K = 64, 1000, 64
    A = rng.standard_normal((N + extra, K))
    C0 = rng.standard_normal((N + extra, N))
    out = run(ctx, False, True, A, A[:N].copy(), C0, -1.0, 1.0, SYM_LOWER, N + extra, N, K)
    mask = np.tril(np.ones((N + extra, N), dtype=bool))
    ref = C0 - A @ A[:N].T
    np.testing.assert_allclose(out[mask], ref[mask], rtol=1e-12, atol=1e-12)
    np.testing.assert_array_equal(out[~mask], C0[~mask])


@pytest.fixture(scope="module", params=[2, 3], ids=["persist2", "persist3"])
def pctx(request):
    """The persistent warp-specialised 128x128 kernel (CGGM_PERSIST_TPC): engaged for grids of at
    least two tiles per SM, so the shapes below span >= 296 tiles with ragged edges."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import os
    from paper_1509_04681_b200 import Context
    os.environ["CGGM_PERSIST_TPC"] = str(request.param)
    os.environ["CGGM_MID_TILE"] = "0"   # the persistent kernel is the 128x128 configuration
    try:
        c = Context(0)
    finally:
        os.environ.pop("CGGM_PERSIST_TPC", None)
        os.environ.pop("CGGM_MID_TILE", None)
    c._check(c.lib.cggm_test_set_tile(c.h, 1))
    return c


@pytest.mark.parametrize("tA", [False, True])
@pytest.mark.parametrize("tB", [False, True])
@pytest.mark.parametrize("M,N,K", [(2600, 2410, 100), (4100, 1290, 37)])
def test_gemm_persistent(pctx, tA, tB, M, N, K):
    rng = np.random.default_rng(M + N + K)
    A = rng.standard_normal((K, M) if tA else (M, K))
    B = rng.standard_normal((N, K) if tB else (K, N))
    C0 = rng.standard_normal((M, N))
    ref = 1.5 * ((A.T if tA else A) @ (B.T if tB else B)) + 0.25 * C0
    out = run(pctx, tA, tB, A, B, C0, 1.5, 0.25, 0, M, N, K)
    assert np.linalg.norm(out - ref) / np.linalg.norm(ref) < 1e-14


@pytest.mark.parametrize("flags", [SYM_LOWER | SYM_MIRROR, SYM_LOWER, B_KLE_N])
def test_gemm_persistent_structured(pctx, flags):
    q, K = 2500, 2500 if flags == B_KLE_N else 90
    rng = np.random.default_rng(flags)
    A = rng.standard_normal((q, K))
    if flags == B_KLE_N:
        B = np.triu(rng.standard_normal((K, q)))   # B[k][n] = 0 for k > n: B_KLE_N shortens the k-range
        ref = A @ B
        out = run(pctx, False, False, A, B, np.zeros((q, q)), 1.0, 0.0, flags, q, q, K)
        assert np.linalg.norm(out - ref) / np.linalg.norm(ref) < 1e-14
        return
    ref = A @ A.T
    out = run(pctx, False, True, A, A, np.zeros((q, q)), 1.0, 0.0, flags, q, q, K)
    lo = np.tril_indices(q)
    assert np.linalg.norm(out[lo] - ref[lo]) / np.linalg.norm(ref[lo]) < 1e-14
    if flags & SYM_MIRROR:
        np.testing.assert_array_equal(out, out.T)
