"""Sigma = L^{-T} L^{-1} assembled inside the recursive inverse (CGGM_OPT_SIGMA_BLOCK,
chol.cu sig_node_pieces): every node at least sig_block wide forms X22^T X21 (and its mirrored
copy) and X21^T X21 into its leading block once its own L^{-1} is final; narrower nodes form
their block in one product.  Checked against the P4 chain closed form, the oracle, and the
one-product path (same sums in a different k-split: rounding-level differences only), at block
sizes that put several recursion levels and ragged splits on the new path."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import cggm_oracle as O  # noqa: E402
from synth.cggm_inputs import csc_from_dense, make_problem  # noqa: E402


def relf(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1509_04681_b200 import Context
    return Context(0)


def set_block(ctx, v, lookahead=256):
    from paper_1509_04681_b200 import _abi
    ctx.set_option(_abi.CGGM_OPT_SIGMA_BLOCK, v)
    ctx.set_option(_abi.CGGM_OPT_LOOKAHEAD_MIN, lookahead)


@pytest.fixture(autouse=True)
def restore(ctx):
    yield
    set_block(ctx, 4096)


def test_option_bounds(ctx):
    from paper_1509_04681_b200 import _abi
    from paper_1509_04681_b200.api import CggmError
    for bad in (1, 64, 127, -5):
        with pytest.raises(CggmError):
            ctx.set_option(_abi.CGGM_OPT_SIGMA_BLOCK, bad)
    ctx.set_option(_abi.CGGM_OPT_SIGMA_BLOCK, 0)
    ctx.set_option(_abi.CGGM_OPT_SIGMA_BLOCK, 128)


@pytest.mark.parametrize("q", [700, 2500])
@pytest.mark.parametrize("block,lookahead", [(128, 256), (256, 256), (1024, 256), (128, 0)])
def test_chain_closed_form(ctx, q, block, lookahead):
    """P3 / P4 (chain log-det and Sigma closed forms) with the Sigma blocks formed in the recursion,
    with the lookahead streams and inline on one stream (lookahead 0)."""
    from paper_1509_04681_b200 import DeviceCsc
    from tests.test_oracle_pins import chain_dense, chain_sigma_closed_form
    set_block(ctx, block, lookahead)
    Sg, ld, pd, fc = ctx.cggm_invert_logdet(DeviceCsc.from_host(csc_from_dense(chain_dense(q))))
    assert pd and fc == -1
    assert ld == pytest.approx(math.log((1 - 0.5 ** (2 * q + 2)) / 0.75), rel=1e-12)
    S = Sg.cpu().numpy()
    np.testing.assert_array_equal(S, S.T)          # both triangles bit-identical (reading A19)
    assert relf(S, chain_sigma_closed_form(q)) <= 1e-12


@pytest.mark.parametrize("name,k", [("small", 1), ("medium", 0)])
@pytest.mark.parametrize("block", [128, 512])
def test_random_spd_against_oracle_and_one_product(ctx, name, k, block):
    from paper_1509_04681_b200 import DeviceCsc
    P = make_problem(name)
    label, lam, th = P.points[k]
    Lg = DeviceCsc.from_host(lam)
    set_block(ctx, 0)
    S0, ld0, pd0, _ = ctx.cggm_invert_logdet(Lg)
    set_block(ctx, block)
    S1, ld1, pd1, _ = ctx.cggm_invert_logdet(Lg)
    assert pd0 and pd1 and ld0 == ld1                 # the factorisation itself is unchanged
    a, b = S0.cpu().numpy(), S1.cpu().numpy()
    np.testing.assert_array_equal(b, b.T)
    assert relf(b, a) <= 1e-13                         # k-split order only
    if name == "small":
        Sig_o, ld_o, ok_o, _ = O.invert_logdet(lam.to_dense())
        assert relf(b, Sig_o) <= 1e-9
    # P7: Lambda Sigma = I
    Ld = torch.from_numpy(lam.to_dense()).cuda()
    I = torch.eye(P.q, dtype=torch.float64, device="cuda")
    assert float(torch.linalg.norm(Ld @ S1 - I)) / math.sqrt(P.q) <= 1e-12


def test_composite_evaluation_bit_identical_to_separate_calls(ctx):
    """cggm_newton_eval (graph capture on the second call) with the interleaved Sigma gives the
    separate calls' results bit for bit, and the oracle's within the contract tolerances."""
    from paper_1509_04681_b200 import DeviceCsc, to_device_colmajor
    from paper_1509_04681_b200.api import newton_evaluation
    set_block(ctx, 256)
    P = make_problem("small")
    label, lam, th = P.points[1]
    X, Y = to_device_colmajor(P.X), to_device_colmajor(P.Y)
    Lg, Tg = DeviceCsc.from_host(lam), DeviceCsc.from_host(th)
    Syy, _ = ctx.cggm_covariances(X, Y, want_sxy=False)
    cap = 1_000_000

    def bufs():
        return {k2: torch.empty(cap, dtype=torch.int32, device="cuda") for k2 in ("L_row", "L_col", "T_row", "T_col")}

    a = newton_evaluation(ctx, X, Y, Syy, Lg, Tg, P.lam_L, P.lam_T, True, bufs(), composite=False)
    outs = [newton_evaluation(ctx, X, Y, Syy, Lg, Tg, P.lam_L, P.lam_T, True, bufs(), composite=True)
            for _ in range(3)]   # eager, capture, replay
    for b in outs:
        for key in ("Sigma", "Psi", "GradL", "GradT"):
            assert torch.equal(a[key], b[key]), key
        assert a["objective"]["f"] == b["objective"]["f"]
    Sig_o, _, _, _ = O.invert_logdet(lam.to_dense())
    assert relf(outs[-1]["Sigma"].cpu().numpy(), Sig_o) <= 1e-9


def test_non_pd_reported_with_interleaved_sigma(ctx):
    """A non-PD Lambda still reports is_pd = 0 and the failing column (P5) on this path."""
    from paper_1509_04681_b200 import DeviceCsc
    from tests.test_oracle_pins import chain_dense
    set_block(ctx, 128)
    q = 700
    A = chain_dense(q)
    lmin = 1.25 - math.cos(math.pi / (q + 1))
    Sg, ld, pd, fc = ctx.cggm_invert_logdet(DeviceCsc.from_host(csc_from_dense(A - (1 + 1e-6) * lmin * np.eye(q))))
    assert not pd and 0 <= fc < q


@pytest.mark.parametrize("block", [128, 512])
def test_fp32_variant_interleaved_sigma(block):
    """The FP32 variant (3xTF32 / FFMA engines with the mirrored off-diagonal epilogue): the P4 chain
    closed form within the FP32 contract (rel-F 1e-4) and the one-product FP32 Sigma to fp32 rounding."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1509_04681_b200 import Context, DeviceCsc, _abi
    from tests.test_oracle_pins import chain_dense, chain_sigma_closed_form
    c = Context(0, dtype="f32")
    q = 2500
    L = DeviceCsc.from_host(csc_from_dense(chain_dense(q)), dtype=torch.float32)
    c.set_option(_abi.CGGM_OPT_SIGMA_BLOCK, 0)
    S0 = c.cggm_invert_logdet(L)[0].double().cpu().numpy()
    c.set_option(_abi.CGGM_OPT_SIGMA_BLOCK, block)
    S1, ld, pd, fc = c.cggm_invert_logdet(L)
    S1 = S1.double().cpu().numpy()
    assert pd
    np.testing.assert_array_equal(S1, S1.T)
    assert relf(S1, chain_sigma_closed_form(q)) <= 1e-4
    assert relf(S1, S0) <= 1e-5


@pytest.mark.parametrize("q,ld_extra", [(700, 1), (4097, 3)])
def test_odd_leading_dimension_and_just_above_block(ctx, q, ld_extra):
    """Sigma into a caller buffer with an odd leading dimension (the mirrored epilogue's scalar path)
    and q just above the default block size (root split, one-product children): P4 closed form."""
    from paper_1509_04681_b200 import DeviceCsc
    from tests.test_oracle_pins import chain_dense, chain_sigma_closed_form
    set_block(ctx, 128 if q < 1000 else 4096)
    base = torch.full((q, q + ld_extra), -7.0, dtype=torch.float64, device="cuda")   # ld = q + ld_extra
    Sg = base.t()[:q, :q]
    S, ld, pd, fc = ctx.cggm_invert_logdet(DeviceCsc.from_host(csc_from_dense(chain_dense(q))), Sigma=Sg)
    assert pd
    out = S.cpu().numpy()
    np.testing.assert_array_equal(out, out.T)
    assert relf(out, chain_sigma_closed_form(q)) <= 1e-12
    np.testing.assert_array_equal(base.t()[q:, :].cpu().numpy(), -7.0)   # padding rows untouched
