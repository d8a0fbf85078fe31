"""GPU: seeded random shapes, dtypes and fallback rates through the quantizer
and the fallback GEMM, against the CPU oracle -- the ragged / odd corners the
hand-picked parity shapes do not reach (rows and columns straddling block and
vector boundaries, tiny and single-block tensors, many-tile grids).  Integer
outputs bit-exact; the GEMM bit-exact in EXACT mode, within FMA_TOL in FMA mode."""
import numpy as np
import pytest

from tests.helpers import bf16_round, outlier_matrix, rel_fro

pytestmark = pytest.mark.gpu

FMA_TOL = 1e-5
_RNG = np.random.default_rng(20261017)
QUANT_CASES = [(int(_RNG.integers(1, 700)), int(_RNG.integers(1, 1300)), ["f32", "bf16"][i % 2],
                float(_RNG.choice([0.0, 0.05, 0.2, 0.5]))) for i in range(16)]
GEMM_CASES = [(int(_RNG.integers(1, 600)), int(_RNG.integers(1, 800)), int(_RNG.integers(1, 900)),
               float(_RNG.choice([0.0, 0.1, 0.3]))) for _ in range(10)]


def _dev(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


@pytest.mark.parametrize("rows,cols,dtype,rate", QUANT_CASES)
def test_fuzz_fallback_quantize(orc, rows, cols, dtype, rate):
    """threshold mode at a theta realising ~rate: codes, scales, mask, residual
    codes / scales of flagged blocks bit-exact."""
    import torch
    from paper_2503_08040_b200 import fbq
    x = outlier_matrix(rows, cols, seed=rows * 7 + cols, channels=[cols // 2], tokens=[rows // 3],
                       mag_c=30.0, mag_t=20.0, occasional=3)
    if dtype == "bf16":
        x = bf16_round(x)
    xt = _dev(x).to(torch.bfloat16) if dtype == "bf16" else _dev(x)
    scores = orc.score_blocks_absmax(x)
    theta, _ = fbq.theta_for_rate(scores, rate)
    theta = max(theta, 1e-30)
    fa = fbq.fallback_quantize(xt, theta=theta)
    mask = orc.mask_threshold(scores, theta)
    codes, scales, rcodes, rscales = orc.fallback_quantize(x, mask)
    assert np.array_equal(fa.mask.cpu().numpy(), mask)
    assert np.array_equal(fa.primary.codes_int16().cpu().numpy(), codes)
    assert np.array_equal(fa.primary.scales.cpu().numpy().view(np.int32), scales.view(np.int32))
    got_rs = fa.res_scales.cpu().numpy()
    assert np.array_equal(got_rs.view(np.int32), rscales.view(np.int32))
    gr = fa.res_codes.cpu().numpy()[:, :cols].astype(np.int16)
    for bi, bj in zip(*np.nonzero(mask)):
        r0, c0 = bi * 128, bj * 128
        assert np.array_equal(gr[r0:r0 + 128, c0:c0 + 128], rcodes[r0:r0 + 128, c0:c0 + 128]), (bi, bj)


@pytest.mark.parametrize("m,n,k,rate", GEMM_CASES)
def test_fuzz_fallback_gemm(orc, m, n, k, rate):
    """Y = fallback_gemm(fq(X), q(W)^T) at random sizes: EXACT bit for bit, FMA
    within tolerance, both against the oracle's run_block_gemm."""
    from paper_2503_08040_b200 import fbq
    a = outlier_matrix(m, k, seed=m + 3 * n + 7 * k, channels=[k // 2], tokens=[m // 2])
    w = outlier_matrix(n, k, seed=m * 5 + k, body=0.02)
    mask = orc.mask_topk(orc.score_blocks_absmax(a), rate)
    fa = fbq.fallback_quantize(_dev(a), _dev(mask))
    wq = fbq.transpose(fbq.quantize_rtn(_dev(w)))
    ac, as_, rc, rs = orc.fallback_quantize(a, mask)
    wc, ws = orc.quantize_rtn(w)
    bc, bs = orc.transpose_qt(wc, ws)
    want = orc.block_gemm(ac, as_, bc, bs, mask=mask, res_codes=rc, res_scales=rs)
    got = fbq.fallback_gemm(fa, wq).cpu().numpy()
    assert np.array_equal(got.view(np.int32), want.view(np.int32)), rel_fro(got, want)
    got_fma = fbq.fallback_gemm(fa, wq, exact=False).cpu().numpy()
    assert rel_fro(got_fma, want) <= FMA_TOL
