"""GPU parity: the sm_100a kernels (through the C ABI) vs the CPU oracle.

Integer outputs (codes, scales, masks, residuals, per-block int32 products)
must be bit-exact; the GEMM's fp32 output is bit-exact in EXACT epilogue
mode and within 1e-5 relative Frobenius (SPEC.md gemm module) in FMA mode.
"""
import numpy as np
import pytest

from tests.helpers import bf16_round, outlier_matrix, rel_fro

pytestmark = pytest.mark.gpu

FMA_TOL = 1e-5  # SPEC.md:240,268 relative Frobenius bound


@pytest.fixture(scope="module")
def F():
    import torch  # noqa: F401
    from paper_2503_08040_b200 import fbq
    return fbq


def dev(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def host(t):
    return t.detach().cpu().numpy()


SHAPES = [(128, 128), (256, 384), (300, 270), (1, 7), (13, 129), (640, 1152)]


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_quantize_rtn(F, orc, shape, dtype):
    import torch
    x = outlier_matrix(*shape, seed=hash(shape) % 1000, channels=[min(3, shape[1] - 1)])
    if dtype == "bf16":
        x = bf16_round(x)
        xt = dev(x).to(torch.bfloat16)
    else:
        xt = dev(x)
    q = F.quantize_rtn(xt)
    codes, scales = orc.quantize_rtn(x)
    assert np.array_equal(host(q.codes_int16()), codes)
    assert np.array_equal(host(q.scales).view(np.int32), scales.view(np.int32))


@pytest.mark.parametrize("shape", SHAPES)
def test_fallback_quantize_threshold(F, orc, shape):
    x = outlier_matrix(*shape, seed=7, channels=[0], tokens=[min(5, shape[0] - 1)], occasional=5)
    scores = orc.score_blocks_absmax(x)
    theta = float(np.median(scores)) if scores.size > 1 else 1.0
    fa = F.fallback_quantize(dev(x), theta=theta)
    mask = orc.mask_threshold(scores, theta)
    codes, scales, rcodes, rscales = orc.fallback_quantize(x, mask)
    assert np.array_equal(host(fa.mask), mask)
    assert int(fa.masked_count.item()) == int(mask.sum())
    assert np.array_equal(host(fa.primary.codes_int16()), codes)
    assert np.array_equal(host(fa.primary.scales).view(np.int32), scales.view(np.int32))
    got_rs = host(fa.res_scales)
    assert np.array_equal(got_rs.view(np.int32), rscales.view(np.int32))
    r, c = shape
    got_rc = host(fa.res_codes[:r, :c]).astype(np.int16)
    for bi, bj in zip(*np.nonzero(mask)):
        sl = (slice(bi * 128, bi * 128 + 128), slice(bj * 128, bj * 128 + 128))
        assert np.array_equal(got_rc[sl], rcodes[sl])
    # scores
    assert np.array_equal(host(F.score_blocks(dev(x))), scores)


@pytest.mark.parametrize("shape", [(300, 270), (640, 1152), (8192, 512)])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_threshold_mask_needs_no_zeroing(F, orc, shape, dtype):
    """THRESHOLD mode writes every bitmap bit (tail bits of the last word
    cleared) and zeroes the count in-stream: dirty buffers give the oracle's
    mask, and back-to-back calls on the same buffers agree."""
    import torch
    from paper_2503_08040_b200 import _capi as K
    x = outlier_matrix(*shape, seed=11, channels=[1], tokens=[min(9, shape[0] - 1)], occasional=7)
    if dtype == "bf16":
        x = bf16_round(x)
    xt = dev(x).to(torch.bfloat16) if dtype == "bf16" else dev(x)
    scores = orc.score_blocks_absmax(x)
    theta = float(np.median(scores))
    mask = orc.mask_threshold(scores, theta)
    r, c = shape
    nb = mask.size
    words = (nb + 31) // 32
    bits = torch.full((words,), -1, dtype=torch.int32, device="cuda")
    count = torch.full((1,), 12345, dtype=torch.int32, device="cuda")
    codes = torch.empty((r, (c + 15) // 16 * 16), dtype=torch.int8, device="cuda")
    res = torch.empty_like(codes)
    sc = torch.empty(nb, dtype=torch.float32, device="cuda")
    rsc = torch.empty_like(sc)
    stream = torch.cuda.current_stream().cuda_stream
    for _ in range(2):
        K.call("fbq_cuda_quantize_fallback", xt.data_ptr(), K.FBQ_BF16 if dtype == "bf16" else K.FBQ_F32,
               r, c, c, K.FBQ_MASK_THRESHOLD, theta, bits.data_ptr(), codes.data_ptr(), codes.stride(0),
               sc.data_ptr(), res.data_ptr(), rsc.data_ptr(), count.data_ptr(), None, None, 0, 0, stream)
        torch.cuda.synchronize()
        want = np.zeros(words * 32, dtype=np.uint8)
        want[:nb] = mask.reshape(-1)
        want_words = (want.reshape(-1, 32).astype(np.uint64) << np.arange(32, dtype=np.uint64)).sum(1)
        got = host(bits).view(np.uint32)
        assert np.array_equal(got, want_words.astype(np.uint32))
        assert int(count.item()) == int(mask.sum())


def test_fallback_quantize_given_mask(F, orc):
    x = outlier_matrix(512, 384, seed=3, channels=[10, 200], occasional=20)
    scores = orc.score_blocks_absmax(x)
    mask = orc.mask_topk(scores, 0.2)
    fa = F.fallback_quantize(dev(x), dev(mask))
    codes, scales, rcodes, rscales = orc.fallback_quantize(x, mask)
    assert np.array_equal(host(fa.mask), mask)
    assert np.array_equal(host(fa.res_scales).view(np.int32), rscales.view(np.int32))
    got = host(fa.res_codes[:512, :384]).astype(np.int16)
    m = np.kron(mask, np.ones((128, 128), np.uint8)).astype(bool)
    assert np.array_equal(got[m], rcodes[m])


@pytest.mark.parametrize("shape,row_offset", [((256, 384), 0), ((300, 270), 0), ((256, 256), 384)])
def test_quantize_stochastic(F, orc, shape, row_offset):
    x = outlier_matrix(*shape, seed=11, channels=[1])
    seed = F.layer_seed(0x5EED, 3, 1, 17)
    q = F.quantize_stochastic(dev(x), seed, row_offset=row_offset)
    codes, scales = orc.quantize_stochastic(x, seed, row_offset=row_offset)
    assert np.array_equal(host(q.codes_int16()), codes)
    assert np.array_equal(host(q.scales).view(np.int32), scales.view(np.int32))


def test_fused_forward_context(F, orc):
    """One pass produces RTN+fallback codes and the SR context (trainsim.cpp:95-102)."""
    x = outlier_matrix(384, 512, seed=5, channels=[7], tokens=[100])
    seed = F.layer_seed(0x5EED, 0, 0, 3)
    fa, ctx = F.fallback_quantize(dev(x), theta=20.0, sr_seed=seed)
    codes, scales = orc.quantize_stochastic(x, seed)
    assert np.array_equal(host(ctx.codes_int16()), codes)
    mask = orc.mask_threshold(orc.score_blocks_absmax(x), 20.0)
    assert np.array_equal(host(fa.mask), mask)


def _quant_pair(orc, m, n, k, seed=0, rate=0.2):
    a = outlier_matrix(m, k, seed=seed, channels=[min(2, k - 1)], tokens=[min(9, m - 1)])
    b = outlier_matrix(k, n, seed=seed + 1, body=0.02)
    scores = orc.score_blocks_absmax(a)
    mask = orc.mask_topk(scores, rate)
    return a, b, mask


GEMM_SHAPES = [(128, 256, 128), (256, 512, 384), (200, 300, 260), (384, 128, 640), (64, 40, 16)]


@pytest.mark.parametrize("mnk", GEMM_SHAPES)
@pytest.mark.parametrize("fallback", [False, True])
def test_gemm_forward_exact(F, orc, mnk, fallback):
    """Y = X W^T: A K-major (X codes), B K-major (W codes, N x K)."""
    m, n, k = mnk
    a, b, mask = _quant_pair(orc, m, n, k)
    w = np.ascontiguousarray(b.T)  # N x K weight, as QuantLinearLayer stores it
    wq = F.quantize_rtn(dev(w))
    wc, ws = orc.quantize_rtn(w)
    bc, bs = orc.transpose_qt(wc, ws)  # reference's quantize_rtn(transpose(W))
    if fallback:
        fa = F.fallback_quantize(dev(a), dev(mask))
        y = F.fallback_gemm(fa, F.transpose(wq))
        ac, as_, rc, rs = orc.fallback_quantize(a, mask)
        want = orc.block_gemm(ac, as_, bc, bs, mask=mask, res_codes=rc, res_scales=rs)
    else:
        qa = F.quantize_rtn(dev(a))
        y = F.block_quant_gemm(qa, F.transpose(wq))
        ac, as_ = orc.quantize_rtn(a)
        want = orc.block_gemm(ac, as_, bc, bs)
    got = host(y)
    assert np.array_equal(got.view(np.int32), want.view(np.int32))


@pytest.mark.parametrize("mnk", GEMM_SHAPES)
def test_gemm_fma_mode(F, orc, mnk):
    m, n, k = mnk
    a, b, mask = _quant_pair(orc, m, n, k, seed=4)
    fa = F.fallback_quantize(dev(a), dev(mask))
    qb = F.quantize_rtn(dev(b))  # K x N: MN-major B (reference orientation)
    y = F.fallback_gemm(fa, qb, exact=False)
    ac, as_, rc, rs = orc.fallback_quantize(a, mask)
    bc, bs = orc.quantize_rtn(b)
    want = orc.block_gemm(ac, as_, bc, bs, mask=mask, res_codes=rc, res_scales=rs)
    assert rel_fro(host(y), want) <= FMA_TOL


@pytest.mark.parametrize("mnk", GEMM_SHAPES)
def test_gemm_backward_layouts(F, orc, mnk):
    """dX = dY W (A K-major, B MN-major) and dW = dY^T X (A MN-major, B MN-major)."""
    t, n_out, k_in = mnk
    gy = outlier_matrix(t, n_out, seed=21, body=1e-3, tokens=[0])
    x = outlier_matrix(t, k_in, seed=22)
    w = outlier_matrix(n_out, k_in, seed=23, body=0.02)
    seed = F.layer_seed(0x5EED, 1, 1, 0)
    gyq = F.quantize_stochastic(dev(gy), seed)
    wq = F.quantize_rtn(dev(w))
    ctx = F.quantize_stochastic(dev(x), F.layer_seed(0x5EED, 1, 0, 0))
    dx = F.block_quant_gemm(gyq, wq)
    dw = F.block_quant_gemm(F.transpose(gyq), ctx)
    gc, gs = orc.quantize_stochastic(gy, seed)
    wc, ws = orc.quantize_rtn(w)
    xc, xs = orc.quantize_stochastic(x, F.layer_seed(0x5EED, 1, 0, 0))
    want_dx = orc.block_gemm(gc, gs, wc, ws)
    gtc, gts = orc.transpose_qt(gc, gs)
    want_dw = orc.block_gemm(gtc, gts, xc, xs)
    assert np.array_equal(host(dx).view(np.int32), want_dx.view(np.int32))
    assert np.array_equal(host(dw).view(np.int32), want_dw.view(np.int32))


@pytest.mark.parametrize("mnk", [(256, 256, 384), (200, 300, 260)])
def test_block_products_bit_exact(F, orc, mnk):
    m, n, k = mnk
    a, b, mask = _quant_pair(orc, m, n, k, seed=9, rate=0.3)
    fa = F.fallback_quantize(dev(a), dev(mask))
    wq = F.quantize_rtn(dev(np.ascontiguousarray(b.T)))
    prim, res = F.block_products(fa.primary, F.transpose(wq), fa)
    ac, as_, rc, rs = orc.fallback_quantize(a, mask)
    bc, _ = orc.quantize_rtn(b)
    want = orc.block_products(ac, bc)
    assert np.array_equal(host(prim), want)
    want_r = orc.block_products(rc, bc)
    got_r = host(res)
    for bi, bk in zip(*np.nonzero(mask)):
        assert np.array_equal(got_r[bi, :, bk], want_r[bi, :, bk])


def test_gemm_accumulate_and_bf16(F, orc):
    import torch
    m, n, k = 256, 256, 256
    a, b, _ = _quant_pair(orc, m, n, k, seed=31)
    qa, qb = F.quantize_rtn(dev(a)), F.quantize_rtn(dev(b))
    base = torch.randn(m, n, device="cuda")
    out = base.clone()
    F.block_quant_gemm(qa, qb, out=out, accumulate=True)
    ac, as_ = orc.quantize_rtn(a)
    bc, bs = orc.quantize_rtn(b)
    want = orc.block_gemm(ac, as_, bc, bs)
    exp = (host(base) + want).astype(np.float32)
    assert np.array_equal(host(out).view(np.int32), exp.view(np.int32))
    y16 = F.block_quant_gemm(qa, qb, out_dtype=torch.bfloat16)
    assert np.array_equal(host(y16.float()), bf16_round(want))


def test_dequantize(F, orc):
    x = outlier_matrix(300, 270, seed=2, channels=[4])
    mask = orc.mask_topk(orc.score_blocks_absmax(x), 0.5)
    fa = F.fallback_quantize(dev(x), dev(mask))
    c, s, rc, rs = orc.fallback_quantize(x, mask)
    assert np.array_equal(host(F.dequantize(fa.primary)), orc.dequantize(c, s))
    want = orc.dequantize_fallback(c, s, mask, rc, rs)
    assert np.array_equal(host(F.dequantize_fallback(fa)).view(np.int32), want.view(np.int32))


def test_gemm_many_tiles_odd_pairs(F, orc):
    """Persistent CTA-pair schedule: several pair tiles per cluster, an odd
    number of block rows (the last pair's second CTA is out of range), two
    scale pages along K, fallback blocks on both CTAs of a pair and on one."""
    m, n, k = 1152, 640, 4608
    a, b, mask = _quant_pair(orc, m, n, k, seed=41, rate=0.15)
    w = np.ascontiguousarray(b.T)
    wq = F.quantize_rtn(dev(w))
    wc, ws = orc.quantize_rtn(w)
    bc, bs = orc.transpose_qt(wc, ws)
    fa = F.fallback_quantize(dev(a), dev(mask))
    y = F.fallback_gemm(fa, F.transpose(wq))
    ac, as_, rc, rs = orc.fallback_quantize(a, mask)
    want = orc.block_gemm(ac, as_, bc, bs, mask=mask, res_codes=rc, res_scales=rs)
    assert np.array_equal(host(y).view(np.int32), want.view(np.int32))
    y2 = F.fallback_gemm(fa, F.transpose(wq), exact=False)
    assert rel_fro(host(y2), want) <= FMA_TOL


@pytest.mark.parametrize("raster", [1 << 17, 1 << 18, 1 << 19, 1 << 20])
def test_gemm_tile_rasters(F, orc, raster):
    """Every tile rasterisation the launcher may pick (kGroupM groups, bm over
    all block-rows, bn fastest) covers each tile exactly once: bit-exact on a
    ragged multi-wave shape with fallback blocks, plain and accumulating."""
    lib = F.K.lib
    lib.fbq_debug_set_gemm_diag.argtypes = [F.K.cint]
    m, n, k = 2200, 1400, 520
    a, b, mask = _quant_pair(orc, m, n, k, seed=43, rate=0.2)
    w = np.ascontiguousarray(b.T)
    wq = F.quantize_rtn(dev(w))
    wc, ws = orc.quantize_rtn(w)
    bc, bs = orc.transpose_qt(wc, ws)
    fa = F.fallback_quantize(dev(a), dev(mask))
    ac, as_, rc, rs = orc.fallback_quantize(a, mask)
    want = orc.block_gemm(ac, as_, bc, bs, mask=mask, res_codes=rc, res_scales=rs)
    try:
        lib.fbq_debug_set_gemm_diag(raster)
        y = F.fallback_gemm(fa, F.transpose(wq))
        assert np.array_equal(host(y).view(np.int32), want.view(np.int32))
        y2 = F.fallback_gemm(fa, F.transpose(wq), exact=False)
        assert rel_fro(host(y2), want) <= FMA_TOL
    finally:
        lib.fbq_debug_set_gemm_diag(0)


@pytest.mark.parametrize("rate", [0.0, 1e-4, 0.05, 0.2, 0.5, 1.0])
def test_mask_topk_device_matches_reference(F, orc, rate):
    """mask_topk (policy.cpp:56-71) on the device: exactly ceil(rate*n) blocks,
    ties toward the lower index -- on AbsMax scores and on a tie-heavy grid."""
    import torch
    x = outlier_matrix(1280, 1664, seed=50, channels=[3, 900], tokens=[77])
    scores = orc.score_blocks_absmax(x)
    got = host(F.mask_topk(F.score_blocks(dev(x)), rate))
    assert np.array_equal(got, orc.mask_topk(scores, rate))
    # many exact ties: scores from a handful of values
    rng = np.random.default_rng(int(rate * 1000) + 1)
    tied = rng.choice(np.array([0.0, 0.5, 1.0, 2.0], np.float32), size=(37, 91)).astype(np.float64)
    got = host(F.mask_topk(torch.from_numpy(tied).cuda(), rate))
    assert np.array_equal(got, orc.mask_topk(tied, rate))


@pytest.mark.parametrize("rate", [0.0, 0.2])
def test_quantizer_dynamic_block_schedule(F, orc, rate):
    """The persistent bf16 K1 claims blocks from a self-resetting counter: its
    codes, scales, mask and residuals equal the static schedule's (diag 4096)
    and the oracle's, launch after launch (the counter slot is reused)."""
    import torch
    lib = F.K.lib
    lib.fbq_debug_set_quant_diag.argtypes = [F.K.cint]
    x = bf16_round(outlier_matrix(2100, 3000, seed=17, channels=[5, 1300], tokens=[7], occasional=40))
    xt = dev(x).to(torch.bfloat16)
    scores = orc.score_blocks_absmax(x)
    mask = orc.mask_topk(scores, rate) if rate > 0 else np.zeros_like(scores, dtype=np.uint8)
    c, s, rc, rs = orc.fallback_quantize(x, mask)
    outs = []
    try:
        for d in (0, 4096, 0, 0):
            lib.fbq_debug_set_quant_diag(d)
            fa = F.fallback_quantize(xt, dev(mask))
            outs.append(fa)
    finally:
        lib.fbq_debug_set_quant_diag(0)
    for fa in outs:
        assert np.array_equal(host(fa.primary.codes_int16()), c)
        assert np.array_equal(host(fa.primary.scales).view(np.int32), s.view(np.int32))
        for bi, bj in zip(*np.nonzero(mask)):
            r0, c0 = bi * 128, bj * 128
            got = host(fa.res_codes[r0:r0 + 128, c0:min(c0 + 128, x.shape[1])].to(torch.int16))
            assert np.array_equal(got, rc[r0:r0 + 128, c0:c0 + 128])
        assert np.array_equal(host(fa.res_scales)[mask.astype(bool)].view(np.int32),
                              rs[mask.astype(bool)].view(np.int32))
