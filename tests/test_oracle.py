"""CPU: pin the oracle (oracle/fbq_oracle.c) before trusting it.

1. against golden vectors produced by the reference itself
   (tests/golden/make_golden.py runs oracle/_ref = the unmodified reference);
2. against the SPEC.md known-answer examples;
3. live against the reference build on random inputs (when oracle/_ref exists);
4. the reference's own kernel pins (tests/test_kernels.cpp): backend
   bit-equality on odd/strided shapes and the int32 headroom.
"""
import os

import numpy as np
import pytest

from oracle.oracle import compact_to_dense
from tests.helpers import outlier_matrix

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "golden.npz")


@pytest.fixture(scope="module")
def G():
    return dict(np.load(GOLDEN))


def bits_eq(a, b):
    a, b = np.asarray(a), np.asarray(b)
    if a.dtype == np.float32:
        return a.shape == b.shape and np.array_equal(a.view(np.int32), b.astype(np.float32).view(np.int32))
    return a.shape == b.shape and np.array_equal(a, b)


# ------------------------------------------------------------ golden vectors
def test_golden_rng(orc, G):
    for i, s in enumerate(G["rng_seeds"]):
        for j, n in enumerate(G["rng_ns"]):
            assert orc.bits_at(int(s), int(n)) == int(G["rng_bits"][i, j])
            assert orc.uniform_at(int(s), int(n)) == G["rng_uniform"][i, j]
            assert np.float32(orc.normal_at(int(s), int(n))) == G["rng_normal"][i, j]
    ds = [orc.derive_seed(0x5EED, a, b) for a in range(6) for b in range(3)]
    assert np.array_equal(np.array(ds, np.uint64), G["derive_seed"])


def test_golden_rtn(orc, G):
    c, s = orc.quantize_rtn(G["rtn_x"])
    assert bits_eq(c, G["rtn_codes"]) and bits_eq(s, G["rtn_scales"])


def test_golden_sr(orc, G):
    c, s = orc.quantize_stochastic(G["sr_x"], int(G["sr_seed"]))
    assert bits_eq(c, G["sr_codes"]) and bits_eq(s, G["sr_scales"])


def test_golden_fallback(orc, G):
    x = G["fb_x"]
    scores = orc.score_blocks_absmax(x)
    assert np.array_equal(scores, G["fb_scores"])
    mask = orc.mask_topk(scores, 0.34)
    assert np.array_equal(mask, G["fb_mask"])
    assert np.array_equal(orc.mask_threshold(scores, float(G["fb_theta"])), G["fb_mask_thr"])
    c, s, rc, rs = orc.fallback_quantize(x, mask)
    wrc, wrs = compact_to_dense(G["fb_res_compact"], G["fb_res_scales"], G["fb_res_index"],
                                *x.shape, 128)
    assert bits_eq(c, G["fb_codes"]) and bits_eq(s, G["fb_scales"])
    assert bits_eq(rc, wrc) and bits_eq(rs, wrs)
    assert bits_eq(orc.dequantize_fallback(c, s, mask, rc, rs), G["fb_dequant"])


def test_golden_gemms(orc, G):
    x = G["fb_x"]
    mask = G["fb_mask"]
    c, s, rc, rs = orc.fallback_quantize(x, mask)
    bc, bs = orc.quantize_rtn(G["gemm_b"])
    assert bits_eq(orc.block_gemm(c, s, bc, bs), G["gemm_block"])
    assert bits_eq(orc.block_gemm(c, s, bc, bs, mask=mask, res_codes=rc, res_scales=rs),
                   G["gemm_fallback"])
    assert bits_eq(orc.block_gemm(c, s, bc, bs, tile=(32, 64, 16)), G["gemm_tiled"])
    # SPEC.md:245 oracle equivalence within 1e-5 relative Frobenius
    y = G["gemm_fallback"].astype(np.float64)
    o = G["gemm_oracle"].astype(np.float64)
    assert np.linalg.norm(y - o) / np.linalg.norm(o) <= 1e-5


def test_golden_controller(orc, G):
    got = [orc.controller_update(1.0, r) for r in (0.05, 0.35, 0.2, 0.1, 0.3)]
    assert np.array_equal(np.array(got), G["ctl"])


# ------------------------------------------------- SPEC.md known answers
def test_spec_rtn_example(orc):
    # SPEC.md:123  [254, -127, 0, 63.5] -> a = 2, codes [127, -64, 0, 32]
    c, s = orc.quantize_rtn(np.array([[254, -127], [0, 63.5]], np.float32), 2, 2)
    assert s[0, 0] == 2.0 and c.ravel().tolist() == [127, -64, 0, 32]
    z, zs = orc.quantize_rtn(np.zeros((128, 128), np.float32))
    assert zs[0, 0] == 0 and not z.any()


def test_spec_fallback_example(orc):
    # SPEC.md:153  [1000, 1, -1, 0.5] masked
    x = np.array([[1000, 1], [-1, 0.5]], np.float32)
    c, s, rc, rs = orc.fallback_quantize(x, np.ones((1, 1), np.uint8), g=2)
    assert c.ravel().tolist() == [127, 0, 0, 0]
    assert rs[0, 0] == np.float32(np.float32(1.0) / np.float32(127.0))
    assert rc.ravel().tolist() == [0, 127, -127, 64]
    d = orc.dequantize_fallback(c, s, np.ones((1, 1), np.uint8), rc, rs, g=2)
    assert np.all(np.abs(d - x) <= rs[0, 0] / 2)


def test_spec_policy_examples(orc):
    assert orc.mask_topk(np.array([5, 1, 9, 9], np.float64), 0.5).tolist() == [0, 0, 1, 1]
    assert orc.mask_topk(np.array([1, 2, 3.0]), 0.0).tolist() == [0, 0, 0]
    assert orc.mask_topk(np.array([1, 2, 3.0]), 1.0).tolist() == [1, 1, 1]
    assert orc.mask_threshold(np.array([0.5, 2.0]), 1.0).tolist() == [0, 1]
    assert orc.mask_threshold(np.array([1.0]), 1.0).tolist() == [0]  # strict
    assert orc.controller_update(1.0, 0.05) == 1.0 / 1.3
    assert orc.controller_update(1.0, 0.35) == 1.3
    assert orc.controller_update(1.0, 0.2) == 1.0


def test_spec_sr_examples(orc):
    # x/a integer -> exact; 0.25 -> P(1) = 0.25
    x = np.zeros((1, 128), np.float32)
    x[0, 0] = 127.0  # forces a = 1
    x[0, 1] = 2.0
    c, s = orc.quantize_stochastic(x, 99, 1, 128)
    assert s[0, 0] == 1.0 and c[0, 1] == 2
    x = np.full((1, 100000), 0.25, np.float32)
    x[0, 0] = 127.0
    c, _ = orc.quantize_stochastic(x, 7, 1, 100000)
    p = c[0, 1:].mean()
    assert abs(p - 0.25) < 3 * np.sqrt(0.25 * 0.75 / 99999)


def test_accumulator_headroom(orc):
    # tests/test_kernels.cpp:110-118
    a = np.full((1, 128), 127, np.int16)
    b = np.full((128, 1), 127, np.int16)
    p = orc.block_products(a, b)
    assert p[0, 0, 0, 0, 0] == 2064512 < 2**31


# ----------------------------------------------- live vs the reference build
@pytest.mark.parametrize("shape", [(300, 270), (128, 128), (1, 7), (129, 257)])
def test_live_quantizers(orc, ref, shape):
    x = outlier_matrix(*shape, seed=sum(shape), channels=[0], tokens=[shape[0] // 2])
    for a, b in zip(orc.quantize_rtn(x), ref.quantize_rtn(x)):
        assert bits_eq(a, b)
    for a, b in zip(orc.quantize_stochastic(x, 0xABCDEF), ref.quantize_stochastic(x, 0xABCDEF)):
        assert bits_eq(a, b)
    m = orc.mask_topk(orc.score_blocks_absmax(x), 0.5)
    for a, b in zip(orc.fallback_quantize(x, m), ref.fallback_quantize(x, m)):
        assert bits_eq(a, b)


def test_live_gemm(orc, ref):
    a = outlier_matrix(200, 260, seed=1, channels=[3])
    b = outlier_matrix(260, 150, seed=2, body=0.05)
    m = orc.mask_topk(orc.score_blocks_absmax(a), 0.5)
    c, s, rc, rs = orc.fallback_quantize(a, m)
    bc, bs = orc.quantize_rtn(b)
    for kw in ({}, dict(mask=m, res_codes=rc, res_scales=rs), dict(tile=(64, 32, 128))):
        assert bits_eq(orc.block_gemm(c, s, bc, bs, **kw), ref.block_gemm(c, s, bc, bs, **kw))


def test_reference_backends_bit_equal(ref):
    """tests/test_kernels.cpp:35-90 through the reference's own Ops tables."""
    import ctypes as C
    lib = ref._l.lib
    f = lib.ref_ops_gemm_i16_accum
    f.argtypes = [C.c_char_p] + [C.c_void_p, C.c_size_t, C.c_void_p, C.c_size_t, C.c_void_p,
                                 C.c_size_t, C.c_size_t, C.c_size_t, C.c_size_t]
    if not lib.ref_avx2_supported():
        pytest.skip("no AVX2")
    rng = np.random.default_rng(0)
    for m, n, k in [(1, 1, 1), (3, 17, 5), (16, 33, 128), (12, 128, 9)]:
        lda, ldb, ldc = k + 1, n + 2, n + 1
        a = rng.integers(-127, 128, (m, lda)).astype(np.int16)
        b = rng.integers(-127, 128, (k, ldb)).astype(np.int16)
        c0 = rng.integers(-500, 500, (m, ldc)).astype(np.int32)
        outs = []
        for be in (b"scalar", b"avx2"):
            c = c0.copy()
            f(be, a.ctypes.data, lda, b.ctypes.data, ldb, c.ctypes.data, ldc, m, n, k)
            outs.append(c)
        assert np.array_equal(outs[0], outs[1])
        want = c0.astype(np.int64)
        want[:, :n] += a[:, :k].astype(np.int64) @ b[:, :n].astype(np.int64)
        assert np.array_equal(outs[0], want)


def test_ref_linear_forward_matches_restated_composition():
    """The QuantLinearLayer shim (oracle/ref_capi.cpp) against the C restatement
    composed like trainsim.cpp:80-98: threshold mask, fallback_quantize,
    quantize_rtn(W^T), fallback_gemm."""
    from oracle.oracle import C_oracle, REF_oracle, RefLinear
    if REF_oracle() is None:
        pytest.skip("oracle/_ref not built")
    orc = C_oracle()
    rng = np.random.default_rng(5)
    x = rng.standard_normal((256, 384)).astype(np.float32)
    x[:, 5] *= 40.0
    w = (rng.standard_normal((128, 384)) * 0.05).astype(np.float32)
    y = RefLinear(w, threshold=4.0).forward(x, 0)
    mask = orc.mask_threshold(orc.score_blocks_absmax(x), 4.0)
    c, s, rc, rs = orc.fallback_quantize(x, mask)
    wc, ws = orc.quantize_rtn(w)
    bc, bs = orc.transpose_qt(wc, ws)
    want = orc.block_gemm(c, s, bc, bs, mask=mask, res_codes=rc, res_scales=rs)
    assert np.array_equal(y.view(np.int32), want.view(np.int32))
