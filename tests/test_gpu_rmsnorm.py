"""GPU: RmsNorm with its 10-bit 1 x 128 context vs the
reference's own RmsNorm (trainsim.cpp:145-219) through oracle/_ref."""
import numpy as np
import pytest

from tests.helpers import bf16_round, outlier_matrix

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("rows,dim", [(256, 384), (200, 512), (129, 1024)])
def test_rmsnorm_bit_exact_vs_reference(rows, dim):
    """forward y, the 10-bit context, backward gx and grad_gain, then an SGD step
    (non-trivial gains) and a second forward/backward -- all bit-identical."""
    import torch
    from oracle.oracle import C_oracle, REF_oracle, RefRmsNorm
    from paper_2503_08040_b200 import fbq
    if REF_oracle() is None:
        pytest.skip("oracle/_ref not present")
    ref = RefRmsNorm(dim)
    dev = fbq.RmsNorm(dim)
    orc = C_oracle()
    for it in range(2):
        x = outlier_matrix(rows, dim, seed=60 + it, body=1.0, channels=[3], tokens=[rows // 2],
                           mag_c=40.0, mag_t=25.0)
        gy = outlier_matrix(rows, dim, seed=70 + it, body=1e-2)
        y = dev.forward(torch.from_numpy(x).cuda()).cpu().numpy()
        assert np.array_equal(y.view(np.int32), ref.forward(x).view(np.int32)), f"y {it}"
        codes, scales = dev.context()
        c_want, s_want = orc.quantize_rtn(x, 1, 128, 10)
        assert np.array_equal(codes.cpu().numpy()[:, :dim], c_want)
        assert np.array_equal(scales.cpu().numpy().reshape(-1), s_want.reshape(-1))
        gx = dev.backward(torch.from_numpy(gy).cuda()).cpu().numpy()
        assert np.array_equal(gx.view(np.int32), ref.backward(gy).view(np.int32)), f"gx {it}"
        g_r, gg_r = ref.state()
        assert np.array_equal(dev.grad_gain.cpu().numpy().view(np.int32), gg_r.view(np.int32))
        dev.apply_sgd(0.05)
        ref.apply_sgd(0.05)
        g_r, _ = ref.state()
        assert np.array_equal(dev.gain.cpu().numpy().view(np.int32), g_r.view(np.int32))


@pytest.mark.parametrize("rows,dim", [(1000, 4096), (333, 1152)])
def test_rmsnorm_bf16_llama_width(rows, dim):
    """bf16 activations at Llama width (32 ring chunks per row, a partial last
    warp of rows): y / dx rounded to bf16 from the reference's fp32 results on
    the same bf16 inputs, the context and grad_gain bit-identical."""
    import torch
    from oracle.oracle import C_oracle, REF_oracle, RefRmsNorm
    from paper_2503_08040_b200 import fbq
    from tests.helpers import bf16_round
    if REF_oracle() is None:
        pytest.skip("oracle/_ref not present")
    ref = RefRmsNorm(dim)
    dev = fbq.RmsNorm(dim)
    orc = C_oracle()
    x = bf16_round(outlier_matrix(rows, dim, seed=80, body=1.0, channels=[5], tokens=[7], mag_c=40.0, mag_t=25.0))
    gy = bf16_round(outlier_matrix(rows, dim, seed=81, body=1e-2))
    y = dev.forward(torch.from_numpy(x).cuda().to(torch.bfloat16)).float().cpu().numpy()
    assert np.array_equal(y, bf16_round(ref.forward(x)))
    codes, scales = dev.context()
    c_want, s_want = orc.quantize_rtn(x, 1, 128, 10)
    assert np.array_equal(codes.cpu().numpy()[:, :dim], c_want)
    assert np.array_equal(scales.cpu().numpy().reshape(-1), s_want.reshape(-1))
    gx = dev.backward(torch.from_numpy(gy).cuda().to(torch.bfloat16)).float().cpu().numpy()
    assert np.array_equal(gx, bf16_round(ref.backward(gy)))
    _, gg_r = ref.state()
    assert np.array_equal(dev.grad_gain.cpu().numpy().view(np.int32), gg_r.view(np.int32))


@pytest.mark.parametrize("rows,dim,dtype,nsr", [(256, 384, "f32", 2), (300, 1152, "bf16", 1),
                                                (1000, 4096, "bf16", 2), (129, 512, "f32", 0)])
@pytest.mark.parametrize("masking", ["threshold", "given"])
def test_rmsnorm_fused_input_quantizer(rows, dim, dtype, nsr, masking):
    """RmsNorm.forward_quantized == forward() then the linear-input quantizer on
    y (codes, scales, mask, residuals, stochastic planes) -- bit for bit -- and
    the same RmsNorm context; y is never materialised on the fused path."""
    import torch
    from paper_2503_08040_b200 import fbq
    from tests.helpers import bf16_round
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    x = outlier_matrix(rows, dim, seed=90, body=1.0, channels=[5], tokens=[7], mag_c=40.0, mag_t=25.0)
    if dtype == "bf16":
        x = bf16_round(x)
    xt = torch.from_numpy(x).cuda().to(tdt)
    a, b = fbq.RmsNorm(dim), fbq.RmsNorm(dim)
    g = torch.linspace(0.5, 1.5, dim, device="cuda")
    a.gain.copy_(g)
    b.gain.copy_(g)
    y = a.forward(xt)
    scores = fbq.score_blocks(y)
    kw = {"theta": float(scores.flatten().median().item())} if masking == "threshold" else \
        {"mask": fbq.mask_topk(scores, 0.2)}
    s1, s2 = fbq.layer_seed(7, 3, 0, 1), fbq.layer_seed(7, 3, 1, 1)
    want = fbq.fallback_quantize(y, sr_seed=s1 if nsr >= 1 else None, **kw)
    got = b.forward_quantized(xt, sr_seed=s1 if nsr >= 1 else None, sr_seed2=s2 if nsr == 2 else None, **kw)
    wf, gf = (want[0], got[0]) if nsr >= 1 else (want, got)
    eq = lambda u, v: torch.equal(u.view(torch.int32) if u.dtype == torch.float32 else u,
                                  v.view(torch.int32) if v.dtype == torch.float32 else v)
    assert eq(gf.primary.codes[:, :dim], wf.primary.codes[:, :dim])
    assert eq(gf.primary.scales, wf.primary.scales)
    assert torch.equal(gf.mask, wf.mask)
    assert int(gf.masked_count.item()) == int(wf.masked_count.item())
    m = wf.mask.bool()
    for bi, bj in zip(*torch.nonzero(m, as_tuple=True)):
        r0, c0 = int(bi) * 128, int(bj) * 128
        assert torch.equal(gf.res_codes[r0:r0 + 128, c0:min(c0 + 128, dim)],
                           wf.res_codes[r0:r0 + 128, c0:min(c0 + 128, dim)])
    assert eq(gf.res_scales[m], wf.res_scales[m])
    if nsr >= 1:
        assert torch.equal(got[1].codes[:, :dim], want[1].codes[:, :dim])
    if nsr == 2:
        q2 = fbq.quantize_stochastic(y, s2)
        assert torch.equal(got[2].codes[:, :dim], q2.codes[:, :dim])
    for u, v in zip(a.context(), b.context()):
        assert torch.equal(u, v)


@pytest.mark.parametrize("rows,dim", [(256, 384), (129, 1024), (300, 200)])
def test_silu_layer_bit_exact_vs_reference(rows, dim):
    """SiluLayer (trainsim.cpp:265-290): y, the 10-bit 1 x 128 context and the
    backward gx bit-identical to the reference's own layer (exact math)."""
    import torch
    from oracle.oracle import C_oracle, REF_oracle, RefSilu
    from paper_2503_08040_b200 import fbq
    if REF_oracle() is None:
        pytest.skip("oracle/_ref not present")
    ref = RefSilu()
    dev = fbq.SiluLayer(exact=True)
    x = outlier_matrix(rows, dim, seed=90, body=2.0, channels=[3], tokens=[rows // 2], mag_c=30.0, mag_t=12.0)
    gy = outlier_matrix(rows, dim, seed=91, body=1e-2)
    y = dev.forward(torch.from_numpy(x).cuda()).cpu().numpy()
    assert np.array_equal(y.view(np.int32), ref.forward(x).view(np.int32))
    codes, scales = dev.context()
    c_want, s_want = C_oracle().quantize_rtn(x, 1, 128, 10)
    assert np.array_equal(codes.cpu().numpy()[:, :dim], c_want)
    assert np.array_equal(scales.cpu().numpy().reshape(-1), s_want.reshape(-1))
    gx = dev.backward(torch.from_numpy(gy).cuda()).cpu().numpy()
    assert np.array_equal(gx.view(np.int32), ref.backward(gy).view(np.int32))


def test_silu_layer_bf16_fast_within_tolerance():
    """bf16 activations, fp32 fast silu: within bf16 rounding of the exact layer."""
    import torch
    from paper_2503_08040_b200 import fbq
    from tests.helpers import rel_fro
    x = bf16_round(outlier_matrix(512, 1024, seed=92, body=2.0))
    gy = bf16_round(outlier_matrix(512, 1024, seed=93, body=1e-2))
    ex, fa = fbq.SiluLayer(exact=True), fbq.SiluLayer(exact=False)
    y_e = ex.forward(torch.from_numpy(x).cuda()).cpu().numpy()
    y_f = fa.forward(torch.from_numpy(x).cuda().to(torch.bfloat16)).float().cpu().numpy()
    assert rel_fro(y_f, y_e) < 8e-3
    g_e = ex.backward(torch.from_numpy(gy).cuda()).cpu().numpy()
    g_f = fa.backward(torch.from_numpy(gy).cuda().to(torch.bfloat16)).float().cpu().numpy()
    assert rel_fro(g_f, g_e) < 8e-3
