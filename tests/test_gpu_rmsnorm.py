"""GPU: RmsNorm with its 10-bit 1 x 128 context vs the
reference's own RmsNorm (trainsim.cpp:145-219) through oracle/_ref."""
import numpy as np
import pytest

from tests.helpers import outlier_matrix

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
