"""GPU: QuantLinearLayer::apply_sgd (trainsim.cpp:137-143) fused with the next
forward's weight quantization (fbq_cuda_sgd_quantize_rtn, fbq_mlp_apply_sgd,
fbq_linear_apply_sgd) -- against the two-kernel form and, over training steps,
against the reference's own layers through oracle/_ref."""
import numpy as np
import pytest

from tests.helpers import outlier_matrix, rel_fro

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mods():
    import torch  # noqa: F401
    from oracle.oracle import REF_oracle, RefLinear, RefMlp
    from paper_2503_08040_b200 import linear
    if REF_oracle() is None:
        pytest.skip("oracle/_ref not present")
    return linear, RefLinear, RefMlp


@pytest.mark.parametrize("rows,cols,lr", [(384, 256, 0.05), (300, 200, 1e-3), (129, 1000, 0.5),
                                          (256, 130, 0.05), (1, 4, 2.0)])
def test_sgd_quantize_rtn_matches_update_then_rtn(rows, cols, lr):
    """one fused pass == fbq_cuda_sgd_update then fbq_cuda_quantize_rtn (W', codes,
    scales bit for bit); cols % 4 != 0 (130) exercises the two-kernel fallback."""
    import torch
    from paper_2503_08040_b200 import _capi as K
    rng = np.random.default_rng(rows * 7 + cols)
    w0 = (rng.standard_normal((rows, cols)) * 0.05).astype(np.float32)
    w0[rows // 2, :: 7] *= 300.0  # outlier elements: blocks of very different scale
    g = (rng.standard_normal((rows, cols)) * 0.3).astype(np.float32)
    g[0, 0] = 0.0
    g[-1, -1] = -0.0
    ldq = (cols + 15) // 16 * 16
    nb = ((rows + 127) // 128) * ((cols + 127) // 128)
    s = torch.cuda.current_stream().cuda_stream
    wa = torch.from_numpy(w0).cuda()
    wb = wa.clone()
    gt = torch.from_numpy(g).cuda()
    qa = torch.zeros(rows, ldq, dtype=torch.int8, device="cuda")
    qb = torch.zeros_like(qa)
    sa = torch.zeros(nb, device="cuda")
    sb = torch.zeros_like(sa)
    K.call("fbq_cuda_sgd_quantize_rtn", wa.data_ptr(), gt.data_ptr(), rows, cols, lr, qa.data_ptr(), ldq,
           sa.data_ptr(), s)
    K.call("fbq_cuda_sgd_update", wb.data_ptr(), gt.data_ptr(), rows * cols, lr, s)
    K.call("fbq_cuda_quantize_rtn", wb.data_ptr(), K.FBQ_F32, rows, cols, cols, qb.data_ptr(), ldq,
           sb.data_ptr(), s)
    torch.cuda.synchronize()
    want = w0 - (lr * g.astype(np.float64)).astype(np.float32)  # the reference's expression
    assert np.array_equal(wb.cpu().numpy().view(np.int32), want.view(np.int32))
    assert torch.equal(wa.view(torch.int32), wb.view(torch.int32))
    assert torch.equal(qa[:, :cols], qb[:, :cols])
    assert torch.equal(sa.view(torch.int32), sb.view(torch.int32))


def test_mlp_training_steps_with_sgd_bit_exact_vs_reference(mods):
    """fwd + bwd + controller + apply_sgd over three steps (exact mode): y, dX,
    the accumulated dW, the updated weights and the controller -- bit for bit
    with the reference's QuantLinearLayer x 3 + GluCombine; the second and third
    forwards run on the codes the fused SGD wrote."""
    import torch
    linear, _, RefMlp = mods
    d, f, t = 256, 384, 384
    rng = np.random.default_rng(5)
    wg, wu = [(rng.standard_normal((f, d)) * 0.05).astype(np.float32) for _ in range(2)]
    wd = (rng.standard_normal((d, f)) * 0.05).astype(np.float32)
    ref = RefMlp(wg, wu, wd, threshold=1.0)
    m = linear.GluMlp(wg, wu, wd, t, act_dtype=torch.float32, mid_dtype=torch.float32, exact=True,
                      threshold_init=1.0)
    for step in range(3):
        x = outlier_matrix(t, d, seed=40 + step, body=0.3, channels=[5], tokens=[t // 3], mag_c=20.0,
                           mag_t=40.0)
        gy = outlier_matrix(t, d, seed=50 + step, body=1e-2)
        y_r, gx_r = ref.step(x, gy, step)
        y = m.forward(torch.from_numpy(x).cuda(), step).cpu().numpy()
        gx = m.backward(torch.from_numpy(gy).cuda(), step).cpu().numpy()
        assert np.array_equal(y.view(np.int32), y_r.view(np.int32)), (step, rel_fro(y, y_r))
        assert np.array_equal(gx.view(np.int32), gx_r.view(np.int32)), (step, rel_fro(gx, gx_r))
        m.controller_step()
        ref.controller()
        m.apply_sgd(0.5)
        ref.apply_sgd(0.5)
        for a, b in zip(m.weights_host(), ref.weights()):
            assert np.array_equal(a.view(np.int32), b.view(np.int32)), step
    for a, b in zip(m.grads_host(), ref.grads()):
        assert np.array_equal(a.view(np.int32), b.view(np.int32))


def test_mlp_sgd_after_zero_grad_is_identity(mods):
    """a pending (deferred) zero_grad: apply_sgd leaves W unchanged (w - lr * 0),
    and the next forward still quantizes W itself."""
    import torch
    linear, _, _ = mods
    d, f, t = 128, 256, 256
    rng = np.random.default_rng(6)
    wg, wu = [(rng.standard_normal((f, d)) * 0.05).astype(np.float32) for _ in range(2)]
    wd = (rng.standard_normal((d, f)) * 0.05).astype(np.float32)
    m = linear.GluMlp(wg, wu, wd, t, act_dtype=torch.float32, mid_dtype=torch.float32, exact=True)
    x = torch.from_numpy(outlier_matrix(t, d, seed=1, body=0.3)).cuda()
    y0 = m.forward(x, 0).clone()
    m.backward(torch.from_numpy(outlier_matrix(t, d, seed=2, body=1e-2)).cuda(), 0)
    m.zero_grad()
    m.apply_sgd(0.5)
    for a, b in zip(m.weights_host(), (wg, wu, wd)):
        assert np.array_equal(a.view(np.int32), b.view(np.int32))
    assert torch.equal(m.forward(x, 0), y0)


def test_linear_sgd_bit_exact_vs_reference(mods):
    """QuantLinear: forward / backward / apply_sgd over three steps, weights and
    outputs bit-identical to the reference layer."""
    import torch
    linear, RefLinear, _ = mods
    t, d_in, d_out = 300, 256, 384
    rng = np.random.default_rng(7)
    w = (rng.standard_normal((d_out, d_in)) * 0.05).astype(np.float32)
    dev = linear.QuantLinear(w, t, act_dtype=torch.float32, exact=True, threshold_init=3.0, layer_id=2)
    ref = RefLinear(w, threshold=3.0, layer_id=2)
    for step in range(3):
        x = outlier_matrix(t, d_in, seed=60 + step, body=0.5, channels=[1], mag_c=15.0)
        gy = outlier_matrix(t, d_out, seed=70 + step, body=1e-2)
        y = dev.forward(torch.from_numpy(x).cuda(), step).cpu().numpy()
        gx = dev.backward(torch.from_numpy(gy).cuda(), step).cpu().numpy()
        assert np.array_equal(y.view(np.int32), ref.forward(x, step).view(np.int32)), step
        assert np.array_equal(gx.view(np.int32), ref.backward(gy, step).view(np.int32)), step
        dev.apply_sgd(0.25)
        ref.apply_sgd(0.25)
        assert np.array_equal(dev.weight_host().view(np.int32), ref.weight().view(np.int32)), step


@pytest.mark.parametrize("n,off", [(1001, 0), (1001, 1), (4 * 148 * 256 * 5 + 3, 0), (7, 3)])
def test_sgd_update_vector_and_tail_paths(n, off):
    """fbq_cuda_sgd_update on aligned (16-byte vectors + scalar tail) and
    misaligned (scalar loop) buffers == the reference's w - float(lr * double(g))."""
    import torch
    from paper_2503_08040_b200 import _capi as K
    rng = np.random.default_rng(n + off)
    w0 = (rng.standard_normal(n + off) * 0.05).astype(np.float32)
    g = (rng.standard_normal(n + off)).astype(np.float32)
    wt, gt = torch.from_numpy(w0).cuda(), torch.from_numpy(g).cuda()
    lr = 0.0123
    K.call("fbq_cuda_sgd_update", wt.data_ptr() + 4 * off, gt.data_ptr() + 4 * off, n, lr,
           torch.cuda.current_stream().cuda_stream)
    want = w0.copy()
    want[off:] = w0[off:] - (lr * g[off:].astype(np.float64)).astype(np.float32)
    assert np.array_equal(wt.cpu().numpy().view(np.int32), want.view(np.int32))
