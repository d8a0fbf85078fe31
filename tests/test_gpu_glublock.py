"""GPU: the pre-norm residual GLU block (GluBlock, trainsim.hpp:136-146,
trainsim.cpp:294-308) -- RmsNorm fused into the gate/up input quantizer, the
residual adds fused into the down GEMM and the norm backward -- against the
reference's own GluBlock through oracle/_ref."""
import numpy as np
import pytest

from tests.helpers import bf16_round, outlier_matrix, rel_fro

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mods():
    import torch  # noqa: F401
    from oracle.oracle import REF_oracle, RefGluBlock
    from paper_2503_08040_b200 import linear
    if REF_oracle() is None:
        pytest.skip("oracle/_ref not present")
    return linear, RefGluBlock


def _weights(d, f, seed):
    rng = np.random.default_rng(seed)
    wg = (rng.standard_normal((f, d)) * 0.05).astype(np.float32)
    wu = (rng.standard_normal((f, d)) * 0.05).astype(np.float32)
    wd = (rng.standard_normal((d, f)) * 0.05).astype(np.float32)
    return wg, wu, wd


def _inputs(t, d, step):
    h = outlier_matrix(t, d, seed=70 + step, body=0.7, channels=[3], tokens=[t // 4], mag_c=12.0, mag_t=20.0)
    gout = outlier_matrix(t, d, seed=80 + step, body=1e-2)
    return h, gout


@pytest.mark.parametrize("d,f,t", [(256, 384, 384), (512, 640, 200)])
def test_glublock_training_steps_bit_exact_vs_reference(mods, d, f, t):
    """Three training steps (fwd, bwd, controller, SGD of the linears and the
    gain), exact mode: out, grad_h, the gain and its gradient, the weights,
    their gradients and the thresholds bit-identical to the reference block."""
    import torch
    linear, RefGluBlock = mods
    wg, wu, wd = _weights(d, f, 21)
    ref = RefGluBlock(wg, wu, wd, threshold=1.5)
    blk = linear.GluBlock(wg, wu, wd, t, act_dtype=torch.float32, mid_dtype=torch.float32, exact=True,
                          threshold_init=1.5)
    for step in range(3):
        h, gout = _inputs(t, d, step)
        out_r, gh_r = ref.step(h, gout, step)
        out = blk.forward(torch.from_numpy(h).cuda(), step).cpu().numpy()
        gh = blk.backward(torch.from_numpy(gout).cuda(), step).cpu().numpy()
        assert np.array_equal(out.view(np.int32), out_r.view(np.int32)), (step, rel_fro(out, out_r))
        assert np.array_equal(gh.view(np.int32), gh_r.view(np.int32)), (step, rel_fro(gh, gh_r))
        gain_r, gg_r, w_r, g_r = ref.state()
        gain, gg = blk.gain_host()
        assert np.array_equal(gg.view(np.int32), gg_r.view(np.int32)), step
        for a, b in zip(blk.grads_host(), g_r):
            assert np.array_equal(a.view(np.int32), b.view(np.int32)), step
        blk.controller_step()
        th_r = ref.controller()
        _, th = blk.controller_state()
        assert th[0] == th_r[0] == th_r[1] and th[1] == th_r[2], (step, th, th_r)
        blk.apply_sgd(0.05)
        ref.apply_sgd(0.05)
        gain_r, _, w_r, _ = ref.state()
        gain, _ = blk.gain_host()
        assert np.array_equal(gain.view(np.int32), gain_r.view(np.int32)), step
        for a, b in zip(blk.weights_host(), w_r):
            assert np.array_equal(a.view(np.int32), b.view(np.int32)), step


def test_glublock_bf16_fast_path_within_tolerance(mods):
    """bf16 activations / intermediates, FMA epilogue, packed contexts (the
    benched MLP configuration) against the reference fed the same bf16-rounded
    inputs: out within bf16 rounding of the residual sum, grad_h within the
    stochastic-rounding tolerance the MLP tests state."""
    import torch
    linear, RefGluBlock = mods
    d, f, t = 512, 1024, 512
    wg, wu, wd = _weights(d, f, 22)
    h, gout = _inputs(t, d, 7)
    h, gout = bf16_round(h), bf16_round(gout)
    ref = RefGluBlock(wg, wu, wd, threshold=2.0)
    out_r, gh_r = ref.step(h, gout, 0)
    blk = linear.GluBlock(wg, wu, wd, t, threshold_init=2.0, ctx_packed=True)
    out = blk.forward(torch.from_numpy(h).cuda().to(torch.bfloat16), 0).float().cpu().numpy()
    gh = blk.backward(torch.from_numpy(gout).cuda().to(torch.bfloat16), 0).float().cpu().numpy()
    assert rel_fro(out, out_r) < 1e-2
    assert rel_fro(gh, gh_r) < 5e-2


def test_glublock_equals_norm_then_mlp(mods):
    """The fused block == RmsNorm.forward -> GluMlp -> + h composed from the
    separate device entry points (same weights, same gain), bit for bit."""
    import torch
    from paper_2503_08040_b200 import fbq
    linear, _ = mods
    d, f, t = 256, 512, 256
    wg, wu, wd = _weights(d, f, 23)
    h, _ = _inputs(t, d, 3)
    hd = torch.from_numpy(h).cuda()
    kw = dict(act_dtype=torch.float32, mid_dtype=torch.float32, exact=True, threshold_init=1.5)
    blk = linear.GluBlock(wg, wu, wd, t, **kw)
    mlp = linear.GluMlp(wg, wu, wd, t, **kw)
    norm = fbq.RmsNorm(d)
    out = blk.forward(hd, 0)
    want = mlp.forward(norm.forward(hd), 0) + hd
    assert torch.equal(out.view(torch.int32), want.view(torch.int32))
