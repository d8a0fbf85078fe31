"""GPU: the device QuantLinear (fbq_linear_*) vs the reference's own
QuantLinearLayer (trainsim.cpp:61-135) through oracle/_ref."""
import numpy as np
import pytest

from tests.helpers import outlier_matrix, rel_fro

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mods():
    import torch  # noqa: F401
    from oracle.oracle import REF_oracle, RefLinear
    from paper_2503_08040_b200 import linear
    if REF_oracle() is None:
        pytest.skip("oracle/_ref not present")
    return linear, RefLinear


@pytest.mark.parametrize("shape", [(384, 256, 512), (200, 384, 272), (256, 128, 128)])
def test_linear_bit_exact_vs_reference_over_steps(mods, shape):
    """forward y, backward dX, accumulated dW and the controller's threshold,
    over three steps with controller updates (exact epilogue, fp32)."""
    import torch
    linear, RefLinear = mods
    t, d_in, d_out = shape
    rng = np.random.default_rng(3)
    w = (rng.standard_normal((d_out, d_in)) * 0.05).astype(np.float32)
    dev = linear.QuantLinear(w, t, act_dtype=torch.float32, exact=True, threshold_init=3.0, layer_id=5)
    ref = RefLinear(w, threshold=3.0, layer_id=5)
    for step in range(3):
        x = outlier_matrix(t, d_in, seed=10 + step, body=0.5, channels=[1], tokens=[t // 2],
                           mag_c=15.0, mag_t=30.0)
        gy = outlier_matrix(t, d_out, seed=20 + step, body=1e-3)
        y = dev.forward(torch.from_numpy(x).cuda(), step).cpu().numpy()
        gx = dev.backward(torch.from_numpy(gy).cuda(), step).cpu().numpy()
        yr = ref.forward(x, step)
        gxr = ref.backward(gy, step)
        assert np.array_equal(y.view(np.int32), yr.view(np.int32)), f"y step {step}"
        assert np.array_equal(gx.view(np.int32), gxr.view(np.int32)), f"dX step {step}"
        g = dev.grad().cpu().numpy()
        assert np.array_equal(g.view(np.int32), ref.grad().view(np.int32)), f"dW step {step}"
        dev.controller_step()
        rate_r, th_r = ref.controller_step()
        rate, th = dev.controller_state()
        assert rate == rate_r and th == th_r


def test_linear_bf16_fast_path_within_tolerance(mods):
    import torch
    linear, RefLinear = mods
    t, d_in, d_out = 512, 384, 256
    rng = np.random.default_rng(4)
    w = (rng.standard_normal((d_out, d_in)) * 0.05).astype(np.float32)
    x = outlier_matrix(t, d_in, seed=30, body=0.5, channels=[3], mag_c=15.0)
    gy = outlier_matrix(t, d_out, seed=31, body=1e-3)
    dev = linear.QuantLinear(w, t, act_dtype=torch.bfloat16, exact=False, threshold_init=3.0)
    ref = RefLinear(w, threshold=3.0)
    xb = torch.from_numpy(x).cuda().to(torch.bfloat16)
    gyb = torch.from_numpy(gy).cuda().to(torch.bfloat16)
    y = dev.forward(xb, 0).float().cpu().numpy()
    gx = dev.backward(gyb, 0).float().cpu().numpy()
    yr = ref.forward(xb.float().cpu().numpy(), 0)
    gxr = ref.backward(gyb.float().cpu().numpy(), 0)
    assert rel_fro(y, yr) < 1e-2 and rel_fro(gx, gxr) < 1e-2
    assert rel_fro(dev.grad().cpu().numpy(), ref.grad()) < 1e-5


@pytest.mark.parametrize("mode,rate", [("fixed_rate", 0.25), ("fixed_rate", 0.0), ("off", 0.0)])
def test_linear_fixed_rate_and_off_modes(mods, mode, rate):
    """FallbackMode::FixedRate (device TopK mask) and Off vs the reference."""
    import torch
    linear, RefLinear = mods
    t, d_in, d_out = 384, 512, 256
    rng = np.random.default_rng(6)
    w = (rng.standard_normal((d_out, d_in)) * 0.05).astype(np.float32)
    dev = linear.QuantLinear(w, t, act_dtype=torch.float32, exact=True, fallback_mode=mode,
                             fixed_rate=rate, layer_id=2)
    ref = RefLinear(w, layer_id=2, fallback_mode=mode, fixed_rate=rate)
    for step in range(2):
        x = outlier_matrix(t, d_in, seed=40 + step, body=0.5, channels=[1, 300], tokens=[5],
                           mag_c=15.0, mag_t=30.0)
        gy = outlier_matrix(t, d_out, seed=50 + step, body=1e-3)
        y = dev.forward(torch.from_numpy(x).cuda(), step).cpu().numpy()
        gx = dev.backward(torch.from_numpy(gy).cuda(), step).cpu().numpy()
        assert np.array_equal(y.view(np.int32), ref.forward(x, step).view(np.int32))
        assert np.array_equal(gx.view(np.int32), ref.backward(gy, step).view(np.int32))
        dev.controller_step()
        rate_r, th_r = ref.controller_step()
        rate_d, th_d = dev.controller_state()
        assert rate_d == rate_r and th_d == th_r
