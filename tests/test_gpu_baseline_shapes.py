"""GPU parity at the BASELINE.json shapes (VERDICT r01 "Next round" #1).

* C1: the fallback-quantized linear forward Y = X W^T at M = N = K = 4096 with a
  10 % topk mask -- EXACT epilogue bit-exact against the reference itself
  (oracle/_ref: fallback_quantize + quantize_rtn(W^T) + fallback_gemm,
  gemm.cpp:101-186), FMA epilogue within SPEC.md's 1e-5 relative Frobenius.
* C2: quantize + fallback-detect on 8192 x {4096, 14336}, bf16 and fp32, at the
  rates 0 / 5 / 20 % through a GIVEN topk mask (policy.cpp:56-71): codes,
  scales, bitmap, residual codes and residual scales bit-exact against the C
  oracle (quant.cpp:128-176); THRESHOLD mode reproduces the same mask when
  theta sits strictly between the k-th and (k+1)-th distinct block scores.
* C3: the Llama-3.1-8B SwiGLU MLP (d_model 4096, d_ff 14336) at T = 256
  tokens, fp32 intermediates + exact epilogue, bit-exact against the
  reference's QuantLinearLayer x 3 + GluCombine over two steps with the
  controller (trainsim.cpp:61-133, 224-263) -- covers K = 14336 (four
  32-k-block scale pages) and the dX GEMM over K = 2 d_ff through strided
  operands.
* The bench's own fast path (bf16 activations and intermediates, FMA epilogue,
  fp32 SiLU) against the reference fed the SAME bf16-rounded inputs, with the
  tolerance DESIGN.md §5 states.
"""
import os

import numpy as np
import pytest

from tests.helpers import bf16_round, outlier_matrix, rel_fro

pytestmark = pytest.mark.gpu

FMA_TOL = 1e-5
# bench fast path vs the reference on identical (bf16-rounded) inputs, DESIGN.md §5:
# y within 4x the bf16 rounding of y; dX / dW within a quarter of the reference's
# own seed-to-seed stochastic-rounding spread (measured B200: y 2.9e-3 vs bf16
# 1.7e-3; dX 1.6e-2 vs 1.8e-1; dW 1.0-2.0e-2 vs 1.4-3.4e-1)
FAST_Y_BF16_FACTOR = 4.0
FAST_SR_FRACTION = 0.25


def dev(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def host(t):
    return t.detach().cpu().numpy()


@pytest.fixture(scope="module")
def F():
    import torch  # noqa: F401
    from paper_2503_08040_b200 import fbq
    return fbq


@pytest.fixture(scope="module")
def R(ref):
    ref.set_gemm_threads(os.cpu_count() or 1)
    return ref


# ------------------------------------------------------------------ C1
@pytest.fixture(scope="module")
def c1(F, R):
    n = 4096
    x = outlier_matrix(n, n, seed=101, channels=[7, 1000, 2049, 3333], tokens=[17, 2900],
                       occasional=40)
    w = outlier_matrix(n, n, seed=102, body=0.02)
    mask = R.mask_topk(R.score_blocks_absmax(x), 0.10)
    c, s, rc, rs = R.fallback_quantize(x, mask)
    wc, ws = R.quantize_rtn(np.ascontiguousarray(w.T))  # quantize_rtn(transpose(W)), trainsim.cpp:96-97
    want = R.block_gemm(c, s, wc, ws, mask=mask, res_codes=rc, res_scales=rs)
    return x, w, mask, want


def test_c1_fallback_linear_4096_exact_vs_reference(F, c1):
    x, w, mask, want = c1
    assert abs(mask.mean() - 0.10) < 1e-3
    fa = F.fallback_quantize(dev(x), dev(mask))
    wq = F.quantize_rtn(dev(w))
    y = F.fallback_gemm(fa, F.transpose(wq))
    got = host(y)
    assert np.array_equal(got.view(np.int32), want.view(np.int32)), rel_fro(got, want)


def test_c1_fallback_linear_4096_fma_within_tolerance(F, c1):
    x, w, mask, want = c1
    fa = F.fallback_quantize(dev(x), dev(mask))
    y = F.fallback_gemm(fa, F.transpose(F.quantize_rtn(dev(w))), exact=False)
    assert rel_fro(host(y), want) <= FMA_TOL


# ------------------------------------------------------------------ C2
def _c2_input(rows, cols, dtype):
    """Outlier channels/tokens whose magnitude drifts smoothly (+-15 %) across
    tokens and channels (bench.make_activations' recipe): block AbsMax scores
    are then distinct even after bf16 rounding, so a threshold realises the
    intended rate."""
    x = outlier_matrix(rows, cols, seed=rows + cols, channels=[3, cols // 3, cols - 5],
                       tokens=[rows // 7], occasional=max(1, rows * cols // 100000))
    r = np.arange(rows, dtype=np.float32)[:, None]
    c = np.arange(cols, dtype=np.float32)[None, :]
    drift = (1.0 + 0.15 * np.sin(r * 0.0015 + c * 0.0007)).astype(np.float32)
    big = np.abs(x) > 50
    x[big] *= drift[big] if drift.shape == x.shape else np.broadcast_to(drift, x.shape)[big]
    return bf16_round(x) if dtype == "bf16" else x


@pytest.mark.parametrize("shape", [(8192, 4096), (8192, 14336)])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_c2_quantize_fallback_given_mask(F, orc, shape, dtype):
    import torch
    rows, cols = shape
    x = _c2_input(rows, cols, dtype)
    xt = dev(x).to(torch.bfloat16) if dtype == "bf16" else dev(x)
    scores = orc.score_blocks_absmax(x)
    assert np.array_equal(host(F.score_blocks(xt)), scores)
    nb = scores.size
    for rate in (0.0, 0.05, 0.20):
        mask = orc.mask_topk(scores, rate)
        assert int(mask.sum()) == int(np.ceil(rate * nb))  # the rate is exact
        fa = F.fallback_quantize(xt, dev(mask))
        codes, sc, rcodes, rsc = orc.fallback_quantize(x, mask)
        assert np.array_equal(host(fa.mask), mask)
        assert np.array_equal(host(fa.primary.codes_int16()), codes), rate
        assert np.array_equal(host(fa.primary.scales).view(np.int32), sc.view(np.int32)), rate
        assert np.array_equal(host(fa.res_scales).view(np.int32), rsc.view(np.int32)), rate
        if mask.any():
            m = np.repeat(np.repeat(mask.astype(bool), 128, 0), 128, 1)[:rows, :cols]
            got_rc = host(fa.res_codes[:rows, :cols]).astype(np.int16)
            assert np.array_equal(got_rc[m], rcodes[m]), rate
        del fa


@pytest.mark.parametrize("shape", [(8192, 4096), (8192, 14336)])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_c2_threshold_mode_true_rates(F, orc, shape, dtype):
    """theta strictly between distinct sorted scores flags exactly the intended
    fraction (the round-1 bench took theta FROM the sorted scores with a strict
    `>`, so tied outlier-channel blocks fell short of 5 % / over-shot 20 %)."""
    import torch
    from paper_2503_08040_b200.fbq import theta_for_rate
    rows, cols = shape
    x = _c2_input(rows, cols, dtype)
    xt = dev(x).to(torch.bfloat16) if dtype == "bf16" else dev(x)
    scores = orc.score_blocks_absmax(x)
    for rate in (0.0, 0.05, 0.20):
        theta, exact_rate = theta_for_rate(scores, rate)
        fa = F.fallback_quantize(xt, theta=theta)
        mask = orc.mask_threshold(scores, theta)
        assert np.array_equal(host(fa.mask), mask)
        assert int(fa.masked_count.item()) == int(mask.sum())
        assert abs(mask.mean() - exact_rate) < 1e-12
        assert abs(exact_rate - rate) <= 0.01  # tied blocks move it by at most a tie group
        codes, sc, _, rsc = orc.fallback_quantize(x, mask)
        assert np.array_equal(host(fa.primary.codes_int16()), codes)
        assert np.array_equal(host(fa.res_scales).view(np.int32), rsc.view(np.int32))


# ------------------------------------------------------------------ C3
D, FF, T = 4096, 14336, 256


@pytest.fixture(scope="module")
def c3_weights():
    rng = np.random.default_rng(2)
    wg = rng.standard_normal((FF, D), dtype=np.float32) * 0.02
    wu = rng.standard_normal((FF, D), dtype=np.float32) * 0.02
    wd = rng.standard_normal((D, FF), dtype=np.float32) * 0.02
    return wg, wu, wd


def _c3_inputs(step):
    x = outlier_matrix(T, D, seed=200 + step, channels=[11, 1500, 4000], tokens=[37], mag_t=60.0,
                       occasional=8)
    gy = outlier_matrix(T, D, seed=300 + step, body=1e-3, tokens=[5], mag_t=3e-2)
    return x, gy


def test_c3_mlp_full_dims_exact_vs_reference(F, R, c3_weights):
    """C3 at full dims, exact mode: two training steps (fwd, bwd, controller, SGD
    between them) bit-identical to the reference."""
    import torch
    from oracle.oracle import RefMlp
    from paper_2503_08040_b200 import linear
    wg, wu, wd = c3_weights
    th = 8.0
    ref = RefMlp(wg, wu, wd, threshold=th)
    m = linear.GluMlp(wg, wu, wd, T, act_dtype=torch.float32, mid_dtype=torch.float32, exact=True,
                      threshold_init=th)
    for step in range(2):
        x, gy = _c3_inputs(step)
        y_r, gx_r = ref.step(x, gy, step)
        y = m.forward(dev(x), step)
        gx = m.backward(dev(gy), step)
        y, gx = host(y), host(gx)
        assert np.array_equal(y.view(np.int32), y_r.view(np.int32)), (step, rel_fro(y, y_r))
        assert np.array_equal(gx.view(np.int32), gx_r.view(np.int32)), (step, rel_fro(gx, gx_r))
        m.controller_step()
        rates, th_g = m.controller_state()
        r_rates, r_th = ref.controller()
        assert rates[0] == r_rates[0] and rates[1] == r_rates[2], (step, rates, r_rates)
        assert th_g[0] == r_th[0] and th_g[1] == r_th[2], (step, th_g, r_th)
        if step == 0:
            # QuantLinearLayer::apply_sgd on the three weights (trainsim.cpp:137-143); the
            # device update is fused with the weight RTN that step 1's forward then uses
            m.apply_sgd(0.05)
            ref.apply_sgd(0.05)
            for w, w_r in zip(m.weights_host(), ref.weights()):
                assert np.array_equal(w.view(np.int32), w_r.view(np.int32))
    for g, g_r in zip(m.grads_host(), ref.grads()):
        assert np.array_equal(g.view(np.int32), g_r.view(np.int32)), rel_fro(g, g_r)


def test_c3_bench_fast_path_vs_reference_same_inputs(F, R, c3_weights):
    """The benched configuration (bf16 activations/intermediates, FMA epilogue,
    fp32 SiLU) against the reference given the SAME bf16-rounded x and dY, so
    the difference is the fast path's own rounding, not input rounding.

    Tolerance, per output:
    * y (no stochastic rounding on the forward path): within 4x the bf16
      rounding of the reference's own y -- the fast path stores [a|b], h and y
      in bf16, so RTN codes of h near a rounding boundary may move by one;
    * dX, dW: within the reference's OWN stochastic-rounding noise, i.e. the
      difference between two reference runs whose SR streams differ (the same
      inputs at step 0 and step 1, layer_seed(.., step), trainsim.cpp:16-19).
      bf16 intermediates shift some SR decisions (u < frac, quant.cpp:69-77);
      an implementation is as accurate as the algorithm when its deviation
      stays inside the algorithm's own seed-to-seed spread."""
    import torch
    from oracle.oracle import RefMlp
    from paper_2503_08040_b200 import linear
    wg, wu, wd = c3_weights
    th = 8.0
    x, gy = _c3_inputs(5)
    x, gy = bf16_round(x), bf16_round(gy)
    ref = RefMlp(wg, wu, wd, threshold=th)
    y_r, gx_r = ref.step(x, gy, 0)
    g_r = ref.grads()
    ref2 = RefMlp(wg, wu, wd, threshold=th)
    _, gx_r2 = ref2.step(x, gy, 1)  # same inputs, other SR streams
    g_r2 = ref2.grads()
    m = linear.GluMlp(wg, wu, wd, T, threshold_init=th)  # bench defaults: bf16 / FMA
    y = host(m.forward(dev(x).to(torch.bfloat16), 0).float())
    gx = host(m.backward(dev(gy).to(torch.bfloat16), 0).float())
    g = m.grads_host()
    e_y, e_gx = rel_fro(y, y_r), rel_fro(gx, gx_r)
    bf16_y = rel_fro(bf16_round(y_r), y_r)
    sr_gx = rel_fro(gx_r2, gx_r)
    e_g = [rel_fro(a, b) for a, b in zip(g, g_r)]
    sr_g = [rel_fro(a, b) for a, b in zip(g_r2, g_r)]
    print(f"\nfast path vs reference (same bf16 inputs): y {e_y:.2e} (bf16 rounding {bf16_y:.2e}); "
          f"dX {e_gx:.2e} (ref SR spread {sr_gx:.2e}); dW {[f'{v:.2e}' for v in e_g]} "
          f"(ref SR spread {[f'{v:.2e}' for v in sr_g]})")
    assert bf16_y <= e_y + 1e-9
    assert e_y <= FAST_Y_BF16_FACTOR * bf16_y, (e_y, bf16_y)
    assert e_gx <= FAST_SR_FRACTION * sr_gx, (e_gx, sr_gx)
    for e, sr in zip(e_g, sr_g):
        assert e <= FAST_SR_FRACTION * sr, (e, sr)


def test_dx_gemm_chunked_raster_bit_identical():
    """The C3 dX GEMM shape (dG 8192 x 28672 K-major x W_gu 28672 x 4096 MN-major)
    takes the chunked-B raster (neither operand pinnable): bit-identical to the
    kGroupM-group raster (diag 1 << 27) in the exact epilogue, and within the
    FMA tolerance -- the raster only reorders whole tiles."""
    import torch
    from paper_2503_08040_b200 import fbq
    lib = fbq.K.lib
    lib.fbq_debug_set_gemm_diag.argtypes = [fbq.K.cint]
    M, N, K = 8192, 4096, 28672
    g = torch.Generator(device="cuda").manual_seed(3)
    qa = fbq.quantize_stochastic(torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16) * 1e-3, 5)
    qb = fbq.quantize_rtn(torch.randn(K, N, device="cuda", generator=g) * 0.02)
    outs = []
    try:
        for d in (0, 1 << 27):
            lib.fbq_debug_set_gemm_diag(d)
            outs.append(fbq.block_quant_gemm(qa, qb))
    finally:
        lib.fbq_debug_set_gemm_diag(0)
    assert torch.equal(outs[0].view(torch.int32), outs[1].view(torch.int32))
    fma = fbq.block_quant_gemm(qa, qb, exact=False)
    assert float((fma - outs[0]).norm() / outs[0].norm()) <= 1e-5


def test_c3_glublock_full_dims_exact_vs_reference(F, R, c3_weights):
    """The reference's GluBlock (RmsNorm + the C3 MLP + residual) at the full C3
    dims, exact mode, two training steps with SGD of the gain and the weights
    between them: out, grad_h, grad_gain and the gain bit-identical."""
    import torch
    from oracle.oracle import RefGluBlock
    from paper_2503_08040_b200 import linear
    wg, wu, wd = c3_weights
    ref = RefGluBlock(wg, wu, wd, threshold=8.0)
    blk = linear.GluBlock(wg, wu, wd, T, act_dtype=torch.float32, mid_dtype=torch.float32, exact=True,
                          threshold_init=8.0)
    for step in range(2):
        h, gout = _c3_inputs(10 + step)
        out_r, gh_r = ref.step(h, gout, step)
        out = host(blk.forward(dev(h), step))
        gh = host(blk.backward(dev(gout), step))
        assert np.array_equal(out.view(np.int32), out_r.view(np.int32)), (step, rel_fro(out, out_r))
        assert np.array_equal(gh.view(np.int32), gh_r.view(np.int32)), (step, rel_fro(gh, gh_r))
        gain_r, gg_r, _, _ = ref.state()
        gain, gg = blk.gain_host()
        assert np.array_equal(gg.view(np.int32), gg_r.view(np.int32)), step
        blk.controller_step()
        ref.controller()
        blk.apply_sgd(0.05)
        ref.apply_sgd(0.05)
        gain_r, _, _, _ = ref.state()
        assert np.array_equal(blk.gain_host()[0].view(np.int32), gain_r.view(np.int32)), step
