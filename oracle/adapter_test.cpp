// TEST INFRASTRUCTURE: the reference-typed adapter (include/fbq_b200_reference_adapter.hpp)
// against the reference itself (oracle/_ref objects), on the same DenseMatrix
// inputs.  Prints "PASS n" / "FAIL ..." and exits non-zero on a mismatch.
// Built by `make -C oracle adapter_test`; run by tests/test_gpu_adapter.py.
#include <cstdio>
#include <cstring>
#include <vector>

#include "fbq/gemm.hpp"
#include "fbq/policy.hpp"
#include "fbq/quant.hpp"
#include "fbq/rng.hpp"
#include "fbq/trainsim.hpp"
#include "fbq_b200_reference_adapter.hpp"

using namespace fbq;

static int g_fail = 0, g_pass = 0;
static void check(bool ok, const char* what) {
  if (ok) ++g_pass;
  else {
    ++g_fail;
    std::printf("FAIL %s\n", what);
  }
}

static DenseMatrix randm(index_t r, index_t c, uint64_t seed, float scale, int outlier_col) {
  DeterministicRng rng(seed);
  std::vector<float> v(static_cast<size_t>(r * c));
  for (size_t i = 0; i < v.size(); ++i) v[i] = scale * rng.normal_at(i);
  if (outlier_col >= 0)
    for (index_t i = 0; i < r; ++i) v[i * c + outlier_col] *= 60.0f;
  return DenseMatrix(r, c, std::move(v));
}

static bool same_qt(const QuantizedTensor& a, const QuantizedTensor& b) {
  return a.rows == b.rows && a.cols == b.cols && a.codes == b.codes &&
         std::memcmp(a.scales.data(), b.scales.data(), a.scales.size() * 4) == 0;
}
static bool same_dense(const DenseMatrix& a, const DenseMatrix& b) {
  return a.rows() == b.rows() && a.cols() == b.cols() &&
         std::memcmp(a.data(), b.data(), a.size() * 4) == 0;
}

int main() {
  const GroupGeometry g(128, 128);
  const BitWidth b8(8);
  const GemmBlockShape shape(128, 128, 128);
  const index_t shapes[][3] = {{256, 384, 256}, {200, 300, 260}, {128, 128, 128}};
  for (const auto& s : shapes) {
    const index_t m = s[0], k = s[1], n = s[2];
    const DenseMatrix x = randm(m, k, 11 + m, 1.0f, 3);
    const DenseMatrix w = randm(k, n, 29 + n, 0.05f, -1);
    // quantizers
    check(same_qt(quantize_rtn(x, g, b8), b200::quantize_rtn(x, g, b8)), "quantize_rtn");
    const DeterministicRng rng(derive_seed(0x5eed, 5, 2));
    check(same_qt(quantize_stochastic(x, g, b8, rng), b200::quantize_stochastic(x, g, b8, rng)),
          "quantize_stochastic");
    const auto scores = score_blocks(x, g, b8, FallbackCriterion::AbsMax);
    check(scores == b200::score_blocks_absmax(x, g), "score_blocks");
    const auto mask = mask_topk(scores, 0.3);
    const FallbackTensor fr = fallback_quantize(x, g, b8, mask);
    const FallbackTensor fg = b200::fallback_quantize(x, g, b8, mask);
    bool res_ok = same_qt(fr.primary, fg.primary) && fr.mask == fg.mask &&
                  fr.residual_index == fg.residual_index &&
                  fr.residuals.size() == fg.residuals.size();
    for (size_t i = 0; res_ok && i < fr.residuals.size(); ++i)
      res_ok = fr.residuals[i].codes == fg.residuals[i].codes &&
               std::memcmp(&fr.residuals[i].scale, &fg.residuals[i].scale, 4) == 0;
    check(res_ok, "fallback_quantize");
    // GEMMs (reference orientation: B = quantize_rtn(W), K x N)
    const QuantizedTensor qa = quantize_rtn(x, g, b8);
    const QuantizedTensor qb = quantize_rtn(w, g, b8);
    check(same_dense(block_quant_gemm(qa, qb, shape), b200::block_quant_gemm(qa, qb, shape)),
          "block_quant_gemm");
    check(same_dense(fallback_gemm(fr, qb, shape), b200::fallback_gemm(fr, qb, shape)),
          "fallback_gemm");
  }
  // ---- dequantize / dequantize_fallback / transpose / tiled_block_gemm (quant.hpp:68-77, gemm.hpp:52-53)
  {
    const DenseMatrix x = randm(300, 270, 77, 1.0f, 5);
    const QuantizedTensor q = quantize_rtn(x, g, b8);
    check(same_dense(dequantize(q), b200::dequantize(q)), "dequantize");
    const auto mask = mask_topk(score_blocks(x, g, b8, FallbackCriterion::AbsMax), 0.5);
    const FallbackTensor f = fallback_quantize(x, g, b8, mask);
    check(same_dense(dequantize_fallback(f), b200::dequantize_fallback(f)), "dequantize_fallback");
    check(same_qt(transpose(q), b200::transpose(q)), "transpose");
    const QuantizedTensor qw = quantize_rtn(randm(270, 200, 78, 0.05f, -1), g, b8);
    for (const TileShape& t : {TileShape(128, 128, 128), TileShape(64, 32, 16), TileShape(1, 128, 8)})
      check(same_dense(tiled_block_gemm(q, qw, shape, t), b200::tiled_block_gemm(q, qw, shape, t)),
            "tiled_block_gemm");
    bool threw = false;
    try {
      b200::tiled_block_gemm(q, qw, shape, TileShape(48, 128, 128));
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    check(threw, "tiled_block_gemm bad tile");
  }
  // ---- policy: mask_threshold / mask_topk / mask_rate / controller_update (policy.hpp:30-47)
  {
    const DenseMatrix x = randm(640, 1152, 91, 1.0f, 300);
    const auto scores = score_blocks(x, g, b8, FallbackCriterion::AbsMax);
    for (double th : {0.5, 2.0, 3.5, 1e9})
      check(mask_threshold(scores, th) == b200::mask_threshold(scores, th), "mask_threshold");
    for (double r : {0.0, 0.01, 0.2, 0.5, 1.0})
      check(mask_topk(scores, r) == b200::mask_topk(scores, r), "mask_topk");
    std::vector<double> tied(91);
    for (size_t i = 0; i < tied.size(); ++i) tied[i] = static_cast<double>((i * 7) % 4) * 0.5;
    for (double r : {0.1, 0.33, 0.9}) check(mask_topk(tied, r) == b200::mask_topk(tied, r), "mask_topk ties");
    const auto m = mask_topk(scores, 0.2);
    check(mask_rate(m) == b200::mask_rate(m), "mask_rate");
    const ControllerConfig cc(0.1, 0.3, 1.3);
    for (double obs : {0.05, 0.2, 0.35}) {
      FallbackThresholdState st;
      st.threshold = 2.5;
      const auto a = controller_update(st, obs, cc), bb = b200::controller_update(st, obs, cc);
      check(a.threshold == bb.threshold && a.last_rate == bb.last_rate, "controller_update");
    }
  }
  // ---- QuantLinearLayer (trainsim.hpp:38-73) over steps with the controller and SGD
  {
    QuantConfig cfg;
    cfg.block = 128;
    cfg.threshold_init = 3.0;
    const DenseMatrix w = randm(384, 256, 55, 0.05f, -1);
    QuantLinearLayer ref("fc", 3, w, cfg);
    b200::QuantLinearLayer gpu("fc", 3, w, cfg, 512);
    bool ok = true;
    for (int step = 0; step < 3 && ok; ++step) {
      const DenseMatrix x = randm(300, 256, 60 + step, 1.0f, 7);
      const DenseMatrix gy = randm(300, 384, 70 + step, 1e-3f, -1);
      ref.zero_grad();
      gpu.zero_grad();
      ok = ok && same_dense(ref.forward(x, step), gpu.forward(x, step));
      ok = ok && ref.last_fallback_rate() == gpu.last_fallback_rate();
      ok = ok && same_dense(ref.backward(gy, step), gpu.backward(gy, step));
      ok = ok && same_dense(ref.grad_weight(), gpu.grad_weight());
      ref.controller_step();
      gpu.controller_step();
      ok = ok && ref.threshold() == gpu.threshold();
      ref.apply_sgd(0.5);
      gpu.apply_sgd(0.5);
      ok = ok && same_dense(ref.weight(), gpu.weight());
    }
    check(ok, "QuantLinearLayer fwd/bwd/grad/controller/sgd over 3 steps");
    bool threw = false;
    try {
      b200::QuantLinearLayer bad("fc", 0, w, QuantConfig{});  // reference default block = 32
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    check(threw, "QuantLinearLayer block = 32 unsupported");
    threw = false;
    try {
      b200::QuantLinearLayer fresh("fc", 0, w, cfg, 512);
      fresh.backward(randm(10, 384, 1, 1.0f, -1), 0);
    } catch (const std::logic_error&) {
      threw = true;
    }
    check(threw, "backward without context");
  }
  // ---- SiluLayer (trainsim.hpp:118-131)
  {
    QuantConfig cfg;
    SiluLayer ref(cfg);
    b200::SiluLayer gpu(cfg);
    const DenseMatrix x = randm(200, 384, 81, 2.0f, 5);
    const DenseMatrix gy = randm(200, 384, 82, 1e-2f, -1);
    bool ok = same_dense(ref.forward(x), gpu.forward(x));
    ok = ok && same_dense(ref.backward(gy), gpu.backward(gy));
    check(ok, "SiluLayer fwd/bwd");
  }
  // ---- GluBlock (trainsim.hpp:136-146) over steps with the controller and SGD
  {
    QuantConfig cfg;
    cfg.block = 128;
    cfg.threshold_init = 1.5;
    const index_t d = 256, f = 384;
    const DenseMatrix wg = randm(f, d, 91, 0.05f, -1), wu = randm(f, d, 92, 0.05f, -1), wd = randm(d, f, 93, 0.05f, -1);
    GluBlock ref{RmsNorm("norm", d, cfg), QuantLinearLayer("gate", 0, wg, cfg), QuantLinearLayer("up", 1, wu, cfg),
                 QuantLinearLayer("down", 2, wd, cfg), GluCombine(cfg)};
    b200::GluBlock gpu(wg, wu, wd, cfg, 512);
    bool ok = true;
    for (int step = 0; step < 3 && ok; ++step) {
      const DenseMatrix h = randm(300, d, 100 + step, 0.7f, 3);
      const DenseMatrix go = randm(300, d, 110 + step, 1e-2f, -1);
      ok = ok && same_dense(ref.forward(h, step), gpu.forward(h, step));
      ok = ok && same_dense(ref.backward(go, step), gpu.backward(go, step));
      ok = ok && ref.norm.grad_gain() == gpu.grad_gain();
      ok = ok && same_dense(ref.gate.grad_weight(), gpu.grad_weight(0)) &&
           same_dense(ref.down.grad_weight(), gpu.grad_weight(2));
      ref.gate.controller_step();
      ref.up.controller_step();
      ref.down.controller_step();
      gpu.controller_step();
      ok = ok && ref.gate.threshold() == gpu.threshold(0) && ref.down.threshold() == gpu.threshold(2);
      ref.norm.apply_sgd(0.05);
      ref.gate.apply_sgd(0.05);
      ref.up.apply_sgd(0.05);
      ref.down.apply_sgd(0.05);
      gpu.apply_sgd(0.05);
      ok = ok && ref.norm.gain() == gpu.gain() && same_dense(ref.up.weight(), gpu.weight(1));
    }
    check(ok, "GluBlock fwd/bwd/grads/controller/sgd over 3 steps");
  }
  // error behaviour mirrors the reference
  bool threw = false;
  try {
    b200::fallback_quantize(randm(128, 128, 1, 1, -1), g, b8, std::vector<uint8_t>(3, 0));
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  check(threw, "mask size error");
  threw = false;
  try {
    b200::quantize_rtn(randm(64, 64, 1, 1, -1), GroupGeometry(32, 32), b8);
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  check(threw, "unsupported geometry error");
  std::printf("%s %d passed, %d failed\n", g_fail ? "FAIL" : "PASS", g_pass, g_fail);
  return g_fail ? 1 : 0;
}
