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
