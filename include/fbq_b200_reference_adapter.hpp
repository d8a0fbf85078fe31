// fbq_b200_reference_adapter.hpp -- the reference's own operator signatures on B200.
//
// Header-only adapter a maintainer of the reference library (/root/reference/proj,
// namespace fbq) adds to route its hot path to the sm_100a kernels: it takes and
// returns the reference's value types (DenseMatrix, QuantizedTensor,
// FallbackTensor; quant.hpp:23-57, matrix.hpp:15-36) and calls the C ABI of
// include/fbq_b200.h.  Semantics, argument meaning and error behaviour follow
// the reference (std::invalid_argument for shape / mask / bit-width errors); the
// B200 kernels cover 128 x 128 blocks at b = 8 and throw
// std::invalid_argument("...unsupported on B200...") otherwise, so a caller can
// keep other geometries on the CPU backend.
//
// Requires the reference headers on the include path (fbq/quant.hpp,
// fbq/gemm.hpp, fbq/policy.hpp, fbq/rng.hpp) and linking lib/libfbq_b200.so.
// Exercised by oracle/adapter_test.cpp against the reference itself.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "fbq/gemm.hpp"
#include "fbq/matrix.hpp"
#include "fbq/policy.hpp"
#include "fbq/quant.hpp"
#include "fbq/rng.hpp"
#include "fbq/trainsim.hpp"
#include "fbq_b200.h"
#include "fbq_b200_host.h"

namespace fbq::b200 {

namespace detail {

inline void check(int st, const char* what) {
  if (st == FBQ_OK) return;
  const std::string msg = std::string(what) + ": " + fbq_status_string(st);
  if (st == FBQ_ERR_CUDA) throw std::runtime_error(msg);
  throw std::invalid_argument(msg);
}

// RAII device buffer through the C ABI (no CUDA runtime needed here)
struct Dev {
  void* p = nullptr;
  explicit Dev(size_t bytes) { check(fbq_malloc(&p, bytes), "fbq_malloc"); }
  ~Dev() { fbq_free(p); }
  Dev(const Dev&) = delete;
  Dev& operator=(const Dev&) = delete;
  template <class T>
  T* as() const { return static_cast<T*>(p); }
};

inline int64_t ld16(int64_t n) { return (n + 15) / 16 * 16; }
inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

inline void require_b200(const GroupGeometry& g, BitWidth b) {
  if (g.group_rows != 128 || g.group_cols != 128 || b.bits != 8)
    throw std::invalid_argument("geometry/bit-width unsupported on B200 (128x128 blocks, 8 bits)");
}

// host DenseMatrix -> device fp32
inline void upload(const DenseMatrix& m, const Dev& d) {
  check(fbq_memcpy_h2d(d.p, m.data(), m.size() * sizeof(float)), "upload");
}

// host int16 codes (rows x cols) -> device int8 plane (rows x ldq)
inline void upload_codes(const std::vector<int16_t>& c, int64_t rows, int64_t cols, int64_t ldq,
                         const Dev& d) {
  std::vector<int8_t> h(static_cast<size_t>(rows * ldq), 0);
  for (int64_t r = 0; r < rows; ++r)
    for (int64_t j = 0; j < cols; ++j) h[r * ldq + j] = static_cast<int8_t>(c[r * cols + j]);
  check(fbq_memcpy_h2d(d.p, h.data(), h.size()), "upload_codes");
}

inline std::vector<int16_t> download_codes(const Dev& d, int64_t rows, int64_t cols, int64_t ldq) {
  std::vector<int8_t> h(static_cast<size_t>(rows * ldq));
  check(fbq_memcpy_d2h(h.data(), d.p, h.size()), "download_codes");
  std::vector<int16_t> c(static_cast<size_t>(rows * cols));
  for (int64_t r = 0; r < rows; ++r)
    for (int64_t j = 0; j < cols; ++j) c[r * cols + j] = h[r * ldq + j];
  return c;
}

inline std::vector<float> download_f32(const Dev& d, size_t n) {
  std::vector<float> v(n);
  check(fbq_memcpy_d2h(v.data(), d.p, n * sizeof(float)), "download");
  return v;
}

inline QuantizedTensor make_qt(int64_t rows, int64_t cols, std::vector<int16_t> codes,
                               std::vector<float> scales) {
  QuantizedTensor q;
  q.rows = rows;
  q.cols = cols;
  q.geometry = GroupGeometry(128, 128);
  q.bits = BitWidth(8);
  q.codes = std::move(codes);
  q.scales = std::move(scales);
  return q;
}

}  // namespace detail

// quant.cpp:36-53
inline QuantizedTensor quantize_rtn(const DenseMatrix& m, const GroupGeometry& g, BitWidth b) {
  detail::require_b200(g, b);
  const int64_t r = m.rows(), c = m.cols(), ldq = detail::ld16(c);
  const int64_t nb = detail::cdiv(r, 128) * detail::cdiv(c, 128);
  detail::Dev x(r * c * 4), codes(r * ldq), scales(nb * 4);
  detail::upload(m, x);
  detail::check(fbq_cuda_quantize_rtn(x.p, FBQ_F32, r, c, c, codes.as<int8_t>(), ldq,
                                      scales.as<float>(), nullptr),
                "quantize_rtn");
  return detail::make_qt(r, c, detail::download_codes(codes, r, c, ldq),
                         detail::download_f32(scales, nb));
}

// quant.cpp:55-84
inline QuantizedTensor quantize_stochastic(const DenseMatrix& m, const GroupGeometry& g,
                                           BitWidth b, const DeterministicRng& rng) {
  detail::require_b200(g, b);
  const int64_t r = m.rows(), c = m.cols(), ldq = detail::ld16(c);
  const int64_t nb = detail::cdiv(r, 128) * detail::cdiv(c, 128);
  detail::Dev x(r * c * 4), codes(r * ldq), scales(nb * 4);
  detail::upload(m, x);
  detail::check(fbq_cuda_quantize_stochastic(x.p, FBQ_F32, r, c, c, rng.seed(), 0,
                                             codes.as<int8_t>(), ldq, scales.as<float>(), nullptr),
                "quantize_stochastic");
  return detail::make_qt(r, c, detail::download_codes(codes, r, c, ldq),
                         detail::download_f32(scales, nb));
}

// quant.cpp:128-176 (residuals in the reference's compact order)
inline FallbackTensor fallback_quantize(const DenseMatrix& m, const GroupGeometry& g, BitWidth b,
                                        const std::vector<uint8_t>& mask) {
  detail::require_b200(g, b);
  const int64_t r = m.rows(), c = m.cols(), ldq = detail::ld16(c);
  const int64_t gr = detail::cdiv(r, 128), gc = detail::cdiv(c, 128), nb = gr * gc;
  if (mask.size() != static_cast<size_t>(nb))
    throw std::invalid_argument("fallback mask does not match the block grid");  // quant.cpp:132
  std::vector<uint32_t> bits(static_cast<size_t>(detail::cdiv(nb, 32)), 0);
  for (int64_t i = 0; i < nb; ++i)
    if (mask[i]) bits[i >> 5] |= 1u << (i & 31);
  detail::Dev x(r * c * 4), codes(r * ldq), scales(nb * 4), res(r * ldq), rscales(nb * 4),
      dbits(bits.size() * 4);
  detail::upload(m, x);
  detail::check(fbq_memcpy_h2d(dbits.p, bits.data(), bits.size() * 4), "upload mask");
  detail::check(fbq_cuda_quantize_fallback(x.p, FBQ_F32, r, c, c, FBQ_MASK_GIVEN, 1.0,
                                           dbits.as<uint32_t>(), codes.as<int8_t>(), ldq,
                                           scales.as<float>(), res.as<int8_t>(),
                                           rscales.as<float>(), nullptr, nullptr, nullptr, 0, 0,
                                           nullptr),
                "fallback_quantize");
  FallbackTensor f;
  f.primary = detail::make_qt(r, c, detail::download_codes(codes, r, c, ldq),
                              detail::download_f32(scales, nb));
  f.mask = mask;
  f.residual_index.assign(static_cast<size_t>(nb), -1);
  const std::vector<int16_t> rc = detail::download_codes(res, r, c, ldq);
  const std::vector<float> rs = detail::download_f32(rscales, nb);
  for (int64_t bi = 0; bi < gr; ++bi)
    for (int64_t bj = 0; bj < gc; ++bj) {
      if (!mask[bi * gc + bj]) continue;
      const int64_t er = std::min<int64_t>(128, r - bi * 128), ec = std::min<int64_t>(128, c - bj * 128);
      FallbackTensor::Residual blk;
      blk.codes.resize(static_cast<size_t>(er * ec));
      for (int64_t i = 0; i < er; ++i)
        for (int64_t j = 0; j < ec; ++j)
          blk.codes[i * ec + j] = rc[(bi * 128 + i) * c + bj * 128 + j];
      blk.scale = rs[bi * gc + bj];
      f.residual_index[bi * gc + bj] = static_cast<int32_t>(f.residuals.size());
      f.residuals.push_back(std::move(blk));
    }
  return f;
}

namespace detail {
// gemm.cpp:78-95 checks + the K3 launch (exact epilogue: bit-identical output)
inline DenseMatrix run_gemm(const QuantizedTensor& qa, const QuantizedTensor& qb,
                            const GemmBlockShape& shape, const FallbackTensor* fb) {
  if (qa.cols != qb.rows) throw std::invalid_argument("block gemm: inner dimensions differ");
  if (shape.m_g != 128 || shape.n_g != 128 || shape.k_g != 128 || qa.bits.bits != 8 ||
      qb.bits.bits != 8 || !(qa.geometry == GroupGeometry(128, 128)) ||
      !(qb.geometry == GroupGeometry(128, 128)))
    throw std::invalid_argument("block shape/geometry unsupported on B200 (128^3, 8 bits)");
  check(fbq_cuda_init(), "fbq_cuda_init");  // once per device (idempotent): dynamic tile scheduler
  const int64_t M = qa.rows, K = qa.cols, N = qb.cols;
  const int64_t lda = ld16(K), ldb = ld16(N);
  Dev a(M * lda + 16), b(K * ldb + 16), sa(qa.scales.size() * 4 + 4), sb(qb.scales.size() * 4 + 4),
      out(M * N * 4 + 4);
  upload_codes(qa.codes, M, K, lda, a);
  upload_codes(qb.codes, K, N, ldb, b);
  check(fbq_memcpy_h2d(sa.p, qa.scales.data(), qa.scales.size() * 4), "upload");
  check(fbq_memcpy_h2d(sb.p, qb.scales.data(), qb.scales.size() * 4), "upload");
  std::unique_ptr<Dev> bits, res, rs;
  if (fb) {
    const int64_t nb = cdiv(M, 128) * cdiv(K, 128);
    if (fb->mask.size() != static_cast<size_t>(nb))
      throw std::invalid_argument("fallback mask does not match the A block grid");
    std::vector<uint32_t> hb(static_cast<size_t>(cdiv(nb, 32)), 0);
    std::vector<int16_t> dense(static_cast<size_t>(M * K), 0);
    std::vector<float> hs(static_cast<size_t>(nb), 0.0f);
    const int64_t gc = cdiv(K, 128);
    for (int64_t i = 0; i < nb; ++i) {
      if (!fb->mask[i]) continue;
      hb[i >> 5] |= 1u << (i & 31);
      const auto& blk = fb->residuals[fb->residual_index[i]];
      const int64_t bi = i / gc, bj = i % gc;
      const int64_t er = std::min<int64_t>(128, M - bi * 128), ec = std::min<int64_t>(128, K - bj * 128);
      for (int64_t r = 0; r < er; ++r)
        for (int64_t c = 0; c < ec; ++c) dense[(bi * 128 + r) * K + bj * 128 + c] = blk.codes[r * ec + c];
      hs[i] = blk.scale;
    }
    bits = std::make_unique<Dev>(hb.size() * 4);
    res = std::make_unique<Dev>(M * lda + 16);
    rs = std::make_unique<Dev>(hs.size() * 4);
    check(fbq_memcpy_h2d(bits->p, hb.data(), hb.size() * 4), "upload");
    upload_codes(dense, M, K, lda, *res);
    check(fbq_memcpy_h2d(rs->p, hs.data(), hs.size() * 4), "upload");
  }
  check(fbq_cuda_gemm(a.as<int8_t>(), lda, sa.as<float>(), FBQ_K_MAJOR, b.as<int8_t>(), ldb,
                      sb.as<float>(), FBQ_MN_MAJOR, fb ? bits->as<uint32_t>() : nullptr,
                      fb ? res->as<int8_t>() : nullptr, fb ? rs->as<float>() : nullptr, M, N, K,
                      out.p, FBQ_F32, N, 0, FBQ_EPI_EXACT, nullptr),
        "block gemm");
  return DenseMatrix(M, N, download_f32(out, static_cast<size_t>(M * N)));
}
}  // namespace detail

// gemm.cpp:190-193
inline DenseMatrix block_quant_gemm(const QuantizedTensor& qa, const QuantizedTensor& qb,
                                    const GemmBlockShape& shape) {
  return detail::run_gemm(qa, qb, shape, nullptr);
}

// gemm.cpp:195-198 (Algorithm 1)
inline DenseMatrix fallback_gemm(const FallbackTensor& fa, const QuantizedTensor& qb,
                                 const GemmBlockShape& shape) {
  return detail::run_gemm(fa.primary, qb, shape, &fa);
}

// policy.cpp:12-28 (AbsMax criterion)
inline std::vector<double> score_blocks_absmax(const DenseMatrix& m, const GroupGeometry& g) {
  detail::require_b200(g, BitWidth(8));
  const int64_t r = m.rows(), c = m.cols();
  const int64_t nb = detail::cdiv(r, 128) * detail::cdiv(c, 128);
  detail::Dev x(r * c * 4), amax(nb * 4);
  detail::upload(m, x);
  detail::check(fbq_cuda_block_absmax(x.p, FBQ_F32, r, c, c, amax.as<float>(), nullptr),
                "score_blocks");
  const std::vector<float> f = detail::download_f32(amax, nb);
  return std::vector<double>(f.begin(), f.end());
}

// ------------------------------------------------------------------ quant.hpp:68-77
namespace detail {
inline DenseMatrix run_dequant(const QuantizedTensor& q, const FallbackTensor* fb) {
  if (!(q.geometry == GroupGeometry(128, 128)) || q.bits.bits != 8)
    throw std::invalid_argument("geometry/bit-width unsupported on B200 (128x128 blocks, 8 bits)");
  const int64_t r = q.rows, c = q.cols, ldq = ld16(c);
  const int64_t gc = cdiv(c, 128), nb = cdiv(r, 128) * gc;
  Dev codes(r * ldq + 16), scales(nb * 4 + 4), out(r * c * 4 + 4);
  upload_codes(q.codes, r, c, ldq, codes);
  check(fbq_memcpy_h2d(scales.p, q.scales.data(), q.scales.size() * 4), "upload");
  std::unique_ptr<Dev> bits, res, rs;
  if (fb) {
    if (fb->mask.size() != static_cast<size_t>(nb))
      throw std::invalid_argument("fallback mask does not match the block grid");
    std::vector<uint32_t> hb(static_cast<size_t>(cdiv(nb, 32)), 0);
    std::vector<int16_t> dense(static_cast<size_t>(r * c), 0);
    std::vector<float> hs(static_cast<size_t>(nb), 0.0f);
    for (int64_t i = 0; i < nb; ++i) {
      if (!fb->mask[i]) continue;
      hb[i >> 5] |= 1u << (i & 31);
      const auto& blk = fb->residuals[fb->residual_index[i]];
      const int64_t bi = i / gc, bj = i % gc;
      const int64_t er = std::min<int64_t>(128, r - bi * 128), ec = std::min<int64_t>(128, c - bj * 128);
      for (int64_t y = 0; y < er; ++y)
        for (int64_t x = 0; x < ec; ++x) dense[(bi * 128 + y) * c + bj * 128 + x] = blk.codes[y * ec + x];
      hs[i] = blk.scale;
    }
    bits = std::make_unique<Dev>(hb.size() * 4);
    res = std::make_unique<Dev>(r * ldq + 16);
    rs = std::make_unique<Dev>(hs.size() * 4);
    check(fbq_memcpy_h2d(bits->p, hb.data(), hb.size() * 4), "upload");
    upload_codes(dense, r, c, ldq, *res);
    check(fbq_memcpy_h2d(rs->p, hs.data(), hs.size() * 4), "upload");
  }
  check(fbq_cuda_dequantize(codes.as<int8_t>(), ldq, scales.as<float>(), fb ? bits->as<uint32_t>() : nullptr,
                            fb ? res->as<int8_t>() : nullptr, fb ? rs->as<float>() : nullptr, r, c,
                            out.as<float>(), c, nullptr),
        "dequantize");
  return DenseMatrix(r, c, download_f32(out, static_cast<size_t>(r * c)));
}
}  // namespace detail

// quant.cpp:86-104
inline DenseMatrix dequantize(const QuantizedTensor& q) { return detail::run_dequant(q, nullptr); }

// quant.cpp:178-202
inline DenseMatrix dequantize_fallback(const FallbackTensor& f) { return detail::run_dequant(f.primary, &f); }

// quant.cpp:106-126.  The B200 path never materialises a transpose: the GEMM
// reads the same int8 plane K- or MN-major through a descriptor bit (quantize
// W once; dgrad/wgrad read it transposed).  For value-API callers this is the
// reference's data movement on the host: codes and the scale grid transposed.
inline QuantizedTensor transpose(const QuantizedTensor& q) {
  if (!(q.geometry == GroupGeometry(128, 128)) || q.bits.bits != 8)
    throw std::invalid_argument("geometry/bit-width unsupported on B200 (128x128 blocks, 8 bits)");
  const int64_t r = q.rows, c = q.cols, gr = detail::cdiv(r, 128), gc = detail::cdiv(c, 128);
  std::vector<int16_t> codes(static_cast<size_t>(r * c));
  for (int64_t i = 0; i < r; ++i)
    for (int64_t j = 0; j < c; ++j) codes[j * r + i] = q.codes[i * c + j];
  std::vector<float> scales(static_cast<size_t>(gr * gc));
  for (int64_t i = 0; i < gr; ++i)
    for (int64_t j = 0; j < gc; ++j) scales[j * gr + i] = q.scales[i * gc + j];
  return detail::make_qt(c, r, std::move(codes), std::move(scales));
}

// gemm.cpp:200-203: any tile dividing the block is bit-identical to the block
// GEMM (integer tile products are associative; the tensor core always forms
// the full 128-deep block product with K = 32 sub-steps)
inline DenseMatrix tiled_block_gemm(const QuantizedTensor& qa, const QuantizedTensor& qb,
                                    const GemmBlockShape& shape, const TileShape& tile) {
  if (shape.m_g % tile.m_t || shape.n_g % tile.n_t || shape.k_g % tile.k_t)
    throw std::invalid_argument("tile sides must divide the block sides");  // gemm.cpp:104-107
  return detail::run_gemm(qa, qb, shape, nullptr);
}

// ------------------------------------------------------------------ policy.hpp:30-47
namespace detail {
inline std::vector<uint8_t> bits_to_mask(const std::vector<uint32_t>& bits, size_t n) {
  std::vector<uint8_t> m(n);
  for (size_t i = 0; i < n; ++i) m[i] = static_cast<uint8_t>((bits[i >> 5] >> (i & 31)) & 1u);
  return m;
}
}  // namespace detail

// policy.cpp:73-80 (strict >) on the device
inline std::vector<uint8_t> mask_threshold(const std::vector<double>& scores, double threshold) {
  if (!(threshold > 0.0)) throw std::invalid_argument("threshold must be > 0");  // policy.cpp:74
  const int64_t n = static_cast<int64_t>(scores.size());
  if (n == 0) return {};
  detail::Dev s(n * 8), bits(detail::cdiv(n, 32) * 4);
  detail::check(fbq_memcpy_h2d(s.p, scores.data(), n * 8), "upload");
  detail::check(fbq_cuda_mask_threshold(s.as<double>(), n, threshold, bits.as<uint32_t>(), nullptr, nullptr),
                "mask_threshold");
  std::vector<uint32_t> hb(static_cast<size_t>(detail::cdiv(n, 32)));
  detail::check(fbq_memcpy_d2h(hb.data(), bits.p, hb.size() * 4), "download");
  return detail::bits_to_mask(hb, static_cast<size_t>(n));
}

// policy.cpp:56-71 on the device (one-CTA radix select, ties to the lower
// index).  The device keys are fp32 scores: AbsMax scores are fp32 block
// maxima widened to double (policy.cpp:18-27), so this is exact for them; other
// criteria (L1 / L1Rel doubles) throw "unsupported on B200".
inline std::vector<uint8_t> mask_topk(const std::vector<double>& scores, double rate) {
  if (!(rate >= 0.0 && rate <= 1.0)) throw std::invalid_argument("rate must be in [0, 1]");  // policy.cpp:57
  const int64_t n = static_cast<int64_t>(scores.size());
  if (n == 0) return {};
  std::vector<float> f(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) {
    f[i] = static_cast<float>(scores[i]);
    if (static_cast<double>(f[i]) != scores[i] || !(scores[i] >= 0.0))
      throw std::invalid_argument("mask_topk: non-fp32 or negative scores unsupported on B200 (AbsMax only)");
  }
  detail::Dev s(n * 4), bits(detail::cdiv(n, 32) * 4);
  detail::check(fbq_memcpy_h2d(s.p, f.data(), n * 4), "upload");
  detail::check(fbq_cuda_mask_topk(s.as<float>(), n, rate, bits.as<uint32_t>(), nullptr, nullptr), "mask_topk");
  std::vector<uint32_t> hb(static_cast<size_t>(detail::cdiv(n, 32)));
  detail::check(fbq_memcpy_d2h(hb.data(), bits.p, hb.size() * 4), "download");
  return detail::bits_to_mask(hb, static_cast<size_t>(n));
}

// policy.cpp:82-87 (flagged / blocks: a host count over the caller's host mask;
// on the device the same count comes out of K1 / the mask kernels)
inline double mask_rate(const std::vector<uint8_t>& mask) {
  if (mask.empty()) return 0.0;
  size_t k = 0;
  for (uint8_t m : mask) k += m ? 1 : 0;
  return static_cast<double>(k) / static_cast<double>(mask.size());
}

// policy.cpp:97-109 (Algorithm 2) through the device controller
inline FallbackThresholdState controller_update(FallbackThresholdState state, double observed_rate,
                                                const ControllerConfig& cfg) {
  if (!(observed_rate >= 0.0 && observed_rate <= 1.0))
    throw std::invalid_argument("observed rate must be in [0, 1]");  // policy.cpp:98-100
  detail::Dev d(3 * sizeof(double));
  const double h[3] = {state.threshold, observed_rate, 0.0};
  detail::check(fbq_memcpy_h2d(d.p, h, sizeof(h)), "upload");
  detail::check(fbq_cuda_controller_update_rate(d.as<double>(), d.as<double>() + 1, cfg.r_min, cfg.r_max,
                                                cfg.alpha, d.as<double>() + 2, nullptr),
                "controller_update");
  double o[3];
  detail::check(fbq_memcpy_d2h(o, d.p, sizeof(o)), "download");
  FallbackThresholdState out;
  out.threshold = o[0];
  out.last_rate = o[2];
  return out;
}

// ------------------------------------------------------------------ trainsim.hpp:38-73
// QuantLinearLayer on the device driver (fbq_linear_*): the same constructor
// arguments and methods; forward/backward take and return host DenseMatrix
// values like the reference (the e2e value API: host -> device -> host).  The
// B200 path covers QuantConfig{block = 128, 8-bit x / w / grad / context,
// not passthrough}; anything else throws std::invalid_argument("...unsupported
// on B200...") -- in particular the reference's DEFAULT block = 32.
// max_tokens sizes the device workspaces (forward rows beyond it throw).
class QuantLinearLayer {
 public:
  QuantLinearLayer(std::string name, int layer_id, DenseMatrix weight, QuantConfig cfg,
                   index_t max_tokens = 4096)
      : name_(std::move(name)), out_(weight.rows()), in_(weight.cols()) {
    if (cfg.passthrough || cfg.block != 128 || cfg.bits_x != 8 || cfg.bits_w != 8 || cfg.bits_grad != 8 ||
        cfg.context_bits != 8)
      throw std::invalid_argument(
          "QuantConfig unsupported on B200 (needs block = 128, 8-bit x/w/grad/context, not passthrough)");
    fbq_linear_config c;
    fbq_linear_default_config(&c);
    c.in_features = in_;
    c.out_features = out_;
    c.max_tokens = max_tokens;
    c.act_dtype = FBQ_F32;
    c.epilogue = FBQ_EPI_EXACT;  // bit-exact with the reference
    c.layer_id = layer_id;
    c.seed = cfg.seed;
    c.threshold_init = cfg.threshold_init;
    c.r_min = cfg.controller.r_min;
    c.r_max = cfg.controller.r_max;
    c.alpha = cfg.controller.alpha;
    c.fallback_mode = cfg.fallback_mode == FallbackMode::Threshold ? 0
                      : cfg.fallback_mode == FallbackMode::FixedRate ? 1 : 2;
    c.fixed_rate = cfg.fixed_rate;
    h_ = fbq_linear_create(&c, weight.data());
    if (!h_) throw std::invalid_argument(std::string("fbq_linear_create: ") + fbq_host_last_error());
    max_tokens_ = max_tokens;
  }
  ~QuantLinearLayer() {
    if (h_) fbq_linear_destroy(h_);
  }
  QuantLinearLayer(const QuantLinearLayer&) = delete;
  QuantLinearLayer& operator=(const QuantLinearLayer&) = delete;

  DenseMatrix forward(const DenseMatrix& x, int step) {
    if (x.cols() != in_) throw std::invalid_argument("forward: input width != in_features");
    return run(x, out_, step, true);
  }
  // returns grad_x, accumulates grad_w (trainsim.cpp:106-127)
  DenseMatrix backward(const DenseMatrix& grad_y, int step) {
    if (grad_y.cols() != out_) throw std::invalid_argument("backward: grad width != out_features");
    if (!has_ctx_) throw std::logic_error("backward without a forward context");  // trainsim.cpp:108
    return run(grad_y, in_, step, false);
  }
  const std::string& name() const { return name_; }
  DenseMatrix weight() const { return host_copy(fbq_linear_get_weight); }
  DenseMatrix grad_weight() const { return host_copy(fbq_linear_get_grad); }
  double last_fallback_rate() const { return controller_state().first; }
  double threshold() const { return controller_state().second; }
  bool holds_full_precision_context() const { return false; }  // the int8 SR context only
  void controller_step() { detail::check(fbq_linear_controller_step(h_, nullptr), "controller_step"); }
  void zero_grad() { detail::check(fbq_linear_zero_grad(h_, nullptr), "zero_grad"); }
  void apply_sgd(double lr) { detail::check(fbq_linear_apply_sgd(h_, lr, nullptr), "apply_sgd"); }

 private:
  DenseMatrix run(const DenseMatrix& in, int64_t out_cols, int step, bool fwd) {
    const int64_t t = in.rows();
    if (t > max_tokens_) throw std::invalid_argument("tokens exceed max_tokens of the B200 layer");
    detail::Dev di(t * in.cols() * 4 + 4), dout(t * out_cols * 4 + 4);
    detail::upload(in, di);
    const int st = fwd ? fbq_linear_forward_device(h_, di.p, t, 0, step, dout.p, nullptr)
                       : fbq_linear_backward_device(h_, di.p, t, 0, step, dout.p, nullptr);
    detail::check(st, fwd ? "forward" : "backward");
    if (fwd) has_ctx_ = true;
    return DenseMatrix(t, out_cols, detail::download_f32(dout, static_cast<size_t>(t * out_cols)));
  }
  DenseMatrix host_copy(int (*fn)(void*, float*)) const {
    std::vector<float> v(static_cast<size_t>(out_ * in_));
    detail::check(fn(h_, v.data()), "copy");
    return DenseMatrix(out_, in_, std::move(v));
  }
  std::pair<double, double> controller_state() const {
    double r = 0.0, th = 0.0;
    detail::check(fbq_linear_get_controller(h_, &r, &th), "get_controller");
    return {r, th};
  }
  std::string name_;
  int64_t out_, in_;
  index_t max_tokens_ = 0;
  void* h_ = nullptr;
  bool has_ctx_ = false;
};

// ------------------------------------------------------------------ trainsim.hpp:118-131
// SiluLayer on the device (fbq_cuda_silu_*): y = silu(x) with the input kept as
// its nonlinear_bits 1 x nonlinear_group RTN context; backward from that context.
// Exact math (the reference's double silu / silu').  Needs nonlinear_group = 128,
// 2..16 bits, not passthrough; cols % 8 == 0.
class SiluLayer {
 public:
  explicit SiluLayer(QuantConfig cfg) : bits_(cfg.nonlinear_bits) {
    if (cfg.passthrough || cfg.nonlinear_bits == 0 || cfg.nonlinear_group != 128)
      throw std::invalid_argument("SiluLayer config unsupported on B200 (10-bit 1 x 128 context)");
  }
  DenseMatrix forward(const DenseMatrix& x) {
    rows_ = x.rows();
    cols_ = x.cols();
    ld_ = detail::ld16(cols_);
    dx_ = std::make_unique<detail::Dev>(rows_ * cols_ * 4 + 4);
    dy_ = std::make_unique<detail::Dev>(rows_ * cols_ * 4 + 4);
    ctx_ = std::make_unique<detail::Dev>(rows_ * ld_ * 2 + 4);
    sc_ = std::make_unique<detail::Dev>(rows_ * detail::cdiv(cols_, 128) * 4 + 4);
    detail::upload(x, *dx_);
    detail::check(fbq_cuda_silu_forward(dx_->p, FBQ_F32, rows_, cols_, cols_, dy_->p, cols_, ctx_->as<int16_t>(),
                                        ld_, sc_->as<float>(), bits_, 1, nullptr),
                  "silu forward");
    return DenseMatrix(rows_, cols_, detail::download_f32(*dy_, static_cast<size_t>(rows_ * cols_)));
  }
  DenseMatrix backward(const DenseMatrix& grad_y) {
    if (!ctx_) throw std::logic_error("silu: backward without context");  // trainsim.cpp:280-282
    if (grad_y.rows() != rows_ || grad_y.cols() != cols_) throw std::invalid_argument("silu: grad shape");
    detail::upload(grad_y, *dx_);
    detail::check(fbq_cuda_silu_backward(ctx_->as<int16_t>(), ld_, sc_->as<float>(), dx_->p, FBQ_F32, rows_, cols_,
                                         cols_, dy_->p, cols_, 1, nullptr),
                  "silu backward");
    return DenseMatrix(rows_, cols_, detail::download_f32(*dy_, static_cast<size_t>(rows_ * cols_)));
  }
  bool holds_full_precision_context() const { return false; }

 private:
  int bits_;
  int64_t rows_ = 0, cols_ = 0, ld_ = 0;
  std::unique_ptr<detail::Dev> dx_, dy_, ctx_, sc_;
};

// ------------------------------------------------------------------ trainsim.hpp:136-146
// GluBlock on the device driver (fbq_glublock_*): h + down(silu(gate(norm(h))) *
// up(norm(h))) with the reference's layer ids (gate 0, up 1, down 2 from
// layer_id_base), forward / backward over host DenseMatrix values.  The
// reference's GluBlock is an aggregate of its layers; their state is reached
// here through the accessors below (which: 0 gate, 1 up, 2 down).  Same config
// rules as QuantLinearLayer (block = 128, 8-bit operands, 10-bit contexts).
class GluBlock {
 public:
  GluBlock(const DenseMatrix& w_gate, const DenseMatrix& w_up, const DenseMatrix& w_down, QuantConfig cfg,
           index_t max_tokens = 4096, int layer_id_base = 0)
      : d_(w_gate.cols()), f_(w_gate.rows()), max_tokens_(max_tokens) {
    if (cfg.passthrough || cfg.block != 128 || cfg.bits_x != 8 || cfg.bits_w != 8 || cfg.bits_grad != 8 ||
        cfg.context_bits != 8 || cfg.nonlinear_group != 128 || cfg.nonlinear_bits != 10 ||
        cfg.fallback_mode != FallbackMode::Threshold)
      throw std::invalid_argument("QuantConfig unsupported on B200 GluBlock (block 128, 8-bit, 10-bit contexts, "
                                  "threshold fallback)");
    fbq_mlp_config c;
    fbq_mlp_default_config(&c);
    c.d_model = d_;
    c.d_ff = f_;
    c.max_tokens = max_tokens;
    c.act_dtype = FBQ_F32;
    c.mid_dtype = FBQ_F32;
    c.epilogue = FBQ_EPI_EXACT;  // bit-exact with the reference
    c.layer_id_base = layer_id_base;
    c.seed = cfg.seed;
    c.threshold_init = cfg.threshold_init;
    c.r_min = cfg.controller.r_min;
    c.r_max = cfg.controller.r_max;
    c.alpha = cfg.controller.alpha;
    b_ = fbq_glublock_create(&c, w_gate.data(), w_up.data(), w_down.data());
    if (!b_) throw std::invalid_argument(std::string("fbq_glublock_create: ") + fbq_host_last_error());
  }
  ~GluBlock() {
    if (b_) fbq_glublock_destroy(b_);
  }
  GluBlock(const GluBlock&) = delete;
  GluBlock& operator=(const GluBlock&) = delete;

  DenseMatrix forward(const DenseMatrix& h, int step) { return run(h, step, true); }
  DenseMatrix backward(const DenseMatrix& grad_out, int step) {
    if (!has_ctx_) throw std::logic_error("GluBlock: backward without context");
    return run(grad_out, step, false);
  }
  void zero_grads() { detail::check(fbq_glublock_zero_grad(b_, nullptr), "zero_grad"); }
  void controller_step() { detail::check(fbq_mlp_controller_step(fbq_glublock_mlp(b_), nullptr), "controller"); }
  void apply_sgd(double lr) { detail::check(fbq_glublock_apply_sgd(b_, lr, nullptr), "apply_sgd"); }
  std::vector<float> gain() const { return gains().first; }
  std::vector<float> grad_gain() const { return gains().second; }
  DenseMatrix weight(int which) const { return mats(which, false); }
  DenseMatrix grad_weight(int which) const { return mats(which, true); }
  // thresholds of gate / up (shared: same input, same controller) and down
  double threshold(int which) const {
    double rates[2], th[2];
    detail::check(fbq_mlp_get_controller(fbq_glublock_mlp(b_), rates, th), "get_controller");
    return th[which == 2 ? 1 : 0];
  }

 private:
  DenseMatrix run(const DenseMatrix& in, int step, bool fwd) {
    const int64_t t = in.rows();
    if (in.cols() != d_) throw std::invalid_argument("GluBlock: width != d_model");
    if (t > max_tokens_) throw std::invalid_argument("tokens exceed max_tokens of the B200 block");
    detail::Dev di(t * d_ * 4 + 4), dout(t * d_ * 4 + 4);
    detail::upload(in, di);
    const int st = fwd ? fbq_glublock_forward_device(b_, di.p, t, 0, step, dout.p, nullptr)
                       : fbq_glublock_backward_device(b_, di.p, t, 0, step, dout.p, nullptr);
    detail::check(st, fwd ? "GluBlock forward" : "GluBlock backward");
    if (fwd) has_ctx_ = true;
    return DenseMatrix(t, d_, detail::download_f32(dout, static_cast<size_t>(t * d_)));
  }
  std::pair<std::vector<float>, std::vector<float>> gains() const {
    std::vector<float> g(static_cast<size_t>(d_)), gg(static_cast<size_t>(d_));
    detail::check(fbq_glublock_get_gain(b_, g.data(), gg.data()), "get_gain");
    return {std::move(g), std::move(gg)};
  }
  DenseMatrix mats(int which, bool grads) const {
    std::vector<float> a(static_cast<size_t>(d_ * f_)), b(a.size()), c(a.size());
    void* m = fbq_glublock_mlp(b_);
    detail::check(grads ? fbq_mlp_get_grads(m, a.data(), b.data(), c.data())
                        : fbq_mlp_get_weights(m, a.data(), b.data(), c.data()),
                  "copy");
    if (which == 2) return DenseMatrix(d_, f_, std::move(c));
    return DenseMatrix(f_, d_, std::move(which == 0 ? a : b));
  }
  int64_t d_, f_;
  index_t max_tokens_;
  void* b_ = nullptr;
  bool has_ctx_ = false;
};

}  // namespace fbq::b200
