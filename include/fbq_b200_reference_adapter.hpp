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
#include "fbq_b200.h"

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

}  // namespace fbq::b200
