/* TEST INFRASTRUCTURE ONLY -- the CPU checker, never the product.
 *
 * Plain-C restatement of the reference's Fallback-Quantization arithmetic
 * (/root/reference/proj, "fbq").  Every function cites the reference
 * file:line it follows.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may call it.
 *
 * Parity pinned: tests/test_oracle.py checks this library against golden
 * vectors produced by the reference itself (oracle/_ref, see
 * tests/golden/make_golden.py) and, where oracle/_ref is present, against the
 * reference live on random inputs.
 *
 * Layouts: matrices are row-major float32; codes are int16 (as the
 * reference's QuantizedTensor::codes, quant.hpp:31); block grids are
 * row-major (quant.hpp:32).  Fallback residuals use a DENSE residual plane:
 * res_codes has the primary's shape, only masked blocks are meaningful (zero
 * elsewhere), res_scales is one float per block (0 where unmasked).  The
 * reference's compact residuals[]/residual_index[] (quant.hpp:46-52) map onto
 * it one-to-one.
 */
#ifndef FBQ_ORACLE_H
#define FBQ_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* rng.hpp:11-58 */
uint64_t orc_mix64(uint64_t z);
uint64_t orc_bits_at(uint64_t seed, uint64_t n);
double orc_uniform_at(uint64_t seed, uint64_t n);
float orc_normal_at(uint64_t seed, uint64_t n);
uint64_t orc_derive_seed(uint64_t base, uint64_t a, uint64_t b);
/* trainsim.cpp:16-19 */
uint64_t orc_layer_seed(uint64_t base, int layer_id, uint64_t tag, int step);

/* kernels.cpp:12-74 (scalar backend = semantics reference) */
float orc_absmax_2d(const float* x, size_t rows, size_t cols, size_t ld);
void orc_quantize_rtn_2d(const float* x, size_t ldx, int16_t* q, size_t ldq, size_t rows,
                         size_t cols, float scale, int32_t limit);
void orc_dequantize_2d(const int16_t* q, size_t ldq, float* y, size_t ldy, size_t rows,
                       size_t cols, float scale);
void orc_gemm_i16_accum(const int16_t* a, size_t lda, const int16_t* b, size_t ldb, int32_t* c,
                        size_t ldc, size_t m, size_t n, size_t k);
void orc_scale_accum(float* acc, const int32_t* p, size_t n, float scale);

/* quant.cpp:36-53 -- gr x gc groups, bits in [2,16] */
int orc_quantize_rtn(const float* x, int64_t rows, int64_t cols, int64_t gr, int64_t gc,
                     int bits, int16_t* codes, float* scales);
/* quant.cpp:55-84 with a global row offset: element (r, c) of this shard uses
 * RNG index (row_offset + r) * cols + c (row_offset = 0 reproduces the
 * reference exactly; the offset form is what token-sharded ranks compute). */
int orc_quantize_stochastic(const float* x, int64_t rows, int64_t cols, int64_t gr, int64_t gc,
                            int bits, uint64_t seed, int64_t row_offset, int16_t* codes,
                            float* scales);
/* quant.cpp:86-104 */
int orc_dequantize(const int16_t* codes, const float* scales, int64_t rows, int64_t cols,
                   int64_t gr, int64_t gc, float* out);
/* quant.cpp:106-126 */
int orc_transpose_qt(const int16_t* codes, const float* scales, int64_t rows, int64_t cols,
                     int64_t gr, int64_t gc, int16_t* out_codes, float* out_scales);
/* quant.cpp:128-176 (b = 8, g x g blocks), dense residual plane (see above) */
int orc_fallback_quantize(const float* x, int64_t rows, int64_t cols, int64_t g,
                          const uint8_t* mask, int16_t* codes, float* scales, int16_t* res_codes,
                          float* res_scales);
/* quant.cpp:178-202 */
int orc_dequantize_fallback(const int16_t* codes, const float* scales, const uint8_t* mask,
                            const int16_t* res_codes, const float* res_scales, int64_t rows,
                            int64_t cols, int64_t g, float* out);

/* gemm.cpp:101-186.  A: m x k codes, B: k x n codes, both g x g blocks.
 * mask/res_* may be NULL (block_quant_gemm).  tile_* = 0 means untiled. */
int orc_block_gemm(const int16_t* a_codes, const float* a_scales, const uint8_t* mask,
                   const int16_t* res_codes, const float* res_scales, const int16_t* b_codes,
                   const float* b_scales, int64_t m, int64_t n, int64_t k, int64_t g,
                   int64_t tile_m, int64_t tile_n, int64_t tile_k, float* out);
/* Per-block int32 products P(bi,bj,bk) (gemm.cpp:140-145), for bit-exact
 * checks of the device's block products: out[((bi*nb+bj)*kb+bk)*g*g + r*g+c]. */
int orc_block_products(const int16_t* a_codes, const int16_t* b_codes, int64_t m, int64_t n,
                       int64_t k, int64_t g, int32_t* out);
/* gemm.cpp:56-74 */
int orc_gemm_oracle(const float* a, const float* b, int64_t m, int64_t n, int64_t k, float* out);

/* policy.cpp:12-28 (AbsMax), 56-87, 97-109 */
int orc_score_blocks_absmax(const float* x, int64_t rows, int64_t cols, int64_t g,
                            double* scores);
int orc_mask_threshold(const double* scores, int64_t n, double theta, uint8_t* mask);
int orc_mask_topk(const double* scores, int64_t n, double rate, uint8_t* mask);
double orc_mask_rate(const uint8_t* mask, int64_t n);
int orc_controller_update(double threshold, double observed, double r_min, double r_max,
                          double alpha, double* out_threshold);

/* gemm.cpp:205-239 -> rmse, max_abs_err, cosine, underflow_fraction */
int orc_compare(const float* actual, const float* reference, int64_t n, double* out4);

#ifdef __cplusplus
}
#endif
#endif
