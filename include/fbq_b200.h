/* fbq_b200.h -- C ABI of the B200 (sm_100a) Fallback-Quantization hot path.
 *
 * Drop-in boundary for the reference C++ operator API (/root/reference/proj,
 * namespace fbq).  Each entry point below names the reference interface it
 * replaces (file:line).  The reference API takes host DenseMatrix /
 * QuantizedTensor values; here every DEVICE entry point (fbq_cuda_*) takes
 * plain device pointers + sizes, runs asynchronously on the caller's
 * cudaStream_t, never allocates, never synchronises, and returns an int status
 * (nothing throws across the ABI).  The HOST entry points (fbq_host_*) take
 * host buffers, exactly like the reference's value-semantics API, and do the
 * host<->device copies themselves (e2e path).
 *
 * Fixed hot-path geometry: 128 x 128 quantization blocks, b = 8 (L = 127) for
 * GEMM operands (SPEC.md gemm module; PAPER.md 4.5).  Other block sides or
 * bit-widths return FBQ_ERR_UNSUPPORTED -- there is no CPU fallback.
 *
 * Device layouts (row-major everywhere):
 *   x          fp32 or bf16, rows x ldx elements
 *   codes      int8, rows x ldq        (reference: int16 QuantizedTensor::codes, quant.hpp:31)
 *   scales     fp32, ceil(rows/128) x ceil(cols/128)            (quant.hpp:32)
 *   mask_bits  uint32, ceil(grid/32) words; bit b <-> linear block b (row-major),
 *              the compact form of FallbackTensor::mask (quant.hpp:42)
 *   res_codes  int8, rows x ldq: dense residual ("lo") plane; only flagged
 *              blocks are written / read (FallbackTensor::residuals, quant.hpp:46-52)
 *   res_scales fp32 grid (0 for unflagged blocks)
 * int8 planes that feed the GEMM need ldq % 16 == 0 (TMA stride rule).
 */
#ifndef FBQ_B200_H
#define FBQ_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* fbq_stream_t; /* == cudaStream_t */

enum fbq_status {
  FBQ_OK = 0,
  FBQ_ERR_SHAPE = 1,       /* dimension / geometry mismatch (reference: std::invalid_argument) */
  FBQ_ERR_UNSUPPORTED = 2, /* block side != 128, bits != 8, bad alignment */
  FBQ_ERR_CUDA = 3,        /* launch or runtime failure; see fbq_last_cuda_error() */
  FBQ_ERR_ARG = 4,         /* null pointer / bad enum / out-of-range value */
  FBQ_ERR_FORMAT = 5       /* malformed file (reference: FormatError, byte offset via fbq_io_last_offset) */
};
enum fbq_dtype { FBQ_F32 = 0, FBQ_BF16 = 1 };
enum fbq_mask_mode {
  FBQ_MASK_NONE = 0,      /* quantize_rtn only */
  FBQ_MASK_THRESHOLD = 1, /* u = absmax > theta (policy.cpp:73-80), written to mask_bits */
  FBQ_MASK_GIVEN = 2      /* u read from mask_bits (e.g. mask_topk, policy.cpp:56-71) */
};
enum fbq_major { FBQ_K_MAJOR = 0, FBQ_MN_MAJOR = 1 };
/* storage of the 10-bit 1 x 128 non-linear contexts (GluCombine a / b) */
enum fbq_ctx_format {
  FBQ_CTX_INT16 = 0,    /* int16 codes, rows x ld_ctx (the reference's QuantizedTensor storage) */
  FBQ_CTX_PACKED10 = 1  /* packed 10-bit planes, fbq_ctx10_bytes(rows, ld_ctx) bytes */
};
enum fbq_epilogue {
  FBQ_EPI_EXACT = 0, /* bit-identical to gemm.cpp's fl(acc + fl(s*P)) chain */
  FBQ_EPI_FMA = 1    /* acc = fma(P, s, acc): ~5e-8 rel. Frobenius from EXACT */
};

const char* fbq_version(void);
/* One-time setup of the CURRENT device (thread-safe, idempotent; allocates and
 * synchronises once): the GEMM's dynamic tile-counter ring.  Call it once per
 * device before capturing or timing work (the fbq_mlp_* / fbq_linear_*
 * drivers call it at creation).  The fbq_cuda_* entry points work without it
 * -- the GEMM then uses its static tile schedule -- and never allocate or
 * synchronise themselves; every call is safe from concurrent host threads
 * and under CUDA stream capture. */
int fbq_cuda_init(void);
const char* fbq_status_string(int status);
int fbq_last_cuda_error(void); /* cudaError_t of the last FBQ_ERR_CUDA on this thread */
int fbq_block_side(void);      /* 128 */

/* Device memory helpers (synchronous; default stream) so that bindings -- the
 * reference-typed C++ adapter, cgo/ctypes stubs -- need no CUDA runtime of
 * their own. */
int fbq_malloc(void** ptr, size_t bytes);
int fbq_free(void* ptr);
int fbq_memcpy_h2d(void* dst, const void* src, size_t bytes);
int fbq_memcpy_d2h(void* dst, const void* src, size_t bytes);
int fbq_memset(void* dst, int value, size_t bytes);
int fbq_synchronize(void);

/* score_blocks(AbsMax) -- policy.cpp:12-28 / policy.hpp:18-19.
 * amax[blk] = max |x| over the block (float; the reference widens to double). */
int fbq_cuda_block_absmax(const void* x, int dtype, int64_t rows, int64_t cols, int64_t ldx,
                          float* amax, fbq_stream_t stream);

/* RmsNorm (trainsim.cpp:154-211) with its 10-bit 1 x 128 RTN input context
 * (QuantConfig::nonlinear_bits / nonlinear_group, trainsim.hpp:26-28).
 * forward: y = fl(fl(x / rms) * gain), rms = sqrtf(float(sum x^2 / cols) + 1e-6f)
 *   with the sum of squares accumulated in double in column order (as the
 *   reference); ctx_codes (int16, rows x ld_ctx) + ctx_scales (rows x
 *   ceil(cols/128)) = quantize_rtn(x, 1 x 128, 10 bits).  rms_ws: rows floats.
 * backward: x = dequantize(ctx); gx = float(g*dy*inv - x*corr) (double math,
 *   row sums in column order); grad_gain[c] += float(float(dy*x) * inv) over the
 *   rows in order.  row_ws: 2*rows doubles, term_ws: rows*cols floats.
 * x / dy / y / gx share dtype (FBQ_F32 or FBQ_BF16); cols % 8 == 0, 16-byte
 * aligned rows, ld_ctx % 8 == 0. */
int fbq_cuda_rmsnorm_forward(const void* x, int dtype, int64_t rows, int64_t cols, int64_t ldx,
                             const float* gain, void* y, int64_t ldy, int16_t* ctx_codes,
                             int64_t ld_ctx, float* ctx_scales, float* rms_ws, fbq_stream_t stream);
/* RmsNorm::forward fused with the next QuantLinearLayer's input quantizer
 * (the transformer block's RMSNorm -> q/k/v or gate/up, trainsim.cpp:294-301,
 * SURVEY 8f-2): writes the RmsNorm context (ctx_codes / ctx_scales, as
 * fbq_cuda_rmsnorm_forward) and, for y = fl(fl(x / rms) * gain) rounded to the
 * activation dtype, exactly the outputs of fbq_cuda_quantize_linear_input(y, ...)
 * -- RTN codes, scales, fallback mask / count, residual plane, up to two
 * stochastic context planes -- without materialising y.  Same argument rules
 * as those two entry points (cols % 8 == 0, 16-byte aligned rows, ldq % 16 == 0). */
int fbq_cuda_rmsnorm_quantize_input(const void* x, int dtype, int64_t rows, int64_t cols, int64_t ldx,
                                    const float* gain, int16_t* ctx_codes, int64_t ld_ctx,
                                    float* ctx_scales, float* rms_ws, int mask_mode, double theta,
                                    const double* theta_dev, uint32_t* mask_bits, int8_t* codes,
                                    int64_t ldq, float* scales, int8_t* res_codes, float* res_scales,
                                    int32_t* masked_count, int8_t* sr_codes, uint64_t sr_seed,
                                    int8_t* sr_codes2, uint64_t sr_seed2, int64_t row_offset,
                                    fbq_stream_t stream);

int fbq_cuda_rmsnorm_backward(const int16_t* ctx_codes, int64_t ld_ctx, const float* ctx_scales,
                              const void* gy, int dtype, int64_t rows, int64_t cols, int64_t ldgy,
                              const float* gain, void* gx, int64_t ldgx, float* grad_gain,
                              double* row_ws, float* term_ws, fbq_stream_t stream);
/* The same, with the pre-norm residual block's gradient add fused into the
 * output: gx = fl(norm.backward(gy) + residual), GluBlock::backward's
 * add(norm.backward(grad_xn), grad_out) (trainsim.cpp:303-307); residual has
 * the activation dtype and row stride ld_res.  gx may alias residual. */
int fbq_cuda_rmsnorm_backward_residual(const int16_t* ctx_codes, int64_t ld_ctx, const float* ctx_scales,
                                       const void* gy, int dtype, int64_t rows, int64_t cols, int64_t ldgy,
                                       const float* gain, const void* residual, int64_t ld_res, void* gx,
                                       int64_t ldgx, float* grad_gain, double* row_ws, float* term_ws,
                                       fbq_stream_t stream);

/* SiluLayer (trainsim.hpp:118-131, trainsim.cpp:265-290).  forward: y = silu(x)
 * and the input's ctx_bits (10) 1 x 128 RTN context (int16 codes rows x ld_ctx,
 * scales rows x ceil(cols/128)); backward: gx = fl(gy * silu'(dequantize(ctx))).
 * exact_math: the reference's double silu / silu' (silu_scalar,
 * silu_grad_scalar, trainsim.cpp:37-46), bit-exact; 0: fp32 MUFU forms (a few
 * ulp).  Layout rules as RmsNorm (cols % 8 == 0, 16-byte aligned rows). */
int fbq_cuda_silu_forward(const void* x, int dtype, int64_t rows, int64_t cols, int64_t ldx, void* y,
                          int64_t ldy, int16_t* ctx_codes, int64_t ld_ctx, float* ctx_scales, int ctx_bits,
                          int exact_math, fbq_stream_t stream);
int fbq_cuda_silu_backward(const int16_t* ctx_codes, int64_t ld_ctx, const float* ctx_scales, const void* gy,
                           int dtype, int64_t rows, int64_t cols, int64_t ldgy, void* gx, int64_t ldgx,
                           int exact_math, fbq_stream_t stream);

/* mask_topk -- policy.cpp:56-71 / policy.hpp:30-31: exactly k = ceil(rate * n)
 * (clamped to n) blocks with the largest scores, ties toward the lower block
 * index, written as a bitmap (bit b = block b; the whole bitmap is rewritten).
 * scores: the n fp32 block absmaxes of fbq_cuda_block_absmax (non-negative).
 * masked_count (optional) receives k.  One device pass, no host round trip;
 * rate outside [0, 1] -> FBQ_ERR_ARG (policy.cpp:57). */
int fbq_cuda_mask_topk(const float* scores, int64_t n, double rate, uint32_t* mask_bits,
                       int32_t* masked_count, fbq_stream_t stream);

/* K1: fused quantize_rtn (quant.cpp:36-53) + score_blocks(AbsMax) + mask_threshold
 * (policy.cpp:73-80) + fallback_quantize (quant.cpp:128-176, quant.hpp:74-75) +
 * masked-block count (mask_rate numerator, policy.cpp:82-87) + optional fused
 * quantize_stochastic context codes (quant.cpp:55-84, trainsim.cpp:100-102).
 * One read of x.  Any output pointer may be NULL to skip that output except
 * that mask modes != NONE need mask_bits, and res_codes/res_scales go together.
 * In THRESHOLD mode every bit of mask_bits (including the unused tail of the
 * last word) is written by the kernel, so the caller need not clear it;
 * *masked_count is overwritten.  sr_codes (if non-NULL) shares `scales` with the RTN codes and
 * uses RNG index (sr_row_offset + r) * cols + c (row offset = token-shard
 * start; 0 reproduces the reference). */
int fbq_cuda_quantize_fallback(const void* x, int dtype, int64_t rows, int64_t cols, int64_t ldx,
                               int mask_mode, double theta, uint32_t* mask_bits, int8_t* codes,
                               int64_t ldq, float* scales, int8_t* res_codes, float* res_scales,
                               int32_t* masked_count, float* amax_out, int8_t* sr_codes,
                               uint64_t sr_seed, int64_t sr_row_offset, fbq_stream_t stream);

/* Linear-layer input quantizer (QuantLinearLayer::forward, trainsim.cpp:80-102):
 * as fbq_cuda_quantize_fallback, plus a SECOND stochastic context plane with its
 * own seed -- layers that share an input (gate/up of a GLU block) each keep the
 * reference's own context stream -- and an optional device-resident threshold
 * (theta_dev != NULL overrides theta; see fbq_cuda_controller_update). */
int fbq_cuda_quantize_linear_input(const void* x, int dtype, int64_t rows, int64_t cols,
                                   int64_t ldx, int mask_mode, double theta,
                                   const double* theta_dev, uint32_t* mask_bits,
                                   int8_t* codes, int64_t ldq, float* scales, int8_t* res_codes,
                                   float* res_scales, int32_t* masked_count, int8_t* ctx_codes,
                                   uint64_t ctx_seed, int8_t* ctx_codes2, uint64_t ctx_seed2,
                                   int64_t row_offset, fbq_stream_t stream);

/* bytes of one packed 10-bit context plane of rows x ld_ctx codes */
int64_t fbq_ctx10_bytes(int64_t rows, int64_t ld_ctx);

/* GluCombine::forward (trainsim.cpp:224-246) fused with the down projection's
 * input quantizer: ab = [a | b] (rows x 2*cols, the gate/up GEMM output, fp32
 * or bf16); writes the ctx_bits-bit 1x128 RTN contexts of a and b
 * (trainsim.cpp:240-243) in ctx_format: FBQ_CTX_INT16 (int16 codes, rows x
 * ld_ctx) or FBQ_CTX_PACKED10 (ctx_bits <= 10; per context the low byte of
 * every code, int8 [rows][ld_ctx], followed by the top two bits of each code's
 * 10-bit two's complement, four codes per byte, [rows][ld_ctx/4], code c at
 * bits 2*(c%4): 1.25 bytes per element, 5/8 of bf16, fbq_ctx10_bytes(rows,
 * ld_ctx) bytes; ld_ctx % 16 == 0) -- and quantizes h = silu(a)*b exactly like
 * fbq_cuda_quantize_linear_input (threshold mode) with one context plane.
 * h itself is not written unless h_out != NULL (fp32, parity/debug).  With
 * exact_math != 0 silu is evaluated like silu_scalar (trainsim.cpp:38-41):
 * double exp, one rounding; otherwise a fast fp32 form (a few ulp away). */
int fbq_cuda_glu_forward(const void* ab, int dtype, int64_t rows, int64_t cols, int64_t ld_ab,
                         void* ctx_a, void* ctx_b, int64_t ld_ctx, int ctx_format, float* ctx_a_scales,
                         float* ctx_b_scales, int ctx_bits, int exact_math, double theta,
                         const double* theta_dev, uint32_t* mask_bits, int8_t* codes,
                         int64_t ldq, float* scales, int8_t* res_codes, float* res_scales,
                         int32_t* masked_count, int8_t* ctx_codes, uint64_t ctx_seed,
                         int64_t row_offset, float* h_out, int64_t ld_h, fbq_stream_t stream);

/* GluCombine::backward (trainsim.cpp:248-263) fused with the gate and up
 * layers' dY quantizers (trainsim.cpp:117-119): from dH and the dequantized
 * contexts, ga = dH*b*silu'(a) and gb = dH*silu(a), stochastically rounded
 * (seeds seed_a / seed_b, RNG index over each rows x cols matrix) into
 * gq = [q(ga) | q(gb)] (int8 rows x ldq, ldq >= 2*cols) with scale grid
 * gq_scales [ceil(rows/128)][2*ceil(cols/128)].  g_out (optional fp32
 * [2][rows][cols]) receives ga, gb for parity checks.  exact_math as in
 * fbq_cuda_glu_forward (silu / silu_grad_scalar, trainsim.cpp:38-46). */
int fbq_cuda_glu_backward(const void* gh, int dtype, int64_t rows, int64_t cols, int64_t ld_gh,
                          const void* ctx_a, const void* ctx_b, int64_t ld_ctx, int ctx_format,
                          const float* ctx_a_scales, const float* ctx_b_scales, int8_t* gq,
                          int64_t ldq, float* gq_scales, uint64_t seed_a, uint64_t seed_b,
                          int64_t row_offset, float* g_out, int exact_math, fbq_stream_t stream);

/* mask_threshold (policy.cpp:73-80): bit i of mask_bits = scores[i] > threshold
 * (strict, double); *masked_count (may be NULL) = flagged blocks (mask_rate
 * numerator, policy.cpp:82-87).  Writes every word; nothing to pre-zero. */
int fbq_cuda_mask_threshold(const double* scores, int64_t n, double threshold, uint32_t* mask_bits,
                            int32_t* masked_count, fbq_stream_t stream);

/* controller_update (policy.cpp:97-109) with the observed rate in device memory */
int fbq_cuda_controller_update_rate(double* theta_dev, const double* observed_rate_dev, double r_min,
                                    double r_max, double alpha, double* last_rate_dev,
                                    fbq_stream_t stream);

/* QuantLinearLayer::apply_sgd (trainsim.cpp:137-143): w[i] -= float(lr * double(grad[i])) */
int fbq_cuda_sgd_update(float* w, const float* grad, int64_t n, double lr, fbq_stream_t stream);

/* apply_sgd fused with the next forward's weight quantization: w (rows x cols,
 * contiguous fp32) -= float(lr * double(grad)), then quantize_rtn of the updated
 * w (128 x 128 blocks, quant.cpp:36-53; trainsim.cpp:96) into codes (ldq) and
 * scales -- one pass over w and grad.  Bit-identical to fbq_cuda_sgd_update
 * followed by fbq_cuda_quantize_rtn (which it runs instead when cols % 4, ldq %
 * 16 or a pointer's 16-byte alignment rules out the fused kernel). */
int fbq_cuda_sgd_quantize_rtn(float* w, const float* grad, int64_t rows, int64_t cols, double lr,
                              int8_t* codes, int64_t ldq, float* scales, fbq_stream_t stream);

/* controller_update (policy.cpp:97-109) on device: rate = *masked_count /
 * n_blocks; *theta_dev /= alpha if rate < r_min, *= alpha if rate > r_max;
 * *last_rate_dev = rate (may be NULL). */
int fbq_cuda_controller_update(double* theta_dev, const int32_t* masked_count, int64_t n_blocks,
                               double r_min, double r_max, double alpha, double* last_rate_dev,
                               fbq_stream_t stream);

/* quantize_rtn -- quant.cpp:36-53 / quant.hpp:61 */
int fbq_cuda_quantize_rtn(const void* x, int dtype, int64_t rows, int64_t cols, int64_t ldx,
                          int8_t* codes, int64_t ldq, float* scales, fbq_stream_t stream);

/* K2: quantize_stochastic -- quant.cpp:55-84 / quant.hpp:65-66 (seed = the
 * DeterministicRng seed, e.g. derive_seed(base, layer*4+tag, step), trainsim.cpp:16-19) */
int fbq_cuda_quantize_stochastic(const void* x, int dtype, int64_t rows, int64_t cols,
                                 int64_t ldx, uint64_t seed, int64_t row_offset, int8_t* codes,
                                 int64_t ldq, float* scales, fbq_stream_t stream);

/* K3: block_quant_gemm (gemm.cpp:190-193, gemm.hpp:41-42) when mask_bits == NULL,
 * fallback_gemm (gemm.cpp:195-198, gemm.hpp:47-48) otherwise.
 *   out[M x N] (+)= sum over ascending k-blocks of the scaled int32 block products.
 *   A[m,k] = a_codes[m*lda + k]  (K-major)   or  a_codes[k*lda + m]  (MN-major)
 *   B[k,n] = b_codes[n*ldb + k]  (K-major)   or  b_codes[k*ldb + n]  (MN-major)
 * Scale grids are the STORED tensors' own grids (row-major): A K-major
 * [ceil(M/128)][ceil(K/128)], A MN-major [ceil(K/128)][ceil(M/128)], B K-major
 * [ceil(N/128)][ceil(K/128)], B MN-major [ceil(K/128)][ceil(N/128)].  mask_bits,
 * res_codes (same layout/ld as A) and res_scales index A's stored grid.
 * The reference's B operand (quantize_rtn(transpose(W)), trainsim.cpp:96-97)
 * is MN-major; W's own quantization (trainsim.cpp:121) used K-major is the same
 * bytes transposed, so one W quantization serves forward and dgrad.
 * accumulate=1 performs out = fl(out + acc) (trainsim.cpp:125 grad_w_ += gw).
 * out_dtype FBQ_F32 (parity) or FBQ_BF16. */
int fbq_cuda_gemm(const int8_t* a_codes, int64_t lda, const float* a_scales, int a_major,
                  const int8_t* b_codes, int64_t ldb, const float* b_scales, int b_major,
                  const uint32_t* mask_bits, const int8_t* res_codes, const float* res_scales,
                  int64_t M, int64_t N, int64_t K, void* out, int out_dtype, int64_t ldo,
                  int accumulate, int epilogue, fbq_stream_t stream);

/* fbq_cuda_gemm with explicit row strides of the stored scale grids (0 =
 * natural), so a column slice of a concatenated code plane (e.g. the gate half
 * of [q(ga) | q(gb)]) can be used as an operand with its parent's scale grid.
 * Fallback (mask_bits != NULL) needs the natural A grid. */
int fbq_cuda_gemm_ex(const int8_t* a_codes, int64_t lda, const float* a_scales, int64_t lds_a,
                     int a_major, const int8_t* b_codes, int64_t ldb, const float* b_scales,
                     int64_t lds_b, int b_major, const uint32_t* mask_bits,
                     const int8_t* res_codes, const float* res_scales, int64_t M, int64_t N,
                     int64_t K, void* out, int out_dtype, int64_t ldo, int accumulate,
                     int epilogue, fbq_stream_t stream);

/* Debug/parity: the raw per-block int32 products of the same tcgen05 path
 * (gemm.cpp:140-145 pbuf), out[((bi*NB+bj)*KB+bk)*16384 + r*128 + c]; the
 * residual products (fallback) follow at element offset MB*NB*KB*16384. */
int fbq_cuda_gemm_block_products(const int8_t* a_codes, int64_t lda, int a_major,
                                 const int8_t* b_codes, int64_t ldb, int b_major,
                                 const uint32_t* mask_bits, const int8_t* res_codes, int64_t M,
                                 int64_t N, int64_t K, int32_t* out, fbq_stream_t stream);

/* K4: dequantize (quant.cpp:86-104) / dequantize_fallback (quant.cpp:178-202)
 * when mask_bits != NULL.  out fp32 rows x ldo. */
int fbq_cuda_dequantize(const int8_t* codes, int64_t ldq, const float* scales,
                        const uint32_t* mask_bits, const int8_t* res_codes,
                        const float* res_scales, int64_t rows, int64_t cols, float* out,
                        int64_t ldo, fbq_stream_t stream);

/* Rounding probes for exhaustive tests: out_rtn[i] = RTN code of x[i]/a[i]
 * (kernels.cpp:24-40), out_sr[i] = SR code with RNG bits[i] (quant.cpp:69-77).
 * path 0: scalar functions, 1: the kernels' vector paths (V = 1), 2: 10-bit
 * context RTN (int16 out), 3: the 8-wide packed RTN path (n % 8 == 0, one
 * scale per 8-element vector = a[8g]), 4: the same packed path at level 511
 * (the 10-bit contexts' group RTN incl. its packed exact fix; int16 out). */
int fbq_cuda_round_probe(const float* x, const float* a, const uint64_t* bits, int8_t* out_rtn,
                         int8_t* out_sr, int64_t n, int path, fbq_stream_t stream);

/* Performance diagnostics only (not part of the reference API): flags
 * 1 = GEMM epilogue skips its math, 2 = GEMM producer skips the TMA loads,
 * 4 = GEMM epilogue skips the output stores, 8 = MMA skips the TMEM-slot wait,
 * 16 = MMA skips the operand-stage wait (races; timing experiments only).
 * Results are garbage while set; 0 restores normal operation. */
void fbq_debug_set_gemm_diag(int flags);
/* device buffer of 5 x num_SMs int64 receiving, per CTA, the MMA warp's total,
 * operand-wait, TMEM-slot-wait, scale-page-wait and MMA-issue cycles (null disables). */
void fbq_debug_set_gemm_prof(long long* dev_buf);
/* Quantizer diagnostics: 1 = use the one-block-per-CTA K1 instead of the
 * persistent TMA-pipelined K1 (A/B timing; results are identical). */
void fbq_debug_set_quant_diag(int flags);

/* ---- host entry points (reference value semantics; host buffers) --------
 * A fallback-quantized linear layer + SwiGLU MLP driver mirroring
 * QuantLinearLayer::forward/backward (trainsim.cpp:61-127) and the gate/up ->
 * GluCombine -> down data flow (trainsim.cpp:294-308) for B200.  Declared in
 * fbq_b200_host.h. */

#ifdef __cplusplus
}
#endif
#endif /* FBQ_B200_H */
