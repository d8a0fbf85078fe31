// extern "C" boundary: argument checking + dispatch to the sm_100a kernels.
// See include/fbq_b200.h for the contract of every entry point.
#include <cuda_runtime.h>
#include <cmath>
#include <cstdint>

#include "../../include/fbq_b200.h"
#include "gemm_kernel.cuh"
#include "quant_kernels.cuh"

namespace fbq {
cudaError_t launch_threshold(const double* scores, int64_t n, double theta, uint32_t* mask_bits,
                             int32_t* count, cudaStream_t s);
cudaError_t launch_controller_rate(double* theta, const double* rate, double r_min, double r_max,
                                   double alpha, double* last_rate, cudaStream_t s);
cudaError_t launch_sgd(float* w, const float* g, int64_t n, double lr, cudaStream_t s);
}  // namespace fbq

namespace {

thread_local int g_last_cuda = 0;
int g_gemm_diag = 0;  // perf diagnostics only (fbq_debug_set_gemm_diag)
long long* g_gemm_prof = nullptr;

int cuda_status(cudaError_t e) {
  if (e == cudaSuccess) return FBQ_OK;
  g_last_cuda = (int)e;
  return FBQ_ERR_CUDA;
}

int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }
bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

int check_x(const void* x, int dtype, int64_t rows, int64_t cols, int64_t ldx) {
  if (dtype != FBQ_F32 && dtype != FBQ_BF16) return FBQ_ERR_ARG;
  if (rows < 0 || cols < 0) return FBQ_ERR_SHAPE;
  if (rows > 0 && cols > 0 && (x == nullptr || ldx < cols)) return FBQ_ERR_ARG;
  if (cdiv(rows, 128) > 65535) return FBQ_ERR_UNSUPPORTED;  // grid.y limit
  return FBQ_OK;
}

}  // namespace

extern "C" {

const char* fbq_version(void) { return "fbq-b200 0.1 (sm_100a)"; }
/* Performance diagnostics (not part of the reference API): 1 = GEMM epilogue
 * skips its math, 2 = producer skips TMA loads.  Results are garbage when set. */
void fbq_debug_set_gemm_diag(int flags) { g_gemm_diag = flags; }
/* device buffer of 5 x num_SMs int64: MMA-warp total / full-wait / tmem-wait / page-wait / issue cycles */
void fbq_debug_set_gemm_prof(long long* dev_buf) { g_gemm_prof = dev_buf; }
void fbq_debug_set_quant_diag(int flags) { fbq::g_quant_diag = flags; }
int fbq_block_side(void) { return 128; }

int fbq_cuda_init(void) { return cuda_status(fbq::gemm_init()); }

int64_t fbq_ctx10_bytes(int64_t rows, int64_t ld_ctx) { return rows * ld_ctx + rows * (ld_ctx / 4); }

int fbq_malloc(void** ptr, size_t bytes) {
  if (!ptr) return FBQ_ERR_ARG;
  *ptr = nullptr;
  if (bytes == 0) return FBQ_OK;
  return cuda_status(cudaMalloc(ptr, bytes));
}
int fbq_free(void* ptr) { return ptr ? cuda_status(cudaFree(ptr)) : FBQ_OK; }
int fbq_memcpy_h2d(void* dst, const void* src, size_t bytes) {
  return bytes ? cuda_status(cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice)) : FBQ_OK;
}
int fbq_memcpy_d2h(void* dst, const void* src, size_t bytes) {
  return bytes ? cuda_status(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost)) : FBQ_OK;
}
int fbq_memset(void* dst, int value, size_t bytes) {
  return bytes ? cuda_status(cudaMemset(dst, value, bytes)) : FBQ_OK;
}
int fbq_synchronize(void) { return cuda_status(cudaDeviceSynchronize()); }
int fbq_last_cuda_error(void) { return g_last_cuda; }

const char* fbq_status_string(int s) {
  switch (s) {
    case FBQ_OK: return "ok";
    case FBQ_ERR_SHAPE: return "shape/geometry mismatch";
    case FBQ_ERR_UNSUPPORTED: return "unsupported geometry, bit-width or alignment";
    case FBQ_ERR_CUDA: return "CUDA error";
    case FBQ_ERR_ARG: return "invalid argument";
    default: return "unknown status";
  }
}

static int fill_quant_params(fbq::QuantParams& p, const void* x, int64_t rows, int64_t cols,
                             int64_t ldx, int mask_mode, double theta, uint32_t* mask_bits,
                             int8_t* codes, int64_t ldq, float* scales, int8_t* res_codes,
                             float* res_scales, int32_t* masked_count, float* amax_out,
                             int8_t* sr_codes, uint64_t sr_seed, int8_t* sr_codes2,
                             uint64_t sr_seed2, int64_t sr_row_offset, cudaStream_t s,
                             const double* theta_dev = nullptr) {
  if (mask_mode < FBQ_MASK_NONE || mask_mode > FBQ_MASK_GIVEN) return FBQ_ERR_ARG;
  if (mask_mode != FBQ_MASK_NONE && mask_bits == nullptr) return FBQ_ERR_ARG;
  if (mask_mode == FBQ_MASK_THRESHOLD && !theta_dev && !(theta > 0.0))
    return FBQ_ERR_ARG;  // policy.cpp:74
  if ((res_codes == nullptr) != (res_scales == nullptr)) return FBQ_ERR_ARG;
  if ((codes || res_codes || sr_codes || sr_codes2) && ldq < cols) return FBQ_ERR_ARG;
  if (sr_row_offset < 0) return FBQ_ERR_ARG;
  // Threshold mode writes every mask bit (set or clear) in the quantizer, so
  // the bitmap is not zeroed here; the count is zeroed by a one-warp grid that
  // the quantizer overlaps (programmatic dependent launch, p.pdl).
  p = fbq::QuantParams{};
  if (masked_count) {
    if (int st = cuda_status(fbq::launch_zero_count(masked_count, s))) return st;
    p.pdl = 1;
  }
  p.x = x;
  p.rows = rows;
  p.cols = cols;
  p.ldx = ldx;
  p.ldq = ldq;
  p.mask_mode = mask_mode;
  p.theta = theta;
  p.theta_dev = theta_dev;
  p.mask_bits = mask_bits;
  p.codes = codes;
  p.scales = scales;
  p.res_codes = res_codes;
  p.res_scales = res_scales;
  p.masked_count = masked_count;
  p.amax_out = amax_out;
  p.sr_codes = sr_codes;
  p.sr_seed = sr_seed;
  p.sr_codes2 = sr_codes2;
  p.sr_seed2 = sr_seed2;
  p.row_offset = sr_row_offset;
  p.vec_store = (ldq % 16 == 0) && aligned16(codes) && aligned16(res_codes) &&
                aligned16(sr_codes) && aligned16(sr_codes2);
  return FBQ_OK;
}

int fbq_cuda_quantize_linear_input(const void* x, int dtype, int64_t rows, int64_t cols,
                                   int64_t ldx, int mask_mode, double theta,
                                   const double* theta_dev, uint32_t* mask_bits,
                                   int8_t* codes, int64_t ldq, float* scales, int8_t* res_codes,
                                   float* res_scales, int32_t* masked_count, int8_t* ctx_codes,
                                   uint64_t ctx_seed, int8_t* ctx_codes2, uint64_t ctx_seed2,
                                   int64_t row_offset, fbq_stream_t stream) {
  if (int st = check_x(x, dtype, rows, cols, ldx)) return st;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  fbq::QuantParams p;
  if (int st = fill_quant_params(p, x, rows, cols, ldx, mask_mode, theta, mask_bits, codes, ldq,
                                 scales, res_codes, res_scales, masked_count, nullptr, ctx_codes,
                                 ctx_seed, ctx_codes2, ctx_seed2, row_offset, s, theta_dev))
    return st;
  if (rows == 0 || cols == 0) return FBQ_OK;
  return cuda_status(fbq::launch_quantize(p, dtype == FBQ_BF16, s));
}

int fbq_cuda_glu_forward(const void* ab, int dtype, int64_t rows, int64_t cols, int64_t ld_ab,
                         void* ctx_a, void* ctx_b, int64_t ld_ctx, int ctx_format, float* ctx_a_scales,
                         float* ctx_b_scales, int ctx_bits, int exact_math, double theta,
                         const double* theta_dev, uint32_t* mask_bits,
                         int8_t* codes, int64_t ldq, float* scales, int8_t* res_codes,
                         float* res_scales, int32_t* masked_count, int8_t* ctx_codes,
                         uint64_t ctx_seed, int64_t row_offset, float* h_out, int64_t ld_h,
                         fbq_stream_t stream) {
  if (dtype != FBQ_F32 && dtype != FBQ_BF16) return FBQ_ERR_ARG;
  if (rows < 0 || cols < 0) return FBQ_ERR_SHAPE;
  if (rows == 0 || cols == 0) return FBQ_OK;
  const size_t esz = dtype == FBQ_F32 ? 4 : 2;
  if (!ab || ld_ab < 2 * cols || (h_out && ld_h < cols)) return FBQ_ERR_ARG;
  if ((ctx_a || ctx_b) && ld_ctx < cols) return FBQ_ERR_ARG;
  if (ctx_bits < 2 || ctx_bits > 16) return FBQ_ERR_ARG;
  if (ctx_format != FBQ_CTX_INT16 && ctx_format != FBQ_CTX_PACKED10) return FBQ_ERR_ARG;
  if ((ctx_a || ctx_b) && ctx_format == FBQ_CTX_PACKED10 && ctx_bits > 10) return FBQ_ERR_UNSUPPORTED;
  // vectorised 16-byte loads of a and b, 16-byte context stores
  if (cols % 8 || (ld_ab * esz) % 16 || !aligned16(ab) || (cols * esz) % 16 ||
      ((ctx_a || ctx_b) && (ld_ctx % 16 || (ctx_a && !aligned16(ctx_a)) || (ctx_b && !aligned16(ctx_b)))))
    return FBQ_ERR_UNSUPPORTED;
  if (cdiv(rows, 128) > 65535) return FBQ_ERR_UNSUPPORTED;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  fbq::QuantParams p;
  if (int st = fill_quant_params(p, nullptr, rows, cols, cols, FBQ_MASK_THRESHOLD, theta,
                                 mask_bits, codes, ldq, scales, res_codes, res_scales,
                                 masked_count, nullptr, ctx_codes, ctx_seed, nullptr, 0,
                                 row_offset, s, theta_dev))
    return st;
  if (ldq % 16) return FBQ_ERR_UNSUPPORTED;
  fbq::GluParams g{ab, rows, cols, ld_ab, static_cast<uint8_t*>(ctx_a), static_cast<uint8_t*>(ctx_b), ld_ctx,
                   ctx_a_scales, ctx_b_scales, (float)((1 << (ctx_bits - 1)) - 1), h_out, ld_h,
                   exact_math ? 1 : 0, ctx_format == FBQ_CTX_PACKED10 ? 1 : 0};
  return cuda_status(fbq::launch_glu_forward(g, p, dtype == FBQ_BF16, s));
}

int fbq_cuda_glu_backward(const void* gh, int dtype, int64_t rows, int64_t cols, int64_t ld_gh,
                          const void* ctx_a, const void* ctx_b, int64_t ld_ctx, int ctx_format,
                          const float* ctx_a_scales, const float* ctx_b_scales, int8_t* gq,
                          int64_t ldq, float* gq_scales, uint64_t seed_a, uint64_t seed_b,
                          int64_t row_offset, float* g_out, int exact_math, fbq_stream_t stream) {
  if (dtype != FBQ_F32 && dtype != FBQ_BF16) return FBQ_ERR_ARG;
  if (rows < 0 || cols < 0) return FBQ_ERR_SHAPE;
  if (rows == 0 || cols == 0) return FBQ_OK;
  const size_t esz = dtype == FBQ_F32 ? 4 : 2;
  if (!gh || !ctx_a || !ctx_b || !ctx_a_scales || !ctx_b_scales || !gq || !gq_scales)
    return FBQ_ERR_ARG;
  if (ld_gh < cols || ld_ctx < cols || ldq < 2 * cols || row_offset < 0) return FBQ_ERR_ARG;
  if (ctx_format != FBQ_CTX_INT16 && ctx_format != FBQ_CTX_PACKED10) return FBQ_ERR_ARG;
  if (cols % 8 || (ld_gh * esz) % 16 || !aligned16(gh) || ldq % 16 || cols % 16 || ld_ctx % 16 ||
      !aligned16(ctx_a) || !aligned16(ctx_b))
    return FBQ_ERR_UNSUPPORTED;
  if (cdiv(rows, 128) > 65535) return FBQ_ERR_UNSUPPORTED;
  fbq::GluBwdParams g{gh, rows, cols, ld_gh, static_cast<const uint8_t*>(ctx_a),
                      static_cast<const uint8_t*>(ctx_b), ld_ctx, ctx_a_scales, ctx_b_scales, gq, ldq,
                      gq_scales, seed_a, seed_b, row_offset, g_out, exact_math ? 1 : 0,
                      ctx_format == FBQ_CTX_PACKED10 ? 1 : 0};
  return cuda_status(fbq::launch_glu_backward(g, dtype == FBQ_BF16, reinterpret_cast<cudaStream_t>(stream)));
}

int fbq_cuda_quantize_fallback(const void* x, int dtype, int64_t rows, int64_t cols, int64_t ldx,
                               int mask_mode, double theta, uint32_t* mask_bits, int8_t* codes,
                               int64_t ldq, float* scales, int8_t* res_codes, float* res_scales,
                               int32_t* masked_count, float* amax_out, int8_t* sr_codes,
                               uint64_t sr_seed, int64_t sr_row_offset, fbq_stream_t stream) {
  if (int st = check_x(x, dtype, rows, cols, ldx)) return st;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  fbq::QuantParams p;
  if (int st = fill_quant_params(p, x, rows, cols, ldx, mask_mode, theta, mask_bits, codes, ldq,
                                 scales, res_codes, res_scales, masked_count, amax_out, sr_codes,
                                 sr_seed, nullptr, 0, sr_row_offset, s))
    return st;
  if (rows == 0 || cols == 0) return FBQ_OK;
  return cuda_status(fbq::launch_quantize(p, dtype == FBQ_BF16, s));
}

int fbq_cuda_block_absmax(const void* x, int dtype, int64_t rows, int64_t cols, int64_t ldx,
                          float* amax, fbq_stream_t stream) {
  if (amax == nullptr && rows > 0 && cols > 0) return FBQ_ERR_ARG;
  return fbq_cuda_quantize_fallback(x, dtype, rows, cols, ldx, FBQ_MASK_NONE, 1.0, nullptr,
                                    nullptr, cols, nullptr, nullptr, nullptr, nullptr, amax,
                                    nullptr, 0, 0, stream);
}

static bool rms_layout_ok(int64_t cols, int64_t ld, const void* p, size_t esz) {
  return cols % 8 == 0 && aligned16(p) && (ld * (int64_t)esz) % 16 == 0;
}

int fbq_cuda_rmsnorm_forward(const void* x, int dtype, int64_t rows, int64_t cols, int64_t ldx,
                             const float* gain, void* y, int64_t ldy, int16_t* ctx_codes,
                             int64_t ld_ctx, float* ctx_scales, float* rms_ws, fbq_stream_t stream) {
  if (dtype != FBQ_F32 && dtype != FBQ_BF16) return FBQ_ERR_ARG;
  if (rows < 0 || cols < 0) return FBQ_ERR_SHAPE;
  if (rows == 0 || cols == 0) return FBQ_OK;
  if (!x || !gain || !y || !ctx_codes || !ctx_scales || !rms_ws) return FBQ_ERR_ARG;
  if (ldx < cols || ldy < cols || ld_ctx < cols) return FBQ_ERR_ARG;
  const size_t esz = dtype == FBQ_F32 ? 4 : 2;
  if (!rms_layout_ok(cols, ldx, x, esz) || !rms_layout_ok(cols, ldy, y, esz) ||
      !rms_layout_ok(cols, ld_ctx, ctx_codes, 2) || cdiv(rows, 128) > 65535)
    return FBQ_ERR_UNSUPPORTED;
  return cuda_status(fbq::launch_rmsnorm_forward(x, dtype == FBQ_BF16, rows, cols, ldx, gain, y, ldy,
                                                 ctx_codes, ld_ctx, ctx_scales, rms_ws,
                                                 reinterpret_cast<cudaStream_t>(stream)));
}

int fbq_cuda_rmsnorm_quantize_input(const void* x, int dtype, int64_t rows, int64_t cols, int64_t ldx,
                                    const float* gain, int16_t* ctx_codes, int64_t ld_ctx,
                                    float* ctx_scales, float* rms_ws, int mask_mode, double theta,
                                    const double* theta_dev, uint32_t* mask_bits, int8_t* codes,
                                    int64_t ldq, float* scales, int8_t* res_codes, float* res_scales,
                                    int32_t* masked_count, int8_t* sr_codes, uint64_t sr_seed,
                                    int8_t* sr_codes2, uint64_t sr_seed2, int64_t row_offset,
                                    fbq_stream_t stream) {
  if (int st = check_x(x, dtype, rows, cols, ldx)) return st;
  if (rows == 0 || cols == 0) return FBQ_OK;
  if (!gain || !ctx_codes || !ctx_scales || !rms_ws || !codes || !scales) return FBQ_ERR_ARG;
  if (ld_ctx < cols) return FBQ_ERR_ARG;
  const size_t esz = dtype == FBQ_F32 ? 4 : 2;
  if (!rms_layout_ok(cols, ldx, x, esz) || !rms_layout_ok(cols, ld_ctx, ctx_codes, 2) ||
      ldq % 16 || !aligned16(codes) || (res_codes && !aligned16(res_codes)) ||
      (sr_codes && !aligned16(sr_codes)) || (sr_codes2 && !aligned16(sr_codes2)))
    return FBQ_ERR_UNSUPPORTED;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  fbq::QuantParams p;
  if (int st = fill_quant_params(p, x, rows, cols, ldx, mask_mode, theta, mask_bits, codes, ldq,
                                 scales, res_codes, res_scales, masked_count, nullptr, sr_codes,
                                 sr_seed, sr_codes2, sr_seed2, row_offset, s, theta_dev))
    return st;
  return cuda_status(fbq::launch_rmsnorm_quantize(p, dtype == FBQ_BF16, gain, ctx_codes, ld_ctx, ctx_scales,
                                                  rms_ws, s));
}

int fbq_cuda_rmsnorm_backward(const int16_t* ctx_codes, int64_t ld_ctx, const float* ctx_scales,
                              const void* gy, int dtype, int64_t rows, int64_t cols, int64_t ldgy,
                              const float* gain, void* gx, int64_t ldgx, float* grad_gain,
                              double* row_ws, float* term_ws, fbq_stream_t stream) {
  if (dtype != FBQ_F32 && dtype != FBQ_BF16) return FBQ_ERR_ARG;
  if (rows < 0 || cols < 0) return FBQ_ERR_SHAPE;
  if (rows == 0 || cols == 0) return FBQ_OK;
  if (!ctx_codes || !ctx_scales || !gy || !gain || !gx || !grad_gain || !row_ws || !term_ws)
    return FBQ_ERR_ARG;
  if (ldgy < cols || ldgx < cols || ld_ctx < cols) return FBQ_ERR_ARG;
  return cuda_status(fbq::launch_rmsnorm_backward(ctx_codes, ld_ctx, ctx_scales, gy, dtype == FBQ_BF16,
                                                  rows, cols, ldgy, gain, gx, ldgx, grad_gain, row_ws,
                                                  term_ws, reinterpret_cast<cudaStream_t>(stream)));
}

int fbq_cuda_rmsnorm_backward_residual(const int16_t* ctx_codes, int64_t ld_ctx, const float* ctx_scales,
                                       const void* gy, int dtype, int64_t rows, int64_t cols, int64_t ldgy,
                                       const float* gain, const void* residual, int64_t ld_res, void* gx,
                                       int64_t ldgx, float* grad_gain, double* row_ws, float* term_ws,
                                       fbq_stream_t stream) {
  if (dtype != FBQ_F32 && dtype != FBQ_BF16) return FBQ_ERR_ARG;
  if (rows < 0 || cols < 0) return FBQ_ERR_SHAPE;
  if (rows == 0 || cols == 0) return FBQ_OK;
  if (!ctx_codes || !ctx_scales || !gy || !gain || !residual || !gx || !grad_gain || !row_ws || !term_ws)
    return FBQ_ERR_ARG;
  if (ldgy < cols || ldgx < cols || ld_ctx < cols || ld_res < cols) return FBQ_ERR_ARG;
  return cuda_status(fbq::launch_rmsnorm_backward(ctx_codes, ld_ctx, ctx_scales, gy, dtype == FBQ_BF16,
                                                  rows, cols, ldgy, gain, gx, ldgx, grad_gain, row_ws,
                                                  term_ws, reinterpret_cast<cudaStream_t>(stream),
                                                  residual, ld_res));
}

int fbq_cuda_silu_forward(const void* x, int dtype, int64_t rows, int64_t cols, int64_t ldx, void* y,
                          int64_t ldy, int16_t* ctx_codes, int64_t ld_ctx, float* ctx_scales, int ctx_bits,
                          int exact_math, fbq_stream_t stream) {
  if (dtype != FBQ_F32 && dtype != FBQ_BF16) return FBQ_ERR_ARG;
  if (rows < 0 || cols < 0) return FBQ_ERR_SHAPE;
  if (rows == 0 || cols == 0) return FBQ_OK;
  if (!x || !y || !ctx_codes || !ctx_scales || ldx < cols || ldy < cols || ld_ctx < cols) return FBQ_ERR_ARG;
  if (ctx_bits < 2 || ctx_bits > 16) return FBQ_ERR_UNSUPPORTED;
  const size_t esz = dtype == FBQ_F32 ? 4 : 2;
  if (!rms_layout_ok(cols, ldx, x, esz) || !rms_layout_ok(cols, ldy, y, esz) ||
      !rms_layout_ok(cols, ld_ctx, ctx_codes, 2) || cdiv(rows, 128) > 65535)
    return FBQ_ERR_UNSUPPORTED;
  return cuda_status(fbq::launch_silu_forward(x, dtype == FBQ_BF16, rows, cols, ldx, y, ldy, ctx_codes, ld_ctx,
                                              ctx_scales, (float)((1 << (ctx_bits - 1)) - 1), exact_math != 0,
                                              reinterpret_cast<cudaStream_t>(stream)));
}

int fbq_cuda_silu_backward(const int16_t* ctx_codes, int64_t ld_ctx, const float* ctx_scales, const void* gy,
                           int dtype, int64_t rows, int64_t cols, int64_t ldgy, void* gx, int64_t ldgx,
                           int exact_math, fbq_stream_t stream) {
  if (dtype != FBQ_F32 && dtype != FBQ_BF16) return FBQ_ERR_ARG;
  if (rows < 0 || cols < 0) return FBQ_ERR_SHAPE;
  if (rows == 0 || cols == 0) return FBQ_OK;
  if (!ctx_codes || !ctx_scales || !gy || !gx || ldgy < cols || ldgx < cols || ld_ctx < cols) return FBQ_ERR_ARG;
  return cuda_status(fbq::launch_silu_backward(ctx_codes, ld_ctx, ctx_scales, gy, dtype == FBQ_BF16, rows, cols,
                                               ldgy, gx, ldgx, exact_math != 0,
                                               reinterpret_cast<cudaStream_t>(stream)));
}

int fbq_cuda_mask_topk(const float* scores, int64_t n, double rate, uint32_t* mask_bits,
                       int32_t* masked_count, fbq_stream_t stream) {
  if (!(rate >= 0.0 && rate <= 1.0)) return FBQ_ERR_ARG;  // policy.cpp:57
  if (n < 0 || n >= (1ll << 32)) return FBQ_ERR_SHAPE;
  if (n == 0) return FBQ_OK;
  if (!scores || !mask_bits) return FBQ_ERR_ARG;
  int64_t k = (int64_t)std::ceil(rate * (double)n);  // policy.cpp:58-59
  if (k > n) k = n;
  return cuda_status(fbq::launch_topk(scores, n, k, mask_bits, masked_count,
                                      reinterpret_cast<cudaStream_t>(stream)));
}

int fbq_cuda_mask_threshold(const double* scores, int64_t n, double threshold, uint32_t* mask_bits,
                            int32_t* masked_count, fbq_stream_t stream) {
  if (n < 0 || n >= (1ll << 31)) return FBQ_ERR_SHAPE;
  if (n == 0) return FBQ_OK;
  if (!scores || !mask_bits) return FBQ_ERR_ARG;
  return cuda_status(fbq::launch_threshold(scores, n, threshold, mask_bits, masked_count,
                                           reinterpret_cast<cudaStream_t>(stream)));
}

int fbq_cuda_controller_update_rate(double* theta_dev, const double* observed_rate_dev, double r_min,
                                    double r_max, double alpha, double* last_rate_dev,
                                    fbq_stream_t stream) {
  if (!theta_dev || !observed_rate_dev) return FBQ_ERR_ARG;
  if (!(0.0 <= r_min && r_min < r_max && r_max <= 1.0) || !(alpha > 1.0)) return FBQ_ERR_ARG;
  return cuda_status(fbq::launch_controller_rate(theta_dev, observed_rate_dev, r_min, r_max, alpha,
                                                 last_rate_dev, reinterpret_cast<cudaStream_t>(stream)));
}

int fbq_cuda_sgd_update(float* w, const float* grad, int64_t n, double lr, fbq_stream_t stream) {
  if (n < 0 || (n > 0 && (!w || !grad))) return FBQ_ERR_ARG;
  return cuda_status(fbq::launch_sgd(w, grad, n, lr, reinterpret_cast<cudaStream_t>(stream)));
}

int fbq_cuda_sgd_quantize_rtn(float* w, const float* grad, int64_t rows, int64_t cols, double lr,
                              int8_t* codes, int64_t ldq, float* scales, fbq_stream_t stream) {
  if (rows < 0 || cols < 0) return FBQ_ERR_SHAPE;
  if (rows == 0 || cols == 0) return FBQ_OK;
  if (!w || !grad || !codes || !scales || ldq < cols) return FBQ_ERR_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  // one fused pass needs 16-byte vectors of W / dW rows and of the code rows
  // (grid.y <= 65535); any other layout runs the same two steps as two kernels
  if (cols % 4 || !aligned16(w) || !aligned16(grad) || ldq % 16 || !aligned16(codes) ||
      cdiv(rows, 128) > 65535) {
    if (int st = fbq_cuda_sgd_update(w, grad, rows * cols, lr, stream)) return st;
    return fbq_cuda_quantize_rtn(w, FBQ_F32, rows, cols, cols, codes, ldq, scales, stream);
  }
  return cuda_status(fbq::launch_sgd_quantize(w, grad, rows, cols, lr, codes, ldq, scales, s));
}

int fbq_cuda_quantize_rtn(const void* x, int dtype, int64_t rows, int64_t cols, int64_t ldx,
                          int8_t* codes, int64_t ldq, float* scales, fbq_stream_t stream) {
  if ((codes == nullptr || scales == nullptr) && rows > 0 && cols > 0) return FBQ_ERR_ARG;
  return fbq_cuda_quantize_fallback(x, dtype, rows, cols, ldx, FBQ_MASK_NONE, 1.0, nullptr, codes,
                                    ldq, scales, nullptr, nullptr, nullptr, nullptr, nullptr, 0, 0,
                                    stream);
}

int fbq_cuda_quantize_stochastic(const void* x, int dtype, int64_t rows, int64_t cols,
                                 int64_t ldx, uint64_t seed, int64_t row_offset, int8_t* codes,
                                 int64_t ldq, float* scales, fbq_stream_t stream) {
  if ((codes == nullptr || scales == nullptr) && rows > 0 && cols > 0) return FBQ_ERR_ARG;
  return fbq_cuda_quantize_fallback(x, dtype, rows, cols, ldx, FBQ_MASK_NONE, 1.0, nullptr,
                                    nullptr, ldq, scales, nullptr, nullptr, nullptr, nullptr,
                                    codes, seed, row_offset, stream);
}

static int gemm_common(const int8_t* a_codes, int64_t lda, const float* a_scales,
                       int64_t lds_a, int a_major, const int8_t* b_codes, int64_t ldb,
                       const float* b_scales, int64_t lds_b, int b_major,
                       const uint32_t* mask_bits, const int8_t* res_codes,
                       const float* res_scales, int64_t M, int64_t N, int64_t K, void* out,
                       int out_dtype, int64_t ldo, int accumulate, int epi, int32_t* dump,
                       cudaStream_t s) {
  if (M < 0 || N < 0 || K < 0) return FBQ_ERR_SHAPE;
  if ((a_major != 0 && a_major != 1) || (b_major != 0 && b_major != 1)) return FBQ_ERR_ARG;
  if (out_dtype != FBQ_F32 && out_dtype != FBQ_BF16) return FBQ_ERR_ARG;
  if (M == 0 || N == 0) return FBQ_OK;
  if (dump == nullptr && (out == nullptr || ldo < N)) return FBQ_ERR_ARG;
  if (K == 0) {  // empty reduction: the reference returns zeros (gemm.cpp:128)
    if (dump || accumulate) return FBQ_OK;
    const size_t esz = out_dtype == FBQ_F32 ? 4 : 2;
    return cuda_status(cudaMemset2DAsync(out, (size_t)ldo * esz, 0, (size_t)N * esz, (size_t)M, s));
  }
  if (!a_codes || !b_codes) return FBQ_ERR_ARG;
  if (dump == nullptr && (!a_scales || !b_scales)) return FBQ_ERR_ARG;
  if (mask_bits && (!res_codes || (dump == nullptr && !res_scales))) return FBQ_ERR_ARG;
  // TMA: 16-byte aligned bases and row strides
  if (!aligned16(a_codes) || !aligned16(b_codes) || (res_codes && !aligned16(res_codes)) ||
      lda % 16 || ldb % 16)
    return FBQ_ERR_UNSUPPORTED;
  if (lda < (a_major == 0 ? K : M) || ldb < (b_major == 0 ? K : N)) return FBQ_ERR_SHAPE;
  fbq::GemmOperands o{a_codes, lda, res_codes, b_codes, ldb};
  fbq::GemmParams p{};
  p.M = M;
  p.N = N;
  p.K = K;
  p.MB = (int)cdiv(M, 128);
  p.NB = (int)cdiv(N, 128);
  p.KB = (int)cdiv(K, 128);
  p.a_major = a_major;
  p.b_major = b_major;
  // natural grid strides unless given: K-major stored grids are [.][KB], MN-major [KB][.]
  const int64_t nat_a = a_major == 0 ? p.KB : p.MB;
  const int64_t nat_b = b_major == 0 ? p.KB : p.NB;
  if ((lds_a && lds_a < nat_a) || (lds_b && lds_b < nat_b)) return FBQ_ERR_SHAPE;
  if (mask_bits && lds_a && lds_a != nat_a) return FBQ_ERR_UNSUPPORTED;  // mask = natural A grid
  p.lds_a = lds_a ? lds_a : nat_a;
  p.lds_b = lds_b ? lds_b : nat_b;
  p.a_scales = a_scales;
  p.b_scales = b_scales;
  p.mask_bits = mask_bits;
  p.res_scales = res_scales;
  p.out = out;
  p.ldo = ldo;
  p.out_bf16 = out_dtype == FBQ_BF16;
  p.accumulate = accumulate ? 1 : 0;
  p.vec_store = (out != nullptr) && aligned16(out) && ((ldo * (out_dtype == FBQ_F32 ? 4 : 2)) % 16 == 0);
  p.dump = dump;
  p.one = 1.0f;
  p.diag = g_gemm_diag;
  p.prof = g_gemm_prof;
  p.dump_res_offset = (int64_t)p.MB * p.NB * p.KB * 128 * 128;
  return cuda_status(fbq::launch_gemm(o, p, dump ? fbq::kEpiDump : epi, s));
}

int fbq_cuda_gemm(const int8_t* a_codes, int64_t lda, const float* a_scales, int a_major,
                  const int8_t* b_codes, int64_t ldb, const float* b_scales, int b_major,
                  const uint32_t* mask_bits, const int8_t* res_codes, const float* res_scales,
                  int64_t M, int64_t N, int64_t K, void* out, int out_dtype, int64_t ldo,
                  int accumulate, int epilogue, fbq_stream_t stream) {
  if (epilogue != FBQ_EPI_EXACT && epilogue != FBQ_EPI_FMA) return FBQ_ERR_ARG;
  return gemm_common(a_codes, lda, a_scales, 0, a_major, b_codes, ldb, b_scales, 0, b_major,
                     mask_bits, res_codes, res_scales, M, N, K, out, out_dtype, ldo, accumulate,
                     epilogue, nullptr, reinterpret_cast<cudaStream_t>(stream));
}

int fbq_cuda_gemm_ex(const int8_t* a_codes, int64_t lda, const float* a_scales, int64_t lds_a,
                     int a_major, const int8_t* b_codes, int64_t ldb, const float* b_scales,
                     int64_t lds_b, int b_major, const uint32_t* mask_bits,
                     const int8_t* res_codes, const float* res_scales, int64_t M, int64_t N,
                     int64_t K, void* out, int out_dtype, int64_t ldo, int accumulate,
                     int epilogue, fbq_stream_t stream) {
  if (epilogue != FBQ_EPI_EXACT && epilogue != FBQ_EPI_FMA) return FBQ_ERR_ARG;
  if (lds_a < 0 || lds_b < 0) return FBQ_ERR_ARG;
  return gemm_common(a_codes, lda, a_scales, lds_a, a_major, b_codes, ldb, b_scales, lds_b,
                     b_major, mask_bits, res_codes, res_scales, M, N, K, out, out_dtype, ldo,
                     accumulate, epilogue, nullptr, reinterpret_cast<cudaStream_t>(stream));
}

int fbq_cuda_gemm_block_products(const int8_t* a_codes, int64_t lda, int a_major,
                                 const int8_t* b_codes, int64_t ldb, int b_major,
                                 const uint32_t* mask_bits, const int8_t* res_codes, int64_t M,
                                 int64_t N, int64_t K, int32_t* out, fbq_stream_t stream) {
  if (out == nullptr) return FBQ_ERR_ARG;
  return gemm_common(a_codes, lda, nullptr, 0, a_major, b_codes, ldb, nullptr, 0, b_major,
                     mask_bits, res_codes, nullptr, M, N, K, nullptr, FBQ_F32, 0, 0,
                     FBQ_EPI_EXACT, out, reinterpret_cast<cudaStream_t>(stream));
}

int fbq_cuda_controller_update(double* theta_dev, const int32_t* masked_count, int64_t n_blocks,
                               double r_min, double r_max, double alpha, double* last_rate_dev,
                               fbq_stream_t stream) {
  if (!theta_dev || !masked_count || n_blocks < 0) return FBQ_ERR_ARG;
  if (!(0.0 <= r_min && r_min < r_max && r_max <= 1.0) || !(alpha > 1.0)) return FBQ_ERR_ARG;
  return cuda_status(fbq::launch_controller(theta_dev, masked_count, n_blocks, r_min, r_max,
                                            alpha, last_rate_dev,
                                            reinterpret_cast<cudaStream_t>(stream)));
}

int fbq_cuda_dequantize(const int8_t* codes, int64_t ldq, const float* scales,
                        const uint32_t* mask_bits, const int8_t* res_codes,
                        const float* res_scales, int64_t rows, int64_t cols, float* out,
                        int64_t ldo, fbq_stream_t stream) {
  if (rows < 0 || cols < 0) return FBQ_ERR_SHAPE;
  if (rows == 0 || cols == 0) return FBQ_OK;
  if (!codes || !scales || !out || ldq < cols || ldo < cols) return FBQ_ERR_ARG;
  if (mask_bits && (!res_codes || !res_scales)) return FBQ_ERR_ARG;
  fbq::DequantParams p{codes, scales, mask_bits, res_codes, res_scales, rows, cols, ldq, ldo, out};
  return cuda_status(fbq::launch_dequantize(p, reinterpret_cast<cudaStream_t>(stream)));
}

int fbq_cuda_round_probe(const float* x, const float* a, const uint64_t* bits, int8_t* out_rtn,
                         int8_t* out_sr, int64_t n, int path, fbq_stream_t stream) {
  if (path < 0 || path > 4 || (path >= 2 && out_sr)) return FBQ_ERR_ARG;
  if (path >= 3 && (n % 8 || !out_rtn)) return FBQ_ERR_ARG;
  if (n < 0) return FBQ_ERR_SHAPE;
  if (n == 0) return FBQ_OK;
  if (!x || !a || (out_sr && !bits)) return FBQ_ERR_ARG;
  return cuda_status(fbq::launch_round_probe(x, a, bits, out_rtn, out_sr, n, path,
                                             reinterpret_cast<cudaStream_t>(stream)));
}

}  // extern "C"
