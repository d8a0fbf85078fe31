/* fbq_b200_host.h -- host-side drivers above the C ABI (include/fbq_b200.h).
 *
 * A fallback-quantized SwiGLU MLP (gate/up -> GluCombine -> down) that mirrors
 * the reference's QuantLinearLayer::forward/backward (trainsim.cpp:61-127) and
 * GluCombine (trainsim.cpp:224-263) data flow with 128 x 128 blocks, 8-bit
 * linear operands, 10-bit 1 x 128 non-linear contexts and the delay-threshold
 * controller (policy.cpp:97-109).  It is the e2e entry point the reference's
 * callers would bind: fbq_mlp_step_host takes HOST fp32 buffers exactly like
 * the reference value API (DenseMatrix in, DenseMatrix out) and performs the
 * host<->device copies itself.
 *
 * Per-layer RNG streams follow layer_seed (trainsim.cpp:16-19): gate = layer
 * layer_id_base, up = +1, down = +2; tag 0 = X context, tag 1 = dY.
 * gate and up see the same input and start from the same threshold, so the
 * reference's two controllers evolve identically; the driver keeps one.
 */
#ifndef FBQ_B200_HOST_H
#define FBQ_B200_HOST_H

#include <stdint.h>

#include "fbq_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct fbq_mlp_config {
  int64_t d_model;        /* K of gate/up, N of down */
  int64_t d_ff;           /* N of gate/up, K of down */
  int64_t max_tokens;     /* capacity of the device workspaces */
  int act_dtype;          /* FBQ_F32 / FBQ_BF16: x, dY, y, dX in the device API */
  int mid_dtype;          /* dtype of the [a|b] and dH intermediates (FBQ_F32 = parity) */
  int epilogue;           /* FBQ_EPI_EXACT (bit-exact) or FBQ_EPI_FMA */
  int nonlinear_bits;     /* 10 (QuantConfig::nonlinear_bits, trainsim.hpp:26) */
  int layer_id_base;      /* 0 */
  uint64_t seed;          /* 0x5eed (QuantConfig::seed) */
  double threshold_init;  /* 1.0 (QuantConfig::threshold_init) */
  double r_min, r_max, alpha; /* 0.1, 0.3, 1.3 (ControllerConfig) */
  int ctx_format;         /* GluCombine a / b contexts: FBQ_CTX_INT16 (default, like the
                             reference's QuantizedTensor codes) or FBQ_CTX_PACKED10 (10 bits
                             per code: the paper's context memory) */
} fbq_mlp_config;

void fbq_mlp_default_config(fbq_mlp_config* cfg);
/* Message of the last failing host-API call on this thread. */
const char* fbq_host_last_error(void);

/* w_gate, w_up: d_ff x d_model; w_down: d_model x d_ff (host fp32, row-major,
 * as QuantLinearLayer's weight, out x in).  Returns NULL on failure. */
void* fbq_mlp_create(const fbq_mlp_config* cfg, const float* w_gate, const float* w_up,
                     const float* w_down);
void fbq_mlp_destroy(void* mlp);

/* Device API (stream-ordered, no host synchronisation).  x, gy, y, gx are
 * device buffers of `tokens` rows in act_dtype.  `row_offset` is the global
 * row of this shard's row 0 (token sharding across ranks; 0 = whole batch). */
int fbq_mlp_forward_device(void* mlp, const void* x, int64_t tokens, int64_t row_offset, int step,
                           void* y, fbq_stream_t stream);
int fbq_mlp_backward_device(void* mlp, const void* gy, int64_t tokens, int64_t row_offset,
                            int step, void* gx, fbq_stream_t stream);
/* controller_step of every layer (trainsim.cpp:129-133) from the last forward */
int fbq_mlp_controller_step(void* mlp, fbq_stream_t stream);
/* Data parallel (trainsim.cpp:93,129-133 / policy.cpp:97-109 on the global
 * batch): the device int32[2] masked-block counters of the last forward
 * (gate/up, down) -- sum them over ranks in place on `stream` -- and a
 * controller step that divides by the GLOBAL block counts (0 = local). */
int32_t* fbq_mlp_count_ptr(void* mlp);
int fbq_mlp_controller_step_blocks(void* mlp, int64_t blocks_gate_up, int64_t blocks_down,
                                   fbq_stream_t stream);
/* zero_grad is deferred: the next backward's dW GEMMs write instead of
 * accumulate (bit-identical to adding into zeroed buffers, no 0.7 GB memset
 * per step).  fbq_mlp_get_grads / fbq_mlp_grad_ptr materialise pending zeros;
 * a device view of the gradients obtained earlier shows the zeros only once
 * the next backward has run. */
int fbq_mlp_zero_grad(void* mlp, fbq_stream_t stream);

/* Host API: one fwd+bwd step over host fp32 buffers (synchronous, like the
 * reference).  Pinned buffers make the copies asynchronous and overlapped. */
int fbq_mlp_step_host(void* mlp, const float* x, const float* gy, int64_t tokens, int step,
                      float* y, float* gx);

/* Pipelined host API: enqueue one step (zero_grad if FBQ_STEP_ZERO_GRAD, fwd,
 * bwd, controller_step if FBQ_STEP_CONTROLLER, apply_sgd at fbq_mlp_set_sgd_lr's
 * rate if FBQ_STEP_SGD -- the reference trainer's step) over host fp32 buffers and
 * return.  Step i's H2D copies overlap step i-1's compute and step i-1's D2H
 * copies overlap step i's (two device slots).  Host buffers must stay valid,
 * and outputs must not be read, until fbq_mlp_host_sync returns; pinned
 * buffers make the copies truly asynchronous. */
#define FBQ_STEP_ZERO_GRAD 1
#define FBQ_STEP_CONTROLLER 2
#define FBQ_STEP_SGD 4
int fbq_mlp_step_host_async(void* mlp, const float* x, const float* gy, int64_t tokens, int step,
                            float* y, float* gx, int flags);
int fbq_mlp_host_sync(void* mlp);

/* Set the device-resident thresholds (gate/up share one, down has its own). */
int fbq_mlp_set_thresholds(void* mlp, double theta_gate_up, double theta_down);
/* Bytes the forward saves for the backward (activation contexts: the two int8
 * stochastic X contexts, the a / b non-linear contexts, the int8 h context and
 * all their scale grids) at `tokens` tokens -- and, for comparison, what a BF16
 * implementation saves (X, a, b, h in bf16). */
int fbq_mlp_context_bytes(void* mlp, int64_t tokens, int64_t* ours, int64_t* bf16);
/* Optional CUDA-event timing of every GEMM launch (on the launching stream);
 * fbq_mlp_gemm_time returns the summed GEMM time since profiling was enabled
 * or last read (synchronise first) and resets. */
int fbq_mlp_set_profiling(void* mlp, int on);
int fbq_mlp_gemm_time(void* mlp, double* total_ms, int64_t* n_gemms);
/* Number of our kernels launched by this driver so far. */
int64_t fbq_mlp_launch_count(void* mlp);

/* Device pointers of the fp32 gradient accumulators (for the data-parallel
 * all-reduce): which = 0 gate (d_ff x d_model), 1 up, 2 down (d_model x d_ff).
 * gate and up are contiguous ([gate; up]). */
void* fbq_mlp_grad_ptr(void* mlp, int which);
/* Make `stream` wait until gradient `which` (0 dW_gate, 1 dW_up, 2 dW_down) of
 * the LAST enqueued backward is complete.  Each is final right after its own
 * GEMM (dW_down first, while the GLU backward and the gate/up GEMMs still run;
 * dW_gate while dW_up is computed): data-parallel callers all-reduce each on a
 * side stream overlapped with the rest of the backward. */
int fbq_mlp_wait_grad(void* mlp, int which, fbq_stream_t stream);
/* Copy gradients / fallback statistics to the host (synchronises). */
int fbq_mlp_get_grads(void* mlp, float* g_gate, float* g_up, float* g_down);
/* rates[2] = last fallback rate of gate/up and down; thresholds[2] likewise */
int fbq_mlp_get_controller(void* mlp, double* rates, double* thresholds);
/* QuantLinearLayer::apply_sgd (trainsim.cpp:137-143) on gate, up and down,
 * stream-ordered after the last backward (data parallel: after the dW
 * all-reduce).  Fused with the weight quantization the next forward would run
 * (fbq_cuda_sgd_quantize_rtn): that forward then uses the codes written here
 * instead of re-quantizing W -- the same codes, one pass over W instead of two.
 * A pending zero_grad makes it a no-op (the reference: w -= lr * 0). */
int fbq_mlp_apply_sgd(void* mlp, double lr, fbq_stream_t stream);
/* learning rate of the FBQ_STEP_SGD flag of fbq_mlp_step_host_async (default 0) */
int fbq_mlp_set_sgd_lr(void* mlp, double lr);
/* synchronous host copies of the fp32 master weights (gate, up: d_ff x
 * d_model; down: d_model x d_ff) */
int fbq_mlp_get_weights(void* mlp, float* w_gate, float* w_up, float* w_down);

/* ---- the reference's pre-norm residual GLU block: GluBlock (trainsim.hpp:136-146,
 * trainsim.cpp:294-308), out = h + down(silu(gate(norm(h))) * up(norm(h))), on the
 * MLP driver above plus an RmsNorm (gain initialised to 1, its 10-bit 1 x 128 input
 * context).  The norm runs fused into the gate/up input quantizer
 * (fbq_cuda_rmsnorm_quantize_input: norm(h) is never materialised), the residual
 * add rides on the down GEMM's accumulate epilogue, and the backward's norm
 * gradient and residual add are one pass (fbq_cuda_rmsnorm_backward_residual).
 * fbq_glublock_mlp returns the block's gate/up/down driver: fbq_mlp_controller_step,
 * _get_grads, _get_weights, _get_controller, _set_thresholds, _wait_grad, ... apply
 * to it.  h / out / grad_out / grad_h: device, tokens x d_model, act_dtype;
 * out must not alias h. */
void* fbq_glublock_create(const fbq_mlp_config* cfg, const float* w_gate, const float* w_up,
                          const float* w_down);
void fbq_glublock_destroy(void* block);
void* fbq_glublock_mlp(void* block);
int fbq_glublock_forward_device(void* block, const void* h, int64_t tokens, int64_t row_offset, int step,
                                void* out, fbq_stream_t stream);
int fbq_glublock_backward_device(void* block, const void* grad_out, int64_t tokens, int64_t row_offset,
                                 int step, void* grad_h, fbq_stream_t stream);
/* zero_grad of gate / up / down (deferred, as fbq_mlp_zero_grad) and of the gain */
int fbq_glublock_zero_grad(void* block, fbq_stream_t stream);
/* apply_sgd of gate / up / down (fused with the next weight RTN) and RmsNorm::apply_sgd */
int fbq_glublock_apply_sgd(void* block, double lr, fbq_stream_t stream);
/* synchronous host copies of the RmsNorm gain and its gradient (d_model floats) */
int fbq_glublock_get_gain(void* block, float* gain, float* grad_gain);
/* device pointers of the gain (which = 0) and grad_gain (1), d_model floats --
 * data parallel: grad_gain is summed over ranks after the backward */
float* fbq_glublock_gain_ptr(void* block, int which);

/* ---- one fallback-quantized linear layer: QuantLinearLayer (trainsim.hpp:38-73,
 * trainsim.cpp:61-135) with 128 x 128 blocks, 8-bit operands, the stochastic X
 * context, threshold fallback and the delay-threshold controller on device.
 * Layer RNG streams: layer_seed(seed, layer_id, tag 0 = context / 1 = dY, step). */
typedef struct fbq_linear_config {
  int64_t in_features;    /* K of the forward GEMM (% 16 == 0) */
  int64_t out_features;   /* N of the forward GEMM (% 16 == 0) */
  int64_t max_tokens;     /* capacity of the device workspaces */
  int act_dtype;          /* FBQ_F32 / FBQ_BF16: x, dY, y, dX */
  int epilogue;           /* FBQ_EPI_EXACT (bit-exact) or FBQ_EPI_FMA */
  int layer_id;           /* QuantLinearLayer layer_id (RNG stream) */
  uint64_t seed;          /* 0x5eed (QuantConfig::seed) */
  double threshold_init;  /* 1.0 */
  double r_min, r_max, alpha; /* 0.1, 0.3, 1.3 */
  int fallback_mode;      /* FallbackMode (trainsim.hpp:15): 0 Threshold, 1 FixedRate, 2 Off */
  double fixed_rate;      /* FixedRate: mask_topk(score_blocks(x), fixed_rate) on the device */
} fbq_linear_config;
void fbq_linear_default_config(fbq_linear_config* cfg);
/* weight: host fp32, out_features x in_features (row-major, like the reference) */
void* fbq_linear_create(const fbq_linear_config* cfg, const float* weight);
void fbq_linear_destroy(void* linear);
/* y = forward(x) (device buffers, tokens x in -> tokens x out); keeps the context */
int fbq_linear_forward_device(void* linear, const void* x, int64_t tokens, int64_t row_offset,
                              int step, void* y, fbq_stream_t stream);
/* dX = backward(dY); accumulates dW (fp32, device, fbq_linear_grad_ptr) */
int fbq_linear_backward_device(void* linear, const void* gy, int64_t tokens, int64_t row_offset,
                               int step, void* gx, fbq_stream_t stream);
int fbq_linear_controller_step(void* linear, fbq_stream_t stream);
/* data parallel, as fbq_mlp_count_ptr / fbq_mlp_controller_step_blocks (int32[1]) */
int32_t* fbq_linear_count_ptr(void* linear);
int fbq_linear_controller_step_blocks(void* linear, int64_t blocks, fbq_stream_t stream);
/* zero_grad is deferred like fbq_mlp_zero_grad: the next backward's dW GEMM
 * writes instead of accumulating; fbq_linear_grad_ptr materialises a pending
 * zero before returning the pointer. */
int fbq_linear_zero_grad(void* linear, fbq_stream_t stream);
float* fbq_linear_grad_ptr(void* linear);
/* last observed fallback rate (of the last forward, trainsim.cpp:93) and the
 * current threshold (synchronous read) */
int fbq_linear_get_controller(void* linear, double* last_rate, double* threshold);
/* QuantLinearLayer::apply_sgd (trainsim.cpp:137-143) on the device master weight */
int fbq_linear_apply_sgd(void* linear, double lr, fbq_stream_t stream);
/* synchronous host copies of the fp32 master weight / dW (out x in) */
int fbq_linear_get_weight(void* linear, float* w_host);
int fbq_linear_get_grad(void* linear, float* g_host);

/* ---- wire formats (host/io.cpp) ----
 * .fmat: the reference's dense fp32 matrix file (matrix.cpp:75-142), byte-
 * compatible, with its FormatError checks: FBQ_ERR_FORMAT + the reference's
 * byte offset (fbq_io_last_offset) and message (fbq_io_last_error).
 * .fqt: block-quantized / fallback tensor sidecar (codes, scales, bitmap,
 * residual plane; 128 x 128 blocks, 8 bits), host buffers. */
const char* fbq_io_last_error(void);
uint64_t fbq_io_last_offset(void);
int fbq_fmat_save(const char* path, const float* data, int64_t rows, int64_t cols);
int fbq_fmat_info(const char* path, int64_t* rows, int64_t* cols);
int fbq_fmat_load(const char* path, float* data, int64_t capacity, int64_t* rows, int64_t* cols);
int fbq_fqt_save(const char* path, int64_t rows, int64_t cols, const int8_t* codes, int64_t ldq,
                 const float* scales, const uint32_t* mask_bits, const int8_t* res_codes,
                 const float* res_scales);
int fbq_fqt_info(const char* path, int64_t* rows, int64_t* cols, int* has_fallback);
int fbq_fqt_load(const char* path, int8_t* codes, int64_t ldq, float* scales, uint32_t* mask_bits,
                 int8_t* res_codes, float* res_scales);

#ifdef __cplusplus
}
#endif
#endif /* FBQ_B200_HOST_H */
