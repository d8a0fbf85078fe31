#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace fbq {

constexpr int kQuantThreads = 256;
enum MaskMode : int { kMaskNone = 0, kMaskThreshold = 1, kMaskGiven = 2 };

struct QuantParams {
  const void* x;       // rows x ldx, fp32 or bf16
  int64_t rows, cols, ldx;
  int64_t ldq;         // leading dim of every int8 code plane
  int vec_store;       // 1: all code planes 16-byte aligned with ldq % 16 == 0
  int mask_mode;
  double theta;
  const double* theta_dev;  // if non-null, the threshold is read on device (controller state)
  uint32_t* mask_bits;     // in (given) / out (threshold: every bit written, no pre-zeroing)
  int8_t* codes;           // may be null (SR-only launch)
  float* scales;           // may be null
  int8_t* res_codes;       // may be null
  float* res_scales;       // may be null
  int* masked_count;       // may be null; zeroed by launch_zero_count right before the grid
  int pdl;                 // 1: launched as a programmatic dependent of launch_zero_count
  float* amax_out;         // may be null
  int8_t* sr_codes;        // may be null
  uint64_t sr_seed;
  int8_t* sr_codes2;       // optional second stochastic plane (own seed), may be null
  uint64_t sr_seed2;
  int64_t row_offset;      // global row of this shard's row 0 (RNG index)
  int* blk_ctr;            // persistent K1: dynamic block counter slot (counter_slot()), or null
  int diag;                // A/B diagnostics inside the kernels (0 = production)
};

// GluCombine forward fused with the next linear's input quantizer.
struct GluParams {
  const void* ab;          // rows x ld_ab: a in cols [0, cols), b in [cols, 2 cols)
  int64_t rows, cols, ld_ab;
  uint8_t* ctx_a;          // 1 x 128 RTN contexts (int16 codes, or packed 10-bit planes), may be null
  uint8_t* ctx_b;
  int64_t ld_ctx;
  float* ctx_a_scales;     // rows x ceil(cols/128)
  float* ctx_b_scales;
  float ctx_level;         // 2^(bits-1) - 1 (511 for 10 bits)
  float* h_out;            // optional fp32 h (rows x ld_h), parity/debug
  int64_t ld_h;
  int exact_math;          // 1: silu like the reference (double); 0: fast fp32
  int ctx_packed;          // 1: packed 10-bit context planes (store_ctx10); 0: int16 codes
};

// GluCombine backward fused with the gate/up dY stochastic quantizers.
struct GluBwdParams {
  const void* gh;          // dH, rows x ld_gh
  int64_t rows, cols, ld_gh;
  const uint8_t* ctx_a;    // int16 codes or packed 10-bit planes (rows x ld_ctx)
  const uint8_t* ctx_b;
  int64_t ld_ctx;
  const float* ctx_a_scales;
  const float* ctx_b_scales;
  int8_t* gq;              // rows x ldq int8: [SR(ga) | SR(gb)]
  int64_t ldq;
  float* gq_scales;        // ceil(rows/128) x 2*ceil(cols/128)
  uint64_t seed_a, seed_b; // DeterministicRng seeds of the gate / up dY streams
  int64_t row_offset;
  float* g_out;            // optional fp32 [2][rows][cols] (ga, gb), parity/debug
  int exact_math;          // 1: silu / silu' like the reference (double); 0: fast fp32
  int ctx_packed;          // as GluParams::ctx_packed
};

struct DequantParams {
  const int8_t* codes;
  const float* scales;
  const uint32_t* mask_bits;  // null -> plain dequantize
  const int8_t* res_codes;
  const float* res_scales;
  int64_t rows, cols, ldq, ldo;
  float* out;
};

cudaError_t launch_quantize(const QuantParams& p, bool bf16, cudaStream_t s);
extern int g_quant_diag;
// RmsNorm forward / backward with the 10-bit 1 x 128 context (trainsim.cpp:154-211)
cudaError_t launch_rmsnorm_forward(const void* x, bool bf16, int64_t rows, int64_t cols, int64_t ldx,
                                   const float* gain, void* y, int64_t ldy, int16_t* ctx,
                                   int64_t ld_ctx, float* ctx_scales, float* rms, cudaStream_t s);
cudaError_t launch_rmsnorm_quantize(const QuantParams& p, bool bf16, const float* gain, int16_t* ctx,
                                    int64_t ld_ctx, float* ctx_scales, float* rms, cudaStream_t s);
cudaError_t launch_rmsnorm_backward(const int16_t* ctx, int64_t ld_ctx, const float* ctx_scales,
                                    const void* gy, bool bf16, int64_t rows, int64_t cols,
                                    int64_t ldgy, const float* gain, void* gx, int64_t ldgx,
                                    float* grad_gain, double* row_ws, float* term, cudaStream_t s,
                                    const void* res = nullptr, int64_t ldres = 0);
// mask_topk (policy.cpp:56-71) on device: exactly k blocks (policy_kernels.cu)
cudaError_t launch_topk(const float* scores, int64_t n, int64_t k, uint32_t* mask_bits,
                        int32_t* count, cudaStream_t s);  // 1 = one-block-per-CTA K1 (diagnostics, fbq_debug_set_quant_diag)
cudaError_t launch_dequantize(const DequantParams& p, cudaStream_t s);
cudaError_t launch_glu_forward(const GluParams& g, const QuantParams& p, bool bf16, cudaStream_t s);
cudaError_t launch_glu_backward(const GluBwdParams& g, bool bf16, cudaStream_t s);
cudaError_t launch_zero_count(int* count, cudaStream_t s);
cudaError_t launch_silu_forward(const void* x, bool bf16, int64_t rows, int64_t cols, int64_t ldx, void* y,
                                int64_t ldy, int16_t* ctx, int64_t ld_ctx, float* ctx_scales, float level,
                                bool exact, cudaStream_t s);
cudaError_t launch_silu_backward(const int16_t* ctx, int64_t ld_ctx, const float* ctx_scales, const void* gy,
                                 bool bf16, int64_t rows, int64_t cols, int64_t ldgy, void* gx, int64_t ldgx,
                                 bool exact, cudaStream_t s);
cudaError_t launch_sgd_quantize(float* w, const float* g, int64_t rows, int64_t cols, double lr,
                                int8_t* codes, int64_t ldq, float* scales, cudaStream_t s);
cudaError_t launch_controller(double* theta, const int* masked_count, int64_t n_blocks,
                              double r_min, double r_max, double alpha, double* last_rate,
                              cudaStream_t s);
cudaError_t launch_round_probe(const float* x, const float* a, const uint64_t* bits,
                               int8_t* out_rtn, int8_t* out_sr, int64_t n, int path, cudaStream_t s);

}  // namespace fbq
