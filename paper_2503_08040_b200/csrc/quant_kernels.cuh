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
  int mask_mode;
  double theta;
  uint32_t* mask_bits;     // in (given) / out (threshold, pre-zeroed)
  int8_t* codes;           // may be null (SR-only launch)
  float* scales;           // may be null
  int8_t* res_codes;       // may be null
  float* res_scales;       // may be null
  int* masked_count;       // may be null (pre-zeroed)
  float* amax_out;         // may be null
  int8_t* sr_codes;        // may be null
  uint64_t sr_seed;
  int64_t row_offset;      // global row of this shard's row 0 (RNG index)
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
cudaError_t launch_dequantize(const DequantParams& p, cudaStream_t s);
cudaError_t launch_round_probe(const float* x, const float* a, const uint64_t* bits,
                               int8_t* out_rtn, int8_t* out_sr, int64_t n, cudaStream_t s);

}  // namespace fbq
