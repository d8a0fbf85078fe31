#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace fbq {

enum EpilogueMode : int { kEpiExact = 0, kEpiFma = 1, kEpiDump = 2 };

struct GemmOperands {
  const int8_t* a_codes;
  int64_t lda;
  const int8_t* res_codes;  // same layout/ld as A, may be null
  const int8_t* b_codes;
  int64_t ldb;
};

struct GemmParams {
  int64_t M, N, K;
  int MB, NB, KB;  // ceil(M/128), ceil(N/128), ceil(K/128)
  int a_major, b_major;  // 0 = K-major, 1 = MN-major
  int64_t lds_a, lds_b;  // row strides of the stored scale grids (elements)
  const float* a_scales;
  const float* b_scales;
  const uint32_t* mask_bits;  // over A's stored block grid; null = block_quant_gemm
  const float* res_scales;
  void* out;
  int64_t ldo;
  int out_bf16;
  int accumulate;
  int vec_store;
  int tma_store;            // 0: direct stores; 1: staged TMA stores; 2: staged TMA reduce-add (fp32 accumulate)
  int32_t* dump;            // kEpiDump: [MB][NB][KB][128][128] primary, then residual
  int64_t dump_res_offset;  // element offset of the residual products
  int num_tiles;
  int group_m;    // tile raster: block-rows per group (bm fastest inside a group)
  int n_fastest;  // 1: bn fastest over the whole N (B stays L2-resident)
  int* tile_ctr;  // dynamic tile counter (zeroed before the launch) or null: static schedule
  float one;  // 1.0f (runtime constant for the exact epilogue)
  int diag;   // perf diagnostics: 1 = skip epilogue math, 2 = skip TMA loads
  long long* prof;  // perf diagnostics: 16 int64 per CTA (MMA-warp cycles, epilogue timeline) or null
};

// Per-device one-time setup (the dynamic tile-counter ring: one allocation
// + zeroing + sync); thread-safe, idempotent.  Until it has run on the current
// device launch_gemm uses the static tile schedule; it never allocates.
cudaError_t gemm_init();
cudaError_t launch_gemm(const GemmOperands& o, GemmParams p, int epi, cudaStream_t s);
int gemm_num_sms();
// The next self-resetting 128-byte counter slot of the current device's ring
// (two ints, both zero at rest; the kernel that uses it leaves them zero), or
// null before gemm_init() ran on the device.  Shared by the GEMM's and the
// quantizer's dynamic schedulers.
int* counter_slot();

}  // namespace fbq
