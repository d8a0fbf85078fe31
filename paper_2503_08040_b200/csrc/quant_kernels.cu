// K1 / K2 / K4 and the fused GLU kernels: the HBM-bound block quantizers of
// the Fallback-Quantization path, hand-written for sm_100a.
//
//  K1  fbq_quantize_block_kernel  (quantize_rtn + score_blocks(AbsMax) +
//      mask_threshold + fallback_quantize + mask_rate count + up to two fused
//      stochastic "context" planes) -- reference quant.cpp:27-53, 128-176,
//      policy.cpp:18-27,73-87, quant.cpp:55-84.  X is read from HBM exactly once
//      (the reference reads it 3-4 times, plus once more per extra context).
//  K2  the same kernel with only the stochastic output enabled
//      (quantize_stochastic, quant.cpp:55-84).
//  K4  dequantize / dequantize_fallback (quant.cpp:86-104, 178-202), parity/debug.
//  GLU forward  (GluCombine::forward, trainsim.cpp:224-246, fused with the next
//      linear's K1): h = silu(a) * b computed in registers from the gate/up GEMM
//      output, 10-bit 1x128 RTN contexts of a and b, then K1 on h -- h itself
//      never goes to HBM.
//  GLU backward (GluCombine::backward, trainsim.cpp:248-263, fused with the
//      gate/up linears' dY quantizer, trainsim.cpp:117-119): ga, gb from dH and
//      the dequantized contexts, stochastic-rounded straight into the int8 code
//      plane of [ga | gb].
//
// Work split: one 256-thread CTA per 128x128 block.  Each thread keeps its 64
// elements in registers (16x 128-bit loads for fp32, 8 for bf16), so the
// residual pass of a flagged block (fallback) re-uses registers and never
// re-reads HBM.  Block absmax: warp shuffles + one smem exchange.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstdint>

#include "fbq_round.cuh"
#include "quant_kernels.cuh"

namespace fbq {

template <typename T>
__device__ __forceinline__ float to_f32(T v);
template <>
__device__ __forceinline__ float to_f32<float>(float v) { return v; }
template <>
__device__ __forceinline__ float to_f32<__nv_bfloat16>(__nv_bfloat16 v) {
  return __bfloat162float(v);
}

template <typename T, bool kVec>
struct Tiling {
  static constexpr int V = kVec ? int(16 / sizeof(T)) : 1;  // elements per load
  static constexpr int VPR = kBlock / V;                    // loads per block row
  static constexpr int RPP = kQuantThreads / VPR;           // rows per pass
  static constexpr int NP = kBlock / RPP;                   // passes
  static_assert(NP * V == 64, "64 elements per thread");
};

__device__ __forceinline__ float block_max(float v, float* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int warp = threadIdx.x >> 5;
  __syncthreads();  // protect `red` reuse across calls
  if ((threadIdx.x & 31) == 0) red[warp] = v;
  __syncthreads();
  float m = red[0];
#pragma unroll
  for (int w = 1; w < kQuantThreads / 32; ++w) m = fmaxf(m, red[w]);
  return m;
}

// max over the VPR threads that share one block row (a 1 x 128 group)
template <int VPR>
__device__ __forceinline__ float row_max(float v) {
#pragma unroll
  for (int o = VPR / 2; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

template <int V>
__device__ __forceinline__ void store_codes(int8_t* p, const int* c) {
  if constexpr (V == 1) {
    *p = (int8_t)c[0];
  } else if constexpr (V == 4) {
    uint32_t w = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) w |= (uint32_t)(uint8_t)(int8_t)c[i] << (8 * i);
    *reinterpret_cast<uint32_t*>(p) = w;
  } else {
    uint32_t w0 = 0, w1 = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      w0 |= (uint32_t)(uint8_t)(int8_t)c[i] << (8 * i);
      w1 |= (uint32_t)(uint8_t)(int8_t)c[i + 4] << (8 * i);
    }
    *reinterpret_cast<uint2*>(p) = make_uint2(w0, w1);
  }
}

template <int V>
__device__ __forceinline__ void store_codes16(int16_t* p, const int* c) {
  if constexpr (V == 1) {
    *p = (int16_t)c[0];
  } else {
    uint32_t w[V / 2];
#pragma unroll
    for (int i = 0; i < V / 2; ++i)
      w[i] = (uint32_t)(uint16_t)(int16_t)c[2 * i] | ((uint32_t)(uint16_t)(int16_t)c[2 * i + 1] << 16);
    if constexpr (V == 4) *reinterpret_cast<uint2*>(p) = make_uint2(w[0], w[1]);
    else *reinterpret_cast<uint4*>(p) = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

// Everything K1 does once the block's 64 values per thread are in registers:
// scale, fallback flag, RTN codes, stochastic context codes, residual.
template <int V, int NP, int RPP>
__device__ __forceinline__ void quantize_fragment(float (&v)[NP][V], const QuantParams& p,
                                                  int64_t blk, int64_t r0, int64_t c0, int lr,
                                                  int lc, float* red) {
  const int t = threadIdx.x;
  // ---- block absmax -> scale (quant.cpp:27-32) ----
  float m = 0.0f;
#pragma unroll
  for (int ps = 0; ps < NP; ++ps)
#pragma unroll
    for (int i = 0; i < V; ++i) m = fmaxf(m, fabsf(v[ps][i]));
  const float amax = block_max(m, red);
  const float a = block_scale(amax);
  const float inv_a = a > 0.0f ? __frcp_rn(a) : 0.0f;

  bool flagged = false;
  if (p.mask_mode == kMaskThreshold) {
    const double theta = p.theta_dev ? *p.theta_dev : p.theta;
    flagged = (double)amax > theta;  // policy.cpp:77, strict, in double
  } else if (p.mask_mode == kMaskGiven) {
    flagged = (p.mask_bits[blk >> 5] >> (blk & 31)) & 1u;
  }
  if (t == 0) {
    if (p.scales) p.scales[blk] = a;
    if (p.amax_out) p.amax_out[blk] = amax;
    if (p.mask_mode == kMaskThreshold && flagged) {
      atomicOr(p.mask_bits + (blk >> 5), 1u << (blk & 31));
    }
    if (flagged && p.masked_count) atomicAdd(p.masked_count, 1);
    if (p.res_scales && !flagged) p.res_scales[blk] = 0.0f;
  }

  // ---- primary RTN codes (kernels.cpp:24-40); zero-scale block -> 0 ----
  // Codes are produced and stored pass by pass (never held as arrays) to keep
  // the register footprint low enough for 2 CTAs/SM.
  const int64_t cc = c0 + lc;
  if (p.codes) {
#pragma unroll
    for (int ps = 0; ps < NP; ++ps) {
      int code[V];
#pragma unroll
      for (int i = 0; i < V; ++i) code[i] = a > 0.0f ? rtn_code(v[ps][i], a, inv_a) : 0;
      const int64_t r = r0 + lr + ps * RPP;
      if (r < p.rows && cc < p.cols) store_codes<V>(p.codes + r * p.ldq + cc, code);
    }
  }

  // ---- stochastic codes at global element index (quant.cpp:66-80) ----
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    int8_t* dst = k ? p.sr_codes2 : p.sr_codes;
    if (!dst) continue;
    const uint64_t seed = k ? p.sr_seed2 : p.sr_seed;
#pragma unroll
    for (int ps = 0; ps < NP; ++ps) {
      const int64_t r = r0 + lr + ps * RPP;
      uint64_t z = seed + (uint64_t)((p.row_offset + r) * p.cols + cc + 1) * kGolden;
      int sc[V];
#pragma unroll
      for (int i = 0; i < V; ++i) {
        sc[i] = a > 0.0f ? sr_code(v[ps][i], a, inv_a, mix64(z)) : 0;
        z += kGolden;
      }
      if (r < p.rows && cc < p.cols) store_codes<V>(dst + r * p.ldq + cc, sc);
    }
  }

  // ---- fallback residual for flagged blocks, from registers (quant.cpp:146-172) ----
  if (flagged) {  // block-uniform branch
    float m2 = 0.0f;
#pragma unroll
    for (int ps = 0; ps < NP; ++ps)
#pragma unroll
      for (int i = 0; i < V; ++i) {
        const int c = a > 0.0f ? rtn_code(v[ps][i], a, inv_a) : 0;
        const float rec = __fmul_rn((float)c, a);
        v[ps][i] = __fsub_rn(v[ps][i], rec);  // out-of-range lanes stay 0 - 0
        m2 = fmaxf(m2, fabsf(v[ps][i]));
      }
    const float ramax = block_max(m2, red);
    const float ra = block_scale(ramax);
    const float inv_ra = ra > 0.0f ? __frcp_rn(ra) : 0.0f;
    if (p.res_codes) {
#pragma unroll
      for (int ps = 0; ps < NP; ++ps) {
        int code[V];
#pragma unroll
        for (int i = 0; i < V; ++i) code[i] = ra > 0.0f ? rtn_code(v[ps][i], ra, inv_ra) : 0;
        const int64_t r = r0 + lr + ps * RPP;
        if (r < p.rows && cc < p.cols) store_codes<V>(p.res_codes + r * p.ldq + cc, code);
      }
    }
    if (t == 0 && p.res_scales) p.res_scales[blk] = ra;
  }
}

template <typename T, int V, int NP, int RPP, bool kVec>
__device__ __forceinline__ void load_tile(float (&v)[NP][V], const T* __restrict__ x, int64_t ldx,
                                          int64_t rows, int64_t cols, int64_t r0, int64_t c0,
                                          int lr, int lc) {
#pragma unroll
  for (int ps = 0; ps < NP; ++ps) {
    const int64_t r = r0 + lr + ps * RPP;
    const int64_t c = c0 + lc;
    if constexpr (kVec) {
      if (r < rows && c < cols) {
        const uint4 raw = __ldcs(reinterpret_cast<const uint4*>(x + r * ldx + c));
        const T* e = reinterpret_cast<const T*>(&raw);
#pragma unroll
        for (int i = 0; i < V; ++i) v[ps][i] = to_f32(e[i]);
      } else {
#pragma unroll
        for (int i = 0; i < V; ++i) v[ps][i] = 0.0f;
      }
    } else {
      v[ps][0] = (r < rows && c < cols) ? to_f32(x[r * ldx + c]) : 0.0f;
    }
  }
}

template <typename T, bool kVec>
__global__ void __launch_bounds__(kQuantThreads, 2)
fbq_quantize_block_kernel(QuantParams p) {
  using Tl = Tiling<T, kVec>;
  constexpr int V = Tl::V, VPR = Tl::VPR, RPP = Tl::RPP, NP = Tl::NP;
  __shared__ float red[kQuantThreads / 32];
  const int64_t bj = blockIdx.x, bi = blockIdx.y;
  const int64_t r0 = bi * kBlock, c0 = bj * kBlock;
  const int lc = (threadIdx.x % VPR) * V;  // local column of this thread's first element
  const int lr = threadIdx.x / VPR;        // local row of pass 0
  float v[NP][V];  // one HBM read of X
  load_tile<T, V, NP, RPP, kVec>(v, reinterpret_cast<const T*>(p.x), p.ldx, p.rows, p.cols, r0,
                                 c0, lr, lc);
  quantize_fragment<V, NP, RPP>(v, p, bi * gridDim.x + bj, r0, c0, lr, lc, red);
}

// ------------------------------------------------------------------ GLU
// silu(x) = x / (1 + exp(-x)) evaluated like the reference (trainsim.cpp:38-46):
// double-precision exp and divide, rounded to float once.
__device__ __forceinline__ float silu_ref(float x) {
  return (float)((double)x / (1.0 + exp(-(double)x)));
}
__device__ __forceinline__ float silu_grad_ref(float x) {
  const double s = 1.0 / (1.0 + exp(-(double)x));
  return (float)(s * (1.0 + (double)x * (1.0 - s)));
}

// 10-bit (or any <= 16-bit) RTN of one 1 x 128 row group shared by VPR threads
// (quantize_rtn with GroupGeometry(1, 128), quant.cpp:36-53).
template <int V, int VPR>
__device__ __forceinline__ float group_rtn(const float (&x)[V], int (&code)[V], float level) {
  float m = 0.0f;
#pragma unroll
  for (int i = 0; i < V; ++i) m = fmaxf(m, fabsf(x[i]));
  m = row_max<VPR>(m);
  const float s = m > 0.0f ? __fdiv_rn(m, level) : 0.0f;
  const float inv = s > 0.0f ? __frcp_rn(s) : 0.0f;
#pragma unroll
  for (int i = 0; i < V; ++i) code[i] = s > 0.0f ? rtn_code(x[i], s, inv, level) : 0;
  return s;
}

template <typename T>
__global__ void __launch_bounds__(kQuantThreads, 1)
fbq_glu_forward_kernel(GluParams g, QuantParams p) {
  using Tl = Tiling<T, true>;
  constexpr int V = Tl::V, VPR = Tl::VPR, RPP = Tl::RPP, NP = Tl::NP;
  __shared__ float red[kQuantThreads / 32];
  const int64_t bj = blockIdx.x, bi = blockIdx.y;
  const int64_t r0 = bi * kBlock, c0 = bj * kBlock;
  const int lc = (threadIdx.x % VPR) * V;
  const int lr = threadIdx.x / VPR;
  const T* ab = reinterpret_cast<const T*>(g.ab);
  float va[NP][V], vb[NP][V];
  load_tile<T, V, NP, RPP, true>(va, ab, g.ld_ab, g.rows, g.cols, r0, c0, lr, lc);
  load_tile<T, V, NP, RPP, true>(vb, ab + g.cols, g.ld_ab, g.rows, g.cols, r0, c0, lr, lc);
  const int64_t gcols = (g.cols + kBlock - 1) / kBlock;
  const int64_t cc = c0 + lc;
#pragma unroll
  for (int ps = 0; ps < NP; ++ps) {
    const int64_t r = r0 + lr + ps * RPP;
    const bool ok = r < g.rows && cc < g.cols;
    // 10-bit contexts of a and b (trainsim.cpp:240-243)
    int code[V];
    float s = group_rtn<V, VPR>(va[ps], code, g.ctx_level);
    if (ok && g.ctx_a) store_codes16<V>(g.ctx_a + r * g.ld_ctx + cc, code);
    if (ok && g.ctx_a_scales && lc == 0) g.ctx_a_scales[r * gcols + bj] = s;
    s = group_rtn<V, VPR>(vb[ps], code, g.ctx_level);
    if (ok && g.ctx_b) store_codes16<V>(g.ctx_b + r * g.ld_ctx + cc, code);
    if (ok && g.ctx_b_scales && lc == 0) g.ctx_b_scales[r * gcols + bj] = s;
    // h = fl(silu(a) * b)  (trainsim.cpp:230)
#pragma unroll
    for (int i = 0; i < V; ++i) va[ps][i] = ok ? __fmul_rn(silu_ref(va[ps][i]), vb[ps][i]) : 0.0f;
    if (ok && g.h_out) {
#pragma unroll
      for (int i = 0; i < V; ++i) g.h_out[r * g.ld_h + cc + i] = va[ps][i];
    }
  }
  quantize_fragment<V, NP, RPP>(va, p, bi * gridDim.x + bj, r0, c0, lr, lc, red);
}

// SR-quantize one 128x128 block held in registers into `dst` with its own
// RNG stream; returns nothing, writes the block scale.
template <int V, int NP, int RPP>
__device__ __forceinline__ void sr_fragment(const float (&v)[NP][V], int8_t* dst, int64_t ldq,
                                            float* scale_out, uint64_t seed, int64_t row_offset,
                                            int64_t rows, int64_t cols, int64_t r0, int64_t c0,
                                            int lr, int lc, float* red) {
  float m = 0.0f;
#pragma unroll
  for (int ps = 0; ps < NP; ++ps)
#pragma unroll
    for (int i = 0; i < V; ++i) m = fmaxf(m, fabsf(v[ps][i]));
  const float amax = block_max(m, red);
  const float a = block_scale(amax);
  const float inv_a = a > 0.0f ? __frcp_rn(a) : 0.0f;
  if (threadIdx.x == 0) *scale_out = a;
  const int64_t cc = c0 + lc;
#pragma unroll
  for (int ps = 0; ps < NP; ++ps) {
    const int64_t r = r0 + lr + ps * RPP;
    uint64_t z = seed + (uint64_t)((row_offset + r) * cols + cc + 1) * kGolden;
    int sc[V];
#pragma unroll
    for (int i = 0; i < V; ++i) {
      sc[i] = a > 0.0f ? sr_code(v[ps][i], a, inv_a, mix64(z)) : 0;
      z += kGolden;
    }
    if (r < rows && cc < cols) store_codes<V>(dst + r * ldq + cc, sc);
  }
}

template <typename T>
__global__ void __launch_bounds__(kQuantThreads, 2)
fbq_glu_backward_kernel(GluBwdParams g) {
  using Tl = Tiling<T, true>;
  constexpr int V = Tl::V, VPR = Tl::VPR, RPP = Tl::RPP, NP = Tl::NP;
  __shared__ float red[kQuantThreads / 32];
  const int64_t bj = blockIdx.x, bi = blockIdx.y;
  const int64_t r0 = bi * kBlock, c0 = bj * kBlock;
  const int lc = (threadIdx.x % VPR) * V;
  const int lr = threadIdx.x / VPR;
  const int64_t gcols = (g.cols + kBlock - 1) / kBlock;
  const int64_t cc = c0 + lc;
  const T* gh = reinterpret_cast<const T*>(g.gh);
  float v[NP][V];
  // pass 0: ga = fl(fl(gy * b) * silu'(a)); pass 1: gb = fl(gy * silu(a))   (trainsim.cpp:256-259)
#pragma unroll 1
  for (int which = 0; which < 2; ++which) {
    load_tile<T, V, NP, RPP, true>(v, gh, g.ld_gh, g.rows, g.cols, r0, c0, lr, lc);
#pragma unroll
    for (int ps = 0; ps < NP; ++ps) {
      const int64_t r = r0 + lr + ps * RPP;
      const bool ok = r < g.rows && cc < g.cols;
      const float sa = ok ? g.ctx_a_scales[r * gcols + bj] : 0.0f;
      const float sb = ok ? g.ctx_b_scales[r * gcols + bj] : 0.0f;
#pragma unroll
      for (int i = 0; i < V; ++i) {
        if (!ok) {
          v[ps][i] = 0.0f;
          continue;
        }
        // dequantize the contexts: fl(code * scale) (quant.cpp:86-104)
        const float a = sa == 0.0f ? 0.0f : __fmul_rn((float)g.ctx_a[r * g.ld_ctx + cc + i], sa);
        if (which == 0) {
          const float b = sb == 0.0f ? 0.0f : __fmul_rn((float)g.ctx_b[r * g.ld_ctx + cc + i], sb);
          v[ps][i] = __fmul_rn(__fmul_rn(v[ps][i], b), silu_grad_ref(a));
        } else {
          v[ps][i] = __fmul_rn(v[ps][i], silu_ref(a));
        }
        if (g.g_out) g.g_out[which * g.rows * g.cols + r * g.cols + cc + i] = v[ps][i];
      }
    }
    const int64_t gq_bj = which * gcols + bj;
    sr_fragment<V, NP, RPP>(v, g.gq + which * g.cols, g.ldq, g.gq_scales + bi * (2 * gcols) + gq_bj,
                            which ? g.seed_b : g.seed_a, g.row_offset, g.rows, g.cols, r0, c0, lr,
                            lc, red);
  }
}

// Delay-threshold controller on device (policy.cpp:97-109, Algorithm 2):
// rate = masked / blocks (policy.cpp:82-87); theta /= alpha below r_min,
// *= alpha above r_max.  Keeps the per-step update off the host.
__global__ void fbq_controller_kernel(double* theta, const int* masked_count, int64_t n_blocks,
                                      double r_min, double r_max, double alpha,
                                      double* last_rate) {
  const double rate = n_blocks > 0 ? (double)*masked_count / (double)n_blocks : 0.0;
  if (rate < r_min) *theta /= alpha;
  else if (rate > r_max) *theta *= alpha;
  if (last_rate) *last_rate = rate;
}

cudaError_t launch_controller(double* theta, const int* masked_count, int64_t n_blocks,
                              double r_min, double r_max, double alpha, double* last_rate,
                              cudaStream_t s) {
  fbq_controller_kernel<<<1, 1, 0, s>>>(theta, masked_count, n_blocks, r_min, r_max, alpha,
                                        last_rate);
  return cudaGetLastError();
}

// dequantize[_fallback]: y = fl(c*a) [+ fl(rc*ra)]  (quant.cpp:86-104, 178-202)
__global__ void fbq_dequantize_kernel(DequantParams p) {
  const int64_t n = p.rows * p.cols;
  const int64_t gc = (p.cols + kBlock - 1) / kBlock;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / p.cols, c = i % p.cols;
    const int64_t blk = (r / kBlock) * gc + c / kBlock;
    const float a = p.scales[blk];
    float y = a == 0.0f ? 0.0f : __fmul_rn((float)p.codes[r * p.ldq + c], a);
    if (p.mask_bits && ((p.mask_bits[blk >> 5] >> (blk & 31)) & 1u)) {
      y = __fadd_rn(y, __fmul_rn((float)p.res_codes[r * p.ldq + c], p.res_scales[blk]));
    }
    p.out[r * p.ldo + c] = y;
  }
}

// Element-wise rounding probes (exhaustive / adversarial tests of rtn_code
// and sr_code against the reference double formulas).
__global__ void fbq_round_probe_kernel(const float* x, const float* a, const uint64_t* bits,
                                       int8_t* out_rtn, int8_t* out_sr, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float ai = a[i];
    const float inv = __frcp_rn(ai);
    if (out_rtn) out_rtn[i] = (int8_t)rtn_code(x[i], ai, inv);
    if (out_sr) out_sr[i] = (int8_t)sr_code(x[i], ai, inv, bits[i]);
  }
}

cudaError_t launch_quantize(const QuantParams& p, bool bf16, cudaStream_t s) {
  const dim3 grid((unsigned)((p.cols + kBlock - 1) / kBlock),
                  (unsigned)((p.rows + kBlock - 1) / kBlock));
  const size_t esz = bf16 ? 2 : 4;
  const bool vec = (reinterpret_cast<uintptr_t>(p.x) % 16 == 0) && ((p.ldx * esz) % 16 == 0) &&
                   (p.cols % 8 == 0) && (p.ldq % 16 == 0);
  if (bf16) {
    if (vec) fbq_quantize_block_kernel<__nv_bfloat16, true><<<grid, kQuantThreads, 0, s>>>(p);
    else fbq_quantize_block_kernel<__nv_bfloat16, false><<<grid, kQuantThreads, 0, s>>>(p);
  } else {
    if (vec) fbq_quantize_block_kernel<float, true><<<grid, kQuantThreads, 0, s>>>(p);
    else fbq_quantize_block_kernel<float, false><<<grid, kQuantThreads, 0, s>>>(p);
  }
  return cudaGetLastError();
}

cudaError_t launch_glu_forward(const GluParams& g, const QuantParams& p, bool bf16,
                               cudaStream_t s) {
  const dim3 grid((unsigned)((g.cols + kBlock - 1) / kBlock),
                  (unsigned)((g.rows + kBlock - 1) / kBlock));
  if (bf16) fbq_glu_forward_kernel<__nv_bfloat16><<<grid, kQuantThreads, 0, s>>>(g, p);
  else fbq_glu_forward_kernel<float><<<grid, kQuantThreads, 0, s>>>(g, p);
  return cudaGetLastError();
}

cudaError_t launch_glu_backward(const GluBwdParams& g, bool bf16, cudaStream_t s) {
  const dim3 grid((unsigned)((g.cols + kBlock - 1) / kBlock),
                  (unsigned)((g.rows + kBlock - 1) / kBlock));
  if (bf16) fbq_glu_backward_kernel<__nv_bfloat16><<<grid, kQuantThreads, 0, s>>>(g);
  else fbq_glu_backward_kernel<float><<<grid, kQuantThreads, 0, s>>>(g);
  return cudaGetLastError();
}

cudaError_t launch_dequantize(const DequantParams& p, cudaStream_t s) {
  const int64_t n = p.rows * p.cols;
  int blocks = (int)((n + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  fbq_dequantize_kernel<<<blocks, 256, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_round_probe(const float* x, const float* a, const uint64_t* bits,
                               int8_t* out_rtn, int8_t* out_sr, int64_t n, cudaStream_t s) {
  int blocks = (int)((n + 255) / 256);
  if (blocks > 148 * 32) blocks = 148 * 32;
  if (blocks < 1) blocks = 1;
  fbq_round_probe_kernel<<<blocks, 256, 0, s>>>(x, a, bits, out_rtn, out_sr, n);
  return cudaGetLastError();
}

}  // namespace fbq
