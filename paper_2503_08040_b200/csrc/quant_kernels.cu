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
//      linear's K1): h = silu(a) * b from the gate/up GEMM output, 10-bit 1x128
//      RTN contexts of a and b, then K1 on h -- h itself never goes to HBM.
//  GLU backward (GluCombine::backward, trainsim.cpp:248-263, fused with the
//      gate/up linears' dY quantizer, trainsim.cpp:117-119): ga, gb from dH and
//      the dequantized contexts, stochastic-rounded straight into the int8 code
//      plane of [ga | gb].
//
// Work split: one 256-thread CTA per 128x128 block.  The raw block is staged
// in shared memory with one coalesced, vectorised HBM read (all loads issued
// before the first use); every later pass (absmax, RTN, stochastic planes,
// the fallback residual) streams it from smem in a compact per-row loop, so
// the kernels stay small (fully unrolling 64 values per thread through the
// rounding/RNG code produced ~15-30K-instruction kernels that thrashed the
// instruction cache).
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
template <>
__device__ __forceinline__ float to_f32<int16_t>(int16_t v) { return (float)v; }

template <typename T>
__device__ __forceinline__ T zero_of();
template <>
__device__ __forceinline__ float zero_of<float>() { return 0.0f; }
template <>
__device__ __forceinline__ __nv_bfloat16 zero_of<__nv_bfloat16>() { return __float2bfloat16(0.0f); }
template <>
__device__ __forceinline__ int16_t zero_of<int16_t>() { return 0; }

// Thread <-> element map of a 128 x 128 block for 16-byte vectors of T.
template <typename T>
struct Tiling {
  static constexpr int V = int(16 / sizeof(T));       // elements per vector
  static constexpr int VPR = kBlock / V;              // vectors per block row
  static constexpr int RPP = kQuantThreads / VPR;     // rows per pass
  static constexpr int NP = kBlock / RPP;             // passes
};
constexpr int kTileElems = kBlock * kBlock;

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

// Store V int8 codes: one vector store when the plane is 16-byte aligned and the
// vector is whole, else element stores (ragged right edge / odd strides).
template <int V>
__device__ __forceinline__ void store_codes(int8_t* p, const int* c, int n, bool vec) {
  if (vec && n == V) {
    if constexpr (V == 4) {
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
  } else {
#pragma unroll
    for (int i = 0; i < V; ++i)
      if (i < n) p[i] = (int8_t)c[i];
  }
}

template <int V>
__device__ __forceinline__ void store_codes16(int16_t* p, const int* c) {
  uint32_t w[V / 2];
#pragma unroll
  for (int i = 0; i < V / 2; ++i)
    w[i] = (uint32_t)(uint16_t)(int16_t)c[2 * i] | ((uint32_t)(uint16_t)(int16_t)c[2 * i + 1] << 16);
  if constexpr (V == 4) *reinterpret_cast<uint2*>(p) = make_uint2(w[0], w[1]);
  else *reinterpret_cast<uint4*>(p) = make_uint4(w[0], w[1], w[2], w[3]);
}

// ------------------------------------------------------------------ staging
// Copy a 128 x 128 block of T (row stride ld) into smem (row stride 128),
// zero-filling outside [rows) x [cols).  All vector loads are issued before the
// smem stores.  kVec requires 16-byte aligned rows and cols % V == 0.
template <typename T, bool kVec>
__device__ __forceinline__ void stage_tile(T* __restrict__ s, const T* __restrict__ g, int64_t ld,
                                           int64_t rows, int64_t cols, int64_t r0, int64_t c0) {
  using Tl = Tiling<T>;
  constexpr int V = Tl::V, VPR = Tl::VPR, RPP = Tl::RPP, NP = Tl::NP;
  const int lc = (threadIdx.x % VPR) * V, lr = threadIdx.x / VPR;
  if constexpr (kVec) {
    uint4 raw[NP];
#pragma unroll
    for (int ps = 0; ps < NP; ++ps) {
      const int64_t r = r0 + lr + ps * RPP, c = c0 + lc;
      raw[ps] = (r < rows && c < cols) ? __ldcs(reinterpret_cast<const uint4*>(g + r * ld + c))
                                       : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int ps = 0; ps < NP; ++ps)
      *reinterpret_cast<uint4*>(s + (lr + ps * RPP) * kBlock + lc) = raw[ps];
  } else {
#pragma unroll 4
    for (int i = threadIdx.x; i < kTileElems; i += kQuantThreads) {
      const int rr = i / kBlock, cc = i % kBlock;
      const int64_t r = r0 + rr, c = c0 + cc;
      s[i] = (r < rows && c < cols) ? g[r * ld + c] : zero_of<T>();
    }
  }
}

template <typename T, int V>
__device__ __forceinline__ void load_vec(const T* s, float (&v)[V]) {
  const uint4 raw = *reinterpret_cast<const uint4*>(s);
  const T* e = reinterpret_cast<const T*>(&raw);
#pragma unroll
  for (int i = 0; i < V; ++i) v[i] = to_f32(e[i]);
}

// ------------------------------------------------------------------ K1 core
// Per-block rounding dispatch, decided once per block (block-uniform): zero
// scale -> all codes 0; tiny scale -> the reference's double formula (out of
// line); otherwise the branch-free fp32 path.
template <int V>
__device__ __forceinline__ void rtn_vec(const float (&v)[V], float a, float inv_a, int mode,
                                        int (&code)[V]) {
  if (mode == 2) {
#pragma unroll
    for (int i = 0; i < V; ++i) code[i] = rtn_code_fast(v[i], a, inv_a, 127.0f);
  } else {
#pragma unroll
    for (int i = 0; i < V; ++i) code[i] = mode == 0 ? 0 : rtn_code_slow(v[i], a, 127.0f);
  }
}
template <int V>
__device__ __forceinline__ void sr_vec(const float (&v)[V], float a, float inv_a, int mode,
                                       uint64_t z, int (&code)[V]) {
#pragma unroll
  for (int i = 0; i < V; ++i) {
    code[i] = mode == 0 ? 0 : sr_code(v[i], a, inv_a, mix64(z));
    z += kGolden;
  }
}
__device__ __forceinline__ int round_mode(float a) {
  return a == 0.0f ? 0 : (a < kTinyScale ? 1 : 2);
}

// Quantize one 128 x 128 block whose values are produced on demand by
// `val(row_in_block, col_in_block, float (&v)[V])` (V consecutive columns).
// Fused outputs per QuantParams: scale, fallback flag, RTN codes, kSR (0-2)
// stochastic context planes and the fallback residual of flagged blocks.
// kSR is a compile-time count so RTN-only launches carry no RNG code.
// Entered by all threads of the CTA (it contains CTA barriers).
template <int V, int kSR, class Val>
__device__ __forceinline__ void quantize_block(const QuantParams& p, int64_t blk, int64_t r0,
                                               int64_t c0, float* red, Val&& val) {
  constexpr int VPR = kBlock / V, RPP = kQuantThreads / VPR, NP = kBlock / RPP;
  const int lc = (threadIdx.x % VPR) * V, lr = threadIdx.x / VPR;
  const int64_t cc = c0 + lc;
  const bool lane_ok = cc < p.cols;
  const int nvalid = (int)(p.cols - cc < V ? p.cols - cc : V);
  // ---- block absmax -> scale (quant.cpp:27-32) ----
  float m = 0.0f;
#pragma unroll 1
  for (int ps = 0; ps < NP; ++ps) {
    float v[V];
    val(lr + ps * RPP, lc, v);
#pragma unroll
    for (int i = 0; i < V; ++i) m = fmaxf(m, fabsf(v[i]));
  }
  const float amax = block_max(m, red);
  const float a = block_scale(amax);
  const float inv_a = a > 0.0f ? __frcp_rn(a) : 0.0f;
  const int mode = round_mode(a);

  bool flagged = false;
  if (p.mask_mode == kMaskThreshold) {
    const double theta = p.theta_dev ? *p.theta_dev : p.theta;
    flagged = (double)amax > theta;  // policy.cpp:77, strict, in double
  } else if (p.mask_mode == kMaskGiven) {
    flagged = (p.mask_bits[blk >> 5] >> (blk & 31)) & 1u;
  }
  if (threadIdx.x == 0) {
    if (p.scales) p.scales[blk] = a;
    if (p.amax_out) p.amax_out[blk] = amax;
    if (p.mask_mode == kMaskThreshold && flagged) atomicOr(p.mask_bits + (blk >> 5), 1u << (blk & 31));
    if (flagged && p.masked_count) atomicAdd(p.masked_count, 1);
    if (p.res_scales && !flagged) p.res_scales[blk] = 0.0f;
  }

  // ---- RTN codes + stochastic context planes (kernels.cpp:24-40, quant.cpp:66-80) ----
  if (lane_ok && (p.codes || kSR > 0)) {
#pragma unroll 1
    for (int ps = 0; ps < NP; ++ps) {
      const int rb = lr + ps * RPP;
      const int64_t r = r0 + rb;
      if (r >= p.rows) break;
      float v[V];
      val(rb, lc, v);
      int code[V];
      if (p.codes) {
        rtn_vec<V>(v, a, inv_a, mode, code);
        store_codes<V>(p.codes + r * p.ldq + cc, code, nvalid, p.vec_store);
      }
      if constexpr (kSR >= 1) {
        const uint64_t lin1 = (uint64_t)((p.row_offset + r) * p.cols + cc + 1);
        sr_vec<V>(v, a, inv_a, mode, p.sr_seed + lin1 * kGolden, code);
        store_codes<V>(p.sr_codes + r * p.ldq + cc, code, nvalid, p.vec_store);
        if constexpr (kSR >= 2) {
          sr_vec<V>(v, a, inv_a, mode, p.sr_seed2 + lin1 * kGolden, code);
          store_codes<V>(p.sr_codes2 + r * p.ldq + cc, code, nvalid, p.vec_store);
        }
      }
    }
  }
  if (!flagged) return;  // block-uniform

  // ---- fallback residual (quant.cpp:146-172): res = fl(x - fl(c*a)), recomputed
  //      from the staged values (no fp32 residual tile) ----
  auto res = [&](int rb, float (&v)[V]) {
    val(rb, lc, v);
    int c[V];
    rtn_vec<V>(v, a, inv_a, mode, c);
#pragma unroll
    for (int i = 0; i < V; ++i) v[i] = __fsub_rn(v[i], __fmul_rn((float)c[i], a));
  };
  m = 0.0f;
#pragma unroll 1
  for (int ps = 0; ps < NP; ++ps) {
    float v[V];
    res(lr + ps * RPP, v);
#pragma unroll
    for (int i = 0; i < V; ++i) m = fmaxf(m, fabsf(v[i]));
  }
  const float ra = block_scale(block_max(m, red));
  const float inv_ra = ra > 0.0f ? __frcp_rn(ra) : 0.0f;
  const int rmode = round_mode(ra);
  if (threadIdx.x == 0 && p.res_scales) p.res_scales[blk] = ra;
  if (!p.res_codes || !lane_ok) return;
#pragma unroll 1
  for (int ps = 0; ps < NP; ++ps) {
    const int rb = lr + ps * RPP;
    const int64_t r = r0 + rb;
    if (r >= p.rows) break;
    float v[V];
    res(rb, v);
    int code[V];
    rtn_vec<V>(v, ra, inv_ra, rmode, code);
    store_codes<V>(p.res_codes + r * p.ldq + cc, code, nvalid, p.vec_store);
  }
}

template <typename T, bool kVec, int kSR>
__global__ void __launch_bounds__(kQuantThreads)
fbq_quantize_block_kernel(QuantParams p) {
  extern __shared__ __align__(16) uint8_t dsm[];
  T* tile = reinterpret_cast<T*>(dsm);
  __shared__ float red[kQuantThreads / 32];
  const int64_t bj = blockIdx.x, bi = blockIdx.y;
  const int64_t r0 = bi * kBlock, c0 = bj * kBlock;
  stage_tile<T, kVec>(tile, reinterpret_cast<const T*>(p.x), p.ldx, p.rows, p.cols, r0, c0);
  __syncthreads();
  constexpr int V = Tiling<T>::V;
  quantize_block<V, kSR>(p, bi * gridDim.x + bj, r0, c0, red,
                         [&](int rb, int cb, float (&v)[V]) { load_vec<T, V>(tile + rb * kBlock + cb, v); });
}

// ------------------------------------------------------------------ GLU
// silu(x) = x / (1 + exp(-x)) evaluated like the reference (trainsim.cpp:38-46):
// double-precision exp and divide, rounded to float once (out of line).
__device__ __noinline__ float silu_ref(float x) {
  return (float)((double)x / (1.0 + exp(-(double)x)));
}
__device__ __noinline__ float silu_grad_ref(float x) {
  const double s = 1.0 / (1.0 + exp(-(double)x));
  return (float)(s * (1.0 + (double)x * (1.0 - s)));
}
// Fast fp32 variants for the bf16 training path (a few ulp from the reference).
__device__ __forceinline__ float sigmoid_fast(float x) { return __fdividef(1.0f, 1.0f + __expf(-x)); }
__device__ __forceinline__ float silu_fast(float x) { return x * sigmoid_fast(x); }
__device__ __forceinline__ float silu_grad_fast(float x) {
  const float s = sigmoid_fast(x);
  return s * (1.0f + x * (1.0f - s));
}

// 1 x 128 row-group RTN shared by the VPR threads of a row (quantize_rtn with
// GroupGeometry(1, 128), quant.cpp:36-53).
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
__global__ void __launch_bounds__(kQuantThreads)
fbq_glu_forward_kernel(GluParams g, QuantParams p) {
  // raw a and b tiles; h = silu(a) * b is recomputed from them on every pass
  extern __shared__ __align__(16) uint8_t dsm[];
  T* ta = reinterpret_cast<T*>(dsm);
  T* tb = ta + kTileElems;
  __shared__ float red[kQuantThreads / 32];
  using Tl = Tiling<T>;
  constexpr int V = Tl::V, VPR = Tl::VPR, RPP = Tl::RPP, NP = Tl::NP;
  const int64_t bj = blockIdx.x, bi = blockIdx.y;
  const int64_t r0 = bi * kBlock, c0 = bj * kBlock;
  const T* ab = reinterpret_cast<const T*>(g.ab);
  stage_tile<T, true>(ta, ab, g.ld_ab, g.rows, g.cols, r0, c0);
  stage_tile<T, true>(tb, ab + g.cols, g.ld_ab, g.rows, g.cols, r0, c0);
  __syncthreads();
  const int lc = (threadIdx.x % VPR) * V, lr = threadIdx.x / VPR;
  const int64_t gcols = (g.cols + kBlock - 1) / kBlock;
  const int64_t cc = c0 + lc;
  // 10-bit contexts of a and b (trainsim.cpp:240-243) [+ optional h_out]
#pragma unroll 1
  for (int ps = 0; ps < NP; ++ps) {
    const int rb = lr + ps * RPP;
    const int64_t r = r0 + rb;
    const bool ok = r < g.rows && cc < g.cols;  // cols % 8 == 0: uniform per row group
    float va[V], vb[V];
    load_vec<T, V>(ta + rb * kBlock + lc, va);
    load_vec<T, V>(tb + rb * kBlock + lc, vb);
    int code[V];
    float s = group_rtn<V, VPR>(va, code, g.ctx_level);
    if (ok && g.ctx_a) store_codes16<V>(g.ctx_a + r * g.ld_ctx + cc, code);
    if (ok && g.ctx_a_scales && lc == 0) g.ctx_a_scales[r * gcols + bj] = s;
    s = group_rtn<V, VPR>(vb, code, g.ctx_level);
    if (ok && g.ctx_b) store_codes16<V>(g.ctx_b + r * g.ld_ctx + cc, code);
    if (ok && g.ctx_b_scales && lc == 0) g.ctx_b_scales[r * gcols + bj] = s;
    if (ok && g.h_out) {
#pragma unroll
      for (int i = 0; i < V; ++i) {
        const float sa = g.exact_math ? silu_ref(va[i]) : silu_fast(va[i]);
        g.h_out[r * g.ld_h + cc + i] = __fmul_rn(sa, vb[i]);
      }
    }
  }
  // h = fl(silu(a) * b) (trainsim.cpp:230), quantized like a linear input
  quantize_block<V, 1>(p, bi * gridDim.x + bj, r0, c0, red, [&](int rb, int cb, float (&v)[V]) {
    float vb[V];
    load_vec<T, V>(ta + rb * kBlock + cb, v);
    load_vec<T, V>(tb + rb * kBlock + cb, vb);
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const float sa = g.exact_math ? silu_ref(v[i]) : silu_fast(v[i]);
      v[i] = __fmul_rn(sa, vb[i]);  // zero-filled lanes: silu(0) * 0 = 0
    }
  });
}

// SR-quantize one block whose values come from `val` into `dst` with its own
// RNG stream (quant.cpp:55-84); writes the block scale.
template <int V, class Val>
__device__ __forceinline__ void sr_block(int8_t* dst, int64_t ldq, float* scale_out, uint64_t seed,
                                         int64_t row_offset, int64_t rows, int64_t cols,
                                         int64_t r0, int64_t c0, float* red, Val&& val) {
  constexpr int VPR = kBlock / V, RPP = kQuantThreads / VPR, NP = kBlock / RPP;
  const int lc = (threadIdx.x % VPR) * V, lr = threadIdx.x / VPR;
  const int64_t cc = c0 + lc;
  float m = 0.0f;
#pragma unroll 1
  for (int ps = 0; ps < NP; ++ps) {
    float v[V];
    val(lr + ps * RPP, lc, v);
#pragma unroll
    for (int i = 0; i < V; ++i) m = fmaxf(m, fabsf(v[i]));
  }
  const float amax = block_max(m, red);
  const float a = block_scale(amax);
  const float inv_a = a > 0.0f ? __frcp_rn(a) : 0.0f;
  const int mode = round_mode(a);
  if (threadIdx.x == 0) *scale_out = a;
  if (cc >= cols) return;
#pragma unroll 1
  for (int ps = 0; ps < NP; ++ps) {
    const int rb = lr + ps * RPP;
    const int64_t r = r0 + rb;
    if (r >= rows) break;
    float v[V];
    val(rb, lc, v);
    int code[V];
    sr_vec<V>(v, a, inv_a, mode, seed + (uint64_t)((row_offset + r) * cols + cc + 1) * kGolden, code);
    store_codes<V>(dst + r * ldq + cc, code, V, true);
  }
}

template <typename T>
__global__ void __launch_bounds__(kQuantThreads)
fbq_glu_backward_kernel(GluBwdParams g) {
  extern __shared__ __align__(16) uint8_t dsm[];
  T* tg = reinterpret_cast<T*>(dsm);
  int16_t* tca = reinterpret_cast<int16_t*>(tg + kTileElems);
  int16_t* tcb = tca + kTileElems;
  __shared__ float sa_row[kBlock], sb_row[kBlock];
  __shared__ float red[kQuantThreads / 32];
  constexpr int V = Tiling<T>::V;
  const int64_t bj = blockIdx.x, bi = blockIdx.y;
  const int64_t r0 = bi * kBlock, c0 = bj * kBlock;
  const int64_t gcols = (g.cols + kBlock - 1) / kBlock;
  stage_tile<T, true>(tg, reinterpret_cast<const T*>(g.gh), g.ld_gh, g.rows, g.cols, r0, c0);
  stage_tile<int16_t, true>(tca, g.ctx_a, g.ld_ctx, g.rows, g.cols, r0, c0);
  stage_tile<int16_t, true>(tcb, g.ctx_b, g.ld_ctx, g.rows, g.cols, r0, c0);
  if (threadIdx.x < kBlock) {
    const int64_t r = r0 + threadIdx.x;
    sa_row[threadIdx.x] = r < g.rows ? g.ctx_a_scales[r * gcols + bj] : 0.0f;
    sb_row[threadIdx.x] = r < g.rows ? g.ctx_b_scales[r * gcols + bj] : 0.0f;
  }
  __syncthreads();
  // dequantized contexts: fl(code * scale) (quant.cpp:86-104); codes read as
  // one 16-byte smem vector per 8 values
  auto deq = [&](const int16_t* t, float s, int rb, int cb, float (&v)[V]) {
#pragma unroll
    for (int i = 0; i < V; ++i) v[i] = s == 0.0f ? 0.0f : __fmul_rn((float)t[rb * kBlock + cb + i], s);
  };
  // ga = fl(fl(gy * b) * silu'(a)),  gb = fl(gy * silu(a))   (trainsim.cpp:256-259)
  auto ga = [&](int rb, int cb, float (&v)[V]) {
    float a[V], b[V];
    load_vec<T, V>(tg + rb * kBlock + cb, v);
    deq(tca, sa_row[rb], rb, cb, a);
    deq(tcb, sb_row[rb], rb, cb, b);
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const float sg = g.exact_math ? silu_grad_ref(a[i]) : silu_grad_fast(a[i]);
      v[i] = __fmul_rn(__fmul_rn(v[i], b[i]), sg);
    }
  };
  auto gb = [&](int rb, int cb, float (&v)[V]) {
    float a[V];
    load_vec<T, V>(tg + rb * kBlock + cb, v);
    deq(tca, sa_row[rb], rb, cb, a);
#pragma unroll
    for (int i = 0; i < V; ++i)
      v[i] = __fmul_rn(v[i], g.exact_math ? silu_ref(a[i]) : silu_fast(a[i]));
  };
  if (g.g_out) {
    constexpr int VPR = kBlock / V, RPP = kQuantThreads / VPR, NP = kBlock / RPP;
    const int lc = (threadIdx.x % VPR) * V, lr = threadIdx.x / VPR;
#pragma unroll 1
    for (int ps = 0; ps < NP; ++ps) {
      const int rb = lr + ps * RPP;
      const int64_t r = r0 + rb;
      if (r >= g.rows || c0 + lc >= g.cols) continue;
      float v[V], w[V];
      ga(rb, lc, v);
      gb(rb, lc, w);
#pragma unroll
      for (int i = 0; i < V; ++i) {
        g.g_out[r * g.cols + c0 + lc + i] = v[i];
        g.g_out[g.rows * g.cols + r * g.cols + c0 + lc + i] = w[i];
      }
    }
  }
  sr_block<V>(g.gq, g.ldq, g.gq_scales + bi * (2 * gcols) + bj, g.seed_a, g.row_offset, g.rows,
              g.cols, r0, c0, red, ga);
  __syncthreads();
  sr_block<V>(g.gq + g.cols, g.ldq, g.gq_scales + bi * (2 * gcols) + gcols + bj, g.seed_b,
              g.row_offset, g.rows, g.cols, r0, c0, red, gb);
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

// ------------------------------------------------------------------ launchers
template <class K>
static cudaError_t opt_in_smem(K kernel, size_t bytes) {
  return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

template <typename T, bool kVec, int kSR>
static cudaError_t launch_k1_sr(const QuantParams& p, dim3 grid, cudaStream_t s) {
  const size_t smem = sizeof(T) * kTileElems;
  static bool ready = false;
  if (!ready) {
    if (cudaError_t e = opt_in_smem(fbq_quantize_block_kernel<T, kVec, kSR>, smem)) return e;
    ready = true;
  }
  fbq_quantize_block_kernel<T, kVec, kSR><<<grid, kQuantThreads, smem, s>>>(p);
  return cudaGetLastError();
}
template <typename T, bool kVec>
static cudaError_t launch_k1(QuantParams p, dim3 grid, cudaStream_t s) {
  // compact the stochastic planes into kSR = 0, 1, 2
  if (!p.sr_codes && p.sr_codes2) {
    p.sr_codes = p.sr_codes2;
    p.sr_seed = p.sr_seed2;
    p.sr_codes2 = nullptr;
  }
  if (p.sr_codes2) return launch_k1_sr<T, kVec, 2>(p, grid, s);
  if (p.sr_codes) return launch_k1_sr<T, kVec, 1>(p, grid, s);
  return launch_k1_sr<T, kVec, 0>(p, grid, s);
}

cudaError_t launch_quantize(const QuantParams& p, bool bf16, cudaStream_t s) {
  const dim3 grid((unsigned)((p.cols + kBlock - 1) / kBlock),
                  (unsigned)((p.rows + kBlock - 1) / kBlock));
  const size_t esz = bf16 ? 2 : 4;
  const bool vec = (reinterpret_cast<uintptr_t>(p.x) % 16 == 0) && ((p.ldx * esz) % 16 == 0) &&
                   (p.cols % (16 / esz) == 0);
  if (bf16) return vec ? launch_k1<__nv_bfloat16, true>(p, grid, s)
                       : launch_k1<__nv_bfloat16, false>(p, grid, s);
  return vec ? launch_k1<float, true>(p, grid, s) : launch_k1<float, false>(p, grid, s);
}

cudaError_t launch_glu_forward(const GluParams& g, const QuantParams& p, bool bf16,
                               cudaStream_t s) {
  const dim3 grid((unsigned)((g.cols + kBlock - 1) / kBlock),
                  (unsigned)((g.rows + kBlock - 1) / kBlock));
  if (bf16) {
    const size_t smem = 2 * sizeof(__nv_bfloat16) * kTileElems;
    if (cudaError_t e = opt_in_smem(fbq_glu_forward_kernel<__nv_bfloat16>, smem)) return e;
    fbq_glu_forward_kernel<__nv_bfloat16><<<grid, kQuantThreads, smem, s>>>(g, p);
  } else {
    const size_t smem = 2 * sizeof(float) * kTileElems;
    if (cudaError_t e = opt_in_smem(fbq_glu_forward_kernel<float>, smem)) return e;
    fbq_glu_forward_kernel<float><<<grid, kQuantThreads, smem, s>>>(g, p);
  }
  return cudaGetLastError();
}

cudaError_t launch_glu_backward(const GluBwdParams& g, bool bf16, cudaStream_t s) {
  const dim3 grid((unsigned)((g.cols + kBlock - 1) / kBlock),
                  (unsigned)((g.rows + kBlock - 1) / kBlock));
  if (bf16) {
    const size_t smem = (sizeof(__nv_bfloat16) + 2 * sizeof(int16_t)) * kTileElems;
    if (cudaError_t e = opt_in_smem(fbq_glu_backward_kernel<__nv_bfloat16>, smem)) return e;
    fbq_glu_backward_kernel<__nv_bfloat16><<<grid, kQuantThreads, smem, s>>>(g);
  } else {
    const size_t smem = (sizeof(float) + 2 * sizeof(int16_t)) * kTileElems;
    if (cudaError_t e = opt_in_smem(fbq_glu_backward_kernel<float>, smem)) return e;
    fbq_glu_backward_kernel<float><<<grid, kQuantThreads, smem, s>>>(g);
  }
  return cudaGetLastError();
}

cudaError_t launch_controller(double* theta, const int* masked_count, int64_t n_blocks,
                              double r_min, double r_max, double alpha, double* last_rate,
                              cudaStream_t s) {
  fbq_controller_kernel<<<1, 1, 0, s>>>(theta, masked_count, n_blocks, r_min, r_max, alpha,
                                        last_rate);
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
