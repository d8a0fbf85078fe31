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
#include <mutex>

#include <cuda.h>

#include "fbq_round.cuh"
#include "quant_kernels.cuh"
#include "gemm_kernel.cuh"
#include "sm100.cuh"

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

// Block-wide max with ONE barrier: `red` must not be re-written before every
// thread has read it -- callers give each call of a block its own 8-float slot
// and have a CTA barrier between blocks (the second slot serves the fallback
// residual; the TMA rings' slot-release barriers separate persistent blocks).
__device__ __forceinline__ float block_max_1b(float v, float* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
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

// Store V int8 codes given as 32-bit words whose low byte is the code (the
// magic-biased rounding words or plain ints): PRMT-packed into one vector store
// when the plane is 16-byte aligned and the vector is whole, else byte stores
// (ragged right edge / odd strides).
__device__ __forceinline__ uint32_t pack4_lo8(const uint32_t* w) {
  return __byte_perm(__byte_perm(w[0], w[1], 0x0040), __byte_perm(w[2], w[3], 0x0040), 0x5410);
}
template <int V>
__device__ __forceinline__ void store_codes(int8_t* p, const uint32_t* w, int n, bool vec) {
  if (vec && n == V) {
    if constexpr (V == 4) *reinterpret_cast<uint32_t*>(p) = pack4_lo8(w);
    else *reinterpret_cast<uint2*>(p) = make_uint2(pack4_lo8(w), pack4_lo8(w + 4));
  } else {
#pragma unroll
    for (int i = 0; i < V; ++i)
      if (i < n) p[i] = (int8_t)(uint8_t)w[i];
  }
}

// V int16 codes from words whose low halfword is the code
template <int V>
__device__ __forceinline__ void store_codes16(int16_t* p, const uint32_t* w) {
  uint32_t o[V / 2];
#pragma unroll
  for (int i = 0; i < V / 2; ++i) o[i] = __byte_perm(w[2 * i], w[2 * i + 1], 0x5410);
  if constexpr (V == 4) *reinterpret_cast<uint2*>(p) = make_uint2(o[0], o[1]);
  else *reinterpret_cast<uint4*>(p) = make_uint4(o[0], o[1], o[2], o[3]);
}

// ---- packed 10-bit context planes (GluCombine's a / b contexts, trainsim.cpp:240-243)
// A context of rows x cols codes (|code| <= 511) with row stride ld (elements,
// ld % 16 == 0) is stored as 10 bits per code: the LOW byte of every code
// (int8 [rows][ld]) followed by the top two bits of the 10-bit two's
// complement, four codes per byte ([rows][ld / 4], code c at bits 2 (c % 4)).
// 1.25 bytes per element = 5/8 of bf16.
template <int V>
__device__ __forceinline__ void store_ctx10(uint8_t* lo, uint8_t* hi, const uint32_t* w) {
  if constexpr (V == 8) *reinterpret_cast<uint2*>(lo) = make_uint2(pack4_lo8(w), pack4_lo8(w + 4));
  else *reinterpret_cast<uint32_t*>(lo) = pack4_lo8(w);
  uint32_t h = 0;
#pragma unroll
  for (int i = 0; i < V; ++i) h |= ((w[i] >> 8) & 3u) << (2 * i);
  if constexpr (V == 8) *reinterpret_cast<uint16_t*>(hi) = (uint16_t)h;
  else *hi = (uint8_t)h;
}
// V codes as int32 scaled by 2^22 (exact: |code| < 2^9): the low byte shifted to
// bits 22-29 and the two top bits to bits 30-31 -- two shifts and one LOP3 per
// code; the caller folds 2^-22 into the scale.
template <int V>
__device__ __forceinline__ void load_ctx10_x4m(const uint8_t* lo, const uint8_t* hi, int32_t (&c)[V]) {
  uint32_t L[V / 4], H;
  if constexpr (V == 8) {
    const uint2 l = *reinterpret_cast<const uint2*>(lo);
    L[0] = l.x;
    L[1] = l.y;
    H = *reinterpret_cast<const uint16_t*>(hi);
  } else {
    L[0] = *reinterpret_cast<const uint32_t*>(lo);
    H = *hi;
  }
#pragma unroll
  for (int i = 0; i < V; ++i) {
    const int k = i & 3;
    const uint32_t lb = k <= 2 ? (L[i >> 2] << (22 - 8 * k)) : (L[i >> 2] >> (8 * k - 22));
    const uint32_t hb = 30 >= 2 * i ? (H << (30 - 2 * i)) : (H >> (2 * i - 30));
    c[i] = (int32_t)((lb & 0x3FC00000u) | (hb & 0xC0000000u));
  }
}

// ------------------------------------------------------------------ staging
// Copy a 128 x 128 block of T (row stride ld) into smem (row stride 128),
// zero-filling outside [rows) x [cols).  All vector loads are issued before the
// smem stores.  kVec requires 16-byte aligned rows and cols % V == 0.
template <typename T, bool kVec>
__device__ __forceinline__ void stage_tile(T* __restrict__ s, const T* __restrict__ g, int64_t ld,
                                           int64_t rows, int64_t cols, int64_t r0, int64_t c0,
                                           int sld = kBlock) {
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
      *reinterpret_cast<uint4*>(s + (lr + ps * RPP) * sld + lc) = raw[ps];
  } else {
#pragma unroll 4
    for (int i = threadIdx.x; i < kTileElems; i += kQuantThreads) {
      const int rr = i / kBlock, cc = i % kBlock;
      const int64_t r = r0 + rr, c = c0 + cc;
      s[rr * sld + cc] = (r < rows && c < cols) ? g[r * ld + c] : zero_of<T>();
    }
  }
}

template <typename T, int V>
__device__ __forceinline__ void load_vec(const T* s, float (&v)[V]) {
  if constexpr (V * sizeof(T) == 32) {  // 8 floats: two 16-byte loads
    const float4 x = reinterpret_cast<const float4*>(s)[0], y = reinterpret_cast<const float4*>(s)[1];
    v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w; v[4] = y.x; v[5] = y.y; v[6] = y.z; v[7] = y.w;
  } else {
    const uint4 raw = *reinterpret_cast<const uint4*>(s);
    const T* e = reinterpret_cast<const T*>(&raw);
#pragma unroll
    for (int i = 0; i < V; ++i) v[i] = to_f32(e[i]);
  }
}
template <int V>
__device__ __forceinline__ void store_f32(float* s, const float (&v)[V]) {
#pragma unroll
  for (int j = 0; j < V / 4; ++j)
    reinterpret_cast<float4*>(s)[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
}

// ------------------------------------------------------------------ K1 core
// Per-block rounding dispatch, decided once per block (block-uniform): zero
// scale -> all codes 0; tiny scale -> the reference's double formula (out of
// line); otherwise the fp32 vector fast path with its exact fallback.
// Outputs are words whose low byte is the code.
template <int V>
__device__ __forceinline__ void rtn_vec(const float (&v)[V], float a, float inv_a, int mode,
                                        uint32_t (&w)[V]) {
  if (mode == 2) {
    if constexpr (V % 2 == 0) {
      if (rtn_fast_vec_x<V>(v, a, inv_a, w)) rtn_fix_vec<V>(v, a, w);
    } else {
      if (rtn_fast_vec<V>(v, inv_a, rtn_window(127.0f), w)) rtn_exact_vec<V>(v, a, inv_a, 127.0f, w);
    }
  } else {
#pragma unroll
    for (int i = 0; i < V; ++i) w[i] = mode == 0 ? 0u : (uint32_t)rtn_code_slow(v[i], a, 127.0f);
  }
}
template <int V>
__device__ __forceinline__ void sr_vec(const float (&v)[V], float a, float inv_a, int mode,
                                       uint64_t z, uint32_t (&w)[V]) {
  if (mode == 2) {
    if (sr_fast_vec<V>(v, inv_a, z, w)) sr_exact_vec<V>(v, a, inv_a, z, w);
  } else {
#pragma unroll
    for (int i = 0; i < V; ++i) {
      w[i] = mode == 0 ? 0u : (uint32_t)sr_code_slow(v[i], a, mix64(z));
      z += kGolden;
    }
  }
}
__device__ __forceinline__ int round_mode(float a) {
  return a == 0.0f ? 0 : (a < kTinyScale ? 1 : 2);
}

// x -> fl(x - fl(c a)) in place, c = RTN code of x (the fallback residual,
// quant.cpp:150-156).  Fast mode: c from the magic words (n = m - M exactly).
template <int V>
__device__ __forceinline__ void residual_vec(float (&v)[V], float a, float inv_a, int mode) {
  if (mode == 2) {
    uint32_t w[V];
    if (rtn_fast_vec_x<V>(v, a, inv_a, w)) rtn_fix_vec<V>(v, a, w);
    const float2 nmag = make_float2(-kMagic, -kMagic), a2 = make_float2(a, a);
#pragma unroll
    for (int i = 0; i < V; i += 2) {
      const float2 n = __fadd2_rn(make_float2(__uint_as_float(w[i]), __uint_as_float(w[i + 1])), nmag);
      const float2 rec = __fmul2_rn(n, a2);                       // fl(c * a)
      const float2 r = __fadd2_rn(make_float2(v[i], v[i + 1]), make_float2(-rec.x, -rec.y));
      v[i] = r.x;
      v[i + 1] = r.y;
    }
  } else if (mode == 1) {
#pragma unroll
    for (int i = 0; i < V; ++i) v[i] = __fsub_rn(v[i], __fmul_rn((float)rtn_code_slow(v[i], a, 127.0f), a));
  }  // mode 0: a == 0, codes 0, residual = x
}

// Quantize one 128 x 128 block whose values are produced on demand by
// `val(row_in_block, col_in_block, float (&v)[V])` (V consecutive columns).
// Fused outputs per QuantParams: scale, fallback flag, RTN codes, kSR (0-2)
// stochastic context planes and the fallback residual of flagged blocks.
// kSR is a compile-time count so RTN-only launches carry no RNG code.
// Entered by all threads of the CTA (it contains CTA barriers).
// have_m: the caller already holds this thread's partial absmax `m_in` (and
// the block barrier in block_max publishes the values `val` reads).
// Threshold mode writes the block's own mask bit either way (set or clear),
// so the bitmap needs no zeroing pass; the last block also clears the unused
// tail bits of the final word.  The masked-block count is the one value that
// must start at zero: it is zeroed by fbq_zero_count_kernel launched just
// before this grid, which this grid may overlap (programmatic dependent
// launch) up to the griddepcontrol.wait in front of the first atomicAdd.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void publish_flag(const QuantParams& p, int64_t blk, bool flagged) {
  if (p.mask_mode == kMaskThreshold) {
    const uint32_t bit = 1u << (blk & 31);
    if (flagged) atomicOr(p.mask_bits + (blk >> 5), bit);
    else atomicAnd(p.mask_bits + (blk >> 5), ~bit);
    const int64_t last = ((p.rows + kBlock - 1) / kBlock) * ((p.cols + kBlock - 1) / kBlock) - 1;
    if (blk == last && (last & 31) != 31) atomicAnd(p.mask_bits + (blk >> 5), (bit << 1) - 1u);
  }
  if (flagged && p.masked_count) {
    pdl_wait();
    atomicAdd(p.masked_count, 1);
  }
}

template <int V, int kSR, class Val>
__device__ __forceinline__ void quantize_block(const QuantParams& p, int64_t blk, int64_t r0,
                                               int64_t c0, float* red, Val&& val,
                                               bool have_m = false, float m_in = 0.0f) {
  constexpr int VPR = kBlock / V, RPP = kQuantThreads / VPR, NP = kBlock / RPP;
  const int lc = (threadIdx.x % VPR) * V, lr = threadIdx.x / VPR;
  const int64_t cc = c0 + lc;
  const bool lane_ok = cc < p.cols;
  const int nvalid = (int)(p.cols - cc < V ? p.cols - cc : V);
  // ---- block absmax -> scale (quant.cpp:27-32) ----
  float m = m_in;
  if (!have_m) {
#pragma unroll 1
    for (int ps = 0; ps < NP; ++ps) {
      float v[V];
      val(lr + ps * RPP, lc, v);
#pragma unroll
      for (int i = 0; i < V; ++i) m = fmaxf(m, fabsf(v[i]));
    }
  }
  const float amax = block_max_1b(m, red);  // slot 0 (callers give red 2 x 8 floats)
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
    publish_flag(p, blk, flagged);
    if (p.res_scales && !flagged) p.res_scales[blk] = 0.0f;
  }

  // ---- RTN codes + stochastic context planes (kernels.cpp:24-40, quant.cpp:66-80) ----
  // (a flagged block's residual absmax rides along with its code pass)
  float rm = 0.0f;
  const bool fuse_rm = (V % 2 == 0) && flagged && mode == 2 && p.codes != nullptr;  // words = magic words
  if (lane_ok && (p.codes || kSR > 0)) {
#pragma unroll 1
    for (int ps = 0; ps < NP; ++ps) {
      const int rb = lr + ps * RPP;
      const int64_t r = r0 + rb;
      if (r >= p.rows) break;
      float v[V];
      val(rb, lc, v);
      uint32_t code[V];
      if (p.codes) {
        rtn_vec<V>(v, a, inv_a, mode, code);
        if (fuse_rm) {
#pragma unroll
          for (int i = 0; i < V; ++i) {  // fl(x - fl(c a)), c = m - M exactly
            const float n = __fsub_rn(__uint_as_float(code[i]), kMagic);
            rm = fmaxf(rm, fabsf(__fsub_rn(v[i], __fmul_rn(n, a))));
          }
        }
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
    if (mode == 2) {
      // code as a float straight from the magic words (n = m - M exactly): no I2F
      residual_vec<V>(v, a, inv_a, mode);
      return;
    }
    uint32_t c[V];
    rtn_vec<V>(v, a, inv_a, mode, c);
#pragma unroll
    for (int i = 0; i < V; ++i) v[i] = __fsub_rn(v[i], __fmul_rn((float)(int8_t)(uint8_t)c[i], a));
  };
  if (!fuse_rm) {
#pragma unroll 1
    for (int ps = 0; ps < NP; ++ps) {
      float v[V];
      res(lr + ps * RPP, v);
#pragma unroll
      for (int i = 0; i < V; ++i) rm = fmaxf(rm, fabsf(v[i]));
    }
  }
  const float ra = block_scale(block_max_1b(rm, red + kQuantThreads / 32));  // slot 1
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
    uint32_t code[V];
    rtn_vec<V>(v, ra, inv_ra, rmode, code);
    store_codes<V>(p.res_codes + r * p.ldq + cc, code, nvalid, p.vec_store);
  }
}

template <typename T, bool kVec, int kSR, int kMinBlocks = 1>
__global__ void __launch_bounds__(kQuantThreads, kMinBlocks)
fbq_quantize_block_kernel(QuantParams p) {
  extern __shared__ __align__(16) uint8_t dsm[];
  T* tile = reinterpret_cast<T*>(dsm);
  __shared__ float red[2 * (kQuantThreads / 32)];
  const int64_t bj = blockIdx.x, bi = blockIdx.y;
  const int64_t r0 = bi * kBlock, c0 = bj * kBlock;
  stage_tile<T, kVec>(tile, reinterpret_cast<const T*>(p.x), p.ldx, p.rows, p.cols, r0, c0);
  __syncthreads();
  constexpr int V = Tiling<T>::V;
  quantize_block<V, kSR>(p, bi * gridDim.x + bj, r0, c0, red,
                         [&](int rb, int cb, float (&v)[V]) { load_vec<T, V>(tile + rb * kBlock + cb, v); });
}

// ------------------------------------------------------------------ K1, register-resident
// The RTN / fallback-detect path (no stochastic planes): every thread keeps its
// 64 values of the block in registers as loaded (32 registers of packed bf16 or
// 64 of fp32) -- no shared-memory staging, one unpack per pass, row pointers
// hoisted out of the pass loop.  The smem-staged K1 above spends ~22
// instructions per element (issue-bound at ~52 % of HBM on 8192 x 14336 bf16);
// this one ~8.
template <typename T>
__device__ __forceinline__ void unpack(const uint4& raw, float (&v)[16 / sizeof(T)]) {
  if constexpr (sizeof(T) == 2) {
    const uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      v[2 * i] = __uint_as_float(w[i] << 16);
      v[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
    }
  } else {
    v[0] = __uint_as_float(raw.x);
    v[1] = __uint_as_float(raw.y);
    v[2] = __uint_as_float(raw.z);
    v[3] = __uint_as_float(raw.w);
  }
}
template <typename T>
__device__ __noinline__ uint2 rtn_slow_raw(uint4 raw, float a, float level) {
  constexpr int V = 16 / sizeof(T);
  float v[V];
  unpack<T>(raw, v);
  uint32_t w[V];
#pragma unroll
  for (int i = 0; i < V; ++i) w[i] = (uint32_t)rtn_code_slow(v[i], a, level);
  uint2 out;
  out.x = pack4_lo8(w);
  out.y = V == 8 ? pack4_lo8(w + 4) : 0u;
  return out;
}
// A vector whose boundary test fired (~20 % of bf16 vectors): fast path again
// plus the exact packed correction, out of line so the 8x-unrolled main path
// of the 80-register persistent variant stays spill-free.
template <typename T>
__device__ __noinline__ uint2 rtn_fix_raw(uint4 raw, float a, float inv_a) {
  constexpr int V = 16 / sizeof(T);
  float v[V];
  unpack<T>(raw, v);
  uint32_t w[V];
  rtn_fast_vec<V>(v, inv_a, rtn_window(127.0f), w);
  rtn_fix_vec<V>(v, a, w);
  uint2 out;
  out.x = pack4_lo8(w);
  out.y = V == 8 ? pack4_lo8(w + 4) : 0u;
  return out;
}
// RTN codes of one vector, packed (V = 8: 8 bytes, V = 4: 4 bytes in .x).
// mode: 0 zero scale, 1 tiny scale (reference double path), 2 fast path.
template <typename T>
__device__ __forceinline__ uint2 rtn_raw(const uint4& raw, float a, float inv_a, int mode) {
  constexpr int V = 16 / sizeof(T);
  if (mode == 2) {
    float v[V];
    unpack<T>(raw, v);
    uint32_t w[V];
    if (rtn_fast_vec_x<V>(v, a, inv_a, w)) return rtn_fix_raw<T>(raw, a, inv_a);
    uint2 out;
    out.x = pack4_lo8(w);
    out.y = V == 8 ? pack4_lo8(w + 4) : 0u;
    return out;
  }
  if (mode == 1) return rtn_slow_raw<T>(raw, a, 127.0f);
  return make_uint2(0u, 0u);
}
// the same, out of line: the fallback residual of flagged blocks recomputes
// the primary codes through this (keeps the unrolled main path small)
template <typename T>
__device__ __noinline__ uint2 rtn_raw_call(uint4 raw, float a, float inv_a, int mode) {
  return rtn_raw<T>(raw, a, inv_a, mode);
}
__device__ __forceinline__ float code_of(const uint2& c, int i) {
  const uint32_t w = i < 4 ? c.x : c.y;
  return (float)(int8_t)(uint8_t)(w >> (8 * (i & 3)));
}

// Out of line (flagged blocks only; keeps the main path's registers): the
// primary codes of one raw vector together with its residual's absmax (the code
// pass of a flagged block), the residual's absmax alone, and the residual RTN
// codes (packed).
struct CodeMax {
  uint2 code;
  float rm;
};
template <typename T>
__device__ __noinline__ CodeMax rtn_resmax_raw(uint4 raw, float a, float inv_a, int mode) {
  constexpr int V = 16 / sizeof(T);
  float v[V];
  unpack<T>(raw, v);
  uint32_t w[V];
  CodeMax out;
  out.rm = 0.0f;
  if (mode == 2) {
    if (rtn_fast_vec_x<V>(v, a, inv_a, w)) rtn_fix_vec<V>(v, a, w);
    const float2 nmag = make_float2(-kMagic, -kMagic), a2 = make_float2(a, a);
#pragma unroll
    for (int i = 0; i < V; i += 2) {
      const float2 n = __fadd2_rn(make_float2(__uint_as_float(w[i]), __uint_as_float(w[i + 1])), nmag);
      const float2 rec = __fmul2_rn(n, a2);  // fl(c * a)
      const float2 r = __fadd2_rn(make_float2(v[i], v[i + 1]), make_float2(-rec.x, -rec.y));
      out.rm = fmaxf(out.rm, fmaxf(fabsf(r.x), fabsf(r.y)));
    }
  } else {
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const int c = mode == 1 ? rtn_code_slow(v[i], a, 127.0f) : 0;
      w[i] = (uint32_t)c;
      out.rm = fmaxf(out.rm, fabsf(__fsub_rn(v[i], __fmul_rn((float)c, a))));
    }
  }
  out.code = make_uint2(pack4_lo8(w), V == 8 ? pack4_lo8(w + 4) : 0u);
  return out;
}
template <typename T>
__device__ __noinline__ float residual_absmax_raw(uint4 raw, float a, float inv_a, int mode) {
  constexpr int V = 16 / sizeof(T);
  float v[V];
  unpack<T>(raw, v);
  residual_vec<V>(v, a, inv_a, mode);
  float m = 0.0f;
#pragma unroll
  for (int i = 0; i < V; ++i) m = fmaxf(m, fabsf(v[i]));
  return m;
}
template <typename T>
__device__ __noinline__ uint2 residual_codes_raw(uint4 raw, float a, float inv_a, int mode, float ra,
                                                 float inv_ra, int rmode) {
  constexpr int V = 16 / sizeof(T);
  float v[V];
  unpack<T>(raw, v);
  residual_vec<V>(v, a, inv_a, mode);
  uint32_t w[V];
  rtn_vec<V>(v, ra, inv_ra, rmode, w);
  return make_uint2(pack4_lo8(w), V == 8 ? pack4_lo8(w + 4) : 0u);
}

// One block's work given its raw values in registers (all threads; contains
// CTA barriers).
template <typename T, int kSR = 0>
__device__ __forceinline__ void quantize_block_reg(const QuantParams& p, int64_t bi, int64_t bj,
                                                   int64_t blk, const uint4 (&raw)[Tiling<T>::NP],
                                                   float* red) {
  using Tl = Tiling<T>;
  constexpr int V = Tl::V, VPR = Tl::VPR, RPP = Tl::RPP, NP = Tl::NP;
  const int lc = (threadIdx.x % VPR) * V, lr = threadIdx.x / VPR;
  const int64_t r0 = bi * kBlock + lr, cc = bj * kBlock + lc;
  const bool col_ok = cc < p.cols;  // cols % V == 0: whole vectors
  const int64_t left = p.rows - r0;  // rows from this thread's first row to the end
  const int nrow = left <= 0 ? 0 : (left >= (int64_t)NP * RPP ? NP : (int)((left + RPP - 1) / RPP));
  // ---- block absmax -> scale (quant.cpp:27-32) ----
  float m = 0.0f;
  if constexpr (sizeof(T) == 2) {
    // |bf16| orders like its low 15 bits as an unsigned integer: packed 16x2
    // integer max on the raw words, no unpacking (LOP3 + VIMNMX3.U16x2)
    // No masking per word: the SIGNED 16-bit max (from 0) picks the largest
    // non-negative value, the UNSIGNED max the largest-magnitude negative one
    // (if any; sign-magnitude orders like the raw bits), so
    // max|x| = max(smax, umax & 0x7FFF) -- one 3-input VIMNMX3 per two words
    // per accumulator instead of a LOP3 per word.
    uint32_t ms = 0, mu = 0;
#pragma unroll
    for (int ps = 0; ps < NP; ++ps) {
      ms = __vimax3_s16x2(ms, raw[ps].x, raw[ps].y);
      ms = __vimax3_s16x2(ms, raw[ps].z, raw[ps].w);
      mu = __vimax3_u16x2(mu, raw[ps].x, raw[ps].y);
      mu = __vimax3_u16x2(mu, raw[ps].z, raw[ps].w);
    }
    const uint32_t mm = __vmaxu2(ms, mu & 0x7FFF7FFFu);
    m = __uint_as_float(max(mm >> 16, mm & 0xFFFFu) << 16);
  } else {
#pragma unroll
    for (int ps = 0; ps < NP; ++ps) {
      float v[V];
      unpack<T>(raw[ps], v);
#pragma unroll
      for (int i = 0; i < V; ++i) m = fmaxf(m, fabsf(v[i]));
    }
  }
  const float amax = block_max_1b(m, red);  // slot 0 (red holds 2 x 8 floats)
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
    publish_flag(p, blk, flagged);
    if (p.res_scales && !flagged) p.res_scales[blk] = 0.0f;
  }
  // ---- RTN codes (kernels.cpp:24-40) ----
  // (the codes are not kept in registers: the fallback residual below -- 5-20 %
  // of blocks -- recomputes them, which keeps this variant inside 80 registers)
  // (rounding mode and row range decided once per block; the destination
  // walks by one pointer increment per pass)
  float rm = 0.0f;       // flagged blocks: the residual's absmax, fused into the code pass
  bool have_rm = false;
  if (p.codes && col_ok) {
    int8_t* dst = p.codes + r0 * p.ldq + cc;
    const int64_t step = (int64_t)RPP * p.ldq;
    if (flagged && !(p.diag & 1)) {  // diag: the separate residual-absmax pass
#pragma unroll
      for (int ps = 0; ps < NP; ++ps, dst += step) {
        if (ps >= nrow) break;  // rows past the end hold zeros: residual 0
        const CodeMax cm = rtn_resmax_raw<T>(raw[ps], a, inv_a, mode);
        rm = fmaxf(rm, cm.rm);
        if constexpr (V == 8) __stcs(reinterpret_cast<uint2*>(dst), cm.code);
        else __stcs(reinterpret_cast<unsigned int*>(dst), cm.code.x);
      }
      have_rm = true;
    } else if (mode == 2 && nrow == NP) {
#pragma unroll
      for (int ps = 0; ps < NP; ++ps, dst += step) {
        constexpr int VV = 16 / sizeof(T);
        float v[VV];
        unpack<T>(raw[ps], v);
        uint32_t w[VV];
        uint2 code;
        if (rtn_fast_vec_x<VV>(v, a, inv_a, w)) {
          code = rtn_fix_raw<T>(raw[ps], a, inv_a);
        } else {
          code.x = pack4_lo8(w);
          code.y = VV == 8 ? pack4_lo8(w + 4) : 0u;
        }
        if constexpr (V == 8) __stcs(reinterpret_cast<uint2*>(dst), code);
        else __stcs(reinterpret_cast<unsigned int*>(dst), code.x);
      }
    } else {
#pragma unroll
      for (int ps = 0; ps < NP; ++ps, dst += step) {
        if (ps >= nrow) break;
        const uint2 code = rtn_raw<T>(raw[ps], a, inv_a, mode);
        if constexpr (V == 8) __stcs(reinterpret_cast<uint2*>(dst), code);
        else __stcs(reinterpret_cast<unsigned int*>(dst), code.x);
      }
    }
  }
  // ---- stochastic context planes (quant.cpp:55-84): RNG index (row_offset + r) * cols + c ----
  if constexpr (kSR >= 1) {
    if (col_ok) {
      const uint64_t lin1 = (uint64_t)((p.row_offset + r0) * p.cols + cc + 1);
      const uint64_t row_step = (uint64_t)RPP * (uint64_t)p.cols * kGolden;
      uint64_t z1 = p.sr_seed + lin1 * kGolden;
      uint64_t z2 = kSR >= 2 ? p.sr_seed2 + lin1 * kGolden : 0;
#pragma unroll 1
      for (int ps = 0; ps < nrow; ++ps) {
        float v[V];
        unpack<T>(raw[ps], v);
        uint32_t w[V];
        const int64_t off = (r0 + (int64_t)ps * RPP) * p.ldq + cc;
        sr_vec<V>(v, a, inv_a, mode, z1, w);
        if constexpr (V == 8) __stcs(reinterpret_cast<uint2*>(p.sr_codes + off), make_uint2(pack4_lo8(w), pack4_lo8(w + 4)));
        else __stcs(reinterpret_cast<unsigned int*>(p.sr_codes + off), pack4_lo8(w));
        if constexpr (kSR >= 2) {
          sr_vec<V>(v, a, inv_a, mode, z2, w);
          if constexpr (V == 8) __stcs(reinterpret_cast<uint2*>(p.sr_codes2 + off), make_uint2(pack4_lo8(w), pack4_lo8(w + 4)));
          else __stcs(reinterpret_cast<unsigned int*>(p.sr_codes2 + off), pack4_lo8(w));
        }
        z1 += row_step;
        z2 += row_step;
      }
    }
  }
  if (!flagged) return;  // block-uniform
  // ---- fallback residual (quant.cpp:146-172): res = fl(x - fl(c * a)) ----
  // the primary codes are recomputed from the raw values (not held: 80-register
  // budget) as magic words, whose n = m - M is the code as a float (no I2F)
  if (!have_rm) {
#pragma unroll
    for (int ps = 0; ps < NP; ++ps) rm = fmaxf(rm, residual_absmax_raw<T>(raw[ps], a, inv_a, mode));
  }
  const float ra = block_scale(block_max_1b(rm, red + kQuantThreads / 32));  // slot 1
  const float inv_ra = ra > 0.0f ? __frcp_rn(ra) : 0.0f;
  const int rmode = round_mode(ra);
  if (threadIdx.x == 0 && p.res_scales) p.res_scales[blk] = ra;
  if (!p.res_codes || !col_ok) return;
  int8_t* rp = p.res_codes + r0 * p.ldq + cc;
#pragma unroll
  for (int ps = 0; ps < NP; ++ps) {
    if (ps >= nrow) break;
    const uint2 code = residual_codes_raw<T>(raw[ps], a, inv_a, mode, ra, inv_ra, rmode);
    int8_t* dst = rp + (int64_t)ps * RPP * p.ldq;
    if constexpr (V == 8) *reinterpret_cast<uint2*>(dst) = code;
    else *reinterpret_cast<uint32_t*>(dst) = code.x;
  }
}

template <typename T>
__device__ __forceinline__ void load_block_reg(const QuantParams& p, int64_t bi, int64_t bj,
                                               uint4 (&raw)[Tiling<T>::NP]) {
  using Tl = Tiling<T>;
  constexpr int V = Tl::V, VPR = Tl::VPR, RPP = Tl::RPP, NP = Tl::NP;
  const int lc = (threadIdx.x % VPR) * V, lr = threadIdx.x / VPR;
  const int64_t r0 = bi * kBlock + lr, cc = bj * kBlock + lc;
  const bool col_ok = cc < p.cols;
  const int64_t left = p.rows - r0;
  const int nrow = left <= 0 ? 0 : (left >= (int64_t)NP * RPP ? NP : (int)((left + RPP - 1) / RPP));
  const T* xp = reinterpret_cast<const T*>(p.x) + r0 * p.ldx + cc;
#pragma unroll
  for (int ps = 0; ps < NP; ++ps)
    raw[ps] = (col_ok && ps < nrow) ? __ldcs(reinterpret_cast<const uint4*>(xp + (int64_t)ps * RPP * p.ldx))
                                    : make_uint4(0, 0, 0, 0);
}

// One 128 x 128 block per CTA (fp32 inputs: 64 registers of raw values per
// thread leave no room for a register double buffer).
template <typename T, int kSR>
__global__ void __launch_bounds__(kQuantThreads, 2)
fbq_quantize_reg_kernel(QuantParams p) {
  __shared__ float red[2 * (kQuantThreads / 32)];  // quantize_block_reg: two reduction slots
  uint4 raw[Tiling<T>::NP];
  load_block_reg<T>(p, blockIdx.y, blockIdx.x, raw);
  quantize_block_reg<T, kSR>(p, blockIdx.y, blockIdx.x, (int64_t)blockIdx.y * gridDim.x + blockIdx.x, raw, red);
}

// QuantLinearLayer::apply_sgd (trainsim.cpp:137-143), w -= float(lr * double(g)),
// fused with the RTN quantization of the updated weight that the next forward
// runs (quantize_rtn(W), trainsim.cpp:96): one 128 x 128 fp32 block per CTA;
// W and dW are read once, W' is written back and its codes and block scale
// come out of the same registers.  Bit-identical to fbq_sgd_kernel followed by
// the RTN quantizer (same per-element expression, same quantize_block_reg).
__global__ void __launch_bounds__(kQuantThreads, 2)
fbq_sgd_quantize_kernel(QuantParams p, float* w, const float* g, double lr) {
  __shared__ float red[2 * (kQuantThreads / 32)];
  using Tl = Tiling<float>;
  constexpr int V = Tl::V, VPR = Tl::VPR, RPP = Tl::RPP, NP = Tl::NP;
  const int64_t bi = blockIdx.y, bj = blockIdx.x;
  uint4 raw[NP];
  load_block_reg<float>(p, bi, bj, raw);
  const int lc = (threadIdx.x % VPR) * V, lrow = threadIdx.x / VPR;
  const int64_t r0 = bi * kBlock + lrow, cc = bj * kBlock + lc;
  const int64_t left = p.rows - r0;
  const int nrow = left <= 0 ? 0 : (left >= (int64_t)NP * RPP ? NP : (int)((left + RPP - 1) / RPP));
  if (cc < p.cols) {
    // dW in two halves of NP / 2 vectors, each half's loads issued together (64
    // raw + 32 registers: one latency round per half instead of one per vector)
    constexpr int H = NP / 2;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      float4 gv[H];
#pragma unroll
      for (int k = 0; k < H; ++k) {
        const int ps = h * H + k;
        gv[k] = ps < nrow ? __ldcs(reinterpret_cast<const float4*>(g + (r0 + (int64_t)ps * RPP) * p.ldx + cc))
                          : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int k = 0; k < H; ++k) {
        const int ps = h * H + k;
        if (ps >= nrow) break;
        const float4 wv = make_float4(__fsub_rn(__uint_as_float(raw[ps].x), (float)(lr * (double)gv[k].x)),
                                      __fsub_rn(__uint_as_float(raw[ps].y), (float)(lr * (double)gv[k].y)),
                                      __fsub_rn(__uint_as_float(raw[ps].z), (float)(lr * (double)gv[k].z)),
                                      __fsub_rn(__uint_as_float(raw[ps].w), (float)(lr * (double)gv[k].w)));
        raw[ps] = make_uint4(__float_as_uint(wv.x), __float_as_uint(wv.y), __float_as_uint(wv.z),
                             __float_as_uint(wv.w));
        __stcs(reinterpret_cast<float4*>(w + (r0 + (int64_t)ps * RPP) * p.ldx + cc), wv);
      }
    }
  }
  quantize_block_reg<float, 0>(p, bi, bj, bi * (int64_t)gridDim.x + bj, raw, red);
}

// Persistent + TMA ring + register compute (bf16): tiles land in a kQStages
// shared-memory ring by TMA while the CTA quantizes the current tile from
// registers; a slot is handed back to TMA as soon as its values are in registers.
// Block schedule: the first kQStages blocks of a CTA are static (blockIdx.x +
// s * gridDim.x); with p.blk_ctr every further one is claimed from the launch's
// counter by thread 0 one refill AHEAD (the atomic's latency hides behind a
// block of rounding), so CTAs that drew flagged (about 3x costlier) blocks take
// fewer -- the fallback blocks of outlier channels otherwise pile up on the
// CTAs whose static stride hits their block-column.  A slot's block id travels
// with its TMA (slot_blk, published before the arrive); -1 ends the CTA.  The
// counter slot self-resets: every CTA's final claim is past the end, and the
// last of those zeroes it (same protocol as the GEMM's tile counter).
template <typename T, int kQStages, int kMinBlocks, int kSR>
__global__ void __launch_bounds__(kQuantThreads, kMinBlocks)
fbq_quantize_tma_reg_kernel(const __grid_constant__ CUtensorMap map_x, QuantParams p, int nblk,
                            int gcols) {
  extern __shared__ __align__(128) uint8_t dsm[];
  T* tiles = reinterpret_cast<T*>(dsm);
  __shared__ __align__(8) uint64_t full[kQStages];
  __shared__ int slot_blk[kQStages];
  __shared__ float red[2 * (kQuantThreads / 32)];  // quantize_block_reg: two reduction slots
  using Tl = Tiling<T>;
  constexpr int V = Tl::V, VPR = Tl::VPR, RPP = Tl::RPP, NP = Tl::NP;
  constexpr uint32_t kTileBytes = sizeof(T) * kTileElems;
  const int static_end = (int64_t)kQStages * gridDim.x < nblk ? kQStages * (int)gridDim.x : nblk;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kQStages; ++s) sm100::mbar_init(full + s, 1);
    sm100::fence_barrier_init();
    sm100::tma_prefetch(&map_x);
  }
  __syncthreads();
  const uint64_t pol = sm100::l2_policy_evict_first();  // X is streamed once
  // thread 0: the static successor of each slot, or the next dynamic claim
  int claim = 0;
  auto next_block = [&](int cur) -> int {
    if (!p.blk_ctr) return cur + kQStages * (int)gridDim.x;
    const int b = claim;
    if (b < nblk) {
      claim = static_end + atomicAdd(p.blk_ctr, 1);
      if (claim >= nblk && atomicAdd(p.blk_ctr + 1, 1) == (int)gridDim.x - 1) {
        atomicExch(p.blk_ctr, 0);  // every CTA made its final claim: reset the slot
        atomicExch(p.blk_ctr + 1, 0);
      }
    }
    return b;
  };
  if (threadIdx.x == 0) {
    if (p.blk_ctr) {
      claim = static_end + atomicAdd(p.blk_ctr, 1);
      if (claim >= nblk && atomicAdd(p.blk_ctr + 1, 1) == (int)gridDim.x - 1) {
        atomicExch(p.blk_ctr, 0);
        atomicExch(p.blk_ctr + 1, 0);
      }
    }
    for (int s = 0; s < kQStages; ++s) {
      const int b = (int)blockIdx.x + s * (int)gridDim.x;
      slot_blk[s] = b < nblk ? b : -1;
      if (b >= nblk) {
        sm100::mbar_arrive(full + s);
        continue;
      }
      sm100::mbar_arrive_expect_tx(full + s, kTileBytes);
      sm100::tma_load_2d(tiles + s * kTileElems, &map_x, full + s, (b % gcols) * kBlock, (b / gcols) * kBlock, pol);
    }
  }
  const int lc = (threadIdx.x % VPR) * V, lr = threadIdx.x / VPR;
  int s = 0;
  uint32_t phase = 0;
  for (;;) {
    sm100::mbar_wait(full + s, phase);
    const int b = slot_blk[s];
    if (b < 0) break;
    uint4 raw[NP];
    const T* tile = tiles + s * kTileElems + lr * kBlock + lc;
#pragma unroll
    for (int ps = 0; ps < NP; ++ps) raw[ps] = *reinterpret_cast<const uint4*>(tile + ps * RPP * kBlock);
    __syncthreads();  // every thread holds its values (and b): slot s goes back to TMA
    if (threadIdx.x == 0) {
      const int nb = next_block(b);
      slot_blk[s] = nb < nblk ? nb : -1;
      if (nb < nblk) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        sm100::mbar_arrive_expect_tx(full + s, kTileBytes);
        sm100::tma_load_2d(tiles + s * kTileElems, &map_x, full + s, (nb % gcols) * kBlock, (nb / gcols) * kBlock, pol);
      } else {
        sm100::mbar_arrive(full + s);  // no tile: wake the CTA to exit
      }
    }
    if (++s == kQStages) { s = 0; phase ^= 1; }
    const int bi = b / gcols;
    quantize_block_reg<T, kSR>(p, bi, b - bi * gcols, b, raw, red);
  }
}

// Persistent, TMA-pipelined K1 (the HBM-bound path for TMA-compatible inputs).
// One-block-per-CTA staging leaves each CTA idle on HBM while it computes and
// idle on the ALUs while it loads (measured 11-37 % of HBM).  Here each CTA
// walks blocks b = blockIdx.x, blockIdx.x + gridDim.x, ... with a kQStages
// ring of 128 x 128 tiles filled by TMA (zero fill outside the tensor = the
// reference's truncated edge blocks, matching stage_tile): while the CTA runs
// quantize_block on tile i, tiles i+1 .. i+kQStages-1 are in flight.
template <typename T, int kSR, int kQStages>
__global__ void __launch_bounds__(kQuantThreads)
fbq_quantize_tma_kernel(const __grid_constant__ CUtensorMap map_x, QuantParams p, int64_t nblk,
                        int gcols) {
  extern __shared__ __align__(128) uint8_t dsm[];
  T* tiles = reinterpret_cast<T*>(dsm);
  __shared__ __align__(8) uint64_t full[kQStages];
  __shared__ float red[2 * (kQuantThreads / 32)];
  constexpr int V = Tiling<T>::V;
  constexpr uint32_t kTileBytes = sizeof(T) * kTileElems;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kQStages; ++s) sm100::mbar_init(full + s, 1);
    sm100::fence_barrier_init();
    sm100::tma_prefetch(&map_x);
  }
  __syncthreads();
  const uint64_t pol = sm100::l2_policy_evict_first();  // X is streamed once
  if (threadIdx.x == 0) {
    for (int s = 0; s < kQStages; ++s) {
      const int64_t b = blockIdx.x + (int64_t)s * gridDim.x;
      if (b >= nblk) break;
      sm100::mbar_arrive_expect_tx(full + s, kTileBytes);
      sm100::tma_load_2d(tiles + s * kTileElems, &map_x, full + s, (int)(b % gcols) * kBlock,
                         (int)(b / gcols) * kBlock, pol);
    }
  }
  int s = 0;
  uint32_t phase = 0;
  for (int64_t b = blockIdx.x; b < nblk; b += gridDim.x) {
    sm100::mbar_wait(full + s, phase);
    const T* tile = tiles + s * kTileElems;
    const int64_t bi = b / gcols, bj = b % gcols;
    quantize_block<V, kSR>(p, b, bi * kBlock, bj * kBlock, red,
                           [&](int rb, int cb, float (&v)[V]) { load_vec<T, V>(tile + rb * kBlock + cb, v); });
    __syncthreads();  // every thread is done reading slot s
    if (threadIdx.x == 0) {
      const int64_t nb = b + (int64_t)kQStages * gridDim.x;
      if (nb < nblk) {
        // order this CTA's generic-proxy reads of the slot before the TMA (async-proxy) write
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        sm100::mbar_arrive_expect_tx(full + s, kTileBytes);
        sm100::tma_load_2d(tiles + s * kTileElems, &map_x, full + s, (int)(nb % gcols) * kBlock,
                           (int)(nb / gcols) * kBlock, pol);
      }
    }
    if (++s == kQStages) { s = 0; phase ^= 1; }
  }
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
// Fast fp32 variants for the bf16 training path (a few ulp from the
// reference): sigmoid = 1 / (1 + 2^(-x log2 e)) with the MUFU ex2 / rcp
// approximations (flush-to-zero ex2: for x > 87 the sigmoid is 1 either way).
__device__ __forceinline__ float sigmoid_fast(float x) {
  float e, r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(x * -1.4426950408889634f));
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(1.0f + e));
  return r;
}
__device__ __forceinline__ float silu_fast(float x) { return x * sigmoid_fast(x); }
__device__ __forceinline__ float silu_grad_fast(float x) {
  const float s = sigmoid_fast(x);
  return s * (1.0f + x * (1.0f - s));
}

// 1 x 128 row-group RTN shared by the VPR threads of a row (quantize_rtn with
// GroupGeometry(1, 128), quant.cpp:36-53).  Words' low halfword = the code.
template <int V, int VPR>
__device__ __forceinline__ float group_rtn(const float (&x)[V], uint32_t (&w)[V], float level) {
  float m = 0.0f;
#pragma unroll
  for (int i = 0; i < V; ++i) m = fmaxf(m, fabsf(x[i]));
  m = row_max<VPR>(m);
  const float s = m > 0.0f ? __fdiv_rn(m, level) : 0.0f;
  const float inv = s > 0.0f ? __frcp_rn(s) : 0.0f;
  if (s >= kTinyScale) {
    // (a per-element second-level test |d| + |q| 2^-22 >= 1/2 in front of the
    // fix was measured 8 % slower on the GLU forward: the bf16 vectors that
    // fire are mostly genuine near-ties; scripts/ab_glu_refine.sh)
    if constexpr (V % 2 == 0) {
      if (rtn_fast_vec_x<V>(x, s, inv, w)) rtn_fix_vec<V>(x, s, w);
    } else {
      if (rtn_fast_vec<V>(x, inv, rtn_window(level), w)) rtn_exact_vec<V>(x, s, inv, level, w);
    }
  } else {
#pragma unroll
    for (int i = 0; i < V; ++i) w[i] = s > 0.0f ? (uint32_t)rtn_code_slow(x[i], s, level) : 0u;
  }
  return s;
}

// Shared-memory row of the forward tile: [a (128 T) | b (128 T)].  The context
// pass turns row r into h = fl(silu(a) * b) as 128 fp32 IN PLACE (512 bytes fit
// in the row; only the VPR threads of that row -- one warp or half-warp --
// touch it, so a __syncwarp orders their reads before their writes).  h is
// thus evaluated once and never reaches HBM.
template <typename T, bool kStaged, int kMinBlocks = 1, bool kPacked = false>
__global__ void __launch_bounds__(kQuantThreads, kMinBlocks)
fbq_glu_forward_kernel(GluParams g, QuantParams p) {
  extern __shared__ __align__(16) uint8_t dsm[];
  constexpr int kRow = 2 * kBlock;                      // T per smem row
  constexpr int kRowF = kRow * (int)sizeof(T) / 4;      // fp32 per smem row
  T* tab = reinterpret_cast<T*>(dsm);
  float* th = reinterpret_cast<float*>(dsm);
  __shared__ float red[2 * (kQuantThreads / 32)];
  using Tl = Tiling<T>;
  constexpr int V = Tl::V, VPR = Tl::VPR, RPP = Tl::RPP, NP = Tl::NP;
  const int64_t bj = blockIdx.x, bi = blockIdx.y;
  const int64_t r0 = bi * kBlock, c0 = bj * kBlock;
  const T* ab = reinterpret_cast<const T*>(g.ab);
  if constexpr (kStaged) {
    stage_tile<T, true>(tab, ab, g.ld_ab, g.rows, g.cols, r0, c0, kRow);
    stage_tile<T, true>(tab + kBlock, ab + g.cols, g.ld_ab, g.rows, g.cols, r0, c0, kRow);
    __syncthreads();
  }
  const int lc = (threadIdx.x % VPR) * V, lr = threadIdx.x / VPR;
  const int64_t gcols = (g.cols + kBlock - 1) / kBlock;
  const int64_t cc = c0 + lc;
  // a and b of (row rb, this thread's V columns): staged tile or global memory
  // (zero outside the tensor: silu(0) * 0 = 0, like the staged zero fill)
  auto load_ab = [&](int rb, int cb, float (&va)[V], float (&vb)[V]) {
    if constexpr (kStaged) {
      load_vec<T, V>(tab + rb * kRow + cb, va);
      load_vec<T, V>(tab + rb * kRow + kBlock + cb, vb);
    } else {
      const int64_t r = r0 + rb, c = c0 + cb;
      if (r < g.rows && c < g.cols) {
        load_vec<T, V>(ab + r * g.ld_ab + c, va);
        load_vec<T, V>(ab + r * g.ld_ab + g.cols + c, vb);
      } else {
#pragma unroll
        for (int i = 0; i < V; ++i) va[i] = vb[i] = 0.0f;
      }
    }
  };
  // h = fl(silu(a) * b) (trainsim.cpp:230), deterministic: the direct variant
  // re-evaluates it in every pass instead of keeping a 64 KiB fp32 tile
  auto hval = [&](const float (&va)[V], const float (&vb)[V], float (&vh)[V]) {
    if (g.exact_math) {
#pragma unroll
      for (int i = 0; i < V; ++i) vh[i] = __fmul_rn(silu_ref(va[i]), vb[i]);
    } else {
      // silu_fast on element pairs: the same roundings, FP32 ops packed
      const float2 one2 = make_float2(1.0f, 1.0f);
      const float2 nl2e = make_float2(-1.4426950408889634f, -1.4426950408889634f);
#pragma unroll
      for (int i = 0; i < V; i += 2) {
        const float2 x2 = make_float2(va[i], va[i + 1]);
        const float2 t = __fmul2_rn(x2, nl2e);
        float e0, e1, r0, r1;
        asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e0) : "f"(t.x));
        asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e1) : "f"(t.y));
        const float2 d = __fadd2_rn(make_float2(e0, e1), one2);
        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r0) : "f"(d.x));
        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r1) : "f"(d.y));
        const float2 h2 = __fmul2_rn(__fmul2_rn(x2, make_float2(r0, r1)), make_float2(vb[i], vb[i + 1]));
        vh[i] = h2.x;
        vh[i + 1] = h2.y;
      }
    }
  };
  // 10-bit contexts of a and b (trainsim.cpp:240-243), h and its absmax
  float m = 0.0f;
#pragma unroll 1
  for (int ps = 0; ps < NP; ++ps) {
    const int rb = lr + ps * RPP;
    const int64_t r = r0 + rb;
    const bool ok = r < g.rows && cc < g.cols;  // cols % 8 == 0: uniform per row group
    float va[V], vb[V];
    load_ab(rb, lc, va, vb);
    uint32_t code[V];
    float s = group_rtn<V, VPR>(va, code, g.ctx_level);
    if (ok && g.ctx_a) {
      if constexpr (kPacked)
        store_ctx10<V>(g.ctx_a + r * g.ld_ctx + cc, g.ctx_a + g.rows * g.ld_ctx + r * (g.ld_ctx >> 2) + (cc >> 2), code);
      else
        store_codes16<V>(reinterpret_cast<int16_t*>(g.ctx_a) + r * g.ld_ctx + cc, code);
    }
    if (ok && g.ctx_a_scales && lc == 0) g.ctx_a_scales[r * gcols + bj] = s;
    s = group_rtn<V, VPR>(vb, code, g.ctx_level);
    if (ok && g.ctx_b) {
      if constexpr (kPacked)
        store_ctx10<V>(g.ctx_b + r * g.ld_ctx + cc, g.ctx_b + g.rows * g.ld_ctx + r * (g.ld_ctx >> 2) + (cc >> 2), code);
      else
        store_codes16<V>(reinterpret_cast<int16_t*>(g.ctx_b) + r * g.ld_ctx + cc, code);
    }
    if (ok && g.ctx_b_scales && lc == 0) g.ctx_b_scales[r * gcols + bj] = s;
    float vh[V];
    hval(va, vb, vh);
#pragma unroll
    for (int i = 0; i < V; ++i) m = fmaxf(m, fabsf(vh[i]));
    if (ok && g.h_out) {
#pragma unroll
      for (int i = 0; i < V; ++i) g.h_out[r * g.ld_h + cc + i] = vh[i];
    }
    if constexpr (kStaged) {
      // h as 128 fp32 IN PLACE of the row's [a | b] (512 bytes; only the VPR
      // threads of that row touch it, so a __syncwarp orders reads before writes)
      __syncwarp();
      store_f32<V>(th + rb * kRowF + lc, vh);
    }
  }
  // h quantized like a linear input (K1, fused)
  if constexpr (kStaged) {
    quantize_block<V, 1>(
        p, bi * gridDim.x + bj, r0, c0, red,
        [&](int rb, int cb, float (&v)[V]) { load_vec<float, V>(th + rb * kRowF + cb, v); }, true, m);
  } else {
    quantize_block<V, 1>(
        p, bi * gridDim.x + bj, r0, c0, red,
        [&](int rb, int cb, float (&v)[V]) {
          float va[V], vb[V];
          load_ab(rb, cb, va, vb);
          hval(va, vb, v);
        },
        true, m);
  }
}

// SiluLayer (trainsim.hpp:118-131, trainsim.cpp:265-290): y = silu(x), the
// input kept as its 10-bit 1 x 128 RTN context (int16 codes, like RmsNorm's);
// backward gx = fl(gy * silu'(dequantize(ctx))).  exact: the reference's double
// silu / silu' (silu_ref / silu_grad_ref); else the fp32 MUFU forms of the GLU
// fast path.  One 128 x 128 tile per CTA, K1's 1 x 128 row groups.
template <typename T, bool kExact>
__global__ void __launch_bounds__(kQuantThreads)
fbq_silu_fwd_kernel(const T* __restrict__ x, int64_t rows, int64_t cols, int64_t ldx, T* __restrict__ y,
                    int64_t ldy, int16_t* __restrict__ ctx, int64_t ld_ctx, float* __restrict__ ctx_scales,
                    float level) {
  using Tl = Tiling<T>;
  constexpr int V = Tl::V, VPR = Tl::VPR, RPP = Tl::RPP, NP = Tl::NP;
  const int64_t bj = blockIdx.x, bi = blockIdx.y;
  const int64_t gcols = (cols + kBlock - 1) / kBlock;
  const int lc = (threadIdx.x % VPR) * V, lr = threadIdx.x / VPR;
  const int64_t cc = bj * kBlock + lc;
  const bool col_ok = cc < cols;  // cols % V == 0
#pragma unroll 1
  for (int ps = 0; ps < NP; ++ps) {
    const int64_t r = bi * kBlock + lr + ps * RPP;
    if (r >= rows) break;  // row-uniform across the VPR threads of the group
    float v[V];
    if (col_ok) {
      load_vec<T, V>(x + r * ldx + cc, v);
    } else {
#pragma unroll
      for (int i = 0; i < V; ++i) v[i] = 0.0f;
    }
    uint32_t code[V];
    const float s = group_rtn<V, VPR>(v, code, level);
    if (!col_ok) continue;
    store_codes16<V>(ctx + r * ld_ctx + cc, code);
    if (lc == 0) ctx_scales[r * gcols + bj] = s;
    T out[V];
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const float o = kExact ? silu_ref(v[i]) : silu_fast(v[i]);
      if constexpr (sizeof(T) == 2) out[i] = __float2bfloat16_rn(o);
      else out[i] = o;
    }
    *reinterpret_cast<uint4*>(y + r * ldy + cc) = *reinterpret_cast<const uint4*>(out);
  }
}

template <typename T, bool kExact>
__global__ void __launch_bounds__(256)
fbq_silu_bwd_kernel(const int16_t* __restrict__ ctx, int64_t ld_ctx, const float* __restrict__ ctx_scales,
                    const T* __restrict__ gy, int64_t ldgy, int64_t rows, int64_t cols, T* __restrict__ gx,
                    int64_t ldgx) {
  const int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 2;
  if (c >= cols) return;
  const bool two = c + 1 < cols;
  const int64_t gcols = (cols + kBlock - 1) / kBlock, cb = c / kBlock;
  for (int64_t r = blockIdx.y; r < rows; r += gridDim.y) {
    const float sc = ctx_scales[r * gcols + cb];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      if (e == 1 && !two) break;
      const int64_t cc = c + e;
      const float xv = __fmul_rn((float)ctx[r * ld_ctx + cc], sc);  // dequantize: fl(code * scale)
      const float d = kExact ? silu_grad_ref(xv) : silu_grad_fast(xv);
      const float o = __fmul_rn(to_f32(gy[r * ldgy + cc]), d);
      if constexpr (sizeof(T) == 2) gx[r * ldgx + cc] = __float2bfloat16_rn(o);
      else gx[r * ldgx + cc] = o;
    }
  }
}

// GluCombine backward (trainsim.cpp:248-263) fused with the two dY
// quantizers: ga = fl(fl(gy * b) * silu'(a)), gb = fl(gy * silu(a)) from the
// staged dH and 10-bit contexts; one pass for both block absmaxes, one pass
// stochastic-rounding both into [q(ga) | q(gb)] with their own RNG streams
// (quant.cpp:55-84).
// kStaged: dH and both contexts staged in shared memory (96 KiB for bf16:
// two CTAs per SM); otherwise every pass reads them straight from global
// memory (the second pass hits L2) with three CTAs per SM -- more warps for
// an issue-bound kernel.
template <typename T, bool kStaged, int kMinBlocks = 1, bool kPacked = false>
__global__ void __launch_bounds__(kQuantThreads, kMinBlocks)
fbq_glu_backward_kernel(GluBwdParams g) {
  extern __shared__ __align__(16) uint8_t dsm[];
  T* tg = reinterpret_cast<T*>(dsm);
  __shared__ float sa_row[kBlock], sb_row[kBlock];
  __shared__ float red[kQuantThreads / 32], red2[kQuantThreads / 32];
  constexpr int V = Tiling<T>::V;
  constexpr int VPR = kBlock / V, RPP = kQuantThreads / VPR, NP = kBlock / RPP;
  const int64_t bj = blockIdx.x, bi = blockIdx.y;
  const int64_t r0 = bi * kBlock, c0 = bj * kBlock;
  const int64_t gcols = (g.cols + kBlock - 1) / kBlock;
  if constexpr (kStaged) {
    stage_tile<T, true>(tg, reinterpret_cast<const T*>(g.gh), g.ld_gh, g.rows, g.cols, r0, c0);
  }
  // the row scales with the packed contexts' 2^22 folded in; a scale small
  // enough for that product to leave the normal range (never for real data)
  // takes the exact path: the code is then read unscaled
  if (threadIdx.x < kBlock) {
    const int64_t r = r0 + threadIdx.x;
    sa_row[threadIdx.x] = r < g.rows ? g.ctx_a_scales[r * gcols + bj] : 0.0f;
    sb_row[threadIdx.x] = r < g.rows ? g.ctx_b_scales[r * gcols + bj] : 0.0f;
  }
  __syncthreads();
  // dequantized contexts: fl(code * scale) (quant.cpp:86-104); a zero scale
  // has all-zero codes, so no special case is needed.  fl((code 2^22) (s 2^-22))
  // == fl(code s) while s 2^-22 stays a normal float (s >= 2^-104).
  auto deq = [&](const uint8_t* gt, float s, int rb, int cb, float (&v)[V]) {
    const int64_t r = r0 + rb, cc = c0 + cb;
    const bool ok = r < g.rows && cc < g.cols;
    if constexpr (!kPacked) {  // int16 codes (the reference's QuantizedTensor storage)
      int16_t c[V];
      const int16_t* src = reinterpret_cast<const int16_t*>(gt) + r * g.ld_ctx + cc;
      if constexpr (V == 8) *reinterpret_cast<uint4*>(c) = ok ? *reinterpret_cast<const uint4*>(src) : make_uint4(0, 0, 0, 0);
      else *reinterpret_cast<uint2*>(c) = ok ? *reinterpret_cast<const uint2*>(src) : make_uint2(0, 0);
#pragma unroll
      for (int i = 0; i < V; ++i) v[i] = __fmul_rn((float)c[i], s);
      return;
    }
    int32_t c[V];
    if (ok) {
      load_ctx10_x4m<V>(gt + r * g.ld_ctx + cc, gt + g.rows * g.ld_ctx + r * (g.ld_ctx >> 2) + (cc >> 2), c);
    } else {
#pragma unroll
      for (int i = 0; i < V; ++i) c[i] = 0;
    }
    if (s >= 0x1p-104f) {
      const float s22 = s * 0x1p-22f;
#pragma unroll
      for (int i = 0; i < V; ++i) v[i] = __fmul_rn((float)c[i], s22);
    } else {
#pragma unroll
      for (int i = 0; i < V; ++i) v[i] = __fmul_rn((float)(c[i] >> 22), s);
    }
  };
  auto eval = [&](int rb, int cb, float (&ga)[V], float (&gb)[V]) {
    float a[V], b[V];
    if constexpr (kStaged) {
      load_vec<T, V>(tg + rb * kBlock + cb, ga);
    } else {
      const int64_t r = r0 + rb, cc = c0 + cb;
      if (r < g.rows && cc < g.cols) {
        load_vec<T, V>(reinterpret_cast<const T*>(g.gh) + r * g.ld_gh + cc, ga);
      } else {
#pragma unroll
        for (int i = 0; i < V; ++i) ga[i] = 0.0f;
      }
    }
    deq(g.ctx_a, sa_row[rb], rb, cb, a);
    deq(g.ctx_b, sb_row[rb], rb, cb, b);
    if (g.exact_math) {
#pragma unroll
      for (int i = 0; i < V; ++i) {
        const float gy = ga[i];
        const float sg = silu_grad_ref(a[i]), sl = silu_ref(a[i]);
        ga[i] = __fmul_rn(__fmul_rn(gy, b[i]), sg);
        gb[i] = __fmul_rn(gy, sl);
      }
    } else {
      // the fast path on element pairs (FMUL2 / FFMA2; ex2 / rcp stay scalar
      // MUFU): sig = 1 / (1 + 2^(-a log2 e)), sg = sig (1 + a (1 - sig)),
      // sl = a sig, ga = fl(fl(gy b) sg), gb = fl(gy sl) -- the same roundings
      // as the scalar sigmoid_fast / silu_grad_fast sequence
      const float2 one2 = make_float2(1.0f, 1.0f), neg1 = make_float2(-1.0f, -1.0f);
      const float2 nl2e = make_float2(-1.4426950408889634f, -1.4426950408889634f);
#pragma unroll
      for (int i = 0; i < V; i += 2) {
        const float2 x2 = make_float2(a[i], a[i + 1]);
        const float2 t = __fmul2_rn(x2, nl2e);
        float e0, e1, r0, r1;
        asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e0) : "f"(t.x));
        asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e1) : "f"(t.y));
        const float2 d = __fadd2_rn(make_float2(e0, e1), one2);
        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r0) : "f"(d.x));
        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r1) : "f"(d.y));
        const float2 sig = make_float2(r0, r1);
        const float2 om = __ffma2_rn(sig, neg1, one2);   // 1 - sig
        const float2 sg = __fmul2_rn(sig, __ffma2_rn(x2, om, one2));
        const float2 sl = __fmul2_rn(x2, sig);
        const float2 gy = make_float2(ga[i], ga[i + 1]);
        const float2 g1 = __fmul2_rn(__fmul2_rn(gy, make_float2(b[i], b[i + 1])), sg);
        const float2 g2 = __fmul2_rn(gy, sl);
        ga[i] = g1.x; ga[i + 1] = g1.y;
        gb[i] = g2.x; gb[i + 1] = g2.y;
      }
    }
  };
  const int lc = (threadIdx.x % VPR) * V, lr = threadIdx.x / VPR;
  const int64_t cc = c0 + lc;
  float ma = 0.0f, mb = 0.0f;
#pragma unroll 1
  for (int ps = 0; ps < NP; ++ps) {
    const int rb = lr + ps * RPP;
    float va[V], vb[V];
    eval(rb, lc, va, vb);
#pragma unroll
    for (int i = 0; i < V; ++i) {
      ma = fmaxf(ma, fabsf(va[i]));
      mb = fmaxf(mb, fabsf(vb[i]));
    }
    const int64_t r = r0 + rb;
    if (g.g_out && r < g.rows && cc < g.cols) {
#pragma unroll
      for (int i = 0; i < V; ++i) {
        g.g_out[r * g.cols + cc + i] = va[i];
        g.g_out[g.rows * g.cols + r * g.cols + cc + i] = vb[i];
      }
    }
  }
  const float a_s = block_scale(block_max_1b(ma, red));  // one block per CTA: no reuse
  const float b_s = block_scale(block_max_1b(mb, red2));
  const float inv_a = a_s > 0.0f ? __frcp_rn(a_s) : 0.0f, inv_b = b_s > 0.0f ? __frcp_rn(b_s) : 0.0f;
  const int mode_a = round_mode(a_s), mode_b = round_mode(b_s);
  if (threadIdx.x == 0) {
    g.gq_scales[bi * (2 * gcols) + bj] = a_s;
    g.gq_scales[bi * (2 * gcols) + gcols + bj] = b_s;
  }
  if (cc >= g.cols) return;
#pragma unroll 1
  for (int ps = 0; ps < NP; ++ps) {
    const int rb = lr + ps * RPP;
    const int64_t r = r0 + rb;
    if (r >= g.rows) break;
    float va[V], vb[V];
    eval(rb, lc, va, vb);
    const uint64_t lin1 = (uint64_t)((g.row_offset + r) * g.cols + cc + 1);
    uint32_t code[V];
    sr_vec<V>(va, a_s, inv_a, mode_a, g.seed_a + lin1 * kGolden, code);
    store_codes<V>(g.gq + r * g.ldq + cc, code, V, true);
    sr_vec<V>(vb, b_s, inv_b, mode_b, g.seed_b + lin1 * kGolden, code);
    store_codes<V>(g.gq + r * g.ldq + g.cols + cc, code, V, true);
  }
}

// ------------------------------------------------------------------ RMSNorm
// RmsNorm (trainsim.cpp:154-211) with its 10-bit 1 x 128 input context.
// The reference accumulates every row's sum of squares (and, backward, the
// gain-weighted dot product) SEQUENTIALLY in double, and grad_gain over the
// rows in order in float; to reproduce those exact roundings each sum is one
// thread's dependent chain.  There are only rows (or cols) such chains, so the
// kernels are built to keep enough bytes in flight per chain: a lane owns a
// row and reads it from a cp.async ring of [32 rows x 128 columns] tiles (row
// statistics), or owns a column of a warp's 32 and reads [kGgRows x 32] tiles
// of the per-element grad_gain terms from a cp.async ring (grad_gain).

// Row statistics: one warp per 32 rows, lane = row, columns in order.  The
// rows are streamed through a kRsStages ring of [32 rows x 128 columns] shared
// memory tiles filled by cp.async in row-contiguous 16-byte pieces (each warp
// instruction moves two 256-byte row segments, so HBM sees long runs; a lane
// loading its own row 16 bytes at a time opened a DRAM page per access and ran
// at 0.3 TB/s); rows are padded by 16 bytes so each lane's LDS.128 of its row
// hits its own banks.
constexpr int kRsCols = 128, kRsStages = 6;
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
  const int sz = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(gmem), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem, bool pred) {
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
  const int sz = pred ? 4 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(sa), "l"(gmem), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Fill stage rows [r0, r0 + 32) x columns [c0, c0 + kRsCols) of a row-major
// T matrix into smem (row stride RS bytes); out-of-range pieces are zeros.
template <typename T, int RS>
__device__ __forceinline__ void rs_fill(uint8_t* dst, const T* src, int64_t ld, int64_t rows, int64_t cols,
                                        int64_t r0, int64_t c0) {
  constexpr int PPR = kRsCols * (int)sizeof(T) / 16;  // 16-byte pieces per row
  constexpr int EPP = 16 / (int)sizeof(T);
  for (int i = threadIdx.x; i < 32 * PPR; i += 32) {
    const int rr = i / PPR, pc = i % PPR;
    const int64_t r = r0 + rr, c = c0 + (int64_t)pc * EPP;
    const bool ok = r < rows && c < cols;  // cols % 8 == 0 keeps pieces whole
    cp_async16(dst + rr * RS + pc * 16, src + (ok ? r * ld + c : 0), ok);
  }
}

template <typename T>
__global__ void __launch_bounds__(32)
fbq_rms_rowstat_fwd_kernel(const T* __restrict__ x, int64_t rows, int64_t cols, int64_t ldx,
                           float* __restrict__ rms) {
  constexpr int RS = kRsCols * (int)sizeof(T) + 16;
  constexpr int E = 16 / (int)sizeof(T);
  extern __shared__ __align__(16) uint8_t rsm[];
  const int64_t r0 = (int64_t)blockIdx.x * 32;
  const int64_t nch = (cols + kRsCols - 1) / kRsCols;
#pragma unroll
  for (int k = 0; k < kRsStages - 1; ++k) {
    if (k < nch) rs_fill<T, RS>(rsm + k * 32 * RS, x, ldx, rows, cols, r0, (int64_t)k * kRsCols);
    cp_async_commit();
  }
  double ss = 0.0;
  for (int64_t ch = 0; ch < nch; ++ch) {
    const int64_t pre = ch + kRsStages - 1;
    if (pre < nch) rs_fill<T, RS>(rsm + (pre % kRsStages) * 32 * RS, x, ldx, rows, cols, r0, pre * kRsCols);
    cp_async_commit();
    cp_async_wait<kRsStages - 1>();
    __syncwarp();
    const uint8_t* row = rsm + (ch % kRsStages) * 32 * RS + threadIdx.x * RS;
#pragma unroll 4
    for (int pc = 0; pc < kRsCols / E; ++pc) {
      float v[E];
      unpack<T>(*reinterpret_cast<const uint4*>(row + pc * 16), v);
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const double d = (double)v[e];  // zero fill past the end adds exactly nothing
        ss = __fma_rn(d, d, ss);         // d*d is exact in double: == ss + d*d (trainsim.cpp:160-163)
      }
    }
    __syncwarp();  // the stage is refilled by a later iteration
  }
  cp_async_wait<0>();
  const int64_t r = r0 + threadIdx.x;
  if (r < rows)  // sqrt(float(ss / cols) + eps) in float (trainsim.cpp:164-165)
    rms[r] = __fsqrt_rn(__fadd_rn(__double2float_rn(__ddiv_rn(ss, (double)cols)), 1e-6f));
}

// y = fl(fl(x / rms) * gain) and the 10-bit 1 x 128 RTN context of x
// (quantize_rtn(x, GroupGeometry(1, 128), 10 bits), trainsim.cpp:166-177).
template <typename T>
__global__ void __launch_bounds__(kQuantThreads)
fbq_rms_apply_fwd_kernel(const T* __restrict__ x, int64_t rows, int64_t cols, int64_t ldx,
                         const float* __restrict__ gain, const float* __restrict__ rms,
                         T* __restrict__ y, int64_t ldy, int16_t* ctx, int64_t ld_ctx,
                         float* ctx_scales, float level) {
  using Tl = Tiling<T>;
  constexpr int V = Tl::V, VPR = Tl::VPR, RPP = Tl::RPP, NP = Tl::NP;
  const int64_t bj = blockIdx.x, bi = blockIdx.y;
  const int64_t gcols = (cols + kBlock - 1) / kBlock;
  const int lc = (threadIdx.x % VPR) * V, lr = threadIdx.x / VPR;
  const int64_t cc = bj * kBlock + lc;
  const bool col_ok = cc < cols;  // cols % V == 0
  float g[V];
#pragma unroll
  for (int i = 0; i < V; ++i) g[i] = col_ok ? gain[cc + i] : 0.0f;
#pragma unroll 1
  for (int ps = 0; ps < NP; ++ps) {
    const int64_t r = bi * kBlock + lr + ps * RPP;
    if (r >= rows) break;  // row-uniform across the VPR threads of the group
    float v[V];
    if (col_ok) {
      load_vec<T, V>(x + r * ldx + cc, v);
    } else {
#pragma unroll
      for (int i = 0; i < V; ++i) v[i] = 0.0f;
    }
    uint32_t code[V];
    const float s = group_rtn<V, VPR>(v, code, level);
    if (!col_ok) continue;
    store_codes16<V>(ctx + r * ld_ctx + cc, code);
    if (lc == 0) ctx_scales[r * gcols + bj] = s;
    const float rr = rms[r];
    T out[V];
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const float o = __fmul_rn(__fdiv_rn(v[i], rr), g[i]);
      if constexpr (sizeof(T) == 2) out[i] = __float2bfloat16_rn(o);
      else out[i] = o;
    }
    *reinterpret_cast<uint4*>(y + r * ldy + cc) = *reinterpret_cast<const uint4*>(out);
  }
}

// RmsNorm fused with the next QuantLinearLayer's input quantizer:
// per 128 x 128 block of x, the 10-bit 1 x 128 context of x (the RmsNorm's own
// saved input, trainsim.cpp:171-176), then y = T(fl(fl(x / rms) * gain))
// (trainsim.cpp:166-168; rounded to the activation dtype exactly like the
// unfused RmsNorm output) repacked into the register-resident K1 -- codes,
// scale, fallback flag / residual and the stochastic context planes of the
// linear input (quant.cpp:36-84, 128-176) -- so y never reaches HBM.  rms[] comes
// from fbq_rms_rowstat_fwd_kernel.  One block per CTA.
template <typename T, int kSR, int kMinBlocks>
__global__ void __launch_bounds__(kQuantThreads, kMinBlocks)
fbq_rms_quant_kernel(QuantParams p, const float* __restrict__ gain, const float* __restrict__ rms,
                     int16_t* __restrict__ ctx, int64_t ld_ctx, float* __restrict__ ctx_scales) {
  extern __shared__ __align__(16) uint8_t dsm[];
  T* tile = reinterpret_cast<T*>(dsm);  // y of the block (zeros outside the tensor), as the K1 tile
  __shared__ float red[2 * (kQuantThreads / 32)];
  using Tl = Tiling<T>;
  constexpr int V = Tl::V, VPR = Tl::VPR, RPP = Tl::RPP, NP = Tl::NP;
  const int64_t bi = blockIdx.y, bj = blockIdx.x;
  const int64_t gcols = (p.cols + kBlock - 1) / kBlock;
  const int lc = (threadIdx.x % VPR) * V, lr = threadIdx.x / VPR;
  const int64_t cc = bj * kBlock + lc;
  const bool col_ok = cc < p.cols;  // cols % V == 0
  float g[V];
#pragma unroll
  for (int i = 0; i < V; ++i) g[i] = col_ok ? gain[cc + i] : 0.0f;
  const T* xp = reinterpret_cast<const T*>(p.x);
#pragma unroll 2
  for (int ps = 0; ps < NP; ++ps) {
    const int rb = lr + ps * RPP;
    const int64_t r = bi * kBlock + rb;
    const bool ok = r < p.rows;  // row-uniform across the VPR threads of the group
    float v[V];
    if (ok && col_ok) {
      load_vec<T, V>(xp + r * p.ldx + cc, v);
    } else {
#pragma unroll
      for (int i = 0; i < V; ++i) v[i] = 0.0f;
    }
    uint32_t code[V];
    const float s = group_rtn<V, VPR>(v, code, 511.0f);
    if (ok && col_ok) {
      store_codes16<V>(ctx + r * ld_ctx + cc, code);
      if (lc == 0) ctx_scales[r * gcols + bj] = s;
    }
    T out[V];
    const float rr = ok ? rms[r] : 1.0f;
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const float o = (ok && col_ok) ? __fmul_rn(__fdiv_rn(v[i], rr), g[i]) : 0.0f;
      if constexpr (sizeof(T) == 2) out[i] = __float2bfloat16_rn(o);
      else out[i] = o;
    }
    *reinterpret_cast<uint4*>(tile + rb * kBlock + lc) = *reinterpret_cast<const uint4*>(out);
  }
  __syncthreads();
  quantize_block<V, kSR>(p, bi * gcols + bj, bi * kBlock, bj * kBlock, red,
                         [&](int rb, int cb, float (&v)[V]) { load_vec<T, V>(tile + rb * kBlock + cb, v); });
}

// backward row statistics (trainsim.cpp:186-199), sequential per row in double:
// x = dequantize(ctx); ss = sum x^2; dot = sum fl(fl(g*dy)*x); rms = sqrt(ss/cols
// + eps); inv = 1 / rms; corr = dot / (((cols*rms)*rms)*rms).  Lane = row; the
// codes, dy, the block's scale per row and the chunk's gains stream through a
// kRsBwdStages cp.async ring like the forward.
constexpr int kRsBwdStages = 4;
template <typename T>
struct RsBwdLayout {
  static constexpr int RSC = kRsCols * 2 + 16;                    // code row stride (bytes)
  static constexpr int RSD = kRsCols * (int)sizeof(T) + 16;       // dy row stride
  static constexpr int kCodes = 0, kDy = 32 * RSC, kScale = kDy + 32 * RSD, kGain = kScale + 32 * 4;
  static constexpr int kStage = kGain + kRsCols * 4;
};
template <typename T>
__global__ void __launch_bounds__(32)
fbq_rms_rowstat_bwd_kernel(const int16_t* __restrict__ ctx, int64_t ld_ctx,
                           const float* __restrict__ ctx_scales, const T* __restrict__ gy,
                           int64_t ldgy, int64_t rows, int64_t cols, const float* __restrict__ gain,
                           double* __restrict__ inv_out, double* __restrict__ corr_out) {
  using L = RsBwdLayout<T>;
  extern __shared__ __align__(16) uint8_t rsm[];
  __shared__ double gd[kRsCols];
  static_assert(kRsCols == 128, "4 gains per lane");
  const int lane = threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.x * 32;
  const int64_t gcols = (cols + kBlock - 1) / kBlock;
  const int64_t nch = (cols + kRsCols - 1) / kRsCols;  // kRsCols == kBlock: one scale per row per chunk
  auto fill = [&](int sidx, int64_t ch) {
    uint8_t* st = rsm + sidx * L::kStage;
    const int64_t c0 = ch * kRsCols;
    rs_fill<int16_t, L::RSC>(st + L::kCodes, ctx, ld_ctx, rows, cols, r0, c0);
    rs_fill<T, L::RSD>(st + L::kDy, gy, ldgy, rows, cols, r0, c0);
    const int64_t r = r0 + lane;
    cp_async4(st + L::kScale + lane * 4, ctx_scales + (r < rows ? r * gcols + ch : 0), r < rows);
    for (int i = lane; i < kRsCols / 4; i += 32) {
      const bool ok = c0 + i * 4 < cols;
      cp_async16(st + L::kGain + i * 16, gain + (ok ? c0 + i * 4 : 0), ok);
    }
  };
#pragma unroll
  for (int k = 0; k < kRsBwdStages - 1; ++k) {
    if (k < nch) fill(k, k);
    cp_async_commit();
  }
  double ss = 0.0, dot = 0.0;
  for (int64_t ch = 0; ch < nch; ++ch) {
    const int64_t pre = ch + kRsBwdStages - 1;
    if (pre < nch) fill((int)(pre % kRsBwdStages), pre);
    cp_async_commit();
    cp_async_wait<kRsBwdStages - 1>();
    __syncwarp();
    const uint8_t* st = rsm + (ch % kRsBwdStages) * L::kStage;
    const uint8_t* crow = st + L::kCodes + lane * L::RSC;
    const uint8_t* drow = st + L::kDy + lane * L::RSD;
    const float sc = *reinterpret_cast<const float*>(st + L::kScale + lane * 4);
    // the chunk's gains widened to double once per chunk (4 per lane) instead of
    // once per element: the F2F.F64.F32 pipe is what paces this kernel
    {
      const float4 g4 = *reinterpret_cast<const float4*>(st + L::kGain + lane * 16);
      gd[lane * 4 + 0] = (double)g4.x;
      gd[lane * 4 + 1] = (double)g4.y;
      gd[lane * 4 + 2] = (double)g4.z;
      gd[lane * 4 + 3] = (double)g4.w;
    }
    __syncwarp();
#pragma unroll 2
    for (int pc = 0; pc < kRsCols / 8; ++pc) {  // 8 columns per step
      const uint4 cw4 = *reinterpret_cast<const uint4*>(crow + pc * 16);
      const uint32_t cw[4] = {cw4.x, cw4.y, cw4.z, cw4.w};
      float dy[8];
      if constexpr (sizeof(T) == 2) {
        unpack<T>(*reinterpret_cast<const uint4*>(drow + pc * 16), dy);
      } else {
        float lo[4], hi[4];
        unpack<float>(*reinterpret_cast<const uint4*>(drow + pc * 32), lo);
        unpack<float>(*reinterpret_cast<const uint4*>(drow + pc * 32 + 16), hi);
#pragma unroll
        for (int e = 0; e < 4; ++e) { dy[e] = lo[e]; dy[4 + e] = hi[e]; }
      }
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int code = (int)(int16_t)(cw[e >> 1] >> (16 * (e & 1)));
        const double v = (double)__fmul_rn((float)code, sc);  // dequantize: fl(code * scale)
        ss = __fma_rn(v, v, ss);                               // zero-filled columns add nothing
        const double h = __dmul_rn(gd[pc * 8 + e], (double)dy[e]);
        dot = __dadd_rn(dot, __dmul_rn(h, v));
      }
    }
    __syncwarp();
  }
  cp_async_wait<0>();
  const int64_t r = r0 + lane;
  if (r < rows) {
    const double rms = __dsqrt_rn(__dadd_rn(__ddiv_rn(ss, (double)cols), (double)1e-6f));
    inv_out[r] = __ddiv_rn(1.0, rms);
    corr_out[r] = __ddiv_rn(dot, __dmul_rn(__dmul_rn(__dmul_rn((double)cols, rms), rms), rms));
  }
}

// gx = float(h * inv - x * corr), h = g * dy (double); and the per-element
// grad_gain term float(float(dy * x) * inv) into `term` (trainsim.cpp:200-205)
template <typename T>
__global__ void __launch_bounds__(256)
fbq_rms_apply_bwd_kernel(const int16_t* __restrict__ ctx, int64_t ld_ctx,
                         const float* __restrict__ ctx_scales, const T* __restrict__ gy,
                         int64_t ldgy, int64_t rows, int64_t cols,
                         const float* __restrict__ gain, const double* __restrict__ inv,
                         const double* __restrict__ corr, T* gx,
                         int64_t ldgx, float* __restrict__ term,
                         const T* res, int64_t ldres) {  // res may alias gx
  // a thread owns columns (c, c + 1) and walks rows blockIdx.y, + gridDim.y, ...:
  // no per-element index division, the two gains widened to double once
  const int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 2;
  if (c >= cols) return;
  const bool two = c + 1 < cols;
  const int64_t gcols = (cols + kBlock - 1) / kBlock, cb = c / kBlock;
  const double g0 = (double)gain[c], g1 = two ? (double)gain[c + 1] : 0.0;
  for (int64_t r = blockIdx.y; r < rows; r += gridDim.y) {
    const float sc = ctx_scales[r * gcols + cb];
    const double iv = inv[r], co = corr[r];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      if (e == 1 && !two) break;
      const int64_t cc = c + e;
      const float x = __fmul_rn((float)ctx[r * ld_ctx + cc], sc);
      const float dy = to_f32(gy[r * ldgy + cc]);
      const double h = __dmul_rn(e ? g1 : g0, (double)dy);
      float o = __double2float_rn(__dsub_rn(__dmul_rn(h, iv), __dmul_rn((double)x, co)));
      // GluBlock's residual: add(norm.backward(grad_xn), grad_out) (trainsim.cpp:303-307)
      if (res) o = __fadd_rn(o, to_f32(res[r * ldres + cc]));
      if constexpr (sizeof(T) == 2) gx[r * ldgx + cc] = __float2bfloat16_rn(o);
      else gx[r * ldgx + cc] = o;
      term[r * cols + cc] = __double2float_rn(__dmul_rn((double)__fmul_rn(dy, x), iv));
    }
  }
}

// grad_gain[c] += term[r][c] for r = 0, 1, ... in order (float adds, the
// reference's accumulation order).  Only `cols` chains exist, so a warp owns 32
// columns and streams [kGgRows x 32] chunks of `term` through a kGgStages
// cp.async ring: each lane's add chain (4 cycles per row) never waits on HBM.
constexpr int kGgRows = 64, kGgStages = 5;  // 40 KB of static shared memory
__global__ void __launch_bounds__(32)
fbq_rms_grad_gain_kernel(const float* __restrict__ term, int64_t rows, int64_t cols,
                         float* __restrict__ grad_gain) {
  __shared__ __align__(16) float st[kGgStages][kGgRows][32];
  const int lane = threadIdx.x;
  const int64_t c0 = (int64_t)blockIdx.x * 32, c = c0 + lane;
  const bool cok = c < cols;
  const int64_t nch = (rows + kGgRows - 1) / kGgRows;
  // kGgRows rows x 128 B = 8 pieces per row (cols % 8 == 0 keeps pieces whole):
  // lane copies piece (lane & 7) of rows (lane >> 3) + 4 k -- its column offset
  // is fixed, so a piece costs one address add (the per-piece index arithmetic
  // was most of this latency-bound kernel's instructions)
  const int pcl = lane & 7, rrl = lane >> 3;
  const bool pc_ok = c0 + pcl * 4 < cols;
  const float* lane_base = term + (int64_t)rrl * cols + c0 + pcl * 4;
  const int64_t step4 = 4 * cols;
  auto fill = [&](int sidx, int64_t ch) {
    const float* src = lane_base + ch * kGgRows * cols;
    const int64_t rlim = rows - ch * kGgRows - rrl;  // rows left for this lane's first piece
#pragma unroll
    for (int k = 0; k < kGgRows / 4; ++k, src += step4) {
      const bool ok = pc_ok && 4 * k < rlim;
      cp_async16(&st[sidx][rrl + 4 * k][pcl * 4], ok ? src : term, ok);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
#pragma unroll
  for (int k = 0; k < kGgStages - 1; ++k) {
    if (k < nch) fill(k, k);
    else asm volatile("cp.async.commit_group;" ::: "memory");
  }
  float acc = cok ? grad_gain[c] : 0.0f;
  for (int64_t ch = 0; ch < nch; ++ch) {
    const int64_t pre = ch + kGgStages - 1;
    if (pre < nch) fill((int)(pre % kGgStages), pre);
    else asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group %0;" ::"n"(kGgStages - 1) : "memory");
    __syncwarp();
    const float(*t)[32] = st[ch % kGgStages];
    const int nr = rows - ch * kGgRows < kGgRows ? (int)(rows - ch * kGgRows) : kGgRows;
    if (nr == kGgRows) {
#pragma unroll 16
      for (int rr = 0; rr < kGgRows; ++rr) acc = __fadd_rn(acc, t[rr][lane]);
    } else {
      for (int rr = 0; rr < nr; ++rr) acc = __fadd_rn(acc, t[rr][lane]);
    }
    __syncwarp();  // this stage is refilled by the next iteration's prefetch
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  if (cok) grad_gain[c] = acc;
}

// per-device one-time opt-in to `bytes` of dynamic shared memory for kernel K
template <auto K>
static cudaError_t smem_once(size_t bytes) {
  static std::once_flag flag[64];
  static cudaError_t err[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  std::call_once(flag[dev], [&] {
    err[dev] = bytes > 48 * 1024 ? cudaFuncSetAttribute(K, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes)
                                 : cudaSuccess;
  });
  return err[dev];
}

cudaError_t launch_rmsnorm_forward(const void* x, bool bf16, int64_t rows, int64_t cols, int64_t ldx,
                                   const float* gain, void* y, int64_t ldy, int16_t* ctx,
                                   int64_t ld_ctx, float* ctx_scales, float* rms, cudaStream_t s) {
  const unsigned rb = (unsigned)((rows + 31) / 32);  // one warp per 32 rows
  const dim3 grid((unsigned)((cols + kBlock - 1) / kBlock), (unsigned)((rows + kBlock - 1) / kBlock));
  const size_t sm16 = (size_t)kRsStages * 32 * (kRsCols * 2 + 16), sm32 = (size_t)kRsStages * 32 * (kRsCols * 4 + 16);
  if (cudaError_t e = smem_once<fbq_rms_rowstat_fwd_kernel<__nv_bfloat16>>(sm16)) return e;
  if (cudaError_t e = smem_once<fbq_rms_rowstat_fwd_kernel<float>>(sm32)) return e;
  if (bf16) {
    fbq_rms_rowstat_fwd_kernel<__nv_bfloat16><<<rb, 32, sm16, s>>>(
        reinterpret_cast<const __nv_bfloat16*>(x), rows, cols, ldx, rms);
    fbq_rms_apply_fwd_kernel<__nv_bfloat16><<<grid, kQuantThreads, 0, s>>>(
        reinterpret_cast<const __nv_bfloat16*>(x), rows, cols, ldx, gain, rms,
        reinterpret_cast<__nv_bfloat16*>(y), ldy, ctx, ld_ctx, ctx_scales, 511.0f);
  } else {
    fbq_rms_rowstat_fwd_kernel<float><<<rb, 32, sm32, s>>>(reinterpret_cast<const float*>(x), rows,
                                                              cols, ldx, rms);
    fbq_rms_apply_fwd_kernel<float><<<grid, kQuantThreads, 0, s>>>(
        reinterpret_cast<const float*>(x), rows, cols, ldx, gain, rms, reinterpret_cast<float*>(y),
        ldy, ctx, ld_ctx, ctx_scales, 511.0f);
  }
  return cudaGetLastError();
}

cudaError_t launch_rmsnorm_backward(const int16_t* ctx, int64_t ld_ctx, const float* ctx_scales,
                                    const void* gy, bool bf16, int64_t rows, int64_t cols,
                                    int64_t ldgy, const float* gain, void* gx, int64_t ldgx,
                                    float* grad_gain, double* row_ws, float* term, cudaStream_t s,
                                    const void* res, int64_t ldres) {
  const unsigned rb = (unsigned)((rows + 31) / 32);  // one warp per 32 rows
  const size_t sm16 = (size_t)kRsBwdStages * RsBwdLayout<__nv_bfloat16>::kStage;
  const size_t sm32 = (size_t)kRsBwdStages * RsBwdLayout<float>::kStage;
  if (cudaError_t e = smem_once<fbq_rms_rowstat_bwd_kernel<__nv_bfloat16>>(sm16)) return e;
  if (cudaError_t e = smem_once<fbq_rms_rowstat_bwd_kernel<float>>(sm32)) return e;
  double* inv = row_ws;
  double* corr = row_ws + rows;
  // apply: 256 threads x 2 columns across, rows strided over grid.y (~16 CTAs per SM)
  const unsigned gxd = (unsigned)((cols + 511) / 512);
  int64_t gyd = (148 * 16 + gxd - 1) / gxd;
  if (gyd > rows) gyd = rows;
  if (gyd > 65535) gyd = 65535;
  const dim3 blocks(gxd, (unsigned)(gyd < 1 ? 1 : gyd));
  if (bf16) {
    auto g = reinterpret_cast<const __nv_bfloat16*>(gy);
    fbq_rms_rowstat_bwd_kernel<__nv_bfloat16><<<rb, 32, sm16, s>>>(ctx, ld_ctx, ctx_scales, g, ldgy,
                                                                      rows, cols, gain, inv, corr);
    fbq_rms_apply_bwd_kernel<__nv_bfloat16><<<blocks, 256, 0, s>>>(
        ctx, ld_ctx, ctx_scales, g, ldgy, rows, cols, gain, inv, corr,
        reinterpret_cast<__nv_bfloat16*>(gx), ldgx, term, reinterpret_cast<const __nv_bfloat16*>(res), ldres);
  } else {
    auto g = reinterpret_cast<const float*>(gy);
    fbq_rms_rowstat_bwd_kernel<float><<<rb, 32, sm32, s>>>(ctx, ld_ctx, ctx_scales, g, ldgy, rows,
                                                              cols, gain, inv, corr);
    fbq_rms_apply_bwd_kernel<float><<<blocks, 256, 0, s>>>(ctx, ld_ctx, ctx_scales, g, ldgy, rows, cols,
                                                           gain, inv, corr, reinterpret_cast<float*>(gx),
                                                           ldgx, term, reinterpret_cast<const float*>(res), ldres);
  }
  fbq_rms_grad_gain_kernel<<<(unsigned)((cols + 31) / 32), 32, 0, s>>>(term, rows, cols, grad_gain);
  return cudaGetLastError();
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

// Element-wise rounding probes (exhaustive / adversarial tests against the
// reference double formulas).  path 0: the scalar rtn_code / sr_code; 1: the
// vector fast paths the kernels use (rtn_vec / sr_vec, requires |x| <= 127 a;
// bits[i] is then the splitmix64 COUNTER z, not the mixed bits); 2: the 10-bit
// context RTN (group_rtn's path, level 511, |x| <= 511 a; out_rtn holds n int16).
__global__ void fbq_round_probe_kernel(const float* x, const float* a, const uint64_t* bits,
                                       int8_t* out_rtn, int8_t* out_sr, int64_t n, int path) {
  if (path == 4) {
    // group_rtn's packed level-511 path (the 10-bit GluCombine contexts): the
    // 8-wide fast path at window(511) + the packed exact fix (rtn_fix_vec),
    // one vector per thread with the scale of its first element, int16 out
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < n / 8;
         g += (int64_t)gridDim.x * blockDim.x) {
      const float ai = a[8 * g];
      const float inv = ai > 0.0f ? __frcp_rn(ai) : 0.0f;
      float v[8];
      uint32_t w[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = x[8 * g + j];
      if (ai >= kTinyScale) {
        if (rtn_fast_vec_x<8>(v, ai, inv, w)) rtn_fix_vec<8>(v, ai, w);
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) w[j] = ai > 0.0f ? (uint32_t)rtn_code_slow(v[j], ai, 511.0f) : 0u;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) reinterpret_cast<int16_t*>(out_rtn)[8 * g + j] = (int16_t)(uint16_t)w[j];
    }
    return;
  }
  if (path == 3) {
    // the 8-wide packed RTN fast path with its two-level boundary test, one
    // vector per thread with the scale of the vector's first element
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < n / 8;
         g += (int64_t)gridDim.x * blockDim.x) {
      const float ai = a[8 * g];
      const float inv = ai > 0.0f ? __frcp_rn(ai) : 0.0f;
      float v[8];
      uint32_t w[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = x[8 * g + j];
      rtn_vec<8>(v, ai, inv, round_mode(ai), w);
#pragma unroll
      for (int j = 0; j < 8; ++j) out_rtn[8 * g + j] = (int8_t)(uint8_t)w[j];
    }
    return;
  }
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float ai = a[i];
    const float inv = ai > 0.0f ? __frcp_rn(ai) : 0.0f;
    if (path == 0) {
      if (out_rtn) out_rtn[i] = (int8_t)rtn_code(x[i], ai, inv);
      if (out_sr) out_sr[i] = (int8_t)sr_code(x[i], ai, inv, bits[i]);
    } else {
      const float v[1] = {x[i]};
      uint32_t w[1];
      if (path == 2) {
        const float s = ai;
        if (s >= kTinyScale) {
          if (rtn_fast_vec<1>(v, inv, rtn_window(511.0f), w)) rtn_exact_vec<1>(v, s, inv, 511.0f, w);
        } else {
          w[0] = s > 0.0f ? (uint32_t)rtn_code_slow(v[0], s, 511.0f) : 0u;
        }
        reinterpret_cast<int16_t*>(out_rtn)[i] = (int16_t)(uint16_t)w[0];  // int16 output
        continue;
      }
      const int mode = round_mode(ai);
      if (out_rtn) {
        rtn_vec<1>(v, ai, inv, mode, w);
        out_rtn[i] = (int8_t)(uint8_t)w[0];
      }
      if (out_sr) {
        sr_vec<1>(v, ai, inv, mode, bits[i], w);
        out_sr[i] = (int8_t)(uint8_t)w[0];
      }
    }
  }
}

// ------------------------------------------------------------------ launchers
template <class K>
static cudaError_t opt_in_smem(K kernel, size_t bytes) {
  return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

// Per-device, thread-safe one-time setup of one kernel instance (shared-memory
// opt-in, occupancy): function attributes are per device, and two host threads
// may launch concurrently.  No allocation or synchronisation.
constexpr int kMaxDev = 64;
struct DevOnce {
  std::once_flag flag[kMaxDev];
  cudaError_t err[kMaxDev] = {};
  int val[kMaxDev] = {};
};
template <class F>
static cudaError_t dev_once(DevOnce& o, F&& f, int* val = nullptr) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDev) return cudaErrorInvalidDevice;
  std::call_once(o.flag[dev], [&] { o.err[dev] = f(o.val[dev]); });
  if (val) *val = o.val[dev];
  return o.err[dev];
}

// Launch with programmatic stream serialisation when the grid follows
// fbq_zero_count_kernel (p.pdl): it may start while the zeroing grid drains.
template <typename... KArgs, typename... Args>
static cudaError_t launch_ex(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                             cudaStream_t s, bool pdl, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, args...);
}

__global__ void fbq_zero_count_kernel(int* count) {
  asm volatile("griddepcontrol.launch_dependents;");
  if (threadIdx.x == 0) *count = 0;
}
cudaError_t launch_zero_count(int* count, cudaStream_t s) {
  fbq_zero_count_kernel<<<1, 32, 0, s>>>(count);
  return cudaGetLastError();
}

template <typename T, bool kVec, int kSR>
static cudaError_t launch_k1_sr(const QuantParams& p, dim3 grid, cudaStream_t s) {
  const size_t smem = sizeof(T) * kTileElems;
  static DevOnce once;
  if (cudaError_t e = dev_once(once, [&](int&) {
        return opt_in_smem(fbq_quantize_block_kernel<T, kVec, kSR, sizeof(T) == 2 ? 4 : 1>, smem);
      }))
    return e;
  // bf16 tiles (32 KiB): four CTAs per SM at 64 registers (measured 7 % faster
  // than three at 76-82 registers for the two-plane SR launch); fp32 tiles
  // (64 KiB) are shared-memory bound at three CTAs anyway
  constexpr int kMinB = sizeof(T) == 2 ? 4 : 1;
  return launch_ex(fbq_quantize_block_kernel<T, kVec, kSR, kMinB>, grid, dim3(kQuantThreads), smem, s, p.pdl, p);
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

typedef CUresult (*PFN_encodeTiledQ)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                     const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                     const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                     CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static PFN_encodeTiledQ encode_fn() {
  static const PFN_encodeTiledQ fn = [] {  // thread-safe one-time lookup
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return reinterpret_cast<PFN_encodeTiledQ>(ptr);
    return (PFN_encodeTiledQ) nullptr;
  }();
  return fn;
}

static int num_sms() {
  static DevOnce once;
  int n = 0;
  dev_once(once, [](int& v) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    if (v <= 0) v = 148;
    return cudaSuccess;
  }, &n);
  return n > 0 ? n : 148;
}

template <typename T, int kSR, int kQStages>
static cudaError_t launch_k1_tma(const QuantParams& p, cudaStream_t s) {
  const size_t smem = (size_t)kQStages * sizeof(T) * kTileElems;
  static DevOnce once;
  int ctas_per_sm = 1;
  if (cudaError_t e = dev_once(once, [&](int& v) {
        if (cudaError_t e2 = opt_in_smem(fbq_quantize_tma_kernel<T, kSR, kQStages>, smem)) return e2;
        int n = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fbq_quantize_tma_kernel<T, kSR, kQStages>, kQuantThreads, smem) != cudaSuccess || n < 1)
          n = 1;
        v = n;
        return cudaSuccess;
      }, &ctas_per_sm))
    return e;
  CUtensorMap m;
  PFN_encodeTiledQ enc = encode_fn();
  if (!enc) return cudaErrorNotSupported;
  const size_t esz = sizeof(T);
  cuuint64_t dims[2] = {(cuuint64_t)p.cols, (cuuint64_t)p.rows};
  cuuint64_t strides[1] = {(cuuint64_t)(p.ldx * esz)};
  cuuint32_t box[2] = {(cuuint32_t)kBlock, (cuuint32_t)kBlock};
  cuuint32_t estr[2] = {1, 1};
  if (enc(&m, sizeof(T) == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
          const_cast<void*>(p.x), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  const int gcols = (int)((p.cols + kBlock - 1) / kBlock);
  const int64_t nblk = (int64_t)gcols * ((p.rows + kBlock - 1) / kBlock);
  int64_t grid = (int64_t)num_sms() * ctas_per_sm;
  if (grid > nblk) grid = nblk;
  return launch_ex(fbq_quantize_tma_kernel<T, kSR, kQStages>, dim3((unsigned)grid), dim3(kQuantThreads), smem, s,
                   p.pdl, m, p, nblk, gcols);
}
template <typename T, int kQStages, int kMinBlocks, int kSR>
static cudaError_t launch_k1_tma_reg(const QuantParams& p, cudaStream_t s) {
  const size_t smem = (size_t)kQStages * sizeof(T) * kTileElems;
  static DevOnce once;
  int ctas_per_sm = 1;
  if (cudaError_t e = dev_once(once, [&](int& v) {
        if (cudaError_t e2 = opt_in_smem(fbq_quantize_tma_reg_kernel<T, kQStages, kMinBlocks, kSR>, smem)) return e2;
        int n = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fbq_quantize_tma_reg_kernel<T, kQStages, kMinBlocks, kSR>, kQuantThreads, smem) != cudaSuccess || n < 1)
          n = 1;
        v = n;
        return cudaSuccess;
      }, &ctas_per_sm))
    return e;
  CUtensorMap m;
  PFN_encodeTiledQ enc = encode_fn();
  if (!enc) return cudaErrorNotSupported;
  const size_t esz = sizeof(T);
  cuuint64_t dims[2] = {(cuuint64_t)p.cols, (cuuint64_t)p.rows};
  cuuint64_t strides[1] = {(cuuint64_t)(p.ldx * esz)};
  cuuint32_t box[2] = {(cuuint32_t)kBlock, (cuuint32_t)kBlock};
  cuuint32_t estr[2] = {1, 1};
  if (enc(&m, sizeof(T) == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
          const_cast<void*>(p.x), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  const int gcols = (int)((p.cols + kBlock - 1) / kBlock);
  const int64_t nblk = (int64_t)gcols * ((p.rows + kBlock - 1) / kBlock);
  int64_t grid = (int64_t)num_sms() * ctas_per_sm;
  if (grid > nblk) grid = nblk;
  // dynamic block schedule when fbq_cuda_init() set up the counter ring (diag 4096: static)
  QuantParams q = p;
  q.blk_ctr = (g_quant_diag & 4096) ? nullptr : counter_slot();
  q.diag = (g_quant_diag & 16384) ? 1 : 0;
  return launch_ex(fbq_quantize_tma_reg_kernel<T, kQStages, kMinBlocks, kSR>, dim3((unsigned)grid), dim3(kQuantThreads),
                   smem, s, p.pdl, m, q, (int)nblk, gcols);
}

template <typename T>
static cudaError_t launch_k1_tma_any(QuantParams p, cudaStream_t s) {
  if (!p.sr_codes && p.sr_codes2) {
    p.sr_codes = p.sr_codes2;
    p.sr_seed = p.sr_seed2;
    p.sr_codes2 = nullptr;
  }
  // ring depth: 3 x 32 KiB (bf16, two CTAs per SM) / 3 x 64 KiB (fp32, one CTA per SM)
  if (p.sr_codes2) return launch_k1_tma<T, 2, 3>(p, s);
  if (p.sr_codes) return launch_k1_tma<T, 1, 3>(p, s);
  return launch_k1_tma<T, 0, 3>(p, s);
}

// diagnostics: 1 = force the smem-staged one-block-per-CTA K1, 2 = the
// persistent TMA-pipelined K1 for SR launches, 4 = bf16 TMA ring 3 stages x
// 2 CTAs per SM, 128 = bf16 RTN on the one-block-per-CTA register kernel
// instead of the persistent TMA one (8192x14336: 99 vs 79 us), 8 = SR
// launches on the register-resident K1 instead of the
// smem-staged one (A/B comparisons; results are identical.  Measured on B200:
// the register-resident SR variant is 25-45 % SLOWER -- with the RNG's ~17
// integer instructions per element it needs 128 registers, i.e. 16 warps per
// SM, too few to hide its latency; scripts/sr_ab.py)
int g_quant_diag = 0;

cudaError_t launch_quantize(const QuantParams& p, bool bf16, cudaStream_t s) {
  const dim3 grid((unsigned)((p.cols + kBlock - 1) / kBlock),
                  (unsigned)((p.rows + kBlock - 1) / kBlock));
  const size_t esz = bf16 ? 2 : 4;
  const bool vec = (reinterpret_cast<uintptr_t>(p.x) % 16 == 0) && ((p.ldx * esz) % 16 == 0) &&
                   (p.cols % (16 / esz) == 0);
  // TMA path: 16-byte aligned base and row stride (the tensor-map rules), and
  // enough blocks to fill the machine (small tensors keep the simple kernel)
  const int64_t nblk = (int64_t)grid.x * grid.y;
  // register-resident K1: RTN / fallback detect with 8-byte aligned code planes
  const bool sr = p.sr_codes || p.sr_codes2;
  if (vec && !(g_quant_diag & 1) && p.vec_store && (!sr || (g_quant_diag & 8))) {
    QuantParams q = p;  // compact the stochastic planes into kSR = 0, 1, 2
    if (!q.sr_codes && q.sr_codes2) {
      q.sr_codes = q.sr_codes2;
      q.sr_seed = q.sr_seed2;
      q.sr_codes2 = nullptr;
    }
    const int nsr = q.sr_codes2 ? 2 : (q.sr_codes ? 1 : 0);
    if (bf16 && nblk >= 2 * num_sms() && p.rows < (1ll << 31) && p.cols < (1ll << 31) &&
        !(g_quant_diag & 128)) {
      if (nsr == 2) return launch_k1_tma_reg<__nv_bfloat16, 3, 2, 2>(q, s);
      if (nsr == 1) return launch_k1_tma_reg<__nv_bfloat16, 3, 2, 1>(q, s);
      // one ring stage x four CTAs (32 warps) per SM: a slot goes back to TMA
      // as soon as its tile is in registers, so one stage already overlaps
      // the next tile's load with this tile's rounding, and the freed shared
      // memory buys a fourth CTA (64 registers; measured 2-5 % faster than
      // 2 stages x 3 CTAs on C2, diag 2048; 3 x 2: diag 4)
      if (g_quant_diag & 2048) return launch_k1_tma_reg<__nv_bfloat16, 2, 3, 0>(q, s);
      return (g_quant_diag & 4) ? launch_k1_tma_reg<__nv_bfloat16, 3, 2, 0>(q, s)
                                : launch_k1_tma_reg<__nv_bfloat16, 1, 4, 0>(q, s);
    }
    const dim3 b(kQuantThreads);
    if (bf16) {
      if (nsr == 2) return launch_ex(fbq_quantize_reg_kernel<__nv_bfloat16, 2>, grid, b, 0, s, q.pdl, q);
      if (nsr == 1) return launch_ex(fbq_quantize_reg_kernel<__nv_bfloat16, 1>, grid, b, 0, s, q.pdl, q);
      return launch_ex(fbq_quantize_reg_kernel<__nv_bfloat16, 0>, grid, b, 0, s, q.pdl, q);
    }
    if (nsr == 2) return launch_ex(fbq_quantize_reg_kernel<float, 2>, grid, b, 0, s, q.pdl, q);
    if (nsr == 1) return launch_ex(fbq_quantize_reg_kernel<float, 1>, grid, b, 0, s, q.pdl, q);
    return launch_ex(fbq_quantize_reg_kernel<float, 0>, grid, b, 0, s, q.pdl, q);
  }
  if (vec && (g_quant_diag & 2) && nblk >= 2 * num_sms() && p.rows < (1ll << 31) &&
      p.cols < (1ll << 31))
    return bf16 ? launch_k1_tma_any<__nv_bfloat16>(p, s) : launch_k1_tma_any<float>(p, s);
  if (bf16) return vec ? launch_k1<__nv_bfloat16, true>(p, grid, s)
                       : launch_k1<__nv_bfloat16, false>(p, grid, s);
  return vec ? launch_k1<float, true>(p, grid, s) : launch_k1<float, false>(p, grid, s);
}

template <bool kPacked>
static cudaError_t launch_glu_forward_t(const GluParams& g, const QuantParams& p, bool bf16, cudaStream_t s) {
  const dim3 grid((unsigned)((g.cols + kBlock - 1) / kBlock),
                  (unsigned)((g.rows + kBlock - 1) / kBlock));
  // staged (default): h computed once into shared memory, three CTAs per SM
  // (442 us on the C3 shape); diagnostics 256 = the direct variant that re-reads
  // a|b from L2 and re-evaluates h per pass at four CTAs per SM (505 us)
  if (bf16) {
    if (g_quant_diag & 256)
      return launch_ex(fbq_glu_forward_kernel<__nv_bfloat16, false, 4, kPacked>, grid, dim3(kQuantThreads), 0, s,
                       p.pdl, g, p);
    const size_t smem = 2 * sizeof(__nv_bfloat16) * kTileElems;  // a|b rows, then h (fp32) in place
    if (cudaError_t e = opt_in_smem(fbq_glu_forward_kernel<__nv_bfloat16, true, 3, kPacked>, smem)) return e;
    return launch_ex(fbq_glu_forward_kernel<__nv_bfloat16, true, 3, kPacked>, grid, dim3(kQuantThreads), smem, s,
                     p.pdl, g, p);
  }
  const size_t smem = 2 * sizeof(float) * kTileElems;
  if (cudaError_t e = opt_in_smem(fbq_glu_forward_kernel<float, true, 1, kPacked>, smem)) return e;
  return launch_ex(fbq_glu_forward_kernel<float, true, 1, kPacked>, grid, dim3(kQuantThreads), smem, s, p.pdl, g, p);
}

cudaError_t launch_glu_forward(const GluParams& g, const QuantParams& p, bool bf16, cudaStream_t s) {
  return g.ctx_packed ? launch_glu_forward_t<true>(g, p, bf16, s) : launch_glu_forward_t<false>(g, p, bf16, s);
}

template <bool kPacked>
static cudaError_t launch_glu_backward_t(const GluBwdParams& g, bool bf16, cudaStream_t s) {
  const dim3 grid((unsigned)((g.cols + kBlock - 1) / kBlock),
                  (unsigned)((g.rows + kBlock - 1) / kBlock));
  const bool staged = (g_quant_diag & 32) != 0;  // diagnostics: dH staged in shared memory
  if (bf16) {
    if (!staged) {
      // four CTAs (32 warps) per SM: 64 registers; measured 484 us vs 590 us
      // at 82 registers / three CTAs (int16 contexts); packed 10-bit contexts:
      // 582 us at four CTAs (a few spilled bytes) vs 621 us at three
      fbq_glu_backward_kernel<__nv_bfloat16, false, 4, kPacked><<<grid, kQuantThreads, 0, s>>>(g);
      return cudaGetLastError();
    }
    const size_t smem = sizeof(__nv_bfloat16) * kTileElems;
    if (cudaError_t e = opt_in_smem(fbq_glu_backward_kernel<__nv_bfloat16, true, 1, kPacked>, smem)) return e;
    fbq_glu_backward_kernel<__nv_bfloat16, true, 1, kPacked><<<grid, kQuantThreads, smem, s>>>(g);
  } else {
    if (!staged) {
      fbq_glu_backward_kernel<float, false, 3, kPacked><<<grid, kQuantThreads, 0, s>>>(g);
      return cudaGetLastError();
    }
    const size_t smem = sizeof(float) * kTileElems;
    if (cudaError_t e = opt_in_smem(fbq_glu_backward_kernel<float, true, 1, kPacked>, smem)) return e;
    fbq_glu_backward_kernel<float, true, 1, kPacked><<<grid, kQuantThreads, smem, s>>>(g);
  }
  return cudaGetLastError();
}

cudaError_t launch_glu_backward(const GluBwdParams& g, bool bf16, cudaStream_t s) {
  return g.ctx_packed ? launch_glu_backward_t<true>(g, bf16, s) : launch_glu_backward_t<false>(g, bf16, s);
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
                               int8_t* out_rtn, int8_t* out_sr, int64_t n, int path, cudaStream_t s) {
  int blocks = (int)((n + 255) / 256);
  if (blocks > 148 * 32) blocks = 148 * 32;
  if (blocks < 1) blocks = 1;
  fbq_round_probe_kernel<<<blocks, 256, 0, s>>>(x, a, bits, out_rtn, out_sr, n, path);
  return cudaGetLastError();
}

cudaError_t launch_rmsnorm_quantize(const QuantParams& p, bool bf16, const float* gain, int16_t* ctx,
                                    int64_t ld_ctx, float* ctx_scales, float* rms, cudaStream_t s) {
  const unsigned rb = (unsigned)((p.rows + 31) / 32);
  const size_t sm16 = (size_t)kRsStages * 32 * (kRsCols * 2 + 16), sm32 = (size_t)kRsStages * 32 * (kRsCols * 4 + 16);
  if (cudaError_t e = smem_once<fbq_rms_rowstat_fwd_kernel<__nv_bfloat16>>(sm16)) return e;
  if (cudaError_t e = smem_once<fbq_rms_rowstat_fwd_kernel<float>>(sm32)) return e;
  if (bf16) fbq_rms_rowstat_fwd_kernel<__nv_bfloat16><<<rb, 32, sm16, s>>>(
      reinterpret_cast<const __nv_bfloat16*>(p.x), p.rows, p.cols, p.ldx, rms);
  else fbq_rms_rowstat_fwd_kernel<float><<<rb, 32, sm32, s>>>(reinterpret_cast<const float*>(p.x), p.rows,
                                                             p.cols, p.ldx, rms);
  if (cudaError_t e = cudaGetLastError()) return e;
  // (launched without programmatic dependence: the kernel reads rms[] at once)
  QuantParams q = p;  // compact the stochastic planes into kSR = 0, 1, 2
  if (!q.sr_codes && q.sr_codes2) {
    q.sr_codes = q.sr_codes2;
    q.sr_seed = q.sr_seed2;
    q.sr_codes2 = nullptr;
  }
  const int nsr = q.sr_codes2 ? 2 : (q.sr_codes ? 1 : 0);
  const dim3 grid((unsigned)((p.cols + kBlock - 1) / kBlock), (unsigned)((p.rows + kBlock - 1) / kBlock));
  const dim3 b(kQuantThreads);
  // y staged as the K1 tile: bf16 32 KiB at four CTAs per SM, fp32 64 KiB (as launch_k1_sr)
  const size_t t16 = 2 * kTileElems, t32 = 4 * kTileElems;
#define FBQ_RQ(TT, NSR, MB, SM)                                                                        \
  do {                                                                                                  \
    if (cudaError_t e = smem_once<fbq_rms_quant_kernel<TT, NSR, MB>>(SM)) return e;                     \
    return launch_ex(fbq_rms_quant_kernel<TT, NSR, MB>, grid, b, SM, s, false, q, gain, rms, ctx,       \
                     ld_ctx, ctx_scales);                                                               \
  } while (0)
  if (bf16) {
    if (nsr == 2) FBQ_RQ(__nv_bfloat16, 2, 4, t16);
    if (nsr == 1) FBQ_RQ(__nv_bfloat16, 1, 4, t16);
    FBQ_RQ(__nv_bfloat16, 0, 4, t16);
  }
  if (nsr == 2) FBQ_RQ(float, 2, 1, t32);
  if (nsr == 1) FBQ_RQ(float, 1, 1, t32);
  FBQ_RQ(float, 0, 1, t32);
#undef FBQ_RQ
}

// (after launch_ex)
cudaError_t launch_sgd_quantize(float* w, const float* g, int64_t rows, int64_t cols, double lr,
                                int8_t* codes, int64_t ldq, float* scales, cudaStream_t s) {
  QuantParams p = {};
  p.x = w;
  p.rows = rows;
  p.cols = cols;
  p.ldx = cols;
  p.ldq = ldq;
  p.vec_store = 1;
  p.mask_mode = kMaskNone;
  p.codes = codes;
  p.scales = scales;
  const dim3 grid((unsigned)((cols + kBlock - 1) / kBlock), (unsigned)((rows + kBlock - 1) / kBlock));
  return launch_ex(fbq_sgd_quantize_kernel, grid, dim3(kQuantThreads), 0, s, false, p, w, g, lr);
}

cudaError_t launch_silu_forward(const void* x, bool bf16, int64_t rows, int64_t cols, int64_t ldx, void* y,
                                int64_t ldy, int16_t* ctx, int64_t ld_ctx, float* ctx_scales, float level,
                                bool exact, cudaStream_t s) {
  const dim3 grid((unsigned)((cols + kBlock - 1) / kBlock), (unsigned)((rows + kBlock - 1) / kBlock));
#define FBQ_SF(T, E) fbq_silu_fwd_kernel<T, E><<<grid, kQuantThreads, 0, s>>>(                      \
      reinterpret_cast<const T*>(x), rows, cols, ldx, reinterpret_cast<T*>(y), ldy, ctx, ld_ctx,  \
      ctx_scales, level)
  if (bf16) {
    if (exact) FBQ_SF(__nv_bfloat16, true);
    else FBQ_SF(__nv_bfloat16, false);
  } else {
    if (exact) FBQ_SF(float, true);
    else FBQ_SF(float, false);
  }
#undef FBQ_SF
  return cudaGetLastError();
}

cudaError_t launch_silu_backward(const int16_t* ctx, int64_t ld_ctx, const float* ctx_scales, const void* gy,
                                 bool bf16, int64_t rows, int64_t cols, int64_t ldgy, void* gx, int64_t ldgx,
                                 bool exact, cudaStream_t s) {
  const unsigned gxd = (unsigned)((cols + 511) / 512);
  int64_t gyd = (148 * 16 + gxd - 1) / gxd;
  if (gyd > rows) gyd = rows;
  if (gyd > 65535) gyd = 65535;
  const dim3 grid(gxd, (unsigned)(gyd < 1 ? 1 : gyd));
#define FBQ_SB(T, E) fbq_silu_bwd_kernel<T, E><<<grid, 256, 0, s>>>(                                 \
      ctx, ld_ctx, ctx_scales, reinterpret_cast<const T*>(gy), ldgy, rows, cols, reinterpret_cast<T*>(gx), ldgx)
  if (bf16) {
    if (exact) FBQ_SB(__nv_bfloat16, true);
    else FBQ_SB(__nv_bfloat16, false);
  } else {
    if (exact) FBQ_SB(float, true);
    else FBQ_SB(float, false);
  }
#undef FBQ_SB
  return cudaGetLastError();
}

}  // namespace fbq
