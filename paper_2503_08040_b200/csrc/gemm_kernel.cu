// K3: block-quantized / fallback INT8 GEMM on the 5th-gen tensor cores.
//
// Semantics (reference gemm.cpp:101-186, run_block_gemm): for every output
// element (i, j) and every 128-deep k-block bk in ASCENDING order
//     P   = sum_k a[i,k] * b[k,j]                        (exact int32)
//     acc = fl(acc + fl(fl(sA(bi,bk) * sB(bk,bj)) * float(P)))
//     if u(bi,bk):  (fallback, Algorithm 1)
//         P2  = sum_k res[i,k] * b[k,j]
//         acc = fl(acc + fl(fl(rA(bi,bk) * sB(bk,bj)) * float(P2)))
// kEpiExact reproduces this sequence bit-for-bit; kEpiFma fuses the scale
// multiply into one FMA (acc = fma(float(P), s, acc); relative Frobenius
// difference ~5e-8, inside SPEC.md's 1e-5 bound); kEpiDump writes the raw
// per-block int32 products P (parity of the "per-block INT32 accumulators").
//
// Structure (one CTA per SM, persistent, warp-specialised, 320 threads):
//   warp 0      TMA producer: A (128x128 int8), B (256x128 int8) and -- only for
//               flagged A blocks -- the residual A tile, into a 3-stage
//               128B-swizzled smem ring (mbarrier full/empty pipeline).
//   warp 1      tcgen05.mma.cta_group::1.kind::i8, M=128 N=256 K=32 (x4 per
//               k-block) issued by one thread into one of two 256-column int32
//               TMEM slots; every k-block (and every residual) is one "item".
//               A residual item re-uses the B tile already in smem.
//   warps 2..9  epilogue: tcgen05.ld the item's int32 block products,
//               int32->fp32 (exact magic-number conversion), scale and
//               accumulate in registers; free the TMEM slot; after the last
//               k-block store the 128x256 fp32/bf16 tile.
// Operand majorness (K- or MN-major) is a descriptor bit, so the backward
// products dX = dY W and dW = dY^T X read the SAME int8 code planes as the
// forward without any transposed copies (reference transposes: quant.cpp:106-126).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

#include "gemm_kernel.cuh"
#include "sm100.cuh"

namespace fbq {

using namespace sm100;

constexpr int kBM = 128, kBN = 256, kBK = 128;
constexpr int kStages = 3;
constexpr int kTileA = kBM * kBK;  // 16 KiB
constexpr int kTileB = kBN * kBK;  // 32 KiB
constexpr int kStageBytes = 2 * kTileA + kTileB;
constexpr int kTmemCols = 512;     // 2 slots x 256 int32 columns
constexpr int kEpiWarps = 8;
constexpr int kThreads = 64 + kEpiWarps * 32;
constexpr size_t kSmemBytes = 1024 + (size_t)kStages * kStageBytes + 256;

struct SmemLayout {
  static __device__ __forceinline__ uint8_t* base(uint8_t* raw) {
    return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  }
};

__device__ __forceinline__ bool mask_bit(const uint32_t* bits, int64_t blk) {
  return (bits[blk >> 5] >> (blk & 31)) & 1u;
}

template <int kEpi>
__global__ void __maxnreg__(200)
fbq_gemm_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_r,
                const __grid_constant__ CUtensorMap map_b, const GemmParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = SmemLayout::base(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  uint64_t* full = bars;                 // [kStages]
  uint64_t* empty = bars + kStages;      // [kStages]
  uint64_t* tfull = bars + 2 * kStages;  // [2]
  uint64_t* tempty = tfull + 2;          // [2]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const bool has_res = p.mask_bits != nullptr;
  const int NT = (p.NB + 1) >> 1;  // 256-wide n tiles

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(tfull + s, 1);
      mbar_init(tempty + s, kEpiWarps);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<kTmemCols>(tmem_holder);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  auto a_blk = [&](int bm, int bk) -> int64_t {
    return p.a_major == 0 ? (int64_t)bm * p.KB + bk : (int64_t)bk * p.MB + bm;
  };
  auto b_blk = [&](int bk, int bn) -> int64_t {
    return p.b_major == 0 ? (int64_t)bn * p.KB + bk : (int64_t)bk * p.NB + bn;
  };

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      tma_prefetch(&map_a);
      tma_prefetch(&map_b);
      if (has_res) tma_prefetch(&map_r);
      const uint64_t pol_a = l2_policy_evict_last();
      const uint64_t pol_b = l2_policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < p.num_tiles; tile += gridDim.x) {
        const int bm = tile / NT, bn2 = tile % NT;
        for (int bk = 0; bk < p.KB; ++bk) {
          const bool masked = has_res && mask_bit(p.mask_bits, a_blk(bm, bk));
          mbar_wait(empty + stage, phase ^ 1);
          uint8_t* sa = smem + stage * kStageBytes;
          uint8_t* sr = sa + kTileA;
          uint8_t* sb = sa + 2 * kTileA;
          mbar_arrive_expect_tx(full + stage, kTileA + kTileB + (masked ? kTileA : 0));
          const int k0 = bk * kBK, m0 = bm * kBM, n0 = bn2 * kBN;
          if (p.a_major == 0) {
            tma_load_2d(sa, &map_a, full + stage, k0, m0, pol_a);
            if (masked) tma_load_2d(sr, &map_r, full + stage, k0, m0, pol_a);
          } else {
            tma_load_2d(sa, &map_a, full + stage, m0, k0, pol_a);
            if (masked) tma_load_2d(sr, &map_r, full + stage, m0, k0, pol_a);
          }
          if (p.b_major == 0) {
            tma_load_2d(sb, &map_b, full + stage, k0, n0, pol_b);
          } else {
            tma_load_2d(sb, &map_b, full + stage, n0, k0, pol_b);
            tma_load_2d(sb + kTileA, &map_b, full + stage, n0 + 128, k0, pol_b);
          }
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    const uint32_t idesc = idesc_i8(kBM, kBN, p.a_major, p.b_major);
    int stage = 0;
    uint32_t phase = 0;
    uint32_t item = 0;
    for (int tile = blockIdx.x; tile < p.num_tiles; tile += gridDim.x) {
      const int bm = tile / NT;
      for (int bk = 0; bk < p.KB; ++bk) {
        const bool masked = has_res && mask_bit(p.mask_bits, a_blk(bm, bk));
        mbar_wait(full + stage, phase);
        tc_fence_after();
        const uint32_t sa = smem_u32(smem + stage * kStageBytes);
        const uint32_t sr = sa + kTileA;
        const uint32_t sb = sa + 2 * kTileA;
        for (int r = 0; r < (masked ? 2 : 1); ++r) {
          const uint32_t slot = item & 1;
          mbar_wait(tempty + slot, ((item >> 1) & 1) ^ 1);
          tc_fence_after();
          if (lane == 0) {
            const uint32_t a_base = r ? sr : sa;
#pragma unroll
            for (int kk = 0; kk < kBK / 32; ++kk) {
              // K-major: advance 32 B inside the 128 B swizzle row;
              // MN-major: advance 32 k-rows = 4 x (8-row core groups of 1 KiB).
              const uint32_t a_off = p.a_major == 0 ? kk * 32 : kk * 4096;
              const uint32_t b_off = p.b_major == 0 ? kk * 32 : kk * 4096;
              const uint64_t ad = smem_desc_sw128(a_base + a_off, 16, 1024);
              const uint64_t bd = p.b_major == 0 ? smem_desc_sw128(sb + b_off, 16, 1024)
                                                 : smem_desc_sw128(sb + b_off, kTileA, 1024);
              mma_i8(tmem_base + slot * 256, ad, bd, idesc, kk > 0 ? 1u : 0u);
            }
            mma_commit(tfull + slot);
          }
          __syncwarp();
          ++item;
        }
        if (lane == 0) mma_commit(empty + stage);
        __syncwarp();
        if (++stage == kStages) { stage = 0; phase ^= 1; }
      }
    }
  } else {
    // ===================== epilogue =====================
    const int ew = warp - 2;
    const int q = warp & 3;  // TMEM lane quadrant this warp may access
    const int h = ew >> 2;   // which 128-column half of the 256-wide tile
    const int row_in_tile = q * 32 + lane;
    const uint32_t lane_addr = (uint32_t)(q * 32) << 16;
    uint32_t item = 0;
    for (int tile = blockIdx.x; tile < p.num_tiles; tile += gridDim.x) {
      const int bm = tile / NT, bn2 = tile % NT;
      const int bn = bn2 * 2 + h;
      const bool bn_ok = bn < p.NB;
      float acc[128];
#pragma unroll
      for (int i = 0; i < 128; ++i) acc[i] = 0.0f;
      for (int bk = 0; bk < p.KB; ++bk) {
        const int64_t ab = a_blk(bm, bk);
        const bool masked = has_res && mask_bit(p.mask_bits, ab);
        const float sb = bn_ok ? p.b_scales[b_blk(bk, bn)] : 0.0f;
        for (int r = 0; r < (masked ? 2 : 1); ++r) {
          const uint32_t slot = item & 1;
          const float sa = r ? p.res_scales[ab] : p.a_scales[ab];
          const float s = __fmul_rn(sa, sb);  // gemm.cpp:163 / :172
          mbar_wait(tfull + slot, (item >> 1) & 1);
          tc_fence_after();
          const uint32_t taddr = tmem_base + lane_addr + slot * 256 + h * 128;
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            uint32_t v[32];
            tmem_ld32(taddr + c * 32, v);
            tmem_ld_wait();
            if (c == 3) {
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(tempty + slot);
            }
            if constexpr (kEpi == kEpiDump) {
              const int64_t grow = (int64_t)bm * kBM + row_in_tile;
              if (bn_ok) {
                int32_t* d = p.dump + (r ? p.dump_res_offset : 0) +
                             ((((int64_t)bm * p.NB + bn) * p.KB + bk) * kBM + row_in_tile) * 128 +
                             c * 32;
#pragma unroll
                for (int i = 0; i < 32; ++i) d[i] = (int32_t)v[i];
              }
              (void)grow;
            } else {
#pragma unroll
              for (int i = 0; i < 32; ++i) {
                // exact int32 -> fp32 for |P| < 2^22 (128*127^2 = 2,064,512)
                const float pf = __fsub_rn(__int_as_float((int)v[i] + 0x4B400000), 12582912.0f);
                if constexpr (kEpi == kEpiExact) {
                  acc[c * 32 + i] = __fadd_rn(acc[c * 32 + i], __fmul_rn(s, pf));
                } else {
                  acc[c * 32 + i] = __fmaf_rn(pf, s, acc[c * 32 + i]);
                }
              }
            }
          }
          ++item;
        }
      }
      if constexpr (kEpi != kEpiDump) {
        const int64_t grow = (int64_t)bm * kBM + row_in_tile;
        const int64_t gcol0 = (int64_t)bn * 128;
        if (bn_ok && grow < p.M) {
          if (p.out_bf16) {
            __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(p.out) + grow * p.ldo + gcol0;
#pragma unroll
            for (int i = 0; i < 128; ++i) {
              if (gcol0 + i < p.N) {
                float val = acc[i];
                if (p.accumulate) val = __fadd_rn(__bfloat162float(o[i]), val);
                o[i] = __float2bfloat16_rn(val);
              }
            }
          } else {
            float* o = reinterpret_cast<float*>(p.out) + grow * p.ldo + gcol0;
            if (p.vec_store && gcol0 + 128 <= p.N) {
#pragma unroll
              for (int i = 0; i < 128; i += 4) {
                float4 val = make_float4(acc[i], acc[i + 1], acc[i + 2], acc[i + 3]);
                if (p.accumulate) {
                  const float4 old = *reinterpret_cast<const float4*>(o + i);
                  val.x = __fadd_rn(old.x, val.x);
                  val.y = __fadd_rn(old.y, val.y);
                  val.z = __fadd_rn(old.z, val.z);
                  val.w = __fadd_rn(old.w, val.w);
                }
                *reinterpret_cast<float4*>(o + i) = val;
              }
            } else {
#pragma unroll
              for (int i = 0; i < 128; ++i) {
                if (gcol0 + i < p.N) o[i] = p.accumulate ? __fadd_rn(o[i], acc[i]) : acc[i];
              }
            }
          }
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<kTmemCols>(tmem_base);
}

// ----------------------------------------------------------------- host side
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                    const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encode() {
  static PFN_encodeTiled fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled>(ptr);
  }
  return fn;
}

// int8 2D map: inner extent `inner` (contiguous), `outer` rows of `ld` bytes.
static bool make_map(CUtensorMap* m, const void* base, int64_t inner, int64_t outer, int64_t ld,
                     uint32_t box_inner, uint32_t box_outer) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)ld};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int gemm_num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

cudaError_t launch_gemm(const GemmOperands& o, GemmParams p, int epi, cudaStream_t s) {
  CUtensorMap ma, mr, mb;
  const int64_t M = p.M, N = p.N, K = p.K;
  bool ok = true;
  if (p.a_major == 0) ok &= make_map(&ma, o.a_codes, K, M, o.lda, 128, 128);
  else ok &= make_map(&ma, o.a_codes, M, K, o.lda, 128, 128);
  if (o.res_codes) {
    if (p.a_major == 0) ok &= make_map(&mr, o.res_codes, K, M, o.lda, 128, 128);
    else ok &= make_map(&mr, o.res_codes, M, K, o.lda, 128, 128);
  } else {
    mr = ma;
  }
  if (p.b_major == 0) ok &= make_map(&mb, o.b_codes, K, N, o.ldb, 128, 256);
  else ok &= make_map(&mb, o.b_codes, N, K, o.ldb, 128, 128);
  if (!ok) return cudaErrorInvalidValue;

  p.num_tiles = p.MB * ((p.NB + 1) / 2);
  const int grid = p.num_tiles < gemm_num_sms() ? p.num_tiles : gemm_num_sms();
  cudaError_t e;
  switch (epi) {
    case kEpiExact:
      e = cudaFuncSetAttribute(fbq_gemm_kernel<kEpiExact>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes);
      if (e != cudaSuccess) return e;
      fbq_gemm_kernel<kEpiExact><<<grid, kThreads, kSmemBytes, s>>>(ma, mr, mb, p);
      break;
    case kEpiFma:
      e = cudaFuncSetAttribute(fbq_gemm_kernel<kEpiFma>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes);
      if (e != cudaSuccess) return e;
      fbq_gemm_kernel<kEpiFma><<<grid, kThreads, kSmemBytes, s>>>(ma, mr, mb, p);
      break;
    default:
      e = cudaFuncSetAttribute(fbq_gemm_kernel<kEpiDump>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes);
      if (e != cudaSuccess) return e;
      fbq_gemm_kernel<kEpiDump><<<grid, kThreads, kSmemBytes, s>>>(ma, mr, mb, p);
      break;
  }
  return cudaGetLastError();
}

}  // namespace fbq
