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
// Structure (one CTA per SM, persistent, warp-specialised, 12 warps):
//   warp 0      TMA producer: A (128x128 int8), B (256x128 int8) and -- only for
//               flagged A blocks -- the residual A tile, into a 3-stage
//               128B-swizzled smem ring (mbarrier full/empty pipeline).
//   warp 1      tcgen05.mma.cta_group::1.kind::i8, M=128 N=256 K=32 (x4 per
//               k-block) issued by one thread into one of two 256-column int32
//               TMEM slots; every k-block (and every residual) is one "item".
//               A residual item re-uses the B tile already in smem.
//   warp 2      scale loader: per tile, stages fl(sA*sB), fl(rA*sB) and the
//               fallback flag of every k-block into a double-buffered smem page
//               (all roles read the flags from there; no global loads on the
//               issue paths).
//   warps 4-11  epilogue (2 warpgroups, setmaxnreg 224): tcgen05.ld the item's
//               int32 products (double-buffered 32-column chunks), free the
//               TMEM slot, I2F + FFMA2 (FMUL2 + FFMA2 in exact mode) into
//               register accumulators, and after the last k-block store the
//               tile.  Measured on B200: the FP32 pipe does 128 element-ops/clk/SM,
//               so convert + scale-accumulate runs at 64 elements/clk/SM -- exactly
//               the int8 MMA rate for 128-deep k-blocks (8192 MAC/clk/SM / 128).
// Operand majorness (K- or MN-major) is a descriptor bit, so the backward
// products dX = dY W and dW = dY^T X read the SAME int8 code planes as the
// forward without any transposed copies (reference transposes: quant.cpp:106-126).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <atomic>
#include <cstdint>
#include <mutex>

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
constexpr int kThreads = 128 + kEpiWarps * 32;  // WG0: TMA, MMA, scales, idle; WG1-2: epilogue
constexpr int kPage = 32;                       // k-blocks per staged scale page
constexpr int kOutChunk = 4096;                 // per-warp output staging buffer (TMA store box)

struct ScalePage {
  float prim[2][kPage];  // fl(sA * sB) for the two 128-column halves
  float res[2][kPage];   // fl(rA * sB) (flagged k-blocks only)
  uint8_t flag[kPage];   // fallback bit u(bm, bk)
  int tile;              // the tile this page belongs to; -1: no more tiles (all roles exit)
  int pg;                // first k-block of the page
};

constexpr size_t kSmemBytes =
    (size_t)kStages * kStageBytes + (size_t)kEpiWarps * kOutChunk + 2 * sizeof(ScalePage) + 256;
static_assert(kSmemBytes <= 232448, "shared memory budget");

// Tile rasterisation, chosen per launch so that one operand stays resident in
// the 126 MB L2 while the other streams once:
//  * A small (<= 48 MiB) and B large (> 96 MiB): group_m = MB -- bm fastest over ALL block-rows, so
//    the ~148 resident CTAs share a couple of B column panels and A is re-read
//    from L2 only (e.g. the gate/up forward: X codes 32 MiB, W 112 MiB);
//  * B small and A large: n_fastest -- every bn of one block-row before the next,
//    B re-read from L2 only (e.g. dW_gate/up: the X context 32 MiB);
//  * else groups of kGroupM block-rows (bm fastest), sharing kGroupM A
//    row-panels and ~148/kGroupM B column-panels in L2.
// With kGroupM groups everywhere the gate/up forward re-read all of B once per
// group (1.03 GB of DRAM reads for 0.15 GB of operands, ncu).
constexpr int kGroupM = 8;
//  * n_fastest = c > 0: bn fastest inside chunks of c n-tiles (c >= NT: the
//    whole N), chunk after chunk -- one pinned chunk of B, A streamed once per chunk.
__device__ __forceinline__ void tile_coords(int tile, int MB, int NT, int group_m, int n_fastest,
                                            int& bm, int& bn2) {
  if (n_fastest) {
    const int c = n_fastest < NT ? n_fastest : NT;
    const int chunk = tile / (MB * c);
    const int in = tile - chunk * (MB * c);
    const int width = c < NT - chunk * c ? c : NT - chunk * c;  // the last chunk may be narrower
    bm = in / width;
    bn2 = chunk * c + (in - bm * width);
    return;
  }
  const int per_group = group_m * NT;
  const int group = tile / per_group;
  const int first = group * group_m;
  const int rows = min(group_m, MB - first);
  const int in = tile - group * per_group;
  bm = first + in % rows;
  bn2 = in / rows;
}

__device__ __forceinline__ bool mask_bit(const uint32_t* bits, int64_t blk) {
  return (bits[blk >> 5] >> (blk & 31)) & 1u;
}

// int32 -> fp32 is I2F (ALU pipe, exact for |P| < 2^24), then one FFMA2 per
// element pair (FMA mode).  `one` is a runtime 1.0f: ptxas contracts FMUL2 +
// FADD2 into FFMA2 even for the _rn intrinsics, but cannot fold a multiply by an
// unknown value, so the exact chain fl(acc + fl(s*P)) is expressed as FMUL2 then
// FFMA2(t, one, acc).  (Decoding biased words on the FMA pipe instead of I2F was
// evaluated twice -- round 1 with TMEM bias fills, round 2 with offset-binary
// operands -- and did not pay.)
template <int kEpi>
__device__ __forceinline__ void consume(const uint32_t (&v)[32], float2* acc, float s, float one) {
  const float2 s2 = make_float2(s, s);
  const float2 one2 = make_float2(one, one);
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const float2 pf = make_float2(__int2float_rn((int)v[2 * i]), __int2float_rn((int)v[2 * i + 1]));
    if constexpr (kEpi == kEpiExact) {
      acc[i] = __ffma2_rn(__fmul2_rn(s2, pf), one2, acc[i]);  // fl(acc + fl(s * P))
    } else {
      acc[i] = __ffma2_rn(pf, s2, acc[i]);
    }
  }
}

// Epilogue warps: warp (4 + q + 4h) owns TMEM lane quadrant q and the
// 128-column half h of every 128 x 256 tile.
// kProf: per-item timeline of warp q == 0 (clock64, diagnostics only).
template <int kEpi, int h, bool kProf, bool kDiag>
__device__ __forceinline__ void epilogue_role(const GemmParams& p, const CUtensorMap* map_o,
                                              uint8_t* obuf, ScalePage* pages, uint64_t* tfull,
                                              uint64_t* tempty, uint64_t* sfull, uint64_t* sempty,
                                              uint32_t* tmem_holder, int warp, int lane, int NT) {
  const int q = warp & 3;  // TMEM lane quadrant this warp may access
  const int row_in_tile = q * 32 + lane;
  const uint32_t lane_addr = (uint32_t)(q * 32) << 16;

  uint32_t item = 0, pc = 0;
  uint32_t tw = 0, tl = 0, tpre = 0, tpost = 0, t0 = 0, t1 = 0, t2 = 0, t3 = 0;
  // tiles arrive through the scale pages (the scale-loader warp is the
  // scheduler): the first page of each tile carries its index, -1 ends
  for (;;) {
    mbar_wait_sleep(sfull + (pc & 1), (pc >> 1) & 1);
    const int tile = pages[pc & 1].tile;
    if (tile < 0) break;
    int bm, bn2;
    tile_coords(tile, p.MB, NT, p.group_m, p.n_fastest, bm, bn2);
    const int bn = bn2 * 2 + h;
    float2 acc[64];
#pragma unroll
    for (int i = 0; i < 64; ++i) acc[i] = make_float2(0.0f, 0.0f);
    for (int pg = 0; pg < p.KB; pg += kPage, ++pc) {
      const ScalePage& sp = pages[pc & 1];
      if (pg > 0) mbar_wait_sleep(sfull + (pc & 1), (pc >> 1) & 1);
      const int nk = min(kPage, p.KB - pg);
      for (int j = 0; j < nk; ++j) {
        const bool masked = sp.flag[j];
        for (int r = 0; r < (masked ? 2 : 1); ++r) {
          const uint32_t slot = item & 1;
          const float s = r ? sp.res[h][j] : sp.prim[h][j];
          // TMEM base re-read from shared memory (issued before the wait, so
          // its latency hides behind it) instead of living in a register
          // across the whole kernel (it was spilled to local memory)
          const uint32_t tbase = ld_shared_u32(tmem_holder);
          if constexpr (kProf) t0 = (uint32_t)clock();
          mbar_wait_sleep(tfull + slot, (item >> 1) & 1);
          tc_fence_after();
          if constexpr (kProf) t1 = (uint32_t)clock();
          const uint32_t tb = tbase + lane_addr + slot * 256 + h * 128;
          if constexpr (kEpi == kEpiDump) {
            int32_t* d = p.dump + (r ? p.dump_res_offset : 0) +
                         ((((int64_t)bm * p.NB + bn) * p.KB + pg + j) * kBM + row_in_tile) * 128;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              uint32_t v[32];
              tmem_ld32(tb + c * 32, v);
              tmem_ld_wait();
              if (bn < p.NB) {
#pragma unroll
                for (int i = 0; i < 32; i += 4)
                  *reinterpret_cast<int4*>(d + c * 32 + i) =
                      make_int4((int)v[i], (int)v[i + 1], (int)v[i + 2], (int)v[i + 3]);
              }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(tempty + slot);
          } else {
            if (kDiag && (p.diag & 1)) {  // diagnostic: release the slot without epilogue math
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(tempty + slot);
              ++item;
              continue;
            }
            // Two 32-column loads in flight; the slot is released right after
            // the last load lands (two consumes in between), the remaining math
            // overlaps the next item's MMA.  The release latency is what paces
            // the tensor pipe with only two TMEM slots.
            uint32_t va[32], vb[32];
            tmem_ld32(tb + 0, va);
            tmem_ld32(tb + 32, vb);
            tmem_ld_wait();
            if constexpr (kProf) t2 = (uint32_t)clock();
            consume<kEpi>(va, acc + 0, s, p.one);
            tmem_ld32(tb + 64, va);
            consume<kEpi>(vb, acc + 16, s, p.one);
            tmem_ld32(tb + 96, vb);
            tmem_ld_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(tempty + slot);
            if constexpr (kProf) t3 = (uint32_t)clock();
            consume<kEpi>(va, acc + 32, s, p.one);
            consume<kEpi>(vb, acc + 48, s, p.one);
            if constexpr (kProf) {
              // a register dependency on the last FFMA2 makes the clock read wait for it
              const uint32_t t4 = (uint32_t)clock() + (acc[63].y == 12345.0f ? 1u : 0u);
              tw += t1 - t0; tl += t2 - t1; tpre += t3 - t2; tpost += t4 - t3;
            }
          }
          ++item;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(sempty + (pc & 1));
    }
    if (kEpi != kEpiDump && !(kDiag && (p.diag & 4)) && p.tma_store) {
      // Staged TMA stores: the warp's 32 rows x 128 columns go out in 4 KiB
      // boxes (64 bf16 or 32 fp32 columns x 32 rows), written into a 128B-
      // swizzled staging buffer (16-byte chunk j of row r at chunk j ^ (r & 7):
      // conflict-free) and handed to TMA, which clips ragged edges; the warp
      // only waits for the previous box to be READ from shared memory.  Tile-end
      // stores thus no longer hold back the TMEM drain (direct per-row stores
      // cost ~16 % of the GEMM).  p.tma_store == 2: fp32 reduce-add (accumulate).
      const int64_t row0 = (int64_t)bm * kBM + q * 32;
      if (bn < p.NB && row0 < p.M) {
        const int cols_per_box = p.out_bf16 ? 64 : 32;
        const int nbox = 128 / cols_per_box;
        uint8_t* rowp = obuf + lane * 128;
        for (int c = 0; c < nbox; ++c) {
          if (p.tma_store != 3 && lane == 0) bulk_wait_read0();  // the previous box left the buffer
          __syncwarp();
          if (p.out_bf16) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {  // 8 x 16 B = 64 bf16 of this lane's row
              const float2* a = acc + c * 32 + j * 4;
              uint4 w;
              __nv_bfloat162 b0 = __float22bfloat162_rn(a[0]), b1 = __float22bfloat162_rn(a[1]);
              __nv_bfloat162 b2 = __float22bfloat162_rn(a[2]), b3 = __float22bfloat162_rn(a[3]);
              w.x = *reinterpret_cast<uint32_t*>(&b0);
              w.y = *reinterpret_cast<uint32_t*>(&b1);
              w.z = *reinterpret_cast<uint32_t*>(&b2);
              w.w = *reinterpret_cast<uint32_t*>(&b3);
              *reinterpret_cast<uint4*>(rowp + ((j ^ (lane & 7)) << 4)) = w;
            }
          } else {
#pragma unroll
            for (int j = 0; j < 8; ++j) {  // 8 x 16 B = 32 fp32 of this lane's row
              const float2* a = acc + c * 16 + j * 2;
              *reinterpret_cast<float4*>(rowp + ((j ^ (lane & 7)) << 4)) =
                  make_float4(a[0].x, a[0].y, a[1].x, a[1].y);
            }
          }
          if (p.tma_store == 3) {
            // coalesced copy-out: lane l moves 16-byte chunk (l & 7) of rows
            // 4i + (l >> 3): every STG.128 writes four full 128 B lines
            __syncwarp();
            const int64_t gcol = (int64_t)bn * 128 + c * cols_per_box;
            const int esz = p.out_bf16 ? 2 : 4;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const int r = 4 * i + (lane >> 3), j = lane & 7;
              const uint4 v = *reinterpret_cast<const uint4*>(obuf + r * 128 + ((j ^ (r & 7)) << 4));
              const int64_t grow = row0 + r;
              const int64_t col = gcol + j * (16 / esz);
              if (grow < p.M && col < p.N)
                *reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(p.out) + (grow * p.ldo + col) * esz) = v;
            }
            __syncwarp();
          } else {
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              const int c0 = bn * 128 + c * cols_per_box;
              // the output streams past the L2-resident operand: evict_first
              // (diag 1 << 24: default policy)
              if (kDiag && (p.diag & (1 << 24))) {
                if (p.tma_store == 2) tma_reduce_add_2d(map_o, obuf, c0, (int)row0);
                else tma_store_2d(map_o, obuf, c0, (int)row0);
              } else {
                const uint64_t pol_o = l2_policy_evict_first();
                if (p.tma_store == 2) tma_reduce_add_2d_hint(map_o, obuf, c0, (int)row0, pol_o);
                else tma_store_2d_hint(map_o, obuf, c0, (int)row0, pol_o);
              }
              bulk_commit();
            }
          }
        }
      }
    } else if (kEpi != kEpiDump && !(kDiag && (p.diag & 4))) {
      const int64_t grow = (int64_t)bm * kBM + row_in_tile;
      const int64_t gcol0 = (int64_t)bn * 128;
      if (bn < p.NB && grow < p.M) {
        const bool full_row = p.vec_store && gcol0 + 128 <= p.N;
        if (p.out_bf16) {
          __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(p.out) + grow * p.ldo + gcol0;
          if (full_row) {
#pragma unroll
            for (int i = 0; i < 64; i += 4) {
              uint4 w;
              uint32_t* wp = reinterpret_cast<uint32_t*>(&w);
              uint4 old = make_uint4(0, 0, 0, 0);
              if (p.accumulate) old = *reinterpret_cast<const uint4*>(o + 2 * i);
              const __nv_bfloat162* op = reinterpret_cast<const __nv_bfloat162*>(&old);
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                float2 v = acc[i + e];
                if (p.accumulate) {
                  const float2 ov = __bfloat1622float2(op[e]);
                  v = make_float2(__fadd_rn(ov.x, v.x), __fadd_rn(ov.y, v.y));
                }
                __nv_bfloat162 b = __float22bfloat162_rn(v);
                wp[e] = *reinterpret_cast<uint32_t*>(&b);
              }
              *reinterpret_cast<uint4*>(o + 2 * i) = w;
            }
          } else {
#pragma unroll
            for (int i = 0; i < 64; ++i) {
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                const int64_t col = gcol0 + 2 * i + e;
                if (col < p.N) {
                  float v = e ? acc[i].y : acc[i].x;
                  if (p.accumulate) v = __fadd_rn(__bfloat162float(o[2 * i + e]), v);
                  o[2 * i + e] = __float2bfloat16_rn(v);
                }
              }
            }
          }
        } else {
          float* o = reinterpret_cast<float*>(p.out) + grow * p.ldo + gcol0;
          if (full_row) {
#pragma unroll
            for (int i = 0; i < 64; i += 2) {
              float4 v = make_float4(acc[i].x, acc[i].y, acc[i + 1].x, acc[i + 1].y);
              if (p.accumulate) {
                const float4 old = *reinterpret_cast<const float4*>(o + 2 * i);
                v.x = __fadd_rn(old.x, v.x);
                v.y = __fadd_rn(old.y, v.y);
                v.z = __fadd_rn(old.z, v.z);
                v.w = __fadd_rn(old.w, v.w);
              }
              *reinterpret_cast<float4*>(o + 2 * i) = v;
            }
          } else {
#pragma unroll
            for (int i = 0; i < 64; ++i) {
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                const int64_t col = gcol0 + 2 * i + e;
                if (col < p.N) {
                  const float v = e ? acc[i].y : acc[i].x;
                  o[2 * i + e] = p.accumulate ? __fadd_rn(o[2 * i + e], v) : v;
                }
              }
            }
          }
        }
      }
    }
  }
  if (p.tma_store && lane == 0) bulk_wait0();  // this warp's stores are complete
  if constexpr (kProf) {
    if (q == 0 && lane == 0) {
      long long* o = p.prof + blockIdx.x * 16 + 1 + h * 4;
      o[0] = tw; o[1] = tl; o[2] = tpre; o[3] = tpost;
      if (h == 0) p.prof[blockIdx.x * 16 + 9] = item;
    }
  }
}

// kDiag: the diagnostic instantiation (performance experiments through
// fbq_debug_set_gemm_diag); the production instances compile those branches out
// of the issue loops.
template <int kEpi, bool kDiag = false>
__global__ void __launch_bounds__(kThreads, 1)
fbq_gemm_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_r,
                const __grid_constant__ CUtensorMap map_b, const __grid_constant__ CUtensorMap map_o,
                const GemmParams p) {
  // The 128B-swizzle atoms need 1 KiB alignment: dynamic shared memory starts
  // 1 KiB-aligned on sm_100 (after the 1 KiB reserved per CTA), which the kernel
  // checks (trap) instead of re-deriving an aligned base -- the runtime
  // arithmetic was rematerialised in every epilogue item under register pressure.
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  if (smem_u32(smem_raw) & 1023u) __trap();
  uint8_t* smem = smem_raw;
  uint8_t* ostage = smem + kStages * kStageBytes;  // [kEpiWarps][kOutChunk], 1 KiB aligned
  ScalePage* pages = reinterpret_cast<ScalePage*>(ostage + kEpiWarps * kOutChunk);
  uint64_t* bars = reinterpret_cast<uint64_t*>(pages + 2);
  uint64_t* full = bars;                 // [kStages]
  uint64_t* empty = bars + kStages;      // [kStages]
  uint64_t* tfull = bars + 2 * kStages;  // [2]
  uint64_t* tempty = tfull + 2;          // [2]
  uint64_t* sfull = tempty + 2;          // [2]
  uint64_t* sempty = sfull + 2;          // [2]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(sempty + 2);

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
      mbar_init(sfull + s, 32);
      mbar_init(sempty + s, kEpiWarps);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<kTmemCols>(tmem_holder);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  // scale-grid indices of the stored operands (row stride lds_a / lds_b)
  auto a_blk = [&](int bm, int bk) -> int64_t {
    return p.a_major == 0 ? (int64_t)bm * p.lds_a + bk : (int64_t)bk * p.lds_a + bm;
  };
  auto b_blk = [&](int bk, int bn) -> int64_t {
    return p.b_major == 0 ? (int64_t)bn * p.lds_b + bk : (int64_t)bk * p.lds_b + bn;
  };

  // Register budget.  setmaxnreg only redistributes the CTA's launch-time
  // pool (168 regs x 12 warps = 2016 warp-registers); asking for all of it
  // (8 x 232 for the epilogue) blocked setmaxnreg.inc forever on the B200, so
  // the budget keeps slack: 40 + 56 + 40 + 24 + 8 x 224 = 1952.
  static_assert(40 + 56 + 40 + 24 + kEpiWarps * 224 <= 168 * (kThreads / 32), "register pool");
  if (warp == 0) setmaxnreg_dec<40>();
  else if (warp == 1) setmaxnreg_dec<56>();
  else if (warp == 2) setmaxnreg_dec<40>();
  else if (warp == 3) setmaxnreg_dec<24>();

  if (warp == 0) {
    // ===================== TMA producer =====================
    // The whole warp walks the schedule (waits included) and lane 0 issues: a
    // warp whose lanes 1-31 sit in the final __syncthreads while lane 0 loops
    // is diverged, and the divergent path steals the issuing lane's slots.
    {
      if (lane == 0) {
        tma_prefetch(&map_a);
        tma_prefetch(&map_b);
        if (has_res) tma_prefetch(&map_r);
      }
      // L2 policy per operand: with a resident-operand raster the streamed
      // operand is read by the ~148 concurrent tiles within a short window and
      // then dead, so it is marked evict-first (diag 1 << 23: all evict-last)
      const uint64_t pol_keep = l2_policy_evict_last();
      const bool split_pol = !(kDiag && (p.diag & (1 << 23)));
      const uint64_t pol_a = (split_pol && p.n_fastest) ? l2_policy_evict_first() : pol_keep;
      // B streams (evict_first) whenever A is the resident operand: all
      // block-rows (A pinned) or row-groups larger than the default
      const uint64_t pol_b = (split_pol && !p.n_fastest && p.group_m > kGroupM) ? l2_policy_evict_first()
                                                                                : pol_keep;
      int stage = 0;
      uint32_t phase = 0, pc = 0;
      for (;;) {
        mbar_wait_sleep(sfull + (pc & 1), (pc >> 1) & 1);
        const int tile = pages[pc & 1].tile;
        if (tile < 0) break;
        int bm, bn2;
        tile_coords(tile, p.MB, NT, p.group_m, p.n_fastest, bm, bn2);
        for (int pg = 0; pg < p.KB; pg += kPage, ++pc) {
          const ScalePage& sp = pages[pc & 1];
          if (pg > 0) mbar_wait_sleep(sfull + (pc & 1), (pc >> 1) & 1);
          const int nk = min(kPage, p.KB - pg);
          for (int j = 0; j < nk; ++j) {
            const int bk = pg + j;
            const bool masked = sp.flag[j];
            mbar_wait_sleep(empty + stage, phase ^ 1);
            uint8_t* sa = smem + stage * kStageBytes;
            uint8_t* sr = sa + kTileA;
            uint8_t* sb = sa + 2 * kTileA;
            if (lane == 0) {
              if (kDiag && (p.diag & 2)) {  // diagnostic: no operand traffic
                mbar_arrive(full + stage);
              } else {
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
              }
            }
            __syncwarp();
            if (++stage == kStages) { stage = 0; phase ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (whole warp walks, lane 0 issues) =====================
    {
      // one M=128 N=256 MMA per 32-deep k step (N=128 instructions run the
      // tensor pipe at ~55-70%, profiles/microbench/r01_mma_raw.txt)
      const uint32_t idesc = idesc_i8(kBM, kBN, p.a_major, p.b_major);
      // Descriptor templates: per stage only the 14-bit start address changes,
      // per 32-deep k step the address advances by 32 B (K-major: inside the
      // 128 B swizzle row) or 4 KiB (MN-major: 32 k-rows of 128 B).
      const uint32_t a_step = p.a_major == 0 ? (32 >> 4) : (4096 >> 4);
      const uint32_t b_step = p.b_major == 0 ? (32 >> 4) : (4096 >> 4);
      const uint64_t a_tmpl = smem_desc_sw128(0, 16, 1024);
      const uint64_t b_tmpl = smem_desc_sw128(0, p.b_major == 0 ? 16 : kTileA, 1024);
      const uint32_t smem0 = smem_u32(smem);
      const uint32_t tmem_base = ld_shared_u32(tmem_holder);
      int stage = 0;
      uint32_t phase = 0, item = 0, pc = 0;
      const long long t_start = p.prof ? clock64() : 0;
      // diag 512 (bare MMA loop, no scale pages): the static tile schedule
      for (int tile = blockIdx.x;; tile += gridDim.x) {
        if (kDiag && (p.diag & 512)) {
          if (tile >= p.num_tiles) break;
        } else {
          mbar_wait_sleep(sfull + (pc & 1), (pc >> 1) & 1);
          if (pages[pc & 1].tile < 0) break;
        }
        for (int pg = 0; pg < p.KB; pg += kPage, ++pc) {
          const ScalePage& sp = pages[pc & 1];
          if (!(kDiag && (p.diag & 512)) && pg > 0) mbar_wait_sleep(sfull + (pc & 1), (pc >> 1) & 1);
          const int nk = min(kPage, p.KB - pg);
          for (int j = 0; j < nk; ++j) {
            const int n_items = (!(kDiag && (p.diag & 512)) && sp.flag[j]) ? 2 : 1;
            if (!(kDiag && (p.diag & 16))) mbar_wait_sleep(full + stage, phase);
            if (!(kDiag && (p.diag & 64))) tc_fence_after();
            const uint32_t sa = smem0 + stage * kStageBytes;
            const uint64_t bd0 = b_tmpl | ((sa + 2 * kTileA) >> 4);
            for (int r = 0; r < n_items; ++r) {
              const uint32_t slot = item & 1;
              if (!(kDiag && (p.diag & 8))) mbar_wait_sleep(tempty + slot, ((item >> 1) & 1) ^ 1);
              if (!(kDiag && (p.diag & 64))) tc_fence_after();
              const uint64_t ad0 = a_tmpl | ((sa + (r ? kTileA : 0)) >> 4);
              const uint32_t d = tmem_base + slot * 256;
              if (lane == 0) {
#pragma unroll
                for (int kk = 0; kk < kBK / 32; ++kk)
                  mma_i8(d, ad0 + kk * a_step, bd0 + kk * b_step, idesc, kk > 0 ? 1u : 0u);
                mma_commit(tfull + slot);
              }
              __syncwarp();
              ++item;
            }
            if (!(kDiag && (p.diag & 128)) && lane == 0) mma_commit(empty + stage);
            __syncwarp();
            if (++stage == kStages) { stage = 0; phase ^= 1; }
          }
        }
      }
      if (p.prof && lane == 0) p.prof[blockIdx.x * 16] = clock64() - t_start;  // MMA-warp cycles per CTA
    }
  } else if (warp == 2) {
    // ===================== scale loader =====================
    // The tile scheduler: the first tile is blockIdx.x, every further one is
    // claimed from the launch's counter (p.tile_ctr, zeroed in-stream before
    // the launch) -- CTAs that drew cheap tiles (few fallback blocks) take
    // more, so the last wave is balanced; without a counter the static
    // schedule tile += gridDim.x.  Each tile's pages carry its index to the
    // other roles; a page with tile = -1 tells them to exit.
    uint32_t pc = 0;
    int tile = (kDiag && (p.diag & 512)) ? p.num_tiles : blockIdx.x;
    for (;;) {
      if (tile >= p.num_tiles) {
        ScalePage& sp = pages[pc & 1];
        mbar_wait_sleep(sempty + (pc & 1), ((pc >> 1) & 1) ^ 1);
        if (lane == 0) sp.tile = -1;
        __syncwarp();
        mbar_arrive(sfull + (pc & 1));
        break;
      }
      int bm, bn2;
      tile_coords(tile, p.MB, NT, p.group_m, p.n_fastest, bm, bn2);
      const int bn0 = 2 * bn2, bn1 = 2 * bn2 + 1;
      for (int pg = 0; pg < p.KB; pg += kPage, ++pc) {
        ScalePage& sp = pages[pc & 1];
        mbar_wait_sleep(sempty + (pc & 1), ((pc >> 1) & 1) ^ 1);
        if (lane == 0) {
          sp.tile = tile;
          sp.pg = pg;
        }
        const int nk = min(kPage, p.KB - pg);
        for (int j = lane; j < nk; j += 32) {
          const int bk = pg + j;
          const int64_t ab = a_blk(bm, bk);
          const bool masked = has_res && mask_bit(p.mask_bits, ab);
          float sa = 0.f, ra = 0.f, sb0 = 0.f, sb1 = 0.f;
          if (p.a_scales) {
            sa = p.a_scales[ab];
            ra = masked ? p.res_scales[ab] : 0.0f;
            sb0 = p.b_scales[b_blk(bk, bn0)];
            sb1 = bn1 < p.NB ? p.b_scales[b_blk(bk, bn1)] : 0.0f;
          }
          sp.prim[0][j] = __fmul_rn(sa, sb0);  // gemm.cpp:163
          sp.prim[1][j] = __fmul_rn(sa, sb1);
          sp.res[0][j] = __fmul_rn(ra, sb0);   // gemm.cpp:172
          sp.res[1][j] = __fmul_rn(ra, sb1);
          sp.flag[j] = masked ? 1 : 0;
        }
        __syncwarp();
        mbar_arrive(sfull + (pc & 1));
      }
      int next = 0;
      if (lane == 0) {
        if (p.tile_ctr) {
          next = atomicAdd(p.tile_ctr, 1) + (int)gridDim.x;
          // Each CTA's last claim is the one past the end; once all gridDim.x
          // of those are in, nobody reads the counter again: the last CTA
          // resets it (and the arrival count) for the slot's next launch.
          if (next >= p.num_tiles && atomicAdd(p.tile_ctr + 1, 1) == (int)gridDim.x - 1) {
            atomicExch(p.tile_ctr, 0);
            atomicExch(p.tile_ctr + 1, 0);
          }
        } else {
          next = tile + (int)gridDim.x;
        }
      }
      tile = __shfl_sync(0xffffffffu, next, 0);
    }
  } else if (warp >= 4) {
    // ===================== epilogue =====================
    setmaxnreg_inc<224>();
    if (p.prof) {
      if (warp >= 8) epilogue_role<kEpi, 1, true, kDiag>(p, &map_o, ostage + (warp - 4) * kOutChunk, pages, tfull, tempty, sfull, sempty, tmem_holder, warp, lane, NT);
      else epilogue_role<kEpi, 0, true, kDiag>(p, &map_o, ostage + (warp - 4) * kOutChunk, pages, tfull, tempty, sfull, sempty, tmem_holder, warp, lane, NT);
    } else {
      if (warp >= 8) epilogue_role<kEpi, 1, false, kDiag>(p, &map_o, ostage + (warp - 4) * kOutChunk, pages, tfull, tempty, sfull, sempty, tmem_holder, warp, lane, NT);
      else epilogue_role<kEpi, 0, false, kDiag>(p, &map_o, ostage + (warp - 4) * kOutChunk, pages, tfull, tempty, sfull, sempty, tmem_holder, warp, lane, NT);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<kTmemCols>(ld_shared_u32(tmem_holder));
}

// ----------------------------------------------------------------- host side
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                    const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encode() {
  static const PFN_encodeTiled fn = [] {  // thread-safe one-time lookup
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return reinterpret_cast<PFN_encodeTiled>(ptr);
    return (PFN_encodeTiled) nullptr;
  }();
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

// ---- per-device state (thread-safe; set up by gemm_init, never in a launch) ----
constexpr int kMaxDevices = 64;
// Dynamic tile counters: a ring of 128-byte slots per device, zeroed once at
// gemm_init.  Every launch takes the next slot with an atomic fetch_add and
// leaves it at zero again (the last CTA to make its final claim resets it),
// so no memset node per launch and no allocation or synchronisation on the
// launch path (safe under stream capture: a captured launch keeps its slot,
// which every replay leaves reset).  kSlots concurrent launches per device
// may be in flight before a slot is reused.
constexpr int kCounterSlots = 4096;
static std::atomic<int*> g_ring[kMaxDevices];
static std::atomic<unsigned> g_next_slot[kMaxDevices];
static std::once_flag g_init_once[kMaxDevices];
static cudaError_t g_init_err[kMaxDevices] = {};
static std::atomic<int> g_num_sms[kMaxDevices];

static int current_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return -1;
  return dev;
}

// kernel attributes + SM count, once per device (no allocation, no sync: may
// run on the launch path)
static std::once_flag g_attr_once[kMaxDevices];
static cudaError_t g_attr_err[kMaxDevices] = {};
static cudaError_t gemm_attributes(int dev) {
  std::call_once(g_attr_once[dev], [dev] {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    g_num_sms[dev].store(n > 0 ? n : 148);
    for (cudaError_t e : {cudaFuncSetAttribute(fbq_gemm_kernel<kEpiExact>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes),
                          cudaFuncSetAttribute(fbq_gemm_kernel<kEpiFma>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes),
                          cudaFuncSetAttribute(fbq_gemm_kernel<kEpiDump>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes),
                          cudaFuncSetAttribute(fbq_gemm_kernel<kEpiExact, true>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes),
                          cudaFuncSetAttribute(fbq_gemm_kernel<kEpiFma, true>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes)})
      if (e != cudaSuccess && g_attr_err[dev] == cudaSuccess) g_attr_err[dev] = e;
  });
  return g_attr_err[dev];
}

cudaError_t gemm_init() {
  const int dev = current_device();
  if (dev < 0) return cudaErrorInvalidDevice;
  if (cudaError_t e = gemm_attributes(dev)) return e;
  std::call_once(g_init_once[dev], [dev] {
    int* r = nullptr;
    cudaError_t e = cudaMalloc(&r, (size_t)kCounterSlots * 128);
    if (e == cudaSuccess) e = cudaMemset(r, 0, (size_t)kCounterSlots * 128);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      if (r) cudaFree(r);
      g_init_err[dev] = e;
      return;
    }
    g_ring[dev].store(r, std::memory_order_release);
  });
  return g_init_err[dev];
}

static bool gemm_ready(int dev) { return dev >= 0 && g_ring[dev].load(std::memory_order_acquire) != nullptr; }

int* counter_slot() {
  const int dev = current_device();
  if (!gemm_ready(dev)) return nullptr;
  const unsigned slot = g_next_slot[dev].fetch_add(1, std::memory_order_relaxed) % kCounterSlots;
  return g_ring[dev].load(std::memory_order_acquire) + (size_t)slot * 32;
}

int gemm_num_sms() {
  const int dev = current_device();
  const int n = dev >= 0 ? g_num_sms[dev].load() : 0;
  return n > 0 ? n : 148;
}

template <int kEpi>
static cudaError_t launch_typed(const CUtensorMap& ma, const CUtensorMap& mr,
                                const CUtensorMap& mb, const CUtensorMap& mo, const GemmParams& p,
                                int grid, cudaStream_t s) {
  // kernel-side diagnostic bits run the diagnostic instantiation (kDiag)
  constexpr int kKernelDiag = 1 | 2 | 4 | 8 | 16 | 64 | 128 | 512 | (1 << 23) | (1 << 24);
  if (kEpi != kEpiDump && (p.diag & kKernelDiag))
    fbq_gemm_kernel<kEpi, kEpi != kEpiDump><<<grid, kThreads, kSmemBytes, s>>>(ma, mr, mb, mo, p);
  else
    fbq_gemm_kernel<kEpi><<<grid, kThreads, kSmemBytes, s>>>(ma, mr, mb, mo, p);
  return cudaGetLastError();
}

cudaError_t launch_gemm(const GemmOperands& o, GemmParams p, int epi, cudaStream_t s) {
  const int dev = current_device();
  if (dev < 0) return cudaErrorInvalidDevice;
  if (cudaError_t e = gemm_attributes(dev)) return e;
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

  // output tensor map for the staged TMA stores: 4 KiB boxes of 32 rows x 128 B,
  // 128B swizzle (the staging layout); fp32 accumulate uses the reduce-add form
  CUtensorMap mo = ma;
  p.tma_store = 0;
  if (epi != kEpiDump && p.out && p.vec_store && !(p.accumulate && p.out_bf16) && !(p.diag & 8192) &&
      p.M < (1ll << 31) && p.N < (1ll << 31)) {
    PFN_encodeTiled enc = get_encode();
    const size_t esz = p.out_bf16 ? 2 : 4;
    cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)M};
    cuuint64_t strides[1] = {(cuuint64_t)(p.ldo * esz)};
    cuuint32_t box[2] = {(cuuint32_t)(128 / esz), 32};
    cuuint32_t estr[2] = {1, 1};
    if (enc && enc(&mo, p.out_bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                   2, p.out, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS)
      p.tma_store = p.accumulate ? 2 : ((p.diag & 16384) ? 3 : 1);
  }
  p.num_tiles = p.MB * ((p.NB + 1) / 2);
  // dynamic tile counter: the next slot of the device's ring (see gemm_init);
  // before fbq_cuda_init() ran on this device, the static tile schedule
  p.tile_ctr = nullptr;
  if (gemm_ready(dev) && !(p.diag & (1 << 21)) && !(p.diag & 512)) {  // diag 1 << 21: static schedule
    const unsigned slot = g_next_slot[dev].fetch_add(1, std::memory_order_relaxed) % kCounterSlots;
    p.tile_ctr = g_ring[dev].load(std::memory_order_acquire) + (size_t)slot * 32;  // one 128 B line per slot
  }
  {
    // Raster (DRAM traffic; scripts/gemm_traffic_probe.py,
    // scripts/gemm_raster_policy.py).  Measured per launch, bf16 out, 10 % fallback:
    // * the smaller operand fits the L2's effective evict_last capacity (<= 56
    //   MB) and the other does not: pin it (bm over all block-rows keeps A
    //   resident, bn fastest keeps B) and stream the other once -- gate/up
    //   forward 0.22 GB read (0.98 GB with groups of 8), down forward 0.36 GB (0.60);
    // * A moderately large (<= 112 MB) and B larger: row-groups of A sized to ~40
    //   MB, B streamed evict_first once per group -- C5 0.98 GB (2.0 GB with groups
    //   of 8; pinning all 64 MB of A read 3.4 GB: evict_last does not hold it);
    // * both operands small: bn fastest (C1 4096^3 +4..15 % over groups of 8);
    // * else groups of kGroupM block-rows with the default policy (the dX GEMM:
    //   1.5 GB; larger groups with B evict_first read 2.4 GB -- B panels are
    //   re-read by CTAs that are not in lock-step).
    // Speed is within +-4 % across rasters on the large shapes.
    constexpr double kPin = 56.0 * (1 << 20), kPinMax = 112.0 * (1 << 20), kGroupBytes = 40.0 * (1 << 20);
    const double a_bytes = (double)p.M * (double)p.K, b_bytes = (double)p.N * (double)p.K;
    p.group_m = kGroupM;
    p.n_fastest = 0;
    const int NTt = (p.NB + 1) / 2;
    if (p.diag & (1 << 19)) p.group_m = p.MB;          // diagnostics/tests: force each raster
    else if (p.diag & (1 << 20)) p.n_fastest = NTt;
    else if (p.diag & (1 << 17)) p.n_fastest = (NTt + 2) / 3;  // tests: B in chunks of ~NT/3
    else if (!(p.diag & (1 << 18))) {  // diagnostics: 1 << 18 = always kGroupM groups
      const double small = a_bytes < b_bytes ? a_bytes : b_bytes;
      const double large = a_bytes < b_bytes ? b_bytes : a_bytes;
      const double b_panel = 256.0 * (double)p.K;  // bytes of one 256-wide B n-tile over K
      if (small <= kPin && large > kPin) {
        if (a_bytes <= b_bytes) p.group_m = p.MB;
        else p.n_fastest = NTt;
      } else if (large <= kPin) {
        p.n_fastest = NTt;
      } else if (a_bytes <= kPinMax && b_bytes > a_bytes) {
        const int g = (int)(kGroupBytes / (128.0 * (double)p.K));
        p.group_m = g < kGroupM ? kGroupM : (g > p.MB ? p.MB : g);
      } else if (b_bytes <= a_bytes && b_panel <= kPin && !(p.diag & (1 << 27))) {
        // both operands too large to pin, B the smaller: B in equal chunks that
        // fit the pin capacity, each chunk's every tile (bn fastest) before the
        // next, so A streams once per chunk and each B chunk once (dX =
        // dG W_gu: A 235 MB, B 117 MB -> two 58 MB chunks; diag 1 << 27: groups)
        const int nmax = (int)(kPin / b_panel);
        const int nchunks = (NTt + nmax - 1) / nmax;
        p.n_fastest = (NTt + nchunks - 1) / nchunks;
      }
    }
  }
  const int grid = p.num_tiles < gemm_num_sms() ? p.num_tiles : gemm_num_sms();
  switch (epi) {
    case kEpiExact: return launch_typed<kEpiExact>(ma, mr, mb, mo, p, grid, s);
    case kEpiFma: return launch_typed<kEpiFma>(ma, mr, mb, mo, p, grid, s);
    default: return launch_typed<kEpiDump>(ma, mr, mb, mo, p, grid, s);
  }
}

}  // namespace fbq
