// Microbenchmark (round 2): operand ingress (TMA, L2-resident int8 operands) + int8
// MMA + TMEM-slot handshake, as in K3, for
//   kCta=1: M=128 N=256 per CTA, stage = A 16 KiB + B 32 KiB
//   kCta=2: CTA pair M=256 N=256, stage per CTA = A 16 KiB + half of B 16 KiB
// Epilogue kEpi: 0 = tcgen05.ld the warp's 128 columns then release (no math);
//                1 = chunk-pipelined I2F + FFMA2 math (the K3 FMA epilogue).
//                2 = as 1, but the slot is prefilled by the epilogue (tcgen05.st) with
//                    0x4B400000 in the warp's last 32 columns and 0 elsewhere, the MMA
//                    always accumulates, and the biased chunk decodes as FADD2 (FMA pipe).
//                3 = 16 epilogue warps (4 per SMSP), warp (q, c) owns 32 lanes x 64 columns:
//                    acc 64 registers, x16 loads double-buffered, setmaxnreg 112.
//                4 = 8 warps, chunk-pipelined: ld(g+1); math(g); wait -- slot released once
//                    its last chunk landed, the next item's first chunk loaded before the
//                    last math of this one.
//                5 = as 1, plus a 5th K=32 u8 x u8 MMA per item (A tile all 255, B rows 96-127
//                    and 224-255 all 255, others 0): those columns get +2080800, i.e. P + bias
//                    is a non-negative denormal; chunk 3 of every warp decodes on the FMA pipe
//                    as fma(d, 2^126, -bias*2^-23) = P*2^-23 exactly (no I2F).
// Reports % of 8192 MAC/clk/SM and TOPS.  A: M x K, B: N x K (both K-major).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2503_08040_b200/csrc \
//        -o scripts/mb_ingress scripts/microbench_ingress.cu
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>

#include "sm100.cuh"

using namespace fbq::sm100;

constexpr int kM = 8192, kN = 8192, kK = 4096;  // 32 + 32 MiB of codes: L2-resident

__device__ __forceinline__ void ld32p(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
        "=r"(r[31])
      : "r"(taddr));
}

__device__ __forceinline__ void consume32(const uint32_t* v, float2* acc, float s) {
  const float2 s2 = make_float2(s, s);
#pragma unroll
  for (int i = 0; i < 16; ++i)
    acc[i] = __ffma2_rn(make_float2(__int2float_rn((int)v[2 * i]), __int2float_rn((int)v[2 * i + 1])), s2, acc[i]);
}

__device__ __forceinline__ void consume32_biased(const uint32_t* v, float2* acc, float s) {
  const float2 s2 = make_float2(s, s);
  const float2 m2 = make_float2(-12582912.0f, -12582912.0f);
#pragma unroll
  for (int i = 0; i < 16; ++i)
    acc[i] = __ffma2_rn(__fadd2_rn(make_float2(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1])), m2), s2, acc[i]);
}

__device__ __forceinline__ void consume32_denorm(const uint32_t* v, float2* acc, float s) {
  const float2 s2 = make_float2(s * 8388608.0f, s * 8388608.0f);  // s * 2^23
  const float2 k2 = make_float2(8.507059173023462e37f, 8.507059173023462e37f);  // 2^126
  const float2 c2 = make_float2(-2080800.0f / 8388608.0f, -2080800.0f / 8388608.0f);
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const float2 y = __ffma2_rn(make_float2(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1])), k2, c2);
    acc[i] = __ffma2_rn(y, s2, acc[i]);
  }
}

// offset-binary operands (u8 x u8): P' = P + bias >= 0 is a denormal; one FFMA removes the
// uniform bias exactly (t = P' 2^-149 * s 2^149 - s 2^21, single rounding), one FADD accumulates
__device__ __forceinline__ void consume32_offset(const uint32_t* v, float2* acc, float s) {
  const float2 s2 = make_float2(s * 0x1p126f * 0x1p23f, s * 0x1p126f * 0x1p23f);
  const float2 b2 = make_float2(-s * 2097152.0f, -s * 2097152.0f);
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const float2 t = __ffma2_rn(make_float2(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1])), s2, b2);
    acc[i] = __fadd2_rn(acc[i], t);
  }
}
// upper bound: one FFMA2 per pair on the raw words (no conversion, no bias removal)
__device__ __forceinline__ void consume32_raw(const uint32_t* v, float2* acc, float s) {
  const float2 s2 = make_float2(s, s);
#pragma unroll
  for (int i = 0; i < 16; ++i)
    acc[i] = __ffma2_rn(make_float2(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1])), s2, acc[i]);
}

template <bool kOff>
__device__ __forceinline__ void consume_sel(const uint32_t* v, float2* acc, float s) {
  if constexpr (kOff) consume32_offset(v, acc, s);
  else consume32(v, acc, s);
}

__device__ __forceinline__ void st8(uint32_t taddr, uint32_t v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(taddr), "r"(v)
               : "memory");
}
// prefill the warp's 128 columns of a slot: 96 zero, 32 magic bias
__device__ __forceinline__ void prefill(uint32_t tb, uint32_t zero, uint32_t bias) {
#pragma unroll
  for (int c = 0; c < 12; ++c) st8(tb + c * 8, zero);
#pragma unroll
  for (int c = 12; c < 16; ++c) st8(tb + c * 8, bias);
}

__device__ __forceinline__ void arrive_any(uint64_t* local, uint32_t remote, bool pair) {
  if (pair) mbar_arrive_cluster(remote);
  else mbar_arrive(local);
}

__device__ __forceinline__ void ld16p(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void consume16(const uint32_t* v, float2* acc, float s) {
  const float2 s2 = make_float2(s, s);
#pragma unroll
  for (int i = 0; i < 8; ++i)
    acc[i] = __ffma2_rn(make_float2(__int2float_rn((int)v[2 * i]), __int2float_rn((int)v[2 * i + 1])), s2, acc[i]);
}

template <int kCta, int kStages, int kEpi>
__global__ void __launch_bounds__(kEpi == 3 ? 640 : 384, 1)
ingress(const __grid_constant__ CUtensorMap ma, const __grid_constant__ CUtensorMap mb, long long* cycles,
        float* sink) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  constexpr int kA = 16384, kB = kCta == 2 ? 16384 : 32768, kStage = kA + kB;
  __shared__ uint64_t full[kStages], empty[kStages], tfull[2], tempty[2];
  __shared__ uint32_t tmem_holder;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = kCta == 2 ? cluster_ctarank() : 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) { mbar_init(full + s, 1); mbar_init(empty + s, 1); }
    for (int s = 0; s < 2; ++s) { mbar_init(tfull + s, 1); mbar_init(tempty + s, (kEpi == 3 ? 16 : 8) * kCta); }
    fence_barrier_init();
  }
  if (warp == 1) {
    if constexpr (kCta == 2) tmem_alloc2<512>(&tmem_holder);
    else tmem_alloc<512>(&tmem_holder);
  }
  tc_fence_before();
  if constexpr (kCta == 2) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_holder;
  if constexpr (kEpi == 5) {
    // bias tiles: A 128 rows x 128 B of 0xFF, B 256 rows x 128 B (0xFF on rows 96-127, 224-255)
    uint32_t* bt = reinterpret_cast<uint32_t*>(smem + kStages * kStage);
    for (int i = threadIdx.x; i < (16384 + 32768) / 4; i += blockDim.x) {
      const int row = i < 4096 ? -1 : (i - 4096) / 32;
      bt[i] = (row < 0 || (row & 127) >= 96) ? 0xFFFFFFFFu : 0u;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
  }
  const int units = gridDim.x / kCta, unit = blockIdx.x / kCta;
  const int MT = kM / (128 * kCta), NT = kN / 256, KB = kK / 128;
  const int tiles = MT * NT;
  if constexpr (kEpi == 3) {
    if (warp < 4) setmaxnreg_dec<24>();
  } else {
    if (warp < 4) setmaxnreg_dec<40>();
  }
  long long t0 = clock64(), t1 = t0;
  if (warp == 0) {
    // producer (whole warp walks, lane 0 issues)
    const uint64_t pol = l2_policy_evict_last();
    const uint32_t leader_full = kCta == 2 ? mapa_shared(smem_u32(full), 0) : smem_u32(full);
    int stage = 0;
    uint32_t phase = 0;
    for (int t = unit; t < tiles; t += units) {
      const int bm = t % MT, bn = t / MT;
      for (int kb = 0; kb < KB; ++kb) {
        mbar_wait(empty + stage, phase ^ 1);
        if (lane == 0) {
          uint8_t* sa = smem + stage * kStage;
          if (rank == 0) mbar_arrive_expect_tx(full + stage, kStage * kCta);
          const int m0 = bm * 128 * kCta + rank * 128, n0 = bn * 256 + (kCta == 2 ? rank * 128 : 0);
          if constexpr (kCta == 2) {
            tma_load_2d_2sm(sa, &ma, leader_full + stage * 8, kb * 128, m0, pol);
            tma_load_2d_2sm(sa + kA, &mb, leader_full + stage * 8, kb * 128, n0, pol);
          } else {
            tma_load_2d(sa, &ma, full + stage, kb * 128, m0, pol);
            tma_load_2d(sa + kA, &mb, full + stage, kb * 128, n0, pol);
          }
        }
        __syncwarp();
        if (++stage == kStages) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1 && rank == 0) {
    const uint32_t idesc = (kEpi == 6 || kEpi == 7 || kEpi == 8) ? (idesc_i8(128 * kCta, 256, 0, 0) & ~((1u << 7) | (1u << 10)))
                                                    : idesc_i8(128 * kCta, 256, 0, 0);
    int stage = 0;
    uint32_t phase = 0, item = 0;
    t0 = clock64();
    for (int t = unit; t < tiles; t += units) {
      for (int kb = 0; kb < KB; ++kb, ++item) {
        const uint32_t slot = item & 1;
        mbar_wait(full + stage, phase);
        mbar_wait(tempty + slot, ((item >> 1) & 1) ^ 1);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t sa = smem_u32(smem) + stage * kStage, sb = sa + kA;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint64_t ad = smem_desc_sw128(sa + kk * 32, 16, 1024), bd = smem_desc_sw128(sb + kk * 32, 16, 1024);
            const uint32_t accum = kEpi == 2 ? 1u : (kk > 0 ? 1u : 0u);
            if constexpr (kCta == 2) mma2_i8(tmem + slot * 256, ad, bd, idesc, accum);
            else mma_i8(tmem + slot * 256, ad, bd, idesc, accum);
          }
          if constexpr (kEpi == 5 && kCta == 1) {
            const uint32_t ba = smem_u32(smem) + kStages * kStage;
            mma_i8(tmem + slot * 256, smem_desc_sw128(ba, 16, 1024), smem_desc_sw128(ba + 16384, 16, 1024),
                   idesc & ~((1u << 7) | (1u << 10)), 1u);
          }
          if constexpr (kCta == 2) {
            mma2_commit_mc(tfull + slot, 3);
            mma2_commit_mc(empty + stage, 3);
          } else {
            mma_commit(tfull + slot);
            mma_commit(empty + stage);
          }
        }
        __syncwarp();
        if (++stage == kStages) { stage = 0; phase ^= 1; }
      }
    }
    t1 = clock64();
    if (lane == 0) cycles[blockIdx.x] = (t1 - t0) / (item > 0 ? item : 1);
  } else if (kEpi == 3 && warp >= 4) {
    if constexpr (kEpi == 3) {
      setmaxnreg_inc<112>();
      const int q = warp & 3, c = (warp - 4) >> 2;
      const uint32_t lane_base = tmem + ((q * 32) << 16) + c * 64;
      const uint32_t tempty_r = kCta == 2 ? mapa_shared(smem_u32(tempty), 0) : smem_u32(tempty);
      float2 acc[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) acc[i] = make_float2(0.f, 0.f);
      const float s = 1.0f + blockIdx.x * 1e-7f;
      uint32_t item = 0;
      for (int t = unit; t < tiles; t += units) {
        for (int kb = 0; kb < KB; ++kb, ++item) {
          const uint32_t slot = item & 1;
          mbar_wait(tfull + slot, (item >> 1) & 1);
          tc_fence_after();
          const uint32_t tb = lane_base + slot * 256;
          uint32_t r0[16], r1[16];
          ld16p(tb, r0);
          ld16p(tb + 16, r1);
          tmem_ld_wait();
          consume16(r0, acc, s);
          ld16p(tb + 32, r0);
          consume16(r1, acc + 8, s);
          ld16p(tb + 48, r1);
          tmem_ld_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) arrive_any(tempty + slot, tempty_r + slot * 8, kCta == 2);
          consume16(r0, acc + 16, s);
          consume16(r1, acc + 24, s);
        }
      }
      float a = 0.f;
#pragma unroll
      for (int i = 0; i < 32; ++i) a += acc[i].x + acc[i].y;
      if (a == 1234.5f) sink[0] = a;
    }
  } else if ((kEpi == 4 || kEpi == 8) && warp >= 4) {
    if constexpr (kEpi == 4 || kEpi == 8) {
      setmaxnreg_inc<224>();
      const int q = warp & 3, h = (warp - 4) >> 2;
      const uint32_t lane_base = tmem + ((q * 32) << 16) + h * 128;
      const uint32_t tempty_r = kCta == 2 ? mapa_shared(smem_u32(tempty), 0) : smem_u32(tempty);
      float2 acc[64];
#pragma unroll
      for (int i = 0; i < 64; ++i) acc[i] = make_float2(0.f, 0.f);
      const float s = 1.0f + blockIdx.x * 1e-7f;
      const int n_items = ((tiles - unit + units - 1) / units) * KB;
      uint32_t va[32], vb[32];
      if (n_items > 0) {
        mbar_wait(tfull, 0);
        tc_fence_after();
        ld32p(lane_base, va);
        tmem_ld_wait();
      }
      for (int it = 0; it < n_items; ++it) {
        const int slot = it & 1;
        const uint32_t tb = lane_base + slot * 256;
        ld32p(tb + 32, vb);
        consume_sel<kEpi == 8>(va, acc + 0, s);
        tmem_ld_wait();
        ld32p(tb + 64, va);
        consume_sel<kEpi == 8>(vb, acc + 16, s);
        tmem_ld_wait();
        ld32p(tb + 96, vb);
        consume_sel<kEpi == 8>(va, acc + 32, s);
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) arrive_any(tempty + slot, tempty_r + slot * 8, kCta == 2);
        if (it + 1 < n_items) {
          const int ns = (it + 1) & 1;
          mbar_wait(tfull + ns, ((it + 1) >> 1) & 1);
          tc_fence_after();
          ld32p(lane_base + ns * 256, va);
        }
        consume_sel<kEpi == 8>(vb, acc + 48, s);
        tmem_ld_wait();
      }
      float a = 0.f;
#pragma unroll
      for (int i = 0; i < 64; ++i) a += acc[i].x + acc[i].y;
      if (a == 1234.5f) sink[0] = a;
    }
  } else if ((kEpi == 9 || kEpi == 10) && warp >= 4) {
    if constexpr (kEpi == 9 || kEpi == 10) {
      // De-phased warp pair: the two epilogue warps of a sub-partition (same TMEM
      // lane quadrant q, column halves h) alternate -- while one loads two
      // 32-column chunks from TMEM the other converts two, so the TMEM read port
      // and the ALU (I2F) work at the same time instead of both warps loading,
      // then both converting.  The odd warp converts the previous item's last two
      // chunks while the even warp loads.  kEpi 9: a named barrier per phase
      // (bar.sync 1+q, 64 threads); kEpi 10: the same orders without barriers.
      setmaxnreg_inc<224>();
      const int q = warp & 3, h = (warp - 4) >> 2;
      const uint32_t lane_base = tmem + ((q * 32) << 16) + h * 128;
      const uint32_t tempty_r = kCta == 2 ? mapa_shared(smem_u32(tempty), 0) : smem_u32(tempty);
      float2 acc[64];
#pragma unroll
      for (int i = 0; i < 64; ++i) acc[i] = make_float2(0.f, 0.f);
      const float s = 1.0f + blockIdx.x * 1e-7f;
      const int n_items = ((tiles - unit + units - 1) / units) * KB;
      const int bar = 1 + q;
      auto pair_sync = [&]() {
        if constexpr (kEpi == 9) asm volatile("bar.sync %0, 64;" ::"r"(bar) : "memory");
      };
      uint32_t va[32], vb[32];
      for (int it = 0; it < n_items; ++it) {
        const int slot = it & 1;
        const uint32_t tb = lane_base + slot * 256;
        if (h == 0) {
          mbar_wait(tfull + slot, (it >> 1) & 1);
          tc_fence_after();
          ld32p(tb, va);
          ld32p(tb + 32, vb);
          tmem_ld_wait();
          pair_sync();
          consume32(va, acc, s);
          consume32(vb, acc + 16, s);
          pair_sync();
          ld32p(tb + 64, va);
          ld32p(tb + 96, vb);
          tmem_ld_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) arrive_any(tempty + slot, tempty_r + slot * 8, kCta == 2);
          pair_sync();
          consume32(va, acc + 32, s);
          consume32(vb, acc + 48, s);
          pair_sync();
        } else {
          if (it > 0) {
            consume32(va, acc + 32, s);
            consume32(vb, acc + 48, s);
          }
          pair_sync();
          mbar_wait(tfull + slot, (it >> 1) & 1);
          tc_fence_after();
          ld32p(tb, va);
          ld32p(tb + 32, vb);
          tmem_ld_wait();
          pair_sync();
          consume32(va, acc, s);
          consume32(vb, acc + 16, s);
          pair_sync();
          ld32p(tb + 64, va);
          ld32p(tb + 96, vb);
          tmem_ld_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) arrive_any(tempty + slot, tempty_r + slot * 8, kCta == 2);
          pair_sync();
        }
      }
      if (h == 1 && n_items > 0) {
        consume32(va, acc + 32, s);
        consume32(vb, acc + 48, s);
      }
      float a = 0.f;
#pragma unroll
      for (int i = 0; i < 64; ++i) a += acc[i].x + acc[i].y;
      if (a == 1234.5f) sink[0] = a;
    }
  } else if (kEpi != 3 && kEpi != 4 && kEpi != 8 && kEpi != 9 && kEpi != 10 && warp >= 4) {
    setmaxnreg_inc<224>();
    const int q = warp & 3, h = (warp - 4) >> 2;
    const uint32_t lane_base = tmem + ((q * 32) << 16) + h * 128;
    const uint32_t tempty_r = kCta == 2 ? mapa_shared(smem_u32(tempty), 0) : smem_u32(tempty);
    float2 acc[64];
#pragma unroll
    for (int i = 0; i < 64; ++i) acc[i] = make_float2(0.f, 0.f);
    const float s = 1.0f + blockIdx.x * 1e-7f;
    uint32_t item = 0;
    const uint32_t zero = (uint32_t)(s == 0.0f), bias = 0x4B400000u + zero;
    if constexpr (kEpi == 2) {
      // both slots start prefilled; the first MMA waits for the release
      prefill(lane_base, zero, bias);
      prefill(lane_base + 256, zero, bias);
      tmem_st_wait();
    }
    for (int t = unit; t < tiles; t += units) {
      for (int kb = 0; kb < KB; ++kb, ++item) {
        const uint32_t slot = item & 1;
        mbar_wait(tfull + slot, (item >> 1) & 1);
        tc_fence_after();
        const uint32_t tb = lane_base + slot * 256;
        uint32_t va[32], vb[32];
        if constexpr (kEpi == 0) {
          ld32p(tb, va);
          ld32p(tb + 32, vb);
          ld32p(tb + 64, va);
          ld32p(tb + 96, vb);
          tmem_ld_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) arrive_any(tempty + slot, tempty_r + slot * 8, kCta == 2);
          acc[0].x += __uint_as_float(va[0] ^ vb[31]);
        } else if constexpr (kEpi == 2) {
          ld32p(tb, va);
          ld32p(tb + 32, vb);
          tmem_ld_wait();
          consume32(va, acc, s);
          ld32p(tb + 64, va);
          consume32(vb, acc + 16, s);
          ld32p(tb + 96, vb);
          tmem_ld_wait();
          prefill(tb, zero, bias);
          tmem_st_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) arrive_any(tempty + slot, tempty_r + slot * 8, kCta == 2);
          consume32(va, acc + 32, s);
          consume32_biased(vb, acc + 48, s);
        } else {
          ld32p(tb, va);
          ld32p(tb + 32, vb);
          tmem_ld_wait();
          if constexpr (kEpi == 6) consume32_offset(va, acc, s);
          else if constexpr (kEpi == 7) consume32_raw(va, acc, s);
          else consume32(va, acc, s);
          ld32p(tb + 64, va);
          if constexpr (kEpi == 6) consume32_offset(vb, acc + 16, s);
          else if constexpr (kEpi == 7) consume32_raw(vb, acc + 16, s);
          else consume32(vb, acc + 16, s);
          ld32p(tb + 96, vb);
          tmem_ld_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) arrive_any(tempty + slot, tempty_r + slot * 8, kCta == 2);
          if constexpr (kEpi == 6) {
            consume32_offset(va, acc + 32, s);
            consume32_offset(vb, acc + 48, s);
          } else if constexpr (kEpi == 7) {
            consume32_raw(va, acc + 32, s);
            consume32_raw(vb, acc + 48, s);
          } else {
            consume32(va, acc + 32, s);
            if constexpr (kEpi == 5) consume32_denorm(vb, acc + 48, s);
            else consume32(vb, acc + 48, s);
          }
        }
      }
    }
    float a = 0.f;
#pragma unroll
    for (int i = 0; i < 64; ++i) a += acc[i].x + acc[i].y;
    if (a == 1234.5f) sink[0] = a;
  }
  tc_fence_before();
  if constexpr (kCta == 2) cluster_sync(); else __syncthreads();
  if (warp == 1) {
    if constexpr (kCta == 2) tmem_dealloc2<512>(tmem);
    else tmem_dealloc<512>(tmem);
  }
}

__global__ void fill(uint32_t* p, size_t n, uint32_t seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u + seed;
    h ^= h >> 15; h *= 2246822519u; h ^= h >> 13; h *= 3266489917u; h ^= h >> 16;
    p[i] = h & 0x7f7f7f7fu ^ ((h << 7) & 0x80808080u);
  }
}

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static PFN_encodeTiled enc;

static CUtensorMap make(void* p, int rows, int box_rows) {
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)kK, (cuuint64_t)rows};
  cuuint64_t str[1] = {(cuuint64_t)kK};
  cuuint32_t box[2] = {128, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, p, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return m;
}

template <int C, int S, int E>
void run(void* a, void* b) {
  long long* cyc;
  float* sink;
  cudaMalloc(&cyc, 148 * sizeof(long long));
  cudaMalloc(&sink, 64);
  cudaMemset(cyc, 0, 148 * sizeof(long long));
  const CUtensorMap ma = make(a, kM, 128), mb = make(b, kN, C == 2 ? 128 : 256);
  const int smem = 1024 + S * (16384 + (C == 2 ? 16384 : 32768)) + (E == 5 ? 49152 : 0);
  cudaFuncSetAttribute(ingress<C, S, E>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(148);
  cfg.blockDim = dim3(E == 3 ? 640 : 384);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int r = 0; r < 2; ++r) cudaLaunchKernelEx(&cfg, ingress<C, S, E>, ma, mb, cyc, sink);
  cudaEventRecord(e0);
  const int reps = 5;
  for (int r = 0; r < reps; ++r) cudaLaunchKernelEx(&cfg, ingress<C, S, E>, ma, mb, cyc, sink);
  cudaEventRecord(e1);
  cudaError_t e = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  long long c[148];
  cudaMemcpy(c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
  double avg = 0;
  int n = 0;
  for (int i = 0; i < 148; i += C) { avg += c[i]; ++n; }
  avg /= n;
  const double tops = 2.0 * kM * kN * (double)kK * reps / (ms * 1e-3) / 1e12;
  printf("cta=%d stages=%d epi=%d: %6.0f cycles/item (%5.1f%% of MMA peak)  %6.0f TOPS  %s\n", C, S, E, avg,
         100.0 * 512 / avg, tops, cudaGetErrorString(e));
  cudaFree(cyc);
  cudaFree(sink);
}

int main() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  enc = (PFN_encodeTiled)fn;
  void *a, *b;
  cudaMalloc(&a, (size_t)kM * kK);
  cudaMalloc(&b, (size_t)kN * kK);
  fill<<<1024, 256>>>((uint32_t*)a, (size_t)kM * kK / 4, 1);
  fill<<<1024, 256>>>((uint32_t*)b, (size_t)kN * kK / 4, 2);
  run<1, 4, 0>(a, b);
  run<1, 4, 1>(a, b);
  run<1, 4, 9>(a, b);
  run<1, 4, 10>(a, b);
  run<1, 4, 4>(a, b);
  run<1, 4, 7>(a, b);
  run<1, 4, 1>(a, b);
  run<1, 4, 9>(a, b);
  return 0;
}
