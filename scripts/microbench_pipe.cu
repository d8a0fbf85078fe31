// Microbenchmark (round 2): int8 tcgen05 MMA pipeline shapes for K3.
//   1-CTA  M=128 N=kN             (cta_group::1)
//   2-CTA  M=256 N=kN, CTA pair   (cta_group::2; each CTA: 128 A rows, kN/2 B rows)
// Each item = one 128-deep k-block = 4 MMAs (K=32) into TMEM slot (item % kSlots).
// Operands rotate over 4 smem stages (no TMA).  Modes:
//   0  MMA only: the issuer bounds itself on its own commits (no epilogue warps)
//   1  + epilogue handshake: 8 epilogue warps wait tfull, release (no tcgen05.ld)
//   2  + every epilogue warp tcgen05.ld's its kN/2 columns before the release
//   3  + I2F + FFMA2 of the loaded words into register accumulators (after release)
//   4  chunk-pipelined epilogue (N=256): 32-column TMEM loads one chunk ahead of the
//      math (ld(g+1); math(g); wait), slot released once its last chunk landed;
//      setmaxnreg 224 for the epilogue warps
//   5  as 4, one element pair in kMixDiv converted on the FMA pipe (IMAD magic + FADD2)
//   6  as 4 without MMAs (the issuer arrives on tfull itself): epilogue capacity
//   7  as 4 without I2F (FFMA2 on the raw words): ALU relief
//   8  as 4 without any math (pipelined loads only)
// kCta == 3: CTA pair with M=128 (64 A rows per CTA; D per CTA = 128 lanes x kN/2 columns,
//   columns [kN/2, kN) of the 64 rows live in lanes 64-127); mode 9 = its epilogue:
//   8 warps x (32 lanes x 64 columns), whole-item loads double-buffered against the math
// Prints % of 8192 int8 MAC/clk/SM (MMA-issuer clock64 over the loop).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2503_08040_b200/csrc \
//        -o scripts/mb_pipe scripts/microbench_pipe.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "sm100.cuh"

using namespace fbq::sm100;

constexpr int kStagesMb = 4;

__device__ __forceinline__ void ld16p(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
constexpr int kEpi = 8;
constexpr int kMixDiv = 4;

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

template <int kMix>
__device__ __forceinline__ void consume32(const uint32_t* v, float2* acc, float s, uint32_t one) {
  const float2 s2 = make_float2(s, s);
  if constexpr (kMix == 8) {
    uint32_t x = 0;
#pragma unroll
    for (int i = 0; i < 32; ++i) x ^= v[i];
    acc[0].x += __uint_as_float(x);
    return;
  }
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    float2 pf;
    if (kMix == 7) {
      pf = make_float2(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1]));
    } else if (kMix == 5 && (i % kMixDiv) == kMixDiv - 1) {
      const float2 b = make_float2(__uint_as_float(v[2 * i] * one + 0x4B400000u),
                                   __uint_as_float(v[2 * i + 1] * one + 0x4B400000u));
      pf = __fadd2_rn(b, make_float2(-12582912.0f, -12582912.0f));
    } else {
      pf = make_float2(__int2float_rn((int)v[2 * i]), __int2float_rn((int)v[2 * i + 1]));
    }
    acc[i] = __ffma2_rn(pf, s2, acc[i]);
  }
}

template <int kMix>
__device__ __forceinline__ void consume16(const uint32_t* v, float2* acc, float s) {
  const float2 s2 = make_float2(s, s);
#pragma unroll
  for (int i = 0; i < 8; ++i)
    acc[i] = __ffma2_rn(make_float2(__int2float_rn((int)v[2 * i]), __int2float_rn((int)v[2 * i + 1])), s2, acc[i]);
}

// Mode 10 (1-CTA, N=256, 2 slots): 16-column loads into a 4-deep register ring with NO
// tcgen05.wait::ld between them (ptxas scoreboards the LDTM destinations); one wait::ld
// per item right after the item's last load is issued, then the slot release.
template <int kSlots>
__device__ __forceinline__ void epi_ring(uint32_t tmem, uint64_t* tfull, uint64_t* tempty, float* sink,
                                         int iters, int warp, int lane) {
  const int q = warp & 3, h = (warp - 4) >> 2;
  const uint32_t lane_base = tmem + ((q * 32) << 16) + h * 128;
  float2 acc[64];
#pragma unroll
  for (int i = 0; i < 64; ++i) acc[i] = make_float2(0.f, 0.f);
  const float s = 1.0f + blockIdx.x * 1e-7f;
  uint32_t r0[16], r1[16], r2[16], r3[16];
  mbar_wait(tfull, 0);
  tc_fence_after();
  ld16p(lane_base + 0, r0);
  ld16p(lane_base + 16, r1);
  ld16p(lane_base + 32, r2);
  for (int it = 0; it < iters; ++it) {
    const uint32_t tb = lane_base + (it % kSlots) * 256;
    const bool more = it + 1 < iters;
    const uint32_t nb = lane_base + ((it + 1) % kSlots) * 256;
    ld16p(tb + 48, r3);  consume16<0>(r0, acc + 0, s);
    ld16p(tb + 64, r0);  consume16<0>(r1, acc + 8, s);
    ld16p(tb + 80, r1);  consume16<0>(r2, acc + 16, s);
    ld16p(tb + 96, r2);  consume16<0>(r3, acc + 24, s);
    ld16p(tb + 112, r3); consume16<0>(r0, acc + 32, s);
    tmem_ld_wait();
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(tempty + it % kSlots);
    if (more) {
      mbar_wait(tfull + (it + 1) % kSlots, ((it + 1) / kSlots) & 1);
      tc_fence_after();
      ld16p(nb + 0, r0);
    }
    consume16<0>(r1, acc + 40, s);
    if (more) ld16p(nb + 16, r1);
    consume16<0>(r2, acc + 48, s);
    if (more) ld16p(nb + 32, r2);
    consume16<0>(r3, acc + 56, s);
  }
  float t = 0.f;
#pragma unroll
  for (int i = 0; i < 64; ++i) t += acc[i].x + acc[i].y;
  if (t == 1234.5f) sink[1] = t;
}

// CTA pair, M=128, N=256: slot = 128 columns; warp (q, h) owns lanes 32q.. x columns h*64..+63.
// Whole-item staging (64 regs) double-buffered: ld(item+1) is in flight during math(item).
template <int kSlots>
__device__ __forceinline__ void epi_pair128(uint32_t tmem, uint64_t* tfull, uint64_t* tempty, float* sink,
                                            int iters, int warp, int lane) {
  const int q = warp & 3, h = (warp - 4) >> 2;
  const uint32_t tempty_addr = mapa_shared(smem_u32(tempty), 0);
  const uint32_t lane_base = tmem + ((q * 32) << 16) + h * 64;
  float2 acc[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) acc[i] = make_float2(0.f, 0.f);
  const float s = 1.0f + blockIdx.x * 1e-7f;
  uint32_t va[64], vb[64];
  mbar_wait(tfull, 0);
  tc_fence_after();
  ld32p(lane_base, va);
  ld32p(lane_base + 32, va + 32);
  tmem_ld_wait();
  tc_fence_before();
  __syncwarp();
  if (lane == 0) mbar_arrive_cluster(tempty_addr);
  for (int it = 0; it < iters; it += 2) {
    // va holds item it; load it+1 into vb during the math on va
    if (it + 1 < iters) {
      const int ns = (it + 1) % kSlots;
      mbar_wait(tfull + ns, ((it + 1) / kSlots) & 1);
      tc_fence_after();
      ld32p(lane_base + ns * 128, vb);
      ld32p(lane_base + ns * 128 + 32, vb + 32);
    }
    consume32<4>(va, acc, s, 1u);
    consume32<4>(va + 32, acc + 16, s, 1u);
    if (it + 1 < iters) {
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(tempty_addr + ((it + 1) % kSlots) * 8);
    } else break;
    if (it + 2 < iters) {
      const int ns = (it + 2) % kSlots;
      mbar_wait(tfull + ns, ((it + 2) / kSlots) & 1);
      tc_fence_after();
      ld32p(lane_base + ns * 128, va);
      ld32p(lane_base + ns * 128 + 32, va + 32);
    }
    consume32<4>(vb, acc, s, 1u);
    consume32<4>(vb + 32, acc + 16, s, 1u);
    if (it + 2 < iters) {
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(tempty_addr + ((it + 2) % kSlots) * 8);
    }
  }
  float t = 0.f;
#pragma unroll
  for (int i = 0; i < 32; ++i) t += acc[i].x + acc[i].y;
  if (t == 1234.5f) sink[1] = t;
}

// 8 warps x (32 lanes x 128 columns): acc 128 regs, two 32-column staging buffers.
template <int kCta, int kN, int kSlots, int kMode>
__device__ __forceinline__ void epi_pipelined(uint32_t tmem, uint64_t* tfull, uint64_t* tempty, float* sink,
                                              int iters, int warp, int lane) {
  static_assert(kN == 256, "pipelined epilogue assumes 256-column items");
  const int q = warp & 3, h = (warp - 4) >> 2;
  const uint32_t tempty_addr = kCta == 2 ? mapa_shared(smem_u32(tempty), 0) : smem_u32(tempty);
  const uint32_t lane_base = tmem + ((q * 32) << 16) + h * 128;
  float2 acc[64];
#pragma unroll
  for (int i = 0; i < 64; ++i) acc[i] = make_float2(0.f, 0.f);
  const float s = 1.0f + blockIdx.x * 1e-7f;
  const uint32_t one = (uint32_t)(iters > 0);
  uint32_t va[32], vb[32];
  mbar_wait(tfull, 0);
  tc_fence_after();
  ld32p(lane_base, va);
  tmem_ld_wait();
  for (int it = 0; it < iters; ++it) {
    const int slot = it % kSlots;
    const uint32_t tb = lane_base + slot * kN;
    // chunk 0 in va
    ld32p(tb + 32, vb);
    consume32<kMode>(va, acc + 0, s, one);
    tmem_ld_wait();
    ld32p(tb + 64, va);
    consume32<kMode>(vb, acc + 16, s, one);
    tmem_ld_wait();
    ld32p(tb + 96, vb);
    consume32<kMode>(va, acc + 32, s, one);
    tmem_ld_wait();
    // all four chunks of this item loaded: release the slot
    tc_fence_before();
    __syncwarp();
    if (lane == 0) {
      if constexpr (kCta == 2) mbar_arrive_cluster(tempty_addr + slot * 8);
      else mbar_arrive(tempty + slot);
    }
    if (it + 1 < iters) {
      const int ns = (it + 1) % kSlots;
      mbar_wait(tfull + ns, ((it + 1) / kSlots) & 1);
      tc_fence_after();
      ld32p(lane_base + ns * kN, va);
    }
    consume32<kMode>(vb, acc + 48, s, one);
    tmem_ld_wait();
  }
  float t = 0.f;
#pragma unroll
  for (int i = 0; i < 64; ++i) t += acc[i].x + acc[i].y;
  if (t == 1234.5f) sink[1] = t;
}

template <int kCta, int kN, int kSlots, int kMode>
__global__ void __launch_bounds__(128 + 32 * kEpi, 1) pipe(long long* cycles, float* sink, int iters) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t tfull[8], tempty[8];
  __shared__ uint32_t tmem_holder;
  constexpr int kBRows = kCta >= 2 ? kN / 2 : kN;
  constexpr int kARows = kCta == 3 ? 64 : 128;
  constexpr int kStageBytes = kARows * 128 + kBRows * 128;
  constexpr int kSlotCols = kCta == 3 ? kN / 2 : kN;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = kCta >= 2 ? cluster_ctarank() : 0;
  for (int i = threadIdx.x; i < kStagesMb * kStageBytes / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(smem)[i] = (uint32_t)(i * 2654435761u) ^ (blockIdx.x * 0x9E3779B9u);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kSlots; ++s) {
      mbar_init(tfull + s, 1);
      mbar_init(tempty + s, kEpi * (kCta >= 2 ? 2 : 1));
    }
    fence_barrier_init();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    if constexpr (kCta >= 2) tmem_alloc2<512>(&tmem_holder);
    else tmem_alloc<512>(&tmem_holder);
  }
  tc_fence_before();
  if constexpr (kCta >= 2) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_holder;
  if constexpr (kMode >= 4) {
    if (warp < 4) setmaxnreg_dec<40>();
  }
  long long t0 = clock64(), t1 = t0;
  if (warp == 0 && rank == 0) {
    const uint32_t idesc = idesc_i8(kCta == 3 ? 128 : kCta * 128, kN, 0, 0);
    for (int it = 0; it < iters; ++it) {
      const int slot = it % kSlots;
      const uint32_t ph = (it / kSlots) & 1;
      if (kMode == 0) {
        if (it >= kSlots) mbar_wait(tfull + slot, ph ^ 1);  // own previous commit to this slot
      } else {
        mbar_wait(tempty + slot, ph ^ 1);
      }
      tc_fence_after();
      const uint32_t sa = smem_u32(smem) + (it % kStagesMb) * kStageBytes;
      const uint32_t sb = sa + kARows * 128;
      if (kMode == 6) {
        if (lane == 0) mbar_arrive(tfull + slot);
      } else if (lane == 0) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint64_t ad = smem_desc_sw128(sa + kk * 32, 16, 1024), bd = smem_desc_sw128(sb + kk * 32, 16, 1024);
          if constexpr (kCta >= 2) mma2_i8(tmem + slot * kSlotCols, ad, bd, idesc, kk > 0);
          else mma_i8(tmem + slot * kN, ad, bd, idesc, kk > 0);
        }
        if constexpr (kCta >= 2) mma2_commit_mc(tfull + slot, 3);
        else mma_commit(tfull + slot);
      }
      __syncwarp();
    }
    if (kMode == 0) {  // drain
      for (int it = iters - kSlots; it < iters; ++it) mbar_wait(tfull + it % kSlots, (it / kSlots) & 1);
    }
    t1 = clock64();
  } else if (kMode == 10 && warp >= 4) {
    if constexpr (kMode == 10) {
      setmaxnreg_inc<224>();
      epi_ring<kSlots>(tmem, tfull, tempty, sink, iters, warp, lane);
    }
  } else if (kMode == 9 && warp >= 4) {
    if constexpr (kMode == 9) {
      setmaxnreg_inc<224>();
      epi_pair128<kSlots>(tmem, tfull, tempty, sink, iters, warp, lane);
    }
  } else if (kMode >= 4 && warp >= 4) {
    if constexpr (kMode >= 4 && kMode < 9) {
      setmaxnreg_inc<224>();
      epi_pipelined<kCta, kN, kSlots, kMode>(tmem, tfull, tempty, sink, iters, warp, lane);
    }
  } else if (kMode > 0 && kMode < 4 && warp >= 4) {
    const int ew = warp - 4, q = warp & 3, h = ew >> 2;
    constexpr int kCols = (kCta == 3 ? kN / 2 : kN) / 2;  // this warp's columns of the slot
    const uint32_t tempty_addr = kCta >= 2 ? mapa_shared(smem_u32(tempty), 0) : smem_u32(tempty);
    float2 acc[kCols / 2];
#pragma unroll
    for (int i = 0; i < kCols / 2; ++i) acc[i] = make_float2(0.f, 0.f);
    const float s = 1.0f + blockIdx.x * 1e-7f;
    for (int it = 0; it < iters; ++it) {
      const int slot = it % kSlots;
      mbar_wait(tfull + slot, (it / kSlots) & 1);
      tc_fence_after();
      const uint32_t tb = tmem + ((q * 32) << 16) + slot * kSlotCols + h * kCols;
      if constexpr (kMode >= 2) {
        uint32_t v[kCols];
#pragma unroll
        for (int c = 0; c < kCols / 16; ++c) ld16p(tb + c * 16, v + c * 16);
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if constexpr (kCta >= 2) mbar_arrive_cluster(tempty_addr + slot * 8);
          else mbar_arrive(tempty + slot);
        }
        if constexpr (kMode == 3) {
          const float2 s2 = make_float2(s, s);
#pragma unroll
          for (int i = 0; i < kCols / 2; ++i)
            acc[i] = __ffma2_rn(make_float2(__int2float_rn((int)v[2 * i]), __int2float_rn((int)v[2 * i + 1])), s2, acc[i]);
        } else {
          if (v[0] == 0x12345678u && v[kCols - 1] == 7u) sink[0] = 1.f;
        }
      } else {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if constexpr (kCta >= 2) mbar_arrive_cluster(tempty_addr + slot * 8);
          else mbar_arrive(tempty + slot);
        }
      }
    }
    float t = 0.f;
#pragma unroll
    for (int i = 0; i < kCols / 2; ++i) t += acc[i].x + acc[i].y;
    if (t == 1234.5f) sink[1] = t;
  }
  tc_fence_before();
  if constexpr (kCta >= 2) cluster_sync(); else __syncthreads();
  if (warp == 0) {
    if constexpr (kCta >= 2) tmem_dealloc2<512>(tmem);
    else tmem_dealloc<512>(tmem);
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  }
}

template <int C, int N, int S, int M>
void run(int iters) {
  long long* cyc;
  float* sink;
  cudaMalloc(&cyc, 2000 * sizeof(long long));
  cudaMalloc(&sink, 64);
  constexpr int kBRows = C >= 2 ? N / 2 : N;
  const int smem = 1024 + kStagesMb * ((C == 3 ? 8192 : 16384) + kBRows * 128);
  cudaFuncSetAttribute(pipe<C, N, S, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(148);
  cfg.blockDim = dim3(128 + 32 * kEpi);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C >= 2 ? 2 : 1;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, pipe<C, N, S, M>, cyc, sink, iters);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  cudaLaunchKernelEx(&cfg, pipe<C, N, S, M>, cyc, sink, iters);
  cudaEventRecord(e1);
  cudaError_t e = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  long long c[148];
  cudaMemcpy(c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
  double avg = 0;
  int n = 0;
  for (int i = 0; i < 148; i += (C >= 2 ? 2 : 1)) { avg += c[i]; ++n; }
  avg /= n;
  const double macs_per_sm = (C == 3 ? 64.0 : 128.0) * N * 128 * iters;  // each SM: rows x N x 128-deep per item
  const double tops = 2.0 * macs_per_sm * 148 / (ms * 1e-3) / 1e12;
  printf("cta=%d N=%3d slots=%d mode=%d: %5.1f%% of 8192 MAC/clk/SM  %6.0f TOPS  %.1f MHz  %s\n", C, N, S, M,
         100 * macs_per_sm / avg / 8192, tops, avg / (ms * 1e3), cudaGetErrorString(e));
  cudaFree(cyc);
  cudaFree(sink);
}

int main() {
  const int it = 6000;
  run<1, 256, 2, 10>(it); run<1, 256, 2, 4>(it);
  return 0;
  run<1, 256, 2, 0>(it); run<1, 256, 2, 1>(it); run<1, 256, 2, 2>(it); run<1, 256, 2, 3>(it);
  run<1, 128, 4, 0>(it); run<1, 128, 4, 1>(it); run<1, 128, 4, 2>(it); run<1, 128, 4, 3>(it);
  run<2, 256, 2, 0>(it); run<2, 256, 2, 1>(it); run<2, 256, 2, 2>(it); run<2, 256, 2, 3>(it);
  run<2, 128, 4, 0>(it); run<2, 128, 4, 1>(it); run<2, 128, 4, 2>(it); run<2, 128, 4, 3>(it);
  run<2, 128, 2, 0>(it); run<2, 192, 2, 0>(it); run<2, 64, 8, 0>(it);
  run<2, 160, 3, 0>(it); run<2, 160, 3, 3>(it);
  return 0;
}
