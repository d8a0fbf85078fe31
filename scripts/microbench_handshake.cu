// Microbenchmark: MMA (M=128,N=256,K=128 per item) with the TMEM-slot handshake
// of the GEMM: MMA thread waits tempty[slot], issues, commits tfull[slot];
// kEpi epilogue warps wait tfull, optionally tcgen05.ld their columns, and
// arrive on tempty.  Measures how much the handshake costs the tensor pipe.
#include <cstdio>
#include <cuda_runtime.h>
#include "sm100.cuh"
using namespace fbq::sm100;

template <int kEpiWarps, int kSlots, bool kLoad, int kVariant>
__global__ void hs(long long* cycles, int iters, int delay) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t tfull[4], tempty[4], extra[4];
  __shared__ uint32_t tmem_holder;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int kN = 512 / kSlots;  // columns per slot
  for (int i = threadIdx.x; i < ((kVariant & 2) ? 192 : 48) * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = (kVariant >= 4) ? (uint32_t)(i * 2654435761u) ^ (uint32_t)(blockIdx.x * 0x9E3779B9u) : 0x01010101u * (i & 7);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kSlots; ++s) { mbar_init(tfull + s, 1); mbar_init(tempty + s, kEpiWarps); mbar_init(extra + s, 1); }
    fence_barrier_init();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) tmem_alloc<512>(&tmem_holder);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_holder;
  long long t0 = clock64();
  if (warp == 0) {
    const uint32_t idesc = idesc_i8(128, kN, 0, 0);
    for (int it = 0; it < iters; ++it) {
      const int slot = it % kSlots;
      const uint32_t sa = smem_u32(smem) + ((kVariant & 2) ? (it % 3) * 65536 : 0);
      const uint32_t sb = sa + ((kVariant & 2) ? 32768 : 16384);
      mbar_wait(tempty + slot, ((it / kSlots) & 1) ^ 1);
      tc_fence_after();
      if (delay) {  // emulate per-item bookkeeping in the issuing thread
        const long long t = clock64();
        while (clock64() - t < delay) {}
      }
      if (lane == 0) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          mma_i8(tmem + slot * kN, smem_desc_sw128(sa + kk * 32, 16, 1024),
                 smem_desc_sw128(sb + kk * 32, 16, 1024), idesc, kk > 0);
        mma_commit(tfull + slot);
        if (kVariant & 1) mma_commit(extra + slot);
      }
      __syncwarp();
    }
  } else if (warp >= 4 && warp < 4 + kEpiWarps) {
    const int ew = warp - 4, q = warp & 3;
    const int cols = kN / (kEpiWarps / 4);
    const int c0 = (ew >> 2) * cols;
    uint32_t sink = 0;
    for (int it = 0; it < iters; ++it) {
      const int slot = it % kSlots;
      mbar_wait(tfull + slot, (it / kSlots) & 1);
      tc_fence_after();
      if constexpr (kLoad) {
        for (int c = 0; c < cols; c += 16) {
          uint32_t v[16];
          tmem_ld16(tmem + ((q * 32) << 16) + slot * kN + c0 + c, v);
          tmem_ld_wait();
          sink += v[0] ^ v[15];
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty + slot);
    }
    if (sink == 12345) cycles[1000] = sink;
  }
  long long t1 = clock64();
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tmem_dealloc<512>(tmem);
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  }
}

template <int E, int S, bool L, int V = 0>
void run(int iters, int delay = 0) {
  long long* cyc;
  cudaMalloc(&cyc, 2000 * sizeof(long long));
  const int smem = 1024 + ((V & 2) ? 192 : 48) * 1024;
  cudaFuncSetAttribute(hs<E, S, L, V>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  hs<E, S, L, V><<<148, 128 + 32 * E, smem>>>(cyc, iters, delay);
  cudaDeviceSynchronize();
  hs<E, S, L, V><<<148, 128 + 32 * E, smem>>>(cyc, iters, delay);
  cudaError_t e = cudaDeviceSynchronize();
  long long c[148];
  cudaMemcpy(c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += c[i];
  avg /= 148;
  const double macs = 128.0 * (512 / S) * 128 * iters;
  printf("delay=%4d variant=%d epi_warps=%2d slots=%d N=%3d tmem_ld=%d: %5.1f%% of 8192 MAC/clk  %s\n", delay, V, E, S, 512 / S, (int)L,
         100 * macs / avg / 8192, cudaGetErrorString(e));
  cudaFree(cyc);
}

int main() {
  run<8, 2, false, 0>(4000);
  run<8, 2, true, 0>(4000);
  run<8, 2, true, 4>(4000);
  run<8, 2, true, 7>(4000);
  run<8, 4, true, 0>(4000);
  run<8, 4, true, 4>(4000);
  run<8, 4, true, 7>(4000);
  run<16, 4, true, 7>(4000);
  run<16, 2, true, 7>(4000);
  return 0;
}
