// Microbenchmark: CTA-pair (cta_group::2) kind::i8 MMA, M=256, N=kN per item,
// kSlots TMEM slots per CTA, 16 epilogue warps per CTA loading their columns
// and arriving (remotely) on the leader's tempty barrier.
#include <cstdio>
#include <cuda_runtime.h>
#include "sm100.cuh"
using namespace fbq::sm100;

template <int kN, int kSlots>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(640, 1) k2(long long* cycles, int iters) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t tfull[8], tempty[8];
  __shared__ uint32_t tmem_holder;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  for (int i = threadIdx.x; i < 32 * 1024 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(smem)[i] = (uint32_t)(i * 2654435761u) ^ (blockIdx.x * 0x9E3779B9u);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kSlots; ++s) { mbar_init(tfull + s, 1); mbar_init(tempty + s, 32); }
    fence_barrier_init();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) tmem_alloc2<512>(&tmem_holder);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = tmem_holder;
  long long t0 = clock64();
  if (warp == 0 && rank == 0) {
    if (lane == 0) {
      const uint32_t idesc = idesc_i8(256, kN, 0, 0);
      const uint32_t sa = smem_u32(smem), sb = sa + 16384;  // A 128 rows, B kN/2 rows per CTA
      for (int it = 0; it < iters; ++it) {
        const int slot = it % kSlots;
        mbar_wait(tempty + slot, ((it / kSlots) & 1) ^ 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          mma2_i8(tmem + slot * kN, smem_desc_sw128(sa + kk * 32, 16, 1024),
                  smem_desc_sw128(sb + kk * 32, 16, 1024), idesc, kk > 0);
        mma2_commit_mc(tfull + slot, 3);
      }
    }
  } else if (warp >= 4 && warp < 20) {
    const int ew = warp - 4, q = warp & 3;
    const int cols = kN / 4;  // 4 warps per quadrant share the slot's kN columns
    const int c0 = (ew >> 2) * cols;
    const uint32_t leader_tempty = mapa_shared(smem_u32(tempty), 0);
    uint32_t sink = 0;
    for (int it = 0; it < iters; ++it) {
      const int slot = it % kSlots;
      mbar_wait(tfull + slot, (it / kSlots) & 1);
      tc_fence_after();
      for (int c = 0; c < cols; c += 16) {
        uint32_t v[16];
        tmem_ld16(tmem + ((q * 32) << 16) + slot * kN + c0 + c, v);
        tmem_ld_wait();
        sink += v[0] ^ v[15];
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(leader_tempty + slot * 8);
    }
    if (sink == 12345) cycles[1000] = sink;
  }
  long long t1 = clock64();
  tc_fence_before();
  cluster_sync();
  if (warp == 0) {
    tmem_dealloc2<512>(tmem);
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  }
}

template <int N, int S>
void run(int iters) {
  long long* cyc;
  cudaMalloc(&cyc, 2000 * sizeof(long long));
  const int smem = 1024 + 32 * 1024;
  cudaFuncSetAttribute(k2<N, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k2<N, S><<<148, 640, smem>>>(cyc, iters);
  cudaDeviceSynchronize();
  k2<N, S><<<148, 640, smem>>>(cyc, iters);
  cudaError_t e = cudaDeviceSynchronize();
  long long c[148];
  cudaMemcpy(c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; i += 2) avg += c[i];
  avg /= 74;
  const double macs_per_sm = 128.0 * N * 128 * iters;  // each SM: 128 rows x N x 128 deep per item
  printf("2CTA M=256 N=%3d slots=%d: %5.1f%% of 8192 MAC/clk/SM  %s\n", N, S, 100 * macs_per_sm / avg / 8192,
         cudaGetErrorString(e));
  cudaFree(cyc);
}

int main() {
  run<256, 2>(4000);
  run<128, 4>(8000);
  run<64, 8>(16000);
  return 0;
}
