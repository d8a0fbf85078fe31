// Microbenchmark: raw tcgen05.mma.kind::i8 throughput per SM (no TMA, no
// epilogue), single-CTA M=128 with N in {64,128,256}, commit cadence varied.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2503_08040_b200/csrc \
//        -o scripts/mb_mma scripts/microbench_mma.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "sm100.cuh"

using namespace fbq::sm100;

template <int N, int kCommitEvery>
__global__ void __launch_bounds__(128, 1) mma_loop(long long* cycles, int iters) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar[2];
  __shared__ uint32_t tmem_holder;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 48 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x01010101u * (i & 7);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
    fence_barrier_init();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) tmem_alloc<512>(&tmem_holder);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_holder;
  long long t0 = 0, t1 = 0;
  if (warp == 0) {
    const uint32_t idesc = idesc_i8(128, N, 0, 0);
    const uint32_t sa = smem_u32(smem), sb = sa + 16384;
    uint32_t ph[2] = {0, 0};
    t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const int slot = it & 1;
      const int grp = (it / kCommitEvery) & 1;
      const bool last_in_grp = (it % kCommitEvery) == kCommitEvery - 1;
      if ((threadIdx.x & 31) == 0) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          mma_i8(tmem + slot * 256, smem_desc_sw128(sa + kk * 32, 16, 1024),
                 smem_desc_sw128(sb + kk * 32, 16, 1024), idesc, kk > 0);
        }
        if (last_in_grp) mma_commit(bar + grp);
      }
      __syncwarp();
      if (last_in_grp && it >= kCommitEvery) {
        // at most two commit groups in flight: wait for the previous group
        mbar_wait(bar + (grp ^ 1), ph[grp ^ 1]);
        ph[grp ^ 1] ^= 1;
      }
    }
    t1 = clock64();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tmem_dealloc<512>(tmem);
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  }
}

template <int N, int C>
void run(int iters) {
  long long* cyc;
  cudaMalloc(&cyc, 148 * sizeof(long long));
  const int smem = 1024 + 48 * 1024;
  cudaFuncSetAttribute(mma_loop<N, C>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  mma_loop<N, C><<<148, 128, smem>>>(cyc, iters);
  cudaDeviceSynchronize();
  mma_loop<N, C><<<148, 128, smem>>>(cyc, iters);
  cudaError_t e = cudaDeviceSynchronize();
  long long c[148];
  cudaMemcpy(c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += c[i];
  avg /= 148;
  const double macs = 128.0 * N * 128 * iters;
  printf("M=128 N=%3d commit/%d items: %6.0f MAC/clk/SM (%.0f%% of 8192)  %s\n", N, C, macs / avg,
         100 * macs / avg / 8192, cudaGetErrorString(e));
  cudaFree(cyc);
}

int main() {
  run<256, 1>(4000);
  run<256, 2>(4000);
  run<256, 4>(4000);
  run<128, 1>(4000);
  run<128, 4>(4000);
  run<64, 1>(4000);
  return 0;
}
