// Microbenchmark: (1) sustained tcgen05.mma kind::i8 rate with LOW-entropy vs
// RANDOM operand bytes (tensor-pipe power throttling), with the SM clock
// measured from clock64 / %globaltimer; (2) the int32->fp32 convert + scale
// epilogue mixes (which pipe I2F runs on, and whether an ALU/FMA split beats
// the I2F + FFMA2 pair).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2503_08040_b200/csrc \
//        -o scripts/mb_pow scripts/microbench_power.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#include "sm100.cuh"

using namespace fbq::sm100;

__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

template <int N, int kVar = 0>
__global__ void __launch_bounds__(128, 1) mma_loop(long long* out, int iters, int random) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar[2], bar2[3];
  __shared__ uint32_t tmem_holder;
  const int warp = threadIdx.x >> 5;
  // 3 stages of A (16 KiB) + B (32 KiB)
  for (int i = threadIdx.x; i < 3 * 48 * 1024 / 4; i += blockDim.x) {
    uint32_t v;
    if (random) {
      uint32_t h = (uint32_t)i * 2654435761u + blockIdx.x * 97u;
      h ^= h >> 15; h *= 2246822519u; h ^= h >> 13; h *= 3266489917u; h ^= h >> 16;
      v = h & 0x7f7f7f7fu;  // |code| <= 127 both signs via bit 7 of the next byte... keep simple
      v ^= (h << 7) & 0x80808080u;
    } else {
      v = 0x01010101u * (i & 7);
    }
    reinterpret_cast<uint32_t*>(smem)[i] = v;
  }
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
    for (int i = 0; i < 3; ++i) mbar_init(bar2 + i, 1);
    fence_barrier_init();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) tmem_alloc<512>(&tmem_holder);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_holder;
  long long t0 = 0, t1 = 0;
  uint64_t g0 = 0, g1 = 0;
  if (warp == 0) {
    const uint32_t idesc = idesc_i8(128, N, 0, 0);
    uint32_t ph[2] = {0, 0};
    t0 = clock64();
    g0 = gtimer();
    for (int it = 0; it < iters; ++it) {
      const int slot = it & 1;
      const uint32_t sa = smem_u32(smem) + (it % 3) * 49152, sb = sa + 16384;
      if ((threadIdx.x & 31) == 0) {
        if (kVar >= 2) tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          mma_i8(tmem + slot * 256, smem_desc_sw128(sa + kk * 32, 16, 1024),
                 smem_desc_sw128(sb + kk * 32, 16, 1024), idesc, kk > 0);
        mma_commit(bar + slot);
        if (kVar >= 1) mma_commit(bar2 + (it % 3));
      }
      __syncwarp();
      if (it >= 1) {
        if (kVar >= 3) mbar_wait_sleep(bar + (slot ^ 1), ph[slot ^ 1]);
        else mbar_wait(bar + (slot ^ 1), ph[slot ^ 1]);
        ph[slot ^ 1] ^= 1;
      }
    }
    t1 = clock64();
    g1 = gtimer();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tmem_dealloc<512>(tmem);
    if (threadIdx.x == 0) {
      out[blockIdx.x * 2] = t1 - t0;
      out[blockIdx.x * 2 + 1] = (long long)(g1 - g0);
    }
  }
}

template <int N, int kVar = 0>
void run_mma(int iters, int random) {
  long long* d;
  cudaMalloc(&d, 148 * 2 * sizeof(long long));
  const int smem = 1024 + 3 * 48 * 1024;
  cudaFuncSetAttribute(mma_loop<N, kVar>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  mma_loop<N, kVar><<<148, 128, smem>>>(d, iters / 10, random);
  cudaDeviceSynchronize();
  mma_loop<N, kVar><<<148, 128, smem>>>(d, iters, random);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[296];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double cyc = 0, ns = 0;
  for (int i = 0; i < 148; ++i) { cyc += h[2 * i]; ns += h[2 * i + 1]; }
  cyc /= 148; ns /= 148;
  const double macs = 128.0 * N * 128 * iters;
  printf("MMA var%d M=128 N=%3d %-8s %7.1f ms  %5.0f MHz  %6.0f MAC/clk/SM (%3.0f%%)  %7.0f TOPS chip  %s\n", kVar, N,
         random ? "random" : "lowent", ns * 1e-6, cyc / ns * 1e3, macs / cyc, 100 * macs / cyc / 8192,
         2 * macs * 148 / ns * 1e-3, cudaGetErrorString(e));
  cudaFree(d);
}

// ------------------------------------------------------------- epilogue mixes
// The real epilogue shape: 8 warps, warp w reads TMEM lane quadrant w%4 and the
// 128-column half w/4 of a 256-column slot (4 x tcgen05.ld 32x32b.x32 per item),
// then converts + scale-accumulates 128 values per thread into acc[64] (float2).
constexpr int kItems = 2048;
template <int kMode>
__device__ __forceinline__ void consume(const uint32_t (&v)[32], float2* acc, float s) {
  const float2 s2 = make_float2(s, s);
  const float2 m2 = make_float2(-12582912.0f, -12582912.0f);
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const bool magic = kMode == 1 || (kMode == 2 && (i & 1)) || (kMode == 4 && (i & 3) == 3);
    if (kMode == 3) {
      acc[i].x = __int_as_float(__float_as_int(acc[i].x) ^ v[2 * i] ^ v[2 * i + 1]);
    } else if (magic) {
      const float2 f = make_float2(__uint_as_float(v[2 * i] + 0x4B400000u), __uint_as_float(v[2 * i + 1] + 0x4B400000u));
      acc[i] = __ffma2_rn(__fadd2_rn(f, m2), s2, acc[i]);
    } else {
      acc[i] = __ffma2_rn(make_float2(__int2float_rn((int)v[2 * i]), __int2float_rn((int)v[2 * i + 1])), s2, acc[i]);
    }
  }
}

template <int kMode>
__global__ void __launch_bounds__(256, 1) epi(float* out, long long* cycles, float s) {
  __shared__ uint32_t tmem_holder;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc<512>(&tmem_holder);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb0 = tmem_holder + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * 128;
  float2 acc[64];
#pragma unroll
  for (int i = 0; i < 64; ++i) acc[i] = make_float2(0.f, 0.f);
  long long t0 = clock64();
  for (int it = 0; it < kItems; ++it) {
    const uint32_t tb = tb0 + (it & 1) * 256;
    uint32_t va[32], vb[32];
    tmem_ld32(tb + 0, va);
    tmem_ld32(tb + 32, vb);
    tmem_ld_wait();
    consume<kMode>(va, acc + 0, s);
    tmem_ld32(tb + 64, va);
    consume<kMode>(vb, acc + 16, s);
    tmem_ld32(tb + 96, vb);
    tmem_ld_wait();
    consume<kMode>(va, acc + 32, s);
    consume<kMode>(vb, acc + 48, s);
  }
  long long t1 = clock64();
  float a = 0;
#pragma unroll
  for (int i = 0; i < 64; ++i) a += acc[i].x + acc[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = a;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem_holder);
}

template <int kMode>
void run_epi(const char* name) {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * sizeof(float));
  cudaMalloc(&cyc, 148 * sizeof(long long));
  epi<kMode><<<148, 256>>>(out, cyc, 0.999f);
  cudaDeviceSynchronize();
  epi<kMode><<<148, 256>>>(out, cyc, 0.999f);
  cudaError_t e = cudaDeviceSynchronize();
  long long c[148];
  cudaMemcpy(c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += c[i];
  avg /= 148;
  printf("%-40s %6.1f elements/clk/SM  (%5.0f cycles per 128x256 item; MMA needs 512)  %s\n", name,
         128.0 * 256 * kItems / avg, avg / kItems, cudaGetErrorString(e));
  cudaFree(out);
  cudaFree(cyc);
}

// CTA-pair MMA loop: leader issues M=256 N=256 (128 rows per SM), commit
// multicast to both CTAs, waits for item it-1 like mma_loop.
template <int N>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) mma2_loop(long long* out, int iters, int nslots) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar[4];
  __shared__ uint32_t tmem_holder;
  const int warp = threadIdx.x >> 5;
  const uint32_t rank = cluster_ctarank();
  for (int i = threadIdx.x; i < 3 * 32 * 1024 / 4; i += blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u + blockIdx.x * 97u;
    h ^= h >> 15; h *= 2246822519u; h ^= h >> 13; h *= 3266489917u; h ^= h >> 16;
    reinterpret_cast<uint32_t*>(smem)[i] = (h & 0x7f7f7f7fu) ^ ((h << 7) & 0x80808080u);
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(bar + i, 1);
    fence_barrier_init();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) tmem_alloc2<512>(&tmem_holder);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = tmem_holder;
  long long t0 = 0, t1 = 0;
  uint64_t g0 = 0, g1 = 0;
  if (warp == 0 && rank == 0) {
    const uint32_t idesc = idesc_i8(256, N, 0, 0);
    constexpr int S = 512 / N > 4 ? 4 : 512 / N;  // TMEM slots, S - 1 items in flight
    uint32_t phbits = 0;
    t0 = clock64();
    g0 = gtimer();
    for (int it0 = 0; it0 < iters; it0 += S) {
#pragma unroll
      for (int slot = 0; slot < S; ++slot) {
        const int it = it0 + slot;
        const uint32_t sa = smem_u32(smem) + (slot % 3) * 32768, sb = sa + 16384;
        if ((threadIdx.x & 31) == 0) {
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            mma2_i8(tmem + slot * N, smem_desc_sw128(sa + kk * 32, 16, 1024),
                    smem_desc_sw128(sb + kk * 32, 16, 1024), idesc, kk > 0);
          mma2_commit_mc(bar + slot, 3);
        }
        __syncwarp();
        if (it >= S - 1) {  // wait for item it - (S - 1)
          constexpr int dummy = 0;
          const int w = (slot + 1) % S;
          mbar_wait(bar + w, (phbits >> w) & 1);
          phbits ^= 1u << w;
          (void)dummy;
        }
      }
    }
    t1 = clock64();
    g1 = gtimer();
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 0) {
    tmem_dealloc2<512>(tmem);
    if (threadIdx.x == 0 && rank == 0) {
      out[blockIdx.x * 2] = t1 - t0;
      out[blockIdx.x * 2 + 1] = (long long)(g1 - g0);
    }
  }
}

template <int N>
void run_mma2(int iters) {
  long long* d;
  cudaMalloc(&d, 148 * 2 * sizeof(long long));
  const int smem = 1024 + 3 * 32 * 1024;
  cudaFuncSetAttribute(mma2_loop<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  mma2_loop<N><<<148, 128, smem>>>(d, iters / 10, 512 / N > 4 ? 4 : 512 / N);
  cudaDeviceSynchronize();
  mma2_loop<N><<<148, 128, smem>>>(d, iters, 512 / N > 4 ? 4 : 512 / N);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[296];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double cyc = 0, ns = 0;
  for (int i = 0; i < 148; i += 2) { cyc += h[2 * i]; ns += h[2 * i + 1]; }
  cyc /= 74; ns /= 74;
  const double macs = 128.0 * N * 128 * iters;  // per SM
  printf("MMA2 pair M=256 N=%d random %7.1f ms %5.0f MHz %6.0f MAC/clk/SM (%3.0f%%)  %s\n", N, ns * 1e-6,
         cyc / ns * 1e3, macs / cyc, 100 * macs / cyc / 8192, cudaGetErrorString(e));
  cudaFree(d);
}

int main(int argc, char** argv) {
  const int iters = argc > 1 ? atoi(argv[1]) : 200000;
  run_mma2<256>(iters);
  run_mma2<128>(iters);
  run_mma2<64>(iters);
  return 0;
  run_epi<0>("TMEM ld + I2F + FFMA2 (current)");
  run_epi<1>("TMEM ld + IADD + FADD2 + FFMA2 (magic)");
  run_epi<2>("TMEM ld + 1:1 I2F : magic");
  run_epi<4>("TMEM ld + 3:1 I2F : magic");
  run_epi<3>("TMEM ld only (LOP3 sink)");
  run_mma<256, 0>(iters, 1);
  run_mma<256, 1>(iters, 1);
  run_mma<256, 2>(iters, 1);
  run_mma<256, 3>(iters, 1);
  run_mma<256>(iters * 4, 1);
  return 0;
}
