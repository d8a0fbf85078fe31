// Microbenchmark: per-SM throughput of the epilogue instruction mixes on
// sm_100a (FFMA vs FFMA2 vs FADD2, int->fp conversions).  Standalone:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb scripts/microbench_epi.cu && ./mb
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096;

template <int kMode>
__global__ void kern(float* out, long long* cycles, float s) {
  float a[16];
  float2 b[8];
  int iv[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    a[i] = threadIdx.x * 0.001f + i;
    iv[i] = threadIdx.x + i;
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) b[i] = make_float2(a[2 * i], a[2 * i + 1]);
  const float2 s2 = make_float2(s, s);
  const float2 c2 = make_float2(-s * 3.f, -s * 3.f);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < kIters; ++it) {
    if constexpr (kMode == 0) {  // scalar FFMA, 16 chains
#pragma unroll
      for (int i = 0; i < 16; ++i) a[i] = __fmaf_rn(a[i], s, 1.0f);
    } else if constexpr (kMode == 1) {  // FFMA2, 8 chains (16 values)
#pragma unroll
      for (int i = 0; i < 8; ++i) b[i] = __ffma2_rn(b[i], s2, c2);
    } else if constexpr (kMode == 2) {  // FADD2 + FFMA2 (the epilogue pair)
#pragma unroll
      for (int i = 0; i < 8; ++i) b[i] = __ffma2_rn(__fadd2_rn(b[i], c2), s2, b[i]);
    } else if constexpr (kMode == 3) {  // scalar FADD + FFMA (16 elements)
#pragma unroll
      for (int i = 0; i < 16; ++i) a[i] = __fmaf_rn(__fadd_rn(a[i], -3.0f), s, a[i]);
    } else if constexpr (kMode == 4) {  // I2F
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        a[i] = __fadd_rn(a[i], __int2float_rn(iv[i]));
        iv[i] += 3;
      }
    } else if constexpr (kMode == 5) {  // IADD (alu) + FADD + FFMA scalar (magic conversion)
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const float f = __int_as_float(iv[i] + 0x4B400000);
        a[i] = __fmaf_rn(__fadd_rn(f, -12582912.0f), s, a[i]);
        iv[i] ^= it;
      }
    } else if constexpr (kMode == 6) {  // mixed: 8 elements scalar FADD+FFMA, 8 via FADD2+FFMA2
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = __fmaf_rn(__fadd_rn(a[i], -3.0f), s, a[i]);
#pragma unroll
      for (int i = 4; i < 8; ++i) b[i] = __ffma2_rn(__fadd2_rn(b[i], c2), s2, b[i]);
    }
  }
  long long t1 = clock64();
  float acc = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) acc += a[i] + (float)iv[i];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc += b[i].x + b[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

template <int kMode>
void run(const char* name, double elems_per_iter_per_thread, int threads) {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * sizeof(float));
  cudaMalloc(&cyc, 148 * sizeof(long long));
  kern<kMode><<<148, threads>>>(out, cyc, 0.999f);
  cudaDeviceSynchronize();
  kern<kMode><<<148, threads>>>(out, cyc, 0.999f);
  cudaDeviceSynchronize();
  long long c[148];
  cudaMemcpy(c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += c[i];
  avg /= 148;
  const double elems = elems_per_iter_per_thread * kIters * threads;
  printf("%-34s threads=%4d  %.1f elements/clk/SM\n", name, threads, elems / avg);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  for (int t : {256, 512, 1024}) {
    run<0>("FFMA scalar (1 op/elem)", 16, t);
    run<1>("FFMA2 (1 op/elem)", 16, t);
    run<2>("FADD2+FFMA2 (epilogue pair)", 16, t);
    run<3>("FADD+FFMA scalar (epilogue pair)", 16, t);
    run<4>("I2F + FADD", 16, t);
    run<5>("IADD+FADD+FFMA (magic conv)", 16, t);
    run<6>("mixed 8 scalar + 8 packed pairs", 16, t);
  }
  return 0;
}
