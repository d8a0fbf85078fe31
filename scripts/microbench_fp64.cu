// FP64 on B200: dependent-chain latency and multi-warp throughput of DFMA / F2F.F64.F32 (vs FFMA).
#include <cstdio>
template <int K>
__global__ void chains(double* out, const float* in, int n, long long* cyc) {
  double ss[K]; float v = in[threadIdx.x];
  for (int k = 0; k < K; ++k) ss[k] = 0.0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int k = 0; k < K; ++k) { const double d = (double)(v + (float)k); ss[k] = __fma_rn(d, d, ss[k]); }
    v += 1.0f;
  }
  long long t1 = clock64();
  double a = 0; for (int k = 0; k < K; ++k) a += ss[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = a; if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}
template <int K>
__global__ void dchains(double* out, const float* in, int n, long long* cyc) {
  double ss[K]; const double d = in[threadIdx.x];
  for (int k = 0; k < K; ++k) ss[k] = k;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int k = 0; k < K; ++k) ss[k] = __fma_rn(d, d, ss[k]);
  }
  long long t1 = clock64();
  double a = 0; for (int k = 0; k < K; ++k) a += ss[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = a; if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double* o; float* in; long long* c; cudaMalloc(&o, 1 << 24); cudaMalloc(&in, 4096 * 4); cudaMalloc(&c, 8);
  cudaMemset(in, 0, 4096 * 4);
  long long h; const int n = 2048;
  for (int warps : {1, 4, 16}) {
    chains<8><<<148, 32 * warps>>>(o, in, n, c); cudaDeviceSynchronize();
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("F2F+DFMA x8 chains, %2d warps/SM: %.2f cyc per (F2F+DFMA) per warp -> %.1f lane-ops/clk/SM\n", warps,
           (double)h / n / 8, 32.0 * warps * 8 * n / h);
    dchains<8><<<148, 32 * warps>>>(o, in, n, c); cudaDeviceSynchronize();
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("DFMA x8 chains,     %2d warps/SM: %.2f cyc per DFMA per warp -> %.1f DFMA lanes/clk/SM\n", warps,
           (double)h / n / 8, 32.0 * warps * 8 * n / h);
  }
  return 0;
}
