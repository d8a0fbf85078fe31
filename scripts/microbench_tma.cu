// Microbenchmark: per-SM TMA ingress (L2 -> smem) throughput vs ring depth.
// One thread per CTA streams 128x128 int8 tiles (16 KiB, 128B swizzle) of an
// L2-resident operand into an S-stage ring (B boxes per stage), re-arming each
// stage as soon as it lands.  Separates a latency bound (more stages help) from
// a bandwidth bound (they do not), and the chip-wide L2 cap (fewer CTAs help)
// from a per-SM port limit (they do not).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2503_08040_b200/csrc \
//        -o scripts/mb_tma scripts/microbench_tma.cu -lcuda
#include <cstdio>
#include <cstdlib>
#include <cuda.h>
#include <cuda_runtime.h>

#include "sm100.cuh"

using namespace fbq::sm100;

__global__ void __launch_bounds__(128, 1)
tma_stream(const __grid_constant__ CUtensorMap map, int stages, int boxes, int iters, int tiles_m,
           int tiles_k, long long* out, int box_bytes) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ uint64_t fullb[4][16];
  const int w = threadIdx.x >> 5;
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u) +
                  (size_t)w * stages * boxes * box_bytes;
  uint64_t* full = fullb[w];
  if ((threadIdx.x & 31) != 0) return;
  for (int s = 0; s < stages; ++s) mbar_init(full + s, 1);
  fence_barrier_init();
  const uint64_t pol = l2_policy_evict_last();
  uint32_t phase = 0;
  long long t0 = 0;
  const int ntiles = tiles_m * tiles_k;
  for (int it = 0; it < iters + stages; ++it) {
    const int s = it % stages;
    if (it >= stages) {
      mbar_wait(full + s, phase);
      if (s == stages - 1) phase ^= 1;
    }
    if (it == stages) t0 = clock64();  // steady state from the first landed stage
    if (it < iters) {
      mbar_arrive_expect_tx(full + s, boxes * box_bytes);
      for (int b = 0; b < boxes; ++b) {
        const int t = (int)((unsigned)((it * boxes + b) * 148 + blockIdx.x * 4 + w) % (unsigned)ntiles);
        tma_load_2d(smem + (s * boxes + b) * box_bytes, &map, full + s, (t % tiles_k) * 128,
                    (t / tiles_k) * (box_bytes / 128), pol);
      }
    }
  }
  if (w == 0) out[blockIdx.x] = clock64() - t0;
}

// plain LDG.128 streaming from L2 (all 256 threads, 8 loads in flight each)
__global__ void __launch_bounds__(256, 1) ldg_stream(const uint4* buf, size_t n16, int iters, long long* out, uint4* sink) {
  uint4 acc = make_uint4(0, 0, 0, 0);
  long long t0 = clock64();
  size_t base = ((size_t)blockIdx.x * 256 + threadIdx.x);
  for (int it = 0; it < iters; ++it) {
    uint4 v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = __ldcg(buf + (base + (size_t)(it * 8 + j) * 148 * 256) % n16);
#pragma unroll
    for (int j = 0; j < 8; ++j) { acc.x ^= v[j].x; acc.y ^= v[j].y; acc.z ^= v[j].z; acc.w ^= v[j].w; }
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
  if (acc.x == 0x12345 && acc.y == 7) sink[0] = acc;
}

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                    const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int rows = 8192, cols = 8192;  // 64 MiB int8, L2-resident after warm-up
  void* buf;
  cudaMalloc(&buf, (size_t)rows * cols);
  cudaMemset(buf, 1, (size_t)rows * cols);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols};
  cuuint32_t box[2] = {128, 128};
  cuuint32_t es[2] = {1, 1};
  ((PFN_encodeTiled)fn)(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, buf, dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  cudaFuncSetAttribute(tma_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024 + 1024);
  CUtensorMap map256;
  cuuint32_t box256[2] = {128, 256};
  ((PFN_encodeTiled)fn)(&map256, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, buf, dims, strides, box256, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  struct Cfg { int stages, boxes, warps, box_bytes, ctas; };
  Cfg cfgs[] = {{3, 3, 1, 16384, 148}, {3, 1, 1, 16384, 148}, {3, 1, 2, 16384, 148}, {3, 1, 4, 16384, 148},
                {3, 3, 2, 16384, 148}, {3, 3, 4, 8192, 148}, {3, 1, 1, 32768, 148}, {3, 2, 1, 32768, 148},
                {3, 1, 4, 16384, 74}};
  for (const Cfg& c : cfgs) {
    const int iters = 6000 / c.boxes;
    const int smem = c.warps * c.stages * c.boxes * c.box_bytes + 1024;
    if (smem > 200 * 1024 + 1024) { printf("skip\n"); continue; }
    const CUtensorMap& m = c.box_bytes == 32768 ? map256 : map;
    for (int rep = 0; rep < 2; ++rep)
      tma_stream<<<c.ctas, 32 * c.warps, smem>>>(m, c.stages, c.boxes, iters, rows / (c.box_bytes / 128), cols / 128, d, c.box_bytes);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, d, sizeof(long long) * c.ctas, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < c.ctas; ++i) avg += h[i];
    avg /= c.ctas;
    const double bytes = (double)iters * c.boxes * c.box_bytes * c.warps;
    printf("TMA warps=%d stages=%d x %d boxes of %5d B, ctas=%3d: %6.1f B/clk/SM  (%5.0f cyc per 48 KiB)  %s\n",
           c.warps, c.stages, c.boxes, c.box_bytes, c.ctas, bytes / avg, 49152.0 / (bytes / avg), cudaGetErrorString(e));
  }
  {
    uint4* sink;
    cudaMalloc(&sink, 64);
    const size_t n16 = (size_t)rows * cols / 16;
    for (int rep = 0; rep < 2; ++rep) ldg_stream<<<148, 256>>>((const uint4*)buf, n16, 400, d, sink);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 148; ++i) avg += h[i];
    avg /= 148;
    printf("LDG.128 (256 thr x 8 in flight): %6.1f B/clk/SM  %s\n", 400.0 * 8 * 256 * 16 / avg, cudaGetErrorString(e));
  }
  return 0;
}
