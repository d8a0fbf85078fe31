// Fallback-mask selection on the device: mask_topk (policy.cpp:56-71) for the
// FixedRate mode -- exactly k = ceil(rate * n) blocks with the largest AbsMax
// scores, ties broken toward the LOWER block index.
//
// Scores are the fp32 block absmaxes (score_blocks(AbsMax) is that float as a
// double, policy.cpp:18-27).  For non-negative floats the bit pattern orders
// like the value, so the reference's comparator (score desc, index asc) is the
// descending order of the unique 64-bit key  bits(score) << 32 | ~index.
// One CTA finds the k-th largest key by an 8-bit MSB radix select (8 histogram
// passes over the n keys in shared memory), then marks every key >= it:
// exactly k bits, no sort, no host round trip.
#include <cuda_runtime.h>
#include <cstdint>

namespace fbq {

constexpr int kTopkThreads = 1024;

__device__ __forceinline__ uint64_t topk_key(const float* scores, int64_t i) {
  return ((uint64_t)__float_as_uint(scores[i]) << 32) | (uint64_t)(0xFFFFFFFFu - (uint32_t)i);
}

__global__ void __launch_bounds__(kTopkThreads)
fbq_topk_kernel(const float* scores, int64_t n, int64_t k, uint32_t* mask_bits, int32_t* count) {
  __shared__ unsigned int hist[256];
  __shared__ uint64_t s_prefix;
  __shared__ int64_t s_need;
  const int tid = threadIdx.x;
  const int64_t words = (n + 31) / 32;
  for (int64_t i = tid; i < words; i += kTopkThreads) mask_bits[i] = 0u;
  if (tid == 0 && count) *count = (int32_t)k;
  if (k <= 0) return;
  uint64_t prefix = 0, pmask = 0;
  int64_t need = k;  // rank of the wanted key among those matching the prefix
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (int b = tid; b < 256; b += kTopkThreads) hist[b] = 0u;
    __syncthreads();
    for (int64_t i = tid; i < n; i += kTopkThreads) {
      const uint64_t key = topk_key(scores, i);
      if ((key & pmask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (tid == 0) {
      int64_t above = 0;
      int b = 255;
      for (; b > 0; --b) {
        if (above + (int64_t)hist[b] >= need) break;
        above += hist[b];
      }
      s_need = need - above;
      s_prefix = prefix | ((uint64_t)b << shift);
    }
    __syncthreads();
    prefix = s_prefix;
    need = s_need;
    pmask |= (uint64_t)255u << shift;
    __syncthreads();
  }
  __syncthreads();  // mask words zeroed by every thread before the marking
  // prefix is now the exact k-th largest key: mark the k keys >= it
  for (int64_t i = tid; i < n; i += kTopkThreads)
    if (topk_key(scores, i) >= prefix) atomicOr(mask_bits + (i >> 5), 1u << (i & 31));
}

cudaError_t launch_topk(const float* scores, int64_t n, int64_t k, uint32_t* mask_bits,
                        int32_t* count, cudaStream_t s) {
  fbq_topk_kernel<<<1, kTopkThreads, 0, s>>>(scores, n, k, mask_bits, count);
  return cudaGetLastError();
}

}  // namespace fbq
