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

// mask_threshold (policy.cpp:73-80): bit i = scores[i] > theta (strict, in
// double), packed 32 per word by warp ballots; one CTA also sums the flagged
// blocks (the mask_rate numerator, policy.cpp:82-87) -- deterministic, nothing
// to pre-zero.
__global__ void __launch_bounds__(kTopkThreads)
fbq_threshold_kernel(const double* scores, int64_t n, double theta, uint32_t* mask_bits, int32_t* count) {
  __shared__ int32_t s_count[kTopkThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t words = (n + 31) / 32;
  int32_t c = 0;
  for (int64_t w = warp; w < words; w += kTopkThreads / 32) {
    const int64_t i = w * 32 + lane;
    const uint32_t bits = __ballot_sync(0xffffffffu, i < n && scores[i] > theta);
    if (lane == 0) {
      mask_bits[w] = bits;
      c += __popc(bits);
    }
  }
  if (lane == 0) s_count[warp] = c;
  __syncthreads();
  if (threadIdx.x == 0 && count) {
    int32_t t = 0;
    for (int i = 0; i < kTopkThreads / 32; ++i) t += s_count[i];
    *count = t;
  }
}

cudaError_t launch_threshold(const double* scores, int64_t n, double theta, uint32_t* mask_bits,
                             int32_t* count, cudaStream_t s) {
  fbq_threshold_kernel<<<1, kTopkThreads, 0, s>>>(scores, n, theta, mask_bits, count);
  return cudaGetLastError();
}

// controller_update (policy.cpp:97-109) on an observed rate held in device memory
__global__ void fbq_controller_rate_kernel(double* theta, const double* rate, double r_min, double r_max,
                                           double alpha, double* last_rate) {
  const double r = *rate;
  if (r < r_min) *theta /= alpha;
  else if (r > r_max) *theta *= alpha;
  if (last_rate) *last_rate = r;
}

cudaError_t launch_controller_rate(double* theta, const double* rate, double r_min, double r_max,
                                   double alpha, double* last_rate, cudaStream_t s) {
  fbq_controller_rate_kernel<<<1, 1, 0, s>>>(theta, rate, r_min, r_max, alpha, last_rate);
  return cudaGetLastError();
}

// QuantLinearLayer::apply_sgd (trainsim.cpp:137-143): w -= float(lr * double(g))
__device__ __forceinline__ float sgd_elem(float w, float g, double lr) {
  return __fsub_rn(w, (float)(lr * (double)g));
}
// 16-byte vectors, four per thread per iteration (loads issued together) when
// both pointers are 16-byte aligned; the scalar loop covers the rest
__global__ void fbq_sgd_kernel(float* w, const float* g, int64_t n, double lr) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  int64_t done = 0;
  if (((reinterpret_cast<uintptr_t>(w) | reinterpret_cast<uintptr_t>(g)) & 15u) == 0) {
    const int64_t nv = n / 4;
    float4* w4 = reinterpret_cast<float4*>(w);
    const float4* g4 = reinterpret_cast<const float4*>(g);
    for (int64_t i = tid; i < nv; i += 4 * nth) {
      float4 wv[4], gv[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int64_t j = i + k * nth;
        if (j < nv) {
          wv[k] = __ldcs(w4 + j);
          gv[k] = __ldcs(g4 + j);
        }
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int64_t j = i + k * nth;
        if (j < nv)
          __stcs(w4 + j, make_float4(sgd_elem(wv[k].x, gv[k].x, lr), sgd_elem(wv[k].y, gv[k].y, lr),
                                     sgd_elem(wv[k].z, gv[k].z, lr), sgd_elem(wv[k].w, gv[k].w, lr)));
      }
    }
    done = nv * 4;
  }
  for (int64_t i = done + tid; i < n; i += nth) w[i] = sgd_elem(w[i], g[i], lr);
}

cudaError_t launch_sgd(float* w, const float* g, int64_t n, double lr, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  int64_t blocks = (n / 4 + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (blocks < 1) blocks = 1;
  fbq_sgd_kernel<<<(unsigned)blocks, 256, 0, s>>>(w, g, n, lr);
  return cudaGetLastError();
}

}  // namespace fbq
