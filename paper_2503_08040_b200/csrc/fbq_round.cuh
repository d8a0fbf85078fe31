// Bit-exact rounding primitives shared by the quantizer kernels.
//
// The reference quantizes with a DOUBLE divide + nearbyint
// (kernels.cpp:24-40 / kernels_avx2.cpp:42-77) and stochastic-rounds with a
// double divide + floor + splitmix64 uniform (quant.cpp:66-80, rng.hpp:11-35).
// Double division would cost ~10-20 FP64 instructions per element and make the
// HBM-bound quantizers issue-bound, so we compute the same results from an
// fp32 reciprocal estimate plus an EXACT fp32 FMA remainder:
//
//   n   = rint(x * (1/a))            (|x/a - n| <= 1/2 + 2^-16)
//   rem = fma(-n, a, x)              exact: x - n*a is representable
//   2|rem| >  a  -> n += sign(rem)   (n was off by one)
//   2|rem| == a  -> exact tie x/a = n +- 1/2: pick the even neighbour
//
// A double rounding of x/a to 53 bits can neither create nor break a tie
// (x and a have 24-bit significands, so a non-tie quotient is >= 2^-31
// relatively away from any half-integer), hence the reference result equals
// round_half_even(exact x/a), which the above computes.  Blocks whose scale
// is tiny enough that 1/a could overflow take the plain double path.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace fbq {

constexpr int kBlock = 128;  // quantization block side (SPEC.md gemm module, §4.5)
constexpr int kLevel = 127;  // L = 2^(8-1) - 1 for b = 8 (quant.hpp:16)
constexpr float kTinyScale = 0x1p-120f;

// a = amax > 0 ? fl(amax / 127) : 0        (quant.cpp:27-32, IEEE RN divide)
__device__ __forceinline__ float block_scale(float amax) {
  return amax > 0.0f ? __fdiv_rn(amax, 127.0f) : 0.0f;
}

// clamp(round_half_even(x / a), -L, L); a > 0.   kernels.cpp:24-40
// (L = 127 for the 8-bit GEMM operands, 511 for the 10-bit non-linear contexts)
// Slow path for scales so small that 1/a could overflow: the reference formula.
__device__ __noinline__ int rtn_code_slow(float x, float a, float level) {
  const float n = (float)rint(__ddiv_rn((double)x, (double)a));
  return (int)fminf(fmaxf(n, -level), level);
}
// Branch-free fast path (a >= kTinyScale).  Rounding goes through the
// "magic" constant M = 1.5 * 2^23: fl(t + M) rounds t to the nearest integer
// with ties to even (|t| < 2^22), as_int(fl(t + M)) - as_int(M) is that integer
// and fl(fl(t + M) - M) is it as a float -- FADD/IADD only, no F2I/FRND
// (conversion-pipe) instructions.
constexpr float kMagic = 12582912.0f;   // 1.5 * 2^23
constexpr int kMagicBits = 0x4B400000;
__device__ __forceinline__ int rtn_code_fast(float x, float a, float inv_a, float level) {
  const float m = __fadd_rn(__fmul_rn(x, inv_a), kMagic);
  const float n = __fsub_rn(m, kMagic);
  int ni = __float_as_int(m) - kMagicBits;
  const float rem = __fmaf_rn(-n, a, x);  // exact
  const float two = __fadd_rn(fabsf(rem), fabsf(rem));
  // off by one, or an exact tie x/a = n +- 1/2 with n odd: step toward x
  const bool step = (two > a) | ((two == a) & ((ni & 1) != 0));
  ni += step ? (rem > 0.0f ? 1 : -1) : 0;
  const int L = (int)level;
  return min(max(ni, -L), L);
}
__device__ __forceinline__ int rtn_code(float x, float a, float inv_a, float level = 127.0f) {
  return a >= kTinyScale ? rtn_code_fast(x, a, inv_a, level) : rtn_code_slow(x, a, level);
}

// splitmix64 finalizer (rng.hpp:11-15)
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;  // rng.hpp:29

// Stochastic rounding of x/a given the element's 64 RNG bits
// (bits_at(lin), rng.hpp:28-35): reference quant.cpp:69-77
//   t = RN53(x/a); f = floor(t); frac = t - f;
//   if (frac > 0 && uniform(lin) < frac) f += 1; clamp(+-127)
// Fast path decides u < frac with an fp32 estimate whenever the two are more
// than 2^-20 apart (the estimate's error is < 2^-21); otherwise (probability
// ~2^-19 per element) it recomputes the reference's double formula exactly,
// out of line so the unrolled fast path stays small.
__device__ __noinline__ int sr_code_slow(float x, float a, uint64_t bits) {
  const double t = __ddiv_rn((double)x, (double)a);
  double fd = floor(t);
  const double frac = t - fd;
  const double u = (double)(bits >> 11) * 0x1.0p-53;
  if (frac > 0.0 && u < frac) fd += 1.0;
  return (int)fmin(fmax(fd, -127.0), 127.0);
}
__device__ __forceinline__ int sr_code(float x, float a, float inv_a, uint64_t bits) {
  if (a < kTinyScale) return sr_code_slow(x, a, bits);
  // nearest integer via the magic constant, then one exact-remainder correction
  // turns it into floor(x/a) with 0 <= rem < a
  const float m = __fadd_rn(__fmul_rn(x, inv_a), kMagic);
  float n0 = __fsub_rn(m, kMagic);
  int ni = __float_as_int(m) - kMagicBits;
  float rem = __fmaf_rn(-n0, a, x);
  const bool neg = rem < 0.0f;
  n0 = neg ? n0 - 1.0f : n0;
  ni -= neg ? 1 : 0;
  rem = neg ? __fmaf_rn(-n0, a, x) : rem;
  const float frac = __fmul_rn(rem, inv_a);
  // u ~ (bits >> 11) * 2^-53 to 2^-23 from the top mantissa bits (no I2F):
  // as_float(0x3F800000 | top 23 bits) - 1 is in [0, 1)
  const float u = __fsub_rn(__uint_as_float(0x3F800000u | (uint32_t)(bits >> 41)), 1.0f);
  const float d = u - frac;
  if (fabsf(d) <= 0x1p-20f) return sr_code_slow(x, a, bits);
  ni += (rem > 0.0f && d < 0.0f) ? 1 : 0;
  return min(max(ni, -127), 127);
}

// ------------------------------------------------------------------ vectors
// Vector fast paths for a block-uniform scale a >= kTinyScale.  Each returns
// the biased magic words m = fl(t + M) (their low byte / halfword IS the code
// in two's complement: M's low 22 bits are zero) and a "near" flag: true when
// some element's fp32 estimate lies within `window` of a rounding boundary,
// where the estimate cannot decide -- the caller then redoes that vector with
// the exact scalar functions above (probability ~2^-12 per element).
//
// RTN: q = fl(x * inv_a) is within |x/a| * 2^-23 < level * 2^-23 of x/a
// (|x| <= amax by construction, so |x/a| <= level * (1 + 2^-24) and the clamp
// is a no-op); d = q - rint(q) is exact.  |d| <= 1/2 - level * 2^-21 proves
// rint(q) == round_half_even(x/a) with no tie.
__device__ __forceinline__ float rtn_window(float level) { return 0.5f - level * 0x1p-21f; }

template <int V>
__device__ __forceinline__ bool rtn_fast_vec(const float (&x)[V], float inv_a, float window,
                                             uint32_t (&w)[V]) {
  if constexpr (V % 2 == 0) {
    // element pairs on the packed FP32 pipe (FMUL2 / FADD2 / FFMA2): q, m,
    // n = m - M (exact), d = q - n (exact, |d| <= 1/2) -- 4 instructions per
    // pair -- and one 3-input max of |d| per pair for the boundary test
    const float2 inv2 = make_float2(inv_a, inv_a);
    const float2 mag = make_float2(kMagic, kMagic), nmag = make_float2(-kMagic, -kMagic);
    const float2 neg1 = make_float2(-1.0f, -1.0f);
    float dm = 0.0f;
#pragma unroll
    for (int i = 0; i < V; i += 2) {
      const float2 q = __fmul2_rn(make_float2(x[i], x[i + 1]), inv2);
      const float2 m = __fadd2_rn(q, mag);
      const float2 n = __fadd2_rn(m, nmag);
      const float2 d = __ffma2_rn(n, neg1, q);
      dm = fmaxf(dm, fmaxf(fabsf(d.x), fabsf(d.y)));
      w[i] = __float_as_uint(m.x);
      w[i + 1] = __float_as_uint(m.y);
    }
    return dm > window;
  }
  bool near = false;
#pragma unroll
  for (int i = 0; i < V; ++i) {
    const float q = __fmul_rn(x[i], inv_a);
    const float m = __fadd_rn(q, kMagic);
    const float d = __fsub_rn(q, __fsub_rn(m, kMagic));
    near |= fabsf(d) > window;
    w[i] = __float_as_uint(m);
  }
  return near;
}
// The same fast path with an exact-remainder boundary test (even V): the
// window above must cover fl(x * inv_a)'s error, |x/a| 2^-23 (up to ~2^-16),
// so on bf16 inputs -- whose x/a cluster at half-integers perturbed only by a's
// own rounding -- about 20 % of 8-element vectors fired the exact fix.  Here
//   r = fma(-n, a, x)   exact (x - n a is a multiple of min(ulp x, ulp a), |r| <~ a)
//   d = fl(r * inv_a)   |d - r/a| <= |r/a| (2^-24 + 2^-24) < 2^-23.4
// so |d| <= 1/2 - 2^-22 proves |x/a - n| < 1/2: n is the unique nearest
// integer and no tie -- one extra FMUL2 per pair, and only exact ties and
// true near-ties within ~2^-22 fire.  Same words / flag contract as above.
constexpr float kRemWindow = 0.5f - 0x1p-22f;
template <int V>
__device__ __forceinline__ bool rtn_fast_vec_x(const float (&x)[V], float a, float inv_a, uint32_t (&w)[V]) {
  static_assert(V % 2 == 0, "pairs");
  const float2 inv2 = make_float2(inv_a, inv_a), na2 = make_float2(-a, -a);
  const float2 mag = make_float2(kMagic, kMagic), nmag = make_float2(-kMagic, -kMagic);
  float dm = 0.0f;
#pragma unroll
  for (int i = 0; i < V; i += 2) {
    const float2 xv = make_float2(x[i], x[i + 1]);
    const float2 m = __fadd2_rn(__fmul2_rn(xv, inv2), mag);
    const float2 r = __ffma2_rn(__fadd2_rn(m, nmag), na2, xv);  // exact remainder
    const float2 d = __fmul2_rn(r, inv2);
    dm = fmaxf(dm, fmaxf(fabsf(d.x), fabsf(d.y)));
    w[i] = __float_as_uint(m.x);
    w[i + 1] = __float_as_uint(m.y);
  }
  return dm > kRemWindow;
}

// Exact correction of rtn_fast_vec's words in place, for vectors whose
// boundary test fired (~20 % of bf16 vectors: a bf16 value sitting near a
// tie repeats many times in a block).  Same arithmetic as rtn_code_fast --
// n = m - M, exact remainder r = x - n a, step toward r when 2|r| > a or on
// an exact tie with n odd -- on element pairs and inline (no call frame): the
// code is the low byte / halfword of m + step.  |x| <= amax keeps the result
// inside +-level, so no clamp is needed.
template <int V>
__device__ __forceinline__ void rtn_fix_vec(const float (&x)[V], float a, uint32_t (&w)[V]) {
  static_assert(V % 2 == 0, "pairs");
  const float2 nmag = make_float2(-kMagic, -kMagic), na = make_float2(-a, -a);
#pragma unroll
  for (int i = 0; i < V; i += 2) {
    const float2 n = __fadd2_rn(make_float2(__uint_as_float(w[i]), __uint_as_float(w[i + 1])), nmag);
    const float2 r = __ffma2_rn(n, na, make_float2(x[i], x[i + 1]));  // exact
    const float2 r2 = __fadd2_rn(r, r);                                // exact
    // step toward r iff 2|r| > a, or 2|r| == a with n odd: t = 2|r| - a is
    // exact (Sterbenz; |2r| <= a (1 + 2^-15)) or, when 2|r| < a/2, still
    // negative with |t| >= 2^-144 (a >= kTinyScale); adding the denormal
    // 2^-149 * (n & 1) turns the tie into "> 0" exactly when n is odd.
    const float t0 = __fadd_rn(__fadd_rn(fabsf(r2.x), -a), __uint_as_float(w[i] & 1u));
    const float t1 = __fadd_rn(__fadd_rn(fabsf(r2.y), -a), __uint_as_float(w[i + 1] & 1u));
    const uint32_t sg0 = (__float_as_uint(r2.x) >> 31) ? 0xFFFFFFFFu : 1u;  // sign(r) as +-1
    const uint32_t sg1 = (__float_as_uint(r2.y) >> 31) ? 0xFFFFFFFFu : 1u;
    w[i] += t0 > 0.0f ? sg0 : 0u;
    w[i + 1] += t1 > 0.0f ? sg1 : 0u;
  }
}
template <int V>
__device__ __forceinline__ void rtn_exact_vec(const float (&x)[V], float a, float inv_a,
                                              float level, uint32_t (&w)[V]) {
#pragma unroll
  for (int i = 0; i < V; ++i) w[i] = (uint32_t)rtn_code_fast(x[i], a, inv_a, level);
}

// Top 32 bits of mix64(z) (exact for bits 33..63, the only ones the fast SR
// path uses): the final z ^ (z >> 31) leaves them unchanged, and only the
// high word of the second 64-bit product is needed.
__device__ __forceinline__ uint32_t mix64_hi(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = z ^ (z >> 27);
  const uint32_t lo = (uint32_t)z, hi = (uint32_t)(z >> 32);
  return __umulhi(lo, 0x133111EBu) + lo * 0x94D049BBu + hi * 0x133111EBu;
}

// Stochastic rounding (quant.cpp:69-77):  floor(t) + [frac > 0 && u < frac]
// == rint(t + 1/2 - u) unless t + 1/2 - u is (within rounding error of) a
// half-integer -- i.e. u == frac, or frac == 0 with u == 0.  The fp32
// w = fl(fl(x * inv_a) + (1/2 - u23)) is within 2^-15 of t + 1/2 - u53 (u23:
// the top 23 RNG bits, exactly 1/2 - u23 = 1.5 - as_float(0x3F800000 | bits));
// near boundaries (window 2^-13) or |w| > 127.25 (a possible clamp) the vector
// is redone exactly.  z: the element's splitmix64 counter (seed + lin * golden).
template <int V>
__device__ __forceinline__ bool sr_fast_vec(const float (&x)[V], float inv_a, uint64_t z,
                                            uint32_t (&w)[V]) {
  if constexpr (V % 2 == 0) {
    // the float part on element pairs (FADD2 / FMUL2 / FFMA2, 3-input max)
    const float2 inv2 = make_float2(inv_a, inv_a);
    const float2 mag = make_float2(kMagic, kMagic), nmag = make_float2(-kMagic, -kMagic);
    const float2 neg1 = make_float2(-1.0f, -1.0f), c15 = make_float2(1.5f, 1.5f);
    float dm = 0.0f, tm = 0.0f;
#pragma unroll
    for (int i = 0; i < V; i += 2) {
      const uint32_t h0 = mix64_hi(z);
      const uint32_t h1 = mix64_hi(z + kGolden);
      z += 2 * kGolden;
      const float2 u = make_float2(__uint_as_float(0x3F800000u | (h0 >> 9)),
                                   __uint_as_float(0x3F800000u | (h1 >> 9)));
      const float2 half_u = __ffma2_rn(u, neg1, c15);  // 1.5 - u, exact
      const float2 t = __fadd2_rn(__fmul2_rn(make_float2(x[i], x[i + 1]), inv2), half_u);
      const float2 m = __fadd2_rn(t, mag);
      const float2 d = __ffma2_rn(__fadd2_rn(m, nmag), neg1, t);
      dm = fmaxf(dm, fmaxf(fabsf(d.x), fabsf(d.y)));
      tm = fmaxf(tm, fmaxf(fabsf(t.x), fabsf(t.y)));
      w[i] = __float_as_uint(m.x);
      w[i + 1] = __float_as_uint(m.y);
    }
    return (dm > 0.5f - 0x1p-13f) | (tm > 127.25f);
  }
  bool near = false;
#pragma unroll
  for (int i = 0; i < V; ++i) {
    const uint32_t h = mix64_hi(z);
    const float half_u = __fsub_rn(1.5f, __uint_as_float(0x3F800000u | (h >> 9)));
    const float t = __fadd_rn(__fmul_rn(x[i], inv_a), half_u);
    const float m = __fadd_rn(t, kMagic);
    const float d = __fsub_rn(t, __fsub_rn(m, kMagic));
    near |= (fabsf(d) > 0.5f - 0x1p-13f) | (fabsf(t) > 127.25f);
    w[i] = __float_as_uint(m);
    z += kGolden;
  }
  return near;
}
template <int V>
__device__ __forceinline__ void sr_exact_vec(const float (&x)[V], float a, float inv_a, uint64_t z,
                                             uint32_t (&w)[V]) {
#pragma unroll
  for (int i = 0; i < V; ++i) {
    w[i] = (uint32_t)sr_code(x[i], a, inv_a, mix64(z));
    z += kGolden;
  }
}

}  // namespace fbq
