// Fallback-quantized SwiGLU MLP driver (include/fbq_b200_host.h).
//
// Mirrors the reference composition of QuantLinearLayer (trainsim.cpp:61-127)
// and GluCombine (trainsim.cpp:224-263) for gate/up/down, re-planned for B200:
//   forward   RTN(W_gu), RTN(W_d)                         2 x K1
//             K1(X): fallback codes + 2 SR contexts       1 read of X
//             [a|b] = fallback_gemm(X, W_gu^T)            K3, one GEMM for gate+up
//             GLU fwd fused with K1(h)                    h never materialised
//             y = fallback_gemm(h, W_d^T)                 K3
//   backward  K2(dY) -> dH = bqg(dY, W_d) ; dW_d += bqg(dY^T, ctx_h)
//             GLU bwd fused with K2(ga), K2(gb)
//             dX = bqg(ga, W_g) + bqg(gb, W_u)            (accumulate = the reference's add)
//             dW_g += bqg(ga^T, ctx_g) ; dW_u += bqg(gb^T, ctx_u)
// Every operand is consumed in the layout it was produced in: the backward
// GEMMs read the forward code planes MN-major instead of transposing them.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <algorithm>
#include <vector>

#include "../../../include/fbq_b200_host.h"

namespace {

struct CudaError : std::runtime_error {
  int status;
  CudaError(int st, const std::string& w) : std::runtime_error(w), status(st) {}
};

#define FBQ_TRY(expr)                                                     \
  do {                                                                    \
    int _st = (expr);                                                     \
    if (_st != FBQ_OK) throw CudaError(_st, #expr);                       \
  } while (0)
#define CU_TRY(expr)                                                      \
  do {                                                                    \
    cudaError_t _e = (expr);                                              \
    if (_e != cudaSuccess) throw CudaError(FBQ_ERR_CUDA, cudaGetErrorString(_e)); \
  } while (0)

int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }
int64_t ld16(int64_t n) { return (n + 15) / 16 * 16; }

// rng.hpp:11-58 / trainsim.cpp:16-19
uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
uint64_t bits_at(uint64_t seed, uint64_t n) { return mix64(seed + (n + 1) * 0x9E3779B97F4A7C15ull); }
uint64_t layer_seed(uint64_t base, int layer, uint64_t tag, int step) {
  return bits_at(bits_at(base, (uint64_t)layer * 4 + tag), (uint64_t)step);
}

struct DevBuf {
  void* p = nullptr;
  DevBuf() = default;
  explicit DevBuf(size_t bytes) {
    if (bytes) CU_TRY(cudaMalloc(&p, bytes));
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p) { o.p = nullptr; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    std::swap(p, o.p);
    return *this;
  }
  template <class T>
  T* as() const { return static_cast<T*>(p); }
};

size_t esize(int dt) { return dt == FBQ_F32 ? 4 : 2; }

struct Mlp {
  fbq_mlp_config c;
  int64_t D, F, T;            // d_model, d_ff, max tokens
  int64_t ldD, ldF, ldF2;     // int8 plane strides
  int64_t gD, gF, gT;         // grid extents (blocks)
  // weights (fp32 master) and gradients
  DevBuf w_gu, w_d, g_gu, g_d;
  // quantized weights
  DevBuf wgu_codes, wgu_scales, wd_codes, wd_scales;
  // forward X quantization
  DevBuf x_codes, x_scales, x_res, x_res_scales, x_mask, ctx_g, ctx_u;
  // [a|b], GLU contexts, h quantization
  DevBuf ab, ctx_a, ctx_b, ctx_a_s, ctx_b_s, h_codes, h_scales, h_res, h_res_scales, h_mask, ctx_h;
  // backward
  DevBuf gy_codes, gy_scales, gh, gq, gq_scales;
  // controller state on device: theta[2], count[2], rate[2]
  DevBuf theta, counts, rates;
  // host e2e staging
  DevBuf hx, hgy, hy, hgx;
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t ev_x = nullptr, ev_gy = nullptr, ev_fwd = nullptr, ev_bwd = nullptr;
  cudaEvent_t ev_grad[3] = {nullptr, nullptr, nullptr};  // dW_gate, dW_up, dW_down final
  // backward side stream: the dW GEMMs run there, so each GEMM's last-wave
  // tail (up to one 224-k-block tile on the long-K dX) is filled by the next
  // independent grid's CTAs instead of idling SMs
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork[2] = {nullptr, nullptr}, ev_join = nullptr;
  // forward: the weight quantizations run on the side stream, overlapping the
  // (issue-bound) X quantizer, the gate/up GEMM's tail and the GLU forward
  cudaEvent_t ev_ffork = nullptr, ev_wgu = nullptr, ev_wd = nullptr;

  Mlp(const fbq_mlp_config& cfg, const float* wg, const float* wu, const float* wd) : c(cfg) {
    D = c.d_model;
    F = c.d_ff;
    T = c.max_tokens;
    if (D <= 0 || F <= 0 || T <= 0) throw CudaError(FBQ_ERR_SHAPE, "bad MLP shape");
    // d_ff % 128: the concatenated [gate; up] planes must not share a block
    if (D % 16 || F % 128) throw CudaError(FBQ_ERR_UNSUPPORTED, "need d_model % 16 == 0 and d_ff % 128 == 0");
    FBQ_TRY(fbq_cuda_init());  // per-device setup (GEMM tile-counter ring) before any launch
    ldD = ld16(D);
    ldF = ld16(F);
    ldF2 = ld16(2 * F);
    gD = cdiv(D, 128);
    gF = cdiv(F, 128);
    gT = cdiv(T, 128);
    const size_t f4 = 4;
    w_gu = DevBuf(2 * F * D * f4);
    w_d = DevBuf(D * F * f4);
    g_gu = DevBuf(2 * F * D * f4);
    g_d = DevBuf(D * F * f4);
    CU_TRY(cudaMemcpy(w_gu.p, wg, F * D * f4, cudaMemcpyHostToDevice));
    CU_TRY(cudaMemcpy(w_gu.as<float>() + F * D, wu, F * D * f4, cudaMemcpyHostToDevice));
    CU_TRY(cudaMemcpy(w_d.p, wd, D * F * f4, cudaMemcpyHostToDevice));
    CU_TRY(cudaMemset(g_gu.p, 0, 2 * F * D * f4));
    CU_TRY(cudaMemset(g_d.p, 0, D * F * f4));
    wgu_codes = DevBuf(2 * F * ldD);
    wgu_scales = DevBuf(cdiv(2 * F, 128) * gD * f4);
    wd_codes = DevBuf(D * ldF);
    wd_scales = DevBuf(gD * gF * f4);
    x_codes = DevBuf(T * ldD);
    x_res = DevBuf(T * ldD);
    ctx_g = DevBuf(T * ldD);
    ctx_u = DevBuf(T * ldD);
    x_scales = DevBuf(gT * gD * f4);
    x_res_scales = DevBuf(gT * gD * f4);
    x_mask = DevBuf(cdiv(gT * gD, 32) * 4);
    ab = DevBuf(T * 2 * F * esize(c.mid_dtype));
    // a / b contexts: int16 codes or packed 10-bit planes (1.25 B per element,
    // fbq_ctx10_bytes; the plane layout follows the call's row count, so the
    // buffers are sized for the capacity)
    if (c.ctx_format != FBQ_CTX_INT16 && c.ctx_format != FBQ_CTX_PACKED10)
      throw CudaError(FBQ_ERR_ARG, "bad ctx_format");
    if (c.ctx_format == FBQ_CTX_PACKED10 && c.nonlinear_bits > 10)
      throw CudaError(FBQ_ERR_UNSUPPORTED, "nonlinear_bits > 10 with packed 10-bit contexts");
    ctx_a = DevBuf(ctx_bytes(T) + 16);
    ctx_b = DevBuf(ctx_bytes(T) + 16);
    ctx_a_s = DevBuf(T * gF * f4);
    ctx_b_s = DevBuf(T * gF * f4);
    h_codes = DevBuf(T * ldF);
    h_res = DevBuf(T * ldF);
    ctx_h = DevBuf(T * ldF);
    h_scales = DevBuf(gT * gF * f4);
    h_res_scales = DevBuf(gT * gF * f4);
    h_mask = DevBuf(cdiv(gT * gF, 32) * 4);
    gy_codes = DevBuf(T * ldD);
    gy_scales = DevBuf(gT * gD * f4);
    gh = DevBuf(T * F * esize(c.mid_dtype));
    gq = DevBuf(T * ldF2);
    gq_scales = DevBuf(gT * 2 * gF * f4);
    theta = DevBuf(2 * sizeof(double));
    counts = DevBuf(2 * sizeof(int32_t));
    rates = DevBuf(2 * sizeof(double));
    const double th[2] = {c.threshold_init, c.threshold_init};
    CU_TRY(cudaMemcpy(theta.p, th, sizeof(th), cudaMemcpyHostToDevice));
    CU_TRY(cudaMemset(counts.p, 0, 2 * sizeof(int32_t)));
    CU_TRY(cudaMemset(rates.p, 0, 2 * sizeof(double)));
    CU_TRY(cudaStreamCreateWithFlags(&copy_stream, cudaStreamNonBlocking));
    CU_TRY(cudaEventCreateWithFlags(&ev_x, cudaEventDisableTiming));
    CU_TRY(cudaEventCreateWithFlags(&ev_gy, cudaEventDisableTiming));
    CU_TRY(cudaEventCreateWithFlags(&ev_fwd, cudaEventDisableTiming));
    CU_TRY(cudaEventCreateWithFlags(&ev_bwd, cudaEventDisableTiming));
    for (cudaEvent_t* e : {&ev_grad[0], &ev_grad[1], &ev_grad[2], &ev_fork[0], &ev_fork[1], &ev_join, &ev_ffork, &ev_wgu, &ev_wd,
                           &ev_gyq})
      CU_TRY(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    CU_TRY(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
  }

  ~Mlp() {
    if (a_cs) {
      cudaStreamSynchronize(a_cs);
      cudaStreamSynchronize(a_d2h);
    }
    async_free();
    for (cudaEvent_t e : ev_pool) cudaEventDestroy(e);
    if (copy_stream) cudaStreamDestroy(copy_stream);
    if (side) cudaStreamDestroy(side);
    for (cudaEvent_t e : {ev_x, ev_gy, ev_fwd, ev_bwd, ev_grad[0], ev_grad[1], ev_grad[2], ev_fork[0], ev_fork[1], ev_join,
                          ev_ffork, ev_wgu, ev_wd, ev_gyq})
      if (e) cudaEventDestroy(e);
  }

  int layer(int i) const { return c.layer_id_base + i; }  // 0 gate, 1 up, 2 down
  // reference-exact non-linear math in parity mode (fp32 intermediates)
  int exact_math() const { return c.mid_dtype == FBQ_F32 ? 1 : 0; }

  // ---- launch accounting and optional per-GEMM CUDA-event timing ----
  int64_t launches = 0;        // our kernels launched (K1/K2/K3/GLU/controller)
  bool profiling = false;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  cudaEvent_t next_event() {
    if (ev_used == ev_pool.size()) {
      cudaEvent_t e;
      CU_TRY(cudaEventCreate(&e));
      ev_pool.push_back(e);
    }
    return ev_pool[ev_used++];
  }
  template <class Fn>
  void gemm(Fn&& launch, cudaStream_t s) {
    if (profiling) CU_TRY(cudaEventRecord(next_event(), s));
    FBQ_TRY(launch());
    if (profiling) CU_TRY(cudaEventRecord(next_event(), s));
    ++launches;
  }
  // GEMM busy time: the union of the [start, end] intervals (GEMMs on the
  // backward side stream overlap the main stream's), relative to the first event
  double gemm_ms_and_reset() {
    std::vector<std::pair<float, float>> iv;
    for (size_t i = 0; i + 1 < ev_used; i += 2) {
      float a = 0.f, b = 0.f;
      CU_TRY(cudaEventElapsedTime(&a, ev_pool[0], ev_pool[i]));
      CU_TRY(cudaEventElapsedTime(&b, ev_pool[0], ev_pool[i + 1]));
      iv.emplace_back(a, b);
    }
    std::sort(iv.begin(), iv.end());
    double total = 0.0, cs = -1e30, ce = -1e30;
    for (auto& [a, b] : iv) {
      if (a > ce) {
        if (ce > cs) total += ce - cs;
        cs = a;
        ce = b;
      } else if (b > ce) {
        ce = b;
      }
    }
    if (ce > cs) total += ce - cs;
    ev_used = 0;
    return total;
  }

  // GluBlock (below): the block's RmsNorm fused into the gate/up input quantizer
  struct NormIn {
    const float* gain;
    int16_t* ctx;
    int64_t ld_ctx;
    float* ctx_scales;
    float* rms_ws;
  };
  // norm: quantize norm(x) instead of x (the RmsNorm context is written too);
  // residual: y = fl(x + down(...)) -- x is copied into y and the down GEMM
  // accumulates onto it (GluBlock::forward's add(h, d), trainsim.cpp:294-301)
  void forward(const void* x, int64_t tok, int64_t row_off, int step, void* y, cudaStream_t s,
               const NormIn* norm = nullptr, bool residual = false) {
    if (tok < 0 || tok > T) throw CudaError(FBQ_ERR_SHAPE, "tokens exceed max_tokens");
    if (tok == 0) return;
    const int64_t gTt = cdiv(tok, 128);
    int32_t* cnt = counts.as<int32_t>();
    double* th = theta.as<double>();
    // weights: one RTN quantization serves forward (K-major) and dgrad (MN-major);
    // quantize_rtn(transpose(W)) == transpose(quantize_rtn(W)) (trainsim.cpp:96-97, 121)
    // after a fused apply_sgd the weight codes already hold RTN(W) of the
    // current W (written in the same pass as the update): used once as they are
    const bool w_fresh = w_codes_fresh;
    w_codes_fresh = false;
    launches += w_fresh ? 3 : 5;  // 2 x RTN(W), K1(X), GLU forward (+ the 2 GEMMs counted in gemm())
    // side stream: RTN(W_gate|up) then RTN(W_down), joined right before the
    // GEMM that consumes each
    CU_TRY(cudaEventRecord(ev_ffork, s));
    CU_TRY(cudaStreamWaitEvent(side, ev_ffork, 0));
    if (!w_fresh)
      FBQ_TRY(fbq_cuda_quantize_rtn(w_gu.p, FBQ_F32, 2 * F, D, D, wgu_codes.as<int8_t>(), ldD,
                                    wgu_scales.as<float>(), side));
    CU_TRY(cudaEventRecord(ev_wgu, side));
    if (!w_fresh)
      FBQ_TRY(fbq_cuda_quantize_rtn(w_d.p, FBQ_F32, D, F, F, wd_codes.as<int8_t>(), ldF,
                                    wd_scales.as<float>(), side));
    CU_TRY(cudaEventRecord(ev_wd, side));
    // X: score + threshold mask + fallback codes + gate/up contexts (trainsim.cpp:80-102)
    if (norm) {
      FBQ_TRY(fbq_cuda_rmsnorm_quantize_input(
          x, c.act_dtype, tok, D, D, norm->gain, norm->ctx, norm->ld_ctx, norm->ctx_scales, norm->rms_ws,
          FBQ_MASK_THRESHOLD, c.threshold_init, th, x_mask.as<uint32_t>(), x_codes.as<int8_t>(), ldD,
          x_scales.as<float>(), x_res.as<int8_t>(), x_res_scales.as<float>(), cnt, ctx_g.as<int8_t>(),
          layer_seed(c.seed, layer(0), 0, step), ctx_u.as<int8_t>(), layer_seed(c.seed, layer(1), 0, step),
          row_off, s));
    } else {
      FBQ_TRY(fbq_cuda_quantize_linear_input(
          x, c.act_dtype, tok, D, D, FBQ_MASK_THRESHOLD, c.threshold_init, th,
          x_mask.as<uint32_t>(), x_codes.as<int8_t>(), ldD, x_scales.as<float>(),
          x_res.as<int8_t>(), x_res_scales.as<float>(), cnt, ctx_g.as<int8_t>(),
          layer_seed(c.seed, layer(0), 0, step), ctx_u.as<int8_t>(),
          layer_seed(c.seed, layer(1), 0, step), row_off, s));
    }
    // [a | b] = fallback_gemm(X, [W_g; W_u]^T)
    CU_TRY(cudaStreamWaitEvent(s, ev_wgu, 0));
    gemm([&] { return fbq_cuda_gemm(x_codes.as<int8_t>(), ldD, x_scales.as<float>(), FBQ_K_MAJOR,
                          wgu_codes.as<int8_t>(), ldD, wgu_scales.as<float>(), FBQ_K_MAJOR,
                          x_mask.as<uint32_t>(), x_res.as<int8_t>(), x_res_scales.as<float>(),
                          tok, 2 * F, D, ab.p, c.mid_dtype, 2 * F, 0, c.epilogue, s); }, s);
    // GLU + contexts + quantization of h for the down projection
    FBQ_TRY(fbq_cuda_glu_forward(
        ab.p, c.mid_dtype, tok, F, 2 * F, ctx_a.p, ctx_b.p, ldF, c.ctx_format,
        ctx_a_s.as<float>(), ctx_b_s.as<float>(), c.nonlinear_bits, exact_math(), c.threshold_init, th + 1,
        h_mask.as<uint32_t>(), h_codes.as<int8_t>(), ldF, h_scales.as<float>(),
        h_res.as<int8_t>(), h_res_scales.as<float>(), cnt + 1, ctx_h.as<int8_t>(),
        layer_seed(c.seed, layer(2), 0, step), row_off, nullptr, 0, s));
    // y = fallback_gemm(h, W_d^T)   (GluBlock: y = x + fallback_gemm(...), accumulated onto x)
    if (residual) CU_TRY(cudaMemcpyAsync(y, x, (size_t)tok * D * esize(c.act_dtype), cudaMemcpyDeviceToDevice, s));
    CU_TRY(cudaStreamWaitEvent(s, ev_wd, 0));
    gemm([&] { return fbq_cuda_gemm(h_codes.as<int8_t>(), ldF, h_scales.as<float>(), FBQ_K_MAJOR,
                          wd_codes.as<int8_t>(), ldF, wd_scales.as<float>(), FBQ_K_MAJOR,
                          h_mask.as<uint32_t>(), h_res.as<int8_t>(), h_res_scales.as<float>(),
                          tok, D, F, y, c.act_dtype, D, residual ? 1 : 0, c.epilogue, s); }, s);
    (void)gTt;
  }

  // SR(dY) for the down layer (trainsim.cpp:117-119).  The host-buffer step
  // APIs have dY before the forward runs, so they quantize it on the side
  // stream right after the forward's weight quantizations (it then overlaps
  // the forward) and the backward only waits for it (gy_ready).
  cudaEvent_t ev_gyq = nullptr;
  void quantize_gy(const void* gy, int64_t tok, int64_t row_off, int step, cudaStream_t s) {
    FBQ_TRY(fbq_cuda_quantize_stochastic(gy, c.act_dtype, tok, D, D,
                                         layer_seed(c.seed, layer(2), 1, step), row_off,
                                         gy_codes.as<int8_t>(), ldD, gy_scales.as<float>(), s));
  }
  void quantize_gy_early(const void* gy, int64_t tok, int64_t row_off, int step) {
    if (tok <= 0) return;
    quantize_gy(gy, tok, row_off, step, side);
    CU_TRY(cudaEventRecord(ev_gyq, side));
  }

  // join = false (GluBlock): the caller enqueues more work that needs only dX
  // on `s` first and joins the side stream's dW GEMMs itself (join_side)
  void backward(const void* gy, int64_t tok, int64_t row_off, int step, void* gx,
                cudaStream_t s, bool gy_ready = false, bool join = true) {
    if (tok < 0 || tok > T) throw CudaError(FBQ_ERR_SHAPE, "tokens exceed max_tokens");
    if (tok == 0) return;
    launches += 2;  // K2(dY), GLU backward (+ 6 GEMMs counted in gemm())
    const int acc_w = grad_zero_pending ? 0 : 1;  // dW: write (deferred zero_grad) or accumulate
    grad_zero_pending = false;
    // down: SR(dY) (trainsim.cpp:117-119)
    if (gy_ready) CU_TRY(cudaStreamWaitEvent(s, ev_gyq, 0));
    else quantize_gy(gy, tok, row_off, step, s);
    CU_TRY(cudaEventRecord(ev_fork[0], s));
    CU_TRY(cudaStreamWaitEvent(side, ev_fork[0], 0));
    // dH = bqg(dY, W_d): B = W_d codes (D x F) read MN-major (trainsim.cpp:121-122)
    gemm([&] { return fbq_cuda_gemm(gy_codes.as<int8_t>(), ldD, gy_scales.as<float>(), FBQ_K_MAJOR,
                          wd_codes.as<int8_t>(), ldF, wd_scales.as<float>(), FBQ_MN_MAJOR,
                          nullptr, nullptr, nullptr, tok, F, D, gh.p, c.mid_dtype, F, 0,
                          c.epilogue, s); }, s);
    // dW_d += bqg(dY^T, ctx_h) (trainsim.cpp:124-125), on the side stream
    cudaStream_t b = side;
    gemm([&] { return fbq_cuda_gemm(gy_codes.as<int8_t>(), ldD, gy_scales.as<float>(), FBQ_MN_MAJOR,
                          ctx_h.as<int8_t>(), ldF, h_scales.as<float>(), FBQ_MN_MAJOR, nullptr,
                          nullptr, nullptr, D, F, tok, g_d.p, FBQ_F32, F, acc_w, c.epilogue, b); }, b);
    // dW_d is final for this step: data-parallel callers start its all-reduce
    // on a side stream here, overlapped with the rest of the backward
    CU_TRY(cudaEventRecord(ev_grad[2], b));
    // GLU backward fused with SR(ga), SR(gb)
    FBQ_TRY(fbq_cuda_glu_backward(gh.p, c.mid_dtype, tok, F, F, ctx_a.p, ctx_b.p, ldF, c.ctx_format,
                                  ctx_a_s.as<float>(),
                                  ctx_b_s.as<float>(), gq.as<int8_t>(), ldF2,
                                  gq_scales.as<float>(), layer_seed(c.seed, layer(0), 1, step),
                                  layer_seed(c.seed, layer(1), 1, step), row_off, nullptr,
                                  exact_math(), s));
    CU_TRY(cudaEventRecord(ev_fork[1], s));
    CU_TRY(cudaStreamWaitEvent(side, ev_fork[1], 0));
    // dX = bqg(ga, W_g) + bqg(gb, W_u)   (the reference adds the two layers' dX)
    const int64_t lds_gq = 2 * gF;
    int8_t* gqc = gq.as<int8_t>();
    float* gqs = gq_scales.as<float>();
    if (c.epilogue == FBQ_EPI_EXACT) {
      // the reference's order: fl(bqg(ga, W_g) + bqg(gb, W_u)), two GEMMs
      gemm([&] { return fbq_cuda_gemm_ex(gqc, ldF2, gqs, lds_gq, FBQ_K_MAJOR, wgu_codes.as<int8_t>(), ldD,
                               wgu_scales.as<float>(), gD, FBQ_MN_MAJOR, nullptr, nullptr, nullptr,
                               tok, D, F, gx, c.act_dtype, D, 0,
                               c.epilogue, s); }, s);
      gemm([&] { return fbq_cuda_gemm_ex(gqc + F, ldF2, gqs + gF, lds_gq, FBQ_K_MAJOR,
                               wgu_codes.as<int8_t>() + F * ldD, ldD,
                               wgu_scales.as<float>() + gF * gD, gD, FBQ_MN_MAJOR, nullptr, nullptr,
                               nullptr, tok, D, F, gx, c.act_dtype, D, 1, c.epilogue, s); }, s);
    } else {
      // FMA epilogue (tolerance mode): ONE GEMM over K = 2 d_ff -- [ga | gb]
      // and [W_g; W_u] are already laid out as one operand each (codes and
      // scale grids), so the two products sum in the fp32 accumulator instead
      // of a second GEMM re-reading and re-writing dX
      gemm([&] { return fbq_cuda_gemm_ex(gqc, ldF2, gqs, lds_gq, FBQ_K_MAJOR, wgu_codes.as<int8_t>(), ldD,
                               wgu_scales.as<float>(), gD, FBQ_MN_MAJOR, nullptr, nullptr, nullptr,
                               tok, D, 2 * F, gx, c.act_dtype, D, 0, c.epilogue, s); }, s);
    }
    // dW_g += bqg(ga^T, ctx_g) ; dW_u += bqg(gb^T, ctx_u)   (side stream)
    gemm([&] { return fbq_cuda_gemm_ex(gqc, ldF2, gqs, lds_gq, FBQ_MN_MAJOR, ctx_g.as<int8_t>(), ldD,
                             x_scales.as<float>(), gD, FBQ_MN_MAJOR, nullptr, nullptr, nullptr, F,
                             D, tok, g_gu.p, FBQ_F32, D, acc_w, c.epilogue, b); }, b);
    // dW_gate is final: its all-reduce overlaps the dW_up GEMM
    CU_TRY(cudaEventRecord(ev_grad[0], b));
    gemm([&] { return fbq_cuda_gemm_ex(gqc + F, ldF2, gqs + gF, lds_gq, FBQ_MN_MAJOR, ctx_u.as<int8_t>(),
                             ldD, x_scales.as<float>(), gD, FBQ_MN_MAJOR, nullptr, nullptr,
                             nullptr, F, D, tok, g_gu.as<float>() + F * D, FBQ_F32, D, acc_w,
                             c.epilogue, b); }, b);
    CU_TRY(cudaEventRecord(ev_grad[1], b));
    // join: everything after the backward (controller, next step, readers of
    // dW) is ordered after the side stream's GEMMs
    CU_TRY(cudaEventRecord(ev_join, side));
    if (join) CU_TRY(cudaStreamWaitEvent(s, ev_join, 0));
  }
  void join_side(cudaStream_t s) { CU_TRY(cudaStreamWaitEvent(s, ev_join, 0)); }

  // observed rate = masked blocks / blocks of the last forward (policy.cpp:82-87).
  // Data parallel: the caller sums `counts` over ranks in place and passes the
  // global block counts, so every rank updates theta with the rate of the whole
  // batch (trainsim.cpp:93,129-133) and the thresholds stay identical.
  void controller(cudaStream_t s, int64_t blocks_gu = 0, int64_t blocks_d = 0) {
    launches += 2;
    ctl_blocks[0] = blocks_gu > 0 ? blocks_gu : last_blocks[0];
    ctl_blocks[1] = blocks_d > 0 ? blocks_d : last_blocks[1];
    FBQ_TRY(fbq_cuda_controller_update(theta.as<double>(), counts.as<int32_t>(), ctl_blocks[0],
                                       c.r_min, c.r_max, c.alpha, rates.as<double>(), s));
    FBQ_TRY(fbq_cuda_controller_update(theta.as<double>() + 1, counts.as<int32_t>() + 1,
                                       ctl_blocks[1], c.r_min, c.r_max, c.alpha,
                                       rates.as<double>() + 1, s));
  }
  int64_t last_blocks[2] = {1, 1};
  int64_t ctl_blocks[2] = {0, 0};
  // one a / b context plane at `tok` tokens
  int64_t ctx_bytes(int64_t tok) const {
    return c.ctx_format == FBQ_CTX_PACKED10 ? fbq_ctx10_bytes(tok, ldF) : tok * ldF * 2;
  }  // blocks the last controller step divided by (0: none yet)

  void step_host(const float* x, const float* gy, int64_t tok, int step, float* y, float* gx) {
    if (tok < 0 || tok > T) throw CudaError(FBQ_ERR_SHAPE, "tokens exceed max_tokens");
    if (!hx.p) {
      hx = DevBuf(T * D * 4);
      hgy = DevBuf(T * D * 4);
      hy = DevBuf(T * D * 4);
      hgx = DevBuf(T * D * 4);
    }
    if (tok == 0) return;
    const size_t bytes = tok * D * 4;
    cudaStream_t s = nullptr;  // legacy default stream for compute
    CU_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    struct Guard { cudaStream_t s; ~Guard() { cudaStreamDestroy(s); } } guard{s};
    CU_TRY(cudaMemcpyAsync(hx.p, x, bytes, cudaMemcpyHostToDevice, s));
    CU_TRY(cudaMemcpyAsync(hgy.p, gy, bytes, cudaMemcpyHostToDevice, copy_stream));
    CU_TRY(cudaEventRecord(ev_gy, copy_stream));
    const int saved = c.act_dtype;
    c.act_dtype = FBQ_F32;  // the host API is fp32 like the reference
    try {
      forward(hx.p, tok, 0, step, hy.p, s);
      // SR(dY) on the side stream once dY has landed, overlapping the forward
      CU_TRY(cudaStreamWaitEvent(side, ev_gy, 0));
      quantize_gy_early(hgy.p, tok, 0, step);
      CU_TRY(cudaEventRecord(ev_fwd, s));
      CU_TRY(cudaStreamWaitEvent(copy_stream, ev_fwd, 0));
      CU_TRY(cudaMemcpyAsync(y, hy.p, bytes, cudaMemcpyDeviceToHost, copy_stream));
      CU_TRY(cudaStreamWaitEvent(s, ev_gy, 0));
      backward(hgy.p, tok, 0, step, hgx.p, s, /*gy_ready=*/true);
      CU_TRY(cudaMemcpyAsync(gx, hgx.p, bytes, cudaMemcpyDeviceToHost, s));
    } catch (...) {
      c.act_dtype = saved;
      throw;
    }
    c.act_dtype = saved;
    CU_TRY(cudaStreamSynchronize(s));
    CU_TRY(cudaStreamSynchronize(copy_stream));
  }

  // ---- pipelined host-buffer steps (fbq_mlp_step_host_async) ----
  // Two device slots of (x, dY, y, dX): step i's H2D copies run on their own
  // stream while step i-1 computes, and step i-1's D2H copies (y right after
  // its forward, dX after its backward) overlap step i's compute -- a training
  // loop's batch prefetch.  Each step still moves its own inputs in and its
  // own results out.
  cudaStream_t a_cs = nullptr, a_h2d = nullptr, a_d2h = nullptr;
  DevBuf ax[2], agy[2], ay[2], agx[2];
  cudaEvent_t a_in[2] = {}, a_fwd[2] = {}, a_done[2] = {}, a_out[2] = {};
  bool a_used[2] = {false, false};
  int64_t a_count = 0;

  void async_init() {
    if (a_cs) return;
    CU_TRY(cudaStreamCreateWithFlags(&a_cs, cudaStreamNonBlocking));
    CU_TRY(cudaStreamCreateWithFlags(&a_h2d, cudaStreamNonBlocking));
    CU_TRY(cudaStreamCreateWithFlags(&a_d2h, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i) {
      ax[i] = DevBuf(T * D * 4);
      agy[i] = DevBuf(T * D * 4);
      ay[i] = DevBuf(T * D * 4);
      agx[i] = DevBuf(T * D * 4);
      for (cudaEvent_t* e : {&a_in[i], &a_fwd[i], &a_done[i], &a_out[i]})
        CU_TRY(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    }
  }
  void async_free() {
    for (cudaStream_t st : {a_cs, a_h2d, a_d2h})
      if (st) cudaStreamDestroy(st);
    for (int i = 0; i < 2; ++i)
      for (cudaEvent_t e : {a_in[i], a_fwd[i], a_done[i], a_out[i]})
        if (e) cudaEventDestroy(e);
  }

  // QuantLinearLayer::apply_sgd on gate, up, down (trainsim.cpp:137-143) fused
  // with the RTN quantization of the updated weights (fbq_cuda_sgd_quantize_rtn):
  // W and dW are read once and the next forward uses the codes written here
  // (w_codes_fresh) instead of re-quantizing W.  Only apply_sgd writes W, so the
  // codes stay those of the current W until the forward consumes them.
  bool w_codes_fresh = false;
  double sgd_lr = 0.0;  // the host step API's learning rate (FBQ_STEP_SGD)
  void apply_sgd(double lr, cudaStream_t s) {
    if (grad_zero_pending) return;  // the gradient is (pending) zero: w - float(lr * 0) == w
    launches += 2;
    FBQ_TRY(fbq_cuda_sgd_quantize_rtn(w_gu.as<float>(), g_gu.as<float>(), 2 * F, D, lr,
                                      wgu_codes.as<int8_t>(), ldD, wgu_scales.as<float>(), s));
    FBQ_TRY(fbq_cuda_sgd_quantize_rtn(w_d.as<float>(), g_d.as<float>(), D, F, lr,
                                      wd_codes.as<int8_t>(), ldF, wd_scales.as<float>(), s));
    w_codes_fresh = true;
  }

  // zero_grad is deferred: the next backward's dW GEMMs then WRITE their
  // products instead of reduce-adding them into zeroed buffers (bit-identical:
  // the accumulators are never -0, so fl(0 + x) == x), which saves a 0.7 GB
  // memset per step.  Readers of the gradient buffers flush it first.
  bool grad_zero_pending = false;
  void zero_grad(cudaStream_t) { grad_zero_pending = true; }
  // (device-wide: an earlier backward may still be writing dW on a
  // non-blocking stream, so wait for it before clearing)
  void flush_grad_zero() {
    if (!grad_zero_pending) return;
    CU_TRY(cudaDeviceSynchronize());
    CU_TRY(cudaMemset(g_gu.p, 0, 2 * F * D * 4));
    CU_TRY(cudaMemset(g_d.p, 0, D * F * 4));
    CU_TRY(cudaDeviceSynchronize());
    grad_zero_pending = false;
  }

  void step_host_async(const float* x, const float* gy, int64_t tok, int step, float* y, float* gx,
                       int flags) {
    if (tok < 0 || tok > T) throw CudaError(FBQ_ERR_SHAPE, "tokens exceed max_tokens");
    if (tok == 0) return;
    async_init();
    const int slot = (int)(a_count++ & 1);
    const size_t bytes = tok * D * 4;
    // inputs: the slot's previous step must be done reading them
    if (a_used[slot]) CU_TRY(cudaStreamWaitEvent(a_h2d, a_done[slot], 0));
    CU_TRY(cudaMemcpyAsync(ax[slot].p, x, bytes, cudaMemcpyHostToDevice, a_h2d));
    CU_TRY(cudaMemcpyAsync(agy[slot].p, gy, bytes, cudaMemcpyHostToDevice, a_h2d));
    CU_TRY(cudaEventRecord(a_in[slot], a_h2d));
    // compute: inputs landed, and the slot's previous outputs are copied out
    CU_TRY(cudaStreamWaitEvent(a_cs, a_in[slot], 0));
    if (a_used[slot]) CU_TRY(cudaStreamWaitEvent(a_cs, a_out[slot], 0));
    const int saved = c.act_dtype;
    c.act_dtype = FBQ_F32;  // the host API is fp32 like the reference
    try {
      if (flags & FBQ_STEP_ZERO_GRAD) zero_grad(a_cs);
      forward(ax[slot].p, tok, 0, step, ay[slot].p, a_cs);
      // SR(dY) on the side stream (ordered after this slot's H2D through the
      // forward's fork), overlapping the forward
      quantize_gy_early(agy[slot].p, tok, 0, step);
      CU_TRY(cudaEventRecord(a_fwd[slot], a_cs));
      backward(agy[slot].p, tok, 0, step, agx[slot].p, a_cs, /*gy_ready=*/true);
      if (flags & FBQ_STEP_CONTROLLER) controller(a_cs);
      if (flags & FBQ_STEP_SGD) apply_sgd(sgd_lr, a_cs);
      CU_TRY(cudaEventRecord(a_done[slot], a_cs));
    } catch (...) {
      c.act_dtype = saved;
      throw;
    }
    c.act_dtype = saved;
    last_blocks[0] = cdiv(tok, 128) * gD;
    last_blocks[1] = cdiv(tok, 128) * gF;
    // outputs: y as soon as the forward is done, dX after the backward
    CU_TRY(cudaStreamWaitEvent(a_d2h, a_fwd[slot], 0));
    CU_TRY(cudaMemcpyAsync(y, ay[slot].p, bytes, cudaMemcpyDeviceToHost, a_d2h));
    CU_TRY(cudaStreamWaitEvent(a_d2h, a_done[slot], 0));
    CU_TRY(cudaMemcpyAsync(gx, agx[slot].p, bytes, cudaMemcpyDeviceToHost, a_d2h));
    CU_TRY(cudaEventRecord(a_out[slot], a_d2h));
    a_used[slot] = true;
  }
  void host_sync() {
    if (!a_cs) return;
    CU_TRY(cudaStreamSynchronize(a_cs));
    CU_TRY(cudaStreamSynchronize(a_d2h));
  }
};

// The reference's pre-norm residual GLU block (GluBlock, trainsim.hpp:136-146,
// trainsim.cpp:294-308): out = h + down(silu(gate(norm(h))) * up(norm(h))).
// The RmsNorm runs fused into the gate/up input quantizer (its output is never
// materialised), the residual add rides on the down GEMM's accumulate epilogue,
// and the backward's norm gradient and residual add are one pass
// (fbq_cuda_rmsnorm_backward_residual).  Gain starts at 1 (trainsim.cpp:148-152).
struct GluBlockDrv {
  Mlp m;
  int64_t ldn;
  DevBuf gain, grad_gain, nctx, nctx_s, rms_ws, row_ws, term_ws, gxn;
  GluBlockDrv(const fbq_mlp_config& cfg, const float* wg, const float* wu, const float* wd)
      : m(cfg, wg, wu, wd) {
    const int64_t D = m.D, T = m.T;
    if (D % 8) throw CudaError(FBQ_ERR_UNSUPPORTED, "GluBlock needs d_model % 8 == 0");
    ldn = ld16(D);
    gain = DevBuf(D * 4);
    grad_gain = DevBuf(D * 4);
    const std::vector<float> ones((size_t)D, 1.0f);
    CU_TRY(cudaMemcpy(gain.p, ones.data(), D * 4, cudaMemcpyHostToDevice));
    CU_TRY(cudaMemset(grad_gain.p, 0, D * 4));
    nctx = DevBuf(T * ldn * 2);
    nctx_s = DevBuf(T * cdiv(D, 128) * 4);
    rms_ws = DevBuf(T * 4);
    row_ws = DevBuf(2 * T * 8);
    term_ws = DevBuf(T * D * 4);
    gxn = DevBuf(T * D * esize(m.c.act_dtype));
  }
  void forward(const void* h, int64_t tok, int64_t row_off, int step, void* out, cudaStream_t s) {
    Mlp::NormIn n{gain.as<float>(), nctx.as<int16_t>(), ldn, nctx_s.as<float>(), rms_ws.as<float>()};
    m.forward(h, tok, row_off, step, out, s, &n, /*residual=*/true);
    m.last_blocks[0] = cdiv(tok, 128) * m.gD;
    m.last_blocks[1] = cdiv(tok, 128) * m.gF;
  }
  void backward(const void* gout, int64_t tok, int64_t row_off, int step, void* gh, cudaStream_t s) {
    if (tok == 0) return;
    // grad of the norm output (trainsim.cpp:303-306); the norm backward needs only
    // dX, so it runs before the join with the side stream's dW GEMMs (its
    // latency-bound row / column chains fill those GEMMs' tails)
    m.backward(gout, tok, row_off, step, gxn.p, s, /*gy_ready=*/false, /*join=*/false);
    FBQ_TRY(fbq_cuda_rmsnorm_backward_residual(nctx.as<int16_t>(), ldn, nctx_s.as<float>(), gxn.p,
                                               m.c.act_dtype, tok, m.D, m.D, gain.as<float>(), gout, m.D, gh,
                                               m.D, grad_gain.as<float>(), row_ws.as<double>(),
                                               term_ws.as<float>(), s));
    m.join_side(s);
    m.launches += 3;
  }
  void zero_grad(cudaStream_t s) {
    m.zero_grad(s);
    CU_TRY(cudaMemsetAsync(grad_gain.p, 0, m.D * 4, s));
  }
  void apply_sgd(double lr, cudaStream_t s) {
    m.apply_sgd(lr, s);
    FBQ_TRY(fbq_cuda_sgd_update(gain.as<float>(), grad_gain.as<float>(), m.D, lr, s));  // RmsNorm::apply_sgd
  }
};

// One fallback-quantized linear layer on the device: QuantLinearLayer
// (trainsim.cpp:61-135) with 128 x 128 blocks.
//   forward   RTN(W) (serves fwd K-major and dgrad MN-major), K1(X): threshold
//             fallback codes + the stochastic context in one pass, Y = fallback_gemm
//   backward  K2(dY), dX = bqg(dY, W), dW += bqg(dY^T, ctx)
struct QuantLinear {
  fbq_linear_config c;
  int64_t In, Out, T, ldIn, ldOut, gIn, gOut, gT;
  DevBuf w, g, w_codes, w_scales, x_codes, x_scales, x_res, x_res_scales, x_mask, ctx, gy_codes,
      gy_scales, theta, count, rate, amax;
  bool w_codes_fresh = false;  // set by the fused apply_sgd, consumed by the next forward
  int64_t last_blocks = 1;
  double last_fixed_rate = 0.0;  // FixedRate / Off: mask_rate of the last forward (k / n)

  QuantLinear(const fbq_linear_config& cfg, const float* wt) : c(cfg) {
    In = c.in_features;
    Out = c.out_features;
    T = c.max_tokens;
    if (In <= 0 || Out <= 0 || T <= 0) throw CudaError(FBQ_ERR_SHAPE, "bad linear shape");
    if (In % 16 || Out % 16) throw CudaError(FBQ_ERR_UNSUPPORTED, "need in/out features % 16 == 0");
    FBQ_TRY(fbq_cuda_init());
    ldIn = ld16(In);
    ldOut = ld16(Out);
    gIn = cdiv(In, 128);
    gOut = cdiv(Out, 128);
    gT = cdiv(T, 128);
    w = DevBuf(Out * In * 4);
    g = DevBuf(Out * In * 4);
    CU_TRY(cudaMemcpy(w.p, wt, Out * In * 4, cudaMemcpyHostToDevice));
    CU_TRY(cudaMemset(g.p, 0, Out * In * 4));
    w_codes = DevBuf(Out * ldIn);
    w_scales = DevBuf(gOut * gIn * 4);
    x_codes = DevBuf(T * ldIn);
    x_res = DevBuf(T * ldIn);
    ctx = DevBuf(T * ldIn);
    x_scales = DevBuf(gT * gIn * 4);
    x_res_scales = DevBuf(gT * gIn * 4);
    x_mask = DevBuf(cdiv(gT * gIn, 32) * 4);
    gy_codes = DevBuf(T * ldOut);
    gy_scales = DevBuf(gT * gOut * 4);
    theta = DevBuf(sizeof(double));
    count = DevBuf(sizeof(int32_t));
    rate = DevBuf(sizeof(double));
    amax = DevBuf(gT * gIn * 4);
    if (c.fallback_mode < 0 || c.fallback_mode > 2) throw CudaError(FBQ_ERR_ARG, "bad fallback_mode");
    if (c.fallback_mode == 1 && !(c.fixed_rate >= 0.0 && c.fixed_rate <= 1.0))
      throw CudaError(FBQ_ERR_ARG, "fixed_rate must be in [0, 1]");
    CU_TRY(cudaMemcpy(theta.p, &c.threshold_init, sizeof(double), cudaMemcpyHostToDevice));
    CU_TRY(cudaMemset(count.p, 0, sizeof(int32_t)));
    CU_TRY(cudaMemset(rate.p, 0, sizeof(double)));
  }

  void forward(const void* x, int64_t tok, int64_t row_off, int step, void* y, cudaStream_t s) {
    if (tok < 0 || tok > T) throw CudaError(FBQ_ERR_SHAPE, "tokens exceed max_tokens");
    if (tok == 0) return;
    // quantize_rtn(transpose(W)) == transpose(quantize_rtn(W)) (trainsim.cpp:96-97);
    // after a fused apply_sgd the codes already hold RTN of the current W (used once)
    if (!w_codes_fresh)
      FBQ_TRY(fbq_cuda_quantize_rtn(w.p, FBQ_F32, Out, In, In, w_codes.as<int8_t>(), ldIn,
                                    w_scales.as<float>(), s));
    w_codes_fresh = false;
    // score_blocks + mask (trainsim.cpp:80-93) + fallback_quantize + the SR context (:95-102)
    int mode = FBQ_MASK_THRESHOLD;
    const int64_t nblk = cdiv(tok, 128) * gIn;
    if (c.fallback_mode == 1) {  // FixedRate: score pass, device TopK, then the given mask
      FBQ_TRY(fbq_cuda_block_absmax(x, c.act_dtype, tok, In, In, amax.as<float>(), s));
      FBQ_TRY(fbq_cuda_mask_topk(amax.as<float>(), nblk, c.fixed_rate, x_mask.as<uint32_t>(),
                                 count.as<int32_t>(), s));
      mode = FBQ_MASK_GIVEN;
      int64_t k = (int64_t)std::ceil(c.fixed_rate * (double)nblk);
      last_fixed_rate = nblk ? (double)(k > nblk ? nblk : k) / (double)nblk : 0.0;
    } else if (c.fallback_mode == 2) {  // Off: an all-zero mask
      CU_TRY(cudaMemsetAsync(x_mask.p, 0, cdiv(nblk, 32) * 4, s));
      mode = FBQ_MASK_GIVEN;
      last_fixed_rate = 0.0;
    }
    FBQ_TRY(fbq_cuda_quantize_linear_input(
        x, c.act_dtype, tok, In, In, mode, c.threshold_init, mode == FBQ_MASK_THRESHOLD ? theta.as<double>() : nullptr,
        x_mask.as<uint32_t>(), x_codes.as<int8_t>(), ldIn, x_scales.as<float>(),
        x_res.as<int8_t>(), x_res_scales.as<float>(), mode == FBQ_MASK_THRESHOLD ? count.as<int32_t>() : nullptr,
        ctx.as<int8_t>(), layer_seed(c.seed, c.layer_id, 0, step), nullptr, 0, row_off, s));
    FBQ_TRY(fbq_cuda_gemm(x_codes.as<int8_t>(), ldIn, x_scales.as<float>(), FBQ_K_MAJOR,
                          w_codes.as<int8_t>(), ldIn, w_scales.as<float>(), FBQ_K_MAJOR,
                          x_mask.as<uint32_t>(), x_res.as<int8_t>(), x_res_scales.as<float>(), tok,
                          Out, In, y, c.act_dtype, Out, 0, c.epilogue, s));
    last_blocks = cdiv(tok, 128) * gIn;
  }

  void backward(const void* gy, int64_t tok, int64_t row_off, int step, void* gx, cudaStream_t s) {
    if (tok < 0 || tok > T) throw CudaError(FBQ_ERR_SHAPE, "tokens exceed max_tokens");
    if (tok == 0) return;
    FBQ_TRY(fbq_cuda_quantize_stochastic(gy, c.act_dtype, tok, Out, Out,
                                         layer_seed(c.seed, c.layer_id, 1, step), row_off,
                                         gy_codes.as<int8_t>(), ldOut, gy_scales.as<float>(), s));
    // grad_x = bqg(q(dY), q(W)): W codes (Out x In) read MN-major (trainsim.cpp:121-122)
    FBQ_TRY(fbq_cuda_gemm(gy_codes.as<int8_t>(), ldOut, gy_scales.as<float>(), FBQ_K_MAJOR,
                          w_codes.as<int8_t>(), ldIn, w_scales.as<float>(), FBQ_MN_MAJOR, nullptr,
                          nullptr, nullptr, tok, In, Out, gx, c.act_dtype, In, 0, c.epilogue, s));
    // grad_w += bqg(q(dY)^T, ctx) (trainsim.cpp:124-125); after a (deferred)
    // zero_grad the GEMM writes instead of reduce-adding into zeros
    const int acc_w = grad_zero_pending ? 0 : 1;
    grad_zero_pending = false;
    FBQ_TRY(fbq_cuda_gemm(gy_codes.as<int8_t>(), ldOut, gy_scales.as<float>(), FBQ_MN_MAJOR,
                          ctx.as<int8_t>(), ldIn, x_scales.as<float>(), FBQ_MN_MAJOR, nullptr,
                          nullptr, nullptr, Out, In, tok, g.p, FBQ_F32, In, acc_w, c.epilogue, s));
  }
  bool grad_zero_pending = false;

  void controller(cudaStream_t s, int64_t blocks = 0) {
    if (c.fallback_mode != 0) return;  // trainsim.cpp:129-133: Threshold mode only
    ctl_blocks = blocks > 0 ? blocks : 0;
    FBQ_TRY(fbq_cuda_controller_update(theta.as<double>(), count.as<int32_t>(),
                                       blocks > 0 ? blocks : last_blocks, c.r_min, c.r_max,
                                       c.alpha, rate.as<double>(), s));
  }
  int64_t ctl_blocks = 0;  // global block count of the last data-parallel controller step
};

thread_local std::string g_host_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return FBQ_OK;
  } catch (const CudaError& e) {
    g_host_err = e.what();
    return e.status;
  } catch (const std::exception& e) {
    g_host_err = e.what();
    return FBQ_ERR_ARG;
  }
}

}  // namespace

extern "C" {

const char* fbq_host_last_error(void) { return g_host_err.c_str(); }

void fbq_mlp_default_config(fbq_mlp_config* c) {
  std::memset(c, 0, sizeof(*c));
  c->act_dtype = FBQ_BF16;
  c->mid_dtype = FBQ_BF16;
  c->epilogue = FBQ_EPI_FMA;
  c->nonlinear_bits = 10;
  c->ctx_format = FBQ_CTX_INT16;
  c->layer_id_base = 0;
  c->seed = 0x5eedull;
  c->threshold_init = 1.0;
  c->r_min = 0.1;
  c->r_max = 0.3;
  c->alpha = 1.3;
}

void* fbq_mlp_create(const fbq_mlp_config* cfg, const float* w_gate, const float* w_up,
                     const float* w_down) {
  if (!cfg || !w_gate || !w_up || !w_down) return nullptr;
  try {
    return new Mlp(*cfg, w_gate, w_up, w_down);
  } catch (const std::exception& e) {
    g_host_err = e.what();
    return nullptr;
  }
}

void fbq_mlp_destroy(void* m) { delete static_cast<Mlp*>(m); }

int fbq_mlp_forward_device(void* m, const void* x, int64_t tokens, int64_t row_offset, int step,
                           void* y, fbq_stream_t stream) {
  if (!m || (tokens > 0 && (!x || !y))) return FBQ_ERR_ARG;
  return guarded([&] {
    auto* mlp = static_cast<Mlp*>(m);
    mlp->forward(x, tokens, row_offset, step, y, reinterpret_cast<cudaStream_t>(stream));
    mlp->last_blocks[0] = cdiv(tokens, 128) * mlp->gD;
    mlp->last_blocks[1] = cdiv(tokens, 128) * mlp->gF;
  });
}

int fbq_mlp_backward_device(void* m, const void* gy, int64_t tokens, int64_t row_offset, int step,
                            void* gx, fbq_stream_t stream) {
  if (!m || (tokens > 0 && (!gy || !gx))) return FBQ_ERR_ARG;
  return guarded([&] {
    static_cast<Mlp*>(m)->backward(gy, tokens, row_offset, step, gx,
                                   reinterpret_cast<cudaStream_t>(stream));
  });
}

int fbq_mlp_controller_step(void* m, fbq_stream_t stream) {
  if (!m) return FBQ_ERR_ARG;
  return guarded([&] { static_cast<Mlp*>(m)->controller(reinterpret_cast<cudaStream_t>(stream)); });
}

int fbq_mlp_controller_step_blocks(void* m, int64_t blocks_gate_up, int64_t blocks_down,
                                   fbq_stream_t stream) {
  if (!m || blocks_gate_up < 0 || blocks_down < 0) return FBQ_ERR_ARG;
  return guarded([&] {
    static_cast<Mlp*>(m)->controller(reinterpret_cast<cudaStream_t>(stream), blocks_gate_up, blocks_down);
  });
}

int32_t* fbq_mlp_count_ptr(void* m) { return m ? static_cast<Mlp*>(m)->counts.as<int32_t>() : nullptr; }

int fbq_mlp_zero_grad(void* m, fbq_stream_t stream) {
  if (!m) return FBQ_ERR_ARG;
  return guarded([&] {
    static_cast<Mlp*>(m)->zero_grad(reinterpret_cast<cudaStream_t>(stream));
  });
}

int fbq_mlp_step_host_async(void* m, const float* x, const float* gy, int64_t tokens, int step,
                            float* y, float* gx, int flags) {
  if (!m || (tokens > 0 && (!x || !gy || !y || !gx))) return FBQ_ERR_ARG;
  if (flags & ~(FBQ_STEP_ZERO_GRAD | FBQ_STEP_CONTROLLER | FBQ_STEP_SGD)) return FBQ_ERR_ARG;
  return guarded([&] { static_cast<Mlp*>(m)->step_host_async(x, gy, tokens, step, y, gx, flags); });
}

int fbq_mlp_host_sync(void* m) {
  if (!m) return FBQ_ERR_ARG;
  return guarded([&] { static_cast<Mlp*>(m)->host_sync(); });
}

int fbq_mlp_step_host(void* m, const float* x, const float* gy, int64_t tokens, int step,
                      float* y, float* gx) {
  if (!m || (tokens > 0 && (!x || !gy || !y || !gx))) return FBQ_ERR_ARG;
  return guarded([&] {
    auto* mlp = static_cast<Mlp*>(m);
    mlp->step_host(x, gy, tokens, step, y, gx);
    mlp->last_blocks[0] = cdiv(tokens, 128) * mlp->gD;
    mlp->last_blocks[1] = cdiv(tokens, 128) * mlp->gF;
  });
}

int fbq_mlp_set_thresholds(void* m, double theta_gate_up, double theta_down) {
  if (!m || !(theta_gate_up > 0.0) || !(theta_down > 0.0)) return FBQ_ERR_ARG;
  return guarded([&] {
    const double th[2] = {theta_gate_up, theta_down};
    CU_TRY(cudaMemcpy(static_cast<Mlp*>(m)->theta.p, th, sizeof(th), cudaMemcpyHostToDevice));
  });
}

int fbq_mlp_context_bytes(void* m, int64_t tokens, int64_t* ours, int64_t* bf16) {
  if (!m || tokens < 0 || !ours || !bf16) return FBQ_ERR_ARG;
  auto* mlp = static_cast<Mlp*>(m);
  const int64_t t = tokens, D = mlp->D, F = mlp->F, gt = cdiv(t, 128);
  const int64_t x_ctx = 2 * t * mlp->ldD + 2 * gt * mlp->gD * 4;          // gate + up SR contexts of X
  const int64_t ab_ctx = 2 * mlp->ctx_bytes(t) + 2 * t * mlp->gF * 4;      // a, b (1 x 128 scales)
  const int64_t h_ctx = t * mlp->ldF + gt * mlp->gF * 4;                   // SR context of h
  *ours = x_ctx + ab_ctx + h_ctx;
  *bf16 = 2 * (t * D + 2 * t * F + t * F);                                  // X, a, b, h in bf16
  return FBQ_OK;
}

int fbq_mlp_set_profiling(void* m, int on) {
  if (!m) return FBQ_ERR_ARG;
  auto* mlp = static_cast<Mlp*>(m);
  mlp->profiling = on != 0;
  mlp->ev_used = 0;
  return FBQ_OK;
}

int fbq_mlp_gemm_time(void* m, double* total_ms, int64_t* n_gemms) {
  if (!m || !total_ms) return FBQ_ERR_ARG;
  return guarded([&] {
    auto* mlp = static_cast<Mlp*>(m);
    if (n_gemms) *n_gemms = (int64_t)(mlp->ev_used / 2);
    *total_ms = mlp->gemm_ms_and_reset();
  });
}

int64_t fbq_mlp_launch_count(void* m) { return m ? static_cast<Mlp*>(m)->launches : 0; }

int fbq_mlp_wait_grad(void* m, int which, fbq_stream_t stream) {
  if (!m || which < 0 || which > 2) return FBQ_ERR_ARG;
  auto* mlp = static_cast<Mlp*>(m);
  cudaEvent_t e = mlp->ev_grad[which];
  return cudaStreamWaitEvent(reinterpret_cast<cudaStream_t>(stream), e, 0) == cudaSuccess ? FBQ_OK
                                                                                          : FBQ_ERR_CUDA;
}

void* fbq_mlp_grad_ptr(void* m, int which) {
  if (!m) return nullptr;
  auto* mlp = static_cast<Mlp*>(m);
  try {
    mlp->flush_grad_zero();
    if (cudaDeviceSynchronize() != cudaSuccess) return nullptr;
  } catch (...) {
    return nullptr;
  }
  if (which == 0) return mlp->g_gu.p;
  if (which == 1) return mlp->g_gu.as<float>() + mlp->F * mlp->D;
  if (which == 2) return mlp->g_d.p;
  return nullptr;
}

int fbq_mlp_get_grads(void* m, float* g_gate, float* g_up, float* g_down) {
  if (!m) return FBQ_ERR_ARG;
  return guarded([&] {
    auto* mlp = static_cast<Mlp*>(m);
    mlp->flush_grad_zero();
    CU_TRY(cudaDeviceSynchronize());
    const size_t n = mlp->F * mlp->D * 4;
    if (g_gate) CU_TRY(cudaMemcpy(g_gate, mlp->g_gu.p, n, cudaMemcpyDeviceToHost));
    if (g_up) CU_TRY(cudaMemcpy(g_up, mlp->g_gu.as<float>() + mlp->F * mlp->D, n, cudaMemcpyDeviceToHost));
    if (g_down) CU_TRY(cudaMemcpy(g_down, mlp->g_d.p, n, cudaMemcpyDeviceToHost));
  });
}

void* fbq_glublock_create(const fbq_mlp_config* cfg, const float* w_gate, const float* w_up,
                          const float* w_down) {
  if (!cfg || !w_gate || !w_up || !w_down) return nullptr;
  try {
    return new GluBlockDrv(*cfg, w_gate, w_up, w_down);
  } catch (const std::exception& e) {
    g_host_err = e.what();
    return nullptr;
  }
}
void fbq_glublock_destroy(void* b) { delete static_cast<GluBlockDrv*>(b); }
void* fbq_glublock_mlp(void* b) { return b ? &static_cast<GluBlockDrv*>(b)->m : nullptr; }
int fbq_glublock_forward_device(void* b, const void* h, int64_t tokens, int64_t row_offset, int step,
                                void* out, fbq_stream_t stream) {
  if (!b || (tokens > 0 && (!h || !out)) || row_offset < 0) return FBQ_ERR_ARG;
  if (h == out && tokens > 0) return FBQ_ERR_ARG;  // out is written before the input is consumed
  return guarded([&] {
    static_cast<GluBlockDrv*>(b)->forward(h, tokens, row_offset, step, out, reinterpret_cast<cudaStream_t>(stream));
  });
}
int fbq_glublock_backward_device(void* b, const void* grad_out, int64_t tokens, int64_t row_offset, int step,
                                 void* grad_h, fbq_stream_t stream) {
  if (!b || (tokens > 0 && (!grad_out || !grad_h)) || row_offset < 0) return FBQ_ERR_ARG;
  return guarded([&] {
    static_cast<GluBlockDrv*>(b)->backward(grad_out, tokens, row_offset, step, grad_h,
                                           reinterpret_cast<cudaStream_t>(stream));
  });
}
int fbq_glublock_zero_grad(void* b, fbq_stream_t stream) {
  if (!b) return FBQ_ERR_ARG;
  return guarded([&] { static_cast<GluBlockDrv*>(b)->zero_grad(reinterpret_cast<cudaStream_t>(stream)); });
}
int fbq_glublock_apply_sgd(void* b, double lr, fbq_stream_t stream) {
  if (!b) return FBQ_ERR_ARG;
  return guarded([&] { static_cast<GluBlockDrv*>(b)->apply_sgd(lr, reinterpret_cast<cudaStream_t>(stream)); });
}
float* fbq_glublock_gain_ptr(void* b, int which) {
  if (!b || (which != 0 && which != 1)) return nullptr;
  auto* g = static_cast<GluBlockDrv*>(b);
  return which == 0 ? g->gain.as<float>() : g->grad_gain.as<float>();
}
int fbq_glublock_get_gain(void* b, float* gain, float* grad_gain) {
  if (!b) return FBQ_ERR_ARG;
  return guarded([&] {
    auto* g = static_cast<GluBlockDrv*>(b);
    CU_TRY(cudaDeviceSynchronize());
    if (gain) CU_TRY(cudaMemcpy(gain, g->gain.p, g->m.D * 4, cudaMemcpyDeviceToHost));
    if (grad_gain) CU_TRY(cudaMemcpy(grad_gain, g->grad_gain.p, g->m.D * 4, cudaMemcpyDeviceToHost));
  });
}

int fbq_mlp_apply_sgd(void* m, double lr, fbq_stream_t stream) {
  if (!m) return FBQ_ERR_ARG;
  return guarded([&] { static_cast<Mlp*>(m)->apply_sgd(lr, reinterpret_cast<cudaStream_t>(stream)); });
}

int fbq_mlp_set_sgd_lr(void* m, double lr) {
  if (!m) return FBQ_ERR_ARG;
  static_cast<Mlp*>(m)->sgd_lr = lr;
  return FBQ_OK;
}

int fbq_mlp_get_weights(void* m, float* w_gate, float* w_up, float* w_down) {
  if (!m) return FBQ_ERR_ARG;
  return guarded([&] {
    auto* mlp = static_cast<Mlp*>(m);
    CU_TRY(cudaDeviceSynchronize());
    const size_t n = mlp->F * mlp->D * 4;
    if (w_gate) CU_TRY(cudaMemcpy(w_gate, mlp->w_gu.p, n, cudaMemcpyDeviceToHost));
    if (w_up) CU_TRY(cudaMemcpy(w_up, mlp->w_gu.as<float>() + mlp->F * mlp->D, n, cudaMemcpyDeviceToHost));
    if (w_down) CU_TRY(cudaMemcpy(w_down, mlp->w_d.p, n, cudaMemcpyDeviceToHost));
  });
}

int fbq_mlp_get_controller(void* m, double* rates, double* thresholds) {
  if (!m) return FBQ_ERR_ARG;
  return guarded([&] {
    auto* mlp = static_cast<Mlp*>(m);
    CU_TRY(cudaDeviceSynchronize());
    if (thresholds) CU_TRY(cudaMemcpy(thresholds, mlp->theta.p, 16, cudaMemcpyDeviceToHost));
    if (rates) {
      // last observed rate of the most recent forward (masked / blocks)
      int32_t cnt[2];
      CU_TRY(cudaMemcpy(cnt, mlp->counts.p, 8, cudaMemcpyDeviceToHost));
      // counts are global after a data-parallel reduction: divide by the
      // blocks the controller used (local blocks when no step ran yet)
      for (int i = 0; i < 2; ++i) {
        const int64_t b = mlp->ctl_blocks[i] > 0 ? mlp->ctl_blocks[i] : mlp->last_blocks[i];
        rates[i] = (double)cnt[i] / (double)b;
      }
    }
  });
}

}  // extern "C"

void fbq_linear_default_config(fbq_linear_config* cfg) {
  if (!cfg) return;
  *cfg = fbq_linear_config{};
  cfg->act_dtype = FBQ_BF16;
  cfg->epilogue = FBQ_EPI_FMA;
  cfg->layer_id = 0;
  cfg->seed = 0x5eedull;
  cfg->threshold_init = 1.0;
  cfg->r_min = 0.1;
  cfg->r_max = 0.3;
  cfg->alpha = 1.3;
  cfg->fallback_mode = 0;
  cfg->fixed_rate = 0.0;
}

void* fbq_linear_create(const fbq_linear_config* cfg, const float* weight) {
  if (!cfg || !weight) {
    g_host_err = "fbq_linear_create: null argument";
    return nullptr;
  }
  try {
    return new QuantLinear(*cfg, weight);
  } catch (const std::exception& e) {
    g_host_err = e.what();
    return nullptr;
  }
}
void fbq_linear_destroy(void* l) { delete static_cast<QuantLinear*>(l); }

int fbq_linear_forward_device(void* l, const void* x, int64_t tokens, int64_t row_offset, int step,
                              void* y, fbq_stream_t stream) {
  if (!l || (tokens > 0 && (!x || !y)) || row_offset < 0) return FBQ_ERR_ARG;
  return guarded([&] {
    static_cast<QuantLinear*>(l)->forward(x, tokens, row_offset, step, y,
                                          reinterpret_cast<cudaStream_t>(stream));
  });
}
int fbq_linear_backward_device(void* l, const void* gy, int64_t tokens, int64_t row_offset,
                               int step, void* gx, fbq_stream_t stream) {
  if (!l || (tokens > 0 && (!gy || !gx)) || row_offset < 0) return FBQ_ERR_ARG;
  return guarded([&] {
    static_cast<QuantLinear*>(l)->backward(gy, tokens, row_offset, step, gx,
                                           reinterpret_cast<cudaStream_t>(stream));
  });
}
int fbq_linear_controller_step(void* l, fbq_stream_t stream) {
  if (!l) return FBQ_ERR_ARG;
  return guarded([&] { static_cast<QuantLinear*>(l)->controller(reinterpret_cast<cudaStream_t>(stream)); });
}
int fbq_linear_controller_step_blocks(void* l, int64_t blocks, fbq_stream_t stream) {
  if (!l || blocks < 0) return FBQ_ERR_ARG;
  return guarded([&] {
    static_cast<QuantLinear*>(l)->controller(reinterpret_cast<cudaStream_t>(stream), blocks);
  });
}
int32_t* fbq_linear_count_ptr(void* l) {
  return l ? static_cast<QuantLinear*>(l)->count.as<int32_t>() : nullptr;
}
int fbq_linear_apply_sgd(void* l, double lr, fbq_stream_t stream) {
  if (!l) return FBQ_ERR_ARG;
  return guarded([&] {
    auto* q = static_cast<QuantLinear*>(l);
    auto s = reinterpret_cast<cudaStream_t>(stream);
    if (q->grad_zero_pending) return;  // grad is (pending) zero: w unchanged
    // fused with the next forward's RTN(W) (fbq_cuda_sgd_quantize_rtn; see Mlp::apply_sgd)
    FBQ_TRY(fbq_cuda_sgd_quantize_rtn(q->w.as<float>(), q->g.as<float>(), q->Out, q->In, lr,
                                      q->w_codes.as<int8_t>(), q->ldIn, q->w_scales.as<float>(), s));
    q->w_codes_fresh = true;
  });
}
int fbq_linear_get_weight(void* l, float* w_host) {
  if (!l || !w_host) return FBQ_ERR_ARG;
  return guarded([&] {
    auto* q = static_cast<QuantLinear*>(l);
    CU_TRY(cudaDeviceSynchronize());
    CU_TRY(cudaMemcpy(w_host, q->w.p, q->Out * q->In * 4, cudaMemcpyDeviceToHost));
  });
}
int fbq_linear_get_grad(void* l, float* g_host) {
  if (!l || !g_host) return FBQ_ERR_ARG;
  return guarded([&] {
    auto* q = static_cast<QuantLinear*>(l);
    CU_TRY(cudaDeviceSynchronize());
    if (q->grad_zero_pending) std::fill(g_host, g_host + q->Out * q->In, 0.0f);
    else CU_TRY(cudaMemcpy(g_host, q->g.p, q->Out * q->In * 4, cudaMemcpyDeviceToHost));
  });
}
int fbq_linear_zero_grad(void* l, fbq_stream_t stream) {
  if (!l) return FBQ_ERR_ARG;
  (void)stream;
  static_cast<QuantLinear*>(l)->grad_zero_pending = true;  // deferred (see backward)
  return FBQ_OK;
}
float* fbq_linear_grad_ptr(void* l) {
  if (!l) return nullptr;
  auto* q = static_cast<QuantLinear*>(l);
  if (q->grad_zero_pending) {  // materialise the pending zero for a reader
    if (cudaDeviceSynchronize() != cudaSuccess || cudaMemset(q->g.p, 0, q->Out * q->In * 4) != cudaSuccess ||
        cudaDeviceSynchronize() != cudaSuccess)
      return nullptr;
    q->grad_zero_pending = false;
  }
  return q->g.as<float>();
}
int fbq_linear_get_controller(void* l, double* last_rate, double* threshold) {
  if (!l || !last_rate || !threshold) return FBQ_ERR_ARG;
  return guarded([&] {
    auto* q = static_cast<QuantLinear*>(l);
    CU_TRY(cudaDeviceSynchronize());
    if (q->c.fallback_mode == 0) {
      // the observed rate of the LAST FORWARD (trainsim.cpp:93: last_rate_ is set
      // in forward, before any controller step): masked / blocks -- global
      // counts and blocks after a data-parallel controller step
      int32_t cnt = 0;
      CU_TRY(cudaMemcpy(&cnt, q->count.p, sizeof(int32_t), cudaMemcpyDeviceToHost));
      const int64_t b = q->ctl_blocks > 0 ? q->ctl_blocks : q->last_blocks;
      *last_rate = b > 0 ? (double)cnt / (double)b : 0.0;
    } else {
      *last_rate = q->last_fixed_rate;
    }
    CU_TRY(cudaMemcpy(threshold, q->theta.p, sizeof(double), cudaMemcpyDeviceToHost));
  });
}
