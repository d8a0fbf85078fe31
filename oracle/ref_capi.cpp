// TEST INFRASTRUCTURE ONLY -- never linked into the product path.
//
// Thin extern "C" shim over the UNMODIFIED reference library (the sources
// under /root/reference/proj/src are compiled in place by oracle/Makefile
// into oracle/_ref/libfbq_ref.so).  It exposes the reference's own public
// operator API (quant.hpp, gemm.hpp, policy.hpp, kernels.hpp, trainsim.hpp)
// on flat host arrays so that
//   * tests/golden/make_golden.py can generate golden vectors from the
//     reference itself,
//   * tests can pin oracle/fbq_oracle.c (the C restatement) against it,
//   * bench.py --impl reference can time the reference CPU path.
// Only tests/, __graft_entry__.smoke() and bench.py's reference/cpu_baseline
// legs may load this library.

#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "fbq/error.hpp"
#include "fbq/gemm.hpp"
#include "fbq/kernels.hpp"
#include "fbq/matrix.hpp"
#include "fbq/policy.hpp"
#include "fbq/quant.hpp"
#include "fbq/rng.hpp"
#include "fbq/trainsim.hpp"

using namespace fbq;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

DenseMatrix make_dense(const float* x, int64_t rows, int64_t cols) {
    return DenseMatrix(rows, cols, std::vector<float>(x, x + rows * cols));
}

QuantizedTensor make_qt(const int16_t* codes, const float* scales, int64_t rows, int64_t cols,
                        int64_t gr, int64_t gc, int bits) {
    QuantizedTensor q;
    q.rows = rows;
    q.cols = cols;
    q.geometry = GroupGeometry(gr, gc);
    q.bits = BitWidth(bits);
    q.codes.assign(codes, codes + rows * cols);
    q.scales.assign(scales, scales + q.grid_rows() * q.grid_cols());
    return q;
}

void dump_qt(const QuantizedTensor& q, int16_t* codes, float* scales) {
    std::memcpy(codes, q.codes.data(), q.codes.size() * sizeof(int16_t));
    std::memcpy(scales, q.scales.data(), q.scales.size() * sizeof(float));
}

// Residual blocks are returned in the reference's compact order (row-major
// over masked blocks); block b occupies res_codes[b*gr*gc ...] with its own
// (possibly truncated) extent, row-major within the block.
FallbackTensor make_ft(const int16_t* codes, const float* scales, const uint8_t* mask,
                       const int16_t* res_codes, const float* res_scales, int64_t rows,
                       int64_t cols, int64_t g) {
    FallbackTensor f;
    f.primary = make_qt(codes, scales, rows, cols, g, g, 8);
    const int64_t gr = f.primary.grid_rows(), gc = f.primary.grid_cols();
    f.mask.assign(mask, mask + gr * gc);
    f.residual_index.assign(gr * gc, -1);
    int64_t slot = 0;
    for (int64_t bi = 0; bi < gr; ++bi) {
        for (int64_t bj = 0; bj < gc; ++bj) {
            if (!f.mask[bi * gc + bj]) continue;
            const int64_t er = std::min(g, rows - bi * g), ec = std::min(g, cols - bj * g);
            FallbackTensor::Residual r;
            r.codes.assign(res_codes + slot * g * g, res_codes + slot * g * g + er * ec);
            r.scale = res_scales[slot];
            f.residual_index[bi * gc + bj] = static_cast<int32_t>(f.residuals.size());
            f.residuals.push_back(std::move(r));
            ++slot;
        }
    }
    return f;
}

} // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void ref_set_gemm_threads(int n) { set_gemm_threads(n); }
int ref_gemm_threads() { return gemm_threads(); }

// kernels::Ops backends ("scalar" | "avx2"), kernels.hpp:14-48
int ref_select_backend(const char* name) { return kernels::select(name) ? 0 : 1; }
const char* ref_active_backend() { return kernels::active().name; }
int ref_avx2_supported() { return kernels::avx2_supported() ? 1 : 0; }

static const kernels::Ops& ops_by_name(const char* n) {
    if (std::strcmp(n, "avx2") == 0 && kernels::avx2_supported()) return kernels::avx2_ops();
    return kernels::scalar_ops();
}
float ref_ops_absmax_2d(const char* be, const float* x, size_t rows, size_t cols, size_t ld) {
    return ops_by_name(be).absmax_2d(x, rows, cols, ld);
}
void ref_ops_quantize_rtn_2d(const char* be, const float* x, size_t ldx, int16_t* q, size_t ldq,
                             size_t rows, size_t cols, float scale, int32_t limit) {
    ops_by_name(be).quantize_rtn_2d(x, ldx, q, ldq, rows, cols, scale, limit);
}
void ref_ops_dequantize_2d(const char* be, const int16_t* q, size_t ldq, float* y, size_t ldy,
                           size_t rows, size_t cols, float scale) {
    ops_by_name(be).dequantize_2d(q, ldq, y, ldy, rows, cols, scale);
}
void ref_ops_gemm_i16_accum(const char* be, const int16_t* a, size_t lda, const int16_t* b,
                            size_t ldb, int32_t* c, size_t ldc, size_t m, size_t n, size_t k) {
    ops_by_name(be).gemm_i16_accum(a, lda, b, ldb, c, ldc, m, n, k);
}
void ref_ops_scale_accum(const char* be, float* acc, const int32_t* p, size_t n, float scale) {
    ops_by_name(be).scale_accum(acc, p, n, scale);
}

// rng.hpp
uint64_t ref_bits_at(uint64_t seed, uint64_t n) { return DeterministicRng(seed).bits_at(n); }
double ref_uniform_at(uint64_t seed, uint64_t n) { return DeterministicRng(seed).uniform_at(n); }
float ref_normal_at(uint64_t seed, uint64_t n) { return DeterministicRng(seed).normal_at(n); }
uint64_t ref_derive_seed(uint64_t base, uint64_t a, uint64_t b) { return derive_seed(base, a, b); }

// quant.hpp
int ref_quantize_rtn(const float* x, int64_t rows, int64_t cols, int64_t gr, int64_t gc, int bits,
                     int16_t* codes, float* scales) {
    return guarded([&] {
        dump_qt(quantize_rtn(make_dense(x, rows, cols), GroupGeometry(gr, gc), BitWidth(bits)),
                codes, scales);
    });
}

int ref_quantize_stochastic(const float* x, int64_t rows, int64_t cols, int64_t gr, int64_t gc,
                            int bits, uint64_t seed, int16_t* codes, float* scales) {
    return guarded([&] {
        dump_qt(quantize_stochastic(make_dense(x, rows, cols), GroupGeometry(gr, gc),
                                    BitWidth(bits), DeterministicRng(seed)),
                codes, scales);
    });
}

int ref_dequantize(const int16_t* codes, const float* scales, int64_t rows, int64_t cols,
                   int64_t gr, int64_t gc, int bits, float* out) {
    return guarded([&] {
        const DenseMatrix d = dequantize(make_qt(codes, scales, rows, cols, gr, gc, bits));
        std::memcpy(out, d.data(), d.size() * sizeof(float));
    });
}

// Outputs: primary codes/scales; residual blocks compacted in the reference's
// order (block slot s at res_codes + s*g*g, extent er x ec row-major);
// residual_index per block (-1 when unmasked); *n_res = residuals.size().
int ref_fallback_quantize(const float* x, int64_t rows, int64_t cols, int64_t g,
                          const uint8_t* mask, int16_t* codes, float* scales, int16_t* res_codes,
                          float* res_scales, int32_t* residual_index, int64_t* n_res) {
    return guarded([&] {
        const int64_t gr = grid_rows(rows, GroupGeometry(g, g));
        const int64_t gc = grid_cols(cols, GroupGeometry(g, g));
        std::vector<uint8_t> m(mask, mask + gr * gc);
        const FallbackTensor f =
            fallback_quantize(make_dense(x, rows, cols), GroupGeometry(g, g), BitWidth(8), m);
        dump_qt(f.primary, codes, scales);
        for (size_t s = 0; s < f.residuals.size(); ++s) {
            std::memcpy(res_codes + s * g * g, f.residuals[s].codes.data(),
                        f.residuals[s].codes.size() * sizeof(int16_t));
            res_scales[s] = f.residuals[s].scale;
        }
        std::memcpy(residual_index, f.residual_index.data(), f.residual_index.size() * 4);
        *n_res = static_cast<int64_t>(f.residuals.size());
    });
}

int ref_dequantize_fallback(const int16_t* codes, const float* scales, const uint8_t* mask,
                            const int16_t* res_codes, const float* res_scales, int64_t rows,
                            int64_t cols, int64_t g, float* out) {
    return guarded([&] {
        const DenseMatrix d = dequantize_fallback(
            make_ft(codes, scales, mask, res_codes, res_scales, rows, cols, g));
        std::memcpy(out, d.data(), d.size() * sizeof(float));
    });
}

int ref_transpose_qt(const int16_t* codes, const float* scales, int64_t rows, int64_t cols,
                     int64_t gr, int64_t gc, int16_t* out_codes, float* out_scales) {
    return guarded([&] {
        dump_qt(transpose(make_qt(codes, scales, rows, cols, gr, gc, 8)), out_codes, out_scales);
    });
}

// gemm.hpp -- A: m x k codes (geometry g x g), B: k x n codes (geometry g x g)
int ref_block_quant_gemm(const int16_t* a_codes, const float* a_scales, const int16_t* b_codes,
                         const float* b_scales, int64_t m, int64_t n, int64_t k, int64_t g,
                         float* out) {
    return guarded([&] {
        const DenseMatrix d = block_quant_gemm(make_qt(a_codes, a_scales, m, k, g, g, 8),
                                               make_qt(b_codes, b_scales, k, n, g, g, 8),
                                               GemmBlockShape(g, g, g));
        std::memcpy(out, d.data(), d.size() * sizeof(float));
    });
}

int ref_fallback_gemm(const int16_t* a_codes, const float* a_scales, const uint8_t* mask,
                      const int16_t* res_codes, const float* res_scales, const int16_t* b_codes,
                      const float* b_scales, int64_t m, int64_t n, int64_t k, int64_t g,
                      float* out) {
    return guarded([&] {
        const DenseMatrix d =
            fallback_gemm(make_ft(a_codes, a_scales, mask, res_codes, res_scales, m, k, g),
                          make_qt(b_codes, b_scales, k, n, g, g, 8), GemmBlockShape(g, g, g));
        std::memcpy(out, d.data(), d.size() * sizeof(float));
    });
}

int ref_tiled_block_gemm(const int16_t* a_codes, const float* a_scales, const int16_t* b_codes,
                         const float* b_scales, int64_t m, int64_t n, int64_t k, int64_t g,
                         int64_t tm, int64_t tn, int64_t tk, float* out) {
    return guarded([&] {
        const DenseMatrix d = tiled_block_gemm(make_qt(a_codes, a_scales, m, k, g, g, 8),
                                               make_qt(b_codes, b_scales, k, n, g, g, 8),
                                               GemmBlockShape(g, g, g), TileShape(tm, tn, tk));
        std::memcpy(out, d.data(), d.size() * sizeof(float));
    });
}

int ref_gemm_oracle(const float* a, const float* b, int64_t m, int64_t n, int64_t k, float* out) {
    return guarded([&] {
        const DenseMatrix d = gemm_oracle(make_dense(a, m, k), make_dense(b, k, n));
        std::memcpy(out, d.data(), d.size() * sizeof(float));
    });
}

// policy.hpp
int ref_score_blocks_absmax(const float* x, int64_t rows, int64_t cols, int64_t g,
                            double* scores) {
    return guarded([&] {
        const auto s = score_blocks(make_dense(x, rows, cols), GroupGeometry(g, g), BitWidth(8),
                                    FallbackCriterion::AbsMax);
        std::memcpy(scores, s.data(), s.size() * sizeof(double));
    });
}

int ref_mask_threshold(const double* scores, int64_t n, double theta, uint8_t* mask) {
    return guarded([&] {
        const auto m = mask_threshold(std::vector<double>(scores, scores + n), theta);
        std::memcpy(mask, m.data(), m.size());
    });
}

int ref_mask_topk(const double* scores, int64_t n, double rate, uint8_t* mask) {
    return guarded([&] {
        const auto m = mask_topk(std::vector<double>(scores, scores + n), rate);
        std::memcpy(mask, m.data(), m.size());
    });
}

double ref_mask_rate(const uint8_t* mask, int64_t n) {
    return mask_rate(std::vector<uint8_t>(mask, mask + n));
}

int ref_controller_update(double threshold, double last_rate, double observed, double r_min,
                          double r_max, double alpha, double* out_threshold,
                          double* out_last_rate) {
    return guarded([&] {
        FallbackThresholdState s;
        s.threshold = threshold;
        s.last_rate = last_rate;
        s = controller_update(s, observed, ControllerConfig(r_min, r_max, alpha));
        *out_threshold = s.threshold;
        *out_last_rate = s.last_rate;
    });
}

// ---------------------------------------------------------------------------
// SwiGLU MLP (gate/up -> GluCombine -> down) built from the reference's own
// QuantLinearLayer / GluCombine (trainsim.hpp:38-118), block side g.  Used by
// bench.py --impl reference and the cpu_baseline leg: one call = one
// fwd+bwd step over `tokens` rows.  The handle owns the layers.
struct RefMlp {
    QuantConfig cfg;
    std::unique_ptr<QuantLinearLayer> gate, up, down;
    std::unique_ptr<GluCombine> combine;
};

void* ref_mlp_create(const float* w_gate, const float* w_up, const float* w_down, int64_t d_model,
                     int64_t d_ff, int64_t g, double threshold) {
    try {
        auto* m = new RefMlp;
        m->cfg.block = g;
        m->cfg.threshold_init = threshold;
        m->gate = std::make_unique<QuantLinearLayer>("gate", 0, make_dense(w_gate, d_ff, d_model),
                                                     m->cfg);
        m->up = std::make_unique<QuantLinearLayer>("up", 1, make_dense(w_up, d_ff, d_model),
                                                   m->cfg);
        m->down = std::make_unique<QuantLinearLayer>("down", 2, make_dense(w_down, d_model, d_ff),
                                                     m->cfg);
        m->combine = std::make_unique<GluCombine>(m->cfg);
        return m;
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

void ref_mlp_destroy(void* h) { delete static_cast<RefMlp*>(h); }

// x: tokens x d_model; grad_out: tokens x d_model; writes y (tokens x d_model)
// and grad_x (tokens x d_model).
int ref_mlp_step(void* h, const float* x, const float* grad_out, int64_t tokens, int64_t d_model,
                 int step, float* y, float* grad_x) {
    return guarded([&] {
        auto* m = static_cast<RefMlp*>(h);
        const DenseMatrix xm = make_dense(x, tokens, d_model);
        const DenseMatrix a = m->gate->forward(xm, step);
        const DenseMatrix b = m->up->forward(xm, step);
        const DenseMatrix hmid = m->combine->forward(a, b);
        const DenseMatrix out = m->down->forward(hmid, step);
        std::memcpy(y, out.data(), out.size() * sizeof(float));
        const DenseMatrix gh = m->down->backward(make_dense(grad_out, tokens, d_model), step);
        auto [ga, gb] = m->combine->backward(gh);
        const DenseMatrix gx1 = m->gate->backward(ga, step);
        const DenseMatrix gx2 = m->up->backward(gb, step);
        for (int64_t i = 0; i < gx1.size(); ++i) grad_x[i] = gx1.data()[i] + gx2.data()[i];
    });
}

int ref_mlp_grads(void* h, float* g_gate, float* g_up, float* g_down) {
    return guarded([&] {
        auto* m = static_cast<RefMlp*>(h);
        std::memcpy(g_gate, m->gate->grad_weight().data(), m->gate->grad_weight().size() * 4);
        std::memcpy(g_up, m->up->grad_weight().data(), m->up->grad_weight().size() * 4);
        std::memcpy(g_down, m->down->grad_weight().data(), m->down->grad_weight().size() * 4);
    });
}

// QuantLinearLayer::apply_sgd (trainsim.cpp:137-143) of gate, up, down, and the weights
int ref_mlp_sgd(void* h, double lr) {
    return guarded([&] {
        auto* m = static_cast<RefMlp*>(h);
        m->gate->apply_sgd(lr);
        m->up->apply_sgd(lr);
        m->down->apply_sgd(lr);
    });
}
int ref_mlp_weights(void* h, float* w_gate, float* w_up, float* w_down) {
    return guarded([&] {
        auto* m = static_cast<RefMlp*>(h);
        std::memcpy(w_gate, m->gate->weight().data(), m->gate->weight().size() * 4);
        std::memcpy(w_up, m->up->weight().data(), m->up->weight().size() * 4);
        std::memcpy(w_down, m->down->weight().data(), m->down->weight().size() * 4);
    });
}

// controller_step of every layer (trainsim.cpp:129-133); rates/thresholds of
// gate, up, down after the update.
int ref_mlp_controller(void* h, double* rates3, double* thresholds3) {
    return guarded([&] {
        auto* m = static_cast<RefMlp*>(h);
        QuantLinearLayer* ls[3] = {m->gate.get(), m->up.get(), m->down.get()};
        for (int i = 0; i < 3; ++i) {
            rates3[i] = ls[i]->last_fallback_rate();
            ls[i]->controller_step();
            thresholds3[i] = ls[i]->threshold();
        }
    });
}

// ---------------------------------------------------------------------------
// One QuantLinearLayer (trainsim.hpp:38-73, trainsim.cpp:61-135), block side g:
// the reference a single fallback-quantized linear is checked against.
struct RefLinear {
    QuantConfig cfg;
    std::unique_ptr<QuantLinearLayer> l;
    int64_t in = 0, out = 0;
};

void* ref_linear_create(const float* w, int64_t out_features, int64_t in_features, int64_t g,
                        double threshold, int layer_id, int fallback_mode, double fixed_rate) {
    try {
        auto* r = new RefLinear;
        r->cfg.block = g;
        r->cfg.threshold_init = threshold;
        r->cfg.fallback_mode = fallback_mode == 1 ? FallbackMode::FixedRate
                             : fallback_mode == 2 ? FallbackMode::Off : FallbackMode::Threshold;
        r->cfg.fixed_rate = fixed_rate;
        r->in = in_features;
        r->out = out_features;
        r->l = std::make_unique<QuantLinearLayer>("linear", layer_id,
                                                  make_dense(w, out_features, in_features), r->cfg);
        return r;
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}
void ref_linear_destroy(void* h) { delete static_cast<RefLinear*>(h); }
int ref_linear_forward(void* h, const float* x, int64_t tokens, int step, float* y) {
    return guarded([&] {
        auto* r = static_cast<RefLinear*>(h);
        const DenseMatrix out = r->l->forward(make_dense(x, tokens, r->in), step);
        std::memcpy(y, out.data(), out.size() * sizeof(float));
    });
}
int ref_linear_backward(void* h, const float* gy, int64_t tokens, int step, float* gx) {
    return guarded([&] {
        auto* r = static_cast<RefLinear*>(h);
        const DenseMatrix out = r->l->backward(make_dense(gy, tokens, r->out), step);
        std::memcpy(gx, out.data(), out.size() * sizeof(float));
    });
}
int ref_linear_grad(void* h, float* gw) {
    return guarded([&] {
        auto* r = static_cast<RefLinear*>(h);
        std::memcpy(gw, r->l->grad_weight().data(), r->l->grad_weight().size() * 4);
    });
}
// last observed rate, then controller_step (trainsim.cpp:129-133) and the new threshold
int ref_linear_controller(void* h, double* rate, double* threshold) {
    return guarded([&] {
        auto* r = static_cast<RefLinear*>(h);
        *rate = r->l->last_fallback_rate();
        r->l->controller_step();
        *threshold = r->l->threshold();
    });
}
int ref_linear_zero_grad(void* h) {
    return guarded([&] { static_cast<RefLinear*>(h)->l->zero_grad(); });
}
int ref_linear_sgd(void* h, double lr) {
    return guarded([&] { static_cast<RefLinear*>(h)->l->apply_sgd(lr); });
}
int ref_linear_weight(void* h, float* w) {
    return guarded([&] {
        auto* r = static_cast<RefLinear*>(h);
        std::memcpy(w, r->l->weight().data(), r->l->weight().size() * 4);
    });
}

// ---------------------------------------------------------------------------
// .fmat I/O (matrix.cpp:92-140): status 0, or 1 with FormatError's byte offset.
int ref_fmat_save(const char* path, const float* data, int64_t rows, int64_t cols) {
    return guarded([&] { save_matrix(make_dense(data, rows, cols), path); });
}
int ref_fmat_load(const char* path, float* data, int64_t capacity, int64_t* rows, int64_t* cols,
                  uint64_t* err_offset) {
    try {
        const DenseMatrix m = load_matrix(path);
        *rows = m.rows();
        *cols = m.cols();
        if (m.size() > capacity) return 2;
        std::memcpy(data, m.data(), m.size() * sizeof(float));
        return 0;
    } catch (const FormatError& e) {
        *err_offset = e.byte_offset();
        g_err = e.what();
        return 1;
    }
}

// ---------------------------------------------------------------------------
// RmsNorm (trainsim.hpp:75-97) with the default QuantConfig (10-bit 1 x 128 context).
struct RefRms {
    QuantConfig cfg;
    std::unique_ptr<RmsNorm> n;
    int64_t dim = 0;
};
void* ref_rms_create(int64_t dim) {
    try {
        auto* r = new RefRms;
        r->dim = dim;
        r->n = std::make_unique<RmsNorm>("norm", dim, r->cfg);
        return r;
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}
void ref_rms_destroy(void* h) { delete static_cast<RefRms*>(h); }
int ref_rms_forward(void* h, const float* x, int64_t rows, float* y) {
    return guarded([&] {
        auto* r = static_cast<RefRms*>(h);
        const DenseMatrix out = r->n->forward(make_dense(x, rows, r->dim));
        std::memcpy(y, out.data(), out.size() * sizeof(float));
    });
}
int ref_rms_backward(void* h, const float* gy, int64_t rows, float* gx) {
    return guarded([&] {
        auto* r = static_cast<RefRms*>(h);
        const DenseMatrix out = r->n->backward(make_dense(gy, rows, r->dim));
        std::memcpy(gx, out.data(), out.size() * sizeof(float));
    });
}
int ref_rms_state(void* h, float* gain, float* grad_gain) {
    return guarded([&] {
        auto* r = static_cast<RefRms*>(h);
        std::memcpy(gain, r->n->gain().data(), r->dim * 4);
        std::memcpy(grad_gain, r->n->grad_gain().data(), r->dim * 4);
    });
}
int ref_rms_sgd(void* h, double lr) {
    return guarded([&] { static_cast<RefRms*>(h)->n->apply_sgd(lr); });
}

// ---------------------------------------------------------------------------
// The reference's own pre-norm residual GLU block (trainsim.hpp:136-146,
// trainsim.cpp:294-308): h + down(silu(gate(norm(h))) * up(norm(h))); layer
// ids 0 / 1 / 2 as RefMlp, block side g.
struct RefBlock {
    QuantConfig cfg;
    std::unique_ptr<GluBlock> b;
    int64_t d = 0, f = 0;
};
void* ref_block_create(const float* w_gate, const float* w_up, const float* w_down, int64_t d_model,
                       int64_t d_ff, int64_t g, double threshold) {
    try {
        auto* r = new RefBlock;
        r->cfg.block = g;
        r->cfg.threshold_init = threshold;
        r->d = d_model;
        r->f = d_ff;
        r->b = std::unique_ptr<GluBlock>(new GluBlock{
            RmsNorm("norm", d_model, r->cfg),
            QuantLinearLayer("gate", 0, make_dense(w_gate, d_ff, d_model), r->cfg),
            QuantLinearLayer("up", 1, make_dense(w_up, d_ff, d_model), r->cfg),
            QuantLinearLayer("down", 2, make_dense(w_down, d_model, d_ff), r->cfg),
            GluCombine(r->cfg)});
        return r;
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}
void ref_block_destroy(void* h) { delete static_cast<RefBlock*>(h); }
// one forward + backward: out = block(x), grad_h = block.backward(grad_out)
int ref_block_step(void* h, const float* x, const float* grad_out, int64_t tokens, int step, float* out,
                   float* grad_h) {
    return guarded([&] {
        auto* r = static_cast<RefBlock*>(h);
        const DenseMatrix y = r->b->forward(make_dense(x, tokens, r->d), step);
        std::memcpy(out, y.data(), y.size() * sizeof(float));
        const DenseMatrix gx = r->b->backward(make_dense(grad_out, tokens, r->d), step);
        std::memcpy(grad_h, gx.data(), gx.size() * sizeof(float));
    });
}
// controller_step of gate, up, down; thresholds after the update
int ref_block_controller(void* h, double* thresholds3) {
    return guarded([&] {
        auto* r = static_cast<RefBlock*>(h);
        QuantLinearLayer* ls[3] = {&r->b->gate, &r->b->up, &r->b->down};
        for (int i = 0; i < 3; ++i) {
            ls[i]->controller_step();
            thresholds3[i] = ls[i]->threshold();
        }
    });
}
int ref_block_sgd(void* h, double lr) {
    return guarded([&] {
        auto* r = static_cast<RefBlock*>(h);
        r->b->norm.apply_sgd(lr);
        r->b->gate.apply_sgd(lr);
        r->b->up.apply_sgd(lr);
        r->b->down.apply_sgd(lr);
    });
}
// gain, grad_gain (d_model); weights and their gradients of gate, up, down
int ref_block_state(void* h, float* gain, float* grad_gain, float* wg, float* wu, float* wd, float* gg,
                    float* gu, float* gd) {
    return guarded([&] {
        auto* r = static_cast<RefBlock*>(h);
        std::memcpy(gain, r->b->norm.gain().data(), r->d * 4);
        std::memcpy(grad_gain, r->b->norm.grad_gain().data(), r->d * 4);
        const size_t n = (size_t)(r->d * r->f) * 4;
        std::memcpy(wg, r->b->gate.weight().data(), n);
        std::memcpy(wu, r->b->up.weight().data(), n);
        std::memcpy(wd, r->b->down.weight().data(), n);
        std::memcpy(gg, r->b->gate.grad_weight().data(), n);
        std::memcpy(gu, r->b->up.grad_weight().data(), n);
        std::memcpy(gd, r->b->down.grad_weight().data(), n);
    });
}

// ---------------------------------------------------------------------------
// SiluLayer (trainsim.hpp:118-131, trainsim.cpp:265-290)
struct RefSilu {
    QuantConfig cfg;
    std::unique_ptr<SiluLayer> l;
};
void* ref_silu_create() {
    try {
        auto* r = new RefSilu;
        r->l = std::make_unique<SiluLayer>(r->cfg);
        return r;
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}
void ref_silu_destroy(void* h) { delete static_cast<RefSilu*>(h); }
int ref_silu_forward(void* h, const float* x, int64_t rows, int64_t cols, float* y) {
    return guarded([&] {
        const DenseMatrix out = static_cast<RefSilu*>(h)->l->forward(make_dense(x, rows, cols));
        std::memcpy(y, out.data(), out.size() * sizeof(float));
    });
}
int ref_silu_backward(void* h, const float* gy, int64_t rows, int64_t cols, float* gx) {
    return guarded([&] {
        const DenseMatrix out = static_cast<RefSilu*>(h)->l->backward(make_dense(gy, rows, cols));
        std::memcpy(gx, out.data(), out.size() * sizeof(float));
    });
}

} // extern "C"
