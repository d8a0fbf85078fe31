/* TEST INFRASTRUCTURE ONLY -- CPU checker for the B200 path; see fbq_oracle.h.
 * Compiled with -ffp-contract=off like the reference (proj/CMakeLists.txt:11-13):
 * every float op below is a single IEEE-rounded operation. */
#include "fbq_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

static int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; } /* matrix.hpp:59 */
static int64_t imin(int64_t a, int64_t b) { return a < b ? a : b; }

/* ---- rng.hpp ---------------------------------------------------------- */
uint64_t orc_mix64(uint64_t z) { /* rng.hpp:11-15 */
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
uint64_t orc_bits_at(uint64_t seed, uint64_t n) { /* rng.hpp:28-30 */
    return orc_mix64(seed + (n + 1) * 0x9E3779B97F4A7C15ull);
}
double orc_uniform_at(uint64_t seed, uint64_t n) { /* rng.hpp:33-35 */
    return (double)(orc_bits_at(seed, n) >> 11) * 0x1.0p-53;
}
float orc_normal_at(uint64_t seed, uint64_t n) { /* rng.hpp:38-44 */
    const uint64_t w = orc_bits_at(seed, n);
    const double u1 = ((double)(w >> 32) + 1.0) * 0x1.0p-32;
    const double u2 = (double)(w & 0xFFFFFFFFull) * 0x1.0p-32;
    const double r = sqrt(-2.0 * log(u1));
    return (float)(r * cos(6.283185307179586 * u2));
}
uint64_t orc_derive_seed(uint64_t base, uint64_t a, uint64_t b) { /* rng.hpp:56-58 */
    return orc_bits_at(orc_bits_at(base, a), b);
}
uint64_t orc_layer_seed(uint64_t base, int layer_id, uint64_t tag, int step) {
    /* trainsim.cpp:16-19 */
    return orc_derive_seed(base, (uint64_t)layer_id * 4 + tag, (uint64_t)step);
}

/* ---- kernels.cpp (scalar backend) -------------------------------------- */
float orc_absmax_2d(const float* x, size_t rows, size_t cols, size_t ld) { /* :12-22 */
    float m = 0.0f;
    for (size_t r = 0; r < rows; ++r)
        for (size_t c = 0; c < cols; ++c) {
            const float v = fabsf(x[r * ld + c]);
            if (v > m) m = v;
        }
    return m;
}

void orc_quantize_rtn_2d(const float* x, size_t ldx, int16_t* q, size_t ldq, size_t rows,
                         size_t cols, float scale, int32_t limit) { /* :24-40 */
    const double inv = (double)scale, lo = -(double)limit, hi = (double)limit;
    for (size_t r = 0; r < rows; ++r)
        for (size_t c = 0; c < cols; ++c) {
            double t = (double)x[r * ldx + c] / inv;
            t = nearbyint(t); /* ties-to-even, default rounding mode */
            if (t > hi) t = hi;
            if (t < lo) t = lo;
            q[r * ldq + c] = (int16_t)t;
        }
}

void orc_dequantize_2d(const int16_t* q, size_t ldq, float* y, size_t ldy, size_t rows,
                       size_t cols, float scale) { /* :42-51 */
    for (size_t r = 0; r < rows; ++r)
        for (size_t c = 0; c < cols; ++c) y[r * ldy + c] = (float)q[r * ldq + c] * scale;
}

void orc_gemm_i16_accum(const int16_t* a, size_t lda, const int16_t* b, size_t ldb, int32_t* c,
                        size_t ldc, size_t m, size_t n, size_t k) { /* :53-67 */
    for (size_t i = 0; i < m; ++i)
        for (size_t kk = 0; kk < k; ++kk) {
            const int32_t av = a[i * lda + kk];
            for (size_t j = 0; j < n; ++j) c[i * ldc + j] += av * (int32_t)b[kk * ldb + j];
        }
}

void orc_scale_accum(float* acc, const int32_t* p, size_t n, float scale) { /* :69-74 */
    for (size_t i = 0; i < n; ++i) {
        const float v = scale * (float)p[i];
        acc[i] = acc[i] + v;
    }
}

/* ---- quant.cpp --------------------------------------------------------- */
static int32_t level_of(int bits) { return (1 << (bits - 1)) - 1; } /* quant.hpp:16 */

static float block_scale(const float* v, int64_t rows, int64_t cols, int64_t ld, int32_t level) {
    /* quant.cpp:27-32 */
    const float amax = orc_absmax_2d(v, (size_t)rows, (size_t)cols, (size_t)ld);
    return amax > 0.0f ? amax / (float)level : 0.0f;
}

int orc_quantize_rtn(const float* x, int64_t rows, int64_t cols, int64_t gr_, int64_t gc_,
                     int bits, int16_t* codes, float* scales) { /* quant.cpp:36-53 */
    if (bits < 2 || bits > 16 || gr_ < 1 || gc_ < 1) return 1;
    const int32_t level = level_of(bits);
    const int64_t gr = cdiv(rows, gr_), gc = cdiv(cols, gc_);
    memset(codes, 0, (size_t)(rows * cols) * sizeof(int16_t));
    for (int64_t bi = 0; bi < gr; ++bi)
        for (int64_t bj = 0; bj < gc; ++bj) {
            const int64_t r0 = bi * gr_, c0 = bj * gc_;
            const int64_t er = imin(gr_, rows - r0), ec = imin(gc_, cols - c0);
            const float* v = x + r0 * cols + c0;
            const float a = block_scale(v, er, ec, cols, level);
            scales[bi * gc + bj] = a;
            if (a == 0.0f) continue;
            orc_quantize_rtn_2d(v, (size_t)cols, codes + r0 * cols + c0, (size_t)cols, (size_t)er,
                                (size_t)ec, a, level);
        }
    return 0;
}

int orc_quantize_stochastic(const float* x, int64_t rows, int64_t cols, int64_t gr_, int64_t gc_,
                            int bits, uint64_t seed, int64_t row_offset, int16_t* codes,
                            float* scales) { /* quant.cpp:55-84 */
    if (bits < 2 || bits > 16 || gr_ < 1 || gc_ < 1) return 1;
    const int32_t level = level_of(bits);
    const int64_t gr = cdiv(rows, gr_), gc = cdiv(cols, gc_);
    memset(codes, 0, (size_t)(rows * cols) * sizeof(int16_t));
    for (int64_t bi = 0; bi < gr; ++bi)
        for (int64_t bj = 0; bj < gc; ++bj) {
            const int64_t r0 = bi * gr_, c0 = bj * gc_;
            const int64_t er = imin(gr_, rows - r0), ec = imin(gc_, cols - c0);
            const float* v = x + r0 * cols + c0;
            const float a = block_scale(v, er, ec, cols, level);
            scales[bi * gc + bj] = a;
            if (a == 0.0f) continue;
            for (int64_t r = 0; r < er; ++r)
                for (int64_t c = 0; c < ec; ++c) {
                    const int64_t lin = (row_offset + r0 + r) * cols + (c0 + c);
                    const double t = (double)v[r * cols + c] / (double)a;
                    double f = floor(t);
                    const double frac = t - f;
                    if (frac > 0.0 && orc_uniform_at(seed, (uint64_t)lin) < frac) f += 1.0;
                    if (f > level) f = level;
                    if (f < -level) f = -level;
                    codes[(r0 + r) * cols + c0 + c] = (int16_t)f;
                }
        }
    return 0;
}

int orc_dequantize(const int16_t* codes, const float* scales, int64_t rows, int64_t cols,
                   int64_t gr_, int64_t gc_, float* out) { /* quant.cpp:86-104 */
    const int64_t gr = cdiv(rows, gr_), gc = cdiv(cols, gc_);
    memset(out, 0, (size_t)(rows * cols) * sizeof(float));
    for (int64_t bi = 0; bi < gr; ++bi)
        for (int64_t bj = 0; bj < gc; ++bj) {
            const float a = scales[bi * gc + bj];
            const int64_t r0 = bi * gr_, c0 = bj * gc_;
            const int64_t er = imin(gr_, rows - r0), ec = imin(gc_, cols - c0);
            if (a == 0.0f) continue;
            orc_dequantize_2d(codes + r0 * cols + c0, (size_t)cols, out + r0 * cols + c0,
                              (size_t)cols, (size_t)er, (size_t)ec, a);
        }
    return 0;
}

int orc_transpose_qt(const int16_t* codes, const float* scales, int64_t rows, int64_t cols,
                     int64_t gr_, int64_t gc_, int16_t* out_codes, float* out_scales) {
    /* quant.cpp:106-126 */
    for (int64_t r = 0; r < rows; ++r)
        for (int64_t c = 0; c < cols; ++c) out_codes[c * rows + r] = codes[r * cols + c];
    const int64_t gr = cdiv(rows, gr_), gc = cdiv(cols, gc_);
    for (int64_t bi = 0; bi < gr; ++bi)
        for (int64_t bj = 0; bj < gc; ++bj) out_scales[bj * gr + bi] = scales[bi * gc + bj];
    return 0;
}

int orc_fallback_quantize(const float* x, int64_t rows, int64_t cols, int64_t g,
                          const uint8_t* mask, int16_t* codes, float* scales, int16_t* res_codes,
                          float* res_scales) { /* quant.cpp:128-176 */
    const int64_t gr = cdiv(rows, g), gc = cdiv(cols, g);
    const int32_t level = 127;
    if (orc_quantize_rtn(x, rows, cols, g, g, 8, codes, scales)) return 1;
    memset(res_codes, 0, (size_t)(rows * cols) * sizeof(int16_t));
    memset(res_scales, 0, (size_t)(gr * gc) * sizeof(float));
    float* res = (float*)malloc((size_t)(g * g) * sizeof(float));
    if (!res) return 1;
    for (int64_t bi = 0; bi < gr; ++bi)
        for (int64_t bj = 0; bj < gc; ++bj) {
            if (!mask[bi * gc + bj]) continue;
            const int64_t r0 = bi * g, c0 = bj * g;
            const int64_t er = imin(g, rows - r0), ec = imin(g, cols - c0);
            const float a = scales[bi * gc + bj];
            for (int64_t r = 0; r < er; ++r)
                for (int64_t c = 0; c < ec; ++c) { /* :150-157 */
                    const float rec = (float)codes[(r0 + r) * cols + c0 + c] * a;
                    res[r * ec + c] = x[(r0 + r) * cols + c0 + c] - rec;
                }
            const float amax = orc_absmax_2d(res, (size_t)er, (size_t)ec, (size_t)ec);
            const float rs = amax > 0.0f ? amax / (float)level : 0.0f; /* :161-164 */
            res_scales[bi * gc + bj] = rs;
            if (rs != 0.0f)
                orc_quantize_rtn_2d(res, (size_t)ec, res_codes + r0 * cols + c0, (size_t)cols,
                                    (size_t)er, (size_t)ec, rs, level);
        }
    free(res);
    return 0;
}

int orc_dequantize_fallback(const int16_t* codes, const float* scales, const uint8_t* mask,
                            const int16_t* res_codes, const float* res_scales, int64_t rows,
                            int64_t cols, int64_t g, float* out) { /* quant.cpp:178-202 */
    orc_dequantize(codes, scales, rows, cols, g, g, out);
    const int64_t gr = cdiv(rows, g), gc = cdiv(cols, g);
    for (int64_t bi = 0; bi < gr; ++bi)
        for (int64_t bj = 0; bj < gc; ++bj) {
            if (!mask[bi * gc + bj]) continue;
            const int64_t r0 = bi * g, c0 = bj * g;
            const int64_t er = imin(g, rows - r0), ec = imin(g, cols - c0);
            const float rs = res_scales[bi * gc + bj];
            for (int64_t r = 0; r < er; ++r)
                for (int64_t c = 0; c < ec; ++c) {
                    float* o = out + (r0 + r) * cols + c0 + c;
                    *o += (float)res_codes[(r0 + r) * cols + c0 + c] * rs;
                }
        }
    return 0;
}

/* ---- gemm.cpp ---------------------------------------------------------- */
int orc_block_gemm(const int16_t* a_codes, const float* a_scales, const uint8_t* mask,
                   const int16_t* res_codes, const float* res_scales, const int16_t* b_codes,
                   const float* b_scales, int64_t m, int64_t n, int64_t k, int64_t g,
                   int64_t tile_m, int64_t tile_n, int64_t tile_k, float* out) {
    /* gemm.cpp:101-186: per output block, ascending bk, primary then residual */
    if ((int64_t)g * 127 * 127 >= (1ll << 31)) return 1; /* :90-94 */
    const int tiled = tile_m > 0;
    if (tiled && (g % tile_m || g % tile_n || g % tile_k)) return 1; /* :106-108 */
    const int64_t mb = cdiv(m, g), nb = cdiv(n, g), kb = cdiv(k, g);
    int32_t* pbuf = (int32_t*)malloc((size_t)(g * g) * sizeof(int32_t));
    float* cbuf = (float*)malloc((size_t)(g * g) * sizeof(float));
    if (!pbuf || !cbuf) return 1;
    for (int64_t bi = 0; bi < mb; ++bi)
        for (int64_t bj = 0; bj < nb; ++bj) {
            const int64_t r0 = bi * g, c0 = bj * g;
            const int64_t er = imin(g, m - r0), ec = imin(g, n - c0);
            const size_t cells = (size_t)(er * ec);
            memset(cbuf, 0, cells * sizeof(float));
            for (int64_t bk = 0; bk < kb; ++bk) {
                const int64_t k0 = bk * g, ek = imin(g, k - k0);
                const int16_t* ap = a_codes + r0 * k + k0;
                const int16_t* bp = b_codes + k0 * n + c0;
                memset(pbuf, 0, cells * sizeof(int32_t));
                if (!tiled) {
                    orc_gemm_i16_accum(ap, (size_t)k, bp, (size_t)n, pbuf, (size_t)ec, (size_t)er,
                                       (size_t)ec, (size_t)ek);
                } else { /* :146-162 */
                    for (int64_t tm = 0; tm < er; tm += tile_m)
                        for (int64_t tn = 0; tn < ec; tn += tile_n)
                            for (int64_t tk = 0; tk < ek; tk += tile_k)
                                orc_gemm_i16_accum(ap + tm * k + tk, (size_t)k, bp + tk * n + tn,
                                                   (size_t)n, pbuf + tm * ec + tn, (size_t)ec,
                                                   (size_t)imin(tile_m, er - tm),
                                                   (size_t)imin(tile_n, ec - tn),
                                                   (size_t)imin(tile_k, ek - tk));
                }
                const float s = a_scales[bi * kb + bk] * b_scales[bk * nb + bj]; /* :163 */
                orc_scale_accum(cbuf, pbuf, cells, s);
                if (mask && mask[bi * kb + bk]) { /* :166-175 */
                    memset(pbuf, 0, cells * sizeof(int32_t));
                    orc_gemm_i16_accum(res_codes + r0 * k + k0, (size_t)k, bp, (size_t)n, pbuf,
                                       (size_t)ec, (size_t)er, (size_t)ec, (size_t)ek);
                    const float s2 = res_scales[bi * kb + bk] * b_scales[bk * nb + bj];
                    orc_scale_accum(cbuf, pbuf, cells, s2);
                }
            }
            for (int64_t r = 0; r < er; ++r)
                memcpy(out + (r0 + r) * n + c0, cbuf + r * ec, (size_t)ec * sizeof(float));
        }
    free(pbuf);
    free(cbuf);
    return 0;
}

int orc_block_products(const int16_t* a_codes, const int16_t* b_codes, int64_t m, int64_t n,
                       int64_t k, int64_t g, int32_t* out) {
    const int64_t mb = cdiv(m, g), nb = cdiv(n, g), kb = cdiv(k, g);
    for (int64_t bi = 0; bi < mb; ++bi)
        for (int64_t bj = 0; bj < nb; ++bj)
            for (int64_t bk = 0; bk < kb; ++bk) {
                int32_t* p = out + ((bi * nb + bj) * kb + bk) * g * g;
                memset(p, 0, (size_t)(g * g) * sizeof(int32_t));
                const int64_t r0 = bi * g, c0 = bj * g, k0 = bk * g;
                orc_gemm_i16_accum(a_codes + r0 * k + k0, (size_t)k, b_codes + k0 * n + c0,
                                   (size_t)n, p, (size_t)g, (size_t)imin(g, m - r0),
                                   (size_t)imin(g, n - c0), (size_t)imin(g, k - k0));
            }
    return 0;
}

int orc_gemm_oracle(const float* a, const float* b, int64_t m, int64_t n, int64_t k,
                    float* out) { /* gemm.cpp:56-74 */
    double* acc = (double*)malloc((size_t)n * sizeof(double));
    if (!acc) return 1;
    for (int64_t i = 0; i < m; ++i) {
        memset(acc, 0, (size_t)n * sizeof(double));
        for (int64_t kk = 0; kk < k; ++kk) {
            const double av = (double)a[i * k + kk];
            for (int64_t j = 0; j < n; ++j) acc[j] += av * (double)b[kk * n + j];
        }
        for (int64_t j = 0; j < n; ++j) out[i * n + j] = (float)acc[j];
    }
    free(acc);
    return 0;
}

/* ---- policy.cpp -------------------------------------------------------- */
int orc_score_blocks_absmax(const float* x, int64_t rows, int64_t cols, int64_t g,
                            double* scores) { /* policy.cpp:18-27 */
    const int64_t gr = cdiv(rows, g), gc = cdiv(cols, g);
    for (int64_t bi = 0; bi < gr; ++bi)
        for (int64_t bj = 0; bj < gc; ++bj) {
            const int64_t r0 = bi * g, c0 = bj * g;
            scores[bi * gc + bj] = orc_absmax_2d(x + r0 * cols + c0, (size_t)imin(g, rows - r0),
                                                 (size_t)imin(g, cols - c0), (size_t)cols);
        }
    return 0;
}

int orc_mask_threshold(const double* scores, int64_t n, double theta, uint8_t* mask) {
    if (!(theta > 0.0)) return 1; /* policy.cpp:74 */
    for (int64_t i = 0; i < n; ++i) mask[i] = scores[i] > theta ? 1 : 0; /* :77 */
    return 0;
}

static const double* g_sort_scores;
static int topk_cmp(const void* pa, const void* pb) { /* policy.cpp:64-67 */
    const int64_t i = *(const int64_t*)pa, j = *(const int64_t*)pb;
    if (g_sort_scores[i] != g_sort_scores[j]) return g_sort_scores[i] > g_sort_scores[j] ? -1 : 1;
    return i < j ? -1 : (i > j);
}

int orc_mask_topk(const double* scores, int64_t n, double rate, uint8_t* mask) {
    if (rate < 0.0 || rate > 1.0) return 1; /* policy.cpp:57 */
    int64_t kk = (int64_t)ceil(rate * (double)n);
    if (kk > n) kk = n;
    int64_t* order = (int64_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
    if (!order) return 1;
    for (int64_t i = 0; i < n; ++i) order[i] = i;
    g_sort_scores = scores;
    qsort(order, (size_t)n, sizeof(int64_t), topk_cmp);
    memset(mask, 0, (size_t)n);
    for (int64_t i = 0; i < kk; ++i) mask[order[i]] = 1;
    free(order);
    return 0;
}

double orc_mask_rate(const uint8_t* mask, int64_t n) { /* policy.cpp:82-87 */
    if (n == 0) return 0.0;
    int64_t set = 0;
    for (int64_t i = 0; i < n; ++i) set += mask[i] != 0;
    return (double)set / (double)n;
}

int orc_controller_update(double threshold, double observed, double r_min, double r_max,
                          double alpha, double* out_threshold) { /* policy.cpp:89-109 */
    if (!(0.0 <= r_min && r_min < r_max && r_max <= 1.0) || !(alpha > 1.0)) return 1;
    if (observed < 0.0 || observed > 1.0) return 1;
    if (observed < r_min) threshold /= alpha;
    else if (observed > r_max) threshold *= alpha;
    *out_threshold = threshold;
    return 0;
}

int orc_compare(const float* actual, const float* reference, int64_t n, double* out4) {
    /* gemm.cpp:205-239 */
    double sq = 0.0, max_err = 0.0, dot = 0.0, na = 0.0, nr = 0.0;
    int64_t ref_nonzero = 0, underflow = 0;
    for (int64_t i = 0; i < n; ++i) {
        const double a = actual[i], r = reference[i], d = a - r;
        sq += d * d;
        if (fabs(d) > max_err) max_err = fabs(d);
        dot += a * r;
        na += a * a;
        nr += r * r;
        if (r != 0.0) {
            ++ref_nonzero;
            if (a == 0.0) ++underflow;
        }
    }
    out4[0] = n > 0 ? sqrt(sq / (double)n) : 0.0;
    out4[1] = max_err;
    if (na == 0.0 && nr == 0.0) out4[2] = 1.0;
    else if (na == 0.0 || nr == 0.0) out4[2] = 0.0;
    else {
        double c = dot / sqrt(na * nr);
        out4[2] = c < -1.0 ? -1.0 : (c > 1.0 ? 1.0 : c);
    }
    out4[3] = ref_nonzero > 0 ? (double)underflow / (double)ref_nonzero : 0.0;
    return 0;
}
