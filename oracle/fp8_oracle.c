/*
 * fp8_oracle.c -- TEST INFRASTRUCTURE ONLY (see fp8_oracle.h).
 *
 * A CPU restatement of the reference fp8emu hot path. Each function cites the
 * reference file:line it follows (paths relative to /root/reference/proj).
 * Compiled with -O2 -ffp-contract=off so FP32 arithmetic is plain IEEE
 * binary32 with no FMA contraction, like the reference objects.
 *
 * Parity of this file is pinned in tests/test_oracle.py against the golden
 * vectors frozen in the reference's own tests and against the compiled
 * reference (oracle/_ref/libfp8emu_ref.so).
 */
#include "fp8_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---- seed mixing: lfsr.cpp:47-52 (mix64 = SplitMix64), lfsr.hpp:46-48 ---- */
uint64_t or_mix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

uint64_t or_mix_seed(uint64_t seed, uint64_t index) {
    return or_mix64(seed + 0x9E3779B97F4A7C15ull * (index + 1));
}

/* ---- LFSR: lfsr.cpp:17-27 (taps 16,15,13,4 = state bits 0,1,3,12) ---- */
uint32_t or_lfsr_next_bits(uint16_t *state, int sample_bits) {
    uint32_t out = 0;
    for (int i = 0; i < sample_bits; ++i) {
        const uint16_t s = *state;
        const uint16_t bit = (uint16_t)(((s >> 0) ^ (s >> 1) ^ (s >> 3) ^ (s >> 12)) & 1u);
        *state = (uint16_t)((s >> 1) | (bit << 15));
        out = (out << 1) | (s & 1u);
    }
    return out;
}

/* lfsr.cpp:34-45 */
uint16_t or_lfsr_split(uint64_t seed, uint64_t stream_index) {
    uint64_t h = or_mix_seed(seed, stream_index);
    uint16_t s = (uint16_t)(h & 0xFFFFu);
    while (s == 0) {
        h = or_mix64(h + 1);
        s = (uint16_t)(h & 0xFFFFu);
    }
    return s;
}

/* ---- format constants: float_format.hpp:30-78, float_format.cpp:27-39 ---- */
static int mant_bits(int fmt) { return fmt == OR_FMT_E5M2 ? 2 : 10; }
static uint32_t sign_mask(int fmt) { return 1u << (5 + mant_bits(fmt)); }
static uint32_t code_mask(int fmt) { return (1u << (6 + mant_bits(fmt))) - 1u; }
static uint32_t max_code(int fmt) { int mb = mant_bits(fmt); return (30u << mb) | ((1u << mb) - 1u); }
static uint32_t inf_code(int fmt) { return 31u << mant_bits(fmt); }
static uint32_t nan_code(int fmt) { return inf_code(fmt) | (1u << (mant_bits(fmt) - 1)); }
static double max_normal(int fmt) {
    const int mb = mant_bits(fmt);
    return (2.0 - ldexp(1.0, -mb)) * ldexp(1.0, 30 - 15);
}
static double min_normal(void) { return ldexp(1.0, 1 - 15); }
static double min_subnormal(int fmt) { return ldexp(1.0, 1 - 15 - mant_bits(fmt)); }

/* float_format.cpp:52-71 */
double or_decode(uint32_t code, int fmt) {
    const int mb = mant_bits(fmt);
    code &= code_mask(fmt);
    const int negative = (code & sign_mask(fmt)) != 0;
    const uint32_t efield = (code >> mb) & 31u;
    const uint32_t mfield = code & ((1u << mb) - 1u);
    double v;
    if (efield == 31u) {
        if (mfield != 0) return NAN;
        v = INFINITY;
    } else if (efield == 0) {
        v = ldexp((double)mfield, 1 - 15 - mb);
    } else {
        const double significand = 1.0 + ldexp((double)mfield, -mb);
        v = significand * ldexp(1.0, (int)efield - 15);
    }
    return negative ? -v : v;
}

/* float_format.cpp:78-93 (floor_code) */
static uint32_t floor_code(double a, int fmt, double *step) {
    const int mb = mant_bits(fmt);
    if (a < min_normal()) {
        *step = min_subnormal(fmt);
        return (uint32_t)(a / *step);
    }
    int e2 = 0;
    frexp(a, &e2);
    const int unbiased = e2 - 1;
    const double mant = ldexp(a, -unbiased);
    const uint32_t m = (uint32_t)ldexp(mant - 1.0, mb);
    const uint32_t efield = (uint32_t)(unbiased + 15);
    *step = ldexp(1.0, unbiased - mb);
    return (efield << (uint32_t)mb) | m;
}

/* float_format.cpp:97-135. r16_given >= 0 supplies the SR sample directly
 * (the supplied-bits / counter-bits extensions); otherwise *lfsr is clocked
 * 16 times (lfsr.cpp:29-32 next_fraction). */
static uint32_t encode_impl(double x, int fmt, int mode, uint16_t *lfsr,
                            int32_t r16_given, int saturate, int *ovf,
                            int *unf, int *consumed) {
    *ovf = 0; *unf = 0; if (consumed) *consumed = 0;
    if (isnan(x)) return nan_code(fmt);
    const uint32_t sign = signbit(x) ? sign_mask(fmt) : 0u;
    const double a = fabs(x);
    if (a > max_normal(fmt)) {
        *ovf = 1;
        return sign | (saturate ? max_code(fmt) : inf_code(fmt));
    }
    if (a == 0.0) return sign;
    double step;
    uint32_t code = floor_code(a, fmt, &step);
    const double lo = or_decode(code, fmt);
    if (lo != a) {
        if (mode == OR_RNE) {
            const double mid = lo + 0.5 * step;
            if (a > mid || (a == mid && (code & 1u))) ++code;
        } else if (mode == OR_SR) {
            uint32_t bits;
            if (r16_given >= 0) bits = (uint32_t)r16_given;
            else bits = or_lfsr_next_bits(lfsr, 16);
            if (consumed) *consumed = 1;
            const double r = ((double)bits / 65536.0) * step;
            if ((a - lo) + r >= step) ++code;
        }
    }
    *unf = (code == 0);
    return sign | code;
}

uint32_t or_encode(double x, int fmt, int mode, uint16_t *lfsr, int saturate,
                   int *overflowed, int *underflowed, int *consumed) {
    return encode_impl(x, fmt, mode, lfsr, -1, saturate, overflowed,
                       underflowed, consumed);
}

/* SURVEY 8a A2': the same encode as integer operations on the FP32 bits.
 * This is the rule the CUDA kernels implement; tests check it against
 * or_encode / the reference. */
uint32_t or_encode_bits(uint32_t u, int fmt, int mode, uint32_t r16,
                        int saturate, int *overflowed, int *underflowed,
                        int *inexact) {
    const int mb = mant_bits(fmt);
    const uint32_t a = u & 0x7FFFFFFFu;
    const uint32_t e = a >> 23, m = a & 0x7FFFFFu;
    const uint32_t sign_out = (u >> 31) ? (1u << (5 + mb)) : 0u;
    const uint32_t maxbits = mb == 2 ? 0x47600000u : 0x477FE000u;
    *overflowed = 0; *underflowed = 0; *inexact = 0;
    if (e == 255u && m != 0) return nan_code(fmt);
    if (a > maxbits) {
        *overflowed = 1;
        return sign_out | (saturate ? max_code(fmt) : inf_code(fmt));
    }
    if (a == 0) return sign_out;
    uint32_t code0, dbits;
    uint64_t d;
    if (e >= 113u) {
        dbits = 23u - (uint32_t)mb;
        code0 = ((e - 112u) << mb) | (m >> dbits);
        d = m & ((1u << dbits) - 1u);
    } else {
        const uint32_t sig = e ? (0x800000u | m) : m;
        dbits = 136u - (uint32_t)mb - (e ? e : 1u);
        if (dbits >= 24u) { code0 = 0; d = sig; }
        else { code0 = sig >> dbits; d = sig & ((1u << dbits) - 1u); }
    }
    if (d == 0) return sign_out | code0;
    *inexact = 1;
    uint32_t up = 0;
    if (mode == OR_RNE) {
        if (dbits <= 32u) {
            const uint64_t half = 1ull << (dbits - 1u);
            up = (d > half) || (d == half && (code0 & 1u));
        }
    } else if (mode == OR_SR) {
        uint64_t r;
        if (dbits >= 16u) r = (dbits - 16u >= 24u) ? 0 : (d >> (dbits - 16u));
        else r = d << (16u - dbits);
        up = (r + r16) >= 65536u;
    }
    const uint32_t code = code0 + up;
    *underflowed = (code == 0);
    return sign_out | code;
}

/* tensor.cpp:46-81 (+ bits-source / block_offset extensions). */
int or_quantize(const float *x, int64_t n, int fmt, int mode, int bits_source,
                uint64_t seed, int saturate, int64_t block_offset,
                const uint32_t *rbits, uint16_t *codes_out, int64_t *counters) {
    if (seed == 0) return 22; /* tensor.cpp:48 */
    int64_t ovf = 0, unf = 0, nan = 0;
    const int64_t kBlock = 4096; /* tensor.hpp:65 kQuantBlock */
    if (mode == OR_SR && bits_source == OR_BITS_LFSR) {
        for (int64_t block = 0; block * kBlock < n; ++block) {
            uint16_t st = or_lfsr_split(seed, (uint64_t)(block + block_offset));
            const int64_t end = (block + 1) * kBlock < n ? (block + 1) * kBlock : n;
            for (int64_t i = block * kBlock; i < end; ++i) {
                int o, u;
                const uint32_t c = encode_impl((double)x[i], fmt, OR_SR, &st, -1,
                                               saturate, &o, &u, 0);
                codes_out[i] = (uint16_t)c;
                ovf += o; unf += u; nan += isnan(x[i]) ? 1 : 0;
            }
        }
    } else {
        for (int64_t i = 0; i < n; ++i) {
            int32_t r16 = -1;
            if (mode == OR_SR) {
                uint32_t r32;
                if (bits_source == OR_BITS_SUPPLIED) {
                    r32 = rbits[i];
                    r16 = (int32_t)(r32 >> 16);
                } else {
                    /* counter bits: one SplitMix64 word per 4 elements, low half first */
                    const uint64_t gi = (uint64_t)(i + block_offset * kBlock);
                    r16 = (int32_t)((or_mix64(seed + (gi >> 2) + 1u) >> (16u * (gi & 3u))) & 0xFFFFu);
                }
            }
            int o, u;
            const uint32_t c = encode_impl((double)x[i], fmt, mode, 0, r16,
                                           saturate, &o, &u, 0);
            codes_out[i] = (uint16_t)c;
            ovf += o; unf += u; nan += isnan(x[i]) ? 1 : 0;
        }
    }
    if (counters) { counters[0] += ovf; counters[1] += unf; counters[2] += nan; }
    return 0;
}

/* tensor.cpp:83-98 with the LUTs of tensor.cpp:100-133 (decode as float). */
void or_dequantize(const uint16_t *codes, int64_t n, int fmt, float *out) {
    for (int64_t i = 0; i < n; ++i) out[i] = (float)or_decode(codes[i], fmt);
}

/* kernels.cpp:37-62 */
void or_gemm(const uint16_t *a, const uint16_t *b, int64_t m, int64_t k,
             int64_t n, int fmt, float *c) {
    float *da = (float *)malloc(sizeof(float) * (size_t)(m * k));
    float *db = (float *)malloc(sizeof(float) * (size_t)(k * n));
    or_dequantize(a, m * k, fmt, da);
    or_dequantize(b, k * n, fmt, db);
    for (int64_t i = 0; i < m; ++i)
        for (int64_t j = 0; j < n; ++j) {
            float acc = 0.0f;
            for (int64_t p = 0; p < k; ++p) acc += da[i * k + p] * db[p * n + j];
            c[i * n + j] = acc;
        }
    free(da);
    free(db);
}

static int64_t conv_out(int64_t in, int64_t k, int64_t s, int64_t p) { return (in + 2 * p - k) / s + 1; }

/* kernels.cpp:106-151 */
void or_conv2d(const uint16_t *x, const uint16_t *w, int64_t n, int64_t c, int64_t h,
               int64_t wd, int64_t f, int64_t kh, int64_t kw, int64_t stride, int64_t pad,
               int fmt, float *y) {
    const int64_t oh = conv_out(h, kh, stride, pad), ow = conv_out(wd, kw, stride, pad);
    for (int64_t ni = 0; ni < n; ++ni)
        for (int64_t fi = 0; fi < f; ++fi)
            for (int64_t oi = 0; oi < oh; ++oi)
                for (int64_t oj = 0; oj < ow; ++oj) {
                    float acc = 0.0f;
                    for (int64_t ci = 0; ci < c; ++ci)
                        for (int64_t ki = 0; ki < kh; ++ki) {
                            const int64_t ii = oi * stride - pad + ki;
                            for (int64_t kj = 0; kj < kw; ++kj) {
                                const int64_t jj = oj * stride - pad + kj;
                                float xv = 0.0f;
                                if (ii >= 0 && ii < h && jj >= 0 && jj < wd)
                                    xv = (float)or_decode(x[((ni * c + ci) * h + ii) * wd + jj], fmt);
                                acc += xv * (float)or_decode(w[((fi * c + ci) * kh + ki) * kw + kj], fmt);
                            }
                        }
                    y[((ni * f + fi) * oh + oi) * ow + oj] = acc;
                }
}

/* kernels.cpp:153-205 */
void or_conv2d_dgrad(const uint16_t *e, const uint16_t *w, int64_t n, int64_t c, int64_t h,
                     int64_t wd, int64_t f, int64_t kh, int64_t kw, int64_t stride,
                     int64_t pad, int fmt, float *dx) {
    const int64_t oh = conv_out(h, kh, stride, pad), ow = conv_out(wd, kw, stride, pad);
    for (int64_t ni = 0; ni < n; ++ni)
        for (int64_t ci = 0; ci < c; ++ci)
            for (int64_t i = 0; i < h; ++i)
                for (int64_t j = 0; j < wd; ++j) {
                    float acc = 0.0f;
                    for (int64_t fi = 0; fi < f; ++fi)
                        for (int64_t ki = 0; ki < kh; ++ki)
                            for (int64_t kj = 0; kj < kw; ++kj) {
                                const int64_t on = i + pad - ki, pn = j + pad - kj;
                                if (on % stride || pn % stride) continue;
                                const int64_t oi = on / stride, oj = pn / stride;
                                if (oi < 0 || oi >= oh || oj < 0 || oj >= ow) continue;
                                acc += (float)or_decode(w[((fi * c + ci) * kh + ki) * kw + kj], fmt) *
                                       (float)or_decode(e[((ni * f + fi) * oh + oi) * ow + oj], fmt);
                            }
                    dx[((ni * c + ci) * h + i) * wd + j] = acc;
                }
}

/* kernels.cpp:207-253 */
void or_conv2d_wgrad(const uint16_t *x, const uint16_t *e, int64_t n, int64_t c, int64_t h,
                     int64_t wd, int64_t f, int64_t kh, int64_t kw, int64_t stride,
                     int64_t pad, int fmt, float *dw) {
    const int64_t oh = conv_out(h, kh, stride, pad), ow = conv_out(wd, kw, stride, pad);
    for (int64_t fi = 0; fi < f; ++fi)
        for (int64_t ci = 0; ci < c; ++ci)
            for (int64_t ki = 0; ki < kh; ++ki)
                for (int64_t kj = 0; kj < kw; ++kj) {
                    float acc = 0.0f;
                    for (int64_t ni = 0; ni < n; ++ni)
                        for (int64_t oi = 0; oi < oh; ++oi)
                            for (int64_t oj = 0; oj < ow; ++oj) {
                                const int64_t ii = oi * stride - pad + ki, jj = oj * stride - pad + kj;
                                if (ii < 0 || ii >= h || jj < 0 || jj >= wd) continue;
                                acc += (float)or_decode(x[((ni * c + ci) * h + ii) * wd + jj], fmt) *
                                       (float)or_decode(e[((ni * f + fi) * oh + oi) * ow + oj], fmt);
                            }
                    dw[((fi * c + ci) * kh + ki) * kw + kj] = acc;
                }
}

void or_gemm_exact(const uint16_t *a, const uint16_t *b, int64_t m, int64_t k,
                   int64_t n, int fmt, double *c_exact, double *c_absdot) {
    for (int64_t i = 0; i < m; ++i)
        for (int64_t j = 0; j < n; ++j) {
            long double acc = 0.0L, aacc = 0.0L;
            for (int64_t p = 0; p < k; ++p) {
                const long double pr = (long double)or_decode(a[i * k + p], fmt) *
                                       (long double)or_decode(b[p * n + j], fmt);
                acc += pr;
                aacc += pr < 0 ? -pr : pr;
            }
            c_exact[i * n + j] = (double)acc;
            c_absdot[i * n + j] = (double)aacc;
        }
}

/* nn.cpp:417-432 (update_tensor); the master rounding is RNE in the
 * reference (nn.cpp:425) and SR as the BASELINE extension, whose oracle is
 * quantize(Tensor(w32), kFp16, {Stochastic, seed}) (SURVEY 8c iii). */
int or_sgd_update(uint16_t *master, float *momentum, const float *g, int64_t n,
                  float scale, float lr, float mu, float two_lambda,
                  int master_mode, int bits_source, uint64_t seed,
                  int64_t block_offset, const uint32_t *rbits, float *w32_out,
                  int64_t *counters) {
    float *w32 = (float *)malloc(sizeof(float) * (size_t)(n > 0 ? n : 1));
    for (int64_t j = 0; j < n; ++j) {
        const float value = (float)or_decode(master[j], OR_FMT_FP16);
        float gv = g[j] / scale;
        if (two_lambda != 0.0f) gv += two_lambda * value;
        momentum[j] = mu * momentum[j] + gv;
        w32[j] = value - lr * momentum[j];
        if (w32_out) w32_out[j] = w32[j];
    }
    int rc = or_quantize(w32, n, OR_FMT_FP16, master_mode, bits_source,
                         master_mode == OR_SR ? seed : 1, 0, block_offset,
                         rbits, master, counters);
    free(w32);
    return rc;
}

/* loss_scaling.cpp:19-38 (validation) */
int or_scaler_init(or_scaler_t *s) {
    if (!(s->scale > 0.0) || !isfinite(s->scale)) return 22;
    if (s->kind == 1) {
        if (!(s->backoff_factor > 0.0) || !(s->backoff_factor < 1.0)) return 22;
        if (!(s->growth_factor > 1.0)) return 22;
        if (s->growth_interval <= 0) return 22;
        int64_t prev = -1;
        for (int i = 0; i < s->n_schedule; ++i) {
            if (s->sched_iter[i] <= prev) return 22;
            if (!(s->sched_scale[i] > 0.0)) return 22;
            prev = s->sched_iter[i];
        }
    }
    s->steps_since_overflow = 0;
    return 0;
}

/* loss_scaling.cpp:40-47 */
double or_scaler_min_threshold(const or_scaler_t *s, int64_t iteration) {
    double thr = 1.0;
    for (int i = 0; i < s->n_schedule; ++i) {
        if (s->sched_iter[i] > iteration) break;
        thr = s->sched_scale[i];
    }
    return thr;
}

/* loss_scaling.cpp:49-83 */
int or_scaler_step(or_scaler_t *s, int grads_finite, int64_t iteration,
                   double *scale_after) {
    int action = OR_ACT_NONE;
    if (s->kind == 0) {
        *scale_after = s->scale;
        return action;
    }
    const double thr = or_scaler_min_threshold(s, iteration);
    if (!grads_finite) {
        const double candidate = s->scale * s->backoff_factor;
        if (candidate < thr) { s->scale = thr; action = OR_ACT_CLAMP; }
        else { s->scale = candidate; action = OR_ACT_BACKOFF; }
        s->steps_since_overflow = 0;
    } else {
        ++s->steps_since_overflow;
        if (s->steps_since_overflow >= s->growth_interval) {
            s->scale *= s->growth_factor;
            s->steps_since_overflow = 0;
            action = OR_ACT_GROWTH;
        }
        if (s->scale < thr) { s->scale = thr; action = OR_ACT_CLAMP; }
    }
    *scale_after = s->scale;
    return action;
}

/* loss_scaling.cpp:89-92 */
void or_unscale(float *g, int64_t n, double scale) {
    const float sc = (float)scale;
    for (int64_t i = 0; i < n; ++i) g[i] /= sc;
}

/* nn.cpp:308-314 */
void or_bias_grad(const float *e, int64_t rows, int64_t cols, float *db) {
    for (int64_t j = 0; j < cols; ++j) {
        float acc = 0.0f;
        for (int64_t r = 0; r < rows; ++r) acc += e[r * cols + j];
        db[j] = acc;
    }
}

uint64_t or_fnv1a64(const void *data, int64_t nbytes) {
    const unsigned char *p = (const unsigned char *)data;
    uint64_t h = 0xcbf29ce484222325ull;
    for (int64_t i = 0; i < nbytes; ++i) {
        h ^= p[i];
        h *= 0x100000001b3ull;
    }
    return h;
}

/* rand.hpp:19-36 */
double or_rand_uniform(or_rand_t *r) {
    return (double)(or_mix64(r->seed + ++r->n) >> 11) * 0x1.0p-53;
}

double or_rand_normal(or_rand_t *r) {
    if (r->have_spare) {
        r->have_spare = 0;
        return r->spare;
    }
    const double u1 = ((double)(or_mix64(r->seed + ++r->n) >> 11) + 1.0) * 0x1.0p-53;
    const double u2 = or_rand_uniform(r);
    const double rr = sqrt(-2.0 * log(u1));
    const double ang = 2.0 * 3.14159265358979323846 * u2;
    r->spare = rr * sin(ang);
    r->have_spare = 1;
    return rr * cos(ang);
}

void or_rand_fill_normal(or_rand_t *r, float *out, int64_t n, double stddev) {
    for (int64_t i = 0; i < n; ++i) out[i] = (float)(or_rand_normal(r) * stddev);
}

static uint16_t bitrev16(uint16_t v) {
    uint16_t r = 0;
    for (int i = 0; i < 16; ++i) r = (uint16_t)(r | (((v >> i) & 1u) << (15 - i)));
    return r;
}

void or_lfsr_tables(uint16_t *tab, uint16_t *pos) {
    uint16_t s = 1;
    memset(pos, 0, sizeof(uint16_t) * 65536);
    for (uint32_t k = 0; k < 65535u; ++k) {
        tab[k] = bitrev16(s);
        pos[s] = (uint16_t)k;
        or_lfsr_next_bits(&s, 16);
    }
}
