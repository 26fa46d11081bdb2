/*
 * fp8_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the reference fp8emu hot path (arXiv 1905.12334 artifact,
 * /root/reference/proj) used as the parity checker for the B200 kernels.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library. The product path
 * (paper_1905_12334_b200/, libfp8b200.so) never links or calls it.
 *
 * Pinning: every function here is checked in tests/ against (a) the golden
 * vectors the reference's own tests freeze (tests/golden/ fixtures, cited per
 * case) and (b) the compiled reference itself (oracle/_ref/libfp8emu_ref.so,
 * built from /root/reference sources by oracle/Makefile) on seeded inputs.
 */
#ifndef FP8_ORACLE_H
#define FP8_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { OR_FMT_E5M2 = 0, OR_FMT_FP16 = 1 };
enum { OR_RNE = 0, OR_SR = 1, OR_TRUNC = 2 };
enum { OR_BITS_LFSR = 0, OR_BITS_COUNTER = 1, OR_BITS_SUPPLIED = 2 };

uint64_t or_mix64(uint64_t x);
uint64_t or_mix_seed(uint64_t seed, uint64_t index);
uint32_t or_lfsr_next_bits(uint16_t *state, int sample_bits);
uint16_t or_lfsr_split(uint64_t seed, uint64_t stream_index);

double or_decode(uint32_t code, int fmt);
/* Reference-style encode in double arithmetic (float_format.cpp:97-135).
 * r16 is consulted only for OR_SR; pass -1 to mean "draw from *lfsr". */
uint32_t or_encode(double x, int fmt, int mode, uint16_t *lfsr, int saturate,
                   int *overflowed, int *underflowed, int *consumed);
/* Pure-integer restatement on FP32 bits (SURVEY A2'); r16 used only for SR. */
uint32_t or_encode_bits(uint32_t fbits, int fmt, int mode, uint32_t r16,
                        int saturate, int *overflowed, int *underflowed,
                        int *inexact);

/* quantize (tensor.cpp:46-81) with the B200 extensions: bits source,
 * block_offset (sharded SR), supplied 32-bit random words.
 * codes_out is uint16 per element (the reference's storage).
 * counters[0]=overflow, [1]=underflow, [2]=NaN codes produced.
 * Returns 0, or 22 (EINVAL) for a zero seed in LFSR-SR mode. */
int or_quantize(const float *x, int64_t n, int fmt, int mode, int bits_source,
                uint64_t seed, int saturate, int64_t block_offset,
                const uint32_t *rbits, uint16_t *codes_out, int64_t *counters);

void or_dequantize(const uint16_t *codes, int64_t n, int fmt, float *out);

/* gemm_fp8 (kernels.cpp:37-62): a [m,k], b [k,n] row-major codes, one format;
 * c[m,n] FP32 with a k-ascending running sum. */
void or_gemm(const uint16_t *a, const uint16_t *b, int64_t m, int64_t k,
             int64_t n, int fmt, float *c);

/* Convolutions over codes, NCHW / FCkk, FP32 accumulation in the reference's
 * fixed orders (kernels.cpp:106-253): fprop (c,kh,kw) with explicit zero
 * products for padded taps; dgrad (f,kh,kw) skipping holes; wgrad (n,oh,ow). */
void or_conv2d(const uint16_t *x, const uint16_t *w, int64_t n, int64_t c, int64_t h,
               int64_t wd, int64_t f, int64_t kh, int64_t kw, int64_t stride, int64_t pad,
               int fmt, float *y);
void or_conv2d_dgrad(const uint16_t *e, const uint16_t *w, int64_t n, int64_t c, int64_t h,
                     int64_t wd, int64_t f, int64_t kh, int64_t kw, int64_t stride,
                     int64_t pad, int fmt, float *dx);
void or_conv2d_wgrad(const uint16_t *x, const uint16_t *e, int64_t n, int64_t c, int64_t h,
                     int64_t wd, int64_t f, int64_t kh, int64_t kw, int64_t stride,
                     int64_t pad, int fmt, float *dw);

/* Exact (long double) sum and sum of |products| for the GEMM tolerance. */
void or_gemm_exact(const uint16_t *a, const uint16_t *b, int64_t m, int64_t k,
                   int64_t n, int fmt, double *c_exact, double *c_absdot);

/* update_tensor (nn.cpp:417-432) over FP16 masters with decoded grads g.
 * master_mode: OR_RNE (reference) or OR_SR (BASELINE extension: the
 * quantize(Tensor(w32), kFp16, {Stochastic, seed}) block stream, or counter /
 * supplied bits). value is derived from the master (value == decode(master)).
 * w32_out (optional) receives the pre-rounding FP32 weights. */
int or_sgd_update(uint16_t *master, float *momentum, const float *g, int64_t n,
                  float scale, float lr, float mu, float two_lambda,
                  int master_mode, int bits_source, uint64_t seed,
                  int64_t block_offset, const uint32_t *rbits, float *w32_out,
                  int64_t *counters);

/* LossScaler (loss_scaling.cpp:19-98). */
typedef struct {
    int kind; /* 0 constant, 1 dynamic-backoff */
    double scale;
    double backoff_factor;
    double growth_factor;
    int64_t growth_interval;
    int64_t steps_since_overflow;
    int32_t n_schedule;
    int64_t sched_iter[16];
    double sched_scale[16];
} or_scaler_t;
enum { OR_ACT_NONE = 0, OR_ACT_BACKOFF = 1, OR_ACT_GROWTH = 2, OR_ACT_CLAMP = 3 };
int or_scaler_init(or_scaler_t *s);
double or_scaler_min_threshold(const or_scaler_t *s, int64_t iteration);
int or_scaler_step(or_scaler_t *s, int grads_finite, int64_t iteration,
                   double *scale_after);
void or_unscale(float *g, int64_t n, double scale);

/* db[j] = sum_r e[r, j] in row order (nn.cpp:308-314). */
void or_bias_grad(const float *e, int64_t rows, int64_t cols, float *db);

/* FNV-1a-64 over raw bytes (the SURVEY 8d known-answer hashes). */
uint64_t or_fnv1a64(const void *data, int64_t nbytes);

/* Rand{seed} (rand.hpp:13-37): fills out[] with float(normal()*stddev),
 * continuing the generator state in *st (seed, n, have_spare, spare). */
typedef struct { uint64_t seed; uint64_t n; int have_spare; double spare; } or_rand_t;
double or_rand_uniform(or_rand_t *r);
double or_rand_normal(or_rand_t *r);
void or_rand_fill_normal(or_rand_t *r, float *out, int64_t n, double stddev);

/* Decimated LFSR tables: tab[k] = bitrev16(D^k(1)), pos[s] = k with
 * D^k(1) == s, D = 16 LFSR clocks. Used by the tests to validate the
 * GPU's jump-ahead scheme independently. */
void or_lfsr_tables(uint16_t *tab /*65535*/, uint16_t *pos /*65536*/);

#ifdef __cplusplus
}
#endif
#endif
