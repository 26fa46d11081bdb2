/*
 * fp8b200.h -- C-ABI of the B200-native FP8 (E5M2) training primitives.
 *
 * This is the drop-in boundary for the hot path of the reference fp8emu
 * library (arXiv 1905.12334 artifact, /root/reference/proj): quantize,
 * dequantize, transpose, gemm_fp8, the loss scaler and the SGD-momentum update
 * into FP16 masters. Each entry point cites the reference interface it replaces
 * (paths relative to /root/reference/proj).
 *
 * Conventions:
 *   - plain pointers and sizes, no C++ or torch types; every tensor pointer is
 *     DEVICE memory owned by the caller; nothing is allocated on hot calls;
 *   - E5M2 codes are 1 byte per element, FP16 codes 2 bytes (the reference
 *     stores both as uint16_t, tensor.hpp:39; the C++ shim widens);
 *   - calls are asynchronous and ordered on `stream` (a cudaStream_t, or NULL
 *     for the legacy default stream); reentrant across streams;
 *   - return 0 on success, FP8B_EINVAL where the reference throws
 *     std::invalid_argument (zero seed tensor.cpp:48, shape or format mismatch
 *     kernels.cpp:38-44, scaler options loss_scaling.cpp:20-37), FP8B_ECUDA on
 *     a CUDA launch/runtime error, FP8B_ENOTSUP for an unsupported combination.
 *     fp8b_last_error() returns a thread-local message for the last failure;
 *   - numeric trouble never fails a call: it is reported through counters
 *     (float_format.hpp:93-99). Counter arrays are device int64[3] =
 *     {overflow, underflow, nan}; kernels ACCUMULATE into them (+=), so several
 *     Q nodes can share one array, as Network::backward sums its overflow
 *     counts (nn.cpp:298-323). overflow/underflow equal the reference's
 *     QuantizedTensor::overflow_count / underflow_count; nan counts NaN codes
 *     produced (a NaN input is not an overflow, float_format.cpp:99).
 */
#ifndef FP8B200_H
#define FP8B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FP8B_OK 0
#define FP8B_EINVAL 22
#define FP8B_ENOTSUP 95
#define FP8B_ECUDA 1000

/* kFp8 / kFp16 (float_format.hpp:75-76) */
enum { FP8B_E5M2 = 0, FP8B_FP16 = 1, FP8B_F32 = 2 };
/* RoundingMode (float_format.hpp:11-15) */
enum { FP8B_RNE = 0, FP8B_SR = 1, FP8B_TRUNC = 2 };
/* Source of the 16-bit stochastic-rounding sample r16 (SR only):
 *  LFSR     -- the reference stream, bit-exact: 4096-element block b draws from
 *              LfsrStream::split(seed, block_offset + b), one 16-bit sample per
 *              inexact element (tensor.cpp:57-70, lfsr.cpp:17-45);
 *  COUNTER  -- r16 = 16-bit lane (g & 3) of mix64(seed + (g >> 2) + 1), with
 *              g = block_offset*4096 + i: the SplitMix64 counter generator of the
 *              reference's Rand (rand.hpp:19-21, lfsr.cpp:47-52), one 64-bit
 *              word per four elements; position-independent, so it fuses anywhere;
 *  SUPPLIED -- r16 = rbits[i] >> 16 from a caller-supplied uint32 tensor.
 * All three round up iff (top 16 discarded bits) + r16 >= 2^16, which is the
 * reference's (a-lo) + r*step >= step (float_format.cpp:122-130) exactly. */
enum { FP8B_BITS_LFSR = 0, FP8B_BITS_COUNTER = 1, FP8B_BITS_SUPPLIED = 2 };

/* QuantConfig (tensor.hpp:28-32) plus the B200 extensions. */
typedef struct {
    int32_t mode;          /* FP8B_RNE / FP8B_SR / FP8B_TRUNC */
    int32_t bits;          /* FP8B_BITS_* (SR only) */
    uint64_t seed;         /* must be nonzero, as QuantConfig.seed (tensor.cpp:48) */
    int32_t saturate;      /* saturate_on_overflow: clamp to max code, flag still fires */
    int32_t reserved;
    int64_t block_offset;  /* number of 4096-element blocks preceding this slice in
                              the logical tensor (sharded SR); 0 otherwise */
    const uint32_t *rbits; /* device, n words; FP8B_BITS_SUPPLIED only */
} fp8b_quant_config_t;

/* Replaces fp8emu::quantize(const Tensor&, const FloatFormat&, const QuantConfig&)
 * (tensor.hpp:59-60, tensor.cpp:46-81). x: n floats; codes: n codes of `fmt`
 * (FP8B_E5M2 or FP8B_FP16); counters: device int64[3] or NULL. */
int fp8b_quantize(const float *x, void *codes, int64_t n, int32_t fmt,
                  const fp8b_quant_config_t *cfg, int64_t *counters, void *stream);

/* Replaces fp8emu::dequantize(const QuantizedTensor&) (tensor.hpp:63,
 * tensor.cpp:83-98): exact decode of E5M2 or FP16 codes to FP32. */
int fp8b_dequantize(const void *codes, float *out, int64_t n, int32_t fmt, void *stream);

/* Replaces fp8emu::transpose(const QuantizedTensor&) (tensor.hpp:73,
 * tensor.cpp:135-150): [rows, cols] codes -> [cols, rows]. The GEMM never needs
 * it (it reads MN-major operands directly); provided for API completeness. */
int fp8b_transpose(const void *in, void *out, int64_t rows, int64_t cols, int32_t fmt,
                   void *stream);

/* Adds the number of non-finite x[i] to counters[2] (the db finiteness check of
 * Network::backward, nn.cpp:401-411). */
int fp8b_count_nonfinite(const float *x, int64_t n, int64_t *counters, void *stream);

/* ---------------------------------------------------------------- GEMM ---- */
/* Operand majors. The reference computes C[M,N] = A[M,K] . B[K,N] with both
 * row-major (kernels.cpp:37-62): A is K-major and B is N-major. The layer step
 * needs the other combinations without a transpose pass (nn.cpp:302, 320):
 *   fprop  Y  = Q(X)  . Q(W)     A K-major, B N-major
 *   bprop  dX = Q(E)  . Q(W)^T   A K-major, B K-major (W [K,N] read as [N,K])
 *   wgrad  dW = Q(X)^T. Q(E)     A M-major (X [B,K] read as [K,B]), B N-major */
enum { FP8B_K_MAJOR = 0, FP8B_MN_MAJOR = 1 };
/* Accumulation engine. */
enum {
    FP8B_GEMM_TENSOR = 0,     /* tcgen05.mma kind::f8f6f4 (E5M2) / kind::f16 (FP16),
                                 FP32 accumulation in TMEM; tolerance-level parity */
    FP8B_GEMM_SEQUENTIAL = 1  /* CUDA cores, one FP32 running sum per output in
                                 k-ascending order: bitwise equal to gemm_fp8 */
};

typedef struct {
    int32_t a_major;       /* FP8B_K_MAJOR: A stored [M,K]; FP8B_MN_MAJOR: A stored [K,M] */
    int32_t b_major;       /* FP8B_MN_MAJOR: B stored [K,N] (reference); FP8B_K_MAJOR: [N,K] */
    int32_t engine;        /* FP8B_GEMM_TENSOR / FP8B_GEMM_SEQUENTIAL */
    int32_t reserved0;
    float *c;              /* optional FP32 output [M,N] row-major (the gemm_fp8 result) */
    const float *bias;     /* optional [N], added in FP32 after the sum (nn.cpp:195-198) */
    void *cq;              /* optional fused output Q node: codes [M,N] row-major */
    int32_t cq_fmt;        /* FP8B_E5M2 / FP8B_FP16 */
    int32_t cq_mode;       /* FP8B_RNE / FP8B_TRUNC / FP8B_SR (with FP8B_BITS_COUNTER only:
                              the reference-stream SR needs the block scan, SURVEY 7(h);
                              write c and call fp8b_quantize instead) */
    uint64_t cq_seed;
    int32_t cq_saturate;
    int32_t reserved1;
    int64_t *cq_counters;  /* device int64[3] or NULL */
} fp8b_gemm_args_t;

/* Replaces fp8emu::gemm_fp8(const QuantizedTensor&, const QuantizedTensor&)
 * (kernels.hpp:11, kernels.cpp:37-62). a and b hold codes of one format `fmt`
 * (the reference requires a shared format, kernels.cpp:9-13). */
int fp8b_gemm(const void *a, const void *b, int64_t m, int64_t n, int64_t k, int32_t fmt,
              const fp8b_gemm_args_t *args, void *stream);

/* 1 if fp8b_gemm with FP8B_GEMM_TENSOR runs these operands on the tcgen05
 * engine, 0 if it would take the CUDA-core engine (TMA needs 16-byte aligned
 * bases and row strides). */
int fp8b_gemm_tensor_supported(const void *a, const void *b, int64_t m, int64_t n, int64_t k,
                               int32_t fmt, int32_t a_major, int32_t b_major);

/* ---------------------------------------------------------- loss scaler ---- */
/* LossScaler (loss_scaling.hpp:26-68) state, resident in DEVICE memory so the
 * step needs no host sync. The host fills kind/scale/factors/interval/schedule
 * and calls fp8b_loss_scaler_init, which validates exactly as the reference
 * constructor (loss_scaling.cpp:19-38) and uploads it. */
#define FP8B_MAX_SCHEDULE 16
enum { FP8B_SCALER_CONSTANT = 0, FP8B_SCALER_DYNAMIC_BACKOFF = 1 };
/* ScaleAction (loss_scaling.hpp:12) */
enum { FP8B_ACT_NONE = 0, FP8B_ACT_BACKOFF = 1, FP8B_ACT_GROWTH = 2, FP8B_ACT_CLAMPED_TO_MIN = 3 };
typedef struct {
    int32_t kind;
    int32_t n_schedule;
    double scale;
    double backoff_factor;
    double growth_factor;
    int64_t growth_interval;
    int64_t steps_since_overflow;
    int64_t sched_iter[FP8B_MAX_SCHEDULE];   /* strictly increasing */
    double sched_scale[FP8B_MAX_SCHEDULE];
    /* last ScaleEvent (loss_scaling.hpp:16-20) */
    int64_t last_iteration;
    int32_t last_action;
    int32_t last_grads_finite;
    double last_scale_after;
    /* device-internal: arrival ticket of a fused update + step (see
     * fp8b_sgd_args_t.step_scaler); zero outside a running update */
    uint32_t step_ticket;
    uint32_t reserved;
} fp8b_loss_scaler_t;

int fp8b_loss_scaler_init(fp8b_loss_scaler_t *dev_state, const fp8b_loss_scaler_t *host_opts,
                          void *stream);
/* LossScaler::step(grads_finite, iteration) (loss_scaling.cpp:49-83) on device.
 * grads_finite = (counters[0] + counters[2] == 0) when counters != NULL (the
 * accumulated overflow + NaN/non-finite counts of the backward Q nodes, i.e.
 * nn.cpp:401-411), else taken from `grads_finite`. */
int fp8b_loss_scaler_step(fp8b_loss_scaler_t *dev_state, const int64_t *counters,
                          int32_t grads_finite, int64_t iteration, void *stream);
/* LossScaler::unscale_gradients_inplace (loss_scaling.cpp:89-92): g /= float(scale)
 * with IEEE division; scale read from the device state. */
int fp8b_unscale(float *g, int64_t n, const fp8b_loss_scaler_t *dev_state, void *stream);

/* -------------------------------------------------------------- update ---- */
typedef struct {
    float lr, mu, two_lambda;   /* narrowed from double as in nn.cpp:437-443 */
    float scale;                /* used when scaler == NULL */
    const fp8b_loss_scaler_t *scaler; /* device: scale = float(scaler->scale) */
    const int64_t *skip_counters;     /* device int64[3] or NULL: the whole update is
                                         skipped when [0]+[2] != 0 (nn.cpp:546) */
    int32_t master_mode;        /* FP8B_RNE (reference, nn.cpp:425) or FP8B_SR (BASELINE) */
    int32_t bits;               /* FP8B_BITS_* for FP8B_SR */
    uint64_t seed;              /* nonzero for FP8B_SR */
    int64_t block_offset;       /* 4096-blocks before this shard of the parameter */
    const uint32_t *rbits;      /* FP8B_BITS_SUPPLIED */
    int64_t *master_counters;   /* device int64[3] or NULL: master rounding counters */
    uint8_t *w_e5m2;            /* optional fused Q_RNE(decode(master_new)) for the next
                                   fprop (nn.cpp:192-193), E5M2 codes */
    int32_t w_saturate;
    int32_t step_scaler;        /* 1: once the whole update has read the scale, run
                                   LossScaler::step(grads_finite(skip_counters),
                                   step_iteration) on `scaler` from the update's last
                                   CTA -- the fp8b_loss_scaler_step that follows the
                                   iteration's last update (nn.cpp:546-547) without its
                                   own launch. At most one such update per scaler in
                                   flight. 2: the same, and the gate's input counters
                                   (skip_counters, skip_counters2) are then cleared for the
                                   next step, so a step needs no zeroing launch. */
    int64_t *w_counters;        /* device int64[3] or NULL */
    int64_t step_iteration;     /* for step_scaler */
    const int64_t *skip_counters2; /* optional second int64[3]: the gate is the element-wise
                                      sum skip_counters + skip_counters2 (the step's two
                                      counter sets, nn.cpp:401-411, with no merge launch) */
    int64_t *gate_out;          /* with step_scaler: the merged int64[3] gate is stored
                                   here by the update's last CTA (may alias neither input) */
} fp8b_sgd_args_t;

/* update_tensor (nn.cpp:417-432) as driven by Network::apply_update
 * (nn.cpp:436-458), fused into one pass: decode grad -> g/scale -> +2λw ->
 * momentum -> w32 -> FP16 master (RNE or SR) [-> E5M2 copy of W].
 * grad_fmt: FP8B_E5M2 codes (qdW), FP8B_FP16 codes, or FP8B_F32 (db).
 * IEEE binary32 arithmetic in the reference's order, no FMA contraction. */
int fp8b_sgd_momentum_update(const void *grad, int32_t grad_fmt, uint16_t *master,
                             float *momentum, int64_t n, const fp8b_sgd_args_t *args,
                             void *stream);

/* db[j] = sum_r dequant(qe)[r, j] in row order (nn.cpp:308-314); bit-exact. */
int fp8b_bias_grad(const void *e_codes, int32_t fmt, int64_t rows, int64_t cols, float *db,
                   void *stream);

/* -------------------------------------------------------- convolutions ---- */
/* The conv family of kernels.hpp:13-50. Layout FP8B_NCHW is the reference's
 * (x [N,C,H,W], w [F,C,kH,kW], y [N,F,OH,OW]); FP8B_NHWC is the B200 layout of
 * BASELINE config 4 (x [N,H,W,C], w [F,kH,kW,C], y [N,OH,OW,F]). Outputs are
 * FP32 (unquantized, as the reference returns them).
 * Engines: FP8B_GEMM_SEQUENTIAL reproduces the reference's accumulation order
 * (fprop (c,kh,kw), dgrad (f,kh,kw), wgrad (n,oh,ow)) bit for bit in either
 * layout; FP8B_GEMM_TENSOR runs implicit GEMM on tcgen05 (NHWC, E5M2, stride
 * 1; other cases fall back to the sequential engine) within the GEMM tolerance. */
enum { FP8B_NCHW = 0, FP8B_NHWC = 1 };
typedef struct {
    int64_t n, c, h, w;       /* input batch, channels, height, width */
    int64_t f, kh, kw;        /* filters and kernel size */
    int64_t stride, pad;      /* ConvGeometry (kernels.hpp:13-16) */
    int32_t layout;           /* FP8B_NCHW / FP8B_NHWC */
    int32_t engine;           /* FP8B_GEMM_TENSOR / FP8B_GEMM_SEQUENTIAL */
    /* Optional fused output Q node (the layer's next quantize, nn.cpp:192-200):
     * when yq != NULL the output is also (or, with a NULL FP32 output, only)
     * written as codes. yq_mode RNE / TRUNC, or SR with counter bits (yq_seed
     * nonzero); counters accumulate {overflow, underflow, nan} like fp8b_quantize. */
    void *yq;
    int32_t yq_fmt;           /* FP8B_E5M2 / FP8B_FP16 */
    int32_t yq_mode;          /* FP8B_RNE / FP8B_TRUNC / FP8B_SR (counter bits) */
    uint64_t yq_seed;
    int32_t yq_saturate;
    int32_t reserved;
    int64_t *yq_counters;     /* device int64[3] or NULL */
} fp8b_conv_t;

/* conv2d_fp8 (kernels.hpp:22-23): y = x * w. The FP32 output pointer may be
 * NULL when g->yq is set. */
int fp8b_conv2d_fprop(const void *x, const void *w, float *y, int32_t fmt, const fp8b_conv_t *g,
                      void *stream);
/* conv2d_backward_data_fp8 (kernels.hpp:39-41): dx from e [N,F,OH,OW] and w */
int fp8b_conv2d_dgrad(const void *e, const void *w, float *dx, int32_t fmt,
                      const fp8b_conv_t *g, void *stream);
/* conv2d_backward_weights_fp8 (kernels.hpp:46-48): dw from x and e */
int fp8b_conv2d_wgrad(const void *x, const void *e, float *dw, int32_t fmt,
                      const fp8b_conv_t *g, void *stream);

/* 1 if FP8B_GEMM_TENSOR runs this conv (kind 0 fprop, 1 dgrad, 2 wgrad) on the
 * tensor cores for 16-byte-aligned operands, 0 if it takes the sequential engine. */
int fp8b_conv_tensor_supported(const fp8b_conv_t *g, int32_t fmt, int32_t kind);
/* Extension (no reference counterpart): 1 if that tensor-engine conv runs the
 * weight-stationary halo-slab kernel (NHWC, stride 1, C * code bytes in {64,
 * 128}, F <= 256; kind 0 fprop, 1 dgrad; kind 2 wgrad: 3x3, E5M2, C = F =
 * 64), 0 if the im2col kernel. */
int fp8b_conv_halo_supported(const fp8b_conv_t *g, int32_t fmt, int32_t kind);

/* im2col (kernels.hpp:25-30): pure code movement, zero code for padded taps.
 * FP8B_NCHW gives the reference's patch matrix [C*kH*kW, N*OH*OW] (rows
 * (c,kh,kw), cols (n,oh,ow)); FP8B_NHWC gives its transpose in the NHWC tap
 * order, [N*OH*OW, kH*kW*C] (K-major A operand of fp8b_gemm). */
int fp8b_im2col(const void *x, void *cols, int32_t fmt, const fp8b_conv_t *g, void *stream);

/* ------------------------------------------------ FP8T container (host) ---- */
/* The reference's binary tensor file (tensor_io.hpp:18-31, tensor_io.cpp:47-187):
 * "FP8T", version 1, dtype (0 FP32, 1 FP8 codes, 2 FP16 codes), rank, rounding
 * mode tag (0 none, 1 nearest-even, 2 stochastic, 3 truncate), 8 reserved zero
 * bytes, rank big-endian uint64 dims, then the big-endian row-major payload.
 * Host buffers in native byte order: float32, uint8 codes, uint16 codes.
 * Errors: FP8B_EIO with the reference's IoError message in fp8b_last_error(). */
enum { FP8B_FP8T_F32 = 0, FP8B_FP8T_FP8 = 1, FP8B_FP8T_FP16 = 2 };
enum { FP8B_EIO = 5 };
#define FP8B_FP8T_MAX_RANK 255

/* save_tensor (tensor_io.cpp:107-140) */
int fp8b_fp8t_save(const char *path, int32_t dtype, int32_t mode_tag, int32_t rank,
                   const int64_t *dims, const void *data);
/* header of a file: dtype, mode tag, rank and up to max_rank dims */
int fp8b_fp8t_peek(const char *path, int32_t *dtype, int32_t *mode_tag, int32_t *rank,
                   int64_t *dims, int32_t max_rank);
/* load_tensor_fp32 / load_tensor_codes (tensor_io.cpp:142-187): expect_dtype
 * FP8B_FP8T_F32, or -1 for "codes of either width"; capacity in elements. */
int fp8b_fp8t_load(const char *path, int32_t expect_dtype, void *data, int64_t capacity);

/* ---------------------------------------------------------- layer step ---- */
/* One quantized Dense-layer training step on device, the composition
 * Network::forward -> backward -> apply_update -> LossScaler::step performs for a
 * Dense layer (nn.cpp:187-203, 294-326, 401-411, 417-458, 540-547) with every
 * Q node in E5M2 round-to-nearest-even:
 *   qx = Q(x); qy = Q(qx . w_q + b)                          (fprop, fused epilogue)
 *   qe = Q(e); db = colsum(qe); qdw = Q(qx^T . qe)           (wgrad, fused epilogue)
 *   qdx = Q(qe . w_q^T)                                      (bprop, fused epilogue)
 *   finite = no overflow in qe/qdw/qdx, no NaN in qdw, db finite  (nn.cpp:401-411)
 *   if finite: update_tensor(W, qdw), update_tensor(b, db);  w_q = Q(decode(w_master))
 *   scaler.step(finite, iteration)
 * The scale used by the backward/update is scaler->scale at entry (nn.cpp:540).
 * `e` is the loss-scaled upstream error (softmax_xent_backward output,
 * nn.cpp:286-288). counters = int64[6]: [0..2] overflow/underflow/nan of Q(e)
 * and Q(dx) plus non-finite db in [2]; [3..5] the Q(dW) counters (so
 * underflow_fraction = counters[4] / (in*out), nn.cpp:305-306). The step zeroes
 * them itself. gate = int64[3] workspace. No host synchronisation: the step can
 * be captured in a CUDA graph. */
typedef struct {
    int64_t batch, in_features, out_features;
    const float *x;          /* [batch, in] FP32 layer input */
    const float *e;          /* [batch, out] loss-scaled upstream error */
    uint16_t *w_master;      /* [in, out] FP16 master weights (row-major like nn.hpp:56-61) */
    float *w_momentum;       /* [in, out] */
    uint8_t *w_q;            /* [in, out] E5M2 Q(decode(w_master)), refreshed by the update */
    uint16_t *b_master;      /* [out] FP16 master bias, or NULL for a bias-free layer */
    float *b_momentum;       /* [out] */
    float *b_value;          /* [out] workspace: decode(b_master) */
    uint8_t *qx, *qy, *qe, *qdw;  /* Q-node outputs */
    uint8_t *qdx;            /* [batch, in] or NULL (first layer: no dx, nn.cpp:317) */
    float *db;               /* [out] bias gradient (bias layers) */
    float *y;                /* optional [batch, out] FP32 pre-Q output */
    int64_t *fwd_counters;   /* int64[3]: Q(x) + Q(y), or NULL */
    int64_t *counters;       /* int64[6], see above */
    int64_t *gate;           /* int64[3] workspace */
    fp8b_loss_scaler_t *scaler;
    int64_t iteration;
    float lr, mu, two_lambda;
    int32_t engine;          /* FP8B_GEMM_TENSOR / FP8B_GEMM_SEQUENTIAL */
    int32_t master_mode;     /* FP8B_RNE (reference) / FP8B_SR (BASELINE) */
    int32_t bits;            /* SR bits source for the masters */
    int32_t saturate;        /* quant.saturate for every Q node */
    uint64_t seed;           /* master SR seed (nonzero) */
} fp8b_dense_step_t;

int fp8b_dense_step(const fp8b_dense_step_t *s, void *stream);

/* -------------------------------------------------------------- misc ---- */
/* Optional eager initialisation for the current device (uploads the 200 KB of
 * LFSR jump tables once); otherwise done lazily by the first SR-LFSR call. Call
 * it before capturing a CUDA graph that contains SR-LFSR calls. */
int fp8b_init(void);
const char *fp8b_last_error(void);
/* Library build tag, e.g. "fp8b200 sm_100a". */
const char *fp8b_version(void);
/* Number of this library's kernels launched since load (per process). */
int64_t fp8b_launch_count(void);

/* Seeded synthetic inputs (bench / tests; no reference counterpart):
 * kind 0: SURVEY 8d config 2 -- |x| = 2^u, u ~ U[lo, hi], random sign, with a
 *         fraction `p` of exact E5M2 rounding midpoints (ties);
 * kind 1: N(0, p^2) via Box-Muller over counter bits;
 * kind 2: |N(0, p^2)| (half-normal activations). */
int fp8b_fill_synthetic(float *out, int64_t n, int32_t kind, uint64_t seed, double p,
                        double lo, double hi, void *stream);

/* ------------------------------------------------- peer memory (multi-GPU) ---- */
/* The data-parallel exchange of SURVEY 8e over NVLink / NVSwitch peer memory
 * (no reference counterpart: the reference is single-process). Buffers that
 * other processes of the node map: */
#define FP8B_PEER_HANDLE_BYTES 64
#define FP8B_MAX_PEERS 16
int fp8b_peer_alloc(void **ptr, int64_t bytes, unsigned char handle[FP8B_PEER_HANDLE_BYTES]);
int fp8b_peer_free(void *ptr);
/* Map / unmap a buffer another PROCESS allocated with fp8b_peer_alloc. */
int fp8b_peer_open(const unsigned char handle[FP8B_PEER_HANDLE_BYTES], void **ptr);
int fp8b_peer_close(void *ptr);
/* Fused reduce-scatter + Q node: for i in [0, n): s = peers[0][i0 + i] + peers[1][i0 + i]
 * + ... in rank order (binary32, the same order on every rank), codes[i] =
 * Q(s) with `cfg` (RNE, TRUNC, or SR with counter bits; cfg->block_offset * 4096 +
 * i is the element's index in the unsharded tensor), counters as fp8b_quantize,
 * and optionally sum_out[i] = s. `peers`: HOST array of `world` device pointers
 * (this rank's own buffer and the fp8b_peer_open mappings), 16-byte aligned;
 * i0 and n multiples of 4. The caller orders the step: every rank's partial
 * must be complete before any rank launches this, and no rank may overwrite
 * its partial until every reader is done. */
int fp8b_peer_reduce_quantize(const float *const *peers, int32_t world, int64_t i0, int64_t n,
                              float *sum_out, void *codes, int32_t fmt,
                              const fp8b_quant_config_t *cfg, int64_t *counters, void *stream);

/* Measurement aid (bench.py; no reference counterpart): streams n FP32 values
 * (n % 4 == 0, 16-byte aligned) with the quantizer's access pattern and writes
 * out_bytes in {0, 1, 2, 4} bytes per element with no arithmetic -- what HBM
 * delivers for that read : write mix, the practical ceiling of the quantize
 * kernels beside the 1 : 1 copy figure. */
int fp8b_stream_probe(const float *x, void *out, int64_t n, int32_t out_bytes, void *stream);

#ifdef __cplusplus
}
#endif
#endif
