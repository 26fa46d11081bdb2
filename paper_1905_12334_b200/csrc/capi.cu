// capi.cu -- extern "C" entry points of libfp8b200.so (declared in include/fp8b200.h).
//
// Validation mirrors where the reference throws std::invalid_argument; every
// accepted call is a stream-ordered launch of the kernels in this directory.
// There is no CPU compute path: a missing or failing GPU is reported as
// FP8B_ECUDA.
#include <atomic>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"

namespace {

thread_local std::string g_err;
std::atomic<int64_t> g_launches{0};

int fail(int code, const char* msg) {
    g_err = msg;
    return code;
}

int check_launch(int nkernels) {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        g_err = std::string("CUDA error: ") + cudaGetErrorString(e);
        return FP8B_ECUDA;
    }
    g_launches += nkernels;
    return FP8B_OK;
}

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// ---- decimated LFSR tables, one copy per device (init once) -------------
constexpr int kMaxDev = 64;
std::mutex g_tab_mu;
fp8b::LfsrTables g_tabs[kMaxDev];
bool g_tab_ok[kMaxDev];

uint16_t bitrev16(uint16_t v) {
    uint16_t r = 0;
    for (int i = 0; i < 16; ++i) r = (uint16_t)(r | (((v >> i) & 1u) << (15 - i)));
    return r;
}

int get_tables(fp8b::LfsrTables* out) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDev)
        return fail(FP8B_ECUDA, "no CUDA device");
    std::lock_guard<std::mutex> lk(g_tab_mu);
    if (!g_tab_ok[dev]) {
        // D = 16 clocks of the (16,15,13,4) Fibonacci LFSR (lfsr.cpp:17-27);
        // D is a single 65535-cycle since gcd(16, 65535) = 1.
        std::vector<uint16_t> tabx(fp8b::kLfsrPeriod + fp8b::kBlock), pos(65536, 0);
        uint16_t s = 1;
        for (int k = 0; k < fp8b::kLfsrPeriod; ++k) {
            tabx[k] = bitrev16(s);
            pos[s] = (uint16_t)k;
            for (int c = 0; c < 16; ++c) {
                const uint16_t bit = (uint16_t)(((s >> 0) ^ (s >> 1) ^ (s >> 3) ^ (s >> 12)) & 1u);
                s = (uint16_t)((s >> 1) | (bit << 15));
            }
        }
        for (int k = 0; k < fp8b::kBlock; ++k) tabx[fp8b::kLfsrPeriod + k] = tabx[k];
        uint16_t *dt = nullptr, *dp = nullptr;
        tabx.resize(tabx.size() + 64, 0);  // the staged kernel bulk-copies a 128-byte-padded image
        if (cudaMalloc(&dt, tabx.size() * 2) != cudaSuccess ||
            cudaMalloc(&dp, pos.size() * 2) != cudaSuccess ||
            cudaMemcpy(dt, tabx.data(), tabx.size() * 2, cudaMemcpyHostToDevice) != cudaSuccess ||
            cudaMemcpy(dp, pos.data(), pos.size() * 2, cudaMemcpyHostToDevice) != cudaSuccess) {
            cudaGetLastError();
            return fail(FP8B_ECUDA, "failed to upload LFSR tables");
        }
        g_tabs[dev].tabx = dt;
        g_tabs[dev].pos = dp;
        g_tab_ok[dev] = true;
        // Split-K workspaces (GEMM, conv wgrad) come from the device's default
        // stream-ordered pool; keep freed blocks mapped across synchronisations
        // so a hot call never pays for re-mapping them.
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t keep = ~0ull;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
        cudaGetLastError();
    }
    *out = g_tabs[dev];
    return FP8B_OK;
}

bool valid_fmt(int32_t f) { return f == FP8B_E5M2 || f == FP8B_FP16; }
bool valid_mode(int32_t m) { return m == FP8B_RNE || m == FP8B_SR || m == FP8B_TRUNC; }
bool valid_bits(int32_t b) { return b == FP8B_BITS_LFSR || b == FP8B_BITS_COUNTER || b == FP8B_BITS_SUPPLIED; }

}  // namespace

namespace fp8b {
void note_launches(int n) { g_launches += n; }
void set_error(const std::string& msg) { g_err = msg; }

// Per-device launch setup. A process may drive several GPUs (one thread per
// device, or cudaSetDevice between calls), and both the SM count and the
// >48 KB dynamic shared memory opt-in belong to the current device's context.
static std::mutex g_dev_mu;
int device_sm_count() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 1;
    static std::map<int, int> sms;
    std::lock_guard<std::mutex> lk(g_dev_mu);
    auto it = sms.find(dev);
    if (it != sms.end()) return it->second;
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v < 1)
        return 1;
    sms[dev] = v;
    return v;
}
int64_t lfsr_cta_max_blocks() {
    static int64_t v = -1;
    if (v < 0) {
        const char* e = getenv("FP8B_LFSR_CTA_MAX");
        v = e ? atoll(e) : 2 * (int64_t)device_sm_count();
    }
    return v;
}
void ensure_smem_attr(const void* fn, int bytes) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return;
    // the largest size set so far per (kernel, device): a kernel whose shared
    // memory plan depends on the call's geometry may need more on a later call
    static std::map<std::pair<const void*, int>, int> done;
    std::lock_guard<std::mutex> lk(g_dev_mu);
    auto it = done.find({fn, dev});
    if (it != done.end() && it->second >= bytes) return;
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) == cudaSuccess)
        done[{fn, dev}] = bytes;
}
}  // namespace fp8b

extern "C" {

const char* fp8b_last_error(void) { return g_err.c_str(); }
const char* fp8b_version(void) { return "fp8b200 0.1 sm_100a (tcgen05/TMA)"; }
int64_t fp8b_launch_count(void) { return g_launches.load(); }

int fp8b_init(void) {
    fp8b::LfsrTables t;
    return get_tables(&t);
}

int fp8b_quantize(const float* x, void* codes, int64_t n, int32_t fmt,
                  const fp8b_quant_config_t* cfg, int64_t* counters, void* stream) {
    if (!cfg) return fail(FP8B_EINVAL, "quantize: null config");
    if (cfg->seed == 0) return fail(FP8B_EINVAL, "QuantConfig.seed must be nonzero");
    if (n < 0) return fail(FP8B_EINVAL, "negative dimension");
    if (!valid_fmt(fmt)) return fail(FP8B_EINVAL, "quantize: unknown float format");
    if (!valid_mode(cfg->mode)) return fail(FP8B_EINVAL, "unknown rounding mode");
    if (cfg->mode == FP8B_SR && !valid_bits(cfg->bits))
        return fail(FP8B_EINVAL, "quantize: unknown random-bits source");
    if (cfg->mode == FP8B_SR && cfg->bits == FP8B_BITS_SUPPLIED && !cfg->rbits)
        return fail(FP8B_EINVAL, "quantize: supplied-bits SR needs rbits");
    if (cfg->block_offset < 0) return fail(FP8B_EINVAL, "quantize: negative block_offset");
    if (n == 0) return FP8B_OK;
    if (!x || !codes) return fail(FP8B_EINVAL, "quantize: null tensor");
    fp8b::LfsrTables tabs{nullptr, nullptr};
    if (cfg->mode == FP8B_SR && cfg->bits == FP8B_BITS_LFSR) {
        const int rc = get_tables(&tabs);
        if (rc) return rc;
    }
    fp8b::launch_quantize(x, codes, n, fmt, *cfg, counters, S(stream), tabs);
    return check_launch(1);
}

int fp8b_dequantize(const void* codes, float* out, int64_t n, int32_t fmt, void* stream) {
    if (n < 0) return fail(FP8B_EINVAL, "negative dimension");
    if (!valid_fmt(fmt)) return fail(FP8B_EINVAL, "dequantize: unknown float format");
    if (n == 0) return FP8B_OK;
    if (!codes || !out) return fail(FP8B_EINVAL, "dequantize: null tensor");
    if ((uintptr_t)codes % (fmt == FP8B_E5M2 ? 4 : 8) || (uintptr_t)out % 16)
        return fail(FP8B_EINVAL, "dequantize: codes must be 4/8-byte and out 16-byte aligned");
    fp8b::launch_dequantize(codes, out, n, fmt, S(stream));
    return check_launch(1);
}

int fp8b_transpose(const void* in, void* out, int64_t rows, int64_t cols, int32_t fmt,
                   void* stream) {
    if (rows < 0 || cols < 0) return fail(FP8B_EINVAL, "negative dimension");
    if (!valid_fmt(fmt)) return fail(FP8B_EINVAL, "transpose: unknown float format");
    if (rows == 0 || cols == 0) return FP8B_OK;
    if (!in || !out) return fail(FP8B_EINVAL, "transpose: null tensor");
    fp8b::launch_transpose(in, out, rows, cols, fmt, S(stream));
    return check_launch(1);
}

int fp8b_count_nonfinite(const float* x, int64_t n, int64_t* counters, void* stream) {
    if (n < 0) return fail(FP8B_EINVAL, "negative dimension");
    if (n == 0) return FP8B_OK;
    if (!x || !counters) return fail(FP8B_EINVAL, "count_nonfinite: null pointer");
    fp8b::launch_count_nonfinite(x, n, counters, S(stream));
    return check_launch(1);
}

int fp8b_bias_grad(const void* e_codes, int32_t fmt, int64_t rows, int64_t cols, float* db,
                   void* stream) {
    if (rows < 0 || cols < 0) return fail(FP8B_EINVAL, "negative dimension");
    if (!valid_fmt(fmt)) return fail(FP8B_EINVAL, "bias_grad: unknown float format");
    if (cols == 0) return FP8B_OK;
    if (!db || (rows > 0 && !e_codes)) return fail(FP8B_EINVAL, "bias_grad: null tensor");
    fp8b::launch_bias_grad(e_codes, fmt, rows, cols, db, S(stream));
    return check_launch(1);
}

int fp8b_gemm(const void* a, const void* b, int64_t m, int64_t n, int64_t k, int32_t fmt,
              const fp8b_gemm_args_t* args, void* stream) {
    if (!args) return fail(FP8B_EINVAL, "gemm: null args");
    if (m < 0 || n < 0 || k < 0) return fail(FP8B_EINVAL, "gemm_fp8 expects rank-2 operands");
    if (!valid_fmt(fmt)) return fail(FP8B_EINVAL, "kernel operands must share one format");
    if (args->a_major != FP8B_K_MAJOR && args->a_major != FP8B_MN_MAJOR)
        return fail(FP8B_EINVAL, "gemm: bad a_major");
    if (args->b_major != FP8B_K_MAJOR && args->b_major != FP8B_MN_MAJOR)
        return fail(FP8B_EINVAL, "gemm: bad b_major");
    if (args->engine != FP8B_GEMM_TENSOR && args->engine != FP8B_GEMM_SEQUENTIAL)
        return fail(FP8B_EINVAL, "gemm: bad engine");
    if (!args->c && !args->cq) return fail(FP8B_EINVAL, "gemm: no output requested");
    if (args->cq) {
        if (!valid_fmt(args->cq_fmt)) return fail(FP8B_EINVAL, "gemm: bad cq_fmt");
        if (!valid_mode(args->cq_mode)) return fail(FP8B_EINVAL, "gemm: bad cq_mode");
        if (args->cq_mode == FP8B_SR && args->cq_seed == 0)
            return fail(FP8B_EINVAL, "QuantConfig.seed must be nonzero");
    }
    if (m == 0 || n == 0) return FP8B_OK;
    if (k > 0 && (!a || !b)) return fail(FP8B_EINVAL, "gemm: null operand");
    fp8b::EpiArgs ep{args->c, args->bias, args->cq, args->cq_fmt, args->cq_mode, args->cq_seed,
                     args->cq_saturate, args->cq_counters};
    const int a_mn = args->a_major == FP8B_MN_MAJOR, b_mn = args->b_major == FP8B_MN_MAJOR;
    if (args->engine == FP8B_GEMM_TENSOR) {
        int nl = 0;
        const int rc = fp8b::launch_gemm_tc(a, b, m, n, k, fmt, a_mn, b_mn, ep, S(stream), &nl);
        if (rc == FP8B_OK) return check_launch(nl);
        if (rc != FP8B_ENOTSUP) return rc;
        // Shapes whose row strides TMA cannot address (not a multiple of 16
        // bytes) run on the CUDA-core engine -- still on the GPU.
    }
    fp8b::launch_gemm_seq(a, b, m, n, k, fmt, a_mn, b_mn, ep, S(stream));
    return check_launch(1);
}

int fp8b_gemm_tensor_supported(const void* a, const void* b, int64_t m, int64_t n, int64_t k,
                               int32_t fmt, int32_t a_major, int32_t b_major) {
    if (!valid_fmt(fmt) || m <= 0 || n <= 0 || k <= 0) return 0;
    const int es = fmt == FP8B_E5M2 ? 1 : 2;
    const int64_t a_inner = a_major == FP8B_MN_MAJOR ? m : k;
    const int64_t b_inner = b_major == FP8B_MN_MAJOR ? n : k;
    if ((uintptr_t)a % 16 || (uintptr_t)b % 16 || (a_inner * es) % 16 || (b_inner * es) % 16) return 0;
    if (m > INT32_MAX || n > INT32_MAX || k > INT32_MAX) return 0;
    return 1;
}

// ---- conv family (kernels.cpp:28-253) -------------------------------------
static int conv_validate(const fp8b_conv_t* g, int32_t fmt, const char* who) {
    if (!g) return fail(FP8B_EINVAL, "conv: null geometry");
    if (g->n < 0 || g->c < 0 || g->h < 0 || g->w < 0 || g->f < 0 || g->kh < 0 || g->kw < 0)
        return fail(FP8B_EINVAL, who);
    // conv_out_dim (kernels.cpp:28-35)
    if (g->stride < 1 || g->h + 2 * g->pad - g->kh < 0 || g->w + 2 * g->pad - g->kw < 0 ||
        g->pad < 0)
        return fail(FP8B_EINVAL, "convolution geometry does not fit input");
    if (g->layout != FP8B_NCHW && g->layout != FP8B_NHWC) return fail(FP8B_EINVAL, "conv: bad layout");
    if (g->engine != FP8B_GEMM_TENSOR && g->engine != FP8B_GEMM_SEQUENTIAL)
        return fail(FP8B_EINVAL, "conv: bad engine");
    if (!valid_fmt(fmt)) return fail(FP8B_EINVAL, "kernel operands must share one format");
    return FP8B_OK;
}

static int conv_common(int kind, const void* a, const void* b, float* out, int32_t fmt,
                       const fp8b_conv_t* g, void* stream, const char* who) {
    const int rc = conv_validate(g, fmt, who);
    if (rc) return rc;
    if (g->yq) {
        if (!valid_fmt(g->yq_fmt)) return fail(FP8B_EINVAL, "conv: bad yq_fmt");
        if (!valid_mode(g->yq_mode)) return fail(FP8B_EINVAL, "conv: bad yq_mode");
        if (g->yq_mode == FP8B_SR && g->yq_seed == 0)
            return fail(FP8B_EINVAL, "QuantConfig.seed must be nonzero");
    }
    const int64_t oh = (g->h + 2 * g->pad - g->kh) / g->stride + 1;
    const int64_t ow = (g->w + 2 * g->pad - g->kw) / g->stride + 1;
    const int64_t nout = kind == 0 ? g->n * g->f * oh * ow
                         : kind == 1 ? g->n * g->c * g->h * g->w
                                     : g->f * g->c * g->kh * g->kw;
    if (nout == 0) return FP8B_OK;
    if (!a || !b || (!out && !g->yq)) return fail(FP8B_EINVAL, "conv: null tensor");
    cudaStream_t st = S(stream);
    // fprop / dgrad on the tensor engine fuse the output Q node into the
    // tcgen05 epilogue; every other case computes FP32 and quantizes after
    if (g->engine == FP8B_GEMM_TENSOR && kind != 2) {
        int nl = 0;
        const int r = fp8b::launch_conv_tc(kind, a, b, out, fmt, *g, st, &nl);
        if (r == FP8B_OK) return check_launch(nl);
        if (r != FP8B_ENOTSUP) return r;
    }
    float* tmp = nullptr;
    if (!out) {
        if (cudaMallocAsync(&tmp, sizeof(float) * (size_t)nout, st) != cudaSuccess)
            return fail(FP8B_ECUDA, "conv: workspace allocation failed");
        out = tmp;
    }
    fp8b_conv_t g2 = *g;
    g2.yq = nullptr;
    int nl = 0;
    int r = FP8B_ENOTSUP;
    // wgrad: the Q(dW) node rides on the split-K sum where there is one (q_done)
    int q_done = 0;
    if (g->engine == FP8B_GEMM_TENSOR)
        r = fp8b::launch_conv_tc(kind, a, b, out, fmt, kind == 2 ? *g : g2, st, &nl, &q_done);
    if (r == FP8B_ENOTSUP) {
        fp8b::launch_conv_seq(kind, a, b, out, fmt, g2, st);
        nl = 1;
        r = FP8B_OK;
    }
    if (r == FP8B_OK && g->yq && !q_done) {
        fp8b::LfsrTables tabs;
        r = get_tables(&tabs);
        if (r == FP8B_OK) {
            fp8b_quant_config_t qc{};
            qc.mode = g->yq_mode;
            qc.bits = FP8B_BITS_COUNTER;
            qc.seed = g->yq_seed;
            qc.saturate = g->yq_saturate;
            fp8b::launch_quantize(out, g->yq, nout, g->yq_fmt, qc, g->yq_counters, st, tabs);
            nl += 1;
        }
    }
    if (tmp) cudaFreeAsync(tmp, st);
    if (r != FP8B_OK) return r;
    return check_launch(nl);
}

int fp8b_conv2d_fprop(const void* x, const void* w, float* y, int32_t fmt, const fp8b_conv_t* g,
                      void* stream) {
    return conv_common(0, x, w, y, fmt, g, stream, "conv2d_fp8 expects [N,C,H,W] and [F,C,kH,kW]");
}
int fp8b_conv2d_dgrad(const void* e, const void* w, float* dx, int32_t fmt, const fp8b_conv_t* g,
                      void* stream) {
    return conv_common(1, e, w, dx, fmt, g, stream, "conv backward expects rank-4 operands");
}
int fp8b_conv2d_wgrad(const void* x, const void* e, float* dw, int32_t fmt, const fp8b_conv_t* g,
                      void* stream) {
    return conv_common(2, x, e, dw, fmt, g, stream,
                       "conv backward expects matching rank-4 operands");
}
int fp8b_conv_tensor_supported(const fp8b_conv_t* g, int32_t fmt, int32_t kind) {
    if (!g || conv_validate(g, fmt, "conv") != FP8B_OK || kind < 0 || kind > 2) return 0;
    return fp8b::conv_tc_supported(kind, fmt, *g);
}
int fp8b_conv_halo_supported(const fp8b_conv_t* g, int32_t fmt, int32_t kind) {
    if (!fp8b_conv_tensor_supported(g, fmt, kind) || g->kh < 2) return 0;
    const int es = fmt == FP8B_E5M2 ? 1 : 2;
    const int64_t oh = g->h + 2 * g->pad - g->kh + 1, ow = g->w + 2 * g->pad - g->kw + 1;
    if (kind == 2)
        return fp8b::conv_halo_wgrad_supported(es, g->n, g->h, g->w, g->c, g->f, (int)g->kh, (int)g->pad);
    if (kind == 0) return fp8b::conv_halo_supported(es, g->n, g->h, g->w, g->c, g->f, (int)g->kh, (int)g->pad);
    // dgrad = fprop over e [n, oh, ow, f] with the flipped weights, pad' = k - 1 - pad
    return fp8b::conv_halo_supported(es, g->n, oh, ow, g->f, g->c, (int)g->kh, (int)(g->kh - 1 - g->pad));
}
int fp8b_im2col(const void* x, void* cols, int32_t fmt, const fp8b_conv_t* g, void* stream) {
    const int rc = conv_validate(g, fmt, "im2col expects [N, C, H, W]");
    if (rc) return rc;
    const int64_t oh = (g->h + 2 * g->pad - g->kh) / g->stride + 1;
    const int64_t ow = (g->w + 2 * g->pad - g->kw) / g->stride + 1;
    if (g->n * oh * ow * g->c * g->kh * g->kw == 0) return FP8B_OK;
    if (!x || !cols) return fail(FP8B_EINVAL, "im2col: null tensor");
    fp8b::launch_im2col(x, cols, fmt, *g, S(stream));
    return check_launch(1);
}

int fp8b_loss_scaler_init(fp8b_loss_scaler_t* dev_state, const fp8b_loss_scaler_t* o,
                          void* stream) {
    if (!dev_state || !o) return fail(FP8B_EINVAL, "loss_scaler_init: null pointer");
    // loss_scaling.cpp:19-38
    if (!(o->scale > 0.0) || !(o->scale < INFINITY))
        return fail(FP8B_EINVAL, "loss scale must be finite and positive");
    if (o->kind != FP8B_SCALER_CONSTANT && o->kind != FP8B_SCALER_DYNAMIC_BACKOFF)
        return fail(FP8B_EINVAL, "unknown scaler kind");
    if (o->n_schedule < 0 || o->n_schedule > FP8B_MAX_SCHEDULE)
        return fail(FP8B_EINVAL, "min threshold schedule too long");
    if (o->kind == FP8B_SCALER_DYNAMIC_BACKOFF) {
        if (!(o->backoff_factor > 0.0) || !(o->backoff_factor < 1.0))
            return fail(FP8B_EINVAL, "backoff factor must lie in (0, 1)");
        if (!(o->growth_factor > 1.0)) return fail(FP8B_EINVAL, "growth factor must exceed 1");
        if (o->growth_interval <= 0) return fail(FP8B_EINVAL, "growth interval must be positive");
        int64_t prev = -1;
        for (int i = 0; i < o->n_schedule; ++i) {
            if (o->sched_iter[i] <= prev)
                return fail(FP8B_EINVAL, "min threshold schedule iterations must increase");
            if (!(o->sched_scale[i] > 0.0)) return fail(FP8B_EINVAL, "min threshold must be positive");
            prev = o->sched_iter[i];
        }
    }
    static thread_local fp8b_loss_scaler_t h;
    h = *o;
    h.steps_since_overflow = 0;
    h.last_iteration = -1;
    h.last_action = FP8B_ACT_NONE;
    h.last_grads_finite = 1;
    h.last_scale_after = o->scale;
    h.step_ticket = 0;
    h.reserved = 0;
    if (cudaMemcpyAsync(dev_state, &h, sizeof(h), cudaMemcpyHostToDevice, S(stream)) != cudaSuccess ||
        cudaStreamSynchronize(S(stream)) != cudaSuccess) {
        cudaGetLastError();
        return fail(FP8B_ECUDA, "loss_scaler_init: copy failed");
    }
    return FP8B_OK;
}

int fp8b_loss_scaler_step(fp8b_loss_scaler_t* dev_state, const int64_t* counters,
                          int32_t grads_finite, int64_t iteration, void* stream) {
    if (!dev_state) return fail(FP8B_EINVAL, "loss_scaler_step: null state");
    fp8b::launch_scaler_step(dev_state, counters, grads_finite, iteration, S(stream));
    return check_launch(1);
}

int fp8b_unscale(float* g, int64_t n, const fp8b_loss_scaler_t* dev_state, void* stream) {
    if (n < 0) return fail(FP8B_EINVAL, "negative dimension");
    if (!dev_state) return fail(FP8B_EINVAL, "unscale: null state");
    if (n == 0) return FP8B_OK;
    if (!g) return fail(FP8B_EINVAL, "unscale: null tensor");
    fp8b::launch_unscale(g, n, dev_state, S(stream));
    return check_launch(1);
}

int fp8b_sgd_momentum_update(const void* grad, int32_t grad_fmt, uint16_t* master,
                             float* momentum, int64_t n, const fp8b_sgd_args_t* args,
                             void* stream) {
    if (!args) return fail(FP8B_EINVAL, "sgd: null args");
    if (n < 0) return fail(FP8B_EINVAL, "negative dimension");
    if (grad_fmt != FP8B_E5M2 && grad_fmt != FP8B_FP16 && grad_fmt != FP8B_F32)
        return fail(FP8B_EINVAL, "sgd: unknown gradient format");
    if (args->master_mode != FP8B_RNE && args->master_mode != FP8B_SR)
        return fail(FP8B_EINVAL, "sgd: master rounding must be nearest-even or stochastic");
    if (args->master_mode == FP8B_SR) {
        if (!valid_bits(args->bits)) return fail(FP8B_EINVAL, "sgd: unknown random-bits source");
        if (args->seed == 0) return fail(FP8B_EINVAL, "QuantConfig.seed must be nonzero");
        if (args->bits == FP8B_BITS_SUPPLIED && !args->rbits)
            return fail(FP8B_EINVAL, "sgd: supplied-bits SR needs rbits");
        if (args->block_offset < 0) return fail(FP8B_EINVAL, "sgd: negative block_offset");
    }
    if (!args->scaler && !(args->scale > 0.0f))
        return fail(FP8B_EINVAL, "loss scale must be finite and positive");
    if (args->step_scaler < 0 || args->step_scaler > 2)
        return fail(FP8B_EINVAL, "sgd: step_scaler must be 0, 1 or 2");
    if (args->step_scaler && !args->scaler)
        return fail(FP8B_EINVAL, "sgd: step_scaler needs a device scaler");
    if (args->gate_out && !args->step_scaler)
        return fail(FP8B_EINVAL, "sgd: gate_out is written by the fused scaler step (step_scaler)");
    if (args->gate_out && (args->gate_out == args->skip_counters || args->gate_out == args->skip_counters2))
        return fail(FP8B_EINVAL, "sgd: gate_out must not alias the gate's inputs");
    if (n == 0) {
        if (args->step_scaler && args->skip_counters2)
            return fail(FP8B_EINVAL, "sgd: an empty update cannot merge the gate");
        if (args->step_scaler) {  // nothing to update: the step alone
            fp8b::launch_scaler_step(const_cast<fp8b_loss_scaler_t*>(args->scaler),
                                     args->skip_counters, 1, args->step_iteration, S(stream));
            return check_launch(1);
        }
        return FP8B_OK;
    }
    if (!grad || !master || !momentum) return fail(FP8B_EINVAL, "sgd: null tensor");
    fp8b::LfsrTables tabs{nullptr, nullptr};
    if (args->master_mode == FP8B_SR && args->bits == FP8B_BITS_LFSR) {
        const int rc = get_tables(&tabs);
        if (rc) return rc;
    }
    fp8b::launch_sgd(grad, grad_fmt, master, momentum, n, *args, S(stream), tabs);
    return check_launch(1);
}

int fp8b_fill_synthetic(float* out, int64_t n, int32_t kind, uint64_t seed, double p, double lo,
                        double hi, void* stream) {
    if (n < 0 || kind < 0 || kind > 2) return fail(FP8B_EINVAL, "fill_synthetic: bad arguments");
    if (n == 0) return FP8B_OK;
    if (!out) return fail(FP8B_EINVAL, "fill_synthetic: null tensor");
    fp8b::launch_fill_synthetic(out, n, kind, seed, p, lo, hi, S(stream));
    return check_launch(1);
}

int fp8b_peer_alloc(void** ptr, int64_t bytes, unsigned char handle[FP8B_PEER_HANDLE_BYTES]) {
    static_assert(sizeof(cudaIpcMemHandle_t) == FP8B_PEER_HANDLE_BYTES, "handle size");
    if (!ptr || bytes <= 0) return fail(FP8B_EINVAL, "peer_alloc: bad arguments");
    void* p = nullptr;
    if (cudaMalloc(&p, (size_t)bytes) != cudaSuccess) {
        cudaGetLastError();
        return fail(FP8B_ECUDA, "peer_alloc: cudaMalloc failed");
    }
    if (handle) {
        cudaIpcMemHandle_t h;
        if (cudaIpcGetMemHandle(&h, p) != cudaSuccess) {
            cudaGetLastError();
            cudaFree(p);
            return fail(FP8B_ECUDA, "peer_alloc: cudaIpcGetMemHandle failed");
        }
        memcpy(handle, &h, sizeof(h));
    }
    *ptr = p;
    return FP8B_OK;
}
int fp8b_peer_free(void* ptr) {
    if (ptr && cudaFree(ptr) != cudaSuccess) {
        cudaGetLastError();
        return fail(FP8B_ECUDA, "peer_free: cudaFree failed");
    }
    return FP8B_OK;
}
int fp8b_peer_open(const unsigned char handle[FP8B_PEER_HANDLE_BYTES], void** ptr) {
    if (!handle || !ptr) return fail(FP8B_EINVAL, "peer_open: null argument");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    void* p = nullptr;
    if (cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
        cudaGetLastError();
        return fail(FP8B_ECUDA, "peer_open: cudaIpcOpenMemHandle failed");
    }
    *ptr = p;
    return FP8B_OK;
}
int fp8b_peer_close(void* ptr) {
    if (ptr && cudaIpcCloseMemHandle(ptr) != cudaSuccess) {
        cudaGetLastError();
        return fail(FP8B_ECUDA, "peer_close: cudaIpcCloseMemHandle failed");
    }
    return FP8B_OK;
}
int fp8b_peer_reduce_quantize(const float* const* peers, int32_t world, int64_t i0, int64_t n,
                              float* sum_out, void* codes, int32_t fmt,
                              const fp8b_quant_config_t* cfg, int64_t* counters, void* stream) {
    if (!cfg || !peers) return fail(FP8B_EINVAL, "peer_reduce_quantize: null argument");
    if (world < 1 || world > FP8B_MAX_PEERS) return fail(FP8B_EINVAL, "peer_reduce_quantize: bad world size");
    if (cfg->seed == 0) return fail(FP8B_EINVAL, "QuantConfig.seed must be nonzero");
    if (!valid_fmt(fmt)) return fail(FP8B_EINVAL, "peer_reduce_quantize: unknown float format");
    if (!valid_mode(cfg->mode)) return fail(FP8B_EINVAL, "unknown rounding mode");
    if (cfg->mode == FP8B_SR && cfg->bits != FP8B_BITS_COUNTER)
        return fail(FP8B_EINVAL, "peer_reduce_quantize: SR takes counter bits");
    if (i0 < 0 || n < 0 || (i0 & 3) || (n & 3) || cfg->block_offset < 0)
        return fail(FP8B_EINVAL, "peer_reduce_quantize: i0 and n must be non-negative multiples of 4");
    if (n == 0) return FP8B_OK;
    if (!codes) return fail(FP8B_EINVAL, "peer_reduce_quantize: null tensor");
    for (int r = 0; r < world; ++r)
        if (!peers[r] || ((uintptr_t)peers[r] % 16))
            return fail(FP8B_EINVAL, "peer_reduce_quantize: null or unaligned peer buffer");
    if (((uintptr_t)codes % 8) || (sum_out && ((uintptr_t)sum_out % 16)))
        return fail(FP8B_EINVAL, "peer_reduce_quantize: unaligned output");
    const int rc = fp8b::launch_peer_reduce_quantize(peers, world, i0, n, sum_out, codes, fmt, *cfg,
                                                     counters, S(stream));
    if (rc) return rc;
    return check_launch(1);
}

int fp8b_stream_probe(const float* x, void* out, int64_t n, int32_t out_bytes, void* stream) {
    if (n < 0 || (n & 3) || (out_bytes != 0 && out_bytes != 1 && out_bytes != 2 && out_bytes != 4))
        return fail(FP8B_EINVAL, "stream_probe: bad arguments");
    if (n == 0) return FP8B_OK;
    if (!x || (out_bytes && !out) || ((uintptr_t)x % 16) || ((uintptr_t)out % 16))
        return fail(FP8B_EINVAL, "stream_probe: null or unaligned tensor");
    fp8b::launch_stream_probe(x, out, n, out_bytes, S(stream));
    return check_launch(1);
}

}  // extern "C"
