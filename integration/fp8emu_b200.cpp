// fp8emu_b200.cpp -- implementation of the reference-side binding (see
// fp8emu_b200.hpp and INTEGRATION.md). Host tensors in, host tensors out, with
// the same validation and exceptions as the reference; the arithmetic runs in
// libfp8b200.so on the GPU.
#include "fp8emu_b200.hpp"

#include <cuda_runtime.h>

#include <cstring>
#include <stdexcept>
#include <string>

#include "fp8b200.h"

namespace fp8emu {
namespace b200 {
namespace {

void cuda_ok(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

void abi_ok(int rc) {
    if (rc == FP8B_OK) return;
    if (rc == FP8B_EINVAL) throw std::invalid_argument(fp8b_last_error());
    throw std::runtime_error(fp8b_last_error());
}

// RAII device buffer.
struct Dev {
    void* p = nullptr;
    explicit Dev(size_t bytes) {
        if (bytes) cuda_ok(cudaMalloc(&p, bytes), "cudaMalloc");
    }
    ~Dev() {
        if (p) cudaFree(p);
    }
    Dev(const Dev&) = delete;
    Dev& operator=(const Dev&) = delete;
    template <typename T>
    T* as() const { return static_cast<T*>(p); }
};

int fmt_id(const FloatFormat& f) {
    if (f == kFp8) return FP8B_E5M2;
    if (f == kFp16) return FP8B_FP16;
    throw std::invalid_argument("the B200 path supports the FP8 and FP16 formats");
}
int mode_id(RoundingMode m) {
    switch (m) {
    case RoundingMode::NearestEven: return FP8B_RNE;
    case RoundingMode::Stochastic: return FP8B_SR;
    case RoundingMode::TruncateTowardZero: return FP8B_TRUNC;
    }
    return FP8B_RNE;
}
size_t code_bytes(int fmt) { return fmt == FP8B_E5M2 ? 1 : 2; }

// u16 host codes (reference storage) <-> 1/2-byte device codes
void upload_codes(const QuantizedTensor& q, int fmt, void* dst) {
    const size_t n = q.codes.size();
    if (fmt == FP8B_FP16) {
        cuda_ok(cudaMemcpy(dst, q.codes.data(), n * 2, cudaMemcpyHostToDevice), "H2D");
    } else {
        std::vector<uint8_t> b(n);
        for (size_t i = 0; i < n; ++i) b[i] = static_cast<uint8_t>(q.codes[i]);
        cuda_ok(cudaMemcpy(dst, b.data(), n, cudaMemcpyHostToDevice), "H2D");
    }
}
void download_codes(const void* src, int fmt, std::vector<std::uint16_t>& out) {
    const size_t n = out.size();
    if (fmt == FP8B_FP16) {
        cuda_ok(cudaMemcpy(out.data(), src, n * 2, cudaMemcpyDeviceToHost), "D2H");
    } else {
        std::vector<uint8_t> b(n);
        cuda_ok(cudaMemcpy(b.data(), src, n, cudaMemcpyDeviceToHost), "D2H");
        for (size_t i = 0; i < n; ++i) out[i] = b[i];
    }
}

Tensor gemm_impl(const QuantizedTensor& a, const QuantizedTensor& b, int engine) {
    // kernels.cpp:38-44 (+ check_same_format, kernels.cpp:9-13)
    if (a.shape.size() != 2 || b.shape.size() != 2)
        throw std::invalid_argument("gemm_fp8 expects rank-2 operands");
    if (a.shape[1] != b.shape[0]) throw std::invalid_argument("gemm_fp8 inner dimensions disagree");
    if (!(a.fmt == b.fmt)) throw std::invalid_argument("kernel operands must share one format");
    const int64_t m = a.shape[0], k = a.shape[1], n = b.shape[1];
    const int fmt = fmt_id(a.fmt);
    Tensor y({m, n});
    if (m == 0 || n == 0) return y;
    Dev da(a.codes.size() * code_bytes(fmt)), db(b.codes.size() * code_bytes(fmt));
    Dev dc(sizeof(float) * (size_t)(m * n));
    upload_codes(a, fmt, da.p);
    upload_codes(b, fmt, db.p);
    fp8b_gemm_args_t args{};
    args.a_major = FP8B_K_MAJOR;
    args.b_major = FP8B_MN_MAJOR;  // B row-major [K, N], as the reference stores it
    args.engine = engine;
    args.c = dc.as<float>();
    abi_ok(fp8b_gemm(da.p, db.p, m, n, k, fmt, &args, nullptr));
    cuda_ok(cudaMemcpy(y.data.data(), dc.p, sizeof(float) * y.data.size(), cudaMemcpyDeviceToHost),
            "D2H");
    return y;
}

}  // namespace

QuantizedTensor quantize(const Tensor& t, const FloatFormat& fmt, const QuantConfig& cfg) {
    if (cfg.seed == 0) throw std::invalid_argument("QuantConfig.seed must be nonzero");
    const int f = fmt_id(fmt);
    QuantizedTensor q;
    q.shape = t.shape;
    q.fmt = fmt;
    q.mode_used = cfg.mode;
    q.codes.resize(t.data.size());
    const int64_t n = static_cast<int64_t>(t.data.size());
    if (n == 0) return q;
    Dev dx(sizeof(float) * n), dq(code_bytes(f) * n), dcnt(3 * sizeof(int64_t));
    cuda_ok(cudaMemcpy(dx.p, t.data.data(), sizeof(float) * n, cudaMemcpyHostToDevice), "H2D");
    cuda_ok(cudaMemset(dcnt.p, 0, 3 * sizeof(int64_t)), "memset");
    fp8b_quant_config_t c{};
    c.mode = mode_id(cfg.mode);
    c.bits = FP8B_BITS_LFSR;  // the reference stream (tensor.cpp:57-70)
    c.seed = cfg.seed;
    c.saturate = cfg.saturate_on_overflow ? 1 : 0;
    abi_ok(fp8b_quantize(dx.as<float>(), dq.p, n, f, &c, dcnt.as<int64_t>(), nullptr));
    download_codes(dq.p, f, q.codes);
    int64_t cnt[3];
    cuda_ok(cudaMemcpy(cnt, dcnt.p, sizeof(cnt), cudaMemcpyDeviceToHost), "D2H");
    q.overflow_count = cnt[0];
    q.underflow_count = cnt[1];
    return q;
}

Tensor dequantize(const QuantizedTensor& q) {
    const int f = fmt_id(q.fmt);
    Tensor t;
    t.shape = q.shape;
    t.data.resize(q.codes.size());
    const int64_t n = static_cast<int64_t>(q.codes.size());
    if (n == 0) return t;
    Dev dq(code_bytes(f) * n), dy(sizeof(float) * n);
    upload_codes(q, f, dq.p);
    abi_ok(fp8b_dequantize(dq.p, dy.as<float>(), n, f, nullptr));
    cuda_ok(cudaMemcpy(t.data.data(), dy.p, sizeof(float) * n, cudaMemcpyDeviceToHost), "D2H");
    return t;
}

QuantizedTensor transpose(const QuantizedTensor& q) {
    if (q.shape.size() != 2) throw std::invalid_argument("transpose expects a rank-2 tensor");
    const int f = fmt_id(q.fmt);
    QuantizedTensor out = q;
    out.shape = {q.shape[1], q.shape[0]};
    const int64_t n = static_cast<int64_t>(q.codes.size());
    if (n == 0) return out;
    Dev di(code_bytes(f) * n), dout(code_bytes(f) * n);
    upload_codes(q, f, di.p);
    abi_ok(fp8b_transpose(di.p, dout.p, q.shape[0], q.shape[1], f, nullptr));
    download_codes(dout.p, f, out.codes);
    return out;
}

Tensor gemm_fp8(const QuantizedTensor& a, const QuantizedTensor& b) {
    return gemm_impl(a, b, FP8B_GEMM_TENSOR);
}
Tensor gemm_fp8_exact(const QuantizedTensor& a, const QuantizedTensor& b) {
    return gemm_impl(a, b, FP8B_GEMM_SEQUENTIAL);
}

// ---- conv family (kernels.cpp:28-281), NCHW, sequential engine ------------
namespace {

int64_t out_dim(int64_t in, int64_t k, const ConvGeometry& g) {
    const int64_t span = in + 2 * g.pad - k;
    if (span < 0 || g.stride < 1) throw std::invalid_argument("convolution geometry does not fit input");
    return span / g.stride + 1;
}

fp8b_conv_t geom_of(int64_t n, int64_t c, int64_t h, int64_t w, int64_t f, int64_t kh, int64_t kw,
                    const ConvGeometry& g) {
    fp8b_conv_t cg{};
    cg.n = n; cg.c = c; cg.h = h; cg.w = w; cg.f = f; cg.kh = kh; cg.kw = kw;
    cg.stride = g.stride; cg.pad = g.pad;
    cg.layout = FP8B_NCHW;
    cg.engine = FP8B_GEMM_SEQUENTIAL;
    return cg;
}

using ConvFn = int (*)(const void*, const void*, float*, int32_t, const fp8b_conv_t*, void*);

Tensor run_conv(ConvFn fn, const QuantizedTensor& a, const QuantizedTensor& b,
                const fp8b_conv_t& cg, std::vector<int64_t> out_shape) {
    const int fmt = fmt_id(a.fmt);
    Tensor y(out_shape);
    if (y.data.empty()) return y;
    Dev da(a.codes.size() * code_bytes(fmt)), db(b.codes.size() * code_bytes(fmt));
    Dev dy(sizeof(float) * y.data.size());
    upload_codes(a, fmt, da.p);
    upload_codes(b, fmt, db.p);
    abi_ok(fn(da.p, db.p, dy.as<float>(), fmt, &cg, nullptr));
    cuda_ok(cudaMemcpy(y.data.data(), dy.p, sizeof(float) * y.data.size(), cudaMemcpyDeviceToHost),
            "D2H");
    return y;
}

}  // namespace

Tensor conv2d_fp8(const QuantizedTensor& x, const QuantizedTensor& w, const ConvGeometry& geom) {
    if (x.shape.size() != 4 || w.shape.size() != 4)
        throw std::invalid_argument("conv2d_fp8 expects [N,C,H,W] and [F,C,kH,kW]");
    if (x.shape[1] != w.shape[1]) throw std::invalid_argument("conv2d_fp8 channel counts disagree");
    if (!(x.fmt == w.fmt)) throw std::invalid_argument("kernel operands must share one format");
    const int64_t n = x.shape[0], c = x.shape[1], h = x.shape[2], iw = x.shape[3];
    const int64_t f = w.shape[0], kh = w.shape[2], kw = w.shape[3];
    const int64_t oh = out_dim(h, kh, geom), ow = out_dim(iw, kw, geom);
    return run_conv(fp8b_conv2d_fprop, x, w, geom_of(n, c, h, iw, f, kh, kw, geom), {n, f, oh, ow});
}

Tensor conv2d_backward_data_fp8(const QuantizedTensor& e, const QuantizedTensor& w,
                                const ConvGeometry& geom, std::int64_t h, std::int64_t w_dim) {
    if (e.shape.size() != 4 || w.shape.size() != 4)
        throw std::invalid_argument("conv backward expects rank-4 operands");
    if (e.shape[1] != w.shape[0]) throw std::invalid_argument("conv backward filter counts disagree");
    if (!(e.fmt == w.fmt)) throw std::invalid_argument("kernel operands must share one format");
    const int64_t n = e.shape[0], f = e.shape[1], c = w.shape[1], kh = w.shape[2], kw = w.shape[3];
    if (out_dim(h, kh, geom) != e.shape[2] || out_dim(w_dim, kw, geom) != e.shape[3])
        throw std::invalid_argument("conv backward geometry disagrees with error");
    return run_conv(fp8b_conv2d_dgrad, e, w, geom_of(n, c, h, w_dim, f, kh, kw, geom), {n, c, h, w_dim});
}

Tensor conv2d_backward_weights_fp8(const QuantizedTensor& x, const QuantizedTensor& e,
                                   std::int64_t kh, std::int64_t kw, const ConvGeometry& geom) {
    if (x.shape.size() != 4 || e.shape.size() != 4 || x.shape[0] != e.shape[0])
        throw std::invalid_argument("conv backward expects matching rank-4 operands");
    if (!(x.fmt == e.fmt)) throw std::invalid_argument("kernel operands must share one format");
    const int64_t n = x.shape[0], c = x.shape[1], h = x.shape[2], iw = x.shape[3], f = e.shape[1];
    if (out_dim(h, kh, geom) != e.shape[2] || out_dim(iw, kw, geom) != e.shape[3])
        throw std::invalid_argument("conv backward geometry disagrees with error");
    return run_conv(fp8b_conv2d_wgrad, x, e, geom_of(n, c, h, iw, f, kh, kw, geom), {f, c, kh, kw});
}

QuantizedTensor im2col(const QuantizedTensor& x, std::int64_t kh, std::int64_t kw,
                       const ConvGeometry& geom) {
    if (x.shape.size() != 4) throw std::invalid_argument("im2col expects [N, C, H, W]");
    const int64_t n = x.shape[0], c = x.shape[1], h = x.shape[2], iw = x.shape[3];
    const int64_t oh = out_dim(h, kh, geom), ow = out_dim(iw, kw, geom);
    const int fmt = fmt_id(x.fmt);
    QuantizedTensor cols;
    cols.fmt = x.fmt;
    cols.mode_used = x.mode_used;
    cols.shape = {c * kh * kw, n * oh * ow};
    cols.codes.assign(static_cast<size_t>(cols.shape[0] * cols.shape[1]), 0);
    if (cols.codes.empty()) return cols;
    Dev dx(x.codes.size() * code_bytes(fmt)), dc(cols.codes.size() * code_bytes(fmt));
    upload_codes(x, fmt, dx.p);
    const fp8b_conv_t cg = geom_of(n, c, h, iw, 1, kh, kw, geom);
    abi_ok(fp8b_im2col(dx.p, dc.p, fmt, &cg, nullptr));
    download_codes(dc.p, fmt, cols.codes);
    return cols;
}

Tensor conv2d_fp8_im2col(const QuantizedTensor& x, const QuantizedTensor& w,
                         const ConvGeometry& geom) {
    // kernels.cpp:255-281: W [F, C*kh*kw] x cols [C*kh*kw, N*OH*OW], then NCHW
    const int64_t n = x.shape[0];
    const int64_t f = w.shape[0], c = w.shape[1], kh = w.shape[2], kw = w.shape[3];
    const int64_t oh = out_dim(x.shape[2], kh, geom), ow = out_dim(x.shape[3], kw, geom);
    const QuantizedTensor cols = b200::im2col(x, kh, kw, geom);
    const QuantizedTensor wmat = w.reshaped({f, c * kh * kw});
    const Tensor flat = gemm_fp8_exact(wmat, cols);
    Tensor y({n, f, oh, ow});
    const int64_t ncols = n * oh * ow;
    for (int64_t ni = 0; ni < n; ++ni)
        for (int64_t fi = 0; fi < f; ++fi)
            for (int64_t p = 0; p < oh * ow; ++p)
                y.data[static_cast<size_t>((ni * f + fi) * oh * ow + p)] =
                    flat.data[static_cast<size_t>(fi * ncols + ni * oh * ow + p)];
    return y;
}

LossScaler::LossScaler(const fp8emu::LossScaler::Options& o) : opts_(o) {
    fp8b_loss_scaler_t h{};
    h.kind = o.kind == fp8emu::LossScaler::Kind::Constant ? FP8B_SCALER_CONSTANT
                                                          : FP8B_SCALER_DYNAMIC_BACKOFF;
    h.scale = o.scale;
    h.backoff_factor = o.backoff_factor;
    h.growth_factor = o.growth_factor;
    h.growth_interval = o.growth_interval;
    if (o.min_threshold_schedule.size() > FP8B_MAX_SCHEDULE)
        throw std::invalid_argument("min threshold schedule too long for the device scaler");
    h.n_schedule = static_cast<int32_t>(o.min_threshold_schedule.size());
    for (size_t i = 0; i < o.min_threshold_schedule.size(); ++i) {
        h.sched_iter[i] = o.min_threshold_schedule[i].first;
        h.sched_scale[i] = o.min_threshold_schedule[i].second;
    }
    cuda_ok(cudaMalloc(&dev_, sizeof(fp8b_loss_scaler_t)), "cudaMalloc");
    const int rc = fp8b_loss_scaler_init(static_cast<fp8b_loss_scaler_t*>(dev_), &h, nullptr);
    if (rc != FP8B_OK) {
        cudaFree(dev_);
        dev_ = nullptr;
        abi_ok(rc);
    }
}

LossScaler::~LossScaler() {
    if (dev_) cudaFree(dev_);
}

double LossScaler::scale() const {
    fp8b_loss_scaler_t h;
    cuda_ok(cudaMemcpy(&h, dev_, sizeof(h), cudaMemcpyDeviceToHost), "D2H");
    return h.scale;
}

double LossScaler::min_threshold(std::int64_t iteration) const {
    double thr = 1.0;  // loss_scaling.cpp:40-47
    for (const auto& [it, sc] : opts_.min_threshold_schedule) {
        if (it > iteration) break;
        thr = sc;
    }
    return thr;
}

ScaleEvent LossScaler::step(bool grads_finite, std::int64_t iteration) {
    abi_ok(fp8b_loss_scaler_step(static_cast<fp8b_loss_scaler_t*>(dev_), nullptr,
                                 grads_finite ? 1 : 0, iteration, nullptr));
    fp8b_loss_scaler_t h;
    cuda_ok(cudaMemcpy(&h, dev_, sizeof(h), cudaMemcpyDeviceToHost), "D2H");
    ScaleEvent ev;
    ev.iteration = h.last_iteration;
    ev.action = static_cast<ScaleAction>(h.last_action);
    ev.scale_after = h.last_scale_after;
    return ev;
}

Tensor LossScaler::unscale_gradients(const Tensor& g) const {
    Tensor out = g;
    const int64_t n = static_cast<int64_t>(g.data.size());
    if (n == 0) return out;
    Dev d(sizeof(float) * n);
    cuda_ok(cudaMemcpy(d.p, g.data.data(), sizeof(float) * n, cudaMemcpyHostToDevice), "H2D");
    abi_ok(fp8b_unscale(d.as<float>(), n, static_cast<const fp8b_loss_scaler_t*>(dev_), nullptr));
    cuda_ok(cudaMemcpy(out.data.data(), d.p, sizeof(float) * n, cudaMemcpyDeviceToHost), "D2H");
    return out;
}

void update_tensor(nn::ParamTensor& p, const std::vector<float>& g, float scale, float lr,
                   float mu, float two_lambda, RoundingMode master_mode, std::uint64_t seed) {
    const int64_t n = static_cast<int64_t>(p.value.size());
    if (static_cast<int64_t>(g.size()) != n || p.master.size() != p.value.size() ||
        p.momentum.size() != p.value.size())
        throw std::invalid_argument("update_tensor: operand sizes disagree");
    if (n == 0) return;
    Dev dg(sizeof(float) * n), dm(2 * n), dv(sizeof(float) * n);
    cuda_ok(cudaMemcpy(dg.p, g.data(), sizeof(float) * n, cudaMemcpyHostToDevice), "H2D");
    cuda_ok(cudaMemcpy(dm.p, p.master.data(), 2 * n, cudaMemcpyHostToDevice), "H2D");
    cuda_ok(cudaMemcpy(dv.p, p.momentum.data(), sizeof(float) * n, cudaMemcpyHostToDevice), "H2D");
    fp8b_sgd_args_t a{};
    a.lr = lr;
    a.mu = mu;
    a.two_lambda = two_lambda;
    a.scale = scale;
    a.master_mode = master_mode == RoundingMode::Stochastic ? FP8B_SR : FP8B_RNE;
    a.bits = FP8B_BITS_LFSR;
    a.seed = seed;
    abi_ok(fp8b_sgd_momentum_update(dg.p, FP8B_F32, dm.as<uint16_t>(), dv.as<float>(), n, &a,
                                    nullptr));
    cuda_ok(cudaMemcpy(p.master.data(), dm.p, 2 * n, cudaMemcpyDeviceToHost), "D2H");
    cuda_ok(cudaMemcpy(p.momentum.data(), dv.p, sizeof(float) * n, cudaMemcpyDeviceToHost), "D2H");
    for (int64_t j = 0; j < n; ++j) p.value[j] = decode_to_float(p.master[j], kFp16);
}

}  // namespace b200
}  // namespace fp8emu
