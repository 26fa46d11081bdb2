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
