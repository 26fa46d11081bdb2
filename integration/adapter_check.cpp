// adapter_check.cpp -- TEST DRIVER: links the UNMODIFIED reference library and
// the fp8emu::b200 drop-in side by side and checks that the drop-in returns
// what the reference returns, through the reference's own C++ types. Built by
// `make -C oracle adapter` (needs /root/reference headers at build time) into
// oracle/_ref/adapter_check; run on the GPU box by tests/test_adapter_gpu.py.
// The checks follow the reference's acceptance criteria 2, 5 and 6
// (acceptance.cpp:68-124, 184-250, 255-316) and its unit tests.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "fp8emu/rand.hpp"
#include "fp8emu_b200.hpp"

using namespace fp8emu;

static int g_fail = 0;
static void report(const char* name, const std::string& why) {
    if (why.empty()) std::printf("PASS %s\n", name);
    else { std::printf("FAIL %s: %s\n", name, why.c_str()); ++g_fail; }
}

static Tensor random_tensor(std::vector<int64_t> shape, uint64_t seed, double lo, double hi) {
    Tensor t(std::move(shape));
    Rand r{seed};
    for (auto& v : t.data) v = static_cast<float>(lo + (hi - lo) * r.uniform());
    return t;
}

static std::string check_quantize() {
    // log-uniform magnitudes across subnormal..overflow plus specials (criterion 2 ranges)
    Tensor t({(1 << 21) + 777});
    Rand r{20190529};
    for (auto& v : t.data) {
        const double mag = std::pow(2.0, -26.0 + 44.0 * r.uniform());
        v = static_cast<float>(r.uniform() < 0.5 ? -mag : mag);
    }
    t.data[0] = 0.0f; t.data[1] = -0.0f; t.data[2] = INFINITY; t.data[3] = NAN;
    t.data[4] = 57344.0f; t.data[5] = 57345.0f; t.data[6] = 65504.0f; t.data[7] = 70000.0f;
    for (const FloatFormat* f : {&kFp8, &kFp16})
        for (RoundingMode m : {RoundingMode::NearestEven, RoundingMode::Stochastic,
                               RoundingMode::TruncateTowardZero})
            for (bool sat : {false, true}) {
                QuantConfig cfg;
                cfg.mode = m;
                cfg.seed = 977;
                cfg.saturate_on_overflow = sat;
                const QuantizedTensor a = fp8emu::quantize(t, *f, cfg);
                const QuantizedTensor b = fp8emu::b200::quantize(t, *f, cfg);
                if (a.codes != b.codes) return std::string("codes differ: ") + f->name + " " + to_string(m);
                if (a.overflow_count != b.overflow_count || a.underflow_count != b.underflow_count)
                    return std::string("counters differ: ") + f->name + " " + to_string(m);
                const Tensor da = fp8emu::dequantize(a), db = fp8emu::b200::dequantize(b);
                if (std::memcmp(da.data.data(), db.data.data(), 4 * da.data.size()) != 0)
                    return "dequantize differs";
            }
    return "";
}

static std::string check_block_contract() {
    // test_quantize.cpp:94-120: whole-tensor SR == per-block split(seed, b) + encode
    const int64_t n = kQuantBlock * 2 + kQuantBlock / 2;
    Tensor t({n});
    for (int64_t i = 0; i < n; ++i) t.at(i) = 0.37f + 0.0001f * static_cast<float>(i % 977);
    QuantConfig cfg;
    cfg.mode = RoundingMode::Stochastic;
    cfg.seed = 1337;
    const QuantizedTensor whole = fp8emu::b200::quantize(t, kFp8, cfg);
    for (int64_t block = 0; block * kQuantBlock < n; ++block) {
        LfsrStream stream = LfsrStream::split(cfg.seed, static_cast<uint64_t>(block));
        for (int64_t i = block * kQuantBlock; i < std::min(n, (block + 1) * kQuantBlock); ++i)
            if (encode(t.at(i), kFp8, RoundingMode::Stochastic, &stream).code != whole.code_at(i))
                return "block stream mismatch at " + std::to_string(i);
    }
    return "";
}

static std::string check_gemm() {
    // criterion 5: 100 random shapes with dims <= 16, bitwise vs gemm_fp8
    LfsrStream dims = LfsrStream::split(0xD1, 0);
    QuantConfig cfg;
    for (int trial = 0; trial < 100; ++trial) {
        const int64_t m = 1 + dims.next_bits() % 16, k = 1 + dims.next_bits() % 16,
                      n = 1 + dims.next_bits() % 16;
        const QuantizedTensor a = fp8emu::quantize(random_tensor({m, k}, 100 + trial, -2, 2), kFp8, cfg);
        const QuantizedTensor b = fp8emu::quantize(random_tensor({k, n}, 200 + trial, -2, 2), kFp8, cfg);
        const Tensor ref = fp8emu::gemm_fp8(a, b);
        const Tensor ex = fp8emu::b200::gemm_fp8_exact(a, b);
        if (std::memcmp(ref.data.data(), ex.data.data(), 4 * ref.data.size()) != 0)
            return "sequential engine not bitwise at trial " + std::to_string(trial);
        const Tensor tc = fp8emu::b200::gemm_fp8(a, b);
        const Tensor da = fp8emu::dequantize(a), db = fp8emu::dequantize(b);
        for (int64_t i = 0; i < m; ++i)
            for (int64_t j = 0; j < n; ++j) {
                double absdot = 0, exact = 0;
                for (int64_t p = 0; p < k; ++p) {
                    const double pr = (double)da.at(i * k + p) * (double)db.at(p * n + j);
                    exact += pr;
                    absdot += std::fabs(pr);
                }
                if (std::fabs((double)tc.at(i * n + j) - exact) > 1e-6 * absdot + 1e-30)
                    return "tensor engine outside tolerance at trial " + std::to_string(trial);
            }
    }
    // a larger shape, tensor engine vs reference under the stated tolerance
    const int64_t m = 192, k = 320, n = 256;
    const QuantizedTensor a = fp8emu::quantize(random_tensor({m, k}, 7, -2, 2), kFp8, cfg);
    const QuantizedTensor b = fp8emu::quantize(random_tensor({k, n}, 8, -2, 2), kFp8, cfg);
    const Tensor ref = fp8emu::gemm_fp8(a, b), tc = fp8emu::b200::gemm_fp8(a, b);
    const Tensor ex = fp8emu::b200::gemm_fp8_exact(a, b);
    if (std::memcmp(ref.data.data(), ex.data.data(), 4 * ref.data.size()) != 0)
        return "sequential engine not bitwise at 192x320x256";
    for (size_t i = 0; i < ref.data.size(); ++i)
        if (std::fabs(ref.data[i] - tc.data[i]) > 1e-3f * (1.0f + std::fabs(ref.data[i])))
            return "tensor engine far from reference at 192x320x256";
    // error behaviour (kernels.cpp:38-44)
    try {
        fp8emu::b200::gemm_fp8(a, a);
        return "shape mismatch did not throw";
    } catch (const std::invalid_argument&) {
    }
    const QuantizedTensor c16 = fp8emu::quantize(random_tensor({k, n}, 3, -2, 2), kFp16, cfg);
    try {
        fp8emu::b200::gemm_fp8(a, c16);
        return "format mismatch did not throw";
    } catch (const std::invalid_argument&) {
    }
    return "";
}

static std::string check_scaler() {
    // criterion 6 (acceptance.cpp:255-283)
    LossScaler::Options o;
    o.kind = LossScaler::Kind::DynamicBackoff;
    o.scale = 65536.0;
    o.growth_interval = 100;
    o.min_threshold_schedule = {{40, 8192.0}, {150, 32768.0}};
    LossScaler ref(o);
    b200::LossScaler dev(o);
    std::vector<std::pair<bool, int64_t>> steps = {{false, 10}, {false, 10}};
    for (int i = 0; i < 10; ++i) steps.push_back({false, 50});
    for (int i = 0; i < 100; ++i) steps.push_back({true, 100});
    steps.push_back({true, 151});
    for (auto [fin, it] : steps) {
        const ScaleEvent a = ref.step(fin, it), b = dev.step(fin, it);
        if (a.action != b.action || a.scale_after != b.scale_after)
            return "trace diverges at iteration " + std::to_string(it);
    }
    if (dev.min_threshold(149) != 8192.0 || dev.min_threshold(150) != 32768.0)
        return "min_threshold";
    // constructor validation (loss_scaling.cpp:19-38)
    LossScaler::Options bad = o;
    bad.backoff_factor = 1.0;
    try {
        b200::LossScaler s(bad);
        return "bad options accepted";
    } catch (const std::invalid_argument&) {
    }
    // unscale is true FP32 division (test_loss_scaling.cpp:170-176)
    LossScaler::Options o3;
    o3.scale = 3.0;
    b200::LossScaler s3(o3);
    Tensor h({1});
    h.data = {9.0f};
    if (s3.unscale_gradients(h).data[0] != 3.0f) return "unscale is not true division";
    return "";
}

static std::string check_update() {
    // update_tensor (nn.cpp:417-432) restated with the reference's encode
    const int64_t n = 3 * 4096 + 5;
    nn::ParamTensor p;
    p.shape = {n};
    Rand r{11};
    p.value.resize(n);
    p.master.resize(n);
    p.momentum.resize(n);
    std::vector<float> g(n);
    for (int64_t j = 0; j < n; ++j) {
        const EncodeResult e = encode(r.normal() / 32.0, kFp16, RoundingMode::NearestEven);
        p.master[j] = static_cast<uint16_t>(e.code);
        p.value[j] = static_cast<float>(decode(e.code, kFp16));
        p.momentum[j] = static_cast<float>(r.normal() * 1e-3);
        g[j] = static_cast<float>(r.normal() * 100.0);
    }
    nn::ParamTensor q = p;
    const float scale = 8192.0f, lr = 0.1f, mu = 0.9f, tl = 2e-4f;
    std::vector<float> w32(n);
    for (int64_t j = 0; j < n; ++j) {
        float gv = g[j] / scale;
        if (tl != 0.0f) gv += tl * q.value[j];
        q.momentum[j] = mu * q.momentum[j] + gv;
        w32[j] = q.value[j] - lr * q.momentum[j];
        q.master[j] = static_cast<uint16_t>(encode(w32[j], kFp16, RoundingMode::NearestEven).code);
        q.value[j] = static_cast<float>(decode(q.master[j], kFp16));
    }
    nn::ParamTensor d = p;
    b200::update_tensor(d, g, scale, lr, mu, tl);
    if (d.master != q.master) return "RNE masters differ";
    if (std::memcmp(d.momentum.data(), q.momentum.data(), 4 * n) != 0) return "momentum differs";
    if (std::memcmp(d.value.data(), q.value.data(), 4 * n) != 0) return "values differ";
    // SR master == reference quantize(Tensor(w32), kFp16, {Stochastic, seed})
    QuantConfig cfg;
    cfg.mode = RoundingMode::Stochastic;
    cfg.seed = 5;
    const QuantizedTensor sr = fp8emu::quantize(Tensor({n}, w32), kFp16, cfg);
    nn::ParamTensor d2 = p;
    b200::update_tensor(d2, g, scale, lr, mu, tl, RoundingMode::Stochastic, 5);
    if (d2.master != sr.codes) return "SR masters differ from the reference stream";
    return "";
}

static std::string check_conv() {
    // test_kernels.cpp:97-184 style: random NCHW shapes, every conv-family entry
    // point bitwise against the reference library.
    LfsrStream dims = LfsrStream::split(0xC0, 0);
    QuantConfig cfg;
    for (int trial = 0; trial < 24; ++trial) {
        const int64_t n = 1 + dims.next_bits() % 2, c = 1 + dims.next_bits() % 4,
                      h = 3 + dims.next_bits() % 6, w = 3 + dims.next_bits() % 6,
                      f = 1 + dims.next_bits() % 4, kh = 1 + dims.next_bits() % 3,
                      kw = 1 + dims.next_bits() % 3;
        ConvGeometry g;
        g.stride = 1 + dims.next_bits() % 2;
        g.pad = dims.next_bits() % 2;
        if (conv_out_dim(h, kh, g.stride, g.pad) < 1 || conv_out_dim(w, kw, g.stride, g.pad) < 1)
            continue;
        const int64_t oh = conv_out_dim(h, kh, g.stride, g.pad), ow = conv_out_dim(w, kw, g.stride, g.pad);
        const FloatFormat& fm = (trial & 1) ? kFp16 : kFp8;
        const QuantizedTensor x = fp8emu::quantize(random_tensor({n, c, h, w}, 300 + trial, -2, 2), fm, cfg);
        const QuantizedTensor k = fp8emu::quantize(random_tensor({f, c, kh, kw}, 400 + trial, -2, 2), fm, cfg);
        const QuantizedTensor e = fp8emu::quantize(random_tensor({n, f, oh, ow}, 500 + trial, -2, 2), fm, cfg);
        auto same = [](const Tensor& a, const Tensor& b) {
            return a.shape == b.shape && std::memcmp(a.data.data(), b.data.data(), 4 * a.data.size()) == 0;
        };
        if (!same(fp8emu::conv2d_fp8(x, k, g), fp8emu::b200::conv2d_fp8(x, k, g)))
            return "conv2d_fp8 differs at trial " + std::to_string(trial);
        if (!same(fp8emu::conv2d_fp8_im2col(x, k, g), fp8emu::b200::conv2d_fp8_im2col(x, k, g)))
            return "conv2d_fp8_im2col differs at trial " + std::to_string(trial);
        if (!same(fp8emu::conv2d_backward_data_fp8(e, k, g, h, w),
                  fp8emu::b200::conv2d_backward_data_fp8(e, k, g, h, w)))
            return "conv2d_backward_data_fp8 differs at trial " + std::to_string(trial);
        if (!same(fp8emu::conv2d_backward_weights_fp8(x, e, kh, kw, g),
                  fp8emu::b200::conv2d_backward_weights_fp8(x, e, kh, kw, g)))
            return "conv2d_backward_weights_fp8 differs at trial " + std::to_string(trial);
        if (fp8emu::im2col(x, kh, kw, g).codes != fp8emu::b200::im2col(x, kh, kw, g).codes)
            return "im2col differs at trial " + std::to_string(trial);
    }
    return "";
}

static std::string check_errors() {
    Tensor t({4});
    QuantConfig cfg;
    cfg.seed = 0;
    bool ref_threw = false, dev_threw = false;
    try { fp8emu::quantize(t, kFp8, cfg); } catch (const std::invalid_argument&) { ref_threw = true; }
    try { fp8emu::b200::quantize(t, kFp8, cfg); } catch (const std::invalid_argument&) { dev_threw = true; }
    if (!(ref_threw && dev_threw)) return "zero seed behaviour differs";
    return "";
}

int main() {
    report("quantize_all_modes_vs_reference", check_quantize());
    report("sr_block_stream_contract", check_block_contract());
    report("gemm_criterion5_bitwise_and_tolerance", check_gemm());
    report("loss_scaler_criterion6", check_scaler());
    report("update_tensor_rne_and_sr", check_update());
    report("conv_family_bitwise", check_conv());
    report("error_behaviour", check_errors());
    std::printf("%d failure(s)\n", g_fail);
    return g_fail;
}
