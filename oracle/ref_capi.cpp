// ref_capi.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" shim over the UNMODIFIED reference library
// (/root/reference/proj/src/{lfsr,float_format,tensor,kernels,loss_scaling,tensor_io}.cpp,
// compiled in place by oracle/Makefile into oracle/_ref/libfp8emu_ref.so).
// It lets the pytest suite and bench.py's reference arm drive the reference's
// public C++ API through ctypes. Nothing here is product code.
//
// The only restated piece is ref_update(): the reference's update_tensor
// (nn.cpp:417-432) has internal linkage, so its 6 lines of arithmetic are
// repeated here verbatim in semantics, calling the reference's own encode().

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <thread>
#include <vector>

#include "fp8emu/float_format.hpp"
#include "fp8emu/kernels.hpp"
#include "fp8emu/lfsr.hpp"
#include "fp8emu/loss_scaling.hpp"
#include "fp8emu/rand.hpp"
#include "fp8emu/tensor.hpp"
#include "fp8emu/tensor_io.hpp"

using namespace fp8emu;

namespace {
const FloatFormat& fmt_of(int f) { return f == 0 ? kFp8 : kFp16; }
RoundingMode mode_of(int m) {
    return m == 0 ? RoundingMode::NearestEven
                  : (m == 1 ? RoundingMode::Stochastic : RoundingMode::TruncateTowardZero);
}
}  // namespace

extern "C" {

uint64_t ref_mix64(uint64_t x) { return mix64(x); }
uint64_t ref_mix_seed(uint64_t s, uint64_t i) { return mix_seed(s, i); }

uint16_t ref_lfsr_split(uint64_t seed, uint64_t idx) {
    return LfsrStream::split(seed, idx).state();
}

// Draw `count` 16-bit samples from LfsrStream(state).
void ref_lfsr_samples(uint16_t state, int64_t count, uint32_t* out) {
    LfsrStream s(state);
    for (int64_t i = 0; i < count; ++i) out[i] = s.next_bits();
}

double ref_decode(uint32_t code, int fmt) { return decode(code, fmt_of(fmt)); }

// bindings.cpp:138-152 semantics: SR draws from LfsrStream::split(seed, 0).
uint32_t ref_encode(double x, int fmt, int mode, uint64_t seed, int saturate,
                    int* overflowed, int* underflowed) {
    LfsrStream rng = LfsrStream::split(seed, 0);
    const RoundingMode rm = mode_of(mode);
    const EncodeResult r = encode(x, fmt_of(fmt), rm,
                                  rm == RoundingMode::Stochastic ? &rng : nullptr,
                                  saturate != 0);
    *overflowed = r.overflowed;
    *underflowed = r.underflowed_to_zero;
    return r.code;
}

// encode with an explicit LFSR state (r16 sample stream = LfsrStream(state)).
uint32_t ref_encode_state(double x, int fmt, int mode, uint16_t* state,
                          int saturate, int* overflowed, int* underflowed) {
    LfsrStream rng(*state);
    const EncodeResult r = encode(x, fmt_of(fmt), mode_of(mode), &rng, saturate != 0);
    *state = rng.state();
    *overflowed = r.overflowed;
    *underflowed = r.underflowed_to_zero;
    return r.code;
}

// fp8emu::quantize (tensor.cpp:46-81). Returns 22 on std::invalid_argument.
int ref_quantize(const float* x, int64_t n, int fmt, int mode, uint64_t seed,
                 int saturate, uint16_t* codes, int64_t* counters) {
    try {
        Tensor t({n}, std::vector<float>(x, x + n));
        QuantConfig cfg;
        cfg.mode = mode_of(mode);
        cfg.seed = seed;
        cfg.saturate_on_overflow = saturate != 0;
        const QuantizedTensor q = quantize(t, fmt_of(fmt), cfg);
        std::memcpy(codes, q.codes.data(), sizeof(uint16_t) * q.codes.size());
        counters[0] += q.overflow_count;
        counters[1] += q.underflow_count;
        return 0;
    } catch (const std::invalid_argument&) {
        return 22;
    }
}

// Block-parallel harness around the reference's public encode()/split()
// (the schedule-independence contract of tensor.hpp:55-58, pinned by
// test_quantize.cpp:94-120): thread t takes whole 4096-element blocks and
// rounds them with LfsrStream::split(seed, global_block). Bit-identical to
// quantize(); used as the multi-core CPU baseline. Codes are u8 for E5M2.
int ref_quantize_mt(const float* x, int64_t n, int fmt, int mode, uint64_t seed,
                    int saturate, void* codes, int64_t* counters, int nthreads) {
    if (seed == 0) return 22;
    const int64_t kB = kQuantBlock;
    const int64_t nblocks = (n + kB - 1) / kB;
    if (nthreads < 1) nthreads = 1;
    std::vector<int64_t> ovf(nthreads, 0), unf(nthreads, 0);
    const FloatFormat& f = fmt_of(fmt);
    const RoundingMode rm = mode_of(mode);
    auto work = [&](int tid) {
        for (int64_t b = tid; b < nblocks; b += nthreads) {
            LfsrStream rng = LfsrStream::split(seed, static_cast<uint64_t>(b));
            const int64_t end = std::min(n, (b + 1) * kB);
            for (int64_t i = b * kB; i < end; ++i) {
                const EncodeResult r =
                    encode(x[i], f, rm, rm == RoundingMode::Stochastic ? &rng : nullptr,
                           saturate != 0);
                if (fmt == 0) static_cast<uint8_t*>(codes)[i] = static_cast<uint8_t>(r.code);
                else static_cast<uint16_t*>(codes)[i] = static_cast<uint16_t>(r.code);
                ovf[tid] += r.overflowed;
                unf[tid] += r.underflowed_to_zero;
            }
        }
    };
    std::vector<std::thread> th;
    for (int t = 1; t < nthreads; ++t) th.emplace_back(work, t);
    work(0);
    for (auto& t : th) t.join();
    for (int t = 0; t < nthreads; ++t) { counters[0] += ovf[t]; counters[1] += unf[t]; }
    return 0;
}

void ref_dequantize(const uint16_t* codes, int64_t n, int fmt, float* out) {
    QuantizedTensor q;
    q.shape = {n};
    q.codes.assign(codes, codes + n);
    q.fmt = fmt_of(fmt);
    const Tensor t = dequantize(q);
    std::memcpy(out, t.data.data(), sizeof(float) * t.data.size());
}

// fp8emu::gemm_fp8 (kernels.cpp:37-62). Returns 22 on invalid_argument.
int ref_gemm(const uint16_t* a, const uint16_t* b, int64_t m, int64_t k, int64_t n,
             int fmt, float* c) {
    try {
        QuantizedTensor qa, qb;
        qa.shape = {m, k};
        qa.codes.assign(a, a + m * k);
        qa.fmt = fmt_of(fmt);
        qb.shape = {k, n};
        qb.codes.assign(b, b + k * n);
        qb.fmt = fmt_of(fmt);
        const Tensor y = gemm_fp8(qa, qb);
        std::memcpy(c, y.data.data(), sizeof(float) * y.data.size());
        return 0;
    } catch (const std::invalid_argument&) {
        return 22;
    }
}

// Row-parallel harness: each thread calls gemm_fp8 on a slab of A's rows;
// results are per-element identical to the single call.
int ref_gemm_mt(const uint16_t* a, const uint16_t* b, int64_t m, int64_t k, int64_t n,
                int fmt, float* c, int nthreads) {
    if (nthreads < 1) nthreads = 1;
    QuantizedTensor qb;
    qb.shape = {k, n};
    qb.codes.assign(b, b + k * n);
    qb.fmt = fmt_of(fmt);
    const int64_t rows = (m + nthreads - 1) / nthreads;
    auto work = [&](int tid) {
        const int64_t r0 = tid * rows, r1 = std::min(m, r0 + rows);
        if (r0 >= r1) return;
        QuantizedTensor qa;
        qa.shape = {r1 - r0, k};
        qa.codes.assign(a + r0 * k, a + r1 * k);
        qa.fmt = fmt_of(fmt);
        const Tensor y = gemm_fp8(qa, qb);
        std::memcpy(c + r0 * n, y.data.data(), sizeof(float) * y.data.size());
    };
    std::vector<std::thread> th;
    for (int t = 1; t < nthreads; ++t) th.emplace_back(work, t);
    work(0);
    for (auto& t : th) t.join();
    return 0;
}

// conv family (kernels.hpp:22-50). kind: 0 fprop, 1 dgrad, 2 wgrad.
int ref_conv(int kind, const uint16_t* a, const uint16_t* b, int64_t n, int64_t c, int64_t h,
             int64_t wd, int64_t f, int64_t kh, int64_t kw, int64_t stride, int64_t pad, int fmt,
             float* out) {
    try {
        const ConvGeometry g{stride, pad};
        const int64_t oh = conv_out_dim(h, kh, stride, pad), ow = conv_out_dim(wd, kw, stride, pad);
        auto qt = [&](const uint16_t* p, std::vector<int64_t> shape) {
            QuantizedTensor q;
            q.shape = shape;
            q.codes.assign(p, p + shape_numel(shape));
            q.fmt = fmt_of(fmt);
            return q;
        };
        Tensor y;
        if (kind == 0) y = conv2d_fp8(qt(a, {n, c, h, wd}), qt(b, {f, c, kh, kw}), g);
        else if (kind == 1) y = conv2d_backward_data_fp8(qt(a, {n, f, oh, ow}), qt(b, {f, c, kh, kw}), g, h, wd);
        else y = conv2d_backward_weights_fp8(qt(a, {n, c, h, wd}), qt(b, {n, f, oh, ow}), kh, kw, g);
        std::memcpy(out, y.data.data(), sizeof(float) * y.data.size());
        return 0;
    } catch (const std::invalid_argument&) {
        return 22;
    }
}

// LossScaler (loss_scaling.hpp:26-68) behind an opaque handle.
void* ref_scaler_new(int kind, double scale, double backoff, double growth,
                     int64_t interval, int nsched, const int64_t* it, const double* sc) {
    try {
        LossScaler::Options o;
        o.kind = kind == 0 ? LossScaler::Kind::Constant : LossScaler::Kind::DynamicBackoff;
        o.scale = scale;
        o.backoff_factor = backoff;
        o.growth_factor = growth;
        o.growth_interval = interval;
        for (int i = 0; i < nsched; ++i) o.min_threshold_schedule.push_back({it[i], sc[i]});
        return new LossScaler(o);
    } catch (const std::invalid_argument&) {
        return nullptr;
    }
}
void ref_scaler_free(void* s) { delete static_cast<LossScaler*>(s); }
double ref_scaler_scale(void* s) { return static_cast<LossScaler*>(s)->scale(); }
double ref_scaler_min_threshold(void* s, int64_t it) {
    return static_cast<LossScaler*>(s)->min_threshold(it);
}
int ref_scaler_step(void* s, int finite, int64_t it, double* scale_after) {
    const ScaleEvent ev = static_cast<LossScaler*>(s)->step(finite != 0, it);
    *scale_after = ev.scale_after;
    return static_cast<int>(ev.action);
}
void ref_scaler_unscale(void* s, float* g, int64_t n) {
    Tensor t({n}, std::vector<float>(g, g + n));
    static_cast<LossScaler*>(s)->unscale_gradients_inplace(t);
    std::memcpy(g, t.data.data(), sizeof(float) * n);
}

// update_tensor (nn.cpp:417-432) arithmetic + the reference's encode for the
// FP16 master (RNE). master_mode 1 applies the BASELINE SR extension through
// the reference's own quantize(Tensor(w32), kFp16, {Stochastic, seed}).
int ref_update(uint16_t* master, float* momentum, const float* g, int64_t n,
               float scale, float lr, float mu, float two_lambda, int master_mode,
               uint64_t seed, float* w32_out) {
    std::vector<float> w32(n);
    for (int64_t j = 0; j < n; ++j) {
        const float value = static_cast<float>(decode(master[j], kFp16));
        float gv = g[j] / scale;
        if (two_lambda != 0.0f) gv += two_lambda * value;
        momentum[j] = mu * momentum[j] + gv;
        w32[j] = value - lr * momentum[j];
        if (w32_out) w32_out[j] = w32[j];
    }
    if (master_mode == 0) {
        for (int64_t j = 0; j < n; ++j)
            master[j] = static_cast<uint16_t>(
                encode(w32[j], kFp16, RoundingMode::NearestEven).code);
        return 0;
    }
    try {
        QuantConfig cfg;
        cfg.mode = RoundingMode::Stochastic;
        cfg.seed = seed;
        const QuantizedTensor q = quantize(Tensor({n}, w32), kFp16, cfg);
        std::memcpy(master, q.codes.data(), sizeof(uint16_t) * n);
        return 0;
    } catch (const std::invalid_argument&) {
        return 22;
    }
}

// Rand{seed}.normal() stream (rand.hpp:13-37): continues across calls via
// the state block {seed, n, have_spare, spare}.
void ref_rand_fill_normal(uint64_t* st_seed_n, int* have_spare, double* spare,
                          float* out, int64_t count, double stddev) {
    Rand r{st_seed_n[0]};
    r.n = st_seed_n[1];
    r.have_spare = *have_spare != 0;
    r.spare = *spare;
    for (int64_t i = 0; i < count; ++i) out[i] = static_cast<float>(r.normal() * stddev);
    st_seed_n[1] = r.n;
    *have_spare = r.have_spare;
    *spare = r.spare;
}

// FP8T container (tensor_io.cpp): save/load through the reference's own code.
// Errors come back as 5 with the IoError message copied into msg (256 bytes).
static int io_err(const std::exception& e, char* msg) {
    std::strncpy(msg, e.what(), 255);
    msg[255] = 0;
    return 5;
}
int ref_fp8t_save_f32(const char* path, int rank, const int64_t* dims, const float* data, char* msg) {
    try {
        Tensor t(std::vector<int64_t>(dims, dims + rank));
        std::memcpy(t.data.data(), data, sizeof(float) * t.data.size());
        save_tensor(path, t);
        return 0;
    } catch (const std::exception& e) {
        return io_err(e, msg);
    }
}
int ref_fp8t_save_codes(const char* path, int fmt, int mode, int rank, const int64_t* dims,
                        const uint16_t* codes, char* msg) {
    try {
        QuantizedTensor q;
        q.shape.assign(dims, dims + rank);
        q.fmt = fmt == 0 ? kFp8 : kFp16;
        q.mode_used = mode == 2 ? RoundingMode::Stochastic
                    : mode == 3 ? RoundingMode::TruncateTowardZero
                                : RoundingMode::NearestEven;
        q.codes.assign(codes, codes + shape_numel(q.shape));
        save_tensor(path, q);
        return 0;
    } catch (const std::exception& e) {
        return io_err(e, msg);
    }
}
// returns 0 and fills out (capacity elements) / shape
int ref_fp8t_load_f32(const char* path, float* out, int64_t cap, int* rank, int64_t* dims, char* msg) {
    try {
        const Tensor t = load_tensor_fp32(path);
        if ((int64_t)t.data.size() > cap) return 7;
        std::memcpy(out, t.data.data(), sizeof(float) * t.data.size());
        *rank = (int)t.shape.size();
        for (size_t i = 0; i < t.shape.size() && i < 16; ++i) dims[i] = t.shape[i];
        return 0;
    } catch (const std::exception& e) {
        return io_err(e, msg);
    }
}
int ref_fp8t_load_codes(const char* path, uint16_t* out, int64_t cap, int* fmt, int* mode, int* rank,
                        int64_t* dims, char* msg) {
    try {
        const QuantizedTensor q = load_tensor_codes(path);
        if ((int64_t)q.codes.size() > cap) return 7;
        std::memcpy(out, q.codes.data(), sizeof(uint16_t) * q.codes.size());
        *fmt = q.fmt == kFp8 ? 0 : 1;
        *mode = q.mode_used == RoundingMode::Stochastic ? 2
              : q.mode_used == RoundingMode::TruncateTowardZero ? 3 : 1;
        *rank = (int)q.shape.size();
        for (size_t i = 0; i < q.shape.size() && i < 16; ++i) dims[i] = q.shape[i];
        return 0;
    } catch (const std::exception& e) {
        return io_err(e, msg);
    }
}

}  // extern "C"
