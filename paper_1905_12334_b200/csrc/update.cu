// update.cu -- fused SGD-momentum update into FP16 masters, device loss scaler.
//
// update_tensor (nn.cpp:417-432) driven by Network::apply_update
// (nn.cpp:436-458), in one HBM pass per parameter tensor:
//   g = decode(grad) ; gv = g / scale ; gv += 2λ·value ; m = μ·m + gv ;
//   w32 = value − lr·m ; master = encode_FP16(w32, RNE | SR) [; W8 = Q_RNE(master)]
// with value == decode(master) (test_nn.cpp:162-178, so no FP32 copy is kept)
// and IEEE binary32 ops in exactly that order: __fdiv_rn/__fmul_rn/__fadd_rn
// forbid FMA contraction (the reference objects contain no FMA).
#include "common.cuh"
#include "kernels.cuh"

namespace fp8b {

struct UpdArgs {
    float lr, mu, two_lambda, scale;
    const fp8b_loss_scaler_t* scaler;
    const int64_t* skip;
    uint64_t seed;
    int64_t elem_offset;
    const uint32_t* rbits;
    int64_t* mcnt;
    uint8_t* w8;
    int w_sat;
    int64_t* wcnt;
};

__device__ __forceinline__ bool upd_skipped(const UpdArgs& a) {
    return a.skip && (a.skip[0] + a.skip[2]) != 0;
}
__device__ __forceinline__ float upd_scale(const UpdArgs& a) {
    return a.scaler ? __double2float_rn(a.scaler->scale) : a.scale;
}

// nn.cpp:419-424
__device__ __forceinline__ float sgd_w32(float g, float value, float& m, float scale,
                                         const UpdArgs& a) {
    float gv = __fdiv_rn(g, scale);
    if (a.two_lambda != 0.0f) gv = __fadd_rn(gv, __fmul_rn(a.two_lambda, value));
    m = __fadd_rn(__fmul_rn(a.mu, m), gv);
    return __fsub_rn(value, __fmul_rn(a.lr, m));
}

template <int GFMT>
__device__ __forceinline__ void load_grad4(const void* grad, int64_t g, float out[4]) {
    if (GFMT == FP8B_E5M2) {
        const uint32_t w = __ldcs(reinterpret_cast<const uint32_t*>(grad) + g);
        out[0] = dec_e5m2(w); out[1] = dec_e5m2(w >> 8); out[2] = dec_e5m2(w >> 16); out[3] = dec_e5m2(w >> 24);
    } else if (GFMT == FP8B_FP16) {
        const uint2 w = __ldcs(reinterpret_cast<const uint2*>(grad) + g);
        out[0] = dec_f16(w.x); out[1] = dec_f16(w.x >> 16); out[2] = dec_f16(w.y); out[3] = dec_f16(w.y >> 16);
    } else {
        const float4 v = __ldcs(reinterpret_cast<const float4*>(grad) + g);
        out[0] = v.x; out[1] = v.y; out[2] = v.z; out[3] = v.w;
    }
}
template <int GFMT>
__device__ __forceinline__ float load_grad1(const void* grad, int64_t i) {
    if (GFMT == FP8B_E5M2) return dec_e5m2(reinterpret_cast<const uint8_t*>(grad)[i]);
    if (GFMT == FP8B_FP16) return dec_f16(reinterpret_cast<const uint16_t*>(grad)[i]);
    return reinterpret_cast<const float*>(grad)[i];
}

// Fused E5M2 copy of the new weight (RNE) + counters.
__device__ __forceinline__ uint32_t w8_code(uint32_t master, bool sat, uint32_t& cb, uint32_t& cn,
                                            uint32_t& cu) {
    const float v = dec_f16(master);
    const uint32_t hw = cvt_e5m2x2(v, 0.0f) & 0xFFu;
    return fix_rne<2>(hw, __float_as_uint(v), sat, cb, cn, cu);
}

// Position-independent master rounding: MODE 0 RNE, 1 SR counter, 2 SR supplied.
template <int GFMT, int MODE, int NT>
__global__ void __launch_bounds__(NT) sgd_elem_kernel(const void* __restrict__ grad,
                                                      uint16_t* __restrict__ master,
                                                      float* __restrict__ mom, int64_t n,
                                                      UpdArgs a, int aligned) {
    if (upd_skipped(a)) return;
    const float scale = upd_scale(a);
    uint32_t mb = 0, mn = 0, mu_ = 0, wb = 0, wn = 0, wu = 0;
    const int64_t ngroups = aligned ? (n >> 2) : 0;
    for (int64_t g = (int64_t)blockIdx.x * NT + threadIdx.x; g < ngroups;
         g += (int64_t)gridDim.x * NT) {
        float gr[4];
        load_grad4<GFMT>(grad, g, gr);
        const uint2 mw = reinterpret_cast<const uint2*>(master)[g];
        float4 mv = reinterpret_cast<const float4*>(mom)[g];
        uint32_t r32[4] = {0, 0, 0, 0};
        if (MODE == 2) {
            const uint4 r = __ldcs(reinterpret_cast<const uint4*>(a.rbits) + g);
            r32[0] = r.x; r32[1] = r.y; r32[2] = r.z; r32[3] = r.w;
        }
        const uint32_t mc[4] = {mw.x & 0xFFFFu, mw.x >> 16, mw.y & 0xFFFFu, mw.y >> 16};
        float m[4] = {mv.x, mv.y, mv.z, mv.w};
        uint32_t out[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const float w32 = sgd_w32(gr[k], dec_f16(mc[k]), m[k], scale, a);
            const uint32_t u = __float_as_uint(w32);
            uint32_t r16 = 0;
            if (MODE == 1) r16 = counter_r16(a.seed, (uint64_t)(a.elem_offset + g * 4 + k));
            if (MODE == 2) r16 = r32[k] >> 16;
            int o, un, na;
            out[k] = encode_int<10>(u, MODE == 0 ? FP8B_RNE : FP8B_SR, r16, false, o, un, na);
            mb += o; mn += na; mu_ += un;
        }
        reinterpret_cast<uint2*>(master)[g] = make_uint2(out[0] | (out[1] << 16), out[2] | (out[3] << 16));
        reinterpret_cast<float4*>(mom)[g] = make_float4(m[0], m[1], m[2], m[3]);
        if (a.w8) {
            uint32_t w = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k) w |= w8_code(out[k], a.w_sat != 0, wb, wn, wu) << (8 * k);
            reinterpret_cast<uint32_t*>(a.w8)[g] = w;
        }
    }
    for (int64_t i = (ngroups << 2) + (int64_t)blockIdx.x * NT + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * NT) {
        float m = mom[i];
        const float w32 = sgd_w32(load_grad1<GFMT>(grad, i), dec_f16(master[i]), m, scale, a);
        uint32_t r16 = 0;
        if (MODE == 1) r16 = counter_r16(a.seed, (uint64_t)(a.elem_offset + i));
        if (MODE == 2) r16 = a.rbits[i] >> 16;
        int o, un, na;
        const uint32_t c = encode_int<10>(__float_as_uint(w32), MODE == 0 ? FP8B_RNE : FP8B_SR, r16,
                                          false, o, un, na);
        mb += o; mn += na; mu_ += un;
        master[i] = (uint16_t)c;
        mom[i] = m;
        if (a.w8) a.w8[i] = (uint8_t)w8_code(c, a.w_sat != 0, wb, wn, wu);
    }
    if (a.mcnt) flush_counters<NT>(mb, mu_, mn, a.mcnt);
    if (a.wcnt) flush_counters<NT>(wb - wn, wu, wn, a.wcnt);
}

// Reference-stream SR master: quantize(Tensor(w32), kFp16, {Stochastic, seed})
// semantics (SURVEY 8c iii) -- the block scan of quantize.cu, fed by w32.
template <int GFMT>
__global__ void __launch_bounds__(256) sgd_lfsr_kernel(const void* __restrict__ grad,
                                                       uint16_t* __restrict__ master,
                                                       float* __restrict__ mom, int64_t n,
                                                       UpdArgs a, int64_t block_offset,
                                                       LfsrTables tabs) {
    if (upd_skipped(a)) return;
    __shared__ uint32_t smem_w[2][8];
    const float scale = upd_scale(a);
    uint32_t mb = 0, mn = 0, mu_ = 0, wb = 0, wn = 0, wu = 0;
    const int64_t nblocks = (n + kBlock - 1) / kBlock;
    int parity = 0;
    for (int64_t b = blockIdx.x; b < nblocks; b += gridDim.x, parity ^= 1) {
        const int64_t base = b * kBlock;
        uint32_t code[4][4], r16[4][4], mask[4];
        float mnew[4][4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            mask[r] = 0;
            const int64_t i0 = base + 1024 * r + 4 * threadIdx.x;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int64_t i = i0 + k;
                float w32 = 0.0f;
                mnew[r][k] = 0.0f;
                if (i < n) {
                    float m = mom[i];
                    w32 = sgd_w32(load_grad1<GFMT>(grad, i), dec_f16(master[i]), m, scale, a);
                    mnew[r][k] = m;
                }
                const uint32_t u = __float_as_uint(w32);
                const Split s = split_bits<10>(u, false);
                code[r][k] = s.code;
                r16[r][k] = s.r16;
                if (i < n) {
                    if (s.inexact) mask[r] |= 1u << k;
                    const uint32_t aa = u & 0x7FFFFFFFu;
                    mb += aa > Fmt<10>::maxbits;
                    mn += aa > 0x7F800000u;
                }
            }
        }
        const uint32_t s0 = lfsr_split(a.seed, (uint64_t)(block_offset + b));
        const uint32_t p0 = __ldg(tabs.pos + s0);
        uint32_t pre[4];
        BlockScan<10>::run(mask, pre, smem_w[parity]);
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            uint32_t j = p0 + pre[r];
            const int64_t i0 = base + 1024 * r + 4 * threadIdx.x;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if (mask[r] & (1u << k)) {
                    const uint32_t sample = __ldg(tabs.tabx + j);
                    ++j;
                    code[r][k] += (r16[r][k] + sample) >= 65536u;
                    mu_ += (code[r][k] & 0x7FFFu) == 0u;
                }
                const int64_t i = i0 + k;
                if (i < n) {
                    master[i] = (uint16_t)code[r][k];
                    mom[i] = mnew[r][k];
                    if (a.w8) a.w8[i] = (uint8_t)w8_code(code[r][k], a.w_sat != 0, wb, wn, wu);
                }
            }
        }
    }
    if (a.mcnt) flush_counters<256>(mb - mn, mu_, mn, a.mcnt);
    if (a.wcnt) flush_counters<256>(wb - wn, wu, wn, a.wcnt);
}

// ---------------------------------------------------------- loss scaler
// loss_scaling.cpp:40-47
__device__ double scaler_min_threshold(const fp8b_loss_scaler_t& s, int64_t it) {
    double thr = 1.0;
    for (int i = 0; i < s.n_schedule; ++i) {
        if (s.sched_iter[i] > it) break;
        thr = s.sched_scale[i];
    }
    return thr;
}

// loss_scaling.cpp:49-83
__global__ void scaler_step_kernel(fp8b_loss_scaler_t* s, const int64_t* counters, int finite_in,
                                   int64_t iteration) {
    const bool finite = counters ? (counters[0] + counters[2]) == 0 : finite_in != 0;
    int action = FP8B_ACT_NONE;
    if (s->kind == FP8B_SCALER_DYNAMIC_BACKOFF) {
        const double thr = scaler_min_threshold(*s, iteration);
        if (!finite) {
            const double cand = s->scale * s->backoff_factor;
            if (cand < thr) { s->scale = thr; action = FP8B_ACT_CLAMPED_TO_MIN; }
            else { s->scale = cand; action = FP8B_ACT_BACKOFF; }
            s->steps_since_overflow = 0;
        } else {
            ++s->steps_since_overflow;
            if (s->steps_since_overflow >= s->growth_interval) {
                s->scale *= s->growth_factor;
                s->steps_since_overflow = 0;
                action = FP8B_ACT_GROWTH;
            }
            if (s->scale < thr) { s->scale = thr; action = FP8B_ACT_CLAMPED_TO_MIN; }
        }
    }
    s->last_iteration = iteration;
    s->last_action = action;
    s->last_grads_finite = finite ? 1 : 0;
    s->last_scale_after = s->scale;
}

// loss_scaling.cpp:89-92
__global__ void unscale_kernel(float* g, int64_t n, const fp8b_loss_scaler_t* s) {
    const float sc = __double2float_rn(s->scale);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        g[i] = __fdiv_rn(g[i], sc);
}

// ---------------------------------------------------------------- launchers
static int sm_count() {
    static int num_sms = 0;
    if (!num_sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
    }
    return num_sms;
}

template <int GFMT>
static void launch_sgd_fmt(const void* grad, uint16_t* master, float* mom, int64_t n,
                           const fp8b_sgd_args_t& args, cudaStream_t st, const LfsrTables& tabs) {
    UpdArgs a;
    a.lr = args.lr; a.mu = args.mu; a.two_lambda = args.two_lambda; a.scale = args.scale;
    a.scaler = args.scaler; a.skip = args.skip_counters; a.seed = args.seed;
    a.elem_offset = args.block_offset * kBlock; a.rbits = args.rbits;
    a.mcnt = args.master_counters; a.w8 = args.w_e5m2; a.w_sat = args.w_saturate;
    a.wcnt = args.w_counters;
    constexpr int NT = 256;
    if (args.master_mode == FP8B_SR && args.bits == FP8B_BITS_LFSR) {
        const int64_t nb = (n + kBlock - 1) / kBlock;
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sgd_lfsr_kernel<GFMT>, 256, 0);
        int64_t g = (int64_t)sm_count() * (per_sm > 0 ? per_sm : 1);
        if (nb < g) g = nb < 1 ? 1 : nb;
        sgd_lfsr_kernel<GFMT><<<(int)g, 256, 0, st>>>(grad, master, mom, n, a, args.block_offset, tabs);
        return;
    }
    const bool aligned = ((uintptr_t)grad % 16 == 0) && ((uintptr_t)master % 8 == 0) &&
                         ((uintptr_t)mom % 16 == 0) && (a.w8 == nullptr || (uintptr_t)a.w8 % 4 == 0) &&
                         (a.rbits == nullptr || (uintptr_t)a.rbits % 16 == 0);
    int64_t g = (int64_t)sm_count() * 8;
    const int64_t need = ((aligned ? n / 4 : n) + NT - 1) / NT;
    if (need < g) g = need < 1 ? 1 : need;
    if (args.master_mode == FP8B_RNE)
        sgd_elem_kernel<GFMT, 0, NT><<<(int)g, NT, 0, st>>>(grad, master, mom, n, a, aligned ? 1 : 0);
    else if (args.bits == FP8B_BITS_COUNTER)
        sgd_elem_kernel<GFMT, 1, NT><<<(int)g, NT, 0, st>>>(grad, master, mom, n, a, aligned ? 1 : 0);
    else
        sgd_elem_kernel<GFMT, 2, NT><<<(int)g, NT, 0, st>>>(grad, master, mom, n, a, aligned ? 1 : 0);
}

void launch_sgd(const void* grad, int grad_fmt, uint16_t* master, float* mom, int64_t n,
                const fp8b_sgd_args_t& args, cudaStream_t st, const LfsrTables& tabs) {
    if (grad_fmt == FP8B_E5M2) launch_sgd_fmt<FP8B_E5M2>(grad, master, mom, n, args, st, tabs);
    else if (grad_fmt == FP8B_FP16) launch_sgd_fmt<FP8B_FP16>(grad, master, mom, n, args, st, tabs);
    else launch_sgd_fmt<FP8B_F32>(grad, master, mom, n, args, st, tabs);
}

void launch_scaler_step(fp8b_loss_scaler_t* s, const int64_t* counters, int finite, int64_t it,
                        cudaStream_t st) {
    scaler_step_kernel<<<1, 1, 0, st>>>(s, counters, finite, it);
}

void launch_unscale(float* g, int64_t n, const fp8b_loss_scaler_t* s, cudaStream_t st) {
    int64_t blocks = (n + 255) / 256;
    if (blocks > (int64_t)sm_count() * 8) blocks = (int64_t)sm_count() * 8;
    if (blocks < 1) blocks = 1;
    unscale_kernel<<<(int)blocks, 256, 0, st>>>(g, n, s);
}

}  // namespace fp8b
