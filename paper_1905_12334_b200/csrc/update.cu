// update.cu -- fused SGD-momentum update into FP16 masters, device loss scaler.
//
// update_tensor (nn.cpp:417-432) driven by Network::apply_update
// (nn.cpp:436-458), in one HBM pass per parameter tensor:
//   g = decode(grad) ; gv = g / scale ; gv += 2λ·value ; m = μ·m + gv ;
//   w32 = value − lr·m ; master = encode_FP16(w32, RNE | SR) [; W8 = Q_RNE(master)]
// with value == decode(master) (test_nn.cpp:162-178, so no FP32 copy is kept)
// and IEEE binary32 ops in exactly that order: __fdiv_rn/__fmul_rn/__fadd_rn
// forbid FMA contraction (the reference objects contain no FMA).
#include <cstdlib>

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
    int step_scaler;     // run the scaler step from the kernel's last CTA
    int64_t iteration;
    const int64_t* skip2;  // optional second counter set of the gate
    int64_t* gate_out;     // merged gate, stored by the last CTA (with step_scaler)
};

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
__device__ void scaler_step_dev(fp8b_loss_scaler_t* s, const int64_t* counters, int finite_in,
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

__global__ void scaler_step_kernel(fp8b_loss_scaler_t* s, const int64_t* counters, int finite_in,
                                   int64_t iteration) {
    scaler_step_dev(s, counters, finite_in, iteration);
}

// Fused LossScaler::step (fp8b_sgd_args_t.step_scaler): every CTA reads the scale
// before it gets here, so the CTA that draws the last ticket may advance it.
__device__ __forceinline__ void upd_tail(const UpdArgs& a) {
    if (!a.step_scaler) return;
    __syncthreads();
    if (threadIdx.x == 0) {
        fp8b_loss_scaler_t* sc = const_cast<fp8b_loss_scaler_t*>(a.scaler);
        __threadfence();
        if (atomicAdd(&sc->step_ticket, 1u) == gridDim.x - 1) {
            sc->step_ticket = 0;
            if (a.skip && a.skip2) {  // merged gate (nn.cpp:401-411)
                int64_t g[3];
                for (int i = 0; i < 3; ++i) g[i] = a.skip[i] + a.skip2[i];
                if (a.gate_out)
                    for (int i = 0; i < 3; ++i) a.gate_out[i] = g[i];
                scaler_step_dev(sc, nullptr, (g[0] + g[2]) == 0, a.iteration);
            } else {
                if (a.skip && a.gate_out)
                    for (int i = 0; i < 3; ++i) a.gate_out[i] = a.skip[i];
                scaler_step_dev(sc, a.skip, 1, a.iteration);
            }
            if (a.step_scaler == 2) {  // hand the gate's inputs back cleared (no zeroing launch next step)
                for (int i = 0; i < 3; ++i) {
                    if (a.skip) const_cast<int64_t*>(a.skip)[i] = 0;
                    if (a.skip2) const_cast<int64_t*>(a.skip2)[i] = 0;
                }
            }
        }
    }
}

__device__ __forceinline__ bool upd_skipped(const UpdArgs& a) {
    int64_t bad = a.skip ? a.skip[0] + a.skip[2] : 0;
    if (a.skip2) bad += a.skip2[0] + a.skip2[2];
    return bad != 0;
}
__device__ __forceinline__ float upd_scale(const UpdArgs& a) {
    return a.scaler ? __double2float_rn(a.scaler->scale) : a.scale;
}

// g / scale. For a power-of-two scale (the loss scaler's factors and floors
// keep it one, loss_scaling.hpp:22-24) g * (1/scale) rounds the same exact real
// value and is bitwise identical to the IEEE division; otherwise true division.
struct Unscale {
    float scale, inv;
    bool pow2;
    __device__ __forceinline__ explicit Unscale(float s) : scale(s) {
        const uint32_t b = __float_as_uint(s);
        pow2 = (b & 0x807FFFFFu) == 0u && (b >> 23) >= 1u && (b >> 23) <= 254u;
        inv = pow2 ? __uint_as_float((254u - (b >> 23)) << 23) : 0.0f;
        if (pow2 && (b >> 23) == 254u) inv = __uint_as_float(0x00400000u);  // 2^-127
    }
    __device__ __forceinline__ float operator()(float g) const {
        return pow2 ? __fmul_rn(g, inv) : __fdiv_rn(g, scale);
    }
};

// nn.cpp:419-424 (no FMA contraction)
__device__ __forceinline__ float sgd_w32(float g, float value, float& m, const Unscale& us,
                                         const UpdArgs& a) {
    float gv = us(g);
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
template <int GFMT>
constexpr int grad_bytes() { return GFMT == FP8B_E5M2 ? 1 : (GFMT == FP8B_FP16 ? 2 : 4); }

// Fused E5M2 copy of the new weight: Q_RNE(decode(master)) (nn.cpp:192-193).
__device__ __forceinline__ uint32_t w8_pack4(const uint32_t (&mc)[4], bool sat, uint32_t& cb,
                                             uint32_t& cn, uint32_t& cu) {
    uint32_t w = 0;
#pragma unroll
    for (int k = 0; k < 4; k += 2) {
        const float v0 = dec_f16(mc[k]), v1 = dec_f16(mc[k + 1]);
        const uint32_t pr = cvt_e5m2x2(v0, v1);
        w |= fix_rne<2>(pr & 0xFFu, __float_as_uint(v0), sat, cb, cn, cu) << (8 * k);
        w |= fix_rne<2>(pr >> 8, __float_as_uint(v1), sat, cb, cn, cu) << (8 * k + 8);
    }
    return w;
}
__device__ __forceinline__ uint32_t w8_code1(uint32_t mc, bool sat, uint32_t& cb, uint32_t& cn,
                                             uint32_t& cu) {
    const float v = dec_f16(mc);
    return fix_rne<2>(cvt_e5m2x2(v, 0.0f) & 0xFFu, __float_as_uint(v), sat, cb, cn, cu);
}

// Master rounding of four w32 values. MODE 0 RNE (hardware cvt + reference
// fixups), 1 SR counter bits, 2 SR supplied bits.
template <int MODE>
__device__ __forceinline__ void master4(const float (&w)[4], uint64_t word, const uint32_t (&rb)[4],
                                        uint32_t (&out)[4], uint32_t& mb, uint32_t& mn,
                                        uint32_t& mu) {
    if (MODE == 0) {
        const uint32_t h01 = cvt_f16x2(w[0], w[1]), h23 = cvt_f16x2(w[2], w[3]);
        const uint32_t h[4] = {h01 & 0xFFFFu, h01 >> 16, h23 & 0xFFFFu, h23 >> 16};
#pragma unroll
        for (int k = 0; k < 4; ++k) out[k] = fix_rne<10>(h[k], __float_as_uint(w[k]), false, mb, mn, mu);
    } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t r16 = MODE == 1 ? (uint32_t)(word >> (16 * k)) & 0xFFFFu : rb[k];
            out[k] = sr_encode<10>(__float_as_uint(w[k]), r16, false, mb, mn, mu);
        }
    }
}

// Position-independent master rounding, 4*G parameters per thread per
// iteration (all G groups' loads issued before any is used); MINB resident CTAs
// per SM bound the registers (occupancy = bytes in flight for this HBM-bound pass).
template <int GFMT, int MODE, int NT, bool CNT, int G = 2, int MINB = 1>
__global__ void __launch_bounds__(NT, MINB) sgd_elem_kernel(const void* __restrict__ grad,
                                                            uint16_t* __restrict__ master,
                                                            float* __restrict__ mom, int64_t n,
                                                            UpdArgs a, int aligned) {
    if (upd_skipped(a)) { upd_tail(a); return; }
    const Unscale us(upd_scale(a));
    const bool wsat = a.w_sat != 0;
    uint32_t mb = 0, mn = 0, mu_ = 0, wb = 0, wn = 0, wu = 0;
    const int64_t ngroups = aligned ? (n >> 2) : 0;
    const int64_t stride = (int64_t)gridDim.x * NT * G;
    for (int64_t g0 = (int64_t)blockIdx.x * NT * G + threadIdx.x; g0 < ngroups; g0 += stride) {
        float gr[G][4];
        uint2 mw[G];
        float4 mv[G];
        uint32_t rb[G][4] = {};
        bool ok[G];
#pragma unroll
        for (int h = 0; h < G; ++h) {
            const int64_t g = g0 + (int64_t)h * NT;
            ok[h] = g < ngroups;
            if (!ok[h]) continue;
            load_grad4<GFMT>(grad, g, gr[h]);
            mw[h] = reinterpret_cast<const uint2*>(master)[g];
            mv[h] = reinterpret_cast<const float4*>(mom)[g];
            if (MODE == 2) {
                const uint4 r = __ldcs(reinterpret_cast<const uint4*>(a.rbits) + g);
                rb[h][0] = r.x >> 16; rb[h][1] = r.y >> 16; rb[h][2] = r.z >> 16; rb[h][3] = r.w >> 16;
            }
        }
#pragma unroll
        for (int h = 0; h < G; ++h) {
            if (!ok[h]) continue;
            const int64_t g = g0 + (int64_t)h * NT;
            const uint32_t mc[4] = {mw[h].x & 0xFFFFu, mw[h].x >> 16, mw[h].y & 0xFFFFu, mw[h].y >> 16};
            float m[4] = {mv[h].x, mv[h].y, mv[h].z, mv[h].w};
            float w[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) w[k] = sgd_w32(gr[h][k], dec_f16(mc[k]), m[k], us, a);
            const uint64_t word = MODE == 1 ? counter_word(a.seed, (uint64_t)((a.elem_offset >> 2) + g)) : 0ull;
            uint32_t out[4];
            master4<MODE>(w, word, rb[h], out, mb, mn, mu_);
            reinterpret_cast<uint2*>(master)[g] = make_uint2(out[0] | (out[1] << 16), out[2] | (out[3] << 16));
            reinterpret_cast<float4*>(mom)[g] = make_float4(m[0], m[1], m[2], m[3]);
            if (a.w8) reinterpret_cast<uint32_t*>(a.w8)[g] = w8_pack4(out, wsat, wb, wn, wu);
        }
    }
    for (int64_t i = (ngroups << 2) + (int64_t)blockIdx.x * NT + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * NT) {
        float m = mom[i];
        const float w32 = sgd_w32(load_grad1<GFMT>(grad, i), dec_f16(master[i]), m, us, a);
        uint32_t r16 = 0;
        if (MODE == 1) r16 = counter_r16(a.seed, (uint64_t)(a.elem_offset + i));
        if (MODE == 2) r16 = a.rbits[i] >> 16;
        int o, un, na;
        const uint32_t c = encode_int<10>(__float_as_uint(w32), MODE == 0 ? FP8B_RNE : FP8B_SR, r16,
                                          false, o, un, na);
        mb += o + na; mn += na; mu_ += un;
        master[i] = (uint16_t)c;
        mom[i] = m;
        if (a.w8) a.w8[i] = (uint8_t)w8_code1(c, wsat, wb, wn, wu);
    }
    // counters are dead code (and compiled out) unless the caller asked for them
    if (CNT && a.mcnt) flush_counters<NT>(mb - mn, mu_, mn, a.mcnt);
    if (CNT && a.wcnt) flush_counters<NT>(wb - wn, wu, wn, a.wcnt);
    upd_tail(a);
}

// Reference-stream SR master: quantize(Tensor(w32), kFp16, {Stochastic, seed})
// semantics (SURVEY 8c iii): block b of 4096 parameters rounds with
// LfsrStream::split(seed, block_offset + b), one sample per inexact w32.
// Warp-per-block kernel over full blocks: each warp owns whole 4096-parameter
// blocks and walks them in 16 chunks of 256 (8 per lane, coalesced, prefetched
// one chunk ahead), so the master SR stream ranks need only a warp shuffle scan
// on top of a running count -- no CTA barrier. Samples come from the
// wrap-extended jump table in shared memory; exact lanes add their sample to a
// zero remainder, which never carries, so no select is needed.
// CTA size = the SM's warp count (the 139 KB table allows one CTA per SM).
// The kernel is latency-bound: A/B on one box, 512 -> 768 threads took the LFSR
// SR master 5.59 -> 6.02 TB/s (with the fused E5M2 W 5.46 -> 5.95); 640 gave
// 5.98, and 1024 (64 registers) spills and gave 5.65.
#ifndef FP8B_UPD_THREADS
#define FP8B_UPD_THREADS 768
#endif
constexpr int kWarpUpdThreads = FP8B_UPD_THREADS;
constexpr int kUpdTabBytes = ((kLfsrPeriod + kBlock) * 2 + 15) & ~15;
template <int GFMT, bool CNT, int NT = kWarpUpdThreads>
__global__ void __launch_bounds__(NT, 1)
    sgd_lfsr_warp_kernel(const void* __restrict__ grad, uint16_t* __restrict__ master,
                         float* __restrict__ mom, int64_t nfull, UpdArgs a, int64_t block_offset,
                         LfsrTables tabs) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ __align__(8) uint64_t tab_bar;
    if (upd_skipped(a)) { upd_tail(a); return; }
    const Unscale us(upd_scale(a));
    const bool wsat = a.w_sat != 0;
    uint32_t mb = 0, mn = 0, mu_ = 0, wb = 0, wn = 0, wu = 0;
    const int lane = threadIdx.x & 31;
    const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t wstride = ((int64_t)gridDim.x * blockDim.x) >> 5;
    if (threadIdx.x == 0) {
        mbar_init(&tab_bar, 1);
        mbar_fence_init();
        mbar_expect_tx(&tab_bar, kUpdTabBytes);
        for (int off = 0; off < kUpdTabBytes; off += 16384) {
            const int len = kUpdTabBytes - off < 16384 ? kUpdTabBytes - off : 16384;
            bulk_g2s(smem + off, reinterpret_cast<const uint8_t*>(tabs.tabx) + off, len, &tab_bar);
        }
    }
    __syncthreads();
    const uint32_t stab_addr = smem_addr(smem);
    uint32_t p0_next = 0;
    if (lane == 0 && wid < nfull)
        p0_next = __ldg(tabs.pos + lfsr_split(a.seed, (uint64_t)(block_offset + wid)));
    mbar_wait(&tab_bar, 0);
    // per-lane chunk loads: grad (8 codes or floats), 8 masters, 8 momenta
    struct Chunk {
        uint4 g;        // E5M2: .x,.y; FP16: all; F32: first 4 floats (second in g2)
        uint4 g2;
        uint4 m;        // 8 FP16 masters
        float4 v0, v1;  // 8 momenta
    };
    auto load = [&](int64_t e0, Chunk& ck) {
        if (GFMT == FP8B_E5M2) {
            const uint2 t = __ldcs(reinterpret_cast<const uint2*>(reinterpret_cast<const uint8_t*>(grad) + e0));
            ck.g = make_uint4(t.x, t.y, 0, 0);
        } else if (GFMT == FP8B_FP16) {
            ck.g = __ldcs(reinterpret_cast<const uint4*>(reinterpret_cast<const uint16_t*>(grad) + e0));
        } else {
            ck.g = __ldcs(reinterpret_cast<const uint4*>(reinterpret_cast<const float*>(grad) + e0));
            ck.g2 = __ldcs(reinterpret_cast<const uint4*>(reinterpret_cast<const float*>(grad) + e0) + 1);
        }
        ck.m = __ldcs(reinterpret_cast<const uint4*>(master + e0));
        ck.v0 = __ldcs(reinterpret_cast<const float4*>(mom + e0));
        ck.v1 = __ldcs(reinterpret_cast<const float4*>(mom + e0) + 1);
    };
    for (int64_t b = wid; b < nfull; b += wstride) {
        const uint32_t p0 = __shfl_sync(0xFFFFFFFFu, p0_next, 0);
        if (lane == 0 && b + wstride < nfull)
            p0_next = __ldg(tabs.pos + lfsr_split(a.seed, (uint64_t)(block_offset + b + wstride)));
        Chunk nx;
        load(b * kBlock + 8 * lane, nx);
        uint32_t run = stab_addr + 2u * p0;
#pragma unroll 1
        for (int c = 0; c < kBlock / 256; ++c) {
            const int64_t e0 = b * kBlock + 256 * c + 8 * lane;
            const Chunk ck = nx;
            if (c + 1 < kBlock / 256) load(e0 + 256, nx);
            float gr[8];
            if (GFMT == FP8B_E5M2) {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    gr[k] = dec_e5m2(ck.g.x >> (8 * k));
                    gr[4 + k] = dec_e5m2(ck.g.y >> (8 * k));
                }
            } else if (GFMT == FP8B_FP16) {
                const uint32_t gw[4] = {ck.g.x, ck.g.y, ck.g.z, ck.g.w};
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    gr[2 * k] = dec_f16(gw[k]);
                    gr[2 * k + 1] = dec_f16(gw[k] >> 16);
                }
            } else {
                const uint32_t gw[8] = {ck.g.x, ck.g.y, ck.g.z, ck.g.w, ck.g2.x, ck.g2.y, ck.g2.z, ck.g2.w};
#pragma unroll
                for (int k = 0; k < 8; ++k) gr[k] = __uint_as_float(gw[k]);
            }
            const uint32_t mw[4] = {ck.m.x, ck.m.y, ck.m.z, ck.m.w};
            float m[8] = {ck.v0.x, ck.v0.y, ck.v0.z, ck.v0.w, ck.v1.x, ck.v1.y, ck.v1.z, ck.v1.w};
            float w[8];
            uint32_t inc[8], n = 0;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const uint32_t mc = (mw[k >> 1] >> (16 * (k & 1))) & 0xFFFFu;
                w[k] = sgd_w32(gr[k], dec_f16(mc), m[k], us, a);
                const uint32_t aa = __float_as_uint(w[k]) & 0x7FFFFFFFu;
                inc[k] = sr_inexact<10>(aa, __uint_as_float(aa)) ? 2u : 0u;
                n += inc[k];
            }
            __stcs(reinterpret_cast<float4*>(mom + e0), make_float4(m[0], m[1], m[2], m[3]));
            __stcs(reinterpret_cast<float4*>(mom + e0) + 1, make_float4(m[4], m[5], m[6], m[7]));
            uint32_t incl = n;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t o = __shfl_up_sync(0xFFFFFFFFu, incl, d);
                if (lane >= d) incl += o;
            }
            const uint32_t total = __shfl_sync(0xFFFFFFFFu, incl, 31);
            uint32_t addr = run + incl - n;
            run += total;
            uint32_t out[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                uint32_t r16;
                asm volatile("ld.shared.u16 %0, [%1];" : "=r"(r16) : "r"(addr));
                addr += inc[k];
                out[k] = sr_encode<10>(__float_as_uint(w[k]), r16, false, mb, mn, mu_);
            }
            __stcs(reinterpret_cast<uint4*>(master + e0),
                   make_uint4(out[0] | (out[1] << 16), out[2] | (out[3] << 16), out[4] | (out[5] << 16),
                              out[6] | (out[7] << 16)));
            if (a.w8) {
                const uint32_t lo[4] = {out[0], out[1], out[2], out[3]}, hi[4] = {out[4], out[5], out[6], out[7]};
                __stcs(reinterpret_cast<uint2*>(a.w8 + e0),
                       make_uint2(w8_pack4(lo, wsat, wb, wn, wu), w8_pack4(hi, wsat, wb, wn, wu)));
            }
        }
    }
    if (CNT && a.mcnt) flush_counters<NT>(mb - mn, mu_, mn, a.mcnt);
    if (CNT && a.wcnt) flush_counters<NT>(wb - wn, wu, wn, a.wcnt);
    upd_tail(a);
}

// Tail / unaligned variant: blocks [block_begin, nblocks) with scalar accesses.
template <int GFMT>
__global__ void __launch_bounds__(256) sgd_lfsr_kernel(const void* __restrict__ grad,
                                                       uint16_t* __restrict__ master,
                                                       float* __restrict__ mom, int64_t n,
                                                       UpdArgs a, int64_t block_offset,
                                                       LfsrTables tabs, int64_t block_begin,
                                                       int vec) {
    if (upd_skipped(a)) { upd_tail(a); return; }
    __shared__ uint32_t smem_w[2][8];
    const Unscale us(upd_scale(a));
    const bool wsat = a.w_sat != 0;
    uint32_t mb = 0, mn = 0, mu_ = 0, wb = 0, wn = 0, wu = 0;
    const int64_t nblocks = (n + kBlock - 1) / kBlock;
    int parity = 0;
    for (int64_t b = block_begin + blockIdx.x; b < nblocks; b += gridDim.x, parity ^= 1) {
        const int64_t base = b * kBlock;
        float w[4][4];
        uint32_t mask[4];
        // full block, 16-byte aligned tensors: one vector access per tensor and round
        const bool vfull = vec && base + kBlock <= n;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            mask[r] = 0;
            const int64_t i0 = base + 1024 * r + 4 * threadIdx.x;
            if (vfull) {
                float gr[4];
                load_grad4<GFMT>(grad, i0 >> 2, gr);
                const uint2 mw = *reinterpret_cast<const uint2*>(master + i0);
                const float4 mv = *reinterpret_cast<const float4*>(mom + i0);
                const uint32_t mc[4] = {mw.x & 0xFFFFu, mw.x >> 16, mw.y & 0xFFFFu, mw.y >> 16};
                float m[4] = {mv.x, mv.y, mv.z, mv.w};
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    w[r][k] = sgd_w32(gr[k], dec_f16(mc[k]), m[k], us, a);
                    const uint32_t aa = __float_as_uint(w[r][k]) & 0x7FFFFFFFu;
                    if (sr_inexact<10>(aa, __uint_as_float(aa))) mask[r] |= 1u << k;
                }
                *reinterpret_cast<float4*>(mom + i0) = make_float4(m[0], m[1], m[2], m[3]);
                continue;
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int64_t i = i0 + k;
                w[r][k] = 0.0f;
                if (i < n) {
                    float m = mom[i];
                    w[r][k] = sgd_w32(load_grad1<GFMT>(grad, i), dec_f16(master[i]), m, us, a);
                    mom[i] = m;
                    const uint32_t aa = __float_as_uint(w[r][k]) & 0x7FFFFFFFu;
                    if (sr_inexact<10>(aa, __uint_as_float(aa))) mask[r] |= 1u << k;
                }
            }
        }
        const uint32_t p0 = __ldg(tabs.pos + lfsr_split(a.seed, (uint64_t)(block_offset + b)));
        uint32_t pre[4];
        BlockScan<10>::run(mask, pre, smem_w[parity]);
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            uint32_t j = p0 + pre[r];
            const int64_t i0 = base + 1024 * r + 4 * threadIdx.x;
            if (vfull) {
                uint32_t c[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const uint32_t take = (mask[r] >> k) & 1u;
                    const uint32_t r16 = take ? (uint32_t)__ldg(tabs.tabx + j) : 0u;
                    j += take;
                    c[k] = sr_encode<10>(__float_as_uint(w[r][k]), r16, false, mb, mn, mu_);
                }
                *reinterpret_cast<uint2*>(master + i0) = make_uint2(c[0] | (c[1] << 16), c[2] | (c[3] << 16));
                if (a.w8) *reinterpret_cast<uint32_t*>(a.w8 + i0) = w8_pack4(c, wsat, wb, wn, wu);
                continue;
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint32_t take = (mask[r] >> k) & 1u;
                const uint32_t r16 = take ? (uint32_t)__ldg(tabs.tabx + j) : 0u;
                j += take;
                const int64_t i = i0 + k;
                if (i < n) {
                    const uint32_t c = sr_encode<10>(__float_as_uint(w[r][k]), r16, false, mb, mn, mu_);
                    master[i] = (uint16_t)c;
                    if (a.w8) a.w8[i] = (uint8_t)w8_code1(c, wsat, wb, wn, wu);
                }
            }
        }
    }
    if (a.mcnt) flush_counters<256>(mb - mn, mu_, mn, a.mcnt);
    if (a.wcnt) flush_counters<256>(wb - wn, wu, wn, a.wcnt);
    upd_tail(a);
}

// loss_scaling.cpp:89-92
__global__ void unscale_kernel(float* g, int64_t n, const fp8b_loss_scaler_t* s) {
    const float sc = __double2float_rn(s->scale);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        g[i] = __fdiv_rn(g[i], sc);
}

// ---------------------------------------------------------------- launchers
static int sm_count() { return device_sm_count(); }

template <int GFMT>
static void launch_sgd_fmt(const void* grad, uint16_t* master, float* mom, int64_t n,
                           const fp8b_sgd_args_t& args, cudaStream_t st, const LfsrTables& tabs) {
    UpdArgs a;
    a.lr = args.lr; a.mu = args.mu; a.two_lambda = args.two_lambda; a.scale = args.scale;
    a.scaler = args.scaler; a.skip = args.skip_counters; a.seed = args.seed;
    a.elem_offset = args.block_offset * kBlock; a.rbits = args.rbits;
    a.mcnt = args.master_counters; a.w8 = args.w_e5m2; a.w_sat = args.w_saturate;
    a.wcnt = args.w_counters;
    a.step_scaler = 0;  // set on the call's last kernel only
    a.iteration = args.step_iteration;
    a.skip2 = args.skip_counters2;
    a.gate_out = args.gate_out;
    const int want_step = args.scaler ? args.step_scaler : 0;
    constexpr int NT = 256;
    const bool cnt = a.mcnt != nullptr || a.wcnt != nullptr;
    const bool aligned = ((uintptr_t)grad % 16 == 0) && ((uintptr_t)master % 16 == 0) &&
                         ((uintptr_t)mom % 16 == 0) && (a.w8 == nullptr || (uintptr_t)a.w8 % 16 == 0) &&
                         (a.rbits == nullptr || (uintptr_t)a.rbits % 16 == 0);
    if (args.master_mode == FP8B_SR && args.bits == FP8B_BITS_LFSR) {
        const int64_t nb = (n + kBlock - 1) / kBlock;
        int64_t begin = 0;
        // up to one resident wave of CTA-per-block CTAs (4 per SM at 64 registers)
        // the CTA kernel wins: its 256 threads take a block at once, while a warp
        // walks it as 16 dependent chunks (2.36M parameters = 576 blocks: 17 -> 9 us)
        int64_t cta_max = lfsr_cta_max_blocks();
        if (!getenv("FP8B_LFSR_CTA_MAX")) {
            int per_sm = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sgd_lfsr_kernel<GFMT>, 256, 0);
            if ((int64_t)per_sm * sm_count() > cta_max) cta_max = (int64_t)per_sm * sm_count();
        }
        if (aligned && n / kBlock > cta_max) {
            const int64_t nfull = n / kBlock;
            constexpr int smem = kUpdTabBytes;
            // one warp per 4096-block: a small tensor (config 1: 256 blocks)
            // spreads its warps over every SM instead of filling a few CTAs
            int64_t g = sm_count();
            // A warp walks a block as a serial chain of 16 chunks whose pace is
            // ~max(1.1 us, 0.082 us x warps per SM) (latency floor, then HBM), and
            // a partly filled last round of blocks costs a whole round: time ~
            // rounds(w) x pace(w). Pick the warps per CTA that minimise it
            // (measured: 2^24 parameters = 4096 blocks, 24 warps: 2 rounds, 63 us;
            // 28-32 warps: 1 round, 39 us; 2^26: 24 warps 160 us, 32 warps 170 us).
            // More than 24 warps take the 1024-thread instantiation (64 registers,
            // a few spills). FP8B_UPD_WARPS forces a count (diagnostic).
            static const int force = [] { const char* e = getenv("FP8B_UPD_WARPS"); return e ? atoi(e) : 0; }();
            constexpr int kW = kWarpUpdThreads / 32;
            int wbest = kW;
            if (nfull <= g * kW) {
                wbest = (int)((nfull + g - 1) / g);  // one round, spread over every SM
            } else {
                auto cost = [&](int w) {
                    const double rounds = (double)((nfull + g * w - 1) / (g * w));
                    double pace = 0.082 * w > 1.1 ? 0.082 * w : 1.1;
                    if (w > kW) pace *= 1.05;
                    return rounds * pace;
                };
                double cbest = cost(kW);
                for (int w = 16; w <= 32; ++w)  // leave the default only for a clear (3 %) gain
                    if (cost(w) < cbest * 0.97) { cbest = cost(w); wbest = w; }
            }
            if (force >= 1 && force <= 32) wbest = force;
            const bool big = wbest > kWarpUpdThreads / 32;
            auto fn = big ? (cnt ? sgd_lfsr_warp_kernel<GFMT, true, 1024> : sgd_lfsr_warp_kernel<GFMT, false, 1024>)
                          : (cnt ? sgd_lfsr_warp_kernel<GFMT, true> : sgd_lfsr_warp_kernel<GFMT, false>);
            ensure_smem_attr((const void*)fn, smem);
            int64_t wpc = wbest;
            const int64_t need = (nfull + wpc - 1) / wpc;
            if (need < g) g = need;
            a.step_scaler = nfull == nb ? want_step : 0;  // no tail kernel follows
            fn<<<(int)g, (int)(32 * wpc), smem, st>>>(grad, master, mom, nfull, a, args.block_offset,
                                                      tabs);
            begin = nfull;
        }
        if (begin < nb) {
            int per_sm = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sgd_lfsr_kernel<GFMT>, 256, 0);
            int64_t g = (int64_t)sm_count() * (per_sm > 0 ? per_sm : 1);
            if (nb - begin < g) g = nb - begin;
            a.step_scaler = want_step;
            sgd_lfsr_kernel<GFMT><<<(int)g, 256, 0, st>>>(grad, master, mom, n, a,
                                                          args.block_offset, tabs, begin,
                                                          aligned ? 1 : 0);
        }
        return;
    }
    int64_t g = (int64_t)sm_count() * 8;  // two rounds of resident CTAs (measured: beats one)
    const int64_t need = ((aligned ? n / 16 : n) + NT - 1) / NT;
    if (need < g) g = need < 1 ? 1 : need;
    const int al = aligned ? 1 : 0;
    a.step_scaler = want_step;
    // 4 groups x 4 parameters per thread, <= 64 registers (4 CTAs of 256 per SM):
    // measured over 2^28 parameters against 2 groups at 72 registers, 4x6, 4x5,
    // 8x2, 8x3 (scripts/upd_time.py): RNE 0.718 -> 0.580 ms, counter SR + E5M2 W
    // 0.861 -> 0.704 ms.
#define FP8B_SGD_C(MODE, C) sgd_elem_kernel<GFMT, MODE, NT, C, 4, 4><<<(int)g, NT, 0, st>>>(grad, master, mom, n, a, al);
#define FP8B_SGD(MODE)                      \
    {                                       \
        if (cnt) FP8B_SGD_C(MODE, true)     \
        else FP8B_SGD_C(MODE, false)        \
    }
    if (args.master_mode == FP8B_RNE) FP8B_SGD(0)
    else if (args.bits == FP8B_BITS_COUNTER) FP8B_SGD(1)
    else FP8B_SGD(2)
#undef FP8B_SGD
#undef FP8B_SGD_C
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
