// quant_group.cuh -- the position-independent Q node on one float4 group, shared
// by the elementwise quantize kernels (quantize.cu) and the fused peer-memory
// reduce + quantize kernel (peer.cu).
#pragma once

#include "common.cuh"

namespace fp8b {

// ---------------------------------------------------------------------------
// Position-independent quantize.
// MODE: 0 RNE (hardware cvt), 1 SR counter bits, 2 SR supplied bits, 3 TRUNC
// One float4 group g -> one code word (E5M2) or two (FP16).
template <int MB, int MODE>
__device__ __forceinline__ void quant_group(const float4& v, const uint32_t (&rb)[4], int64_t g,
                                            void* __restrict__ codes, uint64_t seed, bool sat,
                                            int64_t elem_offset, uint32_t& c_big, uint32_t& c_nan,
                                            uint32_t& c_unf) {
    const float f[4] = {v.x, v.y, v.z, v.w};
    uint32_t c[4];
    if (MODE == 0 && MB == 2) {
        // E5M2 RNE on whole code words. The hardware cvt (satfinite)
        // returns the max code 0x7B for every |x| > 57344 (Inf included),
        // so the reference's overflow rule (float_format.cpp:104-108) is
        // "+1 on the code byte" (0x7B -> the Inf code 0x7C) unless
        // saturating; underflow = zero-magnitude codes minus exact-zero
        // inputs; NaN (rare) rewrites its byte to the canonical 0x7E.
        uint32_t w = cvt_e5m2x4(f[0], f[1], f[2], f[3]);
        uint32_t m = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) m = or_if_gt(m, fabsf(f[k]), 57344.0f, 1u << (8 * k));
        c_big += __popc(m);
        c_unf += zero_mags<0x7F7F7F7Fu>(w);
        if (!sat) w += m;
        const float amax = fmax_nan(fmax_nan(fabsf(f[0]), fabsf(f[1])), fmax_nan(fabsf(f[2]), fabsf(f[3])));
        const float amin = fminf(fminf(fabsf(f[0]), fabsf(f[1])), fminf(fabsf(f[2]), fabsf(f[3])));
        if (amin == 0.0f) {
#pragma unroll
            for (int k = 0; k < 4; ++k) c_unf -= (__float_as_uint(f[k]) << 1) == 0u;
        }
        if (amax != amax) {
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (f[k] != f[k]) {
                    ++c_nan;
                    w = (w & ~(0xFFu << (8 * k))) | ((uint32_t)Fmt<MB>::nancode << (8 * k));
                }
        }
        __stcs(reinterpret_cast<uint32_t*>(codes) + g, w);
        return;
    }
    if (MODE == 0) {
        if (MB == 2) {
            const uint32_t p01 = cvt_e5m2x2(f[0], f[1]);
            const uint32_t p23 = cvt_e5m2x2(f[2], f[3]);
            c[0] = p01 & 0xFFu; c[1] = p01 >> 8; c[2] = p23 & 0xFFu; c[3] = p23 >> 8;
        } else {
            const uint32_t hw01 = cvt_f16x2(f[0], f[1]);
            const uint32_t hw23 = cvt_f16x2(f[2], f[3]);
            c[0] = hw01 & 0xFFFFu; c[1] = hw01 >> 16; c[2] = hw23 & 0xFFFFu; c[3] = hw23 >> 16;
        }
#pragma unroll
        for (int k = 0; k < 4; ++k)
            c[k] = fix_rne<MB>(c[k], __float_as_uint(f[k]), sat, c_big, c_nan, c_unf);
    } else {
        // SR / TRUNC on the packed representation. Screens: amax
        // (NaN-propagating) for overflow / NaN inputs, amin for an exact
        // zero input; underflow = code magnitude 0 from a nonzero input,
        // counted on the packed output words.
        uint64_t word = 0;
        if (MODE == 1) word = counter_word(seed, (uint64_t)((elem_offset >> 2) + g));
        uint32_t r16[4] = {0u, 0u, 0u, 0u};  // TRUNC == SR with r16 = 0
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if (MODE == 1) r16[k] = (uint32_t)(word >> (16 * k)) & 0xFFFFu;
            if (MODE == 2) r16[k] = rb[k];
        }
        const float amax = fmax_nan(fmax_nan(fabsf(f[0]), fabsf(f[1])), fmax_nan(fabsf(f[2]), fabsf(f[3])));
        const float amin = fminf(fminf(fabsf(f[0]), fabsf(f[1])), fminf(fabsf(f[2]), fabsf(f[3])));
        uint32_t sum[4];
        // (FP16: deriving the packed form from one *rz 2^-112 multiply, with a
        // screen for the 3 bits lost under the FP32 denormal grid, was measured
        // 3-7 % slower than the select below despite ~10 fewer instructions.)
#pragma unroll
        for (int k = 0; k < 4; ++k) {  // overflow (Inf / max code) or NaN: select, no branch
            const bool big = count_gtu(fabsf(f[k]), MB == 2 ? 57344.0f : 65504.0f, c_big);
            sum[k] = (big ? special_packed<MB>(sat) : packed_sr<MB>(f[k])) + r16[k];
        }
        const uint32_t u[4] = {__float_as_uint(f[0]), __float_as_uint(f[1]),
                               __float_as_uint(f[2]), __float_as_uint(f[3])};
        uint32_t w0, w1 = 0;
        if (MB == 2) {
            w0 = gather_e5m2(sum[0], sum[1], sum[2], sum[3], u[0], u[1], u[2], u[3]);
            c_unf += zero_mags<0x7F7F7F7Fu>(w0);
            if (amin == 0.0f) {
#pragma unroll
                for (int k = 0; k < 4; ++k) c_unf -= (u[k] << 1) == 0u;
            }
        } else {
            w0 = gather_f16(sum[0], sum[1], u[0], u[1]);
            w1 = gather_f16(sum[2], sum[3], u[2], u[3]);
            // an FP16 code magnitude of 0 needs |x| < 2^-24 (the min subnormal)
            if (amin < 0x1p-24f) {
                c_unf += zero_mags<0x7FFF7FFFu>(w0) + zero_mags<0x7FFF7FFFu>(w1);
#pragma unroll
                for (int k = 0; k < 4; ++k) c_unf -= (u[k] << 1) == 0u;
            }
        }
        if (amax != amax) {  // rare: NaN -> canonical unsigned code (float_format.cpp:99)
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (f[k] != f[k]) {
                    ++c_nan;
                    if (MB == 2) w0 = (w0 & ~(0xFFu << (8 * k))) | ((uint32_t)Fmt<MB>::nancode << (8 * k));
                    else if (k < 2) w0 = (w0 & ~(0xFFFFu << (16 * k))) | ((uint32_t)Fmt<MB>::nancode << (16 * k));
                    else w1 = (w1 & ~(0xFFFFu << (16 * (k - 2)))) | ((uint32_t)Fmt<MB>::nancode << (16 * (k - 2)));
                }
        }
        if (MB == 2) __stcs(reinterpret_cast<uint32_t*>(codes) + g, w0);
        else __stcs(reinterpret_cast<uint2*>(codes) + g, make_uint2(w0, w1));
        return;
    }
    if (MB == 2) {
        const uint32_t w = c[0] | (c[1] << 8) | (c[2] << 16) | (c[3] << 24);
        __stcs(reinterpret_cast<uint32_t*>(codes) + g, w);
    } else {
        const uint2 w = make_uint2(c[0] | (c[1] << 16), c[2] | (c[3] << 16));
        __stcs(reinterpret_cast<uint2*>(codes) + g, w);
    }
}


// How the kernels report the overflow counter of quant_group's c_big: it
// includes NaN inputs except on the E5M2 RNE word path (ordered compare).
template <int MB, int MODE>
__device__ __forceinline__ uint32_t quant_group_overflow(uint32_t c_big, uint32_t c_nan) {
    return (MODE == 0 && MB == 2) ? c_big : c_big - c_nan;
}

}  // namespace fp8b
