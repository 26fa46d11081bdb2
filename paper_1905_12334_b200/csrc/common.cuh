// common.cuh -- device-side building blocks shared by the fp8b200 kernels.
//
// The E5M2 / FP16 encoder here is the integer restatement of the reference's
// encode() (float_format.cpp:97-135) on FP32 bits (SURVEY 8a A2'); it is
// exhaustively equal to the reference for RNE and truncation over all 2^32
// inputs (checked on the B200 by tests/test_quantize_gpu.py::test_exhaustive).
#pragma once

#include <cstdlib>

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/fp8b200.h"

namespace fp8b {

constexpr int kBlock = 4096;  // kQuantBlock (tensor.hpp:65)
constexpr int kLfsrPeriod = 65535;

// Per-format constants (float_format.hpp:30-78). MB = mantissa bits.
template <int MB>
struct Fmt {
    static constexpr uint32_t maxbits = MB == 2 ? 0x47600000u : 0x477FE000u;  // 57344 / 65504
    static constexpr uint32_t maxcode = (30u << MB) | ((1u << MB) - 1u);
    static constexpr uint32_t infcode = 31u << MB;
    static constexpr uint32_t nancode = infcode | (1u << (MB - 1));
    static constexpr uint32_t signbit = 1u << (5 + MB);
    // RNE underflow band: 0 < |x| <= half the min subnormal (ties go to even 0)
    static constexpr uint32_t rne_unf_max = MB == 2 ? 0x37000000u : 0x33000000u;  // 2^-17 / 2^-25
    // trunc underflow band: 0 < |x| < min subnormal
    static constexpr uint32_t trunc_unf_lim = MB == 2 ? 0x37800000u : 0x33800000u;  // 2^-16 / 2^-24
};

// Result of splitting |x| into the truncated code and the discarded bits.
struct Split {
    uint32_t code;   // sign | truncated magnitude code, or the final special code
    uint32_t r16;    // top 16 discarded bits (SR) ; for RNE: round-up decision in bit 0
    bool inexact;    // a sample is consumed (finite, nonzero, not representable)
};

// Classify one FP32 value for a target with MB mantissa bits.
// Specials (NaN, overflow, zero, exact) come back with inexact=false and the
// final code. Overflow/NaN flags are derived by the caller from the bits.
template <int MB>
__device__ __forceinline__ Split split_bits(uint32_t u, bool saturate) {
    using F = Fmt<MB>;
    const uint32_t a = u & 0x7FFFFFFFu;
    const uint32_t sign = (u >> 31) ? F::signbit : 0u;
    const uint32_t e = a >> 23;
    const uint32_t m = a & 0x7FFFFFu;
    const uint32_t sig = e ? (m | 0x800000u) : m;
    const uint32_t emax1 = e > 1u ? e : 1u;
    // dbits = 23-MB for normal targets (e >= 113), 136-MB-max(e,1) below.
    const uint32_t dbits = (23u - MB) + (emax1 < 113u ? 113u - emax1 : 0u);
    const uint32_t sh = dbits < 31u ? dbits : 31u;
    const uint32_t ebase = e > 113u ? ((e - 113u) << MB) : 0u;
    const uint32_t mag0 = ebase + (sig >> sh);
    const uint32_t d = sig & ((1u << sh) - 1u);
    // top 16 discarded bits: (d << 16) >> dbits, 64-bit to cover dbits < 16
    const uint32_t dsh = dbits < 63u ? dbits : 63u;
    const uint32_t r16 = (uint32_t)(((uint64_t)d << 16) >> dsh);
    Split s;
    s.code = sign | mag0;
    s.r16 = r16;
    s.inexact = d != 0u;
    if (a > F::maxbits) {  // includes Inf and NaN
        s.inexact = false;
        s.code = (a > 0x7F800000u) ? F::nancode : (sign | (saturate ? F::maxcode : F::infcode));
    }
    // a == 0 -> mag0 == 0, d == 0: code = sign, exact. Nothing to do.
    return s;
}

// RNE round-up decision from the discarded bits (SURVEY A2' step 7).
template <int MB>
__device__ __forceinline__ uint32_t rne_up(uint32_t u) {
    const uint32_t a = u & 0x7FFFFFFFu;
    const uint32_t e = a >> 23;
    const uint32_t m = a & 0x7FFFFFu;
    const uint32_t sig = e ? (m | 0x800000u) : m;
    const uint32_t emax1 = e > 1u ? e : 1u;
    const uint32_t dbits = (23u - MB) + (emax1 < 113u ? 113u - emax1 : 0u);
    if (dbits > 24u) return 0u;
    const uint32_t d = sig & ((1u << dbits) - 1u);
    const uint32_t half = 1u << (dbits - 1u);
    const uint32_t lsb = (sig >> dbits) & 1u;
    return (d > half || (d == half && lsb)) ? 1u : 0u;
}

// Full integer encode for RNE / TRUNC / SR(with r16). Returns the code and
// sets the reference's flags (float_format.hpp:82-86) plus NaN.
template <int MB>
__device__ __forceinline__ uint32_t encode_int(uint32_t u, int mode, uint32_t r16,
                                               bool saturate, int& ovf, int& unf, int& nan) {
    using F = Fmt<MB>;
    const uint32_t a = u & 0x7FFFFFFFu;
    nan = a > 0x7F800000u;
    ovf = (a > F::maxbits) && !nan;
    Split s = split_bits<MB>(u, saturate);
    uint32_t up = 0;
    if (s.inexact) {
        if (mode == FP8B_RNE) up = rne_up<MB>(u);
        else if (mode == FP8B_SR) up = (s.r16 + r16) >= 65536u;
    }
    const uint32_t code = s.code + up;
    unf = (a != 0u) && !nan && !ovf && ((code & (F::signbit - 1u)) == 0u);
    return code;
}

// Hardware RNE path: cvt.rn.satfinite.e5m2x2.f32 + the two reference fixups
// (SURVEY 0.2): |x| > 57344 overflows to Inf (or max code) and NaN -> 0x7E.
__device__ __forceinline__ uint32_t cvt_e5m2x2(float lo, float hi) {
    uint16_t r;
    asm("cvt.rn.satfinite.e5m2x2.f32 %0, %1, %2;" : "=h"(r) : "f"(hi), "f"(lo));
    return r;
}

// Four floats -> one word of four E5M2 RNE codes (satfinite hardware cvt): the
// two 16-bit results are packed by one mov.b32 (no zero-extension masks).
__device__ __forceinline__ uint32_t cvt_e5m2x4(float f0, float f1, float f2, float f3) {
    uint32_t r;
    asm("{\n"
        ".reg .b16 lo, hi;\n"
        "cvt.rn.satfinite.e5m2x2.f32 lo, %2, %1;\n"
        "cvt.rn.satfinite.e5m2x2.f32 hi, %4, %3;\n"
        "mov.b32 %0, {lo, hi};\n"
        "}\n"
        : "=r"(r)
        : "f"(f0), "f"(f1), "f"(f2), "f"(f3));
    return r;
}

__device__ __forceinline__ uint32_t cvt_f16x2(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}

// Fix up one hardware E5M2 RNE code and update counters.
template <int MB>
__device__ __forceinline__ uint32_t fix_rne(uint32_t hw, uint32_t u, bool saturate,
                                            uint32_t& c_big, uint32_t& c_nan, uint32_t& c_unf) {
    using F = Fmt<MB>;
    const uint32_t a = u & 0x7FFFFFFFu;
    const bool big = a > F::maxbits;
    const bool isnan = a > 0x7F800000u;
    c_big += big;
    c_nan += isnan;
    c_unf += (a - 1u) < F::rne_unf_max;
    const uint32_t sign = (u >> 31) ? F::signbit : 0u;
    const uint32_t ovcode = sign | (saturate ? F::maxcode : F::infcode);
    return big ? (isnan ? F::nancode : ovcode) : hw;
}

// E5M2 / FP16 code -> FP32 (exact). E5M2 is the top byte of an FP16.
__device__ __forceinline__ float dec_e5m2(uint32_t c) {
    return __half2float(__ushort_as_half((unsigned short)((c & 0xFFu) << 8)));
}
__device__ __forceinline__ float dec_f16(uint32_t c) {
    return __half2float(__ushort_as_half((unsigned short)(c & 0xFFFFu)));
}
template <int MB>
__device__ __forceinline__ float dec_code(uint32_t c) {
    return MB == 2 ? dec_e5m2(c) : dec_f16(c);
}
// decode() as the reference returns it (float_format.cpp:60): every NaN code is
// the positive quiet NaN 0x7FC00000 (the GPU's f16->f32 gives 0x7FFFFFFF).
__device__ __forceinline__ float ref_nan(float v) {
    return v != v ? __uint_as_float(0x7FC00000u) : v;
}

// SplitMix64 (lfsr.cpp:47-52).
__device__ __forceinline__ uint64_t mix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}
__host__ __device__ __forceinline__ uint64_t mix64_hd(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

// LfsrStream::split(seed, idx).state() (lfsr.cpp:34-45).
__device__ __forceinline__ uint32_t lfsr_split(uint64_t seed, uint64_t idx) {
    uint64_t h = mix64(seed + 0x9E3779B97F4A7C15ull * (idx + 1));
    uint32_t s = (uint32_t)(h & 0xFFFFu);
    while (s == 0u) {
        h = mix64(h + 1);
        s = (uint32_t)(h & 0xFFFFu);
    }
    return s;
}

// Decimated-cycle tables: tabx[k] = bitrev16(D^k(1)) for
// k in [0, 65535 + 4096) (wrapping), pos[s] = k with D^k(1) == s, D = 16 clocks.
// Sample j of a block stream starting at state s0 is tabx[pos[s0] + j].
struct LfsrTables {
    const uint16_t* tabx;
    const uint16_t* pos;
};

// Counter-bits sample (see FP8B_BITS_COUNTER): the 64-bit SplitMix64 output
// for element group g = gi >> 2 supplies the four 16-bit samples of elements
// 4g .. 4g+3, low half-word first.
__device__ __forceinline__ uint64_t counter_word(uint64_t seed, uint64_t group) {
    return mix64(seed + group + 1ull);
}
__device__ __forceinline__ uint32_t counter_r16(uint64_t seed, uint64_t gi) {
    return (uint32_t)(counter_word(seed, gi >> 2) >> (16u * (uint32_t)(gi & 3u))) & 0xFFFFu;
}

// ---- stochastic rounding as an integer carry (the reference rule exactly) --
// For |x| <= max normal, the SR result magnitude of encode() is
//   normal targets (|x| >= 2^-14): the FP32 bit pattern with r16 added just
//   below the kept mantissa (E5M2: r16<<5 under 21 discarded bits; FP16:
//   r16>>3 under 13 discarded bits -- the dropped low bits of r16 cannot change
//   the carry), shifted down and re-biased (exponent e -> e-112);
//   subnormal targets: t = |x| * 2^(16 + quantum exponent), truncated, plus r16,
//   >> 16.
// Both are "round up iff top-16 discarded bits + r16 >= 2^16" (SURVEY A2'),
// which equals float_format.cpp:122-130; checked against encode_int in tests.
template <int MB>
__device__ __forceinline__ uint32_t sr_mag(uint32_t a, float xabs, uint32_t r16) {
    uint32_t cn, t;
    if (MB == 2) {
        cn = (a + (r16 << 5) - 0x38000000u) >> 21;
        t = __float2uint_rz(xabs * 4294967296.0f);        // |x| * 2^32 < 2^18
    } else {
        cn = (a + (r16 >> 3) - 0x38000000u) >> 13;
        t = __float2uint_rz(xabs * 1099511627776.0f);     // |x| * 2^40 < 2^26
    }
    const uint32_t cs = (t + r16) >> 16;
    return a < 0x38800000u ? cs : cn;
}

// A sample is consumed iff |x| is finite, <= max normal, nonzero and not on the
// target grid (float_format.cpp:111-113).
template <int MB>
__device__ __forceinline__ bool sr_inexact(uint32_t a, float xabs) {
    const uint32_t mask = MB == 2 ? 0x1FFFFFu : 0x1FFFu;
    const float q = xabs * (MB == 2 ? 65536.0f : 16777216.0f);  // in subnormal quanta
    const bool sub_inexact = q != truncf(q);
    const bool nrm_inexact = (a & mask) != 0u;
    return (a <= Fmt<MB>::maxbits) && (a < 0x38800000u ? sub_inexact : nrm_inexact);
}

// Full SR encode with counters, for one element given its sample.
template <int MB>
__device__ __forceinline__ uint32_t sr_encode(uint32_t u, uint32_t r16, bool sat, uint32_t& c_big,
                                              uint32_t& c_nan, uint32_t& c_unf) {
    using F = Fmt<MB>;
    const uint32_t a = u & 0x7FFFFFFFu;
    const uint32_t sign = (u >> 31) ? F::signbit : 0u;
    const uint32_t mag = sr_mag<MB>(a, __uint_as_float(a), r16);
    const bool big = a > F::maxbits;
    const bool isnan = a > 0x7F800000u;
    c_big += big;
    c_nan += isnan;
    c_unf += (!big) & (mag == 0u) & (a != 0u);
    const uint32_t ovcode = sign | (sat ? F::maxcode : F::infcode);
    return big ? (isnan ? F::nancode : ovcode) : (sign | mag);
}

// Block-wide sum of three counters; one atomic per CTA.
template <int NT>
__device__ __forceinline__ void flush_counters(uint32_t c0, uint32_t c1, uint32_t c2,
                                               int64_t* counters) {
    __shared__ unsigned long long red[3][NT / 32];
    unsigned long long v0 = c0, v1 = c1, v2 = c2;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        v0 += __shfl_xor_sync(0xffffffffu, v0, o);
        v1 += __shfl_xor_sync(0xffffffffu, v1, o);
        v2 += __shfl_xor_sync(0xffffffffu, v2, o);
    }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();  // a previous flush in the same kernel may still be reading red
    if (l == 0) { red[0][w] = v0; red[1][w] = v1; red[2][w] = v2; }
    __syncthreads();
    if (threadIdx.x < 3) {
        unsigned long long s = 0;
        const int nw = (int)(blockDim.x >> 5);  // <= NT / 32 (launch bound)
#pragma unroll
        for (int i = 0; i < NT / 32; ++i)
            if (i < nw) s += red[threadIdx.x][i];
        if (s) atomicAdd(reinterpret_cast<unsigned long long*>(counters) + threadIdx.x, s);
    }
}

// CTA-wide exclusive scan of inexact flags over a 4096-element block walked as
// (round r in 0..3, thread t in 0..255, k in 0..3) -- the LFSR consumption order.
template <int MB, int BAR = 0>
struct BlockScan {
    static constexpr int NT = 256;
    // Exclusive prefix (in block order) of the inexact flags of this thread's
    // 16 elements, given per-round 4-bit masks. Returns the prefix of the
    // thread's first element of each round in pre[r].
    __device__ __forceinline__ static void run(const uint32_t mask[4], uint32_t pre[4],
                                               uint32_t* smem_w /*[8]*/) {
        uint32_t cnt[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) cnt[r] = (uint32_t)__popc(mask[r]);
        run_counts(cnt, pre, smem_w);
    }
    // Same, from per-round counts (each <= 4).
    __device__ __forceinline__ static void run_counts(const uint32_t cnt[4], uint32_t pre[4],
                                                      uint32_t* smem_w /*[8]*/) {
        const int lane = threadIdx.x & 31, w = (threadIdx.x >> 5) & 7;
        // pack the 4 per-round counts (<= 4 each, warp sum <= 128) into bytes
        uint32_t packed = 0;
#pragma unroll
        for (int r = 0; r < 4; ++r) packed |= cnt[r] << (8 * r);
        uint32_t inc = packed;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += t;
        }
        if (lane == 31) smem_w[w] = inc;
        if (BAR == 0) __syncthreads();
        else asm volatile("bar.sync %0, 256;" ::"r"(BAR) : "memory");
        const uint32_t excl = inc - packed;
        // Cross-warp part, warp-cooperative: lanes 0..7 hold the 8 warp totals,
        // split into 16-bit fields (rounds 0,2 in lo; 1,3 in hi) and scanned
        // with three shuffles; every warp does it redundantly (no 2nd barrier).
        const uint32_t tw = smem_w[lane & 7];
        uint32_t lo = tw & 0x00FF00FFu, hi = (tw >> 8) & 0x00FF00FFu;
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) {
            const uint32_t tl = __shfl_up_sync(0xffffffffu, lo, o);
            const uint32_t th = __shfl_up_sync(0xffffffffu, hi, o);
            if ((lane & 7) >= o) { lo += tl; hi += th; }
        }
        // inclusive over warps 0..7 -> totals (lane 7) and this warp's exclusive prefix
        const uint32_t tot_lo = __shfl_sync(0xffffffffu, lo, 7);
        const uint32_t tot_hi = __shfl_sync(0xffffffffu, hi, 7);
        uint32_t bef_lo = __shfl_sync(0xffffffffu, lo, (w + 7) & 7);
        uint32_t bef_hi = __shfl_sync(0xffffffffu, hi, (w + 7) & 7);
        if (w == 0) { bef_lo = 0; bef_hi = 0; }
        const uint32_t t0 = tot_lo & 0xFFFFu, t1 = tot_hi & 0xFFFFu, t2 = tot_lo >> 16;
        pre[0] = (bef_lo & 0xFFFFu) + (excl & 0xFFu);
        pre[1] = t0 + (bef_hi & 0xFFFFu) + ((excl >> 8) & 0xFFu);
        pre[2] = t0 + t1 + (bef_lo >> 16) + ((excl >> 16) & 0xFFu);
        pre[3] = t0 + t1 + t2 + (bef_hi >> 16) + (excl >> 24);
    }
};

// ---- mbarrier + bulk-copy (TMA) helpers ------------------------------------
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}
// 1-D bulk copy global -> shared, completing `bytes` on the mbarrier (TMA unit).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(dst)),
        "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}

// ---- packed SR representation ----------------------------------------------
// P = (truncated code magnitude << 16) | (top 16 discarded bits), for
// |x| <= max normal. Then the reference's SR result magnitude is (P + r16) >> 16
// (round up iff top-16 discarded bits + r16 >= 2^16, float_format.cpp:122-130),
// truncation is P >> 16, and an exact input has a zero low half so any r16
// leaves it unchanged. Built on the FMA pipe:
//  E5M2: |x| *rz 2^-112 re-biases the FP32 exponent to E5M2's (e-112) for
//        normal targets and, below 2^-14, truncates into the FP32 denormal grid
//        whose spacing is 2^-149 * 2^112 = 2^-37, i.e. 2^-16 * 2^-21: bits >> 5
//        is P in both ranges.
//  FP16: normal P = (a - 112<<23) << 3 (computed from the raw bits, the sign is
//        shifted out); subnormal P = floor(|x| * 2^40), selected below 2^-14.
__device__ __forceinline__ uint32_t packed_e5m2(float x) {
    return __float_as_uint(__fmul_rz(fabsf(x), 0x1p-112f)) >> 5;
}
__device__ __forceinline__ uint32_t packed_f16(float x) {
    const uint32_t pn = __float_as_uint(x) * 8u + 0x40000000u;
    const uint32_t ps = __float2uint_rz(fabsf(x) * 0x1p40f);
    return fabsf(x) < 0x1p-14f ? ps : pn;
}
template <int MB>
__device__ __forceinline__ uint32_t packed_sr(float x) {
    return MB == 2 ? packed_e5m2(x) : packed_f16(x);
}
// Discarded bits nonzero (a stream sample is consumed), for |x| <= max normal:
// the RZ and RU products differ iff bits fell off below the FP32 denormal grid.
template <int MB>
__device__ __forceinline__ bool inexact_sr(float x) {
    const uint32_t rz = __float_as_uint(__fmul_rz(fabsf(x), 0x1p-112f));
    const uint32_t ru = __float_as_uint(__fmul_ru(fabsf(x), 0x1p-112f));
    return ((rz | ru) & (MB == 2 ? 0x1FFFFFu : 0x1FFFu)) != 0u;
}
// |x| > max normal or NaN (the reference's overflow test plus NaN).
template <int MB>
__device__ __forceinline__ bool big_or_nan(float x) {
    return !(fabsf(x) <= (MB == 2 ? 57344.0f : 65504.0f));
}
template <int MB>
__device__ __forceinline__ uint32_t special_packed(bool sat) {
    return (sat ? Fmt<MB>::maxcode : Fmt<MB>::infcode) << 16;
}
// NaN-propagating max (max.NaN): the screen of an overflow / NaN input.
__device__ __forceinline__ float fmax_nan(float a, float b) {
    float r;
    asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
    return r;
}
// Number of code magnitudes equal to 0 in a packed word of codes (MASK = the
// magnitude bits of each code: 0x7F7F7F7F for E5M2, 0x7FFF7FFF for FP16). A
// magnitude m plus the all-but-top mask sets the code's top bit iff m != 0,
// with no carry into the next code.
template <uint32_t MASK>
__device__ __forceinline__ uint32_t zero_mags(uint32_t w) {
    return __popc(~((w & MASK) + MASK) & ~MASK);
}
// Gather the code bytes (E5M2) of four packed sums plus the four input signs.
__device__ __forceinline__ uint32_t gather_e5m2(uint32_t s0, uint32_t s1, uint32_t s2, uint32_t s3,
                                                uint32_t u0, uint32_t u1, uint32_t u2, uint32_t u3) {
    const uint32_t c01 = __byte_perm(s0, s1, 0x0062), c23 = __byte_perm(s2, s3, 0x0062);
    const uint32_t g01 = __byte_perm(u0, u1, 0x0073), g23 = __byte_perm(u2, u3, 0x0073);
    const uint32_t c = __byte_perm(c01, c23, 0x5410), g = __byte_perm(g01, g23, 0x5410);
    return c | (g & 0x80808080u);
}
// Two FP16 codes (high halves of the packed sums) plus signs.
__device__ __forceinline__ uint32_t gather_f16(uint32_t s0, uint32_t s1, uint32_t u0, uint32_t u1) {
    return __byte_perm(s0, s1, 0x7632) | (__byte_perm(u0, u1, 0x7632) & 0x80008000u);
}

// ---- small PTX helpers that keep ptxas from carrying long-lived predicates --
// One step of an inclusive warp scan (shfl.up): the shuffle's in-range predicate
// guards the add, so no (lane >= d) predicate is held.
__device__ __forceinline__ uint32_t scan_step_up(uint32_t v, int d) {
    uint32_t r;
    asm volatile(
        "{\n"
        ".reg .u32 t;\n"
        ".reg .pred p;\n"
        "shfl.sync.up.b32 t|p, %1, %2, 0, 0xffffffff;\n"
        "@p add.u32 t, t, %1;\n"
        "mov.u32 %0, t;\n"
        "}\n"
        : "=r"(r)
        : "r"(v), "r"(d));
    return r;
}
// f > maxv or NaN: count it and return `special` instead of f.
__device__ __forceinline__ float clamp_big(float f, float maxv, float special, uint32_t& cnt) {
    float r;
    asm("{\n"
        ".reg .pred p;\n"
        "setp.gtu.f32 p, %2, %3;\n"
        "@p add.u32 %0, %0, 1;\n"
        "selp.f32 %1, %4, %2, p;\n"
        "}\n"
        : "+r"(cnt), "=f"(r)
        : "f"(f), "f"(maxv), "f"(special));
    return r;
}
// m | bit if f > thr (ordered: false for NaN), as a compare plus one predicated OR.
__device__ __forceinline__ uint32_t or_if_gt(uint32_t m, float f, float thr, uint32_t bit) {
    asm("{\n"
        ".reg .pred p;\n"
        "setp.gt.f32 p, %1, %2;\n"
        "@p or.b32 %0, %0, %3;\n"
        "}\n"
        : "+r"(m)
        : "f"(f), "f"(thr), "r"(bit));
    return m;
}
// f > thr or unordered: returns the predicate and counts it with one predicated add.
__device__ __forceinline__ bool count_gtu(float f, float thr, uint32_t& cnt) {
    uint32_t r;
    asm("{\n"
        ".reg .pred p;\n"
        "setp.gtu.f32 p, %2, %3;\n"
        "@p add.u32 %0, %0, 1;\n"
        "selp.u32 %1, 1, 0, p;\n"
        "}\n"
        : "+r"(cnt), "=r"(r)
        : "f"(f), "f"(thr));
    return r != 0u;
}
__device__ __forceinline__ uint32_t mad_lo(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t r;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
    return r;
}

// An output Q node applied by a reduction kernel's last step (split-K sums of
// the conv wgrads): the same integer rule and counter-bit stream as the
// standalone quantize launch it replaces (element i draws counter_r16(seed, i)).
struct QNode {
    void* codes;       // null: no Q node
    int fmt, mode;
    uint64_t seed;
    int sat;
    int64_t* counters;
};
__device__ __forceinline__ void qnode_store(const QNode& q, int64_t i, float v, uint32_t& co,
                                            uint32_t& cu, uint32_t& cn) {
    const uint32_t r16 = q.mode == FP8B_SR ? counter_r16(q.seed, (uint64_t)i) : 0u;
    int o, u, n;
    if (q.fmt == FP8B_E5M2) {
        const uint32_t c = encode_int<2>(__float_as_uint(v), q.mode, r16, q.sat != 0, o, u, n);
        reinterpret_cast<uint8_t*>(q.codes)[i] = (uint8_t)c;
    } else {
        const uint32_t c = encode_int<10>(__float_as_uint(v), q.mode, r16, q.sat != 0, o, u, n);
        reinterpret_cast<uint16_t*>(q.codes)[i] = (uint16_t)c;
    }
    co += o; cu += u; cn += n;
}

// ---- programmatic dependent launch (PDL) -----------------------------------
// A kernel launched with programmatic stream serialization (tc_common.cuh
// launch_pdl: the tcgen05 GEMM) may have its CTAs scheduled, and run its
// prologue, while the previous kernel of the stream is still running, once every
// CTA of that kernel has executed pdl_trigger (or exited). The dependent blocks
// in pdl_wait -- before its first global-memory access -- until the previous
// kernel has completed and its writes are visible, so nothing observable
// changes; what is hidden is the ~2.8 us dependent-node latency plus the GEMM's
// prologue behind a short producer (the Q node before a layer's GEMM). Both are
// no-ops for plain launches.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Launch with programmatic stream serialization (see pdl_wait above).
// FP8B_PDL=0 launches the plain way.
inline bool pdl_enabled() {
    static const bool on = [] { const char* e = getenv("FP8B_PDL"); return !(e && e[0] == '0'); }();
    return on;
}
template <class... KArgs, class... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), unsigned grid, unsigned block, size_t smem,
                              cudaStream_t st, Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, KArgs(args)...);
}


}  // namespace fp8b
