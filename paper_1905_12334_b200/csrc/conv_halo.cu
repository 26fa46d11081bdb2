// conv_halo.cu -- weight-stationary "halo slab" implicit-GEMM convolution on
// tcgen05 for the narrow 3x3 layers (conv2d_fp8 / conv2d_backward_data_fp8,
// kernels.cpp:106-151, 155-200; NHWC, stride 1), where C * bytes <= 128.
//
// The im2col kernel (conv_tc.cu) fetches every output pixel's input row once
// per filter tap: 9 TMA row requests per pixel for a 3x3 layer, which bounds
// the C = 64 layers by the TMA request rate, not by HBM or the tensor pipe.
// Here a tile is R whole output rows of one image (R = 128 / Wp, Wp = W + 2 pad
// the padded width). Its input is one zero-padded slab of SR padded rows x Wp
// columns x C channels, loaded by ONE 4-D tiled TMA box (out-of-image rows and
// columns come back as zeros), 64/128-byte swizzled like any K-major operand.
// In the padded row-major index q = oh * Wp + ow, the input of tap (kh, kw) for
// output q is slab row q + kh * Wp + kw, so the A operand of tap t is the slab
// itself seen from row offset kh * Wp + kw: a UMMA descriptor whose start
// address moves by whole rows (the swizzle is a function of the shared-memory
// address bits, so TMA's writes and the MMA's reads agree at any row offset).
// Output rows with ow >= OW (the 2 pad columns of each padded row) and rows
// beyond the tile are computed and dropped by the epilogue.
// The KRSC weights [F, k*k*C] of the whole layer (k*k taps x F x C) stay
// resident in shared memory for the kernel's lifetime (F <= 256, <= 150 KB).
// Per 128-pixel tile the operand stream is one slab (~18 KB for 3x3, C = 64
// at 56x56) instead of 9 x 8 KB of im2col rows.
//
// Roles (one CTA per SM, persistent): warp 0 TMA producer (weights once, then
// a ring of slabs), warp 1 MMA issuer (k*k*C/32 tcgen05.mma per tile, M=128,
// N=F, accumulator double-buffered in TMEM), warps 2-5 epilogue (TMEM lane
// quarters: bias, FP32 y and/or the fused output Q node with the reference's
// counters, as in gemm_tc.cu). Parity as for the im2col kernel: the GEMM
// tolerance |y - y_exact| <= 1e-6 * (|x| * |w|) (tests/test_conv_gpu.py).
#include <cstdlib>
#include <cstring>

#include "tc_common.cuh"

namespace fp8b {
namespace tc {
namespace halo {

// Per-tile timeline trace (scripts/probe_halo.cu builds this file with
// FP8B_HALO_TRACE): %globaltimer per CTA, role and tile.
#ifdef FP8B_HALO_TRACE
__device__ unsigned long long g_halo_trace[148 * 10 * 64];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define HTRACE(role, i)                                                                  \
    do {                                                                                 \
        if ((i) < 64 && blockIdx.x < 148) g_halo_trace[(blockIdx.x * 10 + (role)) * 64 + (i)] = gtimer(); \
    } while (0)
#else
#define HTRACE(role, i) \
    do {                \
    } while (0)
#endif

struct HParams {
    int64_t M, N;      // output matrix [P, F] (P = n * OH * OW)
    EpiArgs ep;
    int nimg, OH, OW;  // output geometry
    int Wp;            // padded width (slab row length)
    int R;             // output rows per tile
    int SR;            // slab rows loaded per tile
    int k, pad;        // square kernel, padding
    int tiles_per_img, ntiles;
    int bo_mode;       // descriptor base-offset rule for row-shifted starts (diagnostic knob)
    int wlog;          // log2(Wp): Wp is a power of two, so a tile is 128 / Wp whole rows
    int c_tma, q_tma;  // FP32 y / output codes go out through 4-D TMA stores
    int qg;            // code chunks per store row (32, 64 or 128 bytes)
    // epilogue staging per warp (bytes): the FP32 box(es) at c_off, the code
    // box(es) at q_off; *_nbuf = 2 is a ring of two boxes, 1 a single box
    int stg, c_off, q_off, c_nbuf, q_nbuf;
    int ew;            // epilogue warps: 8 (two per TMEM lane quarter) or 4
    int dbg;           // diagnostics (FP8B_CONV_HALO_DBG): 1 no slab loads, 2 no MMAs, 4 no epilogue work, 8 busy-poll waits, 16 no tcgen05.commit, 32 no code stores,
                       // 64 no code staging, 128 no Q node, 256 no TMEM loads, 512 no MMA loop
};

// 8 epilogue warps, two per TMEM lane quarter, each draining half of the
// tile's columns: a tile is only a few hundred tensor cycles, and one warp per
// SM sub-partition cannot hide the ALU latency of the output Q node (measured:
// the epilogue alone took longer than loads + MMAs with 4 warps).
// (4 when the layer's resident weights leave no room for 8 warps' staging.)
constexpr int EW_MAX = 8;
constexpr int THREADS_MAX = 64 + 32 * EW_MAX;

// Shared-memory plan for CB-byte pixel rows and a BN-wide filter tile.
template <int CB, int BN>
struct HGeo {
    static constexpr uint32_t W_TAP = (uint32_t)BN * CB;   // one tap's weights [BN x CB]
    static constexpr uint32_t SWZ = CB == 128 ? 2u : 4u;   // UMMA layout code
    static constexpr uint32_t SBO = 8u * CB;               // 8-row swizzle atom
    // A tile is only ~0.3-1 us of MMA work, so the MMA -> epilogue -> MMA
    // handshake latency (commit, barrier wake-ups) would set the pace with a
    // double-buffered accumulator: keep up to 8 tiles in flight in TMEM.
    static constexpr int NACC = 512 / BN < 8 ? 512 / BN : 8;
    static constexpr uint32_t TMEM_COLS = NACC * BN < 32 ? 32 : NACC * BN;
};

__device__ __forceinline__ uint64_t desc_bo(uint32_t saddr, uint32_t sbo, uint32_t layout,
                                            uint32_t bo) {
    uint64_t d = umma_desc(saddr, 16, sbo, layout);
    d |= (uint64_t)(bo & 7u) << 49;
    return d;
}

__device__ __forceinline__ void tma_load_4d(const CUtensorMap* tm, void* dst, uint64_t* bar,
                                            int32_t c0, int32_t c1, int32_t c2, int32_t c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2),
        "r"(c3)
        : "memory");
}

// tmX: 4-D tiled map over x [n, h, w, c] with box {c, Wp, SR, 1};
// tmW: 2-D map over w [f, k*k*c] with box {c, BN}.
__device__ __forceinline__ void tma_store_4d(const CUtensorMap* tm, uint8_t* buf, int lane, int32_t c0,
                                             int32_t c1, int32_t c2, int32_t c3) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) {
        asm volatile(
            "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
                reinterpret_cast<uint64_t>(tm)),
            "r"(smem_u32(buf)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
            : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
}

// Output Q node of one 32-column chunk (bias already added): code words (8
// E5M2 / 16 FP16) and the reference's counters for live lanes and valid
// columns. gbase = this lane's pixel * N + col0 (counter-bit SR position).
template <class P>
__device__ __forceinline__ void codes_chunk(const P& p, const float (&y)[32], int64_t gbase, bool live,
                                            int nvalid, uint32_t* w, uint32_t& co, uint32_t& cu,
                                            uint32_t& cn) {
    const EpiArgs& ep = p.ep;
    const bool sat = ep.cq_sat != 0;
    if (ep.cq_fmt == FP8B_E5M2 && ep.cq_mode == FP8B_RNE) {
        uint32_t w8[8];
        lean_e5m2_codes(y, w8, sat, live, nvalid, co, cu, cn);
#pragma unroll
        for (int q = 0; q < 8; ++q) w[q] = w8[q];
        return;
    }
    uint32_t code[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
        int o, u, na;
        const uint32_t r16 = ep.cq_mode == FP8B_SR ? counter_r16(ep.cq_seed, (uint64_t)(gbase + j)) : 0u;
        code[j] = ep.cq_fmt == FP8B_E5M2 ? encode_int<2>(__float_as_uint(y[j]), ep.cq_mode, r16, sat, o, u, na)
                                         : encode_int<10>(__float_as_uint(y[j]), ep.cq_mode, r16, sat, o, u, na);
        if (live && j < nvalid) { co += o; cu += u; cn += na; }
    }
    if (ep.cq_fmt == FP8B_E5M2) {
#pragma unroll
        for (int q = 0; q < 8; ++q)
            w[q] = code[4 * q] | (code[4 * q + 1] << 8) | (code[4 * q + 2] << 16) | (code[4 * q + 3] << 24);
    } else {
#pragma unroll
        for (int q = 0; q < 16; ++q) w[q] = code[2 * q] | (code[2 * q + 1] << 16);
    }
}

// tmY / tmQ: 4-D store maps over y [n, oh, ow, f] (FP32) / the output codes,
// boxes {32 | qg * 32 columns, min(32, Wp) pixels, max(1, 32 / Wp) rows, 1}:
// one box = one epilogue warp's 32 TMEM lanes for one column chunk.
// KS: the kernel size when known at compile time (3: the tap loop fully
// unrolled, every descriptor a constant offset), 0: any k at run time.
// LEAN: compiled for the layer step's output only -- fused E5M2 RNE codes, no
// FP32 y, no bias, no diagnostics -- so the epilogue warps issue far fewer
// instructions beside the MMA-issuing warp they share an SM sub-partition with.
template <int ES, int CB, int BN, int KS, int LEAN = 0>
__global__ void __launch_bounds__(THREADS_MAX, 1)
    conv_halo_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW,
                     const __grid_constant__ CUtensorMap tmY, const __grid_constant__ CUtensorMap tmQ,
                     const HParams p, uint32_t slab_bytes, int nstages) {
    using G = HGeo<CB, BN>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    const int kk_ = KS ? KS : p.k;  // kernel size
    const int taps = kk_ * kk_;
    uint8_t* wsm = smem;                                                       // resident weights
    uint8_t* ring = smem + (((uint32_t)taps * G::W_TAP + 1023u) & ~1023u);     // slab ring
    uint8_t* stg = ring + (uint32_t)nstages * slab_bytes;                      // p.stg bytes per epilogue warp
    uint64_t* bars = reinterpret_cast<uint64_t*>(stg + p.ew * p.stg);
    uint64_t* full_bar = bars;
    uint64_t* empty_bar = full_bar + nstages;
    uint64_t* tfull_bar = empty_bar + nstages;
    uint64_t* tempty_bar = tfull_bar + G::NACC;
    uint64_t* w_bar = tempty_bar + G::NACC;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(w_bar + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // pipeline waits: try_wait (the thread may be suspended between polls, so
    // waiting warps leave issue slots to the working ones), or busy-poll
    // (test_wait, diagnostic)
    auto hwait = [&](uint64_t* bar, uint32_t par) {
        if (p.dbg & 8) mbar_wait_spin(bar, par);
        else mbar_wait(bar, par);
    };
    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmX)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmW)) : "memory");
        for (int s = 0; s < nstages; ++s) {
            mbar_init(full_bar + s, 1);
            mbar_init(empty_bar + s, 1);
        }
        for (int a = 0; a < G::NACC; ++a) {
            mbar_init(tfull_bar + a, 1);
            mbar_init(tempty_bar + a, p.ew);
        }
        mbar_init(w_bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(G::TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem_base = *tmem_slot;

    uint32_t co = 0, cu = 0, cn = 0;
    if (warp == 0) {
        if (lane == 0) {
            // the layer's weights, once: tap t -> [BN x CB] at wsm + t * W_TAP
            mbar_expect_tx(w_bar, (uint32_t)taps * G::W_TAP);
            for (int t = 0; t < taps; ++t)
                tma_load_2d(&tmW, wsm + t * G::W_TAP, w_bar, t * (CB / ES), 0);
            int stage = 0;
            uint32_t phase = 0;
            for (int tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x) {
                const int n = tile / p.tiles_per_img;
                const int oh0 = (tile - n * p.tiles_per_img) * p.R;
                hwait(empty_bar + stage, phase ^ 1);
                HTRACE(0, (tile - blockIdx.x) / gridDim.x);
                if (p.dbg & 1) {
                    mbar_arrive(full_bar + stage);
                } else {
                    mbar_expect_tx(full_bar + stage, (uint32_t)p.SR * p.Wp * CB);
                    tma_load_4d(&tmX, ring + stage * slab_bytes, full_bar + stage, 0, -p.pad, oh0 - p.pad, n);
                }
                if (++stage == nstages) { stage = 0; phase ^= 1; }
            }
        }
    } else if (warp == 1) {
        const uint32_t leader = elect_one();
        uint32_t idesc = (1u << 4);
        if (ES == 1) idesc |= (1u << 7) | (1u << 10);
        idesc |= (uint32_t)(BN >> 3) << 17;
        idesc |= (uint32_t)(128 >> 4) << 24;
        mbar_wait(w_bar, 0);
        // A tap's MMA is only 16-32 tensor cycles (N = 64..128), so the issue
        // loop must be a handful of instructions per MMA: the descriptors of
        // slab stage 0 / weight tap 0 are built once and only their 14-bit
        // start-address field moves (32-bit adds of byte offset >> 4; shared
        // memory < 256 KB, so it never carries out). The slab row offset of
        // tap (kh, kw), (kh * Wp + kw) * CB, is advanced incrementally.
        const uint64_t dA0 = desc_bo(smem_u32(ring), G::SBO, G::SWZ, 0);
        const uint64_t dB0 = umma_desc(smem_u32(wsm), 16, G::SBO, G::SWZ);
        const uint32_t aHi = (uint32_t)(dA0 >> 32), aLo0 = (uint32_t)dA0;
        const uint32_t bHi = (uint32_t)(dB0 >> 32), bLo0 = (uint32_t)dB0;
        const uint32_t row16 = CB >> 4;                                   // one slab row
        const uint32_t wrap16 = (uint32_t)(p.Wp - kk_ + 1) * row16;       // kw = k-1 -> next kh
        const uint32_t issue = leader && !(p.dbg & 2) ? 1u : 0u;
        int stage = 0;
        uint32_t phase = 0;
        int acc = 0;
        uint32_t accphase = 0;
        for (int tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x) {
            hwait(tempty_bar + acc, accphase ^ 1);
            fence_after();
            if (lane == 0) HTRACE(1, (tile - blockIdx.x) / gridDim.x);
            hwait(full_bar + stage, phase);
            fence_after();
            if (lane == 0) HTRACE(2, (tile - blockIdx.x) / gridDim.x);
            const uint32_t d_tmem = tmem_base + (uint32_t)(acc * BN);
            uint32_t a_lo = aLo0 + (uint32_t)stage * (slab_bytes >> 4);
            if constexpr (KS > 0) {
                // all taps unrolled: tap (kh, kw) reads slab rows kh * Wp + kw on
#pragma unroll
                for (int t = 0; t < KS * KS; ++t) {
                    const uint32_t aoff = (uint32_t)((t / KS) * p.Wp + (t % KS)) * row16;
#pragma unroll
                    for (int kk = 0; kk < CB / 32; ++kk) {
                        const uint64_t ad = ((uint64_t)aHi << 32) | (a_lo + aoff + 2u * kk);
                        const uint64_t bd = ((uint64_t)bHi << 32) | (bLo0 + (uint32_t)t * (G::W_TAP >> 4) + 2u * kk);
                        mma_p<ES>(d_tmem, ad, bd, idesc, (t | kk) ? 1u : 0u, issue);
                    }
                }
            } else {
                uint32_t b_lo = bLo0;
                int kw = 0;
#pragma unroll 1
                for (int t = 0; t < ((p.dbg & 512) ? 0 : taps); ++t) {
#pragma unroll
                    for (int kk = 0; kk < CB / 32; ++kk) {
                        const uint64_t ad = ((uint64_t)aHi << 32) | (a_lo + 2u * kk);
                        const uint64_t bd = ((uint64_t)bHi << 32) | (b_lo + 2u * kk);
                        mma_p<ES>(d_tmem, ad, bd, idesc, (t | kk) ? 1u : 0u, issue);
                    }
                    b_lo += G::W_TAP >> 4;
                    if (++kw == kk_) { kw = 0; a_lo += wrap16; } else { a_lo += row16; }
                }
            }
            if (lane == 0) HTRACE(3, (tile - blockIdx.x) / gridDim.x);
            // one commit per tile: the epilogue releases the slab stage once it
            // sees the accumulator complete (the MMAs that read it are done)
            if (p.dbg & 16) {  // diagnostic: plain arrival instead of tcgen05.commit
                if (lane == 0) mbar_arrive(tfull_bar + acc);
            } else {
                umma_commit_p(tfull_bar + acc, leader);
            }
            if (++stage == nstages) { stage = 0; phase ^= 1; }
            if (++acc == G::NACC) { acc = 0; accphase ^= 1; }
        }
    } else {
        // One warp = one TMEM lane quarter = 32 consecutive padded-row
        // positions: min(32, Wp) pixels of max(1, 32 / Wp) output rows, so each
        // column chunk leaves as one 4-D TMA store box (pad columns and rows
        // beyond the image are clipped by TMA; counters skip them).
        const int quarter = warp & 3;
        const int CPW = BN / 32 / (p.ew / 4);            // column chunks per warp
        const int c_lo = ((warp - 2) >> 2) * CPW;        // this warp's first chunk
        const int q = quarter * 32 + lane;
        const int r = q >> p.wlog, ow = q & ((1 << p.wlog) - 1);
        const int r0 = (quarter * 32) >> p.wlog, ow0 = (quarter * 32) & ((1 << p.wlog) - 1);
        // 8 KB of staging per warp: a ring of two 4 KB boxes for one output;
        // with both FP32 y and codes, one 4 KB box each
        uint8_t* cbase = stg + (warp - 2) * p.stg + p.c_off;
        uint8_t* qbase = stg + (warp - 2) * p.stg + p.q_off;
        const uint32_t qbox = (uint32_t)p.qg * 32 * (p.ep.cq_fmt == FP8B_E5M2 ? 1 : 2) * 32;
        uint32_t nst_c = 0, nst_q = 0;
        int sstage = 0;  // slab stage of the current tile
        // next staging box of an output; its previous store must have read it
        // (one store may stay pending with a ring of two, none with one box)
        auto acquire = [&](uint8_t* base, uint32_t& nst, int nbuf, uint32_t box) {
            uint8_t* b = base + (nbuf == 2 ? (nst++ & 1u) * box : 0u);
            if (lane == 0) {
                if (nbuf == 2) bulk_wait_read1();
                else bulk_wait_read0();
            }
            __syncwarp();
            return b;
        };
        int acc = 0;
        uint32_t accphase = 0;
        for (int tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x) {
            const int n = tile / p.tiles_per_img;
            const int oh0 = (tile - n * p.tiles_per_img) * p.R;
            const bool live = ow < p.OW && oh0 + r < p.OH;
            const bool any = ow0 < p.OW && oh0 + r0 < p.OH;  // warp-uniform
            const int64_t pix = ((int64_t)n * p.OH + oh0 + r) * p.OW + ow;
            hwait(tfull_bar + acc, accphase);
            fence_after();
            if (warp == 2 && lane == 0) {
                HTRACE(4, (tile - blockIdx.x) / gridDim.x);
                mbar_arrive(empty_bar + sstage);  // the tile's MMAs are done with its slab
            }
            if (++sstage == nstages) sstage = 0;
            const uint32_t taddr = tmem_base + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(acc * BN);
            int qpos = 0;
            uint8_t* qbuf = nullptr;
#pragma unroll 1
            for (int c = c_lo; any && (LEAN || !(p.dbg & 4)) && c < c_lo + CPW && c * 32 < p.N; ++c) {
                uint32_t v[32];
                if (!LEAN && (p.dbg & 256)) {
#pragma unroll
                    for (int j = 0; j < 32; ++j) v[j] = (uint32_t)(j * lane);
                } else {
                    tmem_ld32(taddr + c * 32, v);
                }
                if (LEAN) {
                    const int col0 = c * 32;
                    const int nvalid = p.N - col0 < 32 ? (int)(p.N - col0) : 32;
                    float y[32];
#pragma unroll
                    for (int j = 0; j < 32; ++j) y[j] = __uint_as_float(v[j]);
                    uint32_t w[8];
                    lean_e5m2_codes(y, w, p.ep.cq_sat != 0, live, nvalid, co, cu, cn);
                    if (qpos == 0) qbuf = acquire(qbase, nst_q, p.q_nbuf, qbox);
                    if (p.qg == 4) stage_write<128, 8>(qbuf, qpos * 32, w, lane);
                    else if (p.qg == 2) stage_write<64, 8>(qbuf, qpos * 32, w, lane);
                    else stage_write<32, 8>(qbuf, qpos * 32, w, lane);
                    if (++qpos == p.qg || c == c_lo + CPW - 1 || col0 + 32 >= p.N) {
                        tma_store_4d(&tmQ, qbuf, lane, col0 - 32 * (qpos - 1), ow0, oh0 + r0, n);
                        qpos = 0;
                    }
                    continue;
                }
                if (warp == 2 && lane == 0 && c == c_lo) HTRACE(6, (tile - blockIdx.x) / gridDim.x);
                const int col0 = c * 32;
                const int nvalid = p.N - col0 < 32 ? (int)(p.N - col0) : 32;
                float y[32];
#pragma unroll
                for (int j = 0; j < 32; ++j) y[j] = __uint_as_float(v[j]);
                if (p.ep.bias) {
#pragma unroll
                    for (int j = 0; j < 32; ++j)
                        if (j < nvalid) y[j] = __fadd_rn(y[j], __ldg(p.ep.bias + col0 + j));
                }
                const bool last = c == c_lo + CPW - 1 || col0 + 32 >= p.N;
                if (p.c_tma) {
                    uint8_t* buf = acquire(cbase, nst_c, p.c_nbuf, 4096u);
                    stage_write<128, 32>(buf, 0, reinterpret_cast<const uint32_t*>(y), lane);
                    tma_store_4d(&tmY, buf, lane, col0, ow0, oh0 + r0, n);
                }
                if (p.q_tma) {
                    uint32_t w[16];  // 8 words of E5M2 codes or 16 of FP16
                    if (p.dbg & 128) {
#pragma unroll
                        for (int j = 0; j < 16; ++j) w[j] = v[j];
                    } else {
                        codes_chunk(p, y, pix * p.N + col0, live, nvalid, w, co, cu, cn);
                    }
                    if (warp == 2 && lane == 0 && c == c_lo) HTRACE(7, (tile - blockIdx.x) / gridDim.x);
                    if (p.dbg & 64) continue;
                    if (qpos == 0) qbuf = acquire(qbase, nst_q, p.q_nbuf, qbox);
                    if (warp == 2 && lane == 0 && c == c_lo) HTRACE(8, (tile - blockIdx.x) / gridDim.x);
                    if (p.ep.cq_fmt == FP8B_E5M2) {
                        if (p.qg == 4) stage_write<128, 8>(qbuf, qpos * 32, w, lane);
                        else if (p.qg == 2) stage_write<64, 8>(qbuf, qpos * 32, w, lane);
                        else stage_write<32, 8>(qbuf, qpos * 32, w, lane);
                    } else {
                        if (p.qg == 2) stage_write<128, 16>(qbuf, qpos * 64, w, lane);
                        else stage_write<64, 16>(qbuf, qpos * 64, w, lane);
                    }
                    if (++qpos == p.qg || last) {
                        if (!(p.dbg & 32)) tma_store_4d(&tmQ, qbuf, lane, col0 - 32 * (qpos - 1), ow0, oh0 + r0, n);
                        qpos = 0;
                    }
                }
            }
            fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(tempty_bar + acc);
            if (warp == 2 && lane == 0) HTRACE(5, (tile - blockIdx.x) / gridDim.x);
            if (++acc == G::NACC) { acc = 0; accphase ^= 1; }
        }
        if (lane == 0) bulk_wait_read0();
    }
    if (p.ep.cq_counters) flush_counters<THREADS_MAX>(co, cu, cn, p.ep.cq_counters);
    fence_before();
    __syncthreads();
    if (warp == 1) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                     "r"(G::TMEM_COLS));
    }
}

static bool make_slab_map(CUtensorMap* tm, const void* x, int es, int64_t n, int64_t h, int64_t w,
                          int64_t c, int wp, int sr) {
    EncodeTiledFn enc = get_encode();
    if (!enc) return false;
    cuuint64_t dims[4] = {(cuuint64_t)c, (cuuint64_t)w, (cuuint64_t)h, (cuuint64_t)n};
    cuuint64_t strides[3] = {(cuuint64_t)(c * es), (cuuint64_t)(w * c * es), (cuuint64_t)(h * w * c * es)};
    cuuint32_t box[4] = {(cuuint32_t)c, (cuuint32_t)wp, (cuuint32_t)sr, 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    const CUtensorMapSwizzle swz = c * es == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
    return enc(tm, es == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_UINT16, 4,
               const_cast<void*>(x), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Geometry check shared by the launcher and conv_halo_supported().
struct Plan {
    int cb, bn, wp, r, sr, nstages;
    int qg, stg, c_off, q_off, c_nbuf, q_nbuf, ew;
    uint32_t wbytes, slab, smem;
};
// need_c / q_fmt (-1: none): which outputs the epilogue stages.
static bool plan_for(int64_t n, int64_t h, int64_t w, int64_t c, int64_t f, int k, int pad, int es,
                     Plan& pl, bool need_c = true, int q_fmt = FP8B_E5M2) {
    pl.cb = (int)(c * es);
    if (pl.cb != 64 && pl.cb != 128) return false;
    if (f % 16 || f < 16 || f > 256) return false;
    pl.bn = f <= 64 ? 64 : (f <= 128 ? 128 : 256);
    if (k < 1 || k > 7 || pad < 0 || pad > k - 1) return false;
    // slab row length: the padded width rounded up to a power of two, so a
    // 128-row tile is 128 / Wp whole output rows and each warp's 32 TMEM lanes
    // are whole pixel runs of one or more rows (one TMA store box)
    const int64_t oh = h + 2 * pad - k + 1, ow = w + 2 * pad - k + 1;
    if (oh < 1 || ow < 1 || w + 2 * pad > 128) return false;
    pl.wp = 1;
    while (pl.wp < w + 2 * pad) pl.wp <<= 1;
    pl.r = 128 / pl.wp;
    pl.sr = (128 + (k - 1) * (pl.wp + 1) + pl.wp - 1) / pl.wp;
    if (pl.sr > 256) return false;
    pl.wbytes = (uint32_t)(k * k) * pl.bn * pl.cb;
    pl.slab = (((uint32_t)pl.sr * pl.wp * pl.cb) + 1023u) & ~1023u;
    const uint32_t wpad = (pl.wbytes + 1023u) & ~1023u;
    // staging: 8 epilogue warps with rings of two boxes when they fit beside
    // two slabs; else single boxes (c and q sharing one when both are
    // written, codes flushed per chunk); else 4 warps.
    const int qes = q_fmt == FP8B_E5M2 ? 1 : 2;
    const bool need_q = q_fmt >= 0;
    const uint32_t base = 1024 + wpad + 256;
    bool fit = false;
    for (int ew = 8; ew >= 4 && !fit; ew -= 4) {
        for (int tight = 0; tight < 2 && !fit; ++tight) {
            pl.ew = ew;
            pl.qg = need_q ? tc::code_group(q_fmt, pl.bn / (ew / 4)) : 1;  // a warp's columns
            if (tight && need_q && need_c) pl.qg = 1;
            const uint32_t qbox = (uint32_t)pl.qg * 32 * qes * 32;
            if (!tight) {
                pl.c_nbuf = need_c ? (need_q ? 1 : 2) : 0;
                pl.q_nbuf = need_q ? (need_c ? 1 : 2) : 0;
                pl.c_off = 0;
                pl.q_off = pl.c_nbuf * 4096;
                pl.stg = pl.q_off + pl.q_nbuf * (int)qbox;
            } else {
                pl.c_nbuf = need_c ? 1 : 0;
                pl.q_nbuf = need_q ? 1 : 0;
                pl.c_off = pl.q_off = 0;
                pl.stg = need_c ? 4096 : (int)qbox;
            }
            fit = base + (uint32_t)ew * pl.stg + 2 * pl.slab <= 232448u;
        }
    }
    const uint32_t fixed = base + (uint32_t)pl.ew * pl.stg;
    if (fixed + 2 * pl.slab > 232448u) return false;
    pl.nstages = (int)((232448u - fixed) / pl.slab);
    const char* ns = getenv("FP8B_CONV_HALO_STAGES");
    const int cap = ns ? atoi(ns) : 4;
    if (pl.nstages > cap) pl.nstages = cap;
    pl.smem = fixed + (uint32_t)pl.nstages * pl.slab;
    if (n * oh * ow >= ((int64_t)1 << 31)) return false;
    return true;
}

// 4-D store map over an [n, oh, ow, f] output of es-byte elements, boxes of
// `cols` columns x one warp's 32 TMEM lanes (pixels x rows).
static bool make_out_map(CUtensorMap* tm, const void* out, int es, int64_t n, int64_t oh, int64_t ow,
                         int64_t f, int cols, int wp) {
    EncodeTiledFn enc = get_encode();
    if (!enc || !out || (uintptr_t)out % 16 || (f * es) % 16) return false;
    cuuint64_t dims[4] = {(cuuint64_t)f, (cuuint64_t)ow, (cuuint64_t)oh, (cuuint64_t)n};
    cuuint64_t strides[3] = {(cuuint64_t)(f * es), (cuuint64_t)(ow * f * es), (cuuint64_t)(oh * ow * f * es)};
    cuuint32_t box[4] = {(cuuint32_t)cols, (cuuint32_t)(wp < 32 ? wp : 32), (cuuint32_t)(wp < 32 ? 32 / wp : 1), 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    const int span = cols * es;
    const CUtensorMapSwizzle swz = span == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                   : span == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B;
    if (span != 32 && span != 64 && span != 128) return false;
    const CUtensorMapDataType dt = es == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8
                                   : es == 2 ? CU_TENSOR_MAP_DATA_TYPE_UINT16
                                             : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    return enc(tm, dt, 4, const_cast<void*>(out), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
               swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int ES, int CB, int BN>
static int run(const CUtensorMap& tx, const CUtensorMap& tw, const CUtensorMap& ty, const CUtensorMap& tq,
               const HParams& p, const Plan& pl, cudaStream_t st) {
    auto fn = p.k == 3 ? conv_halo_kernel<ES, CB, BN, 3> : conv_halo_kernel<ES, CB, BN, 0>;
    if constexpr (ES == 1) {
        // the layer step's case: E5M2 RNE codes only (FP8B_CONV_HALO_LEAN=0 disables)
        const char* el = getenv("FP8B_CONV_HALO_LEAN");
        if (p.k == 3 && p.q_tma && !p.c_tma && !p.ep.c && !p.ep.bias && p.ep.cq_fmt == FP8B_E5M2 &&
            p.ep.cq_mode == FP8B_RNE && p.dbg == 0 && !(el && el[0] == '0'))
            fn = conv_halo_kernel<ES, CB, BN, 3, 1>;
    }
    ensure_smem_attr((const void*)fn, (int)pl.smem);
    const int sms = device_sm_count();
    const int grid = p.ntiles < sms ? p.ntiles : sms;
    fn<<<grid, 64 + 32 * pl.ew, pl.smem, st>>>(tx, tw, ty, tq, p, pl.slab, pl.nstages);
    return cudaGetLastError() == cudaSuccess ? FP8B_OK : FP8B_ECUDA;
}

// ---------------------------------------------------------------------------
// wgrad (conv2d_backward_weights_fp8, kernels.cpp:202-253) for E5M2 with
// C = F = 64, k = 3: dW_t[f, c] = sum_p e[p, f] * x[p + off_t, c] over the
// output pixels p. Per tile the CTA loads the same halo slab as fprop plus the
// tile's error rows e (zero at the pad columns / beyond the image, TMA
// out-of-bounds fill), and accumulates, for every pair of taps (t1, t2),
//   D[128, F] = [x_t1 ; x_t2]^T . e
// in one M=128 MMA chain: the A operand's two 64-row halves are the slab seen
// from rows off_t1 and off_t2 (MN-major, the halves LBO = (off_t2 - off_t1) *
// 64 bytes apart), B is the error tile (MN-major). The 5 pair accumulators
// (320 TMEM columns) stay resident across all of the CTA's tiles; at the end
// they are written as the CTA's FP32 partial [tap][c][f], and a fixed-order
// sum over CTAs gives dW (deterministic).
struct WParams {
    int nimg, OH, OW, Wp, R, SR, pad, F, C;
    int tiles_per_img, ntiles;
    float* ws;  // [grid][9][C][F] partials
};

template <int ES>
__global__ void __launch_bounds__(192, 1)
    conv_halo_wgrad_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmE,
                           const WParams p, uint32_t slab_bytes, uint32_t stage_bytes, int nstages) {
    constexpr int KS = 3, TAPS = 9, NG = 5;  // tap pairs (0,1) (2,3) (4,5) (6,7) (8,-)
    constexpr int CE = 64 / ES;              // channels (= filters) per 64-byte row
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + (uint32_t)nstages * stage_bytes);
    uint64_t* empty_bar = full_bar + nstages;
    uint64_t* done_bar = empty_bar + nstages;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done_bar + 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmX)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmE)) : "memory");
        for (int s = 0; s < nstages; ++s) {
            mbar_init(full_bar + s, 1);
            mbar_init(empty_bar + s, 1);
        }
        mbar_init(done_bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem_base = *tmem_slot;
    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x) {
                const int n = tile / p.tiles_per_img;
                const int oh0 = (tile - n * p.tiles_per_img) * p.R;
                mbar_wait(empty_bar + stage, phase ^ 1);
                uint8_t* st = smem + stage * stage_bytes;
                mbar_expect_tx(full_bar + stage, (uint32_t)p.SR * p.Wp * 64 + (uint32_t)p.R * p.Wp * 64);
                tma_load_4d(&tmX, st, full_bar + stage, 0, -p.pad, oh0 - p.pad, n);
                tma_load_4d(&tmE, st + slab_bytes, full_bar + stage, 0, 0, oh0, n);
                if (++stage == nstages) { stage = 0; phase ^= 1; }
            }
        }
    } else if (warp == 1) {
        const uint32_t leader = elect_one();
        uint32_t idesc = (1u << 4);
        if (ES == 1) idesc |= (1u << 7) | (1u << 10);
        idesc |= (1u << 15) | (1u << 16);  // A and B MN-major
        idesc |= (uint32_t)(CE >> 3) << 17;  // N = F
        idesc |= (uint32_t)(128 >> 4) << 24;
        // K (pixels) advances 32 / ES rows of 64 bytes per MMA (swizzle atoms of 8 rows, SBO 512)
        uint32_t lbo[NG], aoff[NG];
#pragma unroll
        for (int g = 0; g < NG; ++g) {
            const int t1 = 2 * g, t2 = 2 * g + 1 < TAPS ? 2 * g + 1 : 2 * g;
            const int o1 = (t1 / KS) * p.Wp + t1 % KS, o2 = (t2 / KS) * p.Wp + t2 % KS + (t2 == t1 ? 1 : 0);
            aoff[g] = (uint32_t)o1 * 64u;
            lbo[g] = (uint32_t)(o2 - o1) * 64u;
        }
        int stage = 0;
        uint32_t phase = 0;
        bool first = true;
        for (int tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x) {
            mbar_wait(full_bar + stage, phase);
            fence_after();
            const uint32_t s0 = smem_u32(smem + stage * stage_bytes);
            const uint32_t e0 = s0 + slab_bytes;
#pragma unroll
            for (int g = 0; g < NG; ++g) {
#pragma unroll
                for (int j = 0; j < 4 * ES; ++j) {  // K = 32 / ES pixels per MMA
                    const uint64_t ad = umma_desc(s0 + aoff[g] + (uint32_t)j * (2048u / ES), lbo[g], 512, 4);
                    const uint64_t bd = umma_desc(e0 + (uint32_t)j * (2048u / ES), 64, 512, 4);
                    mma_p<ES>(tmem_base + (uint32_t)(g * 64), ad, bd, idesc, (first && j == 0) ? 0u : 1u, leader);
                }
            }
            first = false;
            umma_commit_p(empty_bar + stage, leader);
            if (++stage == nstages) { stage = 0; phase ^= 1; }
        }
        umma_commit_p(done_bar, leader);
    } else {
        // epilogue warps 2-5 (TMEM lane quarters): TMEM lane l of pair g is
        // channel l % 64 of tap 2g + l / 64
        const int quarter = warp & 3;
        const int row = quarter * 32 + lane;
        const int half = row >> 6, c = row & 63;
        mbar_wait(done_bar, 0);
        fence_after();
        const bool any = p.ntiles > (int)blockIdx.x;
#pragma unroll 1
        for (int g = 0; g < NG; ++g) {
            const int t = 2 * g + half;
#pragma unroll
            for (int cc = 0; cc < CE / 32; ++cc) {
                uint32_t v[32];
                tmem_ld32(tmem_base + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(g * 64 + cc * 32), v);
                if (t < TAPS && c < p.C) {
                    float* dst = p.ws + (((size_t)blockIdx.x * TAPS + t) * p.C + c) * p.F + cc * 32;
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        reinterpret_cast<float4*>(dst)[q] =
                            any ? make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]),
                                              __uint_as_float(v[4 * q + 2]), __uint_as_float(v[4 * q + 3]))
                                : make_float4(0.f, 0.f, 0.f, 0.f);
                }
            }
        }
    }
    fence_before();
    __syncthreads();
    if (warp == 1) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512));
    }
}

// dw [f, kh, kw, c] = sum over CTAs b (ascending) of ws[b][t][c][f], then the
// layer's Q(dW) node when asked for (one launch fewer than sum + quantize).
__global__ void __launch_bounds__(256) conv_halo_wgrad_sum(const float* __restrict__ ws,
                                                           float* __restrict__ dw, int nb, int C,
                                                           int F, QNode q) {
    const int total = 9 * C * F;
    uint32_t co = 0, cu = 0, cn = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
        const int f = i % F, tc = i / F;  // ws order: [t][c][f]
        float s = 0.f;
        for (int b = 0; b < nb; ++b) s = __fadd_rn(s, ws[(size_t)b * total + i]);
        const int t = tc / C, c = tc - t * C;
        const size_t o = ((size_t)f * 9 + t) * C + c;
        dw[o] = s;
        if (q.codes) qnode_store(q, (int64_t)o, s, co, cu, cn);
    }
    if (q.codes && q.counters) flush_counters<256>(co, cu, cn, q.counters);
}

}  // namespace halo
}  // namespace tc

bool conv_halo_supported(int es, int64_t n, int64_t h, int64_t w, int64_t c, int64_t f, int k,
                         int pad) {
    const char* e = getenv("FP8B_CONV_HALO");
    if (e && e[0] == '0') return false;
    tc::halo::Plan pl;
    return tc::halo::plan_for(n, h, w, c, f, k, pad, es, pl);
}

// fprop over NHWC x [n, h, w, c] and KRSC w [f, k, k, c] -> y [n, oh, ow, f]
// (stride 1). Returns FP8B_ENOTSUP when the geometry is not covered.
int launch_conv_halo(const void* x, const void* wt, float* y, int es, int64_t n, int64_t h,
                     int64_t w, int64_t c, int64_t f, int k, int pad, const fp8b_conv_t& g,
                     cudaStream_t st) {
    using namespace tc::halo;
    Plan pl;
    if (!conv_halo_supported(es, n, h, w, c, f, k, pad) ||
        !plan_for(n, h, w, c, f, k, pad, es, pl, y != nullptr, g.yq ? g.yq_fmt : -1))
        return FP8B_ENOTSUP;
    if ((uintptr_t)x % 16 || (uintptr_t)wt % 16) return FP8B_ENOTSUP;
    CUtensorMap tx, tw;
    if (!make_slab_map(&tx, x, es, n, h, w, c, pl.wp, pl.sr)) return FP8B_ENOTSUP;
    const CUtensorMapSwizzle swz = pl.cb == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
    // weights [f, k*k*c]: box {c, bn} (rows f >= F of the last box are zero-filled)
    if (!tc::make_map(&tw, wt, es, (uint64_t)(k * k * c), (uint64_t)f, (uint32_t)c, (uint32_t)pl.bn, swz))
        return FP8B_ENOTSUP;
    HParams p{};
    const int64_t oh = h + 2 * pad - k + 1, ow = w + 2 * pad - k + 1;
    p.M = n * oh * ow;
    p.N = f;
    p.ep = EpiArgs{y, nullptr, g.yq, g.yq_fmt, g.yq_mode, g.yq_seed, g.yq_saturate, g.yq_counters};
    p.nimg = (int)n; p.OH = (int)oh; p.OW = (int)ow;
    p.Wp = pl.wp; p.R = pl.r; p.SR = pl.sr; p.k = k; p.pad = pad;
    p.tiles_per_img = (int)((oh + pl.r - 1) / pl.r);
    p.ntiles = (int)(n * p.tiles_per_img);
    const char* bo = getenv("FP8B_CONV_HALO_BO");
    p.bo_mode = bo ? atoi(bo) : 0;
    const char* dbg = getenv("FP8B_CONV_HALO_DBG");
    p.dbg = dbg ? atoi(dbg) : 0;
    p.stg = pl.stg; p.c_off = pl.c_off; p.q_off = pl.q_off;
    p.c_nbuf = pl.c_nbuf; p.q_nbuf = pl.q_nbuf; p.ew = pl.ew;
    p.wlog = 0;
    while ((1 << p.wlog) < pl.wp) ++p.wlog;
    CUtensorMap ty, tq;
    memset(&ty, 0, sizeof(ty));
    memset(&tq, 0, sizeof(tq));
    p.c_tma = y != nullptr;
    if (y && !make_out_map(&ty, y, 4, n, oh, ow, f, 32, pl.wp)) return FP8B_ENOTSUP;
    p.q_tma = g.yq != nullptr;
    if (g.yq) {
        const int qes = g.yq_fmt == FP8B_E5M2 ? 1 : 2;
        p.qg = pl.qg;  // 64- or 128-byte code rows
        if (p.qg * 32 * qes < 32) return FP8B_ENOTSUP;
        if (!make_out_map(&tq, g.yq, qes, n, oh, ow, f, p.qg * 32, pl.wp)) return FP8B_ENOTSUP;
    }
    if (es == 1) {
        if (pl.cb == 64) {
            if (pl.bn == 64) return run<1, 64, 64>(tx, tw, ty, tq, p, pl, st);
            if (pl.bn == 128) return run<1, 64, 128>(tx, tw, ty, tq, p, pl, st);
            return run<1, 64, 256>(tx, tw, ty, tq, p, pl, st);
        }
        if (pl.bn == 64) return run<1, 128, 64>(tx, tw, ty, tq, p, pl, st);
        if (pl.bn == 128) return run<1, 128, 128>(tx, tw, ty, tq, p, pl, st);
        return run<1, 128, 256>(tx, tw, ty, tq, p, pl, st);
    }
    if (pl.cb == 64) {
        if (pl.bn == 64) return run<2, 64, 64>(tx, tw, ty, tq, p, pl, st);
        if (pl.bn == 128) return run<2, 64, 128>(tx, tw, ty, tq, p, pl, st);
        return run<2, 64, 256>(tx, tw, ty, tq, p, pl, st);
    }
    if (pl.bn == 64) return run<2, 128, 64>(tx, tw, ty, tq, p, pl, st);
    if (pl.bn == 128) return run<2, 128, 128>(tx, tw, ty, tq, p, pl, st);
    return run<2, 128, 256>(tx, tw, ty, tq, p, pl, st);
}

bool conv_halo_wgrad_supported(int es, int64_t n, int64_t h, int64_t w, int64_t c, int64_t f, int k,
                               int pad) {
    const char* e = getenv("FP8B_CONV_HALO");
    if (e && e[0] == '0') return false;
    // E5M2 only: a tap half of the M=128 accumulator is one 64-byte row of 64
    // channels (FP16 rows hold 32, which would need 4 taps per accumulator)
    if (es != 1 || k != 3 || c != 64 || f != 64 || pad < 0 || pad > 2) return false;
    if (w + 2 * pad > 128 || h + 2 * pad - k + 1 < 1 || w + 2 * pad - k + 1 < 1) return false;
    return n * h * w < ((int64_t)1 << 31);
}

// wgrad over NHWC x [n, h, w, c] and e [n, oh, ow, f] -> dw [f, 3, 3, c] (FP32).
int launch_conv_halo_wgrad(const void* x, const void* e, float* dw, int es, int64_t n, int64_t h,
                           int64_t w, int64_t c, int64_t f, int k, int pad, cudaStream_t st, int* nl,
                           const fp8b_conv_t* gq) {
    using namespace tc::halo;
    if (!conv_halo_wgrad_supported(es, n, h, w, c, f, k, pad)) return FP8B_ENOTSUP;
    if ((uintptr_t)x % 16 || (uintptr_t)e % 16 || !dw) return FP8B_ENOTSUP;
    const int64_t oh = h + 2 * pad - k + 1, ow = w + 2 * pad - k + 1;
    int wp = 1;
    while (wp < w + 2 * pad) wp <<= 1;
    const int r = 128 / wp;
    const int sr = (128 + (k - 1) * (wp + 1) + wp - 1) / wp;
    CUtensorMap tx, te;
    if (!make_slab_map(&tx, x, es, n, h, w, c, wp, sr)) return FP8B_ENOTSUP;
    {
        tc::EncodeTiledFn enc = tc::get_encode();
        if (!enc) return FP8B_ENOTSUP;
        cuuint64_t dims[4] = {(cuuint64_t)f, (cuuint64_t)ow, (cuuint64_t)oh, (cuuint64_t)n};
        cuuint64_t strides[3] = {(cuuint64_t)(f * es), (cuuint64_t)(ow * f * es), (cuuint64_t)(oh * ow * f * es)};
        cuuint32_t box[4] = {(cuuint32_t)f, (cuuint32_t)wp, (cuuint32_t)r, 1};
        cuuint32_t estr[4] = {1, 1, 1, 1};
        if (enc(&te, es == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_UINT16, 4,
                const_cast<void*>(e), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return FP8B_ENOTSUP;
    }
    const uint32_t slab = (((uint32_t)sr * wp * 64) + 1023u) & ~1023u;
    const uint32_t stage = slab + ((((uint32_t)r * wp * 64) + 1023u) & ~1023u);
    int nstages = (int)((232448u - 2048u) / stage);
    if (nstages > 4) nstages = 4;
    if (nstages < 2) return FP8B_ENOTSUP;
    const uint32_t smem = 1024 + (uint32_t)nstages * stage + 256;
    WParams p{};
    p.nimg = (int)n; p.OH = (int)oh; p.OW = (int)ow; p.Wp = wp; p.R = r; p.SR = sr; p.pad = pad;
    p.F = (int)f; p.C = (int)c;
    p.tiles_per_img = (int)((oh + r - 1) / r);
    p.ntiles = (int)(n * p.tiles_per_img);
    const int sms = device_sm_count();
    const int grid = p.ntiles < sms ? p.ntiles : sms;
    const size_t part = (size_t)9 * c * f;
    if (cudaMallocAsync(&p.ws, (size_t)grid * part * sizeof(float), st) != cudaSuccess) return FP8B_ECUDA;
    auto fn = es == 1 ? conv_halo_wgrad_kernel<1> : conv_halo_wgrad_kernel<2>;
    ensure_smem_attr((const void*)fn, (int)smem);
    fn<<<grid, 192, smem, st>>>(tx, te, p, slab, stage, nstages);
    int b = (int)((part + 255) / 256);
    if (b > 4 * sms) b = 4 * sms;
    QNode q{};
    if (gq && gq->yq)
        q = QNode{gq->yq, gq->yq_fmt, gq->yq_mode, gq->yq_seed, gq->yq_saturate, gq->yq_counters};
    conv_halo_wgrad_sum<<<b, 256, 0, st>>>(p.ws, dw, grid, (int)c, (int)f, q);
    cudaFreeAsync(p.ws, st);
    *nl = 2;
    return cudaGetLastError() == cudaSuccess ? FP8B_OK : FP8B_ECUDA;
}

}  // namespace fp8b
