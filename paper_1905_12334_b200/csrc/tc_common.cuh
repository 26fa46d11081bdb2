// tc_common.cuh -- tcgen05 / TMA / mbarrier helpers shared by the tensor-core
// kernels (gemm_tc.cu, conv_tc.cu), the fused GEMM epilogue, and the host-side
// tensor-map encoders.
#pragma once
#include <cstdlib>
#include <cuda.h>

#include <mutex>

#include "common.cuh"
#include "kernels.cuh"

namespace fp8b {
namespace tc {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t a = smem_u32(bar);
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(a),
        "r"(parity)
        : "memory");
}

// Non-blocking probe: has the phase with this parity completed?
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
        "selp.u32 %0, 1, 0, P1;\n"
        "}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

// Busy-poll variant (test_wait: never suspends the thread between polls).
__device__ __forceinline__ void mbar_wait_spin(uint64_t* bar, uint32_t parity) {
    const uint32_t a = smem_u32(bar);
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.test_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(a),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void tma_load_2d(const CUtensorMap* tm, void* dst, uint64_t* bar,
                                            int32_t c0, int32_t c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}

__device__ __forceinline__ void fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}

using fp8b::launch_pdl;  // common.cuh

// UMMA shared-memory matrix descriptor, version 1 (sm_100); layout 2 =
// SWIZZLE_128B (default), 4 = SWIZZLE_64B.
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo,
                                              uint32_t layout = 2) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= 1ull << 46;  // descriptor version (Blackwell)
    d |= (uint64_t)layout << 61;
    return d;
}

template <int ES>
__device__ __forceinline__ void mma(uint32_t tmem_d, uint64_t ad, uint64_t bd, uint32_t idesc,
                                    uint32_t accum) {
    if (ES == 1) {
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
            "l"(ad), "l"(bd), "r"(idesc), "r"(accum));
    } else {
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
            "l"(ad), "l"(bd), "r"(idesc), "r"(accum));
    }
}

// Predicated forms for an issue loop run by the whole warp (operands uniform,
// one elected lane issuing).
template <int ES>
__device__ __forceinline__ void mma_p(uint32_t tmem_d, uint64_t ad, uint64_t bd, uint32_t idesc,
                                      uint32_t accum, uint32_t issue) {
    if (ES == 1) {
        asm volatile(
            "{\n.reg .pred p, q;\nsetp.ne.b32 p, %4, 0;\nsetp.ne.b32 q, %5, 0;\n"
            "@q tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
            "l"(ad), "l"(bd), "r"(idesc), "r"(accum), "r"(issue));
    } else {
        asm volatile(
            "{\n.reg .pred p, q;\nsetp.ne.b32 p, %4, 0;\nsetp.ne.b32 q, %5, 0;\n"
            "@q tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
            "l"(ad), "l"(bd), "r"(idesc), "r"(accum), "r"(issue));
    }
}
__device__ __forceinline__ void umma_commit_p(uint64_t* bar, uint32_t issue) {
    asm volatile(
        "{\n.reg .pred q;\nsetp.ne.b32 q, %1, 0;\n"
        "@q tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(
            smem_u32(bar)),
        "r"(issue)
        : "memory");
}
// One lane of the warp (elect.sync): 1 there, 0 elsewhere.
__device__ __forceinline__ uint32_t elect_one() {
    uint32_t e;
    asm volatile("{\n.reg .pred P;\nelect.sync _|P, 0xffffffff;\nselp.u32 %0, 1, 0, P;\n}\n" : "=r"(e));
    return e;
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
          "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
          "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
          "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Issue-only TMEM load (no wait): several chunks can be in flight before one
// tmem_wait_regs(), which also ties the destination registers to the wait so
// the compiler cannot hoist their uses above it.
__device__ __forceinline__ void tmem_ld32_nowait(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
          "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
          "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
          "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_regs_after_wait(uint32_t (&v)[32]) {
    asm volatile(""
                 : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]),
                   "+r"(v[6]), "+r"(v[7]), "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]),
                   "+r"(v[12]), "+r"(v[13]), "+r"(v[14]), "+r"(v[15]), "+r"(v[16]), "+r"(v[17]),
                   "+r"(v[18]), "+r"(v[19]), "+r"(v[20]), "+r"(v[21]), "+r"(v[22]), "+r"(v[23]),
                   "+r"(v[24]), "+r"(v[25]), "+r"(v[26]), "+r"(v[27]), "+r"(v[28]), "+r"(v[29]),
                   "+r"(v[30]), "+r"(v[31])
                 :
                 : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() {
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Grouped rasterisation: walk the tile grid in column bands of GROUP_N tiles so
// the tiles in flight at once (one per SM / SM pair) share a few A row-panels
// and B column-panels that stay resident in L2.
constexpr int GROUP_N = 8;
__device__ __forceinline__ void tile_coords(int tile, int tiles_m, int tiles_n, int& tm, int& tn) {
    const int band = tile / (GROUP_N * tiles_m);
    const int first_n = band * GROUP_N;
    const int width = min(GROUP_N, tiles_n - first_n);
    const int r = tile - band * GROUP_N * tiles_m;
    tm = r / width;
    tn = first_n + r % width;
}

// TMA-store epilogue. Each epilogue warp owns two 4 KB staging buffers used as
// a ring: an output chunk (32 rows x 32 columns; FP32 = 128 B per row, FP16
// codes 64 B, E5M2 codes 32 B) is written with st.shared.v4 in the swizzle of
// its tensor map (span = row bytes) and handed to the TMA engine with one
// cp.async.bulk.tensor store; rows/columns outside the tensor are clipped by
// TMA. Before a buffer is refilled its previous store must have read it
// (wait_group.read 1: only the other buffer's store may still be pending).
constexpr uint32_t EPI_STAGE_BYTES = 4 * 2 * 4096;  // 4 warps x 2 buffers

struct EpiTma {
    const CUtensorMap* c;  // FP32 output map (32x32 boxes, 128B swizzle) or null
    const CUtensorMap* q;  // code output map (qg*32 x 32 boxes, row-span swizzle) or null
    uint8_t* sbuf;         // this warp's 8 KB of staging
    uint32_t* nst;         // this warp's buffer counter
    int64_t row0;          // first row of the warp's 32-row slab
    int lane;
    int z;                 // 3-D store coordinate (split index) or -1
    int qg;                // code chunks per store (row span = qg * 32 * code bytes)
    int qpos;              // chunks already staged in the open code group
    uint8_t* qbuf;         // the open code group's buffer
    int nbuf = 2;          // staging buffers of this warp (2: ring of 4 KB buffers; 1: one)
};

__device__ __forceinline__ void bulk_wait_read1() {
    asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read0() {
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// Next ring buffer, once its previous store has read it.
__device__ __forceinline__ uint8_t* stage_acquire(uint8_t* sbuf, uint32_t& nst, int lane,
                                                  int nbuf = 2) {
    if (nbuf == 1) {
        if (lane == 0) bulk_wait_read0();
        __syncwarp();
        return sbuf;
    }
    uint8_t* buf = sbuf + (nst++ & 1) * 4096;
    if (lane == 0) bulk_wait_read1();
    __syncwarp();
    return buf;
}
// NW words of this lane's row at byte offset OFF of a SPAN-byte row, in the
// map's swizzle (16-byte chunk index XOR the row's phase).
template <int SPAN, int NW>
__device__ __forceinline__ void stage_write(uint8_t* buf, int off, const uint32_t* w, int lane) {
    const uint32_t base = smem_u32(buf) + lane * SPAN;
    const uint32_t x = (uint32_t)(lane / (128 / SPAN)) & (SPAN / 16 - 1);
#pragma unroll
    for (int j = 0; j < NW / 4; ++j) {
        const uint32_t a = base + ((((uint32_t)off >> 4) + j) ^ x) * 16u;
        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(w[4 * j]),
                     "r"(w[4 * j + 1]), "r"(w[4 * j + 2]), "r"(w[4 * j + 3])
                     : "memory");
    }
}
// Hand the warp's staged box to the TMA engine.
__device__ __forceinline__ void stage_flush(const CUtensorMap* tm, uint8_t* buf, int lane, int32_t col0,
                                            int32_t row0, int32_t z = -1) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) {
        if (z < 0)
            asm volatile(
                "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                    reinterpret_cast<uint64_t>(tm)),
                "r"(smem_u32(buf)), "r"(col0), "r"(row0)
                : "memory");
        else
            asm volatile(
                "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                    reinterpret_cast<uint64_t>(tm)),
                "r"(smem_u32(buf)), "r"(col0), "r"(row0), "r"(z)
                : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
}
// One 32-row x 128-byte box (32 FP32 columns) per call.
__device__ __forceinline__ void stage_store_f32(const CUtensorMap* tm, uint8_t* sbuf, uint32_t& nst,
                                                const uint32_t* w, int lane, int32_t col0,
                                                int32_t row0, int32_t z = -1, int nbuf = 2) {
    uint8_t* buf = stage_acquire(sbuf, nst, lane, nbuf);
    stage_write<128, 32>(buf, 0, w, lane);
    stage_flush(tm, buf, lane, col0, row0, z);
}
// Codes: chunks accumulate into one box of qg*32 columns (a 64- or 128-byte row)
// before one store; `last` closes a partial group at the end of a tile.
template <int ES>
__device__ __forceinline__ void stage_codes(EpiTma* t, const uint32_t* w, int64_t col0, bool last) {
    constexpr int NW = 8 * ES;  // 32 codes of ES bytes
    if (t->qpos == 0) t->qbuf = stage_acquire(t->sbuf, *t->nst, t->lane, t->nbuf);
    const int span = t->qg * 32 * ES;
    if (span == 128) stage_write<128, NW>(t->qbuf, t->qpos * 32 * ES, w, t->lane);
    else stage_write<64, NW>(t->qbuf, t->qpos * 32 * ES, w, t->lane);
    if (++t->qpos == t->qg || last) {
        stage_flush(t->q, t->qbuf, t->lane, (int32_t)(col0 - 32 * (t->qpos - 1)), (int32_t)t->row0);
        t->qpos = 0;
    }
}

// Lean E5M2 RNE output node for one 32-column chunk (bias already added):
// paired hardware cvt packed straight into words; overflow / NaN screened on
// the packed codes, four at a time (magnitude bytes m <= 0x7F):
//   m >= 0x7B  <=>  bit 7 of m + 5: the max-normal code (possibly from an input
//                   above 57344, which the reference overflows), Inf or NaN ->
//                   per-element fix-ups (rare);
//   m == 0     <=>  bit 7 of m + 0x7F clear: the code rounded to zero; an
//                   underflow unless the input was +-0.
// Counters cover real rows (live) and columns (< nvalid) only.
__device__ __forceinline__ void lean_e5m2_codes(const float (&y)[32], uint32_t (&w)[8], bool sat,
                                                bool live, int nvalid, uint32_t& co, uint32_t& cu,
                                                uint32_t& cn) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        w[q] = cvt_e5m2x4(y[4 * q], y[4 * q + 1], y[4 * q + 2], y[4 * q + 3]);
    }
    // one screen for both: bit 7 of m + 5 is set iff m >= 0x7B, bit 7 of m + 0x7F
    // is clear iff m == 0 (no carries between bytes: m <= 0x7F); 4 ops per word
    uint32_t flag = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const uint32_t m = w[q] & 0x7F7F7F7Fu;
        flag |= (m + 0x05050505u) | ~(m + 0x7F7F7F7Fu);
    }
    if (!(flag & 0x80808080u)) return;
    uint32_t big = 0, zero = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const uint32_t m = w[q] & 0x7F7F7F7Fu;
        big |= (m + 0x05050505u) & 0x80808080u;
        zero |= ~(m + 0x7F7F7F7Fu) & 0x80808080u;
    }
    if (big) {  // an output at the max code, overflowing or NaN in this row chunk
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            const uint32_t hw = (w[j >> 2] >> (8 * (j & 3))) & 0xFFu;
            uint32_t b = 0, nn = 0, uu = 0;
            const uint32_t c = fix_rne<2>(hw, __float_as_uint(y[j]), sat, b, nn, uu);
            w[j >> 2] = (w[j >> 2] & ~(0xFFu << (8 * (j & 3)))) | (c << (8 * (j & 3)));
            if (live && j < nvalid) { co += b - nn; cn += nn; }
        }
    }
    if (zero && live) {
#pragma unroll
        for (int j = 0; j < 32; ++j)
            cu += (((w[j >> 2] >> (8 * (j & 3))) & 0x7Fu) == 0u) &&
                  (__float_as_uint(y[j]) & 0x7FFFFFFFu) != 0u && j < nvalid;
    }
}

// Epilogue of one 32-column chunk; one row per lane. With TMA stores active
// (t.c or t.q set) the whole warp must call it -- rows >= M included, TMA clips
// them and the counters skip them; otherwise rows >= M return early.
template <class P>
__device__ __forceinline__ void epilogue_chunk(const P& p, int64_t row, int64_t col0,
                                               uint32_t (&v)[32], uint32_t& co, uint32_t& cu,
                                               uint32_t& cn, EpiTma* tm_ = nullptr,
                                               bool last = false) {
    const EpiArgs& ep = p.ep;
    float y[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) y[j] = __uint_as_float(v[j]);
    const bool full = col0 + 32 <= p.N;
    const bool live = row < p.M;
    if (ep.bias) {
#pragma unroll
        for (int j = 0; j < 32; ++j)
            if (full || col0 + j < p.N) y[j] = __fadd_rn(y[j], __ldg(ep.bias + col0 + j));
    }
    const bool c_tma = tm_ && tm_->c, q_tma = tm_ && tm_->q;
    if (c_tma) {
        uint32_t w[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) w[j] = __float_as_uint(y[j]);
        stage_store_f32(tm_->c, tm_->sbuf, *tm_->nst, w, tm_->lane, (int32_t)col0,
                        (int32_t)tm_->row0, tm_->z, tm_->nbuf);
    }
    if (!live && !q_tma) return;
    const int64_t base = row * p.N + col0;
    if (ep.c && !c_tma && live) {
        if (full && (p.N % 4 == 0) && ((uintptr_t)ep.c % 16 == 0)) {
            float4* dst = reinterpret_cast<float4*>(ep.c + base);
#pragma unroll
            for (int j = 0; j < 8; ++j)
                dst[j] = make_float4(y[4 * j], y[4 * j + 1], y[4 * j + 2], y[4 * j + 3]);
        } else {
            for (int j = 0; j < 32; ++j)
                if (col0 + j < p.N) ep.c[base + j] = y[j];
        }
    }
    if (ep.cq && ep.cq_mode == FP8B_RNE && ep.cq_fmt == FP8B_E5M2) {
        uint32_t w[8];
        const int nvalid = full ? 32 : (int)(p.N - col0);
        lean_e5m2_codes(y, w, ep.cq_sat != 0, live, nvalid, co, cu, cn);
        if (q_tma) {
            stage_codes<1>(tm_, w, col0, last);
        } else if (live) {
            uint8_t* dst = reinterpret_cast<uint8_t*>(ep.cq) + base;
            if (full && (p.N % 16 == 0) && ((uintptr_t)ep.cq % 16 == 0)) {
                uint4* d4 = reinterpret_cast<uint4*>(dst);
                d4[0] = make_uint4(w[0], w[1], w[2], w[3]);
                d4[1] = make_uint4(w[4], w[5], w[6], w[7]);
            } else {
#pragma unroll
                for (int j = 0; j < 32; ++j)
                    if (j < nvalid) dst[j] = (uint8_t)(w[j >> 2] >> (8 * (j & 3)));
            }
        }
    } else if (ep.cq) {
        uint32_t code[32];
        const bool sat = ep.cq_sat != 0;
        const bool cnt = live && full;  // counters: real rows, whole chunk in range
        if (ep.cq_mode == FP8B_RNE && ep.cq_fmt == FP8B_E5M2) {
#pragma unroll
            for (int j = 0; j < 32; j += 2) {
                const uint32_t pr = cvt_e5m2x2(y[j], y[j + 1]);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    uint32_t b = 0, nn = 0, uu = 0;
                    code[j + h] = fix_rne<2>(h ? (pr >> 8) : (pr & 0xFFu),
                                             __float_as_uint(y[j + h]), sat, b, nn, uu);
                    if (cnt || (live && col0 + j + h < p.N)) { co += b - nn; cn += nn; cu += uu; }
                }
            }
        } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                int o, u, na;
                const int64_t gi = base + j;
                const uint32_t r16 = ep.cq_mode == FP8B_SR ? counter_r16(ep.cq_seed, (uint64_t)gi) : 0u;
                if (ep.cq_fmt == FP8B_E5M2)
                    code[j] = encode_int<2>(__float_as_uint(y[j]), ep.cq_mode, r16, sat, o, u, na);
                else
                    code[j] = encode_int<10>(__float_as_uint(y[j]), ep.cq_mode, r16, sat, o, u, na);
                if (cnt || (live && col0 + j < p.N)) { co += o; cu += u; cn += na; }
            }
        }
        if (ep.cq_fmt == FP8B_E5M2) {
            uint32_t w[8];
#pragma unroll
            for (int q = 0; q < 8; ++q)
                w[q] = code[4 * q] | (code[4 * q + 1] << 8) | (code[4 * q + 2] << 16) | (code[4 * q + 3] << 24);
            if (q_tma) {
                stage_codes<1>(tm_, w, col0, last);
            } else if (live) {
                uint8_t* dst = reinterpret_cast<uint8_t*>(ep.cq) + base;
                if (full && (p.N % 16 == 0) && ((uintptr_t)ep.cq % 16 == 0)) {
                    uint4* d4 = reinterpret_cast<uint4*>(dst);
                    d4[0] = make_uint4(w[0], w[1], w[2], w[3]);
                    d4[1] = make_uint4(w[4], w[5], w[6], w[7]);
                } else {
                    for (int j = 0; j < 32; ++j)
                        if (col0 + j < p.N) dst[j] = (uint8_t)code[j];
                }
            }
        } else {
            uint32_t w[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) w[q] = code[2 * q] | (code[2 * q + 1] << 16);
            if (q_tma) {
                stage_codes<2>(tm_, w, col0, last);
            } else if (live) {
                uint16_t* dst = reinterpret_cast<uint16_t*>(ep.cq) + base;
                if (full && (p.N % 8 == 0) && ((uintptr_t)ep.cq % 16 == 0)) {
                    uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
                    for (int j = 0; j < 4; ++j) d4[j] = make_uint4(w[4 * j], w[4 * j + 1], w[4 * j + 2], w[4 * j + 3]);
                } else {
                    for (int j = 0; j < 32; ++j)
                        if (col0 + j < p.N) dst[j] = (uint16_t)code[j];
                }
            }
        }
    }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static inline EncodeTiledFn get_encode() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    });
    return fn;
}

// 2-D map over a row-major [outer, inner] matrix of ES-byte elements.
static inline bool make_map(CUtensorMap* tm, const void* ptr, int es, uint64_t inner,
                            uint64_t outer, uint32_t box_inner, uint32_t box_outer,
                            CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
    // es: 1 = u8 codes, 2 = u16 codes, 4 = FP32
    EncodeTiledFn enc = get_encode();
    if (!enc) return false;
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {inner * (uint64_t)es};
    cuuint32_t box[2] = {box_inner, box_outer};
    cuuint32_t estr[2] = {1, 1};
    const CUtensorMapDataType dt = es == 1   ? CU_TENSOR_MAP_DATA_TYPE_UINT8
                                   : es == 2 ? CU_TENSOR_MAP_DATA_TYPE_UINT16
                                             : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    return enc(tm, dt, 2,
               const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
               swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}


// Store map for an FP32 [m, n] output (32x32 boxes, 128B swizzle); false when
// TMA cannot address it (row stride not a multiple of 16 bytes).
static inline bool make_c_map(CUtensorMap* tm, const float* c, int64_t m, int64_t n) {
    if (!c || (uintptr_t)c % 16 || (n * 4) % 16 || m <= 0 || n <= 0) return false;
    if (m > INT32_MAX || n > INT32_MAX) return false;
    return make_map(tm, c, 4, (uint64_t)n, (uint64_t)m, 32, 32);
}

// Store map for an [m, n] code output (E5M2 u8 / FP16 u16) whose boxes are 32
// rows x qg*32 columns with the swizzle of that row span (64 or 128 bytes);
// qg = min(tile_n / 32, 4 / code bytes). False when TMA cannot address it.
static inline int code_group(int fmt, int tile_n) {
    const int es = fmt == FP8B_E5M2 ? 1 : 2;
    const int g = tile_n / 32 < 4 / es ? tile_n / 32 : 4 / es;
    return g;
}
static inline bool make_q_map(CUtensorMap* tm, const void* q, int fmt, int64_t m, int64_t n,
                              int tile_n) {
    const int es = fmt == FP8B_E5M2 ? 1 : 2;
    const int qg = code_group(fmt, tile_n);
    const int span = qg * 32 * es;
    if (span != 64 && span != 128) return false;
    if (!q || (uintptr_t)q % 16 || (n * es) % 16 || m <= 0 || n <= 0) return false;
    if (m > INT32_MAX || n > INT32_MAX) return false;
    return make_map(tm, q, es, (uint64_t)n, (uint64_t)m, (uint32_t)(qg * 32), 32,
                    span == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B);
}

}  // namespace tc
}  // namespace fp8b
