// tc_common.cuh -- tcgen05 / TMA / mbarrier helpers shared by the tensor-core
// kernels (gemm_tc.cu, conv_tc.cu), the fused GEMM epilogue, and the host-side
// tensor-map encoders.
#pragma once
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

// Epilogue for one 32-column chunk of one row held in registers.
// TMA-store staging for the FP32 output: each epilogue warp owns two 4 KB
// buffers (32 rows x 32 FP32, 128B-swizzled to match the C tensor map), fills
// one per 32-column chunk with st.shared.v4 and hands it to the TMA engine with
// one cp.async.bulk.tensor store (rows/cols outside C are clipped by TMA).
constexpr uint32_t EPI_STAGE_BYTES = 4 * 2 * 4096;  // 4 warps x 2 buffers

__device__ __forceinline__ void bulk_wait_read1() {
    asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__device__ __forceinline__ void stage_store_c(const CUtensorMap* tmC, uint8_t* buf, const float (&y)[32],
                                              int lane, int32_t col0, int32_t row0, int32_t z = -1) {
    if (lane == 0) bulk_wait_read1();  // the buffer's previous store has read it
    __syncwarp();
    const uint32_t base = smem_u32(buf) + lane * 128;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const uint32_t a = base + ((uint32_t)(j ^ (lane & 7)) << 4);
        asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(y[4 * j]),
                     "f"(y[4 * j + 1]), "f"(y[4 * j + 2]), "f"(y[4 * j + 3])
                     : "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) {
        if (z < 0)
            asm volatile(
                "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                    reinterpret_cast<uint64_t>(tmC)),
                "r"(smem_u32(buf)), "r"(col0), "r"(row0)
                : "memory");
        else
            asm volatile(
                "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                    reinterpret_cast<uint64_t>(tmC)),
                "r"(smem_u32(buf)), "r"(col0), "r"(row0), "r"(z)
                : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
}

// Epilogue of one 32-column chunk; one row per lane. With tmC set, the whole
// warp must call it (rows >= M included: TMA clips them) and C goes out through
// stage_store_c; otherwise rows >= M return early.
template <class P>
__device__ __forceinline__ void epilogue_chunk(const P& p, int64_t row, int64_t col0,
                                               uint32_t (&v)[32], uint32_t& co, uint32_t& cu,
                                               uint32_t& cn, const CUtensorMap* tmC = nullptr,
                                               uint8_t* sbuf = nullptr, int64_t row0 = 0,
                                               int lane = 0) {
    const EpiArgs& ep = p.ep;
    float y[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) y[j] = __uint_as_float(v[j]);
    const bool full = col0 + 32 <= p.N;
    if (ep.bias) {
#pragma unroll
        for (int j = 0; j < 32; ++j)
            if (full || col0 + j < p.N) y[j] = __fadd_rn(y[j], __ldg(ep.bias + col0 + j));
    }
    if (tmC) stage_store_c(tmC, sbuf, y, lane, (int32_t)col0, (int32_t)row0);
    if (row >= p.M) return;
    const int64_t base = row * p.N + col0;
    if (ep.c && !tmC) {
        if (full && (p.N % 4 == 0)) {
            float4* dst = reinterpret_cast<float4*>(ep.c + base);
#pragma unroll
            for (int j = 0; j < 8; ++j)
                dst[j] = make_float4(y[4 * j], y[4 * j + 1], y[4 * j + 2], y[4 * j + 3]);
        } else {
            for (int j = 0; j < 32; ++j)
                if (col0 + j < p.N) ep.c[base + j] = y[j];
        }
    }
    if (ep.cq) {
        uint32_t code[32];
        const bool sat = ep.cq_sat != 0;
        if (ep.cq_mode == FP8B_RNE && ep.cq_fmt == FP8B_E5M2) {
#pragma unroll
            for (int j = 0; j < 32; j += 2) {
                const uint32_t pr = cvt_e5m2x2(y[j], y[j + 1]);
#pragma unroll
                for (int t = 0; t < 2; ++t) {
                    uint32_t b = 0, nn = 0, uu = 0;
                    code[j + t] = fix_rne<2>(t ? (pr >> 8) : (pr & 0xFFu),
                                             __float_as_uint(y[j + t]), sat, b, nn, uu);
                    if (full || col0 + j + t < p.N) { co += b - nn; cn += nn; cu += uu; }
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
                if (full || col0 + j < p.N) { co += o; cu += u; cn += na; }
            }
        }
        if (ep.cq_fmt == FP8B_E5M2) {
            uint8_t* dst = reinterpret_cast<uint8_t*>(ep.cq) + base;
            if (full && (p.N % 16 == 0)) {
                uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    uint32_t w[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int b = 16 * j + 4 * q;
                        w[q] = code[b] | (code[b + 1] << 8) | (code[b + 2] << 16) | (code[b + 3] << 24);
                    }
                    d4[j] = make_uint4(w[0], w[1], w[2], w[3]);
                }
            } else {
                for (int j = 0; j < 32; ++j)
                    if (col0 + j < p.N) dst[j] = (uint8_t)code[j];
            }
        } else {
            uint16_t* dst = reinterpret_cast<uint16_t*>(ep.cq) + base;
            if (full && (p.N % 8 == 0)) {
                uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    d4[j] = make_uint4(code[8 * j] | (code[8 * j + 1] << 16),
                                       code[8 * j + 2] | (code[8 * j + 3] << 16),
                                       code[8 * j + 4] | (code[8 * j + 5] << 16),
                                       code[8 * j + 6] | (code[8 * j + 7] << 16));
            } else {
                for (int j = 0; j < 32; ++j)
                    if (col0 + j < p.N) dst[j] = (uint16_t)code[j];
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

}  // namespace tc
}  // namespace fp8b
