// conv_tc.cu -- FP8B_GEMM_TENSOR for the conv family (kernels.cpp:106-253):
// implicit-GEMM convolutions on tcgen05, NHWC, stride 1, square kernels.
//
// No im2col buffer is ever materialised. The A operand of fprop is fetched by
// TMA in im2col mode (cp.async.bulk.tensor.4d...im2col): one load brings 128
// consecutive output pixels' input rows (walking W, then H, then N inside the
// conv's bounding box, zero-filled outside the image) for one filter tap
// (the 16-bit im2col offsets) and one channel block, already 64/128-byte
// swizzled for the UMMA descriptor. The K loop runs over (tap, channel block),
// B is the KRSC weight matrix [F, kH*kW*C] (K-major, plain 2-D TMA).
//   fprop  y[P, F]     = sum_{tap,c} X_tap[P, c] * W[F, tap, c]       (M = pixels)
//   dgrad  dx          = fprop(E, W') with W'[c,kh,kw,f] = W[f,kH-1-kh,kW-1-kw,c],
//                        pad' = kH-1-pad (one small flip kernel)
//   wgrad  dW[F, tap*C] = sum_P E[P, F] * X_tap[P, c]                (K = pixels)
//          A = E (MN-major, 2-D TMA), B = X_tap (MN-major, im2col TMA); split-K
//          over pixel blocks into an FP32 workspace, then a fixed-order sum.
// The warp roles, the smem ring, TMEM double buffering and the epilogue are
// those of gemm_tc.cu. Sums are reordered relative to the reference, so parity
// is the GEMM tolerance |y - y_exact| <= 1e-6 * (|x| * |w|) (tests/test_conv_gpu.py).
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "tc_common.cuh"

namespace fp8b {
namespace tc {
namespace cv {

// 2 warps (TMA producer, MMA issuer) + EW epilogue warps; EW = 8 doubles the
// epilogue's issue rate for short-K passes (1x1 convs), where the output Q node
// and stores, not the MMAs, set the pace.
template <int EW>
constexpr int threads_of() { return 64 + 32 * EW; }

struct CParams {
    int64_t M, N;  // output matrix (epilogue): fprop [P, F]; wgrad [F, taps*C]
    EpiArgs ep;
    int tiles_m, tiles_n, num_kb, splits;
    int cblocks;   // fprop: channel blocks per tap
    int C;         // channels of the im2col'd tensor
    int KW, pad, OH, OW;
    int c_tma;     // FP32 output goes through the TMA-store epilogue
    int q_tma;     // or the fused output codes (when no FP32 output is written)
    int qg;        // code chunks per TMA store
    float* ws;     // wgrad: split-K partials [splits][M][N]
};

typedef CUresult (*EncIm2colFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                const cuuint64_t*, const cuuint64_t*, const int*, const int*,
                                cuuint32_t, cuuint32_t, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion,
                                CUtensorMapFloatOOBfill);

static EncIm2colFn get_enc_im2col() {
    static EncIm2colFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncIm2colFn>(p);
    });
    return fn;
}

// im2col map over NHWC x [N, H, W, C] for a k x k kernel with padding pad:
// the bounding box spans the conv's output positions, one load = `pixels`
// output positions x `chans` channels.
static bool make_im2col(CUtensorMap* tm, const void* x, int es, int64_t n, int64_t h, int64_t w,
                        int64_t c, int k, int pad, int chans, int pixels, CUtensorMapSwizzle swz) {
    EncIm2colFn enc = get_enc_im2col();
    if (!enc) return false;
    cuuint64_t dims[4] = {(cuuint64_t)c, (cuuint64_t)w, (cuuint64_t)h, (cuuint64_t)n};
    cuuint64_t strides[3] = {(cuuint64_t)(c * es), (cuuint64_t)(w * c * es),
                             (cuuint64_t)(h * w * c * es)};
    int lower[2] = {-pad, -pad};
    int upper[2] = {pad - (k - 1), pad - (k - 1)};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    return enc(tm, es == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_UINT16, 4,
               const_cast<void*>(x), dims, strides, lower, upper, (cuuint32_t)chans,
               (cuuint32_t)pixels, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
           CUDA_SUCCESS;
}

__device__ __forceinline__ void tma_im2col_4d(const CUtensorMap* tm, void* dst, uint64_t* bar,
                                              int32_t c, int32_t w, int32_t h, int32_t n,
                                              uint16_t ow, uint16_t oh) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6}], [%2], {%7, %8};" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(smem_u32(bar)), "r"(c), "r"(w), "r"(h), "r"(n),
        "h"(ow), "h"(oh)
        : "memory");
}

// Compile-time geometry of one kernel instance. wgrad (MODE 1) tiles may hold
// MH x NH blocks of 128 x BN: the operand stream, not the MMAs, bounds the
// 128 x 128 tile (ncu: tensor pipe 37 % active, 32 KB of TMA rows per 271 MMA
// cycles), and a 256 x 256 tile moves half the bytes per MAC.
template <int ES, int MODE, int BN, int CB, int EW, int MH = 1, int NH = 1>
struct Geo {
    static constexpr uint32_t EPI_BYTES = (uint32_t)EW * 8192;  // 2 x 4 KB per epilogue warp
    static constexpr int KPIX = 128 / ES;            // wgrad: pixels per K block
    static constexpr uint32_t A_HALF = 128u * 128u;  // wgrad: one 128-row block of E
    static constexpr uint32_t B_HALF = (uint32_t)KPIX * CB;  // wgrad: one BN-wide block of X
    static constexpr uint32_t A_BYTES = MODE == 0 ? 128u * CB : MH * A_HALF;
    static constexpr uint32_t B_BYTES = MODE == 0 ? (uint32_t)BN * CB : NH * B_HALF;
    static constexpr uint32_t STAGE = A_BYTES + B_BYTES;
    static constexpr int BUDGET = 232448 - (int)EPI_BYTES - 1280;
    static constexpr int STAGES = (BUDGET / (int)STAGE) > 16 ? 16 : (BUDGET / (int)STAGE);
    static constexpr uint32_t SMEM = STAGES * STAGE + EPI_BYTES + 1024 + 256;
    static constexpr int ACC_COLS = MH * NH * BN;    // one accumulator set
    static constexpr int NACC = 2 * ACC_COLS <= 512 ? 2 : 1;
    static constexpr uint32_t TMEM_COLS = NACC * ACC_COLS < 32 ? 32 : NACC * ACC_COLS;
    static constexpr uint32_t SWZ_LAYOUT = CB == 128 ? 2u : 4u;  // UMMA layout code
    static constexpr uint32_t SBO = 8u * CB;                     // 8 rows of one swizzle atom
    static_assert(MODE == 1 || (MH == 1 && NH == 1), "block tiles are a wgrad feature");
    static_assert(STAGES >= 2, "ring too shallow");
};

// MODE 0: fprop (A = im2col X, K-major; B = W [F, taps*C], K-major).
// MODE 1: wgrad (A = E [P, F], MN-major; B = im2col X, MN-major), split-K.
// LEAN (fprop): compiled for fused E5M2 RNE codes only (no FP32 y, no bias),
// the layer step's output -- the generic epilogue's run-time cases cost ~200
// instructions per 32-column chunk on the short-K passes it paces.
template <int ES, int MODE, int BN, int CB, int EW, int MH = 1, int NH = 1, int LEAN = 0>
__global__ void __launch_bounds__(threads_of<EW>(), 1)
    conv_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmQ,
                   const CParams p) {
    using G = Geo<ES, MODE, BN, CB, EW, MH, NH>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + G::STAGES * G::STAGE + G::EPI_BYTES);
    uint64_t* empty_bar = full_bar + G::STAGES;
    uint64_t* tfull_bar = empty_bar + G::STAGES;
    uint64_t* tempty_bar = tfull_bar + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int CBE = CB / ES;      // channels per block
    constexpr int UK = 32 / ES;       // K elements per MMA
    const int ntiles = p.tiles_m * p.tiles_n;
    const int nitems = ntiles * p.splits;

    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
        for (int s = 0; s < G::STAGES; ++s) {
            mbar_init(full_bar + s, 1);
            mbar_init(empty_bar + s, 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(tfull_bar + a, 1);
            mbar_init(tempty_bar + a, EW);
        }
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
    const int pix_img = p.OH * p.OW;

    // item -> (tile, split) and its K-block range
    auto item_of = [&](int item, int& tm, int& tn, int& s, int& kb0, int& kb1) {
        if (p.splits == 1) {  // no integer divisions on the per-tile path of every warp
            s = 0; kb0 = 0; kb1 = p.num_kb;
            if (p.tiles_n == 1) { tm = item; tn = 0; }
            else tile_coords(item, p.tiles_m, p.tiles_n, tm, tn);
            return;
        }
        const int tile = item / p.splits;
        s = item - tile * p.splits;
        tile_coords(tile, p.tiles_m, p.tiles_n, tm, tn);
        kb0 = (int)((int64_t)p.num_kb * s / p.splits);
        kb1 = (int)((int64_t)p.num_kb * (s + 1) / p.splits);
    };

    uint32_t co = 0, cu = 0, cn = 0;
    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
                int tm, tn, s, kb0, kb1;
                item_of(item, tm, tn, s, kb0, kb1);
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(empty_bar + stage, phase ^ 1);
                    mbar_expect_tx(full_bar + stage, G::STAGE);
                    uint8_t* sA = smem + stage * G::STAGE;
                    uint8_t* sB = sA + G::A_BYTES;
                    if (MODE == 0) {
                        const int t = kb / p.cblocks, cb = kb - t * p.cblocks;
                        const int kh = t / p.KW, kw = t - kh * p.KW;
                        const int64_t P0 = (int64_t)tm * 128;
                        const int n = (int)(P0 / pix_img);
                        const int r = (int)(P0 - (int64_t)n * pix_img);
                        const int oh = r / p.OW, ow = r - oh * p.OW;
                        tma_im2col_4d(&tmA, sA, full_bar + stage, cb * CBE, ow - p.pad, oh - p.pad, n,
                                      (uint16_t)kw, (uint16_t)kh);
                        tma_load_2d(&tmB, sB, full_bar + stage, t * p.C + cb * CBE, tn * BN);
                    } else {
                        const int64_t P0 = (int64_t)kb * G::KPIX;
                        const int f0 = tm * 128 * MH;
#pragma unroll
                        for (int mh = 0; mh < MH; ++mh)
#pragma unroll
                            for (int j = 0; j < ES; ++j)  // 128 rows of F in 128-byte chunks
                                tma_load_2d(&tmA, sA + mh * G::A_HALF + j * (G::KPIX * 128),
                                            full_bar + stage, f0 + mh * 128 + j * (128 / ES), (int32_t)P0);
                        const int col = tn * (NH * BN);  // = t * C + c0 (a tile never straddles taps)
                        const int t = col / p.C, c0 = col - t * p.C;
                        const int kh = t / p.KW, kw = t - kh * p.KW;
                        const int n = (int)(P0 / pix_img);
                        const int r = (int)(P0 - (int64_t)n * pix_img);
                        const int oh = r / p.OW, ow = r - oh * p.OW;
#pragma unroll
                        for (int nh = 0; nh < NH; ++nh)
                            tma_im2col_4d(&tmB, sB + nh * G::B_HALF, full_bar + stage, c0 + nh * BN,
                                          ow - p.pad, oh - p.pad, n, (uint16_t)kw, (uint16_t)kh);
                    }
                    if (++stage == G::STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        {  // whole warp in uniform control flow; one elected lane issues
            const uint32_t leader = elect_one();
            uint32_t idesc = (1u << 4);
            if (ES == 1) idesc |= (1u << 7) | (1u << 10);
            if (MODE == 1) idesc |= (1u << 15) | (1u << 16);  // A and B MN-major
            idesc |= (uint32_t)((NH * BN) >> 3) << 17;
            idesc |= (uint32_t)(128 >> 4) << 24;
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t accphase = 0;
            for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
                int tm, tn, s, kb0, kb1;
                item_of(item, tm, tn, s, kb0, kb1);
                mbar_wait(tempty_bar + acc, accphase ^ 1);
                fence_after();
                const uint32_t d_tmem = tmem_base + (uint32_t)(acc * G::ACC_COLS);
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(full_bar + stage, phase);
                    fence_after();
                    const uint32_t a_base = smem_u32(smem + stage * G::STAGE);
                    const uint32_t b_base = a_base + G::A_BYTES;
                    if (MODE == 0) {
#pragma unroll
                        for (int k = 0; k < CB / 32; ++k) {
                            const uint64_t ad = umma_desc(a_base + 32 * k, 16, G::SBO, G::SWZ_LAYOUT);
                            const uint64_t bd = umma_desc(b_base + 32 * k, 16, G::SBO, G::SWZ_LAYOUT);
                            mma_p<ES>(d_tmem, ad, bd, idesc, (kb > kb0 || k) ? 1u : 0u, leader);
                        }
                    } else {
#pragma unroll
                        for (int k = 0; k < G::KPIX / UK; ++k) {
                            // B: NH blocks of BN columns, one swizzle atom each, LBO apart
                            const uint64_t bd = umma_desc(b_base + k * UK * CB, G::B_HALF, G::SBO,
                                                          G::SWZ_LAYOUT);
#pragma unroll
                            for (int mh = 0; mh < MH; ++mh) {
                                const uint64_t ad = umma_desc(a_base + mh * G::A_HALF + k * UK * 128,
                                                              G::KPIX * 128, 1024);
                                mma_p<ES>(d_tmem + (uint32_t)(mh * NH * BN), ad, bd, idesc,
                                          (kb > kb0 || k) ? 1u : 0u, leader);
                            }
                        }
                    }
                    umma_commit_p(empty_bar + stage, leader);
                    if (++stage == G::STAGES) { stage = 0; phase ^= 1; }
                }
                umma_commit_p(tfull_bar + acc, leader);
                if (++acc == G::NACC) { acc = 0; accphase ^= 1; }
            }
        }
    } else {
        const int quarter = warp & 3;             // TMEM lanes 32*quarter .. +31
        const int ew = warp - 2;                   // epilogue warp index
        constexpr int NC = NH * BN / 32;           // 32-column chunks per 128-row block
        constexpr int PER = NC / (EW / 4);         // chunks per warp (column halves when EW = 8)
        const int c_lo = (ew / 4) * PER;
        uint8_t* sbuf = smem + G::STAGES * G::STAGE + ew * 8192;
        uint32_t nst = 0;
        int acc = 0;
        uint32_t accphase = 0;
        for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
            int tm, tn, s, kb0, kb1;
            item_of(item, tm, tn, s, kb0, kb1);
            mbar_wait(tfull_bar + acc, accphase);
            fence_after();
#pragma unroll 1
            for (int mh = 0; mh < MH; ++mh) {
                const int64_t row0 = ((int64_t)tm * MH + mh) * 128 + quarter * 32;
                const int64_t row = row0 + lane;
                const uint32_t taddr = tmem_base + ((uint32_t)(quarter * 32) << 16) +
                                       (uint32_t)(acc * G::ACC_COLS + mh * NH * BN);
                EpiTma et{p.c_tma ? &tmC : nullptr, p.q_tma ? &tmQ : nullptr, sbuf, &nst,
                          row0, lane, -1, p.qg, 0, nullptr};
#pragma unroll 1
                for (int c = c_lo; c < c_lo + PER; ++c) {
                    uint32_t v[32];
                    tmem_ld32(taddr + c * 32, v);
                    const int64_t col0 = (int64_t)tn * (NH * BN) + c * 32;
                    if (col0 >= p.N) continue;
                    if (LEAN) {
                        const bool last = c == c_lo + PER - 1 || col0 + 32 >= p.N;
                        float y[32];
#pragma unroll
                        for (int j = 0; j < 32; ++j) y[j] = __uint_as_float(v[j]);
                        uint32_t w[8];
                        const int nvalid = col0 + 32 <= p.N ? 32 : (int)(p.N - col0);
                        lean_e5m2_codes(y, w, p.ep.cq_sat != 0, row < p.M, nvalid, co, cu, cn);
                        stage_codes<1>(&et, w, col0, last);
                        continue;
                    }
                    if (p.c_tma || p.q_tma) {
                        if (MODE == 0) {
                            const bool last = c == c_lo + PER - 1 || col0 + 32 >= p.N;
                            epilogue_chunk(p, row, col0, v, co, cu, cn, &et, last);
                        } else {
                            stage_store_f32(&tmC, sbuf, nst, v, lane, (int32_t)col0, (int32_t)row0, s);
                        }
                        continue;
                    }
                    if (row >= p.M) continue;
                    if (MODE == 0) {
                        epilogue_chunk(p, row, col0, v, co, cu, cn);
                    } else {
                        float* dst = p.ws + ((int64_t)s * p.M + row) * p.N + col0;
                        float4* d4 = reinterpret_cast<float4*>(dst);
#pragma unroll
                        for (int j = 0; j < 8; ++j)
                            d4[j] = make_float4(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]),
                                                __uint_as_float(v[4 * j + 2]), __uint_as_float(v[4 * j + 3]));
                    }
                }
            }
            fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(tempty_bar + acc);
            if (++acc == G::NACC) { acc = 0; accphase ^= 1; }
        }
    }
    if ((p.c_tma || p.q_tma) && warp >= 2 && lane == 0) bulk_wait_read0();  // smem read out; the writes land by grid completion
    if (MODE == 0 && p.ep.cq_counters) flush_counters<threads_of<EW>()>(co, cu, cn, p.ep.cq_counters);
    fence_before();
    __syncthreads();
    if (warp == 1) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                     "r"(G::TMEM_COLS));
    }
}

// dw[i] = sum_s ws[s][i], s ascending (deterministic), then the layer's Q(dW)
// node when asked for (one launch fewer than sum + quantize).
__global__ void __launch_bounds__(256) splitk_sum_kernel(const float* __restrict__ ws,
                                                         float* __restrict__ out, int64_t mn,
                                                         int splits, QNode q) {
    uint32_t co = 0, cu = 0, cn = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < mn;
         i += (int64_t)gridDim.x * blockDim.x) {
        float a = ws[i];
        for (int s = 1; s < splits; ++s) a = __fadd_rn(a, ws[s * mn + i]);
        out[i] = a;
        if (q.codes) qnode_store(q, i, a, co, cu, cn);
    }
    if (q.codes && q.counters) flush_counters<256>(co, cu, cn, q.counters);
}

// W'[c, kh, kw, f] = W[f, kH-1-kh, kW-1-kw, c]  (codes, ES bytes each)
template <typename T>
__global__ void flip_kernel(const T* __restrict__ w, T* __restrict__ wf, int64_t f, int64_t c,
                            int64_t kh, int64_t kw) {
    const int64_t total = f * c * kh * kw;
    for (int64_t d = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; d < total;
         d += (int64_t)gridDim.x * blockDim.x) {
        const int64_t fi = d % f, j = (d / f) % kw, i = (d / (f * kw)) % kh, ci = d / (f * kw * kh);
        wf[d] = w[((fi * kh + (kh - 1 - i)) * kw + (kw - 1 - j)) * c + ci];
    }
}

static bool epi_tma() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("FP8B_EPI_TMA");
        v = (e && e[0] == '0') ? 0 : 1;
    }
    return v == 1;
}

// 3-D store map over the split-K workspace [splits][m][n] FP32 (32x32x1 boxes).
static bool make_ws_map(CUtensorMap* tm, float* ws, int splits, int64_t m, int64_t n) {
    EncodeTiledFn enc = get_encode();
    if (!enc || (uintptr_t)ws % 16 || (n * 4) % 16) return false;
    cuuint64_t dims[3] = {(cuuint64_t)n, (cuuint64_t)m, (cuuint64_t)splits};
    cuuint64_t strides[2] = {(cuuint64_t)(n * 4), (cuuint64_t)(m * n * 4)};
    cuuint32_t box[3] = {32, 32, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    return enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, ws, dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static int num_sms() { return device_sm_count(); }

template <int ES, int MODE, int BN, int CB, int EW = 4, int MH = 1, int NH = 1>
static int run(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tcm,
               const CUtensorMap& tqm, const CParams& p, cudaStream_t st) {
    using G = Geo<ES, MODE, BN, CB, EW, MH, NH>;
    const int items = p.tiles_m * p.tiles_n * p.splits;
    const int grid = items < num_sms() ? items : num_sms();
    if constexpr (ES == 1 && MODE == 0) {
        // the layer step's output (FP8B_CONV_LEAN=0 disables)
        const char* el = getenv("FP8B_CONV_LEAN");
        if (p.q_tma && !p.c_tma && !p.ep.c && !p.ep.bias && p.ep.cq_fmt == FP8B_E5M2 &&
            p.ep.cq_mode == FP8B_RNE && !(el && el[0] == '0')) {
            ensure_smem_attr((const void*)conv_tc_kernel<ES, MODE, BN, CB, EW, 1, 1, 1>, G::SMEM);
            conv_tc_kernel<ES, MODE, BN, CB, EW, 1, 1, 1><<<grid, threads_of<EW>(), G::SMEM, st>>>(ta, tb, tcm, tqm, p);
            return FP8B_OK;
        }
    }
    ensure_smem_attr((const void*)conv_tc_kernel<ES, MODE, BN, CB, EW, MH, NH>, G::SMEM);
    conv_tc_kernel<ES, MODE, BN, CB, EW, MH, NH><<<grid, threads_of<EW>(), G::SMEM, st>>>(ta, tb, tcm, tqm, p);
    return FP8B_OK;
}

// fprop over NHWC x [n, h, w, c] and KRSC w [f, k, k, c] -> y [n, oh, ow, f]
template <int ES>
static int fprop(const void* x, const void* w, float* y, int64_t n, int64_t h, int64_t wd,
                 int64_t c, int64_t f, int k, int pad, cudaStream_t st, const fp8b_conv_t& g) {
    // narrow layers with k > 1 (C * bytes <= 128): one halo slab per tile
    // instead of one im2col row request per pixel and tap (conv_halo.cu)
    if (k > 1) {
        const int rc = launch_conv_halo(x, w, y, ES, n, h, wd, c, f, k, pad, g, st);
        if (rc != FP8B_ENOTSUP) return rc;
    }
    const int cb_bytes = (c * ES) % 128 == 0 ? 128 : ((c * ES) % 64 == 0 ? 64 : 0);
    if (!cb_bytes) return FP8B_ENOTSUP;
    const int64_t oh = h + 2 * pad - k + 1, ow = wd + 2 * pad - k + 1;
    const int64_t P = n * oh * ow;
    const CUtensorMapSwizzle swz = cb_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
    const int cbe = cb_bytes / ES;
    const int bn = f <= 64 ? 64 : (f <= 128 ? 128 : 256);
    CUtensorMap ta, tb;
    if (!make_im2col(&ta, x, ES, n, h, wd, c, k, pad, cbe, 128, swz)) return FP8B_ENOTSUP;
    if (!make_map(&tb, w, ES, (uint64_t)(k * k * c), (uint64_t)f, cbe, bn, swz)) return FP8B_ENOTSUP;
    CParams p{};
    p.M = P; p.N = f;
    p.ep = EpiArgs{y, nullptr, g.yq, g.yq_fmt, g.yq_mode, g.yq_seed, g.yq_saturate, g.yq_counters};
    p.tiles_m = (int)((P + 127) / 128);
    p.tiles_n = (int)((f + bn - 1) / bn);
    p.cblocks = (int)(c / cbe);
    p.num_kb = k * k * p.cblocks;
    p.splits = 1;
    p.C = (int)c; p.KW = k; p.pad = pad; p.OH = (int)oh; p.OW = (int)ow;
    CUtensorMap tcm;
    memset(&tcm, 0, sizeof(tcm));
    p.c_tma = (epi_tma() && y && make_c_map(&tcm, y, P, f)) ? 1 : 0;
    CUtensorMap tqm;
    memset(&tqm, 0, sizeof(tqm));
    // short K loops (1x1 convs): 8 epilogue warps split each tile's columns
    const bool ew8 = p.num_kb <= 4 && bn >= 128;
    const int cols_per_warp = ew8 ? bn / 2 : bn;
    p.qg = code_group(g.yq_fmt, cols_per_warp);
    p.q_tma = (!p.c_tma && epi_tma() && g.yq &&
               make_q_map(&tqm, g.yq, g.yq_fmt, P, f, cols_per_warp)) ? 1 : 0;
    if (cb_bytes == 128) {
        if (bn == 64) return run<ES, 0, 64, 128>(ta, tb, tcm, tqm, p, st);
        if (bn == 128) return ew8 ? run<ES, 0, 128, 128, 8>(ta, tb, tcm, tqm, p, st)
                                  : run<ES, 0, 128, 128>(ta, tb, tcm, tqm, p, st);
        return ew8 ? run<ES, 0, 256, 128, 8>(ta, tb, tcm, tqm, p, st)
                   : run<ES, 0, 256, 128>(ta, tb, tcm, tqm, p, st);
    }
    if (bn == 64) return run<ES, 0, 64, 64>(ta, tb, tcm, tqm, p, st);
    if (bn == 128) return ew8 ? run<ES, 0, 128, 64, 8>(ta, tb, tcm, tqm, p, st)
                              : run<ES, 0, 128, 64>(ta, tb, tcm, tqm, p, st);
    return ew8 ? run<ES, 0, 256, 64, 8>(ta, tb, tcm, tqm, p, st)
               : run<ES, 0, 256, 64>(ta, tb, tcm, tqm, p, st);
}

// wgrad: dw [f, k, k, c] from x [n, h, w, c] and e [n, oh, ow, f]
template <int ES>
static int wgrad(const void* x, const void* e, float* dw, int64_t n, int64_t h, int64_t wd,
                 int64_t c, int64_t f, int k, int pad, cudaStream_t st, int* nl,
                 const fp8b_conv_t& g, int* q_done) {
    {  // 3x3 with 64-byte channel and filter rows: the halo-slab wgrad
        const int rc = launch_conv_halo_wgrad(x, e, dw, ES, n, h, wd, c, f, k, pad, st, nl, &g);
        if (rc == FP8B_OK && g.yq && q_done) *q_done = 1;
        if (rc != FP8B_ENOTSUP) return rc;
    }
    const int cb_bytes = (c * ES) % 128 == 0 ? 128 : ((c * ES) % 64 == 0 ? 64 : 0);
    if (!cb_bytes || (f * ES) % 16) return FP8B_ENOTSUP;
    const int64_t oh = h + 2 * pad - k + 1, ow = wd + 2 * pad - k + 1;
    const int64_t P = n * oh * ow;
    constexpr int KPIX = 128 / ES;
    const CUtensorMapSwizzle swz = cb_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
    const int bn = cb_bytes / ES;
    CUtensorMap ta, tb;
    if (!make_map(&ta, e, ES, (uint64_t)f, (uint64_t)P, 128 / ES, KPIX)) return FP8B_ENOTSUP;
    if (!make_im2col(&tb, x, ES, n, h, wd, c, k, pad, bn, KPIX, swz)) return FP8B_ENOTSUP;
    // block tiles (MH x 128 rows of F, NH x bn channels): FP8B_CONV_WGRAD_BLOCK=0 disables
    const char* eb = getenv("FP8B_CONV_WGRAD_BLOCK");
    const int blk = eb && eb[0] ? atoi(eb) : -1;  // -1 auto, 0 off, 1 = 2 x 2, 2 = 2 x 1
    const bool can_m = f % 256 == 0, can_n = cb_bytes == 128 && c % (2 * bn) == 0;
    int mh = 1, nh = 1;
    if (blk == 1 || blk == 2) {
        mh = can_m ? 2 : 1;
        nh = blk == 1 && mh == 2 && can_n ? 2 : 1;
    } else if (blk < 0 && k > 1 && can_m) {
        // measured (config-4 layers, graph replays): 2 x 1 blocks take 3x3 256 @14
        // 52 -> 39.5 us and 3x3 512 @7 48.7 -> 47.6 us (2 x 2: 41.8 / 49.1 -- the wider
        // tile forces more split-K partials of a large dW); 1x1 layers are DRAM-bound
        // and lose 2-5 us to the extra partials, so they keep the 128 x 128 tile
        mh = 2;
    }
    CParams p{};
    p.M = f; p.N = (int64_t)k * k * c;
    p.tiles_m = (int)((f + 128 * mh - 1) / (128 * mh));
    p.tiles_n = (int)(p.N / (nh * bn));
    p.num_kb = (int)((P + KPIX - 1) / KPIX);
    const int tiles = p.tiles_m * p.tiles_n;
    int splits = tiles >= num_sms() ? 1 : num_sms() / tiles;
    if (splits > p.num_kb) splits = p.num_kb;
    if (splits < 1) splits = 1;
    p.splits = splits;
    p.C = (int)c; p.KW = k; p.pad = pad; p.OH = (int)oh; p.OW = (int)ow;
    const int64_t mn = p.M * p.N;
    float* ws = dw;
    if (splits > 1) {
        if (cudaMallocAsync(&ws, (size_t)splits * mn * sizeof(float), st) != cudaSuccess)
            return FP8B_ECUDA;
    }
    p.ws = ws;
    CUtensorMap tcm;
    memset(&tcm, 0, sizeof(tcm));
    p.c_tma = (epi_tma() && make_ws_map(&tcm, ws, splits, p.M, p.N)) ? 1 : 0;
    CUtensorMap tqm;
    memset(&tqm, 0, sizeof(tqm));
    p.q_tma = 0;
    int rc;
    if (cb_bytes == 128) {
        if (nh == 2) rc = run<ES, 1, 128 / ES, 128, 4, 2, 2>(ta, tb, tcm, tqm, p, st);
        else if (mh == 2) rc = run<ES, 1, 128 / ES, 128, 4, 2, 1>(ta, tb, tcm, tqm, p, st);
        else rc = run<ES, 1, 128 / ES, 128>(ta, tb, tcm, tqm, p, st);
    } else {
        if (mh == 2) rc = run<ES, 1, 64 / ES, 64, 4, 2, 1>(ta, tb, tcm, tqm, p, st);
        else rc = run<ES, 1, 64 / ES, 64>(ta, tb, tcm, tqm, p, st);
    }
    *nl = 1;
    if (splits > 1) {
        int64_t b = (mn + 255) / 256;
        if (b > 4 * num_sms()) b = 4 * num_sms();
        QNode q{};
        if (g.yq) {
            q = QNode{g.yq, g.yq_fmt, g.yq_mode, g.yq_seed, g.yq_saturate, g.yq_counters};
            if (q_done) *q_done = 1;
        }
        splitk_sum_kernel<<<(int)b, 256, 0, st>>>(ws, dw, mn, splits, q);
        cudaFreeAsync(ws, st);
        *nl = 2;
    }
    return rc;
}

template <int ES>
static int dgrad(const void* e, const void* w, float* dx, int64_t n, int64_t h, int64_t wd,
                 int64_t c, int64_t f, int k, int pad, cudaStream_t st, int* nl,
                 const fp8b_conv_t& g) {
    // fprop of e [n, oh, ow, f] with W' [c, k, k, f] and pad' = k-1-pad -> [n, h, w, c]
    const int pad2 = k - 1 - pad;
    if (pad2 < 0 || (f * ES) % 64) return FP8B_ENOTSUP;
    const int64_t oh = h + 2 * pad - k + 1, ow = wd + 2 * pad - k + 1;
    void* wf = nullptr;
    const int64_t nw = f * c * k * k;
    if (cudaMallocAsync(&wf, (size_t)nw * ES, st) != cudaSuccess) return FP8B_ECUDA;
    int64_t b = (nw + 255) / 256;
    if (b > 4 * num_sms()) b = 4 * num_sms();
    using T = typename std::conditional<ES == 1, uint8_t, uint16_t>::type;
    flip_kernel<T><<<(int)b, 256, 0, st>>>((const T*)w, (T*)wf, f, c, k, k);
    const int rc = fprop<ES>(e, wf, dx, n, oh, ow, f, c, k, pad2, st, g);
    cudaFreeAsync(wf, st);
    *nl = 2;
    return rc;
}

}  // namespace cv
}  // namespace tc

int conv_tc_supported(int kind, int fmt, const fp8b_conv_t& g) {
    if (fmt != FP8B_E5M2 && fmt != FP8B_FP16) return 0;
    const int64_t es = fmt == FP8B_E5M2 ? 1 : 2;
    if (g.layout != FP8B_NHWC || g.stride != 1 || g.kh != g.kw || g.pad > 64 || g.kh > 64) return 0;
    const int64_t oh = g.h + 2 * g.pad - g.kh + 1, ow = g.w + 2 * g.pad - g.kw + 1;
    if (oh < 1 || ow < 1) return 0;
    const int64_t pix = g.n * (oh > g.h ? oh : g.h) * (ow > g.w ? ow : g.w);
    if (pix >= ((int64_t)1 << 31) - 256 || g.n >= (1 << 30) || g.c >= (1 << 24) || g.f >= (1 << 24))
        return 0;
    if (kind == 0) return (g.c * es) % 64 == 0;                                  // im2col channel block
    if (kind == 1) return (g.f * es) % 64 == 0 && g.pad <= g.kh - 1;              // fprop over E
    return (g.c * es) % 64 == 0 && (g.f * es) % 16 == 0;                          // wgrad
}

int launch_conv_tc(int kind, const void* a, const void* b, float* out, int fmt,
                   const fp8b_conv_t& g, cudaStream_t st, int* nlaunch, int* q_done) {
    *nlaunch = 0;
    if (q_done) *q_done = 0;
    if (!conv_tc_supported(kind, fmt, g)) return FP8B_ENOTSUP;
    if (((uintptr_t)a % 16) || ((uintptr_t)b % 16)) return FP8B_ENOTSUP;
    const int k = (int)g.kh, pad = (int)g.pad;
    int rc;
    // A 1x1 stride-1 unpadded NHWC conv is a plain GEMM on the tensors as they
    // lie: x [P, C], e [P, F] (P = n*h*w pixels), w [F, C]. fprop (y = x . w^T,
    // w K-major) and dgrad (dx = e . w, w N-major: no weight flip pass) run on
    // the pair-tile GEMM engine when their output has >= 256 channels (the
    // 256-wide pair tile is full): measured in the config-4 step, 1x1 64->256
    // @56 0.254 -> 0.213 ms (with the GEMM's 16-warp short-K epilogue), 128->512
    // @28 0.160 -> 0.134 ms, while 64-channel outputs lose (256->64 @56 0.260 ->
    // 0.348 ms) and stay here. dgrad likewise at every pixel count since the
    // 16-warp epilogue (256->64 @56: dgrad 121 -> 81 us, layer step 0.256 -> 0.228
    // ms; FP8B_CONV_1X1_DGRAD_PIX caps the pixel count, diagnostic). wgrad
    // (long K, M = F) is far slower through the GEMM's split-K and stays.
    // FP8B_CONV_1X1_GEMM=0 / 1 disables / forces the routing.
    const char* e1 = getenv("FP8B_CONV_1X1_GEMM");
    const int64_t nout = kind == 0 ? g.f : g.c;
    const char* e2 = getenv("FP8B_CONV_1X1_DGRAD_PIX");  // diagnostic: dgrad pixel limit
    const int64_t dgrad_pix = e2 && e2[0] ? atoll(e2) : INT64_MAX;
    const bool gemm_1x1 = e1 && e1[0] ? e1[0] == '1'
                                      : nout >= 256 && (kind == 0 || g.n * g.h * g.w <= dgrad_pix);
    if (kind != 2 && k == 1 && pad == 0 && g.stride == 1 && gemm_1x1) {
        const EpiArgs ep{out, nullptr, g.yq, g.yq_fmt, g.yq_mode, g.yq_seed, g.yq_saturate, g.yq_counters};
        const int64_t P = g.n * g.h * g.w;
        rc = kind == 0 ? launch_gemm_tc(a, b, P, g.f, g.c, fmt, 0, 0, ep, st, nlaunch)
                       : launch_gemm_tc(a, b, P, g.c, g.f, fmt, 0, 1, ep, st, nlaunch);
        if (rc != FP8B_ENOTSUP) return rc;
        *nlaunch = 0;
    }
    // 1x1 wgrad dW[F, C] = e^T . x is the GEMM with A = e [K = P, M = F] (MN-major)
    // and B = x [K = P, N = C] (N-major). Through the pair-tile GEMM's split-K it
    // wins only for few pixels (measured as graph replays: P = 12544, 2048 x 512:
    // 24.8 vs 34.7 us; P = 50176, 256 x 1024: 40.8 vs 31.6 us; 56 x 56 far slower).
    // FP8B_CONV_1X1_WGRAD_PIX overrides the pixel limit (diagnostic; 0 disables).
    if (kind == 2 && k == 1 && pad == 0 && g.stride == 1 && out) {
        const char* e3 = getenv("FP8B_CONV_1X1_WGRAD_PIX");
        const int64_t lim = e3 && e3[0] ? atoll(e3) : 16384;
        const int64_t P = g.n * g.h * g.w;
        if (P <= lim && g.f >= 256 && g.c >= 256) {
            const EpiArgs ep{out, nullptr, g.yq, g.yq_fmt, g.yq_mode, g.yq_seed, g.yq_saturate, g.yq_counters};
            rc = launch_gemm_tc(b, a, g.f, g.c, P, fmt, 1, 1, ep, st, nlaunch);
            if (rc == FP8B_OK && g.yq && q_done) *q_done = 1;
            if (rc != FP8B_ENOTSUP) return rc;
            *nlaunch = 0;
        }
    }
    if (kind == 0) {
        rc = fmt == FP8B_E5M2 ? tc::cv::fprop<1>(a, b, out, g.n, g.h, g.w, g.c, g.f, k, pad, st, g)
                              : tc::cv::fprop<2>(a, b, out, g.n, g.h, g.w, g.c, g.f, k, pad, st, g);
        if (rc == FP8B_OK) *nlaunch = 1;
    } else if (kind == 1) {
        rc = fmt == FP8B_E5M2 ? tc::cv::dgrad<1>(a, b, out, g.n, g.h, g.w, g.c, g.f, k, pad, st, nlaunch, g)
                              : tc::cv::dgrad<2>(a, b, out, g.n, g.h, g.w, g.c, g.f, k, pad, st, nlaunch, g);
    } else {
        rc = fmt == FP8B_E5M2 ? tc::cv::wgrad<1>(a, b, out, g.n, g.h, g.w, g.c, g.f, k, pad, st, nlaunch, g, q_done)
                              : tc::cv::wgrad<2>(a, b, out, g.n, g.h, g.w, g.c, g.f, k, pad, st, nlaunch, g, q_done);
    }
    return rc;
}

}  // namespace fp8b
