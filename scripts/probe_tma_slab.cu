// probe_tma_slab.cu -- TMA load throughput for conv slab box shapes (diagnostic).
// Each CTA (one per SM) streams T slabs of the same shape through a 4-stage
// ring (a consumer warp only waits and releases), over an NHWC E5M2 tensor
// [256, 56, 56, 64] (51 MB). Reports GB/s and bytes/clk/SM per variant.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probe_tma_slab probe_tma_slab.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(c)); }
__device__ __forceinline__ void expect_tx(uint64_t* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory"); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
    asm volatile("{\n.reg .pred P;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W_%=;\n}\n" ::"r"(sa(b)), "r"(ph) : "memory");
}

struct Var { int kind; int rows_per_slab; uint32_t bytes; };

__global__ void __launch_bounds__(64, 1) probe(const __grid_constant__ CUtensorMap tm, const uint8_t* src, int kind,
                                               int tiles, uint32_t bytes, int nimg, int H) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* ring = (uint8_t*)(((uintptr_t)smem + 1023) & ~(uintptr_t)1023);
    __shared__ uint64_t full[4], empty[4];
    if (threadIdx.x == 0) {
        for (int i = 0; i < 4; ++i) { mbar_init(full + i, 1); mbar_init(empty + i, 1); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const uint32_t stride = (bytes + 1023) & ~1023u;
    if (threadIdx.x == 0) {
        int st = 0; uint32_t ph = 0;
        for (int t = 0; t < tiles; ++t) {
            const int tile = blockIdx.x * tiles + t;
            const int n = (tile / 28) % nimg, oh0 = (tile % 28) * 2;
            wait(empty + st, ph ^ 1);
            expect_tx(full + st, bytes);
            uint8_t* dst = ring + st * stride;
            if (kind == 0 || kind == 1) {  // 4-D tiled box {64, Wbox, 5, 1}
                const int w0 = kind == 0 ? -1 : 0;
                asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];"
                             ::"r"(sa(dst)), "l"((uint64_t)&tm), "r"(sa(full + st)), "r"(0), "r"(w0), "r"(oh0 - 1), "r"(n) : "memory");
            } else if (kind == 2 || kind == 3) {  // 2-D box over [pixels (or pairs), 64 (or 128) bytes]
                const int row0 = (n * H + oh0) * 56 / (kind == 3 ? 2 : 1);
                asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                             ::"r"(sa(dst)), "l"((uint64_t)&tm), "r"(sa(full + st)), "r"(0), "r"(row0) : "memory");
            } else {  // 1-D bulk copy
                const uint8_t* g = src + (size_t)(n * H + oh0) * 56 * 64;
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                             ::"r"(sa(dst)), "l"((uint64_t)g), "r"(bytes), "r"(sa(full + st)) : "memory");
            }
            if (++st == 4) { st = 0; ph ^= 1; }
        }
    } else if (threadIdx.x == 32) {
        int st = 0; uint32_t ph = 0;
        for (int t = 0; t < tiles; ++t) {
            wait(full + st, ph);
            arrive(empty + st);
            if (++st == 4) { st = 0; ph ^= 1; }
        }
    }
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    const int N = 256, H = 56, W = 56, C = 64;
    const size_t bytes_x = (size_t)N * H * W * C;
    uint8_t* x;
    CK(cudaMalloc(&x, bytes_x + (1 << 20)));
    CK(cudaMemset(x, 0x3c, bytes_x));
    void* fp = nullptr; cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q));
    EncFn enc = (EncFn)fp;
    int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 20480 + 1024));
    const char* names[] = {"4D box {64B,58,5,1} w0=-1 (OOB cols), 64B swz", "4D box {64B,56,5,1} w0=0, 64B swz",
                           "2D box {64B, 256 rows}, 64B swz", "2D box {128B, 145 rows}, 128B swz", "1D bulk 18432 B"};
    for (int kind = 0; kind < 5; ++kind) {
        CUtensorMap tm{};
        uint32_t bytes = 0;
        CUresult r = CUDA_SUCCESS;
        if (kind <= 1) {
            cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
            cuuint64_t str[3] = {(cuuint64_t)C, (cuuint64_t)W * C, (cuuint64_t)H * W * C};
            cuuint32_t box[4] = {64, kind == 0 ? 58u : 56u, 5, 1}, es[4] = {1, 1, 1, 1};
            r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, x, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            bytes = 64 * box[1] * 5;
        } else if (kind == 2) {
            cuuint64_t dims[2] = {64, (cuuint64_t)N * H * W};
            cuuint64_t str[1] = {64};
            cuuint32_t box[2] = {64, 256}, es[2] = {1, 1};
            r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, x, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            bytes = 64 * 256;
        } else if (kind == 3) {
            cuuint64_t dims[2] = {128, (cuuint64_t)N * H * W / 2};
            cuuint64_t str[1] = {128};
            cuuint32_t box[2] = {128, 145}, es[2] = {1, 1};
            r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, x, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            bytes = 128 * 145;
        } else {
            bytes = 18432;
        }
        if (r != CUDA_SUCCESS) { printf("encode failed for %d\n", kind); continue; }
        const int tiles = 48;  // per CTA (the config-4 fprop has ~48 tiles per SM)
        for (int rep = 0; rep < 3; ++rep) {
            cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
            cudaEventRecord(a);
            probe<<<sms, 64, 4 * 20480 + 1024>>>(tm, x, kind, tiles, bytes, N, H);
            cudaEventRecord(b);
            CK(cudaEventSynchronize(b));
            float ms = 0; cudaEventElapsedTime(&ms, a, b);
            const double tot = (double)bytes * tiles * sms;
            if (rep == 2)
                printf("%-48s %7.1f us  %7.1f GB/s  %5.1f B/clk/SM (at %d MHz)\n", names[kind], ms * 1e3, tot / ms / 1e6,
                       tot / sms / (ms * 1e-3 * clk * 1e3), clk / 1000);
        }
    }
    CK(cudaGetLastError());
    return 0;
}
