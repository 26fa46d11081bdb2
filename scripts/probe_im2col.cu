// Probe: empirically pin the TMA im2col-mode traversal used by conv_tc.cu.
// Loads pixelsPerColumn pixels of an NHWC u16 tensor for several (start,
// offset) pairs and prints which input pixel each smem row received.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

typedef CUresult (*EncIm2col)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const int*, const int*, cuuint32_t, cuuint32_t,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__global__ void probe(const __grid_constant__ CUtensorMap tm, uint16_t* out, int w0, int h0, int n0,
                      int ow, int oh, int npix) {
    __shared__ alignas(1024) uint16_t buf[128 * 8];
    __shared__ alignas(8) uint64_t bar;
    if (threadIdx.x == 0) {
        for (int i = 0; i < 128 * 8; ++i) buf[i] = 0xFFFF;
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(&bar)),
                     "r"(npix * 16)
                     : "memory");
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%3, %4, %5, %6}], [%2], {%7, %8};" ::"r"((uint32_t)__cvta_generic_to_shared(buf)),
            "l"((uint64_t)&tm), "r"((uint32_t)__cvta_generic_to_shared(&bar)), "r"(0), "r"(w0), "r"(h0),
            "r"(n0), "h"((uint16_t)ow), "h"((uint16_t)oh)
            : "memory");
        asm volatile(
            "{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n@!P bra W;\n}\n" ::"r"(
                (uint32_t)__cvta_generic_to_shared(&bar))
            : "memory");
        for (int i = 0; i < 128 * 8; ++i) out[i] = buf[i];
    }
}

int main() {
    const int N = 2, H = 5, W = 6, C = 8;
    std::vector<uint16_t> x(N * H * W * C);
    for (int n = 0; n < N; ++n)
        for (int h = 0; h < H; ++h)
            for (int w = 0; w < W; ++w)
                for (int c = 0; c < C; ++c) x[((n * H + h) * W + w) * C + c] = (uint16_t)((n * 100 + h * 10 + w) * 8 + c + 8);
    uint16_t *dx, *dout;
    cudaMalloc(&dx, x.size() * 2);
    cudaMalloc(&dout, 128 * 8 * 2);
    cudaMemcpy(dx, x.data(), x.size() * 2, cudaMemcpyHostToDevice);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &fn, cudaEnableDefault, &q);
    if (!fn) { printf("no encoder\n"); return 1; }
    EncIm2col enc = (EncIm2col)fn;
    struct Case { int pad, k, w0, h0, n0, ow, oh, npix; };
    Case cases[] = {
        {1, 3, -1, -1, 0, 0, 0, 40}, {1, 3, -1, -1, 0, 1, 1, 40}, {1, 3, -1, -1, 0, 2, 0, 40},
        {1, 3, 2, 3, 0, 0, 0, 40},   {1, 3, 2, 3, 0, 2, 2, 40},   {0, 1, 0, 0, 0, 0, 0, 64},
        {0, 1, 3, 4, 0, 0, 0, 64},   {0, 3, 0, 0, 0, 1, 2, 24},
    };
    for (auto& cs : cases) {
        CUtensorMap tm;
        cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
        cuuint64_t strides[3] = {(cuuint64_t)C * 2, (cuuint64_t)W * C * 2, (cuuint64_t)H * W * C * 2};
        int lower[2] = {-cs.pad, -cs.pad};
        int upper[2] = {cs.pad - (cs.k - 1), cs.pad - (cs.k - 1)};
        cuuint32_t es[4] = {1, 1, 1, 1};
        CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT16, 4, dx, dims, strides, lower, upper, C,
                         cs.npix, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); continue; }
        probe<<<1, 32>>>(tm, dout, cs.w0, cs.h0, cs.n0, cs.ow, cs.oh, cs.npix);
        std::vector<uint16_t> o(128 * 8);
        cudaError_t e = cudaMemcpy(o.data(), dout, o.size() * 2, cudaMemcpyDeviceToHost);
        printf("case pad=%d k=%d start(w=%d,h=%d,n=%d) off(%d,%d) npix=%d err=%d\n", cs.pad, cs.k, cs.w0,
               cs.h0, cs.n0, cs.ow, cs.oh, cs.npix, (int)e);
        for (int p = 0; p < cs.npix; ++p) {
            const uint16_t v = o[p * 8];
            if (v == 0) printf(" [%d]=pad", p);
            else if (v == 0xFFFF) printf(" [%d]=untouched", p);
            else { const int id = v / 8 - 1; printf(" [%d]=n%d,h%d,w%d", p, id / 100, (id / 10) % 10, id % 10); }
            bool ok = true;
            for (int c = 1; c < 8; ++c) ok &= (o[p * 8 + c] == (v ? v + c : 0));
            if (!ok) printf("(chan!)");
        }
        printf("\n");
    }
    return 0;
}
