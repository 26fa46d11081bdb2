// hbm_ceiling.cu -- what HBM3e delivers for the quantizer's access mixes, with no
// arithmetic in the way: FP32 in, {0, 1, 2, 4} bytes out per element. The result
// is the practical ceiling the quantize / update kernels are judged against
// beside the 1:1 copy figure in MEASURED_PEAKS.json.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o scripts/hbm_ceiling scripts/hbm_ceiling.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

template <int OUTB, int UNROLL, int NT>
__global__ void __launch_bounds__(NT) mix_kernel(const float4* __restrict__ x, void* __restrict__ out,
                                                 int64_t ngroups, float* sink) {
    const int64_t stride = (int64_t)gridDim.x * NT * UNROLL;
    float acc = 0.f;
    for (int64_t g0 = (int64_t)blockIdx.x * NT * UNROLL + threadIdx.x; g0 < ngroups; g0 += stride) {
        float4 v[UNROLL];
#pragma unroll
        for (int j = 0; j < UNROLL; ++j) {
            const int64_t g = g0 + (int64_t)j * NT;
            if (g < ngroups) v[j] = __ldcs(x + g);
        }
#pragma unroll
        for (int j = 0; j < UNROLL; ++j) {
            const int64_t g = g0 + (int64_t)j * NT;
            if (g >= ngroups) continue;
            const uint32_t a = __float_as_uint(v[j].x), b = __float_as_uint(v[j].y),
                           c = __float_as_uint(v[j].z), d = __float_as_uint(v[j].w);
            if (OUTB == 0) acc += v[j].x + v[j].y + v[j].z + v[j].w;
            if (OUTB == 1)
                __stcs(reinterpret_cast<uint32_t*>(out) + g,
                       (a >> 24) | ((b >> 24) << 8) | ((c >> 24) << 16) | (d & 0xFF000000u));
            if (OUTB == 2)
                __stcs(reinterpret_cast<uint2*>(out) + g,
                       make_uint2((a >> 16) | (b & 0xFFFF0000u), (c >> 16) | (d & 0xFFFF0000u)));
            if (OUTB == 4) __stcs(reinterpret_cast<float4*>(out) + g, v[j]);
        }
    }
    if (OUTB == 0 && acc == 123.456f) *sink = acc;
}

__global__ void fill_random(uint32_t* x, int64_t n, int lo_exp, int hi_exp) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t z = (uint64_t)i + 0x9E3779B97F4A7C15ull;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z ^= z >> 31;
        const uint32_t e = 127 + lo_exp + (uint32_t)((z >> 40) % (uint32_t)(hi_exp - lo_exp));
        x[i] = ((uint32_t)z & 0x807FFFFFu) | (e << 23);
    }
}

template <int OUTB, int UNROLL, int NT>
static void run(const float4* x, void* out, int64_t n, float* sink, int ctas_per_sm, int sms) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int grid = sms * ctas_per_sm;
    float best = 1e30f;
    for (int it = 0; it < 12; ++it) {
        cudaEventRecord(e0);
        mix_kernel<OUTB, UNROLL, NT><<<grid, NT>>>(x, out, n / 4, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (it >= 2 && ms < best) best = ms;
    }
    cudaEventRecord(e0);
    for (int it = 0; it < 10; ++it) mix_kernel<OUTB, UNROLL, NT><<<grid, NT>>>(x, out, n / 4, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float avg;
    cudaEventElapsedTime(&avg, e0, e1);
    avg /= 10;
    const double bytes = (double)n * (4 + OUTB);
    printf("out=%dB unroll=%d nt=%d ctas/sm=%d : best %.4f ms %.1f GB/s | avg10 %.4f ms %.1f GB/s\n", OUTB,
           UNROLL, NT, ctas_per_sm, best, bytes / best * 1e-6, avg, bytes / avg * 1e-6);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
}

int main(int argc, char** argv) {
    const bool random = argc > 1;
    const int64_t n = 1ll << 28;
    float4* x;
    void* out;
    float* sink;
    cudaMalloc(&x, n * 4);
    cudaMalloc(&out, n * 4);
    cudaMalloc(&sink, 4);
    cudaMemset(x, 0x11, n * 4);
    if (random) {
        fill_random<<<2048, 256>>>((uint32_t*)x, n, -24, 17);
        printf("input: random sign/mantissa, exponent uniform in [2^-24, 2^17)\n");
    } else {
        printf("input: constant 0x11111111\n");
    }
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
#define SWEEP(OUTB)                                   \
    run<OUTB, 2, 256>(x, out, n, sink, 8, sms);       \
    run<OUTB, 4, 256>(x, out, n, sink, 4, sms);       \
    run<OUTB, 4, 256>(x, out, n, sink, 6, sms);       \
    run<OUTB, 4, 256>(x, out, n, sink, 8, sms);       \
    run<OUTB, 8, 256>(x, out, n, sink, 4, sms);       \
    run<OUTB, 4, 512>(x, out, n, sink, 4, sms);       \
    run<OUTB, 4, 1024>(x, out, n, sink, 2, sms);      \
    run<OUTB, 8, 1024>(x, out, n, sink, 1, sms);      \
    run<OUTB, 1, 256>(x, out, n, sink, 2048, sms);
    SWEEP(0)
    SWEEP(1)
    SWEEP(2)
    SWEEP(4)
    cudaError_t e = cudaDeviceSynchronize();
    printf("done: %s\n", cudaGetErrorString(e));
    return e != cudaSuccess;
}
