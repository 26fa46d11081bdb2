// synth.cu -- seeded synthetic inputs generated in HBM (no host round trip).
// Stand-ins for the datasets the paper used: no dataset item is
// reproduced; only shapes and value distributions are.
#include "common.cuh"
#include "kernels.cuh"

namespace fp8b {

__device__ __forceinline__ double u01(uint64_t h) { return (double)(h >> 11) * 0x1.0p-53; }

__global__ void fill_synth_kernel(float* out, int64_t n, int kind, uint64_t seed, double p,
                                  double lo, double hi) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t h1 = mix64(seed * 0x2545F4914F6CDD1Dull + 2ull * (uint64_t)i + 1ull);
        const uint64_t h2 = mix64(h1 ^ 0xD6E8FEB86659FD93ull);
        float v;
        if (kind == 0) {
            if (u01(h1) < p) {
                // exact E5M2 midpoint between adjacent finite codes c and c+1
                const uint32_t c = (uint32_t)(h2 % 0x7Bull);
                v = 0.5f * (dec_e5m2(c) + dec_e5m2(c + 1));
            } else {
                v = (float)exp2(lo + (hi - lo) * u01(h2));
            }
            if (h1 & 1ull) v = -v;
        } else {
            const double u1 = ((double)(h1 >> 11) + 1.0) * 0x1.0p-53;
            const double r = sqrt(-2.0 * log(u1));
            double z = r * cos(6.283185307179586 * u01(h2)) * p;
            if (kind == 2) z = fabs(z);
            v = (float)z;
        }
        out[i] = v;
    }
}

void launch_fill_synthetic(float* out, int64_t n, int kind, uint64_t seed, double p, double lo,
                           double hi, cudaStream_t st) {
    int64_t blocks = (n + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    if (blocks < 1) blocks = 1;
    fill_synth_kernel<<<(int)blocks, 256, 0, st>>>(out, n, kind, seed, p, lo, hi);
}

// The quantizer's access pattern with no arithmetic (fp8b_stream_probe).
template <int OUTB>
__global__ void __launch_bounds__(256) stream_probe_kernel(const float4* __restrict__ x,
                                                          void* __restrict__ out, int64_t ngroups) {
    constexpr int UN = 2;
    const int64_t stride = (int64_t)gridDim.x * 256 * UN;
    float acc = 0.0f;
    for (int64_t g0 = (int64_t)blockIdx.x * 256 * UN + threadIdx.x; g0 < ngroups; g0 += stride) {
        float4 v[UN];
#pragma unroll
        for (int j = 0; j < UN; ++j)
            if (g0 + j * 256 < ngroups) v[j] = __ldcs(x + g0 + j * 256);
#pragma unroll
        for (int j = 0; j < UN; ++j) {
            const int64_t g = g0 + j * 256;
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
    if (OUTB == 0 && acc == 123.456f && out) *reinterpret_cast<float*>(out) = acc;
}

void launch_stream_probe(const float* x, void* out, int64_t n, int out_bytes, cudaStream_t st) {
    const int grid = device_sm_count() * 8;
    const float4* x4 = reinterpret_cast<const float4*>(x);
    if (out_bytes == 0) stream_probe_kernel<0><<<grid, 256, 0, st>>>(x4, out, n / 4);
    else if (out_bytes == 1) stream_probe_kernel<1><<<grid, 256, 0, st>>>(x4, out, n / 4);
    else if (out_bytes == 2) stream_probe_kernel<2><<<grid, 256, 0, st>>>(x4, out, n / 4);
    else stream_probe_kernel<4><<<grid, 256, 0, st>>>(x4, out, n / 4);
}

}  // namespace fp8b
