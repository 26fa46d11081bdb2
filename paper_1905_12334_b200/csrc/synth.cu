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

}  // namespace fp8b
