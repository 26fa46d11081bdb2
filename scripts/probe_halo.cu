// probe_halo.cu -- per-tile timeline of the halo conv kernel (diagnostic).
// Builds conv_halo.cu with FP8B_HALO_TRACE and links the library for the rest:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DFP8B_HALO_TRACE -cudart shared \
//        -Dlaunch_conv_halo=probe_launch_conv_halo -Dconv_halo_supported=probe_conv_halo_supported -Dhalo=halo_probe \
//        -I paper_1905_12334_b200/csrc -o scripts/probe_halo scripts/probe_halo.cu \
//        -Lpaper_1905_12334_b200 -lfp8b200 -lcuda -Xlinker -rpath=$PWD/paper_1905_12334_b200
// Run: probe_halo C F HW [q]
#include "../paper_1905_12334_b200/csrc/conv_halo.cu"

#include <cstdio>
#include <vector>

int main(int argc, char** argv) {
    const int C = argc > 1 ? atoi(argv[1]) : 64, F = argc > 2 ? atoi(argv[2]) : 64;
    const int HW = argc > 3 ? atoi(argv[3]) : 56;
    const bool q = argc > 4;
    const int N = 256, k = 3, pad = 1;
    uint8_t *x, *w, *yq;
    float* y = nullptr;
    int64_t* cnt;
    cudaMalloc(&x, (size_t)N * HW * HW * C);
    cudaMalloc(&w, (size_t)F * 9 * C);
    cudaMalloc(&yq, (size_t)N * HW * HW * F);
    cudaMalloc(&cnt, 64);
    if (!q) cudaMalloc(&y, (size_t)N * HW * HW * F * 4);
    cudaMemset(x, 0x38, (size_t)N * HW * HW * C);
    cudaMemset(w, 0x38, (size_t)F * 9 * C);
    cudaMemset(cnt, 0, 64);
    fp8b_conv_t g{};
    if (q) { g.yq = yq; g.yq_fmt = FP8B_E5M2; g.yq_mode = FP8B_RNE; g.yq_seed = 1; g.yq_counters = cnt; }
    for (int r = 0; r < 3; ++r) {
        int rc = fp8b::launch_conv_halo(x, w, y, 1, N, HW, HW, C, F, k, pad, g, 0);
        if (rc) { printf("rc %d\n", rc); return 1; }
    }
    printf("sync: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    std::vector<unsigned long long> t(148 * 10 * 64);
    printf("copy: %s\n", cudaGetErrorString(cudaMemcpyFromSymbol(t.data(), fp8b::tc::halo::g_halo_trace, t.size() * 8)));
    unsigned long long nz = 0;
    for (auto v : t) nz += v != 0;
    printf("nonzero trace entries: %llu\n", nz);
    printf("roles: 0 producer issue, 1 MMA after tempty, 2 MMA after full, 3 MMA issued, 4 epi after tfull, 5 epi done\n");
    for (int cta : {0, 73, 147}) {
        const unsigned long long* b = t.data() + cta * 10 * 64;
        const unsigned long long t0 = b[1 * 64 + 0];
        printf("CTA %d (ns from MMA start of tile 0)\n tile  prod   mma_te  mma_full mma_done epi_full epi_done  tmem_ld   codes  acquired\n", cta);
        for (int i = 0; i < 50; ++i) {
            if (!b[4 * 64 + i]) break;
            printf("%4d", i);
            for (int r = 0; r < 9; ++r) printf(" %8lld", (long long)(b[r * 64 + i] - t0));
            printf("\n");
        }
    }
    return 0;
}
