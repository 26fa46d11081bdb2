// peer.cu -- the data-parallel exchange over NVLink / NVSwitch peer memory.
//
// The reference has one Q(dW) node on the full-batch FP32 sum (nn.cpp:302-303).
// Data parallel, that is "sum the ranks' partial dW, then quantize".
// Instead of an NCCL reduce-scatter that writes an FP32 sum back to HBM for a
// second kernel to read, the owner of a shard reads every rank's partial
// straight out of its peers' memory (P2P loads over NVLink; every GPU has full
// bandwidth to every peer through NVSwitch), adds them in rank order -- the
// same, fixed order on every rank, so the result does not depend on who owns
// the shard -- and applies the Q node in the same pass: 4 (world - 1) / world
// bytes per parameter on the wire, no FP32 round trip through HBM, one launch.
//
// Buffers other processes map come from fp8b_peer_alloc (cudaMalloc +
// cudaIpcGetMemHandle); the host side exchanges the 64-byte handles over its
// process group and orders the steps (dp.py). Kernels never wait on a peer.
#include <cstring>

#include "common.cuh"
#include "kernels.cuh"
#include "quant_group.cuh"

namespace fp8b {

constexpr int kMaxPeers = 16;
struct PeerPtrs {
    const float* p[kMaxPeers];
};

// s[i] = peers[0][i0 + i] + peers[1][i0 + i] + ... (rank order), then the Q node
// of the elementwise quantize kernels (quant_group.cuh: the same code words,
// counters and counter-bit stream as fp8b_quantize on the sum).
template <int MB, int MODE>  // MODE 0 RNE, 1 SR counter bits, 3 TRUNC
__global__ void __launch_bounds__(256) peer_reduce_quant_kernel(PeerPtrs peers, int world,
                                                                int64_t i0, int64_t n,
                                                                float* __restrict__ sum_out,
                                                                void* __restrict__ codes,
                                                                uint64_t seed, int saturate,
                                                                int64_t elem_offset,
                                                                int64_t* counters) {
    constexpr int UN = 2;
    const bool sat = saturate != 0;
    uint32_t c_big = 0, c_nan = 0, c_unf = 0;
    const int64_t ngroups = n >> 2;
    const int64_t stride = (int64_t)gridDim.x * 256 * UN;
    const uint32_t rb[4] = {0u, 0u, 0u, 0u};
    for (int64_t g0 = (int64_t)blockIdx.x * 256 * UN + threadIdx.x; g0 < ngroups; g0 += stride) {
        float4 s[UN];
#pragma unroll
        for (int j = 0; j < UN; ++j) {
            const int64_t g = g0 + j * 256;
            if (g < ngroups) s[j] = __ldcs(reinterpret_cast<const float4*>(peers.p[0] + i0) + g);
        }
        for (int r = 1; r < world; ++r) {
            const float4* pr = reinterpret_cast<const float4*>(peers.p[r] + i0);
#pragma unroll
            for (int j = 0; j < UN; ++j) {
                const int64_t g = g0 + j * 256;
                if (g >= ngroups) continue;
                const float4 v = __ldcs(pr + g);
                s[j].x = __fadd_rn(s[j].x, v.x); s[j].y = __fadd_rn(s[j].y, v.y);
                s[j].z = __fadd_rn(s[j].z, v.z); s[j].w = __fadd_rn(s[j].w, v.w);
            }
        }
#pragma unroll
        for (int j = 0; j < UN; ++j) {
            const int64_t g = g0 + j * 256;
            if (g >= ngroups) continue;
            if (sum_out) reinterpret_cast<float4*>(sum_out)[g] = s[j];
            quant_group<MB, MODE>(s[j], rb, g, codes, seed, sat, elem_offset, c_big, c_nan, c_unf);
        }
    }
    if (counters)
        flush_counters<256>(quant_group_overflow<MB, MODE>(c_big, c_nan), c_unf, c_nan, counters);
}

int launch_peer_reduce_quantize(const float* const* peers, int world, int64_t i0, int64_t n,
                                float* sum_out, void* codes, int fmt,
                                const fp8b_quant_config_t& cfg, int64_t* counters,
                                cudaStream_t st) {
    PeerPtrs pp;
    memset(&pp, 0, sizeof(pp));
    for (int r = 0; r < world; ++r) pp.p[r] = peers[r];
    int64_t g = (n / 4 + 511) / 512;
    const int64_t cap = (int64_t)device_sm_count() * 8;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    const int64_t eoff = cfg.block_offset * kBlock;
#define FP8B_PRQ(MB, MODE)                                                                   \
    peer_reduce_quant_kernel<MB, MODE><<<(int)g, 256, 0, st>>>(pp, world, i0, n, sum_out, codes, \
                                                              cfg.seed, cfg.saturate, eoff, counters)
    const int mode = cfg.mode == FP8B_RNE ? 0 : (cfg.mode == FP8B_TRUNC ? 3 : 1);
    if (fmt == FP8B_E5M2) {
        if (mode == 0) FP8B_PRQ(2, 0); else if (mode == 1) FP8B_PRQ(2, 1); else FP8B_PRQ(2, 3);
    } else {
        if (mode == 0) FP8B_PRQ(10, 0); else if (mode == 1) FP8B_PRQ(10, 1); else FP8B_PRQ(10, 3);
    }
#undef FP8B_PRQ
    return FP8B_OK;
}

}  // namespace fp8b
