// kernels.cuh -- launcher declarations shared between the kernel files and the C-ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/fp8b200.h"

namespace fp8b {

struct LfsrTables;

// Fused GEMM epilogue: bias add, FP32 store, output Q node.
struct EpiArgs {
    float* c;
    const float* bias;
    void* cq;
    int cq_fmt;
    int cq_mode;
    uint64_t cq_seed;
    int cq_sat;
    int64_t* cq_counters;
};

void launch_quantize(const float* x, void* codes, int64_t n, int fmt,
                     const fp8b_quant_config_t& cfg, int64_t* counters, cudaStream_t st,
                     const LfsrTables& tabs);
void launch_dequantize(const void* codes, float* out, int64_t n, int fmt, cudaStream_t st);
void launch_transpose(const void* in, void* out, int64_t rows, int64_t cols, int fmt,
                      cudaStream_t st);
void launch_count_nonfinite(const float* x, int64_t n, int64_t* counters, cudaStream_t st);
void launch_bias_grad(const void* e, int fmt, int64_t rows, int64_t cols, float* db,
                      cudaStream_t st);
void launch_sgd(const void* grad, int grad_fmt, uint16_t* master, float* mom, int64_t n,
                const fp8b_sgd_args_t& args, cudaStream_t st, const LfsrTables& tabs);
void launch_scaler_step(fp8b_loss_scaler_t* s, const int64_t* counters, int finite, int64_t it,
                        cudaStream_t st);
void launch_unscale(float* g, int64_t n, const fp8b_loss_scaler_t* s, cudaStream_t st);
void launch_gemm_seq(const void* a, const void* b, int64_t m, int64_t n, int64_t k, int fmt,
                     int a_mn, int b_mn, const EpiArgs& ep, cudaStream_t st);
// Returns 0 on success, FP8B_ENOTSUP if the shape/layout is not supported by
// the tensor-core engine.
int launch_gemm_tc(const void* a, const void* b, int64_t m, int64_t n, int64_t k, int fmt,
                   int a_mn, int b_mn, const EpiArgs& ep, cudaStream_t st, int* nlaunch);
// Conv family: kind 0 fprop, 1 dgrad, 2 wgrad.
void launch_conv_seq(int kind, const void* a, const void* b, float* out, int fmt,
                     const fp8b_conv_t& g, cudaStream_t st);
// Returns FP8B_ENOTSUP when the tensor engine does not cover the case.
// wgrad (kind 2) with g.yq set: the Q node is fused into the split-K sum where
// there is one, and *q_done says so (otherwise the caller quantizes `out`).
int launch_conv_tc(int kind, const void* a, const void* b, float* out, int fmt,
                   const fp8b_conv_t& g, cudaStream_t st, int* nlaunch, int* q_done = nullptr);
int conv_tc_supported(int kind, int fmt, const fp8b_conv_t& g);
// Weight-stationary halo-slab fprop (conv_halo.cu) for C * bytes in {64, 128},
// F <= 256; FP8B_ENOTSUP when the geometry is not covered.
bool conv_halo_supported(int es, int64_t n, int64_t h, int64_t w, int64_t c, int64_t f, int k,
                         int pad);
int launch_conv_halo(const void* x, const void* wt, float* y, int es, int64_t n, int64_t h,
                     int64_t w, int64_t c, int64_t f, int k, int pad, const fp8b_conv_t& g,
                     cudaStream_t st);
// Halo-slab wgrad (conv_halo.cu): 3x3, C * bytes == F * bytes == 64.
bool conv_halo_wgrad_supported(int es, int64_t n, int64_t h, int64_t w, int64_t c, int64_t f, int k,
                               int pad);
int launch_conv_halo_wgrad(const void* x, const void* e, float* dw, int es, int64_t n, int64_t h,
                           int64_t w, int64_t c, int64_t f, int k, int pad, cudaStream_t st, int* nl,
                           const fp8b_conv_t* gq = nullptr);
void launch_im2col(const void* x, void* cols, int fmt, const fp8b_conv_t& g, cudaStream_t st);
// Per-device setup (several GPUs per process are allowed): SM count of the
// current device, and the >48 KB dynamic shared memory opt-in of a kernel on
// the current device, each done once per (kernel, device).
int device_sm_count();
void ensure_smem_attr(const void* fn, int bytes);
// Reference-stream SR (LFSR blocks): tensors of at most this many 4096-blocks
// take the CTA-per-block kernels (all of a block's loads in flight at once)
// instead of the warp-per-block ones, whose 16-chunk chain per block and
// 139 KB table copy per CTA only pay off with many blocks per SM.
// FP8B_LFSR_CTA_MAX overrides it (A/B).
int64_t lfsr_cta_max_blocks();
// Adds n to the library's launch counter (fp8b_launch_count).
void note_launches(int n);
void launch_fill_synthetic(float* out, int64_t n, int kind, uint64_t seed, double p, double lo,
                           double hi, cudaStream_t st);
// peer.cu: fused rank-order sum of the ranks' FP32 partials + Q node over peer memory
int launch_peer_reduce_quantize(const float* const* peers, int world, int64_t i0, int64_t n,
                                float* sum_out, void* codes, int fmt,
                                const fp8b_quant_config_t& cfg, int64_t* counters,
                                cudaStream_t st);
void launch_stream_probe(const float* x, void* out, int64_t n, int out_bytes, cudaStream_t st);

}  // namespace fp8b
