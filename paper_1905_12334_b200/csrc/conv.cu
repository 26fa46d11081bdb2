// conv.cu -- the conv family of the reference (kernels.cpp:106-253) on the GPU.
//
// Sequential engine: one thread per output element, accumulating in exactly the
// reference's order -- fprop (c, kh, kw) with explicit zero products for padded
// taps (kernels.cpp:124-149), dgrad (f, kh, kw) skipping stride holes
// (kernels.cpp:174-203), wgrad (n, oh, ow) (kernels.cpp:225-251) -- so results
// are bitwise equal to the reference in either layout. (Products of E5M2 or FP16
// codes are exact in FP32, so fmaf == acc + x*w.)
#include "common.cuh"
#include "kernels.cuh"

namespace fp8b {

struct ConvDims {
    int64_t n, c, h, w, f, kh, kw, stride, pad, oh, ow;
    int nhwc;
};

__device__ __forceinline__ int64_t x_idx(const ConvDims& d, int64_t n, int64_t c, int64_t i,
                                         int64_t j) {
    return d.nhwc ? ((n * d.h + i) * d.w + j) * d.c + c : ((n * d.c + c) * d.h + i) * d.w + j;
}
__device__ __forceinline__ int64_t w_idx(const ConvDims& d, int64_t f, int64_t c, int64_t ki,
                                         int64_t kj) {
    return d.nhwc ? ((f * d.kh + ki) * d.kw + kj) * d.c + c : ((f * d.c + c) * d.kh + ki) * d.kw + kj;
}
__device__ __forceinline__ int64_t y_idx(const ConvDims& d, int64_t n, int64_t f, int64_t i,
                                         int64_t j) {
    return d.nhwc ? ((n * d.oh + i) * d.ow + j) * d.f + f : ((n * d.f + f) * d.oh + i) * d.ow + j;
}

template <int MB>
__device__ __forceinline__ float ld(const void* p, int64_t i) {
    return MB == 2 ? dec_e5m2(reinterpret_cast<const uint8_t*>(p)[i])
                   : dec_f16(reinterpret_cast<const uint16_t*>(p)[i]);
}

template <int MB>
__global__ void conv_fprop_seq(const void* __restrict__ x, const void* __restrict__ w,
                               float* __restrict__ y, ConvDims d) {
    const int64_t total = d.n * d.f * d.oh * d.ow;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t oj = t % d.ow, oi = (t / d.ow) % d.oh, fi = (t / (d.ow * d.oh)) % d.f,
                      ni = t / (d.ow * d.oh * d.f);
        float acc = 0.0f;
        for (int64_t ci = 0; ci < d.c; ++ci)
            for (int64_t ki = 0; ki < d.kh; ++ki) {
                const int64_t ii = oi * d.stride - d.pad + ki;
                for (int64_t kj = 0; kj < d.kw; ++kj) {
                    const int64_t jj = oj * d.stride - d.pad + kj;
                    float xv = 0.0f;
                    if (ii >= 0 && ii < d.h && jj >= 0 && jj < d.w) xv = ld<MB>(x, x_idx(d, ni, ci, ii, jj));
                    acc = fmaf(xv, ld<MB>(w, w_idx(d, fi, ci, ki, kj)), acc);
                }
            }
        y[y_idx(d, ni, fi, oi, oj)] = acc;
    }
}

template <int MB>
__global__ void conv_dgrad_seq(const void* __restrict__ e, const void* __restrict__ w,
                               float* __restrict__ dx, ConvDims d) {
    const int64_t total = d.n * d.c * d.h * d.w;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = t % d.w, i = (t / d.w) % d.h, ci = (t / (d.w * d.h)) % d.c,
                      ni = t / (d.w * d.h * d.c);
        float acc = 0.0f;
        for (int64_t fi = 0; fi < d.f; ++fi)
            for (int64_t ki = 0; ki < d.kh; ++ki)
                for (int64_t kj = 0; kj < d.kw; ++kj) {
                    const int64_t on = i + d.pad - ki, pn = j + d.pad - kj;
                    if (on % d.stride || pn % d.stride) continue;
                    const int64_t oi = on / d.stride, oj = pn / d.stride;
                    if (oi < 0 || oi >= d.oh || oj < 0 || oj >= d.ow) continue;
                    acc = fmaf(ld<MB>(w, w_idx(d, fi, ci, ki, kj)), ld<MB>(e, y_idx(d, ni, fi, oi, oj)), acc);
                }
        dx[x_idx(d, ni, ci, i, j)] = acc;
    }
}

template <int MB>
__global__ void conv_wgrad_seq(const void* __restrict__ x, const void* __restrict__ e,
                               float* __restrict__ dw, ConvDims d) {
    const int64_t total = d.f * d.c * d.kh * d.kw;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t kj = t % d.kw, ki = (t / d.kw) % d.kh, ci = (t / (d.kw * d.kh)) % d.c,
                      fi = t / (d.kw * d.kh * d.c);
        float acc = 0.0f;
        for (int64_t ni = 0; ni < d.n; ++ni)
            for (int64_t oi = 0; oi < d.oh; ++oi)
                for (int64_t oj = 0; oj < d.ow; ++oj) {
                    const int64_t ii = oi * d.stride - d.pad + ki, jj = oj * d.stride - d.pad + kj;
                    if (ii < 0 || ii >= d.h || jj < 0 || jj >= d.w) continue;
                    acc = fmaf(ld<MB>(x, x_idx(d, ni, ci, ii, jj)), ld<MB>(e, y_idx(d, ni, fi, oi, oj)), acc);
                }
        dw[w_idx(d, fi, ci, ki, kj)] = acc;
    }
}

static ConvDims dims_of(const fp8b_conv_t& g) {
    ConvDims d;
    d.n = g.n; d.c = g.c; d.h = g.h; d.w = g.w; d.f = g.f; d.kh = g.kh; d.kw = g.kw;
    d.stride = g.stride; d.pad = g.pad;
    d.oh = (g.h + 2 * g.pad - g.kh) / g.stride + 1;
    d.ow = (g.w + 2 * g.pad - g.kw) / g.stride + 1;
    d.nhwc = g.layout == FP8B_NHWC;
    return d;
}

static int grid_of(int64_t total) {
    int64_t b = (total + 255) / 256;
    if (b > 148 * 32) b = 148 * 32;
    return (int)(b < 1 ? 1 : b);
}

void launch_conv_seq(int kind, const void* a, const void* b, float* out, int fmt,
                     const fp8b_conv_t& g, cudaStream_t st) {
    const ConvDims d = dims_of(g);
    if (kind == 0) {
        const int gr = grid_of(d.n * d.f * d.oh * d.ow);
        if (fmt == FP8B_E5M2) conv_fprop_seq<2><<<gr, 256, 0, st>>>(a, b, out, d);
        else conv_fprop_seq<10><<<gr, 256, 0, st>>>(a, b, out, d);
    } else if (kind == 1) {
        const int gr = grid_of(d.n * d.c * d.h * d.w);
        if (fmt == FP8B_E5M2) conv_dgrad_seq<2><<<gr, 256, 0, st>>>(a, b, out, d);
        else conv_dgrad_seq<10><<<gr, 256, 0, st>>>(a, b, out, d);
    } else {
        const int gr = grid_of(d.f * d.c * d.kh * d.kw);
        if (fmt == FP8B_E5M2) conv_wgrad_seq<2><<<gr, 256, 0, st>>>(a, b, out, d);
        else conv_wgrad_seq<10><<<gr, 256, 0, st>>>(a, b, out, d);
    }
}

// im2col (kernels.cpp:64-104): pure code movement. NCHW -> the reference's
// [C*kH*kW, N*OH*OW]; NHWC -> [N*OH*OW, kH*kW*C].
template <typename T>
__global__ void im2col_kernel(const T* __restrict__ x, T* __restrict__ cols, ConvDims d) {
    const int64_t kk = d.c * d.kh * d.kw, pix = d.n * d.oh * d.ow, total = kk * pix;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        int64_t ci, ki, kj, p;
        if (d.nhwc) {
            p = t / kk;
            const int64_t r = t % kk;
            ci = r % d.c; kj = (r / d.c) % d.kw; ki = r / (d.c * d.kw);
        } else {
            const int64_t row = t / pix;
            p = t % pix;
            kj = row % d.kw; ki = (row / d.kw) % d.kh; ci = row / (d.kw * d.kh);
        }
        const int64_t oj = p % d.ow, oi = (p / d.ow) % d.oh, ni = p / (d.ow * d.oh);
        const int64_t ii = oi * d.stride - d.pad + ki, jj = oj * d.stride - d.pad + kj;
        T v = 0;
        if (ii >= 0 && ii < d.h && jj >= 0 && jj < d.w) v = x[x_idx(d, ni, ci, ii, jj)];
        cols[t] = v;
    }
}

void launch_im2col(const void* x, void* cols, int fmt, const fp8b_conv_t& g, cudaStream_t st) {
    const ConvDims d = dims_of(g);
    const int gr = grid_of(d.c * d.kh * d.kw * d.n * d.oh * d.ow);
    if (fmt == FP8B_E5M2)
        im2col_kernel<uint8_t><<<gr, 256, 0, st>>>((const uint8_t*)x, (uint8_t*)cols, d);
    else
        im2col_kernel<uint16_t><<<gr, 256, 0, st>>>((const uint16_t*)x, (uint16_t*)cols, d);
}

}  // namespace fp8b
