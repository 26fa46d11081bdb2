// fp8emu_b200.hpp -- the reference-side binding: fp8emu's own C++ API surface,
// served by the B200 kernels through the C-ABI (include/fp8b200.h).
//
// A maintainer of fp8emu (/root/reference/proj) adds this header and
// fp8emu_b200.cpp to the library. Every function keeps the
// reference signature, value semantics and error behaviour
// (std::invalid_argument where the reference throws it); the bodies copy the
// host tensors to HBM, launch the kernels and copy the results back.
//
//   reference                                  drop-in
//   fp8emu::quantize        tensor.hpp:59-60   fp8emu::b200::quantize
//   fp8emu::dequantize      tensor.hpp:63      fp8emu::b200::dequantize
//   fp8emu::transpose       tensor.hpp:73      fp8emu::b200::transpose
//   fp8emu::gemm_fp8        kernels.hpp:11     fp8emu::b200::gemm_fp8       (tcgen05, tolerance)
//                                              fp8emu::b200::gemm_fp8_exact (bitwise order)
//   fp8emu::LossScaler      loss_scaling.hpp   fp8emu::b200::LossScaler     (state in HBM)
//   update_tensor           nn.cpp:417-432     fp8emu::b200::update_tensor
//   fp8emu::conv2d_fp8 ...  kernels.hpp:22-50  fp8emu::b200::conv2d_fp8, im2col,
//                                              conv2d_fp8_im2col, conv2d_backward_data_fp8,
//                                              conv2d_backward_weights_fp8 (NCHW, bitwise)
#pragma once

#include <cstdint>
#include <vector>

#include "fp8emu/kernels.hpp"
#include "fp8emu/loss_scaling.hpp"
#include "fp8emu/nn.hpp"
#include "fp8emu/tensor.hpp"

namespace fp8emu {
namespace b200 {

QuantizedTensor quantize(const Tensor& t, const FloatFormat& fmt, const QuantConfig& cfg);
Tensor dequantize(const QuantizedTensor& q);
QuantizedTensor transpose(const QuantizedTensor& q);
Tensor gemm_fp8(const QuantizedTensor& a, const QuantizedTensor& b);
Tensor gemm_fp8_exact(const QuantizedTensor& a, const QuantizedTensor& b);

// The conv family in the reference's NCHW layout and summation order (bitwise).
Tensor conv2d_fp8(const QuantizedTensor& x, const QuantizedTensor& w, const ConvGeometry& geom);
QuantizedTensor im2col(const QuantizedTensor& x, std::int64_t kh, std::int64_t kw,
                       const ConvGeometry& geom);
Tensor conv2d_fp8_im2col(const QuantizedTensor& x, const QuantizedTensor& w,
                         const ConvGeometry& geom);
Tensor conv2d_backward_data_fp8(const QuantizedTensor& e, const QuantizedTensor& w,
                                const ConvGeometry& geom, std::int64_t h, std::int64_t w_dim);
Tensor conv2d_backward_weights_fp8(const QuantizedTensor& x, const QuantizedTensor& e,
                                   std::int64_t kh, std::int64_t kw, const ConvGeometry& geom);

class LossScaler {
public:
    explicit LossScaler(const fp8emu::LossScaler::Options& opts);
    ~LossScaler();
    LossScaler(const LossScaler&) = delete;
    LossScaler& operator=(const LossScaler&) = delete;
    double scale() const;
    double min_threshold(std::int64_t iteration) const;
    ScaleEvent step(bool grads_finite, std::int64_t iteration);
    Tensor unscale_gradients(const Tensor& g) const;
    void* device_state() const { return dev_; }

private:
    fp8emu::LossScaler::Options opts_;
    void* dev_ = nullptr;
};

// update_tensor semantics on one ParamTensor (FP16 master kept in p.master,
// p.value refreshed as decode(master)); master_mode Stochastic applies the
// BASELINE SR extension with the reference's block stream.
void update_tensor(nn::ParamTensor& p, const std::vector<float>& g, float scale, float lr,
                   float mu, float two_lambda,
                   RoundingMode master_mode = RoundingMode::NearestEven, std::uint64_t seed = 1);

}  // namespace b200
}  // namespace fp8emu
