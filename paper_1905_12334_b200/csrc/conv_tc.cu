// conv_tc.cu -- implicit-GEMM convolutions on tcgen05 (NHWC, E5M2, stride 1).
#include "common.cuh"
#include "kernels.cuh"

namespace fp8b {

int launch_conv_tc(int, const void*, const void*, float*, int, const fp8b_conv_t&, cudaStream_t,
                   int*) {
    return FP8B_ENOTSUP;
}

}  // namespace fp8b
