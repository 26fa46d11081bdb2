// gemm_tc.cu -- placeholder until the tcgen05 engine lands.
#include "common.cuh"
#include "kernels.cuh"
namespace fp8b {
int launch_gemm_tc(const void*, const void*, int64_t, int64_t, int64_t, int, int, int,
                   const EpiArgs&, cudaStream_t, int* nlaunch) {
    *nlaunch = 0;
    return FP8B_ENOTSUP;
}
}  // namespace fp8b
