// Conv engine instantiations for 64-column tiles (see conv_gemm.cuh).
#include "conv_gemm.cuh"

namespace laud {
cudaError_t launch_conv_bn64(const ConvLaunch& c) { LAUD_BN_DISPATCH(64, 6, 4) }
}  // namespace laud
