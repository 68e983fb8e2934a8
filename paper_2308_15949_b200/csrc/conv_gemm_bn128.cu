// Conv engine instantiations for 128-column tiles (see conv_gemm.cuh).
#include "conv_gemm.cuh"

namespace laud {
cudaError_t launch_conv_bn128(const ConvLaunch& c) { LAUD_BN_DISPATCH(128, 4, 2) }
}  // namespace laud
