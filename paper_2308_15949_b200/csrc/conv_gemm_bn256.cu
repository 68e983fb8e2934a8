// Conv engine instantiations for 256-column tiles (see conv_gemm.cuh).
#include "conv_gemm.cuh"

namespace laud {
cudaError_t launch_conv_bn256(const ConvLaunch& c) { LAUD_BN_DISPATCH(256, 3, 1) }
}  // namespace laud
