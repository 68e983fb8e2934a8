// Kernel launches with programmatic dependent launch (PDL): each kernel of
// the block chain is launched with programmaticStreamSerialization, so its
// CTAs can be scheduled (and run their prologue: barrier init, TMEM alloc,
// descriptor prefetch) while the previous kernel drains; every such kernel
// executes griddepcontrol.wait (pdl_wait) before touching global memory the
// previous kernels produce or consume, which preserves stream order for the
// data.  Captured into CUDA graphs as programmatic edges.  LAUD_PDL=0 turns
// it off (plain stream-ordered launches).
#pragma once
#include <cuda_runtime.h>

#include <cstdlib>
#include <utility>

namespace laud {

inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("LAUD_PDL");
    return e ? std::atoi(e) != 0 : true;
  }();
  return on;
}

template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                     Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

}  // namespace laud
