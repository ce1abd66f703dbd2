// pdl.cuh -- programmatic dependent launch for the small kernels between the
// GEMMs: each is launched with programmatic stream serialization, so its
// launch (and block scheduling) overlaps the tail of the previous kernel, and
// waits in griddepcontrol.wait -- before touching global memory -- until that
// kernel has completed and its writes are visible.
#pragma once

#include <cuda_runtime.h>

#include <utility>

namespace hm {

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args &&...args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

}  // namespace hm
