// Programmatic dependent launch (PDL) for the step's back-to-back kernels.
//
// A kernel launched with launch_pdl() may be scheduled while its predecessor
// on the stream is still draining: its CTAs land on SMs as they free up and
// run their prologue (mbarrier init, TMEM allocation, tensor-map prefetch)
// under the predecessor's tail.  Every such kernel MUST call pdl_wait()
// before it touches memory an earlier kernel writes — griddepcontrol.wait
// returns once the predecessor grid has completed and its writes are
// visible — and calls pdl_trigger() so its own successor can do the same.
// Both instructions are no-ops for a kernel launched without the attribute.
// MPRKB_PDL=0 launches everything plainly (A/B measurement).
#pragma once
#include <cuda_runtime.h>

#include <cstdlib>
#include <utility>

#include "types.hpp"

namespace mprkb {

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("MPRKB_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <class... KArgs, class... Args>
void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  CUDA_CHECK(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

}  // namespace mprkb
