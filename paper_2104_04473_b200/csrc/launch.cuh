// Kernel launches with programmatic dependent launch (PDL).
//
// Every kernel of the layer chain is launched with
// cudaLaunchAttributeProgrammaticStreamSerialization: the next kernel on the
// stream may be scheduled as soon as every CTA of the current one has started
// (griddepcontrol.launch_dependents at kernel entry), its CTAs then set up
// (shared memory, barriers, TMEM) and block in griddepcontrol.wait until the
// previous kernel has completed and its memory is visible.  This hides the
// launch latency and prologue of ~5000 kernel boundaries per training step.
// MP_NO_PDL=1 launches without the attribute (A/B).
#pragma once
#include <cuda_runtime.h>

#include <cstdlib>
#include <utility>

namespace mp {

inline bool pdl_enabled() {
  static const bool on = getenv("MP_NO_PDL") == nullptr;
  return on;
}

template <typename... KArgs, typename... Args>
inline void pdl_launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);   // errors surface through cudaGetLastError
}

// allow the next kernel to launch, then wait for the previous one (a no-op for a
// kernel launched without the PDL attribute)
__device__ __forceinline__ void pdl_entry() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

}  // namespace mp
