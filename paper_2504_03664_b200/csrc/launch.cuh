// launch.cuh — programmatic dependent launch (PDL) for the compute-stream kernels.
// A kernel launched with cudaLaunchAttributeProgrammaticStreamSerialization may be
// scheduled while its predecessor drains; pdl_wait() (griddepcontrol.wait) blocks until
// the predecessor grid has completed and its memory is visible, so it must precede every
// read of the predecessor's output and every global write.  pdl_trigger() lets this
// grid's own dependent be scheduled early: used only by single-wave kernels, whose
// dependents then cannot take SM slots from a later wave.  Both are no-ops when the
// kernel was launched without the attribute.
#pragma once
#include <cuda_runtime.h>

#include <cstdlib>

namespace pipo {

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                                Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  static const bool on = !getenv("PIPO_PDL") || atoi(getenv("PIPO_PDL")) != 0;   // PIPO_PDL=0: plain launches (A/B)
  cfg.numAttrs = on ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

}  // namespace pipo
