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
#include <mutex>
#include <set>
#include <tuple>

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

// Plain launch (no PDL attribute) for multi-wave kernels that follow a one-wave GEMM: the
// decode attention launched as the QKV GEMM's programmatic dependent measured 197 us per
// c5 layer in the step against 161 us launched plainly (uninstrumented CUPTI, device
// tier; profiles/r02/pdl_attn/); its pdl_wait() is then a no-op.
template <typename... KArgs, typename... Args>
static cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                            Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.numAttrs = 0;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// cudaFuncAttributeMaxDynamicSharedMemorySize applies to the CURRENT device: track it per
// (device, kernel, size) so a second context on another GPU of the same process gets it
// too; thread-safe (contexts may live on different host threads).
template <typename... KArgs>
inline void ensure_max_smem(void (*kern)(KArgs...), int bytes) {
  static std::mutex mu;
  static std::set<std::tuple<int, const void*, int>> done;
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_tuple(dev, reinterpret_cast<const void*>(kern), bytes);
  std::lock_guard<std::mutex> g(mu);
  if (done.count(key)) return;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) == cudaSuccess) done.insert(key);
}

}  // namespace pipo
