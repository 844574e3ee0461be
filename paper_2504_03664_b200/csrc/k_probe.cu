// k_probe.cu — measurement aid (not on the hot path): how fast can one CTA per SM
// stream HBM into shared memory with cp.async.bulk + an mbarrier ring, as a function
// of request size and ring depth?  Sizes the weight pipeline of the decode GEMM.
#include "common.cuh"
#include "kernels.h"

namespace pipo {

__global__ void __launch_bounds__(128, 1) bulk_probe_kernel(const uint8_t* src, int64_t bytes_per_cta, int chunk,
                                                          int stages, int streams, uint32_t* sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)stages * chunk);
  uint64_t* empty = full + stages;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (tid == 0) {
    for (int i = 0; i < stages; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&full[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&empty[i])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const uint8_t* base = src + (int64_t)blockIdx.x * bytes_per_cta;
  const int n = (int)(bytes_per_cta / chunk);
  uint32_t acc = 0;
  if (warp == 0 && (tid & 31) == 0) {
    for (int i = 0; i < n; ++i) {
      const int s = i % stages;
      const uint32_t ph = ((i / stages) & 1) ^ 1;
      asm volatile("{\n.reg .pred P;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W_%=;\n}\n" ::"r"(
                       smem_u32(&empty[s])), "r"(ph) : "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(&full[s])), "r"(chunk)
                   : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                       smem_u32(sm + (size_t)s * chunk)),
                   // request i: stream i % streams (each stream one contiguous 1/streams of the
                   // CTA's region), like a CTA that consumes several weight row-tiles at once
                   "l"(base + (int64_t)(i % streams) * (bytes_per_cta / streams) + (int64_t)(i / streams) * chunk),
                   "r"(chunk), "r"(smem_u32(&full[s]))
                   : "memory");
    }
  } else if (warp == 1 && (tid & 31) == 0) {
    for (int i = 0; i < n; ++i) {
      const int s = i % stages;
      asm volatile("{\n.reg .pred P;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W_%=;\n}\n" ::"r"(
                       smem_u32(&full[s])), "r"((uint32_t)((i / stages) & 1)) : "memory");
      acc += sm[(size_t)s * chunk];
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(&empty[s])) : "memory");
    }
  }
  if (acc == 0xFFFFFFFFu) *sink = acc;
}

int launch_bulk_probe(const uint8_t* src, int64_t bytes_per_cta, int chunk, int stages, int streams, int ctas,
                      uint32_t* sink, cudaStream_t st) {
  const int smem = stages * chunk + 2 * stages * 8 + 64;
  if (smem > 227 * 1024) return -1;
  cudaFuncSetAttribute(bulk_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  bulk_probe_kernel<<<ctas, 128, smem, st>>>(src, bytes_per_cta, chunk, stages, streams, sink);
  return 1;
}

}  // namespace pipo
