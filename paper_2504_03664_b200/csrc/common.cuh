// common.cuh — small sm_100a device helpers shared by the kernels.
#pragma once
#include <cuda_fp16.h>
#include <stdint.h>

namespace pipo {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// cp.async 16 B global -> shared; src_bytes = 0 zero-fills (ragged tails)
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes = 16) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(smem)), "l"(gmem),
               "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ uint4 ld_nc_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ void ldmatrix_x4(uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3,
                                            const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(smem_u32(p)));
}
__device__ __forceinline__ void ldmatrix_x2(uint32_t& r0, uint32_t& r1, const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];\n"
               : "=r"(r0), "=r"(r1)
               : "r"(smem_u32(p)));
}

// D[16x8] += A[16x16] (row) * B[16x8] (col), fp16 in, fp32 accumulate
__device__ __forceinline__ void mma_16816(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t lop3_and_or(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;   // (a & b) | c
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;\n" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

// One tiled-layout word (8 offset-binary codes, nibble order e0 e2 e4 e6 e1 e3 e5 e7,
// layout.h) -> 4 half2 = fp16_rne(q * s) in natural order (e0,e1) (e2,e3) (e4,e5) (e6,e7).
// 0x6400 | u is fp16 1024 + u; (1024 + u) - 1032 = q exactly; the high-nibble lanes hold
// 1024 + 16u, and (1024 + 16u) * 1/16 - 72 = q exactly (one HFMA2).  Then one HMUL2 by
// the group scale: the K8 unpack+scale arithmetic, bit for bit.
__device__ __forceinline__ void dequant8(uint32_t w, __half2 s2, __half2* out) {
  const uint32_t kMagic = 0x64006400u;
  const __half2 k1032 = __half2half2(__ushort_as_half(0x6408));      // 1032
  const __half2 k1_16 = __half2half2(__ushort_as_half(0x2C00));      // 1/16
  const __half2 km72 = __half2half2(__ushort_as_half(0xD480));       // -72
  const uint32_t w2 = w >> 8;
  uint32_t t0 = lop3_and_or(w, 0x000F000Fu, kMagic);
  uint32_t t1 = lop3_and_or(w, 0x00F000F0u, kMagic);
  uint32_t t2 = lop3_and_or(w2, 0x000F000Fu, kMagic);
  uint32_t t3 = lop3_and_or(w2, 0x00F000F0u, kMagic);
  const __half2 q01 = __hsub2(*reinterpret_cast<__half2*>(&t0), k1032);
  const __half2 q23 = __hfma2(*reinterpret_cast<__half2*>(&t1), k1_16, km72);
  const __half2 q45 = __hsub2(*reinterpret_cast<__half2*>(&t2), k1032);
  const __half2 q67 = __hfma2(*reinterpret_cast<__half2*>(&t3), k1_16, km72);
  out[0] = __hmul2(q01, s2);
  out[1] = __hmul2(q23, s2);
  out[2] = __hmul2(q45, s2);
  out[3] = __hmul2(q67, s2);
}

// signed code of element e (0..7, natural order) of a tiled-layout word
__device__ __forceinline__ int code_at(uint32_t w, int e) {
  const int pos = (e >> 1) + ((e & 1) << 2);            // e0->0 e1->4 e2->1 e3->5 ...
  return (int)((w >> (4 * pos)) & 0xFu) - 8;
}

// Two canonical (two's complement) codes, bits 0-3 -> low half, bits 16-19 -> high
// half, to the exact fp16 pair (q_lo, q_hi) (K8 unpack of the canonical format).
__device__ __forceinline__ __half2 codes_to_half2(uint32_t t) {
  t = (t ^ 0x00080008u) | 0x64006400u;
  __half2 h = *reinterpret_cast<__half2*>(&t);
  return __hsub2(h, __half2half2(__ushort_as_half(0x6408)));  // 1032.0
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

}  // namespace pipo
