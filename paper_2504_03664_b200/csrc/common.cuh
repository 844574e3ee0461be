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

// Two int4 codes (bits 0-3 -> low half, bits 16-19 -> high half of `t`) to the
// exact fp16 pair (q_lo, q_hi): 0x6400|(c^8) is fp16 1024+(q+8); minus 1032 is q.
__device__ __forceinline__ __half2 codes_to_half2(uint32_t t) {
  t = (t ^ 0x00080008u) | 0x64006400u;
  __half2 h = *reinterpret_cast<__half2*>(&t);
  return __hsub2(h, __half2half2(__ushort_as_half(0x6408)));  // 1032.0
}

// 8 codes in one 32-bit word (byte j = codes 2j, 2j+1) -> 4 half2 = fp16_rne(q*s)
__device__ __forceinline__ void dequant8(uint32_t w, __half2 s2, __half2* out) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    uint32_t b = (w >> (8 * j)) & 0xFFu;
    uint32_t t = (b & 0xFu) | ((b >> 4) << 16);
    out[j] = __hmul2(codes_to_half2(t), s2);
  }
}

// code i (0..7) of a 32-bit word as a signed int (arithmetic shift sign-extends)
__device__ __forceinline__ int code_at(uint32_t w, int i) {
  return static_cast<int>(w << (28 - 4 * i)) >> 28;
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
