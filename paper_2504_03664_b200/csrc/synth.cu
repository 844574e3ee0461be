// synth.cu — the library's own implementation of the seeded counter-based input
// generator described in pipo_synth/__init__.py.  This
// is INPUT GENERATION, not the method: it draws the synthetic OPT masters for
// pipo_load_synthetic() so the multi-GB configurations never need fp32 masters on
// the host.  The oracle side draws the same values with numpy; the two share no
// code, only the recipe:
//   mix64(z): z=(z^(z>>30))*0xBF58476D1CE4E5B9; z=(z^(z>>27))*0x94D049BB133111EB; z^(z>>31)
//   key = mix64(mix64(seed) ^ (slot << 16) ^ tid);   h(i) = mix64(key + (i+1)*0x9E3779B97F4A7C15)
//   normal : f16(f32(sum of the 4 16-bit fields - 131070) * scale)
//   uniform: f16(f32((h>>40) - 2^23) * scale);   gamma: f16(1 + f32((h>>40) - 2^23) * scale)
#include <math.h>

#include "kernels.h"

namespace pipo {

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

uint64_t synth_key(uint64_t seed, uint32_t slot, uint32_t tid) {
  return mix64(mix64(seed) ^ ((uint64_t)slot << 16) ^ (uint64_t)tid);
}

float synth_scale(int kind, double param) {
  if (kind == 0) return (float)(param / sqrt((65536.0 * 65536.0 - 1.0) / 3.0));
  return (float)(param / 8388608.0);
}

__global__ void synth_kernel(float* out, int64_t start, int64_t count, uint64_t key, int kind, float scale) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const uint64_t h = mix64(key + (uint64_t)(start + i + 1) * 0x9E3779B97F4A7C15ull);
  float v;
  if (kind == 0) {
    const int64_t s = (int64_t)(h & 0xFFFF) + (int64_t)((h >> 16) & 0xFFFF) + (int64_t)((h >> 32) & 0xFFFF) +
                      (int64_t)(h >> 48);
    v = __fmul_rn((float)(s - 131070), scale);
  } else {
    v = __fmul_rn((float)((int64_t)(h >> 40) - 8388608), scale);
    if (kind == 2) v = __fadd_rn(1.0f, v);
  }
  out[i] = __half2float(__float2half_rn(v));
}

int launch_synth(float* out, int64_t start, int64_t count, uint64_t key, int kind, float scale, cudaStream_t st) {
  synth_kernel<<<(unsigned)((count + 255) / 256), 256, 0, st>>>(out, start, count, key, kind, scale);
  return 1;
}

}  // namespace pipo
