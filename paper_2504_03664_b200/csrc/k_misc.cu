// k_misc.cu — embedding gather (a4 PrepareInput), LayerNorm, greedy argmax (a13),
// int4 unpack+scale (kernel K8), GPU quantizer (a0 for synthetic loads) and fp16
// tiling.
#include <float.h>

#include "common.cuh"
#include "launch.cuh"
#include "kernels.h"
#include "layout.h"

namespace pipo {

// a4: h[m][:] = E_tok[id] + E_pos[past + t + 2]   ([ext] OPT learned positions, offset 2)
// tok is the fp16 tiled LM-head matrix (layout.h), pos row-major fp16.
__global__ void embed_kernel(const int32_t* ids, int n, int past, const __half* tok, int64_t n_kb,
                             const __half* pos, int d, float* h) {
  pdl_wait();
  pdl_trigger();
  const int m = blockIdx.x;
  const int t = m % n;
  const int64_t id = ids[m];
  const __half* prow = pos ? pos + (int64_t)(past + t + 2) * d : nullptr;   // LLaMA: no position table
  for (int k = threadIdx.x; k < d; k += blockDim.x) {
    const float a = __half2float(tok[fp16_tiled_index(id, k, n_kb)]);
    h[(int64_t)m * d + k] = prow ? a + __half2float(prow[k]) : a;
  }
}

int launch_embed(const int32_t* ids, int b, int n, int past, const __half* tok_tiled, int64_t tok_n_kb,
                 const __half* pos, int d, float* h, cudaStream_t st) {
  if (b * n <= 4096) launch_pdl_k(embed_kernel, dim3(b * n), dim3(256), 0, st, ids, n, past, tok_tiled, tok_n_kb, pos, d, h);
  else embed_kernel<<<b * n, 256, 0, st>>>(ids, n, past, tok_tiled, tok_n_kb, pos, d, h);
  return 1;
}

// LayerNorm (biased variance, eps 1e-5, [ext] nn.LayerNorm) of the fp32 residual
// stream, fp16 output for the next GEMM.  One CTA per row; two-pass statistics
// from registers; fixed-order block reduction (deterministic).
constexpr int LN_THREADS = 256;
constexpr int LN_MAX_PER_THREAD = 32;   // d <= 8192

__device__ __forceinline__ float block_sum(float v, float* red) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  float t = 0.f;
  for (int i = 0; i < LN_THREADS / 32; ++i) t += red[i];
  return t;
}

__global__ void __launch_bounds__(LN_THREADS) layernorm_kernel(const float* h, int64_t row_stride, int d,
                                                                 const __half* g, const __half* beta,
                                                                 __half* x) {
  // 16-B loads: float4 of h and 4 halves of gamma / beta per item, all issued before the
  // first reduction (one memory round trip); RMSNorm when beta == nullptr (mean = 0)
  constexpr int NV = LN_MAX_PER_THREAD / 4;   // float4 items per thread (d <= 8192)
  __shared__ float red[LN_THREADS / 32];
  pdl_wait();
  if (gridDim.x <= 1024) pdl_trigger();       // decode: one wave
  const float4* row = reinterpret_cast<const float4*>(h + blockIdx.x * row_stride);
  const int d4 = d >> 2;
  float4 v[NV];
  uint2 gv[NV], bv[NV];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int k = threadIdx.x + i * LN_THREADS;
    const bool in = k < d4;
    v[i] = in ? row[k] : make_float4(0.f, 0.f, 0.f, 0.f);
    gv[i] = in ? reinterpret_cast<const uint2*>(g)[k] : make_uint2(0, 0);
    bv[i] = in && beta ? reinterpret_cast<const uint2*>(beta)[k] : make_uint2(0, 0);
    s += (v[i].x + v[i].y) + (v[i].z + v[i].w);
  }
  const float mean = beta ? block_sum(s, red) / d : 0.f;
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    if (threadIdx.x + i * LN_THREADS < d4) {
      const float a = v[i].x - mean, b = v[i].y - mean, c = v[i].z - mean, e = v[i].w - mean;
      q = fmaf(a, a, q); q = fmaf(b, b, q); q = fmaf(c, c, q); q = fmaf(e, e, q);
    }
  }
  const float var = block_sum(q, red) / d;
  const float rstd = rsqrtf(var + 1e-5f);
  uint2* out = reinterpret_cast<uint2*>(x + (int64_t)blockIdx.x * d);
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int k = threadIdx.x + i * LN_THREADS;
    if (k < d4) {
      const float2 g01 = __half22float2(*reinterpret_cast<const __half2*>(&gv[i].x));
      const float2 g23 = __half22float2(*reinterpret_cast<const __half2*>(&gv[i].y));
      const float2 b01 = __half22float2(*reinterpret_cast<const __half2*>(&bv[i].x));
      const float2 b23 = __half22float2(*reinterpret_cast<const __half2*>(&bv[i].y));
      const __half2 o01 = __floats2half2_rn((v[i].x - mean) * rstd * g01.x + b01.x, (v[i].y - mean) * rstd * g01.y + b01.y);
      const __half2 o23 = __floats2half2_rn((v[i].z - mean) * rstd * g23.x + b23.x, (v[i].w - mean) * rstd * g23.y + b23.y);
      uint2 o;
      o.x = *reinterpret_cast<const uint32_t*>(&o01);
      o.y = *reinterpret_cast<const uint32_t*>(&o23);
      out[k] = o;
    }
  }
}

int launch_layernorm(const float* h, int64_t row_stride, int rows, int d, const __half* g,
                     const __half* beta, __half* x, cudaStream_t st) {
  if (d > LN_THREADS * LN_MAX_PER_THREAD) return -1;
  launch_pdl_k(layernorm_kernel, dim3(rows), dim3(LN_THREADS), 0, st, h, row_stride, d, g, beta, x);
  return 1;
}

// LLaMA RoPE (NEXT-4): one thread per (row, head, pair i); x1 = x[i], x2 = x[i + hd/2],
// angle = pos * inv_freq[i] in fp32 (sincosf, full precision), results rounded to fp16.
// q heads first, then the KV heads of the new K rows in the cache.
__global__ void rope_kernel(__half* q, __half* kc, const float* inv_freq, int n, int past, int n_heads,
                            int n_kv_heads, int hd, int kv_b, int64_t total) {
  pdl_wait();
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= total) return;
  const int half = hd >> 1;
  const int i = (int)(idx % half);
  const int64_t rest = idx / half;
  const int heads = n_heads + n_kv_heads;
  const int hh = (int)(rest % heads);
  const int m = (int)(rest / heads);
  const int bi = m / n, t = m - bi * n;
  __half* x = hh < n_heads ? q + (int64_t)m * n_heads * hd + hh * hd
                           : kc + ((int64_t)(past + t) * kv_b + bi) * n_kv_heads * hd + (hh - n_heads) * hd;
  float sn, cs;
  sincosf((float)(past + t) * inv_freq[i], &sn, &cs);
  const float x1 = __half2float(x[i]), x2 = __half2float(x[i + half]);
  x[i] = __float2half_rn(x1 * cs - x2 * sn);
  x[i + half] = __float2half_rn(x2 * cs + x1 * sn);
}

int launch_rope(__half* q, __half* kc, const float* inv_freq, int b, int n, int past, int n_heads, int n_kv_heads,
                int hd, int kv_b, cudaStream_t st) {
  const int64_t total = (int64_t)b * n * (n_heads + n_kv_heads) * (hd / 2);
  if (total == 0) return 0;
  launch_pdl_k(rope_kernel, dim3((unsigned)((total + 255) / 256)), dim3(256), 0, st, q, kc, inv_freq, n, past, n_heads,
               n_kv_heads, hd, kv_b, total);
  return 1;
}

// SwiGLU (NEXT-4): 8 features per thread (16-B loads of gate and up, 16-B store).
__global__ void swiglu_kernel(const __half* gu, int F, int64_t total8, __half* u) {
  pdl_wait();
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= total8) return;
  const int f8 = F / 8;
  const int64_t m = idx / f8;
  const int f = (int)(idx - m * f8) * 8;
  const int p = f >> 7, j = f & 127;
  const __half* row = gu + m * 2 * (int64_t)F;
  const uint4 gv = *reinterpret_cast<const uint4*>(row + p * 256 + j);
  const uint4 uv = *reinterpret_cast<const uint4*>(row + p * 256 + 128 + j);
  const __half2* g2 = reinterpret_cast<const __half2*>(&gv);
  const __half2* u2 = reinterpret_cast<const __half2*>(&uv);
  uint4 ov;
  __half2* o2 = reinterpret_cast<__half2*>(&ov);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float2 g = __half22float2(g2[k]), up = __half22float2(u2[k]);
    const float a = g.x / (1.f + expf(-g.x)) * up.x, c = g.y / (1.f + expf(-g.y)) * up.y;
    o2[k] = __floats2half2_rn(a, c);
  }
  *reinterpret_cast<uint4*>(u + m * F + f) = ov;
}

int launch_swiglu(const __half* gu, int M, int F, __half* u, cudaStream_t st) {
  const int64_t total8 = (int64_t)M * F / 8;
  if (total8 == 0) return 0;
  launch_pdl_k(swiglu_kernel, dim3((unsigned)((total8 + 255) / 256)), dim3(256), 0, st, gu, F, total8, u);
  return 1;
}

// a13: greedy next token = argmax over the vocabulary, lowest index on exact ties;
// NaN never wins.
__global__ void __launch_bounds__(1024) argmax_kernel(const float* logits, int V, int ldl, int32_t* out) {
  __shared__ float sv[32];
  __shared__ int si[32];
  pdl_wait();
  pdl_trigger();
  const float* row = logits + (int64_t)blockIdx.x * ldl;
  float best = -INFINITY;
  int bi = 0x7fffffff;
  for (int i = threadIdx.x; i < V; i += blockDim.x) {
    const float v = row[i];
    if (v > best || (v == best && i < bi)) { best = v; bi = i; }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) { sv[w] = best; si[w] = bi; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < (int)(blockDim.x >> 5); ++i)
      if (sv[i] > best || (sv[i] == best && si[i] < bi)) { best = sv[i]; bi = si[i]; }
    out[blockIdx.x] = bi == 0x7fffffff ? 0 : bi;
  }
}

int launch_argmax(const float* logits, int rows, int V, int ldl, int32_t* out, cudaStream_t st) {
  launch_pdl_k(argmax_kernel, dim3(rows), dim3(1024), 0, st, logits, V, ldl, out);
  return 1;
}

// K8: unpack + scale: out[r][k] = fp16_rne(q * s) (HMUL2 of exact q and s).
__global__ void unpack_int4_kernel(const uint8_t* codes, const uint16_t* scales, int64_t rows, int64_t cols,
                                   __half* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;   // one byte = 2 codes
  const int64_t nbytes = rows * cols / 2;
  if (i >= nbytes) return;
  const int64_t r = i / (cols / 2), kb = i - r * (cols / 2);
  const uint32_t b = codes[i];
  const __half s = __ushort_as_half(scales[r * (cols / 64) + (2 * kb) / 64]);
  const __half2 v = __hmul2(codes_to_half2((b & 0xFu) | ((b >> 4) << 16)), __half2half2(s));
  reinterpret_cast<__half2*>(out)[i] = v;
}

int launch_unpack_int4(const uint8_t* codes, const uint16_t* scales, int64_t rows, int64_t cols, __half* out,
                       cudaStream_t st) {
  const int64_t n = rows * cols / 2;
  unpack_int4_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(codes, scales, rows, cols, out);
  return 1;
}

// a0 on the GPU (same definition as the host packer):
// one thread per (row, group): a = max|g|; s = fp16_rne(a / 7.0f); q = clamp(rint(g/s)).
// IEEE division and RNE conversions are spelled out (no fast-math contraction).
// Output: canonical packed codes [rows][cols/2] + scales, and/or the tiled block.
__global__ void quantize_kernel(const float* w, int64_t rows, int64_t cols, uint8_t* codes, uint16_t* scales,
                                uint8_t* tiled, int* bad) {
  const int64_t gi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t ng = cols / 64;
  const int64_t rows_pad = (rows + 127) / 128 * 128;
  if (gi >= rows_pad * ng) return;
  const int64_t r = gi / ng, c = gi - r * ng;
  float g[64];
  float a = 0.f;
  bool finite = true;
  if (r < rows) {
    const float4* src = reinterpret_cast<const float4*>(w + r * cols + c * 64);
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const float4 v = src[i];
      g[4 * i] = v.x; g[4 * i + 1] = v.y; g[4 * i + 2] = v.z; g[4 * i + 3] = v.w;
    }
#pragma unroll
    for (int i = 0; i < 64; ++i) {
      finite = finite && isfinite(g[i]);
      a = fmaxf(a, fabsf(g[i]));
    }
  } else {
#pragma unroll
    for (int i = 0; i < 64; ++i) g[i] = 0.f;
  }
  const __half s16 = __float2half_rn(__fdiv_rn(a, 7.0f));
  const float s = __half2float(s16);
  if (!finite || isinf(s)) atomicExch(bad, 1);
  int q[64];
#pragma unroll
  for (int i = 0; i < 64; ++i)
    q[i] = s != 0.f ? (int)fminf(fmaxf(rintf(__fdiv_rn(g[i], s)), -8.f), 7.f) : 0;
  if (codes && r < rows) {
    uint32_t* cdst = reinterpret_cast<uint32_t*>(codes + r * (cols / 2) + c * 32);
#pragma unroll
    for (int wi = 0; wi < 8; ++wi) {
      uint32_t word = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) word |= (uint32_t)(q[wi * 8 + j] & 0xF) << (4 * j);
      cdst[wi] = word;
    }
    scales[r * ng + c] = __half_as_ushort(s16);
  }
  if (tiled) {
    uint32_t pw[8];
#pragma unroll
    for (int wi = 0; wi < 8; ++wi) pw[wi] = pack_tiled_word(q + wi * 8);
    uint8_t* blk = tiled + ((r >> 7) * ng + c) * kInt4BlockBytes;
    const int rr = (int)(r & 127);
    *reinterpret_cast<uint4*>(blk + (0 * 128 + rr) * 16) = make_uint4(pw[0], pw[1], pw[2], pw[3]);
    *reinterpret_cast<uint4*>(blk + (1 * 128 + rr) * 16) = make_uint4(pw[4], pw[5], pw[6], pw[7]);
    *reinterpret_cast<__half*>(blk + 4096 + rr * 2) = s16;
  }
}

int launch_quantize(const float* w, int64_t rows, int64_t cols, uint8_t* codes, uint16_t* scales,
                    uint8_t* tiled, int* bad_flag, cudaStream_t st) {
  const int64_t rows_pad = tiled ? (rows + 127) / 128 * 128 : rows;
  const int64_t n = rows_pad * (cols / 64);
  quantize_kernel<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(w, rows, cols, codes, scales, tiled, bad_flag);
  return 1;
}

// fp16 tiling of fp32 masters: element (r, k) -> block (r/128, k/64), row-major inside.
__global__ void tile_fp16_kernel(const float* w, int64_t rows, int64_t cols, __half* out) {
  const int64_t rows_pad = (rows + 127) / 128 * 128;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows_pad * cols) return;
  const int64_t r = i / cols, k = i - r * cols;
  out[fp16_tiled_index(r, k, cols / 64)] = __float2half_rn(r < rows ? w[r * cols + k] : 0.f);
}

int launch_tile_fp16(const float* w, int64_t rows, int64_t cols, uint8_t* tiled, cudaStream_t st) {
  const int64_t n = (rows + 127) / 128 * 128 * cols;
  tile_fp16_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(w, rows, cols, reinterpret_cast<__half*>(tiled));
  return 1;
}

__global__ void f32_to_f16_kernel(const float* s, __half* d, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) d[i] = __float2half_rn(s[i]);
}
__global__ void f16_to_f32_kernel(const __half* s, float* d, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) d[i] = __half2float(s[i]);
}
int launch_f32_to_f16(const float* src, __half* dst, int64_t n, cudaStream_t st) {
  f32_to_f16_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(src, dst, n);
  return 1;
}
int launch_f16_to_f32(const __half* src, float* dst, int64_t n, cudaStream_t st) {
  f16_to_f32_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(src, dst, n);
  return 1;
}

}  // namespace pipo

namespace pipo {

// ---- NEXT-1 peer transport: cross-process flags in peer (CUDA IPC) memory ----------
// One thread per flag: spin until *addr >= target (acquire at system scope: the flag
// lives in another process's — possibly another GPU's — memory, written after that
// process's copy engine filled the data it guards).
__global__ void p2p_wait_kernel(P2PFlags f, int target) {
  const int i = threadIdx.x;
  if (i >= f.n) return;
  const int* p = f.addr[i];
  int v;
  while (true) {
    asm volatile("ld.acquire.sys.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    if (v >= target) break;
    __nanosleep(256);
  }
}

// One thread per flag: publish `value` (release at system scope, after everything the
// stream ordered before this kernel — the copies it signals — has completed).
__global__ void p2p_signal_kernel(P2PFlags f, int value) {
  const int i = threadIdx.x;
  if (i >= f.n) return;
  __threadfence_system();
  asm volatile("st.release.sys.global.b32 [%0], %1;\n" ::"l"(f.addr[i]), "r"(value) : "memory");
}

int launch_p2p_wait(const P2PFlags& f, int target, cudaStream_t st) {
  if (f.n <= 0) return 0;
  p2p_wait_kernel<<<1, 32, 0, st>>>(f, target);
  return 1;
}

// ---- test hooks ------------------------------------------------
// A one-thread busy wait of `ns` nanoseconds on a stream: injected delays in the host
// tier (copy stream) or in the compute stream; the results must not change.
__global__ void spin_kernel(int64_t ns) {
  uint64_t t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    __nanosleep(1000);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  } while ((int64_t)(t - t0) < ns);
}

// Position-weighted 64-bit checksum of a byte range (multiple of 8 bytes), added into *out
// (zeroed by the caller): sum_i w_i * (2i + 1) mod 2^64 over its little-endian 64-bit words.
__global__ void ring_sum_kernel(const uint64_t* w, int64_t n_words, unsigned long long* out) {
  uint64_t acc = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_words; i += (int64_t)gridDim.x * blockDim.x)
    acc += w[i] * (uint64_t)(2 * i + 1);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, (unsigned long long)acc);
}

int launch_spin(int64_t ns, cudaStream_t st) {
  if (ns <= 0) return 0;
  spin_kernel<<<1, 1, 0, st>>>(ns);
  return 1;
}

int launch_ring_sum(const uint8_t* p, int64_t bytes, uint64_t* out, cudaStream_t st) {
  if (bytes % 8) return -1;
  if (cudaMemsetAsync(out, 0, 8, st) != cudaSuccess) return -1;
  ring_sum_kernel<<<148, 256, 0, st>>>(reinterpret_cast<const uint64_t*>(p), bytes / 8,
                                       reinterpret_cast<unsigned long long*>(out));
  return 1;
}

int launch_p2p_signal(const P2PFlags& f, int value, cudaStream_t st) {
  if (f.n <= 0) return 0;
  p2p_signal_kernel<<<1, 32, 0, st>>>(f, value);
  return 1;
}

}  // namespace pipo
