// k_attn.cu — multi-head attention over the position-major KV cache
// (a7: "the GPU loading the required cache before computing the multi-head
// attention (MHA) layer", §3.1.1).  OPT attention ([ext]
// modeling_opt.py): softmax(q K^T) V per head, q pre-scaled by hd^-0.5 in the QKV
// epilogue, causal in prefill.  fp16 K/V, fp32 scores / softmax / accumulation.
//
// KV cache layout: [pos][kv_b][d] fp16 (position-major, reading Q18) so the first
// L positions of a layer are one contiguous range (one H2D copy for host-resident
// KV).  A head's row for (pos, b) is hd contiguous halves (128 or 256 B).
//
// Decode (flash-decoding): grid (head, b, split); each CTA scans a contiguous range
// of positions with 4 warps, each warp 4 positions per step (4 independent loads
// and reductions in flight), online softmax in fp32; warps merge in fixed order;
// splits merge in fixed order in a second kernel (log-sum-exp weights).
#include <float.h>

#include "common.cuh"
#include "kernels.h"

namespace pipo {

constexpr float kLog2e = 1.4426950408889634f;

template <int E>
__device__ __forceinline__ void load_row(const __half* p, float* out) {
  if constexpr (E == 2) {
    float2 v = __half22float2(*reinterpret_cast<const __half2*>(p));
    out[0] = v.x; out[1] = v.y;
  } else {
    uint2 raw = *reinterpret_cast<const uint2*>(p);
    float2 a = __half22float2(*reinterpret_cast<__half2*>(&raw.x));
    float2 b = __half22float2(*reinterpret_cast<__half2*>(&raw.y));
    out[0] = a.x; out[1] = a.y; out[2] = b.x; out[3] = b.y;
  }
}

template <int HD>
__global__ void __launch_bounds__(128) attn_decode_kernel(AttnArgs a, int n_splits, int pos_per_split) {
  constexpr int E = HD / 32;
  __shared__ float sm_m[4], sm_l[4];
  __shared__ float sm_acc[4][HD];
  const int head = blockIdx.x, bi = blockIdx.y, split = blockIdx.z;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int L = a.past + 1;
  const int lo = split * pos_per_split, hi = min(L, lo + pos_per_split);
  float q[E];
  load_row<E>(a.q + (int64_t)bi * a.d + head * HD + lane * E, q);
#pragma unroll
  for (int e = 0; e < E; ++e) q[e] *= kLog2e;   // scores in log2 units
  const int64_t pstride = (int64_t)a.kv_b * a.d;
  const __half* kbase = a.kc + (int64_t)bi * a.d + head * HD + lane * E;
  const __half* vbase = a.vc + (int64_t)bi * a.d + head * HD + lane * E;
  float m_run = -INFINITY, l_run = 0.f, acc[E];
#pragma unroll
  for (int e = 0; e < E; ++e) acc[e] = 0.f;
  for (int p0 = lo + 4 * warp; p0 < hi; p0 += 16) {
    float kr[4][E], vr[4][E], s[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int p = min(p0 + u, hi - 1);
      load_row<E>(kbase + p * pstride, kr[u]);
      load_row<E>(vbase + p * pstride, vr[u]);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      float t = 0.f;
#pragma unroll
      for (int e = 0; e < E; ++e) t = fmaf(q[e], kr[u][e], t);
      s[u] = t;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int u = 0; u < 4; ++u) s[u] += __shfl_xor_sync(0xffffffffu, s[u], o);
    float mx = m_run;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (p0 + u >= hi) s[u] = -INFINITY;
      mx = fmaxf(mx, s[u]);
    }
    const float corr = exp2f(m_run - mx);   // m_run=-inf, mx finite -> 0
    l_run *= corr;
#pragma unroll
    for (int e = 0; e < E; ++e) acc[e] *= corr;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const float pu = exp2f(s[u] - mx);     // -inf -> 0
      l_run += pu;
#pragma unroll
      for (int e = 0; e < E; ++e) acc[e] = fmaf(pu, vr[u][e], acc[e]);
    }
    m_run = mx;
  }
  if (lane == 0) { sm_m[warp] = m_run; sm_l[warp] = l_run; }
#pragma unroll
  for (int e = 0; e < E; ++e) sm_acc[warp][lane * E + e] = acc[e];
  __syncthreads();
  if (threadIdx.x < HD) {
    const int t = threadIdx.x;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < 4; ++w) M = fmaxf(M, sm_m[w]);
    float l = 0.f, o = 0.f;
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const float f = sm_m[w] == -INFINITY ? 0.f : exp2f(sm_m[w] - M);
      l += sm_l[w] * f;
      o += sm_acc[w][t] * f;
    }
    if (n_splits == 1) {
      a.o[(int64_t)bi * a.d + head * HD + t] = __float2half_rn(o / l);
    } else {
      float* part = a.ws + ((int64_t)(bi * a.n_heads + head) * n_splits + split) * (HD + 2);
      if (t == 0) { part[0] = M; part[1] = l; }
      part[2 + t] = o;
    }
  }
}

template <int HD>
__global__ void attn_merge_kernel(AttnArgs a, int n_splits) {
  const int head = blockIdx.x, bi = blockIdx.y, t = threadIdx.x;
  const float* base = a.ws + (int64_t)(bi * a.n_heads + head) * n_splits * (HD + 2);
  float M = -INFINITY;
  for (int s = 0; s < n_splits; ++s) M = fmaxf(M, base[s * (HD + 2)]);
  float l = 0.f, o = 0.f;
  for (int s = 0; s < n_splits; ++s) {
    const float* p = base + s * (HD + 2);
    const float f = p[0] == -INFINITY ? 0.f : exp2f(p[0] - M);
    l += p[1] * f;
    o += p[2 + t] * f;
  }
  a.o[(int64_t)bi * a.d + head * HD + t] = __float2half_rn(o / l);
}

// Prefill (causal): grid (head, b, ceil(n/32)); 8 warps x 4 query rows. Each warp
// streams positions 0..past+t_last once, sharing every K/V row load across its 4
// rows; row u ignores positions beyond past + t_u.
template <int HD>
__global__ void __launch_bounds__(256) attn_prefill_kernel(AttnArgs a) {
  constexpr int E = HD / 32;
  const int head = blockIdx.x, bi = blockIdx.y;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int t0 = blockIdx.z * 32 + warp * 4;
  if (t0 >= a.n) return;
  const int nrows = min(4, a.n - t0);
  float q[4][E];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int t = t0 + min(u, nrows - 1);
    load_row<E>(a.q + ((int64_t)bi * a.n + t) * a.d + head * HD + lane * E, q[u]);
#pragma unroll
    for (int e = 0; e < E; ++e) q[u][e] *= kLog2e;
  }
  const int64_t pstride = (int64_t)a.kv_b * a.d;
  const __half* kbase = a.kc + (int64_t)bi * a.d + head * HD + lane * E;
  const __half* vbase = a.vc + (int64_t)bi * a.d + head * HD + lane * E;
  float m_run[4], l_run[4], acc[4][E];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    m_run[u] = -INFINITY;
    l_run[u] = 0.f;
#pragma unroll
    for (int e = 0; e < E; ++e) acc[u][e] = 0.f;
  }
  const int pend = a.past + t0 + nrows;   // exclusive
  for (int p = 0; p < pend; ++p) {
    float kr[E], vr[E], s[4];
    load_row<E>(kbase + p * pstride, kr);
    load_row<E>(vbase + p * pstride, vr);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      float t = 0.f;
#pragma unroll
      for (int e = 0; e < E; ++e) t = fmaf(q[u][e], kr[e], t);
      s[u] = t;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int u = 0; u < 4; ++u) s[u] += __shfl_xor_sync(0xffffffffu, s[u], o);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (p > a.past + t0 + u) continue;   // causal (warp-uniform)
      const float mx = fmaxf(m_run[u], s[u]);
      const float corr = exp2f(m_run[u] - mx);
      const float pu = exp2f(s[u] - mx);
      l_run[u] = l_run[u] * corr + pu;
#pragma unroll
      for (int e = 0; e < E; ++e) acc[u][e] = fmaf(pu, vr[e], acc[u][e] * corr);
      m_run[u] = mx;
    }
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    if (u >= nrows) break;
    __half* op = a.o + ((int64_t)bi * a.n + t0 + u) * a.d + head * HD + lane * E;
    const float inv = 1.f / l_run[u];
#pragma unroll
    for (int e = 0; e < E; ++e) op[e] = __float2half_rn(acc[u][e] * inv);
  }
}

int launch_attention_decode(const AttnArgs& a, cudaStream_t st) {
  const int hd = a.d / a.n_heads;
  if (hd != 64 && hd != 128) return -1;
  const int L = a.past + 1;
  const int pairs = a.b * a.n_heads;
  const int target = a.num_sms * 8;
  int n_splits = pairs >= target ? 1 : (target + pairs - 1) / pairs;
  n_splits = max(1, min(n_splits, (L + 63) / 64));
  const int per = (L + n_splits - 1) / n_splits;
  n_splits = (L + per - 1) / per;
  if (n_splits > 1 && (int64_t)pairs * n_splits * (hd + 2) > a.ws_floats) return -1;
  dim3 grid(a.n_heads, a.b, n_splits);
  if (hd == 64) attn_decode_kernel<64><<<grid, 128, 0, st>>>(a, n_splits, per);
  else attn_decode_kernel<128><<<grid, 128, 0, st>>>(a, n_splits, per);
  if (n_splits == 1) return 1;
  dim3 g2(a.n_heads, a.b);
  if (hd == 64) attn_merge_kernel<64><<<g2, 64, 0, st>>>(a, n_splits);
  else attn_merge_kernel<128><<<g2, 128, 0, st>>>(a, n_splits);
  return 2;
}

int launch_attention_prefill(const AttnArgs& a, cudaStream_t st) {
  const int hd = a.d / a.n_heads;
  if (hd != 64 && hd != 128) return -1;
  dim3 grid(a.n_heads, a.b, (a.n + 31) / 32);
  if (hd == 64) attn_prefill_kernel<64><<<grid, 256, 0, st>>>(a);
  else attn_prefill_kernel<128><<<grid, 256, 0, st>>>(a);
  return 1;
}

}  // namespace pipo
