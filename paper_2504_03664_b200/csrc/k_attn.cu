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
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "launch.cuh"
#include "kernels.h"
#include "layout.h"

namespace pipo {

constexpr float kLog2e = 1.4426950408889634f;

// element strides of the K/V source: position-major cache by default
// GQA (LLaMA): K/V rows are dkv = n_kv_heads * hd wide and query head j
// reads KV head j / group; OPT is dkv = d, group = 1.
__device__ __forceinline__ int kv_width(const AttnArgs& a) { return a.dkv ? a.dkv : a.d; }
__device__ __forceinline__ int64_t kv_pstride(const AttnArgs& a) {
  return a.kv_pos_stride ? a.kv_pos_stride : (int64_t)a.kv_b * kv_width(a);
}
__device__ __forceinline__ int64_t kv_bstride(const AttnArgs& a) { return a.kv_b_stride ? a.kv_b_stride : kv_width(a); }

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

// G > 1 (GQA): one CTA per (KV head, b, split) serves the G query heads
// that share the KV head, so each K/V row is read from HBM once for all G heads (G = 1:
// blockIdx.x is the query head; a group size without a G instance also runs G = 1 with
// the head -> KV-head mapping, re-reading shared rows through L2).
template <int HD, int G>
__global__ void __launch_bounds__(128) attn_decode_kernel(AttnArgs a, int n_splits, int pos_per_split) {
  constexpr int E = HD / 32;
  __shared__ float sm_m[G][4], sm_l[G][4];
  __shared__ float sm_acc[G][4][HD];
  pdl_wait();   // multi-wave: no early trigger (dependents would take SM slots)
  const int bi = blockIdx.y, split = blockIdx.z;
  const int head0 = G == 1 ? blockIdx.x : blockIdx.x * G;            // first query head
  const int kvh = G == 1 ? blockIdx.x / a.group : blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int L = a.past + 1;
  const int lo = split * pos_per_split, hi = min(L, lo + pos_per_split);
  float q[G][E];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    load_row<E>(a.q + (int64_t)bi * a.d + (head0 + g) * HD + lane * E, q[g]);
#pragma unroll
    for (int e = 0; e < E; ++e) q[g][e] *= kLog2e;   // scores in log2 units
  }
  const int64_t pstride = kv_pstride(a);
  const __half* kbase = a.kc + (int64_t)bi * kv_bstride(a) + kvh * HD + lane * E;
  const __half* vbase = a.vc + (int64_t)bi * kv_bstride(a) + kvh * HD + lane * E;
  float m_run[G], l_run[G], acc[G][E];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    m_run[g] = -INFINITY;
    l_run[g] = 0.f;
#pragma unroll
    for (int e = 0; e < E; ++e) acc[g][e] = 0.f;
  }
  using Raw = typename std::conditional<E == 4, uint2, uint32_t>::type;
  auto fetch = [&](Raw (&kk)[4], Raw (&vv)[4], int p0) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int p = max(lo, min(p0 + u, hi - 1));
      kk[u] = *reinterpret_cast<const Raw*>(kbase + p * pstride);
      vv[u] = *reinterpret_cast<const Raw*>(vbase + p * pstride);
    }
  };
  auto decode = [&](const Raw& r, float* out) {
    if constexpr (E == 2) {
      const float2 v = __half22float2(*reinterpret_cast<const __half2*>(&r));
      out[0] = v.x; out[1] = v.y;
    } else {
      const float2 x = __half22float2(*reinterpret_cast<const __half2*>(&r.x));
      const float2 y = __half22float2(*reinterpret_cast<const __half2*>(&r.y));
      out[0] = x.x; out[1] = x.y; out[2] = y.x; out[3] = y.y;
    }
  };
  // one 4-position group: scores, online softmax, P.V (the group's raw rows in kk / vv)
  auto step = [&](const Raw (&kk)[4], const Raw (&vv)[4], int p0) {
    float kr[4][E], vr[4][E], s[G][4];
#pragma unroll
    for (int u = 0; u < 4; ++u) { decode(kk[u], kr[u]); decode(vv[u], vr[u]); }
#pragma unroll
    for (int g = 0; g < G; ++g)
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        float t = 0.f;
#pragma unroll
        for (int e = 0; e < E; ++e) t = fmaf(q[g][e], kr[u][e], t);
        s[g][u] = t;
      }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int g = 0; g < G; ++g)
#pragma unroll
        for (int u = 0; u < 4; ++u) s[g][u] += __shfl_xor_sync(0xffffffffu, s[g][u], o);
#pragma unroll
    for (int g = 0; g < G; ++g) {
      float mx = m_run[g];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (p0 + u >= hi) s[g][u] = -INFINITY;
        mx = fmaxf(mx, s[g][u]);
      }
      const float corr = exp2f(m_run[g] - mx);   // m_run=-inf, mx finite -> 0
      l_run[g] *= corr;
#pragma unroll
      for (int e = 0; e < E; ++e) acc[g][e] *= corr;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float pu = exp2f(s[g][u] - mx);     // -inf -> 0
        l_run[g] += pu;
#pragma unroll
        for (int e = 0; e < E; ++e) acc[g][e] = fmaf(pu, vr[u][e], acc[g][e]);
      }
      m_run[g] = mx;
    }
  };
  // raw K/V rows of the next 4-position group are loaded while the current group is
  // computed (register double buffer of the undecoded halves; a third buffer measured
  // 15 % slower at c5: 89 registers, 5 CTAs/SM; profiles/r02/attn_prefetch/)
  Raw kn[4], vn[4], kc_[4], vc_[4];
  if (lo + 4 * warp < hi) fetch(kn, vn, lo + 4 * warp);
  for (int p0 = lo + 4 * warp; p0 < hi; p0 += 16) {
#pragma unroll
    for (int u = 0; u < 4; ++u) { kc_[u] = kn[u]; vc_[u] = vn[u]; }
    if (p0 + 16 < hi) fetch(kn, vn, p0 + 16);
    step(kc_, vc_, p0);
  }
#pragma unroll
  for (int g = 0; g < G; ++g) {
    if (lane == 0) { sm_m[g][warp] = m_run[g]; sm_l[g][warp] = l_run[g]; }
#pragma unroll
    for (int e = 0; e < E; ++e) sm_acc[g][warp][lane * E + e] = acc[g][e];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < G * HD; i += 128) {
    const int g = i / HD, t = i - g * HD, head = head0 + g;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < 4; ++w) M = fmaxf(M, sm_m[g][w]);
    float l = 0.f, o = 0.f;
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const float f = sm_m[g][w] == -INFINITY ? 0.f : exp2f(sm_m[g][w] - M);
      l += sm_l[g][w] * f;
      o += sm_acc[g][w][t] * f;
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


// Decode v2: LPR = HD/8 lanes per K/V row (16-B loads of 8 halves), so one warp
// instruction fetches RPW = 32/LPR rows.  Each lane group ("virtual warp" of LPR lanes)
// runs its own online softmax over an interleaved subset of positions, 4 positions per
// step (8 x 16-B loads in flight per lane); the NV = 4*RPW virtual warps of the CTA are
// merged in fixed order, splits in a second kernel (deterministic).
template <int HD, int G>
__global__ void __launch_bounds__(128) attn_decode_v2_kernel(AttnArgs a, int n_splits, int pos_per_split) {
  // G > 1 (GQA): as in attn_decode_kernel, one CTA per (KV head, b, split) serves the G
  // query heads sharing the KV head; the lane-group layout needs log2(HD/8) shuffle steps
  // per (head, position) instead of 5, which is what GQA's G-fold dot products need
  constexpr int LPR = HD / 8, RPW = 32 / LPR, NV = 4 * RPW;
  __shared__ float sm_m[G][NV], sm_l[G][NV];
  __shared__ float sm_acc[G][NV][HD];
  pdl_wait();
  const int bi = blockIdx.y, split = blockIdx.z;
  const int head0 = G == 1 ? blockIdx.x : blockIdx.x * G;
  const int kvh = G == 1 ? blockIdx.x / a.group : blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int sub = lane / LPR, sl = lane % LPR;            // row slot within the warp, lane within row
  const int vw = warp * RPW + sub;                          // virtual warp id 0..NV-1
  const int L = a.past + 1;
  const int lo = split * pos_per_split, hi = min(L, lo + pos_per_split);
  float q[G][8];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const uint4 qr = *reinterpret_cast<const uint4*>(a.q + (int64_t)bi * a.d + (head0 + g) * HD + sl * 8);
    const __half2* qh = reinterpret_cast<const __half2*>(&qr);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 f = __half22float2(qh[e]);
      q[g][2 * e] = f.x * kLog2e;
      q[g][2 * e + 1] = f.y * kLog2e;
    }
  }
  const int64_t pstride = kv_pstride(a);
  const __half* kbase = a.kc + (int64_t)bi * kv_bstride(a) + kvh * HD + sl * 8;
  const __half* vbase = a.vc + (int64_t)bi * kv_bstride(a) + kvh * HD + sl * 8;
  float m_run[G], l_run[G], acc[G][8];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    m_run[g] = -INFINITY;
    l_run[g] = 0.f;
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[g][e] = 0.f;
  }
  constexpr int U = 4;
  // the trip count must be warp-uniform (full-mask shuffles): loop on the warp's first
  // position, each lane group masks its own positions past `hi`
  for (int pw = lo + warp * RPW * U; pw < hi; pw += NV * U) {
    const int p0 = pw + sub * U;
    uint4 kr[U], vr[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int p = min(p0 + u, hi - 1);
      kr[u] = ld_nc_v4(kbase + p * pstride);
      vr[u] = ld_nc_v4(vbase + p * pstride);
    }
    float s[G][U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const __half2* kh = reinterpret_cast<const __half2*>(&kr[u]);
      float2 kf[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) kf[e] = __half22float2(kh[e]);
#pragma unroll
      for (int g = 0; g < G; ++g) {
        float t = 0.f;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          t = fmaf(q[g][2 * e], kf[e].x, t);
          t = fmaf(q[g][2 * e + 1], kf[e].y, t);
        }
        s[g][u] = t;
      }
    }
#pragma unroll
    for (int o = LPR / 2; o > 0; o >>= 1)
#pragma unroll
      for (int g = 0; g < G; ++g)
#pragma unroll
        for (int u = 0; u < U; ++u) s[g][u] += __shfl_xor_sync(0xffffffffu, s[g][u], o);
#pragma unroll
    for (int g = 0; g < G; ++g) {
      float mx = m_run[g];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (p0 + u >= hi) s[g][u] = -INFINITY;
        mx = fmaxf(mx, s[g][u]);
      }
      const float corr = mx == -INFINITY ? 1.f : exp2f(m_run[g] - mx);   // group may have no live position yet
      l_run[g] *= corr;
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[g][e] *= corr;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const float pu = s[g][u] == -INFINITY ? 0.f : exp2f(s[g][u] - mx);
        l_run[g] += pu;
        const __half2* vh = reinterpret_cast<const __half2*>(&vr[u]);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 f = __half22float2(vh[e]);
          acc[g][2 * e] = fmaf(pu, f.x, acc[g][2 * e]);
          acc[g][2 * e + 1] = fmaf(pu, f.y, acc[g][2 * e + 1]);
        }
      }
      m_run[g] = mx;
    }
  }
#pragma unroll
  for (int g = 0; g < G; ++g) {
    if (sl == 0) { sm_m[g][vw] = m_run[g]; sm_l[g][vw] = l_run[g]; }
#pragma unroll
    for (int e = 0; e < 8; ++e) sm_acc[g][vw][sl * 8 + e] = acc[g][e];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < G * HD; i += 128) {
    const int g = i / HD, t = i - g * HD, head = head0 + g;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < NV; ++w) M = fmaxf(M, sm_m[g][w]);
    float l = 0.f, o = 0.f;
#pragma unroll
    for (int w = 0; w < NV; ++w) {
      const float f = sm_m[g][w] == -INFINITY ? 0.f : exp2f(sm_m[g][w] - M);
      l += sm_l[g][w] * f;
      o += sm_acc[g][w][t] * f;
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

// GQA decode on tensor cores, transposed (S^T = K q^T, O^T = V^T P^T): the
// positions are the 16-row M dimension and the G <= 8 query heads of the KV head the
// n = 8 dimension of mma.sync m16n8k16, so no M rows are padding: per 16 positions a warp
// issues HD/16 mma for the scores and HD/16 for P.V (round 1's kernel with the heads on M:
// HD/8 and HD/4 per 8 positions, half of each on zero rows; 4-7 % slower, removed).  K tiles are the A operand as stored
// (ldmatrix), V^T is ldmatrix.trans of the stored V tile, q^T sits in registers as the B
// operand (rows >= G zero), and the score accumulator becomes P^T's B fragment with one
// movmatrix.trans per 8 x 8 half.  Per-head softmax (fp32, log2 domain, P rounded to
// fp16) reduces over the 8 lanes that share a head column.  NW warps per CTA, each 16
// positions of a 16*NW-position tile, NS-stage cp.async ring; warps merge in fixed order
// through shared memory, splits in attn_merge_kernel.
__device__ __forceinline__ uint32_t movmatrix_t(uint32_t x) {
  uint32_t y;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;\n" : "=r"(y) : "r"(x));
  return y;
}

template <int HD, int NW, int NS>
__global__ void __launch_bounds__(NW * 32) attn_decode_gqa_st_kernel(AttnArgs a, int n_splits, int pos_per_split) {
  constexpr int KP = HD + 8;
  constexpr int CH = HD / 8;
  constexpr int T = 16 * NW;
  constexpr int NTH = NW * 32;
  constexpr int MT = HD / 16;
  extern __shared__ __align__(16) uint8_t smem_attn[];
  __half* sK = reinterpret_cast<__half*>(smem_attn);           // [NS][T][KP]
  __half* sV = sK + NS * T * KP;                               // [NS][T][KP]
  float* sM = reinterpret_cast<float*>(sV + NS * T * KP);      // [NW][8 heads]
  float* sL = sM + NW * 8;
  float* sO = reinterpret_cast<float*>(sK);                    // [NW][8][HD], reuses sK after the loop
  static_assert(NW * 8 * HD * 4 <= NS * T * KP * 2, "merge buffer fits in sK");
  pdl_wait();
  const int kvh = blockIdx.x, bi = blockIdx.y, split = blockIdx.z;
  const int G = a.group;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, tq = lane & 3, mi = lane >> 3, r8 = lane & 7;
  const int L = a.past + 1;
  const int lo = split * pos_per_split, hi = min(L, lo + pos_per_split);
  const int n_kv = (hi - lo + T - 1) / T;
  const int64_t pstride = kv_pstride(a), bstride = kv_bstride(a);
  auto load_kv = [&](int j, int buf) {
    for (int c = tid; c < T * CH; c += NTH) {
      const int r = c / CH, ch = c % CH, p = lo + j * T + r;
      const int64_t off = (int64_t)min(p, hi - 1) * pstride + (int64_t)bi * bstride + kvh * HD + ch * 8;
      const int bytes = p < hi ? 16 : 0;
      cp_async16(sK + (buf * T + r) * KP + ch * 8, a.kc + off, bytes);
      cp_async16(sV + (buf * T + r) * KP + ch * 8, a.vc + off, bytes);
    }
  };
#pragma unroll
  for (int st = 0; st < NS - 1; ++st) {
    if (st < n_kv) load_kv(st, st);
    cp_async_commit();
  }
  // B fragments of q^T: column g = query head kvh*G + g when g < G, else zero
  uint32_t qf[MT][2];
  {
    const __half* qrow = a.q + (int64_t)bi * a.d + (kvh * G + min(g, G - 1)) * HD;
#pragma unroll
    for (int kk = 0; kk < MT; ++kk) {
      qf[kk][0] = g < G ? *reinterpret_cast<const uint32_t*>(qrow + kk * 16 + 2 * tq) : 0u;
      qf[kk][1] = g < G ? *reinterpret_cast<const uint32_t*>(qrow + kk * 16 + 8 + 2 * tq) : 0u;
    }
  }
  float o[MT][4];   // O^T: rows hd 16i+g (+8), columns heads 2tq, 2tq+1
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int c = 0; c < 4; ++c) o[i][c] = 0.f;
  float m_r[2] = {-INFINITY, -INFINITY}, l_r[2] = {0.f, 0.f};   // heads 2tq, 2tq+1 (l: my positions)
  for (int j = 0; j < n_kv; ++j) {
    const int buf = j % NS;
    if (j + NS - 1 < n_kv) load_kv(j + NS - 1, (j + NS - 1) % NS);
    cp_async_commit();
    cp_async_wait<NS - 1>();
    __syncthreads();
    // S^T (16 positions x 8 heads): two accumulators halve the dependent mma chain
    float s0[4] = {0.f, 0.f, 0.f, 0.f}, s1[4] = {0.f, 0.f, 0.f, 0.f};
    const __half* kb = sK + (buf * T + warp * 16) * KP;
#pragma unroll
    for (int kk = 0; kk < MT; ++kk) {
      uint32_t af[4];
      ldmatrix_x4(af[0], af[1], af[2], af[3], kb + ((mi & 1) * 8 + r8) * KP + kk * 16 + (mi >> 1) * 8);
      mma_16816(kk & 1 ? s1 : s0, af, qf[kk][0], qf[kk][1]);
    }
    const int p0 = lo + j * T + warp * 16 + g;
    float sc[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) sc[c] = (p0 + (c >> 1) * 8) < hi ? (s0[c] + s1[c]) * kLog2e : -INFINITY;
    float mx[2], corr[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      float m = fmaxf(m_r[h], fmaxf(sc[h], sc[h + 2]));
      m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 4));
      m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 8));
      m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 16));
      mx[h] = m;
      corr[h] = m == -INFINITY ? 1.f : exp2f(m_r[h] - m);
      m_r[h] = m;
      l_r[h] *= corr[h];
    }
    float e[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) e[c] = mx[c & 1] == -INFINITY ? 0.f : exp2f(sc[c] - mx[c & 1]);
    l_r[0] += e[0] + e[2];
    l_r[1] += e[1] + e[3];
#pragma unroll
    for (int i = 0; i < MT; ++i) {
      o[i][0] *= corr[0]; o[i][1] *= corr[1]; o[i][2] *= corr[0]; o[i][3] *= corr[1];
    }
    __half2 top = __floats2half2_rn(e[0], e[1]), bot = __floats2half2_rn(e[2], e[3]);
    const uint32_t pb0 = movmatrix_t(*reinterpret_cast<uint32_t*>(&top));   // P^T rows 2tq.. (positions 0-7)
    const uint32_t pb1 = movmatrix_t(*reinterpret_cast<uint32_t*>(&bot));   // positions 8-15
    const __half* vb = sV + (buf * T + warp * 16) * KP;
#pragma unroll
    for (int i = 0; i < MT; ++i) {
      uint32_t af[4];
      const __half* ptr = vb + ((mi >> 1) * 8 + r8) * KP + i * 16 + (mi & 1) * 8;
      asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                   : "=r"(af[0]), "=r"(af[1]), "=r"(af[2]), "=r"(af[3])
                   : "r"(smem_u32(ptr)));
      mma_16816(o[i], af, pb0, pb1);
    }
    __syncthreads();
  }
  cp_async_wait<0>();
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    l_r[h] += __shfl_xor_sync(0xffffffffu, l_r[h], 4);
    l_r[h] += __shfl_xor_sync(0xffffffffu, l_r[h], 8);
    l_r[h] += __shfl_xor_sync(0xffffffffu, l_r[h], 16);
  }
  __syncthreads();
  if (g == 0) {
    sM[warp * 8 + 2 * tq] = m_r[0]; sM[warp * 8 + 2 * tq + 1] = m_r[1];
    sL[warp * 8 + 2 * tq] = l_r[0]; sL[warp * 8 + 2 * tq + 1] = l_r[1];
  }
  if (2 * tq < G) {
    float* o0 = sO + (warp * 8 + 2 * tq) * HD;
#pragma unroll
    for (int i = 0; i < MT; ++i) {
      o0[16 * i + g] = o[i][0]; o0[HD + 16 * i + g] = o[i][1];
      o0[16 * i + g + 8] = o[i][2]; o0[HD + 16 * i + g + 8] = o[i][3];
    }
  }
  __syncthreads();
  for (int i = tid; i < G * HD; i += NTH) {
    const int r = i / HD, t = i - r * HD, head = kvh * G + r;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < NW; ++w) M = fmaxf(M, sM[w * 8 + r]);
    float l = 0.f, ov = 0.f;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const float f = sM[w * 8 + r] == -INFINITY ? 0.f : exp2f(sM[w * 8 + r] - M);
      l += sL[w * 8 + r] * f;
      ov += sO[(w * 8 + r) * HD + t] * f;
    }
    if (n_splits == 1) {
      a.o[(int64_t)bi * a.d + head * HD + t] = __float2half_rn(ov / l);
    } else {
      float* part = a.ws + ((int64_t)(bi * a.n_heads + head) * n_splits + split) * (HD + 2);
      if (t == 0) { part[0] = M; part[1] = l; }
      part[2 + t] = ov;
    }
  }
}

template <int HD>
__global__ void attn_merge_kernel(AttnArgs a, int n_splits) {
  pdl_wait();
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
  const int64_t pstride = kv_pstride(a);
  const __half* kbase = a.kc + (int64_t)bi * kv_bstride(a) + (head / a.group) * HD + lane * E;
  const __half* vbase = a.vc + (int64_t)bi * kv_bstride(a) + (head / a.group) * HD + lane * E;
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


// Prefill (causal) on tensor cores, flash-attention-2 style (mma.sync m16n8k16,
// fp16 in / fp32 accumulate): CTA = (head, sequence, 64 query rows), 4 warps x 16
// rows; K/V tiles of 64 positions double-buffered with cp.async; online softmax on
// the S fragments in fp32 (exp2 with log2e folded in); P re-packed to fp16 A
// fragments for P.V; V fragments via ldmatrix.trans from the position-major cache.
template <int HD>
__global__ void __launch_bounds__(128) attn_prefill_mma_kernel(AttnArgs a) {
  constexpr int KP = HD + 8;                 // padded smem row (halves): conflict-free ldmatrix
  constexpr int NT_O = HD / 8;               // n8 tiles of the output
  extern __shared__ __align__(16) uint8_t smem_attn[];
  __half* sQ = reinterpret_cast<__half*>(smem_attn);          // [64][KP]
  __half* sK = sQ + 64 * KP;                                   // [2][64][KP]
  __half* sV = sK + 2 * 64 * KP;                               // [2][64][KP]
  const int head = blockIdx.x, bi = blockIdx.y, qt = blockIdx.z;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, tq = lane & 3;
  const int q0 = qt * 64;
  const int L = a.past + a.n;
  const int kv_end = min(L, a.past + min(a.n, q0 + 64));     // exclusive, causal bound of this CTA
  const int n_kv = (kv_end + 63) / 64;
  const int64_t pstride = kv_pstride(a), bstride = kv_bstride(a);
  constexpr int CH = HD / 8;                 // 16-B chunks per row

  for (int c = tid; c < 64 * CH; c += 128) {
    const int r = c / CH, ch = c % CH, t = q0 + r;
    const __half* src = a.q + ((int64_t)bi * a.n + min(t, a.n - 1)) * a.d + head * HD + ch * 8;
    cp_async16(sQ + r * KP + ch * 8, src, t < a.n ? 16 : 0);
  }
  auto load_kv = [&](int j, int buf) {
    for (int c = tid; c < 64 * CH; c += 128) {
      const int r = c / CH, ch = c % CH, p = j * 64 + r;
      const int64_t off = (int64_t)min(p, L - 1) * pstride + (int64_t)bi * bstride + (head / a.group) * HD + ch * 8;
      const int bytes = p < L ? 16 : 0;
      cp_async16(sK + (buf * 64 + r) * KP + ch * 8, a.kc + off, bytes);
      cp_async16(sV + (buf * 64 + r) * KP + ch * 8, a.vc + off, bytes);
    }
  };
  load_kv(0, 0);
  cp_async_commit();

  float o[NT_O][4];
#pragma unroll
  for (int i = 0; i < NT_O; ++i)
#pragma unroll
    for (int c = 0; c < 4; ++c) o[i][c] = 0.f;
  float m_r[2] = {-INFINITY, -INFINITY}, l_r[2] = {0.f, 0.f};
  uint32_t qf[HD / 16][4];
  const int row0 = q0 + warp * 16 + g;          // query rows of this thread: row0, row0 + 8

  for (int j = 0; j < n_kv; ++j) {
    const int buf = j & 1;
    if (j + 1 < n_kv) load_kv(j + 1, buf ^ 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    if (j == 0) {
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk)
        ldmatrix_x4(qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3],
                    sQ + (warp * 16 + (lane & 15)) * KP + kk * 16 + (lane >> 4) * 8);
    }
    // S = Q K^T for 64 positions
    float sc[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int c = 0; c < 4; ++c) sc[i][c] = 0.f;
    const __half* kb = sK + buf * 64 * KP;
#pragma unroll
    for (int kk = 0; kk < HD / 16; ++kk) {
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) {
        uint32_t b0, b1, b2, b3;
        ldmatrix_x4(b0, b1, b2, b3,
                    kb + (jj * 16 + (lane & 7) + ((lane >> 4) << 3)) * KP + kk * 16 + ((lane >> 3) & 1) * 8);
        mma_16816(sc[2 * jj], qf[kk], b0, b1);
        mma_16816(sc[2 * jj + 1], qf[kk], b2, b3);
      }
    }
    // mask + online softmax (log2 domain)
    float mx[2] = {m_r[0], m_r[1]};
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int p = j * 64 + i * 8 + 2 * tq + (c & 1);
        const int t = row0 + (c >> 1) * 8;
        const bool ok = p < L && p <= a.past + t;
        sc[i][c] = ok ? sc[i][c] * kLog2e : -INFINITY;
        mx[c >> 1] = fmaxf(mx[c >> 1], sc[i][c]);
      }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      mx[h] = fmaxf(mx[h], __shfl_xor_sync(0xffffffffu, mx[h], 1));
      mx[h] = fmaxf(mx[h], __shfl_xor_sync(0xffffffffu, mx[h], 2));
    }
    float corr[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      corr[h] = mx[h] == -INFINITY ? 1.f : exp2f(m_r[h] - mx[h]);
      m_r[h] = mx[h];
      l_r[h] *= corr[h];
    }
#pragma unroll
    for (int i = 0; i < NT_O; ++i) {
      o[i][0] *= corr[0]; o[i][1] *= corr[0];
      o[i][2] *= corr[1]; o[i][3] *= corr[1];
    }
    uint32_t pf[4][4];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float e[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const float mm = m_r[c >> 1];
        e[c] = mm == -INFINITY ? 0.f : exp2f(sc[i][c] - mm);
        l_r[c >> 1] += e[c];
      }
      const __half2 lo = __floats2half2_rn(e[0], e[1]), hi = __floats2half2_rn(e[2], e[3]);
      const int kk2 = i >> 1;
      if ((i & 1) == 0) {
        pf[kk2][0] = *reinterpret_cast<const uint32_t*>(&lo);
        pf[kk2][1] = *reinterpret_cast<const uint32_t*>(&hi);
      } else {
        pf[kk2][2] = *reinterpret_cast<const uint32_t*>(&lo);
        pf[kk2][3] = *reinterpret_cast<const uint32_t*>(&hi);
      }
    }
    // O += P V
    const __half* vb = sV + buf * 64 * KP;
#pragma unroll
    for (int kk2 = 0; kk2 < 4; ++kk2) {
#pragma unroll
      for (int nt2 = 0; nt2 < HD / 16; ++nt2) {
        uint32_t b0, b1, b2, b3;
        const __half* ptr = vb + (kk2 * 16 + (lane & 7) + ((lane >> 3) & 1) * 8) * KP + nt2 * 16 + (lane >> 4) * 8;
        asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                     : "=r"(b0), "=r"(b1), "=r"(b2), "=r"(b3)
                     : "r"(smem_u32(ptr)));
        mma_16816(o[2 * nt2], pf[kk2], b0, b1);
        mma_16816(o[2 * nt2 + 1], pf[kk2], b2, b3);
      }
    }
    __syncthreads();
  }
  cp_async_wait<0>();
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    l_r[h] += __shfl_xor_sync(0xffffffffu, l_r[h], 1);
    l_r[h] += __shfl_xor_sync(0xffffffffu, l_r[h], 2);
  }
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int t = row0 + h * 8;
    if (t >= a.n) continue;
    const float inv = 1.f / l_r[h];
    __half* op = a.o + ((int64_t)bi * a.n + t) * a.d + head * HD;
#pragma unroll
    for (int i = 0; i < NT_O; ++i)
      *reinterpret_cast<__half2*>(op + i * 8 + 2 * tq) = __floats2half2_rn(o[i][2 * h] * inv, o[i][2 * h + 1] * inv);
  }
}

// ---------------------------------------------------------------------------------
// INT4 KV cache (NEXT-2; "quantizing both weights and KV-cache to INT4").
// Cache rows use the weights' encoding: 64-feature groups, fp16 scale = absmax/7,
// codes stored offset-binary in the fast nibble order (layout.h) so dequant8 applies.

// one thread per (row, K|V, group): fresh fp16 K/V from the staging buffer -> cache
__global__ void kv_quant_kernel(const __half* staging, int b, int n, int past, int d, int kv_b, uint8_t* kq,
                                __half* ks, uint8_t* vq, __half* vs) {
  const int ng = d / 64;
  const int64_t gi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gi >= (int64_t)b * n * 2 * ng) return;
  const int g = (int)(gi % ng);
  const int w = (int)((gi / ng) % 2);
  const int64_t m = gi / (2 * ng);
  const int bi = (int)(m / n), t = (int)(m % n);
  const __half* src = staging + m * 2 * d + w * d + g * 64;
  float x[64];
  float amax = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint4 r = *reinterpret_cast<const uint4*>(src + 8 * i);
    const __half2* h = reinterpret_cast<const __half2*>(&r);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 f = __half22float2(h[j]);
      x[8 * i + 2 * j] = f.x;
      x[8 * i + 2 * j + 1] = f.y;
    }
  }
#pragma unroll
  for (int i = 0; i < 64; ++i) amax = fmaxf(amax, fabsf(x[i]));
  const __half s16 = __float2half_rn(__fdiv_rn(amax, 7.0f));
  const float sc = __half2float(s16);
  int q[64];
#pragma unroll
  for (int i = 0; i < 64; ++i) q[i] = sc != 0.f ? (int)fminf(fmaxf(rintf(__fdiv_rn(x[i], sc)), -8.f), 7.f) : 0;
  const int64_t row = (int64_t)(past + t) * kv_b + bi;
  uint8_t* codes = (w == 0 ? kq : vq) + row * (d / 2) + g * 32;
  __half* scales = (w == 0 ? ks : vs) + row * ng + g;
  uint32_t words[8];
#pragma unroll
  for (int wi = 0; wi < 8; ++wi) words[wi] = pack_tiled_word(q + 8 * wi);
  uint4* cd = reinterpret_cast<uint4*>(codes);
  cd[0] = make_uint4(words[0], words[1], words[2], words[3]);
  cd[1] = make_uint4(words[4], words[5], words[6], words[7]);
  *scales = s16;
}

int launch_kv_quant(const __half* staging, int b, int n, int past, int d, int kv_b, uint8_t* kq, __half* ks,
                    uint8_t* vq, __half* vs, cudaStream_t st) {
  if (d % 64) return -1;
  const int64_t total = (int64_t)b * n * 2 * (d / 64);
  kv_quant_kernel<<<(unsigned)((total + 127) / 128), 128, 0, st>>>(staging, b, n, past, d, kv_b, kq, ks, vq, vs);
  return 1;
}

// Decode attention over the int4 cache, "directly on 4-bit": a lane
// owns 16 features (two 8-code words) of one row; q.k = s * sum(q_i * c_i) with the
// exact integer codes, and p*s scales the V codes once per row.  LPR = HD/16 lanes per
// row, lane groups run independent online softmaxes (as in attn_decode_v2_kernel).
template <int HD>
__global__ void __launch_bounds__(128) attn_decode_q4_kernel(AttnArgs a, int n_splits, int pos_per_split) {
  constexpr int LPR = HD / 16, RPW = 32 / LPR, NV = 4 * RPW;
  __shared__ float sm_m[NV], sm_l[NV];
  __shared__ float sm_acc[NV][HD];
  const int head = blockIdx.x, bi = blockIdx.y, split = blockIdx.z;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int sub = lane / LPR, sl = lane % LPR;
  const int vw = warp * RPW + sub;
  const int L = a.past + 1;
  const int lo = split * pos_per_split, hi = min(L, lo + pos_per_split);
  float q[16];
  {
    const __half* qp = a.q + (int64_t)bi * a.d + head * HD + sl * 16;
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2) {
      const uint4 qr = *reinterpret_cast<const uint4*>(qp + 8 * h2);
      const __half2* qh = reinterpret_cast<const __half2*>(&qr);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 f = __half22float2(qh[e]);
        q[8 * h2 + 2 * e] = f.x * kLog2e;
        q[8 * h2 + 2 * e + 1] = f.y * kLog2e;
      }
    }
  }
  const int ng = a.d / 64;
  const int64_t prow = (int64_t)a.kv_b;                      // rows per position
  const int64_t row0 = bi;
  const int cofs = head * (HD / 2) + sl * 8;                 // byte offset of this lane's 16 codes
  const int gofs = head * (HD / 64) + (sl * 16) / 64;        // its group index
  const __half2 one = __half2half2(__float2half_rn(1.f));
  float m_run = -INFINITY, l_run = 0.f, acc[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) acc[e] = 0.f;
  constexpr int U = 4;
  for (int pw = lo + warp * RPW * U; pw < hi; pw += NV * U) {
    const int p0 = pw + sub * U;
    uint2 kc[U], vc[U];
    float ksc[U], vsc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t row = (int64_t)min(p0 + u, hi - 1) * prow + row0;
      kc[u] = *reinterpret_cast<const uint2*>(a.kq + row * (a.d / 2) + cofs);
      vc[u] = *reinterpret_cast<const uint2*>(a.vq + row * (a.d / 2) + cofs);
      ksc[u] = __half2float(a.ks[row * ng + gofs]);
      vsc[u] = __half2float(a.vs[row * ng + gofs]);
    }
    float s[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      __half2 c[8];
      dequant8(kc[u].x, one, c);
      dequant8(kc[u].y, one, c + 4);
      float t = 0.f;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float2 f = __half22float2(c[e]);
        t = fmaf(q[2 * e], f.x, t);
        t = fmaf(q[2 * e + 1], f.y, t);
      }
      s[u] = t * ksc[u];
    }
#pragma unroll
    for (int o = LPR / 2; o > 0; o >>= 1)
#pragma unroll
      for (int u = 0; u < U; ++u) s[u] += __shfl_xor_sync(0xffffffffu, s[u], o);
    float mx = m_run;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (p0 + u >= hi) s[u] = -INFINITY;
      mx = fmaxf(mx, s[u]);
    }
    const float corr = mx == -INFINITY ? 1.f : exp2f(m_run - mx);
    l_run *= corr;
#pragma unroll
    for (int e = 0; e < 16; ++e) acc[e] *= corr;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const float pu = s[u] == -INFINITY ? 0.f : exp2f(s[u] - mx);
      l_run += pu;
      const float ps = pu * vsc[u];
      __half2 c[8];
      dequant8(vc[u].x, one, c);
      dequant8(vc[u].y, one, c + 4);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float2 f = __half22float2(c[e]);
        acc[2 * e] = fmaf(ps, f.x, acc[2 * e]);
        acc[2 * e + 1] = fmaf(ps, f.y, acc[2 * e + 1]);
      }
    }
    m_run = mx;
  }
  if (sl == 0) { sm_m[vw] = m_run; sm_l[vw] = l_run; }
#pragma unroll
  for (int e = 0; e < 16; ++e) sm_acc[vw][sl * 16 + e] = acc[e];
  __syncthreads();
  if (threadIdx.x < HD) {
    const int t = threadIdx.x;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < NV; ++w) M = fmaxf(M, sm_m[w]);
    float l = 0.f, o = 0.f;
#pragma unroll
    for (int w = 0; w < NV; ++w) {
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

int launch_attention_decode_q4(const AttnArgs& a, cudaStream_t st) {
  const int hd = a.d / a.n_heads;
  if (hd != 64 && hd != 128) return -1;
  const int L = a.past + 1;
  const int pairs = a.b * a.n_heads;
  const int target = a.num_sms * 72;
  int n_splits = pairs >= target ? 1 : (target + pairs - 1) / pairs;
  n_splits = max(1, min(n_splits, (L + 63) / 64));
  const int per = (L + n_splits - 1) / n_splits;
  n_splits = (L + per - 1) / per;
  if (n_splits > 1 && (int64_t)pairs * n_splits * (hd + 2) > a.ws_floats) return -1;
  dim3 grid(a.n_heads, a.b, n_splits);
  if (hd == 64) attn_decode_q4_kernel<64><<<grid, 128, 0, st>>>(a, n_splits, per);
  else attn_decode_q4_kernel<128><<<grid, 128, 0, st>>>(a, n_splits, per);
  if (n_splits == 1) return 1;
  dim3 g2(a.n_heads, a.b);
  if (hd == 64) attn_merge_kernel<64><<<g2, 64, 0, st>>>(a, n_splits);
  else attn_merge_kernel<128><<<g2, 128, 0, st>>>(a, n_splits);
  return 2;
}

// The tensor-core GQA kernel (default for group sizes 2/4/8): 32-position K/V tiles in a
// 3-stage cp.async ring, 4 CTAs/SM.  Measured alternatives (64-position tiles with 2 or 3
// stages, forced position splits: profiles/r01/gqa_tc) were slower and are not built.
// The transposed tensor-core GQA kernel (default for group sizes 2/4/8).  4 warps x 16
// positions per 64-position tile when the grid fits one wave at its occupancy (3 stages:
// 104 KB at hd 128, 55 KB at hd 64), else 2 warps x 16 (52 / 28 KB, 4+ CTAs per SM): on
// B200 (profiles/r02/attn_gqa_st/) 4 warps win at c8 / c7 / long contexts, 2 warps at c6
// (512 CTAs would need 1.7 waves at 2 CTAs per SM).  Measured and not built: L2 prefetch
// of the tiles past the ring (+14-70 %), 4 stages of 32 positions (+20 %).
template <int HD, int NW>
static void launch_gqa_st(const AttnArgs& a, dim3 grid, int n_splits, int per, cudaStream_t st) {
  constexpr int smem = 2 * 3 * 16 * NW * (HD + 8) * 2 + 2 * NW * 8 * 4;
  ensure_max_smem(attn_decode_gqa_st_kernel<HD, NW, 3>, smem);
  launch_pdl_k(attn_decode_gqa_st_kernel<HD, NW, 3>, grid, dim3(NW * 32), smem, st, a, n_splits, per);
}

static int launch_attention_decode_gqa_mma(const AttnArgs& a, int G, int var, cudaStream_t st) {
  const int hd = a.d / a.n_heads;
  const int L = a.past + 1;
  const int pairs = a.b * (a.n_heads / G);
  // split positions only when the (b, KV head) pairs cannot cover the SMs: the merge
  // launch costs more than the tail wave (c6: 512 pairs, 1.33 vs 1.62 ms/step)
  int n_splits0 = pairs >= a.num_sms ? 1 : (a.num_sms + pairs - 1) / pairs;
  n_splits0 = max(1, min(n_splits0, (L + 63) / 64));
  auto splits_for = [&](int tile, int* per) {
    *per = ((L + n_splits0 - 1) / n_splits0 + tile - 1) / tile * tile;   // whole tiles per split
    return (L + *per - 1) / *per;
  };
  int per4 = 0, per2 = 0;
  const int ns4 = splits_for(64, &per4), ns2 = splits_for(32, &per2);
  const int smem4 = 2 * 3 * 64 * (hd + 8) * 2 + 2 * 4 * 8 * 4;
  const int64_t fit4 = (int64_t)a.num_sms * ((228 << 10) / (smem4 + 1024));
  // variant 5 forces 4 warps, 6 forces 2 (test and measurement hooks)
  const bool four = var == 5 || (var != 6 && (int64_t)pairs * ns4 <= fit4);
  const int n_splits = four ? ns4 : ns2, per = four ? per4 : per2;
  if (n_splits > 1 && (int64_t)a.b * a.n_heads * n_splits * (hd + 2) > a.ws_floats) return -1;
  dim3 grid(a.n_heads / G, a.b, n_splits);
  if (hd == 64) { if (four) launch_gqa_st<64, 4>(a, grid, n_splits, per, st); else launch_gqa_st<64, 2>(a, grid, n_splits, per, st); }
  else { if (four) launch_gqa_st<128, 4>(a, grid, n_splits, per, st); else launch_gqa_st<128, 2>(a, grid, n_splits, per, st); }
  if (n_splits == 1) return 1;
  dim3 g2(a.n_heads, a.b);
  if (hd == 64) launch_pdl_k(attn_merge_kernel<64>, g2, dim3(64), 0, st, a, n_splits);
  else launch_pdl_k(attn_merge_kernel<128>, g2, dim3(128), 0, st, a, n_splits);
  return 2;
}

int launch_attention_decode(const AttnArgs& a, cudaStream_t st) {
  const int hd = a.d / a.n_heads;
  if (hd != 64 && hd != 128) return -1;
  const int L = a.past + 1;
  // GQA: one CTA per KV head serves its whole query-head group (group sizes 2, 4, 8).
  // The lane-group kernel (v2, variant 1 / PIPO_ATTN_V2=1) is 16 % faster on c6's GQA
  // attention (fewer shuffles per head) but the c6 step measured the same (the following
  // linears timed slower; profiles/r01/gqa_v2), so the one-row-per-warp kernel stays default
  const int G = (a.group == 2 || a.group == 4 || a.group == 8) ? a.group : 1;
  // variant: 0 one-row-per-warp (MHA default), 1 lane groups (CUDA cores; AttnArgs
  // use_cuda_cores = 1 through the pipo_attention_decode hook), 2 tensor cores (GQA default:
  // c6 attention 1.98 -> 1.33 ms/step, c7 0.435 -> 0.36; profiles/r01/gqa_tc); 3 forces the
  // one-row-per-warp kernel for a GQA group (test hook); 5 / 6 force the 4- / 2-warp
  // tensor-core GQA kernel (launch_attention_decode_gqa_mma)
  // MHA default by the number of (b, head) pairs: the lane-group kernel for up to 1536
  // pairs (c2 18.1 -> 13.4 us, c3 50.1 -> 46.8), one row per warp above (c5: 155 vs 173 us;
  // profiles/r02/attn_sk/).  A stream-K variant (one resident wave over the flattened
  // (b, head, position) space, split pairs merged by the last CTA) measured slower at c5
  // (159 vs 155 us isolated, 170 vs 167 in the step) and was not kept.
  const int uc = a.use_cuda_cores;
  const int pairs = a.b * a.n_heads / G;
  const int var = uc == 1 ? 1 : uc == 3 ? 0 : G == 1 ? (pairs <= 1536 ? 1 : 0) : (uc == 5 || uc == 6) ? uc : 2;
  if (var >= 2) return launch_attention_decode_gqa_mma(a, G, var, st);
  const bool v2 = var == 1;
  // enough CTAs for ~8 waves of resident blocks (9 per SM): the block scheduler then
  // balances the tail to within ~1/8 of the kernel; splits merge in a second kernel
  // Split positions only when (b, head) pairs cannot fill the GPU: measured on B200
  // (profiles/r01/attn_splits) one split per pair wins from 512 pairs up (c5 166 -> 155 us,
  // c3 56.5 -> 50.6, c2 15.0 -> 12.5: no partial writes, no merge launch); small batches
  // (c7: b = 1, 8 KV-head pairs) still split.
  const int target = a.num_sms * 2;
  int n_splits = pairs >= target ? 1 : (target + pairs - 1) / pairs;
  n_splits = max(1, min(n_splits, (L + 63) / 64));
  const int per = (L + n_splits - 1) / n_splits;
  n_splits = (L + per - 1) / per;
  if (n_splits > 1 && (int64_t)a.b * a.n_heads * n_splits * (hd + 2) > a.ws_floats) return -1;
  dim3 grid(a.n_heads / G, a.b, n_splits);
  // MHA decode attention is launched WITHOUT programmatic dependent launch (launch_k): as
  // the QKV GEMM's early-launched dependent it measured 197 us per c5 layer in the step vs
  // 161 us launched plainly (c5 device tier uninstrumented 3 740 -> 4 070 tok/s;
  // profiles/r02/pdl_attn/).  The one-wave GQA kernel keeps PDL (same time either way).
  if (!v2) {   // one K/V row per warp: measured 0-5% ahead of v2 at c3-c5 (MHA)
#define PIPO_DECODE(HDV, GV) launch_k(attn_decode_kernel<HDV, GV>, grid, dim3(128), 0, st, a, n_splits, per)
    if (hd == 64) {
      if (G == 1) PIPO_DECODE(64, 1); else if (G == 2) PIPO_DECODE(64, 2); else if (G == 4) PIPO_DECODE(64, 4);
      else PIPO_DECODE(64, 8);
    } else {
      if (G == 1) PIPO_DECODE(128, 1); else if (G == 2) PIPO_DECODE(128, 2); else if (G == 4) PIPO_DECODE(128, 4);
      else PIPO_DECODE(128, 8);
    }
#undef PIPO_DECODE
  } else {     // v2: lane groups with 16-B row loads
#define PIPO_DECODE2(HDV, GV) launch_k(attn_decode_v2_kernel<HDV, GV>, grid, dim3(128), 0, st, a, n_splits, per)
    if (hd == 64) {
      if (G == 1) PIPO_DECODE2(64, 1); else if (G == 2) PIPO_DECODE2(64, 2); else if (G == 4) PIPO_DECODE2(64, 4);
      else PIPO_DECODE2(64, 8);
    } else {
      if (G == 1) PIPO_DECODE2(128, 1); else if (G == 2) PIPO_DECODE2(128, 2); else if (G == 4) PIPO_DECODE2(128, 4);
      else PIPO_DECODE2(128, 8);
    }
#undef PIPO_DECODE2
  }
  if (n_splits == 1) return 1;
  dim3 g2(a.n_heads, a.b);
  if (hd == 64) launch_pdl_k(attn_merge_kernel<64>, g2, dim3(64), 0, st, a, n_splits);
  else launch_pdl_k(attn_merge_kernel<128>, g2, dim3(128), 0, st, a, n_splits);
  return 2;
}

int launch_attention_prefill(const AttnArgs& a, cudaStream_t st) {
  const int hd = a.d / a.n_heads;
  if (hd != 64 && hd != 128) return -1;
  // use_cuda_cores: 0 tcgen05 kernel where it applies (k_attn_tc.cu: causal key range
  // <= 512), else mma.sync; 2 forces the mma.sync kernel; 1 the CUDA-core kernel
  if (a.use_cuda_cores == 0) {
    const int r = launch_attention_prefill_tc(a, st);
    if (r >= 0) return r;
  }
  if (a.use_cuda_cores == 1) {   // the v1 CUDA-core kernel, kept as a cross-check
    dim3 grid(a.n_heads, a.b, (a.n + 31) / 32);
    if (hd == 64) attn_prefill_kernel<64><<<grid, 256, 0, st>>>(a);
    else attn_prefill_kernel<128><<<grid, 256, 0, st>>>(a);
    return 1;
  }
  dim3 grid(a.n_heads, a.b, (a.n + 63) / 64);
  if (hd == 64) {
    const int smem = 5 * 64 * (64 + 8) * 2;
    ensure_max_smem(attn_prefill_mma_kernel<64>, smem);
    attn_prefill_mma_kernel<64><<<grid, 128, smem, st>>>(a);
  } else {
    const int smem = 5 * 64 * (128 + 8) * 2;
    ensure_max_smem(attn_prefill_mma_kernel<128>, smem);
    attn_prefill_mma_kernel<128><<<grid, 128, smem, st>>>(a);
  }
  return 1;
}

}  // namespace pipo
