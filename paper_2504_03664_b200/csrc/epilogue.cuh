// epilogue.cuh — the fused linear-layer epilogue shared by the GEMV, the mma.sync
// GEMM and the tcgen05 GEMM (kernels.h EpiKind).
#pragma once
#include "common.cuh"
#include "kernels.h"

namespace pipo {

__device__ __forceinline__ void epi_store(const EpiParams& e, int m, int n, float acc) {
  if (m >= e.M || n >= e.N) return;
  const float v = acc + (e.bias ? __half2float(e.bias[n]) : 0.f);
  switch (e.kind) {
    case EPI_QKV: {
      const int bi = m / e.n_tok, t = m - bi * e.n_tok;
      const int dkv = e.dkv ? e.dkv : e.d;
      if (n < e.d) {
        e.q[(int64_t)m * e.d + n] = __float2half_rn(v * e.qscale);
      } else {
        const int64_t off = e.kv_rowmajor ? (int64_t)m * 2 * dkv : ((int64_t)(e.past + t) * e.kv_b + bi) * dkv;
        if (n < e.d + dkv) e.kc[off + n - e.d] = __float2half_rn(v);
        else e.vc[off + n - e.d - dkv] = __float2half_rn(v);
      }
      break;
    }
    case EPI_RESID: e.h[(int64_t)m * e.N + n] += v; break;
    case EPI_RELU: e.u[(int64_t)m * e.N + n] = __float2half_rn(fmaxf(v, 0.f)); break;
    case EPI_HALF: e.u[(int64_t)m * e.N + n] = __float2half_rn(v); break;
    default: e.y[(int64_t)m * e.ldy + n] = v; break;
  }
}

// The epilogue for 4 consecutive output features n..n+3 of one row m (the stream-K reduce
// kernel's float4 partial sums): the residual add loads the four old values together
// (epi_store's load/store pairs may alias, so the compiler would serialise them).
__device__ __forceinline__ void epi_store4(const EpiParams& e, int m, int n, float4 acc) {
  if (e.kind == EPI_RESID && m < e.M && n + 3 < e.N) {
    float* hp = e.h + (int64_t)m * e.N + n;
    float b[4] = {0.f, 0.f, 0.f, 0.f};
    if (e.bias)
#pragma unroll
      for (int i = 0; i < 4; ++i) b[i] = __half2float(e.bias[n + i]);
    const float o0 = hp[0], o1 = hp[1], o2 = hp[2], o3 = hp[3];
    hp[0] = o0 + (acc.x + b[0]);
    hp[1] = o1 + (acc.y + b[1]);
    hp[2] = o2 + (acc.z + b[2]);
    hp[3] = o3 + (acc.w + b[3]);
    return;
  }
  epi_store(e, m, n, acc.x);
  epi_store(e, m, n + 1, acc.y);
  epi_store(e, m, n + 2, acc.z);
  epi_store(e, m, n + 3, acc.w);
}

// The same epilogue for 16 consecutive rows m0..m0+15 of one output column n (one
// accumulator chunk read from TMEM): the bias is loaded once and, for the residual add,
// all 16 old values are loaded before any store — epi_store's per-element load/store
// pairs may alias, so the compiler serialises them (one memory round trip per element).
__device__ __forceinline__ void epi_store16(const EpiParams& e, int m0, int n, const float* acc) {
  if (n >= e.N) return;
  const float b = e.bias ? __half2float(e.bias[n]) : 0.f;
  float v[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = acc[i] + b;
  switch (e.kind) {
    case EPI_RESID: {
      float old[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) old[i] = m0 + i < e.M ? e.h[(int64_t)(m0 + i) * e.N + n] : 0.f;
#pragma unroll
      for (int i = 0; i < 16; ++i)
        if (m0 + i < e.M) e.h[(int64_t)(m0 + i) * e.N + n] = old[i] + v[i];
      break;
    }
    case EPI_QKV: {
      const float qs = e.qscale;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int m = m0 + i;
        if (m >= e.M) break;
        if (n < e.d) {
          e.q[(int64_t)m * e.d + n] = __float2half_rn(v[i] * qs);
        } else {
          const int bi = m / e.n_tok, t = m - bi * e.n_tok;
          const int dkv = e.dkv ? e.dkv : e.d;
          const int64_t off = e.kv_rowmajor ? (int64_t)m * 2 * dkv : ((int64_t)(e.past + t) * e.kv_b + bi) * dkv;
          if (n < e.d + dkv) e.kc[off + n - e.d] = __float2half_rn(v[i]);
          else e.vc[off + n - e.d - dkv] = __float2half_rn(v[i]);
        }
      }
      break;
    }
    case EPI_RELU:
#pragma unroll
      for (int i = 0; i < 16; ++i)
        if (m0 + i < e.M) e.u[(int64_t)(m0 + i) * e.N + n] = __float2half_rn(fmaxf(v[i], 0.f));
      break;
    case EPI_HALF:
#pragma unroll
      for (int i = 0; i < 16; ++i)
        if (m0 + i < e.M) e.u[(int64_t)(m0 + i) * e.N + n] = __float2half_rn(v[i]);
      break;
    default:
#pragma unroll
      for (int i = 0; i < 16; ++i)
        if (m0 + i < e.M) e.y[(int64_t)(m0 + i) * e.ldy + n] = v[i];
      break;
  }
}

}  // namespace pipo
