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

}  // namespace pipo
