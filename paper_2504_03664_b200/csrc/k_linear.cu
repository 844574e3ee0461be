// k_linear.cu — fused int4-g64 / fp16 linear layers (decoder QKV, out-proj, FC1, FC2,
// LM head).  y = x . W^T + b with the epilogue fused (kernels.h EpiKind).
//
//  * gemv_int4_kernel — PAPER.md:305-309 (§3.4): "matrix-vector multiplication
//    directly on 4-bit quantized weights, avoiding the dequantization operation",
//    used for small batches ("batch sizes less than 16").  CUDA cores:
//    each thread owns one weight row and 32 codes of every k-block; it multiplies the
//    raw int4 codes with x and applies the group scale once per 32 products:
//    acc += s_g * sum_k q_k x_k.  128-bit coalesced code loads (a warp reads 512
//    contiguous bytes), x staged in shared memory (broadcast reads).
//  * gemm_kernel — the b >= 16 path ("dequantized into floating-point
//    values before computation", here fused: codes are unpacked + scaled into an
//    fp16 shared-memory tile, never materialized in HBM) on tensor cores.
//    Swap-AB: the 128-row weight tile is the MMA "A", activations are "B".
//    Weight blocks and x tiles stream through a 4-stage cp.async ring.
//  Split-K with a deterministic fixup: partials go to a workspace, the last CTA of
//  a tile (arrival counter) sums them in split order and runs the epilogue, so
//  results are bit-reproducible run to run (tier invariance tests rely on it).
#include "common.cuh"
#include "launch.cuh"
#include "kernels.h"
#include "layout.h"
#include "epilogue.cuh"

namespace pipo {

// ---------------------------------------------------------------------------
// split-K fixup: returns true in the CTA that must run the epilogue; `acc` then
// holds the sum over splits in fixed order 0..n_splits-1.
template <int NACC>
__device__ __forceinline__ bool splitk_fixup(float* acc, float* ws, int* counters, int tile,
                                             int n_tiles, int split, int n_splits) {
  if (n_splits == 1) return true;
  __shared__ int s_last;
  const int tid = threadIdx.x, nthr = blockDim.x;
  float* mine = ws + ((int64_t)split * n_tiles + tile) * nthr * NACC + (int64_t)tid * NACC;
#pragma unroll
  for (int i = 0; i < NACC; i += 4)
    __stcg(reinterpret_cast<float4*>(mine + i), make_float4(acc[i], acc[i + 1], acc[i + 2], acc[i + 3]));
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = (atomicAdd(&counters[tile], 1) == n_splits - 1);
  __syncthreads();
  if (!s_last) return false;
  __threadfence();
#pragma unroll
  for (int i = 0; i < NACC; ++i) acc[i] = 0.f;
  for (int s = 0; s < n_splits; ++s) {
    const float* p = ws + ((int64_t)s * n_tiles + tile) * nthr * NACC + (int64_t)tid * NACC;
#pragma unroll
    for (int i = 0; i < NACC; i += 4) {
      float4 v = __ldcg(reinterpret_cast<const float4*>(p + i));
      acc[i] += v.x; acc[i + 1] += v.y; acc[i + 2] += v.z; acc[i + 3] += v.w;
    }
  }
  if (tid == 0) counters[tile] = 0;
  return true;
}

// ---------------------------------------------------------------------------
// GEMV: M <= MM rows, int4 weights only.
constexpr int GEMV_THREADS = 256;
constexpr int GEMV_XS_FLOATS = 8192;

template <int MM>
__global__ void __launch_bounds__(GEMV_THREADS) gemv_int4_kernel(LinearArgs a, int kb_per_split,
                                                                  int n_splits) {
  constexpr int CHUNK_KB = GEMV_XS_FLOATS / (MM * 64);
  __shared__ float xs[MM][CHUNK_KB * 64];
  __shared__ float red[MM][128];
  const int tid = threadIdx.x, h = tid >> 7, r = tid & 127;
  const int rt = blockIdx.x, split = blockIdx.y;
  const int n_kb = a.K / 64;
  const int kb0 = split * kb_per_split, kb1 = min(n_kb, kb0 + kb_per_split);
  const uint8_t* wbase = a.w + (int64_t)rt * n_kb * kInt4BlockBytes;
  float acc[MM];
#pragma unroll
  for (int m = 0; m < MM; ++m) acc[m] = 0.f;

  for (int c0 = kb0; c0 < kb1; c0 += CHUNK_KB) {
    const int nb = min(CHUNK_KB, kb1 - c0);
    __syncthreads();
    for (int i = tid; i < MM * nb * 32; i += GEMV_THREADS) {
      const int m = i / (nb * 32), k2 = i - m * (nb * 32);
      float2 v = make_float2(0.f, 0.f);
      if (m < a.M)
        v = __half22float2(reinterpret_cast<const __half2*>(a.x + (int64_t)m * a.K + (int64_t)c0 * 64)[k2]);
      xs[m][2 * k2] = v.x;
      xs[m][2 * k2 + 1] = v.y;
    }
    __syncthreads();
#pragma unroll 4
    for (int kb = 0; kb < nb; ++kb) {
      const uint8_t* blk = wbase + (int64_t)(c0 + kb) * kInt4BlockBytes;
      const uint4 cw = ld_nc_v4(blk + (h * 128 + r) * 16);
      const float s = __half2float(*reinterpret_cast<const __half*>(blk + 4096 + r * 2));
      const uint32_t words[4] = {cw.x, cw.y, cw.z, cw.w};
      float part[MM];
#pragma unroll
      for (int m = 0; m < MM; ++m) part[m] = 0.f;
#pragma unroll
      for (int wi = 0; wi < 4; ++wi) {
#pragma unroll
        for (int ci = 0; ci < 8; ++ci) {
          const float q = static_cast<float>(code_at(words[wi], ci));
          const int k = kb * 64 + h * 32 + wi * 8 + ci;
#pragma unroll
          for (int m = 0; m < MM; ++m) part[m] = fmaf(q, xs[m][k], part[m]);
        }
      }
#pragma unroll
      for (int m = 0; m < MM; ++m) acc[m] = fmaf(s, part[m], acc[m]);
    }
  }
  __syncthreads();
  if (h == 1) {
#pragma unroll
    for (int m = 0; m < MM; ++m) red[m][r] = acc[m];
  }
  __syncthreads();
  if (h == 0) {
#pragma unroll
    for (int m = 0; m < MM; ++m) acc[m] += red[m][r];
  } else {
#pragma unroll
    for (int m = 0; m < MM; ++m) acc[m] = 0.f;
  }
  constexpr int NACC = (MM + 3) / 4 * 4;
  float accp[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) accp[i] = i < MM ? acc[i] : 0.f;
  if (!splitk_fixup<NACC>(accp, a.ws, a.counters, rt, gridDim.x, split, n_splits)) return;
  if (h == 0) {
#pragma unroll
    for (int m = 0; m < MM; ++m) epi_store(a.epi, m, rt * 128 + r, accp[m]);
  }
}

// ---------------------------------------------------------------------------
// Tensor-core GEMM (mma.sync m16n8k16, fp16 x fp16 -> fp32).
constexpr int GEMM_THREADS = 256;
constexpr int GEMM_STAGES = 4;
constexpr int APAD = 72;  // halves per smem row: 64 + 8 pad (conflict-free ldmatrix)

template <int WT, int BN>
struct GemmCfg {
  static constexpr int RAW = WT ? (int)kInt4BlockBytes : (int)kFp16BlockBytes;
  // fp16 weights land straight in the padded ldmatrix layout (no staging copy, no A buffer)
  static constexpr int RAW_STAGE = WT ? (RAW + 127) / 128 * 128 : 128 * APAD * 2;
  static constexpr int X_STAGE = BN * APAD * 2;
  static constexpr int A_BYTES = WT ? 128 * APAD * 2 : 0;
  static constexpr int SMEM = GEMM_STAGES * (RAW_STAGE + X_STAGE) + A_BYTES;
  static constexpr int NT = BN / 16;           // n8 tiles per warp
  static constexpr int NACC = 2 * NT * 4;
};

template <int WT, int BN>
__global__ void __launch_bounds__(GEMM_THREADS) gemm_kernel(LinearArgs a, int kb_per_split, int n_splits) {
  using C = GemmCfg<WT, BN>;
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* raw = smem;
  __half* xs = reinterpret_cast<__half*>(smem + GEMM_STAGES * C::RAW_STAGE);
  __half* as = reinterpret_cast<__half*>(smem + GEMM_STAGES * (C::RAW_STAGE + C::X_STAGE));
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rt = blockIdx.x, mt = blockIdx.y, split = blockIdx.z;
  const int n_kb = a.K / 64;
  const int kb0 = split * kb_per_split, kb1 = min(n_kb, kb0 + kb_per_split);
  const int nk = max(0, kb1 - kb0);
  const int m0 = mt * BN;
  const uint8_t* wbase = a.w + (int64_t)rt * n_kb * C::RAW;

  auto load_stage = [&](int i) {
    const int s = i % GEMM_STAGES, kb = kb0 + i;
    const uint8_t* src = wbase + (int64_t)kb * C::RAW;
    uint8_t* dst = raw + s * C::RAW_STAGE;
    if constexpr (WT == 1) {
      for (int c = tid; c < C::RAW / 16; c += GEMM_THREADS) cp_async16(dst + c * 16, src + c * 16);
    } else {   // 128 rows x 8 chunks of 16 B -> padded rows of APAD halves
      for (int c = tid; c < C::RAW / 16; c += GEMM_THREADS)
        cp_async16(dst + ((c >> 3) * APAD + (c & 7) * 8) * 2, src + c * 16);
    }
    __half* xd = xs + s * BN * APAD;
    for (int c = tid; c < BN * 8; c += GEMM_THREADS) {
      const int r = c >> 3, col = c & 7, m = m0 + r;
      const __half* xsrc = a.x + (int64_t)min(m, a.M - 1) * a.K + (int64_t)kb * 64 + col * 8;
      cp_async16(xd + r * APAD + col * 8, xsrc, m < a.M ? 16 : 0);
    }
  };

#pragma unroll
  for (int i = 0; i < GEMM_STAGES - 1; ++i) {
    if (i < nk) load_stage(i);
    cp_async_commit();
  }

  float acc[2][C::NT][4];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < C::NT; ++j)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[i][j][c] = 0.f;

  const int wr = warp & 3, wc = warp >> 2;
  for (int i = 0; i < nk; ++i) {
    cp_async_wait<GEMM_STAGES - 2>();
    __syncthreads();
    if (i + GEMM_STAGES - 1 < nk) load_stage(i + GEMM_STAGES - 1);
    cp_async_commit();
    const int s = i % GEMM_STAGES;
    const uint8_t* rs = raw + s * C::RAW_STAGE;
    const __half* aS = WT ? as : reinterpret_cast<const __half*>(rs);
    if constexpr (WT == 1) {
      const int h = tid >> 7, r = tid & 127;
      const uint4 cw = *reinterpret_cast<const uint4*>(rs + (h * 128 + r) * 16);
      const __half sc = *reinterpret_cast<const __half*>(rs + 4096 + r * 2);
      const __half2 s2 = __half2half2(sc);
      __half2 o[16];
      dequant8(cw.x, s2, o + 0);
      dequant8(cw.y, s2, o + 4);
      dequant8(cw.z, s2, o + 8);
      dequant8(cw.w, s2, o + 12);
      uint4* dst = reinterpret_cast<uint4*>(as + r * APAD + h * 32);
      const uint4* src = reinterpret_cast<const uint4*>(o);
#pragma unroll
      for (int q = 0; q < 4; ++q) dst[q] = src[q];
      __syncthreads();
    }
    const __half* xsS = xs + s * BN * APAD;
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      uint32_t af[2][4];
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
        ldmatrix_x4(af[mi][0], af[mi][1], af[mi][2], af[mi][3],
                    aS + (wr * 32 + mi * 16 + (lane & 15)) * APAD + kk * 16 + (lane >> 4) * 8);
      if constexpr (C::NT == 1) {
        uint32_t b0, b1;
        ldmatrix_x2(b0, b1, xsS + (wc * (BN / 2) + (lane & 7)) * APAD + kk * 16 + ((lane >> 3) & 1) * 8);
#pragma unroll
        for (int mi = 0; mi < 2; ++mi) mma_16816(acc[mi][0], af[mi], b0, b1);
      } else {
#pragma unroll
        for (int jj = 0; jj < C::NT / 2; ++jj) {
          uint32_t b0, b1, b2, b3;
          ldmatrix_x4(b0, b1, b2, b3,
                      xsS + (wc * (BN / 2) + jj * 16 + (lane & 7) + ((lane >> 4) << 3)) * APAD + kk * 16 +
                          ((lane >> 3) & 1) * 8);
#pragma unroll
          for (int mi = 0; mi < 2; ++mi) {
            mma_16816(acc[mi][2 * jj], af[mi], b0, b1);
            mma_16816(acc[mi][2 * jj + 1], af[mi], b2, b3);
          }
        }
      }
    }
  }
  cp_async_wait<0>();

  float* flat = &acc[0][0][0];
  if (!splitk_fixup<C::NACC>(flat, a.ws, a.counters, mt * gridDim.x + rt, gridDim.x * gridDim.y, split,
                             n_splits))
    return;
  const int g = lane >> 2, tq = lane & 3;
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int j = 0; j < C::NT; ++j) {
      const int nrow = rt * 128 + wr * 32 + mi * 16 + g;
      const int mcol = m0 + wc * (BN / 2) + j * 8 + 2 * tq;
      epi_store(a.epi, mcol, nrow, acc[mi][j][0]);
      epi_store(a.epi, mcol + 1, nrow, acc[mi][j][1]);
      epi_store(a.epi, mcol, nrow + 8, acc[mi][j][2]);
      epi_store(a.epi, mcol + 1, nrow + 8, acc[mi][j][3]);
    }
}

// ---------------------------------------------------------------------------
template <int WT, int BN>
static int run_gemm(const LinearArgs& a, cudaStream_t st) {
  using C = GemmCfg<WT, BN>;
  ensure_max_smem(gemm_kernel<WT, BN>, C::SMEM);
  const int n_rt = (a.N + 127) / 128, m_tiles = (a.M + BN - 1) / BN, n_kb = a.K / 64;
  const int tiles = n_rt * m_tiles;
  const int per_sm = C::SMEM <= 75 * 1024 ? 3 : (C::SMEM <= 113 * 1024 ? 2 : 1);
  const int target = a.num_sms * per_sm;
  int splits = tiles >= target ? 1 : (target + tiles - 1) / tiles;
  splits = max(1, min(splits, n_kb / 4));
  int kb_per = (n_kb + splits - 1) / splits;
  splits = (n_kb + kb_per - 1) / kb_per;
  if (splits > 1) {
    const int64_t need = (int64_t)splits * tiles * GEMM_THREADS * C::NACC;
    if (need > a.ws_floats || tiles > a.n_counters) {
      splits = 1;
      kb_per = n_kb;
    }
  }
  dim3 grid(n_rt, m_tiles, splits);
  gemm_kernel<WT, BN><<<grid, GEMM_THREADS, C::SMEM, st>>>(a, kb_per, splits);
  return 1;
}

template <int MM>
static int run_gemv(const LinearArgs& a, cudaStream_t st) {
  const int n_rt = (a.N + 127) / 128, n_kb = a.K / 64;
  const int target = a.num_sms * 4;
  int splits = n_rt >= target ? 1 : (target + n_rt - 1) / n_rt;
  splits = max(1, min(splits, n_kb / 2));
  int kb_per = (n_kb + splits - 1) / splits;
  splits = (n_kb + kb_per - 1) / kb_per;
  constexpr int NACC = (MM + 3) / 4 * 4;
  if (splits > 1) {
    const int64_t need = (int64_t)splits * n_rt * GEMV_THREADS * NACC;
    if (need > a.ws_floats || n_rt > a.n_counters) {
      splits = 1;
      kb_per = n_kb;
    }
  }
  dim3 grid(n_rt, splits);
  gemv_int4_kernel<MM><<<grid, GEMV_THREADS, 0, st>>>(a, kb_per, splits);
  return 1;
}

int launch_linear(const LinearArgs& a, int path, int gemv_max_m, cudaStream_t st) {
  if (a.M <= 0 || a.N <= 0 || a.K <= 0 || a.K % 64 != 0) return -1;
  bool gemv = false;
  if (path == PATH_GEMV) gemv = true;
  // M <= gemv_max_m: the CUDA-core GEMV ("batch sizes less than 16") — but
  // only for small matrices: from 8 M weights up the tcgen05 stream-K kernel (BN = 16, rows
  // >= M zero-filled by TMA) streams 1.5-2.6x faster even at M = 1 (c7: FC1 72 -> 27 us,
  // profiles/r01/gemv_crossover; reading Q4 "re-tune the crossover by measurement")
  else if (path == PATH_AUTO) gemv = (a.wfmt == 1 && a.M <= gemv_max_m && (int64_t)a.N * a.K < (8ll << 20));
  if (path == PATH_HEAD) return launch_linear_stream_f16(a, true, st);
  if (path == PATH_STREAM || (path == PATH_AUTO && a.wfmt == 0 && a.M <= 64)) return launch_linear_stream_f16(a, false, st);
  if (path == PATH_TP || (path == PATH_AUTO && !gemv && a.wfmt == 1 && a.M > 128)) return launch_linear_tp(a, st);
  // PATH_PAIR (k_gemm_pair.cu, cta_group::2 + in-kernel fixup) is correct but measured
  // slower than the TM kernel on every decode shape: selectable, not chosen.
  if (path == PATH_PAIR) return launch_linear_pair(a, st);
  if (path == PATH_TM || (path == PATH_AUTO && !gemv && a.wfmt == 1 && a.M <= 64)) return launch_linear_tm(a, st);
  if (path == PATH_WS || (path == PATH_AUTO && !gemv && a.wfmt == 1 && a.M <= 128)) return launch_linear_ws(a, st);
  if (path == PATH_TC || (path == PATH_AUTO && !gemv)) return launch_linear_tc(a, st);
  if (gemv) {
    if (a.wfmt != 1 || a.M > 16) return -1;
    if (a.M == 1) return run_gemv<1>(a, st);
    if (a.M <= 4) return run_gemv<4>(a, st);
    if (a.M <= 8) return run_gemv<8>(a, st);
    return run_gemv<16>(a, st);
  }
  if (a.wfmt == 1) {
    if (a.M <= 16) return run_gemm<1, 16>(a, st);
    if (a.M <= 32) return run_gemm<1, 32>(a, st);
    if (a.M <= 64) return run_gemm<1, 64>(a, st);
    return run_gemm<1, 128>(a, st);
  }
  if (a.M <= 16) return run_gemm<0, 16>(a, st);
  if (a.M <= 32) return run_gemm<0, 32>(a, st);
  if (a.M <= 64) return run_gemm<0, 64>(a, st);
  return run_gemm<0, 128>(a, st);
}

}  // namespace pipo
