// k_head.cu — streaming fp16-weight GEMM on tcgen05 for the decode LM head (a13,
// logits = LN(h) . E_tok^T, "the output embedding layer")
// and the fp16-weight decode linears: y[M x N] = x[M x K] . W[N x K]^T, M <= 64 rows
// (the batch), W streamed once from HBM.  The bound is HBM (c5 LM head: 720 MB per step).
//
// Weights stay in the library's tiled fp16 layout (layout.h: 128-row x 64-k blocks of
// 16 KiB, row-major); a 4-D TMA tensor map over (k in block, row, k-block, row tile) lands
// each block in shared memory already in the SWIZZLE_128B K-major atom layout the MMA
// reads, so no thread touches the weights.  Warp-specialized, persistent (one CTA per SM):
//   warp 0      TMA producer: weight block + x tile per k-block into an NS-stage ring;
//   warp 1      MMA issuer: 4 x tcgen05.mma (M = 128 weight rows, N = BN batch rows,
//               K = 16) per stage, commit releases the stage; two TMEM accumulators;
//   warps 2-5   epilogue: tcgen05.ld of a finished tile, fused epilogue (logits stores:
//               lanes = weight rows, so one batch row's stores are contiguous).
// Tiles are dealt round-robin to the CTAs: the c5 head's 393 tiles over 148 SMs need
// three rounds (88.5 % balance); split-K is not used, so the result is the plain k-order
// sum (deterministic, no partials).
#include <cuda.h>

#include <algorithm>

#include "common.cuh"
#include "epilogue.cuh"
#include "kernels.h"
#include "launch.cuh"
#include "layout.h"
#include "tcgen05.cuh"

namespace pipo {

template <int BN>
struct HeadCfg {
  static constexpr int W_STAGE = 128 * 128;   // one 128 x 64 fp16 block (16 KiB)
  static constexpr int X_STAGE = BN * 128;    // BN x 64 fp16
  static constexpr int STAGE = W_STAGE + X_STAGE;
  static constexpr int NS = (200 * 1024) / STAGE < 12 ? (200 * 1024) / STAGE : 12;
  static constexpr int SMEM = 1024 + NS * STAGE + 512;
  static constexpr int THREADS = 192;
  static constexpr uint32_t TMEM_COLS = 2 * BN < 32 ? 32 : 2 * BN;
  // kind::f16: fp32 accumulate (bit 4), fp16 A / B, both K-major, N >> 3, M >> 4
  static constexpr uint32_t IDESC = (1u << 4) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  static_assert(SMEM <= 227 * 1024, "shared memory budget");
};

template <int BN>
__device__ __forceinline__ void stream_f16_body(const CUtensorMap& wmap, const CUtensorMap& xmap, const LinearArgs& a,
                                                int n_rt) {
  using C = HeadCfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base_u32 = (smem_u32(smem_raw) + 1023u) & ~1023u;
  uint8_t* base = smem_raw + (base_u32 - smem_u32(smem_raw));
  uint64_t* bar = reinterpret_cast<uint64_t*>(base + C::NS * C::STAGE);
  uint64_t* full = bar;
  uint64_t* empty = full + C::NS;
  uint64_t* acc_full = empty + C::NS;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_kb = a.K / 64;
  if (threadIdx.x == 0) {
    for (int i = 0; i < C::NS; ++i) { ptx::mbar_init(&full[i], 1); ptx::mbar_init(&empty[i], 1); }
    for (int i = 0; i < 2; ++i) { ptx::mbar_init(&acc_full[i], 1); ptx::mbar_init(&acc_empty[i], 4); }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&wmap) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&xmap) : "memory");
  }
  if (warp == 1) ptx::tmem_alloc(tmem_slot, C::TMEM_COLS);
  ptx::tc_before();
  __syncthreads();
  ptx::tc_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();   // x (and the output) belong to the predecessor
  if (warp == 0) {
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 1;
      for (int rt = blockIdx.x; rt < n_rt; rt += gridDim.x)
        for (int kb = 0; kb < n_kb; ++kb) {
          ptx::mbar_wait(&empty[s], ph);
          uint8_t* st = base + s * C::STAGE;
          ptx::mbar_expect_tx(&full[s], C::STAGE);
          ptx::tma_4d(st, &wmap, 0, 0, kb, rt, &full[s]);
          ptx::tma_2d(st + C::W_STAGE, &xmap, kb * 64, 0, &full[s]);
          if (++s == C::NS) { s = 0; ph ^= 1; }
        }
    }
  } else if (warp == 1) {
    int s = 0, t = 0;
    uint32_t ph = 0;
    for (int rt = blockIdx.x; rt < n_rt; rt += gridDim.x, ++t) {
      const int ab = t & 1;
      ptx::mbar_wait(&acc_empty[ab], ((t >> 1) & 1) ^ 1);
      ptx::tc_after();
      const uint32_t d = tmem + ab * BN;
      for (int kb = 0; kb < n_kb; ++kb) {
        ptx::mbar_wait(&full[s], ph);
        ptx::tc_after();
        if (ptx::elect_one()) {
          const uint32_t sa = smem_u32(base + s * C::STAGE);
          const uint64_t da = ptx::sw128_desc(sa), db = ptx::sw128_desc(sa + C::W_STAGE);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)   // K = 16 per MMA: +32 B along the swizzled row
            ptx::mma_f16_ss(d, da + (uint64_t)(kk * 2), db + (uint64_t)(kk * 2), C::IDESC, (kb | kk) ? 1u : 0u);
          ptx::mma_commit(&empty[s]);
          if (kb == n_kb - 1) ptx::mma_commit(&acc_full[ab]);
        }
        __syncwarp();
        if (++s == C::NS) { s = 0; ph ^= 1; }
      }
    }
  } else {
    const int quarter = warp & 3;   // tcgen05.ld: a warp reads its own 32-lane quarter
    const int row = quarter * 32 + lane;
    int t = 0;
    for (int rt = blockIdx.x; rt < n_rt; rt += gridDim.x, ++t) {
      const int ab = t & 1;
      ptx::mbar_wait_sleep(&acc_full[ab], (t >> 1) & 1);
      ptx::tc_after();
      const uint32_t taddr = tmem + ab * BN + ((uint32_t)(quarter * 32) << 16);
      const int n = rt * 128 + row;
#pragma unroll
      for (int c0 = 0; c0 < BN; c0 += 16) {
        float v[16];
        ptx::tmem_ld16(taddr + c0, v);
#pragma unroll
        for (int j = 0; j < 16; ++j) epi_store(a.epi, c0 + j, n, v[j]);
      }
      ptx::tc_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&acc_empty[ab]);
    }
  }
  ptx::tc_before();
  __syncthreads();
  if (warp == 1) ptx::tmem_dealloc(tmem, C::TMEM_COLS);
}

// two names for one body, so traces tell the LM head (a13) from the fp16 decode linears
template <int BN>
__global__ void __launch_bounds__(HeadCfg<BN>::THREADS, 1)
    lm_head_stream_kernel(const __grid_constant__ CUtensorMap wmap, const __grid_constant__ CUtensorMap xmap,
                          LinearArgs a, int n_rt) {
  stream_f16_body<BN>(wmap, xmap, a, n_rt);
}
template <int BN>
__global__ void __launch_bounds__(HeadCfg<BN>::THREADS, 1)
    gemm_f16_stream_kernel(const __grid_constant__ CUtensorMap wmap, const __grid_constant__ CUtensorMap xmap,
                           LinearArgs a, int n_rt) {
  stream_f16_body<BN>(wmap, xmap, a, n_rt);
}

typedef CUresult (*PFN_encodeTiledHead)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                        const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                        CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiledHead encoder() {
  static PFN_encodeTiledHead fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess)
      fn = (PFN_encodeTiledHead)p;
    cudaGetLastError();
  }
  return fn;
}

template <int BN>
static int run_head(const LinearArgs& a, bool lm_head, cudaStream_t st) {
  using C = HeadCfg<BN>;
  PFN_encodeTiledHead enc = encoder();
  if (!enc) return -1;
  const int n_rt = (a.N + 127) / 128, n_kb = a.K / 64;
  // the tiled fp16 matrix as a 4-D tensor: (k in block, row in tile, k-block, row tile)
  CUtensorMap wmap, xmap;
  {
    const cuuint64_t dims[4] = {64, 128, (cuuint64_t)n_kb, (cuuint64_t)n_rt};
    const cuuint64_t strides[3] = {128, (cuuint64_t)kFp16BlockBytes, (cuuint64_t)n_kb * kFp16BlockBytes};
    const cuuint32_t box[4] = {64, 128, 1, 1};
    const cuuint32_t es[4] = {1, 1, 1, 1};
    if (enc(&wmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, const_cast<uint8_t*>(a.w), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return -1;
  }
  {
    // rows >= M are out of bounds: TMA zero-fills them (no garbage in the unused columns)
    const cuuint64_t dims[2] = {(cuuint64_t)a.K, (cuuint64_t)a.M};
    const cuuint64_t strides[1] = {(cuuint64_t)a.K * 2};
    const cuuint32_t box[2] = {64, (cuuint32_t)BN};
    const cuuint32_t es[2] = {1, 1};
    if (enc(&xmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<__half*>(a.x), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return -1;
  }
  const int G = std::min(a.num_sms, n_rt);
  if (lm_head) {
    ensure_max_smem(lm_head_stream_kernel<BN>, C::SMEM);
    launch_pdl_k(lm_head_stream_kernel<BN>, dim3(G), dim3(C::THREADS), C::SMEM, st, wmap, xmap, a, n_rt);
  } else {
    ensure_max_smem(gemm_f16_stream_kernel<BN>, C::SMEM);
    launch_pdl_k(gemm_f16_stream_kernel<BN>, dim3(G), dim3(C::THREADS), C::SMEM, st, wmap, xmap, a, n_rt);
  }
  return 1;
}

int launch_linear_stream_f16(const LinearArgs& a, bool lm_head, cudaStream_t st) {
  if (a.wfmt != 0 || a.M <= 0 || a.M > 64 || a.K % 64) return -1;
  if (a.M <= 16) return run_head<16>(a, lm_head, st);
  if (a.M <= 32) return run_head<32>(a, lm_head, st);
  return run_head<64>(a, lm_head, st);
}

}  // namespace pipo
