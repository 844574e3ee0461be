// k_gemm_tc.cu — fused int4-g64 (or fp16) x fp16 GEMM on the 5th-gen tensor cores
// (tcgen05.mma, accumulators in TMEM) for the b >= 16 path:
// prefill (M = b*P) and large-batch decode (M = b).
//
// Swap-AB: D[128 weight rows x BN activation rows] += W_tile[128 x 16] . X_tile[BN x 16]^T
// with both operands K-major in shared memory in the canonical SWIZZLE_128B layout
// (8-row x 128-B atoms, 16-B chunk c of row r stored at chunk c ^ (r & 7)).
// Per 64-wide k-block (one quantization group):
//   * all 128 threads cp.async the raw int4 block (4352 B, contiguous in the blob)
//     and the x tile (BN rows x 128 B, written to swizzled positions) into a ring of
//     NS stages, LOOKAHEAD = NS - 2 k-blocks ahead;
//   * thread r unpacks+scales row r's 64 codes (fp16_rne(q*s), kernel K8 arithmetic)
//     into the fp16 A tile (2 buffers) — the dequantized weight never exists in HBM;
//   * fence.proxy.async + barrier, then ONE thread issues 4 tcgen05.mma (K = 16 each)
//     and tcgen05.commit's an mbarrier; stage/buffer reuse waits on the mbarrier of
//     the MMA two k-blocks back, so MMAs overlap the next k-blocks' loads/unpack.
// Epilogue: tcgen05.ld (32x32b.x16) -> bias / residual / ReLU / QKV scatter, lanes =
// weight rows so stores of one activation row are contiguous across the warp.
// Split-K uses a deterministic fixup (partials in fixed split order).
#include "common.cuh"
#include "launch.cuh"
#include "kernels.h"
#include "layout.h"
#include "epilogue.cuh"

namespace pipo {

namespace tc {

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity));
}

__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void tc_after_sync() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_before_sync() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }

__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);           // start address
  d |= (uint64_t)((1024 >> 4) & 0x3FFF) << 32;      // SBO: 8 rows x 128 B
  d |= (uint64_t)1 << 46;                           // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;                           // SWIZZLE_128B
  return d;
}

__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

}  // namespace tc

constexpr int TC_THREADS = 128;

template <int WT, int BN>
struct TcCfg {
  static constexpr int NS = BN >= 256 ? 4 : 6;               // raw/x ring stages
  static constexpr int LOOK = NS - 2;                          // k-blocks in flight
  static constexpr int RAW = WT ? (int)kInt4BlockBytes : (int)kFp16BlockBytes;
  static constexpr int RAW_STAGE = (RAW + 127) / 128 * 128;
  static constexpr int X_STAGE = BN * 128;                     // BN rows x 64 halves
  static constexpr int A_TILE = 128 * 128;                     // 128 rows x 64 halves
  static constexpr int TMEM_COLS = BN < 32 ? 32 : BN;
  static constexpr int SMEM = 1024 + NS * (RAW_STAGE + X_STAGE) + 2 * A_TILE + 64;
  static constexpr uint32_t IDESC = (1u << 4) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
};

template <int WT, int BN>
__global__ void __launch_bounds__(TC_THREADS, 1) gemm_tc_kernel(LinearArgs a, int kb_per_split, int n_splits) {
  using C = TcCfg<WT, BN>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base_u32 = (smem_u32(smem_raw) + 1023u) & ~1023u;
  uint8_t* base = smem_raw + (base_u32 - smem_u32(smem_raw));
  uint8_t* xs = base;                                            // NS x X_STAGE (1024-aligned)
  uint8_t* as = base + C::NS * C::X_STAGE;                       // 2 x A_TILE
  uint8_t* raw = as + 2 * C::A_TILE;                             // NS x RAW_STAGE
  uint64_t* bars = reinterpret_cast<uint64_t*>(raw + C::NS * C::RAW_STAGE);   // 2 mbarriers
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int rt = blockIdx.x, mt = blockIdx.y, split = blockIdx.z;
  const int n_kb = a.K / 64;
  const int kb0 = split * kb_per_split, kb1 = min(n_kb, kb0 + kb_per_split);
  const int nk = max(0, kb1 - kb0);
  const int m0 = mt * BN;
  const uint8_t* wbase = a.w + (int64_t)rt * n_kb * C::RAW;

  if (tid == 0) {
    tc::mbar_init(&bars[0], 1);
    tc::mbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                 "r"((uint32_t)C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  tc::tc_before_sync();
  __syncthreads();
  tc::tc_after_sync();
  const uint32_t tmem = *tmem_slot;

  auto load_stage = [&](int i) {
    const int s = i % C::NS, kb = kb0 + i;
    const uint8_t* src = wbase + (int64_t)kb * C::RAW;
    uint8_t* dst = raw + s * C::RAW_STAGE;
    for (int c = tid; c < C::RAW / 16; c += TC_THREADS) cp_async16(dst + c * 16, src + c * 16);
    uint8_t* xd = xs + s * C::X_STAGE;
    for (int c = tid; c < BN * 8; c += TC_THREADS) {
      const int r = c >> 3, ch = c & 7, m = m0 + r;
      const __half* xsrc = a.x + (int64_t)min(m, a.M - 1) * a.K + (int64_t)kb * 64 + ch * 8;
      cp_async16(xd + r * 128 + ((ch ^ (r & 7)) << 4), xsrc, m < a.M ? 16 : 0);
    }
  };

#pragma unroll
  for (int i = 0; i < C::LOOK; ++i) {
    if (i < nk) load_stage(i);
    cp_async_commit();
  }

  for (int i = 0; i < nk; ++i) {
    const int s = i % C::NS, ab = i & 1;
    // MMA(i-2) read A[ab], x/raw stage (i-2)%NS: wait for it before reuse
    if (i >= 2) tc::mbar_wait(&bars[ab], ((i - 2) >> 1) & 1);
    if (i + C::LOOK < nk) load_stage(i + C::LOOK);
    cp_async_commit();
    cp_async_wait<C::LOOK>();
    __syncthreads();
    // unpack + scale the weight block into the swizzled fp16 A tile
    const uint8_t* rs = raw + s * C::RAW_STAGE;
    uint8_t* at = as + ab * C::A_TILE;
    const int r = tid;
    if constexpr (WT == 1) {
      const __half2 s2 = __half2half2(*reinterpret_cast<const __half*>(rs + 4096 + r * 2));
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint4 cw = *reinterpret_cast<const uint4*>(rs + (h * 128 + r) * 16);
        __half2 o[16];
        dequant8(cw.x, s2, o + 0);
        dequant8(cw.y, s2, o + 4);
        dequant8(cw.z, s2, o + 8);
        dequant8(cw.w, s2, o + 12);
        const uint4* src = reinterpret_cast<const uint4*>(o);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int ch = h * 4 + q;
          *reinterpret_cast<uint4*>(at + r * 128 + ((ch ^ (r & 7)) << 4)) = src[q];
        }
      }
    } else {
#pragma unroll
      for (int ch = 0; ch < 8; ++ch)
        *reinterpret_cast<uint4*>(at + r * 128 + ((ch ^ (r & 7)) << 4)) =
            *reinterpret_cast<const uint4*>(rs + r * 128 + ch * 16);
    }
    tc::fence_proxy_async();
    __syncthreads();
    if (tid == 0) {
      tc::tc_after_sync();
      const uint32_t a_addr = smem_u32(at), b_addr = smem_u32(xs + s * C::X_STAGE);
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        tc::mma_f16(tmem, tc::sw128_desc(a_addr + kk * 32), tc::sw128_desc(b_addr + kk * 32), C::IDESC,
                    (i > 0 || kk > 0) ? 1u : 0u);
      tc::mma_commit(&bars[ab]);
    }
  }
  cp_async_wait<0>();
  if (nk > 0) tc::mbar_wait(&bars[(nk - 1) & 1], ((nk - 1) >> 1) & 1);
  tc::tc_after_sync();

  // ---- epilogue: row n = rt*128 + tid (TMEM lane), columns = activation rows ----
  const int n = rt * 128 + warp * 32 + lane;
  const uint32_t t_row = tmem + ((uint32_t)(warp * 32) << 16);
  const int n_tiles = gridDim.x * gridDim.y, tile = mt * gridDim.x + rt;
  if (n_splits == 1) {
    for (int c0 = 0; c0 < BN; c0 += 16) {
      float v[16];
      if (nk > 0) tc::tmem_ld16(t_row + c0, v);
      else
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = 0.f;
#pragma unroll
      for (int j = 0; j < 16; ++j) epi_store(a.epi, m0 + c0 + j, n, v[j]);
    }
  } else {
    __shared__ int s_last;
    float* part = a.ws + ((int64_t)split * n_tiles + tile) * (BN * 128);
    for (int c0 = 0; c0 < BN; c0 += 16) {
      float v[16];
      if (nk > 0) tc::tmem_ld16(t_row + c0, v);
      else
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = 0.f;
#pragma unroll
      for (int j = 0; j < 16; ++j) __stcg(part + (c0 + j) * 128 + tid, v[j]);
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = (atomicAdd(&a.counters[tile], 1) == n_splits - 1);
    __syncthreads();
    if (s_last) {
      __threadfence();
      for (int c = 0; c < BN; ++c) {
        float acc = 0.f;
        for (int sp = 0; sp < n_splits; ++sp)
          acc += __ldcg(a.ws + ((int64_t)sp * n_tiles + tile) * (BN * 128) + c * 128 + tid);
        epi_store(a.epi, m0 + c, n, acc);
      }
      if (tid == 0) a.counters[tile] = 0;
    }
  }
  tc::tc_before_sync();
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"((uint32_t)C::TMEM_COLS));
}

template <int WT, int BN>
static int run_gemm_tc(const LinearArgs& a, cudaStream_t st) {
  using C = TcCfg<WT, BN>;
  ensure_max_smem(gemm_tc_kernel<WT, BN>, C::SMEM);
  const int n_rt = (a.N + 127) / 128, m_tiles = (a.M + BN - 1) / BN, n_kb = a.K / 64;
  const int tiles = n_rt * m_tiles;
  const int per_sm = C::SMEM <= 113 * 1024 ? 2 : 1;
  const int target = a.num_sms * per_sm;
  int splits = tiles >= target ? 1 : (target + tiles - 1) / tiles;
  splits = max(1, min(splits, n_kb / 4));
  int kb_per = (n_kb + splits - 1) / splits;
  splits = (n_kb + kb_per - 1) / kb_per;
  if (splits > 1 && ((int64_t)splits * tiles * BN * 128 > a.ws_floats || tiles > a.n_counters)) {
    splits = 1;
    kb_per = n_kb;
  }
  dim3 grid(n_rt, m_tiles, splits);
  gemm_tc_kernel<WT, BN><<<grid, TC_THREADS, C::SMEM, st>>>(a, kb_per, splits);
  return 1;
}

int launch_linear_tc(const LinearArgs& a, cudaStream_t st) {
  if (a.wfmt == 1) {
    if (a.M <= 16) return run_gemm_tc<1, 16>(a, st);
    if (a.M <= 32) return run_gemm_tc<1, 32>(a, st);
    if (a.M <= 64) return run_gemm_tc<1, 64>(a, st);
    if (a.M <= 128) return run_gemm_tc<1, 128>(a, st);
    return run_gemm_tc<1, 256>(a, st);
  }
  if (a.M <= 16) return run_gemm_tc<0, 16>(a, st);
  if (a.M <= 32) return run_gemm_tc<0, 32>(a, st);
  if (a.M <= 64) return run_gemm_tc<0, 64>(a, st);
  if (a.M <= 128) return run_gemm_tc<0, 128>(a, st);
  return run_gemm_tc<0, 256>(a, st);
}

}  // namespace pipo
