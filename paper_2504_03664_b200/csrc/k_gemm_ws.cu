// k_gemm_ws.cu — warp-specialized, persistent stream-K int4-g64 GEMM on tcgen05 for
// the decode linears (M = b <= 256) and prefill.  This is the kernel that consumes each
// streamed weight segment as it lands (a6/a8/a10/a11 of SURVEY.md §8(a)).
//
// Grid = min(#SMs, units) CTAs; the (weight-row-tile, m-tile, k-block) units are split
// into equal contiguous ranges (stream-K), so every SM reads the same number of
// weight bytes — no wave quantization, no per-CTA split-K tail.  A range spans 1..3
// output tiles; a tile covered by several CTAs is finished by the last CTA to arrive,
// which sums the partials in k order (deterministic) and runs the fused epilogue.
//
// Roles (320 threads):
//   warp 0      producer: cp.async.bulk of each raw int4 block (4352 B, contiguous in
//               the blob) and a TMA 2D load of the x tile (SWIZZLE_128B, zero-filled
//               out of bounds) into NR / NX -stage rings, mbarrier complete_tx;
//   warp 1      MMA issuer: 4 x tcgen05.mma (128 x BN x 16) per k-block into one of
//               two TMEM accumulators, tcgen05.commit releases the stages;
//   warps 2-5   unpack + scale: thread r turns row r's 64 codes into fp16_rne(q*s)
//               (kernel K8 arithmetic, 1 SHR + 4 LOP3 + 8 HALF2 ops per 8 codes)
//               written to the swizzled A tile; the dequantized weight never exists
//               in HBM;
//   warps 6-9   epilogue: tcgen05.ld the finished accumulator (lanes = weight rows),
//               bias / residual / ReLU / QKV-scatter, or stream-K partials + fixup.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "launch.cuh"
#include "epilogue.cuh"
#include "kernels.h"
#include "layout.h"

namespace pipo {
namespace ws {

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void tc_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)(1024 >> 4) << 32) | ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
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
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n.reg .pred P;\nelect.sync _|P, 0xffffffff;\nselp.u32 %0, 1, 0, P;\n}\n"
      : "=r"(pred));
  return pred != 0;
}
__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// non-blocking phase test: issued early, its result consumed later, so the mbarrier round
// trip overlaps other work
__device__ __forceinline__ uint32_t mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t done;
  asm volatile(
      "{\n.reg .pred P1;\nmbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\nselp.u32 %0, 1, 0, P1;\n}\n"
      : "=r"(done)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return done;
}
// polling wait with back-off, for warps that idle most of the time (the epilogue)
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  while (true) {
    asm volatile(
        "{\n.reg .pred P1;\nmbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\nselp.u32 %0, 1, 0, P1;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (done) return;
    __nanosleep(64);
  }
}

// stream-K partition of U units over G CTAs (U * G < 2^32: checked by the launchers)
__device__ __forceinline__ int64_t u_begin(int64_t c, int64_t U, int64_t G) {
  return (int64_t)((uint32_t)c * (uint32_t)U / (uint32_t)G);
}
__device__ __forceinline__ int cta_of_unit(int64_t u, int64_t U, int64_t G) {
  uint32_t c = (uint32_t)u * (uint32_t)G / (uint32_t)U;
  while (c + 1 < (uint32_t)G && u_begin(c + 1, U, G) <= u) ++c;
  while (c > 0 && u_begin(c, U, G) > u) --c;
  return (int)c;
}

// Programmatic dependent launch (PDL): a kernel launched with
// cudaLaunchAttributeProgrammaticStreamSerialization may start (prologue: barrier init,
// TMEM alloc, descriptor prefetch) while its predecessor in the stream drains;
// griddep_wait() blocks until the predecessor grid has completed and its memory is
// visible, so every read of a predecessor's output and every global write comes after
// it.  griddep_launch() lets this grid's dependents be scheduled early.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

}  // namespace ws

template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

constexpr int WS_THREADS = 448;   // producer, MMA, 8 unpack warps, 4 epilogue warps

// One stream-K unit = TWO 128-row weight tiles (256 output features) x one 64-wide
// k-block: 8.5 KiB of int4 weights per x tile (halves the x re-reads from L2 and the
// per-unit synchronisation cost).
template <int BN>
struct WsCfg {
  static constexpr int NS = BN <= 32 ? 8 : (BN <= 64 ? 6 : 4); // raw + x ring stages
  static constexpr int NA = 3;                                 // fp16 A stages (2 tiles each)
  static constexpr int RAW = 2 * (int)kInt4BlockBytes;        // 8704
  static constexpr int X_TILE = BN * 128;
  static constexpr int A_TILE = 2 * 128 * 128;                 // two 128 x 64 fp16 tiles
  static constexpr int TMEM_COLS = 4 * BN < 32 ? 32 : 4 * BN;  // 2 accumulators x 2 tiles
  static constexpr int SMEM = 1024 + NS * X_TILE + NA * A_TILE + NS * RAW + 512;
  static constexpr uint32_t IDESC = (1u << 4) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  static_assert(SMEM <= 227 * 1024, "shared memory budget");
  static_assert(TMEM_COLS <= 512, "TMEM budget");
};

template <int BN>
__global__ void __launch_bounds__(WS_THREADS, 1)
    gemm_ws_kernel(const __grid_constant__ CUtensorMap xmap, LinearArgs a, int n_rt, int m_tiles, int dbg) {
  using C = WsCfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base_u32 = (smem_u32(smem_raw) + 1023u) & ~1023u;
  uint8_t* base = smem_raw + (base_u32 - smem_u32(smem_raw));
  uint8_t* xs = base;
  uint8_t* as = xs + C::NS * C::X_TILE;
  uint8_t* raw = as + C::NA * C::A_TILE;
  uint64_t* bar = reinterpret_cast<uint64_t*>(raw + C::NS * C::RAW);
  uint64_t* raw_full = bar;
  uint64_t* raw_empty = raw_full + C::NS;
  uint64_t* x_full = raw_empty + C::NS;
  uint64_t* x_empty = x_full + C::NS;
  uint64_t* a_full = x_empty + C::NS;
  uint64_t* a_empty = a_full + C::NA;
  uint64_t* acc_full = a_empty + C::NA;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n_kb = a.K / 64;
  const int n_pairs = (n_rt + 1) >> 1;
  const int64_t U = (int64_t)n_pairs * m_tiles * n_kb, G = gridDim.x;
  const int64_t u0 = ws::u_begin(blockIdx.x, U, G), u1 = ws::u_begin(blockIdx.x + 1, U, G);

  if (tid == 0) {
    for (int i = 0; i < C::NS; ++i) {
      ws::mbar_init(&raw_full[i], 1);
      ws::mbar_init(&raw_empty[i], 8);
      ws::mbar_init(&x_full[i], 1);
      ws::mbar_init(&x_empty[i], 1);
    }
    for (int i = 0; i < C::NA; ++i) { ws::mbar_init(&a_full[i], 8); ws::mbar_init(&a_empty[i], 1); }
    for (int i = 0; i < 2; ++i) { ws::mbar_init(&acc_full[i], 1); ws::mbar_init(&acc_empty[i], 4); }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&xmap) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                 "r"((uint32_t)C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  ws::tc_before();
  __syncthreads();
  ws::tc_after();
  const uint32_t tmem = *tmem_slot;
  ws::griddep_wait();     // predecessor (producer of x, reader of the partials) has finished
  ws::griddep_launch();   // the stream-K reduce may be scheduled now
  uint64_t* tsbuf = (dbg & 32) ? reinterpret_cast<uint64_t*>(a.ws + (15ll << 20)) + blockIdx.x * 8 : nullptr;
  auto stamp = [&](int k) {
    if (tsbuf) {
      uint64_t t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      tsbuf[k] = t;
    }
  };
  if (tid == 0) stamp(0);

  if (warp == 0) {
    // ------------------------------ producer ------------------------------
    if (lane == 0) {
      int i = 0;
      for (int64_t u = u0; u < u1; ++u, ++i) {
        const int64_t tile = u / n_kb;
        const int kb = (int)(u - tile * n_kb);
        const int pr = (int)(tile % n_pairs), mt = (int)(tile / n_pairs);
        const int s = i % C::NS;
        const uint32_t ph = ((i / C::NS) & 1) ^ 1;
        const int rt0 = 2 * pr;
        const bool two = rt0 + 1 < n_rt;
        ws::mbar_wait(&raw_empty[s], ph);
        ws::mbar_expect_tx(&raw_full[s], two ? C::RAW : C::RAW / 2);
        ws::bulk_g2s(raw + s * C::RAW, a.w + ((int64_t)rt0 * n_kb + kb) * kInt4BlockBytes, kInt4BlockBytes,
                     &raw_full[s]);
        if (two)
          ws::bulk_g2s(raw + s * C::RAW + kInt4BlockBytes, a.w + ((int64_t)(rt0 + 1) * n_kb + kb) * kInt4BlockBytes,
                       kInt4BlockBytes, &raw_full[s]);
        ws::mbar_wait(&x_empty[s], ph);
        if (dbg & 4) {
          ws::mbar_arrive(&x_full[s]);
        } else {
          ws::mbar_expect_tx(&x_full[s], C::X_TILE);
          ws::tma_2d(xs + s * C::X_TILE, &xmap, kb * 64, mt * BN, &x_full[s]);
        }
      }
      stamp(1);
    }
  } else if (warp == 1) {
    // ------------------------------ MMA issuer ------------------------------
    if (lane == 0) {
      int i = 0, seg = 0;
      int64_t u = u0;
      while (u < u1) {
        const int64_t tile = u / n_kb;
        const int64_t seg_end = min(u1, (tile + 1) * n_kb);
        const bool two = 2 * (int)(tile % n_pairs) + 1 < n_rt;
        const int ab = seg & 1;
        ws::mbar_wait(&acc_empty[ab], ((seg >> 1) & 1) ^ 1);
        ws::tc_after();
        const uint32_t d = tmem + ab * (2 * BN);
        for (int64_t v = u; v < seg_end; ++v, ++i) {
          const int sa = i % C::NA, s = i % C::NS;
          ws::mbar_wait(&a_full[sa], (i / C::NA) & 1);
          ws::mbar_wait(&x_full[s], (i / C::NS) & 1);
          ws::tc_after();
          const uint32_t aa = smem_u32(as + sa * C::A_TILE), xa = smem_u32(xs + s * C::X_TILE);
#pragma unroll
          if (!(dbg & 2))
          for (int kk = 0; kk < 4; ++kk) {
            const uint32_t acc = (v > u || kk > 0) ? 1u : 0u;
            const uint64_t db = ws::sw128_desc(xa + kk * 32);
            ws::mma_f16(d, ws::sw128_desc(aa + kk * 32), db, C::IDESC, acc);
            if (two) ws::mma_f16(d + BN, ws::sw128_desc(aa + 128 * 128 + kk * 32), db, C::IDESC, acc);
          }
          if (dbg & 8) {
            ws::mbar_arrive(&a_empty[sa]);
            ws::mbar_arrive(&x_empty[s]);
          } else {
            ws::mma_commit(&a_empty[sa]);
            ws::mma_commit(&x_empty[s]);
          }
        }
        ws::mma_commit(&acc_full[ab]);
        u = seg_end;
        ++seg;
      }
    }
  } else if (warp < 10) {
    // ------------------------------ unpack + scale ------------------------------
    // 8 warps, 2 per SM sub-partition: thread d owns row r of tile t (d = t*128 + r)
    const int d = tid - 64, t = d >> 7, r = d & 127;
    const int sw = r & 7;
    int i = 0;
    for (int64_t u = u0; u < u1; ++u, ++i) {
      const int s = i % C::NS, sa = i % C::NA;
      ws::mbar_wait(&raw_full[s], (i / C::NS) & 1);
      const uint8_t* rs = raw + s * C::RAW + t * kInt4BlockBytes;
      const uint4 c0 = *reinterpret_cast<const uint4*>(rs + r * 16);
      const uint4 c1 = *reinterpret_cast<const uint4*>(rs + (128 + r) * 16);
      const __half2 s2 = __half2half2(*reinterpret_cast<const __half*>(rs + 4096 + r * 2));
      __syncwarp();
      if (lane == 0) ws::mbar_arrive(&raw_empty[s]);
      ws::mbar_wait(&a_empty[sa], ((i / C::NA) & 1) ^ 1);
      uint8_t* at = as + sa * C::A_TILE + t * (128 * 128) + r * 128;
      const uint32_t w[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
      if (!(dbg & 1))
#pragma unroll
      for (int ch = 0; ch < 8; ++ch) {
        __half2 o[4];
        dequant8(w[ch], s2, o);
        *reinterpret_cast<uint4*>(at + ((ch ^ sw) << 4)) = *reinterpret_cast<const uint4*>(o);
      }
      ws::fence_proxy_async();
      __syncwarp();
      if (lane == 0) ws::mbar_arrive(&a_full[sa]);
    }
  } else {
    // ------------------------------ epilogue ------------------------------
    const int quarter = warp & 3;                      // TMEM lanes 32*quarter .. +31
    const int row = quarter * 32 + lane;
    const int et = tid - 320;
    int seg = 0;
    int64_t u = u0;
    const int64_t first_tile_mine = u0 / n_kb;
    while (u < u1) {
      const int64_t tile = u / n_kb;
      const int64_t seg_end = min(u1, (tile + 1) * n_kb);
      const bool full = (u == tile * n_kb) && (seg_end == (tile + 1) * n_kb);
      const int pr = (int)(tile % n_pairs), mt = (int)(tile / n_pairs);
      const int m0 = mt * BN;
      const int ntile = (2 * pr + 1 < n_rt) ? 2 : 1;
      const int ab = seg & 1;
      // long wait: sleep between polls so the waiting warps do not steal issue slots
      {
        uint32_t done = 0;
        const uint32_t addr = smem_u32(&acc_full[ab]), par = (seg >> 1) & 1;
        while (true) {
          asm volatile(
              "{\n.reg .pred P1;\nmbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\nselp.u32 %0, 1, 0, P1;\n}\n"
              : "=r"(done)
              : "r"(addr), "r"(par)
              : "memory");
          if (done) break;
          __nanosleep(256);
        }
      }
      ws::tc_after();
      const bool last_seg = seg_end == u1;
      if (last_seg && et == 0) stamp(4);
      const int slot = 2 * (int)blockIdx.x + (tile == first_tile_mine ? 0 : 1);
      float* part = a.ws + (int64_t)slot * (2 * BN * 128);
      for (int t = 0; t < ntile; ++t) {
        const uint32_t t_row = tmem + ab * (2 * BN) + t * BN + ((uint32_t)(quarter * 32) << 16);
        const int n = (2 * pr + t) * 128 + row;
        for (int c0 = 0; c0 < BN; c0 += 16) {
          float v[16];
          ws::tmem_ld16(t_row + c0, v);
          if (full) {
            epi_store16(a.epi, m0 + c0, n, v);
          } else {
#pragma unroll
            for (int j = 0; j < 16; ++j) __stcg(part + (t * BN + c0 + j) * 128 + row, v[j]);
          }
        }
      }
      ws::tc_before();
      __syncwarp();
      if (lane == 0) ws::mbar_arrive(&acc_empty[ab]);
      if (last_seg && et == 0) stamp(5);
      u = seg_end;
      ++seg;
    }
    if (et == 0) stamp(2);
  }
  __syncwarp();          // lanes 1-31 of the producer / MMA warps wait for lane 0 (bar.sync is .aligned)
  ws::tc_before();
  __syncthreads();
  if (tid == 0) stamp(3);
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"((uint32_t)C::TMEM_COLS));
}


// Stream-K partial reduction (separate launch, fully parallel): tile `tile` of
// (pair, m-tile) was split across CTAs cf..cl; their partial accumulators are summed
// in k order (deterministic) and the fused epilogue runs.  grid = (tiles, BN/16).
template <int BN>
__global__ void __launch_bounds__(256) ws_reduce_kernel(LinearArgs a, int n_rt, int m_tiles, int G, int kbu, int dbg) {
  ws::griddep_wait();     // launched as a programmatic dependent of the GEMM: its partials
  ws::griddep_launch();
  if ((dbg & 128) && threadIdx.x == 0) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    atomicMin(reinterpret_cast<unsigned long long*>(a.ws + (15ll << 20)) + 148 * 16, (unsigned long long)t);
  }
  // grid = (tiles, BN/8): each thread owns one weight row of one tile and 8 columns;
  // contributors are loaded 4 at a time (32 loads in flight), summed in k order.
  // One block per CTA boundary c = blockIdx.x + 1: the tile holding unit u_begin(c) is
  // shared iff the boundary falls inside it; the first such boundary owns the reduce.
  __shared__ int s_cf, s_cl, s_first;
  const int n_ku = a.K / 64 / kbu, n_pairs = (n_rt + 1) >> 1;
  const int64_t U = (int64_t)n_pairs * m_tiles * n_ku;
  const int64_t ub = ws::u_begin(blockIdx.x + 1, U, G);
  const int64_t tile = ub / n_ku;
  if (ub == tile * n_ku || ws::u_begin(blockIdx.x, U, G) > tile * n_ku) return;
  if (threadIdx.x == 0) {
    s_cf = ws::cta_of_unit(tile * n_ku, U, G);
    s_cl = ws::cta_of_unit((tile + 1) * n_ku - 1, U, G);
    s_first = (int)(ws::u_begin(s_cf, U, G) / n_ku) == (int)tile;
  }
  __syncthreads();
  const int cf = s_cf, cl = s_cl;
  if (cf == cl) return;                                   // fully owned: stored by the GEMM
  const int pr = (int)(tile % n_pairs), mt = (int)(tile / n_pairs);
  const int t = threadIdx.x >> 7, row = threadIdx.x & 127;
  if (2 * pr + t >= n_rt) return;
  const int n = (2 * pr + t) * 128 + row, m0 = mt * BN, c0 = blockIdx.y * 8;
  float acc[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) acc[j] = 0.f;
  for (int cb = cf; cb <= cl; cb += 4) {
    float v[4][8];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int cc = cb + q;
      if (cc <= cl) {
        // slot: the tile is cc's first tile unless cc == cf and cf started in an earlier tile
        const int sl = 2 * cc + ((cc == cf && !s_first) ? 1 : 0);
        const float* src = a.ws + (int64_t)sl * (2 * BN * 128) + (t * BN + c0) * 128 + row;
#pragma unroll
        for (int j = 0; j < 8; ++j) v[q][j] = __ldcg(src + j * 128);
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (cb + q <= cl)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] += v[q][j];
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) epi_store(a.epi, m0 + c0 + j, n, acc[j]);
  if ((dbg & 128) && threadIdx.x == 0) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    atomicMax(reinterpret_cast<unsigned long long*>(a.ws + (15ll << 20)) + 148 * 16 + 1, (unsigned long long)t);
  }
}

// Stream-K reduce v2: one 256-thread block per (tile, 4 columns), float4 partial loads — only
// the tiles that exist (no early-exit blocks for CTA boundaries, no shared-memory
// broadcast), one resident wave.  Same operands and order as ws_reduce_kernel
// (0 + p_cf + p_cf+1 + ... in CTA order), so the two are bit-identical.
template <int BN, int CPT>
__global__ void __launch_bounds__(256) ws_reduce2_kernel(LinearArgs a, int n_rt, int m_tiles, int G, int kbu,
                                                          int late) {
  ws::griddep_wait();
  if (!late) ws::griddep_launch();   // late: no early trigger (implicit at block exit)
  const int n_ku = a.K / 64 / kbu, n_pairs = (n_rt + 1) >> 1;
  const int64_t U = (int64_t)n_pairs * m_tiles * n_ku;
  const int64_t tile = blockIdx.x;
  const int pr = (int)(tile % n_pairs), mt = (int)(tile / n_pairs);
  const int cf = ws::cta_of_unit(tile * n_ku, U, G), cl = ws::cta_of_unit((tile + 1) * n_ku - 1, U, G);
  if (cf == cl) return;                                   // owned whole: stored by the GEMM
  const bool cf_first = ws::u_begin(cf, U, G) / n_ku == tile;
  // thread -> (CPT columns c, weight tile t, 4 consecutive rows): float4 partial loads.
  // CPT > 1 puts CPT columns' loads in flight per thread and shrinks the grid to one
  // resident wave for the wide matrices (c5 QKV / FC1: 1344 / 1792 blocks at CPT = 1).
  const int t = (threadIdx.x >> 5) & 1, row4 = (threadIdx.x & 31) * 4;
  if (2 * pr + t >= n_rt) return;
  const int n = (2 * pr + t) * 128 + row4;
  float4 acc[CPT];
#pragma unroll
  for (int i = 0; i < CPT; ++i) acc[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int cb = cf; cb <= cl; cb += 4) {
    float4 v[4][CPT];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int cc = cb + q;
      if (cc <= cl) {
        const int sl = 2 * cc + ((cc == cf && !cf_first) ? 1 : 0);
#pragma unroll
        for (int i = 0; i < CPT; ++i) {
          const int c = (blockIdx.y * CPT + i) * 4 + (threadIdx.x >> 6);
          v[q][i] = __ldcg(reinterpret_cast<const float4*>(a.ws + (int64_t)sl * (2 * BN * 128) + (t * BN + c) * 128 + row4));
        }
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (cb + q <= cl)
#pragma unroll
        for (int i = 0; i < CPT; ++i) {
          acc[i].x += v[q][i].x; acc[i].y += v[q][i].y; acc[i].z += v[q][i].z; acc[i].w += v[q][i].w;
        }
  }
#pragma unroll
  for (int i = 0; i < CPT; ++i) {
    const int m = mt * BN + (blockIdx.y * CPT + i) * 4 + (threadIdx.x >> 6);
    epi_store4(a.epi, m, n, acc[i]);
  }
}

// ---------------------------------------------------------------------------------
// v5: A operand in TMEM.  The unpack warps write each dequantized 128 x 64 tile row
// straight into tensor memory with tcgen05.st (one 32x32b.x32 store per row: the row's
// 64 fp16 values = 32 columns), and the MMA reads A from TMEM (tcgen05.mma ... [a_tmem]).
// No shared-memory A ring, no swizzled STS, no generic->async proxy fence, and the
// freed shared memory deepens the raw-weight ring (NR stages in flight).
// Roles: warp 0 raw producer, 1 MMA, 2 .. 2+UW-1 unpack, then 4 epilogue warps, then
// the x producer.
// One unit = 2 weight tiles (256 rows) x KBU k-blocks: the per-unit synchronisation
// (mbarrier waits, tcgen05.commit, producer bookkeeping) is amortised over 8*KBU MMAs.
// NACC = 2 accumulator buffers (the epilogue of one tile overlaps the next tile's MMAs);
// 8 unpack warps (warp -> tile x lane quarter, all KBU k-blocks), software-pipelined.
// Per-unit mbarrier round trips are the kernel's hidden cost (~150-250 cycles each even on
// a completed phase; clock64 trace in profiles/r02/tm_fin/trace/): the MMA issuer waits on
// a_full only — one unpack warp (the "x gate") waits for the unit's x tile before its
// a_full arrival — and the unpack warps test the next raw stage with a non-blocking
// test_wait a unit's work before they need it.
template <int BN, int KBU, int NACC = 2, int UW = 98>
struct TmCfg {
  static constexpr int RAW_T = KBU * (int)kInt4BlockBytes;     // one tile's blocks (contiguous)
  static constexpr int RAW = 2 * RAW_T;
  static constexpr int NR = (KBU == 1 ? 16 : 8);                // raw unit stages
  static constexpr int X_KB = BN * 128;                         // x tile of one k-block
  static constexpr int X_TILE = KBU * X_KB;
  static constexpr int NX = (KBU == 1 ? 8 : 4);
  static constexpr int ACC_COLS = NACC * 2 * BN;                // NACC buffers x 2 tiles
  static constexpr int A_COLS = 2 * 32 * KBU;                   // per A stage (2 tiles x KBU x 32 cols)
  static constexpr int NA = (512 - ACC_COLS) / A_COLS < 8 ? (512 - ACC_COLS) / A_COLS : 8;
  static constexpr int UWW = 8;                                  // software-pipelined unpack warps
  static constexpr int E0 = 2 + UWW;                             // first epilogue warp
  static constexpr int XW = E0 + 4;                              // x producer warp
  static constexpr int THREADS = (XW + 1) * 32;
  static constexpr int SMEM = 1024 + NX * X_TILE + NR * RAW + 1024;   // + mbarriers (<= 70) and TMEM slot
  static constexpr uint32_t IDESC = (1u << 4) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  static_assert(SMEM <= 227 * 1024, "shared memory budget");
  static_assert(NA >= 2, "TMEM budget");
  static_assert(UW == 98, "software-pipelined unpack (8 warps) is the one built configuration");
  static_assert((2 * NR + 2 * NX + 2 * NA + 2 + NACC + 1) * 8 + 4 <= 1024, "barrier area");
};

__device__ __forceinline__ void mma_f16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(db), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};\n" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
      "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
      "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n" ::"r"(
          taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}

__device__ __forceinline__ uint64_t clk() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));
  return t;
}

template <int BN, int KBU, int NACC, int UW, bool FIN>
__global__ void __launch_bounds__(TmCfg<BN, KBU, NACC, UW>::THREADS, 1)
    gemm_tm_kernel(const __grid_constant__ CUtensorMap xmap, LinearArgs a, int n_rt, int m_tiles, int G, int dbg) {
  using C = TmCfg<BN, KBU, NACC, UW>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base_u32 = (smem_u32(smem_raw) + 1023u) & ~1023u;
  uint8_t* base = smem_raw + (base_u32 - smem_u32(smem_raw));
  uint8_t* xs = base;
  uint8_t* raw = xs + C::NX * C::X_TILE;
  uint64_t* bar = reinterpret_cast<uint64_t*>(raw + C::NR * C::RAW);
  uint64_t* raw_full = bar;
  uint64_t* raw_empty = raw_full + C::NR;
  uint64_t* x_full = raw_empty + C::NR;
  uint64_t* x_empty = x_full + C::NX;
  uint64_t* a_full = x_empty + C::NX;
  uint64_t* a_empty = a_full + C::NA;
  uint64_t* acc_full = a_empty + C::NA;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + NACC);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n_kb = a.K / 64, n_ku = n_kb / KBU;
  const int n_pairs = (n_rt + 1) >> 1;
  const int64_t U = (int64_t)n_pairs * m_tiles * n_ku;
  const int64_t u0 = ws::u_begin(blockIdx.x, U, G);
  const int64_t u1 = (dbg & 256) ? u0 : ws::u_begin(blockIdx.x + 1, U, G);   // debug: no work
  uint64_t* ts = (dbg & 128) ? reinterpret_cast<uint64_t*>(a.ws + (15ll << 20)) + blockIdx.x * 16 : nullptr;
  auto gstamp = [&](int k) {
    if (ts) {
      uint64_t t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      ts[k] = t;
    }
  };
  if (tid == 0) gstamp(9);

  if (tid == 0) {
    for (int i = 0; i < C::NR; ++i) { ws::mbar_init(&raw_full[i], 1); ws::mbar_init(&raw_empty[i], C::UWW); }
    for (int i = 0; i < C::NX; ++i) { ws::mbar_init(&x_full[i], 1); ws::mbar_init(&x_empty[i], 1); }
    for (int i = 0; i < C::NA; ++i) { ws::mbar_init(&a_full[i], C::UWW); ws::mbar_init(&a_empty[i], 1); }
    for (int i = 0; i < NACC; ++i) { ws::mbar_init(&acc_full[i], 1); ws::mbar_init(&acc_empty[i], 4); }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&xmap) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                 "r"(512u));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  ws::tc_before();
  __syncthreads();
  ws::tc_after();
  const uint32_t tmem = *tmem_slot;
  ws::griddep_wait();     // predecessor (producer of x, reader of the partials) has finished
  ws::griddep_launch();   // the stream-K reduce may be scheduled now
  const uint32_t a_base = tmem + C::ACC_COLS;           // A ring columns
  if (tid == 0) gstamp(10);
  uint64_t* wt = (dbg & 32) ? reinterpret_cast<uint64_t*>(a.ws + (15ll << 20)) + blockIdx.x * 16 : nullptr;
  uint64_t w_acc[2] = {0, 0};
  uint64_t w_st = 0;   // debug: unpack warps' tcgen05.wait::st cycles
  const uint64_t t_begin = clk();
#define TWAIT(slot, bar, par)                          \
  do {                                                 \
    const uint64_t t0_ = wt ? clk() : 0;               \
    ws::mbar_wait(bar, par);                           \
    if (wt) w_acc[slot] += clk() - t0_;                \
  } while (0)

  if (warp == 0) {
    // ------- raw int4 producer: per unit one bulk copy per tile (KBU blocks, contiguous) -------
    if (lane == 0) {
      int64_t tile = u0 / n_ku;
      int ku = (int)(u0 - tile * n_ku);
      int pr = (int)(tile % n_pairs);
      int s = 0;
      uint32_t ph = 1;
      const int64_t tile_stride = (int64_t)n_kb * kInt4BlockBytes;
      const uint8_t* wsrc = a.w + (int64_t)(2 * pr) * tile_stride + (int64_t)ku * C::RAW_T;
      for (int64_t u = u0; u < u1; ++u) {
        const bool two = 2 * pr + 1 < n_rt;
        TWAIT(0, &raw_empty[s], ph);
        if (dbg & 16) {   // debug: no weight traffic (stale stage contents)
          ws::mbar_arrive(&raw_full[s]);
        } else {
          ws::mbar_expect_tx(&raw_full[s], two ? C::RAW : C::RAW_T);
          ws::bulk_g2s(raw + s * C::RAW, wsrc, C::RAW_T, &raw_full[s]);
          if (two) ws::bulk_g2s(raw + s * C::RAW + C::RAW_T, wsrc + tile_stride, C::RAW_T, &raw_full[s]);
        }
        wsrc += C::RAW_T;
        if (++ku == n_ku) {
          ku = 0;
          if (++pr == n_pairs) pr = 0;
          wsrc = a.w + (int64_t)(2 * pr) * tile_stride;
        }
        if (++s == C::NR) { s = 0; ph ^= 1; }
      }
    }
  } else if (warp == C::XW) {
    // ---------------- x producer (TMA 2D, SWIZZLE_128B, KBU boxes per unit) ----------------
    if (lane == 0) {
      int64_t tile = u0 / n_ku;
      int ku = (int)(u0 - tile * n_ku);
      int pr = (int)(tile % n_pairs), mt = (int)(tile / n_pairs);
      int s = 0;
      uint32_t ph = 1;
      for (int64_t u = u0; u < u1; ++u) {
        TWAIT(0, &x_empty[s], ph);
        if (dbg & 8) {   // debug: no activation traffic (stale stage contents)
          ws::mbar_arrive(&x_full[s]);
        } else {
          ws::mbar_expect_tx(&x_full[s], C::X_TILE);
#pragma unroll
          for (int k = 0; k < KBU; ++k)
            ws::tma_2d(xs + s * C::X_TILE + k * C::X_KB, &xmap, (ku * KBU + k) * 64, mt * BN, &x_full[s]);
        }
        if (++ku == n_ku) {
          ku = 0;
          if (++pr == n_pairs) { pr = 0; ++mt; }
        }
        if (++s == C::NX) { s = 0; ph ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer: A from TMEM, B (x) from shared memory ----------------
    // The whole warp runs the loop (warp-uniform descriptors stay in uniform registers);
    // one elected lane issues the tcgen05.mma / tcgen05.commit instructions.
    int seg = 0, sa = 0, sx = 0;
    uint32_t ph_a = 0, ph_x = 0;
    int64_t u = u0;
    const uint32_t xs_base = smem_u32(xs);
    while (u < u1) {
      const int64_t tile = u / n_ku;
      const int64_t seg_end = min(u1, (tile + 1) * n_ku);
      const bool two = 2 * (int)(tile % n_pairs) + 1 < n_rt;
      const int ab = seg % NACC;
      ws::mbar_wait(&acc_empty[ab], ((seg / NACC) & 1) ^ 1);
      ws::tc_after();
      const uint32_t d = tmem + ab * (2 * BN);
      for (int64_t v = u; v < seg_end; ++v) {
        TWAIT(0, &a_full[sa], ph_a);
        // x_full: implied by a_full (the x gate unpack warp waits for it before arriving)
        ws::tc_after();
        if (ws::elect_one()) {
          const uint32_t at = a_base + sa * C::A_COLS;
          const uint64_t db0 = ws::sw128_desc(xs_base + sx * C::X_TILE);
#pragma unroll
          for (int k = 0; k < KBU; ++k)
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              const uint32_t acc = (v > u || k > 0 || kk > 0) ? 1u : 0u;
              const uint64_t db = db0 + (uint64_t)((k * C::X_KB + kk * 32) >> 4);
              if (!(dbg & 2)) {   // debug: skip the MMAs (commits still flow)
                mma_f16_ts(d, at + k * 64 + kk * 8, db, C::IDESC, acc);
                if (two) mma_f16_ts(d + BN, at + k * 64 + 32 + kk * 8, db, C::IDESC, acc);
              }
            }
          ws::mma_commit(&a_empty[sa]);
          ws::mma_commit(&x_empty[sx]);
        }
        __syncwarp();
        if (++sa == C::NA) { sa = 0; ph_a ^= 1; }
        if (++sx == C::NX) { sx = 0; ph_x ^= 1; }
      }
      if (ws::elect_one()) ws::mma_commit(&acc_full[ab]);
      __syncwarp();
      u = seg_end;
      ++seg;
    }
    if (lane == 0) gstamp(11);
    if (lane == 0 && ts) ts[2] = clk();
  } else if (warp < C::E0) {
    // ---------------- unpack + scale straight into TMEM ----------------
    // a warp may only touch its TMEM lane quarter (warp % 4): warp -> (tile, quarter),
    // all KBU k-blocks of the unit.
    const int t = (warp - 2) >> 2, q = warp & 3;
    const int r = q * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    {
      // software-pipelined: unit u+1's raw wait + shared loads + ring release are issued
      // while unit u's TMEM stores drain (before tcgen05.wait::st), so the per-unit
      // barrier/latency chain overlaps the store completion
      uint4 cw[KBU][2];
      __half2 s2[KBU];
      auto load_unit = [&](int64_t iu, uint4 (&c)[KBU][2], __half2 (&sc)[KBU], uint32_t ready) {
        const int s = (int)(iu % C::NR);
        if (!ready) TWAIT(0, &raw_full[s], (uint32_t)((iu / C::NR) & 1));
#pragma unroll
        for (int k = 0; k < KBU; ++k) {
          const uint8_t* rs = raw + s * C::RAW + t * C::RAW_T + k * kInt4BlockBytes;
          c[k][0] = *reinterpret_cast<const uint4*>(rs + r * 16);
          c[k][1] = *reinterpret_cast<const uint4*>(rs + (128 + r) * 16);
          sc[k] = __half2half2(*reinterpret_cast<const __half*>(rs + 4096 + r * 2));
        }
        __syncwarp();
        if (lane == 0) ws::mbar_arrive(&raw_empty[s]);
      };
      if (u0 < u1) load_unit(0, cw, s2, 0u);
      // x gate: one unpack warp also waits for the unit's activation tile before its a_full
      // arrival, so the MMA warp's single a_full wait covers both operands (one mbarrier
      // round trip less on the MMA issuer's per-unit loop); its test is issued here and
      // consumed ~a unit's unpack work later
      const bool xgate = warp == 2;
      for (int64_t u = u0; u < u1; ++u) {
        const int64_t iu = u - u0;
        const int sa = (int)(iu % C::NA);
        const int sxg = (int)(iu % C::NX);
        const uint32_t pxg = (uint32_t)((iu / C::NX) & 1);
        const uint32_t xok = xgate ? ws::mbar_test(&x_full[sxg], pxg) : 1u;
        // the next unit's raw stage, tested now and loaded after this unit's TMEM stores
        const uint32_t rok =
            u + 1 < u1 ? ws::mbar_test(&raw_full[(iu + 1) % C::NR], (uint32_t)(((iu + 1) / C::NR) & 1)) : 0u;
        TWAIT(1, &a_empty[sa], (uint32_t)(((iu / C::NA) & 1) ^ 1));
        ws::tc_after();
#pragma unroll
        for (int k = 0; k < KBU; ++k) {
          uint32_t o[32];
          const uint32_t w[8] = {cw[k][0].x, cw[k][0].y, cw[k][0].z, cw[k][0].w,
                                 cw[k][1].x, cw[k][1].y, cw[k][1].z, cw[k][1].w};
#pragma unroll
          for (int ch = 0; ch < 8; ++ch) dequant8(w[ch], s2[k], reinterpret_cast<__half2*>(o + ch * 4));
          tmem_st32(a_base + sa * C::A_COLS + k * 64 + t * 32 + lane_off, o);
        }
        if (u + 1 < u1) load_unit(iu + 1, cw, s2, rok);   // registers are free once the stores are issued
        const uint64_t tst_ = wt ? clk() : 0;
        asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
        if (wt) w_st += clk() - tst_;
        if (!xok) ws::mbar_wait(&x_full[sxg], pxg);
        ws::tc_before();
        __syncwarp();
        if (lane == 0) ws::mbar_arrive(&a_full[sa]);
      }
    }
  } else {
    // ---------------- epilogue: every segment but the last ----------------
    // (a segment = this CTA's maximal run of units inside one output tile).  The first
    // segment of a range that starts inside a tile is a stream-K CONTRIBUTOR: its partial
    // goes to the workspace early, released by a flag.  The last segment is drained below
    // by all unpack + epilogue warps together.
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    int seg = 0;
    int64_t u = u0;
    while (u < u1) {
      const int64_t tile = u / n_ku;
      const int64_t seg_end = min(u1, (tile + 1) * n_ku);
      if (seg_end == u1 && FIN) break;                     // the last segment: below
      const bool full = (u == tile * n_ku) && (seg_end == (tile + 1) * n_ku);
      const int pr = (int)(tile % n_pairs), mt = (int)(tile / n_pairs);
      const int m0 = mt * BN;
      const int ntile = (2 * pr + 1 < n_rt) ? 2 : 1;
      const int ab = seg % NACC;
      ws::mbar_wait_sleep(&acc_full[ab], (uint32_t)((seg / NACC) & 1));
      ws::tc_after();
      const int slot = 2 * (int)blockIdx.x + ((FIN || u == u0) ? 0 : 1);
      float* part = a.ws + (int64_t)slot * (2 * BN * 128);
      for (int tt = 0; tt < ntile; ++tt) {
        const uint32_t t_row = tmem + ab * (2 * BN) + tt * BN + ((uint32_t)(quarter * 32) << 16);
        const int n = (2 * pr + tt) * 128 + row;
        for (int c0 = 0; c0 < BN; c0 += 16) {
          float v[16];
          ws::tmem_ld16(t_row + c0, v);
          if (full) {
            epi_store16(a.epi, m0 + c0, n, v);
          } else {
#pragma unroll
            for (int j = 0; j < 16; ++j) __stcg(part + (tt * BN + c0 + j) * 128 + row, v[j]);
          }
        }
      }
      ws::tc_before();
      __syncwarp();
      if (lane == 0) ws::mbar_arrive(&acc_empty[ab]);
      if (FIN && !full) {   // contributor (only the first segment can be one): release the partial
        __threadfence();
        ws::named_bar(2, 128);
        if (warp == C::E0 && lane == 0) ws::st_release_u32(a.flags + blockIdx.x, 1u);
      }
      u = seg_end;
      ++seg;
    }
    if (warp == C::E0 && lane == 0) gstamp(12);
  }
  if (FIN && warp >= 2 && warp < C::XW && u0 < u1) {
    // ---------------- the last segment: all unpack + epilogue warps ----------------
    //  full        -> fused epilogue
    //  contributor -> partial + release flag (a range inside one tile)
    //  finisher    -> the CTA owning the tile's first unit: waits the flags of the CTAs
    //                 that cover the rest of the tile (their partials were written early,
    //                 in their first segment), adds them in k order — the order of the
    //                 separate reduce (0 + own + next + ...), so the result is bit-identical
    //                 — and runs the fused epilogue.  No second kernel.
    constexpr int NGRP = (C::UWW + 4) / 4;                  // warps per lane quarter
    const int quarter = warp & 3, grp = (warp - 2) >> 2;    // grp 0..NGRP-1
    const int row = quarter * 32 + lane;
    const int64_t tile = (u1 - 1) / n_ku, ts0 = tile * n_ku, te = ts0 + n_ku;
    const int seg = (int)(tile - u0 / n_ku);
    const int ab = seg % NACC;
    const bool contributor = u0 > ts0;
    const bool finisher = !contributor && u1 < te;
    const int pr = (int)(tile % n_pairs), mt = (int)(tile / n_pairs);
    const int m0 = mt * BN;
    const int ntile = (2 * pr + 1 < n_rt) ? 2 : 1;
    int c_last = (int)blockIdx.x;
    if (finisher)
      while (c_last + 1 < G && ws::u_begin(c_last + 1, U, G) < te) ++c_last;
    ws::mbar_wait_sleep(&acc_full[ab], (uint32_t)((seg / NACC) & 1));
    ws::tc_after();
    if (finisher) {
      if (warp == 2 && lane == 0)
        for (int cc = (int)blockIdx.x + 1; cc <= c_last; ++cc)
          while (ws::ld_acquire_u32(a.flags + cc) == 0) __nanosleep(32);
      ws::named_bar(1, NGRP * 128);
    }
    float* part = a.ws + (int64_t)(2 * (int)blockIdx.x) * (2 * BN * 128);
    for (int ch = grp; ch < ntile * (BN / 16); ch += NGRP) {
      const int tt = ch / (BN / 16), c0 = (ch % (BN / 16)) * 16;
      const int n = (2 * pr + tt) * 128 + row;
      float v[16];
      ws::tmem_ld16(tmem + ab * (2 * BN) + tt * BN + c0 + ((uint32_t)(quarter * 32) << 16), v);
      if (contributor) {
#pragma unroll
        for (int j = 0; j < 16; ++j) __stcg(part + (tt * BN + c0 + j) * 128 + row, v[j]);
        continue;
      }
      // k order (own, bid+1, bid+2, ...), two contributors' loads in flight at a time
      int cc = (int)blockIdx.x + 1;
      for (; cc <= c_last; cc += 2) {
        const bool two = cc + 1 <= c_last;
        const float* pa = a.ws + (int64_t)(2 * cc) * (2 * BN * 128) + (tt * BN + c0) * 128 + row;
        const float* pb = pa + (two ? 2 * (2 * BN * 128) : 0);
        float xa[16], xb[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) xa[j] = __ldcg(pa + j * 128);
#pragma unroll
        for (int j = 0; j < 16; ++j) xb[j] = two ? __ldcg(pb + j * 128) : 0.f;
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] += xa[j];
        if (two)
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] += xb[j];
      }
      epi_store16(a.epi, m0 + c0, n, v);
    }
    if (contributor) {
      __threadfence();
      ws::named_bar(1, NGRP * 128);
      if (warp == 2 && lane == 0) ws::st_release_u32(a.flags + blockIdx.x, 1u);
    } else if (finisher) {
      ws::named_bar(1, NGRP * 128);   // every partial read before the flags are re-armed
      if (warp == 2 && lane == 0)
        for (int cc = (int)blockIdx.x + 1; cc <= c_last; ++cc) a.flags[cc] = 0u;
    }
  }
  if (wt && lane == 0) {
    // slots: 0/1 raw producer, 2/3 MMA (a_full, x_full), 4/5 unpack warp 2 (raw_full, a_empty),
    // 6/7 x producer, 8 = total cycles of the MMA thread
    const int role = warp == 0 ? 0 : warp == 1 ? 1 : warp == 2 ? 2 : warp == C::XW ? 3 : -1;
    if (role >= 0) { wt[2 * role] = w_acc[0]; wt[2 * role + 1] = w_acc[1]; }
    if (warp == 1) wt[8] = clk() - t_begin;
    if (warp == 2) { wt[9] = w_st; wt[10] = clk() - t_begin; }
  }
#undef TWAIT
  __syncwarp();
  ws::tc_before();
  __syncthreads();
  if (tid == 0) gstamp(13);
  const uint64_t c13 = ts ? clk() : 0;
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512u));
  if (tid == 0) gstamp(14);
  if (tid == 0 && ts) { ts[0] = clk() - c13; ts[1] = c13 - ts[2]; }   // cycles: teardown, barrier - MMA end
}

// ---------------------------------------------------------------------------------
// host side: TMA descriptor for the activation matrix x [rows][K] fp16 (row-major)
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encode() {
  static PFN_encodeTiled fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess) fn = (PFN_encodeTiled)p;
    cudaGetLastError();
  }
  return fn;
}

static bool make_xmap(CUtensorMap* map, const __half* x, int64_t rows, int64_t K, int box_rows) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)K * 2};
  const cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<__half*>(x), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int BN>
static int run_ws(const LinearArgs& a, cudaStream_t st) {
  using C = WsCfg<BN>;
  ensure_max_smem(gemm_ws_kernel<BN>, C::SMEM);
  const int n_rt = (a.N + 127) / 128, m_tiles = (a.M + BN - 1) / BN, n_kb = a.K / 64;
  const int n_pairs = (n_rt + 1) / 2;
  const int64_t U = (int64_t)n_pairs * m_tiles * n_kb;
  // at least 8 units per CTA: the per-CTA prologue / epilogue must stay amortized
  const int G = (int)std::max<int64_t>(1, std::min<int64_t>(a.num_sms, U / 8));
  const int64_t tiles = (int64_t)n_pairs * m_tiles;
  if ((int64_t)2 * G * 2 * BN * 128 > a.ws_floats || tiles > a.n_counters || U * G >= (1ll << 32)) return -1;
  CUtensorMap map;   // rows >= M are out of bounds: TMA zero-fills them
  if (!make_xmap(&map, a.x, a.M, a.K, BN)) return -1;
  static const int dbg = getenv("PIPO_WS_DEBUG") ? atoi(getenv("PIPO_WS_DEBUG")) : 0;
  launch_pdl(gemm_ws_kernel<BN>, dim3(G), dim3(WS_THREADS), C::SMEM, st, map, a, n_rt, m_tiles, dbg);
  if (dbg & 64) return 1;   // debug: main kernel only
  if (G > 1) {
    dim3 rg((unsigned)(G - 1), BN / 8);
    launch_pdl(ws_reduce_kernel<BN>, rg, dim3(256), 0, st, a, n_rt, m_tiles, G, 1, 0);
  }
  return G > 1 ? 2 : 1;
}


template <int BN, int KBU, int NACC = 2, int UW = 8>
static int run_tm(const LinearArgs& a_in, cudaStream_t st) {
  using C = TmCfg<BN, KBU, NACC, UW>;
  LinearArgs a = a_in;
  const int n_rt = (a.N + 127) / 128, m_tiles = (a.M + BN - 1) / BN, n_kb = a.K / 64;
  const int n_pairs = (n_rt + 1) / 2, n_ku = n_kb / KBU;
  const int64_t U = (int64_t)n_pairs * m_tiles * n_ku;
  const int G = (int)std::max<int64_t>(1, std::min<int64_t>(a.num_sms, U / (8 / KBU)));
  // In-kernel fixup when a split tile spans at most ~3.5 CTAs (units per CTA >= 2/7 of a
  // tile's units): its finisher then adds one to three partials.  Wider spans (long-K
  // matrices: c5 out-proj / FC2, c6 QKV / FC2) keep the separate reduce, which spreads the
  // sums over the whole GPU instead of one finisher CTA per tile (measured on B200,
  // profiles/r02/tm_fin/).
  static const int dbg = getenv("PIPO_WS_DEBUG") ? atoi(getenv("PIPO_WS_DEBUG")) : 0;
  const bool fin = (int64_t)n_ku * G * 2 <= 7 * U && !(dbg & 512);   // debug 512: always the separate reduce
  if (fin) ensure_max_smem(gemm_tm_kernel<BN, KBU, NACC, UW, true>, C::SMEM);
  else ensure_max_smem(gemm_tm_kernel<BN, KBU, NACC, UW, false>, C::SMEM);
  if ((int64_t)2 * G * 2 * BN * 128 > a.ws_floats || U * G >= (1ll << 32)) return -1;
  // fixup flags: the top 512 split-K counters (zero at rest; the finisher re-arms them)
  if (fin && (a.n_counters < 1024 || G > 512)) return -1;
  a.flags = reinterpret_cast<uint32_t*>(a.counters + a.n_counters - 512);
  CUtensorMap map;
  if (!make_xmap(&map, a.x, a.M, a.K, BN)) return -1;
  if (fin) {
    // Stream-K fixup inside the kernel: the CTA owning a split tile's first unit finishes
    // it from TMEM with its neighbours' partials (written early, released by flags).  The
    // finisher spins on other CTAs' flags, so every CTA must be able to become resident:
    // G <= #SMs at one CTA per SM, and a contributor never waits on anything but its own
    // pipeline.
    launch_pdl(gemm_tm_kernel<BN, KBU, NACC, UW, true>, dim3(G), dim3(C::THREADS), C::SMEM, st, map, a, n_rt, m_tiles,
               G, dbg);
    return 1;
  }
  launch_pdl(gemm_tm_kernel<BN, KBU, NACC, UW, false>, dim3(G), dim3(C::THREADS), C::SMEM, st, map, a, n_rt, m_tiles,
             G, dbg);
  if (dbg & 64) return 1;   // debug: main kernel only
  if (G > 1) {
    // (tile, 4 columns) x (2 weight tiles x 32 row quads)
    dim3 rg((unsigned)((int64_t)n_pairs * m_tiles), BN / 4);
    launch_pdl(ws_reduce2_kernel<BN, 1>, rg, dim3(256), 0, st, a, n_rt, m_tiles, G, KBU, 0);
  }
  return G > 1 ? 2 : 1;
}

int launch_linear_tm(const LinearArgs& a, cudaStream_t st) {
  // 8 software-pipelined unpack warps (unit u+1's raw wait / shared loads overlap unit u's
  // TMEM store drain), two accumulators, 2-k-block units when K/64 is even.  The other
  // configurations measured on B200 (one accumulator, 16 or 2 x 8 unpack warps, 1-k-block
  // units with 4-6 A stages: profiles/r01/tm_pipe, profiles/r02/tm_fixup) were slower.
  if (a.wfmt != 1) return -1;
  const bool even = (a.K / 64) % 2 == 0;
  if (a.M <= 16) return even ? run_tm<16, 2, 2, 98>(a, st) : run_tm<16, 1, 2, 98>(a, st);
  if (a.M <= 32) return even ? run_tm<32, 2, 2, 98>(a, st) : run_tm<32, 1, 2, 98>(a, st);
  if (a.M <= 64) return even ? run_tm<64, 2, 2, 98>(a, st) : run_tm<64, 1, 2, 98>(a, st);
  return -1;
}

// ---------------------------------------------------------------------------------
// Prefill: the same roles as gemm_tm_kernel (A = dequantized weights in TMEM, x by TMA,
// one elected MMA lane), scheduled for M = b*P >> 128 where the GEMM is tensor-bound.
//  * static persistent schedule: CTA c owns output tiles c, c+G, ... and the whole K
//    of each (no stream-K partials, no reduce pass);
//  * tile order = weight-tile group fastest: at any moment the 148 CTAs work on ~2
//    token tiles, so the x tile is read from HBM about once and the weights (<= 110 MB
//    per matrix) stay resident in the 126 MB L2 across token tiles;
//  * TILES weight tiles (128 rows each) share one x stage: x is reused 128*TILES times
//    per load, each dequantized weight BN times;
//  * NACC accumulator sets (TILES*BN TMEM columns each); with NACC = 2 the epilogue of
//    tile i overlaps the MMAs of tile i+1;
//  * EPW epilogue warps (4 or 8): with 8, two warps share each TMEM lane quarter and
//    split the columns.
// KBU k-blocks per pipeline unit (TILES = 1 only): one raw bulk copy, one x stage of KBU
// TMA boxes, one A stage of KBU x 32 TMEM columns and ONE round of barrier hand-offs per
// unit — the per-unit synchronisation chain (~700 cycles, see the decode anatomy in
// DESIGN.md) is then paid once per 2 k-blocks = 8 MMAs instead of 4.
template <int BN, int TILES, int NACC, int EPW, int KBU = 1>
struct TpCfg {
  static constexpr int RAW_T = (int)kInt4BlockBytes;
  static constexpr int RAW = TILES * RAW_T * KBU;
  static constexpr int NR = KBU == 1 ? 12 : 4;
  static constexpr int X_KB = BN * 128;                  // x of one k-block
  static constexpr int X_ST = KBU * X_KB;                // x stage
  static constexpr int NX_MAX = ((KBU == 1 ? 200 : 210) * 1024 - NR * RAW) / X_ST;
  static constexpr int NX = NX_MAX > 8 ? 8 : NX_MAX;
  static constexpr int ACC_COLS = NACC * TILES * BN;
  static constexpr int A_COLS = TILES * 32 * KBU;
  static constexpr int NA = (512 - ACC_COLS) / A_COLS < 8 ? (512 - ACC_COLS) / A_COLS : 8;
  static constexpr int THREADS = (10 + EPW + 1) * 32;   // x producer is the last warp
  static constexpr int XW = 10 + EPW;
  static constexpr int SMEM = 1024 + NX * X_ST + NR * RAW + 512;
  static constexpr uint32_t IDESC = (1u << 4) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  static_assert(SMEM <= 227 * 1024, "shared memory budget");
  static_assert(NX >= (KBU == 1 ? 3 : 2), "x ring depth");
  static_assert(KBU == 1 || TILES == 1, "multi-k-block units with one weight tile per unit");
  static_assert(NA >= 2, "TMEM budget");
  static_assert(BN % 16 == 0 && BN >= 16 && BN <= 256, "MMA N");
  static_assert(EPW == 4 || EPW == 8, "epilogue warps");
};


template <int BN, int TILES, int NACC, int EPW, int KBU>
__global__ void __launch_bounds__(TpCfg<BN, TILES, NACC, EPW, KBU>::THREADS, 1)
    gemm_tp_kernel(const __grid_constant__ CUtensorMap xmap, LinearArgs a, int n_rt, int m_tiles) {
  using C = TpCfg<BN, TILES, NACC, EPW, KBU>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base_u32 = (smem_u32(smem_raw) + 1023u) & ~1023u;
  uint8_t* base = smem_raw + (base_u32 - smem_u32(smem_raw));
  uint8_t* xs = base;
  uint8_t* raw = xs + C::NX * C::X_ST;
  uint64_t* bar = reinterpret_cast<uint64_t*>(raw + C::NR * C::RAW);
  uint64_t* raw_full = bar;
  uint64_t* raw_empty = raw_full + C::NR;
  uint64_t* x_full = raw_empty + C::NR;
  uint64_t* x_empty = x_full + C::NX;
  uint64_t* a_full = x_empty + C::NX;
  uint64_t* a_empty = a_full + C::NA;
  uint64_t* acc_full = a_empty + C::NA;
  uint64_t* acc_empty = acc_full + NACC;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + NACC);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n_kb = a.K / 64;                 // n_kb % KBU == 0 (checked by the launcher)
  const int n_grp = (n_rt + TILES - 1) / TILES;
  const int n_tiles = n_grp * m_tiles;
  const int G = gridDim.x;

  if (tid == 0) {
    for (int i = 0; i < C::NR; ++i) { ws::mbar_init(&raw_full[i], 1); ws::mbar_init(&raw_empty[i], 8); }
    for (int i = 0; i < C::NX; ++i) { ws::mbar_init(&x_full[i], 1); ws::mbar_init(&x_empty[i], 1); }
    for (int i = 0; i < C::NA; ++i) { ws::mbar_init(&a_full[i], 8); ws::mbar_init(&a_empty[i], 1); }
    for (int i = 0; i < NACC; ++i) { ws::mbar_init(&acc_full[i], 1); ws::mbar_init(&acc_empty[i], EPW); }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&xmap) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                 "r"(512u));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  ws::tc_before();
  __syncthreads();
  ws::tc_after();
  const uint32_t tmem = *tmem_slot;
  ws::griddep_wait();     // predecessor (producer of x, reader of the partials) has finished
  ws::griddep_launch();   // the stream-K reduce may be scheduled now
  const uint32_t a_base = tmem + C::ACC_COLS;

  if (warp == 0) {
    // ---------------- raw int4 producer: one bulk copy per weight tile and k-block ----------------
    if (lane == 0) {
      const int64_t tile_stride = (int64_t)n_kb * kInt4BlockBytes;
      int s = 0;
      uint32_t ph = 1;
      for (int tile = blockIdx.x; tile < n_tiles; tile += G) {
        const int grp = tile % n_grp;
        const int nt = min(TILES, n_rt - grp * TILES);
        const uint8_t* wsrc = a.w + (int64_t)(grp * TILES) * tile_stride;
        for (int kb = 0; kb < n_kb; kb += KBU) {
          ws::mbar_wait(&raw_empty[s], ph);
          ws::mbar_expect_tx(&raw_full[s], nt * C::RAW_T * KBU);
          for (int t = 0; t < nt; ++t)   // a tile's KBU blocks are contiguous
            ws::bulk_g2s(raw + s * C::RAW + t * C::RAW_T, wsrc + t * tile_stride, C::RAW_T * KBU, &raw_full[s]);
          wsrc += kInt4BlockBytes * KBU;
          if (++s == C::NR) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == C::XW) {
    // ---------------- x producer (TMA 2D, SWIZZLE_128B; rows >= M zero-filled) ----------------
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 1;
      for (int tile = blockIdx.x; tile < n_tiles; tile += G) {
        const int mt = tile / n_grp;
        for (int kb = 0; kb < n_kb; kb += KBU) {
          ws::mbar_wait(&x_empty[s], ph);
          ws::mbar_expect_tx(&x_full[s], C::X_ST);
#pragma unroll
          for (int k = 0; k < KBU; ++k)
            ws::tma_2d(xs + s * C::X_ST + k * C::X_KB, &xmap, (kb + k) * 64, mt * BN, &x_full[s]);
          if (++s == C::NX) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    int sa = 0, sx = 0, seg = 0;
    uint32_t ph_a = 0, ph_x = 0;
    const uint32_t xs_base = smem_u32(xs);
    for (int tile = blockIdx.x; tile < n_tiles; tile += G, ++seg) {
      const int grp = tile % n_grp;
      const int nt = min(TILES, n_rt - grp * TILES);
      const int ab = seg % NACC;
      ws::mbar_wait(&acc_empty[ab], ((seg / NACC) & 1) ^ 1);
      ws::tc_after();
      const uint32_t d = tmem + ab * (TILES * BN);
      for (int kb = 0; kb < n_kb; kb += KBU) {
        ws::mbar_wait(&a_full[sa], ph_a);
        ws::mbar_wait(&x_full[sx], ph_x);
        ws::tc_after();
        if (ws::elect_one()) {
          const uint32_t at = a_base + sa * C::A_COLS;
#pragma unroll
          for (int k = 0; k < KBU; ++k) {
            const uint64_t db0 = ws::sw128_desc(xs_base + sx * C::X_ST + k * C::X_KB);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              const uint32_t acc = (kb > 0 || k > 0 || kk > 0) ? 1u : 0u;
              const uint64_t db = db0 + (uint64_t)((kk * 32) >> 4);
#pragma unroll
              for (int t = 0; t < TILES; ++t)
                if (t < nt) mma_f16_ts(d + t * BN, at + k * 32 + t * 32 + kk * 8, db, C::IDESC, acc);
            }
          }
          ws::mma_commit(&a_empty[sa]);
          ws::mma_commit(&x_empty[sx]);
        }
        __syncwarp();
        if (++sa == C::NA) { sa = 0; ph_a ^= 1; }
        if (++sx == C::NX) { sx = 0; ph_x ^= 1; }
      }
      if (ws::elect_one()) ws::mma_commit(&acc_full[ab]);
      __syncwarp();
    }
  } else if (warp < 10) {
    // ---------------- unpack + scale into TMEM ----------------
    // TILES = 2: warp -> (tile (w-2)/4, lane quarter w%4), both 32-code halves of a row;
    // TILES = 1: warp -> (half (w-2)/4, lane quarter w%4), one 32-code half.
    const int g = (warp - 2) >> 2, q = warp & 3;
    const int r = q * 32 + lane;
    const int t = TILES == 2 ? g : 0;
    int s = 0, sa = 0;
    uint32_t ph_r = 0, ph_a = 1;
    for (int tile = blockIdx.x; tile < n_tiles; tile += G) {
      for (int kb = 0; kb < n_kb; kb += KBU) {
        ws::mbar_wait(&raw_full[s], ph_r);
        const uint32_t lane_off = (uint32_t)(q * 32) << 16;
        if (KBU > 1) {   // TILES == 1: all KBU blocks of the unit, one hand-off round
          uint4 cw[KBU];
          __half2 s2k[KBU];
#pragma unroll
          for (int k = 0; k < KBU; ++k) {
            const uint8_t* rs = raw + s * C::RAW + k * C::RAW_T;
            cw[k] = *reinterpret_cast<const uint4*>(rs + (g * 128 + r) * 16);
            s2k[k] = __half2half2(*reinterpret_cast<const __half*>(rs + 4096 + r * 2));
          }
          __syncwarp();
          if (lane == 0) ws::mbar_arrive(&raw_empty[s]);
          ws::mbar_wait(&a_empty[sa], ph_a);
          ws::tc_after();
#pragma unroll
          for (int k = 0; k < KBU; ++k) {
            uint32_t o[16];
            const uint32_t w[4] = {cw[k].x, cw[k].y, cw[k].z, cw[k].w};
#pragma unroll
            for (int ch = 0; ch < 4; ++ch) dequant8(w[ch], s2k[k], reinterpret_cast<__half2*>(o + ch * 4));
            tmem_st16(a_base + sa * C::A_COLS + k * 32 + g * 16 + lane_off, o);
          }
          asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
          ws::tc_before();
          __syncwarp();
          if (lane == 0) ws::mbar_arrive(&a_full[sa]);
          if (++s == C::NR) { s = 0; ph_r ^= 1; }
          if (++sa == C::NA) { sa = 0; ph_a ^= 1; }
          continue;
        }
        const uint8_t* rs = raw + s * C::RAW + t * C::RAW_T;
        uint4 cw0, cw1;
        if (TILES == 2) {
          cw0 = *reinterpret_cast<const uint4*>(rs + r * 16);
          cw1 = *reinterpret_cast<const uint4*>(rs + (128 + r) * 16);
        } else {
          cw0 = *reinterpret_cast<const uint4*>(rs + (g * 128 + r) * 16);
        }
        const __half2 s2 = __half2half2(*reinterpret_cast<const __half*>(rs + 4096 + r * 2));
        __syncwarp();
        if (lane == 0) ws::mbar_arrive(&raw_empty[s]);
        ws::mbar_wait(&a_empty[sa], ph_a);
        ws::tc_after();
        if (TILES == 2) {
          uint32_t o[32];
          const uint32_t w[8] = {cw0.x, cw0.y, cw0.z, cw0.w, cw1.x, cw1.y, cw1.z, cw1.w};
#pragma unroll
          for (int ch = 0; ch < 8; ++ch) dequant8(w[ch], s2, reinterpret_cast<__half2*>(o + ch * 4));
          tmem_st32(a_base + sa * C::A_COLS + t * 32 + lane_off, o);
        } else {
          uint32_t o[16];
          const uint32_t w[4] = {cw0.x, cw0.y, cw0.z, cw0.w};
#pragma unroll
          for (int ch = 0; ch < 4; ++ch) dequant8(w[ch], s2, reinterpret_cast<__half2*>(o + ch * 4));
          tmem_st16(a_base + sa * C::A_COLS + g * 16 + lane_off, o);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
        ws::tc_before();
        __syncwarp();
        if (lane == 0) ws::mbar_arrive(&a_full[sa]);
        if (++s == C::NR) { s = 0; ph_r ^= 1; }
        if (++sa == C::NA) { sa = 0; ph_a ^= 1; }
      }
    }
  } else if (warp < C::XW) {
    // ---------------- epilogue ----------------
    const int quarter = warp & 3, part = (warp - 10) >> 2;
    constexpr int PARTS = EPW / 4;
    const int row = quarter * 32 + lane;
    int seg = 0;
    for (int tile = blockIdx.x; tile < n_tiles; tile += G, ++seg) {
      const int grp = tile % n_grp, mt = tile / n_grp;
      const int nt = min(TILES, n_rt - grp * TILES);
      const int ab = seg % NACC;
      {
        uint32_t done = 0;
        const uint32_t addr = smem_u32(&acc_full[ab]), par = (seg / NACC) & 1;
        while (true) {
          asm volatile(
              "{\n.reg .pred P1;\nmbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\nselp.u32 %0, 1, 0, P1;\n}\n"
              : "=r"(done)
              : "r"(addr), "r"(par)
              : "memory");
          if (done) break;
          __nanosleep(64);
        }
      }
      ws::tc_after();
      const int m0 = mt * BN;
      for (int tt = 0; tt < nt; ++tt) {
        const uint32_t t_row = tmem + ab * (TILES * BN) + tt * BN + ((uint32_t)(quarter * 32) << 16);
        const int n = (grp * TILES + tt) * 128 + row;
        for (int c0 = part * 16; c0 < BN; c0 += 16 * PARTS) {
          if (m0 + c0 >= a.M) break;
          float v[16];
          ws::tmem_ld16(t_row + c0, v);
          epi_store16(a.epi, m0 + c0, n, v);
        }
      }
      ws::tc_before();
      __syncwarp();
      if (lane == 0) ws::mbar_arrive(&acc_empty[ab]);
    }
  }
  __syncwarp();
  ws::tc_before();
  __syncthreads();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512u));
}

template <int BN, int TILES, int NACC, int EPW, int KBU = 1>
static int run_tp(const LinearArgs& a, cudaStream_t st) {
  using C = TpCfg<BN, TILES, NACC, EPW, KBU>;
  if ((a.K / 64) % KBU) return -1;
  ensure_max_smem(gemm_tp_kernel<BN, TILES, NACC, EPW, KBU>, C::SMEM);
  const int n_rt = (a.N + 127) / 128, m_tiles = (a.M + BN - 1) / BN;
  const int64_t n_tiles = (int64_t)((n_rt + TILES - 1) / TILES) * m_tiles;
  if (n_tiles >= (1ll << 31)) return -1;
  const int G = (int)std::min<int64_t>(a.num_sms, n_tiles);
  CUtensorMap map;
  if (!make_xmap(&map, a.x, a.M, a.K, BN)) return -1;
  launch_pdl(gemm_tp_kernel<BN, TILES, NACC, EPW, KBU>, dim3(G), dim3(C::THREADS), C::SMEM, st, map, a, n_rt, m_tiles);
  return 1;
}

int launch_linear_tp(const LinearArgs& a, cudaStream_t st) {
  if (a.wfmt != 1) return -1;
  // measured at the OPT prefill shapes (tools/tpbench.py, profiles/r01/prefill_nacc2, twelve
  // tile configurations): 224-token tiles with two accumulators (the epilogue of one tile
  // overlaps the next tile's MMAs) win except for the long-K down-projection (K >= 4N:
  // fewer, longer tiles, where 256-token tiles with one accumulator are 4 % faster)
  return a.K >= 4 * a.N ? run_tp<256, 1, 1, 8>(a, st) : run_tp<224, 1, 2, 8>(a, st);
}

int launch_linear_ws(const LinearArgs& a, cudaStream_t st) {
  if (a.wfmt != 1) return -1;
  if (a.M <= 16) return run_ws<16>(a, st);
  if (a.M <= 32) return run_ws<32>(a, st);
  if (a.M <= 64) return run_ws<64>(a, st);
  if (a.M <= 128) return run_ws<128>(a, st);
  return -1;   // M > 128: the prefill shapes use the tcgen05 tile kernel (k_gemm_tc.cu)
}

}  // namespace pipo
