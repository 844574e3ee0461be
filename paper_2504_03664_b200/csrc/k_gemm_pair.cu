// k_gemm_pair.cu — the decode linears (a6 QKV, a8 out-proj, a10 FC1, a11 FC2 of SURVEY.md
// §8(a); M = b <= 64 tokens) as a fused int4-g64 unpack + tcgen05 GEMM on SM PAIRS
// (cta_group::2), with the stream-K fixup inside the kernel.
//
// Why pairs (measured on B200, profiles/r02/ubench/): at N = 64 tokens one
// tcgen05.mma.cta_group::1 128x64x16 with A in TMEM costs 40 cycles, a cta_group::2
// 256x64x16 costs 33 cycles for BOTH SMs (N = 32: 29 -> 17, N = 16: 27 -> 16), and each
// SM then reads only its half of the activation tile B from shared memory.  At M = 64 the
// MMA pipe is ~80 % busy at HBM speed with cta_group::1 — the pair is what leaves room to
// overlap it with the unpack arithmetic (4-bit weights are unpacked
// next to the matrix unit, the fp16 weights never exist in HBM).
//
// Work: a "quad" = 4 weight row-tiles of 128 rows.  CTA rank r of a pair holds row-tiles
// 4q + r (slot 0) and 4q + 2 + r (slot 1) of quad q; one pipeline unit = one quad x one
// 64-wide k-block (one int4 group): per CTA 2 x 4352 B of raw int4 blocks + its half of
// the x tile (BN/2 tokens x 64 k, TMA, SWIZZLE_128B).  The (quad, k-block) units are split
// into equal contiguous ranges over the G pairs (stream-K: every SM streams the same
// number of weight bytes).
//
// Roles per CTA:
//   warp 0      producer: waits a free ring slot, bulk-copies RU consecutive raw blocks of
//               each of its 2 row-tiles (one 17-KB request per tile: the TMA unit's
//               per-request cost makes 4-KB requests top out at 5.3 TB/s);
//   warp 14     x loader: this CTA's x half of each unit through the LSU (cp.async, 16 B per
//               lane, SWIZZLE_128B pattern) into its own ring — x is ~half as many bytes as
//               the weights, and through the TMA unit it would cap the weight stream at
//               ~3.5 TB/s (the limit of the cta_group::1 kernel, k_gemm_ws.cu);
//   warp 1      (leader CTA only) MMA issuer: 2 x 4 tcgen05.mma.cta_group::2 (256 x BN x 16)
//               per unit, A from TMEM, B from both CTAs' shared memory; commits multicast
//               to both CTAs release the A stage and the ring slot;
//   warps 2..   unpack: warp (slot j, lane quarter) turns its row's 64 codes into
//               fp16_rne(q * s) (the K8 arithmetic, common.cuh dequant8) and tcgen05.st's
//               them into the A stage, then arrives on the LEADER's a_full barrier;
//   last 4      epilogue: tcgen05.ld of the CTA's accumulator rows, then one of
//                 full tile     -> fused epilogue (bias / residual / ReLU / QKV scatter)
//                 contributor   -> partial to the workspace + release flag (its range starts
//                                  inside the tile: always the pair's FIRST segment, done
//                                  early)
//                 finisher      -> the pair owning the tile's first k-block, whose LAST
//                                  segment this is: waits the contributors' flags, adds
//                                  their partials in k order (deterministic), fused
//                                  epilogue.  No second kernel, no fixup launch latency.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>
#include <map>
#include <mutex>

#include "common.cuh"
#include "epilogue.cuh"
#include "kernels.h"
#include "launch.cuh"
#include "layout.h"
#include "tcgen05.cuh"

namespace pipo {
namespace pair {

using namespace ptx;

__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_id_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
// address of the same shared-memory object in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
// Arrive on a barrier of the leader CTA.  Relaxed: no generic-memory data travels with
// these hand-offs (the unpack -> MMA data is in TMEM, ordered by tcgen05.wait::st +
// tcgen05.fence::before_thread_sync here and fence::after_thread_sync at the MMA issuer).
// A .release.cluster arrive costs a MEMBAR.ALL.GPU per arrival (ncu: the top stall of
// the first version of this kernel).
__device__ __forceinline__ void arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(cluster_addr) : "memory");
}
// wait on a barrier that receives the peer CTA's (relaxed) arrivals.  (A large
// suspend-time hint on these waits was measured slower.)
__device__ __forceinline__ void wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.relaxed.cluster.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_wait_s(uint64_t* bar, uint32_t parity) { mbar_wait(bar, parity); }
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mma2(uint32_t d, uint32_t a, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
      "r"(a), "l"(db), "r"(idesc), "r"(acc));
}
// arrive (when the MMAs issued so far complete) on the barrier at this smem offset in
// BOTH CTAs of the pair
__device__ __forceinline__ void commit2(uint64_t* bar) {
  asm volatile(
      "{\n.reg .b16 m;\nmov.b16 m, 3;\n"
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n}\n" ::"r"(
          smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void st32(uint32_t taddr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};\n" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
      "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
      "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory"); }

// stream-K partition of U units over G pairs (U * G < 2^32: checked by the launcher)
__device__ __forceinline__ int64_t u_begin(int64_t c, int64_t U, int64_t G) {
  return (int64_t)((uint32_t)c * (uint32_t)U / (uint32_t)G);
}

}  // namespace pair

template <int BN>
struct PairCfg {
  static constexpr int X_BYTES = BN * 64;                       // this CTA's BN/2 tokens x 64 k (128 B rows)
  static constexpr int RU = 4;                                  // units (k-blocks) per raw ring slot
  static constexpr int RAW_T = RU * (int)kInt4BlockBytes;       // one row-tile's blocks: one bulk copy
  static constexpr int STAGE = 2 * RAW_T;                       // raw ring slot (2 row-tiles)
  static constexpr int NX = 8;                                  // x ring stages (one unit each)
  static constexpr int XD = 3;                                  // x units in flight (cp.async groups)
  static constexpr int NR = (200 * 1024 - NX * X_BYTES) / STAGE > 12 ? 12 : (200 * 1024 - NX * X_BYTES) / STAGE;
  static constexpr int NACC = 2;
  static constexpr int ACC_COLS = NACC * 2 * BN;                // NACC x 2 slots x BN fp32 columns
  static constexpr int A_COLS = 64;                             // 2 slots x 32 columns (64 fp16 of k)
  static constexpr int NA = (512 - ACC_COLS) / A_COLS > 6 ? 6 : (512 - ACC_COLS) / A_COLS;
  static constexpr int UW = 8;                                  // unpack warps per group (slot x lane quarter)
  static constexpr int UG = 2;                                  // unit-interleaved unpack groups
  // Warp roles: 0 raw producer, 1 MMA issuer, 2 .. 2+UG*UW-1 unpack, 4 epilogue, x loader.
  // (Giving the single-thread roles the highest warp ids — the SMSP arbiter's priority
  // order — was measured slower.)
  static constexpr int PW = 0, MW = 1;
  static constexpr int U0 = 2;                                  // first unpack warp
  static constexpr int E0 = U0 + UG * UW;                       // first epilogue warp
  static constexpr int XW = E0 + 4;                             // x loader
  static constexpr int THREADS = (XW + 1) * 32;
  static constexpr int EW = UG * UW + 4;                        // warps draining the last segment
  static constexpr int SMEM = 1024 + NX * X_BYTES + NR * STAGE + 1024;
  // kind::f16, fp32 D, fp16 A/B, K-major, N = BN, M = 256
  static constexpr uint32_t IDESC = (1u << 4) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
  static_assert(BN == 16 || BN == 32 || BN == 64, "tokens per pair tile");
  static_assert(SMEM <= 227 * 1024, "shared memory budget");
  static_assert(NA >= 2 && NR >= 3, "TMEM budget / ring depth");
  static_assert(XD < NX, "x ring");
  static_assert((2 * NR + 2 * NX + 2 * NA + 2 * NACC) * 8 + 16 <= 1024, "barrier area");
};

template <int BN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(PairCfg<BN>::THREADS, 1)
    gemm_pair_kernel(LinearArgs a, int n_rt, int G, uint32_t* flags, uint64_t* stamps) {
  using C = PairCfg<BN>;
  using namespace pair;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base_u32 = (smem_u32(smem_raw) + 1023u) & ~1023u;
  uint8_t* base = smem_raw + (base_u32 - smem_u32(smem_raw));
  uint8_t* xring = base;                                   // NX x X_BYTES (1024-aligned stages)
  uint8_t* rring = base + C::NX * C::X_BYTES;               // NR x STAGE
  uint64_t* bar = reinterpret_cast<uint64_t*>(rring + C::NR * C::STAGE);
  uint64_t* slot_full = bar;
  uint64_t* slot_empty = slot_full + C::NR;
  uint64_t* x_full = slot_empty + C::NR;
  uint64_t* x_empty = x_full + C::NX;
  uint64_t* a_full = x_empty + C::NX;        // leader: 2 CTAs x UW unpack warps
  uint64_t* a_empty = a_full + C::NA;
  uint64_t* acc_full = a_empty + C::NA;
  uint64_t* acc_empty = acc_full + C::NACC;  // leader: 2 CTAs x 4 epilogue warps
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + C::NACC);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = cta_rank();
  const int pr = (int)cluster_id_x();
  const int n_kb = a.K / 64;
  const int n_quads = (n_rt + 3) >> 2;
  const int64_t U = (int64_t)n_quads * n_kb;
  const int64_t u0 = u_begin(pr, U, G), u1 = u_begin(pr + 1, U, G);
  // debug-only globaltimer stamps (stamps != nullptr: PIPO_WS_DEBUG bit 128)
  uint64_t* ts = stamps ? stamps + blockIdx.x * 16 : nullptr;
  auto stamp = [&](int k) {
    if (ts) {
      uint64_t t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      ts[k] = t;
    }
  };
  if (tid == 0) stamp(0);
  uint64_t* wc = stamps ? stamps + 148 * 16 + blockIdx.x * 16 : nullptr;   // wait-cycle counters
  auto clk = [] { uint64_t t; asm volatile("mov.u64 %0, %%clock64;" : "=l"(t)); return t; };

  if (tid == 0) {
    for (int i = 0; i < C::NR; ++i) { mbar_init(&slot_full[i], 1); mbar_init(&slot_empty[i], 1); }
    for (int i = 0; i < C::NX; ++i) { mbar_init(&x_full[i], 1); mbar_init(&x_empty[i], 1); }
    for (int i = 0; i < C::NA; ++i) { mbar_init(&a_full[i], 2 * C::UW); mbar_init(&a_empty[i], 1); }
    for (int i = 0; i < C::NACC; ++i) { mbar_init(&acc_full[i], 1); mbar_init(&acc_empty[i], 8); }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == C::MW) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                 "r"(512u));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
  }
  tc_before();
  cluster_sync();            // barriers of both CTAs initialised, TMEM allocated in both
  tc_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();                // predecessor (producer of x / reader of our outputs) has finished
  pdl_trigger();
  const uint32_t a_base = tmem + C::ACC_COLS;
  if (tid == 0) { stamp(1); if (ts) ts[10] = (uint64_t)(u1 - u0); }

  if (warp == C::PW) {
    // ---------------- producer: raw int4 blocks, RU k-blocks of both row-tiles per slot ----------------
    if (lane == 0) {
      int q = (int)(u0 / n_kb), kb = (int)(u0 - (int64_t)q * n_kb);
      const int64_t tile_stride = (int64_t)n_kb * kInt4BlockBytes;
      const int64_t nu = u1 - u0;
      uint64_t w0 = 0, tb = clk();
      for (int64_t ir = 0; ir * C::RU < nu; ++ir) {   // ring slot ir holds units RU*ir .. RU*ir+RU-1
        const int s = (int)(ir % C::NR);
        const uint64_t t0 = wc ? clk() : 0;
        mbar_wait_s(&slot_empty[s], (uint32_t)(((ir / C::NR) & 1) ^ 1));
        if (wc) w0 += clk() - t0;
        const int cnt = (int)(nu - ir * C::RU < C::RU ? nu - ir * C::RU : C::RU);
        // runs of consecutive k-blocks inside one quad are contiguous per row-tile: one
        // bulk copy per (run, row-tile); a quad boundary inside the slot splits the run
        uint32_t bytes = 0;
        {
          int qq = q, kk = kb;
          for (int e = 0; e < cnt; ++e) {
            bytes += (4 * qq + (int)rank < n_rt ? (uint32_t)kInt4BlockBytes : 0u) +
                     (4 * qq + 2 + (int)rank < n_rt ? (uint32_t)kInt4BlockBytes : 0u);
            if (++kk == n_kb) { kk = 0; ++qq; }
          }
        }
        mbar_expect_tx(&slot_full[s], bytes);
        uint8_t* st = rring + s * C::STAGE;
        int e = 0;
        while (e < cnt) {
          const int run = min(cnt - e, n_kb - kb);
#pragma unroll
          for (int jj = 0; jj < 2; ++jj) {
            const int rt = 4 * q + 2 * jj + (int)rank;
            if (rt < n_rt)
              bulk_g2s(st + jj * C::RAW_T + e * kInt4BlockBytes, a.w + rt * tile_stride + (int64_t)kb * kInt4BlockBytes,
                       (uint32_t)(run * kInt4BlockBytes), &slot_full[s]);
          }
          e += run;
          kb += run;
          if (kb == n_kb) { kb = 0; ++q; }
        }
      }
      stamp(2);
      if (wc) { wc[0] = w0; wc[1] = clk() - tb; }
    }
  } else if (warp == C::XW) {
    // ---------------- x loader: this CTA's BN/2 tokens of each unit's k-block (LSU) ----------------
    // 16-B cp.async per lane into the SWIZZLE_128B layout the MMA descriptor expects (chunk c
    // of row r at r * 128 + ((c ^ (r & 7)) * 16)); rows >= M are zero-filled.  XD units stay
    // in flight; a unit is signalled after cp.async.wait_group + a generic -> async proxy fence.
    const int64_t nu = u1 - u0;
    int kb = (int)(u0 % n_kb);
    constexpr int CHUNKS = (BN / 2) * 8;
    auto signal = [&](int64_t iu) {
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&x_full[iu % C::NX]);
    };
    uint64_t w9 = 0, w10 = 0, tb = clk();
    for (int64_t iu = 0; iu < nu; ++iu) {
      const int sx = (int)(iu % C::NX);
      uint64_t t0 = wc ? clk() : 0;
      mbar_wait_s(&x_empty[sx], (uint32_t)(((iu / C::NX) & 1) ^ 1));
      if (wc) w9 += clk() - t0;
      uint8_t* dst = xring + sx * C::X_BYTES;
#pragma unroll
      for (int c = lane; c < CHUNKS; c += 32) {
        const int r = c >> 3, ch = c & 7;
        const int tok = (int)rank * (BN / 2) + r;
        const bool ok = tok < a.M;
        const __half* src = a.x + (ok ? (int64_t)tok * a.K + kb * 64 + ch * 8 : 0);
        cp_async16(dst + r * 128 + ((ch ^ (r & 7)) << 4), src, ok ? 16 : 0);
      }
      cp_async_commit();
      if (iu >= C::XD) {
        t0 = wc ? clk() : 0;
        cp_async_wait<C::XD>();
        if (wc) w10 += clk() - t0;
        signal(iu - C::XD);
      }
      if (++kb == n_kb) kb = 0;
    }
    cp_async_wait<0>();
    for (int64_t iu = nu > C::XD ? nu - C::XD : 0; iu < nu; ++iu) signal(iu);
    if (wc && lane == 0) { wc[9] = w9; wc[10] = w10; wc[11] = clk() - tb; }
  } else if (warp == C::MW) {
    // ---------------- MMA issuer (leader CTA) ----------------
    if (rank == 0) {
      int seg = 0;
      int64_t u = u0;
      uint64_t w2 = 0, w3 = 0, tb = clk();
      while (u < u1) {
        const int64_t q = u / n_kb;
        const int64_t seg_end = min(u1, (q + 1) * n_kb);
        const int ab = seg % C::NACC;
        uint64_t t0 = wc ? clk() : 0;
        wait_cluster(&acc_empty[ab], (uint32_t)(((seg / C::NACC) & 1) ^ 1));
        if (wc) w3 += clk() - t0;
        tc_after();
        const uint32_t d = tmem + ab * (2 * BN);
        for (int64_t v = u; v < seg_end; ++v) {
          const int64_t iu = v - u0;
          const int sa = (int)(iu % C::NA), s = (int)((iu / C::RU) % C::NR), e = (int)(iu % C::RU);
          const int sx = (int)(iu % C::NX);
          t0 = wc ? clk() : 0;
          wait_cluster(&a_full[sa], (uint32_t)((iu / C::NA) & 1));
          if (wc) w2 += clk() - t0;
          tc_after();
          if (elect_one()) {
            const uint64_t db = sw128_desc(base_u32 + sx * C::X_BYTES);
            const uint32_t at = a_base + sa * C::A_COLS;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              const uint32_t acc = (v > u || kk > 0) ? 1u : 0u;
              mma2(d, at + kk * 8, db + (uint64_t)(kk * 2), C::IDESC, acc);
              mma2(d + BN, at + 32 + kk * 8, db + (uint64_t)(kk * 2), C::IDESC, acc);
            }
            commit2(&a_empty[sa]);
            commit2(&x_empty[sx]);
            if (e == C::RU - 1 || iu + 1 == u1 - u0) commit2(&slot_empty[s]);
          }
          __syncwarp();
        }
        if (elect_one()) commit2(&acc_full[ab]);
        __syncwarp();
        u = seg_end;
        ++seg;
      }
      if (lane == 0) stamp(3);
      if (wc && lane == 0) { wc[2] = w2; wc[3] = w3; wc[4] = clk() - tb; }
    }
  } else if (warp < C::E0) {
    // ---------------- unpack + scale into this CTA's A stage ----------------
    // The dequant arithmetic (8 FMA-pipe ops per 8 weights, the K8 rounding) needs ~330
    // cycles of one SMSP's FMA pipe per unit against ~375 cycles of HBM time: UG groups of
    // UW warps take the units round-robin (group g: units g, g + UG, ...) so that 4 warps per
    // SMSP hide each other's shared-memory, TMEM-store and barrier latencies.
    const int g = (warp - C::U0) / C::UW;
    const int j = ((warp - C::U0) >> 2) & 1, qt = warp & 3;   // slot, TMEM lane quarter (warp % 4)
    const int r = qt * 32 + lane;                          // weight row within the tile
    const uint32_t lane_off = (uint32_t)(qt * 32) << 16;
    const uint32_t a_full_leader = mapa(&a_full[0], 0);
    const int64_t nu = u1 - u0;
    int q = (int)((u0 + g) / n_kb), kb = (int)((u0 + g) - (int64_t)q * n_kb);
    // software-pipelined: the group's next unit's codes are loaded while this unit's TMEM
    // stores drain
    uint4 c0 = make_uint4(0, 0, 0, 0), c1 = c0;
    __half2 s2 = __half2half2(__ushort_as_half(0));
    bool have = false;
    uint64_t w5 = 0, w6 = 0, w7 = 0, w12 = 0, tb = clk();
    auto load = [&](int64_t iu, int qq) {
      const int64_t ir = iu / C::RU;
      const int s = (int)(ir % C::NR), e = (int)(iu % C::RU);
      const uint64_t t0 = wc ? clk() : 0;
      mbar_wait_s(&slot_full[s], (uint32_t)((ir / C::NR) & 1));
      if (wc) w5 += clk() - t0;
      have = 4 * qq + 2 * j + (int)rank < n_rt;
      if (have) {
        const uint8_t* rs = rring + s * C::STAGE + j * C::RAW_T + e * kInt4BlockBytes;
        c0 = *reinterpret_cast<const uint4*>(rs + r * 16);
        c1 = *reinterpret_cast<const uint4*>(rs + (128 + r) * 16);
        s2 = __half2half2(*reinterpret_cast<const __half*>(rs + 4096 + r * 2));
      }
    };
    if (g < nu) load(g, q);
    if (warp == C::U0 && lane == 0) stamp(9);
    for (int64_t iu = g; iu < nu; iu += C::UG) {
      const int sa = (int)(iu % C::NA);
      uint64_t t0 = wc ? clk() : 0;
      mbar_wait_s(&a_empty[sa], (uint32_t)(((iu / C::NA) & 1) ^ 1));
      if (wc) w6 += clk() - t0;
      tc_after();
      if (have) {
        uint32_t o[32];
        const uint32_t w[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
#pragma unroll
        for (int ch = 0; ch < 8; ++ch) dequant8(w[ch], s2, reinterpret_cast<__half2*>(o + ch * 4));
        st32(a_base + sa * C::A_COLS + j * 32 + lane_off, o);
      }
      kb += C::UG;
      while (kb >= n_kb) { kb -= n_kb; ++q; }
      if (iu + C::UG < nu) load(iu + C::UG, q);   // registers are free once the stores are issued
      t0 = wc ? clk() : 0;
      asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
      if (wc) w7 += clk() - t0;
      // this CTA's x half of the unit must have landed before the leader may issue: one
      // warp per group gates its a_full arrival on it
      if (((warp - C::U0) & 7) == 0) {
        t0 = wc ? clk() : 0;
        mbar_wait_s(&x_full[iu % C::NX], (uint32_t)((iu / C::NX) & 1));
        if (wc) w12 += clk() - t0;
      }
      tc_before();
      __syncwarp();
      if (lane == 0) arrive_remote(a_full_leader + sa * 8);
    }
    if (warp == C::U0 && lane == 0) stamp(4);
    if (wc && warp == C::U0 && lane == 0) { wc[5] = w5; wc[6] = w6; wc[7] = w7; wc[8] = clk() - tb; wc[12] = w12; }
  }
  // ---------------- epilogue ----------------
  // Segments (maximal runs of this pair's units inside one quad) before the last are
  // drained by the 4 epilogue warps while the mainloop runs; the LAST segment — the one
  // on the kernel's critical path, and the finisher's fixup — is drained by all 12
  // unpack + epilogue warps together (EW / 4 per TMEM lane quarter), each chunk of 16
  // accumulator columns loading its contributors' partials two at a time.
  if (warp >= C::U0 && warp < C::XW && u0 < u1) {
    const int qt = warp & 3, row = qt * 32 + lane;
    const uint32_t lane_off = (uint32_t)(qt * 32) << 16;
    const int64_t slot_floats = (int64_t)BN * 128;
    constexpr int CH = 2 * (BN / 16);               // 16-column chunks per segment (2 slots)
    float* my_part = a.ws + (int64_t)(pr * 2 + (int)rank) * 2 * slot_floats;
    auto do_chunk = [&](int ab, int q, int ch, bool contributor, int c_last) {
      const int jj = ch / (BN / 16), c0 = (ch % (BN / 16)) * 16;
      const int rt = 4 * q + 2 * jj + (int)rank;
      if (rt >= n_rt) return;
      float v[16];
      tmem_ld16(tmem + ab * (2 * BN) + jj * BN + c0 + lane_off, v);
      if (contributor) {
        float* p = my_part + jj * slot_floats + (int64_t)c0 * 128 + row;
#pragma unroll
        for (int i = 0; i < 16; ++i) __stcg(p + i * 128, v[i]);
        return;
      }
      for (int cc = pr + 1; cc <= c_last; ++cc) {   // k order: own, pr+1, pr+2, ...
        const float* pa = a.ws + (int64_t)(cc * 2 + (int)rank) * 2 * slot_floats + jj * slot_floats +
                          (int64_t)c0 * 128 + row;
        float xa[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) xa[i] = __ldcg(pa + i * 128);
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] += xa[i];
      }
      epi_store16(a.epi, c0, rt * 128 + row, v);
    };
    const int q_first = (int)(u0 / n_kb), q_last = (int)((u1 - 1) / n_kb);
    if (warp >= C::E0) {
      const uint32_t acc_empty_leader = mapa(&acc_empty[0], 0);
      for (int q = q_first; q < q_last; ++q) {          // every segment but the last
        const int seg = q - q_first, ab = seg % C::NACC;
        const bool contributor = u0 > (int64_t)q * n_kb;   // only the first segment can be
        mbar_wait_sleep(&acc_full[ab], (uint32_t)((seg / C::NACC) & 1));
        tc_after();
        for (int ch = 0; ch < CH; ++ch) do_chunk(ab, q, ch, contributor, pr);
        tc_before();
        __syncwarp();
        if (lane == 0) arrive_remote(acc_empty_leader + ab * 8);
        if (contributor) {
          __threadfence();
          named_bar(2, 128);
          if (tid == C::E0 * 32) st_release(flags + pr * 2 + rank, 1u);
        }
        if (tid == C::E0 * 32) stamp(12);
      }
    }
    {   // the last segment, all EW unpack + epilogue warps
      const int q = q_last, seg = q_last - q_first, ab = seg % C::NACC;
      const int64_t qs = (int64_t)q * n_kb, qe = qs + n_kb;
      const bool contributor = u0 > qs;
      const bool finisher = !contributor && u1 < qe;
      int c_last = pr;
      if (finisher)
        while (c_last + 1 < G && u_begin(c_last + 1, U, G) < qe) ++c_last;
      mbar_wait_sleep(&acc_full[ab], (uint32_t)((seg / C::NACC) & 1));
      tc_after();
      if (tid == C::U0 * 32) { stamp(5); if (ts) ts[11] = contributor ? 1 : finisher ? 2 : 0; }
      if (finisher) {
        if (tid == C::U0 * 32)
          for (int cc = pr + 1; cc <= c_last; ++cc)
            while (ld_acquire(flags + cc * 2 + rank) == 0) __nanosleep(32);
        named_bar(1, C::EW * 32);
        if (tid == C::U0 * 32) stamp(6);
      }
      for (int ch = (warp - C::U0) >> 2; ch < CH; ch += C::EW / 4) do_chunk(ab, q, ch, contributor, c_last);
      if (tid == C::U0 * 32) stamp(7);
      if (contributor) {
        __threadfence();
        named_bar(1, C::EW * 32);
        if (tid == C::U0 * 32) st_release(flags + pr * 2 + rank, 1u);
      } else if (finisher) {
        named_bar(1, C::EW * 32);   // every partial read before the flags are re-armed
        if (tid == C::U0 * 32)
          for (int cc = pr + 1; cc <= c_last; ++cc) flags[cc * 2 + rank] = 0u;
      }
    }
  }
  __syncwarp();
  tc_before();
  cluster_sync();   // all remote arrivals delivered, all MMAs of both CTAs retired
  tc_after();
  if (tid == 0) stamp(8);
  if (warp == C::MW) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512u));
}

// ---------------------------------------------------------------------------------
// largest number of co-resident pairs (clusters of 2) of the kernel on the current device:
// the in-kernel fixup spins on flags of other pairs, so every pair must be resident
template <int BN>
static int max_pairs() {
  static std::mutex mu;
  static std::map<int, int> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> g(mu);
  auto it = cache.find(dev);
  if (it != cache.end()) return it->second;
  using C = PairCfg<BN>;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2);
  cfg.blockDim = dim3(C::THREADS);
  cfg.dynamicSmemBytes = C::SMEM;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, gemm_pair_kernel<BN>, &cfg) != cudaSuccess) n = 0;
  cudaGetLastError();
  cache[dev] = n;
  return n;
}

template <int BN>
static int run_pair(const LinearArgs& a, cudaStream_t st) {
  using C = PairCfg<BN>;
  ensure_max_smem(gemm_pair_kernel<BN>, C::SMEM);
  const int n_rt = (a.N + 127) / 128, n_kb = a.K / 64;
  const int64_t U = (int64_t)((n_rt + 3) / 4) * n_kb;
  const int mp = max_pairs<BN>();
  if (mp <= 0 || a.M > BN) return -1;
  // >= 16 units (>= 139 KB of weights per SM) per pair: the prologue stays amortised
  const int G = (int)std::max<int64_t>(1, std::min<int64_t>(std::min(mp, a.num_sms / 2), U / 16));
  if ((int64_t)G * 2 * 2 * BN * 128 > a.ws_floats || U * G >= (1ll << 32) || a.n_counters < 1024) return -1;
  // fixup flags: the top 512 split-K counters (zero at rest, self-resetting)
  uint32_t* flags = reinterpret_cast<uint32_t*>(a.counters + a.n_counters - 512);
  static const bool dbg_stamps = getenv("PIPO_WS_DEBUG") && (atoi(getenv("PIPO_WS_DEBUG")) & 128);
  uint64_t* stamps = dbg_stamps ? reinterpret_cast<uint64_t*>(a.ws + (15ll << 20)) : nullptr;
  if (launch_pdl_k(gemm_pair_kernel<BN>, dim3(2 * G), dim3(C::THREADS), C::SMEM, st, a, n_rt, G, flags, stamps) !=
      cudaSuccess)
    return -1;
  return 1;
}

int launch_linear_pair(const LinearArgs& a, cudaStream_t st) {
  if (a.wfmt != 1 || a.M <= 0) return -1;
  if (a.M <= 16) return run_pair<16>(a, st);
  if (a.M <= 32) return run_pair<32>(a, st);
  if (a.M <= 64) return run_pair<64>(a, st);
  return -1;
}

}  // namespace pipo
