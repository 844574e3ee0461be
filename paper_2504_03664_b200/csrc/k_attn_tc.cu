// k_attn_tc.cu — causal prefill attention (a14's attention, PAPER.md:130 / §3.1.1: the
// layer's MHA over the cache it just wrote) on the 5th-generation tensor cores.
//
// A persistent kernel, one CTA per SM (it owns all 512 TMEM columns).  Work item = 128
// queries (a q-tile) of one (sequence, head); items are taken round-robin (item_of: the
// q-tiles of a head adjacent, for L2 reuse of its K/V, rotated for balance).  For an item whose causal key range is L <= 512 positions:
//   S = Q K^T    tcgen05.mma (M = 128 queries, N = 128 keys per block, K = head dim),
//                A = Q and B = K from shared memory (TMA, SWIZZLE_128B), fp32 S in TMEM
//                columns [0, L);
//   softmax      4 warps, thread = query row (= TMEM lane): pass 1 reads its S row for
//                the max over the causal keys, pass 2 re-reads it, p = 2^((s - max) log2e)
//                rounded to fp16, row sum in fp32, and writes P (fp16 pairs) back IN
//                PLACE into TMEM columns [0, L/2) — chunk c's 16 P columns land on S
//                columns already consumed — so the whole row's softmax is exact (no
//                online rescaling);
//   O = P V      tcgen05.mma with A = P from TMEM and B = V from shared memory
//                (MN-major: V is [keys][head dim]), fp32 O in TMEM columns [256, 256+hd);
//   epilogue     the same 4 warps: O row / sum -> fp16 -> o[b][t][h*hd ...].
// The producer warp streams Q (2 buffers), K and V (2-block rings) by TMA ahead of the
// math, across items; the phases of one item are serial (S, P and O share TMEM).
// Longer key ranges (L > 512: the c7 latency-table prompts) use the mma.sync kernel.
// q is pre-scaled by hd^-0.5 in the QKV epilogue (modeling_opt.py:151), so scores are
// plain dot products; the KV cache is position-major [pos][kv_b][dkv] (Q18), GQA maps
// query head h to KV head h / group.
#include <cuda.h>
#include <float.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "kernels.h"
#include "launch.cuh"
#include "tcgen05.cuh"

namespace pipo {
namespace atc {

using namespace ptx;

constexpr float kLog2eA = 1.4426950408889634f;

template <int HD>
struct Cfg {
  static constexpr int QT = 128;                       // queries per item (MMA M)
  static constexpr int KB = 128;                       // keys per block (MMA N of S, K of PV)
  static constexpr int MAXL = 512;                     // S columns in TMEM
  static constexpr int BOX = 128 * 128;                // one TMA box: 128 rows x 64 halves (128 B)
  static constexpr int NHALF = HD / 64;                // boxes per 128-row tile
  static constexpr int TILE = NHALF * BOX;             // 128 rows x HD halves
  static constexpr int NQ = 1, NK = 2, NV = 2;
  static constexpr int SMEM = 1024 + (NQ + NK + NV + 1) * TILE + 1024 + 4096;   // + O staging tile, barriers, exchange
  static constexpr int O_COL = 256;                    // O accumulator columns [256, 256 + HD)
  static constexpr int SW = 8;                          // softmax warps: 2 per TMEM lane quarter (key halves)
  static constexpr int EW0 = 2 + SW;                   // first of 4 epilogue warps
  static constexpr int THREADS = (EW0 + 4) * 32;       // 0 producer, 1 MMA, 2..9 softmax, 10..13 epilogue
  // kind::f16, fp32 D, K-major A and B, N = 128 keys, M = 128
  static constexpr uint32_t IDESC_S = (1u << 4) | ((uint32_t)(KB >> 3) << 17) | ((uint32_t)(QT >> 4) << 24);
  // O += P V: A (P) from TMEM, B (V) MN-major (bit 16), N = HD
  static constexpr uint32_t IDESC_O = (1u << 4) | (1u << 16) | ((uint32_t)(HD >> 3) << 17) | ((uint32_t)(QT >> 4) << 24);
  static_assert(SMEM <= 227 * 1024, "shared memory budget");
  static_assert(O_COL + HD <= 512 && MAXL / 2 <= O_COL, "TMEM plan");
};

__device__ __forceinline__ void tma_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
      "r"(a), "l"(db), "r"(idesc), "r"(acc));
}
// MN-major SWIZZLE_128B operand: 64-element (128 B) rows along MN, 8-row groups along K
// 1024 B apart (SBO), MN atoms (the two 64-wide halves of the head dim) `lbo` bytes apart
__device__ __forceinline__ uint64_t sw128_mn_desc(uint32_t saddr, uint32_t lbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)(1024 >> 4) << 32) | ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
// the same without the wait: two loads in flight per tcgen05.wait::ld
__device__ __forceinline__ void tmem_ld32_nw(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }
// 2^x for two fp16 values at once (MUFU.EX2 on f16x2: half the SFU work of two fp32 ex2)
__device__ __forceinline__ uint32_t ex2_h2(uint32_t x) {
  uint32_t y;
  asm("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n" ::"r"(
          taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}
__device__ __forceinline__ void named_bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

struct Item {
  int bi, head, qt;
};
__device__ __forceinline__ Item item_of(int it, int b, int H, int n_qt) {
  // the q-tiles of one (sequence, head) are adjacent items, so the CTAs running them at
  // the same time share that head's K/V blocks in L2; the q-tile index is rotated by the
  // head index so that every CTA (items it, it + grid, ...) gets a mix of short and long
  // causal key ranges
  Item r;
  const int bh = it / n_qt;
  r.qt = (it - bh * n_qt + bh) % n_qt;
  r.bi = bh / H;
  r.head = bh - r.bi * H;
  return r;
}

}  // namespace atc

template <int HD>
__global__ void __launch_bounds__(atc::Cfg<HD>::THREADS, 1)
    attn_prefill_tc_kernel(const __grid_constant__ CUtensorMap qmap, const __grid_constant__ CUtensorMap kmap,
                           const __grid_constant__ CUtensorMap vmap, const __grid_constant__ CUtensorMap omap,
                           AttnArgs a, int n_items, uint64_t* dbgc) {
  using C = atc::Cfg<HD>;
  using namespace atc;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base_u32 = (smem_u32(smem_raw) + 1023u) & ~1023u;
  uint8_t* base = smem_raw + (base_u32 - smem_u32(smem_raw));
  uint8_t* sq = base;
  uint8_t* sk = sq + C::NQ * C::TILE;
  uint8_t* sv = sk + C::NK * C::TILE;
  uint8_t* so = sv + C::NV * C::TILE;     // O staging tile (SWIZZLE_128B boxes) for the TMA store
  uint64_t* bar = reinterpret_cast<uint64_t*>(so + C::TILE);
  uint64_t* q_full = bar;
  uint64_t* q_empty = q_full + C::NQ;
  uint64_t* k_full = q_empty + C::NQ;
  uint64_t* k_empty = k_full + C::NK;
  uint64_t* v_full = k_empty + C::NK;
  uint64_t* v_empty = v_full + C::NV;
  uint64_t* s_full = v_empty + C::NV;     // [2] MMA -> softmax: S block in TMEM buffer b complete
  uint64_t* p_full = s_full + 2;          // [2] softmax -> MMA: P block written (count 128)
  uint64_t* pv_done = p_full + 2;         // MMA -> softmax: a non-last P.V block of an item retired
  uint64_t* o_full = pv_done + 1;         // MMA -> epilogue: the item's last P.V retired (O complete)
  uint64_t* o_empty = o_full + 1;         // epilogue -> MMA: O read out, the next item may overwrite it (128)
  uint64_t* l_full = o_empty + 1;         // [2] softmax -> epilogue: row sums of the item written (256)
  uint64_t* l_empty = l_full + 2;         // [2] epilogue -> softmax: row sums read (128)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(l_empty + 2);
  float* xch = reinterpret_cast<float*>(base + (C::NQ + C::NK + C::NV + 1) * C::TILE + 1024);   // [2 parity][2 half][128 rows]

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int H = a.n_heads, b = a.b, n = a.n, past = a.past;
  const int n_qt = (n + C::QT - 1) / C::QT;
  if (tid == 0) {
    for (int i = 0; i < C::NQ; ++i) { mbar_init(&q_full[i], 1); mbar_init(&q_empty[i], 1); }
    for (int i = 0; i < C::NK; ++i) { mbar_init(&k_full[i], 1); mbar_init(&k_empty[i], 1); }
    for (int i = 0; i < C::NV; ++i) { mbar_init(&v_full[i], 1); mbar_init(&v_empty[i], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&s_full[i], 1); mbar_init(&p_full[i], C::SW * 32); }
    mbar_init(pv_done, 1);
    mbar_init(o_full, 1);
    mbar_init(o_empty, 128);
    for (int i = 0; i < 2; ++i) { mbar_init(&l_full[i], C::SW * 32); mbar_init(&l_empty[i], 128); }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&qmap) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&kmap) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&vmap) : "memory");
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();

  // number of 128-key blocks of an item: keys 0 .. past + min(t0 + 128, n) - 1
  auto clk = [] { uint64_t t; asm volatile("mov.u64 %0, %%clock64;" : "=l"(t)); return t; };
  uint64_t* dc = dbgc ? dbgc + blockIdx.x * 8 : nullptr;   // debug: phase cycle counters
  auto n_kblocks = [&](int qt) {
    const int L = past + min((qt + 1) * C::QT, n);
    return (L + C::KB - 1) / C::KB;
  };

  if (warp == 0) {
    // ---------------- producer: Q (per item), K and V blocks (rings) ----------------
    if (lane == 0) {
      int kq = 0, kk = 0, kv = 0;   // running counters over all items of this CTA
      for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
        const Item w = item_of(it, b, H, n_qt);
        const int kvh = w.head / a.group;
        const int nkb = n_kblocks(w.qt);
        {
          const int s = kq % C::NQ;
          mbar_wait(&q_empty[s], ((kq / C::NQ) & 1) ^ 1);
          mbar_expect_tx(&q_full[s], C::TILE);
#pragma unroll
          for (int hh = 0; hh < C::NHALF; ++hh)
            tma_2d(sq + s * C::TILE + hh * C::BOX, &qmap, w.head * HD + hh * 64, w.bi * n + w.qt * C::QT, &q_full[s]);
          ++kq;
        }
        // K and V blocks in the MMA warp's consumption order: K_0, K_1, V_0, K_2, V_1, ...
        auto load_v = [&](int j) {
          const int s = kv % C::NV;
          mbar_wait(&v_empty[s], ((kv / C::NV) & 1) ^ 1);
          mbar_expect_tx(&v_full[s], C::TILE);
#pragma unroll
          for (int hh = 0; hh < C::NHALF; ++hh)
            tma_3d(sv + s * C::TILE + hh * C::BOX, &vmap, kvh * HD + hh * 64, j * C::KB, w.bi, &v_full[s]);
          ++kv;
        };
        for (int j = 0; j < nkb; ++j, ++kk) {
          const int s = kk % C::NK;
          mbar_wait(&k_empty[s], ((kk / C::NK) & 1) ^ 1);
          mbar_expect_tx(&k_full[s], C::TILE);
#pragma unroll
          for (int hh = 0; hh < C::NHALF; ++hh)
            tma_3d(sk + s * C::TILE + hh * C::BOX, &kmap, kvh * HD + hh * 64, j * C::KB, w.bi, &k_full[s]);
          if (j > 0) load_v(j - 1);
        }
        load_v(nkb - 1);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    // per item: S_0, S_1, PV_0, S_2, PV_1, ... — S_j (into TMEM buffer j % 2) is issued
    // before waiting for P_{j-1}, so the tensor core computes the next scores while the
    // softmax warps work; tcgen05 ops of one thread execute in order, so S_{j+2} never
    // overwrites P_j before PV_j has read it.
    int kq = 0, kk = 0, kv = 0, ni = 0;
    uint32_t gs = 0, gp = 0;   // S blocks issued / P blocks consumed (global over items)
    auto issue_pv = [&](int jj, bool last) {
      const int bb = (int)(gp & 1);
      mbar_wait(&p_full[bb], (gp >> 1) & 1);
      if (jj == 0) mbar_wait(o_empty, (ni & 1) ^ 1);   // the previous item's O has been read out
      const int s = kv % C::NV;
      mbar_wait(&v_full[s], (kv / C::NV) & 1);
      tc_after();
      if (elect_one()) {
        const uint32_t vb = base_u32 + (uint32_t)(sv - base) + s * C::TILE;
#pragma unroll
        for (int k16 = 0; k16 < C::KB / 16; ++k16) {
          // keys 16*k16 .. +15 of the block: P columns bb*128 + 8*k16 (fp16 pairs), V rows 16*k16 ..
          const uint64_t db = sw128_mn_desc(vb + k16 * 16 * 128, C::BOX);
          mma_ts(tmem + C::O_COL, tmem + bb * C::KB + k16 * 8, db, C::IDESC_O, (jj > 0 || k16 > 0) ? 1u : 0u);
        }
        mma_commit(&v_empty[s]);
        mma_commit(last ? o_full : pv_done);
      }
      __syncwarp();
      ++kv;
      ++gp;
    };
    // S_j of item w into TMEM buffer gs % 2 (K_j from the ring); the item's Q is released
    // after its last S block
    auto issue_s = [&](const Item& w, int j, int nkb) {
      const int sq_s = kq % C::NQ;
      if (j == 0) {
        mbar_wait(&q_full[sq_s], (kq / C::NQ) & 1);
        tc_after();
      }
      const int s = kk % C::NK;
      mbar_wait(&k_full[s], (kk / C::NK) & 1);
      tc_after();
      const int bb = (int)(gs & 1);
      if (elect_one()) {
#pragma unroll
        for (int k16 = 0; k16 < HD / 16; ++k16) {
          const int hh = k16 / 4, kin = k16 % 4;   // 64-wide half of the head dim, 16-wide step inside it
          const uint64_t da = sw128_desc(base_u32 + sq_s * C::TILE + hh * C::BOX) + (uint64_t)(kin * 2);
          const uint64_t db = sw128_desc(base_u32 + (uint32_t)(sk - base) + s * C::TILE + hh * C::BOX) +
                              (uint64_t)(kin * 2);
          mma_ss(tmem + bb * C::KB, da, db, C::IDESC_S, k16 > 0 ? 1u : 0u);
        }
        mma_commit(&k_empty[s]);
        if (j == nkb - 1) mma_commit(&q_empty[sq_s]);
        mma_commit(&s_full[bb]);
      }
      __syncwarp();
      ++kk;
      ++gs;
      if (j == nkb - 1) ++kq;
    };
    // Order: ... S_j, PV_{j-1} ..., then the NEXT item's S_0 (into the buffer PV_{last-1}
    // has released), then this item's last PV — the softmax warps find the next scores
    // ready when they finish an item.
    if (blockIdx.x < n_items) {
      const Item w0 = item_of(blockIdx.x, b, H, n_qt);
      issue_s(w0, 0, n_kblocks(w0.qt));
    }
    for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++ni) {
      const Item w = item_of(it, b, H, n_qt);
      const int nkb = n_kblocks(w.qt);
      for (int j = 1; j < nkb; ++j) {
        issue_s(w, j, nkb);
        issue_pv(j - 1, false);
      }
      if (it + (int)gridDim.x < n_items) {
        const Item wn = item_of(it + gridDim.x, b, H, n_qt);
        issue_s(wn, 0, n_kblocks(wn.qt));
      }
      issue_pv(nkb - 1, true);
    }
  } else if (warp < C::EW0) {
    // ---------------- softmax: thread = query row (TMEM lane) x key half ----------------
    // Two warps per TMEM lane quarter split each 128-key block into halves (and O into
    // column halves); they exchange the row max per block and the row sum at the end
    // through shared memory.  Online softmax per block with a lazily updated reference
    // max m_use: P_j = 2^(s log2e - m_use) while the block max stays within 8 (log2 units)
    // of m_use (P <= 256 fits fp16), otherwise O and l are rescaled by 2^(m_use - m_new)
    // first (after the previous block's P.V retired).  Each S element is read once.
    const int qtr = warp & 3;              // TMEM lane quarter this warp may access
    const int half = (warp - 2) >> 2;      // key half of each block / column half of O
    const int r = qtr * 32 + lane;
    const uint32_t lane_off = (uint32_t)(qtr * 32) << 16;
    const int pair_bar = 2 + qtr;          // named barrier of the two warps of this quarter
    constexpr int KH = C::KB / 2;          // keys per warp per block
    constexpr int OH = HD / 2;             // O columns per warp
    int ni = 0;
    uint32_t gs = 0, gpv = 0;              // S blocks consumed, P.V completions consumed (global)
    for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++ni) {
      const Item w = item_of(it, b, H, n_qt);
      const int nkb = n_kblocks(w.qt);
      const int t = w.qt * C::QT + r;                      // query index in the sequence
      const int kend = past + min(t, n - 1) + 1;           // keys 0 .. kend-1 are visible
      float m_use = 0.f, l = 0.f;
      uint64_t c0 = dc ? clk() : 0, c1 = c0, c2 = c0;
      for (int j = 0; j < nkb; ++j) {
        const int bb = (int)(gs & 1);
        mbar_wait_sleep(&s_full[bb], (gs >> 1) & 1);
        tc_after();
        if (j == 0 && dc) c1 = clk();
        uint32_t v[KH];
        tmem_ld32_nw(tmem + bb * C::KB + half * KH + lane_off, v);
        tmem_ld32_nw(tmem + bb * C::KB + half * KH + 32 + lane_off, v + 32);
        tmem_wait_ld();
        const int kb0 = j * C::KB + half * KH;
        float pm = -FLT_MAX;
        if (kb0 + KH <= kend) {
#pragma unroll
          for (int i = 0; i < KH; ++i) pm = fmaxf(pm, __uint_as_float(v[i]));
        } else {
#pragma unroll
          for (int i = 0; i < KH; ++i) {
            const bool vis = kb0 + i < kend;
            v[i] = vis ? v[i] : __float_as_uint(-INFINITY);
            pm = fmaxf(pm, vis ? __uint_as_float(v[i]) : -FLT_MAX);
          }
        }
        // the partner's half-block max (double-buffered by block parity); after this
        // barrier both warps have their S halves in registers, so P may overwrite S
        float* xb = xch + (gs & 1) * 256;
        xb[half * 128 + r] = pm;
        named_bar_sync(pair_bar, 64);
        const float bm = fmaxf(xb[r], xb[128 + r]) * kLog2eA;   // log2 units
        if (j == 0) {
          m_use = bm;
        } else {
          // P.V of the previous block must have retired before P_j lands and before any O rescale
          mbar_wait(pv_done, gpv & 1);
          ++gpv;
          tc_after();
          // tcgen05.ld/st are warp-collective: the whole warp rescales when any of its rows
          // needs it (alpha = 1 for the others); the partner warp holds the same rows, so it
          // takes the same branch
          const bool need = bm > m_use + 8.f;
          if (__any_sync(0xffffffffu, need)) {
            const float alpha = need ? ex2(m_use - bm) : 1.f;
            l *= alpha;
#pragma unroll 1
            for (int c = 0; c < OH / 32; ++c) {
              uint32_t o[32];
              const uint32_t oa = tmem + C::O_COL + half * OH + c * 32 + lane_off;
              tmem_ld32_nw(oa, o);
              tmem_wait_ld();
#pragma unroll
              for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
              asm volatile(
                  "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                  "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};\n" ::"r"(oa),
                  "r"(o[0]), "r"(o[1]), "r"(o[2]), "r"(o[3]), "r"(o[4]), "r"(o[5]), "r"(o[6]), "r"(o[7]), "r"(o[8]),
                  "r"(o[9]), "r"(o[10]), "r"(o[11]), "r"(o[12]), "r"(o[13]), "r"(o[14]), "r"(o[15]), "r"(o[16]),
                  "r"(o[17]), "r"(o[18]), "r"(o[19]), "r"(o[20]), "r"(o[21]), "r"(o[22]), "r"(o[23]), "r"(o[24]),
                  "r"(o[25]), "r"(o[26]), "r"(o[27]), "r"(o[28]), "r"(o[29]), "r"(o[30]), "r"(o[31])
                  : "memory");
            }
            if (need) m_use = bm;
          }
        }
        // P in fp16: exponents rounded to fp16 and evaluated on f16x2 (near the max, where
        // p matters, the fp16 exponent is exact to 2^-11); masked keys are 2^-inf = 0
        uint32_t pk[KH / 2];
#pragma unroll
        for (int i = 0; i < KH / 2; ++i) {
          const __half2 xh = __floats2half2_rn(fmaf(__uint_as_float(v[2 * i]), kLog2eA, -m_use),
                                               fmaf(__uint_as_float(v[2 * i + 1]), kLog2eA, -m_use));
          pk[i] = ex2_h2(*reinterpret_cast<const uint32_t*>(&xh));
          const float2 pf = __half22float2(*reinterpret_cast<const __half2*>(&pk[i]));
          l += pf.x + pf.y;   // the sum of the fp16 P the MMA multiplies
        }
        tmem_st16(tmem + bb * C::KB + half * (KH / 2) + lane_off, pk);
        tmem_st16(tmem + bb * C::KB + half * (KH / 2) + 16 + lane_off, pk + 16);
        asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
        tc_before();
        mbar_arrive(&p_full[bb]);
        ++gs;
      }
      if (dc) c2 = clk();
      // hand the row sums of both key halves to the epilogue warps (double-buffered by item)
      {
        const int lb = ni & 1;
        mbar_wait(&l_empty[lb], ((ni >> 1) & 1) ^ 1);
        xch[512 + lb * 256 + half * 128 + r] = l;
        mbar_arrive(&l_full[lb]);
      }
      uint64_t c4 = c2;
      if (dc && tid == 64) {
        dc[0] += c1 - c0; dc[1] += c2 - c1; dc[2] += 0; dc[3] += c4 - c2; dc[4] += clk() - c4; dc[5] += 1;
      }
    }
  }
  if (warp >= C::EW0) {
    // ---------------- epilogue warps: O / l -> fp16 -> TMA store ----------------
    // Separate from the softmax warps, so the next item's softmax overlaps this item's
    // output (O is single-buffered: the next item's first P.V waits for o_empty).
    const int qtr = warp & 3;
    const int r = qtr * 32 + lane;
    const uint32_t lane_off = (uint32_t)(qtr * 32) << 16;
    const int etid = tid - C::EW0 * 32;
    int ni = 0;
    for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++ni) {
      const Item w = item_of(it, b, H, n_qt);
      const int lb = ni & 1;
      mbar_wait_sleep(&l_full[lb], (ni >> 1) & 1);
      const float inv = 1.f / (xch[512 + lb * 256 + r] + xch[512 + lb * 256 + 128 + r]);   // fixed order
      mbar_arrive(&l_empty[lb]);
      mbar_wait_sleep(o_full, ni & 1);
      tc_after();
      uint32_t ob[HD / 2];
#pragma unroll
      for (int c = 0; c < HD / 32; ++c) {
        uint32_t va[32];
        tmem_ld32_nw(tmem + C::O_COL + c * 32 + lane_off, va);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const __half2 h = __floats2half2_rn(__uint_as_float(va[2 * i]) * inv, __uint_as_float(va[2 * i + 1]) * inv);
          ob[c * 16 + i] = *reinterpret_cast<const uint32_t*>(&h);
        }
      }
      tc_before();
      mbar_arrive(o_empty);
      // stage the 128 x HD fp16 tile in the SWIZZLE_128B box layout, TMA store (rows past
      // the sequence end are clipped by the map)
      if (etid == 0) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");   // staging tile free
      named_bar_sync(1, 128);
#pragma unroll
      for (int i = 0; i < HD / 8; ++i) {
        const int hh = i / 8, c = i % 8;
        *reinterpret_cast<uint4*>(so + hh * C::BOX + r * 128 + ((c ^ (r & 7)) << 4)) =
            make_uint4(ob[4 * i], ob[4 * i + 1], ob[4 * i + 2], ob[4 * i + 3]);
      }
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      named_bar_sync(1, 128);
      if (etid == 0) {
#pragma unroll
        for (int hh = 0; hh < C::NHALF; ++hh)
          asm volatile(
              "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];\n" ::"l"(&omap),
              "r"(w.head * HD + hh * 64), "r"(w.qt * C::QT), "r"(w.bi), "r"(smem_u32(so + hh * C::BOX))
              : "memory");
        asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
      }
    }
    if (etid == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
  }
  __syncwarp();
  tc_before();
  __syncthreads();
  tc_after();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

// ---------------------------------------------------------------------------------
typedef CUresult (*PFN_encodeTiled_a)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                      const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                      CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled_a encode_a() {
  static PFN_encodeTiled_a fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess)
      fn = (PFN_encodeTiled_a)p;
    cudaGetLastError();
  });
  return fn;
}

template <int HD>
static int run_prefill_tc(const AttnArgs& a, cudaStream_t st) {
  using C = atc::Cfg<HD>;
  PFN_encodeTiled_a enc = encode_a();
  if (!enc) return -1;
  const int dkv = a.dkv ? a.dkv : a.d;
  const int L = a.past + a.n;
  CUtensorMap qm, km, vm;
  {
    const cuuint64_t dims[2] = {(cuuint64_t)a.d, (cuuint64_t)a.b * a.n};
    const cuuint64_t strides[1] = {(cuuint64_t)a.d * 2};
    const cuuint32_t box[2] = {64, 128};
    const cuuint32_t es[2] = {1, 1};
    if (enc(&qm, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<__half*>(a.q), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return -1;
  }
  for (int w = 0; w < 2; ++w) {
    // K / V as 3-D {dkv, position, sequence} over the position-major cache [pos][kv_b][dkv]
    // (default strides) or the int4-KV path's fp16 staging rows [b][n][K | V] (explicit
    // strides); positions >= past + n are out of bounds and read as zeros
    const int64_t ps = a.kv_pos_stride ? a.kv_pos_stride : (int64_t)a.kv_b * dkv;
    const int64_t bs = a.kv_b_stride ? a.kv_b_stride : (int64_t)dkv;
    const cuuint64_t dims[3] = {(cuuint64_t)dkv, (cuuint64_t)L, (cuuint64_t)a.kv_b};
    const cuuint64_t strides[2] = {(cuuint64_t)ps * 2, (cuuint64_t)bs * 2};
    const cuuint32_t box[3] = {64, 128, 1};
    const cuuint32_t es[3] = {1, 1, 1};
    if (enc(w == 0 ? &km : &vm, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, const_cast<__half*>(w == 0 ? a.kc : a.vc), dims,
            strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return -1;
  }
  CUtensorMap om;
  {
    // output [b][n][d] as 3-D {d, n, b}: a tile's rows past the sequence end are out of bounds
    const cuuint64_t dims[3] = {(cuuint64_t)a.d, (cuuint64_t)a.n, (cuuint64_t)a.b};
    const cuuint64_t strides[2] = {(cuuint64_t)a.d * 2, (cuuint64_t)a.n * a.d * 2};
    const cuuint32_t box[3] = {64, 128, 1};
    const cuuint32_t es[3] = {1, 1, 1};
    if (enc(&om, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, a.o, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
        CUDA_SUCCESS)
      return -1;
  }
  const int n_qt = (a.n + C::QT - 1) / C::QT;
  const int n_items = a.b * a.n_heads * n_qt;
  const int grid = std::min(n_items, a.num_sms);
  ensure_max_smem(attn_prefill_tc_kernel<HD>, C::SMEM);
  static const bool dbg = getenv("PIPO_WS_DEBUG") && (atoi(getenv("PIPO_WS_DEBUG")) & 128);
  uint64_t* dbgc = dbg ? reinterpret_cast<uint64_t*>(a.ws + (15ll << 20)) : nullptr;
  if (dbgc) cudaMemsetAsync(dbgc, 0, 148 * 8 * 8, st);
  if (launch_pdl_k(attn_prefill_tc_kernel<HD>, dim3(grid), dim3(C::THREADS), C::SMEM, st, qm, km, vm, om, a, n_items, dbgc) !=
      cudaSuccess)
    return -1;
  return 1;
}

// The tensor-core prefill attention where it applies (returns -1 otherwise, and the
// caller runs the mma.sync kernel): causal key range <= 512, fp16 K/V (cache or staging rows).
int launch_attention_prefill_tc(const AttnArgs& a, cudaStream_t st) {
  const int hd = a.d / a.n_heads;
  if ((hd != 64 && hd != 128) || a.past + a.n > atc::Cfg<128>::MAXL) return -1;
  if ((a.dkv ? a.dkv : a.d) % 64 || a.d % 64) return -1;
  return hd == 64 ? run_prefill_tc<64>(a, st) : run_prefill_tc<128>(a, st);
}

}  // namespace pipo
