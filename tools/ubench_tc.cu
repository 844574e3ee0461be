// ubench_tc.cu — microbenchmarks of the tcgen05 building blocks of the decode GEMM
// (commit cost/latency, A-in-TMEM MMA rate at N = 64, tcgen05.st + wait::st, mbarrier
// hand-off, and the unpack <-> MMA core loop without HBM traffic).  Standalone:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2504_03664_b200/csrc \
//        tools/ubench_tc.cu -o tools/ubench_tc.bin -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>

#include "tcgen05.cuh"

using namespace pipo;
using namespace pipo::ptx;

__device__ __forceinline__ uint64_t clk() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
      "r"(a), "l"(db), "r"(idesc), "r"(acc));
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
__device__ __forceinline__ uint32_t idesc_f16(int M, int N) {
  return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// out[blockIdx.x * 16 + k]
__global__ void __launch_bounds__(640, 1) ub_kernel(int test, int n, int p0, int p1, uint64_t* out, int p2) {
  extern __shared__ uint8_t sm_raw[];
  const uint32_t b32 = (smem_u32(sm_raw) + 1023u) & ~1023u;
  uint8_t* base = sm_raw + (b32 - smem_u32(sm_raw));
  uint64_t* bar = reinterpret_cast<uint64_t*>(base + 200 * 1024 - 1024);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 64);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint64_t* o = out + blockIdx.x * 16;
  if (tid == 0) {
    for (int i = 0; i < 32; ++i) mbar_init(&bar[i], 1);
    for (int i = 32; i < 48; ++i) mbar_init(&bar[i], 8);   // unpack -> MMA (8 warps)
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) tmem_alloc(slot, 512);
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tmem = *slot;
  const uint64_t db0 = sw128_desc(b32);   // B (x) tile at the smem base, 64 rows x 128 B per k-block

  if (test == 0 && warp == 1) {   // commit issue cost (no MMA in flight)
    if (elect_one()) {
      uint64_t t0 = clk();
      for (int i = 0; i < n; ++i) mma_commit(&bar[i & 1]);
      uint64_t t1 = clk();
      o[0] = (t1 - t0) / n;
    }
    __syncwarp();
  } else if (test == 1 && warp == 1) {   // commit -> mbarrier round trip (no MMA)
    if (elect_one()) {
      uint64_t t0 = clk();
      for (int i = 0; i < n; ++i) { mma_commit(&bar[0]); mbar_wait(&bar[0], i & 1); }
      o[0] = (clk() - t0) / n;
    }
    __syncwarp();
  } else if (test == 2 && warp == 1) {   // MMA rate: n MMAs of 128 x p0 x 16, A in TMEM (p1=0) or SMEM (p1=1)
    if (elect_one()) {
      const uint32_t id = idesc_f16(128, p0);
      // warm
      mma_ts(tmem, tmem + 256, db0, id, 0);
      mma_commit(&bar[0]);
      mbar_wait(&bar[0], 0);
      uint64_t t0 = clk();
      for (int i = 0; i < n; ++i) {
        const uint64_t db = db0 + (uint64_t)(((i & 3) * 32) >> 4);
        if (p1 == 0) mma_ts(tmem + ((i >> 2) & 1) * 64, tmem + 256 + (i & 7) * 8, db, id, 1);
        else mma_f16_ss(tmem + ((i >> 2) & 1) * 64, sw128_desc(b32 + 65536) + (uint64_t)(((i & 3) * 32) >> 4), db, id, 1);
      }
      uint64_t t1 = clk();
      mma_commit(&bar[0]);
      mbar_wait(&bar[0], 1);
      uint64_t t2 = clk();
      o[0] = (t1 - t0) / n;   // issue
      o[1] = (t2 - t0) / n;   // completion
      o[2] = t2 - t0;
    }
    __syncwarp();
  } else if (test == 9 && warp == 1) {   // MMA rate, 128 x p0 x 16 A in TMEM, p1 accumulators round-robin
    if (elect_one()) {
      const uint32_t id = idesc_f16(128, p0);
      mma_ts(tmem, tmem + 256, db0, id, 0);
      mma_commit(&bar[0]);
      mbar_wait(&bar[0], 0);
      uint64_t t0 = clk();
      for (int i = 0; i < n; ++i) {
        const uint64_t db = db0 + (uint64_t)(((i & 3) * 32) >> 4);
        mma_ts(tmem + (i % p1) * 64, tmem + 256 + (i & 7) * 8, db, id, 1);
      }
      mma_commit(&bar[0]);
      mbar_wait(&bar[0], 1);
      o[1] = (clk() - t0) / n;   // completion
    }
    __syncwarp();
  } else if (test == 3 && warp == 1) {   // groups of p1 MMAs + commit + wait (serial latency per group)
    if (elect_one()) {
      const uint32_t id = idesc_f16(128, p0);
      uint64_t t0 = clk();
      for (int g = 0; g < n; ++g) {
        for (int i = 0; i < p1; ++i)
          mma_ts(tmem + ((i >> 2) & 1) * 64, tmem + 256 + (i & 7) * 8, db0 + (uint64_t)(((i & 3) * 32) >> 4), id, 1);
        mma_commit(&bar[0]);
        mbar_wait(&bar[0], g & 1);
      }
      o[0] = (clk() - t0) / n;
    }
    __syncwarp();
  } else if (test == 4 && warp >= 4 && warp < 8) {   // STTM x32 (p0 per round) + wait::st, 4 warps
    const uint32_t lo = (uint32_t)((warp & 3) * 32) << 16;
    uint32_t v[32];
    for (int i = 0; i < 32; ++i) v[i] = lane * 32 + i;
    uint64_t t0 = clk();
    for (int r = 0; r < n; ++r) {
      for (int j = 0; j < p0; ++j) st32(tmem + 128 + ((j * 32) & 255) + lo, v);
      asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
    }
    if (lane == 0) o[warp - 4] = (clk() - t0) / n;
  } else if (test == 5 && (warp == 2 || warp == 3)) {   // mbarrier ping-pong between two warps
    uint64_t t0 = clk();
    for (int i = 0; i < n; ++i) {
      if (warp == 2) {
        if (lane == 0) mbar_arrive(&bar[0]);
        mbar_wait(&bar[1], i & 1);
      } else {
        mbar_wait(&bar[0], i & 1);
        if (lane == 0) mbar_arrive(&bar[1]);
      }
    }
    if (warp == 2 && lane == 0) o[0] = (clk() - t0) / n;
  } else if (test == 6) {
    // core loop: 8 unpack warps (2 tiles x 4 quarters) dequantize 2 k-blocks into an A stage
    // (tcgen05.st), MMA warp issues 16 MMAs (2 tiles x 2 kb x 4) per unit, commit frees the
    // stage.  p0 = A stages (acc 128 cols + p0 x 128), p1 bit0: skip dequant math, bit1: skip
    // STTM, bit2: skip MMA.
    const int NA = p0;
    uint64_t* a_full = &bar[32];   // count 8
    uint64_t* a_empty = &bar[0];   // count 1 (commit)
    if (warp == 1) {
      const uint32_t id = idesc_f16(128, 64);
      uint64_t t0 = clk();
      for (int u = 0; u < n; ++u) {
        const int s = u % NA;
        mbar_wait(&a_full[s], (u / NA) & 1);
        tc_after();
        if (elect_one()) {
          const uint32_t at = tmem + 128 + s * 128;
          if (!(p1 & 4))
            for (int k = 0; k < 2; ++k)
              for (int kk = 0; kk < 4; ++kk) {
                const uint64_t db = db0 + (uint64_t)((k * 8192 + kk * 32) >> 4);
                mma_ts(tmem, at + k * 64 + kk * 8, db, id, 1);
                mma_ts(tmem + 64, at + k * 64 + 32 + kk * 8, db, id, 1);
              }
          mma_commit(&a_empty[s]);
        }
        __syncwarp();
      }
      if (lane == 0) o[0] = (clk() - t0) / n;
    } else if (warp >= 2 && warp < 10) {
      const int t = (warp - 2) >> 2, q = warp & 3;
      const uint32_t lo = (uint32_t)(q * 32) << 16;
      const uint8_t* rawp = base + 32768 + (q * 32 + lane) * 16;
      const __half2 s2 = __float2half2_rn(0.01f);
      uint64_t t0 = clk();
      for (int u = 0; u < n; ++u) {
        const int s = u % NA;
        mbar_wait(&a_empty[s], ((u / NA) & 1) ^ 1);
        tc_after();
        for (int k = 0; k < 2; ++k) {
          uint32_t ov[32];
          const uint4 c0 = *reinterpret_cast<const uint4*>(rawp + k * 4352 + t * 8704);
          const uint4 c1 = *reinterpret_cast<const uint4*>(rawp + k * 4352 + t * 8704 + 2048);
          const uint32_t w[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
          if (!(p1 & 1)) {
#pragma unroll
            for (int ch = 0; ch < 8; ++ch) dequant8(w[ch] + u, s2, reinterpret_cast<__half2*>(ov + ch * 4));
          } else {
#pragma unroll
            for (int ch = 0; ch < 32; ++ch) ov[ch] = w[ch & 7] + ch;
          }
          if (!(p1 & 2)) st32(tmem + 128 + s * 128 + k * 64 + t * 32 + lo, ov);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
        tc_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&a_full[s]);
      }
      if (lane == 0 && warp == 2) o[1] = (clk() - t0) / n;
    }
  } else if (test == 7 && warp >= 2 && warp < 2 + p0) {   // pure dequant throughput, p0 warps
    const __half2 s2 = __float2half2_rn(0.01f);
    const uint8_t* rawp = base + 32768 + lane * 16;
    uint32_t acc = 0;
    uint64_t t0 = clk();
    for (int u = 0; u < n; ++u) {
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        uint32_t ov[32];
        const uint4 c0 = *reinterpret_cast<const uint4*>(rawp + k * 4352);
        const uint4 c1 = *reinterpret_cast<const uint4*>(rawp + k * 4352 + 2048);
        const uint32_t w[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
#pragma unroll
        for (int ch = 0; ch < 8; ++ch) dequant8(w[ch] ^ (uint32_t)u, s2, reinterpret_cast<__half2*>(ov + ch * 4));
        if (p1) {
          const uint32_t lo = (uint32_t)((warp & 3) * 32) << 16;
          st32(tmem + 128 + k * 64 + ((warp >> 2) & 1) * 32 + lo, ov);
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) acc ^= ov[i];
        }
      }
      if (p1) asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
    }
    if (lane == 0) o[warp - 2] = (clk() - t0) / n;
    if (acc == 0x12345678) o[15] = acc;
  } else if (test == 8) {
    // grouped core loop: p2 groups of 8 unpack warps take units round-robin; NA stages
    const int NA = p0, NG = p2;
    uint64_t* a_full = &bar[32];
    uint64_t* a_empty = &bar[0];
    if (warp == 1) {
      const uint32_t id = idesc_f16(128, 64);
      uint64_t t0 = clk();
      for (int u = 0; u < n; ++u) {
        const int s = u % NA;
        mbar_wait(&a_full[s], (u / NA) & 1);
        tc_after();
        if (elect_one()) {
          const uint32_t at = tmem + 128 + s * 128;
          if (!(p1 & 4))
            for (int k = 0; k < 2; ++k)
              for (int kk = 0; kk < 4; ++kk) {
                const uint64_t db = db0 + (uint64_t)((k * 8192 + kk * 32) >> 4);
                mma_ts(tmem, at + k * 64 + kk * 8, db, id, 1);
                mma_ts(tmem + 64, at + k * 64 + 32 + kk * 8, db, id, 1);
              }
          mma_commit(&a_empty[s]);
        }
        __syncwarp();
      }
      if (lane == 0) o[0] = (clk() - t0) / n;
    } else if (warp >= 2 && warp < 2 + 8 * NG) {
      const int g = (warp - 2) >> 3, wl = (warp - 2) & 7;
      const int t = wl >> 2, q = warp & 3;
      const uint32_t lo = (uint32_t)(q * 32) << 16;
      const uint8_t* rawp = base + 32768 + (q * 32 + lane) * 16;
      const __half2 s2 = __float2half2_rn(0.01f);
      uint64_t t0 = clk();
      for (int u = g; u < n; u += NG) {
        const int s = u % NA;
        mbar_wait(&a_empty[s], ((u / NA) & 1) ^ 1);
        tc_after();
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          uint32_t ov[32];
          const uint4 c0 = *reinterpret_cast<const uint4*>(rawp + k * 4352 + t * 8704);
          const uint4 c1 = *reinterpret_cast<const uint4*>(rawp + k * 4352 + t * 8704 + 2048);
          const uint32_t w[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
#pragma unroll
          for (int ch = 0; ch < 8; ++ch) dequant8(w[ch] ^ (uint32_t)u, s2, reinterpret_cast<__half2*>(ov + ch * 4));
          st32(tmem + 128 + s * 128 + k * 64 + t * 32 + lo, ov);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
        tc_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&a_full[s]);
      }
      if (lane == 0 && warp == 2) o[1] = (clk() - t0) / n;
    }
  }
  tc_before();
  __syncthreads();
  tc_after();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

int pair_main();
int stream_main();
int main(int argc, char** argv) {
  if (argc > 1 && argv[1][0] == 's') return stream_main();
  if (argc > 1) return pair_main();
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(ub_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  uint64_t* d;
  cudaMalloc(&d, 148 * 16 * 8);
  uint64_t h[148 * 16];
  auto run = [&](const char* name, int test, int n, int p0, int p1, int grid, int p2 = 1) {
    cudaMemset(d, 0, 148 * 16 * 8);
    ub_kernel<<<grid, 640, smem>>>(test, n, p0, p1, d, p2);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e)); exit(1); }
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("%-44s grid %3d : %6llu %6llu %8llu  (cta0)   cta%d: %6llu %6llu\n", name, grid, (unsigned long long)h[0],
           (unsigned long long)h[1], (unsigned long long)h[2], grid - 1, (unsigned long long)h[(grid - 1) * 16],
           (unsigned long long)h[(grid - 1) * 16 + 1]);
  };
  run("commit issue (cyc/commit)", 0, 256, 0, 0, 1);
  run("commit round trip, no MMA (cyc)", 1, 256, 0, 0, 1);
  for (int N : {16, 32, 64, 128, 256}) {
    char b[64];
    snprintf(b, 64, "MMA TS 128x%dx16 x256: issue/complete", N);
    run(b, 2, 256, N, 0, 1);
    snprintf(b, 64, "MMA SS 128x%dx16 x256: issue/complete", N);
    run(b, 2, 256, N, 1, 1);
  }
  run("MMA TS 128x64x16 x256, 148 CTAs", 2, 256, 64, 0, 148);
  for (int na : {1, 2, 3, 4}) {
    char b[64];
    snprintf(b, 64, "MMA TS 128x64x16 x512, %d acc round-robin", na);
    run(b, 9, 512, 64, na, 1);
  }
  for (int g : {4, 8, 16, 32}) {
    char b[64];
    snprintf(b, 64, "group of %d MMAs N64 + commit + wait (cyc)", g);
    run(b, 3, 64, 64, g, 1);
  }
  for (int j : {1, 2, 4}) {
    char b[64];
    snprintf(b, 64, "STTM x32 x%d + wait::st (cyc/round)", j);
    run(b, 4, 64, j, 0, 1);
  }
  run("mbarrier ping-pong (cyc/round trip)", 5, 256, 0, 0, 1);
  for (int w : {4, 8, 12, 16}) {
    char b[80];
    snprintf(b, 80, "pure dequant unit, %d warps (cyc/unit/warp)", w);
    run(b, 7, 64, w, 0, 1);
    snprintf(b, 80, "dequant+STTM unit, %d warps (cyc/unit/warp)", w);
    run(b, 7, 64, w, 1, 1);
  }
  for (int na : {2, 3})
    for (int ng : {1, 2})
      for (int f : {0, 4}) {
        char b[80];
        snprintf(b, 80, "grouped core NA=%d groups=%d flags=%d", na, ng, f);
        run(b, 8, 64, na, f, 1, ng);
      }
  return 0;
}

// ---------------------------------------------------------------------------------
// cta_group::2 (SM pair) MMA rate: cluster of 2 CTAs, the leader issues n MMAs of
// 256 x p0 x 16 (A from TMEM in both CTAs, B half from each CTA's shared memory).
__device__ __forceinline__ void mma_ts2(uint32_t d, uint32_t a, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
      "r"(a), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void commit2_mc(uint64_t* bar) {
  asm volatile(
      "{\n.reg .b16 m;\nmov.b16 m, 3;\n"
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n}\n" ::"r"(
          smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 1) ub_pair_kernel(int n, int N, uint64_t* out, int mode) {
  extern __shared__ uint8_t sm_raw[];
  const uint32_t b32 = (smem_u32(sm_raw) + 1023u) & ~1023u;
  uint8_t* base = sm_raw + (b32 - smem_u32(sm_raw));
  uint64_t* bar = reinterpret_cast<uint64_t*>(base + 100 * 1024);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 8);
  const int warp = threadIdx.x >> 5;
  const uint32_t rank = cluster_rank();
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(slot)), "r"(512u));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
  }
  tc_before();
  cluster_sync_all();
  tc_after();
  const uint32_t tmem = *slot;
  const uint64_t db0 = sw128_desc(b32);
  const uint32_t id = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
  if (mode == 1) {   // commit2 (no MMA) round trip, leader waits its own barrier
    if (rank == 0 && warp == 1 && elect_one()) {
      uint64_t t0 = clk();
      for (int i = 0; i < n; ++i) { commit2_mc(&bar[0]); mbar_wait(&bar[0], i & 1); }
      out[blockIdx.x * 16 + 0] = (clk() - t0) / n;
    }
    if (rank == 1 && warp == 1 && lane_id() == 0) for (int i = 0; i < n; ++i) mbar_wait(&bar[0], i & 1);
  } else if (mode == 2) {   // remote-arrive ping-pong rank0 <-> rank1 (relaxed.cluster)
    if (threadIdx.x == 0) mbar_init(&bar[1], 1);
    if (threadIdx.x == 0) asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    cluster_sync_all();
    if (warp == 2 && lane_id() == 0) {
      uint32_t peer;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(peer) : "r"(smem_u32(&bar[1])), "r"(rank ^ 1));
      uint64_t t0 = clk();
      for (int i = 0; i < n; ++i) {
        if (rank == 0) {
          asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(peer) : "memory");
          mbar_wait(&bar[1], i & 1);
        } else {
          mbar_wait(&bar[1], i & 1);
          asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(peer) : "memory");
        }
      }
      if (rank == 0) out[blockIdx.x * 16 + 0] = (clk() - t0) / n;
    }
  } else if (mode == 3) {   // groups of 8 pair MMAs (N) + commit2 + wait: latency per group
    if (rank == 0 && warp == 1 && elect_one()) {
      uint64_t t0 = clk();
      for (int g = 0; g < n; ++g) {
        for (int i = 0; i < 8; ++i)
          mma_ts2(tmem + ((i >> 2) & 1) * 64, tmem + 256 + (i & 7) * 8, db0 + (uint64_t)(((i & 3) * 32) >> 4), id, 1);
        commit2_mc(&bar[0]);
        mbar_wait(&bar[0], g & 1);
      }
      out[blockIdx.x * 16 + 0] = (clk() - t0) / n;
    }
    if (rank == 1 && warp == 1 && lane_id() == 0) for (int i = 0; i < n; ++i) mbar_wait(&bar[0], i & 1);
  } else if (rank == 0 && warp == 1) {
    if (elect_one()) {
      mma_ts2(tmem, tmem + 256, db0, id, 0);
      commit2_mc(&bar[0]);
      mbar_wait(&bar[0], 0);
      uint64_t t0 = clk();
      for (int i = 0; i < n; ++i)
        mma_ts2(tmem + ((i >> 2) & 1) * 64, tmem + 256 + (i & 7) * 8, db0 + (uint64_t)(((i & 3) * 32) >> 4), id, 1);
      uint64_t t1 = clk();
      commit2_mc(&bar[0]);
      mbar_wait(&bar[0], 1);
      uint64_t t2 = clk();
      out[blockIdx.x * 16 + 0] = (t1 - t0) / n;
      out[blockIdx.x * 16 + 1] = (t2 - t0) / n;
    }
    __syncwarp();
  } else if (mode == 0 && rank == 1 && warp == 1) {
    mbar_wait(&bar[0], 0);
    mbar_wait(&bar[0], 1);
  }
  tc_before();
  cluster_sync_all();
  tc_after();
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512u));
  }
}

int pair_main() {
  const int smem = 110 * 1024;
  cudaFuncSetAttribute(ub_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  uint64_t* d;
  cudaMalloc(&d, 148 * 16 * 8);
  uint64_t h[148 * 16];
  for (int N : {16, 32, 64, 128, 256}) {
    for (int grid : {2, 148}) {
      cudaMemset(d, 0, 148 * 16 * 8);
      ub_pair_kernel<<<grid, 256, smem>>>(256, N, d, 0);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("pair N=%d: %s\n", N, cudaGetErrorString(e)); return 1; }
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      printf("pair MMA TS 256x%dx16 x256 grid %3d: issue %llu complete %llu cyc/MMA\n", N, grid,
             (unsigned long long)h[0], (unsigned long long)h[1]);
    }
  }
  const char* nm[4] = {"", "commit2 multicast round trip (no MMA)", "remote arrive ping-pong (round trip)",
                       "8 pair MMAs N=64 + commit2 + wait"};
  for (int mode = 1; mode <= 3; ++mode) {
    cudaMemset(d, 0, 148 * 16 * 8);
    ub_pair_kernel<<<148, 256, smem>>>(256, 64, d, mode);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("mode %d: %s\n", mode, cudaGetErrorString(e)); return 1; }
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("%-44s : %llu cyc (cta0) %llu (cta146)\n", nm[mode], (unsigned long long)h[0], (unsigned long long)h[146 * 16]);
  }
  return 0;
}

// ---------------------------------------------------------------------------------
// HBM -> smem bulk streaming, one CTA per SM: plain launch vs clusters of 2, and with
// the cta_group::2 TMEM allocation done first (the pair GEMM's setup).
template <int CLUSTER, bool ALLOC2>
__global__ void __launch_bounds__(128, 1) ub_stream_kernel(const uint8_t* src, int64_t per, int chunk, int stages,
                                                          uint64_t* out) {
  extern __shared__ uint8_t sm_raw[];
  const uint32_t b32 = (smem_u32(sm_raw) + 1023u) & ~1023u;
  uint8_t* base = sm_raw + (b32 - smem_u32(sm_raw));
  uint64_t* full = reinterpret_cast<uint64_t*>(base + stages * chunk);
  uint64_t* empty = full + stages;
  uint32_t* slot = reinterpret_cast<uint32_t*>(empty + stages);
  const int tid = threadIdx.x, warp = tid >> 5;
  if (tid == 0) {
    for (int i = 0; i < stages; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (ALLOC2 && warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(slot)), "r"(512u));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
  }
  if (CLUSTER > 1) cluster_sync_all(); else __syncthreads();
  const uint8_t* p = src + (int64_t)blockIdx.x * per;
  const int n = (int)(per / chunk);
  uint64_t t0 = clk();
  if (tid == 0) {
    for (int i = 0; i < n; ++i) {
      const int s = i % stages;
      mbar_wait(&empty[s], ((i / stages) & 1) ^ 1);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(&full[s])), "r"(chunk) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                       smem_u32(base + s * chunk)), "l"(p + (int64_t)i * chunk), "r"(chunk), "r"(smem_u32(&full[s])) : "memory");
    }
  } else if (tid == 32) {
    for (int i = 0; i < n; ++i) {
      const int s = i % stages;
      mbar_wait(&full[s], (i / stages) & 1);
      mbar_arrive(&empty[s]);
    }
    out[blockIdx.x] = clk() - t0;
  }
  if (CLUSTER > 1) cluster_sync_all(); else __syncthreads();
  if (ALLOC2 && warp == 1) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(*slot), "r"(512u));
}

int stream_main() {
  const int64_t per = 3 << 20;
  uint8_t* buf;
  cudaMalloc(&buf, per * 148);
  cudaMemset(buf, 1, per * 148);
  uint64_t* d;
  cudaMalloc(&d, 148 * 8);
  auto run = [&](const char* name, auto kern, int cluster, int chunk, int stages) {
    const int smem = stages * chunk + 2048;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(148);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cluster; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = cluster > 1 ? 1 : 0;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaLaunchKernelEx(&cfg, kern, (const uint8_t*)buf, per, chunk, stages, d);
    cudaEventRecord(e0);
    for (int i = 0; i < 5; ++i) cudaLaunchKernelEx(&cfg, kern, (const uint8_t*)buf, per, chunk, stages, d);
    cudaEventRecord(e1);
    cudaError_t e = cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%-34s chunk %6d stages %2d : %s %.0f GB/s\n", name, chunk, stages, e == cudaSuccess ? "" : cudaGetErrorString(e),
           5.0 * per * 148 / (ms * 1e-3) / 1e9);
  };
  for (int chunk : {8704, 17408})
    for (int stages : {8, 12}) {
      if (chunk * stages > 210 * 1024) continue;
      run("plain", ub_stream_kernel<1, false>, 1, chunk, stages);
      run("cluster 2", ub_stream_kernel<2, false>, 2, chunk, stages);
      run("cluster 2 + tcgen05 alloc cg2", ub_stream_kernel<2, true>, 2, chunk, stages);
    }
  return 0;
}
