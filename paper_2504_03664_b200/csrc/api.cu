// api.cu — the C-ABI (include/pipo.h) and the pipeline scheduler.
//
// Algorithm 1 as a CUDA stream/event DAG instead of a thread
// pool:
//   CallLoadData(i, j)        -> enqueue_copy(): cudaMemcpyAsync of the layer's merged
//                                blob, segment by segment, on the weight-copy stream
//                                into an HBM ring slot; one event per landed segment.
//                                Prefetch runs R-1 layers ahead (performance-optimized
//                                pipeline) and across token steps.
//   PrepareInput(i, j)        -> embedding gather for j = 0; otherwise the hidden state
//                                already lives in HBM.
//   SynchronizeLoadTask(i, j) -> cudaStreamWaitEvent(compute, segment-ready) right
//                                before the first kernel that reads the segment: the
//                                GPU consumes each segment as soon as it lands; the
//                                host never blocks.
//   Compute(i, j)             -> LN1+QKV, attention, out-proj, LN2+FC1, FC2 kernels.
//   CallStoreCache(i, j)      -> (host-resident KV) D2H of the new KV positions on a
//                                save stream after attention; its completion event is
//                                waited for only by the copy stream before the SAME
//                                layer's KV load in the next step (PAPER.md:162-165,
//                                243-245).
// The ring slot of layer G is released by an event recorded after its last kernel;
// the copy stream waits on it before overwriting the slot (WAR).  Weight loads are
// gated only by ring capacity: with ring_layers = 2 the next layer loads while the
// current one computes; ring_layers = 1 is the memory-efficient
// pipeline, which serialises copy and compute.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>
#include <cstdlib>

#include "ctx.h"
#include "disk.h"
#include "nccl_rt.h"
#include "numa.h"

using namespace pipo;

namespace {

thread_local std::string g_err;

pipo_status set_err(pipo_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

pipo_status cuda_fail(pipo_ctx* c, cudaError_t e, const char* what, int line) {
  if (c) c->poisoned = true;
  char buf[512];
  snprintf(buf, sizeof buf, "CUDA error %s (%s) at api.cu:%d: %s", cudaGetErrorName(e), cudaGetErrorString(e),
           line, what);
  return set_err(PIPO_E_CUDA, buf);
}

#define CK(x)                                                 \
  do {                                                        \
    cudaError_t e_ = (x);                                     \
    if (e_ != cudaSuccess) return cuda_fail(ctx, e_, #x, __LINE__); \
  } while (0)

// account a launcher's result: n kernels launched, n < 0 = unsupported config
#define LAUNCH(expr)                                                           \
  do {                                                                         \
    int n_ = (expr);                                                           \
    if (n_ < 0) return set_err(PIPO_E_INVALID_ARG, "unsupported kernel configuration: " #expr); \
    ctx->launches += n_;                                                       \
    CK(cudaGetLastError());                                                    \
  } while (0)

#define CHECK_CTX()                                                                  \
  do {                                                                               \
    if (!ctx) return set_err(PIPO_E_INVALID_ARG, "null context");                    \
    if (ctx->poisoned) return set_err(PIPO_E_STATE, "context poisoned by an earlier CUDA error"); \
  } while (0)

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

template <typename T>
pipo_status dev_alloc(pipo_ctx* ctx, T** p, int64_t bytes) {
  if (bytes <= 0) { *p = nullptr; return PIPO_OK; }
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), (size_t)bytes);
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    return set_err(PIPO_E_OOM, "cudaMalloc of " + std::to_string(bytes) + " bytes failed");
  }
  CK(e);
  ctx->hbm_bytes += bytes;
  return PIPO_OK;
}

// numa = true: one of the big stores (weights, host KV), placed on ctx->numa_node
template <typename T>
pipo_status host_alloc(pipo_ctx* ctx, T** p, int64_t bytes, bool numa = false) {
  if (bytes <= 0) { *p = nullptr; return PIPO_OK; }
  if (numa && ctx->numa_node >= 0) {
    void* q = nullptr;
    bool bound = false;
    if (!numa_host_alloc(bytes, ctx->numa_node, &q, &bound))
      return set_err(PIPO_E_OOM, "NUMA-bound pinned allocation of " + std::to_string(bytes) + " bytes on node " +
                                     std::to_string(ctx->numa_node) + " failed");
    *p = static_cast<T*>(q);
    ctx->numa_allocs.push_back({q, bytes});
    ctx->pinned_bytes += bytes;
    return PIPO_OK;
  }
  cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(p), (size_t)bytes, cudaHostAllocDefault);
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    return set_err(PIPO_E_OOM, "cudaHostAlloc of " + std::to_string(bytes) + " bytes failed");
  }
  CK(e);
  ctx->pinned_bytes += bytes;
  return PIPO_OK;
}

#define TRY(x)                         \
  do {                                 \
    pipo_status s_ = (x);              \
    if (s_ != PIPO_OK) return s_;      \
  } while (0)

void host_free(pipo_ctx* ctx, void* p, int64_t bytes) {
  if (!p) return;
  for (size_t i = 0; i < ctx->numa_allocs.size(); ++i)
    if (ctx->numa_allocs[i].first == p) {
      numa_host_free(p, ctx->numa_allocs[i].second);
      ctx->numa_allocs.erase(ctx->numa_allocs.begin() + (long)i);
      ctx->pinned_bytes -= bytes;
      return;
    }
  cudaFreeHost(p);
  ctx->pinned_bytes -= bytes;
}

// ---- timeline ---------------------------------------------------------------
// Timing events come from a pool that is recycled only by pipeline_stats_reset; a long
// run without resets stops recording at kEventCap events (PIPO_F_TIMELINE / KPROF turn
// themselves off and pipo_stats.timeline_truncated says so) instead of growing forever.
constexpr size_t kEventCap = 1u << 18;

pipo_status ev_get(pipo_ctx* ctx, cudaEvent_t* ev) {
  if (ctx->ev_used == ctx->ev_pool.size()) {
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    ctx->ev_pool.push_back(e);
  }
  *ev = ctx->ev_pool[ctx->ev_used++];
  return PIPO_OK;
}

bool ev_capped(pipo_ctx* ctx) {
  if (ctx->ev_used + 2 <= kEventCap) return false;
  ctx->timeline = ctx->kprof = false;
  ctx->timeline_truncated = true;
  return true;
}

pipo_status span_begin(pipo_ctx* ctx, cudaStream_t st, cudaEvent_t* a) {
  *a = nullptr;
  if (!ctx->timeline || ev_capped(ctx)) return PIPO_OK;
  TRY(ev_get(ctx, a));
  CK(cudaEventRecord(*a, st));
  return PIPO_OK;
}

pipo_status span_end(pipo_ctx* ctx, cudaStream_t st, cudaEvent_t a, int lane, int64_t bytes) {
  if (!a) return PIPO_OK;
  cudaEvent_t b;
  TRY(ev_get(ctx, &b));
  CK(cudaEventRecord(b, st));
  ctx->spans.push_back(Span{a, b, lane, bytes});
  return PIPO_OK;
}

pipo_status kbegin(pipo_ctx* ctx, cudaEvent_t* a) {
  *a = nullptr;
  if (!ctx->kprof || ev_capped(ctx)) return PIPO_OK;
  TRY(ev_get(ctx, a));
  CK(cudaEventRecord(*a, ctx->s_comp));
  return PIPO_OK;
}

pipo_status kend(pipo_ctx* ctx, cudaEvent_t a, int cls, double bytes, double flops) {
  if (!a) return PIPO_OK;
  cudaEvent_t b;
  TRY(ev_get(ctx, &b));
  CK(cudaEventRecord(b, ctx->s_comp));
  ctx->krecs.push_back(KRec{a, b, cls, bytes, flops});
  return PIPO_OK;
}

// algorithmic bytes of one linear layer (weights + x + output traffic)
double linear_bytes(const LinearArgs& la) {
  const double nk = (double)la.N * la.K;
  const double w = la.wfmt == 1 ? nk / 2 + nk / 64 * 2 : nk * 2;
  double out = 0;
  switch (la.epi.kind) {
    case EPI_QKV: out = (double)la.M * la.N * 2; break;
    case EPI_RESID: out = (double)la.M * la.N * 8; break;
    case EPI_RELU: out = (double)la.M * la.N * 2; break;
    default: out = (double)la.M * la.N * 4; break;
  }
  return w + (double)la.M * la.K * 2 + out + (la.epi.bias ? la.N * 2.0 : 0.0);
}

pipo_status run_linear(pipo_ctx* ctx, const LinearArgs& la, int path, int cls) {
  cudaEvent_t a = nullptr;
  TRY(kbegin(ctx, &a));
  LAUNCH(launch_linear(la, path, ctx->gemv_max_m, ctx->s_comp));
  TRY(kend(ctx, a, cls, linear_bytes(la), 2.0 * la.M * la.N * la.K));
  return PIPO_OK;
}

// ---- pointers into a layer blob -----------------------------------------------
const __half* vec_ptr(const pipo_ctx* c, const uint8_t* blob, int v) {
  return c->lay.vec_len[v] ? reinterpret_cast<const __half*>(blob + c->lay.vec_off[v]) : nullptr;   // LLaMA: none
}

bool streamed(const pipo_ctx* c) { return c->weight_tier != PIPO_TIER_DEVICE; }
bool sharded(const pipo_ctx* c) { return c->shard_mode != 0; }   // NEXT-1: rank keeps 1/world of each blob
bool host_kv(const pipo_ctx* c) { return c->kv_tier == PIPO_TIER_HOST; }

uint8_t* kv_region(pipo_ctx* c, int layer, int which, int64_t G) {
  if (host_kv(c)) return c->kv_slot + ((G % c->R) * 2 + which) * c->kv_tensor_bytes;
  return c->kv_dev + ((int64_t)layer * 2 + which) * c->kv_tensor_bytes;
}
uint8_t* kv_host_region(pipo_ctx* c, int layer, int which) {
  return c->kv_host + ((int64_t)layer * 2 + which) * c->kv_tensor_bytes;
}
// byte ranges (offset, size) of positions [p0, p0 + np) inside a region, current batch
int kv_ranges(const pipo_ctx* c, int64_t p0, int64_t np, int64_t* off, int64_t* bytes) {
  const int64_t row = (int64_t)c->b_cur * c->dkv;   // elements per position
  if (c->kv_fmt == PIPO_W_FP16) {
    off[0] = p0 * row * 2; bytes[0] = np * row * 2;
    return 1;
  }
  off[0] = p0 * row / 2; bytes[0] = np * row / 2;
  off[1] = c->kv_codes_cap + p0 * (row / 64) * 2; bytes[1] = np * (row / 64) * 2;
  return 2;
}

// H2D copy of one contiguous byte range in chunks (blockwise transfer)
pipo_status copy_chunks(pipo_ctx* ctx, void* dst, const void* src, int64_t bytes) {
  const int64_t ch = ctx->chunk > 0 ? ctx->chunk : bytes;
  for (int64_t off = 0; off < bytes; off += ch) {
    const int64_t n = std::min(ch, bytes - off);
    CK(cudaMemcpyAsync(static_cast<uint8_t*>(dst) + off, static_cast<const uint8_t*>(src) + off, (size_t)n,
                       cudaMemcpyHostToDevice, ctx->s_copy));
  }
  return PIPO_OK;
}

// CallLoadData for global layer G: weights (+ KV positions [0, kv_pos) if host KV).
pipo_status enqueue_copy(pipo_ctx* ctx, int64_t G, int64_t kv_pos) {
  const int j = (int)(G % ctx->l), slot = (int)(G % ctx->R);
  if (G >= ctx->R) CK(cudaStreamWaitEvent(ctx->s_copy, ctx->ev_free[slot], 0));
  LAUNCH(launch_spin(ctx->dbg_copy_delay_ns, ctx->s_copy));   // test hook: a slow host link
  cudaEvent_t t0 = nullptr;
  TRY(span_begin(ctx, ctx->s_copy, &t0));
  uint8_t* dst = ctx->ring + (int64_t)slot * ctx->layer_bytes;
  int64_t bytes = 0;
  // The merged blob is loaded as ONE request (data merging), split
  // into chunk_bytes blocks (blockwise transfer; 0 = one block).
  // A segment's ready event is recorded right after the block holding its last byte,
  // so the compute stream consumes each segment as soon as it has landed.
  auto after_segment = [&](int s, cudaStream_t ready_on) -> pipo_status {
    if (s == 3 && ctx->dbg_ring_sum)   // test hook: checksum of the layer as it landed in HBM
      LAUNCH(launch_ring_sum(dst, ctx->layer_bytes, ctx->ring_sums + j, ready_on));
    CK(cudaEventRecord(ctx->ev_ready[slot][s], ready_on));
    if (s == 0 && host_kv(ctx)) {
      // KV load advanced with the layer's MHA weights (reading Q6)
      if (G >= ctx->R) CK(cudaStreamWaitEvent(ctx->s_copy, ctx->ev_kv_free[slot], 0));
      CK(cudaStreamWaitEvent(ctx->s_copy, ctx->ev_saved[j], 0));   // A6 fence
      if (kv_pos > 0) {
        int64_t off[2], nb[2];
        const int nr = kv_ranges(ctx, 0, kv_pos, off, nb);
        for (int w = 0; w < 2; ++w)
          for (int r = 0; r < nr; ++r) {
            TRY(copy_chunks(ctx, kv_region(ctx, j, w, G) + off[r], kv_host_region(ctx, j, w) + off[r], nb[r]));
            bytes += nb[r];
          }
      }
      ctx->kv_load_past[slot] = kv_pos;
      CK(cudaEventRecord(ctx->ev_ready[slot][4], ctx->s_copy));
    }
    return PIPO_OK;
  };
  if (ctx->disk) {
    for (int s = 0; s < 4; ++s) {
      const pipo_status ds = disk_enqueue_segment(ctx, j, s, dst + ctx->lay.seg_off[s]);
      if (ds != PIPO_OK) {
        ctx->poisoned = true;
        return set_err(ds, ds == PIPO_E_IO ? "disk tier read failed" : ds == PIPO_E_FORMAT ? "disk blob header mismatch"
                                                                                          : "disk tier transfer setup failed");
      }
      bytes += ctx->lay.seg_bytes[s];
      TRY(after_segment(s, ctx->s_copy));
    }
  } else if (ctx->shard_mode == 2) {
    // NEXT-1 sharded streaming, peer transport: this rank's 1/world over its own host
    // link (copy stream), then the copy engines pull every peer's range of the same layer
    // straight out of the peer's ring slot over NVLink (gather stream).  Flags in peer
    // memory order it across processes: a peer's range is read only after that peer
    // posted the layer; this rank's slot is overwritten only after every peer copied its
    // range of the layer the slot held (R layers earlier).
    const int64_t S = ctx->shard_bytes;
    const int W = ctx->shard_world, me = ctx->shard_rank;
    if (G >= ctx->R) {
      P2PFlags war{};
      for (int p = 0; p < W; ++p)
        if (p != me) war.addr[war.n++] = ctx->own_flags + 1 + p;
      LAUNCH(launch_p2p_wait(war, (int)(G - ctx->R + 1), ctx->s_copy));
    }
    TRY(copy_chunks(ctx, dst + (int64_t)me * S, ctx->host_store + (int64_t)j * S, S));
    bytes += S;
    P2PFlags post{};
    post.addr[post.n++] = ctx->own_flags;
    LAUNCH(launch_p2p_signal(post, (int)(G + 1), ctx->s_copy));
    CK(cudaEventRecord(ctx->ev_h2d[slot], ctx->s_copy));
    CK(cudaStreamWaitEvent(ctx->s_gather, ctx->ev_h2d[slot], 0));   // (also orders after ev_free)
    cudaEvent_t g0 = nullptr;
    TRY(span_begin(ctx, ctx->s_gather, &g0));
    P2PFlags ready{}, done{};
    for (int p = 0; p < W; ++p)
      if (p != me) {
        const int* pf = reinterpret_cast<const int*>(ctx->peer_ring[p] + (int64_t)ctx->R * ctx->layer_bytes);
        ready.addr[ready.n++] = const_cast<int*>(pf);
        done.addr[done.n++] = const_cast<int*>(pf) + 1 + me;
      }
    LAUNCH(launch_p2p_wait(ready, (int)(G + 1), ctx->s_gather));
    for (int p = 0; p < W; ++p)
      if (p != me)
        CK(cudaMemcpyAsync(dst + (int64_t)p * S, ctx->peer_ring[p] + (int64_t)slot * ctx->layer_bytes + (int64_t)p * S,
                           (size_t)S, cudaMemcpyDeviceToDevice, ctx->s_gather));
    LAUNCH(launch_p2p_signal(done, (int)(G + 1), ctx->s_gather));
    TRY(span_end(ctx, ctx->s_gather, g0, 3, S * (W - 1)));
    for (int s = 0; s < 4; ++s) TRY(after_segment(s, ctx->s_gather));
  } else if (ctx->shard_mode == 1) {
    // NEXT-1 sharded streaming: this rank's 1/world of the blob over its own host link
    // (copy stream), then the other ranks' ranges over NVLink by an in-place NCCL
    // all-gather on its OWN stream, ordered after this rank's H2D by an event — so the
    // gather of layer G overlaps the H2D of layer G+1 (PCIe and NVLink in parallel);
    // every segment is ready once the gather has completed.
    const int64_t S = ctx->shard_bytes;
    TRY(copy_chunks(ctx, dst + (int64_t)ctx->shard_rank * S, ctx->host_store + (int64_t)j * S, S));
    bytes += S;
    CK(cudaEventRecord(ctx->ev_h2d[slot], ctx->s_copy));
    CK(cudaStreamWaitEvent(ctx->s_gather, ctx->ev_h2d[slot], 0));
    cudaEvent_t g0 = nullptr;
    TRY(span_begin(ctx, ctx->s_gather, &g0));
    const int rc = nccl_allgather_bytes(dst + (int64_t)ctx->shard_rank * S, dst, (size_t)S, ctx->nccl_comm, ctx->s_gather);
    if (rc != 0) {
      ctx->poisoned = true;
      return set_err(PIPO_E_CUDA, std::string("ncclAllGather failed: ") + nccl_error_string(rc));
    }
    TRY(span_end(ctx, ctx->s_gather, g0, 3, S * (ctx->shard_world - 1)));
    for (int s = 0; s < 4; ++s) {
      TRY(after_segment(s, ctx->s_gather));
    }
  } else {
    const uint8_t* src = ctx->host_store + (int64_t)j * ctx->layer_bytes;
    const int64_t total = ctx->lay.seg_off[3] + ctx->lay.seg_bytes[3];
    const int64_t ch = ctx->chunk > 0 ? ctx->chunk : total;
    int next_seg = 0;
    for (int64_t off = 0; off < total; off += ch) {
      const int64_t n = std::min(ch, total - off);
      CK(cudaMemcpyAsync(dst + off, src + off, (size_t)n, cudaMemcpyHostToDevice, ctx->s_copy));
      bytes += n;
      while (next_seg < 4 && ctx->lay.seg_off[next_seg] + ctx->lay.seg_bytes[next_seg] <= off + n)
        TRY(after_segment(next_seg++, ctx->s_copy));
    }
  }
  ctx->h2d_bytes += bytes;
  TRY(span_end(ctx, ctx->s_copy, t0, 0, bytes));
  return PIPO_OK;
}

pipo_status enqueue_kv_only(pipo_ctx* ctx, int64_t G, int64_t kv_pos) {
  // DEVICE weights + HOST KV: only the KV loading task runs on the copy stream
  const int j = (int)(G % ctx->l), slot = (int)(G % ctx->R);
  if (G >= ctx->R) CK(cudaStreamWaitEvent(ctx->s_copy, ctx->ev_kv_free[slot], 0));
  CK(cudaStreamWaitEvent(ctx->s_copy, ctx->ev_saved[j], 0));
  cudaEvent_t t0 = nullptr;
  TRY(span_begin(ctx, ctx->s_copy, &t0));
  int64_t moved = 0;
  if (kv_pos > 0) {
    int64_t off[2], nb[2];
    const int nr = kv_ranges(ctx, 0, kv_pos, off, nb);
    for (int w = 0; w < 2; ++w)
      for (int r = 0; r < nr; ++r) {
        TRY(copy_chunks(ctx, kv_region(ctx, j, w, G) + off[r], kv_host_region(ctx, j, w) + off[r], nb[r]));
        moved += nb[r];
      }
  }
  ctx->kv_load_past[slot] = kv_pos;
  CK(cudaEventRecord(ctx->ev_ready[slot][4], ctx->s_copy));
  ctx->h2d_bytes += moved;
  TRY(span_end(ctx, ctx->s_copy, t0, 0, moved));
  return PIPO_OK;
}

// one forward pass over all layers: rows M = b * n at positions past .. past+n-1
pipo_status forward_pass(pipo_ctx* ctx, int b, int n, int past, bool want_logits) {
  const int M = b * n, d = ctx->d;
  ctx->forwarded = true;
  cudaStream_t cs = ctx->s_comp;
  const int64_t next_pass_kv = past + n;   // KV positions the next (decode) pass loads
  const bool llama = ctx->arch == PIPO_ARCH_LLAMA;
  const int dkv = ctx->dkv;
  LAUNCH(launch_embed(ctx->ids, b, n, past, ctx->tok, ctx->tok_lay.n_kb, ctx->pos, d, ctx->h, cs));
  LinearArgs la;
  la.ws = ctx->ws; la.ws_floats = ctx->ws_floats; la.counters = ctx->counters; la.n_counters = ctx->n_counters;
  la.num_sms = ctx->num_sms; la.M = M;
  AttnArgs aa;
  aa.b = b; aa.n = n; aa.past = past; aa.d = d; aa.n_heads = ctx->H; aa.kv_b = b;
  aa.dkv = dkv; aa.group = ctx->H / ctx->Hkv;
  aa.ws = ctx->ws; aa.ws_floats = ctx->ws_floats; aa.num_sms = ctx->num_sms;
  const int64_t pass_base = ctx->g_comp;
  const int lin_cls = n == 1 ? PIPO_K_LINEAR_DECODE : PIPO_K_LINEAR_PREFILL;

  for (int j = 0; j < ctx->l; ++j) {
    const int64_t G = ctx->g_comp++;
    const int slot = (int)(G % ctx->R);
    if (streamed(ctx) || host_kv(ctx)) {
      while (ctx->g_copy <= G + ctx->R - 1) {
        const int64_t Gc = ctx->g_copy;
        const bool this_pass = Gc < pass_base + ctx->l;
        const int64_t kv = this_pass ? (n == 1 ? past : 0) : next_pass_kv;
        if (streamed(ctx)) {
          TRY(enqueue_copy(ctx, Gc, kv));
        } else {
          TRY(enqueue_kv_only(ctx, Gc, kv));
        }
        ctx->g_copy++;
      }
    }
    const uint8_t* blob = streamed(ctx) ? ctx->ring + (int64_t)slot * ctx->layer_bytes
                                        : ctx->dev_store + (int64_t)j * ctx->layer_bytes;
    uint8_t* kreg = kv_region(ctx, j, 0, G);
    uint8_t* vreg = kv_region(ctx, j, 1, G);
    const bool q4 = ctx->kv_fmt == PIPO_W_INT4_G64;
    __half* kc = q4 ? ctx->kv_stage : reinterpret_cast<__half*>(kreg);
    __half* vc = q4 ? ctx->kv_stage + dkv : reinterpret_cast<__half*>(vreg);
    if (host_kv(ctx) && n == 1 && ctx->kv_load_past[slot] != past)
      return set_err(PIPO_E_STATE, "internal: KV prefetch range mismatch");
    cudaEvent_t t0;
    // SynchronizeLoadTask granularity: per segment (the paper's tasks): each phase waits
    // for its own segment's event right before its first kernel
    const bool seg_wait = true;
    if (streamed(ctx)) CK(cudaStreamWaitEvent(cs, ctx->ev_ready[slot][seg_wait ? 0 : 3], 0));
    if (host_kv(ctx)) CK(cudaStreamWaitEvent(cs, ctx->ev_ready[slot][4], 0));
    LAUNCH(launch_spin(ctx->dbg_comp_delay_ns, cs));   // test hook: slow compute
    TRY(span_begin(ctx, cs, &t0));
    LAUNCH(launch_layernorm(ctx->h, d, M, d, vec_ptr(ctx, blob, V_LN1_G), vec_ptr(ctx, blob, V_LN1_B), ctx->xa, cs));
    la.x = ctx->xa; la.w = blob + ctx->lay.mat_off[M_QKV]; la.wfmt = ctx->wfmt; la.N = d + 2 * dkv; la.K = d;
    la.epi = EpiParams{};
    la.epi.kind = EPI_QKV; la.epi.bias = vec_ptr(ctx, blob, V_B_QKV); la.epi.M = M; la.epi.N = d + 2 * dkv;
    la.epi.dkv = dkv;
    la.epi.q = ctx->q; la.epi.kc = kc; la.epi.vc = vc; la.epi.d = d; la.epi.n_tok = n; la.epi.past = past;
    la.epi.kv_b = b; la.epi.qscale = 1.0f / sqrtf((float)ctx->hd);
    la.epi.kv_rowmajor = q4 ? 1 : 0;
    TRY(run_linear(ctx, la, PATH_AUTO, lin_cls));
    if (llama)   // RoPE on q and the fresh K rows (q already carries hd^-0.5: rotation is linear)
      LAUNCH(launch_rope(ctx->q, kc, ctx->rope_inv, b, n, past, ctx->H, ctx->Hkv, ctx->hd, b, cs));
    aa.q = ctx->q; aa.kc = kc; aa.vc = vc; aa.o = ctx->xa;
    aa.kv_pos_stride = 0; aa.kv_b_stride = 0; aa.kq = nullptr;
    if (q4) {
      // append: quantize the fresh rows into the int4 cache (codes + fp16 scales)
      LAUNCH(launch_kv_quant(ctx->kv_stage, b, n, past, d, b, kreg,
                             reinterpret_cast<__half*>(kreg + ctx->kv_codes_cap), vreg,
                             reinterpret_cast<__half*>(vreg + ctx->kv_codes_cap), cs));
      if (n == 1) {
        aa.kq = kreg; aa.ks = reinterpret_cast<const __half*>(kreg + ctx->kv_codes_cap);
        aa.vq = vreg; aa.vs = reinterpret_cast<const __half*>(vreg + ctx->kv_codes_cap);
      } else {
        aa.kv_pos_stride = 2 * (int64_t)d;       // prefill attends over the fresh fp16 rows
        aa.kv_b_stride = (int64_t)n * 2 * d;
      }
    }
    {
      cudaEvent_t ka = nullptr;
      TRY(kbegin(ctx, &ka));
      if (n == 1 && q4) LAUNCH(launch_attention_decode_q4(aa, cs));
      else if (n == 1) LAUNCH(launch_attention_decode(aa, cs));
      else LAUNCH(launch_attention_prefill(aa, cs));
      const double L = past + n;
      const double kvb = 2.0 * L * b * dkv * (q4 && n == 1 ? (0.5 + 2.0 / 64) : 2.0);
      // QK^T and PV: 2 flops per multiply-add each; causal prefill attends over past + (n+1)/2
      // positions on average
      const double fl = n == 1 ? 4.0 * b * d * L : 4.0 * b * d * (double)n * (past + (n + 1) / 2.0);
      TRY(kend(ctx, ka, n == 1 ? PIPO_K_ATTN_DECODE : PIPO_K_ATTN_PREFILL, kvb + 4.0 * M * d, fl));
    }
    TRY(span_end(ctx, cs, t0, 1, 0));
    if (host_kv(ctx)) {
      // CallStoreCache: save the new positions after MHA on the save stream
      CK(cudaEventRecord(ctx->ev_attn[slot], cs));
      CK(cudaStreamWaitEvent(ctx->s_save, ctx->ev_attn[slot], 0));
      cudaEvent_t s0;
      TRY(span_begin(ctx, ctx->s_save, &s0));
      int64_t off[2], nb[2], saved = 0;
      const int nr = kv_ranges(ctx, past, n, off, nb);
      for (int w = 0; w < 2; ++w)
        for (int r = 0; r < nr; ++r) {
          CK(cudaMemcpyAsync(kv_host_region(ctx, j, w) + off[r], kv_region(ctx, j, w, G) + off[r], (size_t)nb[r],
                             cudaMemcpyDeviceToHost, ctx->s_save));
          saved += nb[r];
        }
      ctx->d2h_bytes += saved;
      CK(cudaEventRecord(ctx->ev_saved[j], ctx->s_save));
      CK(cudaEventRecord(ctx->ev_kv_free[slot], ctx->s_save));
      TRY(span_end(ctx, ctx->s_save, s0, 2, saved));
    }
    // ---- MHA out-proj + residual (seg 1) ----
    if (streamed(ctx) && seg_wait) CK(cudaStreamWaitEvent(cs, ctx->ev_ready[slot][1], 0));
    TRY(span_begin(ctx, cs, &t0));
    la.x = ctx->xa; la.w = blob + ctx->lay.mat_off[M_OUT]; la.N = d; la.K = d;
    la.epi = EpiParams{};
    la.epi.kind = EPI_RESID; la.epi.bias = vec_ptr(ctx, blob, V_B_OUT); la.epi.M = M; la.epi.N = d; la.epi.h = ctx->h;
    TRY(run_linear(ctx, la, PATH_AUTO, lin_cls));
    TRY(span_end(ctx, cs, t0, 1, 0));
    // ---- MLP: LN2 + FC1 + ReLU (seg 2) ----
    if (streamed(ctx) && seg_wait) CK(cudaStreamWaitEvent(cs, ctx->ev_ready[slot][2], 0));
    TRY(span_begin(ctx, cs, &t0));
    LAUNCH(launch_layernorm(ctx->h, d, M, d, vec_ptr(ctx, blob, V_LN2_G), vec_ptr(ctx, blob, V_LN2_B), ctx->xa, cs));
    la.x = ctx->xa; la.w = blob + ctx->lay.mat_off[M_FC1]; la.N = llama ? 2 * ctx->F : ctx->F; la.K = d;
    la.epi = EpiParams{};
    la.epi.kind = llama ? EPI_HALF : EPI_RELU; la.epi.bias = vec_ptr(ctx, blob, V_B_FC1); la.epi.M = M;
    la.epi.N = la.N; la.epi.u = llama ? ctx->gu : ctx->u;
    TRY(run_linear(ctx, la, PATH_AUTO, lin_cls));
    if (llama) LAUNCH(launch_swiglu(ctx->gu, M, ctx->F, ctx->u, cs));   // u = silu(gate) * up
    TRY(span_end(ctx, cs, t0, 1, 0));
    // ---- MLP: FC2 + residual (seg 3) ----
    if (streamed(ctx) && seg_wait) CK(cudaStreamWaitEvent(cs, ctx->ev_ready[slot][3], 0));
    TRY(span_begin(ctx, cs, &t0));
    la.x = ctx->u; la.w = blob + ctx->lay.mat_off[M_FC2]; la.N = d; la.K = ctx->F;
    la.epi = EpiParams{};
    la.epi.kind = EPI_RESID; la.epi.bias = vec_ptr(ctx, blob, V_B_FC2); la.epi.M = M; la.epi.N = d; la.epi.h = ctx->h;
    TRY(run_linear(ctx, la, PATH_AUTO, lin_cls));
    TRY(span_end(ctx, cs, t0, 1, 0));
    if (streamed(ctx)) CK(cudaEventRecord(ctx->ev_free[slot], cs));   // ring slot release (a12)
    if (ctx->cap_on)
      CK(cudaMemcpyAsync(ctx->cap_dev + (int64_t)j * M * d, ctx->h, (size_t)M * d * 4, cudaMemcpyDeviceToDevice, cs));
  }
  // ---- output embedding: final LN (last position of each sequence), LM head, argmax (a13) ----
  cudaEvent_t t0;
  TRY(span_begin(ctx, cs, &t0));
  LAUNCH(launch_layernorm(ctx->h + (int64_t)(n - 1) * d, (int64_t)n * d, b, d, ctx->lnf_g, ctx->lnf_b, ctx->xa, cs));
  la.x = ctx->xa; la.w = reinterpret_cast<const uint8_t*>(ctx->head); la.wfmt = 0; la.M = b; la.N = ctx->V; la.K = d;
  la.epi = EpiParams{};
  la.epi.kind = EPI_F32; la.epi.M = b; la.epi.N = ctx->V; la.epi.y = ctx->logits; la.epi.ldy = ctx->V;
  // LM head: the streaming tcgen05 kernel for b <= 64, else the tile GEMM
  TRY(run_linear(ctx, la, b <= 64 ? PATH_HEAD : PATH_TC, PIPO_K_HEAD));
  LAUNCH(launch_argmax(ctx->logits, b, ctx->V, ctx->V, ctx->next, cs));
  TRY(span_end(ctx, cs, t0, 1, 0));
  (void)want_logits;
  return PIPO_OK;
}

// A pass that fails after its first enqueue leaves g_comp / g_copy mid-pass and ring slots
// holding layers the next pass would not expect: poison the context (pipo.h conventions).
pipo_status forward(pipo_ctx* ctx, int b, int n, int past, bool want_logits) {
  const pipo_status s = forward_pass(ctx, b, n, past, want_logits);
  if (s != PIPO_OK) ctx->poisoned = true;
  return s;
}

// Weights (re)loaded after a pass: the copy stream may be prefetching the next pass's
// first layers from the old store (and disk readers may hold its files).  Drain every
// stream and forget the prefetch so the next pass re-issues it from the new weights.
pipo_status drain_prefetch(pipo_ctx* ctx) {
  if (!ctx->forwarded) return PIPO_OK;
  CK(cudaDeviceSynchronize());
  ctx->g_copy = ctx->g_comp;
  return PIPO_OK;
}

pipo_status finish_call(pipo_ctx* ctx, int b, int n, int32_t* next, float* logits) {
  CK(cudaMemcpyAsync(ctx->pin_next, ctx->next, (size_t)b * 4, cudaMemcpyDeviceToHost, ctx->s_comp));
  ctx->d2h_bytes += (int64_t)b * 4;
  if (logits) {
    CK(cudaMemcpyAsync(logits, ctx->logits, (size_t)b * ctx->V * 4, cudaMemcpyDeviceToHost, ctx->s_comp));
    ctx->d2h_bytes += (int64_t)b * ctx->V * 4;
  }
  if (ctx->cap_on) {
    CK(cudaMemcpyAsync(ctx->cap_host, ctx->cap_dev, (size_t)ctx->l * b * n * ctx->d * 4, cudaMemcpyDeviceToHost,
                       ctx->s_comp));
  }
  CK(cudaStreamSynchronize(ctx->s_comp));
  if (ctx->disk && disk_io_error(ctx)) {
    ctx->poisoned = true;
    return set_err(PIPO_E_IO, "disk tier read failed");
  }
  if (next) std::memcpy(next, ctx->pin_next, (size_t)b * 4);
  ctx->cap_on = false;
  return PIPO_OK;
}

pipo_status check_ready(pipo_ctx* ctx) {
  if (!ctx->embed_loaded) return set_err(PIPO_E_STATE, "embedding weights not loaded");
  for (int j = 0; j < ctx->l; ++j)
    if (!ctx->layer_loaded[j]) return set_err(PIPO_E_STATE, "decoder layer " + std::to_string(j) + " not loaded");
  return PIPO_OK;
}

pipo_status stage_ids(pipo_ctx* ctx, const int32_t* tokens, int64_t count) {
  for (int64_t i = 0; i < count; ++i)
    if (tokens[i] < 0 || tokens[i] >= ctx->V) return set_err(PIPO_E_INVALID_ARG, "token id out of range");
  std::memcpy(ctx->pin_ids, tokens, (size_t)count * 4);
  CK(cudaMemcpyAsync(ctx->ids, ctx->pin_ids, (size_t)count * 4, cudaMemcpyHostToDevice, ctx->s_comp));
  ctx->h2d_bytes += count * 4;
  return PIPO_OK;
}

pipo_status window_mark(pipo_ctx* ctx, bool start) {
  if (start && !ctx->win_open) {
    CK(cudaEventRecord(ctx->win_start, ctx->s_comp));
    ctx->win_open = true;
    ctx->win_closed = false;
  }
  if (!start) {
    CK(cudaEventRecord(ctx->win_end, ctx->s_comp));
    ctx->win_closed = true;
  }
  return PIPO_OK;
}

double union_len(std::vector<std::pair<double, double>>& v) {
  std::sort(v.begin(), v.end());
  double tot = 0, cs = -1, ce = -1;
  for (auto& p : v) {
    if (p.first > ce) {
      if (ce > cs) tot += ce - cs;
      cs = p.first;
      ce = p.second;
    } else {
      ce = std::max(ce, p.second);
    }
  }
  if (ce > cs) tot += ce - cs;
  return tot;
}

// NEXT-3: Eq. (1) on this machine.  The memory model is the paper's
// (App. B) for b = max_batch, s = max_seq; the hardware numbers are measured here.
pipo_status apply_auto_plan(pipo_ctx* ctx) {
  const pipo_config& c = ctx->cfg;
  pipo_mem_spec sp{};
  sp.n_layers = ctx->l; sp.d_model = ctx->d; sp.vocab = ctx->V; sp.n_heads = ctx->H; sp.n_kv_heads = ctx->Hkv;
  sp.ffn_hidden = ctx->F; sp.mlp_mats = ctx->arch == PIPO_ARCH_LLAMA ? 3 : 2;
  sp.p_weight = ctx->wfmt == PIPO_W_INT4_G64 ? 17.0 / 32.0 : 2.0;
  sp.p_act = 2.0;
  size_t free_b = 0, total_b = 0;
  CK(cudaMemGetInfo(&free_b, &total_b));
  double m_gpu = (double)free_b;
  if (c.hbm_budget > 0) m_gpu = std::min(m_gpu, (double)c.hbm_budget);
  double m_cpu = 0;
  if (FILE* f = fopen("/proc/meminfo", "r")) {
    char key[64];
    long long kb = 0;
    while (fscanf(f, "%63s %lld kB\n", key, &kb) == 2)
      if (!strcmp(key, "MemAvailable:")) { m_cpu = (double)kb * 1024.0; break; }
    fclose(f);
  }
  if (m_cpu <= 0) m_cpu = 1;
  // App. A: pinned H2D probe over block sizes on the copy stream (best of 3 each)
  const int64_t sizes[4] = {4ll << 20, 16ll << 20, 32ll << 20, 64ll << 20};
  double bps[4] = {0, 0, 0, 0};
  uint8_t *hsrc = nullptr, *ddst = nullptr;
  TRY(host_alloc(ctx, &hsrc, sizes[3]));
  pipo_status st = dev_alloc(ctx, &ddst, sizes[3]);
  if (st != PIPO_OK) { host_free(ctx, hsrc, sizes[3]); return st; }
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  for (int i = 0; i < 4; ++i)
    for (int r = 0; r < 4; ++r) {
      CK(cudaEventRecord(e0, ctx->s_copy));
      CK(cudaMemcpyAsync(ddst, hsrc, (size_t)sizes[i], cudaMemcpyHostToDevice, ctx->s_copy));
      CK(cudaEventRecord(e1, ctx->s_copy));
      CK(cudaEventSynchronize(e1));
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (r > 0) bps[i] = std::max(bps[i], sizes[i] / (ms * 1e-3));
    }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  host_free(ctx, hsrc, sizes[3]);
  cudaFree(ddst);
  ctx->hbm_bytes -= sizes[3];
  pipo_hw_spec hw{m_gpu, m_cpu, bps[3], bps[3] / 10.0};
  pipo_plan plan{};
  TRY(pipo_choose_plan(&sp, ctx->max_b, ctx->max_s, &hw, sizes, bps, nullptr, 4, &plan));
  if (plan.weight_tier == PIPO_TIER_DISK && ctx->disk_dir.empty())
    return set_err(PIPO_E_INFEASIBLE, "Eq. (1) puts the weights on disk (W + C >= M_CPU) but cfg.disk_dir is empty");
  ctx->weight_tier = plan.weight_tier;
  ctx->kv_tier = plan.weight_tier == PIPO_TIER_DEVICE ? PIPO_TIER_DEVICE : PIPO_TIER_HOST;
  ctx->R = std::min(plan.ring_layers, ctx->l);
  ctx->chunk = plan.block_bytes;
  ctx->gemv_max_m = plan.gemv_max_m;
  ctx->auto_plan = true;
  ctx->plan = plan;
  return PIPO_OK;
}

}  // namespace

pipo_status pipo::set_last_error(pipo_status s, const char* msg) { return set_err(s, msg); }

extern "C" {

const char* pipo_last_error(void) { return g_err.c_str(); }
int32_t pipo_abi_version(void) { return PIPO_ABI_VERSION; }

pipo_status pipeline_init(const pipo_config* cfg, pipo_ctx** out) {
  if (!out) return set_err(PIPO_E_INVALID_ARG, "out is NULL");
  *out = nullptr;
  if (!cfg) return set_err(PIPO_E_INVALID_ARG, "cfg is NULL");
  const pipo_config& c = *cfg;
  if (c.d_model <= 0 || c.d_model % 64 || c.n_layers <= 0 || c.n_heads <= 0 || c.d_model % c.n_heads ||
      c.ffn_dim <= 0 || c.ffn_dim % 64 || c.vocab <= 0 || c.max_pos <= 0 || c.max_batch <= 0 || c.max_seq <= 1)
    return set_err(PIPO_E_INVALID_ARG, "invalid model/workload shape");
  const int hd = c.d_model / c.n_heads;
  if (hd != 64 && hd != 128) return set_err(PIPO_E_INVALID_ARG, "head_dim must be 64 or 128");
  if (c.d_model > 8192) return set_err(PIPO_E_INVALID_ARG, "d_model > 8192 unsupported");
  if (c.max_seq > c.max_pos) return set_err(PIPO_E_INVALID_ARG, "max_seq exceeds max_pos");
  if (c.wfmt != PIPO_W_FP16 && c.wfmt != PIPO_W_INT4_G64) return set_err(PIPO_E_INVALID_ARG, "bad wfmt");
  if (c.weight_tier < 0 || c.weight_tier > 2) return set_err(PIPO_E_INVALID_ARG, "bad weight_tier");
  if (c.kv_tier != PIPO_TIER_DEVICE && c.kv_tier != PIPO_TIER_HOST) return set_err(PIPO_E_INVALID_ARG, "bad kv_tier");
  if (c.kv_fmt != PIPO_W_FP16 && c.kv_fmt != PIPO_W_INT4_G64) return set_err(PIPO_E_INVALID_ARG, "bad kv_fmt");
  if (c.weight_tier == PIPO_TIER_DISK && (!c.disk_dir || !c.disk_dir[0]))
    return set_err(PIPO_E_INVALID_ARG, "disk tier needs disk_dir");
  if (c.arch != PIPO_ARCH_OPT && c.arch != PIPO_ARCH_LLAMA) return set_err(PIPO_E_INVALID_ARG, "bad arch");
  const int n_kv = c.arch == PIPO_ARCH_LLAMA && c.n_kv_heads > 0 ? c.n_kv_heads : c.n_heads;
  if (c.arch == PIPO_ARCH_LLAMA) {
    if (c.n_heads % n_kv) return set_err(PIPO_E_INVALID_ARG, "n_kv_heads must divide n_heads");
    if (c.ffn_dim % 128) return set_err(PIPO_E_INVALID_ARG, "LLaMA ffn_dim must be a multiple of 128");
    if (c.kv_fmt != PIPO_W_FP16) return set_err(PIPO_E_INVALID_ARG, "LLaMA with an int4 KV cache is not built");
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return set_err(PIPO_E_CUDA, "no CUDA device (the library has no CPU fallback)");
  }
  if (c.device < 0 || c.device >= ndev) return set_err(PIPO_E_INVALID_ARG, "device ordinal out of range");

  pipo_ctx* ctx = new pipo_ctx();
  ctx->cfg = c;
  ctx->disk_dir = c.disk_dir ? c.disk_dir : "";
  ctx->cfg.disk_dir = nullptr;
  ctx->d = c.d_model; ctx->l = c.n_layers; ctx->H = c.n_heads; ctx->F = c.ffn_dim; ctx->V = c.vocab;
  ctx->hd = hd; ctx->max_b = c.max_batch; ctx->max_s = c.max_seq; ctx->wfmt = c.wfmt;
  ctx->arch = c.arch; ctx->Hkv = n_kv; ctx->dkv = n_kv * hd;
  ctx->weight_tier = c.weight_tier; ctx->kv_tier = c.kv_tier; ctx->kv_fmt = c.kv_fmt;
  ctx->R = c.ring_layers > 0 ? c.ring_layers : 2;
  ctx->R = std::min({ctx->R, kMaxRing, ctx->l});
  ctx->chunk = c.chunk_bytes;
  ctx->gemv_max_m = c.gemv_max_m > 0 ? std::min(c.gemv_max_m, 16) : 15;
  ctx->timeline = (c.flags & PIPO_F_TIMELINE) != 0;
  ctx->kprof = (c.flags & PIPO_F_KPROF) != 0;
  ctx->lay = layer_layout(ctx->d, ctx->F, ctx->wfmt, ctx->dkv, ctx->arch == PIPO_ARCH_LLAMA);
  ctx->layer_bytes = ctx->lay.total;
  ctx->layer_loaded.assign(ctx->l, 0);
  ctx->ev_saved.assign(ctx->l, nullptr);
  ctx->kv_load_past.assign(kMaxRing, -1);

  auto fail = [&](pipo_status s) {
    std::string m = g_err;
    pipeline_destroy(ctx);
    g_err = m;
    return s;
  };
#define TRYI(x)                        \
  do {                                 \
    pipo_status s_ = (x);              \
    if (s_ != PIPO_OK) return fail(s_); \
  } while (0)
#define CKI(x)                                                            \
  do {                                                                    \
    cudaError_t e_ = (x);                                                 \
    if (e_ != cudaSuccess) return fail(cuda_fail(ctx, e_, #x, __LINE__)); \
  } while (0)

  CKI(cudaSetDevice(c.device));
  cudaDeviceProp prop;
  CKI(cudaGetDeviceProperties(&prop, c.device));
  if (prop.major < 10) return fail(set_err(PIPO_E_CUDA, "device is not sm_100-class (built for sm_100a only)"));
  ctx->num_sms = prop.multiProcessorCount;
  ctx->numa_node = resolve_numa_node(c.numa_node, c.device);
  {
    // compute stream at the highest priority: the copy stream runs multi-ms DMA commands,
    // the compute stream short kernels and events
    int lo = 0, hi = 0;
    CKI(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CKI(cudaStreamCreateWithPriority(&ctx->s_comp, cudaStreamNonBlocking, hi));
  }
  CKI(cudaStreamCreateWithFlags(&ctx->s_copy, cudaStreamNonBlocking));
  CKI(cudaStreamCreateWithFlags(&ctx->s_save, cudaStreamNonBlocking));
  for (int i = 0; i < kMaxRing; ++i) {
    for (int s = 0; s < 5; ++s) CKI(cudaEventCreateWithFlags(&ctx->ev_ready[i][s], cudaEventDisableTiming));
    CKI(cudaEventCreateWithFlags(&ctx->ev_free[i], cudaEventDisableTiming));
    CKI(cudaEventCreateWithFlags(&ctx->ev_kv_free[i], cudaEventDisableTiming));
    CKI(cudaEventCreateWithFlags(&ctx->ev_attn[i], cudaEventDisableTiming));
  }
  for (int j = 0; j < ctx->l; ++j) CKI(cudaEventCreateWithFlags(&ctx->ev_saved[j], cudaEventDisableTiming));
  if (c.flags & PIPO_F_AUTO_PLAN) TRYI(apply_auto_plan(ctx));
  CKI(cudaEventCreate(&ctx->win_start));
  CKI(cudaEventCreate(&ctx->win_end));

  // resident embeddings
  ctx->tok_lay = mat_layout(ctx->V, ctx->d, 0);
  TRYI(dev_alloc(ctx, &ctx->tok, ctx->tok_lay.bytes));
  TRYI(dev_alloc(ctx, &ctx->lnf_g, ctx->d * 2));
  if (ctx->arch == PIPO_ARCH_OPT) {
    TRYI(dev_alloc(ctx, &ctx->pos, (int64_t)(c.max_pos + 2) * ctx->d * 2));
    TRYI(dev_alloc(ctx, &ctx->lnf_b, ctx->d * 2));
    ctx->head = ctx->tok;   // tied LM head
  } else {
    TRYI(dev_alloc(ctx, &ctx->head, ctx->tok_lay.bytes));
    // llama3 inverse frequencies in double on the host ([ext] transformers
    // _compute_llama3_parameters), uploaded as fp32 (the RoPE kernel multiplies in fp32)
    const double theta = c.rope_theta > 0 ? c.rope_theta : 10000.0;
    std::vector<float> inv((size_t)hd / 2);
    for (int i = 0; i < hd / 2; ++i) {
      double f = 1.0 / std::pow(theta, (2.0 * i) / hd);
      if (c.rope_factor > 0) {
        const double lo = c.rope_low_freq > 0 ? c.rope_low_freq : 1.0, hi = c.rope_high_freq > 0 ? c.rope_high_freq : 4.0;
        const double orig = c.rope_orig_max_pos > 0 ? c.rope_orig_max_pos : 8192;
        const double wl = 2.0 * M_PI / f;
        if (wl > orig / lo) {
          f = f / c.rope_factor;
        } else if (!(wl < orig / hi)) {
          const double sm = (orig / wl - lo) / (hi - lo);
          f = (1.0 - sm) * f / c.rope_factor + sm * f;
        }
      }
      inv[i] = (float)f;
    }
    TRYI(dev_alloc(ctx, &ctx->rope_inv, (int64_t)hd / 2 * 4));
    CKI(cudaMemcpy(ctx->rope_inv, inv.data(), inv.size() * 4, cudaMemcpyHostToDevice));
  }
  // weights
  if (ctx->weight_tier == PIPO_TIER_DISK && ctx->disk_dir.empty())
    return fail(set_err(PIPO_E_INVALID_ARG, "disk tier needs disk_dir"));
  if (ctx->weight_tier == PIPO_TIER_DEVICE) {
    TRYI(dev_alloc(ctx, &ctx->dev_store, (int64_t)ctx->l * ctx->layer_bytes));
  } else {
    TRYI(dev_alloc(ctx, &ctx->ring, (int64_t)ctx->R * ctx->layer_bytes));
    if (ctx->weight_tier == PIPO_TIER_HOST) {
      TRYI(host_alloc(ctx, &ctx->host_store, (int64_t)ctx->l * ctx->layer_bytes, true));
    } else {
      const pipo_status ds = disk_open(ctx, c.disk_threads > 0 ? c.disk_threads : 4);
      if (ds != PIPO_OK) return fail(set_err(ds, "disk tier init failed (stream memory operations / pinned ring)"));
    }
  }
  // KV cache
  const int64_t kv_elems = (int64_t)ctx->max_s * ctx->max_b * ctx->dkv;
  if (ctx->kv_fmt == PIPO_W_INT4_G64) {
    ctx->kv_codes_cap = round_up(kv_elems / 2, 256);
    ctx->kv_tensor_bytes = round_up(ctx->kv_codes_cap + kv_elems / 64 * 2, 4096);
  } else {
    ctx->kv_tensor_bytes = kv_elems * 2;
  }
  if (host_kv(ctx)) {
    TRYI(host_alloc(ctx, &ctx->kv_host, (int64_t)ctx->l * 2 * ctx->kv_tensor_bytes, true));
    TRYI(dev_alloc(ctx, &ctx->kv_slot, (int64_t)ctx->R * 2 * ctx->kv_tensor_bytes));
  } else {
    TRYI(dev_alloc(ctx, &ctx->kv_dev, (int64_t)ctx->l * 2 * ctx->kv_tensor_bytes));
  }
  // activations
  ctx->rows_cap = (int64_t)ctx->max_b * ctx->max_s;
  TRYI(dev_alloc(ctx, &ctx->h, ctx->rows_cap * ctx->d * 4));
  TRYI(dev_alloc(ctx, &ctx->xa, ctx->rows_cap * ctx->d * 2));
  TRYI(dev_alloc(ctx, &ctx->q, ctx->rows_cap * ctx->d * 2));
  TRYI(dev_alloc(ctx, &ctx->u, ctx->rows_cap * ctx->F * 2));
  if (ctx->arch == PIPO_ARCH_LLAMA) TRYI(dev_alloc(ctx, &ctx->gu, ctx->rows_cap * 2 * ctx->F * 2));
  TRYI(dev_alloc(ctx, &ctx->logits, (int64_t)ctx->max_b * ctx->V * 4));
  TRYI(dev_alloc(ctx, &ctx->ids, ctx->rows_cap * 4));
  TRYI(dev_alloc(ctx, &ctx->next, (int64_t)ctx->max_b * 4));
  TRYI(host_alloc(ctx, &ctx->pin_ids, ctx->rows_cap * 4));
  TRYI(host_alloc(ctx, &ctx->pin_next, (int64_t)ctx->max_b * 4));
  ctx->ws_floats = 16ll << 20;
  TRYI(dev_alloc(ctx, &ctx->ws, ctx->ws_floats * 4));
  ctx->n_counters = 1 << 16;
  TRYI(dev_alloc(ctx, &ctx->counters, (int64_t)ctx->n_counters * 4));
  CKI(cudaMemset(ctx->counters, 0, (size_t)ctx->n_counters * 4));
  TRYI(dev_alloc(ctx, &ctx->quant_bad, 4));
  CKI(cudaMemset(ctx->kv_dev ? (void*)ctx->kv_dev : (void*)ctx->kv_slot, 0,
                 (size_t)(host_kv(ctx) ? ctx->R : ctx->l) * 2 * ctx->kv_tensor_bytes));
  if (ctx->kv_fmt == PIPO_W_INT4_G64) TRYI(dev_alloc(ctx, &ctx->kv_stage, ctx->rows_cap * 2 * ctx->dkv * 2));
  CKI(cudaDeviceSynchronize());
  *out = ctx;
  return PIPO_OK;
#undef TRYI
#undef CKI
}

void pipeline_destroy(pipo_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->cfg.device);
  cudaDeviceSynchronize();
  cudaGetLastError();
  if (ctx->disk) disk_close(ctx);
  if (ctx->nccl_comm) nccl_comm_destroy(ctx->nccl_comm);
  for (auto& p : ctx->peer_ring)
    if (p) cudaIpcCloseMemHandle(p);
  if (ctx->pend_ring) cudaFree(ctx->pend_ring);
  if (ctx->pend_store) host_free(ctx, ctx->pend_store, (int64_t)ctx->l * ctx->pend_S);
  if (ctx->head == ctx->tok) ctx->head = nullptr;
  void* dev[] = {ctx->tok, ctx->head, ctx->gu, ctx->rope_inv, ctx->pos, ctx->lnf_g, ctx->lnf_b, ctx->dev_store, ctx->ring, ctx->kv_dev, ctx->kv_slot, ctx->kv_stage,
                 ctx->h, ctx->xa, ctx->q, ctx->u, ctx->logits, ctx->ids, ctx->next, ctx->ws, ctx->counters,
                 ctx->quant_bad, ctx->cap_dev, ctx->ring_sums};
  for (void* p : dev)
    if (p) cudaFree(p);
  void* hst[] = {ctx->host_store, ctx->kv_host, ctx->pin_ids, ctx->pin_next};
  for (void* p : hst) {
    bool numa = false;
    for (auto& a : ctx->numa_allocs)
      if (a.first == p) numa = true;
    if (p && !numa) cudaFreeHost(p);
  }
  for (auto& a : ctx->numa_allocs) numa_host_free(a.first, a.second);
  ctx->numa_allocs.clear();
  for (int i = 0; i < kMaxRing; ++i) {
    for (int s = 0; s < 5; ++s)
      if (ctx->ev_ready[i][s]) cudaEventDestroy(ctx->ev_ready[i][s]);
    if (ctx->ev_free[i]) cudaEventDestroy(ctx->ev_free[i]);
    if (ctx->ev_kv_free[i]) cudaEventDestroy(ctx->ev_kv_free[i]);
    if (ctx->ev_attn[i]) cudaEventDestroy(ctx->ev_attn[i]);
  }
  for (auto e : ctx->ev_saved)
    if (e) cudaEventDestroy(e);
  for (auto e : ctx->ev_pool) cudaEventDestroy(e);
  if (ctx->win_start) cudaEventDestroy(ctx->win_start);
  if (ctx->win_end) cudaEventDestroy(ctx->win_end);
  if (ctx->s_comp) cudaStreamDestroy(ctx->s_comp);
  if (ctx->s_copy) cudaStreamDestroy(ctx->s_copy);
  if (ctx->s_save) cudaStreamDestroy(ctx->s_save);
  if (ctx->s_gather) cudaStreamDestroy(ctx->s_gather);
  for (auto e : ctx->ev_h2d)
    if (e) cudaEventDestroy(e);
  cudaGetLastError();
  delete ctx;
}

pipo_status load_layer_weights(pipo_ctx* ctx, int32_t layer, const void* w) {
  CHECK_CTX();
  if (!w) return set_err(PIPO_E_INVALID_ARG, "weights pointer is NULL");
  CK(cudaSetDevice(ctx->cfg.device));
  if (layer == PIPO_LAYER_EMBED) {
    const pipo_embed_weights* e = static_cast<const pipo_embed_weights*>(w);
    const bool llama = ctx->arch == PIPO_ARCH_LLAMA;
    if (!e->tok || !e->lnf_g || (llama ? !e->lm_head : (!e->pos || !e->lnf_b)))
      return set_err(PIPO_E_INVALID_ARG, "NULL embedding tensor");
    std::vector<uint8_t> tiled((size_t)ctx->tok_lay.bytes);
    tile_fp16(e->tok, ctx->V, ctx->d, tiled.data());
    CK(cudaMemcpy(ctx->tok, tiled.data(), tiled.size(), cudaMemcpyHostToDevice));
    if (llama) {
      tile_fp16(e->lm_head, ctx->V, ctx->d, tiled.data());
      CK(cudaMemcpy(ctx->head, tiled.data(), tiled.size(), cudaMemcpyHostToDevice));
    }
    const int64_t npos = llama ? ctx->d : (int64_t)(ctx->cfg.max_pos + 2) * ctx->d;
    std::vector<uint16_t> tmp((size_t)std::max<int64_t>(npos, ctx->d));
    if (!llama) {
      for (int64_t i = 0; i < npos; ++i) tmp[i] = f32_to_f16_rne(e->pos[i]);
      CK(cudaMemcpy(ctx->pos, tmp.data(), (size_t)npos * 2, cudaMemcpyHostToDevice));
    }
    for (int64_t i = 0; i < ctx->d; ++i) tmp[i] = f32_to_f16_rne(e->lnf_g[i]);
    CK(cudaMemcpy(ctx->lnf_g, tmp.data(), (size_t)ctx->d * 2, cudaMemcpyHostToDevice));
    if (!llama) {
      for (int64_t i = 0; i < ctx->d; ++i) tmp[i] = f32_to_f16_rne(e->lnf_b[i]);
      CK(cudaMemcpy(ctx->lnf_b, tmp.data(), (size_t)ctx->d * 2, cudaMemcpyHostToDevice));
    }
    ctx->embed_loaded = true;
    return PIPO_OK;
  }
  if (layer < 0 || layer >= ctx->l) return set_err(PIPO_E_INVALID_ARG, "layer index out of range");
  TRY(drain_prefetch(ctx));
  const pipo_layer_weights* lw = static_cast<const pipo_layer_weights*>(w);
  uint8_t* dst = nullptr;
  std::vector<uint8_t> tmp;
  if (ctx->weight_tier == PIPO_TIER_HOST && !sharded(ctx)) {
    dst = ctx->host_store + (int64_t)layer * ctx->layer_bytes;
  } else {
    tmp.resize((size_t)ctx->layer_bytes);
    dst = tmp.data();
  }
  if (!build_layer_blob(lw, ctx->lay, ctx->wfmt, dst))
    return set_err(PIPO_E_INVALID_ARG, "non-finite weight, NULL tensor or fp16-overflowing group scale");
  if (sharded(ctx))   // sharded streaming: keep only this rank's range (padding is zero)
    std::memcpy(ctx->host_store + (int64_t)layer * ctx->shard_bytes, dst + (int64_t)ctx->shard_rank * ctx->shard_bytes,
                (size_t)ctx->shard_bytes);
  if (ctx->weight_tier == PIPO_TIER_DEVICE)
    CK(cudaMemcpy(ctx->dev_store + (int64_t)layer * ctx->layer_bytes, dst, (size_t)ctx->layer_bytes,
                  cudaMemcpyHostToDevice));
  else if (ctx->weight_tier == PIPO_TIER_DISK) {
    const pipo_status ds = disk_write_layer(ctx, layer, dst);
    if (ds != PIPO_OK) return set_err(ds, "writing the layer blob file failed");
  }
  ctx->layer_loaded[layer] = 1;
  return PIPO_OK;
}

pipo_status pipo_load_synthetic(pipo_ctx* ctx, int32_t layer, uint64_t seed) {
  CHECK_CTX();
  CK(cudaSetDevice(ctx->cfg.device));
  cudaStream_t st = ctx->s_comp;
  const int64_t d = ctx->d, F = ctx->F;
  auto draw = [&](float* dst, uint32_t slot, uint32_t tid, int kind, double param, int64_t count) -> pipo_status {
    LAUNCH(launch_synth(dst, 0, count, synth_key(seed, slot, tid), kind, synth_scale(kind, param), st));
    return PIPO_OK;
  };
  const bool llama = ctx->arch == PIPO_ARCH_LLAMA;
  if (layer == PIPO_LAYER_EMBED) {
    const int64_t ntok = (int64_t)ctx->V * d, npos = llama ? 0 : (int64_t)(ctx->cfg.max_pos + 2) * d;
    float* buf = nullptr;
    TRY(dev_alloc(ctx, &buf, std::max(ntok, npos) * 4));
    pipo_status s = PIPO_OK;
    do {   // pipo_synth tensor ids: tok 0, pos 1, lnf_g 2, lnf_b 3, lm_head 4
      if ((s = draw(buf, 0, 0, 0, 0.02, ntok)) != PIPO_OK) break;
      LAUNCH(launch_tile_fp16(buf, ctx->V, d, reinterpret_cast<uint8_t*>(ctx->tok), st));
      if (llama) {
        if ((s = draw(buf, 0, 4, 0, 0.02, ntok)) != PIPO_OK) break;
        LAUNCH(launch_tile_fp16(buf, ctx->V, d, reinterpret_cast<uint8_t*>(ctx->head), st));
      } else {
        if ((s = draw(buf, 0, 1, 0, 0.02, npos)) != PIPO_OK) break;
        LAUNCH(launch_f32_to_f16(buf, ctx->pos, npos, st));
      }
      if ((s = draw(buf, 0, 2, 2, 0.1, d)) != PIPO_OK) break;
      LAUNCH(launch_f32_to_f16(buf, ctx->lnf_g, d, st));
      if (!llama) {
        if ((s = draw(buf, 0, 3, 1, 0.1, d)) != PIPO_OK) break;
        LAUNCH(launch_f32_to_f16(buf, ctx->lnf_b, d, st));
      }
    } while (0);
    CK(cudaStreamSynchronize(st));
    cudaFree(buf);
    ctx->hbm_bytes -= std::max(ntok, npos) * 4;
    if (s == PIPO_OK) ctx->embed_loaded = true;
    return s;
  }
  if (layer < 0 || layer >= ctx->l) return set_err(PIPO_E_INVALID_ARG, "layer index out of range");
  TRY(drain_prefetch(ctx));
  // draw + quantize/tile into a device blob, then place it in its tier
  uint8_t* blob = nullptr;
  const bool direct = ctx->weight_tier == PIPO_TIER_DEVICE;
  if (direct) {
    blob = ctx->dev_store + (int64_t)layer * ctx->layer_bytes;
  } else {
    TRY(dev_alloc(ctx, &blob, ctx->layer_bytes));
  }
  int64_t big = 0;
  for (int m = 0; m < M_COUNT; ++m) big = std::max(big, ctx->lay.mat[m].N * ctx->lay.mat[m].K);
  (void)F;
  float* buf = nullptr;
  pipo_status s = dev_alloc(ctx, &buf, big * 4);
  const uint32_t slot = (uint32_t)layer + 1;
  const int vkinds[V_COUNT] = {2, 1, 1, 1, 2, 1, 1, 1};
  const double vparams[V_COUNT] = {0.1, 0.1, 0.02, 0.02, 0.1, 0.1, 0.02, 0.02};
  const uint32_t vtids[V_COUNT] = {0, 1, 3, 5, 6, 7, 9, 11};
  const uint32_t mtids[M_COUNT] = {2, 4, 8, 10};
  int64_t mrows[M_COUNT], mcols[M_COUNT];
  for (int m = 0; m < M_COUNT; ++m) { mrows[m] = ctx->lay.mat[m].N; mcols[m] = ctx->lay.mat[m].K; }
  if (s == PIPO_OK) {
    CK(cudaMemsetAsync(blob, 0, (size_t)ctx->layer_bytes, st));
    CK(cudaMemsetAsync(ctx->quant_bad, 0, 4, st));
    for (int v = 0; v < V_COUNT && s == PIPO_OK; ++v) {
      if (ctx->lay.vec_len[v] == 0) continue;   // LLaMA: no biases / betas
      s = draw(buf, slot, vtids[v], vkinds[v], vparams[v], ctx->lay.vec_len[v]);
      if (s == PIPO_OK)
        LAUNCH(launch_f32_to_f16(buf, reinterpret_cast<__half*>(blob + ctx->lay.vec_off[v]), ctx->lay.vec_len[v], st));
    }
    for (int m = 0; m < M_COUNT && s == PIPO_OK; ++m) {
      s = draw(buf, slot, mtids[m], 0, 0.02, mrows[m] * mcols[m]);
      if (s != PIPO_OK) break;
      uint8_t* dst = blob + ctx->lay.mat_off[m];
      if (ctx->lay.glu && m == M_FC1) {
        // tile-interleaved [gate; up] (layout.h): tile 2p <- gate rows 128p.., 2p+1 <- up rows F+128p..
        const MatLayout& ml = ctx->lay.mat[m];
        const int64_t Fh = mrows[m] / 2, tile_bytes = ml.n_kb * ml.block_bytes;
        for (int64_t t = 0; t < ml.n_rt; ++t) {
          const float* src = buf + ((t & 1) * Fh + (t >> 1) * 128) * mcols[m];
          if (ctx->wfmt == PIPO_W_INT4_G64)
            LAUNCH(launch_quantize(src, 128, mcols[m], nullptr, nullptr, dst + t * tile_bytes, ctx->quant_bad, st));
          else
            LAUNCH(launch_tile_fp16(src, 128, mcols[m], dst + t * tile_bytes, st));
        }
      } else if (ctx->wfmt == PIPO_W_INT4_G64) {
        LAUNCH(launch_quantize(buf, mrows[m], mcols[m], nullptr, nullptr, dst, ctx->quant_bad, st));
      } else {
        LAUNCH(launch_tile_fp16(buf, mrows[m], mcols[m], dst, st));
      }
    }
  }
  if (s == PIPO_OK && !direct) {
    if (sharded(ctx)) {   // sharded streaming: this rank's range only
      CK(cudaMemcpyAsync(ctx->host_store + (int64_t)layer * ctx->shard_bytes,
                         blob + (int64_t)ctx->shard_rank * ctx->shard_bytes, (size_t)ctx->shard_bytes,
                         cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
    } else if (ctx->weight_tier == PIPO_TIER_HOST) {
      CK(cudaMemcpyAsync(ctx->host_store + (int64_t)layer * ctx->layer_bytes, blob, (size_t)ctx->layer_bytes,
                         cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
    } else {
      std::vector<uint8_t> tmp((size_t)ctx->layer_bytes);
      CK(cudaMemcpyAsync(tmp.data(), blob, tmp.size(), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      s = disk_write_layer(ctx, layer, tmp.data());
      if (s != PIPO_OK) set_err(s, "writing the layer blob file failed");
    }
  }
  CK(cudaStreamSynchronize(st));
  if (buf) { cudaFree(buf); ctx->hbm_bytes -= big * 4; }
  if (!direct && blob) { cudaFree(blob); ctx->hbm_bytes -= ctx->layer_bytes; }
  if (s == PIPO_OK) ctx->layer_loaded[layer] = 1;
  return s;
}

pipo_status prefill(pipo_ctx* ctx, const int32_t* tokens, int32_t b, int32_t P, int32_t* next, float* logits) {
  CHECK_CTX();
  if (!tokens || !next) return set_err(PIPO_E_INVALID_ARG, "NULL tokens/next");
  if (b <= 0 || b > ctx->max_b) return set_err(PIPO_E_INVALID_ARG, "batch exceeds max_batch");
  if (P <= 0 || P >= ctx->max_s) return set_err(PIPO_E_INVALID_ARG, "prompt length must be in [1, max_seq)");
  TRY(check_ready(ctx));
  CK(cudaSetDevice(ctx->cfg.device));
  const double t0 = now_s();
  // a new batch: wait until every in-flight KV save of the previous batch is done
  CK(cudaStreamSynchronize(ctx->s_save));
  ctx->b_cur = b;
  ctx->past = 0;
  ctx->have_batch = false;
  TRY(stage_ids(ctx, tokens, (int64_t)b * P));
  TRY(forward(ctx, b, P, 0, logits != nullptr));
  TRY(finish_call(ctx, b, P, next, logits));
  ctx->past = P;
  ctx->have_batch = true;
  ctx->prefill_calls++;
  ctx->tokens += b;
  ctx->prefill_s += now_s() - t0;
  ctx->ttft_s = now_s() - t0;
  return PIPO_OK;
}

static pipo_status decode_common(pipo_ctx* ctx) {
  if (!ctx->have_batch) return set_err(PIPO_E_STATE, "decode_step before prefill");
  if (ctx->past + 1 > ctx->max_s) return set_err(PIPO_E_INVALID_ARG, "KV capacity max_seq exceeded");
  return PIPO_OK;
}

pipo_status decode_step(pipo_ctx* ctx, const int32_t* tokens, int32_t* next, float* logits) {
  CHECK_CTX();
  if (!tokens || !next) return set_err(PIPO_E_INVALID_ARG, "NULL tokens/next");
  TRY(decode_common(ctx));
  CK(cudaSetDevice(ctx->cfg.device));
  const double t0 = now_s();
  TRY(window_mark(ctx, true));
  TRY(stage_ids(ctx, tokens, ctx->b_cur));
  TRY(forward(ctx, ctx->b_cur, 1, ctx->past, logits != nullptr));
  TRY(window_mark(ctx, false));
  TRY(finish_call(ctx, ctx->b_cur, 1, next, logits));
  ctx->past += 1;
  ctx->decode_steps++;
  ctx->tokens += ctx->b_cur;
  ctx->decode_s += now_s() - t0;
  return PIPO_OK;
}

pipo_status decode_step_dev(pipo_ctx* ctx, const int32_t* tokens_dev, int32_t* next_dev) {
  CHECK_CTX();
  if (!tokens_dev || !next_dev) return set_err(PIPO_E_INVALID_ARG, "NULL device buffers");
  TRY(decode_common(ctx));
  CK(cudaSetDevice(ctx->cfg.device));
  const double t0 = now_s();
  TRY(window_mark(ctx, true));
  CK(cudaMemcpyAsync(ctx->ids, tokens_dev, (size_t)ctx->b_cur * 4, cudaMemcpyDeviceToDevice, ctx->s_comp));
  TRY(forward(ctx, ctx->b_cur, 1, ctx->past, false));
  CK(cudaMemcpyAsync(next_dev, ctx->next, (size_t)ctx->b_cur * 4, cudaMemcpyDeviceToDevice, ctx->s_comp));
  TRY(window_mark(ctx, false));
  ctx->past += 1;
  ctx->decode_steps++;
  ctx->tokens += ctx->b_cur;
  ctx->decode_s += now_s() - t0;   // enqueue time only; device time is in stats.window_s
  return PIPO_OK;
}

pipo_status pipeline_stats(pipo_ctx* ctx, pipo_stats* out) {
  CHECK_CTX();
  if (!out) return set_err(PIPO_E_INVALID_ARG, "out is NULL");
  CK(cudaSetDevice(ctx->cfg.device));
  CK(cudaDeviceSynchronize());
  pipo_stats s{};
  s.prefill_calls = ctx->prefill_calls;
  s.decode_steps = ctx->decode_steps;
  s.tokens_generated = ctx->tokens;
  s.prefill_s = ctx->prefill_s;
  s.decode_s = ctx->decode_s;
  s.ttft_s = ctx->ttft_s;
  s.h2d_bytes = ctx->h2d_bytes;
  s.d2h_bytes = ctx->d2h_bytes;
  s.kernel_launches = ctx->launches;
  s.hbm_bytes = ctx->hbm_bytes;
  s.pinned_host_bytes = ctx->pinned_bytes;
  s.numa_node = ctx->numa_node;
  s.timeline_truncated = ctx->timeline_truncated ? 1 : 0;
  s.numa_local_frac = -1.0;
  if (ctx->numa_node >= 0 && ctx->host_store)
    s.numa_local_frac = numa_local_fraction(ctx->host_store, sharded(ctx) ? (int64_t)ctx->l * ctx->shard_bytes
                                                                           : (int64_t)ctx->l * ctx->layer_bytes,
                                            ctx->numa_node, 64);
  if (ctx->win_open && ctx->win_closed) {
    float w = 0;
    CK(cudaEventElapsedTime(&w, ctx->win_start, ctx->win_end));
    s.window_s = w * 1e-3;
    std::vector<std::pair<double, double>> lanes[4], all;
    double copy_bytes = 0;
    for (const Span& sp : ctx->spans) {
      float a = 0, b = 0;
      CK(cudaEventElapsedTime(&a, ctx->win_start, sp.a));
      CK(cudaEventElapsedTime(&b, ctx->win_start, sp.b));
      double lo = std::max(0.0, (double)a), hi = std::min((double)w, (double)b);
      if (hi <= lo) continue;
      lanes[sp.lane].push_back({lo, hi});
      if (sp.lane != 2) all.push_back({lo, hi});
      if (sp.lane == 0 && b > a) copy_bytes += sp.bytes * (hi - lo) / (b - a);
    }
    const double copy_t = union_len(lanes[0]);
    if (w > 0) {
      s.copy_busy = copy_t / w;
      s.kernel_busy = union_len(lanes[1]) / w;
      s.union_busy = union_len(all) / w;
    }
    s.h2d_gbs = copy_t > 0 ? copy_bytes / (copy_t * 1e-3) / 1e9 : 0;
    if (s.window_s > 0 && ctx->b_cur > 0) s.decode_tokens_per_s = (double)ctx->b_cur * ctx->decode_steps / s.window_s;
  } else if (ctx->decode_s > 0) {
    s.decode_tokens_per_s = (double)ctx->b_cur * ctx->decode_steps / ctx->decode_s;
  }
  *out = s;
  return PIPO_OK;
}

pipo_status pipo_set_flags(pipo_ctx* ctx, uint32_t flags) {
  CHECK_CTX();
  CK(cudaSetDevice(ctx->cfg.device));
  CK(cudaDeviceSynchronize());   // spans / kernel records in flight keep their events
  ctx->timeline = (flags & PIPO_F_TIMELINE) != 0;
  ctx->kprof = (flags & PIPO_F_KPROF) != 0;
  ctx->cfg.flags = flags;
  return PIPO_OK;
}

pipo_status pipeline_stats_reset(pipo_ctx* ctx) {
  CHECK_CTX();
  CK(cudaSetDevice(ctx->cfg.device));
  CK(cudaDeviceSynchronize());
  ctx->spans.clear();
  ctx->krecs.clear();
  ctx->ev_used = 0;
  ctx->win_open = false;
  ctx->win_closed = false;
  ctx->timeline_truncated = false;
  ctx->timeline = (ctx->cfg.flags & PIPO_F_TIMELINE) != 0;
  ctx->kprof = (ctx->cfg.flags & PIPO_F_KPROF) != 0;
  ctx->launches = 0;
  ctx->prefill_calls = ctx->decode_steps = ctx->tokens = 0;
  ctx->prefill_s = ctx->decode_s = 0;
  ctx->h2d_bytes = ctx->d2h_bytes = 0;
  return PIPO_OK;
}

pipo_status pipo_kernel_stats(pipo_ctx* ctx, int32_t cls, pipo_kstats* out) {
  CHECK_CTX();
  if (!out || cls < 0 || cls >= PIPO_K_COUNT) return set_err(PIPO_E_INVALID_ARG, "bad kernel class");
  CK(cudaSetDevice(ctx->cfg.device));
  CK(cudaDeviceSynchronize());
  pipo_kstats k{};
  for (const KRec& r : ctx->krecs) {
    if (r.cls != cls) continue;
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, r.a, r.b));
    k.units++;
    k.ms += ms;
    k.bytes += r.bytes;
    k.flops += r.flops;
  }
  *out = k;
  return PIPO_OK;
}

void* pipo_stream(pipo_ctx* ctx, int32_t which) {
  if (!ctx) return nullptr;
  return which == 0 ? (void*)ctx->s_comp : which == 1 ? (void*)ctx->s_copy : (void*)ctx->s_save;
}

// ---- hooks ---------------------------------------------------------------------
pipo_status pipo_quantize_int4_g64(const float* w, int64_t rows, int64_t cols, uint8_t* codes, uint16_t* scales) {
  if (!w || !codes || !scales || rows <= 0 || cols <= 0 || cols % 64)
    return set_err(PIPO_E_INVALID_ARG, "bad quantize arguments");
  if (!quantize_canonical(w, rows, cols, codes, scales))
    return set_err(PIPO_E_INVALID_ARG, "non-finite weight or fp16-overflowing group scale");
  return PIPO_OK;
}

pipo_status pipo_quantize_int4_g64_gpu(pipo_ctx* ctx, const float* w, int64_t rows, int64_t cols, uint8_t* codes,
                                       uint16_t* scales) {
  CHECK_CTX();
  if (!w || !codes || !scales || rows <= 0 || cols <= 0 || cols % 64)
    return set_err(PIPO_E_INVALID_ARG, "bad quantize arguments");
  CK(cudaSetDevice(ctx->cfg.device));
  float* dw = nullptr; uint8_t* dc = nullptr; uint16_t* ds = nullptr;
  TRY(dev_alloc(ctx, &dw, rows * cols * 4));
  TRY(dev_alloc(ctx, &dc, rows * cols / 2));
  TRY(dev_alloc(ctx, &ds, rows * cols / 64 * 2));
  cudaStream_t st = ctx->s_comp;
  CK(cudaMemcpyAsync(dw, w, (size_t)(rows * cols * 4), cudaMemcpyHostToDevice, st));
  CK(cudaMemsetAsync(ctx->quant_bad, 0, 4, st));
  LAUNCH(launch_quantize(dw, rows, cols, dc, ds, nullptr, ctx->quant_bad, st));
  int bad = 0;
  CK(cudaMemcpyAsync(codes, dc, (size_t)(rows * cols / 2), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(scales, ds, (size_t)(rows * cols / 64 * 2), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&bad, ctx->quant_bad, 4, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  cudaFree(dw); cudaFree(dc); cudaFree(ds);
  ctx->hbm_bytes -= rows * cols * 4 + rows * cols / 2 + rows * cols / 64 * 2;
  if (bad) return set_err(PIPO_E_INVALID_ARG, "non-finite weight or fp16-overflowing group scale");
  return PIPO_OK;
}

pipo_status pipo_unpack_int4_g64(pipo_ctx* ctx, const uint8_t* codes, const uint16_t* scales, int64_t rows,
                                 int64_t cols, uint16_t* out) {
  CHECK_CTX();
  if (!codes || !scales || !out || rows <= 0 || cols <= 0 || cols % 64)
    return set_err(PIPO_E_INVALID_ARG, "bad unpack arguments");
  CK(cudaSetDevice(ctx->cfg.device));
  uint8_t* dc = nullptr; uint16_t* ds = nullptr; __half* dout = nullptr;
  TRY(dev_alloc(ctx, &dc, rows * cols / 2));
  TRY(dev_alloc(ctx, &ds, rows * cols / 64 * 2));
  TRY(dev_alloc(ctx, &dout, rows * cols * 2));
  cudaStream_t st = ctx->s_comp;
  CK(cudaMemcpyAsync(dc, codes, (size_t)(rows * cols / 2), cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(ds, scales, (size_t)(rows * cols / 64 * 2), cudaMemcpyHostToDevice, st));
  LAUNCH(launch_unpack_int4(dc, ds, rows, cols, dout, st));
  CK(cudaMemcpyAsync(out, dout, (size_t)(rows * cols * 2), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  cudaFree(dc); cudaFree(ds); cudaFree(dout);
  ctx->hbm_bytes -= rows * cols / 2 + rows * cols / 64 * 2 + rows * cols * 2;
  return PIPO_OK;
}

pipo_status pipo_linear(pipo_ctx* ctx, int32_t wfmt, int32_t path, const uint16_t* x, const float* w,
                        const float* bias, int32_t M, int32_t N, int32_t K, float* y) {
  CHECK_CTX();
  if (!x || !w || !y || M <= 0 || N <= 0 || K <= 0 || K % 64 || (wfmt != 0 && wfmt != 1) || path < 0 || path > 9)
    return set_err(PIPO_E_INVALID_ARG, "bad linear arguments");
  CK(cudaSetDevice(ctx->cfg.device));
  const MatLayout ml = mat_layout(N, K, wfmt);
  std::vector<uint8_t> tiled((size_t)ml.bytes);
  if (wfmt == 1) {
    if (!quantize_tiled(w, N, K, tiled.data())) return set_err(PIPO_E_INVALID_ARG, "non-finite weight");
  } else {
    tile_fp16(w, N, K, tiled.data());
  }
  std::vector<uint16_t> bh;
  if (bias) {
    bh.resize(N);
    for (int i = 0; i < N; ++i) bh[i] = f32_to_f16_rne(bias[i]);
  }
  uint8_t* dw = nullptr; __half* dx = nullptr; __half* db = nullptr; float* dy = nullptr;
  TRY(dev_alloc(ctx, &dw, ml.bytes));
  TRY(dev_alloc(ctx, &dx, (int64_t)M * K * 2));
  TRY(dev_alloc(ctx, &dy, (int64_t)M * N * 4));
  if (bias) TRY(dev_alloc(ctx, &db, (int64_t)N * 2));
  cudaStream_t st = ctx->s_comp;
  CK(cudaMemcpyAsync(dw, tiled.data(), tiled.size(), cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(dx, x, (size_t)M * K * 2, cudaMemcpyHostToDevice, st));
  if (bias) CK(cudaMemcpyAsync(db, bh.data(), (size_t)N * 2, cudaMemcpyHostToDevice, st));
  LinearArgs la;
  la.x = dx; la.w = dw; la.wfmt = wfmt; la.M = M; la.N = N; la.K = K;
  la.ws = ctx->ws; la.ws_floats = ctx->ws_floats; la.counters = ctx->counters; la.n_counters = ctx->n_counters;
  la.num_sms = ctx->num_sms;
  la.epi.kind = EPI_F32; la.epi.bias = db; la.epi.M = M; la.epi.N = N; la.epi.y = dy; la.epi.ldy = N;
  LAUNCH(launch_linear(la, path, ctx->gemv_max_m, st));
  CK(cudaMemcpyAsync(y, dy, (size_t)M * N * 4, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  cudaFree(dw); cudaFree(dx); cudaFree(dy);
  if (db) cudaFree(db);
  ctx->hbm_bytes -= ml.bytes + (int64_t)M * K * 2 + (int64_t)M * N * 4 + (bias ? N * 2 : 0);
  return PIPO_OK;
}

pipo_status pipo_bench_linear(pipo_ctx* ctx, int32_t wfmt, int32_t path, int32_t M, int32_t N, int32_t K,
                              int32_t iters, double* us) {
  CHECK_CTX();
  if (!us || M <= 0 || N <= 0 || K <= 0 || K % 64 || iters <= 0 || (wfmt != 0 && wfmt != 1) || path < 0 || path > 9)
    return set_err(PIPO_E_INVALID_ARG, "bad bench arguments");
  CK(cudaSetDevice(ctx->cfg.device));
  const MatLayout ml = mat_layout(N, K, wfmt);
  uint8_t* dw = nullptr; __half* dx = nullptr; float* dy = nullptr; float* tmp = nullptr;
  TRY(dev_alloc(ctx, &dw, ml.bytes));
  TRY(dev_alloc(ctx, &dx, (int64_t)M * K * 2));
  TRY(dev_alloc(ctx, &dy, (int64_t)M * N * 4));
  TRY(dev_alloc(ctx, &tmp, std::max<int64_t>((int64_t)N * K, (int64_t)M * K) * 4));
  cudaStream_t st = ctx->s_comp;
  LAUNCH(launch_synth(tmp, 0, (int64_t)N * K, synth_key(7, 1, 2), 0, synth_scale(0, 0.02), st));
  if (wfmt == 1) LAUNCH(launch_quantize(tmp, N, K, nullptr, nullptr, dw, ctx->quant_bad, st));
  else LAUNCH(launch_tile_fp16(tmp, N, K, dw, st));
  LAUNCH(launch_synth(tmp, 0, (int64_t)M * K, synth_key(7, 1, 3), 0, synth_scale(0, 1.0), st));
  LAUNCH(launch_f32_to_f16(tmp, dx, (int64_t)M * K, st));
  LinearArgs la;
  la.x = dx; la.w = dw; la.wfmt = wfmt; la.M = M; la.N = N; la.K = K;
  la.ws = ctx->ws; la.ws_floats = ctx->ws_floats; la.counters = ctx->counters; la.n_counters = ctx->n_counters;
  la.num_sms = ctx->num_sms;
  la.epi.kind = EPI_F32; la.epi.M = M; la.epi.N = N; la.epi.y = dy; la.epi.ldy = N;
  // Cold-HBM timing: successive launches read different copies of the weights whose
  // total exceeds the 126 MB L2 (>= 384 MB), so no launch finds its weights in L2 —
  // as in the pipeline, where every layer's weights are fresh.  PIPO_BENCH_HOT=1
  // re-reads one copy (L2-warm upper bound).
  const bool hot = getenv("PIPO_BENCH_HOT") && atoi(getenv("PIPO_BENCH_HOT"));
  const int n_copies = hot ? 1 : (int)std::min<int64_t>(64, std::max<int64_t>(2, ((384ll << 20) + ml.bytes - 1) / ml.bytes));
  uint8_t* wcopies = nullptr;
  if (n_copies > 1) {
    TRY(dev_alloc(ctx, &wcopies, ml.bytes * (n_copies - 1)));
    for (int c = 0; c < n_copies - 1; ++c)
      CK(cudaMemcpyAsync(wcopies + (int64_t)c * ml.bytes, dw, ml.bytes, cudaMemcpyDeviceToDevice, st));
  }
  auto wcopy = [&](int i) { const int c = i % n_copies; return c == 0 ? dw : wcopies + (int64_t)(c - 1) * ml.bytes; };
  if (getenv("PIPO_WS_DEBUG")) CK(cudaMemsetAsync(ctx->ws + (15ll << 20), 0, 2 * 148 * 16 * 8, st));
  for (int i = 0; i < n_copies; ++i) {   // warm-up (touches every copy once)
    la.w = wcopy(i);
    LAUNCH(launch_linear(la, path, ctx->gemv_max_m, st));
  }
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0, st));
  const bool stamps = getenv("PIPO_WS_DEBUG") && (atoi(getenv("PIPO_WS_DEBUG")) & 128);
  for (int i = 0; i < iters; ++i) {
    la.w = wcopy(i + 1);
    if (stamps && i == iters - 1) {   // reduce window of the last launch: min-start / max-end
      const uint64_t init[2] = {~0ull, 0ull};
      CK(cudaMemcpyAsync(ctx->ws + (15ll << 20) + 148 * 16 * 2, init, 16, cudaMemcpyHostToDevice, st));
    }
    LAUNCH(launch_linear(la, path, ctx->gemv_max_m, st));
  }
  CK(cudaEventRecord(e1, st));
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0); cudaEventDestroy(e1);
  if (getenv("PIPO_WS_DEBUG") && (atoi(getenv("PIPO_WS_DEBUG")) & 128) && path == 5) {
    // globaltimer stamps of the last launch: 9 entry, 10 after setup, 11 MMA done,
    // 12 epilogue done, 13 exit; reduce kernel first start / last end
    std::vector<uint64_t> ts(148 * 16 + 2);
    CK(cudaMemcpy(ts.data(), ctx->ws + (15ll << 20), ts.size() * 8, cudaMemcpyDeviceToHost));
    uint64_t t0 = ~0ull;
    for (int c = 0; c < 148; ++c) if (ts[c * 16 + 9]) t0 = std::min(t0, ts[c * 16 + 9]);
    const char* nm[8] = {"entry", "setup", "mma_end", "epi_end", "syncd", "dealloc", "tail_end", "tail1"};
    for (int k = 3; k <= 15; ++k) {
      if (k == 8) continue;
      std::vector<double> v;
      for (int c = 0; c < 148; ++c) if (ts[c * 16 + k] >= t0 && ts[c * 16 + k] - t0 < 10000000ull) v.push_back((ts[c * 16 + k] - t0) * 1e-3);
      std::sort(v.begin(), v.end());
      if (!v.empty()) fprintf(stderr, "tm-stamp %-8s min %7.2f med %7.2f max %7.2f us (n=%zu)\n", k == 7 ? "tail0" : k == 3 ? "w0_wait" : k == 4 ? "w0_loop" : k == 5 ? "w1_wait" : k == 6 ? "w1_loop" : nm[k - 9], v.front(), v[v.size() / 2], v.back(), v.size());
    }
    {   // same-CTA ordering check: exit (after the final __syncthreads) minus MMA / epilogue end
      double lo = 1e30, hi = -1e30, lo2 = 1e30;
      for (int c = 0; c < 148; ++c) {
        if (!ts[c * 16 + 13] || !ts[c * 16 + 11]) continue;
        const double dm = (double)(int64_t)(ts[c * 16 + 13] - ts[c * 16 + 11]) * 1e-3;
        const double de = (double)(int64_t)(ts[c * 16 + 13] - ts[c * 16 + 12]) * 1e-3;
        lo = std::min(lo, dm); hi = std::max(hi, dm); lo2 = std::min(lo2, de);
      }
      fprintf(stderr, "tm-stamp per-CTA exit-mma_end min %.2f max %.2f us, exit-epi_end min %.2f us\n", lo, hi, lo2);
      double fx = 0, bm = 0;
      for (int c = 0; c < 148; ++c) { fx += (double)ts[c * 16] / 148; bm += (double)(int64_t)ts[c * 16 + 1] / 148; }
      fprintf(stderr, "tm-clk fixup %.0f cycles, barrier-after-MMA-end %.0f cycles (avg over CTAs)\n", fx, bm);
    }
    fprintf(stderr, "reduce first start %.2f last end %.2f us\n", (double)(int64_t)(ts[148 * 16] - t0) * 1e-3, (double)(int64_t)(ts[148 * 16 + 1] - t0) * 1e-3);
  } else if (getenv("PIPO_WS_DEBUG") && (atoi(getenv("PIPO_WS_DEBUG")) & 128) && path == 9) {
    // pair kernel stamps of the last launch (k_gemm_pair.cu): relative to the first entry
    std::vector<uint64_t> ts(148 * 16);
    CK(cudaMemcpy(ts.data(), ctx->ws + (15ll << 20), ts.size() * 8, cudaMemcpyDeviceToHost));
    uint64_t t0 = ~0ull;
    for (int c = 0; c < 148; ++c) if (ts[c * 16]) t0 = std::min(t0, ts[c * 16]);
    const char* nm[13] = {"entry", "setup", "prod_end", "mma_end", "unpk_end", "last_acc", "flags_ok", "epi_end",
                          "exit", "first_raw", "units", "lastkind", "seg0_epi"};
    for (int k = 0; k < 13; ++k) {
      std::vector<double> v;
      for (int c = 0; c < 148; ++c) {
        if (k == 10 || k == 11) { v.push_back((double)ts[c * 16 + k]); continue; }
        if (ts[c * 16 + k] >= t0 && ts[c * 16 + k] - t0 < 10000000ull) v.push_back((ts[c * 16 + k] - t0) * 1e-3);
      }
      std::sort(v.begin(), v.end());
      if (!v.empty()) fprintf(stderr, "pair-stamp %-9s min %8.2f med %8.2f max %8.2f (n=%zu)\n", nm[k], v.front(), v[v.size() / 2], v.back(), v.size());
    }
    std::vector<uint64_t> wc(148 * 16);
    CK(cudaMemcpy(wc.data(), ctx->ws + (15ll << 20) + 148 * 16 * 2, wc.size() * 8, cudaMemcpyDeviceToHost));
    const char* wn[13] = {"prod slot_empty", "prod total", "mma a_full", "mma acc_empty", "mma total",
                          "unpk slot_full", "unpk a_empty", "unpk wait_st", "unpk total", "xld x_empty", "xld wait_group",
                          "xld total", "unpk x_full"};
    fprintf(stderr, "pair-waits (kcycles, avg over CTAs that ran the role):");
    for (int k = 0; k < 13; ++k) {
      double sum = 0; int n = 0;
      for (int c = 0; c < 148; ++c) if (wc[c * 16 + k]) { sum += wc[c * 16 + k]; ++n; }
      fprintf(stderr, " | %s %.1f", wn[k], n ? sum / n / 1e3 : 0.0);
    }
    fprintf(stderr, "\n");
  } else if (getenv("PIPO_WS_DEBUG") && (atoi(getenv("PIPO_WS_DEBUG")) & 32) && path == 5) {
    std::vector<uint64_t> wt(148 * 16);
    CK(cudaMemcpy(wt.data(), ctx->ws + (15ll << 20), wt.size() * 8, cudaMemcpyDeviceToHost));
    double avg[11] = {0};
    for (int c = 0; c < 148; ++c)
      for (int k = 0; k < 11; ++k) avg[k] += wt[c * 16 + k] / 148.0;
    fprintf(stderr, "tm-waits(kcycles): prod raw_empty %.1f | mma a_full %.1f x_full %.1f | unpack raw_full %.1f a_empty %.1f wait_st %.1f total %.1f | xprod x_empty %.1f | mma total %.1f\n",
            avg[0] / 1e3, avg[2] / 1e3, avg[3] / 1e3, avg[4] / 1e3, avg[5] / 1e3, avg[9] / 1e3, avg[10] / 1e3, avg[6] / 1e3, avg[8] / 1e3);
  } else if (getenv("PIPO_WS_DEBUG") && (atoi(getenv("PIPO_WS_DEBUG")) & 32)) {
    std::vector<uint64_t> ts(148 * 8);
    CK(cudaMemcpy(ts.data(), ctx->ws + (15ll << 20), ts.size() * 8, cudaMemcpyDeviceToHost));
    uint64_t t0 = ~0ull;
    for (int c = 0; c < 148; ++c) if (ts[c * 8]) t0 = std::min(t0, ts[c * 8]);
    for (int k = 0; k < 8; ++k) {
      std::vector<double> v;
      for (int c = 0; c < 148; ++c) if (ts[c * 8 + k] >= t0 && ts[c * 8 + k] - t0 < 10000000ull) v.push_back((ts[c * 8 + k] - t0) * 1e-3);
      std::sort(v.begin(), v.end());
      if (!v.empty()) fprintf(stderr, "ws-stamp %d: min %.2f med %.2f max %.2f us (n=%zu)\n", k, v.front(), v[v.size() / 2], v.back(), v.size());
    }
  }
  cudaFree(dw); cudaFree(dx); cudaFree(dy); cudaFree(tmp);
  if (wcopies) cudaFree(wcopies);
  ctx->hbm_bytes -= ml.bytes * n_copies + (int64_t)M * K * 2 + (int64_t)M * N * 4 + std::max<int64_t>((int64_t)N * K, (int64_t)M * K) * 4;
  *us = ms * 1e3 / iters;
  return PIPO_OK;
}

pipo_status pipo_probe_bulk(pipo_ctx* ctx, int32_t chunk, int32_t stages, int32_t streams, double* gbs) {
  CHECK_CTX();
  if (!gbs || chunk <= 0 || chunk % 16 || stages <= 0 || streams <= 0) return set_err(PIPO_E_INVALID_ARG, "bad probe arguments");
  CK(cudaSetDevice(ctx->cfg.device));
  const int ctas = ctx->num_sms;
  const int64_t per = (int64_t)(512ll << 20) / ctas / (chunk * (int64_t)streams) * chunk * streams;
  uint8_t* buf = nullptr;
  uint32_t* sink = nullptr;
  TRY(dev_alloc(ctx, &buf, per * ctas));
  TRY(dev_alloc(ctx, &sink, 4));
  cudaStream_t st = ctx->s_comp;
  CK(cudaMemsetAsync(buf, 1, (size_t)(per * ctas), st));
  LAUNCH(launch_bulk_probe(buf, per, chunk, stages, streams, ctas, sink, st));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0, st));
  for (int i = 0; i < 5; ++i) LAUNCH(launch_bulk_probe(buf, per, chunk, stages, streams, ctas, sink, st));
  CK(cudaEventRecord(e1, st));
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0); cudaEventDestroy(e1);
  cudaFree(buf); cudaFree(sink);
  ctx->hbm_bytes -= per * ctas + 4;
  *gbs = 5.0 * per * ctas / (ms * 1e-3) / 1e9;
  return PIPO_OK;
}

pipo_status pipo_bench_attention(pipo_ctx* ctx, int32_t b, int32_t L, int32_t d, int32_t n_heads, int32_t n_kv_heads,
                                 int32_t variant, int32_t iters, double* us) {
  CHECK_CTX();
  if (n_kv_heads == 0) n_kv_heads = n_heads;
  if (!us || b <= 0 || L <= 0 || d <= 0 || n_heads <= 0 || d % n_heads || iters <= 0 || n_kv_heads < 0 ||
      n_heads % n_kv_heads)
    return set_err(PIPO_E_INVALID_ARG, "bad bench arguments");
  CK(cudaSetDevice(ctx->cfg.device));
  const int dkv = d / n_heads * n_kv_heads;
  const int64_t nq = (int64_t)b * d, nkv = (int64_t)L * b * dkv;
  // cold-HBM timing as in the pipeline (every layer's KV is fresh): launches rotate over
  // copies of K/V totalling >= 384 MB (more than the 126 MB L2)
  const int copies = (int)std::max<int64_t>(1, std::min<int64_t>(8, ((384ll << 20) + 4 * nkv - 1) / (4 * nkv)));
  __half *dq = nullptr, *dk = nullptr, *dv = nullptr, *dout = nullptr;
  float* tmp = nullptr;
  TRY(dev_alloc(ctx, &dq, nq * 2));
  TRY(dev_alloc(ctx, &dk, nkv * 2 * copies));
  TRY(dev_alloc(ctx, &dv, nkv * 2 * copies));
  TRY(dev_alloc(ctx, &dout, nq * 2));
  TRY(dev_alloc(ctx, &tmp, std::min<int64_t>(nkv, 64ll << 20) * 4));
  cudaStream_t st = ctx->s_comp;
  const int64_t chunk = std::min<int64_t>(nkv, 64ll << 20);
  for (int w = 0; w < 3; ++w) {
    __half* dst = w == 0 ? dq : (w == 1 ? dk : dv);
    const int64_t n = w == 0 ? nq : nkv;
    for (int64_t off = 0; off < n; off += chunk) {
      const int64_t c = std::min(chunk, n - off);
      LAUNCH(launch_synth(tmp, off, c, synth_key(9, 9, w), 0, synth_scale(0, 1.0), st));
      LAUNCH(launch_f32_to_f16(tmp, dst + off, c, st));
    }
  }
  for (int c = 1; c < copies; ++c) {
    CK(cudaMemcpyAsync(dk + c * nkv, dk, (size_t)nkv * 2, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(dv + c * nkv, dv, (size_t)nkv * 2, cudaMemcpyDeviceToDevice, st));
  }
  AttnArgs aa;
  aa.q = dq; aa.kc = dk; aa.vc = dv; aa.o = dout; aa.b = b; aa.n = 1; aa.past = L - 1; aa.d = d;
  aa.n_heads = n_heads; aa.kv_b = b; aa.ws = ctx->ws; aa.ws_floats = ctx->ws_floats; aa.num_sms = ctx->num_sms;
  aa.dkv = dkv; aa.group = n_heads / n_kv_heads;
  aa.use_cuda_cores = variant;
  for (int c = 0; c < copies; ++c) {
    aa.kc = dk + c * nkv; aa.vc = dv + c * nkv;
    LAUNCH(launch_attention_decode(aa, st));
  }
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0, st));
  for (int i = 0; i < iters; ++i) {
    aa.kc = dk + (i % copies) * nkv; aa.vc = dv + (i % copies) * nkv;
    LAUNCH(launch_attention_decode(aa, st));
  }
  CK(cudaEventRecord(e1, st));
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0); cudaEventDestroy(e1);
  cudaFree(dq); cudaFree(dk); cudaFree(dv); cudaFree(dout); cudaFree(tmp);
  ctx->hbm_bytes -= nq * 4 + nkv * 4 * copies + std::min<int64_t>(nkv, 64ll << 20) * 4;
  *us = ms * 1e3 / iters;
  return PIPO_OK;
}

pipo_status pipo_bench_attention_prefill(pipo_ctx* ctx, int32_t b, int32_t n, int32_t d, int32_t n_heads,
                                         int32_t n_kv_heads, int32_t variant, int32_t iters, double* us) {
  CHECK_CTX();
  if (n_kv_heads == 0) n_kv_heads = n_heads;
  if (!us || b <= 0 || n <= 0 || d <= 0 || n_heads <= 0 || d % n_heads || iters <= 0 || n_kv_heads < 0 ||
      n_heads % n_kv_heads)
    return set_err(PIPO_E_INVALID_ARG, "bad bench arguments");
  CK(cudaSetDevice(ctx->cfg.device));
  const int dkv = d / n_heads * n_kv_heads;
  const int64_t nq = (int64_t)b * n * d, nkv = (int64_t)n * b * dkv;
  __half *dq = nullptr, *dk = nullptr, *dv = nullptr, *dout = nullptr;
  float* tmp = nullptr;
  TRY(dev_alloc(ctx, &dq, nq * 2));
  TRY(dev_alloc(ctx, &dk, nkv * 2));
  TRY(dev_alloc(ctx, &dv, nkv * 2));
  TRY(dev_alloc(ctx, &dout, nq * 2));
  TRY(dev_alloc(ctx, &tmp, std::min<int64_t>(std::max(nq, nkv), 64ll << 20) * 4));
  cudaStream_t st = ctx->s_comp;
  const int64_t chunk = std::min<int64_t>(std::max(nq, nkv), 64ll << 20);
  for (int w = 0; w < 3; ++w) {
    __half* dst = w == 0 ? dq : (w == 1 ? dk : dv);
    const int64_t cnt = w == 0 ? nq : nkv;
    for (int64_t off = 0; off < cnt; off += chunk) {
      const int64_t c = std::min(chunk, cnt - off);
      LAUNCH(launch_synth(tmp, off, c, synth_key(9, 8, w), 0, synth_scale(0, w == 0 ? 0.1 : 1.0), st));
      LAUNCH(launch_f32_to_f16(tmp, dst + off, c, st));
    }
  }
  AttnArgs aa;
  aa.q = dq; aa.kc = dk; aa.vc = dv; aa.o = dout; aa.b = b; aa.n = n; aa.past = 0; aa.d = d;
  aa.n_heads = n_heads; aa.kv_b = b; aa.ws = ctx->ws; aa.ws_floats = ctx->ws_floats; aa.num_sms = ctx->num_sms;
  aa.dkv = dkv; aa.group = n_heads / n_kv_heads;
  aa.use_cuda_cores = variant;
  LAUNCH(launch_attention_prefill(aa, st));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0, st));
  for (int i = 0; i < iters; ++i) LAUNCH(launch_attention_prefill(aa, st));
  CK(cudaEventRecord(e1, st));
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0); cudaEventDestroy(e1);
  if (getenv("PIPO_WS_DEBUG") && (atoi(getenv("PIPO_WS_DEBUG")) & 128) && variant == 0) {
    std::vector<uint64_t> c(148 * 8);
    CK(cudaMemcpy(c.data(), ctx->ws + (15ll << 20), c.size() * 8, cudaMemcpyDeviceToHost));
    double t[6] = {0};
    for (int i = 0; i < 148; ++i) for (int k = 0; k < 6; ++k) t[k] += (double)c[i * 8 + k];
    fprintf(stderr, "attn-tc per item (cycles, warp 2): wait S %.0f | pass1 (max) %.0f | pass2 (exp, P) %.0f | wait O %.0f | epilogue %.0f  (%.0f items)\n",
            t[0] / t[5], t[1] / t[5], t[2] / t[5], t[3] / t[5], t[4] / t[5], t[5]);
  }
  cudaFree(dq); cudaFree(dk); cudaFree(dv); cudaFree(dout); cudaFree(tmp);
  ctx->hbm_bytes -= nq * 4 + nkv * 4 + chunk * 4;
  *us = ms * 1e3 / iters;
  return PIPO_OK;
}

pipo_status pipo_attention_decode(pipo_ctx* ctx, const uint16_t* q, const uint16_t* k, const uint16_t* v, int32_t b,
                                  int32_t L, int32_t d, int32_t n_heads, int32_t variant, float* o) {
  CHECK_CTX();
  if (!q || !k || !v || !o || b <= 0 || L <= 0 || d <= 0 || n_heads <= 0 || d % n_heads)
    return set_err(PIPO_E_INVALID_ARG, "bad attention arguments");
  CK(cudaSetDevice(ctx->cfg.device));
  __half *dq = nullptr, *dk = nullptr, *dv = nullptr, *dout = nullptr;
  float* df = nullptr;
  const int64_t nq = (int64_t)b * d, nkv = (int64_t)L * b * d;
  TRY(dev_alloc(ctx, &dq, nq * 2));
  TRY(dev_alloc(ctx, &dk, nkv * 2));
  TRY(dev_alloc(ctx, &dv, nkv * 2));
  TRY(dev_alloc(ctx, &dout, nq * 2));
  TRY(dev_alloc(ctx, &df, nq * 4));
  cudaStream_t st = ctx->s_comp;
  CK(cudaMemcpyAsync(dq, q, (size_t)nq * 2, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(dk, k, (size_t)nkv * 2, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(dv, v, (size_t)nkv * 2, cudaMemcpyHostToDevice, st));
  AttnArgs aa;
  aa.q = dq; aa.kc = dk; aa.vc = dv; aa.o = dout; aa.b = b; aa.n = 1; aa.past = L - 1; aa.d = d;
  aa.n_heads = n_heads; aa.kv_b = b; aa.ws = ctx->ws; aa.ws_floats = ctx->ws_floats; aa.num_sms = ctx->num_sms;
  aa.use_cuda_cores = variant;
  LAUNCH(launch_attention_decode(aa, st));
  LAUNCH(launch_f16_to_f32(dout, df, nq, st));
  CK(cudaMemcpyAsync(o, df, (size_t)nq * 4, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  cudaFree(dq); cudaFree(dk); cudaFree(dv); cudaFree(dout); cudaFree(df);
  ctx->hbm_bytes -= nq * 2 * 2 + nkv * 2 * 2 + nq * 4;
  return PIPO_OK;
}

pipo_status pipo_attention_prefill(pipo_ctx* ctx, const uint16_t* q, const uint16_t* k, const uint16_t* v,
                                   int32_t b, int32_t n, int32_t past, int32_t d, int32_t n_heads, int32_t cuda_cores,
                                   float* o) {
  CHECK_CTX();
  if (!q || !k || !v || !o || b <= 0 || n <= 0 || past < 0 || d <= 0 || n_heads <= 0 || d % n_heads)
    return set_err(PIPO_E_INVALID_ARG, "bad attention arguments");
  CK(cudaSetDevice(ctx->cfg.device));
  __half *dq = nullptr, *dk = nullptr, *dv = nullptr, *dout = nullptr;
  float* df = nullptr;
  const int64_t L = past + n, nq = (int64_t)b * n * d, nkv = L * b * d;
  TRY(dev_alloc(ctx, &dq, nq * 2));
  TRY(dev_alloc(ctx, &dk, nkv * 2));
  TRY(dev_alloc(ctx, &dv, nkv * 2));
  TRY(dev_alloc(ctx, &dout, nq * 2));
  TRY(dev_alloc(ctx, &df, nq * 4));
  cudaStream_t st = ctx->s_comp;
  CK(cudaMemcpyAsync(dq, q, (size_t)nq * 2, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(dk, k, (size_t)nkv * 2, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(dv, v, (size_t)nkv * 2, cudaMemcpyHostToDevice, st));
  AttnArgs aa;
  aa.q = dq; aa.kc = dk; aa.vc = dv; aa.o = dout; aa.b = b; aa.n = n; aa.past = past; aa.d = d;
  aa.n_heads = n_heads; aa.kv_b = b; aa.ws = ctx->ws; aa.ws_floats = ctx->ws_floats; aa.num_sms = ctx->num_sms;
  aa.use_cuda_cores = cuda_cores;
  LAUNCH(launch_attention_prefill(aa, st));
  LAUNCH(launch_f16_to_f32(dout, df, nq, st));
  CK(cudaMemcpyAsync(o, df, (size_t)nq * 4, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  cudaFree(dq); cudaFree(dk); cudaFree(dv); cudaFree(dout); cudaFree(df);
  ctx->hbm_bytes -= nq * 2 * 2 + nkv * 2 * 2 + nq * 4;
  return PIPO_OK;
}

pipo_status pipo_attention_gqa(pipo_ctx* ctx, const uint16_t* q, const uint16_t* k, const uint16_t* v, int32_t b,
                               int32_t n, int32_t past, int32_t n_heads, int32_t n_kv_heads, int32_t head_dim,
                               int32_t variant, float* o) {
  CHECK_CTX();
  if (!q || !k || !v || !o || b <= 0 || n <= 0 || past < 0 || n_heads <= 0 || n_kv_heads <= 0 ||
      n_heads % n_kv_heads || (head_dim != 64 && head_dim != 128))
    return set_err(PIPO_E_INVALID_ARG, "bad attention arguments");
  CK(cudaSetDevice(ctx->cfg.device));
  const int d = n_heads * head_dim, dkv = n_kv_heads * head_dim;
  __half *dq = nullptr, *dk = nullptr, *dv = nullptr, *dout = nullptr;
  float* df = nullptr;
  const int64_t L = past + n, nq = (int64_t)b * n * d, nkv = L * b * dkv;
  TRY(dev_alloc(ctx, &dq, nq * 2));
  TRY(dev_alloc(ctx, &dk, nkv * 2));
  TRY(dev_alloc(ctx, &dv, nkv * 2));
  TRY(dev_alloc(ctx, &dout, nq * 2));
  TRY(dev_alloc(ctx, &df, nq * 4));
  cudaStream_t st = ctx->s_comp;
  CK(cudaMemcpyAsync(dq, q, (size_t)nq * 2, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(dk, k, (size_t)nkv * 2, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(dv, v, (size_t)nkv * 2, cudaMemcpyHostToDevice, st));
  AttnArgs aa;
  aa.q = dq; aa.kc = dk; aa.vc = dv; aa.o = dout; aa.b = b; aa.n = n; aa.past = past; aa.d = d;
  aa.n_heads = n_heads; aa.kv_b = b; aa.dkv = dkv; aa.group = n_heads / n_kv_heads;
  aa.ws = ctx->ws; aa.ws_floats = ctx->ws_floats; aa.num_sms = ctx->num_sms;
  aa.use_cuda_cores = variant;
  if (n == 1) LAUNCH(launch_attention_decode(aa, st));
  else LAUNCH(launch_attention_prefill(aa, st));
  LAUNCH(launch_f16_to_f32(dout, df, nq, st));
  CK(cudaMemcpyAsync(o, df, (size_t)nq * 4, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  cudaFree(dq); cudaFree(dk); cudaFree(dv); cudaFree(dout); cudaFree(df);
  ctx->hbm_bytes -= nq * 2 * 2 + nkv * 2 * 2 + nq * 4;
  return PIPO_OK;
}

pipo_status pipo_rope(pipo_ctx* ctx, const uint16_t* q, const uint16_t* k, int32_t b, int32_t n, int32_t past,
                      float* q_out, float* k_out) {
  CHECK_CTX();
  if (ctx->arch != PIPO_ARCH_LLAMA) return set_err(PIPO_E_STATE, "pipo_rope needs a LLaMA context");
  if (!q || !k || !q_out || !k_out || b <= 0 || n <= 0 || past < 0 || past + n > ctx->max_s)
    return set_err(PIPO_E_INVALID_ARG, "bad rope arguments");
  CK(cudaSetDevice(ctx->cfg.device));
  __half *dq = nullptr, *dk = nullptr;
  float* df = nullptr;
  const int64_t nq = (int64_t)b * n * ctx->d, nk = (int64_t)(past + n) * b * ctx->dkv;
  TRY(dev_alloc(ctx, &dq, nq * 2));
  TRY(dev_alloc(ctx, &dk, nk * 2));
  TRY(dev_alloc(ctx, &df, std::max(nq, nk) * 4));
  cudaStream_t st = ctx->s_comp;
  CK(cudaMemcpyAsync(dq, q, (size_t)nq * 2, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(dk, k, (size_t)nk * 2, cudaMemcpyHostToDevice, st));
  LAUNCH(launch_rope(dq, dk, ctx->rope_inv, b, n, past, ctx->H, ctx->Hkv, ctx->hd, b, st));
  LAUNCH(launch_f16_to_f32(dq, df, nq, st));
  CK(cudaMemcpyAsync(q_out, df, (size_t)nq * 4, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  LAUNCH(launch_f16_to_f32(dk, df, nk, st));
  CK(cudaMemcpyAsync(k_out, df, (size_t)nk * 4, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  cudaFree(dq); cudaFree(dk); cudaFree(df);
  ctx->hbm_bytes -= nq * 2 + nk * 2 + std::max(nq, nk) * 4;
  return PIPO_OK;
}

int32_t pipo_gpu_numa_node(int32_t device) { return gpu_numa_node(device); }

pipo_status pipo_get_plan(pipo_ctx* ctx, pipo_plan* out) {
  CHECK_CTX();
  if (!out) return set_err(PIPO_E_INVALID_ARG, "out is NULL");
  if (!ctx->auto_plan) return set_err(PIPO_E_STATE, "context was not configured by PIPO_F_AUTO_PLAN");
  *out = ctx->plan;
  return PIPO_OK;
}

pipo_status pipo_shard_range(int64_t layer_bytes, int32_t world, int32_t rank, int64_t* offset, int64_t* bytes) {
  if (layer_bytes <= 0 || world <= 0 || rank < 0 || rank >= world || !offset || !bytes)
    return set_err(PIPO_E_INVALID_ARG, "bad shard arguments");
  const int64_t padded = round_up(layer_bytes, (int64_t)world * 4096);
  *bytes = padded / world;
  *offset = (int64_t)rank * *bytes;
  return PIPO_OK;
}

pipo_status pipo_nccl_unique_id(uint8_t id[128]) {
  if (!id) return set_err(PIPO_E_INVALID_ARG, "id is NULL");
  const int rc = nccl_unique_id(id);
  if (rc != 0) return set_err(PIPO_E_CUDA, std::string("ncclGetUniqueId: ") + nccl_error_string(rc));
  return PIPO_OK;
}

pipo_status pipo_shard_stream_init(pipo_ctx* ctx, int32_t rank, int32_t world, const uint8_t id[128]) {
  CHECK_CTX();
  if (!id || world <= 0 || rank < 0 || rank >= world) return set_err(PIPO_E_INVALID_ARG, "bad rank/world");
  if (ctx->weight_tier != PIPO_TIER_HOST) return set_err(PIPO_E_INVALID_ARG, "sharded streaming needs the HOST tier");
  if (sharded(ctx)) return set_err(PIPO_E_STATE, "sharded streaming already initialised");
  for (int j = 0; j < ctx->l; ++j)
    if (ctx->layer_loaded[j]) return set_err(PIPO_E_STATE, "call pipo_shard_stream_init before loading weights");
  CK(cudaSetDevice(ctx->cfg.device));
  int64_t off = 0, S = 0;
  TRY(pipo_shard_range(ctx->lay.total, world, rank, &off, &S));
  CK(cudaDeviceSynchronize());
  // Everything that can fail is built in temporaries first; the context changes only
  // once all of it succeeded (a failure leaves the plain HOST tier intact).
  const int64_t ring_bytes = (int64_t)ctx->R * S * world;
  uint8_t* new_ring = nullptr;
  uint8_t* new_store = nullptr;
  void* comm = nullptr;
  cudaStream_t gather = nullptr;
  cudaEvent_t evs[kMaxRing] = {};
  auto unwind = [&](pipo_status st) {
    if (new_ring) { cudaFree(new_ring); ctx->hbm_bytes -= ring_bytes; }
    host_free(ctx, new_store, (int64_t)ctx->l * S);
    if (comm) nccl_comm_destroy(comm);
    if (gather) cudaStreamDestroy(gather);
    for (auto& e : evs)
      if (e) cudaEventDestroy(e);
    cudaGetLastError();
    return st;
  };
  pipo_status st = dev_alloc(ctx, &new_ring, ring_bytes);
  if (st != PIPO_OK) return unwind(st);
  if (cudaMemset(new_ring, 0, (size_t)ring_bytes) != cudaSuccess) return unwind(set_err(PIPO_E_CUDA, "cudaMemset of the ring"));
  st = host_alloc(ctx, &new_store, (int64_t)ctx->l * S, true);
  if (st != PIPO_OK) return unwind(st);
  if (cudaStreamCreateWithFlags(&gather, cudaStreamNonBlocking) != cudaSuccess)
    return unwind(set_err(PIPO_E_CUDA, "gather stream"));
  for (auto& e : evs)
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return unwind(set_err(PIPO_E_CUDA, "events"));
  const int rc = nccl_comm_init(&comm, world, id, rank);
  if (rc != 0) {
    comm = nullptr;
    return unwind(set_err(PIPO_E_CUDA, std::string("ncclCommInitRank: ") + nccl_error_string(rc)));
  }
  // commit
  if (ctx->ring) { cudaFree(ctx->ring); ctx->hbm_bytes -= (int64_t)ctx->R * ctx->layer_bytes; }
  host_free(ctx, ctx->host_store, (int64_t)ctx->l * ctx->layer_bytes);
  ctx->ring = new_ring;
  ctx->host_store = new_store;
  ctx->layer_bytes = S * world;
  ctx->shard_bytes = S;
  ctx->shard_rank = rank;
  ctx->shard_world = world;
  ctx->s_gather = gather;
  for (int i = 0; i < kMaxRing; ++i) ctx->ev_h2d[i] = evs[i];
  ctx->nccl_comm = comm;
  ctx->shard_mode = 1;
  return PIPO_OK;
}

pipo_status pipo_shard_p2p_export(pipo_ctx* ctx, int32_t rank, int32_t world, uint8_t handle[PIPO_SHARD_HANDLE_BYTES]) {
  CHECK_CTX();
  if (!handle || world <= 0 || world > 8 || rank < 0 || rank >= world)
    return set_err(PIPO_E_INVALID_ARG, "bad rank/world (world <= 8)");
  if (ctx->weight_tier != PIPO_TIER_HOST) return set_err(PIPO_E_INVALID_ARG, "sharded streaming needs the HOST tier");
  if (sharded(ctx)) return set_err(PIPO_E_STATE, "sharded streaming already initialised");
  for (int j = 0; j < ctx->l; ++j)
    if (ctx->layer_loaded[j]) return set_err(PIPO_E_STATE, "export before loading weights");
  CK(cudaSetDevice(ctx->cfg.device));
  if (ctx->pend_ring) { cudaFree(ctx->pend_ring); ctx->hbm_bytes -= ctx->pend_ring_bytes; ctx->pend_ring = nullptr; }
  if (ctx->pend_store) { host_free(ctx, ctx->pend_store, (int64_t)ctx->l * ctx->pend_S); ctx->pend_store = nullptr; }
  int64_t off = 0, S = 0;
  TRY(pipo_shard_range(ctx->lay.total, world, rank, &off, &S));
  const int64_t ring_bytes = (int64_t)ctx->R * S * world + 4096;   // + the flags page
  TRY(dev_alloc(ctx, &ctx->pend_ring, ring_bytes));
  ctx->pend_ring_bytes = ring_bytes;
  CK(cudaMemset(ctx->pend_ring, 0, (size_t)ring_bytes));
  TRY(host_alloc(ctx, &ctx->pend_store, (int64_t)ctx->l * S, true));
  ctx->pend_S = S;
  ctx->pend_rank = rank;
  ctx->pend_world = world;
  cudaIpcMemHandle_t h;
  CK(cudaIpcGetMemHandle(&h, ctx->pend_ring));
  std::memset(handle, 0, PIPO_SHARD_HANDLE_BYTES);
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  std::memcpy(handle, &h, 64);
  const int64_t meta[4] = {(int64_t)rank, (int64_t)world, ring_bytes, (int64_t)ctx->R};
  std::memcpy(handle + 64, meta, sizeof meta);
  return PIPO_OK;
}

pipo_status pipo_shard_p2p_init(pipo_ctx* ctx, const uint8_t* handles) {
  CHECK_CTX();
  if (!handles) return set_err(PIPO_E_INVALID_ARG, "handles is NULL");
  if (!ctx->pend_ring) return set_err(PIPO_E_STATE, "pipo_shard_p2p_export first");
  if (sharded(ctx)) return set_err(PIPO_E_STATE, "sharded streaming already initialised");
  CK(cudaSetDevice(ctx->cfg.device));
  const int W = ctx->pend_world, me = ctx->pend_rank;
  for (int p = 0; p < W; ++p) {
    int64_t meta[4];
    std::memcpy(meta, handles + (size_t)p * PIPO_SHARD_HANDLE_BYTES + 64, sizeof meta);
    if (meta[0] != p || meta[1] != W || meta[2] != ctx->pend_ring_bytes || meta[3] != ctx->R)
      return set_err(PIPO_E_INVALID_ARG, "handle " + std::to_string(p) + " is not rank " + std::to_string(p) +
                                             " of this sharded configuration");
  }
  cudaStream_t gather = nullptr;
  cudaEvent_t evs[kMaxRing] = {};
  uint8_t* opened[8] = {};
  auto unwind = [&](pipo_status st) {
    for (auto& o : opened)
      if (o) cudaIpcCloseMemHandle(o);
    if (gather) cudaStreamDestroy(gather);
    for (auto& e : evs)
      if (e) cudaEventDestroy(e);
    cudaGetLastError();
    return st;
  };
  for (int p = 0; p < W; ++p) {
    if (p == me) continue;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handles + (size_t)p * PIPO_SHARD_HANDLE_BYTES, 64);
    void* ptr = nullptr;
    const cudaError_t e = cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess)
      return unwind(set_err(PIPO_E_CUDA, std::string("cudaIpcOpenMemHandle of rank ") + std::to_string(p) + ": " +
                                             cudaGetErrorString(e)));
    opened[p] = static_cast<uint8_t*>(ptr);
  }
  if (cudaStreamCreateWithFlags(&gather, cudaStreamNonBlocking) != cudaSuccess)
    return unwind(set_err(PIPO_E_CUDA, "gather stream"));
  for (auto& e : evs)
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return unwind(set_err(PIPO_E_CUDA, "events"));
  // commit
  CK(cudaDeviceSynchronize());
  if (ctx->ring) { cudaFree(ctx->ring); ctx->hbm_bytes -= (int64_t)ctx->R * ctx->layer_bytes; }
  host_free(ctx, ctx->host_store, (int64_t)ctx->l * ctx->layer_bytes);
  ctx->ring = ctx->pend_ring;
  ctx->host_store = ctx->pend_store;
  ctx->pend_ring = nullptr;
  ctx->pend_store = nullptr;
  ctx->shard_bytes = ctx->pend_S;
  ctx->layer_bytes = ctx->pend_S * W;
  ctx->shard_rank = me;
  ctx->shard_world = W;
  ctx->own_flags = reinterpret_cast<int*>(ctx->ring + (int64_t)ctx->R * ctx->layer_bytes);
  for (int p = 0; p < W; ++p) ctx->peer_ring[p] = opened[p];
  ctx->s_gather = gather;
  for (int i = 0; i < kMaxRing; ++i) ctx->ev_h2d[i] = evs[i];
  ctx->shard_mode = 2;
  return PIPO_OK;
}

pipo_status pipo_debug_capture(pipo_ctx* ctx, int32_t on, float* out) {
  CHECK_CTX();
  if (!on) { ctx->cap_on = false; return PIPO_OK; }
  if (!out) return set_err(PIPO_E_INVALID_ARG, "capture buffer is NULL");
  CK(cudaSetDevice(ctx->cfg.device));
  const int64_t need = (int64_t)ctx->l * ctx->rows_cap * ctx->d * 4;
  if (ctx->cap_dev_bytes < need) {
    if (ctx->cap_dev) { cudaFree(ctx->cap_dev); ctx->hbm_bytes -= ctx->cap_dev_bytes; }
    ctx->cap_dev = nullptr;
    ctx->cap_dev_bytes = 0;
    TRY(dev_alloc(ctx, &ctx->cap_dev, need));
    ctx->cap_dev_bytes = need;
  }
  ctx->cap_on = true;
  ctx->cap_host = out;
  return PIPO_OK;
}

pipo_status pipo_debug_inject(pipo_ctx* ctx, int32_t copy_delay_us, int32_t compute_delay_us, int32_t ring_checksum) {
  CHECK_CTX();
  if (copy_delay_us < 0 || compute_delay_us < 0) return set_err(PIPO_E_INVALID_ARG, "negative delay");
  CK(cudaSetDevice(ctx->cfg.device));
  if (ring_checksum && !ctx->ring_sums) {
    TRY(dev_alloc(ctx, &ctx->ring_sums, (int64_t)ctx->l * 8));
    CK(cudaMemset(ctx->ring_sums, 0, (size_t)ctx->l * 8));
  }
  CK(cudaDeviceSynchronize());
  ctx->dbg_copy_delay_ns = (int64_t)copy_delay_us * 1000;
  ctx->dbg_comp_delay_ns = (int64_t)compute_delay_us * 1000;
  ctx->dbg_ring_sum = ring_checksum != 0;
  return PIPO_OK;
}

pipo_status pipo_debug_ring_checksums(pipo_ctx* ctx, uint64_t* out) {
  CHECK_CTX();
  if (!out) return set_err(PIPO_E_INVALID_ARG, "NULL output");
  if (!ctx->ring_sums) return set_err(PIPO_E_STATE, "ring checksums were not enabled (pipo_debug_inject)");
  CK(cudaSetDevice(ctx->cfg.device));
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(out, ctx->ring_sums, (size_t)ctx->l * 8, cudaMemcpyDeviceToHost));
  return PIPO_OK;
}

pipo_status pipo_debug_read_blob(pipo_ctx* ctx, int32_t layer, uint8_t* out, int64_t bytes) {
  CHECK_CTX();
  if (!out || layer < 0 || layer >= ctx->l || bytes != ctx->layer_bytes)
    return set_err(PIPO_E_INVALID_ARG, "layer out of range or bytes != layer blob size");
  if (ctx->disk || ctx->shard_mode || !ctx->host_store)
    return set_err(PIPO_E_INVALID_ARG, "pipo_debug_read_blob reads the unsharded HOST-tier pinned store");
  CK(cudaSetDevice(ctx->cfg.device));
  CK(cudaDeviceSynchronize());
  std::memcpy(out, ctx->host_store + (int64_t)layer * ctx->layer_bytes, (size_t)bytes);
  return PIPO_OK;
}

pipo_status pipo_layer_blob_bytes(pipo_ctx* ctx, int64_t* bytes) {
  CHECK_CTX();
  if (!bytes) return set_err(PIPO_E_INVALID_ARG, "NULL output");
  *bytes = ctx->layer_bytes;
  return PIPO_OK;
}

pipo_status pipo_debug_read_rows(pipo_ctx* ctx, int32_t layer, int32_t matrix, int64_t row0, int64_t nrows,
                                 uint8_t* codes, uint16_t* scales, uint16_t* values) {
  CHECK_CTX();
  CK(cudaSetDevice(ctx->cfg.device));
  MatLayout ml;
  const uint8_t* base = nullptr;
  bool on_device = true, glu = false;
  if (layer == PIPO_LAYER_EMBED) {
    if (!ctx->embed_loaded) return set_err(PIPO_E_STATE, "embedding weights not loaded");
    if (matrix != 0 && !(matrix == 1 && ctx->arch == PIPO_ARCH_LLAMA))
      return set_err(PIPO_E_INVALID_ARG, "embedding matrix: 0 = token table, 1 = LLaMA LM head");
    ml = ctx->tok_lay;
    base = reinterpret_cast<const uint8_t*>(matrix == 0 ? ctx->tok : ctx->head);
  } else {
    if (layer < 0 || layer >= ctx->l || matrix < 0 || matrix >= M_COUNT)
      return set_err(PIPO_E_INVALID_ARG, "layer / matrix out of range");
    if (!ctx->layer_loaded[layer]) return set_err(PIPO_E_STATE, "layer not loaded");
    ml = ctx->lay.mat[matrix];
    glu = ctx->lay.glu && matrix == M_FC1;
    if (ctx->weight_tier == PIPO_TIER_DEVICE) {
      base = ctx->dev_store + (int64_t)layer * ctx->layer_bytes + ctx->lay.mat_off[matrix];
    } else if (ctx->weight_tier == PIPO_TIER_HOST && !sharded(ctx)) {
      base = ctx->host_store + (int64_t)layer * ctx->layer_bytes + ctx->lay.mat_off[matrix];
      on_device = false;
    } else {
      return set_err(PIPO_E_INVALID_ARG, "pipo_debug_read_rows reads the DEVICE or (unsharded) HOST tier");
    }
  }
  if (row0 < 0 || nrows <= 0 || row0 + nrows > ml.N) return set_err(PIPO_E_INVALID_ARG, "row range out of bounds");
  const bool q4 = layer != PIPO_LAYER_EMBED && ml.wfmt == 1;
  if (q4 ? (!codes || !scales) : !values) return set_err(PIPO_E_INVALID_ARG, "NULL output buffer");
  const int64_t K = ml.K, strip = ml.n_kb * ml.block_bytes;
  std::vector<uint8_t> buf((size_t)strip);
  int64_t loaded = -1;
  for (int64_t i = 0; i < nrows; ++i) {
    int64_t r = row0 + i;                     // logical row -> stored row (LLaMA gate|up interleave)
    if (glu) {
      const int64_t F = ml.N / 2, u = r >= F ? r - F : r;
      r = (u / kTileRows) * 2 * kTileRows + (r >= F ? kTileRows : 0) + u % kTileRows;
    }
    const int64_t rt = r / kTileRows, rr = r % kTileRows;
    if (rt != loaded) {
      if (on_device) CK(cudaMemcpy(buf.data(), base + rt * strip, (size_t)strip, cudaMemcpyDeviceToHost));
      else std::memcpy(buf.data(), base + rt * strip, (size_t)strip);
      loaded = rt;
    }
    for (int64_t kb = 0; kb < ml.n_kb; ++kb) {
      const uint8_t* blk = buf.data() + kb * ml.block_bytes;
      if (!q4) {
        std::memcpy(values + i * K + kb * kTileK, blk + rr * kTileK * 2, kTileK * 2);
        continue;
      }
      std::memcpy(scales + i * (K / 64) + kb, blk + 4096 + rr * 2, 2);
      int q[64];
      for (int h = 0; h < 2; ++h)
        for (int w = 0; w < 4; ++w) {
          uint32_t word;
          std::memcpy(&word, blk + (h * kTileRows + rr) * 16 + w * 4, 4);
          for (int nib = 0; nib < 8; ++nib)
            q[h * 32 + w * 8 + kNibbleElem[nib]] = (int)((word >> (4 * nib)) & 0xF) - 8;
        }
      for (int m = 0; m < 32; ++m)
        codes[i * (K / 2) + kb * 32 + m] = (uint8_t)((q[2 * m] & 0xF) | ((q[2 * m + 1] & 0xF) << 4));
    }
  }
  return PIPO_OK;
}

pipo_status pipo_probe_h2d(pipo_ctx* ctx, int64_t bytes, int32_t reps, double* gbs) {
  CHECK_CTX();
  if (bytes <= 0 || reps <= 0 || !gbs) return set_err(PIPO_E_INVALID_ARG, "bad probe arguments");
  CK(cudaSetDevice(ctx->cfg.device));
  uint8_t *hsrc = nullptr, *ddst = nullptr;
  TRY(host_alloc(ctx, &hsrc, bytes));
  TRY(dev_alloc(ctx, &ddst, bytes));
  std::memset(hsrc, 1, (size_t)bytes);
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  double best = 0;
  for (int r = 0; r < reps + 1; ++r) {
    CK(cudaEventRecord(a, ctx->s_copy));
    CK(cudaMemcpyAsync(ddst, hsrc, (size_t)bytes, cudaMemcpyHostToDevice, ctx->s_copy));
    CK(cudaEventRecord(b, ctx->s_copy));
    CK(cudaEventSynchronize(b));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, a, b));
    if (r > 0) best = std::max(best, bytes / (ms * 1e-3) / 1e9);
  }
  cudaEventDestroy(a); cudaEventDestroy(b);
  cudaFreeHost(hsrc); cudaFree(ddst);
  ctx->pinned_bytes -= bytes;
  ctx->hbm_bytes -= bytes;
  *gbs = best;
  return PIPO_OK;
}

}  // extern "C"
