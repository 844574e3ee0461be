// ctx.h — the pipeline context (internal).
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <chrono>
#include <string>
#include <vector>

#include "../../include/pipo.h"
#include "host.h"
#include "kernels.h"
#include "layout.h"

namespace pipo {

constexpr int kMaxRing = 8;

struct Span {            // one interval on a device lane, between two timed events
  cudaEvent_t a, b;
  int lane;              // 0 = H2D copy, 1 = kernels, 2 = D2H save, 3 = NVLink all-gather
  int64_t bytes;
};

struct KRec {            // one timed kernel unit (PIPO_F_KPROF)
  cudaEvent_t a, b;
  int cls;
  double bytes, flops;
};

struct DiskTier;         // disk.cpp

}  // namespace pipo

struct pipo_ctx {
  pipo_config cfg{};
  std::string disk_dir;
  int d = 0, l = 0, H = 0, F = 0, V = 0, hd = 0, max_b = 0, max_s = 0, wfmt = 1;
  int arch = 0;                    // PIPO_ARCH_OPT / PIPO_ARCH_LLAMA
  int Hkv = 0, dkv = 0;            // KV heads, K/V row width (OPT: H, d)
  float* rope_inv = nullptr;       // LLaMA: device [hd/2] inverse frequencies (llama3 rule)
  int weight_tier = 1, kv_tier = 0, R = 2, gemv_max_m = 15;
  int64_t chunk = 0;
  pipo::LayerLayout lay;
  int64_t layer_bytes = 0;
  int num_sms = 148;
  bool poisoned = false;

  cudaStream_t s_comp = nullptr, s_copy = nullptr, s_save = nullptr;
  cudaStream_t s_gather = nullptr;   // NEXT-1: NVLink all-gather, off the PCIe copy stream

  // resident embeddings (Q20)
  pipo::MatLayout tok_lay;
  __half* tok = nullptr;      // tiled [V_pad x d]
  __half* pos = nullptr;      // [max_pos + 2][d]
  __half* lnf_g = nullptr;
  __half* lnf_b = nullptr;
  __half* head = nullptr;     // LM head weight, tiled [V_pad x d]: == tok (OPT, tied) or own (LLaMA)
  bool embed_loaded = false;
  std::vector<char> layer_loaded;

  // weights
  uint8_t* host_store = nullptr;   // pinned, l * layer_bytes (HOST tier)
  uint8_t* dev_store = nullptr;    // HBM, l * layer_bytes (DEVICE tier)
  uint8_t* ring = nullptr;         // HBM, R * layer_bytes (HOST / DISK tiers)
  // NEXT-1 sharded streaming: this rank streams bytes [shard_rank*shard_bytes, +shard_bytes)
  // of every (padded) layer blob and all-gathers the rest from its peers (NCCL, copy stream)
  int shard_rank = 0, shard_world = 1;
  int64_t shard_bytes = 0;         // per-rank range; host_store holds l * shard_bytes
  void* nccl_comm = nullptr;       // ncclComm_t
  int shard_mode = 0;              // 0 plain, 1 NCCL all-gather, 2 peer copies (CUDA IPC)
  // peer transport: pending allocations between export and init, then the peers' rings
  // (IPC mappings; the flags live in the last 4 KiB of every ring allocation:
  // [0] = layers this rank has landed, [1 + p] = layers of this rank's ring peer p copied)
  uint8_t* pend_ring = nullptr;
  uint8_t* pend_store = nullptr;
  int64_t pend_ring_bytes = 0, pend_S = 0;
  int pend_rank = -1, pend_world = 0;
  uint8_t* peer_ring[8] = {};
  int* own_flags = nullptr;
  pipo::DiskTier* disk = nullptr;

  // KV cache: position-major [pos][b][d] per (layer, K/V)
  // one region per (layer, K/V): fp16 [pos][b][d], or int4 codes [pos][b][d/2] followed
  // (at kv_codes_cap) by fp16 scales [pos][b][d/64]
  int kv_fmt = 0;
  int64_t kv_tensor_bytes = 0;     // bytes per (layer, K/V) region
  int64_t kv_codes_cap = 0;        // int4: byte offset of the scales inside a region
  uint8_t* kv_dev = nullptr;       // DEVICE kv tier: [l][2] regions
  uint8_t* kv_host = nullptr;      // HOST kv tier (pinned): [l][2] regions
  uint8_t* kv_slot = nullptr;      // HOST kv tier: [R][2] staging regions in HBM
  __half* kv_stage = nullptr;      // int4 KV: fresh fp16 K/V rows [rows][2d] of the current pass

  // activations
  int64_t rows_cap = 0;
  float* h = nullptr;              // [rows][d] fp32 residual stream
  __half* xa = nullptr;            // [rows][d] LN output / attention output
  __half* q = nullptr;             // [rows][d]
  __half* u = nullptr;             // [rows][F]
  __half* gu = nullptr;            // LLaMA: FC1 gate|up output [rows][2F] (tile-interleaved)
  float* logits = nullptr;         // [max_b][V]
  int32_t* ids = nullptr;          // [rows]
  int32_t* next = nullptr;         // [max_b]
  int32_t* pin_ids = nullptr;      // pinned staging
  int32_t* pin_next = nullptr;
  float* ws = nullptr;
  int64_t ws_floats = 0;
  int* counters = nullptr;
  int n_counters = 0;
  int* quant_bad = nullptr;        // device flag for the GPU quantizer

  // pipeline state (Alg. 1 as a stream/event DAG)
  int64_t g_copy = 0;              // next global layer index whose copy is enqueued
  int64_t g_comp = 0;              // next global layer index to compute
  cudaEvent_t ev_ready[pipo::kMaxRing][5] = {};   // seg 0..3 landed, [4] = KV landed
  cudaEvent_t ev_h2d[pipo::kMaxRing] = {};        // NEXT-1: this rank's range landed (gather may start)
  cudaEvent_t ev_free[pipo::kMaxRing] = {};       // compute done with the slot
  cudaEvent_t ev_kv_free[pipo::kMaxRing] = {};    // KV slot free (after save)
  cudaEvent_t ev_attn[pipo::kMaxRing] = {};       // attention done (save may start)
  std::vector<cudaEvent_t> ev_saved;              // per layer: last KV save done (A6 fence)
  std::vector<int64_t> kv_load_past;              // per ring slot: positions its KV load covers
  int b_cur = 0, past = 0;
  bool have_batch = false;

  // capture (pipo_debug_capture)
  bool cap_on = false;
  float* cap_host = nullptr;
  float* cap_dev = nullptr;
  int64_t cap_dev_bytes = 0;

  // stats / timeline
  bool timeline = true;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  std::vector<pipo::Span> spans;
  bool kprof = false;
  std::vector<pipo::KRec> krecs;
  cudaEvent_t win_start = nullptr, win_end = nullptr;
  bool win_open = false, win_closed = false;
  int64_t launches = 0;
  int64_t prefill_calls = 0, decode_steps = 0, tokens = 0;
  double prefill_s = 0, decode_s = 0, ttft_s = 0;
  int64_t h2d_bytes = 0, d2h_bytes = 0;
  int64_t hbm_bytes = 0, pinned_bytes = 0;
  // NUMA placement of the big pinned stores (numa.cpp): resolved node (-1 = none) and the
  // mmap + mbind + cudaHostRegister allocations that pipeline_destroy must unregister
  int numa_node = -1;
  std::vector<std::pair<void*, int64_t>> numa_allocs;
  bool timeline_truncated = false;
  // test hooks (pipo_debug_inject): injected delays, ring checksums per layer
  int64_t dbg_copy_delay_ns = 0, dbg_comp_delay_ns = 0;
  bool dbg_ring_sum = false;
  uint64_t* ring_sums = nullptr;   // device [l]
  bool forwarded = false;          // a prefill/decode has run (prefetch may be in flight)
  bool auto_plan = false;          // PIPO_F_AUTO_PLAN: the fields below came from Eq. (1)
  pipo_plan plan{};
};
