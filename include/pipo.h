/*
 * pipo.h — C-ABI of the B200-native PIPO hot path (arXiv 2504.03664).
 *
 * PIPO = "pipelined offloading" (§3).  This library implements
 * its data-parallel hot path for OPT decoders: weights (and optionally the KV
 * cache) live off-GPU — pinned host memory (§3.1.1) or files on disk
 * read through a pinned host ring (§3.3) — and are streamed to
 * HBM chunk by chunk on a copy stream while the GPU computes the previous layer
 * (Alg. 1; "weight loading ... overlapping with the computation
 * of the previous layer").  Linear layers run as fused int4-g64
 * unpack+scale GEMV/GEMM kernels (§3.4) or fp16 GEMMs
 * (PAPER.md:396), attention as a decode kernel over the KV cache.
 *
 * The call sequence follows the paper's workflow (Alg. 2):
 *   pipeline_init              ~ Configure + InitModel + InitTransferSuitAndOperators
 *   load_layer_weights (xl+1)  ~ InitModel (host store: quantize, merge, pin)
 *   prefill / decode_step      ~ PipelineScheduling (Alg. 1) for one token step
 *   pipeline_stats             ~ the paper's throughput / GPU-utilisation metrics
 *   pipeline_destroy
 *
 * Conventions (all functions):
 *  - Every pointer argument is a HOST pointer unless its name ends in `_dev`.
 *  - The caller owns every pointer it passes; the library copies what it keeps
 *    before returning.  The context owns all device memory, streams, events and
 *    pinned/disk storage it allocates, and frees them in pipeline_destroy().
 *  - Calls on one context must come from one host thread at a time.  Different
 *    contexts (one per GPU / process) share no state.
 *  - Return value: PIPO_OK or an error status; pipo_last_error() gives a
 *    thread-local human-readable message for the last failing call.
 *  - After any CUDA error the context is poisoned: every later call on it returns
 *    PIPO_E_STATE (pipeline_destroy still frees it).
 *  - No CPU fallback exists: when no sm_100 device is present pipeline_init
 *    returns PIPO_E_CUDA.
 */
#ifndef PIPO_H_
#define PIPO_H_

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PIPO_ABI_VERSION 5

typedef enum {
  PIPO_OK = 0,
  PIPO_E_INVALID_ARG = 1, /* bad shape/size/pointer; SPEC.md:469 ShapeError, :226 LayoutError */
  PIPO_E_STATE = 2,       /* wrong call order (decode before prefill), poisoned context */
  PIPO_E_OOM = 3,         /* device/pinned allocation failed; SPEC.md:236 OutOfMemory */
  PIPO_E_IO = 4,          /* disk-tier read/write failure; SPEC.md:167 IoError */
  PIPO_E_FORMAT = 5,      /* disk-tier blob header/size mismatch; SPEC.md:246 FormatError */
  PIPO_E_INFEASIBLE = 6,  /* configuration cannot fit (Eq. 1) */
  PIPO_E_CUDA = 7         /* CUDA runtime error / no usable device */
} pipo_status;

typedef enum { PIPO_W_FP16 = 0, PIPO_W_INT4_G64 = 1 } pipo_wfmt;

/* Storage tiers of Eq. (1).  DEVICE = all layer weights
 * resident in HBM (no streaming; the tier-invariance reference).  HOST = pinned
 * host memory, streamed per layer.  DISK = one blob file per layer under
 * cfg.disk_dir, read by a reader-thread pool into a pinned ring, then streamed. */
typedef enum { PIPO_TIER_DEVICE = 0, PIPO_TIER_HOST = 1, PIPO_TIER_DISK = 2 } pipo_tier;

/* flags */
#define PIPO_F_TIMELINE 1u  /* record per-segment CUDA events for busy fractions (default on) */
#define PIPO_F_KPROF 2u     /* time every kernel unit with CUDA events (pipo_kernel_stats) */
/* NEXT-3 automatic configuration (§3.5, Eq. (1)): pipeline_init ignores
 * weight_tier, kv_tier, ring_layers, chunk_bytes and gemv_max_m and takes them from
 * pipo_choose_plan on this machine — M_GPU = free device memory (capped by hbm_budget),
 * M_CPU = MemAvailable, B_GPU and the block size from a pinned H2D probe (App. A),
 * B_SSD = B_GPU / 10 (not probed) — for b = max_batch, s = max_seq.  Weights on CPU put the
 * KV cache on CPU too (Eq. (1) tests W + C < M_CPU); the DISK tier needs disk_dir (else
 * PIPO_E_INFEASIBLE).  pipo_get_plan returns what was applied. */
#define PIPO_F_AUTO_PLAN 4u

typedef struct {
  int32_t device;        /* CUDA ordinal */
  /* model shape: d_model % 64 == 0, ffn_dim % 64 == 0, n_heads | d_model,
   * head_dim = d_model / n_heads in {64, 128}                                  */
  int32_t d_model, n_layers, n_heads, ffn_dim, vocab, max_pos;  /* OPT: max_pos 2048 */
  /* workload capacity: KV cache holds max_batch x max_seq positions
   * (s = prompt + generated)                                     */
  int32_t max_batch, max_seq;
  int32_t wfmt;          /* pipo_wfmt for the four decoder linear weights            */
  int32_t weight_tier;   /* pipo_tier: where decoder-layer weights live              */
  int32_t kv_tier;       /* PIPO_TIER_DEVICE or PIPO_TIER_HOST         */
  int32_t kv_fmt;        /* PIPO_W_FP16 or PIPO_W_INT4_G64: KV cache storage ("quantizing both
                            weights and KV-cache to INT4").  int4: each cached
                            row is stored in 64-feature groups with an fp16 scale; prefill
                            attends over its fresh fp16 K/V, decode reads the int4 cache   */
  int32_t ring_layers;   /* HBM weight ring depth in layers: >= 2 = performance-optimized
                            pipeline (preload next layer); 1 = memory-
                            efficient (one layer resident). 0 -> 2    */
  int64_t chunk_bytes;   /* blockwise-transfer chunk; 0 -> whole segment */
  int32_t gemv_max_m;    /* rows M <= this use the CUDA-core int4 GEMV (PAPER.md:360
                            "batch sizes less than 16") for matrices below 8 M weights;
                            larger M or matrices the tensor-core GEMM (measured faster).
                            0 -> 15                                                  */
  int32_t disk_threads;  /* DISK tier reader threads; 0 -> 4        */
  const char* disk_dir;  /* DISK tier directory (copied at init)                      */
  uint32_t flags;        /* PIPO_F_*                                                   */
  /* ---- model family (ABI 3).  PIPO_ARCH_OPT (default, 0): the OPT block above.
   * PIPO_ARCH_LLAMA: the LLaMA3.1 block the paper also evaluates (PAPER.md:318-331
   * §3.5, :390 §4.1; NEXT-4): GQA with n_kv_heads, RoPE with the llama3
   * frequency rule, RMSNorm (eps 1e-5), SwiGLU MLP with ffn_dim = d_h (PAPER.md:323,
   * ffn_dim % 128 == 0), no biases, untied LM head, no position table (max_pos only
   * bounds positions).  LLaMA + kv_fmt INT4 is not built (PIPO_E_INVALID_ARG).       */
  int32_t arch;          /* pipo_arch                                                  */
  int32_t n_kv_heads;    /* LLaMA: KV heads, divides n_heads; 0 -> n_heads             */
  float rope_theta;      /* LLaMA: RoPE base (Llama-3.1: 500000); 0 -> 10000           */
  float rope_factor;     /* llama3 rope scaling factor (8); 0 -> plain RoPE             */
  float rope_low_freq, rope_high_freq;   /* llama3 low/high_freq_factor (1, 4)          */
  int32_t rope_orig_max_pos;             /* llama3 original_max_position_embeddings (8192) */
  /* ---- placement (ABI 4).  NUMA node of the large pinned host stores (weights, host
   * KV cache) and of the disk tier's reader threads (on a
   * multi-socket node each GPU streams from its own socket's memory; App. D "isolated
   * PCIe channels").  PIPO_NUMA_GPU_LOCAL (-1): the node of the GPU's
   * PCIe root, from sysfs, when the host has more than one node; >= 0: that node
   * (pages bound with mbind, allocation fails with OOM if the node is full);
   * PIPO_NUMA_NONE (-2): the OS default placement.  NOTE: a zero-initialised config
   * asks for node 0.                                                                   */
  int32_t numa_node;
  /* device-memory budget for PIPO_F_AUTO_PLAN (M_GPU of Eq. (1)); 0 = free memory       */
  int64_t hbm_budget;
} pipo_config;

#define PIPO_NUMA_GPU_LOCAL (-1)
#define PIPO_NUMA_NONE (-2)

typedef enum { PIPO_ARCH_OPT = 0, PIPO_ARCH_LLAMA = 1 } pipo_arch;

/* fp32 masters (values must be finite; fp16-representable for exact parity).
 * Row-major.  OPT: w_qkv rows are q | k | v ([3d][d]); w_out [d][d]; w_fc1 [F][d];
 * w_fc2 [d][F]; vectors have the obvious lengths.
 * LLaMA: w_qkv [d + 2 d_kv][d] (d_kv = n_kv_heads * head_dim), w_out [d][d],
 * w_fc1 [2F][d] = gate rows then up rows, w_fc2 [d][F] (down); ln1_g / ln2_g are the
 * RMSNorm weights; every bias and ln*_b must be NULL (ignored). */
typedef struct {
  const float *ln1_g, *ln1_b, *w_qkv, *b_qkv, *w_out, *b_out;
  const float *ln2_g, *ln2_b, *w_fc1, *b_fc1, *w_fc2, *b_fc2;
} pipo_layer_weights;

/* tok [vocab][d], pos [max_pos + 2][d] (OPT learned positions, offset 2), final LN.
 * LLaMA: pos and lnf_b NULL, lnf_g = final RMSNorm weight, lm_head [vocab][d] (untied;
 * NULL for OPT, whose LM head is tok). */
typedef struct {
  const float *tok, *pos, *lnf_g, *lnf_b;
  const float *lm_head;
} pipo_embed_weights;

#define PIPO_LAYER_EMBED (-1)

typedef struct {
  int64_t prefill_calls, decode_steps, tokens_generated;
  double prefill_s, decode_s;     /* wall seconds inside prefill / decode_step calls */
  double ttft_s;                  /* last prefill call's wall time (first token)      */
  double decode_tokens_per_s;     /* b * decode_steps / decode_s                       */
  int64_t h2d_bytes, d2h_bytes;   /* streamed weight + KV bytes, token ids              */
  double h2d_gbs;                 /* h2d_bytes / copy-busy seconds (decode window)     */
  double copy_busy, kernel_busy, union_busy;  /* fractions of the decode window (Q9)   */
  double window_s;                /* decode window measured by device events           */
  int64_t kernel_launches;        /* library kernels launched since the last reset     */
  int64_t hbm_bytes;              /* device bytes allocated by the context             */
  int64_t pinned_host_bytes;      /* pinned host bytes allocated by the context        */
  int32_t numa_node;              /* node the pinned stores are bound to, -1 = none     */
  int32_t timeline_truncated;     /* PIPO_F_TIMELINE stopped recording (event cap hit)  */
  double numa_local_frac;         /* sampled pages of the weight store on numa_node (-1 n/a) */
} pipo_stats;

/* ---- lifecycle ---------------------------------------------------------- */

/* Validate cfg, select the device, allocate the HBM ring, KV cache, activation
 * workspace and resident embeddings, create streams/events.
 * Errors: INVALID_ARG (shape rules above), OOM, CUDA.  *out is NULL on error. */
typedef struct pipo_ctx pipo_ctx;
pipo_status pipeline_init(const pipo_config* cfg, pipo_ctx** out);
void pipeline_destroy(pipo_ctx* ctx);
const char* pipo_last_error(void);
int32_t pipo_abi_version(void);

/* ---- host store (InitModel) --------------------------------------------- */

/* Decoder layer `layer` in [0, n_layers), or PIPO_LAYER_EMBED with a
 * pipo_embed_weights*.  Decoder weights are quantized (wfmt INT4: SURVEY.md
 * §8(c) step 1) or rounded to fp16, merged in consumption order into one blob
 * (data merging) and placed in the layer's tier.  Embeddings
 * are always resident in HBM (reading Q20).  Synchronous; the caller may free w
 * on return.  Errors: INVALID_ARG (range, non-finite / fp16-overflowing input),
 * OOM, IO (disk tier). */
pipo_status load_layer_weights(pipo_ctx* ctx, int32_t layer, const void* w);

/* Same tensors drawn on the GPU by the library's own implementation of the
 * pipo_synth counter-based generator — used for the
 * large configurations where fp32 masters would not fit a test host.  The
 * quantizer is the same definition (bit-exact with the host path). */
pipo_status pipo_load_synthetic(pipo_ctx* ctx, int32_t layer, uint64_t seed);

/* ---- PipelineScheduling (Alg. 1) ---------------------------------------- */

/* Start a new batch: b sequences of P prompt tokens (tokens: [b][P] int32, ids
 * in [0, vocab)).  Runs every layer with M = b*P rows, writes P KV positions,
 * returns the greedy next token per sequence (next: [b]) and optionally the
 * last-position logits (logits: [b][vocab] fp32, may be NULL).
 * Errors: INVALID_ARG (b > max_batch, P >= max_seq, P + 2 > max_pos + 2),
 * STATE (missing weights). */
pipo_status prefill(pipo_ctx* ctx, const int32_t* tokens, int32_t b, int32_t P,
                    int32_t* next, float* logits);

/* One decode step for the current batch: feeds tokens[b] at position past,
 * attends over past+1 positions.  Returns next[b] and optional logits[b][vocab].
 * Errors: STATE (no prefill yet), INVALID_ARG (KV capacity max_seq exceeded). */
pipo_status decode_step(pipo_ctx* ctx, const int32_t* tokens, int32_t* next, float* logits);

/* Device-resident variant of decode_step (inputs already in HBM): tokens_dev and
 * next_dev are device int32[b] buffers (may alias: next overwrites tokens). */
pipo_status decode_step_dev(pipo_ctx* ctx, const int32_t* tokens_dev, int32_t* next_dev);

pipo_status pipeline_stats(pipo_ctx* ctx, pipo_stats* out);
pipo_status pipeline_stats_reset(pipo_ctx* ctx);

/* Change the PIPO_F_* instrumentation flags between calls (synchronises the device).
 * Timing events on the compute stream are not free while the copy engine streams
 * (~25 us each): PIPO_F_TIMELINE / PIPO_F_KPROF off gives the
 * uninstrumented step. */
pipo_status pipo_set_flags(pipo_ctx* ctx, uint32_t flags);

/* Per-kernel-class timing (needs PIPO_F_KPROF): one unit = one linear layer / one
 * attention layer / one LM head; ms from CUDA events on the compute stream around
 * each unit; bytes / flops are the ALGORITHMIC counts. */
typedef enum {
  PIPO_K_LINEAR_DECODE = 0, PIPO_K_ATTN_DECODE = 1, PIPO_K_HEAD = 2,
  PIPO_K_LINEAR_PREFILL = 3, PIPO_K_ATTN_PREFILL = 4, PIPO_K_MISC = 5, PIPO_K_COUNT = 6
} pipo_kclass;
typedef struct { int64_t units; double ms, bytes, flops; } pipo_kstats;
pipo_status pipo_kernel_stats(pipo_ctx* ctx, int32_t cls, pipo_kstats* out);

/* cudaStream_t of the compute stream (which=0) or weight-copy stream (which=1),
 * as an opaque handle for external CUDA-event timing. */
void* pipo_stream(pipo_ctx* ctx, int32_t which);

/* ---- test / measurement hooks (parity contract SURVEY.md §8(c)) ----------- */

/* Host quantizer (no GPU): w [rows][cols] fp32, cols % 64 == 0 ->
 * codes [rows][cols/2] packed (low nibble = even k), scales [rows][cols/64]
 * fp16 bits.  Errors: INVALID_ARG (non-finite, fp16-overflowing scale). */
pipo_status pipo_quantize_int4_g64(const float* w, int64_t rows, int64_t cols,
                                   uint8_t* codes, uint16_t* scales);

/* GPU quantizer (same definition), device-side; all host buffers as above. */
pipo_status pipo_quantize_int4_g64_gpu(pipo_ctx* ctx, const float* w, int64_t rows,
                                       int64_t cols, uint8_t* codes, uint16_t* scales);

/* Kernel K8: unpack + scale on the GPU: out[r][k] = fp16_rne(q * s), fp16 bits. */
pipo_status pipo_unpack_int4_g64(pipo_ctx* ctx, const uint8_t* codes, const uint16_t* scales,
                                 int64_t rows, int64_t cols, uint16_t* out);

/* One fused linear layer on the GPU through the production kernels:
 * y[M][N] = x[M][K] . W^T + bias (bias may be NULL).  x fp16 bits [M][K];
 * W given as fp32 masters [N][K] (quantized per wfmt inside); y fp32 [M][N].
 * path: 0 = automatic (as the pipeline chooses), 1 = int4 GEMV (CUDA cores),
 * 2 = mma.sync GEMM (legacy baseline), 3 = tcgen05/TMEM GEMM (synchronous pipeline),
 * 4 = warp-specialized stream-K tcgen05 GEMM (int4, A in shared memory),
 * 5 = same with A in TMEM (int4, M <= 64), 6 = prefill tcgen05 GEMM with A in TMEM
 * (int4, any M; static persistent tile schedule), 7 = streaming fp16-weight tcgen05 GEMM
 * (fp16, M <= 64: TMA-fed, warp-specialized; the fp16 decode linears), 8 = the same kernel
 * as the LM head (a13) runs it, 9 = int4 tcgen05 GEMM on SM pairs (cta_group::2, A in
 * TMEM, stream-K with the fixup inside the kernel; M <= 64: the decode linears).
 * A path that cannot run the shape returns PIPO_E_INVALID_ARG. */
pipo_status pipo_linear(pipo_ctx* ctx, int32_t wfmt, int32_t path, const uint16_t* x,
                        const float* w, const float* bias, int32_t M, int32_t N, int32_t K,
                        float* y);

/* Kernel micro-benchmark: one linear layer y[M][N] = x . W^T on device-resident
 * synthetic data (weights drawn + quantized on the GPU), `iters` back-to-back
 * launches on the compute stream, average microseconds per launch in *us.
 * Successive launches read different copies of the weights (>= 384 MB in total,
 * more than L2), so every launch streams its weights from HBM as in the pipeline;
 * environment PIPO_BENCH_HOT=1 re-reads one copy instead (L2-warm upper bound). */
pipo_status pipo_bench_linear(pipo_ctx* ctx, int32_t wfmt, int32_t path, int32_t M, int32_t N, int32_t K,
                              int32_t iters, double* us);

/* Kernel micro-benchmark: causal prefill attention (past = 0) over device-resident
 * synthetic q [b][n][d], K/V [n][b][d_kv] (n_kv_heads: 0 = MHA), average microseconds
 * per launch; variant as AttnArgs::use_cuda_cores (0 tcgen05 where it applies, 1 CUDA
 * cores, 2 mma.sync). */
pipo_status pipo_bench_attention_prefill(pipo_ctx* ctx, int32_t b, int32_t n, int32_t d, int32_t n_heads,
                                         int32_t n_kv_heads, int32_t variant, int32_t iters, double* us);

/* Measurement aid: HBM -> shared-memory streaming with cp.async.bulk, one CTA per
 * SM, `stages`-deep mbarrier ring of `chunk`-byte requests, each CTA alternating its
 * requests over `streams` contiguous regions (as a CTA that consumes several weight
 * row-tiles at once); GB/s in *gbs. */
pipo_status pipo_probe_bulk(pipo_ctx* ctx, int32_t chunk, int32_t stages, int32_t streams, double* gbs);

/* Kernel micro-benchmark: decode attention over device-resident synthetic q/K/V
 * (b sequences, L positions, d = n_heads * head_dim, n_kv_heads K/V heads: 0 = n_heads,
 * i.e. MHA; GQA otherwise), average microseconds per launch.  Launches rotate over
 * copies of K/V totalling >= 384 MB so that every launch reads its KV from HBM.
 * variant: as AttnArgs::use_cuda_cores (0 automatic). */
pipo_status pipo_bench_attention(pipo_ctx* ctx, int32_t b, int32_t L, int32_t d, int32_t n_heads, int32_t n_kv_heads,
                                 int32_t variant, int32_t iters, double* us);

/* Decode attention kernel: q [b][d] fp16 bits (pre-scaled), k/v [L][b][d] fp16
 * bits (position-major) -> o [b][d] fp32.  n_heads | d.  variant: 0 = production
 * choice (the lane-group kernel up to 1536 (b, head) pairs, one K/V row per warp above),
 * 1 = the lane-group kernel (16-B row loads), 3 = the one-row-per-warp kernel. */
pipo_status pipo_attention_decode(pipo_ctx* ctx, const uint16_t* q, const uint16_t* k,
                                  const uint16_t* v, int32_t b, int32_t L, int32_t d,
                                  int32_t n_heads, int32_t variant, float* o);

/* Prefill (causal) attention kernel: q [b][n][d] (pre-scaled) at positions
 * past..past+n-1, k/v [past+n][b][d] position-major -> o [b][n][d] fp32.
 * cuda_cores != 0 selects the CUDA-core reference kernel instead of the
 * tensor-core (mma.sync) one. */
pipo_status pipo_attention_prefill(pipo_ctx* ctx, const uint16_t* q, const uint16_t* k, const uint16_t* v,
                                   int32_t b, int32_t n, int32_t past, int32_t d, int32_t n_heads, int32_t cuda_cores,
                                   float* o);

/* Grouped-query attention (LLaMA; NEXT-4) through the production
 * kernels: q [b][n][n_heads*head_dim] fp16 bits (pre-scaled, rotated) at positions
 * past..past+n-1; k/v [past+n][b][n_kv_heads*head_dim] position-major; query head j
 * reads KV head j / (n_heads / n_kv_heads).  n == 1 runs the decode kernel, n > 1 the
 * causal prefill kernel.  o [b][n][n_heads*head_dim] fp32.  n_kv_heads | n_heads,
 * head_dim in {64, 128}.  variant (decode): 0 the production choice; 3 the CUDA-core
 * one-row-per-warp kernel; 5 / 6 the tensor-core kernel forced to 4 / 2 warps (test and
 * measurement hooks). */
pipo_status pipo_attention_gqa(pipo_ctx* ctx, const uint16_t* q, const uint16_t* k, const uint16_t* v, int32_t b,
                               int32_t n, int32_t past, int32_t n_heads, int32_t n_kv_heads, int32_t head_dim,
                               int32_t variant, float* o);

/* RoPE kernel of a LLaMA context (its n_heads, n_kv_heads, head_dim, llama3 frequencies):
 * q [b][n][n_heads*hd] fp16 bits at positions past..past+n-1 and k [past+n][b][n_kv_heads*hd]
 * (position-major; only positions past.. are rotated) -> q_out, k_out fp32, same shapes.
 * Errors: STATE (not a LLaMA context), INVALID_ARG. */
pipo_status pipo_rope(pipo_ctx* ctx, const uint16_t* q, const uint16_t* k, int32_t b, int32_t n, int32_t past,
                      float* q_out, float* k_out);

/* Capture per-layer hidden states of the next prefill/decode call:
 * on != 0 -> after that call, out receives [n_layers][b][n][d] fp32 (n = P for
 * prefill, 1 for decode).  out must stay valid until that call returns. */
pipo_status pipo_debug_capture(pipo_ctx* ctx, int32_t on, float* out);

/* Read back stored weights (parity hook for a0): rows
 * [row0, row0 + nrows) of one matrix, converted from the tiled blob layout back to
 * the CANONICAL format of pipo_quantize_int4_g64.  layer in [0, n_layers) with
 * matrix 0..3 = W_qkv, W_out, W_fc1, W_fc2 (logical rows; LLaMA FC1 = gate rows then
 * up rows), read from the DEVICE-tier store or the unsharded HOST-tier pinned store;
 * or layer = PIPO_LAYER_EMBED with matrix 0 = token table, 1 = LLaMA LM head.
 * int4 matrices fill codes [nrows][K/2] and scales [nrows][K/64] (fp16 bits);
 * fp16 matrices and embeddings fill values [nrows][K] (fp16 bits).
 * Errors: INVALID_ARG (range, NULL buffer, DISK tier or sharded store), STATE (not loaded). */
pipo_status pipo_debug_read_rows(pipo_ctx* ctx, int32_t layer, int32_t matrix, int64_t row0, int64_t nrows,
                                 uint8_t* codes, uint16_t* scales, uint16_t* values);

/* Test hooks for the method's invariance under timing and for transfer integrity
 * ("chunk checksums equal the host blob", "injected
 * delays do not change the tokens").  pipo_debug_inject: copy_delay_us > 0 enqueues a
 * busy wait of that length on the weight-copy stream before every layer's transfer
 * (a slow host link); compute_delay_us > 0 one on the compute stream before every
 * layer's kernels (slow compute); ring_checksum != 0 computes, as each layer lands in
 * its HBM ring slot, the position-weighted 64-bit checksum
 *     C = sum_i w_i * (2i + 1)  mod 2^64,  w_i = little-endian 64-bit words of the slot,
 * kept per layer (last transfer wins).  Synchronises the device; values 0 turn it off.
 * pipo_debug_ring_checksums: the per-layer checksums, out[n_layers] (STATE if never
 * enabled).  pipo_debug_read_blob: copies layer `layer`'s merged blob (layout.h) from
 * the unsharded HOST-tier pinned store, `bytes` must equal pipo_layer_blob_bytes.
 * Errors: INVALID_ARG (negative delay, range, NULL, other tiers). */
pipo_status pipo_debug_inject(pipo_ctx* ctx, int32_t copy_delay_us, int32_t compute_delay_us, int32_t ring_checksum);
pipo_status pipo_debug_ring_checksums(pipo_ctx* ctx, uint64_t* out);
pipo_status pipo_debug_read_blob(pipo_ctx* ctx, int32_t layer, uint8_t* out, int64_t bytes);
pipo_status pipo_layer_blob_bytes(pipo_ctx* ctx, int64_t* bytes);

/* H2D probe: best-of-`reps` pinned->device cudaMemcpyAsync bandwidth (GB/s) for
 * `bytes`-sized copies on the weight-copy stream (App. A sweep). */
pipo_status pipo_probe_h2d(pipo_ctx* ctx, int64_t bytes, int32_t reps, double* gbs);

/* Disk probe (the DISK tier's roofline denominator; the tier is
 * PAPER.md:285-303 §3.3): reads the payload of the n_layers blob files
 * dir/layer_<i>.pipo (as written by the DISK tier: 4 KiB header + payload) with the
 * reader pool's method — `threads` threads, O_DIRECT preads of `chunk` bytes (a 4 KiB
 * multiple) into per-thread aligned buffers, no GPU handshake — and returns payload
 * GB/s over wall time.  checksum (optional, NULL to skip; it costs CPU time) receives
 * sum over files and payload bytes of (offset + 1) * byte mod 2^64.  No CUDA calls.
 * Errors: PIPO_E_INVALID_ARG, PIPO_E_IO (missing file, short read), PIPO_E_FORMAT (bad
 * header), PIPO_E_OOM. */
pipo_status pipo_probe_disk(const char* dir, int32_t n_layers, int32_t threads, int64_t chunk, double* gbs,
                            uint64_t* checksum);

/* NUMA node of CUDA device `device`'s PCIe root (sysfs), -1 if unknown; the node a
 * PIPO_NUMA_GPU_LOCAL config binds to on a multi-node host. */
int32_t pipo_gpu_numa_node(int32_t device);

/* ---- NEXT-1: sharded weight streaming across the GPUs of one node ----------
 * App. D: with data parallelism "every GPU loads the layer", so each
 * GPU's host link carries the whole model every step.  Sharded streaming keeps the
 * batch-sharded compute (results bit-identical to one GPU) but splits the transfer:
 * rank r of `world` streams only bytes [r*S, (r+1)*S) of every layer blob (blob padded
 * to world * 4 KiB; S = padded / world) over its own host link into its HBM ring slot,
 * then an NCCL all-gather over NVLink on the copy stream fills in the other ranks'
 * ranges before the layer's segments are marked ready.  Per-rank link bytes drop by
 * `world`x; the pinned host store shrinks to l * S per rank.
 * NCCL is loaded at run time (dlopen "libnccl.so.2"; PIPO_E_CUDA if unavailable). */

/* Host-only: the rank's byte range of a blob of `layer_bytes` (after padding). */
pipo_status pipo_shard_range(int64_t layer_bytes, int32_t world, int32_t rank, int64_t* offset, int64_t* bytes);

/* ncclGetUniqueId: rank 0 creates the 128-byte id; the caller broadcasts it. */
pipo_status pipo_nccl_unique_id(uint8_t id[128]);

/* Switch a HOST-tier context to sharded streaming: call after pipeline_init and
 * before any weights are loaded, on every rank (collective: blocks until all `world`
 * ranks have joined the NCCL communicator).  world == 1 is allowed (a 1-rank
 * all-gather).  Errors: INVALID_ARG (rank/world, weight tier not HOST), STATE (weights
 * already loaded), OOM, CUDA (NCCL missing or failing). */
pipo_status pipo_shard_stream_init(pipo_ctx* ctx, int32_t rank, int32_t world, const uint8_t id[128]);

/* Peer transport for sharded streaming (no NCCL): the gather is the copy engines pulling
 * each peer's range straight out of the peer's HBM ring slot over NVLink (CUDA IPC
 * mappings), ordered by flags in peer memory (a 1-thread wait kernel before, a release
 * store after — the same ordering protocol on one box whatever the GPU count; two
 * processes may even share one GPU, which is how the N-rank path is tested on 1 GPU).
 * Every rank: (1) pipo_shard_p2p_export -> a PIPO_SHARD_HANDLE_BYTES blob (allocates the
 * padded ring + this rank's host store, nothing switched yet); the caller all-gathers the
 * blobs in rank order (any host collective); (2) pipo_shard_p2p_init with all of them
 * (opens the peers' rings; on success the context streams sharded, on failure it is
 * unchanged).  Before any weights are loaded; HOST tier; world <= 8.
 * Errors: INVALID_ARG (rank/world/tier, blob of another world), STATE (weights loaded,
 * already sharded, init without export), OOM, CUDA (IPC / peer access failure). */
#define PIPO_SHARD_HANDLE_BYTES 128
pipo_status pipo_shard_p2p_export(pipo_ctx* ctx, int32_t rank, int32_t world, uint8_t handle[PIPO_SHARD_HANDLE_BYTES]);
pipo_status pipo_shard_p2p_init(pipo_ctx* ctx, const uint8_t* handles);

/* ---- automatic configuration (NEXT-3): memory model + Eq. (1) ---------------
 * Host-only pure functions (no context, no GPU).  The paper states them for
 * LLaMA3.1 (§3.5, App. B); readings Q23-Q27 in
 * DESIGN.md.  All sizes in bytes (doubles, exact for the integer-valued results). */
typedef struct {
  int64_t n_layers, d_model, vocab;   /* l, d, V                                         */
  int64_t n_heads, n_kv_heads;        /* h, h_kv (h_kv | h; OPT: h_kv = h)               */
  int64_t ffn_hidden;                 /* d_h (LLaMA: pipo_ffn_hidden_dim; OPT: ffn_dim)  */
  int32_t mlp_mats;                   /* 3 = the paper's SwiGLU MLP, 2 = OPT fc1/fc2 (Q27) */
  double p_weight, p_act;             /* bytes/element: weights (2 fp16, 0.53125 int4-g64),
                                         activations and KV cache          */
} pipo_mem_spec;

typedef struct {
  double w_embed, w_mha, w_mlp, w_total;   /* W_embed, W_mha, W_mlp, W (§3.5)          */
  double c_total;                          /* C = 2 p b s l d h_kv / h                  */
  double m_mha, m_mlp, m_embed, m_peak;    /* App. B peaks; m_peak = max of the three   */
} pipo_mem_report;

#define PIPO_STAGE_PREFILL 0
#define PIPO_STAGE_DECODE 1

/* d_h = m * ceil(gamma * floor(8d/3) / m); -1 on bad arguments. */
int64_t pipo_ffn_hidden_dim(int64_t d, int64_t m, double gamma);

/* App. B memory model for batch b, sequence s (prompt + generated), stage
 * PIPO_STAGE_*, with (preload != 0) or without preloading.  INVALID_ARG on a bad spec. */
pipo_status pipo_memory_model(const pipo_mem_spec* spec, int64_t b, int64_t s, int32_t stage,
                              int32_t preload, pipo_mem_report* out);

typedef struct {
  double m_gpu, m_cpu;   /* available device / host memory, bytes (M_GPU, M_CPU)   */
  double b_gpu, b_ssd;   /* host->device and disk bandwidth, bytes/s (B_GPU, B_SSD) */
} pipo_hw_spec;

typedef struct {
  int32_t weight_tier;        /* pipo_tier chosen by Eq. (1)                              */
  int32_t ring_layers;        /* 2 = performance-optimized, 1 = memory-efficient pipeline */
  int32_t use_quant_kernel;   /* int4 weights and b < 16                   */
  int32_t gemv_max_m;         /* pipo_config.gemv_max_m to use (15)                       */
  int64_t block_bytes;        /* transfer block size from the probe (App. A); 0 if none   */
  double w_total, c_total;    /* W, C                                                     */
  double m_peak;              /* M (prefill with preloading)                 */
  double m_peak_no_preload;   /* prefill peak of the memory-efficient pipeline            */
} pipo_plan;

/* The plan pipeline_init applied under PIPO_F_AUTO_PLAN (STATE if the context was not
 * configured automatically). */
pipo_status pipo_get_plan(pipo_ctx* ctx, pipo_plan* out);

/* Smallest probed block size whose min-over-edges throughput (h2d, and disk when
 * disk_bps != NULL) is within 5 % of the best (App. A, reading Q26); -1 if n < 1. */
int64_t pipo_choose_block_size(const int64_t* sizes, const double* h2d_bps, const double* disk_bps,
                               int32_t n);

/* Eq. (1): weight tier and pipeline mode for workload (b, s) on
 * hardware hw; optional bandwidth profile (n_sizes entries, may be 0) picks the
 * block size.  INFEASIBLE when even the memory-efficient pipeline exceeds M_GPU. */
pipo_status pipo_choose_plan(const pipo_mem_spec* spec, int64_t b, int64_t s, const pipo_hw_spec* hw,
                             const int64_t* block_sizes, const double* h2d_bps, const double* disk_bps,
                             int32_t n_sizes, pipo_plan* out);

#ifdef __cplusplus
}
#endif
#endif /* PIPO_H_ */
