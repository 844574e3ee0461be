// kernels.h — host-side launchers of the sm_100a kernels (internal, C++).
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace pipo {

enum EpiKind { EPI_QKV = 0, EPI_RESID = 1, EPI_RELU = 2, EPI_F32 = 3, EPI_HALF = 4 };

// Fused epilogue of a linear layer (acc = x . W^T for output row m, feature n):
//  EPI_QKV  : v = acc + b; n < d -> q[m][n] = fp16(v * qscale);  d <= n < 2d -> K cache;
//             2d <= n -> V cache.  Row m = bi * n_tok + t is written at position past + t
//             of the position-major cache [pos][kv_b][d] (a6).
//  EPI_RESID: h[m][n] += acc + b          (out-proj, FC2: residual add, fp32 stream)
//  EPI_RELU : u[m][n] = fp16(relu(acc + b))  (FC1)
//  EPI_F32  : y[m][n] = acc               (LM head logits; pipo_linear hook)
//  EPI_HALF : u[m][n] = fp16(acc + b)     (LLaMA FC1 gate|up, consumed by the SwiGLU kernel)
// GQA (LLaMA): the K and V parts are dkv = n_kv_heads * head_dim wide (dkv = d for OPT).
struct EpiParams {
  int kind = EPI_F32;
  const __half* bias = nullptr;
  int M = 0, N = 0;
  __half* q = nullptr;
  __half* kc = nullptr;
  __half* vc = nullptr;
  int d = 0, n_tok = 1, past = 0, kv_b = 1;
  int dkv = 0;                // K / V width (0 -> d)
  int kv_rowmajor = 0;        // 1: k/v go to a [m][2d] staging buffer (int4-KV path)
  float qscale = 1.f;
  float* h = nullptr;
  __half* u = nullptr;
  float* y = nullptr;
  int ldy = 0;
};

struct LinearArgs {
  const __half* x = nullptr;  // [M][K] fp16, row stride K
  const uint8_t* w = nullptr; // tiled matrix (layout.h)
  int wfmt = 1;               // 1 int4-g64, 0 fp16
  int M = 0, N = 0, K = 0;
  EpiParams epi;
  float* ws = nullptr;        // split-K partials
  int64_t ws_floats = 0;
  int* counters = nullptr;    // split-K arrival counters (zeroed, self-resetting)
  int n_counters = 0;
  uint32_t* flags = nullptr;  // in-kernel stream-K fixup flags (zero at rest, self-resetting)
  int num_sms = 148;
};

enum LinearPath { PATH_AUTO = 0, PATH_GEMV = 1, PATH_GEMM = 2, PATH_TC = 3, PATH_WS = 4, PATH_TM = 5, PATH_TP = 6,
                  PATH_STREAM = 7, PATH_HEAD = 8, PATH_PAIR = 9 };

// streaming fp16-weight tcgen05 GEMM, M <= 64 (k_head.cu): the LM head (lm_head = true,
// PATH_HEAD) and the fp16 decode linears (PATH_STREAM)
int launch_linear_stream_f16(const LinearArgs& a, bool lm_head, cudaStream_t st);

// warp-specialized stream-K tcgen05 GEMM with A in TMEM, int4 weights, M <= 64
int launch_linear_tm(const LinearArgs& a, cudaStream_t st);
// the same on SM pairs (cta_group::2) with the stream-K fixup in-kernel (k_gemm_pair.cu), M <= 64
int launch_linear_pair(const LinearArgs& a, cudaStream_t st);
int launch_linear_tp(const LinearArgs& a, cudaStream_t st);

// warp-specialized stream-K tcgen05 GEMM, int4 weights (k_gemm_ws.cu)
int launch_linear_ws(const LinearArgs& a, cudaStream_t st);

// tcgen05 / TMEM fused dequant GEMM (k_gemm_tc.cu)
int launch_linear_tc(const LinearArgs& a, cudaStream_t st);

// returns the number of kernels launched (0 on a launch error -> check cudaGetLastError)
int launch_linear(const LinearArgs& a, int path, int gemv_max_m, cudaStream_t st);

// attention: q [b][d] (pre-scaled), K/V position-major [pos][kv_b][d]
struct AttnArgs {
  const __half* q = nullptr;  // decode: [b][d]; prefill: [b][n][d]
  const __half* kc = nullptr;
  const __half* vc = nullptr;
  __half* o = nullptr;        // same shape as q
  int b = 0, n = 1, past = 0, d = 0, n_heads = 0, kv_b = 0;
  int dkv = 0, group = 1;     // GQA: K/V rows dkv wide (0 -> d), query head j reads KV head j / group
  int64_t kv_pos_stride = 0;  // elements between positions (0: kv_b * d, position-major cache)
  int64_t kv_b_stride = 0;    // elements between sequences  (0: d)
  int use_cuda_cores = 0;     // prefill: 1 = the CUDA-core reference kernel
  // int4 KV cache (decode): codes [pos][kv_b][d/2] bytes, scales [pos][kv_b][d/64] fp16
  const uint8_t* kq = nullptr;
  const __half* ks = nullptr;
  const uint8_t* vq = nullptr;
  const __half* vs = nullptr;
  float* ws = nullptr;
  int64_t ws_floats = 0;
  int num_sms = 148;
};
int launch_attention_decode(const AttnArgs& a, cudaStream_t st);
int launch_attention_prefill(const AttnArgs& a, cudaStream_t st);
int launch_attention_prefill_tc(const AttnArgs& a, cudaStream_t st);   // tcgen05, key range <= 512 (else -1)

// int4 KV: quantize the fresh fp16 K/V rows (staging [b*n][2d]) into the cache at
// positions past..past+n-1 (codes [pos][kv_b][d/2], fast nibble order; scales fp16)
int launch_kv_quant(const __half* staging, int b, int n, int past, int d, int kv_b, uint8_t* kq, __half* ks,
                    uint8_t* vq, __half* vs, cudaStream_t st);
int launch_attention_decode_q4(const AttnArgs& a, cudaStream_t st);

// misc
int launch_embed(const int32_t* ids, int b, int n, int past, const __half* tok_tiled, int64_t tok_n_kb,
                 const __half* pos, int d, float* h, cudaStream_t st);
int launch_layernorm(const float* h, int64_t row_stride, int rows, int d, const __half* g,
                     const __half* beta, __half* x, cudaStream_t st);
int launch_argmax(const float* logits, int rows, int V, int ldl, int32_t* out, cudaStream_t st);
// LLaMA (NEXT-4): RMSNorm = launch_layernorm with beta == nullptr (mean taken as 0).
// RoPE (rotate-half, angle = pos * inv_freq[i], fp32 math) in place on q [b*n][n_heads*hd]
// (row m = bi*n + t at position past + t) and on the fresh K rows of the position-major
// cache [pos][kv_b][n_kv_heads*hd] at positions past .. past+n-1.
int launch_rope(__half* q, __half* kc, const float* inv_freq, int b, int n, int past, int n_heads, int n_kv_heads,
                int hd, int kv_b, cudaStream_t st);
// SwiGLU: u[m][f] = fp16(silu(g) * up) from the tile-interleaved FC1 output gu [M][2F]
// (gate of feature f = 128p + j at column 256p + j, up at 256p + 128 + j; layout.h).
int launch_swiglu(const __half* gu, int M, int F, __half* u, cudaStream_t st);
int launch_unpack_int4(const uint8_t* codes, const uint16_t* scales, int64_t rows, int64_t cols,
                       __half* out, cudaStream_t st);
// quantize fp32 masters [rows][cols] (device) -> canonical codes/scales and/or tiled blob
int launch_quantize(const float* w, int64_t rows, int64_t cols, uint8_t* codes, uint16_t* scales,
                    uint8_t* tiled, int* bad_flag, cudaStream_t st);
// fp16 tiling of fp32 masters (exact for fp16-representable input)
int launch_tile_fp16(const float* w, int64_t rows, int64_t cols, uint8_t* tiled, cudaStream_t st);
int launch_f32_to_f16(const float* src, __half* dst, int64_t n, cudaStream_t st);
int launch_f16_to_f32(const __half* src, float* dst, int64_t n, cudaStream_t st);

// measurement aid: bulk-copy streaming probe (k_probe.cu)
int launch_bulk_probe(const uint8_t* src, int64_t bytes_per_cta, int chunk, int stages, int streams, int ctas, uint32_t* sink,
                      cudaStream_t st);

// synthetic generator (pipo_synth mirror; input generation, not the method)
int launch_synth(float* out, int64_t start, int64_t count, uint64_t key, int kind, float scale,
                 cudaStream_t st);
uint64_t synth_key(uint64_t seed, uint32_t slot, uint32_t tid);
float synth_scale(int kind, double param);

// NEXT-1 peer transport (k_misc.cu): flags in peer memory, <= 8 per launch
struct P2PFlags {
  int* addr[8];
  int n;
};
int launch_p2p_wait(const P2PFlags& f, int target, cudaStream_t st);     // all *addr >= target
int launch_p2p_signal(const P2PFlags& f, int value, cudaStream_t st);
// test hooks: a busy wait of ns nanoseconds; position-weighted 64-bit checksum of a range
int launch_spin(int64_t ns, cudaStream_t st);
int launch_ring_sum(const uint8_t* p, int64_t bytes, uint64_t* out, cudaStream_t st);    // all *addr = value

}  // namespace pipo
