// layout.h — byte layout of the merged per-layer weight blob (host store, HBM ring,
// disk files).  "Data merging" (§3.3): a layer's tensors are merged
// into ONE tensor that is loaded with a single request and split into blocks.
//
// Consumption order: the blob is four segments, each holding exactly
// what one compute phase of the layer needs, so the compute stream can start a
// phase as soon as its segment has landed (a5):
//   seg 0  MHA-in : ln1_g[d] ln1_b[d] b_qkv[3d] | W_qkv [3d x d]
//   seg 1  MHA-out: b_out[d]                    | W_out [d x d]
//   seg 2  MLP-in : ln2_g[d] ln2_b[d] b_fc1[F]  | W_fc1 [F x d]
//   seg 3  MLP-out: b_fc2[d]                    | W_fc2 [d x F]
// Vectors are fp16.  Segment starts are 4 KiB aligned, matrices 256 B aligned.
//
// Matrix W [N x K] is stored "row-tile major" in blocks of 128 rows x 64 k
// (one int4 quantization group wide), N padded to a multiple of 128 with zero rows:
//   block (rt, kb) at ((rt * (K/64)) + kb) * block_bytes
//   int4 block (4352 B): codes [h=0..1][r=0..127][16 B] then scales [r] fp16 (256 B)
//        16-B chunk (h, r) = 32 codes of row r, k = kb*64 + h*32 + 0..31, as four
//        32-bit words of 8 consecutive k each.  Inside a word the codes are stored
//        OFFSET-BINARY (u = q + 8, 0..15) in nibble order e0 e2 e4 e6 e1 e3 e5 e7
//        (nibble i holds element kNibbleElem[i]) so that one shift + four LOP3 yield
//        the fp16 pairs (e0,e1) (e2,e3) (e4,e5) (e6,e7) (common.cuh dequant8).
//        (The canonical packing of the hooks/oracle — two's complement, low nibble =
//        even k — is a different, documented format.)
//   fp16 block (16384 B): [r=0..127][64] row-major halves
// so that one 128-row strip of the matrix is contiguous (rows land in order) and a
// CTA reads each k-block of its strip as one contiguous 4.25 KiB / 16 KiB piece.
#pragma once
#include <stdint.h>

#ifdef __CUDACC__
#define PIPO_HD __host__ __device__
#else
#define PIPO_HD
#endif

namespace pipo {

constexpr int kTileRows = 128;
constexpr int kTileK = 64;
constexpr int64_t kInt4BlockBytes = 4096 + 256;
constexpr int64_t kFp16BlockBytes = kTileRows * kTileK * 2;

inline int64_t round_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

struct MatLayout {
  int64_t N = 0, K = 0, N_pad = 0, n_rt = 0, n_kb = 0, block_bytes = 0, bytes = 0;
  int wfmt = 1;  // 1 int4, 0 fp16
};

inline MatLayout mat_layout(int64_t N, int64_t K, int wfmt) {
  MatLayout m;
  m.N = N; m.K = K; m.wfmt = wfmt;
  m.N_pad = round_up(N, kTileRows);
  m.n_rt = m.N_pad / kTileRows;
  m.n_kb = K / kTileK;
  m.block_bytes = wfmt == 1 ? kInt4BlockBytes : kFp16BlockBytes;
  m.bytes = m.n_rt * m.n_kb * m.block_bytes;
  return m;
}

// element offset (in halves) of (r, k) inside an fp16 tiled matrix
PIPO_HD inline int64_t fp16_tiled_index(int64_t r, int64_t k, int64_t n_kb) {
  return (((r >> 7) * n_kb + (k >> 6)) << 13) + ((r & 127) << 6) + (k & 63);
}

// word-internal code order of the tiled int4 block
constexpr int kNibbleElem[8] = {0, 2, 4, 6, 1, 3, 5, 7};

// pack 8 signed codes (natural k order) into one tiled-layout word
PIPO_HD inline uint32_t pack_tiled_word(const int* q8) {
  const int pos_of_elem[8] = {0, 4, 1, 5, 2, 6, 3, 7};
  uint32_t w = 0;
  for (int e = 0; e < 8; ++e) w |= (uint32_t)((q8[e] + 8) & 0xF) << (4 * pos_of_elem[e]);
  return w;
}

enum Vec { V_LN1_G, V_LN1_B, V_B_QKV, V_B_OUT, V_LN2_G, V_LN2_B, V_B_FC1, V_B_FC2, V_COUNT };
enum Mat { M_QKV, M_OUT, M_FC1, M_FC2, M_COUNT };

struct LayerLayout {
  int64_t seg_off[4], seg_bytes[4];
  int64_t vec_off[V_COUNT], vec_len[V_COUNT];
  int64_t mat_off[M_COUNT];
  MatLayout mat[M_COUNT];
  int64_t total = 0;
  bool glu = false;   // LLaMA: W_fc1 is [gate | up], stored tile-interleaved (below)
};

// OPT (llama = false): QKV [3d x d], FC1 [F x d], every bias and LN beta present.
// LLaMA (NEXT-4): QKV [(d + 2 dkv) x d] (GQA), no biases / betas (length
// 0), FC1 = [gate; up] [2F x d] stored TILE-INTERLEAVED: 128-row tile 2p holds gate rows
// 128p..128p+127 and tile 2p+1 the up rows of the same features, so the two
// accumulators a SwiGLU output needs sit in adjacent tiles (F % 128 == 0).
inline LayerLayout layer_layout(int64_t d, int64_t F, int wfmt, int64_t dkv = -1, bool llama = false) {
  LayerLayout L;
  if (dkv < 0) dkv = d;
  L.glu = llama;
  L.mat[M_QKV] = mat_layout(d + 2 * dkv, d, wfmt);
  L.mat[M_OUT] = mat_layout(d, d, wfmt);
  L.mat[M_FC1] = mat_layout(llama ? 2 * F : F, d, wfmt);
  L.mat[M_FC2] = mat_layout(d, F, wfmt);
  const int seg_vecs[4][3] = {{V_LN1_G, V_LN1_B, V_B_QKV}, {V_B_OUT, -1, -1},
                              {V_LN2_G, V_LN2_B, V_B_FC1}, {V_B_FC2, -1, -1}};
  const int64_t z = llama ? 0 : 1;
  const int64_t len[V_COUNT] = {d, z * d, z * (d + 2 * dkv), z * d, d, z * d, z * F, z * d};
  int64_t off = 0;
  for (int s = 0; s < 4; ++s) {
    off = round_up(off, 4096);
    L.seg_off[s] = off;
    for (int i = 0; i < 3; ++i) {
      int v = seg_vecs[s][i];
      if (v < 0) continue;
      L.vec_off[v] = off;
      L.vec_len[v] = len[v];
      off += len[v] * 2;
    }
    off = round_up(off, 256);
    L.mat_off[s] = off;
    off += L.mat[s].bytes;
    L.seg_bytes[s] = off - L.seg_off[s];
  }
  L.total = round_up(off, 4096);
  return L;
}

}  // namespace pipo
