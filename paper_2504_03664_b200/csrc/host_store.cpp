// host_store.cpp — host store build (a0): int4-g64 quantize + pack into the merged,
// tiled per-layer blob; fp16 merge for the fp16 path.  Multithreaded over row
// strips.  No fast-math: the quantizer's IEEE fp32 division, RNE rint and RNE
// fp16 conversion are what make it bit-exact with the oracle and the GPU quantizer.
#include <cmath>
#include <cstring>
#include <thread>
#include <vector>
#include <atomic>
#include <algorithm>

#include "host.h"

namespace pipo {

uint16_t f32_to_f16_rne(float f) {
  uint32_t x;
  std::memcpy(&x, &f, 4);
  const uint32_t sign = (x >> 16) & 0x8000u;
  x &= 0x7fffffffu;
  if (x >= 0x7f800000u) return (uint16_t)(sign | (x > 0x7f800000u ? 0x7e00u : 0x7c00u));
  if (x >= 0x477ff000u) return (uint16_t)(sign | 0x7c00u);   // >= 65520 rounds to inf
  if (x < 0x33000000u) return (uint16_t)sign;                // < 2^-25 rounds to 0
  const uint32_t e = x >> 23;
  if (e < 113) {                                             // fp16 subnormal
    const uint32_t m = (x & 0x7fffffu) | 0x800000u;
    const uint32_t shift = 126 - e;
    uint32_t mh = m >> shift;
    const uint32_t rem = m & ((1u << shift) - 1), half = 1u << (shift - 1);
    if (rem > half || (rem == half && (mh & 1u))) ++mh;
    return (uint16_t)(sign | mh);
  }
  uint32_t h = ((e - 112) << 10) | ((x >> 13) & 0x3ffu);
  const uint32_t rem = x & 0x1fffu;
  if (rem > 0x1000u || (rem == 0x1000u && (h & 1u))) ++h;
  return (uint16_t)(sign | h);
}

float f16_to_f32(uint16_t h) {
  const uint32_t sign = (uint32_t)(h & 0x8000u) << 16;
  uint32_t e = (h >> 10) & 0x1f, m = h & 0x3ffu, x;
  if (e == 0) {
    if (m == 0) {
      x = sign;
    } else {
      e = 113;
      while (!(m & 0x400u)) { m <<= 1; --e; }
      x = sign | (e << 23) | ((m & 0x3ffu) << 13);
    }
  } else if (e == 31) {
    x = sign | 0x7f800000u | (m << 13);
  } else {
    x = sign | ((e + 112) << 23) | (m << 13);
  }
  float f;
  std::memcpy(&f, &x, 4);
  return f;
}

void parallel_for(int64_t n, const std::function<void(int64_t, int64_t)>& fn, int max_threads) {
  int nt = (int)std::thread::hardware_concurrency();
  if (max_threads > 0) nt = std::min(nt, max_threads);
  nt = (int)std::max<int64_t>(1, std::min<int64_t>(nt, n));
  if (nt <= 1) { fn(0, n); return; }
  std::vector<std::thread> th;
  const int64_t per = (n + nt - 1) / nt;
  for (int t = 0; t < nt; ++t) {
    const int64_t a = t * per, b = std::min(n, a + per);
    if (a >= b) break;
    th.emplace_back([&fn, a, b] { fn(a, b); });
  }
  for (auto& t : th) t.join();
}

// one group: returns false on a domain error; writes 64 signed codes + scale bits
static inline bool quant_codes(const float* g, int* q, uint16_t* scale_bits) {
  float a = 0.f;
  bool ok = true;
  for (int i = 0; i < 64; ++i) {
    ok = ok && std::isfinite(g[i]);
    a = std::max(a, std::fabs(g[i]));
  }
  const volatile float a7 = a / 7.0f;                 // IEEE fp32 division
  const uint16_t sb = f32_to_f16_rne(a7);
  const float s = f16_to_f32(sb);
  if (!std::isfinite(s)) ok = false;
  for (int i = 0; i < 64; ++i) {
    q[i] = 0;
    if (s != 0.f) {
      const volatile float r = g[i] / s;             // IEEE fp32 division
      q[i] = (int)std::min(7.f, std::max(-8.f, std::nearbyintf(r)));   // RNE
    }
  }
  *scale_bits = sb;
  return ok;
}

// one group in the canonical packing: 32 bytes (low nibble = even k, two's complement)
static inline bool quant_group(const float* g, uint8_t* packed, uint16_t* scale_bits) {
  int q[64];
  const bool ok = quant_codes(g, q, scale_bits);
  for (int i = 0; i < 32; ++i) packed[i] = (uint8_t)((q[2 * i] & 0xF) | ((q[2 * i + 1] & 0xF) << 4));
  return ok;
}

bool quantize_canonical(const float* w, int64_t rows, int64_t cols, uint8_t* codes, uint16_t* scales) {
  if (cols % 64 != 0) return false;
  std::atomic<bool> ok{true};
  const int64_t ng = cols / 64;
  parallel_for(rows, [&](int64_t r0, int64_t r1) {
    bool good = true;
    for (int64_t r = r0; r < r1; ++r)
      for (int64_t c = 0; c < ng; ++c)
        good &= quant_group(w + r * cols + c * 64, codes + r * (cols / 2) + c * 32, scales + r * ng + c);
    if (!good) ok = false;
  });
  return ok;
}

// One 128-row tile of the tiled layout: `src` -> rows 0..nrows-1 (zero rows beyond),
// n_kb k-blocks written at `dst` (the tile's first block).
static bool quantize_one_tile(const float* src, int64_t nrows, int64_t cols, uint8_t* dst) {
  const int64_t n_kb = cols / 64;
  const float zeros[64] = {0};
  bool good = true;
  for (int64_t kb = 0; kb < n_kb; ++kb) {
    uint8_t* blk = dst + kb * kInt4BlockBytes;
    for (int rr = 0; rr < 128; ++rr) {
      uint16_t sb;
      int q[64];
      good &= quant_codes(rr < nrows ? src + rr * cols + kb * 64 : zeros, q, &sb);
      uint32_t words[8];
      for (int wi = 0; wi < 8; ++wi) words[wi] = pack_tiled_word(q + wi * 8);
      std::memcpy(blk + (0 * 128 + rr) * 16, words, 16);
      std::memcpy(blk + (1 * 128 + rr) * 16, words + 4, 16);
      std::memcpy(blk + 4096 + rr * 2, &sb, 2);
    }
  }
  return good;
}

static void tile_fp16_one(const float* src, int64_t nrows, int64_t cols, uint8_t* dst) {
  const int64_t n_kb = cols / 64;
  uint16_t* out = reinterpret_cast<uint16_t*>(dst);
  for (int64_t rr = 0; rr < 128; ++rr)
    for (int64_t k = 0; k < cols; ++k)
      out[fp16_tiled_index(rr, k, n_kb)] = rr < nrows ? f32_to_f16_rne(src[rr * cols + k]) : 0;
}

// tile t of the stored matrix <- master rows row_of_tile(t) .. +127 (identity order, or
// the GLU interleave: tile 2p = gate rows 128p.., tile 2p+1 = up rows F + 128p..)
static bool tile_matrix(const float* w, int64_t rows, int64_t cols, int wfmt, bool glu, uint8_t* tiled) {
  if (cols % 64 != 0) return false;
  const MatLayout m = mat_layout(rows, cols, wfmt);
  const int64_t half = rows / 2;
  std::atomic<bool> ok{true};
  parallel_for(m.n_rt, [&](int64_t t0, int64_t t1) {
    bool good = true;
    for (int64_t t = t0; t < t1; ++t) {
      const int64_t r0 = glu ? (t & 1) * half + (t >> 1) * 128 : t * 128;
      const int64_t end = glu ? (t & 1) * half + half : rows;
      const int64_t nr = std::min<int64_t>(128, end - r0);
      uint8_t* dst = tiled + t * m.n_kb * m.block_bytes;
      if (wfmt == PIPO_W_INT4_G64) good &= quantize_one_tile(w + r0 * cols, nr, cols, dst);
      else tile_fp16_one(w + r0 * cols, nr, cols, dst);
    }
    if (!good) ok = false;
  });
  return ok;
}

bool quantize_tiled(const float* w, int64_t rows, int64_t cols, uint8_t* tiled) {
  return tile_matrix(w, rows, cols, PIPO_W_INT4_G64, false, tiled);
}

void tile_fp16(const float* w, int64_t rows, int64_t cols, uint8_t* tiled) {
  tile_matrix(w, rows, cols, PIPO_W_FP16, false, tiled);
}

bool build_layer_blob(const pipo_layer_weights* w, const LayerLayout& L, int wfmt, uint8_t* blob) {
  std::memset(blob, 0, (size_t)L.total);
  const float* vecs[V_COUNT] = {w->ln1_g, w->ln1_b, w->b_qkv, w->b_out, w->ln2_g, w->ln2_b, w->b_fc1, w->b_fc2};
  for (int v = 0; v < V_COUNT; ++v) {
    if (L.vec_len[v] == 0) continue;   // LLaMA: no biases / betas
    if (!vecs[v]) return false;
    uint16_t* dst = reinterpret_cast<uint16_t*>(blob + L.vec_off[v]);
    for (int64_t i = 0; i < L.vec_len[v]; ++i) {
      if (!std::isfinite(vecs[v][i])) return false;
      dst[i] = f32_to_f16_rne(vecs[v][i]);
    }
  }
  const float* mats[M_COUNT] = {w->w_qkv, w->w_out, w->w_fc1, w->w_fc2};
  for (int i = 0; i < M_COUNT; ++i) {
    if (!mats[i]) return false;
    if (!tile_matrix(mats[i], L.mat[i].N, L.mat[i].K, wfmt, L.glu && i == M_FC1, blob + L.mat_off[i])) return false;
  }
  return true;
}

std::string blob_path(const std::string& dir, int layer) {
  return dir + "/layer_" + std::to_string(layer) + ".pipo";
}

}  // namespace pipo
