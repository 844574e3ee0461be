// host.h — host-side (C++) pieces of the library: the int4-g64 quantizer/packer
// that builds the merged per-layer blob (a0, "data merging" PAPER.md:297-300), fp16
// conversions, a small parallel-for, and the disk-tier blob files.
#pragma once
#include <stdint.h>

#include <functional>
#include <string>

#include "layout.h"
#include "../../include/pipo.h"

namespace pipo {

uint16_t f32_to_f16_rne(float f);
float f16_to_f32(uint16_t h);

void parallel_for(int64_t n, const std::function<void(int64_t, int64_t)>& fn, int max_threads = 0);

// SURVEY.md §8(c) step 1, canonical layout (codes [rows][cols/2], scales [rows][cols/64]).
// Returns false for non-finite input or an fp16-overflowing scale.
bool quantize_canonical(const float* w, int64_t rows, int64_t cols, uint8_t* codes, uint16_t* scales);
// Same definition, written straight into the tiled matrix layout (layout.h).
bool quantize_tiled(const float* w, int64_t rows, int64_t cols, uint8_t* tiled);
void tile_fp16(const float* w, int64_t rows, int64_t cols, uint8_t* tiled);

// Build a decoder layer's merged blob (layout.h) from fp32 masters.
bool build_layer_blob(const pipo_layer_weights* w, const LayerLayout& L, int wfmt, uint8_t* blob);

// Disk tier: one file per layer, header + payload, O_DIRECT-aligned.
struct BlobFileHeader {
  char magic[8];        // "PIPOBLB1"
  uint32_t version;     // 1
  uint32_t layer;
  uint64_t payload_bytes;
  uint64_t layout_hash;
  uint8_t pad[4096 - 32];
};
static_assert(sizeof(BlobFileHeader) == 4096, "header must be one O_DIRECT block");
std::string blob_path(const std::string& dir, int layer);

// thread-local pipo_last_error() message (defined in api.cu); returns s
pipo_status set_last_error(pipo_status s, const char* msg);

}  // namespace pipo
