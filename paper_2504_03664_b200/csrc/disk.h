// disk.h — DISK weight tier (§3.3): one blob file per
// layer, read by a reader-thread pool (multi-thread parallel transfer) into a pinned
// staging ring (blockwise transfer), then copied H2D on the weight-copy stream.
#pragma once
#include "ctx.h"

namespace pipo {
pipo_status disk_open(pipo_ctx* ctx, int threads);
void disk_close(pipo_ctx* ctx);
pipo_status disk_write_layer(pipo_ctx* ctx, int layer, const uint8_t* blob);
// enqueue (on ctx->s_copy) the transfer of segment `seg` of layer `layer` into dst
pipo_status disk_enqueue_segment(pipo_ctx* ctx, int layer, int seg, uint8_t* dst);
// non-zero once a reader thread failed a read (the call then returns PIPO_E_IO)
int disk_io_error(pipo_ctx* ctx);
}  // namespace pipo
