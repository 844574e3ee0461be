// disk.cpp — the DISK weight tier (§3.3, Fig. 3/4).
//
// Each decoder layer's merged blob is one file: a 4 KiB header (magic, version,
// layer, payload size, layout hash) followed by the blob.  A pool of reader threads
// ("multi-thread parallel transfer") reads fixed-size chunks with
// O_DIRECT into a ring of pinned, device-mapped staging slots ("blockwise transfer",
// the disk->host read of chunk k+1 overlaps the host->device copy
// of chunk k).  Handshake without any host thread on the copy path:
//   reader:  wait free[slot] >= seq-1 (GPU finished the previous use), pread, then
//            ready[slot] = seq                      ("signals the GPU thread", :295)
//   copy stream: cuStreamWaitValue32(ready[slot] >= seq) -> cudaMemcpyAsync(H2D)
//            -> cuStreamWriteValue32(free[slot] = seq)
// so the copy stream consumes each chunk as soon as it has landed in host memory.
#include <cuda.h>
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "disk.h"

namespace pipo {

namespace {
using PFN_wait = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
using PFN_write = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

struct Req {
  int fd;
  int64_t off, len;
  int slot;
  uint32_t seq;
};
}  // namespace

struct DiskTier {
  std::string dir;
  int nthreads = 4, nslots = 8;
  int64_t slot_bytes = 32ll << 20;
  uint8_t* staging = nullptr;
  volatile uint32_t* ready = nullptr;
  volatile uint32_t* freef = nullptr;
  CUdeviceptr ready_dev = 0, free_dev = 0;
  std::vector<int> fds;
  std::vector<uint32_t> slot_seq;
  int next_slot = 0;
  std::deque<Req> q;
  std::mutex mu;
  std::condition_variable cv;
  bool stop = false;
  std::vector<std::thread> th;
  std::atomic<int> io_error{0};
  std::atomic<int64_t> reads{0};
  int64_t fail_at = -1, delay_us = 0;
  bool direct = true;
  PFN_wait wait32 = nullptr;
  PFN_write write32 = nullptr;
};

static uint64_t layout_hash(const pipo_ctx* ctx) {
  uint64_t h = 1469598103934665603ull;
  auto mix = [&](int64_t v) { h = (h ^ (uint64_t)v) * 1099511628211ull; };
  mix(ctx->d); mix(ctx->F); mix(ctx->wfmt); mix(ctx->layer_bytes); mix(ctx->arch); mix(ctx->dkv);
  return h;
}

static void reader_loop(DiskTier* dt) {
  for (;;) {
    Req r;
    {
      std::unique_lock<std::mutex> lk(dt->mu);
      dt->cv.wait(lk, [&] { return dt->stop || !dt->q.empty(); });
      if (dt->stop) return;
      r = dt->q.front();
      dt->q.pop_front();
    }
    // wait until the GPU has copied out the slot's previous chunk
    while ((int32_t)(dt->freef[r.slot] - (r.seq - 1)) < 0) {
      if (dt->stop) return;
      std::this_thread::sleep_for(std::chrono::microseconds(20));
    }
    const int64_t nth = dt->reads.fetch_add(1);
    if (dt->delay_us > 0) std::this_thread::sleep_for(std::chrono::microseconds(dt->delay_us * (1 + nth % 3)));
    uint8_t* dst = dt->staging + (int64_t)r.slot * dt->slot_bytes;
    int64_t done = 0;
    bool ok = dt->fail_at < 0 || nth != dt->fail_at;
    while (ok && done < r.len) {
      const ssize_t n = pread(r.fd, dst + done, (size_t)(r.len - done), r.off + done);
      if (n <= 0) { ok = false; break; }
      done += n;
    }
    if (!ok) dt->io_error = 1;
    std::atomic_thread_fence(std::memory_order_release);
    dt->ready[r.slot] = r.seq;   // the copy stream's cuStreamWaitValue32 sees it
  }
}

pipo_status disk_open(pipo_ctx* ctx, int threads) {
  DiskTier* dt = new DiskTier();
  ctx->disk = dt;
  dt->dir = ctx->disk_dir;
  dt->nthreads = threads;
  if (ctx->chunk > 0) dt->slot_bytes = (ctx->chunk + 4095) / 4096 * 4096;
  if (const char* e = getenv("PIPO_DISK_FAIL_AT")) dt->fail_at = atoll(e);
  if (const char* e = getenv("PIPO_DISK_DELAY_US")) dt->delay_us = atoll(e);
  mkdir(dt->dir.c_str(), 0755);
  cudaDriverEntryPointQueryResult q1, q2;
  if (cudaGetDriverEntryPoint("cuStreamWaitValue32", reinterpret_cast<void**>(&dt->wait32), cudaEnableDefault,
                              &q1) != cudaSuccess ||
      cudaGetDriverEntryPoint("cuStreamWriteValue32", reinterpret_cast<void**>(&dt->write32), cudaEnableDefault,
                              &q2) != cudaSuccess ||
      !dt->wait32 || !dt->write32) {
    cudaGetLastError();
    return PIPO_E_CUDA;
  }
  void* p = nullptr;
  if (cudaHostAlloc(&p, (size_t)(dt->nslots * dt->slot_bytes), cudaHostAllocMapped) != cudaSuccess) {
    cudaGetLastError();
    return PIPO_E_OOM;
  }
  dt->staging = static_cast<uint8_t*>(p);
  ctx->pinned_bytes += dt->nslots * dt->slot_bytes;
  if (cudaHostAlloc(&p, 2 * 64 * sizeof(uint32_t), cudaHostAllocMapped) != cudaSuccess) {
    cudaGetLastError();
    return PIPO_E_OOM;
  }
  std::memset(p, 0, 2 * 64 * sizeof(uint32_t));
  dt->ready = static_cast<uint32_t*>(p);
  dt->freef = static_cast<uint32_t*>(p) + 64;
  void* dp = nullptr;
  if (cudaHostGetDevicePointer(&dp, p, 0) != cudaSuccess) { cudaGetLastError(); return PIPO_E_CUDA; }
  dt->ready_dev = reinterpret_cast<CUdeviceptr>(dp);
  dt->free_dev = dt->ready_dev + 64 * sizeof(uint32_t);
  dt->slot_seq.assign(dt->nslots, 0);
  dt->fds.assign(ctx->l, -1);
  for (int i = 0; i < dt->nthreads; ++i) dt->th.emplace_back(reader_loop, dt);
  return PIPO_OK;
}

void disk_close(pipo_ctx* ctx) {
  DiskTier* dt = ctx->disk;
  if (!dt) return;
  {
    std::lock_guard<std::mutex> lk(dt->mu);
    dt->stop = true;
  }
  dt->cv.notify_all();
  for (auto& t : dt->th) t.join();
  for (int fd : dt->fds)
    if (fd >= 0) close(fd);
  if (dt->staging) cudaFreeHost(dt->staging);
  if (dt->ready) cudaFreeHost(const_cast<uint32_t*>(dt->ready));
  delete dt;
  ctx->disk = nullptr;
}

static pipo_status open_layer(pipo_ctx* ctx, int layer) {
  DiskTier* dt = ctx->disk;
  if (dt->fds[layer] >= 0) return PIPO_OK;
  const std::string path = blob_path(dt->dir, layer);
  int fd = open(path.c_str(), O_RDONLY | O_DIRECT);
  if (fd < 0) {
    fd = open(path.c_str(), O_RDONLY);   // filesystems without O_DIRECT (tmpfs)
    dt->direct = false;
  }
  if (fd < 0) return PIPO_E_IO;
  BlobFileHeader hd;
  void* buf = nullptr;
  if (posix_memalign(&buf, 4096, sizeof hd) != 0) { close(fd); return PIPO_E_OOM; }
  const ssize_t n = pread(fd, buf, sizeof hd, 0);
  std::memcpy(&hd, buf, sizeof hd);
  free(buf);
  if (n != (ssize_t)sizeof hd) { close(fd); return PIPO_E_IO; }
  if (std::memcmp(hd.magic, "PIPOBLB1", 8) != 0 || hd.version != 1 || hd.layer != (uint32_t)layer ||
      hd.payload_bytes != (uint64_t)ctx->layer_bytes || hd.layout_hash != layout_hash(ctx)) {
    close(fd);
    return PIPO_E_FORMAT;
  }
  dt->fds[layer] = fd;
  return PIPO_OK;
}

pipo_status disk_write_layer(pipo_ctx* ctx, int layer, const uint8_t* blob) {
  DiskTier* dt = ctx->disk;
  if (!dt) return PIPO_E_STATE;
  if (dt->fds[layer] >= 0) { close(dt->fds[layer]); dt->fds[layer] = -1; }
  const std::string path = blob_path(dt->dir, layer);
  const int fd = open(path.c_str(), O_WRONLY | O_CREAT | O_TRUNC, 0644);
  if (fd < 0) return PIPO_E_IO;
  BlobFileHeader hd;
  std::memset(&hd, 0, sizeof hd);
  std::memcpy(hd.magic, "PIPOBLB1", 8);
  hd.version = 1;
  hd.layer = (uint32_t)layer;
  hd.payload_bytes = (uint64_t)ctx->layer_bytes;
  hd.layout_hash = layout_hash(ctx);
  bool ok = write(fd, &hd, sizeof hd) == (ssize_t)sizeof hd;
  int64_t done = 0;
  while (ok && done < ctx->layer_bytes) {
    const ssize_t n = write(fd, blob + done, (size_t)(ctx->layer_bytes - done));
    if (n <= 0) ok = false;
    else done += n;
  }
  ok = ok && fsync(fd) == 0;
  // drop the file from the page cache so reads measure the disk (O_DIRECT reads bypass it anyway)
  posix_fadvise(fd, 0, 0, POSIX_FADV_DONTNEED);
  close(fd);
  if (!ok) return PIPO_E_IO;
  return open_layer(ctx, layer);
}

pipo_status disk_enqueue_segment(pipo_ctx* ctx, int layer, int seg, uint8_t* dst) {
  DiskTier* dt = ctx->disk;
  if (dt->io_error) return PIPO_E_IO;
  pipo_status s = open_layer(ctx, layer);
  if (s != PIPO_OK) return s;
  const int64_t bytes = ctx->lay.seg_bytes[seg];
  const int64_t file_off = (int64_t)sizeof(BlobFileHeader) + ctx->lay.seg_off[seg];
  for (int64_t off = 0; off < bytes; off += dt->slot_bytes) {
    const int64_t n = std::min(dt->slot_bytes, bytes - off);
    const int slot = dt->next_slot;
    dt->next_slot = (dt->next_slot + 1) % dt->nslots;
    const uint32_t seq = ++dt->slot_seq[slot];
    {
      std::lock_guard<std::mutex> lk(dt->mu);
      dt->q.push_back(Req{dt->fds[layer], file_off + off, (n + 4095) / 4096 * 4096, slot, seq});
    }
    dt->cv.notify_one();
    CUstream st = reinterpret_cast<CUstream>(ctx->s_copy);
    if (dt->wait32(st, dt->ready_dev + slot * 4, seq, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS) return PIPO_E_CUDA;
    if (cudaMemcpyAsync(dst + off, dt->staging + (int64_t)slot * dt->slot_bytes, (size_t)n, cudaMemcpyHostToDevice,
                        ctx->s_copy) != cudaSuccess)
      return PIPO_E_CUDA;
    if (dt->write32(st, dt->free_dev + slot * 4, seq, CU_STREAM_WRITE_VALUE_DEFAULT) != CUDA_SUCCESS)
      return PIPO_E_CUDA;
  }
  return PIPO_OK;
}

int disk_io_error(pipo_ctx* ctx) { return ctx->disk ? ctx->disk->io_error.load() : 0; }

}  // namespace pipo

// ---------------------------------------------------------------------------------
// Disk roofline probe (the disk tier's denominator).  The same read
// path as the reader pool above — one file per layer, O_DIRECT, fixed-size chunks
// handed to `threads` reader threads, each pread into its own aligned buffer — minus
// the GPU handshake, so it bounds what the tier can reach.  No CUDA calls: it runs
// without a GPU.
extern "C" pipo_status pipo_probe_disk(const char* dir, int32_t n_layers, int32_t threads, int64_t chunk, double* gbs,
                                       uint64_t* checksum) {
  using namespace pipo;
  if (!dir || n_layers <= 0 || threads <= 0 || threads > 64 || chunk < 4096 || chunk % 4096 || !gbs)
    return PIPO_E_INVALID_ARG;
  struct PReq {
    int fd;
    int64_t off, len, valid;   // file offset, bytes requested (4 KiB multiple), payload bytes in it
    int64_t pos;               // payload offset of the chunk (checksum weights)
  };
  std::vector<int> fds;
  std::vector<PReq> reqs;
  int64_t total = 0;
  auto close_all = [&] {
    for (int fd : fds) close(fd);
  };
  void* hbuf = nullptr;
  if (posix_memalign(&hbuf, 4096, sizeof(BlobFileHeader)) != 0) return PIPO_E_OOM;
  for (int l = 0; l < n_layers; ++l) {
    const std::string path = blob_path(dir, l);
    int fd = open(path.c_str(), O_RDONLY | O_DIRECT);
    if (fd < 0) fd = open(path.c_str(), O_RDONLY);
    if (fd < 0) { free(hbuf); close_all(); return PIPO_E_IO; }
    fds.push_back(fd);
    BlobFileHeader hd;
    if (pread(fd, hbuf, sizeof hd, 0) != (ssize_t)sizeof hd) { free(hbuf); close_all(); return PIPO_E_IO; }
    std::memcpy(&hd, hbuf, sizeof hd);
    if (std::memcmp(hd.magic, "PIPOBLB1", 8) != 0 || hd.version != 1 || hd.layer != (uint32_t)l) {
      free(hbuf); close_all(); return PIPO_E_FORMAT;
    }
    const int64_t pb = (int64_t)hd.payload_bytes;
    for (int64_t off = 0; off < pb; off += chunk) {
      const int64_t v = std::min(chunk, pb - off);
      reqs.push_back(PReq{fd, (int64_t)sizeof(BlobFileHeader) + off, (v + 4095) / 4096 * 4096, v, off});
    }
    total += pb;
  }
  free(hbuf);
  std::atomic<size_t> next{0};
  std::atomic<int> err{0};
  std::atomic<uint64_t> sum{0};
  auto reader = [&] {
    void* p = nullptr;
    if (posix_memalign(&p, 4096, (size_t)chunk) != 0) { err = 1; return; }
    uint8_t* buf = static_cast<uint8_t*>(p);
    uint64_t local = 0;
    for (size_t i = next.fetch_add(1); i < reqs.size() && !err; i = next.fetch_add(1)) {
      const PReq& r = reqs[i];
      int64_t done = 0;
      while (done < r.len) {
        const ssize_t n = pread(r.fd, buf + done, (size_t)(r.len - done), r.off + done);
        if (n < 0) { err = 1; break; }
        if (n == 0) break;   // end of file (the last request is rounded up to 4 KiB)
        done += n;
      }
      if (done < r.valid) err = 1;
      if (checksum)   // position-weighted: sum_j (pos + j + 1) * byte_j mod 2^64
        for (int64_t j = 0; j < r.valid; ++j) local += (uint64_t)(r.pos + j + 1) * buf[j];
    }
    sum += local;
    free(p);
  };
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> th;
  for (int i = 0; i < threads; ++i) th.emplace_back(reader);
  for (auto& t : th) t.join();
  const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  close_all();
  if (err) return PIPO_E_IO;
  *gbs = s > 0 ? (double)total / s / 1e9 : 0.0;
  if (checksum) *checksum = sum.load();
  return PIPO_OK;
}
