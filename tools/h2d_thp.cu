// H2D throughput of a large pinned host buffer: cudaHostAlloc vs mmap + MADV_HUGEPAGE +
// cudaHostRegister (transparent huge pages -> fewer IOMMU/ATS translations per byte).
// Streams the whole buffer in `chunk`-byte copies (like the weight stream), 3 passes.
//   nvcc -O2 -o /tmp/h2d_thp tools/h2d_thp.cu && /tmp/h2d_thp 4096 128
#include <cuda_runtime.h>
#include <sys/mman.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>

static double stream(const char* name, char* h, size_t bytes, size_t chunk, char* d, size_t dbytes) {
  cudaStream_t st;
  cudaStreamCreate(&st);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  double best = 0;
  for (int pass = 0; pass < 3; ++pass) {
    cudaEventRecord(a, st);
    for (size_t off = 0; off < bytes; off += chunk) {
      size_t n = bytes - off < chunk ? bytes - off : chunk;
      cudaMemcpyAsync(d + (off % dbytes), h + off, n, cudaMemcpyHostToDevice, st);
    }
    cudaEventRecord(b, st);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    double gbs = bytes / (ms * 1e-3) / 1e9;
    if (gbs > best) best = gbs;
    printf("%s pass %d: %.2f GB/s\n", name, pass, gbs);
  }
  return best;
}

int main(int argc, char** argv) {
  size_t mb = argc > 1 ? atol(argv[1]) : 4096, chunk_mb = argc > 2 ? atol(argv[2]) : 128;
  size_t bytes = mb << 20, chunk = chunk_mb << 20, dbytes = 2048ull << 20;
  char* d;
  cudaMalloc(&d, dbytes);
  char* h1;
  cudaHostAlloc(reinterpret_cast<void**>(&h1), bytes, cudaHostAllocDefault);
  memset(h1, 1, bytes);
  stream("cudaHostAlloc", h1, bytes, chunk, d, dbytes);
  cudaFreeHost(h1);
  void* p = mmap(nullptr, bytes + (2 << 20), PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  char* h2 = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(p) + (2 << 20) - 1) & ~uintptr_t((2 << 20) - 1));
  int mr = madvise(h2, bytes, MADV_HUGEPAGE);
  memset(h2, 1, bytes);
  cudaError_t e = cudaHostRegister(h2, bytes, cudaHostRegisterDefault);
  printf("madvise rc=%d register=%s\n", mr, cudaGetErrorString(e));
  stream("mmap+THP+register", h2, bytes, chunk, d, dbytes);
  FILE* f = fopen("/sys/kernel/mm/transparent_hugepage/enabled", "r");
  if (f) { char buf[256] = {0}; fread(buf, 1, 255, f); printf("THP: %s", buf); fclose(f); }
  f = fopen("/proc/meminfo", "r");
  if (f) { char line[256]; while (fgets(line, 256, f)) if (strstr(line, "AnonHugePages") || strstr(line, "Hugepagesize")) printf("%s", line); fclose(f); }
  cudaHostUnregister(h2);
  munmap(p, bytes + (2 << 20));
  return 0;
}
