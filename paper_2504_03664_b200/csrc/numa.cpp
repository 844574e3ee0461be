// numa.cpp — NUMA-local pinned host stores (SURVEY.md §8(b) `numa_node`, §8(e)).
//
// On a multi-socket 8-GPU node each rank's pinned host store (15.7 GB for OPT-30B int4)
// must sit on the socket its GPU's PCIe root hangs off, or every streamed byte crosses
// the socket interconnect (App. D: "Servers usually provide isolated PCIe channels",
// PAPER.md:817).  cudaHostAlloc places pages wherever the allocating thread's policy
// and first touch put them, so the store is built explicitly instead:
//   mmap (anonymous, no pages yet) -> mbind(MPOL_BIND, node) -> first touch by threads
//   pinned to the node's CPUs -> cudaHostRegister (page-lock + map for DMA).
// Raw syscalls: the image has no libnuma.  The GPU's node comes from sysfs
// (/sys/bus/pci/devices/<bus id>/numa_node).
#include <cuda_runtime.h>
#include <pthread.h>
#include <sched.h>
#include <sys/mman.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <algorithm>
#include <cctype>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <string>
#include <thread>
#include <vector>

#include "numa.h"

namespace pipo {

namespace {

constexpr int kMpolBind = 2;          // linux/mempolicy.h
constexpr unsigned kMpolMfStrict = 1u;
constexpr unsigned kMpolMfMove = 2u;

std::string read_file(const std::string& path) {
  std::ifstream f(path);
  std::string s;
  if (f) std::getline(f, s);
  return s;
}

// "0-15,32-47" -> cpu ids
std::vector<int> parse_cpulist(const std::string& s) {
  std::vector<int> out;
  size_t i = 0;
  while (i < s.size()) {
    size_t j = s.find(',', i);
    if (j == std::string::npos) j = s.size();
    const std::string part = s.substr(i, j - i);
    const size_t dash = part.find('-');
    try {
      if (dash == std::string::npos) {
        if (!part.empty()) out.push_back(std::stoi(part));
      } else {
        const int a = std::stoi(part.substr(0, dash)), b = std::stoi(part.substr(dash + 1));
        for (int c = a; c <= b; ++c) out.push_back(c);
      }
    } catch (...) {
    }
    i = j + 1;
  }
  return out;
}

}  // namespace

int numa_node_count() {
  int n = 0;
  while (access(("/sys/devices/system/node/node" + std::to_string(n)).c_str(), F_OK) == 0) ++n;
  return n;
}

int gpu_numa_node(int device) {
  char bus[32] = {0};
  if (cudaDeviceGetPCIBusId(bus, sizeof bus, device) != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  std::string id(bus);
  for (auto& ch : id) ch = (char)std::tolower((unsigned char)ch);
  const std::string s = read_file("/sys/bus/pci/devices/" + id + "/numa_node");
  try {
    return s.empty() ? -1 : std::stoi(s);
  } catch (...) {
    return -1;
  }
}

std::vector<int> node_cpus(int node) {
  if (node < 0) return {};
  return parse_cpulist(read_file("/sys/devices/system/node/node" + std::to_string(node) + "/cpulist"));
}

int resolve_numa_node(int requested, int device) {
  if (requested == PIPO_NUMA_NONE) return -1;
  if (requested >= 0) return requested;
  // PIPO_NUMA_GPU_LOCAL: bind only where there is a choice to make
  return numa_node_count() > 1 ? gpu_numa_node(device) : -1;
}

void bind_thread_to_node(int node) {
  const std::vector<int> cpus = node_cpus(node);
  if (cpus.empty()) return;
  cpu_set_t set;
  CPU_ZERO(&set);
  for (int c : cpus)
    if (c >= 0 && c < CPU_SETSIZE) CPU_SET(c, &set);
  pthread_setaffinity_np(pthread_self(), sizeof set, &set);
}

bool numa_host_alloc(int64_t bytes, int node, void** out, bool* bound) {
  *out = nullptr;
  *bound = false;
  if (bytes <= 0) return true;
  void* p = mmap(nullptr, (size_t)bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS | MAP_NORESERVE, -1, 0);
  if (p == MAP_FAILED) return false;
  if (node >= 0 && node < 1024) {
    unsigned long mask[1024 / (8 * sizeof(unsigned long))] = {0};
    mask[node / (8 * sizeof(unsigned long))] |= 1ul << (node % (8 * sizeof(unsigned long)));
    const long rc = syscall(SYS_mbind, p, (unsigned long)bytes, kMpolBind, mask, (unsigned long)1024,
                            kMpolMfStrict | kMpolMfMove);
    *bound = rc == 0;
  }
  // first touch from threads on the node (the policy already forces the node; local
  // threads make the zeroing itself local)
  const int64_t page = 4096;
  const int64_t n_pages = (bytes + page - 1) / page;
  const int nt = (int)std::max<int64_t>(1, std::min<int64_t>(16, n_pages / 4096));
  std::vector<std::thread> th;
  for (int t = 0; t < nt; ++t) {
    th.emplace_back([=] {
      if (node >= 0) bind_thread_to_node(node);
      const int64_t a = n_pages * t / nt * page, b = std::min<int64_t>(bytes, n_pages * (t + 1) / nt * page);
      if (b > a) std::memset(static_cast<uint8_t*>(p) + a, 0, (size_t)(b - a));
    });
  }
  for (auto& x : th) x.join();
  if (cudaHostRegister(p, (size_t)bytes, cudaHostRegisterPortable) != cudaSuccess) {
    cudaGetLastError();
    munmap(p, (size_t)bytes);
    return false;
  }
  *out = p;
  return true;
}

void numa_host_free(void* p, int64_t bytes) {
  if (!p) return;
  cudaHostUnregister(p);
  cudaGetLastError();
  munmap(p, (size_t)bytes);
}

double numa_local_fraction(const void* p, int64_t bytes, int node, int samples) {
  if (!p || bytes <= 0 || node < 0 || samples <= 0) return -1.0;
  const int64_t page = 4096, n_pages = bytes / page;
  if (n_pages <= 0) return -1.0;
  std::vector<void*> pages;
  for (int i = 0; i < samples; ++i)
    pages.push_back(const_cast<uint8_t*>(static_cast<const uint8_t*>(p)) + (n_pages - 1) * i / std::max(1, samples - 1) * page);
  std::vector<int> status(pages.size(), -1);
  const long rc = syscall(SYS_move_pages, 0, (unsigned long)pages.size(), pages.data(), nullptr, status.data(), 0);
  if (rc != 0) return -1.0;
  int local = 0;
  for (int s : status) local += s == node;
  return (double)local / (double)pages.size();
}

}  // namespace pipo
