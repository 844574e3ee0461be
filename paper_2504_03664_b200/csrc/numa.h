// numa.h — NUMA-local pinned host memory (numa.cpp).
#pragma once
#include <stdint.h>

#include <vector>

#include "../../include/pipo.h"

namespace pipo {

int numa_node_count();
int gpu_numa_node(int device);                  // -1 if unknown / single node
std::vector<int> node_cpus(int node);
// pipo_config.numa_node -> the node to bind to, or -1 for no binding
int resolve_numa_node(int requested, int device);
void bind_thread_to_node(int node);             // no-op for node < 0
// Page-locked host memory whose pages are bound to `node` (node < 0: OS default
// placement).  *bound reports whether the mbind succeeded.  false = out of memory.
bool numa_host_alloc(int64_t bytes, int node, void** out, bool* bound);
void numa_host_free(void* p, int64_t bytes);
// fraction of `samples` pages of [p, p+bytes) resident on `node` (-1: unknown)
double numa_local_fraction(const void* p, int64_t bytes, int node, int samples);

}  // namespace pipo
