// nccl_rt.cpp — see nccl_rt.h.  Types come from <nccl.h>; every entry point is resolved
// with dlsym on first use.
#include "nccl_rt.h"

#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>

namespace pipo {
namespace {

struct Nccl {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char* (*get_error_string)(ncclResult_t) = nullptr;
  bool ok = false;
};

Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    n.get_unique_id = reinterpret_cast<decltype(n.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    n.comm_init_rank = reinterpret_cast<decltype(n.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    n.all_gather = reinterpret_cast<decltype(n.all_gather)>(dlsym(h, "ncclAllGather"));
    n.comm_destroy = reinterpret_cast<decltype(n.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    n.get_error_string = reinterpret_cast<decltype(n.get_error_string)>(dlsym(h, "ncclGetErrorString"));
    n.ok = n.get_unique_id && n.comm_init_rank && n.all_gather && n.comm_destroy && n.get_error_string;
  });
  return n;
}

}  // namespace

int nccl_unique_id(unsigned char id[128]) {
  if (!nccl().ok) return -1;
  ncclUniqueId u;
  const ncclResult_t r = nccl().get_unique_id(&u);
  static_assert(sizeof(u.internal) == 128, "ncclUniqueId is 128 bytes");
  if (r == ncclSuccess) std::memcpy(id, u.internal, 128);
  return (int)r;
}

int nccl_comm_init(void** comm, int world, const unsigned char id[128], int rank) {
  if (!nccl().ok) return -1;
  ncclUniqueId u;
  std::memcpy(u.internal, id, 128);
  ncclComm_t c = nullptr;
  const ncclResult_t r = nccl().comm_init_rank(&c, world, u, rank);
  *comm = c;
  return (int)r;
}

int nccl_allgather_bytes(const void* send, void* recv, size_t bytes_per_rank, void* comm, cudaStream_t st) {
  if (!nccl().ok) return -1;
  return (int)nccl().all_gather(send, recv, bytes_per_rank, ncclUint8, static_cast<ncclComm_t>(comm), st);
}

void nccl_comm_destroy(void* comm) {
  if (comm && nccl().ok) nccl().comm_destroy(static_cast<ncclComm_t>(comm));
}

const char* nccl_error_string(int rc) {
  if (rc == -1) return "libnccl.so.2 could not be loaded";
  return nccl().ok ? nccl().get_error_string(static_cast<ncclResult_t>(rc)) : "NCCL unavailable";
}

}  // namespace pipo
