// nccl_rt.h — NCCL loaded at run time (dlopen "libnccl.so.2") for the NEXT-1 sharded
// weight stream: the library has no link-time NCCL dependency, and inside a PyTorch
// process dlopen returns the libnccl.so.2 torch already loaded.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

namespace pipo {

// all return 0 on success, else an ncclResult_t (or -1: NCCL not loadable)
int nccl_unique_id(unsigned char id[128]);
int nccl_comm_init(void** comm, int world, const unsigned char id[128], int rank);
int nccl_allgather_bytes(const void* send, void* recv, size_t bytes_per_rank, void* comm, cudaStream_t st);
void nccl_comm_destroy(void* comm);
const char* nccl_error_string(int rc);

}  // namespace pipo
