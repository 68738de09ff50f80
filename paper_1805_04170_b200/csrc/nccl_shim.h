// NCCL entry points resolved at run time (dlopen "libnccl.so.2"): the single-GPU path never
// touches NCCL, and inside a torch process the already-loaded NCCL is reused.
#pragma once
#include <cstddef>

#include <cuda_runtime.h>

namespace tpx {

struct NcclUniqueId {
  char internal[128];  // layout of ncclUniqueId (nccl.h)
};

struct NcclApi {
  using Comm = void*;
  int (*GetUniqueId)(NcclUniqueId* id) = nullptr;
  int (*CommInitRank)(Comm* comm, int nranks, NcclUniqueId id, int rank) = nullptr;
  int (*CommDestroy)(Comm comm) = nullptr;
  int (*GroupStart)() = nullptr;
  int (*GroupEnd)() = nullptr;
  int (*Send)(const void* buf, size_t count, int dtype, int peer, Comm comm, cudaStream_t s) = nullptr;
  int (*Recv)(void* buf, size_t count, int dtype, int peer, Comm comm, cudaStream_t s) = nullptr;
  const char* (*GetErrorString)(int r) = nullptr;
  void* handle = nullptr;
};

NcclApi& nccl();  // throws tpx::Error when NCCL cannot be loaded

// Wrappers that throw on error.
void nccl_unique_id(void* out128);
void* nccl_comm_init(int nranks, const void* uid128, int rank);
void nccl_comm_destroy(void* comm);
void nccl_group_start();
void nccl_group_end();
void nccl_send(const void* buf, size_t bytes, int peer, void* comm, cudaStream_t s);
void nccl_recv(void* buf, size_t bytes, int peer, void* comm, cudaStream_t s);

}  // namespace tpx
