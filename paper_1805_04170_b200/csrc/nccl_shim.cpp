#include "nccl_shim.h"

#include <dlfcn.h>

#include <cstring>
#include <string>

#include "util.h"

namespace tpx {

namespace {
constexpr int kNcclUint8 = 1;  // ncclUint8 (nccl.h ncclDataType_t)

template <class F>
void sym(void* h, const char* name, F& f) {
  f = reinterpret_cast<F>(dlsym(h, name));
  if (!f) fail(std::string("NCCL symbol missing: ") + name);
}

void check(int r, const char* what) {
  if (r != 0) {
    const char* msg = nccl().GetErrorString ? nccl().GetErrorString(r) : "?";
    fail(std::string("NCCL ") + what + " failed: " + msg);
  }
}
}  // namespace

NcclApi& nccl() {
  static NcclApi api;
  if (!api.handle) {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) fail(std::string("cannot load NCCL: ") + dlerror());
    sym(h, "ncclGetUniqueId", api.GetUniqueId);
    sym(h, "ncclCommInitRank", api.CommInitRank);
    sym(h, "ncclCommDestroy", api.CommDestroy);
    sym(h, "ncclGroupStart", api.GroupStart);
    sym(h, "ncclGroupEnd", api.GroupEnd);
    sym(h, "ncclSend", api.Send);
    sym(h, "ncclRecv", api.Recv);
    sym(h, "ncclGetErrorString", api.GetErrorString);
    api.handle = h;
  }
  return api;
}

void nccl_unique_id(void* out128) {
  NcclUniqueId id;
  check(nccl().GetUniqueId(&id), "GetUniqueId");
  std::memcpy(out128, &id, sizeof id);
}

void* nccl_comm_init(int nranks, const void* uid128, int rank) {
  NcclUniqueId id;
  std::memcpy(&id, uid128, sizeof id);
  void* comm = nullptr;
  check(nccl().CommInitRank(&comm, nranks, id, rank), "CommInitRank");
  return comm;
}

void nccl_comm_destroy(void* comm) {
  if (comm) nccl().CommDestroy(comm);
}

void nccl_group_start() { check(nccl().GroupStart(), "GroupStart"); }
void nccl_group_end() { check(nccl().GroupEnd(), "GroupEnd"); }

void nccl_send(const void* buf, size_t bytes, int peer, void* comm, cudaStream_t s) {
  check(nccl().Send(buf, bytes, kNcclUint8, peer, comm, s), "Send");
}

void nccl_recv(void* buf, size_t bytes, int peer, void* comm, cudaStream_t s) {
  check(nccl().Recv(buf, bytes, kNcclUint8, peer, comm, s), "Recv");
}

}  // namespace tpx
