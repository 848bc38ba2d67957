// tsds_nccl.cpp -- the NCCL entry points libtsds uses, resolved at run time.
//
// libtsds.so does not link NCCL: the communicator (tsds_comm_*, include/tsds.h)
// dlopen()s libnccl.so.2 on first use -- the copy torch already loaded if
// there is one (same SONAME), else the system's -- so single-GPU users never
// need NCCL.  Only the five calls of the sharded path are bound.
#include "tsds_nccl.h"

#include <dlfcn.h>

#include <cstdlib>
#include <mutex>

namespace tsds_nccl {

namespace {
struct Api {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*get_error_string)(ncclResult_t) = nullptr;
  bool ok = false;
  std::string err;
};
Api g_api;
std::once_flag g_once;

void load_once() {
  const char* env = getenv("TSDS_NCCL_LIB");
  const char* names[] = {env, "libnccl.so.2", "libnccl.so"};
  void* h = nullptr;
  for (const char* n : names) {
    if (!n) continue;
    h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
    if (h) break;
  }
  if (!h) {
    g_api.err = std::string("cannot load libnccl.so.2: ") + dlerror();
    return;
  }
  g_api.get_unique_id = (decltype(g_api.get_unique_id))dlsym(h, "ncclGetUniqueId");
  g_api.comm_init_rank = (decltype(g_api.comm_init_rank))dlsym(h, "ncclCommInitRank");
  g_api.comm_destroy = (decltype(g_api.comm_destroy))dlsym(h, "ncclCommDestroy");
  g_api.all_gather = (decltype(g_api.all_gather))dlsym(h, "ncclAllGather");
  g_api.get_error_string = (decltype(g_api.get_error_string))dlsym(h, "ncclGetErrorString");
  g_api.ok = g_api.get_unique_id && g_api.comm_init_rank && g_api.comm_destroy && g_api.all_gather &&
             g_api.get_error_string;
  if (!g_api.ok) g_api.err = "libnccl.so.2 lacks a required symbol";
}
}  // namespace

bool available(std::string* err) {
  std::call_once(g_once, load_once);
  if (!g_api.ok && err) *err = g_api.err;
  return g_api.ok;
}

std::string error_string(ncclResult_t r) {
  return g_api.get_error_string ? g_api.get_error_string(r) : ("nccl error " + std::to_string((int)r));
}

ncclResult_t get_unique_id(ncclUniqueId* id) { return g_api.get_unique_id(id); }
ncclResult_t comm_init_rank(ncclComm_t* c, int nranks, const ncclUniqueId& id, int rank) {
  return g_api.comm_init_rank(c, nranks, id, rank);
}
ncclResult_t comm_destroy(ncclComm_t c) { return g_api.comm_destroy(c); }
ncclResult_t all_gather_bytes(const void* send, void* recv, size_t bytes, ncclComm_t c, cudaStream_t s) {
  return g_api.all_gather(send, recv, bytes, ncclUint8, c, s);
}

}  // namespace tsds_nccl
