// comm.cuh -- NCCL for the data-parallel step (SURVEY 8b tt_comm_init /
// tt_allreduce_grads, 8e position sharding), host side.
//
// libnccl is resolved at run time (dlopen), not linked: a process that already
// loaded NCCL (torch ships its own libnccl.so.2) keeps that copy
// (RTLD_NOLOAD first), and the engine library still loads on a machine
// without NCCL -- only the comm entry points then fail, with TT_ERR_CUDA and a
// message.  nccl.h supplies the types and declarations only.
#pragma once
#include <dlfcn.h>
#include <nccl.h>

#include <mutex>
#include <string>

namespace tt {

struct NcclApi {
  bool ok = false;
  std::string why;
  decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
  decltype(&ncclCommInitRank) CommInitRank = nullptr;
  decltype(&ncclCommDestroy) CommDestroy = nullptr;
  decltype(&ncclAllReduce) AllReduce = nullptr;
  decltype(&ncclGetErrorString) GetErrorString = nullptr;
  decltype(&ncclGetVersion) GetVersion = nullptr;
  decltype(&ncclAllGather) AllGather = nullptr;
  decltype(&ncclSend) Send = nullptr;
  decltype(&ncclRecv) Recv = nullptr;
  decltype(&ncclGroupStart) GroupStart = nullptr;
  decltype(&ncclGroupEnd) GroupEnd = nullptr;
};

inline const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!lib) lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) {
      const char* e = dlerror();
      api.why = std::string("libnccl.so.2 not loadable: ") + (e ? e : "?");
      return;
    }
#define TT_NCCL_SYM(f)                                                          \
  api.f = reinterpret_cast<decltype(api.f)>(dlsym(lib, "nccl" #f));            \
  if (!api.f) {                                                                 \
    api.why = "libnccl: missing symbol nccl" #f;                                \
    return;                                                                     \
  }
    TT_NCCL_SYM(GetUniqueId)
    TT_NCCL_SYM(CommInitRank)
    TT_NCCL_SYM(CommDestroy)
    TT_NCCL_SYM(AllReduce)
    TT_NCCL_SYM(GetErrorString)
    TT_NCCL_SYM(GetVersion)
    TT_NCCL_SYM(AllGather)
    TT_NCCL_SYM(Send)
    TT_NCCL_SYM(Recv)
    TT_NCCL_SYM(GroupStart)
    TT_NCCL_SYM(GroupEnd)
#undef TT_NCCL_SYM
    api.ok = true;
  });
  return api;
}

}  // namespace tt
