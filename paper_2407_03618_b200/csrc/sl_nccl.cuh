// sl_nccl.cuh — NCCL entry points resolved lazily with dlopen.
//
// The single-GPU path never touches NCCL, and a process that already has a libnccl.so.2
// loaded (e.g. PyTorch's bundled copy) must keep using that one: binding at link time
// would let whichever copy loads first satisfy both, breaking the other user. We take
// the already-loaded copy (RTLD_NOLOAD) and only fall back to the loader search path.
#pragma once
#include <dlfcn.h>
#include <nccl.h>

#include <mutex>

namespace sl {
struct NcclApi {
  decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
  decltype(&ncclCommInitRank) CommInitRank = nullptr;
  decltype(&ncclCommDestroy) CommDestroy = nullptr;
  decltype(&ncclAllReduce) AllReduce = nullptr;
  decltype(&ncclSend) Send = nullptr;
  decltype(&ncclRecv) Recv = nullptr;
  decltype(&ncclGroupStart) GroupStart = nullptr;
  decltype(&ncclGroupEnd) GroupEnd = nullptr;
  decltype(&ncclGetErrorString) GetErrorString = nullptr;
  bool ok = false;
};

inline const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
#define SL_SYM(field, name) api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, #name))
    SL_SYM(GetUniqueId, ncclGetUniqueId);
    SL_SYM(CommInitRank, ncclCommInitRank);
    SL_SYM(CommDestroy, ncclCommDestroy);
    SL_SYM(AllReduce, ncclAllReduce);
    SL_SYM(Send, ncclSend);
    SL_SYM(Recv, ncclRecv);
    SL_SYM(GroupStart, ncclGroupStart);
    SL_SYM(GroupEnd, ncclGroupEnd);
    SL_SYM(GetErrorString, ncclGetErrorString);
#undef SL_SYM
    api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllReduce && api.Send && api.Recv &&
             api.GroupStart && api.GroupEnd && api.GetErrorString;
  });
  return api;
}
}  // namespace sl
