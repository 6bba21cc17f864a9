// NCCL resolved at run time (dlopen) rather than linked: the process may
// already hold a different libnccl.so.2 (PyTorch ships its own), and binding
// ours by soname first would break it. We reuse whichever NCCL is loaded and
// only dlopen one when none is.
#pragma once

#include <dlfcn.h>
#include <nccl.h>

#include <stdexcept>
#include <string>

namespace sqf {

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;

  static const NcclApi& get() {
    static NcclApi api = [] {
      NcclApi a;
      void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
      if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
      if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_LOCAL);
      if (!h) return a;
      a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
      a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
      a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
      a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(dlsym(h, "ncclAllReduce"));
      a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(dlsym(h, "ncclGroupStart"));
      a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(dlsym(h, "ncclGroupEnd"));
      a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
      return a;
    }();
    if (!api.GetUniqueId || !api.CommInitRank || !api.AllReduce)
      throw std::runtime_error("NCCL (libnccl.so.2) could not be loaded");
    return api;
  }
};

}  // namespace sqf
