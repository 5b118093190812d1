// NCCL, loaded at run time (the library owns the multi-GPU communicator).
//
// libkgq.so does not link libnccl: it dlopen()s "libnccl.so.2" on first use, reusing the copy a
// host process (e.g. PyTorch) already loaded (RTLD_NOLOAD) so that one NCCL instance serves the
// process, else the system one; KGQ_NCCL_LIB names another file.  Without NCCL the
// communicator entry points return KGQ_ENCCL and everything else works.  Only the handful of
// calls below is used; their signatures are stable across NCCL 2.x (types from <nccl.h>).
#pragma once
#include <dlfcn.h>
#include <nccl.h>
#include <stdlib.h>

#include <mutex>
#include <string>

namespace kgq {

struct NcclApi {
  bool ok = false;
  std::string why;
  int version = 0;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*GetVersion)(int*) = nullptr;
};

inline const NcclApi& nccl_api() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* name = getenv("KGQ_NCCL_LIB");
    void* h = nullptr;
    if (name && name[0]) {
      h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
    } else {
      h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the process's NCCL, if loaded
      if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
      if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    }
    if (!h) {
      const char* e = dlerror();
      api.why = std::string("cannot load NCCL: ") + (e ? e : "unknown error");
      return;
    }
    bool all = true;
    auto sym = [&](auto& fn, const char* s) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, s));
      if (!fn) {
        all = false;
        if (api.why.empty()) api.why = std::string("NCCL lacks ") + s;
      }
    };
    sym(api.GetUniqueId, "ncclGetUniqueId");
    sym(api.CommInitRank, "ncclCommInitRank");
    sym(api.CommDestroy, "ncclCommDestroy");
    sym(api.CommAbort, "ncclCommAbort");
    sym(api.CommGetAsyncError, "ncclCommGetAsyncError");
    sym(api.AllGather, "ncclAllGather");
    sym(api.AllReduce, "ncclAllReduce");
    sym(api.GroupStart, "ncclGroupStart");
    sym(api.GroupEnd, "ncclGroupEnd");
    sym(api.GetErrorString, "ncclGetErrorString");
    sym(api.GetVersion, "ncclGetVersion");
    if (all && api.GetVersion(&api.version) == ncclSuccess) api.ok = true;
  });
  return api;
}

}  // namespace kgq
