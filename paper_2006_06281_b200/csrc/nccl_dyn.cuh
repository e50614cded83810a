// nccl_dyn.cuh — NCCL loaded on demand (dlopen) instead of linked.
//
// PyTorch ships its own libnccl.so.2 (2.28) while the system has 2.27; both
// use the soname libnccl.so.2, so linking ours would make whichever loads
// first win for the whole process (and break torch if it is ours).  Loading
// lazily, only when a multi-GPU context is created, reuses whatever NCCL the
// process already has (torch's, when torch is imported) or the system one.
#pragma once

#include <dlfcn.h>
#include <nccl.h>

#include <string>

#include "common.cuh"

namespace fcpd {

struct NcclApi {
  decltype(&::ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&::ncclCommInitRank) commInitRank = nullptr;
  decltype(&::ncclCommDestroy) commDestroy = nullptr;
  decltype(&::ncclAllReduce) allReduce = nullptr;
  decltype(&::ncclReduceScatter) reduceScatter = nullptr;
  decltype(&::ncclAllGather) allGather = nullptr;
  decltype(&::ncclGetErrorString) getErrorString = nullptr;
  std::string error;
};

inline NcclApi& nccl_api() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      a.error = std::string("cannot load libnccl.so.2: ") + dlerror();
      return a;
    }
    a.getUniqueId = reinterpret_cast<decltype(a.getUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    a.commInitRank = reinterpret_cast<decltype(a.commInitRank)>(dlsym(h, "ncclCommInitRank"));
    a.commDestroy = reinterpret_cast<decltype(a.commDestroy)>(dlsym(h, "ncclCommDestroy"));
    a.allReduce = reinterpret_cast<decltype(a.allReduce)>(dlsym(h, "ncclAllReduce"));
    a.reduceScatter = reinterpret_cast<decltype(a.reduceScatter)>(dlsym(h, "ncclReduceScatter"));
    a.allGather = reinterpret_cast<decltype(a.allGather)>(dlsym(h, "ncclAllGather"));
    a.getErrorString =
        reinterpret_cast<decltype(a.getErrorString)>(dlsym(h, "ncclGetErrorString"));
    if (!a.getUniqueId || !a.commInitRank || !a.allReduce || !a.reduceScatter || !a.allGather)
      a.error = "libnccl.so.2 lacks required symbols";
    return a;
  }();
  return api;
}

inline NcclApi& nccl_checked() {
  NcclApi& a = nccl_api();
  if (!a.error.empty()) throw Failure(FCPD_ERR_NCCL, a.error);
  return a;
}

}  // namespace fcpd

// route the NCCL calls below this point through the loaded library
#define ncclGetUniqueId ::fcpd::nccl_checked().getUniqueId
#define ncclCommInitRank ::fcpd::nccl_checked().commInitRank
#define ncclCommDestroy ::fcpd::nccl_checked().commDestroy
#define ncclAllReduce ::fcpd::nccl_checked().allReduce
#define ncclReduceScatter ::fcpd::nccl_checked().reduceScatter
#define ncclAllGather ::fcpd::nccl_checked().allGather
#define ncclGetErrorString ::fcpd::nccl_checked().getErrorString
