// nccl_loader.hpp -- NCCL entry points resolved at run time with dlopen.
//
// The library links no NCCL so it loads on hosts without one; Harmony-DP
// opens the libnccl.so.2 torch already ships (path passed from Python) and
// uses only the stable core API (unique id, comm init, all-reduce,
// reduce-scatter).
#pragma once

#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <string>

namespace hm {

struct Nccl {
  void *handle = nullptr;
  ncclResult_t (*get_unique_id)(ncclUniqueId *) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_reduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*reduce_scatter)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                 cudaStream_t) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char *(*error_string)(ncclResult_t) = nullptr;

  bool load(const char *path, std::string &err) {
    if (handle) return true;
    handle = dlopen(path && *path ? path : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!handle) {
      err = std::string("dlopen NCCL failed: ") + dlerror();
      return false;
    }
    get_unique_id = reinterpret_cast<decltype(get_unique_id)>(dlsym(handle, "ncclGetUniqueId"));
    comm_init_rank = reinterpret_cast<decltype(comm_init_rank)>(dlsym(handle, "ncclCommInitRank"));
    all_reduce = reinterpret_cast<decltype(all_reduce)>(dlsym(handle, "ncclAllReduce"));
    reduce_scatter = reinterpret_cast<decltype(reduce_scatter)>(dlsym(handle, "ncclReduceScatter"));
    comm_destroy = reinterpret_cast<decltype(comm_destroy)>(dlsym(handle, "ncclCommDestroy"));
    error_string = reinterpret_cast<decltype(error_string)>(dlsym(handle, "ncclGetErrorString"));
    if (!get_unique_id || !comm_init_rank || !all_reduce || !reduce_scatter || !comm_destroy || !error_string) {
      err = "NCCL symbols missing";
      return false;
    }
    return true;
  }
};

inline Nccl &nccl() {
  static Nccl n;
  return n;
}

}  // namespace hm
