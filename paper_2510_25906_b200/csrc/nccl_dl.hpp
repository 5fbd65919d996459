// NCCL resolved at run time (shared by the 2D and 3D solvers).
#pragma once

#include <dlfcn.h>
#include <nccl.h>

#include <string>

#include "layout.hpp"

namespace ucfvb {

// ---- NCCL, resolved at run time --------------------------------------------
// The library never links NCCL: ucfvb_attach_nccl binds to the NCCL already in
// the process (torch's, when torch.distributed initialised it) or dlopens
// libnccl.so.2. Single-GPU use therefore has no NCCL dependency at all.
struct Nccl {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

inline const Nccl& nccl() {
  static Nccl n;
  static bool done = false;
  if (done) return n;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) throw ApiError(UCFVB_UNSUPPORTED, "NCCL (libnccl.so.2) is not available");
  auto sym = [&](const char* name) {
    void* f = dlsym(h, name);
    if (!f) throw ApiError(UCFVB_UNSUPPORTED, std::string("NCCL symbol missing: ") + name);
    return f;
  };
  n.GetUniqueId = reinterpret_cast<decltype(n.GetUniqueId)>(sym("ncclGetUniqueId"));
  n.CommInitRank = reinterpret_cast<decltype(n.CommInitRank)>(sym("ncclCommInitRank"));
  n.CommDestroy = reinterpret_cast<decltype(n.CommDestroy)>(sym("ncclCommDestroy"));
  n.Send = reinterpret_cast<decltype(n.Send)>(sym("ncclSend"));
  n.Recv = reinterpret_cast<decltype(n.Recv)>(sym("ncclRecv"));
  n.AllReduce = reinterpret_cast<decltype(n.AllReduce)>(sym("ncclAllReduce"));
  n.GroupStart = reinterpret_cast<decltype(n.GroupStart)>(sym("ncclGroupStart"));
  n.GroupEnd = reinterpret_cast<decltype(n.GroupEnd)>(sym("ncclGroupEnd"));
  n.GetErrorString = reinterpret_cast<decltype(n.GetErrorString)>(sym("ncclGetErrorString"));
  done = true;
  return n;
}

#define NK(x)                                                                                  \
  do {                                                                                         \
    ncclResult_t r_ = (x);                                                                     \
    if (r_ != ncclSuccess) throw ApiError(UCFVB_CUDA, std::string(#x) + ": " + nccl().GetErrorString(r_)); \
  } while (0)


}  // namespace ucfvb
