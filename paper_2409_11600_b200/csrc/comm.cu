// Data-parallel gradient exchange (C1): NCCL all-reduce over NVLink 5 / NVSwitch.
//
// Absent from the reference (SPEC.md:665 lists distributed training as a
// non-goal). One process per GPU; rank 0 creates the ncclUniqueId and the
// Python layer ships its 128 bytes to the other ranks over the rendezvous
// store. Buckets of the flat gradient arena are reduced in place on a
// dedicated comm stream (ordering against backward is done with events by the
// caller), so graph capture records them like any other kernel.
//
// NCCL is bound at run time (dlopen), not at link time: a process holds ONE libnccl.so.2, and PyTorch (used for
// the rendezvous) needs the NCCL it ships with. The library is taken from NSK_NCCL_LIB (set by _lib.py to the
// PyTorch-bundled copy when there is one), else the default search path; whichever of PyTorch and libnskb loads
// it first, both end up on the same library.
#include <dlfcn.h>
#include <nccl.h>

#include <mutex>

#include "common.cuh"
#include "../../include/nskb.h"

namespace {

struct NcclApi {
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*commGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  const char* (*getErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
  std::string why;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = nullptr;
    const char* want = getenv("NSK_NCCL_LIB");
    if (want && *want) h = dlopen(want, RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      api.why = std::string("cannot load libnccl.so.2: ") + dlerror();
      return;
    }
    api.getUniqueId = (decltype(api.getUniqueId))dlsym(h, "ncclGetUniqueId");
    api.commInitRank = (decltype(api.commInitRank))dlsym(h, "ncclCommInitRank");
    api.commDestroy = (decltype(api.commDestroy))dlsym(h, "ncclCommDestroy");
    api.allReduce = (decltype(api.allReduce))dlsym(h, "ncclAllReduce");
    api.commGetAsyncError = (decltype(api.commGetAsyncError))dlsym(h, "ncclCommGetAsyncError");
    api.getErrorString = (decltype(api.getErrorString))dlsym(h, "ncclGetErrorString");
    api.ok = api.getUniqueId && api.commInitRank && api.commDestroy && api.allReduce && api.commGetAsyncError &&
             api.getErrorString;
    if (!api.ok) api.why = "libnccl.so.2 lacks an expected entry point";
  });
  return api;
}

int nccl_status(ncclResult_t r, const char* where) {
  return nsk::set_error(NSK_ERR_NCCL, std::string(nccl().getErrorString(r)) + " in " + where);
}

}  // namespace

#define NSK_NCCL_API()                                                         \
  do {                                                                         \
    if (!nccl().ok) return nsk::set_error(NSK_ERR_NCCL, nccl().why);           \
  } while (0)

#define NSK_NCCL(expr)                                     \
  do {                                                     \
    ncclResult_t _r = (expr);                              \
    if (_r != ncclSuccess) return nccl_status(_r, #expr);  \
  } while (0)

extern "C" {

int nsk_comm_unique_id(uint8_t* out128) {
  NSK_NCCL_API();
  ncclUniqueId id;
  NSK_NCCL(nccl().getUniqueId(&id));
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  memcpy(out128, &id, sizeof id);
  return NSK_OK;
}

int nsk_comm_init(int rank, int world, const uint8_t* uid128, void** comm_out) {
  NSK_NCCL_API();
  ncclUniqueId id;
  memcpy(&id, uid128, sizeof id);
  ncclComm_t comm;
  NSK_NCCL(nccl().commInitRank(&comm, world, id, rank));
  *comm_out = (void*)comm;
  return NSK_OK;
}

int nsk_comm_destroy(void* comm) {
  NSK_NCCL_API();
  NSK_NCCL(nccl().commDestroy((ncclComm_t)comm));
  return NSK_OK;
}

int nsk_allreduce(void* comm, void* buf, uint64_t count, int dtype, void* stream) {
  NSK_NCCL_API();
  ncclDataType_t dt = dtype == NSK_DTYPE_BF16 ? ncclBfloat16 : ncclFloat32;
  NSK_NCCL(nccl().allReduce(buf, buf, count, dt, ncclSum, (ncclComm_t)comm, (cudaStream_t)stream));
  return NSK_OK;
}

int nsk_allreduce_i32(void* comm, int* buf, uint64_t count, void* stream) {
  NSK_NCCL_API();
  NSK_NCCL(nccl().allReduce(buf, buf, count, ncclInt32, ncclSum, (ncclComm_t)comm, (cudaStream_t)stream));
  return NSK_OK;
}

int nsk_comm_check(void* comm) {
  NSK_NCCL_API();
  ncclResult_t async_err;
  NSK_NCCL(nccl().commGetAsyncError((ncclComm_t)comm, &async_err));
  if (async_err != ncclSuccess) return nccl_status(async_err, "async");
  return NSK_OK;
}

}  // extern "C"
