// Data-parallel gradient exchange (C1): NCCL all-reduce over NVLink 5 / NVSwitch.
//
// Absent from the reference (SPEC.md:665 lists distributed training as a
// non-goal). One process per GPU; rank 0 creates the ncclUniqueId and the
// Python layer ships its 128 bytes to the other ranks over the rendezvous
// store. Buckets of the flat gradient arena are reduced in place on a
// dedicated comm stream (ordering against backward is done with events by the
// caller), so graph capture records them like any other kernel.
#include <nccl.h>

#include "common.cuh"
#include "../../include/nskb.h"

static int nccl_status(ncclResult_t r, const char* where) {
  return nsk::set_error(NSK_ERR_NCCL, std::string(ncclGetErrorString(r)) + " in " + where);
}

#define NSK_NCCL(expr)                                     \
  do {                                                     \
    ncclResult_t _r = (expr);                              \
    if (_r != ncclSuccess) return nccl_status(_r, #expr);  \
  } while (0)

extern "C" {

int nsk_comm_unique_id(uint8_t* out128) {
  ncclUniqueId id;
  NSK_NCCL(ncclGetUniqueId(&id));
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  memcpy(out128, &id, sizeof id);
  return NSK_OK;
}

int nsk_comm_init(int rank, int world, const uint8_t* uid128, void** comm_out) {
  ncclUniqueId id;
  memcpy(&id, uid128, sizeof id);
  ncclComm_t comm;
  NSK_NCCL(ncclCommInitRank(&comm, world, id, rank));
  *comm_out = (void*)comm;
  return NSK_OK;
}

int nsk_comm_destroy(void* comm) {
  NSK_NCCL(ncclCommDestroy((ncclComm_t)comm));
  return NSK_OK;
}

int nsk_allreduce(void* comm, void* buf, uint64_t count, int dtype, void* stream) {
  ncclDataType_t dt = dtype == NSK_DTYPE_BF16 ? ncclBfloat16 : ncclFloat32;
  NSK_NCCL(ncclAllReduce(buf, buf, count, dt, ncclSum, (ncclComm_t)comm, (cudaStream_t)stream));
  return NSK_OK;
}

int nsk_allreduce_i32(void* comm, int* buf, uint64_t count, void* stream) {
  NSK_NCCL(ncclAllReduce(buf, buf, count, ncclInt32, ncclSum, (ncclComm_t)comm, (cudaStream_t)stream));
  return NSK_OK;
}

int nsk_comm_check(void* comm) {
  ncclResult_t async_err;
  NSK_NCCL(ncclCommGetAsyncError((ncclComm_t)comm, &async_err));
  if (async_err != ncclSuccess) return nccl_status(async_err, "async");
  return NSK_OK;
}

}  // extern "C"
