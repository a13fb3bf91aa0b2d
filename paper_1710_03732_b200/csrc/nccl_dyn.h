// nccl_dyn.h — NCCL entry points resolved at first use with dlopen/dlsym.
//
// The library must not pin a libnccl.so.2 at load time: torch ships its own
// (newer) NCCL under the same soname, and whichever loads first wins for the
// whole process.  Sharded engines therefore bind to the NCCL already present
// in the process (RTLD_NOLOAD; torch's when torch is imported), falling back
// to the system library only if none is loaded.
#pragma once

#include <nccl.h>

namespace qapb {

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                            cudaStream_t);
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t);
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  const char* (*GetErrorString)(ncclResult_t);
};

// Throws CudaError if no NCCL can be loaded.
const NcclApi& nccl();

}  // namespace qapb
