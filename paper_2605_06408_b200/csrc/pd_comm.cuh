// pd_comm.cuh -- the NCCL layer of the sharded build: libnccl.so.2 is opened at the first
// pd_comm_init (dlopen; the library has no link-time NCCL dependency, and under PyTorch it shares the NCCL
// PyTorch already loaded), and the few entry points the path needs are resolved by name.
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>
#include <stdint.h>

#include "../../include/pd.h"

namespace pd {

struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*);
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
    ncclResult_t (*CommDestroy)(ncclComm_t);
    ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
    ncclResult_t (*GroupStart)();
    ncclResult_t (*GroupEnd)();
    const char* (*GetErrorString)(ncclResult_t);
    ncclResult_t (*GetVersion)(int*);
};

// nullptr if libnccl.so.2 cannot be opened (pd_comm_* then return PD_ENCCL)
const NcclApi* nccl_api();
// thread-local message of the last NCCL failure (read by pd_last_cuda_error)
void nccl_set_error(const char* where, ncclResult_t r);
const char* nccl_last_error();

}  // namespace pd

struct pd_comm {
    ncclComm_t comm = nullptr;
    int rank = 0, world = 1, device = 0;
};
