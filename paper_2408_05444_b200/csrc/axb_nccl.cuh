// axb_nccl.cuh — NCCL, loaded at run time.
//
// The library does not link libnccl: the first sharded use dlopen()s
// "libnccl.so.2" (RTLD_GLOBAL), so a process that already loaded NCCL (e.g. via
// torch) shares that one instance, and single-GPU users never need NCCL.
// Only the handful of calls the row-sharded iteration makes are bound.
#pragma once

#include <cstddef>
#include <cuda_runtime.h>
#include <nccl.h>

namespace axb_nccl {

struct Api {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
};

// Loads NCCL on first use; returns nullptr (and sets *why) when unavailable.
const Api* api(const char** why);

}  // namespace axb_nccl
