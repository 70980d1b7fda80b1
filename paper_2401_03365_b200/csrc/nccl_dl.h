// nccl_dl.h — NCCL resolved at run time (dlopen "libnccl.so.2").
//
// The library only needs NCCL for multi-GPU plans; resolving it lazily keeps
// single-GPU use (and the C-ABI symbol checks on CPU-only hosts) free of the
// dependency.  Inside a torch process the already-loaded libnccl.so.2 is reused.
#pragma once

#include <nccl.h>

#include <string>

namespace pcsb {

struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

// Returns nullptr (and sets err) when NCCL cannot be loaded.
const NcclApi* nccl_api(std::string* err);

}  // namespace pcsb
