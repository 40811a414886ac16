// NCCL transport for the multi-GPU solve (one process per GPU).  NCCL is loaded
// with dlopen at first use (the copy torch already loaded, else the system
// libnccl.so.2), so the library itself has no link-time NCCL dependency and
// single-GPU use never touches it.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

namespace amgb {

struct Nccl {
    bool ok = false;
    std::string error;
    void* lib = nullptr;
    // resolved symbols (NCCL's C ABI)
    int (*getUniqueId)(void* id128) = nullptr;
    void* commInitRank = nullptr;  // int ncclCommInitRank(ncclComm_t*, int, ncclUniqueId, int)
    int (*commDestroy)(void*) = nullptr;
    int (*groupStart)() = nullptr;
    int (*groupEnd)() = nullptr;
    int (*send)(const void*, size_t, int, int, void*, cudaStream_t) = nullptr;
    int (*recv)(void*, size_t, int, int, void*, cudaStream_t) = nullptr;
    int (*allReduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
    int (*broadcast)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
    const char* (*getErrorString)(int) = nullptr;

    static Nccl& get();  // loads on first call
};

constexpr int kNcclDouble = 8;  // ncclFloat64
constexpr int kNcclSum = 0;     // ncclSum

// ncclCommInitRank with the 128-byte unique id.
int nccl_comm_init(void** comm, int nranks, const uint8_t id[128], int rank);

}  // namespace amgb
