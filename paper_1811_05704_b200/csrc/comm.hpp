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
    // fault handling (optional symbols; NCCL >= 2.4): a peer that died or never
    // joined turns into AMG_E_NCCL after a timeout instead of a hang
    int (*commGetAsyncError)(void*, int*) = nullptr;
    int (*commAbort)(void*) = nullptr;

    static Nccl& get();  // loads on first call
};

constexpr int kNcclDouble = 8;  // ncclFloat64
constexpr int kNcclSum = 0;     // ncclSum

constexpr int kNcclUint8 = 1;   // ncclUint8
constexpr int kNcclInProgress = 7;

// ncclCommInitRank with the 128-byte unique id.
int nccl_comm_init(void** comm, int nranks, const uint8_t id[128], int rank);

// Seconds a multi-GPU handle waits for a peer (communicator creation, the
// setup scatter, every host synchronisation of a solve) before it aborts the
// communicator and reports AMG_E_NCCL: AMGB_NCCL_TIMEOUT_S, default 300.
double nccl_timeout_s();

// nccl_comm_init on a helper thread (device `device` current there), waiting at
// most timeout_s: 0 = the communicator is up; -2 = timed out (the helper thread
// stays blocked inside NCCL and is detached: the peers never joined); other
// values: the NCCL error.
int nccl_comm_init_timeout(void** comm, int nranks, const uint8_t id[128], int rank, int device, double timeout_s);

}  // namespace amgb
