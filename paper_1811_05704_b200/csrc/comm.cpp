// dlopen-based NCCL loader (see comm.hpp).
#include "comm.hpp"

#include <dlfcn.h>

#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <thread>

namespace amgb {

namespace {
struct UniqueId {
    char internal[128];
};
typedef int (*InitRankFn)(void**, int, UniqueId, int);
}  // namespace

Nccl& Nccl::get() {
    static Nccl n;
    static bool tried = false;
    if (tried) return n;
    tried = true;
    // prefer the NCCL already in the process (torch's), then the default search
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
        n.error = std::string("cannot load libnccl.so.2: ") + dlerror();
        return n;
    }
    n.lib = h;
    bool all = true;
    auto sym = [&](const char* name) {
        void* p = dlsym(h, name);
        if (!p) all = false;
        return p;
    };
    n.getUniqueId = reinterpret_cast<int (*)(void*)>(sym("ncclGetUniqueId"));
    n.commInitRank = sym("ncclCommInitRank");
    n.commDestroy = reinterpret_cast<int (*)(void*)>(sym("ncclCommDestroy"));
    n.groupStart = reinterpret_cast<int (*)()>(sym("ncclGroupStart"));
    n.groupEnd = reinterpret_cast<int (*)()>(sym("ncclGroupEnd"));
    n.send = reinterpret_cast<int (*)(const void*, size_t, int, int, void*, cudaStream_t)>(sym("ncclSend"));
    n.recv = reinterpret_cast<int (*)(void*, size_t, int, int, void*, cudaStream_t)>(sym("ncclRecv"));
    n.allReduce =
        reinterpret_cast<int (*)(const void*, void*, size_t, int, int, void*, cudaStream_t)>(sym("ncclAllReduce"));
    n.broadcast =
        reinterpret_cast<int (*)(const void*, void*, size_t, int, int, void*, cudaStream_t)>(sym("ncclBroadcast"));
    n.getErrorString = reinterpret_cast<const char* (*)(int)>(sym("ncclGetErrorString"));
    n.ok = all;
    n.commGetAsyncError = reinterpret_cast<int (*)(void*, int*)>(dlsym(h, "ncclCommGetAsyncError"));
    n.commAbort = reinterpret_cast<int (*)(void*)>(dlsym(h, "ncclCommAbort"));
    if (!all) n.error = "libnccl.so.2 lacks a required symbol";
    return n;
}

int nccl_comm_init(void** comm, int nranks, const uint8_t id[128], int rank) {
    Nccl& n = Nccl::get();
    if (!n.ok) return -1;
    UniqueId u;
    std::memcpy(u.internal, id, 128);
    return reinterpret_cast<InitRankFn>(n.commInitRank)(comm, nranks, u, rank);
}

double nccl_timeout_s() {
    const char* e = std::getenv("AMGB_NCCL_TIMEOUT_S");
    const double t = e ? std::atof(e) : 0.0;
    return t > 0 ? t : 300.0;
}

int nccl_comm_init_timeout(void** comm, int nranks, const uint8_t id[128], int rank, int device, double timeout_s) {
    struct Shared {
        std::mutex m;
        std::condition_variable cv;
        bool done = false;
        int rc = 0;
        void* comm = nullptr;
    };
    auto sh = std::make_shared<Shared>();
    uint8_t idc[128];
    std::memcpy(idc, id, 128);
    std::thread([sh, nranks, rank, device, idc]() {
        cudaSetDevice(device);
        void* c = nullptr;
        const int rc = nccl_comm_init(&c, nranks, idc, rank);
        std::lock_guard<std::mutex> g(sh->m);
        sh->rc = rc;
        sh->comm = c;
        sh->done = true;
        sh->cv.notify_all();
    }).detach();
    std::unique_lock<std::mutex> lk(sh->m);
    if (!sh->cv.wait_for(lk, std::chrono::duration<double>(timeout_s), [&] { return sh->done; })) return -2;
    *comm = sh->comm;
    return sh->rc;
}

}  // namespace amgb
