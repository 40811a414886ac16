// dlopen-based NCCL loader (see comm.hpp).
#include "comm.hpp"

#include <dlfcn.h>

#include <cstring>

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

}  // namespace amgb
