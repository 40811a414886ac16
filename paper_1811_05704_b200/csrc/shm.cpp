// Host shared-memory test transport (see shm.hpp).
#include "shm.hpp"

#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <thread>

namespace amgb {

namespace {

// a named POSIX shared-memory object of `bytes` bytes, mapped read/write
void* map_object(const std::string& name, size_t bytes, bool create) {
    const int fd = shm_open(name.c_str(), create ? (O_CREAT | O_RDWR) : O_RDWR, 0600);
    if (fd < 0) throw std::runtime_error("shm_open " + name + ": " + std::strerror(errno));
    if (create && ftruncate(fd, (off_t)bytes) != 0) {
        close(fd);
        throw std::runtime_error("ftruncate " + name + ": " + std::strerror(errno));
    }
    void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (p == MAP_FAILED) throw std::runtime_error("mmap " + name + ": " + std::strerror(errno));
    return p;
}

size_t object_size(const std::string& name) {
    const int fd = shm_open(name.c_str(), O_RDONLY, 0600);
    if (fd < 0) throw std::runtime_error("shm_open " + name + ": " + std::strerror(errno));
    struct stat st;
    fstat(fd, &st);
    close(fd);
    return (size_t)st.st_size;
}

}  // namespace

ShmComm::ShmComm(const uint8_t id[128], int rank, int nranks, double timeout_s)
    : rank_(rank), nranks_(nranks), timeout_(timeout_s) {
    char hex[33];
    for (int i = 0; i < 16; ++i) std::snprintf(hex + 2 * i, 3, "%02x", id[i] ^ id[16 + i] ^ id[32 + i]);
    tag_ = std::string("/amgb_") + hex;
    bar_ = static_cast<int64_t*>(map_object(tag_ + "_bar", 4096, true));
    barrier();  // every rank has the barrier object open
}

ShmComm::~ShmComm() {
    if (bar_) munmap(bar_, 4096);
    if (rank_ == 0) shm_unlink((tag_ + "_bar").c_str());
}

void ShmComm::barrier() {
    auto* cnt = reinterpret_cast<std::atomic<int64_t>*>(bar_);
    ++nbar_;
    cnt->fetch_add(1, std::memory_order_acq_rel);
    const int64_t target = nbar_ * nranks_;
    const auto t0 = std::chrono::steady_clock::now();
    while (cnt->load(std::memory_order_acquire) < target) {
        if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > timeout_)
            throw std::runtime_error("shm transport: a peer rank did not reach the barrier within the timeout");
        std::this_thread::sleep_for(std::chrono::microseconds(20));
    }
}

void ShmComm::alltoallv(const std::vector<std::vector<uint8_t>>& out, std::vector<std::vector<uint8_t>>& in) {
    // this rank's outbox: [nranks] (offset, size) then the payloads
    const int64_t s = ++seq_;
    auto box = [&](int r) { return tag_ + "_" + std::to_string(s) + "_" + std::to_string(r); };
    size_t total = sizeof(int64_t) * 2 * nranks_;
    for (const auto& v : out) total += v.size();
    uint8_t* mine = static_cast<uint8_t*>(map_object(box(rank_), total, true));
    int64_t off = (int64_t)(sizeof(int64_t) * 2 * nranks_);
    for (int p = 0; p < nranks_; ++p) {
        const int64_t sz = p < (int)out.size() ? (int64_t)out[p].size() : 0;
        std::memcpy(mine + 16 * p, &off, 8);
        std::memcpy(mine + 16 * p + 8, &sz, 8);
        if (sz) std::memcpy(mine + off, out[p].data(), sz);
        off += sz;
    }
    barrier();  // every outbox is written
    in.assign(nranks_, {});
    for (int p = 0; p < nranks_; ++p) {
        const size_t bytes = object_size(box(p));
        uint8_t* theirs = static_cast<uint8_t*>(map_object(box(p), bytes, false));
        int64_t o = 0, sz = 0;
        std::memcpy(&o, theirs + 16 * rank_, 8);
        std::memcpy(&sz, theirs + 16 * rank_ + 8, 8);
        in[p].assign(theirs + o, theirs + o + sz);
        munmap(theirs, bytes);
    }
    barrier();  // every rank has read its segments
    munmap(mine, total);
    shm_unlink(box(rank_).c_str());
}

}  // namespace amgb
