// Host shared-memory transport between the ranks of a multi-process handle on
// ONE node -- a TEST transport (AMGB_TRANSPORT=shm): it lets two or more
// processes that share a single GPU run the one-process-per-rank path of the
// executor (scattered setup, per-rank vectors, halo plans, all-reduce and
// coarse all-gather) end to end, where NCCL refuses two ranks on one device.
// Every operation is synchronous on the host: the caller synchronises its
// stream, the bytes go device -> host -> shared memory -> host -> device, and
// the ranks meet at host barriers.  No kernel ever waits on another rank (the
// rule of the B200 profiling guide for ranks sharing a GPU), so graph capture
// is not used with this transport.  Every wait is bounded by a timeout.
#pragma once
#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

namespace amgb {

class ShmComm {
  public:
    // Attach rank `rank` of `nranks` to the region named after the 128-byte id
    // (every rank passes the same id); waits for all ranks (barrier).
    ShmComm(const uint8_t id[128], int rank, int nranks, double timeout_s);
    ~ShmComm();
    ShmComm(const ShmComm&) = delete;
    ShmComm& operator=(const ShmComm&) = delete;

    int rank() const { return rank_; }
    int nranks() const { return nranks_; }
    void barrier();
    // Personalised all-to-all: out[p] = bytes for rank p (may be empty);
    // returns in[p] = the bytes rank p sent to this rank.
    void alltoallv(const std::vector<std::vector<uint8_t>>& out, std::vector<std::vector<uint8_t>>& in);

  private:
    std::string tag_;
    int rank_, nranks_;
    double timeout_;
    int64_t* bar_ = nullptr;  // shared monotonic barrier counter
    int64_t nbar_ = 0;        // barriers passed by this rank
    int64_t seq_ = 0;         // alltoallv calls made (equal on every rank)
};

}  // namespace amgb
