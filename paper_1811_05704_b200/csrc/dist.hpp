// Row partition of the AMG hierarchy across ranks (PAPER.md:474-499
// runs the method over MPI processes, without describing the partitioning).
//
// Every rank holds the same global host hierarchy (the setup is global and
// deterministic), so every rank can derive every other rank's needs locally and
// no setup-time communication is required.
//
//  * Level 0 rows are split evenly into contiguous ranges.  A coarse unknown J
//    belongs to the rank owning its aggregate root; roots are discovered in
//    ascending fine order, so each coarse level is again a contiguous range.
//  * Levels l < lg ("distributed"): each rank stores its rows of A_l, P_l (fine
//    rows) and R_l (its coarse rows).  Columns are renumbered [local | ghost]:
//    local column c -> c - row0, ghost g -> nloc + position in the sorted ghost
//    list.  Entries keep their GLOBAL column order, so a row sum is evaluated
//    in exactly the order of the single-GPU run.  The ghost list of level l is
//    the union of the outside columns of A_l, R_l and P_{l-1} rows owned here,
//    so one halo plan serves every vector of the level.
//  * Levels l >= lg ("replicated", fewer than gather_below rows): full copies on
//    every rank.  R_{lg-1} writes the rank's slice of the full f_lg, which is
//    then all-gathered; P_{lg-1} reads the full x_lg.
#pragma once
#include <cstdint>
#include <vector>

#include "setup.hpp"

namespace amgb {

struct HaloPlan {
    int64_t nloc = 0, nghost = 0;
    std::vector<int64_t> ghost_global;                         // sorted global indices
    std::vector<int32_t> recv_peer;                            // owners, ascending
    std::vector<int64_t> recv_off, recv_cnt;                   // segment of the ghost region
    std::vector<int32_t> send_peer;                            // ranks that need our values
    std::vector<int64_t> send_off, send_cnt;                   // segment of the packed buffer
    std::vector<int32_t> send_idx;                             // local indices, concatenated
};

struct LevelPart {
    bool replicated = false;
    int64_t row0 = 0, row1 = 0;    // owned rows (global); [0, n) when replicated
    int64_t crow0 = 0, crow1 = 0;  // owned rows of level l+1 (local rows of R)
    bool next_replicated = false;  // level l+1 is replicated
    Csr A, P, R;                   // local matrices (renumbered columns); P/R empty on the coarsest
    // one rank: the host hierarchy's own matrices, not copies (ma/mp/mr read through)
    const Csr *pA = nullptr, *pP = nullptr, *pR = nullptr;
    const Csr& ma() const { return pA ? *pA : A; }
    const Csr& mp() const { return pP ? *pP : P; }
    const Csr& mr() const { return pR ? *pR : R; }
    HaloPlan halo;                 // plan for vectors of this level (distributed levels)
    std::vector<double> m, diag;   // local rows then ghost values
};

struct RankPart {
    int rank = 0, nranks = 1, lg = 0;
    std::vector<LevelPart> lv;
};

// First replicated level: the first level with fewer than gather_below rows,
// at least 1 (level 0 is always distributed when nranks > 1) and at most the
// coarsest level.  nranks == 1 -> number of levels (nothing replicated).
int first_replicated_level(const HostHierarchy& H, int nranks, int64_t gather_below);

// starts[l][r] = first row of rank r on level l (r = 0..nranks), levels 0..lg.
std::vector<std::vector<int64_t>> level_starts(const HostHierarchy& H, int nranks, int lg);

RankPart build_rank_part(const HostHierarchy& H, int nranks, int rank, int lg,
                         const std::vector<std::vector<int64_t>>& starts);

// ---- scattered setup (one process per GPU): rank 0 builds the global host
// hierarchy once and sends every other rank its part, plus what a rank needs
// to know about the whole hierarchy (level sizes, smoother bounds, partition,
// the replicated coarse inverse).  The other ranks never hold the global matrix.
struct LevelMeta {
    int64_t rows = 0, nnz_A = 0, nnz_P = 0, cols_P = 0, n_agg = 0;
    double lmax = 0, lmin = 0, cheb_d = 0, cheb_c = 0;
};
std::vector<LevelMeta> level_meta(const HostHierarchy& H);

struct PartHeader {
    std::vector<LevelMeta> meta;
    int lg = 0;
    std::vector<std::vector<int64_t>> starts;
    std::vector<double> coarse_inv;
};
// Flat byte image of (header, part) and back (same host ABI on every rank).
void pack_part(const PartHeader& hd, const RankPart& rp, std::vector<uint8_t>& out);
void unpack_part(const uint8_t* p, size_t n, PartHeader& hd, RankPart& rp);

}  // namespace amgb
