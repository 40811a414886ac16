// amgb.cu -- device hierarchy store, V-cycle executor, CG / BiCGStab drivers and
// the C ABI (include/amgb.h).
//
// Solve phase of arXiv 1811.05704 (AMGCL): Algorithm 2 as the
// preconditioner of CG / BiCGStab.  The
// hierarchy comes from setup.cpp (Algorithm 1, on the host)
// and is uploaded once.  Every step of the solve runs in the
// kernels of kernels.cuh / ops.cuh; the host only sequences launches and reads
// one small state struct per pair of Krylov iterations.
//
// Multi-GPU: a handle holds one or more "parts" (row slices of
// the hierarchy, dist.hpp).  With NCCL there is one part per process; in
// virtual mode one process holds every part on one GPU and the transport is
// device-to-device copies (used to test the partitioned path on one GPU).  The
// executor issues every step for every part, with halo exchanges before each
// distributed matrix pass and an all-reduce after each fused dot.
#include <cuda_runtime.h>

#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <chrono>
#include <cstdlib>
#include <numeric>
#include <cstring>
#include <functional>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "../../include/amgb.h"
#include "batched.cuh"
#include "comm.hpp"
#include "dist.hpp"
#include "gmres.cuh"
#include "idrs.cuh"
#include "convert.cuh"
#include "kernels.cuh"
#include "ops.cuh"
#include "setup.hpp"
#include "shm.hpp"

namespace amgb {

// ============================================================ multi-part kernels

// sendbuf[k] = v[idx[k]] (halo pack)
__global__ void __launch_bounds__(kBlock) pack_kernel(const int32_t* __restrict__ idx, const double* __restrict__ v,
                                                      double* __restrict__ out, int64_t n) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
        out[k] = v[idx[k]];
}

// deferred finalize after the cross-rank all-reduce of a fused dot
template <class Fin>
__global__ void fin_kernel(Fin fin, const double* tot, const int32_t* gate) {
    if (gated(gate)) return;
    fin(tot);
}

// virtual-mode all-reduce: every part's totals <- sum over parts in rank order
// Locality reordering of the device store (params.reorder): natural -> stored
// order (dst[q[i]] = src[i]) and back (dst[i] = src[q[i]]).
__global__ void perm_to_kernel(int64_t n, const int64_t* q, const double* src, double* dst) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        dst[q[i]] = src[i];
}
__global__ void perm_from_kernel(int64_t n, const int64_t* q, const double* src, double* dst) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[q[i]];
}

// Split pass (interior + boundary launches): fold the deferred totals of the
// launches that ran (slot k at defer + k * kSlot) into slot 0, fixed order.
constexpr int kSlot = 8;
__global__ void sum_slots_kernel(double* defer, int nv, unsigned mask) {
    if (threadIdx.x != 0) return;
    for (int k = 0; k < nv; ++k) {
        double s = 0.0;
        for (int q = 0; q < 3; ++q)
            if (mask >> q & 1) s += defer[q * kSlot + k];
        defer[k] = s;
    }
}

__global__ void sum_parts_kernel(double* const* parts, int nparts, int nv) {
    const int k = threadIdx.x;
    if (k >= nv) return;
    double s = 0.0;
    for (int p = 0; p < nparts; ++p) s += parts[p][k];
    for (int p = 0; p < nparts; ++p) parts[p][k] = s;
}

// CG ghost update: pn[g] = z[g] + beta p[g] on the ghost region (the local
// rows of pn are written by the CG direction kernel)
__global__ void __launch_bounds__(kBlock) ghost_dir_kernel(const double* z, const double* p, double* pn, int64_t n,
                                                           const KState* ks, const int32_t* gate) {
    if (gated(gate)) return;
    const double beta = ks->beta;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        pn[i] = fma(beta, p[i], z[i]);
}

// device-side loop test of the Krylov iteration graph (conditional WHILE node):
// keep iterating while the solve is not done
__global__ void set_loop_kernel(cudaGraphConditionalHandle h, const int32_t* done) {
    cudaGraphSetConditional(h, *reinterpret_cast<const volatile int32_t*>(done) ? 0u : 1u);
}

// ============================================================ host side

namespace {

thread_local std::string g_err;

struct CudaError {
    std::string msg;
    int code = AMG_E_CUDA;  // AMG_E_NCCL for a failed / timed-out collective
};

inline void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        (void)cudaGetLastError();  // a failed call must not resurface in a later, unrelated check
        throw CudaError{std::string(what) + ": " + cudaGetErrorString(e)};
    }
}

inline void ckn(int r, const char* what) {
    if (r != 0) {
        Nccl& n = Nccl::get();
        throw CudaError{std::string(what) + ": NCCL error " + std::to_string(r) +
                            (n.getErrorString && r > 0 ? std::string(" ") + n.getErrorString(r) : std::string()),
                        AMG_E_NCCL};
    }
}


struct HostSell {
    int64_t nrows = 0, ncols = 0, nslices = 0;
    std::vector<int64_t> sptr;
    hvec<int32_t> col;
    hvec<double> val;
};

// CSR -> SELL-C, slice height C (see kernels.cuh): entry k of row s*C + r at
// sptr[s] + k*C + r.  Padding repeats the row's last column with value 0.
HostSell to_sell(const Csr& A, int C = 32) {
    HostSell S;
    S.nrows = A.nrows;
    S.ncols = A.ncols;
    S.nslices = (A.nrows + C - 1) / C;
    S.sptr.assign(S.nslices + 1, 0);
    for (int64_t s = 0; s < S.nslices; ++s) {
        int64_t w = 0;
        for (int64_t r = s * C; r < std::min<int64_t>(A.nrows, s * C + C); ++r)
            w = std::max<int64_t>(w, A.ptr[r + 1] - A.ptr[r]);
        S.sptr[s + 1] = S.sptr[s] + C * w;
    }
    S.col.resize(S.sptr[S.nslices]);  // every element written below (entries + padding)
    S.val.resize(S.sptr[S.nslices]);
#pragma omp parallel for schedule(static)
    for (int64_t s = 0; s < S.nslices; ++s) {
        const int64_t w = (S.sptr[s + 1] - S.sptr[s]) / C;
        for (int lane = 0; lane < C; ++lane) {
            const int64_t r = s * C + lane;
            int64_t len = 0;
            int32_t last = 0;
            if (r < A.nrows) {
                len = A.ptr[r + 1] - A.ptr[r];
                for (int64_t k = 0; k < len; ++k) {
                    S.col[S.sptr[s] + C * k + lane] = A.col[A.ptr[r] + k];
                    S.val[S.sptr[s] + C * k + lane] = A.val[A.ptr[r] + k];
                }
                if (len > 0) last = A.col[A.ptr[r] + len - 1];
            }
            for (int64_t k = len; k < w; ++k) {
                S.col[S.sptr[s] + C * k + lane] = last;
                S.val[S.sptr[s] + C * k + lane] = 0.0;
            }
        }
    }
    return S;
}

// Column storage of the TMA-staged SELL-32 format ("offset
// dictionary").  A slice whose 32 rows share one sorted set U of column offsets
// (col - row) with |U| = the slice width, and for which every row + u is a
// valid column, stores U once (w ints) instead of 32 w column indices; its
// values are re-laid out at U's positions with zeros where a row lacks an
// offset (0 * x_j added in column order leaves every row sum unchanged).  Other
// slices keep explicit indices.  cptr[s]: first int of slice s; each tile of 8
// slices starts 16-byte aligned (cp.async.bulk), so a slice is a dictionary iff
// cptr[s+1] - cptr[s] < 32 w.
struct HostTmaCols {
    std::vector<int64_t> cptr;
    hvec<int32_t> col;
    int64_t idx_bytes = 0;  // index bytes the format needs (excl. alignment/padding)
    int64_t ndict = 0;      // dictionary slices
};

HostTmaCols tma_cols(const Csr& A, HostSell& S, bool allow_dict) {
    constexpr int C = 32;
    constexpr int kW = 16;  // dictionary slices have at most kW offsets
    const int64_t ns = S.nslices;
    hvec<int32_t> U((size_t)ns * kW);
    hvec<int32_t> ulen(ns);  // offsets in the slice's dictionary (0: explicit slice)
    hvec<int64_t> true_nnz(ns);
#pragma omp parallel
    {
        std::vector<int64_t> offs(C * kW);
#pragma omp for schedule(dynamic, 1024)
        for (int64_t s = 0; s < ns; ++s) {
            ulen[s] = 0;
            const int64_t w = (S.sptr[s + 1] - S.sptr[s]) / C;
            const int64_t r0 = s * C, r1 = std::min<int64_t>(A.nrows, r0 + C);
            true_nnz[s] = A.ptr[r1] - A.ptr[r0];
            if (!allow_dict || w == 0 || w > kW || r1 - r0 < C) continue;
            size_t no = 0;
            bool sorted = true;  // the value layout below needs ascending columns in every row
            for (int64_t r = r0; r < r1; ++r)
                for (int64_t e = A.ptr[r]; e < A.ptr[r + 1]; ++e) {
                    offs[no++] = (int64_t)A.col[e] - r;
                    if (e > A.ptr[r] && A.col[e] <= A.col[e - 1]) sorted = false;
                }
            if (!sorted) continue;
            std::sort(offs.begin(), offs.begin() + no);
            no = std::unique(offs.begin(), offs.begin() + no) - offs.begin();
            if ((int64_t)no != w) continue;
            bool ok = true;
            for (int64_t r = r0; r < r1 && ok; ++r) ok = r + offs[0] >= 0 && r + offs[no - 1] < A.ncols;
            if (!ok) continue;
            int32_t* u = U.data() + (size_t)s * kW;
            for (size_t k = 0; k < no; ++k) u[k] = (int32_t)offs[k];
            ulen[s] = (int32_t)no;
            // values at U's positions (the row's entries are ascending, so are U's)
            for (int lane = 0; lane < C; ++lane) {
                const int64_t r = r0 + lane;
                int64_t k = 0;
                for (int64_t e = A.ptr[r]; e < A.ptr[r + 1]; ++e) {
                    const int64_t off = (int64_t)A.col[e] - r;
                    for (; u[k] != off; ++k) {
                        S.val[S.sptr[s] + C * k + lane] = 0.0;
                        S.col[S.sptr[s] + C * k + lane] = (int32_t)(r + u[k]);
                    }
                    S.val[S.sptr[s] + C * k + lane] = A.val[e];
                    S.col[S.sptr[s] + C * k + lane] = A.col[e];
                    ++k;
                }
                for (; k < w; ++k) {
                    S.val[S.sptr[s] + C * k + lane] = 0.0;
                    S.col[S.sptr[s] + C * k + lane] = (int32_t)(r + u[k]);
                }
            }
        }
    }
    HostTmaCols T;
    T.cptr.assign(ns + 1, 0);
    int64_t cur = 0;
    for (int64_t s = 0; s < ns; ++s) {
        if (s % 8 == 0) cur = (cur + 3) & ~int64_t(3);
        T.cptr[s] = cur;
        const int64_t w = (S.sptr[s + 1] - S.sptr[s]) / C;
        if (ulen[s]) {
            cur += w;
            T.idx_bytes += 4 * w;
            ++T.ndict;
        } else {
            cur += C * w;
            T.idx_bytes += 4 * true_nnz[s];
        }
    }
    T.cptr[ns] = (cur + 3) & ~int64_t(3);
    T.col.resize(T.cptr[ns]);
#pragma omp parallel for schedule(static)
    for (int64_t s = 0; s < ns; ++s) {
        int32_t* out = T.col.data() + T.cptr[s];
        if (ulen[s])
            std::copy(U.data() + (size_t)s * kW, U.data() + (size_t)s * kW + ulen[s], out);
        else
            std::copy(S.col.begin() + S.sptr[s], S.col.begin() + S.sptr[s + 1], out);
        const int64_t len = ulen[s] ? ulen[s] : S.sptr[s + 1] - S.sptr[s];
        for (int64_t q = T.cptr[s] + len; q < T.cptr[s + 1]; ++q) T.col[q] = 0;  // alignment padding
    }
    return T;
}

// bytes of one stage of the TMA-staged CSR kernel (csr_tma): values (vbytes
// each: 8, 4 with fp32, 1 / 2 with value indices), columns (tile_ent each, a
// multiple of 16) and the tile's row pointers, 16-B aligned
inline size_t tcsr_stage_bytes(int64_t tile_ent, int vbytes) {
    return (((size_t)tile_ent * (vbytes + 4) + (size_t)(kTcRows + 8) * 4) + 15) & ~(size_t)15;
}
// shared-memory bytes of a csr_tma value table of ntab entries
inline size_t tcsr_vtab_bytes(int64_t ntab) { return ((size_t)ntab * 8 + 127) & ~(size_t)127; }

// A device matrix in the format chosen for it.
enum class Fmt { CSR, SELL, TMA, TMACSR };

struct DMat {
    Fmt fmt = Fmt::CSR;
    Sell sell;
    SellTma tma;
    CsrDev csr;
    CsrTma tcsr;
    int64_t nrows = 0, ncols = 0, nnz = 0, stored = 0;
    int64_t idx_bytes = -1;  // column-index bytes the format needs (-1: 4 per entry)
    int vbytes = 8;          // value bytes per entry: 8, or 1 / 2 with value-indexed storage
    int64_t ndict = 0;       // TMA slices stored with an offset dictionary
    bool sigma = false;      // rows sorted by length inside 256-row windows (sigma_sort)
    // algorithmic matrix bytes of one pass: values + the indices the format needs
    double mat_bytes(bool f32) const {
        return (f32 ? 4.0 : (double)vbytes) * nnz + (idx_bytes < 0 ? 4.0 * nnz : (double)idx_bytes);
    }
    // row-structure bytes the format's kernel reads per pass: CSR row pointers
    // (4 B per row) and row-block starts; SELL-32 one 8-B slice offset per 32
    // rows; TMA two (values and column offsets per slice)
    double ptr_bytes() const {
        const double ns = (double)((nrows + 31) / 32);
        if (fmt == Fmt::TMA) return 16.0 * ns;
        if (fmt == Fmt::SELL) return 8.0 * ns;
        if (fmt == Fmt::TMACSR) return 4.0 * nrows;
        return 4.0 * nrows + 4.0 * (double)csr.nblocks;
    }
    // Multi-GPU split pass: rows [ib0, ib1) have no ghost column
    // and run while the halo exchange is in flight, the rest after it.
    bool split = false;
    int64_t ib0 = 0, ib1 = 0;
    std::vector<int32_t> hblocks;  // row-block starts of the CSR format (host copy)
    double bytes_scale = 1.0;      // views: share of the pass's algorithmic bytes
    const DMat* origin = nullptr;  // views: the matrix they cut
    DMat view(int64_t r0, int64_t r1, double scale) const {
        DMat v;
        v.fmt = fmt;
        v.nrows = r1 - r0;
        v.ncols = ncols;
        v.nnz = nnz;
        v.idx_bytes = idx_bytes;
        v.bytes_scale = scale;
        v.origin = origin ? origin : this;
        if (fmt == Fmt::TMACSR) {
            v.tcsr = tcsr;
            v.tcsr.row0 = tcsr.row0 + r0;
            v.tcsr.nrows = r1 - r0;
            v.tcsr.ptr = tcsr.ptr + r0;
            v.tcsr.ntiles = (r1 - r0 + kTcRows - 1) / kTcRows;
        } else if (fmt == Fmt::TMA) {
            v.tma = tma;
            v.tma.row0 = tma.row0 + r0;
            v.tma.nrows = r1 - r0;
            v.tma.sptr = tma.sptr + r0 / 32;
            v.tma.cptr = tma.cptr + r0 / 32;
            v.tma.nslices = (r1 - r0 + 31) / 32;
            v.tma.ntiles = (v.tma.nslices + 7) / 8;
        } else if (fmt == Fmt::SELL) {
            v.sell = sell;
            v.sell.row0 = sell.row0 + r0;
            v.sell.nrows = r1 - r0;
            v.sell.sptr = sell.sptr + r0 / 32;
            v.sell.nslices = (r1 - r0 + 31) / 32;
        } else {
            const int64_t b0 = std::lower_bound(hblocks.begin(), hblocks.end(), (int32_t)r0) - hblocks.begin();
            const int64_t b1 = std::lower_bound(hblocks.begin(), hblocks.end(), (int32_t)r1) - hblocks.begin();
            v.csr = csr;
            v.csr.brow = csr.brow + b0;
            v.csr.nblocks = b1 - b0;
        }
        return v;
    }
};

// Interior rows of a distributed matrix: the longest run of rows whose columns
// are all local (< nloc), cut to the format's granularity (256-row tiles, 32-row
// slices, CSR row blocks).  {0, 0}: no split.
std::pair<int64_t, int64_t> interior_range(const Csr& M, int64_t nloc, Fmt fmt, const std::vector<int32_t>& blocks) {
    int64_t best0 = 0, best1 = 0, run0 = 0;
    for (int64_t i = 0; i <= M.nrows; ++i) {
        bool ghost = i == M.nrows;
        for (int64_t k = ghost ? 0 : M.ptr[i]; !ghost && k < M.ptr[i + 1]; ++k) ghost = M.col[k] >= nloc;
        if (ghost) {
            if (i - run0 > best1 - best0) best0 = run0, best1 = i;
            run0 = i + 1;
        }
    }
    int64_t a = best0, b = best1;
    if (fmt == Fmt::CSR) {
        auto lo = std::lower_bound(blocks.begin(), blocks.end(), (int32_t)a);
        auto hi = std::upper_bound(blocks.begin(), blocks.end(), (int32_t)b);
        if (lo == blocks.end() || hi == blocks.begin()) return {0, 0};
        a = *lo;
        b = *(hi - 1);
    } else {
        const int64_t g = (fmt == Fmt::TMA || fmt == Fmt::TMACSR) ? 256 : 32;
        a = (a + g - 1) / g * g;
        b = b == M.nrows ? b : b / g * g;
    }
    if (b <= a) return {0, 0};
    return {a, b};
}

// One level of one part.  Vectors that are gathered by a matrix pass have a
// ghost region after the n local entries.
struct DevLevel {
    bool replicated = true, next_replicated = true;
    int64_t n = 0;                 // local rows
    int64_t ng = 0;                // ghost entries
    int64_t nc = 0;                // columns of P (coarse local + ghost, or the full coarse size)
    int64_t crow0 = 0, crow1 = 0;  // local rows of R (slice of level l+1)
    int64_t nnzA = 0, nnzP = 0, nnzR = 0, padA = 0, dictA = 0;
    DMat A, P, R;
    double* m = nullptr;     // SPAI-0 / Jacobi diagonal (local + ghost)
    double* diag = nullptr;  // a_ii (Chebyshev)
    double* f = nullptr;     // right-hand side (levels >= 1)
    double* x = nullptr;     // work
    double* y = nullptr;     // work (ping-pong)
    double* t = nullptr;     // residual
    double* p = nullptr;     // Chebyshev direction
    double* o = nullptr;     // V-cycle output (levels >= 1)
    double* mf = nullptr;    // m o f, written by the restriction into this level (levels >= 1)
    std::vector<double> cheb_alpha, cheb_beta;
    double alg_bytes = 0;
    int64_t dev_bytes = 0;
    // halo (distributed levels)
    HaloPlan plan;
    int32_t* send_idx = nullptr;
    double* sendbuf = nullptr;
    int64_t nsend = 0;
};

struct Part {
    int rank = 0;
    int64_t row0 = 0, row1 = 0;  // level-0 rows
    std::vector<DevLevel> lv;
    double* coarse_inv = nullptr;
    int64_t nL = 0;
    KState* ks = nullptr;
    Red red;
    // Krylov vectors (level-0 local length + ghosts where gathered)
    double *r = nullptr, *r2 = nullptr, *z = nullptr, *pa = nullptr, *pb = nullptr, *q = nullptr, *xw = nullptr;
    double *rhat = nullptr, *v = nullptr, *s = nullptr, *sh = nullptr, *ph = nullptr, *tv = nullptr;
    const double* fcur = nullptr;  // right-hand side of the current solve (local slice)
    double* xcur = nullptr;        // solution vector of the current solve (with ghosts if needed)
};

double level_alg_bytes(int64_t n_, int64_t z_, int64_t p_, int64_t c_, const amg_params& p, bool coarsest);

}  // namespace

struct Handle {
    amg_params prm{};
    HostHierarchy host;
    bool on_device = false;
    int device = 0;
    int num_sms = 148;
    cudaStream_t stream = nullptr;      // work stream (own_stream unless set by the caller)
    cudaStream_t own_stream = nullptr;  // blocking stream: ordered with the legacy default stream
    // partition
    int nranks = 1;        // total ranks of the partition
    bool virt = false;     // every part lives in this process (one GPU)
    int lg = 1;            // first replicated level
    void* nccl = nullptr;  // ncclComm_t (NCCL mode)
    std::unique_ptr<ShmComm> shm;  // test transport (AMGB_TRANSPORT=shm): ranks sharing one GPU
    std::vector<std::vector<int64_t>> starts;  // level_starts
    std::vector<RankPart> host_parts;          // host copies (export / upload)
    std::vector<LevelMeta> meta;               // every level's global sizes / smoother bounds (all ranks)
    std::vector<double> coarse_inv;            // row-major A_L^-1 (replicated coarsest level)
    std::vector<Part> parts;
    double** d_defer_ptrs = nullptr;       // virtual all-reduce: device array of part->defer
    KState* ks_host = nullptr;             // pinned (part 0)
    double *hf = nullptr, *hx = nullptr;   // device copies for amg_solve_host
    // amg_solve_host_stream: fixed solve vectors (the iteration graph is keyed by
    // x) and double-buffered input / output staging vectors for the copy stream
    double *sf = nullptr, *sx = nullptr, *sin[2] = {nullptr, nullptr}, *sout[2] = {nullptr, nullptr};
    std::vector<void*> allocs;
    // CUDA graph of two Krylov iterations, keyed by the x pointer
    cudaGraphExec_t graph = nullptr;
    const double* graph_x = nullptr;
    int graph_prof_mask = 0;
    int64_t graph_kernels = 0;
    bool graph_loop = false;  // the graph runs the whole loop (conditional WHILE node)
    int graph_variant = -1;   // cg_fused | mf0 << 1 of the captured iterations
    // accounting
    int64_t launches = 0;
    amg_solve_stats stats{};
    bool sync_debug = false;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;

    bool distributed() const { return nranks > 1; }


    template <class T>
    T* talloc(int64_t n) {  // uninitialised device array owned by the handle
        void* p = nullptr;
        ck(cudaMalloc(&p, std::max<int64_t>(n, 1) * sizeof(T)), "cudaMalloc");
        allocs.push_back(p);
        return static_cast<T*>(p);
    }
    void tfree(const void* p) {  // release a talloc / upload allocation early
        auto it = std::find(allocs.begin(), allocs.end(), const_cast<void*>(p));
        if (it != allocs.end()) {
            cudaFree(*it);
            allocs.erase(it);
        }
    }
        double* dalloc(int64_t n) {
        void* p = nullptr;
        ck(cudaMalloc(&p, std::max<int64_t>(n, 1) * sizeof(double)), "cudaMalloc");
        ck(cudaMemset(p, 0, std::max<int64_t>(n, 1) * sizeof(double)), "cudaMemset");
        allocs.push_back(p);
        return static_cast<double*>(p);
    }
    template <class T, class Al>
    T* upload(const std::vector<T, Al>& v) {
        void* p = nullptr;
        ck(cudaMalloc(&p, std::max<size_t>(v.size(), 1) * sizeof(T)), "cudaMalloc");
        allocs.push_back(p);
        const auto t0 = std::chrono::steady_clock::now();
        if (!v.empty()) ck(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice), "upload");
        upload_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        upload_bytes += (double)v.size() * sizeof(T);
        return static_cast<T*>(p);
    }
    double upload_ms = 0, upload_bytes = 0;  // setup statistics (AMGB_SETUP_TIMING)
    // locality reordering (params.reorder = 1, single GPU): the device store
    // holds Q_l A_l Q_l^T etc.; API vectors are permuted on entry / exit
    bool reordered = false;
    std::vector<double> coarse_inv_perm;
    int64_t* dq0 = nullptr;        // q_0 on the device
    std::vector<int64_t*> dq;      // q_l on the device, every level
    std::vector<std::vector<int64_t>> reorder_q;
    double *rf = nullptr, *rx = nullptr;
    // matrices larger than this are read evict-first (AMGB_STREAM_MB overrides)
    int64_t stream_bytes = (std::getenv("AMGB_STREAM_MB") ? std::atoll(std::getenv("AMGB_STREAM_MB")) : 48) << 20;
    ~Handle() {
        free_batch();
        free_gmres();
        free_idr();
        if (graph) cudaGraphExecDestroy(graph);
        for (cudaEvent_t e : ev_all) cudaEventDestroy(e);
        for (void* p : allocs) cudaFree(p);
        if (ks_host) cudaFreeHost(ks_host);
        if (ev0) cudaEventDestroy(ev0);
        if (ev1) cudaEventDestroy(ev1);
        if (own_stream) cudaStreamDestroy(own_stream);
        if (comm_stream) cudaStreamDestroy(comm_stream);
        if (ev_pack) cudaEventDestroy(ev_pack);
        if (ev_halo) cudaEventDestroy(ev_halo);
        if (nccl && Nccl::get().commDestroy) Nccl::get().commDestroy(nccl);
    }

    // Kernels that start with pdl_wait() can be launched with programmatic stream
    // serialization (AMGB_PDL=1), which lets a launch overlap the tail of the
    // previous kernel.  Off by default: measured on the 256^3 solve it made the
    // iteration graph 38% SLOWER (62.5 vs 45.2 ms), so plain stream order it is.
    bool pdl = [] {
        const char* e = std::getenv("AMGB_PDL");
        return e && std::string(e) == "1";
    }();
    // PDL pays only where the passes are short, launch-latency-bound work:
    // measured 0.69 vs 0.75 ms per 32^3 solve and 1.53 vs 1.56 ms at 64^3, but
    // 8.4 vs 7.5 ms at 150^3 and 41.5 vs 35.7 ms at 256^3 (profiles/r02_misc).  On
    // by default for hierarchies whose finest level has fewer than 500,000 rows;
    // AMGB_PDL=0 / 1 forces it.
    void choose_pdl(int64_t n0) {
        const char* e = std::getenv("AMGB_PDL");
        pdl = e ? std::string(e) == "1" : n0 < 500000;
    }
    template <class... KArgs, class... Args>
    void klaunch(void (*k)(KArgs...), dim3 g, dim3 b, size_t smem, Args&&... args) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = g;
        cfg.blockDim = b;
        cfg.dynamicSmemBytes = smem;
        cfg.stream = stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        ck(cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...), "cudaLaunchKernelEx");
    }

    int grid_for(int64_t n) const {
        const int64_t b = (n + kBlock - 1) / kBlock;
        return (int)std::max<int64_t>(1, std::min<int64_t>(b, (int64_t)num_sms * 8));
    }

    // ------------------------------------------------------------ accounting
    // Every launch carries a kernel class (AMG_PROF_*), its algorithmic bytes
    // and the Krylov iteration (0/1 inside a two-iteration
    // group, -1 outside) it belongs to.  Bytes of iterations that actually ran
    // are summed into the solve statistics; in profile mode the classes in
    // prof_mask are bracketed with CUDA events (event-record nodes when the
    // launches are being captured into the iteration graph).
    struct Rec {
        cudaEvent_t a = nullptr, b = nullptr;
        int cls = 0, iter = -1;
        double bytes = 0;
    };
    int prof_mask = 0;
    bool capturing = false;
    int cur_iter = -1;
    std::vector<Rec> rec_direct, rec_graph;  // launches since the last sync / in the graph
    std::vector<cudaEvent_t> ev_pool, ev_all;
    double acc_ms[8] = {}, acc_bytes[8] = {}, alg_bytes = 0;
    int64_t acc_launches[8] = {};

    // ---- batched right-hand sides (single part): interleaved K-column buffers
    struct BLevel {
        double *f = nullptr, *x = nullptr, *y = nullptr, *t = nullptr, *p = nullptr, *o = nullptr;
    };
    struct Batch {
        int K = 0;
        std::vector<BLevel> lv;
        double *r = nullptr, *z = nullptr, *pa = nullptr, *pb = nullptr, *q = nullptr, *xw = nullptr, *fw = nullptr;
        KStateB* ks = nullptr;
        KStateB* ks_host = nullptr;
        std::vector<void*> mem;
        cudaGraphExec_t graph = nullptr;
        std::vector<Rec> rec;
        int64_t graph_kernels = 0;
    } batch;
    // ---- GMRES(m) buffers (single part)
    struct Gmres {
        int m = 0;
        double *V = nullptr, *w = nullptr, *z = nullptr, *u = nullptr, *r = nullptr, *partial = nullptr;
        int64_t nchunks = 0, chunk = 0;
        KStateG* ks = nullptr;
        KStateG* ks_host = nullptr;
        std::vector<void*> mem;
        cudaGraphExec_t graph = nullptr;
        const double* graph_x = nullptr;
        const double* graph_f = nullptr;
        std::vector<Rec> rec;
        int64_t graph_kernels = 0;
    } gm;
    void free_gmres() {
        if (gm.graph) cudaGraphExecDestroy(gm.graph);
        for (void* p : gm.mem) cudaFree(p);
        if (gm.ks_host) cudaFreeHost(gm.ks_host);
        gm = Gmres{};
    }
    // ---- IDR(s) buffers (single part)
    struct Idr {
        int s = 0;
        double *P = nullptr, *G = nullptr, *U = nullptr, *v = nullptr, *z = nullptr, *t = nullptr, *r = nullptr;
        KStateI* ks = nullptr;
        KStateI* ks_host = nullptr;
        std::vector<void*> mem;
        cudaGraphExec_t graph = nullptr;
        const double* graph_x = nullptr;
        const double* graph_f = nullptr;
        std::vector<Rec> rec;
        int64_t graph_kernels = 0;
    } idr;
    void free_idr() {
        if (idr.graph) cudaGraphExecDestroy(idr.graph);
        for (void* p : idr.mem) cudaFree(p);
        if (idr.ks_host) cudaFreeHost(idr.ks_host);
        idr = Idr{};
    }
    void free_batch() {
        if (batch.graph) cudaGraphExecDestroy(batch.graph);
        for (void* p : batch.mem) cudaFree(p);
        if (batch.ks_host) cudaFreeHost(batch.ks_host);
        batch = Batch{};
    }

    cudaEvent_t get_event() {
        if (ev_pool.empty()) {
            cudaEvent_t e;
            ck(cudaEventCreate(&e), "cudaEventCreate");
            ev_all.push_back(e);
            return e;
        }
        cudaEvent_t e = ev_pool.back();
        ev_pool.pop_back();
        return e;
    }
    void record(cudaEvent_t e) {
        if (capturing)
            ck(cudaEventRecordWithFlags(e, stream, cudaEventRecordExternal), "event record node");
        else
            ck(cudaEventRecord(e, stream), "cudaEventRecord");
    }
    bool trace = std::getenv("AMGB_TRACE") != nullptr;
    template <class F>
    void launch(int cls, double bytes, const char* what, F&& fn) {
        if (!in_interior) halo_wait();  // only interior rows may overlap an exchange
        if (trace) {
            std::fprintf(stderr, "[amgb] launch %s\n", what);
            std::fflush(stderr);
        }
        Rec rc;
        rc.cls = cls;
        rc.iter = cur_iter;
        rc.bytes = bytes;
        const bool timed = (prof_mask >> cls) & 1;
        if (timed) {
            rc.a = get_event();
            rc.b = get_event();
            record(rc.a);
        }
        fn();
        if (timed) record(rc.b);
        (capturing ? rec_graph : rec_direct).push_back(rc);
        ++launches;
        if (sync_debug) {
            ck(cudaGetLastError(), what);
            ck(cudaStreamSynchronize(stream), what);
        }
    }
    // After a stream sync: account launches of iterations < ran (and all
    // launches outside iterations); recycle direct-launch events.
    void collect(std::vector<Rec>& v, int ran, bool recycle) {
        for (Rec& rc : v) {
            if (rc.iter >= 0 && rc.iter >= ran) continue;
            alg_bytes += rc.bytes;
            if (rc.a) {
                float ms = 0.f;
                ck(cudaEventElapsedTime(&ms, rc.a, rc.b), "cudaEventElapsedTime");
                acc_ms[rc.cls] += ms;
                acc_bytes[rc.cls] += rc.bytes;
                acc_launches[rc.cls] += 1;
            }
        }
        if (recycle) {
            for (Rec& rc : v)
                if (rc.a) {
                    ev_pool.push_back(rc.a);
                    ev_pool.push_back(rc.b);
                }
            v.clear();
        }
    }
    void drop_graph() {
        if (graph) cudaGraphExecDestroy(graph);
        graph = nullptr;
        for (Rec& rc : rec_graph)
            if (rc.a) {
                ev_pool.push_back(rc.a);
                ev_pool.push_back(rc.b);
            }
        rec_graph.clear();
    }

    // ---------------------------------------------------------------- launches
    int mat_class(const Part& p, const DMat& M0) const {
        const DMat& M = M0.origin ? *M0.origin : M0;
        if (&M == &p.lv[0].A) return AMG_PROF_A0_PASS;
        for (const auto& L : p.lv)
            if (&M == &L.A) return AMG_PROF_A_COARSE;
        return AMG_PROF_TRANSFER;
    }
    template <int U, bool PIPE, bool F32, class Op>
    void rows_sell(const Sell& M, const Op& op, const int32_t* gate, const Red& red, bool stream_loads) {
        const int g = (int)std::max<int64_t>(
            1, std::min<int64_t>((M.nrows + kBlock - 1) / kBlock, (int64_t)num_sms * minb_of<Op>(PIPE ? 4 : 6)));
        if (stream_loads)
            klaunch(sell_rows<U, true, PIPE, Op, F32>, g, kBlock, 0, M, op, gate, red);
        else
            klaunch(sell_rows<U, false, PIPE, Op, F32>, g, kBlock, 0, M, op, gate, red);
    }
    template <int G, bool F32, class Op>
    void rows_csr(const CsrDev& M, const Op& op, const int32_t* gate, const Red& red, bool stream_loads) {
        const int g = (int)std::max<int64_t>(1, std::min<int64_t>(M.nblocks, (int64_t)num_sms * 8));
        if (stream_loads)
            klaunch(csr_rows<G, true, Op, F32>, g, kBlock, 0, M, op, gate, red);
        else
            klaunch(csr_rows<G, false, Op, F32>, g, kBlock, 0, M, op, gate, red);
    }
    template <int T, bool STREAM, bool F32, class Op>
    void rows_tma_impl(const SellTma& M, const Op& op, const int32_t* gate, const Red& red) {
        auto kern = sell_tma<T, STREAM, Op, F32>;
        const bool vix = !F32 && M.vi8 != nullptr;
        const size_t smem =
            (vix ? kVTabBytes : 0) + (size_t)kTmaStages * M.tile_ent * (vix ? 5 : F32 ? 8 : 12) + 2 * kTmaStages * 8;
        static size_t configured = 0;  // per instantiation
        if (smem > configured) {
            ck(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "smem attr");
            configured = smem;
        }
        const int g =
            (int)std::max<int64_t>(1, std::min<int64_t>(M.ntiles, (int64_t)num_sms * minb_of<Op>(kTmaBlocksPerSM)));
        klaunch(kern, g, kTmaThreads, smem, M, op, gate, red);
    }
    template <int T, bool F32, class Op>
    void rows_tma(const SellTma& M, const Op& op, const int32_t* gate, const Red& red, bool stream_loads) {
        if (stream_loads)
            rows_tma_impl<T, true, F32>(M, op, gate, red);
        else
            rows_tma_impl<T, false, F32>(M, op, gate, red);
    }
    int tcsr_un = [] {
        const char* e = std::getenv("AMGB_TCSR_UN");
        return e && e[0] == '8' ? 8 : 4;
    }();
    template <bool STREAM, bool F32, class Op>
    void rows_tcsr_impl(const CsrTma& M, const Op& op, const int32_t* gate, const Red& red) {
        if (tcsr_un == 8)
            rows_tcsr_un<STREAM, F32, 8>(M, op, gate, red);
        else
            rows_tcsr_un<STREAM, F32, 4>(M, op, gate, red);
    }
    template <bool STREAM, bool F32, int UN1, class Op>
    void rows_tcsr_un(const CsrTma& M, const Op& op, const int32_t* gate, const Red& red) {
        auto kern = csr_tma<STREAM, Op, F32, UN1>;
        CsrTma m = M;
        const int vbytes = F32 ? 4 : M.vi8 ? 1 : M.vi16 ? 2 : 8;
        m.vtab_bytes = (!F32 && (M.vi8 || M.vi16)) ? (int32_t)tcsr_vtab_bytes(M.ntab) : 0;
        m.smem_stage = (int32_t)tcsr_stage_bytes(M.tile_ent, vbytes);
        const size_t smem = (size_t)m.vtab_bytes + (size_t)kTmaStages * m.smem_stage + 2 * kTmaStages * 8;
        static size_t configured = 0;  // per instantiation
        if (smem > configured) {
            ck(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "smem attr");
            configured = smem;
        }
        // resident CTAs per SM: shared memory (228 KB per SM) and the launch bounds
        const int per_sm = (int)std::max<size_t>(1, std::min<size_t>(minb_of<Op>(4), (228 * 1024) / (smem + 1024)));
        const int g = (int)std::max<int64_t>(1, std::min<int64_t>(M.ntiles, (int64_t)num_sms * per_sm));
        klaunch(kern, g, kTmaThreads, smem, m, op, gate, red);
    }
    template <bool F32, class Op>
    void rows_tcsr(const CsrTma& M, const Op& op, const int32_t* gate, const Red& red, bool stream_loads) {
        if (stream_loads)
            rows_tcsr_impl<true, F32>(M, op, gate, red);
        else
            rows_tcsr_impl<false, F32>(M, op, gate, red);
    }
        // a part with no rows contributes zeros to an all-reduce
    void zero_defer(Part& p, const Red* r = nullptr) {
        const Red& red = r ? *r : p.red;
        if (red.defer) ck(cudaMemsetAsync(red.defer, 0, 4 * sizeof(double), stream), "memset");
    }
    // One pass over matrix M of part p with the fused epilogue op; F32: read the
    // fp32 copy of the matrix values (mixed-precision V-cycle).
    template <bool F32, class Op>
    void rows_impl(Part& p, const DMat& M, const Op& op, const int32_t* gate, const char* what,
                   const Red* red_slot = nullptr) {
        if (M.nrows == 0) {
            if constexpr (Op::NDOT > 0) zero_defer(p, red_slot);
            return;
        }
        // matrices too big for L2 stream their entries (evict-first); the rest
        // keep them cached so coarse levels stay L2-resident across cycles
        const bool big = M.nnz * 12 > stream_bytes;
        const DMat& Mo = M.origin ? *M.origin : M;  // a view accounts a share of its matrix's pass
        const double bytes = M.bytes_scale * (Mo.mat_bytes(F32) + Mo.ptr_bytes() + 8.0 * Mo.ncols * Op::GATHER +
                                              8.0 * Mo.nrows * Op::ROWV);
        const Red& red = red_slot ? *red_slot : p.red;
        launch(mat_class(p, M), bytes, what, [&] {
            if (M.fmt == Fmt::TMA) {  // T = 1 lane per row (narrow rows only, pick_format)
                rows_tma<1, F32>(M.tma, op, gate, red, big);
            } else if (M.fmt == Fmt::TMACSR) {
                rows_tcsr<F32>(M.tcsr, op, gate, red, big);
            } else if (M.fmt == Fmt::CSR) {
                switch (M.csr.G) {
                    case 1: rows_csr<1, F32>(M.csr, op, gate, red, big); break;
                    case 2: rows_csr<2, F32>(M.csr, op, gate, red, big); break;
                    case 4: rows_csr<4, F32>(M.csr, op, gate, red, big); break;
                    case 8: rows_csr<8, F32>(M.csr, op, gate, red, big); break;
                    default: rows_csr<16, F32>(M.csr, op, gate, red, big); break;
                }
            } else {
                rows_sell<8, true, F32>(M.sell, op, gate, red, big);
            }
        });
    }
    // A distributed pass split around the halo exchange: the
    // interior rows run while the exchange started by exchange() is in flight
    // on comm_stream, the boundary rows after it; fused dots of the (up to 3)
    // launches are folded in a fixed order before the all-reduce.
    template <bool F32, class Op>
    void rows_split(Part& p, const DMat& M, const Op& op, const int32_t* gate, const char* what) {
        Red slot[3] = {p.red, p.red, p.red};
        for (int q = 0; q < 3; ++q)
            if (p.red.defer) slot[q].defer = p.red.defer + q * kSlot;
        unsigned mask = 0;
        bool acct = false;  // the first launch carries the pass's bytes
        if (M.ib1 > M.ib0) {
            in_interior = true;
            rows_impl<F32>(p, M.view(M.ib0, M.ib1, 1.0), op, gate, what, &slot[0]);
            in_interior = false;
            mask |= 1;
            acct = true;
        }
        halo_wait();
        if (M.ib0 > 0) {
            rows_impl<F32>(p, M.view(0, M.ib0, acct ? 0.0 : 1.0), op, gate, what, &slot[1]);
            mask |= 2;
            acct = true;
        }
        if (M.ib1 < M.nrows) {
            rows_impl<F32>(p, M.view(M.ib1, M.nrows, acct ? 0.0 : 1.0), op, gate, what, &slot[2]);
            mask |= 4;
        }
        if constexpr (Op::NDOT > 0)
            launch(AMG_PROF_VECTOR, 0, "fold split dots",
                   [&] { sum_slots_kernel<<<1, 32, 0, stream>>>(p.red.defer, Op::NDOT, mask); });
    }
    template <bool F32, class Op>
    void rows_any(Part& p, const DMat& M, const Op& op, const int32_t* gate, const char* what) {
        if (M.split && distributed() && M.nrows > 0) {
            rows_split<F32>(p, M, op, gate, what);
        } else {
            halo_wait();
            rows_impl<F32>(p, M, op, gate, what);
        }
    }
    template <class Op>
    void rows(Part& p, const DMat& M, const Op& op, const int32_t* gate, const char* what) {
        rows_any<false>(p, M, op, gate, what);
    }
    // V-cycle passes: fp32 hierarchy values when prm.precision == 1
    template <class Op>
    void vrows(Part& p, const DMat& M, const Op& op, const int32_t* gate, const char* what) {
        if (prm.precision == 1)
            rows_any<true>(p, M, op, gate, what);
        else
            rows_any<false>(p, M, op, gate, what);
    }
    // ---- halo exchange in flight on comm_stream (distributed handles)
    cudaStream_t comm_stream = nullptr;
    cudaEvent_t ev_pack = nullptr, ev_halo = nullptr;
    bool halo_pending = false;
    bool in_interior = false;
    void halo_wait() {
        if (!halo_pending) return;
        ck(cudaStreamWaitEvent(stream, ev_halo, 0), "wait halo");
        halo_pending = false;
    }
    // Host synchronisation.  On an NCCL rank a peer that died or stalls would
    // block cudaStreamSynchronize forever; instead poll the stream and the
    // communicator's asynchronous error, and after nccl_timeout_s() without
    // progress abort the communicator (in-flight NCCL kernels exit) and throw
    // AMG_E_NCCL.  The handle is unusable afterwards.
    bool nccl_dead = false;
    double nccl_timeout = 300.0;
    void nccl_fail(const std::string& why) {
        Nccl& nc = Nccl::get();
        if (nccl && nc.commAbort && !nccl_dead) nc.commAbort(nccl);
        nccl_dead = true;
        nccl = nullptr;
        throw CudaError{"NCCL: " + why + " (communicator aborted; destroy the handle)", AMG_E_NCCL};
    }
    void sync(cudaStream_t s) {
        if (nccl_dead) throw CudaError{"NCCL communicator was aborted earlier", AMG_E_NCCL};
        if (!nccl) {
            ck(cudaStreamSynchronize(s), "sync");
            return;
        }
        Nccl& nc = Nccl::get();
        const auto t0 = std::chrono::steady_clock::now();
        for (int spin = 0;; ++spin) {
            const cudaError_t q = cudaStreamQuery(s);
            if (q == cudaSuccess) break;
            if (q != cudaErrorNotReady) ck(q, "sync");
            if (nc.commGetAsyncError && (spin & 255) == 255) {
                int ae = 0;
                nc.commGetAsyncError(nccl, &ae);
                if (ae != 0 && ae != kNcclInProgress)
                    nccl_fail("asynchronous error " + std::to_string(ae) +
                              (nc.getErrorString ? std::string(" ") + nc.getErrorString(ae) : std::string()));
            }
            if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > nccl_timeout)
                nccl_fail("no progress for " + std::to_string((int)nccl_timeout) + " s (a peer rank died or stalled)");
            // busy-poll (a sleep would add its wake-up slack to every iteration's
            // host round trip); back off only once the wait is long
            if (spin > 20000) std::this_thread::sleep_for(std::chrono::microseconds(100));
        }
    }
    // test transport: personalised all-to-all of host bytes (errors -> AMG_E_NCCL)
    void shm_a2a(const std::vector<std::vector<uint8_t>>& out, std::vector<std::vector<uint8_t>>& in) {
        try {
            shm->alltoallv(out, in);
        } catch (const std::exception& e) {
            throw CudaError{e.what(), AMG_E_NCCL};
        }
    }
    template <class T>
    static std::vector<uint8_t> bytes_of(const T* p, int64_t n) {
        const auto* b = reinterpret_cast<const uint8_t*>(p);
        return std::vector<uint8_t>(b, b + n * sizeof(T));
    }
    std::vector<uint8_t> d2h_bytes(const double* d, int64_t n) {
        std::vector<uint8_t> v(n * sizeof(double));
        if (n) ck(cudaMemcpy(v.data(), d, n * sizeof(double), cudaMemcpyDeviceToHost), "D2H (shm)");
        return v;
    }
    template <class Op>
    void vec(Part& p, int64_t n, const Op& op, const int32_t* gate, const char* what) {
        if (n == 0) {
            if constexpr (Op::NDOT > 0) zero_defer(p);
            return;
        }
        launch(AMG_PROF_VECTOR, 8.0 * n * Op::STREAMS, what,
               [&] { klaunch(vec_kernel<Op>, grid_for(n), kBlock, 0, n, op, gate, p.red); });
    }

    // ------------------------------------------------------------ collectives
    using Sel = std::function<double*(Part&)>;
    using CSel = std::function<const double*(Part&)>;
    using GSel = std::function<const int32_t*(Part&)>;

    // Halo exchange of the level-l vector sel(part): pack, then NCCL
    // send/recv (one part per process) or device copies between parts.
    void exchange(int l, const Sel& sel) {
        if (!distributed() || parts[0].lv[l].replicated) return;
        if (trace) {
            std::fprintf(stderr, "[amgb] exchange level %d\n", l);
            std::fflush(stderr);
        }
        for (Part& p : parts) {
            DevLevel& L = p.lv[l];
            if (L.nsend == 0) continue;
            double* v = sel(p);
            launch(AMG_PROF_VECTOR, 12.0 * L.nsend, "halo pack", [&] {
                pack_kernel<<<grid_for(L.nsend), kBlock, 0, stream>>>(L.send_idx, v, L.sendbuf, L.nsend);
            });
        }
        halo_wait();
        // the transfers run on comm_stream, after everything issued so far on
        // the work stream; the next split pass overlaps its interior rows
        ck(cudaEventRecord(ev_pack, stream), "record pack");
        ck(cudaStreamWaitEvent(comm_stream, ev_pack, 0), "wait pack");
        if (virt) {
            for (Part& p : parts) {
                DevLevel& L = p.lv[l];
                double* dst = sel(p) + L.n;
                for (size_t k = 0; k < L.plan.recv_peer.size(); ++k) {
                    const int q = L.plan.recv_peer[k];
                    const DevLevel& Q = parts[q].lv[l];
                    int64_t soff = -1;
                    for (size_t j = 0; j < Q.plan.send_peer.size(); ++j)
                        if (Q.plan.send_peer[j] == p.rank) soff = Q.plan.send_off[j];
                    if (soff < 0) throw CudaError{"halo plan mismatch"};
                    ck(cudaMemcpyAsync(dst + L.plan.recv_off[k], Q.sendbuf + soff, L.plan.recv_cnt[k] * sizeof(double),
                                       cudaMemcpyDeviceToDevice, comm_stream),
                       "halo copy");
                }
            }
        } else if (shm) {  // test transport: synchronous, through host shared memory
            Part& p = parts[0];
            DevLevel& L = p.lv[l];
            double* dst = sel(p) + L.n;
            sync(stream);
            std::vector<std::vector<uint8_t>> out(nranks), in;
            for (size_t j = 0; j < L.plan.send_peer.size(); ++j)
                out[L.plan.send_peer[j]] = d2h_bytes(L.sendbuf + L.plan.send_off[j], L.plan.send_cnt[j]);
            shm_a2a(out, in);
            for (size_t k = 0; k < L.plan.recv_peer.size(); ++k) {
                const auto& b = in[L.plan.recv_peer[k]];
                if ((int64_t)b.size() != L.plan.recv_cnt[k] * 8) throw CudaError{"shm halo: size mismatch", AMG_E_NCCL};
                if (!b.empty())
                    ck(cudaMemcpy(dst + L.plan.recv_off[k], b.data(), b.size(), cudaMemcpyHostToDevice), "H2D (shm)");
            }
            return;  // nothing pending
        } else {
            Nccl& nc = Nccl::get();
            Part& p = parts[0];
            DevLevel& L = p.lv[l];
            double* dst = sel(p) + L.n;
            ckn(nc.groupStart(), "ncclGroupStart");
            for (size_t j = 0; j < L.plan.send_peer.size(); ++j)
                ckn(nc.send(L.sendbuf + L.plan.send_off[j], L.plan.send_cnt[j], kNcclDouble, L.plan.send_peer[j], nccl,
                            comm_stream),
                    "ncclSend");
            for (size_t k = 0; k < L.plan.recv_peer.size(); ++k)
                ckn(nc.recv(dst + L.plan.recv_off[k], L.plan.recv_cnt[k], kNcclDouble, L.plan.recv_peer[k], nccl,
                            comm_stream),
                    "ncclRecv");
            ckn(nc.groupEnd(), "ncclGroupEnd");
        }
        ck(cudaEventRecord(ev_halo, comm_stream), "record halo");
        halo_pending = true;
    }
    // After a fused dot on a distributed handle: all-reduce the deferred
    // totals, then finalize on every part.
    template <class MakeFin>
    void allreduce_fin(int nv, const MakeFin& make_fin, const GSel& gate) {
        if (!distributed()) return;
        halo_wait();
        if (virt) {
            launch(AMG_PROF_VECTOR, 0, "allreduce (virtual)",
                   [&] { sum_parts_kernel<<<1, 32, 0, stream>>>(d_defer_ptrs, (int)parts.size(), nv); });
        } else if (shm) {  // test transport: every rank sums the totals in rank order
            Part& p = parts[0];
            sync(stream);
            std::vector<std::vector<uint8_t>> out(nranks, d2h_bytes(p.red.defer, nv)), in;
            shm_a2a(out, in);
            std::vector<double> tot(nv, 0.0);
            for (int r = 0; r < nranks; ++r)
                for (int k = 0; k < nv; ++k) tot[k] += reinterpret_cast<const double*>(in[r].data())[k];
            ck(cudaMemcpy(p.red.defer, tot.data(), nv * sizeof(double), cudaMemcpyHostToDevice), "H2D (shm)");
        } else {
            Part& p = parts[0];
            ckn(Nccl::get().allReduce(p.red.defer, p.red.defer, nv, kNcclDouble, kNcclSum, nccl, stream),
                "ncclAllReduce");
        }
        for (Part& p : parts) {
            auto fin = make_fin(p);
            const int32_t* g = gate(p);
            launch(AMG_PROF_VECTOR, 0, "finalize", [&] { fin_kernel<<<1, 1, 0, stream>>>(fin, p.red.defer, g); });
        }
    }
    // Level l_rep (first replicated level): every part wrote its slice of the
    // full vector sel(part); gather the other ranks' slices.
    void allgather_slices(int l_rep, const Sel& sel) {
        if (!distributed()) return;
        halo_wait();
        if (l_rep >= (int)starts.size()) throw CudaError{"allgather_slices: level without a partition"};
        const std::vector<int64_t>& st = starts[l_rep];
        if (virt) {
            for (Part& p : parts)
                for (Part& q : parts) {
                    if (q.rank == p.rank) continue;
                    const int64_t a = st[q.rank], b = st[q.rank + 1];
                    if (b > a)
                        ck(cudaMemcpyAsync(sel(p) + a, sel(q) + a, (b - a) * sizeof(double), cudaMemcpyDeviceToDevice,
                                           stream),
                           "allgather copy");
                }
        } else if (shm) {  // test transport: every rank sends its slice to every rank
            double* buf = sel(parts[0]);
            const int me = parts[0].rank;
            sync(stream);
            std::vector<std::vector<uint8_t>> out(nranks, d2h_bytes(buf + st[me], st[me + 1] - st[me])), in;
            shm_a2a(out, in);
            for (int q = 0; q < nranks; ++q)
                if (q != me && !in[q].empty())
                    ck(cudaMemcpy(buf + st[q], in[q].data(), in[q].size(), cudaMemcpyHostToDevice), "H2D (shm)");
        } else {
            Nccl& nc = Nccl::get();
            double* buf = sel(parts[0]);
            ckn(nc.groupStart(), "ncclGroupStart");
            for (int q = 0; q < nranks; ++q) {
                const int64_t a = st[q], b = st[q + 1];
                if (b > a) ckn(nc.broadcast(buf + a, buf + a, b - a, kNcclDouble, q, nccl, stream), "ncclBroadcast");
            }
            ckn(nc.groupEnd(), "ncclGroupEnd");
        }
    }

    bool vcycle(int l, const CSel& f, const Sel& out, const GSel& gate, bool with_rho);
    // fused CG: the level-0 res0 of the next V-cycle also applies r -= alpha q
    const double* fuse_r_old = nullptr;
    double* fuse_r_new = nullptr;
    bool cg_fused = false;
    bool mf0 = false;  // the unfused CG keeps m o r in lv[0].mf (VCgUpdateMF)
    void cg_iteration_fused(int parity);
    template <int K>
    void ensure_batch();
    template <int K>
    bool vcycle_b(int l, const double* f, double* out, const int32_t* gate, bool with_rho);
    template <int K>
    void cg_iteration_b(int parity);
    template <int K>
    amg_status solve_batched(int k, const double* F, int64_t ldf, double* X, int64_t ldx, double tol, int32_t maxiter,
                             int32_t* iters, double* rel);
    void cg_iteration(int parity);
    void gmres_step(int j);
    void gmres_cycle_end(const double* f, double* x);
    amg_status solve_gmres(const double* f, double* x, double tol, int32_t maxiter, int32_t* iters, double* rel);
    template <int S>
    void idr_cycle(double* x);
    template <int S>
    amg_status solve_idrs_t(const double* f, double* x, double tol, int32_t maxiter, int32_t* iters, double* rel);
    amg_status solve_idrs(const double* f, double* x, double tol, int32_t maxiter, int32_t* iters, double* rel);
    amg_status solve_dispatch(const double* f, double* x, double tol, int32_t maxiter, int32_t* iters, double* rel);
    amg_status solve_api(const double* f, double* x, double tol, int32_t maxiter, int32_t* iters, double* rel);
    void perm_in(const double* src, double* dst, int l = 0) {  // natural -> stored order (level l)
        const int64_t n = parts[0].lv[l].n;
        perm_to_kernel<<<grid_for(n), kBlock, 0, stream>>>(n, dq[l], src, dst);
    }
    void perm_out(const double* src, double* dst, int l = 0) {
        const int64_t n = parts[0].lv[l].n;
        perm_from_kernel<<<grid_for(n), kBlock, 0, stream>>>(n, dq[l], src, dst);
    }
    void bicgstab_iteration();
    amg_status solve(const double* f, double* x, double tol, int32_t maxiter, int32_t* iters, double* rel);
    void precond(const double* r, double* z);
};

// Algorithm 2 on level l for every part: out = V(f) from
// x = 0.  If with_rho, the last kernel also computes rho = (f, out) (CG,
// FinRho).  Returns true if the dot was fused.
bool Handle::vcycle(int l, const CSel& fsel, const Sel& osel, const GSel& gate, bool with_rho) {
    const int nlev = (int)parts[0].lv.size();
    if (l == nlev - 1) {  // coarsest: out = A_L^-1 f, replicated
        for (Part& p : parts) {
            DevLevel& L = p.lv[l];
            const int64_t warps = std::min<int64_t>(L.n, (int64_t)num_sms * 64);
            const int g = (int)std::max<int64_t>(1, (warps * 32 + kBlock - 1) / kBlock);
            const double* f = fsel(p);
            double* out = osel(p);
            const int32_t* gt = gate(p);
            launch(AMG_PROF_COARSE_SOLVE, 8.0 * L.n * L.n + 16.0 * L.n, "coarse gemv",
                   [&] { klaunch(dense_gemv, g, kBlock, 0, L.n, (const double*)p.coarse_inv, f, out, gt); });
        }
        return false;
    }
    const int npre = prm.npre, npost = prm.npost;
    const bool cheb = prm.relax == 2;
    const int K = prm.cheb_degree;
    const bool next_rep = parts[0].lv[l].next_replicated;
    // ping-pong buffers per part
    std::vector<double*> X(parts.size()), Y(parts.size());
    for (size_t i = 0; i < parts.size(); ++i) {
        X[i] = parts[i].lv[l].x;
        Y[i] = parts[i].lv[l].y;
    }
    Sel xsel = [&](Part& p) { return X[&p - &parts[0]]; };
    auto for_parts = [&](const std::function<void(Part&, size_t)>& fn) {
        for (size_t i = 0; i < parts.size(); ++i) fn(parts[i], i);
    };
    auto swap_xy = [&] {
        for (size_t i = 0; i < parts.size(); ++i) std::swap(X[i], Y[i]);
    };

    // m o f of this level was produced by the restriction above (levels >= 1,
    // SPAI-0/Jacobi, npre = 1): the zero-start residual gathers it instead of
    // m and f, the prolongation reads it instead of m and f
    const bool have_mf = parts[0].lv[l].mf != nullptr && (l > 0 || mf0);
    // the right-hand side of a distributed level is gathered by the first pass
    if (have_mf)
        exchange(l, [&](Part& p) { return p.lv[l].mf; });
    else
        exchange(l, [&](Part& p) { return const_cast<double*>(fsel(p)); });

    // ---- pre-smoothing from x = 0 and residual t = f - A x
    bool x_is_mf = false;  // x == m o f implicitly (not materialised)
    if (!cheb) {
        if (npre == 1) {
            x_is_mf = true;  // fused: t = f - A (m o f)
            for_parts([&](Part& p, size_t) {
                DevLevel& L = p.lv[l];
                if (l == 0 && fuse_r_new)  // + the previous CG iteration's r -= alpha q
                    vrows(p, L.A,
                          OpRes0Upd<FinRes0Upd>{L.m, fuse_r_old, p.q, fuse_r_new, L.t, p.ks, 0.0, FinRes0Upd{p.ks}},
                          gate(p), "res0 + r update");
                else if (have_mf)
                    vrows(p, L.A, OpRes0MF{L.mf, fsel(p), L.t, {}}, gate(p), "res0 (mf)");
                else
                    vrows(p, L.A, OpRes0{L.m, fsel(p), L.t, {}}, gate(p), "res0");
            });
        } else {
            for_parts([&](Part& p, size_t i) {
                DevLevel& L = p.lv[l];
                if (npre == 0)
                    ck(cudaMemsetAsync(X[i], 0, (L.n + L.ng) * sizeof(double), stream), "memset");
                else
                    vec(p, L.n + L.ng, VMulDiag{L.m, fsel(p), X[i], {}}, gate(p), "x=mf");
            });
            for (int s = 1; s < npre; ++s) {
                exchange(l, xsel);
                for_parts([&](Part& p, size_t i) {
                    DevLevel& L = p.lv[l];
                    vrows(p, L.A, OpRelax<0, NoFin>{X[i], L.m, fsel(p), Y[i], {}}, gate(p), "relax");
                });
                swap_xy();
            }
            exchange(l, xsel);
            for_parts([&](Part& p, size_t i) {
                DevLevel& L = p.lv[l];
                vrows(p, L.A, OpResidual<0, NoFin>{X[i], fsel(p), L.t, {}}, gate(p), "residual");
            });
        }
    } else {
        for (int s = 0; s < npre; ++s) {
            for (int k = 0; k < K; ++k) {
                if (s == 0 && k == 0) {
                    for_parts([&](Part& p, size_t i) {
                        DevLevel& L = p.lv[l];
                        vec(p, L.n + L.ng, VCheb0{fsel(p), L.diag, L.p, X[i], L.cheb_alpha[0], prm.cheb_scaled, {}},
                            gate(p), "cheb0");
                    });
                } else {
                    exchange(l, xsel);
                    for_parts([&](Part& p, size_t i) {
                        DevLevel& L = p.lv[l];
                        vrows(p, L.A,
                             OpCheb<0, NoFin>{X[i], fsel(p), L.diag, L.p, Y[i], L.cheb_alpha[k], L.cheb_beta[k],
                                              prm.cheb_scaled, k == 0, {}},
                             gate(p), "cheb");
                    });
                    swap_xy();
                }
            }
        }
        if (npre == 0)
            for_parts([&](Part& p, size_t i) {
                ck(cudaMemsetAsync(X[i], 0, (p.lv[l].n + p.lv[l].ng) * sizeof(double), stream), "memset");
            });
        exchange(l, xsel);
        for_parts([&](Part& p, size_t i) {
            DevLevel& L = p.lv[l];
            vrows(p, L.A, OpResidual<0, NoFin>{X[i], fsel(p), L.t, {}}, gate(p), "residual");
        });
    }

    // ---- restriction f_c = R t, coarse solve, prolongation x += P x_c
    exchange(l, [&](Part& p) { return p.lv[l].t; });
    for_parts([&](Part& p, size_t) {
        DevLevel& L = p.lv[l];
        DevLevel& C = p.lv[l + 1];
        // into the next level's vector; a replicated next level receives the
        // slice [crow0, crow1) of the full vector
        const int64_t off = next_rep ? L.crow0 : 0;
        if (C.mf)
            vrows(p, L.R, OpSpmvMF{L.t, C.f + off, C.m + off, C.mf + off, {}}, gate(p), "restrict (+mf)");
        else
            vrows(p, L.R, OpSpmv{L.t, C.f + off}, gate(p), "restrict");
    });
    // entering the replicated levels: gather the other ranks' slices of f_{l+1}
    if (next_rep && !parts[0].lv[l].replicated) {
        allgather_slices(l + 1, [&](Part& p) { return p.lv[l + 1].f; });
        if (parts[0].lv[l + 1].mf) allgather_slices(l + 1, [&](Part& p) { return p.lv[l + 1].mf; });
    }
    vcycle(l + 1, [&](Part& p) { return (const double*)p.lv[l + 1].f; }, [&](Part& p) { return p.lv[l + 1].o; }, gate,
           false);
    exchange(l + 1, [&](Part& p) { return p.lv[l + 1].o; });
    for_parts([&](Part& p, size_t i) {
        DevLevel& L = p.lv[l];
        DevLevel& C = p.lv[l + 1];
        if (x_is_mf && have_mf)
            vrows(p, L.P, OpProl0MF{C.o, L.mf, X[i], {}}, gate(p), "prolong0 (mf)");
        else if (x_is_mf)
            vrows(p, L.P, OpProl0{C.o, L.m, fsel(p), X[i], {}}, gate(p), "prolong0");
        else
            vrows(p, L.P, OpProlAdd{C.o, X[i], {}}, gate(p), "prolong");
    });

    // ---- post-smoothing; the last sweep writes `out`
    if (npost == 0) {
        for_parts([&](Part& p, size_t i) {
            ck(cudaMemcpyAsync(osel(p), X[i], p.lv[l].n * sizeof(double), cudaMemcpyDeviceToDevice, stream), "copy");
        });
        return false;
    }
    const int sweeps = cheb ? npost * K : npost;
    for (int s = 0; s < sweeps; ++s) {
        const bool last = s == sweeps - 1;
        exchange(l, xsel);
        for_parts([&](Part& p, size_t i) {
            DevLevel& L = p.lv[l];
            double* dst = last ? osel(p) : Y[i];
            if (!cheb) {
                if (last && with_rho)
                    vrows(p, L.A, OpRelax<1, FinRho>{X[i], L.m, fsel(p), dst, FinRho{p.ks}}, gate(p), "relax+dot");
                else
                    vrows(p, L.A, OpRelax<0, NoFin>{X[i], L.m, fsel(p), dst, {}}, gate(p), "relax");
            } else {
                const int k = s % K;
                if (last && with_rho)
                    vrows(p, L.A,
                         OpCheb<1, FinRho>{X[i], fsel(p), L.diag, L.p, dst, L.cheb_alpha[k], L.cheb_beta[k],
                                           prm.cheb_scaled, k == 0, FinRho{p.ks}},
                         gate(p), "cheb+dot");
                else
                    vrows(p, L.A,
                         OpCheb<0, NoFin>{X[i], fsel(p), L.diag, L.p, dst, L.cheb_alpha[k], L.cheb_beta[k],
                                          prm.cheb_scaled, k == 0, {}},
                         gate(p), "cheb");
            }
        });
        if (!last) swap_xy();
    }
    if (with_rho) allreduce_fin(1, [](Part& p) { return FinRho{p.ks}; }, gate);
    return with_rho;
}

// One CG iteration (§8c c-1): z = M r, rho = (r, z) [fused in the last V-cycle
// kernel]; p' = z + beta p, q = A p', sigma = (p', q) [one kernel];
// x += alpha p', r -= alpha q, (r, r) [one kernel].
void Handle::cg_iteration(int parity) {
    GSel gate = [](Part& p) { return (const int32_t*)&p.ks->done; };
    auto pold = [parity](Part& p) { return parity ? p.pb : p.pa; };
    auto pnew = [parity](Part& p) { return parity ? p.pa : p.pb; };
    if (!vcycle(0, [](Part& p) { return (const double*)p.r; }, [](Part& p) { return p.z; }, gate, true)) {
        for (Part& p : parts) vec(p, p.lv[0].n, VDot<FinRho>{p.r, p.z, FinRho{p.ks}}, gate(p), "dot(r,z)");
        allreduce_fin(1, [](Part& p) { return FinRho{p.ks}; }, gate);
    }
    exchange(0, [](Part& p) { return p.z; });
    if (distributed())  // ghost entries of p' = z + beta p, formed redundantly
        for (Part& p : parts) {
            DevLevel& L = p.lv[0];
            if (L.ng == 0) continue;
            const int32_t* g = gate(p);
            double *zg = p.z + L.n, *pog = pold(p) + L.n, *png = pnew(p) + L.n;
            launch(AMG_PROF_VECTOR, 24.0 * L.ng, "ghost dir", [&] {
                ghost_dir_kernel<<<grid_for(L.ng), kBlock, 0, stream>>>(zg, pog, png, L.ng, p.ks, g);
            });
        }
    for (Part& p : parts)
        rows(p, p.lv[0].A, OpCgDir<FinSigma>{p.z, pold(p), pnew(p), p.q, p.ks, 0.0, FinSigma{p.ks}}, gate(p), "cg dir");
    allreduce_fin(1, [](Part& p) { return FinSigma{p.ks}; }, gate);
    for (Part& p : parts)
        if (mf0)
            vec(p, p.lv[0].n,
                VCgUpdateMF{p.xcur, p.r, pnew(p), p.q, p.lv[0].m, p.lv[0].mf, p.ks, 0.0, FinCgUpdate{p.ks}}, gate(p),
                "cg update (+mf)");
        else
            vec(p, p.lv[0].n, VCgUpdate{p.xcur, p.r, pnew(p), p.q, p.ks, 0.0, FinCgUpdate{p.ks}}, gate(p), "cg update");
    allreduce_fin(1, [](Part& p) { return FinCgUpdate{p.ks}; }, gate);
}

// Fused CG iteration k (single part, SPAI-0/Jacobi, npre = 1, >= 2 levels):
// the same arithmetic as cg_iteration with iteration k-1's r update moved
// into this V-cycle's first kernel and its x update into this CG direction
// kernel (one kernel and 16n bytes less per iteration).
void Handle::cg_iteration_fused(int parity) {
    Part& p = parts[0];
    GSel gate = [](Part& q) { return (const int32_t*)&q.ks->done; };
    double* r_old = parity ? p.r2 : p.r;
    double* r_new = parity ? p.r : p.r2;
    double* pold = parity ? p.pb : p.pa;
    double* pnew = parity ? p.pa : p.pb;
    fuse_r_old = r_old;
    fuse_r_new = r_new;
    vcycle(0, [r_new](Part&) { return (const double*)r_new; }, [](Part& q) { return q.z; }, gate, true);
    fuse_r_old = nullptr;
    fuse_r_new = nullptr;
    rows(p, p.lv[0].A, OpCgDirX<FinSigmaX>{p.z, pold, pnew, p.q, p.xcur, p.ks, 0.0, 0.0, FinSigmaX{p.ks}},
         gate(p), "cg dir + x update");
}

// One BiCGStab iteration (§8c c-1).
void Handle::bicgstab_iteration() {
    GSel gate = [](Part& p) { return (const int32_t*)&p.ks->done; };
    GSel gate2 = [](Part& p) { return (const int32_t*)&p.ks->skip2; };
    for (Part& p : parts) vec(p, p.lv[0].n, VBiP{p.r, p.v, p.pa, p.ks, 0, 0, 0, {}}, gate(p), "bicg p");
    vcycle(0, [](Part& p) { return (const double*)p.pa; }, [](Part& p) { return p.ph; }, gate, false);
    exchange(0, [](Part& p) { return p.ph; });
    for (Part& p : parts)
        rows(p, p.lv[0].A, OpSpmvDot<1, FinBiAlpha>{p.ph, p.rhat, p.v, FinBiAlpha{p.ks}}, gate(p), "v=A ph");
    allreduce_fin(1, [](Part& p) { return FinBiAlpha{p.ks}; }, gate);
    for (Part& p : parts) vec(p, p.lv[0].n, VBiS{p.r, p.v, p.s, p.ks, 0.0, FinBiS{p.ks}}, gate(p), "bicg s");
    allreduce_fin(1, [](Part& p) { return FinBiS{p.ks}; }, gate);
    vcycle(0, [](Part& p) { return (const double*)p.s; }, [](Part& p) { return p.sh; }, gate2, false);
    exchange(0, [](Part& p) { return p.sh; });
    for (Part& p : parts)
        rows(p, p.lv[0].A, OpSpmvDot<2, FinBiOmega>{p.sh, p.s, p.tv, FinBiOmega{p.ks}}, gate2(p), "t=A sh");
    allreduce_fin(2, [](Part& p) { return FinBiOmega{p.ks}; }, gate2);
    for (Part& p : parts)
        vec(p, p.lv[0].n, VBiX{p.xcur, p.r, p.ph, p.sh, p.s, p.tv, p.rhat, p.ks, 0, 0, 0, FinBiX{p.ks}}, gate(p),
            "bicg x");
    allreduce_fin(2, [](Part& p) { return FinBiX{p.ks}; }, gate);
}

// f, x: device vectors.  Single part: length n.  Virtual parts: the GLOBAL
// vectors (each part works on its slice).  NCCL: this rank's slice.
amg_status Handle::solve(const double* f, double* x, double tol, int32_t maxiter, int32_t* iters, double* rel) {
    const bool bicg = prm.solver == 1;
    const bool dist = distributed();
    const int64_t launches0 = launches;
    collect(rec_direct, 0, true);  // discard launches issued outside a solve
    alg_bytes = 0;
    std::fill(acc_ms, acc_ms + 8, 0.0);
    std::fill(acc_bytes, acc_bytes + 8, 0.0);
    std::fill(acc_launches, acc_launches + 8, 0);
    cur_iter = -1;
    // Fused CG iteration (opt-in, AMGB_CG_FUSION=1): its first kernel gathers m,
    // r and q to save the 48 n-byte update kernel.  Measured (interleaved A/B,
    // DESIGN.md §6): no gain on 256^3 Poisson (42.1 vs 41.8 ms), a loss where
    // gathers are random (permuted 150^3: 29.7 vs 18.5 ms).
    const char* fz = std::getenv("AMGB_CG_FUSION");
    cg_fused = !bicg && !dist && prm.relax != 2 && prm.npre == 1 && parts[0].lv.size() >= 2 && fz && fz[0] == '1';
    // unfused CG: the update kernel also writes m o r for the level-0 residual
    mf0 = !bicg && !cg_fused && parts[0].lv[0].mf != nullptr && std::getenv("AMGB_NO_MF0") == nullptr;
    const int variant = (cg_fused ? 1 : 0) | (mf0 ? 2 : 0);
    struct FlagReset {  // precond / GMRES / level_op V-cycles never see mf0
        bool& f;
        ~FlagReset() { f = false; }
    } mf0_reset{mf0};
    GSel nogate = [](Part&) { return (const int32_t*)nullptr; };
    ck(cudaEventRecord(ev0, stream), "event");
    // right-hand side / solution slices of every part
    for (Part& p : parts) {
        const int64_t off = virt ? p.row0 : 0;
        p.fcur = f + off;
        if (!dist) {
            p.xcur = x;  // no ghosts: work on the caller's vector
        } else {
            p.xcur = p.xw;
            ck(cudaMemcpyAsync(p.xw, x + off, p.lv[0].n * sizeof(double), cudaMemcpyDeviceToDevice, stream), "x in");
        }
    }
    // scalars: maxiter in, everything else computed on the device
    std::memset(ks_host, 0, sizeof(KState));
    ks_host->maxiter = maxiter;
    for (Part& p : parts) ck(cudaMemcpyAsync(p.ks, ks_host, sizeof(KState), cudaMemcpyHostToDevice, stream), "ks init");
    for (Part& p : parts) vec(p, p.lv[0].n, VNorm2{p.fcur, FinNorm{p.ks, tol}}, nullptr, "norm f");
    allreduce_fin(1, [tol](Part& p) { return FinNorm{p.ks, tol}; }, nogate);
    exchange(0, [](Part& p) { return p.xcur; });
    for (Part& p : parts)
        rows(p, p.lv[0].A, OpResidual<1, FinInitRes>{p.xcur, p.fcur, p.r, FinInitRes{p.ks}}, nullptr, "r0");
    allreduce_fin(1, [](Part& p) { return FinInitRes{p.ks}; }, nogate);
    if (mf0)
        for (Part& p : parts)
            vec(p, p.lv[0].n, VMulDiag{p.lv[0].m, p.r, p.lv[0].mf, {}}, nullptr, "m o r0");
    for (Part& p : parts) {
        const int64_t n = p.lv[0].n + p.lv[0].ng;
        ck(cudaMemsetAsync(p.pa, 0, n * sizeof(double), stream), "memset");
        ck(cudaMemsetAsync(p.pb, 0, n * sizeof(double), stream), "memset");
        if (bicg) {
            ck(cudaMemcpyAsync(p.rhat, p.r, p.lv[0].n * sizeof(double), cudaMemcpyDeviceToDevice, stream), "copy");
            ck(cudaMemsetAsync(p.v, 0, p.lv[0].n * sizeof(double), stream), "memset");
        }
    }
    ck(cudaMemcpyAsync(ks_host, parts[0].ks, sizeof(KState), cudaMemcpyDeviceToHost, stream), "ks read");
    sync(stream);
    collect(rec_direct, 0, true);
    if (ks_host->nf == 0.0) {  // zero right-hand side: x = 0
        for (Part& p : parts)
            ck(cudaMemsetAsync(x + (virt ? p.row0 : 0), 0, p.lv[0].n * sizeof(double), stream), "memset");
        sync(stream);
        *iters = 0;
        *rel = 0.0;
        stats = amg_solve_stats{};
        stats.kernel_launches = launches - launches0;
        stats.alg_bytes = alg_bytes;
        return AMG_OK;
    }

    // Krylov loop: two iterations per host round trip, replayed from a CUDA
    // graph; kernels of iterations past convergence exit at their gate.
    const bool use_graph = prm.use_graph && !sync_debug && !shm;  // shm transport: host-synchronous
    auto two_iterations = [&] {
        for (int k = 0; k < 2; ++k) {
            cur_iter = k;
            if (bicg)
                bicgstab_iteration();
            else if (cg_fused)
                cg_iteration_fused(k);
            else
                cg_iteration(k);
        }
        cur_iter = -1;
    };
    // Device-side loop: one graph launch runs every remaining iteration (a
    // conditional WHILE node around two iterations + a loop-test kernel); the
    // host waits once.  Used for single-part handles without event profiling
    // (event nodes are not allowed inside conditional bodies).
    const bool use_loop = use_graph && !dist && prof_mask == 0 && std::getenv("AMGB_NO_DEVICE_LOOP") == nullptr;
    if (use_loop && !ks_host->done) {
        if (!graph || !graph_loop || graph_x != x || graph_variant != variant) {
            drop_graph();
            cudaGraph_t g;
            ck(cudaGraphCreate(&g, 0), "graph create");
            cudaGraphConditionalHandle cond;
            ck(cudaGraphConditionalHandleCreate(&cond, g, 1, cudaGraphCondAssignDefault), "cond handle");
            cudaGraphNodeParams cp = {};
            cp.type = cudaGraphNodeTypeConditional;
            cp.conditional.handle = cond;
            cp.conditional.type = cudaGraphCondTypeWhile;
            cp.conditional.size = 1;
            cudaGraphNode_t node;
            ck(cudaGraphAddNode(&node, g, nullptr, 0, &cp), "conditional node");
            cudaGraph_t body = cp.conditional.phGraph_out[0];
            const int64_t before = launches;
            ck(cudaStreamBeginCaptureToGraph(stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal),
               "capture body");
            capturing = true;
            try {
                two_iterations();
                launch(AMG_PROF_VECTOR, 0, "loop test",
                       [&] { set_loop_kernel<<<1, 1, 0, stream>>>(cond, &parts[0].ks->done); });
            } catch (...) {
                capturing = false;
                cudaGraph_t dummy;
                cudaStreamEndCapture(stream, &dummy);
                cudaGraphDestroy(g);
                throw;
            }
            capturing = false;
            cudaGraph_t body_out;
            ck(cudaStreamEndCapture(stream, &body_out), "end capture");
            graph_kernels = launches - before;
            launches = before;
            ck(cudaGraphInstantiate(&graph, g, 0), "instantiate loop graph");
            cudaGraphDestroy(g);
            graph_x = x;
            graph_prof_mask = 0;
            graph_loop = true;
            graph_variant = variant;
        }
        const int iter_before = ks_host->iter;
        ck(cudaGraphLaunch(graph, stream), "graph launch");
        ck(cudaMemcpyAsync(ks_host, parts[0].ks, sizeof(KState), cudaMemcpyDeviceToHost, stream), "ks read");
        sync(stream);
        // the body ran ceil(iters / 2) times; iteration 0 of a body ran that
        // often, iteration 1 one time less when the count is odd
        const int ran = ks_host->iter - iter_before + (ks_host->status ? 1 : 0);
        const int bodies = (ran + 1) / 2;
        launches += graph_kernels * bodies;
        for (int b = 0; b < bodies; ++b) collect(rec_graph, std::min(2, ran - 2 * b), false);
    }
    while (!ks_host->done) {
        const int iter_before = ks_host->iter;
        if (use_graph) {
            if (!graph || graph_loop || graph_x != x || graph_prof_mask != prof_mask || graph_variant != variant) {
                drop_graph();
                graph_loop = false;
                cudaGraph_t g;
                const int64_t before = launches;
                ck(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal), "capture");
                capturing = true;
                try {
                    two_iterations();
                } catch (...) {
                    capturing = false;
                    cudaStreamEndCapture(stream, &g);
                    throw;
                }
                capturing = false;
                halo_wait();  // the comm stream rejoins before the capture ends
                ck(cudaStreamEndCapture(stream, &g), "end capture");
                graph_kernels = launches - before;
                launches = before;
                ck(cudaGraphInstantiate(&graph, g, 0), "instantiate");
                cudaGraphDestroy(g);
                graph_x = x;
                graph_prof_mask = prof_mask;
                graph_variant = variant;
            }
            ck(cudaGraphLaunch(graph, stream), "graph launch");
            launches += graph_kernels;
        } else {
            two_iterations();
        }
        ck(cudaMemcpyAsync(ks_host, parts[0].ks, sizeof(KState), cudaMemcpyDeviceToHost, stream), "ks read");
        sync(stream);
        const int ran = ks_host->iter - iter_before + (ks_host->done && ks_host->status ? 1 : 0);
        collect(use_graph ? rec_graph : rec_direct, ran, !use_graph);
    }
    // fused CG: an r update already applied may still owe its x update
    if (cg_fused && ks_host->xpend) {
        Part& p = parts[0];
        const int last = ks_host->iter - 1;  // the iteration whose alpha, p are pending
        double* plast = (last % 2) ? p.pa : p.pb;
        vec(p, p.lv[0].n, VAxpyAlpha{p.xcur, plast, p.ks, 0.0, {}}, nullptr, "cg final x update");
    }
    // true residual |f - A x| / |f|
    exchange(0, [](Part& p) { return p.xcur; });
    for (Part& p : parts)
        rows(p, p.lv[0].A, OpResidual<1, FinTrueRes>{p.xcur, p.fcur, p.r, FinTrueRes{p.ks}}, nullptr, "true res");
    allreduce_fin(1, [](Part& p) { return FinTrueRes{p.ks}; }, nogate);
    if (dist)
        for (Part& p : parts)
            ck(cudaMemcpyAsync(x + (virt ? p.row0 : 0), p.xw, p.lv[0].n * sizeof(double), cudaMemcpyDeviceToDevice,
                               stream),
               "x out");
    ck(cudaEventRecord(ev1, stream), "event");
    ck(cudaMemcpyAsync(ks_host, parts[0].ks, sizeof(KState), cudaMemcpyDeviceToHost, stream), "ks read");
    sync(stream);
    collect(rec_direct, 0, true);
    *iters = ks_host->iter;
    *rel = ks_host->true_res / ks_host->nf;
    float ms = 0;
    cudaEventElapsedTime(&ms, ev0, ev1);
    stats = amg_solve_stats{};
    stats.iters = ks_host->iter;
    stats.vcycles = bicg ? 2 * ks_host->iter - (ks_host->half ? 1 : 0) : ks_host->iter;
    stats.status = ks_host->status;
    // bit 2: the caller's f or x is not 16-B aligned, so the paired 16-B vector
    // kernels (vec_kernel elem2) took their scalar loop on x
    stats.flags = (cg_fused ? 1 : 0) | ((((uintptr_t)f | (uintptr_t)x) & 15) ? 4 : 0);
    stats.kernel_launches = launches - launches0;
    stats.solve_ms = ms;
    stats.rel_resid = *rel;
    stats.alg_bytes = alg_bytes;
    for (int c = 0; c < 8; ++c) {
        stats.prof_ms[c] = acc_ms[c];
        stats.prof_bytes[c] = acc_bytes[c];
        stats.prof_launches[c] = acc_launches[c];
    }
    if (ks_host->status == AMG_BREAKDOWN) {
        g_err = bicg ? "BiCGStab breakdown" : "CG breakdown: (r, Mr) <= 0 or (p, Ap) <= 0";
        stats.status = AMG_BREAKDOWN;
        return AMG_BREAKDOWN;
    }
    const amg_status st = ks_host->res <= ks_host->tolnf ? AMG_OK : AMG_NOT_CONVERGED;
    stats.status = st;
    return st;
}

// ============================================================ batched solve
// K interleaved right-hand sides through one hierarchy pass (batched.cuh).
template <int K>
void Handle::ensure_batch() {
    if (batch.K == K) return;
    free_batch();
    batch.K = K;
    Part& p = parts[0];
    auto alloc = [&](int64_t n) {
        void* q = nullptr;
        ck(cudaMalloc(&q, std::max<int64_t>(n, 1) * K * sizeof(double)), "cudaMalloc (batch)");
        ck(cudaMemset(q, 0, std::max<int64_t>(n, 1) * K * sizeof(double)), "memset");
        batch.mem.push_back(q);
        return static_cast<double*>(q);
    };
    batch.lv.resize(p.lv.size());
    for (size_t l = 0; l < p.lv.size(); ++l) {
        const int64_t n = p.lv[l].n;
        BLevel& B = batch.lv[l];
        B.x = alloc(n);
        B.y = alloc(n);
        B.t = alloc(n);
        if (prm.relax == 2) B.p = alloc(n);
        if (l > 0) {
            B.f = alloc(n);
            B.o = alloc(n);
        }
    }
    const int64_t n0 = p.lv[0].n;
    batch.r = alloc(n0);
    batch.z = alloc(n0);
    batch.pa = alloc(n0);
    batch.pb = alloc(n0);
    batch.q = alloc(n0);
    batch.xw = alloc(n0);
    batch.fw = alloc(n0);
    void* q = nullptr;
    ck(cudaMalloc(&q, sizeof(KStateB)), "cudaMalloc");
    batch.mem.push_back(q);
    batch.ks = static_cast<KStateB*>(q);
    ck(cudaMallocHost(&batch.ks_host, sizeof(KStateB)), "cudaMallocHost");
}

// Algorithm 2 for K interleaved right-hand sides (single part).
template <int K>
bool Handle::vcycle_b(int l, const double* f, double* out, const int32_t* gate, bool with_rho) {
    Part& p = parts[0];
    const int nlev = (int)p.lv.size();
    DevLevel& L = p.lv[l];
    if (l == nlev - 1) {
        const int64_t warps = std::min<int64_t>(L.n, (int64_t)num_sms * 64);
        const int g = (int)std::max<int64_t>(1, (warps * 32 + kBlock - 1) / kBlock);
        launch(AMG_PROF_COARSE_SOLVE, 8.0 * L.n * L.n + 16.0 * K * L.n, "coarse gemm",
               [&] { dense_gemm_b<K><<<g, kBlock, 0, stream>>>(L.n, p.coarse_inv, f, out, gate); });
        return false;
    }
    BLevel& B = batch.lv[l];
    BLevel& Bc = batch.lv[l + 1];
    DevLevel& C = p.lv[l + 1];
    const bool cheb = prm.relax == 2;
    const int K_ = prm.cheb_degree;
    double* x = B.x;
    double* y = B.y;
    bool x_is_mf = false;
    if (!cheb) {
        if (prm.npre == 1) {
            x_is_mf = true;
            rows(p, L.A, OpRes0B<K>{L.m, f, B.t, {}}, gate, "res0 (batched)");
        } else {
            if (prm.npre == 0)
                ck(cudaMemsetAsync(x, 0, L.n * K * sizeof(double), stream), "memset");
            else
                vec(p, L.n, VMulDiagB<K>{L.m, f, x, {}}, gate, "x=mf (batched)");
            for (int s = 1; s < prm.npre; ++s) {
                rows(p, L.A, OpRelaxB<K, 0, NoFin>{x, L.m, f, y, {}}, gate, "relax (batched)");
                std::swap(x, y);
            }
            rows(p, L.A, OpResidualB<K, 0, NoFin>{x, f, B.t, {}}, gate, "residual (batched)");
        }
    } else {
        for (int s = 0; s < prm.npre; ++s)
            for (int k = 0; k < K_; ++k) {
                if (s == 0 && k == 0) {
                    vec(p, L.n, VCheb0B<K>{f, L.diag, B.p, x, L.cheb_alpha[0], prm.cheb_scaled, {}}, gate,
                        "cheb0 (batched)");
                } else {
                    rows(p, L.A,
                         OpChebB<K, 0, NoFin>{x, f, L.diag, B.p, y, L.cheb_alpha[k], L.cheb_beta[k], prm.cheb_scaled,
                                              k == 0, {}},
                         gate, "cheb (batched)");
                    std::swap(x, y);
                }
            }
        if (prm.npre == 0) ck(cudaMemsetAsync(x, 0, L.n * K * sizeof(double), stream), "memset");
        rows(p, L.A, OpResidualB<K, 0, NoFin>{x, f, B.t, {}}, gate, "residual (batched)");
    }
    rows(p, L.R, OpSpmvB<K>{B.t, Bc.f}, gate, "restrict (batched)");
    vcycle_b<K>(l + 1, Bc.f, Bc.o, gate, false);
    if (x_is_mf)
        rows(p, L.P, OpProl0B<K>{Bc.o, L.m, f, x, {}}, gate, "prolong0 (batched)");
    else
        rows(p, L.P, OpProlAddB<K>{Bc.o, x, {}}, gate, "prolong (batched)");
    (void)C;
    if (prm.npost == 0) {
        ck(cudaMemcpyAsync(out, x, L.n * K * sizeof(double), cudaMemcpyDeviceToDevice, stream), "copy");
        return false;
    }
    const int sweeps = cheb ? prm.npost * K_ : prm.npost;
    for (int s = 0; s < sweeps; ++s) {
        const bool last = s == sweeps - 1;
        double* dst = last ? out : y;
        if (!cheb) {
            if (last && with_rho)
                rows(p, L.A, OpRelaxB<K, 1, FinRhoB<K>>{x, L.m, f, dst, FinRhoB<K>{batch.ks}}, gate, "relax+dot (batched)");
            else
                rows(p, L.A, OpRelaxB<K, 0, NoFin>{x, L.m, f, dst, {}}, gate, "relax (batched)");
        } else {
            const int k = s % K_;
            if (last && with_rho)
                rows(p, L.A,
                     OpChebB<K, 1, FinRhoB<K>>{x, f, L.diag, B.p, dst, L.cheb_alpha[k], L.cheb_beta[k], prm.cheb_scaled,
                                               k == 0, FinRhoB<K>{batch.ks}},
                     gate, "cheb+dot (batched)");
            else
                rows(p, L.A,
                     OpChebB<K, 0, NoFin>{x, f, L.diag, B.p, dst, L.cheb_alpha[k], L.cheb_beta[k], prm.cheb_scaled,
                                          k == 0, {}},
                     gate, "cheb (batched)");
        }
        if (!last) std::swap(x, y);
    }
    return with_rho;
}

template <int K>
void Handle::cg_iteration_b(int parity) {
    Part& p = parts[0];
    const int32_t* gate = &batch.ks->done;
    double* pold = parity ? batch.pb : batch.pa;
    double* pnew = parity ? batch.pa : batch.pb;
    if (!vcycle_b<K>(0, batch.r, batch.z, gate, true))
        vec(p, p.lv[0].n, VDotB<K, FinRhoB<K>>{batch.r, batch.z, FinRhoB<K>{batch.ks}}, gate, "dot(r,z) (batched)");
    rows(p, p.lv[0].A,
         OpCgDirB<K, FinSigmaB<K>>{batch.z, pold, pnew, batch.q, batch.ks, {}, FinSigmaB<K>{batch.ks}}, gate,
         "cg dir (batched)");
    vec(p, p.lv[0].n, VCgUpdateB<K>{batch.xw, batch.r, pnew, batch.q, batch.ks, {}, FinCgUpdateB<K>{batch.ks}}, gate,
        "cg update (batched)");
}

template <int K>
amg_status Handle::solve_batched(int k, const double* F, int64_t ldf, double* X, int64_t ldx, double tol,
                                 int32_t maxiter, int32_t* iters, double* rel) {
    ensure_batch<K>();
    Part& p = parts[0];
    const int64_t n = p.lv[0].n;
    const int64_t launches0 = launches;
    collect(rec_direct, 0, true);
    alg_bytes = 0;
    std::fill(acc_ms, acc_ms + 8, 0.0);
    std::fill(acc_bytes, acc_bytes + 8, 0.0);
    std::fill(acc_launches, acc_launches + 8, 0);
    cur_iter = -1;
    ck(cudaEventRecord(ev0, stream), "event");
    KStateB* kh = batch.ks_host;
    std::memset(kh, 0, sizeof(KStateB));
    kh->k = k;
    kh->maxiter = maxiter;
    ck(cudaMemcpyAsync(batch.ks, kh, sizeof(KStateB), cudaMemcpyHostToDevice, stream), "ks init");
    launch(AMG_PROF_VECTOR, 8.0 * 2 * K * n, "pack F, X", [&] {
        pack_cols<K><<<grid_for(n), kBlock, 0, stream>>>(F, ldf, k, n, batch.fw, nullptr);
        pack_cols<K><<<grid_for(n), kBlock, 0, stream>>>(X, ldx, k, n, batch.xw, nullptr);
    });
    vec(p, n, VNorm2B<K, FinNormB<K>>{batch.fw, FinNormB<K>{batch.ks, tol}}, nullptr, "norm F");
    rows(p, p.lv[0].A, OpResidualB<K, 1, FinInitResB<K>>{batch.xw, batch.fw, batch.r, FinInitResB<K>{batch.ks}},
         nullptr, "r0 (batched)");
    ck(cudaMemsetAsync(batch.pa, 0, n * K * sizeof(double), stream), "memset");
    ck(cudaMemsetAsync(batch.pb, 0, n * K * sizeof(double), stream), "memset");
    ck(cudaMemcpyAsync(kh, batch.ks, sizeof(KStateB), cudaMemcpyDeviceToHost, stream), "ks read");
    sync(stream);
    collect(rec_direct, 0, true);
    // FinInitResB does not know which columns have f = 0: mark them done
    // (x = 0 for them) before iterating
    bool any_zero = false;
    for (int j = 0; j < k; ++j)
        if (kh->nf[j] == 0.0 && !kh->cdone[j]) any_zero = true;
    if (any_zero) {
        int all = 1;
        for (int j = 0; j < K; ++j) {
            if (j < k && kh->nf[j] == 0.0) kh->cdone[j] = 1;
            all &= kh->cdone[j];
        }
        kh->done = all;
        ck(cudaMemcpyAsync(batch.ks, kh, sizeof(KStateB), cudaMemcpyHostToDevice, stream), "ks update");
    }
    if (!kh->done && std::getenv("AMGB_NO_DEVICE_LOOP")) {  // direct launches (ncu profiling)
        while (!kh->done) {
            for (int it = 0; it < 2; ++it) cg_iteration_b<K>(it);
            ck(cudaMemcpyAsync(kh, batch.ks, sizeof(KStateB), cudaMemcpyDeviceToHost, stream), "ks read");
            sync(stream);
        }
    } else if (!kh->done) {
        if (!batch.graph) {  // conditional WHILE node around two iterations (device-side loop)
            cudaGraph_t g;
            ck(cudaGraphCreate(&g, 0), "graph create");
            cudaGraphConditionalHandle cond;
            ck(cudaGraphConditionalHandleCreate(&cond, g, 1, cudaGraphCondAssignDefault), "cond handle");
            cudaGraphNodeParams cp = {};
            cp.type = cudaGraphNodeTypeConditional;
            cp.conditional.handle = cond;
            cp.conditional.type = cudaGraphCondTypeWhile;
            cp.conditional.size = 1;
            cudaGraphNode_t node;
            ck(cudaGraphAddNode(&node, g, nullptr, 0, &cp), "conditional node");
            const int64_t before = launches;
            const int saved_mask = prof_mask;
            prof_mask = 0;  // no event nodes inside conditional bodies
            ck(cudaStreamBeginCaptureToGraph(stream, cp.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                             cudaStreamCaptureModeThreadLocal),
               "capture body");
            capturing = true;
            std::vector<Rec> saved;
            saved.swap(rec_graph);
            try {
                for (int it = 0; it < 2; ++it) {
                    cur_iter = it;
                    cg_iteration_b<K>(it);
                }
                cur_iter = -1;
                launch(AMG_PROF_VECTOR, 0, "loop test",
                       [&] { set_loop_kernel<<<1, 1, 0, stream>>>(cond, &batch.ks->done); });
            } catch (...) {
                capturing = false;
                prof_mask = saved_mask;
                cudaGraph_t dummy;
                cudaStreamEndCapture(stream, &dummy);
                cudaGraphDestroy(g);
                rec_graph.swap(saved);
                throw;
            }
            capturing = false;
            prof_mask = saved_mask;
            batch.rec.swap(rec_graph);
            rec_graph.swap(saved);
            cudaGraph_t body_out;
            ck(cudaStreamEndCapture(stream, &body_out), "end capture");
            batch.graph_kernels = launches - before;
            launches = before;
            ck(cudaGraphInstantiate(&batch.graph, g, 0), "instantiate");
            cudaGraphDestroy(g);
        }
        ck(cudaGraphLaunch(batch.graph, stream), "graph launch");
    }
    rows(p, p.lv[0].A, OpResidualB<K, 1, FinTrueResB<K>>{batch.xw, batch.fw, batch.r, FinTrueResB<K>{batch.ks}},
         nullptr, "true res (batched)");
    launch(AMG_PROF_VECTOR, 8.0 * K * n, "unpack X",
           [&] { unpack_cols<K><<<grid_for(n), kBlock, 0, stream>>>(batch.xw, k, n, X, ldx, batch.ks); });
    ck(cudaEventRecord(ev1, stream), "event");
    ck(cudaMemcpyAsync(kh, batch.ks, sizeof(KStateB), cudaMemcpyDeviceToHost, stream), "ks read");
    sync(stream);
    int itmax = 0;
    for (int j = 0; j < K; ++j) itmax = std::max(itmax, kh->iter[j]);
    const int bodies = (itmax + 1) / 2;
    launches += batch.graph_kernels * bodies;
    for (int b = 0; b < bodies; ++b) collect(batch.rec, std::min(2, itmax - 2 * b), false);
    collect(rec_direct, 0, true);
    amg_status st = AMG_OK;
    for (int j = 0; j < k; ++j) {
        iters[j] = kh->iter[j];
        rel[j] = kh->nf[j] == 0.0 ? 0.0 : kh->true_res[j] / kh->nf[j];
        if (kh->status[j] == AMG_BREAKDOWN)
            st = AMG_BREAKDOWN;
        else if (st == AMG_OK && kh->nf[j] != 0.0 && !(kh->res[j] <= kh->tolnf[j]))
            st = AMG_NOT_CONVERGED;
    }
    float ms = 0;
    cudaEventElapsedTime(&ms, ev0, ev1);
    stats = amg_solve_stats{};
    stats.iters = itmax;
    stats.vcycles = itmax;
    stats.status = st;
    stats.kernel_launches = launches - launches0;
    stats.solve_ms = ms;
    stats.rel_resid = 0;
    for (int j = 0; j < k; ++j) stats.rel_resid = std::max(stats.rel_resid, rel[j]);
    stats.alg_bytes = alg_bytes;
    if (st == AMG_BREAKDOWN) g_err = "CG breakdown in a batched column";
    return st;
}

// ============================================================ GMRES(m)
template <class Fin>
struct VNorm2T {  // (a, a) with a chosen finalizer
    static constexpr int NDOT = 1, STREAMS = 1;
    const double* a;
    Fin fin;
    __device__ void prepare() {}
    __device__ void elem(int64_t i, double* d) const { d[0] += a[i] * a[i]; }
};
struct FinTrueResG {
    KStateG* ks;
    __device__ void operator()(const double* t) const { ks->beta = sqrt(t[0]); }
};

// Arnoldi step j of the current cycle (gated on stop_step): z = M v_j, w = A z,
// two classical Gram-Schmidt passes against v_0..v_j, |w|, Givens, v_{j+1}.
void Handle::gmres_step(int j) {
    Part& p = parts[0];
    const int64_t n = p.lv[0].n;
    const int32_t* gate = &gm.ks->stop_step;
    GSel g = [gate](Part&) { return gate; };
    double* vj = gm.V + (int64_t)j * n;
    vcycle(0, [vj](Part&) { return (const double*)vj; }, [this](Part&) { return gm.z; }, g, false);
    rows(p, p.lv[0].A, OpSpmv{gm.z, gm.w}, gate, "gmres w = A z");
    const int J = j + 1;
    for (int pass = 0; pass < 2; ++pass) {
        launch(AMG_PROF_VECTOR, 8.0 * (J + 1) * n, "gmres dots", [&] {
            gmres_dots<<<dim3(J, (unsigned)gm.nchunks), kBlock, 0, stream>>>(gm.w, gm.V, n, gm.chunk, gm.partial, gate);
            gmres_dots_fin<<<1, 96, 0, stream>>>(gm.partial, J, (int)gm.nchunks, gm.ks, pass, gate);
        });
        if (pass == 0) {
            launch(AMG_PROF_VECTOR, 8.0 * (J + 2) * n, "gmres axpy", [&] {
                vec_kernel<VGmresAxpy<0>><<<grid_for(n), kBlock, 0, stream>>>(
                    n, VGmresAxpy<0>{gm.w, gm.V, n, J, gm.ks, FinGmresStep{gm.ks, j}}, gate, p.red);
            });
        } else {
            launch(AMG_PROF_VECTOR, 8.0 * (J + 2) * n, "gmres axpy+norm", [&] {
                vec_kernel<VGmresAxpy<1>><<<grid_for(n), kBlock, 0, stream>>>(
                    n, VGmresAxpy<1>{gm.w, gm.V, n, J, gm.ks, FinGmresStep{gm.ks, j}}, gate, p.red);
            });
        }
    }
    if (j + 1 <= gm.m) vec(p, n, VGmresScale{gm.w, gm.V + (int64_t)(j + 1) * n, &gm.ks->hn, {}}, gate, "gmres v");
}

// End of a restart cycle (gated on done): y = H^-1 g, x += M (V y), r = f - A x,
// restart test, v_0 = r / |r|.
void Handle::gmres_cycle_end(const double* f, double* x) {
    Part& p = parts[0];
    const int64_t n = p.lv[0].n;
    const int32_t* gate = &gm.ks->done;
    GSel g = [gate](Part&) { return gate; };
    launch(AMG_PROF_VECTOR, 0, "gmres y", [&] { gmres_solve_y<<<1, 1, 0, stream>>>(gm.ks, gate); });
    launch(AMG_PROF_VECTOR, 8.0 * (gm.m + 1) * n, "gmres u = V y", [&] {
        vec_kernel<VGmresCombine><<<grid_for(n), kBlock, 0, stream>>>(n, VGmresCombine{gm.u, gm.V, n, gm.ks, {}},
                                                                       gate, p.red);
    });
    vcycle(0, [this](Part&) { return (const double*)gm.u; }, [this](Part&) { return gm.z; }, g, false);
    vec(p, n, VAdd{x, gm.z, {}}, gate, "gmres x += z");
    rows(p, p.lv[0].A, OpResidual<1, FinGmresRestart>{x, f, gm.r, FinGmresRestart{gm.ks}}, gate, "gmres r");
    vec(p, n, VGmresScale{gm.r, gm.V, &gm.ks->hn, {}}, gate, "gmres v0");
}

amg_status Handle::solve_gmres(const double* f, double* x, double tol, int32_t maxiter, int32_t* iters, double* rel) {
    Part& p = parts[0];
    const int64_t n = p.lv[0].n;
    const int m = prm.gmres_m;
    if (gm.m != m) {
        free_gmres();
        gm.m = m;
        auto alloc = [&](int64_t cnt) {
            void* q = nullptr;
            ck(cudaMalloc(&q, std::max<int64_t>(cnt, 1) * sizeof(double)), "cudaMalloc (gmres)");
            gm.mem.push_back(q);
            return static_cast<double*>(q);
        };
        gm.V = alloc((int64_t)(m + 1) * n);
        gm.w = alloc(n);
        gm.z = alloc(n);
        gm.u = alloc(n);
        gm.r = alloc(n);
        gm.chunk = std::max<int64_t>(4096, (n + 255) / 256);
        gm.nchunks = (n + gm.chunk - 1) / gm.chunk;
        gm.partial = alloc((int64_t)(m + 1) * gm.nchunks);
        void* q = nullptr;
        ck(cudaMalloc(&q, sizeof(KStateG)), "cudaMalloc");
        gm.mem.push_back(q);
        gm.ks = static_cast<KStateG*>(q);
        ck(cudaMallocHost(&gm.ks_host, sizeof(KStateG)), "cudaMallocHost");
    }
    const int64_t launches0 = launches;
    collect(rec_direct, 0, true);
    alg_bytes = 0;
    std::fill(acc_ms, acc_ms + 8, 0.0);
    std::fill(acc_bytes, acc_bytes + 8, 0.0);
    std::fill(acc_launches, acc_launches + 8, 0);
    cur_iter = -1;
    ck(cudaEventRecord(ev0, stream), "event");
    KStateG* kh = gm.ks_host;
    std::memset(kh, 0, sizeof(KStateG));
    kh->m = m;
    kh->maxiter = maxiter;
    ck(cudaMemcpyAsync(gm.ks, kh, sizeof(KStateG), cudaMemcpyHostToDevice, stream), "ks init");
    vec(p, n, VNorm2T<FinGmresNorm>{f, FinGmresNorm{gm.ks, tol}}, nullptr, "norm f");
    rows(p, p.lv[0].A, OpResidual<1, FinGmresRestart>{x, f, gm.r, FinGmresRestart{gm.ks}}, nullptr, "gmres r0");
    vec(p, n, VGmresScale{gm.r, gm.V, &gm.ks->hn, {}}, &gm.ks->done, "gmres v0");
    ck(cudaMemcpyAsync(kh, gm.ks, sizeof(KStateG), cudaMemcpyDeviceToHost, stream), "ks read");
    sync(stream);
    collect(rec_direct, 0, true);
    if (kh->nf == 0.0) {  // zero right-hand side: x = 0
        ck(cudaMemsetAsync(x, 0, n * sizeof(double), stream), "memset");
        sync(stream);
        *iters = 0;
        *rel = 0.0;
        stats = amg_solve_stats{};
        stats.kernel_launches = launches - launches0;
        return AMG_OK;
    }
    int cycles = 0;
    const bool use_graph = prm.use_graph && !sync_debug;
    while (!kh->done) {
        if (use_graph) {  // one restart cycle (m gated steps + the update) per graph launch
            if (!gm.graph || gm.graph_x != x || gm.graph_f != f) {
                if (gm.graph) cudaGraphExecDestroy(gm.graph);
                gm.graph = nullptr;
                cudaGraph_t g;
                const int64_t before = launches;
                const int saved_mask = prof_mask;
                prof_mask = 0;
                std::vector<Rec> saved;
                saved.swap(rec_graph);
                ck(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal), "capture");
                capturing = true;
                try {
                    for (int j = 0; j < m; ++j) {
                        cur_iter = j;  // step tag: only executed steps are accounted
                        gmres_step(j);
                    }
                    cur_iter = -1;
                    gmres_cycle_end(f, x);
                } catch (...) {
                    cur_iter = -1;
                    capturing = false;
                    prof_mask = saved_mask;
                    cudaStreamEndCapture(stream, &g);
                    rec_graph.swap(saved);
                    throw;
                }
                capturing = false;
                prof_mask = saved_mask;
                halo_wait();  // the comm stream rejoins before the capture ends
                ck(cudaStreamEndCapture(stream, &g), "end capture");
                gm.rec.swap(rec_graph);
                rec_graph.swap(saved);
                gm.graph_kernels = launches - before;
                launches = before;
                ck(cudaGraphInstantiate(&gm.graph, g, 0), "instantiate");
                cudaGraphDestroy(g);
                gm.graph_x = x;
                gm.graph_f = f;
            }
            const int k_before = kh->k;
            ck(cudaGraphLaunch(gm.graph, stream), "graph launch");
            launches += gm.graph_kernels;
            ck(cudaMemcpyAsync(kh, gm.ks, sizeof(KStateG), cudaMemcpyDeviceToHost, stream), "ks read");
            sync(stream);
            collect(gm.rec, kh->k - k_before, false);  // steps that ran + the cycle end
        } else {
            for (int j = 0; j < m; ++j) gmres_step(j);
            gmres_cycle_end(f, x);
            ck(cudaMemcpyAsync(kh, gm.ks, sizeof(KStateG), cudaMemcpyDeviceToHost, stream), "ks read");
            sync(stream);
            collect(rec_direct, 0, true);
        }
        ++cycles;
    }
    rows(p, p.lv[0].A, OpResidual<1, FinTrueResG>{x, f, gm.r, FinTrueResG{gm.ks}}, nullptr, "true res");
    ck(cudaEventRecord(ev1, stream), "event");
    ck(cudaMemcpyAsync(kh, gm.ks, sizeof(KStateG), cudaMemcpyDeviceToHost, stream), "ks read");
    sync(stream);
    collect(rec_direct, 0, true);
    *iters = kh->k;
    *rel = kh->beta / kh->nf;
    float ms = 0;
    cudaEventElapsedTime(&ms, ev0, ev1);
    stats = amg_solve_stats{};
    stats.iters = kh->k;
    stats.vcycles = kh->k + cycles;
    stats.kernel_launches = launches - launches0;
    stats.solve_ms = ms;
    stats.rel_resid = *rel;
    stats.alg_bytes = alg_bytes;
    if (kh->status == AMG_BREAKDOWN) {
        g_err = "GMRES breakdown: singular Hessenberg";
        stats.status = AMG_BREAKDOWN;
        return AMG_BREAKDOWN;
    }
    const amg_status st = *rel <= tol ? AMG_OK : AMG_NOT_CONVERGED;
    stats.status = st;
    return st;
}

// IDR(s) shadow space P (s x n, row m = column m): the counter-based generator
// of oracle/oracle.c or_idrs_shadow, written independently -- entry (i, m) =
// 2 u - 1, u = top 53 bits of splitmix64(0x181105704 + m n + i) / 2^53 -- then
// modified Gram-Schmidt in the same order (host, no FP contraction).
static uint64_t idr_splitmix64(uint64_t z) {
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

static std::vector<double> idr_shadow(int64_t n, int s) {
    std::vector<double> P((size_t)n * s);
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < n * s; ++e) {
        const uint64_t z = idr_splitmix64(0x181105704ull + (uint64_t)e);
        P[e] = 2.0 * ((double)(z >> 11) * 0x1.0p-53) - 1.0;
    }
    for (int j = 0; j < s; ++j) {
        double* pj = P.data() + (int64_t)j * n;
        for (int q = 0; q < j; ++q) {
            const double* pq = P.data() + (int64_t)q * n;
            double h = 0.0;
            for (int64_t i = 0; i < n; ++i) h += pq[i] * pj[i];
            for (int64_t i = 0; i < n; ++i) pj[i] = pj[i] - h * pq[i];
        }
        double nn = 0.0;
        for (int64_t i = 0; i < n; ++i) nn += pj[i] * pj[i];
        const double nrm = std::sqrt(nn);
        for (int64_t i = 0; i < n; ++i) pj[i] = pj[i] / nrm;
    }
    return P;
}

// One IDR(s) cycle: s inner steps (tags 0..s-1) and the dimension reduction
// (tag s); every kernel is gated by the done flag.
template <int S>
void Handle::idr_cycle(double* x) {
    Part& p = parts[0];
    const int64_t n = p.lv[0].n;
    const int32_t* gate = &idr.ks->done;
    GSel g = [gate](Part&) { return gate; };
    for (int k = 0; k < S; ++k) {
        cur_iter = k;
        launch(AMG_PROF_VECTOR, 0, "idr c", [&] { idr_solve_c<<<1, 1, 0, stream>>>(idr.ks, k); });
        launch(AMG_PROF_VECTOR, 8.0 * (S - k + 2) * n, "idr v = r - G c", [&] {
            vec_kernel<VIdrV<S>><<<grid_for(n), kBlock, 0, stream>>>(
                n, VIdrV<S>{idr.v, idr.r, idr.G, n, k, idr.ks, {}, {}}, gate, p.red);
        });
        vcycle(0, [this](Part&) { return (const double*)idr.v; }, [this](Part&) { return idr.z; }, g, false);
        launch(AMG_PROF_VECTOR, 8.0 * (S - k + 2) * n, "idr U_k", [&] {
            vec_kernel<VIdrU<S>><<<grid_for(n), kBlock, 0, stream>>>(
                n, VIdrU<S>{idr.U, idr.z, n, k, idr.ks, {}, {}, 0.0}, gate, p.red);
        });
        rows(p, p.lv[0].A,
             OpIdrG<S>{idr.U + (int64_t)k * n, idr.G + (int64_t)k * n, idr.P, n, FinIdrOrth{idr.ks, k}}, gate,
             "idr G_k = A U_k + P^T G_k");
        launch(AMG_PROF_VECTOR, 8.0 * (4 * k + 6) * n, "idr update", [&] {
            vec_kernel<VIdrUpd<S>><<<grid_for(n), kBlock, 0, stream>>>(
                n, VIdrUpd<S>{idr.G, idr.U, idr.r, x, n, k, idr.ks, FinIdrRes{idr.ks}, {}, 0.0}, gate, p.red);
        });
    }
    cur_iter = S;
    vcycle(0, [this](Part&) { return (const double*)idr.r; }, [this](Part&) { return idr.z; }, g, false);
    rows(p, p.lv[0].A, OpIdrT{idr.z, idr.t, idr.r, FinIdrOmega{idr.ks}}, gate, "idr t = A z");
    launch(AMG_PROF_VECTOR, 8.0 * (6 + S) * n, "idr reduction update", [&] {
        vec_kernel<VIdrRed<S>><<<grid_for(n), kBlock, 0, stream>>>(
            n, VIdrRed<S>{x, idr.r, idr.z, idr.t, idr.P, n, idr.ks, FinIdrCycle<S>{idr.ks}, 0.0}, gate, p.red);
    });
    cur_iter = -1;
}

template <int S>
amg_status Handle::solve_idrs_t(const double* f, double* x, double tol, int32_t maxiter, int32_t* iters,
                                double* rel) {
    Part& p = parts[0];
    const int64_t n = p.lv[0].n;
    if (idr.s != S) {
        free_idr();
        idr.s = S;
        auto alloc = [&](int64_t cnt) {
            void* q = nullptr;
            ck(cudaMalloc(&q, std::max<int64_t>(cnt, 1) * sizeof(double)), "cudaMalloc (idrs)");
            idr.mem.push_back(q);
            return static_cast<double*>(q);
        };
        idr.P = alloc((int64_t)S * n);
        idr.G = alloc((int64_t)S * n);
        idr.U = alloc((int64_t)S * n);
        idr.v = alloc(n);
        idr.z = alloc(n);
        idr.t = alloc(n);
        idr.r = alloc(n);
        const std::vector<double> P = idr_shadow(n, S);
        ck(cudaMemcpy(idr.P, P.data(), P.size() * sizeof(double), cudaMemcpyHostToDevice), "upload P");
        void* q = nullptr;
        ck(cudaMalloc(&q, sizeof(KStateI)), "cudaMalloc");
        idr.mem.push_back(q);
        idr.ks = static_cast<KStateI*>(q);
        ck(cudaMallocHost(&idr.ks_host, sizeof(KStateI)), "cudaMallocHost");
    }
    const int64_t launches0 = launches;
    collect(rec_direct, 0, true);
    alg_bytes = 0;
    std::fill(acc_ms, acc_ms + 8, 0.0);
    std::fill(acc_bytes, acc_bytes + 8, 0.0);
    std::fill(acc_launches, acc_launches + 8, 0);
    cur_iter = -1;
    ck(cudaEventRecord(ev0, stream), "event");
    KStateI* kh = idr.ks_host;
    std::memset(kh, 0, sizeof(KStateI));
    kh->s = S;
    kh->maxiter = maxiter;
    kh->om = 1.0;
    kh->kappa = 0.7;
    for (int i = 0; i < S; ++i) kh->M[i * S + i] = 1.0;
    ck(cudaMemcpyAsync(idr.ks, kh, sizeof(KStateI), cudaMemcpyHostToDevice, stream), "ks init");
    ck(cudaMemsetAsync(idr.G, 0, (size_t)S * n * sizeof(double), stream), "memset");
    ck(cudaMemsetAsync(idr.U, 0, (size_t)S * n * sizeof(double), stream), "memset");
    vec(p, n, VNorm2T<FinIdrNorm>{f, FinIdrNorm{idr.ks, tol}}, nullptr, "norm f");
    rows(p, p.lv[0].A, OpResidual<1, FinIdrRes0>{x, f, idr.r, FinIdrRes0{idr.ks}}, nullptr, "idr r0");
    launch(AMG_PROF_VECTOR, 8.0 * (1 + S) * n, "idr phi", [&] {
        vec_kernel<VIdrPhi<S>><<<grid_for(n), kBlock, 0, stream>>>(n, VIdrPhi<S>{idr.r, idr.P, n, {idr.ks}}, nullptr,
                                                                   p.red);
    });
    ck(cudaMemcpyAsync(kh, idr.ks, sizeof(KStateI), cudaMemcpyDeviceToHost, stream), "ks read");
    sync(stream);
    collect(rec_direct, 0, true);
    if (kh->nf == 0.0) {  // zero right-hand side: x = 0
        ck(cudaMemsetAsync(x, 0, n * sizeof(double), stream), "memset");
        sync(stream);
        *iters = 0;
        *rel = 0.0;
        stats = amg_solve_stats{};
        stats.kernel_launches = launches - launches0;
        return AMG_OK;
    }
    const bool use_graph = prm.use_graph && !sync_debug;
    while (!kh->done) {
        const int it_before = kh->it;
        if (use_graph) {  // one cycle (s gated steps + the reduction) per graph launch
            if (!idr.graph || idr.graph_x != x || idr.graph_f != f) {
                if (idr.graph) cudaGraphExecDestroy(idr.graph);
                idr.graph = nullptr;
                cudaGraph_t g;
                const int64_t before = launches;
                const int saved_mask = prof_mask;
                prof_mask = 0;
                std::vector<Rec> saved;
                saved.swap(rec_graph);
                ck(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal), "capture");
                capturing = true;
                try {
                    idr_cycle<S>(x);
                } catch (...) {
                    cur_iter = -1;
                    capturing = false;
                    prof_mask = saved_mask;
                    cudaStreamEndCapture(stream, &g);
                    rec_graph.swap(saved);
                    throw;
                }
                capturing = false;
                prof_mask = saved_mask;
                halo_wait();  // the comm stream rejoins before the capture ends
                ck(cudaStreamEndCapture(stream, &g), "end capture");
                idr.rec.swap(rec_graph);
                rec_graph.swap(saved);
                idr.graph_kernels = launches - before;
                launches = before;
                ck(cudaGraphInstantiate(&idr.graph, g, 0), "instantiate");
                cudaGraphDestroy(g);
                idr.graph_x = x;
                idr.graph_f = f;
            }
            ck(cudaGraphLaunch(idr.graph, stream), "graph launch");
            launches += idr.graph_kernels;
            ck(cudaMemcpyAsync(kh, idr.ks, sizeof(KStateI), cudaMemcpyDeviceToHost, stream), "ks read");
            sync(stream);
            collect(idr.rec, kh->it - it_before, false);  // the steps that ran
        } else {
            idr_cycle<S>(x);
            ck(cudaMemcpyAsync(kh, idr.ks, sizeof(KStateI), cudaMemcpyDeviceToHost, stream), "ks read");
            sync(stream);
            collect(rec_direct, 0, true);
        }
    }
    rows(p, p.lv[0].A, OpResidual<1, FinTrueResI>{x, f, idr.r, FinTrueResI{idr.ks}}, nullptr, "true res");
    ck(cudaEventRecord(ev1, stream), "event");
    ck(cudaMemcpyAsync(kh, idr.ks, sizeof(KStateI), cudaMemcpyDeviceToHost, stream), "ks read");
    sync(stream);
    collect(rec_direct, 0, true);
    *iters = kh->it;
    *rel = kh->res / kh->nf;
    float ms = 0;
    cudaEventElapsedTime(&ms, ev0, ev1);
    stats = amg_solve_stats{};
    stats.iters = kh->it;
    stats.vcycles = kh->it;
    stats.kernel_launches = launches - launches0;
    stats.solve_ms = ms;
    stats.rel_resid = *rel;
    stats.alg_bytes = alg_bytes;
    if (kh->status == AMG_BREAKDOWN) {
        g_err = "IDR(s) breakdown: M[k][k] = 0 or omega = 0";
        stats.status = AMG_BREAKDOWN;
        return AMG_BREAKDOWN;
    }
    const amg_status st = *rel <= tol ? AMG_OK : AMG_NOT_CONVERGED;
    stats.status = st;
    return st;
}

// The handle's Krylov method; with a reordered store the API vectors are
// permuted into the stored order first and the solution back afterwards.
amg_status Handle::solve_dispatch(const double* f, double* x, double tol, int32_t maxiter, int32_t* iters,
                                  double* rel) {
    if (prm.solver == 2 && !distributed()) return solve_gmres(f, x, tol, maxiter, iters, rel);
    if (prm.solver == 3 && !distributed()) return solve_idrs(f, x, tol, maxiter, iters, rel);
    return solve(f, x, tol, maxiter, iters, rel);
}

amg_status Handle::solve_api(const double* f, double* x, double tol, int32_t maxiter, int32_t* iters, double* rel) {
    if (!reordered) return solve_dispatch(f, x, tol, maxiter, iters, rel);
    perm_in(f, rf);
    perm_in(x, rx);
    const amg_status st = solve_dispatch(rf, rx, tol, maxiter, iters, rel);
    perm_out(rx, x);
    sync(stream);
    stats.flags |= 2;  // bit 1: reordered store
    return st;
}

amg_status Handle::solve_idrs(const double* f, double* x, double tol, int32_t maxiter, int32_t* iters, double* rel) {
    switch (prm.idrs_s) {
        case 1: return solve_idrs_t<1>(f, x, tol, maxiter, iters, rel);
        case 2: return solve_idrs_t<2>(f, x, tol, maxiter, iters, rel);
        case 4: return solve_idrs_t<4>(f, x, tol, maxiter, iters, rel);
        default: return solve_idrs_t<8>(f, x, tol, maxiter, iters, rel);
    }
}

// z = M r for every part (r, z: device; global vectors in virtual mode).
void Handle::precond(const double* r, double* z) {
    GSel nogate = [](Part&) { return (const int32_t*)nullptr; };
    if (!distributed()) {
        vcycle(0, [r](Part&) { return r; }, [z](Part&) { return z; }, nogate, false);
        return;
    }
    for (Part& p : parts)  // the V-cycle input needs a ghost region: copy into p.s
        ck(cudaMemcpyAsync(p.s, r + (virt ? p.row0 : 0), p.lv[0].n * sizeof(double), cudaMemcpyDeviceToDevice, stream),
           "copy");
    vcycle(0, [](Part& p) { return (const double*)p.s; }, [](Part& p) { return p.sh; }, nogate, false);
    for (Part& p : parts)
        ck(cudaMemcpyAsync(z + (virt ? p.row0 : 0), p.sh, p.lv[0].n * sizeof(double), cudaMemcpyDeviceToDevice, stream),
           "copy");
}

// ---- upload -------------------------------------------------------------------

namespace {

// Matrix format policy: AMGB_FORMAT = auto (default) | csr | sell | tma.
// auto: row-block CSR for matrices with < 65536 rows (coarse levels: few, long
// rows); otherwise TMA-staged SELL-32 for narrow rows, SELL-32 for wide ones.
// stage capacity (entries) of the TMA-staged CSR format: the largest tile's
// value / column range after aligning its start down to 16 bytes
int64_t tcsr_tile_ent(const Csr& A) {
    int64_t te = 4;
    for (int64_t r0 = 0; r0 < A.nrows; r0 += kTcRows) {
        const int64_t r1 = std::min<int64_t>(r0 + kTcRows, A.nrows);
        const int64_t e0 = A.ptr[r0], e1 = A.ptr[r1];
        te = std::max<int64_t>(te, ((e1 - (e0 & ~(int64_t)3)) + 3) & ~(int64_t)3);     // columns, fp64 values
        te = std::max<int64_t>(te, ((e1 - (e0 & ~(int64_t)15)) + 15) & ~(int64_t)15);  // 1-byte value indices
    }
    return (te + 15) & ~(int64_t)15;
}

// role of a matrix in the V-cycle (the format policy treats wide R differently)
enum class Role { A, P, R };

// *want_index: the pick is TMA-CSR for a wide A, which pays only when its
// values index to at most 2 bytes (upload falls back to SELL-32 otherwise).
Fmt pick_format(const Csr& A, Role role, bool* want_index = nullptr) {
    if (want_index) *want_index = false;
    const char* e = std::getenv("AMGB_FORMAT");
    const std::string f = e ? e : "auto";
    if (f == "csr") return Fmt::CSR;
    if (f == "sell") return Fmt::SELL;
    int64_t lmax = 0;
    for (int64_t r = 0; r < A.nrows; ++r) lmax = std::max<int64_t>(lmax, A.ptr[r + 1] - A.ptr[r]);
    // a TMA stage holds a tile of 8 slices x 32 rows x (longest row) entries at
    // 12 B, kTmaStages of them must fit the 227 KB of shared memory per CTA
    const bool tma_fits =
        (int64_t)kTmaStages * 256 * 12 * std::max<int64_t>(lmax, 1) + kVTabBytes + 64 <= 227 * 1024;
    const bool tcsr_fits = A.nrows > 0 && A.nnz() < INT32_MAX &&
                           (int64_t)kTmaStages * (int64_t)tcsr_stage_bytes(tcsr_tile_ent(A), 8) + 64 <= 227 * 1024;
    if (f == "tma") return tma_fits ? Fmt::TMA : Fmt::SELL;
    if (f == "tmacsr") return tcsr_fits ? Fmt::TMACSR : Fmt::SELL;
    if (A.nrows < 65536) return Fmt::CSR;
    // SELL-32 padding: every row of a 32-row slice is stored at the slice's
    // longest row's length
    int64_t stored = 0;
    for (int64_t s0 = 0; s0 < A.nrows; s0 += 32) {
        int64_t w = 0;
        for (int64_t r = s0; r < std::min<int64_t>(s0 + 32, A.nrows); ++r) w = std::max<int64_t>(w, A.ptr[r + 1] - A.ptr[r]);
        stored += 32 * w;
    }
    const double pad = A.nnz() ? (double)stored / (double)A.nnz() : 1.0;
    // AMGB_TMACSR: 0 never, 1 narrow padded matrices only, 2 also every wide
    // padded one, 3 (default) narrow ones and wide restrictions, 4 as 3 plus
    // the wide A whose values index to 2 bytes (measured slower: 35.0 vs 33.7 ms
    // at 256^3, the A1 passes 10.1 vs 8.4 ms, profiles/r02_tcsr_vi16_tried)
    const char* tc = std::getenv("AMGB_TMACSR");
    const int tmode = tc ? std::atoi(tc) : 3;
    // narrow rows: TMA-staged SELL-32 when its slices are (nearly) unpadded --
    // the level-0 stencil, whose slices also compress to an offset dictionary --
    // else the padding-free TMA-staged CSR (smoothed-aggregation P).  Wide rows:
    // the restrictions R in TMA-CSR too (their few distinct values index to one
    // byte, which the TMA kernels take), the coarse A in register-pipelined
    // SELL-32 (even with 16-bit value indices, AMGB_TMACSR=4, csr_tma is slower
    // on its ~31-entry rows):
    // 256^3, interleaved A/B: all wide in TMA-CSR moved the transfer class
    // 10.9 -> 9.5 ms but the coarse A passes 8.4 -> 10.9 ms (profiles/r02_tcsr_wide)
    if (lmax <= 12) return (tmode >= 1 && pad > 1.15 && tcsr_fits) ? Fmt::TMACSR : Fmt::TMA;
    const bool wide_tcsr = tmode == 2 || (tmode >= 3 && role == Role::R) || (tmode == 4 && role == Role::A);
    const bool pick = wide_tcsr && pad > 1.05 && tcsr_fits;
    if (pick && want_index && tmode == 4 && role == Role::A) *want_index = true;
    return pick ? Fmt::TMACSR : Fmt::SELL;
}

// Row blocks of the CSR kernel: at most kEnt entries and a row cap chosen from
// the mean row length; a row longer than kEnt forms a block of its own.
std::vector<int32_t> row_blocks(const Csr& A, int G) {
    const double avg = A.nrows ? (double)A.nnz() / (double)A.nrows : 0.0;
    const int64_t cap = G > 1 ? kRowsMax : (avg < 4.0 ? 512 : 256);
    std::vector<int32_t> b{0};
    int64_t r = 0;
    while (r < A.nrows) {
        int64_t ents = 0, rows = 0;
        if (A.ptr[r + 1] - A.ptr[r] > kEnt) {
            ++r;
        } else {
            while (r < A.nrows && rows < cap && ents + (A.ptr[r + 1] - A.ptr[r]) <= kEnt) {
                ents += A.ptr[r + 1] - A.ptr[r];
                ++rows;
                ++r;
            }
        }
        b.push_back((int32_t)r);
    }
    return b;
}

DMat upload_mat_impl(Handle& H, const Csr& A, int64_t* bytes, bool f32, Role role);

// upload_mat with AMGB_SETUP_TIMING: per-matrix conversion + copy time
DMat upload_mat(Handle& H, const Csr& A, int64_t* bytes, bool f32 = false, Role role = Role::A) {
    const auto t0 = std::chrono::steady_clock::now();
    const double up0 = H.upload_ms;
    DMat d = upload_mat_impl(H, A, bytes, f32, role);
    if (std::getenv("AMGB_SETUP_TIMING"))
        std::fprintf(stderr, "[setup]   matrix %lld x %lld, %lld nnz, fmt %d: %.1f ms (H2D %.1f ms)\n",
                     (long long)A.nrows, (long long)A.ncols, (long long)A.nnz(), (int)d.fmt,
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count(),
                     H.upload_ms - up0);
    return d;
}

// Device-side format construction (convert.cuh): the CSR goes to the device
// once and the SELL / TMA arrays are built there -- the same arrays as the
// host converters below (AMGB_HOST_CONVERT=1 selects those).
struct DevTmp {  // scratch freed at scope exit
    std::vector<void*> p;
    template <class T>
    T* get(int64_t n) {
        void* q = nullptr;
        ck(cudaMalloc(&q, std::max<int64_t>(n, 1) * sizeof(T)), "cudaMalloc (convert)");
        p.push_back(q);
        return static_cast<T*>(q);
    }
    ~DevTmp() {
        for (void* q : p) cudaFree(q);
    }
};

static void dev_scan_ptr(int64_t* v, int64_t n) {  // inclusive sum of v[1..n] in place (v[0] = 0)
    if (n <= 0) return;
    size_t tmp = 0;
    ck(cub::DeviceScan::InclusiveSum(nullptr, tmp, v + 1, v + 1, (int)n), "scan");
    void* t = nullptr;
    ck(cudaMalloc(&t, std::max<size_t>(tmp, 1)), "cudaMalloc (scan)");
    const cudaError_t e = cub::DeviceScan::InclusiveSum(t, tmp, v + 1, v + 1, (int)n);
    cudaFree(t);
    ck(e, "scan");
}

static int cv_grid(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 1 << 20)); }

bool upload_sliced_dev(Handle& H, const Csr& A, Fmt fmt, bool f32, bool allow_dict, DMat& d, int64_t* bytes) {
    const int64_t n = A.nrows, nnz = A.nnz(), ns = (n + 31) / 32;
    DevTmp tmp;
    int64_t* dptr = tmp.get<int64_t>(n + 1);
    int32_t* dcol = tmp.get<int32_t>(nnz);
    double* dval = tmp.get<double>(nnz);
    ck(cudaMemcpy(dptr, A.ptr.data(), (n + 1) * sizeof(int64_t), cudaMemcpyHostToDevice), "H2D ptr");
    ck(cudaMemcpy(dcol, A.col.data(), nnz * sizeof(int32_t), cudaMemcpyHostToDevice), "H2D col");
    ck(cudaMemcpy(dval, A.val.data(), nnz * sizeof(double), cudaMemcpyHostToDevice), "H2D val");
    int64_t* sptr = H.talloc<int64_t>(ns + 1);
    cv_slice_width<<<cv_grid(ns), 256>>>(n, ns, dptr, sptr);
    dev_scan_ptr(sptr, ns);
    int64_t stored = 0;
    ck(cudaMemcpy(&stored, sptr + ns, sizeof(int64_t), cudaMemcpyDeviceToHost), "D2H");
    double* sval = H.talloc<double>(stored);
    if (fmt == Fmt::SELL) {
        int32_t* scol = H.talloc<int32_t>(stored);
        cv_fill<<<cv_grid(ns * 32), 256>>>(n, ns, dptr, dcol, dval, sptr, nullptr, nullptr, nullptr, scol, nullptr,
                                           sval);
        d.sell.nrows = n;
        d.sell.ncols = A.ncols;
        d.sell.nslices = ns;
        d.sell.sptr = sptr;
        d.sell.col = scol;
        d.sell.val = sval;
        if (f32) {
            float* vf = H.talloc<float>(stored);
            cv_to_f32<<<cv_grid(stored), 256>>>(stored, sval, vf);
            d.sell.valf = vf;
        }
        d.stored = stored;
        *bytes += (ns + 1) * 8 + stored * 12;
    } else {
        const int64_t nt = (ns + 7) / 8;
        int32_t* U = tmp.get<int32_t>(ns * kDictW);
        int32_t* ulen = tmp.get<int32_t>(ns);
        if (allow_dict)
            cv_dict<<<cv_grid(ns), 256>>>(n, A.ncols, ns, dptr, dcol, sptr, U, ulen);
        else
            ck(cudaMemset(ulen, 0, ns * sizeof(int32_t)), "memset");
        int64_t* tc = tmp.get<int64_t>(nt + 1);
        cv_tile_cols<<<cv_grid(nt), 256>>>(ns, nt, sptr, ulen, tc);
        dev_scan_ptr(tc, nt);
        int64_t ncol_total = 0;
        ck(cudaMemcpy(&ncol_total, tc + nt, sizeof(int64_t), cudaMemcpyDeviceToHost), "D2H");
        int64_t* cptr = H.talloc<int64_t>(ns + 1);
        int64_t* tent = tmp.get<int64_t>(nt);
        int64_t* tib = tmp.get<int64_t>(nt);
        cv_cptr<<<cv_grid(nt), 256>>>(ns, nt, dptr, n, sptr, ulen, tc, cptr, tent, tib);
        int32_t* tcol = H.talloc<int32_t>(ncol_total);
        ck(cudaMemset(tcol, 0, std::max<int64_t>(ncol_total, 1) * sizeof(int32_t)), "memset");
        cv_fill<<<cv_grid(ns * 32), 256>>>(n, ns, dptr, dcol, dval, sptr, ulen, U, cptr, nullptr, tcol, sval);
        ck(cudaGetLastError(), "convert");
        std::vector<int64_t> hent(nt), hib(nt);
        std::vector<int32_t> hulen(ns);
        ck(cudaMemcpy(hent.data(), tent, nt * sizeof(int64_t), cudaMemcpyDeviceToHost), "D2H");
        ck(cudaMemcpy(hib.data(), tib, nt * sizeof(int64_t), cudaMemcpyDeviceToHost), "D2H");
        ck(cudaMemcpy(hulen.data(), ulen, ns * sizeof(int32_t), cudaMemcpyDeviceToHost), "D2H");
        int64_t te = 0, ib = 0, nd = 0;
        for (int64_t t = 0; t < nt; ++t) te = std::max(te, hent[t]), ib += hib[t];
        for (int64_t q = 0; q < ns; ++q) nd += hulen[q] > 0;
        SellTma& t = d.tma;
        t.nrows = n;
        t.ncols = A.ncols;
        t.nslices = ns;
        t.T = 1;
        t.ntiles = nt;
        t.tile_ent = (int32_t)(((std::max<int64_t>(te, 32) + 31) / 32) * 32);
        t.sptr = sptr;
        t.cptr = cptr;
        t.col = tcol;
        t.val = sval;
        if (f32) {
            float* vf = H.talloc<float>(stored);
            cv_to_f32<<<cv_grid(stored), 256>>>(stored, sval, vf);
            t.valf = vf;
        }
        d.stored = stored;
        d.idx_bytes = ib;
        d.ndict = nd;
        *bytes += (ns + 1) * 16 + stored * 8 + ncol_total * 4;
    }
    ck(cudaGetLastError(), "convert");
    ck(cudaDeviceSynchronize(), "convert sync");
    return true;
}

// SELL-C-sigma: inside aligned windows of 256 rows (one CTA of
// sell_rows, one tile of sell_tma) the rows are sorted by length, longest first
// (stable), so each 32-row slice holds rows of similar length and pads less.
// Slot s of the stored matrix holds row (s & ~255) + rp[s]; the kernels map a
// slot to its row for the row-local epilogue operands (slot_row), the columns
// and every row's entry order are unchanged, so each row sum is formed exactly
// as in the unsorted store.  Opt-in (AMGB_SIGMA=1), applied when it cuts the
// stored entries by >= 5 % of nnz (smoothed-aggregation P0 36 % -> 9 %, R0
// 14 % -> 3 %, A1 12 % -> 3 % padding at 256^3); single-part handles only (the
// multi-GPU split passes cut matrices at 32-row granularity).  Measured: no gain
// on the 256^3 solve (41.8 ms either way) -- the padded entries' bytes are
// traded for scattered row-local epilogue accesses.
bool sigma_sort(const Csr& A, std::vector<uint8_t>& rp, Csr& B) {
    const int64_t n = A.nrows;
    auto len = [&](int64_t r) { return A.ptr[r + 1] - A.ptr[r]; };
    rp.assign(n, 0);
    int64_t pad0 = 0, pad1 = 0;
    std::vector<int> idx(256);
    for (int64_t w0 = 0; w0 < n; w0 += 256) {
        const int m = (int)std::min<int64_t>(256, n - w0);
        for (int k = 0; k < m; ++k) idx[k] = k;
        std::stable_sort(idx.begin(), idx.begin() + m, [&](int a, int b) { return len(w0 + a) > len(w0 + b); });
        for (int k = 0; k < m; ++k) rp[w0 + k] = (uint8_t)idx[k];
        for (int s0 = 0; s0 < m; s0 += 32) {
            int64_t u = 0, v = 0;
            for (int k = s0; k < std::min(m, s0 + 32); ++k) {
                u = std::max(u, len(w0 + k));
                v = std::max(v, len(w0 + idx[k]));
            }
            pad0 += 32 * u;
            pad1 += 32 * v;
        }
    }
    if ((double)(pad0 - pad1) < 0.05 * (double)A.nnz()) return false;
    B.nrows = n;
    B.ncols = A.ncols;
    B.ptr.resize(n + 1);
    B.col.resize(A.nnz());
    B.val.resize(A.nnz());
    B.ptr[0] = 0;
    for (int64_t q = 0; q < n; ++q) B.ptr[q + 1] = B.ptr[q] + len((q & ~(int64_t)255) + rp[q]);
    for (int64_t q = 0; q < n; ++q) {
        const int64_t r = (q & ~(int64_t)255) + rp[q];
        std::copy(A.col.begin() + A.ptr[r], A.col.begin() + A.ptr[r + 1], B.col.begin() + B.ptr[q]);
        std::copy(A.val.begin() + A.ptr[r], A.val.begin() + A.ptr[r + 1], B.val.begin() + B.ptr[q]);
    }
    return true;
}

// Value-indexed storage (CSR-VI, Kourtis, Goumas & Koziris 2008): a matrix whose
// stored values take at most 256 (65536) distinct bit patterns is stored as a
// table of those values plus a 1-byte (2-byte) index per entry, on the device:
// sort the bit patterns, keep the unique ones, binary-search every entry.
// Lossless (bit patterns, so -0.0 and 0.0 stay distinct): every kernel reads
// exactly the stored values, and results are bitwise those of the plain store.
// Smoothed-aggregation hierarchies of constant-coefficient operators qualify
// (256^3 Poisson: A0 has 2 distinct values, P0 / R0 9, A1 2641 -> 16-bit);
// log-random coefficients do not.  On by default (256^3 Poisson: 35.5 vs 40.3 ms
// per solve); AMGB_VIDX=0 turns it off.
__global__ void k_vidx(int64_t n, const unsigned long long* __restrict__ v, const unsigned long long* __restrict__ tab,
                       int32_t ntab, uint8_t* i8, uint16_t* i16) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long x = v[k];
        int32_t a = 0, b = ntab;
        while (a < b) {
            const int32_t m = (a + b) >> 1;
            if (tab[m] < x) a = m + 1;
            else b = m;
        }
        if (i8) i8[k] = (uint8_t)a;
        else i16[k] = (uint16_t)a;
    }
}

// dval: n device values; on success *tab (table, 256 or 65536 entries padded
// with zeros) and exactly one of *i8 / *i16 (n + pad entries) are handle
// allocations; *nu (optional) = the number of distinct values.  max_u: at
// most 65536 (more than 256 gives 2-byte indices).
bool value_index(Handle& H, const double* dval, int64_t n, int64_t pad, int64_t max_u, const double** tab,
                 const uint8_t** i8, const uint16_t** i16, int* nu_out = nullptr) {
    *tab = nullptr, *i8 = nullptr, *i16 = nullptr;
    const char* ve = std::getenv("AMGB_VIDX");  // default on; AMGB_VIDX=0 keeps fp64 value arrays
    if (n <= 0 || (ve && ve[0] == '0')) return false;
    DevTmp tmp;
    auto* keys = tmp.get<unsigned long long>(n);
    auto* sorted = tmp.get<unsigned long long>(n);
    auto* uniq = tmp.get<unsigned long long>(n);
    int* nu = tmp.get<int>(1);
    size_t t1 = 0, t2 = 0;
    ck(cub::DeviceRadixSort::SortKeys(nullptr, t1, keys, sorted, (int)n), "vidx sort size");
    ck(cub::DeviceSelect::Unique(nullptr, t2, sorted, uniq, nu, (int)n), "vidx unique size");
    void* tt = tmp.get<unsigned char>((int64_t)std::max(t1, t2));
    ck(cudaMemcpy(keys, dval, n * sizeof(double), cudaMemcpyDeviceToDevice), "vidx copy");
    ck(cub::DeviceRadixSort::SortKeys(tt, t1, keys, sorted, (int)n), "vidx sort");
    ck(cub::DeviceSelect::Unique(tt, t2, sorted, uniq, nu, (int)n), "vidx unique");
    int h_nu = 0;
    ck(cudaMemcpy(&h_nu, nu, sizeof(int), cudaMemcpyDeviceToHost), "D2H");
    if (h_nu < 1 || h_nu > max_u) return false;
    const int64_t tab_n = h_nu <= 256 ? 256 : 65536;
    double* t = H.talloc<double>(tab_n);
    ck(cudaMemset(t, 0, tab_n * sizeof(double)), "memset");
    ck(cudaMemcpy(t, uniq, h_nu * sizeof(double), cudaMemcpyDeviceToDevice), "vidx table");
    uint8_t* a8 = nullptr;
    uint16_t* a16 = nullptr;
    if (h_nu <= 256) {
        a8 = H.talloc<uint8_t>(n + pad);
        ck(cudaMemset(a8, 0, n + pad), "memset");
    } else {
        a16 = H.talloc<uint16_t>(n + pad);
        ck(cudaMemset(a16, 0, (n + pad) * sizeof(uint16_t)), "memset");
    }
    k_vidx<<<cv_grid(n), 256>>>(n, reinterpret_cast<const unsigned long long*>(dval), uniq, h_nu, a8, a16);
    ck(cudaGetLastError(), "vidx");
    ck(cudaDeviceSynchronize(), "vidx sync");
    *tab = t, *i8 = a8, *i16 = a16;
    if (nu_out) *nu_out = h_nu;
    return true;
}

// value-index a freshly uploaded SELL / TMA / TMA-CSR store (fp64 V-cycle only)
void index_store(Handle& H, DMat& d, int64_t* bytes) {
    const double* tab = nullptr;
    const uint8_t* i8 = nullptr;
    const uint16_t* i16 = nullptr;
    if (d.fmt == Fmt::TMA) {  // 1-byte indices only (the table lives in shared memory)
        if (!value_index(H, d.tma.val, d.stored, 16, 256, &tab, &i8, &i16)) return;
        H.tfree(d.tma.val);
        d.tma.val = nullptr;
        d.tma.vtab = tab, d.tma.vi8 = i8;
    } else if (d.fmt == Fmt::TMACSR) {
        // the table is staged in shared memory beside kTmaStages stages of
        // 2-byte indices: at most what is left of the 227 KB
        const int64_t left = 227 * 1024 - 64 - (int64_t)kTmaStages * (int64_t)tcsr_stage_bytes(d.tcsr.tile_ent, 2);
        const int64_t cap = std::min<int64_t>(65536, std::max<int64_t>(256, (left - 256) / 8));
        int nu = 0;
        if (!value_index(H, d.tcsr.val, d.nnz, 16, cap, &tab, &i8, &i16, &nu)) return;
        H.tfree(d.tcsr.val);
        d.tcsr.val = nullptr;
        d.tcsr.vtab = tab, d.tcsr.vi8 = i8, d.tcsr.vi16 = i16;
        d.tcsr.ntab = i8 ? 256 : (nu + 15) & ~15;
    } else if (d.fmt == Fmt::SELL) {
        if (!value_index(H, d.sell.val, d.stored, 16, 65536, &tab, &i8, &i16)) return;
        H.tfree(d.sell.val);
        d.sell.val = nullptr;
        d.sell.vtab = tab, d.sell.vi8 = i8, d.sell.vi16 = i16;
    } else {
        return;
    }
    d.vbytes = i8 ? 1 : 2;
    *bytes -= (8 - d.vbytes) * d.stored;
}

DMat upload_mat_impl(Handle& H, const Csr& A0, int64_t* bytes, bool f32, Role role) {
    DMat d;
    const Csr& A = A0;
    d.nrows = A.nrows;
    d.ncols = A.ncols;
    d.nnz = A.nnz();
    if (d.nnz >= INT32_MAX) throw CudaError{"level has >= 2^31 nonzeros"};
    if (d.nrows == 0) return d;
    bool want_index = false;
    d.fmt = pick_format(A, role, &want_index);
    if (want_index && f32) d.fmt = Fmt::SELL;  // the fp32 store is not value-indexed
    if (d.fmt == Fmt::CSR) {
        const double avg = A.nrows ? (double)A.nnz() / (double)A.nrows : 0.0;
        int G = 1;
        if (avg >= 96) G = 16;
        else if (avg >= 48) G = 8;
        else if (avg >= 20) G = 4;
        else if (avg >= 12) G = 2;
        std::vector<int32_t> ptr32(A.ptr.begin(), A.ptr.end());
        std::vector<int32_t> blocks = row_blocks(A, G);
        d.csr.nrows = A.nrows;
        d.csr.ncols = A.ncols;
        d.csr.nnz = A.nnz();
        d.csr.nblocks = (int64_t)blocks.size() - 1;
        d.csr.G = G;
        d.csr.ptr = H.upload(ptr32);
        d.csr.col = H.upload(A.col);
        d.csr.val = H.upload(A.val);
        d.csr.brow = H.upload(blocks);
        d.hblocks = blocks;
        if (f32) d.csr.valf = H.upload(std::vector<float>(A.val.begin(), A.val.end()));
        d.stored = d.nnz;
        *bytes += (int64_t)(ptr32.size() * 4 + A.col.size() * 12 + blocks.size() * 4);
        return d;
    }
    if (d.fmt == Fmt::TMACSR) {  // CSR with padded arrays (csr_tma reads 16-B aligned ranges), built on the device
        const int64_t n = A.nrows, nnz = A.nnz();
        DevTmp tmp;
        int64_t* p64 = tmp.get<int64_t>(n + 1);
        ck(cudaMemcpy(p64, A.ptr.data(), (n + 1) * sizeof(int64_t), cudaMemcpyHostToDevice), "H2D ptr");
        int32_t* p32 = H.talloc<int32_t>(n + 1 + 8);
        cv_ptr32<<<cv_grid(n + 1), 256>>>(n + 1, p64, p32);
        const std::vector<int32_t> tailp(8, (int32_t)nnz);  // readable past the last row
        ck(cudaMemcpy(p32 + n + 1, tailp.data(), 8 * sizeof(int32_t), cudaMemcpyHostToDevice), "H2D ptr tail");
        int32_t* col = H.talloc<int32_t>(nnz + 4);
        double* val = H.talloc<double>(nnz + 2);
        ck(cudaMemcpy(col, A.col.data(), nnz * sizeof(int32_t), cudaMemcpyHostToDevice), "H2D col");
        ck(cudaMemcpy(val, A.val.data(), nnz * sizeof(double), cudaMemcpyHostToDevice), "H2D val");
        ck(cudaMemset(col + nnz, 0, 4 * sizeof(int32_t)), "memset");
        ck(cudaMemset(val + nnz, 0, 2 * sizeof(double)), "memset");
        CsrTma& t = d.tcsr;
        t.nrows = n;
        t.ncols = A.ncols;
        t.ntiles = (n + kTcRows - 1) / kTcRows;
        t.tile_ent = (int32_t)tcsr_tile_ent(A);
        t.ptr = p32;
        t.col = col;
        t.val = val;
        if (f32) {
            float* vf = H.talloc<float>(nnz + 4);
            ck(cudaMemset(vf, 0, (nnz + 4) * sizeof(float)), "memset");
            cv_to_f32<<<cv_grid(nnz), 256>>>(nnz, val, vf);
            t.valf = vf;
        }
        ck(cudaGetLastError(), "convert");
        d.stored = nnz;
        *bytes += (n + 9) * 4 + (nnz + 4) * 4 + (nnz + 2) * 8;
        if (!f32) index_store(H, d, bytes);
        ck(cudaDeviceSynchronize(), "convert sync");
        if (!want_index || d.vbytes < 8) return d;
        // a wide A with too many distinct values: SELL-32 instead
        *bytes -= (n + 9) * 4 + (nnz + 4) * 4 + (nnz + 2) * 8;
        H.tfree(t.ptr);
        H.tfree(t.col);
        H.tfree(t.val);
        d.tcsr = CsrTma{};
        d.fmt = Fmt::SELL;
    }
    // SELL / TMA: rows sorted by length inside 256-row windows when it pays
    std::vector<uint8_t> rp;
    Csr Bs;
    const char* sg = std::getenv("AMGB_SIGMA");
    const bool sorted = !H.distributed() && sg && sg[0] == '1' && sigma_sort(A0, rp, Bs);
    const Csr& As = sorted ? Bs : A0;
    const bool allow_dict = !sorted && !std::getenv("AMGB_NO_DICT");
    if (!std::getenv("AMGB_HOST_CONVERT")) {  // SELL / TMA built on the device
        upload_sliced_dev(H, As, d.fmt, f32, allow_dict, d, bytes);
    } else if (d.fmt == Fmt::SELL) {
        const Csr& A = As;
        HostSell S = to_sell(A, 32);
        d.sell.nrows = S.nrows;
        d.sell.ncols = S.ncols;
        d.sell.nslices = S.nslices;
        d.sell.sptr = H.upload(S.sptr);
        d.sell.col = H.upload(S.col);
        d.sell.val = H.upload(S.val);
        if (f32) d.sell.valf = H.upload(std::vector<float>(S.val.begin(), S.val.end()));
        d.stored = (int64_t)S.col.size();
        *bytes += (int64_t)(S.sptr.size() * 8 + S.col.size() * 12);
    } else {  // TMA-staged SELL-C: lanes per row T from the longest row, C = 32 / T
        const Csr& A = As;
        int64_t lmax = 0;
        for (int64_t r = 0; r < A.nrows; ++r) lmax = std::max<int64_t>(lmax, A.ptr[r + 1] - A.ptr[r]);
        // the kernel supports T lanes per row (SELL-C, C = 32/T); the format policy
        // only sends narrow rows here, which use one lane per row
        (void)lmax;
        const int T = 1;
        const int C = 32 / T;
        HostSell S = to_sell(A, C);
        SellTma& t = d.tma;
        t.nrows = S.nrows;
        t.ncols = S.ncols;
        t.nslices = S.nslices;
        t.T = T;
        t.ntiles = (S.nslices + 7) / 8;
        int64_t te = 0;
        for (int64_t q = 0; q < t.ntiles; ++q)
            te = std::max(te, S.sptr[std::min<int64_t>((q + 1) * 8, S.nslices)] - S.sptr[q * 8]);
        HostTmaCols TC = tma_cols(A, S, allow_dict);
        for (int64_t q = 0; q < t.ntiles; ++q)
            te = std::max(te, TC.cptr[std::min<int64_t>((q + 1) * 8, S.nslices)] - TC.cptr[q * 8]);
        t.tile_ent = (int32_t)(((std::max<int64_t>(te, 32) + 31) / 32) * 32);
        t.sptr = H.upload(S.sptr);
        t.cptr = H.upload(TC.cptr);
        t.col = H.upload(TC.col);
        t.val = H.upload(S.val);
        if (f32) t.valf = H.upload(std::vector<float>(S.val.begin(), S.val.end()));
        d.stored = (int64_t)S.col.size();
        d.idx_bytes = TC.idx_bytes;
        d.ndict = TC.ndict;
        *bytes += (int64_t)(S.sptr.size() * 16 + S.val.size() * 8 + TC.col.size() * 4);
    }
    if (sorted) {
        const uint8_t* drp = H.upload(rp);
        if (d.fmt == Fmt::TMA)
            d.tma.rperm = drp;
        else
            d.sell.rperm = drp;
        d.sigma = true;
        *bytes += (int64_t)rp.size();
    }
    if (!f32) index_store(H, d, bytes);
    return d;
}

// Chebyshev coefficients (§8c c-1): alpha_0 = 1/d; alpha_1 = 2d/(2d^2 - c^2);
// alpha_k = 1/(d - alpha_{k-1} c^2/4); beta_k = alpha_k d - 1.
void cheb_coeffs(double d, double c, int K, std::vector<double>& a, std::vector<double>& b) {
    a.assign(std::max(K, 1), 0.0);
    b.assign(std::max(K, 1), 0.0);
    double alpha = 0.0;
    for (int k = 0; k < K; ++k) {
        if (k == 0)
            alpha = 1.0 / d;
        else if (k == 1)
            alpha = 2.0 * d / (2.0 * d * d - c * c);
        else
            alpha = 1.0 / (d - alpha * c * c / 4.0);
        a[k] = alpha;
        b[k] = k == 0 ? 0.0 : alpha * d - 1.0;
    }
}

// Algorithmic HBM bytes of one V-cycle on a level: every matrix
// read once per pass (12 B per entry + 4 B per row), every vector read or
// written once per kernel that touches it.
double level_alg_bytes(int64_t n_, int64_t z_, int64_t p_, int64_t c_, const amg_params& p, bool coarsest) {
    const double n = (double)n_;
    if (coarsest) return 8.0 * n * n + 16.0 * n;
    // fp32 hierarchy values: 8 instead of 12 bytes per entry (scale nnz by 2/3)
    const double mscale = p.precision == 1 ? 8.0 / 12.0 : 1.0;
    const double z = (double)z_ * mscale;
    const double pp = (double)p_ * mscale, c = (double)c_;
    const double apass_relax = 12 * z + 4 * n + 32 * n;  // x, m, f read, out written
    const double restrict_b = 12 * pp + 4 * c + 8 * n + 8 * c;
    if (p.relax == 2) {
        const double step = 12 * z + 4 * n + 48 * n;  // x, f, diag, p read; p, xo written
        const double K = p.cheb_degree;
        const double pre = p.npre > 0 ? 32 * n + (K * p.npre - 1) * step : 0;
        const double post = p.npost * K * step;
        const double res = 12 * z + 4 * n + 24 * n;
        const double prol = 12 * pp + 4 * n + 8 * c + 16 * n;
        return pre + res + restrict_b + prol + post;
    }
    double pre = 0, prol = 0;
    if (p.npre == 1) {
        pre = 12 * z + 4 * n + 24 * n;            // m, f gathered, t written
        prol = 12 * pp + 4 * n + 8 * c + 24 * n;  // m, f read, x written
    } else {
        pre = (p.npre > 0 ? 24 * n + (p.npre - 1) * apass_relax : 8 * n) + 12 * z + 4 * n + 24 * n;
        prol = 12 * pp + 4 * n + 8 * c + 16 * n;
    }
    return pre + restrict_b + prol + p.npost * apass_relax;
}

// Upload one rank part into a device Part.
// Gather locality of a matrix (params.reorder = 2, automatic): distinct 32-byte
// sectors of the gathered vector touched by a 256-row tile, per entry, over a
// sample of tiles -- about 0.2 for a stencil in natural order (neighbouring rows
// share sectors), about 1 for a randomly permuted matrix.
double gather_sectors_per_entry(const Csr& A) {
    const int64_t tiles = (A.nrows + 255) / 256;
    if (tiles == 0) return 0.0;
    const int64_t step = std::max<int64_t>(1, tiles / 1024);
    int64_t distinct = 0, ents = 0;
    std::vector<int32_t> sec;
    for (int64_t t = 0; t < tiles; t += step) {
        const int64_t r0 = t * 256, r1 = std::min<int64_t>(A.nrows, r0 + 256);
        sec.clear();
        for (int64_t e = A.ptr[r0]; e < A.ptr[r1]; ++e) sec.push_back(A.col[e] >> 2);
        std::sort(sec.begin(), sec.end());
        distinct += std::unique(sec.begin(), sec.end()) - sec.begin();
        ents += (int64_t)sec.size();
    }
    return ents ? (double)distinct / (double)ents : 0.0;
}

// Reverse Cuthill-McKee order of A's row pattern (params.reorder): breadth-first
// from a minimum-degree node of each component, neighbours by ascending degree,
// reversed.  Returns q with q[old] = new.
std::vector<int64_t> rcm_order(const Csr& A) {
    const int64_t n = A.nrows;
    std::vector<int64_t> order;
    order.reserve(n);
    std::vector<char> seen(n, 0);
    std::vector<int64_t> by_deg(n);
    std::iota(by_deg.begin(), by_deg.end(), 0);
    auto deg = [&](int64_t i) { return A.ptr[i + 1] - A.ptr[i]; };
    std::stable_sort(by_deg.begin(), by_deg.end(), [&](int64_t a, int64_t b) { return deg(a) < deg(b); });
    std::vector<int64_t> nb;
    for (int64_t start : by_deg) {
        if (seen[start]) continue;
        seen[start] = 1;
        size_t head = order.size();
        order.push_back(start);
        while (head < order.size()) {
            const int64_t i = order[head++];
            nb.clear();
            for (int64_t k = A.ptr[i]; k < A.ptr[i + 1]; ++k) {
                const int64_t j = A.col[k];
                if (!seen[j]) {
                    seen[j] = 1;
                    nb.push_back(j);
                }
            }
            std::stable_sort(nb.begin(), nb.end(), [&](int64_t a, int64_t b) { return deg(a) < deg(b); });
            order.insert(order.end(), nb.begin(), nb.end());
        }
    }
    std::vector<int64_t> q(n);
    for (int64_t k = 0; k < n; ++k) q[order[n - 1 - k]] = k;
    return q;
}

// Rows moved to qr[i], columns renamed qc[c]; every row keeps its entries in the
// original order, so each row sum is formed exactly as before.
Csr permute_csr(const Csr& M, const std::vector<int64_t>& qr, const std::vector<int64_t>& qc) {
    Csr P;
    P.nrows = M.nrows;
    P.ncols = M.ncols;
    P.ptr.assign(M.nrows + 1, 0);
    for (int64_t i = 0; i < M.nrows; ++i) P.ptr[qr[i] + 1] = M.ptr[i + 1] - M.ptr[i];
    for (int64_t i = 0; i < M.nrows; ++i) P.ptr[i + 1] += P.ptr[i];
    P.col.resize(M.nnz());
    P.val.resize(M.nnz());
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < M.nrows; ++i) {
        int64_t d = P.ptr[qr[i]];
        for (int64_t k = M.ptr[i]; k < M.ptr[i + 1]; ++k, ++d) {
            P.col[d] = (int32_t)qc[M.col[k]];
            P.val[d] = M.val[k];
        }
    }
    return P;
}

// The single-rank part of the reordered store: q_0 = RCM(A_0); an aggregate is
// numbered by the new index of its root, so every level keeps the locality.
RankPart reordered_part(const HostHierarchy& H, std::vector<std::vector<int64_t>>& q,
                        std::vector<double>& inv_perm) {
    const int L = (int)H.levels.size();
    q.assign(L, {});
    q[0] = rcm_order(H.levels[0].A);
    for (int l = 0; l + 1 < L; ++l) {
        const HostLevel& hl = H.levels[l];
        const int64_t nc = hl.n_agg;
        std::vector<int64_t> by(nc);
        std::iota(by.begin(), by.end(), 0);
        std::sort(by.begin(), by.end(), [&](int64_t a, int64_t b) { return q[l][hl.root[a]] < q[l][hl.root[b]]; });
        q[l + 1].assign(nc, 0);
        for (int64_t k = 0; k < nc; ++k) q[l + 1][by[k]] = k;
    }
    RankPart RP;
    RP.rank = 0;
    RP.nranks = 1;
    RP.lg = L;
    RP.lv.resize(L);
    for (int l = 0; l < L; ++l) {
        const HostLevel& hl = H.levels[l];
        LevelPart& lp = RP.lv[l];
        const bool coarsest = l == L - 1;
        const int64_t n = hl.A.nrows;
        lp.replicated = true;
        lp.row0 = 0;
        lp.row1 = n;
        lp.A = permute_csr(hl.A, q[l], q[l]);
        if (!coarsest) {
            lp.P = permute_csr(hl.P, q[l], q[l + 1]);
            lp.R = permute_csr(hl.R, q[l + 1], q[l]);
            lp.crow0 = 0;
            lp.crow1 = hl.P.ncols;
            lp.next_replicated = true;
        }
        auto perm_vec = [&](const std::vector<double>& v, std::vector<double>& out) {
            out.assign(v.size(), 0.0);
            for (size_t i = 0; i < v.size(); ++i) out[q[l][i]] = v[i];
        };
        perm_vec(hl.m, lp.m);
        perm_vec(hl.diag, lp.diag);
        lp.halo.nloc = n;
    }
    const int64_t nL = H.levels.back().A.nrows;
    inv_perm.assign(H.coarse_inv.size(), 0.0);
    const auto& qL = q[L - 1];
    for (int64_t a = 0; a < nL; ++a)
        for (int64_t b = 0; b < nL; ++b) inv_perm[qL[a] * nL + qL[b]] = H.coarse_inv[a * nL + b];
    return RP;
}

void upload_part(Handle& H, const RankPart& RP, Part& P) {
    const amg_params& prm = H.prm;
    const int nlev = (int)RP.lv.size();
    P.rank = RP.rank;
    P.row0 = RP.lv[0].row0;
    P.row1 = RP.lv[0].row1;
    P.lv.resize(nlev);
    for (int l = 0; l < nlev; ++l) {
        const LevelPart& lp = RP.lv[l];
        const LevelMeta& hl = H.meta[l];
        DevLevel& L = P.lv[l];
        const bool coarsest = l == nlev - 1;
        L.replicated = lp.replicated;
        L.next_replicated = lp.next_replicated;
        L.n = lp.ma().nrows;
        L.ng = lp.replicated ? 0 : lp.halo.nghost;
        L.crow0 = lp.crow0;
        L.crow1 = lp.crow1;
        L.nnzA = lp.ma().nnz();
        L.nnzP = coarsest ? 0 : lp.mp().nnz();
        L.nnzR = coarsest ? 0 : lp.mr().nnz();
        L.nc = coarsest ? 0 : lp.mp().ncols;
        if (prm.relax == 2 && !coarsest)
            cheb_coeffs(hl.cheb_d, hl.cheb_c, prm.cheb_degree, L.cheb_alpha, L.cheb_beta);
        L.alg_bytes = level_alg_bytes(L.n, L.nnzA, L.nnzP, coarsest ? 0 : lp.crow1 - lp.crow0, prm, coarsest);
        const int64_t nv = L.n + L.ng;
        const bool f32 = prm.precision == 1;  // fp32 copies of the V-cycle matrix values
        if (!coarsest || nlev == 1) {
            L.A = upload_mat(H, lp.ma(), &L.dev_bytes, f32);
            L.padA = L.A.stored;
            L.dictA = L.A.ndict;
        } else {
            L.padA = L.nnzA;
        }
        if (!coarsest) {
            L.P = upload_mat(H, lp.mp(), &L.dev_bytes, f32, Role::P);
            L.R = upload_mat(H, lp.mr(), &L.dev_bytes, f32, Role::R);
        }
        // multi-GPU: interior rows (no ghost column) of each pass that follows a
        // halo exchange -- A and R gather this level's vectors, P the next level's
        if (H.distributed() && !lp.replicated && std::getenv("AMGB_NO_SPLIT") == nullptr) {
            auto mark = [](DMat& M, const Csr& host, int64_t nloc) {
                const auto r = interior_range(host, nloc, M.fmt, M.hblocks);
                M.split = true;  // boundary-only when the range is empty
                M.ib0 = r.first;
                M.ib1 = r.second;
            };
            mark(L.A, lp.ma(), L.n);
            if (!coarsest) {
                mark(L.R, lp.mr(), L.n);
                if (!lp.next_replicated) mark(L.P, lp.mp(), lp.crow1 - lp.crow0);
            }
        }
        if (!coarsest) {
            if (prm.relax != 2) L.m = H.upload(lp.m);
            if (prm.relax == 2) L.diag = H.upload(lp.diag);  // Chebyshev D^-1 scaling
            L.x = H.dalloc(nv);
            L.y = H.dalloc(nv);
            L.t = H.dalloc(nv);
            if (prm.relax == 2) L.p = H.dalloc(nv);
            L.dev_bytes += 8 * nv * (prm.relax == 2 ? 5 : 4);
        }
        if (l > 0) {
            L.f = H.dalloc(nv);
            L.o = H.dalloc(nv);
            L.dev_bytes += 16 * nv;
            if (!coarsest && prm.relax != 2 && prm.npre == 1 && !std::getenv("AMGB_NO_MF")) {
                L.mf = H.dalloc(nv);
                L.dev_bytes += 8 * nv;
            }
        } else if (!coarsest && prm.solver == 0 && prm.relax != 2 && prm.npre == 1 && !std::getenv("AMGB_NO_MF")) {
            // level 0 (CG): m o r, written by the unfused CG update (Handle::mf0)
            L.mf = H.dalloc(nv);
            L.dev_bytes += 8 * nv;
        }
        if (!lp.replicated) {
            L.plan = lp.halo;
            L.nsend = (int64_t)lp.halo.send_idx.size();
            if (L.nsend) {
                L.send_idx = H.upload(lp.halo.send_idx);
                L.sendbuf = H.dalloc(L.nsend);
            }
        }
    }
    P.nL = RP.lv.back().ma().nrows;
    P.coarse_inv = H.upload(H.reordered ? H.coarse_inv_perm : H.coarse_inv);
    P.lv.back().dev_bytes += 8 * P.nL * P.nL;
    const int64_t nv0 = P.lv[0].n + P.lv[0].ng;
    void* pp = nullptr;
    ck(cudaMalloc(&pp, sizeof(KState)), "cudaMalloc");
    H.allocs.push_back(pp);
    P.ks = static_cast<KState*>(pp);
    ck(cudaMalloc(&pp, (size_t)H.num_sms * 8 * 16 * sizeof(double)), "cudaMalloc");  // <= 16 dots per reduction
    H.allocs.push_back(pp);
    P.red.partial = static_cast<double*>(pp);
    ck(cudaMalloc(&pp, 64), "cudaMalloc");
    H.allocs.push_back(pp);
    ck(cudaMemset(pp, 0, 64), "memset");
    P.red.ticket = static_cast<unsigned int*>(pp);
    if (H.distributed()) P.red.defer = H.dalloc(3 * kSlot);  // 3 slots: split passes
    P.r = H.dalloc(nv0);
    P.r2 = H.dalloc(nv0);  // fused CG: ping-pong r
    P.z = H.dalloc(nv0);
    P.pa = H.dalloc(nv0);
    P.pb = H.dalloc(nv0);
    P.q = H.dalloc(nv0);
    if (H.distributed()) {
        P.xw = H.dalloc(nv0);
        P.s = H.dalloc(nv0);  // also the precond input buffer
        P.sh = H.dalloc(nv0);
    }
    if (prm.solver == 1) {
        P.rhat = H.dalloc(nv0);
        P.v = H.dalloc(nv0);
        if (!P.s) P.s = H.dalloc(nv0);
        if (!P.sh) P.sh = H.dalloc(nv0);
        P.ph = H.dalloc(nv0);
        P.tv = H.dalloc(nv0);
    }
}

}  // namespace

}  // namespace amgb

// ============================================================ C ABI

using amgb::ck;
using amgb::Handle;

struct amg_hierarchy {
    std::unique_ptr<Handle> h;
};

static amg_status set_error(amg_status st, const std::string& msg) {
    amgb::g_err = msg;
    return st;
}

extern "C" {

void amg_params_default(amg_params* p) {
    if (!p) return;
    std::memset(p, 0, sizeof(*p));
    p->struct_size = sizeof(amg_params);
    p->coarsening = 0;
    p->eps_strong = 0.08;
    p->eps_decay = 0.5;
    p->p_omega = 2.0 / 3.0;
    p->relax = 0;
    p->jacobi_omega = 0.72;
    p->cheb_degree = 5;
    p->cheb_lower = 1.0 / 30.0;
    p->cheb_scaled = 1;
    p->npre = 1;
    p->npost = 1;
    p->coarse_enough = 3000;
    p->max_levels = 30;
    p->dense_max = 20000;
    p->solver = 0;
    p->device = 0;
    p->use_graph = 1;
    p->precision = 0;
    p->gmres_m = 30;
    p->setup_device = 1;
    p->idrs_s = 4;
    p->reorder = 2;
}

const char* amg_last_error(void) { return amgb::g_err.c_str(); }

const char* amg_version(void) {
    return "amgb 0.3 (sm_100a; TMA-staged SELL / SELL-32 / row-block CSR fp64 solve phase; host or GPU SA setup; "
           "NCCL row partition)";
}

static amg_status check_params(const amg_params& p) {
    if (p.struct_size != sizeof(amg_params)) return set_error(AMG_E_INVALID_ARG, "amg_params: struct_size mismatch");
    if (p.coarsening < 0 || p.coarsening > 1) return set_error(AMG_E_INVALID_ARG, "coarsening must be 0 or 1");
    if (p.setup_device < 0 || p.setup_device > 1) return set_error(AMG_E_INVALID_ARG, "setup_device must be 0 or 1");
    if (p.reorder < 0 || p.reorder > 2) return set_error(AMG_E_INVALID_ARG, "reorder must be 0, 1 or 2");
    if (p.relax < 0 || p.relax > 2) return set_error(AMG_E_INVALID_ARG, "relax must be 0, 1 or 2");
    if (p.solver < 0 || p.solver > 3)
        return set_error(AMG_E_INVALID_ARG, "solver must be 0 (cg), 1 (bicgstab), 2 (gmres) or 3 (idrs)");
    if (p.solver == 3 && p.idrs_s != 1 && p.idrs_s != 2 && p.idrs_s != 4 && p.idrs_s != 8)
        return set_error(AMG_E_INVALID_ARG, "IDR(s): s must be 1, 2, 4 or 8");
    if (p.solver == 2 && (p.gmres_m < 1 || p.gmres_m > amgb::kGmresMaxM))
        return set_error(AMG_E_INVALID_ARG, "gmres_m in [1, 64]");
    if (p.npre < 0 || p.npost < 0 || p.npre + p.npost < 1)
        return set_error(AMG_E_INVALID_ARG, "npre, npost >= 0 and npre + npost >= 1");
    if (p.relax == 2 && (p.cheb_degree < 1 || !(p.cheb_lower > 0 && p.cheb_lower < 1)))
        return set_error(AMG_E_INVALID_ARG, "chebyshev: degree >= 1, 0 < lower < 1");
    if (!(p.eps_strong >= 0 && p.eps_strong < 1) || !(p.eps_decay > 0 && p.eps_decay <= 1))
        return set_error(AMG_E_INVALID_ARG, "eps_strong in [0,1), eps_decay in (0,1]");
    if (!(p.p_omega >= 0 && p.p_omega < 2)) return set_error(AMG_E_INVALID_ARG, "p_omega in [0,2)");
    if (p.coarse_enough < 1 || p.max_levels < 1 || p.dense_max < 1)
        return set_error(AMG_E_INVALID_ARG, "coarse_enough, max_levels, dense_max >= 1");
    if (p.precision < 0 || p.precision > 1) return set_error(AMG_E_INVALID_ARG, "precision must be 0 or 1");
    return AMG_OK;
}

// Host hierarchy of the global matrix (Algorithm 1): CSR copy,
// then the GPU or host builder.  Throws SetupError / std exceptions.
static void build_host(amgb::Handle& H, int64_t n, const int64_t* ptr, const int32_t* col, const double* val) {
    using namespace amgb;
    const amg_params& prm = H.prm;
    validate_csr(n, ptr, col);
    Csr A0;
    A0.nrows = A0.ncols = n;
    A0.ptr.resize(n + 1);  // uninitialised: first touch in the parallel copy
    A0.col.resize(ptr[n]);
    A0.val.resize(ptr[n]);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        A0.ptr[i + 1] = ptr[i + 1];
        for (int64_t k = ptr[i]; k < ptr[i + 1]; ++k) {
            A0.col[k] = col[k];
            A0.val[k] = val[k];
        }
    }
    A0.ptr[0] = ptr[0];
    SetupParams sp;
    sp.smoothed = prm.coarsening == 0;
    sp.eps_strong = prm.eps_strong;
    sp.eps_decay = prm.eps_decay;
    sp.p_omega = prm.p_omega;
    sp.relax = prm.relax;
    sp.jacobi_omega = prm.jacobi_omega;
    sp.cheb_degree = prm.cheb_degree;
    sp.cheb_lower = prm.cheb_lower;
    sp.cheb_scaled = prm.cheb_scaled != 0;
    sp.coarse_enough = prm.coarse_enough;
    sp.max_levels = prm.max_levels;
    sp.dense_max = prm.dense_max;
    H.host = prm.setup_device == 1 && prm.device >= 0 ? build_hierarchy_gpu(std::move(A0), sp, prm.device)
                                                      : build_hierarchy(std::move(A0), sp);
    H.meta = level_meta(H.host);
    H.coarse_inv = H.host.coarse_inv;
}

// CUDA context, streams and events of a device handle.
static void device_init(amgb::Handle& H) {
    using namespace amgb;
    const auto tc = std::chrono::steady_clock::now();
    ck(cudaSetDevice(H.prm.device), "cudaSetDevice");
    ck(cudaFree(nullptr), "context");
    if (std::getenv("AMGB_SETUP_TIMING"))
        std::fprintf(stderr, "[setup] CUDA context %.1f ms\n",
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tc).count());
    H.device = H.prm.device;
    ck(cudaDeviceGetAttribute(&H.num_sms, cudaDevAttrMultiProcessorCount, H.prm.device), "attr");
    ck(cudaEventCreate(&H.ev0), "event");
    ck(cudaEventCreate(&H.ev1), "event");
    ck(cudaStreamCreate(&H.own_stream), "stream");  // capture needs a non-legacy stream
    H.stream = H.own_stream;
    if (H.nranks > 1) {  // halo transfers overlap interior rows
        ck(cudaStreamCreateWithFlags(&H.comm_stream, cudaStreamNonBlocking), "comm stream");
        ck(cudaEventCreateWithFlags(&H.ev_pack, cudaEventDisableTiming), "event");
        ck(cudaEventCreateWithFlags(&H.ev_halo, cudaEventDisableTiming), "event");
    }
}

// Upload the host parts (device store, work vectors, Krylov state).
static void device_upload(amgb::Handle& H) {
    using namespace amgb;
    H.parts.resize(H.host_parts.size());
    const auto tu = std::chrono::steady_clock::now();
    for (size_t i = 0; i < H.parts.size(); ++i) upload_part(H, H.host_parts[i], H.parts[i]);
    if (std::getenv("AMGB_SETUP_TIMING"))
        std::fprintf(stderr, "[setup] device store %.1f ms (H2D %.2f GB in %.1f ms)\n",
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tu).count(),
                     H.upload_bytes / 1e9, H.upload_ms);
    if (H.virt) {
        std::vector<double*> ptrs;
        for (auto& p : H.parts) ptrs.push_back(p.red.defer);
        H.d_defer_ptrs = H.upload(ptrs);
    }
    ck(cudaMallocHost(&H.ks_host, sizeof(KState)), "cudaMallocHost");
    H.choose_pdl(H.meta.empty() ? 0 : H.meta[0].rows);
    ck(cudaDeviceSynchronize(), "setup sync");
    if (H.reordered) {
        const int64_t n0 = H.parts[0].lv[0].n;
        for (const auto& q : H.reorder_q) H.dq.push_back(H.upload(q));
        H.dq0 = H.dq[0];
        H.rf = H.dalloc(n0);
        H.rx = H.dalloc(n0);
    }
    H.on_device = true;
}

static amg_status setup_error_status(const std::exception_ptr& ep) {
    using namespace amgb;
    try {
        std::rethrow_exception(ep);
    } catch (const SetupError& e) {
        return set_error((amg_status)e.code, e.msg);
    } catch (const std::bad_alloc&) {
        return set_error(AMG_E_OOM, "host allocation failed during setup");
    } catch (const CudaError& e) {
        return set_error(e.msg.find("out of memory") != std::string::npos ? AMG_E_OOM : (amg_status)e.code, e.msg);
    } catch (const std::exception& e) {
        return set_error(AMG_E_INVALID_ARG, e.what());
    }
    return set_error(AMG_E_INVALID_ARG, "setup failed");
}

// Scattered setup of one NCCL rank: the communicator first
// (with a timeout), then rank 0 alone builds the global hierarchy and the
// partition, and sends every other rank the byte image of its part (pack_part)
// over NCCL; the other ranks never see the global matrix (their ptr / col / val
// may be NULL).  A setup error on rank 0 is broadcast, so every rank returns it.
static amg_status setup_scatter(std::unique_ptr<amgb::Handle> H, int64_t n, const int64_t* ptr, const int32_t* col,
                                const double* val, int rank, int64_t gather_below, const uint8_t* nccl_id,
                                amg_handle* out) {
    using namespace amgb;
    const int nranks = H->nranks;
    Nccl& nc = Nccl::get();
    const char* tr = std::getenv("AMGB_TRANSPORT");
    const bool use_shm = tr && std::string(tr) == "shm";  // test transport (shm.hpp)
    if (!use_shm && !nc.ok) return set_error(AMG_E_NCCL, "NCCL unavailable: " + nc.error);
    H->nccl_timeout = nccl_timeout_s();
    try {
        device_init(*H);
        if (use_shm) {
            try {
                H->shm = std::make_unique<ShmComm>(nccl_id, rank, nranks, H->nccl_timeout);
            } catch (const std::exception& e) {
                return set_error(AMG_E_NCCL, std::string("shm transport: ") + e.what());
            }
        } else {
            const int rc = nccl_comm_init_timeout(&H->nccl, nranks, nccl_id, rank, H->prm.device, H->nccl_timeout);
            if (rc == -2) {
                H->nccl = nullptr;
                return set_error(AMG_E_NCCL, "ncclCommInitRank: the other ranks did not join within " +
                                                 std::to_string((int)H->nccl_timeout) + " s (AMGB_NCCL_TIMEOUT_S)");
            }
            ckn(rc, "ncclCommInitRank");
        }
    } catch (...) {
        return setup_error_status(std::current_exception());
    }
    // status block broadcast by rank 0: [status, bytes for rank 0..nranks-1], message
    constexpr int kMsg = 512;
    const size_t hdr_bytes = (size_t)(1 + nranks) * sizeof(int64_t) + kMsg;
    std::vector<uint8_t> hdr(hdr_bytes, 0);
    auto hdr_i64 = [&](int k) -> int64_t& { return reinterpret_cast<int64_t*>(hdr.data())[k]; };
    std::vector<std::vector<uint8_t>> blobs;
    PartHeader ph;
    RankPart own;
    if (rank == 0) {
        amg_status st = AMG_OK;
        try {
            if (n <= 0 || n > INT32_MAX || !ptr || (ptr[n] > 0 && (!col || !val)))
                throw SetupError{AMG_E_INVALID_ARG, "rank 0 needs the global matrix (n, ptr, col, val)"};
            const auto t0 = std::chrono::steady_clock::now();
            build_host(*H, n, ptr, col, val);
            H->lg = first_replicated_level(H->host, nranks, gather_below);
            H->starts = level_starts(H->host, nranks, H->lg);
            ph.meta = H->meta;
            ph.lg = H->lg;
            ph.starts = H->starts;
            ph.coarse_inv = H->coarse_inv;
            blobs.resize(nranks);
            for (int r = 1; r < nranks; ++r) {
                RankPart rp = build_rank_part(H->host, nranks, r, H->lg, H->starts);
                pack_part(ph, rp, blobs[r]);
            }
            own = build_rank_part(H->host, nranks, 0, H->lg, H->starts);
            if (std::getenv("AMGB_SETUP_TIMING"))
                std::fprintf(stderr, "[setup] rank 0: hierarchy + %d parts %.1f ms\n", nranks,
                             std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
        } catch (...) {
            st = setup_error_status(std::current_exception());
        }
        hdr_i64(0) = st;
        for (int r = 1; r < nranks && st == AMG_OK; ++r) hdr_i64(1 + r) = (int64_t)blobs[r].size();
        if (st != AMG_OK) std::snprintf(reinterpret_cast<char*>(hdr.data() + (1 + nranks) * 8), kMsg, "%s",
                                        g_err.c_str());
    }
    uint8_t* dbuf = nullptr;
    amg_status st = AMG_OK;
    if (H->shm) {  // test transport: the same protocol through host shared memory
        try {
            std::vector<std::vector<uint8_t>> out(nranks), in;
            if (rank == 0)
                for (int r = 0; r < nranks; ++r) out[r] = hdr;
            H->shm_a2a(out, in);
            hdr = in[0];
            if (hdr_i64(0) != AMG_OK) {
                const std::string msg(reinterpret_cast<const char*>(hdr.data() + (1 + nranks) * 8));
                return set_error((amg_status)hdr_i64(0), rank == 0 ? g_err : "rank 0 setup failed: " + msg);
            }
            out.assign(nranks, {});
            if (rank == 0)
                for (int r = 1; r < nranks; ++r) out[r] = std::move(blobs[r]);
            H->shm_a2a(out, in);
            if (rank == 0) {
                H->host_parts.push_back(std::move(own));
            } else {
                RankPart rp;
                unpack_part(in[0].data(), in[0].size(), ph, rp);
                if (rp.rank != rank || rp.nranks != nranks) throw SetupError{AMG_E_INVALID_ARG, "scattered setup: wrong part"};
                H->meta = ph.meta;
                H->lg = ph.lg;
                H->starts = ph.starts;
                H->coarse_inv = ph.coarse_inv;
                H->host_parts.push_back(std::move(rp));
            }
            device_upload(*H);
        } catch (...) {
            return setup_error_status(std::current_exception());
        }
        *out = new amg_hierarchy{std::move(H)};
        return AMG_OK;
    }
    try {
        ck(cudaMalloc(&dbuf, hdr_bytes), "cudaMalloc (scatter)");
        ck(cudaMemcpy(dbuf, hdr.data(), hdr_bytes, cudaMemcpyHostToDevice), "H2D");
        ckn(nc.broadcast(dbuf, dbuf, hdr_bytes, kNcclUint8, 0, H->nccl, H->stream), "ncclBroadcast (setup status)");
        H->sync(H->stream);
        ck(cudaMemcpy(hdr.data(), dbuf, hdr_bytes, cudaMemcpyDeviceToHost), "D2H");
        cudaFree(dbuf);
        dbuf = nullptr;
        if (hdr_i64(0) != AMG_OK) {
            const std::string msg(reinterpret_cast<const char*>(hdr.data() + (1 + nranks) * 8));
            return set_error((amg_status)hdr_i64(0), rank == 0 ? g_err : "rank 0 setup failed: " + msg);
        }
        // rank 0 -> rank r: the part image (one p2p transfer per rank)
        if (rank == 0) {
            size_t mx = 0;
            for (int r = 1; r < nranks; ++r) mx = std::max(mx, blobs[r].size());
            ck(cudaMalloc(&dbuf, std::max<size_t>(mx, 1)), "cudaMalloc (scatter)");
            for (int r = 1; r < nranks; ++r) {
                ck(cudaMemcpy(dbuf, blobs[r].data(), blobs[r].size(), cudaMemcpyHostToDevice), "H2D part");
                ckn(nc.send(dbuf, blobs[r].size(), kNcclUint8, r, H->nccl, H->stream), "ncclSend (part)");
                H->sync(H->stream);
                std::vector<uint8_t>().swap(blobs[r]);
            }
            H->host_parts.push_back(std::move(own));
        } else {
            const size_t bytes = (size_t)hdr_i64(1 + rank);
            std::vector<uint8_t> img(bytes);
            ck(cudaMalloc(&dbuf, std::max<size_t>(bytes, 1)), "cudaMalloc (scatter)");
            ckn(nc.recv(dbuf, bytes, kNcclUint8, 0, H->nccl, H->stream), "ncclRecv (part)");
            H->sync(H->stream);
            ck(cudaMemcpy(img.data(), dbuf, bytes, cudaMemcpyDeviceToHost), "D2H part");
            RankPart rp;
            unpack_part(img.data(), img.size(), ph, rp);
            if (rp.rank != rank || rp.nranks != nranks) throw SetupError{AMG_E_INVALID_ARG, "scattered setup: wrong part"};
            H->meta = ph.meta;
            H->lg = ph.lg;
            H->starts = ph.starts;
            H->coarse_inv = ph.coarse_inv;
            H->host_parts.push_back(std::move(rp));
        }
        if (dbuf) cudaFree(dbuf);
        dbuf = nullptr;
        device_upload(*H);
    } catch (...) {
        if (dbuf) cudaFree(dbuf);
        st = setup_error_status(std::current_exception());
    }
    if (st != AMG_OK) return st;
    *out = new amg_hierarchy{std::move(H)};
    return AMG_OK;
}

// Common setup: host hierarchy, partition, upload.  rank = -1: every part in
// this process (virtual); nranks = 1: single GPU; rank >= 0 on a device: the
// scattered setup above.
static amg_status setup_impl(int64_t n, const int64_t* ptr, const int32_t* col, const double* val,
                             const amg_params* prm_in, int nranks, int rank, int64_t gather_below,
                             const uint8_t* nccl_id, amg_handle* out) {
    using namespace amgb;
    if (!out) return set_error(AMG_E_INVALID_ARG, "out is NULL");
    *out = nullptr;
    if (nranks < 1 || rank < -1 || rank >= nranks) return set_error(AMG_E_INVALID_ARG, "nranks / rank");
    amg_params prm;
    if (prm_in)
        prm = *prm_in;
    else
        amg_params_default(&prm);
    if (amg_status st = check_params(prm)) return st;
    auto H = std::make_unique<Handle>();
    H->prm = prm;
    H->sync_debug = std::getenv("AMGB_SYNC_DEBUG") != nullptr;
    H->nranks = nranks;
    H->virt = nranks > 1 && rank < 0;
    if (nranks > 1 && rank >= 0 && prm.device >= 0)
        return setup_scatter(std::move(H), n, ptr, col, val, rank, gather_below, nccl_id, out);
    if (n <= 0 || n > INT32_MAX || !ptr || (!col && ptr[n] > 0) || (!val && ptr[n] > 0))
        return set_error(AMG_E_INVALID_ARG, "n must be in [1, 2^31) and ptr/col/val non-NULL");
    try {
        const auto t0 = std::chrono::steady_clock::now();
        build_host(*H, n, ptr, col, val);
        const auto t1 = std::chrono::steady_clock::now();
        H->lg = first_replicated_level(H->host, nranks, gather_below);
        H->starts = level_starts(H->host, nranks, H->lg);
        if (nranks == 1) {
            const bool reorder = prm.device >= 0 && H->host.levels.size() > 1 &&
                                 (prm.reorder == 1 ||
                                  (prm.reorder == 2 && gather_sectors_per_entry(H->host.levels[0].A) > 0.5));
            if (reorder) {  // locality reordering of the device store
                std::vector<std::vector<int64_t>> q;
                H->host_parts.push_back(reordered_part(H->host, q, H->coarse_inv_perm));
                H->reordered = true;
                H->reorder_q = std::move(q);
            } else {
                H->host_parts.push_back(build_rank_part(H->host, 1, 0, H->lg, H->starts));
            }
        } else if (rank < 0) {
            for (int r = 0; r < nranks; ++r)
                H->host_parts.push_back(build_rank_part(H->host, nranks, r, H->lg, H->starts));
        } else {  // host-only handle of one rank (device = -1): global setup, own part
            H->host_parts.push_back(build_rank_part(H->host, nranks, rank, H->lg, H->starts));
        }
        if (std::getenv("AMGB_SETUP_TIMING"))
            std::fprintf(stderr, "[setup] hierarchy %.1f ms, partition %.1f ms\n",
                         std::chrono::duration<double, std::milli>(t1 - t0).count(),
                         std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t1).count());
    } catch (...) {
        return setup_error_status(std::current_exception());
    }
    if (prm.device < 0) {
        *out = new amg_hierarchy{std::move(H)};
        return AMG_OK;
    }
    try {
        device_init(*H);
        device_upload(*H);
    } catch (...) {
        cudaGetLastError();
        return setup_error_status(std::current_exception());
    }
    *out = new amg_hierarchy{std::move(H)};
    return AMG_OK;
}

amg_status amg_setup(int64_t n, const int64_t* ptr, const int32_t* col, const double* val,
                     const amg_params* prm_in, amg_handle* out) {
    return setup_impl(n, ptr, col, val, prm_in, 1, 0, 0, nullptr, out);
}

amg_status amg_nccl_unique_id(uint8_t id[128]) {
    if (!id) return set_error(AMG_E_INVALID_ARG, "id is NULL");
    amgb::Nccl& nc = amgb::Nccl::get();
    if (!nc.ok) return set_error(AMG_E_NCCL, "NCCL unavailable: " + nc.error);
    const int r = nc.getUniqueId(id);
    if (r != 0) return set_error(AMG_E_NCCL, "ncclGetUniqueId failed");
    return AMG_OK;
}

amg_status amg_setup_dist(int64_t n, const int64_t* ptr, const int32_t* col, const double* val,
                          const amg_params* prm, const amg_dist* d, amg_handle* out) {
    if (!d) return set_error(AMG_E_INVALID_ARG, "dist descriptor is NULL");
    const bool on_device = !prm || prm->device >= 0;
    if (d->nranks > 1 && d->rank >= 0 && on_device) {  // NCCL mode needs rank 0's unique id
        bool zero = true;
        for (int i = 0; i < 128; ++i) zero &= d->nccl_id[i] == 0;
        if (zero) return set_error(AMG_E_INVALID_ARG, "nccl_id not set (amg_nccl_unique_id on rank 0, then broadcast)");
    }
    // default: replicate a level once it has fewer than 16384 rows per rank (below
    // that, a distributed pass is dominated by its halo-exchange latency)
    const int64_t gb = d->gather_below > 0 ? d->gather_below : (int64_t)16384 * std::max(1, d->nranks);
    return setup_impl(n, ptr, col, val, prm, d->nranks, d->rank, gb, d->nccl_id, out);
}

void amg_destroy(amg_handle h) { delete h; }

static amg_status need_device(amg_handle h) {
    if (!h || !h->h) return set_error(AMG_E_INVALID_ARG, "NULL handle");
    if (!h->h->on_device) return set_error(AMG_E_NO_DEVICE, "host-only handle (params.device = -1)");
    return AMG_OK;
}

amg_status amg_solve(amg_handle h, const double* f, double* x, double tol, int32_t maxiter, int32_t* iters,
                     double* rel) {
    if (amg_status st = need_device(h)) return st;
    if (!f || !x || !iters || !rel || f == x) return set_error(AMG_E_INVALID_ARG, "f, x, iters, rel");
    if (!(tol >= 0) || maxiter < 0) return set_error(AMG_E_INVALID_ARG, "tol >= 0, maxiter >= 0");
    try {
        ck(cudaSetDevice(h->h->device), "cudaSetDevice");
        if (h->h->prm.solver == 2 && h->h->distributed())
            return set_error(AMG_E_INVALID_ARG, "GMRES: single-GPU handles only");
        if (h->h->prm.solver == 3 && h->h->distributed())
            return set_error(AMG_E_INVALID_ARG, "IDR(s): single-GPU handles only");
        return h->h->solve_api(f, x, tol, maxiter, iters, rel);
    } catch (const amgb::CudaError& e) {
        cudaGetLastError();
        return set_error((amg_status)e.code, e.msg);
    }
}

amg_status amg_vector_length(amg_handle h, int64_t* n) {
    if (!h || !h->h || !n) return set_error(AMG_E_INVALID_ARG, "NULL argument");
    const Handle& H = *h->h;
    *n = (H.virt || H.parts.empty()) ? H.meta[0].rows : H.parts[0].lv[0].n;
    return AMG_OK;
}

amg_status amg_solve_host(amg_handle h, const double* f, const double* x0, double* x, double tol,
                          int32_t maxiter, int32_t* iters, double* rel) {
    if (amg_status st = need_device(h)) return st;
    if (!f || !x || !iters || !rel) return set_error(AMG_E_INVALID_ARG, "f, x, iters, rel");
    Handle& H = *h->h;
    const int64_t n = H.virt ? H.meta[0].rows : H.parts[0].lv[0].n;
    try {
        ck(cudaSetDevice(H.device), "cudaSetDevice");
        if (!H.hf) {
            H.hf = H.dalloc(n);
            H.hx = H.dalloc(n);
        }
        ck(cudaMemcpyAsync(H.hf, f, n * sizeof(double), cudaMemcpyHostToDevice, H.stream), "H2D f");
        if (x0)
            ck(cudaMemcpyAsync(H.hx, x0, n * sizeof(double), cudaMemcpyHostToDevice, H.stream), "H2D x0");
        else
            ck(cudaMemsetAsync(H.hx, 0, n * sizeof(double), H.stream), "zero x0");
        amg_status st = H.solve_api(H.hf, H.hx, tol, maxiter, iters, rel);
        ck(cudaMemcpyAsync(x, H.hx, n * sizeof(double), cudaMemcpyDeviceToHost, H.stream), "D2H x");
        H.sync(H.stream);
        return st;
    } catch (const amgb::CudaError& e) {
        cudaGetLastError();
        return set_error((amg_status)e.code, e.msg);
    }
}

amg_status amg_solve_host_stream(amg_handle h, int32_t k, const double* const* f, double* const* x, double tol,
                                 int32_t maxiter, int32_t* iters, double* rel, int32_t* vcycles) {
    if (amg_status st = need_device(h)) return st;
    if (k < 0 || (k > 0 && (!f || !x || !iters || !rel))) return set_error(AMG_E_INVALID_ARG, "k, f, x, iters, rel");
    for (int32_t j = 0; j < k; ++j)
        if (!f[j] || !x[j]) return set_error(AMG_E_INVALID_ARG, "f[j] / x[j] is NULL");
    Handle& H = *h->h;
    const int64_t n = H.virt ? H.meta[0].rows : H.parts[0].lv[0].n;
    const size_t bytes = (size_t)n * sizeof(double);
    cudaStream_t cs = nullptr;
    cudaEvent_t in[2] = {nullptr, nullptr}, out[2] = {nullptr, nullptr}, done = nullptr;
    amg_status first = AMG_OK;
    try {
        ck(cudaSetDevice(H.device), "cudaSetDevice");
        if (!H.sf) {
            H.sf = H.dalloc(n);
            H.sx = H.dalloc(n);
            for (int b = 0; b < 2; ++b) H.sin[b] = H.dalloc(n), H.sout[b] = H.dalloc(n);
        }
        ck(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking), "copy stream");
        for (int b = 0; b < 2; ++b) {
            ck(cudaEventCreateWithFlags(&in[b], cudaEventDisableTiming), "event");
            ck(cudaEventCreateWithFlags(&out[b], cudaEventDisableTiming), "event");
        }
        ck(cudaEventCreateWithFlags(&done, cudaEventDisableTiming), "event");
        if (k > 0) {
            ck(cudaMemcpyAsync(H.sin[0], f[0], bytes, cudaMemcpyHostToDevice, cs), "H2D f");
            ck(cudaEventRecord(in[0], cs), "event");
        }
        for (int32_t j = 0; j < k; ++j) {
            const int b = j & 1;
            // the next system's input streams in while this one is solved (its
            // staging vector was last read at the start of solve j - 1, which
            // returned synchronously)
            if (j + 1 < k) {
                ck(cudaMemcpyAsync(H.sin[b ^ 1], f[j + 1], bytes, cudaMemcpyHostToDevice, cs), "H2D f");
                ck(cudaEventRecord(in[b ^ 1], cs), "event");
            }
            ck(cudaStreamWaitEvent(H.stream, in[b], 0), "wait");
            ck(cudaMemcpyAsync(H.sf, H.sin[b], bytes, cudaMemcpyDeviceToDevice, H.stream), "stage f");
            ck(cudaMemsetAsync(H.sx, 0, bytes, H.stream), "zero x0");
            const amg_status st = H.solve_api(H.sf, H.sx, tol, maxiter, &iters[j], &rel[j]);
            if (vcycles) vcycles[j] = H.stats.vcycles;
            if (st != AMG_OK && first == AMG_OK) first = st;
            if (st < 0) break;
            // the solution leaves through a staging vector, copied out while
            // the next system is solved
            if (j >= 2) ck(cudaStreamWaitEvent(H.stream, out[b], 0), "wait");  // x[j-2] copied out
            ck(cudaMemcpyAsync(H.sout[b], H.sx, bytes, cudaMemcpyDeviceToDevice, H.stream), "stage x");
            ck(cudaEventRecord(done, H.stream), "event");
            ck(cudaStreamWaitEvent(cs, done, 0), "wait");
            ck(cudaMemcpyAsync(x[j], H.sout[b], bytes, cudaMemcpyDeviceToHost, cs), "D2H x");
            ck(cudaEventRecord(out[b], cs), "event");
        }
        ck(cudaStreamSynchronize(cs), "sync");
    } catch (const amgb::CudaError& e) {
        cudaGetLastError();
        first = set_error((amg_status)e.code, e.msg);
    }
    if (cs) cudaStreamSynchronize(cs), cudaStreamDestroy(cs);
    for (int b = 0; b < 2; ++b) {
        if (in[b]) cudaEventDestroy(in[b]);
        if (out[b]) cudaEventDestroy(out[b]);
    }
    if (done) cudaEventDestroy(done);
    return first;
}

amg_status amg_solve_batched(amg_handle h, int32_t k, const double* F, int64_t ldf, double* X, int64_t ldx,
                             double tol, int32_t maxiter, int32_t* iters, double* rel) {
    if (amg_status st = need_device(h)) return st;
    Handle& H = *h->h;
    if (H.distributed()) return set_error(AMG_E_INVALID_ARG, "amg_solve_batched: single-GPU handles only");
    if (H.prm.solver != 0) return set_error(AMG_E_INVALID_ARG, "amg_solve_batched: CG only");
    const int64_t n = H.parts[0].lv[0].n;
    if (k < 1 || k > amgb::kMaxK || !F || !X || !iters || !rel || ldf < n || ldx < n)
        return set_error(AMG_E_INVALID_ARG, "k in [1, 8], F/X/iters/rel non-NULL, ld >= n");
    if (!(tol >= 0) || maxiter < 0) return set_error(AMG_E_INVALID_ARG, "tol >= 0, maxiter >= 0");
    try {
        ck(cudaSetDevice(H.device), "cudaSetDevice");
        if (H.reordered) {  // columns permuted into the stored order and back
            amgb::DevTmp tmp;
            double* Fs = tmp.get<double>(k * n);
            double* Xs = tmp.get<double>(k * n);
            for (int j = 0; j < k; ++j) {
                H.perm_in(F + j * ldf, Fs + j * n);
                H.perm_in(X + j * ldx, Xs + j * n);
            }
            amg_status st;
            if (k <= 2) st = H.solve_batched<2>(k, Fs, n, Xs, n, tol, maxiter, iters, rel);
            else if (k <= 4) st = H.solve_batched<4>(k, Fs, n, Xs, n, tol, maxiter, iters, rel);
            else st = H.solve_batched<8>(k, Fs, n, Xs, n, tol, maxiter, iters, rel);
            for (int j = 0; j < k; ++j) H.perm_out(Xs + j * n, X + j * ldx);
            H.sync(H.stream);
            return st;
        }
        if (k <= 2) return H.solve_batched<2>(k, F, ldf, X, ldx, tol, maxiter, iters, rel);
        if (k <= 4) return H.solve_batched<4>(k, F, ldf, X, ldx, tol, maxiter, iters, rel);
        return H.solve_batched<8>(k, F, ldf, X, ldx, tol, maxiter, iters, rel);
    } catch (const amgb::CudaError& e) {
        cudaGetLastError();
        return set_error((amg_status)e.code, e.msg);
    }
}

amg_status amg_precond_apply(amg_handle h, const double* r, double* z) {
    if (amg_status st = need_device(h)) return st;
    if (!r || !z || r == z) return set_error(AMG_E_INVALID_ARG, "r, z");
    try {
        ck(cudaSetDevice(h->h->device), "cudaSetDevice");
        amgb::Handle& H = *h->h;
        if (H.reordered) {
            H.perm_in(r, H.rf);
            H.precond(H.rf, H.rx);
            H.perm_out(H.rx, z);
        } else {
            H.precond(r, z);
        }
        ck(cudaGetLastError(), "launch");
    } catch (const amgb::CudaError& e) {
        return set_error((amg_status)e.code, e.msg);
    }
    return AMG_OK;
}

amg_status amg_set_stream(amg_handle h, void* stream) {
    if (!h || !h->h) return set_error(AMG_E_INVALID_ARG, "NULL handle");
    // the legacy default stream cannot be captured into a graph: keep the
    // handle's own blocking stream, which is ordered with it implicitly
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : h->h->own_stream;
    if (h->h->stream != s) h->h->drop_graph();
    h->h->stream = s;
    return AMG_OK;
}

amg_status amg_set_profile(amg_handle h, int32_t mask) {
    if (!h || !h->h) return set_error(AMG_E_INVALID_ARG, "NULL handle");
    h->h->prof_mask = mask & 0xff;
    return AMG_OK;
}

amg_status amg_level_count(amg_handle h, int32_t* nlevels) {
    if (!h || !h->h || !nlevels) return set_error(AMG_E_INVALID_ARG, "NULL argument");
    *nlevels = (int32_t)h->h->meta.size();
    return AMG_OK;
}

amg_status amg_level_info_get(amg_handle h, int32_t l, amg_level_info* out) {
    if (!h || !h->h || !out) return set_error(AMG_E_INVALID_ARG, "NULL argument");
    const Handle& H = *h->h;
    if (l < 0 || l >= (int)H.meta.size()) return set_error(AMG_E_INVALID_ARG, "level out of range");
    const auto& hl = H.meta[l];
    const bool coarsest = l == (int)H.meta.size() - 1;
    std::memset(out, 0, sizeof(*out));
    out->rows = hl.rows;
    out->nnz_A = hl.nnz_A;
    out->nnz_P = coarsest ? 0 : hl.nnz_P;
    out->cols_P = coarsest ? 0 : hl.cols_P;
    out->aggregates = coarsest ? 0 : hl.n_agg;
    out->is_coarsest = coarsest;
    out->alg_bytes_vcycle = amgb::level_alg_bytes(hl.rows, hl.nnz_A, out->nnz_P, out->cols_P, H.prm, coarsest);
    if (!H.parts.empty()) {
        out->dev_bytes = H.parts[0].lv[l].dev_bytes;
        out->padded_nnz_A = H.parts[0].lv[l].padA;
        out->dict_slices_A = (int32_t)H.parts[0].lv[l].dictA;
        const auto& L = H.parts[0].lv[l];
        out->padded_nnz_P = coarsest ? 0 : L.P.stored;
        out->padded_nnz_R = coarsest ? 0 : L.R.stored;
        out->sigma_mask = (L.A.sigma ? 1 : 0) | (L.P.sigma ? 2 : 0) | (L.R.sigma ? 4 : 0);
        auto code = [](const amgb::DMat& M, bool none) {
            if (none) return (int)AMG_FMT_NONE;
            return M.fmt == amgb::Fmt::TMA      ? (int)AMG_FMT_TMA
                   : M.fmt == amgb::Fmt::TMACSR ? (int)AMG_FMT_TMACSR
                   : M.fmt == amgb::Fmt::SELL   ? (int)AMG_FMT_SELL
                                                : (int)AMG_FMT_CSR;
        };
        auto vmode = [](const amgb::DMat& M) { return M.vbytes == 1 ? 1 : M.vbytes == 2 ? 2 : 0; };
        out->formats = code(L.A, coarsest && l > 0) | code(L.P, coarsest) << 4 | code(L.R, coarsest) << 8 |
                       vmode(L.A) << 12 | vmode(L.P) << 14 | vmode(L.R) << 16;
    }
    return AMG_OK;
}

static void copy_csr(const amgb::Csr& M, int64_t* p, int32_t* c, double* v) {
    if (p) std::copy(M.ptr.begin(), M.ptr.end(), p);
    if (c) std::copy(M.col.begin(), M.col.end(), c);
    if (v) std::copy(M.val.begin(), M.val.end(), v);
}

amg_status amg_export_level(amg_handle h, int32_t l, const amg_level_export* out) {
    if (!h || !h->h || !out) return set_error(AMG_E_INVALID_ARG, "NULL argument");
    const Handle& H = *h->h;
    if (H.host.levels.empty())
        return set_error(AMG_E_INVALID_ARG, "amg_export_level: this rank holds no global hierarchy (scattered "
                                            "multi-GPU setup: export on rank 0)");
    if (l < 0 || l >= (int)H.host.levels.size()) return set_error(AMG_E_INVALID_ARG, "level out of range");
    const auto& hl = H.host.levels[l];
    const bool coarsest = l == (int)H.host.levels.size() - 1;
    copy_csr(hl.A, out->A_ptr, out->A_col, out->A_val);
    if (!coarsest) {
        copy_csr(hl.P, out->P_ptr, out->P_col, out->P_val);
        copy_csr(hl.R, out->R_ptr, out->R_col, out->R_val);
        if (out->aggregates) std::copy(hl.agg.begin(), hl.agg.end(), out->aggregates);
        if (out->smoother) {
            if (H.prm.relax == 2) {
                out->smoother[0] = hl.lmax;
                out->smoother[1] = hl.lmin;
                out->smoother[2] = hl.cheb_d;
                out->smoother[3] = hl.cheb_c;
            } else {
                std::copy(hl.m.begin(), hl.m.end(), out->smoother);
            }
        }
    } else if (out->coarse_inverse) {
        std::copy(H.host.coarse_inv.begin(), H.host.coarse_inv.end(), out->coarse_inverse);
    }
    return AMG_OK;
}

amg_status amg_solve_stats_get(amg_handle h, amg_solve_stats* out) {
    if (!h || !h->h || !out) return set_error(AMG_E_INVALID_ARG, "NULL argument");
    *out = h->h->stats;
    return AMG_OK;
}

amg_status amg_dist_info(amg_handle h, int32_t* nranks, int32_t* first_replicated, int64_t* row_starts) {
    if (!h || !h->h || !nranks || !first_replicated) return set_error(AMG_E_INVALID_ARG, "NULL argument");
    const Handle& H = *h->h;
    *nranks = H.nranks;
    *first_replicated = H.lg;
    if (row_starts)
        for (int r = 0; r <= H.nranks; ++r) row_starts[r] = H.starts[0][r];
    return AMG_OK;
}

static const amgb::LevelPart* find_part(const Handle& H, int32_t rank, int32_t l) {
    for (const auto& rp : H.host_parts)
        if (rp.rank == rank && l >= 0 && l < (int)rp.lv.size()) return &rp.lv[l];
    return nullptr;
}

amg_status amg_dist_level_info(amg_handle h, int32_t rank, int32_t l, int64_t out[18]) {
    if (!h || !h->h || !out) return set_error(AMG_E_INVALID_ARG, "NULL argument");
    const amgb::LevelPart* lp = find_part(*h->h, rank, l);
    if (!lp) return set_error(AMG_E_INVALID_ARG, "rank/level not held by this handle");
    out[0] = lp->row0;
    out[1] = lp->row1;
    out[2] = lp->halo.nghost;
    out[3] = lp->ma().nnz();
    out[4] = lp->mp().nrows ? lp->mp().nnz() : 0;
    out[5] = lp->mr().nrows ? lp->mr().nnz() : 0;
    out[6] = lp->crow0;
    out[7] = lp->crow1;
    out[8] = lp->replicated;
    out[9] = (int64_t)lp->halo.send_idx.size();
    out[10] = (int64_t)lp->halo.recv_peer.size();
    out[11] = (int64_t)lp->halo.send_peer.size();
    for (int q = 12; q < 18; ++q) out[q] = -1;  // split passes: device handles only
    const amgb::Handle& H = *h->h;
    for (const auto& p : H.parts)
        if (p.rank == rank && l < (int)p.lv.size()) {
            const amgb::DevLevel& L = p.lv[l];
            const amgb::DMat* m[3] = {&L.A, &L.P, &L.R};
            for (int q = 0; q < 3; ++q)
                if (m[q]->split) {
                    out[12 + 2 * q] = m[q]->ib0;
                    out[13 + 2 * q] = m[q]->ib1;
                }
        }
    return AMG_OK;
}

amg_status amg_dist_export(amg_handle h, int32_t rank, int32_t l, const amg_dist_level_export* out) {
    if (!h || !h->h || !out) return set_error(AMG_E_INVALID_ARG, "NULL argument");
    const amgb::LevelPart* lp = find_part(*h->h, rank, l);
    if (!lp) return set_error(AMG_E_INVALID_ARG, "rank/level not held by this handle");
    copy_csr(lp->ma(), out->A_ptr, out->A_col, out->A_val);
    if (lp->mp().nrows) copy_csr(lp->mp(), out->P_ptr, out->P_col, out->P_val);
    if (lp->mr().nrows) copy_csr(lp->mr(), out->R_ptr, out->R_col, out->R_val);
    const auto& hp = lp->halo;
    if (out->ghost_global) std::copy(hp.ghost_global.begin(), hp.ghost_global.end(), out->ghost_global);
    for (size_t k = 0; k < hp.recv_peer.size(); ++k) {
        if (out->recv_peer) out->recv_peer[k] = hp.recv_peer[k];
        if (out->recv_off) out->recv_off[k] = hp.recv_off[k];
        if (out->recv_cnt) out->recv_cnt[k] = hp.recv_cnt[k];
    }
    for (size_t k = 0; k < hp.send_peer.size(); ++k) {
        if (out->send_peer) out->send_peer[k] = hp.send_peer[k];
        if (out->send_off) out->send_off[k] = hp.send_off[k];
        if (out->send_cnt) out->send_cnt[k] = hp.send_cnt[k];
    }
    if (out->send_idx) std::copy(hp.send_idx.begin(), hp.send_idx.end(), out->send_idx);
    return AMG_OK;
}

// Exercise the NCCL transport exactly as the multi-GPU executor calls it (grouped
// send/recv, all-reduce, broadcast, also replayed from a captured CUDA graph) on a
// 1-rank communicator of `device` (send/recv to self).  Checks the dlopen'ed
// entry points and their argument order where only one GPU is available.
amg_status amg_nccl_selftest(int32_t device) {
    using namespace amgb;
    Nccl& nc = Nccl::get();
    if (!nc.ok) return set_error(AMG_E_NCCL, "NCCL unavailable: " + nc.error);
    void* comm = nullptr;
    double* buf = nullptr;
    cudaStream_t s = nullptr;
    cudaGraph_t g = nullptr;
    cudaGraphExec_t ge = nullptr;
    amg_status st = AMG_OK;
    try {
        ck(cudaSetDevice(device), "cudaSetDevice");
        uint8_t id[128];
        ckn(nc.getUniqueId(id), "ncclGetUniqueId");
        ckn(nccl_comm_init(&comm, 1, id, 0), "ncclCommInitRank");
        ck(cudaStreamCreate(&s), "stream");
        const int n = 1000;
        ck(cudaMalloc(&buf, 4 * n * sizeof(double)), "cudaMalloc");
        std::vector<double> h(4 * n);
        for (int i = 0; i < n; ++i) {
            h[i] = i + 0.5;  // send buffer
            h[n + i] = -1;   // recv buffer
            h[2 * n + i] = 2.0 * i;
            h[3 * n + i] = 3.0 * i;
        }
        auto round = [&] {
            ckn(nc.groupStart(), "ncclGroupStart");
            ckn(nc.send(buf, n, kNcclDouble, 0, comm, s), "ncclSend");
            ckn(nc.recv(buf + n, n, kNcclDouble, 0, comm, s), "ncclRecv");
            ckn(nc.groupEnd(), "ncclGroupEnd");
            ckn(nc.allReduce(buf + 2 * n, buf + 2 * n, n, kNcclDouble, kNcclSum, comm, s), "ncclAllReduce");
            ckn(nc.groupStart(), "ncclGroupStart");
            ckn(nc.broadcast(buf + 3 * n, buf + 3 * n, n, kNcclDouble, 0, comm, s), "ncclBroadcast");
            ckn(nc.groupEnd(), "ncclGroupEnd");
        };
        for (int pass = 0; pass < 2 && st == AMG_OK; ++pass) {
            ck(cudaMemcpy(buf, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice), "H2D");
            if (pass == 0) {
                round();
            } else {  // captured into a graph, as the Krylov iterations are
                ck(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal), "capture");
                round();
                ck(cudaStreamEndCapture(s, &g), "end capture");
                ck(cudaGraphInstantiate(&ge, g, 0), "instantiate");
                ck(cudaGraphLaunch(ge, s), "graph launch");
            }
            ck(cudaStreamSynchronize(s), "sync");
            std::vector<double> r(4 * n);
            ck(cudaMemcpy(r.data(), buf, r.size() * sizeof(double), cudaMemcpyDeviceToHost), "D2H");
            for (int i = 0; i < n; ++i)
                if (r[n + i] != h[i] || r[2 * n + i] != h[2 * n + i] || r[3 * n + i] != h[3 * n + i]) {
                    st = set_error(AMG_E_NCCL, "NCCL self-test: wrong data (pass " + std::to_string(pass) + ")");
                    break;
                }
        }
    } catch (const CudaError& e) {
        st = set_error((amg_status)e.code, e.msg);
    }
    if (ge) cudaGraphExecDestroy(ge);
    if (g) cudaGraphDestroy(g);
    if (buf) cudaFree(buf);
    if (s) cudaStreamDestroy(s);
    if (comm && nc.commDestroy) nc.commDestroy(comm);
    return st;
}

amg_status amg_shm_selftest(const uint8_t id[128], int32_t rank, int32_t nranks) {
    using namespace amgb;
    if (!id || nranks < 1 || rank < 0 || rank >= nranks) return set_error(AMG_E_INVALID_ARG, "id, rank, nranks");
    try {
        ShmComm c(id, rank, nranks, nccl_timeout_s());
        // payload rank -> p of round k: (1000 r + 10 p + k) repeated, sizes 0, small, 1 MB
        for (int k = 0; k < 3; ++k) {
            auto len = [&](int r, int p) { return (size_t)(k == 2 ? (1 << 20) : (r + p + k) % 3 == 0 ? 0 : 17 * (r + 1)); };
            std::vector<std::vector<uint8_t>> out(nranks), in;
            for (int p = 0; p < nranks; ++p) out[p].assign(len(rank, p), (uint8_t)(100 * rank + 10 * p + k));
            c.alltoallv(out, in);
            for (int p = 0; p < nranks; ++p) {
                if (in[p].size() != len(p, rank)) return set_error(AMG_E_NCCL, "shm self-test: wrong size");
                for (uint8_t b : in[p])
                    if (b != (uint8_t)(100 * p + 10 * rank + k)) return set_error(AMG_E_NCCL, "shm self-test: wrong data");
            }
        }
        c.barrier();
    } catch (const std::exception& e) {
        return set_error(AMG_E_NCCL, std::string("shm self-test: ") + e.what());
    }
    return AMG_OK;
}

static amg_status level_op_impl(amgb::Handle& H, int32_t l, int32_t op, const double* x, const double* f, double* y);

amg_status amg_level_op(amg_handle h, int32_t l, int32_t op, const double* x, const double* f, double* y) {
    using namespace amgb;
    if (amg_status st = need_device(h)) return st;
    Handle& H = *h->h;
    if (H.distributed()) return set_error(AMG_E_INVALID_ARG, "amg_level_op: single-GPU handles only");
    const int nlev = (int)H.parts[0].lv.size();
    if (l < 0 || l >= nlev) return set_error(AMG_E_INVALID_ARG, "level out of range");
    if (!H.reordered) return level_op_impl(H, l, op, x, f, y);
    // reordered store: the operands' levels (x, f, y) per op, permuted in and out
    int lx = l, ly = l;
    if (op == AMG_OP_SPMV_P) lx = std::min(l + 1, nlev - 1);
    if (op == AMG_OP_SPMV_R) ly = std::min(l + 1, nlev - 1);
    try {
        ck(cudaSetDevice(H.device), "cudaSetDevice");
        DevTmp tmp;
        double* xs = x ? tmp.get<double>(H.parts[0].lv[lx].n) : nullptr;
        double* fs = f ? tmp.get<double>(H.parts[0].lv[l].n) : nullptr;
        double* ys = tmp.get<double>(H.parts[0].lv[ly].n);
        if (x) H.perm_in(x, xs, lx);
        if (f) H.perm_in(f, fs, l);
        const amg_status st = level_op_impl(H, l, op, xs, fs, ys);
        if (st == AMG_OK) H.perm_out(ys, y, ly);
        H.sync(H.stream);
        return st;
    } catch (const amgb::CudaError& e) {
        return set_error((amg_status)e.code, e.msg);
    }
}

static amg_status level_op_impl(amgb::Handle& H, int32_t l, int32_t op, const double* x, const double* f, double* y) {
    using namespace amgb;
    Part& p = H.parts[0];
    const int nlev = (int)p.lv.size();
    if (l < 0 || l >= nlev) return set_error(AMG_E_INVALID_ARG, "level out of range");
    const bool coarsest = l == nlev - 1;
    DevLevel& L = p.lv[l];
    Handle::GSel nogate = [](Part&) { return (const int32_t*)nullptr; };
    try {
        ck(cudaSetDevice(H.device), "cudaSetDevice");
        switch (op) {
            case AMG_OP_SPMV_A:
                if (coarsest && nlev > 1) return set_error(AMG_E_INVALID_ARG, "coarsest A is stored dense");
                H.rows(p, L.A, OpSpmv{x, y}, nullptr, "spmv A");
                break;
            case AMG_OP_SPMV_P:
            case AMG_OP_SPMV_R:
                if (coarsest) return set_error(AMG_E_INVALID_ARG, "no P/R on the coarsest level");
                if (op == AMG_OP_SPMV_P)
                    H.rows(p, L.P, OpSpmv{x, y}, nullptr, "spmv P");
                else
                    H.rows(p, L.R, OpSpmv{x, y}, nullptr, "spmv R");
                break;
            case AMG_OP_RESIDUAL:
                if (coarsest && nlev > 1) return set_error(AMG_E_INVALID_ARG, "coarsest A is stored dense");
                H.rows(p, L.A, OpResidual<0, NoFin>{x, f, y, {}}, nullptr, "residual");
                break;
            case AMG_OP_RELAX:
                if (coarsest) return set_error(AMG_E_INVALID_ARG, "no smoother on the coarsest level");
                if (H.prm.relax == 2) {
                    // one full smoother call: K Chebyshev steps from x (fresh recurrence)
                    double* a = L.x;
                    double* b = L.y;
                    ck(cudaMemcpyAsync(a, x, L.n * sizeof(double), cudaMemcpyDeviceToDevice, H.stream), "copy");
                    for (int k = 0; k < H.prm.cheb_degree; ++k) {
                        double* dst = (k == H.prm.cheb_degree - 1) ? y : b;
                        H.rows(p, L.A,
                               OpCheb<0, NoFin>{a, f, L.diag, L.p, dst, L.cheb_alpha[k], L.cheb_beta[k],
                                                H.prm.cheb_scaled, k == 0, {}},
                               nullptr, "cheb");
                        std::swap(a, b);
                    }
                } else {
                    H.rows(p, L.A, OpRelax<0, NoFin>{x, L.m, f, y, {}}, nullptr, "relax");
                }
                break;
            case AMG_OP_COARSE:
                if (!coarsest) return set_error(AMG_E_INVALID_ARG, "not the coarsest level");
                H.vcycle(l, [f](Part&) { return f; }, [y](Part&) { return y; }, nogate, false);
                break;
            case AMG_OP_VCYCLE:
                H.vcycle(l, [f](Part&) { return f; }, [y](Part&) { return y; }, nogate, false);
                break;
            default:
                return set_error(AMG_E_INVALID_ARG, "unknown op");
        }
        ck(cudaGetLastError(), "launch");
    } catch (const amgb::CudaError& e) {
        return set_error((amg_status)e.code, e.msg);
    }
    return AMG_OK;
}

// ---- amg_level_op_ex: the fused production kernels, one launch each --------
static amg_status level_op_ex_impl(amgb::Handle& H, int32_t l, int32_t op, amg_level_op_args& a) {
    using namespace amgb;
    Part& p = H.parts[0];
    const int nlev = (int)p.lv.size();
    if (l < 0 || l >= nlev - 1) return set_error(AMG_E_INVALID_ARG, "amg_level_op_ex: level must have a coarser level");
    DevLevel& L = p.lv[l];
    DevLevel& Cl = p.lv[l + 1];
    const bool cheb = H.prm.relax == 2;
    try {
        ck(cudaSetDevice(H.device), "cudaSetDevice");
        DevTmp tmp;
        KState* ks = tmp.get<KState>(1);
        double* dot = tmp.get<double>(4);
        KState k0{};
        k0.beta = a.scalar;
        k0.alpha = a.scalar;
        k0.maxiter = 1 << 30;
        ck(cudaMemcpyAsync(ks, &k0, sizeof(KState), cudaMemcpyHostToDevice, H.stream), "ks");
        ck(cudaMemsetAsync(dot, 0, 4 * sizeof(double), H.stream), "memset");
        const FinStore fs{dot, 1};
        bool has_dot = false, has_res = false;
        auto need = [&](bool ok, const char* what) {
            if (!ok) throw CudaError{std::string("amg_level_op_ex: ") + what};
        };
        switch (op) {
            case AMG_OP_RES0:  // a1: t = f - A (m o f)
                need(!cheb && a.in0 && a.out0, "RES0 needs SPAI-0/Jacobi, in0 = f, out0");
                H.rows(p, L.A, OpRes0{L.m, a.in0, a.out0, {}}, nullptr, "res0");
                break;
            case AMG_OP_RES0_MF:  // a1 with mf = m o f given: t = f - A mf
                need(a.in0 && a.in1 && a.out0, "RES0_MF needs in0 = f, in1 = mf, out0");
                H.rows(p, L.A, OpRes0MF{a.in1, a.in0, a.out0, {}}, nullptr, "res0 (mf)");
                break;
            case AMG_OP_RESTRICT_MF:  // a2: f_c = R t, mf_c = m_c o f_c
                need(!cheb && Cl.m && a.in0 && a.out0 && a.out1, "RESTRICT_MF needs a SPAI-0/Jacobi next level");
                H.rows(p, L.R, OpSpmvMF{a.in0, a.out0, Cl.m, a.out1, {}}, nullptr, "restrict (+mf)");
                break;
            case AMG_OP_PROL0:  // a5: x = m o f + P e
                need(!cheb && a.in0 && a.in1 && a.out0, "PROL0 needs SPAI-0/Jacobi, in0 = e, in1 = f, out0");
                H.rows(p, L.P, OpProl0{a.in0, L.m, a.in1, a.out0, {}}, nullptr, "prolong0");
                break;
            case AMG_OP_PROL0_MF:  // a5 with mf given: x = mf + P e
                need(a.in0 && a.in1 && a.out0, "PROL0_MF needs in0 = e, in1 = mf, out0");
                H.rows(p, L.P, OpProl0MF{a.in0, a.in1, a.out0, {}}, nullptr, "prolong0 (mf)");
                break;
            case AMG_OP_PROL_ADD:  // a5 general: x += P e
                need(a.in0 && a.out0, "PROL_ADD needs in0 = e, out0 = x (in/out)");
                H.rows(p, L.P, OpProlAdd{a.in0, a.out0, {}}, nullptr, "prolong");
                break;
            case AMG_OP_RELAX_RHO:  // a6: xo = x + m o (f - A x), (f, xo)
                need(!cheb && a.in0 && a.in1 && a.out0 && a.in0 != a.out0, "RELAX_RHO needs in0 = x, in1 = f, out0");
                H.rows(p, L.A, OpRelax<1, FinStore>{a.in0, L.m, a.in1, a.out0, fs}, nullptr, "relax+dot");
                has_dot = true;
                break;
            case AMG_OP_CHEB_STEP: {  // one Chebyshev step k = scalar, (f, xo)
                const int k = (int)a.scalar;
                need(cheb && k >= 0 && k < H.prm.cheb_degree && a.in0 && a.in1 && a.out0 && a.out1 && a.in0 != a.out0,
                     "CHEB_STEP needs Chebyshev, 0 <= k < degree, in0 = x, in1 = f, out0, out1 = p (in/out)");
                H.rows(p, L.A,
                       OpCheb<1, FinStore>{a.in0, a.in1, L.diag, a.out1, a.out0, L.cheb_alpha[k], L.cheb_beta[k],
                                           H.prm.cheb_scaled, k == 0, fs},
                       nullptr, "cheb+dot");
                has_dot = true;
                break;
            }
            case AMG_OP_CG_DIR:  // a7: p' = z + beta p, q = A p', (p', q)
                need(l == 0 && a.in0 && a.in1 && a.out0 && a.out1, "CG_DIR on level 0: in0 = z, in1 = p, out0, out1");
                H.rows(p, L.A, OpCgDir<FinStore>{a.in0, a.in1, a.out0, a.out1, ks, 0.0, fs}, nullptr, "cg dir");
                has_dot = true;
                break;
            case AMG_OP_CG_UPDATE:  // a8: x += alpha p, r -= alpha q, mf = m o r, |r|
                need(l == 0 && !cheb && a.in0 && a.in1 && a.out0 && a.out1 && a.out2,
                     "CG_UPDATE on level 0 (SPAI-0/Jacobi): in0 = p, in1 = q, out0 = x, out1 = r, out2 = mf");
                H.vec(p, L.n, VCgUpdateMF{a.out0, a.out1, a.in0, a.in1, L.m, a.out2, ks, 0.0, FinCgUpdate{ks}}, nullptr,
                      "cg update (+mf)");
                has_res = true;
                break;
            default:
                return set_error(AMG_E_INVALID_ARG, "amg_level_op_ex: unknown op");
        }
        ck(cudaGetLastError(), "launch");
        if (has_dot) {
            ck(cudaMemcpyAsync(&a.dot, dot, sizeof(double), cudaMemcpyDeviceToHost, H.stream), "D2H");
        } else if (has_res) {
            KState kh{};
            ck(cudaMemcpyAsync(&kh, ks, sizeof(KState), cudaMemcpyDeviceToHost, H.stream), "D2H");
            H.sync(H.stream);
            a.dot = kh.res;
        }
        H.sync(H.stream);  // scratch is freed at scope exit
    } catch (const amgb::CudaError& e) {
        return set_error((amg_status)e.code, e.msg);
    }
    return AMG_OK;
}

amg_status amg_level_op_ex(amg_handle h, int32_t l, int32_t op, amg_level_op_args* a) {
    using namespace amgb;
    if (amg_status st = need_device(h)) return st;
    if (!a) return set_error(AMG_E_INVALID_ARG, "NULL args");
    Handle& H = *h->h;
    if (H.distributed()) return set_error(AMG_E_INVALID_ARG, "amg_level_op_ex: single-GPU handles only");
    const int nlev = (int)H.parts[0].lv.size();
    if (l < 0 || l >= nlev - 1) return set_error(AMG_E_INVALID_ARG, "level out of range");
    if (!H.reordered) return level_op_ex_impl(H, l, op, *a);
    // reordered store: every operand permuted into the stored order of its level
    // (e and the restriction's outputs live on level l+1), outputs permuted back
    const bool coarse_in0 = op == AMG_OP_PROL0 || op == AMG_OP_PROL0_MF || op == AMG_OP_PROL_ADD;
    const bool coarse_out = op == AMG_OP_RESTRICT_MF;
    const int l_in0 = coarse_in0 ? l + 1 : l, l_out = coarse_out ? l + 1 : l;
    try {
        ck(cudaSetDevice(H.device), "cudaSetDevice");
        DevTmp tmp;
        amg_level_op_args b = *a;
        auto in = [&](const double* v, int lv) -> const double* {
            if (!v) return nullptr;
            double* s = tmp.get<double>(H.parts[0].lv[lv].n);
            H.perm_in(v, s, lv);
            return s;
        };
        auto io = [&](double* v, int lv) -> double* {  // outputs that are also read
            if (!v) return nullptr;
            double* s = tmp.get<double>(H.parts[0].lv[lv].n);
            H.perm_in(v, s, lv);
            return s;
        };
        b.in0 = in(a->in0, l_in0);
        b.in1 = in(a->in1, l);
        b.out0 = io(a->out0, l_out);
        b.out1 = io(a->out1, l_out);
        b.out2 = io(a->out2, l);
        const amg_status st = level_op_ex_impl(H, l, op, b);
        if (st == AMG_OK) {
            if (a->out0) H.perm_out(b.out0, a->out0, l_out);
            if (a->out1) H.perm_out(b.out1, a->out1, l_out);
            if (a->out2) H.perm_out(b.out2, a->out2, l);
            a->dot = b.dot;
        }
        H.sync(H.stream);
        return st;
    } catch (const amgb::CudaError& e) {
        return set_error((amg_status)e.code, e.msg);
    }
}

}  // extern "C"
