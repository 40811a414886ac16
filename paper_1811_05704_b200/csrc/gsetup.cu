// GPU setup phase (Algorithm 1): the
// numeric steps of the hierarchy construction -- strength of connection,
// smoothed prolongation, R = P^T, the Galerkin products A P and R (A P), the
// SPAI-0 / Jacobi diagonals and the Chebyshev bound's row sums -- run on the
// device, and so does the greedy aggregation: its sequential Phase 1 (R3) is
// reproduced exactly by dependency propagation rounds (aggregate_dev below).
// The coarsest dense inverse (253 rows at 256^3) stays on the host.
//
// Every device step performs exactly the host's operations in the host's
// order (setup.cpp): one thread per row, sums in ascending column / inner
// index starting from 0.0, and this file is compiled with -fmad=false (the
// host with -ffp-contract=off), so the hierarchy is BITWISE the host's, which
// is bitwise the oracle's (tests/test_gpu_setup.py).  Rows longer than the
// per-thread lists below are rare; such a product is computed by the host
// routine instead (same result by construction).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cub/cub.cuh>
#include <string>
#include <vector>

#include "setup.hpp"

namespace amgb {

namespace {

[[noreturn]] void gfail(int code, const std::string& m) { throw SetupError{code, m}; }

void gck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) gfail(-10, std::string("GPU setup: ") + what + ": " + cudaGetErrorString(e));
}

template <class T>
struct DVec {
    T* p = nullptr;
    int64_t n = 0;
    DVec() = default;
    explicit DVec(int64_t n_) { resize(n_); }
    DVec(const DVec&) = delete;
    DVec& operator=(const DVec&) = delete;
    DVec(DVec&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr, o.n = 0; }
    DVec& operator=(DVec&& o) noexcept {
        if (this != &o) {
            release();
            p = o.p, n = o.n;
            o.p = nullptr, o.n = 0;
        }
        return *this;
    }
    ~DVec() { release(); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr, n = 0;
    }
    void resize(int64_t n_) {
        release();
        n = n_;
        if (n > 0) {
            const cudaError_t e = cudaMalloc(&p, (size_t)n * sizeof(T));
            if (e != cudaSuccess) {
                cudaGetLastError();
                gfail(-6, std::string("GPU setup: cudaMalloc: ") + cudaGetErrorString(e));
            }
        }
    }
    void from(const std::vector<T>& h) {
        resize((int64_t)h.size());
        if (n) gck(cudaMemcpy(p, h.data(), n * sizeof(T), cudaMemcpyHostToDevice), "H2D");
    }
    std::vector<T> to_host() const {
        std::vector<T> h(n);
        if (n) gck(cudaMemcpy(h.data(), p, n * sizeof(T), cudaMemcpyDeviceToHost), "D2H");
        return h;
    }
    // into an uninitialised host vector: pages first touched by all threads,
    // then one copy
    void to_host(hvec<T>& h) const {
        h.resize(n);
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < n; i += 512) h[i] = T{};
        if (n) gck(cudaMemcpy(h.data(), p, n * sizeof(T), cudaMemcpyDeviceToHost), "D2H");
    }
    void from(const hvec<T>& h) {
        resize((int64_t)h.size());
        if (n) gck(cudaMemcpy(p, h.data(), n * sizeof(T), cudaMemcpyHostToDevice), "H2D");
    }
};

struct DCsr {
    int64_t nrows = 0, ncols = 0;
    DVec<int64_t> ptr;
    DVec<int32_t> col;
    DVec<double> val;
    int64_t nnz() const { return col.n; }
};

DCsr upload(const Csr& A) {
    DCsr D;
    D.nrows = A.nrows;
    D.ncols = A.ncols;
    D.ptr.from(A.ptr);
    D.col.from(A.col);
    D.val.from(A.val);
    return D;
}

Csr download(const DCsr& D) {
    Csr A;
    A.nrows = D.nrows;
    A.ncols = D.ncols;
    D.ptr.to_host(A.ptr);
    D.col.to_host(A.col);
    D.val.to_host(A.val);
    if (A.ptr.empty()) A.ptr.assign(1, 0);
    return A;
}

constexpr int kThreads = 256;
int blocks_for(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + kThreads - 1) / kThreads, 1 << 20)); }

#define ROWS_LOOP(i, n) for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (n); i += (int64_t)gridDim.x * blockDim.x)

// d_i = a_ii (0 if absent); first row with a missing / non-positive diagonal -> *bad
__global__ void k_diag(int64_t n, const int64_t* ptr, const int32_t* col, const double* val, double* d,
                       unsigned long long* bad) {
    ROWS_LOOP(i, n) {
        int64_t lo = ptr[i], hi = ptr[i + 1];
        while (lo < hi) {  // lower_bound of i in the row's ascending columns
            const int64_t mid = (lo + hi) / 2;
            if (col[mid] < i) lo = mid + 1;
            else hi = mid;
        }
        const double v = (lo < ptr[i + 1] && col[lo] == i) ? val[lo] : 0.0;
        d[i] = v;
        if (!(v > 0.0)) atomicMin(bad, (unsigned long long)i);
    }
}

// strength (setup.cpp strength(); §8c L1): a_ij^2 > (eps^2 a_ii) a_jj, j != i
__global__ void k_strength(int64_t n, const int64_t* ptr, const int32_t* col, const double* val, const double* d,
                           double eps2, uint8_t* S) {
    ROWS_LOOP(i, n) {
        const double ti = eps2 * d[i];
        for (int64_t k = ptr[i]; k < ptr[i + 1]; ++k) {
            const int32_t j = col[k];
            if (j == i) {
                S[k] = 0;
                continue;
            }
            const double a = val[k];
            S[k] = (a * a > ti * d[j]) ? 1 : 0;
        }
    }
}

// sorted distinct aggregates of {i} u S_i (setup.cpp prolongation(), pass 1)
constexpr int kMaxRow = 256;
__device__ int row_aggs(int64_t i, const int64_t* ptr, const int32_t* col, const uint8_t* S, const int32_t* id,
                        int32_t* ids) {
    int cnt = 0;
    ids[cnt++] = id[i];
    for (int64_t k = ptr[i]; k < ptr[i + 1]; ++k)
        if (S[k]) ids[cnt++] = id[col[k]];
    for (int a = 1; a < cnt; ++a) {  // insertion sort
        const int32_t v = ids[a];
        int b = a - 1;
        while (b >= 0 && ids[b] > v) {
            ids[b + 1] = ids[b];
            --b;
        }
        ids[b + 1] = v;
    }
    int u = cnt ? 1 : 0;
    for (int a = 1; a < cnt; ++a)
        if (ids[a] != ids[u - 1]) ids[u++] = ids[a];
    return u;
}

__global__ void k_p_len(int64_t n, const int64_t* ptr, const int32_t* col, const uint8_t* S, const int32_t* id,
                        int64_t* len) {
    int32_t ids[kMaxRow];
    ROWS_LOOP(i, n) len[i + 1] = row_aggs(i, ptr, col, S, id, ids);
}

// values (setup.cpp prolongation(), pass 2): D_F(i) = a_ii + weak off-diagonals
// (ascending j); P(i,J) = sum over ascending k of w_ii = 1 - omega (k = i,
// id[i] = J) and w_ik = -((omega / D_F(i)) a_ik) (strong k, id[k] = J), from 0.0
__global__ void k_p_fill(int64_t n, const int64_t* ptr, const int32_t* col, const double* val, const uint8_t* S,
                         const int32_t* id, double omega, const int64_t* pptr, int32_t* pcol, double* pval) {
    int32_t ids[kMaxRow];
    const double wii = 1.0 - omega;
    ROWS_LOOP(i, n) {
        double aii = 0.0;
        for (int64_t k = ptr[i]; k < ptr[i + 1]; ++k)
            if (col[k] == i) aii = val[k];
        double df = aii;
        for (int64_t k = ptr[i]; k < ptr[i + 1]; ++k)
            if (col[k] != i && !S[k]) df += val[k];
        const double scale = omega / df;
        const int u = row_aggs(i, ptr, col, S, id, ids);
        const int64_t base = pptr[i];
        for (int t = 0; t < u; ++t) {
            const int32_t J = ids[t];
            double s = 0.0;
            for (int64_t k = ptr[i]; k < ptr[i + 1]; ++k) {
                const int32_t j = col[k];
                if (j == i) {
                    if (id[i] == J) s += wii;
                } else if (S[k] && id[j] == J) {
                    s += -(scale * val[k]);
                }
            }
            pcol[base + t] = J;
            pval[base + t] = s;
        }
    }
}

__global__ void k_tentative(int64_t n, const int32_t* id, int64_t* pptr, int32_t* pcol, double* pval) {
    ROWS_LOOP(i, n) {
        pptr[i + 1] = i + 1;
        pcol[i] = id[i];
        pval[i] = 1.0;
        if (i == 0) pptr[0] = 0;
    }
}

__global__ void k_row_of(int64_t n, const int64_t* ptr, int32_t* rowidx) {
    ROWS_LOOP(i, n) for (int64_t k = ptr[i]; k < ptr[i + 1]; ++k) rowidx[k] = (int32_t)i;
}

__global__ void k_iota(int64_t n, int32_t* v) {
    ROWS_LOOP(i, n) v[i] = (int32_t)i;
}

__global__ void k_count_cols(int64_t nnz, const int32_t* col, int64_t* cnt) {
    ROWS_LOOP(k, nnz) atomicAdd((unsigned long long*)&cnt[col[k] + 1], 1ull);
}

__global__ void k_gather_t(int64_t nnz, const int32_t* perm, const int32_t* rowidx, const double* val, int32_t* tcol,
                           double* tval) {
    ROWS_LOOP(d, nnz) {
        const int32_t e = perm[d];
        tcol[d] = rowidx[e];
        tval[d] = val[e];
    }
}

// C = A B row by row (setup.cpp multiply()): the sorted distinct columns of
// row i, then C(i,J) = 0.0 + sum over ascending k of A(i,k) B(k,J)
constexpr int kMaxC = 512;
__device__ int insert_sorted(int32_t* cols, int m, int32_t J) {  // -1: overflow
    int lo = 0, hi = m;
    while (lo < hi) {
        const int mid = (lo + hi) / 2;
        if (cols[mid] < J) lo = mid + 1;
        else hi = mid;
    }
    if (lo < m && cols[lo] == J) return m;
    if (m == kMaxC) return -1;
    for (int t = m; t > lo; --t) cols[t] = cols[t - 1];
    cols[lo] = J;
    return m + 1;
}

__global__ void k_spgemm_count(int64_t n, const int64_t* aptr, const int32_t* acol, const int64_t* bptr,
                               const int32_t* bcol, int64_t* cnt, int* overflow) {
    int32_t cols[kMaxC];
    ROWS_LOOP(i, n) {
        int m = 0;
        for (int64_t ka = aptr[i]; ka < aptr[i + 1] && m >= 0; ++ka) {
            const int32_t k = acol[ka];
            for (int64_t kb = bptr[k]; kb < bptr[k + 1]; ++kb) {
                m = insert_sorted(cols, m, bcol[kb]);
                if (m < 0) break;
            }
        }
        if (m < 0) {
            *overflow = 1;
            m = 0;
        }
        cnt[i + 1] = m;
    }
}

__global__ void k_spgemm_fill(int64_t n, const int64_t* aptr, const int32_t* acol, const double* aval,
                              const int64_t* bptr, const int32_t* bcol, const double* bval, const int64_t* cptr,
                              int32_t* ccol, double* cval) {
    int32_t cols[kMaxC];
    ROWS_LOOP(i, n) {
        int m = 0;
        for (int64_t ka = aptr[i]; ka < aptr[i + 1]; ++ka) {
            const int32_t k = acol[ka];
            for (int64_t kb = bptr[k]; kb < bptr[k + 1]; ++kb) m = insert_sorted(cols, m, bcol[kb]);
        }
        const int64_t base = cptr[i];
        for (int t = 0; t < m; ++t) {
            ccol[base + t] = cols[t];
            cval[base + t] = 0.0;
        }
        for (int64_t ka = aptr[i]; ka < aptr[i + 1]; ++ka) {
            const int32_t k = acol[ka];
            const double a = aval[ka];
            for (int64_t kb = bptr[k]; kb < bptr[k + 1]; ++kb) {
                const int32_t J = bcol[kb];
                int lo = 0, hi = m;
                while (lo < hi) {
                    const int mid = (lo + hi) / 2;
                    if (cols[mid] < J) lo = mid + 1;
                    else hi = mid;
                }
                cval[base + lo] += a * bval[kb];
            }
        }
    }
}

// smoother data (setup.cpp setup_smoother())
__global__ void k_smoother(int64_t n, const int64_t* ptr, const double* val, const double* d, int relax,
                           double jomega, int cheb_scaled, double* m, double* rowv) {
    ROWS_LOOP(i, n) {
        if (relax == 0) {
            double s = 0.0;
            for (int64_t k = ptr[i]; k < ptr[i + 1]; ++k) s += val[k] * val[k];
            m[i] = d[i] / s;
        } else if (relax == 1) {
            m[i] = jomega / d[i];
        } else {
            double s = 0.0;
            for (int64_t k = ptr[i]; k < ptr[i + 1]; ++k) s += fabs(val[k]);
            if (cheb_scaled) s = s / fabs(d[i]);
            rowv[i] = s;
        }
    }
}

// ---- aggregation on the device (R3; setup.cpp aggregate()) ----------------
// Phase 1 is the sequential greedy scan "i becomes a root iff i and all of S_i
// are unassigned when i is visited; a root claims S_i".  Its outcome has a
// parallel characterisation: j is assigned at time i iff some root r < i has
// j in {r} u S_r, so with D(i) = { r < i : ({i} u S_i) n ({r} u S_r) != {} }
//   i is a root  <=>  every r in D(i) is a non-root,
//   i is not     <=>  some r in D(i) is a root.
// Decisions therefore propagate from lower to higher indices: cnt(i) counts the
// (j, r) paths of D(i) (with multiplicity), a decided non-root r decrements the
// counts of its dependents, a decided root makes its undecided dependents
// non-roots, and a count reaching 0 makes i a root.  Each node is decided once,
// by exactly the rule of the sequential scan, so roots, ids (root rank in
// ascending order), claims and Phase 2 are BITWISE the host's.
constexpr int32_t kUnd = 0, kRoot = 1, kNonRoot = 2;

// strong pattern (j != i, ascending columns) of A: row lengths, then columns
__global__ void k_s_len(int64_t n, const int64_t* ptr, const uint8_t* S, int64_t* sptr) {
    ROWS_LOOP(i, n) {
        int64_t c = 0;
        for (int64_t k = ptr[i]; k < ptr[i + 1]; ++k) c += S[k];
        sptr[i + 1] = c;
    }
}
__global__ void k_s_fill(int64_t n, const int64_t* ptr, const int32_t* col, const uint8_t* S, const int64_t* sptr,
                         int32_t* scol) {
    ROWS_LOOP(i, n) {
        int64_t o = sptr[i];
        for (int64_t k = ptr[i]; k < ptr[i + 1]; ++k)
            if (S[k]) scol[o++] = col[k];
    }
}

// entries of the ascending list c[lo, hi) that are < x
__device__ __forceinline__ int64_t count_below(const int32_t* c, int64_t lo, int64_t hi, int64_t x) {
    int64_t a = lo, b = hi;
    while (a < b) {
        const int64_t m = (a + b) / 2;
        if (c[m] < x) a = m + 1;
        else b = m;
    }
    return a - lo;
}

// cnt(i) = sum over j in {i} u S_i of |{ r in {j} u S^T_j : r < i }|
__global__ void k_agg_count(int64_t n, const int64_t* sptr, const int32_t* scol, const int64_t* tptr,
                            const int32_t* tcol, int32_t* cnt, int32_t* state, int32_t* F, int32_t* fsize) {
    ROWS_LOOP(i, n) {
        int64_t c = count_below(tcol, tptr[i], tptr[i + 1], i);  // j = i
        for (int64_t k = sptr[i]; k < sptr[i + 1]; ++k) {
            const int64_t j = scol[k];
            c += (j < i) + count_below(tcol, tptr[j], tptr[j + 1], i);
        }
        cnt[i] = (int32_t)c;
        if (c == 0) {
            state[i] = kRoot;
            F[atomicAdd(fsize, 1)] = (int32_t)i;
        } else {
            state[i] = kUnd;
        }
    }
}

// one propagation round over the frontier F (nodes decided in the last round)
__global__ void k_agg_round(const int32_t* F, const int32_t* fsize, const int64_t* sptr, const int32_t* scol,
                            const int64_t* tptr, const int32_t* tcol, int32_t* cnt, int32_t* state, int32_t* Fn,
                            int32_t* fnsize) {
    const int32_t m = *fsize;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m; t += (int64_t)gridDim.x * blockDim.x) {
        const int32_t r = F[t];
        const bool root = state[r] == kRoot;
        auto touch = [&](int32_t i) {  // dependent i > r of r
            if (root) {
                if (atomicCAS(&state[i], kUnd, kNonRoot) == kUnd) Fn[atomicAdd(fnsize, 1)] = i;
            } else if (atomicSub(&cnt[i], 1) == 1) {
                if (atomicCAS(&state[i], kUnd, kRoot) == kUnd) Fn[atomicAdd(fnsize, 1)] = i;
            }
        };
        auto visit = [&](int64_t j) {  // i in {j} u S^T_j, i > r
            if (j > r) touch((int32_t)j);
            for (int64_t k = tptr[j] + count_below(tcol, tptr[j], tptr[j + 1], (int64_t)r + 1); k < tptr[j + 1]; ++k)
                touch(tcol[k]);
        };
        visit(r);
        for (int64_t k = sptr[r]; k < sptr[r + 1]; ++k) visit(scol[k]);
    }
}

__global__ void k_agg_flags(int64_t n, const int32_t* state, int32_t* flag, int32_t* und) {
    ROWS_LOOP(i, n) {
        flag[i] = state[i] == kRoot;
        if (state[i] == kUnd) atomicAdd(und, 1);
    }
}

// Phase 1 claims: a root r takes id rank(r) for itself and S_r
__global__ void k_agg_claim(int64_t n, const int32_t* state, const int32_t* rank, const int64_t* sptr,
                            const int32_t* scol, int32_t* id, int64_t* root) {
    ROWS_LOOP(i, n) {
        if (state[i] != kRoot) continue;
        const int32_t a = rank[i];
        id[i] = a;
        root[a] = i;
        for (int64_t k = sptr[i]; k < sptr[i + 1]; ++k) id[scol[k]] = a;
    }
}

// Phase 2 from the Phase-1 snapshot: the strongest aggregated strong
// neighbour, ascending k, strict > (the lowest column wins ties)
__global__ void k_agg_phase2(int64_t n, const int64_t* ptr, const int32_t* col, const double* val, const uint8_t* S,
                             const int32_t* snap, int32_t* id, int32_t* left) {
    ROWS_LOOP(i, n) {
        if (snap[i] >= 0) continue;
        double best = -1.0;
        int32_t pick = -1;
        for (int64_t k = ptr[i]; k < ptr[i + 1]; ++k) {
            if (!S[k]) continue;
            const int32_t j = col[k];
            if (snap[j] < 0) continue;
            const double w = fabs(val[k]);
            if (w > best) {
                best = w;
                pick = snap[j];
            }
        }
        id[i] = pick;
        if (pick < 0) atomicAdd(left, 1);
    }
}

// inclusive prefix sum in place over v[1..n] (v[0] = 0): CSR row pointers
void scan_ptr(DVec<int64_t>& v) {
    const int64_t n = v.n - 1;
    gck(cudaMemset(v.p, 0, sizeof(int64_t)), "memset");
    if (n <= 0) return;
    size_t tmp = 0;
    gck(cub::DeviceScan::InclusiveSum(nullptr, tmp, v.p + 1, v.p + 1, (int)n), "scan size");
    DVec<unsigned char> t((int64_t)tmp);
    gck(cub::DeviceScan::InclusiveSum(t.p, tmp, v.p + 1, v.p + 1, (int)n), "scan");
}

int64_t last_of(const DVec<int64_t>& v) {
    int64_t x = 0;
    gck(cudaMemcpy(&x, v.p + v.n - 1, sizeof(int64_t), cudaMemcpyDeviceToHost), "D2H");
    return x;
}

DCsr transpose_dev(const DCsr& P) {
    DCsr R;
    R.nrows = P.ncols;
    R.ncols = P.nrows;
    const int64_t nnz = P.nnz();
    R.ptr.resize(R.nrows + 1);
    gck(cudaMemset(R.ptr.p, 0, (R.nrows + 1) * sizeof(int64_t)), "memset");
    R.col.resize(nnz);
    R.val.resize(nnz);
    if (nnz == 0) return R;
    k_count_cols<<<blocks_for(nnz), kThreads>>>(nnz, P.col.p, R.ptr.p);
    scan_ptr(R.ptr);
    // stable radix sort of the entries by column: within a column, entries stay
    // in row-major order, i.e. ascending row (the host's sequential fill)
    DVec<int32_t> rowidx(nnz), idx(nnz), keys_out(nnz), perm(nnz);
    k_row_of<<<blocks_for(P.nrows), kThreads>>>(P.nrows, P.ptr.p, rowidx.p);
    k_iota<<<blocks_for(nnz), kThreads>>>(nnz, idx.p);
    int bits = 1;
    while (bits < 31 && (int64_t(1) << bits) < P.ncols) ++bits;
    size_t tmp = 0;
    gck(cub::DeviceRadixSort::SortPairs(nullptr, tmp, P.col.p, keys_out.p, idx.p, perm.p, (int)nnz, 0, bits),
        "sort size");
    DVec<unsigned char> t((int64_t)tmp);
    gck(cub::DeviceRadixSort::SortPairs(t.p, tmp, P.col.p, keys_out.p, idx.p, perm.p, (int)nnz, 0, bits), "sort");
    k_gather_t<<<blocks_for(nnz), kThreads>>>(nnz, perm.p, rowidx.p, P.val.p, R.col.p, R.val.p);
    gck(cudaGetLastError(), "transpose");
    return R;
}

DCsr spgemm_dev(const DCsr& A, const DCsr& B, bool* overflowed) {
    DCsr C;
    C.nrows = A.nrows;
    C.ncols = B.ncols;
    C.ptr.resize(C.nrows + 1);
    DVec<int> of(1);
    gck(cudaMemset(of.p, 0, sizeof(int)), "memset");
    k_spgemm_count<<<blocks_for(A.nrows), kThreads>>>(A.nrows, A.ptr.p, A.col.p, B.ptr.p, B.col.p, C.ptr.p, of.p);
    gck(cudaGetLastError(), "spgemm count");
    int ovf = 0;
    gck(cudaMemcpy(&ovf, of.p, sizeof(int), cudaMemcpyDeviceToHost), "D2H");
    *overflowed = ovf != 0;
    if (ovf) return C;
    scan_ptr(C.ptr);
    const int64_t nnz = last_of(C.ptr);
    C.col.resize(nnz);
    C.val.resize(nnz);
    k_spgemm_fill<<<blocks_for(A.nrows), kThreads>>>(A.nrows, A.ptr.p, A.col.p, A.val.p, B.ptr.p, B.col.p, B.val.p,
                                                     C.ptr.p, C.col.p, C.val.p);
    gck(cudaGetLastError(), "spgemm fill");
    return C;
}

// C = A B on the device, or with the host routine when a row's column list
// exceeds kMaxC (bitwise the same product)
DCsr product(const DCsr& A, const DCsr& B, const Csr* hA, const Csr* hB) {
    bool ovf = false;
    DCsr C = spgemm_dev(A, B, &ovf);
    if (!ovf) return C;
    if (std::getenv("AMGB_SETUP_TIMING")) std::fprintf(stderr, "[gsetup] product row > %d columns: host multiply\n", kMaxC);
    Csr a = hA ? *hA : download(A), b = hB ? *hB : download(B);
    return upload(multiply(a, b));
}

}  // namespace

// Device aggregation (kernels above): ids on the device (did) and on the host,
// roots ascending.  Returns the aggregate count.
int64_t aggregate_dev(const DCsr& dA, const DVec<uint8_t>& S, DVec<int32_t>& did, std::vector<int32_t>& id,
                      std::vector<int64_t>& root, int* rounds_out) {
    const int64_t n = dA.nrows;
    // strong pattern and its transpose
    DCsr Sc;
    Sc.nrows = Sc.ncols = n;
    Sc.ptr.resize(n + 1);
    k_s_len<<<blocks_for(n), kThreads>>>(n, dA.ptr.p, S.p, Sc.ptr.p);
    scan_ptr(Sc.ptr);
    const int64_t ns = last_of(Sc.ptr);
    if (ns >= INT32_MAX) gfail(-1, "GPU aggregation: too many strong connections");
    Sc.col.resize(ns);
    Sc.val.resize(ns);  // unused by the pattern transpose
    k_s_fill<<<blocks_for(n), kThreads>>>(n, dA.ptr.p, dA.col.p, S.p, Sc.ptr.p, Sc.col.p);
    gck(cudaGetLastError(), "strong pattern");
    DCsr St = transpose_dev(Sc);  // rows ascending within each column
    // Phase 1: counts, initial roots, propagation rounds
    DVec<int32_t> cnt(n), state(n), F0(n), F1(n), sizes(2);
    gck(cudaMemset(sizes.p, 0, 2 * sizeof(int32_t)), "memset");
    k_agg_count<<<blocks_for(n), kThreads>>>(n, Sc.ptr.p, Sc.col.p, St.ptr.p, St.col.p, cnt.p, state.p, F0.p,
                                             sizes.p);
    gck(cudaGetLastError(), "agg count");
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int grid = sms * 8;
    int32_t* F[2] = {F0.p, F1.p};
    int rounds = 0;
    for (;;) {
        // a batch of rounds without host synchronisation; an empty frontier
        // makes a round a no-op
        for (int b = 0; b < 16; ++b, ++rounds) {
            const int c = rounds & 1;
            gck(cudaMemsetAsync(sizes.p + (c ^ 1), 0, sizeof(int32_t)), "memset");
            k_agg_round<<<grid, kThreads>>>(F[c], sizes.p + c, Sc.ptr.p, Sc.col.p, St.ptr.p, St.col.p, cnt.p,
                                            state.p, F[c ^ 1], sizes.p + (c ^ 1));
        }
        gck(cudaGetLastError(), "agg round");
        int32_t sz = 0;
        gck(cudaMemcpy(&sz, sizes.p + (rounds & 1), sizeof(int32_t), cudaMemcpyDeviceToHost), "D2H");
        if (sz == 0) break;
        if (rounds > 4 * n + 64) gfail(-1, "GPU aggregation did not converge");
    }
    if (rounds_out) *rounds_out = rounds;
    DVec<int32_t> flag(n), rank(n), und(1);
    gck(cudaMemset(und.p, 0, sizeof(int32_t)), "memset");
    k_agg_flags<<<blocks_for(n), kThreads>>>(n, state.p, flag.p, und.p);
    int32_t h_und = 0;
    gck(cudaMemcpy(&h_und, und.p, sizeof(int32_t), cudaMemcpyDeviceToHost), "D2H");
    if (h_und != 0) gfail(-1, "GPU aggregation left undecided rows");
    size_t tmp = 0;
    gck(cub::DeviceScan::ExclusiveSum(nullptr, tmp, flag.p, rank.p, (int)n), "scan size");
    DVec<unsigned char> t((int64_t)tmp);
    gck(cub::DeviceScan::ExclusiveSum(t.p, tmp, flag.p, rank.p, (int)n), "scan");
    int32_t last_rank = 0, last_flag = 0;
    gck(cudaMemcpy(&last_rank, rank.p + n - 1, sizeof(int32_t), cudaMemcpyDeviceToHost), "D2H");
    gck(cudaMemcpy(&last_flag, flag.p + n - 1, sizeof(int32_t), cudaMemcpyDeviceToHost), "D2H");
    int64_t count = (int64_t)last_rank + last_flag;
    did.resize(n);
    gck(cudaMemset(did.p, 0xff, n * sizeof(int32_t)), "memset");  // -1
    DVec<int64_t> droot(std::max<int64_t>(count, 1));
    k_agg_claim<<<blocks_for(n), kThreads>>>(n, state.p, rank.p, Sc.ptr.p, Sc.col.p, did.p, droot.p);
    // Phase 2 from the snapshot
    DVec<int32_t> snap(n), left(1);
    gck(cudaMemcpy(snap.p, did.p, n * sizeof(int32_t), cudaMemcpyDeviceToDevice), "D2D");
    gck(cudaMemset(left.p, 0, sizeof(int32_t)), "memset");
    k_agg_phase2<<<blocks_for(n), kThreads>>>(n, dA.ptr.p, dA.col.p, dA.val.p, S.p, snap.p, did.p, left.p);
    gck(cudaGetLastError(), "agg phase 2");
    id = did.to_host();
    root.resize(count);
    if (count) gck(cudaMemcpy(root.data(), droot.p, count * sizeof(int64_t), cudaMemcpyDeviceToHost), "D2H");
    int32_t h_left = 0;
    gck(cudaMemcpy(&h_left, left.p, sizeof(int32_t), cudaMemcpyDeviceToHost), "D2H");
    if (h_left) {  // Phase 3 (provably empty, R3): leftovers become singletons in ascending order
        for (int64_t i = 0; i < n; ++i)
            if (id[i] < 0) {
                id[i] = (int32_t)count++;
                root.push_back(i);
            }
        did.from(id);
    }
    return count;
}

HostHierarchy build_hierarchy_gpu(Csr A0, const SetupParams& prm, int device) {
    gck(cudaSetDevice(device), "cudaSetDevice");
    const bool timing = std::getenv("AMGB_SETUP_TIMING") != nullptr;
    auto t_last = std::chrono::steady_clock::now();
    auto lap = [&](const char* what, size_t l) {
        if (!timing) return;
        gck(cudaDeviceSynchronize(), "sync");
        const auto t = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[gsetup] level %zu %-12s %8.1f ms\n", l, what,
                     std::chrono::duration<double, std::milli>(t - t_last).count());
        t_last = t;
    };
    HostHierarchy H;
    H.levels.emplace_back();
    H.levels.back().A = std::move(A0);
    DCsr dA = upload(H.levels[0].A);
    lap("upload A0", 0);
    double eps = prm.eps_strong;
    bool prev_slow = false;
    for (;;) {
        HostLevel& L = H.levels.back();
        const int64_t n = L.A.nrows;
        const size_t lv = H.levels.size() - 1;
        if (!(n > prm.coarse_enough && static_cast<int>(H.levels.size()) < prm.max_levels)) break;
        // diagonal check + strength
        DVec<double> d(n);
        DVec<unsigned long long> bad(1);
        const unsigned long long none = ~0ull;
        gck(cudaMemcpy(bad.p, &none, sizeof(none), cudaMemcpyHostToDevice), "H2D");
        k_diag<<<blocks_for(n), kThreads>>>(n, dA.ptr.p, dA.col.p, dA.val.p, d.p, bad.p);
        unsigned long long b = 0;
        gck(cudaMemcpy(&b, bad.p, sizeof(b), cudaMemcpyDeviceToHost), "D2H");
        if (b != none) gfail(-3, "row " + std::to_string(b) + ": diagonal is missing or not positive");
        DVec<uint8_t> S(dA.nnz());
        k_strength<<<blocks_for(n), kThreads>>>(n, dA.ptr.p, dA.col.p, dA.val.p, d.p, eps * eps, S.p);
        gck(cudaGetLastError(), "strength");
        lap("strength", lv);
        // aggregation (R3): on the device (AMGB_HOST_AGGREGATE=1: the host routine)
        std::vector<int32_t> id;
        std::vector<int64_t> root;
        DVec<int32_t> did;
        std::vector<uint8_t> Sh;
        int64_t cnt = 0;
        if (std::getenv("AMGB_HOST_AGGREGATE")) {
            Sh = S.to_host();
            cnt = aggregate(L.A, Sh, id, &root);
            did.from(id);
        } else {
            int rounds = 0;
            cnt = aggregate_dev(dA, S, did, id, root, &rounds);
            if (timing) std::fprintf(stderr, "[gsetup] level %zu aggregation: %d propagation rounds\n", lv, rounds);
        }
        lap("aggregate", lv);
        const bool slow = static_cast<double>(cnt) > 0.95 * static_cast<double>(n);
        if (cnt == n || (slow && prev_slow)) break;
        prev_slow = slow;
        // prolongation
        DCsr dP;
        int64_t lmax = 0;
        for (int64_t i = 0; i < n; ++i) lmax = std::max<int64_t>(lmax, L.A.ptr[i + 1] - L.A.ptr[i]);
        if (!prm.smoothed) {
            dP.nrows = n;
            dP.ncols = cnt;
            dP.ptr.resize(n + 1);
            dP.col.resize(n);
            dP.val.resize(n);
            k_tentative<<<blocks_for(n), kThreads>>>(n, did.p, dP.ptr.p, dP.col.p, dP.val.p);
        } else if (lmax < kMaxRow) {
            dP.nrows = n;
            dP.ncols = cnt;
            dP.ptr.resize(n + 1);
            k_p_len<<<blocks_for(n), kThreads>>>(n, dA.ptr.p, dA.col.p, S.p, did.p, dP.ptr.p);
            scan_ptr(dP.ptr);
            const int64_t pn = last_of(dP.ptr);
            dP.col.resize(pn);
            dP.val.resize(pn);
            k_p_fill<<<blocks_for(n), kThreads>>>(n, dA.ptr.p, dA.col.p, dA.val.p, S.p, did.p, prm.p_omega, dP.ptr.p,
                                                  dP.col.p, dP.val.p);
        } else {  // a row longer than the per-thread list: the host routine
            if (Sh.empty()) Sh = S.to_host();
            dP = upload(prolongation(L.A, Sh, id, cnt, prm.smoothed, prm.p_omega));
        }
        gck(cudaGetLastError(), "prolongation");
        lap("P", lv);
        DCsr dR = transpose_dev(dP);
        lap("R=P^T", lv);
        L.P = download(dP);
        L.R = download(dR);
        L.agg = std::move(id);
        L.root = std::move(root);
        L.n_agg = cnt;
        lap("download P,R", lv);
        DCsr dAP = product(dA, dP, &L.A, &L.P);
        lap("AP", lv);
        DCsr dAc = product(dR, dAP, &L.R, nullptr);
        dAP = DCsr();
        lap("R(AP)", lv);
        // smoother data
        {
            DVec<double> m(prm.relax <= 1 ? n : 0), rowv(prm.relax == 2 ? n : 0);
            k_smoother<<<blocks_for(n), kThreads>>>(n, dA.ptr.p, dA.val.p, d.p, prm.relax, prm.jacobi_omega,
                                                    prm.cheb_scaled ? 1 : 0, m.p, rowv.p);
            gck(cudaGetLastError(), "smoother");
            L.diag = d.to_host();
            if (prm.relax <= 1) {
                L.m = m.to_host();
            } else {
                const std::vector<double> rv = rowv.to_host();
                double lm = 0.0;
                for (int64_t i = 0; i < n; ++i) lm = std::max(lm, rv[i]);
                L.lmax = lm;
                L.lmin = lm * prm.cheb_lower;
                L.cheb_d = (L.lmax + L.lmin) / 2.0;
                L.cheb_c = (L.lmax - L.lmin) / 2.0;
            }
        }
        lap("smoother", lv);
        H.levels.emplace_back();
        H.levels.back().A = download(dAc);
        dA = std::move(dAc);
        lap("download Ac", lv);
        eps *= prm.eps_decay;
    }
    dA = DCsr();
    finish_hierarchy(H, prm);
    lap("coarse inv", H.levels.size() - 1);
    return H;
}

}  // namespace amgb
