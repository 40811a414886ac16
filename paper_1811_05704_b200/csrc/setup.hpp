// Host-side hierarchy construction (Algorithm 1) for the
// library.  Runs on the CPU inside amg_setup, as the paper prescribes
// (PAPER.md:163-167); the result is uploaded by hierarchy.cu.
#pragma once
#include <cstdint>
#include <memory>
#include <utility>
#include <string>
#include <vector>

namespace amgb {

// Vectors whose elements are default-initialised (no zero fill): every CSR
// array is completely written by its producer, so the first touch of its pages
// happens in that (often parallel) loop instead of in a serial memset.
template <class T>
struct UninitAlloc : std::allocator<T> {
    template <class U>
    struct rebind {
        using other = UninitAlloc<U>;
    };
    UninitAlloc() = default;
    template <class U>
    UninitAlloc(const UninitAlloc<U>&) {}
    template <class U, class... Args>
    void construct(U* p, Args&&... args) {
        ::new ((void*)p) U(std::forward<Args>(args)...);
    }
    template <class U>
    void construct(U* p) {
        ::new ((void*)p) U;
    }
};
template <class T>
using hvec = std::vector<T, UninitAlloc<T>>;

struct Csr {
    int64_t nrows = 0, ncols = 0;
    hvec<int64_t> ptr;  // nrows + 1
    hvec<int32_t> col;
    hvec<double> val;
    int64_t nnz() const { return ptr.empty() ? 0 : ptr.back(); }
};

struct SetupParams {
    bool smoothed = true;
    double eps_strong = 0.08, eps_decay = 0.5, p_omega = 2.0 / 3.0;
    int relax = 0;  // 0 spai0, 1 damped jacobi, 2 chebyshev
    double jacobi_omega = 0.72;
    int cheb_degree = 5;
    double cheb_lower = 1.0 / 30.0;
    bool cheb_scaled = true;
    int64_t coarse_enough = 3000;
    int max_levels = 30;
    int64_t dense_max = 20000;
};

struct HostLevel {
    Csr A, P, R;                 // P, R empty on the coarsest level
    std::vector<int32_t> agg;    // aggregate of each row (non-coarsest)
    std::vector<int64_t> root;   // root row of each aggregate (ascending: Phase-1 discovery order)
    int64_t n_agg = 0;
    std::vector<double> m;       // SPAI-0 / Jacobi diagonal
    std::vector<double> diag;    // a_ii (Chebyshev scaling)
    double lmax = 0, lmin = 0, cheb_d = 0, cheb_c = 0;
};

struct HostHierarchy {
    std::vector<HostLevel> levels;  // finest first; last one is the coarsest
    std::vector<double> coarse_inv; // row-major A_L^-1
};

// Error codes mirror amg_status.
struct SetupError {
    int code;
    std::string msg;
};

// Validate CSR; throws SetupError.
void validate_csr(int64_t n, const int64_t* ptr, const int32_t* col);

// Individual components (exposed for the C++ unit tests through the C ABI).
void strength(const Csr& A, double eps, std::vector<uint8_t>& strong);
int64_t aggregate(const Csr& A, const std::vector<uint8_t>& strong, std::vector<int32_t>& id,
                  std::vector<int64_t>* root = nullptr);
Csr prolongation(const Csr& A, const std::vector<uint8_t>& strong, const std::vector<int32_t>& id,
                 int64_t n_agg, bool smoothed, double omega);
Csr transpose(const Csr& A);
Csr multiply(const Csr& A, const Csr& B);

HostHierarchy build_hierarchy(Csr A0, const SetupParams& prm);

// The same hierarchy with the numeric steps on CUDA device `device` (gsetup.cu;
// aggregation and the coarse inverse on the host).  Bitwise equal to
// build_hierarchy.
HostHierarchy build_hierarchy_gpu(Csr A0, const SetupParams& prm, int device);

// Coarsest-level check and dense inverse (the tail of both builders).
void finish_hierarchy(HostHierarchy& H, const SetupParams& prm);

}  // namespace amgb
