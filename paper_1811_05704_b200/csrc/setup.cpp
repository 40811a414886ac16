// Host hierarchy construction of the library (Algorithm 1).
//
// This is the product's own implementation of the setup; it shares no code with
// oracle/ (which the tests compare it against).  Both follow DESIGN.md §3:
//   strength      a_ij^2 > (eps_l^2 a_ii) a_jj, eps_l = eps * decay^l     (R1, §8c L1)
//   aggregation   3-phase greedy, Phase-2 snapshot, ties -> lowest column  (§8c L2)
//   prolongation  P = (I - w D_F^-1 A_F) Pt, weak entries lumped on D_F     (§8c L4-L6)
//   Galerkin      A_c = R (A P), R = P^T, ascending inner-index sums      (§8c L7, L8)
// All floating-point sums run in ascending index order and this file is compiled
// with -ffp-contract=off, so the values are reproducible bit for bit and
// independent of the OpenMP thread count (every parallel loop is over
// independent rows).
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include "setup.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>

#ifdef _OPENMP
#include <omp.h>
#endif

namespace amgb {

namespace {

[[noreturn]] void fail(int code, const std::string& m) { throw SetupError{code, m}; }

// Position of the diagonal entry of each row (-1 if absent).
std::vector<int64_t> diag_positions(const Csr& A) {
    std::vector<int64_t> pos(A.nrows, -1);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < A.nrows; ++i) {
        const int32_t* b = A.col.data() + A.ptr[i];
        const int32_t* e = A.col.data() + A.ptr[i + 1];
        const int32_t* it = std::lower_bound(b, e, static_cast<int32_t>(i));
        if (it != e && *it == i) pos[i] = A.ptr[i] + (it - b);
    }
    return pos;
}

int num_threads() {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

int thread_id() {
#ifdef _OPENMP
    return omp_get_thread_num();
#else
    return 0;
#endif
}

}  // namespace

void validate_csr(int64_t n, const int64_t* ptr, const int32_t* col) {
    if (ptr[0] != 0) fail(-2, "CSR: ptr[0] must be 0");
    // parallel scan for the first bad row, then the message from a serial check of it
    int64_t first_bad = n;
#pragma omp parallel for schedule(static) reduction(min : first_bad)
    for (int64_t i = 0; i < n; ++i) {
        bool bad = ptr[i + 1] < ptr[i];
        for (int64_t k = ptr[i]; !bad && k < ptr[i + 1]; ++k)
            bad = col[k] < 0 || col[k] >= n || (k > ptr[i] && col[k] <= col[k - 1]);
        if (bad && i < first_bad) first_bad = i;
    }
    if (first_bad < n) {
        const int64_t i = first_bad;
        if (ptr[i + 1] < ptr[i]) fail(-2, "CSR: row " + std::to_string(i) + ": ptr decreases");
        for (int64_t k = ptr[i]; k < ptr[i + 1]; ++k) {
            if (col[k] < 0 || col[k] >= n)
                fail(-2, "CSR: row " + std::to_string(i) + ": column " + std::to_string(col[k]) +
                             " out of range");
            if (k > ptr[i] && col[k] <= col[k - 1])
                fail(-2, "CSR: row " + std::to_string(i) + ": columns not strictly increasing");
        }
    }
    if (ptr[n] > INT32_MAX * 8LL) fail(-1, "matrix too large");
}

// Strength of connection (§8c L1): off-diagonal (i,j) is strong iff
// a_ij * a_ij > (eps^2 * a_ii) * a_jj.  Diagonal entries are never flagged.
void strength(const Csr& A, double eps, std::vector<uint8_t>& strong) {
    const auto dpos = diag_positions(A);
    std::vector<double> d(A.nrows);
    for (int64_t i = 0; i < A.nrows; ++i) {
        double v = dpos[i] >= 0 ? A.val[dpos[i]] : 0.0;
        if (!(v > 0.0)) fail(-3, "row " + std::to_string(i) + ": diagonal is missing or not positive");
        d[i] = v;
    }
    const double eps2 = eps * eps;
    strong.assign(A.nnz(), 0);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < A.nrows; ++i) {
        const double ti = eps2 * d[i];
        for (int64_t k = A.ptr[i]; k < A.ptr[i + 1]; ++k) {
            const int32_t j = A.col[k];
            if (j == i) continue;
            const double a = A.val[k];
            strong[k] = (a * a > ti * d[j]) ? 1 : 0;
        }
    }
}

// Greedy aggregation (§8c L2).  Returns the aggregate count.
int64_t aggregate(const Csr& A, const std::vector<uint8_t>& strong, std::vector<int32_t>& id,
                  std::vector<int64_t>* root) {
    const int64_t n = A.nrows;
    id.assign(n, -1);
    if (root) root->clear();
    int64_t next = 0;
    // Phase 1 (sequential by definition: later roots depend on earlier ones)
    for (int64_t i = 0; i < n; ++i) {
        if (id[i] >= 0) continue;
        bool free_nbhd = true;
        for (int64_t k = A.ptr[i]; k < A.ptr[i + 1] && free_nbhd; ++k)
            if (strong[k] && id[A.col[k]] >= 0) free_nbhd = false;
        if (!free_nbhd) continue;
        const int32_t a = static_cast<int32_t>(next++);
        id[i] = a;
        if (root) root->push_back(i);
        for (int64_t k = A.ptr[i]; k < A.ptr[i + 1]; ++k)
            if (strong[k]) id[A.col[k]] = a;
    }
    // Phase 2: join the strongest aggregated strong neighbour of the Phase-1
    // state (rows are independent given the snapshot).
    const std::vector<int32_t> phase1 = id;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        if (phase1[i] >= 0) continue;
        double best = -1.0;
        int32_t pick = -1;
        for (int64_t k = A.ptr[i]; k < A.ptr[i + 1]; ++k) {
            if (!strong[k]) continue;
            const int32_t j = A.col[k];
            if (phase1[j] < 0) continue;
            const double w = std::fabs(A.val[k]);
            if (w > best) {  // strict: the lowest column wins ties
                best = w;
                pick = phase1[j];
            }
        }
        id[i] = pick;
    }
    // Phase 3: leftovers become singletons (provably empty; kept for safety).
    for (int64_t i = 0; i < n; ++i)
        if (id[i] < 0) {
            id[i] = static_cast<int32_t>(next++);
            if (root) root->push_back(i);
        }
    return next;
}

// Tentative (smoothed = false) or smoothed prolongation (§8c L3-L6).
Csr prolongation(const Csr& A, const std::vector<uint8_t>& strong, const std::vector<int32_t>& id,
                 int64_t n_agg, bool smoothed, double omega) {
    const int64_t n = A.nrows;
    Csr P;
    P.nrows = n;
    P.ncols = n_agg;
    P.ptr.assign(n + 1, 0);
    if (!smoothed) {
        P.col.resize(n);
        P.val.assign(n, 1.0);
        for (int64_t i = 0; i < n; ++i) {
            P.ptr[i + 1] = i + 1;
            P.col[i] = id[i];
        }
        return P;
    }
    // pass 1: distinct aggregates of {i} u S_i per row
    std::vector<int32_t> len(n);
#pragma omp parallel
    {
        std::vector<int32_t> ids;
#pragma omp for schedule(static)
        for (int64_t i = 0; i < n; ++i) {
            ids.clear();
            ids.push_back(id[i]);
            for (int64_t k = A.ptr[i]; k < A.ptr[i + 1]; ++k)
                if (strong[k]) ids.push_back(id[A.col[k]]);
            std::sort(ids.begin(), ids.end());
            len[i] = static_cast<int32_t>(std::unique(ids.begin(), ids.end()) - ids.begin());
        }
    }
    for (int64_t i = 0; i < n; ++i) P.ptr[i + 1] = P.ptr[i] + len[i];
    P.col.resize(P.ptr[n]);
    P.val.resize(P.ptr[n]);
    // pass 2: values.  D_F(i) = a_ii + sum of weak off-diagonals (ascending j);
    // P(i,J) = sum over k in {i} u S_i with id[k] = J, ascending k, of
    //          w_ii = 1 - omega,  w_ik = -(omega / D_F(i)) * a_ik.
    const double wii = 1.0 - omega;
#pragma omp parallel
    {
        std::vector<int32_t> ids;
#pragma omp for schedule(static)
        for (int64_t i = 0; i < n; ++i) {
            double aii = 0.0;
            for (int64_t k = A.ptr[i]; k < A.ptr[i + 1]; ++k)
                if (A.col[k] == i) aii = A.val[k];
            double df = aii;
            for (int64_t k = A.ptr[i]; k < A.ptr[i + 1]; ++k)
                if (A.col[k] != i && !strong[k]) df += A.val[k];
            const double scale = omega / df;
            ids.clear();
            ids.push_back(id[i]);
            for (int64_t k = A.ptr[i]; k < A.ptr[i + 1]; ++k)
                if (strong[k]) ids.push_back(id[A.col[k]]);
            std::sort(ids.begin(), ids.end());
            ids.erase(std::unique(ids.begin(), ids.end()), ids.end());
            const int64_t base = P.ptr[i];
            for (size_t t = 0; t < ids.size(); ++t) {
                const int32_t J = ids[t];
                double s = 0.0;
                for (int64_t k = A.ptr[i]; k < A.ptr[i + 1]; ++k) {
                    const int32_t j = A.col[k];
                    if (j == i) {
                        if (id[i] == J) s += wii;
                    } else if (strong[k] && id[j] == J) {
                        s += -(scale * A.val[k]);
                    }
                }
                P.col[base + t] = J;
                P.val[base + t] = s;
            }
        }
    }
    return P;
}

Csr transpose(const Csr& A) {
    Csr T;
    T.nrows = A.ncols;
    T.ncols = A.nrows;
    T.ptr.assign(T.nrows + 1, 0);
    for (int64_t k = 0; k < A.nnz(); ++k) T.ptr[A.col[k] + 1]++;
    std::partial_sum(T.ptr.begin(), T.ptr.end(), T.ptr.begin());
    T.col.resize(A.nnz());
    T.val.resize(A.nnz());
    std::vector<int64_t> fill(T.ptr.begin(), T.ptr.end() - 1);
    for (int64_t i = 0; i < A.nrows; ++i)
        for (int64_t k = A.ptr[i]; k < A.ptr[i + 1]; ++k) {
            const int64_t d = fill[A.col[k]]++;
            T.col[d] = static_cast<int32_t>(i);
            T.val[d] = A.val[k];
        }
    return T;
}

// Row-wise sparse product C = A B.  Each C(i,J) accumulates A(i,k) B(k,J) over
// ascending k starting from 0.0; the pattern keeps structural zeros; columns
// ascending.  Parallel over rows with per-thread dense accumulators.
Csr multiply(const Csr& A, const Csr& B) {
    const int64_t n = A.nrows, m = B.ncols;
    Csr C;
    C.nrows = n;
    C.ncols = m;
    C.ptr.assign(n + 1, 0);
    const int nt = num_threads();
    std::vector<std::vector<int64_t>> marks(nt);
    // symbolic
#pragma omp parallel
    {
        auto& mark = marks[thread_id()];
        mark.assign(m, -1);
#pragma omp for schedule(dynamic, 1024)
        for (int64_t i = 0; i < n; ++i) {
            int64_t cnt = 0;
            for (int64_t ka = A.ptr[i]; ka < A.ptr[i + 1]; ++ka) {
                const int32_t k = A.col[ka];
                for (int64_t kb = B.ptr[k]; kb < B.ptr[k + 1]; ++kb) {
                    const int32_t J = B.col[kb];
                    if (mark[J] != i) {
                        mark[J] = i;
                        ++cnt;
                    }
                }
            }
            C.ptr[i + 1] = cnt;
        }
    }
    std::partial_sum(C.ptr.begin(), C.ptr.end(), C.ptr.begin());
    C.col.resize(C.ptr[n]);
    C.val.resize(C.ptr[n]);
    // numeric
#pragma omp parallel
    {
        auto& mark = marks[thread_id()];
        std::fill(mark.begin(), mark.end(), -1);
        std::vector<double> acc(m);
#pragma omp for schedule(dynamic, 1024)
        for (int64_t i = 0; i < n; ++i) {
            int32_t* out = C.col.data() + C.ptr[i];
            int64_t cnt = 0;
            for (int64_t ka = A.ptr[i]; ka < A.ptr[i + 1]; ++ka) {
                const int32_t k = A.col[ka];
                const double a = A.val[ka];
                for (int64_t kb = B.ptr[k]; kb < B.ptr[k + 1]; ++kb) {
                    const int32_t J = B.col[kb];
                    if (mark[J] != i) {
                        mark[J] = i;
                        acc[J] = 0.0;
                        out[cnt++] = J;
                    }
                    acc[J] += a * B.val[kb];
                }
            }
            std::sort(out, out + cnt);
            double* vout = C.val.data() + C.ptr[i];
            for (int64_t t = 0; t < cnt; ++t) vout[t] = acc[out[t]];
        }
    }
    return C;
}

namespace {

// Smoother data (§8c).
void setup_smoother(HostLevel& L, const SetupParams& prm) {
    const Csr& A = L.A;
    const int64_t n = A.nrows;
    const auto dpos = diag_positions(A);
    L.diag.resize(n);
    for (int64_t i = 0; i < n; ++i) L.diag[i] = dpos[i] >= 0 ? A.val[dpos[i]] : 0.0;
    if (prm.relax == 0 || prm.relax == 1) {
        L.m.resize(n);
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < n; ++i) {
            if (prm.relax == 0) {  // SPAI-0: a_ii / sum_j a_ij^2
                double s = 0.0;
                for (int64_t k = A.ptr[i]; k < A.ptr[i + 1]; ++k) s += A.val[k] * A.val[k];
                L.m[i] = L.diag[i] / s;
            } else {  // damped Jacobi: omega / a_ii
                L.m[i] = prm.jacobi_omega / L.diag[i];
            }
        }
    } else {  // Chebyshev: Gershgorin bound of D^-1 A (or A)
        double lmax = 0.0;
        for (int64_t i = 0; i < n; ++i) {
            double s = 0.0;
            for (int64_t k = A.ptr[i]; k < A.ptr[i + 1]; ++k) s += std::fabs(A.val[k]);
            if (prm.cheb_scaled) s = s / std::fabs(L.diag[i]);
            lmax = std::max(lmax, s);
        }
        L.lmax = lmax;
        L.lmin = lmax * prm.cheb_lower;
        L.cheb_d = (L.lmax + L.lmin) / 2.0;
        L.cheb_c = (L.lmax - L.lmin) / 2.0;
    }
}

// Dense inverse of the coarsest matrix via LU with partial pivoting
// (the V-cycle applies A_L^-1 as a GEMV on the device, §8c).
std::vector<double> dense_inverse(const Csr& A) {
    const int64_t n = A.nrows;
    std::vector<double> lu(n * n, 0.0);
    double amax = 0.0;
    for (int64_t i = 0; i < n; ++i)
        for (int64_t k = A.ptr[i]; k < A.ptr[i + 1]; ++k) {
            lu[i * n + A.col[k]] = A.val[k];
            amax = std::max(amax, std::fabs(A.val[k]));
        }
    std::vector<int64_t> perm(n);
    std::iota(perm.begin(), perm.end(), 0);
    for (int64_t k = 0; k < n; ++k) {
        int64_t p = k;
        double best = std::fabs(lu[k * n + k]);
        for (int64_t i = k + 1; i < n; ++i)
            if (std::fabs(lu[i * n + k]) > best) {
                best = std::fabs(lu[i * n + k]);
                p = i;
            }
        if (best == 0.0 || best < 1e-14 * amax)
            fail(-4, "coarsest level is singular (pivot " + std::to_string(best) + ")");
        if (p != k) {
            std::swap_ranges(lu.begin() + k * n, lu.begin() + (k + 1) * n, lu.begin() + p * n);
            std::swap(perm[k], perm[p]);
        }
        const double piv = lu[k * n + k];
#pragma omp parallel for schedule(static) if (n - k > 256)
        for (int64_t i = k + 1; i < n; ++i) {
            const double l = lu[i * n + k] / piv;
            lu[i * n + k] = l;
            double* ri = &lu[i * n];
            const double* rk = &lu[k * n];
            for (int64_t j = k + 1; j < n; ++j) ri[j] -= l * rk[j];
        }
    }
    if (std::getenv("AMGB_SETUP_TIMING")) std::fprintf(stderr, "[setup] coarse LU done (n = %lld)\n", (long long)n);
    // inverse: solve L U X = P I for all columns at once, row by row, in blocks
    // of columns: element (i, c) sees exactly the operations of a column-by-
    // column substitution (ascending j, multiply then subtract), but the inner
    // loop runs over contiguous columns (vectorisable, no reduction chain)
    std::vector<double> inv(n * n);
    constexpr int64_t kCols = 64;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t c0 = 0; c0 < n; c0 += kCols) {
        const int64_t w = std::min(kCols, n - c0);
        std::vector<double> X(n * w);  // rows of the column block
        for (int64_t i = 0; i < n; ++i)
            for (int64_t c = 0; c < w; ++c) X[i * w + c] = (perm[i] == c0 + c) ? 1.0 : 0.0;
        for (int64_t i = 0; i < n; ++i) {  // forward: unit lower L
            double* xi = &X[i * w];
            for (int64_t j = 0; j < i; ++j) {
                const double l = lu[i * n + j];
                const double* xj = &X[j * w];
                for (int64_t c = 0; c < w; ++c) xi[c] -= l * xj[c];
            }
        }
        for (int64_t i = n - 1; i >= 0; --i) {  // backward: U
            double* xi = &X[i * w];
            for (int64_t j = i + 1; j < n; ++j) {
                const double u = lu[i * n + j];
                const double* xj = &X[j * w];
                for (int64_t c = 0; c < w; ++c) xi[c] -= u * xj[c];
            }
            const double d = lu[i * n + i];
            for (int64_t c = 0; c < w; ++c) xi[c] = xi[c] / d;
        }
        for (int64_t i = 0; i < n; ++i)
            for (int64_t c = 0; c < w; ++c) inv[i * n + c0 + c] = X[i * w + c];
    }
    return inv;
}

}  // namespace

// Algorithm 1 with the stopping rules of §8c L9 (coarse_enough, max_levels,
// stagnation: no reduction, or > 95% of the rows kept on two levels in a row).
HostHierarchy build_hierarchy(Csr A0, const SetupParams& prm) {
    // AMGB_SETUP_TIMING=1: per-level phase times on stderr
    const bool timing = std::getenv("AMGB_SETUP_TIMING") != nullptr;
    auto t_last = std::chrono::steady_clock::now();
    auto lap = [&](const char* what, size_t l) {
        if (!timing) return;
        const auto t = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[setup] level %zu %-12s %8.1f ms\n", l, what,
                     std::chrono::duration<double, std::milli>(t - t_last).count());
        t_last = t;
    };
    HostHierarchy H;
    H.levels.emplace_back();
    H.levels.back().A = std::move(A0);
    double eps = prm.eps_strong;
    bool prev_slow = false;
    for (;;) {
        HostLevel& L = H.levels.back();
        const int64_t n = L.A.nrows;
        if (!(n > prm.coarse_enough && static_cast<int>(H.levels.size()) < prm.max_levels)) break;
        const size_t lv = H.levels.size() - 1;
        std::vector<uint8_t> S;
        strength(L.A, eps, S);
        lap("strength", lv);
        std::vector<int32_t> id;
        std::vector<int64_t> root;
        const int64_t cnt = aggregate(L.A, S, id, &root);
        lap("aggregate", lv);
        const bool slow = static_cast<double>(cnt) > 0.95 * static_cast<double>(n);
        if (cnt == n || (slow && prev_slow)) break;
        prev_slow = slow;
        L.P = prolongation(L.A, S, id, cnt, prm.smoothed, prm.p_omega);
        lap("P", lv);
        L.R = transpose(L.P);
        lap("R=P^T", lv);
        L.agg = std::move(id);
        L.root = std::move(root);
        L.n_agg = cnt;
        Csr AP = multiply(L.A, L.P);
        lap("AP", lv);
        Csr Ac = multiply(L.R, AP);
        lap("R(AP)", lv);
        AP = Csr();
        setup_smoother(L, prm);
        lap("smoother", lv);
        H.levels.emplace_back();
        H.levels.back().A = std::move(Ac);
        eps *= prm.eps_decay;
    }
    finish_hierarchy(H, prm);
    lap("coarse inv", H.levels.size() - 1);
    return H;
}

// The coarsest level: size check and dense inverse (shared by the GPU setup).
void finish_hierarchy(HostHierarchy& H, const SetupParams& prm) {
    HostLevel& C = H.levels.back();
    if (C.A.nrows > prm.dense_max)
        fail(-5, "coarsest level has " + std::to_string(C.A.nrows) + " rows > dense_max");
    // positive diagonal is required on the coarsest level too (strength() checks
    // the others)
    H.coarse_inv = dense_inverse(C.A);
}

}  // namespace amgb
