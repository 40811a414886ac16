// Batched right-hand sides ("the hierarchy can be reused
// with multiple right-hand sides").  K right-hand sides are
// solved together: every level vector is stored interleaved (x[i*K + j]), so one
// pass over a matrix serves all K columns (matrix bytes are amortised K-fold)
// and a gather fetches K consecutive doubles.  Each column runs its own CG with
// its own scalars and convergence test; columns that are done (or padding
// columns beyond k) get alpha = beta = 0, so their x and r stay fixed.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.cuh"

namespace amgb {

constexpr int kMaxK = 8;

struct KStateB {
    double nf[kMaxK], tolnf[kMaxK], res[kMaxK], rho[kMaxK], rho_prev[kMaxK], alpha[kMaxK], beta[kMaxK];
    double true_res[kMaxK];
    int32_t iter[kMaxK], cdone[kMaxK], status[kMaxK];
    int32_t k, maxiter, done, pad;
};

// K interleaved columns of row i: K = 4, 8 move 32-byte groups with one 256-bit
// access each (LDG/STG.E.ENL2.256 on sm_100a): a warp's gather of 32 rows is
// then full 128-byte lines instead of half-used ones (two 16-byte loads per row
// left the level-0 batched kernels L1-bound); K = 2 one 128-bit access.
__device__ __forceinline__ void ld256(const double* p, double* r) {  // data written by earlier kernels
    asm("ld.global.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(r[0]), "=d"(r[1]), "=d"(r[2]), "=d"(r[3]) : "l"(p));
}
__device__ __forceinline__ void ldg256(const double* p, double* r) {
    asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(r[0]), "=d"(r[1]), "=d"(r[2]), "=d"(r[3]) : "l"(p));
}
__device__ __forceinline__ void st256(double* p, const double* v) {
    asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(v[0]), "d"(v[1]), "d"(v[2]), "d"(v[3])
                 : "memory");
}

template <int K>
__device__ __forceinline__ Vk<K> ldk(const double* p, int64_t i) {
    Vk<K> r;
    if constexpr (K % 4 == 0) {
#pragma unroll
        for (int j = 0; j < K / 4; ++j) ld256(p + i * K + 4 * j, r.v + 4 * j);
    } else if constexpr (K % 2 == 0) {
        const double2* q = reinterpret_cast<const double2*>(p + i * K);
#pragma unroll
        for (int j = 0; j < K / 2; ++j) {
            const double2 t = q[j];
            r.v[2 * j] = t.x;
            r.v[2 * j + 1] = t.y;
        }
    } else {
#pragma unroll
        for (int j = 0; j < K; ++j) r.v[j] = p[i * K + j];
    }
    return r;
}
template <int K>
__device__ __forceinline__ Vk<K> ldgk(const double* p, int64_t i) {  // read-only path (gathers)
    Vk<K> r;
    if constexpr (K % 4 == 0) {
#pragma unroll
        for (int j = 0; j < K / 4; ++j) ldg256(p + i * K + 4 * j, r.v + 4 * j);
    } else if constexpr (K % 2 == 0) {
        const double2* q = reinterpret_cast<const double2*>(p + i * K);
#pragma unroll
        for (int j = 0; j < K / 2; ++j) {
            const double2 t = __ldg(q + j);
            r.v[2 * j] = t.x;
            r.v[2 * j + 1] = t.y;
        }
    } else {
#pragma unroll
        for (int j = 0; j < K; ++j) r.v[j] = __ldg(p + i * K + j);
    }
    return r;
}
template <int K>
__device__ __forceinline__ void stk(double* p, int64_t i, const Vk<K>& v) {
    if constexpr (K % 4 == 0) {
#pragma unroll
        for (int j = 0; j < K / 4; ++j) st256(p + i * K + 4 * j, v.v + 4 * j);
    } else if constexpr (K % 2 == 0) {
        double2* q = reinterpret_cast<double2*>(p + i * K);
#pragma unroll
        for (int j = 0; j < K / 2; ++j) q[j] = make_double2(v.v[2 * j], v.v[2 * j + 1]);
    } else {
#pragma unroll
        for (int j = 0; j < K; ++j) p[i * K + j] = v.v[j];
    }
}

// ---------------------------------------------------------------- finalizers
template <int K>
struct FinNormB {
    KStateB* ks;
    double tol;
    __device__ void operator()(const double* t) const {
        for (int j = 0; j < K; ++j) {
            ks->nf[j] = sqrt(t[j]);
            ks->tolnf[j] = tol * ks->nf[j];
        }
    }
};

template <int K>
struct FinInitResB {
    KStateB* ks;
    __device__ void operator()(const double* t) const {
        int all = 1;
        for (int j = 0; j < K; ++j) {
            const double res = sqrt(t[j]);
            ks->res[j] = res;
            ks->iter[j] = 0;
            ks->status[j] = 0;
            ks->alpha[j] = 0.0;
            ks->beta[j] = 0.0;
            ks->cdone[j] = (j >= ks->k) || !(0 < ks->maxiter && res > ks->tolnf[j]);
            all &= ks->cdone[j];
        }
        ks->done = all;
    }
};

template <int K>
struct FinTrueResB {
    KStateB* ks;
    __device__ void operator()(const double* t) const {
        for (int j = 0; j < K; ++j) ks->true_res[j] = sqrt(t[j]);
    }
};

template <int K>
struct FinRhoB {  // rho_j = (r_j, z_j); beta_j
    KStateB* ks;
    __device__ void operator()(const double* t) const {
        for (int j = 0; j < K; ++j) {
            if (ks->cdone[j]) {
                ks->beta[j] = 0.0;
                continue;
            }
            const double rho = t[j];
            if (!(rho > 0.0)) {
                ks->status[j] = AMG_BREAKDOWN;
                ks->cdone[j] = 1;
                ks->beta[j] = 0.0;
                continue;
            }
            ks->rho[j] = rho;
            ks->beta[j] = ks->iter[j] == 0 ? 0.0 : rho / ks->rho_prev[j];
        }
    }
};

template <int K>
struct FinSigmaB {  // alpha_j = rho_j / (p'_j, q_j)
    KStateB* ks;
    __device__ void operator()(const double* t) const {
        for (int j = 0; j < K; ++j) {
            if (ks->cdone[j]) {
                ks->alpha[j] = 0.0;
                continue;
            }
            const double sigma = t[j];
            if (!(sigma > 0.0)) {
                ks->status[j] = AMG_BREAKDOWN;
                ks->cdone[j] = 1;
                ks->alpha[j] = 0.0;
                continue;
            }
            ks->alpha[j] = ks->rho[j] / sigma;
        }
    }
};

template <int K>
struct FinCgUpdateB {  // res_j, k_j += 1, per-column loop test
    KStateB* ks;
    __device__ void operator()(const double* t) const {
        int all = 1;
        for (int j = 0; j < K; ++j) {
            if (!ks->cdone[j]) {
                ks->res[j] = sqrt(t[j]);
                ks->iter[j] += 1;
                ks->rho_prev[j] = ks->rho[j];
                ks->cdone[j] = !(ks->iter[j] < ks->maxiter && ks->res[j] > ks->tolnf[j]);
            }
            all &= ks->cdone[j];
        }
        ks->done = all;
    }
};

// ---------------------------------------------------------------- row ops
// GATHER / ROWV count 8-byte streams per gathered column / per row (bytes model).
template <int K>
struct OpSpmvB {
    static constexpr int GATHER = K, ROWV = K, NDOT = 0;
    const double* x;
    double* y;
    NoFin fin;
    struct Row {};
    __device__ void prepare() {}
    __device__ Row load(int64_t) const { return {}; }
    __device__ Vk<K> gather(int32_t c) const { return ldgk<K>(x, c); }
    __device__ void row(int64_t i, const Vk<K>& s, const Row&, double*) const { stk<K>(y, i, s); }
};

template <int K, int ND, class Fin>
struct OpResidualB {  // y = f - A x  [+ (y_j, y_j)]
    static constexpr int GATHER = K, ROWV = 2 * K, NDOT = ND * K;
    const double* x;
    const double* f;
    double* y;
    Fin fin;
    struct Row {
        Vk<K> f;
    };
    __device__ void prepare() {}
    __device__ Row load(int64_t i) const { return {ldk<K>(f, i)}; }
    __device__ Vk<K> gather(int32_t c) const { return ldgk<K>(x, c); }
    __device__ void row(int64_t i, const Vk<K>& s, const Row& rr, double* d) const {
        Vk<K> r;
#pragma unroll
        for (int j = 0; j < K; ++j) {
            r.v[j] = rr.f.v[j] - s.v[j];
            if constexpr (ND > 0) d[j] += r.v[j] * r.v[j];
        }
        stk<K>(y, i, r);
    }
};

template <int K>
struct OpRes0B {  // t = f - A (m o f)
    static constexpr int GATHER = 1 + K, ROWV = K, NDOT = 0;
    const double* m;
    const double* f;
    double* t;
    NoFin fin;
    struct Row {
        Vk<K> f;
    };
    __device__ void prepare() {}
    __device__ Row load(int64_t i) const { return {ldk<K>(f, i)}; }
    __device__ Vk<K> gather(int32_t c) const {
        const double mc = __ldg(m + c);
        Vk<K> x = ldgk<K>(f, c);
#pragma unroll
        for (int j = 0; j < K; ++j) x.v[j] *= mc;
        return x;
    }
    __device__ void row(int64_t i, const Vk<K>& s, const Row& rr, double*) const {
        Vk<K> r;
#pragma unroll
        for (int j = 0; j < K; ++j) r.v[j] = rr.f.v[j] - s.v[j];
        stk<K>(t, i, r);
    }
};

template <int K, int ND, class Fin>
struct OpRelaxB {  // xo = x + m o (f - A x)  [+ (f_j, xo_j)]
    static constexpr int GATHER = K, ROWV = 1 + 2 * K, NDOT = ND * K;
    const double* x;
    const double* m;
    const double* f;
    double* xo;
    Fin fin;
    struct Row {
        Vk<K> x, f;
        double m;
    };
    __device__ void prepare() {}
    __device__ Row load(int64_t i) const { return {ldk<K>(x, i), ldk<K>(f, i), m[i]}; }
    __device__ Vk<K> gather(int32_t c) const { return ldgk<K>(x, c); }
    __device__ void row(int64_t i, const Vk<K>& s, const Row& rr, double* d) const {
        Vk<K> xn;
#pragma unroll
        for (int j = 0; j < K; ++j) {
            xn.v[j] = rr.x.v[j] + rr.m * (rr.f.v[j] - s.v[j]);
            if constexpr (ND > 0) d[j] += rr.f.v[j] * xn.v[j];
        }
        stk<K>(xo, i, xn);
    }
};

template <int K>
struct OpProl0B {  // x = m o f + P e
    static constexpr int GATHER = K, ROWV = 1 + 2 * K, NDOT = 0;
    const double* e;
    const double* m;
    const double* f;
    double* x;
    NoFin fin;
    struct Row {
        Vk<K> f;
        double m;
    };
    __device__ void prepare() {}
    __device__ Row load(int64_t i) const { return {ldk<K>(f, i), m[i]}; }
    __device__ Vk<K> gather(int32_t c) const { return ldgk<K>(e, c); }
    __device__ void row(int64_t i, const Vk<K>& s, const Row& rr, double*) const {
        Vk<K> xn;
#pragma unroll
        for (int j = 0; j < K; ++j) xn.v[j] = rr.m * rr.f.v[j] + s.v[j];
        stk<K>(x, i, xn);
    }
};

template <int K>
struct OpProlAddB {  // x = x + P e
    static constexpr int GATHER = K, ROWV = 2 * K, NDOT = 0;
    const double* e;
    double* x;
    NoFin fin;
    struct Row {
        Vk<K> x;
    };
    __device__ void prepare() {}
    __device__ Row load(int64_t i) const { return {ldk<K>(x, i)}; }
    __device__ Vk<K> gather(int32_t c) const { return ldgk<K>(e, c); }
    __device__ void row(int64_t i, const Vk<K>& s, const Row& rr, double*) const {
        Vk<K> xn;
#pragma unroll
        for (int j = 0; j < K; ++j) xn.v[j] = rr.x.v[j] + s.v[j];
        stk<K>(x, i, xn);
    }
};

template <int K, int ND, class Fin>
struct OpChebB {  // Chebyshev step per column (same alpha/beta for every column)
    static constexpr int GATHER = K, ROWV = 1 + 4 * K, NDOT = ND * K;
    const double* x;
    const double* f;
    const double* diag;
    double* p;
    double* xo;
    double alpha, beta;
    int32_t scaled, first;
    Fin fin;
    struct Row {
        Vk<K> f, p, x;
        double dg;
    };
    __device__ void prepare() {}
    __device__ Row load(int64_t i) const {
        Row r{ldk<K>(f, i), Vk<K>{}, ldk<K>(x, i), diag[i]};
        if (!first) r.p = ldk<K>(p, i);
        return r;
    }
    __device__ Vk<K> gather(int32_t c) const { return ldgk<K>(x, c); }
    __device__ void row(int64_t i, const Vk<K>& s, const Row& rr, double* d) const {
        Vk<K> pn, xn;
#pragma unroll
        for (int j = 0; j < K; ++j) {
            double r = rr.f.v[j] - s.v[j];
            if (scaled) r = r / rr.dg;
            pn.v[j] = first ? alpha * r : alpha * r + beta * rr.p.v[j];
            xn.v[j] = rr.x.v[j] + pn.v[j];
            if constexpr (ND > 0) d[j] += rr.f.v[j] * xn.v[j];
        }
        stk<K>(p, i, pn);
        stk<K>(xo, i, xn);
    }
};

template <int K, class Fin>
struct OpCgDirB {  // p'_j = z_j + beta_j p_j (in the gather), q = A p', sigma_j
    static constexpr int GATHER = 2 * K, ROWV = 2 * K, NDOT = K;
    const double* z;
    const double* p;
    double* pn;
    double* q;
    const KStateB* ks;
    double beta[K];
    Fin fin;
    struct Row {
        Vk<K> z, p;
    };
    __device__ void prepare() {
#pragma unroll
        for (int j = 0; j < K; ++j) beta[j] = ks->beta[j];
    }
    __device__ Row load(int64_t i) const { return {ldk<K>(z, i), ldk<K>(p, i)}; }
    __device__ Vk<K> gather(int32_t c) const {
        Vk<K> zc = ldgk<K>(z, c);
        const Vk<K> pc = ldgk<K>(p, c);
#pragma unroll
        for (int j = 0; j < K; ++j) zc.v[j] = fma(beta[j], pc.v[j], zc.v[j]);
        return zc;
    }
    __device__ void row(int64_t i, const Vk<K>& s, const Row& rr, double* d) const {
        Vk<K> pi;
#pragma unroll
        for (int j = 0; j < K; ++j) {
            pi.v[j] = fma(beta[j], rr.p.v[j], rr.z.v[j]);
            d[j] += pi.v[j] * s.v[j];
        }
        stk<K>(pn, i, pi);
        stk<K>(q, i, s);
    }
};

// ---------------------------------------------------------------- vector ops
template <int K, class Fin>
struct VNorm2B {
    static constexpr int NDOT = K, STREAMS = K;
    const double* a;
    Fin fin;
    __device__ void prepare() {}
    __device__ void elem(int64_t i, double* d) const {
        const Vk<K> v = ldk<K>(a, i);
#pragma unroll
        for (int j = 0; j < K; ++j) d[j] += v.v[j] * v.v[j];
    }
};

template <int K, class Fin>
struct VDotB {
    static constexpr int NDOT = K, STREAMS = 2 * K;
    const double* a;
    const double* b;
    Fin fin;
    __device__ void prepare() {}
    __device__ void elem(int64_t i, double* d) const {
        const Vk<K> x = ldk<K>(a, i), y = ldk<K>(b, i);
#pragma unroll
        for (int j = 0; j < K; ++j) d[j] += x.v[j] * y.v[j];
    }
};

template <int K>
struct VMulDiagB {  // x = m o f
    static constexpr int NDOT = 0, STREAMS = 1 + 2 * K;
    const double* m;
    const double* f;
    double* x;
    NoFin fin;
    __device__ void prepare() {}
    __device__ void elem(int64_t i, double*) const {
        Vk<K> v = ldk<K>(f, i);
        const double mi = m[i];
#pragma unroll
        for (int j = 0; j < K; ++j) v.v[j] *= mi;
        stk<K>(x, i, v);
    }
};

template <int K>
struct VCheb0B {  // p = alpha (f / a_ii); x = p
    static constexpr int NDOT = 0, STREAMS = 1 + 3 * K;
    const double* f;
    const double* diag;
    double* p;
    double* x;
    double alpha;
    int32_t scaled;
    NoFin fin;
    __device__ void prepare() {}
    __device__ void elem(int64_t i, double*) const {
        Vk<K> v = ldk<K>(f, i);
        const double dg = diag[i];
#pragma unroll
        for (int j = 0; j < K; ++j) v.v[j] = alpha * (scaled ? v.v[j] / dg : v.v[j]);
        stk<K>(p, i, v);
        stk<K>(x, i, v);
    }
};

template <int K>
struct VCgUpdateB {  // x_j += alpha_j p_j; r_j -= alpha_j q_j; (r_j, r_j)
    static constexpr int NDOT = K, STREAMS = 6 * K;
    double* x;
    double* r;
    const double* p;
    const double* q;
    const KStateB* ks;
    double alpha[K];
    FinCgUpdateB<K> fin;
    __device__ void prepare() {
#pragma unroll
        for (int j = 0; j < K; ++j) alpha[j] = ks->alpha[j];
    }
    __device__ void elem(int64_t i, double* d) const {
        Vk<K> xv = ldk<K>(x, i), rv = ldk<K>(r, i);
        const Vk<K> pv = ldk<K>(p, i), qv = ldk<K>(q, i);
#pragma unroll
        for (int j = 0; j < K; ++j) {
            xv.v[j] = fma(alpha[j], pv.v[j], xv.v[j]);
            rv.v[j] = fma(-alpha[j], qv.v[j], rv.v[j]);
            d[j] += rv.v[j] * rv.v[j];
        }
        stk<K>(x, i, xv);
        stk<K>(r, i, rv);
    }
};

// coarsest level: Y = A_L^-1 F for K interleaved columns (warp per row)
template <int K>
__global__ void __launch_bounds__(kBlock) dense_gemm_b(int64_t n, const double* __restrict__ M,
                                                       const double* __restrict__ F, double* __restrict__ Y,
                                                       const int32_t* gate) {
    if (gated(gate)) return;
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = warp; r < n; r += nwarps) {
        const double* row = M + r * n;
        Vk<K> s{};
        for (int64_t c = lane; c < n; c += 32) fma_acc(s, __ldg(row + c), ldgk<K>(F, c));
#pragma unroll
        for (int j = 0; j < K; ++j) {
            const double t = warp_sum(s.v[j]);
            if (lane == 0) Y[r * K + j] = t;
        }
    }
}

// column-major (leading dimension ld, k columns) <-> interleaved K columns
template <int K>
__global__ void __launch_bounds__(kBlock) pack_cols(const double* __restrict__ src, int64_t ld, int k, int64_t n,
                                                    double* __restrict__ dst, const double* __restrict__ zero_if) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        Vk<K> v;
#pragma unroll
        for (int j = 0; j < K; ++j) v.v[j] = (j < k && src) ? src[j * ld + i] : 0.0;
        stk<K>(dst, i, v);
    }
}
template <int K>
__global__ void __launch_bounds__(kBlock) unpack_cols(const double* __restrict__ src, int k, int64_t n,
                                                      double* __restrict__ dst, int64_t ld, const KStateB* ks) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const Vk<K> v = ldk<K>(src, i);
#pragma unroll
        for (int j = 0; j < K; ++j)
            if (j < k) dst[j * ld + i] = ks->nf[j] == 0.0 ? 0.0 : v.v[j];  // zero RHS -> x = 0
    }
}

}  // namespace amgb
