// Right-preconditioned IDR(s) with bi-orthogonalisation on the device
// (PAPER.md:212 lists IDR(s); the algorithm of van Gijzen &
// Sonneveld 2011, "Algorithm 913", restated in oracle/oracle.c or_idrs).  The
// small s x s quantities (M, phi, c, the bi-orthogonalisation coefficients,
// beta, omega) live in KStateI and are updated by one-thread finalizers; the
// n-vectors G, U (s columns each), P (the shadow space) stay in HBM.
//
// One inner step k = 5 kernels + a V-cycle: c from the lower-triangular
// M[k:s,k:s] c = phi[k:s]; v = r - G[:,k:s] c; z = B v; U_k = U[:,k:s] c + om z;
// G_k = A U_k fused with the s dots P^T G_k; then one vector pass applies the
// bi-orthogonalisation to G_k and U_k and updates r, x and |r|.  The oracle
// orthogonalises G_k against G_0..G_{k-1} one at a time (a dot per i); the
// device gets every coefficient from the single set of dots P^T (A U_k) and
// the stored M (P_i^T G_j = M[i][j] for i >= j): the same numbers in exact
// arithmetic, one kernel instead of k, results agree to rounding (as CGS vs
// MGS in gmres.cuh).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.cuh"

namespace amgb {

constexpr int kIdrMaxS = 8;

struct KStateI {
    double nf, tolnf, res, om, kappa, beta;
    double M[kIdrMaxS * kIdrMaxS];  // M[i * s + j]
    double phi[kIdrMaxS], c[kIdrMaxS], alpha[kIdrMaxS];
    int32_t s, maxiter, it, done, status, pad;
};

// c[0 .. s-k) solves M[k:s, k:s] c = phi[k:s] (forward substitution)
__global__ void idr_solve_c(KStateI* ks, int k) {
    if (ks->done) return;
    const int s = ks->s;
    for (int i = k; i < s; ++i) {
        double sum = ks->phi[i];
        for (int j = k; j < i; ++j) sum -= ks->M[i * s + j] * ks->c[j - k];
        ks->c[i - k] = sum / ks->M[i * s + i];
    }
}

struct FinIdrNorm {  // |f|
    KStateI* ks;
    double tol;
    __device__ void operator()(const double* t) const {
        ks->nf = sqrt(t[0]);
        ks->tolnf = tol * ks->nf;
    }
};

struct FinIdrRes0 {  // |r0|; converged before the first step?
    KStateI* ks;
    __device__ void operator()(const double* t) const {
        ks->res = sqrt(t[0]);
        if (!(ks->res > ks->tolnf) || ks->maxiter <= 0) ks->done = 1;
    }
};

template <int S>
struct FinIdrPhi {  // phi = P^T r
    KStateI* ks;
    __device__ void operator()(const double* t) const {
#pragma unroll
        for (int m = 0; m < S; ++m) ks->phi[m] = t[m];
    }
};

// v = r - sum_{j=k}^{s-1} c[j-k] G_j
template <int S>
struct VIdrV {
    static constexpr int NDOT = 0, STREAMS = 0;  // bytes counted by the caller
    double* v;
    const double* r;
    const double* G;
    int64_t n;
    int k;
    const KStateI* ks;
    NoFin fin;
    double c[S];
    __device__ void prepare() {
#pragma unroll
        for (int j = 0; j < S; ++j) c[j] = j < S - k ? ks->c[j] : 0.0;
    }
    __device__ void elem(int64_t q, double*) const {
        double sum = r[q];
        for (int j = k; j < S; ++j) sum -= c[j - k] * G[(int64_t)j * n + q];
        v[q] = sum;
    }
};

// U_k = om z + sum_{j=k}^{s-1} c[j-k] U_j  (U_k read before it is written)
template <int S>
struct VIdrU {
    static constexpr int NDOT = 0, STREAMS = 0;
    double* U;
    const double* z;
    int64_t n;
    int k;
    const KStateI* ks;
    NoFin fin;
    double c[S];
    double om;
    __device__ void prepare() {
#pragma unroll
        for (int j = 0; j < S; ++j) c[j] = j < S - k ? ks->c[j] : 0.0;
        om = ks->om;
    }
    __device__ void elem(int64_t q, double*) const {
        double sum = om * z[q];
        for (int j = k; j < S; ++j) sum += c[j - k] * U[(int64_t)j * n + q];
        U[(int64_t)k * n + q] = sum;
    }
};

// bi-orthogonalisation coefficients, the new column of M, beta, phi
struct FinIdrOrth {
    KStateI* ks;
    int k;
    __device__ void operator()(const double* t) const {
        const int s = ks->s;
        for (int i = 0; i < k; ++i) {
            double a = t[i];
            for (int j = 0; j < i; ++j) a -= ks->alpha[j] * ks->M[i * s + j];
            ks->alpha[i] = a / ks->M[i * s + i];
        }
        for (int m = k; m < s; ++m) {
            double v = t[m];
            for (int i = 0; i < k; ++i) v -= ks->alpha[i] * ks->M[m * s + i];
            ks->M[m * s + k] = v;
        }
        ks->it += 1;
        const double mkk = ks->M[k * s + k];
        if (mkk == 0.0) {
            ks->status = AMG_BREAKDOWN;
            ks->done = 1;
            return;
        }
        ks->beta = ks->phi[k] / mkk;
        for (int m = k + 1; m < s; ++m) ks->phi[m] = ks->phi[m] - ks->beta * ks->M[m * s + k];
    }
};

// G_k = A U_k and the dots P_m^T G_k (m < S)
template <int S>
struct OpIdrG {
    static constexpr int GATHER = 1, ROWV = 1 + S;  // U_k gathered; G_k written, P read
    static constexpr int NDOT = S;
    const double* u;
    double* g;
    const double* P;
    int64_t n;
    FinIdrOrth fin;
    struct Row {
        double p[S];
    };
    __device__ void prepare() {}
    __device__ Row load(int64_t i) const {
        Row r;
#pragma unroll
        for (int m = 0; m < S; ++m) r.p[m] = P[(int64_t)m * n + i];
        return r;
    }
    __device__ double gather(int32_t c) const { return __ldg(u + c); }
    __device__ void row(int64_t i, double s, const Row& rr, double* d) const {
        g[i] = s;
#pragma unroll
        for (int m = 0; m < S; ++m) d[m] += rr.p[m] * s;
    }
};

struct FinIdrRes {  // after an inner step: |r|, convergence, iteration cap
    KStateI* ks;
    __device__ void operator()(const double* t) const {
        ks->res = sqrt(t[0]);
        if (!(ks->res > ks->tolnf) || ks->it >= ks->maxiter) ks->done = 1;
    }
};

// G_k -= sum_{i<k} alpha_i G_i; U_k likewise; r -= beta G_k; x += beta U_k; (r, r)
template <int S>
struct VIdrUpd {
    static constexpr int NDOT = 1, STREAMS = 0;
    double* G;
    double* U;
    double* r;
    double* x;
    int64_t n;
    int k;
    const KStateI* ks;
    FinIdrRes fin;
    double alpha[S];
    double beta;
    __device__ void prepare() {
#pragma unroll
        for (int i = 0; i < S; ++i) alpha[i] = i < k ? ks->alpha[i] : 0.0;
        beta = ks->beta;
    }
    __device__ void elem(int64_t q, double* d) const {
        double g = G[(int64_t)k * n + q], u = U[(int64_t)k * n + q];
        for (int i = 0; i < k; ++i) {
            g = g - alpha[i] * G[(int64_t)i * n + q];
            u = u - alpha[i] * U[(int64_t)i * n + q];
        }
        G[(int64_t)k * n + q] = g;
        U[(int64_t)k * n + q] = u;
        const double rn = r[q] - beta * g;
        r[q] = rn;
        x[q] = x[q] + beta * u;
        d[0] += rn * rn;
    }
};

// dimension reduction: omega from (t, t), (t, r) with the "angle" safeguard
struct FinIdrOmega {
    KStateI* ks;
    __device__ void operator()(const double* t) const {
        ks->it += 1;
        const double tt = sqrt(t[0]), tr = t[1];
        if (tt == 0.0) {
            ks->status = AMG_BREAKDOWN;
            ks->done = 1;
            return;
        }
        double om = tr / (tt * tt);
        const double rho = fabs(tr) / (tt * ks->res);
        if (rho < ks->kappa) om = om * ks->kappa / rho;
        if (om == 0.0) {
            ks->status = AMG_BREAKDOWN;
            ks->done = 1;
            return;
        }
        ks->om = om;
    }
};

// t = A z, (t, t), (t, r)
struct OpIdrT {
    static constexpr int GATHER = 1, ROWV = 2;  // z gathered; t written, r read
    static constexpr int NDOT = 2;
    const double* z;
    double* t;
    const double* r;
    FinIdrOmega fin;
    struct Row {
        double r;
    };
    __device__ void prepare() {}
    __device__ Row load(int64_t i) const { return {r[i]}; }
    __device__ double gather(int32_t c) const { return __ldg(z + c); }
    __device__ void row(int64_t i, double s, const Row& rr, double* d) const {
        t[i] = s;
        d[0] += s * s;
        d[1] += s * rr.r;
    }
};

template <int S>
struct FinIdrCycle {  // after the reduction: |r|, phi = P^T r, convergence, cap
    KStateI* ks;
    __device__ void operator()(const double* t) const {
        ks->res = sqrt(t[0]);
#pragma unroll
        for (int m = 0; m < S; ++m) ks->phi[m] = t[1 + m];
        if (!(ks->res > ks->tolnf) || ks->it >= ks->maxiter) ks->done = 1;
    }
};

// x += om z; r -= om t; (r, r) and P^T r for the next cycle
template <int S>
struct VIdrRed {
    static constexpr int NDOT = 1 + S, STREAMS = 0;
    double* x;
    double* r;
    const double* z;
    const double* t;
    const double* P;
    int64_t n;
    const KStateI* ks;
    FinIdrCycle<S> fin;
    double om;
    __device__ void prepare() { om = ks->om; }
    __device__ void elem(int64_t q, double* d) const {
        x[q] = x[q] + om * z[q];
        const double rn = r[q] - om * t[q];
        r[q] = rn;
        d[0] += rn * rn;
#pragma unroll
        for (int m = 0; m < S; ++m) d[1 + m] += P[(int64_t)m * n + q] * rn;
    }
};

// phi = P^T r (start of the solve)
template <int S>
struct VIdrPhi {
    static constexpr int NDOT = S, STREAMS = 0;
    const double* r;
    const double* P;
    int64_t n;
    FinIdrPhi<S> fin;
    __device__ void prepare() {}
    __device__ void elem(int64_t q, double* d) const {
#pragma unroll
        for (int m = 0; m < S; ++m) d[m] += P[(int64_t)m * n + q] * r[q];
    }
};

struct FinTrueResI {  // true residual at exit
    KStateI* ks;
    __device__ void operator()(const double* t) const { ks->res = sqrt(t[0]); }
};

}  // namespace amgb
