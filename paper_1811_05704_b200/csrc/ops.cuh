// Finalizers (Krylov scalar updates run by the last block of a reducing
// kernel, or by fin_kernel after a cross-rank all-reduce) and fused vector
// kernels of the CG / BiCGStab iterations.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/amgb.h"
#include "kernels.cuh"

namespace amgb {

// ============================================================ device code

__global__ void __launch_bounds__(kBlock) dense_gemv(int64_t n, const double* __restrict__ M,
                                                     const double* __restrict__ x, double* __restrict__ y,
                                                     const int32_t* gate) {
    pdl_wait();
    if (gated(gate)) return;
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = warp; r < n; r += nwarps) {
        const double* row = M + r * n;
        double s = 0.0;
        for (int64_t j = lane; j < n; j += 32) s = fma(__ldg(row + j), __ldg(x + j), s);
        s = warp_sum(s);
        if (lane == 0) y[r] = s;
    }
}

// ---- finalizers (run once, by the last block of a reducing kernel) ----------

struct FinNorm {  // |f| -> nf, tol |f|
    KState* ks;
    double tol;
    __device__ void operator()(const double* t) const {
        ks->nf = sqrt(t[0]);
        ks->tolnf = tol * ks->nf;
    }
};

struct FinInitRes {  // r0 = f - A x0: res, done; BiCGStab also rho = (r,r), |rhat|
    KState* ks;
    __device__ void operator()(const double* t) const {
        const double res = sqrt(t[0]);
        ks->res = res;
        ks->rho = t[0];
        ks->rhat_norm = res;
        ks->iter = 0;
        ks->half = 0;
        ks->status = 0;
        ks->done = !(0 < ks->maxiter && res > ks->tolnf);
        ks->skip2 = ks->done;
    }
};

// Test hook (amg_level_op_ex): store the n reduced totals of a fused dot.
struct FinStore {
    double* out;
    int n;
    __device__ void operator()(const double* t) const {
        for (int k = 0; k < n; ++k) out[k] = t[k];
    }
};

struct FinTrueRes {
    KState* ks;
    __device__ void operator()(const double* t) const { ks->true_res = sqrt(t[0]); }
};

struct FinRho {  // CG: rho = (r, z); beta = rho / rho_prev (0 on the first iteration)
    KState* ks;
    __device__ void operator()(const double* t) const {
        const double rho = t[0];
        if (!(rho > 0.0)) {
            ks->status = AMG_BREAKDOWN;
            ks->done = 1;
            return;
        }
        ks->rho = rho;
        ks->beta = ks->iter == 0 ? 0.0 : rho / ks->rho_prev;
    }
};

struct FinSigma {  // CG: sigma = (p, q); alpha = rho / sigma
    KState* ks;
    __device__ void operator()(const double* t) const {
        const double sigma = t[0];
        if (!(sigma > 0.0)) {
            ks->status = AMG_BREAKDOWN;
            ks->done = 1;
            return;
        }
        ks->sigma = sigma;
        ks->alpha = ks->rho / sigma;
    }
};

struct FinCgUpdate {  // CG: res = |r|; k += 1; loop test of §8c c-1
    KState* ks;
    __device__ void operator()(const double* t) const {
        ks->res = sqrt(t[0]);
        ks->iter += 1;
        ks->rho_prev = ks->rho;
        ks->done = !(ks->iter < ks->maxiter && ks->res > ks->tolnf);
    }
};

// Fused CG (see OpRes0Upd / OpCgDirX): the r update of iteration k-1 landed
// in this iteration's first kernel: res, k += 1, loop test of §8c c-1.
struct FinRes0Upd {
    KState* ks;
    __device__ void operator()(const double* t) const {
        if (!ks->upd) return;  // iteration 0: nothing was updated
        ks->res = sqrt(t[0]);
        ks->iter += 1;
        ks->rho_prev = ks->rho;
        ks->upd = 0;
        ks->xpend = 1;
        ks->done = !(ks->iter < ks->maxiter && ks->res > ks->tolnf);
    }
};

struct FinSigmaX {  // FinSigma + bookkeeping of the deferred updates
    KState* ks;
    __device__ void operator()(const double* t) const {
        ks->xpend = 0;  // the CG direction kernel just applied it
        const double sigma = t[0];
        if (!(sigma > 0.0)) {
            ks->status = AMG_BREAKDOWN;
            ks->done = 1;
            ks->upd = 0;
            return;
        }
        ks->sigma = sigma;
        ks->alpha = ks->rho / sigma;
        ks->upd = 1;
    }
};

// 16-B vector access for the paired (elem2) vector ops: elements 2j, 2j+1.
__device__ __forceinline__ double2 ld2(const double* a, int64_t j) { return reinterpret_cast<const double2*>(a)[j]; }
__device__ __forceinline__ void st2(double* a, int64_t j, double2 v) { reinterpret_cast<double2*>(a)[j] = v; }
__device__ __forceinline__ bool al16(const void* a) { return (reinterpret_cast<uintptr_t>(a) & 15) == 0; }

// x += alpha p (the last deferred x update after the loop)
struct VAxpyAlpha {
    static constexpr int NDOT = 0, STREAMS = 3;
    double* x;
    const double* p;
    const KState* ks;
    double alpha;
    NoFin fin;
    __device__ void prepare() { alpha = ks->alpha; }
    __device__ void elem(int64_t i, double*) const { x[i] = fma(alpha, p[i], x[i]); }
};

// BiCGStab finalizers (§8c c-1, right-preconditioned van der Vorst)
struct FinBiAlpha {  // alpha = rho / (rhat, v)
    KState* ks;
    __device__ void operator()(const double* t) const {
        if (t[0] == 0.0) {
            ks->status = AMG_BREAKDOWN;
            ks->done = 1;
            ks->skip2 = 1;
            return;
        }
        ks->alpha = ks->rho / t[0];
    }
};

struct FinBiS {  // |s| <= tol |f| -> half-step exit
    KState* ks;
    __device__ void operator()(const double* t) const {
        ks->ss = sqrt(t[0]);
        if (ks->ss <= ks->tolnf) {
            ks->half = 1;
            ks->skip2 = 1;
        }
    }
};

struct FinBiOmega {  // omega = (t, s) / (t, t)
    KState* ks;
    __device__ void operator()(const double* t) const {
        if (t[0] == 0.0) {
            ks->status = AMG_BREAKDOWN;
            ks->done = 1;
            ks->skip2 = 1;
            return;
        }
        const double om = t[1] / t[0];
        if (fabs(om) < 1e-30) {
            ks->status = AMG_BREAKDOWN;
            ks->done = 1;
            ks->skip2 = 1;
            return;
        }
        ks->omega = om;
    }
};

struct FinBiX {  // after x, r update: rho_next = (rhat, r), res = |r|
    KState* ks;
    __device__ void operator()(const double* t) const {
        ks->iter += 1;
        if (ks->half) {
            ks->res = ks->ss;
            ks->done = 1;
            ks->skip2 = 1;
            return;
        }
        const double rho_next = t[0];
        ks->res = sqrt(t[1]);
        ks->done = !(ks->iter < ks->maxiter && ks->res > ks->tolnf);
        if (!ks->done && fabs(rho_next) < 1e-30 * ks->rhat_norm * ks->res) {
            ks->status = AMG_BREAKDOWN;
            ks->done = 1;
        }
        if (!ks->done) {
            ks->beta = (rho_next / ks->rho) * (ks->alpha / ks->omega);
            ks->rho_prev = ks->rho;
            ks->rho = rho_next;
        }
        ks->skip2 = ks->done;
    }
};

// ---- vector ops ----------------------------------------------------------

struct VNorm2 {
    static constexpr int STREAMS = 1;  // n-vectors moved; (a, a)
    static constexpr int NDOT = 1;
    const double* a;
    FinNorm fin;
    __device__ void prepare() {}
    __device__ void elem(int64_t i, double* d) const { d[0] += a[i] * a[i]; }
};

template <class Fin>
struct VDot {
    static constexpr int STREAMS = 2;  // n-vectors moved; (a, b)
    static constexpr int NDOT = 1;
    const double* a;
    const double* b;
    Fin fin;
    __device__ void prepare() {}
    __device__ void elem(int64_t i, double* d) const { d[0] += a[i] * b[i]; }
};

struct VMulDiag {
    static constexpr int STREAMS = 3;  // n-vectors moved; x = m o f  (first SPAI-0/Jacobi sweep from zero)
    static constexpr int NDOT = 0;
    const double* m;
    const double* f;
    double* x;
    NoFin fin;
    __device__ void prepare() {}
    __device__ void elem(int64_t i, double*) const { x[i] = m[i] * f[i]; }
};

struct VCheb0 {
    static constexpr int STREAMS = 4;  // n-vectors moved; first Chebyshev step from x = 0: p = alpha (f / a_ii); x = p
    static constexpr int NDOT = 0;
    const double* f;
    const double* diag;
    double* p;
    double* x;
    double alpha;
    int32_t scaled;
    NoFin fin;
    __device__ void prepare() {}
    __device__ void elem(int64_t i, double*) const {
        double r = f[i];
        if (scaled) r = r / diag[i];
        const double pn = alpha * r;
        p[i] = pn;
        x[i] = pn;
    }
};

struct VCgUpdate {
    static constexpr int STREAMS = 6;  // n-vectors moved; x += alpha p; r -= alpha q; (r, r)
    static constexpr int NDOT = 1;
    double* x;
    double* r;
    const double* p;
    const double* q;
    const KState* ks;
    double alpha;
    FinCgUpdate fin;
    __device__ void prepare() { alpha = ks->alpha; }
    __device__ void elem(int64_t i, double* d) const {
        x[i] = fma(alpha, p[i], x[i]);
        const double rn = fma(-alpha, q[i], r[i]);
        r[i] = rn;
        d[0] += rn * rn;
    }
    __device__ bool aligned16() const { return al16(x) && al16(r) && al16(p) && al16(q); }
    __device__ void elem2(int64_t j, double* d) const {
        const double2 pv = ld2(p, j), qv = ld2(q, j);
        double2 xv = ld2(x, j), rv = ld2(r, j);
        xv.x = fma(alpha, pv.x, xv.x);
        xv.y = fma(alpha, pv.y, xv.y);
        rv.x = fma(-alpha, qv.x, rv.x);
        rv.y = fma(-alpha, qv.y, rv.y);
        st2(x, j, xv);
        st2(r, j, rv);
        d[0] += rv.x * rv.x;
        d[0] += rv.y * rv.y;
    }
};

// The same update, also writing mf = m o r_new for the next V-cycle's level-0
// zero-start residual (one gathered vector instead of m and r).
struct VCgUpdateMF {
    static constexpr int STREAMS = 8;  // + m read, mf written
    static constexpr int NDOT = 1;
    double* x;
    double* r;
    const double* p;
    const double* q;
    const double* m;
    double* mf;
    const KState* ks;
    double alpha;
    FinCgUpdate fin;
    __device__ void prepare() { alpha = ks->alpha; }
    __device__ void elem(int64_t i, double* d) const {
        x[i] = fma(alpha, p[i], x[i]);
        const double rn = fma(-alpha, q[i], r[i]);
        r[i] = rn;
        mf[i] = m[i] * rn;
        d[0] += rn * rn;
    }
    __device__ bool aligned16() const {
        return ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(r) | reinterpret_cast<uintptr_t>(p) |
                 reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(m) | reinterpret_cast<uintptr_t>(mf)) &
                15) == 0;
    }
    // Elements 2j and 2j+1 (same arithmetic as elem, loads issued first).
    __device__ void elem2(int64_t j, double* d) const {
        const double2 pv = __ldg(reinterpret_cast<const double2*>(p) + j);
        const double2 qv = __ldg(reinterpret_cast<const double2*>(q) + j);
        const double2 mv = __ldg(reinterpret_cast<const double2*>(m) + j);
        double2 xv = reinterpret_cast<const double2*>(x)[j];
        double2 rv = reinterpret_cast<const double2*>(r)[j];
        xv.x = fma(alpha, pv.x, xv.x);
        xv.y = fma(alpha, pv.y, xv.y);
        rv.x = fma(-alpha, qv.x, rv.x);
        rv.y = fma(-alpha, qv.y, rv.y);
        reinterpret_cast<double2*>(x)[j] = xv;
        reinterpret_cast<double2*>(r)[j] = rv;
        reinterpret_cast<double2*>(mf)[j] = make_double2(mv.x * rv.x, mv.y * rv.y);
        d[0] += rv.x * rv.x;
        d[0] += rv.y * rv.y;
    }
};

struct VBiP {
    static constexpr int STREAMS = 3;  // n-vectors moved; p = r (k = 0) or r + beta (p - omega v)
    static constexpr int NDOT = 0;
    const double* r;
    const double* v;
    double* p;
    const KState* ks;
    double beta, omega;
    int32_t first;
    NoFin fin;
    __device__ void prepare() {
        beta = ks->beta;
        omega = ks->omega;
        first = ks->iter == 0;
    }
    __device__ void elem(int64_t i, double*) const {
        p[i] = first ? r[i] : fma(beta, p[i] - omega * v[i], r[i]);
    }
    __device__ bool aligned16() const { return al16(r) && al16(v) && al16(p); }
    __device__ void elem2(int64_t j, double*) const {
        const double2 rv = ld2(r, j);
        if (first) {
            st2(p, j, rv);
            return;
        }
        const double2 vv = ld2(v, j), pv = ld2(p, j);
        st2(p, j, make_double2(fma(beta, pv.x - omega * vv.x, rv.x), fma(beta, pv.y - omega * vv.y, rv.y)));
    }
};

struct VBiS {
    static constexpr int STREAMS = 3;  // n-vectors moved; s = r - alpha v; (s, s)
    static constexpr int NDOT = 1;
    const double* r;
    const double* v;
    double* s;
    const KState* ks;
    double alpha;
    FinBiS fin;
    __device__ void prepare() { alpha = ks->alpha; }
    __device__ void elem(int64_t i, double* d) const {
        const double si = fma(-alpha, v[i], r[i]);
        s[i] = si;
        d[0] += si * si;
    }
    __device__ bool aligned16() const { return al16(r) && al16(v) && al16(s); }
    __device__ void elem2(int64_t j, double* d) const {
        const double2 rv = ld2(r, j), vv = ld2(v, j);
        const double2 sv = make_double2(fma(-alpha, vv.x, rv.x), fma(-alpha, vv.y, rv.y));
        st2(s, j, sv);
        d[0] += sv.x * sv.x;
        d[0] += sv.y * sv.y;
    }
};

struct VBiX {
    static constexpr int STREAMS = 9;  // n-vectors moved; half: x += alpha ph; else x += alpha ph + omega sh, r = s - omega t
    static constexpr int NDOT = 2;
    double* x;
    double* r;
    const double* ph;
    const double* sh;
    const double* s;
    const double* t;
    const double* rhat;
    const KState* ks;
    double alpha, omega;
    int32_t half;
    FinBiX fin;
    __device__ void prepare() {
        alpha = ks->alpha;
        omega = ks->omega;
        half = ks->half;
    }
    __device__ void elem(int64_t i, double* d) const {
        if (half) {
            x[i] = fma(alpha, ph[i], x[i]);
            return;
        }
        x[i] = fma(omega, sh[i], fma(alpha, ph[i], x[i]));
        const double rn = fma(-omega, t[i], s[i]);
        r[i] = rn;
        d[0] += rhat[i] * rn;
        d[1] += rn * rn;
    }
    __device__ bool aligned16() const {
        return al16(x) && al16(r) && al16(ph) && al16(sh) && al16(s) && al16(t) && al16(rhat);
    }
    __device__ void elem2(int64_t j, double* d) const {
        const double2 phv = ld2(ph, j);
        double2 xv = ld2(x, j);
        if (half) {
            st2(x, j, make_double2(fma(alpha, phv.x, xv.x), fma(alpha, phv.y, xv.y)));
            return;
        }
        const double2 shv = ld2(sh, j), sv = ld2(s, j), tv = ld2(t, j), hv = ld2(rhat, j);
        xv.x = fma(omega, shv.x, fma(alpha, phv.x, xv.x));
        xv.y = fma(omega, shv.y, fma(alpha, phv.y, xv.y));
        st2(x, j, xv);
        const double2 rn = make_double2(fma(-omega, tv.x, sv.x), fma(-omega, tv.y, sv.y));
        st2(r, j, rn);
        d[0] += hv.x * rn.x;
        d[1] += rn.x * rn.x;
        d[0] += hv.y * rn.y;
        d[1] += rn.y * rn.y;
    }
};

}  // namespace amgb
