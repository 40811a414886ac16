// Restarted right-preconditioned GMRES(m) on the device (PAPER.md:212 lists
// GMRES among the solvers).  Arnoldi with classical
// Gram-Schmidt applied twice (CGS2: the two passes are two fused multi-dot /
// multi-axpy kernel pairs instead of the 2(j+1) sequential kernels of modified
// Gram-Schmidt), Givens rotations and the small Hessenberg solve in one-thread
// finalizers, so the whole restart cycle runs on the device.  The oracle uses
// modified Gram-Schmidt; both are backward stable, results agree to rounding.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.cuh"

namespace amgb {

constexpr int kGmresMaxM = 64;

struct KStateG {
    double nf, tolnf, beta, hn;
    double H[(kGmresMaxM + 1) * kGmresMaxM];  // H[i*m + j]
    double g[kGmresMaxM + 1], cs[kGmresMaxM], sn[kGmresMaxM], y[kGmresMaxM];
    double coef[kGmresMaxM + 1];  // current Gram-Schmidt pass coefficients
    double hcol[kGmresMaxM + 1];  // accumulated column j of H
    int32_t m, maxiter, k, jlast, stop_step, done, status, cycles;
};

// partial[i * nchunks + chunk] = sum over the chunk of w * V_i  (grid: x = i, y = chunk)
__global__ void __launch_bounds__(kBlock) gmres_dots(const double* __restrict__ w, const double* __restrict__ V,
                                                     int64_t n, int64_t chunk, double* __restrict__ partial,
                                                     const int32_t* gate) {
    if (gated(gate)) return;
    const int i = blockIdx.x;
    const int64_t c0 = (int64_t)blockIdx.y * chunk, c1 = c0 + chunk < n ? c0 + chunk : n;
    const double* v = V + (int64_t)i * n;
    double s = 0.0;
    for (int64_t r = c0 + threadIdx.x; r < c1; r += blockDim.x) s += w[r] * v[r];
    __shared__ double sh[kBlock / 32];
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int q = 0; q < kBlock / 32; ++q) t += sh[q];
        partial[(int64_t)i * gridDim.y + blockIdx.y] = t;
    }
}

// coef[i] = sum over chunks (fixed order); hcol[i] = coef[i] (pass 0) or += (pass 1)
__global__ void gmres_dots_fin(const double* __restrict__ partial, int J, int nchunks, KStateG* ks, int pass,
                               const int32_t* gate) {
    if (gated(gate)) return;
    const int i = threadIdx.x;
    if (i >= J) return;
    double s = 0.0;
    for (int c = 0; c < nchunks; ++c) s += partial[(int64_t)i * nchunks + c];
    ks->coef[i] = s;
    ks->hcol[i] = pass == 0 ? s : ks->hcol[i] + s;
}

// Step j done: |w|, the new column of H through the Givens rotations, g
struct FinGmresStep {
    KStateG* ks;
    int j;
    __device__ void operator()(const double* t) const {
        const int m = ks->m;
        const double hn = sqrt(t[0]);
        ks->hn = hn;
        for (int i = 0; i <= j; ++i) ks->H[i * m + j] = ks->hcol[i];
        ks->H[(j + 1) * m + j] = hn;
        for (int i = 0; i < j; ++i) {
            const double a = ks->H[i * m + j], b = ks->H[(i + 1) * m + j];
            ks->H[i * m + j] = ks->cs[i] * a + ks->sn[i] * b;
            ks->H[(i + 1) * m + j] = -ks->sn[i] * a + ks->cs[i] * b;
        }
        const double a = ks->H[j * m + j], b = ks->H[(j + 1) * m + j];
        const double d = sqrt(a * a + b * b);
        ks->cs[j] = d == 0.0 ? 1.0 : a / d;
        ks->sn[j] = d == 0.0 ? 0.0 : b / d;
        ks->H[j * m + j] = d;
        ks->H[(j + 1) * m + j] = 0.0;
        ks->g[j + 1] = -ks->sn[j] * ks->g[j];
        ks->g[j] = ks->cs[j] * ks->g[j];
        ks->k += 1;
        ks->jlast = j;
        if (fabs(ks->g[j + 1]) <= ks->tolnf || ks->k >= ks->maxiter || hn == 0.0 || j == m - 1) ks->stop_step = 1;
    }
};

// w = w - sum_{i<J} coef_i V_i  [+ (w, w) -> FinGmresStep on the second pass]
template <int ND>
struct VGmresAxpy {
    static constexpr int NDOT = ND, STREAMS = 2;  // + J basis vectors (counted by the caller)
    double* w;
    const double* V;
    int64_t n;
    int J;
    const KStateG* ks;
    FinGmresStep fin;
    __device__ void prepare() {}
    __device__ void elem(int64_t r, double* d) const {
        double s = w[r];
        for (int i = 0; i < J; ++i) s -= ks->coef[i] * V[(int64_t)i * n + r];
        w[r] = s;
        if constexpr (ND > 0) d[0] += s * s;
    }
};

// v = w / hn
struct VGmresScale {
    static constexpr int NDOT = 0, STREAMS = 2;
    const double* w;
    double* v;
    const double* hn;
    NoFin fin;
    __device__ void prepare() {}
    __device__ void elem(int64_t r, double*) const { v[r] = w[r] / *hn; }
};

// y = H^-1 g (upper triangular, jlast+1 unknowns)
__global__ void gmres_solve_y(KStateG* ks, const int32_t* gate) {
    if (gated(gate)) return;
    const int m = ks->m, jl = ks->jlast;
    for (int i = jl; i >= 0; --i) {
        double s = ks->g[i];
        for (int q = i + 1; q <= jl; ++q) s -= ks->H[i * m + q] * ks->y[q];
        const double h = ks->H[i * m + i];
        if (h == 0.0) {
            ks->status = AMG_BREAKDOWN;
            ks->done = 1;
            ks->y[i] = 0.0;
            continue;
        }
        ks->y[i] = s / h;
    }
}

// u = sum_{i <= jlast} y_i V_i
struct VGmresCombine {
    static constexpr int NDOT = 0, STREAMS = 1;
    double* u;
    const double* V;
    int64_t n;
    const KStateG* ks;
    NoFin fin;
    __device__ void prepare() {}
    __device__ void elem(int64_t r, double*) const {
        double s = 0.0;
        const int J = ks->jlast + 1;
        for (int i = 0; i < J; ++i) s += ks->y[i] * V[(int64_t)i * n + r];
        u[r] = s;
    }
};

// x = x + z
struct VAdd {
    static constexpr int NDOT = 0, STREAMS = 3;
    double* x;
    const double* z;
    NoFin fin;
    __device__ void prepare() {}
    __device__ void elem(int64_t r, double*) const { x[r] = x[r] + z[r]; }
};

struct FinGmresNorm {  // |f| -> nf, tol |f|
    KStateG* ks;
    double tol;
    __device__ void operator()(const double* t) const {
        ks->nf = sqrt(t[0]);
        ks->tolnf = tol * ks->nf;
    }
};

// after r = f - A x: beta, convergence (true residual), start of the next cycle
struct FinGmresRestart {
    KStateG* ks;
    __device__ void operator()(const double* t) const {
        const double beta = sqrt(t[0]);
        ks->beta = beta;
        if (!(beta > ks->tolnf && ks->k < ks->maxiter)) ks->done = 1;
        ks->stop_step = ks->done;
        ks->jlast = -1;
        for (int i = 0; i <= ks->m; ++i) ks->g[i] = 0.0;
        ks->g[0] = beta;
        ks->hn = beta;  // v_0 = r / beta uses the same scale kernel
    }
};

}  // namespace amgb
