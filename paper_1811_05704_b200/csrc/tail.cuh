// The coarse end of the V-cycle in ONE cooperative kernel ("tail cycle").
//
// Below a level Lt every matrix is small (row-block CSR format, L2-resident:
// levels >= 3 at 256^3, the whole hierarchy of a 32^3 problem), so each pass of
// Algorithm 2 there is a few microseconds of work behind a
// launch and a drain.  The tail kernel runs the recursion from Lt down to the
// coarsest solve and back up -- zero-start residual, restriction, dense coarse
// GEMV, prolongation, post-smoothing (and at level 0 the fused rho = (f, x')) --
// as a list of steps separated by grid-wide barriers (cooperative launch, all
// blocks co-resident).  Every step is the same arithmetic as the launch it
// replaces (ops of kernels.cuh, products in ascending column order per row
// group, then a fixed xor-shuffle tree), so the tail is a drop-in for those
// launches; only the order of the partial sums inside a row differs.
#pragma once
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.cuh"

namespace amgb {

enum TailOp : int32_t {
    kTailRes0 = 0,     // y = f - A (m o f)
    kTailRes0MF = 1,   // y = f - A mf             (b = mf)
    kTailSpmv = 2,     // y = A a
    kTailSpmvMF = 3,   // y = A a, y2 = m o y      (m = next level's diagonal)
    kTailGemv = 4,     // y = Mdense f
    kTailProl0 = 5,    // y = m o f + A a
    kTailProl0MF = 6,  // y = b + A a              (b = mf)
    kTailRelax = 7,    // y = b + m o (f - A b)    (b = x)
};

struct TailStep {
    int32_t op = 0;
    int32_t G = 1;                 // threads per row (power of 2 <= 32)
    int64_t nrows = 0;
    const int32_t* ptr = nullptr;  // CSR (int32 row pointers); dense: nullptr
    const int32_t* col = nullptr;
    const double* val = nullptr;   // CSR values, or the dense row-major matrix (kTailGemv)
    const double* a = nullptr;     // gathered input vector
    const double* b = nullptr;     // mf / x (row-local, or gathered for kTailRes0MF / kTailRelax)
    const double* f = nullptr;     // row-local right-hand side
    const double* m = nullptr;     // smoother diagonal (row-local; gathered for kTailRes0)
    double* y = nullptr;
    double* y2 = nullptr;
};

constexpr int kTailMax = 40;  // steps per launch (4 per level + the coarse solve)

struct TailProg {
    int32_t nsteps = 0;
    int32_t rho_step = -1;  // the step whose (f, y) is reduced into rho (CG, level 0), -1: none
    TailStep s[kTailMax];
};

// The program travels by value in the kernel parameters (about 3.5 KB; graph
// capture keeps a copy), so every call site can name its own top-level f / out.
template <class Fin>
__global__ void __launch_bounds__(kBlock) tail_cycle(const __grid_constant__ TailProg prog, const int32_t* gate,
                                                     double* partial, Fin fin) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    if (gated(gate)) return;  // uniform across the grid: before any barrier
    const int tid = (int)(blockIdx.x * blockDim.x + threadIdx.x);
    const int nthreads = (int)(gridDim.x * blockDim.x);
    double dot = 0.0;
    for (int q = 0; q < prog.nsteps; ++q) {
        const TailStep& S = prog.s[q];
        if (S.op == kTailGemv) {  // warp per row, coalesced dense rows
            const int lane = tid & 31, w = tid >> 5, nw = nthreads >> 5;
            for (int64_t r = w; r < S.nrows; r += nw) {
                const double* row = S.val + r * S.nrows;
                double s = 0.0;
                for (int64_t j = lane; j < S.nrows; j += 32) s = fma(__ldg(row + j), S.f[j], s);
                s = warp_sum(s);
                if (lane == 0) S.y[r] = s;
            }
        } else {
            const int G = S.G;
            const int lig = tid & (G - 1);
            const unsigned gmask = G == 32 ? 0xffffffffu : (((1u << G) - 1u) << ((threadIdx.x & 31) & ~(G - 1)));
            const int64_t groups = nthreads / G;
            for (int64_t r = tid / G; r < S.nrows; r += groups) {
                double s = 0.0;
                const int32_t k1 = S.ptr[r + 1];
                for (int32_t k = S.ptr[r] + lig; k < k1; k += G) {
                    const int32_t c = S.col[k];
                    double xv;
                    if (S.op == kTailRes0) xv = S.m[c] * S.f[c];
                    else if (S.op == kTailRes0MF || S.op == kTailRelax) xv = S.b[c];
                    else xv = S.a[c];
                    s = fma(S.val[k], xv, s);
                }
#pragma unroll
                for (int o = 1; o < 32; o <<= 1)
                    if (o < G) s += __shfl_xor_sync(gmask, s, o);
                if (lig != 0) continue;
                switch (S.op) {
                    case kTailRes0:
                    case kTailRes0MF: S.y[r] = S.f[r] - s; break;
                    case kTailSpmv: S.y[r] = s; break;
                    case kTailSpmvMF:
                        S.y[r] = s;
                        S.y2[r] = S.m[r] * s;
                        break;
                    case kTailProl0: S.y[r] = S.m[r] * S.f[r] + s; break;
                    case kTailProl0MF: S.y[r] = S.b[r] + s; break;
                    default: {  // kTailRelax
                        const double fi = S.f[r];
                        const double xn = S.b[r] + S.m[r] * (fi - s);
                        S.y[r] = xn;
                        if (q == prog.rho_step) dot += fi * xn;
                    }
                }
            }
        }
        if (q + 1 < prog.nsteps) grid.sync();
    }
    if (prog.rho_step < 0) return;
    // rho = (f, x'): fixed-order block tree, then block 0 sums the partials in
    // block order (deterministic), then the finalizer
    __shared__ double sh[kBlock / 32];
    dot = warp_sum(dot);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = dot;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < kBlock / 32; ++w) s += sh[w];
        partial[blockIdx.x] = s;
    }
    grid.sync();
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        double s = 0.0;
        for (int b = 0; b < (int)gridDim.x; ++b) s += partial[b];
        double t[1] = {s};
        fin(t);
    }
}

}  // namespace amgb
