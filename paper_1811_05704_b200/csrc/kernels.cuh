// Device kernels of the solve phase (sm_100a).  Every kernel here is HBM-bound
// fp64 work (SpMV ~ 0.17 flop/B): no tensor cores; the design levers are
// coalesced loads, bytes in flight, fusion (one pass over A per smoother /
// residual / Krylov step) and keeping coarse levels in L2.  DESIGN.md §6 gives
// the roofline and the algorithmic bytes of each kernel.
//
// Matrix store: sliced ELLPACK with slice height 32 = one warp ("SELL-32").
// Row r lives in slice r/32, lane r%32; entry k of the row sits at
//   sptr[slice] + 32*k + lane,
// so the 32 threads of a warp read 32 consecutive doubles (256 B) and 32
// consecutive int32 (128 B) per step: fully coalesced for any row-length mix.
// Padding entries (k >= row length) carry value 0 and repeat the row's last
// column, so their gathers hit a cached line.  Entries of a row keep ascending
// column order, so each row sum runs in the order of the paper's CSR product.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace amgb {

constexpr int kBlock = 256;  // threads per block of every kernel
constexpr int kWarp = 32;

struct Sell {
    int64_t nrows = 0, ncols = 0, nslices = 0;
    const int64_t* sptr = nullptr;
    const int32_t* col = nullptr;
    const double* val = nullptr;
};

// Krylov scalars kept on the device between kernels.
struct KState {
    double nf, tolnf, res, rho, rho_prev, sigma, alpha, beta, omega, rhat_norm, true_res, ss;
    int32_t iter, maxiter, done, skip2, status, half;
};

// Deterministic single-pass grid reduction scratch: per-block partials + ticket.
struct Red {
    double* partial = nullptr;  // >= gridDim.x * 4
    unsigned int* ticket = nullptr;
};

// ---------------------------------------------------------------- loads
__device__ __forceinline__ double ld_stream(const double* p) { return __ldcs(p); }
__device__ __forceinline__ int32_t ld_stream(const int32_t* p) { return __ldcs(p); }
template <bool STREAM>
__device__ __forceinline__ double ld_mat(const double* p) {
    if constexpr (STREAM) return __ldcs(p); else return __ldg(p);
}
template <bool STREAM>
__device__ __forceinline__ int32_t ld_mat(const int32_t* p) {
    if constexpr (STREAM) return __ldcs(p); else return __ldg(p);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    return v;
}

// Block-reduce NV values (fixed tree: warp shuffles, then warp 0 over the
// per-warp results), write this block's partials, and let the last block to
// finish (ticket) sum all partials in block order and call fin(totals).  The
// summation order depends only on gridDim/blockDim, so results are bitwise
// reproducible run to run.
template <int NV, class Fin>
__device__ __forceinline__ void grid_reduce(double (&v)[NV], const Red& red, const Fin& fin) {
    __shared__ double sh[NV][kBlock / kWarp];
    __shared__ bool last;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int nw = blockDim.x >> 5;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
        double s = warp_sum(v[k]);
        if (lane == 0) sh[k][wid] = s;
    }
    __syncthreads();
    if (wid == 0) {
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            double s = lane < nw ? sh[k][lane] : 0.0;
            s = warp_sum(s);
            if (lane == 0) red.partial[blockIdx.x * NV + k] = s;
        }
        if (lane == 0) {
            __threadfence();
            unsigned t = atomicAdd(red.ticket, 1u);
            last = (t == gridDim.x - 1);
        }
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    double acc[NV];
#pragma unroll
    for (int k = 0; k < NV; ++k) acc[k] = 0.0;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) {
#pragma unroll
        for (int k = 0; k < NV; ++k) acc[k] += __ldcg(red.partial + b * NV + k);
    }
#pragma unroll
    for (int k = 0; k < NV; ++k) {
        double s = warp_sum(acc[k]);
        if (lane == 0) sh[k][wid] = s;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double tot[NV];
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            double s = 0.0;
            for (int w = 0; w < nw; ++w) s += sh[k][w];
            tot[k] = s;
        }
        fin(tot);
        *red.ticket = 0u;
        __threadfence();
    }
}

struct NoFin {
    __device__ void operator()(const double*) const {}
};

__device__ __forceinline__ bool gated(const int32_t* gate) {
    return gate != nullptr && *reinterpret_cast<const volatile int32_t*>(gate) != 0;
}

// ----------------------------------------------------------------- SELL row kernel
// One thread per row; U entries of the row are loaded before their gathers are
// issued (bytes in flight), then accumulated in ascending column order.
// Op supplies: NDOT (number of fused dot products), NEED_DIAG, prepare(),
// gather(col) -> value of the input vector at col (may fuse a vector op, e.g.
// m_j f_j or z_j + beta p_j), row(i, sum, diag, dots) -> epilogue, fin.
template <int U, bool STREAM, class Op>
__global__ void __launch_bounds__(kBlock) sell_rows(Sell A, Op op, const int32_t* gate, Red red) {
    if (gated(gate)) return;
    op.prepare();
    double dots[Op::NDOT > 0 ? Op::NDOT : 1];
#pragma unroll
    for (int k = 0; k < (Op::NDOT > 0 ? Op::NDOT : 1); ++k) dots[k] = 0.0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < A.nrows; row += stride) {
        const int64_t s = row >> 5;
        const int lane = (int)(row & 31);
        const int64_t beg = A.sptr[s];
        const int w = (int)((A.sptr[s + 1] - beg) >> 5);
        const int32_t* cp = A.col + beg + lane;
        const double* vp = A.val + beg + lane;
        double sum = 0.0, dg = 0.0;
        for (int k0 = 0; k0 < w; k0 += U) {
            int32_t c[U];
            double v[U], xv[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (k0 + u < w) {
                    c[u] = ld_mat<STREAM>(cp + 32 * (k0 + u));
                    v[u] = ld_mat<STREAM>(vp + 32 * (k0 + u));
                } else {
                    c[u] = 0;
                    v[u] = 0.0;
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) xv[u] = (k0 + u < w) ? op.gather(c[u]) : 0.0;
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (k0 + u < w) {
                    sum = fma(v[u], xv[u], sum);
                    if (Op::NEED_DIAG && c[u] == row && dg == 0.0) dg = v[u];
                }
            }
        }
        op.row(row, sum, dg, dots);
    }
    if constexpr (Op::NDOT > 0) grid_reduce<Op::NDOT>(dots, red, op.fin);
}

// ----------------------------------------------------------------- vector kernel
template <class Op>
__global__ void __launch_bounds__(kBlock) vec_kernel(int64_t n, Op op, const int32_t* gate, Red red) {
    if (gated(gate)) return;
    op.prepare();
    double dots[Op::NDOT > 0 ? Op::NDOT : 1];
#pragma unroll
    for (int k = 0; k < (Op::NDOT > 0 ? Op::NDOT : 1); ++k) dots[k] = 0.0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) op.elem(i, dots);
    if constexpr (Op::NDOT > 0) grid_reduce<Op::NDOT>(dots, red, op.fin);
}

// Dense GEMV y = M x (M row-major n x n): the coarsest-level solve with the
// host-computed inverse (Algorithm 2 "solve the coarsest system directly",
// PAPER.md:128).  One warp per row, coalesced row reads, x from L1/L2.
__global__ void __launch_bounds__(kBlock) dense_gemv(int64_t n, const double* __restrict__ M,
                                                     const double* __restrict__ x, double* __restrict__ y,
                                                     const int32_t* gate);

// ----------------------------------------------------------------- epilogue ops
// Each op declares its algorithmic traffic: a pass over M (rows x
// cols, nnz) moves 12 nnz + 4 rows (CSR-equivalent matrix bytes) + 8 cols per
// gathered vector (each read once, ideal reuse) + 8 rows per row-indexed vector
// read or written.
// y = A x
struct OpSpmv {
    static constexpr int GATHER = 1, ROWV = 1;  // vectors gathered / row-indexed (bytes model)
    static constexpr int NDOT = 0;
    static constexpr bool NEED_DIAG = false;
    const double* x;
    double* y;
    NoFin fin;
    __device__ void prepare() {}
    __device__ double gather(int32_t c) const { return __ldg(x + c); }
    __device__ void row(int64_t i, double s, double, double*) const { y[i] = s; }
};

// y = f - A x  [+ (y, y)]
template <int ND, class Fin>
struct OpResidual {
    static constexpr int GATHER = 1, ROWV = 2;  // vectors gathered / row-indexed (bytes model)
    static constexpr int NDOT = ND;
    static constexpr bool NEED_DIAG = false;
    const double* x;
    const double* f;
    double* y;
    Fin fin;
    __device__ void prepare() {}
    __device__ double gather(int32_t c) const { return __ldg(x + c); }
    __device__ void row(int64_t i, double s, double, double* d) const {
        double r = f[i] - s;
        y[i] = r;
        if constexpr (ND > 0) d[0] += r * r;
    }
};

// Zero-start smoother + residual (a1): with x = m o f (the first SPAI-0/Jacobi
// sweep from x = 0), t = f - A x, computing x_j = m_j f_j inside the gather.
struct OpRes0 {
    static constexpr int GATHER = 2, ROWV = 1;  // vectors gathered / row-indexed (bytes model)
    static constexpr int NDOT = 0;
    static constexpr bool NEED_DIAG = false;
    const double* m;
    const double* f;
    double* t;
    NoFin fin;
    __device__ void prepare() {}
    __device__ double gather(int32_t c) const { return __ldg(m + c) * __ldg(f + c); }
    __device__ void row(int64_t i, double s, double, double*) const { t[i] = f[i] - s; }
};

// Damped-Jacobi / SPAI-0 sweep (a6): xo = x + m o (f - A x), optional (f, xo).
template <int ND, class Fin>
struct OpRelax {
    static constexpr int GATHER = 1, ROWV = 3;  // vectors gathered / row-indexed (bytes model)
    static constexpr int NDOT = ND;
    static constexpr bool NEED_DIAG = false;
    const double* x;
    const double* m;
    const double* f;
    double* xo;
    Fin fin;
    __device__ void prepare() {}
    __device__ double gather(int32_t c) const { return __ldg(x + c); }
    __device__ void row(int64_t i, double s, double, double* d) const {
        const double fi = f[i];
        const double xn = x[i] + m[i] * (fi - s);
        xo[i] = xn;
        if constexpr (ND > 0) d[0] += fi * xn;
    }
};

// Prolongation-correction after a zero-start sweep (a5): x = m o f + P e.
struct OpProl0 {
    static constexpr int GATHER = 1, ROWV = 3;  // vectors gathered / row-indexed (bytes model)
    static constexpr int NDOT = 0;
    static constexpr bool NEED_DIAG = false;
    const double* e;
    const double* m;
    const double* f;
    double* x;
    NoFin fin;
    __device__ void prepare() {}
    __device__ double gather(int32_t c) const { return __ldg(e + c); }
    __device__ void row(int64_t i, double s, double, double*) const { x[i] = m[i] * f[i] + s; }
};

// General prolongation-correction: x = x + P e (x updated in place, row-local).
struct OpProlAdd {
    static constexpr int GATHER = 1, ROWV = 2;  // vectors gathered / row-indexed (bytes model)
    static constexpr int NDOT = 0;
    static constexpr bool NEED_DIAG = false;
    const double* e;
    double* x;
    NoFin fin;
    __device__ void prepare() {}
    __device__ double gather(int32_t c) const { return __ldg(e + c); }
    __device__ void row(int64_t i, double s, double, double*) const { x[i] = x[i] + s; }
};

// One Chebyshev step (§8c c-1): r = f - A x; scaled: r = r / a_ii (a_ii read from
// the row itself); p = alpha r + beta p (first step: p = alpha r); xo = x + p.
template <int ND, class Fin>
struct OpCheb {
    static constexpr int GATHER = 1, ROWV = 4;  // vectors gathered / row-indexed (bytes model)
    static constexpr int NDOT = ND;
    static constexpr bool NEED_DIAG = true;
    const double* x;
    const double* f;
    double* p;
    double* xo;
    double alpha, beta;
    int32_t scaled, first;
    Fin fin;
    __device__ void prepare() {}
    __device__ double gather(int32_t c) const { return __ldg(x + c); }
    __device__ void row(int64_t i, double s, double dg, double* d) const {
        double r = f[i] - s;
        if (scaled) r = r / dg;
        const double pn = first ? alpha * r : alpha * r + beta * p[i];
        p[i] = pn;
        const double xn = x[i] + pn;
        xo[i] = xn;
        if constexpr (ND > 0) d[0] += f[i] * xn;
    }
};

// CG direction + SpMV (a7): p' = z + beta p (formed inside the gather), q = A p',
// sigma = (p', q).
template <class Fin>
struct OpCgDir {
    static constexpr int GATHER = 2, ROWV = 2;  // vectors gathered / row-indexed (bytes model)
    static constexpr int NDOT = 1;
    static constexpr bool NEED_DIAG = false;
    const double* z;
    const double* p;
    double* pn;
    double* q;
    const KState* ks;
    double beta;
    Fin fin;
    __device__ void prepare() { beta = ks->beta; }
    __device__ double gather(int32_t c) const { return fma(beta, __ldg(p + c), __ldg(z + c)); }
    __device__ void row(int64_t i, double s, double, double* d) {
        const double pi = fma(beta, p[i], z[i]);
        pn[i] = pi;
        q[i] = s;
        d[0] += pi * s;
    }
};

// y = A x with dots: ND = 1: (w, y); ND = 2: (y, y), (y, w).
template <int ND, class Fin>
struct OpSpmvDot {
    static constexpr int GATHER = 1, ROWV = 2;  // vectors gathered / row-indexed (bytes model)
    static constexpr int NDOT = ND;
    static constexpr bool NEED_DIAG = false;
    const double* x;
    const double* w;
    double* y;
    Fin fin;
    __device__ void prepare() {}
    __device__ double gather(int32_t c) const { return __ldg(x + c); }
    __device__ void row(int64_t i, double s, double, double* d) const {
        y[i] = s;
        if constexpr (ND == 1) {
            d[0] += w[i] * s;
        } else {
            d[0] += s * s;
            d[1] += s * w[i];
        }
    }
};

}  // namespace amgb
