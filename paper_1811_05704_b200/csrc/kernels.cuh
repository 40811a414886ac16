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

#include <cassert>
#include <cstdint>
#include <type_traits>
#include <utility>

namespace amgb {

// Bounds-checked build (make check -> _lib_chk/libamgb.so, -DAMGB_BOUNDS_CHECK):
// every gathered column index and every TMA stage range is asserted on the
// device (a failing assert aborts the kernel with cudaErrorAssert), in lieu of
// compute-sanitizer, which is closed on this pool.
#ifdef AMGB_BOUNDS_CHECK
#define AMGB_ASSERT(c) assert(c)
#else
#define AMGB_ASSERT(c) ((void)0)
#endif

constexpr int kBlock = 256;  // threads per block of every kernel
constexpr int kWarp = 32;

struct Sell {
    int64_t nrows = 0, ncols = 0, nslices = 0;
    int64_t row0 = 0;  // first row of this (sub-)matrix view: row = row0 + local row
    const int64_t* sptr = nullptr;
    const int32_t* col = nullptr;
    const double* val = nullptr;
    const float* valf = nullptr;  // fp32 copy of val (mixed-precision V-cycle)
    // SELL-C-sigma (amgb.cu sigma_sort): slot s holds row (s & ~255) + rperm[s];
    // nullptr = slots are rows
    const uint8_t* rperm = nullptr;
    // value-indexed storage (amgb.cu value_index): entry k's value is
    // vtab[vi8[k]] (<= 256 distinct values) or vtab[vi16[k]] (<= 65536); val unused
    const double* vtab = nullptr;
    const uint8_t* vi8 = nullptr;
    const uint16_t* vi16 = nullptr;
};

// stored slot -> matrix row of a SELL-C-sigma matrix (rows sorted by length
// inside aligned 256-row windows); the identity without a permutation
__device__ __forceinline__ int64_t slot_row(const uint8_t* rperm, int64_t slot) {
    return rperm ? (slot & ~(int64_t)255) + (int64_t)__ldg(rperm + slot) : slot;
}

// Krylov scalars kept on the device between kernels.
struct KState {
    double nf, tolnf, res, rho, rho_prev, sigma, alpha, beta, omega, rhat_norm, true_res, ss;
    int32_t iter, maxiter, done, skip2, status, half;
    int32_t upd;    // fused CG: alpha of this iteration awaits its r update (next res0)
    int32_t xpend;  // fused CG: an applied r update awaits its x update (next CG direction)
};

// Deterministic single-pass grid reduction scratch: per-block partials + ticket.
struct Red {
    double* partial = nullptr;  // >= gridDim.x * 4
    unsigned int* ticket = nullptr;
    double* defer = nullptr;    // multi-rank: store the block-summed totals here
                                // (all-reduced, then finalized by fin_kernel)
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
template <bool STREAM>
__device__ __forceinline__ float ld_mat(const float* p) {
    if constexpr (STREAM) return __ldcs(p); else return __ldg(p);
}
// matrix value k of a store: fp64, or the fp32 copy widened to fp64 (F32)
template <bool STREAM, bool F32, class M>
__device__ __forceinline__ double ld_val(const M& A, int64_t k) {
    if constexpr (F32) return (double)ld_mat<STREAM>(A.valf + k); else return ld_mat<STREAM>(A.val + k);
}
__device__ __forceinline__ uint32_t ld_idx8(const uint8_t* p) { return __ldcs(reinterpret_cast<const unsigned char*>(p)); }
__device__ __forceinline__ uint32_t ld_idx16(const uint16_t* p) { return __ldcs(reinterpret_cast<const unsigned short*>(p)); }
// value k of a SELL store in its storage mode (VM: 0 = the value array / its
// fp32 copy, 1 = 8-bit index into vtab, 2 = 16-bit index); the table is small
// and read through L1
template <int VM, bool STREAM, bool F32>
__device__ __forceinline__ double ld_sell_val(const Sell& A, int64_t k) {
    if constexpr (VM == 1) return __ldg(A.vtab + ld_idx8(A.vi8 + k));
    else if constexpr (VM == 2) return __ldg(A.vtab + ld_idx16(A.vi16 + k));
    else return ld_val<STREAM, F32>(A, k);
}

// Accumulator of a row kernel: one double (single right-hand side) or Vk<K> (K
// interleaved right-hand sides of a batched solve, x[c*K + j]).  Ops return
// their accumulator type from gather(); the kernels are written once for both.
template <int K>
struct Vk {
    double v[K];
};
template <class Op>
using acc_t = decltype(std::declval<Op>().gather(0));
// gather with the bounds check of the checked build (column in [0, ncols))
template <class Op>
__device__ __forceinline__ acc_t<Op> gather_chk(const Op& op, int32_t c, int64_t ncols) {
    AMGB_ASSERT(c >= 0 && (int64_t)c < ncols);
    (void)ncols;
    return op.gather(c);
}
// columns carried by an op's accumulator (1 = single right-hand side)
template <class Op>
constexpr int cols_of() { return (int)(sizeof(acc_t<Op>) / sizeof(double)); }
// entries in flight per thread: 8 gathers for one column, fewer for K columns
// (each gather already moves K doubles; keeps the register file from spilling)
template <class Op>
constexpr int unroll_of(int u1) { return cols_of<Op>() == 1 ? u1 : (cols_of<Op>() == 2 ? 4 : (cols_of<Op>() == 4 ? 2 : 1)); }
// resident blocks requested per SM (launch bounds)
template <class Op>
constexpr int minb_of(int b1) { return cols_of<Op>() == 1 ? b1 : (cols_of<Op>() <= 4 ? 3 : 2); }
__device__ __forceinline__ void fma_acc(double& s, double a, double x) { s = fma(a, x, s); }
template <int K>
__device__ __forceinline__ void fma_acc(Vk<K>& s, double a, const Vk<K>& x) {
#pragma unroll
    for (int j = 0; j < K; ++j) s.v[j] = fma(a, x.v[j], s.v[j]);
}
__device__ __forceinline__ double shfl_xor_acc(unsigned m, double s, int o) { return __shfl_xor_sync(m, s, o); }
template <int K>
__device__ __forceinline__ Vk<K> shfl_xor_acc(unsigned m, const Vk<K>& s, int o) {
    Vk<K> r;
#pragma unroll
    for (int j = 0; j < K; ++j) r.v[j] = __shfl_xor_sync(m, s.v[j], o);
    return r;
}
__device__ __forceinline__ void add_acc(double& s, double x) { s += x; }
template <int K>
__device__ __forceinline__ void add_acc(Vk<K>& s, const Vk<K>& x) {
#pragma unroll
    for (int j = 0; j < K; ++j) s.v[j] += x.v[j];
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
    __shared__ double sh[NV][32];
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
        if (red.defer) {
            for (int k = 0; k < NV; ++k) red.defer[k] = tot[k];
        } else {
            fin(tot);
        }
        *red.ticket = 0u;
        __threadfence();
    }
}

struct NoFin {
    __device__ void operator()(const double*) const {}
};

// Programmatic dependent launch (sm_90+): a kernel launched with the
// programmatic-stream-serialization attribute may start while its predecessor
// finishes; pdl_wait() blocks until the predecessor grid has completed and its
// writes are visible (a no-op for normal launches), pdl_trigger() lets the
// successor start launching once every block of this grid has triggered.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ bool gated(const int32_t* gate) {
    return gate != nullptr && *reinterpret_cast<const volatile int32_t*>(gate) != 0;
}

// ----------------------------------------------------------------- SELL row kernel
// One thread per row; U entries of the row are loaded before their gathers are
// issued (bytes in flight), the next U entries are requested before this
// chunk's products are accumulated (software pipelining), and the sum runs in
// ascending column order.
// Op supplies: NDOT (number of fused dot products), prepare(), load(i) -> the
// row-local operands of the epilogue (Row), gather(col) -> value of the input
// vector at col (may fuse a vector op, e.g. m_j f_j or z_j + beta p_j),
// row(i, sum, Row, dots) -> epilogue, fin.
// PIPE = false: all U entries of the (narrow, w <= U) row in one chunk, no
// prefetch registers; launch bounds ask for >= 6 resident blocks (48 warps) so
// enough loads are in flight per SM.
template <int VM, int U, bool STREAM, bool PIPE, bool F32, class Op, int ND>
__device__ __forceinline__ void sell_rows_body(const Sell& A, Op& op, double (&dots)[ND]) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < A.nrows; row += stride) {
        // row-local epilogue operands are requested first, so their latency
        // overlaps the matrix stream (single column; K-column rows load later)
        typename Op::Row rr{};
        const int64_t grow = A.row0 + slot_row(A.rperm, row);  // global row (views of a split pass)
        if constexpr (cols_of<Op>() == 1) rr = op.load(grow);
        const int64_t s = row >> 5;
        const int lane = (int)(row & 31);
        const int64_t beg = A.sptr[s];
        const int w = (int)((A.sptr[s + 1] - beg) >> 5);
        const int32_t* cp = A.col + beg + lane;
        const int64_t vb = beg + lane;
        acc_t<Op> sum{};
        int32_t c[U];
        double v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            c[u] = u < w ? ld_mat<STREAM>(cp + 32 * u) : 0;
            v[u] = u < w ? ld_sell_val<VM, STREAM, F32>(A, vb + 32 * u) : 0.0;
        }
        if constexpr (!PIPE) {
            acc_t<Op> xv[U];
#pragma unroll
            for (int u = 0; u < U; ++u) xv[u] = u < w ? gather_chk(op, c[u], A.ncols) : acc_t<Op>{};
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (u < w) fma_acc(sum, v[u], xv[u]);
        }
        for (int k0 = 0; PIPE && k0 < w; k0 += U) {
            acc_t<Op> xv[U];
#pragma unroll
            for (int u = 0; u < U; ++u) xv[u] = (k0 + u < w) ? gather_chk(op, c[u], A.ncols) : acc_t<Op>{};
            // software pipelining: the next chunk's entries are in flight while
            // this chunk's gathers complete
            int32_t cn[U];
            double vn[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int k = k0 + U + u;
                cn[u] = k < w ? ld_mat<STREAM>(cp + 32 * k) : 0;
                vn[u] = k < w ? ld_sell_val<VM, STREAM, F32>(A, vb + 32 * k) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (k0 + u < w) fma_acc(sum, v[u], xv[u]);
#pragma unroll
            for (int u = 0; u < U; ++u) {
                c[u] = cn[u];
                v[u] = vn[u];
            }
        }
        if constexpr (cols_of<Op>() > 1) rr = op.load(grow);
        op.row(grow, sum, rr, dots);
    }
}

template <int U1, bool STREAM, bool PIPE, class Op, bool F32 = false>
__global__ void __launch_bounds__(kBlock, minb_of<Op>(PIPE ? 4 : 6)) sell_rows(Sell A, Op op, const int32_t* gate,
                                                                                 Red red) {
    constexpr int U = unroll_of<Op>(U1);
    pdl_wait();
    if (gated(gate)) return;
    op.prepare();
    constexpr int ND = Op::NDOT > 0 ? Op::NDOT : 1;
    double dots[ND];
#pragma unroll
    for (int k = 0; k < ND; ++k) dots[k] = 0.0;
    if (A.vi8 && !F32)
        sell_rows_body<1, U, STREAM, PIPE, F32>(A, op, dots);
    else if (A.vi16 && !F32)
        sell_rows_body<2, U, STREAM, PIPE, F32>(A, op, dots);
    else
        sell_rows_body<0, U, STREAM, PIPE, F32>(A, op, dots);
    pdl_trigger();
    if constexpr (Op::NDOT > 0) grid_reduce<Op::NDOT>(dots, red, op.fin);
}

// ----------------------------------------------------------------- TMA-staged SELL-C kernel
// The matrix stream is decoupled from the register file: a producer warp moves
// whole tiles (8 consecutive slices; their col and val ranges are contiguous)
// into a kTmaStages-deep shared-memory ring with cp.async.bulk (TMA bulk
// copies, completion counted in bytes on an mbarrier), while 8 consumer warps
// read entries from shared memory, issue the gathers and run the fused
// epilogue.  Matrices are stored as SELL-C with slice height C = 32/T: warp w
// owns slice w of the tile, lane l works on row l % C, entries k = l / C + T j
// (T lanes per row).  Entry k of row r sits at slice_off + k C + r, so the 32
// lanes of a warp read 32 consecutive words (conflict-free) and the T partial
// sums of a row are combined with xor-shuffles in a fixed order.
constexpr int kTmaStages = 2;
constexpr int kTmaBlocksPerSM = 4;
constexpr int kTmaThreads = kBlock + 32;  // 8 consumer warps + 1 producer warp

struct SellTma {
    int64_t nrows = 0, ncols = 0, nslices = 0, ntiles = 0;
    int64_t row0 = 0;  // first row of this (sub-)matrix view (a multiple of 256)
    const int64_t* sptr = nullptr;  // nslices + 1 element offsets (multiples of C)
    const int64_t* cptr = nullptr;  // nslices + 1 offsets into col (offset dictionary, amgb.cu tma_cols)
    const int32_t* col = nullptr;
    const double* val = nullptr;
    const float* valf = nullptr;    // fp32 copy of val (mixed-precision V-cycle)
    int32_t T = 1;          // lanes per row; slice height C = 32 / T
    int32_t tile_ent = 0;   // capacity of one stage in entries (max over tiles)
    const uint8_t* rperm = nullptr;  // SELL-C-sigma slot -> row (T = 1: window = tile); see Sell
    // value-indexed storage (<= 256 distinct values): the stage carries 1-byte
    // indices, the kernel keeps the table in shared memory; val unused
    const double* vtab = nullptr;
    const uint8_t* vi8 = nullptr;
};

// shared-memory bytes of the value table of an indexed TMA store
constexpr int kVTabBytes = 256 * 8;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t a) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t a, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
// try_wait with a suspend-time hint: the waiting thread is suspended until the
// phase completes (or the hint elapses) instead of re-issuing the test -- a
// spinning producer lane otherwise costs its warp an issue slot per test
// (12 % of the level-0 pass's instructions before, ncu round 2)
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity) {
    uint32_t ok = 0;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
            " selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(ok)
            : "r"(a), "r"(parity), "r"(1000000u)
            : "memory");
    } while (!ok);
}
template <bool STREAM>
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t mbar,
                                         uint64_t policy) {
    if constexpr (STREAM)
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
            " [%0], [%1], %2, [%3], %4;" ::"r"(dst),
            "l"(src), "r"(bytes), "r"(mbar), "l"(policy)
            : "memory");
    else
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
            "l"(src), "r"(bytes), "r"(mbar)
            : "memory");
}

template <int T, bool STREAM, class Op, bool F32 = false>
__global__ void __launch_bounds__(kTmaThreads, minb_of<Op>(kTmaBlocksPerSM)) sell_tma(SellTma A, Op op,
                                                                                      const int32_t* gate, Red red) {
    using VT = std::conditional_t<F32, float, double>;
    constexpr int VB = (int)sizeof(VT);
    constexpr int UN = unroll_of<Op>(8);
    pdl_wait();
    if (gated(gate)) return;
    op.prepare();
    constexpr int C = 32 / T;  // slice height
    constexpr int NS = 8;      // slices per tile (one per consumer warp)
    extern __shared__ __align__(128) unsigned char smem_raw[];
    // layout: [value table (indexed stores)] kTmaStages x { val[tile_ent] (VB bytes, or
    // 1-byte indices), col[tile_ent] (4 B) } | barriers
    const bool vix = !F32 && A.vi8 != nullptr;
    double* vtab_s = reinterpret_cast<double*>(smem_raw);
    unsigned char* smem = smem_raw + (vix ? kVTabBytes : 0);
    const int vbytes = vix ? 1 : VB;
    const int te = A.tile_ent;
    const size_t stage_bytes = (size_t)te * (vbytes + 4);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kTmaStages * stage_bytes);  // full[S], empty[S]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (vix)
        for (int k = threadIdx.x; k < 256; k += blockDim.x) vtab_s[k] = __ldg(A.vtab + k);
    if (threadIdx.x == 0) {
        for (int s = 0; s < kTmaStages; ++s) {
            mbar_init(smem_u32(bars + s), 1);
            mbar_init(smem_u32(bars + kTmaStages + s), kBlock / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    constexpr int ND = Op::NDOT > 0 ? Op::NDOT : 1;
    double dots[ND];
#pragma unroll
    for (int k = 0; k < ND; ++k) dots[k] = 0.0;

    if (warp == kBlock / 32) {  // ---------------- producer warp
        if (lane == 0) {
            uint64_t policy = 0;
            if constexpr (STREAM) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
            int i = 0;
            for (int64_t t = blockIdx.x; t < A.ntiles; t += gridDim.x, ++i) {
                const int s = i % kTmaStages;
                if (i >= kTmaStages) mbar_wait(smem_u32(bars + kTmaStages + s), ((i / kTmaStages) & 1) ^ 1);
                const int64_t s0 = t * NS;
                const int64_t s1 = s0 + NS < A.nslices ? s0 + NS : A.nslices;
                const int64_t e0 = A.sptr[s0], e1 = A.sptr[s1];
                const int64_t c0 = A.cptr[s0], c1 = A.cptr[s1];
                const uint32_t n = (uint32_t)(e1 - e0), nc = (uint32_t)(c1 - c0);
                AMGB_ASSERT(e1 >= e0 && c1 >= c0 && n <= (uint32_t)te && nc <= (uint32_t)te);
                const uint32_t full = smem_u32(bars + s);
                unsigned char* st = smem + (size_t)s * stage_bytes;
                mbar_expect_tx(full, n * (uint32_t)vbytes + nc * 4u);
                if (vix)
                    bulk_g2s<STREAM>(smem_u32(st), A.vi8 + e0, n, full, policy);
                else if constexpr (F32)
                    bulk_g2s<STREAM>(smem_u32(st), A.valf + e0, n * 4u, full, policy);
                else
                    bulk_g2s<STREAM>(smem_u32(st), A.val + e0, n * 8u, full, policy);
                if (nc) bulk_g2s<STREAM>(smem_u32(st + (size_t)te * vbytes), A.col + c0, nc * 4u, full, policy);
            }
        }
    } else {  // ------------------------------------ consumer warps
        const int r = lane % C;  // row within the slice
        const int pt = lane / C; // part of the row
        // loop-invariant addresses and flags, hoisted out of the tile loop
        const uint32_t bar_full0 = smem_u32(bars), bar_empty0 = smem_u32(bars + kTmaStages);
        const bool sorted = A.rperm != nullptr;
        const int nslices = (int)A.nslices, nrows = (int)A.nrows, ntiles = (int)A.ntiles;
        // slice offsets as 32-bit low words (their differences fit in 32 bits;
        // the arrays are little-endian int64), loaded one tile ahead so their
        // latency is off the critical path
        const uint32_t* sp32 = reinterpret_cast<const uint32_t*>(A.sptr);
        const uint32_t* cp32 = reinterpret_cast<const uint32_t*>(A.cptr);
        struct SliceOff {
            uint32_t e0 = 0, e1 = 0, eb = 0, c0 = 0, c1 = 0, cb = 0;
        };
        auto load_off = [&](int t) {
            SliceOff o;
            const int slice = t * NS + warp;
            if (t < ntiles && slice < nslices) {
                o.e0 = __ldg(sp32 + 2 * slice);
                o.e1 = __ldg(sp32 + 2 * slice + 2);
                o.eb = __ldg(sp32 + 2 * (t * NS));
                o.c0 = __ldg(cp32 + 2 * slice);
                o.c1 = __ldg(cp32 + 2 * slice + 2);
                o.cb = __ldg(cp32 + 2 * (t * NS));
            }
            return o;
        };
        SliceOff nxt = load_off((int)blockIdx.x);
        int i = 0;
        for (int t = (int)blockIdx.x; t < ntiles; t += (int)gridDim.x, ++i) {
            const int s = i % kTmaStages;
            const int slice = t * NS + warp;
            const int lrow = slice * C + r;
            const bool has_row = slice < nslices && lrow < nrows;
            // global row (views of a split pass); a sorted matrix has no
            // dictionary slices, so `row` is only the epilogue's index there
            const int64_t row = A.row0 + (int64_t)((has_row && sorted) ? (int)slot_row(A.rperm, lrow) : lrow);
            typename Op::Row rr{};
            if constexpr (cols_of<Op>() == 1)
                if (pt == 0 && has_row) rr = op.load(row);  // in flight during the wait
            const SliceOff cur = nxt;
            nxt = load_off(t + (int)gridDim.x);
            int off = 0, w = 0, coff = 0;
            bool dict = false;  // the slice's columns are row + a shared offset list
            if (slice < nslices) {
                off = (int)(cur.e0 - cur.eb);
                w = (int)(cur.e1 - cur.e0) / C;
                coff = (int)(cur.c0 - cur.cb);
                dict = (int)(cur.c1 - cur.c0) < C * w;
            }
            mbar_wait(bar_full0 + 8 * s, (i / kTmaStages) & 1);
            const unsigned char* st = smem + (size_t)s * stage_bytes;
            const VT* sv = reinterpret_cast<const VT*>(st) + off + r;
            const uint8_t* si = st + off + r;
            const int32_t* sc = reinterpret_cast<const int32_t*>(st + (size_t)te * vbytes) + coff + (dict ? 0 : r);
            acc_t<Op> sum{};
            // entry k's column: sc[CS k] (+ row for a dictionary slice); the
            // stride is a template constant so every load is an immediate offset;
            // its value: sv[C k], or the table entry of the index si[C k]
            auto run = [&](auto cs, int32_t cbase, auto vx) {
                constexpr int CS = decltype(cs)::value;
                constexpr bool VX = decltype(vx)::value;
                for (int k0 = pt; k0 < w; k0 += UN * T) {
                    acc_t<Op> xv[UN];
                    int32_t c[UN];
#pragma unroll
                    for (int u = 0; u < UN; ++u) {
                        const int k = k0 + u * T;
                        c[u] = k < w ? sc[CS * k] + cbase : 0;
                    }
#pragma unroll
                    for (int u = 0; u < UN; ++u) xv[u] = (k0 + u * T < w) ? gather_chk(op, c[u], A.ncols) : acc_t<Op>{};
#pragma unroll
                    for (int u = 0; u < UN; ++u) {
                        const int k = k0 + u * T;
                        if constexpr (VX) {
                            if (k < w) fma_acc(sum, vtab_s[si[C * k]], xv[u]);
                        } else {
                            if (k < w) fma_acc(sum, (double)sv[C * k], xv[u]);
                        }
                    }
                }
            };
            // slices of exactly W entries (the 7-point stencil: W = 7, 6 on a
            // boundary plane): fully unrolled, no per-entry predicates (T = 1)
            auto run_w = [&](auto wc, auto cs, int32_t cbase, auto vx) {
                constexpr int W = decltype(wc)::value;
                constexpr int CS = decltype(cs)::value;
                constexpr bool VX = decltype(vx)::value;
                int32_t c[W];
                acc_t<Op> xv[W];
#pragma unroll
                for (int u = 0; u < W; ++u) c[u] = sc[CS * u] + cbase;
#pragma unroll
                for (int u = 0; u < W; ++u) xv[u] = gather_chk(op, c[u], A.ncols);
#pragma unroll
                for (int u = 0; u < W; ++u) {
                    if constexpr (VX)
                        fma_acc(sum, vtab_s[si[C * u]], xv[u]);
                    else
                        fma_acc(sum, (double)sv[C * u], xv[u]);
                }
            };
            using one = std::integral_constant<int, 1>;
            using cc = std::integral_constant<int, C>;
            using w7 = std::integral_constant<int, 7>;
            using w6 = std::integral_constant<int, 6>;
            auto dispatch = [&](auto vx) {
                if constexpr (T == 1) {
                    if (w == 7) {
                        if (dict) run_w(w7{}, one{}, (int32_t)row, vx);
                        else run_w(w7{}, cc{}, 0, vx);
                        return;
                    }
                    if (w == 6) {
                        if (dict) run_w(w6{}, one{}, (int32_t)row, vx);
                        else run_w(w6{}, cc{}, 0, vx);
                        return;
                    }
                }
                if (dict)
                    run(one{}, (int32_t)row, vx);
                else
                    run(cc{}, 0, vx);
            };
            if (vix)
                dispatch(std::true_type{});
            else
                dispatch(std::false_type{});
            __syncwarp();
            if (lane == 0) mbar_arrive(bar_empty0 + 8 * s);  // stage free
            if constexpr (T > 1) {
#pragma unroll
                for (int o = C; o < 32; o <<= 1) add_acc(sum, shfl_xor_acc(0xffffffffu, sum, o));
            }
            if constexpr (cols_of<Op>() > 1)
                if (pt == 0 && has_row) rr = op.load(row);
            if (pt == 0 && has_row) op.row(row, sum, rr, dots);
        }
    }
    pdl_trigger();
    if constexpr (Op::NDOT > 0) grid_reduce<Op::NDOT>(dots, red, op.fin);
}

// ----------------------------------------------------------------- TMA-staged CSR kernel
// Padding-free alternative to the TMA-staged SELL-32 for matrices whose rows
// differ in length (smoothed-aggregation P and R, coarse A: SELL-32 pads every
// row of a 32-row slice to the slice's longest row, 26 % of P0's stored entries
// at 256^3).  A tile is 256 consecutive rows; its entries are the contiguous
// CSR range [ptr[r0], ptr[r0 + 256]), which the producer warp moves into a
// kTmaStages-deep shared-memory ring with three cp.async.bulk copies (values,
// columns, the tile's 257 row pointers; each source aligned down to 16 bytes,
// the arrays padded so the rounded-up tail stays in bounds).  Consumer warp w
// owns rows 32 w .. 32 w + 31 of the tile, one thread per row: its entries are
// read from shared memory in ascending column order (the CSR order of the
// paper's product), gathers issued UN at a time, then the fused epilogue.
constexpr int kTcRows = 256;  // rows per tile (8 consumer warps x 32)

struct CsrTma {
    int64_t nrows = 0, ncols = 0, ntiles = 0;
    int64_t row0 = 0;             // first row of this (sub-)matrix view (a multiple of 256)
    const int32_t* ptr = nullptr; // row pointers of the view's rows (absolute entry offsets, nnz < 2^31),
                                  // readable up to 8 past the last row
    const int32_t* col = nullptr; // padded by 4 entries
    const double* val = nullptr;  // padded by 2 entries
    const float* valf = nullptr;  // fp32 copy (mixed precision), padded by 4
    int32_t tile_ent = 0;         // stage capacity in entries (max over tiles, incl. alignment slack)
    int32_t smem_stage = 0;       // bytes of one stage
    const double* vtab = nullptr; // value-indexed storage, the table staged in shared memory; val unused:
    const uint8_t* vi8 = nullptr; // 1-byte indices (<= 256 distinct values), padded by 16
    const uint16_t* vi16 = nullptr; // or 2-byte indices (<= ntab distinct values), padded by 16
    int32_t ntab = 0;             // table entries (256 with vi8)
    int32_t vtab_bytes = 0;       // shared-memory bytes of the table (set at launch; 128-B multiple)
};

// UN1: entries per unrolled step for one right-hand side (P rows hold 1-6
// entries: 4 wastes fewer predicated slots than 8; AMGB_TCSR_UN=8 for the other)
template <bool STREAM, class Op, bool F32 = false, int UN1 = 4>
__global__ void __launch_bounds__(kTmaThreads, minb_of<Op>(2)) csr_tma(CsrTma A, Op op, const int32_t* gate,
                                                                         Red red) {
    using VT = std::conditional_t<F32, float, double>;
    constexpr int VB = (int)sizeof(VT);
    constexpr int VA = 16 / VB;  // value alignment unit (entries)
    constexpr int UN = cols_of<Op>() == 1 ? UN1 : unroll_of<Op>(8);
    pdl_wait();
    if (gated(gate)) return;
    op.prepare();
    extern __shared__ __align__(128) unsigned char smem_raw[];
    // layout: [value table] stages { val[tile_ent] (VB bytes, or 1- / 2-byte indices) | col[tile_ent] |
    // ptr[kTcRows + 8] }; barriers after the stages
    const int vm = F32 ? 0 : A.vi8 ? 1 : A.vi16 ? 2 : 0;  // value mode: array / 8-bit / 16-bit index
    const bool vix = vm != 0;
    double* vtab_s = reinterpret_cast<double*>(smem_raw);
    unsigned char* smem = smem_raw + (vix ? A.vtab_bytes : 0);
    const int vbytes = vm == 1 ? 1 : vm == 2 ? 2 : VB;
    const int te = A.tile_ent;
    const size_t sb = (size_t)A.smem_stage;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kTmaStages * sb);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (vix)
        for (int k = threadIdx.x; k < A.ntab; k += blockDim.x) vtab_s[k] = __ldg(A.vtab + k);
    if (threadIdx.x == 0) {
        for (int s = 0; s < kTmaStages; ++s) {
            mbar_init(smem_u32(bars + s), 1);
            mbar_init(smem_u32(bars + kTmaStages + s), kBlock / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    constexpr int ND = Op::NDOT > 0 ? Op::NDOT : 1;
    double dots[ND];
#pragma unroll
    for (int k = 0; k < ND; ++k) dots[k] = 0.0;

    if (warp == kBlock / 32) {  // ---------------- producer warp
        if (lane == 0) {
            uint64_t policy = 0;
            if constexpr (STREAM) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
            int i = 0;
            for (int64_t t = blockIdx.x; t < A.ntiles; t += gridDim.x, ++i) {
                const int s = i % kTmaStages;
                if (i >= kTmaStages) mbar_wait(smem_u32(bars + kTmaStages + s), ((i / kTmaStages) & 1) ^ 1);
                const int64_t r0 = t * kTcRows;
                const int64_t r1 = r0 + kTcRows < A.nrows ? r0 + kTcRows : A.nrows;
                const int32_t e0 = A.ptr[r0], e1 = A.ptr[r1];
                const int32_t vau = vm == 1 ? 16 : vm == 2 ? 8 : VA;  // value alignment unit (entries)
                const int32_t va = e0 & ~(vau - 1), ca = e0 & ~3;
                const uint32_t nv = (uint32_t)(((e1 - va) + vau - 1) & ~(vau - 1));
                const uint32_t nc = (uint32_t)(((e1 - ca) + 3) & ~3);
                const uint32_t np = (uint32_t)(((r1 - r0 + 1) + 3) & ~3);
                AMGB_ASSERT(e1 >= e0 && nv <= (uint32_t)te && nc <= (uint32_t)te);
                const uint32_t full = smem_u32(bars + s);
                unsigned char* st = smem + (size_t)s * sb;
                mbar_expect_tx(full, nv * (uint32_t)vbytes + nc * 4u + np * 4u);
                if (nv) {
                    if (vm == 1)
                        bulk_g2s<STREAM>(smem_u32(st), A.vi8 + va, nv, full, policy);
                    else if (vm == 2)
                        bulk_g2s<STREAM>(smem_u32(st), A.vi16 + va, nv * 2u, full, policy);
                    else if constexpr (F32)
                        bulk_g2s<STREAM>(smem_u32(st), A.valf + va, nv * 4u, full, policy);
                    else
                        bulk_g2s<STREAM>(smem_u32(st), A.val + va, nv * 8u, full, policy);
                }
                if (nc) bulk_g2s<STREAM>(smem_u32(st + (size_t)te * vbytes), A.col + ca, nc * 4u, full, policy);
                bulk_g2s<STREAM>(smem_u32(st + (size_t)te * (vbytes + 4)), A.ptr + r0, np * 4u, full, policy);
            }
        }
    } else {  // ------------------------------------ consumer warps
        int i = 0;
        for (int64_t t = blockIdx.x; t < A.ntiles; t += gridDim.x, ++i) {
            const int s = i % kTmaStages;
            const int64_t lrow = t * kTcRows + warp * 32 + lane;
            const bool has_row = lrow < A.nrows;
            const int64_t row = A.row0 + lrow;
            typename Op::Row rr{};
            if constexpr (cols_of<Op>() == 1)
                if (has_row) rr = op.load(row);  // in flight during the wait
            mbar_wait(smem_u32(bars + s), (i / kTmaStages) & 1);
            const unsigned char* st = smem + (size_t)s * sb;
            const int32_t* sp = reinterpret_cast<const int32_t*>(st + (size_t)te * (vbytes + 4));
            const int32_t e0 = sp[0];
            const VT* sv = reinterpret_cast<const VT*>(st) - (e0 & ~(VA - 1));
            const uint8_t* si = st - (e0 & ~15);
            const uint16_t* si16 = reinterpret_cast<const uint16_t*>(st) - (e0 & ~7);
            const int32_t* sc = reinterpret_cast<const int32_t*>(st + (size_t)te * vbytes) - (e0 & ~3);
            acc_t<Op> sum{};
            auto run = [&](auto vx) {
                constexpr int VX = decltype(vx)::value;
                const int32_t pb = sp[warp * 32 + lane], pe = sp[warp * 32 + lane + 1];
                for (int32_t k0 = pb; k0 < pe; k0 += UN) {
                    acc_t<Op> xv[UN];
                    int32_t c[UN];
#pragma unroll
                    for (int u = 0; u < UN; ++u) c[u] = k0 + u < pe ? sc[k0 + u] : 0;
#pragma unroll
                    for (int u = 0; u < UN; ++u) xv[u] = (k0 + u < pe) ? gather_chk(op, c[u], A.ncols) : acc_t<Op>{};
#pragma unroll
                    for (int u = 0; u < UN; ++u) {
                        if constexpr (VX == 1) {
                            if (k0 + u < pe) fma_acc(sum, vtab_s[si[k0 + u]], xv[u]);
                        } else if constexpr (VX == 2) {
                            if (k0 + u < pe) fma_acc(sum, vtab_s[si16[k0 + u]], xv[u]);
                        } else {
                            if (k0 + u < pe) fma_acc(sum, (double)sv[k0 + u], xv[u]);
                        }
                    }
                }
            };
            if (has_row) {
                if (vm == 1)
                    run(std::integral_constant<int, 1>{});
                else if (vm == 2)
                    run(std::integral_constant<int, 2>{});
                else
                    run(std::integral_constant<int, 0>{});
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(bars + kTmaStages + s));  // stage free
            if constexpr (cols_of<Op>() > 1)
                if (has_row) rr = op.load(row);
            if (has_row) op.row(row, sum, rr, dots);
        }
    }
    pdl_trigger();
    if constexpr (Op::NDOT > 0) grid_reduce<Op::NDOT>(dots, red, op.fin);
}

// ----------------------------------------------------------------- row-block CSR kernel
// Padding-free alternative to SELL for any row-length mix ("CSR-stream").  The
// rows are cut on the host into blocks of at most kEnt entries (and kRowsMax
// rows).  Per block: (1) the block's contiguous [ptr[rb], ptr[re]) slice of col /
// val is read with fully coalesced loads, kEnt/kBlock entries per thread, all
// issued before their gathers, and the products a_ij * x_j go to shared memory;
// (2) G threads per row sum the row's products (G = 1: one thread, ascending
// order -- the same arithmetic as a plain CSR row loop) and run the epilogue.
// A row longer than kEnt gets a block of its own and is reduced block-wide.
// Persistent grid (grid-stride over row blocks) so fused dot products reduce
// over a bounded number of partials.
constexpr int kEnt = 2048;
constexpr int kRowsMax = 512;

struct CsrDev {
    int64_t nrows = 0, ncols = 0, nnz = 0, nblocks = 0;
    const int32_t* ptr = nullptr;   // nrows + 1 (nnz < 2^31 per level)
    const int32_t* col = nullptr;
    const double* val = nullptr;
    const float* valf = nullptr;    // fp32 copy of val (mixed-precision V-cycle)
    const int32_t* brow = nullptr;  // nblocks + 1 first rows of the row blocks
    int32_t G = 1;                  // threads per row in the summation phase
};

template <int G, bool STREAM, class Op, bool F32 = false>
__global__ void __launch_bounds__(kBlock) csr_rows(CsrDev A, Op op, const int32_t* gate, Red red) {
    pdl_wait();
    if (gated(gate)) return;
    op.prepare();
    __shared__ double prod[kEnt];
    constexpr int ND = Op::NDOT > 0 ? Op::NDOT : 1;
    double dots[ND];
#pragma unroll
    for (int k = 0; k < ND; ++k) dots[k] = 0.0;
    const int tid = threadIdx.x;
    const int lig = tid & (G - 1);
    const unsigned gmask = G == 32 ? 0xffffffffu : (((1u << G) - 1u) << ((tid & 31) & ~(G - 1)));
    if constexpr (!std::is_same_v<acc_t<Op>, double>) {
        // batched right-hand sides: G threads per row straight from global
        // memory (the shared-memory product tile would be K times larger)
        const int64_t groups = ((int64_t)gridDim.x * blockDim.x) / G;
        for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + tid) / G; r < A.nrows; r += groups) {
            acc_t<Op> s{};
            for (int k = A.ptr[r] + lig; k < A.ptr[r + 1]; k += G)
                fma_acc(s, ld_val<STREAM, F32>(A, k), gather_chk(op, ld_mat<STREAM>(A.col + k), A.ncols));
            if constexpr (G > 1) {
#pragma unroll
                for (int o = G / 2; o > 0; o >>= 1) add_acc(s, shfl_xor_acc(gmask, s, o));
            }
            if (lig == 0) op.row(r, s, op.load(r), dots);
        }
        pdl_trigger();
        if constexpr (Op::NDOT > 0) grid_reduce<Op::NDOT>(dots, red, op.fin);
        return;
    } else {
    for (int64_t b = blockIdx.x; b < A.nblocks; b += gridDim.x) {
        const int rb = A.brow[b], re = A.brow[b + 1];
        const int eb = A.ptr[rb], ne = A.ptr[re] - eb;
        if (ne <= kEnt) {
            constexpr int PER = kEnt / kBlock;
            int32_t c[PER];
            double v[PER];
#pragma unroll
            for (int k = 0; k < PER; ++k) {
                const int e = tid + k * kBlock;
                if (e < ne) {
                    c[k] = ld_mat<STREAM>(A.col + eb + e);
                    v[k] = ld_val<STREAM, F32>(A, eb + e);
                }
            }
#pragma unroll
            for (int k = 0; k < PER; ++k) {
                const int e = tid + k * kBlock;
                if (e < ne) prod[e] = v[k] * gather_chk(op, c[k], A.ncols);
            }
            __syncthreads();
            for (int r = rb + tid / G; r < re; r += kBlock / G) {
                const typename Op::Row rr = op.load(r);
                const int s0 = A.ptr[r] - eb, s1 = A.ptr[r + 1] - eb;
                double s = 0.0;
                for (int k = s0 + lig; k < s1; k += G) s += prod[k];
                if constexpr (G > 1) {
#pragma unroll
                    for (int o = G / 2; o > 0; o >>= 1) s += __shfl_xor_sync(gmask, s, o);
                }
                if (lig == 0) op.row(r, s, rr, dots);
            }
            __syncthreads();
        } else {  // one long row
            double s = 0.0;
            for (int e = tid; e < ne; e += kBlock)
                s += ld_val<STREAM, F32>(A, eb + e) * gather_chk(op, ld_mat<STREAM>(A.col + eb + e), A.ncols);
            s = warp_sum(s);
            if ((tid & 31) == 0) prod[tid >> 5] = s;
            __syncthreads();
            if (tid == 0) {
                double t = 0.0;
                for (int w = 0; w < kBlock / 32; ++w) t += prod[w];
                op.row(rb, t, op.load(rb), dots);
            }
            __syncthreads();
        }
    }
    }  // single right-hand side
    pdl_trigger();
    if constexpr (Op::NDOT > 0) grid_reduce<Op::NDOT>(dots, red, op.fin);
}

// ----------------------------------------------------------------- vector kernel
template <class Op, class = void>
struct op_pairs : std::false_type {};
template <class Op>
struct op_pairs<Op, std::void_t<decltype(&Op::elem2)>> : std::true_type {};

template <class Op>
__global__ void __launch_bounds__(kBlock) vec_kernel(int64_t n, Op op, const int32_t* gate, Red red) {
    pdl_wait();
    if (gated(gate)) return;
    op.prepare();
    double dots[Op::NDOT > 0 ? Op::NDOT : 1];
#pragma unroll
    for (int k = 0; k < (Op::NDOT > 0 ? Op::NDOT : 1); ++k) dots[k] = 0.0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if constexpr (op_pairs<Op>::value) {
        // Ops with elem2: two consecutive elements per thread with 16-B loads and
        // stores (half the memory instructions per byte), when every vector is
        // 16-B aligned; the odd tail element goes through elem.
        if (op.aligned16()) {
            for (int64_t j = tid; j < (n >> 1); j += stride) op.elem2(j, dots);
            if ((n & 1) && tid == 0) op.elem(n - 1, dots);
        } else {
            for (int64_t i = tid; i < n; i += stride) op.elem(i, dots);
        }
    } else {
        for (int64_t i = tid; i < n; i += stride) op.elem(i, dots);
    }
    pdl_trigger();
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
    const double* x;
    double* y;
    NoFin fin;
    struct Row {};
    __device__ void prepare() {}
    __device__ Row load(int64_t) const { return {}; }
    __device__ double gather(int32_t c) const { return __ldg(x + c); }
    __device__ void row(int64_t i, double s, const Row&, double*) const { y[i] = s; }
};

// y = f - A x  [+ (y, y)]
template <int ND, class Fin>
struct OpResidual {
    static constexpr int GATHER = 1, ROWV = 2;  // vectors gathered / row-indexed (bytes model)
    static constexpr int NDOT = ND;
    const double* x;
    const double* f;
    double* y;
    Fin fin;
    struct Row {
        double f;
    };
    __device__ void prepare() {}
    __device__ Row load(int64_t i) const { return {f[i]}; }
    __device__ double gather(int32_t c) const { return __ldg(x + c); }
    __device__ void row(int64_t i, double s, const Row& rr, double* d) const {
        double r = rr.f - s;
        y[i] = r;
        if constexpr (ND > 0) d[0] += r * r;
    }
};

// Restriction that also emits the next level's m o f (a2 feeding a1): y = R t,
// mf = m_c o y -- so the next level's zero-start residual gathers one vector.
struct OpSpmvMF {
    static constexpr int GATHER = 1, ROWV = 3;  // t gathered; y, mf written, m_c read
    static constexpr int NDOT = 0;
    const double* x;
    double* y;
    const double* mc;
    double* mf;
    NoFin fin;
    struct Row {
        double m;
    };
    __device__ void prepare() {}
    __device__ Row load(int64_t i) const { return {mc[i]}; }
    __device__ double gather(int32_t c) const { return __ldg(x + c); }
    __device__ void row(int64_t i, double s, const Row& rr, double*) const {
        y[i] = s;
        mf[i] = rr.m * s;
    }
};

// Zero-start residual with a precomputed mf = m o f: t = f - A mf.
struct OpRes0MF {
    static constexpr int GATHER = 1, ROWV = 2;  // mf gathered; f read, t written
    static constexpr int NDOT = 0;
    const double* mf;
    const double* f;
    double* t;
    NoFin fin;
    struct Row {
        double f;
    };
    __device__ void prepare() {}
    __device__ Row load(int64_t i) const { return {f[i]}; }
    __device__ double gather(int32_t c) const { return __ldg(mf + c); }
    __device__ void row(int64_t i, double s, const Row& rr, double*) const { t[i] = rr.f - s; }
};

// Prolongation after a zero-start sweep with a precomputed mf: x = mf + P e.
struct OpProl0MF {
    static constexpr int GATHER = 1, ROWV = 2;  // e gathered; mf read, x written
    static constexpr int NDOT = 0;
    const double* e;
    const double* mf;
    double* x;
    NoFin fin;
    struct Row {
        double mf;
    };
    __device__ void prepare() {}
    __device__ Row load(int64_t i) const { return {mf[i]}; }
    __device__ double gather(int32_t c) const { return __ldg(e + c); }
    __device__ void row(int64_t i, double s, const Row& rr, double*) const { x[i] = rr.mf + s; }
};

// Zero-start smoother + residual (a1): with x = m o f (the first SPAI-0/Jacobi
// sweep from x = 0), t = f - A x, computing x_j = m_j f_j inside the gather.
struct OpRes0 {
    static constexpr int GATHER = 2, ROWV = 1;  // vectors gathered / row-indexed (bytes model)
    static constexpr int NDOT = 0;
    const double* m;
    const double* f;
    double* t;
    NoFin fin;
    struct Row {
        double f;
    };
    __device__ void prepare() {}
    __device__ Row load(int64_t i) const { return {f[i]}; }
    __device__ double gather(int32_t c) const { return __ldg(m + c) * __ldg(f + c); }
    __device__ void row(int64_t i, double s, const Row& rr, double*) const { t[i] = rr.f - s; }
};

// Damped-Jacobi / SPAI-0 sweep (a6): xo = x + m o (f - A x), optional (f, xo).
template <int ND, class Fin>
struct OpRelax {
    static constexpr int GATHER = 1, ROWV = 3;  // vectors gathered / row-indexed (bytes model)
    static constexpr int NDOT = ND;
    const double* x;
    const double* m;
    const double* f;
    double* xo;
    Fin fin;
    struct Row {
        double x, m, f;
    };
    __device__ void prepare() {}
    __device__ Row load(int64_t i) const { return {x[i], m[i], f[i]}; }
    __device__ double gather(int32_t c) const { return __ldg(x + c); }
    __device__ void row(int64_t i, double s, const Row& rr, double* d) const {
        const double fi = rr.f;
        const double xn = rr.x + rr.m * (fi - s);
        xo[i] = xn;
        if constexpr (ND > 0) d[0] += fi * xn;
    }
};

// Prolongation-correction after a zero-start sweep (a5): x = m o f + P e.
struct OpProl0 {
    static constexpr int GATHER = 1, ROWV = 3;  // vectors gathered / row-indexed (bytes model)
    static constexpr int NDOT = 0;
    const double* e;
    const double* m;
    const double* f;
    double* x;
    NoFin fin;
    struct Row {
        double m, f;
    };
    __device__ void prepare() {}
    __device__ Row load(int64_t i) const { return {m[i], f[i]}; }
    __device__ double gather(int32_t c) const { return __ldg(e + c); }
    __device__ void row(int64_t i, double s, const Row& rr, double*) const { x[i] = rr.m * rr.f + s; }
};

// General prolongation-correction: x = x + P e (x updated in place, row-local).
struct OpProlAdd {
    static constexpr int GATHER = 1, ROWV = 2;  // vectors gathered / row-indexed (bytes model)
    static constexpr int NDOT = 0;
    const double* e;
    double* x;
    NoFin fin;
    struct Row {
        double x;
    };
    __device__ void prepare() {}
    __device__ Row load(int64_t i) const { return {x[i]}; }
    __device__ double gather(int32_t c) const { return __ldg(e + c); }
    __device__ void row(int64_t i, double s, const Row& rr, double*) const { x[i] = rr.x + s; }
};

// One Chebyshev step (§8c c-1): r = f - A x; scaled: r = r / a_ii (a_ii read from
// the row itself); p = alpha r + beta p (first step: p = alpha r); xo = x + p.
template <int ND, class Fin>
struct OpCheb {
    static constexpr int GATHER = 1, ROWV = 5;  // vectors gathered / row-indexed (bytes model)
    static constexpr int NDOT = ND;
    const double* x;
    const double* f;
    const double* diag;
    double* p;
    double* xo;
    double alpha, beta;
    int32_t scaled, first;
    Fin fin;
    struct Row {
        double f, dg, p, x;
    };
    __device__ void prepare() {}
    __device__ Row load(int64_t i) const { return {f[i], diag[i], first ? 0.0 : p[i], x[i]}; }
    __device__ double gather(int32_t c) const { return __ldg(x + c); }
    __device__ void row(int64_t i, double s, const Row& rr, double* d) const {
        double r = rr.f - s;
        if (scaled) r = r / rr.dg;
        const double pn = first ? alpha * r : alpha * r + beta * rr.p;
        p[i] = pn;
        const double xn = rr.x + pn;
        xo[i] = xn;
        if constexpr (ND > 0) d[0] += rr.f * xn;
    }
};

// CG direction + SpMV (a7): p' = z + beta p (formed inside the gather), q = A p',
// sigma = (p', q).
template <class Fin>
struct OpCgDir {
    static constexpr int GATHER = 2, ROWV = 2;  // vectors gathered / row-indexed (bytes model)
    static constexpr int NDOT = 1;
    const double* z;
    const double* p;
    double* pn;
    double* q;
    const KState* ks;
    double beta;
    Fin fin;
    struct Row {
        double z, p;
    };
    __device__ void prepare() { beta = ks->beta; }
    __device__ Row load(int64_t i) const { return {z[i], p[i]}; }
    __device__ double gather(int32_t c) const { return fma(beta, __ldg(p + c), __ldg(z + c)); }
    __device__ void row(int64_t i, double s, const Row& rr, double* d) const {
        const double pi = fma(beta, rr.p, rr.z);
        pn[i] = pi;
        q[i] = s;
        d[0] += pi * s;
    }
};

// Fused CG (single part, SPAI-0/Jacobi, npre = 1): the first level-0 kernel
// of iteration k also applies iteration k-1's r -= alpha q (formed inside the
// gather -- bitwise the same fma as the separate update -- and stored once to a
// ping-pong r buffer) and computes (r, r) for the loop test:
//   rn = r - alpha q;  t = rn - A (m o rn);  (rn, rn)
template <class Fin>
struct OpRes0Upd {
    static constexpr int GATHER = 3, ROWV = 2;  // m, r, q gathered; rn, t written
    static constexpr int NDOT = 1;
    const double* m;
    const double* r;
    const double* q;
    double* rn;
    double* t;
    const KState* ks;
    double alpha;
    Fin fin;
    struct Row {
        double r, q;
    };
    __device__ void prepare() { alpha = ks->upd ? ks->alpha : 0.0; }
    __device__ Row load(int64_t i) const { return {r[i], q[i]}; }
    __device__ double gather(int32_t c) const { return __ldg(m + c) * fma(-alpha, __ldg(q + c), __ldg(r + c)); }
    __device__ void row(int64_t i, double s, const Row& rr, double* d) const {
        const double v = fma(-alpha, rr.q, rr.r);
        rn[i] = v;
        t[i] = v - s;
        d[0] += v * v;
    }
};

// Fused CG direction: OpCgDir plus iteration k-1's x += alpha p (p = the old
// direction this kernel reads anyway).
template <class Fin>
struct OpCgDirX {
    static constexpr int GATHER = 2, ROWV = 4;  // z, p gathered; pn, q written; x read + written
    static constexpr int NDOT = 1;
    const double* z;
    const double* p;
    double* pn;
    double* q;
    double* x;
    const KState* ks;
    double beta, xa;
    Fin fin;
    struct Row {
        double z, p;
    };
    __device__ void prepare() {
        beta = ks->beta;
        xa = ks->xpend ? ks->alpha : 0.0;
    }
    __device__ Row load(int64_t i) const { return {z[i], p[i]}; }
    __device__ double gather(int32_t c) const { return fma(beta, __ldg(p + c), __ldg(z + c)); }
    __device__ void row(int64_t i, double s, const Row& rr, double* d) const {
        const double pi = fma(beta, rr.p, rr.z);
        pn[i] = pi;
        q[i] = s;
        d[0] += pi * s;
        if (xa != 0.0) x[i] = fma(xa, rr.p, x[i]);
    }
};

// y = A x with dots: ND = 1: (w, y); ND = 2: (y, y), (y, w).
template <int ND, class Fin>
struct OpSpmvDot {
    static constexpr int GATHER = 1, ROWV = 2;  // vectors gathered / row-indexed (bytes model)
    static constexpr int NDOT = ND;
    const double* x;
    const double* w;
    double* y;
    Fin fin;
    struct Row {
        double w;
    };
    __device__ void prepare() {}
    __device__ Row load(int64_t i) const { return {w[i]}; }
    __device__ double gather(int32_t c) const { return __ldg(x + c); }
    __device__ void row(int64_t i, double s, const Row& rr, double* d) const {
        y[i] = s;
        if constexpr (ND == 1) {
            d[0] += rr.w * s;
        } else {
            d[0] += s * s;
            d[1] += s * rr.w;
        }
    }
};

}  // namespace amgb
