// amgb.cu -- device hierarchy store, V-cycle executor, CG / BiCGStab drivers and
// the C ABI (include/amgb.h).
//
// Solve phase of arXiv 1811.05704 (AMGCL): Algorithm 2 as the
// preconditioner of CG / BiCGStab.  The
// hierarchy comes from setup.cpp (Algorithm 1, on the host)
// and is uploaded once into sliced-ELL device matrices (kernels.cuh).  Every
// step of the solve runs in this file's kernels; the host only sequences
// launches and reads one small state struct per pair of Krylov iterations.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/amgb.h"
#include "kernels.cuh"
#include "setup.hpp"

namespace amgb {

// ============================================================ device code

__global__ void __launch_bounds__(kBlock) dense_gemv(int64_t n, const double* __restrict__ M,
                                                     const double* __restrict__ x, double* __restrict__ y,
                                                     const int32_t* gate) {
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
};

// ============================================================ host side

namespace {

thread_local std::string g_err;

struct CudaError {
    std::string msg;
};

inline void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw CudaError{std::string(what) + ": " + cudaGetErrorString(e)};
}

struct HostSell {
    int64_t nrows = 0, ncols = 0, nslices = 0;
    std::vector<int64_t> sptr;
    std::vector<int32_t> col;
    std::vector<double> val;
};

// CSR -> SELL-C, slice height C (see kernels.cuh): entry k of row s*C + r at
// sptr[s] + k*C + r.
HostSell to_sell(const Csr& A, int C = 32) {
    HostSell S;
    S.nrows = A.nrows;
    S.ncols = A.ncols;
    S.nslices = (A.nrows + C - 1) / C;
    S.sptr.assign(S.nslices + 1, 0);
    for (int64_t s = 0; s < S.nslices; ++s) {
        int64_t w = 0;
        for (int64_t r = s * C; r < std::min<int64_t>(A.nrows, s * C + C); ++r)
            w = std::max<int64_t>(w, A.ptr[r + 1] - A.ptr[r]);
        S.sptr[s + 1] = S.sptr[s] + C * w;
    }
    S.col.assign(S.sptr[S.nslices], 0);
    S.val.assign(S.sptr[S.nslices], 0.0);
#pragma omp parallel for schedule(static)
    for (int64_t s = 0; s < S.nslices; ++s) {
        const int64_t w = (S.sptr[s + 1] - S.sptr[s]) / C;
        for (int lane = 0; lane < C; ++lane) {
            const int64_t r = s * C + lane;
            int64_t len = 0;
            int32_t last = 0;
            if (r < A.nrows) {
                len = A.ptr[r + 1] - A.ptr[r];
                for (int64_t k = 0; k < len; ++k) {
                    S.col[S.sptr[s] + C * k + lane] = A.col[A.ptr[r] + k];
                    S.val[S.sptr[s] + C * k + lane] = A.val[A.ptr[r] + k];
                }
                if (len > 0) last = A.col[A.ptr[r] + len - 1];
            }
            for (int64_t k = len; k < w; ++k) {
                S.col[S.sptr[s] + C * k + lane] = last;
                S.val[S.sptr[s] + C * k + lane] = 0.0;
            }
        }
    }
    return S;
}

// A device matrix in the format chosen for it.
enum class Fmt { CSR, SELL, TMA };

struct DMat {
    Fmt fmt = Fmt::CSR;
    bool is_csr = true;
    Sell sell;
    SellTma tma;
    int64_t sell_wmax = 0;  // widest slice
    CsrDev csr;
    int64_t nrows = 0, ncols = 0, nnz = 0, stored = 0;
};

struct DevLevel {
    int64_t n = 0, nc = 0;
    int64_t nnzA = 0, nnzP = 0, padA = 0;
    DMat A, P, R;
    double* m = nullptr;     // SPAI-0 / Jacobi diagonal
    double* diag = nullptr;  // a_ii (Chebyshev)
    double* f = nullptr;     // right-hand side (levels >= 1)
    double* x = nullptr;     // work
    double* y = nullptr;     // work (ping-pong)
    double* t = nullptr;     // residual
    double* p = nullptr;     // Chebyshev direction
    double* o = nullptr;     // V-cycle output (levels >= 1)
    std::vector<double> cheb_alpha, cheb_beta;
    double alg_bytes = 0;
    int64_t dev_bytes = 0;
};

}  // namespace

struct Handle {
    amg_params prm{};
    HostHierarchy host;
    bool on_device = false;
    int device = 0;
    int num_sms = 148;
    cudaStream_t stream = nullptr;      // work stream (own_stream unless set by the caller)
    cudaStream_t own_stream = nullptr;  // blocking stream: ordered with the legacy default stream
    std::vector<DevLevel> lv;
    double* coarse_inv = nullptr;
    int64_t nL = 0;
    KState* ks = nullptr;
    KState* ks_host = nullptr;  // pinned
    Red red;
    int32_t* zero_gate = nullptr;
    // Krylov vectors (level-0 length)
    double *r = nullptr, *z = nullptr, *pa = nullptr, *pb = nullptr, *q = nullptr;
    double *rhat = nullptr, *v = nullptr, *s = nullptr, *sh = nullptr, *ph = nullptr, *tv = nullptr;
    double *hf = nullptr, *hx = nullptr;  // device copies for amg_solve_host
    std::vector<void*> allocs;
    // CUDA graph of two Krylov iterations, keyed by the x pointer
    cudaGraphExec_t graph = nullptr;
    const double* graph_x = nullptr;
    int graph_prof_mask = 0;
    int64_t graph_kernels = 0;
    // accounting
    int64_t launches = 0;
    bool count_only = false;  // while capturing: count kernels into graph_kernels
    amg_solve_stats stats{};
    bool sync_debug = false;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;

    double* dalloc(int64_t n) {
        void* p = nullptr;
        ck(cudaMalloc(&p, std::max<int64_t>(n, 1) * sizeof(double)), "cudaMalloc");
        allocs.push_back(p);
        return static_cast<double*>(p);
    }
    template <class T>
    T* upload(const std::vector<T>& v) {
        void* p = nullptr;
        ck(cudaMalloc(&p, std::max<size_t>(v.size(), 1) * sizeof(T)), "cudaMalloc");
        allocs.push_back(p);
        if (!v.empty()) ck(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice), "upload");
        return static_cast<T*>(p);
    }
    ~Handle() {
        if (graph) cudaGraphExecDestroy(graph);
        for (cudaEvent_t e : ev_all) cudaEventDestroy(e);
        for (void* p : allocs) cudaFree(p);
        if (ks_host) cudaFreeHost(ks_host);
        if (ev0) cudaEventDestroy(ev0);
        if (ev1) cudaEventDestroy(ev1);
        if (own_stream) cudaStreamDestroy(own_stream);
    }

    int grid_for(int64_t n) const {
        const int64_t b = (n + kBlock - 1) / kBlock;
        return (int)std::max<int64_t>(1, std::min<int64_t>(b, (int64_t)num_sms * 8));
    }

    // ------------------------------------------------------------ accounting
    // Every launch carries a kernel class (AMG_PROF_*), its algorithmic bytes
    // and the Krylov iteration (0/1 inside a two-iteration
    // group, -1 outside) it belongs to.  Bytes of iterations that actually ran
    // are summed into the solve statistics; in profile mode the classes in
    // prof_mask are bracketed with CUDA events (event-record nodes when the
    // launches are being captured into the iteration graph).
    struct Rec {
        cudaEvent_t a = nullptr, b = nullptr;
        int cls = 0, iter = -1;
        double bytes = 0;
    };
    int prof_mask = 0;
    bool capturing = false;
    int cur_iter = -1;
    std::vector<Rec> rec_direct, rec_graph;  // launches since the last sync / in the graph
    std::vector<cudaEvent_t> ev_pool, ev_all;
    double acc_ms[8] = {}, acc_bytes[8] = {}, alg_bytes = 0;
    int64_t acc_launches[8] = {};

    cudaEvent_t get_event() {
        if (ev_pool.empty()) {
            cudaEvent_t e;
            ck(cudaEventCreate(&e), "cudaEventCreate");
            ev_all.push_back(e);
            return e;
        }
        cudaEvent_t e = ev_pool.back();
        ev_pool.pop_back();
        return e;
    }
    void record(cudaEvent_t e) {
        if (capturing)
            ck(cudaEventRecordWithFlags(e, stream, cudaEventRecordExternal), "event record node");
        else
            ck(cudaEventRecord(e, stream), "cudaEventRecord");
    }
    template <class F>
    void launch(int cls, double bytes, const char* what, F&& fn) {
        Rec rc;
        rc.cls = cls;
        rc.iter = cur_iter;
        rc.bytes = bytes;
        const bool timed = (prof_mask >> cls) & 1;
        if (timed) {
            rc.a = get_event();
            rc.b = get_event();
            record(rc.a);
        }
        fn();
        if (timed) record(rc.b);
        (capturing ? rec_graph : rec_direct).push_back(rc);
        ++launches;
        if (sync_debug) {
            ck(cudaGetLastError(), what);
            ck(cudaStreamSynchronize(stream), what);
        }
    }
    // After a stream sync: account launches of iterations < ran (and all
    // launches outside iterations); recycle direct-launch events.
    void collect(std::vector<Rec>& v, int ran, bool recycle) {
        for (Rec& rc : v) {
            if (rc.iter >= 0 && rc.iter >= ran) continue;
            alg_bytes += rc.bytes;
            if (rc.a) {
                float ms = 0.f;
                ck(cudaEventElapsedTime(&ms, rc.a, rc.b), "cudaEventElapsedTime");
                acc_ms[rc.cls] += ms;
                acc_bytes[rc.cls] += rc.bytes;
                acc_launches[rc.cls] += 1;
            }
        }
        if (recycle) {
            for (Rec& rc : v)
                if (rc.a) {
                    ev_pool.push_back(rc.a);
                    ev_pool.push_back(rc.b);
                }
            v.clear();
        }
    }
    void drop_graph() {
        if (graph) cudaGraphExecDestroy(graph);
        graph = nullptr;
        for (Rec& rc : rec_graph)
            if (rc.a) {
                ev_pool.push_back(rc.a);
                ev_pool.push_back(rc.b);
            }
        rec_graph.clear();
    }

    // ---------------------------------------------------------------- launches
    int mat_class(const DMat& M) const {
        if (&M == &lv[0].A) return AMG_PROF_A0_PASS;
        for (const auto& L : lv)
            if (&M == &L.A) return AMG_PROF_A_COARSE;
        return AMG_PROF_TRANSFER;
    }
    template <int U, bool PIPE, class Op>
    void rows_sell(const Sell& M, const Op& op, const int32_t* gate, bool stream_loads) {
        const int g = (int)std::max<int64_t>(
            1, std::min<int64_t>((M.nrows + kBlock - 1) / kBlock, (int64_t)num_sms * (PIPE ? 4 : 6)));
        if (stream_loads)
            sell_rows<U, true, PIPE, Op><<<g, kBlock, 0, stream>>>(M, op, gate, red);
        else
            sell_rows<U, false, PIPE, Op><<<g, kBlock, 0, stream>>>(M, op, gate, red);
    }
    template <int G, class Op>
    void rows_csr(const CsrDev& M, const Op& op, const int32_t* gate, bool stream_loads) {
        const int g = (int)std::max<int64_t>(1, std::min<int64_t>(M.nblocks, (int64_t)num_sms * 8));
        if (stream_loads)
            csr_rows<G, true, Op><<<g, kBlock, 0, stream>>>(M, op, gate, red);
        else
            csr_rows<G, false, Op><<<g, kBlock, 0, stream>>>(M, op, gate, red);
    }
    template <int T, bool STREAM, class Op>
    void rows_tma_impl(const SellTma& M, const Op& op, const int32_t* gate) {
        auto kern = sell_tma<T, STREAM, Op>;
        const size_t smem = (size_t)kTmaStages * M.tile_ent * 12 + 2 * kTmaStages * 8;
        static size_t configured = 0;  // per instantiation
        if (smem > configured) {
            ck(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "smem attr");
            configured = smem;
        }
        const int g = (int)std::max<int64_t>(1, std::min<int64_t>(M.ntiles, (int64_t)num_sms * kTmaBlocksPerSM));
        kern<<<g, kTmaThreads, smem, stream>>>(M, op, gate, red);
    }
    template <int T, class Op>
    void rows_tma(const SellTma& M, const Op& op, const int32_t* gate, bool stream_loads) {
        if (stream_loads)
            rows_tma_impl<T, true>(M, op, gate);
        else
            rows_tma_impl<T, false>(M, op, gate);
    }
    template <class Op>
    void rows_auto(const DMat& M, const Op& op, const int32_t* gate, const char* what) {
        // matrices too big for L2 stream their entries (evict-first); the rest
        // keep them cached so coarse levels stay L2-resident across cycles
        const bool big = M.nnz * 12 > (int64_t)48 << 20;
        const double bytes = 12.0 * M.nnz + 4.0 * M.nrows + 8.0 * M.ncols * Op::GATHER + 8.0 * M.nrows * Op::ROWV;
        launch(mat_class(M), bytes, what, [&] {
            if (M.fmt == Fmt::TMA) {
                switch (M.tma.T) {
                    case 1: rows_tma<1>(M.tma, op, gate, big); break;
                    case 2: rows_tma<2>(M.tma, op, gate, big); break;
                    case 4: rows_tma<4>(M.tma, op, gate, big); break;
                    default: rows_tma<8>(M.tma, op, gate, big); break;
                }
            } else if (M.is_csr) {
                switch (M.csr.G) {
                    case 1: rows_csr<1>(M.csr, op, gate, big); break;
                    case 2: rows_csr<2>(M.csr, op, gate, big); break;
                    case 4: rows_csr<4>(M.csr, op, gate, big); break;
                    case 8: rows_csr<8>(M.csr, op, gate, big); break;
                    default: rows_csr<16>(M.csr, op, gate, big); break;
                }
            } else if (M.sell_wmax <= 8) {
                rows_sell<8, false>(M.sell, op, gate, big);
            } else {
                rows_sell<8, true>(M.sell, op, gate, big);
            }
        });
    }
    template <class Op>
    void vec(int64_t n, const Op& op, const int32_t* gate, const char* what) {
        launch(AMG_PROF_VECTOR, 8.0 * n * Op::STREAMS, what,
               [&] { vec_kernel<Op><<<grid_for(n), kBlock, 0, stream>>>(n, op, gate, red); });
    }

    // ---------------------------------------------------------------- V-cycle
    // Algorithm 2 on level l: out = V(f) from x = 0.  If
    // rho_fin is set, the last kernel also computes (f, out) and calls it.
    // Returns true if the dot was fused.
    template <class FinT>
    bool vcycle(int l, const double* f, double* out, const int32_t* gate, const FinT* rho_fin);
    bool vcycle_plain(int l, const double* f, double* out, const int32_t* gate) {
        return vcycle<FinRho>(l, f, out, gate, nullptr);
    }

    void cg_iteration(double* x, int parity);
    void bicgstab_iteration(double* x);
    amg_status solve(const double* f, double* x, double tol, int32_t maxiter, int32_t* iters, double* rel);
};

template <class FinT>
bool Handle::vcycle(int l, const double* f, double* out, const int32_t* gate, const FinT* rho_fin) {
    DevLevel& L = lv[l];
    const int nlev = (int)lv.size();
    if (l == nlev - 1) {  // coarsest: out = A_L^-1 f
        const int64_t warps = std::min<int64_t>(L.n, (int64_t)num_sms * 64);
        const int g = (int)std::max<int64_t>(1, (warps * 32 + kBlock - 1) / kBlock);
        launch(AMG_PROF_COARSE_SOLVE, 8.0 * L.n * L.n + 16.0 * L.n, "coarse gemv",
               [&] { dense_gemv<<<g, kBlock, 0, stream>>>(L.n, coarse_inv, f, out, gate); });
        return false;
    }
    DevLevel& C = lv[l + 1];
    const int npre = prm.npre, npost = prm.npost;
    const bool cheb = prm.relax == 2;
    const int K = prm.cheb_degree;

    // ---- pre-smoothing from x = 0 and residual t = f - A x
    double* x = L.x;
    double* y = L.y;
    bool x_is_mf = false;  // x == m o f implicitly (not materialised)
    if (!cheb) {
        if (npre == 0) {
            ck(cudaMemsetAsync(x, 0, L.n * sizeof(double), stream), "memset");
            rows_auto(L.A, OpResidual<0, NoFin>{x, f, L.t, {}}, gate, "residual");
        } else if (npre == 1) {
            x_is_mf = true;  // fused: t = f - A (m o f)
            rows_auto(L.A, OpRes0{L.m, f, L.t, {}}, gate, "res0");
        } else {
            vec(L.n, VMulDiag{L.m, f, x, {}}, gate, "x=mf");
            for (int s = 1; s < npre; ++s) {
                rows_auto(L.A, OpRelax<0, NoFin>{x, L.m, f, y, {}}, gate, "relax");
                std::swap(x, y);
            }
            rows_auto(L.A, OpResidual<0, NoFin>{x, f, L.t, {}}, gate, "residual");
        }
    } else {
        if (npre == 0) {
            ck(cudaMemsetAsync(x, 0, L.n * sizeof(double), stream), "memset");
        } else {
            for (int s = 0; s < npre; ++s) {
                for (int k = 0; k < K; ++k) {
                    if (s == 0 && k == 0) {
                        vec(L.n, VCheb0{f, L.diag, L.p, x, L.cheb_alpha[0], prm.cheb_scaled, {}}, gate,
                            "cheb0");
                    } else {
                        rows_auto(L.A,
                                  OpCheb<0, NoFin>{x, f, L.diag, L.p, y, L.cheb_alpha[k], L.cheb_beta[k],
                                                   prm.cheb_scaled, k == 0, {}},
                                  gate, "cheb");
                        std::swap(x, y);
                    }
                }
            }
        }
        rows_auto(L.A, OpResidual<0, NoFin>{x, f, L.t, {}}, gate, "residual");
    }

    // ---- restriction f_c = R t, coarse solve, prolongation x += P x_c
    rows_auto(L.R, OpSpmv{L.t, C.f}, gate, "restrict");
    vcycle_plain(l + 1, C.f, C.o, gate);
    if (x_is_mf)
        rows_auto(L.P, OpProl0{C.o, L.m, f, x, {}}, gate, "prolong0");
    else
        rows_auto(L.P, OpProlAdd{C.o, x, {}}, gate, "prolong");

    // ---- post-smoothing; the last sweep writes `out`
    if (!cheb) {
        if (npost == 0) {
            ck(cudaMemcpyAsync(out, x, L.n * sizeof(double), cudaMemcpyDeviceToDevice, stream), "copy");
            return false;
        }
        for (int s = 0; s < npost; ++s) {
            double* dst = (s == npost - 1) ? out : y;
            if (s == npost - 1 && rho_fin)
                rows_auto(L.A, OpRelax<1, FinT>{x, L.m, f, dst, *rho_fin}, gate, "relax+dot");
            else
                rows_auto(L.A, OpRelax<0, NoFin>{x, L.m, f, dst, {}}, gate, "relax");
            if (dst == y) std::swap(x, y);
        }
        return rho_fin != nullptr;
    }
    if (npost == 0) {
        ck(cudaMemcpyAsync(out, x, L.n * sizeof(double), cudaMemcpyDeviceToDevice, stream), "copy");
        return false;
    }
    for (int s = 0; s < npost; ++s) {
        for (int k = 0; k < K; ++k) {
            const bool lastk = (s == npost - 1) && (k == K - 1);
            double* dst = lastk ? out : y;
            if (lastk && rho_fin)
                rows_auto(L.A,
                          OpCheb<1, FinT>{x, f, L.diag, L.p, dst, L.cheb_alpha[k], L.cheb_beta[k], prm.cheb_scaled,
                                          k == 0, *rho_fin},
                          gate, "cheb+dot");
            else
                rows_auto(L.A,
                          OpCheb<0, NoFin>{x, f, L.diag, L.p, dst, L.cheb_alpha[k], L.cheb_beta[k], prm.cheb_scaled,
                                           k == 0, {}},
                          gate, "cheb");
            if (!lastk) std::swap(x, y);
        }
    }
    return rho_fin != nullptr;
}

// One CG iteration (§8c c-1): z = M r, rho = (r, z) [fused in the last V-cycle
// kernel]; p' = z + beta p, q = A p', sigma = (p', q) [one kernel];
// x += alpha p', r -= alpha q, (r, r) [one kernel].
void Handle::cg_iteration(double* x, int parity) {
    const int32_t* gate = &ks->done;
    double* pold = parity ? pb : pa;
    double* pnew = parity ? pa : pb;
    DevLevel& L0 = lv[0];
    FinRho frho{ks};
    if (!vcycle<FinRho>(0, r, z, gate, &frho)) vec(L0.n, VDot<FinRho>{r, z, frho}, gate, "dot(r,z)");
    rows_auto(L0.A, OpCgDir<FinSigma>{z, pold, pnew, q, ks, 0.0, FinSigma{ks}}, gate, "cg dir");
    vec(L0.n, VCgUpdate{x, r, pnew, q, ks, 0.0, FinCgUpdate{ks}}, gate, "cg update");
}

// One BiCGStab iteration (§8c c-1).
void Handle::bicgstab_iteration(double* x) {
    const int32_t* gate = &ks->done;
    const int32_t* gate2 = &ks->skip2;
    DevLevel& L0 = lv[0];
    vec(L0.n, VBiP{r, v, pa, ks, 0, 0, 0, {}}, gate, "bicg p");
    vcycle_plain(0, pa, ph, gate);
    rows_auto(L0.A, OpSpmvDot<1, FinBiAlpha>{ph, rhat, v, FinBiAlpha{ks}}, gate, "v=A ph");
    vec(L0.n, VBiS{r, v, s, ks, 0.0, FinBiS{ks}}, gate, "bicg s");
    vcycle_plain(0, s, sh, gate2);
    rows_auto(L0.A, OpSpmvDot<2, FinBiOmega>{sh, s, tv, FinBiOmega{ks}}, gate2, "t=A sh");
    vec(L0.n, VBiX{x, r, ph, sh, s, tv, rhat, ks, 0, 0, 0, FinBiX{ks}}, gate, "bicg x");
}

amg_status Handle::solve(const double* f, double* x, double tol, int32_t maxiter, int32_t* iters,
                         double* rel) {
    DevLevel& L0 = lv[0];
    const int64_t n = L0.n;
    const bool bicg = prm.solver == 1;
    const int64_t launches0 = launches;
    std::fill(acc_ms, acc_ms + 8, 0.0);
    std::fill(acc_bytes, acc_bytes + 8, 0.0);
    std::fill(acc_launches, acc_launches + 8, 0);
    alg_bytes = 0;
    collect(rec_direct, 0, true);  // discard launches issued outside a solve
    alg_bytes = 0;
    std::fill(acc_ms, acc_ms + 8, 0.0);
    std::fill(acc_bytes, acc_bytes + 8, 0.0);
    std::fill(acc_launches, acc_launches + 8, 0);
    cur_iter = -1;
    ck(cudaEventRecord(ev0, stream), "event");
    // scalars: maxiter in, everything else computed on the device
    std::memset(ks_host, 0, sizeof(KState));
    ks_host->maxiter = maxiter;
    ck(cudaMemcpyAsync(ks, ks_host, sizeof(KState), cudaMemcpyHostToDevice, stream), "ks init");
    vec(n, VNorm2{f, FinNorm{ks, tol}}, nullptr, "norm f");
    rows_auto(L0.A, OpResidual<1, FinInitRes>{x, f, r, FinInitRes{ks}}, nullptr, "r0");
    ck(cudaMemsetAsync(pa, 0, n * sizeof(double), stream), "memset");
    ck(cudaMemsetAsync(pb, 0, n * sizeof(double), stream), "memset");
    if (bicg) {
        ck(cudaMemcpyAsync(rhat, r, n * sizeof(double), cudaMemcpyDeviceToDevice, stream), "copy");
        ck(cudaMemsetAsync(v, 0, n * sizeof(double), stream), "memset");
    }
    ck(cudaMemcpyAsync(ks_host, ks, sizeof(KState), cudaMemcpyDeviceToHost, stream), "ks read");
    ck(cudaStreamSynchronize(stream), "sync");
    collect(rec_direct, 0, true);
    if (ks_host->nf == 0.0) {  // zero right-hand side: x = 0
        ck(cudaMemsetAsync(x, 0, n * sizeof(double), stream), "memset");
        ck(cudaStreamSynchronize(stream), "sync");
        *iters = 0;
        *rel = 0.0;
        stats = amg_solve_stats{};
        stats.kernel_launches = launches - launches0;
        stats.alg_bytes = alg_bytes;
        return AMG_OK;
    }

    // Krylov loop: two iterations per host round trip, replayed from a CUDA
    // graph; kernels of iterations past convergence exit at their gate.
    const bool use_graph = prm.use_graph && !sync_debug;
    auto two_iterations = [&] {
        for (int k = 0; k < 2; ++k) {
            cur_iter = k;
            if (bicg)
                bicgstab_iteration(x);
            else
                cg_iteration(x, k);
        }
        cur_iter = -1;
    };
    while (!ks_host->done) {
        const int iter_before = ks_host->iter;
        if (use_graph) {
            if (!graph || graph_x != x || graph_prof_mask != prof_mask) {
                drop_graph();
                cudaGraph_t g;
                const int64_t before = launches;
                ck(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal), "capture");
                capturing = true;
                try {
                    two_iterations();
                } catch (...) {
                    capturing = false;
                    cudaStreamEndCapture(stream, &g);
                    throw;
                }
                capturing = false;
                ck(cudaStreamEndCapture(stream, &g), "end capture");
                graph_kernels = launches - before;
                launches = before;
                ck(cudaGraphInstantiate(&graph, g, 0), "instantiate");
                cudaGraphDestroy(g);
                graph_x = x;
                graph_prof_mask = prof_mask;
            }
            ck(cudaGraphLaunch(graph, stream), "graph launch");
            launches += graph_kernels;
        } else {
            two_iterations();
        }
        ck(cudaMemcpyAsync(ks_host, ks, sizeof(KState), cudaMemcpyDeviceToHost, stream), "ks read");
        ck(cudaStreamSynchronize(stream), "sync");
        const int ran = ks_host->iter - iter_before + (ks_host->done && ks_host->status ? 1 : 0);
        collect(use_graph ? rec_graph : rec_direct, ran, !use_graph);
    }
    // true residual |f - A x| / |f|
    rows_auto(L0.A, OpResidual<1, FinTrueRes>{x, f, r, FinTrueRes{ks}}, nullptr, "true res");
    ck(cudaEventRecord(ev1, stream), "event");
    ck(cudaMemcpyAsync(ks_host, ks, sizeof(KState), cudaMemcpyDeviceToHost, stream), "ks read");
    ck(cudaStreamSynchronize(stream), "sync");
    collect(rec_direct, 0, true);
    *iters = ks_host->iter;
    *rel = ks_host->true_res / ks_host->nf;
    float ms = 0;
    cudaEventElapsedTime(&ms, ev0, ev1);
    stats = amg_solve_stats{};
    stats.iters = ks_host->iter;
    stats.vcycles = bicg ? 2 * ks_host->iter - (ks_host->half ? 1 : 0) : ks_host->iter;
    stats.status = ks_host->status;
    stats.kernel_launches = launches - launches0;
    stats.solve_ms = ms;
    stats.rel_resid = *rel;
    stats.alg_bytes = alg_bytes;
    for (int c = 0; c < 8; ++c) {
        stats.prof_ms[c] = acc_ms[c];
        stats.prof_bytes[c] = acc_bytes[c];
        stats.prof_launches[c] = acc_launches[c];
    }
    if (ks_host->status == AMG_BREAKDOWN) {
        g_err = bicg ? "BiCGStab breakdown" : "CG breakdown: (r, Mr) <= 0 or (p, Ap) <= 0";
        stats.status = AMG_BREAKDOWN;
        return AMG_BREAKDOWN;
    }
    const amg_status st = ks_host->res <= ks_host->tolnf ? AMG_OK : AMG_NOT_CONVERGED;
    stats.status = st;
    return st;
}

// ---- upload -------------------------------------------------------------------

namespace {

// Matrix format policy: AMGB_FORMAT = auto (default) | csr | sell | tma.
// auto: row-block CSR for matrices with < 65536 rows (coarse levels: few, long
// rows); otherwise TMA-staged SELL-32 for narrow rows, SELL-32 for wide ones.
Fmt pick_format(const Csr& A) {
    const char* e = std::getenv("AMGB_FORMAT");
    const std::string f = e ? e : "auto";
    if (f == "csr") return Fmt::CSR;
    if (f == "sell") return Fmt::SELL;
    if (f == "tma") return Fmt::TMA;
    if (A.nrows < 65536) return Fmt::CSR;
    int64_t lmax = 0;
    for (int64_t r = 0; r < A.nrows; ++r) lmax = std::max<int64_t>(lmax, A.ptr[r + 1] - A.ptr[r]);
    // narrow rows (level-0 A, P): TMA-staged SELL-32, one thread per row.  Wide
    // rows (coarse A, R): their gathers are L2-bound and one thread per row of a
    // register-pipelined SELL-32 measured faster than T > 1 lanes per row.
    return lmax <= 12 ? Fmt::TMA : Fmt::SELL;
}

// Row blocks of the CSR kernel: at most kEnt entries and a row cap chosen from
// the mean row length; a row longer than kEnt forms a block of its own.
std::vector<int32_t> row_blocks(const Csr& A, int G) {
    const double avg = A.nrows ? (double)A.nnz() / (double)A.nrows : 0.0;
    const int64_t cap = G > 1 ? kRowsMax : (avg < 4.0 ? 512 : 256);
    std::vector<int32_t> b{0};
    int64_t r = 0;
    while (r < A.nrows) {
        int64_t ents = 0, rows = 0;
        if (A.ptr[r + 1] - A.ptr[r] > kEnt) {
            ++r;
        } else {
            while (r < A.nrows && rows < cap && ents + (A.ptr[r + 1] - A.ptr[r]) <= kEnt) {
                ents += A.ptr[r + 1] - A.ptr[r];
                ++rows;
                ++r;
            }
        }
        b.push_back((int32_t)r);
    }
    return b;
}

DMat upload_mat(Handle& H, const Csr& A, int64_t* bytes) {
    DMat d;
    d.nrows = A.nrows;
    d.ncols = A.ncols;
    d.nnz = A.nnz();
    if (d.nnz >= INT32_MAX) throw CudaError{"level has >= 2^31 nonzeros"};
    d.fmt = pick_format(A);
    d.is_csr = d.fmt == Fmt::CSR;
    if (d.is_csr) {
        const double avg = A.nrows ? (double)A.nnz() / (double)A.nrows : 0.0;
        int G = 1;
        if (avg >= 96) G = 16;
        else if (avg >= 48) G = 8;
        else if (avg >= 20) G = 4;
        else if (avg >= 12) G = 2;
        std::vector<int32_t> ptr32(A.ptr.begin(), A.ptr.end());
        std::vector<int32_t> blocks = row_blocks(A, G);
        d.csr.nrows = A.nrows;
        d.csr.ncols = A.ncols;
        d.csr.nnz = A.nnz();
        d.csr.nblocks = (int64_t)blocks.size() - 1;
        d.csr.G = G;
        d.csr.ptr = H.upload(ptr32);
        d.csr.col = H.upload(A.col);
        d.csr.val = H.upload(A.val);
        d.csr.brow = H.upload(blocks);
        d.stored = d.nnz;
        *bytes += (int64_t)(ptr32.size() * 4 + A.col.size() * 12 + blocks.size() * 4);
    } else if (d.fmt == Fmt::SELL) {
        HostSell S = to_sell(A, 32);
        d.sell.nrows = S.nrows;
        d.sell.ncols = S.ncols;
        d.sell.nslices = S.nslices;
        d.sell.sptr = H.upload(S.sptr);
        d.sell.col = H.upload(S.col);
        d.sell.val = H.upload(S.val);
        d.stored = (int64_t)S.col.size();
        for (int64_t q = 0; q < S.nslices; ++q) d.sell_wmax = std::max(d.sell_wmax, (S.sptr[q + 1] - S.sptr[q]) / 32);
        *bytes += (int64_t)(S.sptr.size() * 8 + S.col.size() * 12);
    } else {  // TMA-staged SELL-C: lanes per row T from the longest row, C = 32 / T
        int64_t lmax = 0;
        for (int64_t r = 0; r < A.nrows; ++r) lmax = std::max<int64_t>(lmax, A.ptr[r + 1] - A.ptr[r]);
        const char* te_env = std::getenv("AMGB_TMA_T");
        int T = lmax <= 12 ? 1 : lmax <= 24 ? 2 : lmax <= 48 ? 4 : 8;
        if (te_env) T = std::atoi(te_env);
        const int C = 32 / T;
        HostSell S = to_sell(A, C);
        SellTma& t = d.tma;
        t.nrows = S.nrows;
        t.ncols = S.ncols;
        t.nslices = S.nslices;
        t.T = T;
        t.ntiles = (S.nslices + 7) / 8;
        int64_t te = 0;
        for (int64_t q = 0; q < t.ntiles; ++q)
            te = std::max(te, S.sptr[std::min<int64_t>((q + 1) * 8, S.nslices)] - S.sptr[q * 8]);
        t.tile_ent = (int32_t)(((std::max<int64_t>(te, 32) + 31) / 32) * 32);
        t.sptr = H.upload(S.sptr);
        t.col = H.upload(S.col);
        t.val = H.upload(S.val);
        d.stored = (int64_t)S.col.size();
        *bytes += (int64_t)(S.sptr.size() * 8 + S.col.size() * 12);
    }
    return d;
}

// Chebyshev coefficients (§8c c-1): alpha_0 = 1/d; alpha_1 = 2d/(2d^2 - c^2);
// alpha_k = 1/(d - alpha_{k-1} c^2/4); beta_k = alpha_k d - 1.
void cheb_coeffs(double d, double c, int K, std::vector<double>& a, std::vector<double>& b) {
    a.assign(std::max(K, 1), 0.0);
    b.assign(std::max(K, 1), 0.0);
    double alpha = 0.0;
    for (int k = 0; k < K; ++k) {
        if (k == 0)
            alpha = 1.0 / d;
        else if (k == 1)
            alpha = 2.0 * d / (2.0 * d * d - c * c);
        else
            alpha = 1.0 / (d - alpha * c * c / 4.0);
        a[k] = alpha;
        b[k] = k == 0 ? 0.0 : alpha * d - 1.0;
    }
}

// Algorithmic HBM bytes of one V-cycle on level l: every matrix
// read once per pass (12 B per entry + 4 B per row), every vector read or
// written once per kernel that touches it.
double level_alg_bytes(const DevLevel& L, const amg_params& p, bool coarsest) {
    const double n = (double)L.n, z = (double)L.nnzA;
    if (coarsest) return 8.0 * n * n + 16.0 * n;
    const double pp = (double)L.nnzP, c = (double)L.nc;
    const double apass_relax = 12 * z + 4 * n + 32 * n;  // x, m, f read, out written
    const double restrict_b = 12 * pp + 4 * c + 8 * n + 8 * c;
    if (p.relax == 2) {
        const double step = 12 * z + 4 * n + 40 * n;  // x, f, p read; p, xo written
        const double K = p.cheb_degree;
        const double pre = p.npre > 0 ? 32 * n + (K * p.npre - 1) * step : 0;
        const double post = p.npost * K * step;
        const double res = 12 * z + 4 * n + 24 * n;
        const double prol = 12 * pp + 4 * n + 8 * c + 16 * n;
        return pre + res + restrict_b + prol + post;
    }
    double pre = 0, prol = 0;
    if (p.npre == 1) {
        pre = 12 * z + 4 * n + 32 * n;  // m, f read (gathered once), t written
        prol = 12 * pp + 4 * n + 8 * c + 24 * n;  // m, f read, x written
    } else {
        pre = (p.npre > 0 ? 24 * n + (p.npre - 1) * apass_relax : 8 * n) + 12 * z + 4 * n + 24 * n;
        prol = 12 * pp + 4 * n + 8 * c + 16 * n;
    }
    return pre + restrict_b + prol + p.npost * apass_relax;
}

}  // namespace

}  // namespace amgb

// ============================================================ C ABI

using amgb::Handle;
using amgb::ck;

struct amg_hierarchy {
    std::unique_ptr<Handle> h;
};

static amg_status set_error(amg_status st, const std::string& msg) {
    amgb::g_err = msg;
    return st;
}

extern "C" {

void amg_params_default(amg_params* p) {
    if (!p) return;
    std::memset(p, 0, sizeof(*p));
    p->struct_size = sizeof(amg_params);
    p->coarsening = 0;
    p->eps_strong = 0.08;
    p->eps_decay = 0.5;
    p->p_omega = 2.0 / 3.0;
    p->relax = 0;
    p->jacobi_omega = 0.72;
    p->cheb_degree = 5;
    p->cheb_lower = 1.0 / 30.0;
    p->cheb_scaled = 1;
    p->npre = 1;
    p->npost = 1;
    p->coarse_enough = 3000;
    p->max_levels = 30;
    p->dense_max = 20000;
    p->solver = 0;
    p->device = 0;
    p->use_graph = 1;
}

const char* amg_last_error(void) { return amgb::g_err.c_str(); }

const char* amg_version(void) {
    return "amgb 0.1 (sm_100a; SELL-32 fp64 solve phase; host SA setup)";
}

static amg_status check_params(const amg_params& p) {
    if (p.struct_size != sizeof(amg_params)) return set_error(AMG_E_INVALID_ARG, "amg_params: struct_size mismatch");
    if (p.coarsening < 0 || p.coarsening > 1) return set_error(AMG_E_INVALID_ARG, "coarsening must be 0 or 1");
    if (p.relax < 0 || p.relax > 2) return set_error(AMG_E_INVALID_ARG, "relax must be 0, 1 or 2");
    if (p.solver < 0 || p.solver > 1) return set_error(AMG_E_INVALID_ARG, "solver must be 0 or 1");
    if (p.npre < 0 || p.npost < 0 || p.npre + p.npost < 1)
        return set_error(AMG_E_INVALID_ARG, "npre, npost >= 0 and npre + npost >= 1");
    if (p.relax == 2 && (p.cheb_degree < 1 || !(p.cheb_lower > 0 && p.cheb_lower < 1)))
        return set_error(AMG_E_INVALID_ARG, "chebyshev: degree >= 1, 0 < lower < 1");
    if (!(p.eps_strong >= 0 && p.eps_strong < 1) || !(p.eps_decay > 0 && p.eps_decay <= 1))
        return set_error(AMG_E_INVALID_ARG, "eps_strong in [0,1), eps_decay in (0,1]");
    if (!(p.p_omega >= 0 && p.p_omega < 2)) return set_error(AMG_E_INVALID_ARG, "p_omega in [0,2)");
    if (p.coarse_enough < 1 || p.max_levels < 1 || p.dense_max < 1)
        return set_error(AMG_E_INVALID_ARG, "coarse_enough, max_levels, dense_max >= 1");
    return AMG_OK;
}

amg_status amg_setup(int64_t n, const int64_t* ptr, const int32_t* col, const double* val,
                     const amg_params* prm_in, amg_handle* out) {
    using namespace amgb;
    if (!out) return set_error(AMG_E_INVALID_ARG, "out is NULL");
    *out = nullptr;
    if (n <= 0 || n > INT32_MAX || !ptr || (!col && ptr[n] > 0) || (!val && ptr[n] > 0))
        return set_error(AMG_E_INVALID_ARG, "n must be in [1, 2^31) and ptr/col/val non-NULL");
    amg_params prm;
    if (prm_in)
        prm = *prm_in;
    else
        amg_params_default(&prm);
    if (amg_status st = check_params(prm)) return st;
    auto H = std::make_unique<Handle>();
    H->prm = prm;
    H->sync_debug = std::getenv("AMGB_SYNC_DEBUG") != nullptr;
    try {
        validate_csr(n, ptr, col);
        Csr A0;
        A0.nrows = A0.ncols = n;
        A0.ptr.assign(ptr, ptr + n + 1);
        A0.col.assign(col, col + ptr[n]);
        A0.val.assign(val, val + ptr[n]);
        SetupParams sp;
        sp.smoothed = prm.coarsening == 0;
        sp.eps_strong = prm.eps_strong;
        sp.eps_decay = prm.eps_decay;
        sp.p_omega = prm.p_omega;
        sp.relax = prm.relax;
        sp.jacobi_omega = prm.jacobi_omega;
        sp.cheb_degree = prm.cheb_degree;
        sp.cheb_lower = prm.cheb_lower;
        sp.cheb_scaled = prm.cheb_scaled != 0;
        sp.coarse_enough = prm.coarse_enough;
        sp.max_levels = prm.max_levels;
        sp.dense_max = prm.dense_max;
        H->host = build_hierarchy(std::move(A0), sp);
    } catch (const SetupError& e) {
        return set_error((amg_status)e.code, e.msg);
    } catch (const std::bad_alloc&) {
        return set_error(AMG_E_OOM, "host allocation failed during setup");
    }
    const int nlev = (int)H->host.levels.size();
    H->lv.resize(nlev);
    for (int l = 0; l < nlev; ++l) {
        const HostLevel& hl = H->host.levels[l];
        DevLevel& L = H->lv[l];
        L.n = hl.A.nrows;
        L.nnzA = hl.A.nnz();
        L.nc = l + 1 < nlev ? hl.P.ncols : 0;
        L.nnzP = l + 1 < nlev ? hl.P.nnz() : 0;
        if (prm.relax == 2 && l + 1 < nlev)
            cheb_coeffs(hl.cheb_d, hl.cheb_c, prm.cheb_degree, L.cheb_alpha, L.cheb_beta);
        L.alg_bytes = level_alg_bytes(L, prm, l == nlev - 1);
    }
    H->nL = H->host.levels.back().A.nrows;
    if (prm.device < 0) {
        *out = new amg_hierarchy{std::move(H)};
        return AMG_OK;
    }
    try {
        ck(cudaSetDevice(prm.device), "cudaSetDevice");
        H->device = prm.device;
        ck(cudaDeviceGetAttribute(&H->num_sms, cudaDevAttrMultiProcessorCount, prm.device), "attr");
        ck(cudaEventCreate(&H->ev0), "event");
        ck(cudaEventCreate(&H->ev1), "event");
        ck(cudaStreamCreate(&H->own_stream), "stream");  // capture needs a non-legacy stream
        H->stream = H->own_stream;
        for (int l = 0; l < nlev; ++l) {
            const HostLevel& hl = H->host.levels[l];
            DevLevel& L = H->lv[l];
            const bool coarsest = l == nlev - 1;
            if (!coarsest) {
                L.A = upload_mat(*H, hl.A, &L.dev_bytes);
                L.P = upload_mat(*H, hl.P, &L.dev_bytes);
                L.R = upload_mat(*H, hl.R, &L.dev_bytes);
                L.padA = L.A.stored;
                if (prm.relax != 2) L.m = H->upload(hl.m);
                if (prm.relax == 2) L.diag = H->upload(hl.diag);  // Chebyshev D^-1 scaling
                L.x = H->dalloc(L.n);
                L.y = H->dalloc(L.n);
                L.t = H->dalloc(L.n);
                if (prm.relax == 2) L.p = H->dalloc(L.n);
                L.dev_bytes += 8 * L.n * (prm.relax == 2 ? 5 : 4);
            } else {
                L.padA = L.nnzA;
            }
            if (l > 0) {
                L.f = H->dalloc(L.n);
                L.o = H->dalloc(L.n);
                L.dev_bytes += 16 * L.n;
            }
        }
        H->coarse_inv = H->upload(H->host.coarse_inv);
        H->lv.back().dev_bytes += 8 * H->nL * H->nL;
        if (nlev == 1) {  // single level: the level-0 A is needed by the Krylov loop
            int64_t dummy = 0;
            H->lv[0].A = upload_mat(*H, H->host.levels[0].A, &H->lv[0].dev_bytes);
            H->lv[0].padA = H->lv[0].A.stored;
            (void)dummy;
        }
        const int64_t n = H->lv[0].n;
        void* p = nullptr;
        ck(cudaMalloc(&p, sizeof(KState)), "cudaMalloc");
        H->allocs.push_back(p);
        H->ks = static_cast<amgb::KState*>(p);
        ck(cudaMallocHost(&H->ks_host, sizeof(amgb::KState)), "cudaMallocHost");
        ck(cudaMalloc(&p, (size_t)H->num_sms * 8 * 4 * sizeof(double)), "cudaMalloc");
        H->allocs.push_back(p);
        H->red.partial = static_cast<double*>(p);
        ck(cudaMalloc(&p, 64), "cudaMalloc");
        H->allocs.push_back(p);
        ck(cudaMemset(p, 0, 64), "memset");
        H->red.ticket = static_cast<unsigned int*>(p);
        H->zero_gate = reinterpret_cast<int32_t*>(static_cast<char*>(p) + 32);
        H->r = H->dalloc(n);
        H->z = H->dalloc(n);
        H->pa = H->dalloc(n);
        H->pb = H->dalloc(n);
        H->q = H->dalloc(n);
        if (prm.solver == 1) {
            H->rhat = H->dalloc(n);
            H->v = H->dalloc(n);
            H->s = H->dalloc(n);
            H->sh = H->dalloc(n);
            H->ph = H->dalloc(n);
            H->tv = H->dalloc(n);
        }
        ck(cudaDeviceSynchronize(), "setup sync");
        H->on_device = true;
    } catch (const amgb::CudaError& e) {
        cudaGetLastError();
        return set_error(e.msg.find("out of memory") != std::string::npos ? AMG_E_OOM : AMG_E_CUDA, e.msg);
    }
    *out = new amg_hierarchy{std::move(H)};
    return AMG_OK;
}

void amg_destroy(amg_handle h) { delete h; }

static amg_status need_device(amg_handle h) {
    if (!h || !h->h) return set_error(AMG_E_INVALID_ARG, "NULL handle");
    if (!h->h->on_device) return set_error(AMG_E_NO_DEVICE, "host-only handle (params.device = -1)");
    return AMG_OK;
}

amg_status amg_solve(amg_handle h, const double* f, double* x, double tol, int32_t maxiter, int32_t* iters,
                     double* rel) {
    if (amg_status st = need_device(h)) return st;
    if (!f || !x || !iters || !rel || f == x) return set_error(AMG_E_INVALID_ARG, "f, x, iters, rel");
    if (!(tol >= 0) || maxiter < 0) return set_error(AMG_E_INVALID_ARG, "tol >= 0, maxiter >= 0");
    try {
        ck(cudaSetDevice(h->h->device), "cudaSetDevice");
        return h->h->solve(f, x, tol, maxiter, iters, rel);
    } catch (const amgb::CudaError& e) {
        cudaGetLastError();
        return set_error(AMG_E_CUDA, e.msg);
    }
}

amg_status amg_solve_host(amg_handle h, const double* f, double* x, double tol, int32_t maxiter,
                          int32_t* iters, double* rel) {
    if (amg_status st = need_device(h)) return st;
    if (!f || !x || !iters || !rel) return set_error(AMG_E_INVALID_ARG, "f, x, iters, rel");
    Handle& H = *h->h;
    const int64_t n = H.lv[0].n;
    try {
        ck(cudaSetDevice(H.device), "cudaSetDevice");
        if (!H.hf) {
            H.hf = H.dalloc(n);
            H.hx = H.dalloc(n);
        }
        ck(cudaMemcpyAsync(H.hf, f, n * sizeof(double), cudaMemcpyHostToDevice, H.stream), "H2D f");
        ck(cudaMemcpyAsync(H.hx, x, n * sizeof(double), cudaMemcpyHostToDevice, H.stream), "H2D x");
        amg_status st = H.solve(H.hf, H.hx, tol, maxiter, iters, rel);
        ck(cudaMemcpyAsync(x, H.hx, n * sizeof(double), cudaMemcpyDeviceToHost, H.stream), "D2H x");
        ck(cudaStreamSynchronize(H.stream), "sync");
        return st;
    } catch (const amgb::CudaError& e) {
        cudaGetLastError();
        return set_error(AMG_E_CUDA, e.msg);
    }
}

amg_status amg_precond_apply(amg_handle h, const double* r, double* z) {
    if (amg_status st = need_device(h)) return st;
    if (!r || !z || r == z) return set_error(AMG_E_INVALID_ARG, "r, z");
    try {
        ck(cudaSetDevice(h->h->device), "cudaSetDevice");
        h->h->vcycle_plain(0, r, z, nullptr);
        ck(cudaGetLastError(), "launch");
    } catch (const amgb::CudaError& e) {
        return set_error(AMG_E_CUDA, e.msg);
    }
    return AMG_OK;
}

amg_status amg_set_stream(amg_handle h, void* stream) {
    if (!h || !h->h) return set_error(AMG_E_INVALID_ARG, "NULL handle");
    // the legacy default stream cannot be captured into a graph: keep the
    // handle's own blocking stream, which is ordered with it implicitly
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : h->h->own_stream;
    if (h->h->stream != s) h->h->drop_graph();
    h->h->stream = s;
    return AMG_OK;
}

amg_status amg_set_profile(amg_handle h, int32_t mask) {
    if (!h || !h->h) return set_error(AMG_E_INVALID_ARG, "NULL handle");
    h->h->prof_mask = mask & 0xff;
    return AMG_OK;
}

amg_status amg_level_count(amg_handle h, int32_t* nlevels) {
    if (!h || !h->h || !nlevels) return set_error(AMG_E_INVALID_ARG, "NULL argument");
    *nlevels = (int32_t)h->h->host.levels.size();
    return AMG_OK;
}

amg_status amg_level_info_get(amg_handle h, int32_t l, amg_level_info* out) {
    if (!h || !h->h || !out) return set_error(AMG_E_INVALID_ARG, "NULL argument");
    const Handle& H = *h->h;
    if (l < 0 || l >= (int)H.host.levels.size()) return set_error(AMG_E_INVALID_ARG, "level out of range");
    const auto& hl = H.host.levels[l];
    const auto& L = H.lv[l];
    const bool coarsest = l == (int)H.host.levels.size() - 1;
    std::memset(out, 0, sizeof(*out));
    out->rows = hl.A.nrows;
    out->nnz_A = hl.A.nnz();
    out->nnz_P = coarsest ? 0 : hl.P.nnz();
    out->cols_P = coarsest ? 0 : hl.P.ncols;
    out->aggregates = coarsest ? 0 : hl.n_agg;
    out->is_coarsest = coarsest;
    out->dev_bytes = L.dev_bytes;
    out->padded_nnz_A = L.padA;
    out->alg_bytes_vcycle = L.alg_bytes;
    return AMG_OK;
}

static void copy_csr(const amgb::Csr& M, int64_t* p, int32_t* c, double* v) {
    if (p) std::copy(M.ptr.begin(), M.ptr.end(), p);
    if (c) std::copy(M.col.begin(), M.col.end(), c);
    if (v) std::copy(M.val.begin(), M.val.end(), v);
}

amg_status amg_export_level(amg_handle h, int32_t l, const amg_level_export* out) {
    if (!h || !h->h || !out) return set_error(AMG_E_INVALID_ARG, "NULL argument");
    const Handle& H = *h->h;
    if (l < 0 || l >= (int)H.host.levels.size()) return set_error(AMG_E_INVALID_ARG, "level out of range");
    const auto& hl = H.host.levels[l];
    const bool coarsest = l == (int)H.host.levels.size() - 1;
    copy_csr(hl.A, out->A_ptr, out->A_col, out->A_val);
    if (!coarsest) {
        copy_csr(hl.P, out->P_ptr, out->P_col, out->P_val);
        copy_csr(hl.R, out->R_ptr, out->R_col, out->R_val);
        if (out->aggregates) std::copy(hl.agg.begin(), hl.agg.end(), out->aggregates);
        if (out->smoother) {
            if (H.prm.relax == 2) {
                out->smoother[0] = hl.lmax;
                out->smoother[1] = hl.lmin;
                out->smoother[2] = hl.cheb_d;
                out->smoother[3] = hl.cheb_c;
            } else {
                std::copy(hl.m.begin(), hl.m.end(), out->smoother);
            }
        }
    } else if (out->coarse_inverse) {
        std::copy(H.host.coarse_inv.begin(), H.host.coarse_inv.end(), out->coarse_inverse);
    }
    return AMG_OK;
}

amg_status amg_solve_stats_get(amg_handle h, amg_solve_stats* out) {
    if (!h || !h->h || !out) return set_error(AMG_E_INVALID_ARG, "NULL argument");
    *out = h->h->stats;
    return AMG_OK;
}

amg_status amg_level_op(amg_handle h, int32_t l, int32_t op, const double* x, const double* f, double* y) {
    using namespace amgb;
    if (amg_status st = need_device(h)) return st;
    Handle& H = *h->h;
    const int nlev = (int)H.lv.size();
    if (l < 0 || l >= nlev) return set_error(AMG_E_INVALID_ARG, "level out of range");
    const bool coarsest = l == nlev - 1;
    DevLevel& L = H.lv[l];
    try {
        ck(cudaSetDevice(H.device), "cudaSetDevice");
        switch (op) {
            case AMG_OP_SPMV_A:
                if (coarsest && nlev > 1) return set_error(AMG_E_INVALID_ARG, "coarsest A is stored dense");
                H.rows_auto(L.A, OpSpmv{x, y}, nullptr, "spmv A");
                break;
            case AMG_OP_SPMV_P:
            case AMG_OP_SPMV_R:
                if (coarsest) return set_error(AMG_E_INVALID_ARG, "no P/R on the coarsest level");
                if (op == AMG_OP_SPMV_P)
                    H.rows_auto(L.P, OpSpmv{x, y}, nullptr, "spmv P");
                else
                    H.rows_auto(L.R, OpSpmv{x, y}, nullptr, "spmv R");
                break;
            case AMG_OP_RESIDUAL:
                if (coarsest && nlev > 1) return set_error(AMG_E_INVALID_ARG, "coarsest A is stored dense");
                H.rows_auto(L.A, OpResidual<0, NoFin>{x, f, y, {}}, nullptr, "residual");
                break;
            case AMG_OP_RELAX:
                if (coarsest) return set_error(AMG_E_INVALID_ARG, "no smoother on the coarsest level");
                if (H.prm.relax == 2) {
                    // one full smoother call: K Chebyshev steps from x (fresh recurrence)
                    double* a = L.x;
                    double* b = L.y;
                    ck(cudaMemcpyAsync(a, x, L.n * sizeof(double), cudaMemcpyDeviceToDevice, H.stream), "copy");
                    for (int k = 0; k < H.prm.cheb_degree; ++k) {
                        double* dst = (k == H.prm.cheb_degree - 1) ? y : b;
                        H.rows_auto(L.A,
                                    OpCheb<0, NoFin>{a, f, L.diag, L.p, dst, L.cheb_alpha[k], L.cheb_beta[k],
                                                     H.prm.cheb_scaled, k == 0, {}},
                                    nullptr, "cheb");
                        std::swap(a, b);
                    }
                } else {
                    H.rows_auto(L.A, OpRelax<0, NoFin>{x, L.m, f, y, {}}, nullptr, "relax");
                }
                break;
            case AMG_OP_COARSE:
                if (!coarsest) return set_error(AMG_E_INVALID_ARG, "not the coarsest level");
                H.vcycle_plain(l, f, y, nullptr);
                break;
            case AMG_OP_VCYCLE:
                H.vcycle_plain(l, f, y, nullptr);
                break;
            default:
                return set_error(AMG_E_INVALID_ARG, "unknown op");
        }
        ck(cudaGetLastError(), "launch");
    } catch (const amgb::CudaError& e) {
        return set_error(AMG_E_CUDA, e.msg);
    }
    return AMG_OK;
}

}  // extern "C"
