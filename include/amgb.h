/*
 * amgb.h -- C ABI of the B200 smoothed-aggregation AMG solve phase.
 *
 * What it computes (arXiv 1811.05704, "AMGCL", PAPER.md):
 *   the solution of A u = f (Eq. (1)) by a Krylov method (CG, or
 *   BiCGStab for non-symmetric A) preconditioned by one AMG
 *   V-cycle (Algorithm 2; "single V-cycle is used as a
 *   preconditioning step").  The hierarchy is built inside
 *   amg_setup (Algorithm 1) with smoothed (or plain) aggregation
 *    -- by default on the GPU, bitwise equal to the host build the
 *   paper prescribes ("the AMG hierarchy is always constructed on the main
 *   processor (CPU)"), which params.setup_device = 0 selects --
 *   and the solve phase runs entirely in this library's sm_100a kernels.
 *   The readings of the paper this implementation commits to are listed in
 *   DESIGN.md §3 (strength test, aggregation order, smoother constants, ...).
 *
 * Conventions common to every call:
 *   - Return value: amg_status; 0 = OK, > 0 = result valid but flagged,
 *     < 0 = error (nothing was computed; amg_last_error() has a message).
 *   - Matrices: square CSR with int64 row pointers (n+1), int32 column indices
 *     strictly increasing within each row and in [0, n), fp64 values.  Empty rows
 *     are legal; every row must hold a positive diagonal entry (the strength test
 *     a_ij^2 > eps^2 a_ii a_jj needs it).
 *   - "device" pointers are CUDA global-memory fp64 arrays on the handle's
 *     device, length n, not aliased with each other, 8-byte aligned (16-byte
 *     alignment, e.g. any cudaMalloc / torch allocation, lets the vector kernels
 *     use paired 16-byte accesses; amg_solve_stats.flags bit 2 reports when a
 *     solve could not); "host"
 *     pointers are ordinary (pageable or pinned) host memory.
 *   - Work is issued on the handle's stream (amg_set_stream; default: a stream
 *     the handle creates, which is ordered with the legacy default stream).  Calls that return results (amg_solve*) synchronise that
 *     stream before returning; amg_precond_apply and amg_level_op are
 *     asynchronous.
 *   - A handle is not re-entrant; distinct handles may be used concurrently.
 *   - amg_last_error() is thread-local.
 */
#ifndef AMGB_H
#define AMGB_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    AMG_OK = 0,
    AMG_NOT_CONVERGED = 1,      /* maxiter reached; outputs valid */
    AMG_BREAKDOWN = 2,          /* CG (r,Mr) <= 0 or (p,Ap) <= 0; BiCGStab rho/omega underflow */
    AMG_E_INVALID_ARG = -1,
    AMG_E_BAD_CSR = -2,         /* CSR invariants violated (message names the row) */
    AMG_E_ZERO_DIAG = -3,       /* a diagonal entry is missing or not positive */
    AMG_E_SINGULAR_COARSE = -4, /* coarsest LU pivot below 1e-14 max|A_L| */
    AMG_E_COARSE_TOO_LARGE = -5,/* coarsest level larger than dense_max */
    AMG_E_OOM = -6,
    AMG_E_NO_DEVICE = -7,       /* solve requested on a host-only handle */
    AMG_E_CUDA = -10,
    AMG_E_NCCL = -11            /* multi-GPU: NCCL unavailable or failed, or a peer rank did not
                                   respond within AMGB_NCCL_TIMEOUT_S seconds [300] (communicator
                                   creation, setup scatter, any host synchronisation of a solve);
                                   the communicator is aborted and the handle must be destroyed */
} amg_status;

typedef struct amg_hierarchy *amg_handle;

/* Parameters; names follow the paper's runtime keys where it
 * has them.  Defaults (amg_params_default) in brackets; DESIGN.md §3 cites each. */
typedef struct {
    uint32_t struct_size;   /* = sizeof(amg_params) (ABI check) */
    int32_t coarsening;     /* "precond.coarsening.type": 0 smoothed_aggregation [0], 1 aggregation */
    double eps_strong;      /* strength threshold on the finest level [0.08] */
    double eps_decay;       /* eps on level l+1 = eps on level l * eps_decay [0.5] */
    double p_omega;         /* prolongation-smoother damping [2/3] */
    int32_t relax;          /* "precond.relax.type": 0 spai0 [0], 1 damped_jacobi, 2 chebyshev */
    double jacobi_omega;    /* damped Jacobi weight [0.72] */
    int32_t cheb_degree;    /* Chebyshev polynomial degree K [5] */
    double cheb_lower;      /* lambda_min = lambda_max * cheb_lower [1/30] */
    int32_t cheb_scaled;    /* 1: polynomial in D^-1 A [1]; 0: in A */
    int32_t npre, npost;    /* smoothing sweeps per level [1, 1] */
    int64_t coarse_enough;  /* stop coarsening at <= this many rows [3000] */
    int32_t max_levels;     /* [30] */
    int64_t dense_max;      /* error if the coarsest level is larger [20000] */
    int32_t solver;         /* "solver.type": 0 cg [0], 1 bicgstab, 2 gmres (restarted, right-preconditioned),
                               3 idrs (IDR(s) with bi-orthogonalisation, right-preconditioned; single GPU) */
    int32_t device;         /* CUDA device ordinal [0]; -1 = host-only handle (setup + export) */
    int32_t use_graph;      /* 1: replay Krylov iterations as a CUDA graph [1] */
    int32_t precision;      /* 0: fp64 throughout [0]; 1: mixed -- the V-cycle reads fp32 copies of
                               the hierarchy values (arithmetic and vectors stay fp64; the Krylov
                               method and its A stay fp64).  SURVEY §8f rank 2; value types
                               "double or float", PAPER.md:186-191 */
    int32_t gmres_m;        /* GMRES restart length m in [1, 64] [30] ("solver.M") */
    int32_t setup_device;   /* 1: the hierarchy is built on the CUDA device -- strength, the greedy
                               aggregation (Phase 1 by exact dependency propagation), smoothed P,
                               R = P^T, A P, R(AP), smoother data; only the coarsest dense inverse
                               on the host [1]; 0: everything on the host.  Bitwise the same
                               hierarchy either way (Algorithm 1,
                               PAPER.md:95-107).  Host-only handles (device = -1) use the host. */
    int32_t idrs_s;         /* IDR(s) shadow-space dimension s in {1, 2, 4, 8} [4] ("solver.s") */
    int32_t reorder;        /* locality reordering of the device store (single GPU):
                               the same hierarchy stored as Q_l A_l Q_l^T, Q_l P_l Q_{l+1}^T, ...
                               with q_0 = reverse Cuthill-McKee of A_0 and aggregates numbered by
                               their root; every API call permutes its vectors on entry and exit.
                               0 off, 1 on, 2 automatic: on when A_0's gathers are non-local (a
                               256-row tile touches > 0.5 distinct 32-byte sectors per entry) [2] */
} amg_params;

/* Per-level statistics (amg_level_info). */
typedef struct {
    int64_t rows, nnz_A, nnz_P, cols_P; /* nnz_P = nnz(R); 0 on the coarsest level */
    int64_t aggregates;                 /* = cols_P */
    int32_t is_coarsest;
    int32_t dict_slices_A;              /* 32-row slices of A stored with a column-offset
                                           dictionary (TMA SELL-32 format) */
    int64_t dev_bytes;                  /* device bytes of this level's store */
    int64_t padded_nnz_A;               /* stored (sliced-ELL) entries of A incl. padding */
    double alg_bytes_vcycle;            /* algorithmic HBM bytes of this level per V-cycle */
    int64_t padded_nnz_P, padded_nnz_R; /* stored entries of P and R incl. padding */
    int32_t sigma_mask;                 /* bit 0/1/2: A/P/R stored SELL-C-sigma (rows sorted by
                                           length inside 256-row windows) */
    int32_t formats;                    /* device format of A | P << 4 | R << 8 (single-GPU
                                           handles): AMG_FMT_*; value storage
                                           of A << 12 | P << 14 | R << 16: 0 fp64 array,
                                           1 8-bit / 2 16-bit index into a value table */
} amg_level_info;

/* device matrix formats (amg_level_info.formats) */
enum { AMG_FMT_CSR = 0,      /* row-block CSR (csr_rows) */
       AMG_FMT_SELL = 1,     /* SELL-32, one thread per row (sell_rows) */
       AMG_FMT_TMA = 2,      /* TMA-staged SELL-32 with the column-offset dictionary (sell_tma) */
       AMG_FMT_TMACSR = 3,   /* TMA-staged CSR, padding-free (csr_tma) */
       AMG_FMT_NONE = 15 };  /* no such matrix (coarsest level: P, R) */

/* Test/export hook (amg_export_level): caller-owned HOST buffers, sized from
 * amg_level_info; any pointer may be NULL to skip that array.  R = P^T. */
typedef struct {
    int64_t *A_ptr; int32_t *A_col; double *A_val;  /* rows+1, nnz_A, nnz_A */
    int64_t *P_ptr; int32_t *P_col; double *P_val;  /* rows+1, nnz_P, nnz_P */
    int64_t *R_ptr; int32_t *R_col; double *R_val;  /* cols_P+1, nnz_P, nnz_P */
    int32_t *aggregates;                            /* rows */
    double *smoother;   /* spai0/jacobi: m (rows); chebyshev: lmax, lmin, d, c */
    double *coarse_inverse; /* coarsest level only: rows*rows, row-major A_L^-1 */
} amg_level_export;

/* Solve statistics (amg_solve_stats), filled by the last amg_solve*. */
typedef struct {
    int32_t iters;          /* Krylov iterations (loop trips, DESIGN.md §3 R19) */
    int32_t vcycles;        /* preconditioner applications */
    int32_t status;
    int32_t flags;          /* bit 0: the fused CG iteration ran; bit 1: reordered store;
                               bit 2: f or x not 16-B aligned (scalar vector-kernel loop) */
    int64_t kernel_launches;/* kernels this library launched during the solve */
    double solve_ms;        /* device time of the solve (events on the handle stream) */
    double rel_resid;       /* true |f - A x| / |f| */
    double alg_bytes;       /* algorithmic HBM bytes of the kernels that ran */
    double prof_ms[8];      /* profile mode: device ms per kernel class (see AMG_PROF_*) */
    double prof_bytes[8];   /* profile mode: algorithmic bytes per kernel class */
    int64_t prof_launches[8];
} amg_solve_stats;

/* kernel classes timed in profile mode */
enum { AMG_PROF_A0_PASS = 0,   /* level-0 A passes (smoother/residual/CG direction) */
       AMG_PROF_A_COARSE = 1,  /* A passes on levels >= 1 */
       AMG_PROF_TRANSFER = 2,  /* restriction / prolongation */
       AMG_PROF_VECTOR = 3,    /* Krylov vector updates and norms */
       AMG_PROF_COARSE_SOLVE = 4 };

/* Fill *p with the defaults above (struct_size set). */
void amg_params_default(amg_params *p);

/* Build the hierarchy of A (host arrays: ptr[n+1], col[nnz], val[nnz], nnz =
 * ptr[n]) and, unless prm->device == -1, upload it to the current CUDA device
 * (prm->device).  The caller keeps ownership of the inputs and may free them on
 * return; *out owns every allocation (release with amg_destroy).  prm may be NULL
 * (defaults).  Errors: AMG_E_INVALID_ARG (n <= 0, NULL pointers, bad params),
 * AMG_E_BAD_CSR, AMG_E_ZERO_DIAG, AMG_E_SINGULAR_COARSE, AMG_E_COARSE_TOO_LARGE,
 * AMG_E_OOM, AMG_E_CUDA.  Cite: Algorithm 1. */
amg_status amg_setup(int64_t n, const int64_t *ptr, const int32_t *col, const double *val,
                     const amg_params *prm, amg_handle *out);

/* Solve A x = f to |f - A x| <= tol |f| (recurrence residual; R14) with
 * the handle's Krylov method (params.solver: CG, BiCGStab, GMRES(m) or IDR(s)), at
 * most maxiter iterations.  f, x: DEVICE pointers; x holds the initial guess on
 * entry and the solution on return.  f = 0 gives x = 0, 0 iterations.  *iters =
 * loop trips (CG, BiCGStab), Arnoldi steps (GMRES) or preconditioned products
 * (IDR(s)); *rel_resid = true |f - A x|/|f| recomputed at exit.  Returns AMG_OK,
 * AMG_NOT_CONVERGED or AMG_BREAKDOWN (outputs filled in all three cases) or an
 * error.  GMRES and IDR(s) need a single-GPU handle.  Synchronous.  Cite:
 * PAPER.md:141-143, 209-215. */
amg_status amg_solve(amg_handle h, const double *f, double *x, double tol, int32_t maxiter,
                     int32_t *iters, double *rel_resid);

/* Length of the f / x vectors that amg_solve* take on this handle: n on a
 * single-GPU or virtual-rank handle, this rank's row count on an NCCL rank. */
amg_status amg_vector_length(amg_handle h, int64_t *n);

/* Same as amg_solve with HOST buffers (the end-to-end path): copies f (and the
 * initial guess x0, unless x0 is NULL = zero guess) to the device, solves, and
 * copies the solution into x, all inside the call.  x0 may equal x. */
amg_status amg_solve_host(amg_handle h, const double *f, const double *x0, double *x, double tol,
                          int32_t maxiter, int32_t *iters, double *rel_resid);

/* A sequence of k independent solves with HOST buffers (the end-to-end path for a
 * stream of right-hand sides; the hierarchy is reused for many right-hand sides,
 * PAPER.md:156-159): system j solves A x_j = f_j from a zero initial guess, f[j]
 * and x[j] are host pointers of n_local doubles (entries may repeat: the same
 * buffer is copied again for every system).  The copy of f[j+1] to the device
 * and of x[j-1] back to the host run on a copy stream while system j is solved
 * (double-buffered device vectors), so with PINNED host buffers the transfers
 * overlap the solves; pageable buffers still give correct results.  iters[j],
 * rel_resid[j] as amg_solve; vcycles (may be NULL): preconditioner applications
 * per system.  Returns the first non-OK status of the k solves (all k are run
 * unless a CUDA error stops the sequence); amg_solve_stats describes the last. */
amg_status amg_solve_host_stream(amg_handle h, int32_t k, const double *const *f, double *const *x, double tol,
                                 int32_t maxiter, int32_t *iters, double *rel_resid, int32_t *vcycles);

/* Batched solve of A X = F for k right-hand sides (1 <= k <= 8) with one pass over
 * the hierarchy per iteration serving every column (the hierarchy is reused for
 * many right-hand sides).  F, X: DEVICE,
 * column-major, column j at F + j*ldf / X + j*ldx (ld >= n); X holds the initial
 * guesses on entry and the solutions on return.  Every column runs its own CG
 * (own scalars, convergence test and iteration count, identical in exact
 * arithmetic to k separate amg_solve calls).  iters[k], rel_resid[k] (true
 * residuals) are outputs; the status is the worst over the columns.  CG on
 * single-GPU handles only.  Synchronous. */
amg_status amg_solve_batched(amg_handle h, int32_t k, const double *F, int64_t ldf, double *X, int64_t ldx,
                             double tol, int32_t maxiter, int32_t *iters, double *rel_resid);

/* z = M r: one V-cycle from a zero initial guess.  r, z:
 * DEVICE pointers (length n, distinct).  Asynchronous on the handle stream. */
amg_status amg_precond_apply(amg_handle h, const double *r, double *z);

/* Issue subsequent work on `stream` (a cudaStream_t of the handle's device). */
amg_status amg_set_stream(amg_handle h, void *stream);

/* Profile mode: time the kernel classes in `mask` (bit c = class AMG_PROF_c;
 * 0 = off [default]) with CUDA events during amg_solve* -- event-record nodes
 * inside the iteration graph, so the timed solve is the production path.
 * Results: amg_solve_stats.prof_ms / prof_bytes / prof_launches. */
amg_status amg_set_profile(amg_handle h, int32_t mask);

amg_status amg_level_count(amg_handle h, int32_t *nlevels);
amg_status amg_level_info_get(amg_handle h, int32_t level, amg_level_info *out);
/* Copy the host-side hierarchy data of `level` into caller buffers. */
amg_status amg_export_level(amg_handle h, int32_t level, const amg_level_export *out);
amg_status amg_solve_stats_get(amg_handle h, amg_solve_stats *out);

/* TEST HOOK: one device operation of level `level` on DEVICE vectors (async):
 *   AMG_OP_SPMV_A   y = A_l x           AMG_OP_SPMV_P  y = P_l x   AMG_OP_SPMV_R  y = R_l x
 *   AMG_OP_RESIDUAL y = f - A_l x       AMG_OP_RELAX   y = S_l(A_l, f, x) (one smoother call)
 *   AMG_OP_COARSE   y = A_L^-1 f (coarsest level)     AMG_OP_VCYCLE y = V-cycle from level l, f, x = 0 */
enum { AMG_OP_SPMV_A = 0, AMG_OP_SPMV_P = 1, AMG_OP_SPMV_R = 2, AMG_OP_RESIDUAL = 3,
       AMG_OP_RELAX = 4, AMG_OP_COARSE = 5, AMG_OP_VCYCLE = 6 };
amg_status amg_level_op(amg_handle h, int32_t level, int32_t op, const double *x, const double *f,
                        double *y);

/* TEST HOOK: one launch of a FUSED production kernel of the V-cycle / CG
 * iteration on level `level` (< coarsest), with the same op struct and kernel
 * template the solve runs, on caller DEVICE vectors (natural order; a reordered
 * store permutes them in and out).  Operand roles per op (c = level + 1):
 *   AMG_OP_RES0         out0 = in0 - A (m o in0)           a1, zero-start sweep + residual
 *                                                          (SPAI-0/Jacobi; Alg. 2)
 *   AMG_OP_RES0_MF      out0 = in0 - A in1  (in1 = m o f)  a1 with the precomputed m o f
 *   AMG_OP_RESTRICT_MF  out0 = R in0 (level c), out1 = m_c o out0   a2
 *   AMG_OP_PROL0        out0 = m o in1 + P in0 (in0 on level c)      a5
 *   AMG_OP_PROL0_MF     out0 = in1 + P in0  (in1 = m o f)
 *   AMG_OP_PROL_ADD     out0 += P in0       (out0 read and written)
 *   AMG_OP_RELAX_RHO    out0 = in0 + m o (in1 - A in0), dot = (in1, out0)   a6
 *   AMG_OP_CHEB_STEP    Chebyshev step k = (int)scalar of one smoother call: r = in1 - A in0
 *                       (/ a_ii when scaled), out1 = alpha_k r + beta_k out1 (k = 0: alpha_0 r;
 *                       out1 read and written), out0 = in0 + out1, dot = (in1, out0)
 *   AMG_OP_CG_DIR       (level 0) out0 = in0 + scalar * in1, out1 = A out0, dot = (out0, out1)
 *                       a7 (CG direction)
 *   AMG_OP_CG_UPDATE    (level 0, SPAI-0/Jacobi) out0 += scalar in0, out1 -= scalar in1,
 *                       out2 = m o out1, dot = |out1| (CG update + norm)
 * Synchronous (dot is a host output).  AMG_E_INVALID_ARG for an op the handle's
 * smoother does not use or a missing operand; single-GPU handles only. */
enum { AMG_OP_RES0 = 7, AMG_OP_RES0_MF = 8, AMG_OP_RESTRICT_MF = 9, AMG_OP_PROL0 = 10, AMG_OP_PROL0_MF = 11,
       AMG_OP_PROL_ADD = 12, AMG_OP_RELAX_RHO = 13, AMG_OP_CHEB_STEP = 14, AMG_OP_CG_DIR = 15,
       AMG_OP_CG_UPDATE = 16 };
typedef struct {
    const double *in0, *in1;
    double *out0, *out1, *out2;
    double scalar;   /* beta (CG_DIR), alpha (CG_UPDATE), step k (CHEB_STEP) */
    double dot;      /* out: the fused reduction */
} amg_level_op_args;
amg_status amg_level_op_ex(amg_handle h, int32_t level, int32_t op, amg_level_op_args *args);

/* ---------------------------------------------------------------- multi-GPU
 * Row partition of the hierarchy over `nranks` ranks (the paper
 * runs the method over MPI processes).  The host setup is
 * global and deterministic (the hierarchy is the single-GPU one at every rank
 * count); each rank keeps its contiguous row slice of every level (coarse rows
 * follow their aggregate roots) with ghost columns renumbered after the local
 * ones, and levels with fewer than gather_below rows are replicated on every rank.
 *   rank >= 0: one process per GPU; halo exchange / all-reduce / all-gather run
 *              over NCCL (loaded with dlopen) created from nccl_id, which rank 0
 *              obtains with amg_nccl_unique_id and broadcasts.  Scattered setup:
 *              the communicator is created first, then rank 0 alone builds the
 *              hierarchy of the global matrix it was given and sends every other
 *              rank its part over NCCL; ranks > 0 pass only n (ptr, col, val may
 *              be NULL and are ignored) and never hold the global matrix.  A setup
 *              error on rank 0 is returned on every rank.  amg_solve then takes
 *              this rank's slice of f and x (rows row_starts[rank] ..
 *              row_starts[rank+1]-1, see amg_dist_info).  Every wait on a peer is
 *              bounded by AMGB_NCCL_TIMEOUT_S (AMG_E_NCCL).
 *   rank == -1: every rank lives in this process on one GPU ("virtual ranks":
 *              transport = device copies).  amg_solve / amg_precond_apply take
 *              the GLOBAL f and x.  Used to test the partitioned path on one GPU.
 * Results equal the single-GPU solve up to the order of the dot-product sums
 * (row sums keep the global column order). */
typedef struct {
    int32_t nranks;         /* ranks of the partition */
    int32_t rank;           /* >= 0: NCCL rank of this process; -1: all ranks here */
    int64_t gather_below;   /* replicate levels with fewer rows [0 -> 16384 * nranks] */
    uint8_t nccl_id[128];   /* ncclUniqueId from amg_nccl_unique_id (rank >= 0) */
} amg_dist;

/* Test/export hook of one rank's level (host buffers sized by amg_dist_level_info). */
typedef struct {
    int64_t *A_ptr; int32_t *A_col; double *A_val;   /* local rows, local|ghost columns */
    int64_t *P_ptr; int32_t *P_col; double *P_val;   /* local fine rows */
    int64_t *R_ptr; int32_t *R_col; double *R_val;   /* local coarse rows */
    int64_t *ghost_global;                           /* global index of each ghost */
    int32_t *recv_peer; int64_t *recv_off, *recv_cnt;/* ghost-region segments by owner */
    int32_t *send_peer; int64_t *send_off, *send_cnt;/* packed send-buffer segments */
    int32_t *send_idx;                               /* local indices to send, by peer */
} amg_dist_level_export;

/* Write a fresh NCCL unique id (call on rank 0 only).  AMG_E_CUDA if NCCL is unavailable. */
amg_status amg_nccl_unique_id(uint8_t id[128]);
/* Distributed setup (see above); same errors as amg_setup, plus AMG_E_INVALID_ARG
 * for a hierarchy that cannot be distributed (a single level) and AMG_E_NCCL.
 * amg_export_level works on rank 0 only (the other ranks hold their parts). */
amg_status amg_setup_dist(int64_t n, const int64_t *ptr, const int32_t *col, const double *val,
                          const amg_params *prm, const amg_dist *dist, amg_handle *out);
/* nranks, first replicated level and the level-0 row starts (nranks+1 entries, may be NULL). */
amg_status amg_dist_info(amg_handle h, int32_t *nranks, int32_t *first_replicated, int64_t *row_starts);
/* out[0..11] = row0, row1, ghosts, nnz(A), nnz(P), nnz(R), crow0, crow1, replicated,
 *              send entries, recv peers, send peers of (rank, level);
 * out[12..17] = interior row range [ib0, ib1) of the split A, P and R passes (rows
 *              without ghost columns, overlapped with the halo exchange),
 *              -1 where the pass is not split (host-only handles, replicated levels). */
amg_status amg_dist_level_info(amg_handle h, int32_t rank, int32_t level, int64_t out[18]);
amg_status amg_dist_export(amg_handle h, int32_t rank, int32_t level, const amg_dist_level_export *out);
/* Self-test of the NCCL transport on a 1-rank communicator of `device`: grouped
 * send/recv to self, all-reduce and broadcast, directly and replayed from a
 * captured CUDA graph, with the same calls the executor makes.  AMG_OK or an error. */
amg_status amg_nccl_selftest(int32_t device);

/* Self-test of the host shared-memory TEST transport (AMGB_TRANSPORT=shm: ranks
 * of one node that share a GPU run the one-process-per-rank path through host
 * shared memory instead of NCCL; every transfer synchronous on the host, no
 * kernel waits on another rank).  Call from `nranks` processes with the same id;
 * three personalised all-to-all rounds are checked.  AMG_OK or AMG_E_NCCL.
 * Needs no GPU. */
amg_status amg_shm_selftest(const uint8_t id[128], int32_t rank, int32_t nranks);

void amg_destroy(amg_handle h);
const char *amg_last_error(void);
/* Library build identification string (compile flags, arch). */
const char *amg_version(void);

#ifdef __cplusplus
}
#endif
#endif /* AMGB_H */
