/*
 * oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, fp64 CPU implementation of the smoothed-aggregation AMG method of
 * D. Demidov, "AMGCL: an efficient, flexible, and extensible algebraic multigrid
 * implementation" (arXiv 1811.05704), written from the paper and the
 * readings fixed in SURVEY.md §8(c) / DESIGN.md §3.  It exists only to check the
 * product library (paper_1811_05704_b200/, include/amgb.h).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
 * load it.  It shares no code, header, table or helper with the product library.
 *
 * Citations: "PAPER.md:L" = line L of the paper text, "SPEC.md:L" = line L of the
 * CPU-program spec written from it, "§8c Lk" = reading k of SURVEY.md §8(c)-3.
 *
 * Conventions: CSR with int64 row pointers, int32 column indices (strictly
 * increasing within a row), fp64 values.  Every function returns 0 on success and
 * a negative code on error (see OR_E_*); or_last_error() gives the message.
 */
#ifndef AMG_ORACLE_H
#define AMG_ORACLE_H
#include <stdint.h>

#define OR_OK 0
#define OR_NOT_CONVERGED 1
#define OR_BREAKDOWN 2
#define OR_E_INVALID -1
#define OR_E_BAD_CSR -2
#define OR_E_ZERO_DIAG -3
#define OR_E_SINGULAR -4
#define OR_E_TOO_LARGE -5
#define OR_E_NOMEM -6

typedef struct {
    int64_t nrows, ncols, nnz;
    int64_t *ptr; /* nrows+1 */
    int32_t *col; /* nnz */
    double *val;  /* nnz */
} or_csr;

/* Parameters (defaults: SPEC.md:181, 264, 337; §8c L1-L15). */
typedef struct {
    double eps_strong;    /* 0.08 on the finest level */
    double eps_decay;     /* 0.5: eps on level l+1 = eps on level l * eps_decay */
    double p_omega;       /* 2/3  */
    int32_t smoothed;     /* 1 = smoothed aggregation, 0 = plain aggregation */
    int32_t relax;        /* 0 = spai0, 1 = damped jacobi, 2 = chebyshev */
    double jacobi_omega;  /* 0.72 */
    int32_t cheb_degree;  /* 5 */
    double cheb_lower;    /* 1/30 */
    int32_t cheb_scaled;  /* 1 = polynomial in D^-1 A */
    int32_t npre, npost;  /* 1, 1 */
    int64_t coarse_enough;/* 3000 */
    int32_t max_levels;   /* 30 */
    int64_t dense_max;    /* 20000 */
} or_params;

const char *or_last_error(void);
void or_params_default(or_params *p);

/* ---- single operations (each exported for the pin tests) ---- */
int or_spmv(int64_t nrows, const int64_t *ptr, const int32_t *col, const double *val,
            const double *x, double *y);
int or_strength(int64_t n, const int64_t *ptr, const int32_t *col, const double *val,
                double eps, uint8_t *strong /* nnz; diagonal entries get 0 */);
int or_aggregate(int64_t n, const int64_t *ptr, const int32_t *col, const double *val,
                 const uint8_t *strong, int32_t *id, int64_t *count);
/* or_csr objects returned by the functions below are owned by the caller: or_csr_free. */
or_csr *or_tentative_p(int64_t n, const int32_t *id, int64_t count);
or_csr *or_smooth_p(int64_t n, const int64_t *ptr, const int32_t *col, const double *val,
                    const uint8_t *strong, const int32_t *id, int64_t count, double omega);
or_csr *or_transpose(const or_csr *A);
or_csr *or_spgemm(const or_csr *A, const or_csr *B);
or_csr *or_csr_wrap_copy(int64_t nrows, int64_t ncols, const int64_t *ptr, const int32_t *col,
                         const double *val);
void or_csr_dims(const or_csr *A, int64_t out[3]);
void or_csr_copy_out(const or_csr *A, int64_t *ptr, int32_t *col, double *val);
void or_csr_free(or_csr *A);

int or_lu_factor(int64_t n, double *a /* row-major n*n, overwritten */, int32_t *piv);
int or_lu_solve(int64_t n, const double *lu, const int32_t *piv, const double *b, double *x);

/* ---- hierarchy (Algorithm 1) ---- */
typedef struct or_hier or_hier;
int or_setup(int64_t n, const int64_t *ptr, const int32_t *col, const double *val,
             const or_params *prm, or_hier **out);
void or_free(or_hier *h);
int or_nlevels(const or_hier *h);
/* out[0]=rows, out[1]=nnz(A), out[2]=nnz(P) (0 on coarsest), out[3]=cols of P
 * (=rows of next level), out[4]=aggregate count, out[5]=is_coarsest */
int or_level_info(const or_hier *h, int l, int64_t out[6]);
/* which: 0=A, 1=P, 2=R */
int or_level_matrix(const or_hier *h, int l, int which, int64_t *ptr, int32_t *col, double *val);
int or_level_aggregates(const or_hier *h, int l, int32_t *id);
/* SPAI-0 / Jacobi diagonal m (n values) or, for Chebyshev, out[0..3]=lmax,lmin,d,c */
int or_level_smoother(const or_hier *h, int l, double *out);

/* ---- solve phase ---- */
/* One V-cycle of Algorithm 2 on level l with x as the initial guess. */
int or_vcycle(const or_hier *h, int l, const double *f, double *x);
/* Preconditioner z = M r: one V-cycle from zero. */
int or_precond(const or_hier *h, const double *r, double *z);
/* One relaxation call S(A_l, f, x) (Algorithm 2 lines "S_i(A_i, f_i, u_i)"). */
int or_relax(const or_hier *h, int l, const double *f, double *x);
/* Step k of the Chebyshev smoother's recurrence (the body of or_relax's loop):
 * x, p updated in place; *alpha = alpha_{k-1} in, alpha_k out (ignored for k = 0). */
int or_cheb_step(const or_hier *h, int l, int k, const double *f, double *x, double *p, double *alpha);
/* Preconditioned CG / BiCGStab.  x: initial guess in,
 * solution out.  precond = 0 runs the unpreconditioned method (M = I) for pins. */
int or_cg(const or_hier *h, int64_t n, const int64_t *ptr, const int32_t *col, const double *val,
          int precond, const double *f, double *x, double tol, int32_t maxiter,
          int32_t *iters, double *rel_resid, double *resid_hist /* maxiter+1 or NULL */);
int or_bicgstab(const or_hier *h, int64_t n, const int64_t *ptr, const int32_t *col,
                const double *val, int precond, const double *f, double *x, double tol,
                int32_t maxiter, int32_t *iters, double *rel_resid, int32_t *vcycles);
/* Restarted right-preconditioned GMRES(m) (Saad 2003 Alg. 9.5 with
 * modified Gram-Schmidt and Givens rotations).  iters = Arnoldi steps; vcycles
 * counts preconditioner applications (one per step + one per restart cycle for
 * x += M (V y)).  resid_hist (maxiter+1 or NULL): estimated residual norms. */
int or_gmres(const or_hier *h, int64_t n, const int64_t *ptr, const int32_t *col, const double *val,
             int precond, int32_t m, const double *f, double *x, double tol, int32_t maxiter,
             int32_t *iters, double *rel_resid, int32_t *vcycles, double *resid_hist);

/* IDR(s) shadow space (column-major n x s): counter-based splitmix64 entries in
 * [-1, 1), orthonormalised by modified Gram-Schmidt. */
void or_idrs_shadow(int64_t n, int32_t s, double *P);
/* Right-preconditioned IDR(s) with bi-orthogonalisation (van Gijzen &
 * Sonneveld 2011, Alg. 913).  kappa: "angle" omega strategy (0.7; 0 = minimal
 * residual).  P: shadow space or NULL (or_idrs_shadow).  iters = preconditioned
 * matrix-vector products; resid_hist (maxiter+1 or NULL): |r| after each. */
int or_idrs(const or_hier *h, int64_t n, const int64_t *ptr, const int32_t *col, const double *val,
            int precond, int32_t s, double kappa, const double *P, const double *f, double *x, double tol,
            int32_t maxiter, int32_t *iters, double *rel_resid, int32_t *vcycles, double *resid_hist);

#endif
