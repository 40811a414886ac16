/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * A plain, slow, obviously-correct fp64 CPU implementation of the method of
 * arXiv 1811.05704 (AMGCL): smoothed-aggregation setup (Algorithm 1,
 * PAPER.md:95-107), the V-cycle (Algorithm 2) used as a
 * preconditioner for CG and BiCGStab.
 * Component details the paper only names are taken from SPEC.md and the readings
 * of SURVEY.md §8(c)-3 (cited as "§8c Lk"); DESIGN.md §3 lists every reading.
 *
 * Rules followed here: one loop per definition, no blocking or fusion, every
 * accumulation in ascending index order, compiled with -ffp-contract=off and no
 * fast-math.  OpenMP is used only on row loops of matrix-vector products, where
 * every row's arithmetic is unchanged by the thread count.  Dot products are
 * plain serial sums.
 *
 * Parity status per function (DESIGN.md §4 has the list of pins):
 *   every function below is pinned by tests/test_oracle_*.py except the
 *   hierarchy sizes and iteration counts at the benchmark sizes, which the
 *   paper does not print: "parity unpinned" for those two quantities
 *   (bounds only).
 */
#include "oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static char g_err[512];

static void set_err(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
}

const char *or_last_error(void) { return g_err; }

/* Defaults: SPEC.md:181 (eps 0.08, omega 2/3), SPEC.md:264 (jacobi 0.72, degree 5,
 * lower 1/30), SPEC.md:337 (npre = npost = 1, coarse_enough 3000, max_levels 30),
 * §8c L9 (dense_max 20000), §8c L15 (Chebyshev scaled by D^-1). */
void or_params_default(or_params *p) {
    p->eps_strong = 0.08;
    p->eps_decay = 0.5;
    p->p_omega = 2.0 / 3.0;
    p->smoothed = 1;
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
}

/* ------------------------------------------------------------------------- */
/* CSR helpers                                                               */
/* ------------------------------------------------------------------------- */

static or_csr *csr_alloc(int64_t nrows, int64_t ncols, int64_t nnz) {
    or_csr *A = (or_csr *)calloc(1, sizeof(or_csr));
    if (!A) return NULL;
    A->nrows = nrows;
    A->ncols = ncols;
    A->nnz = nnz;
    A->ptr = (int64_t *)calloc((size_t)nrows + 1, sizeof(int64_t));
    A->col = (int32_t *)malloc((size_t)(nnz > 0 ? nnz : 1) * sizeof(int32_t));
    A->val = (double *)malloc((size_t)(nnz > 0 ? nnz : 1) * sizeof(double));
    if (!A->ptr || !A->col || !A->val) {
        free(A->ptr);
        free(A->col);
        free(A->val);
        free(A);
        return NULL;
    }
    return A;
}

void or_csr_free(or_csr *A) {
    if (!A) return;
    free(A->ptr);
    free(A->col);
    free(A->val);
    free(A);
}

or_csr *or_csr_wrap_copy(int64_t nrows, int64_t ncols, const int64_t *ptr, const int32_t *col,
                         const double *val) {
    or_csr *A = csr_alloc(nrows, ncols, ptr[nrows]);
    if (!A) return NULL;
    memcpy(A->ptr, ptr, (size_t)(nrows + 1) * sizeof(int64_t));
    memcpy(A->col, col, (size_t)ptr[nrows] * sizeof(int32_t));
    memcpy(A->val, val, (size_t)ptr[nrows] * sizeof(double));
    return A;
}

void or_csr_dims(const or_csr *A, int64_t out[3]) {
    out[0] = A->nrows;
    out[1] = A->ncols;
    out[2] = A->nnz;
}

void or_csr_copy_out(const or_csr *A, int64_t *ptr, int32_t *col, double *val) {
    memcpy(ptr, A->ptr, (size_t)(A->nrows + 1) * sizeof(int64_t));
    memcpy(col, A->col, (size_t)A->nnz * sizeof(int32_t));
    memcpy(val, A->val, (size_t)A->nnz * sizeof(double));
}

/* CSR invariants of SPEC.md:25-27: ptr[0] = 0, non-decreasing, columns strictly
 * increasing inside a row and within [0, ncols).  Empty rows are legal. */
static int check_csr(int64_t nrows, int64_t ncols, const int64_t *ptr, const int32_t *col) {
    if (ptr[0] != 0) {
        set_err("ptr[0] = %lld, expected 0", (long long)ptr[0]);
        return OR_E_BAD_CSR;
    }
    for (int64_t i = 0; i < nrows; i++) {
        if (ptr[i + 1] < ptr[i]) {
            set_err("row %lld: ptr decreases", (long long)i);
            return OR_E_BAD_CSR;
        }
        for (int64_t k = ptr[i]; k < ptr[i + 1]; k++) {
            if (col[k] < 0 || col[k] >= ncols) {
                set_err("row %lld: column %d out of range", (long long)i, col[k]);
                return OR_E_BAD_CSR;
            }
            if (k > ptr[i] && col[k] <= col[k - 1]) {
                set_err("row %lld: columns not strictly increasing", (long long)i);
                return OR_E_BAD_CSR;
            }
        }
    }
    return OR_OK;
}

/* Diagonal entry a_ii; returns 0.0 if the row has none. */
static double diag_of(const int64_t *ptr, const int32_t *col, const double *val, int64_t i) {
    for (int64_t k = ptr[i]; k < ptr[i + 1]; k++)
        if (col[k] == i) return val[k];
    return 0.0;
}

/* y = A x, each y_i = sum_j a_ij x_j accumulated in ascending j. */
int or_spmv(int64_t nrows, const int64_t *ptr, const int32_t *col, const double *val,
            const double *x, double *y) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < nrows; i++) {
        double s = 0.0;
        for (int64_t k = ptr[i]; k < ptr[i + 1]; k++) s += val[k] * x[col[k]];
        y[i] = s;
    }
    return OR_OK;
}

static void spmv_csr(const or_csr *A, const double *x, double *y) {
    or_spmv(A->nrows, A->ptr, A->col, A->val, x, y);
}

/* r = f - A x. */
static void residual(const or_csr *A, const double *f, const double *x, double *r) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < A->nrows; i++) {
        double s = 0.0;
        for (int64_t k = A->ptr[i]; k < A->ptr[i + 1]; k++) s += A->val[k] * x[A->col[k]];
        r[i] = f[i] - s;
    }
}

/* (a, b): plain serial sum in ascending i. */
static double dot(int64_t n, const double *a, const double *b) {
    double s = 0.0;
    for (int64_t i = 0; i < n; i++) s += a[i] * b[i];
    return s;
}

/* ------------------------------------------------------------------------- */
/* Setup components                      */
/* ------------------------------------------------------------------------- */

/* Strength of connection, §8c L1 / SPEC.md:189: for j != i,
 *   strong(i,j)  <=>  a_ij * a_ij > (eps^2 * a_ii) * a_jj     (strict >)
 * A non-positive (or missing) diagonal is an error. */
int or_strength(int64_t n, const int64_t *ptr, const int32_t *col, const double *val,
                double eps, uint8_t *strong) {
    double *d = (double *)malloc((size_t)(n > 0 ? n : 1) * sizeof(double));
    if (!d) return OR_E_NOMEM;
    for (int64_t i = 0; i < n; i++) {
        d[i] = diag_of(ptr, col, val, i);
        if (!(d[i] > 0.0)) {
            set_err("row %lld: diagonal %g is not positive", (long long)i, d[i]);
            free(d);
            return OR_E_ZERO_DIAG;
        }
    }
    double eps2 = eps * eps;
    for (int64_t i = 0; i < n; i++) {
        for (int64_t k = ptr[i]; k < ptr[i + 1]; k++) {
            int32_t j = col[k];
            if (j == i) {
                strong[k] = 0;
            } else {
                double a = val[k];
                strong[k] = (a * a > (eps2 * d[i]) * d[j]) ? 1 : 0;
            }
        }
    }
    free(d);
    return OR_OK;
}

/* Greedy aggregation (SPEC.md:240 with §8c L2):
 * Phase 1: scan rows ascending; an unaggregated row whose strong neighbours are
 *          all unaggregated becomes a root and takes its strong neighbourhood.
 *          (A row with no strong neighbour becomes a singleton root.)
 * Phase 2: every row still unaggregated joins, via a snapshot of Phase 1, the
 *          aggregate of its strongest aggregated strong neighbour (max |a_ij|,
 *          ties -> lowest j).
 * Phase 3: rows still unaggregated become singletons (never happens; the count of
 *          such rows is reported through the error string for the tests). */
int or_aggregate(int64_t n, const int64_t *ptr, const int32_t *col, const double *val,
                 const uint8_t *strong, int32_t *id, int64_t *count_out) {
    const int32_t UNAGG = -1;
    int64_t count = 0;
    for (int64_t i = 0; i < n; i++) id[i] = UNAGG;

    /* Phase 1 */
    for (int64_t i = 0; i < n; i++) {
        if (id[i] != UNAGG) continue;
        int any_taken = 0;
        for (int64_t k = ptr[i]; k < ptr[i + 1]; k++)
            if (strong[k] && id[col[k]] != UNAGG) any_taken = 1;
        if (any_taken) continue;
        id[i] = (int32_t)count;
        for (int64_t k = ptr[i]; k < ptr[i + 1]; k++)
            if (strong[k]) id[col[k]] = (int32_t)count;
        count += 1;
    }

    /* Phase 2 (reads the Phase-1 snapshot) */
    int32_t *snap = (int32_t *)malloc((size_t)(n > 0 ? n : 1) * sizeof(int32_t));
    if (!snap) return OR_E_NOMEM;
    memcpy(snap, id, (size_t)n * sizeof(int32_t));
    for (int64_t i = 0; i < n; i++) {
        if (snap[i] != UNAGG) continue;
        int64_t best = -1;
        double best_v = -1.0;
        for (int64_t k = ptr[i]; k < ptr[i + 1]; k++) {
            if (!strong[k] || snap[col[k]] == UNAGG) continue;
            double v = fabs(val[k]);
            if (v > best_v) {
                best_v = v;
                best = col[k];
            }
        }
        if (best >= 0) id[i] = snap[best];
    }
    free(snap);

    /* Phase 3 */
    int64_t phase3 = 0;
    for (int64_t i = 0; i < n; i++) {
        if (id[i] == UNAGG) {
            id[i] = (int32_t)count;
            count += 1;
            phase3 += 1;
        }
    }
    if (phase3) set_err("aggregate: phase 3 created %lld singletons", (long long)phase3);
    *count_out = count;
    return OR_OK;
}

/* Tentative prolongation (§8c L3): Pt[i, id[i]] = 1. */
or_csr *or_tentative_p(int64_t n, const int32_t *id, int64_t count) {
    or_csr *P = csr_alloc(n, count, n);
    if (!P) return NULL;
    for (int64_t i = 0; i < n; i++) {
        P->ptr[i + 1] = i + 1;
        P->col[i] = id[i];
        P->val[i] = 1.0;
    }
    return P;
}

static int cmp_i32(const void *a, const void *b) {
    int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
    return (x > y) - (x < y);
}

/* Smoothed prolongation (§8c L4-L6):
 *   P = (I - omega D_F^-1 A_F) Pt
 * with A_F the filtered matrix: strong off-diagonals kept, weak off-diagonals
 * lumped onto the diagonal:  D_F(i) = a_ii + sum_{j != i, weak} a_ij (ascending j).
 * Row i:  P(i,J) = sum_{k in {i} u S_i, id[k] = J} w_ik  (ascending k), with
 *   w_ii = 1 - omega,   w_ik = -(omega / D_F(i)) * a_ik.
 * The pattern is { id[k] : k in {i} u S_i }, structural (zeros kept). */
or_csr *or_smooth_p(int64_t n, const int64_t *ptr, const int32_t *col, const double *val,
                    const uint8_t *strong, const int32_t *id, int64_t count, double omega) {
    /* upper bound on nnz: one entry per member of {i} u S_i */
    int64_t cap = 0;
    for (int64_t i = 0; i < n; i++) {
        cap += 1;
        for (int64_t k = ptr[i]; k < ptr[i + 1]; k++) cap += strong[k];
    }
    or_csr *P = csr_alloc(n, count, cap);
    if (!P) return NULL;
    int32_t *cols = (int32_t *)malloc((size_t)(cap > 0 ? cap : 1) * sizeof(int32_t));
    int64_t pos = 0;
    for (int64_t i = 0; i < n; i++) {
        double dfi = 0.0, aii = 0.0;
        for (int64_t k = ptr[i]; k < ptr[i + 1]; k++)
            if (col[k] == i) aii = val[k];
        dfi = aii;
        for (int64_t k = ptr[i]; k < ptr[i + 1]; k++)
            if (col[k] != i && !strong[k]) dfi += val[k];
        double s = omega / dfi;

        /* distinct aggregate ids of {i} u S_i, ascending */
        int64_t nc = 0;
        cols[nc++] = id[i];
        for (int64_t k = ptr[i]; k < ptr[i + 1]; k++)
            if (strong[k]) cols[nc++] = id[col[k]];
        qsort(cols, (size_t)nc, sizeof(int32_t), cmp_i32);
        int64_t m = 0;
        for (int64_t t = 0; t < nc; t++)
            if (m == 0 || cols[t] != cols[m - 1]) cols[m++] = cols[t];

        for (int64_t t = 0; t < m; t++) {
            int32_t J = cols[t];
            double acc = 0.0;
            for (int64_t k = ptr[i]; k < ptr[i + 1]; k++) {
                int32_t j = col[k];
                if (j == i) {
                    if (id[i] == J) acc += 1.0 - omega;
                } else if (strong[k] && id[j] == J) {
                    acc += -(s * val[k]);
                }
            }
            /* a row without a stored diagonal still owns w_ii (only possible
             * when a_ii is absent, which strength() rejects) */
            P->col[pos] = J;
            P->val[pos] = acc;
            pos++;
        }
        P->ptr[i + 1] = pos;
    }
    free(cols);
    P->nnz = pos;
    return P;
}

/* Transpose (R = P^T, §8c L8); rows of the result list their
 * columns in ascending order. */
or_csr *or_transpose(const or_csr *A) {
    or_csr *T = csr_alloc(A->ncols, A->nrows, A->nnz);
    if (!T) return NULL;
    for (int64_t k = 0; k < A->nnz; k++) T->ptr[A->col[k] + 1] += 1;
    for (int64_t j = 0; j < A->ncols; j++) T->ptr[j + 1] += T->ptr[j];
    int64_t *next = (int64_t *)malloc((size_t)(A->ncols > 0 ? A->ncols : 1) * sizeof(int64_t));
    for (int64_t j = 0; j < A->ncols; j++) next[j] = T->ptr[j];
    for (int64_t i = 0; i < A->nrows; i++) {
        for (int64_t k = A->ptr[i]; k < A->ptr[i + 1]; k++) {
            int64_t dst = next[A->col[k]]++;
            T->col[dst] = (int32_t)i;
            T->val[dst] = A->val[k];
        }
    }
    free(next);
    return T;
}

/* C = A B, row by row (§8c L7): C(i,J) = sum_k A(i,k) B(k,J)
 * accumulated in ascending k; the pattern is the structural product pattern
 * (cancellation zeros kept), columns ascending. */
or_csr *or_spgemm(const or_csr *A, const or_csr *B) {
    int64_t cap = 1024;
    int64_t nnz = 0;
    int64_t *ptr = (int64_t *)calloc((size_t)A->nrows + 1, sizeof(int64_t));
    int32_t *col = (int32_t *)malloc((size_t)cap * sizeof(int32_t));
    double *val = (double *)malloc((size_t)cap * sizeof(double));
    double *acc = (double *)malloc((size_t)(B->ncols > 0 ? B->ncols : 1) * sizeof(double));
    int64_t *mark = (int64_t *)malloc((size_t)(B->ncols > 0 ? B->ncols : 1) * sizeof(int64_t));
    int32_t *list = (int32_t *)malloc((size_t)(B->ncols > 0 ? B->ncols : 1) * sizeof(int32_t));
    if (!ptr || !col || !val || !acc || !mark || !list) return NULL;
    for (int64_t j = 0; j < B->ncols; j++) mark[j] = -1;

    for (int64_t i = 0; i < A->nrows; i++) {
        int64_t len = 0;
        for (int64_t ka = A->ptr[i]; ka < A->ptr[i + 1]; ka++) {
            int32_t k = A->col[ka];
            double a = A->val[ka];
            for (int64_t kb = B->ptr[k]; kb < B->ptr[k + 1]; kb++) {
                int32_t J = B->col[kb];
                if (mark[J] != i) {
                    mark[J] = i;
                    acc[J] = 0.0;
                    list[len++] = J;
                }
                acc[J] += a * B->val[kb];
            }
        }
        qsort(list, (size_t)len, sizeof(int32_t), cmp_i32);
        if (nnz + len > cap) {
            while (nnz + len > cap) cap *= 2;
            col = (int32_t *)realloc(col, (size_t)cap * sizeof(int32_t));
            val = (double *)realloc(val, (size_t)cap * sizeof(double));
            if (!col || !val) return NULL;
        }
        for (int64_t t = 0; t < len; t++) {
            col[nnz] = list[t];
            val[nnz] = acc[list[t]];
            nnz++;
        }
        ptr[i + 1] = nnz;
    }
    free(acc);
    free(mark);
    free(list);
    or_csr *C = (or_csr *)calloc(1, sizeof(or_csr));
    C->nrows = A->nrows;
    C->ncols = B->ncols;
    C->nnz = nnz;
    C->ptr = ptr;
    C->col = col;
    C->val = val;
    return C;
}

/* Dense LU with partial pivoting: P A = L U, row-major, L unit
 * lower.  piv[k] = row swapped with k at step k.  A pivot below
 * 1e-14 * max|A| is an error. */
int or_lu_factor(int64_t n, double *a, int32_t *piv) {
    double amax = 0.0;
    for (int64_t i = 0; i < n * n; i++)
        if (fabs(a[i]) > amax) amax = fabs(a[i]);
    for (int64_t k = 0; k < n; k++) {
        int64_t p = k;
        double best = fabs(a[k * n + k]);
        for (int64_t i = k + 1; i < n; i++) {
            if (fabs(a[i * n + k]) > best) {
                best = fabs(a[i * n + k]);
                p = i;
            }
        }
        if (!(best >= 1e-14 * amax) || best == 0.0) {
            set_err("coarse LU: pivot %g at step %lld below 1e-14*max|A|", best, (long long)k);
            return OR_E_SINGULAR;
        }
        piv[k] = (int32_t)p;
        if (p != k) {
            for (int64_t j = 0; j < n; j++) {
                double t = a[k * n + j];
                a[k * n + j] = a[p * n + j];
                a[p * n + j] = t;
            }
        }
        for (int64_t i = k + 1; i < n; i++) {
            double l = a[i * n + k] / a[k * n + k];
            a[i * n + k] = l;
            for (int64_t j = k + 1; j < n; j++) a[i * n + j] -= l * a[k * n + j];
        }
    }
    return OR_OK;
}

int or_lu_solve(int64_t n, const double *lu, const int32_t *piv, const double *b, double *x) {
    for (int64_t i = 0; i < n; i++) x[i] = b[i];
    for (int64_t k = 0; k < n; k++) {
        if (piv[k] != k) {
            double t = x[k];
            x[k] = x[piv[k]];
            x[piv[k]] = t;
        }
    }
    for (int64_t i = 0; i < n; i++) { /* L y = P b */
        double s = x[i];
        for (int64_t j = 0; j < i; j++) s -= lu[i * n + j] * x[j];
        x[i] = s;
    }
    for (int64_t i = n - 1; i >= 0; i--) { /* U x = y */
        double s = x[i];
        for (int64_t j = i + 1; j < n; j++) s -= lu[i * n + j] * x[j];
        x[i] = s / lu[i * n + i];
    }
    return OR_OK;
}

/* ------------------------------------------------------------------------- */
/* Hierarchy: Algorithm 1                                  */
/* ------------------------------------------------------------------------- */

#define OR_MAXL 64

struct or_hier {
    or_params prm;
    int nlev;
    or_csr *A[OR_MAXL], *P[OR_MAXL], *R[OR_MAXL];
    int32_t *agg[OR_MAXL];
    int64_t nagg[OR_MAXL];
    double *m[OR_MAXL];       /* SPAI-0 or Jacobi diagonal */
    double *dinv_src[OR_MAXL];/* a_ii (Chebyshev scaling) */
    double cheb[OR_MAXL][4];  /* lmax, lmin, d, c */
    double *lu;
    int32_t *piv;
    int64_t nL;
};

/* Smoother setup (§8c):
 *   SPAI-0:  m_i = a_ii / sum_j a_ij^2
 *   Jacobi:  m_i = omega_J / a_ii
 *   Chebyshev: lmax = Gershgorin bound of D^-1 A (or of A when unscaled),
 *              lmin = lmax * cheb_lower, d = (lmax+lmin)/2, c = (lmax-lmin)/2. */
static int smoother_setup(or_hier *h, int l) {
    const or_csr *A = h->A[l];
    int64_t n = A->nrows;
    h->dinv_src[l] = (double *)malloc((size_t)(n > 0 ? n : 1) * sizeof(double));
    for (int64_t i = 0; i < n; i++) h->dinv_src[l][i] = diag_of(A->ptr, A->col, A->val, i);
    if (h->prm.relax == 0 || h->prm.relax == 1) {
        h->m[l] = (double *)malloc((size_t)(n > 0 ? n : 1) * sizeof(double));
        for (int64_t i = 0; i < n; i++) {
            double aii = h->dinv_src[l][i];
            if (h->prm.relax == 0) {
                double s2 = 0.0;
                for (int64_t k = A->ptr[i]; k < A->ptr[i + 1]; k++) s2 += A->val[k] * A->val[k];
                h->m[l][i] = aii / s2;
            } else {
                h->m[l][i] = h->prm.jacobi_omega / aii;
            }
        }
    } else {
        double lmax = 0.0;
        for (int64_t i = 0; i < n; i++) {
            double s = 0.0;
            for (int64_t k = A->ptr[i]; k < A->ptr[i + 1]; k++) s += fabs(A->val[k]);
            if (h->prm.cheb_scaled) s = s / fabs(h->dinv_src[l][i]);
            if (s > lmax) lmax = s;
        }
        double lmin = lmax * h->prm.cheb_lower;
        h->cheb[l][0] = lmax;
        h->cheb[l][1] = lmin;
        h->cheb[l][2] = (lmax + lmin) / 2.0;
        h->cheb[l][3] = (lmax - lmin) / 2.0;
    }
    return OR_OK;
}

void or_free(or_hier *h) {
    if (!h) return;
    for (int l = 0; l < h->nlev; l++) {
        if (l > 0) or_csr_free(h->A[l]); /* A[0] is a copy too */
        or_csr_free(h->P[l]);
        or_csr_free(h->R[l]);
        free(h->agg[l]);
        free(h->m[l]);
        free(h->dinv_src[l]);
    }
    if (h->nlev > 0) or_csr_free(h->A[0]);
    free(h->lu);
    free(h->piv);
    free(h);
}

/* Algorithm 1 with the stopping rules of SPEC.md:345, 385 (§8c L9):
 *   while n_l > coarse_enough and l+1 < max_levels:
 *       S = strength(A_l); agg = aggregate(A_l, S)
 *       stop if agg.count == n_l, or if count > 0.95 n_l on this and the previous level
 *       P = smoothed ? smooth(A_l, S, Pt) : Pt;  R = P^T;  A_{l+1} = R (A_l P)
 *   dense LU of A_L. */
int or_setup(int64_t n, const int64_t *ptr, const int32_t *col, const double *val,
             const or_params *prm, or_hier **out) {
    *out = NULL;
    if (n <= 0) {
        set_err("empty matrix");
        return OR_E_INVALID;
    }
    int rc = check_csr(n, n, ptr, col);
    if (rc) return rc;
    or_hier *h = (or_hier *)calloc(1, sizeof(or_hier));
    h->prm = *prm;
    h->A[0] = or_csr_wrap_copy(n, n, ptr, col, val);
    int l = 0;
    int prev_slow = 0;
    double eps_l = prm->eps_strong; /* eps on level l = eps_strong * eps_decay^l (R1) */
    for (;;) {
        or_csr *A = h->A[l];
        if (!(A->nrows > prm->coarse_enough && l + 1 < prm->max_levels)) break;
        uint8_t *S = (uint8_t *)malloc((size_t)(A->nnz > 0 ? A->nnz : 1));
        rc = or_strength(A->nrows, A->ptr, A->col, A->val, eps_l, S);
        if (rc) {
            free(S);
            h->nlev = l + 1;
            or_free(h);
            return rc;
        }
        int32_t *id = (int32_t *)malloc((size_t)A->nrows * sizeof(int32_t));
        int64_t count = 0;
        or_aggregate(A->nrows, A->ptr, A->col, A->val, S, id, &count);
        int slow = count > 0.95 * (double)A->nrows;
        if (count == A->nrows || (slow && prev_slow)) {
            free(S);
            free(id);
            break;
        }
        prev_slow = slow;
        or_csr *P = prm->smoothed
                        ? or_smooth_p(A->nrows, A->ptr, A->col, A->val, S, id, count, prm->p_omega)
                        : or_tentative_p(A->nrows, id, count);
        free(S);
        or_csr *R = or_transpose(P);
        or_csr *AP = or_spgemm(A, P);
        or_csr *Ac = or_spgemm(R, AP);
        or_csr_free(AP);
        h->P[l] = P;
        h->R[l] = R;
        h->agg[l] = id;
        h->nagg[l] = count;
        h->nlev = l + 1; /* so or_free sees the levels built so far */
        smoother_setup(h, l);
        h->A[l + 1] = Ac;
        l += 1;
        eps_l = eps_l * prm->eps_decay;
    }
    h->nlev = l + 1;
    /* coarsest level: smoother data is unused; keep the diagonal for info */
    h->dinv_src[l] = NULL;
    or_csr *AL = h->A[l];
    if (AL->nrows > prm->dense_max) {
        set_err("coarsest level has %lld rows > dense_max", (long long)AL->nrows);
        or_free(h);
        return OR_E_TOO_LARGE;
    }
    h->nL = AL->nrows;
    h->lu = (double *)calloc((size_t)(h->nL * h->nL), sizeof(double));
    h->piv = (int32_t *)malloc((size_t)h->nL * sizeof(int32_t));
    for (int64_t i = 0; i < h->nL; i++)
        for (int64_t k = AL->ptr[i]; k < AL->ptr[i + 1]; k++) h->lu[i * h->nL + AL->col[k]] = AL->val[k];
    rc = or_lu_factor(h->nL, h->lu, h->piv);
    if (rc) {
        or_free(h);
        return rc;
    }
    *out = h;
    return OR_OK;
}

int or_nlevels(const or_hier *h) { return h->nlev; }

int or_level_info(const or_hier *h, int l, int64_t out[6]) {
    if (l < 0 || l >= h->nlev) return OR_E_INVALID;
    int coarsest = (l == h->nlev - 1);
    out[0] = h->A[l]->nrows;
    out[1] = h->A[l]->nnz;
    out[2] = coarsest ? 0 : h->P[l]->nnz;
    out[3] = coarsest ? 0 : h->P[l]->ncols;
    out[4] = coarsest ? 0 : h->nagg[l];
    out[5] = coarsest;
    return OR_OK;
}

int or_level_matrix(const or_hier *h, int l, int which, int64_t *ptr, int32_t *col, double *val) {
    if (l < 0 || l >= h->nlev) return OR_E_INVALID;
    const or_csr *M = which == 0 ? h->A[l] : which == 1 ? h->P[l] : h->R[l];
    if (!M) return OR_E_INVALID;
    or_csr_copy_out(M, ptr, col, val);
    return OR_OK;
}

int or_level_aggregates(const or_hier *h, int l, int32_t *id) {
    if (l < 0 || l >= h->nlev - 1) return OR_E_INVALID;
    memcpy(id, h->agg[l], (size_t)h->A[l]->nrows * sizeof(int32_t));
    return OR_OK;
}

int or_level_smoother(const or_hier *h, int l, double *out) {
    if (l < 0 || l >= h->nlev - 1) return OR_E_INVALID;
    if (h->prm.relax == 2) {
        memcpy(out, h->cheb[l], 4 * sizeof(double));
    } else {
        memcpy(out, h->m[l], (size_t)h->A[l]->nrows * sizeof(double));
    }
    return OR_OK;
}

/* ------------------------------------------------------------------------- */
/* Solve phase                                                               */
/* ------------------------------------------------------------------------- */

/* Relaxation S(A_l, f, x) (Algorithm 2; §8c c-1):
 *   SPAI-0 / Jacobi:  x <- x + m o (f - A x)   (every row from the old x)
 *   Chebyshev (K = cheb_degree, fresh recurrence per call):
 *     for k = 0..K-1:  r = f - A x;  if scaled: r_i = r_i / a_ii
 *        k = 0: alpha = 1/d,                p = alpha r
 *        k = 1: alpha = 2d/(2d^2 - c^2),    beta = alpha d - 1, p = alpha r + beta p
 *        k > 1: alpha = 1/(d - alpha c^2/4), beta = alpha d - 1, p = alpha r + beta p
 *        x = x + p */
/* One step k of the Chebyshev recurrence above (the loop body of or_relax,
 * exported so tests can check the library's single-step kernel row by row):
 * r = f - A x; scaled: r_i = r_i / a_ii; alpha_k from *alpha (= alpha_{k-1} on
 * entry, alpha_k on return); p = alpha r (k = 0) or alpha r + beta p; x = x + p. */
int or_cheb_step(const or_hier *h, int l, int k, const double *f, double *x, double *p, double *alpha) {
    if (l < 0 || l >= h->nlev - 1 || h->prm.relax != 2 || k < 0) {
        set_err("or_cheb_step: not a Chebyshev level / step");
        return OR_E_INVALID;
    }
    const or_csr *A = h->A[l];
    int64_t n = A->nrows;
    double d = h->cheb[l][2], c = h->cheb[l][3];
    double *r = (double *)malloc((size_t)(n > 0 ? n : 1) * sizeof(double));
    residual(A, f, x, r);
    if (h->prm.cheb_scaled)
        for (int64_t i = 0; i < n; i++) r[i] = r[i] / h->dinv_src[l][i];
    if (k == 0) {
        *alpha = 1.0 / d;
        for (int64_t i = 0; i < n; i++) p[i] = *alpha * r[i];
    } else {
        if (k == 1)
            *alpha = 2.0 * d / (2.0 * d * d - c * c);
        else
            *alpha = 1.0 / (d - *alpha * c * c / 4.0);
        double beta = *alpha * d - 1.0;
        for (int64_t i = 0; i < n; i++) p[i] = *alpha * r[i] + beta * p[i];
    }
    for (int64_t i = 0; i < n; i++) x[i] = x[i] + p[i];
    free(r);
    return OR_OK;
}

int or_relax(const or_hier *h, int l, const double *f, double *x) {
    const or_csr *A = h->A[l];
    int64_t n = A->nrows;
    if (h->prm.relax == 0 || h->prm.relax == 1) {
        double *r = (double *)malloc((size_t)(n > 0 ? n : 1) * sizeof(double));
        residual(A, f, x, r);
        for (int64_t i = 0; i < n; i++) x[i] = x[i] + h->m[l][i] * r[i];
        free(r);
    } else {
        double *p = (double *)malloc((size_t)(n > 0 ? n : 1) * sizeof(double));
        double alpha = 0.0;
        for (int k = 0; k < h->prm.cheb_degree; k++) or_cheb_step(h, l, k, f, x, p, &alpha);
        free(p);
    }
    return OR_OK;
}

/* V-cycle, Algorithm 2:
 *   coarsest:  x = A_L^-1 f
 *   otherwise: npre x relax; t = f - A x; f_c = R t; x_c = 0 (§8c);
 *              vcycle(l+1, f_c, x_c); x = x + P x_c; npost x relax. */
int or_vcycle(const or_hier *h, int l, const double *f, double *x) {
    if (l == h->nlev - 1) return or_lu_solve(h->nL, h->lu, h->piv, f, x);
    const or_csr *A = h->A[l];
    int64_t n = A->nrows, nc = h->P[l]->ncols;
    for (int s = 0; s < h->prm.npre; s++) or_relax(h, l, f, x);
    double *t = (double *)malloc((size_t)n * sizeof(double));
    double *fc = (double *)malloc((size_t)(nc > 0 ? nc : 1) * sizeof(double));
    double *xc = (double *)calloc((size_t)(nc > 0 ? nc : 1), sizeof(double));
    double *e = (double *)malloc((size_t)n * sizeof(double));
    residual(A, f, x, t);
    spmv_csr(h->R[l], t, fc);
    or_vcycle(h, l + 1, fc, xc);
    spmv_csr(h->P[l], xc, e);
    for (int64_t i = 0; i < n; i++) x[i] = x[i] + e[i];
    for (int s = 0; s < h->prm.npost; s++) or_relax(h, l, f, x);
    free(t);
    free(fc);
    free(xc);
    free(e);
    return OR_OK;
}

/* Preconditioner z = M r: a single V-cycle from a zero guess (PAPER.md:141-143,
 * SPEC.md:360-363). */
int or_precond(const or_hier *h, const double *r, double *z) {
    int64_t n = h->A[0]->nrows;
    for (int64_t i = 0; i < n; i++) z[i] = 0.0;
    return or_vcycle(h, 0, r, z);
}

/* Preconditioned CG (§8c c-1, L17):
 *   nf = |f|; f = 0 -> x = 0, 0 iterations
 *   r = f - A x; res = |r|
 *   while k < maxiter and res > tol nf:
 *       z = M r; rho = (r,z); rho <= 0 -> breakdown
 *       p = (k == 0) ? z : z + (rho/rho_prev) p
 *       q = A p; sigma = (p,q) (sigma <= 0 -> breakdown); alpha = rho/sigma
 *       x += alpha p; r -= alpha q; res = |r|; rho_prev = rho; k++
 *   rel_resid = |f - A x| / nf  (recomputed true residual) */
int or_cg(const or_hier *h, int64_t n, const int64_t *ptr, const int32_t *col, const double *val,
          int precond, const double *f, double *x, double tol, int32_t maxiter, int32_t *iters,
          double *rel_resid, double *hist) {
    or_csr A = {n, n, ptr[n], (int64_t *)ptr, (int32_t *)col, (double *)val};
    double nf = sqrt(dot(n, f, f));
    *iters = 0;
    *rel_resid = 0.0;
    if (nf == 0.0) {
        for (int64_t i = 0; i < n; i++) x[i] = 0.0;
        if (hist) hist[0] = 0.0;
        return OR_OK;
    }
    double *r = (double *)malloc((size_t)n * sizeof(double));
    double *z = (double *)malloc((size_t)n * sizeof(double));
    double *p = (double *)malloc((size_t)n * sizeof(double));
    double *q = (double *)malloc((size_t)n * sizeof(double));
    residual(&A, f, x, r);
    double res = sqrt(dot(n, r, r));
    if (hist) hist[0] = res;
    double rho_prev = 1.0;
    int32_t k = 0;
    int status = OR_OK;
    while (k < maxiter && res > tol * nf) {
        if (precond)
            or_precond(h, r, z);
        else
            memcpy(z, r, (size_t)n * sizeof(double));
        double rho = dot(n, r, z);
        if (!(rho > 0.0)) {
            set_err("CG breakdown: (r, Mr) = %g <= 0", rho);
            status = OR_BREAKDOWN;
            break;
        }
        if (k == 0) {
            memcpy(p, z, (size_t)n * sizeof(double));
        } else {
            double beta = rho / rho_prev;
            for (int64_t i = 0; i < n; i++) p[i] = z[i] + beta * p[i];
        }
        spmv_csr(&A, p, q);
        double sigma = dot(n, p, q);
        if (!(sigma > 0.0)) {
            set_err("CG breakdown: (p, Ap) = %g <= 0", sigma);
            status = OR_BREAKDOWN;
            break;
        }
        double alpha = rho / sigma;
        for (int64_t i = 0; i < n; i++) x[i] = x[i] + alpha * p[i];
        for (int64_t i = 0; i < n; i++) r[i] = r[i] - alpha * q[i];
        res = sqrt(dot(n, r, r));
        rho_prev = rho;
        k += 1;
        if (hist) hist[k] = res;
    }
    if (status == OR_OK && res > tol * nf) status = OR_NOT_CONVERGED;
    residual(&A, f, x, r);
    *iters = k;
    *rel_resid = sqrt(dot(n, r, r)) / nf;
    free(r);
    free(z);
    free(p);
    free(q);
    return status;
}

/* Right-preconditioned BiCGStab (van der Vorst; §8c):
 *   r = f - A x; rh = r; res = |r|
 *   while k < maxiter and res > tol nf:
 *     rho = (rh, r); |rho| < 1e-30 |rh||r| -> breakdown
 *     p = (k == 0) ? r : r + (rho/rho_prev)(alpha/omega)(p - omega v)
 *     ph = M p; v = A ph; alpha = rho / (rh, v)
 *     s = r - alpha v; |s| <= tol nf -> x += alpha ph; k++; stop
 *     sh = M s; t = A sh; omega = (t,s)/(t,t); |omega| < 1e-30 -> breakdown
 *     x += alpha ph + omega sh; r = s - omega t; res = |r|; k++
 * vcycles counts preconditioner applications (§8c). */
int or_bicgstab(const or_hier *h, int64_t n, const int64_t *ptr, const int32_t *col,
                const double *val, int precond, const double *f, double *x, double tol,
                int32_t maxiter, int32_t *iters, double *rel_resid, int32_t *vcycles) {
    or_csr A = {n, n, ptr[n], (int64_t *)ptr, (int32_t *)col, (double *)val};
    double nf = sqrt(dot(n, f, f));
    *iters = 0;
    *rel_resid = 0.0;
    *vcycles = 0;
    if (nf == 0.0) {
        for (int64_t i = 0; i < n; i++) x[i] = 0.0;
        return OR_OK;
    }
    size_t bytes = (size_t)n * sizeof(double);
    double *r = (double *)malloc(bytes), *rh = (double *)malloc(bytes);
    double *p = (double *)calloc((size_t)n, sizeof(double)), *v = (double *)calloc((size_t)n, sizeof(double));
    double *ph = (double *)malloc(bytes), *s = (double *)malloc(bytes), *sh = (double *)malloc(bytes);
    double *t = (double *)malloc(bytes);
    residual(&A, f, x, r);
    memcpy(rh, r, bytes);
    double res = sqrt(dot(n, r, r));
    double rho_prev = 1.0, alpha = 1.0, omega = 1.0;
    int32_t k = 0, vc = 0;
    int status = OR_OK;
    while (k < maxiter && res > tol * nf) {
        double rho = dot(n, rh, r);
        if (fabs(rho) < 1e-30 * sqrt(dot(n, rh, rh)) * sqrt(dot(n, r, r))) {
            set_err("BiCGStab breakdown: rho = %g", rho);
            status = OR_BREAKDOWN;
            break;
        }
        if (k == 0) {
            memcpy(p, r, bytes);
        } else {
            double beta = (rho / rho_prev) * (alpha / omega);
            for (int64_t i = 0; i < n; i++) p[i] = r[i] + beta * (p[i] - omega * v[i]);
        }
        if (precond) {
            or_precond(h, p, ph);
            vc++;
        } else {
            memcpy(ph, p, bytes);
        }
        spmv_csr(&A, ph, v);
        double rv = dot(n, rh, v);
        if (rv == 0.0) {
            set_err("BiCGStab breakdown: (rh, v) = 0");
            status = OR_BREAKDOWN;
            break;
        }
        alpha = rho / rv;
        for (int64_t i = 0; i < n; i++) s[i] = r[i] - alpha * v[i];
        double ns = sqrt(dot(n, s, s));
        if (ns <= tol * nf) {
            for (int64_t i = 0; i < n; i++) x[i] = x[i] + alpha * ph[i];
            k += 1;
            res = ns;
            break;
        }
        if (precond) {
            or_precond(h, s, sh);
            vc++;
        } else {
            memcpy(sh, s, bytes);
        }
        spmv_csr(&A, sh, t);
        double tt = dot(n, t, t);
        if (tt == 0.0) {
            set_err("BiCGStab breakdown: (t, t) = 0");
            status = OR_BREAKDOWN;
            break;
        }
        omega = dot(n, t, s) / tt;
        if (fabs(omega) < 1e-30) {
            set_err("BiCGStab breakdown: omega = %g", omega);
            status = OR_BREAKDOWN;
            break;
        }
        for (int64_t i = 0; i < n; i++) x[i] = x[i] + alpha * ph[i] + omega * sh[i];
        for (int64_t i = 0; i < n; i++) r[i] = s[i] - omega * t[i];
        res = sqrt(dot(n, r, r));
        rho_prev = rho;
        k += 1;
    }
    if (status == OR_OK && res > tol * nf) status = OR_NOT_CONVERGED;
    residual(&A, f, x, r);
    *iters = k;
    *vcycles = vc;
    *rel_resid = sqrt(dot(n, r, r)) / nf;
    free(r);
    free(rh);
    free(p);
    free(v);
    free(ph);
    free(s);
    free(sh);
    free(t);
    return status;
}

/* Restarted right-preconditioned GMRES(m) (PAPER.md:212 names GMRES; the
 * algorithm is Saad, Iterative Methods for Sparse Linear Systems, 2nd ed.,
 * Alg. 9.5 "GMRES with right preconditioning", restarted every m steps):
 *   r = f - A x; beta = |r|; converged if beta <= tol |f|
 *   cycle:  v_0 = r / beta;  g = beta e_0
 *     for j = 0 .. m-1:
 *        z = M v_j; w = A z
 *        for i = 0 .. j:  h_ij = (w, v_i); w = w - h_ij v_i      (modified Gram-Schmidt)
 *        h_{j+1,j} = |w|; v_{j+1} = w / h_{j+1,j}
 *        apply the previous Givens rotations to column j of H; build rotation j
 *        that zeroes h_{j+1,j}; g_{j+1} = -s_j g_j, g_j = c_j g_j
 *        k += 1; stop the cycle if |g_{j+1}| <= tol |f| or k == maxiter
 *     solve the upper-triangular H y = g (size j+1); x = x + M (V y)
 *     r = f - A x; beta = |r|; converged if beta <= tol |f|  (true residual)
 * A zero h_{j+1,j} (lucky breakdown) ends the cycle with the exact solution. */
int or_gmres(const or_hier *h, int64_t n, const int64_t *ptr, const int32_t *col, const double *val,
             int precond, int32_t m, const double *f, double *x, double tol, int32_t maxiter,
             int32_t *iters, double *rel_resid, int32_t *vcycles, double *hist) {
    or_csr A = {n, n, ptr[n], (int64_t *)ptr, (int32_t *)col, (double *)val};
    double nf = sqrt(dot(n, f, f));
    *iters = 0;
    *rel_resid = 0.0;
    *vcycles = 0;
    if (m < 1) {
        set_err("gmres: restart m must be >= 1");
        return OR_E_INVALID;
    }
    if (nf == 0.0) {
        for (int64_t i = 0; i < n; i++) x[i] = 0.0;
        if (hist) hist[0] = 0.0;
        return OR_OK;
    }
    size_t bytes = (size_t)n * sizeof(double);
    double *V = (double *)malloc(bytes * (size_t)(m + 1));
    double *H = (double *)calloc((size_t)(m + 1) * (size_t)m, sizeof(double)); /* H[i*m + j] */
    double *cs = (double *)malloc((size_t)m * sizeof(double));
    double *sn = (double *)malloc((size_t)m * sizeof(double));
    double *g = (double *)malloc((size_t)(m + 1) * sizeof(double));
    double *y = (double *)malloc((size_t)m * sizeof(double));
    double *r = (double *)malloc(bytes), *z = (double *)malloc(bytes), *w = (double *)malloc(bytes);
    double *u = (double *)malloc(bytes);
    residual(&A, f, x, r);
    double beta = sqrt(dot(n, r, r));
    if (hist) hist[0] = beta;
    int32_t k = 0, vc = 0;
    int status = OR_OK;
    while (beta > tol * nf && k < maxiter) {
        for (int64_t i = 0; i < n; i++) V[i] = r[i] / beta;
        for (int i = 0; i <= m; i++) g[i] = 0.0;
        g[0] = beta;
        int jlast = -1;
        for (int j = 0; j < m; j++) {
            double *vj = V + (size_t)j * n;
            if (precond) {
                or_precond(h, vj, z);
                vc++;
            } else {
                memcpy(z, vj, bytes);
            }
            spmv_csr(&A, z, w);
            for (int i = 0; i <= j; i++) {
                double *vi = V + (size_t)i * n;
                double hij = dot(n, w, vi);
                H[i * m + j] = hij;
                for (int64_t q = 0; q < n; q++) w[q] = w[q] - hij * vi[q];
            }
            double hn = sqrt(dot(n, w, w));
            H[(j + 1) * m + j] = hn;
            if (hn != 0.0)
                for (int64_t q = 0; q < n; q++) V[(size_t)(j + 1) * n + q] = w[q] / hn;
            for (int i = 0; i < j; i++) { /* previous rotations on column j */
                double a = H[i * m + j], b = H[(i + 1) * m + j];
                H[i * m + j] = cs[i] * a + sn[i] * b;
                H[(i + 1) * m + j] = -sn[i] * a + cs[i] * b;
            }
            double a = H[j * m + j], b = H[(j + 1) * m + j];
            double d = sqrt(a * a + b * b);
            cs[j] = d == 0.0 ? 1.0 : a / d;
            sn[j] = d == 0.0 ? 0.0 : b / d;
            H[j * m + j] = d;
            H[(j + 1) * m + j] = 0.0;
            g[j + 1] = -sn[j] * g[j];
            g[j] = cs[j] * g[j];
            k += 1;
            jlast = j;
            if (hist) hist[k] = fabs(g[j + 1]);
            if (fabs(g[j + 1]) <= tol * nf || k >= maxiter || hn == 0.0) break;
        }
        /* y = H^-1 g (upper triangular, back substitution) */
        for (int i = jlast; i >= 0; i--) {
            double s = g[i];
            for (int q = i + 1; q <= jlast; q++) s -= H[i * m + q] * y[q];
            if (H[i * m + i] == 0.0) {
                set_err("gmres: singular Hessenberg");
                status = OR_BREAKDOWN;
                break;
            }
            y[i] = s / H[i * m + i];
        }
        if (status != OR_OK) break;
        for (int64_t q = 0; q < n; q++) u[q] = 0.0; /* u = V y */
        for (int i = 0; i <= jlast; i++)
            for (int64_t q = 0; q < n; q++) u[q] = u[q] + y[i] * V[(size_t)i * n + q];
        if (precond) {
            or_precond(h, u, z);
            vc++;
        } else {
            memcpy(z, u, bytes);
        }
        for (int64_t q = 0; q < n; q++) x[q] = x[q] + z[q];
        residual(&A, f, x, r);
        beta = sqrt(dot(n, r, r));
    }
    if (status == OR_OK && beta > tol * nf) status = OR_NOT_CONVERGED;
    *iters = k;
    *vcycles = vc;
    *rel_resid = beta / nf;
    free(V);
    free(H);
    free(cs);
    free(sn);
    free(g);
    free(y);
    free(r);
    free(z);
    free(w);
    free(u);
    return status;
}

/* IDR(s) shadow space: P (column-major, P[j*n + i]) from a counter-based
 * generator -- entry (i, j) = 2 u - 1, u = the top 53 bits of
 * splitmix64(0x181105704 + j*n + i) / 2^53 -- then orthonormalised by modified
 * Gram-Schmidt over the columns j = 0..s-1 (the library implements the same
 * generator on its own: DESIGN.md §8f). */
static uint64_t splitmix64(uint64_t z) {
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

void or_idrs_shadow(int64_t n, int32_t s, double *P) {
    for (int32_t j = 0; j < s; j++)
        for (int64_t i = 0; i < n; i++) {
            uint64_t z = splitmix64(0x181105704ull + (uint64_t)j * (uint64_t)n + (uint64_t)i);
            P[(int64_t)j * n + i] = 2.0 * ((double)(z >> 11) * 0x1.0p-53) - 1.0;
        }
    for (int32_t j = 0; j < s; j++) {
        double *pj = P + (int64_t)j * n;
        for (int32_t q = 0; q < j; q++) {
            const double *pq = P + (int64_t)q * n;
            double h = dot(n, pq, pj);
            for (int64_t i = 0; i < n; i++) pj[i] = pj[i] - h * pq[i];
        }
        double nrm = sqrt(dot(n, pj, pj));
        for (int64_t i = 0; i < n; i++) pj[i] = pj[i] / nrm;
    }
}

/* Right-preconditioned IDR(s) with bi-orthogonalisation (PAPER.md:212 lists
 * IDR(s), citing Sonneveld & van Gijzen 2008; the variant is van Gijzen &
 * Sonneveld, ACM TOMS 38(1) 2011, "Algorithm 913", with the preconditioner B = M
 * applied as in their right-preconditioned form):
 *   r = f - A x;  G = U = 0 (n x s);  M = I (s x s);  om = 1
 *   while |r| > tol |f|:
 *     phi = P^T r
 *     for k = 0 .. s-1:
 *        solve M[k:s, k:s] c = phi[k:s]                    (lower triangular)
 *        v = r - G[:, k:s] c;   v = B v
 *        U[:, k] = U[:, k:s] c + om v;   G[:, k] = A U[:, k]
 *        for i = 0 .. k-1:  a = (P[:, i], G[:, k]) / M[i, i]
 *                           G[:, k] -= a G[:, i];  U[:, k] -= a U[:, i]
 *        M[k:s, k] = P[:, k:s]^T G[:, k];  breakdown if M[k, k] = 0
 *        beta = phi[k] / M[k, k];  r -= beta G[:, k];  x += beta U[:, k]
 *        stop if |r| <= tol |f|;   phi[k+1:s] -= beta M[k+1:s, k]
 *     v = B r;  t = A v
 *     om = (t, r) / (t, t);  rho = |(t, r)| / (|t| |r|);  if rho < kappa: om *= kappa / rho
 *     breakdown if om = 0;  x += om v;  r -= om t
 * kappa = 0.7 ("angle" strategy, the authors' default; 0 = minimal residual).
 * iters counts preconditioned matrix-vector products (s per cycle + 1);
 * vcycles = iters when precond.  P: shadow space (column-major n x s) or NULL
 * for or_idrs_shadow's.  resid_hist (maxiter + 1 or NULL): |r| after each. */
int or_idrs(const or_hier *h, int64_t n, const int64_t *ptr, const int32_t *col, const double *val,
            int precond, int32_t s, double kappa, const double *Pin, const double *f, double *x, double tol,
            int32_t maxiter, int32_t *iters, double *rel_resid, int32_t *vcycles, double *resid_hist) {
    or_csr A = {n, n, ptr[n], (int64_t *)ptr, (int32_t *)col, (double *)val};
    *iters = 0;
    *vcycles = 0;
    *rel_resid = 0.0;
    if (s < 1 || s > 64) {
        set_err("IDR(s): s must be in [1, 64]");
        return OR_E_INVALID;
    }
    double nf = sqrt(dot(n, f, f));
    if (nf == 0.0) {
        for (int64_t i = 0; i < n; i++) x[i] = 0.0;
        if (resid_hist) resid_hist[0] = 0.0;
        return OR_OK;
    }
    size_t bytes = (size_t)n * sizeof(double);
    double *P = (double *)malloc(bytes * s), *G = (double *)calloc((size_t)n * s, sizeof(double));
    double *U = (double *)calloc((size_t)n * s, sizeof(double));
    double *r = (double *)malloc(bytes), *v = (double *)malloc(bytes), *z = (double *)malloc(bytes);
    double *t = (double *)malloc(bytes), *uk = (double *)malloc(bytes);
    double *M = (double *)calloc((size_t)s * s, sizeof(double)), *phi = (double *)malloc(sizeof(double) * s);
    double *c = (double *)malloc(sizeof(double) * s);
    if (Pin)
        memcpy(P, Pin, bytes * s);
    else
        or_idrs_shadow(n, s, P);
    for (int32_t i = 0; i < s; i++) M[i * s + i] = 1.0; /* M[row * s + col] */
    residual(&A, f, x, r);
    double res = sqrt(dot(n, r, r));
    if (resid_hist) resid_hist[0] = res;
    double om = 1.0;
    int32_t it = 0, vc = 0;
    int status = OR_OK;
    int stop = !(res > tol * nf);
    while (!stop && it < maxiter) {
        for (int32_t i = 0; i < s; i++) phi[i] = dot(n, P + (int64_t)i * n, r);
        for (int32_t k = 0; k < s && !stop && it < maxiter; k++) {
            /* M[k:s, k:s] c = phi[k:s], forward substitution */
            for (int32_t i = k; i < s; i++) {
                double sum = phi[i];
                for (int32_t j = k; j < i; j++) sum -= M[i * s + j] * c[j - k];
                c[i - k] = sum / M[i * s + i];
            }
            for (int64_t q = 0; q < n; q++) {
                double sum = r[q];
                for (int32_t j = k; j < s; j++) sum -= c[j - k] * G[(int64_t)j * n + q];
                v[q] = sum;
            }
            if (precond) {
                or_precond(h, v, z);
                vc++;
            } else {
                memcpy(z, v, bytes);
            }
            for (int64_t q = 0; q < n; q++) {
                double sum = om * z[q];
                for (int32_t j = k; j < s; j++) sum += c[j - k] * U[(int64_t)j * n + q];
                uk[q] = sum;
            }
            memcpy(U + (int64_t)k * n, uk, bytes);
            double *gk = G + (int64_t)k * n, *ukp = U + (int64_t)k * n;
            spmv_csr(&A, ukp, gk);
            for (int32_t i = 0; i < k; i++) {
                double a = dot(n, P + (int64_t)i * n, gk) / M[i * s + i];
                for (int64_t q = 0; q < n; q++) {
                    gk[q] = gk[q] - a * G[(int64_t)i * n + q];
                    ukp[q] = ukp[q] - a * U[(int64_t)i * n + q];
                }
            }
            for (int32_t i = k; i < s; i++) M[i * s + k] = dot(n, P + (int64_t)i * n, gk);
            it++;
            if (M[k * s + k] == 0.0) {
                set_err("IDR(s) breakdown: M[%d][%d] = 0", k, k);
                status = OR_BREAKDOWN;
                stop = 1;
                break;
            }
            double beta = phi[k] / M[k * s + k];
            for (int64_t q = 0; q < n; q++) {
                r[q] = r[q] - beta * gk[q];
                x[q] = x[q] + beta * ukp[q];
            }
            res = sqrt(dot(n, r, r));
            if (resid_hist) resid_hist[it] = res;
            if (!(res > tol * nf)) {
                stop = 1;
                break;
            }
            for (int32_t i = k + 1; i < s; i++) phi[i] = phi[i] - beta * M[i * s + k];
        }
        if (stop || it >= maxiter) break;
        /* dimension reduction step */
        if (precond) {
            or_precond(h, r, z);
            vc++;
        } else {
            memcpy(z, r, bytes);
        }
        spmv_csr(&A, z, t);
        double tt = sqrt(dot(n, t, t)), tr = dot(n, t, r);
        it++;
        if (tt == 0.0) {
            set_err("IDR(s) breakdown: A B r = 0");
            status = OR_BREAKDOWN;
            break;
        }
        om = tr / (tt * tt);
        double rho = fabs(tr) / (tt * res);
        if (rho < kappa) om = om * kappa / rho;
        if (om == 0.0) {
            set_err("IDR(s) breakdown: omega = 0");
            status = OR_BREAKDOWN;
            break;
        }
        for (int64_t q = 0; q < n; q++) {
            x[q] = x[q] + om * z[q];
            r[q] = r[q] - om * t[q];
        }
        res = sqrt(dot(n, r, r));
        if (resid_hist) resid_hist[it] = res;
        if (!(res > tol * nf)) stop = 1;
    }
    if (status == OR_OK && res > tol * nf) status = OR_NOT_CONVERGED;
    residual(&A, f, x, r);
    *iters = it;
    *vcycles = vc;
    *rel_resid = sqrt(dot(n, r, r)) / nf;
    free(P);
    free(G);
    free(U);
    free(r);
    free(v);
    free(z);
    free(t);
    free(uk);
    free(M);
    free(phi);
    free(c);
    return status;
}
