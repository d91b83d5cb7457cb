/*
 * TEST INFRASTRUCTURE ONLY -- the CPU oracle for the simplexmg hot path.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  The product path
 * (paper_2402_12947_b200/) never links or calls it.
 *
 * Plain-C restatement of the compiled arithmetic the reference reaches
 * through scipy / LAPACK on its hot path (reference paths are relative to
 * /root/reference):
 *
 *   oracle_csr_matvec   scipy sparsetools csr_matvec, reached from
 *                       pkg/src/simplexmg/sparse.py:115-118 (to_scipy() @ x),
 *                       used at smoothers.py:123,128,132,263,266 and
 *                       mg.py:141,149,164,174.  Row-sequential, column-order
 *                       sum starting from 0.0, one rounding per multiply and
 *                       one per add (no FMA contraction).
 *   oracle_csrT_matvec  scipy csc_matvec reached from mg.py:142
 *                       (P.to_scipy().T @ r): y[c] += P[i,c] r[i] for fine
 *                       rows i in ascending order.  Restated over an explicit
 *                       CSR(P^T) whose rows list fine indices ascending.
 *   oracle_spgemm       scipy sparsetools csr_matmat (SMMP), reached from the
 *                       Galerkin product sparse.py:147-154 (ps.T @ (a @ ps),
 *                       via transfer.py:153-155 coarsen_system, mg.py:100):
 *                       row i of C = X Y accumulates sums[k] += X_ij * Y_jk
 *                       over X's row in stored (ascending column) order,
 *                       starting from 0.0, and keeps only sums != 0.
 *   oracle_chol_solve   LAPACK dpotrs via scipy.linalg.cho_solve
 *                       (sparse.py:225-231): forward substitution with L,
 *                       back substitution with L^T.  Sequential order differs
 *                       from blocked LAPACK, so agreement is to ~1e-15 relative,
 *                       not bitwise (pinned by tests/golden fixtures).
 *
 * Build: oracle/Makefile (gcc -O2 -fopenmp -ffp-contract=off).  Row loops are
 * OpenMP-parallel; every row's own sum is sequential, so the thread count
 * never changes a result bit.
 */
#include <stdint.h>
#include <stdlib.h>
#include <math.h>
#include <omp.h>

int oracle_num_threads(void) { return omp_get_max_threads(); }
void oracle_set_threads(int n) { if (n > 0) omp_set_num_threads(n); }

/* y = A x  (scipy csr_matvec order) */
void oracle_csr_matvec(int64_t nrows, const int64_t *rowptr, const int64_t *col,
                       const double *val, const double *x, double *y)
{
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < nrows; ++i) {
        double sum = 0.0;
        for (int64_t jj = rowptr[i]; jj < rowptr[i + 1]; ++jj)
            sum += val[jj] * x[col[jj]];
        y[i] = sum;
    }
}

/* y = A x restricted to a row list: y[k] = (A x)[rows[k]] (same per-row order) */
void oracle_csr_matvec_rows(int64_t nsel, const int64_t *rows, const int64_t *rowptr,
                            const int64_t *col, const double *val, const double *x,
                            double *y)
{
    #pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < nsel; ++k) {
        int64_t i = rows[k];
        double sum = 0.0;
        for (int64_t jj = rowptr[i]; jj < rowptr[i + 1]; ++jj)
            sum += val[jj] * x[col[jj]];
        y[k] = sum;
    }
}

/* y = P^T r given CSR(P^T) with ascending fine indices per row
 * (scipy csc_matvec accumulates y[c] in ascending fine-row order from 0.0). */
void oracle_csrT_matvec(int64_t ncoarse, const int64_t *tptr, const int64_t *tcol,
                        const double *tval, const double *r, double *y)
{
    #pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < ncoarse; ++c) {
        double sum = 0.0;
        for (int64_t jj = tptr[c]; jj < tptr[c + 1]; ++jj)
            sum += tval[jj] * r[tcol[jj]];
        y[c] = sum;
    }
}

/* Solve (L L^T) x = r in place, L the lower triangle of the row-major n x n
 * array c (scipy cho_factor(lower=True) layout; the upper triangle is ignored). */
static void chol_solve_one(int64_t n, const double *c, double *x)
{
    for (int64_t i = 0; i < n; ++i) {
        double s = x[i];
        const double *row = c + i * n;
        for (int64_t j = 0; j < i; ++j) s -= row[j] * x[j];
        x[i] = s / row[i];
    }
    for (int64_t i = n - 1; i >= 0; --i) {
        double s = x[i];
        for (int64_t j = i + 1; j < n; ++j) s -= c[j * n + i] * x[j];
        x[i] = s / c[i * n + i];
    }
}

void oracle_chol_solve(int64_t n, const double *c, double *x)
{
    chol_solve_one(n, c, x);
}

/* Batched patch solves: patch p owns dofs idx[ptr[p]..ptr[p+1]) and a dense
 * row-major factor at factors + foff[p].  x holds the patch residuals laid
 * out like idx and is overwritten by the corrections. */
void oracle_patch_solves(int64_t npatch, const int64_t *ptr, const int64_t *foff,
                         const double *factors, double *x)
{
    #pragma omp parallel for schedule(dynamic, 1)
    for (int64_t p = 0; p < npatch; ++p) {
        int64_t n = ptr[p + 1] - ptr[p];
        chol_solve_one(n, factors + foff[p], x + ptr[p]);
    }
}

/* plain sequential sum of squares / dot (the reference uses BLAS ddot via
 * np.linalg.norm / r @ z; those differ from this only in rounding order) */
double oracle_dot(int64_t n, const double *a, const double *b)
{
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];
    return s;
}

/* C = X Y (scipy csr_matmat order, see the header).  The output rows are
 * canonical (columns ascending), as CsrMatrix.from_scipy leaves them
 * (sparse.py:93-99: sort_indices; sorting does not touch values).
 * Pass 1 (cptr != NULL, ccol == NULL): cptr[0..nrows] = row offsets of the
 * kept entries.  Pass 2 (ccol, cval != NULL): fill them. */
static int cmp_i64(const void *a, const void *b)
{
    int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
    return (x > y) - (x < y);
}

void oracle_spgemm(int64_t nrows, int64_t ncols, const int64_t *xptr, const int64_t *xcol,
                   const double *xval, const int64_t *yptr, const int64_t *ycol,
                   const double *yval, int64_t *cptr, int64_t *ccol, double *cval)
{
    #pragma omp parallel
    {
        double *sums = (double *)calloc((size_t)ncols, sizeof(double));
        int64_t *mark = (int64_t *)malloc((size_t)ncols * sizeof(int64_t));
        int64_t *keys = (int64_t *)malloc((size_t)ncols * sizeof(int64_t));
        for (int64_t k = 0; k < ncols; ++k) mark[k] = -1;
        #pragma omp for schedule(dynamic, 256)
        for (int64_t i = 0; i < nrows; ++i) {
            int64_t nk = 0;
            for (int64_t jj = xptr[i]; jj < xptr[i + 1]; ++jj) {
                const int64_t j = xcol[jj];
                const double v = xval[jj];
                for (int64_t kk = yptr[j]; kk < yptr[j + 1]; ++kk) {
                    const int64_t k = ycol[kk];
                    if (mark[k] != i) {
                        mark[k] = i;
                        keys[nk++] = k;
                    }
                    sums[k] += v * yval[kk];
                }
            }
            qsort(keys, (size_t)nk, sizeof(int64_t), cmp_i64);
            int64_t kept = 0;
            int64_t out = ccol ? cptr[i] : 0;
            for (int64_t t = 0; t < nk; ++t) {
                const int64_t k = keys[t];
                if (sums[k] != 0) {
                    if (ccol) {
                        ccol[out + kept] = k;
                        cval[out + kept] = sums[k];
                    }
                    ++kept;
                }
                sums[k] = 0.0;
            }
            if (!ccol) cptr[i + 1] = kept;
        }
        free(sums);
        free(mark);
        free(keys);
    }
    if (!ccol) {
        cptr[0] = 0;
        for (int64_t i = 0; i < nrows; ++i) cptr[i + 1] += cptr[i];
    }
}
