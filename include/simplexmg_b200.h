/*
 * simplexmg_b200.h -- C-ABI of the B200-native combined-smoother hot path.
 *
 * A drop-in for the compiled arithmetic the reference (`simplexmg`, arXiv
 * 2402.12947; paths relative to /root/reference/pkg/src/simplexmg) reaches on
 * its V-cycle hot path.  The reference is pure Python over scipy/LAPACK and has
 * no FFI of its own; each entry point below names the reference function it
 * replaces, and INTEGRATION.md shows the ctypes binding a maintainer adds.
 *
 * Conventions
 *   - Plain C types only.  Matrices enter as HOST arrays in the reference's
 *     canonical CSR layout (int64 row offsets and column indices, float64
 *     values; sparse.py:47-84); the library keeps its own device copies.
 *   - Vectors are DEVICE pointers (float64) unless the name ends in _host.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *   - Every call returns SMG_OK or an error code; smg_last_error() gives the
 *     message (thread-local).  Error codes map onto the reference's typed
 *     exceptions (sparse.py:23-44, smoothers.py:27-30).
 *   - No CPU fallback: every compute entry point launches sm_100a kernels.
 */
#ifndef SIMPLEXMG_B200_H
#define SIMPLEXMG_B200_H

#include <stdint.h>

#if defined(__GNUC__)
#define SMG_API __attribute__((visibility("default")))
#else
#define SMG_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define SMG_ABI_VERSION 1

#define SMG_OK 0
#define SMG_ERR_INVALID 1        /* ValueError (bad arguments / layout)               */
#define SMG_ERR_DIMENSION 2      /* ValueError "dimension mismatch" (sparse.py:139)   */
#define SMG_ERR_CUDA 3           /* RuntimeError from the CUDA runtime                */
#define SMG_ERR_ZERO_DIAGONAL 4  /* ZeroDiagonalError(row) (smoothers.py:112-114)     */
#define SMG_ERR_INDEFINITE 5     /* IndefiniteOperatorError (sparse.py:199-200)       */
#define SMG_ERR_UNSUPPORTED 6    /* NotImplementedError (e.g. SGS smoother)           */
#define SMG_ERR_POINT_LOCATION 7 /* PointLocationError (transfer.py:21-33)            */
#define SMG_ERR_NOT_SPD 8        /* NotPositiveDefiniteError (sparse.py:234-254)      */

/* smoother kinds (smoothers.py:33-59).  SMG_SMOOTHER_CHEBYSHEV with
 * lambda_min_fraction == 1 is the reference's damped-Jacobi branch
 * (smoothers.py:120-124; omega = 1/lambda_max). */
#define SMG_SMOOTHER_CHEBYSHEV 0
#define SMG_SMOOTHER_SGS 1       /* not on the GPU hot path: SMG_ERR_UNSUPPORTED */

typedef struct smg_operator smg_operator;
typedef struct smg_correction smg_correction;
typedef struct smg_hierarchy smg_hierarchy;
typedef struct smg_csr smg_csr;           /* device-resident CSR product result */

SMG_API int smg_abi_version(void);
SMG_API const char *smg_last_error(void);
SMG_API int smg_device_info(int *sm_count, int64_t *l2_bytes, int *cc_major, int *cc_minor);

/* ---- operators: CsrMatrix (sparse.py:47-132) ------------------------------
 * Canonical CSR (sorted, unique columns per row).  with_transpose != 0 also
 * stores CSR(A^T) so the operator can serve as a prolongation P (restriction
 * P^T r, mg.py:142). */
SMG_API int smg_operator_create(int64_t nrows, int64_t ncols, const int64_t *row_offsets,
                        const int64_t *col_indices, const double *values,
                        int with_transpose, smg_operator **out);
SMG_API int smg_operator_destroy(smg_operator *op);
/* first_zero_diag = first row whose diagonal is 0 or absent, -1 if none */
SMG_API int smg_operator_info(const smg_operator *op, int64_t *nrows, int64_t *ncols, int64_t *nnz,
                      int64_t *first_zero_diag, int64_t *device_bytes);

/* Device layout the sweeps of an operator run on (chosen at upload from its
 * row-length statistics; every layout is bit-identical):
 *   SMG_LAYOUT_TILES        CSR tiles with an offset table (csr_tile_kernel)
 *   SMG_LAYOUT_TILES_FIXED  fixed-capacity CSR tiles (csr_tile_kernel)
 *   SMG_LAYOUT_SELL         SELL-32-sigma256 (sell_kernel); *unroll = loop depth
 *   SMG_LAYOUT_SELL4        SELL-8x4, 4 lanes per row, sigma 64 (sell4_kernel);
 *                           *unroll = batches in flight (2 or 4)
 *   SMG_LAYOUT_SELL_D16     SELL-32-sigma256 with 16-bit delta-coded columns
 *                           (10 instead of 12 bytes per entry; same sums);
 *                           chosen by the rule for SELL operators whose rows
 *                           need at most two escapes
 *   SMG_LAYOUT_TILES_STAGED offset-table tiles staged whole in shared memory
 *                           (csr_stage_kernel: one barrier, every row of the
 *                           tile sums at once); chosen for long-row operators
 *                           that stay L2-resident; *unroll = load batches per tile
 * For tiles *unroll is the chunks per tile (1, or 4 for long-row operators). */
#define SMG_LAYOUT_TILES 0
#define SMG_LAYOUT_TILES_FIXED 1
#define SMG_LAYOUT_SELL 2
#define SMG_LAYOUT_SELL4 3
#define SMG_LAYOUT_SELL_D16 4
#define SMG_LAYOUT_TILES_STAGED 5
SMG_API int smg_operator_layout(const smg_operator *op, int *layout, int *unroll);
/* Force a layout (and SELL loop depth 4/8/16; 0 = by the rule) for the
 * operator and its stored transpose -- for tests and A/B runs; results are
 * bit-identical in every layout.  Not thread-safe with concurrent launches on
 * the operator; hierarchies built on it afterwards use the new layout.        */
SMG_API int smg_operator_set_layout(smg_operator *op, int layout, int unroll);

/* y = A x                       (sparse.py:135-140 spmv; bitwise)                */
SMG_API int smg_spmv(const smg_operator *a, const double *x, double *y, void *stream);
/* r = b - A u                   (smoothers.py:263,266; mg.py:141; bitwise)       */
SMG_API int smg_residual(const smg_operator *a, const double *b, const double *u, double *r,
                 void *stream);
/* y = P^T r                     (transfer.py:158-162 restrict_residual, mg.py:142;
 *                                bitwise vs scipy csc_matvec)                     */
SMG_API int smg_spmv_transpose(const smg_operator *p, const double *r, double *y, void *stream);
/* u_fine += P u_coarse          (transfer.py:165-172 prolong_add, mg.py:149)     */
SMG_API int smg_prolong_add(const smg_operator *p, const double *u_coarse, double *u_fine,
                    void *stream);

/* ---- setup: Galerkin coarse operator (sparse.py:147-154 triple_product, via
 * transfer.py:153-155 coarsen_system, mg.py:100) -------------------------------
 * *out = P^T (A P) on the device, bit-identical to scipy's `ps.T @ (a @ ps)`:
 * both products accumulate in csr_matmat's order (each output entry sums its
 * products in ascending order of the inner index, no FMA), entries whose sum
 * is exactly 0 are dropped as csr_matmat drops them, rows are canonical
 * (columns ascending).  p must have been created with_transpose.              */
SMG_API int smg_galerkin(const smg_operator *a, const smg_operator *p, smg_csr **out,
                         void *stream);
/* *out = X Y (scipy csr_matmat order, as above; the building block of
 * smg_galerkin, exposed for testing and other Galerkin-type products)          */
SMG_API int smg_matmul(const smg_operator *x, const smg_operator *y, smg_csr **out,
                       void *stream);
SMG_API int smg_csr_info(const smg_csr *c, int64_t *nrows, int64_t *ncols, int64_t *nnz);
/* copy to host CSR arrays (nrows + 1, nnz, nnz; int64 columns as sparse.py:63-65) */
SMG_API int smg_csr_to_host(const smg_csr *c, int64_t *row_offsets, int64_t *col_indices,
                            double *values);
SMG_API int smg_csr_destroy(smg_csr *c);

/* ---- setup: interpolation prolongation (transfer.py:117-150 build_prolongation
 * with CellLocator.locate, transfer.py:36-91) ---------------------------------
 * Row i of *out holds the coarse Lagrange basis (degree 1 or 2, dim 2 or 3)
 * evaluated at fine point i inside the lowest-index coarse cell whose
 * barycentric coordinates are all >= -tol (candidates: the cells listed for the
 * point's bin, ascending; if none hits, every cell), clamped to [0, 1] and
 * renormalised; entries with |value| <= drop_tol are dropped.  Host inputs:
 * points (n_points x dim), the coarse cells' first vertices v0 (n_cells x dim)
 * and inverse Jacobians inv_jac (n_cells x dim x dim, np.linalg.inv of the
 * edge matrices as transfer.py:46-48 forms them), cell_nodes (n_cells x
 * nodes per cell), and the bin index: nb bins per dimension over
 * [lo, hi] with scale = nb / span, bin_ptr (nb^dim + 1) / bin_cells.  Bitwise
 * equal to the reference's P.  A point outside every cell returns
 * SMG_ERR_POINT_LOCATION with *failed_point = the lowest such index.          */
SMG_API int smg_prolongation_build(int dim, int degree, int64_t n_points, const double *points,
                                   int64_t n_cells, const double *v0, const double *inv_jac,
                                   const int64_t *cell_nodes, int64_t n_coarse_nodes, int nb,
                                   const double *lo, const double *hi, const double *scale,
                                   const int64_t *bin_ptr, const int64_t *bin_cells, double tol,
                                   double drop_tol, smg_csr **out, int64_t *failed_point,
                                   void *stream);

/* Chebyshev / damped-Jacobi smoother in place on u (smoothers.py:99-136;
 * bitwise).  work: 2*((n+1)/2)*2 device doubles (two 16-byte aligned halves),
 * or NULL for a library allocation. */
SMG_API int smg_chebyshev_smooth(const smg_operator *a, const double *b, double *u, int sweeps,
                         double lambda_max, double lambda_min_fraction, double *work,
                         void *stream);

/* One fused smoother step (the loop body of smoothers.py:120-135), for
 * callers that drive the recurrence themselves and for per-kernel timing:
 *   step 0: u_out = u_in + (D^-1 (b - A u_in)) / theta              (:123)
 *   step 1: d = (D^-1 (b - A u_in)) / theta; u_out = u_in + d       (:128-129)
 *   step 2: d = c1 d + c2 D^-1 (b - A u_in); u_out = u_in + d       (:132-134)
 * u_out must not alias u_in (the reference forms A u before updating u). */
#define SMG_STEP_JACOBI 0
#define SMG_STEP_CHEB_FIRST 1
#define SMG_STEP_CHEB_NEXT 2
SMG_API int smg_smoother_step(const smg_operator *a, const double *b, const double *u_in,
                              double *u_out, double *d, int step, double theta, double c1,
                              double c2, void *stream);

/* ---- local correction: LocalCorrection (smoothers.py:139-200) ------------
 * Region d owns the sorted dofs[region_offsets[d] .. region_offsets[d+1]) and
 * the dense row-major n_d x n_d array factors[factor_offsets[d] ..] whose
 * LOWER triangle is the Cholesky factor (scipy cho_factor(lower=True),
 * sparse.py:248; the upper triangle is ignored).  Regions must be disjoint. */
SMG_API int smg_correction_create(const smg_operator *a, int64_t n_regions,
                          const int64_t *region_offsets, const int64_t *dofs,
                          const int64_t *factor_offsets, const double *factors,
                          smg_correction **out);
SMG_API int smg_correction_destroy(smg_correction *c);
SMG_API int smg_correction_info(const smg_correction *c, int64_t *n_regions, int64_t *covered_dofs,
                        int *coupled, int64_t *device_bytes);
/* ---- setup: stiffness from element matrices, scipy's exact order
 * (fem.py:339-375 assemble: coo_matrix((local, (rows, cols))).tocsr(), then the
 * symmetric Dirichlet elimination).  local: n_cells x nloc x nloc element
 * matrices (the reference's arithmetic, computed by the caller), cell_dofs:
 * n_cells x nloc.  Duplicates are summed in the order scipy's coo->csr uses
 * (entries bucketed by row in input order, then libstdc++ std::sort of every
 * row's (column, value) pairs unless all rows are already sorted, then runs
 * added sequentially), so *out is the reference's matrix bit for bit:
 * canonical CSR, rows/columns of the sorted dirichlet_dofs removed and a unit
 * diagonal in their place.                                                     */
SMG_API int smg_assemble_elements(int64_t n_dofs, int64_t n_cells, int nloc,
                                  const int64_t *cell_dofs, const double *local,
                                  const int64_t *dirichlet_dofs, int64_t n_dirichlet,
                                  smg_csr **out, void *stream);
/* ---- setup: Poisson stiffness assembly (fem.py:303-377 assemble, scalar
 * P1/P2, homogeneous Dirichlet on the listed DOFs) ---------------------------
 * Host inputs: vertices (n_vertices x dim), cells (n_cells x (dim+1), positively
 * oriented), cell_dofs (n_cells x nodes per cell, the DofMap numbering),
 * sorted dirichlet_dofs, and the reference gradients grad_ref (n_quad x nodes
 * x dim) with weights (n_quad) of the stiffness quadrature (fem.py:63-95).
 * *out = the assembled operator after symmetric elimination: Dirichlet rows
 * and columns removed, unit diagonal (canonical CSR).  Values agree with the
 * reference to rounding (element geometry by cofactors, duplicates summed in
 * cell order).  SMG_ERR_INVALID with *bad_cell for a cell with det <= 0.      */
SMG_API int smg_assemble_poisson(int dim, int degree, int64_t n_vertices, const double *vertices,
                                 int64_t n_cells, const int64_t *cells, const int64_t *cell_dofs,
                                 int64_t n_dofs, const int64_t *dirichlet_dofs,
                                 int64_t n_dirichlet, const double *grad_ref,
                                 const double *weights, int n_quad, smg_csr **out,
                                 int64_t *bad_cell, void *stream);

/* ---- setup: coarse operator factor and inverse (mg.py:123 coarse_factor =
 * sparse.py:234-254 dense_factor; the hot path's A_L^-1) --------------------
 * smg_dense_cholesky: a (host, n x n row-major) -> c (host) in cho_factor's
 * layout (L lower, A strict upper), on the device (hand-written blocked dpotrf,
 * csrc/coarse_factor.cu).
 * SMG_ERR_INVALID "… expects a symmetric matrix" when max|a - a^T| > 1e-10
 * max|a|; SMG_ERR_NOT_SPD with *info = dpotrf's leading minor when not SPD
 * (the reference then falls back to LU on the host).
 * smg_cholesky_inverse: c (cho_factor layout, lower) -> the full symmetric
 * A^-1 (host), as LAPACK dpotri on the same factor.                          */
SMG_API int smg_dense_cholesky(int64_t n, const double *a, double *c, int64_t *info,
                               void *stream);
SMG_API int smg_cholesky_inverse(int64_t n, const double *c, double *inverse, void *stream);

/* Factor every region's principal submatrix on the device (setup;
 * smoothers.py:176-200 build_local_correction -> sparse.py:234-254
 * dense_factor(lu_fallback=False) -> scipy cho_factor(lower=True)): one CTA per
 * region gathers A[B_d, B_d] and runs a blocked Cholesky.  factors (host, size
 * sum n_d^2, region order, row-major) receives cho_factor's `c` layout: L in
 * the lower triangle, A in the strict upper triangle.  Errors, first failing
 * region in order: SMG_ERR_INVALID "… expects a symmetric matrix" when
 * max|a - a^T| > 1e-10 max|a| (sparse.py:245-247), SMG_ERR_NOT_SPD with
 * *failed_region / *failed_minor (dpotrf info) when a pivot is not positive.
 * Region dofs must be sorted, unique, disjoint and in range.                  */
SMG_API int smg_patch_factor(const smg_operator *a, int64_t n_regions,
                             const int64_t *region_offsets, const int64_t *dofs, double *factors,
                             int64_t *failed_region, int64_t *failed_minor, void *stream);
/* out = S_c r, zero outside the regions (smoothers.py:203-211)                    */
SMG_API int smg_apply_local_correction(const smg_correction *c, const double *r, double *out,
                               void *stream);
/* u += S_c (b - A u)            (smoothers.py:263 / :266)                          */
SMG_API int smg_local_correct(const smg_correction *c, const double *b, double *u, void *stream);
/* sandwich smoother             (smoothers.py:252-267); c may be NULL.  c must
 * have been created for this operator a (its patch residuals read a's rows):
 * another operator is SMG_ERR_DIMENSION.                                          */
SMG_API int smg_combined_smooth(const smg_operator *a, const double *b, double *u,
                        const smg_correction *c, int kind, int sweeps, double lambda_max,
                        double lambda_min_fraction, double *work, void *stream);

/* ---- hierarchy and solvers: Hierarchy / vcycle (mg.py:51-184) -------------
 * Level l (0 = finest) has operator a[l], prolongation p[l] (from level l+1
 * into l; created with_transpose; ignored on the coarsest level), optional
 * correction[l] and smoother parameters.  The coarsest level is solved with
 * the dense operator coarse_inverse = A_L^{-1} (n_coarse x n_coarse row-major,
 * e.g. LAPACK dpotri on the reference's coarse_factor, mg.py:123; symmetric:
 * only its lower triangle is read and kept on the device, in 64 x 64 tiles);
 * coarse_refine != 0 adds one refinement step with a[n_levels-1].
 * The hierarchy borrows (does not own) the operators and corrections. */
SMG_API int smg_hierarchy_create(int n_levels, const smg_operator *const *a,
                         const smg_operator *const *p, const smg_correction *const *corrections,
                         const int *kinds, const int *sweeps, const double *lambda_max,
                         const double *lambda_min_fraction, int64_t n_coarse,
                         const double *coarse_inverse, int coarse_refine,
                         smg_hierarchy **out);
SMG_API int smg_hierarchy_destroy(smg_hierarchy *h);
/* enable != 0: capture each V-cycle once per (b, u) pointer pair as a CUDA graph */
SMG_API int smg_hierarchy_set_graphs(smg_hierarchy *h, int enable);
/* runtime options (each change drops cached graphs):
 *   SMG_OPT_GRAPHS          1 = capture V-cycles as CUDA graphs (default 1)
 *   SMG_OPT_FUSE_ZERO_GUESS 1 = fuse each coarse level's restriction with its
 *                           first smoother sweep from the zero initial guess
 *                           (mg.py:143; bit-identical, default 1)
 *   SMG_OPT_LC_OVERLAP      1 = run each local correction concurrently with the
 *                           patch-independent (interior) rows of the adjacent
 *                           smoother sweep; the halo rows follow (bit-identical,
 *                           default 0: the extra halo launch and the fork/join
 *                           cost more than the overlap saves on C1-C3)
 *   SMG_OPT_LC_FOLLOW       1 = every local correction that follows a kernel
 *                           producing u (the last smoother step, the
 *                           prolong-add) runs concurrently with it: the
 *                           producer skips the patch dofs, the correction
 *                           recomputes the producer on its rings and writes
 *                           them (bit-identical; default 1, but rings are
 *                           only built for corrections created with the
 *                           environment variable SMG_LC_FOLLOW=1: measured
 *                           slower on C1-C4, a dependent launch cannot start
 *                           before its producer's last wave) */
#define SMG_OPT_GRAPHS 0
#define SMG_OPT_FUSE_ZERO_GUESS 1
#define SMG_OPT_LC_OVERLAP 2
#define SMG_OPT_LC_FOLLOW 3
SMG_API int smg_hierarchy_set_option(smg_hierarchy *h, int option, int value);
/* kernels one V-cycle launches (for launch accounting) */
SMG_API int smg_hierarchy_launches_per_vcycle(const smg_hierarchy *h, int64_t *launches);
/* x_c = A_L^{-1} b_c on the coarsest level, exactly as the V-cycle applies it
 * (mg.py:145 h.coarse_factor.solve; symmetric 64 x 64 tiles of A_L^{-1},
 * deterministic reduction, plus the refinement step when the hierarchy was
 * created with coarse_refine).  Device vectors of the coarsest size.          */
SMG_API int smg_coarse_solve(smg_hierarchy *h, const double *b_c, double *x_c, void *stream);

/* u <- one V-cycle on u (mg.py:127-151; in place).
 * Thread safety ("concurrent vcycle calls on distinct arrays over
 * one shared Hierarchy are safe"): every call below that runs the hierarchy
 * (smg_vcycle*, smg_solve_stationary, smg_cg with a preconditioner, option
 * setters) holds a per-hierarchy mutex while it enqueues, and orders its
 * device work after the previous call's through an event, whatever stream
 * the callers use; results equal the sequential calls.                          */
SMG_API int smg_vcycle(smg_hierarchy *h, const double *b, double *u, void *stream);
/* same with HOST b/u: H2D copies, V-cycle, D2H of u (the e2e path)                */
SMG_API int smg_vcycle_host(smg_hierarchy *h, const double *b_host, double *u_host, void *stream);
/* count independent HOST (b[i], u[i]) pairs, one V-cycle each (u[i] in place),
 * pipelined: the copies of neighbouring pairs overlap each V-cycle.  Pinned
 * host memory gives the overlap; pageable memory is correct but serial.
 * Returns after the last u[i] is written back.                                   */
SMG_API int smg_vcycle_host_many(smg_hierarchy *h, int64_t count, const double *const *b_host,
                                 double *const *u_host, void *stream);
/* stationary MG (mg.py:154-175): u holds u0 on entry and the result on exit.
 * history: capacity max_cycles + 1 host doubles; *n_history entries written.  */
SMG_API int smg_solve_stationary(smg_hierarchy *h, const double *b, double *u, double rtol,
                         int max_cycles, double *history, int *n_history, void *stream);
/* MG-preconditioned CG (sparse.py:168-211 with mg.py:178-184 as precond).
 * h == NULL: unpreconditioned.  x holds x0 on entry when x0_given != 0, else
 * it is zeroed.  history: capacity maxit + 1.  On SMG_ERR_INDEFINITE,
 * *bad_iteration / *bad_curvature describe the failure.  A preconditioner
 * whose fine level is not a's size is SMG_ERR_DIMENSION (nothing launched). */
SMG_API int smg_cg(smg_hierarchy *h, const smg_operator *a, const double *b, double *x, int x0_given,
           double rtol, int maxit, double *history, int *n_history, int64_t *bad_iteration,
           double *bad_curvature, void *stream);
/* deterministic fixed-order dot product, result to host */
SMG_API int smg_dot(int64_t n, const double *x, const double *y, double *result_host, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* SIMPLEXMG_B200_H */
