// Internal types shared by the sm_100a kernels and the C-ABI layer.
// Nothing here crosses the library boundary (include/simplexmg_b200.h is the
// only public surface).
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <string>
#include <vector>

// SMG_CHECKED (a variant build, tools/checked_run.py): device-side bounds and
// protocol assertions in the kernels -- the substitute for compute-sanitizer,
// which this pool does not run (profiles/r02/sanitizer/).  A failed check
// prints its condition and traps (the launch fails with an error the host
// reports).  Compiled out of the product build.
#ifdef SMG_CHECKED
#include <cstdio>
#define SMG_DCHECK(cond)                                                             \
  do {                                                                               \
    if (!(cond)) {                                                                   \
      printf("SMG_DCHECK failed %s:%d block %d thread %d: %s\n", __FILE__, __LINE__, \
             (int)blockIdx.x, (int)threadIdx.x, #cond);                              \
      __trap();                                                                      \
    }                                                                                \
  } while (0)
#else
#define SMG_DCHECK(cond) \
  do {                   \
  } while (0)
#endif

namespace smg {

// ---------------------------------------------------------------------------
// CSR-stream partition.  A "tile" is a run of consecutive rows owned by one
// CTA: at most kRowsPerTile rows and (unless a single row is longer) at most
// kTileNnz nonzeros.  The CTA streams the tile's values/columns with
// coalesced loads into shared memory as exact products val*x[col], then every
// thread sums its own row sequentially in column order -- the order scipy's
// csr_matvec uses -- so results are bit-identical to the reference.
constexpr int kThreads = 256;        // one row per thread at most
constexpr int kRowsPerTile = kThreads;
#ifndef SMG_TILE_NNZ
#define SMG_TILE_NNZ 2048
#endif
constexpr int kTileNnz = SMG_TILE_NNZ;  // products staged per pass (16 KB smem)
constexpr int kItems = kTileNnz / kThreads;
// operators with long rows get tiles of up to kMaxTileChunks chunks of
// kTileNnz nonzeros (<= kRowsPerTile rows): more rows sum in parallel per CTA
// and each chunk's loads overlap the previous chunk's sums
constexpr int kMaxTileChunks = 4;
constexpr int64_t kStreamBytes = 64ll << 20;   // operators above this are streamed evict-first
// whole-tile staging (csr_stage_kernel): the tile's products live in dynamic
// shared memory (8 B each), kStageCtas CTAs per SM
constexpr int kStageCtas = 3;
constexpr int kStageMaxNnz = 9216;   // 72 KB per CTA, 3 x 73 KB <= 227 KB per SM

struct DevCsr {
  int64_t nrows = 0, ncols = 0, nnz = 0;
  const int64_t* rowptr = nullptr;   // nrows + 1
  const int32_t* col = nullptr;      // nnz
  const double* val = nullptr;       // nnz
  const int32_t* tile_row = nullptr; // ntiles + 1 (row boundaries of tiles)
  const int64_t* tile_nz = nullptr;  // ntiles + 1 (rowptr at the tile boundaries)
  const double* inv_diag = nullptr;  // 1.0 / a_ii (IEEE, as smoothers.py:115), square ops
  const int32_t* row_map = nullptr;  // gathered row subsets: local row -> operator row
  int32_t ntiles = 0;
  bool streaming = false;            // val+col exceed kStreamBytes: evict-first reads
  bool multichunk = false;           // long rows: tiles of up to kMaxTileChunks chunks
  int32_t stage_cap = 0;             // > 0: tiles of at most stage_cap nonzeros, staged whole (csr_stage_kernel)
  // fixed-capacity layout: tile t's nonzeros sit at [t*cap, (t+1)*cap) of the
  // padded arrays (zero values / column 0 after the last row), so a CTA can
  // issue its value/column loads without first loading its tile offset;
  // rel_end[r] = end of row r relative to its tile's start
  bool fixed = false;
  int32_t cap = 0;
  const int32_t* pcol = nullptr;
  const double* pval = nullptr;
  const int32_t* rel_end = nullptr;
  // SELL-32-sigma256 layout (sell_kernel): windows of 256 consecutive rows,
  // rows sorted by length inside the window (perm: slot -> row offset, -1 =
  // no row), 8 slices of 32 slots per window stored column-major (entry j of
  // the 32 slots contiguous; padding column -1), slice offsets in sell_ptr
  bool sell = false;
  // lanes per row: 1 = SELL-32-sigma256 (sell_kernel); 4 = SELL-8x4 (sell4_kernel:
  // windows of 64 rows, slices of 8 rows, 4 lanes per row -- entry 4b+t of
  // slot r at slice offset 32b + 4r + t; sigma = 64)
  int32_t sell_lanes = 1;
  int32_t sell_unroll = 4;             // loop unroll (4: 8 CTAs/SM; 8/16: long rows)
  int32_t sell_pipe = 0;               // 8-deep long rows: software-pipelined batch depth (0 = off)
  int32_t sell_nwin = 0;
  const int64_t* sell_ptr = nullptr;   // nwin * 8 + 1
  const int16_t* sell_perm = nullptr;  // nwin * 256
  const int32_t* sell_col = nullptr;
  const double* sell_val = nullptr;
  // SELL-d16 (sell_delta): 16-bit column codes at the positions of sell_col
  // (which is then not uploaded): delta to the row's previous column, 0xFFFE
  // padding, 0xFFFF = take the slot's next escape column; first column and
  // escapes per slot (sell_esc: sell_esc_planes planes of nwin * 256)
  bool sell_delta = false;
  int32_t sell_esc_planes = 0;
  const uint16_t* sell_dcol = nullptr;
  const int32_t* sell_c0 = nullptr;
  const int32_t* sell_esc = nullptr;
};
constexpr int kSellWindow = 256;
constexpr int kSellSlices = kSellWindow / 32;
constexpr int kSell4Window = 64;    // SELL-8x4: 8 slices of 8 rows per window

// Host-side owner of one operator's device arrays.
struct Operator {
  DevCsr a;                 // the matrix
  bool has_t = false;
  DevCsr t;                 // CSR of the transpose (restriction P^T), fine index ascending
  int64_t first_zero_diag = -1;   // -1: every row has a nonzero diagonal
  bool all_finite = true;          // every stored value is finite
  const double* diag = nullptr;    // explicit diagonal (0.0 where absent), square ops
  const double* inv_diag = nullptr;  // 1.0 / diag, exactly as numpy forms inv_diag
  int64_t device_bytes = 0;
  std::vector<void*> allocs;
};

// rows of a producer operator (A for a sweep, P for the prolong-add) on every
// region's ring, gathered at upload (rptr indexes the concatenated ring rows)
struct RingRows {
  const int64_t* rptr = nullptr;
  const int32_t* rcol = nullptr;
  const double* rval = nullptr;
};

struct Correction {
  int64_t n_global = 0;
  int32_t n_regions = 0;
  int64_t m = 0;                 // total patch dofs
  int32_t max_dofs = 0;
  const int32_t* pptr = nullptr;   // n_regions + 1
  const int32_t* dofs = nullptr;   // m (global dof of each patch slot)
  const int32_t* order = nullptr;  // n_regions: launch order, largest region first
  const int64_t* foff = nullptr;   // n_regions + 1, offsets into packed factors
  const double* lfac = nullptr;    // packed lower factors, row-major
  double* rbuf = nullptr;          // m scratch (patch residual / correction)
  const int64_t* prow = nullptr;   // m + 1: offsets of the patch rows' gathered copy
  const int32_t* pcol = nullptr;   // gathered columns of the patch rows of A
  const double* pval = nullptr;    // gathered values of the patch rows of A
  // interior/halo split of A around the patches: halo rows are those whose
  // stencil touches a patch dof (they depend on the correction); `halo` holds
  // their gathered rows (with row_map), `halo_mask` flags them per row
  bool has_halo = false;
  DevCsr halo;
  const uint8_t* halo_mask = nullptr;
  bool coupled = true;             // some A[B_d, B_d'] != 0 (d != d')
  bool sym = false;                // regions past the L^{-1} sizes hold packed A[B,B]^{-1}
  // follow mode (correction overlapped with the kernel producing its u): the
  // ring of region d is the sorted set of columns of its rows (B_d included);
  // the correction kernel recomputes the producer's output there from the
  // producer's inputs, while the producer skips the patch dofs (bmask)
  bool has_ring = false;
  int32_t ring_max = 0;
  int64_t ring_total = 0;
  const int32_t* ring_ptr = nullptr;   // n_regions + 1
  const int32_t* ring_rows = nullptr;  // ring_total global rows
  const int32_t* plcol = nullptr;      // per gathered patch-row entry: ring position of its column
  const int32_t* bpos = nullptr;       // per patch dof: its own ring position
  const uint8_t* bmask = nullptr;      // per row: 1 = patch dof
  RingRows ringA;                      // A's rows on the rings
  const Operator* op = nullptr;
  int64_t device_bytes = 0;
  std::vector<void*> allocs;
};

// patch slot geometry: packed L (even length) + inverted 32x32 diagonal blocks
constexpr int kPanel = 32;
constexpr int kDinvLd = 33;                       // padded row stride (bank conflicts)
constexpr int kDinvBlock = kPanel * kDinvLd;      // 1056 doubles (even)
__host__ __device__ inline int64_t patch_tri_even(int64_t nd)
{
  return (nd * (nd + 1) / 2 + 1) & ~int64_t(1);
}
// Regions of 33..64 dofs carry the whole inverse of L in a 64 x 65 block
// (zero above the diagonal) instead of inverted 32 x 32 diagonal blocks, and so
// do regions of 65..128 dofs (128 x 129 block) when no region of the
// correction is larger (the slot then still fits shared memory): each
// triangular solve is one GEMV instead of a chain of panel steps.
__host__ __device__ inline int patch_block(int64_t nd, int64_t nmax)
{
  if (nd > kPanel && nd <= 2 * kPanel) return 2 * kPanel;
  if (nd > 2 * kPanel && nd <= 4 * kPanel && nmax <= 4 * kPanel) return 4 * kPanel;
  return 0;
}
// Symmetric-inverse regions (round 2, SMG_PATCH_SYM, default on): a region
// that would otherwise run the panel substitution (more than 32 dofs and no
// whole-L^{-1} block) stores the packed lower triangle of A[B,B]^{-1} =
// L^{-T} L^{-1} instead of L: the correction is one symmetric matrix-vector
// product streamed from HBM once, with no serial panel chain.
// (corrections with a region of more than kPatchSymMaxDofs dofs keep the
// substitution path: the per-warp rings would not fit shared memory)
constexpr int kPatchSymMaxDofs = 896;
__host__ __device__ inline bool patch_is_sym(int64_t nd, int64_t nmax, bool sym)
{
  return sym && nd > kPanel && patch_block(nd, nmax) == 0;
}
__host__ __device__ inline int64_t patch_slot_doubles(int64_t nd, int64_t nmax, bool sym)
{
  if (patch_is_sym(nd, nmax, sym)) return patch_tri_even(nd);
  const int64_t B = patch_block(nd, nmax);
  return patch_tri_even(nd) + (B ? B * (B + 1) : ((nd + kPanel - 1) / kPanel) * kDinvBlock);
}
// the largest slot that is staged whole in shared memory for regions of at
// most nmax dofs (slots are not monotonic; symmetric-inverse regions stream)
__host__ __device__ inline int64_t patch_slot_max(int64_t nmax, bool sym)
{
  if (sym && nmax > 4 * kPanel)   // staged: <= 32 dofs (L + one block) and 33..64 (L + 64 x 65)
    return patch_slot_doubles(2 * kPanel, nmax, sym);
  const int64_t a = patch_slot_doubles(nmax, nmax, sym);
  const int64_t b =
      nmax > kPanel ? patch_slot_doubles(nmax < 2 * kPanel ? nmax : 2 * kPanel, nmax, sym) : 0;
  return a > b ? a : b;
}

enum SmootherKind : int { kChebyshev = 0, kJacobi = 1 };

struct Smoother {
  int kind = kChebyshev;
  int sweeps = 1;
  double lambda_max = 0.0;
  double lambda_min_fraction = 0.1;
};

// error reporting (thread-local last error)
void set_error(const std::string& msg);
int fail(const std::string& msg);
int check_cuda(cudaError_t e, const char* what);

// ---------------------------------------------------------------------------
// kernel launchers (spmv_kernels.cu)
enum class Epi : int {
  kSpmv = 0,       // y = s
  kResidual,       // y = b - s
  kJacobi,         // u_out = u_in + (inv_d * (b - s)) / theta
  kChebFirst,      // d = (inv_d * (b - s)) / theta ; u_out = u_in + d
  kChebNext,       // z = inv_d * (b - s) ; d = c1*d + c2*z ; u_out = u_in + d
  kAddTo,          // y = y + s  (prolong-add)
  kRestrictFirst,  // b_c = s (restriction), then the coarse level's first smoother
                   // step from a zero initial guess: d = (1/diag * (b_c - 0)) / theta,
                   // u_c = 0 + d  (A_c 0 sums to +0.0 exactly, so this equals the
                   // reference's first sweep bit for bit)
};

struct EpiArgs {
  const double* b = nullptr;
  const double* u_in = nullptr;
  double* out = nullptr;   // y / r / u_out
  double* d = nullptr;
  double theta = 1.0, c1 = 0.0, c2 = 0.0;
  const double* inv_diag = nullptr;  // kRestrictFirst: coarse operator 1/diagonal
  double* b_out = nullptr;        // kRestrictFirst: restricted right-hand side
  const uint8_t* skip_rows = nullptr;  // interior pass: rows flagged here are not written
  bool keep_d = true;   // false: the last Chebyshev step of a smooth (d is dead) leaves d alone
  bool stream_vec = false;  // set by the launcher: per-row vectors b, d, 1/a_ii read (and d
                            // written) evict-first, so x keeps the L2 (SMG_EVICT_VEC)
};

// follow-mode correction (patch_kernels.cu): producer epilogue `epi` (kJacobi,
// kChebFirst, kChebNext or kAddTo) recomputed on the rings, then
// out[B_d] = producer(B_d) + (L L^T)^{-1} (b - A producer)[B_d]
struct FollowArgs {
  int epi = 0;
  RingRows ring;
  const double* x = nullptr;      // the producer's SpMV input (u_in / coarse u)
  const double* u_in = nullptr;   // sweeps: u_in; prolong-add: the fine u before the add
  const double* b = nullptr;      // the level's right-hand side
  const double* d = nullptr;      // kChebNext: direction before the step
  const double* inv_diag = nullptr;
  double theta = 1.0, c1 = 0.0, c2 = 0.0;
  double* out = nullptr;          // the producer's output vector
  int ring_max = 0;               // set by the launcher (shared-memory carve-up)
};

cudaError_t launch_csr_stream(const DevCsr& m, const double* x, Epi epi, const EpiArgs& ea,
                              cudaStream_t s);
void configure_l2_persist();   // SMG_L2_PERSIST_MB carve-out (call outside stream capture)

// patch kernels (patch_kernels.cu)
cudaError_t launch_patch_residual(const DevCsr& a, const Correction& c, const double* b,
                                  const double* u, cudaStream_t s);
cudaError_t launch_gather(const int32_t* idx, int64_t m, const double* src, double* dst,
                          cudaStream_t s);
cudaError_t launch_patch_solve(const Correction& c, const double* b, const double* u_res,
                               double* u_add, double* out_scatter, bool fused, cudaStream_t s);
cudaError_t configure_patch_solve_smem(const Correction& c);
cudaError_t launch_patch_follow(const Correction& c, const FollowArgs& fa, cudaStream_t s);
bool patch_follow_fits(const Correction& c);
cudaError_t launch_patch_row_len(const DevCsr& a, const int32_t* dofs, int64_t m, int64_t* len);
cudaError_t launch_patch_row_gather(const DevCsr& a, const int32_t* dofs, int64_t m,
                                    const int64_t* prow, int32_t* pcol, double* pval);
cudaError_t launch_mark_halo(const DevCsr& a, const uint8_t* in_patch, uint8_t* mask);

// symmetric coarse operator, lower-triangle 64 x 64 tiles (dense_kernels.cu)
constexpr int kSymTile = 64;
struct SymTiles {
  int64_t n = 0;
  int nb = 0;                        // tiles per dimension
  const double* tiles = nullptr;     // nb(nb+1)/2 tiles of kSymTile^2 doubles
  const int32_t* tile_i = nullptr;   // block row of each tile
  double* partial = nullptr;         // nb * nb * kSymTile scratch
  unsigned int* counter = nullptr;   // nb: partials delivered per block row (0 between calls)
};
cudaError_t launch_sym_apply(const SymTiles& m, const double* x, double* y, bool add,
                             cudaStream_t s);
int sym_apply_launches();   // kernels one launch_sym_apply enqueues (1 fused, 2 default)

// sparse matrix product C = X Y in scipy csr_matmat's order, bit-identical
// (galerkin_kernels.cu; the Galerkin operator P^T (A P), sparse.py:147-154)
struct DevCsrOwned {
  int64_t nrows = 0, ncols = 0, nnz = 0;
  int64_t* rowptr = nullptr;
  int32_t* col = nullptr;
  double* val = nullptr;
  void release();
  DevCsr view() const;
};
cudaError_t spgemm_device(const DevCsr& X, const DevCsr& Y, DevCsrOwned* out, cudaStream_t s);

// prolongation rows by point location (transfer_kernels.cu; transfer.py:73-150)
struct LocateArgs {
  int64_t n_points = 0;
  const double* points = nullptr;      // n_points x dim fine DOF coordinates
  int64_t n_cells = 0;
  const double* v0 = nullptr;          // n_cells x dim first vertex of each coarse cell
  const double* inv_jac = nullptr;     // n_cells x dim x dim (np.linalg.inv of the edge matrix)
  const int64_t* cell_nodes = nullptr; // n_cells x nodes-per-cell coarse DOFs
  int64_t n_coarse = 0;
  int nb = 1;                          // bins per dimension
  double lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0}, scale[3] = {0, 0, 0};
  const int64_t* bin_ptr = nullptr;    // nb^dim + 1
  const int64_t* bin_cells = nullptr;  // ascending cell ids per bin
  double tol = 1e-10, drop_tol = 1e-14;
};
cudaError_t prolongation_device(const LocateArgs& a, int dim, int degree, DevCsrOwned* out,
                                int64_t* failed_point, cudaStream_t s);

// batched dense Cholesky of the local-correction blocks (factor_kernels.cu;
// smoothers.py:176-200).  status[r] = 0 or the failing leading minor (dpotrf
// info); sym[2r] = max |a - a^T|, sym[2r+1] = max |a| of the gathered block.
cudaError_t launch_patch_factor(const DevCsr& a, int64_t n_regions, const int32_t* pptr,
                                const int32_t* dofs, const int64_t* foff, double* w,
                                int64_t* status, double* sym, cudaStream_t s);

// dense Cholesky (invert=false: A -> cho_factor's c in place, *info = dpotrf
// info) or inverse from such a factor (invert=true: dpotri, full symmetric);
// row-major, cuSOLVER (coarse_factor.cu).  With check_symmetry the max|a - a^T|
// and max|a| come back in *asym / *amax and an asymmetric input stops early.
int dense_cholesky_device(int64_t n, double* d_a, bool check_symmetry, double* asym,
                          double* amax, int64_t* info_out, bool invert, cudaStream_t s);

// Poisson stiffness with Dirichlet elimination (assembly_kernels.cu; fem.py:303-377)
int assemble_poisson_device(int dim, int degree, int64_t n_vertices, const double* verts,
                            int64_t n_cells, const int64_t* cells, const int64_t* cell_dofs,
                            int64_t n_dofs, const uint8_t* dirichlet_mask, int64_t n_dir,
                            const int64_t* dir_dofs, const double* gref, const double* wq, int nq,
                            DevCsrOwned* out, int64_t* bad_cell_out, cudaStream_t s);

// element matrices (host, the reference's arithmetic) -> canonical CSR with
// scipy's duplicate order and the Dirichlet elimination (coo_kernels.cu;
// fem.py:339-375).  dirichlet_mask: host, n_dofs bytes, or nullptr.
int assemble_elements_device(int64_t n_dofs, int64_t n_cells, int nloc, const int64_t* cell_dofs,
                             const double* local, const uint8_t* dirichlet_mask, DevCsrOwned* out,
                             cudaStream_t s);

// dense / reduction kernels (dense_kernels.cu)
cudaError_t launch_dot(int64_t n, const double* a, const double* b, double* partials,
                       unsigned int* counter, double* result, cudaStream_t s);
cudaError_t launch_axpby(int64_t n, double alpha, const double* x, double beta, double* y,
                         int mode, cudaStream_t s);
constexpr int kDotBlocks = 296;   // fixed grid => deterministic reduction order

}  // namespace smg
