// Coarse-level solve and deterministic reductions (sm_100a, fp64).
//
// Coarse solve (mg.py:145, Hierarchy.coarse_factor from mg.py:123): the
// reference runs LAPACK dpotrs on the dense Cholesky factor of A_L.  Two
// dependent triangular sweeps over an n_L^2 factor are latency-bound on a GPU
// (n_L sequential steps), so the library applies the precomputed symmetric
// operator A_L^{-1} = (L L^T)^{-1} as an HBM-streaming symmetric matrix-vector
// product over its lower triangle (every tile read once, used for A x and
// A^T x), optionally followed by one refinement step x += A_L^{-1}(b - A_L x)
// (the residual uses the sparse coarse operator).  Parity is tolerance-based, like
// every dense solve on this path.
//
// Reductions (solve_stationary norms mg.py:164,174; CG dots sparse.py:184-208):
// fixed grid, fixed per-thread stride, fixed shuffle tree, last-block
// finalisation in block order -> run-to-run deterministic results.
#include "smg_internal.cuh"

#include <cstdlib>

namespace smg {

__device__ __forceinline__ double warp_sum_d(double v)
{
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---------------------------------------------------------------------------
// Symmetric coarse operator applied from its lower triangle only (half the
// bytes of the dense GEMV): A_L^{-1} is stored as 64 x 64 tiles (I, J), J <= I,
// row-major inside a tile, zero-padded, tile (I, J) at index I(I+1)/2 + J.
// One kernel, one CTA per tile: partial[I][J] = A_IJ x_J and, off the
// diagonal, partial[J][I] = A_IJ^T x_I.  Each block row I receives nb partials;
// the CTA that delivers the last one (per-row counter) forms
// y_i = sum_J partial[I][J][i] in ascending J and resets the counter -- a fixed
// summation order whoever finalises, so the result is run-to-run
// deterministic.  The tile (static data) is requested before the programmatic
// dependency wait, x after it.
constexpr int kSymThreads = 256;
constexpr int kSymRowsPerThread = kSymTile * kSymTile / kSymThreads;   // 16

__device__ __forceinline__ void sym_finish_row(int row, int nb, int64_t n,
                                               const double* partial, double* y, bool add)
{
  const int tid = threadIdx.x;
  if (tid >= kSymTile) return;
  const int64_t i = (int64_t)row * kSymTile + tid;
  if (i >= n) return;
  const double* p = partial + (int64_t)row * nb * kSymTile + tid;
  double s = 0.0;
  for (int J = 0; J < nb; ++J) s += __ldcg(p + (int64_t)J * kSymTile);
  y[i] = (add & 1) ? y[i] + s : s;
}

__global__ void __launch_bounds__(kSymThreads)
sym_tile_kernel(int nb, const int32_t* __restrict__ tile_i, const double* __restrict__ tiles,
                const double* __restrict__ x, int64_t n, double* __restrict__ partial,
                unsigned int* __restrict__ counter, double* __restrict__ y, int add)
{
  __shared__ double s_xi[kSymTile], s_xj[kSymTile];
  __shared__ double s_row[kSymTile][2];
  __shared__ double s_col[kSymThreads / kSymTile][kSymTile];
  __shared__ int s_last[2];
  const int t = blockIdx.x;
  const int I = tile_i[t];
  const int J = t - I * (I + 1) / 2;
  SMG_DCHECK(I >= 0 && I < nb && J >= 0 && J <= I);
  const int tid = threadIdx.x;
  const int c = tid & (kSymTile - 1);      // column inside the tile
  const int g = tid / kSymTile;            // rows g, g + 4, g + 8, ...
  const double* __restrict__ a = tiles + (int64_t)t * kSymTile * kSymTile;
  double v[kSymRowsPerThread];
#pragma unroll
  for (int i = 0; i < kSymRowsPerThread; ++i)
    v[i] = add < 2 ? __ldcs(a + (g + 4 * i) * kSymTile + c) : __ldg(a + (g + 4 * i) * kSymTile + c);
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (tid < kSymTile) {
    const int64_t gi = (int64_t)I * kSymTile + tid, gj = (int64_t)J * kSymTile + tid;
    s_xi[tid] = gi < n ? x[gi] : 0.0;
    s_xj[tid] = gj < n ? x[gj] : 0.0;
  }
  __syncthreads();
  const int lane = tid & 31, warp = tid >> 5;
  // rows: each warp covers 32 of the 64 columns of its 16 rows
  const double xc = s_xj[c];
#pragma unroll
  for (int i = 0; i < kSymRowsPerThread; ++i) {
    double p = v[i] * xc;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) p += __shfl_xor_sync(0xffffffffu, p, o);
    if (lane == 0) s_row[g + 4 * i][warp & 1] = p;
  }
  // columns (off-diagonal tiles): this thread's 16 rows, then the 4 row groups
  if (I != J) {
    double q = 0.0;
#pragma unroll
    for (int i = 0; i < kSymRowsPerThread; ++i) q += v[i] * s_xi[g + 4 * i];
    s_col[g][c] = q;
  }
  __syncthreads();
  double* out = partial + ((int64_t)I * nb + J) * kSymTile;
  if (tid < kSymTile) out[tid] = s_row[tid][0] + s_row[tid][1];
  if (I != J && tid < kSymTile) {
    double q = 0.0;
#pragma unroll
    for (int gg = 0; gg < kSymThreads / kSymTile; ++gg) q += s_col[gg][tid];
    partial[((int64_t)J * nb + I) * kSymTile + tid] = q;
  }
  if (!counter) return;   // two-kernel mode: sym_reduce_kernel sums the rows
  // deliver: the last contributor of a block row sums it (threadFenceReduction)
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    const unsigned ci = atomicAdd(&counter[I], 1u);
    SMG_DCHECK(ci < (unsigned)nb);   // a block row receives exactly nb partials per call
    s_last[0] = ci == (unsigned)(nb - 1);
    unsigned cj = 0;
    if (I != J) {
      cj = atomicAdd(&counter[J], 1u);
      SMG_DCHECK(cj < (unsigned)nb);
    }
    s_last[1] = I != J && cj == (unsigned)(nb - 1);
  }
  __syncthreads();
  if (s_last[0]) {
    __threadfence();
    sym_finish_row(I, nb, n, partial, y, (add & 1) != 0);
    if (tid == 0) counter[I] = 0;
  }
  if (s_last[1]) {
    __threadfence();
    sym_finish_row(J, nb, n, partial, y, (add & 1) != 0);
    if (tid == 0) counter[J] = 0;
  }
}

int sym_apply_launches()
{
  const char* v = getenv("SMG_COARSE_FUSED");
  return (v && atoi(v)) ? 1 : 2;
}

// one CTA per 64-row block row: thread group q (of 4) sums the partials
// J = q, q + 4, ... in ascending order, then the four group sums are added in
// group order -- a fixed order, so run-to-run deterministic
template <bool kAdd>
__global__ void __launch_bounds__(256) sym_reduce_kernel(int nb, int64_t n,
                                                        const double* __restrict__ partial,
                                                        double* __restrict__ y)
{
  __shared__ double s_part[4][kSymTile];
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int I = blockIdx.x;
  const int r = threadIdx.x & (kSymTile - 1), q = threadIdx.x / kSymTile;
  const double* p = partial + (int64_t)I * nb * kSymTile + r;
  double s = 0.0;
  for (int J = q; J < nb; J += 4) s += p[(int64_t)J * kSymTile];
  s_part[q][r] = s;
  __syncthreads();
  const int64_t i = (int64_t)I * kSymTile + threadIdx.x;
  if (threadIdx.x < kSymTile && i < n) {
    const double t = ((s_part[0][r] + s_part[1][r]) + s_part[2][r]) + s_part[3][r];
    if (kAdd)
      y[i] += t;
    else
      y[i] = t;
  }
}

cudaError_t launch_sym_apply(const SymTiles& m, const double* x, double* y, bool add,
                             cudaStream_t s)
{
  if (m.n == 0) return cudaSuccess;
  static const int fused = [] {
    const char* v = getenv("SMG_COARSE_FUSED");
    return v ? atoi(v) : 0;
  }();
  if (!fused) {
    // two kernels, both programmatic dependents (counter == nullptr: the tile
    // kernel only writes partials)
    const int64_t ntiles = (int64_t)m.nb * (m.nb + 1) / 2;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)ntiles);
    cfg.blockDim = dim3(kSymThreads);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    // SMG_COARSE_KEEP=1: tiles read with normal L2 priority (they may stay
    // resident between V-cycles when small); default evict-first
    static const int keep = [] {
      const char* v = getenv("SMG_COARSE_KEEP");
      return v ? atoi(v) : 0;
    }();
    const int mode = (add ? 1 : 0) | (keep ? 2 : 0);
    cudaError_t e = cudaLaunchKernelEx(&cfg, sym_tile_kernel, m.nb, m.tile_i, m.tiles, x, m.n,
                                       m.partial, (unsigned int*)nullptr, y, mode);
    if (e != cudaSuccess) return e;
    cfg.gridDim = dim3((unsigned)m.nb);
    cfg.blockDim = dim3(256);
    if (add) return cudaLaunchKernelEx(&cfg, sym_reduce_kernel<true>, m.nb, m.n,
                                       (const double*)m.partial, y);
    return cudaLaunchKernelEx(&cfg, sym_reduce_kernel<false>, m.nb, m.n,
                              (const double*)m.partial, y);
  }
  const int64_t ntiles = (int64_t)m.nb * (m.nb + 1) / 2;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)ntiles);
  cfg.blockDim = dim3(kSymThreads);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, sym_tile_kernel, m.nb, m.tile_i, m.tiles, x, m.n, m.partial,
                            m.counter, y, add ? 1 : 0);
}

// ---------------------------------------------------------------------------
constexpr int kDotThreads = 256;

__global__ void __launch_bounds__(kDotThreads)
dot_kernel(int64_t n, const double* __restrict__ a, const double* __restrict__ b,
           double* __restrict__ partials, unsigned int* __restrict__ counter,
           double* __restrict__ result)
{
  __shared__ double s_w[kDotThreads / 32];
  __shared__ bool s_last;
  const int64_t stride = (int64_t)gridDim.x * kDotThreads;
  double acc = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * kDotThreads + threadIdx.x; i < n; i += stride)
    acc = fma(a[i], b[i], acc);
  acc = warp_sum_d(acc);
  if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kDotThreads / 32; ++w) t += s_w[w];
    partials[blockIdx.x] = t;
    __threadfence();
    const unsigned int done = atomicAdd(counter, 1u);
    s_last = (done == gridDim.x - 1);
  }
  __syncthreads();
  if (s_last && threadIdx.x < 32) {
    __threadfence();
    double t = 0.0;
    for (int i = threadIdx.x; i < (int)gridDim.x; i += 32)
      t += ((volatile double*)partials)[i];
    t = warp_sum_d(t);
    if (threadIdx.x == 0) {
      *result = t;
      *counter = 0u;
    }
  }
}

cudaError_t launch_dot(int64_t n, const double* a, const double* b, double* partials,
                       unsigned int* counter, double* result, cudaStream_t s)
{
  dot_kernel<<<kDotBlocks, kDotThreads, 0, s>>>(n, a, b, partials, counter, result);
  return cudaGetLastError();
}

// mode 0: y = y + alpha*x ; mode 1: y = y - alpha*x ; mode 2: y = x + beta*y
// (numpy order of `x += alpha*d`, `r -= alpha*q`, `d = z + beta*d`, sparse.py:202-209)
__global__ void axpby_kernel(int64_t n, double alpha, const double* __restrict__ x, double beta,
                             double* __restrict__ y, int mode)
{
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    if (mode == 0)
      y[i] = __dadd_rn(y[i], __dmul_rn(alpha, x[i]));
    else if (mode == 1)
      y[i] = __dsub_rn(y[i], __dmul_rn(alpha, x[i]));
    else
      y[i] = __dadd_rn(x[i], __dmul_rn(beta, y[i]));
  }
}

cudaError_t launch_axpby(int64_t n, double alpha, const double* x, double beta, double* y,
                         int mode, cudaStream_t s)
{
  if (n == 0) return cudaSuccess;
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  axpby_kernel<<<(unsigned)blocks, 256, 0, s>>>(n, alpha, x, beta, y, mode);
  return cudaGetLastError();
}

}  // namespace smg
