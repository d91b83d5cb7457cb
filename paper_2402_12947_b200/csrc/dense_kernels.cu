// Coarse-level solve and deterministic reductions (sm_100a, fp64).
//
// Coarse solve (mg.py:145, Hierarchy.coarse_factor from mg.py:123): the
// reference runs LAPACK dpotrs on the dense Cholesky factor of A_L.  Two
// dependent triangular sweeps over an n_L^2 factor are latency-bound on a GPU
// (n_L sequential steps), so the library applies the precomputed dense
// operator A_L^{-1} = (L L^T)^{-1} as one HBM-streaming GEMV across every SM,
// optionally followed by one refinement step x += A_L^{-1}(b - A_L x) (the
// residual uses the sparse coarse operator).  Parity is tolerance-based, like
// every dense solve on this path.
//
// Reductions (solve_stationary norms mg.py:164,174; CG dots sparse.py:184-208):
// fixed grid, fixed per-thread stride, fixed shuffle tree, last-block
// finalisation in block order -> run-to-run deterministic results.
#include "smg_internal.cuh"

namespace smg {

constexpr int kGemvThreads = 128;                 // 4 rows (warps) per CTA
constexpr int kGemvUnroll = 8;                    // independent 256 B loads in flight per warp

__device__ __forceinline__ double warp_sum_d(double v)
{
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// y = M x (kAdd=false) or y += M x (kAdd=true); M dense row-major n x n.
// One warp per row, kGemvUnroll independent accumulators (fixed order: the
// result is run-to-run deterministic).
template <bool kAdd>
__global__ void __launch_bounds__(kGemvThreads)
dense_gemv_kernel(int64_t n, const double* __restrict__ m, const double* __restrict__ x,
                  double* __restrict__ y)
{
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * (kGemvThreads / 32) + (threadIdx.x >> 5);
  if (row >= n) return;
  const double* __restrict__ mr = m + row * n;
  double acc[kGemvUnroll];
#pragma unroll
  for (int u = 0; u < kGemvUnroll; ++u) acc[u] = 0.0;
  int64_t j = lane;
  for (; j + 32 * (kGemvUnroll - 1) < n; j += 32 * kGemvUnroll) {
    double mv[kGemvUnroll];
#pragma unroll
    for (int u = 0; u < kGemvUnroll; ++u) mv[u] = __ldcs(mr + j + 32 * u);
#pragma unroll
    for (int u = 0; u < kGemvUnroll; ++u) acc[u] = fma(mv[u], __ldg(x + j + 32 * u), acc[u]);
  }
  for (; j < n; j += 32) acc[0] = fma(__ldcs(mr + j), __ldg(x + j), acc[0]);
  double s = 0.0;
#pragma unroll
  for (int u = 0; u < kGemvUnroll; ++u) s += acc[u];
  s = warp_sum_d(s);
  if (lane == 0) {
    if (kAdd)
      y[row] += s;
    else
      y[row] = s;
  }
}

static cudaError_t gemv(int64_t n, const double* m, const double* x, double* y, bool add,
                        cudaStream_t s)
{
  if (n == 0) return cudaSuccess;
  const int64_t blocks = (n + (kGemvThreads / 32) - 1) / (kGemvThreads / 32);
  if (add)
    dense_gemv_kernel<true><<<(unsigned)blocks, kGemvThreads, 0, s>>>(n, m, x, y);
  else
    dense_gemv_kernel<false><<<(unsigned)blocks, kGemvThreads, 0, s>>>(n, m, x, y);
  return cudaGetLastError();
}

cudaError_t launch_dense_gemv(int64_t n, const double* m, const double* x, double* y,
                              cudaStream_t s)
{
  return gemv(n, m, x, y, false, s);
}

cudaError_t launch_dense_gemv_add(int64_t n, const double* m, const double* x, double* y,
                                  cudaStream_t s)
{
  return gemv(n, m, x, y, true, s);
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
