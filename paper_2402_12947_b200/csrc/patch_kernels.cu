// Batched local correction S_c (sm_100a, fp64).
//
// Reference: smoothers.py:203-211 (apply_local_correction) inside the sandwich
// smoother smoothers.py:252-267:  u += S_c (b - A u), where for every region
// d the correction is (L_d L_d^T)^{-1} r[B_d] with L_d the Cholesky factor of
// the principal submatrix A[B_d, B_d] (smoothers.py:176-200, LAPACK dpotrs
// via sparse.py:225-231).
//
// Two kernels, because regions are DOF-disjoint but may be coupled through A
// (SURVEY.md section 8(a) A4): every patch residual must see the
// pre-correction u.
//   patch_residual_kernel  rbuf[k] = b[i] - (A u)[i] for every patch dof
//                          i = dofs[k]; per-row sequential sum in column order
//                          (bit-identical to the reference's full residual
//                          restricted to patch rows).
//   patch_solve_kernel     one CTA per region: forward substitution with the
//                          packed row-major L_d, back substitution with L_d^T,
//                          then u[i] += x (or out[i] = x).  32-wide panels:
//                          off-panel updates are warp-cooperative, coalesced
//                          reads of factor row segments; the panel triangle
//                          is solved by one warp from registers with shuffles.
// Dense solves are tolerance-parity (<= 1e-13 relative vs the oracle), not
// bitwise: LAPACK's blocked order is not reproducible.
#include "smg_internal.cuh"

namespace smg {

__global__ void patch_residual_kernel(const DevCsr a, const int32_t* __restrict__ dofs, int64_t m,
                                      const double* __restrict__ b,
                                      const double* __restrict__ u, double* __restrict__ rbuf)
{
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m) return;
  const int32_t i = dofs[k];
  double sum = 0.0;
  const int64_t e = a.rowptr[i + 1];
  for (int64_t j = a.rowptr[i]; j < e; ++j)
    sum = __dadd_rn(sum, __dmul_rn(a.val[j], __ldg(u + a.col[j])));
  rbuf[k] = __dsub_rn(b[i], sum);
}

__device__ __forceinline__ double warp_sum(double v)
{
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ int64_t tri(int64_t i) { return i * (i + 1) / 2; }

constexpr int kSolveThreads = 256;
constexpr int kSolveWarps = kSolveThreads / 32;

// mode 0: u[dofs] += x ;  mode 1: out[dofs] = x
// kFused: the CTA forms its own patch residual b - A u on its rows first
// (valid when no other region's rows couple to this one through A, checked
// at upload); otherwise the residuals come from patch_residual_kernel (rbuf).
// The packed factor is staged in shared memory when it fits (<= ~236 dofs),
// so the sequential panel solves never wait on HBM/L2; larger factors are
// read through the same generic pointer from global memory.
template <bool kFused>
__global__ void __launch_bounds__(kSolveThreads)
patch_solve_kernel(const DevCsr a, const int32_t* __restrict__ pptr,
                   const int32_t* __restrict__ dofs, const int64_t* __restrict__ foff,
                   const double* __restrict__ lfac, const double* __restrict__ b,
                   const double* u_res, const double* __restrict__ rbuf,
                   double* target, int mode, int64_t smem_tri_cap)
{
  extern __shared__ double s_dyn[];
  __shared__ double s_red[kSolveWarps][32];
  const int p = blockIdx.x;
  const int32_t k0 = pptr[p];
  const int n = pptr[p + 1] - k0;
  const double* __restrict__ Lg = lfac + foff[p];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  double* s_x = s_dyn;
  const int64_t ntri = tri(n);
  const bool staged = ntri <= smem_tri_cap;
  double* s_L = s_dyn + ((n + 1) & ~1);
  const double* L = staged ? s_L : Lg;

  if (staged)
    for (int64_t i = threadIdx.x; i < ntri; i += kSolveThreads) s_L[i] = __ldg(Lg + i);
  if (kFused) {
    for (int i = threadIdx.x; i < n; i += kSolveThreads) {
      const int32_t g = dofs[k0 + i];
      double sum = 0.0;
      const int64_t e = a.rowptr[g + 1];
      for (int64_t j = a.rowptr[g]; j < e; ++j)
        sum = __dadd_rn(sum, __dmul_rn(__ldg(a.val + j), u_res[__ldg(a.col + j)]));
      s_x[i] = __dsub_rn(b[g], sum);
    }
  } else {
    for (int i = threadIdx.x; i < n; i += kSolveThreads) s_x[i] = rbuf[k0 + i];
  }
  __syncthreads();

  // ---- forward: L y = r (left-looking over 32-row panels)
  for (int p0 = 0; p0 < n; p0 += 32) {
    const int pn = min(32, n - p0);
    if (p0 > 0) {
      for (int ii = warp; ii < pn; ii += kSolveWarps) {
        const int i = p0 + ii;
        const double* Li = L + tri(i);
        double acc = 0.0;
        for (int j = lane; j < p0; j += 32) acc += Li[j] * s_x[j];
        acc = warp_sum(acc);
        if (lane == 0) s_x[i] -= acc;
      }
      __syncthreads();
    }
    if (warp == 0) {
      double lrow[32];
      const int i = p0 + lane;
#pragma unroll
      for (int j = 0; j < 32; ++j)
        lrow[j] = (lane < pn && j <= lane) ? L[tri(i) + p0 + j] : 0.0;
      double xi = lane < pn ? s_x[i] : 0.0;
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        if (j < pn) {
          if (lane == j) xi = xi / lrow[j];
          const double yj = __shfl_sync(0xffffffffu, xi, j);
          if (lane > j) xi -= lrow[j] * yj;
        }
      }
      if (lane < pn) s_x[i] = xi;
    }
    __syncthreads();
  }

  // ---- backward: L^T x = y (panels from the bottom)
  const int last = ((n - 1) / 32) * 32;
  for (int p0 = last; p0 >= 0; p0 -= 32) {
    const int pn = min(32, n - p0);
    const int pe = p0 + pn;
    if (pe < n) {
      double acc = 0.0;
      for (int j = pe + warp; j < n; j += kSolveWarps) {
        const double xj = s_x[j];
        if (lane < pn) acc += L[tri(j) + p0 + lane] * xj;
      }
      s_red[warp][lane] = acc;
      __syncthreads();
      if (threadIdx.x < pn) {
        double t = 0.0;
#pragma unroll
        for (int w = 0; w < kSolveWarps; ++w) t += s_red[w][threadIdx.x];
        s_x[p0 + threadIdx.x] -= t;
      }
      __syncthreads();
    }
    if (warp == 0) {
      // lane t holds column t of the panel triangle: lcol[j] = L[p0+j][p0+t], j >= t
      double lcol[32];
#pragma unroll
      for (int j = 0; j < 32; ++j)
        lcol[j] = (lane < pn && j < pn && j >= lane) ? L[tri(p0 + j) + p0 + lane] : 0.0;
      double yt = lane < pn ? s_x[p0 + lane] : 0.0;
#pragma unroll
      for (int j = 31; j >= 0; --j) {
        if (j < pn) {
          if (lane == j) yt = yt / lcol[j];
          const double xj = __shfl_sync(0xffffffffu, yt, j);
          if (lane < j) yt -= lcol[j] * xj;
        }
      }
      if (lane < pn) s_x[p0 + lane] = yt;
    }
    __syncthreads();
  }

  for (int i = threadIdx.x; i < n; i += kSolveThreads) {
    const int32_t g = dofs[k0 + i];
    if (mode == 0)
      target[g] = __dadd_rn(target[g], s_x[i]);
    else
      target[g] = s_x[i];
  }
}

cudaError_t launch_patch_residual(const DevCsr& a, const Correction& c, const double* b,
                                  const double* u, cudaStream_t s)
{
  if (c.m == 0) return cudaSuccess;
  const int threads = 128;
  const int64_t blocks = (c.m + threads - 1) / threads;
  patch_residual_kernel<<<(unsigned)blocks, threads, 0, s>>>(a, c.dofs, c.m, b, u, c.rbuf);
  return cudaGetLastError();
}

__global__ void gather_kernel(const int32_t* __restrict__ idx, int64_t m,
                              const double* __restrict__ src, double* __restrict__ dst)
{
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < m) dst[k] = src[idx[k]];
}

cudaError_t launch_gather(const int32_t* idx, int64_t m, const double* src, double* dst,
                          cudaStream_t s)
{
  if (m == 0) return cudaSuccess;
  gather_kernel<<<(unsigned)((m + 127) / 128), 128, 0, s>>>(idx, m, src, dst);
  return cudaGetLastError();
}

constexpr int64_t kSmemBudget = 220 * 1024;   // dynamic smem per CTA (of 227 KB)

static size_t solve_smem(const Correction& c, int64_t* tri_cap)
{
  const int64_t xb = ((c.max_dofs + 1) & ~1) * (int64_t)sizeof(double);
  int64_t cap = (kSmemBudget - xb) / (int64_t)sizeof(double);
  const int64_t need = (int64_t)c.max_dofs * (c.max_dofs + 1) / 2;
  if (cap < 0) cap = 0;
  *tri_cap = cap;
  const int64_t use = need < cap ? need : cap;
  return (size_t)(xb + use * (int64_t)sizeof(double));
}

// u_add != nullptr -> u += x ; else out_scatter[dofs] = x.  fused: residual in-kernel.
cudaError_t launch_patch_solve(const Correction& c, const double* b, const double* u_res,
                               double* u_add, double* out_scatter, bool fused, cudaStream_t s)
{
  if (c.n_regions == 0) return cudaSuccess;
  int64_t cap = 0;
  const size_t smem = solve_smem(c, &cap);
  const int mode = u_add ? 0 : 1;
  double* tgt = u_add ? u_add : out_scatter;
  if (fused)
    patch_solve_kernel<true><<<c.n_regions, kSolveThreads, smem, s>>>(
        c.op->a, c.pptr, c.dofs, c.foff, c.lfac, b, u_res, c.rbuf, tgt, mode, cap);
  else
    patch_solve_kernel<false><<<c.n_regions, kSolveThreads, smem, s>>>(
        c.op->a, c.pptr, c.dofs, c.foff, c.lfac, b, u_res, c.rbuf, tgt, mode, cap);
  return cudaGetLastError();
}

cudaError_t configure_patch_solve_smem(const Correction& c)
{
  int64_t cap = 0;
  const size_t smem = solve_smem(c, &cap);
  cudaError_t e = cudaFuncSetAttribute(patch_solve_kernel<true>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(patch_solve_kernel<false>,
                              cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

}  // namespace smg
