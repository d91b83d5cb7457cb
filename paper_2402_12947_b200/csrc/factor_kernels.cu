// Batched dense Cholesky of the local-correction blocks on the device.
//
// Reference (paths relative to /root/reference/pkg/src/simplexmg):
// smoothers.py:176-200 build_local_correction extracts each region's principal
// submatrix A[B_d, B_d] (sparse.py:127-130) and factors it with
// dense_factor(lu_fallback=False) (sparse.py:234-254: symmetry check, then
// scipy cho_factor(lower=True) = LAPACK dpotrf; a non-SPD block raises
// NotPositiveDefiniteError).  SURVEY.md section 8(f) rank 1.
//
// One CTA per region (regions are independent): gather the dense block from
// the CSR rows (warp per row, binary search of each column in the region's
// sorted dof list), then a right-looking blocked Cholesky with 32-wide
// panels in global memory (the block stays L2-resident): the 32 x 32 diagonal
// block is factored in shared memory by one warp (left-looking inside the
// block), the panel below it is solved by one thread per row, and the
// trailing lower triangle is updated in 32 x 32 tiles staged in shared
// memory.  Output layout = cho_factor's `c`: L in the lower triangle, the
// untouched strict upper triangle still holding A.  LAPACK's blocked order
// differs, so factors agree to rounding (tests: solves <= 1e-13 relative).
#include "smg_internal.cuh"

namespace smg {

namespace {

constexpr int kFT = 256;   // threads per CTA
constexpr int kFP = 32;    // panel width
constexpr int kFLd = kFP + 1;

__device__ __forceinline__ int find_local(const int32_t* idx, int n, int32_t g)
{
  int lo = 0, hi = n - 1;
  while (lo <= hi) {
    const int mid = (lo + hi) >> 1;
    const int32_t v = idx[mid];
    if (v == g) return mid;
    if (v < g)
      lo = mid + 1;
    else
      hi = mid - 1;
  }
  return -1;
}

__global__ void __launch_bounds__(kFT, 2)
patch_factor_kernel(DevCsr A, const int32_t* pptr, const int32_t* dofs, const int64_t* foff,
                    double* W, int64_t* status, double* sym)
{
  __shared__ double D[kFP][kFLd];
  __shared__ double PI[kFP][kFLd];
  __shared__ double PJ[kFP][kFLd];
  __shared__ double red[2][kFT / 32];
  __shared__ int failed;
  const int r = blockIdx.x;
  const int n = pptr[r + 1] - pptr[r];
  const int32_t* idx = dofs + pptr[r];
  double* w = W + foff[r];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t nn = (int64_t)n * n;
  for (int64_t t = tid; t < nn; t += kFT) w[t] = 0.0;
  if (tid == 0) failed = 0;
  __syncthreads();
  // gather A[B, B] (sparse.py:127-130 principal_submatrix)
  for (int row = warp; row < n; row += kFT / 32) {
    const int32_t g = idx[row];
    for (int64_t kk = A.rowptr[g] + lane; kk < A.rowptr[g + 1]; kk += 32) {
      const int lc = find_local(idx, n, A.col[kk]);
      if (lc >= 0) w[(int64_t)row * n + lc] = A.val[kk];
    }
  }
  __syncthreads();
  // symmetry check inputs (sparse.py:245-247): max |a - a^T|, max |a|
  double dmax = 0.0, amax = 0.0;
  for (int64_t t = tid; t < nn; t += kFT) {
    const int i = (int)(t / n), j = (int)(t % n);
    const double v = w[t];
    amax = fmax(amax, fabs(v));
    if (j > i) dmax = fmax(dmax, fabs(v - w[(int64_t)j * n + i]));
  }
  for (int o = 16; o > 0; o >>= 1) {
    dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
    amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  }
  if (lane == 0) {
    red[0][warp] = dmax;
    red[1][warp] = amax;
  }
  __syncthreads();
  if (tid == 0) {
    double a0 = 0.0, a1 = 0.0;
    for (int k = 0; k < kFT / 32; ++k) {
      a0 = fmax(a0, red[0][k]);
      a1 = fmax(a1, red[1][k]);
    }
    sym[2 * r] = a0;
    sym[2 * r + 1] = a1;
  }
  for (int k0 = 0; k0 < n; k0 += kFP) {
    const int kb = min(kFP, n - k0);
    // (a) diagonal block: factor in shared memory
    for (int t = tid; t < kb * kb; t += kFT) {
      const int i = t / kb, j = t % kb;
      D[i][j] = j <= i ? w[(int64_t)(k0 + i) * n + k0 + j] : 0.0;
    }
    __syncthreads();
    if (warp == 0) {
      for (int j = 0; j < kb; ++j) {
        if (lane >= j && lane < kb) {
          double s = D[lane][j];
          for (int k = 0; k < j; ++k) s -= D[lane][k] * D[j][k];
          D[lane][j] = s;
        }
        __syncwarp();
        const double piv = D[j][j];
        if (!(piv > 0.0)) {  // LAPACK dpotrf: leading minor j+1 not positive (or NaN)
          if (lane == 0) {
            failed = 1;
            status[r] = k0 + j + 1;
          }
          break;
        }
        const double dj = sqrt(piv);
        __syncwarp();
        if (lane == j) D[j][j] = dj;
        if (lane > j && lane < kb) D[lane][j] = D[lane][j] / dj;
        __syncwarp();
      }
    }
    __syncthreads();
    if (failed) return;
    for (int t = tid; t < kb * kb; t += kFT) {
      const int i = t / kb, j = t % kb;
      if (j <= i) w[(int64_t)(k0 + i) * n + k0 + j] = D[i][j];
    }
    // (b) panel below: L21 = A21 L11^-T, one thread per row
    const int r0 = k0 + kb;
    for (int i = r0 + tid; i < n; i += kFT) {
      double* wr = w + (int64_t)i * n + k0;
      for (int j = 0; j < kb; ++j) {
        double s = wr[j];
        for (int k = 0; k < j; ++k) s -= wr[k] * D[j][k];
        wr[j] = s / D[j][j];
      }
    }
    __syncthreads();
    // (c) trailing update of the lower triangle in 32 x 32 tiles
    const int m = n - r0;
    const int T = (m + kFP - 1) / kFP;
    for (int I = 0; I < T; ++I) {
      const int i0 = r0 + I * kFP, ib = min(kFP, n - i0);
      for (int t = tid; t < kFP * kFP; t += kFT) {
        const int i = t / kFP, k = t % kFP;
        PI[i][k] = (i < ib && k < kb) ? w[(int64_t)(i0 + i) * n + k0 + k] : 0.0;
      }
      for (int J = 0; J <= I; ++J) {
        const int j0 = r0 + J * kFP, jb = min(kFP, n - j0);
        __syncthreads();
        for (int t = tid; t < kFP * kFP; t += kFT) {
          const int j = t / kFP, k = t % kFP;
          PJ[j][k] = (j < jb && k < kb) ? w[(int64_t)(j0 + j) * n + k0 + k] : 0.0;
        }
        __syncthreads();
        // thread -> (i, 4 columns)
        const int i = tid >> 3, jq = (tid & 7) * 4;
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll 8
        for (int k = 0; k < kFP; ++k) {
          const double a = PI[i][k];
#pragma unroll
          for (int q = 0; q < 4; ++q) acc[q] += a * PJ[jq + q][k];
        }
        if (i < ib) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int j = jq + q;
            if (j < jb && i0 + i >= j0 + j) w[(int64_t)(i0 + i) * n + j0 + j] -= acc[q];
          }
        }
      }
      __syncthreads();
    }
  }
}

}  // namespace

cudaError_t launch_patch_factor(const DevCsr& a, int64_t n_regions, const int32_t* pptr,
                                const int32_t* dofs, const int64_t* foff, double* w,
                                int64_t* status, double* sym, cudaStream_t s)
{
  if (n_regions == 0) return cudaSuccess;
  patch_factor_kernel<<<(unsigned)n_regions, kFT, 0, s>>>(a, pptr, dofs, foff, w, status, sym);
  return cudaGetLastError();
}

}  // namespace smg
