// Dense Cholesky factor and inverse of the coarsest operator on the device.
//
// Reference (paths relative to /root/reference/pkg/src/simplexmg): mg.py:123
// coarse_factor = dense_factor(A_L.to_dense()) -> sparse.py:234-254 (symmetry
// check, scipy cho_factor(lower=True) = LAPACK dpotrf, LU fallback when not
// SPD).  The hot path applies A_L^-1 (lower triangle, 64 x 64 tiles), formed
// once at setup as LAPACK dpotri would from the factor.
// ("batched patch/coarse Cholesky"): at C4 (n_L = 15,625) this is a 1.27
// TFLOP dense factorisation plus the inverse -- a plain library problem, so
// it runs on cuSOLVER (dpotrf / dpotri) like a cuBLAS GEMM would; the small
// kernels here check symmetry and mirror the inverse.
//
// Row-major symmetric A is its own column-major transpose: the UPPER
// column-major factor U (A = U^T U) is the row-major LOWER L, and the other
// triangle is left holding A -- exactly cho_factor's `c` layout.
#include "../../include/simplexmg_b200.h"
#include "smg_internal.cuh"

#include <algorithm>

#include <cusolverDn.h>

namespace smg {

namespace {

__global__ void sym_check_kernel(int64_t n, const double* a, unsigned long long* out)
{
  double dmax = 0.0, amax = 0.0;
  const int64_t total = n * n;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / n, j = t % n;
    const double v = a[t];
    amax = fmax(amax, fabs(v));
    if (j > i) dmax = fmax(dmax, fabs(v - a[j * n + i]));
  }
  for (int o = 16; o > 0; o >>= 1) {
    dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
    amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  }
  if ((threadIdx.x & 31) == 0) {  // non-negative doubles order like their bit patterns
    atomicMax(&out[0], (unsigned long long)__double_as_longlong(dmax));
    atomicMax(&out[1], (unsigned long long)__double_as_longlong(amax));
  }
}

// row-major: copy the lower triangle onto the upper (full symmetric inverse)
__global__ void mirror_lower_kernel(int64_t n, double* a)
{
  const int64_t total = n * n;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / n, j = t % n;
    if (j > i) a[t] = a[j * n + i];
  }
}

const char* solver_status(cusolverStatus_t s)
{
  switch (s) {
    case CUSOLVER_STATUS_SUCCESS: return "success";
    case CUSOLVER_STATUS_NOT_INITIALIZED: return "not initialized";
    case CUSOLVER_STATUS_ALLOC_FAILED: return "alloc failed";
    case CUSOLVER_STATUS_INVALID_VALUE: return "invalid value";
    case CUSOLVER_STATUS_ARCH_MISMATCH: return "arch mismatch";
    case CUSOLVER_STATUS_EXECUTION_FAILED: return "execution failed";
    case CUSOLVER_STATUS_INTERNAL_ERROR: return "internal error";
    default: return "error";
  }
}

}  // namespace

int dense_cholesky_device(int64_t n, double* d_a, bool check_symmetry, double* asym,
                          double* amax, int64_t* info_out, bool invert, cudaStream_t s)
{
  *info_out = 0;
  if (n == 0) return SMG_OK;
  if (n >= 46341) return fail("coarse operator too large for the dense factorisation");
  const unsigned grid = 148 * 8;
  unsigned long long* d_sym = nullptr;
  int* d_info = nullptr;
  double* d_work = nullptr;
  cusolverDnHandle_t h = nullptr;
  int rc = SMG_OK;
  int lwork = 0, info = 0;
  cusolverStatus_t st;
#define SMG_CS(x)                                                                        \
  do {                                                                                   \
    st = (x);                                                                            \
    if (st != CUSOLVER_STATUS_SUCCESS) {                                                 \
      rc = fail(std::string("cuSOLVER ") + #x + ": " + solver_status(st));               \
      goto done;                                                                         \
    }                                                                                    \
  } while (0)
#define SMG_CC(x)                                        \
  do {                                                   \
    rc = check_cuda((x), #x);                            \
    if (rc != SMG_OK) goto done;                         \
  } while (0)
  SMG_CC(cudaMalloc(&d_sym, 2 * sizeof(unsigned long long)));
  SMG_CC(cudaMalloc(&d_info, sizeof(int)));
  if (check_symmetry) {
    unsigned long long hs[2] = {0, 0};
    SMG_CC(cudaMemsetAsync(d_sym, 0, 2 * sizeof(unsigned long long), s));
    sym_check_kernel<<<grid, 256, 0, s>>>(n, d_a, d_sym);
    SMG_CC(cudaGetLastError());
    SMG_CC(cudaMemcpyAsync(hs, d_sym, sizeof(hs), cudaMemcpyDeviceToHost, s));
    SMG_CC(cudaStreamSynchronize(s));
    *asym = __builtin_bit_cast(double, hs[0]);
    *amax = __builtin_bit_cast(double, hs[1]);
    if (*amax != 0.0 && *asym > 1e-10 * *amax) goto done;  // caller reports ValueError
  }
  SMG_CS(cusolverDnCreate(&h));
  SMG_CS(cusolverDnSetStream(h, s));
  if (!invert) {
    SMG_CS(cusolverDnDpotrf_bufferSize(h, CUBLAS_FILL_MODE_UPPER, (int)n, d_a, (int)n, &lwork));
  } else {
    SMG_CS(cusolverDnDpotri_bufferSize(h, CUBLAS_FILL_MODE_UPPER, (int)n, d_a, (int)n, &lwork));
  }
  SMG_CC(cudaMalloc(&d_work, sizeof(double) * (size_t)std::max(lwork, 1)));
  if (!invert) {
    SMG_CS(cusolverDnDpotrf(h, CUBLAS_FILL_MODE_UPPER, (int)n, d_a, (int)n, d_work, lwork, d_info));
  } else {
    SMG_CS(cusolverDnDpotri(h, CUBLAS_FILL_MODE_UPPER, (int)n, d_a, (int)n, d_work, lwork, d_info));
  }
  SMG_CC(cudaMemcpyAsync(&info, d_info, sizeof(int), cudaMemcpyDeviceToHost, s));
  SMG_CC(cudaStreamSynchronize(s));
  *info_out = info;
  if (invert && info == 0) {
    mirror_lower_kernel<<<grid, 256, 0, s>>>(n, d_a);
    SMG_CC(cudaGetLastError());
    SMG_CC(cudaStreamSynchronize(s));
  }
done:
  if (h) cusolverDnDestroy(h);
  cudaFree(d_sym);
  cudaFree(d_info);
  cudaFree(d_work);
#undef SMG_CS
#undef SMG_CC
  return rc;
}

}  // namespace smg
