// Dense Cholesky factor and inverse of the coarsest operator on the device,
// hand-written (no cuSOLVER).
//
// Reference (paths relative to /root/reference/pkg/src/simplexmg): mg.py:123
// coarse_factor = dense_factor(A_L.to_dense()) -> sparse.py:234-254 (symmetry
// check, scipy cho_factor(lower=True) = LAPACK dpotrf, LU fallback when not
// SPD).  The hot path applies A_L^-1 (lower triangle, 64 x 64 tiles), formed
// once at setup as LAPACK dpotri forms it from the factor: L^-1 (dtrtri),
// then L^-T L^-1 (dlauum).  SURVEY.md 8(f) rank 1 ("batched patch/coarse
// Cholesky"): at C4 (n_L = 15,625) this is a 1.27 TFLOP dense factorisation
// plus the inverse.
//
// Storage: row-major n x n.  The factor is cho_factor's `c`: L in the lower
// triangle (diagonal included), the strict upper triangle still holding A.
//
// Blocked algorithms on 64 x 64 tiles (fp64 CUDA-core FMAs; GEMM-shaped work
// at ~0.25 flop per byte of tile traffic from L2):
//   dpotrf (right-looking): for every tile column k
//     1. potrf_diag_kernel   -- one CTA factors the diagonal tile in shared
//        memory (unblocked right-looking Cholesky; the first non-positive
//        pivot is reported as LAPACK's info = its 1-based order);
//     2. trsm_panel_kernel   -- one CTA per tile below: A_ik <- A_ik L_kk^-T;
//     3. syrk_update_kernel  -- one CTA per lower trailing tile:
//        A_ij -= L_ik L_jk^T (k < j <= i; diagonal tiles keep their strict
//        upper half, which holds A).
//   dtrtri (lower, W = L^-1): diagonal tiles inverted independently, then
//     tile diagonals d = 1 .. nb-1 in order, W_ij = -W_ii sum_{k=j}^{i-1} L_ik W_kj
//     (every tile of a diagonal in parallel; it only needs shorter diagonals).
//   dlauum (X = W^T W, lower): X_ij = sum_{k>=i} W_ki^T W_kj, every tile at once,
//     then mirrored to the full symmetric inverse.
// Rounding differs from LAPACK's blocked order; the factor agrees to ~1e-15
// relative and the inverse to ~1e-16 * cond (tests/test_gpu_setup.py).
#include "../../include/simplexmg_b200.h"
#include "smg_internal.cuh"

#include <algorithm>

namespace smg {

namespace {

constexpr int kT = 64;          // tile edge
constexpr int kLd = kT + 1;     // padded shared-memory row stride
constexpr int kGemmThreads = 256;
constexpr int kTwoTiles = 2 * kT * kLd * (int)sizeof(double);   // dynamic smem of the tile kernels

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

// tile (I, J) of the row-major matrix <-> shared memory (rows >= n / cols >= n
// read as 0, never written)
__device__ __forceinline__ void load_tile(double* s, const double* a, int64_t n, int I, int J)
{
  for (int e = threadIdx.x; e < kT * kT; e += blockDim.x) {
    const int r = e / kT, c = e % kT;
    const int64_t gi = (int64_t)I * kT + r, gj = (int64_t)J * kT + c;
    s[r * kLd + c] = (gi < n && gj < n) ? a[gi * n + gj] : 0.0;
  }
}

__device__ __forceinline__ void store_tile(const double* s, double* a, int64_t n, int I, int J,
                                           bool lower_only)
{
  for (int e = threadIdx.x; e < kT * kT; e += blockDim.x) {
    const int r = e / kT, c = e % kT;
    if (lower_only && c > r) continue;
    const int64_t gi = (int64_t)I * kT + r, gj = (int64_t)J * kT + c;
    if (gi < n && gj < n) a[gi * n + gj] = s[r * kLd + c];
  }
}

// 1. factor the diagonal tile k in shared memory
__global__ void __launch_bounds__(kGemmThreads) potrf_diag_kernel(int64_t n, double* a, int k,
                                                                  unsigned long long* info)
{
  __shared__ double s[kT * kLd];
  load_tile(s, a, n, k, k);
  const int kb = (int)((n - (int64_t)k * kT) < kT ? (n - (int64_t)k * kT) : kT);
  __syncthreads();
  for (int j = 0; j < kb; ++j) {
    if (threadIdx.x == 0) {
      const double d = s[j * kLd + j];
      if (!(d > 0.0)) atomicMin(info, (unsigned long long)((int64_t)k * kT + j + 1));
      s[j * kLd + j] = sqrt(d);
    }
    __syncthreads();
    const double djj = s[j * kLd + j];
    for (int i = j + 1 + threadIdx.x; i < kb; i += blockDim.x) s[i * kLd + j] /= djj;
    __syncthreads();
    // trailing lower part of the tile: s[i][l] -= s[i][j] s[l][j], j < l <= i
    const int m = kb - j - 1;
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
      const int i = j + 1 + e / m, l = j + 1 + e % m;
      if (l <= i) s[i * kLd + l] -= s[i * kLd + j] * s[l * kLd + j];
    }
    __syncthreads();
  }
  store_tile(s, a, n, k, k, true);
}

// 2. A_ik <- A_ik L_kk^-T for the tiles below the diagonal (i = k + 1 + blockIdx.x)
__global__ void __launch_bounds__(kGemmThreads) trsm_panel_kernel(int64_t n, double* a, int k)
{
  extern __shared__ double dsm[];
  double* sl = dsm;
  double* sx = dsm + kT * kLd;
  const int i = k + 1 + blockIdx.x;
  load_tile(sl, a, n, k, k);
  load_tile(sx, a, n, i, k);
  __syncthreads();
  const int kb = (int)((n - (int64_t)k * kT) < kT ? (n - (int64_t)k * kT) : kT);
  // row r of X solves x L^T = a_r: x_c = (a_rc - sum_{m<c} x_m L_cm) / L_cc.
  // Four threads per row split the dot product; the row's sequence over c stays serial.
  const int r = threadIdx.x >> 2, q = threadIdx.x & 3;
  for (int c = 0; c < kb; ++c) {
    double acc = 0.0;
    for (int m = q; m < c; m += 4) acc += sx[r * kLd + m] * sl[c * kLd + m];
    acc += __shfl_xor_sync(0xffffffffu, acc, 1);
    acc += __shfl_xor_sync(0xffffffffu, acc, 2);
    if (q == 0) sx[r * kLd + c] = (sx[r * kLd + c] - acc) / sl[c * kLd + c];
    __syncwarp();
  }
  __syncthreads();
  store_tile(sx, a, n, i, k, false);
}

// C (64 x 64 in registers, 4 x 4 per thread) += sign * A B^T over one tile pair
// in shared memory (A, B row-major with stride kLd); transposed_a: A^T B instead
__device__ __forceinline__ void tile_gemm_acc(const double* sa, const double* sb, double c[4][4],
                                              bool transposed_a)
{
  const int tr = (threadIdx.x >> 4) * 4, tc = (threadIdx.x & 15) * 4;
#pragma unroll 4
  for (int m = 0; m < kT; ++m) {
    double av[4], bv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      av[u] = transposed_a ? sa[m * kLd + tr + u] : sa[(tr + u) * kLd + m];
      bv[u] = sb[(tc + u) * kLd + m];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) c[u][v] += av[u] * bv[v];
  }
}

// 3. trailing update A_ij -= L_ik L_jk^T for k < j <= i (tile pairs enumerated
// in the lower trailing triangle)
__global__ void __launch_bounds__(kGemmThreads) syrk_update_kernel(int64_t n, double* a, int k,
                                                                   int nb)
{
  extern __shared__ double dsm[];
  double* si = dsm;
  double* sj = dsm + kT * kLd;
  // t -> (ii, jj) with 0 <= jj <= ii < m, m = nb - k - 1
  const int t = blockIdx.x;
  int ii = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
  while ((ii + 1) * (ii + 2) / 2 <= t) ++ii;
  while (ii * (ii + 1) / 2 > t) --ii;
  const int jj = t - ii * (ii + 1) / 2;
  const int I = k + 1 + ii, J = k + 1 + jj;
  load_tile(si, a, n, I, k);
  load_tile(sj, a, n, J, k);
  __syncthreads();
  double c[4][4] = {};
  tile_gemm_acc(si, sj, c, false);
  const int tr = (threadIdx.x >> 4) * 4, tc = (threadIdx.x & 15) * 4;
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int r = tr + u, cc = tc + v;
      if (I == J && cc > r) continue;   // diagonal tile: the strict upper half holds A
      const int64_t gi = (int64_t)I * kT + r, gj = (int64_t)J * kT + cc;
      if (gi < n && gj < n) a[gi * n + gj] -= c[u][v];
    }
}

// dtrtri, diagonal tiles: W_ii = L_ii^-1 (lower) into w
__global__ void __launch_bounds__(kGemmThreads) trtri_diag_kernel(int64_t n, const double* l,
                                                                  double* w)
{
  extern __shared__ double dsm[];
  double* sl = dsm;
  double* sw = dsm + kT * kLd;
  const int k = blockIdx.x;
  load_tile(sl, l, n, k, k);
  __syncthreads();
  const int kb = (int)((n - (int64_t)k * kT) < kT ? (n - (int64_t)k * kT) : kT);
  // column c of the inverse: forward substitution L w = e_c (thread per column)
  if (threadIdx.x < kT) {
    const int c = threadIdx.x;
    for (int r = 0; r < kT; ++r) {
      double v = 0.0;
      if (r >= c && r < kb) {
        double s = (r == c) ? 1.0 : 0.0;
        for (int m = c; m < r; ++m) s -= sl[r * kLd + m] * sw[m * kLd + c];
        v = s / sl[r * kLd + r];
      }
      sw[r * kLd + c] = v;
    }
  }
  __syncthreads();
  store_tile(sw, w, n, k, k, false);
}

// dtrtri, diagonal d: W_ij = -W_ii sum_{k=j}^{i-1} L_ik W_kj, i = j + d
__global__ void __launch_bounds__(kGemmThreads) trtri_off_kernel(int64_t n, const double* l,
                                                                 double* w, int d)
{
  extern __shared__ double dsm[];
  double* sa = dsm;
  double* sb = dsm + kT * kLd;
  const int J = blockIdx.x, I = J + d;
  double c[4][4] = {};
  for (int k = J; k < I; ++k) {
    load_tile(sa, l, n, I, k);
    load_tile(sb, w, n, k, J);
    __syncthreads();
    // c += L_ik W_kj : A B with B not transposed -> use sb^T layout
    const int tr = (threadIdx.x >> 4) * 4, tc = (threadIdx.x & 15) * 4;
#pragma unroll 4
    for (int m = 0; m < kT; ++m) {
      double av[4], bv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        av[u] = sa[(tr + u) * kLd + m];
        bv[u] = sb[m * kLd + tc + u];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) c[u][v] += av[u] * bv[v];
    }
    __syncthreads();
  }
  // T -> shared, then W_ij = -W_ii T
  const int tr = (threadIdx.x >> 4) * 4, tc = (threadIdx.x & 15) * 4;
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) sb[(tr + u) * kLd + tc + v] = c[u][v];
  load_tile(sa, w, n, I, I);
  __syncthreads();
  double o[4][4] = {};
#pragma unroll 4
  for (int m = 0; m < kT; ++m) {
    double av[4], bv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      av[u] = sa[(tr + u) * kLd + m];
      bv[u] = sb[m * kLd + tc + u];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) o[u][v] += av[u] * bv[v];
  }
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int64_t gi = (int64_t)I * kT + tr + u, gj = (int64_t)J * kT + tc + v;
      if (gi < n && gj < n) w[gi * n + gj] = -o[u][v];
    }
}

// dlauum: X_ij = sum_{k>=i} W_ki^T W_kj (lower tiles, j <= i), into x
__global__ void __launch_bounds__(kGemmThreads) lauum_kernel(int64_t n, const double* w, double* x,
                                                             int nb)
{
  extern __shared__ double dsm[];
  double* sa = dsm;
  double* sb = dsm + kT * kLd;
  const int t = blockIdx.x;
  int I = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
  while ((I + 1) * (I + 2) / 2 <= t) ++I;
  while (I * (I + 1) / 2 > t) --I;
  const int J = t - I * (I + 1) / 2;
  double c[4][4] = {};
  const int tr = (threadIdx.x >> 4) * 4, tc = (threadIdx.x & 15) * 4;
  for (int k = I; k < nb; ++k) {
    load_tile(sa, w, n, k, I);
    load_tile(sb, w, n, k, J);
    __syncthreads();
#pragma unroll 4
    for (int m = 0; m < kT; ++m) {
      double av[4], bv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        av[u] = sa[m * kLd + tr + u];
        bv[u] = sb[m * kLd + tc + u];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) c[u][v] += av[u] * bv[v];
    }
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int r = tr + u, cc = tc + v;
      if (I == J && cc > r) continue;
      const int64_t gi = (int64_t)I * kT + r, gj = (int64_t)J * kT + cc;
      if (gi < n && gj < n) x[gi * n + gj] = c[u][v];
    }
}

__global__ void zero_diag_kernel(int64_t n, const double* l, unsigned long long* info)
{
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && l[i * n + i] == 0.0) atomicMin(info, (unsigned long long)(i + 1));
}

// zero the strict upper triangle of row-major w (W = L^-1 is lower)
__global__ void zero_upper_kernel(int64_t n, double* w)
{
  const int64_t total = n * n;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x)
    if (t % n > t / n) w[t] = 0.0;
}

}  // namespace

int dense_cholesky_device(int64_t n, double* d_a, bool check_symmetry, double* asym,
                          double* amax, int64_t* info_out, bool invert, cudaStream_t s)
{
  *info_out = 0;
  if (n == 0) return SMG_OK;
  if (n >= 46341) return fail("coarse operator too large for the dense factorisation");
  const unsigned grid = 148 * 8;
  const int nb = (int)((n + kT - 1) / kT);
  unsigned long long* d_sym = nullptr;
  unsigned long long* d_info = nullptr;
  double* d_w = nullptr;
  int rc = SMG_OK;
  unsigned long long info = ~0ull;
#define SMG_CC(x)                                        \
  do {                                                   \
    rc = check_cuda((x), #x);                            \
    if (rc != SMG_OK) goto done;                         \
  } while (0)
  {
    static bool attrs = false;
    if (!attrs) {
      SMG_CC(cudaFuncSetAttribute(trsm_panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kTwoTiles));
      SMG_CC(cudaFuncSetAttribute(syrk_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kTwoTiles));
      SMG_CC(cudaFuncSetAttribute(trtri_diag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kTwoTiles));
      SMG_CC(cudaFuncSetAttribute(trtri_off_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kTwoTiles));
      SMG_CC(cudaFuncSetAttribute(lauum_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kTwoTiles));
      attrs = true;
    }
  }
  SMG_CC(cudaMalloc(&d_sym, 2 * sizeof(unsigned long long)));
  SMG_CC(cudaMalloc(&d_info, sizeof(unsigned long long)));
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
  if (!invert) {
    // dpotrf: info = 1-based order of the first non-positive pivot, 0 if SPD
    SMG_CC(cudaMemcpyAsync(d_info, &info, sizeof(info), cudaMemcpyHostToDevice, s));
    for (int k = 0; k < nb; ++k) {
      potrf_diag_kernel<<<1, kGemmThreads, 0, s>>>(n, d_a, k, d_info);
      SMG_CC(cudaGetLastError());
      const int m = nb - k - 1;
      if (m > 0) {
        trsm_panel_kernel<<<m, kGemmThreads, kTwoTiles, s>>>(n, d_a, k);
        SMG_CC(cudaGetLastError());
        syrk_update_kernel<<<(unsigned)(m * (m + 1) / 2), kGemmThreads, kTwoTiles, s>>>(n, d_a, k, nb);
        SMG_CC(cudaGetLastError());
      }
    }
    SMG_CC(cudaMemcpyAsync(&info, d_info, sizeof(info), cudaMemcpyDeviceToHost, s));
    SMG_CC(cudaStreamSynchronize(s));
    *info_out = info == ~0ull ? 0 : (int64_t)info;
  } else {
    // dpotri from the factor in d_a (lower L): W = L^-1, then A^-1 = W^T W.
    // A zero diagonal entry makes L singular: dtrtri's info (1-based order)
    SMG_CC(cudaMemcpyAsync(d_info, &info, sizeof(info), cudaMemcpyHostToDevice, s));
    zero_diag_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, d_a, d_info);
    SMG_CC(cudaGetLastError());
    SMG_CC(cudaMemcpyAsync(&info, d_info, sizeof(info), cudaMemcpyDeviceToHost, s));
    SMG_CC(cudaStreamSynchronize(s));
    if (info != ~0ull) {
      *info_out = (int64_t)info;
      goto done;
    }
    SMG_CC(cudaMalloc(&d_w, sizeof(double) * (size_t)n * (size_t)n));
    zero_upper_kernel<<<grid, 256, 0, s>>>(n, d_w);
    SMG_CC(cudaGetLastError());
    trtri_diag_kernel<<<nb, kGemmThreads, kTwoTiles, s>>>(n, d_a, d_w);
    SMG_CC(cudaGetLastError());
    for (int d = 1; d < nb; ++d) {
      trtri_off_kernel<<<nb - d, kGemmThreads, kTwoTiles, s>>>(n, d_a, d_w, d);
      SMG_CC(cudaGetLastError());
    }
    lauum_kernel<<<(unsigned)((int64_t)nb * (nb + 1) / 2), kGemmThreads, kTwoTiles, s>>>(n, d_w, d_a, nb);
    SMG_CC(cudaGetLastError());
    mirror_lower_kernel<<<grid, 256, 0, s>>>(n, d_a);
    SMG_CC(cudaGetLastError());
    SMG_CC(cudaStreamSynchronize(s));
  }
done:
  cudaFree(d_sym);
  cudaFree(d_info);
  cudaFree(d_w);
#undef SMG_CC
  return rc;
}

}  // namespace smg
