// Prolongation construction on the device: point location of every fine DOF
// in the coarse mesh and the coarse Lagrange basis evaluated there.
//
// Reference (paths relative to /root/reference/pkg/src/simplexmg):
// transfer.py:117-150 build_prolongation, a Python loop over fine DOFs that
// calls CellLocator.locate (:73-91) -- candidates from a uniform bin of the
// coarse cells' padded bounding boxes, tested in ascending cell order; the
// first cell whose barycentric coordinates are all >= -tol wins (the
// lowest-index tie rule); with no hit in the bin every cell is scanned; no
// hit at all raises PointLocationError.  The winner's coordinates are clamped
// to [0, 1] and renormalised, the basis is evaluated at bary[1:]
// (reference_basis, fem.py:43-60: vertices first, then edges) and values
// with |v| <= drop_tol are dropped.  SURVEY.md section 8(f) rank 3.
//
// Bitwise parity: the barycentric coordinates follow numpy's own arithmetic
// for `einsum("med,md->me", inv_jac[cells], x - v0[cells])` (2D: P0 + P1;
// 3D: (P0 + P2) + P1 -- numpy's two-lane SIMD sum of products, measured) and
// `1 - local.sum(axis=1)` / `clamped.sum()` (sequential), with the inverse
// Jacobians computed by numpy on the host exactly as the reference does
// (np.linalg.inv), so every P value equals the reference's bit for bit.
//
// One thread per fine DOF (integer/latency work, a few hundred bytes per
// point): each thread writes its sorted row into a fixed-stride slot, then a
// scan of the row lengths and a compaction give canonical CSR.
#include "smg_internal.cuh"

#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <vector>

namespace smg {

namespace {

template <int DIM>
__device__ __forceinline__ void barycentric(const LocateArgs& a, int64_t c, const double* x,
                                            double* bary)
{
  double diff[DIM];
#pragma unroll
  for (int d = 0; d < DIM; ++d) diff[d] = __dsub_rn(x[d], a.v0[c * DIM + d]);
  double loc[DIM];
  const double* inv = a.inv_jac + c * DIM * DIM;
#pragma unroll
  for (int e = 0; e < DIM; ++e) {
    const double p0 = __dmul_rn(inv[e * DIM + 0], diff[0]);
    const double p1 = __dmul_rn(inv[e * DIM + 1], diff[1]);
    if constexpr (DIM == 2) {
      loc[e] = __dadd_rn(p0, p1);
    } else {
      const double p2 = __dmul_rn(inv[e * DIM + 2], diff[2]);
      loc[e] = __dadd_rn(__dadd_rn(p0, p2), p1);
    }
  }
  double s = loc[0];
#pragma unroll
  for (int e = 1; e < DIM; ++e) s = __dadd_rn(s, loc[e]);
  bary[0] = __dsub_rn(1.0, s);
#pragma unroll
  for (int e = 0; e < DIM; ++e) bary[1 + e] = loc[e];
}

template <int DIM>
__device__ __forceinline__ bool inside(const double* bary, double tol)
{
  double mn = bary[0];
#pragma unroll
  for (int e = 1; e <= DIM; ++e) mn = fmin(mn, bary[e]);
  return mn >= -tol;
}

template <int DIM, int DEG>
__global__ void __launch_bounds__(256)
prolong_rows_kernel(LocateArgs a, int32_t* row_len, int32_t* cols, double* vals,
                    unsigned long long* fail)
{
  constexpr int NPC = DEG == 1 ? DIM + 1 : (DIM + 1) * (DIM + 2) / 2;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n_points) return;
  double x[DIM];
  int64_t key = 0, stride = 1;
#pragma unroll
  for (int d = 0; d < DIM; ++d) {
    x[d] = a.points[i * DIM + d];
    const double q = fmin(fmax(x[d], a.lo[d]), a.hi[d]);  // np.clip(x, lo, hi)
    int64_t b = (int64_t)__dmul_rn(__dsub_rn(q, a.lo[d]), a.scale[d]);
    b = b < 0 ? 0 : (b > a.nb - 1 ? a.nb - 1 : b);
    key += b * stride;
    stride *= a.nb;
  }
  double bary[DIM + 1];
  int64_t cell = -1;
  for (int64_t k = a.bin_ptr[key]; k < a.bin_ptr[key + 1]; ++k) {
    const int64_t c = a.bin_cells[k];
    barycentric<DIM>(a, c, x, bary);
    if (inside<DIM>(bary, a.tol)) {
      cell = c;
      break;
    }
  }
  if (cell < 0) {  // transfer.py:81-82: scan every cell in ascending order
    for (int64_t c = 0; c < a.n_cells; ++c) {
      barycentric<DIM>(a, c, x, bary);
      if (inside<DIM>(bary, a.tol)) {
        cell = c;
        break;
      }
    }
  }
  if (cell < 0) {
    atomicMin(fail, (unsigned long long)i);
    row_len[i] = 0;
    return;
  }
  // clamp to [0, 1] and renormalise (transfer.py:88-89)
  double sum = 0.0;
#pragma unroll
  for (int e = 0; e <= DIM; ++e) {
    bary[e] = fmin(fmax(bary[e], 0.0), 1.0);
    sum = e == 0 ? bary[0] : __dadd_rn(sum, bary[e]);
  }
#pragma unroll
  for (int e = 0; e <= DIM; ++e) bary[e] = __ddiv_rn(bary[e], sum);
  // basis at point = bary[1:] (fem.py:43-60 via reference_basis): lam0 = 1 - sum(point)
  double lam[DIM + 1];
  double ps = bary[1];
#pragma unroll
  for (int e = 2; e <= DIM; ++e) ps = __dadd_rn(ps, bary[e]);
  lam[0] = __dsub_rn(1.0, ps);
#pragma unroll
  for (int e = 1; e <= DIM; ++e) lam[e] = bary[e];
  double v[NPC];
  if constexpr (DEG == 1) {
#pragma unroll
    for (int e = 0; e <= DIM; ++e) v[e] = lam[e];
  } else {
#pragma unroll
    for (int e = 0; e <= DIM; ++e) v[e] = __dmul_rn(lam[e], __dsub_rn(__dmul_rn(2.0, lam[e]), 1.0));
    int t = DIM + 1;
#pragma unroll
    for (int p = 0; p <= DIM; ++p)
#pragma unroll
      for (int q = p + 1; q <= DIM; ++q) v[t++] = __dmul_rn(__dmul_rn(4.0, lam[p]), lam[q]);
  }
  // keep |v| > drop_tol, sorted by coarse node (canonical CSR row)
  int32_t nc[NPC];
  double nv[NPC];
  int n = 0;
#pragma unroll
  for (int t = 0; t < NPC; ++t) {
    if (fabs(v[t]) > a.drop_tol) {
      const int32_t node = (int32_t)a.cell_nodes[cell * NPC + t];
      int p = n++;
      while (p > 0 && nc[p - 1] > node) {
        nc[p] = nc[p - 1];
        nv[p] = nv[p - 1];
        --p;
      }
      nc[p] = node;
      nv[p] = v[t];
    }
  }
  for (int t = 0; t < n; ++t) {
    cols[i * NPC + t] = nc[t];
    vals[i * NPC + t] = nv[t];
  }
  row_len[i] = n;
}

__global__ void widen_rows_kernel(const int32_t* in, int64_t n, int64_t* out)
{
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = in[i];
}

__global__ void compact_fixed_kernel(int64_t n, int stride, const int32_t* cols, const double* vals,
                                     const int64_t* ptr, int32_t* col, double* val)
{
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t dst = ptr[i], len = ptr[i + 1] - dst;
  for (int64_t t = 0; t < len; ++t) {
    col[dst + t] = cols[i * stride + t];
    val[dst + t] = vals[i * stride + t];
  }
}

}  // namespace

cudaError_t prolongation_device(const LocateArgs& a, int dim, int degree, DevCsrOwned* out,
                                int64_t* failed_point, cudaStream_t s)
{
  cudaError_t e;
#define SMG_T(x)                            \
  do {                                      \
    if ((e = (x)) != cudaSuccess) goto done; \
  } while (0)
  const int npc = degree == 1 ? dim + 1 : (dim + 1) * (dim + 2) / 2;
  const int64_t n = a.n_points;
  int32_t* len = nullptr;
  int32_t* cols = nullptr;
  double* vals = nullptr;
  int64_t* wide = nullptr;
  unsigned long long* fail = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  unsigned long long h_fail = 0;
  const unsigned grid = (unsigned)((n + 255) / 256);
  *failed_point = -1;
  out->nrows = n;
  out->ncols = a.n_coarse;
  SMG_T(cudaMalloc(&len, sizeof(int32_t) * std::max<int64_t>(n, 1)));
  SMG_T(cudaMalloc(&cols, sizeof(int32_t) * std::max<int64_t>(n * npc, 1)));
  SMG_T(cudaMalloc(&vals, sizeof(double) * std::max<int64_t>(n * npc, 1)));
  SMG_T(cudaMalloc(&wide, sizeof(int64_t) * std::max<int64_t>(n, 1)));
  SMG_T(cudaMalloc(&fail, sizeof(unsigned long long)));
  h_fail = (unsigned long long)n;
  SMG_T(cudaMemcpyAsync(fail, &h_fail, sizeof(h_fail), cudaMemcpyHostToDevice, s));
  if (n > 0) {
    if (dim == 2 && degree == 1)
      prolong_rows_kernel<2, 1><<<grid, 256, 0, s>>>(a, len, cols, vals, fail);
    else if (dim == 2 && degree == 2)
      prolong_rows_kernel<2, 2><<<grid, 256, 0, s>>>(a, len, cols, vals, fail);
    else if (dim == 3 && degree == 1)
      prolong_rows_kernel<3, 1><<<grid, 256, 0, s>>>(a, len, cols, vals, fail);
    else
      prolong_rows_kernel<3, 2><<<grid, 256, 0, s>>>(a, len, cols, vals, fail);
    SMG_T(cudaGetLastError());
    widen_rows_kernel<<<grid, 256, 0, s>>>(len, n, wide);
    SMG_T(cudaGetLastError());
  }
  SMG_T(cudaMemcpyAsync(&h_fail, fail, sizeof(h_fail), cudaMemcpyDeviceToHost, s));
  SMG_T(cudaMalloc(&out->rowptr, sizeof(int64_t) * (size_t)(n + 1)));
  SMG_T(cudaMemsetAsync(out->rowptr, 0, sizeof(int64_t), s));
  if (n > 0) {
    SMG_T(cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, wide, out->rowptr + 1, n, s));
    SMG_T(cudaMalloc(&tmp, tmp_bytes));
    SMG_T(cub::DeviceScan::InclusiveSum(tmp, tmp_bytes, wide, out->rowptr + 1, n, s));
  }
  SMG_T(cudaMemcpyAsync(&out->nnz, out->rowptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  SMG_T(cudaStreamSynchronize(s));
  if (h_fail < (unsigned long long)n) {
    *failed_point = (int64_t)h_fail;
    goto done;
  }
  SMG_T(cudaMalloc(&out->col, sizeof(int32_t) * (size_t)std::max<int64_t>(out->nnz, 1)));
  SMG_T(cudaMalloc(&out->val, sizeof(double) * (size_t)std::max<int64_t>(out->nnz, 1)));
  if (n > 0) {
    compact_fixed_kernel<<<grid, 256, 0, s>>>(n, npc, cols, vals, out->rowptr, out->col, out->val);
    SMG_T(cudaGetLastError());
  }
  SMG_T(cudaStreamSynchronize(s));
done:
  cudaFree(len);
  cudaFree(cols);
  cudaFree(vals);
  cudaFree(wide);
  cudaFree(fail);
  cudaFree(tmp);
#undef SMG_T
  return e;
}

}  // namespace smg
