// Element matrices -> canonical CSR on the device, in scipy's exact order.
//
// Reference (relative to /root/reference/pkg/src/simplexmg): fem.py:339-345
//   rows = np.repeat(cell_dofs, nloc, axis=1).ravel()
//   cols = np.tile(cell_dofs, (1, nloc)).ravel()
//   stiffness = sp.coo_matrix((local.ravel(), (rows, cols))).tocsr()
// then the symmetric Dirichlet elimination fem.py:362-375 (rows and columns of
// the Dirichlet dofs dropped, a unit diagonal in their place; CsrMatrix
// .from_coo keeps values as they are).
//
// scipy's tocsr (coo_tocsr + sum_duplicates, observed on scipy 1.18 and pinned
// by tests/test_setup.py::test_scipy_duplicate_order) does:
//   1. bucket the entries by row, keeping their input order;
//   2. if any row is not already non-decreasing in its columns, run
//      std::sort (libstdc++ introsort: median-of-three quicksort down to
//      16-element runs, heapsort past 2*floor(log2 n) levels, final insertion
//      sort) on EVERY row's (column, value) pairs, comparing columns only --
//      so duplicates of one column end up in an order fixed by that algorithm;
//   3. add each run of equal columns sequentially, in that order.
// The element values come from the host (numpy's own einsum / LAPACK det and
// inv, the reference's arithmetic, fem.py:317-322), so the result is the
// reference's matrix bit for bit; this file only moves steps 1-3 and the
// elimination to the GPU: a stable radix sort by row (step 1), one thread per
// row running the same introsort on its segment (step 2) and summing its runs
// with __dadd_rn (step 3), then the elimination and a compaction.
#include "../../include/simplexmg_b200.h"
#include "smg_internal.cuh"

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>

namespace smg {

namespace coo_sort {

// ---- libstdc++ std::sort on (column, value) pairs, comparing columns only
// (bits/stl_algo.h / stl_heap.h, GCC 14; verified against scipy on random rows)
struct Seg {
  int32_t* c;
  double* v;
  __host__ __device__ __forceinline__ void swap(int64_t a, int64_t b)
  {
    const int32_t tc = c[a];
    c[a] = c[b];
    c[b] = tc;
    const double tv = v[a];
    v[a] = v[b];
    v[b] = tv;
  }
};

__host__ __device__ int lg2(int64_t n)
{
  int r = 0;
  while (n > 1) {
    n >>= 1;
    ++r;
  }
  return r;
}

__host__ __device__ void move_median_to_first(Seg s, int64_t result, int64_t a, int64_t b, int64_t c)
{
  if (s.c[a] < s.c[b]) {
    if (s.c[b] < s.c[c])
      s.swap(result, b);
    else if (s.c[a] < s.c[c])
      s.swap(result, c);
    else
      s.swap(result, a);
  } else if (s.c[a] < s.c[c]) {
    s.swap(result, a);
  } else if (s.c[b] < s.c[c]) {
    s.swap(result, c);
  } else {
    s.swap(result, b);
  }
}

__host__ __device__ int64_t unguarded_partition(Seg s, int64_t first, int64_t last, int64_t pivot)
{
  while (true) {
    while (s.c[first] < s.c[pivot]) ++first;
    --last;
    while (s.c[pivot] < s.c[last]) --last;
    if (!(first < last)) return first;
    s.swap(first, last);
    ++first;
  }
}

__host__ __device__ void adjust_heap(Seg s, int64_t first, int64_t hole, int64_t len, int32_t vc, double vv)
{
  const int64_t top = hole;
  int64_t child = hole;
  while (child < (len - 1) / 2) {
    child = 2 * (child + 1);
    if (s.c[first + child] < s.c[first + child - 1]) --child;
    s.c[first + hole] = s.c[first + child];
    s.v[first + hole] = s.v[first + child];
    hole = child;
  }
  if ((len & 1) == 0 && child == (len - 2) / 2) {
    child = 2 * (child + 1);
    s.c[first + hole] = s.c[first + child - 1];
    s.v[first + hole] = s.v[first + child - 1];
    hole = child - 1;
  }
  // __push_heap
  int64_t parent = (hole - 1) / 2;
  while (hole > top && s.c[first + parent] < vc) {
    s.c[first + hole] = s.c[first + parent];
    s.v[first + hole] = s.v[first + parent];
    hole = parent;
    parent = (hole - 1) / 2;
  }
  s.c[first + hole] = vc;
  s.v[first + hole] = vv;
}

__host__ __device__ void heap_sort_range(Seg s, int64_t first, int64_t last)
{
  // __partial_sort(first, last, last) = __heap_select (== make_heap here) + __sort_heap
  const int64_t len = last - first;
  if (len >= 2) {
    int64_t parent = (len - 2) / 2;
    while (true) {
      adjust_heap(s, first, parent, len, s.c[first + parent], s.v[first + parent]);
      if (parent == 0) break;
      --parent;
    }
  }
  while (last - first > 1) {
    --last;
    const int32_t vc = s.c[last];
    const double vv = s.v[last];
    s.c[last] = s.c[first];
    s.v[last] = s.v[first];
    adjust_heap(s, first, 0, last - first, vc, vv);
  }
}

__host__ __device__ void unguarded_linear_insert(Seg s, int64_t last)
{
  const int32_t vc = s.c[last];
  const double vv = s.v[last];
  int64_t next = last - 1;
  while (vc < s.c[next]) {
    s.c[last] = s.c[next];
    s.v[last] = s.v[next];
    last = next;
    --next;
  }
  s.c[last] = vc;
  s.v[last] = vv;
}

__host__ __device__ void insertion_sort(Seg s, int64_t first, int64_t last)
{
  if (first == last) return;
  for (int64_t i = first + 1; i != last; ++i) {
    if (s.c[i] < s.c[first]) {
      const int32_t vc = s.c[i];
      const double vv = s.v[i];
      for (int64_t k = i; k > first; --k) {   // move_backward(first, i, i + 1)
        s.c[k] = s.c[k - 1];
        s.v[k] = s.v[k - 1];
      }
      s.c[first] = vc;
      s.v[first] = vv;
    } else {
      unguarded_linear_insert(s, i);
    }
  }
}

constexpr int64_t kSThreshold = 16;

__host__ __device__ void std_sort(Seg s, int64_t n)
{
  if (n < 2) return;
  // __introsort_loop with an explicit stack for its right-hand recursion
  int64_t st_first[64], st_last[64];
  int st_depth[64];
  int top = 0;
  st_first[0] = 0;
  st_last[0] = n;
  st_depth[0] = 2 * lg2(n);
  top = 1;
  while (top > 0) {
    --top;
    int64_t first = st_first[top], last = st_last[top];
    int depth = st_depth[top];
    while (last - first > kSThreshold) {
      if (depth == 0) {
        heap_sort_range(s, first, last);
        break;
      }
      --depth;
      const int64_t mid = first + (last - first) / 2;
      move_median_to_first(s, first, first + 1, mid, last - 1);
      const int64_t cut = unguarded_partition(s, first + 1, last, first);
      // the reference recurses on [cut, last) first, then loops on [first, cut):
      // the two ranges are disjoint, so the order in which they are processed
      // does not change the result; push the right part, continue on the left
      st_first[top] = cut;
      st_last[top] = last;
      st_depth[top] = depth;
      ++top;
      last = cut;
    }
  }
  // __final_insertion_sort
  if (n > kSThreshold) {
    insertion_sort(s, 0, kSThreshold);
    for (int64_t i = kSThreshold; i < n; ++i) unguarded_linear_insert(s, i);
  } else {
    insertion_sort(s, 0, n);
  }
}

}  // namespace coo_sort

namespace {
using coo_sort::Seg;
using coo_sort::std_sort;

// ---- pipeline kernels
__global__ void coo_row_keys_kernel(int64_t ne, int nloc, const int64_t* __restrict__ cell_dofs,
                                    uint32_t* keys, uint32_t* idx)
{
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= ne) return;
  const int64_t nn = (int64_t)nloc * nloc;
  const int64_t c = t / nn;
  const int i = (int)((t - c * nn) / nloc);
  keys[t] = (uint32_t)cell_dofs[c * nloc + i];
  idx[t] = (uint32_t)t;
}

__global__ void coo_gather_kernel(int64_t ne, int nloc, const int64_t* __restrict__ cell_dofs,
                                  const double* __restrict__ local, const uint32_t* __restrict__ sidx,
                                  int32_t* col, double* val)
{
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= ne) return;
  const int64_t t = sidx[p];
  const int64_t c = t / nloc / nloc;
  const int j = (int)(t % nloc);
  col[p] = (int32_t)cell_dofs[c * nloc + j];
  val[p] = local[t];
}

__global__ void coo_rowptr_kernel(int64_t n, int64_t ne, const uint32_t* __restrict__ skeys,
                                  int64_t* rowptr)
{
  const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (row > n) return;
  int64_t lo = 0, hi = ne;   // first sorted key >= row
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if ((int64_t)skeys[mid] < row)
      lo = mid + 1;
    else
      hi = mid;
  }
  rowptr[row] = lo;
}

__global__ void coo_sorted_check_kernel(int64_t n, const int64_t* __restrict__ rowptr,
                                        const int32_t* __restrict__ col, int* unsorted)
{
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  for (int64_t p = rowptr[r]; p + 1 < rowptr[r + 1]; ++p)
    if (col[p] > col[p + 1]) {
      atomicOr(unsorted, 1);
      return;
    }
}

// sort (if any row is unsorted), sum runs in place; count what survives the
// Dirichlet elimination (Dirichlet rows keep only their unit diagonal)
__global__ void coo_row_sum_kernel(int64_t n, const int64_t* __restrict__ rowptr, int32_t* col,
                                   double* val, const int* __restrict__ unsorted,
                                   const uint8_t* __restrict__ dir, int64_t* ucount,
                                   int64_t* kcount)
{
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int64_t p0 = rowptr[r], len = rowptr[r + 1] - p0;
  Seg s{col + p0, val + p0};
  if (*unsorted) std_sort(s, len);
  int64_t w = 0, kept = 0;
  int64_t j = 0;
  while (j < len) {
    const int32_t c = s.c[j];
    double x = s.v[j];
    ++j;
    while (j < len && s.c[j] == c) {
      x = __dadd_rn(x, s.v[j]);
      ++j;
    }
    s.c[w] = c;
    s.v[w] = x;
    ++w;
    if (dir == nullptr || !dir[c]) ++kept;
  }
  ucount[r] = w;
  kcount[r] = (dir != nullptr && dir[r]) ? 1 : kept;
}

__global__ void coo_write_kernel(int64_t n, const int64_t* __restrict__ rowptr,
                                 const int32_t* __restrict__ col, const double* __restrict__ val,
                                 const int64_t* __restrict__ ucount, const uint8_t* __restrict__ dir,
                                 const int64_t* __restrict__ out_ptr, int32_t* out_col,
                                 double* out_val)
{
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  int64_t o = out_ptr[r];
  if (dir != nullptr && dir[r]) {
    out_col[o] = (int32_t)r;
    out_val[o] = 1.0;
    return;
  }
  const int64_t p0 = rowptr[r];
  for (int64_t k = 0; k < ucount[r]; ++k) {
    const int32_t c = col[p0 + k];
    if (dir != nullptr && dir[c]) continue;
    out_col[o] = c;
    out_val[o] = val[p0 + k];
    ++o;
  }
}

}  // namespace

int assemble_elements_device(int64_t n_dofs, int64_t n_cells, int nloc, const int64_t* cell_dofs,
                             const double* local, const uint8_t* dirichlet_mask, DevCsrOwned* out,
                             cudaStream_t s)
{
  const int64_t ne = n_cells * nloc * nloc;
  int rc = SMG_OK;
  int64_t *d_dofs = nullptr, *rowptr = nullptr, *ucount = nullptr, *kcount = nullptr;
  double *d_local = nullptr, *val = nullptr;
  uint32_t *k_in = nullptr, *k_out = nullptr, *i_in = nullptr, *i_out = nullptr;
  int32_t* col = nullptr;
  uint8_t* d_dir = nullptr;
  int* d_unsorted = nullptr;
  void* tmp = nullptr;
  size_t tb = 0, tmp_bytes = 0;
  int end_bit = 1;
  while (end_bit < 32 && (1ll << end_bit) < n_dofs) ++end_bit;
  const unsigned ge = (unsigned)((ne + 255) / 256);
  const unsigned gr = (unsigned)((n_dofs + 1 + 255) / 256);
  out->nrows = n_dofs;
  out->ncols = n_dofs;
#define SMG_E(x)                          \
  do {                                    \
    rc = check_cuda((x), #x);             \
    if (rc != SMG_OK) goto done;          \
  } while (0)
  SMG_E(cudaMalloc(&d_dofs, sizeof(int64_t) * (size_t)std::max<int64_t>(n_cells * nloc, 1)));
  SMG_E(cudaMalloc(&d_local, sizeof(double) * (size_t)std::max<int64_t>(ne, 1)));
  SMG_E(cudaMalloc(&k_in, sizeof(uint32_t) * (size_t)std::max<int64_t>(ne, 1)));
  SMG_E(cudaMalloc(&k_out, sizeof(uint32_t) * (size_t)std::max<int64_t>(ne, 1)));
  SMG_E(cudaMalloc(&i_in, sizeof(uint32_t) * (size_t)std::max<int64_t>(ne, 1)));
  SMG_E(cudaMalloc(&i_out, sizeof(uint32_t) * (size_t)std::max<int64_t>(ne, 1)));
  SMG_E(cudaMalloc(&rowptr, sizeof(int64_t) * (size_t)(n_dofs + 1)));
  SMG_E(cudaMalloc(&ucount, sizeof(int64_t) * (size_t)(n_dofs + 1)));
  SMG_E(cudaMalloc(&kcount, sizeof(int64_t) * (size_t)(n_dofs + 1)));
  SMG_E(cudaMalloc(&d_unsorted, sizeof(int)));
  SMG_E(cudaMemsetAsync(d_unsorted, 0, sizeof(int), s));
  if (dirichlet_mask) {
    SMG_E(cudaMalloc(&d_dir, (size_t)std::max<int64_t>(n_dofs, 1)));
    SMG_E(cudaMemcpyAsync(d_dir, dirichlet_mask, (size_t)n_dofs, cudaMemcpyHostToDevice, s));
  }
  SMG_E(cudaMemcpyAsync(d_dofs, cell_dofs, sizeof(int64_t) * (size_t)(n_cells * nloc),
                        cudaMemcpyHostToDevice, s));
  SMG_E(cudaMemcpyAsync(d_local, local, sizeof(double) * (size_t)ne, cudaMemcpyHostToDevice, s));
  if (ne > 0) {
    coo_row_keys_kernel<<<ge, 256, 0, s>>>(ne, nloc, d_dofs, k_in, i_in);
    SMG_E(cudaGetLastError());
    // stable LSD radix sort by row: each row's entries stay in input order
    SMG_E(cub::DeviceRadixSort::SortPairs(nullptr, tb, k_in, k_out, i_in, i_out, ne, 0, end_bit, s));
    tmp_bytes = tb;
    SMG_E(cudaMalloc(&tmp, tmp_bytes));
    SMG_E(cub::DeviceRadixSort::SortPairs(tmp, tb, k_in, k_out, i_in, i_out, ne, 0, end_bit, s));
    cudaFree(tmp);
    tmp = nullptr;
    cudaFree(k_in);
    k_in = nullptr;
    cudaFree(i_in);
    i_in = nullptr;
  }
  SMG_E(cudaMalloc(&col, sizeof(int32_t) * (size_t)std::max<int64_t>(ne, 1)));
  SMG_E(cudaMalloc(&val, sizeof(double) * (size_t)std::max<int64_t>(ne, 1)));
  if (ne > 0) {
    coo_gather_kernel<<<ge, 256, 0, s>>>(ne, nloc, d_dofs, d_local, i_out, col, val);
    SMG_E(cudaGetLastError());
  }
  coo_rowptr_kernel<<<gr, 256, 0, s>>>(n_dofs, ne, k_out, rowptr);
  SMG_E(cudaGetLastError());
  coo_sorted_check_kernel<<<gr, 256, 0, s>>>(n_dofs, rowptr, col, d_unsorted);
  SMG_E(cudaGetLastError());
  coo_row_sum_kernel<<<(unsigned)((n_dofs + 127) / 128), 128, 0, s>>>(n_dofs, rowptr, col, val,
                                                                 d_unsorted, d_dir, ucount, kcount);
  SMG_E(cudaGetLastError());
  SMG_E(cudaMalloc(&out->rowptr, sizeof(int64_t) * (size_t)(n_dofs + 1)));
  // out_ptr = exclusive scan of kcount (n_dofs + 1 entries: kcount[n] = 0)
  SMG_E(cudaMemsetAsync(kcount + n_dofs, 0, sizeof(int64_t), s));
  tb = 0;
  SMG_E(cub::DeviceScan::ExclusiveSum(nullptr, tb, kcount, out->rowptr, n_dofs + 1, s));
  SMG_E(cudaMalloc(&tmp, tb));
  SMG_E(cub::DeviceScan::ExclusiveSum(tmp, tb, kcount, out->rowptr, n_dofs + 1, s));
  SMG_E(cudaMemcpyAsync(&out->nnz, out->rowptr + n_dofs, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  SMG_E(cudaStreamSynchronize(s));
  SMG_E(cudaMalloc(&out->col, sizeof(int32_t) * (size_t)std::max<int64_t>(out->nnz, 1)));
  SMG_E(cudaMalloc(&out->val, sizeof(double) * (size_t)std::max<int64_t>(out->nnz, 1)));
  coo_write_kernel<<<gr, 256, 0, s>>>(n_dofs, rowptr, col, val, ucount, d_dir, out->rowptr,
                                      out->col, out->val);
  SMG_E(cudaGetLastError());
  SMG_E(cudaStreamSynchronize(s));
done:
  cudaFree(d_dofs);
  cudaFree(d_local);
  cudaFree(k_in);
  cudaFree(k_out);
  cudaFree(i_in);
  cudaFree(i_out);
  cudaFree(rowptr);
  cudaFree(ucount);
  cudaFree(kcount);
  cudaFree(col);
  cudaFree(val);
  cudaFree(d_dir);
  cudaFree(d_unsorted);
  cudaFree(tmp);
#undef SMG_E
  return rc;
}

}  // namespace smg
