// Galerkin coarse operator on the device: A_c = P^T (A P), bit-identical to
// the reference's scipy product.
//
// Reference: sparse.py:147-154 triple_product (`ps.T @ (a.to_scipy() @ ps)`),
// called by transfer.py:153-155 coarsen_system from mg.py:100 (setup; SURVEY.md
// section 8(f) rank 1).  scipy evaluates both products with sparsetools
// csr_matmat (SMMP): row i of C = X Y accumulates sums[k] += X_ij * Y_jk over
// X's row in stored (ascending column) order starting from 0.0 and keeps the
// entries whose sum is != 0.  For the second product scipy works on CSC
// arrays: column c of P^T M sums M_ic * P_ik over fine rows i ascending, which
// is exactly row k of CSR(P^T) M with CSR(P^T) listing fine rows ascending
// (the operator's stored transpose): products commute and the addition order
// is the same, so every sum rounds identically (oracle/smg_oracle.c
// oracle_spgemm restates the order; tests pin it to the reference's own
// coarse operators bit for bit).
//
// Device design (setup work, integer-heavy, no tensor cores): one warp per
// output row with a shared-memory open-addressing hash table.
//   count   : every lane walks whole Y rows for its X entries and inserts the
//             columns (order-free); the unique count is an upper bound on the
//             row's kept entries.  Rows whose table overflows are recounted
//             by one CTA each with a global-memory table.
//   numeric : X's row is walked SEQUENTIALLY (warp-uniform), the lanes split
//             Y's row j -- distinct columns, so no two lanes touch the same
//             slot within a step and __syncwarp orders the steps.  Each entry
//             therefore sees its products in scipy's order, each product and
//             each sum correctly rounded (__dmul_rn / __dadd_rn, no FMA).
//             The table is then compacted in place (zero sums dropped, as
//             csr_matmat drops them) and ranked by column (canonical CSR).
//             Rows above kNumMax unique columns use one CTA each with a
//             global-memory table and __syncthreads between steps.
//   compact : kept counts -> row offsets (cub scan) -> copy.
#include "smg_internal.cuh"

#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <vector>

namespace smg {

namespace {

constexpr int kGWarps = 8;       // warps (rows) per CTA
constexpr int kSymCap = 2048;    // count: hash slots per warp (int32 keys, 8 KB)
constexpr int kSymMax = 1024;    // count: more unique columns -> CTA recount
constexpr int kNumCap = 1024;    // numeric: hash slots per warp (12 KB)
constexpr int kNumMax = 512;     // numeric: more unique columns -> CTA path
constexpr int kBigThreads = 256;

__device__ __forceinline__ uint32_t slot_hash(int32_t k, uint32_t mask)
{
  return ((uint32_t)k * 2654435761u >> 7) & mask;
}

// insert k (order-free); returns false if the table is full
__device__ __forceinline__ bool table_insert(int32_t* tab, uint32_t mask, int32_t k, int* ctr)
{
  uint32_t s = slot_hash(k, mask);
  for (uint32_t probe = 0; probe <= mask; ++probe, s = (s + 1) & mask) {
    int32_t cur = tab[s];
    if (cur == k) return true;
    if (cur == -1) {
      cur = atomicCAS(&tab[s], -1, k);
      if (cur == -1) {
        atomicAdd(ctr, 1);
        return true;
      }
      if (cur == k) return true;
    }
  }
  return false;
}

// slot of k, inserting it if absent; the table always has room (size >= 2 x unique)
__device__ __forceinline__ uint32_t table_slot(int32_t* tab, uint32_t mask, int32_t k)
{
  uint32_t s = slot_hash(k, mask);
  while (true) {
    int32_t cur = tab[s];
    if (cur == k) return s;
    if (cur == -1) {
      cur = atomicCAS(&tab[s], -1, k);
      if (cur == -1 || cur == k) return s;
    }
    s = (s + 1) & mask;
  }
}

__global__ void __launch_bounds__(kGWarps * 32)
spgemm_count_kernel(DevCsr X, DevCsr Y, int32_t* count, int32_t* big_rows, int32_t* n_big,
                    int64_t* big_bound)
{
  extern __shared__ int32_t count_smem[];  // kGWarps x kSymCap keys
  __shared__ int ctr[kGWarps];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * kGWarps + w;
  if (row >= X.nrows) return;
  int32_t* tab = count_smem + w * kSymCap;
  for (int s = lane; s < kSymCap; s += 32) tab[s] = -1;
  if (lane == 0) ctr[w] = 0;
  __syncwarp();
  bool full = false;
  int64_t bound = 0;
  for (int64_t jj = X.rowptr[row] + lane; jj < X.rowptr[row + 1]; jj += 32) {
    const int32_t j = X.col[jj];
    const int64_t b = Y.rowptr[j], e = Y.rowptr[j + 1];
    bound += e - b;
    for (int64_t kk = b; kk < e && !full; ++kk) {
      if (!table_insert(tab, kSymCap - 1, Y.col[kk], &ctr[w])) full = true;
      if (*(volatile int*)&ctr[w] > kSymMax) full = true;
    }
  }
  for (int o = 16; o > 0; o >>= 1) bound += __shfl_xor_sync(0xffffffffu, bound, o);
  full = __any_sync(0xffffffffu, full);
  __syncwarp();
  const int c = ctr[w];
  if (lane == 0) {
    if (full || c > kSymMax) {
      const int at = atomicAdd(n_big, 1);
      big_rows[at] = (int32_t)row;
      big_bound[at] = bound;
      count[row] = -1;
    } else {
      count[row] = c;
    }
  }
}

// recount of overflowed rows: one CTA per row, table in global memory
__global__ void __launch_bounds__(kBigThreads)
spgemm_count_big_kernel(DevCsr X, DevCsr Y, const int32_t* big_rows, const int64_t* tab_off,
                        int32_t* tabs, int32_t* count)
{
  __shared__ int ctr;
  const int64_t row = big_rows[blockIdx.x];
  int32_t* tab = tabs + tab_off[blockIdx.x];
  const uint32_t mask = (uint32_t)(tab_off[blockIdx.x + 1] - tab_off[blockIdx.x] - 1);
  for (int64_t s = threadIdx.x; s <= mask; s += blockDim.x) tab[s] = -1;
  if (threadIdx.x == 0) ctr = 0;
  __syncthreads();
  for (int64_t jj = X.rowptr[row]; jj < X.rowptr[row + 1]; ++jj) {
    const int32_t j = X.col[jj];
    for (int64_t kk = Y.rowptr[j] + threadIdx.x; kk < Y.rowptr[j + 1]; kk += blockDim.x)
      table_insert(tab, mask, Y.col[kk], &ctr);
  }
  __syncthreads();
  if (threadIdx.x == 0) count[row] = ctr;
}

__global__ void __launch_bounds__(kGWarps * 32)
spgemm_numeric_kernel(DevCsr X, DevCsr Y, const int32_t* count, const int64_t* ub_ptr,
                      int32_t* ub_col, double* ub_val, int32_t* kept)
{
  extern __shared__ double num_smem[];  // kGWarps x kNumCap sums, then keys
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * kGWarps + w;
  if (row >= X.nrows) return;
  if (count[row] > kNumMax) return;  // CTA path
  double* vals = num_smem + w * kNumCap;
  int32_t* keys = reinterpret_cast<int32_t*>(num_smem + kGWarps * kNumCap) + w * kNumCap;
  for (int s = lane; s < kNumCap; s += 32) {
    keys[s] = -1;
    vals[s] = 0.0;
  }
  __syncwarp();
  const int64_t xb = X.rowptr[row], xe = X.rowptr[row + 1];
  for (int64_t j0 = xb; j0 < xe; j0 += 32) {
    // this lane's X entry and its Y row bounds, broadcast step by step
    int32_t jl = 0;
    double xl = 0.0;
    int64_t yb = 0, ye = 0;
    if (j0 + lane < xe) {
      jl = X.col[j0 + lane];
      xl = X.val[j0 + lane];
      yb = Y.rowptr[jl];
      ye = Y.rowptr[jl + 1];
    }
    const int steps = (int)(xe - j0 < 32 ? xe - j0 : 32);
    for (int t = 0; t < steps; ++t) {  // X's row in stored order: scipy's sum order
      const double xv = __shfl_sync(0xffffffffu, xl, t);
      const int64_t b = __shfl_sync(0xffffffffu, yb, t), e = __shfl_sync(0xffffffffu, ye, t);
      for (int64_t kk = b + lane; kk < e; kk += 32) {
        const uint32_t s = table_slot(keys, kNumCap - 1, Y.col[kk]);
        vals[s] = __dadd_rn(vals[s], __dmul_rn(xv, Y.val[kk]));
      }
      __syncwarp();
    }
  }
  // in-place compaction: keep key != -1 with sum != 0 (csr_matmat drops zeros)
  int base = 0;
  for (int c0 = 0; c0 < kNumCap; c0 += 32) {
    const int32_t k = keys[c0 + lane];
    const double v = vals[c0 + lane];
    const bool keep = (k != -1) && (v != 0.0);
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    const int pos = base + __popc(bal & ((1u << lane) - 1u));
    __syncwarp();
    if (keep) {
      keys[pos] = k;
      vals[pos] = v;
    }
    base += __popc(bal);
    __syncwarp();
  }
  // rank by column (columns are unique): canonical sorted rows
  const int64_t off = ub_ptr[row];
  for (int e = lane; e < base; e += 32) {
    const int32_t k = keys[e];
    int r = 0;
    for (int t = 0; t < base; ++t) r += keys[t] < k;
    ub_col[off + r] = k;
    ub_val[off + r] = vals[e];
  }
  if (lane == 0) kept[row] = base;
}

// rows with more than kNumMax unique columns: one CTA per row, global table
__global__ void __launch_bounds__(kBigThreads)
spgemm_numeric_big_kernel(DevCsr X, DevCsr Y, const int32_t* rows, const int64_t* tab_off,
                          int32_t* tkeys, double* tvals, const int64_t* ub_ptr, int32_t* ub_col,
                          double* ub_val, int32_t* kept)
{
  __shared__ int base_s;
  const int64_t row = rows[blockIdx.x];
  int32_t* keys = tkeys + tab_off[blockIdx.x];
  double* vals = tvals + tab_off[blockIdx.x];
  const int64_t cap = tab_off[blockIdx.x + 1] - tab_off[blockIdx.x];
  const uint32_t mask = (uint32_t)(cap - 1);
  for (int64_t s = threadIdx.x; s < cap; s += blockDim.x) {
    keys[s] = -1;
    vals[s] = 0.0;
  }
  __syncthreads();
  for (int64_t jj = X.rowptr[row]; jj < X.rowptr[row + 1]; ++jj) {
    const double xv = X.val[jj];
    const int32_t j = X.col[jj];
    for (int64_t kk = Y.rowptr[j] + threadIdx.x; kk < Y.rowptr[j + 1]; kk += blockDim.x) {
      const uint32_t s = table_slot(keys, mask, Y.col[kk]);
      vals[s] = __dadd_rn(vals[s], __dmul_rn(xv, Y.val[kk]));
    }
    __syncthreads();
  }
  // compaction by warp 0 (rare rows; simplicity over speed)
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    int base = 0;
    for (int64_t c0 = 0; c0 < cap; c0 += 32) {
      const int32_t k = keys[c0 + lane];
      const double v = vals[c0 + lane];
      const bool keep = (k != -1) && (v != 0.0);
      const unsigned bal = __ballot_sync(0xffffffffu, keep);
      const int pos = base + __popc(bal & ((1u << lane) - 1u));
      __syncwarp();
      if (keep) {
        keys[pos] = k;
        vals[pos] = v;
      }
      base += __popc(bal);
      __syncwarp();
    }
    if (lane == 0) base_s = base;
  }
  __syncthreads();
  const int base = base_s;
  const int64_t off = ub_ptr[row];
  for (int e = threadIdx.x; e < base; e += blockDim.x) {
    const int32_t k = keys[e];
    int r = 0;
    for (int t = 0; t < base; ++t) r += keys[t] < k;
    ub_col[off + r] = k;
    ub_val[off + r] = vals[e];
  }
  if (threadIdx.x == 0) kept[row] = base;
}

__global__ void collect_rows_kernel(const int32_t* count, int64_t n, int threshold, int32_t* rows,
                                    int32_t* n_rows)
{
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && count[i] > threshold) rows[atomicAdd(n_rows, 1)] = (int32_t)i;
}

__global__ void widen_kernel(const int32_t* in, int64_t n, int64_t* out)
{
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = in[i];
}

// warp per row: copy the kept entries from the upper-bound layout
__global__ void compact_rows_kernel(int64_t n, const int64_t* ub_ptr, const int32_t* ub_col,
                                    const double* ub_val, const int64_t* ptr, int32_t* col,
                                    double* val)
{
  const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  const int64_t src = ub_ptr[row], dst = ptr[row], len = ptr[row + 1] - dst;
  for (int64_t t = lane; t < len; t += 32) {
    col[dst + t] = ub_col[src + t];
    val[dst + t] = ub_val[src + t];
  }
}

struct Scratch {
  std::vector<void*> ptrs;
  ~Scratch()
  {
    for (void* p : ptrs) cudaFree(p);
  }
  template <typename T>
  cudaError_t alloc(T** out, size_t n)
  {
    *out = nullptr;
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T));
    if (e == cudaSuccess) {
      ptrs.push_back(p);
      *out = static_cast<T*>(p);
    }
    return e;
  }
};

// out[0..n] = exclusive scan of in[0..n) (int64), out[n] = total
cudaError_t scan_offsets(const int64_t* in, int64_t n, int64_t* out, Scratch& sc, cudaStream_t s)
{
  size_t bytes = 0;
  cudaError_t e = cub::DeviceScan::InclusiveSum(nullptr, bytes, in, out + 1, (int64_t)n, s);
  if (e != cudaSuccess) return e;
  void* tmp = nullptr;
  if ((e = sc.alloc(reinterpret_cast<char**>(&tmp), bytes)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(out, 0, sizeof(int64_t), s)) != cudaSuccess) return e;
  if (n == 0) return cudaSuccess;
  return cub::DeviceScan::InclusiveSum(tmp, bytes, in, out + 1, (int64_t)n, s);
}

uint64_t next_pow2(uint64_t v)
{
  uint64_t c = 1;
  while (c < v) c <<= 1;
  return c;
}

}  // namespace

cudaError_t spgemm_device(const DevCsr& X, const DevCsr& Y, DevCsrOwned* out, cudaStream_t s)
{
  cudaError_t e;
  Scratch sc;
  const int64_t n = X.nrows;
  out->nrows = n;
  out->ncols = Y.ncols;
  int32_t *count = nullptr, *big = nullptr, *nbig = nullptr, *kept = nullptr;
  int64_t *bound = nullptr, *wide = nullptr, *ub_ptr = nullptr;
#define SMG_G(x)                          \
  do {                                    \
    if ((e = (x)) != cudaSuccess) return e; \
  } while (0)
  SMG_G(sc.alloc(&count, n));
  SMG_G(sc.alloc(&big, n));
  SMG_G(sc.alloc(&bound, n));
  SMG_G(sc.alloc(&nbig, 2));
  SMG_G(sc.alloc(&kept, n));
  SMG_G(sc.alloc(&wide, n));
  SMG_G(sc.alloc(&ub_ptr, n + 1));
  SMG_G(cudaMemsetAsync(nbig, 0, 2 * sizeof(int32_t), s));
  const int64_t grid_rows = (n + kGWarps - 1) / kGWarps;
  constexpr size_t count_smem = sizeof(int32_t) * kGWarps * kSymCap;
  constexpr size_t num_smem = (sizeof(double) + sizeof(int32_t)) * kGWarps * kNumCap;
  static bool attrs = false;
  if (!attrs) {
    SMG_G(cudaFuncSetAttribute(spgemm_count_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)count_smem));
    SMG_G(cudaFuncSetAttribute(spgemm_numeric_kernel,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)num_smem));
    attrs = true;
  }
  if (n > 0) {
    spgemm_count_kernel<<<(unsigned)grid_rows, kGWarps * 32, count_smem, s>>>(X, Y, count, big, nbig,
                                                                     bound);
    SMG_G(cudaGetLastError());
  }
  int32_t h_nbig = 0;
  SMG_G(cudaMemcpyAsync(&h_nbig, nbig, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  SMG_G(cudaStreamSynchronize(s));
  if (h_nbig > 0) {  // recount overflowed rows with global tables of 2 x min(bound, ncols)
    std::vector<int64_t> hb((size_t)h_nbig), off((size_t)h_nbig + 1, 0);
    SMG_G(cudaMemcpy(hb.data(), bound, h_nbig * sizeof(int64_t), cudaMemcpyDeviceToHost));
    for (int32_t b = 0; b < h_nbig; ++b)
      off[(size_t)b + 1] = off[(size_t)b] +
                           (int64_t)next_pow2((uint64_t)std::max<int64_t>(
                               64, 2 * std::min<int64_t>(hb[(size_t)b], Y.ncols)));
    int64_t* d_off = nullptr;
    int32_t* tabs = nullptr;
    SMG_G(sc.alloc(&d_off, off.size()));
    SMG_G(sc.alloc(&tabs, (size_t)off.back()));
    SMG_G(cudaMemcpy(d_off, off.data(), off.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
    spgemm_count_big_kernel<<<h_nbig, kBigThreads, 0, s>>>(X, Y, big, d_off, tabs, count);
    SMG_G(cudaGetLastError());
  }
  // upper-bound layout
  if (n > 0) {
    widen_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(count, n, wide);
    SMG_G(cudaGetLastError());
  }
  SMG_G(scan_offsets(wide, n, ub_ptr, sc, s));
  int64_t ub_nnz = 0;
  SMG_G(cudaMemcpyAsync(&ub_nnz, ub_ptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  SMG_G(cudaStreamSynchronize(s));
  int32_t* ub_col = nullptr;
  double* ub_val = nullptr;
  SMG_G(sc.alloc(&ub_col, (size_t)ub_nnz));
  SMG_G(sc.alloc(&ub_val, (size_t)ub_nnz));
  if (n > 0) {
    spgemm_numeric_kernel<<<(unsigned)grid_rows, kGWarps * 32, num_smem, s>>>(X, Y, count, ub_ptr,
                                                                       ub_col, ub_val, kept);
    SMG_G(cudaGetLastError());
    // rows above kNumMax: CTA path
    SMG_G(cudaMemsetAsync(nbig + 1, 0, sizeof(int32_t), s));
    collect_rows_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(count, n, kNumMax, big,
                                                                    nbig + 1);
    SMG_G(cudaGetLastError());
    int32_t h_nlong = 0;
    SMG_G(cudaMemcpyAsync(&h_nlong, nbig + 1, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    SMG_G(cudaStreamSynchronize(s));
    if (h_nlong > 0) {
      std::vector<int32_t> rows((size_t)h_nlong), cnt((size_t)n);
      SMG_G(cudaMemcpy(rows.data(), big, h_nlong * sizeof(int32_t), cudaMemcpyDeviceToHost));
      std::vector<int64_t> off((size_t)h_nlong + 1, 0);
      for (int32_t b = 0; b < h_nlong; ++b) {
        int32_t c = 0;
        SMG_G(cudaMemcpy(&c, count + rows[(size_t)b], sizeof(int32_t), cudaMemcpyDeviceToHost));
        off[(size_t)b + 1] = off[(size_t)b] + (int64_t)next_pow2((uint64_t)std::max(64, 2 * c));
      }
      int64_t* d_off = nullptr;
      int32_t* tk = nullptr;
      double* tv = nullptr;
      SMG_G(sc.alloc(&d_off, off.size()));
      SMG_G(sc.alloc(&tk, (size_t)off.back()));
      SMG_G(sc.alloc(&tv, (size_t)off.back()));
      SMG_G(cudaMemcpy(d_off, off.data(), off.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
      spgemm_numeric_big_kernel<<<h_nlong, kBigThreads, 0, s>>>(X, Y, big, d_off, tk, tv, ub_ptr,
                                                               ub_col, ub_val, kept);
      SMG_G(cudaGetLastError());
    }
    widen_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(kept, n, wide);
    SMG_G(cudaGetLastError());
  }
  // final layout
  SMG_G(cudaMalloc(&out->rowptr, (size_t)(n + 1) * sizeof(int64_t)));
  SMG_G(scan_offsets(wide, n, out->rowptr, sc, s));
  SMG_G(cudaMemcpyAsync(&out->nnz, out->rowptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  SMG_G(cudaStreamSynchronize(s));
  SMG_G(cudaMalloc(&out->col, (size_t)std::max<int64_t>(out->nnz, 1) * sizeof(int32_t)));
  SMG_G(cudaMalloc(&out->val, (size_t)std::max<int64_t>(out->nnz, 1) * sizeof(double)));
  if (n > 0) {
    compact_rows_kernel<<<(unsigned)((n * 32 + 255) / 256), 256, 0, s>>>(
        n, ub_ptr, ub_col, ub_val, out->rowptr, out->col, out->val);
    SMG_G(cudaGetLastError());
  }
  SMG_G(cudaStreamSynchronize(s));
#undef SMG_G
  return cudaSuccess;
}

void DevCsrOwned::release()
{
  cudaFree(rowptr);
  cudaFree(col);
  cudaFree(val);
  rowptr = nullptr;
  col = nullptr;
  val = nullptr;
}

DevCsr DevCsrOwned::view() const
{
  DevCsr d;
  d.nrows = nrows;
  d.ncols = ncols;
  d.nnz = nnz;
  d.rowptr = rowptr;
  d.col = col;
  d.val = val;
  return d;
}

}  // namespace smg
