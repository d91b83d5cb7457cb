// TEST HARNESS (tests/test_coo_order.py): the device's scipy-order row sort
// (paper_2402_12947_b200/csrc/coo_kernels.cu, namespace smg::coo_sort, host
// build of the same __host__ __device__ code) next to libstdc++'s real
// std::sort -- the algorithm scipy's csr_sort_indices runs -- so the test can
// compare the two on any input, including McIlroy's "antiqsort" adversary,
// which drives the median-of-three quicksort into its heapsort fallback.
#include <cuda_runtime.h>

#include <algorithm>
#include <string>
#include <utility>
#include <vector>

namespace smg {
int check_cuda(cudaError_t, const char*) { return 0; }
int fail(const std::string&) { return 1; }
void set_error(const std::string&) {}
}  // namespace smg

#include "../../paper_2402_12947_b200/csrc/coo_kernels.cu"

extern "C" {

// the device code path, run on the host
void emulated_row_sort(int64_t n, int32_t* c, double* v)
{
  smg::coo_sort::Seg s{c, v};
  smg::coo_sort::std_sort(s, n);
}

// what scipy does (sparsetools csr_sort_indices: std::sort of (col, val)
// pairs with a comparator on the column only)
static bool kv_less(const std::pair<int32_t, double>& a, const std::pair<int32_t, double>& b)
{
  return a.first < b.first;
}
void libstdcxx_row_sort(int64_t n, int32_t* c, double* v)
{
  std::vector<std::pair<int32_t, double>> t((size_t)n);
  for (int64_t i = 0; i < n; ++i) t[(size_t)i] = {c[i], v[i]};
  std::sort(t.begin(), t.end(), kv_less);
  for (int64_t i = 0; i < n; ++i) {
    c[i] = t[(size_t)i].first;
    v[i] = t[(size_t)i].second;
  }
}

// M. D. McIlroy, "A killer adversary for quicksort" (1999): a comparator
// that fixes values lazily so that the sort under attack degenerates; the
// resulting values are a concrete input that drives std::sort's depth limit
static std::vector<int> g_val;
static int g_gas, g_nsolid, g_candidate;
static bool adversary_less(int x, int y)
{
  if (g_val[(size_t)x] == g_gas && g_val[(size_t)y] == g_gas) {
    if (x == g_candidate)
      g_val[(size_t)x] = g_nsolid++;
    else
      g_val[(size_t)y] = g_nsolid++;
  }
  if (g_val[(size_t)x] == g_gas)
    g_candidate = x;
  else if (g_val[(size_t)y] == g_gas)
    g_candidate = y;
  return g_val[(size_t)x] < g_val[(size_t)y];
}
void antiqsort_input(int64_t n, int32_t* out)
{
  g_val.assign((size_t)n, (int)n - 1);
  g_gas = (int)n - 1;
  g_nsolid = 0;
  g_candidate = 0;
  std::vector<int> ptr((size_t)n);
  for (int64_t i = 0; i < n; ++i) ptr[(size_t)i] = (int)i;
  std::sort(ptr.begin(), ptr.end(), adversary_less);
  for (int64_t i = 0; i < n; ++i) out[i] = g_val[(size_t)i];
}

}  // extern "C"
