// CSR-stream SpMV family with fused smoother epilogues (sm_100a, fp64).
//
// One kernel template serves every sparse product on the V-cycle hot path:
//
//   Epi::kSpmv      y = A x                      sparse.py:135-140
//   Epi::kResidual  r = b - A u                  mg.py:141, smoothers.py:263,266
//   Epi::kJacobi    u' = u + (D^-1 (b - A u))/theta        smoothers.py:120-124
//   Epi::kChebFirst d = (D^-1 (b - A u))/theta; u' = u + d  smoothers.py:128-129
//   Epi::kChebNext  z = D^-1 (b - A u); d = c1 d + c2 z; u' = u + d
//                                                          smoothers.py:130-135
//   Epi::kAddTo     u += P u_c                   mg.py:149 (prolong-add)
//   (restriction P^T r runs kSpmv over the stored CSR(P^T), mg.py:142)
//
// Bitwise parity with the reference (scipy csr_matvec: per-row sequential sum
// in column order, separately rounded multiply and add) drives the design:
//   * phase 1: the CTA streams its tile's values and column indices with
//     coalesced loads and stages the exact products val*x[col] (__dmul_rn) in
//     shared memory -- independent roundings, so any thread may compute them;
//   * phase 2: each thread owns one row and adds that row's products in
//     column order with __dadd_rn (no FMA contraction anywhere);
//   * the epilogue reproduces numpy's elementwise expression order, with IEEE
//     division (__ddiv_rn) for 1/a_ii and /theta.
// The diagonal is picked from the row during phase 2 (no separate inv-diag
// array is read).  Rows of any length are handled: a tile whose nonzeros
// exceed kTileNnz is streamed in several passes, each thread continuing its
// running sum, which keeps the column order.
#include "smg_internal.cuh"

namespace smg {

template <Epi E>
struct EpiNeedsDiag {
  static constexpr bool value = (E == Epi::kJacobi || E == Epi::kChebFirst || E == Epi::kChebNext);
};

template <Epi E>
__global__ void __launch_bounds__(kThreads)
csr_stream_kernel(const DevCsr m, const double* __restrict__ x, const EpiArgs ea)
{
  constexpr bool kDiag = EpiNeedsDiag<E>::value;
  __shared__ double s_prod[kTileNnz];
  __shared__ int32_t s_col[kDiag ? kTileNnz : 1];

  const int tile = blockIdx.x;
  const int32_t r0 = m.tile_row[tile];
  const int32_t r1 = m.tile_row[tile + 1];
  const int32_t row = r0 + (int32_t)threadIdx.x;
  const bool has_row = row < r1;
  const int64_t base = m.rowptr[r0];
  const int64_t end = m.rowptr[r1];
  int64_t lo = 0, hi = 0;
  if (has_row) {
    lo = m.rowptr[row];
    hi = m.rowptr[row + 1];
  }

  double sum = 0.0;
  int64_t jdiag = -1;
  for (int64_t cs = base; cs < end; cs += kTileNnz) {
    const int64_t rem = end - cs;
    const int cnt = rem < (int64_t)kTileNnz ? (int)rem : kTileNnz;
    const int32_t* __restrict__ colp = m.col + cs;
    const double* __restrict__ valp = m.val + cs;
    // phase 1: coalesced streaming of (col, val), gather x, exact products
    int32_t c[kItems];
    double v[kItems];
#pragma unroll
    for (int it = 0; it < kItems; ++it) {
      const int k = it * kThreads + (int)threadIdx.x;
      c[it] = 0;
      v[it] = 0.0;
      if (k < cnt) {
        c[it] = __ldg(colp + k);
        v[it] = __ldg(valp + k);
      }
    }
#pragma unroll
    for (int it = 0; it < kItems; ++it) {
      const int k = it * kThreads + (int)threadIdx.x;
      if (k < cnt) {
        const double xv = __ldg(x + c[it]);
        s_prod[k] = __dmul_rn(v[it], xv);
        if constexpr (kDiag) s_col[k] = c[it];
      }
    }
    __syncthreads();
    // phase 2: sequential per-row sum in column order
    if (has_row) {
      const int64_t a = lo > cs ? lo : cs;
      const int64_t bnd = hi < cs + cnt ? hi : cs + cnt;
      for (int64_t j = a; j < bnd; ++j) {
        sum = __dadd_rn(sum, s_prod[j - cs]);
        if constexpr (kDiag) {
          if (s_col[j - cs] == row) jdiag = j;
        }
      }
    }
    __syncthreads();
  }
  if (!has_row) return;

  if constexpr (E == Epi::kSpmv) {
    ea.out[row] = sum;
  } else if constexpr (E == Epi::kResidual) {
    ea.out[row] = __dsub_rn(ea.b[row], sum);
  } else if constexpr (E == Epi::kAddTo) {
    ea.out[row] = __dadd_rn(ea.out[row], sum);
  } else {
    const double dg = jdiag >= 0 ? m.val[jdiag] : 0.0;
    const double inv = __ddiv_rn(1.0, dg);
    const double t = __dmul_rn(inv, __dsub_rn(ea.b[row], sum));
    if constexpr (E == Epi::kJacobi) {
      ea.out[row] = __dadd_rn(ea.u_in[row], __ddiv_rn(t, ea.theta));
    } else if constexpr (E == Epi::kChebFirst) {
      const double d = __ddiv_rn(t, ea.theta);
      ea.d[row] = d;
      ea.out[row] = __dadd_rn(ea.u_in[row], d);
    } else {  // kChebNext
      const double d = __dadd_rn(__dmul_rn(ea.c1, ea.d[row]), __dmul_rn(ea.c2, t));
      ea.d[row] = d;
      ea.out[row] = __dadd_rn(ea.u_in[row], d);
    }
  }
}

template <Epi E>
static cudaError_t launch_t(const DevCsr& m, const double* x, const EpiArgs& ea, cudaStream_t s)
{
  if (m.ntiles == 0) return cudaSuccess;
  csr_stream_kernel<E><<<m.ntiles, kThreads, 0, s>>>(m, x, ea);
  return cudaGetLastError();
}

cudaError_t launch_csr_stream(const DevCsr& m, const double* x, Epi epi, const EpiArgs& ea,
                              cudaStream_t s)
{
  switch (epi) {
    case Epi::kSpmv: return launch_t<Epi::kSpmv>(m, x, ea, s);
    case Epi::kResidual: return launch_t<Epi::kResidual>(m, x, ea, s);
    case Epi::kJacobi: return launch_t<Epi::kJacobi>(m, x, ea, s);
    case Epi::kChebFirst: return launch_t<Epi::kChebFirst>(m, x, ea, s);
    case Epi::kChebNext: return launch_t<Epi::kChebNext>(m, x, ea, s);
    case Epi::kAddTo: return launch_t<Epi::kAddTo>(m, x, ea, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace smg
