// CSR-tile SpMV family with fused smoother epilogues (sm_100a, fp64).
//
// One kernel template serves every sparse product on the V-cycle hot path:
//
//   Epi::kSpmv          y = A x                      sparse.py:135-140
//   Epi::kResidual      r = b - A u                  mg.py:141, smoothers.py:263,266
//   Epi::kJacobi        u' = u + (D^-1 (b - A u))/theta        smoothers.py:120-124
//   Epi::kChebFirst     d = (D^-1 (b - A u))/theta; u' = u + d  smoothers.py:128-129
//   Epi::kChebNext      z = D^-1 (b - A u); d = c1 d + c2 z; u' = u + d
//                                                              smoothers.py:130-135
//   Epi::kAddTo         u += P u_c                   mg.py:149 (prolong-add; out of
//                       place into `out` when u_in is given)
//   Epi::kRestrictFirst b_c = P^T r, then the coarse level's first sweep from
//                       its zero initial guess (mg.py:142-143 + smoothers.py:128)
//   (plain restriction P^T r runs kSpmv over the stored CSR(P^T), mg.py:142)
//
// Bitwise parity with the reference (scipy csr_matvec: per-row sequential sum
// in column order, separately rounded multiply and add):
//   * a CTA owns a tile of consecutive rows (<= 256 rows, <= 2048 nonzeros);
//     all its threads load the tile's values/columns with coalesced loads,
//     gather x and stage the exact products val*x[col] (__dmul_rn) in shared
//     memory -- products are independently rounded, so any thread may form
//     any of them;
//   * each thread then adds its own row's products in column order with
//     __dadd_rn (no FMA contraction anywhere);
//   * the epilogue reproduces numpy's elementwise expression order, with IEEE
//     division (__ddiv_rn) for /theta; 1/a_ii is a precomputed vector formed
//     with the same IEEE division numpy uses (smoothers.py:115).
//
// L2 residency: operators too large to stay in L2 (DevCsr::streaming, set at
// upload) are read with evict-first priority, so the coarse levels -- visited
// twice per V-cycle -- stay L2-resident across the fine-level sweeps.
//
// Latency hiding (the kernel is latency-, not instruction-bound):
//   * operator data (tile bounds, row offsets, values, columns) is requested
//     before griddepcontrol.wait; kernels are launched with programmatic
//     dependent launch, so that traffic overlaps the previous kernel's tail;
//   * one thread per CTA issues cp.async.bulk.prefetch.L2 for the tile that
//     starts one resident wave later, so the next wave's loads hit L2.
// Rejected designs (persistent TMA rings, tiles delivered by bulk copy) are
// recorded in DESIGN.md section 3 with their measurements.
#include "smg_internal.cuh"

#include <algorithm>
#include <cstdlib>

namespace smg {

// programmatic dependent launch: no-ops when launched without the attribute
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger()
{
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes, bool evict_first)
{
  if (evict_first) {
    asm volatile(
        "{\n.reg .b64 pol;\n"
        "createpolicy.fractional.L2::evict_first.b64 pol, 1.0;\n"
        "cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, pol;\n}\n" ::"l"(p),
        "r"(bytes)
        : "memory");
  } else {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
  }
}

template <Epi E>
struct EpiTraits {
  static constexpr bool kDiag = (E == Epi::kJacobi || E == Epi::kChebFirst || E == Epi::kChebNext);
  static constexpr bool kDiagVec = (E == Epi::kRestrictFirst);
  static constexpr bool kB = (E != Epi::kSpmv && E != Epi::kAddTo && E != Epi::kRestrictFirst);
  static constexpr bool kU = kDiag;
  static constexpr bool kD = (E == Epi::kChebNext);
  static constexpr bool kOut = (E == Epi::kAddTo);
};

template <Epi E>
__device__ __forceinline__ void epilogue(const EpiArgs& ea, int32_t row, double sum, double inv,
                                         double bv, double uv, double dv, double ov)
{
  if constexpr (E == Epi::kSpmv) {
    ea.out[row] = sum;
  } else if constexpr (E == Epi::kResidual) {
    ea.out[row] = __dsub_rn(bv, sum);
  } else if constexpr (E == Epi::kAddTo) {
    ea.out[row] = __dadd_rn(ov, sum);
  } else if constexpr (E == Epi::kRestrictFirst) {
    ea.b_out[row] = sum;
    const double t = __dmul_rn(inv, __dsub_rn(sum, 0.0));  // A_c 0 sums to +0.0 exactly
    const double d = __ddiv_rn(t, ea.theta);
    if (ea.d) ea.d[row] = d;
    ea.out[row] = __dadd_rn(0.0, d);
  } else {
    const double t = __dmul_rn(inv, __dsub_rn(bv, sum));
    if constexpr (E == Epi::kJacobi) {
      ea.out[row] = __dadd_rn(uv, __ddiv_rn(t, ea.theta));
    } else if constexpr (E == Epi::kChebFirst) {
      const double d = __ddiv_rn(t, ea.theta);
      if (ea.keep_d) {
        if (ea.stream_vec) __stcs(ea.d + row, d); else ea.d[row] = d;
      }
      ea.out[row] = __dadd_rn(uv, d);
    } else {  // kChebNext
      const double d = __dadd_rn(__dmul_rn(ea.c1, dv), __dmul_rn(ea.c2, t));
      if (ea.keep_d) {
        if (ea.stream_vec) __stcs(ea.d + row, d); else ea.d[row] = d;
      }
      ea.out[row] = __dadd_rn(uv, d);
    }
  }
}

// 64 registers, 4 CTAs (32 warps) per SM: measured faster than 40 registers /
// 6 CTAs with spills (profiles/r01/bench_variant_v*.json).
#ifndef SMG_SPMV_MIN_BLOCKS
#define SMG_SPMV_MIN_BLOCKS 4
#endif
constexpr int kMinBlocks = SMG_SPMV_MIN_BLOCKS;

template <Epi E, bool kPf, bool kMulti, bool kFixed>
__global__ void __launch_bounds__(kThreads, kMinBlocks)
csr_tile_kernel(const DevCsr m, const double* __restrict__ x, const EpiArgs ea, int pf_dist)
{
  using T = EpiTraits<E>;
  // kMulti (operators with long rows, multi-chunk tiles): two chunk buffers,
  // chunk q's products are summed while chunk q+1's values and columns are
  // already in flight.  Otherwise one buffer (only a single row longer than a
  // chunk makes a tile span several chunks).
  __shared__ double s_prod[kMulti ? 2 * kTileNnz : kTileNnz];
  const int t = blockIdx.x;
  const int tid = threadIdx.x;
  // ---- operator data (never written by any kernel): before the dependency wait
  // fixed-capacity layout: the tile's nonzeros start at t * cap -- the value /
  // column loads need no tile-offset load first (one dependent round trip less)
  const int32_t* __restrict__ colp = kFixed ? m.pcol : m.col;
  const double* __restrict__ valp = kFixed ? m.pval : m.val;
  int64_t e0;
  int cnt;
  if constexpr (kFixed) {
    e0 = (int64_t)t * m.cap;
    cnt = m.cap;
  } else {
    e0 = m.tile_nz[t];
    cnt = (int)(m.tile_nz[t + 1] - e0);
  }
  int32_t c[kItems];
  double v[kItems];
  auto load_chunk = [&](int q0) {
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
      const int k = q0 + i * kThreads + tid;
      c[i] = 0;
      v[i] = 0.0;
      if (k < cnt && k < q0 + kTileNnz) {
        if (m.streaming) {  // operator larger than L2 share: don't evict the small levels
          c[i] = __ldcs(colp + e0 + k);
          v[i] = __ldcs(valp + e0 + k);
        } else {
          c[i] = __ldg(colp + e0 + k);
          v[i] = __ldg(valp + e0 + k);
        }
      }
    }
  };
  if constexpr (kFixed) load_chunk(0);
  const int32_t r0 = m.tile_row[t];
  const int32_t r1 = m.tile_row[t + 1];
  const int nq = (cnt + kTileNnz - 1) / kTileNnz;   // chunks of this tile
  const int32_t row = r0 + tid;
  const bool has_row = row < r1;
  int64_t lo = 0, hi = 0;
  if (has_row) {
    if constexpr (kFixed) {
      lo = tid > 0 ? m.rel_end[row - 1] : 0;
      hi = m.rel_end[row];
    } else {
      lo = m.rowptr[row] - e0;
      hi = m.rowptr[row + 1] - e0;
    }
  }
  if constexpr (!kFixed) load_chunk(0);
  if constexpr (kPf) {
    // pull the tile that starts one resident wave later into L2 (bulk
    // prefetch: no registers, no shared memory), so its CTA's loads hit L2
    if (tid == 0) {
      const int tp = t + pf_dist;
      if (tp < m.ntiles) {
        const int64_t p0 = kFixed ? (int64_t)tp * m.cap : m.tile_nz[tp];
        const int64_t p1 = kFixed ? p0 + m.cap : m.tile_nz[tp + 1];
        if (p1 - p0 <= kTileNnz * kMaxTileChunks && p1 > p0) {
          const int64_t va = p0 & ~int64_t(1), vb = (p1 + 1) & ~int64_t(1);
          const int64_t ca = p0 & ~int64_t(3), cb = (p1 + 3) & ~int64_t(3);
          prefetch_l2(valp + va, (uint32_t)((vb - va) * 8), m.streaming);
          prefetch_l2(colp + ca, (uint32_t)((cb - ca) * 4), m.streaming);
        }
      }
    }
  }
  // ---- vectors produced by earlier kernels: after the dependency wait
  pdl_wait();
  pdl_trigger();
  // gathered row subsets (halo pass) address vectors through row_map; the
  // interior pass skips the rows a concurrent local correction may change
  const int32_t grow = (has_row && m.row_map) ? m.row_map[row] : row;
  SMG_DCHECK(!has_row || (grow >= 0 && (m.row_map || grow < m.nrows)));
  const bool write = has_row && !(ea.skip_rows && ea.skip_rows[grow]);
  double bv = 0.0, uv = 0.0, dv = 0.0, ov = 0.0, inv = 0.0;
  if (write) {
    if constexpr (T::kB) bv = ea.b[grow];
    if constexpr (T::kU) uv = ea.u_in[grow];
    if constexpr (T::kD) dv = ea.d[grow];
    if constexpr (T::kOut) ov = (ea.u_in ? ea.u_in : ea.out)[grow];  // prolong-add in or out of place
    if constexpr (T::kDiag) inv = m.inv_diag[grow];
    if constexpr (T::kDiagVec) inv = ea.inv_diag[grow];
  }
  const int a = (int)lo, bnd = (int)hi;   // this row's tile-relative range
  double sum = 0.0;
  for (int q = 0; q < nq; ++q) {
    const int q0 = q * kTileNnz;
    const int qn = min(kTileNnz, cnt - q0);
    double* buf = s_prod + (kMulti ? (q & 1) * kTileNnz : 0);
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
      const int k = i * kThreads + tid;
      if (k < qn) {
        SMG_DCHECK(c[i] >= 0 && c[i] < m.ncols);
        buf[k] = __dmul_rn(v[i], __ldg(x + c[i]));
      }
    }
    if (q + 1 < nq) load_chunk(q0 + kTileNnz);   // in flight during this chunk's sums
    __syncthreads();
    if (has_row) {
      SMG_DCHECK(a >= 0 && a <= bnd && bnd <= cnt);
      const int j0 = max(a, q0), j1 = min(bnd, q0 + qn);
      for (int j = j0; j < j1; ++j) sum = __dadd_rn(sum, buf[j - q0]);
    }
    if (!kMulti && q + 1 < nq) __syncthreads();   // single buffer: sums done before reuse
  }
  if (write) epilogue<E>(ea, grow, sum, inv, bv, uv, dv, ov);
}

// Warp-specialised tile kernel for long-row operators on offset-table tiles
// (SMG_TILE_WS=1; C2 levels 2-3, C3 level 1, C4 level 2: L2-resident,
// latency-bound).  In csr_tile_kernel every thread first forms products and
// then the few row owners sum them while the other threads wait at the
// barrier; here six loader warps stream (value, column) chunks, gather x and
// fill a ring of three product buffers, while two summer warps add each
// row's products in column order as the chunks arrive (row r of the tile
// belongs to summer thread r mod 64, which keeps its running sum across
// chunks).  "full" / "empty" mbarriers per buffer, one arrival per warp; no
// CTA barrier after the start.  Same products, same order: bit-identical.
constexpr int kWsLoaders = 192;
constexpr int kWsSummers = kThreads - kWsLoaders;   // 64
constexpr int kWsSlots = 3;
constexpr int kWsItems = (kTileNnz + kWsLoaders - 1) / kWsLoaders;   // 11
constexpr int kWsRows = kRowsPerTile / kWsSummers;                   // 4 rows per summer thread

__device__ __forceinline__ uint32_t ws_smem_u32(const void* p)
{
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void ws_wait(uint64_t* bar, uint32_t parity)
{
  asm volatile(
      "{\n.reg .pred p;\nWS_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WS_%=;\n}\n" ::"r"(ws_smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void ws_arrive(uint64_t* bar)
{
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(ws_smem_u32(bar)) : "memory");
}

template <Epi E, bool kPf>
__global__ void __launch_bounds__(kThreads, 4)
csr_ws_kernel(const DevCsr m, const double* __restrict__ x, const EpiArgs ea, int pf_dist)
{
  using T = EpiTraits<E>;
  // dynamic: 3 x 16 KB of products (+ barriers) is past the 48 KB static limit
  extern __shared__ __align__(16) unsigned char ws_smem[];
  double(*s_prod)[kTileNnz] = reinterpret_cast<double(*)[kTileNnz]>(ws_smem);
  uint64_t* s_full = reinterpret_cast<uint64_t*>(ws_smem + sizeof(double) * kWsSlots * kTileNnz);
  uint64_t* s_empty = s_full + kWsSlots;
  const int t = blockIdx.x;
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int64_t e0 = m.tile_nz[t];
  const int cnt = (int)(m.tile_nz[t + 1] - e0);
  const int nq = (cnt + kTileNnz - 1) / kTileNnz;
  if (tid == 0) {
    for (int s = 0; s < kWsSlots; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(ws_smem_u32(&s_full[s])),
                   "r"(kWsLoaders / 32)
                   : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(ws_smem_u32(&s_empty[s])),
                   "r"(kWsSummers / 32)
                   : "memory");
    }
  }
  if (tid < kWsLoaders) {
    // ---- loaders: operator data before the dependency wait
    int32_t c[kWsItems];
    double v[kWsItems];
    auto load_chunk = [&](int q0) {
#pragma unroll
      for (int i = 0; i < kWsItems; ++i) {
        const int k = q0 + i * kWsLoaders + tid;
        c[i] = 0;
        v[i] = 0.0;
        if (k < cnt && k < q0 + kTileNnz) {
          if (m.streaming) {
            c[i] = __ldcs(m.col + e0 + k);
            v[i] = __ldcs(m.val + e0 + k);
          } else {
            c[i] = __ldg(m.col + e0 + k);
            v[i] = __ldg(m.val + e0 + k);
          }
        }
      }
    };
    load_chunk(0);
    if constexpr (kPf) {
      if (tid == 0) {
        const int tp = t + pf_dist;
        if (tp < m.ntiles) {
          const int64_t p0 = m.tile_nz[tp], p1 = m.tile_nz[tp + 1];
          if (p1 - p0 <= kTileNnz * kMaxTileChunks && p1 > p0) {
            const int64_t va = p0 & ~int64_t(1), vb = (p1 + 1) & ~int64_t(1);
            const int64_t ca = p0 & ~int64_t(3), cb = (p1 + 3) & ~int64_t(3);
            prefetch_l2(m.val + va, (uint32_t)((vb - va) * 8), m.streaming);
            prefetch_l2(m.col + ca, (uint32_t)((cb - ca) * 4), m.streaming);
          }
        }
      }
    }
    __syncthreads();   // barriers initialised
    pdl_wait();
    pdl_trigger();
    int slot = 0;
    uint32_t eph = 1;   // parity of the "empty" phase a refill waits for (first round: free)
    for (int q = 0; q < nq; ++q) {
      const int q0 = q * kTileNnz;
      const int qn = min(kTileNnz, cnt - q0);
      if (q >= kWsSlots) ws_wait(&s_empty[slot], eph);
      double* buf = s_prod[slot];
#pragma unroll
      for (int i = 0; i < kWsItems; ++i) {
        const int k = i * kWsLoaders + tid;
        if (k < qn) buf[k] = __dmul_rn(v[i], __ldg(x + c[i]));
      }
      if (q + 1 < nq) load_chunk(q0 + kTileNnz);
      __syncwarp();
      if (lane == 0) ws_arrive(&s_full[slot]);
      if (++slot == kWsSlots) {
        slot = 0;
        if (q >= kWsSlots - 1) eph ^= 1u;
      }
    }
    return;
  }
  // ---- summers: rows r0 + s + 64 j
  const int sidx = tid - kWsLoaders;
  const int32_t r0 = m.tile_row[t];
  const int32_t r1 = m.tile_row[t + 1];
  int lo[kWsRows], hi[kWsRows];
#pragma unroll
  for (int j = 0; j < kWsRows; ++j) {
    const int32_t row = r0 + sidx + kWsSummers * j;
    lo[j] = hi[j] = 0;
    if (row < r1) {
      lo[j] = (int)(m.rowptr[row] - e0);
      hi[j] = (int)(m.rowptr[row + 1] - e0);
    }
  }
  __syncthreads();   // barriers initialised
  pdl_wait();
  pdl_trigger();
  double bv[kWsRows], uv[kWsRows], dv[kWsRows], ov[kWsRows], inv[kWsRows], sum[kWsRows];
  int32_t grow[kWsRows];
  bool write[kWsRows];
#pragma unroll
  for (int j = 0; j < kWsRows; ++j) {
    const int32_t row = r0 + sidx + kWsSummers * j;
    const bool has_row = row < r1;
    grow[j] = (has_row && m.row_map) ? m.row_map[row] : row;
    write[j] = has_row && !(ea.skip_rows && ea.skip_rows[grow[j]]);
    bv[j] = uv[j] = dv[j] = ov[j] = inv[j] = 0.0;
    sum[j] = 0.0;
    if (write[j]) {
      if constexpr (T::kB) bv[j] = ea.b[grow[j]];
      if constexpr (T::kU) uv[j] = ea.u_in[grow[j]];
      if constexpr (T::kD) dv[j] = ea.d[grow[j]];
      if constexpr (T::kOut) ov[j] = (ea.u_in ? ea.u_in : ea.out)[grow[j]];
      if constexpr (T::kDiag) inv[j] = m.inv_diag[grow[j]];
      if constexpr (T::kDiagVec) inv[j] = ea.inv_diag[grow[j]];
    }
  }
  int slot = 0;
  uint32_t fph = 0;
  for (int q = 0; q < nq; ++q) {
    const int q0 = q * kTileNnz;
    const int qn = min(kTileNnz, cnt - q0);
    ws_wait(&s_full[slot], fph);
    const double* buf = s_prod[slot];
#pragma unroll
    for (int j = 0; j < kWsRows; ++j) {
      const int j0 = max(lo[j], q0), j1 = min(hi[j], q0 + qn);
      double sacc = sum[j];
      for (int e = j0; e < j1; ++e) sacc = __dadd_rn(sacc, buf[e - q0]);
      sum[j] = sacc;
    }
    __syncwarp();
    if (lane == 0) ws_arrive(&s_empty[slot]);
    if (++slot == kWsSlots) {
      slot = 0;
      fph ^= 1u;
    }
  }
#pragma unroll
  for (int j = 0; j < kWsRows; ++j)
    if (write[j]) epilogue<E>(ea, grow[j], sum[j], inv[j], bv[j], uv[j], dv[j], ov[j]);
}

// Whole-tile staging for L2-resident long-row operators (DevCsr::stage_cap > 0,
// SMG_LAYOUT_TILES_STAGED; C2 levels 2-3, C3 levels 1-2).  csr_tile_kernel
// walks such a tile in 2048-product chunks and, after every chunk, the ~34
// row owners add their 60 products one after the other while the rest of the
// CTA waits at the barrier: four serial rounds of (gather latency + add chain)
// per tile.  Here the tile (up to kStageMaxNnz products, sized at upload so
// the operator is one resident wave of 3 CTAs per SM) is staged whole: the
// loads of batch q+1 are in flight during the x gathers of batch q, there is
// ONE barrier, and then every row of the tile sums at once.  Same products,
// same order per row: bit-identical.
template <Epi E, bool kPf>
__global__ void __launch_bounds__(kThreads, kStageCtas)
csr_stage_kernel(const DevCsr m, const double* __restrict__ x, const EpiArgs ea, int pf_dist)
{
  using T = EpiTraits<E>;
  extern __shared__ __align__(16) double st_prod[];
  const int t = blockIdx.x;
  const int tid = threadIdx.x;
  // ---- operator data (never written by any kernel): before the dependency wait
  const int64_t e0 = m.tile_nz[t];
  const int cnt = (int)(m.tile_nz[t + 1] - e0);
  const int32_t* __restrict__ colp = m.col + e0;
  const double* __restrict__ valp = m.val + e0;
  int32_t c[kItems];
  double v[kItems];
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    const int k = i * kThreads + tid;
    c[i] = 0;
    v[i] = 0.0;
    if (k < cnt) {
      if (m.streaming) {   // several waves of an operator larger than L2: evict-first
        c[i] = __ldcs(colp + k);
        v[i] = __ldcs(valp + k);
      } else {
        c[i] = __ldg(colp + k);
        v[i] = __ldg(valp + k);
      }
    }
  }
  const int32_t r0 = m.tile_row[t];
  const int32_t r1 = m.tile_row[t + 1];
  const int32_t row = r0 + tid;
  const bool has_row = row < r1;
  int a = 0, bnd = 0;   // this row's tile-relative range
  if (has_row) {
    a = (int)(m.rowptr[row] - e0);
    bnd = (int)(m.rowptr[row + 1] - e0);
  }
  if constexpr (kPf) {
    if (tid == 0) {
      const int tp = t + pf_dist;
      if (tp < m.ntiles) {
        const int64_t p0 = m.tile_nz[tp], p1 = m.tile_nz[tp + 1];
        if (p1 > p0 && p1 - p0 <= kStageMaxNnz) {
          const int64_t va = p0 & ~int64_t(1), vb = (p1 + 1) & ~int64_t(1);
          const int64_t ca = p0 & ~int64_t(3), cb = (p1 + 3) & ~int64_t(3);
          prefetch_l2(m.val + va, (uint32_t)((vb - va) * 8), m.streaming);
          prefetch_l2(m.col + ca, (uint32_t)((cb - ca) * 4), m.streaming);
        }
      }
    }
  }
  // ---- vectors produced by earlier kernels: after the dependency wait
  pdl_wait();
  pdl_trigger();
  const int32_t grow = (has_row && m.row_map) ? m.row_map[row] : row;
  SMG_DCHECK(!has_row || (grow >= 0 && (m.row_map || grow < m.nrows)));
  const bool write = has_row && !(ea.skip_rows && ea.skip_rows[grow]);
  double bv = 0.0, uv = 0.0, dv = 0.0, ov = 0.0, inv = 0.0;
  if (write) {
    if constexpr (T::kB) bv = ea.b[grow];
    if constexpr (T::kU) uv = ea.u_in[grow];
    if constexpr (T::kD) dv = ea.d[grow];
    if constexpr (T::kOut) ov = (ea.u_in ? ea.u_in : ea.out)[grow];
    if constexpr (T::kDiag) inv = m.inv_diag[grow];
    if constexpr (T::kDiagVec) inv = ea.inv_diag[grow];
  }
  for (int q0 = 0; q0 < cnt; q0 += kTileNnz) {
    double xv[kItems];
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
      SMG_DCHECK(c[i] >= 0 && c[i] < m.ncols);
      xv[i] = __ldg(x + c[i]);   // c = 0 past the end: a valid address, product unused
    }
    // the next batch's values and columns are requested before this batch's
    // gathers are consumed
    int32_t cn[kItems];
    double vn[kItems];
    const int qn = q0 + kTileNnz;
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
      const int k = qn + i * kThreads + tid;
      cn[i] = 0;
      vn[i] = 0.0;
      if (k < cnt) {
        if (m.streaming) {
          cn[i] = __ldcs(colp + k);
          vn[i] = __ldcs(valp + k);
        } else {
          cn[i] = __ldg(colp + k);
          vn[i] = __ldg(valp + k);
        }
      }
    }
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
      const int k = q0 + i * kThreads + tid;
      if (k < cnt) st_prod[k] = __dmul_rn(v[i], xv[i]);
    }
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
      c[i] = cn[i];
      v[i] = vn[i];
    }
  }
  __syncthreads();
  double sum = 0.0;
  if (has_row) {
    SMG_DCHECK(a >= 0 && a <= bnd && bnd <= cnt);
    int j = a;
    for (; j + 8 <= bnd; j += 8) {
      double p[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) p[i] = st_prod[j + i];
#pragma unroll
      for (int i = 0; i < 8; ++i) sum = __dadd_rn(sum, p[i]);
    }
    for (; j < bnd; ++j) sum = __dadd_rn(sum, st_prod[j]);
  }
  if (write) epilogue<E>(ea, grow, sum, inv, bv, uv, dv, ov);
}

// SELL-32-sigma256 (DevCsr::sell): one CTA per window of 256 rows, warp k =
// slice k, lane = slot.  Each thread streams its own row -- entry j of the 32
// slots is contiguous, so every load is coalesced -- and adds the products in
// column order (scipy's order) without staging them in shared memory: no
// barrier, few registers, 8 CTAs (64 warps) per SM.
constexpr int kSellPre = 4;   // entries loaded before the dependency wait

// kPipe (long rows): the next kUnroll entries' columns and values are
// requested before this batch's x gathers and sums, so the HBM stream never
// waits on the gathers (software pipelining; SMG_SELL_PIPE)
// kDelta (DevCsr::sell_delta, "SELL-d16"): the column stream is 16-bit codes
// in the same positions -- code = column - previous column of the row
// (0..0xFFFD), 0xFFFE = padding, 0xFFFF = the next of the row's (at most two)
// escape columns, held per slot in sell_esc; the row's first column comes
// from sell_c0.  A thread walks its row in order anyway, so decoding is one
// integer add on the gather address; the sums are unchanged (same products,
// same order), the operator stream is 10 instead of 12 bytes per entry.
#ifndef SMG_D16_RELAX
#define SMG_D16_RELAX 0   // 1: delta kernels get 6 / 3 CTAs per SM (40 / 80 registers, no spills)
#endif
constexpr int sell_min_blocks(int unroll, bool pipe, bool delta)
{
  if (SMG_D16_RELAX && delta) return pipe ? 3 : (unroll <= 4 ? 6 : (unroll <= 8 ? 3 : 2));
  return pipe ? 4 : (unroll <= 4 ? 8 : (unroll <= 8 ? 4 : 2));
}

template <Epi E, bool kPf, int kUnroll, bool kPipe = false, bool kDelta = false>
__global__ void __launch_bounds__(kSellWindow, sell_min_blocks(kUnroll, kPipe, kDelta))
sell_kernel(const DevCsr m, const double* __restrict__ x, const EpiArgs ea, int pf_dist,
            int xpf_chunk)
{
  using T = EpiTraits<E>;
  constexpr int32_t kPad = kDelta ? 0xFFFE : -1;
  const int w = blockIdx.x;
  const int k = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t sb = m.sell_ptr[(int64_t)w * kSellSlices + k];
  const int64_t se = m.sell_ptr[(int64_t)w * kSellSlices + k + 1];
  const int width = (int)((se - sb) >> 5);
  const int rl = m.sell_perm[(int64_t)w * kSellWindow + threadIdx.x];
  const int32_t* __restrict__ cp = m.sell_col + sb + lane;
  const uint16_t* __restrict__ dp = m.sell_dcol + sb + lane;
  const double* __restrict__ vp = m.sell_val + sb + lane;
  // raw column-stream item j of this slot: a column (or -1), or a 16-bit code
  auto ldraw = [&](int j) -> int32_t {
    if constexpr (kDelta)
      return m.streaming ? (int32_t)__ldcs(dp + j * 32) : (int32_t)__ldg(dp + j * 32);
    else
      return m.streaming ? __ldcs(cp + j * 32) : __ldg(cp + j * 32);
  };
  auto ldval = [&](int j) -> double {
    return m.streaming ? __ldcs(vp + j * 32) : __ldg(vp + j * 32);
  };
  // decoder state (kDelta): current column, escapes consumed, the slot's escapes
  int32_t ccur = 0, e0 = 0, e1 = 0;
  int ek = 0;
  if constexpr (kDelta) {
    const int64_t slot = (int64_t)w * kSellWindow + threadIdx.x;
    ccur = __ldg(m.sell_c0 + slot);
    if (m.sell_esc_planes > 0) e0 = __ldg(m.sell_esc + slot);
    if (m.sell_esc_planes > 1) e1 = __ldg(m.sell_esc + (int64_t)m.sell_nwin * kSellWindow + slot);
  }
  // items must be decoded in entry order; returns the column, or -1 for padding
  auto decode = [&](int32_t raw) -> int32_t {
    if constexpr (!kDelta) {
      return raw;
    } else {
      if (raw == 0xFFFE) return -1;
      if (raw == 0xFFFF) {
        ccur = ek == 0 ? e0 : e1;
        ++ek;
      } else {
        ccur += raw;
      }
      return ccur;
    }
  };
  int32_t c0[kSellPre];
  double v0[kSellPre];
#pragma unroll
  for (int j = 0; j < kSellPre; ++j) {
    c0[j] = kPad;
    v0[j] = 0.0;
    if (j < width) {
      c0[j] = ldraw(j);
      v0[j] = ldval(j);
    }
  }
  if constexpr (kPf) {
    if (threadIdx.x == 0) {
      const int wp = w + pf_dist;
      if (wp < m.sell_nwin) {
        const int64_t p0 = m.sell_ptr[(int64_t)wp * kSellSlices];
        const int64_t p1 = m.sell_ptr[(int64_t)(wp + 1) * kSellSlices];
        if (p1 > p0 && p1 - p0 <= (int64_t)kTileNnz * 16) {
          const int64_t va = p0 & ~int64_t(1), vb = (p1 + 1) & ~int64_t(1);
          prefetch_l2(m.sell_val + va, (uint32_t)((vb - va) * 8), m.streaming);
          if constexpr (kDelta) {
            const int64_t ca = p0 & ~int64_t(7), cb = (p1 + 7) & ~int64_t(7);
            prefetch_l2(m.sell_dcol + ca, (uint32_t)((cb - ca) * 2), m.streaming);
          } else {
            const int64_t ca = p0 & ~int64_t(3), cb = (p1 + 3) & ~int64_t(3);
            prefetch_l2(m.sell_col + ca, (uint32_t)((cb - ca) * 4), m.streaming);
          }
        }
      }
    }
  }
  pdl_wait();
  pdl_trigger();
  // SMG_X_PREFETCH: the first CTAs pull the gathered vector x (produced by the
  // previous kernel, so only after the dependency wait) into L2 in
  // xpf_chunk-byte pieces -- a cold x would otherwise be gathered from HBM
  // with a dependent round trip per entry
  if (xpf_chunk > 0 && threadIdx.x == 32) {
    const int64_t xb = m.ncols * 8;
    const int64_t off = (int64_t)w * xpf_chunk;
    if (off < xb) {
      const int64_t len = min((int64_t)xpf_chunk, xb - off) & ~int64_t(15);
      if (len > 0) prefetch_l2(reinterpret_cast<const char*>(x) + off, (uint32_t)len, false);
    }
  }
  const int32_t grow = w * kSellWindow + rl;
  const bool has_row = rl >= 0;
  SMG_DCHECK(!has_row || grow < m.nrows);
  SMG_DCHECK(se >= sb && ((se - sb) & 31) == 0);
  const bool write = has_row && !(ea.skip_rows && ea.skip_rows[grow]);
  double bv = 0.0, uv = 0.0, dv = 0.0, ov = 0.0, inv = 0.0;
  if (write) {
    if constexpr (T::kB) bv = ea.stream_vec ? __ldcs(ea.b + grow) : ea.b[grow];
    if constexpr (T::kU) uv = ea.u_in[grow];
    if constexpr (T::kD) dv = ea.stream_vec ? __ldcs(ea.d + grow) : ea.d[grow];
    if constexpr (T::kOut) ov = (ea.u_in ? ea.u_in : ea.out)[grow];  // prolong-add in or out of place
    if constexpr (T::kDiag) inv = ea.stream_vec ? __ldcs(m.inv_diag + grow) : m.inv_diag[grow];
    if constexpr (T::kDiagVec) inv = ea.inv_diag[grow];
  }
  double sum = 0.0;
#pragma unroll
  for (int j = 0; j < kSellPre; ++j) {
    const int32_t c = decode(c0[j]);
    SMG_DCHECK(c < m.ncols);
    if (c >= 0) sum = __dadd_rn(sum, __dmul_rn(v0[j], __ldg(x + c)));
  }
  if constexpr (kPipe) {
    auto ldb = [&](int j0, int32_t* cc, double* vv) {
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int j = j0 + u;
        cc[u] = kPad;
        vv[u] = 0.0;
        if (j < width) {
          cc[u] = ldraw(j);
          vv[u] = ldval(j);
        }
      }
    };
    int32_t c[kUnroll];
    double v[kUnroll];
    ldb(kSellPre, c, v);
    for (int j0 = kSellPre; j0 < width; j0 += kUnroll) {
      int32_t cn[kUnroll];
      double vn[kUnroll];
      ldb(j0 + kUnroll, cn, vn);
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int32_t cu = decode(c[u]);
        if (cu >= 0) sum = __dadd_rn(sum, __dmul_rn(v[u], __ldg(x + cu)));
      }
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        c[u] = cn[u];
        v[u] = vn[u];
      }
    }
    if (write) epilogue<E>(ea, grow, sum, inv, bv, uv, dv, ov);
    return;
  }
#pragma unroll kUnroll
  for (int j = kSellPre; j < width; ++j) {
    const int32_t raw = ldraw(j);
    const double v = ldval(j);
    const int32_t c = decode(raw);
    SMG_DCHECK(c < m.ncols);
    if (c >= 0) sum = __dadd_rn(sum, __dmul_rn(v, __ldg(x + c)));
  }
  if (write) epilogue<E>(ea, grow, sum, inv, bv, uv, dv, ov);
}

// SELL-8x4 (DevCsr::sell_lanes == 4): operators with long rows but too few
// rows for one thread per row to fill the GPU (C2 levels 2-3, C3 level 1, C4
// level 2).  One CTA per window of 64 rows, warp k = slice k of 8 rows, 4
// lanes per row: the lanes of a row load entries 4b..4b+3 of batch b
// (coalesced: a batch of the slice is 32 contiguous entries) and form their
// products in parallel -- the serial load chain per row is a quarter of
// sell_kernel's -- then the row's first lane adds the four products in column
// order (shuffles; padding entries, column -1, are skipped via a ballot), so
// every row is still one sequential sum in scipy's order, bit for bit.
constexpr int kSell4Pre = 2;   // batches loaded before the dependency wait

template <Epi E, bool kPf, int kUnroll>
__global__ void __launch_bounds__(kThreads, kUnroll <= 2 ? 8 : 4)
sell4_kernel(const DevCsr m, const double* __restrict__ x, const EpiArgs ea, int pf_dist)
{
  using T = EpiTraits<E>;
  const int w = blockIdx.x;
  const int k = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t sb = m.sell_ptr[(int64_t)w * kSellSlices + k];
  const int64_t se = m.sell_ptr[(int64_t)w * kSellSlices + k + 1];
  const int width = (int)((se - sb) >> 5);   // batches of 4 entries per row
  const int g0 = lane & ~3;                  // first lane of this row's group
  const int rl = m.sell_perm[(int64_t)w * kSell4Window + k * 8 + (lane >> 2)];
  const int32_t* __restrict__ cp = m.sell_col + sb + lane;
  const double* __restrict__ vp = m.sell_val + sb + lane;
  auto ld = [&](int j, int32_t& c, double& v) {
    c = -1;
    v = 0.0;
    if (j < width) {
      if (m.streaming) {
        c = __ldcs(cp + j * 32);
        v = __ldcs(vp + j * 32);
      } else {
        c = __ldg(cp + j * 32);
        v = __ldg(vp + j * 32);
      }
    }
  };
  int32_t c0[kSell4Pre];
  double v0[kSell4Pre];
#pragma unroll
  for (int j = 0; j < kSell4Pre; ++j) ld(j, c0[j], v0[j]);
  if constexpr (kPf) {
    if (threadIdx.x == 0) {
      const int wp = w + pf_dist;
      if (wp < m.sell_nwin) {
        const int64_t p0 = m.sell_ptr[(int64_t)wp * kSellSlices];
        const int64_t p1 = m.sell_ptr[(int64_t)(wp + 1) * kSellSlices];
        if (p1 > p0 && p1 - p0 <= (int64_t)kTileNnz * 16) {
          const int64_t va = p0 & ~int64_t(1), vb = (p1 + 1) & ~int64_t(1);
          const int64_t ca = p0 & ~int64_t(3), cb = (p1 + 3) & ~int64_t(3);
          prefetch_l2(m.sell_val + va, (uint32_t)((vb - va) * 8), m.streaming);
          prefetch_l2(m.sell_col + ca, (uint32_t)((cb - ca) * 4), m.streaming);
        }
      }
    }
  }
  pdl_wait();
  pdl_trigger();
  const int32_t grow = w * kSell4Window + rl;
  const bool owner = (lane & 3) == 0;
  const bool write = owner && rl >= 0 && !(ea.skip_rows && ea.skip_rows[grow]);
  double bv = 0.0, uv = 0.0, dv = 0.0, ov = 0.0, inv = 0.0;
  if (write) {
    if constexpr (T::kB) bv = ea.b[grow];
    if constexpr (T::kU) uv = ea.u_in[grow];
    if constexpr (T::kD) dv = ea.d[grow];
    if constexpr (T::kOut) ov = (ea.u_in ? ea.u_in : ea.out)[grow];
    if constexpr (T::kDiag) inv = m.inv_diag[grow];
    if constexpr (T::kDiagVec) inv = ea.inv_diag[grow];
  }
  double sum = 0.0;
  // the group's four products of one batch, added in entry (column) order
  auto add4 = [&](double p, bool valid) {
    const unsigned msk = __ballot_sync(0xffffffffu, valid);
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const double q = __shfl_sync(0xffffffffu, p, g0 + t);
      if ((msk >> (g0 + t)) & 1u) sum = __dadd_rn(sum, q);
    }
  };
  {
    double p0[kSell4Pre];
#pragma unroll
    for (int j = 0; j < kSell4Pre; ++j)
      p0[j] = c0[j] >= 0 ? __dmul_rn(v0[j], __ldg(x + c0[j])) : 0.0;
#pragma unroll
    for (int j = 0; j < kSell4Pre; ++j) add4(p0[j], c0[j] >= 0);
  }
  for (int j0 = kSell4Pre; j0 < width; j0 += kUnroll) {
    int32_t c[kUnroll];
    double v[kUnroll], p[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) ld(j0 + u, c[u], v[u]);
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) p[u] = c[u] >= 0 ? __dmul_rn(v[u], __ldg(x + c[u])) : 0.0;
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) add4(p[u], c[u] >= 0);
  }
  if (write) epilogue<E>(ea, grow, sum, inv, bv, uv, dv, ov);
}

static int g_sm_count = 0;
static int g_prefetch = -1;
static int g_pdl = -1;

static bool env_flag(int& cache, const char* name, int dflt)
{
  if (cache < 0) {
    const char* v = getenv(name);
    cache = v ? atoi(v) : dflt;
  }
  return cache != 0;
}

// SMG_L2_PERSIST_MB (default 0 = off): a persisting-L2 carve-out of that size;
// the sweeps of streamed operators then mark their gathered vector x with a
// persisting access-policy window (and everything else they touch keeps its
// normal / evict-first treatment), so the operator stream cannot displace x
// between the gathers of neighbouring rows.  Set up outside any stream
// capture (operator creation calls configure_l2_persist).
static size_t g_persist_bytes = 0;
static size_t g_persist_window = 0;

void configure_l2_persist()
{
  static bool done = false;
  if (done) return;
  done = true;
  const char* v = getenv("SMG_L2_PERSIST_MB");
  const long mb = v ? atol(v) : 0;
  if (mb <= 0) return;
  int dev = 0, maxp = 0, maxw = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, dev);
  cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, dev);
  size_t want = (size_t)mb << 20;
  if (want > (size_t)maxp) want = (size_t)maxp;
  if (want == 0 || cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want) != cudaSuccess) {
    cudaGetLastError();
    return;
  }
  g_persist_bytes = want;
  g_persist_window = (size_t)maxw;
}

template <Epi E>
static cudaError_t launch_t_sell(const DevCsr& m, const double* x, const EpiArgs& ea,
                                 cudaLaunchConfig_t cfg, bool pf, int waves);

template <Epi E>
static cudaError_t launch_t(const DevCsr& m, const double* x, const EpiArgs& ea, cudaStream_t s)
{
  if (m.ntiles == 0 && !(m.sell && m.sell_nwin > 0)) return cudaSuccess;
  if (g_sm_count == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sm_count, cudaDevAttrMultiProcessorCount, dev);
    if (g_sm_count <= 0) g_sm_count = 148;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)m.ntiles);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[3];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = env_flag(g_pdl, "SMG_PDL", 1) ? 1 : 0;
  // L1 / shared-memory split per launch (SMG_CARVEOUT: 0 = driver's choice,
  // 1 = SELL kernels, which use no shared memory, ask for the largest L1, so
  // the x gathers do not inherit the small L1 a shared-memory-heavy kernel
  // (patch_kernel, csr_stage_kernel) left on the SM; 2 = also the tile
  // kernels ask for just their own 4 CTAs' worth)
  static const int carve = [] {
    const char* v = getenv("SMG_CARVEOUT");
    return v ? atoi(v) : 1;
  }();
  if (carve >= 1 && (m.sell || (carve >= 2 && m.stage_cap == 0))) {
    cudaLaunchAttribute& a = attr[cfg.numAttrs++];
    a.id = cudaLaunchAttributePreferredSharedMemoryCarveout;
    a.val.sharedMemCarveout = m.sell ? 0u : (m.multichunk ? 60u : 30u);
  }
  if (g_persist_bytes > 0 && m.streaming && m.ncols > 0) {
    size_t bytes = (size_t)m.ncols * 8;
    if (bytes > g_persist_window) bytes = g_persist_window;
    cudaLaunchAttribute& a = attr[cfg.numAttrs++];
    a.id = cudaLaunchAttributeAccessPolicyWindow;
    a.val.accessPolicyWindow.base_ptr = const_cast<double*>(x);
    a.val.accessPolicyWindow.num_bytes = bytes;
    a.val.accessPolicyWindow.hitRatio =
        bytes <= g_persist_bytes ? 1.0f : (float)((double)g_persist_bytes / (double)bytes);
    a.val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    a.val.accessPolicyWindow.missProp = cudaAccessPropertyNormal;
  }
  static const int waves = [] {
    const char* v = getenv("SMG_PF_WAVES");
    const int w = v ? atoi(v) : 1;
    return w > 0 ? w : 1;
  }();
  const bool pf = env_flag(g_prefetch, "SMG_L2_PREFETCH", 1);
  // streamed SELL operators read their per-row vectors evict-first so x
  // keeps the L2 (C2 fine step 31.5 -> 29.5 us; profiles/r01/ab_evictvec/)
  static const int evict_vec = [] {
    const char* v = getenv("SMG_EVICT_VEC");
    return v ? atoi(v) : 1;
  }();
  if (m.sell && m.streaming && evict_vec) {
    EpiArgs e2 = ea;
    e2.stream_vec = true;
    return launch_t_sell<E>(m, x, e2, cfg, pf, waves);
  }
  return launch_t_sell<E>(m, x, ea, cfg, pf, waves);
}

template <Epi E>
static cudaError_t launch_t_sell(const DevCsr& m, const double* x, const EpiArgs& ea,
                                 cudaLaunchConfig_t cfg, bool pf, int waves)
{
  const int dist = g_sm_count * kMinBlocks * waves;  // resident waves ahead (default one)
  if (m.sell && m.sell_lanes == 4) {
    cfg.gridDim = dim3((unsigned)m.sell_nwin);
    cfg.blockDim = dim3(kThreads);
    if (m.sell_unroll >= 4) {
      const int sdist = g_sm_count * 4 * waves;
      return pf ? cudaLaunchKernelEx(&cfg, sell4_kernel<E, true, 4>, m, x, ea, sdist)
                : cudaLaunchKernelEx(&cfg, sell4_kernel<E, false, 4>, m, x, ea, sdist);
    }
    const int sdist = g_sm_count * 8 * waves;
    return pf ? cudaLaunchKernelEx(&cfg, sell4_kernel<E, true, 2>, m, x, ea, sdist)
              : cudaLaunchKernelEx(&cfg, sell4_kernel<E, false, 2>, m, x, ea, sdist);
  }
  if (m.sell) {
    cfg.gridDim = dim3((unsigned)m.sell_nwin);
    cfg.blockDim = dim3(kSellWindow);
    // SMG_X_PREFETCH (0 = off, 1 = on): x in chunks over the first resident wave
    static const int xpf_env = [] {
      const char* v = getenv("SMG_X_PREFETCH");
      return v ? atoi(v) : 0;
    }();
    int xpf = 0;
    if (xpf_env && ((uintptr_t)x & 15) == 0) {
      const int64_t ctas = std::min<int64_t>(m.sell_nwin, (int64_t)g_sm_count * 4);
      xpf = (int)(((m.ncols * 8 + ctas - 1) / ctas + 15) & ~int64_t(15));
    }
#define SMG_SELL_LAUNCH(U, P)                                                              \
  do {                                                                                     \
    if (m.sell_delta)                                                                      \
      return pf ? cudaLaunchKernelEx(&cfg, sell_kernel<E, true, U, P, true>, m, x, ea, sdist, xpf) \
                : cudaLaunchKernelEx(&cfg, sell_kernel<E, false, U, P, true>, m, x, ea, sdist, xpf); \
    return pf ? cudaLaunchKernelEx(&cfg, sell_kernel<E, true, U, P, false>, m, x, ea, sdist, xpf) \
              : cudaLaunchKernelEx(&cfg, sell_kernel<E, false, U, P, false>, m, x, ea, sdist, xpf); \
  } while (0)
    if (m.sell_unroll >= 16) {
      const int sdist = g_sm_count * 2 * waves;
      SMG_SELL_LAUNCH(16, false);
    }
    if (m.sell_unroll >= 8) {
      const int sdist = g_sm_count * 4 * waves;
      // SMG_SELL_PIPE: unset = per operator (DevCsr::sell_pipe, set at upload),
      // 0 = never, 4 / 6 = that depth for every 8-deep operator
      static const int pipe_env = [] {
        const char* v = getenv("SMG_SELL_PIPE");
        return v ? atoi(v) : -1;
      }();
      const int pipe = pipe_env >= 0 ? pipe_env : m.sell_pipe;
      if (pipe >= 6) SMG_SELL_LAUNCH(6, true);
      if (pipe > 0) SMG_SELL_LAUNCH(4, true);
      SMG_SELL_LAUNCH(8, false);
    }
    const int sdist = g_sm_count * 8 * waves;
    SMG_SELL_LAUNCH(4, false);
#undef SMG_SELL_LAUNCH
  }
  if (m.stage_cap > 0) {
    const int smem = (int)sizeof(double) * m.stage_cap;
    static const cudaError_t attr_rc = [] {
      const int cap = (int)sizeof(double) * kStageMaxNnz;
      cudaError_t e = cudaFuncSetAttribute(csr_stage_kernel<E, true>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, cap);
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute(csr_stage_kernel<E, false>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, cap);
      return e;
    }();
    if (attr_rc != cudaSuccess) return attr_rc;
    cfg.dynamicSmemBytes = (size_t)smem;
    const int sdist = g_sm_count * kStageCtas * waves;
    return pf ? cudaLaunchKernelEx(&cfg, csr_stage_kernel<E, true>, m, x, ea, sdist)
              : cudaLaunchKernelEx(&cfg, csr_stage_kernel<E, false>, m, x, ea, sdist);
  }
  if (m.fixed) {
    if (m.multichunk)
      return pf ? cudaLaunchKernelEx(&cfg, csr_tile_kernel<E, true, true, true>, m, x, ea, dist)
                : cudaLaunchKernelEx(&cfg, csr_tile_kernel<E, false, true, true>, m, x, ea, dist);
    return pf ? cudaLaunchKernelEx(&cfg, csr_tile_kernel<E, true, false, true>, m, x, ea, dist)
              : cudaLaunchKernelEx(&cfg, csr_tile_kernel<E, false, false, true>, m, x, ea, dist);
  }
  if (m.multichunk) {
    static const int ws = [] {
      const char* v = getenv("SMG_TILE_WS");
      return v ? atoi(v) : 0;
    }();
    if (ws) {
      constexpr int kWsSmem = (int)(sizeof(double) * kWsSlots * kTileNnz + 2 * kWsSlots * sizeof(uint64_t));
      static const cudaError_t attr_rc = [] {
        cudaError_t e = cudaFuncSetAttribute(csr_ws_kernel<E, true>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, kWsSmem);
        if (e == cudaSuccess)
          e = cudaFuncSetAttribute(csr_ws_kernel<E, false>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, kWsSmem);
        return e;
      }();
      if (attr_rc != cudaSuccess) return attr_rc;
      cfg.dynamicSmemBytes = kWsSmem;
      return pf ? cudaLaunchKernelEx(&cfg, csr_ws_kernel<E, true>, m, x, ea, dist)
                : cudaLaunchKernelEx(&cfg, csr_ws_kernel<E, false>, m, x, ea, dist);
    }
    return pf ? cudaLaunchKernelEx(&cfg, csr_tile_kernel<E, true, true, false>, m, x, ea, dist)
              : cudaLaunchKernelEx(&cfg, csr_tile_kernel<E, false, true, false>, m, x, ea, dist);
  }
  return pf ? cudaLaunchKernelEx(&cfg, csr_tile_kernel<E, true, false, false>, m, x, ea, dist)
            : cudaLaunchKernelEx(&cfg, csr_tile_kernel<E, false, false, false>, m, x, ea, dist);
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
    case Epi::kRestrictFirst: return launch_t<Epi::kRestrictFirst>(m, x, ea, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace smg
