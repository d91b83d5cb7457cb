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
// in column order, separately rounded multiply and add):
//   * phase 1: the tile's exact products val*x[col] (__dmul_rn) are formed by
//     all threads and staged in shared memory -- products are independently
//     rounded, so any thread may form any of them;
//   * phase 2: each thread owns one row and adds that row's products in
//     column order with __dadd_rn (no FMA contraction anywhere);
//   * the epilogue reproduces numpy's elementwise expression order, with IEEE
//     division (__ddiv_rn) for 1/a_ii and /theta.
//
// B200 data movement: the kernel is persistent (2 CTAs per SM, static
// round-robin over tiles) and streams every tile's values, column indices and
// row offsets HBM -> shared memory with 1D TMA bulk copies
// (cp.async.bulk ... mbarrier::complete_tx) into a kStages-deep ring, issued
// kStages tiles ahead by one elected thread, so HBM latency is overlapped with
// the gather / sum / epilogue of earlier tiles.  Only the x gathers (L2/L1
// resident) and the per-row epilogue vectors go through the LSU; the
// epilogue operands are prefetched into registers before the tile's barrier
// wait.  Tiles whose nonzeros exceed kTileNnz (a single row longer than the
// ring slot) take a chunked fallback that reads global memory directly.
#include "smg_internal.cuh"

#include <cstdlib>

namespace smg {

// ---------------------------------------------------------------------------
// PTX helpers (mbarrier + 1D bulk TMA)
__device__ __forceinline__ uint32_t smem_u32(const void* p)
{
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count)
{
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void fence_mbar_init()
{
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes)
{
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar)
{
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity)
{
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async()
{
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// programmatic dependent launch: no-ops when launched without the attribute
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger()
{
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ---------------------------------------------------------------------------
template <Epi E>
struct EpiTraits {
  static constexpr bool kDiag = (E == Epi::kJacobi || E == Epi::kChebFirst || E == Epi::kChebNext);
  static constexpr bool kB = (E != Epi::kSpmv && E != Epi::kAddTo && E != Epi::kRestrictFirst);
  static constexpr bool kU = (E == Epi::kJacobi || E == Epi::kChebFirst || E == Epi::kChebNext);
  static constexpr bool kD = (E == Epi::kChebNext);
  static constexpr bool kOut = (E == Epi::kAddTo);
  static constexpr bool kDiagVec = (E == Epi::kRestrictFirst);
  static constexpr bool kInv = kDiag || kDiagVec;   // needs 1/a_ii
};

// ring-slot geometry (bytes are multiples of 16 as cp.async.bulk requires)
constexpr int kValCap = kTileNnz + 2;        // doubles (start aligned down to 16 B)
constexpr int kColCap = kTileNnz + 4;        // int32
constexpr int kRpCap = kRowsPerTile + 4;     // int64 (rows r0..r1 inclusive + alignment)
constexpr int kSlotBytes = kValCap * 8 + kColCap * 4 + kRpCap * 8;
static_assert(kSlotBytes % 16 == 0, "slot must keep 16-byte alignment");
constexpr int kSmemBytes = kStages * kSlotBytes + kTileNnz * 8;
constexpr int kDefaultVariant = 10;
constexpr int kFlatMinBlocks = 6;   // <= 40 registers: 6 CTAs (48 warps) per SM

template <Epi E>
__device__ __forceinline__ void epilogue(const DevCsr& m, const EpiArgs& ea, int32_t row, double sum,
                                         double dg, double bv, double uv, double dv, double ov)
{
  if constexpr (E == Epi::kSpmv) {
    ea.out[row] = sum;
  } else if constexpr (E == Epi::kResidual) {
    ea.out[row] = __dsub_rn(bv, sum);
  } else if constexpr (E == Epi::kAddTo) {
    ea.out[row] = __dadd_rn(ov, sum);
  } else if constexpr (E == Epi::kRestrictFirst) {
    ea.b_out[row] = sum;
    const double inv = dg;
    const double t = __dmul_rn(inv, __dsub_rn(sum, 0.0));
    const double d = __ddiv_rn(t, ea.theta);
    if (ea.d) ea.d[row] = d;
    ea.out[row] = __dadd_rn(0.0, d);
  } else {
    const double inv = dg;  // 1.0 / a_ii, precomputed with the same IEEE division
    const double t = __dmul_rn(inv, __dsub_rn(bv, sum));
    if constexpr (E == Epi::kJacobi) {
      ea.out[row] = __dadd_rn(uv, __ddiv_rn(t, ea.theta));
    } else if constexpr (E == Epi::kChebFirst) {
      const double d = __ddiv_rn(t, ea.theta);
      ea.d[row] = d;
      ea.out[row] = __dadd_rn(uv, d);
    } else {  // kChebNext
      const double d = __dadd_rn(__dmul_rn(ea.c1, dv), __dmul_rn(ea.c2, t));
      ea.d[row] = d;
      ea.out[row] = __dadd_rn(uv, d);
    }
  }
}

// producer: issue the bulk copies of tile t into ring slot s
__device__ __forceinline__ void issue_tile(const DevCsr& m, int t, unsigned char* slot,
                                           uint64_t* bar)
{
  const int32_t r0 = m.tile_row[t];
  const int32_t r1 = m.tile_row[t + 1];
  const int64_t e0 = m.tile_nz[t];
  const int64_t e1 = m.tile_nz[t + 1];
  if (e1 - e0 > kTileNnz) {  // long tile: consumer reads global memory directly
    mbar_arrive_expect_tx(bar, 0);
    return;
  }
  const int64_t va = e0 & ~int64_t(1), vb = (e1 + 1) & ~int64_t(1);
  const int64_t ca = e0 & ~int64_t(3), cb = (e1 + 3) & ~int64_t(3);
  const int64_t ra = r0 & ~1, rb = (int64_t(r1) + 2) & ~int64_t(1);
  const uint32_t bv = (uint32_t)((vb - va) * 8), bc = (uint32_t)((cb - ca) * 4),
                 br = (uint32_t)((rb - ra) * 8);
  mbar_arrive_expect_tx(bar, bv + bc + br);
  double* sval = reinterpret_cast<double*>(slot);
  int32_t* scol = reinterpret_cast<int32_t*>(slot + kValCap * 8);
  int64_t* srp = reinterpret_cast<int64_t*>(slot + kValCap * 8 + kColCap * 4);
  if (bv) bulk_g2s(sval, m.val + va, bv, bar);
  if (bc) bulk_g2s(scol, m.col + ca, bc, bar);
  bulk_g2s(srp, m.rowptr + ra, br, bar);
}

template <Epi E>
__global__ void __launch_bounds__(kThreads, kCtasPerSm)
csr_stream_kernel(const DevCsr m, const double* __restrict__ x, const EpiArgs ea)
{
  using T = EpiTraits<E>;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint64_t bars[kStages];
  double* s_prod = reinterpret_cast<double*>(smem + kStages * kSlotBytes);

  const int ntiles = m.ntiles;
  const int G = gridDim.x;
  const int first = blockIdx.x;
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      const int t = first + s * G;
      if (t < ntiles) issue_tile(m, t, smem + s * kSlotBytes, &bars[s]);
    }
  }

  int it = 0;
  for (int t = first; t < ntiles; t += G, ++it) {
    const int s = it % kStages;
    const uint32_t parity = (uint32_t)((it / kStages) & 1);
    unsigned char* slot = smem + s * kSlotBytes;
    const int32_t r0 = m.tile_row[t];
    const int32_t r1 = m.tile_row[t + 1];
    const int32_t row = r0 + tid;
    const bool has_row = row < r1;
    // prefetch the row's epilogue operands while the tile is in flight
    double bv = 0.0, uv = 0.0, dv = 0.0, ov = 0.0;
    if (has_row) {
      if constexpr (T::kB) bv = ea.b[row];
      if constexpr (T::kU) uv = ea.u_in[row];
      if constexpr (T::kD) dv = ea.d[row];
      if constexpr (T::kOut) ov = ea.out[row];
    }
    const int64_t e0 = m.tile_nz[t];
    const int64_t e1 = m.tile_nz[t + 1];
    double sum = 0.0;
    double dg = 0.0;
    if (has_row) {
      if constexpr (T::kDiag) dg = m.inv_diag[row];
      if constexpr (T::kDiagVec) dg = ea.inv_diag[row];
    }
    mbar_wait(&bars[s], parity);
    if (e1 - e0 <= kTileNnz) {
      const double* sval = reinterpret_cast<const double*>(slot) + (e0 & 1);
      const int32_t* scol = reinterpret_cast<const int32_t*>(slot + kValCap * 8) + (e0 & 3);
      const int64_t* srp =
          reinterpret_cast<const int64_t*>(slot + kValCap * 8 + kColCap * 4) + (r0 & 1);
      const int cnt = (int)(e1 - e0);
      // phase 1: gather x, exact products
#pragma unroll
      for (int i = 0; i < kItems; ++i) {
        const int k = i * kThreads + tid;
        if (k < cnt) s_prod[k] = __dmul_rn(sval[k], __ldg(x + scol[k]));
      }
      __syncthreads();
      // phase 2: sequential per-row sum in column order
      if (has_row) {
        const int a = (int)(srp[tid] - e0);
        const int bnd = (int)(srp[tid + 1] - e0);
        for (int j = a; j < bnd; ++j) sum = __dadd_rn(sum, s_prod[j]);
      }
    } else {
      // long tile (a row longer than one ring slot): chunked, global reads
      int64_t lo = 0, hi = 0;
      if (has_row) {
        lo = m.rowptr[row];
        hi = m.rowptr[row + 1];
      }
      for (int64_t cs = e0; cs < e1; cs += kTileNnz) {
        const int64_t rem = e1 - cs;
        const int cnt = rem < (int64_t)kTileNnz ? (int)rem : kTileNnz;
        for (int k = tid; k < cnt; k += kThreads)
          s_prod[k] = __dmul_rn(__ldg(m.val + cs + k), __ldg(x + __ldg(m.col + cs + k)));
        __syncthreads();
        if (has_row) {
          const int64_t a = lo > cs ? lo : cs;
          const int64_t bnd = hi < cs + cnt ? hi : cs + cnt;
          for (int64_t j = a; j < bnd; ++j) sum = __dadd_rn(sum, s_prod[j - cs]);
        }
        __syncthreads();
      }
    }
    if (has_row) epilogue<E>(m, ea, row, sum, dg, bv, uv, dv, ov);
    __syncthreads();  // slot s and s_prod are free again
    if (tid == 0) {
      const int tn = t + kStages * G;
      if (tn < ntiles) {
        fence_proxy_async();
        issue_tile(m, tn, slot, &bars[s]);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Non-persistent variants: one tile per CTA.
//   kTma = false: coalesced LSU loads of (val, col) straight into registers;
//   kTma = true : one elected thread issues the tile's bulk copies, the other
//                 threads prefetch the epilogue operands meanwhile.
// Both start every independent load (row bounds, epilogue vectors, tile
// values) as early as possible so a tile costs ~3 memory latencies.
constexpr int kFlatTmaSmem = kSlotBytes + kTileNnz * 8;

__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes)
{
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

template <Epi E, bool kTma, int kMinB, bool kPf = false, bool kPfVec = false>
__global__ void __launch_bounds__(kThreads, kMinB)
csr_flat_kernel(const DevCsr m, const double* __restrict__ x, const EpiArgs ea, int pf_dist = 0)
{
  using T = EpiTraits<E>;
  extern __shared__ __align__(128) unsigned char fsmem[];
  __shared__ uint64_t bar;
  __shared__ double s_prod_static[kTma ? 1 : kTileNnz];
  const int t = blockIdx.x;
  const int tid = threadIdx.x;
  // ---- operator data (never written by any kernel): safe before the
  //      programmatic-dependency wait, so it overlaps the previous kernel's tail
  const int32_t r0 = m.tile_row[t];
  const int32_t r1 = m.tile_row[t + 1];
  const int64_t e0 = m.tile_nz[t];
  const int64_t e1 = m.tile_nz[t + 1];
  const bool longtile = e1 - e0 > kTileNnz;
  const int cnt = (int)(e1 - e0);
  if constexpr (kTma) {
    if (tid == 0) {
      mbar_init(&bar, 1);
      fence_mbar_init();
    }
    __syncthreads();
    if (tid == 0) issue_tile(m, t, fsmem, &bar);
  }
  const int32_t row = r0 + tid;
  const bool has_row = row < r1;
  int64_t lo = 0, hi = 0;
  if (has_row && (!kTma || longtile)) {
    lo = m.rowptr[row];
    hi = m.rowptr[row + 1];
  }
  int32_t c[kTma ? 1 : kItems];
  double v[kTma ? 1 : kItems];
  if constexpr (!kTma) {
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
      const int k = i * kThreads + tid;
      c[i] = 0;
      v[i] = 0.0;
      if (!longtile && k < cnt) {
        c[i] = __ldg(m.col + e0 + k);
        v[i] = __ldg(m.val + e0 + k);
      }
    }
  }
  if constexpr (kPf) {
    // pull the tile that will start one resident-wave later into L2 (bulk
    // prefetch: no registers, no shared memory), so its CTA's loads hit L2
    if (tid == 0) {
      const int tp = t + pf_dist;
      if (tp < m.ntiles) {
        const int64_t p0 = m.tile_nz[tp], p1 = m.tile_nz[tp + 1];
        if (p1 - p0 <= kTileNnz && p1 > p0) {
          const int64_t va = p0 & ~int64_t(1), vb = (p1 + 1) & ~int64_t(1);
          const int64_t ca = p0 & ~int64_t(3), cb = (p1 + 3) & ~int64_t(3);
          prefetch_l2(m.val + va, (uint32_t)((vb - va) * 8));
          prefetch_l2(m.col + ca, (uint32_t)((cb - ca) * 4));
        }
      }
    }
  }
  // ---- vectors produced by earlier kernels: after the dependency wait
  pdl_wait();
  pdl_trigger();
  if constexpr (kPfVec) {
    // the same future tile's per-row epilogue vectors (contiguous rows)
    if (tid == 0) {
      const int tp = t + pf_dist;
      if (tp < m.ntiles) {
        const int32_t ra = m.tile_row[tp] & ~1, rb = m.tile_row[tp + 1] & ~1;
        if (rb > ra) {
          const uint32_t nb = (uint32_t)(rb - ra) * 8;
          auto pf = [&](const double* v) {
            if ((reinterpret_cast<uintptr_t>(v) & 15) == 0) prefetch_l2(v + ra, nb);
          };
          if constexpr (T::kB) pf(ea.b);
          if constexpr (T::kU) pf(ea.u_in);
          if constexpr (T::kD) pf(ea.d);
          if constexpr (T::kOut) pf(ea.out);
          if constexpr (T::kDiag) pf(m.inv_diag);
          if constexpr (T::kDiagVec) pf(ea.inv_diag);
        }
      }
    }
  }
  double bv = 0.0, uv = 0.0, dv = 0.0, ov = 0.0;
  double sum = 0.0;
  double dg = 0.0;
  if (has_row) {
    if constexpr (T::kB) bv = ea.b[row];
    if constexpr (T::kU) uv = ea.u_in[row];
    if constexpr (T::kD) dv = ea.d[row];
    if constexpr (T::kOut) ov = ea.out[row];
    if constexpr (T::kDiag) dg = m.inv_diag[row];
    if constexpr (T::kDiagVec) dg = ea.inv_diag[row];
  }
  double* s_prod = kTma ? reinterpret_cast<double*>(fsmem + kSlotBytes) : s_prod_static;
  if (!longtile) {
    if constexpr (kTma) {
      mbar_wait(&bar, 0);
      const double* vals = reinterpret_cast<const double*>(fsmem) + (e0 & 1);
      const int32_t* cols = reinterpret_cast<const int32_t*>(fsmem + kValCap * 8) + (e0 & 3);
      const int64_t* srp =
          reinterpret_cast<const int64_t*>(fsmem + kValCap * 8 + kColCap * 4) + (r0 & 1);
      if (has_row) {
        lo = srp[tid];
        hi = srp[tid + 1];
      }
#pragma unroll
      for (int i = 0; i < kItems; ++i) {
        const int k = i * kThreads + tid;
        if (k < cnt) s_prod[k] = __dmul_rn(vals[k], __ldg(x + cols[k]));
      }
    } else {
#pragma unroll
      for (int i = 0; i < kItems; ++i) {
        const int k = i * kThreads + tid;
        if (k < cnt) s_prod[k] = __dmul_rn(v[i], __ldg(x + c[i]));
      }
    }
    __syncthreads();
    if (has_row) {
      const int a = (int)(lo - e0);
      const int bnd = (int)(hi - e0);
      for (int j = a; j < bnd; ++j) sum = __dadd_rn(sum, s_prod[j]);
    }
  } else {
    if constexpr (kTma) mbar_wait(&bar, 0);
    for (int64_t cs = e0; cs < e1; cs += kTileNnz) {
      const int64_t rem = e1 - cs;
      const int cn = rem < (int64_t)kTileNnz ? (int)rem : kTileNnz;
      for (int k = tid; k < cn; k += kThreads)
        s_prod[k] = __dmul_rn(__ldg(m.val + cs + k), __ldg(x + __ldg(m.col + cs + k)));
      __syncthreads();
      if (has_row) {
        const int64_t a = lo > cs ? lo : cs;
        const int64_t bnd = hi < cs + cn ? hi : cs + cn;
        for (int64_t j = a; j < bnd; ++j) sum = __dadd_rn(sum, s_prod[j - cs]);
      }
      __syncthreads();
    }
  }
  if (has_row) epilogue<E>(m, ea, row, sum, dg, bv, uv, dv, ov);
}

// ---------------------------------------------------------------------------
// Variant 5: persistent CTAs over CONTIGUOUS tile ranges with a TMA ring that
// carries everything a tile needs -- values, column indices, row offsets AND
// the per-row epilogue vectors (b, u, d, 1/a_ii, out) -- so each tile costs
// the consumers one barrier wait, the x gathers (L1/L2: neighbouring tiles
// share x) and the sums.  The CTA's tile descriptors are staged in shared
// memory up front, so the producer never waits on a dependent global load.
// Operator data of the first kPStages tiles is requested before the
// programmatic-dependency wait; vectors (produced by earlier kernels) after.
constexpr int kPStages = 2;
constexpr int kPCtas = 2;
constexpr int kVecCap = kRowsPerTile + 2;               // doubles per vector slot
constexpr int kPVal = 0;
constexpr int kPCol = kPVal + kValCap * 8;
constexpr int kPRp = kPCol + kColCap * 4;
constexpr int kPVec = kPRp + kRpCap * 8;
constexpr int kPSlot = kPVec + 4 * kVecCap * 8;          // 4 vector slots
constexpr int kPMaxTiles = 512;                          // descriptors staged per pass
static_assert(kPSlot % 16 == 0, "slot alignment");
constexpr int kPSmem = kPStages * kPSlot + kTileNnz * 8 + kPMaxTiles * 12 + 16;

template <Epi E>
struct PVecs {
  using T = EpiTraits<E>;
  // which vectors ride in the ring, in slot order
  static constexpr int kN = (T::kB ? 1 : 0) + (T::kU ? 1 : 0) + (T::kD ? 1 : 0) + (T::kOut ? 1 : 0) +
                            (T::kInv ? 1 : 0);
  __device__ static int fill(const DevCsr& m, const EpiArgs& ea, const double** v)
  {
    int k = 0;
    if constexpr (T::kB) v[k++] = ea.b;
    if constexpr (T::kU) v[k++] = ea.u_in;
    if constexpr (T::kD) v[k++] = ea.d;
    if constexpr (T::kOut) v[k++] = ea.out;
    if constexpr (T::kDiag) v[k++] = m.inv_diag;
    if constexpr (T::kDiagVec) v[k++] = ea.inv_diag;
    return k;
  }
};

__device__ __forceinline__ uint32_t tile_op_bytes(int32_t r0, int32_t r1, int64_t e0, int64_t e1)
{
  if (e1 - e0 > kTileNnz) return 0;
  const int64_t va = e0 & ~int64_t(1), vb = (e1 + 1) & ~int64_t(1);
  const int64_t ca = e0 & ~int64_t(3), cb = (e1 + 3) & ~int64_t(3);
  const int64_t ra = r0 & ~1, rb = (int64_t(r1) + 2) & ~int64_t(1);
  return (uint32_t)((vb - va) * 8 + (cb - ca) * 4 + (rb - ra) * 8);
}

__device__ __forceinline__ uint32_t tile_vec_bytes(int32_t r0, int32_t r1, int nvec)
{
  const int32_t ra = r0 & ~1, rb = r1 & ~1;
  return rb > ra ? (uint32_t)((rb - ra) * 8 * nvec) : 0u;
}

template <Epi E>
__global__ void __launch_bounds__(kThreads, kPCtas)
csr_pipe_kernel(const DevCsr m, const double* __restrict__ x, const EpiArgs ea)
{
  using T = EpiTraits<E>;
  using V = PVecs<E>;
  extern __shared__ __align__(128) unsigned char psm[];
  __shared__ uint64_t bars[kPStages];
  double* s_prod = reinterpret_cast<double*>(psm + kPStages * kPSlot);
  int32_t* s_trow = reinterpret_cast<int32_t*>(psm + kPStages * kPSlot + kTileNnz * 8);
  int64_t* s_tnz = reinterpret_cast<int64_t*>(psm + kPStages * kPSlot + kTileNnz * 8 + kPMaxTiles * 4 + 8);
  const int tid = threadIdx.x;
  const int G = gridDim.x;
  const int tb_all = (int)(((int64_t)m.ntiles * blockIdx.x) / G);
  const int te_all = (int)(((int64_t)m.ntiles * (blockIdx.x + 1)) / G);
  const double* vecs[5];
  V::fill(m, ea, vecs);
  bool vec_bulk = true;  // bulk copies need 16-byte aligned vector bases
  for (int k = 0; k < V::kN; ++k) vec_bulk &= ((reinterpret_cast<uintptr_t>(vecs[k]) & 15) == 0);

  if (tid == 0) {
    for (int s = 0; s < kPStages; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  int it = 0;  // global tile counter (ring position)
  bool waited = false;
  for (int tb = tb_all; tb < te_all; tb += kPMaxTiles) {
    const int te = min(te_all, tb + kPMaxTiles);
    const int nt = te - tb;
    __syncthreads();
    for (int i = tid; i <= nt; i += kThreads) {
      s_trow[i] = m.tile_row[tb + i];
      s_tnz[i] = m.tile_nz[tb + i];
    }
    __syncthreads();
    auto issue_op = [&](int i, int s) {
      const int32_t r0 = s_trow[i], r1 = s_trow[i + 1];
      const int64_t e0 = s_tnz[i], e1 = s_tnz[i + 1];
      unsigned char* slot = psm + s * kPSlot;
      const uint32_t bo = tile_op_bytes(r0, r1, e0, e1);
      const uint32_t bvv = vec_bulk ? tile_vec_bytes(r0, r1, V::kN) : 0u;
      mbar_arrive_expect_tx(&bars[s], bo + bvv);
      if (bo) {
        const int64_t va = e0 & ~int64_t(1), vb = (e1 + 1) & ~int64_t(1);
        const int64_t ca = e0 & ~int64_t(3), cb = (e1 + 3) & ~int64_t(3);
        const int64_t ra = r0 & ~1, rb = (int64_t(r1) + 2) & ~int64_t(1);
        if (vb > va) bulk_g2s(slot + kPVal, m.val + va, (uint32_t)((vb - va) * 8), &bars[s]);
        if (cb > ca) bulk_g2s(slot + kPCol, m.col + ca, (uint32_t)((cb - ca) * 4), &bars[s]);
        bulk_g2s(slot + kPRp, m.rowptr + ra, (uint32_t)((rb - ra) * 8), &bars[s]);
      }
    };
    auto issue_vec = [&](int i, int s) {
      const int32_t r0 = s_trow[i], r1 = s_trow[i + 1];
      const int32_t ra = r0 & ~1, rb = r1 & ~1;
      if (rb <= ra || !vec_bulk) return;
      unsigned char* slot = psm + s * kPSlot;
      for (int k = 0; k < V::kN; ++k)
        bulk_g2s(slot + kPVec + k * kVecCap * 8, vecs[k] + ra, (uint32_t)((rb - ra) * 8), &bars[s]);
    };
    if (tid == 0) {
      for (int j = 0; j < kPStages && j < nt; ++j) issue_op(j, (it + j) % kPStages);
    }
    if (!waited) {
      pdl_wait();
      pdl_trigger();
      waited = true;
    }
    if (tid == 0) {
      for (int j = 0; j < kPStages && j < nt; ++j) issue_vec(j, (it + j) % kPStages);
    }
    for (int i = 0; i < nt; ++i, ++it) {
      const int s = it % kPStages;
      const uint32_t parity = (uint32_t)((it / kPStages) & 1);
      unsigned char* slot = psm + s * kPSlot;
      const int32_t r0 = s_trow[i], r1 = s_trow[i + 1];
      const int64_t e0 = s_tnz[i], e1 = s_tnz[i + 1];
      const int32_t row = r0 + tid;
      const bool has_row = row < r1;
      const int32_t ra = r0 & ~1, rbv = vec_bulk ? (r1 & ~1) : r0;
      double sum = 0.0;
      mbar_wait(&bars[s], parity);
      // epilogue operands: from the ring, or (one odd trailing row) from global
      double ev[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
      if (has_row) {
        if (row < rbv) {
          const double* vs = reinterpret_cast<const double*>(slot + kPVec) + (row - ra);
#pragma unroll
          for (int k = 0; k < V::kN; ++k) ev[k] = vs[k * kVecCap];
        } else {
#pragma unroll
          for (int k = 0; k < V::kN; ++k) ev[k] = vecs[k][row];
        }
      }
      if (e1 - e0 <= kTileNnz) {
        const double* sval = reinterpret_cast<const double*>(slot + kPVal) + (e0 & 1);
        const int32_t* scol = reinterpret_cast<const int32_t*>(slot + kPCol) + (e0 & 3);
        const int64_t* srp = reinterpret_cast<const int64_t*>(slot + kPRp) + (r0 & 1);
        const int cnt = (int)(e1 - e0);
#pragma unroll
        for (int q = 0; q < kItems; ++q) {
          const int k = q * kThreads + tid;
          if (k < cnt) s_prod[k] = __dmul_rn(sval[k], __ldg(x + scol[k]));
        }
        __syncthreads();
        if (has_row) {
          const int a = (int)(srp[tid] - e0);
          const int bnd = (int)(srp[tid + 1] - e0);
          for (int j = a; j < bnd; ++j) sum = __dadd_rn(sum, s_prod[j]);
        }
      } else {
        int64_t lo = 0, hi = 0;
        if (has_row) {
          lo = m.rowptr[row];
          hi = m.rowptr[row + 1];
        }
        for (int64_t cs = e0; cs < e1; cs += kTileNnz) {
          const int64_t rem = e1 - cs;
          const int cn = rem < (int64_t)kTileNnz ? (int)rem : kTileNnz;
          for (int k = tid; k < cn; k += kThreads)
            s_prod[k] = __dmul_rn(__ldg(m.val + cs + k), __ldg(x + __ldg(m.col + cs + k)));
          __syncthreads();
          if (has_row) {
            const int64_t a = lo > cs ? lo : cs;
            const int64_t bnd = hi < cs + cn ? hi : cs + cn;
            for (int64_t j = a; j < bnd; ++j) sum = __dadd_rn(sum, s_prod[j - cs]);
          }
          __syncthreads();
        }
      }
      if (has_row) {
        int k = 0;
        double bv = 0.0, uv = 0.0, dv = 0.0, ov = 0.0, dg = 0.0;
        if constexpr (T::kB) bv = ev[k++];
        if constexpr (T::kU) uv = ev[k++];
        if constexpr (T::kD) dv = ev[k++];
        if constexpr (T::kOut) ov = ev[k++];
        if constexpr (T::kInv) dg = ev[k++];
        epilogue<E>(m, ea, row, sum, dg, bv, uv, dv, ov);
      }
      __syncthreads();  // slot s and s_prod are free again
      if (tid == 0 && i + kPStages < nt) {
        fence_proxy_async();
        issue_op(i + kPStages, s);
        issue_vec(i + kPStages, s);
      }
    }
  }
  if (!waited) {
    pdl_wait();
    pdl_trigger();
  }
}

static int g_sm_count = 0;

static int g_variant = -1;

static int spmv_variant()
{
  if (g_variant < 0) {
    const char* v = getenv("SMG_SPMV_VARIANT");
    g_variant = v ? atoi(v) : kDefaultVariant;
  }
  return g_variant;
}

static int g_pdl = -1;

static bool use_pdl()
{
  if (g_pdl < 0) {
    const char* v = getenv("SMG_PDL");
    g_pdl = v ? atoi(v) : 1;
  }
  return g_pdl != 0;
}

template <Epi E>
static cudaError_t launch_t(const DevCsr& m, const double* x, const EpiArgs& ea, cudaStream_t s)
{
  if (m.ntiles == 0) return cudaSuccess;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(csr_stream_kernel<E>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(csr_flat_kernel<E, true, 4>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, kFlatTmaSmem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  const int variant = spmv_variant();
  if (variant == 5) {
    static bool configured5 = false;
    if (!configured5) {
      cudaError_t e = cudaFuncSetAttribute(csr_pipe_kernel<E>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, kPSmem);
      if (e != cudaSuccess) return e;
      configured5 = true;
    }
    if (g_sm_count == 0) {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&g_sm_count, cudaDevAttrMultiProcessorCount, dev);
      if (g_sm_count <= 0) g_sm_count = 148;
    }
    int grid = g_sm_count * kPCtas;
    if (grid > m.ntiles) grid = m.ntiles;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = kPSmem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = use_pdl() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, csr_pipe_kernel<E>, m, x, ea);
  }
  if (variant >= 1) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)m.ntiles);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = variant == 2 ? kFlatTmaSmem : 0;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = use_pdl() ? 1 : 0;
    if (variant == 1) return cudaLaunchKernelEx(&cfg, csr_flat_kernel<E, false, 6>, m, x, ea, 0);
    if (variant == 3) return cudaLaunchKernelEx(&cfg, csr_flat_kernel<E, false, 4>, m, x, ea, 0);
    if (variant == 4) return cudaLaunchKernelEx(&cfg, csr_flat_kernel<E, false, 8>, m, x, ea, 0);
    if (variant == 10 || variant == 11 || variant == 12) {
      if (g_sm_count == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_sm_count, cudaDevAttrMultiProcessorCount, dev);
        if (g_sm_count <= 0) g_sm_count = 148;
      }
      const int dist = g_sm_count * 4 * (variant == 11 ? 2 : 1);
      if (variant == 12)
        return cudaLaunchKernelEx(&cfg, csr_flat_kernel<E, false, 4, true, true>, m, x, ea, dist);
      return cudaLaunchKernelEx(&cfg, csr_flat_kernel<E, false, 4, true>, m, x, ea, dist);
    }
    return cudaLaunchKernelEx(&cfg, csr_flat_kernel<E, true, 4>, m, x, ea, 0);
  }
  if (g_sm_count == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sm_count, cudaDevAttrMultiProcessorCount, dev);
    if (g_sm_count <= 0) g_sm_count = 148;
  }
  int grid = g_sm_count * kCtasPerSm;
  if (grid > m.ntiles) grid = m.ntiles;
  csr_stream_kernel<E><<<grid, kThreads, kSmemBytes, s>>>(m, x, ea);
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
    case Epi::kRestrictFirst: return launch_t<Epi::kRestrictFirst>(m, x, ea, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace smg
