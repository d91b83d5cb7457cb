// Batched local correction S_c (sm_100a, fp64).
//
// Reference: smoothers.py:203-211 (apply_local_correction) inside the sandwich
// smoother smoothers.py:252-267:  u += S_c (b - A u), where for every region
// d the correction is (L_d L_d^T)^{-1} r[B_d] with L_d the Cholesky factor of
// the principal submatrix A[B_d, B_d] (smoothers.py:176-200, LAPACK dpotrs
// via sparse.py:225-231).
//
// One CTA per region.  Each CTA
//   1. stages the packed lower factor L_d in shared memory when it fits
//      (larger factors are read through the same generic pointer from HBM);
//   2. forms the patch residual b - A u on its rows (the reference computes a
//      full-length residual and keeps only these rows -- identical values):
//      row bounds -> block scan -> all threads stream the rows' (val, col)
//      segments and form exact products in shared memory -> each row is then
//      summed sequentially in column order (bit-identical to scipy);
//   3. forward substitution with L, back substitution with L^T, 32-row panels:
//      off-panel updates are coalesced warp dot products; each panel's
//      triangle is applied as a 32-wide GEMV with its inverted diagonal block
//      (computed once at upload), so the serial chain is n/32 panel steps
//      instead of n dependent shuffle steps;
//   4. u[B_d] += x (or out[B_d] = x for apply_local_correction).
// Regions are DOF-disjoint but may be coupled through A: when
// the upload-time check finds coupling, the residuals of ALL regions are
// formed first by a residual-only launch (every region sees the
// pre-correction u), then the solve launch reads them from rbuf.
// Dense solves are tolerance-parity (~1e-15 relative vs the oracle), not
// bitwise: LAPACK's blocked order is not reproducible.
#include "smg_internal.cuh"

#include <cstdlib>

namespace smg {

// programmatic dependent launch (no-ops without the launch attribute): wait
// for the producer of u / b / rbuf, then let the next kernel's CTAs start
// their own static prologue on the SMs this kernel leaves idle.
__device__ __forceinline__ void patch_pdl_wait()
{
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ uint32_t psmem_u32(const void* p)
{
  return (uint32_t)__cvta_generic_to_shared(p);
}

// 1D bulk copy of a packed factor into shared memory (TMA, mbarrier completion)
__device__ __forceinline__ void factor_bulk_load(double* dst, const double* src, uint32_t bytes,
                                                 uint64_t* bar)
{
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(psmem_u32(bar)) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(psmem_u32(bar)),
               "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(psmem_u32(dst)),
      "l"(src), "r"(bytes), "r"(psmem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void factor_wait(uint64_t* bar)
{
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n"
      "@!p bra W_%=;\n}\n" ::"r"(psmem_u32(bar))
      : "memory");
}

__device__ __forceinline__ double warp_sum(double v)
{
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__host__ __device__ __forceinline__ int64_t tri(int64_t i) { return i * (i + 1) / 2; }

constexpr int kSolveThreads = 256;
constexpr int kSolveWarps = kSolveThreads / 32;
static_assert(kSolveWarps * 4 == 32, "panel_gemv splits a 32-wide panel over the warps");

// x[0:pn] <- D x (or D^T x) for one inverted 32x32 diagonal block D (row
// stride kDinvLd; zero-padded).  All threads: warp w forms the partial sums
// over columns [4w, 4w+4), then one thread per row adds the eight partials --
// dependency depth 4 + 8 instead of a 32-step chain in one warp.  Called with
// x ready (after a barrier); returns after a barrier.
__device__ __forceinline__ void panel_gemv(const double* D, double* x, int pn, bool transposed,
                                           double (*red)[32])
{
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  double acc = 0.0;
  if (lane < pn) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int j = warp * 4 + q;
      if (j < pn) acc += (transposed ? D[j * kDinvLd + lane] : D[lane * kDinvLd + j]) * x[j];
    }
  }
  red[warp][lane] = acc;
  __syncthreads();
  if (threadIdx.x < pn) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < kSolveWarps; ++w) t += red[w][threadIdx.x];
    x[threadIdx.x] = t;
  }
  __syncthreads();
}

// x[0:n] <- M x (or M^T x) for the whole inverse M = L^{-1} of a region
// (B = 64 or 128 rows, row stride B + 1, zero above the diagonal): warp w sums
// columns [w*B/8, (w+1)*B/8) for rows lane + 32q, then one thread per row adds
// the eight partials (red: 8 x B doubles).  Rows and columns >= n are never
// stored to / read from x.  Called with x ready; returns after a barrier.
template <int B>
__device__ __forceinline__ void gemv_inv(const double* M, double* x, int n, bool transposed,
                                         double* red)
{
  constexpr int kLd = B + 1, kCols = B / kSolveWarps, kRows = B / 32;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  double acc[kRows];
#pragma unroll
  for (int q = 0; q < kRows; ++q) acc[q] = 0.0;
#pragma unroll
  for (int c = 0; c < kCols; ++c) {
    const int j = warp * kCols + c;
    if (j < n) {
      const double xj = x[j];
#pragma unroll
      for (int q = 0; q < kRows; ++q) {
        const int i = lane + 32 * q;
        acc[q] += (transposed ? M[j * kLd + i] : M[i * kLd + j]) * xj;
      }
    }
  }
#pragma unroll
  for (int q = 0; q < kRows; ++q) red[warp * B + lane + 32 * q] = acc[q];
  __syncthreads();
  if (threadIdx.x < n) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < kSolveWarps; ++w) t += red[w * B + threadIdx.x];
    x[threadIdx.x] = t;
  }
  __syncthreads();
}

constexpr int kProdCap = 2048;                 // residual products staged per pass
constexpr int kProdItems = kProdCap / kSolveThreads;
constexpr int64_t kSmemBudget = 220 * 1024;    // dynamic smem per CTA (of 227 KB)

enum PatchMode : int { kAddResidualSolve = 0, kSolveFromBuf = 1, kResidualOnly = 2, kFollow = 3 };
constexpr int kFlagStream = 1;      // factors larger than shared memory stream through a ring
constexpr int kFlagL2Prefetch = 2;  // ... after an L2 prefetch of the whole factor
constexpr int kFlagSym = 4;         // the correction holds packed A[B,B]^{-1} for its larger regions
constexpr int kFlagSymPfShift = 12; // launch flags bits 12..16: L2 prefetch distance of the symmetric rings (rounds)
constexpr int kFlagSymNoFence = 1 << 18; // A/B: no fence.proxy.async before a ring refill (SMG_SYM_NOFENCE=1)
constexpr int kFlagSymReg = 1 << 19;     // register-resident column sums (sym_apply_reg; SMG_SYM_REG, default 1)
constexpr int kFlagSymFold = 1 << 17; // symmetric rings carry folded chunks: rows {c, n-1-c}, (n + 1) entries each

// Phase timestamps (SM clock) of the first 256 CTAs, compiled in only for the
// tools/trace_patch.py build (-DSMG_PATCH_TRACE); no cost otherwise.
#ifdef SMG_PATCH_TRACE
__device__ unsigned long long g_patch_trace[256][16];
#define PTRACE(k)                                                  \
  do {                                                             \
    if (threadIdx.x == 0 && blockIdx.x < 256)                      \
      g_patch_trace[blockIdx.x][k] = (unsigned long long)clock64(); \
  } while (0)
#define PTRACE_ACC(k, v)                                            \
  do {                                                              \
    if (threadIdx.x == 0 && blockIdx.x < 256) g_patch_trace[blockIdx.x][k] += (unsigned long long)(v); \
  } while (0)
#define PTRACE_CLK() clock64()
#else
#define PTRACE(k) \
  do {            \
  } while (0)
#define PTRACE_ACC(k, v) \
  do {                   \
  } while (0)
#define PTRACE_CLK() 0ll
#endif

static int patch_env(const char* name, int dflt)
{
  const char* v = getenv(name);
  return v ? atoi(v) : dflt;
}


static bool nostream_env()
{
  const char* v = getenv("SMG_PATCH_NOSTREAM");
  return v && v[0] == '1';
}

// shared-memory carve-up for a region of at most nmax dofs
struct PatchSmem {
  int64_t x_off, lo_off, off_off, prod_off, l_off, tri_cap, bytes;
  int64_t stage;   // > 0: streaming ring of `nst` stages of `stage` doubles at l_off
  int nst;
  int64_t y_off, z_off;   // symmetric-inverse path: column sums / row dots (double[n2] each)
  bool sym;               // ring carries packed A^{-1} rows (sym_apply), not factor rows
  int sym_rows;           // rows per chunk of the symmetric-inverse rings (1 or 2)
};

#ifndef SMG_CHUNK_ROWS
#define SMG_CHUNK_ROWS 8
#endif
constexpr int kChunkRows = SMG_CHUNK_ROWS;   // factor rows per streamed chunk (divides the 32-row panel)
static_assert(kPanel % kChunkRows == 0 && kChunkRows % 8 == 0, "chunk rows: 8, 16 or 32");
// chunks in flight per CTA; measured best on C5: 2 x 8 rows (227 us) beat
// 4 x 4 rows, a variable-size byte ring holding 2-4 longest chunks (282-475
// us) and an L2 prefetch window 2-6 chunks ahead (265 vs 247 us): the
// streamed solve is bound by its per-chunk arithmetic, not by copy latency
constexpr int kRingStages = 2;      // default depth (SMG_PATCH_STAGES overrides)
constexpr int kMaxRingStages = 8;
constexpr int kFlagStagesShift = 8; // launch flags bits 8..11: ring depth

// ring depth for streamed factors (SMG_PATCH_STAGES, default kRingStages)
static int stages_env()
{
  static int st = -1;
  if (st < 0) {
    const char* v = getenv("SMG_PATCH_STAGES");
    st = v ? atoi(v) : kRingStages;
    if (st < 2) st = 2;
    if (st > kMaxRingStages) st = kMaxRingStages;
  }
  return st;
}


// symmetric-inverse ring geometry: every warp has its own ring of nst (2..4)
// stages, a stage holds one chunk of sym_rows (2, or 1 for very large
// regions) rows: sym_rows (nmax + 2) doubles
constexpr int kSymMaxRows = 2;
constexpr int kSymWarps = 8;        // = kSolveWarps (defined below)
constexpr int kSymMaxStages = 6;

__host__ __device__ inline PatchSmem patch_smem_layout(int nmax, bool allow_stream = true,
                                                       int nst = kRingStages, bool sym = false,
                                                       int64_t sym_stage = 0, int sym_nst = 0)
{
  PatchSmem p;
  p.nst = nst < 2 ? 2 : (nst > kMaxRingStages ? kMaxRingStages : nst);
  const int64_t n2 = (nmax + 2) & ~int64_t(1);
  p.x_off = 0;                                   // double[n2]
  p.lo_off = p.x_off + 8 * n2;                   // int64[n2]
  p.off_off = p.lo_off + 8 * n2;                 // int32[n2 + 2]
  p.prod_off = p.off_off + ((4 * (n2 + 2) + 15) & ~int64_t(15));  // double[kProdCap]
  // the product buffer doubles as the streamed path's inverted-block double buffer
  p.l_off = p.prod_off + 8 * (kProdCap > 2 * kDinvBlock ? kProdCap : 2 * kDinvBlock);
  p.y_off = p.z_off = 0;
  p.sym = sym && nmax > 4 * kPanel;
  p.stage = 0;
  p.sym_rows = 0;
  if (p.sym) {
    // regions of more than 128 dofs (and 65..128 beside them) stream the packed
    // lower triangle of their inverse through per-warp rings; smaller ones are
    // staged whole in the same area.  y: one column-sum vector per warp.
    p.y_off = p.l_off;
    p.z_off = p.y_off + 8 * n2 * kSymWarps;
    p.l_off = p.z_off + 8 * n2;
    p.nst = sym_nst < 2 ? 2 : (sym_nst > kSymMaxStages ? kSymMaxStages : sym_nst);
    p.sym_rows = kSymMaxRows;
    if (sym_stage != 0) {
      // folded chunks (rows c and n-1-c, two 16-byte aligned copies): n + 1
      // entries plus alignment slack, whatever c
      p.sym_rows = 0;
      p.stage = ((int64_t)nmax + 6) & ~int64_t(1);
      while (p.nst > 2 && p.l_off + 8 * kSymWarps * p.nst * p.stage > kSmemBudget) --p.nst;
    } else {
      for (;;) {
        p.stage = ((int64_t)p.sym_rows * (nmax + 2) + 1) & ~int64_t(1);
        if (p.l_off + 8 * kSymWarps * p.nst * p.stage <= kSmemBudget) break;
        if (p.nst > 2) --p.nst;
        else if (p.sym_rows > 1) --p.sym_rows;
        else break;
      }
    }
    const int64_t need = patch_slot_max(nmax, true);
    const int64_t ring = (int64_t)kSymWarps * p.nst * p.stage;
    p.tri_cap = ring > need ? ring : need;
    p.bytes = p.l_off + 8 * p.tri_cap;
    return p;
  }
  int64_t cap = (kSmemBudget - p.l_off) / 8;
  if (cap < 0) cap = 0;
  cap &= ~int64_t(1);
  const int64_t need = patch_slot_max(nmax, false);
  if (need <= cap || !allow_stream) {  // every region's slot (factor + inverted blocks) fits: stage it whole
    p.tri_cap = need;
    p.bytes = p.l_off + 8 * need;
  } else {            // stream factor rows through a ring (smaller regions still staged)
    p.stage = ((int64_t)kChunkRows * (nmax + 2) + 1) & ~int64_t(1);
    // deeper rings only while they fit the budget
    while (p.nst > 2 && p.l_off + 8 * p.nst * p.stage > kSmemBudget) --p.nst;
    p.tri_cap = p.nst * p.stage;
    p.bytes = p.l_off + 8 * p.tri_cap;
  }
  return p;
}

// ---------------------------------------------------------------------------
// Streaming triangular solves for regions whose factor does not fit in shared
// memory (C5: 64..512-dof patches).  Row chunks of kChunkRows factor rows --
// contiguous in the packed row-major layout -- flow HBM -> smem through a
// kRingStages-deep bulk-copy ring.  Forward: left-looking (chunk rows against the
// solved prefix), then the panel's inverted diagonal block.  Backward:
// right-looking from the last panel (inverted block first, then the panel's
// rows update the unsolved prefix), so both passes stream the same row chunks.
__device__ __forceinline__ int n_chunks(int n)
{
  const int nb = (n + kPanel - 1) / kPanel;
  const int pn_last = n - (nb - 1) * kPanel;
  return (nb - 1) * (kPanel / kChunkRows) + (pn_last + kChunkRows - 1) / kChunkRows;
}

// Chunk sequence without divisions: forward panels 0..nb-1, then backward
// panels nb-1..0, chunks ascending inside each panel; advanced one chunk at a time by the consumer and the issuer.
struct ChunkCursor {
  int panel, j, nb, k_last, n;
  bool fwd;
  __device__ __forceinline__ void init(int n_)
  {
    n = n_;
    nb = (n + kPanel - 1) / kPanel;
    k_last = (n - (nb - 1) * kPanel + kChunkRows - 1) / kChunkRows;
    panel = 0;
    j = 0;
    fwd = true;
  }
  __device__ __forceinline__ int chunks_in_panel() const
  {
    return panel == nb - 1 ? k_last : kPanel / kChunkRows;
  }
  __device__ __forceinline__ int i0() const { return panel * kPanel + j * kChunkRows; }
  __device__ __forceinline__ int rows() const { return min(kChunkRows, n - i0()); }
  __device__ __forceinline__ void advance()
  {
    if (++j < chunks_in_panel()) return;
    j = 0;
    if (fwd) {
      if (++panel == nb) {
        fwd = false;
        panel = nb - 1;
      }
    } else {
      --panel;
    }
  }
};

// chunk seq -> ring stage seq % kRingStages (one mbarrier per stage)
__device__ __forceinline__ void ring_issue_at(const double* Lg, double* ring, int64_t stage,
                                              int i0, int rows, int s, uint64_t* bars)
{
  const int64_t a = tri(i0) & ~int64_t(1);
  const int64_t b = (tri(i0 + rows) + 1) & ~int64_t(1);
  SMG_DCHECK(s >= 0 && s < kMaxRingStages && rows > 0 && b - a <= stage);
  uint64_t* bar = &bars[s];
  const uint32_t bytes = (uint32_t)((b - a) * 8);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(psmem_u32(bar)),
               "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(psmem_u32(ring + s * stage)),
      "l"(Lg + a), "r"(bytes), "r"(psmem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void ring_wait(uint64_t* bar, uint32_t parity)
{
  asm volatile(
      "{\n.reg .pred p;\nRW_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra RW_%=;\n}\n" ::"r"(psmem_u32(bar)),
      "r"(parity)
      : "memory");
}

// Inverted diagonal blocks are consumed in a fixed order -- forward panels
// 0..nb-1, then backward panels nb-1..0 -- and prefetched two uses ahead into
// a double buffer by bulk copy (each block is 1056 contiguous doubles).
__device__ __forceinline__ int dinv_panel(int q, int nb) { return q < nb ? q : 2 * nb - 1 - q; }

__device__ __forceinline__ void dinv_issue(const double* Dinv, double* s_dinv, int q, int nb,
                                           uint64_t* dbars)
{
  const int slot = q & 1;
  uint64_t* bar = &dbars[slot];
  const uint32_t bytes = kDinvBlock * 8;
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(psmem_u32(bar)),
               "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(psmem_u32(s_dinv + slot * kDinvBlock)),
      "l"(Dinv + (int64_t)dinv_panel(q, nb) * kDinvBlock), "r"(bytes), "r"(psmem_u32(bar))
      : "memory");
}

__device__ void stream_solve(const double* __restrict__ Lg, double* ring, int64_t stage, int nst,
                             int n, double* s_x, double* s_dinv, uint64_t* bars, uint64_t* dbars,
                             double (*red)[32])
{
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const double* Dinv = Lg + patch_tri_even(n);
  const int nb = (n + kPanel - 1) / kPanel;
  const int C = n_chunks(n);
  const int total = 2 * C;
  int dq = 0;  // next inverted block to consume
  // issue cursor (thread 0 only): the chunk that goes into the ring next
  ChunkCursor iss;
  iss.init(n);
  int iss_seq = 0, iss_stage = 0;
  if (threadIdx.x == 0) {
    for (int q = 0; q < nst; ++q)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(psmem_u32(&bars[q])) : "memory");
    for (int q = 0; q < 2; ++q)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(psmem_u32(&dbars[q])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (; iss_seq < nst && iss_seq < total; ++iss_seq) {
      ring_issue_at(Lg, ring, stage, iss.i0(), iss.rows(), iss_stage, bars);
      iss.advance();
      if (++iss_stage == nst) iss_stage = 0;
    }
    for (int q = 0; q < 2 && q < 2 * nb; ++q) dinv_issue(Dinv, s_dinv, q, nb, dbars);
  }
  __syncthreads();
  // consume block dq: wait, x_P = inv(L_PP) r_P (forward) or inv(L_PP)^T y_P (backward)
  auto panel_solve = [&](int p0, int pn, bool transposed) {
    ring_wait(&dbars[dq & 1], (uint32_t)((dq >> 1) & 1));
    panel_gemv(s_dinv + (dq & 1) * kDinvBlock, s_x + p0, pn, transposed, red);
    if (threadIdx.x == 0 && dq + 2 < 2 * nb) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      dinv_issue(Dinv, s_dinv, dq + 2, nb, dbars);
    }
    ++dq;
  };
  ChunkCursor cur;
  cur.init(n);
  int stg = 0;
  uint32_t phase = 0;
  for (int seq = 0; seq < total; ++seq) {
    const int i0 = cur.i0(), crows = cur.rows();
    const int p0 = cur.panel * kPanel;
    const int pn = min(kPanel, n - p0);
    const bool fwd = cur.fwd;
    if (seq == C) PTRACE(4);
    if (!fwd && i0 == p0) panel_solve(p0, pn, true);   // backward: own block first
    ring_wait(&bars[stg], phase);
    const double* rows = ring + stg * stage + (tri(i0) & 1) - tri(i0);
    SMG_DCHECK(i0 >= p0 && crows > 0 && i0 + crows <= n && stg < nst);
    if (fwd) {
      // x_i -= L[i, 0:p0] . x[0:p0] for the chunk's rows (warp w: rows w, w + 8, ...)
      if (p0 > 0) {
#pragma unroll
        for (int rr = 0; rr < kChunkRows / 8; ++rr) {
          const int r = warp + 8 * rr;
          if (r < crows) {
            const int i = i0 + r;
            const double* Li = rows + tri(i);
            // four independent partial sums: the loads of the next products do
            // not wait on the previous multiply-add
            double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
            int j = lane;
            for (; j + 96 < p0; j += 128) {
              a0 += Li[j] * s_x[j];
              a1 += Li[j + 32] * s_x[j + 32];
              a2 += Li[j + 64] * s_x[j + 64];
              a3 += Li[j + 96] * s_x[j + 96];
            }
            for (; j < p0; j += 32) a0 += Li[j] * s_x[j];
            const double acc = warp_sum((a0 + a1) + (a2 + a3));
            if (lane == 0) s_x[i] -= acc;
          }
        }
      }
    } else if (p0 > 0) {
      // y[c] -= sum_{i in chunk} L[i][c] x_i  for c < p0 (thread per column)
      for (int col = threadIdx.x; col < p0; col += kSolveThreads) {
        double a0 = 0.0, a1 = 0.0;
        const double* rc = rows + tri(i0) + col;   // row i0 + r starts tri(i0 + r)
        int r = 0;
        for (; r + 1 < crows; r += 2) {
          a0 += rc[0] * s_x[i0 + r];
          rc += i0 + r + 1;
          a1 += rc[0] * s_x[i0 + r + 1];
          rc += i0 + r + 2;
        }
        if (r < crows) a0 += rc[0] * s_x[i0 + r];
        s_x[col] -= a0 + a1;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0 && iss_seq < total) {  // stage free: next chunk into it
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      ring_issue_at(Lg, ring, stage, iss.i0(), iss.rows(), iss_stage, bars);
      iss.advance();
      ++iss_seq;
      if (++iss_stage == nst) iss_stage = 0;
    }
    if (fwd && i0 + crows == p0 + pn) panel_solve(p0, pn, false);  // forward: panel done
    cur.advance();
    if (++stg == nst) {
      stg = 0;
      phase ^= 1u;
    }
  }
}

// ---------------------------------------------------------------------------
// Symmetric-inverse correction: x = A[B,B]^{-1} r from the packed lower
// triangle M of the inverse (row-major, row i = M[i][0..i]), read from HBM
// once.  The rows are cut into chunks of R (2, or 1) consecutive rows --
// contiguous in the packed layout -- and chunk c belongs to warp c mod 8
// alone: every warp runs its own bulk-copy ring (its lane 0 requests, the
// warp waits on its own mbarriers), so the stream loop has no CTA barrier and
// no exchange between warps.  For a chunk with rows [i0, i0 + R) the warp
// walks the 32-column blocks, lane l on column j = c0 + l:
//   row part     a_k += M[i0+k][j] r_j   (j <= i), summed over the blocks, then
//                one butterfly per chunk leaves z_{i0+k} on a lane;
//   column part  y_w[j] += sum_k M[i0+k][j] r_{i0+k}   (j < i), the warp's own
//                column-sum vector in shared memory.
// At the end x = z + sum_w y_w (warp order).  Nothing in a chunk depends on
// another chunk's result.  Fixed order everywhere: deterministic, independent
// of the ring depth.
// Measured alternatives (profiles/r02/SUMMARY.md): chunks shared by all eight
// warps (column blocks split over the warps, per-warp partial row sums
// combined after a CTA barrier per chunk: 119-125 us on C5 against 75 here --
// the per-chunk fixed costs, ~240 instructions per warp, were three times the
// arithmetic); variable-size byte chunks with a warp per row and a thread per
// column (203 us); 4-row chunks with full / empty mbarriers and a rotating
// closing warp (175 us).

// 32-bit triangle numbers (regions are far below 65k dofs)
__device__ __forceinline__ int tri32(int i) { return (i * (i + 1)) >> 1; }

// lane 0 of a warp: request chunk c (rows [c R, c R + R)) into `dst`
__device__ __forceinline__ void sym_issue(const double* Mg, double* dst, int R, int n, int c,
                                          uint64_t* bar)
{
  const int i0 = c * R;
  const int i1 = min(i0 + R, n);
  const int a = tri32(i0) & ~1;
  const int b = (tri32(i1) + 1) & ~1;
  const uint32_t bytes = (uint32_t)(b - a) * 8u;
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(psmem_u32(bar)),
               "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(psmem_u32(dst)),
      "l"(Mg + a), "r"(bytes), "r"(psmem_u32(bar))
      : "memory");
}

// lane 0 of a warp: pull chunk c towards L2 (fire and forget: no shared
// memory, so the bytes in flight are not limited by the ring)
__device__ __forceinline__ void sym_prefetch(const double* Mg, int R, int n, int c)
{
  const int i0 = c * R;
  const int i1 = min(i0 + R, n);
  const int a = tri32(i0) & ~1;
  const int b = (tri32(i1) + 1) & ~1;
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(Mg + a),
               "r"((uint32_t)(b - a) * 8u)
               : "memory");
}

// folded chunks (R == 0): chunk c = rows {c, n - 1 - c} -- n + 1 entries for
// every c, so each ring stage carries the same bytes and the bytes in flight
// per CTA are the ring's capacity (with consecutive row pairs the first
// chunks are a few hundred bytes and the ring is half empty on average).
// Two copies per chunk (the rows are not adjacent in the packed layout), one
// mbarrier.
__device__ __forceinline__ void sym_issue_fold(const double* Mg, double* dst, int n, int c,
                                               uint64_t* bar)
{
  const int ia = c, ib = n - 1 - c;
  const int a0 = tri32(ia) & ~1, a1 = (tri32(ia + 1) + 1) & ~1;
  const int b0 = tri32(ib) & ~1, b1 = (tri32(ib + 1) + 1) & ~1;
  const bool two = ib > ia;
  const uint32_t bytes_a = (uint32_t)(a1 - a0) * 8u;
  const uint32_t bytes_b = two ? (uint32_t)(b1 - b0) * 8u : 0u;
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(psmem_u32(bar)),
               "r"(bytes_a + bytes_b)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(psmem_u32(dst)),
      "l"(Mg + a0), "r"(bytes_a), "r"(psmem_u32(bar))
      : "memory");
  if (two)
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(psmem_u32(dst + (a1 - a0))),
        "l"(Mg + b0), "r"(bytes_b), "r"(psmem_u32(bar))
        : "memory");
}

// thread 0, at kernel entry: the warps' ring barriers (kSymWarps x nst)
__device__ __forceinline__ void sym_ring_init(int nst, uint64_t* bars)
{
  for (int q = 0; q < kSymWarps * nst; ++q)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(psmem_u32(&bars[q])) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// every warp's lane 0, after the barrier that publishes the initialised
// mbarriers (the inverse is static data: before the dependency wait,
// overlapping the residual): the warp's first nst chunks
__device__ __forceinline__ void sym_ring_start(const double* Mg, double* ring, int S, int nst, int R,
                                               int n, uint64_t* bars, int pf)
{
  const int warp = threadIdx.x >> 5;
  if (R == 0) {   // folded chunks
    const int nch = (n + 1) >> 1;
    for (int q = 0; q < nst; ++q) {
      const int c = warp + q * kSymWarps;
      if (c < nch) sym_issue_fold(Mg, ring + (warp * nst + q) * S, n, c, &bars[warp * nst + q]);
    }
    return;
  }
  const int nchunks = (n + R - 1) / R;
  for (int q = 0; q < nst; ++q) {
    const int c = warp + q * kSymWarps;
    if (c < nchunks)
      sym_issue(Mg, ring + (warp * nst + q) * S, R, n, c, &bars[warp * nst + q]);
  }
  // the next pf rounds of this warp's chunks go towards L2 meanwhile
  for (int q = nst; q < nst + pf; ++q) {
    const int c = warp + q * kSymWarps;
    if (c < nchunks) sym_prefetch(Mg, R, n, c);
  }
}

// Folded-chunk version of sym_apply (below): chunk c = rows ia = c and
// ib = n - 1 - c.  Blocks left of ia's diagonal take both rows, the block on
// ia's diagonal is predicated, the blocks between the two diagonals take row
// ib alone.  Same row / column parts, same final combine.
__device__ void sym_apply_fold(const double* __restrict__ Mg, double* ring, int S, int nst, int n,
                               int n2, double* s_x, double* s_y, double* s_z, uint64_t* bars)
{
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  double* __restrict__ yw = s_y + warp * n2;
  const double* __restrict__ xr = s_x;
  for (int j = lane; j < n; j += 32) yw[j] = 0.0;
  __syncwarp();
  const int nch = (n + 1) >> 1;
  double* ringw = ring + warp * nst * S;
  uint64_t* barw = bars + warp * nst;
  int stg = 0;
  uint32_t phase = 0;
  for (int c = warp; c < nch; c += kSymWarps) {
    const int ia = c, ib = n - 1 - c;
    const bool two = ib > ia;
    ring_wait(&barw[stg], phase);
    const double* base = ringw + stg * S;
    const int ta = tri32(ia);
    const int len_a = ((tri32(ia + 1) + 1) & ~1) - (ta & ~1);
    const int tb = tri32(ib);
    const double* __restrict__ rowa = base - (ta & ~1) + ta;            // M[ia][j] = rowa[j]
    const double* __restrict__ rowb = base + len_a - (tb & ~1) + tb;    // M[ib][j] = rowb[j]
    const double ra = xr[ia];
    const double rb = two ? xr[ib] : 0.0;
    double aa = 0.0, ab = 0.0;
    int c0 = 0;
    // both rows, blocks strictly left of ia's diagonal
    for (; c0 + 127 < ia; c0 += 128) {
      const int j = c0 + lane;
      double m0[4], m1[4], xv[4], yv[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        m0[q] = rowa[j + 32 * q];
        m1[q] = two ? rowb[j + 32 * q] : 0.0;   // (the middle row of an odd region is alone)
        xv[q] = xr[j + 32 * q];
        yv[q] = yw[j + 32 * q];
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        aa += m0[q] * xv[q];
        ab += m1[q] * xv[q];
        yv[q] = (yv[q] + m0[q] * ra) + m1[q] * rb;
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) yw[j + 32 * q] = yv[q];
    }
    for (; c0 + 31 < ia; c0 += 32) {
      const int j = c0 + lane;
      const double m00 = rowa[j];
      const double m10 = two ? rowb[j] : 0.0;
      const double x0 = xr[j];
      aa += m00 * x0;
      ab += m10 * x0;
      yw[j] = (yw[j] + m00 * ra) + m10 * rb;
    }
    // the block on ia's diagonal (c0 <= ia < c0 + 32)
    {
      const int j = c0 + lane;
      const double m00 = j <= ia ? rowa[j] : 0.0;
      const double m10 = (two && j <= ib) ? rowb[j] : 0.0;
      const double x0 = j < n ? xr[j] : 0.0;
      aa += m00 * x0;
      ab += m10 * x0;
      if (j < ib) {   // j < ia implies j < ib
        double y = yw[j];
        if (j < ia) y += m00 * ra;
        if (two) y += m10 * rb;
        yw[j] = y;
      }
      c0 += 32;
    }
    // row ib alone, up to its diagonal
    if (two) {
      for (; c0 + 127 < ib; c0 += 128) {
        const int j = c0 + lane;
        double m1[4], xv[4], yv[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          m1[q] = rowb[j + 32 * q];
          xv[q] = xr[j + 32 * q];
          yv[q] = yw[j + 32 * q];
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          ab += m1[q] * xv[q];
          yv[q] += m1[q] * rb;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) yw[j + 32 * q] = yv[q];
      }
      for (; c0 + 31 < ib; c0 += 32) {
        const int j = c0 + lane;
        const double m10 = rowb[j];
        ab += m10 * xr[j];
        yw[j] += m10 * rb;
      }
      for (; c0 <= ib; c0 += 32) {
        const int j = c0 + lane;
        const double m10 = j <= ib ? rowb[j] : 0.0;
        const double x0 = j < n ? xr[j] : 0.0;
        ab += m10 * x0;
        if (j < ib) yw[j] += m10 * rb;
      }
    }
    // 2-value butterfly: lane 0 ends with z_ia, lane 16 with z_ib
    {
      const bool up = (lane & 16) != 0;
      const double send = up ? aa : ab;
      const double keep = up ? ab : aa;
      double v = keep + __shfl_xor_sync(0xffffffffu, send, 16);
      v += __shfl_xor_sync(0xffffffffu, v, 8);
      v += __shfl_xor_sync(0xffffffffu, v, 4);
      v += __shfl_xor_sync(0xffffffffu, v, 2);
      v += __shfl_xor_sync(0xffffffffu, v, 1);
      if (lane == 0) s_z[ia] = v;
      if (lane == 16 && two) s_z[ib] = v;
    }
    __syncwarp();
    if (lane == 0 && c + nst * kSymWarps < nch) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      sym_issue_fold(Mg, ringw + stg * S, n, c + nst * kSymWarps, &barw[stg]);
    }
    if (++stg == nst) {
      stg = 0;
      phase ^= 1u;
    }
  }
  __syncthreads();   // every warp's z rows and column sums
  for (int j = threadIdx.x; j < n; j += kSolveThreads) {
    double y = s_y[j];
#pragma unroll
    for (int w = 1; w < kSymWarps; ++w) y += s_y[w * n2 + j];
    s_x[j] = s_z[j] + y;
  }
  __syncthreads();
}

// Register-resident version of sym_apply (below) for regions of at most
// 32 NB dofs, consecutive row pairs (R = 2); used for regions of <= 256 dofs
// (NB = 8: 192 x1000 61.5 -> 56.7 us, 256 x1000 81.3 -> 74.2 us).  The phase trace of sym_apply
// (profiles/r02/SUMMARY.md, session 5: per chunk 850 cycles in the blocks,
// 430 in the butterfly, 300 in the refill, 95 waiting for the ring) showed
// the warps bound by their own instruction latencies, not by the copies:
//   * lane l owns columns l, l + 32, ...: its r_j and its column sums y_j
//     stay in registers (NB of each), so a block left of the diagonal costs
//     two shared-memory loads (the two matrix rows) instead of four loads
//     and a store; four blocks are loaded ahead of their arithmetic;
//   * the block(s) on the diagonal keep the predicated shared-memory path
//     (the warp's own column-sum vector yw), added to the registers' sums in
//     the final combine;
//   * the row sums of four consecutive chunks of the warp (eight values) are
//     reduced by ONE transposed butterfly (nine shuffles, depth five) instead
//     of four 2-value butterflies.
// Fixed order everywhere: deterministic, independent of the ring depth.
template <int NB>
__device__ void sym_apply_reg(const double* __restrict__ Mg, double* ring, int S, int nst, int n,
                              int n2, double* s_x, double* s_y, double* s_z, uint64_t* bars,
                              bool fence)
{
  constexpr int R = 2;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  double* __restrict__ yw = s_y + warp * n2;
  double xr[NB], y[NB];
#pragma unroll
  for (int k = 0; k < NB; ++k) {
    const int j = 32 * k + lane;
    xr[k] = j < n ? s_x[j] : 0.0;
    y[k] = 0.0;
  }
  for (int j = lane; j < n; j += 32) yw[j] = 0.0;
  __syncwarp();
  const int nchunks = (n + R - 1) / R;
  double* ringw = ring + warp * nst * S;
  uint64_t* barw = bars + warp * nst;
  int stg = 0;
  uint32_t phase = 0;
  double acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = 0.0;
  int q = 0;            // chunks in the current group of four
  int cg = warp;        // first chunk of the group
  for (int c = warp; c < nchunks; c += kSymWarps) {
    const int i0 = c * R;
    const bool two = i0 + 1 < n;
    ring_wait(&barw[stg], phase);
    const int t0 = tri32(i0);
    const double* __restrict__ row0 = ringw + stg * S - (t0 & ~1) + t0;   // M[i0][j] = row0[j]
    const double* __restrict__ row1 = row0 + i0 + 1;                      // M[i0 + 1][j] = row1[j]
    const double r0 = s_x[i0];
    const double r1 = two ? s_x[i0 + 1] : 0.0;
    double a0 = 0.0, a1 = 0.0;
    const int kd = i0 >> 5;   // blocks k < kd lie strictly left of the diagonal
#pragma unroll
    for (int kk = 0; kk < NB; kk += 4) {
      if (kk + 3 < kd) {
        double m0[4], m1[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          m0[t] = row0[32 * (kk + t) + lane];
          m1[t] = two ? row1[32 * (kk + t) + lane] : 0.0;
        }
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          a0 += m0[t] * xr[kk + t];
          a1 += m1[t] * xr[kk + t];
          y[kk + t] = (y[kk + t] + m0[t] * r0) + m1[t] * r1;
        }
      } else if (kk < kd) {
#pragma unroll
        for (int t = 0; t < 3; ++t) {
          if (kk + t < kd) {
            const double m00 = row0[32 * (kk + t) + lane];
            const double m10 = two ? row1[32 * (kk + t) + lane] : 0.0;
            a0 += m00 * xr[kk + t];
            a1 += m10 * xr[kk + t];
            y[kk + t] = (y[kk + t] + m00 * r0) + m10 * r1;
          }
        }
      }
    }
    // blocks crossing the diagonal: row part j <= i, column part j < i
    const int last = two ? i0 + 1 : i0;
    for (int c0 = kd << 5; c0 <= last; c0 += 32) {
      const int j = c0 + lane;
      const double m00 = j <= i0 ? row0[j] : 0.0;
      const double m10 = (two && j <= i0 + 1) ? row1[j] : 0.0;
      const double x0 = j < n ? s_x[j] : 0.0;
      a0 += m00 * x0;
      a1 += m10 * x0;
      if (j < last) {
        double yy = yw[j];
        if (j < i0) yy += m00 * r0;
        if (two) yy += m10 * r1;   // j < i0 + 1 = last
        yw[j] = yy;
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (q == i) {
        acc[2 * i] = a0;
        acc[2 * i + 1] = a1;
      }
    // the stage is free once every lane has read it: refill with this warp's
    // chunk nst rounds ahead
    __syncwarp();
    if (lane == 0 && c + nst * kSymWarps < nchunks) {
      if (fence) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      sym_issue(Mg, ringw + stg * S, R, n, c + nst * kSymWarps, &barw[stg]);
    }
    if (++stg == nst) {
      stg = 0;
      phase ^= 1u;
    }
    ++q;
    if (q == 4 || c + kSymWarps >= nchunks) {
      // transposed butterfly: value i (row 2 (cg + 8 (i / 2)) + (i & 1)) ends on lane 4 i
      double w4[4], w2[2];
      {
        const bool up = (lane & 16) != 0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const double send = up ? acc[i] : acc[4 + i];
          const double keep = up ? acc[4 + i] : acc[i];
          w4[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
        }
      }
      {
        const bool up = (lane & 8) != 0;
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const double send = up ? w4[i] : w4[2 + i];
          const double keep = up ? w4[2 + i] : w4[i];
          w2[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
        }
      }
      double v;
      {
        const bool up = (lane & 4) != 0;
        const double send = up ? w2[0] : w2[1];
        const double keep = up ? w2[1] : w2[0];
        v = keep + __shfl_xor_sync(0xffffffffu, send, 4);
      }
      v += __shfl_xor_sync(0xffffffffu, v, 2);
      v += __shfl_xor_sync(0xffffffffu, v, 1);
      if ((lane & 3) == 0) {
        const int i = lane >> 2;                       // value index 0..7
        const int row = R * (cg + kSymWarps * (i >> 1)) + (i & 1);
        if ((i >> 1) < q && row < n) s_z[row] = v;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] = 0.0;
      q = 0;
      cg = c + kSymWarps;
    }
  }
  // the registers' column sums join the diagonal blocks' in the warp's vector
#pragma unroll
  for (int k = 0; k < NB; ++k) {
    const int j = 32 * k + lane;
    if (j < n) yw[j] += y[k];
  }
  __syncthreads();   // every warp's z rows and column sums
  for (int j = threadIdx.x; j < n; j += kSolveThreads) {
    double yy = s_y[j];
#pragma unroll
    for (int w = 1; w < kSymWarps; ++w) yy += s_y[w * n2 + j];
    s_x[j] = s_z[j] + yy;
  }
  __syncthreads();
}

// s_x holds r on entry (visible to all threads) and x on return (after a
// barrier).  s_y: kSymWarps vectors of n2 doubles.
__device__ void sym_apply(const double* __restrict__ Mg, double* ring, int S, int nst, int R, int n,
                          int n2, double* s_x, double* s_y, double* s_z, uint64_t* bars, int pf,
                          bool fence)
{
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  double* __restrict__ yw = s_y + warp * n2;
  const double* __restrict__ xr = s_x;   // r: read-only until the final combine
  for (int j = lane; j < n; j += 32) yw[j] = 0.0;
  __syncwarp();
  const int nchunks = (n + R - 1) / R;
  double* ringw = ring + warp * nst * S;
  uint64_t* barw = bars + warp * nst;
  int stg = 0;
  uint32_t phase = 0;
  for (int c = warp; c < nchunks; c += kSymWarps) {
    const int i0 = c * R;
    const bool two = R == 2 && i0 + 1 < n;      // the chunk has a second row
    const long long tr0 = PTRACE_CLK();
    ring_wait(&barw[stg], phase);
    const long long tr1 = PTRACE_CLK();
    PTRACE_ACC(9, tr1 - tr0);
    const int t0 = tri32(i0);
    const double* __restrict__ row0 = ringw + stg * S - (t0 & ~1) + t0;   // M[i0][j] = row0[j]
    const double* __restrict__ row1 = row0 + i0 + 1;                      // M[i0 + 1][j] = row1[j]
    const double r0 = xr[i0];
    const double r1 = two ? xr[i0 + 1] : 0.0;
    double a0 = 0.0, a1 = 0.0;
    // blocks strictly left of the diagonal: no predicates; four per pass with
    // all sixteen loads ahead of the arithmetic (two warps per scheduler: the
    // shared-memory latency has to be covered inside the warp)
    int c0 = 0;
    for (; c0 + 127 < i0; c0 += 128) {
      const int j = c0 + lane;
      double m0[4], m1[4], xv[4], yv[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        m0[q] = row0[j + 32 * q];
        m1[q] = two ? row1[j + 32 * q] : 0.0;
        xv[q] = xr[j + 32 * q];
        yv[q] = yw[j + 32 * q];
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        a0 += m0[q] * xv[q];
        a1 += m1[q] * xv[q];
        yv[q] = (yv[q] + m0[q] * r0) + m1[q] * r1;
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) yw[j + 32 * q] = yv[q];
    }
    for (; c0 + 31 < i0; c0 += 32) {
      const int j = c0 + lane;
      const double m00 = row0[j];
      const double m10 = two ? row1[j] : 0.0;
      const double x0 = xr[j];
      a0 += m00 * x0;
      a1 += m10 * x0;
      yw[j] = (yw[j] + m00 * r0) + m10 * r1;
    }
    // blocks crossing the diagonal: row part j <= i, column part j < i
    const int last = two ? i0 + 1 : i0;
    for (; c0 <= last; c0 += 32) {
      const int j = c0 + lane;
      const double m00 = j <= i0 ? row0[j] : 0.0;
      const double m10 = (two && j <= i0 + 1) ? row1[j] : 0.0;
      const double x0 = j < n ? xr[j] : 0.0;
      a0 += m00 * x0;
      a1 += m10 * x0;
      if (j < last) {
        double y = yw[j];
        if (j < i0) y += m00 * r0;
        if (two) y += m10 * r1;   // j < i0 + 1 = last
        yw[j] = y;
      }
    }
    const long long tr2 = PTRACE_CLK();
    PTRACE_ACC(10, tr2 - tr1);
    // 2-value butterfly: lane 0 ends with z_{i0}, lane 16 with z_{i0+1}
    {
      const bool up = (lane & 16) != 0;
      const double send = up ? a0 : a1;
      const double keep = up ? a1 : a0;
      double v = keep + __shfl_xor_sync(0xffffffffu, send, 16);
      v += __shfl_xor_sync(0xffffffffu, v, 8);
      v += __shfl_xor_sync(0xffffffffu, v, 4);
      v += __shfl_xor_sync(0xffffffffu, v, 2);
      v += __shfl_xor_sync(0xffffffffu, v, 1);
      if (lane == 0) s_z[i0] = v;
      if (lane == 16 && two) s_z[i0 + 1] = v;
    }
    // the stage is free once every lane has read it: refill with this warp's
    // chunk nst rounds ahead
    const long long tr3 = PTRACE_CLK();
    PTRACE_ACC(11, tr3 - tr2);
    __syncwarp();
    if (lane == 0 && c + nst * kSymWarps < nchunks) {
      if (fence) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      sym_issue(Mg, ringw + stg * S, R, n, c + nst * kSymWarps, &barw[stg]);
      if (pf > 0 && c + (nst + pf) * kSymWarps < nchunks)
        sym_prefetch(Mg, R, n, c + (nst + pf) * kSymWarps);
    }
    PTRACE_ACC(13, PTRACE_CLK() - tr3);
    PTRACE_ACC(14, 1);
    if (++stg == nst) {
      stg = 0;
      phase ^= 1u;
    }
  }
  __syncthreads();   // every warp's z rows and column sums
  for (int j = threadIdx.x; j < n; j += kSolveThreads) {
    double y = s_y[j];
#pragma unroll
    for (int w = 1; w < kSymWarps; ++w) y += s_y[w * n2 + j];
    s_x[j] = s_z[j] + y;
  }
  __syncthreads();
}

__host__ __device__ __forceinline__ int nmax_ring(const FollowArgs& fa) { return fa.ring_max; }

// kSym: the correction has symmetric-inverse regions (more than 128 dofs):
// its own instantiation (128 registers, two CTAs per SM), so corrections of
// small regions keep the lean kernel (C1-C3: 64 registers)
template <int kMode, bool kSym>
__global__ void __launch_bounds__(kSolveThreads, kSym ? 2 : 0)
patch_kernel(const int64_t* __restrict__ prow, const int32_t* __restrict__ pcol,
             const double* __restrict__ pval, const int32_t* __restrict__ pptr,
             const int32_t* __restrict__ dofs,
             const int64_t* __restrict__ foff, const double* __restrict__ lfac,
             const double* __restrict__ b, const double* u_res, double* rbuf, double* target,
             int scatter_add, int nmax, int flags, const int32_t* __restrict__ order,
             const FollowArgs fa, const int32_t* __restrict__ ring_ptr,
             const int32_t* __restrict__ ring_rows, const int32_t* __restrict__ plcol,
             const int32_t* __restrict__ bpos)
{
  const bool allow_stream = (flags & kFlagStream) != 0;
  PTRACE(0);
  // follow mode: the next kernel may start its static prologue at once; its
  // dependency wait still covers the producer, because this grid completes
  // only after waiting for the producer (end of the kernel)
  if (kMode == kFollow) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  extern __shared__ __align__(16) unsigned char psm[];
  __shared__ double s_red[kSolveWarps][32];
  __shared__ uint64_t s_bar;
  __shared__ uint64_t s_ring_bar[kMaxRingStages];
  __shared__ uint64_t s_sym_bar[kSymWarps * kSymMaxStages];
  __shared__ uint64_t s_dinv_bar[2];
  const bool sym_on = kSym && (flags & kFlagSym) != 0;
  const PatchSmem L_ = patch_smem_layout(nmax, allow_stream, (flags >> kFlagStagesShift) & 15, sym_on,
                                         (flags & kFlagSymFold) ? 1 : 0,
                                         (flags >> kFlagStagesShift) & 15);
  double* s_x = reinterpret_cast<double*>(psm + L_.x_off);
  int32_t* s_off = reinterpret_cast<int32_t*>(psm + L_.off_off);
  double* s_prod = reinterpret_cast<double*>(psm + L_.prod_off);
  double* s_L = reinterpret_cast<double*>(psm + L_.l_off);

  // regions run largest first (order, built at upload) so the long solves
  // start in the first wave and the short ones fill in behind them
  const int p = order ? order[blockIdx.x] : (int)blockIdx.x;
  const int32_t k0 = pptr[p];
  const int n = pptr[p + 1] - k0;
  SMG_DCHECK(n > 0 && n <= nmax);
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int64_t nslot = patch_slot_doubles(n, nmax, sym_on);
  const bool is_sym = kSym && kMode != kResidualOnly && patch_is_sym(n, nmax, sym_on);
  const bool staged = kMode != kResidualOnly && !is_sym && nslot <= L_.tri_cap;
  SMG_DCHECK(L_.bytes <= (int64_t)227 * 1024);
  const double* __restrict__ Lg = lfac + foff[p];
  // this thread's own patch dof (rows < kSolveThreads): b and the scatter
  // target there are fetched right after the dependency wait, off the
  // residual's and the scatter's critical paths
  const int32_t g_own = threadIdx.x < n ? dofs[k0 + threadIdx.x] : 0;
  double b_own = 0.0, t_own = 0.0;
  auto fetch_own = [&]() {
    if (kMode != kFollow && threadIdx.x < n) {
      if (kMode != kSolveFromBuf) b_own = b[g_own];
      if (kMode != kResidualOnly && scatter_add) t_own = target[g_own];
    }
  };
  // factors are stored at 16-byte aligned offsets with even lengths, so one
  // bulk copy stages the whole factor while the residual is formed
  if (staged && threadIdx.x == 0)
    factor_bulk_load(s_L, Lg, (uint32_t)(nslot * 8), &s_bar);
  // symmetric-inverse region: the first chunks of the inverse are requested now
  // (the warps' own first chunks are requested right after the barrier below)
  if (is_sym && threadIdx.x == 0) sym_ring_init(L_.nst, s_sym_bar);
  // a factor streamed through the ring: pull all of it towards L2 now, so the
  // ring's dependent copies hit L2 instead of paying HBM latency one chunk at
  // a time (the slot is contiguous, 16-byte aligned, even length)
  if (!staged && !is_sym && kMode != kResidualOnly && L_.stage > 0 &&
      (flags & kFlagL2Prefetch) && warp == 0) {
    const int64_t total = nslot * 8;
    constexpr int64_t kPiece = 32 * 1024;
    for (int64_t off = (int64_t)lane * kPiece; off < total; off += 32 * kPiece) {
      const int64_t len = total - off < kPiece ? total - off : kPiece;
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(
                       reinterpret_cast<const char*>(Lg) + off),
                   "r"((uint32_t)len)
                   : "memory");
    }
  }
  // every thread may only wait on the barrier after thread 0 has initialised it
  __syncthreads();
  if (is_sym && lane == 0)
    sym_ring_start(Lg, s_L, (int)L_.stage, L_.nst, L_.sym_rows, n, s_sym_bar,
                   (flags >> kFlagSymPfShift) & 31);

  if (kMode == kFollow) {
    // ---- follow mode: this kernel was launched (programmatic dependent
    //      launch) as soon as every CTA of the producer kernel had passed its
    //      own dependency wait, so the producer's INPUTS are complete; its
    //      output is not.  Recompute the producer on the region's ring (the
    //      columns of the patch rows) from those inputs -- the same
    //      separately rounded products, sequential sums and epilogue as the
    //      SpMV kernels, so the same bits -- then form the patch residual from
    //      the ring.  Vectors written by earlier kernels are read through L2
    //      (ld.global.cg, coherent), never from a possibly stale L1 line.
    //      The ring rows stream like the patch residual's rows: coalesced
    //      (column, value) chunks, exact products with the gathered x staged
    //      in shared memory, then every ring row summed sequentially in
    //      column order; the next chunk's loads are in flight during the sums.
    double* s_ring = reinterpret_cast<double*>(psm + L_.bytes);
    const int32_t q0 = ring_ptr[p];
    const int nr = ring_ptr[p + 1] - q0;
    int32_t* s_roff = reinterpret_cast<int32_t*>(s_ring + ((nmax_ring(fa) + 1) & ~1));
    const int64_t rbase = fa.ring.rptr[q0];
    const int rtotal = (int)(fa.ring.rptr[q0 + nr] - rbase);
    int32_t cc[kProdItems];
    double vv[kProdItems];
    auto load_ring = [&](int c0) {
#pragma unroll
      for (int it = 0; it < kProdItems; ++it) {
        const int e = c0 + it * kSolveThreads + threadIdx.x;
        cc[it] = 0;
        vv[it] = 0.0;
        if (e < rtotal && e < c0 + kProdCap) {
          cc[it] = __ldg(fa.ring.rcol + rbase + e);
          vv[it] = __ldg(fa.ring.rval + rbase + e);
        }
      }
    };
    load_ring(0);
    for (int q = threadIdx.x; q <= nr; q += kSolveThreads) {
      s_roff[q] = (int)(fa.ring.rptr[q0 + q] - rbase);
      if (q < nr) s_ring[q] = 0.0;
    }
    __syncthreads();
    for (int c0 = 0; c0 < rtotal; c0 += kProdCap) {
      const int cnt = min(kProdCap, rtotal - c0);
#pragma unroll
      for (int it = 0; it < kProdItems; ++it) {
        const int e = it * kSolveThreads + threadIdx.x;
        if (e < cnt) s_prod[e] = __dmul_rn(vv[it], __ldcg(fa.x + cc[it]));
      }
      if (c0 + kProdCap < rtotal) load_ring(c0 + kProdCap);
      __syncthreads();
      for (int q = threadIdx.x; q < nr; q += kSolveThreads) {
        const int a0 = max(s_roff[q], c0), a1 = min(s_roff[q + 1], c0 + cnt);
        double sum = s_ring[q];
        for (int e = a0; e < a1; ++e) sum = __dadd_rn(sum, s_prod[e - c0]);
        s_ring[q] = sum;
      }
      __syncthreads();
    }
    for (int q = threadIdx.x; q < nr; q += kSolveThreads) {
      const int32_t g = ring_rows[q0 + q];
      const double sum = s_ring[q];
      double v;
      if (fa.epi == (int)Epi::kAddTo) {
        v = __dadd_rn(__ldcg(fa.u_in + g), sum);
      } else {
        const double t = __dmul_rn(__ldg(fa.inv_diag + g), __dsub_rn(__ldcg(fa.b + g), sum));
        const double uv = __ldcg(fa.u_in + g);
        if (fa.epi == (int)Epi::kJacobi) {
          v = __dadd_rn(uv, __ddiv_rn(t, fa.theta));
        } else if (fa.epi == (int)Epi::kChebFirst) {
          v = __dadd_rn(uv, __ddiv_rn(t, fa.theta));
        } else {  // kChebNext
          const double d = __dadd_rn(__dmul_rn(fa.c1, __ldcg(fa.d + g)), __dmul_rn(fa.c2, t));
          v = __dadd_rn(uv, d);
        }
      }
      s_ring[q] = v;
    }
    // patch residual from the ring values: the same chunked products / row sums
    const int64_t base = prow[k0];
    const int total = (int)(prow[k0 + n] - base);
    for (int i = threadIdx.x; i <= n; i += kSolveThreads) {
      s_off[i] = (int)(prow[k0 + i] - base);
      if (i < n) s_x[i] = 0.0;
    }
    auto load_patch = [&](int c0) {
#pragma unroll
      for (int it = 0; it < kProdItems; ++it) {
        const int e = c0 + it * kSolveThreads + threadIdx.x;
        cc[it] = 0;
        vv[it] = 0.0;
        if (e < total && e < c0 + kProdCap) {
          cc[it] = __ldg(plcol + base + e);
          vv[it] = __ldg(pval + base + e);
        }
      }
    };
    load_patch(0);
    __syncthreads();
    for (int c0 = 0; c0 < total; c0 += kProdCap) {
      const int cnt = min(kProdCap, total - c0);
#pragma unroll
      for (int it = 0; it < kProdItems; ++it) {
        const int e = it * kSolveThreads + threadIdx.x;
        if (e < cnt) s_prod[e] = __dmul_rn(vv[it], s_ring[cc[it]]);
      }
      if (c0 + kProdCap < total) load_patch(c0 + kProdCap);
      __syncthreads();
      for (int i = threadIdx.x; i < n; i += kSolveThreads) {
        const int a0 = max(s_off[i], c0), a1 = min(s_off[i + 1], c0 + cnt);
        double sum = s_x[i];
        for (int e = a0; e < a1; ++e) sum = __dadd_rn(sum, s_prod[e - c0]);
        s_x[i] = sum;
      }
      __syncthreads();
    }
    for (int i = threadIdx.x; i < n; i += kSolveThreads)
      s_x[i] = __dsub_rn(__ldcg(fa.b + dofs[k0 + i]), s_x[i]);
    PTRACE(2);
  } else if (kMode != kSolveFromBuf) {
    // ---- residual rows from the region's gathered row copy (prow/pcol/pval,
    //      built at upload): coalesced streamed products, then ordered sums.
    //      The copy is static, so its first chunk is requested before the
    //      programmatic-dependency wait; u and b are read after it.
    const int64_t base = prow[k0];
    const int total = (int)(prow[k0 + n] - base);
    for (int i = threadIdx.x; i <= n; i += kSolveThreads) {
      s_off[i] = (int)(prow[k0 + i] - base);
      if (i < n) s_x[i] = 0.0;
    }
    int32_t cc[kProdItems];
    double vv[kProdItems];
    auto load_chunk = [&](int c0, int cnt) {
#pragma unroll
      for (int it = 0; it < kProdItems; ++it) {
        const int e = it * kSolveThreads + threadIdx.x;
        cc[it] = 0;
        vv[it] = 0.0;
        if (e < cnt) {
          cc[it] = __ldg(pcol + base + c0 + e);
          vv[it] = __ldg(pval + base + c0 + e);
        }
      }
    };
    load_chunk(0, min(kProdCap, total));
    patch_pdl_wait();
    fetch_own();
    PTRACE(1);
    __syncthreads();
    for (int c0 = 0; c0 < total; c0 += kProdCap) {
      const int cnt = min(kProdCap, total - c0);
      if (c0 > 0) load_chunk(c0, cnt);
#pragma unroll
      for (int it = 0; it < kProdItems; ++it) {
        const int e = it * kSolveThreads + threadIdx.x;
        if (e < cnt) {
          SMG_DCHECK(e < kProdCap && cc[it] >= 0);
          s_prod[e] = __dmul_rn(vv[it], u_res[cc[it]]);
        }
      }
      __syncthreads();
      for (int i = threadIdx.x; i < n; i += kSolveThreads) {
        const int a0 = max(s_off[i], c0), a1 = min(s_off[i + 1], c0 + cnt);
        double sum = s_x[i];
        for (int e = a0; e < a1; ++e) sum = __dadd_rn(sum, s_prod[e - c0]);
        s_x[i] = sum;
      }
      __syncthreads();
    }
    for (int i = threadIdx.x; i < n; i += kSolveThreads) {
      const double r = __dsub_rn(i == (int)threadIdx.x ? b_own : b[dofs[k0 + i]], s_x[i]);
      if (kMode == kResidualOnly)
        rbuf[k0 + i] = r;
      else
        s_x[i] = r;
    }
    PTRACE(2);
    if (kMode == kResidualOnly) return;
  } else {
    patch_pdl_wait();
    fetch_own();
    PTRACE(1);
    for (int i = threadIdx.x; i < n; i += kSolveThreads) s_x[i] = rbuf[k0 + i];
    PTRACE(2);
  }
  if (staged) factor_wait(&s_bar);
  __syncthreads();
  PTRACE(3);
  const double* L = staged ? s_L : Lg;
  const double* Dinv = L + patch_tri_even(n);   // inverted diagonal blocks, row stride 33

  const int blk = patch_block(n, nmax);
  if (is_sym && L_.sym_rows == 0) {
    sym_apply_fold(Lg, s_L, (int)L_.stage, L_.nst, n, (nmax + 2) & ~1, s_x,
                   reinterpret_cast<double*>(psm + L_.y_off),
                   reinterpret_cast<double*>(psm + L_.z_off), s_sym_bar);
  } else if (is_sym && L_.sym_rows == 2 && n <= 256 && (flags & kFlagSymReg)) {
    sym_apply_reg<8>(Lg, s_L, (int)L_.stage, L_.nst, n, (nmax + 2) & ~1, s_x,
                     reinterpret_cast<double*>(psm + L_.y_off),
                     reinterpret_cast<double*>(psm + L_.z_off), s_sym_bar,
                     (flags & kFlagSymNoFence) == 0);
  } else if (is_sym) {
    // (larger regions keep the shared-memory column sums: sym_apply_reg<16>
    // measured slower for 257..512 dofs -- 512 x1000 244 -> 261 us, 384 x1000
    // 176 -> 194 us; profiles/r02/SUMMARY.md session 5)
    sym_apply(Lg, s_L, (int)L_.stage, L_.nst, L_.sym_rows, n, (nmax + 2) & ~1, s_x,
              reinterpret_cast<double*>(psm + L_.y_off), reinterpret_cast<double*>(psm + L_.z_off),
              s_sym_bar, (flags >> kFlagSymPfShift) & 31, (flags & kFlagSymNoFence) == 0);
  } else if (blk == 2 * kPanel) {
    // x = L^{-T} (L^{-1} r): two GEMVs with the stored inverse
    gemv_inv<2 * kPanel>(L + patch_tri_even(n), s_x, n, false, s_prod);
    gemv_inv<2 * kPanel>(L + patch_tri_even(n), s_x, n, true, s_prod);
  } else if (blk == 4 * kPanel) {
    gemv_inv<4 * kPanel>(L + patch_tri_even(n), s_x, n, false, s_prod);
    gemv_inv<4 * kPanel>(L + patch_tri_even(n), s_x, n, true, s_prod);
  } else if (!staged && L_.stage > 0) {
    stream_solve(Lg, s_L, L_.stage, L_.nst, n, s_x, s_prod, s_ring_bar, s_dinv_bar, s_red);
  } else {

  // ---- forward: L y = r (left-looking over 32-row panels)
  for (int p0 = 0; p0 < n; p0 += 32) {
    const int pn = min(32, n - p0);
    if (p0 > 0) {
      // x_i -= L[i, 0:p0] . x[0:p0] for the panel's rows: 8 lanes per row,
      // all 32 rows at once
      const int r = threadIdx.x >> 3, sub = threadIdx.x & 7;
      double acc = 0.0;
      if (r < pn) {
        const double* Li = L + tri(p0 + r);
        double a1 = 0.0;
        int j = sub;
        for (; j + 8 < p0; j += 16) {
          acc += Li[j] * s_x[j];
          a1 += Li[j + 8] * s_x[j + 8];
        }
        if (j < p0) acc += Li[j] * s_x[j];
        acc += a1;
      }
      acc += __shfl_xor_sync(0xffffffffu, acc, 4);
      acc += __shfl_xor_sync(0xffffffffu, acc, 2);
      acc += __shfl_xor_sync(0xffffffffu, acc, 1);
      if (r < pn && sub == 0) s_x[p0 + r] -= acc;
      __syncthreads();
    }
    // x_P = inv(L_PP) r_P with the precomputed inverse block
    panel_gemv(Dinv + (p0 / kPanel) * kDinvBlock, s_x + p0, pn, false, s_red);
  }

  PTRACE(4);
  // ---- backward: L^T x = y (panels from the bottom)
  const int last = ((n - 1) / 32) * 32;
  for (int p0 = last; p0 >= 0; p0 -= 32) {
    const int pn = min(32, n - p0);
    const int pe = p0 + pn;
    if (pe < n) {
      double acc = 0.0;
      for (int j = pe + warp; j < n; j += kSolveWarps) {
        const double xj = s_x[j];
        if (lane < pn) acc += L[tri(j) + p0 + lane] * xj;
      }
      s_red[warp][lane] = acc;
      __syncthreads();
      if (threadIdx.x < pn) {
        double t = 0.0;
#pragma unroll
        for (int w = 0; w < kSolveWarps; ++w) t += s_red[w][threadIdx.x];
        s_x[p0 + threadIdx.x] -= t;
      }
      __syncthreads();
    }
    // x_P = inv(L_PP)^T y_P
    panel_gemv(Dinv + (p0 / kPanel) * kDinvBlock, s_x + p0, pn, true, s_red);
  }

  }  // generic (staged / global) path
  PTRACE(5);

  if constexpr (kMode == kFollow) {
    double* s_ring = reinterpret_cast<double*>(psm + L_.bytes);
    for (int i = threadIdx.x; i < n; i += kSolveThreads)
      fa.out[dofs[k0 + i]] = __dadd_rn(s_ring[bpos[k0 + i]], s_x[i]);   // u += S_c r
    // completion of this grid must imply completion of the producer (the next
    // kernel waits on this one only)
    asm volatile("griddepcontrol.wait;" ::: "memory");
  } else {
    for (int i = threadIdx.x; i < n; i += kSolveThreads) {
      const bool own = i == (int)threadIdx.x;
      const int32_t g = own ? g_own : dofs[k0 + i];
      if (scatter_add)
        target[g] = __dadd_rn(own ? t_own : target[g], s_x[i]);
      else
        target[g] = s_x[i];
    }
  }
  PTRACE(6);
}

// upload-time helpers: bounds of the patch rows, then their (col, val) copy
__global__ void patch_row_len_kernel(const DevCsr a, const int32_t* __restrict__ dofs, int64_t m,
                                     int64_t* __restrict__ len)
{
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < m) len[k] = a.rowptr[dofs[k] + 1] - a.rowptr[dofs[k]];
}

__global__ void patch_row_gather_kernel(const DevCsr a, const int32_t* __restrict__ dofs, int64_t m,
                                        const int64_t* __restrict__ prow, int32_t* __restrict__ pcol,
                                        double* __restrict__ pval)
{
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m) return;
  const int64_t lo = a.rowptr[dofs[k]], hi = a.rowptr[dofs[k] + 1];
  int64_t o = prow[k];
  for (int64_t j = lo; j < hi; ++j, ++o) {
    pcol[o] = a.col[j];
    pval[o] = a.val[j];
  }
}

cudaError_t launch_patch_row_len(const DevCsr& a, const int32_t* dofs, int64_t m, int64_t* len)
{
  if (m == 0) return cudaSuccess;
  patch_row_len_kernel<<<(unsigned)((m + 127) / 128), 128>>>(a, dofs, m, len);
  return cudaGetLastError();
}

cudaError_t launch_patch_row_gather(const DevCsr& a, const int32_t* dofs, int64_t m,
                                    const int64_t* prow, int32_t* pcol, double* pval)
{
  if (m == 0) return cudaSuccess;
  patch_row_gather_kernel<<<(unsigned)((m + 127) / 128), 128>>>(a, dofs, m, prow, pcol, pval);
  return cudaGetLastError();
}

// mask[i] = 1 iff row i of A has a column inside some patch (the rows whose
// value depends on a local correction of u)
__global__ void mark_halo_kernel(const DevCsr a, const uint8_t* __restrict__ in_patch,
                                 uint8_t* __restrict__ mask)
{
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.nrows) return;
  uint8_t h = 0;
  for (int64_t j = a.rowptr[i]; j < a.rowptr[i + 1] && !h; ++j) h = in_patch[a.col[j]];
  mask[i] = h;
}

cudaError_t launch_mark_halo(const DevCsr& a, const uint8_t* in_patch, uint8_t* mask)
{
  if (a.nrows == 0) return cudaSuccess;
  mark_halo_kernel<<<(unsigned)((a.nrows + 255) / 256), 256>>>(a, in_patch, mask);
  return cudaGetLastError();
}

__global__ void gather_kernel(const int32_t* __restrict__ idx, int64_t m,
                              const double* __restrict__ src, double* __restrict__ dst)
{
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < m) dst[k] = src[idx[k]];
}

cudaError_t launch_gather(const int32_t* idx, int64_t m, const double* src, double* dst,
                          cudaStream_t s)
{
  if (m == 0) return cudaSuccess;
  gather_kernel<<<(unsigned)((m + 127) / 128), 128, 0, s>>>(idx, m, src, dst);
  return cudaGetLastError();
}

// launch flags and shared-memory carve-up of a correction (host side; the
// kernel rebuilds the same layout from the flags)
struct PatchGeom {
  int flags;
  PatchSmem L;
};

// corrections whose larger regions hold packed inverses run the kSym kernels
static bool patch_has_sym(const Correction& c) { return c.sym && c.max_dofs > 4 * kPanel; }

static PatchGeom patch_geom(const Correction& c)
{
  static const int l2pf = patch_env("SMG_PATCH_L2PF", 0);  // measured slower on C5 (222 vs 240 us)
  // read per launch (tests vary it); a graph bakes the value of its capture
  // SMG_SYM_FOLD (default 0): folded chunks (rows c and n-1-c), ring depth
  // SMG_SYM_STAGES (default 4 folded, 2 with consecutive row pairs).  Measured
  // slower at every depth (C5 129 -> 152 us, 512 x1 39.5 -> 45.7 us, the same
  // for 2 / 3 / 4 / 6 stages; profiles/r02/SUMMARY.md session 5): the rings
  // are not waiting for bytes, and the folded chunk's three block phases cost
  // more instructions per chunk
  const int sym_fold = patch_env("SMG_SYM_FOLD", 0);
  const int sym_stages = patch_env("SMG_SYM_STAGES", sym_fold ? 4 : 2);
  // SMG_SYM_L2PF: rounds (of eight chunks) pulled towards L2 ahead of the rings
  int sym_pf = patch_env("SMG_SYM_L2PF", 0);
  sym_pf = sym_pf < 0 ? 0 : (sym_pf > 31 ? 31 : sym_pf);
  const bool st = !nostream_env();
  int nst = stages_env();
  if (patch_has_sym(c)) nst = sym_stages < 2 ? 2 : (sym_stages > kSymMaxStages ? kSymMaxStages : sym_stages);
  PatchGeom g;
  g.flags = (st ? kFlagStream : 0) | (l2pf ? kFlagL2Prefetch : 0) | (nst << kFlagStagesShift) |
            (c.sym ? kFlagSym : 0) | (sym_pf << kFlagSymPfShift) |
            ((c.sym && sym_fold) ? kFlagSymFold : 0) |
            (patch_env("SMG_SYM_NOFENCE", 0) ? kFlagSymNoFence : 0) |
            (patch_env("SMG_SYM_REG", 1) ? kFlagSymReg : 0);
  g.L = patch_smem_layout(c.max_dofs, st, nst, c.sym, (c.sym && sym_fold) ? 1 : 0, nst);
  return g;
}

template <int kMode>
static cudaError_t launch_patch(const Correction& c, size_t smem, const double* b,
                                const double* u_res, double* tgt, int add, int flags,
                                cudaStream_t s)
{
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)c.n_regions);
  cfg.blockDim = dim3(kSolveThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  static const int lpt = patch_env("SMG_PATCH_LPT", 1);
  auto fn = patch_has_sym(c) ? patch_kernel<kMode, true> : patch_kernel<kMode, false>;
  return cudaLaunchKernelEx(&cfg, fn, c.prow, c.pcol, c.pval, c.pptr, c.dofs,
                            c.foff, c.lfac, b, u_res, c.rbuf, tgt, add, c.max_dofs, flags,
                            lpt ? c.order : (const int32_t*)nullptr, FollowArgs(),
                            (const int32_t*)nullptr, (const int32_t*)nullptr,
                            (const int32_t*)nullptr, (const int32_t*)nullptr);
}

static size_t follow_smem(const Correction& c)
{
  const PatchSmem L = patch_geom(c).L;
  return (size_t)L.bytes + 8 * (size_t)((c.ring_max + 1) & ~1) + 4 * (size_t)(c.ring_max + 2);
}

bool patch_follow_fits(const Correction& c) { return follow_smem(c) <= 227 * 1024; }

// follow mode: launched right after its producer kernel (programmatic
// dependent launch), runs concurrently with it, waits for it at the end
cudaError_t launch_patch_follow(const Correction& c, const FollowArgs& fa, cudaStream_t s)
{
  if (c.n_regions == 0) return cudaSuccess;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)c.n_regions);
  cfg.blockDim = dim3(kSolveThreads);
  cfg.dynamicSmemBytes = follow_smem(c);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  static const int lpt = patch_env("SMG_PATCH_LPT", 1);
  FollowArgs f = fa;
  f.ring_max = c.ring_max;
  auto fn = patch_has_sym(c) ? patch_kernel<kFollow, true> : patch_kernel<kFollow, false>;
  return cudaLaunchKernelEx(&cfg, fn, c.prow, c.pcol, c.pval, c.pptr, c.dofs,
                            c.foff, c.lfac, fa.b, (const double*)nullptr, c.rbuf, fa.out, 1,
                            c.max_dofs, patch_geom(c).flags,
                            lpt ? c.order : (const int32_t*)nullptr, f, c.ring_ptr, c.ring_rows,
                            c.plcol, c.bpos);
}

// residual-only pass (coupled regions): rbuf[k] = (b - A u)[dofs[k]]
cudaError_t launch_patch_residual(const DevCsr& a, const Correction& c, const double* b,
                                  const double* u, cudaStream_t s)
{
  (void)a;
  if (c.n_regions == 0) return cudaSuccess;
  const PatchGeom g = patch_geom(c);
  // only the residual buffers (everything before the factor / ring area)
  const size_t smem = (size_t)(g.L.sym ? g.L.y_off : g.L.l_off);
  return launch_patch<kResidualOnly>(c, smem, b, u, nullptr, 0, g.flags, s);
}

static size_t smem_pad()
{
  static long pad = -1;
  if (pad < 0) {
    const char* v = getenv("SMG_PATCH_SMEM_PAD");
    pad = v ? atol(v) : 0;
  }
  return (size_t)pad;
}

// u_add != nullptr -> u += x ; else out_scatter[dofs] = x.  fused: residual in-kernel.
cudaError_t launch_patch_solve(const Correction& c, const double* b, const double* u_res,
                               double* u_add, double* out_scatter, bool fused, cudaStream_t s)
{
  if (c.n_regions == 0) return cudaSuccess;
  const PatchGeom g = patch_geom(c);
  double* tgt = u_add ? u_add : out_scatter;
  const int add = u_add ? 1 : 0;
  const size_t smem = (size_t)g.L.bytes + smem_pad();
  if (fused) return launch_patch<kAddResidualSolve>(c, smem, b, u_res, tgt, add, g.flags, s);
  return launch_patch<kSolveFromBuf>(c, smem, b, u_res, tgt, add, g.flags, s);
}

// The attribute is per kernel, shared by every correction: it only ever grows
// (a smaller correction created later must not lower it under a larger one's
// launch size).
cudaError_t configure_patch_solve_smem(const Correction& c)
{
  static int cur[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const PatchSmem L = patch_geom(c).L;
  const bool sym = patch_has_sym(c);
  const int bytes = (int)(L.bytes + smem_pad());
  cudaError_t e = cudaSuccess;
  auto grow = [&](int mode, auto fn, int need) {
    const int slot = mode + (sym ? 4 : 0);
    if (e == cudaSuccess && need > cur[slot]) {
      e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, need);
      if (e == cudaSuccess) cur[slot] = need;
    }
  };
  const int rbytes = (int)(L.sym ? L.y_off : L.l_off);
  if (sym) {
    grow(kAddResidualSolve, patch_kernel<kAddResidualSolve, true>, bytes);
    grow(kSolveFromBuf, patch_kernel<kSolveFromBuf, true>, bytes);
    grow(kResidualOnly, patch_kernel<kResidualOnly, true>, rbytes);
    if (c.has_ring && patch_follow_fits(c))
      grow(kFollow, patch_kernel<kFollow, true>, (int)follow_smem(c));
  } else {
    grow(kAddResidualSolve, patch_kernel<kAddResidualSolve, false>, bytes);
    grow(kSolveFromBuf, patch_kernel<kSolveFromBuf, false>, bytes);
    grow(kResidualOnly, patch_kernel<kResidualOnly, false>, rbytes);
    if (c.has_ring && patch_follow_fits(c))
      grow(kFollow, patch_kernel<kFollow, false>, (int)follow_smem(c));
  }
  return e;
}

}  // namespace smg

#ifdef SMG_PATCH_TRACE
extern "C" __attribute__((visibility("default"))) int smg_debug_patch_trace(unsigned long long* out)
{
  return (int)cudaMemcpyFromSymbol(out, smg::g_patch_trace, sizeof(smg::g_patch_trace));
}
#endif
