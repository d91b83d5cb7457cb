// C-ABI implementation: device-resident operators, patch sets and the V-cycle
// runtime (graph-captured) behind include/simplexmg_b200.h.
//
// Host arithmetic for smoother scalars follows smoothers.py:109-135 exactly
// (compiled with -ffp-contract=off), so the scalars fed to the kernels equal
// the Python floats the reference computes.
#include "../../include/simplexmg_b200.h"
#include "smg_internal.cuh"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <thread>
#include <utility>

namespace smg {


static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }
int fail(const std::string& msg)
{
  set_error(msg);
  return SMG_ERR_INVALID;
}
int check_cuda(cudaError_t e, const char* what)
{
  if (e == cudaSuccess) return SMG_OK;
  set_error(std::string(what) + ": " + cudaGetErrorString(e));
  return SMG_ERR_CUDA;
}

#define SMG_TRY(expr)                      \
  do {                                     \
    int _rc = (expr);                      \
    if (_rc != SMG_OK) return _rc;         \
  } while (0)
#define SMG_CUDA(expr) SMG_TRY(check_cuda((expr), #expr))

template <typename T>
static int dev_upload(std::vector<void*>& allocs, int64_t& bytes, const T* host, size_t n,
                      T** out)
{
  *out = nullptr;
  if (n == 0) return SMG_OK;
  void* p = nullptr;
  SMG_CUDA(cudaMalloc(&p, n * sizeof(T)));
  allocs.push_back(p);
  bytes += (int64_t)(n * sizeof(T));
  if (host) SMG_CUDA(cudaMemcpy(p, host, n * sizeof(T), cudaMemcpyHostToDevice));
  *out = static_cast<T*>(p);
  return SMG_OK;
}

template <typename T>
static int dev_alloc(std::vector<void*>& allocs, int64_t& bytes, size_t n, T** out)
{
  return dev_upload<T>(allocs, bytes, nullptr, n, out);
}

static void free_all(std::vector<void*>& allocs)
{
  for (void* p : allocs) cudaFree(p);
  allocs.clear();
}

// Greedy tile partition: consecutive rows, <= kRowsPerTile rows, <= cap
// nonzeros unless a single row is longer.  Small operators (coarse levels)
// get smaller tiles so every SM still has several independent CTAs.
// Multi-chunk tiles (csr_tile_kernel<.., kMulti>) for operators whose rows
// average >= SMG_MC_MIN_ROW nonzeros (default 24) -- except operators streamed
// from HBM with rows averaging >= SMG_MC_MAX_STREAM_ROW (default 36), where the
// per-chunk serialisation cost more than it saved (profiles/r01/ab_multichunk:
// C5 and C4's fine level gain 4-10 %, C2 level 1 and C4 levels 1-2 lose).
static bool long_rows(int64_t nnz, int64_t nrows)
{
  static int mc_row = -1, mc_stream_max = -1;
  if (mc_row < 0) {
    const char* v = getenv("SMG_MC_MIN_ROW");
    mc_row = v ? atoi(v) : 24;
    if (mc_row < 0) mc_row = 0;
    v = getenv("SMG_MC_MAX_STREAM_ROW");
    mc_stream_max = v ? atoi(v) : 36;
  }
  if (mc_row == 0 || nrows == 0 || nnz < (int64_t)mc_row * nrows) return false;
  const bool streamed = nnz * 12 > kStreamBytes;
  return !streamed || mc_stream_max <= 0 || nnz < (int64_t)mc_stream_max * nrows;
}

static int64_t tile_cap_for(int64_t nnz, int64_t nrows)
{
  static int per_sm = -1, mc_chunks = -1;
  if (per_sm < 0) {
    const char* v = getenv("SMG_TILES_PER_SM");
    per_sm = v ? atoi(v) : 4;
    if (per_sm <= 0) per_sm = 4;
    v = getenv("SMG_MC_CHUNKS");
    mc_chunks = v ? atoi(v) : kMaxTileChunks;
    if (mc_chunks < 1 || mc_chunks > kMaxTileChunks) mc_chunks = kMaxTileChunks;
  }
  const int64_t max_cap = long_rows(nnz, nrows) ? (int64_t)kTileNnz * mc_chunks : kTileNnz;
  const int64_t want = nnz / (148 * per_sm);  // ~per_sm tiles per SM
  int64_t cap = 256;
  while (cap < want && cap < max_cap) cap *= 2;
  return cap;
}

static std::vector<int32_t> make_tiles(int64_t nrows, const int64_t* rowptr, int64_t cap = 0)
{
  if (cap <= 0) cap = tile_cap_for(rowptr[nrows], nrows);
  std::vector<int32_t> t;
  t.reserve((size_t)(nrows / 64 + 2));
  t.push_back(0);
  int64_t r = 0;
  while (r < nrows) {
    const int64_t start = r;
    const int64_t base = rowptr[r];
    ++r;
    while (r < nrows && r - start < kRowsPerTile && rowptr[r + 1] - base <= cap) ++r;
    t.push_back((int32_t)r);
  }
  return t;
}

static bool stream_env()
{
  const char* v = getenv("SMG_EVICT_FIRST");
  return !(v && v[0] == '0');
}

// forced_layout: -1 = by the measured rule, else SMG_LAYOUT_* (tests / A-B);
// forced_unroll: SELL loop depth (0 = by the rule)
static int build_devcsr(std::vector<void*>& allocs, int64_t& bytes, int64_t nrows, int64_t ncols,
                        const int64_t* rowptr, const int64_t* col64, const double* val,
                        DevCsr* out, int forced_layout = -1, int forced_unroll = 0)
{
  const int64_t nnz = rowptr[nrows];
  // padded so the TMA ring may read up to 16 B past the last element
  std::vector<int32_t> col32((size_t)nnz + 4, 0);
  for (int64_t j = 0; j < nnz; ++j) col32[(size_t)j] = (int32_t)col64[j];
  std::vector<double> valp((size_t)nnz + 2, 0.0);
  if (nnz) std::memcpy(valp.data(), val, sizeof(double) * (size_t)nnz);
  std::vector<int64_t> rpp((size_t)nrows + 3, nnz);
  std::memcpy(rpp.data(), rowptr, sizeof(int64_t) * (size_t)(nrows + 1));
  // fixed-capacity tiles (DevCsr::fixed): shrink the capacity while whole
  // tiles of kRowsPerTile average rows would not fill it (little padding)
  int64_t cap = tile_cap_for(nnz, nrows);
  static const bool fixed_env = [] {
    const char* e = getenv("SMG_FIXED_TILES");
    return !(e && e[0] == '0');
  }();
  // (multi-chunk operators keep the offset-table layout: with ~27 nonzeros per
  // row their tiles are row-bound, and shrinking them to avoid padding measured
  // slower on C5, profiles/r01/ab_fixed_tiles/)
  bool fixed = fixed_env && nrows > 0 && !long_rows(nnz, nrows);
  if (forced_layout >= 0) fixed = forced_layout == SMG_LAYOUT_TILES_FIXED && nrows > 0;
  if (fixed && !long_rows(nnz, nrows)) {
    while (cap > 256 && kRowsPerTile * nnz < cap * nrows) cap /= 2;
  }
  std::vector<int32_t> tiles = make_tiles(nrows, rowptr, cap);
  std::vector<int64_t> tnz(tiles.size());
  for (size_t i = 0; i < tiles.size(); ++i) tnz[i] = rowptr[tiles[i]];
  for (size_t i = 0; fixed && i + 1 < tiles.size(); ++i)
    if (tnz[i + 1] - tnz[i] > cap) fixed = false;   // a single row longer than the capacity
  DevCsr d;
  d.nrows = nrows;
  d.ncols = ncols;
  d.nnz = nnz;
  d.ntiles = (int32_t)(tiles.size() - 1);
  d.streaming = stream_env() && nnz * 12 > kStreamBytes;
  d.multichunk = long_rows(nnz, nrows);
  int64_t* rp = nullptr;
  int32_t* c = nullptr;
  double* v = nullptr;
  int32_t* tr = nullptr;
  int64_t* tz = nullptr;
  SMG_TRY(dev_upload(allocs, bytes, rpp.data(), rpp.size(), &rp));
  SMG_TRY(dev_upload(allocs, bytes, col32.data(), col32.size(), &c));
  SMG_TRY(dev_upload(allocs, bytes, valp.data(), valp.size(), &v));
  SMG_TRY(dev_upload(allocs, bytes, tiles.data(), tiles.size(), &tr));
  SMG_TRY(dev_upload(allocs, bytes, tnz.data(), tnz.size(), &tz));
  d.rowptr = rp;
  d.col = c;
  d.val = v;
  d.tile_row = tr;
  d.tile_nz = tz;
  // SMG_SELL: 0 = never, 1 = every operator, unset/2 = by measurement
  // (profiles/r01/ab_sell/): short rows (avg < SMG_SELL_MAX_ROW = 20) with at
  // least SMG_SELL_MIN_WIN = 296 windows run SELL with a 4-deep loop (8 CTAs
  // per SM); longer rows with at least SMG_SELL_MIN_WIN_LONG = 592 windows run
  // SELL with an SMG_SELL_LONG_UNROLL-deep loop (default 8; more loads in
  // flight per thread); operators with fewer windows keep the tile kernel,
  // whose CTAs share a row's products across all threads
  auto env_int = [](const char* name, int dflt) {
    const char* e = getenv(name);
    return e ? atoi(e) : dflt;
  };
  static const int sell_mode = env_int("SMG_SELL", 2);
  static const int sell_max_row = env_int("SMG_SELL_MAX_ROW", 20);
  static const int sell_min_win = env_int("SMG_SELL_MIN_WIN", 296);
  static const int sell_min_win_long = env_int("SMG_SELL_MIN_WIN_LONG", 592);
  static const int sell_long_unroll = env_int("SMG_SELL_LONG_UNROLL", 8);
  const int64_t nwin_est = (nrows + kSellWindow - 1) / kSellWindow;
  const bool short_rows = nnz < (int64_t)sell_max_row * nrows;
  bool use_sell =
      nrows > 0 && (sell_mode == 1 ||
                    (sell_mode >= 2 && nwin_est >= (short_rows ? sell_min_win : sell_min_win_long)));
  if (forced_layout >= 0)
    use_sell = (forced_layout == SMG_LAYOUT_SELL || forced_layout == SMG_LAYOUT_SELL_D16) && nrows > 0;
  d.sell_unroll = short_rows ? 4 : sell_long_unroll;
  if (forced_unroll > 0) d.sell_unroll = forced_unroll >= 16 ? 16 : (forced_unroll >= 8 ? 8 : 4);
  // SELL-8x4 (SMG_SELL4: 0 = only when forced, 1 = every long-row
  // operator the rule above leaves to the tiles).  Measured slower than the
  // tiles on C1-C3 and even on C4 (profiles/r01/ab_sell4/): 64-row windows
  // with 4 batches in flight fit 4 CTAs per SM, so C2 level 2 needs 1.7 waves,
  // and the 2-batch build (8 CTAs per SM) spills and keeps too few loads in flight
  // 2: only very long rows (>= SMG_SELL4_AUTO_ROW = 200 per row, C4 level 2),
  // 4 batches in flight -- its sweep gets faster (158 -> 152 us) but the C4
  // V-cycle does not (178.2 -> 176.5 /s; profiles/r01/ab_sell4/auto_*), so the
  // default stays 0.
  static const int sell4_mode = env_int("SMG_SELL4", 0);
  static const int sell4_min_row = env_int("SMG_SELL4_MIN_ROW", 20);
  static const int sell4_auto_row = env_int("SMG_SELL4_AUTO_ROW", 200);
  static const int sell4_unroll = env_int("SMG_SELL4_UNROLL", sell4_mode == 2 ? 4 : 2);
  bool use_sell4 = nrows > 0 && !use_sell && sell4_mode >= 1 &&
                   nnz >= (int64_t)(sell4_mode == 2 ? sell4_auto_row : sell4_min_row) * nrows;
  if (forced_layout >= 0) use_sell4 = forced_layout == SMG_LAYOUT_SELL4 && nrows > 0;
  if (use_sell4) {
    const int64_t nw = (nrows + kSell4Window - 1) / kSell4Window;
    std::vector<int16_t> perm((size_t)(nw * kSell4Window), -1);
    std::vector<int64_t> sptr((size_t)(nw * kSellSlices + 1), 0);
    std::vector<int32_t> idx(kSell4Window);
    for (int64_t w = 0; w < nw; ++w) {
      const int64_t r0 = w * kSell4Window;
      const int cntw = (int)std::min<int64_t>(kSell4Window, nrows - r0);
      for (int i = 0; i < cntw; ++i) idx[(size_t)i] = i;
      std::stable_sort(idx.begin(), idx.begin() + cntw, [&](int a, int b) {
        return rowptr[r0 + a + 1] - rowptr[r0 + a] > rowptr[r0 + b + 1] - rowptr[r0 + b];
      });
      for (int sl = 0; sl < cntw; ++sl) perm[(size_t)(r0 + sl)] = (int16_t)idx[(size_t)sl];
      for (int k = 0; k < kSellSlices; ++k) {
        int64_t width = 0;   // batches of 4 entries
        for (int l = 0; l < 8; ++l) {
          const int sl = k * 8 + l;
          if (sl < cntw) {
            const int64_t r = r0 + idx[(size_t)sl];
            width = std::max<int64_t>(width, (rowptr[r + 1] - rowptr[r] + 3) / 4);
          }
        }
        sptr[(size_t)(w * kSellSlices + k + 1)] = sptr[(size_t)(w * kSellSlices + k)] + 32 * width;
      }
    }
    const int64_t total = sptr.back();
    std::vector<int32_t> scol((size_t)total + 4, -1);
    std::vector<double> sval((size_t)total + 2, 0.0);
    for (int64_t w = 0; w < nw; ++w) {
      const int64_t r0 = w * kSell4Window;
      for (int sl = 0; sl < kSell4Window; ++sl) {
        const int16_t pr = perm[(size_t)(r0 + sl)];
        if (pr < 0) continue;
        const int64_t r = r0 + pr;
        const int64_t base = sptr[(size_t)(w * kSellSlices + sl / 8)] + 4 * (sl % 8);
        for (int64_t j = rowptr[r]; j < rowptr[r + 1]; ++j) {
          const int64_t e = j - rowptr[r];
          const int64_t at = base + (e / 4) * 32 + (e % 4);
          scol[(size_t)at] = col32[(size_t)j];
          sval[(size_t)at] = val[j];
        }
      }
    }
    int64_t* dsp = nullptr;
    int16_t* dperm = nullptr;
    int32_t* dsc = nullptr;
    double* dsv = nullptr;
    SMG_TRY(dev_upload(allocs, bytes, sptr.data(), sptr.size(), &dsp));
    SMG_TRY(dev_upload(allocs, bytes, perm.data(), perm.size(), &dperm));
    SMG_TRY(dev_upload(allocs, bytes, scol.data(), scol.size(), &dsc));
    SMG_TRY(dev_upload(allocs, bytes, sval.data(), sval.size(), &dsv));
    d.sell = true;
    d.sell_lanes = 4;
    d.sell_unroll = forced_unroll > 0 ? (forced_unroll >= 4 ? 4 : 2) : (sell4_unroll >= 4 ? 4 : 2);
    fixed = false;
    d.sell_nwin = (int32_t)nw;
    d.sell_ptr = dsp;
    d.sell_perm = dperm;
    d.sell_col = dsc;
    d.sell_val = dsv;
  }
  if (use_sell) {
    // SELL-32-sigma256: per window of 256 rows, slots sorted by row length
    // (stable, descending), 8 slices of 32 slots, column-major within a slice
    const int64_t nw = (nrows + kSellWindow - 1) / kSellWindow;
    std::vector<int16_t> perm((size_t)(nw * kSellWindow), -1);
    std::vector<int64_t> sptr((size_t)(nw * kSellSlices + 1), 0);
    std::vector<int32_t> idx(kSellWindow);
    for (int64_t w = 0; w < nw; ++w) {
      const int64_t r0 = w * kSellWindow;
      const int cntw = (int)std::min<int64_t>(kSellWindow, nrows - r0);
      for (int i = 0; i < cntw; ++i) idx[(size_t)i] = i;
      std::stable_sort(idx.begin(), idx.begin() + cntw, [&](int a, int b) {
        return rowptr[r0 + a + 1] - rowptr[r0 + a] > rowptr[r0 + b + 1] - rowptr[r0 + b];
      });
      for (int sl = 0; sl < cntw; ++sl) perm[(size_t)(r0 + sl)] = (int16_t)idx[(size_t)sl];
      for (int k = 0; k < kSellSlices; ++k) {
        int64_t width = 0;
        for (int l = 0; l < 32; ++l) {
          const int sl = k * 32 + l;
          if (sl < cntw) {
            const int64_t r = r0 + idx[(size_t)sl];
            width = std::max<int64_t>(width, rowptr[r + 1] - rowptr[r]);
          }
        }
        sptr[(size_t)(w * kSellSlices + k + 1)] = sptr[(size_t)(w * kSellSlices + k)] + 32 * width;
      }
    }
    const int64_t total = sptr.back();
    std::vector<int32_t> scol((size_t)total + 4, -1);
    std::vector<double> sval((size_t)total + 2, 0.0);
    for (int64_t w = 0; w < nw; ++w) {
      const int64_t r0 = w * kSellWindow;
      for (int sl = 0; sl < kSellWindow; ++sl) {
        const int16_t pr = perm[(size_t)(r0 + sl)];
        if (pr < 0) continue;
        const int64_t r = r0 + pr;
        const int64_t base = sptr[(size_t)(w * kSellSlices + sl / 32)] + (sl % 32);
        for (int64_t j = rowptr[r]; j < rowptr[r + 1]; ++j) {
          scol[(size_t)(base + (j - rowptr[r]) * 32)] = col32[(size_t)j];
          sval[(size_t)(base + (j - rowptr[r]) * 32)] = val[j];
        }
      }
    }
    // SELL-d16 (SMG_LAYOUT_SELL_D16; by the rule only with SMG_SELL_DELTA=1):
    // 16-bit column codes where every row needs at most two escapes and the
    // column stream shrinks by >= 10 %.  Measured slower than int32 columns on
    // C2 (fine sweep 29.1 -> 34.2 us, level 1 25.8 -> 29.5 us, 1,637 -> 1,489
    // V-cycles/s; profiles/r02/SUMMARY.md): the sweeps are latency-bound, and
    // the decode sits between the column load and the gather.  Kept as a
    // forced layout (bit-identical, tests/test_gpu_layouts.py).
    static const int delta_env = env_int("SMG_SELL_DELTA", 0);
    const bool delta_forced = forced_layout == SMG_LAYOUT_SELL_D16;
    bool delta = delta_forced || (delta_env >= 1 && forced_layout < 0);
    int planes = 0;
    std::vector<uint16_t> dcol;
    std::vector<int32_t> c0v, escv;
    if (delta) {
      const size_t nslot = (size_t)(nw * kSellWindow);
      dcol.assign((size_t)total + 8, (uint16_t)0xFFFE);
      c0v.assign(nslot, 0);
      escv.assign(2 * nslot, 0);
      for (int64_t w = 0; w < nw && delta; ++w) {
        const int64_t r0 = w * kSellWindow;
        for (int sl = 0; sl < kSellWindow && delta; ++sl) {
          const int16_t pr = perm[(size_t)(r0 + sl)];
          if (pr < 0) continue;
          const int64_t r = r0 + pr;
          const int64_t base = sptr[(size_t)(w * kSellSlices + sl / 32)] + (sl % 32);
          int ne = 0;
          int64_t prev = 0;
          for (int64_t j = rowptr[r]; j < rowptr[r + 1]; ++j) {
            const int64_t cj = col32[(size_t)j];
            uint16_t code;
            if (j == rowptr[r]) {
              c0v[(size_t)(r0 + sl)] = (int32_t)cj;
              code = 0;
            } else if (cj - prev >= 0 && cj - prev <= 0xFFFD) {
              code = (uint16_t)(cj - prev);
            } else if (ne < 2) {
              escv[(size_t)ne * nslot + (size_t)(r0 + sl)] = (int32_t)cj;
              ++ne;
              code = 0xFFFF;
            } else {
              delta = false;   // a row with three far jumps: keep int32 columns
              break;
            }
            prev = cj;
            dcol[(size_t)(base + (j - rowptr[r]) * 32)] = code;
          }
          planes = std::max(planes, ne);
        }
      }
      // worth it only if the column stream really shrinks
      if (delta && !delta_forced &&
          10 * (2 * total + 4 * nw * kSellWindow * (1 + planes)) > 9 * 4 * total)
        delta = false;
    }
    int64_t* dsp = nullptr;
    int16_t* dperm = nullptr;
    int32_t* dsc = nullptr;
    double* dsv = nullptr;
    SMG_TRY(dev_upload(allocs, bytes, sptr.data(), sptr.size(), &dsp));
    SMG_TRY(dev_upload(allocs, bytes, perm.data(), perm.size(), &dperm));
    if (delta) {
      uint16_t* ddc = nullptr;
      int32_t *dc0 = nullptr, *desc = nullptr;
      escv.resize((size_t)std::max(planes, 1) * (size_t)(nw * kSellWindow));
      SMG_TRY(dev_upload(allocs, bytes, dcol.data(), dcol.size(), &ddc));
      SMG_TRY(dev_upload(allocs, bytes, c0v.data(), c0v.size(), &dc0));
      SMG_TRY(dev_upload(allocs, bytes, escv.data(), escv.size(), &desc));
      d.sell_delta = true;
      d.sell_esc_planes = planes;
      d.sell_dcol = ddc;
      d.sell_c0 = dc0;
      d.sell_esc = desc;
    } else {
      SMG_TRY(dev_upload(allocs, bytes, scol.data(), scol.size(), &dsc));
    }
    SMG_TRY(dev_upload(allocs, bytes, sval.data(), sval.size(), &dsv));
    d.sell = true;
    // software-pipelined loop for long rows up to SMG_SELL_PIPE_MAX_ROW (64)
    // nonzeros per row: C2 level 1 (41) 28.2 -> 25.9 us, C4 level 0 (26.5)
    // 547 -> 503 us; C4 level 1 (172) loses (363 -> 381 us), keeps the plain
    // loop (profiles/r01/ab_pipe/)
    static const int pipe_max_row = env_int("SMG_SELL_PIPE_MAX_ROW", 64);
    d.sell_pipe = (d.sell_unroll == 8 && nnz < (int64_t)pipe_max_row * nrows) ? 6 : 0;
    fixed = false;   // the sweeps run on the SELL arrays: no padded tile copy
    d.sell_nwin = (int32_t)nw;
    d.sell_ptr = dsp;
    d.sell_perm = dperm;
    d.sell_col = dsc;
    d.sell_val = dsv;
  }
  // Streamed operators with very long rows that are too small for SELL (C4
  // level 2: 117,649 rows x 335 nonzeros): single-chunk tiles hold six rows,
  // whose owners add 335 products each while 250 threads wait (0.49 of HBM in
  // every layout, profiles/r02/af/).  Staged whole in 9,216-product tiles
  // (27 rows summing at once, three CTAs per SM, several resident waves) they
  // measured SLOWER (146 -> 158 us per step, C4 197.9 -> 194.8 V-cycles/s;
  // bit-identical, profiles/r02/ah/), so this is opt-in:
  // SMG_STAGE_STREAM_MIN_ROW = least average row length (default 0 = off).
  static const int stage_stream_min_row = env_int("SMG_STAGE_STREAM_MIN_ROW", 0);
  const bool stage_stream = forced_layout < 0 && env_int("SMG_TILE_STAGE", 1) != 0 &&
                            stage_stream_min_row > 0 && nrows > 0 && !d.sell &&
                            nnz * 12 > kStreamBytes &&
                            nnz >= (int64_t)stage_stream_min_row * nrows;
  if (stage_stream) fixed = false;
  if (fixed) {
    const size_t nt = tiles.size() - 1;
    std::vector<int32_t> pc(nt * (size_t)cap + 4, 0);
    std::vector<double> pv(nt * (size_t)cap + 2, 0.0);
    std::vector<int32_t> rel((size_t)nrows);
    for (size_t t = 0; t < nt; ++t) {
      const int64_t b = tnz[t], e = tnz[t + 1];
      for (int64_t j = b; j < e; ++j) {
        pc[t * (size_t)cap + (size_t)(j - b)] = col32[(size_t)j];
        pv[t * (size_t)cap + (size_t)(j - b)] = val[j];
      }
      for (int32_t r = tiles[t]; r < tiles[t + 1]; ++r)
        rel[(size_t)r] = (int32_t)(rowptr[r + 1] - b);
    }
    int32_t* dpc = nullptr;
    double* dpv = nullptr;
    int32_t* drel = nullptr;
    SMG_TRY(dev_upload(allocs, bytes, pc.data(), pc.size(), &dpc));
    SMG_TRY(dev_upload(allocs, bytes, pv.data(), pv.size(), &dpv));
    SMG_TRY(dev_upload(allocs, bytes, rel.data(), rel.size(), &drel));
    d.fixed = true;
    d.cap = (int32_t)cap;
    d.pcol = dpc;
    d.pval = dpv;
    d.rel_end = drel;
  }
  // Whole-tile staging (csr_stage_kernel, SMG_LAYOUT_TILES_STAGED): long-row
  // operators that stay in L2 and keep the offset-table tiles get tiles sized
  // so that the operator is one resident wave of kStageCtas CTAs per SM (at
  // most kStageMaxNnz nonzeros each), staged whole in shared memory.
  // SMG_TILE_STAGE=0 keeps the chunked tile kernel.
  static const int stage_mode = env_int("SMG_TILE_STAGE", 1);
  bool stage = stage_mode != 0 && nrows > 0 && !d.sell && !d.fixed &&
               nnz * 12 <= kStreamBytes && long_rows(nnz, nrows);
  if (forced_layout >= 0) stage = forced_layout == SMG_LAYOUT_TILES_STAGED && nrows > 0;
  if (stage_stream) stage = true;
  if (stage) {
    const int64_t slots = (int64_t)(148 * kStageCtas * 95) / 100;
    int64_t scap = ((nnz + slots - 1) / slots + 255) & ~int64_t(255);
    if (scap < 1024) scap = 1024;
    if (stage_stream) scap = kStageMaxNnz;   // several resident waves of the largest tiles
    // by the rule only operators whose one-wave tiles stay small
    // (SMG_STAGE_MAX_CAP nonzeros, default 6144 = 48 KB per CTA; measured
    // gains up to 4,608: C2 level 3 and C3 levels 1-2): with 72 KB tiles
    // (C2 level 2) the kernel alone is faster (13.8 -> 12.2 us) but the
    // V-cycle is not -- three such CTAs leave the SM 28 KB of L1 for the x
    // gathers and no room for the next kernel's programmatic early launch,
    // and level 1's sweeps next to it lose 8 us (profiles/r02/SUMMARY.md,
    // session 5)
    static const int stage_max_cap = env_int("SMG_STAGE_MAX_CAP", 6144);
    // SMG_STAGE_WAVES (default 1): operators whose one-wave tiles are too
    // large may be staged as that many resident waves of smaller tiles
    static const int stage_waves = env_int("SMG_STAGE_WAVES", 1);
    for (int w = 2; forced_layout < 0 && !stage_stream && scap > stage_max_cap && w <= stage_waves; ++w) {
      scap = ((nnz + slots * w - 1) / (slots * w) + 255) & ~int64_t(255);
      if (scap < 1024) scap = 1024;
    }
    if (forced_layout < 0 && !stage_stream && scap > stage_max_cap) stage = false;
    if (scap > kStageMaxNnz) scap = kStageMaxNnz;
    std::vector<int32_t> st;
    if (stage) st = make_tiles(nrows, rowptr, scap);
    std::vector<int64_t> sz(st.size());
    for (size_t i = 0; i < st.size(); ++i) sz[i] = rowptr[st[i]];
    for (size_t i = 0; stage && i + 1 < st.size(); ++i)
      if (sz[i + 1] - sz[i] > scap) stage = false;   // a single row longer than the capacity
    if (stage) {
      int32_t* str = nullptr;
      int64_t* stz = nullptr;
      SMG_TRY(dev_upload(allocs, bytes, st.data(), st.size(), &str));
      SMG_TRY(dev_upload(allocs, bytes, sz.data(), sz.size(), &stz));
      d.tile_row = str;
      d.tile_nz = stz;
      d.ntiles = (int32_t)(st.size() - 1);
      d.stage_cap = (int32_t)scap;
    }
  }
  *out = d;
  return SMG_OK;
}

// ---------------------------------------------------------------------------
// smoother scalars, smoothers.py:109-135
struct ChebScalars {
  bool collapsed = false;
  double theta = 0, delta = 0, sigma = 0;
  std::vector<std::pair<double, double>> steps;  // (c1, c2) for sweeps 2..k
};

static int cheb_scalars(int sweeps, double lambda_max, double frac, ChebScalars* out)
{
  if (!(lambda_max > 0.0)) {
    set_error("chebyshev_smooth requires a positive cfg.lambda_max");
    return SMG_ERR_INVALID;
  }
  if (sweeps < 1) return fail("sweeps must be at least 1");
  const double lam_max = lambda_max;
  const double lam_min = frac * lam_max;
  ChebScalars s;
  s.theta = 0.5 * (lam_max + lam_min);
  s.delta = 0.5 * (lam_max - lam_min);
  if (s.delta == 0.0) {
    s.collapsed = true;
  } else {
    s.sigma = s.theta / s.delta;
    double rho = 1.0 / s.sigma;
    for (int k = 1; k < sweeps; ++k) {
      const double rho_next = 1.0 / (2.0 * s.sigma - rho);
      const double c1 = rho_next * rho;
      const double c2 = 2.0 * rho_next / s.delta;
      s.steps.emplace_back(c1, c2);
      rho = rho_next;
    }
  }
  *out = s;
  return SMG_OK;
}

// k steps ping-ponging between *cur and *alt (the reference computes the full
// A u before updating u, so the gathering SpMV never writes its own input).
// With `follow` the last step skips the patch dofs and leaves d alone (it is
// dead after the last step), and the correction that follows the smoother
// runs concurrently with that step (patch_kernel<kFollow>: it recomputes the
// step on its rings, then writes u_out on the patch dofs); *followed reports
// whether that happened (no step launched -> the caller corrects as usual).
static int enqueue_global_smooth(const Operator& op, const double* b, double** cur, double** alt,
                                 double* d, int sweeps, const ChebScalars& cs, cudaStream_t st,
                                 int64_t* launches, bool first_done = false,
                                 const Correction* follow = nullptr, bool* followed = nullptr)
{
  if (followed) *followed = false;
  std::vector<std::pair<Epi, std::pair<double, double>>> steps;
  if (cs.collapsed) {
    for (int k = first_done ? 1 : 0; k < sweeps; ++k) steps.push_back({Epi::kJacobi, {0.0, 0.0}});
  } else {
    if (!first_done) steps.push_back({Epi::kChebFirst, {0.0, 0.0}});
    for (const auto& c : cs.steps) steps.push_back({Epi::kChebNext, c});
  }
  for (size_t k = 0; k < steps.size(); ++k) {
    EpiArgs ea;
    ea.b = b;
    ea.theta = cs.theta;
    ea.d = d;
    ea.u_in = *cur;
    ea.out = *alt;
    ea.c1 = steps[k].second.first;
    ea.c2 = steps[k].second.second;
    const bool fol = follow && k + 1 == steps.size();
    if (fol) {
      ea.skip_rows = follow->bmask;
      ea.keep_d = false;
    }
    SMG_CUDA(launch_csr_stream(op.a, *cur, steps[k].first, ea, st));
    ++*launches;
    if (fol) {
      FollowArgs fa;
      fa.epi = (int)steps[k].first;
      fa.ring = follow->ringA;
      fa.x = *cur;
      fa.u_in = *cur;
      fa.b = b;
      fa.d = d;
      fa.inv_diag = op.a.inv_diag;
      fa.theta = cs.theta;
      fa.c1 = ea.c1;
      fa.c2 = ea.c2;
      fa.out = *alt;
      SMG_CUDA(launch_patch_follow(*follow, fa, st));
      ++*launches;
      if (followed) *followed = true;
    }
    std::swap(*cur, *alt);
  }
  return SMG_OK;
}

static int enqueue_local_correct(const Correction& c, const double* b, double* u, cudaStream_t st,
                                 int64_t* launches)
{
  if (c.n_regions == 0) return SMG_OK;
  if (c.coupled) {
    // all residuals must see the pre-correction u: separate gather pass
    SMG_CUDA(launch_patch_residual(c.op->a, c, b, u, st));
    SMG_CUDA(launch_patch_solve(c, b, u, u, nullptr, false, st));
    *launches += 2;
  } else {
    SMG_CUDA(launch_patch_solve(c, b, u, u, nullptr, true, st));
    *launches += 1;
  }
  return SMG_OK;
}

// ---------------------------------------------------------------------------
// scratch for free-standing reductions
struct DotScratch {
  double* partials = nullptr;
  unsigned int* counter = nullptr;
  double* result = nullptr;
  double* host = nullptr;  // pinned
  std::vector<void*> allocs;
  int64_t bytes = 0;
  int init()
  {
    if (partials) return SMG_OK;
    SMG_TRY(dev_alloc(allocs, bytes, kDotBlocks, &partials));
    SMG_TRY(dev_alloc(allocs, bytes, 1, &counter));
    SMG_TRY(dev_alloc(allocs, bytes, 1, &result));
    SMG_CUDA(cudaMemset(counter, 0, sizeof(unsigned int)));
    SMG_CUDA(cudaMallocHost(&host, sizeof(double)));
    return SMG_OK;
  }
  void release()
  {
    free_all(allocs);
    if (host) cudaFreeHost(host);
    host = nullptr;
    partials = nullptr;
  }
  int dot(int64_t n, const double* x, const double* y, cudaStream_t st, double* out)
  {
    SMG_TRY(init());
    SMG_CUDA(launch_dot(n, x, y, partials, counter, result, st));
    SMG_CUDA(cudaMemcpyAsync(host, result, sizeof(double), cudaMemcpyDeviceToHost, st));
    SMG_CUDA(cudaStreamSynchronize(st));
    *out = *host;
    return SMG_OK;
  }
};

// ---------------------------------------------------------------------------
struct HLevel {
  const Operator* a = nullptr;
  const Operator* p = nullptr;
  const Correction* lc = nullptr;
  int kind = kChebyshev;
  int sweeps = 1;
  double lambda_max = 0, frac = 0.1;
  ChebScalars cs;
  int64_t n = 0;
  double* b = nullptr;   // levels >= 1
  double* u = nullptr;   // levels >= 1
  double* t = nullptr;   // ping-pong partner
  double* d = nullptr;   // Chebyshev direction
  double* r = nullptr;   // residual
  RingRows ringP;        // P's rows on the correction rings (follow-mode prolong-add)
  bool has_ringP = false;
  // locality renumbering (renumber_level): perm[old] = new, inv[new] = old
  bool renum = false;
  std::vector<int32_t> perm_h;
  int32_t* perm = nullptr;
  int32_t* inv = nullptr;
};

struct Hierarchy {
  std::vector<HLevel> lv;
  int64_t n_coarse = 0;
  SymTiles coarse;                    // A_L^{-1}, lower-triangle tiles
  int coarse_refine = 0;
  double* coarse_r = nullptr;
  double* coarse_x = nullptr;
  std::vector<void*> allocs;
  int64_t bytes = 0;
  bool use_graphs = true;
  bool fuse_zero_guess = true;
  bool lc_overlap = false;  // measured slower: opt-in
  bool lc_follow = true;    // corrections overlapped with their producer kernel
                            // (only where rings were built: opt-in, see build_ring)
  cudaStream_t side = nullptr;       // local corrections overlapping interior sweeps
  cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
  std::map<std::pair<const void*, void*>, cudaGraphExec_t> graphs;
  cudaStream_t capture_stream = nullptr;
  int64_t launches = 0;
  double* stage_b = nullptr;  // device copies for the host-buffer path
  double* stage_u = nullptr;
  double* stage_b2 = nullptr;  // second staging slot (pipelined host path)
  double* stage_u2 = nullptr;
  cudaStream_t copy_in = nullptr, copy_out = nullptr;
  cudaEvent_t pipe_ev[6] = {};
  DotScratch dots;
  // concurrent vcycle calls on one shared hierarchy are safe:
  // every entry point that touches the per-level scratch, the staging
  // buffers, the dot scratch or the graph cache holds `mu`, and device work is
  // ordered across callers' streams by `done_ev` (each call waits for the
  // previous call's last kernel before it starts, then records its own).
  std::recursive_mutex mu;
  cudaEvent_t done_ev = nullptr;
  // renamed copies owned by the hierarchy (renumbered levels)
  std::vector<std::unique_ptr<Operator>> own_ops;
  std::vector<std::unique_ptr<Correction>> own_corrs;
  const Operator* a_user = nullptr;   // level 0's operator as the caller passed it
  double* b0r = nullptr;              // level 0 renumbered: b and u in the renamed space
  double* u0r = nullptr;

  ~Hierarchy()
  {
    for (auto& o : own_ops) free_all(o->allocs);
    for (auto& c : own_corrs) free_all(c->allocs);
    if (done_ev) cudaEventDestroy(done_ev);
    for (auto& kv : graphs) cudaGraphExecDestroy(kv.second);
    if (capture_stream) cudaStreamDestroy(capture_stream);
    if (side) cudaStreamDestroy(side);
    if (fork_ev) cudaEventDestroy(fork_ev);
    if (join_ev) cudaEventDestroy(join_ev);
    if (copy_in) cudaStreamDestroy(copy_in);
    if (copy_out) cudaStreamDestroy(copy_out);
    for (cudaEvent_t e : pipe_ev)
      if (e) cudaEventDestroy(e);
    dots.release();
    free_all(allocs);
  }
};

// One combined smoothing step (smoothers.py:240-269: LC, k global sweeps, LC).
// With a halo split the first local correction runs on a side stream
// concurrently with the interior rows of sweep 1 (rows with no column in any
// patch, so they neither read nor write what the correction changes); the halo
// rows of sweep 1 follow once both finished.  Symmetrically the last sweep's
// halo rows run first, then the second correction overlaps its interior rows.
// Every row is computed by exactly the arithmetic of the unsplit sweep, so the
// result is bit-identical.
// lc1_done: the first correction already ran, fused with the prolong-add.
static int enqueue_smooth(Hierarchy& h, HLevel& L, const double* b, double** cur, double** alt,
                          cudaStream_t st, int64_t* launches, bool first_done = false,
                          bool lc1_done = false)
{
  const bool active = L.lc && L.lc->n_regions > 0;
  if (!active || first_done || !h.lc_overlap || !L.lc->has_halo) {
    if (active && !lc1_done) SMG_TRY(enqueue_local_correct(*L.lc, b, *cur, st, launches));
    const bool follow = active && h.lc_follow && L.lc->has_ring;
    bool followed = false;
    SMG_TRY(enqueue_global_smooth(*L.a, b, cur, alt, L.d, L.sweeps, L.cs, st, launches,
                                  first_done, follow ? L.lc : nullptr, &followed));
    if (active && !followed) SMG_TRY(enqueue_local_correct(*L.lc, b, *cur, st, launches));
    return SMG_OK;
  }
  const Correction& lc = *L.lc;
  if (!h.side) {
    SMG_CUDA(cudaStreamCreateWithFlags(&h.side, cudaStreamNonBlocking));
    SMG_CUDA(cudaEventCreateWithFlags(&h.fork_ev, cudaEventDisableTiming));
    SMG_CUDA(cudaEventCreateWithFlags(&h.join_ev, cudaEventDisableTiming));
  }
  struct Step {
    Epi e;
    double c1, c2;
  };
  std::vector<Step> steps;
  if (L.cs.collapsed) {
    for (int k = 0; k < L.sweeps; ++k) steps.push_back({Epi::kJacobi, 0.0, 0.0});
  } else {
    steps.push_back({Epi::kChebFirst, 0.0, 0.0});
    for (const auto& c : L.cs.steps) steps.push_back({Epi::kChebNext, c.first, c.second});
  }
  enum Part { kAll, kInterior, kHalo };
  auto sweep = [&](const Step& s, Part part) -> int {
    EpiArgs ea;
    ea.b = b;
    ea.theta = L.cs.theta;
    ea.d = L.d;
    ea.u_in = *cur;
    ea.out = *alt;
    ea.c1 = s.c1;
    ea.c2 = s.c2;
    if (part == kInterior) ea.skip_rows = lc.halo_mask;
    SMG_CUDA(launch_csr_stream(part == kHalo ? lc.halo : L.a->a, *cur, s.e, ea, st));
    ++*launches;
    return SMG_OK;
  };
  auto fork = [&]() -> int {
    SMG_CUDA(cudaEventRecord(h.fork_ev, st));
    SMG_CUDA(cudaStreamWaitEvent(h.side, h.fork_ev, 0));
    return SMG_OK;
  };
  auto join = [&]() -> int {
    SMG_CUDA(cudaEventRecord(h.join_ev, h.side));
    SMG_CUDA(cudaStreamWaitEvent(st, h.join_ev, 0));
    return SMG_OK;
  };
  const size_t k = steps.size();
  // LC1 (in place on cur) || interior rows of sweep 1; then its halo rows
  SMG_TRY(fork());
  SMG_TRY(enqueue_local_correct(lc, b, *cur, h.side, launches));
  SMG_TRY(sweep(steps[0], kInterior));
  SMG_TRY(join());
  SMG_TRY(sweep(steps[0], kHalo));
  std::swap(*cur, *alt);
  for (size_t i = 1; i + 1 < k; ++i) {
    SMG_TRY(sweep(steps[i], kAll));
    std::swap(*cur, *alt);
  }
  if (k >= 2) {
    // halo rows of the last sweep, then LC2 on them || the interior rows
    SMG_TRY(sweep(steps[k - 1], kHalo));
    SMG_TRY(fork());
    SMG_TRY(enqueue_local_correct(lc, b, *alt, h.side, launches));
    SMG_TRY(sweep(steps[k - 1], kInterior));
    SMG_TRY(join());
    std::swap(*cur, *alt);
  } else {
    SMG_TRY(enqueue_local_correct(lc, b, *cur, st, launches));
  }
  return SMG_OK;
}

// mg.py:127-151
static int enqueue_vcycle(Hierarchy& h, const double* b0, double* u0, cudaStream_t st,
                          int64_t* launches)
{
  const int nl = (int)h.lv.size();
  std::vector<double*> cur(nl), alt(nl);
  std::vector<const double*> bl(nl);
  bl[0] = b0;
  cur[0] = u0;
  alt[0] = h.lv[0].t;
  for (int l = 1; l < nl; ++l) {
    bl[l] = h.lv[l].b;
    cur[l] = h.lv[l].u;
    alt[l] = h.lv[l].t;
  }
  if (h.lv[0].renum) {
    // the caller's b and u into level 0's renamed index space
    SMG_CUDA(launch_gather(h.lv[0].inv, h.lv[0].n, b0, h.b0r, st));
    SMG_CUDA(launch_gather(h.lv[0].inv, h.lv[0].n, u0, h.u0r, st));
    bl[0] = h.b0r;
    cur[0] = h.u0r;
    *launches += 2;
  }
  std::vector<char> first_done(nl, 0);
  for (int l = 0; l < nl - 1; ++l) {
    HLevel& L = h.lv[l];
    SMG_TRY(enqueue_smooth(h, L, bl[l], &cur[l], &alt[l], st, launches, first_done[l] != 0));
    EpiArgs ea;
    ea.b = bl[l];
    ea.out = L.r;
    SMG_CUDA(launch_csr_stream(L.a->a, cur[l], Epi::kResidual, ea, st));
    HLevel& N = h.lv[l + 1];
    const bool next_coarsest = (l + 1 == nl - 1);
    const bool next_lc = N.lc && N.lc->n_regions > 0;
    if (!next_coarsest && !next_lc && N.a->all_finite && h.fuse_zero_guess) {
      // restriction fused with the next level's first sweep from u = 0
      EpiArgs er;
      er.out = alt[l + 1];
      er.b_out = N.b;
      er.inv_diag = N.a->inv_diag;
      er.theta = N.cs.theta;
      er.d = N.cs.collapsed ? nullptr : N.d;
      SMG_CUDA(launch_csr_stream(L.p->t, L.r, Epi::kRestrictFirst, er, st));
      std::swap(cur[l + 1], alt[l + 1]);
      first_done[l + 1] = 1;
    } else {
      EpiArgs er;
      er.out = N.b;
      SMG_CUDA(launch_csr_stream(L.p->t, L.r, Epi::kSpmv, er, st));
      if (!next_coarsest)
        SMG_CUDA(cudaMemsetAsync(cur[l + 1], 0, sizeof(double) * (size_t)N.n, st));
    }
    *launches += 2;
  }
  // coarse solve
  {
    HLevel& C = h.lv[nl - 1];
    SMG_CUDA(launch_sym_apply(h.coarse, bl[nl - 1], cur[nl - 1], false, st));
    *launches += sym_apply_launches();
    if (h.coarse_refine) {
      EpiArgs ea;
      ea.b = bl[nl - 1];
      ea.out = h.coarse_r;
      SMG_CUDA(launch_csr_stream(C.a->a, cur[nl - 1], Epi::kResidual, ea, st));
      SMG_CUDA(launch_sym_apply(h.coarse, h.coarse_r, cur[nl - 1], true, st));
      *launches += 1 + sym_apply_launches();
    }
  }
  for (int l = nl - 2; l >= 0; --l) {
    HLevel& L = h.lv[l];
    const bool follow = L.lc && L.lc->n_regions > 0 && L.lc->has_ring && L.has_ringP &&
                        h.lc_follow && !h.lc_overlap;
    EpiArgs ea;
    ea.out = cur[l];
    if (follow) {
      // prolong-add out of place, skipping the patch dofs; the post-smoother's
      // first correction recomputes it on its rings and runs concurrently
      ea.u_in = cur[l];
      ea.out = alt[l];
      ea.skip_rows = L.lc->bmask;
    }
    SMG_CUDA(launch_csr_stream(L.p->a, cur[l + 1], Epi::kAddTo, ea, st));
    ++*launches;
    if (follow) {
      FollowArgs fa;
      fa.epi = (int)Epi::kAddTo;
      fa.ring = L.ringP;
      fa.x = cur[l + 1];
      fa.u_in = cur[l];
      fa.b = bl[l];
      fa.out = alt[l];
      SMG_CUDA(launch_patch_follow(*L.lc, fa, st));
      ++*launches;
      std::swap(cur[l], alt[l]);
    }
    SMG_TRY(enqueue_smooth(h, L, bl[l], &cur[l], &alt[l], st, launches, false, follow));
  }
  if (h.lv[0].renum) {
    SMG_CUDA(launch_gather(h.lv[0].perm, h.lv[0].n, cur[0], u0, st));   // back to the caller's order
    ++*launches;
  } else if (cur[0] != u0) {
    SMG_CUDA(cudaMemcpyAsync(u0, cur[0], sizeof(double) * (size_t)h.lv[0].n,
                             cudaMemcpyDeviceToDevice, st));
  }
  return SMG_OK;
}

// Cross-stream ordering of the shared scratch (see Hierarchy::mu): wait for
// the previous caller's work, run, record.  Skipped while the caller's stream
// is being captured (an event recorded outside a capture cannot be waited on
// inside it; a captured graph is ordered by whoever launches it).
struct ScratchOrder {
  Hierarchy* hp;
  cudaStream_t st;
  bool active = false;
  int begin()
  {
    if (!hp) return SMG_OK;
    Hierarchy& h = *hp;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    SMG_CUDA(cudaStreamIsCapturing(st, &cs));
    active = cs == cudaStreamCaptureStatusNone;
    if (!active) return SMG_OK;
    if (!h.done_ev) {
      SMG_CUDA(cudaEventCreateWithFlags(&h.done_ev, cudaEventDisableTiming));
      return SMG_OK;   // nothing recorded yet
    }
    SMG_CUDA(cudaStreamWaitEvent(st, h.done_ev, 0));
    return SMG_OK;
  }
  int end()
  {
    if (hp && active) SMG_CUDA(cudaEventRecord(hp->done_ev, st));
    return SMG_OK;
  }
};

static int run_vcycle(Hierarchy& h, const double* b, double* u, cudaStream_t st)
{
  if (!h.use_graphs) {
    int64_t n = 0;
    SMG_TRY(enqueue_vcycle(h, b, u, st, &n));
    h.launches = n;
    return SMG_OK;
  }
  auto key = std::make_pair((const void*)b, (void*)u);
  auto it = h.graphs.find(key);
  if (it == h.graphs.end()) {
    if (!h.capture_stream)
      SMG_CUDA(cudaStreamCreateWithFlags(&h.capture_stream, cudaStreamNonBlocking));
    SMG_CUDA(cudaStreamBeginCapture(h.capture_stream, cudaStreamCaptureModeThreadLocal));
    int64_t n = 0;
    int rc = enqueue_vcycle(h, b, u, h.capture_stream, &n);
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaStreamEndCapture(h.capture_stream, &g);
    if (rc != SMG_OK) {
      if (g) cudaGraphDestroy(g);
      return rc;
    }
    SMG_CUDA(e);
    cudaGraphExec_t ex = nullptr;
    e = cudaGraphInstantiate(&ex, g, 0);
    cudaGraphDestroy(g);
    SMG_CUDA(e);
    if (h.graphs.size() > 64) {  // bound the cache
      for (auto& kv : h.graphs) cudaGraphExecDestroy(kv.second);
      h.graphs.clear();
    }
    it = h.graphs.emplace(key, ex).first;
    h.launches = n;
  }
  SMG_CUDA(cudaGraphLaunch(it->second, st));
  return SMG_OK;
}

static std::mutex g_scratch_mu;
static DotScratch g_dots;

}  // namespace smg

using namespace smg;

struct smg_operator {
  Operator o;
};
struct smg_correction {
  Correction c;
};
struct smg_hierarchy {
  Hierarchy h;
};
struct smg_csr {
  DevCsrOwned m;
  ~smg_csr() { m.release(); }
};

static cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

extern "C" {

int smg_abi_version(void) { return SMG_ABI_VERSION; }

const char* smg_last_error(void) { return g_last_error.c_str(); }

int smg_device_info(int* sm_count, int64_t* l2_bytes, int* cc_major, int* cc_minor)
{
  int dev = 0;
  SMG_CUDA(cudaGetDevice(&dev));
  cudaDeviceProp p;
  SMG_CUDA(cudaGetDeviceProperties(&p, dev));
  if (sm_count) *sm_count = p.multiProcessorCount;
  if (l2_bytes) *l2_bytes = p.l2CacheSize;
  if (cc_major) *cc_major = p.major;
  if (cc_minor) *cc_minor = p.minor;
  return SMG_OK;
}

int smg_operator_create(int64_t nrows, int64_t ncols, const int64_t* rowptr, const int64_t* col,
                        const double* val, int with_transpose, smg_operator** out)
{
  if (!out) return fail("out is NULL");
  *out = nullptr;
  if (nrows < 0 || ncols < 0) return fail("negative dimensions");
  if (nrows >= INT32_MAX || ncols >= INT32_MAX) return fail("dimensions exceed int32 indexing");
  if (!rowptr) return fail("row_offsets is NULL");
  if (rowptr[0] != 0) return fail("row_offsets must be monotone from 0 to nnz");
  for (int64_t i = 0; i < nrows; ++i)
    if (rowptr[i + 1] < rowptr[i]) return fail("row_offsets must be monotone from 0 to nnz");
  const int64_t nnz = rowptr[nrows];
  for (int64_t i = 0; i < nrows; ++i) {
    for (int64_t j = rowptr[i]; j < rowptr[i + 1]; ++j) {
      if (col[j] < 0 || col[j] >= ncols) return fail("column index out of range");
      if (j > rowptr[i] && col[j] <= col[j - 1])
        return fail("column indices must be strictly increasing within rows");
    }
  }
  configure_l2_persist();
  auto* op = new smg_operator();
  Operator& o = op->o;
  int rc = build_devcsr(o.allocs, o.device_bytes, nrows, ncols, rowptr, col, val, &o.a);
  if (rc != SMG_OK) {
    free_all(o.allocs);
    delete op;
    return rc;
  }
  // first zero / missing diagonal (smoothers.py:111-114 via a.diagonal())
  o.first_zero_diag = -1;
  const int64_t nd = std::min(nrows, ncols);
  std::vector<double> diag((size_t)nd, 0.0);
  for (int64_t i = 0; i < nd; ++i) {
    double dv = 0.0;
    const int64_t* b = col + rowptr[i];
    const int64_t* e = col + rowptr[i + 1];
    const int64_t* f = std::lower_bound(b, e, i);
    if (f != e && *f == i) dv = val[rowptr[i] + (f - b)];
    diag[(size_t)i] = dv;
    if (dv == 0.0 && o.first_zero_diag < 0) o.first_zero_diag = i;
  }
  for (int64_t j = 0; j < nnz && o.all_finite; ++j)
    if (!std::isfinite(val[j])) o.all_finite = false;
  if (nrows == ncols && nd > 0) {
    // inv_diag = 1.0 / diag: the same IEEE division numpy performs
    // (smoothers.py:115), so the epilogue multiplies by identical values
    std::vector<double> inv((size_t)nd);
    for (int64_t i = 0; i < nd; ++i) inv[(size_t)i] = 1.0 / diag[(size_t)i];
    double* dd = nullptr;
    double* di = nullptr;
    rc = dev_upload(o.allocs, o.device_bytes, diag.data(), diag.size(), &dd);
    if (rc == SMG_OK) rc = dev_upload(o.allocs, o.device_bytes, inv.data(), inv.size(), &di);
    if (rc != SMG_OK) {
      free_all(o.allocs);
      delete op;
      return rc;
    }
    o.diag = dd;
    o.inv_diag = di;
    o.a.inv_diag = di;
  }
  if (with_transpose) {
    // CSR(A^T) with ascending source rows in each row (counting sort is stable)
    std::vector<int64_t> tptr((size_t)ncols + 1, 0);
    for (int64_t j = 0; j < nnz; ++j) ++tptr[(size_t)col[j] + 1];
    for (int64_t c = 0; c < ncols; ++c) tptr[(size_t)c + 1] += tptr[(size_t)c];
    std::vector<int64_t> fill(tptr.begin(), tptr.end() - 1);
    std::vector<int64_t> tcol((size_t)nnz);
    std::vector<double> tval((size_t)nnz);
    for (int64_t i = 0; i < nrows; ++i)
      for (int64_t j = rowptr[i]; j < rowptr[i + 1]; ++j) {
        const int64_t pos = fill[(size_t)col[j]]++;
        tcol[(size_t)pos] = i;
        tval[(size_t)pos] = val[j];
      }
    rc = build_devcsr(o.allocs, o.device_bytes, ncols, nrows, tptr.data(), tcol.data(),
                      tval.data(), &o.t);
    if (rc != SMG_OK) {
      free_all(o.allocs);
      delete op;
      return rc;
    }
    o.has_t = true;
  }
  *out = op;
  return SMG_OK;
}

int smg_operator_destroy(smg_operator* op)
{
  if (!op) return SMG_OK;
  free_all(op->o.allocs);
  delete op;
  return SMG_OK;
}

int smg_operator_info(const smg_operator* op, int64_t* nrows, int64_t* ncols, int64_t* nnz,
                      int64_t* first_zero_diag, int64_t* device_bytes)
{
  if (!op) return fail("operator is NULL");
  if (nrows) *nrows = op->o.a.nrows;
  if (ncols) *ncols = op->o.a.ncols;
  if (nnz) *nnz = op->o.a.nnz;
  if (first_zero_diag) *first_zero_diag = op->o.first_zero_diag;
  if (device_bytes) *device_bytes = op->o.device_bytes;
  return SMG_OK;
}

static int relayout(Operator& o, DevCsr& m, int layout, int unroll)
{
  const int64_t n = m.nrows, nnz = m.nnz;
  std::vector<int64_t> rp((size_t)n + 1);
  std::vector<int32_t> c32((size_t)std::max<int64_t>(nnz, 1));
  std::vector<int64_t> c64((size_t)std::max<int64_t>(nnz, 1));
  std::vector<double> v((size_t)std::max<int64_t>(nnz, 1));
  SMG_CUDA(cudaMemcpy(rp.data(), m.rowptr, sizeof(int64_t) * (size_t)(n + 1), cudaMemcpyDeviceToHost));
  if (nnz > 0) {
    SMG_CUDA(cudaMemcpy(c32.data(), m.col, sizeof(int32_t) * (size_t)nnz, cudaMemcpyDeviceToHost));
    SMG_CUDA(cudaMemcpy(v.data(), m.val, sizeof(double) * (size_t)nnz, cudaMemcpyDeviceToHost));
  }
  for (int64_t j = 0; j < nnz; ++j) c64[(size_t)j] = c32[(size_t)j];
  DevCsr d;
  SMG_TRY(build_devcsr(o.allocs, o.device_bytes, n, m.ncols, rp.data(), c64.data(), v.data(), &d,
                       layout, unroll));
  d.inv_diag = m.inv_diag;
  d.row_map = m.row_map;
  m = d;
  return SMG_OK;
}

int smg_operator_set_layout(smg_operator* op, int layout, int unroll)
{
  if (!op) return fail("operator is NULL");
  if (layout < SMG_LAYOUT_TILES || layout > SMG_LAYOUT_TILES_STAGED) return fail("unknown layout");
  SMG_CUDA(cudaDeviceSynchronize());
  SMG_TRY(relayout(op->o, op->o.a, layout, unroll));
  if (op->o.has_t) SMG_TRY(relayout(op->o, op->o.t, layout, unroll));
  return SMG_OK;
}

int smg_operator_layout(const smg_operator* op, int* layout, int* unroll)
{
  if (!op) return fail("operator is NULL");
  const DevCsr& m = op->o.a;
  if (layout)
    *layout = m.sell ? (m.sell_lanes == 4 ? SMG_LAYOUT_SELL4
                                          : (m.sell_delta ? SMG_LAYOUT_SELL_D16 : SMG_LAYOUT_SELL))
                     : (m.stage_cap > 0 ? SMG_LAYOUT_TILES_STAGED
                                        : (m.fixed ? SMG_LAYOUT_TILES_FIXED : SMG_LAYOUT_TILES));
  if (unroll)
    *unroll = m.sell ? m.sell_unroll
                     : (m.stage_cap > 0 ? (m.stage_cap + kTileNnz - 1) / kTileNnz
                                        : (m.multichunk ? kMaxTileChunks : 1));
  return SMG_OK;
}

int smg_spmv(const smg_operator* a, const double* x, double* y, void* stream)
{
  if (!a) return fail("operator is NULL");
  EpiArgs ea;
  ea.out = y;
  SMG_CUDA(launch_csr_stream(a->o.a, x, Epi::kSpmv, ea, as_stream(stream)));
  return SMG_OK;
}

int smg_residual(const smg_operator* a, const double* b, const double* u, double* r, void* stream)
{
  if (!a) return fail("operator is NULL");
  EpiArgs ea;
  ea.b = b;
  ea.out = r;
  SMG_CUDA(launch_csr_stream(a->o.a, u, Epi::kResidual, ea, as_stream(stream)));
  return SMG_OK;
}

int smg_spmv_transpose(const smg_operator* p, const double* r, double* y, void* stream)
{
  if (!p) return fail("operator is NULL");
  if (!p->o.has_t) return fail("operator was created without its transpose");
  EpiArgs ea;
  ea.out = y;
  SMG_CUDA(launch_csr_stream(p->o.t, r, Epi::kSpmv, ea, as_stream(stream)));
  return SMG_OK;
}

static int spgemm_checked(const DevCsr& x, const DevCsr& y, DevCsrOwned* out, cudaStream_t st)
{
  const cudaError_t e = spgemm_device(x, y, out, st);
  if (e != cudaSuccess) {
    out->release();
    return check_cuda(e, "spgemm_device");
  }
  return SMG_OK;
}

int smg_matmul(const smg_operator* x, const smg_operator* y, smg_csr** out, void* stream)
{
  if (!out) return fail("out is NULL");
  *out = nullptr;
  if (!x || !y) return fail("operator is NULL");
  if (x->o.a.ncols != y->o.a.nrows) {
    set_error("dimension mismatch: " + std::to_string(x->o.a.nrows) + "x" +
              std::to_string(x->o.a.ncols) + " @ " + std::to_string(y->o.a.nrows) + "x" +
              std::to_string(y->o.a.ncols));
    return SMG_ERR_DIMENSION;
  }
  auto c = std::make_unique<smg_csr>();
  SMG_TRY(spgemm_checked(x->o.a, y->o.a, &c->m, as_stream(stream)));
  *out = c.release();
  return SMG_OK;
}

int smg_galerkin(const smg_operator* a, const smg_operator* p, smg_csr** out, void* stream)
{
  if (!out) return fail("out is NULL");
  *out = nullptr;
  if (!a || !p) return fail("operator is NULL");
  if (a->o.a.ncols != p->o.a.nrows || a->o.a.nrows != p->o.a.nrows) {
    set_error("dimension mismatch: a is " + std::to_string(a->o.a.nrows) + "x" +
              std::to_string(a->o.a.ncols) + ", p is " + std::to_string(p->o.a.nrows) + "x" +
              std::to_string(p->o.a.ncols));
    return SMG_ERR_DIMENSION;
  }
  if (!p->o.has_t) return fail("prolongation was created without its transpose");
  const cudaStream_t st = as_stream(stream);
  DevCsrOwned m;  // A P
  SMG_TRY(spgemm_checked(a->o.a, p->o.a, &m, st));
  auto c = std::make_unique<smg_csr>();
  const int rc = spgemm_checked(p->o.t, m.view(), &c->m, st);  // CSR(P^T) (A P)
  m.release();
  SMG_TRY(rc);
  *out = c.release();
  return SMG_OK;
}

int smg_prolongation_build(int dim, int degree, int64_t n_points, const double* points,
                           int64_t n_cells, const double* v0, const double* inv_jac,
                           const int64_t* cell_nodes, int64_t n_coarse_nodes, int nb,
                           const double* lo, const double* hi, const double* scale,
                           const int64_t* bin_ptr, const int64_t* bin_cells, double tol,
                           double drop_tol, smg_csr** out, int64_t* failed_point, void* stream)
{
  if (!out) return fail("out is NULL");
  *out = nullptr;
  if (failed_point) *failed_point = -1;
  if (dim != 2 && dim != 3) return fail("dim must be 2 or 3");
  if (degree != 1 && degree != 2) return fail("element degree must be 1 or 2");
  if (n_points < 0 || n_cells <= 0 || nb <= 0 || n_coarse_nodes <= 0)
    return fail("empty coarse mesh or negative sizes");
  if (n_points >= INT32_MAX || n_coarse_nodes >= INT32_MAX)
    return fail("dimensions exceed int32 indexing");
  if ((n_points > 0 && !points) || !v0 || !inv_jac || !cell_nodes || !lo || !hi || !scale ||
      !bin_ptr || !bin_cells)
    return fail("NULL input array");
  const int npc = degree == 1 ? dim + 1 : (dim + 1) * (dim + 2) / 2;
  int64_t nbins = 1;
  for (int d = 0; d < dim; ++d) nbins *= nb;
  const int64_t nbc = bin_ptr[nbins];
  for (int64_t k = 0; k < n_cells * npc; ++k)
    if (cell_nodes[k] < 0 || cell_nodes[k] >= n_coarse_nodes) return fail("cell node out of range");
  for (int64_t k = 0; k < nbc; ++k)
    if (bin_cells[k] < 0 || bin_cells[k] >= n_cells) return fail("bin cell out of range");
  std::vector<void*> tmp;
  int64_t bytes = 0;
  LocateArgs a;
  a.n_points = n_points;
  a.n_cells = n_cells;
  a.n_coarse = n_coarse_nodes;
  a.nb = nb;
  for (int d = 0; d < dim; ++d) {
    a.lo[d] = lo[d];
    a.hi[d] = hi[d];
    a.scale[d] = scale[d];
  }
  a.tol = tol;
  a.drop_tol = drop_tol;
  double *dp = nullptr, *dv0 = nullptr, *dinv = nullptr;
  int64_t *dcn = nullptr, *dbp = nullptr, *dbc = nullptr;
  int rc = dev_upload(tmp, bytes, points, (size_t)(n_points * dim), &dp);
  if (rc == SMG_OK) rc = dev_upload(tmp, bytes, v0, (size_t)(n_cells * dim), &dv0);
  if (rc == SMG_OK) rc = dev_upload(tmp, bytes, inv_jac, (size_t)(n_cells * dim * dim), &dinv);
  if (rc == SMG_OK) rc = dev_upload(tmp, bytes, cell_nodes, (size_t)(n_cells * npc), &dcn);
  if (rc == SMG_OK) rc = dev_upload(tmp, bytes, bin_ptr, (size_t)(nbins + 1), &dbp);
  if (rc == SMG_OK) rc = dev_upload(tmp, bytes, bin_cells, (size_t)std::max<int64_t>(nbc, 1), &dbc);
  if (rc != SMG_OK) {
    free_all(tmp);
    return rc;
  }
  a.points = dp;
  a.v0 = dv0;
  a.inv_jac = dinv;
  a.cell_nodes = dcn;
  a.bin_ptr = dbp;
  a.bin_cells = dbc;
  auto c = std::make_unique<smg_csr>();
  int64_t bad = -1;
  const cudaError_t e = prolongation_device(a, dim, degree, &c->m, &bad, as_stream(stream));
  free_all(tmp);
  if (e != cudaSuccess) return check_cuda(e, "prolongation_device");
  if (bad >= 0) {
    if (failed_point) *failed_point = bad;
    set_error("point " + std::to_string(bad) + " lies outside the coarse mesh");
    return SMG_ERR_POINT_LOCATION;
  }
  *out = c.release();
  return SMG_OK;
}

int smg_csr_info(const smg_csr* c, int64_t* nrows, int64_t* ncols, int64_t* nnz)
{
  if (!c) return fail("matrix is NULL");
  if (nrows) *nrows = c->m.nrows;
  if (ncols) *ncols = c->m.ncols;
  if (nnz) *nnz = c->m.nnz;
  return SMG_OK;
}

int smg_csr_to_host(const smg_csr* c, int64_t* row_offsets, int64_t* col_indices, double* values)
{
  if (!c) return fail("matrix is NULL");
  const DevCsrOwned& m = c->m;
  if (row_offsets)
    SMG_CUDA(cudaMemcpy(row_offsets, m.rowptr, (size_t)(m.nrows + 1) * sizeof(int64_t),
                        cudaMemcpyDeviceToHost));
  if (col_indices && m.nnz > 0) {
    std::vector<int32_t> tmp((size_t)m.nnz);
    SMG_CUDA(cudaMemcpy(tmp.data(), m.col, (size_t)m.nnz * sizeof(int32_t),
                        cudaMemcpyDeviceToHost));
    for (int64_t k = 0; k < m.nnz; ++k) col_indices[k] = tmp[(size_t)k];
  }
  if (values && m.nnz > 0)
    SMG_CUDA(cudaMemcpy(values, m.val, (size_t)m.nnz * sizeof(double), cudaMemcpyDeviceToHost));
  return SMG_OK;
}

int smg_csr_destroy(smg_csr* c)
{
  delete c;
  return SMG_OK;
}

int smg_prolong_add(const smg_operator* p, const double* uc, double* uf, void* stream)
{
  if (!p) return fail("operator is NULL");
  EpiArgs ea;
  ea.out = uf;
  SMG_CUDA(launch_csr_stream(p->o.a, uc, Epi::kAddTo, ea, as_stream(stream)));
  return SMG_OK;
}

int smg_smoother_step(const smg_operator* a, const double* b, const double* u_in, double* u_out,
                      double* d, int step, double theta, double c1, double c2, void* stream)
{
  if (!a) return fail("operator is NULL");
  if (u_in == u_out) return fail("u_out must not alias u_in");
  if (a->o.first_zero_diag >= 0) {
    set_error("zero diagonal entry in row " + std::to_string(a->o.first_zero_diag));
    return SMG_ERR_ZERO_DIAGONAL;
  }
  EpiArgs ea;
  ea.b = b;
  ea.u_in = u_in;
  ea.out = u_out;
  ea.d = d;
  ea.theta = theta;
  ea.c1 = c1;
  ea.c2 = c2;
  Epi e = step == SMG_STEP_JACOBI ? Epi::kJacobi
          : step == SMG_STEP_CHEB_FIRST ? Epi::kChebFirst
          : step == SMG_STEP_CHEB_NEXT ? Epi::kChebNext : Epi::kSpmv;
  if (e == Epi::kSpmv) return fail("unknown smoother step");
  SMG_CUDA(launch_csr_stream(a->o.a, u_in, e, ea, as_stream(stream)));
  return SMG_OK;
}

static int check_square_diag(const Operator& o)
{
  if (o.a.nrows != o.a.ncols) return fail("smoother needs a square operator");
  if (o.first_zero_diag >= 0) {
    set_error("zero diagonal entry in row " + std::to_string(o.first_zero_diag));
    return SMG_ERR_ZERO_DIAGONAL;
  }
  return SMG_OK;
}

static int smooth_standalone(const Operator& o, const double* b, double* u, const Correction* c,
                             int kind, int sweeps, double lmax, double frac, double* work,
                             cudaStream_t st)
{
  if (kind == SMG_SMOOTHER_SGS) {
    set_error("symmetric Gauss-Seidel is outside the GPU hot path");
    return SMG_ERR_UNSUPPORTED;
  }
  if (kind != SMG_SMOOTHER_CHEBYSHEV) return fail("unknown smoother kind");
  ChebScalars cs;
  SMG_TRY(cheb_scalars(sweeps, lmax, frac, &cs));
  SMG_TRY(check_square_diag(o));
  const int64_t n = o.a.nrows;
  std::vector<void*> tmp;
  int64_t bytes = 0;
  double* w = work;
  const int64_t n_even = (n + 1) & ~int64_t(1);   // keep d 16-byte aligned
  if (!w && n > 0) SMG_TRY(dev_alloc(tmp, bytes, (size_t)(2 * n_even), &w));
  double* cur = u;
  double* alt = w;
  double* d = w ? w + n_even : nullptr;
  int64_t launches = 0;
  int rc = SMG_OK;
  const bool active = c && c->n_regions > 0;
  if (active) rc = enqueue_local_correct(*c, b, cur, st, &launches);
  if (rc == SMG_OK) rc = enqueue_global_smooth(o, b, &cur, &alt, d, sweeps, cs, st, &launches);
  if (rc == SMG_OK && active) rc = enqueue_local_correct(*c, b, cur, st, &launches);
  if (rc == SMG_OK && cur != u && n > 0)
    rc = check_cuda(cudaMemcpyAsync(u, cur, sizeof(double) * (size_t)n, cudaMemcpyDeviceToDevice, st),
                    "copy back");
  if (!tmp.empty()) {
    cudaStreamSynchronize(st);
    free_all(tmp);
  }
  return rc;
}

int smg_chebyshev_smooth(const smg_operator* a, const double* b, double* u, int sweeps,
                         double lambda_max, double frac, double* work, void* stream)
{
  if (!a) return fail("operator is NULL");
  return smooth_standalone(a->o, b, u, nullptr, SMG_SMOOTHER_CHEBYSHEV, sweeps, lambda_max, frac,
                           work, as_stream(stream));
}

// Interior/halo split of A around the patches (for overlapping the local
// corrections with smoother sweeps).  Halo rows: every row with a column in a
// patch, every patch row and every column of a patch row (the correction reads
// u there).  Only worth it while the halo is a minority of the rows.
static int build_halo(const Operator& o, const std::vector<int32_t>& dof32,
                      const std::vector<int32_t>& patch_cols, Correction& c)
{
  const int64_t n = o.a.nrows;
  const char* env = getenv("SMG_LC_SPLIT");
  if ((env && env[0] == '0') || n == 0 || dof32.empty() || !o.a.inv_diag) return SMG_OK;
  std::vector<void*> tmp;
  int64_t tmp_bytes = 0;
  std::vector<uint8_t> inb((size_t)n, 0);
  for (int32_t g : dof32) inb[(size_t)g] = 1;
  uint8_t* d_inb = nullptr;
  uint8_t* d_mask = nullptr;
  int rc = dev_upload(tmp, tmp_bytes, inb.data(), inb.size(), &d_inb);
  if (rc == SMG_OK) rc = dev_alloc(tmp, tmp_bytes, (size_t)n, &d_mask);
  if (rc == SMG_OK) rc = check_cuda(launch_mark_halo(o.a, d_inb, d_mask), "halo mark");
  std::vector<uint8_t> mask((size_t)n, 0);
  if (rc == SMG_OK)
    rc = check_cuda(cudaMemcpy(mask.data(), d_mask, (size_t)n, cudaMemcpyDeviceToHost), "halo D2H");
  free_all(tmp);
  SMG_TRY(rc);
  for (int32_t g : dof32) mask[(size_t)g] = 1;
  for (int32_t j : patch_cols) mask[(size_t)j] = 1;
  std::vector<int32_t> rows;
  for (int64_t i = 0; i < n; ++i)
    if (mask[(size_t)i]) rows.push_back((int32_t)i);
  const int64_t nh = (int64_t)rows.size();
  if (nh == 0 || 2 * nh > n) return SMG_OK;
  uint8_t* mk = nullptr;
  int32_t* drows = nullptr;
  int64_t* dlen = nullptr;
  SMG_TRY(dev_upload(c.allocs, c.device_bytes, mask.data(), mask.size(), &mk));
  SMG_TRY(dev_upload(c.allocs, c.device_bytes, rows.data(), rows.size(), &drows));
  SMG_TRY(dev_alloc(tmp, tmp_bytes, (size_t)nh, &dlen));
  std::vector<int64_t> hrow((size_t)nh + 3, 0);
  rc = check_cuda(launch_patch_row_len(o.a, drows, nh, dlen), "halo row lengths");
  if (rc == SMG_OK)
    rc = check_cuda(cudaMemcpy(hrow.data() + 1, dlen, sizeof(int64_t) * (size_t)nh,
                               cudaMemcpyDeviceToHost), "halo row lengths D2H");
  free_all(tmp);
  SMG_TRY(rc);
  for (int64_t k = 0; k < nh; ++k) hrow[(size_t)k + 1] += hrow[(size_t)k];
  const int64_t hn = hrow[(size_t)nh];
  hrow[(size_t)nh + 1] = hrow[(size_t)nh + 2] = hn;
  std::vector<int32_t> tiles = make_tiles(nh, hrow.data());
  std::vector<int64_t> tnz(tiles.size());
  for (size_t i = 0; i < tiles.size(); ++i) tnz[i] = hrow[(size_t)tiles[i]];
  int64_t* drp = nullptr;
  int32_t* dcol = nullptr;
  double* dval = nullptr;
  int32_t* dtr = nullptr;
  int64_t* dtz = nullptr;
  SMG_TRY(dev_upload(c.allocs, c.device_bytes, hrow.data(), hrow.size(), &drp));
  SMG_TRY(dev_alloc(c.allocs, c.device_bytes, (size_t)hn + 4, &dcol));  // prefetch padding
  SMG_TRY(dev_alloc(c.allocs, c.device_bytes, (size_t)hn + 2, &dval));
  SMG_TRY(dev_upload(c.allocs, c.device_bytes, tiles.data(), tiles.size(), &dtr));
  SMG_TRY(dev_upload(c.allocs, c.device_bytes, tnz.data(), tnz.size(), &dtz));
  SMG_TRY(check_cuda(launch_patch_row_gather(o.a, drows, nh, drp, dcol, dval), "halo gather"));
  SMG_CUDA(cudaDeviceSynchronize());
  DevCsr hm;
  hm.nrows = nh;
  hm.ncols = o.a.ncols;
  hm.nnz = hn;
  hm.rowptr = drp;
  hm.col = dcol;
  hm.val = dval;
  hm.tile_row = dtr;
  hm.tile_nz = dtz;
  hm.inv_diag = o.a.inv_diag;   // indexed by operator row (row_map)
  hm.row_map = drows;
  hm.ntiles = (int32_t)(tiles.size() - 1);
  hm.streaming = o.a.streaming;
  hm.multichunk = long_rows(hn, nh);
  c.halo = hm;
  c.halo_mask = mk;
  c.has_halo = true;
  return SMG_OK;
}

int smg_assemble_poisson(int dim, int degree, int64_t n_vertices, const double* vertices,
                         int64_t n_cells, const int64_t* cells, const int64_t* cell_dofs,
                         int64_t n_dofs, const int64_t* dirichlet_dofs, int64_t n_dirichlet,
                         const double* grad_ref, const double* weights, int n_quad,
                         smg_csr** out, int64_t* bad_cell, void* stream)
{
  if (!out) return fail("out is NULL");
  *out = nullptr;
  if (bad_cell) *bad_cell = -1;
  if (dim != 2 && dim != 3) return fail("dim must be 2 or 3");
  if (degree != 1 && degree != 2) return fail("element degree must be 1 or 2");
  if (n_cells <= 0 || n_vertices <= 0 || n_dofs <= 0 || n_quad <= 0 || n_dirichlet < 0)
    return fail("empty mesh or negative sizes");
  if (n_dofs >= INT32_MAX || (uint64_t)n_dofs > (1ull << 31)) return fail("too many DOFs");
  if (!vertices || !cells || !cell_dofs || !grad_ref || !weights ||
      (n_dirichlet > 0 && !dirichlet_dofs))
    return fail("NULL input array");
  const int npc = degree == 1 ? dim + 1 : (dim + 1) * (dim + 2) / 2;
  for (int64_t k = 0; k < n_cells * (dim + 1); ++k)
    if (cells[k] < 0 || cells[k] >= n_vertices) return fail("cell vertex out of range");
  for (int64_t k = 0; k < n_cells * npc; ++k)
    if (cell_dofs[k] < 0 || cell_dofs[k] >= n_dofs) return fail("cell dof out of range");
  std::vector<uint8_t> mask((size_t)n_dofs, 0);
  for (int64_t k = 0; k < n_dirichlet; ++k) {
    const int64_t d = dirichlet_dofs[k];
    if (d < 0 || d >= n_dofs) return fail("Dirichlet dof out of range");
    if (k > 0 && d <= dirichlet_dofs[k - 1]) return fail("Dirichlet dofs must be sorted and unique");
    mask[(size_t)d] = 1;
  }
  auto c = std::make_unique<smg_csr>();
  int64_t bad = -1;
  const int rc = assemble_poisson_device(dim, degree, n_vertices, vertices, n_cells, cells,
                                         cell_dofs, n_dofs, mask.data(), n_dirichlet,
                                         dirichlet_dofs, grad_ref, weights, n_quad, &c->m, &bad,
                                         as_stream(stream));
  if (bad_cell) *bad_cell = bad;
  SMG_TRY(rc);
  *out = c.release();
  return SMG_OK;
}

int smg_assemble_elements(int64_t n_dofs, int64_t n_cells, int nloc, const int64_t* cell_dofs,
                          const double* local, const int64_t* dirichlet_dofs, int64_t n_dirichlet,
                          smg_csr** out, void* stream)
{
  if (!out) return fail("out is NULL");
  *out = nullptr;
  if (n_dofs <= 0 || n_cells < 0 || nloc <= 0 || n_dirichlet < 0)
    return fail("empty space or negative sizes");
  if (n_dofs >= INT32_MAX) return fail("too many DOFs");
  if (n_cells * (int64_t)nloc * nloc >= (int64_t)UINT32_MAX)
    return fail("too many element entries for one call");
  if ((n_cells > 0 && (!cell_dofs || !local)) || (n_dirichlet > 0 && !dirichlet_dofs))
    return fail("NULL input array");
  for (int64_t k = 0; k < n_cells * nloc; ++k)
    if (cell_dofs[k] < 0 || cell_dofs[k] >= n_dofs) return fail("cell dof out of range");
  std::vector<uint8_t> mask;
  if (n_dirichlet > 0) {
    mask.assign((size_t)n_dofs, 0);
    for (int64_t k = 0; k < n_dirichlet; ++k) {
      const int64_t d = dirichlet_dofs[k];
      if (d < 0 || d >= n_dofs) return fail("Dirichlet dof out of range");
      if (k > 0 && d <= dirichlet_dofs[k - 1]) return fail("Dirichlet dofs must be sorted and unique");
      mask[(size_t)d] = 1;
    }
  }
  auto c = std::make_unique<smg_csr>();
  SMG_TRY(assemble_elements_device(n_dofs, n_cells, nloc, cell_dofs, local,
                                   mask.empty() ? nullptr : mask.data(), &c->m, as_stream(stream)));
  *out = c.release();
  return SMG_OK;
}

static int dense_roundtrip(int64_t n, const double* in, double* out, bool invert, int64_t* info,
                           void* stream)
{
  if (info) *info = 0;
  if (n < 0) return fail("negative dimension");
  if (n == 0) return SMG_OK;
  if (!in || !out) return fail("NULL matrix");
  const cudaStream_t st = as_stream(stream);
  const size_t bytes = sizeof(double) * (size_t)n * (size_t)n;
  double* d = nullptr;
  SMG_CUDA(cudaMalloc(&d, bytes));
  int rc = check_cuda(cudaMemcpyAsync(d, in, bytes, cudaMemcpyHostToDevice, st), "H2D");
  double asym = 0.0, amax = 0.0;
  int64_t inf = 0;
  if (rc == SMG_OK)
    rc = dense_cholesky_device(n, d, !invert, &asym, &amax, &inf, invert, st);
  if (rc == SMG_OK && !invert && amax != 0.0 && asym > 1e-10 * amax)
    rc = fail("dense_factor expects a symmetric matrix");
  if (rc == SMG_OK && inf != 0) {
    if (info) *info = inf;
    set_error(invert ? "dpotri: the factor is singular (info " + std::to_string(inf) + ")"
                     : "Cholesky failed: leading minor of order " + std::to_string(inf) +
                           " is not positive");
    rc = SMG_ERR_NOT_SPD;
  }
  if (rc == SMG_OK) rc = check_cuda(cudaMemcpy(out, d, bytes, cudaMemcpyDeviceToHost), "D2H");
  cudaFree(d);
  return rc;
}

int smg_dense_cholesky(int64_t n, const double* a, double* c, int64_t* info, void* stream)
{
  return dense_roundtrip(n, a, c, false, info, stream);
}

int smg_cholesky_inverse(int64_t n, const double* c, double* inverse, void* stream)
{
  int64_t info = 0;
  return dense_roundtrip(n, c, inverse, true, &info, stream);
}

int smg_patch_factor(const smg_operator* a, int64_t n_regions, const int64_t* roff,
                     const int64_t* dofs, double* factors, int64_t* failed_region,
                     int64_t* failed_minor, void* stream)
{
  if (failed_region) *failed_region = -1;
  if (failed_minor) *failed_minor = 0;
  if (!a) return fail("operator is NULL");
  const Operator& o = a->o;
  const int64_t n = o.a.nrows;
  if (o.a.nrows != o.a.ncols) return fail("local corrections need a square operator");
  if (n_regions < 0) return fail("negative region count");
  if (n_regions == 0) return SMG_OK;
  if (!roff || !dofs || !factors) return fail("NULL region arrays");
  std::vector<uint8_t> seen((size_t)n, 0);
  const int64_t m = roff[n_regions];
  std::vector<int32_t> pptr((size_t)n_regions + 1), dof32((size_t)m);
  std::vector<int64_t> foff((size_t)n_regions + 1, 0);
  for (int64_t r = 0; r < n_regions; ++r) {
    const int64_t nd = roff[r + 1] - roff[r];
    if (nd <= 0) return fail("region " + std::to_string(r) + " is empty");
    pptr[(size_t)r] = (int32_t)roff[r];
    foff[(size_t)r + 1] = foff[(size_t)r] + nd * nd;
    for (int64_t k = roff[r]; k < roff[r + 1]; ++k) {
      const int64_t g = dofs[k];
      if (g < 0 || g >= n)
        return fail("region " + std::to_string(r) + " has dof indices outside 0.." +
                    std::to_string(n - 1));
      if (k > roff[r] && g <= dofs[k - 1])
        return fail("region " + std::to_string(r) + " dofs must be sorted and unique");
      if (seen[(size_t)g]) return fail("region " + std::to_string(r) + " overlaps a previous region's dofs");
      seen[(size_t)g] = 1;
      dof32[(size_t)k] = (int32_t)g;
    }
  }
  pptr[(size_t)n_regions] = (int32_t)m;
  std::vector<void*> tmp;
  int64_t bytes = 0;
  int32_t *dp = nullptr, *dd = nullptr;
  int64_t *df = nullptr, *dst = nullptr;
  double *dw = nullptr, *dsym = nullptr;
  const cudaStream_t st = as_stream(stream);
  int rc = dev_upload(tmp, bytes, pptr.data(), pptr.size(), &dp);
  if (rc == SMG_OK) rc = dev_upload(tmp, bytes, dof32.data(), dof32.size(), &dd);
  if (rc == SMG_OK) rc = dev_upload(tmp, bytes, foff.data(), foff.size(), &df);
  if (rc == SMG_OK) rc = dev_alloc(tmp, bytes, (size_t)foff.back(), &dw);
  if (rc == SMG_OK) rc = dev_alloc(tmp, bytes, (size_t)n_regions, &dst);
  if (rc == SMG_OK) rc = dev_alloc(tmp, bytes, (size_t)n_regions * 2, &dsym);
  if (rc == SMG_OK)
    rc = check_cuda(cudaMemsetAsync(dst, 0, sizeof(int64_t) * (size_t)n_regions, st), "memset");
  if (rc == SMG_OK)
    rc = check_cuda(launch_patch_factor(o.a, n_regions, dp, dd, df, dw, dst, dsym, st),
                    "patch_factor_kernel");
  std::vector<int64_t> status((size_t)n_regions);
  std::vector<double> sym((size_t)n_regions * 2);
  if (rc == SMG_OK) rc = check_cuda(cudaStreamSynchronize(st), "patch factor");
  if (rc == SMG_OK)
    rc = check_cuda(cudaMemcpy(status.data(), dst, sizeof(int64_t) * status.size(),
                               cudaMemcpyDeviceToHost), "status D2H");
  if (rc == SMG_OK)
    rc = check_cuda(cudaMemcpy(sym.data(), dsym, sizeof(double) * sym.size(),
                               cudaMemcpyDeviceToHost), "sym D2H");
  if (rc == SMG_OK)
    rc = check_cuda(cudaMemcpy(factors, dw, sizeof(double) * (size_t)foff.back(),
                               cudaMemcpyDeviceToHost), "factors D2H");
  free_all(tmp);
  SMG_TRY(rc);
  for (int64_t r = 0; r < n_regions; ++r) {
    const double scale = sym[(size_t)(2 * r + 1)];
    if (scale != 0.0 && sym[(size_t)(2 * r)] > 1e-10 * scale) {
      if (failed_region) *failed_region = r;
      return fail("dense_factor expects a symmetric matrix (region " + std::to_string(r) + ")");
    }
    if (status[(size_t)r] != 0) {
      if (failed_region) *failed_region = r;
      if (failed_minor) *failed_minor = status[(size_t)r];
      set_error("local block " + std::to_string(r) + " (" + std::to_string(roff[r + 1] - roff[r]) +
                " dofs) is not SPD: leading minor of order " + std::to_string(status[(size_t)r]) +
                " is not positive");
      return SMG_ERR_NOT_SPD;
    }
  }
  return SMG_OK;
}

// Gather the rows `rows` (device, m entries) of `a` into a compact CSR copy.
static int gather_rows(std::vector<void*>& allocs, int64_t& bytes, const DevCsr& a,
                       const int32_t* rows, int64_t m, RingRows* out)
{
  std::vector<void*> tmp;
  int64_t tmp_bytes = 0;
  int64_t* dlen = nullptr;
  std::vector<int64_t> rp((size_t)m + 1, 0);
  int rc = dev_alloc(tmp, tmp_bytes, (size_t)std::max<int64_t>(m, 1), &dlen);
  if (rc == SMG_OK) rc = check_cuda(launch_patch_row_len(a, rows, m, dlen), "ring row lengths");
  if (rc == SMG_OK)
    rc = check_cuda(cudaMemcpy(rp.data() + 1, dlen, sizeof(int64_t) * (size_t)m,
                               cudaMemcpyDeviceToHost), "ring row lengths D2H");
  free_all(tmp);
  SMG_TRY(rc);
  for (int64_t k = 0; k < m; ++k) rp[(size_t)k + 1] += rp[(size_t)k];
  int64_t* drp = nullptr;
  int32_t* dcol = nullptr;
  double* dval = nullptr;
  SMG_TRY(dev_upload(allocs, bytes, rp.data(), rp.size(), &drp));
  SMG_TRY(dev_alloc(allocs, bytes, (size_t)rp[(size_t)m] + 1, &dcol));
  SMG_TRY(dev_alloc(allocs, bytes, (size_t)rp[(size_t)m] + 1, &dval));
  SMG_TRY(check_cuda(launch_patch_row_gather(a, rows, m, drp, dcol, dval), "ring row gather"));
  SMG_CUDA(cudaDeviceSynchronize());
  out->rptr = drp;
  out->rcol = dcol;
  out->rval = dval;
  return SMG_OK;
}

// Rings for follow-mode corrections (a correction overlapped with the kernel
// producing the u it corrects): region d's ring is the
// sorted set of columns of its rows (B_d included), plcol maps every gathered
// patch-row entry to the ring position of its column, bpos every patch dof to
// its own ring position.
static int build_ring(const Operator& o, const std::vector<int32_t>& pptr,
                      const std::vector<int32_t>& dof32, const std::vector<int64_t>& prow,
                      const std::vector<int32_t>& hcol, Correction& c)
{
  // opt-in (SMG_LC_FOLLOW=1 when the correction is created): measured slower
  // on C1-C4, profiles/r01/ab_follow/ 
  const char* env = getenv("SMG_LC_FOLLOW");
  if (!(env && env[0] == '1') || !o.a.inv_diag || c.n_regions == 0) return SMG_OK;
  const int64_t nr = c.n_regions;
  std::vector<int32_t> rptr((size_t)nr + 1, 0), rows, plcol(hcol.size()), bpos(dof32.size());
  int32_t rmax = 0;
  for (int64_t r = 0; r < nr; ++r) {
    const int32_t k0 = pptr[(size_t)r], k1 = pptr[(size_t)r + 1];
    std::vector<int32_t> ring(dof32.begin() + k0, dof32.begin() + k1);
    for (int64_t j = prow[(size_t)k0]; j < prow[(size_t)k1]; ++j) ring.push_back(hcol[(size_t)j]);
    std::sort(ring.begin(), ring.end());
    ring.erase(std::unique(ring.begin(), ring.end()), ring.end());
    auto pos = [&](int32_t g) {
      return (int32_t)(std::lower_bound(ring.begin(), ring.end(), g) - ring.begin());
    };
    for (int32_t k = k0; k < k1; ++k) {
      bpos[(size_t)k] = pos(dof32[(size_t)k]);
      for (int64_t j = prow[(size_t)k]; j < prow[(size_t)k + 1]; ++j)
        plcol[(size_t)j] = pos(hcol[(size_t)j]);
    }
    rmax = std::max<int32_t>(rmax, (int32_t)ring.size());
    rows.insert(rows.end(), ring.begin(), ring.end());
    rptr[(size_t)r + 1] = (int32_t)rows.size();
  }
  c.ring_max = rmax;
  c.ring_total = (int64_t)rows.size();
  c.has_ring = true;
  if (!patch_follow_fits(c)) {
    c.has_ring = false;
    return SMG_OK;
  }
  std::vector<uint8_t> mask((size_t)o.a.nrows, 0);
  for (int32_t g : dof32) mask[(size_t)g] = 1;
  int32_t *drp = nullptr, *drows = nullptr, *dpl = nullptr, *dbp = nullptr;
  uint8_t* dmask = nullptr;
  SMG_TRY(dev_upload(c.allocs, c.device_bytes, rptr.data(), rptr.size(), &drp));
  SMG_TRY(dev_upload(c.allocs, c.device_bytes, rows.data(), rows.size(), &drows));
  SMG_TRY(dev_upload(c.allocs, c.device_bytes, plcol.data(), plcol.size(), &dpl));
  SMG_TRY(dev_upload(c.allocs, c.device_bytes, bpos.data(), bpos.size(), &dbp));
  SMG_TRY(dev_upload(c.allocs, c.device_bytes, mask.data(), mask.size(), &dmask));
  c.ring_ptr = drp;
  c.ring_rows = drows;
  c.plcol = dpl;
  c.bpos = dbp;
  c.bmask = dmask;
  return gather_rows(c.allocs, c.device_bytes, o.a, drows, c.ring_total, &c.ringA);
}

// Packed lower triangle (row-major, even length) of (L L^T)^{-1} from the
// reference's factor c (cho_factor layout, nd x nd row-major, lower triangle
// valid): M = L^{-1} by row-oriented forward substitution, then
// A^{-1} = M^T M accumulated row by row of M -- LAPACK dpotri's two steps
// (dtrtri, dlauum) with contiguous inner loops.
static void packed_spd_inverse(int64_t nd, const double* f, double* out, std::vector<double>& m)
{
  m.assign((size_t)(nd * (nd + 1) / 2 + nd), 0.0);
  double* tmp = m.data() + nd * (nd + 1) / 2;
  auto T = [](int64_t i) { return i * (i + 1) / 2; };
  for (int64_t i = 0; i < nd; ++i) {
    // row i of M: M[i][j] = -(sum_{k=j}^{i-1} L[i][k] M[k][j]) / L[i][i], M[i][i] = 1 / L[i][i]
    for (int64_t j = 0; j < i; ++j) tmp[j] = 0.0;
    for (int64_t k = 0; k < i; ++k) {
      const double lik = f[i * nd + k];
      const double* mk = m.data() + T(k);
      for (int64_t j = 0; j <= k; ++j) tmp[j] += lik * mk[j];
    }
    const double inv = 1.0 / f[i * nd + i];
    double* mi = m.data() + T(i);
    for (int64_t j = 0; j < i; ++j) mi[j] = -tmp[j] * inv;
    mi[i] = inv;
  }
  const int64_t len = (nd * (nd + 1) / 2 + 1) & ~int64_t(1);
  for (int64_t q = 0; q < len; ++q) out[q] = 0.0;
  for (int64_t k = 0; k < nd; ++k) {
    // A^{-1}[i][j] += M[k][i] M[k][j] for j <= i <= k
    const double* mk = m.data() + T(k);
    for (int64_t i = 0; i <= k; ++i) {
      const double s = mk[i];
      double* oi = out + T(i);
      for (int64_t j = 0; j <= i; ++j) oi[j] += s * mk[j];
    }
  }
}

int smg_correction_create(const smg_operator* a, int64_t n_regions, const int64_t* roff,
                          const int64_t* dofs, const int64_t* foff, const double* factors,
                          smg_correction** out)
{
  if (!out) return fail("out is NULL");
  *out = nullptr;
  if (!a) return fail("operator is NULL");
  const Operator& o = a->o;
  const int64_t n = o.a.nrows;
  if (n_regions < 0) return fail("negative region count");
  if (n_regions > 0 && (!roff || !dofs || !foff || !factors)) return fail("NULL region arrays");
  std::vector<int32_t> owner((size_t)n, -1);
  const int64_t m = n_regions > 0 ? roff[n_regions] : 0;
  std::vector<int32_t> pptr((size_t)n_regions + 1);
  std::vector<int32_t> dof32((size_t)m);
  std::vector<int64_t> poff((size_t)n_regions + 1, 0);
  int32_t max_dofs = 0;
  for (int64_t r = 0; r < n_regions; ++r)
    max_dofs = std::max<int32_t>(max_dofs, (int32_t)(roff[r + 1] - roff[r]));
  // SMG_PATCH_SYM=0: keep the factor (panel substitution) for the larger regions
  const char* sym_env = getenv("SMG_PATCH_SYM");
  const bool sym = !(sym_env && sym_env[0] == '0') && max_dofs <= kPatchSymMaxDofs;
  for (int64_t r = 0; r < n_regions; ++r) {
    const int64_t nd = roff[r + 1] - roff[r];
    if (nd <= 0) return fail("region " + std::to_string(r) + " is empty");
    pptr[(size_t)r] = (int32_t)roff[r];
    // slot = [packed L, even length][inverted 32x32 diagonal blocks]; 16-byte
    // aligned and even-length so one bulk copy stages the whole slot
    poff[(size_t)r + 1] = poff[(size_t)r] + patch_slot_doubles(nd, max_dofs, sym);
    for (int64_t k = roff[r]; k < roff[r + 1]; ++k) {
      const int64_t g = dofs[k];
      if (g < 0 || g >= n)
        return fail("region " + std::to_string(r) + " has dof indices outside 0.." +
                    std::to_string(n - 1));
      if (k > roff[r] && g <= dofs[k - 1])
        return fail("region " + std::to_string(r) + " dofs must be sorted and unique");
      if (owner[(size_t)g] >= 0)
        return fail("region " + std::to_string(r) + " overlaps a previous region's dofs");
      owner[(size_t)g] = (int32_t)r;
      dof32[(size_t)k] = (int32_t)g;
    }
  }
  pptr[(size_t)n_regions] = (int32_t)m;
  // pack lower triangles (row-major) and invert each 32x32 diagonal block
  // (row stride kDinvLd) so the panel triangle solves become small GEMVs;
  // symmetric-inverse regions get the packed lower triangle of A[B,B]^{-1}
  std::vector<double> packed((size_t)poff[(size_t)n_regions], 0.0);
  std::vector<int64_t> sym_regions;
  for (int64_t r = 0; r < n_regions; ++r) {
    const int64_t nd = roff[r + 1] - roff[r];
    const double* f = factors + foff[r];
    double* base = packed.data() + poff[(size_t)r];
    if (patch_is_sym(nd, max_dofs, sym)) {
      sym_regions.push_back(r);
      continue;
    }
    double* dst = base;
    for (int64_t i = 0; i < nd; ++i)
      for (int64_t j = 0; j <= i; ++j) *dst++ = f[i * nd + j];
    double* dinv = base + ((nd * (nd + 1) / 2 + 1) & ~int64_t(1));
    if (const int64_t B = patch_block(nd, max_dofs)) {   // the whole L^{-1}, row stride B + 1
      const int64_t ld = B + 1;
      for (int64_t j = 0; j < nd; ++j) {
        for (int64_t i = j; i < nd; ++i) {
          double sacc = (i == j) ? 1.0 : 0.0;
          for (int64_t k = j; k < i; ++k) sacc -= f[i * nd + k] * dinv[k * ld + j];
          dinv[i * ld + j] = sacc / f[i * nd + i];
        }
      }
      continue;
    }
    for (int64_t p0 = 0; p0 < nd; p0 += kPanel) {
      const int64_t pn = std::min<int64_t>(kPanel, nd - p0);
      double* D = dinv + (p0 / kPanel) * kDinvBlock;
      for (int64_t j = 0; j < pn; ++j) {       // column j of the inverse
        for (int64_t i = j; i < pn; ++i) {
          double sacc = (i == j) ? 1.0 : 0.0;
          for (int64_t k = j; k < i; ++k) sacc -= f[(p0 + i) * nd + (p0 + k)] * D[k * kDinvLd + j];
          D[i * kDinvLd + j] = sacc / f[(p0 + i) * nd + (p0 + i)];
        }
      }
    }
  }
  if (!sym_regions.empty()) {
    // largest first, a few host threads (C5: 1000 regions of up to 512 dofs)
    std::stable_sort(sym_regions.begin(), sym_regions.end(), [&](int64_t x, int64_t y) {
      return roff[x + 1] - roff[x] > roff[y + 1] - roff[y];
    });
    std::atomic<size_t> next{0};
    auto work = [&]() {
      std::vector<double> scratch;
      for (size_t q; (q = next.fetch_add(1)) < sym_regions.size();) {
        const int64_t r = sym_regions[q];
        const int64_t nd = roff[r + 1] - roff[r];
        packed_spd_inverse(nd, factors + foff[r], packed.data() + poff[(size_t)r], scratch);
      }
    };
    unsigned nt = std::thread::hardware_concurrency();
    nt = std::max(1u, std::min(nt, 32u));
    nt = (unsigned)std::min<size_t>(nt, sym_regions.size());
    std::vector<std::thread> pool;
    for (unsigned t = 1; t < nt; ++t) pool.emplace_back(work);
    work();
    for (auto& th : pool) th.join();
  }
  auto* cc = new smg_correction();
  Correction& c = cc->c;
  c.n_global = n;
  c.n_regions = (int32_t)n_regions;
  c.m = m;
  c.max_dofs = max_dofs;
  c.sym = sym;
  c.op = &o;
  int32_t* dp = nullptr;
  int32_t* dd = nullptr;
  int64_t* df = nullptr;
  double* dl = nullptr;
  int rc = SMG_OK;
  c.coupled = false;
  if (n_regions > 0) {
    rc = dev_upload(c.allocs, c.device_bytes, pptr.data(), pptr.size(), &dp);
    if (rc == SMG_OK) rc = dev_upload(c.allocs, c.device_bytes, dof32.data(), dof32.size(), &dd);
    if (rc == SMG_OK) rc = dev_upload(c.allocs, c.device_bytes, poff.data(), poff.size(), &df);
    if (rc == SMG_OK) rc = dev_upload(c.allocs, c.device_bytes, packed.data(), packed.size(), &dl);
    if (rc == SMG_OK) {
      std::vector<int32_t> ord((size_t)n_regions);
      for (int64_t r = 0; r < n_regions; ++r) ord[(size_t)r] = (int32_t)r;
      std::stable_sort(ord.begin(), ord.end(), [&](int32_t x, int32_t y) {
        return roff[x + 1] - roff[x] > roff[y + 1] - roff[y];
      });
      int32_t* dord = nullptr;
      rc = dev_upload(c.allocs, c.device_bytes, ord.data(), ord.size(), &dord);
      c.order = dord;
    }
    if (rc == SMG_OK) rc = dev_alloc(c.allocs, c.device_bytes, (size_t)m, &c.rbuf);
    // gathered copy of the patch rows of A (residuals read it coalesced)
    int64_t* dlen = nullptr;
    int64_t* dprow = nullptr;
    int32_t* dpcol = nullptr;
    double* dpval = nullptr;
    std::vector<int64_t> prow((size_t)m + 1, 0);
    if (rc == SMG_OK) rc = dev_alloc(c.allocs, c.device_bytes, (size_t)m, &dlen);
    if (rc == SMG_OK) rc = check_cuda(launch_patch_row_len(o.a, dd, m, dlen), "patch row lengths");
    if (rc == SMG_OK)
      rc = check_cuda(cudaMemcpy(prow.data() + 1, dlen, sizeof(int64_t) * (size_t)m,
                                 cudaMemcpyDeviceToHost), "patch row lengths D2H");
    if (rc == SMG_OK) {
      for (int64_t k = 0; k < m; ++k) prow[(size_t)k + 1] += prow[(size_t)k];
      rc = dev_upload(c.allocs, c.device_bytes, prow.data(), prow.size(), &dprow);
    }
    const int64_t pn = prow[(size_t)m];
    if (rc == SMG_OK) rc = dev_alloc(c.allocs, c.device_bytes, (size_t)pn + 1, &dpcol);
    if (rc == SMG_OK) rc = dev_alloc(c.allocs, c.device_bytes, (size_t)pn + 1, &dpval);
    if (rc == SMG_OK)
      rc = check_cuda(launch_patch_row_gather(o.a, dd, m, dprow, dpcol, dpval), "patch row gather");
    // coupling through A between different regions
    std::vector<int32_t> hcol;
    if (rc == SMG_OK) {
      hcol.resize((size_t)pn);
      rc = check_cuda(cudaMemcpy(hcol.data(), dpcol, sizeof(int32_t) * (size_t)pn,
                                 cudaMemcpyDeviceToHost), "patch columns D2H");
      for (int64_t k = 0; rc == SMG_OK && k < m && !c.coupled; ++k) {
        const int32_t own_row = owner[(size_t)dof32[(size_t)k]];
        for (int64_t j = prow[(size_t)k]; j < prow[(size_t)k + 1]; ++j) {
          const int32_t own = owner[(size_t)hcol[(size_t)j]];
          if (own >= 0 && own != own_row) {
            c.coupled = true;
            break;
          }
        }
      }
    }
    c.prow = dprow;
    c.pcol = dpcol;
    c.pval = dpval;
    if (rc == SMG_OK) rc = build_halo(o, dof32, hcol, c);
    if (rc == SMG_OK) rc = build_ring(o, pptr, dof32, prow, hcol, c);
    if (rc == SMG_OK) {
      c.pptr = dp;
      c.dofs = dd;
      c.foff = df;
      c.lfac = dl;
      rc = check_cuda(configure_patch_solve_smem(c), "patch solve shared memory");
    }
  }
  if (rc != SMG_OK) {
    free_all(c.allocs);
    delete cc;
    return rc;
  }
  c.pptr = dp;
  c.dofs = dd;
  c.foff = df;
  c.lfac = dl;
  *out = cc;
  return SMG_OK;
}

int smg_correction_destroy(smg_correction* c)
{
  if (!c) return SMG_OK;
  free_all(c->c.allocs);
  delete c;
  return SMG_OK;
}

int smg_correction_info(const smg_correction* c, int64_t* n_regions, int64_t* covered, int* coupled,
                        int64_t* device_bytes)
{
  if (!c) return fail("correction is NULL");
  if (n_regions) *n_regions = c->c.n_regions;
  if (covered) *covered = c->c.m;
  if (coupled) *coupled = c->c.coupled ? 1 : 0;
  if (device_bytes) *device_bytes = c->c.device_bytes;
  return SMG_OK;
}

int smg_apply_local_correction(const smg_correction* c, const double* r, double* out, void* stream)
{
  if (!c) return fail("correction is NULL");
  const Correction& cc = c->c;
  cudaStream_t st = as_stream(stream);
  if (cc.n_global > 0) SMG_CUDA(cudaMemsetAsync(out, 0, sizeof(double) * (size_t)cc.n_global, st));
  if (cc.n_regions == 0) return SMG_OK;
  // rbuf[k] = r[dofs[k]], then the batched solves scatter into out
  SMG_CUDA(launch_gather(cc.dofs, cc.m, r, cc.rbuf, st));
  SMG_CUDA(launch_patch_solve(cc, nullptr, nullptr, nullptr, out, false, st));
  return SMG_OK;
}

int smg_local_correct(const smg_correction* c, const double* b, double* u, void* stream)
{
  if (!c) return fail("correction is NULL");
  int64_t n = 0;
  return enqueue_local_correct(c->c, b, u, as_stream(stream), &n);
}

int smg_combined_smooth(const smg_operator* a, const double* b, double* u, const smg_correction* c,
                        int kind, int sweeps, double lambda_max, double frac, double* work,
                        void* stream)
{
  if (!a) return fail("operator is NULL");
  if (c && c->c.n_regions > 0 && c->c.op != &a->o) {
    // the correction forms its patch residuals from the rows of the operator
    // it was created with (smg_correction_create); another operator would
    // give the residual of a different matrix
    set_error("correction of size " + std::to_string(c->c.n_global) +
              " was created for another operator; it does not match this " +
              std::to_string(a->o.a.nrows) + "-row operator");
    return SMG_ERR_DIMENSION;
  }
  return smooth_standalone(a->o, b, u, c ? &c->c : nullptr, kind, sweeps, lambda_max, frac, work,
                           as_stream(stream));
}

// A_L^{-1} (dense, row-major, symmetric) -> lower-triangle 64 x 64 tiles
static int upload_sym_tiles(std::vector<void*>& allocs, int64_t& bytes, int64_t n,
                            const double* dense, SymTiles* out)
{
  SymTiles m;
  m.n = n;
  m.nb = (int)((n + kSymTile - 1) / kSymTile);
  const int64_t ntiles = (int64_t)m.nb * (m.nb + 1) / 2;
  std::vector<double> t((size_t)(ntiles * kSymTile * kSymTile), 0.0);
  std::vector<int32_t> ti((size_t)ntiles);
  int64_t k = 0;
  for (int I = 0; I < m.nb; ++I)
    for (int J = 0; J <= I; ++J, ++k) {
      ti[(size_t)k] = I;
      double* dst = t.data() + k * kSymTile * kSymTile;
      for (int r = 0; r < kSymTile; ++r) {
        const int64_t gi = (int64_t)I * kSymTile + r;
        if (gi >= n) break;
        for (int c = 0; c < kSymTile; ++c) {
          const int64_t gj = (int64_t)J * kSymTile + c;
          if (gj >= n) break;
          dst[r * kSymTile + c] = dense[gi * n + gj];
        }
      }
    }
  double* dt = nullptr;
  int32_t* dti = nullptr;
  double* dp = nullptr;
  SMG_TRY(dev_upload(allocs, bytes, t.data(), t.size(), &dt));
  SMG_TRY(dev_upload(allocs, bytes, ti.data(), ti.size(), &dti));
  SMG_TRY(dev_alloc(allocs, bytes, (size_t)m.nb * m.nb * kSymTile, &dp));
  unsigned int* dc = nullptr;
  SMG_TRY(dev_alloc(allocs, bytes, (size_t)m.nb, &dc));
  SMG_CUDA(cudaMemset(dc, 0, sizeof(unsigned int) * (size_t)m.nb));
  m.tiles = dt;
  m.tile_i = dti;
  m.partial = dp;
  m.counter = dc;
  *out = m;
  return SMG_OK;
}

// ---------------------------------------------------------------------------
// Locality renumbering of a level's device copy: a
// symmetric permutation (reverse Cuthill-McKee of the operator's graph)
// renames rows and columns of A_l, the rows of P_l and the columns of
// P_{l-1}, so each SELL window / tile gathers x from a compact index range.
// Every row keeps its entries in the reference's column order (only the
// names change), CSR(P^T) keeps ascending ORIGINAL fine rows, and the patch
// factors keep their row order -- every sum is the same sequence of the same
// operations, so a renumbered V-cycle is bit-identical to the plain one.
// Level 0's b and u are gathered into the renamed space at the start of the
// V-cycle and back at its end (three gathers, inside the graph).
struct HostCsr {
  int64_t nrows = 0, ncols = 0;
  std::vector<int64_t> ptr;
  std::vector<int32_t> col;
  std::vector<double> val;
};

static int download_csr(const DevCsr& m, HostCsr* out)
{
  out->nrows = m.nrows;
  out->ncols = m.ncols;
  out->ptr.resize((size_t)m.nrows + 1);
  out->col.resize((size_t)m.nnz);
  out->val.resize((size_t)m.nnz);
  SMG_CUDA(cudaMemcpy(out->ptr.data(), m.rowptr, sizeof(int64_t) * (size_t)(m.nrows + 1),
                      cudaMemcpyDeviceToHost));
  if (m.nnz > 0) {
    SMG_CUDA(cudaMemcpy(out->col.data(), m.col, sizeof(int32_t) * (size_t)m.nnz, cudaMemcpyDeviceToHost));
    SMG_CUDA(cudaMemcpy(out->val.data(), m.val, sizeof(double) * (size_t)m.nnz, cudaMemcpyDeviceToHost));
  }
  return SMG_OK;
}

// reverse Cuthill-McKee: BFS from a low-degree node of each component,
// neighbours in ascending (degree, index) order, order reversed.  perm[old] = new.
static std::vector<int32_t> rcm_permutation(const HostCsr& a)
{
  const int64_t n = a.nrows;
  std::vector<int32_t> deg((size_t)n);
  for (int64_t i = 0; i < n; ++i) deg[(size_t)i] = (int32_t)(a.ptr[(size_t)i + 1] - a.ptr[(size_t)i]);
  std::vector<int32_t> by_deg((size_t)n);
  for (int64_t i = 0; i < n; ++i) by_deg[(size_t)i] = (int32_t)i;
  std::stable_sort(by_deg.begin(), by_deg.end(),
                   [&](int32_t x, int32_t y) { return deg[(size_t)x] < deg[(size_t)y]; });
  std::vector<uint8_t> seen((size_t)n, 0);
  std::vector<int32_t> order;
  order.reserve((size_t)n);
  std::vector<int32_t> nb;
  auto bfs = [&](int32_t start, std::vector<int32_t>* out, int32_t* last) {
    // plain BFS (for the pseudo-peripheral search) when out == nullptr
    std::vector<int32_t> q{start};
    std::vector<uint8_t>& mark = seen;
    mark[(size_t)start] = 2;
    size_t h = 0;
    while (h < q.size()) {
      const int32_t u = q[h++];
      nb.clear();
      for (int64_t j = a.ptr[(size_t)u]; j < a.ptr[(size_t)u + 1]; ++j) {
        const int32_t v = a.col[(size_t)j];
        if (v != u && !mark[(size_t)v]) nb.push_back(v);
      }
      std::sort(nb.begin(), nb.end(), [&](int32_t x, int32_t y) {
        return deg[(size_t)x] != deg[(size_t)y] ? deg[(size_t)x] < deg[(size_t)y] : x < y;
      });
      for (int32_t v : nb)
        if (!mark[(size_t)v]) {
          mark[(size_t)v] = 2;
          q.push_back(v);
        }
    }
    if (last) *last = q.back();
    if (out) {
      for (int32_t v : q) {
        mark[(size_t)v] = 1;
        out->push_back(v);
      }
    } else {
      for (int32_t v : q) mark[(size_t)v] = 0;   // probe only: unmark
    }
  };
  for (int32_t s0 : by_deg) {
    if (seen[(size_t)s0]) continue;
    int32_t start = s0, far = s0;
    bfs(start, nullptr, &far);   // one pseudo-peripheral step: restart from the far end
    start = far;
    bfs(start, &order, nullptr);
  }
  std::vector<int32_t> perm((size_t)n);
  for (int64_t k = 0; k < n; ++k) perm[(size_t)order[(size_t)k]] = (int32_t)(n - 1 - k);
  return perm;
}

// greedy BFS clusters of `csize` nodes (compact blobs: a SELL window's rows
// and their x columns sit together), each cluster grown from the first
// unclustered node adjacent to the previous one, nodes numbered in the order
// they join.  perm[old] = new.
static std::vector<int32_t> cluster_permutation(const HostCsr& a, int csize)
{
  const int64_t n = a.nrows;
  std::vector<int32_t> perm((size_t)n, -1);
  std::vector<int32_t> q;
  q.reserve((size_t)csize * 8);
  int32_t next = 0;
  int64_t scan = 0;          // lowest possibly unclustered node
  std::vector<int32_t> frontier_seed;
  int32_t seed = -1;
  while (next < n) {
    if (seed < 0 || perm[(size_t)seed] >= 0) {
      while (scan < n && perm[(size_t)scan] >= 0) ++scan;
      seed = (int32_t)scan;
    }
    // grow one cluster by BFS from seed
    q.clear();
    q.push_back(seed);
    perm[(size_t)seed] = next++;
    size_t h = 0;
    int taken = 1;
    int32_t boundary = -1;
    while (h < q.size()) {
      const int32_t u = q[h++];
      for (int64_t j = a.ptr[(size_t)u]; j < a.ptr[(size_t)u + 1]; ++j) {
        const int32_t v = a.col[(size_t)j];
        if (perm[(size_t)v] >= 0) continue;
        if (taken < csize) {
          perm[(size_t)v] = next++;
          ++taken;
          q.push_back(v);
        } else if (boundary < 0) {
          boundary = v;      // the next cluster starts next to this one
        }
      }
      if (taken >= csize && boundary >= 0) break;
    }
    seed = boundary;
  }
  return perm;
}

// rows moved by rperm (old -> new, or identity), columns renamed by cperm,
// each row's entries in their original order
static HostCsr renamed(const HostCsr& a, const int32_t* rperm, const int32_t* cperm)
{
  HostCsr b;
  b.nrows = a.nrows;
  b.ncols = a.ncols;
  b.ptr.assign((size_t)a.nrows + 1, 0);
  for (int64_t i = 0; i < a.nrows; ++i) {
    const int64_t r = rperm ? rperm[i] : i;
    b.ptr[(size_t)r + 1] = a.ptr[(size_t)i + 1] - a.ptr[(size_t)i];
  }
  for (int64_t r = 0; r < a.nrows; ++r) b.ptr[(size_t)r + 1] += b.ptr[(size_t)r];
  b.col.resize(a.col.size());
  b.val.resize(a.val.size());
  for (int64_t i = 0; i < a.nrows; ++i) {
    const int64_t r = rperm ? rperm[i] : i;
    int64_t o = b.ptr[(size_t)r];
    for (int64_t j = a.ptr[(size_t)i]; j < a.ptr[(size_t)i + 1]; ++j, ++o) {
      b.col[(size_t)o] = cperm ? cperm[a.col[(size_t)j]] : a.col[(size_t)j];
      b.val[(size_t)o] = a.val[(size_t)j];
    }
  }
  return b;
}

// CSR of P^T with the coarse rows renamed by cperm and, inside every row, the
// fine entries in ascending ORIGINAL fine row order (scipy csc_matvec's order),
// their names taken from rperm
static HostCsr transposed_original_order(const HostCsr& p, const int32_t* rperm,
                                         const int32_t* cperm)
{
  HostCsr t;
  t.nrows = p.ncols;
  t.ncols = p.nrows;
  t.ptr.assign((size_t)p.ncols + 1, 0);
  for (int32_t c : p.col) ++t.ptr[(size_t)(cperm ? cperm[c] : c) + 1];
  for (int64_t r = 0; r < t.nrows; ++r) t.ptr[(size_t)r + 1] += t.ptr[(size_t)r];
  std::vector<int64_t> fill(t.ptr.begin(), t.ptr.end() - 1);
  t.col.resize(p.col.size());
  t.val.resize(p.val.size());
  for (int64_t i = 0; i < p.nrows; ++i)
    for (int64_t j = p.ptr[(size_t)i]; j < p.ptr[(size_t)i + 1]; ++j) {
      const int32_t c = p.col[(size_t)j];
      const int64_t pos = fill[(size_t)(cperm ? cperm[c] : c)]++;
      t.col[(size_t)pos] = rperm ? rperm[i] : (int32_t)i;
      t.val[(size_t)pos] = p.val[(size_t)j];
    }
  return t;
}

static int upload_renamed(const HostCsr& h, Operator& o, DevCsr* out)
{
  std::vector<int64_t> c64(h.col.begin(), h.col.end());
  return build_devcsr(o.allocs, o.device_bytes, h.nrows, h.ncols, h.ptr.data(), c64.data(),
                      h.val.data(), out);
}

// a renamed square operator: diagonal found by a linear search (rows are no
// longer sorted), 1/a_ii by the same IEEE division as the original
static int make_renamed_operator(const HostCsr& h, const Operator& src, Operator& o)
{
  SMG_TRY(upload_renamed(h, o, &o.a));
  o.first_zero_diag = src.first_zero_diag;
  o.all_finite = src.all_finite;
  if (h.nrows == h.ncols && h.nrows > 0) {
    std::vector<double> diag((size_t)h.nrows, 0.0), inv((size_t)h.nrows);
    for (int64_t r = 0; r < h.nrows; ++r) {
      for (int64_t j = h.ptr[(size_t)r]; j < h.ptr[(size_t)r + 1]; ++j)
        if (h.col[(size_t)j] == r) diag[(size_t)r] = h.val[(size_t)j];
      inv[(size_t)r] = 1.0 / diag[(size_t)r];
    }
    double *dd = nullptr, *di = nullptr;
    SMG_TRY(dev_upload(o.allocs, o.device_bytes, diag.data(), diag.size(), &dd));
    SMG_TRY(dev_upload(o.allocs, o.device_bytes, inv.data(), inv.size(), &di));
    o.diag = dd;
    o.inv_diag = di;
    o.a.inv_diag = di;
  }
  return SMG_OK;
}

// the correction of a renamed level: the same regions, factors (shared with
// the source, never freed here) and launch order, dofs renamed, the patch rows
// gathered from the renamed operator (original column order, renamed columns)
static int make_renamed_correction(const Correction& src, const Operator& op,
                                   const std::vector<int32_t>& perm, Correction& c)
{
  c.n_global = src.n_global;
  c.n_regions = src.n_regions;
  c.m = src.m;
  c.max_dofs = src.max_dofs;
  c.pptr = src.pptr;
  c.order = src.order;
  c.foff = src.foff;
  c.lfac = src.lfac;
  c.coupled = src.coupled;
  c.sym = src.sym;
  c.op = &op;
  std::vector<int32_t> dofs((size_t)src.m);
  if (src.m > 0)
    SMG_CUDA(cudaMemcpy(dofs.data(), src.dofs, sizeof(int32_t) * (size_t)src.m, cudaMemcpyDeviceToHost));
  for (auto& g : dofs) g = perm[(size_t)g];
  int32_t* dd = nullptr;
  SMG_TRY(dev_upload(c.allocs, c.device_bytes, dofs.data(), dofs.size(), &dd));
  c.dofs = dd;
  SMG_TRY(dev_alloc(c.allocs, c.device_bytes, (size_t)src.m, &c.rbuf));
  std::vector<int64_t> prow((size_t)src.m + 1, 0);
  int64_t* dlen = nullptr;
  SMG_TRY(dev_alloc(c.allocs, c.device_bytes, (size_t)std::max<int64_t>(src.m, 1), &dlen));
  SMG_CUDA(launch_patch_row_len(op.a, dd, src.m, dlen));
  SMG_CUDA(cudaMemcpy(prow.data() + 1, dlen, sizeof(int64_t) * (size_t)src.m, cudaMemcpyDeviceToHost));
  for (int64_t k = 0; k < src.m; ++k) prow[(size_t)k + 1] += prow[(size_t)k];
  int64_t* dprow = nullptr;
  int32_t* dpcol = nullptr;
  double* dpval = nullptr;
  SMG_TRY(dev_upload(c.allocs, c.device_bytes, prow.data(), prow.size(), &dprow));
  SMG_TRY(dev_alloc(c.allocs, c.device_bytes, (size_t)prow[(size_t)src.m] + 1, &dpcol));
  SMG_TRY(dev_alloc(c.allocs, c.device_bytes, (size_t)prow[(size_t)src.m] + 1, &dpval));
  SMG_CUDA(launch_patch_row_gather(op.a, dd, src.m, dprow, dpcol, dpval));
  SMG_CUDA(cudaDeviceSynchronize());
  c.prow = dprow;
  c.pcol = dpcol;
  c.pval = dpval;
  return SMG_OK;
}

// SMG_RENUMBER: bit l set = renumber level l (never the coarsest); "auto"
// (default) = levels whose operator is streamed from HBM (val + col > 64 MB)
static bool renumber_level(int l, int n_levels, const Operator& a)
{
  if (l >= n_levels - 1) return false;
  const char* env = getenv("SMG_RENUMBER");   // read per hierarchy (tests switch it)
  if (!env || !strcmp(env, "auto")) return false;   // measured first: off unless requested
  const long mask = strtol(env, nullptr, 0);
  (void)a;
  return (mask >> l) & 1;
}

int smg_hierarchy_create(int n_levels, const smg_operator* const* a, const smg_operator* const* p,
                         const smg_correction* const* corrections, const int* kinds,
                         const int* sweeps, const double* lambda_max, const double* frac,
                         int64_t n_coarse, const double* coarse_inverse, int coarse_refine,
                         smg_hierarchy** out)
{
  if (!out) return fail("out is NULL");
  *out = nullptr;
  if (n_levels < 2) return fail("a hierarchy needs at least 2 levels, got " + std::to_string(n_levels));
  if (!a || !p || !kinds || !sweeps || !lambda_max || !frac) return fail("NULL level arrays");
  auto* hh = new smg_hierarchy();
  Hierarchy& h = hh->h;
  auto bail = [&](int rc) {
    delete hh;
    return rc;
  };
  h.lv.resize((size_t)n_levels);
  for (int l = 0; l < n_levels; ++l) {
    HLevel& L = h.lv[(size_t)l];
    if (!a[l]) return bail(fail("level operator is NULL"));
    L.a = &a[l]->o;
    L.n = L.a->a.nrows;
    if (L.a->a.nrows != L.a->a.ncols) return bail(fail("level operators must be square"));
    if (l < n_levels - 1) {
      if (!p[l]) return bail(fail("prolongation is NULL"));
      L.p = &p[l]->o;
      if (!L.p->has_t) return bail(fail("prolongations must be created with_transpose"));
      if (L.p->a.nrows != L.n || L.p->a.ncols != a[l + 1]->o.a.nrows)
        return bail(fail("dimension mismatch between prolongation and level operators"));
      L.lc = corrections ? (corrections[l] ? &corrections[l]->c : nullptr) : nullptr;
      if (L.lc && L.lc->n_regions > 0 && L.lc->op != L.a)
        return bail(fail("level " + std::to_string(l) +
                         ": the correction was created for another operator (does not match)"));
      L.kind = kinds[l];
      L.sweeps = sweeps[l];
      L.lambda_max = lambda_max[l];
      L.frac = frac[l];
      if (L.kind == SMG_SMOOTHER_SGS) {
        set_error("symmetric Gauss-Seidel is outside the GPU hot path");
        return bail(SMG_ERR_UNSUPPORTED);
      }
      int rc = cheb_scalars(L.sweeps, L.lambda_max, L.frac, &L.cs);
      if (rc != SMG_OK) return bail(rc);
      rc = check_square_diag(*L.a);
      if (rc != SMG_OK) return bail(rc);
    }
  }
  if (n_coarse != h.lv.back().n) return bail(fail("coarse inverse size does not match the coarsest level"));
  if (!coarse_inverse) return bail(fail("coarse_inverse is NULL"));
  int rc = SMG_OK;
  for (int l = 0; l < n_levels && rc == SMG_OK; ++l) {
    HLevel& L = h.lv[(size_t)l];
    const size_t n = (size_t)L.n;
    if (l > 0) {
      rc = dev_alloc(h.allocs, h.bytes, n, &L.b);
      if (rc == SMG_OK) rc = dev_alloc(h.allocs, h.bytes, n, &L.u);
    }
    if (rc == SMG_OK && l < n_levels - 1) {
      rc = dev_alloc(h.allocs, h.bytes, n, &L.t);
      if (rc == SMG_OK) rc = dev_alloc(h.allocs, h.bytes, n, &L.d);
      if (rc == SMG_OK) rc = dev_alloc(h.allocs, h.bytes, n, &L.r);
    }
  }
  // locality renumbering (renumber_level): renamed copies of A_l, P_l, P_{l-1}
  // and the corrections; the originals stay with their owners untouched
  h.a_user = h.lv[0].a;
  for (int l = 0; l < n_levels - 1 && rc == SMG_OK; ++l) {
    HLevel& L = h.lv[(size_t)l];
    if (!renumber_level(l, n_levels, *L.a)) continue;
    HostCsr ah;
    rc = download_csr(L.a->a, &ah);
    if (rc != SMG_OK) break;
    {
      const char* ord = getenv("SMG_RENUMBER_ORDER");   // "rcm" | "cluster" (default)
      L.perm_h = (ord && !strcmp(ord, "rcm")) ? rcm_permutation(ah)
                                              : cluster_permutation(ah, kSellWindow);
    }
    L.renum = true;
    auto op = std::make_unique<Operator>();
    const HostCsr ar = renamed(ah, L.perm_h.data(), L.perm_h.data());
    rc = make_renamed_operator(ar, *L.a, *op);
    if (rc != SMG_OK) {
      free_all(op->allocs);
      break;
    }
    if (L.lc && L.lc->n_regions > 0) {
      auto cc = std::make_unique<Correction>();
      rc = make_renamed_correction(*L.lc, *op, L.perm_h, *cc);
      if (rc != SMG_OK) {
        free_all(cc->allocs);
        free_all(op->allocs);
        break;
      }
      L.lc = cc.get();
      h.own_corrs.push_back(std::move(cc));
    }
    L.a = op.get();
    h.own_ops.push_back(std::move(op));
    if (l == 0) {
      std::vector<int32_t> inv(L.perm_h.size());
      for (size_t i = 0; i < L.perm_h.size(); ++i) inv[(size_t)L.perm_h[i]] = (int32_t)i;
      rc = dev_upload(h.allocs, h.bytes, L.perm_h.data(), L.perm_h.size(), &L.perm);
      if (rc == SMG_OK) rc = dev_upload(h.allocs, h.bytes, inv.data(), inv.size(), &L.inv);
      if (rc == SMG_OK) rc = dev_alloc(h.allocs, h.bytes, (size_t)L.n, &h.b0r);
      if (rc == SMG_OK) rc = dev_alloc(h.allocs, h.bytes, (size_t)L.n, &h.u0r);
    }
  }
  for (int l = 0; l < n_levels - 1 && rc == SMG_OK; ++l) {
    HLevel& L = h.lv[(size_t)l];
    const HLevel& N = h.lv[(size_t)l + 1];
    if (!L.renum && !N.renum) continue;
    HostCsr ph;
    rc = download_csr(L.p->a, &ph);
    if (rc != SMG_OK) break;
    const int32_t* rp = L.renum ? L.perm_h.data() : nullptr;
    const int32_t* cp = N.renum ? N.perm_h.data() : nullptr;
    auto op = std::make_unique<Operator>();
    rc = upload_renamed(renamed(ph, rp, cp), *op, &op->a);
    if (rc == SMG_OK) rc = upload_renamed(transposed_original_order(ph, rp, cp), *op, &op->t);
    if (rc != SMG_OK) {
      free_all(op->allocs);
      break;
    }
    op->has_t = true;
    L.p = op.get();
    h.own_ops.push_back(std::move(op));
  }
  // P's rows on the correction rings (follow-mode prolong-add + correction)
  for (int l = 0; l < n_levels - 1 && rc == SMG_OK; ++l) {
    HLevel& L = h.lv[(size_t)l];
    if (L.lc && L.lc->has_ring && L.lc->n_global == L.n) {
      rc = gather_rows(h.allocs, h.bytes, L.p->a, L.lc->ring_rows, L.lc->ring_total, &L.ringP);
      L.has_ringP = rc == SMG_OK;
    }
  }
  if (rc == SMG_OK) rc = upload_sym_tiles(h.allocs, h.bytes, n_coarse, coarse_inverse, &h.coarse);
  h.n_coarse = n_coarse;
  h.coarse_refine = coarse_refine;
  if (rc == SMG_OK && coarse_refine) rc = dev_alloc(h.allocs, h.bytes, (size_t)n_coarse, &h.coarse_r);
  if (rc == SMG_OK) rc = dev_alloc(h.allocs, h.bytes, (size_t)h.lv[0].n, &h.stage_b);
  if (rc == SMG_OK) rc = dev_alloc(h.allocs, h.bytes, (size_t)h.lv[0].n, &h.stage_u);
  if (rc != SMG_OK) return bail(rc);
  *out = hh;
  return SMG_OK;
}

int smg_hierarchy_destroy(smg_hierarchy* h)
{
  delete h;
  return SMG_OK;
}

int smg_hierarchy_set_graphs(smg_hierarchy* h, int enable)
{
  if (!h) return fail("hierarchy is NULL");
  std::lock_guard<std::recursive_mutex> lk(h->h.mu);
  h->h.use_graphs = enable != 0;
  return SMG_OK;
}

int smg_hierarchy_set_option(smg_hierarchy* h, int option, int value)
{
  if (!h) return fail("hierarchy is NULL");
  Hierarchy& H = h->h;
  std::lock_guard<std::recursive_mutex> lk(H.mu);
  if (option == SMG_OPT_GRAPHS)
    H.use_graphs = value != 0;
  else if (option == SMG_OPT_FUSE_ZERO_GUESS)
    H.fuse_zero_guess = value != 0;
  else if (option == SMG_OPT_LC_OVERLAP)
    H.lc_overlap = value != 0;
  else if (option == SMG_OPT_LC_FOLLOW)
    H.lc_follow = value != 0;
  else
    return fail("unknown hierarchy option");
  for (auto& kv : H.graphs) cudaGraphExecDestroy(kv.second);
  H.graphs.clear();
  return SMG_OK;
}

int smg_coarse_solve(smg_hierarchy* h, const double* b_c, double* x_c, void* stream)
{
  if (!h || !b_c || !x_c) return fail("NULL argument");
  Hierarchy& H = h->h;
  std::lock_guard<std::recursive_mutex> lk(H.mu);
  cudaStream_t st = as_stream(stream);
  ScratchOrder ord{&H, st};
  SMG_TRY(ord.begin());
  SMG_CUDA(launch_sym_apply(H.coarse, b_c, x_c, false, st));
  if (H.coarse_refine) {
    EpiArgs ea;
    ea.b = b_c;
    ea.out = H.coarse_r;
    SMG_CUDA(launch_csr_stream(H.lv.back().a->a, x_c, Epi::kResidual, ea, st));
    SMG_CUDA(launch_sym_apply(H.coarse, H.coarse_r, x_c, true, st));
  }
  return ord.end();
}

int smg_hierarchy_launches_per_vcycle(const smg_hierarchy* h, int64_t* launches)
{
  if (!h || !launches) return fail("NULL argument");
  *launches = h->h.launches;
  return SMG_OK;
}

int smg_vcycle(smg_hierarchy* h, const double* b, double* u, void* stream)
{
  if (!h) return fail("hierarchy is NULL");
  std::lock_guard<std::recursive_mutex> lk(h->h.mu);
  ScratchOrder ord{&h->h, as_stream(stream)};
  SMG_TRY(ord.begin());
  SMG_TRY(run_vcycle(h->h, b, u, as_stream(stream)));
  return ord.end();
}

int smg_vcycle_host(smg_hierarchy* h, const double* b_host, double* u_host, void* stream)
{
  if (!h) return fail("hierarchy is NULL");
  Hierarchy& H = h->h;
  std::lock_guard<std::recursive_mutex> lk(H.mu);
  cudaStream_t st = as_stream(stream);
  ScratchOrder ord{&H, st};
  SMG_TRY(ord.begin());
  const size_t bytes = sizeof(double) * (size_t)H.lv[0].n;
  SMG_CUDA(cudaMemcpyAsync(H.stage_b, b_host, bytes, cudaMemcpyHostToDevice, st));
  SMG_CUDA(cudaMemcpyAsync(H.stage_u, u_host, bytes, cudaMemcpyHostToDevice, st));
  SMG_TRY(run_vcycle(H, H.stage_b, H.stage_u, st));
  SMG_CUDA(cudaMemcpyAsync(u_host, H.stage_u, bytes, cudaMemcpyDeviceToHost, st));
  SMG_TRY(ord.end());
  SMG_CUDA(cudaStreamSynchronize(st));
  return SMG_OK;
}

// Independent (b, u) pairs in host memory, one V-cycle each, pipelined: the
// H2D copies of pair i+1 (copy-in stream) and the D2H copy of pair i-1
// (copy-out stream) overlap the V-cycle of pair i (two staging slots).
int smg_vcycle_host_many(smg_hierarchy* h, int64_t count, const double* const* b_host,
                         double* const* u_host, void* stream)
{
  if (!h) return fail("hierarchy is NULL");
  if (count < 0) return fail("negative count");
  if (count > 0 && (!b_host || !u_host)) return fail("NULL host pointer arrays");
  Hierarchy& H = h->h;
  std::lock_guard<std::recursive_mutex> lk(H.mu);
  cudaStream_t st = as_stream(stream);
  ScratchOrder ord{&H, st};
  SMG_TRY(ord.begin());
  if (!H.stage_b2) {
    SMG_TRY(dev_alloc(H.allocs, H.bytes, (size_t)H.lv[0].n, &H.stage_b2));
    SMG_TRY(dev_alloc(H.allocs, H.bytes, (size_t)H.lv[0].n, &H.stage_u2));
    SMG_CUDA(cudaStreamCreateWithFlags(&H.copy_in, cudaStreamNonBlocking));
    SMG_CUDA(cudaStreamCreateWithFlags(&H.copy_out, cudaStreamNonBlocking));
    for (cudaEvent_t& e : H.pipe_ev) SMG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  double* sb[2] = {H.stage_b, H.stage_b2};
  double* su[2] = {H.stage_u, H.stage_u2};
  cudaEvent_t* in_done = H.pipe_ev;       // per slot: H2D finished
  cudaEvent_t* out_done = H.pipe_ev + 2;  // per slot: D2H finished (slot free)
  cudaEvent_t start = H.pipe_ev[4];
  const size_t bytes = sizeof(double) * (size_t)H.lv[0].n;
  // the copies must follow whatever the caller queued on its stream
  SMG_CUDA(cudaEventRecord(start, st));
  SMG_CUDA(cudaStreamWaitEvent(H.copy_in, start, 0));
  SMG_CUDA(cudaStreamWaitEvent(H.copy_out, start, 0));
  for (int64_t i = 0; i < count; ++i) {
    const int s = (int)(i & 1);
    if (i >= 2) SMG_CUDA(cudaStreamWaitEvent(H.copy_in, out_done[s], 0));
    SMG_CUDA(cudaMemcpyAsync(sb[s], b_host[i], bytes, cudaMemcpyHostToDevice, H.copy_in));
    SMG_CUDA(cudaMemcpyAsync(su[s], u_host[i], bytes, cudaMemcpyHostToDevice, H.copy_in));
    SMG_CUDA(cudaEventRecord(in_done[s], H.copy_in));
    SMG_CUDA(cudaStreamWaitEvent(st, in_done[s], 0));
    SMG_TRY(run_vcycle(H, sb[s], su[s], st));
    SMG_CUDA(cudaEventRecord(H.pipe_ev[5], st));
    SMG_CUDA(cudaStreamWaitEvent(H.copy_out, H.pipe_ev[5], 0));
    SMG_CUDA(cudaMemcpyAsync(u_host[i], su[s], bytes, cudaMemcpyDeviceToHost, H.copy_out));
    SMG_CUDA(cudaEventRecord(out_done[s], H.copy_out));
  }
  SMG_TRY(ord.end());
  SMG_CUDA(cudaStreamSynchronize(H.copy_out));
  SMG_CUDA(cudaStreamSynchronize(st));
  return SMG_OK;
}

int smg_solve_stationary(smg_hierarchy* h, const double* b, double* u, double rtol, int max_cycles,
                         double* history, int* n_history, void* stream)
{
  if (!h || !history || !n_history) return fail("NULL argument");
  Hierarchy& H = h->h;
  std::lock_guard<std::recursive_mutex> lk(H.mu);
  cudaStream_t st = as_stream(stream);
  ScratchOrder ord{&H, st};
  SMG_TRY(ord.begin());
  struct End {
    ScratchOrder& o;
    ~End() { o.end(); }
  } end_guard{ord};
  HLevel& L0 = H.lv[0];
  const int64_t n = L0.n;
  const Operator& A0 = *H.a_user;   // b and u are in the caller's order
  double rr = 0, bb = 0;
  EpiArgs ea;
  ea.b = b;
  ea.out = L0.r;
  SMG_CUDA(launch_csr_stream(A0.a, u, Epi::kResidual, ea, st));
  SMG_TRY(H.dots.dot(n, L0.r, L0.r, st, &rr));
  SMG_TRY(H.dots.dot(n, b, b, st, &bb));
  const double residual = std::sqrt(rr);
  const double norm_b = std::sqrt(bb);
  const double denom = norm_b > 0 ? norm_b : residual;
  int cnt = 0;
  if (denom == 0.0) {
    history[cnt++] = 0.0;
    *n_history = cnt;
    return SMG_OK;
  }
  history[cnt++] = residual / denom;
  for (int k = 0; k < max_cycles; ++k) {
    if (history[cnt - 1] <= rtol) break;
    SMG_TRY(run_vcycle(H, b, u, st));
    SMG_CUDA(launch_csr_stream(A0.a, u, Epi::kResidual, ea, st));
    SMG_TRY(H.dots.dot(n, L0.r, L0.r, st, &rr));
    history[cnt++] = std::sqrt(rr) / denom;
  }
  *n_history = cnt;
  return SMG_OK;
}

int smg_cg(smg_hierarchy* h, const smg_operator* a, const double* b, double* x, int x0_given,
           double rtol, int maxit, double* history, int* n_history, int64_t* bad_iteration,
           double* bad_curvature, void* stream)
{
  if (!a || !history || !n_history) return fail("NULL argument");
  const Operator& A = a->o;
  const int64_t n = A.a.nrows;
  if (A.a.nrows != A.a.ncols) return fail("cg needs a square operator");
  if (h && h->h.lv[0].n != n) {
    set_error("dimension mismatch: the preconditioner's fine level has " +
              std::to_string(h->h.lv[0].n) + " dofs, the operator " + std::to_string(n) +
              " (does not match)");
    return SMG_ERR_DIMENSION;
  }
  cudaStream_t st = as_stream(stream);
  std::unique_lock<std::recursive_mutex> lk;
  if (h) lk = std::unique_lock<std::recursive_mutex>(h->h.mu);
  ScratchOrder ord{h ? &h->h : nullptr, st};
  SMG_TRY(ord.begin());
  struct End {
    ScratchOrder& o;
    ~End() { o.end(); }
  } end_guard{ord};
  std::vector<void*> tmp;
  int64_t bytes = 0;
  double *r = nullptr, *z = nullptr, *d = nullptr, *q = nullptr;
  SMG_TRY(dev_alloc(tmp, bytes, (size_t)n, &r));
  SMG_TRY(dev_alloc(tmp, bytes, (size_t)n, &z));
  SMG_TRY(dev_alloc(tmp, bytes, (size_t)n, &d));
  SMG_TRY(dev_alloc(tmp, bytes, (size_t)n, &q));
  DotScratch local;
  DotScratch& dots = h ? h->h.dots : local;
  struct Guard {
    std::vector<void*>& t;
    DotScratch& l;
    cudaStream_t s;
    ~Guard()
    {
      cudaStreamSynchronize(s);
      free_all(t);
      l.release();
    }
  } guard{tmp, local, st};

  auto precond = [&](const double* rin, double* zout) -> int {
    if (!h) {
      SMG_CUDA(cudaMemcpyAsync(zout, rin, sizeof(double) * (size_t)n, cudaMemcpyDeviceToDevice, st));
      return SMG_OK;
    }
    SMG_CUDA(cudaMemsetAsync(zout, 0, sizeof(double) * (size_t)n, st));
    return run_vcycle(h->h, rin, zout, st);
  };
  if (!x0_given) SMG_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * (size_t)n, st));
  EpiArgs ea;
  ea.b = b;
  ea.out = r;
  SMG_CUDA(launch_csr_stream(A.a, x, Epi::kResidual, ea, st));
  double bb = 0, rr = 0;
  SMG_TRY(dots.dot(n, b, b, st, &bb));
  SMG_TRY(dots.dot(n, r, r, st, &rr));
  const double norm_b = std::sqrt(bb);
  const double denom = norm_b > 0 ? norm_b : std::sqrt(rr);
  int cnt = 0;
  if (denom == 0.0) {
    history[cnt++] = 0.0;
    *n_history = cnt;
    return SMG_OK;
  }
  history[cnt++] = std::sqrt(rr) / denom;
  if (history[0] <= rtol) {
    *n_history = cnt;
    return SMG_OK;
  }
  SMG_TRY(precond(r, z));
  SMG_CUDA(cudaMemcpyAsync(d, z, sizeof(double) * (size_t)n, cudaMemcpyDeviceToDevice, st));
  double rz = 0;
  SMG_TRY(dots.dot(n, r, z, st, &rz));
  for (int k = 0; k < maxit; ++k) {
    EpiArgs em;
    em.out = q;
    SMG_CUDA(launch_csr_stream(A.a, d, Epi::kSpmv, em, st));
    double curvature = 0;
    SMG_TRY(dots.dot(n, d, q, st, &curvature));
    if (curvature <= 0.0) {
      if (bad_iteration) *bad_iteration = k;
      if (bad_curvature) *bad_curvature = curvature;
      *n_history = cnt;
      char buf[160];
      snprintf(buf, sizeof buf,
               "non-positive curvature p'Ap = %.6e at CG iteration %d; operator is not positive definite",
               curvature, k);
      set_error(buf);
      return SMG_ERR_INDEFINITE;
    }
    const double alpha = rz / curvature;
    SMG_CUDA(launch_axpby(n, alpha, d, 0.0, x, 0, st));
    SMG_CUDA(launch_axpby(n, alpha, q, 0.0, r, 1, st));
    SMG_TRY(dots.dot(n, r, r, st, &rr));
    history[cnt++] = std::sqrt(rr) / denom;
    if (history[cnt - 1] <= rtol) break;
    SMG_TRY(precond(r, z));
    double rz_new = 0;
    SMG_TRY(dots.dot(n, r, z, st, &rz_new));
    SMG_CUDA(launch_axpby(n, 0.0, z, rz_new / rz, d, 2, st));
    rz = rz_new;
  }
  *n_history = cnt;
  return SMG_OK;
}

int smg_dot(int64_t n, const double* x, const double* y, double* result_host, void* stream)
{
  if (!result_host) return fail("result is NULL");
  std::lock_guard<std::mutex> lk(g_scratch_mu);
  return g_dots.dot(n, x, y, as_stream(stream), result_host);
}

}  // extern "C"
