"""Every device layout of the sweep operators gives the same bits.

The sweeps, residuals and transfers run on one of three layouts chosen per
operator at upload (offset-table CSR tiles, fixed-capacity CSR tiles,
SELL-32-sigma256 with a 4/8/16-deep loop and int32 or 16-bit delta-coded
columns, SELL-8x4 with 2/4 batches in flight).  The fixtures
are small, so the automatic rule picks tiles for them; here each layout is
forced with smg_operator_set_layout and checked against the reference's golden
vectors and the oracle: bitwise for SpMV-type work and every smoother sweep,
and the whole V-cycle must come out bit-identical across layouts.
"""

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

NAMES = ["crit7_adj", "c1s", "c2s", "c3s"]
LAYOUTS = [(0, 0), (1, 0), (2, 4), (2, 8), (2, 16), (3, 2), (3, 4), (4, 4), (4, 8), (4, 16), (5, 0)]


def fresh(m):
    """A new host object, so the device-operator cache uploads it afresh."""
    from paper_2402_12947_b200.sparse import CsrMatrix
    return CsrMatrix(m.nrows, m.ncols, np.array(m.row_offsets), np.array(m.col_indices),
                     np.array(m.values))


def forced(m, layout, unroll, with_transpose=False):
    from paper_2402_12947_b200 import _lib
    from paper_2402_12947_b200 import device as D
    op = D.device_operator(m, with_transpose=with_transpose)
    lib = _lib.load()
    _lib.check(lib.smg_operator_set_layout(op.handle, layout, unroll))
    lay, unr = ctypes.c_int(), ctypes.c_int()
    _lib.check(lib.smg_operator_layout(op.handle, ctypes.byref(lay), ctypes.byref(unr)))
    assert lay.value == layout
    if layout in (2, 3, 4):
        assert unr.value == unroll
    return op


@pytest.mark.parametrize("layout,unroll", LAYOUTS)
@pytest.mark.parametrize("name", NAMES)
def test_layout_sparse_ops_and_sweeps_bitwise(name, layout, unroll):
    import torch
    import paper_2402_12947_b200 as P
    from oracle import oracle as O
    from paper_2402_12947_b200 import _lib
    from paper_2402_12947_b200 import device as D
    from tests.golden import fixtures
    z, h = fixtures.load(name)
    lv = h.levels[0]
    a = fresh(lv.a)
    pm = fresh(lv.prolongation.matrix)
    forced(a, layout, unroll)
    pop = forced(pm, layout, unroll, with_transpose=True)
    ur, b = z["g/u_rand"], z["g/b"]
    assert np.array_equal(P.spmv(a, ur), z["g/spmv"])
    for k in range(1, lv.smoother.sweeps + 1):
        u = ur.copy()
        P.chebyshev_smooth(a, b, u, k, lv.smoother)
        assert np.array_equal(u, z[f"g/cheb{k}"]), f"sweep {k}"
    lib = _lib.load()
    rt = torch.from_numpy(ur).cuda()
    y = torch.empty(pm.ncols, dtype=torch.float64, device="cuda")
    _lib.check(lib.smg_spmv_transpose(pop.handle, D.ptr(rt), D.ptr(y), D.stream_handle()))
    assert np.array_equal(y.cpu().numpy(), z["g/restrict"])
    uc = torch.from_numpy(z["g/uc"]).cuda()
    _lib.check(lib.smg_prolong_add(pop.handle, D.ptr(uc), D.ptr(rt), D.stream_handle()))
    assert np.array_equal(rt.cpu().numpy(), z["g/prolong_add"])
    # every coarser operator too (Galerkin products: long rows)
    for l, lvl in enumerate(h.levels[1:-1], start=1):
        al = fresh(lvl.a)
        forced(al, layout, unroll)
        x = np.random.default_rng(l).standard_normal(al.ncols)
        assert np.array_equal(P.spmv(al, x), O.spmv(lvl.a, x)), f"level {l}"


@pytest.mark.parametrize("name", NAMES)
def test_vcycle_identical_across_layouts(name):
    from dataclasses import replace
    from paper_2402_12947_b200.mg import DeviceHierarchy, Level, Prolongation
    from tests.golden import fixtures
    z, h = fixtures.load(name)
    outs = []
    for layout, unroll in LAYOUTS:
        levels = []
        for lv in h.levels:
            a = fresh(lv.a)
            forced(a, layout, unroll)
            prol = None
            if lv.prolongation is not None:
                pm = fresh(lv.prolongation.matrix)
                forced(pm, layout, unroll, with_transpose=True)
                prol = Prolongation(pm, lv.prolongation.fine_level, lv.prolongation.coarse_level)
            levels.append(replace(lv, a=a, prolongation=prol))
        dh = DeviceHierarchy(levels, h.coarse_factor)
        u = z["g/u_rand"].copy()
        dh.vcycle(z["g/b"], u)
        outs.append(u)
        ref = z["g/vcycle1"]
        assert np.linalg.norm(u - ref) <= 1e-12 * np.linalg.norm(ref)
    for u in outs[1:]:
        assert np.array_equal(u, outs[0])


@pytest.mark.parametrize("name", ["c2s", "c4s", "cpl_p2", "crit7_adj", "c3s"])
@pytest.mark.parametrize("mask", ["1", "3", "0x7"])
def test_renumbered_levels_are_bitwise(name, mask, monkeypatch):
    """Locality renumbering (SMG_RENUMBER bit mask of levels; reverse
    Cuthill-McKee of each renamed level) only renames rows and columns --
    every row keeps its entries in the reference's column order, CSR(P^T)
    keeps ascending original fine rows, the patch factors keep their rows --
    so V-cycles, stationary histories and CG counts are bit-identical to the
    plain hierarchy's, and equal the reference's outputs."""
    import torch
    from paper_2402_12947_b200.mg import DeviceHierarchy
    from tests.golden import fixtures
    z, h = fixtures.load(name)
    b = torch.from_numpy(z["g/b"]).cuda()
    res = []
    for m in ("0", mask):
        monkeypatch.setenv("SMG_RENUMBER", m)
        for graphs in (True, False):
            dh = DeviceHierarchy(h.levels, h.coarse_factor, use_graphs=graphs)
            u = torch.from_numpy(z["g/u_rand"]).cuda()
            dh.vcycle(b, u)
            dh.vcycle(b, u)
            res.append(u.cpu().numpy())
        _, hist = dh.solve_stationary(z["g/b"], z["g/u0"], 1e-10, 300)
        assert len(hist) - 1 == int(z["g/stat_iters"])
        res.append(np.array(hist))
    assert np.array_equal(res[0], res[1])
    assert np.array_equal(res[0], res[3]) and np.array_equal(res[1], res[4])
    assert np.array_equal(res[2], res[5])
    assert np.linalg.norm(res[3] - z["g/vcycle2"]) <= 1e-12 * np.linalg.norm(z["g/vcycle2"])


@pytest.mark.parametrize("nrows,per_row,want", [
    (30_000, 40, 5),     # L2-resident long rows, one-wave tiles of 3,072 products: staged by the rule
    (30_000, 8, 1),      # short rows: fixed-capacity tiles
    (120_000, 40, 0),    # one-wave tiles of 11.5k products: past SMG_STAGE_MAX_CAP, chunked offset-table tiles
])
def test_rule_picks_the_staged_layout_for_small_long_row_operators(nrows, per_row, want):
    """The upload rule (capi.cu build_devcsr): long-row operators that stay in
    L2 and fit one resident wave of small tiles run csr_stage_kernel; the result
    is the oracle's bit for bit whatever the rule picks."""
    import paper_2402_12947_b200 as P
    from oracle import oracle as O
    from paper_2402_12947_b200 import _lib
    from paper_2402_12947_b200 import device as D
    from paper_2402_12947_b200.sparse import CsrMatrix
    rng = np.random.default_rng(nrows + per_row)
    counts = rng.integers(per_row - per_row // 4, per_row + per_row // 4 + 1, size=nrows)
    rp = np.zeros(nrows + 1, dtype=np.int64)
    np.cumsum(counts, out=rp[1:])
    cols = np.empty(rp[-1], dtype=np.int64)
    for r in range(nrows):   # sorted unique columns near the diagonal
        lo = max(0, min(r - counts[r], nrows - 2 * counts[r] - 1))
        cols[rp[r]:rp[r + 1]] = lo + np.sort(rng.choice(2 * counts[r], size=counts[r], replace=False))
    a = CsrMatrix(nrows, nrows, rp, cols, rng.standard_normal(rp[-1]))
    op = D.device_operator(a)
    lib = _lib.load()
    lay, unr = ctypes.c_int(), ctypes.c_int()
    _lib.check(lib.smg_operator_layout(op.handle, ctypes.byref(lay), ctypes.byref(unr)))
    assert lay.value == want
    x = rng.standard_normal(nrows)
    assert np.array_equal(P.spmv(a, x), O.spmv(a, x))
