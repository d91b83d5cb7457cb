"""GPU parity against the reference's golden vectors and the oracle.

Every call goes through the C-ABI library (paper_2402_12947_b200/lib) on
cuda:0.  Bars (stated per test): bitwise for SpMV, residual, restriction,
prolong-add and every smoother sweep; <= 1e-12 relative for anything that
includes a dense Cholesky solve (patch / coarse); identical stationary and
CG iteration counts at rtol 1e-10; bit-identical reruns (criterion 10).
"""

import numpy as np
import pytest

from tests.golden import fixtures

pytestmark = pytest.mark.gpu

NAMES = fixtures.HIERARCHY_FIXTURES
TOL_DENSE = 1e-12


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(scope="module")
def P():
    import paper_2402_12947_b200 as P
    return P


@pytest.fixture(scope="module", params=NAMES)
def fx(request):
    from tests.golden import fixtures
    z, h = fixtures.load(request.param)
    return request.param, z, h


def test_library_is_the_compute_path(P):
    from paper_2402_12947_b200 import _lib
    lib = _lib.load()
    import ctypes
    sm, l2, ma, mi = ctypes.c_int(), ctypes.c_int64(), ctypes.c_int(), ctypes.c_int()
    _lib.check(lib.smg_device_info(ctypes.byref(sm), ctypes.byref(l2), ctypes.byref(ma),
                                   ctypes.byref(mi)))
    assert (ma.value, mi.value) == (10, 0), "expected a B200 (sm_100)"


def test_sparse_ops_bitwise(P, fx):
    import torch
    name, z, h = fx
    lv = h.levels[0]
    ur, b = z["g/u_rand"], z["g/b"]
    assert np.array_equal(P.spmv(lv.a, ur), z["g/spmv"])
    from paper_2402_12947_b200 import _lib, device as D
    lib = _lib.load()
    op = D.device_operator(lv.a)
    bt = torch.from_numpy(b).cuda()
    ut = torch.from_numpy(ur).cuda()
    r = torch.empty_like(bt)
    _lib.check(lib.smg_residual(op.handle, D.ptr(bt), D.ptr(ut), D.ptr(r), D.stream_handle()))
    assert np.array_equal(r.cpu().numpy(), z["g/residual"])
    pop = D.device_operator(lv.prolongation.matrix, with_transpose=True)
    y = torch.empty(pop.ncols, dtype=torch.float64, device="cuda")
    _lib.check(lib.smg_spmv_transpose(pop.handle, D.ptr(ut), D.ptr(y), D.stream_handle()))
    assert np.array_equal(y.cpu().numpy(), z["g/restrict"])
    uf = ut.clone()
    uc = torch.from_numpy(z["g/uc"]).cuda()
    _lib.check(lib.smg_prolong_add(pop.handle, D.ptr(uc), D.ptr(uf), D.stream_handle()))
    assert np.array_equal(uf.cpu().numpy(), z["g/prolong_add"])


def test_per_sweep_bitwise(P, fx):
    name, z, h = fx
    lv = h.levels[0]
    for k in range(1, lv.smoother.sweeps + 1):
        u = z["g/u_rand"].copy()
        P.chebyshev_smooth(lv.a, z["g/b"], u, k, lv.smoother)
        assert np.array_equal(u, z[f"g/cheb{k}"]), f"{name}: sweep {k}"


def test_every_level_sweep_and_spmv_bitwise(P, fx):
    """Coarse Galerkin levels have long rows (multi-chunk tiles when they
    average >= 24 nonzeros per row): their SpMV and sweeps are bitwise too."""
    from oracle import oracle as O
    name, z, h = fx
    rng = np.random.default_rng(8)
    for l, lv in enumerate(h.levels[:-1]):
        n = lv.a.nrows
        x, b = rng.standard_normal(n), rng.standard_normal(n)
        assert np.array_equal(P.spmv(lv.a, x), O.spmv(lv.a, x)), f"{name} level {l}"
        u = x.copy()
        P.chebyshev_smooth(lv.a, b, u, lv.smoother.sweeps, lv.smoother)
        assert np.array_equal(u, O.global_smooth(lv.a, b, x.copy(), lv.smoother)), \
            f"{name} level {l} sweeps"


def test_sandwich_and_local_correction(P, fx):
    name, z, h = fx
    lv = h.levels[0]
    b, ur = z["g/b"], z["g/u_rand"]
    u = ur.copy()
    P.combined_smooth(lv.a, b, u, lv.local_correction, lv.smoother)
    assert rel(u, z["g/combined"]) <= TOL_DENSE
    if "g/lc_apply" in z:
        out = P.apply_local_correction(lv.local_correction, z["g/residual"])
        assert rel(out, z["g/lc_apply"]) <= TOL_DENSE
        outside = np.ones(len(out), dtype=bool)
        outside[lv.local_correction.covered_dofs] = False
        assert np.all(out[outside] == 0.0)


def test_vcycles(P, fx):
    name, z, h = fx
    b, ur = z["g/b"], z["g/u_rand"]
    v1 = ur.copy()
    P.vcycle(h, b, v1)
    assert rel(v1, z["g/vcycle1"]) <= TOL_DENSE
    v2 = v1.copy()
    P.vcycle(h, b, v2)
    assert rel(v2, z["g/vcycle2"]) <= TOL_DENSE
    v0 = np.zeros(len(b))
    P.vcycle(h, b, v0)
    assert rel(v0, z["g/vcycle_zero"]) <= TOL_DENSE


def test_vcycle_matches_oracle_and_is_deterministic(P, fx):
    from oracle import oracle as O
    name, z, h = fx
    b, ur = z["g/b"], z["g/u_rand"]
    ref = O.vcycle(h, b, ur.copy())
    outs = []
    for _ in range(3):
        u = ur.copy()
        P.vcycle(h, b, u)
        outs.append(u)
    assert rel(outs[0], ref) <= TOL_DENSE
    assert all(np.array_equal(outs[0], o) for o in outs[1:]), "reruns must be bit-identical"


def test_graph_and_eager_agree_bitwise(P, fx):
    import torch
    from paper_2402_12947_b200.mg import DeviceHierarchy
    name, z, h = fx
    b = torch.from_numpy(z["g/b"]).cuda()
    res = []
    for graphs in (True, False):
        dh = DeviceHierarchy(h.levels, h.coarse_factor, use_graphs=graphs)
        u = torch.from_numpy(z["g/u_rand"]).cuda()
        dh.vcycle(b, u)
        dh.vcycle(b, u)
        res.append(u.cpu().numpy())
    assert np.array_equal(res[0], res[1])


def test_zero_guess_fusion_is_bitwise(P, fx):
    import torch
    from paper_2402_12947_b200.mg import DeviceHierarchy
    name, z, h = fx
    b = torch.from_numpy(z["g/b"]).cuda()
    res = []
    for fuse in (1, 0):
        dh = DeviceHierarchy(h.levels, h.coarse_factor)
        dh.set_option(1, fuse)
        u = torch.from_numpy(z["g/u_rand"]).cuda()
        dh.vcycle(b, u)
        dh.vcycle(b, u)
        res.append(u.cpu().numpy())
    assert np.array_equal(res[0], res[1])


@pytest.mark.parametrize("graphs", [True, False])
def test_lc_overlap_is_bitwise(P, fx, graphs):
    """Local corrections running concurrently with the interior rows of the
    adjacent sweep (halo rows after) give the sequential result bit for bit."""
    import torch
    from paper_2402_12947_b200.mg import DeviceHierarchy
    name, z, h = fx
    b = torch.from_numpy(z["g/b"]).cuda()
    res, launches = [], []
    for overlap in (1, 0):
        dh = DeviceHierarchy(h.levels, h.coarse_factor, use_graphs=graphs)
        dh.set_option(2, overlap)
        u = torch.from_numpy(z["g/u_rand"]).cuda()
        dh.vcycle(b, u)
        dh.vcycle(b, u)
        res.append(u.cpu().numpy())
        launches.append(dh.launches_per_vcycle())
    assert np.array_equal(res[0], res[1])
    has_lc = any(lv.local_correction is not None and lv.local_correction.regions
                 for lv in h.levels)
    if has_lc:  # the fixtures' halos are a few % of the rows: the split is active
        assert launches[0] > launches[1]


@pytest.mark.parametrize("graphs", [True, False])
def test_lc_follow_is_bitwise(P, fx, graphs, monkeypatch):
    """Corrections overlapped with the kernel producing their u (last smoother
    step, prolong-add; SMG_OPT_LC_FOLLOW) give the sequential V-cycle bit for
    bit, over repeated cycles, and stay within 1e-12 of the oracle."""
    import torch
    from oracle import oracle as O
    from paper_2402_12947_b200.mg import DeviceHierarchy
    name, z, h = fx
    from paper_2402_12947_b200 import device as D
    monkeypatch.setenv("SMG_LC_FOLLOW", "1")   # build the rings (opt-in) ...
    monkeypatch.setattr(D, "_corr_cache", {})  # ... on freshly created corrections
    b = torch.from_numpy(z["g/b"]).cuda()
    res, launches = [], []
    for follow in (1, 0):
        dh = DeviceHierarchy(h.levels, h.coarse_factor, use_graphs=graphs)
        dh.set_option(3, follow)
        u = torch.from_numpy(z["g/u_rand"]).cuda()
        for _ in range(3):
            dh.vcycle(b, u)
        res.append(u.cpu().numpy())
        launches.append(dh.launches_per_vcycle())
    assert np.array_equal(res[0], res[1])
    # a followed correction is one kernel; a coupled correction's plain path is
    # two (residual-only pass, then the solves)
    if fixtures.MULTI_REGION_FIXTURES.get(name):
        assert launches[0] < launches[1]
    else:
        assert launches[0] == launches[1]
    ref = z["g/u_rand"].copy()
    for _ in range(3):
        ref = O.vcycle(h, z["g/b"], ref)
    assert rel(res[0], ref) <= TOL_DENSE


def test_lc_follow_coupled_regions(P, monkeypatch):
    """Two regions coupled through A whose rings overlap: each
    follow-mode correction still sees the pre-correction u (bitwise equal to
    the sequential path)."""
    import torch
    from tests.golden import fixtures
    from paper_2402_12947_b200.mg import DeviceHierarchy
    from paper_2402_12947_b200 import smoothers as S
    from paper_2402_12947_b200 import device as D
    monkeypatch.setenv("SMG_LC_FOLLOW", "1")   # build the rings (opt-in) ...
    monkeypatch.setattr(D, "_corr_cache", {})  # ... on freshly created corrections
    z, h = fixtures.load("c1s")
    lv0 = h.levels[0]
    n = lv0.a.nrows
    # adjacent dof sets: rows 40..47 and their first unclaimed neighbours
    rp, ci = lv0.a.row_offsets, lv0.a.col_indices
    b1 = list(range(n // 2, n // 2 + 6))
    nb = sorted({int(c) for r in b1 for c in ci[rp[r]:rp[r + 1]]} - set(b1))[:6]
    corr = S.build_local_correction(lv0.a, [np.array(b1), np.array(nb)])
    levels = list(h.levels)
    import dataclasses
    levels[0] = dataclasses.replace(lv0, local_correction=corr)
    b = torch.from_numpy(z["g/b"]).cuda()
    res = []
    for follow in (1, 0):
        dh = DeviceHierarchy(levels, h.coarse_factor)
        dh.set_option(3, follow)
        u = torch.from_numpy(z["g/u_rand"]).cuda()
        for _ in range(2):
            dh.vcycle(b, u)
        res.append(u.cpu().numpy())
    assert np.array_equal(res[0], res[1])


def test_pipelined_host_vcycles_match_single_calls(P, fx):
    """smg_vcycle_host_many (copies overlapping V-cycles, two staging slots)
    gives every pair exactly the single-call result."""
    import torch
    from paper_2402_12947_b200.mg import DeviceHierarchy
    name, z, h = fx
    n = h.levels[0].a.nrows
    dh = DeviceHierarchy(h.levels, h.coarse_factor)
    rng = np.random.default_rng(11)
    bs = [torch.from_numpy(rng.standard_normal(n)).pin_memory().numpy() for _ in range(5)]
    us = [torch.from_numpy(rng.standard_normal(n)).pin_memory().numpy() for _ in range(5)]
    expect = []
    for b, u in zip(bs, us):
        ud = torch.from_numpy(u.copy()).cuda()
        dh.vcycle(torch.from_numpy(b).cuda(), ud)
        expect.append(ud.cpu().numpy())
    dh.vcycles_host(bs, us)
    for u, e in zip(us, expect):
        assert np.array_equal(u, e)
    with pytest.raises(ValueError, match="dimension mismatch"):
        dh.vcycles_host(bs[:2], us[:1])


def test_iteration_counts(P, fx):
    name, z, h = fx
    b = z["g/b"]
    u, hist = P.solve_stationary(h, b, z["g/u0"], 1e-10, 300)
    assert len(hist) - 1 == int(z["g/stat_iters"])
    np.testing.assert_allclose(hist, z["g/stat_hist"], rtol=1e-3)
    assert rel(u, z["g/stat_u"]) <= 1e-10
    x, ch = P.cg(h.levels[0].a, b, precond=P.as_preconditioner(h), rtol=1e-10, maxit=300)
    assert len(ch) - 1 == int(z["g/cg_iters"])
    np.testing.assert_allclose(ch, z["g/cg_hist"], rtol=1e-6)
    assert rel(x, z["g/cg_x"]) <= 1e-10


def test_criterion7_unadjusted_count(P):
    from dataclasses import replace
    from tests.golden import fixtures
    z, h = fixtures.load("crit7_adj")
    for lv, lam in zip(h.levels, z["lambda_max"]):
        lv.smoother = replace(lv.smoother, lambda_max=float(lam))
    _, hist = P.solve_stationary(h, z["g/b"], z["g/u0"], 1e-10, 300)
    assert len(hist) - 1 == int(z["unadjusted_stat_iters"]) == 17


def test_c5_patch_solves(P):
    from tests.test_oracle_golden import load_c5p
    z, lc = load_c5p()
    out = P.apply_local_correction(lc, z["r"])
    assert rel(out, z["lc_apply"]) <= 1e-13


def test_jacobi_config_is_reference_delta_zero_branch(P):
    from tests.golden import fixtures
    z, h = fixtures.load("c1s")
    lv = h.levels[0]
    u = z["g/u_rand"].copy()
    P.chebyshev_smooth(lv.a, z["g/b"], u, 2, P.SmootherConfig("jacobi", 2, omega=2.0 / 3.0))
    assert np.array_equal(u, z["g/cheb2"])


def test_torch_inplace_path(P):
    import torch
    from tests.golden import fixtures
    z, h = fixtures.load("c2s")
    lv = h.levels[0]
    b = torch.from_numpy(z["g/b"]).cuda()
    u = torch.from_numpy(z["g/u_rand"]).cuda()
    ptr = u.data_ptr()
    P.chebyshev_smooth(lv.a, b, u, 3, lv.smoother)
    assert u.data_ptr() == ptr
    assert np.array_equal(u.cpu().numpy(), z["g/cheb3"])
    v = torch.from_numpy(z["g/u_rand"]).cuda()
    P.vcycle(h, b, v)
    assert rel(v.cpu().numpy(), z["g/vcycle1"]) <= TOL_DENSE


def test_error_behaviour(P):
    from paper_2402_12947_b200.sparse import CsrMatrix
    a = CsrMatrix.from_dense(np.diag([2.0, 0.0, 3.0]) + np.eye(3, k=1) + np.eye(3, k=-1))
    with pytest.raises(P.ZeroDiagonalError) as e:
        P.chebyshev_smooth(a, np.ones(3), np.zeros(3), 1, P.SmootherConfig("chebyshev", 1, 1.0))
    assert e.value.row == 1
    good = CsrMatrix.from_dense(np.diag([2.0, 2.0, 3.0]))
    with pytest.raises(ValueError, match="positive cfg.lambda_max"):
        P.chebyshev_smooth(good, np.ones(3), np.zeros(3), 1, P.SmootherConfig("chebyshev", 1))
    with pytest.raises(ValueError, match="dimension mismatch"):
        P.spmv(good, np.ones(4))
    with pytest.raises(NotImplementedError):
        P.combined_smooth(good, np.ones(3), np.zeros(3), None, P.SmootherConfig("sgs", 1))
    indef = CsrMatrix.from_dense(np.diag([1.0, -1.0]))
    with pytest.raises(P.IndefiniteOperatorError):
        P.cg(indef, np.array([1.0, 1.0]))


def test_edge_cases(P):
    from paper_2402_12947_b200.sparse import CsrMatrix
    # empty rows, a dense row longer than one tile, and a 0x0 operator
    n = 5000
    rows = [np.zeros(n, dtype=np.int64)]
    cols = [np.arange(n)]
    vals = [np.random.default_rng(0).standard_normal(n)]
    rows.append(np.arange(2, n))
    cols.append(np.arange(2, n))
    vals.append(np.full(n - 2, 4.0))
    a = CsrMatrix.from_coo(n, n, np.concatenate(rows), np.concatenate(cols), np.concatenate(vals))
    x = np.random.default_rng(1).standard_normal(n)
    from oracle import oracle as O
    assert np.array_equal(P.spmv(a, x), O.spmv(a, x))
    assert P.spmv(a, x)[1] == 0.0
    e = CsrMatrix(0, 0, np.array([0]), np.zeros(0, dtype=np.int64), np.zeros(0))
    assert P.spmv(e, np.zeros(0)).shape == (0,)
    # no regions: combined_smooth == chebyshev_smooth (test_smoothers.py:278-287)
    from tests.golden import fixtures
    z, h = fixtures.load("c2s")
    lv = h.levels[0]
    u1 = z["g/u_rand"].copy()
    P.combined_smooth(lv.a, z["g/b"], u1, None, lv.smoother)
    assert np.array_equal(u1, z["g/cheb3"])


def test_long_row_operators_multichunk(P):
    """Operators averaging >= 24 nonzeros per row use multi-chunk tiles
    (double-buffered chunks); a single row longer than a whole tile spans
    many chunks.  SpMV and smoother sweeps stay bit-identical."""
    from paper_2402_12947_b200.sparse import CsrMatrix
    from oracle import oracle as O
    n, w = 12000, 40
    rng = np.random.default_rng(3)
    r, c = [], []
    for k in range(-w, w + 1):
        i = np.arange(max(0, -k), min(n, n - k))
        r.append(i)
        c.append(i + k)
    r.append(np.zeros(n, dtype=np.int64))          # row 0: dense, 12000 nonzeros
    c.append(np.arange(n))
    rr, cc = np.concatenate(r), np.concatenate(c)
    key = np.unique(rr * n + cc)
    rr, cc = key // n, key % n
    vals = rng.uniform(-1, 1, len(rr))
    vals[rr == cc] = 4.0 * w + 1.0
    a = CsrMatrix.from_coo(n, n, rr, cc, vals)
    assert a.nnz >= 24 * n
    x = rng.standard_normal(n)
    assert np.array_equal(P.spmv(a, x), O.spmv(a, x))
    b = rng.standard_normal(n)
    cfg = P.SmootherConfig("chebyshev", 3, lambda_max=2.0)
    u = x.copy()
    P.chebyshev_smooth(a, b, u, 3, cfg)
    assert np.array_equal(u, O.global_smooth(a, b, x.copy(), cfg))


def test_coarse_solve_vs_reference(P, fx):
    """The coarse solve the V-cycle performs (A_L^-1 from the reference's
    factor, symmetric tiles, deterministic reduction) against the reference's
    own h.coarse_factor.solve (LAPACK dpotrs, mg.py:145) at a fixed bar, and
    bit-identical on reruns."""
    from paper_2402_12947_b200.mg import DeviceHierarchy
    name, z, h = fx
    dh = DeviceHierarchy(h.levels, h.coarse_factor)
    x = dh.coarse_solve(z["g/coarse_b"])
    assert rel(x, z["g/coarse_x"]) <= TOL_DENSE
    assert np.array_equal(x, dh.coarse_solve(z["g/coarse_b"]))
