"""Several local-correction regions on one level, pinned to the reference.

SURVEY.md A4: the regions of a LocalCorrection are DOF-disjoint
(smoothers.py:190-192) but may be coupled through A; S_c is additive, so every
region's residual must be formed from the pre-correction u
(smoothers.py:203-211, one shared residual).  The fixtures come from the
reference itself (tests/golden/make_golden.py ``multi_region``): two flattened
vertices 4 cells apart on a 16x16 grid give two coupled regions (P1 and P2);
three far-apart vertices give uncoupled ones (the reference's own
test_smoothers.py:89-99 case, on a mesh).

Every mode the library has for the corrections is compared with the
reference's golden outputs at 1e-12 (they pass through dense Cholesky solves):
the default path (for coupled regions: a residual-only pass for every region,
then the solves from the stored residuals -- patch_kernel<kResidualOnly> +
<kSolveFromBuf>), corrections overlapped with the interior rows of the
adjacent sweep (option 2), and corrections that follow their producer
(option 3, SMG_LC_FOLLOW rings).
"""

import ctypes

import numpy as np
import pytest

from tests.golden import fixtures

pytestmark = pytest.mark.gpu

TOL_DENSE = 1e-12
MULTI = sorted(fixtures.MULTI_REGION_FIXTURES)


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(scope="module", params=MULTI)
def fx(request):
    z, h = fixtures.load(request.param)
    return request.param, z, h


def test_fixture_shape(fx):
    name, z, h = fx
    lc = h.levels[0].local_correction
    assert lc is not None and lc.n_regions >= 2
    assert bool(int(z["coupled"])) == fixtures.MULTI_REGION_FIXTURES[name]


def test_library_detects_coupling(fx):
    """smg_correction_info reports coupled=1 exactly when the reference's
    regions are coupled through A (upload-time check)."""
    from paper_2402_12947_b200 import _lib, device as D
    name, z, h = fx
    lv = h.levels[0]
    dc = D.device_correction(lv.a, lv.local_correction)
    lib = _lib.load()
    nreg, cov, cpl, byt = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int(), ctypes.c_int64()
    _lib.check(lib.smg_correction_info(dc.handle, ctypes.byref(nreg), ctypes.byref(cov),
                                       ctypes.byref(cpl), ctypes.byref(byt)))
    assert nreg.value == lv.local_correction.n_regions
    assert cov.value == sum(len(i) for i, _ in lv.local_correction.regions)
    assert bool(cpl.value) == bool(int(z["coupled"]))


def test_apply_and_sandwich_vs_reference(fx):
    import paper_2402_12947_b200 as P
    name, z, h = fx
    lv = h.levels[0]
    out = P.apply_local_correction(lv.local_correction, z["g/residual"])
    assert rel(out, z["g/lc_apply"]) <= TOL_DENSE
    outside = np.ones(len(out), dtype=bool)
    outside[lv.local_correction.covered_dofs] = False
    assert np.all(out[outside] == 0.0)
    u = z["g/u_rand"].copy()
    P.combined_smooth(lv.a, z["g/b"], u, lv.local_correction, lv.smoother)
    assert rel(u, z["g/combined"]) <= TOL_DENSE


def test_additive_not_multiplicative(fx):
    """Coupled regions: applying the regions one after another (each seeing
    the previous region's update) would differ from the reference; the GPU
    result must be the additive one."""
    import paper_2402_12947_b200 as P
    from oracle import oracle as O
    name, z, h = fx
    lv = h.levels[0]
    b, ur = z["g/b"], z["g/u_rand"]
    seq = ur.copy()
    for idx, fac in lv.local_correction.regions:
        r = b - O.spmv(lv.a, seq)
        seq[idx] += O.chol_solve(fac, r[idx])
    add = ur + O.apply_local_correction(lv.local_correction, b - O.spmv(lv.a, ur))
    gpu = ur + P.apply_local_correction(lv.local_correction, b - O.spmv(lv.a, ur))
    assert rel(gpu, add) <= TOL_DENSE
    if z["coupled"]:
        assert rel(seq, add) > 1e-6, "fixture regions should interact through A"


@pytest.mark.parametrize("mode", ["default", "overlap", "follow"])
@pytest.mark.parametrize("graphs", [True, False])
def test_vcycle_modes_vs_reference(fx, mode, graphs, monkeypatch):
    import torch
    from paper_2402_12947_b200 import device as D
    from paper_2402_12947_b200.mg import DeviceHierarchy
    name, z, h = fx
    if mode == "follow":
        monkeypatch.setenv("SMG_LC_FOLLOW", "1")   # rings are built on request only
        monkeypatch.setattr(D, "_corr_cache", {})
    dh = DeviceHierarchy(h.levels, h.coarse_factor, use_graphs=graphs)
    if mode == "overlap":
        dh.set_option(2, 1)
    elif mode == "follow":
        dh.set_option(3, 1)
    b = torch.from_numpy(z["g/b"]).cuda()
    u = torch.from_numpy(z["g/u_rand"]).cuda()
    dh.vcycle(b, u)
    assert rel(u.cpu().numpy(), z["g/vcycle1"]) <= TOL_DENSE
    dh.vcycle(b, u)
    assert rel(u.cpu().numpy(), z["g/vcycle2"]) <= TOL_DENSE
    u0 = torch.zeros_like(b)
    dh.vcycle(b, u0)
    assert rel(u0.cpu().numpy(), z["g/vcycle_zero"]) <= TOL_DENSE


def test_counts_vs_reference(fx):
    import paper_2402_12947_b200 as P
    name, z, h = fx
    b = z["g/b"]
    _, hist = P.solve_stationary(h, b, z["g/u0"], 1e-10, 300)
    assert len(hist) - 1 == int(z["g/stat_iters"])
    _, ch = P.cg(h.levels[0].a, b, precond=P.as_preconditioner(h), rtol=1e-10, maxit=300)
    assert len(ch) - 1 == int(z["g/cg_iters"])
