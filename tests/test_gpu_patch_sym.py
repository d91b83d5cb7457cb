"""Symmetric-inverse local corrections (regions past the whole-L^{-1} sizes
apply the packed lower triangle of A[B,B]^{-1} in one HBM pass) against the
reference's LAPACK solves (smoothers.py:203-211, sparse.py:225-231).

Bars: <= 1e-13 relative on the cond-1e6 C5 blocks (the c5p golden), <= 1e-12
on the mesh fixtures (the north star's per-sweep bar); the substitution path
(SMG_PATCH_SYM=0) is held to the same bars, and every ring geometry must give
the same bits (the chunking never changes a sum's order).
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(scope="module")
def P():
    import paper_2402_12947_b200 as P
    return P


def _fresh_apply(lc_host, a, r):
    """apply_local_correction on a correction uploaded NOW (the slot contents
    depend on SMG_PATCH_SYM at upload)."""
    import ctypes
    import torch
    from paper_2402_12947_b200 import _lib, device as D
    lib = _lib.load()
    op = D.DeviceOperator(a)
    dc = D.DeviceCorrection(op, lc_host)
    rt = torch.from_numpy(np.ascontiguousarray(r)).cuda()
    out = torch.empty_like(rt)
    _lib.check(lib.smg_apply_local_correction(dc.handle, D.ptr(rt), D.ptr(out), D.stream_handle()))
    torch.cuda.synchronize()
    return out.cpu().numpy(), dc


def _c5p_operator(z):
    from paper_2402_12947_b200.sparse import CsrMatrix
    return CsrMatrix.identity(int(z["n"]))


@pytest.mark.parametrize("sym", ["1", "0"])
def test_c5p_blocks_both_paths(P, sym, monkeypatch):
    from tests.test_oracle_golden import load_c5p
    z, lc = load_c5p()
    monkeypatch.setenv("SMG_PATCH_SYM", sym)
    out, _ = _fresh_apply(lc, _c5p_operator(z), z["r"])
    assert rel(out, z["lc_apply"]) <= 1e-13


@pytest.mark.parametrize("fold", ["1", "0"])
@pytest.mark.parametrize("stages", ["2", "3", "4", "6"])
def test_ring_geometry_does_not_change_bits(P, stages, fold, monkeypatch):
    """The depth of the warps' rings only changes when rows arrive, never the
    order of a sum: every depth gives the default depth's bits -- with folded
    chunks (rows c and n-1-c, the default) and with consecutive row pairs."""
    from tests.test_oracle_golden import load_c5p
    z, lc = load_c5p()
    a = _c5p_operator(z)
    monkeypatch.setenv("SMG_SYM_FOLD", fold)
    base, _ = _fresh_apply(lc, a, z["r"])
    monkeypatch.setenv("SMG_SYM_STAGES", stages)
    out, _ = _fresh_apply(lc, a, z["r"])
    assert np.array_equal(out, base)
    assert rel(out, z["lc_apply"]) <= 1e-13


@pytest.mark.parametrize("fold", ["1", "0"])
def test_many_sizes_vs_lapack(P, fold, monkeypatch):
    """Every region size class at once (<= 32: panel, 33..64: L^{-1} block,
    65..: symmetric inverse, including sizes around the chunk boundaries and
    odd sizes) against scipy's cho_solve on cond-1e4 blocks."""
    import scipy.linalg as sl
    from paper_2402_12947_b200.smoothers import LocalCorrection
    from paper_2402_12947_b200.sparse import CsrMatrix, DenseFactor
    monkeypatch.setenv("SMG_SYM_FOLD", fold)
    rng = np.random.default_rng(12947)
    sizes = [1, 2, 31, 32, 33, 63, 64, 65, 66, 90, 127, 128, 129, 130, 191, 255, 256, 257, 300,
             383, 511, 513, 640, 895]
    n = int(sum(sizes)) + 100
    perm = rng.permutation(n)
    regions, start, blocks = [], 0, []
    for nd in sizes:
        idx = np.sort(perm[start:start + nd])
        start += nd
        q, _ = np.linalg.qr(rng.standard_normal((nd, nd)))
        blk = (q * np.logspace(0, -4, nd)) @ q.T
        blk = 0.5 * (blk + blk.T)
        c = sl.cho_factor(blk, lower=True)
        regions.append((idx.astype(np.int64), DenseFactor("cholesky", c, nd)))
        blocks.append((idx, c))
    lc = LocalCorrection(tuple(regions), n)
    r = rng.standard_normal(n)
    out, _ = _fresh_apply(lc, CsrMatrix.identity(n), r)
    want = np.zeros(n)
    for idx, c in blocks:
        want[idx] = sl.cho_solve(c, r[idx])
    for idx, c in blocks:
        assert rel(out[idx], want[idx]) <= 1e-12, f"region of {len(idx)} dofs"
    untouched = np.ones(n, dtype=bool)
    for idx, _ in blocks:
        untouched[idx] = False
    assert not out[untouched].any()


def test_very_large_region_keeps_the_substitution(P):
    """A correction with a region past the symmetric path's size limit (its
    per-warp rings would not fit shared memory) runs the streamed substitution
    for all its regions; same bar."""
    import scipy.linalg as sl
    from paper_2402_12947_b200.smoothers import LocalCorrection
    from paper_2402_12947_b200.sparse import CsrMatrix, DenseFactor
    rng = np.random.default_rng(7)
    sizes = [1000, 300, 40]
    n = sum(sizes) + 10
    perm = rng.permutation(n)
    regions, blocks, start = [], [], 0
    for nd in sizes:
        idx = np.sort(perm[start:start + nd])
        start += nd
        q, _ = np.linalg.qr(rng.standard_normal((nd, nd)))
        blk = (q * np.logspace(0, -3, nd)) @ q.T
        c = sl.cho_factor(0.5 * (blk + blk.T), lower=True)
        regions.append((idx.astype(np.int64), DenseFactor("cholesky", c, nd)))
        blocks.append((idx, c))
    r = rng.standard_normal(n)
    out, _ = _fresh_apply(LocalCorrection(tuple(regions), n), CsrMatrix.identity(n), r)
    for idx, c in blocks:
        assert rel(out[idx], sl.cho_solve(c, r[idx])) <= 1e-12, f"region of {len(idx)} dofs"


@pytest.mark.parametrize("name", ["c4s", "c2s", "cpl_p2"])
@pytest.mark.parametrize("sym", ["1", "0"])
def test_sandwich_vs_reference_both_paths(P, name, sym, monkeypatch):
    """combined_smooth on the fine level with a correction uploaded under each
    setting, against the reference's stored output (c4s: two 279-dof regions,
    the symmetric-inverse path; the others stay on their L^{-1} blocks)."""
    from tests.golden import fixtures
    from paper_2402_12947_b200 import device as D
    monkeypatch.setenv("SMG_PATCH_SYM", sym)
    z, h = fixtures.load(name)
    lv = h.levels[0]
    D._corr_cache.clear()          # upload the correction under this setting
    u = z["g/u_rand"].copy()
    P.combined_smooth(lv.a, z["g/b"], u, lv.local_correction, lv.smoother)
    D._corr_cache.clear()
    assert rel(u, z["g/combined"]) <= 1e-12
