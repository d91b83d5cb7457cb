"""The drop-in boundary's contract.

* "concurrent vcycle calls on distinct arrays over one shared
  Hierarchy are safe": threads sharing one device hierarchy (host arrays and
  CUDA tensors on their own streams) get exactly the sequential results.
* Reference-shaped objects (types.SimpleNamespace with the reference's
  attribute names, mg.py:30-69, sparse.py:47-132, smoothers.py:139-158) are
  accepted by vcycle / combined_smooth / solve_stationary.
* restrict_residual / prolong_add (transfer.py:158-172) bitwise, with the
  reference's error texts; size mismatches raise ValueError instead of
  touching memory out of bounds.
"""

import threading
import types

import numpy as np
import pytest

from tests.golden import fixtures

pytestmark = pytest.mark.gpu

TOL_DENSE = 1e-12


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _inputs(n, k, seed=3):
    g = np.random.default_rng(seed)
    return [(g.standard_normal(n), g.standard_normal(n)) for _ in range(k)]


def test_concurrent_vcycles_host_arrays():
    import paper_2402_12947_b200 as P
    z, h = fixtures.load("c2s")
    dh = P.DeviceHierarchy(h.levels, h.coarse_factor)
    n = h.levels[0].a.nrows
    pairs = _inputs(n, 6)
    expect = []
    for b, u in pairs:
        w = u.copy()
        for _ in range(3):
            dh.vcycle(b, w)
        expect.append(w)
    got = [u.copy() for _, u in pairs]
    errors = []

    def work(i):
        try:
            for _ in range(3):
                dh.vcycle(pairs[i][0], got[i])
        except Exception as e:  # pragma: no cover - reported below
            errors.append(e)

    for _ in range(3):
        got = [u.copy() for _, u in pairs]
        th = [threading.Thread(target=work, args=(i,)) for i in range(len(pairs))]
        for t in th:
            t.start()
        for t in th:
            t.join()
        assert not errors, errors
        for g, e in zip(got, expect):
            assert np.array_equal(g, e)


def test_concurrent_vcycles_device_tensors_on_own_streams():
    import torch
    import paper_2402_12947_b200 as P
    z, h = fixtures.load("c2s")
    dh = P.DeviceHierarchy(h.levels, h.coarse_factor)
    n = h.levels[0].a.nrows
    pairs = _inputs(n, 4, seed=9)
    expect = []
    for b, u in pairs:
        w = u.copy()
        for _ in range(4):
            dh.vcycle(b, w)
        expect.append(w)
    bt = [torch.from_numpy(b).cuda() for b, _ in pairs]
    ut = [torch.from_numpy(u).cuda() for _, u in pairs]
    streams = [torch.cuda.Stream() for _ in pairs]
    torch.cuda.synchronize()
    errors = []

    def work(i):
        try:
            with torch.cuda.stream(streams[i]):
                for _ in range(4):
                    dh.vcycle(bt[i], ut[i])
        except Exception as e:  # pragma: no cover
            errors.append(e)

    th = [threading.Thread(target=work, args=(i,)) for i in range(len(pairs))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    torch.cuda.synchronize()
    assert not errors, errors
    for u, e in zip(ut, expect):
        assert np.array_equal(u.cpu().numpy(), e)


def test_concurrent_solves_and_cg():
    """solve_stationary and CG (which use the hierarchy's residual and dot
    scratch) from two threads: identical histories to the sequential calls."""
    import paper_2402_12947_b200 as P
    z, h = fixtures.load("c1s")
    dh = P.DeviceHierarchy(h.levels, h.coarse_factor)
    b = z["g/b"]
    b2 = np.random.default_rng(4).standard_normal(len(b))
    _, hs = dh.solve_stationary(b, np.zeros(len(b)), 1e-10, 100)
    _, hc = P.cg(h.levels[0].a, b2, precond=dh.as_preconditioner(), rtol=1e-10, maxit=100)
    out = {}

    def stat():
        out["s"] = dh.solve_stationary(b, np.zeros(len(b)), 1e-10, 100)[1]

    def cg():
        out["c"] = P.cg(h.levels[0].a, b2, precond=dh.as_preconditioner(), rtol=1e-10,
                        maxit=100)[1]

    for _ in range(3):
        th = [threading.Thread(target=stat), threading.Thread(target=cg)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        assert out["s"] == hs
        assert out["c"] == hc


def _duck_csr(m):
    return types.SimpleNamespace(nrows=m.nrows, ncols=m.ncols, row_offsets=m.row_offsets,
                                 col_indices=m.col_indices, values=m.values)


def _duck_hierarchy(h):
    """The reference's data model with nothing but attribute names
    (mg.py:30-69; DenseFactor sparse.py:214 = (kind, factor, n))."""
    levels = []
    for lv in h.levels:
        lc = lv.local_correction
        dlc = None
        if lc is not None:
            dlc = types.SimpleNamespace(
                regions=tuple((idx, types.SimpleNamespace(kind="cholesky", factor=f.factor,
                                                          n_local=len(idx)))
                              for idx, f in lc.regions),
                n_global=lc.n_global)
        cfg = lv.smoother
        levels.append(types.SimpleNamespace(
            index=lv.index, mesh=None, dofmap=None, a=_duck_csr(lv.a),
            prolongation=None if lv.prolongation is None else types.SimpleNamespace(
                matrix=_duck_csr(lv.prolongation.matrix), fine_level=lv.index,
                coarse_level=lv.index + 1),
            smoother=types.SimpleNamespace(kind=cfg.kind, sweeps=cfg.sweeps,
                                           lambda_max=cfg.lambda_max,
                                           lambda_min_fraction=cfg.lambda_min_fraction,
                                           adjusted=False),
            regions=None, local_correction=dlc, sgs=None))
    cf = h.coarse_factor
    return types.SimpleNamespace(levels=levels, coarse_factor=types.SimpleNamespace(
        kind="cholesky", factor=cf.factor, n_local=cf.n_local), system=None)


@pytest.mark.parametrize("name", ["crit7_adj", "cpl_p2", "c3s"])
def test_reference_shaped_duck_objects(name):
    import paper_2402_12947_b200 as P
    z, h = fixtures.load(name)
    dh = _duck_hierarchy(h)
    b, ur = z["g/b"], z["g/u_rand"]
    u = ur.copy()
    P.vcycle(dh, b, u)
    assert rel(u, z["g/vcycle1"]) <= TOL_DENSE
    lv = dh.levels[0]
    w = ur.copy()
    P.combined_smooth(lv.a, b, w, lv.local_correction, lv.smoother)
    assert rel(w, z["g/combined"]) <= TOL_DENSE
    w = ur.copy()
    P.chebyshev_smooth(lv.a, b, w, lv.smoother.sweeps, lv.smoother)
    assert np.array_equal(w, z[f"g/cheb{lv.smoother.sweeps}"])
    _, hist = P.solve_stationary(dh, b, z["g/u0"], 1e-10, 300)
    assert len(hist) - 1 == int(z["g/stat_iters"])


@pytest.mark.parametrize("name", ["c2s", "c4s", "cpl_p1"])
def test_restrict_residual_and_prolong_add(name):
    import torch
    import paper_2402_12947_b200 as P
    z, h = fixtures.load(name)
    p = h.levels[0].prolongation
    ur = z["g/u_rand"]
    assert np.array_equal(P.restrict_residual(p, ur), z["g/restrict"])
    uf = ur.copy()
    assert P.prolong_add(p, z["g/uc"], uf) is uf
    assert np.array_equal(uf, z["g/prolong_add"])
    # CUDA tensors: zero-copy, in place
    ut = torch.from_numpy(ur).cuda()
    assert np.array_equal(P.restrict_residual(p, ut).cpu().numpy(), z["g/restrict"])
    P.prolong_add(p, torch.from_numpy(z["g/uc"]).cuda(), ut)
    assert np.array_equal(ut.cpu().numpy(), z["g/prolong_add"])
    with pytest.raises(ValueError, match="does not match fine size"):
        P.restrict_residual(p, ur[:-1])
    with pytest.raises(ValueError, match="does not match"):
        P.prolong_add(p, z["g/uc"][:-1], ur.copy())
    with pytest.raises(ValueError, match="does not match"):
        P.prolong_add(p, z["g/uc"], ur[:-1].copy())


def test_size_mismatches_raise():
    """smg_cg with a preconditioner of another fine size, and a correction
    reused on an operator of another size, raise instead of writing out of
    bounds (reference: ValueError, sparse.py:139, smoothers.py:206-207)."""
    import paper_2402_12947_b200 as P
    z1, h1 = fixtures.load("c1s")
    z3, h3 = fixtures.load("c3s")
    a3 = h3.levels[0].a
    b3 = z3["g/b"]
    with pytest.raises(ValueError, match="does not match"):
        P.cg(a3, b3, precond=P.as_preconditioner(h1), rtol=1e-10, maxit=5)
    lv1 = h1.levels[0]
    with pytest.raises(ValueError, match="does not match"):
        P.combined_smooth(a3, b3, np.zeros(len(b3)), lv1.local_correction, h3.levels[0].smoother)


def test_correction_follows_the_operator_it_is_used_with():
    """One LocalCorrection used with two operators of the same size: the
    patch residuals come from the operator passed in (reference semantics,
    smoothers.py:263-266), not from the first one it was uploaded with."""
    import paper_2402_12947_b200 as P
    from oracle import oracle as O
    from paper_2402_12947_b200.sparse import CsrMatrix
    z, h = fixtures.load("c1s")
    lv = h.levels[0]
    a2 = CsrMatrix(lv.a.nrows, lv.a.ncols, lv.a.row_offsets, lv.a.col_indices, 2.0 * lv.a.values)
    b, ur = z["g/b"], z["g/u_rand"]
    for a in (lv.a, a2, lv.a):
        u = ur.copy()
        P.combined_smooth(a, b, u, lv.local_correction, lv.smoother)
        ref = O.combined_smooth(a, b, ur.copy(), lv.local_correction, lv.smoother)
        assert rel(u, ref) <= TOL_DENSE
