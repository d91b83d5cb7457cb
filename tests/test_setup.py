"""Host setup (vectorised mesh / FEM / transfer / regions) against the
reference-built hierarchies stored in tests/golden (c1s, c2s, c3s were
assembled, transferred and Galerkin-coarsened by the reference itself from
the same meshes).  Setup is not the hot path; these tests pin that the
bench's full-size hierarchies are the ones the reference would build."""

import numpy as np
import pytest

from paper_2402_12947_b200 import configs
from paper_2402_12947_b200.mesh import generate_simplex_grid, identify_regions, radius_ratios
from tests.golden import fixtures, refshim

CASES = ["c1s", "c2s", "c3s", "c4s"]


def _same_csr(m, ref):
    assert m.nrows == ref.nrows and m.ncols == ref.ncols
    assert np.array_equal(m.row_offsets, ref.row_offsets)
    assert np.array_equal(m.col_indices, ref.col_indices)
    return bool(np.array_equal(m.values, ref.values))


@pytest.mark.parametrize("name", CASES)
def test_own_setup_matches_reference_hierarchy(name):
    """Host setup == the reference's construction bit for bit: every A_l, P_l,
    region dof set, smoother lambda (Lanczos with the reference's (n, maxit)
    basis, sparse.py:280) and the right-hand side."""
    z, ref = fixtures.load(name)
    h, b, u0 = configs.build(fixtures.workload(name), device_setup=False)
    assert len(h.levels) == len(ref.levels)
    for lv, rl in zip(h.levels, ref.levels):
        assert _same_csr(lv.a, rl.a)
        if rl.prolongation is not None:
            assert _same_csr(lv.prolongation.matrix, rl.prolongation.matrix)
        if rl.smoother.lambda_min_fraction != 1.0:   # Chebyshev: lambda from setup
            assert lv.smoother.lambda_max == rl.smoother.lambda_max
        nref = 0 if rl.local_correction is None else len(rl.local_correction.regions)
        nown = 0 if lv.local_correction is None else len(lv.local_correction.regions)
        assert nref == nown
        for (i1, _), (i2, _) in zip(lv.local_correction.regions if nown else [],
                                    rl.local_correction.regions if nref else []):
            assert np.array_equal(i1, i2)
    assert np.array_equal(b, z["g/b"])


@pytest.mark.skipif(not refshim.available(), reason="reference not present")
@pytest.mark.parametrize("dim,n", [(2, 1), (2, 5), (3, 1), (3, 3)])
def test_grid_matches_reference(dim, n):
    sm = refshim.import_reference()
    r = sm.mesh.generate_simplex_grid(dim, n)
    m = generate_simplex_grid(dim, n)
    assert np.array_equal(m.vertices, r.vertices)
    assert np.array_equal(m.cells, r.cells)
    assert np.array_equal(m.boundary_facets, r.boundary_facets)
    assert np.array_equal(m.facet_markers, r.facet_markers)
    np.testing.assert_allclose(radius_ratios(m), sm.mesh.radius_ratios(r), rtol=1e-14)


@pytest.mark.skipif(not refshim.available(), reason="reference not present")
def test_regions_match_reference():
    sm = refshim.import_reference()
    wl = configs.C1.scaled(4)
    mesh = configs.build_meshes(wl)[0]
    rmesh = sm.mesh.SimplexMesh(mesh.dim, mesh.vertices, mesh.cells, mesh.boundary_facets,
                                mesh.facet_markers)
    ref = sm.mesh.identify_regions(rmesh, 0.1)
    own = identify_regions(mesh, 0.1)
    assert set(own.omega_b.tolist()) == set(ref.omega_b)
    assert [sorted(r.tolist()) for r in own.omega_B_regions] == [sorted(r) for r in ref.omega_B_regions]


def test_workload_shapes():
    """The full-size constructions have the BASELINE sizes (grid arithmetic only)."""
    assert (2 * configs.C2.grids[0] + 1) ** 2 == 1050625
    assert (configs.C1.grids[0] + 1) ** 2 == 16641
    assert (configs.C3.grids[0] + 1) ** 3 == 274625
    assert (2 * configs.C4.grids[0] + 1) ** 3 == 7189057


@pytest.mark.parametrize("n", [2, 3, 5])
def test_p2_tet_stencil_matches_assembly(n):
    """C5's structured generator equals fem.assemble_poisson on the same grid."""
    from paper_2402_12947_b200 import fem, stencil
    m = generate_simplex_grid(3, n)
    ref = fem.assemble_poisson(m, fem.build_dofmap(m, 2), None, dirichlet_all=True).a
    a = stencil.p2_tet_laplacian(n)
    assert np.array_equal(a.row_offsets, ref.row_offsets)
    assert np.array_equal(a.col_indices, ref.col_indices)
    assert np.max(np.abs(a.values - ref.values)) <= 1e-13 * np.max(np.abs(ref.values))


@pytest.mark.skipif(not refshim.available(), reason="reference not present")
@pytest.mark.parametrize("name,degree,theta", [("cpl_p1", 1, 1.5), ("cpl_p2", 2, None)])
def test_reference_signature_and_objects(name, degree, theta):
    """build_hierarchy(meshes, problem, smoother, use_local_correction,
    quality_threshold, element_degree) called positionally with the
    reference's own mesh / ProblemSpec / SmootherConfig objects (mg.py:72-75)
    rebuilds the reference-built fixture bit for bit."""
    from paper_2402_12947_b200.mg import build_hierarchy
    sm = refshim.import_reference()
    ex = sm.experiments
    z, ref = fixtures.load(name)
    meshes = []
    for lvl, n in enumerate(z["meta/grids"]):
        m = sm.mesh.generate_simplex_grid(2, int(n))
        if lvl == 0:
            cl = [ex.ClusterSpec(c, 1e-4, 1) for c in [(0.3125, 0.5), (0.5625, 0.5)]]
            m = ex._apply_clusters(m, cl, np.random.default_rng([5, lvl]))
        meshes.append(m)
    zero = lambda x: 0.0
    problem = sm.fem.ProblemSpec("poisson", source=lambda x: 1.0,
                                 dirichlet=tuple((m, zero) for m in range(1, 5)))
    h = build_hierarchy(meshes, problem, sm.smoothers.SmootherConfig("chebyshev", 2), True, 0.1,
                        degree, device_setup=False)
    for lv, rl in zip(h.levels, ref.levels):
        assert _same_csr(lv.a, rl.a)
        if theta is None:
            assert lv.smoother.lambda_max == rl.smoother.lambda_max
    assert np.array_equal(h.system.b, z["g/b"])
    regs = h.levels[0].local_correction.regions
    assert [r[0].tolist() for r in regs] == \
        [r[0].tolist() for r in ref.levels[0].local_correction.regions]


def test_build_hierarchy_rejects_old_argument_order():
    from paper_2402_12947_b200.mg import build_hierarchy
    wl = configs.C1.scaled(8)
    with pytest.raises(TypeError):
        build_hierarchy(configs.build_meshes(wl), wl.smoother, True)


@pytest.mark.skipif(not refshim.available(), reason="reference not present")
def test_locate_point_matches_reference():
    """locate_point (transfer.py:99-101): same cell (lowest index on ties) and
    barycentrics as the reference, including points on shared facets and
    vertices of a jittered mesh."""
    from paper_2402_12947_b200 import locate_point
    sm = refshim.import_reference()
    wl = configs.C1.scaled(16)
    mesh = configs.build_meshes(wl)[1]
    rmesh = sm.mesh.SimplexMesh(mesh.dim, mesh.vertices, mesh.cells, mesh.boundary_facets,
                                mesh.facet_markers)
    g = np.random.default_rng(2)
    pts = list(g.uniform(0, 1, size=(40, 2))) + list(mesh.vertices[::7])
    v = mesh.vertices[mesh.cells[3]]
    pts.append(0.5 * (v[0] + v[1]))          # on a shared edge
    for x in pts:
        c, bary = locate_point(mesh, x)
        rc, rbary = sm.transfer.locate_point(rmesh, x)
        assert c == rc
        assert np.array_equal(bary, rbary)
