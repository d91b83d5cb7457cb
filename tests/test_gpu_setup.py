"""GPU prolongation construction (smg_prolongation_build) against the
reference's own prolongations and the host restatement.

Reference: transfer.py:117-150 build_prolongation with CellLocator.locate
(:36-91) -- lowest-index containing cell, clamped/renormalised barycentrics,
basis values with drop tolerance.
Bar: BITWISE (row offsets, columns, values).
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CASES = [("c1s", "C1", 4), ("c2s", "C2", 8), ("c3s", "C3", 4)]


def same(m, r) -> bool:
    return (m.shape == r.shape and np.array_equal(m.row_offsets, r.row_offsets)
            and np.array_equal(m.col_indices, r.col_indices) and np.array_equal(m.values, r.values))


@pytest.mark.parametrize("name,wl,scale", CASES)
def test_prolongation_bitwise_vs_reference(name, wl, scale):
    """Meshes rebuilt from the seeded construction the reference fixtures were
    made from; every device P equals the reference-built P bit for bit."""
    from paper_2402_12947_b200 import configs
    from paper_2402_12947_b200.fem import build_dofmap
    from paper_2402_12947_b200.transfer import build_prolongation
    from tests.golden import fixtures
    z, ref = fixtures.load(name)
    w = getattr(configs, wl).scaled(scale)
    meshes = configs.build_meshes(w)
    dms = [build_dofmap(m, w.degree) for m in meshes]
    for l in range(len(meshes) - 1):
        p = build_prolongation(dms[l], meshes[l + 1], dms[l + 1], device=True)
        assert same(p, ref.levels[l].prolongation.matrix), f"{name} level {l}"


@pytest.mark.parametrize("dim,degree", [(2, 1), (2, 2), (3, 1), (3, 2)])
def test_prolongation_ties_on_nested_grids(dim, degree):
    """Unjittered nested grids: fine nodes lie exactly on coarse facets and
    edges, so the lowest-index tie rule decides (device == host)."""
    from paper_2402_12947_b200.fem import build_dofmap
    from paper_2402_12947_b200.mesh import generate_simplex_grid
    from paper_2402_12947_b200.transfer import build_prolongation
    n = 8 if dim == 2 else 4
    fine, coarse = generate_simplex_grid(dim, 2 * n), generate_simplex_grid(dim, n)
    fd, cd = build_dofmap(fine, degree), build_dofmap(coarse, degree)
    p_dev = build_prolongation(fd, coarse, cd, device=True)
    p_host = build_prolongation(fd, coarse, cd, device=False)
    assert same(p_dev, p_host)
    # nested P1/P2 interpolation reproduces constants: rows sum to 1
    np.testing.assert_allclose(p_dev.to_scipy() @ np.ones(p_dev.ncols), 1.0, rtol=0, atol=1e-14)


def test_point_outside_raises_with_dof_index():
    from dataclasses import replace
    from paper_2402_12947_b200.fem import build_dofmap
    from paper_2402_12947_b200.mesh import generate_simplex_grid
    from paper_2402_12947_b200.transfer import PointLocationError, build_prolongation
    fine, coarse = generate_simplex_grid(2, 8), generate_simplex_grid(2, 4)
    shrunk = replace(coarse, vertices=coarse.vertices * 0.5)
    fd, cd = build_dofmap(fine, 1), build_dofmap(shrunk, 1)
    with pytest.raises(PointLocationError) as dev:
        build_prolongation(fd, shrunk, cd, device=True)
    with pytest.raises(PointLocationError) as host:
        build_prolongation(fd, shrunk, cd, device=False)
    assert dev.value.dof_index == host.value.dof_index


@pytest.mark.slow
@pytest.mark.parametrize("wl", ["C2", "C3"])
def test_prolongation_full_size_bitwise(wl):
    """Full BASELINE C2 / C3 meshes: device P == host restatement, every level."""
    from paper_2402_12947_b200 import configs
    from paper_2402_12947_b200.fem import build_dofmap
    from paper_2402_12947_b200.transfer import build_prolongation
    w = getattr(configs, wl)
    meshes = configs.build_meshes(w)
    dms = [build_dofmap(m, w.degree) for m in meshes]
    for l in range(len(meshes) - 1):
        p_dev = build_prolongation(dms[l], meshes[l + 1], dms[l + 1], device=True)
        p_host = build_prolongation(dms[l], meshes[l + 1], dms[l + 1], device=False)
        assert same(p_dev, p_host), f"level {l}"
