"""P1/P2 Lagrange Poisson discretisation for hierarchy setup (host side).

Restates the reference's scalar-Poisson path (fem.py:29-60 bases,
:63-95 quadrature, :203-221 DOF map, :303-377 assembly with symmetric
Dirichlet elimination) with the same DOF numbering (vertices, then edge
midpoints in ``np.unique`` order of sorted vertex pairs) and the same einsum
expressions, so operators built here match the reference's.  Setup only;
the hot path consumes the resulting CSR operator.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional, Tuple

import numpy as np
import scipy.sparse as sp

from .mesh import SimplexMesh
from .sparse import CsrMatrix

_EDGES = {
    2: ((0, 1), (0, 2), (1, 2)),
    3: ((0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)),
}


def basis_values(degree: int, dim: int, lam: np.ndarray) -> np.ndarray:
    """Lagrange basis values at barycentric points ``lam`` (m, dim+1)
    (fem.py:43-60: vertices first, then edges in ``_EDGES`` order)."""
    if degree == 1:
        return lam.copy()
    vals = [lam * (2.0 * lam - 1.0)]
    vals += [(4.0 * lam[:, a] * lam[:, b])[:, None] for a, b in _EDGES[dim]]
    return np.hstack(vals)


def reference_gradients(degree: int, dim: int, point: np.ndarray) -> np.ndarray:
    """fem.py:47-60 gradients at one local point."""
    point = np.asarray(point, dtype=np.float64)
    lam = np.concatenate([[1.0 - point.sum()], point])
    grad_lam = np.vstack([-np.ones(dim), np.eye(dim)])
    if degree == 1:
        return grad_lam.copy()
    edges = _EDGES[dim]
    grads = np.empty((dim + 1 + len(edges), dim))
    grads[:dim + 1] = (4.0 * lam - 1.0)[:, None] * grad_lam
    for k, (a, b) in enumerate(edges):
        grads[dim + 1 + k] = 4.0 * (lam[a] * grad_lam[b] + lam[b] * grad_lam[a])
    return grads


def reference_values(degree: int, dim: int, point: np.ndarray) -> np.ndarray:
    point = np.asarray(point, dtype=np.float64)
    lam = np.concatenate([[1.0 - point.sum()], point])
    return basis_values(degree, dim, lam[None, :])[0]


def quadrature(dim: int, degree: int) -> Tuple[np.ndarray, np.ndarray]:
    """fem.py:63-95 (degrees 1, 2 and the 2D degree-4 rule)."""
    if dim == 2:
        if degree == 1:
            return np.array([[1 / 3, 1 / 3]]), np.array([0.5])
        if degree == 2:
            pts = np.array([[1 / 6, 1 / 6], [2 / 3, 1 / 6], [1 / 6, 2 / 3]])
            return pts, np.full(3, 1 / 6)
        groups = ((0.445948490915965, 0.223381589678011),
                  (0.091576213509771, 0.109951743655322))
        pts, wts = [], []
        for a, w in groups:
            b = 1.0 - 2.0 * a
            pts += [[a, a], [b, a], [a, b]]
            wts += [w, w, w]
        return np.asarray(pts), 0.5 * np.asarray(wts)
    if degree == 1:
        return np.array([[0.25, 0.25, 0.25]]), np.array([1 / 6])
    if degree == 2:
        a = (5.0 - np.sqrt(5.0)) / 20.0
        b = (5.0 + 3.0 * np.sqrt(5.0)) / 20.0
        pts = np.array([[a, a, a], [b, a, a], [a, b, a], [a, a, b]])
        return pts, np.full(4, 1 / 24)
    from scipy.special import roots_jacobi, roots_legendre
    n = 3
    xu, wu = roots_jacobi(n, 2.0, 0.0)
    xv, wv = roots_jacobi(n, 1.0, 0.0)
    xw, ww = roots_legendre(n)
    u, wu = (xu + 1.0) / 2.0, wu / 8.0
    v, wv = (xv + 1.0) / 2.0, wv / 4.0
    w, ww = (xw + 1.0) / 2.0, ww / 2.0
    pts, wts = [], []
    for i in range(n):
        for j in range(n):
            for k in range(n):
                pts.append([u[i], v[j] * (1.0 - u[i]), w[k] * (1.0 - u[i]) * (1.0 - v[j])])
                wts.append(wu[i] * wv[j] * ww[k])
    return np.asarray(pts), np.asarray(wts)


@dataclass(frozen=True)
class DofMap:
    """Scalar P1/P2 DOF map (fem.py:125-221; value_dims fixed to 1)."""

    mesh: SimplexMesh
    element_degree: int
    node_coords: np.ndarray
    cell_nodes: np.ndarray
    edges: Optional[np.ndarray]  # (n_edges, 2) sorted vertex pairs, P2 only

    value_dims: int = 1

    @property
    def n_nodes(self) -> int:
        return len(self.node_coords)

    @property
    def n_dofs(self) -> int:
        return self.n_nodes

    @property
    def cell_dofs(self) -> np.ndarray:
        return self.cell_nodes

    def boundary_dofs(self) -> np.ndarray:
        """DOFs on any boundary facet (all markers), sorted (fem.py:175-185)."""
        facets = self.mesh.boundary_facets
        nodes = [np.unique(facets)]
        if self.element_degree == 2:
            k = facets.shape[1]
            pairs = np.concatenate([np.sort(facets[:, [a, b]], axis=1)
                                    for a in range(k) for b in range(a + 1, k)])
            pairs = np.unique(pairs, axis=0)
            key_all = self.edges[:, 0] * self.mesh.n_vertices + self.edges[:, 1]
            key = pairs[:, 0] * self.mesh.n_vertices + pairs[:, 1]
            pos = np.searchsorted(key_all, key)
            nodes.append(self.mesh.n_vertices + pos)
        return np.unique(np.concatenate(nodes)).astype(np.int64)


def build_dofmap(mesh: SimplexMesh, degree: int) -> DofMap:
    """fem.py:203-221 (edge ids from np.unique over sorted pairs)."""
    if degree not in (1, 2):
        raise ValueError(f"element degree must be 1 or 2, got {degree}")
    if degree == 1:
        return DofMap(mesh, 1, np.array(mesh.vertices), np.array(mesh.cells), None)
    local_edges = np.asarray(_EDGES[mesh.dim])
    pairs = np.sort(mesh.cells[:, local_edges], axis=2).reshape(-1, 2)
    # np.unique(pairs, axis=0) order (lexicographic) via one int64 key per pair
    nv = np.int64(mesh.n_vertices)
    ukeys, inverse = np.unique(pairs[:, 0].astype(np.int64) * nv + pairs[:, 1],
                               return_inverse=True)
    unique = np.column_stack([ukeys // nv, ukeys % nv])
    edge_ids = inverse.reshape(mesh.n_cells, len(local_edges))
    midpoints = 0.5 * (mesh.vertices[unique[:, 0]] + mesh.vertices[unique[:, 1]])
    node_coords = np.vstack([mesh.vertices, midpoints])
    cell_nodes = np.hstack([mesh.cells, mesh.n_vertices + edge_ids])
    return DofMap(mesh, 2, node_coords, cell_nodes, unique.astype(np.int64))


def _load_vector(mesh, dofmap, source, v0, jac, det) -> np.ndarray:
    dim, degree = mesh.dim, dofmap.element_degree
    b = np.zeros(dofmap.n_dofs)
    qpts, qwts = quadrature(dim, 4)
    vals = np.asarray([reference_values(degree, dim, p) for p in qpts])
    coords = v0[:, None, :] + np.einsum("mde,qe->mqd", jac, qpts)
    fvals = np.asarray(source(coords.reshape(-1, dim)), dtype=np.float64).reshape(coords.shape[:2])
    b_local = np.einsum("q,m,qi,mq->mi", qwts, det, vals, fvals)
    np.add.at(b, dofmap.cell_dofs.ravel(), b_local.ravel())
    return b


def _assemble_poisson_device(mesh, dofmap, source, dirichlet_all, grads_ref, wts):
    import ctypes
    from . import _lib
    from . import device as _dev
    _dev.require_cuda()
    lib = _lib.load()
    i64p = ctypes.POINTER(ctypes.c_int64)
    f64p = ctypes.POINTER(ctypes.c_double)
    verts = np.ascontiguousarray(mesh.vertices, dtype=np.float64)
    cells = np.ascontiguousarray(mesh.cells, dtype=np.int64)
    cdofs = np.ascontiguousarray(dofmap.cell_dofs, dtype=np.int64)
    dir_dofs = dofmap.boundary_dofs() if dirichlet_all else np.empty(0, dtype=np.int64)
    dd = np.ascontiguousarray(dir_dofs, dtype=np.int64)
    g = np.ascontiguousarray(grads_ref, dtype=np.float64)
    w = np.ascontiguousarray(wts, dtype=np.float64)
    out = ctypes.c_void_p()
    bad = ctypes.c_int64(-1)
    rc = lib.smg_assemble_poisson(mesh.dim, int(dofmap.element_degree), len(verts),
                                  verts.ctypes.data_as(f64p), len(cells), cells.ctypes.data_as(i64p),
                                  cdofs.ctypes.data_as(i64p), int(dofmap.n_dofs),
                                  dd.ctypes.data_as(i64p), len(dd), g.ctypes.data_as(f64p),
                                  w.ctypes.data_as(f64p), len(w), ctypes.byref(out),
                                  ctypes.byref(bad), _dev.stream_handle())
    if rc != _lib.SMG_OK and bad.value >= 0:
        raise ValueError("mesh contains a degenerate or inverted cell")
    _lib.check(rc)
    nr, nc, ptr, col, val = _dev._csr_result_to_host(lib, out)
    a = CsrMatrix(nr, nc, ptr, col, val)
    if source is not None:
        v0, jac, det, _ = _cell_geometry(mesh)
        b = _load_vector(mesh, dofmap, source, v0, jac, det)
    else:
        b = np.zeros(dofmap.n_dofs)
    if len(dir_dofs):
        b[dir_dofs] = 0.0
    return AssembledSystem(a, b, dir_dofs)


@dataclass(frozen=True)
class AssembledSystem:
    a: CsrMatrix
    b: np.ndarray
    dirichlet_dofs: np.ndarray


def _cell_geometry(mesh: SimplexMesh):
    v = mesh.vertices[mesh.cells]
    jac = (v[:, 1:, :] - v[:, :1, :]).transpose(0, 2, 1)
    det = np.linalg.det(jac)
    if np.any(det <= 0.0):
        raise ValueError("mesh contains a degenerate or inverted cell")
    return v[:, 0, :], jac, det, np.linalg.inv(jac)


def _element_matrices(mesh: SimplexMesh, degree: int, grads_ref, wts):
    """The reference's element stiffness matrices, with its own arithmetic
    (fem.py:312-322: LAPACK det / inv via numpy, then two einsums)."""
    v0, jac, det, inv_jac = _cell_geometry(mesh)
    grads = np.einsum("qie,med->mqid", grads_ref, inv_jac)
    local = np.einsum("q,m,mqid,mqjd->mij", wts, det, grads, grads)
    return local, (v0, jac, det)


def _assemble_elements_device(mesh, dofmap, source, dirichlet_all, grads_ref, wts):
    """Element matrices on the host (the reference's arithmetic), then the
    COO -> CSR summation in scipy's exact duplicate order and the Dirichlet
    elimination on the GPU (``smg_assemble_elements``): bit-identical to the
    host path."""
    import ctypes
    from . import _lib
    from . import device as _dev
    _dev.require_cuda()
    lib = _lib.load()
    i64p = ctypes.POINTER(ctypes.c_int64)
    f64p = ctypes.POINTER(ctypes.c_double)
    local, (v0, jac, det) = _element_matrices(mesh, dofmap.element_degree, grads_ref, wts)
    local = np.ascontiguousarray(local, dtype=np.float64)
    cdofs = np.ascontiguousarray(dofmap.cell_dofs, dtype=np.int64)
    dir_dofs = dofmap.boundary_dofs() if dirichlet_all else np.empty(0, dtype=np.int64)
    dd = np.ascontiguousarray(dir_dofs, dtype=np.int64)
    out = ctypes.c_void_p()
    _lib.check(lib.smg_assemble_elements(int(dofmap.n_dofs), len(cdofs), int(cdofs.shape[1]),
                                         cdofs.ctypes.data_as(i64p), local.ctypes.data_as(f64p),
                                         dd.ctypes.data_as(i64p), len(dd), ctypes.byref(out),
                                         _dev.stream_handle()))
    nr, nc, ptr, col, val = _dev._csr_result_to_host(lib, out)
    a = CsrMatrix(nr, nc, ptr, col, val)
    b = np.zeros(dofmap.n_dofs)
    if source is not None:
        b = _load_vector(mesh, dofmap, source, v0, jac, det)
    if len(dir_dofs):
        # homogeneous data: the reference's b -= A u_bc (u_bc = 0) leaves b as
        # it is up to the sign of zeros, which -= 0.0 keeps (fem.py:362-366)
        b -= 0.0
        b[dir_dofs] = 0.0
    return AssembledSystem(a, b, dir_dofs)


def assemble_poisson(mesh: SimplexMesh, dofmap: DofMap,
                     source: Optional[Callable[[np.ndarray], np.ndarray]] = None,
                     dirichlet_all: bool = True, device=False) -> AssembledSystem:
    """Stiffness + load with homogeneous Dirichlet on every box face
    (fem.py:303-377).  ``source`` is vectorised: (m, dim) points -> (m,).

    ``device``: False = all on the host (numpy / scipy, the reference's own
    calls); True = element matrices on the host with the reference's
    arithmetic, the duplicate summation (scipy's order) and the Dirichlet
    elimination on the GPU (``smg_assemble_elements``) -- both bit-identical
    to the reference; ``"kernel"`` = element matrices too on the GPU
    (``smg_assemble_poisson``: cofactor geometry, values within ~1e-13, same
    pattern)."""
    dim = mesh.dim
    degree = dofmap.element_degree
    pts, wts = quadrature(dim, 1 if degree == 1 else 2)
    grads_ref = np.asarray([reference_gradients(degree, dim, p) for p in pts])
    if device == "kernel":
        return _assemble_poisson_device(mesh, dofmap, source, dirichlet_all, grads_ref, wts)
    if device:
        return _assemble_elements_device(mesh, dofmap, source, dirichlet_all, grads_ref, wts)
    local, (v0, jac, det) = _element_matrices(mesh, degree, grads_ref, wts)

    cell_dofs = dofmap.cell_dofs
    rows = np.repeat(cell_dofs, cell_dofs.shape[1], axis=1).ravel()
    cols = np.tile(cell_dofs, (1, cell_dofs.shape[1])).ravel()
    stiffness = sp.coo_matrix((local.ravel(), (rows, cols)),
                              shape=(dofmap.n_dofs, dofmap.n_dofs)).tocsr()
    stiffness.sum_duplicates()

    b = np.zeros(dofmap.n_dofs)
    if source is not None:
        qpts, qwts = quadrature(dim, 4)
        vals = np.asarray([reference_values(degree, dim, p) for p in qpts])
        coords = v0[:, None, :] + np.einsum("mde,qe->mqd", jac, qpts)
        fvals = np.asarray(source(coords.reshape(-1, dim)), dtype=np.float64).reshape(
            coords.shape[:2])
        b_local = np.einsum("q,m,qi,mq->mi", qwts, det, vals, fvals)
        np.add.at(b, cell_dofs.ravel(), b_local.ravel())

    dir_dofs = dofmap.boundary_dofs() if dirichlet_all else np.empty(0, dtype=np.int64)
    if len(dir_dofs):
        # homogeneous data: b -= A u_bc is a no-op up to signed zeros; keep the
        # reference's sequence so b rounds identically (fem.py:362-366)
        u_bc = np.zeros(dofmap.n_dofs)
        b -= stiffness @ u_bc
        b[dir_dofs] = 0.0
        mask = np.zeros(dofmap.n_dofs, dtype=bool)
        mask[dir_dofs] = True
        coo = stiffness.tocoo()
        keep = ~(mask[coo.row] | mask[coo.col])
        rows = np.concatenate([coo.row[keep], dir_dofs])
        cols = np.concatenate([coo.col[keep], dir_dofs])
        data = np.concatenate([coo.data[keep], np.ones(len(dir_dofs))])
        a = CsrMatrix.from_coo(dofmap.n_dofs, dofmap.n_dofs, rows, cols, data)
    else:
        a = CsrMatrix.from_scipy(stiffness)
    return AssembledSystem(a, b, dir_dofs)
