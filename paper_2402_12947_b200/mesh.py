"""Simplicial meshes for hierarchy setup (host side, vectorised numpy).

Setup is not the GPU hot path (SURVEY.md section 2 marks it out of scope), but
the bench and the full-size parity tests must build BASELINE-sized
hierarchies on a box where the reference is absent, and the reference's own
mesh routines are per-cell Python loops (mesh.py:62, :155-179, :199-201) that
take minutes at 1M DOFs.  This module restates them with array operations and
the same numbering, so meshes built here equal the reference's vertex for
vertex and cell for cell:

* ``generate_simplex_grid``   mesh.py:136-184 (vertex ids ``j*side+i`` in 2D,
  ``(k*side+j)*side+i`` in 3D; 2 triangles / 6 Kuhn tets per box in the
  same order and orientation);
* ``boundary facets/markers`` mesh.py:198-223;
* ``radius_ratios``           mesh.py:256-297 (same formula);
* ``identify_regions``        mesh.py:326-378 (vertex-adjacency clusters,
  one-layer vertex extension, merge of regions sharing a vertex), with an
  extra ``layers`` knob for BASELINE's "patch = cells within 2 layers".

The BASELINE perturbations (uniform jitter, node collapses, flattened tets)
are harness constructions, not reference features (SURVEY.md finding 10);
they live in :mod:`paper_2402_12947_b200.configs`.
"""

from __future__ import annotations

import itertools
import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np
import scipy.sparse as sp
from scipy.sparse.csgraph import connected_components


class DegenerateCellError(ValueError):
    """A cell has non-positive volume (mesh.py:22-23)."""


@dataclass(frozen=True)
class SimplexMesh:
    """Simplicial mesh: ``cells`` positively oriented, marked boundary facets."""

    dim: int
    vertices: np.ndarray
    cells: np.ndarray
    boundary_facets: np.ndarray
    facet_markers: np.ndarray

    @property
    def n_vertices(self) -> int:
        return len(self.vertices)

    @property
    def n_cells(self) -> int:
        return len(self.cells)

    def boundary_vertex_mask(self) -> np.ndarray:
        m = np.zeros(self.n_vertices, dtype=bool)
        m[np.unique(self.boundary_facets)] = True
        return m

    def vertex_cell_incidence(self) -> sp.csr_matrix:
        """(n_vertices x n_cells) 0/1 incidence; row v lists the cells of v sorted."""
        nc, k = self.cells.shape
        rows = self.cells.ravel()
        cols = np.repeat(np.arange(nc, dtype=np.int64), k)
        return sp.csr_matrix((np.ones(len(rows), dtype=np.int8), (rows, cols)),
                             shape=(self.n_vertices, nc))

    def with_vertices(self, vertices: np.ndarray, check: bool = True) -> "SimplexMesh":
        m = SimplexMesh(self.dim, np.asarray(vertices, dtype=np.float64), self.cells,
                        self.boundary_facets, self.facet_markers)
        if check:
            vols = signed_volumes(m.vertices, m.cells)
            bad = np.nonzero(vols <= 0.0)[0]
            if len(bad):
                raise DegenerateCellError(
                    f"{len(bad)} cell(s) with non-positive volume, first is cell {bad[0]}")
        return m


def signed_volumes(vertices: np.ndarray, cells: np.ndarray) -> np.ndarray:
    """mesh.py:125-129."""
    v = vertices[cells]
    edges = v[:, 1:, :] - v[:, :1, :]
    dim = vertices.shape[1]
    return np.linalg.det(edges) / math.factorial(dim)


def _permutation_sign(perm: Sequence[int]) -> int:
    sign, p = 1, list(perm)
    for i in range(len(p)):
        while p[i] != i:
            j = p[i]
            p[i], p[j] = p[j], p[i]
            sign = -sign
    return sign


def generate_simplex_grid(dim: int, n: int) -> SimplexMesh:
    """Structured triangulation of the unit square / cube (mesh.py:136-184)."""
    if dim not in (2, 3):
        raise ValueError(f"dim must be 2 or 3, got {dim}")
    if n < 1:
        raise ValueError(f"cells-per-edge must be at least 1, got {n}")
    side = n + 1
    if dim == 2:
        axis = np.linspace(0.0, 1.0, side)
        xx, yy = np.meshgrid(axis, axis, indexing="ij")
        vertices = np.column_stack([xx.ravel(order="F"), yy.ravel(order="F")])
        j, i = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
        i, j = i.ravel(), j.ravel()
        a = j * side + i
        b = a + 1
        c = a + side + 1
        d = a + side
        cells = np.empty((2 * n * n, 3), dtype=np.int64)
        cells[0::2] = np.column_stack([a, b, c])
        cells[1::2] = np.column_stack([a, c, d])
    else:
        kk, jj, ii = np.meshgrid(np.arange(side), np.arange(side), np.arange(side),
                                 indexing="ij")
        order = np.column_stack([ii.ravel(), jj.ravel(), kk.ravel()])
        vertices = order / n
        k, j, i = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
        base = np.column_stack([i.ravel(), j.ravel(), k.ravel()])
        steps = np.eye(3, dtype=np.int64)
        tets = []
        for perm in itertools.permutations(range(3)):
            path = [base]
            for ax in perm:
                path.append(path[-1] + steps[ax])
            vids = [(p[:, 2] * side + p[:, 1]) * side + p[:, 0] for p in path]
            if _permutation_sign(perm) < 0:
                vids[2], vids[3] = vids[3], vids[2]
            tets.append(np.column_stack(vids))
        cells = np.stack(tets, axis=1).reshape(-1, 4).astype(np.int64)
    vertices = np.asarray(vertices, dtype=np.float64)
    facets, markers = _box_boundary_facets(vertices, cells, dim)
    return SimplexMesh(dim, vertices, cells, facets, markers)


def _all_faces(cells: np.ndarray) -> np.ndarray:
    k = cells.shape[1]
    faces = [np.delete(cells, skip, axis=1) for skip in range(k)]
    return np.sort(np.concatenate(faces, axis=0), axis=1)


def _box_boundary_facets(vertices, cells, dim):
    """Faces of exactly one cell, marked by box face, lexicographically sorted
    (mesh.py:198-223)."""
    faces = _all_faces(cells)
    uniq, counts = np.unique(faces, axis=0, return_counts=True)
    facets = uniq[counts == 1]
    coords = vertices[facets]  # (f, dim, dim)
    markers = np.zeros(len(facets), dtype=np.int64)
    for axis in range(dim - 1, -1, -1):  # lowest axis wins, as in the reference loop
        hi = np.all(np.abs(coords[:, :, axis] - 1.0) < 1e-12, axis=1)
        lo = np.all(np.abs(coords[:, :, axis]) < 1e-12, axis=1)
        markers[hi] = 2 * axis + 2
        markers[lo] = 2 * axis + 1
    if np.any(markers == 0):
        raise RuntimeError("boundary facet not on a box face")
    return facets.astype(np.int64), markers


def _facet_measures(v: np.ndarray, dim: int) -> np.ndarray:
    m = v.shape[0]
    measures = np.empty((m, dim + 1))
    for skip in range(dim + 1):
        keep = [j for j in range(dim + 1) if j != skip]
        pts = v[:, keep, :]
        if dim == 2:
            measures[:, skip] = np.linalg.norm(pts[:, 1] - pts[:, 0], axis=1)
        else:
            cross = np.cross(pts[:, 1] - pts[:, 0], pts[:, 2] - pts[:, 0])
            measures[:, skip] = 0.5 * np.linalg.norm(cross, axis=1)
    return measures


def radius_ratios(mesh: SimplexMesh, cells: Optional[np.ndarray] = None) -> np.ndarray:
    """Normalised inradius/circumradius ratio, 1 for the regular simplex
    (mesh.py:271-297)."""
    dim = mesh.dim
    cidx = mesh.cells if cells is None else mesh.cells[cells]
    v = mesh.vertices[cidx]
    edges = v[:, 1:, :] - v[:, :1, :]
    vols = np.linalg.det(edges) / math.factorial(dim)
    if np.any(vols <= 0.0):
        bad = int(np.nonzero(vols <= 0.0)[0][0])
        raise DegenerateCellError(f"cell {bad} has non-positive volume {vols[bad]:.3e}")
    r_in = dim * vols / _facet_measures(v, dim).sum(axis=1)
    rhs = np.einsum("mij,mij->mi", edges, edges)
    centers = np.linalg.solve(2.0 * edges, rhs[:, :, None])[:, :, 0]
    r_circ = np.linalg.norm(centers, axis=1)
    return dim * r_in / r_circ


@dataclass(frozen=True)
class RegionSet:
    """Low-quality cells and their disjoint extended regions (mesh.py:105-116).

    ``omega_B_regions`` holds sorted int64 cell arrays (the reference uses
    frozensets), ordered by smallest cell index as in mesh.py:377.
    """

    omega_b: np.ndarray
    omega_B_regions: Tuple[np.ndarray, ...]


def identify_regions(mesh: SimplexMesh, threshold: float = 0.1, layers: int = 1,
                     gammas: Optional[np.ndarray] = None) -> RegionSet:
    """mesh.py:326-378 restated with sparse connectivity; ``layers`` > 1 repeats
    the vertex extension (BASELINE's "cells within 2 layers")."""
    if not 0.0 < threshold < 1.0:
        raise ValueError(f"threshold must lie in (0, 1), got {threshold}")
    if layers < 1:
        raise ValueError("layers must be >= 1")
    g = radius_ratios(mesh) if gammas is None else gammas
    bad = np.nonzero(g < threshold)[0]
    if len(bad) == 0:
        return RegionSet(np.empty(0, dtype=np.int64), ())
    inc = mesh.vertex_cell_incidence()          # V x C
    inc_t = inc.T.tocsr()                         # C x V
    # clusters: bad cells sharing a vertex
    sub = inc_t[bad]
    adj = (sub @ sub.T).tocsr()
    ncl, lab = connected_components(adj, directed=False)
    # extension: cells sharing a vertex with the cluster, `layers` times
    extended = []
    for c in range(ncl):
        cells = bad[lab == c]
        for _ in range(layers):
            verts = np.unique(mesh.cells[cells])
            cells = np.unique(inc[verts].indices)
        extended.append(cells)
    # merge regions whose extensions share any vertex
    nreg = len(extended)
    rows = np.concatenate([np.full(len(np.unique(mesh.cells[e])), i) for i, e in enumerate(extended)])
    cols = np.concatenate([np.unique(mesh.cells[e]) for e in extended])
    rv = sp.csr_matrix((np.ones(len(rows), dtype=np.int8), (rows, cols)),
                       shape=(nreg, mesh.n_vertices))
    ncomp, lab2 = connected_components((rv @ rv.T).tocsr(), directed=False)
    merged = []
    for c in range(ncomp):
        merged.append(np.unique(np.concatenate([extended[i] for i in np.nonzero(lab2 == c)[0]])))
    merged.sort(key=lambda r: int(r[0]))
    return RegionSet(np.sort(bad).astype(np.int64), tuple(m.astype(np.int64) for m in merged))
