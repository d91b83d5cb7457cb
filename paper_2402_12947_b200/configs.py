"""BASELINE.json workload constructions C1-C5 (seeded synthetic inputs).

The paper's meshes are unpublished, so BASELINE.json's configs
are built here from the reference's primitives (structured simplex grids,
vertex displacement, region detection) -- SURVEY.md finding 10 / section
8(d).  Every random choice is seeded; nothing is read from disk.

Constructions (h = 1/n on a level with n cells per edge):

* jitter: every interior vertex moves by U(-a h, a h)^dim, rng = default_rng([seed, level]);
* collapse (2D, C1/C2): a vertex moves along an edge to within ``1e-3 h`` of
  its neighbour (needle triangles, aspect ~1e3);
* flatten (3D, C3/C4): a vertex moves toward the centroid of the opposite
  facet of an incident tet until 1e-3 of its height remains (dihedral < 1 deg);
* clusters are placed at seeded centres (default_rng([seed, 7])) on the
  FINE level only; BASELINE builds every coarse mesh "independently at 2x
  spacing with its own seeded jitter".  (Collapsing an edge on a coarse
  level would leave its P2 midpoint basis function with no fine node in its
  support, a zero column of P and a singular Galerkin operator.)
* vertices of one cluster are the closest to the centre that are pairwise
  non-adjacent (the reference's own rule, experiments.py:175-216);
* regions: cells with radius ratio < 0.1, extended by ``region_layers``
  vertex layers (C2: 2 layers per BASELINE), merged when they share a vertex.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

from .mesh import SimplexMesh, generate_simplex_grid, signed_volumes
from .smoothers import SmootherConfig


@dataclass(frozen=True)
class Workload:
    name: str
    dim: int
    degree: int
    grids: Tuple[int, ...]
    jitter: float
    perturb: Optional[str]           # "collapse" | "flatten" | None
    n_clusters: int
    vertices_per_cluster: int
    smoother: SmootherConfig
    rhs: str                         # "source-one" | "random"
    region_layers: int = 1
    seed: int = 0
    squash: float = 1e-3

    def scaled(self, factor: int) -> "Workload":
        """Same construction with every grid divided by ``factor`` (test sizes)."""
        grids = tuple(max(2, g // factor) for g in self.grids)
        ncl = max(1, int(round(self.n_clusters / factor ** self.dim))) if self.n_clusters else 0
        return Workload(self.name + f"/{factor}", self.dim, self.degree, grids, self.jitter,
                        self.perturb, ncl, self.vertices_per_cluster, self.smoother,
                        self.rhs, self.region_layers, self.seed, self.squash)


def _cheb(k):
    return SmootherConfig("chebyshev", sweeps=k)


def _jac(k, omega=2.0 / 3.0):
    return SmootherConfig("jacobi", sweeps=k, omega=omega)


C1 = Workload("C1-2d-p1-jacobi", 2, 1, (128, 64, 32, 16), 0.2, "collapse", 1, 3, _jac(2),
              "source-one", 1)
C2 = Workload("C2-2d-p2-cheb3", 2, 2, (512, 256, 128, 64, 32), 0.2, "collapse", 20, 1, _cheb(3),
              "random", 2)
C3 = Workload("C3-3d-p1-jacobi", 3, 1, (64, 32, 16, 8), 0.15, "flatten", 8, 1, _jac(2),
              "random", 1)
C4 = Workload("C4-3d-p2-cheb2", 3, 2, (96, 48, 24, 12), 0.15, "flatten", 50, 1, _cheb(2),
              "random", 1)
WORKLOADS = {"C1": C1, "C2": C2, "C3": C3, "C4": C4}

DESCRIPTIONS = {
    "C1": "BASELINE configs[0] (2D Poisson P1, 129x129 vertex grid, jitter 0.2h, one cluster of "
          "3 nodes moved within 1e-3h of a neighbour, f=1, damped Jacobi omega=2/3 x2, "
          "4-level non-nested Galerkin hierarchy)",
    "C2": "BASELINE configs[1] (2D Poisson P2, 513x513 vertex grid, jitter 0.2h, 20 "
          "collapsed-node clusters, 2-layer patches, Chebyshev degree 3, random N(0,1) RHS, "
          "5-level non-nested Galerkin hierarchy)",
    "C3": "BASELINE configs[2] (3D Poisson P1, 65^3 vertex grid, jitter 0.15h, 8 flattened "
          "tets, damped Jacobi omega=2/3 x2, 4-level non-nested Galerkin hierarchy)",
    "C4": "BASELINE configs[3] (3D Poisson P2, 97^3 vertex grid (7.2M DOFs), jitter 0.15h, 50 "
          "flattened-tet patches, Chebyshev degree 2, random N(0,1) RHS, 4 levels)",
}


def _interior_mask(mesh: SimplexMesh) -> np.ndarray:
    return ~mesh.boundary_vertex_mask()


def jitter(mesh: SimplexMesh, amplitude: float, rng: np.random.Generator) -> SimplexMesh:
    n = round(1.0 / (mesh.vertices[1, 0] - mesh.vertices[0, 0]))
    h = 1.0 / n
    interior = np.nonzero(_interior_mask(mesh))[0]
    verts = np.array(mesh.vertices)
    verts[interior] += rng.uniform(-amplitude * h, amplitude * h, size=(len(interior), mesh.dim))
    return mesh.with_vertices(verts)


def _cells_ok(verts, cells) -> bool:
    return bool(np.all(signed_volumes(verts, cells) > 0.0))


def perturb_clusters(mesh: SimplexMesh, wl: Workload, centers: np.ndarray,
                     rng: np.random.Generator) -> SimplexMesh:
    """Apply ``wl.perturb`` at each centre (vertex choice as experiments.py:175-216)."""
    if wl.perturb is None or wl.n_clusters == 0:
        return mesh
    n = round(1.0 / (mesh.vertices[1, 0] - mesh.vertices[0, 0]))
    h = 1.0 / n
    verts = np.array(mesh.vertices)
    interior = np.nonzero(_interior_mask(mesh))[0]
    inc = mesh.vertex_cell_incidence()
    blocked = np.zeros(mesh.n_vertices, dtype=bool)
    for center in centers:
        d = np.linalg.norm(mesh.vertices[interior] - center, axis=1)
        order = interior[np.lexsort((interior, d))]
        taken = 0
        for v in order[:64]:
            if taken == wl.vertices_per_cluster:
                break
            if blocked[v]:
                continue
            cells = inc[v].indices
            star = np.unique(mesh.cells[cells])
            if wl.perturb == "collapse":
                nbrs = star[star != v]
                nbrs = nbrs[np.argsort(np.linalg.norm(verts[nbrs] - verts[v], axis=1), kind="stable")]
                moved = False
                for w in nbrs:
                    direction = verts[v] - verts[w]
                    cand = verts[w] + wl.squash * h * direction / np.linalg.norm(direction)
                    old = verts[v].copy()
                    verts[v] = cand
                    if _cells_ok(verts, mesh.cells[cells]):
                        moved = True
                        break
                    verts[v] = old
            else:  # flatten toward the opposite facet of an incident tet
                moved = False
                for c in cells:
                    facet = [u for u in mesh.cells[c] if u != v]
                    centroid = verts[facet].mean(axis=0)
                    old = verts[v].copy()
                    verts[v] = old + (centroid - old) * (1.0 - wl.squash)
                    if _cells_ok(verts, mesh.cells[cells]):
                        moved = True
                        break
                    verts[v] = old
            if moved:
                taken += 1
                blocked[star] = True
    return mesh.with_vertices(verts)


def cluster_centers(wl: Workload) -> np.ndarray:
    rng = np.random.default_rng([wl.seed, 7])
    pts = []
    tries = 0
    min_sep = 0.5 / max(1.0, wl.n_clusters ** (1.0 / wl.dim))
    while len(pts) < wl.n_clusters and tries < 100000:
        tries += 1
        c = rng.uniform(0.1, 0.9, size=wl.dim)
        if all(np.linalg.norm(c - p) >= min_sep for p in pts):
            pts.append(c)
    return np.asarray(pts).reshape(-1, wl.dim)


def build_meshes(wl: Workload) -> List[SimplexMesh]:
    centers = cluster_centers(wl)
    meshes = []
    for level, n in enumerate(wl.grids):
        mesh = generate_simplex_grid(wl.dim, n)
        mesh = jitter(mesh, wl.jitter, np.random.default_rng([wl.seed, level]))
        if level == 0:
            mesh = perturb_clusters(mesh, wl, centers, np.random.default_rng([wl.seed, 1000]))
        meshes.append(mesh)
    return meshes


def problem_spec(wl: Workload):
    """Poisson, homogeneous Dirichlet on every box face (fem.py:230-262);
    f = 1 for the source-one workloads (vectorised), else no source (the
    random right-hand side is drawn directly)."""
    from .mg import ProblemSpec
    zero = lambda x: 0.0
    source = (lambda x: np.ones(len(x))) if wl.rhs == "source-one" else None
    return ProblemSpec("poisson", source=source,
                       dirichlet=tuple((m, zero) for m in range(1, 2 * wl.dim + 1)),
                       vectorized_source=True)


def build(wl: Workload, use_local_correction: bool = True, coarse_refine: bool = False,
          device_setup=None, device_assembly=None):
    """Host hierarchy + (b, u0) for a workload.  Returns (hierarchy, b, u0).
    ``device_setup``: see mg.build_hierarchy (None = GPU setup when a device
    exists; False = the host path).  Either way the hierarchy is the
    reference's construction bit for bit unless ``device_assembly="kernel"``."""
    from .mg import build_hierarchy
    meshes = build_meshes(wl)
    h = build_hierarchy(meshes, problem_spec(wl), wl.smoother, use_local_correction, 0.1,
                        wl.degree, region_layers=wl.region_layers, coarse_refine=coarse_refine,
                        device_setup=device_setup, device_assembly=device_assembly)
    n0 = h.fine.a.nrows
    if wl.rhs == "random":
        b = np.random.default_rng([wl.seed, 99]).standard_normal(n0)
        b[h.system.dirichlet_dofs] = 0.0
    else:
        b = np.array(h.system.b)
    u0 = np.zeros(n0)
    return h, b, u0
