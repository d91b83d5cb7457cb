"""Non-nested intergrid transfer for hierarchy setup (host side, vectorised).

Restates ``pkg/src/simplexmg/transfer.py`` (relative to
/root/reference/pkg/src/simplexmg) without its per-DOF Python loop
(:132-144): point location returns, for every fine DOF coordinate, the
lowest-index coarse cell whose barycentric coordinates are all >= -1e-10
(the reference's tie rule, :81-91), clamps and renormalises them, and
evaluates the coarse P1/P2 basis there (:138-144, drop tolerance 1e-14).
Galerkin coarsening is ``P^T A P`` (:153-155).  Setup only; the hot path
consumes the resulting P (and its CSR transpose) on the device.
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from .fem import DofMap, basis_values
from .mesh import SimplexMesh
from .sparse import CsrMatrix, host_triple_product, triple_product


class PointLocationError(RuntimeError):
    """A point lies outside every cell beyond the barycentric tolerance (transfer.py:21-33)."""

    def __init__(self, point, dof_index=None):
        where = f" (while interpolating dof {dof_index})" if dof_index is not None else ""
        super().__init__(f"point {np.asarray(point)} lies outside the mesh{where}")
        self.point = np.asarray(point)
        self.dof_index = dof_index


class CellLocator:
    """Uniform-bin cell index; ``locate`` is vectorised over many points."""

    def __init__(self, mesh: SimplexMesh, tol: float = 1e-10):
        self.mesh = mesh
        self.tol = tol
        v = mesh.vertices[mesh.cells]
        self._v0 = v[:, 0, :]
        edges = (v[:, 1:, :] - v[:, :1, :]).transpose(0, 2, 1)
        self._inv_jac = np.linalg.inv(edges)
        self._lo = mesh.vertices.min(axis=0)
        self._hi = mesh.vertices.max(axis=0)
        span = np.maximum(self._hi - self._lo, 1e-300)
        dim = mesh.dim
        self._nb = max(1, int(round((mesh.n_cells / (2.0 if dim == 2 else 6.0)) ** (1.0 / dim))))
        self._scale = self._nb / span
        pad = 1e-9 * span.max()
        lo_b = np.clip(((v.min(axis=1) - pad - self._lo) * self._scale).astype(np.int64), 0, self._nb - 1)
        hi_b = np.clip(((v.max(axis=1) + pad - self._lo) * self._scale).astype(np.int64), 0, self._nb - 1)
        ext = hi_b - lo_b + 1
        counts = np.prod(ext, axis=1)
        cell_ids = np.repeat(np.arange(mesh.n_cells, dtype=np.int64), counts)
        offs = np.arange(len(cell_ids)) - np.repeat(np.cumsum(counts) - counts, counts)
        keys = np.zeros(len(cell_ids), dtype=np.int64)
        rem = offs.copy()
        stride = 1
        e_rep = ext[cell_ids]
        l_rep = lo_b[cell_ids]
        for d in range(dim):
            idx_d = rem % e_rep[:, d]
            rem //= e_rep[:, d]
            keys += (l_rep[:, d] + idx_d) * stride
            stride *= self._nb
        order = np.lexsort((cell_ids, keys))
        keys, cell_ids = keys[order], cell_ids[order]
        self._bin_ptr = np.searchsorted(keys, np.arange(self._nb ** dim + 1))
        self._bin_cells = cell_ids

    def _bin_key(self, x: np.ndarray) -> np.ndarray:
        q = np.clip(x, self._lo, self._hi)
        b = np.clip(((q - self._lo) * self._scale).astype(np.int64), 0, self._nb - 1)
        key = np.zeros(len(x), dtype=np.int64)
        stride = 1
        for d in range(self.mesh.dim):
            key += b[:, d] * stride
            stride *= self._nb
        return key

    def _bary(self, cells: np.ndarray, x: np.ndarray) -> np.ndarray:
        local = np.einsum("med,md->me", self._inv_jac[cells], x - self._v0[cells])
        return np.column_stack([1.0 - local.sum(axis=1), local])

    def locate(self, x: np.ndarray, chunk: int = 1 << 20):
        """(cells, clamped barycentrics) for points x (m, dim)."""
        x = np.asarray(x, dtype=np.float64)
        m = len(x)
        out_cell = np.full(m, -1, dtype=np.int64)
        out_bary = np.zeros((m, self.mesh.dim + 1))
        keys = self._bin_key(x)
        starts = self._bin_ptr[keys]
        counts = self._bin_ptr[keys + 1] - starts
        for c0 in range(0, m, chunk):
            sl = slice(c0, min(m, c0 + chunk))
            cnt = counts[sl]
            pid = np.repeat(np.arange(sl.start, sl.stop), cnt)
            off = np.arange(len(pid)) - np.repeat(np.cumsum(cnt) - cnt, cnt)
            cand = self._bin_cells[np.repeat(starts[sl], cnt) + off]
            bary = self._bary(cand, x[pid])
            inside = bary.min(axis=1) >= -self.tol
            pid_in, cand_in, bary_in = pid[inside], cand[inside], bary[inside]
            # candidates are ascending per point: keep the first inside hit
            first = np.ones(len(pid_in), dtype=bool)
            first[1:] = pid_in[1:] != pid_in[:-1]
            out_cell[pid_in[first]] = cand_in[first]
            out_bary[pid_in[first]] = bary_in[first]
        miss = np.nonzero(out_cell < 0)[0]
        for i in miss:  # rare: fall back to a scan of every cell (transfer.py:81-82)
            bary = self._bary(np.arange(self.mesh.n_cells), np.repeat(x[i:i + 1], self.mesh.n_cells, 0))
            inside = np.nonzero(bary.min(axis=1) >= -self.tol)[0]
            if len(inside) == 0:
                raise PointLocationError(x[i], dof_index=int(i))
            out_cell[i] = inside[0]
            out_bary[i] = bary[inside[0]]
        clamped = np.clip(out_bary, 0.0, 1.0)
        return out_cell, clamped / clamped.sum(axis=1, keepdims=True)


def build_prolongation(fine: DofMap, coarse_mesh: SimplexMesh, coarse: DofMap,
                       drop_tol: float = 1e-14, device: bool = False) -> CsrMatrix:
    """Row i holds the coarse basis values at fine dof i (transfer.py:117-150).

    ``device=True``: point location and basis evaluation run on the GPU
    (``smg_prolongation_build``, one thread per fine DOF; bit-identical); the
    bin index and the inverse Jacobians are formed here exactly as the
    reference forms them.  ``device=False``: the vectorised host restatement."""
    if fine.element_degree != coarse.element_degree:
        raise ValueError("fine and coarse dof maps must have equal element degree")
    loc = CellLocator(coarse_mesh)
    if device:
        return _build_prolongation_device(fine, coarse_mesh, coarse, loc, drop_tol)
    cells, bary = loc.locate(fine.node_coords)
    point = bary[:, 1:]
    lam = np.column_stack([1.0 - point.sum(axis=1), point])
    values = basis_values(coarse.element_degree, coarse_mesh.dim, lam)
    nodes = coarse.cell_nodes[cells]
    keep = np.abs(values) > drop_tol
    rows = np.repeat(np.arange(fine.n_nodes, dtype=np.int64), values.shape[1])[keep.ravel()]
    m = sp.coo_matrix((values[keep], (rows, nodes[keep])),
                      shape=(fine.n_nodes, coarse.n_nodes)).tocsr()
    return CsrMatrix.from_scipy(m)


def _build_prolongation_device(fine, coarse_mesh, coarse, loc, drop_tol) -> CsrMatrix:
    import ctypes
    from . import _lib
    from . import device as _dev
    _dev.require_cuda()
    lib = _lib.load()
    dim = coarse_mesh.dim
    i64p = ctypes.POINTER(ctypes.c_int64)
    f64p = ctypes.POINTER(ctypes.c_double)

    def f64(a):
        return np.ascontiguousarray(a, dtype=np.float64)

    def i64(a):
        return np.ascontiguousarray(a, dtype=np.int64)

    pts, v0, inv = f64(fine.node_coords), f64(loc._v0), f64(loc._inv_jac)
    nodes = i64(coarse.cell_nodes)
    lo, hi, scale = f64(loc._lo), f64(loc._hi), f64(loc._scale)
    bptr, bcells = i64(loc._bin_ptr), i64(loc._bin_cells)
    out = ctypes.c_void_p()
    bad = ctypes.c_int64(-1)
    rc = lib.smg_prolongation_build(
        dim, int(coarse.element_degree), len(pts), pts.ctypes.data_as(f64p), len(v0),
        v0.ctypes.data_as(f64p), inv.ctypes.data_as(f64p), nodes.ctypes.data_as(i64p),
        int(coarse.n_nodes), int(loc._nb), lo.ctypes.data_as(f64p), hi.ctypes.data_as(f64p),
        scale.ctypes.data_as(f64p), bptr.ctypes.data_as(i64p), bcells.ctypes.data_as(i64p),
        float(loc.tol), float(drop_tol), ctypes.byref(out), ctypes.byref(bad),
        _dev.stream_handle())
    if rc == _lib.SMG_ERR_POINT_LOCATION:
        raise PointLocationError(pts[bad.value], dof_index=int(bad.value))
    _lib.check(rc)
    nr, nc, ptr, col, val = _dev._csr_result_to_host(lib, out)
    return CsrMatrix(nr, nc, ptr, col, val)


def coarsen_system(a_fine, p, device: bool = True) -> CsrMatrix:
    """Galerkin coarse operator (transfer.py:153-155): on the GPU by default
    (``smg_galerkin``, bit-identical); ``device=False`` is the host-only setup
    path (the reference's scipy product)."""
    m = getattr(p, "matrix", p)
    return triple_product(m, a_fine) if device else host_triple_product(m, a_fine)


def locate_point(mesh: SimplexMesh, x, tol: float = 1e-10):
    """One-shot point location (transfer.py:99-101): (cell index, clamped
    barycentric coordinates), lowest-index containing cell on ties."""
    pt = np.asarray(x, dtype=np.float64).reshape(1, mesh.dim)
    cells, bary = CellLocator(mesh, tol=tol).locate(pt)
    return int(cells[0]), bary[0]


def _prolongation_operator(p):
    from . import device as _dev
    m = getattr(p, "matrix", p)
    return m, _dev.device_operator(m, with_transpose=True)


def restrict_residual(p, r_fine):
    """``P^T r`` (transfer.py:158-162; the restriction inside vcycle, mg.py:142)
    on the GPU: stored CSR(P^T) rows summed in ascending fine order, bitwise
    equal to scipy's csc_matvec.  numpy in -> numpy out; CUDA tensor in ->
    CUDA tensor out."""
    from . import _lib, device as _dev
    m, op = _prolongation_operator(p)
    t = _dev.torch()
    is_tensor = isinstance(r_fine, t.Tensor)
    if tuple(np.shape(r_fine)) != (m.nrows,):
        raise ValueError(f"residual length {tuple(r_fine.shape)} does not match fine size "
                         f"{m.nrows}")
    rt, _ = _dev.as_device_vector(r_fine, m.nrows, "r_fine")
    out = t.empty(m.ncols, dtype=t.float64, device=rt.device)
    _lib.check(_lib.load().smg_spmv_transpose(op.handle, _dev.ptr(rt), _dev.ptr(out),
                                              _dev.stream_handle()))
    return out if is_tensor else out.cpu().numpy()


def prolong_add(p, u_coarse, u_fine):
    """``u_fine += P u_coarse`` in place (transfer.py:165-172; mg.py:149) on the
    GPU (row-sequential sums, bitwise equal to scipy's csr_matvec + add)."""
    from . import _lib, device as _dev
    m, op = _prolongation_operator(p)
    t = _dev.torch()
    if tuple(np.shape(u_coarse)) != (m.ncols,):
        raise ValueError(f"coarse vector length {tuple(u_coarse.shape)} does not match {m.ncols}")
    if tuple(np.shape(u_fine)) != (m.nrows,):
        raise ValueError(f"fine vector length {tuple(u_fine.shape)} does not match {m.nrows}")
    ct, _ = _dev.as_device_vector(u_coarse, m.ncols, "u_coarse")
    ft, host = _dev.as_device_vector(u_fine, m.nrows, "u_fine")
    _lib.check(_lib.load().smg_prolong_add(op.handle, _dev.ptr(ct), _dev.ptr(ft),
                                           _dev.stream_handle()))
    if host is not None and not isinstance(u_fine, t.Tensor):
        u_fine[...] = ft.cpu().numpy()
    return u_fine
